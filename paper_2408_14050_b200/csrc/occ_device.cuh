// occ_device.cuh -- device helpers shared by libocc's kernels (k_tile.cu,
// k_direct.cu).  Every function restates one step of PAPER.md §3 under the
// readings of DESIGN.md §2; exact fp32 semantics (no FMA: -fmad=false, and
// explicit _rn intrinsics).
#pragma once
#include <climits>

#include "occ_internal.h"

namespace occ {

// Eq. 3 (S5): h = floor(min(cap, ceil(2 s R)) / 2), R = fl32(dmax - dmin).
__device__ __forceinline__ int32_t view_h(float R, int32_t s, int32_t cap) {
    double L = ceil(__dmul_rn(__dmul_rn(2.0, (double)s), (double)R));
    if (!(L <= (double)cap)) L = (double)cap;
    return ((int32_t)L) >> 1;
}

// Largest offset a partner can have: |dk| < t_dist + s R
// (delta <= R) and |dk| <= 2h.  R = inf (the frame's range overflowed fp32)
// gives 2h; the comparison runs in binary64 before any conversion to int.
__device__ __forceinline__ int32_t partner_reach(float t_dist, int32_t s, float R, int32_t h) {
    const double r = floor(__dadd_rn((double)t_dist, __dmul_rn((double)s, (double)R))) + 1.0;
    return r < (double)(2 * h) ? (int32_t)r : 2 * h;
}

__device__ __forceinline__ float frame_range(const FrameStats &fs) {
    return __fsub_rn(key_float(fs.maxkey), key_float(fs.minkey));
}

// Eq. 5 with the prose sign (S7): delta = fl32(vq - vp) > t_disp and
// |dk + s delta| < t_dist, exact: s*delta is exact in binary64 and the
// bounds +-t_dist - dk are exact for the validated parameter ranges.
__device__ __forceinline__ bool pair_exact(float vq, float vp, int32_t dk, int32_t s,
                                           float t_dist, float t_disp) {
    const float delta = __fsub_rn(vq, vp);
    if (!(delta > t_disp)) return false;
    const double x = __dmul_rn((double)s, (double)delta);
    const double hi = __dsub_rn((double)t_dist, (double)dk);
    const double lo = __dsub_rn(-(double)t_dist, (double)dk);
    return (x > lo) && (x < hi);
}

// Eqs. 1-2 at pixel (x, y) for the family base direction b0: returns bit 0
// when the pixel is a candidate of +b0, bit 1 when it is one of -b0.
//   Eq. 1: E_x = D[x+1,y] - D[x,y], E_y = D[x,y+1] - D[x,y] (0 at the border)
//   E > t_e: literal sqrt_rn(fl(fl(E_x^2) + fl(E_y^2))) > t_e when kLiteral,
//            else the equivalent e2 > e2_thresh (sqrt_rn is monotone)
//   |Theta - phi| < pi/2  <=>  b0 . (E_x, E_y) > 0, sign exact in binary64
template <bool kLiteral>
__device__ __forceinline__ uint32_t cand_dirs(const float *__restrict__ Df, int32_t H, int32_t W,
                                              int32_t x, int32_t y, int32_t b0x, int32_t b0y,
                                              float e2_thresh, float t_edge) {
    const int64_t i = (int64_t)y * W + x;
    const float c = __ldg(Df + i);
    const float ex = (x + 1 < W) ? __fsub_rn(__ldg(Df + i + 1), c) : 0.0f;
    const float ey = (y + 1 < H) ? __fsub_rn(__ldg(Df + i + W), c) : 0.0f;
    const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
    const bool edge = kLiteral ? (__fsqrt_rn(e2) > t_edge) : (e2 > e2_thresh);
    if (!edge) return 0u;
    const double dot = __dadd_rn(__dmul_rn((double)b0x, (double)ex), __dmul_rn((double)b0y, (double)ey));
    return (dot > 0.0 ? 1u : 0u) | (dot < 0.0 ? 2u : 0u);
}

// cand_dirs with the centre value already loaded (tiled kernel's staging);
// squared-threshold form of E > t_e.
__device__ __forceinline__ uint32_t cand_dirs_v(const float *__restrict__ Df, int32_t H, int32_t W,
                                                int32_t x, int32_t y, float c, int32_t b0x,
                                                int32_t b0y, float e2_thresh) {
    const int64_t i = (int64_t)y * W + x;
    const float ex = (x + 1 < W) ? __fsub_rn(__ldg(Df + i + 1), c) : 0.0f;
    const float ey = (y + 1 < H) ? __fsub_rn(__ldg(Df + i + W), c) : 0.0f;
    const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
    if (!(e2 > e2_thresh)) return 0u;
    const double dot = __dadd_rn(__dmul_rn((double)b0x, (double)ex), __dmul_rn((double)b0y, (double)ey));
    return (dot > 0.0 ? 1u : 0u) | (dot < 0.0 ? 2u : 0u);
}

// The digital epipolar line through a pixel (S6) and its samples by u.
struct LineGeom {
    int32_t H, W, line, xmajor, num, den, sg;
    __device__ __forceinline__ void init(const ViewDesc &vd, int32_t H_, int32_t W_, int32_t x, int32_t y) {
        H = H_; W = W_; xmajor = vd.xmajor; num = vd.num; den = vd.den; sg = vd.sg;
        line = xmajor ? y - floordiv(x * num, den) : x - floordiv(y * num, den);
    }
    // sample at u (u = sg * pos): fills x, y; false when outside the image
    __device__ __forceinline__ bool at(int32_t u, int32_t &xx, int32_t &yy) const {
        const int32_t ps = sg * u;
        if (xmajor) {
            xx = ps;
            if (xx < 0 || xx >= W) return false;
            yy = line + floordiv(ps * num, den);
            return yy >= 0 && yy < H;
        }
        yy = ps;
        if (yy < 0 || yy >= H) return false;
        xx = line + floordiv(ps * num, den);
        return xx >= 0 && xx < W;
    }
};

// Per-pixel form of Eqs. 1-6 for one view (derived in App. A.2):
// M(p) = 1 iff some q on p's line satisfies Eq. 5 and p, q share the scan
// window of one candidate.  O(h) per pixel; reads D directly (L1/L2).
template <bool kLiteral>
__device__ __forceinline__ bool direct_pixel(const float *__restrict__ Df, int32_t H, int32_t W,
                                             const ViewDesc &vd, const FamilyDesc &fd,
                                             const Params &p, int32_t h, int32_t x, int32_t y) {
    if (h <= 0) return false;
    LineGeom lg;
    lg.init(vd, H, W, x, y);
    const int32_t up = vd.sg * (vd.xmajor ? x : y);
    const uint32_t mybit = vd.sg > 0 ? 1u : 2u;
    const float vp = __ldg(Df + (int64_t)y * W + x);
    const int32_t s = vd.s;
    int32_t xx, yy;
    // U(p) = pc(u_p + h) + h  (largest candidate u <= u_p + h)
    int32_t U = INT_MIN;
    for (int32_t c = up + h; c >= up - h; --c) {
        if (!lg.at(c, xx, yy)) continue;
        if (cand_dirs<kLiteral>(Df, H, W, xx, yy, fd.b0x, fd.b0y, p.e2_thresh, p.t_edge) & mybit) { U = c + h; break; }
    }
    if (U != INT_MIN) {
        const int32_t dmax = min(U - up, 2 * h);
        for (int32_t d = 1; d <= dmax; ++d) {
            if (!lg.at(up + d, xx, yy)) continue;
            if (pair_exact(__ldg(Df + (int64_t)yy * W + xx), vp, -d, s, p.t_dist, p.t_disp)) return true;
        }
    }
    // forward partners (dk = +fo): need fo < t_dist; window: candidate in [u_p - h, u_p - fo + h]
    const int32_t fmax = min(2 * h, (int32_t)ceilf(p.t_dist) - 1);
    for (int32_t fo = 1; fo <= fmax; ++fo) {
        if (!lg.at(up - fo, xx, yy)) continue;
        if (!pair_exact(__ldg(Df + (int64_t)yy * W + xx), vp, fo, s, p.t_dist, p.t_disp)) continue;
        for (int32_t c = up - h; c <= up - fo + h; ++c) {
            int32_t cx, cy;
            if (!lg.at(c, cx, cy)) continue;
            if (cand_dirs<kLiteral>(Df, H, W, cx, cy, fd.b0x, fd.b0y, p.e2_thresh, p.t_edge) & mybit) return true;
        }
    }
    return false;
}

}  // namespace occ
