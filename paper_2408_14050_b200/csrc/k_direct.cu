// k_direct.cu -- the DIRECT path: one thread per (pixel, view), evaluating
// the per-pixel form of Eqs. 1-6 ("Equivalent GPU form"):
//
//   M_b(p) = 1  <=>  exists q on line(p), q != p, with P_b(p, q) and a
//                    candidate c with max(k_p,k_q) - h <= k_c <= min(k_p,k_q) + h
//
// Straightforward and slow (O(h) per pixel-view); used for frames whose scan
// half-length exceeds the tiled kernel's halo, and as an on-device
// cross-check of the tiled kernel (OCC_PATH_DIRECT).  The magnitude test is
// the literal sqrt_rn form here (the tiled kernel uses the equivalent exact
// squared threshold), so agreement of the two paths also pins that rewrite.
#include <climits>

#include "occ_internal.h"

namespace occ {

// ----------------------------------------------------------------- Eq. 1-2
// Candidate code per pixel: bit 2f = candidate of family f's +b0 direction,
// bit 2f+1 = candidate of -b0.  PAPER.md:92-109.
__global__ void __launch_bounds__(256) k_cand(const float *__restrict__ D, int32_t H, int32_t W,
                                              const FamilyDesc *__restrict__ fams, int32_t nfam,
                                              Params p, uint32_t *__restrict__ cand) {
    const int64_t HW = (int64_t)H * W;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= HW) return;
    const int f = blockIdx.y;
    const float *Df = D + (int64_t)f * HW;
    const int x = (int)(i % W), y = (int)(i / W);
    const float c = Df[i];
    // Eq. 1, f = (-1, 1)^T forward difference, 0 on the last column / row
    const float ex = (x + 1 < W) ? __fsub_rn(Df[i + 1], c) : 0.0f;
    const float ey = (y + 1 < H) ? __fsub_rn(Df[i + W], c) : 0.0f;
    // PAPER.md:103 E = sqrt(E_x^2 + E_y^2), literal fp32
    const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
    const bool edge = __fsqrt_rn(e2) > p.t_edge;
    uint32_t code = 0;
    if (edge) {
        for (int k = 0; k < nfam; ++k) {
            // Eq. 2 |Theta - phi| < pi/2  <=>  b . (E_x, E_y) > 0 (exact in binary64)
            const double dot = __dadd_rn(__dmul_rn((double)fams[k].b0x, (double)ex),
                                         __dmul_rn((double)fams[k].b0y, (double)ey));
            code |= (uint32_t)(dot > 0.0) << (2 * k);
            code |= (uint32_t)(dot < 0.0) << (2 * k + 1);
        }
    }
    cand[(int64_t)f * HW + i] = code;
}

// Eq. 3 (S5): h = floor(min(cap, ceil(2 s R)) / 2), R = fl32(dmax - dmin)
__device__ __forceinline__ int32_t view_h(const FrameStats &fs, int32_t s, int32_t cap) {
    const float R = __fsub_rn(key_float(fs.maxkey), key_float(fs.minkey));
    double L = ceil(__dmul_rn(__dmul_rn(2.0, (double)s), (double)R));
    if (!(L <= (double)cap)) L = (double)cap;
    return ((int32_t)L) >> 1;
}

// Eq. 5 with the prose sign (S7): delta = fl32(vq - vp) > t_disp and
// |dk + s delta| < t_dist, exact (s*delta exact in binary64, bounds exact).
__device__ __forceinline__ bool pair_exact(float vq, float vp, int32_t dk, int32_t s,
                                           const Params &p) {
    const float delta = __fsub_rn(vq, vp);
    if (!(delta > p.t_disp)) return false;
    const double x = __dmul_rn((double)s, (double)delta);
    const double hi = __dsub_rn((double)p.t_dist, (double)dk);
    const double lo = __dsub_rn(-(double)p.t_dist, (double)dk);
    return (x > lo) && (x < hi);
}

struct LineWalker {
    const float *Df;
    const uint32_t *Cf;
    int32_t H, W, line, xmajor, num, den, sg;
    // pixel index of the line sample at u (u = sg * pos); -1 when outside
    __device__ __forceinline__ int64_t at(int32_t u) const {
        const int32_t ps = sg * u;
        int32_t xx, yy;
        if (xmajor) {
            xx = ps;
            if (xx < 0 || xx >= W) return -1;
            yy = line + floordiv(ps * num, den);
            if (yy < 0 || yy >= H) return -1;
        } else {
            yy = ps;
            if (yy < 0 || yy >= H) return -1;
            xx = line + floordiv(ps * num, den);
            if (xx < 0 || xx >= W) return -1;
        }
        return (int64_t)yy * W + xx;
    }
    __device__ __forceinline__ bool cand(int32_t u, int bit) const {
        const int64_t i = at(u);
        return i >= 0 && ((Cf[i] >> bit) & 1);
    }
};

// grid: (ceil(HW/256), nviews, batch)
__global__ void __launch_bounds__(256) k_direct(const float *__restrict__ D,
                                                const uint32_t *__restrict__ cand,
                                                int32_t H, int32_t W,
                                                const ViewDesc *__restrict__ views, int32_t nviews,
                                                const FrameStats *__restrict__ st, Params p,
                                                uint8_t *__restrict__ masks) {
    const int64_t HW = (int64_t)H * W;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= HW) return;
    const int v = blockIdx.y, f = blockIdx.z;
    uint8_t *out = masks + ((int64_t)f * nviews + v) * HW;
    const FrameStats fs = st[f];
    if (fs.nonfinite) { out[pix] = 0; return; }          // SPEC.md:76 reject
    const ViewDesc &vd = views[v];
    const int32_t s = vd.s;
    const int32_t h = view_h(fs, s, p.max_scan);
    if (h == 0) { out[pix] = 0; return; }
    const int32_t x = (int32_t)(pix % W), y = (int32_t)(pix / W);
    LineWalker lw;
    lw.Df = D + (int64_t)f * HW;
    lw.Cf = cand + (int64_t)f * HW;
    lw.H = H; lw.W = W; lw.xmajor = vd.xmajor; lw.num = vd.num; lw.den = vd.den; lw.sg = vd.sg;
    const int32_t pos = vd.xmajor ? x : y;
    lw.line = vd.xmajor ? y - floordiv(x * vd.num, vd.den) : x - floordiv(y * vd.num, vd.den);
    const int32_t up = vd.sg * pos;
    const int bit = vd.candbit;
    const float vp = lw.Df[pix];

    // U(p) = pc(u_p + h) + h: the farthest sample sharing a window with p
    int32_t U = INT_MIN;
    for (int32_t c = up + h; c >= up - h; --c)
        if (lw.cand(c, bit)) { U = c + h; break; }
    bool m = false;
    if (U != INT_MIN) {
        // partners behind p (dk = -d < 0): the pair shares c's window iff d <= U - u_p
        const int32_t dmax = min(U - up, 2 * h);
        for (int32_t d = 1; d <= dmax && !m; ++d) {
            const int64_t q = lw.at(up + d);
            if (q < 0) continue;
            m = pair_exact(lw.Df[q], vp, -d, s, p);
        }
    }
    // partners ahead of p (dk = +fo > 0); |fo + s delta| < t_dist with
    // delta > 0 needs fo < t_dist.  Window: a candidate in [u_p - h, u_p - fo + h].
    const int32_t fmax = min(2 * h, (int32_t)ceilf(p.t_dist) - 1);
    for (int32_t fo = 1; fo <= fmax && !m; ++fo) {
        const int64_t q = lw.at(up - fo);
        if (q < 0) continue;
        if (!pair_exact(lw.Df[q], vp, fo, s, p)) continue;
        for (int32_t c = up - h; c <= up - fo + h; ++c)
            if (lw.cand(c, bit)) { m = true; break; }
    }
    out[pix] = (uint8_t)m;
}

cudaError_t launch_cand(const float *D, int32_t H, int32_t W, int32_t batch,
                        const FamilyDesc *fams, int32_t nfam, const Params &p,
                        uint32_t *cand, cudaStream_t s) {
    const int64_t HW = (int64_t)H * W;
    dim3 grid((unsigned)((HW + 255) / 256), (unsigned)batch);
    k_cand<<<grid, 256, 0, s>>>(D, H, W, fams, nfam, p, cand);
    return cudaGetLastError();
}

cudaError_t launch_direct(const float *D, const uint32_t *cand, int32_t H, int32_t W,
                          int32_t batch, const ViewDesc *views, int32_t nviews,
                          const FrameStats *st, const Params &p, uint8_t *masks,
                          cudaStream_t s) {
    const int64_t HW = (int64_t)H * W;
    dim3 grid((unsigned)((HW + 255) / 256), (unsigned)nviews, (unsigned)batch);
    k_direct<<<grid, 256, 0, s>>>(D, cand, H, W, views, nviews, st, p, masks);
    return cudaGetLastError();
}

}  // namespace occ
