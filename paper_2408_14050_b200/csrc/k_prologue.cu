// k_prologue.cu -- K0 of the tiled path: one streaming pass over a chunk of
// frames computing
//   * the exact per-frame min / max / non-finite count (S1; PAPER.md:113-115,
//     Eq. 3 "minimum and maximum occurring disparity"), and
//   * a per-pixel candidate code: for every line family f, bit 2f = pixel is
//     a candidate of +b0_f, bit 2f+1 = candidate of -b0_f (Eqs. 1-2,
//     E > t_e and |Theta - phi| < pi/2).
// The edge test runs once per pixel here instead of once per family in K1.
// D is read once from HBM (16-byte loads); the row below is an L2 hit (the
// neighbouring block reads it at the same time); codes stay L2-resident for
// K1, which runs on the same chunk right after.
#include <algorithm>

#include "occ_internal.h"

namespace occ {

struct FamDirs {
    int32_t n;
    int32_t small;      // all components in {-2..2}: fp32 products are exact
    int32_t bx[kMaxFamilies], by[kMaxFamilies];
    float fbx[kMaxFamilies], fby[kMaxFamilies];
};

// NF > 0: compile-time family count (unrolled); NF = 0: fd.n at run time
template <typename CodeT, int NF>
__device__ __forceinline__ CodeT pixel_code(float c, float right, float below, bool has_r, bool has_b,
                                            const FamDirs &fd, float e2_thresh) {
    // Eq. 1 forward differences (0 on the last column / row), E^2 vs the exact
    // squared threshold of E > t_e (sqrt_rn is monotone)
    const float ex = has_r ? __fsub_rn(right, c) : 0.0f;
    const float ey = has_b ? __fsub_rn(below, c) : 0.0f;
    const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
    uint32_t code = 0;
    if (NF == -4) {
        // the 3x3 array's families (1,0), (0,1), (1,1), (1,-1): the same fp32
        // dot products as the generic loop below with the +-1 products folded
        // (1 * x = x, -1 * y = -y exactly); the 0 * E products are kept, so an
        // infinite E gives NaN and no candidate, as there.  Branch-free.
        auto sgn2 = [](float x) -> uint32_t { return (x > 0.0f ? 1u : 0u) | (x < 0.0f ? 2u : 0u); };
        code = sgn2(__fadd_rn(ex, __fmul_rn(0.0f, ey))) | (sgn2(__fadd_rn(__fmul_rn(0.0f, ex), ey)) << 2) |
               (sgn2(__fadd_rn(ex, ey)) << 4) | (sgn2(__fsub_rn(ex, ey)) << 6);
        return (CodeT)(e2 > e2_thresh ? code : 0u);
    }
    if (e2 > e2_thresh) {
        const int nf = NF > 0 ? NF : fd.n;
#pragma unroll
        for (int k = 0; k < (NF > 0 ? NF : kMaxFamilies); ++k) {
            if (k >= nf) break;
            // Eq. 2 <=> b0 . (E_x, E_y) > 0, exact sign: with |b0| components
            // in {0, 1, 2} both products are exact in fp32 and the sign of a
            // correctly rounded sum is the sign of the exact sum; otherwise binary64
            // (the fp32 products can overflow, e.g. 2 * 2e38 = inf where the
            // exact product is finite: then the binary64 dot decides)
            bool pos, neg;
            const float px = __fmul_rn(fd.fbx[k], ex), py = __fmul_rn(fd.fby[k], ey);
            if (fd.small && isfinite(px) && isfinite(py)) {
                const float dot = __fadd_rn(px, py);
                pos = dot > 0.0f; neg = dot < 0.0f;
            } else {
                const double dot = __dadd_rn(__dmul_rn((double)fd.bx[k], (double)ex),
                                             __dmul_rn((double)fd.by[k], (double)ey));
                pos = dot > 0.0; neg = dot < 0.0;
            }
            code |= (pos ? 1u : 0u) << (2 * k);
            code |= (neg ? 1u : 0u) << (2 * k + 1);
        }
    }
    return (CodeT)code;
}

// four consecutive codes in one vector store (dst is 4-code aligned)
__device__ __forceinline__ void store4(uint8_t *dst, uint8_t a, uint8_t b, uint8_t c, uint8_t d) {
    *reinterpret_cast<uint32_t *>(dst) = (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)c << 16) | ((uint32_t)d << 24);
}
__device__ __forceinline__ void store4(uint16_t *dst, uint16_t a, uint16_t b, uint16_t c, uint16_t d) {
    *reinterpret_cast<uint2 *>(dst) = make_uint2((uint32_t)a | ((uint32_t)b << 16), (uint32_t)c | ((uint32_t)d << 16));
}
__device__ __forceinline__ void store4(uint32_t *dst, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    *reinterpret_cast<uint4 *>(dst) = make_uint4(a, b, c, d);
}

__device__ __forceinline__ void stat_acc(float d, int32_t &lo, int32_t &hi, uint32_t &bad) {
    if (isfinite(d)) {
        const int32_t k = float_key(d);
        lo = min(lo, k);
        hi = max(hi, k);
    } else {
        ++bad;
    }
}

// grid: (blocks per frame, frames); block 256
template <typename CodeT, int NF>
__global__ void __launch_bounds__(256) k_prologue(const float *__restrict__ D, int32_t H, int32_t W,
                                                  FamDirs fd, float e2_thresh, FrameStats *st,
                                                  CodeT *__restrict__ codes, int32_t do_stats) {
    const int f = blockIdx.y;
    const int64_t HW = (int64_t)H * W;
    const float *Df = D + (int64_t)f * HW;
    CodeT *Cf = codes + (int64_t)f * HW;
    int32_t lo = 0x7FFFFFFF, hi = (int32_t)0x80000000;
    uint32_t bad = 0;
    if ((W & 3) == 0 && (reinterpret_cast<uintptr_t>(Df) & 15) == 0) {
        // rows are block-strided, float4 columns thread-strided (no 64-bit
        // index division per element)
        const float4 *D4 = reinterpret_cast<const float4 *>(Df);
        const int32_t W4 = W >> 2;
        for (int32_t y = blockIdx.x; y < H; y += gridDim.x)
        for (int32_t xq = threadIdx.x; xq < W4; xq += blockDim.x) {
            const int64_t t = (int64_t)y * W4 + xq;
            const int32_t x = xq * 4;
            const float4 c = __ldg(D4 + t);
            const bool has_b = y + 1 < H;
            const float4 b = has_b ? __ldg(D4 + t + W4) : make_float4(0.f, 0.f, 0.f, 0.f);
            const bool has_r4 = x + 4 < W;
            const float r4 = has_r4 ? __ldg(Df + (int64_t)y * W + x + 4) : 0.0f;
            stat_acc(c.x, lo, hi, bad);
            stat_acc(c.y, lo, hi, bad);
            stat_acc(c.z, lo, hi, bad);
            stat_acc(c.w, lo, hi, bad);
            CodeT k0 = pixel_code<CodeT, NF>(c.x, c.y, b.x, true, has_b, fd, e2_thresh);
            CodeT k1 = pixel_code<CodeT, NF>(c.y, c.z, b.y, true, has_b, fd, e2_thresh);
            CodeT k2 = pixel_code<CodeT, NF>(c.z, c.w, b.z, true, has_b, fd, e2_thresh);
            CodeT k3 = pixel_code<CodeT, NF>(c.w, r4, b.w, has_r4, has_b, fd, e2_thresh);
            store4(Cf + (int64_t)t * 4, k0, k1, k2, k3);
        }
    } else {
        const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const int64_t nth = (int64_t)gridDim.x * blockDim.x;
        for (int64_t i = tid; i < HW; i += nth) {
            const int32_t y = (int32_t)(i / W), x = (int32_t)(i - (int64_t)y * W);
            const float c = Df[i];
            stat_acc(c, lo, hi, bad);
            const bool has_r = x + 1 < W, has_b = y + 1 < H;
            Cf[i] = pixel_code<CodeT, NF>(c, has_r ? Df[i + 1] : 0.0f, has_b ? Df[i + W] : 0.0f, has_r,
                                      has_b, fd, e2_thresh);
        }
    }
    if (!do_stats) return;          // statistics already computed by k_words
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    // block reduction, then one set of atomics per block
    __shared__ int32_t r_lo[8], r_hi[8];
    __shared__ uint32_t r_bad[8];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { r_lo[w] = lo; r_hi[w] = hi; r_bad[w] = bad; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        lo = l < nw ? r_lo[l] : 0x7FFFFFFF;
        hi = l < nw ? r_hi[l] : (int32_t)0x80000000;
        bad = l < nw ? r_bad[l] : 0u;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            bad += __shfl_xor_sync(0xffffffffu, bad, o);
        }
        if (l == 0) {
            atomicMin(&st[f].minkey, lo);
            atomicMax(&st[f].maxkey, hi);
            if (bad) atomicAdd(&st[f].nonfinite, bad);
        }
    }
}

cudaError_t launch_prologue(const float *D, int32_t H, int32_t W, int32_t frames,
                            const FamilyDesc *fams_host, int32_t nfam, float e2_thresh,
                            FrameStats *st, void *codes, int32_t code_bytes, int32_t do_stats, cudaStream_t s) {
    FamDirs fd{};
    fd.n = nfam;
    fd.small = 1;
    for (int k = 0; k < nfam; ++k) {
        fd.bx[k] = fams_host[k].b0x; fd.by[k] = fams_host[k].b0y;
        fd.fbx[k] = (float)fd.bx[k]; fd.fby[k] = (float)fd.by[k];
        if (fd.bx[k] < -2 || fd.bx[k] > 2 || fd.by[k] < -2 || fd.by[k] > 2) fd.small = 0;
    }
    // vector path: blocks stride over rows (about 2 float4 per thread per row
    // at 1920 wide); scalar path: grid-stride over the pixels
    const int bx = std::max(1, std::min(H, 256));
    dim3 grid(bx, frames);
    const bool grid3 = nfam == 4 && fd.bx[0] == 1 && fd.by[0] == 0 && fd.bx[1] == 0 && fd.by[1] == 1 &&
                       fd.bx[2] == 1 && fd.by[2] == 1 && fd.bx[3] == 1 && fd.by[3] == -1;
    if (code_bytes == 1) {
        if (grid3) k_prologue<uint8_t, -4><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint8_t *)codes, do_stats);
        else if (nfam == 4) k_prologue<uint8_t, 4><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint8_t *)codes, do_stats);
        else if (nfam == 1) k_prologue<uint8_t, 1><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint8_t *)codes, do_stats);
        else k_prologue<uint8_t, 0><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint8_t *)codes, do_stats);
    } else if (code_bytes == 2) {
        if (nfam == 8) k_prologue<uint16_t, 8><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint16_t *)codes, do_stats);
        else k_prologue<uint16_t, 0><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint16_t *)codes, do_stats);
    } else {
        k_prologue<uint32_t, 0><<<grid, 256, 0, s>>>(D, H, W, fd, e2_thresh, st, (uint32_t *)codes, do_stats);
    }
    return cudaGetLastError();
}

}  // namespace occ
