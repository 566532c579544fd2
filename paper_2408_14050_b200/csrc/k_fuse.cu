// k_fuse.cu -- pixel-wise median fusion of K disparity estimates
// (SURVEY §8(f) NEXT #3).  PAPER.md:238 (§4.2): the per-camera disparity maps
// "are fused to a single disparity map by pixel-wise median filtering";
// for even counts the arithmetic mean of the two middle values.
//
// fp32 recipe (Q22): odd K -> the middle order statistic; even
// K -> fl32(fl32(a + b) * 0.5) of the middle pair a <= b; a non-finite input
// at a pixel gives NaN there (the detector then rejects the frame, Q18).
//
// HBM-bound streaming kernel: 4K bytes read + 4 bytes written per pixel.
// Each thread takes 4 consecutive pixels: one 16-byte load per estimate
// plane, a compile-time odd-even transposition network on registers
// (min/max pairs; the order statistics of a multiset do not depend on the
// network), one 16-byte streaming store.  Grid-stride over the pixels.
#include <algorithm>

#include "occ_internal.h"

namespace occ {

namespace {

// compare-exchange: after it, a <= b (NaN-free inputs)
__device__ __forceinline__ void cex(float &a, float &b) {
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    a = lo;
    b = hi;
}

// The signed zero a stable sort (equal values keep input order, as the
// oracle's insertion sort) puts at sorted position idx, given that position
// holds a zero: the (idx - #negatives)-th zero of the pixel's inputs.  The
// min/max network orders the values but not -0 / +0 among themselves.
__device__ __noinline__ float stable_zero(const float *col, int64_t stride, int K, int idx) {
    int neg = 0;
    for (int k = 0; k < K; ++k) neg += __ldg(col + (int64_t)k * stride) < 0.0f ? 1 : 0;
    int want = idx - neg;
    for (int k = 0; k < K; ++k) {
        const float x = __ldg(col + (int64_t)k * stride);
        if (x == 0.0f && want-- == 0) return x;
    }
    return 0.0f;
}

template <int K>
__device__ __forceinline__ float median_of(float (&v)[K], bool bad, const float *col, int64_t stride) {
    // odd-even transposition sort: K rounds of disjoint neighbour exchanges
#pragma unroll
    for (int r = 0; r < K; ++r) {
#pragma unroll
        for (int i = (r & 1); i + 1 < K; i += 2) cex(v[i], v[i + 1]);
    }
    float m;
    if (K & 1) {
        m = v[K / 2];
        if (m == 0.0f) m = stable_zero(col, stride, K, K / 2);
    } else {
        float lo = v[K / 2 - 1], hi = v[K / 2];
        if (lo == 0.0f) lo = stable_zero(col, stride, K, K / 2 - 1);
        if (hi == 0.0f) hi = stable_zero(col, stride, K, K / 2);
        m = __fmul_rn(__fadd_rn(lo, hi), 0.5f);
    }
    return bad ? __int_as_float(0x7fc00000) : m;
}

template <int K>
__global__ void __launch_bounds__(256) k_fuse(const float *__restrict__ stack, int64_t n,
                                              float *__restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(stack) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    if (vec) {
        const int64_t n4 = n >> 2;
        const float4 *s4 = reinterpret_cast<const float4 *>(stack);
        float4 *o4 = reinterpret_cast<float4 *>(out);
        for (int64_t i = t0; i < n4; i += stride) {
            float a[K], b[K], c[K], d[K];
            bool ba = false, bb = false, bc = false, bd = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float4 q = __ldcs(s4 + (int64_t)k * n4 + i);
                a[k] = q.x; b[k] = q.y; c[k] = q.z; d[k] = q.w;
                ba |= !isfinite(q.x); bb |= !isfinite(q.y); bc |= !isfinite(q.z); bd |= !isfinite(q.w);
            }
            const float *col = stack + 4 * i;
            __stcs(o4 + i, make_float4(median_of<K>(a, ba, col, n), median_of<K>(b, bb, col + 1, n),
                                       median_of<K>(c, bc, col + 2, n), median_of<K>(d, bd, col + 3, n)));
        }
        return;
    }
    for (int64_t i = t0; i < n; i += stride) {
        float a[K];
        bool bad = false;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            a[k] = __ldg(stack + (int64_t)k * n + i);
            bad |= !isfinite(a[k]);
        }
        out[i] = median_of<K>(a, bad, stack + i, n);
    }
}

// K beyond the unrolled range: insertion sort in local memory (slow path)
__global__ void __launch_bounds__(128) k_fuse_generic(const float *__restrict__ stack, int32_t K, int64_t n,
                                                      float *__restrict__ out) {
    float v[kFuseMaxK];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        bool bad = false;
        for (int32_t k = 0; k < K; ++k) {
            const float x = __ldg(stack + (int64_t)k * n + p);
            bad |= !isfinite(x);
            int32_t j = k;
            while (j > 0 && v[j - 1] > x) { v[j] = v[j - 1]; --j; }
            v[j] = x;
        }
        float m = (K & 1) ? v[K / 2] : __fmul_rn(__fadd_rn(v[K / 2 - 1], v[K / 2]), 0.5f);
        out[p] = bad ? __int_as_float(0x7fc00000) : m;
    }
}

template <int K>
cudaError_t launch_k(const float *stack, int64_t n, float *out, int nsm, cudaStream_t s) {
    const int64_t work = (n + 3) / 4;
    int blocks = (int)std::min<int64_t>((work + 255) / 256, (int64_t)nsm * 8);
    if (blocks < 1) blocks = 1;
    k_fuse<K><<<blocks, 256, 0, s>>>(stack, n, out);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fuse_median(const float *stack, int32_t K, int64_t n, float *out, int nsm, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1>(stack, n, out, nsm, s);
        case 2: return launch_k<2>(stack, n, out, nsm, s);
        case 3: return launch_k<3>(stack, n, out, nsm, s);
        case 4: return launch_k<4>(stack, n, out, nsm, s);
        case 5: return launch_k<5>(stack, n, out, nsm, s);
        case 6: return launch_k<6>(stack, n, out, nsm, s);
        case 7: return launch_k<7>(stack, n, out, nsm, s);
        case 8: return launch_k<8>(stack, n, out, nsm, s);
        case 9: return launch_k<9>(stack, n, out, nsm, s);
        case 10: return launch_k<10>(stack, n, out, nsm, s);
        case 11: return launch_k<11>(stack, n, out, nsm, s);
        case 12: return launch_k<12>(stack, n, out, nsm, s);
        case 13: return launch_k<13>(stack, n, out, nsm, s);
        case 14: return launch_k<14>(stack, n, out, nsm, s);
        case 15: return launch_k<15>(stack, n, out, nsm, s);
        case 16: return launch_k<16>(stack, n, out, nsm, s);
        default: {
            const int blocks = (int)std::min<int64_t>((n + 127) / 128, (int64_t)nsm * 16);
            k_fuse_generic<<<blocks < 1 ? 1 : blocks, 128, 0, s>>>(stack, K, n, out);
            return cudaGetLastError();
        }
    }
}

}  // namespace occ
