// k_stats.cu -- K0: per-frame exact min / max of D and non-finite count
// (Eq. 3 "minimum and maximum occurring
// disparity").  HBM-bound streaming reduction: 16-byte loads, warp-shuffle
// reductions, one atomic per warp on ordered-int keys (exact for fp32).
#include "occ_internal.h"

namespace occ {

__global__ void k_stats_init(FrameStats *st, int32_t batch) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < batch) {
        st[i].minkey = 0x7FFFFFFF;
        st[i].maxkey = (int32_t)0x80000000;
        st[i].nonfinite = 0u;
        st[i].pad = 0;
    }
}

__device__ __forceinline__ void acc(float d, int32_t &lo, int32_t &hi, uint32_t &bad) {
    if (isfinite(d)) {
        int32_t k = float_key(d);
        lo = min(lo, k);
        hi = max(hi, k);
    } else {
        ++bad;
    }
}

// grid: (blocks per frame, batch); block 256 threads
__global__ void __launch_bounds__(256) k_stats(const float *__restrict__ D, int64_t HW,
                                               FrameStats *st) {
    const int f = blockIdx.y;
    const float *Df = D + (int64_t)f * HW;
    int32_t lo = 0x7FFFFFFF, hi = (int32_t)0x80000000;
    uint32_t bad = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if ((HW & 3) == 0 && (reinterpret_cast<uintptr_t>(Df) & 15) == 0) {
        const float4 *D4 = reinterpret_cast<const float4 *>(Df);
        const int64_t n4 = HW >> 2;
        for (int64_t i = tid; i < n4; i += nth) {
            float4 q = __ldg(D4 + i);    // default policy: K1 re-reads D from L2
            acc(q.x, lo, hi, bad);
            acc(q.y, lo, hi, bad);
            acc(q.z, lo, hi, bad);
            acc(q.w, lo, hi, bad);
        }
    } else {
        for (int64_t i = tid; i < HW; i += nth) acc(Df[i], lo, hi, bad);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&st[f].minkey, lo);
        atomicMax(&st[f].maxkey, hi);
        if (bad) atomicAdd(&st[f].nonfinite, bad);
    }
}

cudaError_t launch_stats_init(FrameStats *st, int32_t batch, cudaStream_t s) {
    k_stats_init<<<(batch + 255) / 256, 256, 0, s>>>(st, batch);
    return cudaGetLastError();
}

cudaError_t launch_stats(const float *D, int64_t HW, int32_t batch, FrameStats *st,
                         cudaStream_t s) {
    int64_t per_block = 256 * 4 * 8;     // 8 float4 per thread
    int bx = (int)((HW + per_block - 1) / per_block);
    if (bx < 1) bx = 1;
    if (bx > 1024) bx = 1024;
    k_stats<<<dim3(bx, batch), 256, 0, s>>>(D, HW, st);
    return cudaGetLastError();
}

}  // namespace occ
