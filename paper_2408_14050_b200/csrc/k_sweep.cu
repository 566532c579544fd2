// k_sweep.cu -- the line-sweep hot path for the four line families of a
// |b| <= 2 grid array whose views share rows, columns, diagonals and
// anti-diagonals (§3, Eqs. 1-6):
//
//   k_words  (K0)  one pass over D: the exact per-frame min / max / non-finite
//                  count (Eq. 3) and the candidate bits of
//                  Eqs. 1-2 of all four families, written
//                  as 32-bit words in the layout the sweep reads (one word =
//                  one line x 32 positions), so the sweep never recomputes
//                  an edge test and needs no per-pixel code bytes.
//   k_sweep  (K1)  one warp = 32 consecutive lines x a segment of positions
//                  of one family, both views +-b of the family:
//                    pass 1 (ascending)  the far filter of view -b (running
//                      max of s v + pos over the partners behind) and the
//                      last candidates each window needs, parked per block;
//                    pass 2 (descending) Eq. 5's near tests of both views
//                      (shared differences), the far filter of view +b,
//                      window coverage (S8), the far survivors' witness
//                      probes, and the uint8 / packed stores of both views.
//                  Unconfirmed far survivors go to k_hard (k_line.cu).
//
// Geometry (digital lines; l0 a multiple of 32, lane l is
// line l0 + l, tau increases along the family's base direction b0):
//   kind 0 rows      b0 = ( 1, 0): pixel (tau, l0 + l)
//   kind 1 columns   b0 = ( 0, 1): pixel (l0 + l, tau)
//   kind 2 diagonals b0 = ( 1, 1): pixel (tau - l, l0 + tau)          line y - x
//   kind 3 anti-diag b0 = ( 1,-1): pixel (tau - 31 + l, l0 + 31 - tau) line x + y
// View +b0 ("P") has its occluders at larger tau, view -b0 ("N") at smaller.
#include <algorithm>
#include <climits>

#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cstring>

#include "occ_device.cuh"

namespace occ {

namespace {
constexpr uint32_t FULL = 0xffffffffu;
constexpr int32_t NONE_LO = -(1 << 29), NONE_HI = (1 << 29);
constexpr int kSlot = 1280;              // floats per staging slot (5 KB: keeps both slots 1 KB aligned)
constexpr int kWordSlots = 12;            // words per K0 block and lane
}  // namespace

// merged diagonal words: K0 ORs both halves of every diagonal / anti-diagonal
// word (atomics into a zeroed buffer) so the sweep loads one word instead of
// two and an OR (C5 A/B on one B200: 18.68 vs 18.91 ms per step)
#ifndef SWEEP_DMERGE
#define SWEEP_DMERGE 1
#endif
#ifndef SWEEP_STORE_LEAN
#define SWEEP_STORE_LEAN 1
#endif
// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t s_ge(int32_t a) { return a <= 0 ? FULL : (a >= 32 ? 0u : (FULL << a)); }
__device__ __forceinline__ uint32_t s_le(int32_t b) { return b < 0 ? 0u : (b >= 31 ? FULL : ((2u << b) - 1u)); }
// w << 1 | sign bit of x
__device__ __forceinline__ uint32_t s_push(uint32_t w, float x) { return __funnelshift_l(__float_as_uint(x), w, 1); }
__device__ __forceinline__ uint32_t s_sgn(float x) { return __float_as_uint(x) >> 31; }
__device__ __forceinline__ float s_nextup(float a) {
    const int32_t b = __float_as_int(a);
    if (a == 0.0f) return __int_as_float(1);
    return __int_as_float(a > 0.0f ? b + 1 : b - 1);
}
__device__ __forceinline__ uint32_t s_expand4(uint32_t b4) { return (b4 * 0x00204081u) & 0x01010101u; }
__device__ __forceinline__ uint32_t s_transpose32(uint32_t x, int lane) {
    const uint32_t M[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int s = 16 >> k;
        const uint32_t m = M[k];
        const uint32_t y = __shfl_xor_sync(FULL, x, s);
        x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
    }
    return x;
}
// bits [st, st + 32) of the OR-dilation of the 96-bit x = x0 | x1 << 32 |
// x2 << 64 by a window of w bits (bit t = OR of x[t .. t + w - 1]);
// 1 <= w <= 33, 0 <= st, st + 31 + w - 1 < 96 (window coverage for h < 17)
__device__ __forceinline__ uint32_t s_dil(uint32_t x0, uint32_t x1, uint32_t x2, int32_t w, int32_t st) {
    int32_t c = 1;
    while (2 * c <= w) {
        x0 |= __funnelshift_r(x0, x1, c);
        x1 |= __funnelshift_r(x1, x2, c);
        x2 |= x2 >> c;
        c *= 2;
    }
    if (c < w) {
        const int32_t k = w - c;
        x0 |= __funnelshift_r(x0, x1, k);
        x1 |= __funnelshift_r(x1, x2, k);
        x2 |= x2 >> k;
    }
    return st < 32 ? __funnelshift_r(x0, x1, st) : __funnelshift_r(x1, x2, st - 32);
}
__device__ __forceinline__ void s_cp16(float *dst, const float *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void s_cp4(float *dst, const float *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void s_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void s_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ====================================================================== K0
// One warp per 32 x 32 pixel block (x-block kx, y-block m, frame f): lane c
// owns column 32 kx + c and walks the 32 rows.  Per pixel (Eq. 1, reading
// Q1): E_x = D[x+1,y] - D[x,y], E_y = D[x,y+1] - D[x,y] (0 on the last
// column / row), edge <=> E^2 > e2_thresh (the exact rewrite of
// sqrt_rn(E^2) > t_e, DESIGN §2 Q4); Eq. 2 for b0 in {(1,0), (0,1), (1,1),
// (1,-1)} is the sign of b0 . (E_x, E_y), exact in fp32 here: the +-1
// products are exact and the rounded sum has the sign of the exact sum; the
// axis families keep the 0 * E term (0 * inf = NaN: no candidate, as the
// oracle's binary64 dot).  Bit v of a pixel: candidate of view +b0 (v even)
// or -b0 (v odd).  Row words (ballots over the lanes) are transposed /
// skewed into the sweep's (line, 32-position) words:
//   slots 0,1  rows:      line block m,        block kx; lane = row,    bit = column
//   slots 2,3  columns:   line block kx,       block m;  lane = column, bit = row
//   slots 4..7 diagonals: lower (c <= r) / upper (c > r) parts, lane = (r - c) mod 32, bit = r
//   slots 8..11 anti:     lower (c + r <= 31) / upper parts,   lane = (c + r) mod 32, bit = 31 - r
struct WordsArgs {
    const float *D;
    int32_t H, W, nxb, nyb;
    float e2_thresh;
    FrameStats *st;
    uint32_t *words;       // [frame][nyb][nxb + 1][12][32] (one spare column: merged diagonal words)
    int32_t do_stats;
};

__global__ void __launch_bounds__(128) k_words(WordsArgs a) {
    __shared__ uint32_t rw[4][32][8];
    __shared__ int32_t r_lo[4], r_hi[4];
    __shared__ uint32_t r_bad[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t kx = blockIdx.x * 4 + warp, m = blockIdx.y, f = blockIdx.z;
    const int32_t H = a.H, W = a.W;
    const float *Df = a.D + (int64_t)f * H * W;
    int32_t lo = 0x7FFFFFFF, hi = (int32_t)0x80000000;
    uint32_t bad = 0;
    {   // (warps past the last x-block run with every load off: no divergent branch around the ballots)
        const bool wok = kx < a.nxb;
        const int32_t x = 32 * kx + lane, y0 = 32 * m;
        const bool xin = wok && x < W, xr = xin && x + 1 < W;
        // (branch-free body: the ballots stay convergent)
        const float *col = Df + x;
        float v = (xin && y0 < H) ? __ldg(col + (int64_t)y0 * W) : 0.0f;
        const bool l31 = lane == 31;
#ifndef WORDS_UNROLL
#define WORDS_UNROLL 32           // (C5 k_words ms per 256 frames: unroll 2 1.52, 4 1.57, 8 1.72, 32 1.50)
#endif
#define S_PRAGMA(x) _Pragma(#x)
#define S_UNROLL(n) S_PRAGMA(unroll n)
        S_UNROLL(WORDS_UNROLL)
        for (int r = 0; r < 32; ++r) {
            const int32_t y = y0 + r;
            const bool yin = y < H, yb = y + 1 < H;
            const bool in = xin && yin;
            const float below = (xin && yb) ? __ldg(col + (int64_t)(y + 1) * W) : 0.0f;
            const float r31 = (l31 && xr && yin) ? __ldg(col + (int64_t)y * W + 1) : 0.0f;
            const float sh = __shfl_down_sync(FULL, v, 1);
            const float right = l31 ? r31 : sh;
            const float ex = xr ? __fsub_rn(right, v) : 0.0f;
            const float ey = yb ? __fsub_rn(below, v) : 0.0f;
            const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
            const bool edge = in && e2 > a.e2_thresh;
            const float d0 = __fmaf_rn(0.0f, ey, ex), d1 = __fmaf_rn(0.0f, ex, ey);
            const float d2 = __fadd_rn(ex, ey), d3 = __fsub_rn(ex, ey);
            const uint32_t b0 = __ballot_sync(FULL, edge && d0 > 0.0f), b1 = __ballot_sync(FULL, edge && d0 < 0.0f);
            const uint32_t b2 = __ballot_sync(FULL, edge && d1 > 0.0f), b3 = __ballot_sync(FULL, edge && d1 < 0.0f);
            const uint32_t b4 = __ballot_sync(FULL, edge && d2 > 0.0f), b5 = __ballot_sync(FULL, edge && d2 < 0.0f);
            const uint32_t b6 = __ballot_sync(FULL, edge && d3 > 0.0f), b7 = __ballot_sync(FULL, edge && d3 < 0.0f);
            if (lane == 0) {
                *reinterpret_cast<uint4 *>(&rw[warp][r][0]) = make_uint4(b0, b1, b2, b3);
                *reinterpret_cast<uint4 *>(&rw[warp][r][4]) = make_uint4(b4, b5, b6, b7);
            }
            // statistics (exact min / max through ordered keys, non-finite count)
            const bool fin = in && isfinite(v);
            const int32_t key = float_key(v);
            lo = fin ? min(lo, key) : lo;
            hi = fin ? max(hi, key) : hi;
            bad += (in && !fin) ? 1u : 0u;
            v = below;
        }
        __syncwarp();
        const uint4 q0 = *reinterpret_cast<const uint4 *>(&rw[warp][lane][0]);
        const uint4 q1 = *reinterpret_cast<const uint4 *>(&rw[warp][lane][4]);
        uint32_t o[kWordSlots];
        o[0] = q0.x;
        o[1] = q0.y;
        o[2] = s_transpose32(q0.z, lane);
        o[3] = s_transpose32(q0.w, lane);
        const uint32_t ge = FULL << lane, gea = FULL << (31 - lane);
        {   // diagonals: Q[r] bit j = R[r] bit ((r - j) mod 32)
            const uint32_t t4 = s_transpose32(__funnelshift_r(__brev(q1.x), __brev(q1.x), 31 - lane), lane);
            const uint32_t t5 = s_transpose32(__funnelshift_r(__brev(q1.y), __brev(q1.y), 31 - lane), lane);
            o[4] = t4 & ge;  o[5] = t5 & ge;
            o[6] = t4 & ~ge; o[7] = t5 & ~ge;
        }
        {   // anti-diagonals: Q[r] bit j = R[r] bit ((j - r) mod 32), then bit reversal (bit = 31 - r)
            const uint32_t t6 = __brev(s_transpose32(__funnelshift_l(q1.z, q1.z, lane), lane));
            const uint32_t t7 = __brev(s_transpose32(__funnelshift_l(q1.w, q1.w, lane), lane));
            o[8] = t6 & gea;  o[9] = t7 & gea;
            o[10] = t6 & ~gea; o[11] = t7 & ~gea;
        }
        uint32_t *dst = a.words + ((((int64_t)f * a.nyb + m) * (a.nxb + 1) + kx) * kWordSlots) * 32 + lane;
        if (wok) {
#if SWEEP_DMERGE
            // the diagonal words of record (m, kx) are lower(m, kx) | upper(m,
            // kx - 1): OR both halves into the zeroed slots 4, 5 / 8, 9 (the
            // upper halves into the next record), so the sweep loads one word
#pragma unroll
            for (int s = 0; s < 4; ++s) dst[s * 32] = o[s];
            atomicOr(dst + 4 * 32, o[4]);
            atomicOr(dst + 5 * 32, o[5]);
            atomicOr(dst + 8 * 32, o[8]);
            atomicOr(dst + 9 * 32, o[9]);
            atomicOr(dst + (kWordSlots + 4) * 32, o[6]);
            atomicOr(dst + (kWordSlots + 5) * 32, o[7]);
            atomicOr(dst + (kWordSlots + 8) * 32, o[10]);
            atomicOr(dst + (kWordSlots + 9) * 32, o[11]);
#else
#pragma unroll
            for (int s = 0; s < kWordSlots; ++s) dst[s * 32] = o[s];
#endif
        }
    }
    if (!a.do_stats) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(FULL, lo, o));
        hi = max(hi, __shfl_xor_sync(FULL, hi, o));
        bad += __shfl_xor_sync(FULL, bad, o);
    }
    if (lane == 0) { r_lo[warp] = lo; r_hi[warp] = hi; r_bad[warp] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 4; ++w) { lo = min(lo, r_lo[w]); hi = max(hi, r_hi[w]); bad += r_bad[w]; }
        if (lo != 0x7FFFFFFF) atomicMin(&a.st[f].minkey, lo);
        if (hi != (int32_t)0x80000000) atomicMax(&a.st[f].maxkey, hi);
        if (bad) atomicAdd(&a.st[f].nonfinite, bad);
    }
}

cudaError_t launch_words(const float *D, int32_t H, int32_t W, int32_t frames, float e2_thresh, FrameStats *st,
                         uint32_t *words, int32_t do_stats, cudaStream_t s) {
    WordsArgs a{D, H, W, (W + 31) / 32, (H + 31) / 32, e2_thresh, st, words, do_stats};
#if SWEEP_DMERGE
    cudaError_t e = cudaMemsetAsync(words, 0, sizeof(uint32_t) * (size_t)frames * sweep_words_per_frame(H, W), s);
    if (e != cudaSuccess) return e;
#endif
    dim3 grid((unsigned)((a.nxb + 3) / 4), (unsigned)a.nyb, (unsigned)frames);
    k_words<<<grid, 128, 0, s>>>(a);
    return cudaGetLastError();
}

// ===================================================================== K1
struct SweepArgs {
    const float *D;
    int32_t H, W, nxb, nyb;
    const SweepUnit *units;    // sorted by kind (kinds 0..3 at [kstart[k], kstart[k + 1]))
    int32_t nunits, frames;
    int32_t kstart[5];
    int32_t fgroup;            // frames per group: work order group, kind, unit, frame
    const GroupDesc *groups;
    const ViewDesc *views;
    int32_t nviews;
    const FamilyDesc *fams;
    const FrameStats *st;
    Params p;
    uint8_t *masks;
    MaskFmt mf;
    const uint32_t *words;
    HardEntry *gq;
    uint32_t *gq_count;
    int32_t gq_cap;
    int32_t tma;               // 1: TMA staging (W % 4 == 0, 16-byte aligned frames); 0: 4-byte cp.async
    // Sheared family (knight baselines, k_shear): D is the sheared copy whose
    // rows (shkind 0, x-major) or columns (shkind 1, y-major) are the
    // family's digital lines; line l' of it is the image line l = l' + sh_lmin,
    // whose pixel at position tau is (tau, l + floor(tau num / den)) or
    // (l + floor(tau num / den), tau) of the Ho x Wo image the masks cover.
    int32_t shkind, sh_num, sh_den, sh_lmin, Ho, Wo;
    unsigned long long *dbg;   // event counters (SWEEP_STATS builds), or null
};
// TMA descriptors of D viewed as [frames][H][W] fp32 (out-of-image boxes read NaN)
struct SweepMaps {
    CUtensorMap rows;          // box 32 x 32, 128-byte swizzle: kind 0 tile [line][position]
    CUtensorMap cols;          // box 32 x 32: kind 1 tile [position][line]
    CUtensorMap run;           // box 32 x 1: one image-row run of the diagonal kinds
};

// warp-aggregated event counter (SWEEP_STATS builds only; warp-uniform call)
#ifdef SWEEP_STATS
#define SST(idx, n)                                                                           \
    do {                                                                                      \
        const unsigned t_ = __reduce_add_sync(FULL, (unsigned)(n));                           \
        if (a.dbg && (threadIdx.x & 31) == 0 && t_) atomicAdd(a.dbg + (idx), (unsigned long long)t_); \
    } while (0)
#else
#define SST(idx, n) do { } while (0)
#endif

// ---------------------------------------------------------------- mbarrier / TMA
__device__ __forceinline__ uint32_t s_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void s_mbar_init(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_smem(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void s_mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void s_mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(s_smem(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void s_tma3(float *dst, const CUtensorMap *m, int32_t x, int32_t y, int32_t z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(s_smem(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(s_smem(bar))
        : "memory");
}

// Per-warp constants of one unit
struct SU {
    int32_t kind, l0, A, lane, H, W, nxb, nyb, f;
    int32_t elo, ehi;          // lane's in-image tau range
    int64_t B;                 // pixel index of the lane's line at tau = 0
    int32_t S;                 // pixel stride per tau
    const float *Df;
    const uint32_t *Wf;        // frame's candidate words
};

__device__ __forceinline__ void s_extent(int kind, int32_t l0, int32_t l, int32_t H, int32_t W, int32_t &lo,
                                         int32_t &hi) {
    const int32_t L = l0 + l;
    if (kind == 0) { lo = 0; hi = (L < H) ? W : 0; }
    else if (kind == 1) { lo = 0; hi = (L < W) ? H : 0; }
    else if (kind == 2) { lo = max(l, -l0); hi = min(W + l, H - l0); }
    else { lo = max(31 - l, l0 + 32 - H); hi = min(W + 31 - l, l0 + 32); }
    if (hi < lo) hi = lo;
}
__device__ __forceinline__ int64_t s_base(int kind, int32_t l0, int32_t l, int32_t W) {
    if (kind == 0) return (int64_t)(l0 + l) * W;
    if (kind == 1) return (int64_t)(l0 + l);
    if (kind == 2) return (int64_t)l0 * W - l;
    return (int64_t)(l0 + 31) * W - 31 + l;
}
__device__ __forceinline__ int32_t s_stride(int kind, int32_t W) {
    return kind == 0 ? 1 : (kind == 1 ? W : (kind == 2 ? W + 1 : 1 - W));
}

// candidate word of one view (v = 0: +b0, 1: -b0) for tau block k
__device__ __forceinline__ uint32_t s_word1(const SU &u, int32_t k, int v) {
    const uint32_t *Wl = u.Wf + u.lane + 32 * v;
    constexpr int St = kWordSlots * 32;
    const int32_t P = u.nxb + 1;              // record pitch
    if (u.kind == 0) return (uint32_t)k < (uint32_t)u.nxb ? __ldg(Wl + (u.A * P + k) * St) : 0u;
    if (u.kind == 1) return (uint32_t)k < (uint32_t)u.nyb ? __ldg(Wl + (k * P + u.A) * St + 64) : 0u;
    const int32_t m = u.kind == 2 ? u.A + k : u.A - k;
    if ((uint32_t)m >= (uint32_t)u.nyb) return 0u;
    const uint32_t *p = Wl + (m * P + k) * St + (u.kind == 2 ? 4 * 32 : 8 * 32);
#if SWEEP_DMERGE
    return (uint32_t)k <= (uint32_t)u.nxb ? __ldg(p) : 0u;
#else
    uint32_t w = 0u;
    if ((uint32_t)k < (uint32_t)u.nxb) w = __ldg(p);
    if ((uint32_t)(k - 1) < (uint32_t)u.nxb) w |= __ldg(p - St + 64);
    return w;
#endif
}

#ifndef SWEEP_ROWCOPY
#define SWEEP_ROWCOPY 1
#endif
// Stages tau block k (32 positions of the 32 lines) into a slot:
//   kind 0: [line][32 positions] with the 128-byte swizzle (16-byte chunk c of row l at c ^ (l & 7));
//   kind 1: [position][32 lines];
//   kinds 2, 3: [position r][36 x from ((32k + r - 31) & ~3)] (the 32 lines' run of image row r,
//   4-aligned: the lane's element sits at 31 - l (kind 2) or l (kind 3) plus (r + 1) & 3).
// Kinds 0, 1 by one TMA box (32 x 32, completion on the slot's mbarrier;
// out-of-image elements read NaN); kinds 2, 3 by 16-byte cp.async (TMA boxes
// need 16-byte aligned x and 128-byte aligned destinations: a row run would
// take 256 bytes of shared memory).  Unaligned frames: 4-byte cp.async.
// Returns whether the block was staged by TMA (then wait on the mbarrier).
__device__ __noinline__ bool s_stage(const SU &u, const SweepMaps &tm, float *slot, uint64_t *bar, int32_t k, int tma) {
    const int lane = u.lane;
    const float NaN = __int_as_float(0x7fc00000);
    const int32_t H = u.H, W = u.W;
    if (tma && u.kind <= 1) {
        if (lane == 0) {
            s_mbar_expect(bar, 4096u);
            if (u.kind == 0) s_tma3(slot, &tm.rows, 32 * k, u.l0, u.f, bar);
            else s_tma3(slot, &tm.cols, u.l0, 32 * k, u.f, bar);
        }
        return true;
    }
    if (tma) {                       // kinds 2, 3: 16-byte copies of the 4-aligned row runs
#if SWEEP_ROWCOPY
        // lane r copies row r's 9 chunks (one address per lane, immediate offsets)
        const int r = lane;
        const int32_t y = u.kind == 2 ? u.l0 + 32 * k + r : u.l0 + 31 - 32 * k - r;
        const int32_t x0 = 32 * k + ((r - 31) & ~3);
        float *dst = slot + r * 36;
        const float *src = u.Df + (int64_t)y * W + x0;
        if ((uint32_t)y < (uint32_t)H && x0 >= 0 && x0 + 36 <= W) {
#pragma unroll
            for (int q = 0; q < 9; ++q) s_cp16(dst + 4 * q, src + 4 * q);
        } else {
#pragma unroll
            for (int q = 0; q < 9; ++q) {
                if ((uint32_t)y < (uint32_t)H && (uint32_t)(x0 + 4 * q) < (uint32_t)W) s_cp16(dst + 4 * q, src + 4 * q);
                else *reinterpret_cast<float4 *>(dst + 4 * q) = make_float4(NaN, NaN, NaN, NaN);
            }
        }
#else
        const int32_t dy = u.kind == 2 ? 32 * k : -32 * k;
#pragma unroll 3
        for (int i = 0; i < 9; ++i) {
            const int c = lane + 32 * i, r = c / 9, q = c - 9 * r;
            const int32_t y = (u.kind == 2 ? u.l0 + r : u.l0 + 31 - r) + dy;
            const int32_t x = 32 * k + ((r - 31) & ~3) + 4 * q;
            float *dst = slot + r * 36 + 4 * q;
            OCC_CHECK(r < 32 && q < 9 && r * 36 + 4 * q + 4 <= kSlot);
            if ((uint32_t)x < (uint32_t)W && (uint32_t)y < (uint32_t)H) s_cp16(dst, u.Df + (int64_t)y * W + x);
            else *reinterpret_cast<float4 *>(dst) = make_float4(NaN, NaN, NaN, NaN);
        }
#endif
        s_commit();
        return false;
    }
    for (int r = 0; r < 32; ++r) {
        const int32_t tau = 32 * k + r;
        float *dst;
        if (u.kind == 0) dst = slot + lane * 32 + ((((r >> 2) ^ (lane & 7)) << 2) | (r & 3));
        else if (u.kind == 1) dst = slot + r * 32 + lane;
        else dst = slot + r * 36 + (u.kind == 2 ? 31 - lane : lane) + ((r + 1) & 3);
        if (tau >= u.elo && tau < u.ehi) s_cp4(dst, u.Df + u.B + (int64_t)tau * u.S);
        else *dst = NaN;
    }
    s_commit();
    return false;
}
__device__ __forceinline__ void s_stage_wait(uint64_t *bar, uint32_t &phase, bool by_tma) {
    if (by_tma) {
        s_mbar_wait(bar, phase);
        phase ^= 1u;
    } else {
        s_wait<0>();
    }
    __syncwarp();
}

// staged value at block position r of the line of lane l (see s_stage's layouts)
__device__ __forceinline__ int s_at(int kind, int l, int r) {
    if (kind == 0) return l * 32 + ((((r >> 2) ^ (l & 7)) << 2) | (r & 3));
    if (kind == 1) return r * 32 + l;
    return r * 36 + (kind == 2 ? 31 - l : l) + ((r + 1) & 3);
}
// the lane's staged values at positions 4g .. 4g + 3 (rb: the lane's read base)
__device__ __forceinline__ float4 s_read4(const float *rb, int kind, int g, int sw) {
    if (kind == 0) return *reinterpret_cast<const float4 *>(rb + ((g ^ sw) << 2));
    if (kind == 1) {
        const float *p = rb + g * 128;
        return make_float4(p[0], p[32], p[64], p[96]);
    }
    const float *p = rb + g * 144;
    return make_float4(p[1], p[36 + 2], p[72 + 3], p[108]);
}
// value at tau straight from global memory (NaN outside the line)
__device__ __forceinline__ float s_gv(const SU &u, int32_t tau) {
    return (tau >= u.elo && tau < u.ehi) ? __ldg(u.Df + u.B + (int64_t)tau * u.S) : __int_as_float(0x7fc00000);
}

// mask bits of one view for tau block k (bit r <-> tau = 32k + r), positions
// outside the lane's line already cleared
__device__ __noinline__ void s_store_packed(const SU &u, uint8_t *Mv, const MaskFmt &mf, uint32_t word, int32_t k) {
    const int lane = u.lane;
    const int32_t H = u.H, W = u.W;
    {
        uint32_t *P = reinterpret_cast<uint32_t *>(Mv);
        const int32_t Wb = mf.Wb;
        if (u.kind == 0) {
            const int32_t y = u.l0 + lane;
            if (y < H && 32 * k >= 0 && 32 * k < W) P[(int64_t)y * Wb + k] = word;
        } else if (u.kind == 1) {
            const uint32_t t = s_transpose32(word, lane);
            const int32_t y = 32 * k + lane;
            if (y >= 0 && y < H && u.l0 < W) P[(int64_t)y * Wb + (u.l0 >> 5)] = t;
        } else {
            // tau = 32k + r is one image row; its 32 lanes form a run of 32 x
            uint32_t mine = 0u;
            for (int r = 0; r < 32; ++r) {
                const uint32_t b = __ballot_sync(FULL, (word >> r) & 1u);
                if (r == lane) mine = b;
            }
            const int32_t tau = 32 * k + lane;
            const int32_t y = u.kind == 2 ? u.l0 + tau : u.l0 + 31 - tau;
            const uint32_t run = u.kind == 2 ? __brev(mine) : mine;      // bit j <-> x = tau - 31 + j
            if (run && y >= 0 && y < H) {
                const int32_t x0 = tau - 31, w0 = x0 >> 5, sh = x0 & 31;
                const uint32_t lo = run << sh, hi = sh ? (run >> (32 - sh)) : 0u;
                if (lo && w0 >= 0 && w0 < Wb) atomicOr(P + (int64_t)y * Wb + w0, lo);
                if (hi && w0 + 1 >= 0 && w0 + 1 < Wb) atomicOr(P + (int64_t)y * Wb + w0 + 1, hi);
            }
        }
        return;
    }
}

__device__ __noinline__ void s_store(const SU &u, uint8_t *Mv, const MaskFmt &mf, uint32_t word, int32_t k) {
    const int lane = u.lane;
    const int32_t H = u.H, W = u.W;
    if (mf.packed) {
        s_store_packed(u, Mv, mf, word, k);
        return;
    }
    if (u.kind <= 1) {
        // rows: the lane's 32 positions are one row segment; columns: the bit
        // transpose gives lane r row 32k + r's 32 columns
        const uint32_t t = u.kind == 0 ? word : s_transpose32(word, lane);
        const int32_t y = u.kind == 0 ? u.l0 + lane : 32 * k + lane;
        const int32_t x0 = u.kind == 0 ? 32 * k : u.l0;
        if (y >= H) return;
        uint8_t *row = Mv + (int64_t)y * W + x0;
        if ((W & 15) == 0 && x0 + 32 <= W) {
            uint4 *d = reinterpret_cast<uint4 *>(row);
            __stcs(d, make_uint4(s_expand4(t & 15u), s_expand4((t >> 4) & 15u), s_expand4((t >> 8) & 15u),
                                 s_expand4((t >> 12) & 15u)));
            __stcs(d + 1, make_uint4(s_expand4((t >> 16) & 15u), s_expand4((t >> 20) & 15u),
                                     s_expand4((t >> 24) & 15u), s_expand4(t >> 28)));
        } else {
            for (int j = 0; j < 32; ++j)
                if (x0 + j < W) row[j] = (uint8_t)((t >> j) & 1u);
        }
        return;
    }
    // one image row per tau: the 32 lanes write one contiguous run
    uint8_t *dst = Mv + u.B + (int64_t)(32 * k) * u.S;
    const int64_t S = u.S;
#ifdef OCC_CHECKS
    for (int r = 0; r < 32; ++r) {
        const int32_t tau = 32 * k + r;
        const int64_t pix = u.B + (int64_t)tau * u.S;
        OCC_CHECK(tau < u.elo || tau >= u.ehi || (pix >= 0 && pix < (int64_t)H * W));
    }
#endif
    if (32 * k >= u.elo && 32 * k + 32 <= u.ehi) {
#if SWEEP_STORE_LEAN
        // pointer steps and a shifted word (no per-byte variable shift)
        uint32_t w = word;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) { __stcs(dst, (uint8_t)(w & 1u)); w >>= 1; dst += S; }
#else
#pragma unroll 8
        for (int r = 0; r < 32; ++r) __stcs(dst + r * S, (uint8_t)((word >> r) & 1u));
#endif
    } else {
        for (int r = 0; r < 32; ++r) {
            const int32_t tau = 32 * k + r;
            if (tau >= u.elo && tau < u.ehi) __stcs(dst + r * S, (uint8_t)((word >> r) & 1u));
        }
    }
}

// (the knight families have den = 2: floor(t num / 2) is an arithmetic shift)
// masks of a sheared family (knight baselines): bit r of the lane's word is
// line l0 + lane at tau = 32k + r; un-shear to the image pixel and write it
// (uint8: every in-image byte of the unit's lines once; packed: set bits).
// Every warp store covers consecutive x of one image row:
//   y-major (kind 1): at tau = row y the 32 lines are 32 consecutive x;
//   x-major (kind 0): lane c writes column 32k + c of each row the block's
//   lines cross, taking the bit from the line that owns that pixel (shuffle).
__device__ __noinline__ void s_store_sh(const SU &u, const SweepArgs &a, uint8_t *Mv, uint32_t word, int32_t k) {
    const int lane = u.lane;
    const int32_t Ho = a.Ho, Wo = a.Wo;
    const bool packed = a.mf.packed != 0;
    uint32_t *P = reinterpret_cast<uint32_t *>(Mv);
    if (u.kind == 1) {                    // pixel (l + f(tau), tau)
        const bool lok = u.l0 + lane < u.W;
        const int32_t xl = u.l0 + lane + a.sh_lmin;
        for (int r = 0; r < 32; ++r) {
            const int32_t y = 32 * k + r;
            if (y < 0 || y >= Ho) continue;                       // warp-uniform
            const int32_t x = xl + ((y * a.sh_num) >> 1);
            const bool ok = lok && (uint32_t)x < (uint32_t)Wo;
            const uint32_t b = (word >> r) & 1u;
            if (!packed) {
                if (ok) __stcs(Mv + (int64_t)y * Wo + x, (uint8_t)b);
            } else {
                const uint32_t run = __ballot_sync(FULL, ok && b);    // bit j <-> x = x(lane 0) + j
                const int32_t x0 = __shfl_sync(FULL, x, 0);               // lanes are consecutive x
                if (lane == 0 && run) {
                    const int32_t xs = x0, w0 = xs >> 5, sh = xs - 32 * w0;
                    const uint32_t lo = run << sh, hi = sh ? (run >> (32 - sh)) : 0u;
                    if (lo && w0 >= 0 && w0 < a.mf.Wb) atomicOr(P + (int64_t)y * a.mf.Wb + w0, lo);
                    if (hi && w0 + 1 >= 0 && w0 + 1 < a.mf.Wb) atomicOr(P + (int64_t)y * a.mf.Wb + w0 + 1, hi);
                }
            }
        }
        return;
    }
    // x-major: pixel (tau, l + f(tau)); lane c writes column x = 32k + c
    const int32_t x = 32 * k + lane;
    const int32_t fc = (x * a.sh_num) >> 1;
    const int32_t fa = (32 * k * a.sh_num) >> 1, fb = ((32 * k + 31) * a.sh_num) >> 1;
    const int32_t Lb = u.l0 + a.sh_lmin;  // image line of lane 0
    const bool xok = x < Wo;
    for (int32_t y = max(0, Lb + min(fa, fb)); y <= min(Ho - 1, Lb + 31 + max(fa, fb)); ++y) {
        const int32_t o = y - fc - Lb;                            // the lane whose line holds (x, y)
        const uint32_t w = __shfl_sync(FULL, word, o & 31);
        const bool ok = xok && (uint32_t)o < 32u && u.l0 + o < u.H;
        const uint32_t b = (w >> lane) & 1u;
        if (!packed) {
            if (ok) __stcs(Mv + (int64_t)y * Wo + x, (uint8_t)b);
        } else {
            const uint32_t bits = __ballot_sync(FULL, ok && b);
            if (lane == 0 && bits) atomicOr(P + (int64_t)y * a.mf.Wb + k, bits);
        }
    }
}

// Eq. 5 for a far pair (offset j >= jstar: delta > t_disp is implied):
// |s fl(vq - vp) - j| < t_dist; fp32 with a 2^-10 band, binary64 inside it.
__device__ __noinline__ bool s_pair_slow(float vq, float vp, int32_t j, int32_t s, float t_dist, float t_disp) {
    return pair_exact(vq, vp, -j, s, t_dist, t_disp);
}
__device__ __forceinline__ bool s_pair_far(float vq, float vp, int32_t j, float fs, int32_t s, float tlo, float thi,
                                           const Params &p) {
    const float x = fabsf(__fmaf_rn(fs, __fsub_rn(vq, vp), -(float)j));
    if (x < tlo) return true;
    if (!(x <= thi)) return false;
    return s_pair_slow(vq, vp, j, s, p.t_dist, p.t_disp);
}

// exhaustive search of one survivor (queue full): offsets 3..J along the line
__device__ __noinline__ bool s_exhaust(const float *Df, int64_t B, int32_t S, int32_t elo, int32_t ehi, int32_t tau,
                                       int dir, int32_t J, float vp, float fs, int32_t s, float tlo, float thi,
                                       const Params &p) {
    for (int32_t j = 3; j <= J; ++j) {
        const int32_t t = tau + dir * j;
        const float vq = (t >= elo && t < ehi) ? __ldg(Df + B + (int64_t)t * S) : __int_as_float(0x7fc00000);
        if (s_pair_far(vq, vp, j, fs, s, tlo, thi, p)) return true;
    }
    return false;
}

// exact per-pixel fallback for the unit's positions (frames the sweep does not serve)
__device__ __noinline__ void s_direct(const SU &u, const SweepArgs &a, const GroupDesc &gd, const FamilyDesc &fd,
                                      int32_t T0, int32_t T1, bool zero) {
    const float R = frame_range(a.st[u.f]);
    for (int g = 0; g < gd.nv; ++g) {
        const ViewDesc &vd = a.views[gd.view[g]];
        const int32_t h = view_h(R, vd.s, a.p.max_scan);
        uint8_t *Mv = a.masks + ((int64_t)u.f * a.nviews + gd.view[g]) * a.mf.vbytes;
        for (int32_t tau = max(T0, u.elo); tau < min(T1, u.ehi); ++tau) {
            const int64_t pix = u.B + (int64_t)tau * u.S;
            const int32_t y = (int32_t)(pix / u.W), x = (int32_t)(pix - (int64_t)y * u.W);
            const bool mk = !zero && direct_pixel<false>(u.Df, u.H, u.W, vd, fd, a.p, h, x, y);
            mask_put(Mv, a.mf, u.W, x, y, mk);
        }
    }
}

struct Rec {                   // pass 1 -> pass 2, per block and lane (12 bytes)
    uint32_t XN;               // view -b far-filter survivors (bit r <-> tau0 + r)
    int16_t pclP;              // last +b candidate <= tau0 + h - 1, minus tau0 (clamped: see s_rel)
    int16_t lcN;               // last -b candidate <= tau0 + 31 - h, minus tau0
    __half2 VW;                // v at the -b filter's witness after positions 0 / 16 (partner guesses)
};
// candidate positions relative to the block, clamped below: a last candidate
// further than 2h + 32 below the block's start covers none of its windows
__device__ __forceinline__ int16_t s_rel(int32_t c, int32_t tau0, int32_t h) {
    return (int16_t)max(c - tau0, -min(2 * h + 64, 32000));
}

constexpr int kMaxSegBlocks = kSweepSeg / 32;
constexpr int kListCap = 256;                 // dense survivor list (entries per pass)
#ifndef SWEEP_NSLOT
#define SWEEP_NSLOT 1
#endif
constexpr int kNSlot = SWEEP_NSLOT;        // staging slots per warp (2: prefetch the next block)
constexpr size_t kRecOff = sizeof(float) * kSlot * kNSlot;
constexpr size_t kListOff = kRecOff + sizeof(Rec) * 32 * kMaxSegBlocks;
constexpr size_t kMarkOff = kListOff + sizeof(uint16_t) * kListCap;
constexpr size_t kBarOff = kMarkOff + sizeof(uint32_t) * 64;
constexpr size_t kSweepWarpSmem = ((kBarOff + 16) + 1023) & ~(size_t)1023;   // 1 KB aligned (128-byte swizzle)
size_t sweep_smem_bytes() { return kSweepWarpSmem; }

__device__ __forceinline__ int32_t s_guess(float vw, float vp, float fs, int32_t J) {
    return min(max(__float2int_rn(fminf(fmaxf(__fmul_rn(fs, __fsub_rn(vw, vp)), -1e9f), 1e9f)), 3), J);
}

struct SurvCtx {
    int32_t tau0, h;
    uint32_t WP, WN;           // window candidate bits: +b [tau0 + h, +31], -b [tau0 - h, +31]
    int32_t pcl, ncl;          // last +b candidate <= tau0 + h - 1, first -b candidate >= tau0 + 32 - h
    float Q0, Q1, Q2, Q3;      // +b witness values after positions 7, 15, 23, 31
    __half2 VW;                // -b witness values after positions 0, 16
    float fs;
    int32_t s;
    float tlo, thi;
    int32_t vP, vN;
};

// one listed survivor, decoded with its owner lane's context (warp-collective: shuffles)
struct SurvDec {
    int64_t B;                 // owner line's pixel index at tau = 0
    int32_t i, J, dir, j1;     // position, largest partner offset, direction (+1: +b), probe offset
    float vp;                  // v(i)
    int src, r, view;
    bool ok;                   // a listed survivor with J >= 3
};
__device__ __forceinline__ SurvDec s_decode(const SU &u, const float *slot, const SurvCtx &c, const uint16_t *list,
                                            uint32_t tot, uint32_t e, uint32_t Blo, uint32_t Bhi) {
    SurvDec d;
    const bool valid = e < tot;
    const uint32_t ent = valid ? list[e] : 0u;
    d.src = (int)(ent >> 6); d.r = (int)(ent & 31); d.view = (int)((ent >> 5) & 1);
    const int src = d.src, r = d.r;
    const uint32_t wp = __shfl_sync(FULL, c.WP, src), wn = __shfl_sync(FULL, c.WN, src);
    const int32_t pcl = __shfl_sync(FULL, c.pcl, src), ncl = __shfl_sync(FULL, c.ncl, src);
    const float q0 = __shfl_sync(FULL, c.Q0, src), q1 = __shfl_sync(FULL, c.Q1, src);
    const float q2 = __shfl_sync(FULL, c.Q2, src), q3 = __shfl_sync(FULL, c.Q3, src);
    const uint32_t vwb = __shfl_sync(FULL, *reinterpret_cast<const uint32_t *>(&c.VW), src);
    const int32_t elo = __shfl_sync(FULL, u.elo, src), ehi = __shfl_sync(FULL, u.ehi, src);
    d.B = (int64_t)(((uint64_t)__shfl_sync(FULL, Bhi, src) << 32) | __shfl_sync(FULL, Blo, src));
    d.i = c.tau0 + r;
    d.vp = slot[s_at(u.kind, src, r)];
    float vw;
    if (d.view == 0) {
        const uint32_t m = wp & s_le(r);
        const int32_t pc = m ? c.tau0 + c.h + 31 - __clz(m) : pcl;
        d.J = min(pc + c.h - d.i, ehi - 1 - d.i);
        d.dir = 1;
        vw = r >= 16 ? (r >= 24 ? q3 : q2) : (r >= 8 ? q1 : q0);
    } else {
        const uint32_t m = wn & s_ge(r);
        const int32_t nc = m ? c.tau0 - c.h + __ffs(m) - 1 : ncl;
        d.J = min(d.i + c.h - nc, d.i - elo);
        d.dir = -1;
        const __half2 h2 = *reinterpret_cast<const __half2 *>(&vwb);
        vw = r >= 16 ? __high2float(h2) : __low2float(h2);
    }
    d.ok = valid && d.J >= 3;
    d.j1 = s_guess(vw, d.vp, c.fs, d.J);
    return d;
}

// Dense resolution of one block's far survivors (Eq. 5 far pairs,
// PAPER.md:131-142): the survivors of all lanes are listed lane-major in
// shared memory (entry = r | view << 5 | lane << 6) and resolved 32 per
// round, whatever lanes own them; a round reads the owner's window words,
// witnesses and line by shuffles.  For survivor i of view +b (-b) the
// partner offset j lies in [3, J], J = dcov(i) (S8) clipped to the line; the
// probe is at the witness guess j = s (v_w - v_i) (all probes of the block in
// flight together); a miss goes to k_hard's queue.  Hits are OR-ed into the
// owner's mask word by shared-memory atomics.
__device__ __forceinline__ void s_resolve(const SweepArgs &a, const SU &u, const float *slot, const SurvCtx &c,
                                       uint32_t sP, uint32_t sN, uint32_t &mP, uint32_t &mN, uint16_t *list,
                                       uint32_t *marks) {
    const int lane = u.lane;
    const float NaN = __int_as_float(0x7fc00000);
    marks[lane] = 0u;
    marks[32 + lane] = 0u;
    // (rare) more survivors than the list holds: blocks of 4 positions in
    // turn (at most 4 x 64 = 256 <= kListCap entries each)
    static_assert(4 * 64 <= kListCap, "list capacity");
    const int rw = __reduce_add_sync(FULL, __popc(sP) + __popc(sN)) > (uint32_t)kListCap ? 4 : 32;
    const uint32_t Blo = (uint32_t)u.B, Bhi = (uint32_t)((uint64_t)u.B >> 32);
    for (int rlo = 0; rlo < 32; rlo += rw) {
        const uint32_t pm = s_ge(rlo) & s_le(rlo + rw - 1);
        const uint32_t tP = sP & pm, tN = sN & pm;
        const uint32_t n = __popc(tP) + __popc(tN);
        uint32_t inc = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += t;
        }
        const uint32_t tot = __shfl_sync(FULL, inc, 31);
        {
            uint32_t o = inc - n;
            const uint32_t tag = (uint32_t)lane << 6;
            uint32_t t = tP;
            while (t) { OCC_CHECK(o < (uint32_t)kListCap); list[o++] = (uint16_t)(tag | (__ffs(t) - 1)); t &= t - 1u; }
            t = tN;
            while (t) { OCC_CHECK(o < (uint32_t)kListCap); list[o++] = (uint16_t)(tag | 32 | (__ffs(t) - 1)); t &= t - 1u; }
        }
        __syncwarp();
        for (uint32_t b0 = 0; b0 < tot; b0 += 32) {
            const SurvDec d = s_decode(u, slot, c, list, tot, b0 + lane, Blo, Bhi);
            OCC_CHECK(!d.ok || (d.j1 >= 3 && d.j1 <= d.J && d.B + (int64_t)(d.i + d.dir * d.j1) * u.S >= 0 &&
                                d.B + (int64_t)(d.i + d.dir * d.j1) * u.S < (int64_t)u.H * u.W));
            const float vq = d.ok ? __ldg(u.Df + d.B + (int64_t)(d.i + d.dir * d.j1) * u.S) : NaN;
            bool hit = d.ok && s_pair_far(vq, d.vp, d.j1, c.fs, c.s, c.tlo, c.thi, a.p);
            SST(3 + d.view, hit);
            SST(9, lane == 0);
#ifndef SWEEP_PROBE2
#define SWEEP_PROBE2 0
#endif
            if (SWEEP_PROBE2) {       // (measured slower: its latency costs more than k_hard's extra work)
                const int32_t j2 = s_guess(vq, d.vp, c.fs, d.J);
                const bool p2 = d.ok && !hit && vq == vq && j2 != d.j1;
                if (__any_sync(FULL, p2)) {
                    const float w2 = p2 ? __ldg(u.Df + d.B + (int64_t)(d.i + d.dir * j2) * u.S) : NaN;
                    const bool h2 = p2 && s_pair_far(w2, d.vp, j2, c.fs, c.s, c.tlo, c.thi, a.p);
                    SST(5 + d.view, h2);
                    hit = hit || h2;
                }
            }
            if (hit) atomicOr(marks + 32 * d.view + d.src, 1u << d.r);
            const bool q = d.ok && !hit;
            SST(7 + d.view, q);
            const uint32_t bq = __ballot_sync(FULL, q);
            if (bq) {
                uint32_t base = 0u;
                if (lane == 0) base = atomicAdd(a.gq_count, __popc(bq));
                base = __shfl_sync(FULL, base, 0);
                if (q) {
                    const uint32_t slotq = base + __popc(bq & ((1u << lane) - 1u));
                    const int vid = d.view ? c.vN : c.vP;
                    if (slotq < (uint32_t)a.gq_cap) {
                        HardEntry he;
                        he.pix = (int32_t)(d.B + (int64_t)d.i * u.S);
                        he.meta = (uint32_t)d.J | ((uint32_t)vid << 25);
                        he.guess = d.j1 | (u.f << 17);
                        he.vq = vq;
                        a.gq[slotq] = he;
                    } else {
                        const int32_t elo = d.dir > 0 ? -(1 << 30) : d.i - d.J, ehi = d.dir > 0 ? d.i + d.J + 1 : (1 << 30);
                        if (s_exhaust(u.Df, d.B, u.S, elo, ehi, d.i, d.dir, d.J, d.vp, c.fs, c.s, c.tlo, c.thi, a.p))
                            atomicOr(marks + 32 * d.view + d.src, 1u << d.r);
                    }
                }
            }
        }
        __syncwarp();
    }
    mP |= marks[lane];
    mN |= marks[32 + lane];
    __syncwarp();
}

template <bool SMALLH, bool SHEAR>
__device__ __forceinline__ void sweep_unit(const SweepArgs &a, const SweepMaps &tm, const SweepUnit &un,
                                        const GroupDesc &gd, int32_t f, unsigned char *smem, uint32_t *phase) {
    const FamilyDesc &fd = a.fams[gd.fam];
    SU u;
    u.kind = SHEAR ? a.shkind : fd.kind;
    const int kind = u.kind;
    u.l0 = un.l0;
    u.A = un.l0 >> 5;
    u.lane = threadIdx.x & 31;
    u.H = a.H; u.W = a.W; u.nxb = a.nxb; u.nyb = a.nyb; u.f = f;
    const int lane = u.lane;
    s_extent(kind, u.l0, lane, u.H, u.W, u.elo, u.ehi);
    u.B = s_base(kind, u.l0, lane, u.W);
    u.S = s_stride(kind, u.W);
    const int64_t HW = (int64_t)a.H * a.W;
    u.Df = a.D + (int64_t)f * HW;
    u.Wf = a.words + (int64_t)f * a.nyb * (a.nxb + 1) * kWordSlots * 32;
    float *stg = reinterpret_cast<float *>(smem);
    Rec *rec = reinterpret_cast<Rec *>(smem + kRecOff);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kBarOff);
    const int32_t T0 = un.t0, T1 = un.t1;         // multiples of 32
    const int32_t kB = T0 >> 5, kT = (T1 >> 5) - 1;
    // the lane's read base in a slot (kind 0: its row; 1: its column; 2, 3: its element of the row runs)
    const int32_t rbo = kind == 0 ? lane * 32 : (kind == 2 ? 31 - lane : lane);
    const int sw = lane & 7;

    int32_t vP = -1, vN = -1;
    for (int g = 0; g < gd.nv; ++g) {
        if (a.views[gd.view[g]].sg > 0) vP = gd.view[g]; else vN = gd.view[g];
    }
    const ViewDesc &vd0 = a.views[vP >= 0 ? vP : vN];
    const FrameStats fs = a.st[f];
    const float R = frame_range(fs);
    const int32_t s = vd0.s;
    const int32_t h = view_h(R, s, a.p.max_scan);
    if (fs.nonfinite || h <= 0) {                 // SPEC.md:76 reject / Q17: zero masks
        if constexpr (SHEAR) {        // zeros through the un-shearing store
            for (int32_t k = T0 >> 5; k < (T1 >> 5); ++k) {
                if (vP >= 0) s_store_sh(u, a, a.masks + ((int64_t)f * a.nviews + vP) * a.mf.vbytes, 0u, k);
                if (vN >= 0) s_store_sh(u, a, a.masks + ((int64_t)f * a.nviews + vN) * a.mf.vbytes, 0u, k);
            }
        } else {
            s_direct(u, a, gd, fd, T0, T1, true);
        }
        return;
    }
    // h < 17: window coverage from OR-dilations of the raw candidate words
    // (s_dil) instead of the first / last candidate thresholds (which need
    // 2h >= 34); those units run in k_sweep_small
    if (!SMALLH && h < 17) return;
    constexpr bool smallh = SMALLH;
    const int32_t reach = partner_reach(a.p.t_dist, s, R, h);
    const int32_t nbr = (reach + 3 + 31) >> 5;    // staged warm-up blocks per pass
    const int32_t nbl = (T1 - T0) / 32 + nbr;     // blocks per pass
    const float fs_ = (float)s;
    float T;                                      // far-filter margin
    {
        const float M = fmaxf(fabsf(key_float(fs.minkey)), fabsf(key_float(fs.maxkey)));
        const double P = 32.0 * (nbl + 2);
        const double eps = ldexp(1.0, -23) * (double)(8 * nbl + 5) * ((double)s * (double)M + P + (double)a.p.t_dist + 1.0);
        T = __double2float_ru(__dadd_rn((double)a.p.t_dist, eps));
    }
    const float tlo = __fsub_rn(a.p.t_dist, 0x1p-10f), thi = __fadd_rn(a.p.t_dist, 0x1p-10f);
    const float a1n = s_nextup(vd0.back_lo[0]), bhi0 = vd0.back_hi[0];
    const float a2n = s_nextup(vd0.back_lo[1]), bhi1 = vd0.back_hi[1];
    const bool NFWD = vd0.nfwd > 0;
    const float fhi0 = NFWD ? vd0.fwd_hi[0] : 0.0f;
    const int tma = a.tma;
    const float NaN = __int_as_float(0x7fc00000);
    // unit's tau extent over its lanes (staging range)
    int32_t kEmin = u.elo >> 5, kEmax = (u.ehi - 1) >> 5;
    if (u.elo >= u.ehi) { kEmin = 1 << 20; kEmax = -(1 << 20); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kEmin = min(kEmin, __shfl_xor_sync(FULL, kEmin, o));
        kEmax = max(kEmax, __shfl_xor_sync(FULL, kEmax, o));
    }
    const int32_t hq = h >> 5, hr = h & 31;       // window offsets in words / bits
    const int32_t nsh = (32 - hr) & 31, nq = hr ? -hq - 1 : -hq;

    // ------------------------------------------------ pass 1 (ascending)
    // Far filter of view -b: SY = max over q <= i - 3 of A'(q) = s v(q) + (q -
    // base), base = the first position of the current group of 4 (A' shifted
    // by -4 per group).  Also the last candidates the windows need:
    // P window [tau0 + h - 32, tau0 + h - 1] (word k + hq - 1, shift hr), N
    // window [tau0 - h, tau0 + 31 - h] (word k + nq, shift nsh).
    {
        const int32_t kS = max(kB - nbr, kEmin);           // first staged block
        const int32_t kW = min(kS, kB - ((2 * h + 63) >> 5));
        int32_t pcl = NONE_LO, lc = NONE_LO;
        uint32_t pw_lo = s_word1(u, kW + hq - 1, 0), nw_lo = s_word1(u, kW + nq, 1);
        // words prefetched 3 blocks ahead (the first iterations only track windows)
        uint32_t pq0 = s_word1(u, kW + hq, 0), pq1 = s_word1(u, kW + 1 + hq, 0), pq2 = s_word1(u, kW + 2 + hq, 0);
        uint32_t nq0 = s_word1(u, kW + nq + 1, 1), nq1 = s_word1(u, kW + nq + 2, 1), nq2 = s_word1(u, kW + nq + 3, 1);
        float A1 = NaN, A2 = NaN, A3 = NaN, w1 = NaN, w2 = NaN, w3 = NaN, SY = -INFINITY, VM = NaN;
        uint32_t XN = 0u;
        int slot = 0;
        bool bt[2] = {false, false};
        if (kS <= kT) bt[0] = s_stage(u, tm, stg, bars, kS, tma);
        for (int32_t k = kW; k <= kT; ++k) {
            const uint32_t pw_hi = pq0, nw_hi = nq0;
            pq0 = pq1; pq1 = pq2; pq2 = s_word1(u, k + 3 + hq, 0);
            nq0 = nq1; nq1 = nq2; nq2 = s_word1(u, k + 3 + nq + 1, 1);
            const uint32_t WP = __funnelshift_r(pw_lo, pw_hi, hr);
            pw_lo = pw_hi;
            if (WP) pcl = 32 * k + h - 32 + 31 - __clz(WP);
            const uint32_t WN = __funnelshift_r(nw_lo, nw_hi, nsh);
            nw_lo = nw_hi;
            if (WN) lc = 32 * k - h + 31 - __clz(WN);
            if (k < kS) continue;
            s_stage_wait(bars + slot, phase[slot], bt[slot]);
            if (kNSlot == 2 && k + 1 <= kT) bt[slot ^ 1] = s_stage(u, tm, stg + (slot ^ 1) * kSlot, bars + (slot ^ 1), k + 1, tma);
            const float *rb = stg + slot * kSlot + rbo;
            float Q0 = NaN, Q2 = NaN;
            if (vN >= 0) {
#pragma unroll 1
                for (int g = 0; g < 8; ++g) {
                    SY = __fsub_rn(SY, 4.0f);
                    A1 = __fsub_rn(A1, 4.0f); A2 = __fsub_rn(A2, 4.0f); A3 = __fsub_rn(A3, 4.0f);
                    const float4 q4 = s_read4(rb, kind, g, sw);
                    const float vv[4] = {q4.x, q4.y, q4.z, q4.w};
                    float qa = NaN;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v0 = vv[e];
                        const float A0 = __fmaf_rn(fs_, v0, (float)e);
                        if (A3 > SY) { SY = A3; VM = w3; }
                        XN = s_push(XN, __fsub_rn(__fsub_rn(A0, T), SY));
                        if (e == 0) qa = VM;
                        A3 = A2; A2 = A1; A1 = A0;
                        w3 = w2; w2 = w1; w1 = v0;
                    }
                    if (g == 0) Q0 = qa;
                    if (g == 4) Q2 = qa;
                }
            }
            __syncwarp();
            if (kNSlot == 2) slot ^= 1;
            else if (k + 1 <= kT) bt[0] = s_stage(u, tm, stg, bars, k + 1, tma);
            if (k >= kB) {
                Rec rr;
                rr.XN = __brev(XN);
                rr.pclP = s_rel(pcl, 32 * k, h);
                rr.lcN = s_rel(lc, 32 * k, h);
                rr.VW = __floats2half2_rn(Q0, Q2);
                OCC_CHECK(k - kB < kMaxSegBlocks);
                rec[(k - kB) * 32 + lane] = rr;
            }
        }
    }

    // ------------------------------------------------ pass 2 (descending)
    uint8_t *MP = vP >= 0 ? a.masks + ((int64_t)f * a.nviews + vP) * a.mf.vbytes : nullptr;
    uint8_t *MN = vN >= 0 ? a.masks + ((int64_t)f * a.nviews + vN) * a.mf.vbytes : nullptr;
    {
        const int32_t kS = min(kT + nbr, kEmax);            // first staged block (from the top)
        const int32_t kW = max(kS, kT + 2 + ((2 * h + 31) >> 5));
        int32_t fc = NONE_HI, ncl = NONE_HI;
        uint32_t pw_hi = s_word1(u, kW + hq + 1, 0), nw_hi = s_word1(u, kW + nq + 1, 1);
        uint32_t pq0 = s_word1(u, kW + hq, 0), pq1 = s_word1(u, kW - 1 + hq, 0), pq2 = s_word1(u, kW - 2 + hq, 0);
        uint32_t nq0 = s_word1(u, kW + nq, 1), nq1 = s_word1(u, kW - 1 + nq, 1), nq2 = s_word1(u, kW - 2 + nq, 1);
        uint32_t WNprev = 0u, nw_hh = 0u;
        float v1 = NaN, v2 = NaN, v3 = NaN, A1 = NaN, A2 = NaN, A3 = NaN, SX = -INFINITY, VM = NaN;
        int slot = 0;
        bool bt[2] = {false, false};
        bt[0] = s_stage(u, tm, stg, bars, kS, tma);
        for (int32_t k = kW; k >= kB; --k) {
            const int32_t tau0 = 32 * k;
            const uint32_t pw_lo = pq0, nw_lo = nq0;
            pq0 = pq1; pq1 = pq2; pq2 = s_word1(u, k - 3 + hq, 0);
            nq0 = nq1; nq1 = nq2; nq2 = s_word1(u, k - 3 + nq, 1);
            const uint32_t WP = __funnelshift_r(pw_lo, pw_hi, hr);      // +b candidates [tau0 + h, tau0 + h + 31]
            const uint32_t rP2 = pw_hi;                                 // (small h: raw word of block k + 1)
            pw_hi = pw_lo;
            if (WP) fc = tau0 + h + __ffs(WP) - 1;
            const uint32_t WN = __funnelshift_r(nw_lo, nw_hi, nsh);     // -b candidates [tau0 - h, tau0 - h + 31]
            // raw candidate words of blocks k - 1, k, k + 1 (small h: hq = 0, nq = -1)
            const uint32_t rP0 = pq0, rP1 = pw_lo, rN0 = nw_lo, rN1 = nw_hi, rN2 = nw_hh;
            nw_hh = nw_hi;
            nw_hi = nw_lo;
            if (WNprev) ncl = tau0 + 32 - h + __ffs(WNprev) - 1;
            WNprev = WN;
            if (k > kS) continue;
            s_stage_wait(bars + slot, phase[slot], bt[slot]);
            if (kNSlot == 2 && k - 1 >= kB) bt[slot ^ 1] = s_stage(u, tm, stg + (slot ^ 1) * kSlot, bars + (slot ^ 1), k - 1, tma);
            const float *rb = stg + slot * kSlot + rbo;
            if (k > kT) {
                // warm-up: far filter of +b only
#pragma unroll 1
                for (int g = 7; g >= 0; --g) {
                    SX = __fsub_rn(SX, 4.0f);
                    A1 = __fsub_rn(A1, 4.0f); A2 = __fsub_rn(A2, 4.0f); A3 = __fsub_rn(A3, 4.0f);
                    const float4 q4 = s_read4(rb, kind, g, sw);
                    const float vv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                    for (int e = 3; e >= 0; --e) {
                        const float v0 = vv[e];
                        const float A0 = __fmaf_rn(fs_, v0, -(float)e);
                        if (A3 > SX) { SX = A3; VM = v3; }
                        A3 = A2; A2 = A1; A1 = A0;
                        v3 = v2; v2 = v1; v1 = v0;
                    }
                }
                __syncwarp();
                if (kNSlot == 2) slot ^= 1;
                else if (k - 1 >= kB) bt[0] = s_stage(u, tm, stg, bars, k - 1, tma);
                continue;
            }
            // tails for the pairs reaching below the block (d1 at tau0 - 1, d2 at tau0 - 1, tau0 - 2)
            const float vm1 = s_gv(u, tau0 - 1), vm2 = s_gv(u, tau0 - 2);
            uint32_t Xs1 = 0, Xg1 = 0, Xl1 = 0, Xlf = 0, Xs2 = 0, Xg2 = 0, Xl2 = 0, XFR = 0;
            float Q0 = NaN, Q1 = NaN, Q2 = NaN, Q3 = NaN;   // +b witness values after positions 7, 15, 23, 31
#pragma unroll 1
            for (int g = 7; g >= 0; --g) {
                SX = __fsub_rn(SX, 4.0f);
                A1 = __fsub_rn(A1, 4.0f); A2 = __fsub_rn(A2, 4.0f); A3 = __fsub_rn(A3, 4.0f);
                const float4 q4 = s_read4(rb, kind, g, sw);
                const float vv[4] = {q4.x, q4.y, q4.z, q4.w};
                float qa = NaN;
#pragma unroll
                for (int e = 3; e >= 0; --e) {
                    const float v0 = vv[e];
                    const float d1 = __fsub_rn(v1, v0), d2 = __fsub_rn(v2, v0);
                    const float e1 = fabsf(d1), e2 = fabsf(d2);
                    Xs1 = s_push(Xs1, d1);
                    Xg1 = s_push(Xg1, __fsub_rn(e1, a1n));
                    Xl1 = s_push(Xl1, __fsub_rn(e1, bhi0));
                    Xlf = s_push(Xlf, __fsub_rn(e1, fhi0));
                    Xs2 = s_push(Xs2, d2);
                    Xg2 = s_push(Xg2, __fsub_rn(e2, a2n));
                    Xl2 = s_push(Xl2, __fsub_rn(e2, bhi1));
                    const float A0 = __fmaf_rn(fs_, v0, -(float)e);
                    if (A3 > SX) { SX = A3; VM = v3; }
                    XFR = s_push(XFR, __fsub_rn(__fsub_rn(A0, T), SX));
                    if (e == 3) qa = VM;
                    A3 = A2; A2 = A1; A1 = A0;
                    v3 = v2; v2 = v1; v1 = v0;
                }
                if (g == 7) Q3 = qa;
                if (g == 5) Q2 = qa;
                if (g == 3) Q1 = qa;
                if (g == 1) Q0 = qa;
            }
            // v1 = v(tau0), v2 = v(tau0 + 1)
            const float d1m = __fsub_rn(v1, vm1), d2m1 = __fsub_rn(v2, vm1), d2m2 = __fsub_rn(v1, vm2);
            const uint32_t s1m = s_sgn(d1m), g1m = s_sgn(__fsub_rn(fabsf(d1m), a1n));
            const uint32_t t1m = (g1m ^ 1u) & s_sgn(__fsub_rn(fabsf(d1m), bhi0));
            const uint32_t tfm = NFWD ? ((g1m ^ 1u) & s_sgn(__fsub_rn(fabsf(d1m), fhi0))) : 0u;
            const uint32_t t2m1 = (s_sgn(__fsub_rn(fabsf(d2m1), a2n)) ^ 1u) & s_sgn(__fsub_rn(fabsf(d2m1), bhi1));
            const uint32_t t2m2 = (s_sgn(__fsub_rn(fabsf(d2m2), a2n)) ^ 1u) & s_sgn(__fsub_rn(fabsf(d2m2), bhi1));
            const uint32_t s2m1 = s_sgn(d2m1), s2m2 = s_sgn(d2m2);
            const uint32_t T1 = ~Xg1 & Xl1, T2 = ~Xg2 & Xl2, TF = NFWD ? (~Xg1 & Xlf) : 0u;
            const uint32_t ext = s_ge(u.elo - tau0) & s_le(u.ehi - 1 - tau0);
            OCC_CHECK(k >= kB && k - kB < kMaxSegBlocks);
            const Rec rr = rec[(k - kB) * 32 + lane];
            // view +b: pairs (i, i + j) covered <=> a +b candidate in [i + j - h, i + h]
            const int32_t pcl = tau0 + rr.pclP;
            uint32_t cP1, cP2, cP3, cPf, cN1, cN2, cN3, cNf;
            const int32_t lc = tau0 + rr.lcN;
            if (!smallh) {
                const uint32_t cPa = s_ge(fc - h - tau0);
                cP1 = cPa | s_le(pcl + h - 1 - tau0);
                cP2 = cPa | s_le(pcl + h - 2 - tau0);
                cP3 = cPa | s_le(pcl + h - 3 - tau0);
                cPf = s_ge(fc - h + 1 - tau0) | s_le(pcl + h - tau0);
                const uint32_t cNa = s_le(lc + h - tau0);
                cN1 = cNa | s_ge(ncl + 1 - h - tau0);
                cN2 = cNa | s_ge(ncl + 2 - h - tau0);
                cN3 = cNa | s_ge(ncl + 3 - h - tau0);
                cNf = s_le(lc + h - 1 - tau0) | s_ge(ncl - h - tau0);
            } else {
                // pair (a, b), a < b, covered <=> a candidate in [b - h, a + h]
                // (S8/S9): bit r of a window mask = OR of the block's
                // candidate bits over [r + lo, r + lo + w - 1]
                cP1 = s_dil(rP0, rP1, rP2, 2 * h, 32 + 1 - h);        // (i, i + j): [i + j - h, i + h]
                cP2 = s_dil(rP0, rP1, rP2, 2 * h - 1, 32 + 2 - h);
                cP3 = s_dil(rP0, rP1, rP2, 2 * h - 2, 32 + 3 - h);
                cPf = s_dil(rP0, rP1, rP2, 2 * h, 32 - h);            // (i - 1, i): [i - h, i - 1 + h]
                cN1 = s_dil(rN0, rN1, rN2, 2 * h, 32 - h);            // (i - j, i): [i - h, i - j + h]
                cN2 = s_dil(rN0, rN1, rN2, 2 * h - 1, 32 - h);
                cN3 = s_dil(rN0, rN1, rN2, 2 * h - 2, 32 - h);
                cNf = s_dil(rN0, rN1, rN2, 2 * h, 32 + 1 - h);        // (i, i + 1): [i + 1 - h, i + h]
            }
            uint32_t mP = ((T1 & ~Xs1) & cP1) | ((T2 & ~Xs2) & cP2);
            if (NFWD) mP |= (((TF & Xs1) << 1) | (tfm & s1m)) & cPf;
            mP &= ext;
            // view -b: pairs (i - j, i) covered <=> a -b candidate in [i - h, i - j + h]
            const uint32_t n1 = ((T1 & Xs1) << 1) | (t1m & s1m);
            const uint32_t n2 = ((T2 & Xs2) << 2) | ((t2m1 & s2m1) << 1) | (t2m2 & s2m2);
            uint32_t mN = (n1 & cN1) | (n2 & cN2);
            if (NFWD) mN |= (TF & ~Xs1) & cNf;
            mN &= ext;
            const uint32_t sP = vP >= 0 ? (XFR & cP3 & ~mP & ext) : 0u;
            const uint32_t sN = vN >= 0 ? (rr.XN & cN3 & ~mN & ext) : 0u;
            SST(0, __popc(ext));
            SST(1, __popc(sP));
            SST(2, __popc(sN));
            SST(10, __popc(mP));
            SST(11, __popc(mN));
            SST(13, lane == 0);
            if (__any_sync(FULL, (sP | sN) != 0u)) {
                SST(12, lane == 0);
                SurvCtx sc;
                sc.tau0 = tau0; sc.h = h; sc.WP = WP; sc.WN = WN; sc.pcl = pcl; sc.ncl = ncl;
                sc.Q0 = Q0; sc.Q1 = Q1; sc.Q2 = Q2; sc.Q3 = Q3; sc.VW = rr.VW;
                sc.fs = fs_; sc.s = s; sc.tlo = tlo; sc.thi = thi; sc.vP = vP; sc.vN = vN;
                s_resolve(a, u, stg + slot * kSlot, sc, sP, sN, mP, mN, reinterpret_cast<uint16_t *>(smem + kListOff),
                          reinterpret_cast<uint32_t *>(smem + kMarkOff));
            }
            __syncwarp();
            if (kNSlot == 2) slot ^= 1;
            else if (k - 1 >= kB) bt[0] = s_stage(u, tm, stg, bars, k - 1, tma);
            if constexpr (SHEAR) {
                if (vP >= 0) s_store_sh(u, a, MP, mP, k);
                if (vN >= 0) s_store_sh(u, a, MN, mN, k);
            } else {
                if (vP >= 0) s_store(u, MP, a.mf, mP, k);
                if (vN >= 0) s_store(u, MN, a.mf, mN, k);
            }
        }
    }
}

// grid: CTAs of kSweepWarps warps, one unit per warp.  Work order: frame
// groups of fgroup frames; inside a group the units of one kind segment
// after another (host order: diagonals, anti-diagonals, rows, columns;
// longest first inside a segment), each over the group's frames: the warps in flight work
// on a few frames, whose D and words stay in L2.
constexpr int kSweepWarps = 1;
// minimum CTAs per SM of the launch bounds: a code-generation knob (the
// kernel keeps 96 registers either way; 18 gives the smaller stack frame):
// C5 A/B on one B200, ms per 256 frames: 16 22.06, 17 20.18, 18 20.23,
// 19 20.66, 20 20.88, 22 / 24 (80 registers, spills) 22.8; after the merged
// diagonal words: 17 18.48, 18 18.67, 19 18.47, 20 18.56, 21 (80 registers) 20.56
#ifndef SWEEP_MINB
#define SWEEP_MINB 19
#endif
template <bool SHEAR>
__global__ void __launch_bounds__(32 * kSweepWarps, SWEEP_MINB) k_sweep(const __grid_constant__ SweepArgs a,
                                                                 const __grid_constant__ SweepMaps tm) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t wid = blockIdx.x * kSweepWarps + (threadIdx.x >> 5);
    if (wid >= (uint32_t)a.nunits * (uint32_t)a.frames) return;
    const uint32_t per_group = (uint32_t)a.nunits * (uint32_t)a.fgroup;
    const int32_t g = (int32_t)(wid / per_group);
    const int32_t f0 = g * a.fgroup, gf = min(a.fgroup, a.frames - f0);
    const int32_t rem = (int32_t)(wid - (uint32_t)g * per_group);
    int kk = 0;
    while (kk < 3 && rem >= a.kstart[kk + 1] * gf) ++kk;
    const int32_t ri = rem - a.kstart[kk] * gf;
    const SweepUnit un = a.units[a.kstart[kk] + ri / gf];
    const int32_t f = f0 + ri % gf;
    const GroupDesc gd = a.groups[un.group];
    unsigned char *sm = smem + (size_t)(threadIdx.x >> 5) * kSweepWarpSmem;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + kBarOff);
    if ((threadIdx.x & 31) == 0) {
        s_mbar_init(bars, 1);
        s_mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase[2] = {0u, 0u};
    sweep_unit<false, SHEAR>(a, tm, un, gd, f, sm, phase);
}

// The units of frames with 0 < h < 17 (the ones k_sweep skips): persistent
// warps walk the frames, and every (small-h frame, unit) pair is taken by one
// warp in turn.  smin = the smallest s of the sweep's groups (h grows with s).
template <bool SHEAR>
__global__ void __launch_bounds__(32, SWEEP_MINB) k_sweep_small(const __grid_constant__ SweepArgs a,
                                                       const __grid_constant__ SweepMaps tm, int32_t smin) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kBarOff);
    if ((threadIdx.x & 31) == 0) {
        s_mbar_init(bars, 1);
        s_mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase[2] = {0u, 0u};
    uint32_t item = 0;
    const int lane = threadIdx.x & 31;
    for (int32_t f32 = 0; f32 < a.frames; f32 += 32) {
        // the lanes test 32 frames at once; only small-h frames are walked
        bool small = false;
        if (f32 + lane < a.frames) {
            const FrameStats fl = a.st[f32 + lane];
            small = !fl.nonfinite && view_h(frame_range(fl), smin, a.p.max_scan) < 17;
        }
        for (uint32_t sm = __ballot_sync(FULL, small); sm; sm &= sm - 1u) {
            const int32_t f = f32 + __ffs(sm) - 1;
            const float R = frame_range(a.st[f]);
            // this warp's units of the frame: items item + i with (item + i) % grid == block
            const uint32_t G = gridDim.x;
            const uint32_t i0 = (blockIdx.x + G - item % G) % G;
            item += (uint32_t)a.nunits;
            for (uint32_t i = i0; i < (uint32_t)a.nunits; i += G) {
                const SweepUnit un = a.units[i];
                const GroupDesc gd = a.groups[un.group];
                const int32_t h = view_h(R, a.views[gd.view[0]].s, a.p.max_scan);
                if (h > 0 && h < 17) sweep_unit<true, SHEAR>(a, tm, un, gd, f, smem, phase);
            }
        }
    }
}

// host: TMA descriptors of the chunk's D ([frames][H][W] fp32)
static bool make_maps(const float *D, int32_t H, int32_t W, int32_t frames, SweepMaps &m) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    const cuuint32_t es[3] = {1, 1, 1};
    const cuuint32_t box32[3] = {32, 32, 1}, box1[3] = {32, 1, 1};
    void *g = const_cast<float *>(D);
    auto mk = [&](CUtensorMap *t, const cuuint32_t *box, CUtensorMapSwizzle swz) {
        return enc(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) ==
               CUDA_SUCCESS;
    };
    return mk(&m.rows, box32, CU_TENSOR_MAP_SWIZZLE_128B) && mk(&m.cols, box32, CU_TENSOR_MAP_SWIZZLE_NONE) &&
           mk(&m.run, box1, CU_TENSOR_MAP_SWIZZLE_NONE);
}

cudaError_t launch_sweep(const float *D, int32_t H, int32_t W, int32_t frames, const SweepUnit *units,
                         int32_t nunits, const GroupDesc *groups, const ViewDesc *views, int32_t nviews,
                         const FamilyDesc *fams, const FrameStats *st, const Params &p, uint8_t *masks,
                         const MaskFmt &mf, const uint32_t *words, HardEntry *gq, uint32_t *gq_count,
                         int32_t gq_cap, const int32_t *kstart, int32_t fgroup, unsigned long long *dbg,
                         int32_t smin_hint, const ShearDesc *sh, cudaStream_t s) {
    if (nunits <= 0 || frames <= 0) return cudaSuccess;
    SweepArgs a{};
    a.shkind = -1;
    if (sh) {
        a.shkind = sh->kind; a.sh_num = sh->num; a.sh_den = sh->den; a.sh_lmin = sh->lmin;
        a.Ho = sh->Ho; a.Wo = sh->Wo;
    }
    for (int k = 0; k < 5; ++k) a.kstart[k] = kstart[k];
    a.fgroup = fgroup;
    a.D = D; a.H = H; a.W = W; a.nxb = (W + 31) / 32; a.nyb = (H + 31) / 32;
    a.units = units; a.nunits = nunits; a.frames = frames;
    a.groups = groups; a.views = views; a.nviews = nviews; a.fams = fams; a.st = st; a.p = p;
    a.masks = masks; a.mf = mf; a.words = words; a.gq = gq; a.gq_count = gq_count; a.gq_cap = gq_cap;
    a.dbg = dbg;
    SweepMaps tm;
    memset(&tm, 0, sizeof(tm));
    static const bool no_tma = [] { const char *ev = getenv("OCC_NO_TMA"); return ev && atoi(ev) != 0; }();
    a.tma = (!no_tma && (W & 3) == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0 && make_maps(D, H, W, frames, tm))
                ? 1 : 0;
    const size_t smem = kSweepWarpSmem * kSweepWarps;
    auto kmain = sh ? k_sweep<true> : k_sweep<false>;
    auto ksmall = sh ? k_sweep_small<true> : k_sweep_small<false>;
    cudaError_t e = cudaFuncSetAttribute(kmain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(kmain, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int64_t nw = (int64_t)nunits * frames;
    kmain<<<(unsigned)((nw + kSweepWarps - 1) / kSweepWarps), 32 * kSweepWarps, smem, s>>>(a, tm);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // units of frames with h < 17 (data dependent: known on the device only)
    const int32_t smin = std::max(1, smin_hint);
    e = cudaFuncSetAttribute(ksmall, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepWarpSmem);
    if (e != cudaSuccess) return e;
    // one resident wave of 1-warp CTAs (148 SMs x SWEEP_MINB)
    ksmall<<<(unsigned)std::min<int64_t>(nw, 148 * SWEEP_MINB), 32, kSweepWarpSmem, s>>>(a, tm, smin);
    return cudaGetLastError();
}

// ================================================================ k_shear
// Knight baselines ((2, +-1), (1, +-2)): their digital lines (S6, reading
// Q8: l = y - floor(x by / bx), x-major; l = x - floor(y bx / by), y-major)
// are not arithmetic progressions in memory.  k_shear copies D into a
// sheared frame whose rows (x-major) or columns (y-major) ARE the family's
// lines -- Ds[l'][x] = D[l' + lmin + f(x)][x] or Ds[y][l'] = D[y][l' + lmin +
// f(y)], f(t) = floor(t num / den), NaN outside the image (a NaN sample
// never pairs and is never a candidate: the dropped samples of reading Q10)
// -- and writes the family's Eq. 1-2 candidate bits (PAPER.md:92-109,
// computed on the image's own neighbours) in the k_words layout of sweep
// kind 0 (rows) or 1 (columns) of that frame.  k_sweep then runs the family
// as rows / columns and un-shears its mask stores (s_store_sh).
struct ShearArgs {
    const float *D;
    int32_t H, W;              // image
    int32_t Hs, Ws, nxb, nyb;  // sheared frame and its 32 x 32 blocks
    int32_t xmajor, num, den, lmin, b0x, b0y;
    float e2_thresh;
    float *Ds;
    uint32_t *words;           // [frame][nyb][nxb][12][32] (slots 0, 1 or 2, 3 used)
};
__global__ void __launch_bounds__(128) k_shear(ShearArgs a) {
    __shared__ uint2 rw[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t kx = blockIdx.x * 4 + warp, m = blockIdx.y, f = blockIdx.z;
    const bool wok = kx < a.nxb;
    const float NaN = __int_as_float(0x7fc00000);
    const float *Df = a.D + (int64_t)f * a.H * a.W;
    float *Dsf = a.Ds + (int64_t)f * a.Hs * a.Ws;
    const int32_t col = 32 * kx + lane;
    for (int r = 0; r < 32; ++r) {
        const int32_t row = 32 * m + r;
        const bool ins = wok && col < a.Ws && row < a.Hs;
        int32_t x, y;
        if (a.xmajor) { x = col; y = row + a.lmin + ((col * a.num) >> 1); }
        else { y = row; x = col + a.lmin + ((row * a.num) >> 1); }
        const bool in = ins && (uint32_t)x < (uint32_t)a.W && (uint32_t)y < (uint32_t)a.H;
        const float v = in ? __ldg(Df + (int64_t)y * a.W + x) : NaN;
        if (ins) Dsf[(int64_t)row * a.Ws + col] = v;
        const bool hr = in && x + 1 < a.W, hb = in && y + 1 < a.H;
        const float right = hr ? __ldg(Df + (int64_t)y * a.W + x + 1) : 0.0f;
        const float below = hb ? __ldg(Df + (int64_t)(y + 1) * a.W + x) : 0.0f;
        // Eq. 1 (reading Q1) and the exact E^2 threshold (Q4), as k_words
        const float ex = hr ? __fsub_rn(right, v) : 0.0f;
        const float ey = hb ? __fsub_rn(below, v) : 0.0f;
        const float e2 = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey));
        const bool edge = in && e2 > a.e2_thresh;
        // Eq. 2 <=> b0 . (E_x, E_y) > 0, exact sign: components in {1, 2}
        // make both fp32 products exact unless they overflow (then binary64)
        const float px = __fmul_rn((float)a.b0x, ex), py = __fmul_rn((float)a.b0y, ey);
        bool pos, neg;
        if (isfinite(px) && isfinite(py)) {
            const float dot = __fadd_rn(px, py);
            pos = dot > 0.0f; neg = dot < 0.0f;
        } else {
            const double dot = __dadd_rn(__dmul_rn((double)a.b0x, (double)ex), __dmul_rn((double)a.b0y, (double)ey));
            pos = dot > 0.0; neg = dot < 0.0;
        }
        const uint32_t bp = __ballot_sync(FULL, edge && pos), bn = __ballot_sync(FULL, edge && neg);
        if (lane == 0) rw[warp][r] = make_uint2(bp, bn);
    }
    __syncwarp();
    const uint2 q = rw[warp][lane];
    if (!wok) return;
    uint32_t *dst = a.words + (((int64_t)f * a.nyb + m) * (a.nxb + 1) + kx) * kWordSlots * 32 + lane;
    if (a.xmajor) {          // kind 0: lane = line (row of the block), bit = position (column)
        dst[0] = q.x;
        dst[32] = q.y;
    } else {                 // kind 1: lane = line (column), bit = position (row)
        dst[64] = s_transpose32(q.x, lane);
        dst[96] = s_transpose32(q.y, lane);
    }
}

cudaError_t launch_shear(const float *D, int32_t H, int32_t W, int32_t frames, const ShearDesc &sh, int32_t Hs,
                         int32_t Ws, int32_t b0x, int32_t b0y, float e2_thresh, float *Ds, uint32_t *words,
                         cudaStream_t s) {
    ShearArgs a{D, H, W, Hs, Ws, (Ws + 31) / 32, (Hs + 31) / 32, sh.kind == 0 ? 1 : 0, sh.num, sh.den, sh.lmin,
                b0x, b0y, e2_thresh, Ds, words};
    dim3 grid((unsigned)((a.nxb + 3) / 4), (unsigned)a.nyb, (unsigned)frames);
    k_shear<<<grid, 128, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace occ
