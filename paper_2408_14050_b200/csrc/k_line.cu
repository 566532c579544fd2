#include <algorithm>
#include <cstdlib>
// k_line.cu -- K2, the line-sweep kernel for the four line families of
// |b| <= 1 camera arrays (rows, columns, diagonals, anti-diagonals): Eqs. 1-6
// for a pair of views +-b of one family.
//
// One warp = one work unit: 32 consecutive digital epipolar lines (SURVEY
// §8.0 S6; lane = line) x a segment of up to kLineSeg positions, one frame.
// Every lane works in its own "time" coordinate tau = pos + off(lane)
// (off = 0 for rows/columns, lane for diagonals, 31 - lane for
// anti-diagonals) so that at every tau the 32 lanes read one coalesced run of
// one image row (diagonals) or one row/column segment; all bit words below
// are indexed by tau (bit r of block k <-> tau = 32k + r).
//
//  pass 0  candidate words (Eqs. 1-2, from K0's per-pixel codes) of both
//          views for the segment +- (h + 32) positions, into shared memory.
//  pass A  descending tau.  Per position: the shared Eq. 5 near tests of
//          both views -- delta1 = fl(v[i+1] - v[i]) and delta2 = fl(v[i+2] -
//          v[i]) against the exact fp32 interval bounds, reduced to sign bits
//          of |delta| - bound and the sign of delta (view +b uses delta > 0,
//          view -b delta < 0) -- and the far-partner filter of view +b (suffix
//          max of A = s v - pos over q >= i + 3).  Per 32 positions: window
//          coverage of both views as two threshold masks (previous / next
//          candidate), the near marks, the far survivors and
//          one probe each, the +b mask store; the -b near marks are parked in
//          shared memory.
//  pass B  ascending tau: far filter of view -b (prefix max of s v + pos),
//          its survivors' probes, the -b mask store.
// Far survivors (filter passed, no near mark, dcov >= 3) get one branch-free
// exact probe (fp32 with a 2^-10 band) at the partner offset guessed from the
// filter's witness; the rest are queued (8-byte entries) for k_hard, which
// searches them exhaustively with one thread each after the kernel.  D is
// staged per warp one chunk of 32 positions x 32 lines at a time (cp.async,
// coalesced, 33-float pitch); probes read global memory (L1 / L2).
//
// Frames the kernel cannot serve with this scheme (h < 17 or h + 32 beyond
// the candidate margin) are computed by the exact per-pixel
// routine (direct_pixel) inside the same warp.
#include <cstdlib>

#include "occ_device.cuh"

#ifndef SWEEP_UNROLL
#define SWEEP_UNROLL 4
#endif

namespace occ {

namespace {
constexpr int kSweepUnroll = SWEEP_UNROLL;      // sweep / probe loops
constexpr int SEGB = kLineSeg / 32;            // blocks per segment
constexpr int CMW = kLineCandMarginWords;       // candidate margin words per side
constexpr int NCW = SEGB + 2 * CMW;             // candidate words per view
constexpr size_t OFF_CW = 0;
constexpr size_t OFF_NN = OFF_CW + sizeof(uint32_t) * 2 * NCW * 32;
#ifndef LINE_QCAP
#define LINE_QCAP 128
#endif
#ifndef LINE_SAB8
#define LINE_SAB8 0
#endif
#if LINE_SAB8
typedef uint8_t SabT;                           // partner guesses saturated at 255
#define SAB_MAX 255
#else
typedef int16_t SabT;
#define SAB_MAX 30000
#endif
constexpr int QCAP = LINE_QCAP;                 // deferred hard survivors per warp
constexpr size_t OFF_Q = OFF_NN + sizeof(uint32_t) * SEGB * 32;
constexpr size_t OFF_SAB = OFF_Q + sizeof(int32_t) * 2 * QCAP;
constexpr int SP = 33;                          // staging pitch (floats per position)
constexpr size_t OFF_STG = (OFF_SAB + sizeof(SabT) * 32 * 32 + 15) & ~(size_t)15;
#ifndef LINE_ONE_SLOT
#define LINE_ONE_SLOT 1      // one staging slot: smem 12.4 KB per warp, 16 warps per SM (C5 33.2 -> 28.8 ms per step)
#endif
constexpr size_t WSMEM = OFF_STG + sizeof(float) * (LINE_ONE_SLOT ? 1 : 2) * 32 * SP;
constexpr uint32_t FULL = 0xffffffffu;
constexpr int32_t NONE_LO = -(1 << 28), NONE_HI = (1 << 28);
}  // namespace

size_t line_smem_bytes() { return WSMEM; }

// ------------------------------------------------------------ small helpers
__device__ __forceinline__ uint32_t ge_mask(int32_t a) {      // bits r >= a
    return a <= 0 ? FULL : (a >= 32 ? 0u : (FULL << a));
}
__device__ __forceinline__ uint32_t le_mask(int32_t b) {      // bits r <= b
    return b < 0 ? 0u : (b >= 31 ? FULL : ((2u << b) - 1u));
}
// sign bit of x appended to w (w << 1 | sign(x))
__device__ __forceinline__ uint32_t push(uint32_t w, float x) {
    return __funnelshift_l(__float_as_uint(x), w, 1);
}
__device__ __forceinline__ uint32_t sgnbit(float x) { return __float_as_uint(x) >> 31; }
// smallest float > a (finite a): x > a <=> x >= nextup(a) <=> !(fl(x - nextup(a)) < 0)
__device__ __forceinline__ float nextup_f(float a) {
    const int32_t b = __float_as_int(a);
    if (a == 0.0f) return __int_as_float(1);
    return __int_as_float(a > 0.0f ? b + 1 : b - 1);
}
__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// 32x32 bit transpose across the warp: returns, for lane j, the word whose
// bit l is bit j of lane l's input.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
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
// 4 mask bits -> 4 bytes 0/1
__device__ __forceinline__ uint32_t expand4(uint32_t b4) { return (b4 * 0x00204081u) & 0x01010101u; }

// per-CTA phase timers (debug statistics only)
#ifdef OCC_LINE_STATS
#define OCC_PH_T0(v) const long long v = clock64()
#define OCC_PH_T1(c, i, v) do { if ((c).ph && ((c).lane == 0)) (c).ph[i] += (unsigned long long)(clock64() - (v)); } while (0)
#else
#define OCC_PH_T0(v) do { } while (0)
#define OCC_PH_T1(c, i, v) do { } while (0)
#endif

// warp-aggregated event counter (debug statistics only)
__device__ __forceinline__ void dbg_add(unsigned long long *dbg, int idx, uint32_t n) {
#ifndef OCC_LINE_STATS
    return;
#endif
    if (!dbg) return;
    const uint32_t tot = __reduce_add_sync(__activemask(), n);
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && tot) atomicAdd(dbg + idx, (unsigned long long)tot);
}

// ------------------------------------------------------------ line geometry
// KIND 0 rows (line y, pos x), 1 columns (line x, pos y), 2 diagonals
// (x-major, line y - x, pos x), 3 anti-diagonals (x-major, line y + x, pos x).
template <int KIND>
struct LG {
    // pixel of lane l (line l0 + l) at time tau
    static __device__ __forceinline__ void px(int32_t l0, int32_t l, int32_t tau, int32_t &x, int32_t &y) {
        if (KIND == 0) { x = tau; y = l0 + l; }
        else if (KIND == 1) { x = l0 + l; y = tau; }
        else if (KIND == 2) { x = tau - l; y = l0 + tau; }
        else { x = tau - 31 + l; y = l0 + 31 - tau; }
    }
    // in-image extent of lane l in tau: [lo, hi) (lo >= hi when empty)
    static __device__ __forceinline__ void ext(int32_t l0, int32_t l, int32_t H, int32_t W,
                                               int32_t &lo, int32_t &hi) {
        const int32_t L = l0 + l;
        if (KIND == 0) { lo = 0; hi = (L >= 0 && L < H) ? W : 0; }
        else if (KIND == 1) { lo = 0; hi = (L >= 0 && L < W) ? H : 0; }
        else if (KIND == 2) {
            const int32_t a = max(0, -L), b = min(W, H - L);
            lo = a + l; hi = max(a, b) + l;
        } else {
            const int32_t a = max(0, L - H + 1), b = min(W, L + 1);
            lo = a + 31 - l; hi = max(a, b) + 31 - l;
        }
    }
};

// Every digital line is an arithmetic progression in memory: pixel index of
// line l0 + l at time tau = base(l) + tau * stride.
__device__ __forceinline__ int64_t line_base(int kind, int32_t l0, int32_t l, int32_t W) {
    if (kind == 0) return (int64_t)(l0 + l) * W;
    if (kind == 1) return (int64_t)(l0 + l);
    if (kind == 2) return (int64_t)l0 * W - l;
    return (int64_t)(l0 + 31) * W - 31 + l;
}
__device__ __forceinline__ int32_t line_stride(int kind, int32_t W) {
    return kind == 0 ? 1 : (kind == 1 ? W : (kind == 2 ? W + 1 : 1 - W));
}

// runtime forms (the kind is warp-uniform: one code path for all families)
__device__ __forceinline__ void lg_px(int kind, int32_t l0, int32_t l, int32_t tau, int32_t &x, int32_t &y) {
    if (kind == 0) { x = tau; y = l0 + l; }
    else if (kind == 1) { x = l0 + l; y = tau; }
    else if (kind == 2) { x = tau - l; y = l0 + tau; }
    else { x = tau - 31 + l; y = l0 + 31 - tau; }
}
__device__ __forceinline__ void lg_ext(int kind, int32_t l0, int32_t l, int32_t H, int32_t W, int32_t &lo,
                                       int32_t &hi) {
    if (kind == 0) LG<0>::ext(l0, l, H, W, lo, hi);
    else if (kind == 1) LG<1>::ext(l0, l, H, W, lo, hi);
    else if (kind == 2) LG<2>::ext(l0, l, H, W, lo, hi);
    else LG<3>::ext(l0, l, H, W, lo, hi);
}

// ------------------------------------------------------------ candidate words
// cw: one view's words [NCW][32] for tau blocks WB .. WB + NCW - 1.
// Largest candidate tau <= x with tau >= lo (NONE_LO if none).
__device__ __forceinline__ int32_t prev_cand(const uint32_t *cw, int32_t x, int32_t lo, int32_t WB, int lane) {
    int32_t w = (x >> 5) - WB;
    uint32_t m;
    if (w >= NCW) { w = NCW - 1; m = cw[w * 32 + lane]; }
    else if (w < 0) return NONE_LO;
    else m = cw[w * 32 + lane] & le_mask(x & 31);
    const int32_t wlo = max((lo >> 5) - WB, 0);
    while (!m) {
        if (--w < wlo) return NONE_LO;
        m = cw[w * 32 + lane];
    }
    const int32_t c = (WB + w) * 32 + 31 - __clz(m);
    return c >= lo ? c : NONE_LO;
}
// Smallest candidate tau >= x with tau <= hi (NONE_HI if none).
__device__ __forceinline__ int32_t next_cand(const uint32_t *cw, int32_t x, int32_t hi, int32_t WB, int lane) {
    int32_t w = (x >> 5) - WB;
    uint32_t m;
    if (w < 0) { w = 0; m = cw[lane]; }
    else if (w >= NCW) return NONE_HI;
    else m = cw[w * 32 + lane] & ge_mask(x & 31);
    const int32_t whi = min((hi >> 5) - WB, NCW - 1);
    while (!m) {
        if (++w > whi) return NONE_HI;
        m = cw[w * 32 + lane];
    }
    const int32_t c = (WB + w) * 32 + __ffs(m) - 1;
    return c <= hi ? c : NONE_HI;
}

struct LineArgs {
    const float *D;
    int32_t H, W;
    const LineUnit *units;
    const GroupDesc *groups;
    const ViewDesc *views;
    int32_t nviews;
    const FamilyDesc *fams;
    const FrameStats *st;
    Params p;
    uint8_t *masks;
    const void *codes;
    unsigned long long *dbg;   // optional event counters (occ_debug_line_stats), or null
    int32_t frames;
    HardEntry *gq;             // global queue of exhaustive searches (k_hard), capacity gq_cap
    uint32_t *gq_count;
    int32_t gq_cap;
    int32_t nwork;             // units x frames
    MaskFmt mf;
    int32_t frame_major;       // work order: 0 frames fastest, 1 units fastest (frame-major)
    const uint32_t *cand;      // k_cand's candidate words for the chunk, or null (pass 0 from codes)
    const CandFam *candfam;    // per family (indexed by family), slot descriptors
};

// Per-warp context
struct Ctx {
    unsigned long long *dbg;
    unsigned long long *ph;    // per-CTA phase timers (debug) or null
    int32_t kind;              // line family (0 rows, 1 columns, 2 diagonals, 3 anti-diagonals)
    const float *Df;
    int32_t H, W, l0, lane;
    int32_t elo, ehi;          // lane's extent in tau
    const float *Dl;           // lane's line: v(tau) = Dl[tau * S]
    bool vec4;                 // rows with 16-byte aligned rows (float4 loads)
    int64_t B;                 // lane's line: pixel index = B + tau * S
    int32_t S;
    int32_t f;                 // frame
    MaskFmt mf;
    HardEntry *gq;
    uint32_t *gq_count;
    int32_t gq_cap;
};

__device__ __forceinline__ float gload(const Ctx &c, int32_t l, int32_t tau) {
    const int64_t b = l == c.lane ? c.B : line_base(c.kind, c.l0, l, c.W);
    return __ldg(c.Df + b + (int64_t)tau * c.S);
}

// Stages chunk k (tau = 32k .. 32k + 31 of the warp's 32 lines) into st
// [position][lane] with cp.async, one coalesced run per instruction; NaN
// outside the image.
__device__ __noinline__ void stage_chunk(const Ctx &c, float *st, int32_t k) {
    const float NaN = __int_as_float(0x7fc00000);
    const int lane = c.lane;
    const int32_t t0 = 32 * k;
    const float *src;
    float *dst;
    int64_t step;
    int32_t dstep, jlo, jhi;
    if (c.kind == 0) {
        // rows: lane = position, one coalesced row segment per line j
        const int32_t x = t0 + lane;
        src = c.Df + (int64_t)c.l0 * c.W + x;
        step = c.W;
        dst = st + lane * SP;
        dstep = 1;
        jlo = 0;
        jhi = (x >= 0 && x < c.W) ? min(32, c.H - c.l0) : 0;
    } else {
        // lane = line: one coalesced run per tau
        src = c.Dl + (int64_t)t0 * c.S;
        step = c.S;
        dst = st + lane;
        dstep = SP;
        jlo = c.elo - t0;
        jhi = c.ehi - t0;
    }
    if (__all_sync(FULL, jlo <= 0 && jhi >= 32)) {
        // interior chunk: 32 unconditional copies, 32-bit offsets
        const int32_t st32 = (int32_t)step;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) cp_async4(dst + j * dstep, src + j * st32);
        return;
    }
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        if (j >= jlo && j < jhi) cp_async4(dst + j * dstep, src + (int64_t)j * step);
        else dst[j * dstep] = NaN;
    }
}

// value of the lane's line at tau (NaN outside the image)
__device__ __forceinline__ float gv(const Ctx &c, int32_t tau) {
    return (tau >= c.elo && tau < c.ehi) ? __ldg(c.Dl + (int64_t)tau * c.S) : __int_as_float(0x7fc00000);
}
// values at tau .. tau + 3 (tau multiple of 4); `inside`: all four are in the image
__device__ __forceinline__ float4 load4(const Ctx &c, int32_t tau, bool inside) {
    if (inside) {
        if (c.vec4) return __ldg(reinterpret_cast<const float4 *>(c.Dl + tau));
        const float *q = c.Dl + (int64_t)tau * c.S;
        return make_float4(__ldg(q), __ldg(q + c.S), __ldg(q + 2 * c.S), __ldg(q + 3 * c.S));
    }
    return make_float4(gv(c, tau), gv(c, tau + 1), gv(c, tau + 2), gv(c, tau + 3));
}

template <int CB>
__device__ __forceinline__ uint32_t code_at(const void *codes, int64_t idx) {
    if (CB == 1) return __ldg(reinterpret_cast<const uint8_t *>(codes) + idx);
    if (CB == 2) return __ldg(reinterpret_cast<const uint16_t *>(codes) + idx);
    return __ldg(reinterpret_cast<const uint32_t *>(codes) + idx);
}

// Candidate words of both views (bits cb and cb + 1 of the codes) for the 32
// positions t0 .. t0 + 31 of the lane's line: bit r <-> tau = t0 + r.
template <int CB>
__device__ __forceinline__ void cand_word(const Ctx &c, const void *codesf, int32_t cb, int32_t t0,
                                          uint32_t &wp, uint32_t &wn) {
    const int lane = c.lane;
    wp = 0u;
    wn = 0u;
    if (!(t0 + 31 >= c.elo && t0 < c.ehi)) return;
    if (c.kind == 0 && CB == 1 && (c.W & 15) == 0 && t0 >= 0 && t0 + 32 <= c.W) {
        // rows: 32 consecutive codes of the lane's row in two 16-byte loads
        const uint8_t *row = reinterpret_cast<const uint8_t *>(codesf) + (int64_t)(c.l0 + lane) * c.W + t0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(row + 16 * hh));
            const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t tp = (u[e] >> cb) & 0x01010101u;
                const uint32_t tn = (u[e] >> (cb + 1)) & 0x01010101u;
                wp |= ((tp * 0x10204080u) >> 28) << (16 * hh + 4 * e);
                wn |= ((tn * 0x10204080u) >> 28) << (16 * hh + 4 * e);
            }
        }
    } else if (t0 >= c.elo && t0 + 32 <= c.ehi) {
        const int64_t i0 = c.B + (int64_t)t0 * c.S;
#pragma unroll 8
        for (int j = 31; j >= 0; --j) {
            const uint32_t code = code_at<CB>(codesf, i0 + (int64_t)j * c.S) >> cb;
            wp = (wp << 1) | (code & 1u);
            wn = (wn << 1) | ((code >> 1) & 1u);
        }
    } else {
        for (int j = 31; j >= 0; --j) {
            const int32_t tau = t0 + j;
            uint32_t code = 0u;
            if (tau >= c.elo && tau < c.ehi) code = code_at<CB>(codesf, c.B + (int64_t)tau * c.S) >> cb;
            wp = (wp << 1) | (code & 1u);
            wn = (wn << 1) | ((code >> 1) & 1u);
        }
    }
}

// pass 0: candidate words of both views (bit cb and cb + 1 of the codes)
template <int CB>
__device__ __noinline__ void build_cand(const Ctx &c, const void *codesf, int32_t cb, int32_t WB,
                                           uint32_t *cw, int32_t wlo, int32_t whi) {
    const int lane = c.lane;
    for (int w = 0; w < NCW; ++w) {
        uint32_t wp = 0u, wn = 0u;
        if (w >= wlo && w <= whi) cand_word<CB>(c, codesf, cb, 32 * (WB + w), wp, wn);
        cw[(0 * NCW + w) * 32 + lane] = wp;
        cw[(1 * NCW + w) * 32 + lane] = wn;
    }
}

// pass 0 from the words k_cand precomputed for the whole chunk (no margin
// recomputation between neighbouring units)
__device__ __noinline__ void load_cand(const Ctx &c, const uint32_t *cand, const CandFam &cf, int32_t WB,
                                       uint32_t *cw, int32_t wlo, int32_t whi) {
    const int lane = c.lane;
    const int32_t lb = (c.l0 - cf.lmin) >> 5;
    const uint32_t *base = cand + (((int64_t)c.f * cf.per_frame + cf.base_slot + (int64_t)lb * cf.nk) << 6);
    for (int w = 0; w < NCW; ++w) {
        const int32_t k = WB + w - cf.kmin;
        uint32_t wp = 0u, wn = 0u;
        if (w >= wlo && w <= whi && k >= 0 && k < cf.nk) {
            wp = __ldg(base + ((int64_t)k << 6) + lane);
            wn = __ldg(base + ((int64_t)k << 6) + 32 + lane);
        }
        cw[(0 * NCW + w) * 32 + lane] = wp;
        cw[(1 * NCW + w) * 32 + lane] = wn;
    }
}

// Window coverage of view +b for the 32 positions tau0 + r (SURVEY App. A.2,
// h >= 17): covered_k(i) <=> a candidate lies in [i + k - h, i + h]
//   = [i >= fc - h] or [i <= pcl + h - k],
// fc = first candidate >= tau0 + h, pcl = last candidate <= tau0 + h - 1.
struct CovP { int32_t fc, pcl; };
__device__ __forceinline__ CovP cov_p(const uint32_t *cw, int32_t tau0, int32_t h, int32_t WB, int lane) {
    CovP r;
    r.fc = next_cand(cw, tau0 + h, tau0 + 31 + h, WB, lane);
    r.pcl = prev_cand(cw, tau0 + h - 1, tau0 - h, WB, lane);
    return r;
}
__device__ __forceinline__ uint32_t cov_p_k(const CovP &v, int32_t tau0, int32_t h, int32_t k) {
    return ge_mask(v.fc - h - tau0) | le_mask(v.pcl + h - k - tau0);
}
// forward pair (i - 1, i): covered_1(i - 1)
__device__ __forceinline__ uint32_t cov_p_f(const CovP &v, int32_t tau0, int32_t h) {
    return ge_mask(v.fc - h + 1 - tau0) | le_mask(v.pcl + h - tau0);
}
// view -b (backward = lower tau): covered_k(i) <=> candidate in [i - h, i - k + h]
//   = [i <= lc + h] or [i >= ncl + k - h],
// lc = last candidate <= tau0 + 31 - h, ncl = first candidate >= tau0 + 32 - h.
struct CovN { int32_t lc, ncl; };
__device__ __forceinline__ CovN cov_n(const uint32_t *cw, int32_t tau0, int32_t h, int32_t WB, int lane) {
    CovN r;
    r.lc = prev_cand(cw, tau0 + 31 - h, tau0 - h, WB, lane);
    r.ncl = next_cand(cw, tau0 + 32 - h, tau0 + 31 + h, WB, lane);
    return r;
}
__device__ __forceinline__ uint32_t cov_n_k(const CovN &v, int32_t tau0, int32_t h, int32_t k) {
    return le_mask(v.lc + h - tau0) | ge_mask(v.ncl + k - h - tau0);
}
// forward pair (i, i + 1): covered_1(i + 1)
__device__ __forceinline__ uint32_t cov_n_f(const CovN &v, int32_t tau0, int32_t h) {
    return le_mask(v.lc + h - 1 - tau0) | ge_mask(v.ncl - h - tau0);
}

struct ViewK {
    int32_t s, h;
    float fs;              // (float)s
    float T;               // far-filter margin
    float tlo, thi;        // t_dist -+ 2^-10: fp32 fast path of the exact Eq. 5 test
};

// Per-block context of the far-survivor resolution.
struct Blk {
    int32_t tau0;          // block start
    uint32_t Wc;           // candidate bits of [tau0 + h, +31] (+b) / [tau0 - h, +31] (-b)
    int32_t cfall;         // last candidate < tau0 + h (+b) / first candidate >= tau0 + 32 - h (-b)
    const float *cb;       // the block's staged values, lane column ([r * SP])
    const SabT *sab;       // partner guess of each survivor ([r][lane])
    int32_t T0;
};

// value of line l at tau (L1 / L2); NaN outside the line
__device__ __forceinline__ float probe_b(const Ctx &c, const Blk &b, int32_t l, int32_t tau, int32_t elo,
                                         int32_t ehi) {
    if (tau < elo || tau >= ehi) return __int_as_float(0x7fc00000);
    return gload(c, l, tau);
}
// dcov of the survivor at tau0 + r (largest far offset sharing a scan window, App. A.2)
__device__ __forceinline__ int32_t dcov_of(const int DIR, uint32_t Wc, int32_t cfall, int32_t tau0, int32_t r, int32_t h) {
    if (DIR > 0) {
        const uint32_t m = Wc & le_mask(r);
        const int32_t pc = m ? tau0 + h + 31 - __clz(m) : cfall;
        return pc + h - (tau0 + r);
    }
    const uint32_t m = Wc & ge_mask(r);
    const int32_t nc = m ? tau0 - h + __ffs(m) - 1 : cfall;
    return tau0 + r + h - nc;
}
// Eq. 5 for a far pair (offset j >= jstar, so delta > t_disp is implied):
// |s fl(vq - vp) - j| < t_dist.  s delta is exact; one rounding in the fma,
// far below the 2^-10 band; inside the band the binary64 test decides.
__device__ __noinline__ bool pair_exact_slow(float vq, float vp, int32_t j, int32_t s, float t_dist,
                                             float t_disp) {
    return pair_exact(vq, vp, -j, s, t_dist, t_disp);
}
__device__ __forceinline__ bool pair_far(float vq, float vp, int32_t j, const ViewK &vk, const Params &p) {
    const float d = __fsub_rn(vq, vp);
    const float x = fabsf(__fmaf_rn(vk.fs, d, -(float)j));
    if (x < vk.tlo) return true;
    if (!(x <= vk.thi)) return false;
    return pair_exact_slow(vq, vp, j, vk.s, p.t_dist, p.t_disp);
}

// Deferred exhaustive searches: one lane per queued survivor (tau, dcov,
// line), scanning offsets 3..dcov of its line in global memory (L2) with 16
// loads in flight; a confirmed Eq. 5 pair sets the mask byte directly (the
// block store already wrote 0 there).
__device__ __noinline__ void flush_queue(const int DIR, const Ctx &c, const int32_t *qbuf, int32_t qn, const ViewK &vk,
                                         const Params &p, uint8_t *Mv, int32_t vid) {
    OCC_PH_T0(tph);
    __syncwarp();
    const float NaN = __int_as_float(0x7fc00000);
    // normally the searches go to the global queue, resolved after this
    // kernel by k_hard with the whole GPU (no single warp carries a heavy unit)
    // The entries that fit below the capacity are always written (k_hard
    // reads slots [0, min(count, cap)), so every one of them must hold an
    // entry of this chunk); a reservation straddling the capacity resolves
    // only its remainder here.
    int32_t done = 0;
    if (c.gq && qn > 0) {
        uint32_t base = 0u;
        if (c.lane == 0) base = atomicAdd(c.gq_count, (uint32_t)qn);
        base = __shfl_sync(FULL, base, 0);
        const int32_t fit = base >= (uint32_t)c.gq_cap ? 0 : (int32_t)min((uint32_t)qn, (uint32_t)c.gq_cap - base);
        for (int32_t e = c.lane; e < fit; e += 32) {
            const int32_t tau = qbuf[2 * e], w = qbuf[2 * e + 1];
            const int32_t src = w & 31, jm = (w >> 5) & 0x1FFFF;
            HardEntry he;
            he.pix = (int32_t)(line_base(c.kind, c.l0, src, c.W) + (int64_t)tau * c.S);
            he.meta = (uint32_t)jm | ((uint32_t)vid << 25);
            he.guess = c.f << 17;
            he.vq = 0.0f;
            c.gq[base + (uint32_t)e] = he;
        }
        __syncwarp();
        done = fit;
        if (fit == qn) {
            OCC_PH_T1(c, 1, tph);
            return;
        }
    }
    for (int32_t e0 = done; e0 < qn; e0 += 32) {
        const int32_t e = e0 + c.lane;
        if (e < qn) {
            const int32_t tau = qbuf[2 * e], w = qbuf[2 * e + 1];
            const int32_t src = w & 31, jm = (w >> 5) & 0x1FFFF;
            const float *Ds = c.Df + line_base(c.kind, c.l0, src, c.W) + (int64_t)tau * c.S;
            const int32_t st = DIR * c.S;
            const float vp = __ldg(Ds);
            bool hit = false;
            for (int32_t j0 = 3; j0 <= jm && !hit; j0 += 4) {
                float vq[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) vq[u] = (j0 + u <= jm) ? __ldg(Ds + (int64_t)(j0 + u) * st) : NaN;
                for (int u = 0; u < 4; ++u) hit = hit || pair_far(vq[u], vp, j0 + u, vk, p);
            }
            dbg_add(c.dbg, 4, hit ? 1u : 0u);
            if (hit) {
                int32_t x, y;
                lg_px(c.kind, c.l0, src, tau, x, y);
                mask_put(Mv, c.mf, c.W, x, y, true);
            }
        }
    }
    __syncwarp();
    OCC_PH_T1(c, 1, tph);
}

// Appends the survivors of `bits` (bit r <-> tau0 + r) to the deferred queue,
// at most `quota` per lane; returns the bits not queued.  Warp-collective;
// the caller guarantees room for 32 * quota entries.
__device__ __forceinline__ uint32_t queue_bits(const int DIR, const Ctx &c, const Blk &b, int32_t h, uint32_t bits,
                                               int quota, int32_t *qbuf, int32_t &qn) {
    const int lane = c.lane;
    uint32_t take = 0u, t = bits;
    for (int i = 0; i < quota && t; ++i) { const uint32_t lb = t & (0u - t); take |= lb; t ^= lb; }
    const uint32_t n = __popc(take);
    uint32_t inc = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t tt = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += tt;
    }
    const int32_t tot = (int32_t)__shfl_sync(FULL, inc, 31);
    int32_t pos = qn + (int32_t)(inc - n);
    uint32_t w = take;
    while (w) {
        const int32_t r = __ffs(w) - 1;
        w &= w - 1u;
        const int32_t tau = b.tau0 + r;
        int32_t jm = dcov_of(DIR, b.Wc, b.cfall, b.tau0, r, h);
        jm = min(jm, DIR > 0 ? c.ehi - 1 - tau : tau - c.elo);
        qbuf[2 * pos] = tau;
        qbuf[2 * pos + 1] = (max(jm, 0) << 5) | lane;
        ++pos;
    }
    qn += tot;
    __syncwarp();
    return bits & ~take;
}

// Far survivors S (bit r <-> tau0 + r) of one view that the sweep's witness
// probe did not confirm: all of them go to the deferred queue, searched after
// the kernel by k_hard (one thread per survivor, the whole GPU, IPC ~3)
// instead of in this latency-bound warp.  Measured at C5: resolving them here
// first (the line's last offset, then the parked guess +-1 and a secant step)
// cost 46.0 ms per step against 36.9 ms for queueing them all.
__device__ __noinline__ uint32_t resolve(const int DIR, const Ctx &c, uint32_t S, const Blk &b, const ViewK &vk,
                                         const Params &p, int32_t *qbuf, int32_t &qn,
                                         uint8_t *Mv, uint32_t &left, int32_t vid) {
    const int lane = c.lane;
    const int32_t h = vk.h;
    OCC_PH_T0(tph);
    dbg_add(c.dbg, DIR > 0 ? 0 : 1, __popc(S));
    const uint32_t hits = 0u, hard = S;
    dbg_add(c.dbg, 3, __popc(hard));
    // queue the rest for the deferred lane-parallel search.  Flushing here is
    // safe: the queue holds only earlier blocks, whose masks are stored.
    // More than QCAP at once (rare): the remainder is returned in `left` and
    // queued by the caller after this block's mask store.
    {
        const int32_t tot = __reduce_add_sync(FULL, __popc(hard));
        if (lane == 0) dbg_add(c.dbg, 10, tot > QCAP ? 1u : 0u);
        if (qn + tot > QCAP) {
            flush_queue(DIR, c, qbuf, qn, vk, p, Mv, vid);
            qn = 0;
        }
        left = queue_bits(DIR, c, b, h, hard, tot <= QCAP ? 32 : QCAP / 32, qbuf, qn);
    }
    OCC_PH_T1(c, 0, tph);
    return hits;
}

// candidate bits of [x, x + 31] from one view's words (0 outside the staged range)
__device__ __forceinline__ uint32_t cand_bits32(const uint32_t *cw, int32_t x, int32_t WB, int lane) {
    const int32_t w = (x >> 5) - WB, sh = x & 31;
    const uint32_t lo = (w >= 0 && w < NCW) ? cw[w * 32 + lane] : 0u;
    const uint32_t hi = (w + 1 >= 0 && w + 1 < NCW) ? cw[(w + 1) * 32 + lane] : 0u;
    return __funnelshift_r(lo, hi, sh);
}

// mask bytes of one view for the 32 tau of block k (bit r <-> tau = 32k + r)
__device__ __noinline__ void store_block(const Ctx &c, uint8_t *Mv, uint32_t word, int32_t k) {
    const int lane = c.lane;
    const int32_t H = c.H, W = c.W;
    if (c.mf.packed) {
        // bit-packed planes (pre-zeroed): rows and columns own whole words;
        // a diagonal row run straddles two words shared with the neighbouring
        // line block (atomicOr)
        uint32_t *P = reinterpret_cast<uint32_t *>(Mv);
        const int32_t Wb = c.mf.Wb;
        if (c.kind == 0) {
            const int32_t y = c.l0 + lane;
            if (y >= 0 && y < H && 32 * k >= 0 && 32 * k < W) P[(int64_t)y * Wb + k] = word;
        } else if (c.kind == 1) {
            const uint32_t t = transpose32(word, lane);          // lane r: row 32k + r, bit l = column l0 + l
            const int32_t y = 32 * k + lane;
            if (y >= 0 && y < H && c.l0 >= 0 && c.l0 < W) P[(int64_t)y * Wb + (c.l0 >> 5)] = t;
        } else {
            // tau = 32k + r is one image row; its 32 lanes form the run x0 .. x0 + 31
            uint32_t mine = 0u;
            for (int r = 0; r < 32; ++r) {
                const uint32_t b = __ballot_sync(0xffffffffu, (word >> r) & 1u);
                if (r == lane) mine = b;
            }
            const int32_t tau = 32 * k + lane;
            const int32_t y = c.kind == 2 ? c.l0 + tau : c.l0 + 31 - tau;
            const uint32_t run = c.kind == 2 ? __brev(mine) : mine;      // bit m <-> x = tau - 31 + m
            if (run && y >= 0 && y < H) {
                const int32_t x0 = tau - 31, w0 = x0 >> 5, sh = x0 & 31;
                const uint32_t lo = run << sh, hi = sh ? (run >> (32 - sh)) : 0u;
                if (lo && w0 >= 0 && w0 < Wb) atomicOr(P + (int64_t)y * Wb + w0, lo);
                if (hi && w0 + 1 >= 0 && w0 + 1 < Wb) atomicOr(P + (int64_t)y * Wb + w0 + 1, hi);
            }
        }
        return;
    }
    if (c.kind == 0) {
        const int32_t y = c.l0 + lane, x0 = 32 * k;
        if (y < 0 || y >= H) return;
        uint8_t *row = Mv + (int64_t)y * W;
        if ((W & 15) == 0 && x0 >= 0 && x0 + 32 <= W) {
            uint4 *d = reinterpret_cast<uint4 *>(row + x0);
            __stcs(d, make_uint4(expand4(word & 15u), expand4((word >> 4) & 15u),
                                 expand4((word >> 8) & 15u), expand4((word >> 12) & 15u)));
            __stcs(d + 1, make_uint4(expand4((word >> 16) & 15u), expand4((word >> 20) & 15u),
                                     expand4((word >> 24) & 15u), expand4(word >> 28)));
        } else {
            for (int r = 0; r < 32; ++r) {
                const int32_t x = x0 + r;
                if (x >= 0 && x < W) row[x] = (uint8_t)((word >> r) & 1u);
            }
        }
    } else if (c.kind == 1) {
        const uint32_t t = transpose32(word, lane);      // lane r: row y = 32k + r, bit l = column l0 + l
        const int32_t y = 32 * k + lane;
        if (y < 0 || y >= H) return;
        uint8_t *row = Mv + (int64_t)y * W;
        if ((W & 15) == 0 && c.l0 >= 0 && c.l0 + 32 <= W && (c.l0 & 15) == 0) {
            uint4 *d = reinterpret_cast<uint4 *>(row + c.l0);
            __stcs(d, make_uint4(expand4(t & 15u), expand4((t >> 4) & 15u), expand4((t >> 8) & 15u),
                                 expand4((t >> 12) & 15u)));
            __stcs(d + 1, make_uint4(expand4((t >> 16) & 15u), expand4((t >> 20) & 15u),
                                     expand4((t >> 24) & 15u), expand4(t >> 28)));
        } else {
            for (int l = 0; l < 32; ++l) {
                const int32_t x = c.l0 + l;
                if (x >= 0 && x < W) row[x] = (uint8_t)((t >> l) & 1u);
            }
        }
    } else {
        // one image row per tau: the 32 lanes write one contiguous (reversed) run
        uint8_t *dst = Mv + c.B + (int64_t)(32 * k) * c.S;
        if (32 * k >= c.elo && 32 * k + 32 <= c.ehi) {
#pragma unroll 8
            for (int r = 0; r < 32; ++r) __stcs(dst + (int64_t)r * c.S, (uint8_t)((word >> r) & 1u));
        } else {
            for (int r = 0; r < 32; ++r) {
                const int32_t tau = 32 * k + r;
                if (tau >= c.elo && tau < c.ehi) __stcs(dst + (int64_t)r * c.S, (uint8_t)((word >> r) & 1u));
            }
        }
    }
}

// exact per-pixel fallback for the unit (frames outside the sweep's range of h)
__device__ __noinline__ void unit_direct(const Ctx &c, const LineArgs &a, const GroupDesc &gd,
                                         const FamilyDesc &fd, int32_t f, int32_t T0, int32_t T1,
                                         bool zero) {
    const int64_t HW = (int64_t)c.H * c.W;
    const float R = frame_range(a.st[f]);
    for (int g = 0; g < gd.nv; ++g) {
        const ViewDesc &vd = a.views[gd.view[g]];
        const int32_t h = view_h(R, vd.s, a.p.max_scan);
        uint8_t *Mv = a.masks + ((int64_t)f * a.nviews + gd.view[g]) * a.mf.vbytes;
        for (int32_t tau = max(T0, c.elo); tau < min(T1, c.ehi); ++tau) {
            int32_t x, y;
            lg_px(c.kind, c.l0, c.lane, tau, x, y);
            const bool m = !zero && direct_pixel<false>(c.Df, c.H, c.W, vd, fd, a.p, h, x, y);
            mask_put(Mv, a.mf, c.W, x, y, m);
        }
    }
}

template <int CB>
__device__ __forceinline__ void unit_body(const LineArgs &a, const LineUnit &u, const GroupDesc &gd,
                                          const FamilyDesc &fd, int32_t f, unsigned char *smem) {
    const int kind = fd.kind;
    const bool NFWD = a.views[gd.view[0]].nfwd > 0;
    const int lane = threadIdx.x & 31;
    const int32_t H = a.H, W = a.W;
    const int64_t HW = (int64_t)H * W;
    Ctx c;
    c.dbg = a.dbg;
    c.f = f;
    c.mf = a.mf;
    c.gq = a.gq; c.gq_count = a.gq_count; c.gq_cap = a.gq_cap;
    {
        const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
#ifdef OCC_LINE_STATS
        c.ph = (a.dbg && wid < 32768u) ? a.dbg + 16 + 2 * 32768 + 4 * wid : nullptr;
#else
        c.ph = nullptr;
        (void)wid;
#endif
    }
    c.kind = kind;
    c.Df = a.D + (int64_t)f * HW;
    c.H = H; c.W = W; c.l0 = u.l0; c.lane = lane;
    lg_ext(kind, u.l0, lane, H, W, c.elo, c.ehi);
    c.B = line_base(kind, u.l0, lane, W);
    c.S = line_stride(kind, W);
    c.Dl = c.Df + c.B;
    c.vec4 = kind == 0 && (W & 3) == 0;

    uint32_t *cw = reinterpret_cast<uint32_t *>(smem + OFF_CW);
    uint32_t *nn = reinterpret_cast<uint32_t *>(smem + OFF_NN);
    int32_t *qbuf = reinterpret_cast<int32_t *>(smem + OFF_Q);
    SabT *sab = reinterpret_cast<SabT *>(smem + OFF_SAB);
    float *stg = reinterpret_cast<float *>(smem + OFF_STG);
    int32_t qn = 0;
    const int32_t T0 = u.t0, T1 = u.t1;            // multiples of 32
    const int32_t kB = T0 >> 5, kT = (T1 >> 5) - 1;

    // views: P = +b0 (sg > 0), N = -b0
    int32_t vP = -1, vN = -1;
    for (int g = 0; g < gd.nv; ++g) {
        if (a.views[gd.view[g]].sg > 0) vP = gd.view[g]; else vN = gd.view[g];
    }
    const ViewDesc &vd0 = a.views[vP >= 0 ? vP : vN];
    const FrameStats fs = a.st[f];
    const float R = frame_range(fs);
    const int32_t s = vd0.s;
    const int32_t h = view_h(R, s, a.p.max_scan);
    if (fs.nonfinite || h <= 0) {            // SPEC.md:76 reject / Q17: zero masks
        unit_direct(c, a, gd, fd, f, T0, T1, true);
        return;
    }
    if (h < 17 || h + 32 > 32 * CMW) {
        dbg_add(c.dbg, 8, 1u);
        unit_direct(c, a, gd, fd, f, T0, T1, false);
        return;
    }
    const float M = fmaxf(fabsf(key_float(fs.minkey)), fabsf(key_float(fs.maxkey)));
    ViewK vk;
    vk.s = s; vk.h = h; vk.fs = (float)s;
    vk.tlo = __fsub_rn(a.p.t_dist, 0x1p-10f);
    vk.thi = __fadd_rn(a.p.t_dist, 0x1p-10f);
    {
        const double eps = ldexp(1.0, -19) * ((double)s * (double)M + 4096.0 + (double)a.p.t_dist);
        vk.T = __double2float_ru(__dadd_rn((double)a.p.t_dist, eps));
    }
    const int32_t reach = partner_reach(a.p.t_dist, s, R, h);
    const int32_t nbr = (reach + 3 + 31) >> 5;
    // thresholds (identical for the two views of the group)
    const float a1n = nextup_f(vd0.back_lo[0]), bhi0 = vd0.back_hi[0];
    const float a2n = nextup_f(vd0.back_lo[1]), bhi1 = vd0.back_hi[1];
    const float fhi0 = NFWD ? vd0.fwd_hi[0] : 0.0f;
    const float fs_ = (float)s;
    int32_t kEmin = c.elo >> 5, kEmax = (c.ehi - 1) >> 5;
    if (c.elo >= c.ehi) { kEmin = 1 << 20; kEmax = -(1 << 20); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kEmin = min(kEmin, __shfl_xor_sync(FULL, kEmin, o));
        kEmax = max(kEmax, __shfl_xor_sync(FULL, kEmax, o));
    }

    // ---------------------------------------------------- pass 0: candidates
    const int32_t WB = kB - CMW;
    {
        const unsigned char *codesf = reinterpret_cast<const unsigned char *>(a.codes) + (int64_t)f * HW * CB;
        OCC_PH_T0(tph);
        // coverage reads candidates within h + 32 of the segment (S8, App. A.2)
        const int32_t wlo = ((T0 - h - 32) >> 5) - WB, whi = ((T1 + h + 31) >> 5) - WB;
        if (a.cand) load_cand(c, a.cand, a.candfam[gd.fam], WB, cw, wlo, whi);
        else build_cand<CB>(c, codesf, 2 * gd.fam, WB, cw, wlo, whi);
        OCC_PH_T1(c, 2, tph);
    }
    const uint32_t *cwP = cw, *cwN = cw + NCW * 32;
    __syncwarp();

    const float NaN = __int_as_float(0x7fc00000);
    uint8_t *MP = vP >= 0 ? a.masks + ((int64_t)f * a.nviews + vP) * a.mf.vbytes : nullptr;
    uint8_t *MN = vN >= 0 ? a.masks + ((int64_t)f * a.nviews + vN) * a.mf.vbytes : nullptr;

    // ---------------------------------------------------- pass A (descending)
    // Far filter of view +b: SX = max A(q) over q >= i + 3, A = s v - pos, with
    // its witness SA, which is parked for every survivor (filter passed) and
    // seeds the survivor's exact resolution.
    {
        const int32_t kS = max(min(kT + nbr, kEmax), kT);
        float v1 = NaN, v2 = NaN, v3 = NaN, A1 = NaN, A2 = NaN, A3 = NaN, SX = -INFINITY, VW = NaN;
        int32_t SA = 0;
        int slot = 0;
        stage_chunk(c, stg, kS);
        cp_commit();
        for (int32_t k = kS; k >= kB; --k) {
#if LINE_ONE_SLOT
            // one staging slot: chunk k was staged at the end of the previous
            // iteration; chunk k - 1 is staged after this one is done
            const float *cb = stg + lane;
            (void)slot;
            cp_wait<0>();
            __syncwarp();
#else
            // chunk k is (being) staged in `slot`; stage k - 1 into the other slot
            const float *cb = stg + slot * 32 * SP + lane;
            float *nxt = stg + (slot ^ 1) * 32 * SP;
            __syncwarp();
            stage_chunk(c, nxt, k - 1);
            cp_commit();
            cp_wait<1>();
            __syncwarp();
            slot ^= 1;
#endif
            float ip = (float)(32 * k + 31 - T0);
            SA += 32;                                  // witness offset relative to tau0 = 32 k
            if (k > kT) {
                // start-up: suffix max only
#pragma unroll 8
                for (int r = 31; r >= 0; --r) {
                    const float v0 = cb[r * SP];
                    const float A0 = __fmaf_rn(fs_, v0, -ip);
                    if (A3 > SX) { SX = A3; SA = r + 3; VW = v3; }
                    A3 = A2; A2 = A1; A1 = A0; v3 = v2; v2 = v1; v1 = v0;
                    ip = __fsub_rn(ip, 1.0f);
                }
#if LINE_ONE_SLOT
                __syncwarp();
                stage_chunk(c, stg, k - 1);
                cp_commit();
#endif
                continue;
            }
            const int32_t tau0 = 32 * k;
            const CovP cp = cov_p(cwP, tau0, h, WB, lane);
            uint32_t Xs1 = 0, Xg1 = 0, Xl1 = 0, Xlf = 0, Xs2 = 0, Xg2 = 0, Xl2 = 0, XFR = 0;
#pragma unroll kSweepUnroll
            for (int r = 31; r >= 0; --r) {
                const float v0 = cb[r * SP];
                const float d1 = __fsub_rn(v1, v0), d2 = __fsub_rn(v2, v0);
                const float e1 = fabsf(d1), e2 = fabsf(d2);
                Xs1 = push(Xs1, d1);
                Xg1 = push(Xg1, __fsub_rn(e1, a1n));
                Xl1 = push(Xl1, __fsub_rn(e1, bhi0));
                Xlf = push(Xlf, __fsub_rn(e1, fhi0));
                Xs2 = push(Xs2, d2);
                Xg2 = push(Xg2, __fsub_rn(e2, a2n));
                Xl2 = push(Xl2, __fsub_rn(e2, bhi1));
                const float A0 = __fmaf_rn(fs_, v0, -ip);
                if (A3 > SX) { SX = A3; SA = r + 3; VW = v3; }
                const float fr = __fsub_rn(__fsub_rn(A0, vk.T), SX);
                XFR = push(XFR, fr);
                // partner guess of a survivor: past the filter witness SA, A falls
                // ~1 per step along a flat occluder, so the partner sits near
                // jw = max(SA - i, s (v_SA - v_i))
                if (fr < 0.0f)
                    sab[r * 32 + lane] = (SabT)min(max(SA - r, __float2int_rn(fminf(__fmul_rn(fs_, __fsub_rn(VW, v0)), 30000.0f))), SAB_MAX);
                A3 = A2; A2 = A1; A1 = A0; v3 = v2; v2 = v1; v1 = v0;
                ip = __fsub_rn(ip, 1.0f);
            }
            // tails: delta1 at 32k - 1, delta2 at 32k - 1 and 32k - 2 (chunk k - 1)
#if LINE_ONE_SLOT
            const float vm1 = gv(c, 32 * k - 1), vm2 = gv(c, 32 * k - 2);
#else
            cp_wait<0>();
            __syncwarp();
            const float vm1 = nxt[31 * SP + lane], vm2 = nxt[30 * SP + lane];
#endif
            const float d1m = __fsub_rn(v1, vm1), d2m1 = __fsub_rn(v2, vm1), d2m2 = __fsub_rn(v1, vm2);
            const uint32_t s1m = sgnbit(d1m), g1m = sgnbit(__fsub_rn(fabsf(d1m), a1n));
            const uint32_t t1m = (g1m ^ 1u) & sgnbit(__fsub_rn(fabsf(d1m), bhi0));
            const uint32_t tfm = NFWD ? ((g1m ^ 1u) & sgnbit(__fsub_rn(fabsf(d1m), fhi0))) : 0u;
            const uint32_t t2m1 = (sgnbit(__fsub_rn(fabsf(d2m1), a2n)) ^ 1u) & sgnbit(__fsub_rn(fabsf(d2m1), bhi1));
            const uint32_t t2m2 = (sgnbit(__fsub_rn(fabsf(d2m2), a2n)) ^ 1u) & sgnbit(__fsub_rn(fabsf(d2m2), bhi1));
            const uint32_t s2m1 = sgnbit(d2m1), s2m2 = sgnbit(d2m2);
            const uint32_t T1 = ~Xg1 & Xl1, T2 = ~Xg2 & Xl2, TF = NFWD ? (~Xg1 & Xlf) : 0u;
            // view -b near marks (parked for pass B)
            if (vN >= 0) {
                const CovN cn = cov_n(cwN, tau0, h, WB, lane);
                const uint32_t n1 = ((T1 & Xs1) << 1) | (t1m & s1m);
                const uint32_t n2 = ((T2 & Xs2) << 2) | ((t2m1 & s2m1) << 1) | (t2m2 & s2m2);
                uint32_t mN = (n1 & cov_n_k(cn, tau0, h, 1)) | (n2 & cov_n_k(cn, tau0, h, 2));
                if (NFWD) mN |= (TF & ~Xs1) & cov_n_f(cn, tau0, h);
                nn[(k - kB) * 32 + lane] = mN;
            }
            if (vP >= 0) {
                const uint32_t C3 = cov_p_k(cp, tau0, h, 3);
                uint32_t mP = ((T1 & ~Xs1) & cov_p_k(cp, tau0, h, 1)) | ((T2 & ~Xs2) & cov_p_k(cp, tau0, h, 2));
                if (NFWD) mP |= (((TF & Xs1) << 1) | (tfm & s1m)) & cov_p_f(cp, tau0, h);
                uint32_t surv = XFR & C3 & ~mP;
                uint32_t left = 0u;
                Blk b;
                if (__any_sync(FULL, surv != 0u)) {
                    // witness probes of the block's survivors, branch-free, 8 loads in
                    // flight; offsets clamped to dcov(i) >= pc(tau0 + h) + h - i (a hit
                    // at any covered offset >= 3 is a far mark) and to the line
                    const int32_t pc0 = (cand_bits32(cwP, tau0 + h, WB, lane) & 1u) ? tau0 + h : cp.pcl;
                    const int32_t jcb = min(pc0 + h - tau0, c.ehi - 1 - tau0);
                    uint32_t XH = 0u;
#pragma unroll kSweepUnroll
                    for (int r = 31; r >= 0; --r) {
                        const int32_t jv = min((int32_t)sab[r * 32 + lane], jcb - r);
                        const bool ok = jv >= 3 && tau0 + r >= c.elo && ((surv >> r) & 1u);
                        const float vq = ok ? __ldg(c.Dl + (int64_t)(tau0 + r + jv) * c.S) : NaN;
                        const float x = __fsub_rn(fabsf(__fmaf_rn(fs_, __fsub_rn(vq, cb[r * SP]), -(float)jv)), vk.tlo);
                        XH = push(XH, x);
                    }
                    mP |= XH & surv;
                    surv &= ~XH;
                }
                if (__any_sync(FULL, surv != 0u)) {
                    b.tau0 = tau0; b.cb = cb;
                    b.Wc = cand_bits32(cwP, tau0 + h, WB, lane); b.cfall = cp.pcl;
                    b.sab = sab; b.T0 = T0;
                    mP |= resolve(1, c, surv, b, vk, a.p, qbuf, qn, MP, left, vP);
                }
                store_block(c, MP, mP, k);
                while (__any_sync(FULL, left != 0u)) {        // queue overflow (rare)
                    flush_queue(1, c, qbuf, qn, vk, a.p, MP, vP);
                    qn = 0;
                    left = queue_bits(1, c, b, h, left, QCAP / 32, qbuf, qn);
                }
                if (qn >= 32) {          // a full lane batch: search while its lines are L1-hot
                    flush_queue(1, c, qbuf, qn, vk, a.p, MP, vP);
                    qn = 0;
                }
            }
#if LINE_ONE_SLOT
            __syncwarp();
            if (k - 1 >= kB) {
                stage_chunk(c, stg, k - 1);
                cp_commit();
            }
#endif
        }
        cp_wait<0>();
        if (vP >= 0 && qn > 0) flush_queue(1, c, qbuf, qn, vk, a.p, MP, vP);
        qn = 0;
    }
    if (vN < 0) return;
    __syncwarp();

    // ---------------------------------------------------- pass B (ascending)
    // Far filter of view -b: SX = max A(q) over q <= i - 3, A = s v + pos,
    // with its witness SA parked for every survivor.
    {
        const int32_t kS = min(max(kB - nbr, kEmin), kB);
        float v1 = NaN, v2 = NaN, v3 = NaN, A1 = NaN, A2 = NaN, A3 = NaN, SX = -INFINITY, VW = NaN;
        int32_t SA = 0;
        int slot = 0;
        stage_chunk(c, stg, kS);
        cp_commit();
        for (int32_t k = kS; k <= kT; ++k) {
#if LINE_ONE_SLOT
            const float *cb = stg + lane;
            (void)slot;
            cp_wait<0>();
            __syncwarp();
#else
            const float *cb = stg + slot * 32 * SP + lane;
            float *nxt = stg + (slot ^ 1) * 32 * SP;
            __syncwarp();
            if (k + 1 <= kT) stage_chunk(c, nxt, k + 1);
            cp_commit();
            cp_wait<1>();
            __syncwarp();
            slot ^= 1;
#endif
            float ip = (float)(32 * k - T0);
            SA -= 32;                                  // witness offset relative to tau0 = 32 k
            if (k < kB) {
#pragma unroll 8
                for (int r = 0; r < 32; ++r) {
                    const float v0 = cb[r * SP];
                    const float A0 = __fmaf_rn(fs_, v0, ip);
                    if (A3 > SX) { SX = A3; SA = r - 3; VW = v3; }
                    A3 = A2; A2 = A1; A1 = A0; v3 = v2; v2 = v1; v1 = v0;
                    ip = __fadd_rn(ip, 1.0f);
                }
#if LINE_ONE_SLOT
                __syncwarp();
                stage_chunk(c, stg, k + 1);
                cp_commit();
#endif
                continue;
            }
            const int32_t tau0 = 32 * k;
            const CovN cn = cov_n(cwN, tau0, h, WB, lane);
            uint32_t XFR = 0;
#pragma unroll kSweepUnroll
            for (int r = 0; r < 32; ++r) {
                const float v0 = cb[r * SP];
                const float A0 = __fmaf_rn(fs_, v0, ip);
                if (A3 > SX) { SX = A3; SA = r - 3; VW = v3; }
                const float fr = __fsub_rn(__fsub_rn(A0, vk.T), SX);
                XFR = push(XFR, fr);
                if (fr < 0.0f)
                    sab[r * 32 + lane] = (SabT)min(max(r - SA, __float2int_rn(fminf(__fmul_rn(fs_, __fsub_rn(VW, v0)), 30000.0f))), SAB_MAX);
                A3 = A2; A2 = A1; A1 = A0; v3 = v2; v2 = v1; v1 = v0;
                ip = __fadd_rn(ip, 1.0f);
            }
            XFR = __brev(XFR);                     // bit r <-> tau0 + r
            const uint32_t C3 = cov_n_k(cn, tau0, h, 3);
            uint32_t mN = nn[(k - kB) * 32 + lane];
            uint32_t surv = XFR & C3 & ~mN;
            uint32_t left = 0u;
            Blk b;
            if (__any_sync(FULL, surv != 0u)) {
                // witness probes toward lower tau; dcov(i) >= i + h - nc(tau0 + 31 - h)
                const int32_t nc0 = (cand_bits32(cwN, tau0 + 31 - h, WB, lane) & 1u) ? tau0 + 31 - h : cn.ncl;
                const int32_t jcb = min(tau0 + h - nc0, tau0 - c.elo);
                uint32_t XH = 0u;
#pragma unroll kSweepUnroll
                for (int r = 31; r >= 0; --r) {
                    const int32_t jv = min((int32_t)sab[r * 32 + lane], jcb + r);
                    const bool ok = jv >= 3 && tau0 + r < c.ehi && ((surv >> r) & 1u);
                    const float vq = ok ? __ldg(c.Dl + (int64_t)(tau0 + r - jv) * c.S) : NaN;
                    const float x = __fsub_rn(fabsf(__fmaf_rn(fs_, __fsub_rn(vq, cb[r * SP]), -(float)jv)), vk.tlo);
                    XH = push(XH, x);
                }
                mN |= XH & surv;
                surv &= ~XH;
            }
            if (__any_sync(FULL, surv != 0u)) {
                b.tau0 = tau0; b.cb = cb;
                b.Wc = cand_bits32(cwN, tau0 - h, WB, lane); b.cfall = cn.ncl;
                b.sab = sab; b.T0 = T0;
                mN |= resolve(-1, c, surv, b, vk, a.p, qbuf, qn, MN, left, vN);
            }
            dbg_add(c.dbg, 7, 32u);
            store_block(c, MN, mN, k);
            while (__any_sync(FULL, left != 0u)) {            // queue overflow (rare)
                flush_queue(-1, c, qbuf, qn, vk, a.p, MN, vN);
                qn = 0;
                left = queue_bits(-1, c, b, h, left, QCAP / 32, qbuf, qn);
            }
            if (qn >= 32) {              // a full lane batch: search while its lines are L1-hot
                flush_queue(-1, c, qbuf, qn, vk, a.p, MN, vN);
                qn = 0;
            }
#if LINE_ONE_SLOT
            __syncwarp();
            if (k + 1 <= kT) {
                stage_chunk(c, stg, k + 1);
                cp_commit();
            }
#endif
        }
        cp_wait<0>();
        if (qn > 0) flush_queue(-1, c, qbuf, qn, vk, a.p, MN, vN);
    }
}

// grid: (units, frames); one warp per block
template <int CB>
#ifndef LINE_MINB
#define LINE_MINB 1
#endif
__global__ void __launch_bounds__(128, LINE_MINB) k_line(LineArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    // one work unit per warp, frame-major (units fastest, longest first)
    const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (wid >= (uint32_t)a.nwork) return;
    const uint32_t nu = (uint32_t)a.nwork / (uint32_t)a.frames;
    const int32_t f = a.frame_major ? (int32_t)(wid / nu) : (int32_t)(wid % (unsigned)a.frames);
    const LineUnit u = a.units[a.frame_major ? wid % nu : wid / (unsigned)a.frames];
    const GroupDesc gd = a.groups[u.group];
    const FamilyDesc fd = a.fams[gd.fam];
#ifdef OCC_LINE_STATS
    const long long t0 = a.dbg ? clock64() : 0;
#endif
    unit_body<CB>(a, u, gd, fd, f, smem + (size_t)(threadIdx.x >> 5) * WSMEM);
#ifdef OCC_LINE_STATS
    if (a.dbg && (threadIdx.x & 31) == 0 && wid < 32768u) {
        a.dbg[16 + wid] = (unsigned long long)(clock64() - t0);
        a.dbg[16 + 32768 + wid] = ((unsigned long long)fd.kind << 60) | ((unsigned long long)(u.t1 - u.t0) << 40) |
                                  ((unsigned long long)(u.l0 + 40000) << 20) | (unsigned long long)(u.t0 + 40000);
    }
#endif
}

// Exhaustive far-partner searches queued by k_line: one thread per entry
// (survivor p of view v in frame f), offsets 3..dcov(p) along its line, 16
// loads in flight; a confirmed Eq. 5 pair sets the mask byte.
#ifndef HARD_BATCH
#define HARD_BATCH 16        // offsets (loads in flight) per k_hard step
#endif
// C5 k_hard ms per 256 frames (one B200, A/B): MINB 1 (71 registers) 3.49,
// 2 3.52, 4 (64) 3.23, 5 (48) 3.53, 6 (40, spills) 3.82
#ifndef HARD_MINB
#define HARD_MINB 4
#endif
#ifndef HARD_PROBE_LEAN
#define HARD_PROBE_LEAN 1    // (C5 k_hard 2.46 -> 2.39 ms per step, A/B on one B200)
#endif
// SHEAR: the entries of a knight family swept through its sheared copy
// (k_shear): D, W, HW are the sheared frame's, the line step is 1 (rows) or
// W (columns), and the mask pixel is un-sheared (ShearDesc, occ_internal.h)
template <bool SHEAR>
__global__ void __launch_bounds__(256, HARD_MINB) k_hard(const float *__restrict__ D, uint8_t *__restrict__ masks,
                                              MaskFmt mf, int32_t W, int64_t HW, int32_t frames, int32_t nviews,
                                              const ViewDesc *__restrict__ views,
                                              Params p, const HardEntry *__restrict__ gq,
                                              const uint32_t *__restrict__ gq_count, int32_t gq_cap,
                                              const FrameStats *__restrict__ st, ShearDesc sh) {
    const uint32_t n = min(*gq_count, (uint32_t)gq_cap);
    const float NaN = __int_as_float(0x7fc00000);
    // newest entries first: their frames were swept last and are still in L2
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t e = n - 1u - t;
        const HardEntry he = gq[e];
        const int32_t f = (int32_t)((uint32_t)he.guess >> 17), v = (int32_t)(he.meta >> 25);
        const int32_t guess = he.guess & 0x1FFFF;
        OCC_CHECK(f < frames && v < nviews && he.pix >= 0 && (int64_t)he.pix < HW);
        const ViewDesc &vdv = views[v];
        const int32_t s = vdv.s;
        const int32_t step = (vdv.sg > 0 ? 1 : -1) * (SHEAR ? (sh.kind == 0 ? 1 : W) : line_stride(vdv.lkind, W));
        ViewK vk;
        vk.s = s; vk.h = 0; vk.fs = (float)s; vk.T = 0.0f;
        vk.tlo = __fsub_rn(p.t_dist, 0x1p-10f);
        vk.thi = __fadd_rn(p.t_dist, 0x1p-10f);
        const float *Ds = D + (int64_t)f * HW + he.pix;
        const float vp = __ldg(Ds);
        // a partner at offset j needs j < s delta + t_dist with delta =
        // fl(v_q - v_p) <= fl(vmax - v_p) (rounding is monotone): offsets past
        // floor(s fl(vmax - v_p) + t_dist) cannot pair
        const float vmax = key_float(st[f].maxkey);
        const double jv = floor(__dadd_rn(__dmul_rn((double)s, (double)__fsub_rn(vmax, vp)), (double)p.t_dist));
        const int32_t jm = (int32_t)fmin((double)(he.meta & 0x1FFFFu), jv);
        bool hit = false;
        if (guess >= 3 && jm >= 3) {
            // the sweep's probe at he.guess read he.vq and missed: a slanted
            // occluder puts the partner near the fixed point j = s (vq - v_p)
            const double jf = rint(__dmul_rn((double)s, (double)__fsub_rn(he.vq, vp)));
            const int32_t j2 = (int32_t)fmin(fmax(jf, 3.0), (double)jm);
            float w[5];
#if HARD_PROBE_LEAN
            // as the scan batches: pointer steps, one minimum, the exact test
            // only when the minimum lies in the 2^-10 band
            const float *q = Ds + (int64_t)(j2 - 2) * step;
            float mn = INFINITY;
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int32_t j = j2 - 2 + u;
                w[u] = (j >= 3 && j <= jm) ? __ldg(q) : NaN;
                q += step;
            }
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const float x = fabsf(__fmaf_rn(vk.fs, __fsub_rn(w[u], vp), -(float)(j2 - 2 + u)));   // NaN off range
                mn = fminf(mn, x);
            }
            hit = mn < vk.tlo;
            if (!hit && mn <= vk.thi) {
#pragma unroll
                for (int u = 0; u < 5; ++u) {
                    const int32_t j = j2 - 2 + u;
                    if (!hit && j >= 3 && j <= jm) hit = pair_far(w[u], vp, j, vk, p);
                }
            }
#else
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int32_t j = j2 - 2 + u;
                w[u] = (j >= 3 && j <= jm) ? __ldg(Ds + (int64_t)j * step) : NaN;
            }
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int32_t j = j2 - 2 + u;
                if (!hit && j >= 3 && j <= jm) hit = pair_far(w[u], vp, j, vk, p);
            }
#endif
        }
        for (int32_t j0 = 3; j0 <= jm && !hit; j0 += HARD_BATCH) {
            float vq[HARD_BATCH];
#pragma unroll
            for (int u = 0; u < HARD_BATCH; ++u)
                OCC_CHECK(j0 + u > jm || ((int64_t)he.pix + (int64_t)(j0 + u) * step >= 0 &&
                                          (int64_t)he.pix + (int64_t)(j0 + u) * step < HW));
            // addresses by pointer steps; whole batches below jm unpredicated
            const float *q = Ds + (int64_t)j0 * step;
            if (j0 + HARD_BATCH - 1 <= jm) {
#pragma unroll
                for (int u = 0; u < HARD_BATCH; ++u) { vq[u] = __ldg(q); q += step; }
            } else {
#pragma unroll
                for (int u = 0; u < HARD_BATCH; ++u) { vq[u] = (j0 + u <= jm) ? __ldg(q) : NaN; q += step; }
            }
            // branch-free fast test of the HARD_BATCH offsets (fp32 with the 2^-10
            // band, as pair_far); offsets inside the band take the exact test.
            // No offset below the band (mn >= tlo): some offset lies in the
            // band iff the minimum does (fminf skips the NaNs beyond jm)
            float mn = INFINITY;
#pragma unroll
            for (int u = 0; u < HARD_BATCH; ++u) {
                vq[u] = fabsf(__fmaf_rn(vk.fs, __fsub_rn(vq[u], vp), -(float)(j0 + u)));   // NaN beyond jm
                mn = fminf(mn, vq[u]);
            }
            hit = mn < vk.tlo;
            if (!hit && mn <= vk.thi) {
                for (int u = 0; u < HARD_BATCH && !hit; ++u)
                    if (vq[u] >= vk.tlo && vq[u] <= vk.thi)
                        hit = pair_exact_slow(__ldg(Ds + (int64_t)(j0 + u) * step), vp, j0 + u, s, p.t_dist, p.t_disp);
            }
        }
        if (hit) {
            uint8_t *Mv = masks + ((int64_t)f * nviews + v) * mf.vbytes;
            if constexpr (SHEAR) {
                const int32_t q = he.pix / W, r = he.pix % W;
                if (sh.kind == 0) mask_put(Mv, mf, sh.Wo, r, q + sh.lmin + ((r * sh.num) >> 1), true);
                else mask_put(Mv, mf, sh.Wo, r + sh.lmin + ((q * sh.num) >> 1), q, true);
            } else {
                mask_put(Mv, mf, W, he.pix % W, he.pix / W, true);
            }
        }
    }
}

cudaError_t launch_hard(const float *D, uint8_t *masks, const MaskFmt &mf, int32_t W, int64_t HW, int32_t frames,
                        int32_t nviews, const ViewDesc *views,
                        const Params &p, const HardEntry *gq, const uint32_t *gq_count, int32_t gq_cap,
                        const FrameStats *st, int32_t nsm, cudaStream_t s, const ShearDesc *sh) {
    // Grid: about two entries per thread for the expected queue (1.5 % of the
    // chunk's pixel-views at C5), so the block scheduler balances the
    // variable-length searches (a resident grid-striding 8 blocks per SM left
    // a tail: C5 k_hard 3.21 -> 2.63 ms per step at 256 blocks per SM, A/B on
    // one B200); at least 8 blocks per SM, at most 256 (OCC_HARD_GRID: fixed
    // blocks per SM).  More entries than threads are grid-strided.
    static const int bps = [] { const char *ev = getenv("OCC_HARD_GRID"); return ev ? std::max(1, atoi(ev)) : 0; }();
    const int64_t pv = (int64_t)frames * HW * nviews;
    const int64_t want = (int64_t)(0.015 * (double)pv) / 512 + 1;
    const int64_t blocks = bps ? (int64_t)nsm * bps : std::min<int64_t>((int64_t)nsm * 256, std::max<int64_t>((int64_t)nsm * 8, want));
    if (sh)
        k_hard<true><<<(unsigned)blocks, 256, 0, s>>>(D, masks, mf, W, HW, frames, nviews, views, p, gq, gq_count, gq_cap,
                                                      st, *sh);
    else
        k_hard<false><<<(unsigned)blocks, 256, 0, s>>>(D, masks, mf, W, HW, frames, nviews, views, p, gq, gq_count, gq_cap,
                                                       st, ShearDesc{});
    return cudaGetLastError();
}

// Candidate words of every (line block, tau block) of the chunk's line
// families: one warp per (frame, family, 32 lines, 32 positions), the same
// computation as k_line's pass 0 (cand_word) done once instead of once per
// unit and margin.  Layout: [frame][per_frame blocks][view 2][lane 32].
template <int CB>
__global__ void __launch_bounds__(256) k_cand(const float *D, int32_t H, int32_t W, const void *codes,
                                              const CandFam *cf, int32_t ncf, int64_t per_frame,
                                              int64_t nblocks, uint32_t *cand) {
    const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (gw >= nblocks) return;
    const int32_t f = (int32_t)(gw / per_frame);
    const int64_t bi = gw - (int64_t)f * per_frame;
    int q = 0;
    while (q + 1 < ncf && bi >= cf[q + 1].base_slot) ++q;
    const CandFam fam = cf[q];
    const int64_t r = bi - fam.base_slot;
    const int32_t lb = (int32_t)(r / fam.nk), k = (int32_t)(r - (int64_t)lb * fam.nk) + fam.kmin;
    Ctx c;
    c.kind = fam.kind;
    c.H = H; c.W = W;
    c.l0 = fam.lmin + 32 * lb;
    c.lane = threadIdx.x & 31;
    lg_ext(c.kind, c.l0, c.lane, H, W, c.elo, c.ehi);
    c.B = line_base(c.kind, c.l0, c.lane, W);
    c.S = line_stride(c.kind, W);
    const int64_t HW = (int64_t)H * W;
    const void *codesf = reinterpret_cast<const unsigned char *>(codes) + (int64_t)f * HW * CB;
    uint32_t wp, wn;
    cand_word<CB>(c, codesf, 2 * fam.fam, 32 * k, wp, wn);
    uint32_t *o = cand + (gw << 6);
    o[c.lane] = wp;
    o[32 + c.lane] = wn;
}

cudaError_t launch_cand(const float *D, int32_t H, int32_t W, int32_t frames, const void *codes, int32_t code_bytes,
                        const CandFam *cf_slots, int32_t ncf, int64_t per_frame, uint32_t *cand, cudaStream_t s) {
    if (ncf <= 0 || per_frame <= 0) return cudaSuccess;
    const int64_t nblocks = per_frame * frames;
    const unsigned grid = (unsigned)((nblocks + 7) / 8);
    if (code_bytes == 1) k_cand<1><<<grid, 256, 0, s>>>(D, H, W, codes, cf_slots, ncf, per_frame, nblocks, cand);
    else if (code_bytes == 2) k_cand<2><<<grid, 256, 0, s>>>(D, H, W, codes, cf_slots, ncf, per_frame, nblocks, cand);
    else k_cand<4><<<grid, 256, 0, s>>>(D, H, W, codes, cf_slots, ncf, per_frame, nblocks, cand);
    return cudaGetLastError();
}

cudaError_t launch_line(const float *D, int32_t H, int32_t W, int32_t batch, const LineUnit *units,
                        int32_t nunits, const GroupDesc *groups, const ViewDesc *views, int32_t nviews,
                        const FamilyDesc *fams, const FrameStats *st, const Params &p, uint8_t *masks,
                        const MaskFmt &mf, const void *codes, int32_t code_bytes, unsigned long long *dbg,
                        HardEntry *gq, uint32_t *gq_count, int32_t gq_cap, const uint32_t *cand,
                        const CandFam *candfam, cudaStream_t s) {
    if (nunits <= 0) return cudaSuccess;
    LineArgs a{D, H, W, units, groups, views, nviews, fams, st, p, masks, codes, dbg, batch, gq, gq_count, gq_cap,
               nunits * batch, mf, 0, cand, candfam};
    // tuning knobs, read once (thread-safe static initialisation)
    // frame-major by default: the warps in flight cover about one frame,
    // whose D and codes stay in L2 for all four families (measured: k_line
    // DRAM reads per 25-frame chunk 1.34 GB -> 0.26 GB, same time)
    static const int order = [] { const char *ev = getenv("OCC_LINE_ORDER"); return ev ? atoi(ev) : 1; }();
    a.frame_major = order;
    static const int nw = [] {
        const char *ev = getenv("OCC_LINE_WARPS");
        return ev ? max(1, min(4, atoi(ev))) : 4;
    }();
    dim3 grid((unsigned)((a.nwork + nw - 1) / nw));
    const size_t smem = WSMEM * (size_t)nw;
    cudaError_t e;
    // shared-memory carve-out: with the far-survivor resolution moved to
    // k_hard, occupancy beats L1 (C5: 4 warps x 100 % 33.2 ms/step, x 50 %
    // 36.1; before the move 4 x 50 % was best); set OCC_LINE_CARVEOUT to override
    static const int carve = [] { const char *ev = getenv("OCC_LINE_CARVEOUT"); return ev ? atoi(ev) : 100; }();
    if (code_bytes == 1) {
        e = cudaFuncSetAttribute(k_line<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (carve >= 0) cudaFuncSetAttribute(k_line<1>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        k_line<1><<<grid, 32 * nw, smem, s>>>(a);
    } else if (code_bytes == 2) {
        e = cudaFuncSetAttribute(k_line<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (carve >= 0) cudaFuncSetAttribute(k_line<2>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        k_line<2><<<grid, 32 * nw, smem, s>>>(a);
    } else {
        e = cudaFuncSetAttribute(k_line<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (carve >= 0) cudaFuncSetAttribute(k_line<4>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        k_line<4><<<grid, 32 * nw, smem, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace occ
