// k_tile.cu -- K1, the tiled sweep kernel: Eqs. 1-6 for one line family.
//
// One CTA = one (tile, frame): 32 consecutive digital epipolar lines of one
// family x up to 256 output positions along them, for a
// group of <= 2 views of that family.  Layout "lane = line": every thread of
// a warp owns one line, a warp owns 32 consecutive positions, so all shared
// memory accesses of the compute phase are conflict-free and the per-line
// work is a sequential sweep (the cheapest possible scan).
//
//  1. stage   D along the 32 lines into smem [pos][lane] with a halo of
//             HALO >= max(h, reach) positions per side (coalesced row runs),
//             candidate bits (Eqs. 1-2, from K0's per-pixel codes) per line
//             as 32-bit words.
//  2. per view:
//     a. coverage dcov(p) = U(p) - u_p, U(p) = pc(u_p + h) + h: a pair (p, q)
//        shares one candidate's scan window (Eq. 4) iff u_q - u_p <= dcov(p).
//     b. near pairs (|dk| <= jstar-1): exact fp32 interval tests of
//        delta = fl(v_q - v_p) (host-precomputed thresholds, S7).
//     c. far pairs (dk <= -jstar, delta > t_disp implied): conservative
//        suffix-max filter on B = s v - u along the sweep; survivors are
//        resolved exactly (binary64 predicate) at guessed offsets, the rest
//        by a warp-cooperative exhaustive search.
//  3. store   mask bytes through smem, row-contiguous streaming stores.
// Views whose halo does not fit (huge disparity ranges) are computed by the
// exact per-pixel routine (direct_pixel) inside the same CTA.
//
// The line geometry (major axis, slope num/den), the sweep direction, the
// near-offset split of the default thresholds and the candidate-code width
// are compile-time parameters for the families of |b| <= 2 arrays; other
// cases run the same code with runtime values.
#include "occ_device.cuh"

namespace occ {

namespace {
constexpr int TP = kTilePositions;     // output positions per tile
#ifndef TILE_NT
#define TILE_NT 192           // 6 warps: one per (view, block pair) sweep item of a 160-position tile (C4: 4.91 -> 4.59 ms)
#endif
constexpr int NT = TILE_NT;            // threads
constexpr int NWARP = NT / 32;
constexpr int HMAX = kTileHaloMax;     // max staged halo per side
constexpr int NPMAX = TP + 2 * HMAX;   // staged positions
constexpr int NB = NPMAX / 32;         // 32-position blocks
constexpr int VPITCH = 34;             // max floats per staged position (32 lanes + pad)
constexpr int16_t NONE_LO = -30000, NONE_HI = 30000;

constexpr int NOB = TP / 32;            // output blocks per tile
constexpr size_t OFF_V = 0;
constexpr size_t OFF_CW = OFF_V + sizeof(float) * NPMAX * VPITCH;
constexpr size_t OFF_LAST = OFF_CW + sizeof(uint32_t) * 2 * NB * 32;
constexpr size_t OFF_NEXT = OFF_LAST + sizeof(int16_t) * 2 * NB * 32;
constexpr size_t OFF_OUT = OFF_NEXT + sizeof(int16_t) * 2 * NB * 32;     // mask bits
constexpr size_t OFF_JG = OFF_OUT + sizeof(uint32_t) * kGroupViews * NOB * 32;
constexpr size_t SMEM = OFF_JG + (size_t)NWARP * 32 * 32;               // parked guesses
}  // namespace

size_t tile_smem_bytes() { return SMEM; }

// ------------------------------------------------------------ geometry
// Line family geometry: x-major lines l = y - floor(x num/den) (pos = x),
// y-major lines l = x - floor(y num/den) (pos = y).  fl(a) = floor(a num/den).
template <bool XM, int NUM, int DEN>
struct GeoK {
    __device__ __forceinline__ bool xm() const { return XM; }
    __device__ __forceinline__ int32_t num() const { return NUM; }
    __device__ __forceinline__ int32_t den() const { return DEN; }
    __device__ __forceinline__ int32_t fl(int32_t a) const {
        if (NUM == 0) return 0;
        if (DEN == 1) return a * NUM;
        if (DEN == 2) return (a * NUM) >> 1;
        return floordiv(a * NUM, DEN);
    }
};
struct GeoR {
    bool xm_;
    int32_t num_, den_;
    __device__ __forceinline__ bool xm() const { return xm_; }
    __device__ __forceinline__ int32_t num() const { return num_; }
    __device__ __forceinline__ int32_t den() const { return den_; }
    __device__ __forceinline__ int32_t fl(int32_t a) const { return floordiv(a * num_, den_); }
};

// floor(a / d) for d > 0
__device__ __forceinline__ int32_t fdivg(int32_t a, int32_t d) {
    if (d == 1) return a;
    if (d == 2) return a >> 1;
    return floordiv(a, d);
}

// x-range of image row y covered by lanes [0, 32) of an x-major tile:
// l = y - l0 - floor(x num / den) in [0, 31], clipped to [lo, hi].
template <class G>
__device__ __forceinline__ void row_run(const G &geo, int32_t y, int32_t l0, int32_t lo, int32_t hi,
                                        int32_t &xa, int32_t &xb) {
    const int32_t A = y - l0 - 31, B = y - l0;
    const int32_t num = geo.num(), den = geo.den();
    if (num == 0) {
        if (B < 0 || B > 31) { xa = 1; xb = 0; return; }
        xa = lo; xb = hi;
    } else if (num > 0) {
        xa = -fdivg(-(A * den), num);
        xb = -fdivg(-((B + 1) * den), num) - 1;
    } else {
        const int32_t n = -num;
        xa = fdivg(-(B + 1) * den, n) + 1;
        xb = fdivg(-A * den, n);
    }
    xa = max(xa, lo);
    xb = min(xb, hi);
}

// previous / next candidate of a line (local index), from the bit words and
// their per-word summaries; NONE_LO / NONE_HI when there is none
__device__ __forceinline__ int32_t prevcand(const uint32_t *cw, const int16_t *last, int32_t x,
                                            int32_t lane) {
    const int32_t w = x >> 5;
    const uint32_t m = cw[w * 32 + lane] & (0xffffffffu >> (31 - (x & 31)));
    return m ? 32 * w + 31 - __clz(m) : (w > 0 ? (int32_t)last[(w - 1) * 32 + lane] : (int32_t)NONE_LO);
}
__device__ __forceinline__ int32_t nextcand(const uint32_t *cw, const int16_t *next, int32_t x,
                                            int32_t nb, int32_t lane) {
    const int32_t w = x >> 5;
    const uint32_t m = cw[w * 32 + lane] & (0xffffffffu << (x & 31));
    return m ? 32 * w + __ffs(m) - 1 : (w + 1 < nb ? (int32_t)next[(w + 1) * 32 + lane] : (int32_t)NONE_HI);
}

template <int CB>
__device__ __forceinline__ uint32_t load_code(const unsigned char *Cb, int64_t idx) {
    if (CB == 1) return __ldg(Cb + idx);
    if (CB == 2) return __ldg(reinterpret_cast<const uint16_t *>(Cb) + idx);
    return __ldg(reinterpret_cast<const uint32_t *>(Cb) + idx);
}

// ------------------------------------------------------------ bit-sliced sweep
// Smallest float > x (x finite): the exact rewrite x > a <=> x >= nextup(a).
__device__ __forceinline__ float nextup(float a) {
    const int32_t b = __float_as_int(a);
    if (a == 0.0f) return __int_as_float(1);                  // +-0 -> smallest denormal
    return __int_as_float(a > 0.0f ? b + 1 : b - 1);
}
// Appends the sign bit of a float / int to a word: (w << 1) | sign(x).
// The sign of fl(x - c) is the exact sign of x - c, so fl(x - nextup(a)) < 0
// <=> !(x > a) and fl(x - b) < 0 <=> x < b.  For a NaN x (absent sample)
// both differences are NaN with one common sign, so the interval bit
// ~sign(x - a') & sign(x - b) is 0 whatever that sign is.
__device__ __forceinline__ uint32_t pushf(uint32_t w, float x) {
    return __funnelshift_l(__float_as_uint(x), w, 1);
}
__device__ __forceinline__ uint32_t pushi(uint32_t w, int32_t x) {
    return __funnelshift_l((uint32_t)x, w, 1);
}

// Default split (near backward j = 1, 2; far j >= 3; NFWD near forward
// offsets in {0, 1}).  One thread = one line, 32 positions of block b walked
// toward lower u.  Every per-position test is reduced to a sign bit and
// packed into 32-bit words (one bit per position); the Eq. 5 interval tests,
// window coverage and the far-filter verdict are then combined word-wise.
// Far survivors are resolved exactly afterwards: at the offset of the line's
// previous hit, or (first survivor of the line) at the offset guessed from
// the suffix-max witness, else by a warp-cooperative exhaustive search.
template <int SG, int NFWD, int VP>
__device__ __forceinline__ void sweep_bits(const float *__restrict__ sv, const uint32_t *cw,
                                           const int16_t *last, const int16_t *next,
                                           uint32_t *ow, uint8_t *jgb, int lane, int32_t b,
                                           int32_t nblk, int32_t L0,
                                           int32_t NP32, int32_t NB32, int32_t h, int32_t s,
                                           float T, int32_t Jr, float blo0, float bhi0,
                                           float blo1, float bhi1, float flo0, float fhi0,
                                           float t_dist, float t_disp) {
    const float fs_ = (float)s;
    const float a1 = nextup(blo0), a2 = nextup(blo1), af = nextup(flo0);
    const int32_t i0 = SG > 0 ? 32 * b + 31 : 32 * b;       // first (highest-u) position
    const float *col = sv + lane;
    float uf = (float)(SG * (i0 - L0));
    // suffix max of B = s v - u over i0 + SG*[4, Jr] and its witness SA
    float SX = -INFINITY;
    int32_t SA = i0;
    {
        const int32_t jend = min(Jr, SG > 0 ? NP32 - 1 - i0 : i0);
        const float *pq = col + (i0 + 4 * SG) * VP;
        float uq = uf + 4.0f;
        for (int32_t j = 4; j <= jend; ++j) {
            const float Bq = __fmaf_rn(fs_, *pq, -uq);
            if (Bq > SX) { SX = Bq; SA = i0 + SG * j; }
            pq += SG * VP;
            uq += 1.0f;
        }
    }
    const float *pc = col + i0 * VP;
    float vp = pc[0], v1 = pc[SG * VP], v2 = pc[2 * SG * VP], v3 = pc[3 * SG * VP];
    int32_t cst = SG > 0 ? prevcand(cw, last, i0 + h, lane) : nextcand(cw, next, i0 - h, NB32, lane);
    auto dcov_of = [&](int32_t i) -> int32_t {
        if (SG > 0) {
            const int32_t x = i + h;
            if (cst > x) cst = prevcand(cw, last, x, lane);
            return (cst >= i - h) ? cst + h - i : -1;
        }
        const int32_t x = i - h;
        if (cst < x) cst = nextcand(cw, next, x, NB32, lane);
        return (cst <= i + h) ? i + h - cst : -1;
    };
    int32_t dc = dcov_of(i0);
    // nblk consecutive blocks in u-descending order share the carried state
    // (window, suffix max, coverage), so the suffix-max start-up scan is paid once
    for (int kb = 0; kb < nblk; ++kb) {
    const int32_t bb = b - SG * kb;
    const int32_t ib = SG > 0 ? 32 * bb + 31 : 32 * bb;       // block's first position
    uint32_t G1 = 0, L1 = 0, G2 = 0, L2 = 0, GF = 0, LF = 0;   // interval sign words
    uint32_t C1 = 0, C2 = 0, C3 = 0, CF = 0, FR = 0;           // coverage / far words
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
        const int32_t i = ib - SG * r;
        const float vf = pc[-SG * VP];                       // forward neighbour
        {   // fold position i + 3 SG into the suffix max
            const float B3 = __fmaf_rn(fs_, v3, -(uf + 3.0f));
            if (B3 > SX) { SX = B3; SA = i + 3 * SG; }
        }
        const int32_t dcn = dcov_of(i - SG);
        const float d1 = __fsub_rn(v1, vp), d2 = __fsub_rn(v2, vp);
        G1 = pushf(G1, __fsub_rn(d1, a1)); L1 = pushf(L1, __fsub_rn(d1, bhi0));
        G2 = pushf(G2, __fsub_rn(d2, a2)); L2 = pushf(L2, __fsub_rn(d2, bhi1));
        if (NFWD) {
            const float df = __fsub_rn(vf, vp);
            GF = pushf(GF, __fsub_rn(df, af)); LF = pushf(LF, __fsub_rn(df, fhi0));
            CF = pushi(CF, -dcn);                                // dc(i - SG) >= 1
        }
        C1 = pushi(C1, -dc);                                     // dc >= 1
        C2 = pushi(C2, 1 - dc);                                  // dc >= 2
        C3 = pushi(C3, 2 - dc);                                  // dc >= 3
        // far filter: survivor <=> SX > fl(B_p - T)
        const float Bp = __fmaf_rn(fs_, vp, -uf);
        const float fr = __fsub_rn(__fsub_rn(Bp, T), SX);
        FR = pushf(FR, fr);
        if (fr < 0.0f) {
            // guessed partner offset: past the witness SA, B falls ~1 per step on
            // a flat occluder, so the partner sits ~(SX - Bp) beyond it; parked
            // in the warp's scratch until the exact resolution below
            const int32_t jg = SG * (SA - i) + min(max(0, __float2int_rn(__fsub_rn(SX, Bp))), 255);
            jgb[(i - 32 * bb) * 32 + lane] = (uint8_t)min(jg, 255);
        }
        v3 = v2; v2 = v1; v1 = vp; vp = vf;
        pc -= SG * VP;
        dc = dcn;
        uf -= 1.0f;
    }
    if (SG < 0) {   // packed first-processed-highest: restore bit r <-> position 32b + r
        G1 = __brev(G1); L1 = __brev(L1); G2 = __brev(G2); L2 = __brev(L2);
        GF = __brev(GF); LF = __brev(LF); C1 = __brev(C1); C2 = __brev(C2);
        C3 = __brev(C3); CF = __brev(CF); FR = __brev(FR);
    }
    uint32_t m = (~G1 & L1 & C1) | (~G2 & L2 & C2);
    if (NFWD) m |= ~GF & LF & CF;
    uint32_t sv_bits = (2 * h >= 3) ? (FR & C3 & ~m) : 0u;      // far survivors
    // exact resolution, u-descending order; jl = offset of the line's last hit
    int32_t jl = 0;
    uint32_t miss = 0;
    while (sv_bits) {
        const int32_t rr = SG > 0 ? 31 - __clz(sv_bits) : __ffs(sv_bits) - 1;
        sv_bits &= ~(1u << rr);
        const int32_t i = 32 * bb + rr;
        const float vq0 = sv[i * VP + lane];
        int32_t dci;
        if (SG > 0) {
            const int32_t pcv = prevcand(cw, last, i + h, lane);
            dci = pcv >= i - h ? pcv + h - i : -1;
        } else {
            const int32_t ncv = nextcand(cw, next, i - h, NB32, lane);
            dci = ncv <= i + h ? i + h - ncv : -1;
        }
        const int32_t jm = min(min(dci, 2 * h), SG > 0 ? NP32 - 1 - i : i);
        const int32_t jg = jgb[rr * 32 + lane];
        bool hit = false;
#pragma unroll
        for (int c = 0; c < 6; ++c) {
            const int32_t j = c == 5 ? jl : jg + (c == 0 ? 0 : (c == 1 ? -1 : (c == 2 ? 1 : (c == 3 ? -2 : 2))));
            if (!hit && j >= 3 && j <= jm &&
                pair_exact(sv[(i + SG * j) * VP + lane], vq0, -j, s, t_dist, t_disp)) {
                hit = true; jl = j;
            }
        }
        if (hit) m |= 1u << rr; else miss |= 1u << rr;
    }
    // misses: warp-cooperative exhaustive search over j in [3, jm], 32 at a time
    unsigned pend = __ballot_sync(0xffffffffu, miss != 0u);
    while (pend) {
        const int src = __ffs(pend) - 1;
        const uint32_t mw = __shfl_sync(0xffffffffu, miss, src);
        const int32_t rr = __ffs(mw) - 1;
        if (lane == src) miss &= ~(1u << rr);
        pend = __ballot_sync(0xffffffffu, miss != 0u);
        const int32_t i = 32 * bb + rr;
        const float vs = sv[i * VP + src];
        int32_t dci;
        if (SG > 0) {
            const int32_t pcv = prevcand(cw, last, i + h, src);
            dci = pcv >= i - h ? pcv + h - i : -1;
        } else {
            const int32_t ncv = nextcand(cw, next, i - h, NB32, src);
            dci = ncv <= i + h ? i + h - ncv : -1;
        }
        const int32_t jm = min(min(dci, 2 * h), SG > 0 ? NP32 - 1 - i : i);
        bool found = false;
        for (int32_t j0 = 3; j0 <= jm && !found; j0 += 32) {
            const int32_t j = j0 + lane;
            const bool ok = j <= jm && pair_exact(sv[(i + SG * j) * VP + src], vs, -j, s,
                                                  t_dist, t_disp);
            found = __ballot_sync(0xffffffffu, ok) != 0u;
        }
        if (found && lane == src) m |= 1u << rr;
    }
    ow[(bb - (L0 >> 5)) * 32 + lane] = m;      // bit r = position 32 bb + r
    __syncwarp();                              // jgb reused by the next block
    }
}

// ------------------------------------------------------------ tile body
struct ViewRegs {
    int32_t s, sg, h, jstar, nback, nfwd, vid, jr;
    float T;              // far-filter margin t_dist + eps
    bool staged;
};

struct TileArgs {
    const float *D;
    int32_t H, W;
    const TileDesc *tiles;
    const GroupDesc *groups;
    const ViewDesc *views;
    int32_t nviews;
    const FamilyDesc *fams;
    const FrameStats *st;
    Params p;
    uint8_t *masks;
    const void *codes;
    MaskFmt mf;
};

template <class G, int CB, int VP>
__device__ __forceinline__ void tile_body(const TileArgs &a, const G &geo, const TileDesc &td,
                                          const GroupDesc &gd, const FamilyDesc &fd,
                                          unsigned char *smem) {
    float *sv = reinterpret_cast<float *>(smem + OFF_V);
    uint32_t *scw = reinterpret_cast<uint32_t *>(smem + OFF_CW);
    int16_t *slast = reinterpret_cast<int16_t *>(smem + OFF_LAST);
    int16_t *snext = reinterpret_cast<int16_t *>(smem + OFF_NEXT);
    uint32_t *outw = reinterpret_cast<uint32_t *>(smem + OFF_OUT);
    uint8_t *sjg = smem + OFF_JG + (size_t)(threadIdx.x >> 5) * 32 * 32;
    const Params &p = a.p;
    const int32_t H = a.H, W = a.W;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int f = blockIdx.y;
    const FrameStats fs = a.st[f];
    const int64_t HW = (int64_t)H * W;
    const float *Df = a.D + (int64_t)f * HW;
    const int32_t l0 = td.l0, P0 = td.p0, P1 = td.p1, TPe = P1 - P0;
    const bool xm = geo.xm();

    // ------------------------------------------------ per-view parameters
    const float R = frame_range(fs);
    const float M = fmaxf(fabsf(key_float(fs.minkey)), fabsf(key_float(fs.maxkey)));
    ViewRegs vr[kGroupViews];
    int32_t halo = 0;
    bool any_staged = false;
#pragma unroll
    for (int g = 0; g < kGroupViews; ++g) {
        vr[g].staged = false;
        if (g >= gd.nv) continue;
        const ViewDesc &vd = a.views[gd.view[g]];
        vr[g].vid = gd.view[g];
        vr[g].s = vd.s; vr[g].sg = vd.sg; vr[g].jstar = vd.jstar;
        vr[g].nback = vd.nback; vr[g].nfwd = vd.nfwd;
        vr[g].h = view_h(R, vd.s, p.max_scan);
        // reach: a valid partner has |dk| < t_dist + s R (delta <= R) and <= 2h
        // staged halo: far partners (min(2h, reach)), candidates within h of a
        // forward neighbour (h + nfwd), near partners (nback)
        vr[g].jr = partner_reach(p.t_dist, vd.s, R, vr[g].h);
        int32_t need = max(vr[g].h + vd.nfwd, vr[g].jr);
        need = max(need, vd.nback);
        // filter margin: bounds the fp32 rounding of B = s v - u (|u| < 2^12)
        const double eps = ldexp(1.0, -19) * ((double)vd.s * (double)M + 4096.0 + (double)p.t_dist);
        vr[g].T = __double2float_ru(__dadd_rn((double)p.t_dist, eps));
        vr[g].staged = !fs.nonfinite && need <= HMAX && vd.nback <= kMaxNear &&
                       vd.nfwd <= kMaxNear && vd.jstar <= 32;
        if (vr[g].staged) { halo = max(halo, need); any_staged = true; }
    }
    // >= 32 NaN-padded positions on each side of the output blocks
    const int32_t HALO32 = max(32, (halo + 31) & ~31);
    const int32_t L0 = HALO32;                     // local index of P0
    const int32_t base = P0 - HALO32;              // position of local index 0
    const int32_t NP32 = ((TPe + 31) & ~31) + 2 * HALO32;
    const int32_t NB32 = NP32 >> 5;

    if (any_staged) {
        // ------------------------------------------------ 1. stage
        for (int k = tid; k < NP32 * 32; k += NT) sv[(k >> 5) * VP + (k & 31)] = __int_as_float(0x7fc00000);
        for (int k = tid; k < 2 * NB * 32; k += NT) scw[k] = 0u;
        __syncthreads();
        // only [L0 - halo, L0 + TPe + halo) is ever read; the rest stays NaN
        const int32_t lo_i = L0 - halo, hi_i = L0 + TPe + halo;
        // candidate bits of this family from K0's per-pixel codes (Eqs. 1-2)
        const int cshift = 2 * gd.fam;
        const unsigned char *Cb = reinterpret_cast<const unsigned char *>(a.codes) + (int64_t)f * HW * CB;
        if (!xm) {
            // y-major: pos = y, lane -> x = l0 + lane + fl(y).  A warp owns whole
            // 32-position blocks, so each lane builds its line's words in registers.
            for (int blk = (lo_i >> 5) + warp; blk <= ((hi_i - 1) >> 5); blk += NWARP) {
                uint32_t w0 = 0u, w1 = 0u;
                for (int r = 0; r < 32; ++r) {
                    const int32_t i = 32 * blk + r;
                    if (i < lo_i || i >= hi_i) continue;
                    const int32_t y = base + i;
                    if (y < 0 || y >= H) continue;
                    const int32_t x = l0 + lane + geo.fl(y);
                    if (x < 0 || x >= W) continue;
                    const int64_t idx = (int64_t)y * W + x;
                    sv[i * VP + lane] = __ldg(Df + idx);
                    const uint32_t c = load_code<CB>(Cb, idx) >> cshift;
                    w0 |= (c & 1u) << r;
                    w1 |= ((c >> 1) & 1u) << r;
                }
                scw[(0 * NB + blk) * 32 + lane] = w0;
                scw[(1 * NB + blk) * 32 + lane] = w1;
            }
        } else {
            // x-major: pos = x, lane = y - l0 - fl(x); walk image rows
            const int32_t xs = max(base + lo_i, 0), xe = min(base + hi_i, W) - 1;
            if (xs <= xe && geo.den() == 1 && (geo.num() == 1 || geo.num() == -1)) {
                // diagonals: image row y = l0 + t holds lane l at x = t - l (num = 1)
                // or x = l - t (num = -1): one coalesced row segment per step t
                const int32_t nm = geo.num();
                const int32_t tlo = nm > 0 ? xs : -xe, thi = nm > 0 ? xe + 31 : 31 - xs;
                for (int32_t t = max(tlo, -l0) + warp; t <= min(thi, H - 1 - l0); t += NWARP) {
                    const int32_t y = l0 + t, x = nm > 0 ? t - lane : lane - t;
                    if (x < xs || x > xe) continue;
                    const int32_t i = x - base;
                    const int64_t idx = (int64_t)y * W + x;
                    sv[i * VP + lane] = __ldg(Df + idx);
                    const uint32_t c = load_code<CB>(Cb, idx) >> cshift;
                    if (c & 1u) atomicOr(&scw[(0 * NB + (i >> 5)) * 32 + lane], 1u << (i & 31));
                    if (c & 2u) atomicOr(&scw[(1 * NB + (i >> 5)) * 32 + lane], 1u << (i & 31));
                }
            } else if (xs <= xe) {
                const int32_t fa = geo.fl(xs), fb = geo.fl(xe);
                const int32_t ylo = max(0, l0 + min(fa, fb)), yhi = min(H - 1, l0 + 31 + max(fa, fb));
                for (int32_t y = ylo + warp; y <= yhi; y += NWARP) {
                    int32_t xa, xb;
                    row_run(geo, y, l0, xs, xe, xa, xb);
                    const float *Drow = Df + (int64_t)y * W;
                    if (geo.num() == 0) {
                        // rows: the whole run is one line owned by this warp ->
                        // ballot the candidate bits into its words (no atomics)
                        const int32_t l = y - l0;
                        for (int32_t x0 = xa; x0 <= xb; x0 += 32) {
                            const int32_t x = x0 + lane;
                            const bool ok = x <= xb;
                            const int32_t i = x - base;
                            uint32_t c = 0u;
                            if (ok) {
                                sv[i * VP + l] = __ldg(Drow + x);
                                c = load_code<CB>(Cb, (int64_t)y * W + x) >> cshift;
                            }
                            const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u);
                            const uint32_t b1 = __ballot_sync(0xffffffffu, (c >> 1) & 1u);
                            if (lane == 0 && (b0 | b1)) {
                                const int32_t i0 = x0 - base, sh = i0 & 31, w = i0 >> 5;
                                scw[(0 * NB + w) * 32 + l] |= b0 << sh;
                                scw[(1 * NB + w) * 32 + l] |= b1 << sh;
                                if (sh) {
                                    scw[(0 * NB + w + 1) * 32 + l] |= b0 >> (32 - sh);
                                    scw[(1 * NB + w + 1) * 32 + l] |= b1 >> (32 - sh);
                                }
                            }
                        }
                    } else {
                        for (int32_t x = xa + lane; x <= xb; x += 32) {
                            const int32_t l = y - l0 - geo.fl(x);
                            const int32_t i = x - base;
                            sv[i * VP + l] = __ldg(Drow + x);
                            const uint32_t c = load_code<CB>(Cb, (int64_t)y * W + x) >> cshift;
                            if (c & 1u) atomicOr(&scw[(0 * NB + (i >> 5)) * 32 + l], 1u << (i & 31));
                            if (c & 2u) atomicOr(&scw[(1 * NB + (i >> 5)) * 32 + l], 1u << (i & 31));
                        }
                    }
                }
            }
        }
        __syncthreads();
        // candidate prefix/suffix summaries per word (for O(1) prev/next candidate)
        if (tid < 64) {
            const int d = tid >> 5;
            int16_t last = NONE_LO;
            for (int w = 0; w < NB32; ++w) {
                const uint32_t m = scw[(d * NB + w) * 32 + lane];
                if (m) last = (int16_t)(32 * w + 31 - __clz(m));
                slast[(d * NB + w) * 32 + lane] = last;
            }
            int16_t nxt = NONE_HI;
            for (int w = NB32 - 1; w >= 0; --w) {
                const uint32_t m = scw[(d * NB + w) * 32 + lane];
                if (m) nxt = (int16_t)(32 * w + __ffs(m) - 1);
                snext[(d * NB + w) * 32 + lane] = nxt;
            }
        }
        __syncthreads();
    }

    // ------------------------------------------------ 2. masks as bit words
    // outw[g][ob][lane]: bit r = mask of output position 32 ob + r of line lane
    for (int k = tid; k < kGroupViews * NOB * 32; k += NT) outw[k] = 0u;
    __syncthreads();
    if (!fs.nonfinite) {       // non-finite frame: masks stay zero
        // views without the default staged sweep: exact per-pixel routine
#pragma unroll 1
        for (int g = 0; g < gd.nv; ++g) {
            const ViewRegs cv = g == 0 ? vr[0] : vr[kGroupViews - 1];
            if (cv.staged && cv.nback == 2 && cv.jstar == 3 && cv.nfwd <= 1) continue;
            const ViewDesc vd = a.views[cv.vid];
            for (int k = tid; k < TPe * 32; k += NT) {
                const int32_t pos = P0 + (k >> 5), l = k & 31, ln = l0 + l;
                int32_t x, y;
                if (xm) { x = pos; y = ln + geo.fl(pos); }
                else { y = pos; x = ln + geo.fl(pos); }
                if (x >= 0 && x < W && y >= 0 && y < H &&
                    direct_pixel<false>(Df, H, W, vd, fd, p, cv.h, x, y))
                    atomicOr(&outw[(g * NOB + ((k >> 5) >> 5)) * 32 + l], 1u << ((k >> 5) & 31));
            }
        }
        // default thresholds: barrier-free bit-sliced sweeps of all views at
        // once; a warp owns (view, pair of adjacent 32-position blocks)
        const int32_t nob = (TPe + 31) >> 5, npair = (nob + 1) >> 1;
        for (int u = warp; u < gd.nv * npair; u += NWARP) {
            const int g = u / npair, pr = u - g * npair;
            const ViewRegs cv = g == 0 ? vr[0] : vr[kGroupViews - 1];
            if (!(cv.staged && cv.nback == 2 && cv.jstar == 3 && cv.nfwd <= 1)) continue;
            uint32_t *ow = outw + g * NOB * 32;
            const ViewDesc &vd = a.views[cv.vid];
            const float blo0 = vd.back_lo[0], bhi0 = vd.back_hi[0], blo1 = vd.back_lo[1],
                        bhi1 = vd.back_hi[1], flo0 = vd.fwd_lo[0], fhi0 = vd.fwd_hi[0];
            const int32_t blo = (L0 >> 5) + 2 * pr, bhi = min(blo + 1, (L0 >> 5) + nob - 1);
            const int32_t nb = bhi - blo + 1;
            const int d = cv.sg > 0 ? 0 : 1;
            const uint32_t *cwd = scw + d * NB * 32;
            const int16_t *ld = slast + d * NB * 32, *nd = snext + d * NB * 32;
            if (cv.sg > 0) {
                if (cv.nfwd)
                    sweep_bits<1, 1, VP>(sv, cwd, ld, nd, ow, sjg, lane, bhi, nb, L0, NP32, NB32, cv.h, cv.s,
                                         cv.T, cv.jr, blo0, bhi0, blo1, bhi1, flo0, fhi0, p.t_dist, p.t_disp);
                else
                    sweep_bits<1, 0, VP>(sv, cwd, ld, nd, ow, sjg, lane, bhi, nb, L0, NP32, NB32, cv.h, cv.s,
                                         cv.T, cv.jr, blo0, bhi0, blo1, bhi1, flo0, fhi0, p.t_dist, p.t_disp);
            } else {
                if (cv.nfwd)
                    sweep_bits<-1, 1, VP>(sv, cwd, ld, nd, ow, sjg, lane, blo, nb, L0, NP32, NB32, cv.h, cv.s,
                                          cv.T, cv.jr, blo0, bhi0, blo1, bhi1, flo0, fhi0, p.t_dist, p.t_disp);
                else
                    sweep_bits<-1, 0, VP>(sv, cwd, ld, nd, ow, sjg, lane, blo, nb, L0, NP32, NB32, cv.h, cv.s,
                                          cv.T, cv.jr, blo0, bhi0, blo1, bhi1, flo0, fhi0, p.t_dist, p.t_disp);
            }
        }
    }
    __syncthreads();

    // ------------------------------------------------ 3. store (row-contiguous)
    // mask bit of output position k (0 <= k < TPe) of line l
    auto bit_at = [&](const uint32_t *ow, int32_t k, int32_t l) -> uint32_t {
        return (ow[(k >> 5) * 32 + l] >> (k & 31)) & 1u;
    };
#pragma unroll 1
    for (int g = 0; g < gd.nv; ++g) {
        const uint32_t *ow = outw + g * NOB * 32;
        uint8_t *Mv = a.masks + ((int64_t)f * a.nviews + gd.view[g]) * a.mf.vbytes;
        if (a.mf.packed) {
            // bit-packed masks (pre-zeroed): set the marked pixels of the tile
            for (int k = tid; k < TPe * 32; k += NT) {
                const int32_t kk = k >> 5, l = k & 31;
                if (!bit_at(ow, kk, l)) continue;
                const int32_t pos = P0 + kk, ln = l0 + l;
                int32_t x, y;
                if (xm) { x = pos; y = ln + geo.fl(pos); }
                else { y = pos; x = ln + geo.fl(pos); }
                if (x >= 0 && x < W && y >= 0 && y < H) mask_put(Mv, a.mf, W, x, y, true);
            }
            continue;
        }
        const bool al4 = ((W & 3) == 0) && ((l0 & 3) == 0) && ((P0 & 3) == 0) && geo.num() == 0;
        if (!xm && al4) {
            // columns: output row y = P0 + k holds lanes l0..l0+31 -> 4 lanes per thread
            for (int t = tid; t < TPe * 8; t += NT) {
                const int32_t k = t >> 3, q = t & 7;
                const int32_t y = P0 + k, x = l0 + 4 * q;
                if (y >= H || x >= W) continue;
                uint32_t w = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) w |= bit_at(ow, k, 4 * q + e) << (8 * e);
                if (x + 3 < W) {
                    __stcs(reinterpret_cast<uint32_t *>(Mv + (int64_t)y * W + x), w);
                } else {
                    for (int e = 0; e < 4 && x + e < W; ++e) Mv[(int64_t)y * W + x + e] = (uint8_t)(w >> (8 * e));
                }
            }
            continue;
        }
        if (xm && al4) {
            // rows: row l0 + l, positions [P0, P1): 4 mask bits -> 4 bytes per store
            const int32_t nq = (TPe + 3) >> 2;
            for (int t = tid; t < 32 * nq; t += NT) {
                const int32_t l = t / nq, q = t - l * nq;
                const int32_t y = l0 + l, x = P0 + 4 * q;
                if (y >= H) continue;
                const uint32_t b4 = (ow[((4 * q) >> 5) * 32 + l] >> ((4 * q) & 31)) & 0xfu;
                const uint32_t w = (b4 * 0x00204081u) & 0x01010101u;     // bit e -> byte e
                if (x + 3 < P1) {
                    __stcs(reinterpret_cast<uint32_t *>(Mv + (int64_t)y * W + x), w);
                } else {
                    for (int e = 0; e < 4 && x + e < P1; ++e) Mv[(int64_t)y * W + x + e] = (uint8_t)(w >> (8 * e));
                }
            }
            continue;
        }
        if (!xm) {
            for (int k = warp; k < TPe; k += NWARP) {
                const int32_t y = P0 + k;
                if (y < 0 || y >= H) continue;
                const int32_t x = l0 + lane + geo.fl(y);
                if (x < 0 || x >= W) continue;
                __stcs(Mv + (int64_t)y * W + x, (uint8_t)bit_at(ow, k, lane));
            }
        } else {
            const int32_t xs = max(P0, 0), xe = min(P1, W) - 1;
            if (xs > xe) continue;
            if (geo.den() == 1 && (geo.num() == 1 || geo.num() == -1)) {
                // diagonals: row y = l0 + t, lane l at x = t - l (num = 1) / l - t
                const int32_t nm = geo.num();
                const int32_t tlo = nm > 0 ? xs : -xe, thi = nm > 0 ? xe + 31 : 31 - xs;
                for (int32_t t = max(tlo, -l0) + warp; t <= min(thi, H - 1 - l0); t += NWARP) {
                    const int32_t x = nm > 0 ? t - lane : lane - t;
                    if (x < xs || x > xe) continue;
                    __stcs(Mv + (int64_t)(l0 + t) * W + x, (uint8_t)bit_at(ow, x - P0, lane));
                }
                continue;
            }
            const int32_t fa = geo.fl(xs), fb = geo.fl(xe);
            const int32_t ylo = max(0, l0 + min(fa, fb)), yhi = min(H - 1, l0 + 31 + max(fa, fb));
            for (int32_t y = ylo + warp; y <= yhi; y += NWARP) {
                int32_t xa, xb;
                row_run(geo, y, l0, xs, xe, xa, xb);
                for (int32_t x = xa + lane; x <= xb; x += 32) {
                    const int32_t l = y - l0 - geo.fl(x);
                    __stcs(Mv + (int64_t)y * W + x, (uint8_t)bit_at(ow, x - P0, l));
                }
            }
        }
    }
}

// Family kinds with compile-time geometry (FamilyDesc::kind, set by the host):
// 0 rows, 1 columns, 2 diagonal, 3 anti-diagonal, 4/5 x-major knight +-1/2,
// 6/7 y-major knight +-1/2, 8 any other slope (runtime geometry).
template <int CB>
__global__ void __launch_bounds__(NT, 3) k_tile(TileArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const TileDesc td = a.tiles[blockIdx.x];
    const GroupDesc gd = a.groups[td.group];
    const FamilyDesc fd = a.fams[gd.fam];
    switch (fd.kind) {
        case 0: tile_body<GeoK<true, 0, 1>, CB, 33>(a, GeoK<true, 0, 1>(), td, gd, fd, smem); break;
        case 1: tile_body<GeoK<false, 0, 1>, CB, 33>(a, GeoK<false, 0, 1>(), td, gd, fd, smem); break;
        case 2: tile_body<GeoK<true, 1, 1>, CB, 34>(a, GeoK<true, 1, 1>(), td, gd, fd, smem); break;
        case 3: tile_body<GeoK<true, -1, 1>, CB, 34>(a, GeoK<true, -1, 1>(), td, gd, fd, smem); break;
        case 4: tile_body<GeoK<true, 1, 2>, CB, 34>(a, GeoK<true, 1, 2>(), td, gd, fd, smem); break;
        case 5: tile_body<GeoK<true, -1, 2>, CB, 34>(a, GeoK<true, -1, 2>(), td, gd, fd, smem); break;
        case 6: tile_body<GeoK<false, 1, 2>, CB, 33>(a, GeoK<false, 1, 2>(), td, gd, fd, smem); break;
        case 7: tile_body<GeoK<false, -1, 2>, CB, 33>(a, GeoK<false, -1, 2>(), td, gd, fd, smem); break;
        default: {
            GeoR g{fd.xmajor != 0, fd.num, fd.den};
            if (g.xm()) tile_body<GeoR, CB, 34>(a, g, td, gd, fd, smem);
            else tile_body<GeoR, CB, 33>(a, g, td, gd, fd, smem);
        }
    }
}

cudaError_t launch_tile(const float *D, int32_t H, int32_t W, int32_t batch,
                        const TileDesc *tiles, int32_t ntiles, const GroupDesc *groups,
                        const ViewDesc *views, int32_t nviews, const FamilyDesc *fams,
                        const FrameStats *st, const Params &p, uint8_t *masks, const MaskFmt &mf,
                        const void *codes, int32_t code_bytes, cudaStream_t s) {
    TileArgs a{D, H, W, tiles, groups, views, nviews, fams, st, p, masks, codes, mf};
    dim3 grid((unsigned)ntiles, (unsigned)batch);
    cudaError_t e;
    if (code_bytes == 1) {
        e = cudaFuncSetAttribute(k_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        k_tile<1><<<grid, NT, SMEM, s>>>(a);
    } else if (code_bytes == 2) {
        e = cudaFuncSetAttribute(k_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        k_tile<2><<<grid, NT, SMEM, s>>>(a);
    } else {
        e = cudaFuncSetAttribute(k_tile<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        k_tile<4><<<grid, NT, SMEM, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace occ
