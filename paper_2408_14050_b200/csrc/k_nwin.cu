// k_nwin.cu -- the detector with a finite neighbour count N (SURVEY §8(f)
// NEXT #1; occ_set_neighbors).  PAPER.md:131-142 (Eq. 5) read literally:
// every candidate C_i owns the scan window S_i = C_i + G (Eq. 4, h from
// Eq. 3), whose warped coordinates W = G + s V are sorted
// (ties by scan index); each sorted entry is
// compared with the N/2 entries on either side (beyond the line
// skipped) by the pair test S7, and Eq. 6 marks the entries with a positive
// count.  With finite N the marks depend on the whole window (which entries
// sit between two partners), so this path works per candidate window, not
// per pixel like k_line.
//
// One warp per window, persistent CTAs pulling 256-pixel granules of the
// candidate codes (K0) from an atomic counter:
//   1. the window's valid extent [glo, ghi] (the digital line clipped to the
//      image is one interval of g), v = D on it, w = fl64(g + s v) -- the
//      same binary64 value the oracle sorts;
//   2. rank of every entry under (w, index): the window splits into runs of
//      non-decreasing w; an entry's rank sums, over the runs, the entries
//      below it (own run: its offset; other runs: all, none, or one binary
//      search).  Windows with many runs count directly over the g-range
//      outside which the order is fixed by g alone;
//   3. sorted[rank] = i; every unordered pair of sorted positions
//      {r, r + d}, d = 1..N/2, gets one Eq. 5 test serving both orientations
//      (the d loop stops once the warped distances exceed t_dist + eps), and
//      the flagged entries' pixels are marked.
// Masks are zeroed before the launch; the kernel only sets 1s (u8 byte
// stores or atomicOr on packed words), so overlapping windows OR their marks.
//
// Windows of up to kNwinCap entries live in shared memory; frames whose h
// gives longer windows go to the same code with a per-warp slice of global
// scratch (second launch, small grid).
#include <climits>

#include "occ_device.cuh"

namespace occ {

namespace {

constexpr int kNwinWarps = 8;
#ifndef NWIN_GRAN
#define NWIN_GRAN 32
#endif
constexpr int kGran = NWIN_GRAN;   // pixels per work granule
constexpr int kMaxRuns = 24;   // run-merge ranking up to this many runs per window

struct NwinArgs {
    const float *D;
    int32_t H, W, frames;
    const void *codes;
    int32_t code_bytes;
    const ViewDesc *views;
    int32_t nviews;
    const FrameStats *st;
    Params p;
    int32_t half;              // N / 2
    uint8_t *masks;
    MaskFmt mf;
    uint32_t *work;            // granule counter (zeroed before the launch)
    int64_t ngran, gpf;        // granules total / per frame
    int32_t cap;               // window capacity of the storage this launch uses
    unsigned char *gbuf;       // global scratch (big launch): [warp][cap * kNwinEntryBytes]
    int32_t smax;              // largest ||b||_inf (ceil of the length) of the views
    int32_t angles;            // real-valued directions: candidates computed here (Eq. 1-2)
    const int2 *offs;          // their Eq. 4 offset tables
};

// Eq. 3 with the W scale rho (rho = s for grid baselines: equal to view_h)
__device__ __forceinline__ int32_t view_h_rho(float R, double rho, int32_t cap) {
    double L = ceil(__dmul_rn(__dmul_rn(2.0, rho), (double)R));
    if (!(L <= (double)cap)) L = (double)cap;
    return ((int32_t)L) >> 1;
}

// Per-warp window storage, kNwinEntryBytes per entry: w (binary64), v,
// sorted index, run starts.  cap is even, so every warp's slice stays
// 8-byte aligned.
struct WinBuf {
    double *w;
    float *v;
    int32_t *s, *run;
};
__device__ __forceinline__ WinBuf carve(unsigned char *base, int32_t cap) {
    WinBuf b;
    b.w = reinterpret_cast<double *>(base);
    b.v = reinterpret_cast<float *>(base + (size_t)cap * 8);
    b.s = reinterpret_cast<int32_t *>(base + (size_t)cap * 12);
    b.run = reinterpret_cast<int32_t *>(base + (size_t)cap * 16);
    return b;
}

__device__ __forceinline__ uint32_t load_code(const void *codes, int32_t cb, int64_t i) {
    if (cb == 1) return reinterpret_cast<const uint8_t *>(codes)[i];
    if (cb == 2) return reinterpret_cast<const uint16_t *>(codes)[i];
    return reinterpret_cast<const uint32_t *>(codes)[i];
}

__device__ __forceinline__ int32_t fdiv(int32_t a, int32_t den) {   // floor(a / den), den > 0
    return den == 1 ? a : (den == 2 ? (a >> 1) : floordiv(a, den));
}

// Sample g of a candidate's scan window (Eq. 4): grid baselines walk the
// digital line (S6: major coordinate pc - sg g, orc_scanline's x = cx - sg g,
// minor line + floor(major num / den)); real-valued directions add the
// host-computed rounded offset of g u (reading Q23).  false: outside the image.
struct Geo {
    int32_t angle, X, sg, num, den, pc, line, nmaj, nmin, cx, cy, W, H;
    const int2 *off;      // angle: offsets, indexed by g (centred)
    __device__ __forceinline__ void init(const NwinArgs &a, const ViewDesc &vd, int32_t x, int32_t y) {
        angle = vd.angle; cx = x; cy = y; W = a.W; H = a.H;
        X = vd.xmajor; sg = vd.sg; num = vd.num; den = vd.den;
        pc = X ? x : y;
        line = angle ? 0 : (X ? y - fdiv(x * num, den) : x - fdiv(y * num, den));
        nmaj = X ? W : H; nmin = X ? H : W;
        off = angle ? a.offs + vd.off_base + a.p.max_scan / 2 : nullptr;
    }
    __device__ __forceinline__ bool at(int32_t g, int32_t &x, int32_t &y) const {
        if (angle) {
            const int2 o = __ldg(off + g);
            x = cx + o.x; y = cy + o.y;
            return x >= 0 && x < W && y >= 0 && y < H;
        }
        const int32_t mj = pc - sg * g;
        const int32_t mn = line + fdiv(mj * num, den);
        x = X ? mj : mn; y = X ? mn : mj;
        return mj >= 0 && mj < nmaj && mn >= 0 && mn < nmin;
    }
};

// One candidate window (warp-cooperative).
__device__ __forceinline__ void window(const NwinArgs &a, const float *__restrict__ Df, uint8_t *Mv,
                                       const ViewDesc &vd, int32_t h, int32_t cx, int32_t cy,
                                       const WinBuf &B) {
    const int lane = threadIdx.x & 31;
    Geo geo;
    geo.init(a, vd, cx, cy);
    const double rho = vd.rho;          // W = G + rho V (rho = s for grid baselines)
    // 1. valid extent (the clipped line is one interval of g: the in-image
    // test of a rounded point moving along a straight line is monotone)
    int32_t glo = INT_MAX, ghi = INT_MIN;
    if (!geo.angle && geo.den == 1 && geo.num >= -1 && geo.num <= 1) {
        // rows / columns / diagonals: major coordinate mj = pc - sg g in
        // [0, nmaj) and minor line + num mj in [0, nmin), in closed form
        int32_t lo = 0, hi = geo.nmaj - 1;
        if (geo.num == 1) { lo = max(lo, -geo.line); hi = min(hi, geo.nmin - 1 - geo.line); }
        if (geo.num == -1) { lo = max(lo, geo.line - geo.nmin + 1); hi = min(hi, geo.line); }
        // mj in [lo, hi]  <=>  g in [pc - hi, pc - lo] (sg = 1) or [lo - pc, hi - pc] (sg = -1)
        glo = max(-h, geo.sg > 0 ? geo.pc - hi : lo - geo.pc);
        ghi = min(h, geo.sg > 0 ? geo.pc - lo : hi - geo.pc);
    } else {
        for (int32_t g0 = -h; g0 <= h; g0 += 32) {
            const int32_t g = g0 + lane;
            int32_t xx, yy;
            if (g <= h && geo.at(g, xx, yy)) { glo = min(glo, g); ghi = max(ghi, g); }
        }
        glo = __reduce_min_sync(0xffffffffu, glo);
        ghi = __reduce_max_sync(0xffffffffu, ghi);
    }
    const int32_t n = ghi - glo + 1;        // >= 1: the candidate itself
    // 2. V = D on the window, W = fl64(G + fl64(rho V))
    float vmin = INFINITY, vmax = -INFINITY;
    for (int32_t i0 = 0; i0 < n; i0 += 128) {      // 4 gathers in flight per lane
        float vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t i = i0 + 32 * u + lane;
            int32_t xx = 0, yy = 0;
            if (i < n) geo.at(glo + i, xx, yy);
            vv[u] = i < n ? __ldg(Df + (int64_t)yy * a.W + xx) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t i = i0 + 32 * u + lane;
            if (i < n) {
                B.v[i] = vv[u];
                B.w[i] = __dadd_rn((double)(glo + i), __dmul_rn(rho, (double)vv[u]));
                vmin = fminf(vmin, vv[u]);
                vmax = fmaxf(vmax, vv[u]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    __syncwarp();
    // 3. rank of every entry under the key (w, index).  The window splits
    // into maximal runs of non-decreasing w (keys increasing); the rank of
    // w_i is the sum over runs of the entries below it: the run holding i
    // contributes i - start, a run wholly below / above contributes all / none,
    // the rest one binary search.  Inside smooth regions w grows by about 1
    // per sample, so a window has a few runs (one more per depth edge whose
    // near side comes first).  Windows with more than kMaxRuns runs (noise
    // at s >= 2, random maps) count directly: q with g_q - g_i >= rho (v_i -
    // vmin) + 1 >= rho (v_i - v_q) + 1 has w_q > w_i (the exact difference is
    // >= 1, far above the roundings of w), so key_q > key_i without a
    // comparison; symmetrically below.
    int32_t m = 0;
    for (int32_t b0 = 0; b0 < n; b0 += 32) {
        const int32_t i = b0 + lane;
        const bool st = i < n && (i == 0 || B.w[i] < B.w[i - 1]);
        const uint32_t bal = __ballot_sync(0xffffffffu, st);
        if (st) B.run[m + __popc(bal & ((1u << lane) - 1u))] = i;
        m += __popc(bal);
    }
    __syncwarp();
    if (m <= kMaxRuns) {
        for (int32_t i = lane; i < n; i += 32) {
            const double wi = B.w[i];
            int32_t rank = 0;
            for (int32_t k = 0; k < m; ++k) {
                const int32_t ra = B.run[k], rb = (k + 1 < m ? B.run[k + 1] : n) - 1;
                if (i >= ra && i <= rb) { rank += i - ra; continue; }
                const double wa = B.w[ra], wb = B.w[rb];
                if (rb < i) {                     // keys below w_i: w_q <= w_i
                    if (wb <= wi) { rank += rb - ra + 1; continue; }
                    if (!(wa <= wi)) continue;
                    int32_t lo = ra + 1, hi = rb;     // first q in (ra, rb] with w_q > w_i
                    while (lo < hi) { const int32_t md = (lo + hi) >> 1; if (B.w[md] > wi) hi = md; else lo = md + 1; }
                    rank += lo - ra;
                } else {                          // keys below w_i: w_q < w_i
                    if (wb < wi) { rank += rb - ra + 1; continue; }
                    if (!(wa < wi)) continue;
                    int32_t lo = ra + 1, hi = rb;     // first q in (ra, rb] with w_q >= w_i
                    while (lo < hi) { const int32_t md = (lo + hi) >> 1; if (B.w[md] >= wi) hi = md; else lo = md + 1; }
                    rank += lo - ra;
                }
            }
            B.s[rank] = i;
        }
    } else {
        for (int32_t i = lane; i < n; i += 32) {
            const double wi = B.w[i];
            const float vi = B.v[i];
            const double kd = ceil(__dmul_ru(rho, __dsub_ru((double)vmax, (double)vi))) + 1.0;
            const double ku = ceil(__dmul_ru(rho, __dsub_ru((double)vi, (double)vmin))) + 1.0;
            const int32_t lo = kd >= (double)i ? 0 : i - (int32_t)kd;
            const int32_t hi = ku >= (double)(n - 1 - i) ? n - 1 : i + (int32_t)ku;
            int32_t rank = lo;
            for (int32_t q = lo; q < i; ++q) rank += B.w[q] <= wi ? 1 : 0;   // ties: q < i counts
            for (int32_t q = i + 1; q <= hi; ++q) rank += B.w[q] < wi ? 1 : 0;
            B.s[rank] = i;
        }
    }
    __syncwarp();
    // 4. Eq. 5 over the sorted neighbours d = 1..N/2, one test
    // per unordered pair {r, r + d}: with delta = fl32(v_hi - v_lo) the
    // reversed orientation has delta' = -delta exactly and the same warped
    // distance |dk + s delta|, so one distance test serves both; the entry
    // with the smaller disparity is marked when |delta| > t_disp.  Per chunk
    // of 32 sorted positions the d loop ends once no lane's pair is within
    // t_dist + eps in w (sorted: further d are further in w; eps bounds every
    // rounding of w and of s delta vs s (v_q - v_p), the oracle's bound of
    // DESIGN.md §2.3 with the window's max |v|).  Flags in the run slots.
    const int32_t half = a.half;
    const float t_dist = a.p.t_dist, t_disp = a.p.t_disp;
    const double M = fmax(fabs((double)vmin), fabs((double)vmax));
    const double lim = __dadd_rn((double)t_dist, __dmul_rn(0x1p-16, __dadd_rn(__dmul_rn(rho, M), 1.0)));
    int32_t *hit = B.run;
    for (int32_t r = lane; r < n; r += 32) hit[r] = 0;
    __syncwarp();
    for (int32_t r0 = 0; r0 < n - 1; r0 += 32) {
        const int32_t r = r0 + lane;
        const int32_t ip = r < n ? B.s[r] : 0;
        const float vp = B.v[ip];
        const double wp = B.w[ip];
        bool hp = false;
        for (int32_t d = 1; d <= half; ++d) {
            const int32_t rq = r + d;
            bool near = false;
            if (rq < n) {
                const int32_t iq = B.s[rq];
                near = __dsub_rn(B.w[iq], wp) < lim;
                if (near) {
                    const float delta = __fsub_rn(B.v[iq], vp);
                    const bool pq = delta > t_disp, qp = -delta > t_disp;   // only then the distance
                    if (pq || qp) {
                        const int32_t dk = iq - ip;                    // g_q - g_p
                        const double x = __dmul_rn(rho, (double)delta);
                        if (x > __dsub_rn(-(double)t_dist, (double)dk) && x < __dsub_rn((double)t_dist, (double)dk)) {
                            if (pq) hp = true;                         // p behind q
                            else hit[rq] = 1;                          // q behind p
                        }
                    }
                }
            }
            if (!__any_sync(0xffffffffu, near)) break;
        }
        __syncwarp();
        if (hp) hit[r] = 1;
    }
    __syncwarp();
    for (int32_t r = lane; r < n; r += 32) {
        if (!hit[r]) continue;                                           // Eq. 6
        int32_t xx, yy;
        geo.at(glo + B.s[r], xx, yy);
        mask_put(Mv, a.mf, a.W, xx, yy, true);
    }
    __syncwarp();
}

// kBig = false: windows of 2h + 1 <= kNwinCap entries, shared-memory
// storage; kBig = true: the longer ones, global scratch.
template <bool kBig>
__global__ void __launch_bounds__(32 * kNwinWarps) k_nwin(NwinArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t wbytes = (size_t)a.cap * kNwinEntryBytes;
    const WinBuf B = kBig ? carve(a.gbuf + ((size_t)blockIdx.x * kNwinWarps + wid) * wbytes, a.cap)
                          : carve(smem + (size_t)wid * wbytes, a.cap);
    const int64_t HW = (int64_t)a.H * a.W;
    if (kBig) {     // nothing to do unless some frame has a window longer than kNwinCap
        bool need = false;
        for (int32_t f = lane; f < a.frames; f += 32) {
            const FrameStats fs = a.st[f];
            need |= !fs.nonfinite && 2 * view_h(frame_range(fs), a.smax, a.p.max_scan) + 1 > kNwinCap;
        }
        if (!__any_sync(0xffffffffu, need)) return;
    }
    for (;;) {
        int64_t gi = 0;
        if (lane == 0) gi = atomicAdd(a.work, 1u);
        gi = __shfl_sync(0xffffffffu, gi, 0);
        if (gi >= a.ngran) break;
        const int32_t f = (int32_t)(gi / a.gpf);
        const int64_t p0 = (gi - (int64_t)f * a.gpf) * kGran;
        const FrameStats fs = a.st[f];
        if (fs.nonfinite) continue;                     // masks stay zero
        const float R = frame_range(fs);
        if (kBig && 2 * view_h(R, a.smax, a.p.max_scan) + 1 <= kNwinCap) continue;
        const float *Df = a.D + (int64_t)f * HW;
        for (int32_t sub = 0; sub < kGran; sub += 32) {
            const int64_t pix = p0 + sub + lane;
            uint32_t code = 0u;
            float ex = 0.0f, ey = 0.0f;
            if (a.angles) {
                // real-valued directions: Eq. 1 and E > t_e here (the squared
                // exact threshold, as K0), the direction test per view below
                if (pix < HW) {
                    const int32_t y = (int32_t)(pix / a.W), x = (int32_t)(pix - (int64_t)y * a.W);
                    const float c = __ldg(Df + pix);
                    ex = x + 1 < a.W ? __fsub_rn(__ldg(Df + pix + 1), c) : 0.0f;
                    ey = y + 1 < a.H ? __fsub_rn(__ldg(Df + pix + a.W), c) : 0.0f;
                    code = __fadd_rn(__fmul_rn(ex, ex), __fmul_rn(ey, ey)) > a.p.e2_thresh ? 1u : 0u;
                }
            } else {
                code = pix < HW ? load_code(a.codes, a.code_bytes, (int64_t)f * HW + pix) : 0u;
            }
            if (__ballot_sync(0xffffffffu, code != 0u) == 0u) continue;
            for (int32_t vi = 0; vi < a.nviews; ++vi) {
                const ViewDesc &vd = a.views[vi];
                const int32_t h = view_h_rho(R, vd.rho, a.p.max_scan);
                if (h <= 0) continue;                   // Q17: no window, no marks
                if ((2 * h + 1 > kNwinCap) != kBig) continue;   // the other launch's window
                // Eq. 2: grid baselines from the K0 codes; directions as
                // fl64(cos phi E_x) + fl64(sin phi E_y) > 0 (reading Q23)
                const bool isc = a.angles ? (code != 0u && __dadd_rn(__dmul_rn(vd.ca, (double)ex),
                                                                     __dmul_rn(vd.sa, (double)ey)) > 0.0)
                                          : ((code >> vd.candbit) & 1u) != 0u;
                uint32_t cand = __ballot_sync(0xffffffffu, isc);
                uint8_t *Mv = a.masks + ((int64_t)f * a.nviews + vi) * a.mf.vbytes;
                while (cand) {
                    const int b = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const int64_t pc = p0 + sub + b;
                    const int32_t cy = (int32_t)(pc / a.W), cx = (int32_t)(pc - (int64_t)cy * a.W);
                    window(a, Df, Mv, vd, h, cx, cy, B);
                }
            }
        }
    }
}

}  // namespace

size_t nwin_smem_bytes() { return (size_t)kNwinWarps * kNwinCap * kNwinEntryBytes; }

cudaError_t launch_nwin(const float *D, int32_t H, int32_t W, int32_t frames, const ViewDesc *views,
                        int32_t nviews, const FrameStats *st, const Params &p, int32_t N, uint8_t *masks,
                        const MaskFmt &mf, const void *codes, int32_t code_bytes, uint32_t *work,
                        NwinScratch &big, int32_t smax, int32_t angles, const int2 *offs, int32_t nsm,
                        cudaStream_t s) {
    NwinArgs a{};
    a.smax = smax;
    a.angles = angles;
    a.offs = offs;
    a.D = D; a.H = H; a.W = W; a.frames = frames;
    a.codes = codes; a.code_bytes = code_bytes;
    a.views = views; a.nviews = nviews; a.st = st; a.p = p;
    a.half = N > 0 ? N / 2 : (1 << 30);     // N = 0: infinity (every pair within t_dist + eps)
    a.masks = masks; a.mf = mf;
    a.gpf = ((int64_t)H * W + kGran - 1) / kGran;
    a.ngran = a.gpf * frames;
    const size_t smem = nwin_smem_bytes();
    // per-device attribute and occupancy (current device; computed per call:
    // cheap host queries, no static state shared between devices or threads)
    cudaError_t e = cudaFuncSetAttribute(k_nwin<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ_blocks = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, k_nwin<false>, 32 * kNwinWarps, smem);
    if (e != cudaSuccess) return e;
    if (occ_blocks < 1) occ_blocks = 1;
    e = cudaMemsetAsync(work, 0, 2 * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    a.work = work;
    a.cap = kNwinCap;
    k_nwin<false><<<nsm * occ_blocks, 32 * kNwinWarps, smem, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // windows longer than kNwinCap (h > (kNwinCap - 1) / 2): global scratch
    // sized for the largest window max_scan allows
    const int32_t capbig = 2 * (p.max_scan / 2) + 2;   // even: 8-byte aligned slices
    if (capbig <= kNwinCap) return cudaSuccess;
    const int32_t blocks = nsm;
    const size_t need = (size_t)blocks * kNwinWarps * capbig * kNwinEntryBytes;
    if (big.bytes < need) {
        cudaFree(big.buf);
        big.buf = nullptr;
        big.bytes = 0;
        if ((e = cudaMalloc(&big.buf, need)) != cudaSuccess) return e;
        big.bytes = need;
    }
    a.work = work + 1;
    a.cap = capbig;
    a.gbuf = big.buf;
    k_nwin<true><<<blocks, 32 * kNwinWarps, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace occ
