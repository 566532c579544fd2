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
//   2. rank of every entry by counting smaller keys (w, index).  An entry q
//      with g_q - g_i > s (v_i - vmin) >= s (v_i - v_q) has exact w_q > w_i,
//      so (rounding is monotone, ties go by index) key_q > key_i without a
//      comparison, and symmetrically below; the count only visits
//      [i - ceil(s (vmax - v_i)), i + ceil(s (v_i - vmin))];
//   3. sorted[rank] = i; each sorted position r tests the pairs (r, r +- d),
//      d = 1..N/2, with pair_exact and marks the entry's pixel.
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
constexpr int kGran = 256;     // pixels per work granule

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
    double *gw;                // global scratch (big launch): [warp][cap] doubles
    float *gv;                 //                              [warp][cap] floats
    int32_t *gs;               //                              [warp][cap] ints
};

__device__ __forceinline__ uint32_t load_code(const void *codes, int32_t cb, int64_t i) {
    if (cb == 1) return reinterpret_cast<const uint8_t *>(codes)[i];
    if (cb == 2) return reinterpret_cast<const uint16_t *>(codes)[i];
    return reinterpret_cast<const uint32_t *>(codes)[i];
}

// One candidate window (warp-cooperative).  sw / sv / ss: this warp's
// storage (shared or global), at least n entries.
__device__ __forceinline__ void window(const NwinArgs &a, const float *__restrict__ Df, uint8_t *Mv,
                                   const ViewDesc &vd, int32_t h, int32_t cx, int32_t cy,
                                   double *sw, float *sv, int32_t *ss) {
    const int lane = threadIdx.x & 31;
    LineGeom lg;
    lg.init(vd, a.H, a.W, cx, cy);
    const int32_t uc = vd.sg * (vd.xmajor ? cx : cy);
    const int32_t s = vd.s;
    // 1. valid extent: sample g sits at u = uc - g (orc_scanline: x = cx - sg g)
    int32_t glo = INT_MAX, ghi = INT_MIN;
    for (int32_t g0 = -h; g0 <= h; g0 += 32) {
        const int32_t g = g0 + lane;
        int32_t xx, yy;
        const bool ok = g <= h && lg.at(uc - g, xx, yy);
        if (ok) { glo = min(glo, g); ghi = max(ghi, g); }
    }
    glo = __reduce_min_sync(0xffffffffu, glo);
    ghi = __reduce_max_sync(0xffffffffu, ghi);
    const int32_t n = ghi - glo + 1;        // >= 1: the candidate itself
    float vmin = INFINITY, vmax = -INFINITY;
    for (int32_t i = lane; i < n; i += 32) {
        const int32_t g = glo + i;
        int32_t xx, yy;
        lg.at(uc - g, xx, yy);
        const float v = __ldg(Df + (int64_t)yy * a.W + xx);
        sv[i] = v;
        sw[i] = __dadd_rn((double)g, __dmul_rn((double)s, (double)v));   // PAPER.md:127, W = G + s V
        vmin = fminf(vmin, v);
        vmax = fmaxf(vmax, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    __syncwarp();
    // 2. ranks by counting (ties by index), 3. scatter
    for (int32_t i = lane; i < n; i += 32) {
        const double wi = sw[i];
        const float vi = sv[i];
        // kd >= s (vmax - v_i): q < i - kd has w_q < w_i; ku >= s (v_i - vmin):
        // q > i + ku has w_q > w_i (rounded up: only >= is needed)
        const double kd = ceil(__dmul_ru((double)s, __dsub_ru((double)vmax, (double)vi)));
        const double ku = ceil(__dmul_ru((double)s, __dsub_ru((double)vi, (double)vmin)));
        const int32_t lo = kd >= (double)i ? 0 : i - (int32_t)kd;
        const int32_t hi = ku >= (double)(n - 1 - i) ? n - 1 : i + (int32_t)ku;
        int32_t rank = lo;
        for (int32_t q = lo; q < i; ++q) rank += sw[q] <= wi ? 1 : 0;   // ties: q < i counts
        for (int32_t q = i + 1; q <= hi; ++q) rank += sw[q] < wi ? 1 : 0;
        ss[rank] = i;
    }
    __syncwarp();
    const int32_t half = a.half;
    const float t_dist = a.p.t_dist, t_disp = a.p.t_disp;
    for (int32_t r = lane; r < n; r += 32) {
        const int32_t ip = ss[r];
        const float vp = sv[ip];
        bool hit = false;
        for (int32_t d = 1; d <= half && !hit; ++d) {
            if (r + d < n) {
                const int32_t iq = ss[r + d];
                hit = pair_exact(sv[iq], vp, iq - ip, s, t_dist, t_disp);   // dk = g_q - g_p
            }
            if (!hit && r - d >= 0) {
                const int32_t iq = ss[r - d];
                hit = pair_exact(sv[iq], vp, iq - ip, s, t_dist, t_disp);
            }
        }
        if (hit) {                                                       // Eq. 6
            int32_t xx, yy;
            lg.at(uc - (glo + ip), xx, yy);
            mask_put(Mv, a.mf, a.W, xx, yy, true);
        }
    }
    __syncwarp();
}

// kBig = false: windows of 2h + 1 <= cap entries, shared-memory storage;
// kBig = true: the longer ones, global scratch.
template <bool kBig>
__global__ void __launch_bounds__(32 * kNwinWarps) k_nwin(NwinArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *sw;
    float *sv;
    int32_t *ss;
    if (kBig) {
        const int64_t gw = (int64_t)blockIdx.x * kNwinWarps + wid;
        sw = a.gw + gw * a.cap;
        sv = a.gv + gw * a.cap;
        ss = a.gs + gw * a.cap;
    } else {
        unsigned char *base = smem + (size_t)wid * a.cap * 16;
        sw = reinterpret_cast<double *>(base);
        sv = reinterpret_cast<float *>(base + (size_t)a.cap * 8);
        ss = reinterpret_cast<int32_t *>(base + (size_t)a.cap * 12);
    }
    const int64_t HW = (int64_t)a.H * a.W;
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
        const float *Df = a.D + (int64_t)f * HW;
        const void *cf = a.codes;
        for (int32_t sub = 0; sub < kGran; sub += 32) {
            const int64_t pix = p0 + sub + lane;
            const uint32_t code = pix < HW ? load_code(cf, a.code_bytes, (int64_t)f * HW + pix) : 0u;
            if (__ballot_sync(0xffffffffu, code != 0u) == 0u) continue;
            for (int32_t vi = 0; vi < a.nviews; ++vi) {
                const ViewDesc &vd = a.views[vi];
                const int32_t h = view_h(R, vd.s, a.p.max_scan);
                if (h <= 0) continue;                   // Q17: no window, no marks
                if ((2 * h + 1 > kNwinCap) != kBig) continue;   // the other launch's window
                uint32_t cand = __ballot_sync(0xffffffffu, (code >> vd.candbit) & 1u);
                uint8_t *Mv = a.masks + ((int64_t)f * a.nviews + vi) * a.mf.vbytes;
                while (cand) {
                    const int b = __ffs(cand) - 1;
                    cand &= cand - 1;
                    const int64_t pc = p0 + sub + b;
                    const int32_t cy = (int32_t)(pc / a.W), cx = (int32_t)(pc - (int64_t)cy * a.W);
                    window(a, Df, Mv, vd, h, cx, cy, sw, sv, ss);
                }
            }
        }
    }
}

}  // namespace

size_t nwin_smem_bytes() { return (size_t)kNwinWarps * kNwinCap * 16; }

cudaError_t launch_nwin(const float *D, int32_t H, int32_t W, int32_t frames, const ViewDesc *views,
                        int32_t nviews, const FrameStats *st, const Params &p, int32_t N, uint8_t *masks,
                        const MaskFmt &mf, const void *codes, int32_t code_bytes, uint32_t *work,
                        NwinScratch &big, int32_t nsm, cudaStream_t s) {
    NwinArgs a{};
    a.D = D; a.H = H; a.W = W; a.frames = frames;
    a.codes = codes; a.code_bytes = code_bytes;
    a.views = views; a.nviews = nviews; a.st = st; a.p = p; a.half = N / 2;
    a.masks = masks; a.mf = mf;
    a.gpf = ((int64_t)H * W + kGran - 1) / kGran;
    a.ngran = a.gpf * frames;
    static int occ_blocks = 0;
    const size_t smem = nwin_smem_bytes();
    if (!occ_blocks) {
        cudaError_t e = cudaFuncSetAttribute(k_nwin<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_blocks, k_nwin<false>, 32 * kNwinWarps, smem);
        if (e != cudaSuccess) return e;
        if (occ_blocks < 1) occ_blocks = 1;
    }
    cudaError_t e = cudaMemsetAsync(work, 0, 2 * sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    a.work = work;
    a.cap = kNwinCap;
    k_nwin<false><<<nsm * occ_blocks, 32 * kNwinWarps, smem, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // windows longer than kNwinCap (h > (kNwinCap - 1) / 2): global scratch
    // sized for the largest window max_scan allows
    const int32_t capbig = 2 * (p.max_scan / 2) + 1;
    if (capbig <= kNwinCap) return cudaSuccess;
    const int32_t blocks = nsm;
    const size_t need = (size_t)blocks * kNwinWarps * capbig;
    if (big.entries < need) {
        cudaFree(big.w); cudaFree(big.v); cudaFree(big.s);
        big.w = nullptr; big.v = nullptr; big.s = nullptr; big.entries = 0;
        if ((e = cudaMalloc(&big.w, need * sizeof(double))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&big.v, need * sizeof(float))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&big.s, need * sizeof(int32_t))) != cudaSuccess) return e;
        big.entries = need;
    }
    a.work = work + 1;
    a.cap = capbig;
    a.gw = big.w; a.gv = big.v; a.gs = big.s;
    k_nwin<true><<<blocks, 32 * kNwinWarps, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace occ
