// occ_internal.h -- device-side descriptors shared by the host library and
// the sm_100a kernels of libocc.  Product code only (never includes oracle/).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/occ.h"

// OCC_CHECKS builds (OCC_DEFINES=-DOCC_CHECKS): device-side bounds checks
// of every queue entry, staged / listed index and mask write, before the
// access (compute-sanitizer is closed on the GPU pool).  A failed check
// prints the condition and traps (the call then reports OCC_ERR_CUDA).
#ifdef OCC_CHECKS
#include <cstdio>
#define OCC_CHECK(c)                                                                          \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("OCC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define OCC_CHECK(c) do { } while (0)
#endif

namespace occ {

constexpr int kMaxViews = 64;
constexpr int kMaxFamilies = 16;
constexpr int kMaxNear = 8;        // near partners handled by fp32 thresholds

// One peripheral view (baseline b).  Geometry of its digital epipolar lines
// (SURVEY §8.0 S6): x-major when |bx| >= |by|: pos = x, line = y - floor(x num/den);
// y-major: pos = y, line = x - floor(y num/den).  u = sg * pos increases toward
// the "backward" partners (the side the occluders of this view come from).
struct ViewDesc {
    int32_t bx, by;
    int32_t s;          // ||b||_inf (Eq. 3 / W scaling, readings Q6, Q9)
    int32_t xmajor;     // 1: pos = x
    int32_t sg;         // sign of the major component of b (+1 / -1)
    int32_t num, den;   // reduced slope of the family (den > 0)
    int32_t fam;        // family index (lines shared by +-m b0)
    int32_t candbit;    // bit of the per-pixel candidate code: 2*fam + (sg < 0)
    int32_t lkind;      // k_line geometry of its family (0 rows .. 3 anti-diagonals; 8 other)
    int32_t jstar;      // first backward offset whose Eq. 5 test implies delta > t_disp
    int32_t nback;      // near backward offsets j = 1..nback (nback = jstar-1)
    int32_t nfwd;       // near forward offsets f = 1..nfwd
    // exact fp32 thresholds: delta in (lo, hi) <=> Eq. 5 test holds
    float back_lo[kMaxNear], back_hi[kMaxNear];   // dk = -j, j = 1..nback
    float fwd_lo[kMaxNear], fwd_hi[kMaxNear];     // dk = +f, f = 1..nfwd
    // W scaling (Eq. 4 / W): rho = s for grid baselines, the Euclidean length
    // for real-valued directions (occ_create_dirs, reading Q23)
    double rho;
    int32_t angle;      // 1: real-valued direction (k_nwin only)
    int32_t off_base;   // its offset table: entries [off_base, off_base + 2 (max_scan / 2) + 1)
    double ca, sa;      // cos / sin of the baseline angle (Eq. 2)
    double ux, uy;      // displacement unit vector (-ca, -sa)
};

struct FamilyDesc {
    int32_t b0x, b0y;   // reduced base direction, major component > 0
    int32_t xmajor, num, den;
    int32_t kind;       // compile-time geometry variant of k_tile (8 = runtime)
    int32_t nviews;
    int32_t view[kMaxViews];   // indices into ViewDesc[]
};

// Tiled kernel work decomposition (k_tile.cu): a group is <= 2 views of one
// family sharing staged data; a tile is 32 consecutive lines x TP positions.
constexpr int kGroupViews = 2;
struct GroupDesc {
    int32_t fam, nv;
    int32_t view[kGroupViews];
};
struct TileDesc {
    int32_t group, l0, p0, p1;   // lines [l0, l0+32), output positions [p0, p1)
};

struct Params {
    float t_edge, t_dist, t_disp;
    int32_t max_scan;
    float e2_thresh;    // largest fp32 x with sqrt_rn(x) <= t_edge: E > t_e <=> e2 > e2_thresh
};

// Mask output format (occ_set_mask_format): uint8 [H][W] per (frame, view),
// or bit-packed: [H][Wb] 32-bit words, Wb = ceil(W / 32), bit x & 31 of word
// (y, x >> 5) = mask of pixel (x, y), padding bits 0.  vbytes = bytes per
// (frame, view) plane.  Packed planes are zeroed before the kernels run and
// only set bits are written (atomicOr where two writers share a word).
struct MaskFmt {
    int32_t packed, Wb;
    int64_t vbytes;
};
#ifdef __CUDACC__
__device__ __forceinline__ void mask_put(uint8_t *Mv, const MaskFmt &m, int32_t W, int32_t x, int32_t y, bool v) {
    if (m.packed) {
        if (v) atomicOr(reinterpret_cast<unsigned int *>(Mv) + (int64_t)y * m.Wb + (x >> 5), 1u << (x & 31));
    } else {
        Mv[(int64_t)y * W + x] = (uint8_t)v;
    }
}
#endif

// Per-frame statistics written by k_stats (S1) -- ordered-int keys so that
// atomicMin/atomicMax give the exact fp32 min/max.
struct FrameStats {
    int32_t minkey, maxkey;
    uint32_t nonfinite;
    int32_t pad;
};

__host__ __device__ inline int32_t float_key(float f) {
#ifdef __CUDA_ARCH__
    int32_t b = __float_as_int(f);
#else
    int32_t b; memcpy(&b, &f, 4);
#endif
    return b >= 0 ? b : (b ^ 0x7FFFFFFF);
}
__host__ __device__ inline float key_float(int32_t k) {
    int32_t b = k >= 0 ? k : (k ^ 0x7FFFFFFF);
#ifdef __CUDA_ARCH__
    return __int_as_float(b);
#else
    float f; memcpy(&f, &b, 4); return f;
#endif
}

__host__ __device__ inline int32_t floordiv(int32_t a, int32_t d) {   // d > 0
    int32_t q = a / d;
    if ((a % d) != 0 && a < 0) q -= 1;
    return q;
}

// Launchers (k_*.cu)
cudaError_t launch_stats_init(FrameStats *st, int32_t batch, cudaStream_t s);
cudaError_t launch_stats(const float *D, int64_t HW, int32_t batch, FrameStats *st, cudaStream_t s);
cudaError_t launch_direct(const float *D, int32_t H, int32_t W, int32_t batch,
                          const ViewDesc *views, int32_t nviews, const FamilyDesc *fams,
                          const FrameStats *st, const Params &p, uint8_t *masks, const MaskFmt &mf,
                          cudaStream_t s);
size_t tile_smem_bytes();
constexpr int64_t kTinyPixelViews = 1 << 16;   // AUTO: per-pixel kernel for calls this small
constexpr int kTilePositions = 160;    // TP (5 blocks of 32: with the 128 halo, smem for 3 CTAs per SM)
constexpr int kTileHaloMax = 128;      // staged halo per side (multiple of 32): C4 knights need 97
cudaError_t launch_tile(const float *D, int32_t H, int32_t W, int32_t batch,
                        const TileDesc *tiles, int32_t ntiles, const GroupDesc *groups,
                        const ViewDesc *views, int32_t nviews, const FamilyDesc *fams,
                        const FrameStats *st, const Params &p, uint8_t *masks, const MaskFmt &mf,
                        const void *codes, int32_t code_bytes, cudaStream_t s);
// Line-sweep kernel (k_line.cu) for the four line families of |b| <= 1
// arrays: one warp per unit = 32 consecutive lines x [t0, t1) in the lane's
// time coordinate (t0, t1 multiples of 32, t1 - t0 <= kLineSeg).
constexpr int kLineSeg = 256;
constexpr int kLineCandMarginWords = 4;  // candidate words staged beyond the segment (h + 32 <= 128)
struct LineUnit {
    int32_t group, l0, t0, t1;
};
// An exhaustive far-partner search deferred to k_hard (16 bytes): survivor at
// pixel index pix of frame f (of the chunk), view v; partners at
// pix + j * sg(v) * stride(kind(v)), j = 3 .. jm (dcov clipped to the image).
// meta = jm | v << 25 (jm <= 2 * (65536 / 2) < 2^17, v < 128);
// guess = j | f << 17 (j < 2^17 the sweep's failed probe offset or 0, f < 2^15).
// A knight family served by k_sweep through a sheared copy of D (k_shear):
// kind = the sweep kind its lines become (0 rows: x-major, 1 columns:
// y-major); image line l = sheared line + lmin; f(t) = floor(t num / den).
struct ShearDesc {
    int32_t kind, num, den, lmin, Ho, Wo;
};
struct HardEntry {
    int32_t pix;
    uint32_t meta;
    int32_t guess;      // offset of the sweep's failed probe (0: none) | frame << 17
    float vq;           // the value it read (k_hard starts at its fixed point s (vq - v_p))
};
constexpr int kMaxChunkFrames = 4096;    // frames per chunk (HardEntry's f: 15 bits)
// Candidate words precomputed per chunk by k_cand (one entry per family;
// families without line units have nlb = nk = 0): blocks of 32 lines x 32
// positions, [frame][base_slot + lb * nk + (k - kmin)][view 2][lane 32] uint32.
struct CandFam {
    int32_t fam, kind, lmin, nlb, kmin, nk;
    int64_t base_slot, per_frame;
};
cudaError_t launch_cand(const float *D, int32_t H, int32_t W, int32_t frames, const void *codes, int32_t code_bytes,
                        const CandFam *cf, int32_t ncf, int64_t per_frame, uint32_t *cand, cudaStream_t s);
size_t line_smem_bytes();
cudaError_t launch_line(const float *D, int32_t H, int32_t W, int32_t batch, const LineUnit *units,
                        int32_t nunits, const GroupDesc *groups, const ViewDesc *views, int32_t nviews,
                        const FamilyDesc *fams, const FrameStats *st, const Params &p, uint8_t *masks,
                        const MaskFmt &mf, const void *codes, int32_t code_bytes, unsigned long long *dbg,
                        HardEntry *gq, uint32_t *gq_count, int32_t gq_cap, const uint32_t *cand,
                        const CandFam *candfam, cudaStream_t s);
cudaError_t launch_hard(const float *D, uint8_t *masks, const MaskFmt &mf, int32_t W, int64_t HW, int32_t frames,
                        int32_t nviews, const ViewDesc *views,
                        const Params &p, const HardEntry *gq, const uint32_t *gq_count, int32_t gq_cap,
                        const FrameStats *st, int32_t nsm, cudaStream_t s,
                        const ShearDesc *sh = nullptr);
// Pixel-wise median fusion (k_fuse.cu): stack [K][n] -> out [n].
constexpr int kFuseMaxK = 64;
cudaError_t launch_fuse_median(const float *stack, int32_t K, int64_t n, float *out, int nsm, cudaStream_t s);
// Finite-N detector (k_nwin.cu, occ_set_neighbors): one warp per candidate
// window; windows of up to kNwinCap entries in shared memory, longer ones in
// lazily allocated global scratch.
constexpr int kNwinCap = 320;
constexpr int kNwinEntryBytes = 20;
struct NwinScratch {
    unsigned char *buf = nullptr;
    size_t bytes = 0;
};
size_t nwin_smem_bytes();
cudaError_t launch_nwin(const float *D, int32_t H, int32_t W, int32_t frames, const ViewDesc *views,
                        int32_t nviews, const FrameStats *st, const Params &p, int32_t N, uint8_t *masks,
                        const MaskFmt &mf, const void *codes, int32_t code_bytes, uint32_t *work,
                        NwinScratch &big, int32_t smax, int32_t angles, const int2 *offs, int32_t nsm,
                        cudaStream_t s);
cudaError_t launch_prologue(const float *D, int32_t H, int32_t W, int32_t frames,
                            const FamilyDesc *fams_host, int32_t nfam, float e2_thresh,
                            FrameStats *st, void *codes, int32_t code_bytes, int32_t do_stats, cudaStream_t s);
// Line-sweep hot path (k_sweep.cu) for the rows / columns / diagonals /
// anti-diagonals families: K0 words (stats + candidate words of the four
// families, [frame][ceil(H/32)][ceil(W/32)][12][32] uint32) and one warp per
// unit = 32 consecutive lines (l0 a multiple of 32) x [t0, t1) positions
// (multiples of 32, t1 - t0 <= 256).
struct SweepUnit {
    int32_t group, l0, t0, t1;
};
// k_sweep unit length (positions; multiple of 32): C5 ms per 256 frames on
// one B200 (A/B): 256 20.03, 320 19.52, 384 19.30, 448 20.14, 512 20.13
#ifndef SWEEP_SEG
#define SWEEP_SEG 384
#endif
constexpr int kSweepSeg = SWEEP_SEG;
inline int64_t sweep_words_per_frame(int32_t H, int32_t W) {
    return (int64_t)((H + 31) / 32) * ((W + 31) / 32 + 1) * 12 * 32;   // (+1: spare record column)
}
cudaError_t launch_words(const float *D, int32_t H, int32_t W, int32_t frames, float e2_thresh, FrameStats *st,
                         uint32_t *words, int32_t do_stats, cudaStream_t s);
size_t sweep_smem_bytes();
cudaError_t launch_sweep(const float *D, int32_t H, int32_t W, int32_t frames, const SweepUnit *units,
                         int32_t nunits, const GroupDesc *groups, const ViewDesc *views, int32_t nviews,
                         const FamilyDesc *fams, const FrameStats *st, const Params &p, uint8_t *masks,
                         const MaskFmt &mf, const uint32_t *words, HardEntry *gq, uint32_t *gq_count,
                         int32_t gq_cap, const int32_t *kstart, int32_t fgroup, unsigned long long *dbg,
                         int32_t smin, const ShearDesc *sh, cudaStream_t s);
cudaError_t launch_shear(const float *D, int32_t H, int32_t W, int32_t frames, const ShearDesc &sh, int32_t Hs,
                         int32_t Ws, int32_t b0x, int32_t b0y, float e2_thresh, float *Ds, uint32_t *words,
                         cudaStream_t s);

}  // namespace occ
