/*
 * occ.h -- C ABI of the B200-native fast edge-aware occlusion detection
 * (arXiv 2408.14050, §3 "Edge-aware Occlusion Detection", Eqs. 1-6).
 *
 * One call marks, for each peripheral camera of an array, the pixels of the
 * fused centre-camera disparity map that the camera cannot see:
 *
 *   occ_detect(D [batch][H][W] fp32, device)  ->  M [batch][V][H][W] uint8 {0,1}
 *
 * The operation is the paper's detector with N = infinity (SURVEY.md §8.0
 * S1-S9; readings Q1-Q21 in DESIGN.md §2):
 *   PAPER.md:92-101  Eq. 1  E_x, E_y forward differences (f = (-1, 1)^T)
 *   PAPER.md:103           E = sqrt(E_x^2 + E_y^2), Theta = angle of (E_x, E_y)
 *   PAPER.md:105-109 Eq. 2  candidates: E > t_edge and |Theta - phi| < pi/2
 *   PAPER.md:113-116 Eq. 3  L = ceil(2 s (max D - min D)), s = ||b||_inf
 *   PAPER.md:117-129 Eq. 4  scan lines of length L along the baseline, W = G + s V
 *   PAPER.md:131-144 Eq. 5  neighbours with |W_i - W_j| < t_dist and larger
 *                           disparity (by more than t_disp) occlude
 *   PAPER.md:145-151 Eq. 6  M = 1 where the occlusion count is positive
 * Every step runs in the library's own sm_100a CUDA kernels; there is no CPU
 * fallback.  The result is bit-identical to the test oracle (oracle/).
 *
 * Conventions
 *   - D is row-major fp32, x rightward, y downward, contiguous,
 *     device memory owned by the caller; frames are [H][W] back to back.
 *   - A baseline b = (bx, by) is the offset of a peripheral camera from the
 *     centre camera in units of the grid spacing; that camera sees centre
 *     pixel p at p - D(p) b.  |bx|, |by| <= 8, b != (0, 0).
 *   - masks is caller-owned device memory, [batch][n_views][H][W] uint8;
 *     every byte is written (0 or 1).  masks must not alias disparity.
 *   - Stream ordered: occ_detect enqueues work on the given cudaStream_t and
 *     returns without synchronising.  Argument errors are returned
 *     synchronously; data errors (non-finite input) are reported per frame
 *     by occ_status, and that frame's masks are all zero.
 *   - A context must not be used concurrently from two host threads/streams.
 */
#ifndef OCC_H
#define OCC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct occ_ctx occ_ctx;                       /* opaque; owns device scratch */

typedef struct { int32_t bx, by; } occ_baseline;       /* peripheral camera offset */

/* PAPER.md:187 (§4.1): t_e = 1.0, t_dist = 2.0, t_disp = 0.5; SPEC.md:153 cap 4096.
 * Valid ranges: t_edge > 0 finite; t_dist in [2^-12, 2^16];
 * t_disp in [0, 2^16]; max_scan in [1, 65536]. */
typedef struct { float t_edge, t_dist, t_disp; int32_t max_scan; } occ_params;

enum {
    OCC_OK = 0,
    OCC_ERR_INVALID_ARG = -1,   /* bad sizes, pointers, params or baselines */
    OCC_ERR_CUDA = -2,          /* a CUDA runtime call failed */
    OCC_ERR_OOM = -3,           /* device allocation failed */
    OCC_ERR_NONFINITE = -4,     /* per-frame status: NaN/Inf in the input */
    OCC_ERR_UNSUPPORTED = -5    /* |bx| or |by| > 8, or too many views */
};

/* Paths (occ_set_path): AUTO runs the line-sweep kernel for the view pairs
 * +-b of row / column / diagonal / anti-diagonal families under the default
 * near/far split, and the tiled kernel for every other view group; both fall
 * back in-kernel to the exact per-pixel routine for frames outside their
 * staging range.  TILED forces the tiled kernel for every group; DIRECT the
 * per-pixel kernel (debug / cross-check). */
enum { OCC_PATH_AUTO = 0, OCC_PATH_TILED = 1, OCC_PATH_DIRECT = 2 };

/* A real-valued peripheral direction (calibrated
 * non-grid arrays): baseline angle in radians (image coordinates, x right, y
 * down; the angle of b) and baseline length in grid units, (0, 8]. */
typedef struct { double baseline_angle, baseline_length; } occ_direction;

/* Fills the paper's defaults. */
void occ_default_params(occ_params *p);

/* Creates a context for H x W maps and n_views baselines (copied).
 * params == NULL selects the defaults.  max_batch bounds occ_detect's batch.
 * Allocates only small per-frame scratch (O(max_batch) bytes).  Requires a
 * current CUDA device with compute capability 10.0 (sm_100a).
 * Errors: OCC_ERR_INVALID_ARG (H < 2, W < 2, H or W > 32768, n_views < 1,
 * b == (0,0), params out of range, max_batch < 1, out == NULL),
 * OCC_ERR_UNSUPPORTED (|b| component > 8 or n_views > 64), OCC_ERR_CUDA,
 * OCC_ERR_OOM. */
int occ_create(int32_t H, int32_t W, const occ_baseline *baselines, int32_t n_views,
               const occ_params *params, int32_t max_batch, occ_ctx **out);

/* Context for real-valued directions (reading Q23 of DESIGN.md; PAPER.md:
 * 103-128 with SPEC.md:179, 241-242): candidates E > t_e and
 * fl64(cos(phi) E_x) + fl64(sin(phi) E_y) > 0; sample g of candidate C at
 * C + g u, u = -(cos phi, sin phi), each coordinate rounded half away from
 * zero (offset tables computed on the host); h = floor(min(cap,
 * ceil(fl64(2 rho) R)) / 2); W = g + rho V; pair |dg + fl64(rho delta)| <
 * t_dist and delta > t_disp.  Detection runs the per-window kernel (N =
 * infinity by default, occ_set_neighbors for finite N); occ_set_path has no
 * effect.  Same buffers, formats and errors as occ_create (an angle must be
 * finite, a length in (0, 8]). */
int occ_create_dirs(int32_t H, int32_t W, const occ_direction *dirs, int32_t n_views,
                    const occ_params *params, int32_t max_batch, occ_ctx **out);

/* Enqueues detection for `batch` frames.  disparity: device [batch][H][W]
 * fp32; masks: device [batch][n_views][H][W] uint8.  cuda_stream is a
 * cudaStream_t (NULL = legacy default stream).  Returns OCC_OK or
 * OCC_ERR_INVALID_ARG (null pointers, batch < 1 or > max_batch) /
 * OCC_ERR_CUDA (launch failure). */
int occ_detect(occ_ctx *ctx, const float *disparity, uint8_t *masks, int32_t batch,
               void *cuda_stream);

/* Same operation on HOST buffers (pageable or pinned): copies D to the
 * context's device staging buffer, detects, copies the masks back, and
 * synchronises the stream before returning.  Staging buffers are allocated
 * on first use (max_batch frames).  Used for end-to-end timing. */
int occ_detect_host(occ_ctx *ctx, const float *disparity_host, uint8_t *masks_host,
                    int32_t batch, void *cuda_stream);

/* Synchronises the stream of the last occ_detect and writes one status per
 * frame of that call (OCC_OK or OCC_ERR_NONFINITE) to host memory
 * frame_status[batch].  Returns OCC_OK or OCC_ERR_CUDA. */
int occ_status(occ_ctx *ctx, int32_t *frame_status);

/* Synchronises and reports the per-frame statistics of the last call:
 * dmin/dmax (exact, S1) and the scan half-length h of every view (S5);
 * h_per_view has n_views entries.  Any output pointer may be NULL. */
int occ_frame_info(occ_ctx *ctx, int32_t frame, float *dmin, float *dmax, int32_t *h_per_view);

/* Eq. 3 (S5 of SURVEY §8.0) for given frame statistics:
 * h = floor(min(max_scan, ceil(2 s R)) / 2) per view, R = fl32(dmax - dmin),
 * s = the view's ||b||_inf (real-valued directions: 2 rho R).  dmin <= dmax
 * finite, or non-finite stats give h = max_scan / 2.  h_per_view: host,
 * n_views entries.  No device work.  OCC_OK or OCC_ERR_INVALID_ARG.  Used
 * to size the halos of single-frame spatial sharding (spatial.py). */
int occ_scan_half_lengths(const occ_ctx *ctx, float dmin, float dmax, int32_t *h_per_view);

/* Mask output format (occ_set_mask_format), NEXT #4 of SURVEY §8(f):
 *   OCC_MASK_U8   (default) uint8 [batch][n_views][H][W], each byte 0 or 1;
 *   OCC_MASK_BITS bit-packed uint32 words [batch][n_views][H][ceil(W/32)]:
 *                 bit (x & 31) of word (y, x >> 5) is the mask of pixel
 *                 (x, y); padding bits are 0.  8x fewer bytes to move.
 * The buffers passed to occ_detect / occ_detect_host must hold
 * occ_mask_bytes(ctx, batch) bytes.  Returns OCC_OK or OCC_ERR_INVALID_ARG. */
enum { OCC_MASK_U8 = 0, OCC_MASK_BITS = 1 };
int occ_set_mask_format(occ_ctx *ctx, int32_t format);

/* Bytes of the mask buffer for `batch` frames in the current format (-1 on
 * a null context or negative batch). */
int64_t occ_mask_bytes(const occ_ctx *ctx, int32_t batch);

/* Neighbour count N of Eq. 5:
 * each entry of a sorted warped scan line is compared with the entries at
 * sorted offsets d in {-N/2..-1, 1..N/2} only (offsets beyond
 * the line skipped; SPEC.md:155's default is N = 8).  N = 0 (the context's
 * default) selects N = infinity, the per-pixel form every other path
 * computes.  With N > 0 subsequent calls run the per-window kernel k_nwin
 * (one warp per candidate window: sort by (W, scan index), then the +-N/2
 * neighbour tests) whatever occ_set_path selected; the output is
 * bit-identical to the oracle's orc_detect_n.  Longer windows than the
 * kernel's shared-memory capacity (h > 159) use device scratch allocated on
 * first use (about nsm * 8 * (max_scan + 1) * 16 bytes).
 * Returns OCC_OK, OCC_ERR_INVALID_ARG (N odd, N < 0, N > 65536, NULL ctx)
 * or OCC_ERR_OOM. */
int occ_set_neighbors(occ_ctx *ctx, int32_t N);

/* Current N (0 = infinity), -1 on a NULL context. */
int32_t occ_get_neighbors(const occ_ctx *ctx);

/* Spatial sharding: a frame too large for one GPU is
 * split into row bands, each processed with halo rows on its own rank.  The
 * scan half-length h (Eq. 3) depends on the WHOLE frame's
 * min/max, so the ranks all-reduce their band statistics and impose the
 * result on their band:
 *   occ_frame_stats: exact per-frame min / max / non-finite count of `batch`
 *     device frames [batch][H][W] (this context's H, W); writes host arrays
 *     dmin[batch], dmax[batch], nonfinite[batch] (any may be NULL; a frame
 *     without finite values reports dmin = +inf, dmax = -inf).  Synchronises
 *     the stream.  Errors: OCC_ERR_INVALID_ARG, OCC_ERR_CUDA.
 *   occ_set_frame_stats: subsequent occ_detect / occ_detect_host calls use
 *     dmin[f], dmax[f], nonfinite[f] (host arrays, copied) for frame f < n
 *     instead of the statistics of the data passed (n = 0 disables the
 *     override).  Candidates, windows and pairs still come from the data, so
 *     a band extended by 2 h + 2 halo rows on each side (clipped to the
 *     frame) yields the whole frame's masks on its interior rows.
 *     Errors: OCC_ERR_INVALID_ARG (n < 0, n > max_batch, NULL arrays with
 *     n > 0, dmin > dmax with a zero non-finite count), OCC_ERR_CUDA. */
int occ_frame_stats(occ_ctx *ctx, const float *disparity, int32_t batch, float *dmin, float *dmax,
                    int32_t *nonfinite, void *cuda_stream);
int occ_set_frame_stats(occ_ctx *ctx, const float *dmin, const float *dmax, const int32_t *nonfinite,
                        int32_t n);

/* Selects the kernel path for subsequent calls (OCC_PATH_*). */
int occ_set_path(occ_ctx *ctx, int32_t path);

/* Number of kernel launches the last occ_detect enqueued. */
int32_t occ_last_launches(const occ_ctx *ctx);

/* Kernel timing (benchmarks): while enabled, every kernel launch is
 * bracketed by CUDA events recorded on its launch stream.  occ_profile
 * enables/disables and resets the accumulators; occ_profile_read
 * synchronises and returns, for one kernel kind, the summed device time in
 * milliseconds and the number of launches since the last reset. */
enum { OCC_KERNEL_INIT = 0, OCC_KERNEL_STATS = 1, OCC_KERNEL_TILE = 2, OCC_KERNEL_DIRECT = 3,
       OCC_KERNEL_CAND = 4, OCC_KERNEL_LINE = 5, OCC_KERNEL_NWIN = 6, OCC_KERNEL_HARD = 7,
       OCC_KERNEL_KINDS = 8 };
int occ_profile(occ_ctx *ctx, int32_t enable);
int occ_profile_read(occ_ctx *ctx, int32_t kind, double *total_ms, int32_t *launches);

/* Pixel-wise median fusion of K disparity estimates into the fused map the
 * detector consumes (§4.2: "fused to a single disparity map by
 * pixel-wise median filtering").  No context needed.
 *   stack: device, K planes of n fp32 values back to back ([K][n]; plane k =
 *          estimate k, n = frames * H * W for a batch), caller-owned;
 *   out:   device, n fp32 values, caller-owned, must not overlap stack.
 * out[p] = the middle value of {stack[k][p]} for odd K; for even K the fp32
 * mean fl(fl(a + b) * 0.5) of the two middle values a <= b; NaN where any
 * estimate is non-finite (occ_detect then reports OCC_ERR_NONFINITE for the
 * frame).  Stream ordered; returns OCC_OK, OCC_ERR_INVALID_ARG (null
 * pointers, K < 1 or K > 64, n < 1, overlap) or OCC_ERR_CUDA. */
int occ_fuse_median(const float *stack, int32_t K, int64_t n, float *out, void *cuda_stream);

/* Releases the context and its device scratch (synchronises first). */
int occ_destroy(occ_ctx *ctx);

const char *occ_strerror(int code);

/* ABI version (major*10000 + minor*100 + patch). */
int32_t occ_version(void);

#ifdef __cplusplus
}
#endif
#endif
