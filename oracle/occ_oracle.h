/*
 * occ_oracle.h -- CPU ORACLE for the fast edge-aware occlusion detection of
 * arXiv 2408.14050 (§3, Eqs. 1-6).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (libocc, the CUDA
 * kernels, the Python binding) may include, link or call this code; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg do.  It
 * shares no source with paper_2408_14050_b200/csrc.
 *
 * Plain, slow, single-threaded C11.  Build flags: -O2 -ffp-contract=off
 * -fno-fast-math (x86-64 SSE arithmetic, so every float operation below is
 * one IEEE-754 round-to-nearest-even fp32 operation).
 *
 * Semantics follow SURVEY.md §8.0 (S1-S9) / §8(c) (O1-O11) and the readings
 * Q1-Q21 listed in DESIGN.md §2.  Every function cites the paper passage it
 * implements.  Parity status of each function is listed in DESIGN.md §2.4.
 */
#ifndef OCC_ORACLE_H
#define OCC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (mirror the product ABI's values, defined independently) */
#define ORC_OK 0
#define ORC_ERR_INVALID_ARG (-1)
#define ORC_ERR_NONFINITE (-4)
#define ORC_ERR_UNSUPPORTED (-5)

/* O1 validation ranges */
int orc_validate(int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                 float t_edge, float t_dist, float t_disp, int32_t max_scan);

/* O2 / S1: exact min and max of D; returns number of non-finite values.
 * PAPER.md:113-115 (Eq. 3 "minimum and maximum occurring disparity"). */
int64_t orc_stats(const float *D, int32_t H, int32_t W, float *dmin, float *dmax);

/* O3-O4 / S2-S3: forward-difference edge maps and magnitude.
 * PAPER.md:92-103 (Eq. 1, E = sqrt(Ex^2 + Ey^2)). */
void orc_edges(const float *D, int32_t H, int32_t W, float *Ex, float *Ey, float *E);

/* O6 / S4: candidate flags for baseline (bx, by). PAPER.md:104-109 (Eq. 2). */
int64_t orc_candidates(const float *Ex, const float *Ey, const float *E, int32_t H, int32_t W,
                       int32_t bx, int32_t by, float t_edge, uint8_t *cand);

/* S4 via the literal angle form (atan2, circular distance) -- used only by a
 * test that pins orc_candidates' exact sign test against the textbook
 * definition away from the pi/2 boundary. */
int orc_angle_predicate(float Ex, float Ey, int32_t bx, int32_t by);

/* O5 / S5: scan length L (Eq. 3) for a baseline with s = max(|bx|,|by|). */
int32_t orc_scan_length(float dmin, float dmax, int32_t s, int32_t max_scan);

/* O7 / S6: scan line of candidate (cx, cy): samples g = -h..h, dropped when
 * outside the image.  Writes up to 2h+1 entries, returns the count.
 * PAPER.md:117-127 (Eq. 4, V_i = D[S_i]). */
int32_t orc_scanline(const float *D, int32_t H, int32_t W, int32_t bx, int32_t by,
                     int32_t cx, int32_t cy, int32_t h,
                     int32_t *g, int32_t *xs, int32_t *ys, float *v);

/* O9: stable sort of warped positions w. idx receives the
 * permutation I such that w[I] is non-decreasing, ties by index. */
void orc_sort(const double *w, int32_t n, int32_t *idx);

/* S7: pair predicate for neighbour q of entry p (Eq. 5
 * with the prose sign): delta = fl32(vq - vp) > t_disp and
 * |dk + s*delta| < t_dist, evaluated exactly. */
int orc_pair(float vq, float vp, int32_t dk, int32_t s, float t_dist, float t_disp);

/* O10: occlusion counts O_i for one sorted scan line (Eq. 5, N = infinity).
 * Inputs in scan-line order; idx from orc_sort; O receives counts per
 * scan-line entry (not per sorted position). eps bounds w's rounding. */
void orc_count(const int32_t *g, const float *v, const double *w, const int32_t *idx,
               int32_t n, int32_t s, float t_dist, float t_disp, double eps, int32_t *O);

/* O1-O11: the whole detector for V baselines; masks [V][H][W] in {0,1}.
 * info (optional) receives per view {n_candidates, L, h, n_marked}. */
int orc_detect(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
               float t_edge, float t_dist, float t_disp, int32_t max_scan,
               uint8_t *masks, int32_t *info);

/* ---------------------------------------------------------------------
 * Brute-force references (oracle/brute.c; independent code, test only)
 * ------------------------------------------------------------------- */

/* BF1: all ordered pairs inside every candidate window, no sort. */
int bf1_detect(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
               float t_edge, float t_dist, float t_disp, int32_t max_scan, uint8_t *masks);

/* BF2: 2-D forward-warp visibility for INTEGER-valued D and integer b:
 * p occluded iff some q != p has p - D(p) b == q - D(q) b and
 * D(q) - D(p) > t_disp  (PAPER.md:32 definition of occlusion). */
int bf2_zbuffer(const float *D, int32_t H, int32_t W, int32_t bx, int32_t by,
                float t_disp, uint8_t *mask);

/* O10 with a finite neighbour count N (SPEC.md:197,
 * 244): each sorted entry is compared with the entries at sorted offsets
 * d in {-N/2..-1, 1..N/2} (skipped beyond the line) with the exact pair
 * predicate (orc_pair); O[p] counts the pairs.  N even >= 2. */
void orc_count_n(const int32_t *g, const float *v, const int32_t *idx, int32_t n, int32_t s,
                 float t_dist, float t_disp, int32_t N, int32_t *O);

/* O1-O11 with a finite neighbour count N (N = 0: N = infinity, identical to
 * orc_detect).  Returns ORC_ERR_INVALID_ARG for odd N or N < 2 (N != 0). */
int orc_detect_n(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                 float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                 uint8_t *masks, int32_t *info);

/* orc_detect_n with Eq. 3's min / max supplied by the caller (dmin <= dmax):
 * the statistics of the whole frame a band D belongs to (spatial sharding). */
int orc_detect_range(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                     float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                     float dmin, float dmax, uint8_t *masks, int32_t *info);

/* NEXT #2: real-valued baseline directions (reading Q23): view i has baseline
 * angle phi[i] (radians, finite) and length rho[i] in (0, 8]; N as for
 * orc_detect_n (0 = infinity).  masks [V][H][W], info as orc_detect. */
int orc_detect_dirs(const float *D, int32_t H, int32_t W, const double *phi, const double *rho, int32_t V,
                    float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                    uint8_t *masks, int32_t *info);
/* Sample offsets of the direction phi: dx, dy [2h + 1] for g = -h..h. */
int orc_dir_offsets(double phi, int32_t h, int32_t *dx, int32_t *dy);

/* Pixel-wise median fusion of K disparity estimates.
 * PAPER.md:238 (§4.2, "fused to a single disparity map by pixel-wise median
 * filtering"); SPEC.md:51-58 (fuse_median: for even counts the arithmetic
 * mean of the two middle values).  stack is K planes of n values
 * ([K][n], plane k = estimate k); out[p] = median of stack[0..K-1][p].
 * fp32 reading (Q22): odd K -> the middle value; even K ->
 * fl32(fl32(a + b) * 0.5) of the two middle values a <= b; any non-finite
 * input at p -> out[p] = NaN (the detector then rejects the frame, Q18).
 * Returns ORC_OK, or ORC_ERR_INVALID_ARG for K < 1. */
int orc_fuse_median(const float *stack, int32_t K, int64_t n, float *out);

#ifdef __cplusplus
}
#endif
#endif
