/*
 * occ_oracle.c -- CPU ORACLE (test infrastructure only; see occ_oracle.h).
 *
 * The paper's procedure, step by step, in the paper's order and notation
 * (§3, Fig. 2 pipeline):
 *   Eq. 1   E_x, E_y  forward differences with f = (-1, 1)^T
 *   (prose) E = sqrt(E_x^2 + E_y^2), Theta = angle of (E_x, E_y)
 *   Eq. 2   C = {E > t_e and |Theta - phi| < pi/2}
 *   Eq. 3   L = ceil(2 (max D - min D))            (x s, reading Q6)
 *   Eq. 4   S_i = C_i + G (direction of the baseline), G = [-L/2 .. L/2]
 *   (prose) V_i = D[S_i], W_i = G + V_i, sort W_i keeping indices I
 *   Eq. 5   O_i = #{neighbours with |W_i - W_j| < t_dist and larger disparity}
 *   Eq. 6   M[S_i[I]] = 1 if O_i > 0
 * with N = infinity (reading Q12) and the readings Q1-Q21 of DESIGN.md §2.
 *
 * Parity status: pinned by tests/test_oracle_*.py (closed forms, SPEC worked
 * examples, brute force BF1/BF2, exact rational predicate, invariants).
 */
#include "occ_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- O1 */
int orc_validate(int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                 float t_edge, float t_dist, float t_disp, int32_t max_scan)
{
    /* maps smaller than 2x2 are rejected. */
    if (H < 2 || W < 2 || H > 32768 || W > 32768) return ORC_ERR_INVALID_ARG;
    if (V < 1 || V > 64 || baselines == NULL) return ORC_ERR_INVALID_ARG;
    /* t_edge > 0, t_dist > 0, t_disp >= 0; ranges chosen so the
     * exact comparisons of orc_pair are exact in binary64. */
    if (!(isfinite(t_edge) && t_edge > 0.0f)) return ORC_ERR_INVALID_ARG;
    if (!(t_dist >= 0x1p-12f && t_dist <= 0x1p16f)) return ORC_ERR_INVALID_ARG;
    if (!(t_disp >= 0.0f && t_disp <= 0x1p16f)) return ORC_ERR_INVALID_ARG;
    if (max_scan < 1 || max_scan > 65536) return ORC_ERR_INVALID_ARG;
    for (int32_t i = 0; i < V; ++i) {
        int32_t bx = baselines[2 * i], by = baselines[2 * i + 1];
        if (bx == 0 && by == 0) return ORC_ERR_INVALID_ARG;
        if (bx < -8 || bx > 8 || by < -8 || by > 8) return ORC_ERR_UNSUPPORTED;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------ O2 / S1 */
int64_t orc_stats(const float *D, int32_t H, int32_t W, float *dmin, float *dmax)
{
    /* "determined by the minimum and maximum occurring
     * disparity".  Non-finite values are counted (reject). */
    int64_t bad = 0;
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < (int64_t)H * W; ++i) {
        float d = D[i];
        if (!isfinite(d)) { ++bad; continue; }
        if (d < lo) lo = d;
        if (d > hi) hi = d;
    }
    *dmin = lo;
    *dmax = hi;
    return bad;
}

/* ------------------------------------------------------- O3-O4 / S2-S3 */
void orc_edges(const float *D, int32_t H, int32_t W, float *Ex, float *Ey, float *E)
{
    /* PAPER.md:92-101 (Eq. 1): E_x[x,y] = sum_i f[i] D[x+i,y] with
     * f = (-1, 1)^T, i.e. the forward difference D[x+1,y] - D[x,y]
     * (reading Q1); 0 on the last column / row. */
    for (int32_t y = 0; y < H; ++y) {
        for (int32_t x = 0; x < W; ++x) {
            int64_t i = (int64_t)y * W + x;
            float ex = (x + 1 < W) ? D[i + 1] - D[i] : 0.0f;
            float ey = (y + 1 < H) ? D[i + W] - D[i] : 0.0f;
            Ex[i] = ex;
            Ey[i] = ey;
            /* E = sqrt(E_x^2 + E_y^2), literal fp32 (reading Q4) */
            float ex2 = ex * ex;
            float ey2 = ey * ey;
            E[i] = sqrtf(ex2 + ey2);
        }
    }
}

/* --------------------------------------------------------- O6 / S4 */
int orc_angle_predicate(float Ex, float Ey, int32_t bx, int32_t by)
{
    /* Theta = tan^-1(E_y/E_x) taken as the two-argument
     * arctangent (reading Q2), phi = direction of the baseline, circular
     * distance |Theta - phi| < pi/2. */
    double theta = atan2((double)Ey, (double)Ex);
    double phi = atan2((double)by, (double)bx);
    double d = fabs(theta - phi);
    if (d > M_PI) d = 2.0 * M_PI - d;
    return d < M_PI / 2.0;
}

int64_t orc_candidates(const float *Ex, const float *Ey, const float *E, int32_t H, int32_t W,
                       int32_t bx, int32_t by, float t_edge, uint8_t *cand)
{
    /* PAPER.md:105-109 (Eq. 2): C = {(x,y) : E > t_e  and  |Theta - phi| < pi/2}.
     * |Theta - phi| < pi/2 (circular) holds iff the gradient (E_x, E_y) has a
     * strictly positive dot product with the baseline b (reading Q2/Q3); the
     * dot product is evaluated exactly: b_x E_x and b_y E_y are exact in
     * binary64 (|b| <= 8), and the rounded sum of two doubles has the sign
     * of their exact sum. */
    int64_t n = 0;
    for (int64_t i = 0; i < (int64_t)H * W; ++i) {
        int edge = E[i] > t_edge;
        double dot = (double)bx * (double)Ex[i] + (double)by * (double)Ey[i];
        cand[i] = (uint8_t)(edge && dot > 0.0);
        n += cand[i];
    }
    return n;
}

/* --------------------------------------------------------- O5 / S5 */
int32_t orc_scan_length(float dmin, float dmax, int32_t s, int32_t max_scan)
{
    /* PAPER.md:113-116 (Eq. 3): L = ceil((max D - min D) * 2); scaled by
     * s = ||b||_inf because W is measured in major-axis pixels (reading Q6,
     * Q9); capped at max_scan.  R = fl32(max - min);
     * 2 s R is exact in binary64. */
    float R = dmax - dmin;
    double L = ceil(2.0 * (double)s * (double)R);
    if (!(L <= (double)max_scan)) L = (double)max_scan;   /* also R = inf */
    return (int32_t)L;
}

/* ------------------------------------------------------------ O7 / S6 */
static int32_t floordiv(int32_t a, int32_t d)   /* d > 0 */
{
    int32_t q = a / d;
    if ((a % d != 0) && (a < 0)) q -= 1;
    return q;
}

int32_t orc_scanline(const float *D, int32_t H, int32_t W, int32_t bx, int32_t by,
                     int32_t cx, int32_t cy, int32_t h,
                     int32_t *g, int32_t *xs, int32_t *ys, float *v)
{
    /* PAPER.md:117-126 (Eq. 4): S_i = C_i + G (cos phi, sin phi), centred on
     * the candidate, G = [-h .. h] with h = floor(L/2) (reading Q7).
     * Discretised as the digital epipolar line through C_i (reading Q8):
     * x-major (|bx| >= |by|): line id l = y - floor(x by/bx), k = -sgn(bx) x;
     * y-major: l = x - floor(y bx/by), k = -sgn(by) y.  Sample g is the line
     * pixel with k = k_c + g, i.e. the scan runs along the displacement
     * direction -b (reading Q5).  Samples outside the image are dropped
     * (reading Q10).  PAPER.md:127: V_i = D[S_i]. */
    int32_t n = 0;
    if (abs(bx) >= abs(by)) {
        int32_t sg = bx > 0 ? 1 : -1, num = by * sg, den = abs(bx);
        int32_t line = cy - floordiv(cx * num, den);
        for (int32_t gg = -h; gg <= h; ++gg) {
            int32_t x = cx - sg * gg;
            if (x < 0 || x >= W) continue;
            int32_t y = line + floordiv(x * num, den);
            if (y < 0 || y >= H) continue;
            g[n] = gg; xs[n] = x; ys[n] = y; v[n] = D[(int64_t)y * W + x];
            ++n;
        }
    } else {
        int32_t sg = by > 0 ? 1 : -1, num = bx * sg, den = abs(by);
        int32_t line = cx - floordiv(cy * num, den);
        for (int32_t gg = -h; gg <= h; ++gg) {
            int32_t y = cy - sg * gg;
            if (y < 0 || y >= H) continue;
            int32_t x = line + floordiv(y * num, den);
            if (x < 0 || x >= W) continue;
            g[n] = gg; xs[n] = x; ys[n] = y; v[n] = D[(int64_t)y * W + x];
            ++n;
        }
    }
    return n;
}

/* ----------------------------------------------------------------- O9 */
typedef struct { double w; int32_t i; } keyed;

static int cmp_keyed(const void *a, const void *b)
{
    const keyed *p = (const keyed *)a, *q = (const keyed *)b;
    if (p->w < q->w) return -1;
    if (p->w > q->w) return 1;
    return (p->i > q->i) - (p->i < q->i);      /* stable: ties by index */
}

void orc_sort(const double *w, int32_t n, int32_t *idx)
{
    /* "these warped scan lines W are sorted, where the sorting
     * indices are kept in I"; ties broken by original index. */
    keyed *k = (keyed *)malloc(sizeof(keyed) * (size_t)(n > 0 ? n : 1));
    for (int32_t i = 0; i < n; ++i) { k[i].w = w[i]; k[i].i = i; }
    qsort(k, (size_t)n, sizeof(keyed), cmp_keyed);
    for (int32_t i = 0; i < n; ++i) idx[i] = k[i].i;
    free(k);
}

/* --------------------------------------------------------------- S7 */
int orc_pair(float vq, float vp, int32_t dk, int32_t s, float t_dist, float t_disp)
{
    /* PAPER.md:131-144 (Eq. 5) with the prose rule "the pixel with bigger
     * disparity occludes the pixel with smaller disparity" (reading Q13):
     * the neighbour's disparity exceeds ours by more than t_disp, and the two
     * warped positions are closer than t_dist.  W_q - W_p = dk + s delta with
     * delta rounded once (reading Q14).  s*delta is exact in binary64
     * (24+4 bits); t_dist - dk and -t_dist - dk are exact in binary64 for the
     * validated ranges (t_dist in [2^-12, 2^16], |dk| <= 2^16), so both
     * comparisons are exact. */
    float delta = vq - vp;
    if (!(delta > t_disp)) return 0;
    double x = (double)s * (double)delta;
    double hi = (double)t_dist - (double)dk;
    double lo = -(double)t_dist - (double)dk;
    return (x > lo) && (x < hi);
}

/* ---------------------------------------------------------------- O10 */
void orc_count(const int32_t *g, const float *v, const double *w, const int32_t *idx,
               int32_t n, int32_t s, float t_dist, float t_disp, double eps, int32_t *O)
{
    /* PAPER.md:131-142 (Eq. 5): compare each entry of the sorted warped line
     * with its neighbours d in {-N/2..N/2}\{0}, N = infinity (reading Q12).
     * The sorted order lets the walk stop once the warped distance reaches
     * t_dist + eps (eps >= every rounding of w); all nearer entries are
     * visited, so the count's positivity equals that of the full sum. */
    for (int32_t i = 0; i < n; ++i) O[i] = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t p = idx[i];
        for (int32_t j = i + 1; j < n; ++j) {
            int32_t q = idx[j];
            if (!(w[q] - w[p] < (double)t_dist + eps)) break;
            if (orc_pair(v[q], v[p], g[q] - g[p], s, t_dist, t_disp)) O[p]++;
        }
        for (int32_t j = i - 1; j >= 0; --j) {
            int32_t q = idx[j];
            if (!(w[p] - w[q] < (double)t_dist + eps)) break;
            if (orc_pair(v[q], v[p], g[q] - g[p], s, t_dist, t_disp)) O[p]++;
        }
    }
}

/* ----------------------------------------------- O10 with finite N */
void orc_count_n(const int32_t *g, const float *v, const int32_t *idx, int32_t n, int32_t s,
                 float t_dist, float t_disp, int32_t N, int32_t *O)
{
    /* PAPER.md:131-142 (Eq. 5) literally: each entry i of the sorted warped
     * line is compared with the entries at sorted offsets d in
     * {-N/2..-1, 1..N/2}; offsets beyond the line are skipped (SPEC.md:197,
     * 244).  The pair test is the exact S7 predicate (reading Q14), so the
     * warped distance is |dk + s delta| with delta rounded once. */
    for (int32_t i = 0; i < n; ++i) O[i] = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t p = idx[i];
        for (int32_t d = 1; d <= N / 2; ++d) {
            if (i + d < n) {
                int32_t q = idx[i + d];
                if (orc_pair(v[q], v[p], g[q] - g[p], s, t_dist, t_disp)) O[p]++;
            }
            if (i - d >= 0) {
                int32_t q = idx[i - d];
                if (orc_pair(v[q], v[p], g[q] - g[p], s, t_dist, t_disp)) O[p]++;
            }
        }
    }
}

/* --------------------------------------------------------- O1-O11 */
static int detect_impl(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                       float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t Nnb,
                       const float *range, uint8_t *masks, int32_t *info);

int orc_detect(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
               float t_edge, float t_dist, float t_disp, int32_t max_scan,
               uint8_t *masks, int32_t *info)
{
    return detect_impl(D, H, W, baselines, V, t_edge, t_dist, t_disp, max_scan, 0, NULL, masks, info);
}

int orc_detect_n(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                 float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                 uint8_t *masks, int32_t *info)
{
    if (N < 0 || (N > 0 && (N < 2 || (N & 1)))) return ORC_ERR_INVALID_ARG;
    return detect_impl(D, H, W, baselines, V, t_edge, t_dist, t_disp, max_scan, N, NULL, masks, info);
}

int orc_detect_range(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                     float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                     float dmin, float dmax, uint8_t *masks, int32_t *info)
{
    /* O1-O11 with Eq. 3's "minimum and maximum occurring disparity"
     * supplied by the caller: the statistics of a whole
     * frame of which D is a band (spatial sharding). */
    if (N < 0 || (N > 0 && (N < 2 || (N & 1)))) return ORC_ERR_INVALID_ARG;
    if (!(dmin <= dmax)) return ORC_ERR_INVALID_ARG;
    const float range[2] = {dmin, dmax};
    return detect_impl(D, H, W, baselines, V, t_edge, t_dist, t_disp, max_scan, N, range, masks, info);
}

static int detect_impl(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
                       float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t Nnb,
                       const float *range, uint8_t *masks, int32_t *info)
{
    int rc = orc_validate(H, W, baselines, V, t_edge, t_dist, t_disp, max_scan);
    if (rc != ORC_OK) return rc;
    const int64_t N = (int64_t)H * W;
    memset(masks, 0, (size_t)(N * V));
    if (info) memset(info, 0, sizeof(int32_t) * 4 * (size_t)V);

    float dmin, dmax;
    if (orc_stats(D, H, W, &dmin, &dmax) > 0) return ORC_ERR_NONFINITE;   /* O1, Q18 */
    if (range) { dmin = range[0]; dmax = range[1]; }                     /* whole-frame stats */

    float *Ex = (float *)malloc(sizeof(float) * (size_t)N);
    float *Ey = (float *)malloc(sizeof(float) * (size_t)N);
    float *E = (float *)malloc(sizeof(float) * (size_t)N);
    uint8_t *cand = (uint8_t *)malloc((size_t)N);
    orc_edges(D, H, W, Ex, Ey, E);                                     /* O3, O4 */

    double M = fabs((double)dmin) > fabs((double)dmax) ? fabs((double)dmin) : fabs((double)dmax);

    for (int32_t vi = 0; vi < V; ++vi) {
        int32_t bx = baselines[2 * vi], by = baselines[2 * vi + 1];
        int32_t s = abs(bx) > abs(by) ? abs(bx) : abs(by);
        int32_t L = orc_scan_length(dmin, dmax, s, max_scan);            /* O5 */
        int32_t h = L / 2;
        uint8_t *mask = masks + (int64_t)vi * N;
        int64_t nc = orc_candidates(Ex, Ey, E, H, W, bx, by, t_edge, cand); /* O6 */
        int64_t marked = 0;
        if (h > 0) {
            int32_t cap = 2 * h + 1;
            int32_t *g = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *xs = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *ys = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *O = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            float *v = (float *)malloc(sizeof(float) * (size_t)cap);
            double *w = (double *)malloc(sizeof(double) * (size_t)cap);
            /* eps >= 8x the worst rounding of w (binary64 sums) plus that of
             * s*delta vs s*(v_q - v_p) (one fp32 rounding): DESIGN.md §2.3 */
            double eps = 0x1p-16 * ((double)s * M + 1.0);
            for (int32_t cy = 0; cy < H; ++cy) {                          /* O6 row-major */
                for (int32_t cx = 0; cx < W; ++cx) {
                    if (!cand[(int64_t)cy * W + cx]) continue;
                    int32_t n = orc_scanline(D, H, W, bx, by, cx, cy, h, g, xs, ys, v); /* O7 */
                    for (int32_t i = 0; i < n; ++i)                      /* O8: W = G + V */
                        w[i] = (double)g[i] + (double)s * (double)v[i];
                    orc_sort(w, n, idx);                                 /* O9 */
                    if (Nnb > 0) orc_count_n(g, v, idx, n, s, t_dist, t_disp, Nnb, O);   /* O10, finite N */
                    else orc_count(g, v, w, idx, n, s, t_dist, t_disp, eps, O);     /* O10, N = inf */
                    for (int32_t i = 0; i < n; ++i)                      /* O11: Eq. 6, OR */
                        if (O[i] > 0) mask[(int64_t)ys[i] * W + xs[i]] = 1;
                }
            }
            free(g); free(xs); free(ys); free(idx); free(O); free(v); free(w);
        }
        for (int64_t i = 0; i < N; ++i) marked += mask[i];
        if (info) {
            info[4 * vi + 0] = (int32_t)nc;
            info[4 * vi + 1] = L;
            info[4 * vi + 2] = h;
            info[4 * vi + 3] = (int32_t)marked;
        }
    }
    free(Ex); free(Ey); free(E); free(cand);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * NEXT #2: real-valued baseline directions (calibrated, non-grid arrays).
 * A view is a baseline angle phi (radians, image coordinates) and a baseline
 * length rho (grid units).  Reading Q23:
 *   Eq. 2: E > t_e (literal fp32, Q4) and the circular
 *     |Theta - phi| < pi/2, i.e. cos(phi) E_x + sin(phi) E_y > 0, evaluated as
 *     fl64(fl64(c E_x) + fl64(s E_y)) > 0 with c = cos(phi), s = sin(phi);
 *   Eq. 4: sample g of candidate C sits at
 *     C + g u, u = (-c, -s) (displacement = baseline + pi),
 *     each coordinate rounded half away from zero; samples
 *     outside the image are dropped, coinciding samples kept;
 *   Eq. 3: L = min(cap, ceil(fl64(fl64(2 rho) R))), h = floor(L / 2);
 *   W = g + rho V: w = fl64(g + fl64(rho v)) (Euclidean
 *     major-axis-free scaling: samples are one pixel apart along u);
 *   Eq. 5 (prose sign, Q13): delta = fl32(v_q - v_p) > t_disp and
 *     |dg + fl64(rho delta)| < t_dist, exact on these values;
 *   sort by (w, index), N = infinity walk or finite N, Eq. 6 OR-marks.
 * ------------------------------------------------------------------------- */
static int pair_rho(float vq, float vp, int32_t dg, double rho, float t_dist, float t_disp)
{
    float delta = vq - vp;
    if (!(delta > t_disp)) return 0;
    double x = rho * (double)delta;                      /* one binary64 rounding */
    return (x > -(double)t_dist - (double)dg) && (x < (double)t_dist - (double)dg);
}

int orc_dir_offsets(double phi, int32_t h, int32_t *dx, int32_t *dy)
{
    /* offsets of samples g = -h..h (index g + h): round half away from zero
     * of g u, u = (-cos phi, -sin phi) */
    if (!isfinite(phi) || h < 0) return ORC_ERR_INVALID_ARG;
    double ux = -cos(phi), uy = -sin(phi);
    for (int32_t g = -h; g <= h; ++g) {
        dx[g + h] = (int32_t)round((double)g * ux);
        dy[g + h] = (int32_t)round((double)g * uy);
    }
    return ORC_OK;
}

int orc_detect_dirs(const float *D, int32_t H, int32_t W, const double *phi, const double *rho, int32_t V,
                    float t_edge, float t_dist, float t_disp, int32_t max_scan, int32_t N,
                    uint8_t *masks, int32_t *info)
{
    if (H < 2 || W < 2 || H > 32768 || W > 32768 || V < 1 || V > 64 || !phi || !rho) return ORC_ERR_INVALID_ARG;
    if (!(isfinite(t_edge) && t_edge > 0.0f)) return ORC_ERR_INVALID_ARG;
    if (!(t_dist >= 0x1p-12f && t_dist <= 0x1p16f)) return ORC_ERR_INVALID_ARG;
    if (!(t_disp >= 0.0f && t_disp <= 0x1p16f)) return ORC_ERR_INVALID_ARG;
    if (max_scan < 1 || max_scan > 65536) return ORC_ERR_INVALID_ARG;
    if (N < 0 || (N > 0 && (N < 2 || (N & 1)))) return ORC_ERR_INVALID_ARG;
    for (int32_t i = 0; i < V; ++i)
        if (!isfinite(phi[i]) || !(rho[i] > 0.0 && rho[i] <= 8.0)) return ORC_ERR_INVALID_ARG;
    const int64_t P = (int64_t)H * W;
    memset(masks, 0, (size_t)(P * V));
    if (info) memset(info, 0, sizeof(int32_t) * 4 * (size_t)V);
    float dmin, dmax;
    if (orc_stats(D, H, W, &dmin, &dmax) > 0) return ORC_ERR_NONFINITE;   /* O1, Q18 */
    float *Ex = (float *)malloc(sizeof(float) * (size_t)P);
    float *Ey = (float *)malloc(sizeof(float) * (size_t)P);
    float *E = (float *)malloc(sizeof(float) * (size_t)P);
    orc_edges(D, H, W, Ex, Ey, E);                                     /* O3, O4 */
    const float R = dmax - dmin;
    double M = fabs((double)dmin) > fabs((double)dmax) ? fabs((double)dmin) : fabs((double)dmax);
    for (int32_t vi = 0; vi < V; ++vi) {
        const double c = cos(phi[vi]), sn = sin(phi[vi]), r = rho[vi];
        double Ld = ceil((2.0 * r) * (double)R);                        /* O5, Eq. 3 */
        if (!(Ld <= (double)max_scan)) Ld = (double)max_scan;
        const int32_t L = (int32_t)Ld, h = L / 2;
        uint8_t *mask = masks + (int64_t)vi * P;
        int64_t nc = 0, marked = 0;
        if (h > 0) {
            const int32_t cap = 2 * h + 1;
            int32_t *dx = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *dy = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *g = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *xs = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *ys = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            int32_t *O = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
            float *v = (float *)malloc(sizeof(float) * (size_t)cap);
            double *w = (double *)malloc(sizeof(double) * (size_t)cap);
            orc_dir_offsets(phi[vi], h, dx, dy);
            const double eps = 0x1p-16 * (r * M + 1.0);
            for (int32_t cy = 0; cy < H; ++cy) {
                for (int32_t cx = 0; cx < W; ++cx) {
                    const int64_t ci = (int64_t)cy * W + cx;
                    /* O6: Eq. 2 */
                    const double dot = c * (double)Ex[ci] + sn * (double)Ey[ci];
                    if (!(E[ci] > t_edge && dot > 0.0)) continue;
                    ++nc;
                    int32_t n = 0;                                      /* O7: Eq. 4 */
                    for (int32_t gg = -h; gg <= h; ++gg) {
                        const int32_t x = cx + dx[gg + h], y = cy + dy[gg + h];
                        if (x < 0 || x >= W || y < 0 || y >= H) continue;
                        g[n] = gg; xs[n] = x; ys[n] = y; v[n] = D[(int64_t)y * W + x];
                        ++n;
                    }
                    for (int32_t i = 0; i < n; ++i) w[i] = (double)g[i] + r * (double)v[i];   /* O8 */
                    orc_sort(w, n, idx);                                /* O9 */
                    for (int32_t i = 0; i < n; ++i) O[i] = 0;           /* O10 */
                    for (int32_t i = 0; i < n; ++i) {
                        const int32_t p = idx[i];
                        for (int32_t j = i + 1; j < n && (N == 0 || j - i <= N / 2); ++j) {
                            const int32_t q = idx[j];
                            if (N == 0 && !(w[q] - w[p] < (double)t_dist + eps)) break;
                            if (pair_rho(v[q], v[p], g[q] - g[p], r, t_dist, t_disp)) O[p]++;
                        }
                        for (int32_t j = i - 1; j >= 0 && (N == 0 || i - j <= N / 2); --j) {
                            const int32_t q = idx[j];
                            if (N == 0 && !(w[p] - w[q] < (double)t_dist + eps)) break;
                            if (pair_rho(v[q], v[p], g[q] - g[p], r, t_dist, t_disp)) O[p]++;
                        }
                    }
                    for (int32_t i = 0; i < n; ++i)                      /* O11: Eq. 6, OR */
                        if (O[i] > 0) mask[(int64_t)ys[i] * W + xs[i]] = 1;
                }
            }
            free(dx); free(dy); free(g); free(xs); free(ys); free(idx); free(O); free(v); free(w);
        }
        for (int64_t i = 0; i < P; ++i) marked += mask[i];
        if (info) {
            info[4 * vi + 0] = (int32_t)nc;
            info[4 * vi + 1] = L;
            info[4 * vi + 2] = h;
            info[4 * vi + 3] = (int32_t)marked;
        }
    }
    free(Ex); free(Ey); free(E);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * NEXT #3: pixel-wise median fusion.
 * Per pixel: copy the K values, insertion-sort them (plain, O(K^2)), take the
 * middle one (odd K) or the fp32 mean of the two middle ones (even K).
 * ------------------------------------------------------------------------- */
int orc_fuse_median(const float *stack, int32_t K, int64_t n, float *out)
{
    if (K < 1 || K > 1024) return ORC_ERR_INVALID_ARG;
    float *v = (float *)malloc(sizeof(float) * (size_t)K);
    if (!v) return ORC_ERR_INVALID_ARG;
    for (int64_t p = 0; p < n; ++p) {
        int bad = 0;
        for (int32_t k = 0; k < K; ++k) {
            const float x = stack[(int64_t)k * n + p];
            if (!isfinite(x)) bad = 1;
            /* insertion into the sorted prefix v[0..k-1] */
            int32_t j = k;
            while (j > 0 && v[j - 1] > x) { v[j] = v[j - 1]; --j; }
            v[j] = x;
        }
        if (bad) { out[p] = NAN; continue; }
        if (K & 1) {
            out[p] = v[K / 2];
        } else {
            const float a = v[K / 2 - 1], b = v[K / 2];
            const float sum = a + b;          /* one fp32 rounding */
            out[p] = sum * 0.5f;              /* exact halving (normal range) */
        }
    }
    free(v);
    return ORC_OK;
}
