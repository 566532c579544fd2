/*
 * brute.c -- brute-force references for the oracle's tests (test only).
 *
 * Written independently of occ_oracle.c (no shared helpers): different line
 * parametrisation (floating floor of the rational), no sort, all ordered pairs.
 *
 * BF1  For every candidate window (Eq. 4) compare every
 *      ordered pair of samples with the Eq. 5 test (N = infinity); mark the
 *      smaller-disparity sample (Eq. 6).  O(L^2) per candidate, no sort.
 *      Domain: t_disp >= 2^-20 (so dk + s*delta is exact in binary64).
 * BF2  2-D forward-warp z-buffer for integer-valued D and integer b: centre
 *      pixel p is not visible in the peripheral camera when a pixel q with
 *      larger disparity lands on the same position p - D(p) b (PAPER.md:32,
 *      the definition of occlusion used by the paper).
 */
#include "occ_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int bf_is_candidate(const float *D, int32_t H, int32_t W, int32_t x, int32_t y,
                           int32_t bx, int32_t by, float t_edge)
{
    float c = D[(int64_t)y * W + x];
    float ex = 0.0f, ey = 0.0f;
    if (x < W - 1) ex = D[(int64_t)y * W + x + 1] - c;
    if (y < H - 1) ey = D[(int64_t)(y + 1) * W + x] - c;
    float sq = ex * ex;
    sq = sq + ey * ey;
    if (!(sqrtf(sq) > t_edge)) return 0;
    /* sign of bx*ex + by*ey, exact: compare the two exact binary64 products */
    double a = (double)bx * (double)ex, b = -(double)by * (double)ey;
    return a > b;
}

/* line id and position along the line, floating floor of the exact rational */
static void bf_line(int32_t x, int32_t y, int32_t bx, int32_t by, int64_t *line, int64_t *k)
{
    if (abs(bx) >= abs(by)) {
        *line = (int64_t)y - (int64_t)floor((double)x * (double)by / (double)bx);
        *k = (bx > 0) ? -(int64_t)x : (int64_t)x;
    } else {
        *line = (int64_t)x - (int64_t)floor((double)y * (double)bx / (double)by);
        *k = (by > 0) ? -(int64_t)y : (int64_t)y;
    }
}

int bf1_detect(const float *D, int32_t H, int32_t W, const int32_t *baselines, int32_t V,
               float t_edge, float t_dist, float t_disp, int32_t max_scan, uint8_t *masks)
{
    const int64_t N = (int64_t)H * W;
    memset(masks, 0, (size_t)(N * V));
    float lo = D[0], hi = D[0];
    for (int64_t i = 0; i < N; ++i) {
        if (!isfinite(D[i])) return ORC_ERR_NONFINITE;
        lo = D[i] < lo ? D[i] : lo;
        hi = D[i] > hi ? D[i] : hi;
    }
    int64_t *lid = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    int64_t *kk = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    int64_t *win = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    for (int32_t vi = 0; vi < V; ++vi) {
        int32_t bx = baselines[2 * vi], by = baselines[2 * vi + 1];
        int32_t s = abs(bx) > abs(by) ? abs(bx) : abs(by);
        float R = hi - lo;
        double Ld = ceil((double)R * 2.0 * (double)s);
        int64_t L = Ld > (double)max_scan ? max_scan : (int64_t)Ld;
        int64_t h = L / 2;
        uint8_t *m = masks + (int64_t)vi * N;
        for (int32_t y = 0; y < H; ++y)
            for (int32_t x = 0; x < W; ++x)
                bf_line(x, y, bx, by, &lid[(int64_t)y * W + x], &kk[(int64_t)y * W + x]);
        for (int32_t cy = 0; cy < H; ++cy) {
            for (int32_t cx = 0; cx < W; ++cx) {
                if (!bf_is_candidate(D, H, W, cx, cy, bx, by, t_edge)) continue;
                int64_t c = (int64_t)cy * W + cx;
                int64_t nw = 0;
                for (int64_t i = 0; i < N; ++i)
                    if (lid[i] == lid[c] && llabs(kk[i] - kk[c]) <= h) win[nw++] = i;
                for (int64_t a = 0; a < nw; ++a) {
                    int64_t p = win[a];
                    if (m[p]) continue;
                    for (int64_t b = 0; b < nw; ++b) {
                        int64_t q = win[b];
                        if (q == p) continue;
                        float delta = D[q] - D[p];
                        if (!(delta > t_disp)) continue;
                        double dw = (double)(kk[q] - kk[p]) + (double)s * (double)delta;
                        if (fabs(dw) < (double)t_dist) { m[p] = 1; break; }
                    }
                }
            }
        }
    }
    free(lid); free(kk); free(win);
    return ORC_OK;
}

int bf2_zbuffer(const float *D, int32_t H, int32_t W, int32_t bx, int32_t by,
                float t_disp, uint8_t *mask)
{
    const int64_t N = (int64_t)H * W;
    memset(mask, 0, (size_t)N);
    for (int64_t i = 0; i < N; ++i)
        if (D[i] != floorf(D[i]) || fabsf(D[i]) > 1e6f) return ORC_ERR_INVALID_ARG;
    for (int32_t py = 0; py < H; ++py) {
        for (int32_t px = 0; px < W; ++px) {
            int64_t dp = (int64_t)D[(int64_t)py * W + px];
            int64_t wx = px - dp * bx, wy = py - dp * by;
            for (int32_t qy = 0; qy < H && !mask[(int64_t)py * W + px]; ++qy) {
                for (int32_t qx = 0; qx < W; ++qx) {
                    if (qx == px && qy == py) continue;
                    int64_t dq = (int64_t)D[(int64_t)qy * W + qx];
                    if (qx - dq * bx != wx || qy - dq * by != wy) continue;
                    if ((float)(dq - dp) > t_disp) { mask[(int64_t)py * W + px] = 1; break; }
                }
            }
        }
    }
    return ORC_OK;
}
