// occ_api.cu -- host side of libocc: the C ABI of include/occ.h.
//
// Owns validation, the view/family descriptors (digital-line geometry of
// SURVEY §8.0 S6), the exact fp32 thresholds of the Eq. 5 test, per-frame
// scratch, and launch sequencing on the caller's stream.  All arithmetic of
// the method runs in the kernels (k_stats.cu, k_tile.cu, k_direct.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "occ_internal.h"

using namespace occ;

struct occ_ctx {
    int32_t H = 0, W = 0, V = 0, nfam = 0, max_batch = 0, device = 0;
    int32_t path = OCC_PATH_AUTO;
    int32_t neighbors = 0;               // occ_set_neighbors: N (0 = infinity)
    int32_t line_seg = kLineSeg;         // positions per k_line unit (<= kLineSeg, multiple of 32)
    std::vector<CandFam> candfam;        // k_cand word blocks per family (index = family)
    CandFam *d_candfam = nullptr;
    int64_t cand_per_frame = 0;
    uint32_t *d_cand = nullptr;          // k_cand words for one chunk (null: pass 0 from the codes)
    int32_t angles = 0;                  // occ_create_dirs context: real-valued directions
    int2 *d_offs = nullptr;              // their Eq. 4 offset tables [V][2 (max_scan/2) + 1]
    uint32_t *d_nwin_work = nullptr;     // k_nwin granule counters (lazy)
    NwinScratch nwin_big;                // k_nwin scratch for windows > kNwinCap (lazy)
    FrameStats *d_override = nullptr;    // occ_set_frame_stats (lazy), n_override frames
    int32_t n_override = 0;
    MaskFmt mf{0, 0, 0};                 // occ_set_mask_format
    Params params{};
    std::vector<ViewDesc> views;
    std::vector<FamilyDesc> fams;
    ViewDesc *d_views = nullptr;
    FamilyDesc *d_fams = nullptr;
    FrameStats *d_stats = nullptr;
    std::vector<GroupDesc> groups;
    std::vector<TileDesc> tiles;
    GroupDesc *d_groups = nullptr;
    TileDesc *d_tiles = nullptr;
    std::vector<SweepUnit> sunits;        // k_sweep work (eligible groups; the default line path)
    SweepUnit *d_sunits = nullptr;
    uint32_t *d_words = nullptr;          // k_words -> k_sweep candidate words, one chunk of frames
    // consecutive chunks on two streams (the second chunk's sweep fills the
    // first chunk's k_hard and tail): a second words buffer, the main queue
    // region split in two halves with their own counters
    uint32_t *d_words2 = nullptr;
    cudaStream_t s_alt = nullptr;
    cudaEvent_t ev_alt_fork = nullptr, ev_alt_join = nullptr;
    cudaEvent_t ev_swept[2] = {nullptr, nullptr};   // chunk's sweep done: the next chunk may start
    int32_t skstart[5] = {0, 0, 0, 0, 0}; // sunits of kind k at [skstart[k], skstart[k + 1])
    int32_t sfgroup = 1;                  // k_sweep work order: frames per group
    int32_t ssmin = 1;                    // smallest s of the k_sweep groups (k_sweep_small's frame filter)
    // knight families swept through a sheared copy of D (k_shear + k_sweep)
    struct ShearFam {
        int32_t fam = 0, Hs = 0, Ws = 0;   // family, sheared frame
        ShearDesc sd{};
        std::vector<SweepUnit> units;
        SweepUnit *d_units = nullptr;
        int32_t kstart[5] = {0, 0, 0, 0, 0};
        int32_t fgroup = 1, smin = 1;
        float *d_D = nullptr;             // its sheared D, one chunk of frames
        uint32_t *d_W = nullptr;          // its candidate words
        int64_t q0 = 0;                   // its region of the far-partner queue [q0, q0 + qcap)
        int32_t qcap = 0;
        cudaStream_t st = nullptr;        // families run concurrently, forked from the caller's stream
        cudaEvent_t done = nullptr;
    };
    std::vector<ShearFam> shear;
    cudaEvent_t sh_fork = nullptr;
    int32_t main_qcap = 0;                // queue region of the main sweep [0, main_qcap)
    std::vector<LineUnit> units;          // k_line work (eligible groups, OCC_SWEEP=0)
    std::vector<TileDesc> all_tiles;      // k_tile work for every group (OCC_PATH_TILED)
    LineUnit *d_units = nullptr;
    TileDesc *d_all_tiles = nullptr;
    unsigned long long *d_dbg = nullptr;  // k_line event counters (occ_debug_line_stats)
    HardEntry *d_gq = nullptr;            // k_line -> k_hard queue (one chunk)
    uint32_t *d_gq_count = nullptr;
    int32_t gq_cap = 0, nsm = 148;
    void *d_codes = nullptr;             // K0 -> K1 candidate codes, one chunk of frames
    int32_t code_bytes = 1, chunk = 1;
    float *d_stage_D = nullptr;          // occ_detect_host staging (lazy)
    uint8_t *d_stage_M = nullptr;
    cudaStream_t last_stream = nullptr;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;   // occ_detect_host copy streams
    std::vector<cudaEvent_t> ev_pipe;
    int32_t last_batch = 0;
    int32_t last_launches = 0;
    // kernel timing (occ_profile)
    bool profiling = false;
    std::vector<cudaEvent_t> ev[OCC_KERNEL_KINDS];   // start/end pairs
    size_t ev_used[OCC_KERNEL_KINDS] = {};
};

namespace {

int32_t igcd(int32_t a, int32_t b) {
    a = std::abs(a); b = std::abs(b);
    while (b) { int32_t t = a % b; a = b; b = t; }
    return a;
}

// Largest fp32 f with s*f <= A (A exact in binary64): delta > A/s <=> delta > f
float rd_div(double A, int32_t s) {
    float f = (float)(A / s);
    while ((double)s * (double)f > A) f = std::nextafter(f, -INFINITY);
    for (;;) {
        float n = std::nextafter(f, INFINITY);
        if ((double)s * (double)n <= A) f = n; else break;
    }
    return f;
}

// Smallest fp32 f with s*f >= B: delta < B/s <=> delta < f
float ru_div(double B, int32_t s) {
    float f = (float)(B / s);
    while ((double)s * (double)f < B) f = std::nextafter(f, INFINITY);
    for (;;) {
        float n = std::nextafter(f, -INFINITY);
        if ((double)s * (double)n >= B) f = n; else break;
    }
    return f;
}

// Largest fp32 x >= 0 with sqrt_rn(x) <= t: sqrt_rn is monotone, so
// sqrt_rn(e2) > t  <=>  e2 > x   (exact rewrite of PAPER.md:103's E > t_e).
float sqrt_thresh(float t) {
    double t2 = (double)t * (double)t;
    float x = t2 > 3.0e38 ? 3.4028234663852886e38f : (float)t2;
    while (x > 0.0f && std::sqrt(x) > t) x = std::nextafter(x, 0.0f);
    for (;;) {
        float n = std::nextafter(x, INFINITY);
        if (std::isfinite(n) && std::sqrt(n) <= t) x = n; else break;
    }
    return x;
}

int validate(int32_t H, int32_t W, const occ_baseline *b, int32_t V, const occ_params &p) {
    if (H < 2 || W < 2 || H > 32768 || W > 32768) return OCC_ERR_INVALID_ARG;
    if (V < 1 || b == nullptr) return OCC_ERR_INVALID_ARG;
    if (V > kMaxViews) return OCC_ERR_UNSUPPORTED;
    if (!(std::isfinite(p.t_edge) && p.t_edge > 0.0f)) return OCC_ERR_INVALID_ARG;
    if (!(p.t_dist >= 0x1p-12f && p.t_dist <= 0x1p16f)) return OCC_ERR_INVALID_ARG;
    if (!(p.t_disp >= 0.0f && p.t_disp <= 0x1p16f)) return OCC_ERR_INVALID_ARG;
    if (p.max_scan < 1 || p.max_scan > 65536) return OCC_ERR_INVALID_ARG;
    for (int32_t i = 0; i < V; ++i) {
        if (b[i].bx == 0 && b[i].by == 0) return OCC_ERR_INVALID_ARG;
        if (std::abs(b[i].bx) > 8 || std::abs(b[i].by) > 8) return OCC_ERR_UNSUPPORTED;
    }
    return OCC_OK;
}

// Near/far split of the Eq. 5 offsets for one view:
// backward offsets j >= jstar satisfy delta > t_disp automatically
// (s delta > j - t_dist >= s t_disp); forward offsets need f < t_dist - s t_disp.
void near_far(ViewDesc &vd, const occ_params &p) {
    const double t = p.t_dist, sd = (double)vd.s * (double)p.t_disp;
    int32_t j = 1;
    while ((double)j - t < sd) ++j;
    vd.jstar = j;
    vd.nback = j - 1;
    int32_t f = 0;
    while ((double)(f + 1) < t - sd) ++f;
    vd.nfwd = f;
    for (int32_t i = 0; i < kMaxNear; ++i) {
        vd.back_lo[i] = vd.back_hi[i] = vd.fwd_lo[i] = vd.fwd_hi[i] = 0.0f;
    }
    // delta in (lo, hi) <=> delta > t_disp and -t < dk + s delta < t   (S7)
    for (int32_t i = 0; i < vd.nback && i < kMaxNear; ++i) {
        const double dk = -(double)(i + 1);
        vd.back_lo[i] = std::fmax(p.t_disp, rd_div(-t - dk, vd.s));
        vd.back_hi[i] = ru_div(t - dk, vd.s);
    }
    for (int32_t i = 0; i < vd.nfwd && i < kMaxNear; ++i) {
        const double dk = (double)(i + 1);
        vd.fwd_lo[i] = std::fmax(p.t_disp, rd_div(-t - dk, vd.s));
        vd.fwd_hi[i] = ru_div(t - dk, vd.s);
    }
}

// CUDA errors map to OCC_ERR_CUDA; OCC_VERBOSE=1 prints the failing call
bool occ_verbose() {
    static const bool v = [] { const char *ev = getenv("OCC_VERBOSE"); return ev && atoi(ev) != 0; }();
    return v;
}
#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) {                                                                    \
            if (occ_verbose()) fprintf(stderr, "libocc: %s:%d %s -> %s\n", __FILE__, __LINE__, #x,   \
                                       cudaGetErrorString(e_));                                     \
            return OCC_ERR_CUDA;                                                                    \
        }                                                                                           \
    } while (0)

// Brackets one launch with events when profiling; returns a CUDA error.
struct ProfScope {
    occ_ctx *c; int kind; cudaStream_t s; bool on;
    ProfScope(occ_ctx *c_, int kind_, cudaStream_t s_) : c(c_), kind(kind_), s(s_), on(c_->profiling) {
        if (!on) return;
        auto &v = c->ev[kind];
        size_t &u = c->ev_used[kind];
        while (v.size() < u + 2) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) { on = false; return; }
            v.push_back(e);
        }
        cudaEventRecord(v[u], s);
    }
    void end() {
        if (!on) return;
        auto &v = c->ev[kind];
        size_t &u = c->ev_used[kind];
        if (v.size() >= u + 2) cudaEventRecord(v[u + 1], s);     // (scopes of one kind never nest)
        u += 2;
        on = false;
    }
};

// k_line serves a group when its family is rows / columns / diagonals /
// anti-diagonals, its views use the default near/far split (near backward
// offsets {1, 2}, far >= 3, <= 1 near forward offset whose lower bound equals
// the backward one), and the two views (if two) are +-b with equal s.
bool views_line_ok(const occ_ctx *c, const GroupDesc &g);
bool line_eligible(const occ_ctx *c, const GroupDesc &g) {
    const FamilyDesc &fd = c->fams[g.fam];
    if (fd.kind < 0 || fd.kind > 3 || g.nv < 1 || g.nv > 2) return false;
    return views_line_ok(c, g);
}
// the knight families (2, +-1), (1, +-2) through k_shear: the same view conditions
bool shear_eligible(const occ_ctx *c, const GroupDesc &g) {
    const FamilyDesc &fd = c->fams[g.fam];
    if (fd.kind < 4 || fd.kind > 7 || g.nv < 1 || g.nv > 2) return false;
    if (fd.den != 2) return false;        // (the sheared kernels shift by 1 for floor(t num / 2))
    return views_line_ok(c, g);
}
bool views_line_ok(const occ_ctx *c, const GroupDesc &g) {
    for (int32_t k = 0; k < g.nv; ++k) {
        const ViewDesc &v = c->views[g.view[k]];
        if (v.nback != 2 || v.jstar != 3 || v.nfwd > 1) return false;
        if (v.nfwd == 1 && v.fwd_lo[0] != v.back_lo[0]) return false;
    }
    if (g.nv == 2) {
        const ViewDesc &a = c->views[g.view[0]], &b = c->views[g.view[1]];
        if (a.sg == b.sg || a.s != b.s || a.nfwd != b.nfwd) return false;
        for (int i = 0; i < 2; ++i)
            if (a.back_lo[i] != b.back_lo[i] || a.back_hi[i] != b.back_hi[i]) return false;
        if (a.nfwd && (a.fwd_lo[0] != b.fwd_lo[0] || a.fwd_hi[0] != b.fwd_hi[0])) return false;
    }
    return true;
}

// Host copy of k_line's lane extent (LG<KIND>::ext): in-image positions of
// line L in the lane's time coordinate tau = pos + off(l).
void line_extent(int32_t kind, int32_t l0, int32_t l, int32_t H, int32_t W, int32_t &lo, int32_t &hi) {
    const int32_t L = l0 + l;
    if (kind == 0) { lo = 0; hi = (L >= 0 && L < H) ? W : 0; }
    else if (kind == 1) { lo = 0; hi = (L >= 0 && L < W) ? H : 0; }
    else if (kind == 2) {
        const int32_t a = std::max(0, -L), b = std::min(W, H - L);
        lo = a + l; hi = std::max(a, b) + l;
    } else {
        const int32_t a = std::max(0, L - H + 1), b = std::min(W, L + 1);
        lo = a + 31 - l; hi = std::max(a, b) + 31 - l;
    }
}

void add_line_units(occ_ctx *c, int32_t gi) {
    const int32_t kind = c->fams[c->groups[gi].fam].kind;
    const int32_t H = c->H, W = c->W;
    int32_t lmin = 0, lmax = 0;
    if (kind == 0) { lmin = 0; lmax = H - 1; }
    else if (kind == 1) { lmin = 0; lmax = W - 1; }
    else if (kind == 2) { lmin = -(W - 1); lmax = H - 1; }
    else { lmin = 0; lmax = H + W - 2; }
    for (int32_t l0 = lmin; l0 <= lmax; l0 += 32) {
        int32_t tlo = INT32_MAX, thi = INT32_MIN;
        for (int32_t l = 0; l < 32; ++l) {
            int32_t lo, hi;
            line_extent(kind, l0, l, H, W, lo, hi);
            if (lo < hi) { tlo = std::min(tlo, lo); thi = std::max(thi, hi); }
        }
        if (tlo >= thi) continue;
        const int32_t a = tlo & ~31, b = (thi + 31) & ~31;
        for (int32_t t0 = a; t0 < b; t0 += c->line_seg) {
            LineUnit u{};
            u.group = gi; u.l0 = l0; u.t0 = t0; u.t1 = std::min(t0 + c->line_seg, b);
            c->units.push_back(u);
        }
    }
}

// Host copy of k_sweep's lane extent (s_extent): in-image positions of line
// l0 + l (l0 a multiple of 32) in the sweep's coordinate tau.
void sweep_extent(int32_t kind, int32_t l0, int32_t l, int32_t H, int32_t W, int32_t &lo, int32_t &hi) {
    const int32_t L = l0 + l;
    if (kind == 0) { lo = 0; hi = (L >= 0 && L < H) ? W : 0; }
    else if (kind == 1) { lo = 0; hi = (L >= 0 && L < W) ? H : 0; }
    else if (kind == 2) { lo = std::max(l, -l0); hi = std::min(W + l, H - l0); }
    else { lo = std::max(31 - l, l0 + 32 - H); hi = std::min(W + 31 - l, l0 + 32); }
    if (hi < lo) hi = lo;
}

void add_sweep_units(occ_ctx *c, int32_t gi, int32_t seg) {
    const int32_t kind = c->fams[c->groups[gi].fam].kind;
    const int32_t H = c->H, W = c->W;
    int32_t lmin = 0, lmax = 0;
    if (kind == 0) { lmin = 0; lmax = H - 1; }
    else if (kind == 1) { lmin = 0; lmax = W - 1; }
    else if (kind == 2) { lmin = -(W - 1); lmax = H - 1; }
    else { lmin = 0; lmax = H + W - 2; }
    for (int32_t l0 = lmin & ~31; l0 <= lmax; l0 += 32) {
        int32_t tlo = INT32_MAX, thi = INT32_MIN;
        for (int32_t l = 0; l < 32; ++l) {
            int32_t lo, hi;
            sweep_extent(kind, l0, l, H, W, lo, hi);
            if (lo < hi) { tlo = std::min(tlo, lo); thi = std::max(thi, hi); }
        }
        if (tlo >= thi) continue;
        const int32_t a = tlo & ~31, b = (thi + 31) & ~31;
        for (int32_t t0 = a; t0 < b; t0 += seg) {
            SweepUnit u{};
            u.group = gi; u.l0 = l0; u.t0 = t0; u.t1 = std::min(t0 + seg, b);
            c->sunits.push_back(u);
        }
    }
}

// View groups (<= 2 views of one family, +-b pairs of equal s first) and the
// static tile list: for every group, blocks of 32 consecutive lines and
// segments of kTilePositions positions covering the lines' in-image extent.
// Pure integer geometry of the digital lines (S6); independent of the data.
void build_tiles(occ_ctx *c) {
    for (int32_t fam = 0; fam < c->nfam; ++fam) {
        const FamilyDesc &fd = c->fams[fam];
        std::vector<int32_t> vs(fd.view, fd.view + fd.nviews);
        std::stable_sort(vs.begin(), vs.end(), [&](int32_t a, int32_t b) {
            if (c->views[a].s != c->views[b].s) return c->views[a].s < c->views[b].s;
            return c->views[a].sg > c->views[b].sg;
        });
        for (size_t k = 0; k < vs.size(); k += kGroupViews) {
            GroupDesc g{};
            g.fam = fam;
            g.nv = 0;
            for (size_t j = k; j < vs.size() && j < k + kGroupViews; ++j) g.view[g.nv++] = vs[j];
            c->groups.push_back(g);
        }
    }
    const int32_t H = c->H, W = c->W;
    std::vector<char> eligible(c->groups.size(), 0);
    // k_sweep (default) or the round-1 k_line + k_cand path (OCC_SWEEP=0, kept for A/B runs)
    static const bool sweep = [] { const char *ev = getenv("OCC_SWEEP"); return !(ev && atoi(ev) == 0); }();
    std::vector<char> sheared(c->groups.size(), 0);
    static const bool shear_on = [] { const char *ev = getenv("OCC_SHEAR"); return !(ev && atoi(ev) == 0); }();
    for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi) {
        eligible[gi] = line_eligible(c, c->groups[gi]);
        if (eligible[gi] && !sweep) add_line_units(c, gi);
        sheared[gi] = sweep && shear_on && shear_eligible(c, c->groups[gi]);
    }
    if (sweep) {
        // segment length: 256 positions, halved while one call of max_batch
        // frames would not fill the GPU (148 SMs x 16 warps)
        int32_t seg = kSweepSeg;
        static const int fill = [] { const char *ev = getenv("OCC_SWEEP_FILL"); return ev ? atoi(ev) : 16; }();
        for (;;) {
            c->sunits.clear();
            for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi)
                if (eligible[gi]) add_sweep_units(c, gi, seg);
            if (seg <= 32 || (double)c->sunits.size() * c->max_batch >= 148.0 * fill) break;
            seg = std::max(32, (seg / 2) & ~31);
        }
        c->ssmin = INT32_MAX;
        for (const SweepUnit &x : c->sunits) c->ssmin = std::min(c->ssmin, c->views[c->groups[x.group].view[0]].s);
        if (c->sunits.empty()) c->ssmin = 1;
        // by kind, longest first inside a kind (k_sweep's work order, k_sweep.cu)
        // segment order of the kinds inside a frame group: diagonals (the
        // longer units, ~1.7x a row unit's work) first, so a group's last
        // wave is made of short units (C5 A/B on one B200, ms per step:
        // 0123 18.46, 2301 18.33, 2310 18.35, 0132 18.52); OCC_SWEEP_KORDER
        // overrides it (a permutation of "0123"; the kernel takes the
        // segments in turn whatever kinds they hold)
        static const std::string korder = [] {
            const char *ev = getenv("OCC_SWEEP_KORDER");
            std::string o = ev ? ev : "2301";
            std::string t = o;
            std::sort(t.begin(), t.end());
            return t == "0123" ? o : std::string("2301");
        }();
        auto rank_of = [&](const SweepUnit &x) {
            return (int)korder.find((char)('0' + c->fams[c->groups[x.group].fam].kind));
        };
        std::stable_sort(c->sunits.begin(), c->sunits.end(), [&](const SweepUnit &x, const SweepUnit &y) {
            if (rank_of(x) != rank_of(y)) return rank_of(x) < rank_of(y);
            return x.t1 - x.t0 > y.t1 - y.t0;
        });
        for (int k = 0; k <= 4; ++k) {
            int32_t n = 0;
            for (const SweepUnit &x : c->sunits) n += rank_of(x) < k ? 1 : 0;
            c->skstart[k] = n;
        }
        // frames per group: every kind's share of a group about one resident
        // wave (148 SMs x 16 warps), and a group's D + words within ~40 MB of L2
        int32_t kmin = INT32_MAX;
        for (int k = 0; k < 4; ++k)
            if (c->skstart[k + 1] > c->skstart[k]) kmin = std::min(kmin, c->skstart[k + 1] - c->skstart[k]);
        const double fbytes = (double)H * W * 4.0 + 4.0 * (double)sweep_words_per_frame(H, W);
        const int32_t by_wave = (int32_t)std::ceil(148.0 * 16 / std::max(1, kmin));
        // (C5, 256 frames, ms: 1 19.99, 2 19.95, 3 19.90, 4 19.98, 7 20.02, 10 20.09, 14 20.29)
        const int32_t by_l2 = std::max(1, (int32_t)(40.0e6 / fbytes));
        c->sfgroup = std::max(1, std::min(by_wave, by_l2));
        if (const char *ev = getenv("OCC_SWEEP_FGROUP")) c->sfgroup = std::max(1, atoi(ev));   // tuning knob
        // knight families: one sheared frame per family; its lines become the
        // rows (x-major) or columns (y-major) of that frame
        for (int32_t fm = 0; fm < (int32_t)c->fams.size(); ++fm) {
            std::vector<int32_t> gs;
            for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi)
                if (sheared[gi] && c->groups[gi].fam == fm) gs.push_back(gi);
            if (gs.empty()) continue;
            const FamilyDesc &fd = c->fams[fm];
            occ_ctx::ShearFam sf;
            sf.fam = fm;
            ShearDesc &sd = sf.sd;
            sd.kind = fd.xmajor ? 0 : 1;
            sd.num = fd.num; sd.den = fd.den; sd.Ho = H; sd.Wo = W;
            const int32_t PM = fd.xmajor ? W : H, QM = fd.xmajor ? H : W;
            auto fdv = [&](int32_t t) { return floordiv(t * fd.num, fd.den); };
            const int32_t f0 = fdv(0), f1 = fdv(PM - 1);
            sd.lmin = -std::max(f0, f1);
            const int32_t nl = QM - 1 - std::min(f0, f1) - sd.lmin + 1;     // lines
            // rows padded to 32 floats (NaN): TMA boxes need 16-byte row strides
            sf.Hs = fd.xmajor ? nl : H;
            sf.Ws = ((fd.xmajor ? W : nl) + 31) & ~31;
            // units: 32-line blocks x seg positions over the block's in-image extent
            for (int32_t gi : gs) {
                for (int32_t l0 = 0; l0 < nl; l0 += 32) {
                    int32_t lo = INT32_MAX, hi = INT32_MIN;
                    for (int32_t l = l0; l < std::min(nl, l0 + 32); l += std::max(1, std::min(31, nl - 1 - l))) {
                        const int32_t L = l + sd.lmin;
                        for (int32_t t = 0; t < PM; ++t) {
                            const int32_t q = L + fdv(t);
                            if (q >= 0 && q < QM) { lo = std::min(lo, t); hi = std::max(hi, t + 1); }
                        }
                    }
                    if (lo >= hi) continue;
                    const int32_t a0 = lo & ~31, b0 = (hi + 31) & ~31;
                    for (int32_t t0 = a0; t0 < b0; t0 += seg) {
                        SweepUnit u{};
                        u.group = gi; u.l0 = l0; u.t0 = t0; u.t1 = std::min(t0 + seg, b0);
                        sf.units.push_back(u);
                    }
                }
            }
            std::stable_sort(sf.units.begin(), sf.units.end(),
                             [](const SweepUnit &x, const SweepUnit &y) { return x.t1 - x.t0 > y.t1 - y.t0; });
            const int32_t nu = (int32_t)sf.units.size();
            sf.kstart[0] = 0;
            for (int k = 1; k <= 4; ++k) sf.kstart[k] = nu;
            const double sbytes = (double)sf.Hs * sf.Ws * 4.0 + 4.0 * (double)sweep_words_per_frame(sf.Hs, sf.Ws);
            const int32_t sw = (int32_t)std::ceil(148.0 * 16 / std::max(1, nu));
            sf.fgroup = std::max(1, std::min(sw, std::max(1, (int32_t)(40.0e6 / sbytes))));
            sf.smin = INT32_MAX;
            for (int32_t gi : gs) sf.smin = std::min(sf.smin, c->views[c->groups[gi].view[0]].s);
            c->shear.push_back(std::move(sf));
        }
    }
    // segment length: 256 positions, shorter when a call of max_batch frames
    // would not fill the GPU (a unit is one warp's serial work, ~0.1 ms at
    // 256 positions): single small frames trade margin work for parallelism
    static const int min_seg = [] { const char *ev = getenv("OCC_LINE_MINSEG"); return ev ? std::max(32, atoi(ev)) : 32; }();
    // one resident wave is 148 SMs x 16 warps (k_line at 4 warps per CTA)
    while (c->line_seg > min_seg && (double)c->units.size() * c->max_batch < 148.0 * 16) {
        c->line_seg /= 2;
        c->units.clear();
        for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi)
            if (eligible[gi]) add_line_units(c, gi);
    }
    // k_cand word blocks: for every family with line units, all 32-line
    // blocks x all 32-position tau blocks of its lines' extents
    c->candfam.assign((size_t)c->nfam, CandFam{});
    {
        std::vector<char> lfam((size_t)c->nfam, 0);
        for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi)
            if (eligible[gi]) lfam[(size_t)c->groups[gi].fam] = 1;
        int64_t base = 0;
        for (int32_t fm = 0; fm < c->nfam; ++fm) {
            CandFam cf{};
            cf.fam = fm;
            cf.kind = c->fams[(size_t)fm].kind;
            cf.base_slot = base;
            if (lfam[(size_t)fm] && cf.kind <= 3) {
                int32_t lmin = 0, lmax = 0;
                if (cf.kind == 0) { lmin = 0; lmax = H - 1; }
                else if (cf.kind == 1) { lmin = 0; lmax = W - 1; }
                else if (cf.kind == 2) { lmin = -(W - 1); lmax = H - 1; }
                else { lmin = 0; lmax = H + W - 2; }
                int32_t tlo = INT32_MAX, thi = INT32_MIN;
                for (int32_t l0 = lmin; l0 <= lmax; l0 += 32)
                    for (int32_t l = 0; l < 32; ++l) {
                        int32_t lo, hi;
                        line_extent(cf.kind, l0, l, H, W, lo, hi);
                        if (lo < hi) { tlo = std::min(tlo, lo); thi = std::max(thi, hi); }
                    }
                if (tlo < thi) {
                    cf.lmin = lmin;
                    cf.nlb = (lmax - lmin) / 32 + 1;
                    cf.kmin = floordiv(tlo, 32);
                    cf.nk = floordiv(thi - 1, 32) - cf.kmin + 1;
                    base += (int64_t)cf.nlb * cf.nk;
                }
            }
            c->candfam[(size_t)fm] = cf;
        }
        c->cand_per_frame = base;
        for (CandFam &cf : c->candfam) cf.per_frame = base;
    }
    // longest units first (diagonal families sweep ~1.7x the work per
    // position): the last wave of warps is made of short units
    std::stable_sort(c->units.begin(), c->units.end(), [&](const LineUnit &x, const LineUnit &y) {
        auto cost = [&](const LineUnit &u) {
            const int32_t kind = c->fams[c->groups[u.group].fam].kind;
            return (double)(u.t1 - u.t0 + 96) * (kind >= 2 ? 1.7 : 1.0);
        };
        return cost(x) > cost(y);
    });
    for (int32_t gi = 0; gi < (int32_t)c->groups.size(); ++gi) {
        const FamilyDesc &fd = c->fams[c->groups[gi].fam];
        const int32_t num = fd.num, den = fd.den;
        const int32_t PM = fd.xmajor ? W : H;      // positions
        const int32_t QM = fd.xmajor ? H : W;      // the other axis
        auto fdv = [&](int32_t a) { return floordiv(a * num, den); };
        const int32_t f0 = fdv(0), f1 = fdv(PM - 1);
        const int32_t lmin = 0 - std::max(f0, f1), lmax = QM - 1 - std::min(f0, f1);
        for (int32_t l0 = lmin; l0 <= lmax; l0 += 32) {
            int32_t plo = INT32_MAX, phi = -1;
            for (int32_t pos = 0; pos < PM; ++pos) {
                const int32_t q0 = l0 + fdv(pos);
                if (q0 <= QM - 1 && q0 + 31 >= 0) { plo = std::min(plo, pos); phi = pos; }
            }
            if (phi < 0) continue;
            for (int32_t p0 = plo; p0 <= phi; p0 += kTilePositions) {
                TileDesc t{};
                t.group = gi; t.l0 = l0; t.p0 = p0; t.p1 = std::min(p0 + kTilePositions, phi + 1);
                c->all_tiles.push_back(t);
                if (!eligible[gi] && !sheared[gi]) c->tiles.push_back(t);
            }
        }
    }
}

// Capacity of the k_line / k_sweep -> k_hard queue: 1/2 of a chunk's
// pixel-views, clamped to [64 Ki, 512 Mi] entries (16 B each: at most 8 GiB
// of the 180 GB).  Survivors grow with the occluded fraction, which grows
// with h: C5 frames (h ~ 66) queue 1.4 % of their pixel-views, the same
// frames scaled to h ~ 300 about 10 %, to h ~ 600 about 30 %; past the
// capacity the sweep warps search in-warp (exact, ~30x slower at h = 300).  OCC_GQ_CAP (test knob,
// read at occ_create) overrides it, e.g. to force the capacity-overflow path.
int32_t gq_capacity(int32_t chunk, int32_t H, int32_t W, int32_t n_views) {
    const char *ev = getenv("OCC_GQ_CAP");
    if (ev && atoi(ev) > 0) return atoi(ev);
    return (int32_t)std::min<double>(512.0 * 1048576.0, std::max(65536.0, (double)chunk * H * W * n_views / 2.0));
}

}  // namespace

extern "C" {

void occ_default_params(occ_params *p) {
    if (!p) return;
    p->t_edge = 1.0f;
    p->t_dist = 2.0f;
    p->t_disp = 0.5f;
    p->max_scan = 4096;
}

int32_t occ_version(void) { return 10000; }

const char *occ_strerror(int code) {
    switch (code) {
        case OCC_OK: return "ok";
        case OCC_ERR_INVALID_ARG: return "invalid argument";
        case OCC_ERR_CUDA: return "CUDA runtime error";
        case OCC_ERR_OOM: return "out of device memory";
        case OCC_ERR_NONFINITE: return "non-finite disparity in frame";
        case OCC_ERR_UNSUPPORTED: return "unsupported baseline or view count";
        default: return "unknown error";
    }
}

// device buffers of the sheared (knight) families: one sheared frame and its
// words per chunk frame (sized for the largest family), unit lists
bool alloc_shear(occ_ctx *c) {
    c->main_qcap = c->gq_cap;
    if (c->shear.empty()) return true;
    // queue regions in proportion to the views each sweep serves
    int32_t vmain = 0;
    {
        std::vector<char> inmain(c->groups.size(), 0);
        for (const SweepUnit &u : c->sunits) inmain[(size_t)u.group] = 1;
        for (size_t g = 0; g < c->groups.size(); ++g) vmain += inmain[g] ? c->groups[g].nv : 0;
    }
    int32_t vtot = vmain;
    std::vector<int32_t> vsh;
    for (auto &sf : c->shear) {
        std::vector<char> in(c->groups.size(), 0);
        for (const SweepUnit &u : sf.units) in[(size_t)u.group] = 1;
        int32_t v = 0;
        for (size_t g = 0; g < c->groups.size(); ++g) v += in[g] ? c->groups[g].nv : 0;
        vsh.push_back(std::max(1, v));
        vtot += std::max(1, v);
    }
    c->main_qcap = (int32_t)((double)c->gq_cap * vmain / vtot);
    int64_t q = c->main_qcap;
    for (size_t k = 0; k < c->shear.size(); ++k) {
        auto &sf = c->shear[k];
        sf.q0 = q;
        sf.qcap = (int32_t)((double)c->gq_cap * vsh[k] / vtot);
        q += sf.qcap;
        if (cudaMalloc(&sf.d_units, sizeof(SweepUnit) * std::max<size_t>(1, sf.units.size())) != cudaSuccess ||
            (sf.units.size() && cudaMemcpy(sf.d_units, sf.units.data(), sizeof(SweepUnit) * sf.units.size(),
                                           cudaMemcpyHostToDevice) != cudaSuccess) ||
            cudaMalloc(&sf.d_D, sizeof(float) * (size_t)c->chunk * sf.Hs * sf.Ws) != cudaSuccess ||
            cudaMalloc(&sf.d_W, sizeof(uint32_t) * (size_t)c->chunk * (size_t)sweep_words_per_frame(sf.Hs, sf.Ws)) !=
                cudaSuccess ||
            cudaStreamCreateWithFlags(&sf.st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sf.done, cudaEventDisableTiming) != cudaSuccess)
            return false;
    }
    return cudaEventCreateWithFlags(&c->sh_fork, cudaEventDisableTiming) == cudaSuccess;
}

// Device side of a context whose views (and families) are set up: work
// lists, chunking, device copies, offset tables.  Frees c on failure.
int create_tail(occ_ctx *c, int32_t H, int32_t W, int32_t n_views, int32_t max_batch, occ_ctx **out) {
    c->nfam = (int32_t)c->fams.size();
    build_tiles(c);
    c->code_bytes = c->nfam <= 4 ? 1 : (c->nfam <= 8 ? 2 : 4);
    {   // frames per K0/K1 chunk.  With frame-major k_line the chunk only
        // sets the launch count (L2 locality is per frame); measured at C5:
        // 256 MiB (25 frames) 53.1 ms/step, 1 GiB 51.5, 2 GiB (207 frames)
        // 51.3, 4 GiB (one launch) 52.4
        double shear_per = 0.0;
        for (const auto &sf : c->shear)
            shear_per += (double)sf.Hs * sf.Ws * 4.0 + 4.0 * (double)sweep_words_per_frame(sf.Hs, sf.Ws);
        const double per = (double)H * W * (4.0 + c->code_bytes) +
                           (c->sunits.empty() && c->shear.empty() ? 0.0 : 4.0 * (double)sweep_words_per_frame(H, W)) +
                           shear_per;
        const char *ev = getenv("OCC_CHUNK_MIB");          // tuning knob (default 2 GiB)
        const double budget = (ev ? std::max(1, atoi(ev)) : 2048) * 1048576.0;
        c->chunk = (int32_t)std::max(1.0, std::min((double)kMaxChunkFrames, std::floor(budget / per)));
        c->chunk = std::min(c->chunk, max_batch);
    }

    if (cudaGetDevice(&c->device) != cudaSuccess) { cudaGetLastError(); delete c; return OCC_ERR_CUDA; }
    if (cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess) c->nsm = 148;
    if (cudaMalloc(&c->d_views, sizeof(ViewDesc) * c->views.size()) != cudaSuccess ||
        cudaMalloc(&c->d_fams, sizeof(FamilyDesc) * c->fams.size()) != cudaSuccess ||
        cudaMalloc(&c->d_groups, sizeof(GroupDesc) * c->groups.size()) != cudaSuccess ||
        cudaMalloc(&c->d_tiles, sizeof(TileDesc) * std::max<size_t>(1, c->tiles.size())) != cudaSuccess ||
        cudaMalloc(&c->d_all_tiles, sizeof(TileDesc) * std::max<size_t>(1, c->all_tiles.size())) != cudaSuccess ||
        cudaMalloc(&c->d_units, sizeof(LineUnit) * std::max<size_t>(1, c->units.size())) != cudaSuccess ||
        cudaMalloc(&c->d_stats, sizeof(FrameStats) * (size_t)max_batch) != cudaSuccess ||
        cudaMalloc(&c->d_codes, (size_t)c->chunk * H * W * c->code_bytes) != cudaSuccess ||
        ((!c->units.empty() || !c->sunits.empty() || !c->shear.empty()) &&
         (cudaMalloc(&c->d_gq, sizeof(HardEntry) * (size_t)(c->gq_cap = gq_capacity(c->chunk, H, W, n_views))) != cudaSuccess ||
          cudaMalloc(&c->d_gq_count, sizeof(uint32_t) * (2 + kMaxFamilies)) != cudaSuccess)) ||
        ((!c->sunits.empty() || !c->shear.empty()) &&
         (cudaMalloc(&c->d_sunits, sizeof(SweepUnit) * std::max<size_t>(1, c->sunits.size())) != cudaSuccess ||
          cudaMalloc(&c->d_words, sizeof(uint32_t) * (size_t)c->chunk * (size_t)sweep_words_per_frame(H, W)) != cudaSuccess ||
          (max_batch > c->chunk &&
           cudaMalloc(&c->d_words2, sizeof(uint32_t) * (size_t)c->chunk * (size_t)sweep_words_per_frame(H, W)) !=
               cudaSuccess))) ||
        !alloc_shear(c)) {
        cudaGetLastError();
        occ_destroy(c);
        return OCC_ERR_OOM;
    }
    if (cudaMemcpy(c->d_views, c->views.data(), sizeof(ViewDesc) * c->views.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_fams, c->fams.data(), sizeof(FamilyDesc) * c->fams.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_groups, c->groups.data(), sizeof(GroupDesc) * c->groups.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        (c->tiles.size() && cudaMemcpy(c->d_tiles, c->tiles.data(), sizeof(TileDesc) * c->tiles.size(),
                                       cudaMemcpyHostToDevice) != cudaSuccess) ||
        (c->all_tiles.size() && cudaMemcpy(c->d_all_tiles, c->all_tiles.data(),
                                           sizeof(TileDesc) * c->all_tiles.size(),
                                           cudaMemcpyHostToDevice) != cudaSuccess) ||
        (c->units.size() && cudaMemcpy(c->d_units, c->units.data(), sizeof(LineUnit) * c->units.size(),
                                       cudaMemcpyHostToDevice) != cudaSuccess) ||
        (c->sunits.size() && cudaMemcpy(c->d_sunits, c->sunits.data(), sizeof(SweepUnit) * c->sunits.size(),
                                        cudaMemcpyHostToDevice) != cudaSuccess)) {
        occ_destroy(c);
        return OCC_ERR_CUDA;
    }
    {   // k_cand word buffer for one chunk (optional: pass 0 falls back to the codes)
        const char *ev = getenv("OCC_LINE_CAND");
        const bool want = !(ev && atoi(ev) == 0);
        if (want && !c->units.empty() && c->cand_per_frame > 0) {
            if (cudaMalloc(&c->d_candfam, sizeof(CandFam) * c->candfam.size()) != cudaSuccess ||
                cudaMemcpy(c->d_candfam, c->candfam.data(), sizeof(CandFam) * c->candfam.size(),
                           cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMalloc(&c->d_cand, (size_t)c->chunk * (size_t)c->cand_per_frame * 64 * sizeof(uint32_t)) != cudaSuccess) {
                cudaGetLastError();
                cudaFree(c->d_cand);
                c->d_cand = nullptr;
            }
        }
    }
    if (c->angles && cudaMalloc(&c->d_nwin_work, 2 * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        occ_destroy(c);
        return OCC_ERR_OOM;
    }
    if (c->angles) {   // Eq. 4 sample offsets of every direction, |g| <= max_scan / 2
        const int32_t hc = c->params.max_scan / 2, n = 2 * hc + 1;
        std::vector<int2> off((size_t)n * c->V);
        for (int32_t v = 0; v < c->V; ++v) {
            const ViewDesc &vd = c->views[(size_t)v];
            for (int32_t g = -hc; g <= hc; ++g) {
                // round half away from zero of g u, u = (-cos phi, -sin phi) (reading Q23)
                off[(size_t)v * n + (g + hc)] = make_int2((int32_t)std::round((double)g * vd.ux),
                                                          (int32_t)std::round((double)g * vd.uy));
            }
        }
        if (cudaMalloc(&c->d_offs, sizeof(int2) * off.size()) != cudaSuccess) { cudaGetLastError(); occ_destroy(c); return OCC_ERR_OOM; }
        if (cudaMemcpy(c->d_offs, off.data(), sizeof(int2) * off.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            occ_destroy(c);
            return OCC_ERR_CUDA;
        }
    }
    *out = c;
    return OCC_OK;
}

int occ_create(int32_t H, int32_t W, const occ_baseline *baselines, int32_t n_views,
               const occ_params *params, int32_t max_batch, occ_ctx **out) {
    if (!out) return OCC_ERR_INVALID_ARG;
    *out = nullptr;
    occ_params p;
    occ_default_params(&p);
    if (params) p = *params;
    int rc = validate(H, W, baselines, n_views, p);
    if (rc != OCC_OK) return rc;
    if (max_batch < 1) return OCC_ERR_INVALID_ARG;

    occ_ctx *c = new (std::nothrow) occ_ctx();
    if (!c) return OCC_ERR_OOM;
    c->H = H; c->W = W; c->V = n_views; c->max_batch = max_batch;
    c->mf.packed = 0; c->mf.Wb = (W + 31) / 32; c->mf.vbytes = (int64_t)H * W;
    c->params.t_edge = p.t_edge;
    c->params.t_dist = p.t_dist;
    c->params.t_disp = p.t_disp;
    c->params.max_scan = p.max_scan;
    c->params.e2_thresh = sqrt_thresh(p.t_edge);

    // families: lines shared by +-m b0 (S6); b0 reduced with positive major
    for (int32_t i = 0; i < n_views; ++i) {
        ViewDesc vd{};
        vd.bx = baselines[i].bx; vd.by = baselines[i].by;
        vd.s = std::max(std::abs(vd.bx), std::abs(vd.by));
        vd.xmajor = std::abs(vd.bx) >= std::abs(vd.by) ? 1 : 0;
        const int32_t g = igcd(vd.bx, vd.by);
        int32_t b0x = vd.bx / g, b0y = vd.by / g;
        const int32_t major = vd.xmajor ? b0x : b0y;
        vd.sg = major > 0 ? 1 : -1;
        if (vd.sg < 0) { b0x = -b0x; b0y = -b0y; }
        if (vd.xmajor) { vd.num = b0y; vd.den = b0x; }
        else { vd.num = b0x; vd.den = b0y; }
        int32_t fam = -1;
        for (size_t k = 0; k < c->fams.size(); ++k)
            if (c->fams[k].b0x == b0x && c->fams[k].b0y == b0y) fam = (int32_t)k;
        if (fam < 0) {
            if ((int32_t)c->fams.size() >= kMaxFamilies) { delete c; return OCC_ERR_UNSUPPORTED; }
            FamilyDesc fd{};
            fd.b0x = b0x; fd.b0y = b0y; fd.xmajor = vd.xmajor; fd.num = vd.num; fd.den = vd.den;
            fd.nviews = 0;
            // k_tile's compile-time geometry variants (rows, columns, diagonals, knights)
            const int32_t X = fd.xmajor, n = fd.num, dd = fd.den;
            fd.kind = (X && n == 0) ? 0 : (!X && n == 0) ? 1 : (X && n == 1 && dd == 1) ? 2
                    : (X && n == -1 && dd == 1) ? 3 : (X && n == 1 && dd == 2) ? 4
                    : (X && n == -1 && dd == 2) ? 5 : (!X && n == 1 && dd == 2) ? 6
                    : (!X && n == -1 && dd == 2) ? 7 : 8;
            c->fams.push_back(fd);
            fam = (int32_t)c->fams.size() - 1;
        }
        FamilyDesc &fd = c->fams[fam];
        fd.view[fd.nviews++] = i;
        vd.fam = fam;
        vd.candbit = 2 * fam + (vd.sg < 0 ? 1 : 0);
        vd.lkind = fd.kind;
        near_far(vd, p);
        vd.rho = (double)vd.s;
        c->views.push_back(vd);
    }
    return create_tail(c, H, W, n_views, max_batch, out);
}

int occ_create_dirs(int32_t H, int32_t W, const occ_direction *dirs, int32_t n_views,
                    const occ_params *params, int32_t max_batch, occ_ctx **out) {
    if (!out) return OCC_ERR_INVALID_ARG;
    *out = nullptr;
    occ_params p;
    occ_default_params(&p);
    if (params) p = *params;
    if (H < 2 || W < 2 || H > 32768 || W > 32768 || n_views < 1 || !dirs || max_batch < 1) return OCC_ERR_INVALID_ARG;
    if (n_views > kMaxViews) return OCC_ERR_UNSUPPORTED;
    if (!(std::isfinite(p.t_edge) && p.t_edge > 0.0f) || !(p.t_dist >= 0x1p-12f && p.t_dist <= 0x1p16f) ||
        !(p.t_disp >= 0.0f && p.t_disp <= 0x1p16f) || p.max_scan < 1 || p.max_scan > 65536)
        return OCC_ERR_INVALID_ARG;
    for (int32_t i = 0; i < n_views; ++i)
        if (!std::isfinite(dirs[i].baseline_angle) || !(dirs[i].baseline_length > 0.0 && dirs[i].baseline_length <= 8.0))
            return OCC_ERR_INVALID_ARG;
    occ_ctx *c = new (std::nothrow) occ_ctx();
    if (!c) return OCC_ERR_OOM;
    c->H = H; c->W = W; c->V = n_views; c->max_batch = max_batch;
    c->mf.packed = 0; c->mf.Wb = (W + 31) / 32; c->mf.vbytes = (int64_t)H * W;
    c->params.t_edge = p.t_edge;
    c->params.t_dist = p.t_dist;
    c->params.t_disp = p.t_disp;
    c->params.max_scan = p.max_scan;
    c->params.e2_thresh = sqrt_thresh(p.t_edge);
    c->angles = 1;
    for (int32_t i = 0; i < n_views; ++i) {
        ViewDesc vd{};
        vd.angle = 1;
        vd.ca = std::cos(dirs[i].baseline_angle);       // Eq. 2 direction (reading Q23)
        vd.sa = std::sin(dirs[i].baseline_angle);
        vd.ux = -vd.ca;                                 // displacement = baseline + pi
        vd.uy = -vd.sa;
        vd.rho = dirs[i].baseline_length;
        vd.s = (int32_t)std::ceil(vd.rho);
        vd.off_base = i * (2 * (p.max_scan / 2) + 1);
        vd.fam = -1;
        vd.candbit = 31;
        c->views.push_back(vd);
    }
    return create_tail(c, H, W, n_views, max_batch, out);
}

int occ_set_mask_format(occ_ctx *c, int32_t format) {
    if (!c || (format != OCC_MASK_U8 && format != OCC_MASK_BITS)) return OCC_ERR_INVALID_ARG;
    c->mf.packed = format == OCC_MASK_BITS;
    c->mf.Wb = (c->W + 31) / 32;
    c->mf.vbytes = c->mf.packed ? (int64_t)c->H * c->mf.Wb * 4 : (int64_t)c->H * c->W;
    return OCC_OK;
}

int64_t occ_mask_bytes(const occ_ctx *c, int32_t batch) {
    if (!c || batch < 0) return -1;
    return (int64_t)batch * c->V * c->mf.vbytes;
}

int occ_set_path(occ_ctx *c, int32_t path) {
    if (!c || path < OCC_PATH_AUTO || path > OCC_PATH_DIRECT) return OCC_ERR_INVALID_ARG;
    c->path = path;
    return OCC_OK;
}

int32_t occ_last_launches(const occ_ctx *c) { return c ? c->last_launches : -1; }

int occ_set_neighbors(occ_ctx *c, int32_t N) {
    if (!c || N < 0 || N == 1 || (N & 1) || N > 65536) return OCC_ERR_INVALID_ARG;
    if (N > 0 && !c->d_nwin_work) {
        CK(cudaSetDevice(c->device));
        if (cudaMalloc(&c->d_nwin_work, 2 * sizeof(uint32_t)) != cudaSuccess) {
            cudaGetLastError();
            return OCC_ERR_OOM;
        }
    }
    c->neighbors = N;
    return OCC_OK;
}

int32_t occ_get_neighbors(const occ_ctx *c) { return c ? c->neighbors : -1; }

int occ_frame_stats(occ_ctx *c, const float *D, int32_t batch, float *dmin, float *dmax, int32_t *nonfinite,
                    void *stream) {
    if (!c || !D || batch < 1 || batch > c->max_batch) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    // own scratch: the context's d_stats belong to the last occ_detect (occ_status)
    FrameStats *st = nullptr;
    if (cudaMalloc(&st, sizeof(FrameStats) * (size_t)batch) != cudaSuccess) { cudaGetLastError(); return OCC_ERR_OOM; }
    std::vector<FrameStats> h((size_t)batch);
    cudaError_t e = launch_stats_init(st, batch, s);
    if (e == cudaSuccess) e = launch_stats(D, (int64_t)c->H * c->W, batch, st, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), st, sizeof(FrameStats) * h.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(st);
    if (e != cudaSuccess) return OCC_ERR_CUDA;
    for (int32_t f = 0; f < batch; ++f) {
        if (dmin) dmin[f] = key_float(h[(size_t)f].minkey);
        if (dmax) dmax[f] = key_float(h[(size_t)f].maxkey);
        if (nonfinite) nonfinite[f] = (int32_t)h[(size_t)f].nonfinite;
    }
    return OCC_OK;
}

int occ_set_frame_stats(occ_ctx *c, const float *dmin, const float *dmax, const int32_t *nonfinite, int32_t n) {
    if (!c || n < 0 || n > c->max_batch || (n > 0 && (!dmin || !dmax || !nonfinite))) return OCC_ERR_INVALID_ARG;
    std::vector<FrameStats> h((size_t)n);
    for (int32_t f = 0; f < n; ++f) {
        if (!nonfinite[f] && !(dmin[f] <= dmax[f])) return OCC_ERR_INVALID_ARG;
        h[(size_t)f].minkey = float_key(dmin[f]);
        h[(size_t)f].maxkey = float_key(dmax[f]);
        h[(size_t)f].nonfinite = (uint32_t)std::max(0, nonfinite[f]);
        h[(size_t)f].pad = 0;
    }
    CK(cudaSetDevice(c->device));
    if (n > 0) {
        if (!c->d_override) {
            if (cudaMalloc(&c->d_override, sizeof(FrameStats) * (size_t)c->max_batch) != cudaSuccess) {
                cudaGetLastError();
                return OCC_ERR_OOM;
            }
        }
        CK(cudaDeviceSynchronize());     // no call in flight may still read the old values
        CK(cudaMemcpy(c->d_override, h.data(), sizeof(FrameStats) * (size_t)n, cudaMemcpyHostToDevice));
    }
    c->n_override = n;
    return OCC_OK;
}

}  // extern "C"

namespace {
int32_t smax_of(const occ_ctx *c) {
    int32_t m = 1;
    for (const ViewDesc &v : c->views) m = std::max(m, (int32_t)std::ceil(v.rho));
    return m;
}

// K0 + K1 for frames [c0, c0 + n) of a batch whose frames start at D / M (device).
// slot: 0, or 1 for the odd chunks of an alternating call (second words
// buffer, second half of the main queue region); -1: the whole region
int detect_chunk(occ_ctx *c, const float *D, uint8_t *M, int32_t c0, int32_t n, cudaStream_t s, int &launches,
                 int slot = -1, cudaEvent_t swept = nullptr) {
    uint32_t *words = slot == 1 ? c->d_words2 : c->d_words;
    const int32_t qcap = slot < 0 ? c->main_qcap : c->main_qcap / 2;
    HardEntry *gqm = c->d_gq + (slot == 1 ? qcap : 0);
    uint32_t *gqc = slot == 1 ? c->d_gq_count + 1 + kMaxFamilies : c->d_gq_count;
    const int64_t HW = (int64_t)c->H * c->W;
    const float *Dc = D + (int64_t)c0 * HW;
    uint8_t *Mc = M + (int64_t)c0 * c->V * c->mf.vbytes;
    const bool tiled_only = c->path == OCC_PATH_TILED;
    const bool nwin = c->neighbors > 0 || c->angles;
    const bool sweep = !tiled_only && !nwin && (!c->sunits.empty() || !c->shear.empty());
    const TileDesc *tl = tiled_only ? c->d_all_tiles : c->d_tiles;
    const int32_t nt = (int32_t)(tiled_only ? c->all_tiles.size() : c->tiles.size());
    {
        ProfScope ps(c, OCC_KERNEL_STATS, s);
        if (sweep) {
            CK(launch_words(Dc, c->H, c->W, n, c->params.e2_thresh, c->d_stats + c0, words, 1, s)); ++launches;
            if (nt > 0) {    // k_tile's groups read the per-pixel codes
                CK(launch_prologue(Dc, c->H, c->W, n, c->fams.data(), c->nfam, c->params.e2_thresh,
                                   c->d_stats + c0, c->d_codes, c->code_bytes, 0, s)); ++launches;
            }
        } else {
            CK(launch_prologue(Dc, c->H, c->W, n, c->fams.data(), c->nfam, c->params.e2_thresh,
                               c->d_stats + c0, c->d_codes, c->code_bytes, 1, s)); ++launches;
        }
        if (c->n_override > c0)    // imposed whole-frame statistics (spatial sharding)
            CK(cudaMemcpyAsync(c->d_stats + c0, c->d_override + c0,
                               sizeof(FrameStats) * (size_t)std::min(n, c->n_override - c0),
                               cudaMemcpyDeviceToDevice, s));
        ps.end();
    }
    if (nwin) {   // finite N / real directions: per-window kernel (masks pre-zeroed)
        ProfScope pn(c, OCC_KERNEL_NWIN, s);
        CK(launch_nwin(Dc, c->H, c->W, n, c->d_views, c->V, c->d_stats + c0, c->params, c->neighbors, Mc,
                       c->mf, c->d_codes, c->code_bytes, c->d_nwin_work, c->nwin_big, smax_of(c), c->angles,
                       c->d_offs, c->nsm, s));
        launches += 2 * c->params.max_scan / 2 + 1 > kNwinCap ? 2 : 1;
        pn.end();
        return OCC_OK;
    }
    if (sweep) {
        CK(cudaMemsetAsync(gqc, 0, sizeof(uint32_t), s));
#ifdef OCC_CHECKS
        // poison the queue: a slot k_hard reads that this chunk did not write fails its checks
        CK(cudaMemsetAsync(c->d_gq, 0xFF, sizeof(HardEntry) * (size_t)c->gq_cap, s));
#endif
        // knight families: sheared copy + words (k_shear), the sweep over its
        // rows / columns, the far-partner searches of its queue region; each
        // family on its own stream (one family is about one wave of units:
        // run alone, its tail would idle the GPU), joined back into s
        if (!c->shear.empty()) CK(cudaEventRecord(c->sh_fork, s));
        for (size_t q = 0; q < c->shear.size(); ++q) {
            const auto &sf = c->shear[q];
            cudaStream_t ss = sf.st;
            CK(cudaStreamWaitEvent(ss, c->sh_fork, 0));
            ProfScope ps2(c, OCC_KERNEL_LINE, ss);
            const FamilyDesc &fd = c->fams[(size_t)sf.fam];
            uint32_t *cnt = c->d_gq_count + 1 + q;
            HardEntry *gq = c->d_gq + sf.q0;
            CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), ss));
            CK(launch_shear(Dc, c->H, c->W, n, sf.sd, sf.Hs, sf.Ws, fd.b0x, fd.b0y, c->params.e2_thresh, sf.d_D,
                            sf.d_W, ss));
            CK(launch_sweep(sf.d_D, sf.Hs, sf.Ws, n, sf.d_units, (int32_t)sf.units.size(), c->d_groups, c->d_views,
                            c->V, c->d_fams, c->d_stats + c0, c->params, Mc, c->mf, sf.d_W, gq, cnt, sf.qcap,
                            sf.kstart, sf.fgroup, c->d_dbg, sf.smin, &sf.sd, ss));
            ps2.end();
            ProfScope ph2(c, OCC_KERNEL_HARD, ss);
            CK(launch_hard(sf.d_D, Mc, c->mf, sf.Ws, (int64_t)sf.Hs * sf.Ws, n, c->V, c->d_views, c->params, gq, cnt,
                           sf.qcap, c->d_stats + c0, c->nsm, ss, &sf.sd));
            ph2.end();
            CK(cudaEventRecord(sf.done, ss));
            launches += 4;       // k_shear, k_sweep, k_sweep_small, k_hard
        }
        if (!c->sunits.empty()) {
            // (profile scopes of one kind must not nest: the knight scopes above are closed)
            ProfScope pl(c, OCC_KERNEL_LINE, s);
            CK(launch_sweep(Dc, c->H, c->W, n, c->d_sunits, (int32_t)c->sunits.size(), c->d_groups, c->d_views, c->V,
                            c->d_fams, c->d_stats + c0, c->params, Mc, c->mf, words, gqm, gqc,
                            qcap, c->skstart, c->sfgroup, c->d_dbg, c->ssmin, nullptr, s));
            if (swept) CK(cudaEventRecord(swept, s));
            pl.end();
            ProfScope ph(c, OCC_KERNEL_HARD, s);
            CK(launch_hard(Dc, Mc, c->mf, c->W, HW, n, c->V, c->d_views, c->params, gqm, gqc,
                           qcap, c->d_stats + c0, c->nsm, s));
            launches += 3;       // k_sweep, k_sweep_small, k_hard
            ph.end();
        }
        for (const auto &sf : c->shear) CK(cudaStreamWaitEvent(s, sf.done, 0));
    } else if (!tiled_only && !c->units.empty()) {
        ProfScope pl(c, OCC_KERNEL_LINE, s);
        CK(cudaMemsetAsync(c->d_gq_count, 0, sizeof(uint32_t), s));
#ifdef OCC_CHECKS
        CK(cudaMemsetAsync(c->d_gq, 0xFF, sizeof(HardEntry) * (size_t)c->gq_cap, s));
#endif
        if (c->d_cand) {
            CK(launch_cand(Dc, c->H, c->W, n, c->d_codes, c->code_bytes, c->d_candfam, c->nfam,
                           c->cand_per_frame, c->d_cand, s));
            ++launches;
        }
        CK(launch_line(Dc, c->H, c->W, n, c->d_units, (int32_t)c->units.size(), c->d_groups,
                       c->d_views, c->V, c->d_fams, c->d_stats + c0, c->params, Mc, c->mf, c->d_codes,
                       c->code_bytes, c->d_dbg, c->d_gq, c->d_gq_count, c->gq_cap, c->d_cand, c->d_candfam, s));
        CK(launch_hard(Dc, Mc, c->mf, c->W, HW, n, c->V, c->d_views, c->params, c->d_gq, c->d_gq_count,
                       c->gq_cap, c->d_stats + c0, c->nsm, s));
        launches += 2;
        pl.end();
    }
    if (nt > 0) {
        ProfScope pt(c, OCC_KERNEL_TILE, s);
        CK(launch_tile(Dc, c->H, c->W, n, tl, nt, c->d_groups, c->d_views, c->V, c->d_fams,
                       c->d_stats + c0, c->params, Mc, c->mf, c->d_codes, c->code_bytes, s)); ++launches;
        pt.end();
    }
    return OCC_OK;
}
}  // namespace

extern "C" {

int occ_detect(occ_ctx *c, const float *D, uint8_t *M, int32_t batch, void *stream) {
    if (!c || !D || !M || batch < 1 || batch > c->max_batch) return OCC_ERR_INVALID_ARG;
    const int64_t HW = (int64_t)c->H * c->W;
    {   // masks must not alias the input
        const char *d0 = (const char *)D, *d1 = d0 + (size_t)batch * HW * sizeof(float);
        const char *m0 = (const char *)M, *m1 = m0 + (size_t)batch * c->V * c->mf.vbytes;
        if (m0 < d1 && d0 < m1) return OCC_ERR_INVALID_ARG;
    }
    CK(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    if (c->mf.packed || c->neighbors > 0 || c->angles)   // packed / finite N / directions: kernels set marks only
        CK(cudaMemsetAsync(M, 0, (size_t)batch * c->V * c->mf.vbytes, s));
    {
        ProfScope ps(c, OCC_KERNEL_INIT, s);
        CK(launch_stats_init(c->d_stats, batch, s)); ++launches;
        ps.end();
    }
    // tiny calls (C1-sized: a few thousand pixel-views) are latency bound:
    // one thread per pixel-view beats a handful of line-sweep warps
    const bool tiny = c->path == OCC_PATH_AUTO && (int64_t)batch * HW * c->V <= kTinyPixelViews;
    if ((c->path == OCC_PATH_DIRECT || tiny) && c->neighbors == 0 && !c->angles) {
        {
            ProfScope ps(c, OCC_KERNEL_STATS, s);
            CK(launch_stats(D, HW, batch, c->d_stats, s)); ++launches;
            if (c->n_override > 0)
                CK(cudaMemcpyAsync(c->d_stats, c->d_override, sizeof(FrameStats) * (size_t)std::min(batch, c->n_override),
                                   cudaMemcpyDeviceToDevice, s));
            ps.end();
        }
        ProfScope pd(c, OCC_KERNEL_DIRECT, s);
        CK(launch_direct(D, c->H, c->W, batch, c->d_views, c->V, c->d_fams, c->d_stats,
                         c->params, M, c->mf, s)); ++launches;
        pd.end();
    } else {
        // chunks of ~256 MiB of D + codes: enough warps per K1 launch to fill
        // the GPU (the long-tailed per-unit times average out); K1's re-reads
        // of D mostly hit L2, the rest is a small fraction of the HBM bandwidth
        // several chunks of a sweep-only call: odd chunks on a second stream
        // (own words buffer and queue half), so one chunk's sweep overlaps
        // the other's k_hard and tail; joined back into s
#ifdef OCC_CHECKS
        const bool alt_on = false;        // (the checks poison the whole queue per chunk)
#else
        // opt-in (OCC_ALT=1): C5 18.82 vs 18.90 ms per step (A/B on one B200),
        // but the overlapping launches blur the per-kernel event times
        static const bool alt_on = [] { const char *ev = getenv("OCC_ALT"); return ev && atoi(ev) != 0; }();
#endif
        const bool alt = alt_on && batch > c->chunk && c->d_words2 && c->tiles.empty() && c->path == OCC_PATH_AUTO &&
                         c->neighbors == 0 && !c->angles && !c->sunits.empty();
        if (alt) {
            if (!c->s_alt) {
                CK(cudaStreamCreateWithFlags(&c->s_alt, cudaStreamNonBlocking));
                CK(cudaEventCreateWithFlags(&c->ev_alt_fork, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&c->ev_alt_join, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&c->ev_swept[0], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&c->ev_swept[1], cudaEventDisableTiming));
            }
            CK(cudaEventRecord(c->ev_alt_fork, s));
            CK(cudaStreamWaitEvent(c->s_alt, c->ev_alt_fork, 0));
        }
        int32_t ci = 0;
        for (int32_t c0 = 0; c0 < batch; c0 += c->chunk, ++ci) {
            const bool odd = alt && (ci & 1);
            cudaStream_t cs = odd ? c->s_alt : s;
            // a chunk starts once the previous chunk's sweep is done (two sweeps
            // at once would share L2): it overlaps that chunk's k_hard
            if (alt && ci > 0) CK(cudaStreamWaitEvent(cs, c->ev_swept[(ci - 1) & 1], 0));
            const int rc = detect_chunk(c, D, M, c0, std::min(c->chunk, batch - c0), cs, launches,
                                        alt ? (ci & 1) : -1, alt ? c->ev_swept[ci & 1] : nullptr);
            if (rc != OCC_OK) return rc;
        }
        if (alt) {
            CK(cudaEventRecord(c->ev_alt_join, c->s_alt));
            CK(cudaStreamWaitEvent(s, c->ev_alt_join, 0));
        }
    }
    c->last_stream = s;
    c->last_batch = batch;
    c->last_launches = launches;
    return OCC_OK;
}

// Host-buffer entry point, pipelined per chunk of frames: the H2D copy of
// chunk i + 1 and the D2H copy of chunk i - 1 run on their own streams while
// chunk i is detected on the caller's stream (copy engines overlap the kernels).
int occ_detect_host(occ_ctx *c, const float *Dh, uint8_t *Mh, int32_t batch, void *stream) {
    if (!c || !Dh || !Mh || batch < 1 || batch > c->max_batch) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    const size_t HW = (size_t)c->H * c->W;
    if (!c->d_stage_D) {
        // masks in either format: uint8 H*W or packed H*ceil(W/32)*4 bytes per plane
        const size_t plane = std::max(HW, (size_t)c->H * (size_t)((c->W + 31) / 32) * 4);
        if (cudaMalloc(&c->d_stage_D, (size_t)c->max_batch * HW * sizeof(float)) != cudaSuccess ||
            cudaMalloc(&c->d_stage_M, (size_t)c->max_batch * c->V * plane) != cudaSuccess) {
            cudaGetLastError();
            return OCC_ERR_OOM;
        }
    }
    if (!c->s_h2d) {
        CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    }
    cudaStream_t s = (cudaStream_t)stream;
    // pipeline granularity: MiB of D per copy (finer than the device-side
    // chunk, so the first H2D and the last D2H expose little of the step)
    // measured at C5 (e2e ms/step for 32/64/128/256 MiB): packed masks
    // 56.3/51.5/50.0/51.4 (H2D bound: larger copies, less exposed
    // start-up); uint8 masks 82.8/83.8/86.4/91.6 (D2H bound: finer copies)
    static const int pipe_env = [] {                       // tuning knob, read once
        const char *ev = getenv("OCC_PIPE_MIB");
        return ev ? std::max(1, atoi(ev)) : -1;
    }();
    const int pipe_mib = pipe_env > 0 ? pipe_env : (c->mf.packed ? 128 : 32);
    const int32_t pipe = (int32_t)std::max<int64_t>(1, ((int64_t)pipe_mib << 20) / (int64_t)(HW * sizeof(float)));
    const bool direct = c->path == OCC_PATH_DIRECT && c->neighbors == 0 && !c->angles;
    const int32_t chunk = direct ? batch : std::min(c->chunk, pipe);
    // chunk boundaries: full chunks, then the last chunk's worth of frames in
    // quarter pieces, so that less detection and download trails the final
    // upload (the pipeline is upload bound)
    std::vector<int32_t> starts;
    {
        int32_t c0 = 0;
        while (batch - c0 > chunk) { starts.push_back(c0); c0 += chunk; }
        const int32_t piece = direct ? batch : std::max(1, (chunk + 3) / 4);
        while (c0 < batch) { starts.push_back(c0); c0 += std::min(piece, batch - c0); }
        starts.push_back(batch);
    }
    const int32_t nchunks = (int32_t)starts.size() - 1;
    while ((int32_t)c->ev_pipe.size() < 2 * nchunks + 1) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ev_pipe.push_back(e);
    }
    // the copies must not start before the caller's earlier work on s
    CK(cudaEventRecord(c->ev_pipe[2 * nchunks], s));
    CK(cudaStreamWaitEvent(c->s_h2d, c->ev_pipe[2 * nchunks], 0));
    CK(cudaStreamWaitEvent(c->s_d2h, c->ev_pipe[2 * nchunks], 0));
    int launches = 0;
    {
        ProfScope ps(c, OCC_KERNEL_INIT, s);
        CK(launch_stats_init(c->d_stats, batch, s)); ++launches;
        ps.end();
    }
    if ((c->mf.packed || c->neighbors > 0 || c->angles) && !direct)
        CK(cudaMemsetAsync(c->d_stage_M, 0, (size_t)batch * c->V * c->mf.vbytes, s));
    for (int32_t i = 0; i < nchunks; ++i) {
        const int32_t c0 = starts[(size_t)i], n = starts[(size_t)i + 1] - c0;
        CK(cudaMemcpyAsync(c->d_stage_D + (size_t)c0 * HW, Dh + (size_t)c0 * HW, (size_t)n * HW * sizeof(float),
                           cudaMemcpyHostToDevice, c->s_h2d));
        CK(cudaEventRecord(c->ev_pipe[2 * i], c->s_h2d));
        CK(cudaStreamWaitEvent(s, c->ev_pipe[2 * i], 0));
        if (direct) {
            int rc = occ_detect(c, c->d_stage_D, c->d_stage_M, batch, stream);
            if (rc != OCC_OK) return rc;
            launches += c->last_launches;
        } else {
            const int rc = detect_chunk(c, c->d_stage_D, c->d_stage_M, c0, n, s, launches);
            if (rc != OCC_OK) return rc;
        }
        CK(cudaEventRecord(c->ev_pipe[2 * i + 1], s));
        CK(cudaStreamWaitEvent(c->s_d2h, c->ev_pipe[2 * i + 1], 0));
        CK(cudaMemcpyAsync(Mh + (size_t)c0 * c->V * c->mf.vbytes, c->d_stage_M + (size_t)c0 * c->V * c->mf.vbytes,
                           (size_t)n * c->V * c->mf.vbytes, cudaMemcpyDeviceToHost, c->s_d2h));
    }
    CK(cudaStreamSynchronize(c->s_d2h));
    CK(cudaStreamSynchronize(s));
    c->last_stream = s;
    c->last_batch = batch;
    c->last_launches = launches;
    return OCC_OK;
}

int occ_status(occ_ctx *c, int32_t *frame_status) {
    if (!c || !frame_status) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->last_stream));
    std::vector<FrameStats> st((size_t)c->last_batch);
    if (c->last_batch > 0)
        CK(cudaMemcpy(st.data(), c->d_stats, sizeof(FrameStats) * st.size(), cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < c->last_batch; ++i)
        frame_status[i] = st[(size_t)i].nonfinite ? OCC_ERR_NONFINITE : OCC_OK;
    return OCC_OK;
}

int occ_frame_info(occ_ctx *c, int32_t frame, float *dmin, float *dmax, int32_t *h_per_view) {
    if (!c || frame < 0 || frame >= c->last_batch) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->last_stream));
    FrameStats fs;
    CK(cudaMemcpy(&fs, c->d_stats + frame, sizeof(fs), cudaMemcpyDeviceToHost));
    const float lo = key_float(fs.minkey), hi = key_float(fs.maxkey);
    if (dmin) *dmin = lo;
    if (dmax) *dmax = hi;
    if (h_per_view) {
        const float R = hi - lo;
        for (int32_t v = 0; v < c->V; ++v) {
            double L = std::ceil((2.0 * c->views[v].rho) * (double)R);
            if (!(L <= (double)c->params.max_scan)) L = c->params.max_scan;
            h_per_view[v] = fs.nonfinite ? 0 : ((int32_t)L) / 2;
        }
    }
    return OCC_OK;
}

int occ_scan_half_lengths(const occ_ctx *c, float dmin, float dmax, int32_t *h_per_view) {
    if (!c || !h_per_view) return OCC_ERR_INVALID_ARG;
    const float R = dmax - dmin;            // fl32 (host SSE, no contraction)
    for (int32_t v = 0; v < c->V; ++v) {
        double L = std::ceil((2.0 * c->views[v].rho) * (double)R);
        if (!(L <= (double)c->params.max_scan)) L = c->params.max_scan;
        h_per_view[v] = ((int32_t)L) / 2;
    }
    return OCC_OK;
}

int occ_profile(occ_ctx *c, int32_t enable) {
    if (!c) return OCC_ERR_INVALID_ARG;
    c->profiling = enable != 0;
    for (int k = 0; k < OCC_KERNEL_KINDS; ++k) c->ev_used[k] = 0;
    return OCC_OK;
}

int occ_profile_read(occ_ctx *c, int32_t kind, double *total_ms, int32_t *launches) {
    if (!c || kind < 0 || kind >= OCC_KERNEL_KINDS) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    double tot = 0.0;
    const size_t n = c->ev_used[kind];
    for (size_t i = 0; i + 1 < n; i += 2) {
        CK(cudaEventSynchronize(c->ev[kind][i + 1]));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, c->ev[kind][i], c->ev[kind][i + 1]));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = (int32_t)(n / 2);
    return OCC_OK;
}

// Debug statistics of the line-sweep kernel (not part of include/occ.h):
// enable != 0 allocates/zeroes 16 counters that subsequent occ_detect calls
// accumulate, plus per-CTA cycle counts of the last launch (entries 16..);
// out (host, 16 + 65536 entries, may be NULL) receives the current values.
int occ_debug_line_stats(occ_ctx *c, int32_t enable, unsigned long long *out) {
    if (!c) return OCC_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    if (out) {
        if (c->d_dbg) {
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(out, c->d_dbg, (16 + 65536 + 4 * 32768) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        } else {
            memset(out, 0, (16 + 65536 + 4 * 32768) * sizeof(unsigned long long));
        }
    }
    if (enable) {
        if (!c->d_dbg) CK(cudaMalloc(&c->d_dbg, (16 + 65536 + 4 * 32768) * sizeof(unsigned long long)));
        CK(cudaMemset(c->d_dbg, 0, (16 + 65536 + 4 * 32768) * sizeof(unsigned long long)));
    } else if (c->d_dbg) {
        CK(cudaFree(c->d_dbg));
        c->d_dbg = nullptr;
    }
    return OCC_OK;
}

int occ_fuse_median(const float *stack, int32_t K, int64_t n, float *out, void *stream) {
    if (!stack || !out || K < 1 || K > kFuseMaxK || n < 1) return OCC_ERR_INVALID_ARG;
    {
        const char *s0 = (const char *)stack, *s1 = s0 + (size_t)K * (size_t)n * sizeof(float);
        const char *o0 = (const char *)out, *o1 = o0 + (size_t)n * sizeof(float);
        if (o0 < s1 && s0 < o1) return OCC_ERR_INVALID_ARG;
    }
    int dev = 0, nsm = 148;
    CK(cudaGetDevice(&dev));
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) nsm = 148;
    CK(launch_fuse_median(stack, K, n, out, nsm, (cudaStream_t)stream));
    return OCC_OK;
}

int occ_destroy(occ_ctx *c) {
    if (!c) return OCC_ERR_INVALID_ARG;
    cudaSetDevice(c->device);
    if (c->last_stream || c->last_batch) cudaStreamSynchronize(c->last_stream);
    cudaFree(c->d_views);
    cudaFree(c->d_fams);
    cudaFree(c->d_stats);
    cudaFree(c->d_codes);
    cudaFree(c->d_groups);
    cudaFree(c->d_tiles);
    cudaFree(c->d_all_tiles);
    cudaFree(c->d_units);
    cudaFree(c->d_sunits);
    cudaFree(c->d_words);
    cudaFree(c->d_words2);
    if (c->s_alt) cudaStreamDestroy(c->s_alt);
    if (c->ev_alt_fork) cudaEventDestroy(c->ev_alt_fork);
    if (c->ev_alt_join) cudaEventDestroy(c->ev_alt_join);
    for (cudaEvent_t e : c->ev_swept) if (e) cudaEventDestroy(e);
    for (auto &sf : c->shear) {
        cudaFree(sf.d_units);
        cudaFree(sf.d_D);
        cudaFree(sf.d_W);
        if (sf.st) cudaStreamDestroy(sf.st);
        if (sf.done) cudaEventDestroy(sf.done);
    }
    if (c->sh_fork) cudaEventDestroy(c->sh_fork);
    cudaFree(c->d_dbg);
    cudaFree(c->d_gq);
    cudaFree(c->d_gq_count);
    cudaFree(c->d_nwin_work);
    cudaFree(c->d_override);
    cudaFree(c->d_offs);
    cudaFree(c->d_cand);
    cudaFree(c->d_candfam);
    cudaFree(c->nwin_big.buf);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (cudaEvent_t e : c->ev_pipe) cudaEventDestroy(e);
    cudaFree(c->d_stage_D);
    cudaFree(c->d_stage_M);
    for (int k = 0; k < OCC_KERNEL_KINDS; ++k)
        for (cudaEvent_t e : c->ev[k]) cudaEventDestroy(e);
    delete c;
    return OCC_OK;
}

}  // extern "C"
