/*
 * pch_oracle.c -- CPU restatement of the reference PCH / ICH engines.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path (paper_1305_1293_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it; the product never links or calls it.
 *
 * It restates, in plain C, the algorithm of the reference package
 * (/root/reference/pkg/src/pargeo, Python + numba):
 *   geom.py:73   _unfold              -> o_unfold
 *   geom.py:93   _window_key          -> o_window_key
 *   geom.py:106  _ray_seg_param       -> o_ray_seg
 *   geom.py:125  _emit_child          -> o_emit_child
 *   geom.py:185  _emit_fan            -> o_emit_fan
 *   geom.py:312  _propagate_window    -> o_propagate
 *   engine.py:402 _source_rows        -> o_source_rows
 *   engine.py:235 select_nearest      -> o_select
 *   engine.py:201 dedupe_rows         -> o_dedupe
 *   engine.py:341 apply_distance_events / :359 apply_angle_events
 *   engine.py:433 run_pch             -> pch_oracle_run_pch
 *   engine.py:533 _ich_run / :624 run_ich -> pch_oracle_run_ich
 * Window rows keep the reference layout (he, b0, b1, d0, d1, d, key) so
 * the restatement can be read side by side with the reference.
 *
 * Parity pinning: tests/golden/ (npz files) hold distance fields and window
 * counts produced by the reference itself (tests/golden/make_golden.py);
 * tests/test_oracle_golden.py checks this file against them.
 *
 * Build: see oracle/Makefile (gcc -O2 -pthread -ffp-contract=off).
 * Workers run on a persistent pthread pool (the reference uses numba prange).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define W_HE 0
#define W_B0 1
#define W_B1 2
#define W_D0 3
#define W_D1 4
#define W_D 5
#define W_KEY 6
#define WIN_COLS 7
#define AE_COMP 7
#define AE_ENTRYX 8
#define AEV_COLS 9

enum { C_PROPAGATED, C_CREATED, C_PRUNE_ICH, C_PRUNE_SPLIT, C_PRUNE_TINY,
       C_PRUNE_DEGEN, C_MAXCHILD, C_EV_CREATED, C_EV_APPLIED, N_COUNTERS };

#define SADDLE 2
#define MAXVAL 256
static const double TWO_PI = 6.283185307179586;
static const double PI_ = 3.141592653589793;

typedef struct {
    const int64_t *origin, *opposite;
    const double *length, *corner;
    const uint8_t *vclass;
    int64_t nv, nhe;
} omesh;

/* growable row buffer */
typedef struct { double *p; int64_t n, cap, cols; } rows_t;

static int rows_reserve(rows_t *r, int64_t want) {
    if (want <= r->cap) return 0;
    int64_t c = r->cap ? r->cap : 64;
    while (c < want) c *= 2;
    double *q = (double *)realloc(r->p, (size_t)c * r->cols * sizeof(double));
    if (!q) return -1;
    r->p = q; r->cap = c;
    return 0;
}
static double *rows_push(rows_t *r) {
    if (rows_reserve(r, r->n + 1)) return NULL;
    return r->p + (r->n++) * r->cols;
}
static void rows_free(rows_t *r) { free(r->p); r->p = NULL; r->n = r->cap = 0; }

static inline int64_t nxt(int64_t j) { return 3 * (j / 3) + (j + 1) % 3; }
static inline int64_t prv(int64_t j) { return 3 * (j / 3) + (j + 2) % 3; }

/* geom.py:73 */
static int o_unfold(double b0, double b1, double d0, double d1, double eps_num,
                    double *x, double *y) {
    double w = b1 - b0;
    *x = 0.0; *y = 0.0;
    if (w <= 0.0) return 0;
    *x = b0 + 0.5 * (w * w + d0 * d0 - d1 * d1) / w;
    double dx = *x - b0;
    double h2 = d0 * d0 - dx * dx;
    double scale = d0 * d0 > w * w ? d0 * d0 : w * w;
    if (h2 < -eps_num * (scale > 1e-30 ? scale : 1e-30)) return 0;
    *y = h2 > 0.0 ? sqrt(h2) : 0.0;
    return 1;
}

/* geom.py:93 */
static double o_window_key(double b0, double b1, double d0, double d1,
                           double dps, double eps_num) {
    double x, y;
    if (!o_unfold(b0, b1, d0, d1, eps_num, &x, &y)) return -1.0;
    if (x < b0 || x > b1) return dps + (d0 < d1 ? d0 : d1);
    return dps + y;
}

/* geom.py:106 */
static int o_ray_seg(double ix, double iy, double tx, double ty, double px,
                     double py, double qx, double qy, double *s) {
    double rx = tx - ix, ry = ty - iy, ex = qx - px, ey = qy - py;
    double den = rx * ey - ry * ex;
    *s = 0.0;
    if (fabs(den) < 1e-300) return 0;
    double t = ((px - ix) * ry - (py - iy) * rx) / den;
    if (t < 0.0) t = 0.0; else if (t > 1.0) t = 1.0;
    *s = t;
    return 1;
}

/* geom.py:125 -- returns 1 if stored, 0 if filtered, -1 on alloc failure */
static int o_emit_child(int64_t che, double lc, double sx, double sy, double ex,
                        double ey, double s0, double s1, double ix, double iy,
                        double dps, double g_s, double g_e, double g_r,
                        double rx, double ry, int r_pairs_low, double eps_win,
                        double eps_num, rows_t *out, int64_t *cnt) {
    cnt[C_CREATED]++;
    double cb0 = s0 * lc, cb1 = s1 * lc;
    if (cb1 - cb0 <= eps_win) { cnt[C_PRUNE_TINY]++; return 0; }
    double p0x = sx + s0 * (ex - sx), p0y = sy + s0 * (ey - sy);
    double p1x = sx + s1 * (ex - sx), p1y = sy + s1 * (ey - sy);
    double cd0 = hypot(ix - p0x, iy - p0y);
    double cd1 = hypot(ix - p1x, iy - p1y);
    double t0 = dps + cd0, t1 = dps + cd1;
    if (g_s < INFINITY && t1 > g_s + hypot(sx - p1x, sy - p1y) + eps_num) {
        cnt[C_PRUNE_ICH]++; return 0;
    }
    if (g_e < INFINITY && t0 > g_e + hypot(ex - p0x, ey - p0y) + eps_num) {
        cnt[C_PRUNE_ICH]++; return 0;
    }
    if (g_r < INFINITY) {
        if (r_pairs_low) {
            if (t0 > g_r + hypot(rx - p0x, ry - p0y) + eps_num) { cnt[C_PRUNE_ICH]++; return 0; }
        } else {
            if (t1 > g_r + hypot(rx - p1x, ry - p1y) + eps_num) { cnt[C_PRUNE_ICH]++; return 0; }
        }
    }
    double key = o_window_key(cb0, cb1, cd0, cd1, dps, eps_num);
    if (key < 0.0) { cnt[C_PRUNE_DEGEN]++; return 0; }
    double *r = rows_push(out);
    if (!r) return -1;
    r[W_HE] = (double)che; r[W_B0] = cb0; r[W_B1] = cb1; r[W_D0] = cd0;
    r[W_D1] = cd1; r[W_D] = dps; r[W_KEY] = key;
    return 1;
}

/* geom.py:185 -- windows sourced at v over its fan; returns stored count
 * or -1 on allocation failure */
static int64_t o_emit_fan(const omesh *m, int64_t v, double dist_v,
                          int64_t h_anchor, double rel_r, int full_fan,
                          const double *gd, double eps_win, double eps_num,
                          int fan_full_edges, rows_t *out, int64_t *cnt) {
    (void)v;
    int64_t start = h_anchor;
    int interior = 0;
    for (int guard = 0; guard < 4 * MAXVAL; ++guard) {
        int64_t ho = m->opposite[start];
        if (ho < 0) break;
        int64_t hcw = nxt(ho);
        if (hcw == h_anchor) { interior = 1; start = h_anchor; break; }
        start = hcw;
    }
    int64_t hs[MAXVAL];
    double phis[MAXVAL + 1];
    int m_ = 0;
    double phi = 0.0, anchor_phi = 0.0;
    int64_t h = start;
    while (m_ < MAXVAL) {
        hs[m_] = h;
        phis[m_] = phi;
        if (h == h_anchor) anchor_phi = phi;
        phi += m->corner[h];
        m_++;
        int64_t ho = m->opposite[prv(h)];
        if (ho < 0) break;
        h = ho;
        if (h == start) break;
    }
    phis[m_] = phi;
    double theta = phi, flo, fhi;
    int reps;
    if (full_fan) {
        flo = -1.0e300; fhi = 1.0e300; reps = 1;
    } else {
        double width = theta - TWO_PI;
        if (width <= eps_num) return 0;
        flo = anchor_phi + rel_r + PI_;
        fhi = flo + width;
        if (interior) {
            double k = floor(flo / theta);
            flo -= k * theta; fhi -= k * theta;
            reps = 2;
        } else {
            reps = 1;
        }
    }
    int64_t stored = 0;
    for (int i = 0; i < m_; ++i) {
        double wlo = phis[i], whi = phis[i + 1];
        int64_t hgi = hs[i], che = nxt(hgi), hprev = prv(hgi);
        double li = m->length[hgi], lq = m->length[hprev], lc = m->length[che];
        int64_t pid = m->origin[che], qid = m->origin[hprev];
        for (int rep = 0; rep < reps; ++rep) {
            double lo = flo - rep * theta, hi = fhi - rep * theta;
            double slo = wlo > lo ? wlo : lo;
            double shi = whi < hi ? whi : hi;
            if (shi - slo <= 1e-12) continue;
            if (fan_full_edges) { slo = wlo; shi = whi; }
            double px = li * cos(wlo), py = li * sin(wlo);
            double qx = lq * cos(whi), qy = lq * sin(whi);
            double s0, s1;
            int ok0 = 1, ok1 = 1;
            if (slo <= wlo + 1e-12) s0 = 0.0;
            else ok0 = o_ray_seg(0.0, 0.0, cos(slo), sin(slo), px, py, qx, qy, &s0);
            if (shi >= whi - 1e-12) s1 = 1.0;
            else ok1 = o_ray_seg(0.0, 0.0, cos(shi), sin(shi), px, py, qx, qy, &s1);
            if (!(ok0 && ok1)) { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; continue; }
            int add = o_emit_child(che, lc, px, py, qx, qy, s0, s1, 0.0, 0.0,
                                   dist_v, gd[pid], gd[qid], INFINITY, 0.0, 0.0,
                                   1, eps_win, eps_num, out, cnt);
            if (add < 0) return -1;
            stored += add;
        }
    }
    return stored;
}

/* geom.py:312 -- one window propagation; returns 0 ok, -1 alloc failure */
static int o_propagate(const double *row, const omesh *m, const double *gd,
                       const double *split_comp, const double *split_entryx,
                       double eps_win, double eps_num, int fan_full,
                       rows_t *ow, rows_t *od, rows_t *oa, int64_t *cnt) {
    cnt[C_PROPAGATED]++;
    int64_t j = (int64_t)row[W_HE];
    double b0 = row[W_B0], b1 = row[W_B1], d0 = row[W_D0], d1 = row[W_D1];
    double dps = row[W_D];
    double ell = m->length[j];
    double ix, iy;
    if (!o_unfold(b0, b1, d0, d1, eps_num, &ix, &iy)) { cnt[C_PRUNE_DEGEN]++; return 0; }
    int64_t stored = 0, add;
    int64_t jn = nxt(j), jp = prv(j);
    int64_t v0 = m->origin[j], v1 = m->origin[jn];

    if (b0 <= eps_win) {
        double cand = dps + d0 + b0;
        if (cand < gd[v0]) {
            double *e = rows_push(od); if (!e) return -1;
            e[0] = (double)v0; e[1] = cand;
            if (m->vclass[v0] == SADDLE) {
                double rel = atan2(iy, ix);
                add = o_emit_fan(m, v0, cand, j, rel, 0, gd, eps_win, eps_num, fan_full, ow, cnt);
                if (add < 0) return -1;
                stored += add;
            }
        }
    }
    if (b1 >= ell - eps_win) {
        double cand = dps + d1 + (ell - b1);
        if (cand < gd[v1]) {
            double *e = rows_push(od); if (!e) return -1;
            e[0] = (double)v1; e[1] = cand;
            if (m->vclass[v1] == SADDLE) {
                double lps = m->length[jp], lns = m->length[jn];
                double axs = 0.5 * (ell * ell + lps * lps - lns * lns) / ell;
                double ay2 = lps * lps - axs * axs;
                double ays = ay2 > 0.0 ? sqrt(ay2) : 0.0;
                double adir = atan2(ays, axs - ell);
                double rel = atan2(iy, ix - ell) - adir;
                add = o_emit_fan(m, v1, cand, jn, rel, 0, gd, eps_win, eps_num, fan_full, ow, cnt);
                if (add < 0) return -1;
                stored += add;
            }
        }
    }

    int64_t jo = m->opposite[j];
    if (jo >= 0) {
        int64_t jno = nxt(jo), jpo = prv(jo);
        double lan = m->length[jno], lpv = m->length[jpo];
        double dx = 0.5 * (ell * ell + lan * lan - lpv * lpv) / ell;
        double dy2 = lan * lan - dx * dx;
        double dy = dy2 > 0.0 ? -sqrt(dy2) : 0.0;
        int64_t vd = m->origin[jpo];
        double uax = b0 - ix, uay = -iy, ubx = b1 - ix, uby = -iy;
        double vdx = dx - ix, vdy = dy - iy;
        double nvd = hypot(vdx, vdy);
        double ca = uax * vdy - uay * vdx;
        double cb = ubx * vdy - uby * vdx;
        double tola = eps_num * hypot(uax, uay) * nvd;
        double tolb = eps_num * hypot(ubx, uby) * nvd;
        double g0 = gd[v0], g1 = gd[v1], gdd = gd[vd];
        double sa, sb;
        int oka, okb;
        if (ca > tola && cb < -tolb) {
            double comp = dps + nvd;
            double denom = iy - dy;
            double entry_x = denom > 1e-300 ? ix + (dx - ix) * (iy / denom) : ix;
            int want_left = 1, want_right = 1;
            if (comp < split_comp[j]) {
                double *a = rows_push(oa); if (!a) return -1;
                for (int c = 0; c < WIN_COLS; ++c) a[c] = row[c];
                a[AE_COMP] = comp; a[AE_ENTRYX] = entry_x;
            } else {
                cnt[C_PRUNE_SPLIT]++; cnt[C_CREATED]++;
                if (entry_x < split_entryx[j]) want_right = 0; else want_left = 0;
            }
            if (want_left) {
                oka = o_ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, &sa);
                if (oka) {
                    add = o_emit_child(jno, lan, 0.0, 0.0, dx, dy, sa, 1.0, ix, iy, dps,
                                       g0, gdd, g1, ell, 0.0, 1, eps_win, eps_num, ow, cnt);
                    if (add < 0) return -1;
                    stored += add;
                } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
            }
            if (want_right) {
                okb = o_ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, &sb);
                if (okb) {
                    add = o_emit_child(jpo, lpv, dx, dy, ell, 0.0, 0.0, sb, ix, iy, dps,
                                       gdd, g1, g0, 0.0, 0.0, 0, eps_win, eps_num, ow, cnt);
                    if (add < 0) return -1;
                    stored += add;
                } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
            }
            double cand = dps + nvd;
            if (cand < gdd) {
                double *e = rows_push(od); if (!e) return -1;
                e[0] = (double)vd; e[1] = cand;
                if (m->vclass[vd] == SADDLE) {
                    double gamma = atan2(-dy, ell - dx);
                    double rel = atan2(iy - dy, ix - dx) - gamma;
                    add = o_emit_fan(m, vd, cand, jpo, rel, 0, gd, eps_win, eps_num, fan_full, ow, cnt);
                    if (add < 0) return -1;
                    stored += add;
                }
            }
        } else if (cb >= -tolb) {
            oka = o_ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, &sa);
            okb = o_ray_seg(ix, iy, b1, 0.0, 0.0, 0.0, dx, dy, &sb);
            if (oka && okb) {
                add = o_emit_child(jno, lan, 0.0, 0.0, dx, dy, sa, sb, ix, iy, dps,
                                   g0, gdd, g1, ell, 0.0, 1, eps_win, eps_num, ow, cnt);
                if (add < 0) return -1;
                stored += add;
            } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
        } else {
            oka = o_ray_seg(ix, iy, b0, 0.0, dx, dy, ell, 0.0, &sa);
            okb = o_ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, &sb);
            if (oka && okb) {
                add = o_emit_child(jpo, lpv, dx, dy, ell, 0.0, sa, sb, ix, iy, dps,
                                   gdd, g1, g0, 0.0, 0.0, 0, eps_win, eps_num, ow, cnt);
                if (add < 0) return -1;
                stored += add;
            } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
        }
    }
    if (stored > cnt[C_MAXCHILD]) cnt[C_MAXCHILD] = stored;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* stats block shared with the Python wrapper (oracle/oracle.py) */
typedef struct {
    int64_t iterations, windows_propagated, total_windows_created,
        total_windows_pruned, pruned_ich, pruned_split, pruned_tiny,
        pruned_degenerate, pruned_duplicate, windows_stored,
        max_children_per_window, events_created, events_applied,
        peak_active_pool;
} ostats;

static void absorb(ostats *s, const int64_t *c) {
    s->windows_propagated += c[C_PROPAGATED];
    s->total_windows_created += c[C_CREATED];
    s->pruned_ich += c[C_PRUNE_ICH];
    s->pruned_split += c[C_PRUNE_SPLIT];
    s->pruned_tiny += c[C_PRUNE_TINY];
    s->pruned_degenerate += c[C_PRUNE_DEGEN];
    s->total_windows_pruned += c[C_PRUNE_ICH] + c[C_PRUNE_SPLIT] + c[C_PRUNE_TINY] + c[C_PRUNE_DEGEN];
    if (c[C_MAXCHILD] > s->max_children_per_window) s->max_children_per_window = c[C_MAXCHILD];
}

/* engine.py:402 -- source windows are full fans with d = 0 */
static int o_source_rows(const omesh *m, const int64_t *outgoing,
                         const int64_t *src, int64_t nsrc, const double *gd,
                         double eps_win, rows_t *out, int64_t *cnt) {
    for (int64_t i = 0; i < nsrc; ++i) {
        int64_t h = outgoing[src[i]];
        if (h < 0) continue;
        if (o_emit_fan(m, src[i], 0.0, h, 0.0, 1, gd, eps_win, 1e-12, 0, out, cnt) < 0)
            return -1;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* ICH: binary heap on (key, seq) -- engine.py:487-621 */
typedef struct { double key; int64_t seq; int64_t row; } hent;

static inline int hless(const hent *a, const hent *b) {
    if (a->key != b->key) return a->key < b->key;
    return a->seq < b->seq;
}

int pch_oracle_run_ich(const int64_t *origin, const int64_t *opposite,
                       const double *length, const double *corner,
                       const uint8_t *vclass, const int64_t *outgoing,
                       int64_t nv, int64_t nf, const int64_t *src, int64_t nsrc,
                       double eps_win, int fan_full, double *dist,
                       ostats *st) {
    const double eps_num = 1e-12;
    omesh m = {origin, opposite, length, corner, vclass, nv, 3 * nf};
    int64_t cnt[N_COUNTERS] = {0};
    memset(st, 0, sizeof(*st));
    for (int64_t v = 0; v < nv; ++v) dist[v] = INFINITY;
    for (int64_t i = 0; i < nsrc; ++i) dist[src[i]] = 0.0;
    double *scomp = (double *)malloc(sizeof(double) * 3 * nf);
    double *sentry = (double *)calloc(3 * nf, sizeof(double));
    for (int64_t i = 0; i < 3 * nf; ++i) scomp[i] = INFINITY;
    rows_t store = {0, 0, 0, WIN_COLS};   /* window rows referenced by heap */
    rows_t init = {0, 0, 0, WIN_COLS};
    int rc = 0;
    if (o_source_rows(&m, outgoing, src, nsrc, dist, eps_win, &init, cnt)) { rc = -1; goto done; }
    absorb(st, cnt);
    memset(cnt, 0, sizeof(cnt));
    st->windows_stored += init.n;

    int64_t hcap = 1024, hsize = 0, seq = 0, peak = 0;
    hent *heap = (hent *)malloc(sizeof(hent) * hcap);
    /* free-list of row slots in `store` */
    int64_t *freel = NULL; int64_t nfree = 0, freecap = 0;
    rows_t wb = {0, 0, 0, WIN_COLS}, dv = {0, 0, 0, 2}, av = {0, 0, 0, AEV_COLS};

#define HPUSH(rowsrc) do {                                                   \
        int64_t slot;                                                        \
        if (nfree) slot = freel[--nfree];                                    \
        else { if (!rows_push(&store)) { rc = -1; goto done2; } slot = store.n - 1; } \
        memcpy(store.p + slot * WIN_COLS, (rowsrc), sizeof(double) * WIN_COLS); \
        if (hsize == hcap) { hcap *= 2; heap = (hent *)realloc(heap, sizeof(hent) * hcap); } \
        int64_t i_ = hsize++;                                                \
        heap[i_].key = (rowsrc)[W_KEY]; heap[i_].seq = seq++; heap[i_].row = slot; \
        while (i_ > 0) { int64_t p_ = (i_ - 1) / 2;                          \
            if (hless(&heap[i_], &heap[p_])) { hent t_ = heap[i_]; heap[i_] = heap[p_]; heap[p_] = t_; i_ = p_; } \
            else break; }                                                    \
    } while (0)

    for (int64_t i = 0; i < init.n; ++i) HPUSH(init.p + i * WIN_COLS);
    peak = hsize;
    double row[WIN_COLS];
    while (hsize > 0) {
        int64_t slot = heap[0].row;
        memcpy(row, store.p + slot * WIN_COLS, sizeof(row));
        if (nfree == freecap) { freecap = freecap ? 2 * freecap : 1024; freel = (int64_t *)realloc(freel, sizeof(int64_t) * freecap); }
        freel[nfree++] = slot;
        hsize--;
        if (hsize > 0) {
            heap[0] = heap[hsize];
            int64_t i_ = 0;
            for (;;) {
                int64_t l = 2 * i_ + 1, r = l + 1, mm = l;
                if (l >= hsize) break;
                if (r < hsize && hless(&heap[r], &heap[l])) mm = r;
                if (hless(&heap[mm], &heap[i_])) { hent t_ = heap[i_]; heap[i_] = heap[mm]; heap[mm] = t_; i_ = mm; }
                else break;
            }
        }
        wb.n = dv.n = av.n = 0;
        if (o_propagate(row, &m, dist, scomp, sentry, eps_win, eps_num, fan_full, &wb, &dv, &av, cnt)) { rc = -1; goto done2; }
        cnt[C_EV_CREATED] += dv.n + av.n;
        for (int64_t e = 0; e < dv.n; ++e) {
            int64_t v = (int64_t)dv.p[2 * e];
            if (dv.p[2 * e + 1] < dist[v]) { dist[v] = dv.p[2 * e + 1]; cnt[C_EV_APPLIED]++; }
        }
        for (int64_t e = 0; e < av.n; ++e) {
            const double *a = av.p + e * AEV_COLS;
            int64_t he = (int64_t)a[W_HE];
            if (a[AE_COMP] < scomp[he]) { scomp[he] = a[AE_COMP]; sentry[he] = a[AE_ENTRYX]; cnt[C_EV_APPLIED]++; }
        }
        for (int64_t i = 0; i < wb.n; ++i) HPUSH(wb.p + i * WIN_COLS);
        if (hsize > peak) peak = hsize;
    }
    absorb(st, cnt);
    st->events_created = cnt[C_EV_CREATED];
    st->events_applied = cnt[C_EV_APPLIED];
    st->windows_stored += st->total_windows_created - st->total_windows_pruned;
    st->peak_active_pool = peak;
    st->iterations = st->windows_propagated;
done2:
    free(heap); free(freel); rows_free(&wb); rows_free(&dv); rows_free(&av);
#undef HPUSH
done:
    rows_free(&store); rows_free(&init); free(scomp); free(sentry);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* PCH batch engine -- engine.py:433 run_pch */

/* k-th smallest (0-based) of a[0..n) by quickselect on a scratch copy */
static double kth_smallest(double *a, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        double piv = a[lo + (hi - lo) / 2];
        int64_t i = lo, j = hi;
        while (i <= j) {
            while (a[i] < piv) i++;
            while (a[j] > piv) j--;
            if (i <= j) { double t = a[i]; a[i] = a[j]; a[j] = t; i++; j--; }
        }
        if (k <= j) hi = j; else if (k >= i) lo = i; else return a[k];
    }
    return a[k];
}

/* mark the m smallest keys among positions first, first+stride, ...;
 * ties at the m-th value are taken in position order */
static void mark_smallest(const double *active, int64_t n, int64_t first,
                          int64_t stride, int64_t m, double *scratch,
                          uint8_t *mask) {
    int64_t cnt = 0;
    for (int64_t i = first; i < n; i += stride) scratch[cnt++] = active[i * WIN_COLS + W_KEY];
    if (cnt <= m) {
        for (int64_t i = first; i < n; i += stride) mask[i] = 1;
        return;
    }
    double kth = kth_smallest(scratch, cnt, m - 1);
    int64_t below = 0;
    for (int64_t i = first; i < n; i += stride)
        if (active[i * WIN_COLS + W_KEY] < kth) { mask[i] = 1; below++; }
    for (int64_t i = first; i < n && below < m; i += stride)
        if (active[i * WIN_COLS + W_KEY] == kth) { mask[i] = 1; below++; }
}

/* hash-set dedupe of exact duplicate rows, keeping first occurrences
 * (engine.py:201) -- returns new count */
static uint64_t row_hash(const double *r) {
    uint64_t h = 1469598103934665603ull;
    for (int c = 0; c < WIN_COLS; ++c) {
        uint64_t b; memcpy(&b, &r[c], 8);
        h ^= b + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 1099511628211ull;
    }
    return h;
}
static int64_t o_dedupe(double *rows, int64_t n) {
    if (n < 2) return n;
    int64_t cap = 16;
    while (cap < 2 * n) cap *= 2;
    int64_t *tab = (int64_t *)malloc(sizeof(int64_t) * cap);
    for (int64_t i = 0; i < cap; ++i) tab[i] = -1;
    int64_t out = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double *r = rows + i * WIN_COLS;
        uint64_t h = row_hash(r) & (cap - 1);
        int dup = 0;
        while (tab[h] >= 0) {
            if (memcmp(rows + tab[h] * WIN_COLS, r, sizeof(double) * WIN_COLS) == 0) { dup = 1; break; }
            h = (h + 1) & (cap - 1);
        }
        if (dup) continue;
        if (out != i) memcpy(rows + out * WIN_COLS, r, sizeof(double) * WIN_COLS);
        tab[h] = out;
        out++;
    }
    free(tab);
    return out;
}

/* engine.py:359 lexsort order: he, key, comp, b0, b1, d0, d1, d, entry_x */
static int aev_cmp(const void *pa, const void *pb) {
    const double *a = (const double *)pa, *b = (const double *)pb;
    static const int order[] = {W_HE, W_KEY, AE_COMP, W_B0, W_B1, W_D0, W_D1, W_D, AE_ENTRYX};
    for (int i = 0; i < 9; ++i) {
        double x = a[order[i]], y = b[order[i]];
        if (x < y) return -1;
        if (x > y) return 1;
    }
    return 0;
}

/* persistent worker pool: worker w propagates selected[w*share, (w+1)*share) */
typedef struct {
    pthread_barrier_t start, done;
    int T, quit;
    const double *sel; int64_t ns, share;
    const omesh *m; const double *dist, *scomp, *sentry;
    double eps_win; int fan_full;
    rows_t *wb, *db, *ab; int64_t *wcnt; int *fail;
} wpool;

static void pool_work(wpool *p, int w) {
    p->wb[w].n = p->db[w].n = p->ab[w].n = 0;
    p->fail[w] = 0;
    int64_t lo = (int64_t)w * p->share, hi = lo + p->share;
    if (hi > p->ns) hi = p->ns;
    for (int64_t i = lo; i < hi; ++i)
        if (o_propagate(p->sel + i * WIN_COLS, p->m, p->dist, p->scomp, p->sentry,
                        p->eps_win, 1e-12, p->fan_full, &p->wb[w], &p->db[w], &p->ab[w],
                        p->wcnt + w * N_COUNTERS)) { p->fail[w] = 1; break; }
}

typedef struct { wpool *p; int w; } warg;

static void *pool_main(void *arg) {
    warg *a = (warg *)arg;
    for (;;) {
        pthread_barrier_wait(&a->p->start);
        if (a->p->quit) return NULL;
        pool_work(a->p, a->w);
        pthread_barrier_wait(&a->p->done);
    }
}

int pch_oracle_run_pch(const int64_t *origin, const int64_t *opposite,
                       const double *length, const double *corner,
                       const uint8_t *vclass, const int64_t *outgoing,
                       int64_t nv, int64_t nf, const int64_t *src, int64_t nsrc,
                       int64_t k, int workers, int strided, double eps_win,
                       int fan_full, int64_t max_iterations, double *dist,
                       ostats *st) {
    omesh m = {origin, opposite, length, corner, vclass, nv, 3 * nf};
    memset(st, 0, sizeof(*st));
    for (int64_t v = 0; v < nv; ++v) dist[v] = INFINITY;
    for (int64_t i = 0; i < nsrc; ++i) dist[src[i]] = 0.0;
    double *scomp = (double *)malloc(sizeof(double) * 3 * nf);
    double *sentry = (double *)calloc(3 * nf, sizeof(double));
    for (int64_t i = 0; i < 3 * nf; ++i) scomp[i] = INFINITY;
    int64_t cnt0[N_COUNTERS] = {0};
    rows_t active = {0, 0, 0, WIN_COLS}, nextact = {0, 0, 0, WIN_COLS}, sel = {0, 0, 0, WIN_COLS};
    int rc = 0;
    if (o_source_rows(&m, outgoing, src, nsrc, dist, eps_win, &active, cnt0)) return -1;
    absorb(st, cnt0);
    st->windows_stored += active.n;
    int T = workers < 1 ? 1 : workers;
    rows_t *wb = (rows_t *)calloc(T, sizeof(rows_t));
    rows_t *db = (rows_t *)calloc(T, sizeof(rows_t));
    rows_t *ab = (rows_t *)calloc(T, sizeof(rows_t));
    int64_t *wcnt = (int64_t *)calloc((size_t)T * N_COUNTERS, sizeof(int64_t));
    int *fail = (int *)calloc(T, sizeof(int));
    for (int w = 0; w < T; ++w) { wb[w].cols = WIN_COLS; db[w].cols = 2; ab[w].cols = AEV_COLS; }
    wpool pool;
    memset(&pool, 0, sizeof(pool));
    pool.T = T;
    pthread_barrier_init(&pool.start, NULL, T);
    pthread_barrier_init(&pool.done, NULL, T);
    pthread_t *thr = (pthread_t *)calloc(T, sizeof(pthread_t));
    warg *args = (warg *)calloc(T, sizeof(warg));
    for (int w = 1; w < T; ++w) { args[w].p = &pool; args[w].w = w; pthread_create(&thr[w], NULL, pool_main, &args[w]); }
    uint8_t *mask = NULL; double *scratch = NULL; int64_t maskcap = 0;
    rows_t newrows = {0, 0, 0, WIN_COLS}, dev = {0, 0, 0, 2}, aev = {0, 0, 0, AEV_COLS};
    double *vbest = (double *)malloc(sizeof(double) * nv);
    for (int64_t v = 0; v < nv; ++v) vbest[v] = INFINITY;

    while (active.n) {
        if (active.n > st->peak_active_pool) st->peak_active_pool = active.n;
        /* phase 1: select (engine.py:235) */
        int64_t n = active.n;
        sel.n = 0; nextact.n = 0;
        if (n <= k) {
            rows_reserve(&sel, n);
            memcpy(sel.p, active.p, sizeof(double) * WIN_COLS * n);
            sel.n = n;
        } else {
            if (maskcap < n) { maskcap = n; mask = (uint8_t *)realloc(mask, n); scratch = (double *)realloc(scratch, sizeof(double) * n); }
            memset(mask, 0, n);
            if (!strided) mark_smallest(active.p, n, 0, 1, k, scratch, mask);
            else {
                int64_t mm = (k + T - 1) / T;
                for (int w = 0; w < T; ++w) mark_smallest(active.p, n, w, T, mm, scratch, mask);
            }
            rows_reserve(&sel, n); rows_reserve(&nextact, n);
            for (int64_t i = 0; i < n; ++i) {
                rows_t *dst = mask[i] ? &sel : &nextact;
                memcpy(dst->p + dst->n * WIN_COLS, active.p + i * WIN_COLS, sizeof(double) * WIN_COLS);
                dst->n++;
            }
        }
        /* phase 2: propagate across workers (engine.py:272) */
        int64_t ns = sel.n, share = (ns + T - 1) / T;
        if (share < 1) share = 1;
        memset(wcnt, 0, sizeof(int64_t) * T * N_COUNTERS);
        pool.sel = sel.p; pool.ns = ns; pool.share = share;
        pool.m = &m; pool.dist = dist; pool.scomp = scomp; pool.sentry = sentry;
        pool.eps_win = eps_win; pool.fan_full = fan_full;
        pool.wb = wb; pool.db = db; pool.ab = ab; pool.wcnt = wcnt; pool.fail = fail;
        pthread_barrier_wait(&pool.start);
        pool_work(&pool, 0);
        pthread_barrier_wait(&pool.done);
        int64_t tot[N_COUNTERS] = {0};
        for (int w = 0; w < T; ++w) {
            if (fail[w]) { rc = -1; goto out; }
            for (int c = 0; c < N_COUNTERS; ++c)
                tot[c] = c == C_MAXCHILD ? (wcnt[w * N_COUNTERS + c] > tot[c] ? wcnt[w * N_COUNTERS + c] : tot[c])
                                         : tot[c] + wcnt[w * N_COUNTERS + c];
        }
        absorb(st, tot);
        /* phase 3: compact per-worker buffers in worker order (engine.py:188) */
        newrows.n = dev.n = aev.n = 0;
        for (int w = 0; w < T; ++w) {
            st->events_created += db[w].n + ab[w].n;
            rows_reserve(&newrows, newrows.n + wb[w].n);
            memcpy(newrows.p + newrows.n * WIN_COLS, wb[w].p, sizeof(double) * WIN_COLS * wb[w].n);
            newrows.n += wb[w].n;
            rows_reserve(&dev, dev.n + db[w].n);
            memcpy(dev.p + dev.n * 2, db[w].p, sizeof(double) * 2 * db[w].n);
            dev.n += db[w].n;
            rows_reserve(&aev, aev.n + ab[w].n);
            memcpy(aev.p + aev.n * AEV_COLS, ab[w].p, sizeof(double) * AEV_COLS * ab[w].n);
            aev.n += ab[w].n;
        }
        int64_t kept = o_dedupe(newrows.p, newrows.n);
        st->pruned_duplicate += newrows.n - kept;
        st->total_windows_pruned += newrows.n - kept;
        st->windows_stored += kept;
        /* next active = unselected (in order) + new rows */
        if (n <= k) nextact.n = 0;
        rows_reserve(&nextact, nextact.n + kept);
        memcpy(nextact.p + nextact.n * WIN_COLS, newrows.p, sizeof(double) * WIN_COLS * kept);
        nextact.n += kept;
        { rows_t t = active; active = nextact; nextact = t; }
        /* phase 4: events (engine.py:341, :359) */
        int64_t applied = 0;
        for (int64_t e = 0; e < dev.n; ++e) {
            int64_t v = (int64_t)dev.p[2 * e];
            if (dev.p[2 * e + 1] < vbest[v]) vbest[v] = dev.p[2 * e + 1];
        }
        for (int64_t e = 0; e < dev.n; ++e) {
            int64_t v = (int64_t)dev.p[2 * e];
            if (vbest[v] < INFINITY) {
                if (vbest[v] < dist[v]) { dist[v] = vbest[v]; applied++; }
                vbest[v] = INFINITY;
            }
        }
        if (aev.n) {
            qsort(aev.p, aev.n, sizeof(double) * AEV_COLS, aev_cmp);
            for (int64_t e = 0; e < aev.n; ++e) {
                const double *a = aev.p + e * AEV_COLS;
                if (e > 0 && aev.p[(e - 1) * AEV_COLS + W_HE] == a[W_HE]) continue;
                int64_t he = (int64_t)a[W_HE];
                if (a[AE_COMP] < scomp[he]) { scomp[he] = a[AE_COMP]; sentry[he] = a[AE_ENTRYX]; applied++; }
            }
        }
        st->events_applied += applied;
        st->iterations++;
        if (max_iterations > 0 && st->iterations > max_iterations) { rc = -2; goto out; }
    }
out:
    pool.quit = 1;
    pthread_barrier_wait(&pool.start);
    for (int w = 1; w < T; ++w) pthread_join(thr[w], NULL);
    pthread_barrier_destroy(&pool.start); pthread_barrier_destroy(&pool.done);
    free(thr); free(args);
    for (int w = 0; w < T; ++w) { rows_free(&wb[w]); rows_free(&db[w]); rows_free(&ab[w]); }
    free(wb); free(db); free(ab); free(wcnt); free(fail); free(mask); free(scratch);
    free(vbest); free(scomp); free(sentry);
    rows_free(&active); rows_free(&nextact); rows_free(&sel);
    rows_free(&newrows); rows_free(&dev); rows_free(&aev);
    return rc;
}

int pch_oracle_abi_version(void) { return 1; }
