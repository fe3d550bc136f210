/*
 * pch_model.c -- sequential CPU model of the B200 engine's *semantics*
 * (design-exploration tool; not product, not the parity oracle).
 *
 * It reuses the oracle's geometry (included below) and replays the batch
 * schedule the CUDA engine implements, so window counts of design choices
 * can be measured on CPU before GPU time is spent:
 *   - threshold selection: every window with key <= t, t = k-th smallest
 *   - DEFER_FANS: a saddle vertex's fan is emitted once per iteration, by
 *     the event with the smallest candidate distance, one iteration later
 *   - RECHECK: at pop time re-test the two endpoint inequalities of the
 *     ICH filter against the current distances of the window's own edge
 *   - split rule: smallest comp wins (ties: smallest entry_x)
 */
#include "../oracle/pch_oracle.c"

enum { F_DEFER_FANS = 1, F_RECHECK = 2, F_MINCOMP = 4 };

typedef struct { int64_t v, anchor; double cand, rel; } fanev;

/* propagation with fans recorded as events instead of emitted */
static int m_propagate(const double *row, const omesh *m, const double *gd,
                       const double *split_comp, const double *split_entryx,
                       double eps_win, int flags, rows_t *ow, rows_t *od,
                       rows_t *oa, fanev **fe, int64_t *nfe, int64_t *fecap,
                       int64_t *cnt, int64_t *rechecked) {
    const double eps_num = 1e-12;
    int64_t j = (int64_t)row[W_HE];
    double b0 = row[W_B0], b1 = row[W_B1], d0 = row[W_D0], d1 = row[W_D1];
    double dps = row[W_D];
    double ell = m->length[j];
    double ix, iy;
    if (!o_unfold(b0, b1, d0, d1, eps_num, &ix, &iy)) { cnt[C_PRUNE_DEGEN]++; return 0; }
    int64_t jn = nxt(j), jp = prv(j);
    int64_t v0 = m->origin[j], v1 = m->origin[jn];
    if (flags & F_RECHECK) {
        double g0 = gd[v0], g1 = gd[v1];
        double tA = dps + hypot(ix - b0, iy), tB = dps + hypot(ix - b1, iy);
        if ((g0 < INFINITY && tB > g0 + b1 + eps_num) ||
            (g1 < INFINITY && tA > g1 + (ell - b0) + eps_num)) {
            (*rechecked)++;
            return 0;
        }
    }
    cnt[C_PROPAGATED]++;
    if (!(flags & F_DEFER_FANS))
        return o_propagate(row, m, gd, split_comp, split_entryx, eps_win, eps_num, 0, ow, od, oa, cnt);
#define FANEV(V, C, A, R) do { if (*nfe == *fecap) { *fecap = *fecap ? 2 * *fecap : 1024; *fe = realloc(*fe, sizeof(fanev) * *fecap); } \
        (*fe)[*nfe].v = (V); (*fe)[*nfe].cand = (C); (*fe)[*nfe].anchor = (A); (*fe)[*nfe].rel = (R); (*nfe)++; } while (0)
    int64_t stored = 0, add;
    if (b0 <= eps_win) {
        double cand = dps + d0 + b0;
        if (cand < gd[v0]) {
            double *e = rows_push(od); e[0] = (double)v0; e[1] = cand;
            if (m->vclass[v0] == SADDLE) FANEV(v0, cand, j, atan2(iy, ix));
        }
    }
    if (b1 >= ell - eps_win) {
        double cand = dps + d1 + (ell - b1);
        if (cand < gd[v1]) {
            double *e = rows_push(od); e[0] = (double)v1; e[1] = cand;
            if (m->vclass[v1] == SADDLE) {
                double lps = m->length[jp], lns = m->length[jn];
                double axs = 0.5 * (ell * ell + lps * lps - lns * lns) / ell;
                double ay2 = lps * lps - axs * axs;
                double ays = ay2 > 0.0 ? sqrt(ay2) : 0.0;
                double adir = atan2(ays, axs - ell);
                FANEV(v1, cand, jn, atan2(iy, ix - ell) - adir);
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
        double ca = uax * vdy - uay * vdx, cb = ubx * vdy - uby * vdx;
        double tola = eps_num * hypot(uax, uay) * nvd, tolb = eps_num * hypot(ubx, uby) * nvd;
        double g0 = gd[v0], g1 = gd[v1], gdd = gd[vd];
        double sa, sb;
        if (ca > tola && cb < -tolb) {
            double comp = dps + nvd, denom = iy - dy;
            double entry_x = denom > 1e-300 ? ix + (dx - ix) * (iy / denom) : ix;
            int wl = 1, wr = 1;
            if (comp < split_comp[j]) {
                double *a = rows_push(oa);
                for (int c = 0; c < WIN_COLS; ++c) a[c] = row[c];
                a[AE_COMP] = comp; a[AE_ENTRYX] = entry_x;
            } else {
                cnt[C_PRUNE_SPLIT]++; cnt[C_CREATED]++;
                if (entry_x < split_entryx[j]) wr = 0; else wl = 0;
            }
            if (wl) {
                if (o_ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, &sa)) {
                    add = o_emit_child(jno, lan, 0.0, 0.0, dx, dy, sa, 1.0, ix, iy, dps, g0, gdd, g1, ell, 0.0, 1, eps_win, eps_num, ow, cnt);
                    stored += add;
                } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
            }
            if (wr) {
                if (o_ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, &sb)) {
                    add = o_emit_child(jpo, lpv, dx, dy, ell, 0.0, 0.0, sb, ix, iy, dps, gdd, g1, g0, 0.0, 0.0, 0, eps_win, eps_num, ow, cnt);
                    stored += add;
                } else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
            }
            double cand = dps + nvd;
            if (cand < gdd) {
                double *e = rows_push(od); e[0] = (double)vd; e[1] = cand;
                if (m->vclass[vd] == SADDLE) {
                    double gamma = atan2(-dy, ell - dx);
                    FANEV(vd, cand, jpo, atan2(iy - dy, ix - dx) - gamma);
                }
            }
        } else if (cb >= -tolb) {
            int oka = o_ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, &sa);
            int okb = o_ray_seg(ix, iy, b1, 0.0, 0.0, 0.0, dx, dy, &sb);
            if (oka && okb) stored += o_emit_child(jno, lan, 0.0, 0.0, dx, dy, sa, sb, ix, iy, dps, g0, gdd, g1, ell, 0.0, 1, eps_win, eps_num, ow, cnt);
            else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
        } else {
            int oka = o_ray_seg(ix, iy, b0, 0.0, dx, dy, ell, 0.0, &sa);
            int okb = o_ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, &sb);
            if (oka && okb) stored += o_emit_child(jpo, lpv, dx, dy, ell, 0.0, sa, sb, ix, iy, dps, gdd, g1, g0, 0.0, 0.0, 0, eps_win, eps_num, ow, cnt);
            else { cnt[C_CREATED]++; cnt[C_PRUNE_DEGEN]++; }
        }
    }
    if (stored > cnt[C_MAXCHILD]) cnt[C_MAXCHILD] = stored;
    return 0;
#undef FANEV
}

static int dcmp(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : x > y;
}

int pch_model_run(const int64_t *origin, const int64_t *opposite,
                  const double *length, const double *corner,
                  const uint8_t *vclass, const int64_t *outgoing, int64_t nv,
                  int64_t nf, const int64_t *src, int64_t nsrc, int64_t k,
                  int flags, double *dist, int64_t *out /* 6 */) {
    const double eps_win = 1e-6;
    omesh m = {origin, opposite, length, corner, vclass, nv, 3 * nf};
    for (int64_t v = 0; v < nv; ++v) dist[v] = INFINITY;
    for (int64_t i = 0; i < nsrc; ++i) dist[src[i]] = 0.0;
    double *scomp = malloc(sizeof(double) * 3 * nf), *sentry = calloc(3 * nf, sizeof(double));
    for (int64_t i = 0; i < 3 * nf; ++i) scomp[i] = INFINITY;
    int64_t cnt[N_COUNTERS] = {0};
    rows_t act = {0, 0, 0, WIN_COLS}, nact = {0, 0, 0, WIN_COLS}, sel = {0, 0, 0, WIN_COLS};
    rows_t nw = {0, 0, 0, WIN_COLS}, dv = {0, 0, 0, 2}, av = {0, 0, 0, AEV_COLS};
    o_source_rows(&m, outgoing, src, nsrc, dist, eps_win, &act, cnt);
    fanev *fe = NULL; int64_t nfe = 0, fecap = 0;
    fanev *pend = NULL; int64_t npend = 0;
    double *fbest = malloc(sizeof(double) * nv);
    int64_t *fwin = malloc(sizeof(int64_t) * nv);
    for (int64_t v = 0; v < nv; ++v) { fbest[v] = INFINITY; fwin[v] = -1; }
    double *keys = NULL; int64_t keycap = 0;
    int64_t iters = 0, rechecked = 0, fans = 0;
    while (act.n || npend) {
        nw.n = dv.n = av.n = 0;
        /* deferred fans from the previous iteration */
        for (int64_t i = 0; i < npend; ++i) {
            if (pend[i].cand > dist[pend[i].v]) continue;
            fans++;
            o_emit_fan(&m, pend[i].v, pend[i].cand, pend[i].anchor, pend[i].rel, 0, dist, eps_win, 1e-12, 0, &nw, cnt);
        }
        npend = 0;
        /* threshold selection */
        int64_t n = act.n;
        sel.n = 0; nact.n = 0;
        rows_reserve(&sel, n); rows_reserve(&nact, n);
        double t = INFINITY;
        if (n > k) {
            if (keycap < n) { keycap = n; keys = realloc(keys, sizeof(double) * n); }
            for (int64_t i = 0; i < n; ++i) keys[i] = act.p[i * WIN_COLS + W_KEY];
            t = kth_smallest(keys, n, k - 1);
        }
        for (int64_t i = 0; i < n; ++i) {
            rows_t *d = act.p[i * WIN_COLS + W_KEY] <= t ? &sel : &nact;
            memcpy(d->p + d->n * WIN_COLS, act.p + i * WIN_COLS, sizeof(double) * WIN_COLS);
            d->n++;
        }
        nfe = 0;
        for (int64_t i = 0; i < sel.n; ++i)
            m_propagate(sel.p + i * WIN_COLS, &m, dist, scomp, sentry, eps_win, flags, &nw, &dv, &av, &fe, &nfe, &fecap, cnt, &rechecked);
        int64_t kept = o_dedupe(nw.p, nw.n);
        rows_reserve(&nact, nact.n + kept);
        memcpy(nact.p + nact.n * WIN_COLS, nw.p, sizeof(double) * WIN_COLS * kept);
        nact.n += kept;
        { rows_t tt = act; act = nact; nact = tt; }
        for (int64_t e = 0; e < dv.n; ++e) {
            int64_t v = (int64_t)dv.p[2 * e];
            if (dv.p[2 * e + 1] < dist[v]) dist[v] = dv.p[2 * e + 1];
        }
        if (flags & F_MINCOMP) {
            for (int64_t e = 0; e < av.n; ++e) {
                const double *a = av.p + e * AEV_COLS;
                int64_t he = (int64_t)a[W_HE];
                if (a[AE_COMP] < scomp[he] || (a[AE_COMP] == scomp[he] && a[AE_ENTRYX] < sentry[he])) {
                    scomp[he] = a[AE_COMP]; sentry[he] = a[AE_ENTRYX];
                }
            }
        } else if (av.n) {
            qsort(av.p, av.n, sizeof(double) * AEV_COLS, aev_cmp);
            for (int64_t e = 0; e < av.n; ++e) {
                const double *a = av.p + e * AEV_COLS;
                if (e > 0 && av.p[(e - 1) * AEV_COLS + W_HE] == a[W_HE]) continue;
                int64_t he = (int64_t)a[W_HE];
                if (a[AE_COMP] < scomp[he]) { scomp[he] = a[AE_COMP]; sentry[he] = a[AE_ENTRYX]; }
            }
        }
        /* fan winners: smallest cand per vertex (ties: anchor, rel) */
        for (int64_t e = 0; e < nfe; ++e) {
            int64_t v = fe[e].v;
            int64_t w = fwin[v];
            if (w < 0 || fe[e].cand < fe[w].cand ||
                (fe[e].cand == fe[w].cand && (fe[e].anchor < fe[w].anchor ||
                 (fe[e].anchor == fe[w].anchor && fe[e].rel < fe[w].rel))))
                fwin[v] = e;
        }
        pend = realloc(pend, sizeof(fanev) * (nfe + 1));
        for (int64_t e = 0; e < nfe; ++e) {
            int64_t v = fe[e].v;
            if (fwin[v] == e) pend[npend++] = fe[e];
        }
        for (int64_t e = 0; e < nfe; ++e) fwin[fe[e].v] = -1;
        iters++;
    }
    out[0] = cnt[C_CREATED]; out[1] = cnt[C_PROPAGATED]; out[2] = iters;
    out[3] = rechecked; out[4] = fans; out[5] = cnt[C_PRUNE_ICH];
    free(scomp); free(sentry); free(fe); free(pend); free(fbest); free(fwin); free(keys);
    rows_free(&act); rows_free(&nact); rows_free(&sel); rows_free(&nw); rows_free(&dv); rows_free(&av);
    return 0;
}

/* one-barrier schedule: during iteration i the threshold t_{i+1} is the
 * k-th smallest key of the pool P_i (children of S_i are routed by it as
 * they are created); fans of iteration i-1 are emitted in iteration i by
 * every fan event whose candidate equals the committed distance. */
int pch_model_run1(const int64_t *origin, const int64_t *opposite,
                   const double *length, const double *corner,
                   const uint8_t *vclass, const int64_t *outgoing, int64_t nv,
                   int64_t nf, const int64_t *src, int64_t nsrc, int64_t k,
                   int flags, double *dist, int64_t *out /* 6 */) {
    const double eps_win = 1e-6;
    omesh m = {origin, opposite, length, corner, vclass, nv, 3 * nf};
    for (int64_t v = 0; v < nv; ++v) dist[v] = INFINITY;
    for (int64_t i = 0; i < nsrc; ++i) dist[src[i]] = 0.0;
    double *scomp = malloc(sizeof(double) * 3 * nf), *sentry = calloc(3 * nf, sizeof(double));
    for (int64_t i = 0; i < 3 * nf; ++i) scomp[i] = INFINITY;
    int64_t cnt[N_COUNTERS] = {0};
    rows_t S = {0, 0, 0, WIN_COLS}, P = {0, 0, 0, WIN_COLS}, S2 = {0, 0, 0, WIN_COLS}, P2 = {0, 0, 0, WIN_COLS};
    rows_t nw = {0, 0, 0, WIN_COLS}, dv = {0, 0, 0, 2}, av = {0, 0, 0, AEV_COLS};
    o_source_rows(&m, outgoing, src, nsrc, dist, eps_win, &S, cnt);
    fanev *fe = NULL, *pend = NULL; int64_t nfe = 0, fecap = 0, npend = 0, pendcap = 0;
    double *keys = NULL; int64_t keycap = 0;
    int64_t iters = 0, rechecked = 0, fans = 0, maxbatch = 0;
    double tprev = 0.0, delta = 0.5;
    while (S.n || P.n || npend) {
        if (S.n > maxbatch) maxbatch = S.n;
        double t = INFINITY;
        if (flags & 8) {
            /* step controller: t = t_prev + delta, delta steered by |S|/k */
            double r = (double)(S.n > 0 ? S.n : 1) / (double)k;
            double f = 1.0 / r;
            if (f > 1.25) f = 1.25;
            if (f < 0.5) f = 0.5;
            if (iters > 0) delta *= f;
            if (delta > 4.0) delta = 4.0;
            if (delta < 1e-3) delta = 1e-3;
            double pmin = INFINITY;
            for (int64_t i = 0; i < P.n; ++i) if (P.p[i * WIN_COLS + W_KEY] < pmin) pmin = P.p[i * WIN_COLS + W_KEY];
            t = tprev + delta;
            if (S.n == 0 && pmin > t) t = pmin;
            tprev = t;
        } else if (P.n > k) {
            if (keycap < P.n) { keycap = P.n; keys = realloc(keys, sizeof(double) * P.n); }
            for (int64_t i = 0; i < P.n; ++i) keys[i] = P.p[i * WIN_COLS + W_KEY];
            t = kth_smallest(keys, P.n, k - 1);
        }
        nw.n = dv.n = av.n = 0;
        for (int64_t i = 0; i < npend; ++i) {
            if (pend[i].cand != dist[pend[i].v]) continue;
            fans++;
            o_emit_fan(&m, pend[i].v, pend[i].cand, pend[i].anchor, pend[i].rel, 0, dist, eps_win, 1e-12, 0, &nw, cnt);
        }
        nfe = 0;
        for (int64_t i = 0; i < S.n; ++i)
            m_propagate(S.p + i * WIN_COLS, &m, dist, scomp, sentry, eps_win, flags, &nw, &dv, &av, &fe, &nfe, &fecap, cnt, &rechecked);
        int64_t kept = o_dedupe(nw.p, nw.n);
        S2.n = P2.n = 0;
        rows_reserve(&S2, P.n + kept); rows_reserve(&P2, P.n + kept);
        for (int pass = 0; pass < 2; ++pass) {
            rows_t *src_ = pass ? &nw : &P;
            int64_t n = pass ? kept : P.n;
            for (int64_t i = 0; i < n; ++i) {
                rows_t *d = src_->p[i * WIN_COLS + W_KEY] <= t ? &S2 : &P2;
                memcpy(d->p + d->n * WIN_COLS, src_->p + i * WIN_COLS, sizeof(double) * WIN_COLS);
                d->n++;
            }
        }
        { rows_t tt = S; S = S2; S2 = tt; tt = P; P = P2; P2 = tt; }
        for (int64_t e = 0; e < dv.n; ++e) {
            int64_t v = (int64_t)dv.p[2 * e];
            if (dv.p[2 * e + 1] < dist[v]) dist[v] = dv.p[2 * e + 1];
        }
        for (int64_t e = 0; e < av.n; ++e) {
            const double *a = av.p + e * AEV_COLS;
            int64_t he = (int64_t)a[W_HE];
            if (a[AE_COMP] < scomp[he] || (a[AE_COMP] == scomp[he] && a[AE_ENTRYX] < sentry[he])) {
                scomp[he] = a[AE_COMP]; sentry[he] = a[AE_ENTRYX];
            }
        }
        if (pendcap < nfe) { pendcap = nfe; pend = realloc(pend, sizeof(fanev) * pendcap); }
        memcpy(pend, fe, sizeof(fanev) * nfe);
        npend = nfe;
        iters++;
    }
    out[0] = cnt[C_CREATED]; out[1] = cnt[C_PROPAGATED]; out[2] = iters;
    out[3] = rechecked; out[4] = fans; out[5] = maxbatch;
    free(scomp); free(sentry); free(fe); free(pend); free(keys);
    rows_free(&S); rows_free(&P); rows_free(&S2); rows_free(&P2); rows_free(&nw); rows_free(&dv); rows_free(&av);
    return 0;
}
