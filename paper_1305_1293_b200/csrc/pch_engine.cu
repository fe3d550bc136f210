// pch_engine.cu -- B200-native Parallel Chen-Han exact geodesic solver.
//
// One persistent cooperative kernel runs the whole PCH loop (paper
// Algorithm 1; reference pkg/src/pargeo/engine.py:433 run_pch) on the
// device.  Each iteration is two phases separated by grid barriers, so
// the per-level CPU/GPU synchronisation the paper identifies as the CH
// bottleneck never happens:
//
//   phase A  (propagate)  every thread takes windows of the selected batch
//            S_i and runs Algorithm 2 (geom.py:312) against the *frozen*
//            distance field and angle-split table of the previous
//            iteration; children are appended to the pool (warp-aggregated
//            slot allocation), their keys histogrammed; distance events
//            are 64-bit atomicMin on the fp64 bit patterns of a shadow
//            field, angle events a 128-bit CAS-min of (comp, entry_x) on a
//            shadow split table; saddle fans of the previous iteration's
//            winners are emitted here too.
//   phase B  (organise)   the k-selection threshold t_{i+1} is read off the
//            key histogram (distance-threshold pick, every CTA computes the
//            same value); touched vertices / angles are committed from the
//            shadow tables; the pool P_i + children C_i is partitioned into
//            the next batch S_{i+1} (key <= t) and the next pool P_{i+1}
//            (stream compaction, gap free -- paper Algorithm 3), whose keys
//            are histogrammed for the following threshold.
//
// Deferred event application replaces the paper's sort-then-first-wins
// pass (Algorithm 4; engine.py:341/:359): atomicMin is order independent,
// so results do not depend on scheduling.  Saddle fans are deferred one
// iteration and emitted once per vertex by the smallest candidate
// (window-count control).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pch_b200.h"
#include "pch_device.cuh"

using namespace pch;

// ---------------------------------------------------------------------------
// device state

enum { ST_PROPAGATED, ST_CREATED, ST_PRUNE_ICH, ST_PRUNE_SPLIT, ST_PRUNE_TINY,
       ST_PRUNE_DEGEN, ST_RECHECK, ST_STORED, ST_EV_CREATED, ST_EV_APPLIED,
       ST_FANS, ST_MAXCHILD, ST_PEAK, N_ST };

enum { ERR_NONE = 0, ERR_OVERFLOW = 1, ERR_GUARD = 2, ERR_TIMEOUT = 3 };

struct Slot {               // per-iteration counters, indexed by iteration % 3
    unsigned long long nS;  // size of the selected batch S (written in phase B)
    unsigned long long nP;  // size of the pool P (written in phase B)
    unsigned long long nC;  // children appended during phase A
    unsigned long long nTV; // touched vertices (phase A)
    unsigned long long nTE; // touched angle entries (phase A)
    unsigned long long nF;  // fan events (phase A)
    unsigned long long pad[2];
};

struct Ctrl {
    Slot slot[3];
    unsigned int bar_count;
    unsigned int bar_gen;
    int error;
    int pad0;
    long long iterations;
    unsigned long long st[N_ST];
    double t_final;
    int final_parity;  // which of X/Y held the last pool (unused on exit)
    int pad1;
};

struct Params {
    // mesh (immutable)
    const HeRec *he;
    const FanRec *fan;
    const int32_t *fan_off;    // [nv + 1]
    const int32_t *fanpos;     // [nhe] position of h in origin(h)'s fan
    const double *fan_theta;   // [nv]
    const uint8_t *fan_interior;  // [nv]
    int32_t nv, nhe;
    // distance field / angle-split table: frozen + shadow copies
    double *dist_cur;
    unsigned long long *dist_new;
    double2 *split_cur;        // (comp, entry_x)
    ulonglong2 *split_new;     // (ord(comp), ord(entry_x))
    ulonglong2 *fanpick[2];    // per vertex (cand bits, anchor<<32 | ord32(rel))
    int32_t *tv_stamp, *te_stamp;
    int32_t *tv_list, *te_list;
    FanEv *fanev[2];
    long long fancap;
    // window pools
    WinSoA X, Y, S;
    long long cap;
    unsigned int *hist[2];     // NBINS + 1 bins each
    Ctrl *ctrl;
    // config
    long long K;
    double eps_win;
    double w0;
    long long max_iter;
    unsigned long long time_limit_ns;
    int fan_full;
    int recheck;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ord64(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord64(unsigned long long b) {
    b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    return __longlong_as_double((long long)b);
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  The
// last arriver resets the counter and bumps the generation.  A waiter that
// sees no release within 20 s flags ERR_TIMEOUT instead of hanging.
__device__ __forceinline__ void grid_barrier(Ctrl *c, unsigned int &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int target = gen + 1;
        __threadfence();
        unsigned int arrived = atomicAdd(&c->bar_count, 1u);
        if (arrived == gridDim.x - 1) {
            atomicExch(&c->bar_count, 0u);
            __threadfence();
            atomicExch(&c->bar_gen, target);
        } else {
            unsigned long long t0 = globaltimer();
            while (ld_acquire_u32(&c->bar_gen) != target) {
                __nanosleep(32);
                if (globaltimer() - t0 > 20000000000ull) {
                    atomicExch(&c->error, ERR_TIMEOUT);
                    break;
                }
            }
        }
        __threadfence();
        gen = target;
    }
    __syncthreads();
}

// Warp-aggregated slot allocation among the currently active lanes:
// each lane with `want` gets a distinct index from *counter.
__device__ __forceinline__ unsigned long long warp_alloc(unsigned long long *counter,
                                                         bool want) {
    unsigned mask = __activemask();
    unsigned b = __ballot_sync(mask, want);
    int lane = threadIdx.x & 31;
    int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader && b) base = atomicAdd(counter, (unsigned long long)__popc(b));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(b & ((1u << lane) - 1u));
}

__device__ __forceinline__ int key_bin(double key, double base, double w) {
    double f = (key - base) / w;
    if (!(f >= 0.0)) return 0;
    if (f >= (double)NBINS) return NBINS;
    return (int)f;
}

__device__ __forceinline__ void store_win(const WinSoA &W, unsigned long long i, const Win &c) {
    W.he[i] = c.he;
    W.b0[i] = c.b0;
    W.b1[i] = c.b1;
    W.d0[i] = c.d0;
    W.d1[i] = c.d1;
    W.d[i] = c.d;
    W.key[i] = c.key;
}

__device__ __forceinline__ Win load_win(const WinSoA &W, unsigned long long i) {
    Win c;
    c.he = __ldcg(W.he + i);
    c.b0 = __ldcg(W.b0 + i);
    c.b1 = __ldcg(W.b1 + i);
    c.d0 = __ldcg(W.d0 + i);
    c.d1 = __ldcg(W.d1 + i);
    c.d = __ldcg(W.d + i);
    c.key = __ldcg(W.key + i);
    return c;
}

struct LocalStats {
    unsigned long long v[N_ST];
    __device__ void zero() {
#pragma unroll
        for (int i = 0; i < N_ST; ++i) v[i] = 0;
    }
};

__device__ __forceinline__ void flush_stats(Ctrl *c, LocalStats &ls) {
#pragma unroll
    for (int i = 0; i < N_ST; ++i) {
        unsigned long long x = ls.v[i];
        if (i == ST_MAXCHILD || i == ST_PEAK) {
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
                x = x > y ? x : y;
            }
            if ((threadIdx.x & 31) == 0 && x) atomicMax(&c->st[i], x);
        } else {
#pragma unroll
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) == 0 && x) atomicAdd(&c->st[i], x);
        }
    }
    ls.zero();
}

// ---------------------------------------------------------------------------
// events

__device__ __forceinline__ void dist_event(const Params &p, Slot &sl, int it, int32_t v,
                                           double cand, LocalStats &ls) {
    ls.v[ST_EV_CREATED]++;
    unsigned long long nb = (unsigned long long)__double_as_longlong(cand);
    unsigned long long old = atomicMin(p.dist_new + v, nb);
    if (nb < old && atomicExch(p.tv_stamp + v, it) != it) {
        unsigned long long slot = atomicAdd(&sl.nTV, 1ull);
        p.tv_list[slot] = v;
        ls.v[ST_EV_APPLIED]++;
    }
}

__device__ __forceinline__ void angle_event(const Params &p, Slot &sl, int it, int32_t j,
                                            double comp, double entry, LocalStats &ls) {
    ls.v[ST_EV_CREATED]++;
    if (cas_min_u128(p.split_new + j, ord64(comp), ord64(entry)) &&
        atomicExch(p.te_stamp + j, it) != it) {
        unsigned long long slot = atomicAdd(&sl.nTE, 1ull);
        p.te_list[slot] = j;
        ls.v[ST_EV_APPLIED]++;
    }
}

__device__ __forceinline__ void fan_event(const Params &p, Slot &sl, int it, int32_t v,
                                          int32_t anchor, double cand, double rel) {
    unsigned long long hi = (unsigned long long)__double_as_longlong(cand);
    unsigned long long lo = ((unsigned long long)(uint32_t)anchor << 32) | ord_hi32(rel);
    cas_min_u128(p.fanpick[it & 1] + v, hi, lo);
    unsigned long long slot = atomicAdd(&sl.nF, 1ull);
    if ((long long)slot < p.fancap) {
        FanEv e;
        e.v = v;
        e.anchor = anchor;
        e.cand = cand;
        e.rel = rel;
        p.fanev[it & 1][slot] = e;
    } else {
        atomicExch(&p.ctrl->error, ERR_OVERFLOW);
    }
}

// ---------------------------------------------------------------------------
// saddle fans (geom.py:185): windows with pseudo source v on the edges
// opposite v inside the fan spanned by the two straight extensions of the
// incoming ray; `full` emits every wedge (source initialisation).

template <typename Emit>
__device__ void emit_fan(const Params &p, int32_t v, double cand, int32_t anchor,
                         double rel, bool full, const double *dist, Emit &&emit,
                         LocalStats &ls) {
    int32_t off = __ldg(p.fan_off + v);
    int32_t m = __ldg(p.fan_off + v + 1) - off;
    double theta = __ldg(p.fan_theta + v);
    double flo, fhi;
    int reps;
    if (full) {
        flo = -1.0e300;
        fhi = 1.0e300;
        reps = 1;
    } else {
        double width = theta - TWO_PI_D;
        if (width <= EPS_NUM) return;
        double aphi = __ldg(&p.fan[off + __ldg(p.fanpos + anchor)].wlo);
        flo = aphi + rel + PI_D;
        fhi = flo + width;
        if (__ldg(p.fan_interior + v)) {
            double k = floor(flo / theta);
            flo -= k * theta;
            fhi -= k * theta;
            reps = 2;
        } else {
            reps = 1;
        }
    }
    for (int i = 0; i < m; ++i) {
        const FanRec &f = p.fan[off + i];
        double wlo = __ldg(&f.wlo), whi = __ldg(&f.whi);
        for (int rep = 0; rep < reps; ++rep) {
            double lo = flo - rep * theta, hi = fhi - rep * theta;
            double slo = wlo > lo ? wlo : lo;
            double shi = whi < hi ? whi : hi;
            if (shi - slo <= 1e-12) continue;
            if (p.fan_full) {
                slo = wlo;
                shi = whi;
            }
            double px = __ldg(&f.px), py = __ldg(&f.py), qx = __ldg(&f.qx), qy = __ldg(&f.qy);
            double s0 = 0.0, s1 = 1.0;
            bool ok0 = true, ok1 = true;
            if (!(slo <= wlo + 1e-12)) {
                double sn, cs;
                sincos(slo, &sn, &cs);
                ok0 = ray_seg(0.0, 0.0, cs, sn, px, py, qx, qy, s0);
            }
            if (!(shi >= whi - 1e-12)) {
                double sn, cs;
                sincos(shi, &sn, &cs);
                ok1 = ray_seg(0.0, 0.0, cs, sn, px, py, qx, qy, s1);
            }
            ls.v[ST_CREATED]++;
            if (!(ok0 && ok1)) {
                ls.v[ST_PRUNE_DEGEN]++;
                continue;
            }
            int32_t pid = __ldg(&f.pid), qid = __ldg(&f.qid);
            Win c;
            int fate = make_child(__ldg(&f.che), __ldg(&f.lc), px, py, qx, qy, s0, s1, 0.0, 0.0,
                                  cand, ldcg(dist + pid), ldcg(dist + qid), INFINITY, 0.0, 0.0,
                                  true, p.eps_win, c);
            if (fate == CH_STORED) {
                emit(c);
            } else {
                ls.v[fate == CH_TINY ? ST_PRUNE_TINY : fate == CH_ICH ? ST_PRUNE_ICH : ST_PRUNE_DEGEN]++;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Algorithm 2 (geom.py:312) for one window against the frozen tables.
// Up to two children are returned in `c`; events go to the shadow tables.

__device__ int propagate(const Params &p, Slot &sl, int it, const Win &w, Win c[2],
                         LocalStats &ls) {
    const int32_t j = w.he;
    const double b0 = w.b0, b1 = w.b1, d0 = w.d0, d1 = w.d1, dps = w.d;
    double ix, iy;
    if (!unfold(b0, b1, d0, d1, ix, iy)) {
        ls.v[ST_PRUNE_DEGEN]++;
        return 0;
    }
    const HeRec *hp = p.he + j;
    const double ell = __ldg(&hp->ell);
    const uint32_t v0f = __ldg(&hp->v0), v1f = __ldg(&hp->v1);
    const int32_t v0 = (int32_t)(v0f & VMASK), v1 = (int32_t)(v1f & VMASK);
    const double g0 = ldcg(p.dist_cur + v0), g1 = ldcg(p.dist_cur + v1);

    if (p.recheck) {
        // endpoint inequalities of the ICH filter (paper Fig. 4b) against
        // the current field: paths through v0 (resp. v1) already reach the
        // far end of the interval more cheaply -> the window is useless
        double tB = dps + hyp(ix - b1, iy), tA = dps + hyp(ix - b0, iy);
        if ((g0 < INFINITY && tB > g0 + b1 + EPS_NUM) ||
            (g1 < INFINITY && tA > g1 + (ell - b0) + EPS_NUM)) {
            ls.v[ST_RECHECK]++;
            return 0;
        }
    }
    ls.v[ST_PROPAGATED]++;
    int nc = 0;

    if (b0 <= p.eps_win) {
        double cand = dps + d0 + b0;
        if (cand < g0) {
            dist_event(p, sl, it, v0, cand, ls);
            if (v0f & SADDLE_BIT) fan_event(p, sl, it, v0, j, cand, atan2(iy, ix));
        }
    }
    if (b1 >= ell - p.eps_win) {
        double cand = dps + d1 + (ell - b1);
        if (cand < g1) {
            dist_event(p, sl, it, v1, cand, ls);
            if (v1f & SADDLE_BIT) {
                int32_t jn = 3 * (j / 3) + (j + 1) % 3;
                fan_event(p, sl, it, v1, jn, cand, atan2(iy, ix - ell) - __ldg(&hp->adir));
            }
        }
    }

    const int32_t jo = __ldg(&hp->jo);
    if (jo < 0) return 0;
    const int32_t jno = 3 * (jo / 3) + (jo + 1) % 3;
    const int32_t jpo = 3 * (jo / 3) + (jo + 2) % 3;
    const double dx = __ldg(&hp->dx), dy = __ldg(&hp->dy);
    const double lan = __ldg(&hp->lan), lpv = __ldg(&hp->lpv);
    const uint32_t vdf = __ldg(&hp->vd);
    const int32_t vd = (int32_t)(vdf & VMASK);
    const double gdd = ldcg(p.dist_cur + vd);

    const double uax = b0 - ix, uay = -iy, ubx = b1 - ix, uby = -iy;
    const double vdx = dx - ix, vdy = dy - iy;
    const double nvd = hyp(vdx, vdy);
    const double ca = uax * vdy - uay * vdx;
    const double cb = ubx * vdy - uby * vdx;
    const double tola = EPS_NUM * hyp(uax, uay) * nvd;
    const double tolb = EPS_NUM * hyp(ubx, uby) * nvd;
    double sa, sb;

    if (ca > tola && cb < -tolb) {
        // the ray to the apex passes strictly inside (A, B): w occupies vd
        double comp = dps + nvd;
        double denom = iy - dy;
        double entry_x = denom > 1e-300 ? ix + (dx - ix) * (iy / denom) : ix;
        bool want_l = true, want_r = true;
        double2 sp = __ldcg(p.split_cur + j);
        if (comp < sp.x) {
            angle_event(p, sl, it, j, comp, entry_x, ls);
        } else {
            // one-angle-one-split: keep only the child on our side
            ls.v[ST_PRUNE_SPLIT]++;
            ls.v[ST_CREATED]++;
            if (entry_x < sp.y) want_r = false;
            else want_l = false;
        }
        if (want_l) {
            ls.v[ST_CREATED]++;
            if (ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, sa)) {
                int f = make_child(jno, lan, 0.0, 0.0, dx, dy, sa, 1.0, ix, iy, dps, g0, gdd, g1,
                                   ell, 0.0, true, p.eps_win, c[nc]);
                if (f == CH_STORED) nc++;
                else ls.v[f == CH_TINY ? ST_PRUNE_TINY : f == CH_ICH ? ST_PRUNE_ICH : ST_PRUNE_DEGEN]++;
            } else {
                ls.v[ST_PRUNE_DEGEN]++;
            }
        }
        if (want_r) {
            ls.v[ST_CREATED]++;
            if (ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, sb)) {
                int f = make_child(jpo, lpv, dx, dy, ell, 0.0, 0.0, sb, ix, iy, dps, gdd, g1, g0,
                                   0.0, 0.0, false, p.eps_win, c[nc]);
                if (f == CH_STORED) nc++;
                else ls.v[f == CH_TINY ? ST_PRUNE_TINY : f == CH_ICH ? ST_PRUNE_ICH : ST_PRUNE_DEGEN]++;
            } else {
                ls.v[ST_PRUNE_DEGEN]++;
            }
        }
        double cand = dps + nvd;
        if (cand < gdd) {
            dist_event(p, sl, it, vd, cand, ls);
            if (vdf & SADDLE_BIT)
                fan_event(p, sl, it, vd, jpo, cand, atan2(iy - dy, ix - dx) - __ldg(&hp->gamma));
        }
    } else {
        ls.v[ST_CREATED]++;
        bool left = cb >= -tolb;  // both rays exit through edge v0-D
        bool ok;
        if (left) {
            ok = ray_seg(ix, iy, b0, 0.0, 0.0, 0.0, dx, dy, sa) &&
                 ray_seg(ix, iy, b1, 0.0, 0.0, 0.0, dx, dy, sb);
        } else {
            ok = ray_seg(ix, iy, b0, 0.0, dx, dy, ell, 0.0, sa) &&
                 ray_seg(ix, iy, b1, 0.0, dx, dy, ell, 0.0, sb);
        }
        if (!ok) {
            ls.v[ST_PRUNE_DEGEN]++;
        } else {
            int f = left ? make_child(jno, lan, 0.0, 0.0, dx, dy, sa, sb, ix, iy, dps, g0, gdd, g1,
                                      ell, 0.0, true, p.eps_win, c[nc])
                         : make_child(jpo, lpv, dx, dy, ell, 0.0, sa, sb, ix, iy, dps, gdd, g1, g0,
                                      0.0, 0.0, false, p.eps_win, c[nc]);
            if (f == CH_STORED) nc++;
            else ls.v[f == CH_TINY ? ST_PRUNE_TINY : f == CH_ICH ? ST_PRUNE_ICH : ST_PRUNE_DEGEN]++;
        }
    }
    return nc;
}

// ---------------------------------------------------------------------------
// k-selection threshold from the key histogram: smallest bin boundary whose
// cumulative count reaches K.  Every CTA computes the identical value.

struct Thresh {
    double t, w_next;
};

__device__ Thresh pick_threshold(const unsigned int *hist, double base, double w, long long K) {
    __shared__ unsigned int s_part[32];
    __shared__ int s_bin;
    __shared__ unsigned long long s_total, s_over;
    constexpr int PER = (NBINS + 255) / 256;  // blockDim is 256
    unsigned int loc[PER];
    unsigned int sum = 0;
    int t = threadIdx.x;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        int b = t * PER + q;
        loc[q] = b < NBINS ? __ldcg(hist + b) : 0u;
        sum += loc[q];
    }
    if (t == 0) {
        s_bin = NBINS;
        s_over = __ldcg(hist + NBINS);
    }
    // block exclusive scan of `sum`
    unsigned int x = sum;
    int lane = t & 31, wid = t >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_part[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned int y = lane < (int)(blockDim.x >> 5) ? s_part[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned int z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        s_part[lane] = y;  // inclusive warp totals
        if (lane == 31) s_total = y;
    }
    __syncthreads();
    unsigned long long before = (unsigned long long)(x - sum) + (wid ? s_part[wid - 1] : 0u);
    unsigned long long cum = before;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        unsigned long long nx = cum + loc[q];
        if (cum < (unsigned long long)K && nx >= (unsigned long long)K) atomicMin(&s_bin, t * PER + q);
        cum = nx;
    }
    __syncthreads();
    Thresh r;
    int b = s_bin;
    if (b < NBINS) {
        r.t = base + (double)(b + 1) * w;
        double f = (double)(b + 1) / (double)(NBINS / 4);
        f = f < 0.5 ? 0.5 : (f > 2.0 ? 2.0 : f);
        r.w_next = w * f;
    } else if (s_over == 0) {
        r.t = INFINITY;  // everything fits: select all
        r.w_next = w;
    } else {
        r.t = base + (double)NBINS * w;  // take the whole range, widen
        r.w_next = w * 4.0;
    }
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// the persistent kernel

__global__ void __launch_bounds__(256) pch_persistent(Params p) {
    Ctrl *ctrl = p.ctrl;
    unsigned int gen = 0;
    LocalStats ls;
    ls.zero();
    WinSoA X = p.X, Y = p.Y;
    double base = 0.0, w = p.w0;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long gthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long t_start = globaltimer();
    int it = 0;
    for (;;) {
        Slot &cur = ctrl->slot[it % 3];
        Slot &prev = ctrl->slot[(it + 2) % 3];
        const unsigned long long nS = *(volatile unsigned long long *)&cur.nS;
        const unsigned long long nP = *(volatile unsigned long long *)&cur.nP;

        // ================= phase A: propagate =================
        if (blockIdx.x == 0) {
            Slot &nxt = ctrl->slot[(it + 1) % 3];
            if (threadIdx.x < sizeof(Slot) / 8)
                reinterpret_cast<unsigned long long *>(&nxt)[threadIdx.x] = 0ull;
            for (int b = threadIdx.x; b <= NBINS; b += blockDim.x) p.hist[(it + 1) & 1][b] = 0u;
            if (threadIdx.x == 0) {
                unsigned long long tot = nS + nP;
                if (tot > ls.v[ST_PEAK]) ls.v[ST_PEAK] = tot;
            }
        }
        unsigned int *hcur = p.hist[it & 1];
        auto emit_child_to_pool = [&](const Win &c) {
            unsigned long long slot = nP + warp_alloc(&cur.nC, true);
            if ((long long)slot < p.cap) {
                store_win(X, slot, c);
                atomicAdd(hcur + key_bin(c.key, base, w), 1u);
            } else {
                atomicExch(&ctrl->error, ERR_OVERFLOW);
            }
            ls.v[ST_STORED]++;
        };
        // deferred saddle fans of iteration it-1: emitted by every event
        // whose candidate equals the committed distance and the per-vertex
        // pick (smallest candidate, then anchor / direction)
        if (it > 0) {
            const unsigned long long nF = *(volatile unsigned long long *)&prev.nF;
            const FanEv *fe = p.fanev[(it - 1) & 1];
            const unsigned long long nFc = nF < (unsigned long long)p.fancap ? nF : p.fancap;
            for (unsigned long long i = gtid; i < nFc; i += gthreads) {
                FanEv e = fe[i];
                double dv = ldcg(p.dist_cur + e.v);
                if (__double_as_longlong(dv) != __double_as_longlong(e.cand)) continue;
                ulonglong2 pk = __ldcg(p.fanpick[(it - 1) & 1] + e.v);
                unsigned long long lo = ((unsigned long long)(uint32_t)e.anchor << 32) | ord_hi32(e.rel);
                if (pk.x != (unsigned long long)__double_as_longlong(e.cand) || pk.y != lo) continue;
                ls.v[ST_FANS]++;
                emit_fan(p, e.v, e.cand, e.anchor, e.rel, false, p.dist_cur, emit_child_to_pool, ls);
            }
        }
        // the selected batch
        {
            const unsigned long long nS_pad = (nS + 31ull) & ~31ull;
            for (unsigned long long i = gtid; i < nS_pad; i += gthreads) {
                Win c[2];
                int nc = 0;
                if (i < nS) {
                    Win win = load_win(p.S, i);
                    nc = propagate(p, cur, it, win, c, ls);
                    if ((unsigned long long)nc > ls.v[ST_MAXCHILD]) ls.v[ST_MAXCHILD] = nc;
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    bool has = q < nc;
                    unsigned long long slot = nP + warp_alloc(&cur.nC, has);
                    if (has) {
                        if ((long long)slot < p.cap) {
                            store_win(X, slot, c[q]);
                            atomicAdd(hcur + key_bin(c[q].key, base, w), 1u);
                        } else {
                            atomicExch(&ctrl->error, ERR_OVERFLOW);
                        }
                        ls.v[ST_STORED]++;
                    }
                }
            }
        }
        grid_barrier(ctrl, gen);

        // ================= phase B: organise =================
        Thresh th = pick_threshold(hcur, base, w, p.K);
        Slot &nxt = ctrl->slot[(it + 1) % 3];
        {
            // commit the shadow tables for entries touched this iteration
            const unsigned long long nTV = *(volatile unsigned long long *)&cur.nTV;
            for (unsigned long long i = gtid; i < nTV; i += gthreads) {
                int32_t v = __ldcg(p.tv_list + i);
                p.dist_cur[v] = __longlong_as_double((long long)__ldcg(p.dist_new + v));
            }
            const unsigned long long nTE = *(volatile unsigned long long *)&cur.nTE;
            for (unsigned long long i = gtid; i < nTE; i += gthreads) {
                int32_t j = __ldcg(p.te_list + i);
                ulonglong2 s = __ldcg(p.split_new + j);
                p.split_cur[j] = make_double2(unord64(s.x), unord64(s.y));
            }
            // fan picks of iteration it-1 are consumed: reset them
            if (it > 0) {
                const unsigned long long nF = *(volatile unsigned long long *)&prev.nF;
                const FanEv *fe = p.fanev[(it - 1) & 1];
                const unsigned long long nFc = nF < (unsigned long long)p.fancap ? nF : p.fancap;
                for (unsigned long long i = gtid; i < nFc; i += gthreads)
                    p.fanpick[(it - 1) & 1][fe[i].v] = make_ulonglong2(~0ull, ~0ull);
            }
        }
        {
            // partition P_i + C_i -> S_{i+1} (key <= t) and P_{i+1}
            const unsigned long long nC = *(volatile unsigned long long *)&cur.nC;
            unsigned long long total = nP + nC;
            if ((long long)total > p.cap) total = p.cap;
            unsigned int *hnext = p.hist[(it + 1) & 1];
            const double nbase = th.t < INFINITY ? th.t : base;
            const unsigned long long tot_pad = (total + 31ull) & ~31ull;
            for (unsigned long long i = gtid; i < tot_pad; i += gthreads) {
                Win c;
                bool valid = i < total;
                if (valid) c = load_win(X, i);
                bool sel = valid && c.key <= th.t;
                bool keep = valid && !sel;
                unsigned long long si = warp_alloc(&nxt.nS, sel);
                unsigned long long pi = warp_alloc(&nxt.nP, keep);
                if (sel) store_win(p.S, si, c);
                if (keep) {
                    store_win(Y, pi, c);
                    atomicAdd(hnext + key_bin(c.key, nbase, th.w_next), 1u);
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (p.max_iter > 0 && it + 1 > p.max_iter) atomicExch(&ctrl->error, ERR_GUARD);
            if (globaltimer() - t_start > p.time_limit_ns) atomicExch(&ctrl->error, ERR_TIMEOUT);
        }
        grid_barrier(ctrl, gen);

        // ================= termination =================
        const int err = *(volatile int *)&ctrl->error;
        const unsigned long long ns = *(volatile unsigned long long *)&nxt.nS;
        const unsigned long long np = *(volatile unsigned long long *)&nxt.nP;
        const unsigned long long nf = *(volatile unsigned long long *)&cur.nF;
        ++it;
        if (err || (ns == 0 && np == 0 && nf == 0)) break;
        WinSoA T = X;
        X = Y;
        Y = T;
        // after a select-all step (t = +inf) keep the old histogram base
        if (th.t < INFINITY) base = th.t;
        w = th.w_next;
    }
    flush_stats(ctrl, ls);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctrl->iterations = it;
        ctrl->t_final = base;
    }
}

// ---------------------------------------------------------------------------
// initialisation kernels

__global__ void k_init_state(Params p, const int64_t *src, int nsrc) {
    const long long n = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long v = t0; v < p.nv; v += n) {
        p.dist_cur[v] = INFINITY;
        p.dist_new[v] = (unsigned long long)__double_as_longlong(INFINITY);
        p.tv_stamp[v] = -1;
        p.fanpick[0][v] = make_ulonglong2(~0ull, ~0ull);
        p.fanpick[1][v] = make_ulonglong2(~0ull, ~0ull);
    }
    for (long long j = t0; j < p.nhe; j += n) {
        p.split_cur[j] = make_double2(INFINITY, 0.0);
        p.split_new[j] = make_ulonglong2(ord64(INFINITY), ord64(0.0));
        p.te_stamp[j] = -1;
    }
    for (long long b = t0; b < 2 * (NBINS + 1); b += n) (b <= NBINS ? p.hist[0][b] : p.hist[1][b - NBINS - 1]) = 0u;
}

__global__ void k_set_sources(Params p, const int64_t *src, int nsrc) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nsrc) {
        int64_t s = src[i];
        p.dist_cur[s] = 0.0;
        p.dist_new[s] = 0ull;
    }
}

// source windows: a full fan around every source (engine.py:402 via
// geom.py:524), into the first batch S_0
__global__ void k_source_windows(Params p, const int64_t *src, int nsrc) {
    LocalStats ls;
    ls.zero();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    Ctrl *ctrl = p.ctrl;
    auto emit = [&](const Win &c) {
        unsigned long long slot = atomicAdd(&ctrl->slot[0].nS, 1ull);
        if ((long long)slot < p.cap) store_win(p.S, slot, c);
        else atomicExch(&ctrl->error, ERR_OVERFLOW);
        ls.v[ST_STORED]++;
    };
    if (i < nsrc) {
        int32_t s = (int32_t)src[i];
        if (__ldg(p.fan_off + s + 1) > __ldg(p.fan_off + s))
            emit_fan(p, s, 0.0, 0, 0.0, true, p.dist_cur, emit, ls);
    }
    flush_stats(ctrl, ls);
}

// ---------------------------------------------------------------------------
// host side

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            return fail(PCH_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
};

}  // namespace

struct pch_mesh {
    int device = 0;
    int32_t nv = 0, nhe = 0;
    double mean_edge = 1.0;
    HeRec *he = nullptr;
    FanRec *fan = nullptr;
    int32_t *fan_off = nullptr, *fanpos = nullptr;
    double *fan_theta = nullptr;
    uint8_t *fan_interior = nullptr;
    size_t mesh_bytes = 0;
    // workspace
    long long cap = 0;
    std::vector<void *> ws;
    Params prm{};
    int64_t *d_src = nullptr;
    size_t src_cap = 0;
    double *d_out = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    int grid = 0;
};

static void free_ws(pch_mesh *m) {
    for (void *q : m->ws) cudaFree(q);
    m->ws.clear();
    m->cap = 0;
}

template <typename T>
static int ws_alloc(pch_mesh *m, T **out, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) return fail(PCH_ERR_NOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
    m->ws.push_back(q);
    *out = static_cast<T *>(q);
    return PCH_OK;
}

static int alloc_soa(pch_mesh *m, WinSoA &W, long long cap) {
    int rc;
    if ((rc = ws_alloc(m, &W.he, cap))) return rc;
    if ((rc = ws_alloc(m, &W.b0, cap))) return rc;
    if ((rc = ws_alloc(m, &W.b1, cap))) return rc;
    if ((rc = ws_alloc(m, &W.d0, cap))) return rc;
    if ((rc = ws_alloc(m, &W.d1, cap))) return rc;
    if ((rc = ws_alloc(m, &W.d, cap))) return rc;
    if ((rc = ws_alloc(m, &W.key, cap))) return rc;
    return PCH_OK;
}

static int ensure_ws(pch_mesh *m, long long cap) {
    if (m->cap >= cap) return PCH_OK;
    free_ws(m);
    Params &p = m->prm;
    int rc;
    p = Params{};
    p.he = m->he;
    p.fan = m->fan;
    p.fan_off = m->fan_off;
    p.fanpos = m->fanpos;
    p.fan_theta = m->fan_theta;
    p.fan_interior = m->fan_interior;
    p.nv = m->nv;
    p.nhe = m->nhe;
    if ((rc = ws_alloc(m, &p.dist_cur, m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.dist_new, m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.split_cur, m->nhe))) return rc;
    if ((rc = ws_alloc(m, &p.split_new, m->nhe))) return rc;
    if ((rc = ws_alloc(m, &p.fanpick[0], m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.fanpick[1], m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.tv_stamp, m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.te_stamp, m->nhe))) return rc;
    if ((rc = ws_alloc(m, &p.tv_list, m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.te_list, m->nhe))) return rc;
    p.fancap = std::max<long long>(cap, 1 << 16);
    if ((rc = ws_alloc(m, &p.fanev[0], p.fancap))) return rc;
    if ((rc = ws_alloc(m, &p.fanev[1], p.fancap))) return rc;
    if ((rc = alloc_soa(m, p.X, cap))) return rc;
    if ((rc = alloc_soa(m, p.Y, cap))) return rc;
    if ((rc = alloc_soa(m, p.S, cap))) return rc;
    if ((rc = ws_alloc(m, &p.hist[0], NBINS + 1))) return rc;
    if ((rc = ws_alloc(m, &p.hist[1], NBINS + 1))) return rc;
    if ((rc = ws_alloc(m, &p.ctrl, 1))) return rc;
    p.cap = cap;
    m->cap = cap;
    return PCH_OK;
}

static int solve(pch_mesh *m, const int64_t *d_src, int nsrc, const pch_config *cfg,
                 cudaStream_t st, pch_stats *stats) {
    if (cfg->k < 1) return fail(PCH_ERR_CONFIG, "k must be >= 1");
    if (!(cfg->epsilon_window > 0.0)) return fail(PCH_ERR_CONFIG, "epsilon_window must be > 0");
    if (cfg->fan_mode != 0 && cfg->fan_mode != 1) return fail(PCH_ERR_CONFIG, "fan_mode must be clip or full_edges");
    long long cap = cfg->pool_capacity > 0 ? cfg->pool_capacity
                                           : std::max<long long>(1 << 20, 2ll * m->nhe);
    if (m->cap > cap) cap = m->cap;
    int regrows = 0;
    for (;;) {
        int rc = ensure_ws(m, cap);
        if (rc) return rc;
        Params p = m->prm;
        p.K = cfg->k;
        p.eps_win = cfg->epsilon_window;
        p.w0 = m->mean_edge / 64.0;
        p.max_iter = cfg->max_iterations;
        p.time_limit_ns = 120ull * 1000000000ull;
        p.fan_full = cfg->fan_mode == 1;
        p.recheck = (cfg->flags & PCH_FLAG_NO_RECHECK) ? 0 : 1;
        CK(cudaEventRecord(m->ev0, st));
        CK(cudaMemsetAsync(p.ctrl, 0, sizeof(Ctrl), st));
        k_init_state<<<4 * 148, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        k_set_sources<<<(nsrc + 255) / 256, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        k_source_windows<<<(nsrc + 255) / 256, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        CK(cudaEventRecord(m->ev1, st));
        void *args[] = {&p};
        CK(cudaLaunchCooperativeKernel((const void *)pch_persistent, dim3(m->grid), dim3(256), args, 0, st));
        CK(cudaEventRecord(m->ev2, st));
        CK(cudaStreamSynchronize(st));
        Ctrl c;
        CK(cudaMemcpy(&c, p.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
        if (c.error == ERR_OVERFLOW) {
            if (cap >= (1ll << 31)) return fail(PCH_ERR_NOMEM, "window pool overflow at maximum capacity");
            cap *= 2;
            regrows++;
            continue;
        }
        if (c.error == ERR_GUARD)
            return fail(PCH_ERR_GUARD, "iteration cap " + std::to_string(cfg->max_iterations) + " exceeded");
        if (c.error == ERR_TIMEOUT) return fail(PCH_ERR_GUARD, "device wall-time guard tripped");
        if (stats) {
            float t_all = 0.f, t_k = 0.f;
            cudaEventElapsedTime(&t_all, m->ev0, m->ev2);
            cudaEventElapsedTime(&t_k, m->ev1, m->ev2);
            stats->iterations += c.iterations;
            stats->windows_propagated += c.st[ST_PROPAGATED];
            stats->total_windows_created += c.st[ST_CREATED];
            stats->pruned_ich += c.st[ST_PRUNE_ICH];
            stats->pruned_split += c.st[ST_PRUNE_SPLIT];
            stats->pruned_tiny += c.st[ST_PRUNE_TINY];
            stats->pruned_degenerate += c.st[ST_PRUNE_DEGEN];
            stats->pruned_recheck += c.st[ST_RECHECK];
            stats->total_windows_pruned += c.st[ST_PRUNE_ICH] + c.st[ST_PRUNE_SPLIT] +
                                           c.st[ST_PRUNE_TINY] + c.st[ST_PRUNE_DEGEN];
            stats->windows_stored += c.st[ST_STORED];
            stats->max_children_per_window = std::max<int64_t>(stats->max_children_per_window, c.st[ST_MAXCHILD]);
            stats->events_created += c.st[ST_EV_CREATED];
            stats->events_applied += c.st[ST_EV_APPLIED];
            stats->peak_active_pool = std::max<int64_t>(stats->peak_active_pool, c.st[ST_PEAK]);
            stats->fans_emitted += c.st[ST_FANS];
            stats->buffer_regrows += regrows;
            stats->time_total_ms += t_all;
            stats->time_kernel_ms += t_k;
        }
        return PCH_OK;
    }
}

// ---------------------------------------------------------------------------
// mesh construction: HeRec / FanRec tables from the SurfaceMesh arrays

static inline int64_t nxt_he(int64_t j) { return 3 * (j / 3) + (j + 1) % 3; }
static inline int64_t prv_he(int64_t j) { return 3 * (j / 3) + (j + 2) % 3; }

extern "C" {

int pch_abi_version(void) { return PCH_ABI_VERSION; }

const char *pch_last_error(void) { return g_err.c_str(); }

int pch_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int pch_mesh_create(const int64_t *origin, const int64_t *opposite, const double *length,
                    const double *corner_angle, const uint8_t *vertex_class,
                    const int64_t *outgoing, int64_t n_vertices, int64_t n_faces,
                    int32_t device, pch_mesh **out) {
    if (!out) return fail(PCH_ERR_MESH, "null output handle");
    *out = nullptr;
    if (n_vertices <= 0 || n_faces <= 0) return fail(PCH_ERR_MESH, "mesh has no faces");
    if (3 * n_faces >= (1ll << 31) || n_vertices >= (1ll << 31))
        return fail(PCH_ERR_MESH, "mesh too large for 32-bit indices");
    const int64_t nhe = 3 * n_faces;
    for (int64_t j = 0; j < nhe; ++j) {
        if (origin[j] < 0 || origin[j] >= n_vertices) return fail(PCH_ERR_MESH, "origin index out of range");
        if (opposite[j] < -1 || opposite[j] >= nhe) return fail(PCH_ERR_MESH, "opposite index out of range");
        if (!(length[j] > 0.0)) return fail(PCH_ERR_MESH, "non-positive edge length");
    }
    std::vector<HeRec> he(nhe);
    double lsum = 0.0;
    auto vflag = [&](int64_t v) -> uint32_t {
        return (uint32_t)v | (vertex_class[v] == 2 ? SADDLE_BIT : 0u);
    };
    for (int64_t j = 0; j < nhe; ++j) {
        HeRec &r = he[j];
        int64_t jn = nxt_he(j), jp = prv_he(j);
        double ell = length[j];
        lsum += ell;
        r.ell = ell;
        r.v0 = vflag(origin[j]);
        r.v1 = vflag(origin[jn]);
        // direction of the source-side apex seen from v1 (geom.py:372-377)
        double lps = length[jp], lns = length[jn];
        double axs = 0.5 * (ell * ell + lps * lps - lns * lns) / ell;
        double ay2 = lps * lps - axs * axs;
        double ays = ay2 > 0.0 ? std::sqrt(ay2) : 0.0;
        r.adir = std::atan2(ays, axs - ell);
        int64_t jo = opposite[j];
        r.jo = (int32_t)jo;
        if (jo >= 0) {
            int64_t jno = nxt_he(jo), jpo = prv_he(jo);
            double lan = length[jno], lpv = length[jpo];
            double dx = 0.5 * (ell * ell + lan * lan - lpv * lpv) / ell;
            double dy2 = lan * lan - dx * dx;
            double dy = dy2 > 0.0 ? -std::sqrt(dy2) : 0.0;
            r.dx = dx;
            r.dy = dy;
            r.lan = lan;
            r.lpv = lpv;
            r.vd = vflag(origin[jpo]);
            r.gamma = std::atan2(-dy, ell - dx);
        } else {
            r.dx = r.dy = r.lan = r.lpv = r.gamma = 0.0;
            r.vd = 0;
        }
        r.pad = 0.0;
    }
    // fan tables: for every vertex walk its outgoing half-edges
    // counterclockwise from outgoing[v] (the clockwise-most one on a
    // boundary, mesh.py:213), accumulating corner angles (geom.py:199-236)
    std::vector<int32_t> fan_off(n_vertices + 1, 0), fanpos(nhe, -1);
    std::vector<double> theta(n_vertices, 0.0);
    std::vector<uint8_t> interior(n_vertices, 0);
    std::vector<FanRec> fan;
    fan.reserve(nhe);
    for (int64_t v = 0; v < n_vertices; ++v) {
        fan_off[v] = (int32_t)fan.size();
        int64_t h = outgoing[v];
        if (h < 0) continue;
        const int64_t start = h;
        double phi = 0.0;
        bool closed = false;
        for (int64_t guard = 0; guard < nhe; ++guard) {
            FanRec f{};
            int64_t che = nxt_he(h), hprev = prv_he(h);
            double li = length[h], lq = length[hprev];
            f.wlo = phi;
            phi += corner_angle[h];
            f.whi = phi;
            f.px = li * std::cos(f.wlo);
            f.py = li * std::sin(f.wlo);
            f.qx = lq * std::cos(f.whi);
            f.qy = lq * std::sin(f.whi);
            f.lc = length[che];
            f.che = (int32_t)che;
            f.pid = (int32_t)origin[che];
            f.qid = (int32_t)origin[hprev];
            fanpos[h] = (int32_t)(fan.size() - fan_off[v]);
            fan.push_back(f);
            int64_t o = opposite[hprev];
            if (o < 0) break;
            h = o;
            if (h == start) {
                closed = true;
                break;
            }
        }
        theta[v] = phi;
        interior[v] = closed ? 1 : 0;
    }
    fan_off[n_vertices] = (int32_t)fan.size();
    for (int64_t j = 0; j < nhe; ++j)
        if (fanpos[j] < 0) return fail(PCH_ERR_MESH, "half-edge not reachable in its vertex fan (non-manifold vertex)");

    pch_mesh *m = new pch_mesh();
    m->device = device;
    m->nv = (int32_t)n_vertices;
    m->nhe = (int32_t)nhe;
    m->mean_edge = lsum / (double)nhe;
    auto cleanup = [&](int code, const std::string &msg) {
        pch_mesh_destroy(m);
        return fail(code, msg);
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cleanup(PCH_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t r = cudaMalloc(dst, std::max<size_t>(bytes, 16));
        if (r != cudaSuccess) return r;
        m->mesh_bytes += bytes;
        return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    };
    if ((e = up((void **)&m->he, he.data(), sizeof(HeRec) * nhe)) != cudaSuccess ||
        (e = up((void **)&m->fan, fan.data(), sizeof(FanRec) * fan.size())) != cudaSuccess ||
        (e = up((void **)&m->fan_off, fan_off.data(), sizeof(int32_t) * fan_off.size())) != cudaSuccess ||
        (e = up((void **)&m->fanpos, fanpos.data(), sizeof(int32_t) * nhe)) != cudaSuccess ||
        (e = up((void **)&m->fan_theta, theta.data(), sizeof(double) * n_vertices)) != cudaSuccess ||
        (e = up((void **)&m->fan_interior, interior.data(), n_vertices)) != cudaSuccess)
        return cleanup(PCH_ERR_CUDA, std::string("mesh upload: ") + cudaGetErrorString(e));
    if ((e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreate(&m->ev0)) != cudaSuccess || (e = cudaEventCreate(&m->ev1)) != cudaSuccess ||
        (e = cudaEventCreate(&m->ev2)) != cudaSuccess)
        return cleanup(PCH_ERR_CUDA, std::string("stream/event: ") + cudaGetErrorString(e));
    int nsm = 0, per_sm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pch_persistent, 256, 0);
    if (per_sm < 1) return cleanup(PCH_ERR_CUDA, "persistent kernel cannot be resident");
    m->grid = nsm * std::min(per_sm, 4);
    *out = m;
    return PCH_OK;
}

int pch_mesh_destroy(pch_mesh *m) {
    if (!m) return PCH_OK;
    cudaSetDevice(m->device);
    free_ws(m);
    cudaFree(m->he);
    cudaFree(m->fan);
    cudaFree(m->fan_off);
    cudaFree(m->fanpos);
    cudaFree(m->fan_theta);
    cudaFree(m->fan_interior);
    cudaFree(m->d_src);
    cudaFree(m->d_out);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    if (m->ev2) cudaEventDestroy(m->ev2);
    if (m->stream) cudaStreamDestroy(m->stream);
    delete m;
    return PCH_OK;
}

int64_t pch_mesh_device_bytes(const pch_mesh *m) { return m ? (int64_t)m->mesh_bytes : 0; }

static int check_sources(const pch_mesh *m, const int64_t *sources, int64_t n) {
    if (n <= 0) return fail(PCH_ERR_SOURCE, "at least one source vertex is required");
    for (int64_t i = 0; i < n; ++i)
        if (sources[i] < 0 || sources[i] >= m->nv)
            return fail(PCH_ERR_SOURCE, "invalid source index " + std::to_string(sources[i]));
    return PCH_OK;
}

static int stage_sources(pch_mesh *m, const int64_t *sources, int64_t n) {
    if ((size_t)n > m->src_cap) {
        cudaFree(m->d_src);
        m->d_src = nullptr;
        CK(cudaMalloc(&m->d_src, sizeof(int64_t) * n));
        m->src_cap = n;
    }
    CK(cudaMemcpyAsync(m->d_src, sources, sizeof(int64_t) * n, cudaMemcpyHostToDevice, m->stream));
    return PCH_OK;
}

int pch_run(pch_mesh *m, const int64_t *sources, int64_t n_sources, const pch_config *cfg,
            double *out_dist, pch_stats *stats) {
    if (!m || !cfg || !out_dist) return fail(PCH_ERR_CONFIG, "null argument");
    int rc = check_sources(m, sources, n_sources);
    if (rc) return rc;
    CK(cudaSetDevice(m->device));
    if ((rc = stage_sources(m, sources, n_sources))) return rc;
    if ((rc = solve(m, m->d_src, (int)n_sources, cfg, m->stream, stats))) return rc;
    CK(cudaMemcpyAsync(out_dist, m->prm.dist_cur, sizeof(double) * m->nv, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return PCH_OK;
}

int pch_run_device(pch_mesh *m, const int64_t *d_sources, int64_t n_sources, const pch_config *cfg,
                   double *d_out, void *stream, pch_stats *stats) {
    if (!m || !cfg || !d_out || !d_sources) return fail(PCH_ERR_CONFIG, "null argument");
    if (n_sources <= 0) return fail(PCH_ERR_SOURCE, "at least one source vertex is required");
    CK(cudaSetDevice(m->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : m->stream;
    int rc = solve(m, d_sources, (int)n_sources, cfg, st, stats);
    if (rc) return rc;
    CK(cudaMemcpyAsync(d_out, m->prm.dist_cur, sizeof(double) * m->nv, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return PCH_OK;
}

int pch_run_rows(pch_mesh *m, const int64_t *sources, int64_t n_sources, const pch_config *cfg,
                 double *out_rows, pch_stats *stats) {
    if (!m || !cfg || !out_rows) return fail(PCH_ERR_CONFIG, "null argument");
    int rc = check_sources(m, sources, n_sources);
    if (rc) return rc;
    CK(cudaSetDevice(m->device));
    if ((rc = stage_sources(m, sources, n_sources))) return rc;
    for (int64_t r = 0; r < n_sources; ++r) {
        if ((rc = solve(m, m->d_src + r, 1, cfg, m->stream, stats))) return rc;
        CK(cudaMemcpyAsync(out_rows + r * (int64_t)m->nv, m->prm.dist_cur, sizeof(double) * m->nv,
                           cudaMemcpyDeviceToHost, m->stream));
    }
    CK(cudaStreamSynchronize(m->stream));
    return PCH_OK;
}

}  // extern "C"
