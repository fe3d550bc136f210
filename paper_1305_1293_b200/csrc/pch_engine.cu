// pch_engine.cu -- B200-native Parallel Chen-Han exact geodesic solver.
//
// A persistent cooperative kernel runs the whole PCH loop (paper
// Algorithm 1; reference pkg/src/pargeo/engine.py:433 run_pch) on the
// device, so the per-level CPU/GPU synchronisation the paper identifies as
// the CH bottleneck never happens.  Two solvers share the window geometry
// (pch_device.cuh, reference geom.py) and the event primitives:
//
//   pch_live (default)   one phase + one grid barrier per iteration: the
//            next threshold is fixed up front by a step controller (about
//            one face layer per crossing), every produced window is routed
//            to the next batch or the pool as it is produced (into the
//            CTA's own chunk, one shared atomic per warp; chunk prefix
//            tables rebuilt after the barrier), the filters read the tables
//            the events update atomically, and a child inside the next
//            threshold is propagated at once by the same thread (chaining,
//            up to 3 crossings per iteration).  Also solves R fields at
//            once (batched rows, pch_run_rows) and seeded fields
//            (farthest-point sampling, pch_fps).
//   pch_persistent (PCH_FLAG_DETERMINISTIC)   two phases per iteration:
//            propagation against tables frozen at the start of the
//            iteration, then commit + histogram k-selection + partition
//            (paper Algorithm 3) -- bitwise reproducible.
//
// In both, events replace the paper's sort-then-first-wins pass
// (Algorithm 4; engine.py:341/:359) by order-independent atomics: 64-bit
// atomicMin on the fp64 bit patterns of the distance field, 128-bit
// CAS-min of (comp, entry_x) on the angle-split table, and a per-vertex
// CAS-min pick so each improved saddle fans out once.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pch_b200.h"
#include "pch_device.cuh"

using namespace pch;

// ---------------------------------------------------------------------------
// device state

enum { // the ten hot counters first: packed per thread (LocalStats)
       ST_PROPAGATED, ST_CREATED, ST_PRUNE_ICH, ST_PRUNE_SPLIT, ST_RECHECK, ST_STORED,
       ST_EV_CREATED, ST_EV_APPLIED, ST_PRUNE_TINY, ST_PRUNE_DEGEN, ST_N_PACKED,
       ST_FANS = ST_N_PACKED, ST_PRUNE_DUP, ST_BARRIERS, ST_MAXCHILD, ST_PEAK,
       // PCH_PROFILE section clocks (clock64 deltas summed over threads)
       ST_CYC_PROP, ST_CYC_POOL, ST_CYC_FANSPAN, ST_CYC_FANITEM,
       ST_CYC_PART, ST_N_POOL, ST_N_PART, ST_N_FANITEM, ST_CAS_ANGLE_CALLS, ST_CAS_ANGLE_TRIES, ST_CAS_FAN_CALLS, ST_CAS_FAN_TRIES,
       // phase attribution of the one-barrier solver (warp cycles, lane 0):
       // the reference's RunStats.time_select / _propagate / _compact /
       // _events (engine.py:470-473) as shares of the kernel time
       ST_PH_SELECT, ST_PH_PROP, ST_PH_COMPACT, ST_PH_EVENTS, ST_N_SITEM, N_ST };

enum { ERR_NONE = 0, ERR_OVERFLOW = 1, ERR_GUARD = 2, ERR_TIMEOUT = 3, ERR_SOURCE = 4 };

struct Slot {                // per-iteration counters (ring of NSLOT)
    unsigned long long nS;   // size of the selected batch S
    unsigned long long nP;   // size of the pool P
    unsigned long long nC;   // children appended (two-barrier kernel)
    unsigned long long nTV;  // touched vertices (two-barrier kernel)
    unsigned long long nTE;  // touched angle entries (two-barrier kernel)
    unsigned long long nF;   // fan events
    unsigned long long pmin; // smallest key in P, fp64 bits (one-barrier kernel)
    unsigned long long smax; // largest key in S, fp64 bits (one-barrier kernel)
};
constexpr int NSLOT = 4;

struct Ctrl {
    Slot slot[NSLOT];
    unsigned long long lat_hist[64];  // PCH_PROFILE: log2 histogram of propagation cycles
    unsigned int bar_count;
    unsigned int bar_gen;
    int error;
    int pad0;
    long long iterations;
    unsigned long long st[N_ST];
    double t_final;
    int final_parity;  // which of X/Y held the last pool (unused on exit)
    int grow;          // live solver: a chunk passed its soft limit -> stop at the iteration end, grow, resume
    long long res_it;  // ... the iteration to resume at, its threshold and controller step
    double res_t, res_delta;
};

struct Params {
    // mesh (immutable)
    const FaceRec *face;       // [F]
    const FanRec *fan;
    const FanHdr *fanhdr;      // [nv] wedge range, total angle, interior flag
    const double *anchor_wlo;  // [nhe] start angle of h's wedge in origin(h)'s fan
    const double2 *apex_xy;    // [nhe] apex of face(h) unfolded in the frame of edge h (geom.py:390-396)
    int32_t nv, nhe;
    // distance field / angle-split table: frozen + shadow copies
    double *dist_cur;
    unsigned long long *dist_new;
    double2 *split_cur;        // (comp, entry_x)
    ulonglong2 *split_new;     // (ord(comp), ord(entry_x))
    ulonglong2 *fanpick[3];    // per vertex (cand bits, anchor<<32 | ord32(rel)), by iteration % 3
    int32_t *tv_list, *te_list;
    long long tvcap, tecap;
    FanEv *fanev[3];           // saddle fan candidates, by iteration % 3
    long long fancap;
    // window pools
    WinSoA X, Y, S, S2;        // pools (X/Y) and batches (S/S2); the one-barrier
                               // kernel double-buffers S/S2 and P = X/Y
    long long cap;
    unsigned int *hist[2];     // NBINS + 1 bins each
    unsigned int *fine[2];     // exact selection: every bin's NBINS sub-bins (+1 spare), by parity
    int exact_select;          // selection_mode "exact" (two-level k-selection) vs "approximate_strided"
    Ctrl *ctrl;
    // config
    long long K;
    double eps_win;
    double inv_r0;             // 1 / radius of the angular tiny-window rule (huge: absolute)
    double eps_win2, inv_r02;  // their squares (make_child compares squared)
    double fan_widen;          // saddle-fan interval widened by this angle on both sides
    int phase;                 // attribute cycles to the four phases (PCH_FLAG_PHASE_TIMES)
    int resume;                // live solver: continue at ctrl->res_it after a pool growth
    int local_iters;           // live solver: iterations per grid barrier (the others CTA-local)
    ulonglong2 *dup_tab;       // fan-window fingerprints of the current iteration (dedupe)
    unsigned long long dup_mask;  // table slots - 1 (power of two)
    unsigned int dup_epoch;    // solve sequence << 20: + iteration = the entries' epoch
    double w0;
    double delta0, delta_min, delta_max;  // one-barrier step controller
    long long max_iter;
    unsigned long long time_limit_ns;
    int fan_full;
    int recheck;
    int live;                  // filters read the live shadow tables
    int prof;                  // PCH_PROFILE: accumulate per-section clocks
    int chain;                 // max propagations a thread chains per iteration
    int rows;                  // distance fields solved together (batched rows)
    unsigned int *ccnt;        // live solver: per-CTA output counts [2 parity][S, P, fans][MAX_CTAS]
    int live_grid;             // CTAs of the live solver's launch (chunk count)
    const double *seed;        // optional initial field (farthest-point sampling), else +inf
    unsigned long long *trace; // optional per-iteration timeline (TR_* records)
    long long trace_cap;       // iterations the trace buffer holds
};

// per-iteration trace record (PCH_TRACE=path): globaltimer stamps and sizes
enum { TR_T0, TR_A_END, TR_B1, TR_B_END, TR_B2, TR_NS, TR_NP, TR_NC, TR_NF, TR_NTV, TR_TSEL_BITS,
       TR_FAN_END, TR_START_MAX, TR_WORK_END, TR_SCAN_END, TR_TRIP0, TR_LOADED, TR_ROUTED, TR_N };

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

// Grid-wide barrier for a cooperative launch (all CTAs co-resident): one
// monotonically increasing arrival counter, no separate release step --
// thread 0 of each CTA adds its arrival (release) and spins (acquire) until
// the counter reaches gen * gridDim.  `after` runs on thread 0 between the
// spin and the closing __syncthreads (used to read the iteration's
// counters once per CTA).  A waiter that sees no progress within 20 s
// flags ERR_TIMEOUT instead of hanging.
template <bool LeadingSync = true, typename After>
__device__ __forceinline__ void grid_barrier(Ctrl *c, unsigned int &gen, After &&after) {
    if (LeadingSync) __syncthreads();
    if (threadIdx.x == 0) {
        gen += 1;
        const unsigned int target = gen * gridDim.x;
        // release (cumulative over the CTA's writes ordered by the
        // __syncthreads above) / acquire pairing: no separate fences
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&c->bar_count), "r"(1u) : "memory");
        unsigned int spins = 0;
        unsigned long long t0 = 0;
        while ((int)(ld_acquire_u32(&c->bar_count) - target) < 0) {
            if ((++spins & 1023u) == 0u) {
                if (t0 == 0) t0 = globaltimer();
                else if (globaltimer() - t0 > 20000000000ull) {
                    atomicExch(&c->error, ERR_TIMEOUT);
                    break;
                }
            }
        }
        after();
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(Ctrl *c, unsigned int &gen) {
    grid_barrier(c, gen, [] {});
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

// The tables of one distance field.  Batched rows (pch_run_rows) solve R
// independent single-source fields in one kernel: every window carries its
// field's row, and the distance field / angle-split table / fan picks of
// row r live at offset r * (V or 3F) -- the mesh is shared.
struct RowTabs {
    unsigned long long *dist;  // fp64 bit patterns (live shadow field)
    ulonglong2 *split;         // (ord(comp), ord(entry_x))
    ulonglong2 *pick;          // fan picks
};

// LIVE: 1 / 0 when the caller is the one- / two-barrier solver (the
// other solver's branches then compile away), -1 to read p.live
template <int LIVE = -1>
__device__ __forceinline__ RowTabs row_tabs(const Params &p, uint32_t r, int it) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    RowTabs t;
    t.dist = p.dist_new + (size_t)r * p.nv;
    t.split = p.split_new + (size_t)r * p.nhe;
    t.pick = p.fanpick[live ? 0 : it % 3] + (size_t)r * p.nv;
    return t;
}

// distance / angle-split reads of the filters: the iteration-frozen copy
// (deterministic solver, one row), or the shadow tables the events update
// atomically.  Any value read is the length of a real path, so a stale or
// racing read only weakens pruning; it never admits a wrong distance.
template <int LIVE = -1>
__device__ __forceinline__ double gdist(const Params &p, const RowTabs &t, int32_t v) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    if (live) return __longlong_as_double((long long)__ldcg(t.dist + v));
    return __ldcg(p.dist_cur + v);
}
// the angle-split entry as ord64 bits (the CAS guess), converted where it
// is used: keeping the conversion away from the load lets the load's
// latency overlap the unfolding and both children's geometry
template <int LIVE = -1>
__device__ __forceinline__ ulonglong2 gsplit_raw(const Params &p, const RowTabs &t, int32_t j) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    if (live) {
        // single-copy-atomic 128-bit read (a strong .b128 load): the pair is
        // never torn between two claims' CAS writes
        unsigned long long lo, hi;
        asm volatile("{\n\t.reg .b128 t;\n\tld.relaxed.gpu.global.b128 t, [%2];\n\tmov.b128 {%0, %1}, t;\n\t}"
                     : "=l"(lo), "=l"(hi)
                     : "l"(t.split + j)
                     : "memory");
        return make_ulonglong2(lo, hi);
    }
    // the frozen entry is the shadow entry's value at the start of the
    // iteration: the best first guess for a CAS on it
    const double2 s = __ldcg(p.split_cur + j);
    return make_ulonglong2(ord64(s.x), ord64(s.y));
}

__device__ __forceinline__ int key_bin(double key, double base, double w) {
    double f = (key - base) / w;
    if (!(f >= 0.0)) return 0;
    if (f >= (double)NBINS) return NBINS;
    return (int)f;
}

// exact selection (two-barrier solver): the key's sub-bin inside its
// coarse bin cb, counted as the key is histogrammed -- the bin that holds
// the K-th key is then refined without a second pass over the keys and a
// second grid barrier.  Same lo / sub-width arithmetic as a refinement
// pass over that bin.
constexpr size_t FINE_ROW = NBINS + 1;
constexpr size_t FINE_N = (size_t)NBINS * FINE_ROW;
__device__ __forceinline__ void fine_add(unsigned int *fine, double key, double base, double w, int cb) {
    if (cb >= NBINS) return;
    const double lo = base + (double)cb * w, sw = w / (double)NBINS;
    const double f = (key - lo) / sw;
    if (f >= 0.0 && f < (double)NBINS) atomicAdd(fine + (size_t)cb * FINE_ROW + (int)f, 1u);
}

__device__ __forceinline__ void store_win(const WinSoA &W, unsigned long long i, const Win &c) {
    W.hv[i] = make_int4(c.he, c.jo, (int)c.v0f, (int)c.v1f);
    W.vr[i] = make_uint2(c.vdf, c.row);
    W.b0[i] = c.b0;
    W.b1[i] = c.b1;
    W.d0[i] = c.d0;
    W.d1[i] = c.d1;
    W.d[i] = c.d;
    W.key[i] = c.key;
}

__device__ __forceinline__ Win load_win(const WinSoA &W, unsigned long long i) {
    Win c;
    const int4 hv = __ldcg(W.hv + i);
    c.he = hv.x;
    c.jo = hv.y;
    c.v0f = (uint32_t)hv.z;
    c.v1f = (uint32_t)hv.w;
    const uint2 vr = __ldcg(W.vr + i);
    c.vdf = vr.x;
    c.row = vr.y;
    c.b0 = __ldcg(W.b0 + i);
    c.b1 = __ldcg(W.b1 + i);
    c.d0 = __ldcg(W.d0 + i);
    c.d1 = __ldcg(W.d1 + i);
    c.d = __ldcg(W.d + i);
    c.key = __ldcg(W.key + i);
    return c;
}

// Run counters.  The ten hot ones (ST_PROPAGATED .. ST_PRUNE_DEGEN) are
// packed as 16-bit fields into three per-thread registers and folded into
// the CTA's shared counters when any field passes 2^15 and at exit (one
// warp reduction per field, one shared atomic per nonzero field from lane
// 0): a shared-memory atomic per increment serialises the propagation path
// (measured ~25% of the solve).  A trip adds at most 4 per chained
// propagation (3 distance + 1 angle event) to a field, far below the 2^15
// headroom, so a fold is needed only every few thousand trips -- folding
// on a fixed short period had cost 0.24 ms of the 1M-face field.  The
// tiny / degenerate prunes are packed too (as shared atomics under a branch
// they cost every crossing a divergent region); the rare ones (fans, dup
// prunes), profiling clocks, maxima and `direct` objects go straight to
// shared memory, only when nonzero.
struct LocalStats {
    unsigned long long *s;
    bool direct;
    unsigned long long a = 0ull, b = 0ull, c = 0ull;
    __device__ __forceinline__ void add(int i, unsigned long long x = 1ull) {
        if (!direct && i <= 3) {
            a += x << (16 * i);
        } else if (!direct && i <= 7) {
            b += x << (16 * (i - 4));
        } else if (!direct && i < ST_N_PACKED) {
            c += x << (16 * (i - 8));
        } else if (x) {
            atomicAdd(s + i, x);
        }
    }
    __device__ __forceinline__ void max(int i, unsigned long long x) { atomicMax(s + i, x); }
    // some lane of the (converged) warp is past half of a field's range
    __device__ __forceinline__ bool fold_due() const {
        return __any_sync(0xffffffffu, ((a | b | c) & 0x8000800080008000ull) != 0ull);
    }
    // fold the packed fields into shared memory (whole warp, converged):
    // one warp reduction per field, lane 0 adds the nonzero sums
    __device__ __forceinline__ void fold() {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 0; k < ST_N_PACKED; ++k) {
            const unsigned long long w = k <= 3 ? a : k <= 7 ? b : c;
            const unsigned int f = __reduce_add_sync(0xffffffffu, (unsigned int)((w >> (16 * (k & 3))) & 0xffffull));
            if (lane == 0 && f) atomicAdd(s + k, (unsigned long long)f);
        }
        a = b = c = 0ull;
    }
};

__device__ __forceinline__ void stats_init(unsigned long long *s) {
    for (int i = threadIdx.x; i < N_ST; i += blockDim.x) s[i] = 0ull;
    __syncthreads();
}

__device__ __forceinline__ void flush_stats(Ctrl *c, unsigned long long *s) {
    __syncthreads();
    for (int i = threadIdx.x; i < N_ST; i += blockDim.x) {
        unsigned long long x = s[i];
        if (!x) continue;
        if (i == ST_MAXCHILD || i == ST_PEAK) atomicMax(&c->st[i], x);
        else atomicAdd(&c->st[i], x);
    }
}

// ---------------------------------------------------------------------------
// events
//
// Events are applied on the spot with order-independent atomics (64-bit
// atomicMin on the fp64 bit pattern of a positive distance, 128-bit CAS-min
// on the angle-split pair), so the result does not depend on which thread
// wins a race.  The bookkeeping they need -- which vertices / angles the
// iteration touched, which saddles should fan out -- is staged in shared
// memory and flushed by the CTA once per trip with one global atomic per
// list: no hot global counter sits on the propagation path.

#ifndef PCH_TPB
#define PCH_TPB 256
#endif
constexpr int TPB = PCH_TPB;      // threads per CTA of every solver kernel
constexpr int NWARP = TPB / 32;
constexpr double DELTA_FLOOR = 0.45;  // controller step floor, mean edge lengths
constexpr double DELTA_CAP = 0.75;    // controller step cap, mean edge lengths
constexpr double DELTA_CAP_LONG = 0.6;  // ... with chains longer than DEFAULT_CHAIN
constexpr double ALT_FLOOR = 1.0;     // ... and floor <= this many mean face altitudes
constexpr int LONG_CHAIN_FACES = 1 << 18;  // meshes this large chain one more crossing
constexpr unsigned int LIGHT_PER_WARP = 4;  // light work items per warp before batch warps take some
constexpr int DEFAULT_CHAIN = 2;      // propagations a thread may chain per iteration
constexpr int ANISO_CHAIN = 6;        // ... on large anisotropic meshes
constexpr int LOCAL_ITERS = 12;       // live solver: iterations per grid barrier (single fields)
constexpr int LOCAL_ITERS_ROWS = 8;   // ... batched rows
constexpr int DEFAULT_ROWS = 32;
constexpr long long DUP_SLOTS = 1ll << 21;  // fan-window dedupe table (32 MB)
#ifndef PCH_POOL_MIN
#define PCH_POOL_MIN (1ll << 21)
#endif
constexpr long long DEFAULT_POOL_MIN = PCH_POOL_MIN;  // first window-pool capacity (at least)
constexpr double TINY_R0_EDGES = 40.0;  // angular tiny-window radius, mean edge lengths      // fields pch_run_rows solves together (at most)
constexpr int MAX_CTAS = 1024;        // chunk-count tables of the live solver
constexpr int FAN_LANES = 8;      // lanes per saddle fan (wedges x repetitions)
constexpr int FANS_PER_WARP = 32 / FAN_LANES;

constexpr int FE_CAP = 2 * TPB;



// development instrumentation (PCH_TRACE timelines, PCH_PROFILE clocks) of
// the solvers: compiled in only with -DPCH_DEVTOOLS, so the
// default kernels carry no checks for it
#ifdef PCH_DEVTOOLS
#define DEV_TRACE (p.trace != nullptr)
#define DEV_PROF (p.prof != 0)
#else
#define DEV_TRACE false
#define DEV_PROF false
#endif

struct Stage {
    unsigned int ntv, nte, nfe, pad;
    int32_t tv[3 * TPB];  // improved vertices (<= 3 per propagation)
    int32_t te[TPB];      // improved angle-split entries (<= 1)
    FanEv fe[FE_CAP];     // saddle fan candidates (overflow appends directly)
};

template <int LIVE = -1>
__device__ __forceinline__ void dist_event(const Params &p, const RowTabs &t, Stage &sg, int32_t v,
                                           double cand, LocalStats &ls) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    // the caller checked cand against the distance it read; the minimum
    // itself needs no reply (RED), the vertex is listed for the commit
    ls.add(ST_EV_CREATED);
    atomicMin(t.dist + v, (unsigned long long)__double_as_longlong(cand));
    if (!live) {
        unsigned int k = atomicAdd(&sg.ntv, 1u);
        sg.tv[k] = v;
    }
    ls.add(ST_EV_APPLIED);
}

template <int LIVE = -1>
__device__ __forceinline__ void angle_event(const Params &p, const RowTabs &t, Stage &sg, int32_t j,
                                            double comp, double entry, ulonglong2 guess, LocalStats &ls) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    ls.add(ST_EV_CREATED);
    if (live) {
        // live solver: one CAS attempt, reply unused (off the propagation's
        // critical path).  A lost race leaves the entry at a value that is
        // still smaller than the one read -- a window that kept both its
        // children -- so it is a valid dominator for the one-angle-one-split
        // rule; losing only weakens pruning, never correctness.
        if (ord64(comp) < guess.x || (ord64(comp) == guess.x && ord64(entry) < guess.y)) {
            atomicCAS(t.split + j, guess, make_ulonglong2(ord64(comp), ord64(entry)));
            ls.add(ST_EV_APPLIED);
        }
        return;
    }
    int tries = 0;
    const bool won = cas_min_u128(t.split + j, ord64(comp), ord64(entry), guess, &tries);
    if (DEV_PROF) {
        atomicAdd(&p.ctrl->st[ST_CAS_ANGLE_CALLS], 1ull);
        atomicAdd(&p.ctrl->st[ST_CAS_ANGLE_TRIES], (unsigned long long)tries);
    }
    if (won) {
        if (!live) {
            unsigned int k = atomicAdd(&sg.nte, 1u);
            sg.te[k] = j;
        }
        ls.add(ST_EV_APPLIED);
    }
}

template <int LIVE = -1, typename FanSink>
__device__ __forceinline__ void fan_event(const Params &p, const RowTabs &t, uint32_t row, FanSink &&sink,
                                          ulonglong2 guess, int32_t v, int32_t anchor,
                                          double cand, double ax, double ay, double bx, double by) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    FanEv e;
    e.v = v;
    e.row = row;
    e.pad = 0u;
    e.anchor = anchor;
    e.cand = cand;
    e.ax = ax;
    e.ay = ay;
    e.bx = bx;
    e.by = by;
    // per-vertex pick (smallest candidate, then anchor / direction) by
    // 128-bit CAS-min: ties are common (the same pseudo source reaching a
    // saddle through several windows) and every tying event would emit the
    // same fan (the reference dedupes those rows, engine.py:201).  The
    // deterministic solver resets the picks every iteration; the live one
    // never does (a new candidate is always strictly smaller) and seeds the
    // CAS with the pick it read.
    const unsigned long long hi = (unsigned long long)__double_as_longlong(cand);
    const unsigned long long lo = fan_tiebreak(e);
    if (live) {
        // one attempt, reply unused (no wait on the propagation path): if
        // it loses a race against a worse candidate, the winner check of
        // the next iteration finds the pick stale and repairs it
        if (hi < guess.x || (hi == guess.x && lo < guess.y))
            atomicCAS(t.pick + v, guess, make_ulonglong2(hi, lo));
    } else {
        int tries = 0;
        cas_min_u128(t.pick + v, hi, lo, guess, &tries);
        if (DEV_PROF) {
            atomicAdd(&p.ctrl->st[ST_CAS_FAN_CALLS], 1ull);
            atomicAdd(&p.ctrl->st[ST_CAS_FAN_TRIES], (unsigned long long)tries);
        }
    }
    sink(e);
}

// fan candidates of the deterministic solver: staged in shared memory and
// flushed by the CTA per trip (trip_flush); overflow appends directly
struct StageFanSink {
    const Params &p;
    Stage &sg;
    unsigned long long *nf_glob;
    FanEv *fe_out;
    __device__ __forceinline__ void operator()(const FanEv &e) const {
        const unsigned int k = atomicAdd(&sg.nfe, 1u);
        if (k < (unsigned int)FE_CAP) {
            sg.fe[k] = e;
        } else {
            atomicSub(&sg.nfe, 1u);
            const unsigned long long at = atomicAdd(nf_glob, 1ull);
            if ((long long)at < p.fancap) fe_out[at] = e;
            else atomicExch(&p.ctrl->error, ERR_OVERFLOW);
        }
    }
};

// End of one trip of the selected batch (uniform over the CTA): reserve
// `n` (<= 2) pool slots per thread for the children with one global
// atomicAdd per CTA, and flush the staged event lists with one atomicAdd
// per list, all issued back to back by one thread.  Returns the thread's
// first child slot relative to the pool's child counter.
__device__ unsigned int block_excl_scan(unsigned int x, unsigned int &total);

__device__ __forceinline__ unsigned long long trip_flush(const Params &p, Stage &sg, Slot &sl, int it,
                                                        unsigned int n) {
    __shared__ unsigned long long s_b[4];
    unsigned int total;
    const unsigned int excl = block_excl_scan(n, total);  // all staging of the trip is done
    if (threadIdx.x == 0) {
        s_b[0] = sg.ntv ? atomicAdd(&sl.nTV, (unsigned long long)sg.ntv) : 0ull;
        s_b[1] = sg.nte ? atomicAdd(&sl.nTE, (unsigned long long)sg.nte) : 0ull;
        s_b[2] = sg.nfe ? atomicAdd(&sl.nF, (unsigned long long)min(sg.nfe, (unsigned int)FE_CAP)) : 0ull;
        s_b[3] = total ? atomicAdd(&sl.nC, (unsigned long long)total) : 0ull;
    }
    __syncthreads();
    const unsigned int ntv = sg.ntv, nte = sg.nte, nfe = min(sg.nfe, (unsigned int)FE_CAP);
    for (unsigned int k = threadIdx.x; k < ntv; k += TPB) {
        unsigned long long at = s_b[0] + k;
        if ((long long)at < p.tvcap) p.tv_list[at] = sg.tv[k];
        else atomicExch(&p.ctrl->error, ERR_OVERFLOW);
    }
    for (unsigned int k = threadIdx.x; k < nte; k += TPB) {
        unsigned long long at = s_b[1] + k;
        if ((long long)at < p.tecap) p.te_list[at] = sg.te[k];
        else atomicExch(&p.ctrl->error, ERR_OVERFLOW);
    }
    for (unsigned int k = threadIdx.x; k < nfe; k += TPB) {
        unsigned long long at = s_b[2] + k;
        if ((long long)at < p.fancap) p.fanev[p.live ? (it & 1) : it % 3][at] = sg.fe[k];
        else atomicExch(&p.ctrl->error, ERR_OVERFLOW);
    }
    const unsigned long long rel = s_b[3] + excl;
    __syncthreads();
    if (threadIdx.x == 0) sg.ntv = sg.nte = sg.nfe = 0u;
    __syncthreads();
    return rel;
}

// exclusive block-wide prefix sum of x; *total receives the CTA total
// (uniform: contains __syncthreads)
__device__ unsigned int block_excl_scan(unsigned int x, unsigned int &total) {
    __shared__ unsigned int s_w[NWARP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned int y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
    }
    if (lane == 31) s_w[wid] = y;
    __syncthreads();
    if (wid == 0) {
        unsigned int t = lane < NWARP ? s_w[lane] : 0u;
#pragma unroll
        for (int o = 1; o < NWARP; o <<= 1) {
            unsigned int z = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += z;
        }
        if (lane < NWARP) s_w[lane] = t;
    }
    __syncthreads();
    unsigned int excl = y - x + (wid ? s_w[wid - 1] : 0u);
    total = s_w[NWARP - 1];
    __syncthreads();
    return excl;
}

// ---------------------------------------------------------------------------
// saddle fans (geom.py:185): windows with pseudo source v on the edges
// opposite v inside the fan spanned by the two straight extensions of the
// incoming ray; `full` emits every wedge (source initialisation).

struct FanSpan {
    int32_t off, m;  // wedge records of v: fan[off, off + m)
    int reps;        // 2 when the fan interval may wrap around an interior vertex
    double theta, flo, fhi;
};

// Exact-duplicate removal (reference engine.py:201 dedupe_rows, applied
// to every compacted block at :461), on request (PCH_FLAG_DEDUPE): the
// per-vertex fan pick already keeps all but ties from fanning out twice,
// so twins are rare here (3.3k of 20M windows on terrain1m, 1 of 96M on
// torus500k) while the table probes on the fan warps cost ~10 % of a
// field.  Exact twins come from saddle fans:
// tied candidates of one vertex (same distance, different directions) fan
// out over the same fully covered wedges.  Every fan window is
// fingerprinted (96 bits of two 64-bit mixes of its fields and field row)
// into an open-addressed table tagged with the iteration's epoch; a window
// whose fingerprint is already there in this epoch is dropped and counted
// as pruned_duplicate.  Stale entries (older epochs) are claimed over.
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ bool fan_duplicate(const Params &p, const Win &c, unsigned int epoch) {
    const unsigned long long f[6] = {
        ((unsigned long long)(uint32_t)c.he << 32) | c.row, (unsigned long long)__double_as_longlong(c.b0),
        (unsigned long long)__double_as_longlong(c.b1), (unsigned long long)__double_as_longlong(c.d0),
        (unsigned long long)__double_as_longlong(c.d1), (unsigned long long)__double_as_longlong(c.d)};
    unsigned long long h1 = 0x9e3779b97f4a7c15ull, h2 = 0x632be59bd9b4e019ull;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        h1 = mix64(h1 ^ f[k]);
        h2 = mix64(h2 + f[k] * 0xd6e8feb86659fd93ull);
    }
    const unsigned long long tag = ((unsigned long long)epoch << 32) | (h1 & 0xffffffffull);
    unsigned long long slot = (h1 >> 32) & p.dup_mask;
    for (int probe = 0; probe < 16; ++probe, slot = (slot + 1) & p.dup_mask) {
        ulonglong2 cur = __ldcg(p.dup_tab + slot);
        for (;;) {
            if (cur.x == tag && cur.y == h2) return true;          // twin in this epoch
            if ((unsigned int)(cur.x >> 32) == epoch) break;        // other window: next slot
            const ulonglong2 old = atomicCAS(p.dup_tab + slot, cur, make_ulonglong2(tag, h2));
            if (old.x == cur.x && old.y == cur.y) return false;    // claimed a stale slot
            cur = old;
        }
    }
    return false;  // table crowded: keep the window (a duplicate only costs work)
}

// fan interval of v (geom.py:239-256); returns false for an empty fan
__device__ __forceinline__ bool fan_span(const Params &p, int32_t v, int32_t anchor, double rel,
                                         bool full, FanSpan &f) {
    // one 16-byte header per vertex and the anchor's wedge angle: both
    // addresses are known from the event, so the two loads overlap
    const double2 hraw = __ldg(reinterpret_cast<const double2 *>(p.fanhdr + v));
    const double aphi = full ? 0.0 : __ldg(p.anchor_wlo + anchor);
    f.theta = hraw.x;
    const long long meta = __double_as_longlong(hraw.y);
    f.off = (int32_t)(meta & 0xffffffffll);
    f.m = (int32_t)((meta >> 32) & 0x7fffffffll);
    const bool interior = (meta >> 63) & 1;
    if (full) {
        f.flo = -1.0e300;
        f.fhi = 1.0e300;
        f.reps = 1;
        return true;
    }
    double width = f.theta - TWO_PI_D;
    if (width <= EPS_NUM) return false;
    f.flo = aphi + rel + PI_D - p.fan_widen;
    f.fhi = f.flo + width + 2.0 * p.fan_widen;
    if (interior) {
        double k = floor(f.flo / f.theta);
        f.flo -= k * f.theta;
        f.fhi -= k * f.theta;
        f.reps = 2;
    } else {
        f.reps = 1;
    }
    return true;
}

// one (wedge i, repetition rep) item of a fan (geom.py:258-307): the window
// with pseudo source v on the edge opposite v in wedge i, clipped to the fan
// interval.  `fresh` filters against the shadow field of this iteration
// (phase B, where the frozen copy is being committed) instead of gdist.
template <typename Emit>
__device__ __forceinline__ void fan_item(const Params &p, const RowTabs &t, uint32_t row, double cand,
                                         const FanSpan &f, int i, int rep, bool fresh, Emit &&emit,
                                         LocalStats &ls, unsigned int epoch = 0u) {
    const FanRec &fr = p.fan[f.off + i];
    double wlo = __ldg(&fr.wlo), whi = __ldg(&fr.whi);
    double lo = f.flo - rep * f.theta, hi = f.fhi - rep * f.theta;
    double slo = wlo > lo ? wlo : lo;
    double shi = whi < hi ? whi : hi;
    if (shi - slo <= 1e-12) return;
    if (p.fan_full) {
        slo = wlo;
        shi = whi;
    }
    double px = __ldg(&fr.px), py = __ldg(&fr.py), qx = __ldg(&fr.qx), qy = __ldg(&fr.qy);
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
    ls.add(ST_CREATED);
    if (!(ok0 && ok1)) {
        ls.add(ST_PRUNE_DEGEN);
        return;
    }
    int32_t pid = __ldg(&fr.pid), qid = __ldg(&fr.qid);
    const uint32_t sad = __ldg(&fr.sad);
    const uint32_t cv0 = (uint32_t)pid | ((sad & 1u) ? SADDLE_BIT : 0u);
    const uint32_t cv1 = (uint32_t)qid | ((sad & 2u) ? SADDLE_BIT : 0u);
    double gp, gq;
    if (fresh) {
        gp = __longlong_as_double((long long)__ldcg(t.dist + pid));
        gq = __longlong_as_double((long long)__ldcg(t.dist + qid));
    } else {
        gp = gdist(p, t, pid);
        gq = gdist(p, t, qid);
    }
    Win c;
    int fate = make_child(__ldg(&fr.che), __ldg(&fr.cho), cv0, cv1, __ldg(&fr.capx), __ldg(&fr.lc), px, py,
                          qx, qy, s0, s1, 0.0, 0.0, cand,
                          gp, gq, INFINITY, 0.0, 0.0, true, p.eps_win2, p.inv_r02, c);
    c.row = row;
    if (fate == CH_STORED) {
        if (epoch && p.dup_tab && fan_duplicate(p, c, epoch)) {
            ls.add(ST_PRUNE_DUP);
            return;
        }
        emit(c);
    } else {
        ls.add(fate == CH_TINY ? ST_PRUNE_TINY : fate == CH_ICH ? ST_PRUNE_ICH : ST_PRUNE_DEGEN);
    }
}

// saddle fans (geom.py:185): windows with pseudo source v on the edges
// opposite v inside the fan spanned by the two straight extensions of the
// incoming ray; `full` emits every wedge (source initialisation).  Serial
// form (one thread); the solver loop spreads fan items over a warp.
template <typename Emit>
__device__ void emit_fan(const Params &p, const RowTabs &t, uint32_t row, int32_t v, double cand,
                         int32_t anchor, double rel, bool full, Emit &&emit, LocalStats &ls) {
    FanSpan f;
    if (!fan_span(p, v, anchor, rel, full, f)) return;
    for (int i = 0; i < f.m; ++i)
        for (int rep = 0; rep < f.reps; ++rep) fan_item(p, t, row, cand, f, i, rep, false, emit, ls);
}

// ---------------------------------------------------------------------------
// Algorithm 2 (geom.py:312) for one window against the frozen tables.
// Up to two children are returned in `c`; events go to the shadow tables.

template <int LIVE = -1, typename FanSink>
__device__ __forceinline__ int propagate(const Params &p, Stage &sg, int it, FanSink &&fsink,
                                         const Win &w, Win &out0, Win &out1, LocalStats &ls) {
    const bool live = LIVE < 0 ? (p.live != 0) : (LIVE != 0);
    // Latency layout: the per-iteration critical path is one propagation
    // (of the slowest lane of the slowest warp), so
    //  * every memory access is issued as soon as its address is known
    //    (window -> face record + split entry -> distances: three levels);
    //  * the case analysis of Algorithm 2 selects parameters instead of
    //    branching: both candidate children (on the far face's left and
    //    right edge) go through one straight-line make_child each, so a
    //    warp runs one instruction stream whatever its lanes' cases;
    //  * all event atomics are issued together at the end, fire and forget
    //    where the result is not needed.
    const int32_t j = w.he, jo = w.jo;
    const double b0 = w.b0, b1 = w.b1, d0 = w.d0, d1 = w.d1, dps = w.d;
    const bool far = jo >= 0;
    const RowTabs T = row_tabs<LIVE>(p, w.row, it);
    // level 1: the far face (or, on a boundary, the window's own face)
    // and the angle-split entry of j
    const int32_t fr = far ? jo : j;
    const int a = fr % 3;
    const FaceRec *fp = p.face + fr / 3;
    const int a1 = a == 2 ? 0 : a + 1, a2 = a == 0 ? 2 : a - 1;
    // edge jo runs v1 -> v0 and its successor starts at v0 (geom.py:390);
    // on a boundary the record is j's own face, where j runs v0 -> v1
    const double ell = __ldg(&fp->len[a]);
    const double lan = __ldg(&fp->len[a1]);
    const double lpv = __ldg(&fp->len[a2]);
    // the far triangle's apex D below the edge, precomputed per half-edge
    // (geom.py:387-396), loaded with the face record
    const double2 dxy = __ldg(p.apex_xy + fr);
    // the window's vertices (carried from its creation): the distances
    // below are issued together with the face record
    const uint32_t v0f = w.v0f, v1f = w.v1f, vdf = far ? w.vdf : 0u;
    const int32_t cho_l = __ldg(&fp->opp[a1]), cho_r = __ldg(&fp->opp[a2]);
    const uint32_t apx_l = __ldg(&fp->apx[a1]), apx_r = __ldg(&fp->apx[a2]);
    const ulonglong2 sp_raw = far ? gsplit_raw<LIVE>(p, T, j) : make_ulonglong2(ord64(INFINITY), ord64(0.0));
    // level 2: distances at the three vertices
    const int32_t v0 = (int32_t)(v0f & VMASK), v1 = (int32_t)(v1f & VMASK);
    const int32_t vd = (int32_t)(vdf & VMASK);
    const double g0 = gdist<LIVE>(p, T, v0), g1 = gdist<LIVE>(p, T, v1);
    const double gdd = far ? gdist<LIVE>(p, T, vd) : INFINITY;
    // saddle endpoints: the current fan pick, the guess for its CAS-min
    const ulonglong2 *pick = T.pick;
    const ulonglong2 none = make_ulonglong2(~0ull, ~0ull);
    const ulonglong2 pk0 = (live && (v0f & SADDLE_BIT)) ? __ldcg(pick + v0) : none;
    const ulonglong2 pk1 = (live && (v1f & SADDLE_BIT)) ? __ldcg(pick + v1) : none;
    const ulonglong2 pkd = (live && far && (vdf & SADDLE_BIT)) ? __ldcg(pick + vd) : none;

    double ix, iy;
    if (!unfold(b0, b1, d0, d1, ix, iy)) {
        ls.add(ST_PRUNE_DEGEN);
        return 0;
    }
    // endpoint inequalities of the ICH filter (paper Fig. 4b) against the
    // current field: paths through v0 (resp. v1) already reach the far end
    // of the interval more cheaply -> the window is useless.  Evaluated
    // here, applied at the end (no branch on the distance loads).
    // |I B| = d1 and |I A| = d0 by construction of I
    const bool rechecked = p.recheck && ((dps + d1 > g0 + b1 + EPS_NUM) ||
                                         (dps + d0 > g1 + (ell - b0) + EPS_NUM));

    // interval endpoints sitting on v0 / v1 (geom.py:345-385)
    const double cand0 = dps + d0 + b0;
    const bool ev0 = !rechecked && b0 <= p.eps_win && cand0 < g0;
    const double cand1 = dps + d1 + (ell - b1);
    const bool ev1 = !rechecked && b1 >= ell - p.eps_win && cand1 < g1;

    // the far triangle: apex D below the edge (geom.py:387-516)
    const double dx = dxy.x, dy = dxy.y;
    const double uax = b0 - ix, uay = -iy, ubx = b1 - ix, uby = -iy;
    const double vdx = dx - ix, vdy = dy - iy;
    const double nvd2 = vdx * vdx + vdy * vdy;
    const double nvd = psqrt(nvd2);
    const double ca = uax * vdy - uay * vdx;
    const double cb = ubx * vdy - uby * vdx;
    // tolerances EPS_NUM |IA| |ID| and EPS_NUM |IB| |ID| compared squared
    // (|IA| = d0, |IB| = d1 up to the unfold's rounding; geom.py:408-409)
    const double e2 = EPS_NUM * EPS_NUM * nvd2;
    const bool a_in = ca > 0.0 && ca * ca > e2 * (uax * uax + uay * uay);
    const bool b_out = cb < 0.0 && cb * cb > e2 * (ubx * ubx + uby * uby);
    // occ: the ray to the apex passes strictly inside (A, B) -- w occupies vd
    const bool occ = far && a_in && b_out;
    const bool left = !b_out;  // (not occ) both rays exit through edge v0-D
    const double comp = dps + nvd;
    const double denom = iy - dy;
    const double entry_x = denom > 1e-300 ? ix + (dx - ix) * pdiv(iy, denom) : ix;
    // the two rays: I->A against the left edge (v0, D) unless only the
    // right edge is hit, I->B against the right edge (D, v1) unless only
    // the left edge is hit
    const bool eA_left = occ || left, eB_left = !occ && left;
    double rA, rB;
    const bool okA = ray_seg(ix, iy, b0, 0.0, eA_left ? 0.0 : dx, eA_left ? 0.0 : dy,
                             eA_left ? dx : ell, eA_left ? dy : 0.0, rA);
    const bool okB = ray_seg(ix, iy, b1, 0.0, eB_left ? 0.0 : dx, eB_left ? 0.0 : dy,
                             eB_left ? dx : ell, eB_left ? dy : 0.0, rB);
    const bool okL = okA && (occ || okB), okR = okB && (occ || okA);
    const double candd = comp;
    const bool evd = !rechecked && occ && candd < gdd;
    int nc = 0;
    Win cl, cr;
    const int fl = make_child(3 * (fr / 3) + a1, cho_l, v0f, vdf, apx_l, lan, 0.0, 0.0, dx, dy, rA,
                              occ ? 1.0 : rB,
                              ix, iy, dps, g0, gdd, g1, ell, 0.0, true, p.eps_win2, p.inv_r02, cl);
    const int frr = make_child(3 * (fr / 3) + a2, cho_r, vdf, v1f, apx_r, lpv, dx, dy, ell, 0.0,
                               occ ? 0.0 : rA, rB,
                               ix, iy, dps, gdd, g1, g0, 0.0, 0.0, false, p.eps_win2, p.inv_r02, cr);
    cl.row = cr.row = w.row;
    // one-angle-one-split (Fig. 4a): a stored window that already gives
    // the apex a shorter distance leaves only the child on our side
    const double sp_comp = unord64(sp_raw.x), sp_x = unord64(sp_raw.y);
    const bool claim = !rechecked && occ && comp < sp_comp;
    const bool split_pruned = !rechecked && occ && !claim;
    const bool want_l = !rechecked && (occ ? (claim || entry_x < sp_x) : (far && left));
    const bool want_r = !rechecked && (occ ? (claim || !(entry_x < sp_x)) : (far && !left));
    const bool ml = want_l && okL, mr = want_r && okR;  // children computed
    const bool sl = ml && fl == CH_STORED, sr = mr && frr == CH_STORED;
    // accounting as the reference counts it (geom.py:433-516)
    ls.add(ST_PROPAGATED, rechecked ? 0u : 1u);
    ls.add(ST_RECHECK, rechecked ? 1u : 0u);
    ls.add(ST_PRUNE_SPLIT, split_pruned ? 1 : 0);
    ls.add(ST_CREATED, rechecked ? 0u
                                 : (split_pruned ? 1u : 0u) +
                                       (occ ? (want_l ? 1u : 0u) + (want_r ? 1u : 0u) : (far ? 1u : 0u)));
    const unsigned int degen = rechecked ? 0u
                               : occ     ? (want_l && !okL ? 1u : 0u) + (want_r && !okR ? 1u : 0u)
                                         : (far && !(okA && okB) ? 1u : 0u);
    ls.add(ST_PRUNE_DEGEN, degen + (ml && fl == CH_DEGEN ? 1u : 0u) + (mr && frr == CH_DEGEN ? 1u : 0u));
    ls.add(ST_PRUNE_TINY, (ml && fl == CH_TINY ? 1u : 0u) + (mr && frr == CH_TINY ? 1u : 0u));
    ls.add(ST_PRUNE_ICH, (ml && fl == CH_ICH ? 1u : 0u) + (mr && frr == CH_ICH ? 1u : 0u));
    // compacted children: the right one is always out1 when both are
    // kept, so only out0 needs a select (not two predicated copies)
    out0 = sl ? cl : cr;
    out1 = cr;
    nc = (sl ? 1 : 0) + (sr ? 1 : 0);

    // ---- events, issued together (order independent: min / CAS-min) ----
    if (ev0) dist_event<LIVE>(p, T, sg, v0, cand0, ls);
    if (ev1) dist_event<LIVE>(p, T, sg, v1, cand1, ls);
    if (evd) dist_event<LIVE>(p, T, sg, vd, candd, ls);
    if (claim) angle_event<LIVE>(p, T, sg, j, comp, entry_x, sp_raw, ls);
    // saddle fans (Fig. 3c): the reverse direction of the incoming ray
    // relative to an anchor half-edge out of the vertex (geom.py:353-484)
    if (ev0 && (v0f & SADDLE_BIT)) fan_event<LIVE>(p, T, w.row, fsink, pk0, v0, j, cand0, ix, iy, 1.0, 0.0);
    if (ev1 && (v1f & SADDLE_BIT)) {
        if (far) {
            // anchor jo = v1 -> v0: its wedge follows next(j)'s, so this is
            // the reference's anchor next(j) with the corner at v1 folded
            // into the anchor angle
            fan_event<LIVE>(p, T, w.row, fsink, pk1, v1, jo, cand1, ix - ell, iy, -1.0, 0.0);
        } else {
            // boundary window: anchor next(j), the source-side apex
            // direction from v1 (geom.py:372-377)
            const int32_t jn = 3 * (j / 3) + (j + 1) % 3;
            const FaceRec *fj = p.face + j / 3;
            const int b = j % 3;
            const double lns = __ldg(&fj->len[b == 2 ? 0 : b + 1]);
            const double lps = __ldg(&fj->len[b == 0 ? 2 : b - 1]);
            const double axs = 0.5 * (ell * ell + lps * lps - lns * lns) / ell;
            const double ay2 = lps * lps - axs * axs;
            fan_event<LIVE>(p, T, w.row, fsink, pk1, v1, jn, cand1, ix - ell, iy, axs - ell,
                      ay2 > 0.0 ? sqrt(ay2) : 0.0);
        }
    }
    if (evd && (vdf & SADDLE_BIT))
        fan_event<LIVE>(p, T, w.row, fsink, pkd, vd, 3 * (jo / 3) + a2, candd, ix - dx, iy - dy, ell - dx, -dy);
    return nc;
}

// ---------------------------------------------------------------------------
// k-selection threshold from the key histogram: smallest bin boundary whose
// cumulative count reaches K.  Every CTA computes the identical value.

struct Thresh {
    double t, w_next;
    int bin;                    // bin holding the K-th key (NBINS: none)
    unsigned long long before;  // keys in the bins below it
};

__device__ Thresh pick_threshold(const unsigned int *hist, double base, double w, long long K) {
    __shared__ unsigned int s_part[32];
    __shared__ int s_bin;
    __shared__ unsigned long long s_total, s_over;
    constexpr int PER = (NBINS + TPB - 1) / TPB;
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
    __shared__ unsigned long long s_before;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        unsigned long long nx = cum + loc[q];
        if (cum < (unsigned long long)K && nx >= (unsigned long long)K) {
            atomicMin(&s_bin, t * PER + q);
            s_before = cum;  // a single bin crosses K
        }
        cum = nx;
    }
    __syncthreads();
    Thresh r;
    int b = s_bin;
    r.bin = b;
    r.before = b < NBINS ? s_before : 0ull;
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


__device__ __forceinline__ void trace_max(const Params &p, int it, int slot) {
    if (p.trace && it < p.trace_cap) atomicMax(p.trace + (size_t)it * TR_N + slot, globaltimer());
}

// one trace stamp per warp (the first active lane): per-lane global
// atomics on one address would serialise and distort the timeline
__device__ __forceinline__ void trace_max_warp(const Params &p, int it, int slot) {
    const unsigned m = __activemask();
    if ((threadIdx.x & 31) == __ffs(m) - 1) trace_max(p, it, slot);
}

// CTA-level allocation of `n` (<= 3) pool slots per thread for one trip:
// one global atomicAdd per CTA; returns the thread's first slot index
// relative to the counter (uniform: contains __syncthreads)
__device__ __forceinline__ unsigned long long cta_alloc(unsigned long long *counter, unsigned int n) {
    __shared__ unsigned long long s_base;
    unsigned int total;
    unsigned int excl = block_excl_scan(n, total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(counter, (unsigned long long)total) : 0ull;
    __syncthreads();
    unsigned long long r = s_base + excl;
    __syncthreads();
    return r;
}

__device__ __forceinline__ void flush_hist(unsigned int *s_hist, unsigned int *g_hist) {
    __syncthreads();
    for (int b = threadIdx.x; b <= NBINS; b += TPB) {
        unsigned int x = s_hist[b];
        if (x) {
            atomicAdd(g_hist + b, x);
            s_hist[b] = 0u;
        }
    }
    __syncthreads();
}

#ifndef PCH_MIN_BLOCKS
#define PCH_MIN_BLOCKS 1  // resident CTAs per SM the register budget targets
#endif
#ifndef PCH_LIVE_MIN_BLOCKS
#define PCH_LIVE_MIN_BLOCKS 1  // ... of the one-barrier solver
#endif

__global__ void __launch_bounds__(TPB, PCH_MIN_BLOCKS) pch_persistent(Params p) {
    Ctrl *ctrl = p.ctrl;
    unsigned int gen = 0;
    __shared__ unsigned long long s_st[N_ST];
    __shared__ Stage sg;
    __shared__ unsigned int s_hist[NBINS + 1];
    stats_init(s_st);
    for (int b = threadIdx.x; b <= NBINS; b += TPB) s_hist[b] = 0u;
    if (threadIdx.x == 0) sg.ntv = sg.nte = sg.nfe = 0u;
    __syncthreads();
    LocalStats ls{s_st, true};
    int maxchild = 0;
    WinSoA X = p.X, Y = p.Y;
    double base = 0.0, w = p.w0;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * TPB + threadIdx.x;
    const unsigned long long gthreads = (unsigned long long)gridDim.x * TPB;
    const unsigned long long nwarps = gthreads >> 5;
    // warp-interleaved thread index: consecutive warps of work land on
    // different CTAs (SMs), lanes of a warp stay contiguous (coalesced),
    // so a batch much smaller than the grid still spreads over every SM
    const unsigned long long wtid =
        ((unsigned long long)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32ull + (threadIdx.x & 31);
    const unsigned long long gwid = wtid >> 5;
    const int lane = threadIdx.x & 31;
    const unsigned long long t_start = globaltimer();
    int it = 0;
    // an initialisation failure (source-window overflow, invalid device
    // source) leaves slot 0 unusable: every CTA reads the same flag before
    // iteration 0 and skips the loop
    const bool init_err = *(volatile int *)&ctrl->error != 0;
    for (; !init_err;) {
        Slot &cur = ctrl->slot[it % 3];
        Slot &prev = ctrl->slot[(it + 2) % 3];
        Slot &nxt = ctrl->slot[(it + 1) % 3];
        const unsigned long long nS = *(volatile unsigned long long *)&cur.nS;
        const unsigned long long nP = *(volatile unsigned long long *)&cur.nP;
        if (DEV_TRACE && it < p.trace_cap && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long *tr = p.trace + (size_t)it * TR_N;
            tr[TR_T0] = globaltimer();
            tr[TR_NS] = nS;
            tr[TR_NP] = nP;
        }

        // ================= phase A: propagate =================
        long long ph0 = clock64();
        auto phase = [&](int which) {
            if (p.phase && threadIdx.x == 0) {
                const long long now = clock64();
                s_st[which] += (unsigned long long)(now - ph0);
                ph0 = now;
            }
        };
        if (blockIdx.x == 0) {
            if (threadIdx.x < sizeof(Slot) / 8)
                reinterpret_cast<unsigned long long *>(&nxt)[threadIdx.x] = 0ull;
            for (int b = threadIdx.x; b <= NBINS; b += TPB) p.hist[(it + 1) & 1][b] = 0u;
            if (threadIdx.x == 0) ls.max(ST_PEAK, nS + nP);
        }
        if (p.exact_select) {
            // the next iteration's sub-bins (last read in phase B of it-1)
            uint4 *fz = reinterpret_cast<uint4 *>(p.fine[(it + 1) & 1]);
            for (unsigned long long q = gtid; q < FINE_N / 4; q += gthreads) fz[q] = make_uint4(0u, 0u, 0u, 0u);
        }
        unsigned int *hcur = p.hist[it & 1];
        // write one window into pool slot nP + rel (children C_i follow P_i)
        auto put_pool = [&](const Win &c, unsigned long long rel) {
            unsigned long long slot = nP + rel;
            if ((long long)slot < p.cap) {
                store_win(X, slot, c);
                const int cb = key_bin(c.key, base, w);
                atomicAdd(s_hist + cb, 1u);
                if (p.exact_select) fine_add(p.fine[it & 1], c.key, base, w, cb);
            } else {
                atomicExch(&ctrl->error, ERR_OVERFLOW);
            }
            ls.add(ST_STORED);
        };
        // saddle fans of iteration it-1, one warp per fan event with the
        // lanes spread over the fan's wedges.  Only the event whose candidate
        // is the committed distance and wins the per-vertex pick (smallest
        // candidate, then anchor / direction) emits, so each improved saddle
        // fans out once per improvement.  Every input is frozen, so which
        // warp runs an event (and when) does not change the outcome.
        const unsigned long long nFc = [&] {
            if (it == 0) return 0ull;
            const unsigned long long nF = *(volatile unsigned long long *)&prev.nF;
            return nF < (unsigned long long)p.fancap ? nF : (unsigned long long)p.fancap;
        }();
        const FanEv *fe = p.fanev[(it + 2) % 3];
        auto fan_event_warp = [&](unsigned long long i, Win &c, unsigned int &n) {
            long long c3 = DEV_PROF ? clock64() : 0;
            FanEv e = fe[i];
            const double rel = fan_rel(e);
            const double dv = __ldcg(p.dist_cur + e.v);
            const ulonglong2 pk = __ldcg(p.fanpick[(it + 2) % 3] + e.v);
            const unsigned long long lo =
                fan_tiebreak(e);
            FanSpan f;
            if (__double_as_longlong(dv) == __double_as_longlong(e.cand) &&
                pk.x == (unsigned long long)__double_as_longlong(e.cand) && pk.y == lo &&
                fan_span(p, e.v, e.anchor, rel, false, f)) {
                if (lane == 0) ls.add(ST_FANS);
                const int items = f.m * f.reps;
                if (lane < items) {
                    fan_item(p, row_tabs(p, 0u, it), 0u, e.cand, f, lane % f.m, lane / f.m, false,
                             [&](const Win &x) { c = x; n = 1; }, ls, p.dup_epoch + it + 1u);
                }
                // wedges beyond the warp width (valence > 32): rare,
                // appended with a warp-aggregated global slot
                for (int q = lane + 32; q < items; q += 32)
                    fan_item(p, row_tabs(p, 0u, it), 0u, e.cand, f, q % f.m, q / f.m, false,
                             [&](const Win &x) { put_pool(x, warp_alloc(&cur.nC, true)); }, ls,
                             p.dup_epoch + it + 1u);
            }
            if (DEV_PROF) {
                ls.add(ST_CYC_FANITEM, clock64() - c3);
                ls.add(ST_N_FANITEM);
            }
        };
        // (A1) the selected batch S_i: one thread per window, children into
        // registers, pool slots reserved once per CTA and trip.  The warps
        // the last trip leaves without a window run fan events meanwhile
        // (the first nFa of them) instead of idling until A2.
        unsigned long long nFa = 0;
        {
            const unsigned long long trips = (nS + gthreads - 1) / gthreads;
            const unsigned long long last = trips ? nS - (trips - 1) * gthreads : 0ull;
            const unsigned long long busyw = (last + 31) >> 5;  // warps of the last trip with windows
            nFa = trips ? min(nFc, nwarps - busyw) : 0ull;
            for (unsigned long long t = 0; t < trips; ++t) {
                const unsigned long long i = t * gthreads + wtid;
                Win ca, cb;
                int nc = 0;
                if (i < nS) {
                    long long c0 = DEV_PROF ? clock64() : 0;
                    Win win = load_win(p.S, i);
                    nc = propagate<0>(p, sg, it, StageFanSink{p, sg, &cur.nF, p.fanev[it % 3]}, win, ca,
                                   cb, ls);
                    if (DEV_PROF) ls.add(ST_CYC_PROP, clock64() - c0);
                    if (nc > maxchild) maxchild = nc;
                } else if (t + 1 == trips && gwid >= busyw && gwid - busyw < nFa) {
                    unsigned int n = 0;
                    fan_event_warp(gwid - busyw, ca, n);
                    nc = (int)n;
                }
                long long c2 = DEV_PROF ? clock64() : 0;
                const unsigned long long rel = trip_flush(p, sg, cur, it, (unsigned int)nc);
                if (nc > 0) put_pool(ca, rel);
                if (nc > 1) put_pool(cb, rel + 1);
                if (DEV_PROF) {
                    ls.add(ST_CYC_POOL, clock64() - c2);
                    ls.add(ST_N_POOL);
                }
            }
        }
        phase(ST_PH_PROP);
        // (A2) the fan events the idle warps of A1 did not take
        {
            const unsigned long long nrest = nFc - nFa;
            const unsigned long long trips = (nrest + nwarps - 1) / nwarps;
            for (unsigned long long t = 0; t < trips; ++t) {
                const unsigned long long i = nFa + t * nwarps + gwid;
                Win c;
                unsigned int n = 0;
                if (i < nFc) fan_event_warp(i, c, n);
                unsigned long long rel = cta_alloc(&cur.nC, n);
                if (n) put_pool(c, rel);
            }
        }
        flush_hist(s_hist, hcur);
        if (DEV_TRACE && threadIdx.x == 0) trace_max(p, it, TR_A_END);
        phase(ST_PH_EVENTS);
        grid_barrier(ctrl, gen);
        if (DEV_TRACE && it < p.trace_cap && blockIdx.x == 0 && threadIdx.x == 0)
            p.trace[(size_t)it * TR_N + TR_B1] = globaltimer();

        // ================= phase B: organise =================
        // the shadow-table commit needs no threshold: its first entries and
        // their new values are read here, in flight during the threshold
        // pick, and written after it
        const unsigned long long nTVc = [&] {
            const unsigned long long n = *(volatile unsigned long long *)&cur.nTV;
            return n < (unsigned long long)p.tvcap ? n : (unsigned long long)p.tvcap;
        }();
        const unsigned long long nTEc = [&] {
            const unsigned long long n = *(volatile unsigned long long *)&cur.nTE;
            return n < (unsigned long long)p.tecap ? n : (unsigned long long)p.tecap;
        }();
        const int32_t cv = gtid < nTVc ? __ldcg(p.tv_list + gtid) : -1;
        const int32_t cj = gtid < nTEc ? __ldcg(p.te_list + gtid) : -1;
        const unsigned long long cdist = cv >= 0 ? __ldcg(p.dist_new + cv) : 0ull;
        const ulonglong2 csplit = cj >= 0 ? __ldcg(p.split_new + cj) : make_ulonglong2(0ull, 0ull);
        const int32_t cfv = gtid < nFc ? fe[gtid].v : -1;  // fan picks consumed in A: reset below
        Thresh th = pick_threshold(hcur, base, w, p.K);
        if (p.exact_select && th.bin < NBINS) {
            // selection_mode "exact" (engine.py:256, argpartition): the bin
            // holding the K-th key refined into its NBINS sub-bins (counted
            // with the keys, fine_add), so the batch is the K nearest
            // windows up to keys within (bin width / NBINS)
            const double lo = base + (double)th.bin * w, sw = w / (double)NBINS;
            const Thresh t2 = pick_threshold(p.fine[it & 1] + (size_t)th.bin * FINE_ROW, lo, sw,
                                             (long long)((unsigned long long)p.K - th.before));
            if (t2.bin < NBINS) th.t = t2.t;
        }
        phase(ST_PH_SELECT);
        {
            // commit the shadow tables for entries touched this iteration
            if (cv >= 0) p.dist_cur[cv] = __longlong_as_double((long long)cdist);
            if (cj >= 0) p.split_cur[cj] = make_double2(unord64(csplit.x), unord64(csplit.y));
            for (unsigned long long i = gtid + gthreads; i < nTVc; i += gthreads) {
                int32_t v = __ldcg(p.tv_list + i);
                p.dist_cur[v] = __longlong_as_double((long long)__ldcg(p.dist_new + v));
            }
            for (unsigned long long i = gtid + gthreads; i < nTEc; i += gthreads) {
                int32_t j = __ldcg(p.te_list + i);
                ulonglong2 s = __ldcg(p.split_new + j);
                p.split_cur[j] = make_double2(unord64(s.x), unord64(s.y));
            }
            // fan picks of iteration it-1 are consumed: reset them
            if (cfv >= 0) p.fanpick[(it + 2) % 3][cfv] = make_ulonglong2(~0ull, ~0ull);
            for (unsigned long long i = gtid + gthreads; i < nFc; i += gthreads)
                p.fanpick[(it + 2) % 3][fe[i].v] = make_ulonglong2(~0ull, ~0ull);
        }
        phase(ST_PH_EVENTS);
        {
            // partition P_i + C_i -> S_{i+1} (key <= t) and P_{i+1}: stream
            // compaction with one reservation per CTA and trip per output
            const unsigned long long nC = *(volatile unsigned long long *)&cur.nC;
            unsigned long long total = nP + nC;
            if ((long long)total > p.cap) total = p.cap;
            const double nbase = th.t < INFINITY ? th.t : base;
            const unsigned long long trips = (total + gthreads - 1) / gthreads;
            __shared__ unsigned long long s_sb[2];
            for (unsigned long long t = 0; t < trips; ++t) {
                const unsigned long long i = t * gthreads + gtid;
                long long c5 = DEV_PROF ? clock64() : 0;
                Win c;
                const bool valid = i < total;
                if (valid) c = load_win(X, i);
                const bool sel = valid && c.key <= th.t;
                const bool keep = valid && !sel;
                unsigned int tot2;
                const unsigned int ex = block_excl_scan((sel ? 1u : 0u) | (keep ? 0x10000u : 0u), tot2);
                if (threadIdx.x == 0) {
                    s_sb[0] = (tot2 & 0xffffu) ? atomicAdd(&nxt.nS, (unsigned long long)(tot2 & 0xffffu)) : 0ull;
                    s_sb[1] = (tot2 >> 16) ? atomicAdd(&nxt.nP, (unsigned long long)(tot2 >> 16)) : 0ull;
                }
                __syncthreads();
                if (sel) store_win(p.S, s_sb[0] + (ex & 0xffffu), c);
                if (keep) {
                    store_win(Y, s_sb[1] + (ex >> 16), c);
                    const int cb = key_bin(c.key, nbase, th.w_next);
                    atomicAdd(s_hist + cb, 1u);
                    if (p.exact_select) fine_add(p.fine[(it + 1) & 1], c.key, nbase, th.w_next, cb);
                }
                __syncthreads();
                if (DEV_PROF && valid) {
                    ls.add(ST_CYC_PART, clock64() - c5);
                    ls.add(ST_N_PART);
                }
            }
            flush_hist(s_hist, p.hist[(it + 1) & 1]);
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (p.max_iter >= 0 && it + 1 > p.max_iter) atomicExch(&ctrl->error, ERR_GUARD);
            if (globaltimer() - t_start > p.time_limit_ns) atomicExch(&ctrl->error, ERR_TIMEOUT);
        }
        if (DEV_TRACE && threadIdx.x == 0) trace_max(p, it, TR_B_END);
        grid_barrier(ctrl, gen);
        phase(ST_PH_COMPACT);

        // ================= termination =================
        const int err = *(volatile int *)&ctrl->error;
        const unsigned long long ns = *(volatile unsigned long long *)&nxt.nS;
        const unsigned long long np = *(volatile unsigned long long *)&nxt.nP;
        const unsigned long long nf = *(volatile unsigned long long *)&cur.nF;
        if (DEV_TRACE && it < p.trace_cap && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long *tr = p.trace + (size_t)it * TR_N;
            tr[TR_B2] = globaltimer();
            tr[TR_NC] = *(volatile unsigned long long *)&cur.nC;
            tr[TR_NF] = nf;
            tr[TR_NTV] = *(volatile unsigned long long *)&cur.nTV;
            tr[TR_TSEL_BITS] = (unsigned long long)__double_as_longlong(th.t);
        }
        ++it;
        if (err || (ns == 0 && np == 0 && nf == 0)) break;
        WinSoA T = X;
        X = Y;
        Y = T;
        // after a select-all step (t = +inf) keep the old histogram base
        if (th.t < INFINITY) base = th.t;
        w = th.w_next;
    }
    if (maxchild) ls.max(ST_MAXCHILD, maxchild);
    flush_stats(ctrl, s_st);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctrl->iterations = it;
        ctrl->t_final = base;
    }
}

// ---------------------------------------------------------------------------
// The one-barrier solver (default).  Iteration i is a single phase
// followed by one grid barrier:
//
//   * the threshold t_{i+1} of the next batch is fixed when the iteration
//     starts, by a step controller that steers |S| toward k (paper §5.2's
//     k, as a distance step instead of a k-th-key search: every CTA
//     evaluates it identically from the same counters);
//   * every work item is routed as it is produced: children of S_i (one
//     thread per window), windows of P_i (re-examined against t_{i+1}) and
//     the saddle fans won in iteration i-1 (one warp per fan, one lane per
//     wedge) go to S_{i+1} when key <= t_{i+1}, else to P_{i+1}, through
//     one reservation per CTA and trip (stream compaction);
//   * events update the distance field / angle-split table atomically and
//     the filters read them live (paper §5.1's delayed update collapses to
//     zero delay: every value read is a real path length, so a racing read
//     only weakens pruning).  Fields agree across runs to rounding; the
//     bitwise-deterministic two-barrier kernel above is PCH_FLAG_DETERMINISTIC.

// Item index -> slot of a chunked buffer: chunk c holds items
// [pre[c], pre[c+1]) at slots c * ch + (i - pre[c]).  Chunks are filled
// about evenly (windows are spread over the CTAs), so the search starts at
// the proportional guess i * G / n and walks at most a few chunks.
__device__ __forceinline__ unsigned long long chunk_slot(const unsigned int *pre, int G, unsigned int i,
                                                         unsigned long long ch) {
    // the last chunk c with pre[c] <= i: branch-free binary search,
    // log2(G) dependent shared loads whatever the chunk sizes' skew
    int c = 0;
    for (int step = 1 << (31 - __clz(G)); step > 0; step >>= 1) {
        const int n = c + step;
        c = (n < G && pre[n] <= i) ? n : c;
    }
    return (unsigned long long)c * ch + (i - pre[c]);
}

// warp-level reservation in the CTA's own chunks of S_{i+1} and P_{i+1}:
// every lane brings ns / np items (< 2^16 per warp), one packed scan and
// one shared 64-bit atomic per warp (S count in the low, P in the high
// half); returns the lane's first slot in each chunk (converged warp)
__device__ __forceinline__ void warp_chunk_alloc2(unsigned long long *s_cnt, unsigned int ns, unsigned int np,
                                                  unsigned int &sa, unsigned int &pa) {
    const int lane = threadIdx.x & 31;
    const unsigned int n = ns | (np << 16);
    unsigned int x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    const unsigned int tot = __shfl_sync(0xffffffffu, x, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot)
        base = atomicAdd(s_cnt, (unsigned long long)(tot & 0xffffu) | ((unsigned long long)(tot >> 16) << 32));
    base = __shfl_sync(0xffffffffu, base, 31);
    const unsigned int ex = x - n;
    sa = (unsigned int)base + (ex & 0xffffu);
    pa = (unsigned int)(base >> 32) + (ex >> 16);
}

// One CTA per SM with the full register budget (no spills), for single
// fields and batched rows alike: a 2-CTA/SM build at 128 registers spilled
// the propagation state to local memory and lost 9-16 % on batched rows
// (profiles/r01_bigcheck.md)
// PHASE: attribute warp cycles to the four phases (RunStats.time_*), on
// request only (EngineConfig.phase_times): the clock reads and per-item
// shared adds on the batch warps' critical path cost ~3 % of a field
template <bool PHASE, bool ROWS>
__global__ void __launch_bounds__(TPB, PCH_LIVE_MIN_BLOCKS) pch_live(Params p) {
    // Outputs are chunked per CTA: CTA b writes the windows it routes to
    // slots [b*ch, (b+1)*ch) of the next batch / pool and its fan
    // candidates to [b*chF, (b+1)*chF), allocating with one shared atomic
    // per warp -- no CTA-wide scan or global reservation on the iteration's
    // critical path.  Each CTA publishes its three counts at the end of the
    // iteration; after the barrier every CTA rebuilds the prefix tables.
    Ctrl *ctrl = p.ctrl;
    unsigned int gen = 0;
    const int G = gridDim.x;
    const int b = blockIdx.x;
    __shared__ unsigned long long s_st[N_ST];
    __shared__ Stage sg;                        // unused staging (shared helpers)
    __shared__ unsigned int s_pre[3][MAX_CTAS + 1];  // prefix tables: S, P, fans(prev)
    // this CTA's outputs of iteration i: S (low) / P (high), fan candidates;
    // three rotating copies, so reading iteration i's totals and clearing
    // the copy of iteration i+2 need no CTA barrier after the publish one
    __shared__ unsigned long long s_nsp3[3];
    __shared__ unsigned int s_nf3[3];
    __shared__ unsigned long long s_pmin, s_smax;
    __shared__ unsigned long long s_c[4];       // err, pmin, smax, grow of the finished iteration
    __shared__ unsigned int s_maxc[3];          // the largest chunk count of each table (build_prefix)
    stats_init(s_st);
    if (threadIdx.x == 0) {
        sg.ntv = sg.nte = sg.nfe = 0u;
        s_pmin = ~0ull;
        s_smax = 0ull;
        s_nsp3[0] = s_nsp3[1] = s_nsp3[2] = 0ull;
        s_nf3[0] = s_nf3[1] = s_nf3[2] = 0u;
    }
    int k3 = 0;  // this iteration's copy of the output counters
    unsigned int locS = 0u, locP = 0u, locF = 0u;  // this CTA's own counts (local iterations)
    LocalStats ls{s_st, false};   // packed per-thread counters, folded when nearly full
    LocalStats lsd{s_st, true};   // rare paths: straight to shared memory
    int maxchild = 0;
    const unsigned long long ch = (unsigned long long)p.cap / G;
    const unsigned long long chF = (unsigned long long)p.fancap / G;
    const unsigned long long gthreads = (unsigned long long)G * TPB;
    const unsigned long long nwarps = gthreads >> 5;
    const unsigned long long gwid = (unsigned long long)(threadIdx.x >> 5) * G + b;
    const int lane = threadIdx.x & 31;
    const unsigned long long t_start = globaltimer();
    // a resumed launch (pool grown at an iteration boundary) continues with
    // the saved iteration, threshold and step; its inputs were migrated
    // into the enlarged chunks by k_migrate_chunks
    double t = p.resume ? ctrl->res_t : 0.0;           // threshold S_i was selected with
    double delta = p.resume ? ctrl->res_delta : p.delta0;  // controller step
    // prefix tables of the iteration's inputs from the per-CTA counts
    // (and, with `slot`, the controller's inputs in the same round trip)
    auto build_prefix = [&](int par_in, int par_fan, const Slot *slot) {
        if (slot && threadIdx.x == 96) {
            s_c[0] = (unsigned long long)__ldcg(&ctrl->error);
            s_c[1] = __ldcg(&slot->pmin);
            s_c[2] = __ldcg(&slot->smax);
            s_c[3] = (unsigned long long)__ldcg(&ctrl->grow);
        }
        if (threadIdx.x < 96) {
            const int q = threadIdx.x >> 5;  // 0: S, 1: P, 2: fans of the previous iteration
            const unsigned int *cnt = p.ccnt + (size_t)((q < 2 ? par_in : par_fan) * 3 + q) * MAX_CTAS;
            if (lane == 0) s_pre[q][0] = 0u;
            unsigned int vmax = 0u;
            // all loads first (one round trip), then the carried scans
            constexpr int PER = 8;  // G <= 256 in one pass
            for (int base = 0; base < G; base += 32 * PER) {
                unsigned int v[PER];
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int c = base + k * 32 + lane;
                    v[k] = c < G ? __ldcg(cnt + c) : 0u;
                    vmax = v[k] > vmax ? v[k] : vmax;
                }
                unsigned int carry = base ? s_pre[q][base] : 0u;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int c = base + k * 32 + lane;
                    unsigned int x = v[k];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (c < G) s_pre[q][c + 1] = carry + x;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                __syncwarp();
            }
            vmax = __reduce_max_sync(0xffffffffu, vmax);
            if (lane == 0) s_maxc[q] = vmax;
        }
        __syncthreads();
    };
    int it = p.resume ? (int)ctrl->res_it : 0;
    // S_0: the source windows (chunk-published by k_source_windows), or the
    // inputs of the resumed iteration
    build_prefix(it & 1, (it & 1) ^ 1, &ctrl->slot[it % NSLOT]);
    // an initialisation failure (a source-window chunk overflowed, an
    // invalid device source) makes the published counts meaningless: every
    // CTA read the same flag with the prefix tables and skips the loop
    const bool init_err = s_c[0] != 0ull;
    // phase clocks (lane 0 of every warp): the iteration's barrier, prefix
    // rebuild and controller count as selection of the next batch
    long long ph_t = clock64();
    // Local iterations (p.local_iters > 1): between two grid barriers a CTA
    // runs local_iters - 1 iterations on its own chunks only -- its outputs
    // stay in its chunks anyway -- with a CTA barrier instead of the grid
    // barrier and without the prefix rebuild; the threshold advances by the
    // step the last global iteration chose, the global controller, the
    // termination test and the error / growth checks run at grid barriers.
    bool local = false;
    int local_left = 0;  // local iterations still to run in this block
    for (; !init_err;) {
        const int par = it & 1;                     // parity of the iteration's inputs
        // a local iteration reads this CTA's own counts (locS/P/F) and maps
        // item i to slot b * ch + i directly; a global one goes through the
        // prefix tables
        const unsigned int nS = local ? locS : s_pre[0][G], nP = local ? locP : s_pre[1][G];
        const unsigned int nF = it > 0 ? (local ? locF : s_pre[2][G]) : 0u;
        unsigned long long *const s_nsp = &s_nsp3[k3];
        unsigned int *const s_nf = &s_nf3[k3];
        const unsigned long long pminb = s_c[1], smaxb = s_c[2];
        Slot &nxt = ctrl->slot[(it + 1) % NSLOT];
        // work distribution: every warp of the grid over all chunks, or (a
        // local iteration) this CTA's warps over its own chunks
        const unsigned int wid0 = local ? (threadIdx.x >> 5) : (unsigned int)gwid;
        const unsigned int nwt = local ? (unsigned int)NWARP : (unsigned int)nwarps;
        // step controller: |S_i| / k steers the distance step
        if (it > 0 && !local) {
            double f = (double)p.K / (double)(nS > 0 ? nS : 1);
            f = f < 0.5 ? 0.5 : (f > 1.5 ? 1.5 : f);
            delta *= f;
            delta = delta < p.delta_min ? p.delta_min : (delta > p.delta_max ? p.delta_max : delta);
        }
        // anchor the threshold to the data: never above the largest key
        // actually selected (a select-all step must not run ahead), and up
        // to the pool's smallest key when nothing was selected
        const double pmin = nP ? __longlong_as_double((long long)pminb) : INFINITY;
        const double smax = __longlong_as_double((long long)smaxb);
        if (!local && nS > 0 && it > 0 && smax < t) t = smax;
        if (!local && nS == 0 && pmin > t && pmin < INFINITY) t = pmin;
        const double tn = t + delta;  // threshold of S_{i+1}
        // the iteration's sets as regions of p.S's columns (alloc_soa4):
        // batch in / out, pool in / out
        // (region numbers: batch in = par, batch out = par ^ 1, pool in =
        // 2 + par, pool out = 2 + (par ^ 1); offsets formed at the use)
        const unsigned int rSc = (unsigned int)par, rPc = 2u + (unsigned int)par;
        const FanEv *fev = p.fanev[par ^ 1];        // fan candidates of iteration i-1
        FanEv *fout = p.fanev[par] + (size_t)b * chF;  // this CTA's chunk for iteration i
        if (!local && blockIdx.x == 0 && threadIdx.x == 0) {
            // the slot of iteration i+2 is idle now: clear it
            Slot &clr = ctrl->slot[(it + 2) % NSLOT];
            clr.pmin = ~0ull;
            clr.smax = 0ull;
            ls.max(ST_PEAK, (unsigned long long)nS + nP);
        }
        if (DEV_TRACE && threadIdx.x == 0) trace_max(p, it, TR_START_MAX);
        if (DEV_TRACE && it < p.trace_cap && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long *tr = p.trace + (size_t)it * TR_N;
            tr[TR_T0] = globaltimer();
            tr[TR_NS] = nS;
            tr[TR_NP] = nP;
            tr[TR_NF] = nF;
            tr[TR_TSEL_BITS] = (unsigned long long)__double_as_longlong(tn);
        }
        // fan candidates of this iteration go straight to the CTA's chunk
        auto fsink = [&](const FanEv &e) {
            const unsigned int k = atomicAdd(s_nf, 1u);
            if (k < chF) fout[k] = e;
            else atomicExch(&ctrl->error, ERR_OVERFLOW);
        };
        // one window into this CTA's chunk of S_{i+1} / P_{i+1}
        auto put_at = [&](bool sel, unsigned int k, const Win &c) {
            if (k < ch)
                store_win(p.S, (unsigned long long)((sel ? 0u : 2u) + (unsigned int)(par ^ 1)) * (unsigned long long)p.cap +
                                   (unsigned long long)b * ch + k,
                          c);
            else atomicExch(&ctrl->error, ERR_OVERFLOW);
        };
        // rare paths (divergent): one shared atomic per window
        auto put_direct = [&](const Win &c) {
            const bool sel = c.key <= tn;
            lsd.add(ST_STORED);
            const unsigned long long old = atomicAdd(s_nsp, sel ? 1ull : (1ull << 32));
            put_at(sel, sel ? (unsigned int)old : (unsigned int)(old >> 32), c);
            if (sel) atomicMax(&s_smax, (unsigned long long)__double_as_longlong(c.key));
            else atomicMin(&s_pmin, (unsigned long long)__double_as_longlong(c.key));
        };

        // warp work items: S_i windows (32 per warp), fan candidates of i-1
        // (FANS_PER_WARP per warp), P_i windows (32 per warp); warps run
        // independently, no CTA-wide synchronisation until the iteration end
        const unsigned int nwS = (nS + 31u) >> 5, nwP = (nP + 31u) >> 5;
        const unsigned int nwF = (nF + FANS_PER_WARP - 1u) / FANS_PER_WARP;
        const unsigned int W = nwS + nwF + nwP;
        // a batch item (up to `chain` propagations) costs several light
        // items (fan candidate, pool re-examination): when the light items
        // fit on the warps without a batch item at <= LIGHT_PER_WARP each,
        // they stay there instead of wrapping onto the batch warps, whose
        // chains set the iteration's latency
        const unsigned int nLw = nwt > nwS ? nwt - nwS : 0u;
        const bool split = nLw > 0u && nwF + nwP <= LIGHT_PER_WARP * nLw;
        const unsigned int wstep = !split ? nwt : (wid0 < nwS ? W : nLw);
        if (PHASE && lane == 0) {
            const long long now = clock64();
            atomicAdd(&s_st[ST_PH_SELECT], (unsigned long long)(now - ph_t));
            ph_t = now;
        }
        for (unsigned int wi = wid0; wi < W; wi += wstep) {
            Win o0, o1, o2;   // o2: a sibling left behind by chaining
            int no = 0;
            bool h2 = false;
            if (wi < nwS) {
                const unsigned int i = (wi << 5) + lane;
                if (i < nS) {
                    long long c0 = DEV_PROF ? clock64() : 0;
                    const unsigned long long slot0 = local ? (unsigned long long)b * ch + i : chunk_slot(s_pre[0], G, i, ch);
                    if (DEV_TRACE) {
                        asm volatile("" ::"l"(slot0));
                        trace_max_warp(p, it, TR_TRIP0);
                    }
                    Win win = load_win(p.S, (unsigned long long)rSc * (unsigned long long)p.cap + slot0);
                    if (DEV_TRACE) {
                        asm volatile("" ::"d"(win.b0 + win.b1 + win.d0 + win.d1 + win.d + (double)win.jo));
                        trace_max_warp(p, it, TR_LOADED);
                    }
                    long long c1 = 0;
                    if (DEV_PROF) {
                        asm volatile("" ::"d"(win.b0 + win.b1 + win.d0 + win.d1 + win.d + (double)win.jo));
                        c1 = clock64();
                    }
                    // chaining: a child that the next batch would select
                    // (key <= t_{i+1}) is propagated right away by the same
                    // thread, up to p.chain propagations
                    for (int step = 1;; ++step) {
                        no = propagate<1>(p, sg, it, fsink, win, o0, o1, ls);
                        if (no > maxchild) maxchild = no;
                        if (step >= p.chain || no == 0) break;
                        const bool c0ok = o0.key <= tn, c1ok = no > 1 && o1.key <= tn;
                        if (!c0ok && !c1ok) break;
                        const bool take1 = c1ok && (!c0ok || o1.key < o0.key);
                        if (no > 1) {
                            // the child not chained: routed with the warp's
                            // outputs (first one) or directly (chain > 2)
                            if (!h2) {
                                o2 = take1 ? o0 : o1;
                                h2 = true;
                            } else {
                                put_direct(take1 ? o0 : o1);
                            }
                        }
                        win = take1 ? o1 : o0;
                        no = 0;
                    }
                    if (DEV_TRACE) {
                        asm volatile("" ::"d"((no > 0 ? o0.key : 0.0) + (no > 1 ? o1.key : 0.0)));
                        trace_max_warp(p, it, TR_WORK_END);
                    }
                    if (DEV_PROF) {
                        asm volatile("" ::"d"((no > 0 ? o0.key : 0.0) + (no > 1 ? o1.key : 0.0)));
                        const long long c2p = clock64();
                        ls.add(ST_CYC_PROP, c2p - c0);
                        const unsigned long long dtp = (unsigned long long)(c2p - c1);
                        atomicAdd(&ctrl->lat_hist[63 - __clzll(dtp | 1ull)], 1ull);
                    }
                }
            } else if (wi < nwS + nwF) {
                // FANS_PER_WARP candidates per warp, FAN_LANES lanes each
                const unsigned int fi = (wi - nwS) * FANS_PER_WARP + lane / FAN_LANES;
                const int sl = lane % FAN_LANES;
                if (fi < nF) {
                    const FanEv e = fev[local ? (unsigned long long)b * chF + fi : chunk_slot(s_pre[2], G, fi, chF)];
                    const RowTabs T = row_tabs<1>(p, e.row, it);
                    const unsigned long long dv = __ldcg(T.dist + e.v);
                    const ulonglong2 pk = __ldcg(T.pick + e.v);
                    const double rel = fan_rel(e);
                    const unsigned long long hi = (unsigned long long)__double_as_longlong(e.cand);
                    const unsigned long long lo = fan_tiebreak(e);
                    // the fan's span is read speculatively, in parallel with
                    // the winner check: the winner of the vertex's pick,
                    // still at the vertex's distance (a later improvement
                    // fans out on its own)
                    FanSpan f;
                    const bool span = fan_span(p, e.v, e.anchor, rel, false, f);
                    // still the vertex's distance and either the pick, or
                    // better than a stale pick (our claim lost a race to a
                    // worse candidate): the group's first lane claims it
                    // now; a tie racing the same repair may fan out twice
                    // (duplicate windows, never a missing fan)
                    const bool stale = dv == hi && (pk.x > hi || (pk.x == hi && pk.y > lo));
                    bool won = false;
                    if (stale && sl == 0) won = cas_min_u128(T.pick + e.v, hi, lo, pk);
                    const unsigned int gmask = FAN_LANES == 32 ? 0xffffffffu
                                                                : ((1u << FAN_LANES) - 1u) << (lane & ~(FAN_LANES - 1));
                    won = __shfl_sync(gmask, won, lane & ~(FAN_LANES - 1));
                    if (dv == hi && ((pk.x == hi && pk.y == lo) || won) && span) {
                        if (sl == 0) ls.add(ST_FANS);
                        const int items = f.m * f.reps;
                        if (sl < items)
                            fan_item(p, T, e.row, e.cand, f, sl % f.m, sl / f.m, false,
                                     [&](const Win &x) { o0 = x; no = 1; }, ls, p.dup_epoch + it + 1u);
                        for (int q = sl + FAN_LANES; q < items; q += FAN_LANES)
                            fan_item(p, T, e.row, e.cand, f, q % f.m, q / f.m, false, put_direct, lsd,
                                     p.dup_epoch + it + 1u);
                    }
                }
            } else {
                const unsigned int i = ((wi - nwS - nwF) << 5) + lane;
                if (i < nP) {
                    o0 = load_win(p.S, (unsigned long long)rPc * (unsigned long long)p.cap +
                                           (local ? (unsigned long long)b * ch + i : chunk_slot(s_pre[1], G, i, ch)));
                    no = 1;
                }
            }
            // route: S_{i+1} if key <= t_{i+1}, else P_{i+1}
            __syncwarp();
            if (PHASE && lane == 0) {
                const long long now = clock64();
                atomicAdd(&s_st[wi < nwS ? ST_PH_PROP : wi < nwS + nwF ? ST_PH_EVENTS : ST_PH_COMPACT],
                          (unsigned long long)(now - ph_t));
                if (wi < nwS) atomicAdd(&s_st[ST_N_SITEM], 1ull);
                ph_t = now;
            }
            const bool s0 = no > 0 && o0.key <= tn, s1 = no > 1 && o1.key <= tn;
            const bool k0 = no > 0 && !s0, k1 = no > 1 && !s1;
            const bool s2 = h2 && o2.key <= tn, k2 = h2 && !s2;
            const unsigned int ns_ = (unsigned int)s0 + (unsigned int)s1 + (unsigned int)s2;
            const unsigned int np_ = (unsigned int)k0 + (unsigned int)k1 + (unsigned int)k2;
            // warp-reduced key extremes on the top 32 bits of the (positive,
            // order-preserving) fp64 patterns, one shared atomic per warp:
            // the pool minimum rounds down, the batch maximum up -- both
            // only steer the controller
            const auto hi32 = [](double x) {
                return (unsigned int)((unsigned long long)__double_as_longlong(x) >> 32);
            };
            unsigned int hmin = k0 ? hi32(o0.key) : 0xffffffffu, hmax = s0 ? hi32(o0.key) : 0u;
            if (k1) hmin = min(hmin, hi32(o1.key));
            if (k2) hmin = min(hmin, hi32(o2.key));
            if (s1) hmax = max(hmax, hi32(o1.key));
            if (s2) hmax = max(hmax, hi32(o2.key));
            hmin = __reduce_min_sync(0xffffffffu, hmin);
            hmax = __reduce_max_sync(0xffffffffu, hmax);
            if (lane == 0) {
                if (hmin != 0xffffffffu) atomicMin(&s_pmin, (unsigned long long)hmin << 32);
                if (hmax) atomicMax(&s_smax, ((unsigned long long)hmax << 32) | 0xffffffffull);
            }
            unsigned int sa, pa;
            warp_chunk_alloc2(s_nsp, ns_, np_, sa, pa);
            if (no > 0) put_at(s0, s0 ? sa++ : pa++, o0);
            if (no > 1) put_at(s1, s1 ? sa++ : pa++, o1);
            if (h2) put_at(s2, s2 ? sa : pa, o2);
            ls.add(ST_STORED, (unsigned long long)(no + (h2 ? 1 : 0)));
            if (DEV_TRACE && wi < nwS) trace_max_warp(p, it, TR_ROUTED);
            if (DEV_TRACE && wi < nwS) trace_max_warp(p, it, TR_SCAN_END);
            if (PHASE && lane == 0) {
                const long long now = clock64();
                atomicAdd(&s_st[ST_PH_COMPACT], (unsigned long long)(now - ph_t));
                ph_t = now;
            }
            if (ls.fold_due()) ls.fold();
        }
        // publish this CTA's outputs, then the grid barrier (or, before a
        // local iteration, only a CTA barrier)
        __syncthreads();
        // a block of local iterations starts after a global one only when it
        // pays and is safe: every CTA has work (at least a warp's worth on
        // average, no chunk above twice the average -- else the CTAs holding
        // the work would run the block alone) and every chunk is at most 1/8
        // full (it must absorb a block's growth before the next grid
        // barrier can act on a grow request)
        if (!local) {
            const unsigned long long tot = (unsigned long long)nS + nP;
            const unsigned long long mx = (unsigned long long)s_maxc[0] + s_maxc[1];
            local_left = tot >= 32ull * G && mx * G <= 2ull * tot && mx * 8ull <= ch &&
                                 (unsigned long long)s_maxc[2] * 8ull <= chF
                             ? p.local_iters - 1
                             : 0;
        } else {
            --local_left;
        }
        const bool next_local = local_left > 0;
        // this iteration's totals (final after the publish barrier), read by
        // every thread: the next iteration's own counts
        const unsigned long long nsp_tot = *s_nsp;
        const unsigned int nf_tot = *s_nf;
        locS = min((unsigned int)nsp_tot, (unsigned int)ch);
        locP = min((unsigned int)(nsp_tot >> 32), (unsigned int)ch);
        locF = min(nf_tot, (unsigned int)chF);
        if (threadIdx.x == 0) {
            const int po = par ^ 1;  // parity of the next iteration's inputs
            p.ccnt[(size_t)(po * 3 + 0) * MAX_CTAS + b] = locS;
            p.ccnt[(size_t)(po * 3 + 1) * MAX_CTAS + b] = locP;
            p.ccnt[(size_t)(par * 3 + 2) * MAX_CTAS + b] = locF;
            // past half a chunk: finish this iteration, then grow the pool
            // and resume (host), instead of overflowing in a later one (a
            // CTA adds well under half a chunk per iteration)
            const unsigned long long soft = ch / 2, softF = chF / 2;
#ifndef PCH_NO_SOFT
            if ((nsp_tot & 0xffffffffull) > soft || (nsp_tot >> 32) > soft || nf_tot > softF)
                atomicExch(&ctrl->grow, 1);
#endif
            // the copy of iteration i-1 (every thread read its totals
            // before this iteration's publish barrier) serves iteration i+2
            const int kp = k3 == 0 ? 2 : k3 - 1;
            s_nsp3[kp] = 0ull;
            s_nf3[kp] = 0u;
            if (!next_local) {  // the controller's extremes, over the local block
                if (s_pmin != ~0ull) atomicMin(&nxt.pmin, s_pmin);
                if (s_smax) atomicMax(&nxt.smax, s_smax);
                s_pmin = ~0ull;
                s_smax = 0ull;
            }
            if (DEV_TRACE) trace_max(p, it, TR_A_END);
            if (blockIdx.x == 0) {
                if (p.max_iter >= 0 && it + 1 > p.max_iter) atomicExch(&ctrl->error, ERR_GUARD);
                if (globaltimer() - t_start > p.time_limit_ns) atomicExch(&ctrl->error, ERR_TIMEOUT);
            }
        }
        if (next_local) {
            // after a global iteration the other CTAs may still be reading
            // this CTA's chunks (the distributed inputs): a grid barrier
            // before it writes its parity buffers again
            // (local -> local: the publish barrier already ordered this
            // CTA's outputs before the next iteration's loads, and the
            // counters rotate)
            if (!local) {
                grid_barrier<false>(ctrl, gen, [] {});
                if (b == 0 && threadIdx.x == 0) s_st[ST_BARRIERS] += 1ull;
            } else if (ROWS) {
                __syncthreads();  // batched rows: measured faster with the CTA in step
            }
            k3 = k3 == 2 ? 0 : k3 + 1;
            ++it;
            t = tn;
            local = true;
            continue;
        }
        local = false;
        // the __syncthreads before the publish already ordered every
        // thread's outputs before thread 0's release
        grid_barrier<false>(ctrl, gen, [] {});
        if (b == 0 && threadIdx.x == 0) s_st[ST_BARRIERS] += 1ull;
        // the next iteration's inputs: S_{i+1}, P_{i+1} (parity par^1) and
        // the fan candidates of iteration i (parity par); the counts and
        // the controller's inputs are read in one round trip
        build_prefix(par ^ 1, par, &nxt);
        const int err = (int)s_c[0];
        const unsigned int ns = s_pre[0][G], np = s_pre[1][G], nf = s_pre[2][G];
        if (DEV_TRACE && it < p.trace_cap && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long *trr = p.trace + (size_t)it * TR_N;
            trr[TR_B1] = trr[TR_B_END] = trr[TR_B2] = globaltimer();
            trr[TR_NC] = (unsigned long long)ns + np;
        }
        k3 = k3 == 2 ? 0 : k3 + 1;
        ++it;
        if (err || (ns == 0 && np == 0 && nf == 0)) break;
        t = tn;
        if (s_c[3]) {
            // grow request: every CTA saw it with the counts; the inputs of
            // iteration `it` are complete in their chunks
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                ctrl->res_it = it;
                ctrl->res_t = t;
                ctrl->res_delta = delta;
            }
            break;
        }
    }
    __syncwarp();
    ls.fold();
    if (maxchild) ls.max(ST_MAXCHILD, maxchild);
    flush_stats(ctrl, s_st);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctrl->iterations = it;
        ctrl->t_final = t;
    }
}

// the instance for a solve: phase clocks only where requested; batched
// rows and single fields separately tuned
static const void *live_kernel(const Params &p) {
    const bool rows = p.rows > 1;
    if (p.phase) return rows ? (const void *)pch_live<true, true> : (const void *)pch_live<true, false>;
    return rows ? (const void *)pch_live<false, true> : (const void *)pch_live<false, false>;
}

// ---------------------------------------------------------------------------
// initialisation kernels

__global__ void k_init_state(Params p, const int64_t *src, int nsrc) {
    const long long n = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nvr = (long long)p.nv * p.rows, nher = (long long)p.nhe * p.rows;
    // a seed field (single field only) starts every vertex at a known
    // path length: ICH pruning against it is as valid as against the
    // solve's own distances, so the result is min(seed, new field)
    const double *seed = p.rows == 1 ? p.seed : nullptr;
    for (long long v = t0; v < nvr; v += n) {
        p.dist_new[v] = (unsigned long long)__double_as_longlong(seed ? seed[v] : INFINITY);
        p.fanpick[0][v] = make_ulonglong2(~0ull, ~0ull);
    }
    if (!p.live) {
        for (long long v = t0; v < p.nv; v += n) {
            p.dist_cur[v] = seed ? seed[v] : INFINITY;
            p.fanpick[1][v] = make_ulonglong2(~0ull, ~0ull);
            p.fanpick[2][v] = make_ulonglong2(~0ull, ~0ull);
        }
        for (long long j = t0; j < p.nhe; j += n) p.split_cur[j] = make_double2(INFINITY, 0.0);
    }
    for (long long j = t0; j < nher; j += n) p.split_new[j] = make_ulonglong2(ord64(INFINITY), ord64(0.0));
    for (long long b = t0; b < 2 * (NBINS + 1); b += n) {
        (b <= NBINS ? p.hist[0][b] : p.hist[1][b - NBINS - 1]) = 0u;
    }
    if (t0 == 0)
        for (int q = 0; q < NSLOT; ++q) p.ctrl->slot[q].pmin = ~0ull;
}

// one field (rows == 1: the union of the sources, reference run_pch) or
// one field per source (batched rows: source i seeds row i)
__global__ void k_set_sources(Params p, const int64_t *src, int nsrc) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nsrc) {
        const int64_t s = src[i];
        // device-resident source lists (pch_run_device) are validated
        // here: an out-of-range index fails the solve with PCH_ERR_SOURCE
        if (s < 0 || s >= p.nv) {
            atomicExch(&p.ctrl->error, ERR_SOURCE);
            return;
        }
        const size_t r = p.rows > 1 ? (size_t)i : 0;
        if (!p.live) p.dist_cur[s] = 0.0;
        p.dist_new[r * p.nv + s] = 0ull;
    }
}

// source windows: a full fan around every source (engine.py:402 via
// geom.py:524), into the first batch S_0
__global__ void k_source_windows(Params p, const int64_t *src, int nsrc) {
    __shared__ unsigned long long s_st[N_ST];
    stats_init(s_st);
    LocalStats ls{s_st, true};
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    Ctrl *ctrl = p.ctrl;
    // the live solver reads its batch in per-CTA chunks: source i seeds
    // chunk i % G (G = the solver's grid); the deterministic one linearly
    const unsigned long long G = (unsigned long long)p.live_grid;
    const unsigned long long ch = G ? (unsigned long long)p.cap / G : 0ull;
    auto emit = [&](const Win &c) {
        if (p.live) {
            const unsigned long long c0 = (unsigned long long)i % G;
            const unsigned int k = atomicAdd(p.ccnt + c0, 1u);  // parity 0, S counts
            if (k < ch) store_win(p.S, c0 * ch + k, c);
            else atomicExch(&ctrl->error, ERR_OVERFLOW);
        } else {
            unsigned long long slot = atomicAdd(&ctrl->slot[0].nS, 1ull);
            if ((long long)slot < p.cap) store_win(p.S, slot, c);
            else atomicExch(&ctrl->error, ERR_OVERFLOW);
        }
        ls.add(ST_STORED);
    };
    if (i < nsrc && src[i] >= 0 && src[i] < p.nv) {
        int32_t s = (int32_t)src[i];
        if ((__double_as_longlong(__ldg(&p.fanhdr[s].meta_bits)) >> 32) & 0x7fffffffll)
        {
            const uint32_t r = p.rows > 1 ? (uint32_t)i : 0u;
            emit_fan(p, row_tabs(p, r, 0), r, s, 0.0, 0, 0.0, true, emit, ls);
        }
    }
    flush_stats(ctrl, s_st);
}

// Pool growth without a restart (live solver): the inputs of the resumed
// iteration -- batch S, pool P (both parity `par`) and the fan candidates
// of the previous iteration (parity par^1) -- move from their chunks of
// the old capacity (ch, chF per CTA) to the same chunks of the new one.
__global__ void k_migrate_chunks(WinSoA S_old, WinSoA P_old, const FanEv *F_old, WinSoA S_new, WinSoA P_new,
                                 FanEv *F_new, const unsigned int *ccnt, int par, int G,
                                 unsigned long long ch_old, unsigned long long ch_new,
                                 unsigned long long chF_old, unsigned long long chF_new) {
    const int b = blockIdx.y;  // chunk
    const unsigned int nS = ccnt[(size_t)(par * 3 + 0) * MAX_CTAS + b];
    const unsigned int nP = ccnt[(size_t)(par * 3 + 1) * MAX_CTAS + b];
    const unsigned int nF = ccnt[(size_t)((par ^ 1) * 3 + 2) * MAX_CTAS + b];
    for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(max(nS, nP), nF);
         i += gridDim.x * blockDim.x) {
        if (i < nS) store_win(S_new, b * ch_new + i, load_win(S_old, b * ch_old + i));
        if (i < nP) store_win(P_new, b * ch_new + i, load_win(P_old, b * ch_old + i));
        if (i < nF) F_new[b * chF_new + i] = F_old[b * chF_old + i];
    }
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
    double mean_alt = 1.0;  // mean smallest altitude of a face (2 area / longest edge)
    FaceRec *face = nullptr;
    FanRec *fan = nullptr;
    FanHdr *fanhdr = nullptr;
    double *anchor_wlo = nullptr;
    double2 *apex_xy = nullptr;
    size_t mesh_bytes = 0;
    // workspace
    long long cap = 0;
    int rows_alloc = 0;
    std::vector<void *> ws;
    Params prm{};
    int64_t *d_src = nullptr;
    size_t src_cap = 0;
    char *fps_buf = nullptr;  // farthest-point sampling scratch (grows)
    size_t ws_bytes = 0;      // bytes held by the solve workspace
    size_t fps_cap = 0;
    double *d_out = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    int grid = 0, grid_live = 0;
    double clock_mhz = 0.0;  // SM clock (cudaDevAttrClockRate) for cycle -> time
    ulonglong2 *dup_tab = nullptr;  // fan-window fingerprints (dedupe), DUP_SLOTS entries
    unsigned int solve_seq = 0;     // epochs of the dedupe table
    unsigned long long *trace = nullptr;  // PCH_TRACE development timeline
    long long trace_cap = 0;
};

// the final distance field of the last solve: the shadow field holds it in
// both solvers (fp64 bit patterns of non-negative distances, +inf for
// unreachable), the frozen copy only in the two-barrier one
static const double *field_ptr(const pch_mesh *m) {
    return reinterpret_cast<const double *>(m->prm.dist_new);
}

static void free_ws(pch_mesh *m) {
    for (void *q : m->ws) cudaFree(q);
    m->ws.clear();
    m->cap = 0;
    m->ws_bytes = 0;
}

template <typename T>
static int ws_alloc(pch_mesh *m, T **out, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) return fail(PCH_ERR_NOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
    m->ws_bytes += std::max<size_t>(count, 1) * sizeof(T);
    m->ws.push_back(q);
    *out = static_cast<T *>(q);
    return PCH_OK;
}

// The four window sets share each column's allocation: region r of a
// column starts at r * cap (S = 0, S2 = 1, X = 2, Y = 3), so the one-barrier
// solver addresses every set through p.S's pointers plus a region offset --
// no per-window select between two sets' eight column pointers.
static int alloc_soa4(pch_mesh *m, Params &p, long long cap) {
    int rc;
    WinSoA &W = p.S;
    if ((rc = ws_alloc(m, &W.hv, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.vr, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.b0, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.b1, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.d0, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.d1, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.d, 4 * cap))) return rc;
    if ((rc = ws_alloc(m, &W.key, 4 * cap))) return rc;
    WinSoA *sets[3] = {&p.S2, &p.X, &p.Y};
    for (int r = 1; r < 4; ++r) {
        WinSoA &R = *sets[r - 1];
        R.hv = W.hv + r * cap;
        R.vr = W.vr + r * cap;
        R.b0 = W.b0 + r * cap;
        R.b1 = W.b1 + r * cap;
        R.d0 = W.d0 + r * cap;
        R.d1 = W.d1 + r * cap;
        R.d = W.d + r * cap;
        R.key = W.key + r * cap;
    }
    return PCH_OK;
}

// `exact`: an explicit pool capacity (EngineConfig.pool_capacity) is
// honoured even when the mesh's workspace is larger
static int ensure_ws(pch_mesh *m, long long cap, int rows, bool exact = false) {
    if ((exact ? m->cap == cap : m->cap >= cap) && m->rows_alloc >= rows) return PCH_OK;
    if (!exact) cap = std::max(cap, m->cap);
    rows = std::max(rows, m->rows_alloc);
    free_ws(m);
    Params &p = m->prm;
    int rc;
    p = Params{};
    p.face = m->face;
    p.fan = m->fan;
    p.fanhdr = m->fanhdr;
    p.anchor_wlo = m->anchor_wlo;
    p.apex_xy = m->apex_xy;
    p.nv = m->nv;
    p.nhe = m->nhe;
    if ((rc = ws_alloc(m, &p.dist_cur, m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.dist_new, (size_t)m->nv * rows))) return rc;
    if ((rc = ws_alloc(m, &p.split_cur, m->nhe))) return rc;
    if ((rc = ws_alloc(m, &p.split_new, (size_t)m->nhe * rows))) return rc;
    if ((rc = ws_alloc(m, &p.fanpick[0], (size_t)m->nv * rows))) return rc;
    if ((rc = ws_alloc(m, &p.fanpick[1], m->nv))) return rc;
    if ((rc = ws_alloc(m, &p.fanpick[2], m->nv))) return rc;
    // one entry per improving event of an iteration (<= 3 per propagated
    // window, <= 1 angle claim), duplicates allowed
    p.tvcap = 3 * cap + m->nv;
    p.tecap = cap + m->nhe;
    if ((rc = ws_alloc(m, &p.tv_list, p.tvcap))) return rc;
    if ((rc = ws_alloc(m, &p.te_list, p.tecap))) return rc;
    p.fancap = std::max<long long>(cap, 1 << 16);
    if ((rc = ws_alloc(m, &p.fanev[0], p.fancap))) return rc;
    if ((rc = ws_alloc(m, &p.fanev[1], p.fancap))) return rc;
    if ((rc = ws_alloc(m, &p.fanev[2], p.fancap))) return rc;
    if ((rc = alloc_soa4(m, p, cap))) return rc;
    if ((rc = ws_alloc(m, &p.hist[0], NBINS + 1))) return rc;
    if ((rc = ws_alloc(m, &p.hist[1], NBINS + 1))) return rc;
    if ((rc = ws_alloc(m, &p.fine[0], 2 * FINE_N))) return rc;
    p.fine[1] = p.fine[0] + FINE_N;
    if ((rc = ws_alloc(m, &p.ctrl, 1))) return rc;
    if ((rc = ws_alloc(m, &p.ccnt, 2 * 3 * MAX_CTAS))) return rc;
    p.cap = cap;
    m->cap = cap;
    m->rows_alloc = rows;
    return PCH_OK;
}

// Enlarge the cap-sized buffers (window SoAs, fan candidates, event lists)
// to `cap`, moving the resumed iteration's inputs (parity `par`) chunk by
// chunk; the distance / angle-split / pick tables and the counters stay.
static int grow_ws(pch_mesh *m, long long cap, int par, cudaStream_t st) {
    Params &p = m->prm;
    const int G = m->grid_live;
    const long long old_cap = p.cap, old_fancap = p.fancap;
    // (the four window sets live in p.S's column allocations)
    std::vector<void *> old = {p.S.hv, p.S.vr, p.S.b0, p.S.b1, p.S.d0, p.S.d1, p.S.d, p.S.key,
                               p.fanev[0], p.fanev[1], p.fanev[2], p.tv_list, p.te_list};
    const WinSoA oX = p.X, oY = p.Y, oS = p.S, oS2 = p.S2;
    FanEv *oF[3] = {p.fanev[0], p.fanev[1], p.fanev[2]};
    int rc;
    if ((rc = alloc_soa4(m, p, cap))) return rc;
    p.fancap = std::max<long long>(cap, 1 << 16);
    for (int q = 0; q < 3; ++q)
        if ((rc = ws_alloc(m, &p.fanev[q], p.fancap))) return rc;
    p.tvcap = 3 * cap + m->nv;
    p.tecap = cap + m->nhe;
    if ((rc = ws_alloc(m, &p.tv_list, p.tvcap)) || (rc = ws_alloc(m, &p.te_list, p.tecap))) return rc;
    const unsigned long long ch_old = old_cap / G, ch_new = cap / G;
    const unsigned long long chF_old = old_fancap / G, chF_new = p.fancap / G;
    k_migrate_chunks<<<dim3(64, G), 256, 0, st>>>(par ? oS2 : oS, par ? oY : oX, oF[par ^ 1], par ? p.S2 : p.S,
                                                  par ? p.Y : p.X, p.fanev[par ^ 1], p.ccnt, par, G, ch_old,
                                                  ch_new, chF_old, chF_new);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    for (void *q : old) {
        cudaFree(q);
        m->ws.erase(std::remove(m->ws.begin(), m->ws.end(), q), m->ws.end());
    }
    m->ws_bytes -= (size_t)old_cap * 4 * 72 + (size_t)old_fancap * 3 * sizeof(FanEv) +
                   sizeof(int32_t) * ((size_t)(3 * old_cap + m->nv) + (size_t)(old_cap + m->nhe));
    p.cap = cap;
    m->cap = cap;
    return PCH_OK;
}

// rows == 1: one field from the union of the sources (reference run_pch);
// rows == nsrc > 1: one field per source, solved together (batched rows,
// live solver only)
static int solve(pch_mesh *m, const int64_t *d_src, int nsrc, const pch_config *cfg,
                 cudaStream_t st, pch_stats *stats, int rows = 1, const double *d_seed = nullptr) {
    if (cfg->k < 1) return fail(PCH_ERR_CONFIG, "k must be >= 1");
    if (!(cfg->epsilon_window > 0.0)) return fail(PCH_ERR_CONFIG, "epsilon_window must be > 0");
    if (!(cfg->fan_margin >= 0.0 && cfg->fan_margin < 0.1)) return fail(PCH_ERR_CONFIG, "fan_margin must be in [0, 0.1)");
    if (cfg->fan_mode != 0 && cfg->fan_mode != 1) return fail(PCH_ERR_CONFIG, "fan_mode must be clip or full_edges");
    if (cfg->chain < 0) return fail(PCH_ERR_CONFIG, "chain must be >= 0");
    if (rows > 1 && (cfg->flags & PCH_FLAG_DETERMINISTIC))
        return fail(PCH_ERR_CONFIG, "batched rows need the live solver");
    // the pool holds every row's wavefront: scale the first guess with rows
    // the live solver grows its pool at an iteration boundary and continues
    // (grow_ws), so the first capacity only needs to cover the early
    // wavefront: a quarter window per half-edge (peak active pools measured
    // 0.4M windows on the 16M-face sphere, 3M for 32 torus rows)
    long long cap = cfg->pool_capacity > 0
                        ? cfg->pool_capacity
                        : std::max<long long>(DEFAULT_POOL_MIN, m->nhe / 4) * std::max(1, rows / 4);
    if (cfg->pool_capacity <= 0 && m->cap > cap) cap = m->cap;
    // every per-CTA chunk of the live solver holds at least 8 windows
    cap = std::max<long long>(cap, 8ll * m->grid_live);
    bool exact = cfg->pool_capacity > 0;
    int regrows = 0, restarts = 0;
    for (;;) {
        int rc = ensure_ws(m, cap, rows, exact);
        if (rc) return rc;
        exact = false;  // a rerun after a hard overflow only grows
        Params p = m->prm;
        p.seed = d_seed;
        p.K = cfg->k;
        p.eps_win = cfg->epsilon_window;
        // angular tiny-window rule within 40 mean edges of the pseudo
        // source (pch_device.cuh make_child); the flag restores geom.py:133
        p.inv_r0 = (cfg->flags & PCH_FLAG_ABSOLUTE_TINY) ? 1e300 : 1.0 / (TINY_R0_EDGES * m->mean_edge);
        if (const char *r0 = getenv("PCH_TINY_R0"))  // development: radius in mean edges
            if (!(cfg->flags & PCH_FLAG_ABSOLUTE_TINY)) p.inv_r0 = 1.0 / (atof(r0) * m->mean_edge);
        p.eps_win2 = p.eps_win * p.eps_win;
        p.inv_r02 = p.inv_r0 * p.inv_r0;
        p.fan_widen = cfg->fan_margin;
        // one grid barrier every LOCAL_ITERS iterations, the others CTA-local
        // (measured: terrain1m 7.64 -> 7.06 ms, sphere16m 112 -> 102 ms at 8;
        // with local iterations that skip the prefix tables, 12 for single
        // fields: sphere16m 84.0 -> 81.6 ms, terrain1m / torus500k equal,
        // 16 lets terrain1m's CTAs drift apart; batched rows stay at 8)
        p.local_iters = rows > 1 ? LOCAL_ITERS_ROWS : LOCAL_ITERS;
        if (const char *li = getenv("PCH_LOCAL_ITERS")) p.local_iters = std::max(1, atoi(li));  // development
        p.exact_select = cfg->selection_mode == 0 ? 1 : 0;
        // dedupe epochs: solve sequence << 20 plus the iteration (+1), so a
        // table entry never matches a window of another solve
        if (!m->dup_tab && (cfg->flags & PCH_FLAG_DEDUPE)) {
            CK(cudaMalloc(&m->dup_tab, sizeof(ulonglong2) * DUP_SLOTS));
            CK(cudaMemsetAsync(m->dup_tab, 0, sizeof(ulonglong2) * DUP_SLOTS, st));
        }
        m->solve_seq = (m->solve_seq + 1) & 0xfffu;
        if (m->solve_seq == 0) {  // wrapped: clear the stale epochs once
            m->solve_seq = 1;
            CK(cudaMemsetAsync(m->dup_tab, 0, sizeof(ulonglong2) * DUP_SLOTS, st));
        }
        p.dup_tab = (cfg->flags & PCH_FLAG_DEDUPE) ? m->dup_tab : nullptr;
        p.dup_mask = DUP_SLOTS - 1;
        p.dup_epoch = m->solve_seq << 20;
        p.phase = (cfg->flags & PCH_FLAG_PHASE_TIMES) ? 1 : 0;
        p.w0 = m->mean_edge / 64.0;
        p.max_iter = cfg->max_iterations;  // < 0: no cap (reference max_iterations=None)
        p.time_limit_ns = cfg->time_limit_s > 0.0 ? (unsigned long long)(cfg->time_limit_s * 1e9) : ~0ull;
        p.fan_full = cfg->fan_mode == 1;
        p.recheck = (cfg->flags & PCH_FLAG_NO_RECHECK) ? 0 : 1;
        p.live = (cfg->flags & PCH_FLAG_DETERMINISTIC) ? 0 : 1;
        p.rows = rows;
        // step controller bounds (mean edge lengths): the floor keeps wide
        // wavefronts (tori, large spheres: far more than k windows per face
        // layer) from splitting one layer over many iterations; the cap
        // keeps narrow ones (terrain: fewer than k windows per layer) from
        // selecting several layers out of order; measured over the bench
        // meshes (profiles/r01_controller.md)
        // chaining: up to `chain` face crossings per iteration, for single
        // fields and batched rows alike; a third crossing pays on large
        // meshes (deep wavefronts), not on small ones where it only
        // lengthens the iteration (profiles/r01_controller.md)
        // a fourth on anisotropic meshes (mean smallest face altitude below
        // half a mean edge: a crossing advances less distance there)
        // six on anisotropic ones (mean smallest face altitude below half a
        // mean edge: a crossing advances less distance; torus500k 11.1 ->
        // 10.55 ms, its rows 8.55 -> 8.20 ms/row, knot4m 384 -> 359 ms;
        // on isotropic meshes longer chains only add out-of-order windows)
        p.chain = cfg->chain > 0 ? cfg->chain
                                 : (m->nhe / 3 >= LONG_CHAIN_FACES
                                        ? (m->mean_alt < 0.5 * m->mean_edge ? ANISO_CHAIN : DEFAULT_CHAIN + 1)
                                        : DEFAULT_CHAIN);
        if (const char *ch = getenv("PCH_CHAIN")) p.chain = std::max(1, atoi(ch));  // development
        p.delta0 = m->mean_edge;
        // skinny faces (torus-knot tubes): a step of several face
        // altitudes selects layers out of order and doubles the windows.
        // The bounds are per two crossings and scale with the chain length.
        const double per_cross = 0.5 * p.chain;
        p.delta_min = per_cross * std::min(DELTA_FLOOR * m->mean_edge, ALT_FLOOR * m->mean_alt);
        // long chains select deeper per iteration: a tighter cap keeps the
        // out-of-order share down (profiles/r01_controller.md)
        p.delta_max = per_cross * (p.chain > DEFAULT_CHAIN ? DELTA_CAP_LONG : DELTA_CAP) * m->mean_edge;
        if (const char *fd = getenv("PCH_DELTA")) {  // development: fixed step
            const double dlt = atof(fd) * m->mean_edge;
            if (dlt > 0.0) p.delta0 = p.delta_min = p.delta_max = dlt;
        }
        if (const char *fm = getenv("PCH_DELTA_MIN")) {  // development: step floor
            const double dlt = atof(fm) * m->mean_edge;
            if (dlt > 0.0) p.delta_min = dlt;
        }
        if (const char *fx = getenv("PCH_DELTA_MAX")) {  // development: step cap
            const double dlt = atof(fx) * m->mean_edge;
            if (dlt > 0.0) p.delta_max = dlt;
        }
        p.delta0 = std::min(std::max(p.delta0, p.delta_min), p.delta_max);
        p.prof = getenv("PCH_PROFILE") ? 1 : 0;
        const char *trace_path = getenv("PCH_TRACE");
        if (trace_path && !m->trace) {
            m->trace_cap = 1 << 17;
            CK(cudaMalloc(&m->trace, sizeof(unsigned long long) * TR_N * m->trace_cap));
        }
        p.trace = trace_path ? m->trace : nullptr;
        p.trace_cap = trace_path ? m->trace_cap : 0;
        if (p.trace) CK(cudaMemsetAsync(p.trace, 0, sizeof(unsigned long long) * TR_N * p.trace_cap, st));
        CK(cudaEventRecord(m->ev0, st));
        CK(cudaMemsetAsync(p.ctrl, 0, sizeof(Ctrl), st));
        p.live_grid = m->grid_live;
        if (p.live) CK(cudaMemsetAsync(p.ccnt, 0, sizeof(unsigned int) * 2 * 3 * MAX_CTAS, st));
        if (!p.live && p.exact_select) CK(cudaMemsetAsync(p.fine[0], 0, sizeof(unsigned int) * 2 * FINE_N, st));
        k_init_state<<<4 * 148, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        k_set_sources<<<(nsrc + 255) / 256, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        k_source_windows<<<(nsrc + 255) / 256, 256, 0, st>>>(p, d_src, nsrc);
        CK(cudaGetLastError());
        CK(cudaEventRecord(m->ev1, st));
        void *args[] = {&p};
        if (p.live)
        {
            const void *kern = live_kernel(p);
            CK(cudaLaunchCooperativeKernel(kern, dim3(p.live_grid), dim3(TPB), args, 0, st));
        }
        else
            CK(cudaLaunchCooperativeKernel((const void *)pch_persistent, dim3(m->grid), dim3(TPB), args, 0, st));
        CK(cudaEventRecord(m->ev2, st));
        CK(cudaStreamSynchronize(st));
        Ctrl c;
        CK(cudaMemcpy(&c, p.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
        // a chunk passed its soft limit: the live solver stopped at an
        // iteration boundary with every window in place -- grow the pool,
        // move the next iteration's inputs, continue where it stopped
        while (p.live && c.error == ERR_NONE && c.grow) {
            if (cap >= (1ll << 31)) return fail(PCH_ERR_NOMEM, "window pool at maximum capacity");
            int rc2 = grow_ws(m, cap * 2, (int)(c.res_it & 1), st);
            if (rc2) return rc2;
            cap *= 2;
            regrows++;
            p.X = m->prm.X;
            p.Y = m->prm.Y;
            p.S = m->prm.S;
            p.S2 = m->prm.S2;
            for (int q = 0; q < 3; ++q) p.fanev[q] = m->prm.fanev[q];
            p.fancap = m->prm.fancap;
            p.tv_list = m->prm.tv_list;
            p.te_list = m->prm.te_list;
            p.tvcap = m->prm.tvcap;
            p.tecap = m->prm.tecap;
            p.cap = cap;
            p.resume = 1;
            CK(cudaMemsetAsync(&p.ctrl->grow, 0, sizeof(int), st));
            CK(cudaMemsetAsync(&p.ctrl->bar_count, 0, sizeof(unsigned int), st));
            void *args2[] = {&p};
            const void *kern = live_kernel(p);
            CK(cudaLaunchCooperativeKernel(kern, dim3(p.live_grid), dim3(TPB), args2, 0, st));
            CK(cudaEventRecord(m->ev2, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemcpy(&c, p.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
        }
        if (c.error == ERR_OVERFLOW) {
            // hard overflow (a chunk filled within one iteration, the
            // source windows, or the two-barrier solver): rerun at 2x
            if (cap >= (1ll << 31)) return fail(PCH_ERR_NOMEM, "window pool overflow at maximum capacity");
            cap *= 2;
            regrows++;
            restarts++;
            continue;
        }
        if (p.trace) {
            long long n = std::min<long long>(c.iterations, p.trace_cap);
            std::vector<unsigned long long> h((size_t)n * TR_N);
            CK(cudaMemcpy(h.data(), p.trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
            if (FILE *f = fopen(trace_path, "wb")) {
                fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
                fclose(f);
            }
        }
        if (p.prof) {
            fprintf(stderr, "PCH_PROFILE CAS: angle %llu calls %llu tries, fan %llu calls %llu tries\n",
                    c.st[ST_CAS_ANGLE_CALLS], c.st[ST_CAS_ANGLE_TRIES], c.st[ST_CAS_FAN_CALLS],
                    c.st[ST_CAS_FAN_TRIES]);
            fprintf(stderr, "PCH_PROFILE propagation latency log2(cycles) histogram:");
            for (int b = 0; b < 64; ++b)
                if (c.lat_hist[b]) fprintf(stderr, " [2^%d]=%llu", b, c.lat_hist[b]);
            fprintf(stderr, "\n");
            const unsigned long long *q = c.st;
            double np_ = (double)std::max<unsigned long long>(q[ST_PROPAGATED] + q[ST_RECHECK], 1);
            fprintf(stderr,
                    "PCH_PROFILE cycles/unit: prop %.0f pool %.0f "
                    "fanspan %.0f/fan fanitem %.0f part %.0f | n_prop %.0f n_pool %llu n_fanitem %llu "
                    "n_part %llu\n",
                    q[ST_CYC_PROP] / np_,
                    q[ST_CYC_POOL] / (double)std::max<unsigned long long>(q[ST_N_POOL], 1),
                    q[ST_CYC_FANSPAN] / (double)std::max<unsigned long long>(q[ST_FANS], 1),
                    q[ST_CYC_FANITEM] / (double)std::max<unsigned long long>(q[ST_N_FANITEM], 1),
                    q[ST_CYC_PART] / (double)std::max<unsigned long long>(q[ST_N_PART], 1), np_,
                    q[ST_N_POOL], q[ST_N_FANITEM], q[ST_N_PART]);
        }
        if (c.error == ERR_GUARD)
            return fail(PCH_ERR_GUARD, "iteration cap " + std::to_string(cfg->max_iterations) + " exceeded");
        if (c.error == ERR_TIMEOUT) return fail(PCH_ERR_GUARD, "device wall-time guard tripped");
        if (c.error == ERR_SOURCE) return fail(PCH_ERR_SOURCE, "invalid source index in the device source list");
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
            stats->pruned_duplicate += c.st[ST_PRUNE_DUP];
            stats->pruned_recheck += c.st[ST_RECHECK];
            stats->total_windows_pruned += c.st[ST_PRUNE_ICH] + c.st[ST_PRUNE_SPLIT] +
                                           c.st[ST_PRUNE_TINY] + c.st[ST_PRUNE_DEGEN] + c.st[ST_PRUNE_DUP];
            stats->windows_stored += c.st[ST_STORED];
            stats->max_children_per_window = std::max<int64_t>(stats->max_children_per_window, c.st[ST_MAXCHILD]);
            stats->events_created += c.st[ST_EV_CREATED];
            stats->events_applied += c.st[ST_EV_APPLIED];
            stats->peak_active_pool = std::max<int64_t>(stats->peak_active_pool, c.st[ST_PEAK]);
            stats->fans_emitted += c.st[ST_FANS];
            stats->buffer_regrows += regrows;
            stats->pool_restarts += restarts;
            stats->grid_barriers += c.st[ST_BARRIERS];
            stats->time_total_ms += t_all;
            stats->time_kernel_ms += t_k;
            // phase shares of the kernel time from the warp-cycle attribution
            const double ph[4] = {(double)c.st[ST_PH_SELECT], (double)c.st[ST_PH_PROP],
                                  (double)c.st[ST_PH_COMPACT], (double)c.st[ST_PH_EVENTS]};
            const double phs = ph[0] + ph[1] + ph[2] + ph[3];
            if (c.st[ST_N_SITEM] > 0 && m->clock_mhz > 0.0)
                stats->prop_item_us = (double)c.st[ST_PH_PROP] / (double)c.st[ST_N_SITEM] / m->clock_mhz;
            if (phs > 0.0) {
                stats->time_select_ms += t_k * ph[0] / phs;
                stats->time_propagate_ms += t_k * ph[1] / phs;
                stats->time_compact_ms += t_k * ph[2] / phs;
                stats->time_events_ms += t_k * ph[3] / phs;
            }
        }
        return PCH_OK;
    }
}

// ---------------------------------------------------------------------------
// farthest-point sampling: argmax of the min-field, on the device

// (distance, vertex) order of the greedy pick: larger distance first
// (+inf = a component no sample reaches yet), then the lower vertex index
__device__ __forceinline__ bool fps_better(double d, long long v, double bd, long long bv) {
    return d > bd || (d == bd && v < bv);
}

__device__ __forceinline__ void fps_warp_best(double &bd, long long &bv) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double d = __shfl_down_sync(0xffffffffu, bd, o);
        const long long v = __shfl_down_sync(0xffffffffu, bv, o);
        if (fps_better(d, v, bd, bv)) {
            bd = d;
            bv = v;
        }
    }
}

// stage 1: one (distance, vertex) candidate per block
__global__ void k_fps_argmax1(const double *field, long long nv, double *bd_out, long long *bv_out) {
    __shared__ double sd[32];
    __shared__ long long sv[32];
    double bd = -1.0;
    long long bv = LLONG_MAX;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
         v += (long long)gridDim.x * blockDim.x) {
        const double d = __ldg(field + v);
        if (fps_better(d, v, bd, bv)) {
            bd = d;
            bv = v;
        }
    }
    fps_warp_best(bd, bv);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sd[w] = bd;
        sv[w] = bv;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        bd = lane < nw ? sd[lane] : -1.0;
        bv = lane < nw ? sv[lane] : LLONG_MAX;
        fps_warp_best(bd, bv);
        if (lane == 0) {
            bd_out[blockIdx.x] = bd;
            bv_out[blockIdx.x] = bv;
        }
    }
}

// stage 2: one warp reduces the block candidates into the next sample
__global__ void k_fps_argmax2(const double *bd_in, const long long *bv_in, int nb, int64_t *next) {
    double bd = -1.0;
    long long bv = LLONG_MAX;
    for (int i = threadIdx.x; i < nb; i += 32)
        if (fps_better(bd_in[i], bv_in[i], bd, bv)) {
            bd = bd_in[i];
            bv = bv_in[i];
        }
    fps_warp_best(bd, bv);
    if (threadIdx.x == 0) *next = (int64_t)bv;
}

// ---------------------------------------------------------------------------
// latency / peak probes (bench roofline denominators, pch_probe)

// the solver's grid barrier alone, `n` times, on a cooperative grid shaped
// like the live solver's
__global__ void __launch_bounds__(TPB, 1) k_probe_barrier(Ctrl *c, int n) {
    unsigned int gen = 0;
    for (int i = 0; i < n; ++i) grid_barrier<true>(c, gen, [] {});
}

// FP64 FMA throughput: 8 independent dependent chains per thread
__global__ void k_probe_fp64(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5) out[0] = s;  // keeps the chains live
}

// ---------------------------------------------------------------------------
// mesh construction: FaceRec / FanRec tables from the SurfaceMesh arrays

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
    std::vector<FaceRec> face(n_faces);
    double lsum = 0.0;
    auto vflag = [&](int64_t v) -> uint32_t {
        return (uint32_t)v | (vertex_class[v] == 2 ? SADDLE_BIT : 0u);
    };
    for (int64_t f = 0; f < n_faces; ++f) {
        FaceRec &r = face[f];
        for (int a = 0; a < 3; ++a) {
            const int64_t j = 3 * f + a;
            lsum += length[j];
            r.len[a] = length[j];
            r.vid[a] = vflag(origin[j]);
            r.opp[a] = (int32_t)opposite[j];
            r.apx[a] = opposite[j] >= 0 ? vflag(origin[prv_he(opposite[j])]) : 0u;
        }
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
            f.cho = (int32_t)opposite[che];
            f.capx = opposite[che] >= 0 ? vflag(origin[prv_he(opposite[che])]) : 0u;
            f.pid = (int32_t)origin[che];
            f.qid = (int32_t)origin[hprev];
            f.sad = (vertex_class[origin[che]] == 2 ? 1u : 0u) | (vertex_class[origin[hprev]] == 2 ? 2u : 0u);
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
    std::vector<FanHdr> hdr(n_vertices);
    std::vector<double> awlo(nhe);
    for (int64_t v = 0; v < n_vertices; ++v) {
        const long long m_ = fan_off[v + 1] - fan_off[v];
        const long long meta = (long long)(uint32_t)fan_off[v] | (m_ << 32) |
                               (interior[v] ? (long long)(1ull << 63) : 0ll);
        hdr[v].theta = theta[v];
        std::memcpy(&hdr[v].meta_bits, &meta, sizeof(meta));
    }
    for (int64_t j = 0; j < nhe; ++j) {
        const int64_t v = origin[j];
        awlo[j] = fan[fan_off[v] + fanpos[j]].wlo;
    }

    // precomputed unfolding: the apex of face(h) in the frame of edge h
    // (origin(h) at 0, dest(h) at (|h|, 0), apex below the edge) -- the far
    // triangle of every window on opposite(h) (geom.py:390-396), computed
    // once instead of a division and a square root per crossing
    std::vector<double2> apex(nhe);
    for (int64_t h = 0; h < nhe; ++h) {
        const double ell = length[h], lan = length[nxt_he(h)], lpv = length[prv_he(h)];
        const double dx = 0.5 * (ell * ell + lan * lan - lpv * lpv) / ell;
        const double dy2 = lan * lan - dx * dx;
        apex[h] = make_double2(dx, dy2 > 0.0 ? -std::sqrt(dy2) : 0.0);
    }

    pch_mesh *m = new pch_mesh();
    m->device = device;
    m->nv = (int32_t)n_vertices;
    m->nhe = (int32_t)nhe;
    m->mean_edge = lsum / (double)nhe;
    {
        double asum = 0.0;
        const int64_t nf = nhe / 3;
        for (int64_t f = 0; f < nf; ++f) {
            const double a = length[3 * f], b = length[3 * f + 1], c = length[3 * f + 2];
            const double s = 0.5 * (a + b + c);
            const double area = std::sqrt(std::max(0.0, s * (s - a) * (s - b) * (s - c)));
            asum += 2.0 * area / std::max(std::max(a, b), std::max(c, 1e-300));
        }
        m->mean_alt = nf > 0 ? asum / (double)nf : m->mean_edge;
    }
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
    if ((e = up((void **)&m->face, face.data(), sizeof(FaceRec) * n_faces)) != cudaSuccess ||
        (e = up((void **)&m->fan, fan.data(), sizeof(FanRec) * fan.size())) != cudaSuccess ||
        (e = up((void **)&m->fanhdr, hdr.data(), sizeof(FanHdr) * n_vertices)) != cudaSuccess ||
        (e = up((void **)&m->anchor_wlo, awlo.data(), sizeof(double) * nhe)) != cudaSuccess ||
        (e = up((void **)&m->apex_xy, apex.data(), sizeof(double2) * nhe)) != cudaSuccess)
        return cleanup(PCH_ERR_CUDA, std::string("mesh upload: ") + cudaGetErrorString(e));
    if ((e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreate(&m->ev0)) != cudaSuccess || (e = cudaEventCreate(&m->ev1)) != cudaSuccess ||
        (e = cudaEventCreate(&m->ev2)) != cudaSuccess)
        return cleanup(PCH_ERR_CUDA, std::string("stream/event: ") + cudaGetErrorString(e));
    int nsm = 0, per_sm = 0, per_sm_live = 0, khz = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
    m->clock_mhz = khz / 1000.0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pch_persistent, TPB, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_live, pch_live<true, true>, TPB, 0);
    if (per_sm < 1 || per_sm_live < 1) return cleanup(PCH_ERR_CUDA, "persistent kernel cannot be resident");
    // persistent grids: every SM, as many co-resident CTAs as fit (<= 4)
    m->grid = nsm * std::min(per_sm, 4);
    m->grid_live = nsm * std::min(per_sm_live, 4);
    *out = m;
    return PCH_OK;
}

int pch_mesh_destroy(pch_mesh *m) {
    if (!m) return PCH_OK;
    cudaSetDevice(m->device);
    free_ws(m);
    cudaFree(m->face);
    cudaFree(m->fan);
    cudaFree(m->fanhdr);
    cudaFree(m->anchor_wlo);
    cudaFree(m->apex_xy);
    cudaFree(m->dup_tab);
    cudaFree(m->d_src);
    cudaFree(m->fps_buf);
    cudaFree(m->d_out);
    cudaFree(m->trace);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    if (m->ev2) cudaEventDestroy(m->ev2);
    if (m->stream) cudaStreamDestroy(m->stream);
    delete m;
    return PCH_OK;
}

int64_t pch_mesh_device_bytes(const pch_mesh *m) { return m ? (int64_t)m->mesh_bytes : 0; }

int pch_probe(int32_t device, double *out, int32_t n_out) {
    if (!out || n_out < 2) return fail(PCH_ERR_CONFIG, "pch_probe needs out[2]");
    CK(cudaSetDevice(device));
    int nsm = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pch_live<true, true>, TPB, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double *buf = nullptr;
    Ctrl *c = nullptr;
    CK(cudaMalloc(&buf, 64));
    CK(cudaMalloc(&c, sizeof(Ctrl)));
    // FP64: 148 x 8 CTAs of 256 threads, 8 chains x iters FMAs each
    const int iters = 1 << 14, blocks = nsm * 8;
    k_probe_fp64<<<blocks, 256>>>(buf, 16, 1.0000001, 1e-9);  // warm-up
    CK(cudaEventRecord(e0));
    k_probe_fp64<<<blocks, 256>>>(buf, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    out[0] = 2.0 * 8.0 * iters * blocks * 256.0 / (ms * 1e-3) / 1e12;  // TFLOP/s
    // grid barrier at the live solver's grid
    const int grid = nsm * std::min(std::max(per_sm, 1), 4), n = 2048;
    int nn = n;
    void *args[] = {&c, &nn};
    CK(cudaMemset(c, 0, sizeof(Ctrl)));
    CK(cudaLaunchCooperativeKernel((const void *)k_probe_barrier, dim3(grid), dim3(TPB), args, 0, 0));
    CK(cudaMemset(c, 0, sizeof(Ctrl)));
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((const void *)k_probe_barrier, dim3(grid), dim3(TPB), args, 0, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    out[1] = ms * 1e3 / n;  // us per grid barrier
    cudaFree(buf);
    cudaFree(c);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return PCH_OK;
}

static int check_sources(const pch_mesh *m, const int64_t *sources, int64_t n) {
    if (n <= 0) return fail(PCH_ERR_SOURCE, "at least one source vertex is required");
    if (n > INT_MAX) return fail(PCH_ERR_SOURCE, "too many sources");
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
    CK(cudaMemcpyAsync(out_dist, field_ptr(m), sizeof(double) * m->nv, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return PCH_OK;
}

int pch_run_device(pch_mesh *m, const int64_t *d_sources, int64_t n_sources, const pch_config *cfg,
                   double *d_out, void *stream, pch_stats *stats) {
    if (!m || !cfg || !d_out || !d_sources) return fail(PCH_ERR_CONFIG, "null argument");
    if (n_sources <= 0) return fail(PCH_ERR_SOURCE, "at least one source vertex is required");
    if (n_sources > INT_MAX) return fail(PCH_ERR_SOURCE, "too many sources");
    CK(cudaSetDevice(m->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : m->stream;
    int rc = solve(m, d_sources, (int)n_sources, cfg, st, stats);
    if (rc) return rc;
    CK(cudaMemcpyAsync(d_out, field_ptr(m), sizeof(double) * m->nv, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return PCH_OK;
}

// batches of R fields solved together (one field per source), each
// batch's rows copied out (to the host or in place on the device) while
// the next batch solves on the same stream
static int run_rows(pch_mesh *m, const int64_t *d_sources, int64_t n_sources, const pch_config *cfg,
                    double *out_rows, bool out_on_device, cudaStream_t st, pch_stats *stats) {
    // the deterministic solver runs them one at a time
    int R = (cfg->flags & PCH_FLAG_DETERMINISTIC) ? 1 : DEFAULT_ROWS;
    // and no more than half the device memory can hold: per row the
    // distance / split / pick tables, per 4 rows one base window capacity
    // (4 window SoA buffers, event lists, fan candidates; ensure_ws)
    if (R > 1 && cfg->pool_capacity <= 0) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const double budget = 0.5 * (double)(free_b + m->ws_bytes);
            const double per_row = 24.0 * m->nv + 16.0 * m->nhe;
            const double base = (double)std::max<long long>(DEFAULT_POOL_MIN, m->nhe / 4);
            auto est = [&](int r) { return r * per_row + base * std::max(1, r / 4) * 472.0; };
            while (R > 1 && est(R) > budget) R /= 2;
        }
    }
    if (const char *rr = getenv("PCH_ROWS")) R = std::max(1, atoi(rr));  // development
    const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    for (int64_t r0 = 0; r0 < n_sources; r0 += R) {
        const int n = (int)std::min<int64_t>(R, n_sources - r0);
        int rc = solve(m, d_sources + r0, n, cfg, st, stats, n);
        if (rc) return rc;
        CK(cudaMemcpyAsync(out_rows + r0 * (int64_t)m->nv, field_ptr(m), sizeof(double) * m->nv * n, kind, st));
    }
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
    return run_rows(m, m->d_src, n_sources, cfg, out_rows, false, m->stream, stats);
}

int pch_run_rows_device(pch_mesh *m, const int64_t *d_sources, int64_t n_sources, const pch_config *cfg,
                        double *d_out_rows, void *stream, pch_stats *stats) {
    if (!m || !cfg || !d_out_rows || !d_sources) return fail(PCH_ERR_CONFIG, "null argument");
    if (n_sources <= 0) return fail(PCH_ERR_SOURCE, "at least one source vertex is required");
    if (n_sources > INT_MAX) return fail(PCH_ERR_SOURCE, "too many sources");
    CK(cudaSetDevice(m->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : m->stream;
    return run_rows(m, d_sources, n_sources, cfg, d_out_rows, true, st, stats);
}

int pch_fps(pch_mesh *m, int64_t first, int64_t n_samples, const pch_config *cfg, int64_t *out_samples,
            double *out_dist, pch_stats *stats) {
    if (!m || !cfg || !out_samples) return fail(PCH_ERR_CONFIG, "null argument");
    if (n_samples < 1) return fail(PCH_ERR_CONFIG, "n_samples must be >= 1");
    int rc = check_sources(m, &first, 1);
    if (rc) return rc;
    CK(cudaSetDevice(m->device));
    constexpr int NB = 4 * 148;  // argmax stage-1 blocks
    const size_t need = sizeof(int64_t) * n_samples + sizeof(double) * m->nv +
                        NB * (sizeof(double) + sizeof(long long));
    // samples, the running min-field and the argmax scratch in one buffer,
    // kept with the mesh (no allocation / implicit sync per call)
    if (need > m->fps_cap) {
        cudaFree(m->fps_buf);
        m->fps_buf = nullptr;
        m->fps_cap = 0;
        CK(cudaMalloc(&m->fps_buf, need));
        m->fps_cap = need;
    }
    char *buf = m->fps_buf;
    int64_t *d_samples = reinterpret_cast<int64_t *>(buf);
    double *d_min = reinterpret_cast<double *>(buf + sizeof(int64_t) * n_samples);
    double *d_bd = d_min + m->nv;
    long long *d_bv = reinterpret_cast<long long *>(d_bd + NB);
    cudaStream_t st = m->stream;
    auto done = [&](int code) {
        cudaStreamSynchronize(st);
        return code;
    };
    if (cudaMemcpyAsync(d_samples, &first, sizeof(int64_t), cudaMemcpyHostToDevice, st) != cudaSuccess)
        return done(fail(PCH_ERR_CUDA, "sample upload failed"));
    // greedy: sample s+1 is the vertex farthest from samples 0..s; each
    // solve starts from the min-field so far and only moves where the new
    // sample is closer (the argmax never leaves the device)
    for (int64_t s = 0; s < n_samples; ++s) {
        if ((rc = solve(m, d_samples + s, 1, cfg, st, stats, 1, s > 0 ? d_min : nullptr))) return done(rc);
        if (cudaMemcpyAsync(d_min, field_ptr(m), sizeof(double) * m->nv, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
            return done(fail(PCH_ERR_CUDA, "field copy failed"));
        if (s + 1 < n_samples) {
            k_fps_argmax1<<<NB, 256, 0, st>>>(d_min, m->nv, d_bd, d_bv);
            k_fps_argmax2<<<1, 32, 0, st>>>(d_bd, d_bv, NB, reinterpret_cast<int64_t *>(d_samples + s + 1));
            if (cudaGetLastError() != cudaSuccess) return done(fail(PCH_ERR_CUDA, "argmax launch failed"));
        }
    }
    if (cudaMemcpyAsync(out_samples, d_samples, sizeof(int64_t) * n_samples, cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        (out_dist &&
         cudaMemcpyAsync(out_dist, d_min, sizeof(double) * m->nv, cudaMemcpyDeviceToHost, st) != cudaSuccess))
        return done(fail(PCH_ERR_CUDA, "result download failed"));
    if (cudaStreamSynchronize(st) != cudaSuccess) return done(fail(PCH_ERR_CUDA, "fps sync failed"));
    return done(PCH_OK);
}

}  // extern "C"
