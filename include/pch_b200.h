/*
 * pch_b200.h -- C ABI of the B200-native Parallel Chen-Han geodesic solver.
 *
 * This is the drop-in boundary for the reference's engine entry point
 *   run_pch(mesh: SurfaceMesh, sources, config: EngineConfig)
 *       -> (distance_field, RunStats)
 * (reference pkg/src/pargeo/engine.py:433), with the mesh arrays of
 * SurfaceMesh (pkg/src/pargeo/mesh.py:44) crossing as plain pointers.
 * No torch types, no C++ types: every argument is a pointer + size.
 *
 * Entry points and the reference interface each one replaces:
 *   pch_half_edge_build  build_half_edge_mesh(positions, faces) (mesh.py:142)
 *   pch_mesh_create   build_half_edge_mesh result -> device-resident mesh
 *                     (mesh.py:142 output; the paper's §4.1 `he[]`,
 *                      `outgoing_he[]` plus precomputed unfoldings)
 *   pch_run           run_pch(mesh, sources, config) with host buffers
 *                     (engine.py:433)
 *   pch_run_device    the same with device-resident sources / output
 *   pch_run_rows      batched single-source fields, one row per source
 *   pch_run_rows_device  the same with device-resident sources / rows
 *                     (the CLI's multi-source use, cli.py:382 context;
 *                      paper Table 3 "multiple-source-all-destination")
 *   pch_fps           farthest-point sampling on seeded single-source solves
 *                     (north star's batched workloads; no reference entry)
 * Error behaviour mirrors the reference: an empty or out-of-range source
 * list returns PCH_ERR_SOURCE (reference raises ValueError "invalid source
 * index"); exceeding max_iterations returns PCH_ERR_GUARD (EngineGuard,
 * engine.py:475); bad config values return PCH_ERR_CONFIG (ValueError in
 * EngineConfig.__post_init__, engine.py:65).  pch_last_error() returns the
 * message of the last failure on the calling thread.
 */
#ifndef PCH_B200_H
#define PCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCH_ABI_VERSION 3

enum pch_status {
    PCH_OK = 0,
    PCH_ERR_CUDA = 1,     /* CUDA runtime failure (message in pch_last_error) */
    PCH_ERR_SOURCE = 2,   /* empty / out-of-range source list */
    PCH_ERR_CONFIG = 3,   /* k < 1, epsilon <= 0, ... */
    PCH_ERR_GUARD = 4,    /* iteration cap or wall-time guard tripped */
    PCH_ERR_MESH = 5,     /* malformed mesh arrays */
    PCH_ERR_NOMEM = 6     /* window pool cannot grow further */
};

/* EngineConfig (engine.py:44) fields that exist on this path. */
typedef struct pch_config {
    int64_t k;               /* selection size per iteration (>= 1) */
    int32_t selection_mode;  /* 0 exact, 1 approximate_strided (both map to
                                the device threshold selection) */
    int32_t fan_mode;        /* 0 clip, 1 full_edges */
    double epsilon_window;   /* tiny-window tolerance (default 1e-6) */
    int64_t max_iterations;  /* < 0: no cap (reference None); n >= 0: the
                                solve fails with PCH_ERR_GUARD once it runs
                                more than n iterations (engine.py:475) */
    int64_t pool_capacity;   /* initial window-pool capacity; 0 = auto */
    int32_t flags;           /* PCH_FLAG_* */
    int32_t chain;           /* propagations one thread may chain per
                                iteration: a child the next batch would
                                select is propagated at once by the same
                                thread (0 = library default: 3 on meshes
                                of >= 2^18 faces, 6 if they are
                                anisotropic, else 2; 1 = off;
                                one-barrier solver only) */
    double time_limit_s;     /* device wall-time guard in seconds, 0 = none
                                (no reference counterpart; PCH_ERR_GUARD) */
    double fan_margin;       /* saddle-fan interval widened by this angle
                                (radians, [0, 0.1)) on both sides; 0 = the
                                reference's clip (geom.py:239-256).  A small
                                margin (1e-5) closes the rounding slivers
                                between a fan and the straight windows
                                passing its saddle */
} pch_config;

#define PCH_FLAG_NO_RECHECK 1   /* disable the pop-time endpoint re-check */
#define PCH_FLAG_DETERMINISTIC 2  /* two-barrier solver whose filters read
                                     iteration-frozen tables: bitwise
                                     identical fields across runs (paper
                                     Algorithm 1 with its delayed updates);
                                     default is the one-barrier solver with
                                     live tables, equal to rounding */
#define PCH_FLAG_PHASE_TIMES 8  /* fill pch_stats.time_select/_propagate/
                                     _compact/_events_ms and prop_item_us
                                     (warp-cycle attribution, ~3 % slower) */
#define PCH_FLAG_DEDUPE 16  /* drop exact-duplicate fan windows as the
                                reference does (engine.py:201), counted in
                                pruned_duplicate; off by default: the
                                per-vertex fan pick leaves ~0.02 % twins
                                and the fingerprint table costs ~10 % */
#define PCH_FLAG_ABSOLUTE_TINY 4  /* the reference's absolute tiny-window
                                     drop (width <= epsilon_window,
                                     geom.py:133) everywhere; default: the
                                     threshold scales with the distance to
                                     the pseudo source within 40 mean edges
                                     (an angular width of eps/40 edges), so
                                     the thin fan of a nearly flat saddle is
                                     not dropped -- the reference's holes
                                     and detoured vertices behind such
                                     saddles */

/* RunStats (engine.py:76) plus device-side counters. */
typedef struct pch_stats {
    int64_t iterations;
    int64_t windows_propagated;
    int64_t total_windows_created;
    int64_t total_windows_pruned;
    int64_t pruned_ich;
    int64_t pruned_split;
    int64_t pruned_tiny;
    int64_t pruned_degenerate;
    int64_t pruned_duplicate;
    int64_t pruned_recheck;
    int64_t windows_stored;
    int64_t max_children_per_window;
    int64_t events_created;
    int64_t events_applied;
    int64_t peak_active_pool;
    int64_t fans_emitted;
    int64_t buffer_regrows;   /* window-pool growths (RunStats.buffer_regrows) */
    int64_t pool_restarts;    /* ... of which reran the solve from scratch (a
                                 hard overflow); the live solver grows at an
                                 iteration boundary and continues */
    int64_t grid_barriers;    /* grid-wide barriers the one-barrier solver ran
                                 (fewer than iterations: CTA-local iterations) */
    double time_total_ms;     /* device time of the solve (CUDA events) */
    double time_kernel_ms;    /* persistent-kernel time only */
    /* RunStats.time_select / _propagate / _compact / _events
     * (engine.py:470-473), with PCH_FLAG_PHASE_TIMES (else 0): the kernel
     * time split by warp-cycle attribution
     * (the phases are fused into one kernel; select = barrier, prefix
     * rebuild and step controller; events = saddle fans and, in the
     * deterministic solver, the table commit) */
    double time_select_ms;
    double time_propagate_ms;
    double time_compact_ms;
    double time_events_ms;
    /* (PCH_FLAG_PHASE_TIMES) mean duration of one batch work item of the one-barrier solver (a
     * warp's chain of up to `chain` propagations), microseconds: the
     * latency term of the solver's roofline */
    double prop_item_us;
} pch_stats;

typedef struct pch_mesh pch_mesh;

/* Half-edge construction on the host (reference mesh.py:142
 * build_half_edge_mesh): positions double[n_vertices * 3], faces
 * int64[n_faces * 3] (consistently oriented) in; the SurfaceMesh arrays
 * out -- origin / opposite (-1 on a boundary) / length / corner_angle
 * [3 n_faces], total_angle / vertex_class (0 spherical, 1 euclidean,
 * 2 saddle) / outgoing / on_boundary [n_vertices].  Lengths are
 * bit-identical to the reference's numpy arithmetic; with corner_cos_only
 * the corner_angle array receives the clipped law-of-cosines ratio and
 * total_angle / vertex_class are left to the caller (numpy's arccos and the
 * C library's differ in the last bit; the Python layer applies numpy's).
 * Returns PCH_ERR_MESH with the reference's MeshError message in
 * pch_half_edge_error() for bad indices, repeated vertices, zero-length
 * edges, degenerate triangles, non-manifold edges or vertices.  No GPU. */
int pch_half_edge_build(const double *positions, int64_t n_vertices,
                        const int64_t *faces, int64_t n_faces,
                        int64_t *origin, int64_t *opposite, double *length,
                        double *corner_angle, double *total_angle,
                        uint8_t *vertex_class, int64_t *outgoing,
                        uint8_t *on_boundary, int32_t corner_cos_only);
const char *pch_half_edge_error(void);

/* Library identity. */
int pch_abi_version(void);
const char *pch_last_error(void);
int pch_device_count(void);

/* Upload a half-edge mesh (arrays exactly as SurfaceMesh holds them:
 * origin/opposite/length/corner_angle are length 3*n_faces, vertex_class
 * and outgoing length n_vertices; opposite == -1 marks a boundary) to
 * `device` and build the device-side tables.  *out receives the handle. */
int pch_mesh_create(const int64_t *origin, const int64_t *opposite,
                    const double *length, const double *corner_angle,
                    const uint8_t *vertex_class, const int64_t *outgoing,
                    int64_t n_vertices, int64_t n_faces, int32_t device,
                    pch_mesh **out);
int pch_mesh_destroy(pch_mesh *mesh);
int64_t pch_mesh_device_bytes(const pch_mesh *mesh);

/* Exact geodesic distance field from the union of `sources` (host
 * int64[n_sources]) into host double[n_vertices] `out_dist`; +inf marks
 * unreachable vertices.  `stats` may be NULL. */
int pch_run(pch_mesh *mesh, const int64_t *sources, int64_t n_sources,
            const pch_config *config, double *out_dist, pch_stats *stats);

/* Same with device pointers on the mesh's device; `stream` is a
 * cudaStream_t (NULL = the library's own stream).  Returns after the
 * solve has completed on the stream. */
int pch_run_device(pch_mesh *mesh, const int64_t *d_sources,
                   int64_t n_sources, const pch_config *config,
                   double *d_out_dist, void *stream, pch_stats *stats);

/* One single-source field per entry of `sources`: row r of the host
 * double[n_sources * n_vertices] `out_rows` is the field of sources[r].
 * `stats` (may be NULL) accumulates over rows. */
int pch_run_rows(pch_mesh *mesh, const int64_t *sources, int64_t n_sources,
                 const pch_config *config, double *out_rows,
                 pch_stats *stats);

/* pch_run_rows with device-resident sources (int64[n_sources]) and output
 * (double[n_sources * n_vertices]) on the mesh's device; `stream` as in
 * pch_run_device.  The rows never cross PCIe (multi-GPU gathers read them
 * in place, paper_1305_1293_b200/shard.py).  An out-of-range device source
 * returns PCH_ERR_SOURCE. */
int pch_run_rows_device(pch_mesh *mesh, const int64_t *d_sources,
                        int64_t n_sources, const pch_config *config,
                        double *d_out_rows, void *stream, pch_stats *stats);

/* Roofline denominators measured on `device` (bench.py): out[0] = FP64
 * FMA throughput in TFLOP/s (all SMs, independent chains), out[1] = one
 * grid barrier of the live solver's cooperative grid in microseconds.
 * n_out >= 2. */
int pch_probe(int32_t device, double *out, int32_t n_out);

/* Greedy farthest-point sampling (north star: batched multi-source
 * workloads): sample 0 is `first`, sample s+1 the vertex with the largest
 * geodesic distance to samples 0..s (ties: lowest index; +inf first, i.e.
 * components not reached yet).  Each step is one solve seeded with the
 * min-field so far, so it only propagates where the new sample is closer;
 * the argmax stays on the device.  Writes int64 out_samples[n_samples]
 * and, if out_dist is not NULL, the final min-field double[n_vertices]
 * (= run_pch(mesh, out_samples) of the reference, engine.py:433).  No
 * reference counterpart; the reference-side composition it replaces is a
 * loop of run_pch calls with a host argmax. */
int pch_fps(pch_mesh *mesh, int64_t first, int64_t n_samples,
            const pch_config *config, int64_t *out_samples, double *out_dist,
            pch_stats *stats);

#ifdef __cplusplus
}
#endif

#endif /* PCH_B200_H */
