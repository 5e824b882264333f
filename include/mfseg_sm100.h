/*
 * mfseg_sm100.h — C ABI of the B200 (sm_100a) segmentation core.
 *
 * Drop-in boundary for the data-parallel hot path of the reference `mfseg`
 * package (arXiv 1903.12294).  Every entry point below replaces one Python
 * function of the reference; the citation after each declaration names it
 * (paths relative to /root/reference/pkg/src/mfseg/).
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, POD structs.  No torch types.
 *   - All array pointers are DEVICE pointers unless a name ends in `_host`.
 *     The caller owns every buffer, including the workspace sized by the
 *     matching *_workspace_size() query (any alignment; the library aligns its
 *     carvings itself).  The library never frees caller memory.
 *   - Inputs must be finite: NaN / inf values, coordinates or
 *     times are rejected with status 2, as are inputs whose per-cluster sums
 *     could exceed the exact 128-bit accumulators (max |x| * samples >= 2^62).
 *   - Every call is stream-ordered on the caller's `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Calls that return host
 *     values synchronise that stream.
 *   - Return value: 0 on success, non-zero on error; the message is available
 *     from mfseg_last_error() (thread-local).  No C++ exception crosses the ABI.
 *   - Layouts follow the reference: field values are timestep-major, x-fastest
 *     (flat = i + nx*(j + ny*k), model.py:112); point xyz is (N,3) row-major
 *     (model.py:86-89); labels are int32 (engine.py:374-375).
 *   - Arithmetic is IEEE fp64 with the reference's operation order and no FMA
 *     contraction, so labels are bit-identical to the reference's.
 */
#ifndef MFSEG_SM100_H
#define MFSEG_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFSEG_ABI_VERSION 2

/* Clustering geometry and weights: ClusterParams (model.py:198-228) plus the
 * extent minima and interval distances C = extent/k (model.py:275-280). */
typedef struct mfseg_params {
    int32_t k[4];          /* clusters per axis (x, y, z, t) */
    double mins[4];        /* DomainExtent minima (x, y, z, t) */
    double C[4];           /* interval distances, computed by the host exactly as the reference */
    double c_f, w_d, w_p, w_f;
    double eps_c;
    int32_t max_iterations;
    int32_t n_centers;     /* centres in the state; 0 = k1*k2*k3*k4 (always so in mfseg_run) */
} mfseg_params;

/* FieldSet (model.py:108-157).  values: [nt][nz][ny][nx] fp64 (already
 * normalized, ingest.py:321-335), times: [nt].  offset: global cell index of
 * the first local cell per axis (0 for a whole grid; a spatial slab of a larger
 * grid keeps the grid's origin and sets offset, so that cell centres are
 * origin + (offset + i + 0.5) * spacing with the reference's roundings). */
typedef struct mfseg_field {
    int32_t nx, ny, nz, nt;
    double origin[3];
    double spacing[3];
    const double *times;
    const double *values;
    int32_t offset[3];
} mfseg_field;

/* PointSet (model.py:78-105): xyz [n][3], t [n], value [n] (normalized). */
typedef struct mfseg_points {
    int64_t n;
    const double *xyz;
    const double *t;
    const double *value;
} mfseg_points;

/* CenterState (engine.py:48-70), structure of arrays of length K. */
typedef struct mfseg_centers {
    double *loc;           /* [4][K]: x plane, y plane, z plane, t plane */
    double *pval;          /* [K], NaN when !has_p */
    double *fval;          /* [K], NaN when !has_f */
    uint8_t *has_p, *has_f, *dormant;   /* [K] */
    int64_t *n_points, *n_fields;        /* [K] */
} mfseg_centers;

/* Exact per-cluster sums (accumulate, engine.py:244-263) in 128-bit fixed
 * point (2^-64 units): per cluster 16 int64 words
 *   [0..7]  x, y, z, t   (lo, hi) pairs   — points and fields together
 *   [8..9]  point-value sum (lo, hi)
 *   [10..11] field-value sum (lo, hi)
 *   [12] n_points  [13] n_fields  [14..15] reserved (0)
 * Integer addition is associative, so the sums are independent of thread
 * scheduling and of the number of GPUs the samples are sharded over. */
#define MFSEG_ACC_WORDS 16

/* Per-iteration progress sink: progress(it, max_delta) (engine.py:368-369). */
typedef void (*mfseg_progress_fn)(void *user, int32_t iteration, double max_delta);

/* Cross-shard reduction hook for multi-GPU runs: called once per pass with a
 * device buffer of `n_words` int64 limbs (3 limbs of <=42 bits per 128-bit
 * word) that must be SUM-all-reduced in place across ranks on `stream`
 * before it returns.  NULL for single-GPU runs. */
typedef int (*mfseg_reduce_fn)(void *user, int64_t *limbs, int64_t n_words, void *stream);

const char *mfseg_last_error(void);
int mfseg_abi_version(void);

/* Instrumentation (bench.py): total kernel launches issued by this library so
 * far; optional per-phase device timing of mfseg_run with CUDA events on the
 * caller's stream (phases: 0 CenterGrid rebuild, 1 field assign, 2 point
 * assign, 3 stranded fallback, 4 exchange + update).  mfseg_timing_read fills
 * ms_out[0..n) with accumulated milliseconds and returns the pass count. */
long long mfseg_launch_count(void);

void mfseg_timing_enable(int32_t on);
int32_t mfseg_timing_read(double *ms_out, int32_t n);

/* Diagnostics / test knobs for the calling thread (defaults 0 / -1 are the
 * product behaviour; no environment variable is read by the library):
 * flags: bit 0 no tile culling, bit 1 exact fp64 for every surviving
 * candidate, bit 3 per-pass statistics on stderr (the kernels' path counters
 * only in a library built with -DMFSEG_DEVICE_STATS=1), bit 4 no reuse of unchanged
 * blocks / chunks across passes, bit 5 exact reuse only (no margin reuse);
 * multi_cap >= 0 caps the multi-candidate brick queue (the overflow takes the
 * exact per-sample path).  Results are identical for every setting. */
#define MFSEG_DEBUG_NO_CULL 1
#define MFSEG_DEBUG_EXACT 2
#define MFSEG_DEBUG_STATS 8
#define MFSEG_DEBUG_KERNEL_BITS 11
#define MFSEG_DEBUG_NO_REUSE 16
#define MFSEG_DEBUG_NO_MARGIN_REUSE 32
#define MFSEG_DEBUG_NO_SEEDS_FAST 64   /* initial pass: no interior-block shortcut */
#define MFSEG_DEBUG_NO_ZT_SWAP 128     /* thin fields: blocks along z, not time */
#define MFSEG_DEBUG_NO_BLOCK_CACHE 256 /* field blocks: no cached sums of fully reused blocks */
#define MFSEG_DEBUG_DEFERRED_BATCH 512 /* crowded tiles: one sample per lane at any list length */
int mfseg_set_debug_options(int32_t flags, int64_t multi_cap);

/* ---------------------------------------------------------------- full run
 * engine.run (engine.py:323-381): seed -> initial pass -> iterate
 * (CenterGrid, assign_iteration, accumulate, update_centers, has_converged)
 * until converged or max_iterations.  Outputs: labels of the last pass,
 * final centre state, iterations_used and converged flag (host ints). */
size_t mfseg_run_workspace_size(const mfseg_params *p, const mfseg_field *f,
                                const mfseg_points *pts);
int mfseg_run(const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts,
              int32_t *point_labels, int32_t *field_labels, mfseg_centers out,
              int32_t *iterations_used_host, int32_t *converged_host,
              mfseg_progress_fn progress, void *progress_user,
              mfseg_reduce_fn reduce, void *reduce_user,
              void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- one pass
 * assign_iteration (engine.py:208-241) for the given centres, with the fused
 * exact accumulation (engine.py:244-263) into `acc` [K][MFSEG_ACC_WORDS]
 * (zeroed by the call).  Uses the params' weights as given (the caller
 * passes w_p = w_f = 0, w_d = 1 for the initial pass, engine.py:348-349).
 * Labels are int32; the reference's int64 is a host-side widening. */
size_t mfseg_assign_workspace_size(const mfseg_params *p, const mfseg_field *f,
                                   const mfseg_points *pts);
int mfseg_assign(const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts,
                 mfseg_centers centers, int32_t *point_labels, int32_t *field_labels,
                 int64_t *acc, void *workspace, size_t workspace_bytes, void *stream);

/* accumulate (engine.py:244-263) for caller-given labels (int32, values in
 * [0, K)) into acc [K][MFSEG_ACC_WORDS] (zeroed by the call). */
int mfseg_accumulate(int32_t K, const mfseg_field *f, const mfseg_points *pts,
                     const int32_t *point_labels, const int32_t *field_labels,
                     int64_t *acc, void *stream);

/* accumulate's fp64 view: sums [K][4], psum [K], fsum [K], n_p [K], n_f [K]
 * (each 128-bit sum rounded once to the nearest double). */
int mfseg_acc_to_double(int32_t K, const int64_t *acc, double *sums, double *psum,
                        double *fsum, int64_t *n_p, int64_t *n_f, void *stream);

/* update_centers (engine.py:266-286) + has_converged / max_center_delta
 * (engine.py:289-320): old -> new_state.  `conv_host` gets
 * {converged (0/1)} and `delta_host` the progress delta (synchronises). */
int mfseg_update_centers(int32_t K, const int64_t *acc, mfseg_centers old_state,
                         mfseg_centers new_state, double eps_c, int32_t *conv_host,
                         double *delta_host, void *stream);

/* update_centers from the reference's fp64 sums (engine.py:266-286):
 * sums [K][4], psum/fsum [K], n_p/n_f [K] -> new_state (old_state supplies
 * the frozen values of empty clusters). */
int mfseg_update_centers_f64(int32_t K, const double *sums, const double *psum,
                             const double *fsum, const int64_t *n_p, const int64_t *n_f,
                             mfseg_centers old_state, mfseg_centers new_state, void *stream);

/* has_converged + max_center_delta of two states (engine.py:289-320). */
int mfseg_compare_centers(int32_t K, mfseg_centers old_state, mfseg_centers new_state,
                          double eps_c, int32_t *conv_host, double *delta_host, void *stream);

/* ---------------------------------------------------------------- ingest
 * normalize_variables / _minmax (ingest.py:312-335): in-place (v-lo)/(hi-lo)
 * on n values, or zeros when hi == lo.  lo/hi returned to the host. */
int mfseg_minmax_normalize(double *values, int64_t n, int32_t apply, double *lo_host,
                           double *hi_host, void *stream);

/* The same map with a caller-given (global) range, for sharded inputs whose
 * min/max were all-reduced across ranks. */
int mfseg_normalize_range(double *values, int64_t n, double lo, double hi, void *stream);

/* build_link_index (ingest.py:261-280): bucket points by (cell, interval).
 * Outputs (device): keys [n] int64 (flat key sorted ascending; flat =
 * ((k*ny + j)*nx + i)*n_int + m), members [n] int32 (point indices, stable
 * within a bucket), n_buckets_host.  Returns 2 if a point is outside the grid. */
/* build_features' trajectory split (postproc.py:152-160, 176-191): order =
 * point indices sorted by (traj_id, t) (np.lexsort, stable); runs of that order
 * broken at a new trajectory, a label change or a time gap > stride * (1+1e-9)
 * with stride = min positive difference of the unique point times (+inf when
 * there are fewer than two).  run_start[0..n_runs] (device) delimits the runs;
 * runs of >= 2 points are polylines, single points isolated points.
 * label: one int32 per point (feature slot).  Synchronises the stream. */
size_t mfseg_traj_split_workspace_size(int64_t n);
int mfseg_traj_split(int64_t n, const int64_t *traj_id, const double *t, const int32_t *label,
                     int32_t *order, int32_t *run_start, int64_t *n_runs_host, double *stride_host,
                     void *workspace, size_t workspace_bytes, void *stream);

/* The same split with a caller-given stride (multi-GPU: the ranks' common
 * stride over all point times; the points of each trajectory are all local). */
int mfseg_traj_split_stride(int64_t n, const int64_t *traj_id, const double *t,
                            const int32_t *label, double stride, int32_t *order,
                            int32_t *run_start, int64_t *n_runs_host, void *workspace,
                            size_t workspace_bytes, void *stream);

size_t mfseg_link_index_workspace_size(int64_t n);
int mfseg_link_index(const mfseg_field *f, const mfseg_points *pts, int64_t *keys,
                     int32_t *members, int64_t *n_buckets_host, void *workspace,
                     size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- post
 * merge_clusters (postproc.py:59-92) over the live centre table (n rows in
 * ascending id order).  Inputs: ids [n] int32, loc [4][n], p_c/f_c [n]
 * (NaN = absent), n_points/n_fields [n].  Outputs: rep [n] int32 (the merge
 * map, = smallest id of the eligibility component), merged table rows
 * (ascending representative id): m_ids, m_loc [4][n], m_p/m_f, m_np, m_nf
 * and n_merged_host.  neumaier: 1 = the merged p_c / f_c sums follow CPython
 * >= 3.12's compensated sum() of floats, 0 = the plain left-to-right sum of
 * earlier interpreters (postproc.py:85-88 uses the builtin sum). */
size_t mfseg_merge_workspace_size(int32_t n);
int mfseg_merge(int32_t n, const int32_t *ids, const double *loc, const double *p_c,
                const double *f_c, const int64_t *n_points, const int64_t *n_fields,
                double eps_m, int32_t neumaier, int32_t *rep, int32_t *m_ids, double *m_loc, double *m_p,
                double *m_f, int64_t *m_np, int64_t *m_nf, int32_t *n_merged_host,
                void *workspace, size_t workspace_bytes, void *stream);

/* merge_map[label] gather (postproc.py:155,164): out[i] = lut[labels[i]]. */
int mfseg_relabel(const int32_t *labels, int64_t n, const int32_t *lut, int32_t lut_len,
                  int32_t *out, void *stream);

/* Per-timestep voxel bucketing (postproc.py:162-168): for timestep m and
 * feature f, the ascending flat cell indices with feature label f.
 * Output CSR keyed by (m, f_slot) with f_slot = dense feature slot from
 * `slot_of` [lut_len] (feature id -> slot, -1 unused): seg_start [(nt*nf)+1]
 * int64, cells [nt*ncell] int32. */
size_t mfseg_voxel_csr_workspace_size(int64_t n_field_samples, int32_t nt, int32_t n_slots);
int mfseg_voxel_csr(const int32_t *feature_labels, int32_t nt, int64_t ncell,
                    const int32_t *slot_of, int32_t lut_len, int32_t n_slots,
                    int64_t *seg_start, int32_t *cells, void *workspace,
                    size_t workspace_bytes, void *stream);

/* feature_stats (postproc.py:194-227) for n_slots features from per-sample
 * slots (-1 = none): stats [n_slots][MFSEG_STAT_WORDS] doubles:
 *   bbox_min[4], bbox_max[4], p_mean, p_std, f_mean, f_std, n_points, n_fields */
#define MFSEG_STAT_WORDS 14
size_t mfseg_feature_stats_workspace_size(int32_t n_slots);
int mfseg_feature_stats(int32_t n_slots, const mfseg_field *f, const int32_t *field_slot,
                        const mfseg_points *pts, const int32_t *point_slot, double *stats,
                        void *workspace, size_t workspace_bytes, void *stream);

/* feature_stats in steps, for samples sharded over ranks (the caller reduces
 * `partial` across ranks between the steps).  partial [n_slots][18] uint64:
 *   [0..1] point-value sum, [2..3] field-value sum (128-bit fixed point, lo/hi),
 *   [4..5] point, [6..7] field sums of squared deviations from the mean (same),
 *   [8] n_points, [9] n_fields, [10..13] bbox minima, [14..17] bbox maxima as
 *   order-preserving keys of the doubles (unsigned min / max).
 * pass 0 initialises `partial` and adds sums, counts and bbox; pass 1 adds the
 * squared deviations from `mean` [n_slots][2] (point, field), which
 * mfseg_feature_stats_means derives from the (reduced) pass-0 words;
 * mfseg_feature_stats_final writes the MFSEG_STAT_WORDS rows.  Integer sums make
 * the result independent of the sharding.  Synchronises (pass). */
#define MFSEG_STAT_PARTIAL_WORDS 18
int mfseg_feature_stats_pass(int32_t n_slots, const mfseg_field *f, const int32_t *field_slot,
                             const mfseg_points *pts, const int32_t *point_slot, int32_t pass,
                             const double *mean, uint64_t *partial, void *stream);
int mfseg_feature_stats_means(int32_t n_slots, const uint64_t *partial, double *mean, void *stream);
int mfseg_feature_stats_final(int32_t n_slots, const uint64_t *partial, const double *mean,
                              double *stats, void *stream);

/* ---------------------------------------------------------------- multi-GPU
 * acc [n_words] 128-bit (lo,hi) pairs <-> 3 limbs of 42 bits, for SUM
 * all-reduce across ranks (exact for up to 2^20 ranks). */
int mfseg_acc_to_limbs(const int64_t *acc, int64_t n_pairs, int64_t *limbs, void *stream);
int mfseg_limbs_to_acc(const int64_t *limbs, int64_t n_pairs, int64_t *acc, void *stream);

/* ---------------------------------------------------------------- synthetic data
 * Counter-based synthetic generator (bench inputs; reproducible bit-for-bit
 * by the numpy mirror in oracle/synth.py): drifting ellipsoid blobs over a
 * background plus hashed noise.  See DESIGN.md "Synthetic inputs". */
typedef struct mfseg_synth {
    int32_t nx, ny, nz, nt;
    int64_t n_traj;        /* trajectories, one sample per timestep each */
    uint64_t seed;
    double noise;          /* noise amplitude */
    int32_t n_blobs;
    int32_t dyadic;        /* 1: quantize values to 2^-20 and xyz to 2^-16 */
} mfseg_synth;
int mfseg_synth_field(const mfseg_synth *s, double *values, void *stream);
int mfseg_synth_points(const mfseg_synth *s, int64_t *traj_id, double *t, double *xyz,
                       double *value, void *stream);
/* Windows of the same datasets (multi-GPU slabs generate only their share):
 * timesteps [m0, m1) x z-planes [z0, z1) of the field ([m][z][y][x], x fastest),
 * trajectories [p0, p1) x timesteps [m0, m1) of the points (trajectory-major). */
int mfseg_synth_field_window(const mfseg_synth *s, int32_t m0, int32_t m1, int32_t z0, int32_t z1,
                             double *values, void *stream);
int mfseg_synth_points_window(const mfseg_synth *s, int64_t p0, int64_t p1, int32_t m0, int32_t m1,
                              int64_t *traj_id, double *t, double *xyz, double *value, void *stream);
/* Taxi-like 2D+t points (configs[3]): trajectories [p0, p1), each `steps`
 * consecutive samples from a uniform random start step; a fraction `skew` of
 * them drive along road rows / columns (a fraction `road_frac` of all rows /
 * columns), z = 0.5 * nz.  Output (p1 - p0) * steps samples, trajectory-major. */
int mfseg_synth_taxi_points(const mfseg_synth *s, int32_t steps, double skew, double road_frac,
                            int64_t p0, int64_t p1, int64_t *traj_id, double *t, double *xyz,
                            double *value, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MFSEG_SM100_H */
