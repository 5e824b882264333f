// Kernel argument blocks and launchers shared by the runtime (run.cu) and the
// assignment kernels (assign.cu).
#pragma once

#include "common.cuh"

// Device-side path counters of the assignment kernels (MFSEG_DEBUG_STATS): compiled
// only into a diagnostics build (-DMFSEG_DEVICE_STATS=1, tools/variant_time.sh); the
// product build drops the checks from the hot loops.
#ifndef MFSEG_DEVICE_STATS
#define MFSEG_DEVICE_STATS 0
#endif
#define DEVICE_STATS(args) (MFSEG_DEVICE_STATS && ((args).debug & 8))

namespace mfseg {

// A field brick left with several candidates after culling and dominance:
// resolved per sample by k_field_screen (one warp per item).
#ifndef MFSEG_MULTI_MAX
#define MFSEG_MULTI_MAX 16
#endif
constexpr int MULTI_MAX = MFSEG_MULTI_MAX;
struct MultiItem {
    int x0, y0, z0, t0;       // brick origin (global sample indices)
    int meta;                 // nk | live extent x << 8 | y << 12 | z << 16 | t << 20
    int pad[3];
    int id[MULTI_MAX];        // kept candidates (global centre ids)
};

struct FieldArgs {
    int nx, ny, nz, nt;
    double ox, oy, oz, sx, sy, sz;
    int x0, y0, z0;       // global cell index of the field's first cell (spatial slabs)
    int seeds_fast;       // initial pass: blocks whose axis tiles are all interior (AxisTile.pad)
                          // take their own bin's seed (see run.cu seeds_fast_ok)
    // Thin fields (nz = 1, k_z = 1): the kernels' z axis runs over the timesteps and
    // their t axis over the single z plane, so blocks and bricks fill along time
    // (the layouts coincide: plane stride = volume stride).  zt then holds time
    // tiles and tt the z tile, nz / nt / kz / kt and the centres' z / t pointers are
    // passed swapped; coordinates, the c_f scale, the validity boxes, the exact
    // metric and the accumulator words follow the real axes (run.cu plan_pass).
    int swap_zt;
    const double *times;
    const double *values;
    const AxisTile *xt, *yt, *zt;
    int ntx, nty, ntz;
    const int *tbin;
    const AxisTile *tt;   // time tiles: runs of <= 4 timesteps inside one t-bin
    int ntt;
    int kx, ky, kz, kt;
    double cf, wd, wv;
    CentersView c;
    const double *cval;
    const uint8_t *chas;
    Grid g;
    int *labels;
    unsigned long long *acc;
    long long *stranded;
    unsigned long long *n_stranded;
    long long stranded_cap;
    long long *deferred;              // samples of crowded tiles, resolved by k_deferred
    unsigned long long *n_deferred;
    long long deferred_cap;
    int *overflow;
    unsigned long long *absmax;   // k_brick_pre: [5] max |value| (double bits), [6] non-finite flag
    int accumulate;
    int debug;   // bit0: no warp culling, bit1: exact evaluation of every survivor, bit3: stats
    unsigned long long *stats;   // debug bit3: [0] bricks, [1] kept candidates, [2] exact samples
    const float2 *brange;        // per brick (block * 64 + brick): range of fl32(value)
    const ulonglong2 *bsum;      // per brick: fixed-order value sum as 128-bit fixed point (k_brick_pre)
    float2 *brange_out;
    ulonglong2 *bsum_out;
    MultiItem *multi;            // queue of bricks for k_field_screen (capacity: all bricks)
    unsigned long long *n_multi;
    long long multi_cap;
    // reuse of the previous pass: a block whose 3^4 neighbour bins hold no
    // centre changed by the last update (bin_stable) keeps the labels of its
    // single-candidate bricks (bslot: slot, 255 = none)
    const unsigned char *bin_stable;
    unsigned char *bslot;
    int reuse;
    // margin reuse: bins whose neighbourhood's candidate lists, validity boxes and
    // has-flags did not change (bin_sstable); per centre an upper bound of the
    // change of its metric anywhere (cdelta = w_d |delta c| + w_v |delta cv|);
    // per brick a proven lower bound of D_s - D_s* over its samples (bmargin)
    const unsigned char *bin_sstable;
    const float *cdelta;
    float *bmargin;
    // a block whose every brick keeps its label contributes the same sums as in
    // the pass that labelled it: per brick the centre id of its label (bcid) and
    // per block its per-cluster sums (bcache, n = -1: none) let such a block add
    // them without its setup (k_field_assign5)
    int *bcid;
    struct BlockCache *bcache;
    const float *bin_dmax;       // per sample bin: the largest cdelta among its candidates
};

#ifndef MFSEG_BC_MAX
#define MFSEG_BC_MAX 6
#endif
constexpr int BC_MAX = MFSEG_BC_MAX;   // clusters cached per field block
struct BlockCache {                   // one field block's per-cluster sums, as added to acc
    int n;                            // entries (-1: none)
    int id[BC_MAX];
    unsigned long long w[BC_MAX][10]; // x, y, z, t, value: 128-bit (lo, hi), real axes
    unsigned long long cnt[BC_MAX];
};

struct WBox {                 // one 64-point warp tile of a point chunk (k_point_assign4)
    float4 lo, hi;            // chunk-relative fp32 box (t scaled by c_f)
    float2 v;                 // range of fl32(value)
    float2 pad;
    double s[5];              // fixed-order warp sums of x, y, z, t, value (whole tile)
    double pad2;
};

struct PointArgs {
    long long n;
    const double *x, *y, *z, *t, *v;   // bin-sorted SoA
    const int4 *tiles;                 // (bin, start, len, -)
    const int *n_tiles;
    const double *tile_box;            // [tile][8]: exact lo[4], hi[4] (k_point_assign4)
    const WBox *wbox;                  // [tile][POINT_CHUNK / 64] warp-tile boxes
    double Cx, Cy, Cz, Ct;
    double cf, wd, wv;
    int seeds_fast;                    // initial pass: interior chunks take their bin's seed
    double mn[4];                      // extent minima and k (the chunks' interior test)
    int kk[4];
    CentersView c;
    const double *cval;
    const uint8_t *chas;
    Grid g;
    int *labels;                       // bin-sorted order
    int *labels_out;                   // final pass: also labels_out[perm[p]] (record order)
    const unsigned *perm;              // bin-sorted position -> record index
    unsigned long long *acc;
    long long *stranded;
    unsigned long long *n_stranded;
    long long stranded_cap;
    long long *deferred;
    unsigned long long *n_deferred;
    long long deferred_cap;
    int *overflow;
    int accumulate;
    int debug;
    unsigned long long *stats;   // debug bit3: [0] warp tiles, [1] kept candidates, [2] exact points
    // reuse (as FieldArgs): per warp tile the slot of its single label last pass (255: none)
    const unsigned char *bin_stable;
    unsigned char *tslot;
    int reuse;
    // a chunk whose bin is stable keeps every label: its per-cluster sums are those
    // cached when it last ran (pcache, n = -1: none)
    struct PointCache *pcache;
};

#ifndef MFSEG_PC_MAX
#define MFSEG_PC_MAX 12
#endif
constexpr int PC_MAX = MFSEG_PC_MAX;  // clusters cached per point chunk
struct PointCache {                   // one point chunk's per-cluster sums, as added to acc
    int n;                            // entries (-1: none)
    int id[PC_MAX];
    unsigned long long w[PC_MAX][10]; // x, y, z, t, value: 128-bit (lo, hi)
    unsigned long long cnt[PC_MAX];
};

// Stranded-sample fallback (engine.py:195-205): field samples (kind 1) are
// addressed by flat index, points (kind 0) by bin-sorted position.
struct FallbackArgs {
    int K;
    CentersView c;
    const double *cval;
    const uint8_t *chas;
    double C[4];
    double cf, wd, wv;
    // sample source: field (kind 1) or bin-sorted points (kind 0)
    int kind;
    int nx, ny, nz, nt;
    double ox, oy, oz, sx, sy, sz;
    const double *times, *values;
    int x0, y0, z0;                    // global cell index of the field's first cell (slabs)
    const double *px, *py, *pz, *pt, *pv;
    // CenterGrid bins (k_fallback enumerates the bins a widened box can reach)
    const int *bin_start, *bin_ids;
    double mins[4];
    int k[4];
    long long n_samples;
    int *labels;
    int *labels_out;                   // points, final pass: also labels_out[perm[idx]]
    const unsigned *perm;
    const long long *stranded;
    const unsigned long long *n_stranded;
    long long cap;
    unsigned long long *acc;
    int *overflow;
    int accumulate;
};

// points per chunk of k_point_assign4 (8 warps x 4 warp tiles of 64 points)
#ifndef MFSEG_POINT_CHUNK
#define MFSEG_POINT_CHUNK 2048
#endif
constexpr int POINT_CHUNK = MFSEG_POINT_CHUNK;

// grid.cu
size_t grid_workspace_bytes(int K, int NB);
Grid grid_carve(Carver &cv, int K, int NB, int **count_tmp, void **scan_tmp);
int grid_build(Grid &g, const double *x, const double *y, const double *z, const double *t,
               const mfseg_params *p, const mfseg_field *f, int *count_tmp, void *scan_tmp,
               cudaStream_t st);
// assign.cu
struct DebugOptions {   // mfseg_set_debug_options (thread-local; defaults = product behaviour)
    int flags = 0;
    long long multi_cap = -1;
};
const DebugOptions &debug_options();
int field_tile_dims(int *tx, int *ty, int *tz);
int launch_brick_pre(const FieldArgs &a, cudaStream_t st);
int launch_field_screen(const FieldArgs &a, cudaStream_t st);
int point_tile_size();
int launch_tile_box(unsigned long long *absmax, const int4 *tiles, const int *n_tiles, long long max_tiles, double *x, double *y,
                    double *z, double *t, double *v, double cf, double *box, WBox *wbox,
                    const unsigned *perm, const double *gxyz, const double *gt, const double *gv,
                    cudaStream_t st);
int launch_field_assign(const FieldArgs &a, long long ntiles, cudaStream_t st);
int launch_point_assign(const PointArgs &a, long long max_tiles, cudaStream_t st);
int launch_fallback(const FallbackArgs &a, cudaStream_t st);
int launch_deferred(const FallbackArgs &a, const Grid &g, const int *tbin, const int4 &k,
                    const double *mins, const long long *list, const unsigned long long *count,
                    long long cap, cudaStream_t st);
int launch_accumulate_field(long long n, const mfseg_field *f, const int *labels,
                            unsigned long long *acc, int *overflow, cudaStream_t st);
int launch_accumulate_points(const mfseg_points *p, const int *labels, unsigned long long *acc,
                             int *overflow, cudaStream_t st);
// update.cu
size_t update_flags_bytes();
int launch_update(int K, const unsigned long long *acc, mfseg_centers o, mfseg_centers n,
                  double eps_c, void *flags_dev, cudaStream_t st);
void decode_flags(const void *flags_host, int *converged, double *delta);
int launch_acc_to_double(int K, const unsigned long long *acc, double *sums, double *psum,
                         double *fsum, long long *n_p, long long *n_f, cudaStream_t st);
int launch_to_limbs(long long npairs, const unsigned long long *acc, long long *limbs,
                    cudaStream_t st);
int launch_from_limbs(long long npairs, const long long *limbs, unsigned long long *acc,
                      cudaStream_t st);

}  // namespace mfseg
