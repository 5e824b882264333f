// Host-side runtime of the segmentation core: workspace plan, point binning,
// field tiling, the pass loop of engine.run (engine.py:323-381) and the C ABI.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"

namespace mfseg {

// ------------------------------------------------------------------ instrumentation
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// per-phase device times of mfseg_run (CUDA events on the caller's stream),
// read by bench.py for the roofline of the dominant kernel
struct PhaseTimer {
    bool on = false;
    double ms[8] = {0};      // 0 grid, 1 field assign, 2 point assign, 3 fallback, 4 update
    long long launches[8] = {0};
    int passes = 0;
};
static PhaseTimer g_timer;
static cudaEvent_t g_ev[6];
static bool g_ev_made = false;

// NVTX ranges per phase of a pass (host-side launch regions; free when no tool
// is attached): grid, field assign, point assign, fallback, exchange + update
static void nvtx_phase(int i) {
    static const char *names[5] = {"mfseg grid", "mfseg field assign", "mfseg point assign",
                                   "mfseg fallback", "mfseg exchange+update"};
    if (i > 0) nvtxRangePop();
    if (i < 5) nvtxRangePushA(names[i]);
}

static void mark(int i, cudaStream_t st) {
    nvtx_phase(i);
    if (!g_timer.on) return;
    if (!g_ev_made) {
        for (auto &e : g_ev) cudaEventCreate(&e);
        g_ev_made = true;
    }
    cudaEventRecord(g_ev[i], st);
}

// after the stream has been synchronised: fold the pass's event intervals in
static void harvest() {
    if (!g_timer.on || !g_ev_made) return;
    float t;
    for (int i = 0; i < 5; ++i)
        if (cudaEventElapsedTime(&t, g_ev[i], g_ev[i + 1]) == cudaSuccess) g_timer.ms[i] += t;
    g_timer.passes++;
}

// ------------------------------------------------------------------ debug options
// Diagnostics and test knobs (mfseg_set_debug_options), per calling thread;
// the defaults are the product behaviour.
static thread_local DebugOptions g_dbg;
const DebugOptions &debug_options() { return g_dbg; }

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
int tiny_scratch(void **dev, void **host) {
    struct Slot {
        void *d = nullptr, *h = nullptr;
    };
    static thread_local Slot slots[64];
    int id = 0;
    MFSEG_CUDA(cudaGetDevice(&id));
    if (id < 0 || id >= 64) {
        set_error("device ordinal out of range");
        return 1;
    }
    Slot &sl = slots[id];
    if (!sl.d) {
        MFSEG_CUDA(cudaMalloc(&sl.d, 256));
        MFSEG_CUDA(cudaMallocHost(&sl.h, 256));
    }
    *dev = sl.d;
    *host = sl.h;
    return 0;
}

void set_error(const std::string &msg) { g_err = msg; }
int fail(const char *where, cudaError_t e) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return 1;
}

}  // namespace mfseg

namespace mfseg {
namespace {

// ------------------------------------------------------------------ small kernels
__global__ void k_seed(int K, double4 mins, double4 C, int4 k, mfseg_centers s) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    int ix = c % k.x, r = c / k.x;
    int iy = r % k.y;
    r /= k.y;
    int iz = r % k.z, it = r / k.z;
    // mins[d] + (j + 0.5) * C[d]   (engine.py:38)
    s.loc[c] = DADD(mins.x, DMUL((double)ix + 0.5, C.x));
    s.loc[K + c] = DADD(mins.y, DMUL((double)iy + 0.5, C.y));
    s.loc[2 * K + c] = DADD(mins.z, DMUL((double)iz + 0.5, C.z));
    s.loc[3 * K + c] = DADD(mins.w, DMUL((double)it + 0.5, C.w));
    double nan = __longlong_as_double(0x7ff8000000000000ll);
    s.pval[c] = nan;
    s.fval[c] = nan;
    s.has_p[c] = s.has_f[c] = s.dormant[c] = 0;
    s.n_points[c] = s.n_fields[c] = 0;
}

__global__ void k_tbins(int nt, const double *times, double mn, double C, int k, int *tbin) {
    int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < nt) tbin[m] = bin_coord(times[m], mn, C, k);
}

// Sort key of a point: (sample bin, field-timestep interval, sub-cell), the
// sub-cell being the top sub_bits of the Morton interleave of 8 subdivisions
// per axis inside the bin (t, z, y, x bits from high to low), so consecutive
// points form compact 4D blocks; inside a sub-cell the stable sort keeps the
// caller's (trajectory) order, which keeps the chunk gather local.  One bit
// per axis (16 sub-cells) balances the two: finer sub-cells give tighter warp
// tiles but a scattered gather.  Tiles are cut per (bin, interval) group.
__global__ void k_point_keys(long long n, const double *xyz, const double *t, double4 mins,
                             double4 C, double4 inv, int4 k, const double *times, int nt, int sub_bits,
                             unsigned *keys, unsigned *vals) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c[4] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], t[i]};
    const double mn[4] = {mins.x, mins.y, mins.z, mins.w}, CC[4] = {C.x, C.y, C.z, C.w};
    const int kk[4] = {k.x, k.y, k.z, k.w};
    int b[4];
    unsigned sd[4];
    const double iC[4] = {inv.x, inv.y, inv.z, inv.w};
    for (int d = 0; d < 4; ++d) {
        // u = fl((c - mn) / C) as bin_coord computes it; the quotient only enters
        // through floor(u) and floor(8 u), so a reciprocal product (within a few
        // ulps of it) serves unless 8 u lies near an integer: then divide exactly
        const double dd = DSUB(c[d], mn[d]);
        double u = DMUL(dd, iC[d]);
        const double e = DMUL(u, 8.0), fe = floor(e);
        const double tol = 1e-13 * fabs(e) + 1e-13;
        if (!(fabs(e) < 1e15) || e - fe < tol || fe + 1.0 - e < tol) u = DDIV(dd, CC[d]);
        const double q = floor(u);   // bin_coord's clamps
        b[d] = !(q >= 0.0) ? 0 : (q >= (double)(kk[d] - 1) ? kk[d] - 1 : (int)q);
        const double f = floor(DMUL(u, 8.0)) - 8.0 * b[d];
        sd[d] = f < 0.0 ? 0u : (f > 7.0 ? 7u : (unsigned)f);
    }
    unsigned sub = 0;
    for (int bit = 2; bit >= 0; --bit)          // Morton: high bits first, x lowest
        for (int d = 3; d >= 0; --d) sub = (sub << 1) | ((sd[d] >> bit) & 1u);
    sub >>= (12 - sub_bits);
    int m = 0;
    if (nt > 1) {   // searchsorted(times, t, 'right') - 1, clipped to [0, nt-1]
        int a = 0, e = nt;
        while (a < e) {
            const int mid = (a + e) >> 1;
            if (times[mid] <= c[3]) a = mid + 1; else e = mid;
        }
        m = a - 1 < 0 ? 0 : a - 1;
    }
    const unsigned bin = (unsigned)(((b[3] * k.z + b[2]) * k.y + b[1]) * k.x + b[0]);
    keys[i] = (((unsigned)((unsigned long long)bin * nt + m)) << sub_bits) | sub;
    vals[i] = (unsigned)i;
}

// Group starts of the sorted keys by boundary detection (no atomics: sorted keys
// would serialise a histogram on the same counters).  Thread i in [0, n] writes
// first[q] = i for every group q in (group(i-1), group(i)]; group(n) = ng.
__global__ void k_bin_first(long long n, const unsigned *skeys, int shift, int ng, int *first) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i > n) return;
    int g = i < n ? (int)(skeys[i] >> shift) : ng;
    int gp = i > 0 ? (int)(skeys[i - 1] >> shift) : -1;
    for (int q = gp + 1; q <= g; ++q) first[q] = (int)i;
}

__global__ void k_tiles_per_bin(int nb, const int *first, int tp, int *cnt, int *ntiles) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int c = first[b + 1] - first[b];
    cnt[b] = c;
    ntiles[b] = (c + tp - 1) / tp;
}

__global__ void k_make_tiles(int ng, const int *cnt, const int *first, const int *tstart, int tp,
                             int per_bin, int4 *tiles) {
    int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int n = cnt[g], f = first[g], o = tstart[g];
    for (int q = 0; q * tp < n; ++q)
        tiles[o + q] = make_int4(g / per_bin, f + q * tp, min(tp, n - q * tp), g);
}

// labels back to the caller's point order: 4 per thread (vector loads), scattered stores
__global__ void k_unpermute(long long n, const unsigned *perm, const int *src, int *dst) {
    const long long i = 4 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
    if (i + 3 < n) {
        const uint4 pm = *reinterpret_cast<const uint4 *>(perm + i);
        const int4 sv = *reinterpret_cast<const int4 *>(src + i);
        dst[pm.x] = sv.x;
        dst[pm.y] = sv.y;
        dst[pm.z] = sv.z;
        dst[pm.w] = sv.w;
    } else {
        for (long long q = i; q < n; ++q) dst[perm[q]] = src[q];
    }
}

__global__ void k_copy_state(int K, mfseg_centers s, mfseg_centers d) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    for (int q = 0; q < 4; ++q) d.loc[q * K + c] = s.loc[q * K + c];
    d.pval[c] = s.pval[c];
    d.fval[c] = s.fval[c];
    d.has_p[c] = s.has_p[c];
    d.has_f[c] = s.has_f[c];
    d.dormant[c] = s.dormant[c];
    d.n_points[c] = s.n_points[c];
    d.n_fields[c] = s.n_fields[c];
}

__global__ void k_minmax(const double *v, long long n, unsigned long long *mm) {
    // mm[0] = ordered-bits min, mm[1] = ordered-bits max (total order on doubles)
    // mm[2] = non-zero when a value is NaN or +-inf
    double lo = __builtin_huge_val(), hi = -__builtin_huge_val();
    bool bad = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double x = v[i];
        lo = fmin(lo, x);
        hi = fmax(hi, x);
        bad |= !isfinite(x);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&mm[2], 1ull);
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        auto key = [](double d) {
            unsigned long long b = (unsigned long long)__double_as_longlong(d);
            return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        };
        atomicMin(&mm[0], key(lo));
        atomicMax(&mm[1], key(hi));
    }
}

__global__ void k_normalize(double *v, long long n, double lo, double span, int degenerate) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        v[i] = degenerate ? 0.0 : DDIV(DSUB(v[i], lo), span);
}

double unkey(unsigned long long b) {
    unsigned long long r = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    double d;
    memcpy(&d, &r, sizeof d);
    return d;
}

int bits_for(long long maxval) {
    int b = 1;
    while ((1ll << b) <= maxval) ++b;
    return b;
}

// ------------------------------------------------------------------ plan
struct State {                 // device centre state buffers (length K)
    mfseg_centers v;
};

struct Plan {
    mfseg_params p;
    mfseg_field f;
    mfseg_points pts;
    int K;                          // centres
    int NB;                         // bins = k1*k2*k3*k4
    int swap_zt;                    // thin field: the field kernels' z axis is time (FieldArgs)
    long long nbricks;              // brick records allocated (64 per block)
    int seeds_fast;                 // the initial pass may label interior blocks / chunks by
                                    // their own seed (seeds_fast_ok)
    long long nf, np;
    cudaStream_t st;
    // centre state ping-pong
    mfseg_centers s[2];
    unsigned long long *acc;
    long long *limbs;
    void *flags;
    // grid
    Grid g;
    int *count_tmp;
    void *grid_scan_tmp;
    // field
    AxisTile *xt, *yt, *zt;
    int ntx, nty, ntz, ntt;
    int *tbin;
    AxisTile *tt;
    float2 *brange;                 // per brick value range (field v5)
    ulonglong2 *bsum;               // per brick value sum, fixed point (field v5)
    MultiItem *multi;               // multi-candidate bricks for k_field_screen
    long long multi_cap;
    unsigned char *bslot;           // per brick: slot of its single label last pass (255: none)
    int *bcid;                      // per brick: centre id of that label
    BlockCache *bcache;             // per field block: its per-cluster sums (k_field_assign5)
    unsigned char *bmark, *bstable; // per sample bin: changed centres / stable neighbourhood
    unsigned char *smark, *sstable; // per sample bin: structural changes (bin, validity box, has)
    float *cdelta;                  // per centre: bound of its metric change in the last update
    unsigned *cbmax;                // per bin: largest cdelta of its centres (float bits)
    float *bdmax;                   // per sample bin: largest cdelta among its candidates
    float *bmargin;                 // per brick: proven margin of its single label
    int4 *vbox_prev;                // validity boxes of the previous pass
    unsigned char *tslot;           // per point warp tile: slot of its single label last pass
    PointCache *pcache;             // per point chunk: its per-cluster sums (k_point_assign4)
    long long *stranded_f, *deferred_f;
    long long cap_f;
    unsigned long long *absmax;     // [0..3] max |point x, y, z, t|, [4] |point v|, [5] |field v|
                                    // (double bits), [6] non-finite input flag
    unsigned long long *counters;   // [0] field stranded, [1] point stranded
    int *overflow;
    // points
    unsigned *keys, *vals, *skeys, *perm;
    double *px, *py, *pz, *pt, *pv;
    int *plabels;                   // bin-sorted labels
    int *bcnt, *bfirst, *btiles, *tstart;   // per (bin, interval) group
    int ngroups, nint, sub_bits, key_bits;
    int4 *tiles;
    double *tbox;                   // exact box per point chunk (v4)
    WBox *wbox;                     // per warp tile of a chunk (v4)
    long long max_tiles;
    long long *stranded_p, *deferred_p;
    long long cap_p;
    void *radix_tmp;
    size_t radix_bytes;
    void *scan_tmp;
    size_t scan_bytes;
};

// Initial pass (seeds at the bin midpoints mins + (j + 0.5) C, w_v = 0): a sample
// whose scaled bin coordinate u = (s - min) / C (fp64, as the reference bins it)
// has a fractional part in [eta, 1 - eta] on every axis is nearer to its own bin's
// seed than to any other seed by a squared-distance gap of at least
// 2 eta (C_d c_d)^2 on some axis (c_d = c_f for time, 1 otherwise), and its own
// seed passes the box test.  seeds_fast_ok checks that this gap dwarfs the fp64
// error of the reference's D over the 3^4 candidates (then the own seed is the
// unique argmin, no tie); interior_cell is the per-coordinate test.
constexpr double SEED_ETA = 0x1.0p-20;

bool interior_coord(double x, double mn, double C, int k) {
    volatile double u = (x - mn) / C;   // fl(fl(x - mn) / C): no contraction on the host
    const double f = u - std::floor(u);
    return u >= 0.0 && u < (double)k && f >= SEED_ETA && f <= 1.0 - SEED_ETA;
}

bool seeds_fast_ok(const mfseg_params &p) {
    double dmax2 = 0.0, gmin = INFINITY;
    for (int d = 0; d < 4; ++d) {
        const double cs = p.C[d] * (d == 3 ? std::fabs(p.c_f) : 1.0);
        dmax2 += 4.0 * cs * cs;                     // |c - s| <= 2 C on every axis of a candidate
        gmin = std::fmin(gmin, 2.0 * SEED_ETA * cs * cs);
        // the seeds and the binning quotient carry fp64 errors ~2^-52 (|min| / C + k)
        // bins: far below eta while that stays under 2^28
        if (!(std::fabs(p.mins[d]) / p.C[d] + (double)p.k[d] < 0x1.0p28)) return false;
    }
    return std::isfinite(dmax2) && dmax2 > 0.0 && gmin > 0x1.0p-40 * dmax2;   // fp64 error ~2^-50
}

// tiles of <= T cells along one axis that never straddle a bin boundary; `off` =
// global index of the first local cell (spatial slabs: a slab that starts on a
// bin boundary gets exactly the tiles of the whole grid)
std::vector<AxisTile> axis_tiles(int n, double o, double s, int off, double mn, double C, int k, int T) {
    std::vector<AxisTile> v;
    int i = 0;
    while (i < n) {
        int b = bin_coord(cell_coord(o, s, (long long)off + i), mn, C, k);
        int j = i;
        while (j < n && j - i < T && bin_coord(cell_coord(o, s, (long long)off + j), mn, C, k) == b) ++j;
        v.push_back(AxisTile{i, j - i, b, 0});
        i = j;
    }
    return v;
}

long long axis_tile_count(int n, double o, double s, int off, double mn, double C, int k, int T) {
    return (long long)axis_tiles(n, o, s, off, mn, C, k, T).size();
}

int check_inputs(const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts) {
    if (!p) {
        set_error("params is NULL");
        return 2;
    }
    for (int d = 0; d < 4; ++d)
        if (p->k[d] < 1 || !(p->C[d] > 0)) {
            set_error("invalid k or C (k must be >= 1, C > 0)");
            return 2;
        }
    long long NB = (long long)p->k[0] * p->k[1] * p->k[2] * p->k[3];
    if (NB > (1ll << 26) || p->n_centers > (1 << 26) || p->n_centers < 0) {
        set_error("too many clusters (K > 2^26)");
        return 2;
    }
    if (f && f->nt > 0 && (f->nx < 1 || f->ny < 1 || f->nz < 1)) {
        set_error("invalid field dims");
        return 2;
    }
    if (f && f->nt > 0 && (f->offset[0] < 0 || f->offset[1] < 0 || f->offset[2] < 0)) {
        set_error("invalid field offset (global index of the first cell must be >= 0)");
        return 2;
    }
    if (pts && pts->n >= (1ll << 31)) {
        set_error("more than 2^31-1 point samples on one GPU; shard the points");
        return 2;
    }
    return 0;
}

// Carve every buffer; with base == nullptr only sizes are computed.
size_t plan_carve(Plan &P, void *ws, size_t bytes) {
    Carver cv(ws, bytes);
    int K = P.K;
    for (int q = 0; q < 2; ++q) {
        P.s[q].loc = cv.take<double>(4ll * K);
        P.s[q].pval = cv.take<double>(K);
        P.s[q].fval = cv.take<double>(K);
        P.s[q].has_p = cv.take<uint8_t>(K);
        P.s[q].has_f = cv.take<uint8_t>(K);
        P.s[q].dormant = cv.take<uint8_t>(K);
        P.s[q].n_points = cv.take<int64_t>(K);
        P.s[q].n_fields = cv.take<int64_t>(K);
    }
    P.acc = cv.take<unsigned long long>((long long)K * MFSEG_ACC_WORDS);
    P.limbs = cv.take<long long>((long long)K * MFSEG_ACC_WORDS / 2 * 3);
    P.flags = cv.take<char>(update_flags_bytes());
    int NB = P.NB;
    P.g = grid_carve(cv, K, NB, &P.count_tmp, &P.grid_scan_tmp);
    P.counters = cv.take<unsigned long long>(40);   // [8..40): debug stats
    P.absmax = cv.take<unsigned long long>(8);
    P.overflow = cv.take<int>(4);
    // field
    P.nf = (P.f.nt > 0) ? (long long)P.f.nx * P.f.ny * P.f.nz * P.f.nt : 0;
    int TX, TY, TZ;
    field_tile_dims(&TX, &TY, &TZ);
    P.ntx = P.nty = P.ntz = 0;
    if (P.nf > 0) {
        P.ntx = (int)axis_tile_count(P.f.nx, P.f.origin[0], P.f.spacing[0], P.f.offset[0], P.p.mins[0], P.p.C[0],
                                     P.p.k[0], TX);
        P.nty = (int)axis_tile_count(P.f.ny, P.f.origin[1], P.f.spacing[1], P.f.offset[1], P.p.mins[1], P.p.C[1],
                                     P.p.k[1], TY);
        P.ntz = (int)axis_tile_count(P.f.nz, P.f.origin[2], P.f.spacing[2], P.f.offset[2], P.p.mins[2], P.p.C[2],
                                     P.p.k[2], TZ);
    }
    // thin fields (one z plane and one z bin): blocks and bricks run along time
    P.swap_zt = P.nf > 0 && P.f.nz == 1 && P.f.nt > 1 && P.p.k[2] == 1 &&
                !(debug_options().flags & MFSEG_DEBUG_NO_ZT_SWAP);
    P.xt = cv.take<AxisTile>(P.ntx);
    P.yt = cv.take<AxisTile>(P.nty);
    P.zt = cv.take<AxisTile>(std::max(P.ntz, P.f.nt > 0 ? P.f.nt : 1));   // z tiles, or time tiles
    P.tbin = cv.take<int>(P.f.nt > 0 ? P.f.nt : 1);
    P.tt = cv.take<AxisTile>(P.f.nt > 0 ? P.f.nt : 1);
    // blocks <= ntx nty ntz nt either way (swapped: ntz = 1 z tile, <= nt time tiles)
    P.nbricks = 64ll * P.ntx * P.nty * P.ntz * (P.f.nt > 0 ? P.f.nt : 1);
    P.brange = cv.take<float2>(P.nbricks);
    P.bsum = cv.take<ulonglong2>(P.nbricks);
    {
        const long long bricks = P.nbricks;
        // every live brick can be queued (96 B per brick of <= 256 samples): a full
        // queue would send the rest to the per-sample exact path (k_deferred), 10-100x
        // slower.  Live bricks per block are a product over the axes (thin grids,
        // e.g. nz = 1, leave most of a block's 64 brick slots empty).
        long long live = 0;
        if (P.nf > 0) {
            int TX, TY, TZ;
            field_tile_dims(&TX, &TY, &TZ);
            auto per_axis = [](const std::vector<AxisTile> &v, int g) {
                long long c = 0;
                for (const AxisTile &t : v) c += (t.len + g - 1) / g;
                return c;
            };
            const long long lx = per_axis(axis_tiles(P.f.nx, P.f.origin[0], P.f.spacing[0], P.f.offset[0],
                                                     P.p.mins[0], P.p.C[0], P.p.k[0], TX), 8);
            const long long ly = per_axis(axis_tiles(P.f.ny, P.f.origin[1], P.f.spacing[1], P.f.offset[1],
                                                     P.p.mins[1], P.p.C[1], P.p.k[1], TY), 4);
            const long long lz = per_axis(axis_tiles(P.f.nz, P.f.origin[2], P.f.spacing[2], P.f.offset[2],
                                                     P.p.mins[2], P.p.C[2], P.p.k[2], TZ), 4);
            // time tiles: ceil(len / 2) bricks each, at most len: <= nt in all
            live = lx * ly * lz * (long long)P.f.nt;
        }
        P.multi_cap = P.nf > 0 ? (live < bricks ? live : bricks) : 0;
        P.multi = cv.take<MultiItem>(P.multi_cap);
        P.bslot = cv.take<unsigned char>(P.nf > 0 ? bricks : 0);
        P.bmargin = cv.take<float>(P.nf > 0 ? bricks : 0);
        P.bcid = cv.take<int>(P.nf > 0 ? bricks : 0);
        P.bcache = cv.take<BlockCache>(P.nf > 0 ? bricks / 64 : 0);
    }
    P.bmark = cv.take<unsigned char>(NB);
    P.bstable = cv.take<unsigned char>(NB);
    P.smark = cv.take<unsigned char>(NB);
    P.sstable = cv.take<unsigned char>(NB);
    P.cdelta = cv.take<float>(K);
    P.cbmax = cv.take<unsigned>(NB);
    P.bdmax = cv.take<float>(NB);
    P.vbox_prev = cv.take<int4>(P.nf > 0 ? 2ll * K : 0);
    P.cap_f = P.nf < (1ll << 22) ? P.nf : (1ll << 22);
    P.stranded_f = cv.take<long long>(P.cap_f);
    P.deferred_f = cv.take<long long>(P.cap_f);
    // points
    long long n = P.np;
    int TP = point_tile_size();
    P.keys = cv.take<unsigned>(n);
    P.vals = cv.take<unsigned>(n);
    P.skeys = cv.take<unsigned>(n);
    P.perm = cv.take<unsigned>(n);
    P.px = cv.take<double>(n);
    P.py = cv.take<double>(n);
    P.pz = cv.take<double>(n);
    P.pt = cv.take<double>(n);
    P.pv = cv.take<double>(n);
    P.plabels = cv.take<int>(n);
    // point tile groups: one per sample bin.  (A bin never straddles a time
    // slab because multi-GPU slabs are whole t-bins, parallel.time_slab.)
    P.nint = 1;
    {
        long long G = (long long)NB * P.nint;
        int gb = bits_for(G - 1);
        P.ngroups = (int)G;
#ifndef MFSEG_SUB_BITS
#define MFSEG_SUB_BITS 4   // one Morton bit per axis (tools/variant_time.sh: 2-8 and 12 measured)
#endif
        constexpr int SB = MFSEG_SUB_BITS;   // 2^SB Morton sub-cells per bin
        P.sub_bits = gb + SB <= 32 ? SB : (32 - gb > 0 ? 32 - gb : 0);
        P.key_bits = gb + P.sub_bits;
    }
    const int NG = P.ngroups;
    P.bcnt = cv.take<int>(NG + 1);
    P.bfirst = cv.take<int>(NG + 1);
    P.btiles = cv.take<int>(NG + 1);
    P.tstart = cv.take<int>(NG + 1);
    P.max_tiles = n > 0 ? (n + TP - 1) / TP + NG : 0;
    P.tiles = cv.take<int4>(P.max_tiles);
    P.tbox = cv.take<double>(8 * P.max_tiles);
    P.wbox = cv.take<WBox>(P.max_tiles * (POINT_CHUNK / 64));
    P.tslot = cv.take<unsigned char>(P.max_tiles * (POINT_CHUNK / 64));
    P.pcache = cv.take<PointCache>(P.max_tiles);
    P.cap_p = n < (1ll << 22) ? n : (1ll << 22);
    P.stranded_p = cv.take<long long>(P.cap_p);
    P.deferred_p = cv.take<long long>(P.cap_p);
    P.radix_bytes = n > 0 ? radix_tmp_bytes(n) : 0;
    P.radix_tmp = cv.take<char>(P.radix_bytes);
    P.scan_bytes = scan_tmp_bytes((long long)(NG > NB ? NG : NB) + 1) + 1024;
    P.scan_tmp = cv.take<char>(P.scan_bytes);
    return cv.off + 1024;
}

int plan_init(Plan &P, const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts,
              void *ws, size_t bytes, cudaStream_t st) {
    MFSEG_TRY(check_inputs(p, f, pts));
    memset(&P, 0, sizeof P);
    P.p = *p;
    if (f) P.f = *f;
    if (pts) P.pts = *pts;
    P.NB = p->k[0] * p->k[1] * p->k[2] * p->k[3];
    P.K = p->n_centers > 0 ? p->n_centers : P.NB;
    P.np = pts ? pts->n : 0;
    P.st = st;
    size_t need = plan_carve(P, nullptr, 0);
    if (!ws || bytes < need) {
        set_error("workspace too small: need " + std::to_string(need) + " bytes");
        return 3;
    }
    plan_carve(P, ws, bytes);
    return 0;
}

// Inputs must be finite, and every per-cluster sum must fit the
// 128-bit fixed-point accumulators (2^-64 units, |sum| < 2^63): with m = the
// largest |input| of a sum and n its sample count, m * n < 2^62 is required.
int check_ranges(Plan &P, double field_coord_max) {
    unsigned long long *h = nullptr;
    void *d = nullptr;
    MFSEG_TRY(tiny_scratch(&d, (void **)&h));
    MFSEG_CUDA(cudaMemcpyAsync(h, P.absmax, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost, P.st));
    MFSEG_CUDA(cudaStreamSynchronize(P.st));
    if (h[6]) {
        set_error("non-finite (NaN or inf) sample value or coordinate");
        return 2;
    }
    double m[6];
    for (int i = 0; i < 6; ++i) memcpy(&m[i], &h[i], sizeof(double));
    const double n = (double)(P.np + P.nf), lim = 0x1.0p62;
    double coord = field_coord_max;
    for (int i = 0; i < 4; ++i) coord = std::fmax(coord, m[i]);
    if (coord * n >= lim || m[4] * (double)P.np >= lim || m[5] * (double)P.nf >= lim) {
        set_error("sample coordinates or values too large for the exact 128-bit cluster sums "
                  "(max |x| * samples must stay below 2^62): rescale or shift the inputs");
        return 2;
    }
    return 0;
}

// once per run: field axis tiles, timestep bins, point binning + sort + tiles
int plan_prepare_impl(Plan &P);

int plan_prepare(Plan &P) {   // once per run, under one NVTX range
    nvtxRangePushA("mfseg prepare");
    const int rc = plan_prepare_impl(P);
    nvtxRangePop();
    return rc;
}

int plan_prepare_impl(Plan &P) {
    cudaStream_t st = P.st;
    const mfseg_params &p = P.p;
    MFSEG_CUDA(cudaMemsetAsync(P.absmax, 0, sizeof(unsigned long long) * 8, st));
    double field_coord_max = 0.0;   // max |cell centre| and |time| of the field (host)
    if (P.nf > 0) {
        int TX, TY, TZ;
        field_tile_dims(&TX, &TY, &TZ);
        auto xt = axis_tiles(P.f.nx, P.f.origin[0], P.f.spacing[0], P.f.offset[0], p.mins[0], p.C[0], p.k[0], TX);
        auto yt = axis_tiles(P.f.ny, P.f.origin[1], P.f.spacing[1], P.f.offset[1], p.mins[1], p.C[1], p.k[1], TY);
        auto zt = axis_tiles(P.f.nz, P.f.origin[2], P.f.spacing[2], P.f.offset[2], p.mins[2], p.C[2], p.k[2], TZ);
        // initial-pass flag per tile: every cell interior to its bin (AxisTile.pad)
        auto flag = [&](std::vector<AxisTile> &v, int d) {
            for (AxisTile &t : v) {
                bool ok = true;
                for (int i = t.start; ok && i < t.start + t.len; ++i)
                    ok = interior_coord(cell_coord(P.f.origin[d], P.f.spacing[d], (long long)P.f.offset[d] + i),
                                        p.mins[d], p.C[d], p.k[d]);
                t.pad = ok;
            }
        };
        flag(xt, 0);
        flag(yt, 1);
        flag(zt, 2);
        MFSEG_CUDA(cudaMemcpyAsync(P.xt, xt.data(), sizeof(AxisTile) * xt.size(),
                                   cudaMemcpyHostToDevice, st));
        MFSEG_CUDA(cudaMemcpyAsync(P.yt, yt.data(), sizeof(AxisTile) * yt.size(),
                                   cudaMemcpyHostToDevice, st));

        // time tiles: runs of <= 4 timesteps with the same t-bin (host copy of the
        // times; bin_coord on the host rounds exactly like the device)
        std::vector<double> th(P.f.nt);
        MFSEG_CUDA(cudaMemcpyAsync(th.data(), P.f.times, sizeof(double) * P.f.nt,
                                   cudaMemcpyDeviceToHost, st));
        MFSEG_CUDA(cudaStreamSynchronize(st));
        std::vector<AxisTile> tts;
        for (int m0 = 0; m0 < P.f.nt;) {
            const int b = bin_coord(th[m0], p.mins[3], p.C[3], p.k[3]);
            int m1 = m0;
            while (m1 < P.f.nt && m1 - m0 < 4 && bin_coord(th[m1], p.mins[3], p.C[3], p.k[3]) == b) ++m1;
            bool ok = true;
            for (int m = m0; ok && m < m1; ++m) ok = interior_coord(th[m], p.mins[3], p.C[3], p.k[3]);
            tts.push_back(AxisTile{m0, m1 - m0, b, ok ? 1 : 0});
            m0 = m1;
        }
        P.ntt = (int)tts.size();
        if (P.swap_zt) {
            // the kernels' z axis runs over time: runs of <= TZ timesteps with the same
            // t-bin; their t axis over the single z tile
            std::vector<AxisTile> zts;
            for (int m0 = 0; m0 < P.f.nt;) {
                const int b = bin_coord(th[m0], p.mins[3], p.C[3], p.k[3]);
                int m1 = m0;
                while (m1 < P.f.nt && m1 - m0 < TZ && bin_coord(th[m1], p.mins[3], p.C[3], p.k[3]) == b) ++m1;
                bool ok = true;
                for (int m = m0; ok && m < m1; ++m) ok = interior_coord(th[m], p.mins[3], p.C[3], p.k[3]);
                zts.push_back(AxisTile{m0, m1 - m0, b, ok ? 1 : 0});
                m0 = m1;
            }
            tts = zt;
            zt = zts;
            P.ntz = (int)zt.size();
            P.ntt = (int)tts.size();
        }
        MFSEG_CUDA(cudaMemcpyAsync(P.zt, zt.data(), sizeof(AxisTile) * zt.size(),
                                   cudaMemcpyHostToDevice, st));
        for (int m = 0; m < P.f.nt; ++m) {
            if (!std::isfinite(th[m])) {
                set_error("non-finite field time");
                return 2;
            }
            field_coord_max = std::fmax(field_coord_max, std::fabs(th[m]));
        }
        for (int d = 0; d < 3; ++d) {
            const int n = d == 0 ? P.f.nx : d == 1 ? P.f.ny : P.f.nz;
            if (!std::isfinite(P.f.origin[d]) || !std::isfinite(P.f.spacing[d])) {
                set_error("non-finite field origin or spacing");
                return 2;
            }
            field_coord_max = std::fmax(field_coord_max, std::fabs(cell_coord(P.f.origin[d], P.f.spacing[d], P.f.offset[d])));
            field_coord_max = std::fmax(field_coord_max, std::fabs(cell_coord(P.f.origin[d], P.f.spacing[d], (long long)P.f.offset[d] + n - 1)));
        }
        MFSEG_CUDA(cudaMemcpyAsync(P.tt, tts.data(), sizeof(AxisTile) * tts.size(),
                                   cudaMemcpyHostToDevice, st));
        MFSEG_CUDA(cudaStreamSynchronize(st));   // host vectors die at scope exit
        ::mfseg::count_launch();
        k_tbins<<<(P.f.nt + 255) / 256, 256, 0, st>>>(P.f.nt, P.f.times, p.mins[3], p.C[3],
                                                        p.k[3], P.tbin);
        MFSEG_LAUNCH("k_tbins");
        {   // per-brick value ranges and sums (the values are fixed for the whole run)
            FieldArgs va;
            memset(&va, 0, sizeof va);
            va.nx = P.f.nx;
            va.ny = P.f.ny;
            va.nz = P.swap_zt ? P.f.nt : P.f.nz;   // (swapped: the planes are the timesteps)
            va.nt = P.swap_zt ? 1 : P.f.nt;
            va.swap_zt = P.swap_zt;
            va.values = P.f.values;
            va.xt = P.xt;
            va.yt = P.yt;
            va.zt = P.zt;
            va.tt = P.tt;
            va.ntx = P.ntx;
            va.nty = P.nty;
            va.ntz = P.ntz;
            va.ntt = P.ntt;
            va.brange_out = P.brange;
            va.bsum_out = P.bsum;
            va.overflow = P.overflow;
            va.absmax = P.absmax;
            MFSEG_TRY(launch_brick_pre(va, st));
        }
        if (P.bslot) MFSEG_CUDA(cudaMemsetAsync(P.bslot, 255, P.nbricks, st));
        if (P.bcache)   // n = -1: no block has cached sums yet
            MFSEG_CUDA(cudaMemsetAsync(P.bcache, 255, sizeof(BlockCache) * (P.nbricks / 64), st));
    }
    long long n = P.np;
    if (n > 0) {
        double4 mins = make_double4(p.mins[0], p.mins[1], p.mins[2], p.mins[3]);
        double4 C = make_double4(p.C[0], p.C[1], p.C[2], p.C[3]);
        int4 k = make_int4(p.k[0], p.k[1], p.k[2], p.k[3]);
        unsigned gb = (unsigned)((n + 255) / 256);
        ::mfseg::count_launch();
        const double4 inv = make_double4(1.0 / p.C[0], 1.0 / p.C[1], 1.0 / p.C[2], 1.0 / p.C[3]);
        k_point_keys<<<gb, 256, 0, st>>>(n, P.pts.xyz, P.pts.t, mins, C, inv, k, P.f.times, P.nint,
                                         P.sub_bits, P.keys, P.vals);
        MFSEG_LAUNCH("k_point_keys");
        if (P.key_bits > 32) {
            set_error("too many (bin, timestep) groups for 32-bit point keys");
            return 2;
        }
        MFSEG_TRY(radix_sort_pairs(P.keys, P.vals, P.skeys, P.perm, n, P.key_bits, P.radix_tmp,
                                   P.radix_bytes, st));
        const int NG = P.ngroups;
        ::mfseg::count_launch();
        k_bin_first<<<(unsigned)((n + 256) / 256), 256, 0, st>>>(n, P.skeys, P.sub_bits, NG,
                                                                 P.bfirst);
        int TP = point_tile_size();
        unsigned gk = (unsigned)((NG + 256) / 256);
        MFSEG_CUDA(cudaMemsetAsync(P.btiles, 0, sizeof(int) * (NG + 1), st));
        ::mfseg::count_launch();
        k_tiles_per_bin<<<gk, 256, 0, st>>>(NG, P.bfirst, TP, P.bcnt, P.btiles);
        MFSEG_TRY(scan_exclusive_i32(P.btiles, P.tstart, NG + 1, P.scan_tmp, P.scan_bytes, st));
        ::mfseg::count_launch();
        k_make_tiles<<<gk, 256, 0, st>>>(NG, P.bcnt, P.bfirst, P.tstart, TP, P.nint, P.tiles);
        MFSEG_LAUNCH("point tiles");
        // the points are gathered into the bin-sorted SoA chunk by chunk here
        MFSEG_TRY(launch_tile_box(P.absmax, P.tiles, P.tstart + NG, P.max_tiles, P.px, P.py, P.pz, P.pt,
                                      P.pv, p.c_f, P.tbox, P.wbox, P.perm, P.pts.xyz, P.pts.t,
                                      P.pts.value, st));
        MFSEG_CUDA(cudaMemsetAsync(P.tslot, 255, P.max_tiles * (POINT_CHUNK / 64), st));
        MFSEG_CUDA(cudaMemsetAsync(P.pcache, 255, sizeof(PointCache) * P.max_tiles, st));   // n = -1
    }
    return check_ranges(P, field_coord_max);
}

CentersView view_of(const mfseg_centers &s, int K) {
    CentersView v;
    v.x = s.loc;
    v.y = s.loc + K;
    v.z = s.loc + 2ll * K;
    v.t = s.loc + 3ll * K;
    v.pval = s.pval;
    v.fval = s.fval;
    v.has_p = s.has_p;
    v.has_f = s.has_f;
    return v;
}

// Centres changed by the last update (position, point or field value or their
// presence, bitwise): mark the sample bins they left and entered (mark).  A
// centre whose bin, field validity box or field has-flag changed also marks
// them in smark (structural change).  cdelta: an upper bound of how much its
// field metric w_d sst + w_f |v - cv| can change at any sample.
__global__ void k_mark_changed(int K, mfseg_centers cur, mfseg_centers old, double4 mins, double4 C,
                               int4 k, double cf, double wd, double wf, const int4 *vbox,
                               const int4 *vbox_prev, unsigned char *mark, unsigned char *smark,
                               float *cdelta, unsigned *cbmax) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    bool ch = cur.has_f[c] != old.has_f[c] || cur.has_p[c] != old.has_p[c] ||
              __double_as_longlong(cur.fval[c]) != __double_as_longlong(old.fval[c]) ||
              __double_as_longlong(cur.pval[c]) != __double_as_longlong(old.pval[c]);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        ch |= __double_as_longlong(cur.loc[(size_t)q * K + c]) != __double_as_longlong(old.loc[(size_t)q * K + c]);
    float delta = 0.f;
    if (ch) {
        double d2 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double d = cur.loc[(size_t)q * K + c] - old.loc[(size_t)q * K + c];
            if (q == 3) d *= cf;
            d2 += d * d;
        }
        double dv = 0.0;
        if (cur.has_f[c] && old.has_f[c]) dv = fabs(cur.fval[c] - old.fval[c]);
        delta = __double2float_ru((wd * sqrt(d2) + wf * dv) * (1.0 + 0x1.0p-30) + 1e-300);
    }
    cdelta[c] = delta;
    if (!ch) return;
    const double mn[4] = {mins.x, mins.y, mins.z, mins.w}, CC[4] = {C.x, C.y, C.z, C.w};
    const int kk[4] = {k.x, k.y, k.z, k.w};
    int bn[4], bo[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        bn[q] = bin_coord(cur.loc[(size_t)q * K + c], mn[q], CC[q], kk[q]);
        bo[q] = bin_coord(old.loc[(size_t)q * K + c], mn[q], CC[q], kk[q]);
    }
    const int fn = ((bn[3] * k.z + bn[2]) * k.y + bn[1]) * k.x + bn[0];
    // per bin the largest move of its centres (non-negative floats order as their bits)
    if (cbmax && delta > 0.f) atomicMax(&cbmax[fn], __float_as_uint(delta));
    const int fo = ((bo[3] * k.z + bo[2]) * k.y + bo[1]) * k.x + bo[0];
    mark[fn] = 1;
    mark[fo] = 1;
    bool sch = fn != fo || cur.has_f[c] != old.has_f[c];
    if (vbox) {
        const int4 a0 = vbox[2 * c], a1 = vbox[2 * c + 1], b0 = vbox_prev[2 * c], b1 = vbox_prev[2 * c + 1];
        sch |= a0.x != b0.x || a0.y != b0.y || a0.z != b0.z || a0.w != b0.w || a1.x != b1.x ||
               a1.y != b1.y || a1.z != b1.z || a1.w != b1.w;
    }
    if (sch) {
        smark[fn] = 1;
        smark[fo] = 1;
    }
}

// A sample bin is stable when none of its 3^4 neighbour bins is marked: its
// candidate list and every candidate's state equal the last pass's.  One warp
// per bin, the 81 neighbours over the lanes.
__global__ void k_bin_stable(int NB, int4 k, const unsigned char *mark, unsigned char *stable,
                             const unsigned char *smark, unsigned char *sstable, const unsigned *cbmax,
                             float *bdmax) {
    const int lane = threadIdx.x & 31;
    const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (b >= NB) return;   // warp-uniform
    int r = (int)b;
    const int bx = r % k.x;
    r /= k.x;
    const int by = r % k.y;
    r /= k.y;
    const int bz = r % k.z;
    const int bt = r / k.z;
    bool ok = true, sok = true;
    unsigned dm = 0;
    for (int j = lane; j < 81; j += 32) {   // j = (dt, dz, dy, dx) + 1, base 3
        const int qx = bx + j % 3 - 1, qy = by + (j / 3) % 3 - 1, qz = bz + (j / 9) % 3 - 1,
                  qt = bt + j / 27 - 1;
        if (qx < 0 || qy < 0 || qz < 0 || qt < 0 || qx >= k.x || qy >= k.y || qz >= k.z || qt >= k.w)
            continue;
        const int q = ((qt * k.z + qz) * k.y + qy) * k.x + qx;
        ok = ok && !mark[q];
        sok = sok && !smark[q];
        if (cbmax) dm = max(dm, cbmax[q]);
    }
    ok = __all_sync(0xffffffffu, ok);
    sok = __all_sync(0xffffffffu, sok);
    dm = __reduce_max_sync(0xffffffffu, dm);
    if (lane == 0) {
        stable[b] = ok;
        sstable[b] = sok;
        if (bdmax) bdmax[b] = __uint_as_float(dm);   // largest move among the bin's candidates
    }
}

// one assignment pass for centre state `c` (grid rebuilt here); `prev`: the
// state of the previous pass when it used the same weights (labels of stable
// field blocks are reused), else null
int plan_pass(Plan &P, const mfseg_centers &c, double wd, double wp, double wf, int32_t *flabels,
              int accumulate, const mfseg_centers *prev, int32_t *plabels_out, int initial) {
    // the initial pass of mfseg_run: seeds as centres, pure space-time metric
    const DebugOptions &dbg = debug_options();
    const int fast0 = initial && P.seeds_fast && wp == 0.0 && wf == 0.0 && wd == 1.0 &&
                      !(dbg.flags & MFSEG_DEBUG_NO_SEEDS_FAST);
    cudaStream_t st = P.st;
    const mfseg_params &p = P.p;
    int K = P.K;
    CentersView cv = view_of(c, K);
    mark(0, st);
    // validity boxes of the previous pass (structural-change test of the reuse)
    const bool reuse = prev && accumulate && !(dbg.flags & MFSEG_DEBUG_NO_REUSE);
    if (P.vbox_prev && P.nf > 0 && accumulate)
        MFSEG_CUDA(cudaMemcpyAsync(P.vbox_prev, P.g.vbox, sizeof(int4) * 2 * K, cudaMemcpyDeviceToDevice, st));
    MFSEG_TRY(grid_build(P.g, cv.x, cv.y, cv.z, cv.t, &p, P.nf > 0 ? &P.f : nullptr,
                         P.count_tmp, P.grid_scan_tmp, st));
    mark(1, st);
    MFSEG_CUDA(cudaMemsetAsync(P.counters, 0, sizeof(unsigned long long) * 40, st));
    // reuse of the previous pass: sample bins whose candidates did not change
    // (exactly, or only by bounded moves: see k_mark_changed)
    if (reuse) {
        const int NB = P.NB;
        MFSEG_CUDA(cudaMemsetAsync(P.bmark, 0, NB, st));
        MFSEG_CUDA(cudaMemsetAsync(P.smark, 0, NB, st));
        MFSEG_CUDA(cudaMemsetAsync(P.cbmax, 0, sizeof(unsigned) * NB, st));
        ::mfseg::count_launch();
        k_mark_changed<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(
            K, c, *prev, make_double4(p.mins[0], p.mins[1], p.mins[2], p.mins[3]),
            make_double4(p.C[0], p.C[1], p.C[2], p.C[3]), make_int4(p.k[0], p.k[1], p.k[2], p.k[3]),
            p.c_f, wd, wf, P.nf > 0 ? P.g.vbox : nullptr, P.nf > 0 ? P.vbox_prev : nullptr, P.bmark,
            P.smark, P.cdelta, P.cbmax);
        ::mfseg::count_launch();
        k_bin_stable<<<(unsigned)((32ll * NB + 255) / 256), 256, 0, st>>>(
            NB, make_int4(p.k[0], p.k[1], p.k[2], p.k[3]), P.bmark, P.bstable, P.smark, P.sstable, P.cbmax,
            P.bdmax);
        MFSEG_LAUNCH("stable bins");
    }
    if (accumulate)
        MFSEG_CUDA(cudaMemsetAsync(P.acc, 0, sizeof(unsigned long long) * K * MFSEG_ACC_WORDS, st));
    if (P.nf > 0) {
        FieldArgs a;
        memset(&a, 0, sizeof a);
        a.nx = P.f.nx;
        a.ny = P.f.ny;
        a.nz = P.swap_zt ? P.f.nt : P.f.nz;   // (swapped: the planes are the timesteps)
        a.nt = P.swap_zt ? 1 : P.f.nt;
        a.swap_zt = P.swap_zt;
        a.ox = P.f.origin[0];
        a.oy = P.f.origin[1];
        a.oz = P.f.origin[2];
        a.x0 = P.f.offset[0];
        a.y0 = P.f.offset[1];
        a.z0 = P.f.offset[2];
        a.sx = P.f.spacing[0];
        a.sy = P.f.spacing[1];
        a.sz = P.f.spacing[2];
        a.times = P.f.times;
        a.values = P.f.values;
        a.xt = P.xt;
        a.yt = P.yt;
        a.zt = P.zt;
        a.ntx = P.ntx;
        a.nty = P.nty;
        a.ntz = P.ntz;
        a.tbin = P.tbin;
        a.tt = P.tt;
        a.brange = P.brange;
        a.bsum = P.bsum;
        a.ntt = P.ntt;
        a.kx = p.k[0];
        a.ky = p.k[1];
        a.kz = P.swap_zt ? p.k[3] : p.k[2];
        a.kt = P.swap_zt ? p.k[2] : p.k[3];
        a.cf = p.c_f;
        a.wd = wd;
        a.wv = wf;
        a.c = cv;
        if (P.swap_zt) std::swap(a.c.z, a.c.t);   // the kernels' z axis is time
        a.cval = c.fval;
        a.chas = c.has_f;
        a.g = P.g;
        a.labels = flabels;
        a.acc = P.acc;
        a.stranded = P.stranded_f;
        a.n_stranded = P.counters;
        a.stranded_cap = P.cap_f;
        a.deferred = P.deferred_f;
        a.n_deferred = P.counters + 2;
        a.stats = P.counters + 8;
        a.deferred_cap = P.cap_f;
        a.multi = P.multi;
        a.n_multi = P.counters + 4;
        a.multi_cap = P.multi_cap;
        a.bslot = P.bslot;
        a.bmargin = a.bslot ? P.bmargin : nullptr;
        a.bcid = a.bslot ? P.bcid : nullptr;
        a.bcache = a.bslot && !(dbg.flags & MFSEG_DEBUG_NO_BLOCK_CACHE) ? P.bcache : nullptr;
        a.bin_dmax = P.bdmax;
        a.seeds_fast = fast0;
        if (reuse && a.bslot) {
            a.reuse = 1;
            a.bin_stable = P.bstable;
            a.bin_sstable = (dbg.flags & MFSEG_DEBUG_NO_MARGIN_REUSE) ? P.bstable : P.sstable;
            a.cdelta = P.cdelta;
        }
        if (dbg.multi_cap >= 0 && dbg.multi_cap < a.multi_cap) a.multi_cap = dbg.multi_cap;   // test knob
        a.overflow = P.overflow;
        a.accumulate = accumulate;
        a.debug = dbg.flags & MFSEG_DEBUG_KERNEL_BITS;
        long long ntiles = (long long)P.ntx * P.nty * P.ntz * P.f.nt;
        MFSEG_TRY(launch_field_assign(a, ntiles, st));
        MFSEG_TRY(launch_field_screen(a, st));
    }
    mark(2, st);
    if (P.np > 0) {
        PointArgs a;
        memset(&a, 0, sizeof a);
        a.n = P.np;
        a.x = P.px;
        a.y = P.py;
        a.z = P.pz;
        a.t = P.pt;
        a.v = P.pv;
        a.tiles = P.tiles;
        a.n_tiles = P.tstart + P.ngroups;
        a.tile_box = P.tbox;
        a.wbox = P.wbox;
        a.Cx = p.C[0];
        a.Cy = p.C[1];
        a.Cz = p.C[2];
        a.Ct = p.C[3];
        a.cf = p.c_f;
        a.wd = wd;
        a.wv = wp;
        a.c = cv;
        a.cval = c.pval;
        a.chas = c.has_p;
        a.g = P.g;
        a.labels = P.plabels;
        a.labels_out = plabels_out;   // final pass: record-order labels stored directly
        a.perm = P.perm;
        a.acc = P.acc;
        a.stranded = P.stranded_p;
        a.n_stranded = P.counters + 1;
        a.stranded_cap = P.cap_p;
        a.deferred = P.deferred_p;
        a.n_deferred = P.counters + 3;
        a.stats = P.counters + 16;
        a.deferred_cap = P.cap_p;
        a.tslot = P.tslot;
        a.seeds_fast = fast0;
        for (int d = 0; d < 4; ++d) {
            a.mn[d] = p.mins[d];
            a.kk[d] = p.k[d];
        }
        if (reuse && a.tslot) {
            a.reuse = 1;
            a.bin_stable = P.bstable;
        }
        if (a.tslot && !(dbg.flags & MFSEG_DEBUG_NO_BLOCK_CACHE)) a.pcache = P.pcache;
        a.overflow = P.overflow;
        a.accumulate = accumulate;
        a.debug = dbg.flags & MFSEG_DEBUG_KERNEL_BITS;
        MFSEG_TRY(launch_point_assign(a, P.max_tiles, st));
    }
    mark(3, st);
    // stranded samples
    for (int kind = 0; kind < 2; ++kind) {
        if (kind == 1 && P.nf == 0) continue;
        if (kind == 0 && P.np == 0) continue;
        FallbackArgs a;
        memset(&a, 0, sizeof a);
        a.K = K;
        a.c = cv;
        a.cval = kind == 1 ? c.fval : c.pval;
        a.chas = kind == 1 ? c.has_f : c.has_p;
        for (int d = 0; d < 4; ++d) a.C[d] = p.C[d];
        a.cf = p.c_f;
        a.wd = wd;
        a.wv = kind == 1 ? wf : wp;
        a.kind = kind;
        a.nx = P.f.nx;
        a.ny = P.f.ny;
        a.nz = P.f.nz;
        a.nt = P.f.nt;
        a.ox = P.f.origin[0];
        a.oy = P.f.origin[1];
        a.oz = P.f.origin[2];
        a.x0 = P.f.offset[0];
        a.y0 = P.f.offset[1];
        a.z0 = P.f.offset[2];
        a.sx = P.f.spacing[0];
        a.sy = P.f.spacing[1];
        a.sz = P.f.spacing[2];
        a.times = P.f.times;
        a.values = P.f.values;
        a.px = P.px;
        a.py = P.py;
        a.pz = P.pz;
        a.pt = P.pt;
        a.pv = P.pv;
        a.n_samples = kind == 1 ? P.nf : P.np;
        a.labels = kind == 1 ? flabels : P.plabels;
        a.labels_out = kind == 1 ? nullptr : plabels_out;
        a.perm = P.perm;
        a.stranded = kind == 1 ? P.stranded_f : P.stranded_p;
        a.n_stranded = P.counters + (kind == 1 ? 0 : 1);
        a.cap = kind == 1 ? P.cap_f : P.cap_p;
        a.acc = P.acc;
        a.overflow = P.overflow;
        a.accumulate = accumulate;
        a.bin_start = P.g.bin_start;   // the CenterGrid of this pass (all K centres)
        a.bin_ids = P.g.bin_ids;
        for (int d = 0; d < 4; ++d) {
            a.mins[d] = p.mins[d];
            a.k[d] = p.k[d];
        }
        // crowded tiles first (may add stranded samples), then the fallback
        const int4 kk = make_int4(p.k[0], p.k[1], p.k[2], p.k[3]);
        MFSEG_TRY(launch_deferred(a, P.g, P.tbin, kk, p.mins, kind == 1 ? P.deferred_f : P.deferred_p,
                                  P.counters + (kind == 1 ? 2 : 3), a.cap, st));
        MFSEG_TRY(launch_fallback(a, st));
    }
    mark(4, st);
    {
        if (dbg.flags & MFSEG_DEBUG_STATS) {   // (kernel path counters: MFSEG_DEVICE_STATS builds only)
            if (!MFSEG_DEVICE_STATS)
                fprintf(stderr, "[mfseg stats] this library was built without -DMFSEG_DEVICE_STATS=1: "
                                "the kernel path counters below stay 0\n");
            unsigned long long h[40];
            MFSEG_CUDA(cudaMemcpyAsync(h, P.counters, sizeof h, cudaMemcpyDeviceToHost, st));
            MFSEG_CUDA(cudaStreamSynchronize(st));
            const unsigned long long *F = h + 8, *Q = h + 16;
            auto rat = [](unsigned long long a, unsigned long long b) { return b ? (double)a / b : 0.0; };
            fprintf(stderr,
                    "[mfseg stats] field: bricks %llu kept/brick %.2f exact %llu records/brick %.2f "
                    "regions %llu listed %.3f list/region %.2f | points: warp tiles %llu kept/tile %.2f "
                    "exact %llu | stranded f %llu p %llu deferred f %llu p %llu\n",
                    F[0], rat(F[1], F[0]), F[2], rat(F[3], F[0]), F[4], rat(F[5], F[4]), rat(F[6], F[5]),
                    Q[0], rat(Q[1], Q[0]), Q[2], h[0], h[1], h[2], h[3]);
            fprintf(stderr, "[mfseg stats] field bricks: kept after cull %.3f, single after cull %.3f, "
                    "reused %llu, screen items %llu exact samples %llu, bricks without s* %.3f\n",
                    rat(F[7], F[0]), rat(F[2], F[0]), h[32], h[33], h[34], rat(h[38], F[0]));
            fprintf(stderr, "[mfseg stats] point tiles single %.3f kept hist", rat(Q[3], Q[0]));
            for (int q = 0; q < 8; ++q) fprintf(stderr, " %.3f", rat(Q[4 + q], Q[0]));
            fprintf(stderr, " | chunks by candidate rounds 1/2/3/4: %llu %llu %llu %llu", Q[12], Q[13],
                    Q[14], Q[15]);
            fprintf(stderr, "\n");
        }
    }
    return 0;
}

int check_overflow(Plan &P) {
    int ov = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&ov, P.overflow, sizeof(int), cudaMemcpyDeviceToHost, P.st));
    MFSEG_CUDA(cudaStreamSynchronize(P.st));
    if (ov) {
        set_error(ov == 1 ? "fixed-point accumulator overflow (|coordinate| too large)"
                          : "internal error in assignment (code " + std::to_string(ov) + ")");
        return 4;
    }
    return 0;
}

}  // namespace
}  // namespace mfseg

using namespace mfseg;

// ====================================================================== C ABI
extern "C" {

const char *mfseg_last_error(void) { return mfseg::g_err.c_str(); }

long long mfseg_launch_count(void) { return mfseg::g_launches.load(); }

void mfseg_timing_enable(int32_t on) {
    mfseg::g_timer = mfseg::PhaseTimer();
    mfseg::g_timer.on = on != 0;
}

int32_t mfseg_timing_read(double *ms_out, int32_t n) {
    for (int i = 0; i < n && i < 8; ++i) ms_out[i] = mfseg::g_timer.ms[i];
    return mfseg::g_timer.passes;
}
int mfseg_abi_version(void) { return MFSEG_ABI_VERSION; }

int mfseg_set_debug_options(int32_t flags, int64_t multi_cap) {
    mfseg::g_dbg.flags = flags;
    mfseg::g_dbg.multi_cap = multi_cap;
    return 0;
}

size_t mfseg_run_workspace_size(const mfseg_params *p, const mfseg_field *f,
                                const mfseg_points *pts) {
    if (check_inputs(p, f, pts)) return 0;
    Plan P;
    memset(&P, 0, sizeof P);
    P.p = *p;
    if (f) P.f = *f;
    if (pts) P.pts = *pts;
    P.NB = p->k[0] * p->k[1] * p->k[2] * p->k[3];
    P.K = p->n_centers > 0 ? p->n_centers : P.NB;
    P.np = pts ? pts->n : 0;
    return plan_carve(P, nullptr, 0);
}

size_t mfseg_assign_workspace_size(const mfseg_params *p, const mfseg_field *f,
                                   const mfseg_points *pts) {
    return mfseg_run_workspace_size(p, f, pts);
}

int mfseg_run(const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts,
              int32_t *point_labels, int32_t *field_labels, mfseg_centers out,
              int32_t *iterations_used_host, int32_t *converged_host, mfseg_progress_fn progress,
              void *progress_user, mfseg_reduce_fn reduce, void *reduce_user, void *workspace,
              size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Plan P;
    MFSEG_TRY(plan_init(P, p, f, pts, workspace, workspace_bytes, st));
    if (P.K != P.NB) {
        set_error("mfseg_run seeds one centre per k-grid cell: n_centers must be 0 or k1*k2*k3*k4");
        return 2;
    }
    if (P.nf == 0 && P.np == 0) {
        set_error("no samples of either kind");
        return 2;
    }
    int K = P.K;
    P.seeds_fast = K == P.NB && seeds_fast_ok(*p);   // centres are the seeds in the initial pass (K == NB)
    MFSEG_CUDA(cudaMemsetAsync(P.overflow, 0, sizeof(int) * 4, st));
    MFSEG_TRY(plan_prepare(P));
    double4 mins = make_double4(p->mins[0], p->mins[1], p->mins[2], p->mins[3]);
    double4 C = make_double4(p->C[0], p->C[1], p->C[2], p->C[3]);
    int4 k = make_int4(p->k[0], p->k[1], p->k[2], p->k[3]);
    unsigned gk = (unsigned)((K + 255) / 256);
    ::mfseg::count_launch();
    k_seed<<<gk, 256, 0, st>>>(K, mins, C, k, P.s[0]);
    MFSEG_LAUNCH("k_seed");
    int cur = 0;
    int iterations = 0, converged = 0;
    bool unpermuted = false;
    alignas(16) char flags_host[64];
    for (int pass = 0; pass <= p->max_iterations; ++pass) {
        bool initial = pass == 0;
        // initial assignment: pure space-time nearest seed (engine.py:346-351)
        double wd = initial ? 1.0 : p->w_d, wp = initial ? 0.0 : p->w_p, wf = initial ? 0.0 : p->w_f;
        // from the second weighted pass on, stable field blocks reuse the last labels
        // the last possible pass writes the point labels in record order itself
        const bool last = pass == p->max_iterations;
        MFSEG_TRY(plan_pass(P, P.s[cur], wd, wp, wf, field_labels, 1, pass >= 2 ? &P.s[cur ^ 1] : nullptr,
                            last ? point_labels : nullptr, initial));
        unpermuted = last;
        if (reduce) {
            long long npairs = (long long)K * MFSEG_ACC_WORDS / 2;
            MFSEG_TRY(launch_to_limbs(npairs, P.acc, P.limbs, st));
            int rc = reduce(reduce_user, (int64_t *)P.limbs, npairs * 3, stream);
            if (rc) {
                set_error("reduce callback failed");
                return 5;
            }
            MFSEG_TRY(launch_from_limbs(npairs, P.limbs, P.acc, st));
        }
        MFSEG_TRY(launch_update(K, P.acc, P.s[cur], P.s[cur ^ 1], p->eps_c, P.flags, st));
        mark(5, st);
        cur ^= 1;
        if (g_timer.on) {
            MFSEG_CUDA(cudaStreamSynchronize(st));
            harvest();
        }
        if (initial) continue;
        MFSEG_CUDA(cudaMemcpyAsync(flags_host, P.flags, update_flags_bytes(),
                                   cudaMemcpyDeviceToHost, st));
        MFSEG_CUDA(cudaStreamSynchronize(st));
        double delta;
        decode_flags(flags_host, &converged, &delta);
        iterations = pass;
        if (progress) progress(progress_user, pass, delta);
        if (converged) break;
    }
    MFSEG_TRY(check_overflow(P));
    if (P.np > 0 && !unpermuted) {   // converged before the last pass
        ::mfseg::count_launch();
        k_unpermute<<<(unsigned)((P.np + 1023) / 1024), 256, 0, st>>>(P.np, P.perm, P.plabels,
                                                                     point_labels);
        MFSEG_LAUNCH("k_unpermute");
    }
    ::mfseg::count_launch();
    k_copy_state<<<gk, 256, 0, st>>>(K, P.s[cur], out);
    MFSEG_LAUNCH("k_copy_state");
    if (iterations_used_host) *iterations_used_host = iterations;
    if (converged_host) *converged_host = converged;
    return 0;
}

int mfseg_assign(const mfseg_params *p, const mfseg_field *f, const mfseg_points *pts,
                 mfseg_centers centers, int32_t *point_labels, int32_t *field_labels,
                 int64_t *acc, void *workspace, size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Plan P;
    MFSEG_TRY(plan_init(P, p, f, pts, workspace, workspace_bytes, st));
    MFSEG_CUDA(cudaMemsetAsync(P.overflow, 0, sizeof(int) * 4, st));
    MFSEG_TRY(plan_prepare(P));
    const int rc = plan_pass(P, centers, p->w_d, p->w_p, p->w_f, field_labels, 1, nullptr, point_labels, 0);
    nvtx_phase(5);   // close the pass's last NVTX range
    MFSEG_TRY(rc);
    if (acc)
        MFSEG_CUDA(cudaMemcpyAsync(acc, P.acc, sizeof(int64_t) * P.K * MFSEG_ACC_WORDS,
                                   cudaMemcpyDeviceToDevice, st));
    return check_overflow(P);
}

int mfseg_accumulate(int32_t K, const mfseg_field *f, const mfseg_points *pts,
                     const int32_t *point_labels, const int32_t *field_labels, int64_t *acc,
                     void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int *ovf = nullptr, *ovf_h = nullptr;
    MFSEG_TRY(tiny_scratch((void **)&ovf, (void **)&ovf_h));
    MFSEG_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), st));
    MFSEG_CUDA(cudaMemsetAsync(acc, 0, sizeof(int64_t) * K * MFSEG_ACC_WORDS, st));
    if (pts && pts->n > 0)
        MFSEG_TRY(launch_accumulate_points(pts, point_labels, (unsigned long long *)acc, ovf, st));
    if (f && f->nt > 0) {
        long long n = (long long)f->nx * f->ny * f->nz * f->nt;
        MFSEG_TRY(launch_accumulate_field(n, f, field_labels, (unsigned long long *)acc, ovf, st));
    }
    MFSEG_CUDA(cudaMemcpyAsync(ovf_h, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (*ovf_h) {
        set_error("fixed-point accumulator overflow");
        return 4;
    }
    return 0;
}

int mfseg_acc_to_double(int32_t K, const int64_t *acc, double *sums, double *psum, double *fsum,
                        int64_t *n_p, int64_t *n_f, void *stream) {
    return launch_acc_to_double(K, (const unsigned long long *)acc, sums, psum, fsum,
                                (long long *)n_p, (long long *)n_f, (cudaStream_t)stream);
}

int mfseg_update_centers(int32_t K, const int64_t *acc, mfseg_centers old_state,
                         mfseg_centers new_state, double eps_c, int32_t *conv_host,
                         double *delta_host, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    void *flags = nullptr, *h = nullptr;
    MFSEG_TRY(tiny_scratch(&flags, &h));
    MFSEG_TRY(launch_update(K, (const unsigned long long *)acc, old_state, new_state, eps_c,
                            flags, st));
    MFSEG_CUDA(cudaMemcpyAsync(h, flags, update_flags_bytes(), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    int conv;
    double delta;
    decode_flags(h, &conv, &delta);
    if (conv_host) *conv_host = conv;
    if (delta_host) *delta_host = delta;
    return 0;
}

int mfseg_minmax_normalize(double *values, int64_t n, int32_t apply, double *lo_host,
                           double *hi_host, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        set_error("minmax of an empty array");
        return 2;
    }
    unsigned long long *mm = nullptr, *h = nullptr;
    MFSEG_TRY(tiny_scratch((void **)&mm, (void **)&h));
    const unsigned long long init[3] = {~0ull, 0ull, 0ull};
    MFSEG_CUDA(cudaMemcpyAsync(mm, init, 24, cudaMemcpyHostToDevice, st));
    ::mfseg::count_launch();
    k_minmax<<<148 * 4, 256, 0, st>>>(values, n, mm);
    MFSEG_LAUNCH("k_minmax");
    MFSEG_CUDA(cudaMemcpyAsync(h, mm, 24, cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (h[2]) {   // samples are finite
        set_error("non-finite (NaN or inf) sample value");
        return 2;
    }
    double lo = unkey(h[0]), hi = unkey(h[1]);
    if (lo_host) *lo_host = lo;
    if (hi_host) *hi_host = hi;
    if (apply) {
        // (v - lo) / (hi - lo); degenerate range maps to 0 (ingest.py:312-318)
        volatile double span = hi - lo;
        ::mfseg::count_launch();
        k_normalize<<<148 * 8, 256, 0, st>>>(values, n, lo, span, hi == lo);
        MFSEG_LAUNCH("k_normalize");
    }
    return 0;
}

int mfseg_normalize_range(double *values, int64_t n, double lo, double hi, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) return 0;
    volatile double span = hi - lo;
    ::mfseg::count_launch();
    k_normalize<<<148 * 8, 256, 0, st>>>(values, n, lo, span, hi == lo);
    MFSEG_LAUNCH("k_normalize");
    return 0;
}

int mfseg_acc_to_limbs(const int64_t *acc, int64_t n_pairs, int64_t *limbs, void *stream) {
    return launch_to_limbs(n_pairs, (const unsigned long long *)acc, (long long *)limbs,
                           (cudaStream_t)stream);
}

int mfseg_limbs_to_acc(const int64_t *limbs, int64_t n_pairs, int64_t *acc, void *stream) {
    return launch_from_limbs(n_pairs, (const long long *)limbs, (unsigned long long *)acc,
                             (cudaStream_t)stream);
}

}  // extern "C"
