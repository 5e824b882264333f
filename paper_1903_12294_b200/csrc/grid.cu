// CenterGrid rebuild (engine.py:89-134), once per pass, all on the device.
//
//  cbin / bin CSR   centre -> clip(floor((loc - min)/C), 0, k-1) flat bin,
//                   ascending ids within a bin (engine.py:102-108)
//  cand CSR         per SAMPLE bin b: every centre whose bin is one of the
//                   in-range 3^4 neighbours of b (engine.py:119-131).  A
//                   sample in bin b therefore satisfies the neighbour-bin
//                   condition for exactly the centres of b's list.
//  vbox             per centre and field axis, the index interval of field
//                   samples that pass the box test |c - s| <= C
//                   (engine.py:179-181).  fl(c - x_i) is monotone in i, so the
//                   passing set is an interval, found by exact binary search.
#include "kernels.cuh"

namespace mfseg {

namespace {

__global__ void k_center_bins(int K, const double *x, const double *y, const double *z,
                              const double *t, double4 mins, double4 C, int4 k, int *cbin,
                              int *bin_count) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    int bx = bin_coord(x[c], mins.x, C.x, k.x);
    int by = bin_coord(y[c], mins.y, C.y, k.y);
    int bz = bin_coord(z[c], mins.z, C.z, k.z);
    int bt = bin_coord(t[c], mins.w, C.w, k.w);
    int f = ((bt * k.z + bz) * k.y + by) * k.x + bx;
    cbin[c] = f;
    atomicAdd(&bin_count[f], 1);
}

// first index i in [0, n) with fl(c - x_i) <= C  (n if none)
__device__ int first_le(double c, double C, double o, double s, int off, int n) {
    int a = 0, b = n;
    while (a < b) {
        int mid = (a + b) >> 1;
        if (DSUB(c, cell_coord(o, s, (long long)off + mid)) <= C) b = mid; else a = mid + 1;
    }
    return a;
}
// last index i with fl(c - x_i) >= -C  (-1 if none)
__device__ int last_ge(double c, double C, double o, double s, int off, int n) {
    int a = 0, b = n;   // first i with fl(c - x_i) < -C
    while (a < b) {
        int mid = (a + b) >> 1;
        if (DSUB(c, cell_coord(o, s, (long long)off + mid)) < -C) b = mid; else a = mid + 1;
    }
    return a - 1;
}
__device__ int first_le_t(double c, double C, const double *tt, int n) {
    int a = 0, b = n;
    while (a < b) {
        int mid = (a + b) >> 1;
        if (DSUB(c, tt[mid]) <= C) b = mid; else a = mid + 1;
    }
    return a;
}
__device__ int last_ge_t(double c, double C, const double *tt, int n) {
    int a = 0, b = n;
    while (a < b) {
        int mid = (a + b) >> 1;
        if (DSUB(c, tt[mid]) < -C) b = mid; else a = mid + 1;
    }
    return a - 1;
}

struct FieldGeom {
    int nx, ny, nz, nt;
    double ox, oy, oz, sx, sy, sz;
    int x0, y0, z0;   // global index of the first cell (spatial slabs); vbox is local
    const double *times;
};

__global__ void k_center_vbox(int K, const double *x, const double *y, const double *z,
                              const double *t, double4 C, FieldGeom fg, int4 *vbox) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    int4 a, b;
    a.x = first_le(x[c], C.x, fg.ox, fg.sx, fg.x0, fg.nx);
    a.y = last_ge(x[c], C.x, fg.ox, fg.sx, fg.x0, fg.nx);
    a.z = first_le(y[c], C.y, fg.oy, fg.sy, fg.y0, fg.ny);
    a.w = last_ge(y[c], C.y, fg.oy, fg.sy, fg.y0, fg.ny);
    b.x = first_le(z[c], C.z, fg.oz, fg.sz, fg.z0, fg.nz);
    b.y = last_ge(z[c], C.z, fg.oz, fg.sz, fg.z0, fg.nz);
    b.z = first_le_t(t[c], C.w, fg.times, fg.nt);
    b.w = last_ge_t(t[c], C.w, fg.times, fg.nt);
    vbox[2 * c] = a;
    vbox[2 * c + 1] = b;
}

__global__ void k_center_place(int K, const int *cbin, const int *bin_start, int *cursor,
                               int *bin_ids) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    int b = cbin[c];
    int p = atomicAdd(&cursor[b], 1);
    bin_ids[bin_start[b] + p] = c;
}

// make every bin's id list ascending (lists hold ~1 centre; insertion sort)
__global__ void k_bin_sort(int nbins, const int *bin_start, int *bin_ids) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbins) return;
    int s = bin_start[b], e = bin_start[b + 1];
    for (int i = s + 1; i < e; ++i) {
        int v = bin_ids[i], j = i - 1;
        while (j >= s && bin_ids[j] > v) {
            bin_ids[j + 1] = bin_ids[j];
            --j;
        }
        bin_ids[j + 1] = v;
    }
}

__device__ __forceinline__ void unflat(int b, int4 k, int &bx, int &by, int &bz, int &bt) {
    bx = b % k.x;
    b /= k.x;
    by = b % k.y;
    b /= k.y;
    bz = b % k.z;
    bt = b / k.z;
}

// One warp per bin: lane r < 27 takes neighbour row r = (dt, dz, dy) in the
// reference's loop order (dt outer, dy inner); a row is the x-run of bins
// [bx - 1, bx + 1], contiguous in bin_ids.  Returns the row's (start, length).
__device__ __forceinline__ int2 cand_row(long long b, int4 k, const int *bin_start, int lane) {
    int bx, by, bz, bt;
    unflat((int)b, k, bx, by, bz, bt);
    int2 r = make_int2(0, 0);
    if (lane < 27) {
        const int qt = bt + lane / 9 - 1, qz = bz + (lane / 3) % 3 - 1, qy = by + lane % 3 - 1;
        if (qt >= 0 && qt < k.w && qz >= 0 && qz < k.z && qy >= 0 && qy < k.y) {
            const int row = ((qt * k.z + qz) * k.y + qy) * k.x;
            const int lo = max(bx - 1, 0), hi = min(bx + 1, k.x - 1);
            r.x = bin_start[row + lo];
            r.y = bin_start[row + hi + 1] - r.x;
        }
    }
    return r;
}

__global__ void k_cand_count(int nbins, int4 k, const int *bin_start, int *cand_count) {
    const int lane = threadIdx.x & 31;
    const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (b >= nbins) return;   // warp-uniform
    const int n = __reduce_add_sync(0xffffffffu, (unsigned)cand_row(b, k, bin_start, lane).y);
    if (lane == 0) cand_count[b] = n;
}

__global__ void k_cand_fill(int nbins, int4 k, const int *bin_start, const int *bin_ids,
                            const int *cand_start, int *cand_ids) {
    const int lane = threadIdx.x & 31;
    const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (b >= nbins) return;   // warp-uniform
    const int2 r = cand_row(b, k, bin_start, lane);
    int incl = r.y;   // rows' output offsets: exclusive prefix over the lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int o = cand_start[b] + incl - r.y;
    for (int i = 0; i < r.y; ++i) cand_ids[o + i] = bin_ids[r.x + i];
}

}  // namespace

size_t grid_workspace_bytes(int K, int NB) {
    Carver cv;
    int *ct;
    void *sc;
    grid_carve(cv, K, NB, &ct, &sc);
    return cv.off + 256;
}

// K centres, NB = k1*k2*k3*k4 bins (the reference allows K != NB for a
// caller-built CenterState, e.g. test_engine.py:250-262).
Grid grid_carve(Carver &cv, int K, int NB, int **count_tmp, void **scan_tmp) {
    Grid g;
    g.K = K;
    g.NB = NB;
    g.cbin = cv.take<int>(K);
    g.bin_start = cv.take<int>(NB + 1);
    g.bin_ids = cv.take<int>(K);
    g.cand_start = cv.take<int>(NB + 1);
    g.cand_ids = cv.take<int>(81ll * K);     // each centre is in <= 81 neighbour lists
    g.vbox = cv.take<int4>(2ll * K);
    *count_tmp = cv.take<int>(NB + 1);
    *scan_tmp = cv.take<char>(scan_tmp_bytes(NB + 1));
    return g;
}

// Rebuild the grid for centre locations x/y/z/t (planes of length K).
int grid_build(Grid &g, const double *x, const double *y, const double *z, const double *t,
               const mfseg_params *p, const mfseg_field *f, int *count_tmp, void *scan_tmp,
               cudaStream_t st) {
    int K = g.K, NB = g.NB;
    double4 mins = make_double4(p->mins[0], p->mins[1], p->mins[2], p->mins[3]);
    double4 C = make_double4(p->C[0], p->C[1], p->C[2], p->C[3]);
    int4 k = make_int4(p->k[0], p->k[1], p->k[2], p->k[3]);
    const int B = 256;
    unsigned gk = (unsigned)((K + B - 1) / B), gb = (unsigned)((NB + B - 1) / B);
    size_t sb = scan_tmp_bytes(NB + 1);
    MFSEG_CUDA(cudaMemsetAsync(count_tmp, 0, sizeof(int) * (NB + 1), st));
    if (K > 0) {
        ::mfseg::count_launch();
        k_center_bins<<<gk, B, 0, st>>>(K, x, y, z, t, mins, C, k, g.cbin, count_tmp);
    }
    MFSEG_TRY(scan_exclusive_i32(count_tmp, g.bin_start, NB + 1, scan_tmp, sb, st));
    MFSEG_CUDA(cudaMemsetAsync(count_tmp, 0, sizeof(int) * (NB + 1), st));
    if (K > 0) {
        ::mfseg::count_launch();
        k_center_place<<<gk, B, 0, st>>>(K, g.cbin, g.bin_start, count_tmp, g.bin_ids);
    }
    ::mfseg::count_launch();
    k_bin_sort<<<gb, B, 0, st>>>(NB, g.bin_start, g.bin_ids);
    const unsigned gw = (unsigned)((32ll * NB + B - 1) / B);   // one warp per bin
    ::mfseg::count_launch();
    k_cand_count<<<gw, B, 0, st>>>(NB, k, g.bin_start, count_tmp);
    MFSEG_TRY(scan_exclusive_i32(count_tmp, g.cand_start, NB + 1, scan_tmp, sb, st));
    ::mfseg::count_launch();
    k_cand_fill<<<gw, B, 0, st>>>(NB, k, g.bin_start, g.bin_ids, g.cand_start, g.cand_ids);
    if (f && f->nt > 0 && K > 0) {
        FieldGeom fg{f->nx, f->ny, f->nz, f->nt, f->origin[0], f->origin[1], f->origin[2],
                     f->spacing[0], f->spacing[1], f->spacing[2], f->offset[0], f->offset[1],
                     f->offset[2], f->times};
        ::mfseg::count_launch();
        k_center_vbox<<<gk, B, 0, st>>>(K, x, y, z, t, C, fg, g.vbox);
    }
    MFSEG_LAUNCH("grid_build");
    return 0;
}

}  // namespace mfseg
