// Stranded-sample fallback, crowded-tile (deferred) path and accumulate for
// given labels.
//
// Reference: engine._assign_chunk / _metric / _fallback_assign / accumulate
// (engine.py:137-263).  For every sample the label is
//     argmin_(D, id) { D(s, c) : c in cand(bin(s)), |c - s| <= C per axis }
// with D computed in the reference's fp64 operation order; if the set is empty
// the sample is "stranded" and takes the doubling-window fallback over all K
// centres (k_fallback).  The tiled fast paths live in assign_field5.cu /
// assign_field5b.cu (fields) and assign_point4.cu (points); samples of tiles
// too crowded for them come here (k_deferred, one warp per sample).
//
// Accumulation here is per sample: fixed point + integer atomics, exact and
// order-free, so it agrees bit for bit with the tiled kernels' sums.
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace mfseg {

namespace {
constexpr double INF = __builtin_huge_val();
// word offsets inside one cluster's MFSEG_ACC_WORDS accumulator
constexpr int ACC_X = 0, ACC_PV = 8, ACC_FV = 10, ACC_NP = 12, ACC_NF = 13;
}  // namespace

// ====================================================================== fallback
// Stranded samples: doubling box over ALL centres (engine.py:195-205).  One
// warp per sample; (D, id) lexicographic minimum = numpy's first minimum over
// ascending ids.  Also accumulates the sample (per-sample fixed point).


__device__ void fallback_one(const FallbackArgs &a, long long idx) {
    const int lane = threadIdx.x & 31;
    double s0, s1, s2, s3, v;
    if (a.kind == 1) {
        long long r = idx;
        int i = (int)(r % a.nx);
        r /= a.nx;
        int j = (int)(r % a.ny);
        r /= a.ny;
        int k = (int)(r % a.nz);
        int m = (int)(r / a.nz);
        s0 = cell_coord(a.ox, a.sx, a.x0 + i);
        s1 = cell_coord(a.oy, a.sy, a.y0 + j);
        s2 = cell_coord(a.oz, a.sz, a.z0 + k);
        s3 = a.times[m];
        v = a.values[idx];
    } else {
        s0 = a.px[idx];
        s1 = a.py[idx];
        s2 = a.pz[idx];
        s3 = a.pt[idx];
        v = a.pv[idx];
    }
    // Level `mult`: the centres with |c - s| <= mult * C on every axis
    // (engine.py:199-205).  Their bins lie within (mult + 2) bins of the sample's
    // own unclipped bin coordinate on each axis (the +2 covers the rounding of
    // the bin arithmetic; bins are clipped like CenterGrid's, so centres outside
    // the extent sit in the edge bins and stay covered), so while that bin box is
    // small the level scans its bins' centres; otherwise all K.  Either way the
    // exact box test selects the same set, and the (D, id) minimum is unique.
    const double sc[4] = {s0, s1, s2, s3};
    double mult = 2.0;
    int best = INT_MAX;
    for (int guard = 0; guard < 1100 && best == INT_MAX; ++guard, mult = DMUL(mult, 2.0)) {
        double b0 = DMUL(mult, a.C[0]), b1 = DMUL(mult, a.C[1]), b2 = DMUL(mult, a.C[2]),
               b3 = DMUL(mult, a.C[3]);
        double bD = INF;
        int bI = INT_MAX;
        auto consider = [&](int c) {
            double dx = DSUB(a.c.x[c], s0), dy = DSUB(a.c.y[c], s1), dz = DSUB(a.c.z[c], s2),
                   dt = DSUB(a.c.t[c], s3);
            if (fabs(dx) <= b0 && fabs(dy) <= b1 && fabs(dz) <= b2 && fabs(dt) <= b3) {
                double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
                double ct = DMUL(a.cf, dt);
                bool h = a.chas[c] != 0;
                double D = metric_tail(qq, DMUL(ct, ct), v, h ? a.cval[c] : 0.0, h, a.wv, a.wd);
                if (better(D, c, bD, bI)) {
                    bD = D;
                    bI = c;
                }
            }
        };
        int lo[4], ext[4];
        long long nbins = 1;
        const int reach = mult < 1e6 ? (int)mult + 2 : (1 << 28);
        for (int d = 0; d < 4; ++d) {
            const double u = floor(DDIV(DSUB(sc[d], a.mins[d]), a.C[d]));
            const double l = fmax(fmin(u - reach, (double)(a.k[d] - 1)), 0.0);
            const double h = fmax(fmin(u + reach, (double)(a.k[d] - 1)), 0.0);
            lo[d] = (int)l;
            ext[d] = (int)h - (int)l + 1;
            nbins *= ext[d];
        }
        if (a.bin_start && nbins * 4 < a.K) {
            for (long long q = 0; q < nbins; ++q) {
                long long r = q;
                const int bx = lo[0] + (int)(r % ext[0]);
                r /= ext[0];
                const int by = lo[1] + (int)(r % ext[1]);
                r /= ext[1];
                const int bz = lo[2] + (int)(r % ext[2]);
                const int bt = lo[3] + (int)(r / ext[2]);
                const int b = ((bt * a.k[2] + bz) * a.k[1] + by) * a.k[0] + bx;
                const int e = a.bin_start[b + 1];
                for (int p = a.bin_start[b] + lane; p < e; p += 32) consider(a.bin_ids[p]);
            }
        } else {
            for (int c = lane; c < a.K; c += 32) consider(c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double oD = __shfl_xor_sync(0xffffffffu, bD, o);
            int oI = __shfl_xor_sync(0xffffffffu, bI, o);
            if (better(oD, oI, bD, bI)) {
                bD = oD;
                bI = oI;
            }
        }
        best = bI;
    }
    if (lane == 0) {
        a.labels[idx] = best == INT_MAX ? -1 : best;
        if (a.kind == 0 && a.labels_out) a.labels_out[a.perm[idx]] = best == INT_MAX ? -1 : best;
        if (best == INT_MAX) {
            *a.overflow = 3;
            return;
        }
        if (a.accumulate) {
            unsigned long long *p = a.acc + (size_t)best * MFSEG_ACC_WORDS;
            atomic_add_double_fix(p + ACC_X + 0, s0, a.overflow);
            atomic_add_double_fix(p + ACC_X + 2, s1, a.overflow);
            atomic_add_double_fix(p + ACC_X + 4, s2, a.overflow);
            atomic_add_double_fix(p + ACC_X + 6, s3, a.overflow);
            atomic_add_double_fix(p + (a.kind == 1 ? ACC_FV : ACC_PV), v, a.overflow);
            atomicAdd(p + (a.kind == 1 ? ACC_NF : ACC_NP), 1ull);
        }
    }
}

__global__ void k_fallback(FallbackArgs a) {
    const long long n = (long long)*a.n_stranded;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n <= a.cap) {
        for (long long q = wid; q < n; q += warps) fallback_one(a, a.stranded[q]);
    } else {
        // list overflowed: rescan all labels for -1 (still deterministic)
        for (long long q = wid; q < a.n_samples; q += warps)
            if (a.labels[q] < 0) fallback_one(a, q);
    }
}

// ====================================================================== deferred samples
// Samples of tiles whose candidate set is too crowded for the fast path
// (labels -2).  One warp per sample: the reference's windowed predicate
// (candidates of the sample's bin, exact box test, fp64 D, lowest id on ties),
// then per-sample fixed-point accumulation; samples without a valid candidate
// go to the stranded list for k_fallback.
struct DeferredGeo {
    Grid g;
    const int *tbin;
    int4 k;
    double mins[4];
    const long long *list;
    const unsigned long long *count;
    long long cap;
    long long batch_min;   // list length from which samples go one per lane
};

// the deferred sample's coordinates, value and sample bin
__device__ __forceinline__ int deferred_sample(const FallbackArgs &a, const DeferredGeo &G, long long idx,
                                               double &s0, double &s1, double &s2, double &s3, double &v) {
    int bt;
    if (a.kind == 1) {
        long long r = idx;
        const int i = (int)(r % a.nx);
        r /= a.nx;
        const int j = (int)(r % a.ny);
        r /= a.ny;
        const int k = (int)(r % a.nz);
        const int m = (int)(r / a.nz);
        s0 = cell_coord(a.ox, a.sx, a.x0 + i);
        s1 = cell_coord(a.oy, a.sy, a.y0 + j);
        s2 = cell_coord(a.oz, a.sz, a.z0 + k);
        s3 = a.times[m];
        v = a.values[idx];
        bt = G.tbin[m];
    } else {
        s0 = a.px[idx];
        s1 = a.py[idx];
        s2 = a.pz[idx];
        s3 = a.pt[idx];
        v = a.pv[idx];
        bt = bin_coord(s3, G.mins[3], a.C[3], G.k.w);
    }
    const int bx = bin_coord(s0, G.mins[0], a.C[0], G.k.x);
    const int by = bin_coord(s1, G.mins[1], a.C[1], G.k.y);
    const int bz = bin_coord(s2, G.mins[2], a.C[2], G.k.z);
    return ((bt * G.k.z + bz) * G.k.y + by) * G.k.x + bx;
}

// the windowed predicate for one (sample, candidate) pair: (D, id) minimum update
__device__ __forceinline__ void deferred_pair(const FallbackArgs &a, int c, double s0, double s1, double s2,
                                              double s3, double v, double &bD, int &bI) {
    const double dx = DSUB(a.c.x[c], s0), dy = DSUB(a.c.y[c], s1), dz = DSUB(a.c.z[c], s2),
                 dt = DSUB(a.c.t[c], s3);
    if (!(fabs(dx) <= a.C[0] && fabs(dy) <= a.C[1] && fabs(dz) <= a.C[2] && fabs(dt) <= a.C[3]))
        return;
    const double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    const double ct = DMUL(a.cf, dt);
    const bool h = a.chas[c] != 0;
    const double D = metric_tail(qq, DMUL(ct, ct), v, h ? a.cval[c] : 0.0, h, a.wv, a.wd);
    if (better(D, c, bD, bI)) {
        bD = D;
        bI = c;
    }
}

// label, stranded list or per-sample fixed-point sums of one resolved sample
__device__ __forceinline__ void deferred_finish(const FallbackArgs &a, long long idx, int bI, double s0,
                                                double s1, double s2, double s3, double v) {
    if (bI == INT_MAX) {   // stranded: the fallback kernel runs next
        a.labels[idx] = -1;
        if (a.kind == 0 && a.labels_out) a.labels_out[a.perm[idx]] = -1;
        const unsigned long long q = atomicAdd((unsigned long long *)a.n_stranded, 1ull);
        if ((long long)q < a.cap) ((long long *)a.stranded)[q] = idx;
        return;
    }
    a.labels[idx] = bI;
    if (a.kind == 0 && a.labels_out) a.labels_out[a.perm[idx]] = bI;
    if (a.accumulate) {
        unsigned long long *p = a.acc + (size_t)bI * MFSEG_ACC_WORDS;
        atomic_add_double_fix(p + ACC_X + 0, s0, a.overflow);
        atomic_add_double_fix(p + ACC_X + 2, s1, a.overflow);
        atomic_add_double_fix(p + ACC_X + 4, s2, a.overflow);
        atomic_add_double_fix(p + ACC_X + 6, s3, a.overflow);
        atomic_add_double_fix(p + (a.kind == 1 ? ACC_FV : ACC_PV), v, a.overflow);
        atomicAdd(p + (a.kind == 1 ? ACC_NF : ACC_NP), 1ull);
    }
}

// one sample, the warp's lanes over its candidates
__device__ void deferred_one(const FallbackArgs &a, const DeferredGeo &G, long long idx) {
    const int lane = threadIdx.x & 31;
    double s0, s1, s2, s3, v;
    const int sbin = deferred_sample(a, G, idx, s0, s1, s2, s3, v);
    double bD = INF;
    int bI = INT_MAX;
    for (int p = G.g.cand_start[sbin] + lane; p < G.g.cand_start[sbin + 1]; p += 32)
        deferred_pair(a, G.g.cand_ids[p], s0, s1, s2, s3, v, bD, bI);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oD = __shfl_xor_sync(0xffffffffu, bD, o);
        const int oI = __shfl_xor_sync(0xffffffffu, bI, o);
        if (better(oD, oI, bD, bI)) {
            bD = oD;
            bI = oI;
        }
    }
    if (lane == 0) deferred_finish(a, idx, bI, s0, s1, s2, s3, v);
}

// 32 consecutive list entries, one per lane: when they share a sample bin (the
// lists are written brick by brick) every lane scans the bin's candidates for
// its own sample (the candidate loads are warp broadcasts); otherwise one
// sample at a time
__device__ void deferred_batch(const FallbackArgs &a, const DeferredGeo &G, long long q0, long long n) {
    const int lane = threadIdx.x & 31;
    const long long q = q0 + lane;
    const bool valid = q < n;
    const long long idx = valid ? G.list[q] : G.list[q0];
    double s0, s1, s2, s3, v;
    const int sbin = deferred_sample(a, G, idx, s0, s1, s2, s3, v);
    const int sb0 = __shfl_sync(0xffffffffu, sbin, 0);
    if (!__all_sync(0xffffffffu, sbin == sb0)) {
        const int m = (int)min(32ll, n - q0);
        for (int j = 0; j < m; ++j) deferred_one(a, G, __shfl_sync(0xffffffffu, idx, j));
        return;
    }
    double bD = INF;
    int bI = INT_MAX;
    const int p1 = G.g.cand_start[sb0 + 1];
    int p = G.g.cand_start[sb0];
    for (; p + 4 <= p1; p += 4) {   // four candidates' state in flight
        int c[4];
        double cx[4], cy[4], cz[4], ct[4], cv[4];
        bool ch[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = G.g.cand_ids[p + u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            cx[u] = a.c.x[c[u]];
            cy[u] = a.c.y[c[u]];
            cz[u] = a.c.z[c[u]];
            ct[u] = a.c.t[c[u]];
            ch[u] = a.chas[c[u]] != 0;
            cv[u] = a.cval[c[u]];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double dx = DSUB(cx[u], s0), dy = DSUB(cy[u], s1), dz = DSUB(cz[u], s2), dt = DSUB(ct[u], s3);
            if (!(fabs(dx) <= a.C[0] && fabs(dy) <= a.C[1] && fabs(dz) <= a.C[2] && fabs(dt) <= a.C[3]))
                continue;
            const double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
            const double tt = DMUL(a.cf, dt);
            const double D = metric_tail(qq, DMUL(tt, tt), v, ch[u] ? cv[u] : 0.0, ch[u], a.wv, a.wd);
            if (better(D, c[u], bD, bI)) {
                bD = D;
                bI = c[u];
            }
        }
    }
    for (; p < p1; ++p) deferred_pair(a, G.g.cand_ids[p], s0, s1, s2, s3, v, bD, bI);
    if (valid) deferred_finish(a, idx, bI, s0, s1, s2, s3, v);
}

__global__ void k_deferred(FallbackArgs a, DeferredGeo G) {
    const long long n = (long long)*G.count;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n <= G.cap && n >= G.batch_min) {   // many samples: one per lane
        for (long long q = 32 * wid; q < n; q += 32 * warps) deferred_batch(a, G, q, n);
    } else if (n <= G.cap) {               // few: the warp's lanes over each sample's candidates
        for (long long q = wid; q < n; q += warps) deferred_one(a, G, G.list[q]);
    } else {
        for (long long q = wid; q < a.n_samples; q += warps)
            if (a.labels[q] == -2) deferred_one(a, G, q);
    }
}

// ====================================================================== accumulate (given labels)
// accumulate (engine.py:244-263) for caller-supplied labels: per-sample fixed
// point + integer atomics, exact and order-free.
__global__ void k_accumulate_field(long long n, int nx, int ny, int nz, double ox, double oy,
                                   double oz, double sx, double sy, double sz, int x0, int y0,
                                   int z0, const double *times, const double *values, const int *labels,
                                   unsigned long long *acc, int *overflow) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        long long r = q;
        int i = (int)(r % nx);
        r /= nx;
        int j = (int)(r % ny);
        r /= ny;
        int k = (int)(r % nz);
        int m = (int)(r / nz);
        unsigned long long *p = acc + (size_t)labels[q] * MFSEG_ACC_WORDS;
        atomic_add_double_fix(p + ACC_X + 0, cell_coord(ox, sx, (long long)x0 + i), overflow);
        atomic_add_double_fix(p + ACC_X + 2, cell_coord(oy, sy, (long long)y0 + j), overflow);
        atomic_add_double_fix(p + ACC_X + 4, cell_coord(oz, sz, (long long)z0 + k), overflow);
        atomic_add_double_fix(p + ACC_X + 6, times[m], overflow);
        atomic_add_double_fix(p + ACC_FV, values[q], overflow);
        atomicAdd(p + ACC_NF, 1ull);
    }
}

__global__ void k_accumulate_points(long long n, const double *xyz, const double *t,
                                    const double *value, const int *labels,
                                    unsigned long long *acc, int *overflow) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        unsigned long long *p = acc + (size_t)labels[q] * MFSEG_ACC_WORDS;
        atomic_add_double_fix(p + ACC_X + 0, xyz[3 * q], overflow);
        atomic_add_double_fix(p + ACC_X + 2, xyz[3 * q + 1], overflow);
        atomic_add_double_fix(p + ACC_X + 4, xyz[3 * q + 2], overflow);
        atomic_add_double_fix(p + ACC_X + 6, t[q], overflow);
        atomic_add_double_fix(p + ACC_PV, value[q], overflow);
        atomicAdd(p + ACC_NP, 1ull);
    }
}

// ---------------------------------------------------------------------- launchers
int field_tile_dims(int *tx, int *ty, int *tz) {   // the field kernel's sample-bin block
    *tx = 16;
    *ty = 16;
    *tz = 16;
    return 0;
}
int point_tile_size() { return POINT_CHUNK; }

int launch_field_assign_v5(const FieldArgs &a, cudaStream_t st);
int launch_point_assign_v4(const PointArgs &a, long long max_tiles, cudaStream_t st);

int launch_field_assign(const FieldArgs &a, long long, cudaStream_t st) {
    return launch_field_assign_v5(a, st);
}

int launch_point_assign(const PointArgs &a, long long max_tiles, cudaStream_t st) {
    return launch_point_assign_v4(a, max_tiles, st);
}

int launch_deferred(const FallbackArgs &a, const Grid &g, const int *tbin, const int4 &k,
                    const double *mins, const long long *list, const unsigned long long *count,
                    long long cap, cudaStream_t st) {
    DeferredGeo G;
    G.g = g;
    G.tbin = tbin;
    G.k = k;
    for (int d = 0; d < 4; ++d) G.mins[d] = mins[d];
    G.list = list;
    G.count = count;
    G.cap = cap;
    constexpr int blocks = 148 * 4, threads = 256;
#ifndef MFSEG_DEFERRED_BATCH_MUL
#define MFSEG_DEFERRED_BATCH_MUL 1   // x 32 lanes: from one batch per warp
#endif
    G.batch_min = (debug_options().flags & MFSEG_DEBUG_DEFERRED_BATCH)
                      ? 0 : (long long)MFSEG_DEFERRED_BATCH_MUL * blocks * (threads / 32);
    ::mfseg::count_launch();
    k_deferred<<<blocks, threads, 0, st>>>(a, G);
    MFSEG_LAUNCH("k_deferred");
    return 0;
}

int launch_fallback(const FallbackArgs &a, cudaStream_t st) {
    ::mfseg::count_launch();
    k_fallback<<<148 * 4, 256, 0, st>>>(a);
    MFSEG_LAUNCH("k_fallback");
    return 0;
}

int launch_accumulate_field(long long n, const mfseg_field *f, const int *labels,
                            unsigned long long *acc, int *overflow, cudaStream_t st) {
    if (n <= 0) return 0;
    ::mfseg::count_launch();
    k_accumulate_field<<<148 * 8, 256, 0, st>>>(n, f->nx, f->ny, f->nz, f->origin[0],
                                                f->origin[1], f->origin[2], f->spacing[0],
                                                f->spacing[1], f->spacing[2], f->offset[0],
                                                f->offset[1], f->offset[2], f->times,
                                                f->values, labels, acc, overflow);
    MFSEG_LAUNCH("k_accumulate_field");
    return 0;
}

int launch_accumulate_points(const mfseg_points *p, const int *labels, unsigned long long *acc,
                             int *overflow, cudaStream_t st) {
    if (p->n <= 0) return 0;
    ::mfseg::count_launch();
    k_accumulate_points<<<148 * 8, 256, 0, st>>>(p->n, p->xyz, p->t, p->value, labels, acc,
                                                 overflow);
    MFSEG_LAUNCH("k_accumulate_points");
    return 0;
}

}  // namespace mfseg
