// Feature materialisation after segmentation (postproc.py:20-227) and the
// particle->cell link index (ingest.py:261-280).
//
//   mfseg_merge          union-find over the live centre table, smallest-id
//                        root (postproc.py:20-79); merged rows summed in the
//                        reference's order: numpy `sum` of loc*n (sequential)
//                        and CPython 3.12 `sum` of floats (Neumaier) for
//                        p_c / f_c (postproc.py:82-92)
//   mfseg_relabel        merge_map[label] gather (postproc.py:155,164)
//   mfseg_voxel_csr      per (timestep, feature) ascending cell lists
//                        (postproc.py:162-168) via a stable radix sort
//   mfseg_feature_stats  bbox / mean / population std / counts
//                        (postproc.py:194-227), exact fixed-point sums
//   mfseg_link_index     stable (cell, interval) bucketing (ingest.py:261-280)
#include <climits>
#include <cstring>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double DELTA = 1e-12;   // model.py:16

__device__ __forceinline__ bool values_match(double a, double b, double eps) {
    bool na = isnan(a), nb = isnan(b);
    if (na && nb) return true;    // both lack the kind
    if (na || nb) return false;   // one-sided absence never merges
    // pct = fl(r / s) <= eps with r, s computed exactly as the reference; the
    // division is only needed near the threshold: r < eps s (1 - 2^-50) implies
    // fl(r / s) <= eps, r > eps s (1 + 2^-50) implies fl(r / s) > eps
    const double r = DMUL(2.0, fabs(DSUB(a, b))), s = DADD(DADD(fabs(a), fabs(b)), DELTA);
    const double es = eps * s;
    if (r < es * (1.0 - 0x1.0p-50)) return true;
    if (r > es * (1.0 + 0x1.0p-50)) return false;
    return DDIV(r, s) <= eps;
}

__device__ int uf_find(int *parent, int a) {
    // path halving: every visited node is re-pointed to its grandparent (benign
    // races: parents only ever move to smaller rows of the same component)
    int p = ((volatile int *)parent)[a];
    while (p != a) {
        const int gp = ((volatile int *)parent)[p];
        if (gp != p) atomicMin(&parent[a], gp);
        a = p;
        p = gp;
    }
    return a;
}

// hook the larger root under the smaller one: the final root of every
// component is its smallest row (= smallest id, rows are id-ascending)
__device__ void uf_union(int *parent, int a, int b) {
    while (true) {
        a = uf_find(parent, a);
        b = uf_find(parent, b);
        if (a == b) return;
        if (a > b) {
            int t = a;
            a = b;
            b = t;
        }
        int old = atomicCAS(&parent[b], b, a);
        if (old == b) return;
        b = old;
    }
}

__global__ void k_uf_init(int n, int *parent) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) parent[i] = i;
}

// p_c sort keys (order-preserving bits; every NaN last) and rows
__global__ void k_merge_pkeys(int n, const double *pc, unsigned long long *k, unsigned *v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p = pc[i];
    const unsigned long long b = (unsigned long long)__double_as_longlong(p);
    k[i] = isnan(p) ? ~0ull : ((b >> 63) ? ~b : (b | 0x8000000000000000ull));
    v[i] = (unsigned)i;
}

// The rows sorted by p_c: the rows whose p_c matches row i's form a contiguous
// run around it (2|a - b| / (|a| + |b| + DELTA) grows as b moves away from a on
// either side; the NaNs, which only match each other, come last).  One warp per
// sorted position i sweeps the positions after it until a p_c is beyond the
// threshold with a 2^-30 relative slack (then so is every later one, and the
// exact test, decided within 2^-50 of the threshold, fails for them too).  Each
// matching pair is a union-find edge; the components (and their smallest rows)
// are those of the all-pairs sweep.
__global__ void k_merge_pairs_sorted(int n, const unsigned *srow, const double *pc, const double *fc,
                                     double eps, int *parent) {
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    const int i = (int)w;
    const int ri = (int)srow[i];
    const double pi = pc[ri], fi = fc[ri];
    const bool pn = isnan(pi);
    for (int j0 = i + 1; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        bool beyond = j >= n;
        if (!beyond) {
            const int rj = (int)srow[j];
            const double pj = pc[rj];
            if (!pn) {
                const double r = DMUL(2.0, fabs(DSUB(pi, pj))), s = DADD(DADD(fabs(pi), fabs(pj)), DELTA);
                beyond = isnan(pj) || r > eps * s * (1.0 + 0x1.0p-30);
            }
            if (!beyond && values_match(pi, pj, eps) && values_match(fi, fc[rj], eps)) {
                // cached (possibly stale) parents: a stale parent is still an ancestor,
                // so equal answers prove one component; otherwise the CAS-based union
                // resolves the roots exactly
                int a = ri, b = rj, pa, pb;
                while ((pa = __ldca(parent + a)) != a) a = pa;
                while ((pb = __ldca(parent + b)) != b) b = pb;
                if (a != b) uf_union(parent, a, b);
            }
        }
        if (__any_sync(0xffffffffu, beyond)) break;
    }
}

// the members' records in group order (the sequential sums below read them
// contiguously): counts (as bits), loc[4], p_c, f_c
__global__ void k_merge_gather(int n, const unsigned *members, const long long *np_, const long long *nf_,
                               const double *loc, const double *pc, const double *fc, double *rec) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int r = (int)members[q];
    double *o = rec + (size_t)q * 8;
    o[0] = __longlong_as_double(np_[r]);
    o[1] = __longlong_as_double(nf_[r]);
#pragma unroll
    for (int d = 0; d < 4; ++d) o[2 + d] = loc[(size_t)d * n + r];
    o[6] = pc[r];
    o[7] = fc[r];
}

__global__ void k_uf_flatten(int n, int *parent, const int *ids, int *rep_row, int *rep_id,
                             unsigned *keys, unsigned *vals, int *is_root) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int r = uf_find(parent, i);
    rep_row[i] = r;
    rep_id[i] = ids[r];
    keys[i] = (unsigned)r;
    vals[i] = (unsigned)i;
    is_root[i] = r == i;
}

struct MergeOut {
    int *m_ids;
    double *m_loc, *m_p, *m_f;
    long long *m_np, *m_nf;
};

// One warp per group (launched per sorted position; only a group's first
// position works), members ascending (stable sort by root row), records
// gathered contiguously (k_merge_gather).  The sums keep the reference's
// sequential order.  The lanes load a batch of 32 members' records into shared
// memory (the next batch's loads are in flight meanwhile) and split the chains:
// lanes 0-3 the count-weighted location sums, lane 4 the point-value sum, lane
// 5 the field-value sum (Neumaier steps as CPython >= 3.12's sum of floats when
// `neumaier`, else plain), every lane the counts.
constexpr int MG_WARPS = 8;
__global__ void __launch_bounds__(32 * MG_WARPS) k_merge_groups(int n, const unsigned *skeys, const int *group_of_root,
                                                               const int *ids, const double *rec, MergeOut o, int G,
                                                               int neumaier) {
    __shared__ double buf[MG_WARPS][32][9];   // 9: no bank conflicts on the column reads
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (wid >= n) return;
    const int i = (int)wid;                        // position in the sorted order
    if (i > 0 && skeys[i - 1] == skeys[i]) return;   // not the first member of its group
    const unsigned root = skeys[i];
    const int g = group_of_root[root];
    long long n_p = 0, n_f = 0, n_tot = 0;
    double acc = 0.0, cmp = 0.0;   // lane 0-3: loc sum d; 4: p sum; 5: f sum
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const int col = lane < 6 ? 2 + lane : 2;       // record column of this lane's chain
    double nxt[8];
    bool nin = i + lane < n && skeys[i + lane] == root;
#pragma unroll
    for (int c = 0; c < 8; ++c) nxt[c] = nin ? rec[(size_t)(i + lane) * 8 + c] : 0.0;
    for (int q0 = i; q0 < n; q0 += 32) {
        const int cnt = __popc(__ballot_sync(0xffffffffu, nin));   // lanes 0 .. cnt-1 (contiguous)
#pragma unroll
        for (int c = 0; c < 8; ++c) buf[w][lane][c] = nxt[c];
        __syncwarp();
        const bool more = cnt == 32 && q0 + 32 < n;
        if (more) {   // prefetch the next batch
            const int q = q0 + 32 + lane;
            nin = q < n && skeys[q] == root;
#pragma unroll
            for (int c = 0; c < 8; ++c) nxt[c] = nin ? rec[(size_t)q * 8 + c] : 0.0;
        }
        // branch-free steps (the chains only depend on acc / cmp: the loads of the
        // next members are scheduled ahead)
        const bool comp = neumaier && (lane == 4 || lane == 5);
#pragma unroll 4
        for (int t = 0; t < cnt; ++t) {
            const long long a = __double_as_longlong(buf[w][t][0]), b = __double_as_longlong(buf[w][t][1]);
            const long long tt = a + b;
            n_p += a;
            n_f += b;
            n_tot += tt;
            const double v = buf[w][t][col];
            const double x = DMUL(v, (double)(lane < 4 ? tt : lane == 4 ? a : b));
            const double t2 = DADD(acc, x);
            const bool skip = lane >= 4 && isnan(v);   // a member without the value kind
            if (comp && !skip)
                cmp = fabs(acc) >= fabs(x) ? DADD(cmp, DADD(DSUB(acc, t2), x))
                                           : DADD(cmp, DADD(DSUB(x, t2), acc));
            acc = skip ? acc : t2;
        }
        __syncwarp();
        if (!more) break;
    }
    if (lane == 4 || lane == 5)
        if (cmp != 0.0 && isfinite(cmp)) acc = DADD(acc, cmp);
    const double pf = __shfl_sync(0xffffffffu, acc, 4), ff = __shfl_sync(0xffffffffu, acc, 5);
    if (lane < 4) o.m_loc[(size_t)lane * G + g] = DDIV(acc, (double)n_tot);
    if (lane != 0) return;
    o.m_ids[g] = ids[root];
    o.m_p[g] = n_p > 0 ? DDIV(pf, (double)n_p) : nan;
    o.m_f[g] = n_f > 0 ? DDIV(ff, (double)n_f) : nan;
    o.m_np[g] = n_p;
    o.m_nf[g] = n_f;
}

__global__ void k_relabel(const int *labels, long long n, const int *lut, int lut_len, int *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        int l = labels[i];
        out[i] = (l >= 0 && l < lut_len) ? lut[l] : -1;
    }
}

// ------------------------------------------------------------------ voxel CSR
__global__ void k_voxel_keys(const int *flab, long long n, long long ncell, const int *slot_of,
                             int lut_len, int n_slots, unsigned *keys, unsigned *vals,
                             int *bad) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        long long m = q / ncell;
        int l = flab[q];
        int s = (l >= 0 && l < lut_len) ? slot_of[l] : -1;
        if (s < 0) {
            *bad = 1;
            s = 0;
        }
        keys[q] = (unsigned)(m * n_slots + s);
        vals[q] = (unsigned)(q - m * ncell);
    }
}

__global__ void k_key_hist(const unsigned *skeys, long long n, long long *cnt) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        // run-length: only the last element of a run adds the run length
        if (q + 1 == n || skeys[q + 1] != skeys[q]) {
            long long a = 0, b = q;   // find run start by binary search on sorted keys
            unsigned k = skeys[q];
            while (a < b) {
                long long mid = (a + b) >> 1;
                if (skeys[mid] < k) a = mid + 1; else b = mid;
            }
            cnt[k] = q - a + 1;
        }
    }
}

// Counting-sort path (few features): tiles of VT consecutive cells of one
// timestep, 8 warps x VW cells each, 16 cells per lane kept in registers.
//   k_voxel_hist:    per tile and slot the cell count -> H[(m*ns + s)*tpm + tile]
//   (exclusive scan of H: every (m, s, tile) run's output offset, in (m, s)
//    order and, within (m, s), tile order -> stable, cells ascending)
//   k_voxel_scatter: warp-ordered ranks inside the tile, cells written once.
constexpr int VT = 4096, VW = VT / 8, VSLOTS = 256;

__device__ __forceinline__ int voxel_slot(const int *slot_of, int lut_len, int l, int *bad) {
    const int s = (l >= 0 && l < lut_len) ? __ldg(slot_of + l) : -1;
    if (s < 0) *bad = 1;
    return s < 0 ? 0 : s;
}

__global__ void __launch_bounds__(256) k_voxel_hist(const int *flab, long long ncell, int tpm,
                                                    const int *slot_of, int lut_len, int ns,
                                                    int *H, int *bad) {
    __shared__ int hist[VSLOTS];
    const int tile = blockIdx.x % tpm, m = blockIdx.x / tpm;
    for (int i = threadIdx.x; i < ns; i += 256) hist[i] = 0;
    __syncthreads();
    const long long c0 = (long long)tile * VT;
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < VT / 256; ++k) {
        const long long c = c0 + k * 256 + threadIdx.x;
        int s = -1;
        if (c < ncell) s = voxel_slot(slot_of, lut_len, __ldg(flab + (long long)m * ncell + c), bad);
        // labels are spatially coherent: a ballot loop over the round's distinct
        // slots (mostly one or two) is cheaper than MATCH.ANY
        unsigned act = __ballot_sync(0xffffffffu, s >= 0);
        while (act) {
            const int L = __shfl_sync(0xffffffffu, s, __ffs(act) - 1);
            const unsigned grp = __ballot_sync(0xffffffffu, s == L);
            if (lane == __ffs(act) - 1) atomicAdd(&hist[L], __popc(grp));
            act &= ~grp;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ns; i += 256) H[((long long)m * ns + i) * tpm + tile] = hist[i];
}

__global__ void __launch_bounds__(256) k_voxel_scatter(const int *flab, long long ncell, int tpm,
                                                       const int *slot_of, int lut_len, int ns,
                                                       const long long *O, int *cells, int *bad) {
    __shared__ int wcnt[8][VSLOTS];     // per warp: its cells per slot, then its base in the tile
    const int tile = blockIdx.x % tpm, m = blockIdx.x / tpm;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 8 * VSLOTS; i += 256) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const long long c0 = (long long)tile * VT + (long long)w * VW;
    int sl[VW / 32];
#pragma unroll
    for (int k = 0; k < VW / 32; ++k) {
        const long long c = c0 + k * 32 + lane;
        sl[k] = c < ncell ? voxel_slot(slot_of, lut_len, __ldg(flab + (long long)m * ncell + c), bad) : -1;
        unsigned act = __ballot_sync(0xffffffffu, sl[k] >= 0);
        while (act) {
            const int L = __shfl_sync(0xffffffffu, sl[k], __ffs(act) - 1);
            const unsigned grp = __ballot_sync(0xffffffffu, sl[k] == L);
            if (lane == __ffs(act) - 1) wcnt[w][L] += __popc(grp);
            act &= ~grp;
        }
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over the warps per slot (warp order = cell order)
    for (int s = threadIdx.x; s < ns; s += 256) {
        int run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int c = wcnt[q][s];
            wcnt[q][s] = run;
            run += c;
        }
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < VW / 32; ++k) {
        const int s = sl[k];
        unsigned grp = 0;
        unsigned act = __ballot_sync(0xffffffffu, s >= 0);
        while (act) {   // this lane's group = the lanes with its slot
            const int L = __shfl_sync(0xffffffffu, s, __ffs(act) - 1);
            const unsigned g = __ballot_sync(0xffffffffu, s == L);
            if (s == L) grp = g;
            act &= ~g;
        }
        if (s >= 0) {
            const int base = wcnt[w][s];
            const long long dst = O[((long long)m * ns + s) * tpm + tile] + base + __popc(grp & lt);
            cells[dst] = (int)(c0 + k * 32 + lane);
        }
        __syncwarp();
        if (s >= 0 && lane == __ffs(grp) - 1) wcnt[w][s] += __popc(grp);
        __syncwarp();
    }
}

__global__ void k_voxel_segs(int nseg, int tpm, const long long *O, long long n, long long *seg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nseg) seg[i] = O[(long long)i * tpm];
    if (i == 0) seg[nseg] = n;
}

__global__ void k_widen_i32(const int *in, long long n, long long *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = in[i];
}

// ------------------------------------------------------------------ feature stats
// per slot words: [0..1] sum pv, [2..3] sum fv, [4..5] ssq pv, [6..7] ssq fv,
// [8] n_p, [9] n_f, [10..13] bbox min (ordered bits), [14..17] bbox max
constexpr int SW = 18;

__device__ __forceinline__ unsigned long long okey(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unokey(unsigned long long b) {
    unsigned long long r = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    return __longlong_as_double((long long)r);
}

struct StatArgs {
    int n_slots;
    long long nf, ncell;
    int nx, ny, nz;
    double ox, oy, oz, sx, sy, sz;
    int x0, y0, z0;   // global index of the first cell (spatial slabs)
    const double *times, *values;
    const int *fslot;
    long long np;
    const double *xyz, *pt, *pv;
    const int *pslot;
    unsigned long long *S;
    const double *mean;
    int *ovf;
};

// One pass over the samples: every lane accumulates the run of samples of one
// feature it meets (128-bit fixed-point value sums, counts, bounding box) in
// registers and adds the run to its slot record when the feature changes and
// at the end -- a few atomics per run instead of a warp reduction per 32
// samples.  Each warp takes a contiguous range of the samples, 32 consecutive
// ones per step (coalesced loads), so a lane's runs are long.  SMEM: the block
// accumulates into a shared-memory copy of the slot records (few features: the
// global ones would serialise the final flushes on a handful of addresses) and
// adds it to the global records once.  Integer sums and min/max keys: the
// result does not depend on the order, the grid or the partition of the samples.
constexpr int STAT_SMEM_SLOTS = 320;   // 320 x 18 x 8 B = 45 KB
constexpr int STAT_BLOCKS = 148 * 8;

__device__ __forceinline__ void add_fix(unsigned long long &lo, long long &hi, unsigned long long l,
                                        long long h) {
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(l), "l"(h));
}

// d2fix (common.cuh) for the per-sample statistics: the same value (|x| 2^64
// truncated toward zero, negated for x < 0) from the integer and fractional
// parts by hardware conversions instead of shifts on the exponent
__device__ __noinline__ void d2fix_rare(double x, unsigned long long &lo, long long &hi, int *ovf) {
    d2fix(x, lo, hi, ovf);
}

__device__ __forceinline__ void d2fix_stat(double x, unsigned long long &lo, long long &hi, int *ovf) {
    const double ax = fabs(x);
    if (!(ax < 0x1.0p62)) {   // also NaN / inf (out of line: keeps the hot loops small)
        d2fix_rare(x, lo, hi, ovf);
        return;
    }
    const double ih = trunc(ax);
    const unsigned long long uh = (unsigned long long)ih;
    const unsigned long long ul = __double2ull_rz(DMUL(DSUB(ax, ih), 0x1.0p64));   // exact difference
    if (x < 0.0) {
        lo = 0ull - ul;
        hi = (long long)(~uh + (ul == 0 ? 1ull : 0ull));
    } else {
        lo = ul;
        hi = (long long)uh;
    }
}

// bounding-box keys into a slot record (atomics only when the box grows)
__device__ __forceinline__ void bbox_flush(unsigned long long *s, const unsigned long long *k0,
                                           const unsigned long long *k1) {
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        if (k0[d] < ((volatile unsigned long long *)s)[10 + d]) atomicMin(s + 10 + d, k0[d]);
        if (k1[d] > ((volatile unsigned long long *)s)[14 + d]) atomicMax(s + 14 + d, k1[d]);
    }
}

template <bool SMEM>
__device__ __forceinline__ unsigned long long *stat_records(const StatArgs &a) {
    extern __shared__ unsigned long long sS[];
    if (SMEM) {
        for (int i = threadIdx.x; i < a.n_slots * SW; i += blockDim.x) {
            const int w = i % SW;
            sS[i] = (w >= 10 && w < 14) ? ~0ull : 0ull;
        }
        __syncthreads();
        return sS;
    }
    return a.S;
}

template <bool SMEM>
__device__ __forceinline__ void stat_records_flush(const StatArgs &a) {
    extern __shared__ unsigned long long sS[];
    if (!SMEM) return;
    __syncthreads();
    for (int i = threadIdx.x; i < a.n_slots * SW; i += blockDim.x) {
        const int w = i % SW;
        unsigned long long *g = a.S + i;
        const unsigned long long v = sS[i];
        if (w < 8) {
            if ((w & 1) == 0 && (v | sS[i + 1])) atomic_add_fix(g, v, (long long)sS[i + 1]);
        } else if (w < 10) {
            if (v) atomicAdd(g, v);
        } else if (w < 14) {
            if (v != ~0ull) atomicMin(g, v);
        } else if (v) {
            atomicMax(g, v);
        }
    }
}

// Field samples: each lane takes 8 consecutive samples of every 256-sample
// segment of its warp's range (vector loads), so along x its runs follow the
// feature; the next segment is the next 256 cells (the same x strip of the next
// rows when nx = 256).  The run's bounding box is kept in cell indices
// (cell_coord is monotone in the index: the coordinate box is the keys of the
// extreme indices) and time keys; y, z, t are only re-examined at row changes.
// (out of line: runs end rarely, and eight inlined copies in the unrolled sample
// loop overflowed the instruction cache)
struct FieldGeom {
    double ox, oy, oz, sx, sy, sz;
    int x0, y0, z0;
};

__device__ __noinline__ void field_run_flush(unsigned long long *S, FieldGeom gm, int pass, int rs,
                                             unsigned rn, unsigned long long lo, long long hi, unsigned bx0,
                                             unsigned bx1, unsigned by0, unsigned by1, unsigned bz0, unsigned bz1,
                                             unsigned long long t0, unsigned long long t1) {
    unsigned long long *s = S + (size_t)rs * SW;
    if (pass == 1) {
        atomic_add_fix(s + 6, lo, hi);
        return;
    }
    atomic_add_fix(s + 2, lo, hi);
    atomicAdd(s + 9, (unsigned long long)rn);
    const unsigned long long ka = okey(cell_coord(gm.ox, gm.sx, gm.x0 + (long long)bx0)),
                             kb = okey(cell_coord(gm.ox, gm.sx, gm.x0 + (long long)bx1)),
                             kc = okey(cell_coord(gm.oy, gm.sy, gm.y0 + (long long)by0)),
                             kd = okey(cell_coord(gm.oy, gm.sy, gm.y0 + (long long)by1)),
                             ke = okey(cell_coord(gm.oz, gm.sz, gm.z0 + (long long)bz0)),
                             kf = okey(cell_coord(gm.oz, gm.sz, gm.z0 + (long long)bz1));
    const unsigned long long k0[4] = {min(ka, kb), min(kc, kd), min(ke, kf), t0};
    const unsigned long long k1[4] = {max(ka, kb), max(kc, kd), max(ke, kf), t1};
    bbox_flush(s, k0, k1);
}

template <bool SMEM>
__global__ void __launch_bounds__(256) k_stats_field(StatArgs a, int pass) {
    unsigned long long *S = stat_records<SMEM>(a);
    const int lane = threadIdx.x & 31;
    long long q0, q1;
    {   // this warp's contiguous share of whole 256-sample segments
        const long long W = (long long)gridDim.x * (blockDim.x >> 5);
        const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        const long long segs = (a.nf + 255) >> 8, per = (segs + W - 1) / W;
        q0 = min(a.nf, gw * per * 256);
        q1 = min(a.nf, (gw + 1) * per * 256);
    }
    const unsigned nx = (unsigned)a.nx, ny = (unsigned)a.ny, nz = (unsigned)a.nz;
    const long long plane = (long long)nx * ny;
    unsigned dx, dy, dz, dm;   // 256 in (timestep, z, y, x) digits
    {
        long long r = 256;
        dm = (unsigned)(r / a.ncell);
        r %= a.ncell;
        dz = (unsigned)(r / plane);
        r %= plane;
        dy = (unsigned)(r / nx);
        dx = (unsigned)(r % nx);
    }
    unsigned ix = 0, iy = 0, iz = 0, m = 0;   // the lane's first sample of the segment
    if (q0 < q1) {
        const long long q = q0 + 8 * lane;
        m = (unsigned)(q / a.ncell);
        long long r = q % a.ncell;
        iz = (unsigned)(r / plane);
        r %= plane;
        iy = (unsigned)(r / nx);
        ix = (unsigned)(r % nx);
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(a.fslot) | reinterpret_cast<uintptr_t>(a.values)) & 15) == 0;
    const FieldGeom gm{a.ox, a.oy, a.oz, a.sx, a.sy, a.sz, a.x0, a.y0, a.z0};
    int ovf = 0;
    int rs = -1;                       // the run's slot
    unsigned rn = 0;
    unsigned long long lo = 0;
    long long hi = 0;
    unsigned b0[3] = {0, 0, 0}, b1[3] = {0, 0, 0};   // index box (x, y, z)
    unsigned long long t0 = 0, t1 = 0, tk = 0;
    unsigned mk = 0xFFFFFFFFu;
    double mu = 0.0;
    for (long long sb = q0; sb < q1; sb += 256) {
        const long long qb = sb + 8 * lane;
        int sl[8];
        double vv[8];
        if (vec && qb + 8 <= q1) {
            const int4 s0 = *reinterpret_cast<const int4 *>(a.fslot + qb);
            const int4 s1 = *reinterpret_cast<const int4 *>(a.fslot + qb + 4);
            sl[0] = s0.x; sl[1] = s0.y; sl[2] = s0.z; sl[3] = s0.w;
            sl[4] = s1.x; sl[5] = s1.y; sl[6] = s1.z; sl[7] = s1.w;
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
                const double2 v2 = *reinterpret_cast<const double2 *>(a.values + qb + k);
                vv[k] = v2.x;
                vv[k + 1] = v2.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                sl[k] = qb + k < q1 ? a.fslot[qb + k] : -1;
                vv[k] = sl[k] >= 0 ? a.values[qb + k] : 0.0;
            }
        }
        unsigned jx = ix, jy = iy, jz = iz, jm = m;
        bool row = true;   // y / z / t not yet examined in this row for the run
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int slot = sl[k];
            if (slot >= 0) {
                if (slot != rs) {
                    if (rs >= 0)
                        field_run_flush(S, gm, pass, rs, rn, lo, hi, b0[0], b1[0], b0[1], b1[1], b0[2], b1[2],
                                        t0, t1);
                    rs = slot;
                    rn = 0;
                    lo = 0;
                    hi = 0;
                    b0[0] = b1[0] = jx;
                    row = true;
                    if (pass == 0) {
                        b0[1] = b1[1] = jy;
                        b0[2] = b1[2] = jz;
                        if (jm != mk) {
                            tk = okey(a.times[jm]);
                            mk = jm;
                        }
                        t0 = t1 = tk;
                    } else {
                        mu = a.mean[2 * slot + 1];
                    }
                }
                unsigned long long l;
                long long h;
                if (pass == 0) {
                    d2fix_stat(vv[k], l, h, &ovf);
                    ++rn;
                    b0[0] = min(b0[0], jx);
                    b1[0] = max(b1[0], jx);
                    if (row) {
                        row = false;
                        b0[1] = min(b0[1], jy);
                        b1[1] = max(b1[1], jy);
                        b0[2] = min(b0[2], jz);
                        b1[2] = max(b1[2], jz);
                        if (jm != mk) {
                            tk = okey(a.times[jm]);
                            mk = jm;
                        }
                        t0 = min(t0, tk);
                        t1 = max(t1, tk);
                    }
                } else {
                    const double dv = DSUB(vv[k], mu);
                    d2fix_stat(DMUL(dv, dv), l, h, &ovf);
                }
                add_fix(lo, hi, l, h);
            }
            if (++jx == nx) {   // next row
                jx = 0;
                row = true;
                if (++jy == ny) {
                    jy = 0;
                    if (++jz == nz) {
                        jz = 0;
                        ++jm;
                    }
                }
            }
        }
        // the lane's first sample of the next segment: + 256
        unsigned c;
        ix += dx;
        c = ix >= nx;
        ix -= c ? nx : 0u;
        iy += dy + c;
        c = iy >= ny;
        iy -= c ? ny : 0u;
        iz += dz + c;
        c = iz >= nz;
        iz -= c ? nz : 0u;
        m += dm + c;
    }
    if (rs >= 0)
        field_run_flush(S, gm, pass, rs, rn, lo, hi, b0[0], b1[0], b0[1], b1[1], b0[2], b1[2], t0, t1);
    if (ovf) *a.ovf = 1;
    stat_records_flush<SMEM>(a);
}

// Point samples (record order: a trajectory's samples are consecutive): as the
// field kernel, each lane takes 8 consecutive records of every 256-record
// segment of its warp's range, so a lane's run follows one trajectory.
__device__ __noinline__ void point_run_flush(unsigned long long *S, int pass, int rs, unsigned rn,
                                             unsigned long long lo, long long hi, unsigned long long a0,
                                             unsigned long long a1, unsigned long long a2, unsigned long long a3,
                                             unsigned long long c0, unsigned long long c1, unsigned long long c2,
                                             unsigned long long c3) {
    unsigned long long *s = S + (size_t)rs * SW;
    if (pass == 1) {
        atomic_add_fix(s + 4, lo, hi);
        return;
    }
    atomic_add_fix(s, lo, hi);
    atomicAdd(s + 8, (unsigned long long)rn);
    const unsigned long long k0[4] = {a0, a1, a2, a3}, k1[4] = {c0, c1, c2, c3};
    bbox_flush(s, k0, k1);
}

template <bool SMEM>
__global__ void __launch_bounds__(256) k_stats_points(StatArgs a, int pass) {
    unsigned long long *S = stat_records<SMEM>(a);
    const int lane = threadIdx.x & 31;
    long long q0, q1;
    {   // this warp's contiguous share of whole 256-record segments
        const long long W = (long long)gridDim.x * (blockDim.x >> 5);
        const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        const long long segs = (a.np + 255) >> 8, per = (segs + W - 1) / W;
        q0 = min(a.np, gw * per * 256);
        q1 = min(a.np, (gw + 1) * per * 256);
    }
    int ovf = 0;
    int rs = -1;
    unsigned rn = 0;
    unsigned long long lo = 0;
    long long hi = 0;
    unsigned long long k0[4] = {0, 0, 0, 0}, k1[4] = {0, 0, 0, 0};
    double mu = 0.0;
    for (long long sb = q0; sb < q1; sb += 256) {
        const long long qb = sb + 8 * lane;
#pragma unroll 2
        for (int k = 0; k < 8; ++k) {
            const long long q = qb + k;
            const int slot = q < q1 ? a.pslot[q] : -1;
            if (slot < 0) continue;
            const double v = a.pv[q];
            unsigned long long kk[4];
            if (pass == 0) {
                kk[0] = okey(a.xyz[3 * q]);
                kk[1] = okey(a.xyz[3 * q + 1]);
                kk[2] = okey(a.xyz[3 * q + 2]);
                kk[3] = okey(a.pt[q]);
            }
            if (slot != rs) {
                if (rs >= 0)
                    point_run_flush(S, pass, rs, rn, lo, hi, k0[0], k0[1], k0[2], k0[3], k1[0], k1[1], k1[2],
                                    k1[3]);
                rs = slot;
                rn = 0;
                lo = 0;
                hi = 0;
                if (pass == 0) {
#pragma unroll
                    for (int d = 0; d < 4; ++d) k0[d] = k1[d] = kk[d];
                } else {
                    mu = a.mean[2 * slot];
                }
            }
            unsigned long long l;
            long long h;
            if (pass == 0) {
                d2fix_stat(v, l, h, &ovf);
                ++rn;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    k0[d] = min(k0[d], kk[d]);
                    k1[d] = max(k1[d], kk[d]);
                }
            } else {
                const double dv = DSUB(v, mu);
                d2fix_stat(DMUL(dv, dv), l, h, &ovf);
            }
            add_fix(lo, hi, l, h);
        }
    }
    if (rs >= 0)
        point_run_flush(S, pass, rs, rn, lo, hi, k0[0], k0[1], k0[2], k0[3], k1[0], k1[1], k1[2], k1[3]);
    if (ovf) *a.ovf = 1;
    stat_records_flush<SMEM>(a);
}

int launch_stats(const StatArgs &a, int pass, cudaStream_t st) {
    const bool sm = a.n_slots <= STAT_SMEM_SLOTS;
    const size_t bytes = sm ? (size_t)a.n_slots * SW * 8 : 0;
    if (a.nf > 0) {
        ::mfseg::count_launch();
        if (sm) k_stats_field<true><<<STAT_BLOCKS, 256, bytes, st>>>(a, pass);
        else k_stats_field<false><<<STAT_BLOCKS, 256, 0, st>>>(a, pass);
        MFSEG_LAUNCH("k_stats_field");
    }
    if (a.np > 0) {
        ::mfseg::count_launch();
        if (sm) k_stats_points<true><<<STAT_BLOCKS, 256, bytes, st>>>(a, pass);
        else k_stats_points<false><<<STAT_BLOCKS, 256, 0, st>>>(a, pass);
        MFSEG_LAUNCH("k_stats_points");
    }
    return 0;
}

__global__ void k_stats_means(int n_slots, const unsigned long long *S, double *mean) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    const unsigned long long *w = S + (size_t)s * SW;
    long long np = (long long)w[8], nf = (long long)w[9];
    mean[2 * s] = np ? DDIV(fix2d(w[0], (long long)w[1]), (double)np) : 0.0;
    mean[2 * s + 1] = nf ? DDIV(fix2d(w[2], (long long)w[3]), (double)nf) : 0.0;
}

__global__ void k_stats_final(int n_slots, const unsigned long long *S, const double *mean,
                              double *out) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    const unsigned long long *w = S + (size_t)s * SW;
    double *o = out + (size_t)s * MFSEG_STAT_WORDS;
    long long np = (long long)w[8], nf = (long long)w[9];
    double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (int d = 0; d < 4; ++d) {
        bool any = np + nf > 0;
        o[d] = any ? unokey(w[10 + d]) : nan;
        o[4 + d] = any ? unokey(w[14 + d]) : nan;
    }
    o[8] = np ? mean[2 * s] : nan;
    o[9] = np ? DSQRT(DDIV(fix2d(w[4], (long long)w[5]), (double)np)) : nan;
    o[10] = nf ? mean[2 * s + 1] : nan;
    o[11] = nf ? DSQRT(DDIV(fix2d(w[6], (long long)w[7]), (double)nf)) : nan;
    o[12] = (double)np;
    o[13] = (double)nf;
}

__global__ void k_stats_init(int n_slots, unsigned long long *S) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots) return;
    unsigned long long *w = S + (size_t)s * SW;
    for (int i = 0; i < 10; ++i) w[i] = 0;
    for (int d = 0; d < 4; ++d) {
        w[10 + d] = ~0ull;
        w[14 + d] = 0ull;
    }
}

// ------------------------------------------------------------------ link index
__global__ void k_link_keys(long long n, const double *xyz, const double *t, int nx, int ny,
                            int nz, double ox, double oy, double oz, double sx, double sy,
                            double sz, const double *times, int nt, unsigned long long *keys,
                            unsigned *vals, int *bad) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double cx = floor(DDIV(DSUB(xyz[3 * i], ox), sx));
    double cy = floor(DDIV(DSUB(xyz[3 * i + 1], oy), sy));
    double cz = floor(DDIV(DSUB(xyz[3 * i + 2], oz), sz));
    if (!(cx >= 0 && cx < nx && cy >= 0 && cy < ny && cz >= 0 && cz < nz)) {
        *bad = 1;
        cx = cy = cz = 0;
    }
    int n_int = nt - 1 > 1 ? nt - 1 : 1;
    // searchsorted(times, t, 'right') - 1, clipped to [0, n_int-1]
    int a = 0, b = nt;
    double tv = t[i];
    while (a < b) {
        int mid = (a + b) >> 1;
        if (times[mid] <= tv) a = mid + 1; else b = mid;
    }
    int m = a - 1;
    if (m < 0) m = 0;
    if (m > n_int - 1) m = n_int - 1;
    long long flat = (((long long)cz * ny + (long long)cy) * nx + (long long)cx) * n_int + m;
    keys[i] = (unsigned long long)flat;
    vals[i] = (unsigned)i;
}

__global__ void k_count_runs(const unsigned long long *k, long long n, unsigned long long *cnt) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n && (i == 0 || k[i] != k[i - 1])) atomicAdd(cnt, 1ull);
}

int bits_of(unsigned long long v) {
    int b = 1;
    while (b < 64 && (1ull << b) <= v) ++b;
    return b;
}

}  // namespace

namespace {

// ------------------------------------------------------------------ trajectory split
// build_features' polylines (postproc.py:152-160, 176-191): points ordered by
// (traj_id, t) (np.lexsort, stable), runs broken at a new trajectory, a feature
// change or a time gap larger than stride * (1 + 1e-9), stride = the smallest
// positive difference of the sorted unique point times.

__device__ __forceinline__ unsigned long long dkey(double x) {   // order-preserving bits
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// time keys restricted to the bits that vary (the bits above and below are the
// same in every key, so the order is kept and the radix sort takes fewer passes)
__global__ void k_tkeys(long long n, const double *t, int lo, unsigned long long mask, unsigned long long *k,
                        unsigned *v) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    k[i] = (dkey(t[i]) >> lo) & mask;
    v[i] = (unsigned)i;
}

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ long long warp_max_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One pass over the points: the trajectory id range, the bits in which the time
// keys differ from the first one, and whether the records are already in
// lexsort((t, traj_id)) order (then the stable sort is the identity).
__global__ void k_tscan(long long n, const double *t, const long long *tid, unsigned long long *misc) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    unsigned long long span = 0;
    int unsorted = 0;
    const unsigned long long k0 = dkey(t[0]);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long id = tid[i];
        const double ti = t[i];
        lo = min(lo, id);
        hi = max(hi, id);
        span |= dkey(ti) ^ k0;
        if (i > 0) {
            const long long ip = tid[i - 1];
            unsorted |= id < ip || (id == ip && ti < t[i - 1]);
        }
    }
    lo = warp_min_ll(lo);
    hi = warp_max_ll(hi);
    span = __reduce_or_sync(0xffffffffu, (unsigned)span) | ((unsigned long long)__reduce_or_sync(
                                                                 0xffffffffu, (unsigned)(span >> 32)) << 32);
    unsorted = __reduce_or_sync(0xffffffffu, unsorted);
    if ((threadIdx.x & 31) == 0) {
        // signed -> order-preserving unsigned for the atomics
        atomicMin(&misc[1], (unsigned long long)lo ^ 0x8000000000000000ull);
        atomicMax(&misc[2], (unsigned long long)hi ^ 0x8000000000000000ull);
        if (span) atomicOr(&misc[3], span);
        if (unsorted) atomicOr(&misc[4], 1ull);
    }
}

__global__ void k_iota_u32(long long n, unsigned *v) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) v[i] = (unsigned)i;
}

// over the sorted times: unique flags and the smallest positive gap between uniques
__global__ void k_tunique(long long n, const unsigned long long *sk, const unsigned *perm,
                          const double *t, int *uflag, unsigned long long *min_gap) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool u = i == 0 || sk[i] != sk[i - 1];
    uflag[i] = u ? 1 : 0;
    if (u && i > 0) {
        const double g = DSUB(t[perm[i]], t[perm[i - 1]]);   // np.diff(np.unique(t))
        if (g > 0.0) atomicMin(min_gap, (unsigned long long)__double_as_longlong(g));
    }
}

// t rank of every point (index of its value among the sorted unique times)
__global__ void k_trank(long long n, const int *urank_incl, const unsigned *perm, unsigned *trank) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    trank[perm[i]] = (unsigned)(urank_incl[i] - 1);
}

__global__ void k_lex_keys(long long n, const long long *tid, const unsigned *trank, long long tmin,
                           int tbits, unsigned long long *k, unsigned *v) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    k[i] = ((unsigned long long)(tid[i] - tmin) << tbits) | trank[i];
    v[i] = (unsigned)i;
}

__global__ void k_traj_breaks(long long n, const unsigned *order, const long long *tid,
                              const double *t, const int *lab, double gap_limit, int *brk) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool b = i == 0;
    if (!b) {
        const unsigned j = order[i], q = order[i - 1];
        b = tid[j] != tid[q] || lab[j] != lab[q] || DSUB(t[j], t[q]) > gap_limit;
    }
    brk[i] = b ? 1 : 0;
}

__global__ void k_run_starts(long long n, const int *brk, const int *incl, int *starts) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == n) {
        starts[incl[n - 1]] = (int)n;
        return;
    }
    if (brk[i]) starts[incl[i] - 1] = (int)i;
}

__global__ void k_inclusive_from_exclusive(long long n, const int *in, const int *ex, int *incl) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) incl[i] = ex[i] + in[i];
}

}  // namespace
}  // namespace mfseg

using namespace mfseg;

extern "C" {

size_t mfseg_merge_workspace_size(int32_t n) {
    Carver cv;
    cv.take<int>(n);          // parent
    cv.take<int>(n);          // rep_row
    cv.take<unsigned>(n);     // keys
    cv.take<unsigned>(n);     // vals
    cv.take<unsigned>(n);     // skeys
    cv.take<unsigned>(n);     // members
    cv.take<int>(n + 1);      // is_root
    cv.take<int>(n + 1);      // group_of_root
    cv.take<char>(radix_tmp_bytes(n > 0 ? n : 1));
    cv.take<char>(scan_tmp_bytes(n + 1));
    cv.take<unsigned long long>(n);   // p keys
    cv.take<unsigned long long>(n);   // sorted p keys
    cv.take<unsigned>(n);             // rows
    cv.take<unsigned>(n);             // rows by p
    cv.take<double>(8ll * n);         // member records in group order
    return cv.off + 256;
}

int mfseg_merge(int32_t n, const int32_t *ids, const double *loc, const double *p_c,
                const double *f_c, const int64_t *n_points, const int64_t *n_fields, double eps_m,
                int32_t neumaier, int32_t *rep, int32_t *m_ids, double *m_loc, double *m_p, double *m_f,
                int64_t *m_np, int64_t *m_nf, int32_t *n_merged_host, void *workspace,
                size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n <= 0) {
        if (n_merged_host) *n_merged_host = 0;
        return 0;
    }
    if (workspace_bytes < mfseg_merge_workspace_size(n)) {
        set_error("merge: workspace too small");
        return 3;
    }
    Carver cv(workspace, workspace_bytes);
    int *parent = cv.take<int>(n);
    int *rep_row = cv.take<int>(n);
    unsigned *keys = cv.take<unsigned>(n);
    unsigned *vals = cv.take<unsigned>(n);
    unsigned *skeys = cv.take<unsigned>(n);
    unsigned *members = cv.take<unsigned>(n);
    int *is_root = cv.take<int>(n + 1);
    int *group_of_root = cv.take<int>(n + 1);
    size_t rb = radix_tmp_bytes(n);
    void *rtmp = cv.take<char>(rb);
    size_t sb = scan_tmp_bytes(n + 1);
    void *stmp = cv.take<char>(sb);
    unsigned long long *pk = cv.take<unsigned long long>(n), *pks = cv.take<unsigned long long>(n);
    unsigned *prow = cv.take<unsigned>(n), *srow = cv.take<unsigned>(n);
    double *rec = cv.take<double>(8ll * n);
    unsigned g = (unsigned)((n + 255) / 256);
    ::mfseg::count_launch();
    k_uf_init<<<g, 256, 0, st>>>(n, parent);
    ::mfseg::count_launch();
    k_merge_pkeys<<<g, 256, 0, st>>>(n, p_c, pk, prow);
    MFSEG_TRY(radix_sort_pairs64(pk, prow, pks, srow, n, 64, rtmp, rb, st));
    ::mfseg::count_launch();
    k_merge_pairs_sorted<<<(unsigned)(((long long)n * 32 + 255) / 256), 256, 0, st>>>(n, srow, p_c, f_c,
                                                                                      eps_m, parent);
    MFSEG_CUDA(cudaMemsetAsync(is_root, 0, sizeof(int) * (n + 1), st));
    ::mfseg::count_launch();
    k_uf_flatten<<<g, 256, 0, st>>>(n, parent, ids, rep_row, rep, keys, vals, is_root);
    MFSEG_LAUNCH("merge union-find");
    MFSEG_TRY(radix_sort_pairs(keys, vals, skeys, members, n, bits_of((unsigned)n), rtmp, rb, st));
    MFSEG_TRY(scan_exclusive_i32(is_root, group_of_root, n + 1, stmp, sb, st));
    int G = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&G, group_of_root + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    MergeOut o{m_ids, m_loc, m_p, m_f, (long long *)m_np, (long long *)m_nf};
    ::mfseg::count_launch();
    k_merge_gather<<<g, 256, 0, st>>>(n, members, (const long long *)n_points, (const long long *)n_fields, loc,
                                      p_c, f_c, rec);
    ::mfseg::count_launch();
    k_merge_groups<<<(unsigned)(((long long)n + MG_WARPS - 1) / MG_WARPS), 32 * MG_WARPS, 0, st>>>(
        n, skeys, group_of_root, ids, rec, o, G, neumaier);
    MFSEG_LAUNCH("k_merge_groups");
    if (n_merged_host) *n_merged_host = G;
    return 0;
}

int mfseg_relabel(const int32_t *labels, int64_t n, const int32_t *lut, int32_t lut_len,
                  int32_t *out, void *stream) {
    if (n <= 0) return 0;
    ::mfseg::count_launch();
    k_relabel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(labels, n, lut, lut_len, out);
    MFSEG_LAUNCH("k_relabel");
    return 0;
}

static bool voxel_counting(int32_t n_slots) { return n_slots <= VSLOTS; }

size_t mfseg_voxel_csr_workspace_size(int64_t n, int32_t nt, int32_t n_slots) {
    Carver cv;
    const long long ncell = nt > 0 ? n / nt : 0;
    if (voxel_counting(n_slots)) {
        const long long tpm = (ncell + VT - 1) / VT;
        const long long nh = (long long)nt * n_slots * tpm;
        cv.take<int>(nh);
        cv.take<long long>(nh + 1);
        cv.take<long long>(nh + 1);
        cv.take<int>(4);
        cv.take<char>(scan_tmp_bytes(nh + 1));
        return cv.off + 256;
    }
    cv.take<unsigned>(n);
    cv.take<unsigned>(n);
    cv.take<unsigned>(n);
    cv.take<long long>((long long)nt * n_slots + 1);
    cv.take<int>(4);
    cv.take<char>(radix_tmp_bytes(n > 0 ? n : 1));
    cv.take<char>(scan_tmp_bytes((long long)nt * n_slots + 1));
    return cv.off + 256;
}

static int voxel_csr_counting(const int32_t *flab, int32_t nt, int64_t ncell, const int32_t *slot_of,
                              int32_t lut_len, int32_t n_slots, int64_t *seg_start, int32_t *cells,
                              void *workspace, size_t workspace_bytes, cudaStream_t st) {
    const long long tpm = (ncell + VT - 1) / VT;
    const long long nh = (long long)nt * n_slots * tpm;
    if (tpm * nt >= (1ll << 31)) {
        set_error("voxel_csr: too many tiles");
        return 2;
    }
    Carver cv(workspace, workspace_bytes);
    int *H = cv.take<int>(nh);
    long long *H64 = cv.take<long long>(nh + 1);
    long long *O = cv.take<long long>(nh + 1);
    int *bad = cv.take<int>(4);
    const size_t sb = scan_tmp_bytes(nh + 1);
    void *stmp = cv.take<char>(sb);
    MFSEG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    MFSEG_CUDA(cudaMemsetAsync(H64 + nh, 0, sizeof(long long), st));
    const unsigned nb = (unsigned)(tpm * nt);
    ::mfseg::count_launch();
    k_voxel_hist<<<nb, 256, 0, st>>>(flab, ncell, (int)tpm, slot_of, lut_len, n_slots, H, bad);
    ::mfseg::count_launch();
    k_widen_i32<<<148 * 4, 256, 0, st>>>(H, nh, H64);
    MFSEG_TRY(scan_exclusive_i64(H64, O, nh + 1, stmp, sb, st));
    ::mfseg::count_launch();
    k_voxel_scatter<<<nb, 256, 0, st>>>(flab, ncell, (int)tpm, slot_of, lut_len, n_slots, O, cells,
                                        bad);
    const int nseg = nt * n_slots;
    ::mfseg::count_launch();
    k_voxel_segs<<<(nseg + 256) / 256, 256, 0, st>>>(nseg, (int)tpm, O, (long long)nt * ncell,
                                                     (long long *)seg_start);
    MFSEG_LAUNCH("voxel_csr");
    int hb = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (hb) {
        set_error("voxel_csr: a field label has no feature slot");
        return 2;
    }
    return 0;
}

int mfseg_voxel_csr(const int32_t *flab, int32_t nt, int64_t ncell, const int32_t *slot_of,
                    int32_t lut_len, int32_t n_slots, int64_t *seg_start, int32_t *cells,
                    void *workspace, size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    long long n = (long long)nt * ncell;
    long long nseg = (long long)nt * n_slots;
    if (n <= 0) return 0;
    if (n >= (1ll << 31) || nseg >= (1ll << 32)) {
        set_error("voxel_csr: too many samples for one call; split by timestep");
        return 2;
    }
    if (workspace_bytes < mfseg_voxel_csr_workspace_size(n, nt, n_slots)) {
        set_error("voxel_csr: workspace too small");
        return 3;
    }
    if (voxel_counting(n_slots))
        return voxel_csr_counting(flab, nt, ncell, slot_of, lut_len, n_slots, seg_start, cells,
                                  workspace, workspace_bytes, st);
    Carver cv(workspace, workspace_bytes);
    unsigned *keys = cv.take<unsigned>(n);
    unsigned *vals = cv.take<unsigned>(n);
    unsigned *skeys = cv.take<unsigned>(n);
    long long *cnt = cv.take<long long>(nseg + 1);
    int *bad = cv.take<int>(4);
    size_t rb = radix_tmp_bytes(n);
    void *rtmp = cv.take<char>(rb);
    size_t sb = scan_tmp_bytes(nseg + 1);
    void *stmp = cv.take<char>(sb);
    MFSEG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    MFSEG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(long long) * (nseg + 1), st));
    ::mfseg::count_launch();
    k_voxel_keys<<<148 * 8, 256, 0, st>>>(flab, n, ncell, slot_of, lut_len, n_slots, keys, vals,
                                          bad);
    MFSEG_LAUNCH("k_voxel_keys");
    MFSEG_TRY(radix_sort_pairs(keys, vals, skeys, (unsigned *)cells, n, bits_of((unsigned long long)nseg),
                               rtmp, rb, st));
    ::mfseg::count_launch();
    k_key_hist<<<148 * 8, 256, 0, st>>>(skeys, n, cnt);
    MFSEG_TRY(scan_exclusive_i64(cnt, (long long *)seg_start, nseg + 1, stmp, sb, st));
    int hb = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (hb) {
        set_error("voxel_csr: a field label has no feature slot");
        return 2;
    }
    return 0;
}

size_t mfseg_feature_stats_workspace_size(int32_t n_slots) {
    Carver cv;
    cv.take<unsigned long long>((long long)n_slots * SW);
    cv.take<double>(2ll * n_slots);
    cv.take<int>(4);
    return cv.off + 256;
}

static void stat_args(StatArgs &a, int32_t n_slots, const mfseg_field *f, const int32_t *field_slot,
                      const mfseg_points *pts, const int32_t *point_slot) {
    memset(&a, 0, sizeof a);
    a.n_slots = n_slots;
    if (f && f->nt > 0 && field_slot) {
        a.ncell = (long long)f->nx * f->ny * f->nz;
        a.nf = a.ncell * f->nt;
        a.nx = f->nx;
        a.ny = f->ny;
        a.nz = f->nz;
        a.ox = f->origin[0];
        a.oy = f->origin[1];
        a.oz = f->origin[2];
        a.x0 = f->offset[0];
        a.y0 = f->offset[1];
        a.z0 = f->offset[2];
        a.sx = f->spacing[0];
        a.sy = f->spacing[1];
        a.sz = f->spacing[2];
        a.times = f->times;
        a.values = f->values;
        a.fslot = field_slot;
    }
    if (pts && pts->n > 0 && point_slot) {
        a.np = pts->n;
        a.xyz = pts->xyz;
        a.pt = pts->t;
        a.pv = pts->value;
        a.pslot = point_slot;
    }
}

int mfseg_feature_stats(int32_t n_slots, const mfseg_field *f, const int32_t *field_slot,
                        const mfseg_points *pts, const int32_t *point_slot, double *stats,
                        void *workspace, size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_slots <= 0) return 0;
    if (workspace_bytes < mfseg_feature_stats_workspace_size(n_slots)) {
        set_error("feature_stats: workspace too small");
        return 3;
    }
    Carver cv(workspace, workspace_bytes);
    StatArgs a;
    stat_args(a, n_slots, f, field_slot, pts, point_slot);
    a.S = cv.take<unsigned long long>((long long)n_slots * SW);
    double *mean = cv.take<double>(2ll * n_slots);
    a.mean = mean;
    a.ovf = cv.take<int>(4);
    unsigned gs = (unsigned)((n_slots + 255) / 256);
    MFSEG_CUDA(cudaMemsetAsync(a.ovf, 0, sizeof(int), st));
    ::mfseg::count_launch();
    k_stats_init<<<gs, 256, 0, st>>>(n_slots, a.S);
    MFSEG_TRY(launch_stats(a, 0, st));
    ::mfseg::count_launch();
    k_stats_means<<<gs, 256, 0, st>>>(n_slots, a.S, mean);
    MFSEG_TRY(launch_stats(a, 1, st));
    ::mfseg::count_launch();
    k_stats_final<<<gs, 256, 0, st>>>(n_slots, a.S, mean, stats);
    MFSEG_LAUNCH("feature_stats");
    int h = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&h, a.ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (h) {
        set_error("feature_stats: fixed-point overflow");
        return 4;
    }
    return 0;
}

int mfseg_feature_stats_pass(int32_t n_slots, const mfseg_field *f, const int32_t *field_slot,
                             const mfseg_points *pts, const int32_t *point_slot, int32_t pass,
                             const double *mean, uint64_t *partial, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_slots <= 0) return 0;
    if (pass != 0 && pass != 1) {
        set_error("feature_stats_pass: pass must be 0 or 1");
        return 2;
    }
    int *ovf = nullptr, *ovf_h = nullptr;
    MFSEG_TRY(tiny_scratch((void **)&ovf, (void **)&ovf_h));
    StatArgs a;
    stat_args(a, n_slots, f, field_slot, pts, point_slot);
    a.S = (unsigned long long *)partial;
    a.mean = mean;
    a.ovf = ovf;
    unsigned gs = (unsigned)((n_slots + 255) / 256);
    MFSEG_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), st));
    if (pass == 0) {
        ::mfseg::count_launch();
        k_stats_init<<<gs, 256, 0, st>>>(n_slots, a.S);
    }
    MFSEG_TRY(launch_stats(a, pass, st));
    MFSEG_LAUNCH("feature_stats_pass");
    MFSEG_CUDA(cudaMemcpyAsync(ovf_h, ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (*ovf_h) {
        set_error("feature_stats: fixed-point overflow");
        return 4;
    }
    return 0;
}

int mfseg_feature_stats_means(int32_t n_slots, const uint64_t *partial, double *mean, void *stream) {
    if (n_slots <= 0) return 0;
    ::mfseg::count_launch();
    k_stats_means<<<(unsigned)((n_slots + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n_slots, (const unsigned long long *)partial, mean);
    MFSEG_LAUNCH("k_stats_means");
    return 0;
}

int mfseg_feature_stats_final(int32_t n_slots, const uint64_t *partial, const double *mean,
                              double *stats, void *stream) {
    if (n_slots <= 0) return 0;
    ::mfseg::count_launch();
    k_stats_final<<<(unsigned)((n_slots + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        n_slots, (const unsigned long long *)partial, mean, stats);
    MFSEG_LAUNCH("k_stats_final");
    return 0;
}

size_t mfseg_link_index_workspace_size(int64_t n) {
    Carver cv;
    cv.take<unsigned long long>(n);
    cv.take<unsigned>(n);
    cv.take<unsigned long long>(2);
    cv.take<int>(4);
    cv.take<char>(radix_tmp_bytes(n > 0 ? n : 1));
    return cv.off + 256;
}

int mfseg_link_index(const mfseg_field *f, const mfseg_points *pts, int64_t *keys, int32_t *members,
                     int64_t *n_buckets_host, void *workspace, size_t workspace_bytes,
                     void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    long long n = pts ? pts->n : 0;
    if (n_buckets_host) *n_buckets_host = 0;
    if (n <= 0) return 0;
    if (f->offset[0] || f->offset[1] || f->offset[2]) {
        set_error("link_index: the field must be a whole grid (offset 0)");
        return 2;
    }
    if (workspace_bytes < mfseg_link_index_workspace_size(n)) {
        set_error("link_index: workspace too small");
        return 3;
    }
    Carver cv(workspace, workspace_bytes);
    unsigned long long *k0 = cv.take<unsigned long long>(n);
    unsigned *v0 = cv.take<unsigned>(n);
    unsigned long long *cnt = cv.take<unsigned long long>(2);
    int *bad = cv.take<int>(4);
    size_t rb = radix_tmp_bytes(n);
    void *rtmp = cv.take<char>(rb);
    MFSEG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    MFSEG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    unsigned g = (unsigned)((n + 255) / 256);
    ::mfseg::count_launch();
    k_link_keys<<<g, 256, 0, st>>>(n, pts->xyz, pts->t, f->nx, f->ny, f->nz, f->origin[0],
                                   f->origin[1], f->origin[2], f->spacing[0], f->spacing[1],
                                   f->spacing[2], f->times, f->nt, k0, v0, bad);
    MFSEG_LAUNCH("k_link_keys");
    int n_int = f->nt - 1 > 1 ? f->nt - 1 : 1;
    unsigned long long maxkey = (unsigned long long)f->nx * f->ny * f->nz * n_int;
    MFSEG_TRY(radix_sort_pairs64(k0, v0, (unsigned long long *)keys, (unsigned *)members, n,
                                 bits_of(maxkey), rtmp, rb, st));
    ::mfseg::count_launch();
    k_count_runs<<<g, 256, 0, st>>>((const unsigned long long *)keys, n, cnt);
    MFSEG_LAUNCH("k_count_runs");
    int hb = 0;
    unsigned long long nb = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaMemcpyAsync(&nb, cnt, sizeof(nb), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (hb) {
        set_error("point sample outside the field grid; filter_to_grid first");
        return 2;
    }
    if (n_buckets_host) *n_buckets_host = (int64_t)nb;
    return 0;
}


size_t mfseg_traj_split_workspace_size(int64_t n) {
    Carver cv;
    cv.take<unsigned long long>(n);
    cv.take<unsigned>(n);
    cv.take<unsigned long long>(n);
    cv.take<unsigned>(n);
    cv.take<int>(n);
    cv.take<int>(n);
    cv.take<int>(n);
    cv.take<unsigned>(n);
    cv.take<unsigned long long>(6);
    const size_t rb = radix_tmp_bytes(n > 0 ? n : 1), sb = scan_tmp_bytes(n > 0 ? n : 1);
    cv.take<char>(rb > sb ? rb : sb);
    return cv.off + 256;
}

static int traj_split_impl(int64_t n, const int64_t *traj_id, const double *t,
                           const int32_t *label, const double *stride_in, int32_t *order,
                           int32_t *run_start, int64_t *n_runs_host, double *stride_host,
                           void *workspace, size_t workspace_bytes, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n_runs_host) *n_runs_host = 0;
    if (n <= 0) return 0;
    if (n >= (1ll << 31)) {
        set_error("traj_split: more than 2^31-1 points");
        return 2;
    }
    if (workspace_bytes < mfseg_traj_split_workspace_size(n)) {
        set_error("traj_split: workspace too small");
        return 3;
    }
    Carver cv(workspace, workspace_bytes);
    unsigned long long *k0 = cv.take<unsigned long long>(n);
    unsigned *v0 = cv.take<unsigned>(n);
    unsigned long long *k1 = cv.take<unsigned long long>(n);
    unsigned *v1 = cv.take<unsigned>(n);
    int *flag = cv.take<int>(n);
    int *ex = cv.take<int>(n);
    int *incl = cv.take<int>(n);
    unsigned *trank = cv.take<unsigned>(n);
    unsigned long long *misc = cv.take<unsigned long long>(6);   // min gap, traj min / max, span, unsorted
    const size_t rb = radix_tmp_bytes(n), sb = scan_tmp_bytes(n);
    void *tmp = cv.take<char>(rb > sb ? rb : sb);
    const size_t tmpb = rb > sb ? rb : sb;
    const unsigned g = (unsigned)((n + 255) / 256);
    const unsigned long long init[5] = {0x7FF0000000000000ull, ~0ull, 0ull, 0ull, 0ull};   // +inf, min, max
    MFSEG_CUDA(cudaMemcpyAsync(misc, init, sizeof init, cudaMemcpyHostToDevice, st));
    ::mfseg::count_launch();
    k_tscan<<<148 * 4, 256, 0, st>>>(n, t, (const long long *)traj_id, misc);
    MFSEG_LAUNCH("k_tscan");
    unsigned long long h[5];
    MFSEG_CUDA(cudaMemcpyAsync(h, misc, sizeof h, cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    const bool in_order = h[4] == 0;
    int klo = 0, kbits = 1;
    if (h[3]) {
        klo = __builtin_ctzll(h[3]);
        kbits = 64 - __builtin_clzll(h[3]) - klo;
    }
    const unsigned long long kmask = kbits >= 64 ? ~0ull : ((1ull << kbits) - 1);
    // 1. sorted unique times -> stride and per-point t ranks
    ::mfseg::count_launch();
    k_tkeys<<<g, 256, 0, st>>>(n, t, klo, kmask, k0, v0);
    MFSEG_TRY(radix_sort_pairs64(k0, v0, k1, v1, n, kbits, tmp, tmpb, st));
    ::mfseg::count_launch();
    k_tunique<<<g, 256, 0, st>>>(n, k1, v1, t, flag, misc);
    MFSEG_TRY(scan_exclusive_i32(flag, ex, n, tmp, tmpb, st));
    ::mfseg::count_launch();
    k_inclusive_from_exclusive<<<g, 256, 0, st>>>(n, flag, ex, incl);
    if (!in_order) {
        ::mfseg::count_launch();
        k_trank<<<g, 256, 0, st>>>(n, incl, v1, trank);
    }
    MFSEG_LAUNCH("traj_split ranks");
    int nu = 0;
    MFSEG_CUDA(cudaMemcpyAsync(h, misc, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaMemcpyAsync(&nu, incl + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    double stride;
    memcpy(&stride, &h[0], sizeof stride);   // +inf when fewer than two unique times
    if (stride_in) stride = *stride_in;      // sharded: the stride of all ranks' times
    const long long tmin = (long long)(h[1] ^ 0x8000000000000000ull);
    const long long tmax = (long long)(h[2] ^ 0x8000000000000000ull);
    const unsigned long long range = (unsigned long long)tmax - (unsigned long long)tmin;
    int tbits = 0;
    while ((1ll << tbits) < nu) ++tbits;
    int rbits = 0;
    while (rbits < 64 && (range >> rbits) != 0) ++rbits;
    // 2. lexsort((t, traj_id)): one stable sort of (traj - min, t rank); the
    // identity when the records are in that order already
    if (in_order) {
        ::mfseg::count_launch();
        k_iota_u32<<<g, 256, 0, st>>>(n, v1);
        MFSEG_LAUNCH("k_iota_u32");
    } else if (rbits + tbits <= 64) {
        ::mfseg::count_launch();
        k_lex_keys<<<g, 256, 0, st>>>(n, (const long long *)traj_id, trank, tmin, tbits, k0, v0);
        MFSEG_TRY(radix_sort_pairs64(k0, v0, k1, v1, n, rbits + tbits > 0 ? rbits + tbits : 1, tmp,
                                     tmpb, st));
    } else {
        set_error("traj_split: trajectory id range and time count exceed 64 key bits");
        return 2;
    }
    // 3. run breaks along the sorted order and their compaction
    volatile double gap_limit = stride * (1.0 + 1e-9);   // stride * (1 + 1e-9), postproc.py:182
    ::mfseg::count_launch();
    k_traj_breaks<<<g, 256, 0, st>>>(n, v1, (const long long *)traj_id, t, label, gap_limit, flag);
    MFSEG_TRY(scan_exclusive_i32(flag, ex, n, tmp, tmpb, st));
    ::mfseg::count_launch();
    k_inclusive_from_exclusive<<<g, 256, 0, st>>>(n, flag, ex, incl);
    ::mfseg::count_launch();
    k_run_starts<<<(unsigned)((n + 256) / 256), 256, 0, st>>>(n, flag, incl, run_start);
    MFSEG_CUDA(cudaMemcpyAsync(order, v1, sizeof(unsigned) * n, cudaMemcpyDeviceToDevice, st));
    MFSEG_LAUNCH("traj_split runs");
    int nr = 0;
    MFSEG_CUDA(cudaMemcpyAsync(&nr, incl + (n - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    if (n_runs_host) *n_runs_host = nr;
    if (stride_host) *stride_host = stride;
    return 0;
}

int mfseg_traj_split(int64_t n, const int64_t *traj_id, const double *t, const int32_t *label,
                     int32_t *order, int32_t *run_start, int64_t *n_runs_host, double *stride_host,
                     void *workspace, size_t workspace_bytes, void *stream) {
    return traj_split_impl(n, traj_id, t, label, nullptr, order, run_start, n_runs_host,
                           stride_host, workspace, workspace_bytes, stream);
}

int mfseg_traj_split_stride(int64_t n, const int64_t *traj_id, const double *t,
                            const int32_t *label, double stride, int32_t *order,
                            int32_t *run_start, int64_t *n_runs_host, void *workspace,
                            size_t workspace_bytes, void *stream) {
    return traj_split_impl(n, traj_id, t, label, &stride, order, run_start, n_runs_host, nullptr,
                           workspace, workspace_bytes, stream);
}

}  // extern "C"
