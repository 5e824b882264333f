// k_field_assign5 — windowed exact assignment of field samples, one CTA per
// sample-bin block (v5, the default field kernel).
//
// Same result as the reference's _assign_chunk / _metric (engine.py:137-192)
// for every field sample: argmin over valid candidates of the fp64 D computed
// in the reference's operation order, lowest id on ties.  v5 changes where the
// work per candidate is spent (v4: assign_field.cu):
//
//  * the tile is the whole 16x16x16 voxel x 4 timestep block of one sample bin
//    (16384 samples), so the candidate list, the fp32 tables and the partial
//    sums are set up once per bin instead of once per 2048 samples;
//  * no fp64 tile-level culling: every candidate whose validity box meets the
//    block gets fp32 tables (dx^2[16] | dy^2[16] | dz^2[16] | (cf dt)^2[4],
//    each computed in fp64 exactly like the reference and rounded once; +inf
//    where |c - s| <= C fails) plus per-quad (min, max) of every axis;
//  * each warp walks the 8 bricks of its region (bricks of 8x4x4 voxels x 2
//    timesteps, 8 samples per lane): warp culling from the group tables, then
//    the linear dominance test against the best fully valid candidate.  A
//    brick left with one candidate is labelled here; a brick with several
//    (<= MULTI_MAX) is queued for k_field_screen (assign_field5b.cu), which
//    runs the per-sample fp32 screen below (packed 32-bit keys: float bits of
//    d with the low 7 mantissa bits replaced by the candidate, so the top-2
//    update is three integer min/max) and the certification;
//  * partial sums: per slot 16-bit count marginals in shared memory (x, y, z,
//    t indices; shared-memory integer atomics) and the value sums as 24-bit
//    shared limbs of the bricks' per-run fixed-point sums; once per block the
//    marginals x 128-bit fixed-point coordinates and the limbs go to the
//    global 128-bit sums.
//
// Error analysis of the screen (all table terms >= 0):
//   s = (((Tx + Ty) + Tz) + Tt) has 4 fp32 rounded table terms and 3 fp32
//   additions -> s = S (1 + th), |th| <= 4.0001 * 2^-24; sqrt.approx adds
//   <= 2^-22.4 relative, fwd = fl(wd) and the final fma 2^-24 each, the value
//   term w_v |fl(v) - fl(cv)| is within 3 * 2^-24 w_v (|v| + |cv|) absolute.
//   Hence |d32 - D| <= 2^-20 (D + W), W = w_v (|v| + max|cv|) + slack, well
//   inside the 2^-19 bound the margins below assume (KSCR = 2^-18 is twice it).
//   Packed keys truncate d to t with t <= d < t (1 + 2^-16); certification uses
//   u1 = fl(t1 (1 + 2^-15)) >= d1 for the best and t2 <= d for every other
//   candidate, so a certified best is the exact argmin.  Anything else
//   (near ties, overflow to +inf) is re-evaluated in exact fp64 over every
//   kept candidate within the margin.  Warp culling is exact-safe for the same
//   reasons as v4 (margin 2^-16 >> the fp32 error of the bounds).
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr float INF_F = __builtin_huge_valf();
constexpr float FLT_BIG = 3.4028234663852886e38f;

constexpr int BX = 16, BY = 16, BZ = 16, BT = 4;   // block = one bin's 16^3 x 4 samples (at most)
constexpr int NT = 256, NW = 8;
constexpr int CAP = 128;                           // candidates per block (more: deferred)
constexpr unsigned SLOT_MASK = 127u;               // 7 slot bits in the packed keys
constexpr int TE = BX + BY + BZ + BT;              // 52 table entries per candidate
constexpr int OZ = BX + BY, OT = BX + BY + BZ;     // table offsets of z and t
constexpr int GX = 8, GY = 4, GZ = 4, GT = 2;      // brick: 8x4x4 voxels x 2 timesteps
constexpr int QY = BX / GX, QZ = QY + BY / GY, QT = QZ + BZ / GZ;
constexpr int NQ = QT + BT / GT;                   // brick-row groups: x 2, y 4, z 4, t 2
constexpr int HW = 27;                             // histogram words: x 8, y 8, z 8, t 2, n 1
static_assert(MULTI_MAX <= 32, "one lane per kept candidate in k_field_screen");
constexpr float KCULL = 0x1.0p-16f;

struct Ctx {
    AxisTile X, Y, Z, T;
    int cnt, nrounds;
    bool deferred;
    float cvmax, fwd, wvf, slack;
    long long plane, vol;
};

struct __align__(16) Smem5 {
    float tab[CAP][TE];             // 16-byte aligned rows (52 floats)
    float2 qmm[CAP][NQ];            // (min, max) of each quad of table entries
    double c[CAP][5];               // cx, cy, cz, ct, cv (0 when absent)
    unsigned vlimb[CAP][6];         // per slot value sum: 128-bit fixed point in 24-bit limbs
    unsigned hist[CAP][HW];         // 16-bit count marginals, two per word
    unsigned long long xf[BX][2], yf[BY][2], zf[BZ][2], tf[BT][2];
    double x[BX], y[BY], z[BZ], t[BT];
    int id[CAP];
    unsigned box[CAP];              // x 4+4 | y 4+4 | z 4+4 | t 2+2 bits
    float cvf[CAP], wvf[CAP];
    unsigned char has[CAP];
    int wc[NW];
    float red[NW];
    int cidx[CAP];                  // block cache: entry of each slot (-1: absent)
    int cnz;
    int lst[NW][32];                // per region: candidate slots that survive its cull
    int nlist[NW];                  // list lengths (-1: more than 32 survivors)
    unsigned char bslot[64];        // reused bricks: slot of their label (255: recompute)
    float rcg[NW];                  // per region: min over its culled candidates of dl (1-2^-16) - 2^-15 Wb
    float red2[NW];
    float dmax;                     // largest metric change of the block's candidates
    ulonglong2 bsums[64];           // per reused brick: its per-run value sum (prologue)
    Ctx ctx;
};

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float to_f(double x) { return fminf(__double2float_rn(x), FLT_BIG); }
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// warp min / max by one REDUX: non-negative floats order like their bit
// patterns; general floats through an order-preserving bit transform
__device__ __forceinline__ float warp_min_nn(float v) {
    return __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ float warp_max_nn(float v) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ unsigned f2ord(float v) {
    const unsigned b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ float warp_min_any(float v) {
    return ord2f(__reduce_min_sync(0xffffffffu, f2ord(v)));
}
__device__ __forceinline__ float warp_max_any(float v) {
    return ord2f(__reduce_max_sync(0xffffffffu, f2ord(v)));
}
__device__ __forceinline__ __int128 get128(const unsigned long long *p) {
    return (__int128)(((unsigned __int128)p[1] << 64) | (unsigned __int128)p[0]);
}
__device__ __forceinline__ int hget(const unsigned *h, int i) {   // 16-bit counter i
    return (int)((h[i >> 1] >> (16 * (i & 1))) & 0xFFFFu);
}

// warp-aggregated append of this lane's `n` entries to a global list
__device__ __forceinline__ long long warp_reserve(unsigned long long *counter, int n) {
    const int lane = threadIdx.x & 31;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total > 0) base = atomicAdd(counter, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    return (long long)base + incl - n;
}

}  // namespace


// One table row: entries e[i] = fl32((s (c - coord[i]))^2) (fp64 as the reference,
// s = c_f for time) inside the validity box [lo, hi], +inf outside, and the
// (min, max) of each group of G entries over the indices that exist (< len).
template <int N, int G>
__device__ __forceinline__ void table_row(float *e, float2 *mm, const double *coord, double cc,
                                          double scale, bool scaled, unsigned lo, unsigned hi,
                                          int len) {
#pragma unroll 1
    for (int g = 0; g < N / G; ++g) {   // rolled over groups: small setup code (I-cache)
        float mn = INF_F, mx = 0.0f;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int i = g * G + j;
            float val = INF_F;
            if ((unsigned)i >= lo && (unsigned)i <= hi) {
                double d = DSUB(cc, coord[i]);
                if (scaled) d = DMUL(scale, d);
                val = to_f(DMUL(d, d));
            }
            e[i] = val;
            if (i < len) {
                mn = fminf(mn, val);
                mx = fmaxf(mx, val);
            }
        }
        mm[g] = make_float2(mn, mx);
    }
}


// Add one fp64 value sum to a slot's exact 128-bit fixed-point total kept as
// six 24-bit limbs in 32-bit shared counters (the top one signed): integer,
// order-free, and at most 64 records per slot and block, so no counter overflows.
__device__ __forceinline__ void add_fix_limbs(unsigned *lim, unsigned long long lo, long long hi) {
    const unsigned M = 0xFFFFFFu;
    atomicAdd(&lim[0], (unsigned)(lo & M));
    atomicAdd(&lim[1], (unsigned)((lo >> 24) & M));
    atomicAdd(&lim[2], (unsigned)(((lo >> 48) | ((unsigned long long)hi << 16)) & M));
    atomicAdd(&lim[3], (unsigned)(((unsigned long long)hi >> 8) & M));
    atomicAdd(&lim[4], (unsigned)(((unsigned long long)hi >> 32) & M));
    atomicAdd((int *)&lim[5], (int)(hi >> 56));
}

__device__ __forceinline__ void add_value_limbs(unsigned *lim, double v, int &ovf) {
    unsigned long long lo;
    long long hi;
    d2fix(v, lo, hi, &ovf);
    add_fix_limbs(lim, lo, hi);
}

__device__ __forceinline__ __int128 value_limbs_total(const unsigned *lim) {
    __int128 acc = (__int128)((int)lim[5]) << 120;
#pragma unroll
    for (int k = 0; k < 5; ++k) acc += (__int128)((unsigned __int128)lim[k] << (24 * k));
    return acc;
}

// One warp brick: lane (lx, ly) = (8 bx + lane % 8, 4 by + lane / 8), samples
// k = 4 r + q at z = 4 bz + q, timestep 2 bt + r.  FULL: all 256 samples exist.

// (min, max) over table groups [g0, g1]
__device__ __forceinline__ float2 gmm(const float2 *m, int g0, int g1) {
    float2 r = m[g0];
    for (int g = g0 + 1; g <= g1; ++g) {
        r.x = fminf(r.x, m[g].x);
        r.y = fmaxf(r.y, m[g].y);
    }
    return r;
}

// Warp region = the 8 bricks of warp w: x half rbx, y quarter rby, every z and
// timestep of the block.  Cull the block's candidates over the whole region
// (bounds from the group tables, value range of the block) and compact the
// survivors into S.lst[w]: a candidate culled here is beaten by the region's
// best fully valid candidate on every sample of every brick of the region.
// Returns the list length, or -1 when more than 32 survive.
template <bool USEVAL, int NR>
__device__ __forceinline__ int region_list(Smem5 &S, const Ctx &C, int rbx, int rby, int zg0, int zg1,
                                           int tg0, int tg1, float vl, float vh, int debug) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float fwd = C.fwd, wvf = C.wvf;
    float dl[4] = {INF_F, INF_F, INF_F, INF_F};
    float ubw = INF_F;
#pragma unroll 1
    for (int r = 0; r < NR; ++r) {   // rolled: smaller code next to the hot brick loop
        float dlr = INF_F;
        const int s = lane + 32 * r;
        if (r < C.nrounds && s < C.cnt) {
            const float2 qx = S.qmm[s][rbx], qy = S.qmm[s][QY + rby];
            const float2 qz = gmm(S.qmm[s] + QZ, zg0, zg1), qt = gmm(S.qmm[s] + QT, tg0, tg1);
            float vtl = 0.0f, vth = 0.0f;
            if (USEVAL) {
                const float wvs = S.wvf[s];
                if (wvs > 0.0f) {
                    const float cvs = S.cvf[s];
                    const float pl = vl - cvs, ph = vh - cvs;   // pl <= ph
                    vtl = wvs * fmaxf(fmaxf(pl, -ph), 0.f);
                    vth = wvs * fmaxf(ph, -pl);
                }
            }
            dlr = fmaf(fwd, sqrt_approx((qx.x + qy.x) + (qz.x + qt.x)), vtl);
            ubw = fminf(ubw, fmaf(fwd, sqrt_approx((qx.y + qy.y) + (qz.y + qt.y)), vth));
        }
        if (r == 0) dl[0] = dlr;
        else if (r == 1) dl[1] = dlr;
        else if (r == 2) dl[2] = dlr;
        else dl[3] = dlr;
    }
    ubw = warp_min_nn(ubw);
    const float Wb = (USEVAL ? wvf * (fmaxf(fabsf(vl), fabsf(vh)) + C.cvmax) : 0.f) + C.slack;
    const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) * (1.f + 0x1.0p-15f);
    unsigned keep[4] = {0u, 0u, 0u, 0u};
    int total = 0;
    float rc = INF_F;   // smallest lower bound among the culled candidates (margin reuse)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const bool k = dl[r] < INF_F && (dl[r] <= thr || (debug & 1));
        keep[r] = __ballot_sync(0xffffffffu, k);
        total += __popc(keep[r]);
        if (!k && dl[r] < INF_F) rc = fminf(rc, dl[r]);
    }
    rc = warp_min_nn(rc);
    if (lane == 0) S.rcg[w] = rc < INF_F ? rc * (1.f - 0x1.0p-16f) - 0x1.0p-15f * Wb : INF_F;
    if (total > 32) return -1;
    int base = 0;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        if (keep[r] >> lane & 1u) S.lst[w][base + __popc(keep[r] & ((1u << lane) - 1u))] = lane + 32 * r;
        base += __popc(keep[r]);
    }
    __syncwarp();
    return total;
}

// NR: rounds of 32 candidate slots (3 when the block has <= 96 candidates: the
// common case gets a smaller instruction footprint)
// LIST: the candidates are the warp region's list S.lst[w][0..nlist) (one round,
// bit b of a keep mask = list position b); otherwise slot = bit + 32 * round.
// A whole brick labelled by one slot: the count marginals are constants and the
// value sum is the brick's (fixed-order warp sum, computed once per run).
// Partial sums of a brick labelled by one slot: count marginals from its live
// extents (ex x ey x ez x et samples; a brick cut by the block edge -- or by a
// thin grid, e.g. nz = 1 -- has fewer) and the brick's per-run value sum.
__device__ __forceinline__ void single_brick_sums(Smem5 &S, ulonglong2 vs, int one,
                                                  int bx, int by, int bz, int bt, int ex, int ey,
                                                  int ez, int et) {
    const int lane = threadIdx.x & 31;
    unsigned *h = S.hist[one];
    if (lane < 10) {   // count marginals: two 16-bit counts (indices i0, i0 + 1) per word
        const bool full = ex == GX && ey == GY && ez == GZ && et == GT;   // constant counts
        auto pair = [](int i0, int e, unsigned c) {
            return (i0 < e ? c : 0u) | ((i0 + 1 < e ? c : 0u) << 16);
        };
        if (lane < 4) {                                                      // 8 x
            const unsigned w = full ? (32u | (32u << 16)) : pair(2 * lane, ex, (unsigned)(ey * ez * et));
            if (w) atomicAdd(&h[4 * bx + lane], w);
        } else if (lane < 6) {                                               // 4 y
            const unsigned w = full ? (64u | (64u << 16))
                                    : pair(2 * (lane - 4), ey, (unsigned)(ex * ez * et));
            if (w) atomicAdd(&h[8 + 2 * by + (lane - 4)], w);
        } else if (lane < 8) {                                               // 4 z
            const unsigned w = full ? (64u | (64u << 16))
                                    : pair(2 * (lane - 6), ez, (unsigned)(ex * ey * et));
            if (w) atomicAdd(&h[16 + 2 * bz + (lane - 6)], w);
        } else if (lane == 8) {                                              // 2 timesteps
            atomicAdd(&h[24 + bt], full ? (128u | (128u << 16)) : pair(0, et, (unsigned)(ex * ey * ez)));
        } else {
            atomicAdd(&h[26], full ? 256u : (unsigned)(ex * ey * ez * et));
        }
    } else if (lane < 16) {   // the six value-sum limbs, one per lane
        const int q = lane - 10;
        const unsigned long long lo = vs.x, hi = vs.y;
        const unsigned long long bits = q < 2 ? lo >> (24 * q)
                                      : q == 2 ? (lo >> 48) | (hi << 16)
                                               : hi >> (24 * q - 64);
        atomicAdd(&S.vlimb[one][q], q < 5 ? (unsigned)(bits & 0xFFFFFFu) : (unsigned)(bits & 0xFFu) |
                                                ((bits & 0x80u) ? 0xFFFFFF00u : 0u));
    }
}

// A run of nb full bricks of one warp labelled by one slot (the warp's bricks
// share bx and by; zc / tc count them per bz / bt): their count marginals and
// summed per-run value sums in one set of shared atomics (single_brick_sums per
// brick would issue nb sets).  Integer sums: the totals are the same.
// (rc packs 4-bit counts: bz = 0..3 in bits 0-15, bt = 0..1 in 16-23, nb in 24-27)
__device__ __forceinline__ void run_brick_sums(Smem5 &S, int one, int bx, int by, unsigned rc,
                                               unsigned long long vlo, unsigned long long vhi) {
    const int lane = threadIdx.x & 31;
    const unsigned nb = (rc >> 24) & 15u;
    unsigned *h = S.hist[one];
    auto two = [](unsigned c) { return c | (c << 16); };
    if (lane < 4) {                                      // 8 x: 32 samples per brick each
        atomicAdd(&h[4 * bx + lane], two(32u * nb));
    } else if (lane < 6) {                               // 4 y: 64 each
        atomicAdd(&h[8 + 2 * by + (lane - 4)], two(64u * nb));
    } else if (lane < 14) {                              // 4 z per bz: 64 each
        const int bz = (lane - 6) >> 1;
        const unsigned c = (rc >> (4 * bz)) & 15u;
        if (c) atomicAdd(&h[16 + 2 * bz + ((lane - 6) & 1)], two(64u * c));
    } else if (lane < 16) {                              // 2 timesteps per bt: 128 each
        const unsigned c = (rc >> (16 + 4 * (lane - 14))) & 15u;
        if (c) atomicAdd(&h[24 + (lane - 14)], two(128u * c));
    } else if (lane == 16) {
        atomicAdd(&h[26], 256u * nb);
    } else if (lane < 23) {                              // the six value-sum limbs
        const int q = lane - 17;
        const unsigned long long bits = q < 2 ? vlo >> (24 * q)
                                      : q == 2 ? (vlo >> 48) | (vhi << 16)
                                               : vhi >> (24 * q - 64);
        atomicAdd(&S.vlimb[one][q], q < 5 ? (unsigned)(bits & 0xFFFFFFu) : (unsigned)(bits & 0xFFu) |
                                                ((bits & 0x80u) ? 0xFFFFFF00u : 0u));
    }
}

// Every live sample of a brick labelled `lab` (the initial pass's interior blocks).
__device__ __forceinline__ void label_brick(const FieldArgs &a, const Ctx &C, int bx, int by, int bz,
                                            int bt, int lab) {
    const int lane = threadIdx.x & 31;
    const int lx = GX * bx + (lane & 7), ly = GY * by + (lane >> 3);
    const int z0 = GZ * bz, t0 = GT * bt;
    if (lx >= C.X.len || ly >= C.Y.len) return;
    int *lab_base = a.labels + (((long long)(C.T.start + t0) * a.nz + C.Z.start + z0) * a.ny +
                                (C.Y.start + ly)) * (long long)a.nx + (C.X.start + lx);
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (z0 + (k & 3) < C.Z.len && t0 + (k >> 2) < C.T.len) lab_base[(k & 3) * C.plane + (k >> 2) * C.vol] = lab;
}

// Every sample of a brick to the exact per-sample path (k_deferred, label -2).
__device__ __forceinline__ void defer_brick(const FieldArgs &a, const Ctx &C, int bx, int by, int bz, int bt) {
    const int lane = threadIdx.x & 31;
    const int lx = GX * bx + (lane & 7), ly = GY * by + (lane >> 3);
    const int z0 = GZ * bz, t0 = GT * bt;
    const long long fbase = (((long long)(C.T.start + t0) * a.nz + C.Z.start + z0) * a.ny +
                             (C.Y.start + ly)) * (long long)a.nx + (C.X.start + lx);
    unsigned livem = 0;
    if (lx < C.X.len && ly < C.Y.len) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (z0 + (k & 3) < C.Z.len && t0 + (k >> 2) < C.T.len) livem |= 1u << k;
    }
    int *lab_base = a.labels + fbase;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (livem >> k & 1) lab_base[(k & 3) * C.plane + (k >> 2) * C.vol] = -2;
    long long p = warp_reserve(a.n_deferred, __popc(livem));
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (livem >> k & 1) {
            if (p < a.deferred_cap) a.deferred[p] = fbase + (k & 3) * C.plane + (k >> 2) * C.vol;
            ++p;
        }
}

// Returns the brick's slot when it is FULL and labelled by one slot (the caller
// sums it in its run), -1 when it is labelled by one slot and summed here, -2
// when it is not (queued for k_field_screen, deferred or stranded).
template <bool USEVAL, bool FULL, int NR, bool LIST>
__device__ __forceinline__ int brick(const FieldArgs &a, Smem5 &S, const Ctx &C, int bi, int bx,
                                      int by, int bz, int bt, int region, int nlist, int &ovf_local) {
    const int lane = threadIdx.x & 31;
    const int lx = GX * bx + (lane & 7), ly = GY * by + (lane >> 3);
    const int z0 = GZ * bz, t0 = GT * bt;
    const long long fbase = (((long long)(C.T.start + t0) * a.nz + C.Z.start + z0) * a.ny +
                             (C.Y.start + ly)) * (long long)a.nx + (C.X.start + lx);
    unsigned livem = 0xFFu;
    if (!FULL) {
        livem = 0;
        if (lx < C.X.len && ly < C.Y.len) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (z0 + (k & 3) < C.Z.len && t0 + (k >> 2) < C.T.len) livem |= 1u << k;
        }
    }
    // Values are loaded only where they are needed: bricks left with several
    // candidates (per-sample screen) and bricks cut by the block edge.  Bricks
    // labelled by one candidate use the per-run brick value range and value
    // sum (k_brick_pre: the field values do not change between passes).
    const size_t bidx = (size_t)blockIdx.x * 64 + bi;
    // live extents of the brick (all full unless the block edge cuts it)
    const int ex = FULL ? GX : min(GX, C.X.len - GX * bx), ey = FULL ? GY : min(GY, C.Y.len - GY * by);
    const int ez = FULL ? GZ : min(GZ, C.Z.len - GZ * bz), et = FULL ? GT : min(GT, C.T.len - GT * bt);

    int sl[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sl[k] = -1;
    int one = -1;   // slot when a single candidate labels the whole brick (warp-uniform)
    const float fwd = C.fwd, wvf = C.wvf, slack = C.slack, cvmax = C.cvmax;
    if (!C.deferred && C.cnt > 0) {
        // brick value range: min/max of fl(v) = fl(min/max of v) (rounding is monotone)
        float vwl = 0.0f, vwh = 0.0f;
        if (USEVAL) {
            const float2 r = a.brange[bidx];
            vwl = r.x;
            vwh = r.y;
        }
        // ---- warp culling from the group (min, max) tables
        float dl[4], shi[4];
        float ubw = INF_F;
        unsigned ubkey = 0xFFFFFFFFu;   // (ub | slot) of the best fully valid candidate
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            dl[r] = INF_F;
            shi[r] = INF_F;
            const int s = LIST ? (lane < nlist ? S.lst[region][lane] : -1) : lane + 32 * r;
            if (LIST ? s >= 0 : (r < C.nrounds && s < C.cnt)) {
                const float2 qx = S.qmm[s][bx], qy = S.qmm[s][QY + by], qz = S.qmm[s][QZ + bz],
                             qt = S.qmm[s][QT + bt];
                float vtl = 0.0f, vth = 0.0f;
                if (USEVAL) {
                    const float wvs = S.wvf[s];
                    if (wvs > 0.0f) {
                        const float cvs = S.cvf[s];
                        const float pl = vwl - cvs, ph = vwh - cvs;   // pl <= ph
                        vtl = wvs * fmaxf(fmaxf(pl, -ph), 0.f);
                        vth = wvs * fmaxf(ph, -pl);
                    }
                }
                dl[r] = fmaf(fwd, sqrt_approx((qx.x + qy.x) + (qz.x + qt.x)), vtl);
                shi[r] = (qx.y + qy.y) + (qz.y + qt.y);
                const float ub = fmaf(fwd, sqrt_approx(shi[r]), vth);
                ubw = fminf(ubw, ub);
                if (ub < INF_F) ubkey = min(ubkey, (__float_as_uint(ub) & ~SLOT_MASK) | (unsigned)s);
            }
        }
        ubw = warp_min_nn(ubw);
        const float Wb = (USEVAL ? wvf * (fmaxf(fabsf(vwl), fabsf(vwh)) + cvmax) : 0.f) + slack;
        const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) * (1.f + 0x1.0p-15f);
        unsigned keep[4] = {0u, 0u, 0u, 0u}, keep0[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            keep[r] = __ballot_sync(0xffffffffu, dl[r] < INF_F && (dl[r] <= thr || (a.debug & 1)));
            keep0[r] = keep[r];
        }

        // ---- dominance: drop kept candidates s with D(s) > D(s*) on the whole brick,
        // s* = the fully valid candidate with the smallest upper bound.  The squared
        // distance difference is linear in each coordinate, so its minimum over the
        // brick is the sum over axes of the smaller endpoint difference (fp32 table
        // values, margin 2^-20 (S_s + S_s*) >> their rounding); the sqrt gap is at
        // least dS / (sqrt S_s,max + sqrt S_s*,max); the value terms differ by at
        // least w_v min(f(v_lo), f(v_hi)), f(v) = |v - cv_s| - |v - cv_s*| (both have
        // values; f is monotone in v), or -w_v max|v - cv_s*| (only s* has one).
        ubkey = __reduce_min_sync(0xffffffffu, ubkey);
        if (DEVICE_STATS(a) && lane == 0) {
            const int nc = __popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]);
            atomicAdd(a.stats + 7, (unsigned long long)nc);
            if (nc == 1) atomicAdd(a.stats + 2, 1ull);
        }
        int sstar = -1;
        float gmin = INF_F;   // smallest proven gap D_s - D_s* among the dominated candidates
        if (ubkey != 0xFFFFFFFFu && !(a.debug & 1)) {
            sstar = (int)(ubkey & SLOT_MASK);
            const int xa = GX * bx, ya = GY * by, za = GZ * bz, ta = GT * bt;
            const int xb = FULL ? xa + GX - 1 : min(xa + GX - 1, C.X.len - 1);
            const int yb = FULL ? ya + GY - 1 : min(ya + GY - 1, C.Y.len - 1);
            const int zb = FULL ? za + GZ - 1 : min(za + GZ - 1, C.Z.len - 1);
            const int tb = FULL ? ta + GT - 1 : min(ta + GT - 1, C.T.len - 1);
            const float *Q = S.tab[sstar];
            const float qx0 = Q[xa], qx1 = Q[xb], qy0 = Q[BX + ya], qy1 = Q[BX + yb];
            const float qz0 = Q[OZ + za], qz1 = Q[OZ + zb], qt0 = Q[OT + ta], qt1 = Q[OT + tb];
            const float2 mqx = S.qmm[sstar][bx], mqy = S.qmm[sstar][QY + by], mqz = S.qmm[sstar][QZ + bz],
                         mqt = S.qmm[sstar][QT + bt];
            const float shq = (mqx.y + mqy.y) + (mqz.y + mqt.y);
            const float rq = sqrt_approx(shq);
            float cvq = 0.f, wvq = 0.f;
            if (USEVAL) {
                cvq = S.cvf[sstar];
                wvq = S.wvf[sstar];
            }
            const float vabs = fmaxf(fabsf(vwl), fabsf(vwh));
            const float vq = fmaxf(fabsf(vwl - cvq), fabsf(vwh - cvq));
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int s = LIST ? (lane < nlist ? S.lst[region][lane] : -1) : lane + 32 * r;
                bool dom = false;
                float gd = INF_F;
                if ((keep[r] >> lane & 1u) && s != sstar) {
                    const float *T = S.tab[s];
                    float dS = -INF_F, shs = shi[r];   // -inf: no proof possible
                    {
                        const float ex0 = T[xa], ex1 = T[xb], ey0 = T[BX + ya], ey1 = T[BX + yb];
                        const float ez0 = T[OZ + za], ez1 = T[OZ + zb], et0 = T[OT + ta], et1 = T[OT + tb];
                        const float emax = fmaxf(fmaxf(fmaxf(ex0, ex1), fmaxf(ey0, ey1)),
                                                 fmaxf(fmaxf(ez0, ez1), fmaxf(et0, et1)));
                        if (emax < INF_F)   // valid on the whole brick (windows are intervals)
                            dS = (fminf(ex0 - qx0, ex1 - qx1) + fminf(ey0 - qy0, ey1 - qy1)) +
                                 (fminf(ez0 - qz0, ez1 - qz1) + fminf(et0 - qt0, et1 - qt1));
                    }
                    if (dS == -INF_F) {
                        // valid on part of the brick only: s can win only where it is valid,
                        // so the dominance is proven over the brick's intersection with its
                        // validity box (index intervals per axis; squared distances peak at
                        // the interval ends, their differences are linear)
                        const unsigned b = S.box[s];
                        const int ia = max(xa, (int)(b & 15u)), ib = min(xb, (int)((b >> 4) & 15u));
                        const int ja = max(ya, (int)((b >> 8) & 15u)), jb = min(yb, (int)((b >> 12) & 15u));
                        const int ka = max(za, (int)((b >> 16) & 15u)), kb = min(zb, (int)((b >> 20) & 15u));
                        const int ma = max(ta, (int)((b >> 24) & 3u)), mb = min(tb, (int)((b >> 26) & 3u));
                        if (ia <= ib && ja <= jb && ka <= kb && ma <= mb) {
                            const float *Q = S.tab[sstar];
                            const float e0 = T[ia], e1 = T[ib], f0 = T[BX + ja], f1 = T[BX + jb];
                            const float g0 = T[OZ + ka], g1 = T[OZ + kb], h0 = T[OT + ma], h1 = T[OT + mb];
                            shs = (fmaxf(e0, e1) + fmaxf(f0, f1)) + (fmaxf(g0, g1) + fmaxf(h0, h1));
                            if (shs < INF_F)
                                dS = (fminf(e0 - Q[ia], e1 - Q[ib]) + fminf(f0 - Q[BX + ja], f1 - Q[BX + jb])) +
                                     (fminf(g0 - Q[OZ + ka], g1 - Q[OZ + kb]) +
                                      fminf(h0 - Q[OT + ma], h1 - Q[OT + mb]));
                        }
                    }
                    if (dS > -INF_F) {
                        const float dSlb = dS - 0x1.0p-20f * (shs + shq);
                        if (dSlb > 0.f) {
                            const float den = (sqrt_approx(shs) + rq) * (1.f + 0x1.0p-20f);
                            const float gap = __fdividef(dSlb, den) * (1.f - 0x1.0p-19f);
                            float Vb = 0.f;
                            if (USEVAL && wvq > 0.f) {
                                // both with values: |v - cv_s| - |v - cv_s*| is monotone in v,
                                // so its minimum over the brick's value range is at an end
                                const float cvs = S.cvf[s];
                                const float V = S.wvf[s] > 0.f
                                    ? wvf * fmaxf(0.f, -fminf(fabsf(vwl - cvs) - fabsf(vwl - cvq),
                                                              fabsf(vwh - cvs) - fabsf(vwh - cvq)))
                                    : wvf * vq;
                                Vb = V * (1.f + 0x1.0p-18f) +
                                     0x1.0p-18f * wvf * (fabsf(cvs) + fabsf(cvq) + vabs);
                            }
                            const float rel = 0x1.0p-30f * (fwd * den + Wb) + slack;
                            gd = fwd * gap * (1.f - 0x1.0p-20f) - (Vb + rel);
                            dom = gd > 0.f;
                        }
                    }
                }
                keep[r] &= ~__ballot_sync(0xffffffffu, dom);
                if (dom) gmin = fminf(gmin, gd);
            }
        }
        if (DEVICE_STATS(a) && lane == 0 && sstar < 0) atomicAdd(a.stats + 30, 1ull);   // no s*
        if (DEVICE_STATS(a) && lane == 0) {
            atomicAdd(a.stats, 1ull);
            atomicAdd(a.stats + 1, (unsigned long long)(__popc(keep[0]) + __popc(keep[1]) +
                                                         __popc(keep[2]) + __popc(keep[3])));
        }

        const int nkeep = __popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]);
        if (nkeep == 1 && sstar >= 0) {
            // s* is valid on the whole brick and every other candidate is culled or
            // dominated: it is the exact argmin of every sample
#pragma unroll
            for (int k = 0; k < 8; ++k) sl[k] = (livem >> k & 1) ? sstar : -1;
            one = sstar;
            if (a.bmargin) {
                // proven lower bound of D_s - D_s* over the brick for every other
                // candidate: culled (lower bound minus s*'s upper bound, with the
                // cull's error allowances), region-culled, or dominated (its gap)
                float cm = INF_F;
#pragma unroll
                for (int r = 0; r < NR; ++r)
                    if (!(keep0[r] >> lane & 1u) && dl[r] < INF_F) cm = fminf(cm, dl[r]);
                cm = warp_min_nn(cm);
                gmin = warp_min_nn(gmin);
                const float ubs = ubw * (1.f + 0x1.0p-15f) * (1.f + 0x1.0p-16f);
                float m = gmin;
                if (cm < INF_F) m = fminf(m, cm * (1.f - 0x1.0p-16f) - ubs - 0x1.0p-15f * Wb);
                const float rg = S.rcg[region];
                if (rg < INF_F) m = fminf(m, rg - ubs - 0x1.0p-15f * Wb);
                if (lane == 0) a.bmargin[bidx] = m - 1e-6f * (fwd + wvf) - slack;
            }
        } else {
            // several survivors: the per-sample screen runs in k_field_screen (one
            // warp per brick, kept candidates by global id), keeping this kernel lean;
            // more than MULTI_MAX survivors or a full queue: exact per-sample path
            unsigned long long item = ~0ull;
            if (lane == 0 && nkeep <= MULTI_MAX) item = atomicAdd(a.n_multi, 1ull);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item < (unsigned long long)a.multi_cap) {
            MultiItem &it = a.multi[item];
            int pos = 0;
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const unsigned kr = keep[r];
                if (kr >> lane & 1u) {
                    const int slot = LIST ? S.lst[region][lane] : lane + 32 * r;
                    it.id[pos + __popc(kr & ((1u << lane) - 1u))] = S.id[slot];
                }
                pos += __popc(kr);
            }
            if (lane == 0) {
                it.x0 = C.X.start + GX * bx;
                it.y0 = C.Y.start + GY * by;
                it.z0 = C.Z.start + GZ * bz;
                it.t0 = C.T.start + GT * bt;
                it.meta = nkeep | min(GX, C.X.len - GX * bx) << 8 | min(GY, C.Y.len - GY * by) << 12 |
                          min(GZ, C.Z.len - GZ * bz) << 16 | min(GT, C.T.len - GT * bt) << 20;
            }
            return -2;
            }
            int nd = 0;
            int *lab_base = a.labels + fbase;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (livem >> k & 1) {
                    lab_base[(k & 3) * C.plane + (k >> 2) * C.vol] = -2;
                    ++nd;
                }
            long long p = warp_reserve(a.n_deferred, nd);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (livem >> k & 1) {
                    if (p < a.deferred_cap) a.deferred[p] = fbase + (k & 3) * C.plane + (k >> 2) * C.vol;
                    ++p;
                }
            return -2;
        }
    }

    // ---- labels; deferred / stranded samples to their lists (warp-aggregated)
    int *lab_base = a.labels + fbase;
    if (one >= 0) {
        const int lab = S.id[one];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (FULL || (livem >> k & 1)) lab_base[(k & 3) * C.plane + (k >> 2) * C.vol] = lab;
        if (lane == 0 && a.bslot) {
            a.bslot[bidx] = (unsigned char)one;
            if (a.bcid) a.bcid[bidx] = lab;
        }
        if (FULL) return one;   // the caller adds it to its warp's run of full bricks
        if (a.accumulate) single_brick_sums(S, a.bsum[bidx], one, bx, by, bz, bt, ex, ey, ez, et);
        return -1;
    }
    int nout = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {   // no candidate for the brick: deferred block or stranded
        if (!FULL && !(livem >> k & 1)) continue;
        lab_base[(k & 3) * C.plane + (k >> 2) * C.vol] = C.deferred ? -2 : -1;
        ++nout;
    }
    if (__any_sync(0xffffffffu, nout > 0)) {
        unsigned long long *ctr = C.deferred ? a.n_deferred : a.n_stranded;
        long long *lst = C.deferred ? a.deferred : a.stranded;
        const long long cap = C.deferred ? a.deferred_cap : a.stranded_cap;
        long long p = warp_reserve(ctr, nout);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (!(livem >> k & 1)) continue;
            if (p < cap) lst[p] = fbase + (k & 3) * C.plane + (k >> 2) * C.vol;
            ++p;
        }
    }

    // (no partial sums here: a brick labelled by one slot returned above with its
    // per-run sums; the others are stranded or deferred and summed where resolved)
    return -2;
}

template <bool USEVAL, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_field_assign5(FieldArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem5 &S = *reinterpret_cast<Smem5 *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    __shared__ int tix[4];   // the block's axis tiles: one thread decodes the block index
    if (tid == 0) {
        unsigned tile = blockIdx.x;
        tix[0] = (int)(tile % (unsigned)a.ntx);
        tile /= (unsigned)a.ntx;
        tix[1] = (int)(tile % (unsigned)a.nty);
        tile /= (unsigned)a.nty;
        tix[2] = (int)(tile % (unsigned)a.ntz);
        tix[3] = (int)(tile / (unsigned)a.ntz);
    }
    __syncthreads();
    const AxisTile X = a.xt[tix[0]], Y = a.yt[tix[1]], Z = a.zt[tix[2]], Tm = a.tt[tix[3]];
    int ovf_local = 0;
    // the bricks' reuse state of the last pass, loaded now (no dependence on the
    // candidates): the latency overlaps the block setup below
    unsigned char pf_sl = 255;
    ulonglong2 pf_bs = make_ulonglong2(0ull, 0ull);
    float pf_mg = 0.f;
    int pf_cid = 0;
    if (tid < 64 && (a.reuse || a.seeds_fast)) {
        const size_t bidx = (size_t)blockIdx.x * 64 + tid;
        if (a.bslot) pf_sl = a.bslot[bidx];
        if (a.accumulate) pf_bs = a.bsum[bidx];
        if (a.bmargin) pf_mg = a.bmargin[bidx];
        if (a.bcid && a.bcache) pf_cid = a.bcid[bidx];
    }

    // ---- a block whose every brick keeps its label: its sums are those of the pass
    // that labelled it (block cache), added without the block setup.  The margin
    // test is the one below with the largest move over all the bin's candidates
    // (a superset of the block's: never looser)
    if (a.bcache && a.reuse && !a.seeds_fast && a.accumulate) {
        const int sbin0 = ((Tm.bin * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;
        const int bn = a.bin_sstable[sbin0] ? a.bcache[blockIdx.x].n : -1;
        const int L0 = a.g.cand_start[sbin0], L1 = a.g.cand_start[sbin0 + 1];
        if (bn >= 0 && L1 - L0 <= NT) {
            const bool stable = a.bin_stable[sbin0];
            const float dmax = stable ? 0.f : a.bin_dmax[sbin0];
            const int bx = tid & 1, by = (tid >> 1) & 3, bz = (tid >> 3) & 3, bt = tid >> 5;
            const bool live = tid < 64 && !(GX * bx >= X.len || GY * by >= Y.len || GZ * bz >= Z.len ||
                                            GT * bt >= Tm.len);
            float dec = 0.f;
            bool ok = !live || pf_sl != 255;
            if (live && ok && !stable) {
                dec = (a.cdelta[pf_cid] + dmax) * (1.f + 0x1.0p-20f);
                ok = pf_mg > dec;
            }
            if (__syncthreads_and(ok)) {
                if (live && !stable)
                    a.bmargin[(size_t)blockIdx.x * 64 + tid] =
                        (pf_mg - dec) * (1.f - 0x1.0p-20f) - 1e-6f * ((float)a.wd + (USEVAL ? (float)a.wv : 0.0f));
                const BlockCache &bc = a.bcache[blockIdx.x];
                for (int e = tid; e < bn * 6; e += NT) {
                    const int ce = e / 6, q = e - 6 * ce;
                    unsigned long long *dst = a.acc + (size_t)bc.id[ce] * MFSEG_ACC_WORDS;
                    if (q == 5) atomicAdd(dst + 13, bc.cnt[ce]);
                    else atomic_add_fix(dst + (q < 4 ? 2 * q : 10), bc.w[ce][2 * q], (long long)bc.w[ce][2 * q + 1]);
                }
                if (DEVICE_STATS(a) && tid < 64 && live) atomicAdd(a.stats + 24, 1ull);
                return;
            }
        }
    }

    // ---- block coordinates (reference formula) + 128-bit fixed-point copies
    if (tid < TE) {
        double cv;
        unsigned long long *dst;
        if (tid < BX) {
            cv = cell_coord(a.ox, a.sx, a.x0 + X.start + min(tid, X.len - 1));
            S.x[tid] = cv;
            dst = S.xf[tid];
        } else if (tid < OZ) {
            const int i = tid - BX;
            cv = cell_coord(a.oy, a.sy, a.y0 + Y.start + min(i, Y.len - 1));
            S.y[i] = cv;
            dst = S.yf[i];
        } else if (tid < OT) {
            const int i = tid - OZ;
            cv = a.swap_zt ? a.times[Z.start + min(i, Z.len - 1)]
                           : cell_coord(a.oz, a.sz, a.z0 + Z.start + min(i, Z.len - 1));
            S.z[i] = cv;
            dst = S.zf[i];
        } else {
            const int i = tid - OT;
            cv = a.swap_zt ? cell_coord(a.oz, a.sz, a.z0 + Tm.start + min(i, Tm.len - 1))
                           : a.times[Tm.start + min(i, Tm.len - 1)];
            S.t[i] = cv;
            dst = S.tf[i];
        }
        long long hi;
        d2fix(cv, dst[0], hi, &ovf_local);
        dst[1] = (unsigned long long)hi;
    }
    const int sbin = ((Tm.bin * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;
    // initial pass, every cell of the block interior to its bin (margin 2^-20 of a
    // bin from every bin boundary, see run.cu seeds_fast_ok): the block's own seed
    // (id = sbin) is the unique nearest valid candidate of every sample, so the
    // block is labelled and summed without candidate lists or tables
    const bool fast0 = a.seeds_fast && X.pad && Y.pad && Z.pad && Tm.pad;
    const int L0 = fast0 ? 0 : a.g.cand_start[sbin], L1 = fast0 ? 0 : a.g.cand_start[sbin + 1];
    bool deferred = (L1 - L0) > NT;
    int cnt = 0;
    float cvmax = 0.0f;
    if (fast0) {
        if (tid == 0) S.id[0] = sbin;
        cnt = 1;
    } else if (!deferred) {
        // ---- candidates whose validity box meets the block, compacted to slots
        const int ci = L0 + tid;
        bool have = ci < L1;
        int id = 0;
        unsigned box = 0;
        if (have) {
            id = a.g.cand_ids[ci];
            const int4 b0 = a.g.vbox[2 * id], br = a.g.vbox[2 * id + 1];
            const int4 b1 = a.swap_zt ? make_int4(br.z, br.w, br.x, br.y) : br;   // kernel (z, t) ranges
            const int xa = max(b0.x - X.start, 0), xb = min(b0.y - X.start, X.len - 1);
            const int ya = max(b0.z - Y.start, 0), yb = min(b0.w - Y.start, Y.len - 1);
            const int za = max(b1.x - Z.start, 0), zb = min(b1.y - Z.start, Z.len - 1);
            const int ta = max(b1.z - Tm.start, 0), tb = min(b1.w - Tm.start, Tm.len - 1);
            have = xa <= xb && ya <= yb && za <= zb && ta <= tb;
            box = (unsigned)xa | ((unsigned)xb << 4) | ((unsigned)ya << 8) | ((unsigned)yb << 12) |
                  ((unsigned)za << 16) | ((unsigned)zb << 20) | ((unsigned)ta << 24) |
                  ((unsigned)tb << 26);
        }
        // the kept candidates' state, loaded before the compaction's barrier
        double cx = 0.0, cy = 0.0, cz = 0.0, ct = 0.0, cv = 0.0;
        bool chas = false;
        float cdl = 0.f;
        if (have) {
            cx = a.c.x[id];
            cy = a.c.y[id];
            cz = a.c.z[id];
            ct = a.c.t[id];
            chas = a.chas[id] != 0;
            if (chas) cv = a.cval[id];
            if (a.reuse) cdl = a.cdelta[id];
        }
        const unsigned bal = __ballot_sync(0xffffffffu, have);
        float mycv = 0.0f;
        if (lane == 0) S.wc[w] = __popc(bal);
        __syncthreads();
        int off = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < w ? S.wc[q] : 0;
            cnt += S.wc[q];
        }
        deferred = cnt > CAP;
        if (!deferred && have) {
            const int p = off + __popc(bal & ((1u << lane) - 1u));
            S.id[p] = id;
            S.c[p][0] = cx;
            S.c[p][1] = cy;
            S.c[p][2] = cz;
            S.c[p][3] = ct;
            S.c[p][4] = cv;
            S.box[p] = box;
            S.has[p] = chas;
            S.cvf[p] = (float)cv;
            S.wvf[p] = (USEVAL && chas) ? (float)a.wv : 0.0f;
            if (USEVAL && chas) mycv = fabsf((float)cv);
        }
        if (USEVAL) {
            mycv = warp_max_nn(mycv);
            if (lane == 0) S.red[w] = mycv;
        }
        if (a.reuse) {   // largest metric change among the block's candidates
            const float md = warp_max_nn((!deferred && have) ? cdl : 0.f);
            if (lane == 0) S.red2[w] = md;
        }
        __syncthreads();
        if (USEVAL) {
#pragma unroll
            for (int q = 0; q < NW; ++q) cvmax = fmaxf(cvmax, S.red[q]);
        }
    }

    // ---- reuse: in a stable block (no candidate changed since the last pass) a
    // brick labelled by one slot then keeps its labels; the tables and region
    // lists are built only if some brick must be recomputed
    // stable: nothing changed (labels reusable as they are); sstable: only bounded
    // moves (a brick's label is reusable while its proven margin exceeds twice the
    // largest metric change of the block's candidates; the margin is carried on)
    const bool sstable = fast0 || (a.reuse && !deferred && cnt > 0 && a.bin_sstable[sbin]);
    const bool stable = fast0 || (sstable && a.bin_stable[sbin]);
    bool need_full = true;
    float dmax = 0.f;
    if (sstable) {
        if (!stable) {
#pragma unroll
            for (int q = 0; q < NW; ++q) dmax = fmaxf(dmax, S.red2[q]);
        }
        int need = 0;
        if (tid < 64) {
            const int bx = tid & 1, by = (tid >> 1) & 3, bz = (tid >> 3) & 3, bt = tid >> 5;
            const size_t bidx = (size_t)blockIdx.x * 64 + tid;
            unsigned char sl = fast0 ? 0 : pf_sl;
            if (sl != 255) {
                // the per-brick constants of the reuse path below, in shared memory
                S.bsums[tid] = pf_bs;
                if (!stable) {
                    // the margin must exceed the change of s* plus the largest change of
                    // any other candidate of the block
                    const float dec = (a.cdelta[S.id[sl]] + dmax) * (1.f + 0x1.0p-20f);
                    const float mg = pf_mg;
                    if (!(mg > dec)) sl = 255;
                    else   // reused: the margin shrinks by the bound of this pass's moves
                        a.bmargin[bidx] = (mg - dec) * (1.f - 0x1.0p-20f) -
                                          1e-6f * ((float)a.wd + (USEVAL ? (float)a.wv : 0.0f));
                }
            }
            S.bslot[tid] = sl;
            need = sl == 255 && !(GX * bx >= X.len || GY * by >= Y.len || GZ * bz >= Z.len ||
                                  GT * bt >= Tm.len);
        }
        need_full = __syncthreads_or(need) != 0;
    }
    if (!deferred && cnt > 0 && !need_full && a.accumulate) {
        for (int e = tid; e < cnt * HW; e += NT) (&S.hist[0][0])[e] = 0u;
        for (int e = tid; e < cnt * 6; e += NT) (&S.vlimb[0][0])[e] = 0u;
        __syncthreads();
    }
    if (!deferred && cnt > 0 && need_full) {
        // ---- fp32 tables + group (min, max): one (axis, candidate) row per thread
        for (int j = tid; j < 4 * cnt; j += NT) {
            const int ax = j / cnt, p = j - ax * cnt;   // axis-major: warps stay on one axis
            const unsigned b = S.box[p];
            const double cc = S.c[p][ax];
            if (ax == 0)
                table_row<BX, GX>(S.tab[p], S.qmm[p], S.x, cc, 1.0, false, b & 15u, (b >> 4) & 15u, X.len);
            else if (ax == 1)
                table_row<BY, GY>(S.tab[p] + BX, S.qmm[p] + QY, S.y, cc, 1.0, false, (b >> 8) & 15u,
                                  (b >> 12) & 15u, Y.len);
            else if (ax == 2)   // (the time axis carries the c_f scale)
                table_row<BZ, GZ>(S.tab[p] + OZ, S.qmm[p] + QZ, S.z, cc, a.cf, a.swap_zt != 0,
                                  (b >> 16) & 15u, (b >> 20) & 15u, Z.len);
            else
                table_row<BT, GT>(S.tab[p] + OT, S.qmm[p] + QT, S.t, cc, a.cf, a.swap_zt == 0,
                                  (b >> 24) & 3u, (b >> 26) & 3u, Tm.len);
        }
        if (a.accumulate) {
            for (int e = tid; e < cnt * HW; e += NT) (&S.hist[0][0])[e] = 0u;
            for (int e = tid; e < cnt * 6; e += NT) (&S.vlimb[0][0])[e] = 0u;
        }
        __syncthreads();
    }

    // ---- bricks: warp w takes bricks w, w + 8, ... (8x4x4 voxels x 2 timesteps each)
    if (tid == 0) {
        Ctx &C = S.ctx;
        C.X = X;
        C.Y = Y;
        C.Z = Z;
        C.T = Tm;
        C.cnt = cnt;
        C.nrounds = (cnt + 31) >> 5;
        C.deferred = deferred;
        C.cvmax = cvmax;
        C.plane = (long long)a.ny * a.nx;
        C.vol = C.plane * a.nz;
        C.fwd = (float)a.wd;
        C.wvf = USEVAL ? (float)a.wv : 0.0f;
        C.slack = 3e-13f * (float)(a.wd + a.wv);
    }
    __syncthreads();
    const Ctx &C = S.ctx;
    // warp region candidate list (see region_list)
    {
        int nl = -1;
        const int rbx = w & 1, rby = (w >> 1) & 3;
        // (skipped when every brick of this warp keeps its labels)
        bool wneed = need_full;
        if (sstable && need_full) wneed = __any_sync(0xffffffffu, lane < 8 && S.bslot[w + NW * lane] == 255);
        if (!deferred && cnt > 0 && cnt <= 32 && wneed) {
            // one round of candidates: the bricks cull them directly (a region cull
            // would cost a round of its own and remove nothing from the bricks' round)
            if (lane < cnt) S.lst[w][lane] = lane;
            if (lane == 0) S.rcg[w] = INF_F;
            nl = cnt;
        } else if (!deferred && cnt > 0 && wneed && GX * rbx < X.len && GY * rby < Y.len) {
            float vl = 0.f, vh = 0.f;
            if (USEVAL) {   // value range of the region = union of its bricks' ranges
                float lo = INF_F, hi = -INF_F;
                if (lane < 8) {
                    const int bi = w + NW * lane;
                    const int bz = (bi >> 3) & 3, bt = bi >> 5;
                    if (GZ * bz < Z.len && GT * bt < Tm.len) {
                        const float2 r = a.brange[(size_t)blockIdx.x * 64 + bi];
                        lo = r.x;
                        hi = r.y;
                    }
                }
                vl = warp_min_any(lo);
                vh = warp_max_any(hi);
            }
            const int zg1 = (Z.len - 1) / GZ, tg1 = (Tm.len - 1) / GT;
            nl = C.nrounds <= 3 ? region_list<USEVAL, 3>(S, C, rbx, rby, 0, zg1, 0, tg1, vl, vh, a.debug)
                                : region_list<USEVAL, 4>(S, C, rbx, rby, 0, zg1, 0, tg1, vl, vh, a.debug);
            if (DEVICE_STATS(a) && lane == 0) {
                atomicAdd(a.stats + 4, 1ull);
                if (nl >= 0) {
                    atomicAdd(a.stats + 5, 1ull);
                    atomicAdd(a.stats + 6, (unsigned long long)nl);
                }
            }
        }
        if (lane == 0) S.nlist[w] = nl;
    }
    __syncthreads();
    // bricks: warp w takes w, w + 8, ... (the partial sums are order-free integers,
    // so which warp takes which brick does not affect the result)
    // the warp's reused bricks, lane-parallel (lane j <-> brick w + 8 j): labels stay,
    // the sums are constants -- one run per slot (run_brick_sums) for the full ones
    unsigned needm = 0xFFu;   // bricks j left for the loop below
    if (sstable) {
        const int bx = w & 1, by = (w >> 1) & 3;
        const int bj = w + 8 * (lane & 7), jbz = (bj >> 3) & 3, jbt = bj >> 5;
        const bool inr = !(GX * bx >= X.len || GY * by >= Y.len || GZ * jbz >= Z.len || GT * jbt >= Tm.len);
        const int sl = S.bslot[bj];
        const bool ru = lane < 8 && inr && sl != 255;
        const unsigned rmask = __ballot_sync(0xffffffffu, ru);
        needm = ~rmask & 0xFFu;
        if (rmask) {
            const bool jfull = GX * bx + GX <= X.len && GY * by + GY <= Y.len && GZ * jbz + GZ <= Z.len &&
                               GT * jbt + GT <= Tm.len;
            if (fast0) {   // initial pass: the labels are written once
                for (unsigned m = rmask; m; m &= m - 1) {
                    const int b = w + 8 * (__ffs(m) - 1);
                    label_brick(a, C, bx, by, (b >> 3) & 3, b >> 5, sbin);
                }
            }
            if (a.accumulate) {
                for (unsigned m = __ballot_sync(0xffffffffu, ru && !jfull); m; m &= m - 1) {   // cut bricks
                    const int b = w + 8 * (__ffs(m) - 1), bz = (b >> 3) & 3, bt = b >> 5;
                    single_brick_sums(S, S.bsums[b], S.bslot[b], bx, by, bz, bt, min(GX, X.len - GX * bx),
                                      min(GY, Y.len - GY * by), min(GZ, Z.len - GZ * bz),
                                      min(GT, Tm.len - GT * bt));
                }
                unsigned fm = __ballot_sync(0xffffffffu, ru && jfull);
                while (fm) {
                    const int L = __shfl_sync(0xffffffffu, sl, __ffs(fm) - 1);
                    const bool in = (fm >> lane & 1u) && sl == L;
                    fm &= ~__ballot_sync(0xffffffffu, in);
                    const unsigned rcg = __reduce_add_sync(
                        0xffffffffu, in ? (1u << (4 * jbz)) + (1u << (16 + 4 * jbt)) + (1u << 24) : 0u);
                    unsigned long long lo = 0, hi = 0;
                    if (in) {
                        const ulonglong2 v = S.bsums[bj];
                        lo = v.x;
                        hi = v.y;
                    }
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {   // 128-bit sum over lanes 0-7
                        const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
                        const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
                        const unsigned long long n = lo + l2;
                        hi = hi + h2 + (n < lo ? 1ull : 0ull);
                        lo = n;
                    }
                    lo = __shfl_sync(0xffffffffu, lo, 0);
                    hi = __shfl_sync(0xffffffffu, hi, 0);
                    run_brick_sums(S, L, bx, by, rcg, lo, hi);
                }
            }
            if (DEVICE_STATS(a) && lane == 0) atomicAdd(a.stats + 24, (unsigned long long)__popc(rmask));
        }
    }
    bool nocache = false;                 // a brick not labelled by one slot (block cache)
    int rslot = -1;                       // run of freshly labelled single-slot full bricks
    unsigned rc = 0;                      // its packed counts (run_brick_sums)
    unsigned long long rvlo = 0, rvhi = 0;
    for (unsigned bm = needm; bm; bm &= bm - 1) {   // the bricks not reused above
        const int bi = w + NW * (__ffs(bm) - 1);
        const int bx = bi & 1, by = (bi >> 1) & 3, bz = (bi >> 3) & 3, bt = bi >> 5;
        if (!(GX * bx >= X.len || GY * by >= Y.len || GZ * bz >= Z.len || GT * bt >= Tm.len)) {
            const bool full = GX * bx + GX <= X.len && GY * by + GY <= Y.len &&
                              GZ * bz + GZ <= Z.len && GT * bt + GT <= Tm.len;
            const int region = bi & 7, nl = S.nlist[region];
            const size_t bidx = (size_t)blockIdx.x * 64 + bi;
            if (lane == 0 && a.bslot) a.bslot[bidx] = 255;
            int nlb = nl;
            if (nl < 0) {
                // more than 32 survivors in the region: a list for this brick alone
                // (one code path for every brick keeps the hot code small)
                float vl = 0.f, vh = 0.f;
                if (USEVAL) {
                    const float2 r = a.brange[bidx];
                    vl = r.x;
                    vh = r.y;
                }
                nlb = C.nrounds <= 3 ? region_list<USEVAL, 3>(S, C, bx, by, bz, bz, bt, bt, vl, vh, a.debug)
                                     : region_list<USEVAL, 4>(S, C, bx, by, bz, bz, bt, bt, vl, vh, a.debug);
            }
            if (nlb >= 0) {
                if (full) {
                    const int one = brick<USEVAL, true, 1, true>(a, S, C, bi, bx, by, bz, bt, region, nlb,
                                                                 ovf_local);
                    nocache |= one == -2;
                    if (one >= 0 && a.accumulate) {   // single-slot full brick: into the warp's run
                        if (one != rslot) {
                            if (rc) run_brick_sums(S, rslot, bx, by, rc, rvlo, rvhi);
                            rslot = one;
                            rc = 0;
                            rvlo = rvhi = 0;
                        }
                        rc += (1u << (4 * bz)) + (1u << (16 + 4 * bt)) + (1u << 24);
                        const ulonglong2 v = a.bsum[bidx];
                        const unsigned long long n = rvlo + v.x;
                        rvhi += v.y + (n < rvlo ? 1ull : 0ull);
                        rvlo = n;
                    }
                } else {
                    nocache |= brick<USEVAL, false, 1, true>(a, S, C, bi, bx, by, bz, bt, region, nlb,
                                                             ovf_local) == -2;
                }
            } else {
                defer_brick(a, C, bx, by, bz, bt);   // > 32 survivors in one brick: exact path
                nocache = true;
            }
        }
    }
    if (rc) run_brick_sums(S, rslot, w & 1, (w >> 1) & 3, rc, rvlo, rvhi);

    // ---- once per block: marginals x fixed-point coordinates -> global 128-bit sums
    // (and into the block cache when every brick has one label: up to BC_MAX clusters)
    if (a.accumulate && !deferred && cnt > 0) {
        bool cache = __syncthreads_or(nocache) == 0 && a.bcache != nullptr;
        if (cache) {   // entry of each cluster present (warp 0), in slot order
            if (w == 0) {
                int base = 0;
                for (int r = 0; 32 * r < cnt; ++r) {
                    const int sl = 32 * r + lane;
                    const bool nz = sl < cnt && S.hist[sl][26] != 0;
                    const unsigned b = __ballot_sync(0xffffffffu, nz);
                    if (sl < cnt) S.cidx[sl] = nz ? base + __popc(b & ((1u << lane) - 1u)) : -1;
                    base += __popc(b);
                }
                if (lane == 0) S.cnz = base;
            }
            __syncthreads();
            cache = S.cnz <= BC_MAX;
            if (tid == 0) a.bcache[blockIdx.x].n = cache ? S.cnz : -1;
        } else if (tid == 0 && a.bcache) {
            a.bcache[blockIdx.x].n = -1;
        }
        for (int e = tid; e < cnt * 6; e += NT) {
            const int s = e / 6, wd = e - s * 6;
            const unsigned *h = S.hist[s];
            const int n = (int)h[26];
            if (n == 0) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            BlockCache *bcp = cache ? a.bcache + blockIdx.x : nullptr;
            const int ce = cache ? S.cidx[s] : -1;
            __int128 acc = 0;
            if (wd < 4) {   // one rolled loop for the four axes (small code)
                static_assert(BX == BY && BY == BZ, "x, y, z marginals share one loop");
                const unsigned long long(*F)[2] = wd == 0 ? S.xf : wd == 1 ? S.yf : wd == 2 ? S.zf : S.tf;
                const int nn = wd == 3 ? BT : BX;
#pragma unroll 4
                for (int i = 0; i < nn; ++i) acc += get128(F[i]) * (__int128)hget(h + 8 * wd, i);
            } else if (wd == 4) {
                acc = value_limbs_total(S.vlimb[s]);
            } else {
                atomicAdd(dst + 13, (unsigned long long)n);
                if (bcp) {
                    bcp->id[ce] = S.id[s];
                    bcp->cnt[ce] = (unsigned long long)n;
                }
                continue;
            }
            const int word = wd < 2 ? 2 * wd : wd < 4 ? 2 * (a.swap_zt ? 5 - wd : wd) : 10;   // real axis
            atomic_add_fix(dst + word, (unsigned long long)acc, (long long)(acc >> 64));
            if (bcp) {
                const int q = word < 10 ? word / 2 : 4;
                bcp->w[ce][2 * q] = (unsigned long long)acc;
                bcp->w[ce][2 * q + 1] = (unsigned long long)(acc >> 64);
            }
        }
    } else if (tid == 0 && a.bcache) {
        a.bcache[blockIdx.x].n = -1;
    }
    if (ovf_local) *a.overflow = 1;
}

// Per brick, once per run: range of fl32(value) and the fixed-order value sum
// (each lane sums its samples in k order, then the fp64 warp butterfly) --
// exactly what k_field_assign5 would compute from the same samples.
__global__ void __launch_bounds__(NT) k_brick_pre(FieldArgs a) {
    unsigned tile = blockIdx.x;
    const int txi = (int)(tile % (unsigned)a.ntx);
    tile /= (unsigned)a.ntx;
    const int tyi = (int)(tile % (unsigned)a.nty);
    tile /= (unsigned)a.nty;
    const int tzi = (int)(tile % (unsigned)a.ntz);
    const int tti = (int)(tile / (unsigned)a.ntz);
    const AxisTile X = a.xt[txi], Y = a.yt[tyi], Z = a.zt[tzi], T = a.tt[tti];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long plane = (long long)a.ny * a.nx, vol = plane * a.nz;
    double amax = 0.0;   // max |value| and non-finite flag (range check of the fixed-point sums)
    bool bad = false;
    // two rounds of four bricks per warp; each round issues its 32 loads per lane
    // before any is used (HBM latency is covered by the loads in flight)
#pragma unroll 1
    for (int b0 = w; b0 < 64; b0 += 4 * NW) {
        double v[4][8];
        unsigned lv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int bi = b0 + u * NW;
            const int bx = bi & 1, by = (bi >> 1) & 3, bz = (bi >> 3) & 3, bt = bi >> 5;
            const int lx = GX * bx + (lane & 7), ly = GY * by + (lane >> 3);
            const int z0 = GZ * bz, t0 = GT * bt;
            const long long fbase = (((long long)(T.start + t0) * a.nz + Z.start + z0) * a.ny +
                                     (Y.start + ly)) * (long long)a.nx + (X.start + lx);
            lv[u] = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (lx < X.len && ly < Y.len && z0 + (k & 3) < Z.len && t0 + (k >> 2) < T.len) lv[u] |= 1u << k;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                v[u][k] = (lv[u] >> k & 1) ? __ldg(a.values + fbase + (k & 3) * plane + (k >> 2) * vol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int bi = b0 + u * NW;
            const int bx = bi & 1, by = (bi >> 1) & 3, bz = (bi >> 3) & 3, bt = bi >> 5;
            if (GX * bx >= X.len || GY * by >= Y.len || GZ * bz >= Z.len || GT * bt >= T.len) continue;
            float lo = INF_F, hi = -INF_F;
            double vs = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                vs = DADD(vs, v[u][k]);
                if (lv[u] >> k & 1) {
                    lo = fminf(lo, (float)v[u][k]);
                    hi = fmaxf(hi, (float)v[u][k]);
                }
            }
            vs = warp_sum_d(vs);
            lo = warp_min_f(lo);
            hi = warp_max_f(hi);
            // range check of the fixed-point sums, per brick: NaN / inf propagate into
            // the fp64 sum; |value| is bounded by the fl32 range (inf if it overflows fl32)
            bad |= !isfinite(vs);
            amax = fmax(amax, (double)fmaxf(fabsf(lo), fabsf(hi)));
            if (lane == 0) {
                a.brange_out[(size_t)blockIdx.x * 64 + bi] = make_float2(lo, hi);
                unsigned long long flo;
                long long fhi;
                int ovf = 0;
                d2fix(vs, flo, fhi, &ovf);
                if (ovf) *a.overflow = 1;
                a.bsum_out[(size_t)blockIdx.x * 64 + bi] = make_ulonglong2(flo, (unsigned long long)fhi);
            }
        }
    }
    // one atomic per block, and only when it raises the maximum (every block
    // hitting one address would serialise thousands of atomics at the L2)
    __shared__ double bmax[NW];
    __shared__ int bbad[NW];
    if (lane == 0) {   // amax and bad are warp-uniform
        bmax[w] = amax;
        bbad[w] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0 && a.absmax) {
        double m = bmax[0];
        int b = bbad[0];
        for (int q = 1; q < NW; ++q) {
            m = fmax(m, bmax[q]);
            b |= bbad[q];
        }
        const unsigned long long mk = (unsigned long long)__double_as_longlong(m);
        if (mk > *(volatile unsigned long long *)(a.absmax + 5)) atomicMax(a.absmax + 5, mk);
        if (b) atomicOr(a.absmax + 6, 1ull);
    }
}

int launch_brick_pre(const FieldArgs &a, cudaStream_t st) {
    const long long n = (long long)a.ntx * a.nty * a.ntz * a.ntt;
    if (n <= 0) return 0;
    ::mfseg::count_launch();
    k_brick_pre<<<(unsigned)n, NT, 0, st>>>(a);
    MFSEG_LAUNCH("k_brick_pre");
    return 0;
}

int launch_field_assign_v5(const FieldArgs &a, cudaStream_t st) {
    const long long n = (long long)a.ntx * a.nty * a.ntz * a.ntt;
    if (n <= 0) return 0;
    if (n > 0x7fffffffll) {
        set_error("field tile grid too large");
        return 3;
    }
    const size_t smem = sizeof(Smem5);
    static bool configured = false;
    if (!configured) {
        MFSEG_CUDA(cudaFuncSetAttribute(k_field_assign5<true, 3>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MFSEG_CUDA(cudaFuncSetAttribute(k_field_assign5<false, 3>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    ::mfseg::count_launch();
    if (a.wv > 0.0)
        k_field_assign5<true, 3><<<(unsigned)n, NT, smem, st>>>(a);
    else
        k_field_assign5<false, 3><<<(unsigned)n, NT, smem, st>>>(a);
    MFSEG_LAUNCH("k_field_assign5");
    return 0;
}

}  // namespace mfseg
