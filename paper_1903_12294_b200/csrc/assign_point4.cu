// k_point_assign4 — windowed exact assignment of point samples, one CTA per
// chunk of <= 2048 bin-sorted points of one sample bin (v4, the default).
//
// Same contract as the field kernels (exact reference labels, lowest id on
// ties; engine.py:137-192).  Points are sorted once per run by (sample bin,
// 4^4 Morton sub-cell) and cut into chunks of one bin; per chunk the exact
// fp64 bounding box is computed once per run (k_tile_box).  Per CTA:
//
//  1. the bin's candidates are classified against the chunk box in exact fp64
//     (no sample can pass the box test / every sample passes / partial) and
//     get chunk-relative fp32 coordinates rc = fl32(fl64(c - o) s) (o = box
//     minimum corner, s = c_f for time, 1 otherwise); points get rp likewise,
//     so |(rc - rp)_d - s (c - x)_d| <= 2^-22 (E_d + C_d) s =: delta_d / 2 and
//     |d32 - D| <= 2^-19 (D + W) + w_d ||delta|| (v3 analysis, assign_point.cu).
//  2. each warp walks 64-point warp tiles (2 points per lane): fp32 bounds over
//     the warp tile's box cull the candidates (margin 2^-16 relative), then the
//     per-point screen keeps best/second best as packed (d, slot) keys (three
//     integer min/max per pair; truncation 2^-16 relative, covered by the
//     certification exactly as in k_field_assign5) and certifies with margin
//     2^-18 relative + 2 w_d ||delta|| absolute.  Box tests inside the
//     +-delta guard band, near ties and overflow go to exact fp64.
//  3. partial sums: per warp and slot fp64 running sums (the warp's tiles in a
//     fixed order), per slot point counts with shared atomics; once per CTA
//     the warp sums are converted exactly to 128-bit fixed point and added to
//     the global sums.  Chunks are canonical (never split across GPUs when the
//     time slabs are whole t-bins), so the sums are deterministic.
#include <climits>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();
constexpr unsigned INF_BITS = 0x7F800000u;

constexpr int NT = 128, NW = 4;   // 4 warps: a short per-CTA tail, 6 CTAs per SM
constexpr int CR = 2;             // raw candidate rounds of NT (up to 256 per bin)
#ifndef MFSEG_POINT_MINB
#define MFSEG_POINT_MINB 6
#endif
constexpr int MINB = MFSEG_POINT_MINB;
constexpr int CAP = 128;
constexpr unsigned SLOT_MASK = 127u;
constexpr float KSCR = 0x1.0p-18f;
constexpr float KCULL = 0x1.0p-16f;
static_assert(POINT_CHUNK % 64 == 0, "warp tiles of 64 points");

struct PCtx {
    double o[4];
    float delta[4], Cf[4];
    float iC[4], uhi, ulo;          // 1 / Cf; 1 +- eps (box test band)
    float cw[4], cn[4];             // Cf +- delta (guard-banded box half-widths)
    float Aabs, cvmax, fwd, wvf, slack, ndelta;
    int cnt, nrounds, len;
    long long start;
    bool deferred;
    bool stable;                    // no candidate changed since the last pass
    bool fast0;                     // initial pass, interior chunk: every point takes slot 0
};

struct __align__(16) PSmem4 {
    float4 rc[CAP];                 // chunk-relative fp32 centre coordinates
    double c[CAP][5];               // cx, cy, cz, ct (raw), cv
    double wsum[NW][5][CAP];        // per-warp fp64 sums of x, y, z, t, v
    unsigned n[CAP];
    int id[CAP];
    float cvf[CAP], wvf[CAP];
    unsigned char has[CAP], full[CAP];
    int wc[CR * NW];
    float red[NW];
    int plisted;                    // some point went to the stranded / deferred lists
    int pcidx[CAP];                 // chunk cache: entry of each slot (-1: absent)
    int pcnz;
    PCtx ctx;
};

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float wmin_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float wmax_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double wmin_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double wmax_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

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

// exact reference box test + metric of one pair (engine.py:137-149, 179-181)
__device__ __forceinline__ bool exact_pair(const double *c, const double *P, bool has, double cf,
                                           double wv, double wd, const double *C, double &D) {
    const double dx = DSUB(c[0], P[0]), dy = DSUB(c[1], P[1]), dz = DSUB(c[2], P[2]),
                 dt = DSUB(c[3], P[3]);
    if (!(fabs(dx) <= C[0] && fabs(dy) <= C[1] && fabs(dz) <= C[2] && fabs(dt) <= C[3])) return false;
    const double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    const double ct = DMUL(cf, dt);
    D = metric_tail(q, DMUL(ct, ct), P[4], c[4], has, wv, wd);
    return true;
}

// fp32 screen distance of one (point, slot) pair; box test with the guard band
// as u = max_d |d_d| / Cf_d against 1 +- eps (eps = max_d delta_d / Cf_d + 2^-22
// covers the two fp32 roundings of u): u > 1 + eps -> outside for sure (+inf);
// u >= 1 - eps -> within the band, `unsure` (exact fp64 decides).
__device__ __forceinline__ float pair_d32(const float4 &r, const float *rp, const PCtx &C, bool full,
                                          float fv, float cvs, float wvs, bool useval, bool &unsure) {
    const float dx = r.x - rp[0], dy = r.y - rp[1], dz = r.z - rp[2], dt = r.w - rp[3];
    const float q = fmaf(dt, dt, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
    float d = useval ? fmaf(C.fwd, sqrt_approx(q), wvs * fabsf(fv - cvs)) : C.fwd * sqrt_approx(q);
    if (!full) {
        const float u = fmaxf(fmaxf(fabsf(dx) * C.iC[0], fabsf(dy) * C.iC[1]),
                              fmaxf(fabsf(dz) * C.iC[2], fabsf(dt) * C.iC[3]));
        const bool out = u > C.uhi;
        unsure |= !out && u >= C.ulo;
        d = out ? INF_F : d;
    }
    return d;
}

// NR: rounds of 32 candidate slots (3 for chunks with <= 96 candidates)
template <bool USEVAL, int NR>
__device__ __forceinline__ void point_warp(const PointArgs &a, PSmem4 &S, const PCtx &C, int wt,
                                           int &ovf_local) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double Cd[4] = {a.Cx, a.Cy, a.Cz, a.Ct};
    const int off0 = 64 * wt + lane, off1 = off0 + 32;
    const bool live0 = off0 < C.len, live1 = off1 < C.len;
    const long long p0 = C.start + off0, p1 = C.start + off1;
    // The point records are loaded only for tiles left with several candidates;
    // a tile labelled by one candidate uses its per-run box and sums (k_wtile_box:
    // the points do not change between passes).
    double P0[5] = {0, 0, 0, 0, 0}, P1[5] = {0, 0, 0, 0, 0};
    const WBox *wbp = a.wbox + (size_t)blockIdx.x * (POINT_CHUNK / 64) + wt;
    const size_t tidx = (size_t)blockIdx.x * (POINT_CHUNK / 64) + wt;
    int sl0 = -1, sl1 = -1;
    bool reused = false;   // several labels kept from the last pass: sums only
    if (C.stable) {   // unchanged since the last pass: the tile keeps its labels
        const unsigned char ts = C.fast0 ? 0 : a.tslot[tidx];
        if (ts < 254) {   // one label: the per-run tile sums
            if (C.fast0) {   // initial pass: the labels are new
                if (live0) a.labels[p0] = S.id[0];
                if (live1) a.labels[p1] = S.id[0];
            }
            if (a.labels_out) {   // final pass: record-order labels
                if (live0) a.labels_out[a.perm[p0]] = S.id[ts];
                if (live1) a.labels_out[a.perm[p1]] = S.id[ts];
            }
            if (a.accumulate && lane == 0) {
#pragma unroll
                for (int d = 0; d < 5; ++d) S.wsum[w][d][ts] = DADD(S.wsum[w][d][ts], wbp->s[d]);
                atomicAdd(&S.n[ts], (unsigned)min(64, C.len - 64 * wt));
            }
            return;
        }
        if (ts == 254) {   // several labels (none stranded): slots from the labels
            if (!a.accumulate) return;
            const int lab0 = live0 ? a.labels[p0] : -1, lab1 = live1 ? a.labels[p1] : -1;
            if (a.labels_out) {
                if (live0) a.labels_out[a.perm[p0]] = lab0;
                if (live1) a.labels_out[a.perm[p1]] = lab1;
            }
            int todo0 = lab0, todo1 = lab1;
            while (true) {
                const unsigned m0 = __ballot_sync(0xffffffffu, todo0 >= 0),
                               m1 = __ballot_sync(0xffffffffu, todo1 >= 0);
                if (!(m0 | m1)) break;
                const int L = m0 ? __shfl_sync(0xffffffffu, todo0, __ffs(m0) - 1)
                                 : __shfl_sync(0xffffffffu, todo1, __ffs(m1) - 1);
                int slot = -1;
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const int s = lane + 32 * r;
                    const unsigned f = __ballot_sync(0xffffffffu, s < C.cnt && S.id[s] == L);
                    if (f && slot < 0) slot = __ffs(f) - 1 + 32 * r;
                }
                if (todo0 == L) {
                    sl0 = slot;
                    todo0 = -1;
                }
                if (todo1 == L) {
                    sl1 = slot;
                    todo1 = -1;
                }
            }
            if (live0) {
                P0[0] = a.x[p0]; P0[1] = a.y[p0]; P0[2] = a.z[p0]; P0[3] = a.t[p0]; P0[4] = a.v[p0];
            }
            if (live1) {
                P1[0] = a.x[p1]; P1[1] = a.y[p1]; P1[2] = a.z[p1]; P1[3] = a.t[p1]; P1[4] = a.v[p1];
            }
            reused = true;
        }
    }
    if (!reused && lane == 0 && a.tslot) a.tslot[tidx] = 255;
    int one = -1;   // slot labelling the whole tile (warp-uniform)
    if (!reused) {
    if (!C.deferred && C.cnt > 0) {
        // warp-tile box (fp32, chunk-relative) and value range: precomputed once per
        // run by k_wtile_box with exactly the formulas used for rp / fv below
        const float4 blo = wbp->lo, bhi = wbp->hi;
        const float2 bv = wbp->v;
        const float wl[4] = {blo.x, blo.y, blo.z, blo.w};
        const float wh[4] = {bhi.x, bhi.y, bhi.z, bhi.w};
        float vl = 0.f, vh = 0.f;
        if (USEVAL) {
            vl = bv.x;
            vh = bv.y;
        }
        // ---- warp culling (fp32 bounds over the warp-tile box, guard bands widen the box test)
        float dl[4], qhu[4];
        bool wf[4];
        float ubw = INF_F;
        unsigned ubkey = 0xFFFFFFFFu;   // (ub | slot) of the best candidate valid on the whole tile
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            dl[r] = INF_F;
            qhu[r] = INF_F;
            wf[r] = false;
            const int s = lane + 32 * r;
            if (r < C.nrounds && s < C.cnt) {
                const float4 rc = S.rc[s];
                const float rcv[4] = {rc.x, rc.y, rc.z, rc.w};
                // per axis the distance range over [b1, a1]: nearest max(0, b1, -a1),
                // farthest max(a1, -b1).  (Clamping to the guard band +-cw changes
                // neither for a candidate that is not out of range, and the farthest
                // distance is the upper bound of a fully valid one.)
                float ql = 0.f, qu = 0.f;
                bool wfull = true, none = false;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const float cw = C.cw[d], cn = C.cn[d];
                    const float a1 = rcv[d] - wl[d], b1 = rcv[d] - wh[d];   // a1 >= b1
                    if (a1 < -cw || b1 > cw) none = true;
                    if (!(a1 <= cn && b1 >= -cn)) wfull = false;
                    const float mn = fmaxf(fmaxf(b1, -a1), 0.f);
                    const float mu = fmaxf(a1, -b1);
                    ql = fmaf(mn, mn, ql);
                    qu = fmaf(mu, mu, qu);
                }
                const float qh = qu;
                float vtl = 0.f, vth = 0.f;
                if (USEVAL) {
                    const float wvs = S.wvf[s];
                    if (wvs > 0.f) {
                        const float cvs = S.cvf[s];
                        const float pl = vl - cvs, ph = vh - cvs;   // pl <= ph
                        vtl = wvs * fmaxf(fmaxf(pl, -ph), 0.f);
                        vth = wvs * fmaxf(ph, -pl);
                    }
                }
                if (!none) dl[r] = fmaf(C.fwd, sqrt_approx(ql), vtl);
                qhu[r] = qu;
                wf[r] = wfull && !none;   // every point of the warp tile passes the box test
                if (wfull && !none) {
                    const float ub = fmaf(C.fwd, sqrt_approx(qh), vth);
                    ubw = fminf(ubw, ub);
                    ubkey = min(ubkey, (__float_as_uint(ub) & ~SLOT_MASK) | (unsigned)s);
                }
            }
        }
        ubw = wmin_f(ubw);
        ubkey = __reduce_min_sync(0xffffffffu, ubkey);
        const float Wb = USEVAL ? C.wvf * (fmaxf(fabsf(vl), fabsf(vh)) + C.cvmax) : 0.f;
        const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb + 2.f * C.Aabs) * (1.f + 0x1.0p-15f);
        unsigned keep[4] = {0u, 0u, 0u, 0u}, kfull[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            keep[r] = __ballot_sync(0xffffffffu, dl[r] < INF_F && (dl[r] <= thr || (a.debug & 1)));
            kfull[r] = __ballot_sync(0xffffffffu, wf[r]);
        }

        // ---- dominance against s' = the fully valid candidate with the smallest upper
        // bound: per axis the squared-distance difference (r_s - x)^2 - (r_s' - x)^2 is
        // linear in x, so its minimum over the tile box is at wl or wh.  The fp32
        // relative coordinates are within delta/2 of the exact scaled differences:
        // exact dS >= dS32 - |delta| (sqrt Sa + sqrt Sb) - |delta|^2 / 2 - rounding.
        // Then D_s - D_s' >= w_d dS / (sqrt S_s + sqrt S_s') - (value-term bound).
        int sdom = -1;
        if (ubkey != 0xFFFFFFFFu && !(a.debug & 1)) {
            sdom = (int)(ubkey & SLOT_MASK);
            const float4 rq = S.rc[sdom];
            const float rqv[4] = {rq.x, rq.y, rq.z, rq.w};
            float sb = 0.f;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const float mu = fmaxf(fabsf(rqv[d] - wl[d]), fabsf(rqv[d] - wh[d]));
                sb = fmaf(mu, mu, sb);
            }
            const float rb = sqrt_approx(sb);
            float cvq = 0.f, wvq = 0.f;
            if (USEVAL) {
                cvq = S.cvf[sdom];
                wvq = S.wvf[sdom];
            }
            const float vabs = fmaxf(fabsf(vl), fabsf(vh));
            const float vq = fmaxf(fabsf(vl - cvq), fabsf(vh - cvq));
            const float nd = C.ndelta;
#pragma unroll 1
            for (int r = 0; r < NR; ++r) {   // rolled: a small hot loop for the instruction cache
                const unsigned kr = r == 0 ? keep[0] : r == 1 ? keep[1] : r == 2 ? keep[2] : keep[3];
                if (kr == 0u) continue;   // warp-uniform
                const float sa = r == 0 ? qhu[0] : r == 1 ? qhu[1] : r == 2 ? qhu[2] : qhu[3];
                const int s = lane + 32 * r;
                bool dom = false;
                if ((kr >> lane & 1u) && s != sdom) {
                    const float4 rc = S.rc[s];
                    const float rcv[4] = {rc.x, rc.y, rc.z, rc.w};
                    float dS = 0.f;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const float al = rcv[d] - wl[d], ah = rcv[d] - wh[d];
                        const float bl = rqv[d] - wl[d], bh = rqv[d] - wh[d];
                        dS += fminf(fmaf(al, al, -bl * bl), fmaf(ah, ah, -bh * bh));
                    }
                    const float ra = sqrt_approx(sa);
                    const float dSlb = dS - nd * (ra + rb) * (1.f + 0x1.0p-20f) - 0.5f * nd * nd -
                                       0x1.0p-20f * (sa + sb);
                    if (dSlb > 0.f) {
                        const float den = (ra + rb + nd) * (1.f + 0x1.0p-20f);
                        const float gap = __fdividef(dSlb, den) * (1.f - 0x1.0p-19f);
                        float Vb = 0.f;
                        if (USEVAL && wvq > 0.f) {
                            // monotone value-term difference: its minimum over the tile's
                            // value range is at an end (see k_field_assign5)
                            const float cvs = S.cvf[s];
                            const float V = S.wvf[s] > 0.f
                                ? C.wvf * fmaxf(0.f, -fminf(fabsf(vl - cvs) - fabsf(vl - cvq),
                                                            fabsf(vh - cvs) - fabsf(vh - cvq)))
                                : C.wvf * vq;
                            Vb = V * (1.f + 0x1.0p-18f) + 0x1.0p-18f * C.wvf * (fabsf(cvs) + fabsf(cvq) + vabs);
                        }
                        const float rel = 0x1.0p-30f * (C.fwd * den + Wb) + C.slack;
                        dom = C.fwd * gap * (1.f - 0x1.0p-20f) > Vb + rel;
                    }
                }
                const unsigned db = __ballot_sync(0xffffffffu, dom);
                if (r == 0) keep[0] &= ~db;
                else if (r == 1) keep[1] &= ~db;
                else if (r == 2) keep[2] &= ~db;
                else keep[3] &= ~db;
            }
        }
        if (DEVICE_STATS(a) && lane == 0) {
            const int nk = __popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]);
            if (nk == 1 && sdom >= 0) atomicAdd(a.stats + 3, 1ull);
            atomicAdd(a.stats + 4 + min(nk, 7), 1ull);
            atomicAdd(a.stats, 1ull);
            atomicAdd(a.stats + 1, (unsigned long long)(__popc(keep[0]) + __popc(keep[1]) +
                                                         __popc(keep[2]) + __popc(keep[3])));
        }
        unsigned a1k = 0xFFFFFFFFu, a2k = 0xFFFFFFFFu, b1k = 0xFFFFFFFFu, b2k = 0xFFFFFFFFu;
        bool unsure0 = false, unsure1 = false;
        const int nkeep = __popc(keep[0]) + __popc(keep[1]) + __popc(keep[2]) + __popc(keep[3]);
        if (nkeep == 1 && sdom >= 0) {
            // s' is valid for every point of the tile and every other candidate is
            // culled or dominated: it is the exact argmin of every point
            sl0 = live0 ? sdom : -1;
            sl1 = live1 ? sdom : -1;
            one = sdom;
            if (lane == 0 && a.tslot) a.tslot[tidx] = (unsigned char)sdom;
        } else {
        if (live0) {
            P0[0] = a.x[p0]; P0[1] = a.y[p0]; P0[2] = a.z[p0]; P0[3] = a.t[p0]; P0[4] = a.v[p0];
        }
        if (live1) {
            P1[0] = a.x[p1]; P1[1] = a.y[p1]; P1[2] = a.z[p1]; P1[3] = a.t[p1]; P1[4] = a.v[p1];
        }
        float rp0[4], rp1[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const double sc = d == 3 ? a.cf : 1.0;
            rp0[d] = (float)DMUL(DSUB(P0[d], C.o[d]), sc);
            rp1[d] = (float)DMUL(DSUB(P1[d], C.o[d]), sc);
        }
        const float fv0 = (float)P0[4], fv1 = (float)P1[4];
        unsigned scan[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int r = 0; r < NR; ++r) scan[r] = keep[r];

        // ---- per-point screen, packed (d, slot) keys
#pragma unroll 1
        for (int r = 0; r < NR; ++r) {   // rolled: a small hot loop for the instruction cache
            unsigned it = r == 0 ? scan[0] : r == 1 ? scan[1] : r == 2 ? scan[2] : scan[3];
            const unsigned kf = r == 0 ? kfull[0] : r == 1 ? kfull[1] : r == 2 ? kfull[2] : kfull[3];
            while (it) {
                const int b = __ffs(it) - 1, s = b + 32 * r;
                it &= it - 1;
                const float4 rc = S.rc[s];
                const bool fl = (kf >> b) & 1u;
                float cvs = 0.f, wvs = 0.f;
                if (USEVAL) {
                    cvs = S.cvf[s];
                    wvs = S.wvf[s];
                }
                const float d0 = pair_d32(rc, rp0, C, fl, fv0, cvs, wvs, USEVAL, unsure0);
                const float d1 = pair_d32(rc, rp1, C, fl, fv1, cvs, wvs, USEVAL, unsure1);
                const unsigned k0 = (__float_as_uint(d0) & ~SLOT_MASK) | (unsigned)s;
                const unsigned k1 = (__float_as_uint(d1) & ~SLOT_MASK) | (unsigned)s;
                a2k = min(a2k, max(a1k, k0));
                a1k = min(a1k, k0);
                b2k = min(b2k, max(b1k, k1));
                b1k = min(b1k, k1);
            }
        }
        // ---- certify, or resolve exactly
        const float W0 = USEVAL ? C.wvf * (fabsf(fv0) + C.cvmax) : 0.f;
        const float W1 = USEVAL ? C.wvf * (fabsf(fv1) + C.cvmax) : 0.f;
        const float u0 = __uint_as_float(min(a1k & ~SLOT_MASK, INF_BITS)) * (1.f + 0x1.0p-15f);
        const float u1 = __uint_as_float(min(b1k & ~SLOT_MASK, INF_BITS)) * (1.f + 0x1.0p-15f);
        const float s0 = __uint_as_float(min(a2k & ~SLOT_MASK, INF_BITS));
        const float s1 = __uint_as_float(min(b2k & ~SLOT_MASK, INF_BITS));
        const bool ok0 = !(a.debug & 2) && !unsure0 && a1k < INF_BITS &&
                         s0 * (1.f - KSCR) > u0 * (1.f + KSCR) + 2.f * KSCR * W0 + 2.f * C.Aabs;
        const bool ok1 = !(a.debug & 2) && !unsure1 && b1k < INF_BITS &&
                         s1 * (1.f - KSCR) > u1 * (1.f + KSCR) + 2.f * KSCR * W1 + 2.f * C.Aabs;
        sl0 = ok0 ? (int)(a1k & SLOT_MASK) : -1;
        sl1 = ok1 ? (int)(b1k & SLOT_MASK) : -1;
        const bool need0 = live0 && !ok0, need1 = live1 && !ok1;
        if (DEVICE_STATS(a) && (need0 || need1)) atomicAdd(a.stats + 2, (unsigned long long)(need0 + need1));
        if (__any_sync(0xffffffffu, need0 || need1) && (need0 || need1)) {
            // exact fp64 over every kept candidate inside the margin (all of them
            // when a box test was inside the guard band or the screen overflowed)
            const float t0 = (a1k < INF_BITS && !unsure0)
                                 ? (u0 * (1.f + KSCR) + 2.f * KSCR * W0 + 2.f * C.Aabs) * (1.f + 0x1.0p-17f)
                                 : INF_F;
            const float t1 = (b1k < INF_BITS && !unsure1)
                                 ? (u1 * (1.f + KSCR) + 2.f * KSCR * W1 + 2.f * C.Aabs) * (1.f + 0x1.0p-17f)
                                 : INF_F;
            double eD0 = INF_D, eD1 = INF_D;
            int eI0 = INT_MAX, eI1 = INT_MAX, eS0 = -1, eS1 = -1;
#pragma unroll 1
            for (int r = 0; r < NR; ++r) {
                unsigned it = r == 0 ? keep[0] : r == 1 ? keep[1] : r == 2 ? keep[2] : keep[3];
                while (it) {
                    const int s = __ffs(it) - 1 + 32 * r;
                    it &= it - 1;
                    const float4 rc = S.rc[s];
                    const int cid = S.id[s];
                    const float cvs = S.cvf[s], wvs = S.wvf[s];
                    bool dummy = false;
                    double D;
                    if (need0) {
                        const float d = pair_d32(rc, rp0, C, false, fv0, cvs, wvs, USEVAL, dummy);
                        if (!(d > t0) && exact_pair(S.c[s], P0, S.has[s], a.cf, a.wv, a.wd, Cd, D) &&
                            better(D, cid, eD0, eI0)) {
                            eD0 = D; eI0 = cid; eS0 = s;
                        }
                    }
                    if (need1) {
                        const float d = pair_d32(rc, rp1, C, false, fv1, cvs, wvs, USEVAL, dummy);
                        if (!(d > t1) && exact_pair(S.c[s], P1, S.has[s], a.cf, a.wv, a.wd, Cd, D) &&
                            better(D, cid, eD1, eI1)) {
                            eD1 = D; eI1 = cid; eS1 = s;
                        }
                    }
                }
            }
            if (need0) sl0 = eS0;
            if (need1) sl1 = eS1;
        }
        if (!live0) sl0 = -1;
        if (!live1) sl1 = -1;
        }   // screen
    }

    // ---- labels (bin-sorted order); deferred / stranded lists (warp-aggregated)
    int nlist = 0;
    if (live0) {
        const int lab = C.deferred ? -2 : (sl0 >= 0 ? S.id[sl0] : -1);
        a.labels[p0] = lab;
        if (a.labels_out) a.labels_out[a.perm[p0]] = lab;
        if (lab < 0) ++nlist;
    }
    if (live1) {
        const int lab = C.deferred ? -2 : (sl1 >= 0 ? S.id[sl1] : -1);
        a.labels[p1] = lab;
        if (a.labels_out) a.labels_out[a.perm[p1]] = lab;
        if (lab < 0) ++nlist;
    }
    const bool listed = __any_sync(0xffffffffu, nlist > 0);
    if (listed && lane == 0) S.plisted = 1;   // (no chunk cache)
    if (listed) {
        unsigned long long *ctr = C.deferred ? a.n_deferred : a.n_stranded;
        long long *lst = C.deferred ? a.deferred : a.stranded;
        const long long cap = C.deferred ? a.deferred_cap : a.stranded_cap;
        long long p = warp_reserve(ctr, nlist);
        if (live0 && (C.deferred || sl0 < 0)) {
            if (p < cap) lst[p] = p0;
            ++p;
        }
        if (live1 && (C.deferred || sl1 < 0)) {
            if (p < cap) lst[p] = p1;
        }
    }
    // several labels, none stranded: reusable while the chunk's candidates stay
    if (one < 0 && !listed && !C.deferred && C.cnt > 0 && lane == 0 && a.tslot) a.tslot[tidx] = 254;
    }   // !reused

    // ---- partial sums: per-warp fp64 running sums + shared counts
    if (a.accumulate && one >= 0) {   // the whole tile -> one cluster: per-run tile sums
        if (lane == 0) {
#pragma unroll
            for (int d = 0; d < 5; ++d) S.wsum[w][d][one] = DADD(S.wsum[w][d][one], wbp->s[d]);
            atomicAdd(&S.n[one], (unsigned)min(64, C.len - 64 * wt));
        }
        return;
    }
    if (a.accumulate && !C.deferred && C.cnt > 0) {
        unsigned m0 = __ballot_sync(0xffffffffu, sl0 >= 0), m1 = __ballot_sync(0xffffffffu, sl1 >= 0);
        while (m0 | m1) {
            const int L = m0 ? __shfl_sync(0xffffffffu, sl0, __ffs(m0) - 1)
                             : __shfl_sync(0xffffffffu, sl1, __ffs(m1) - 1);
            const unsigned g0 = __ballot_sync(0xffffffffu, sl0 == L);
            const unsigned g1 = __ballot_sync(0xffffffffu, sl1 == L);
            m0 &= ~g0;
            m1 &= ~g1;
            double s5[5];
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                double v = 0.0;
                if (sl0 == L) v = P0[d];
                if (sl1 == L) v = DADD(v, P1[d]);
                s5[d] = warp_sum_d(v);
            }
            if (lane == 0) {
#pragma unroll
                for (int d = 0; d < 5; ++d) S.wsum[w][d][L] = DADD(S.wsum[w][d][L], s5[d]);
                atomicAdd(&S.n[L], (unsigned)(__popc(g0) + __popc(g1)));
            }
        }
    }
    (void)ovf_local;
}

}  // namespace

template <bool USEVAL>
__global__ void __launch_bounds__(NT, MINB) k_point_assign4(PointArgs a) {
    if ((int)blockIdx.x >= *a.n_tiles) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PSmem4 &S = *reinterpret_cast<PSmem4 *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int4 T = a.tiles[blockIdx.x];
    // a chunk whose bin is stable (no candidate changed) keeps every label: it adds
    // the per-cluster sums it cached when it last ran (not in the final pass, which
    // writes the record-order labels)
    if (a.pcache && a.reuse && !a.labels_out && a.accumulate && a.bin_stable[T.x]) {
        const PointCache &pc = a.pcache[blockIdx.x];
        const int pn = pc.n;
        if (pn >= 0) {
            for (int e = threadIdx.x; e < pn * 6; e += NT) {
                const int ce = e / 6, q = e - 6 * ce;
                unsigned long long *dst = a.acc + (size_t)pc.id[ce] * MFSEG_ACC_WORDS;
                if (q == 5) atomicAdd(dst + 12, pc.cnt[ce]);
                else atomic_add_fix(dst + (q < 4 ? 2 * q : 8), pc.w[ce][2 * q], (long long)pc.w[ce][2 * q + 1]);
            }
            return;
        }
    }
    const double *box = a.tile_box + 8 * (size_t)blockIdx.x;   // lo[4], hi[4]
    const double Cd[4] = {a.Cx, a.Cy, a.Cz, a.Ct};
    int ovf_local = 0;
    if (tid == 0) S.plisted = 0;
    if (tid < 4) {   // chunk frame: origin, guard bands, fp32 box half-widths
        const int d = tid;
        const double sc = d == 3 ? a.cf : 1.0;
        S.ctx.o[d] = box[d];
        S.ctx.delta[d] = (float)(DMUL(DMUL(DADD(DSUB(box[4 + d], box[d]), Cd[d]), sc), 0x1.0p-21));
        S.ctx.Cf[d] = (float)DMUL(Cd[d], sc);
    }
    __syncthreads();
    // initial pass (seeds as centres, w_v = 0): a chunk whose exact box lies inside
    // its bin with the margin seeds_fast_ok (run.cu) proves takes the bin's own seed
    // (id = bin) for every point -- the unique nearest valid candidate
    bool fast0 = false;
    if (a.seeds_fast) {
        fast0 = true;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const double ul = DDIV(DSUB(box[d], a.mn[d]), Cd[d]), uh = DDIV(DSUB(box[4 + d], a.mn[d]), Cd[d]);
            const double fl = floor(ul), fh = floor(uh);
            if (!(fl >= 0.0 && fl == fh && fl < (double)a.kk[d] && DSUB(ul, fl) >= 0x1.0p-20 &&
                  DSUB(uh, fh) <= 1.0 - 0x1.0p-20))
                fast0 = false;
        }
    }
    const int L0 = fast0 ? 0 : a.g.cand_start[T.x], L1 = fast0 ? 0 : a.g.cand_start[T.x + 1];
    bool deferred = (L1 - L0) > CR * NT;
    int cnt = 0;
    float cvmax = 0.f;
    if (fast0) {
        cnt = 1;
        if (tid == 0) S.id[0] = T.x;
        if (a.accumulate) {
            if (tid == 0) S.n[0] = 0u;
            for (int e = tid; e < NW * 5 * CAP; e += NT) (&S.wsum[0][0][0])[e] = 0.0;
        }
    } else if (!deferred) {
        // ---- candidates classified against the chunk box (exact fp64), compacted
        bool have[CR], full[CR];
        int id[CR];
        double c4[CR][4];
        unsigned bal[CR];
#pragma unroll
        for (int r = 0; r < CR; ++r) {
            const int ci = L0 + tid + NT * r;
            have[r] = ci < L1;
            full[r] = false;
            id[r] = 0;
#pragma unroll
            for (int d = 0; d < 4; ++d) c4[r][d] = 0.0;
            if (have[r]) {
                id[r] = a.g.cand_ids[ci];
                c4[r][0] = a.c.x[id[r]];
                c4[r][1] = a.c.y[id[r]];
                c4[r][2] = a.c.z[id[r]];
                c4[r][3] = a.c.t[id[r]];
                full[r] = true;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const double da = DSUB(c4[r][d], box[d]), db = DSUB(c4[r][d], box[4 + d]);   // da >= db
                    if (da < -Cd[d] || db > Cd[d]) have[r] = false;    // no sample passes
                    if (!(da <= Cd[d] && db >= -Cd[d])) full[r] = false;   // not every sample
                }
                if (!have[r]) full[r] = false;
            }
            bal[r] = __ballot_sync(0xffffffffu, have[r]);
            if (lane == 0) S.wc[r * NW + w] = __popc(bal[r]);
        }
        // the kept candidates' values, loaded before the compaction's barrier
        bool chs[CR];
        double cvv[CR];
#pragma unroll
        for (int r = 0; r < CR; ++r) {
            chs[r] = have[r] && a.chas[id[r]] != 0;
            cvv[r] = chs[r] ? a.cval[id[r]] : 0.0;
        }
        __syncthreads();
        int off[CR];
#pragma unroll
        for (int r = 0; r < CR; ++r) off[r] = 0;
#pragma unroll
        for (int q = 0; q < CR * NW; ++q) {
#pragma unroll
            for (int r = 0; r < CR; ++r) off[r] += q < r * NW + w ? S.wc[q] : 0;
            cnt += S.wc[q];
        }
        deferred = cnt > CAP;
        float mycv = 0.f;
#pragma unroll
        for (int r = 0; r < CR; ++r) {
            if (!deferred && have[r]) {
                const int p = off[r] + __popc(bal[r] & ((1u << lane) - 1u));
                const bool chas = chs[r];
                const double cv = cvv[r];
                S.id[p] = id[r];
                S.c[p][0] = c4[r][0];
                S.c[p][1] = c4[r][1];
                S.c[p][2] = c4[r][2];
                S.c[p][3] = c4[r][3];
                S.c[p][4] = cv;
                S.rc[p] = make_float4((float)DSUB(c4[r][0], S.ctx.o[0]), (float)DSUB(c4[r][1], S.ctx.o[1]),
                                      (float)DSUB(c4[r][2], S.ctx.o[2]),
                                      (float)DMUL(DSUB(c4[r][3], S.ctx.o[3]), a.cf));
                S.cvf[p] = (float)cv;
                S.wvf[p] = (USEVAL && chas) ? (float)a.wv : 0.f;
                S.has[p] = chas;
                S.full[p] = full[r];
                if (USEVAL && chas) mycv = fmaxf(mycv, fabsf((float)cv));
            }
        }
        if (USEVAL) {
            mycv = wmax_f(mycv);
            if (lane == 0) S.red[w] = mycv;
        }
        __syncthreads();
        if (USEVAL) {
#pragma unroll
            for (int q = 0; q < NW; ++q) cvmax = fmaxf(cvmax, S.red[q]);
        }
        if (!deferred && a.accumulate) {
            for (int e = tid; e < cnt; e += NT) S.n[e] = 0u;
            for (int e = tid; e < NW * 5 * CAP; e += NT) (&S.wsum[0][0][0])[e] = 0.0;
        }
    }
    if (tid == 0) {
        PCtx &C = S.ctx;
        float eps = 0.f;
        for (int d = 0; d < 4; ++d) {
            C.iC[d] = 1.0f / C.Cf[d];
            C.cw[d] = C.Cf[d] + C.delta[d];
            C.cn[d] = C.Cf[d] - C.delta[d];
            eps = fmaxf(eps, C.delta[d] / C.Cf[d]);
        }
        eps = eps * 1.0001f + 0x1.0p-22f;
        C.uhi = 1.0f + eps;
        C.ulo = 1.0f - eps;
        const float D0 = C.delta[0], D1 = C.delta[1], D2 = C.delta[2], D3 = C.delta[3];
        C.ndelta = sqrtf(D0 * D0 + D1 * D1 + D2 * D2 + D3 * D3) * 1.0001f;
        C.slack = 3e-13f * (float)(a.wd + a.wv);
        C.Aabs = 1.1f * (float)a.wd * C.ndelta + C.slack;
        C.cvmax = cvmax;
        C.fwd = (float)a.wd;
        C.wvf = USEVAL ? (float)a.wv : 0.f;
        C.cnt = cnt;
        C.nrounds = (cnt + 31) >> 5;
        if (DEVICE_STATS(a)) atomicAdd(a.stats + 11 + min(max(C.nrounds, 1), 4), 1ull);
        C.len = T.z;
        C.start = T.y;
        C.deferred = deferred;
        C.stable = fast0 || (a.reuse && !deferred && cnt > 0 && a.bin_stable[T.x]);
        C.fast0 = fast0;
    }
    __syncthreads();
    const PCtx &C = S.ctx;
    if (C.nrounds <= 3) {
        for (int wt = w; 64 * wt < C.len; wt += NW) point_warp<USEVAL, 3>(a, S, C, wt, ovf_local);
    } else {
        for (int wt = w; 64 * wt < C.len; wt += NW) point_warp<USEVAL, 4>(a, S, C, wt, ovf_local);
    }

    // ---- once per CTA: exact per-slot totals -> global 128-bit sums (and into the
    // chunk cache when no point went to the stranded / deferred lists: up to PC_MAX)
    if (a.accumulate && !deferred && cnt > 0) {
        __syncthreads();
        bool cache = a.pcache != nullptr && S.plisted == 0;
        if (cache) {
            if (w == 0) {
                int base = 0;
                for (int r = 0; 32 * r < cnt; ++r) {
                    const int sl = 32 * r + lane;
                    const bool nz = sl < cnt && S.n[sl] != 0;
                    const unsigned b = __ballot_sync(0xffffffffu, nz);
                    if (sl < cnt) S.pcidx[sl] = nz ? base + __popc(b & ((1u << lane) - 1u)) : -1;
                    base += __popc(b);
                }
                if (lane == 0) S.pcnz = base;
            }
            __syncthreads();
            cache = S.pcnz <= PC_MAX;
            if (tid == 0) a.pcache[blockIdx.x].n = cache ? S.pcnz : -1;
        } else if (tid == 0 && a.pcache) {
            a.pcache[blockIdx.x].n = -1;
        }
        for (int e = tid; e < cnt * 6; e += NT) {
            const int s = e / 6, wd = e - s * 6;
            const unsigned n = S.n[s];
            if (n == 0) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            PointCache *pcp = cache ? a.pcache + blockIdx.x : nullptr;
            const int ce = cache ? S.pcidx[s] : -1;
            if (wd == 5) {
                atomicAdd(dst + 12, (unsigned long long)n);   // n_points
                if (pcp) {
                    pcp->id[ce] = S.id[s];
                    pcp->cnt[ce] = (unsigned long long)n;
                }
                continue;
            }
            __int128 acc = 0;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                unsigned long long lo;
                long long hi;
                d2fix(S.wsum[q][wd][s], lo, hi, &ovf_local);
                acc += (__int128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
            }
            atomic_add_fix(dst + (wd < 4 ? 2 * wd : 8), (unsigned long long)acc, (long long)(acc >> 64));
            if (pcp) {
                pcp->w[ce][2 * wd] = (unsigned long long)acc;
                pcp->w[ce][2 * wd + 1] = (unsigned long long)(acc >> 64);
            }
        }
    } else if (tid == 0 && a.pcache) {
        a.pcache[blockIdx.x].n = -1;
    }
    if (ovf_local) *a.overflow = 1;
}

// Once per run, one CTA per point chunk: the exact fp64 bounding box of the
// chunk, then for each 64-point warp tile (warp w takes tiles w, w + 8, ...)
// the chunk-relative fp32 box, the fl32(value) range and the fixed-order sums
// -- the same formulas k_point_assign4 uses.  The second read of the chunk's
// points hits the cache.
// GATHER: the chunk's points are first gathered from the caller's arrays through
// the sort permutation (and written to the bin-sorted SoA), so the sorted points
// are read from HBM once, here, instead of by a separate gather pass.
template <bool GATHER>
__global__ void __launch_bounds__(256) k_chunk_boxes(const int4 *tiles, const int *n_tiles,
                                                      double *x, double *y, double *z, double *t,
                                                      double *v, const unsigned *perm,
                                                      const double *gxyz, const double *gt,
                                                      const double *gv, double cf, double *box,
                                                      WBox *out, unsigned long long *absmax) {
    constexpr int TPW = POINT_CHUNK / 64 / 8;   // warp tiles per warp
    __shared__ double red[8][8];
    __shared__ double amax_s[8][5];
    __shared__ int bad_s;
    __shared__ double o[4];
    const long long tile = blockIdx.x;
    if (tile >= *n_tiles) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int4 T = tiles[tile];
    // every point of the chunk once, in registers: warp w holds its warp tiles
    // w + 8 j, lane l points l and l + 32 of each
    double P[TPW][2][5];
#pragma unroll
    for (int j = 0; j < TPW; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int off = 64 * (w + 8 * j) + lane + 32 * q;
            const long long p = (long long)T.y + min(off, T.z - 1);   // clamped: box unaffected
            if (GATHER) {
                const long long src = perm[p];
                P[j][q][0] = __ldg(gxyz + 3 * src);
                P[j][q][1] = __ldg(gxyz + 3 * src + 1);
                P[j][q][2] = __ldg(gxyz + 3 * src + 2);
                P[j][q][3] = __ldg(gt + src);
                P[j][q][4] = __ldg(gv + src);
            } else {
                P[j][q][0] = x[p];
                P[j][q][1] = y[p];
                P[j][q][2] = z[p];
                P[j][q][3] = t[p];
                P[j][q][4] = v[p];
            }
        }
    if (GATHER) {
#pragma unroll
        for (int j = 0; j < TPW; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int off = 64 * (w + 8 * j) + lane + 32 * q;
                if (off < T.z) {
                    const long long p = (long long)T.y + off;
                    x[p] = P[j][q][0];
                    y[p] = P[j][q][1];
                    z[p] = P[j][q][2];
                    t[p] = P[j][q][3];
                    v[p] = P[j][q][4];
                }
            }
    }
    {   // range check of the fixed-point sums: max |x|, |y|, |z|, |t|, |v| and non-finite inputs
        if (tid == 0) bad_s = 0;
        bool bad = false;
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            double m = 0.0;
#pragma unroll
            for (int j = 0; j < TPW; ++j)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    m = fmax(m, fabs(P[j][q][d]));
                    bad |= !isfinite(P[j][q][d]);
                }
            m = wmax_d(m);
            if (lane == 0) amax_s[w][d] = m;
        }
        __syncthreads();
        if (bad) bad_s = 1;
        __syncthreads();
        if (tid < 5) {   // atomics only when they raise the maximum
            double m = amax_s[0][tid];
            for (int q = 1; q < 8; ++q) m = fmax(m, amax_s[q][tid]);
            const unsigned long long mk = (unsigned long long)__double_as_longlong(m);
            if (mk > *(volatile unsigned long long *)(absmax + tid)) atomicMax(absmax + tid, mk);
        }
        if (tid == 0 && bad_s) atomicOr(absmax + 6, 1ull);
    }
    double lo[4], hi[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        lo[d] = P[0][0][d];
        hi[d] = P[0][0][d];
#pragma unroll
        for (int j = 0; j < TPW; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                lo[d] = fmin(lo[d], P[j][q][d]);
                hi[d] = fmax(hi[d], P[j][q][d]);
            }
        lo[d] = wmin_d(lo[d]);
        hi[d] = wmax_d(hi[d]);
    }
    if (lane < 4) {
        double l = lo[0], h = hi[0];
#pragma unroll
        for (int d = 1; d < 4; ++d)
            if (lane == d) {
                l = lo[d];
                h = hi[d];
            }
        red[w][lane] = l;
        red[w][4 + lane] = h;
    }
    __syncthreads();
    if (tid < 8) {
        double r = red[0][tid];
        for (int q = 1; q < 8; ++q) r = tid < 4 ? fmin(r, red[q][tid]) : fmax(r, red[q][tid]);
        box[8 * tile + tid] = r;
        if (tid < 4) o[tid] = r;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
        const int wt = w + 8 * j;
        if (64 * wt >= T.z) break;   // warp-uniform
        float flo[5], fhi[5];
        double sm[5];   // point_warp's record order: P0, then + P1
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            flo[d] = INF_F;
            fhi[d] = -INF_F;
            sm[d] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (64 * wt + lane + 32 * q >= T.z) continue;
#pragma unroll
            for (int d = 0; d < 5; ++d) sm[d] = q == 0 ? P[j][q][d] : DADD(sm[d], P[j][q][d]);
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const float r = (float)DMUL(DSUB(P[j][q][d], o[d]), d == 3 ? cf : 1.0);
                flo[d] = fminf(flo[d], r);
                fhi[d] = fmaxf(fhi[d], r);
            }
            const float fv = (float)P[j][q][4];
            flo[4] = fminf(flo[4], fv);
            fhi[4] = fmaxf(fhi[4], fv);
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            flo[d] = wmin_f(flo[d]);
            fhi[d] = wmax_f(fhi[d]);
            sm[d] = warp_sum_d(sm[d]);
        }
        if (lane == 0) {
            WBox b;
            b.lo = make_float4(flo[0], flo[1], flo[2], flo[3]);
            b.hi = make_float4(fhi[0], fhi[1], fhi[2], fhi[3]);
            b.v = make_float2(flo[4], fhi[4]);
            b.pad = make_float2(0.f, 0.f);
#pragma unroll
            for (int d = 0; d < 5; ++d) b.s[d] = sm[d];
            b.pad2 = 0.0;
            out[tile * (POINT_CHUNK / 64) + wt] = b;
        }
    }
}

int launch_tile_box(unsigned long long *absmax, const int4 *tiles, const int *n_tiles, long long max_tiles, double *x, double *y,
                    double *z, double *t, double *v, double cf, double *box, WBox *wbox,
                    const unsigned *perm, const double *gxyz, const double *gt, const double *gv,
                    cudaStream_t st) {
    if (max_tiles <= 0) return 0;
    if (max_tiles > 0x7fffffffll) {
        set_error("point chunk grid too large");
        return 3;
    }
    ::mfseg::count_launch();
    if (perm)
        k_chunk_boxes<true><<<(unsigned)max_tiles, 256, 0, st>>>(tiles, n_tiles, x, y, z, t, v, perm, gxyz,
                                                                 gt, gv, cf, box, wbox, absmax);
    else
        k_chunk_boxes<false><<<(unsigned)max_tiles, 256, 0, st>>>(tiles, n_tiles, x, y, z, t, v, nullptr,
                                                                  nullptr, nullptr, nullptr, cf, box, wbox, absmax);
    MFSEG_LAUNCH("k_chunk_boxes");
    return 0;
}

int launch_point_assign_v4(const PointArgs &a, long long max_tiles, cudaStream_t st) {
    if (max_tiles <= 0) return 0;
    if (max_tiles > 0x7fffffffll) {
        set_error("point chunk grid too large");
        return 3;
    }
    const size_t smem = sizeof(PSmem4);
    static bool configured = false;
    if (!configured) {
        MFSEG_CUDA(cudaFuncSetAttribute(k_point_assign4<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MFSEG_CUDA(cudaFuncSetAttribute(k_point_assign4<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    ::mfseg::count_launch();
    if (a.wv > 0.0)
        k_point_assign4<true><<<(unsigned)max_tiles, NT, smem, st>>>(a);
    else
        k_point_assign4<false><<<(unsigned)max_tiles, NT, smem, st>>>(a);
    MFSEG_LAUNCH("k_point_assign4");
    return 0;
}

}  // namespace mfseg
