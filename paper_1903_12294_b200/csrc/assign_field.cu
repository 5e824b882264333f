// k_field_assign — windowed exact assignment of field samples, v2.
//
// Same result as the reference's _assign_chunk / _metric (engine.py:137-192)
// for every field sample: argmin over valid candidates of the fp64 D computed
// in the reference's operation order, lowest id on ties.  What changes is how
// few (sample, centre) pairs are evaluated in fp64:
//
//  1. tile level (16x8x4 voxels of one timestep, one sample bin): for each
//     candidate of the bin's neighbour list, exact fp64 lower/upper bounds of D
//     over the tile (all ops monotone); candidates whose lower bound exceeds the
//     best whole-tile upper bound are dropped (typically ~52 -> ~12).
//  2. per survivor, fp32 tables of the per-axis squared distances over the
//     tile (dx^2[16], dy^2[8], dz^2+dt^2[4], computed in fp64 and rounded once;
//     +inf where the box test |c - s| <= C fails).
//  3. warp level (4x4x4 sub-brick): fp32 bounds from the tables, culled with a
//     relative margin k = 2^-16 (>> the 2^-19 error bound of the fp32 path).
//  4. per sample: fp32 screen d32 ~ D with |d32 - D| <= 2^-19 (D + W),
//     W = w_v (|v| + max|c_v|), tracking best and second best.  If
//     d2 (1-k) > d1 (1+k) + 2 k W (k = 2^-18) the best is provably the exact
//     argmin; otherwise every candidate within that margin is re-evaluated in
//     exact fp64 (rare: near-ties).
//  5. accumulation in exact 128-bit fixed point: x/y/z/t sums as
//     (per-row counts from ballots) x (fixed-point coordinate tables), value
//     sums as a warp int128 butterfly; shared-memory integer tables per tile
//     survivor, then one global atomic per (cluster, word) per tile.  Integer
//     sums are order-free, so results do not depend on tiling or GPU count.
#include <climits>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();
constexpr float FLT_BIG = 3.4028234663852886e38f;

constexpr int TX = 16, TY = 8, TZ = 4;
constexpr int NT = 256, NW = 8;
constexpr int SCAP = 64;            // survivors handled by the fast path
constexpr float KSCR = 0x1.0p-18f;  // screen margin (2x the proven 2^-19 bound)
constexpr float KCULL = 0x1.0p-16f; // warp-cull margin

__device__ __forceinline__ void axis_range(double c, double lo, double hi, double &dmin,
                                           double &dmax) {
    double a = DSUB(c, lo), b = DSUB(c, hi);
    double fa = fabs(a), fb = fabs(b);
    dmax = fmax(fa, fb);
    dmin = (b <= 0.0 && a >= 0.0) ? 0.0 : fmin(fa, fb);
}

__device__ __forceinline__ double bound_D(double dx, double dy, double dz, double tsq, double vt,
                                          double wd) {
    double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    return DADD(vt, DMUL(wd, DSQRT(DADD(q, tsq))));
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float to_f(double x) {   // round once, saturate, keep +inf
    float f = __double2float_rn(x);
    return fminf(f, FLT_BIG);
}

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
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

// 128-bit helpers (two's complement in (lo, hi))
__device__ __forceinline__ void add128(unsigned long long &lo, long long &hi,
                                       unsigned long long blo, long long bhi) {
    unsigned long long n = lo + blo;
    hi = hi + bhi + (n < lo ? 1 : 0);
    lo = n;
}
__device__ __forceinline__ void warp_sum128(unsigned long long &lo, long long &hi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long ol = __shfl_xor_sync(0xffffffffu, lo, o);
        long long oh = __shfl_xor_sync(0xffffffffu, hi, o);
        add128(lo, hi, ol, oh);
    }
}
__device__ __forceinline__ void smem_add128(unsigned long long *p, unsigned long long lo,
                                            long long hi) {
    if (lo == 0 && hi == 0) return;
    unsigned long long old = atomicAdd(p, lo);
    unsigned long long h = (unsigned long long)hi + ((old + lo < old) ? 1ull : 0ull);
    if (h) atomicAdd(p + 1, h);
}

// exact fp64 D of one (sample, survivor) pair; the box test must already hold
__device__ __forceinline__ double exact_D(const double *c, double px, double py, double pz,
                                          double v, bool has, double wv, double wd) {
    double dx = DSUB(c[0], px), dy = DSUB(c[1], py), dz = DSUB(c[2], pz);
    double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    return metric_tail(q, c[3], v, c[4], has, wv, wd);
}

struct Smem {
    double x[TX], y[TY], z[TZ];
    unsigned long long xf[TX][2], yf[TY][2], zf[TZ][2], tf[2];
    int id[SCAP];
    double c[SCAP][5];                     // cx, cy, cz, tsq, cv (0 when absent)
    unsigned char has[SCAP];
    float cvf[SCAP], wvf[SCAP];
    float dx2[SCAP][TX], dy2[SCAP][TY], dz2[SCAP][TZ];
    unsigned long long acc[SCAP][11];      // x,y,z,t,v as (lo,hi) + count
    double red[2 * NW];
    float redf[NW];
    int wc[NW];
};

}  // namespace

__global__ void __launch_bounds__(NT, 3) k_field_assign2(FieldArgs a) {
    __shared__ Smem S;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    long long tile = blockIdx.x;
    const int txi = (int)(tile % a.ntx);
    tile /= a.ntx;
    const int tyi = (int)(tile % a.nty);
    tile /= a.nty;
    const int tzi = (int)(tile % a.ntz);
    const int m = (int)(tile / a.ntz);
    const AxisTile X = a.xt[txi], Y = a.yt[tyi], Z = a.zt[tzi];
    const double tm = a.times[m];
    int ovf_local = 0;
    if (tid < TX) {
        double xv = cell_coord(a.ox, a.sx, X.start + tid);
        S.x[tid] = xv;
        long long hi;
        d2fix(xv, S.xf[tid][0], hi, &ovf_local);
        S.xf[tid][1] = (unsigned long long)hi;
    } else if (tid < TX + TY) {
        int j = tid - TX;
        double yv = cell_coord(a.oy, a.sy, Y.start + j);
        S.y[j] = yv;
        long long hi;
        d2fix(yv, S.yf[j][0], hi, &ovf_local);
        S.yf[j][1] = (unsigned long long)hi;
    } else if (tid < TX + TY + TZ) {
        int k = tid - TX - TY;
        double zv = cell_coord(a.oz, a.sz, Z.start + k);
        S.z[k] = zv;
        long long hi;
        d2fix(zv, S.zf[k][0], hi, &ovf_local);
        S.zf[k][1] = (unsigned long long)hi;
    } else if (tid == TX + TY + TZ) {
        long long hi;
        d2fix(tm, S.tf[0], hi, &ovf_local);
        S.tf[1] = (unsigned long long)hi;
    }
    const int sbin = ((a.tbin[m] * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;

    // ---- this lane's two samples: (lx, ly, lz) and (lx, ly, lz + 2) of warp w's 4x4x4 brick
    const int bx = (w & 3) * 4, by = (w >> 2) * 4;
    const int lx = bx + (lane & 3), ly = by + ((lane >> 2) & 3), lz0 = lane >> 4;
    const bool rowok = lx < X.len && ly < Y.len;
    const bool live0 = rowok && lz0 < Z.len, live1 = rowok && lz0 + 2 < Z.len;
    const long long row = (((long long)m * a.nz + Z.start) * a.ny + (Y.start + ly)) * (long long)a.nx +
                          (X.start + lx);
    const long long plane = (long long)a.ny * a.nx;
    const long long f0 = row + lz0 * plane, f1 = row + (lz0 + 2) * plane;
    const double v0 = live0 ? __ldg(a.values + f0) : 0.0;
    const double v1 = live1 ? __ldg(a.values + f1) : 0.0;
    // tile value range (phase A bounds) and warp value range (warp culling)
    double vlo = INF_D, vhi = -INF_D;
    if (live0) { vlo = v0; vhi = v0; }
    if (live1) { vlo = fmin(vlo, v1); vhi = fmax(vhi, v1); }
    const bool useval = a.wv > 0.0;
    double wvlo = vlo, wvhi = vhi;
    if (useval) {
        wvlo = warp_min_d(vlo);
        wvhi = warp_max_d(vhi);
        if (lane == 0) {
            S.red[w] = wvlo;
            S.red[NW + w] = wvhi;
        }
    }
    __syncthreads();
    double tvlo = wvlo, tvhi = wvhi;
    if (useval) {
        tvlo = S.red[0];
        tvhi = S.red[NW];
#pragma unroll
        for (int q = 1; q < NW; ++q) {
            tvlo = fmin(tvlo, S.red[q]);
            tvhi = fmax(tvhi, S.red[NW + q]);
        }
    }

    int lab0 = -1, lab1 = -1;      // final labels (centre ids)
    int sl0 = -1, sl1 = -1;        // survivor slots (fast path accumulation)
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    const bool fast = (L1 - L0) <= NT;
    double bD0 = INF_D, bD1 = INF_D;   // exact-mode running best
    int bI0 = INT_MAX, bI1 = INT_MAX;
    int nsurv_fast = 0;                // > 0: labels came from the fast path's slots

    for (int cb = L0; cb < L1; cb += NT) {
        // ---- phase A: exact fp64 tile bounds, one candidate per thread
        const int ci = cb + tid;
        bool have = ci < L1;
        int id = 0;
        double cx = 0, cy = 0, cz = 0, cv = 0, tsq = 0, Dlo = INF_D, Dhi = INF_D;
        bool chas = false, full = false;
        int xa = 0, xb = -1, ya = 0, yb = -1, za = 0, zb = -1;
        if (have) {
            id = a.g.cand_ids[ci];
            const int4 b0 = a.g.vbox[2 * id], b1 = a.g.vbox[2 * id + 1];
            xa = max(b0.x - X.start, 0);
            xb = min(b0.y - X.start, X.len - 1);
            ya = max(b0.z - Y.start, 0);
            yb = min(b0.w - Y.start, Y.len - 1);
            za = max(b1.x - Z.start, 0);
            zb = min(b1.y - Z.start, Z.len - 1);
            have = m >= b1.z && m <= b1.w && xa <= xb && ya <= yb && za <= zb;
            if (have) {
                cx = a.c.x[id];
                cy = a.c.y[id];
                cz = a.c.z[id];
                const double ct = DMUL(a.cf, DSUB(a.c.t[id], tm));
                tsq = DMUL(ct, ct);
                chas = a.chas[id] != 0;
                cv = chas ? a.cval[id] : 0.0;
                full = xa == 0 && xb == X.len - 1 && ya == 0 && yb == Y.len - 1 && za == 0 &&
                       zb == Z.len - 1;
                double dxl, dxh, dyl, dyh, dzl, dzh;
                axis_range(cx, S.x[xa], S.x[xb], dxl, dxh);
                axis_range(cy, S.y[ya], S.y[yb], dyl, dyh);
                axis_range(cz, S.z[za], S.z[zb], dzl, dzh);
                double vtl = 0.0, vth = 0.0;
                if (useval && chas) {
                    const double p = DSUB(tvlo, cv), q = DSUB(tvhi, cv);
                    const double fp = fabs(p), fq = fabs(q);
                    vtl = DMUL(a.wv, (p <= 0.0 && q >= 0.0) ? 0.0 : fmin(fp, fq));
                    vth = DMUL(a.wv, fmax(fp, fq));
                }
                Dlo = bound_D(dxl, dyl, dzl, tsq, vtl, a.wd);
                Dhi = bound_D(dxh, dyh, dzh, tsq, vth, a.wd);
            }
        }
        // ---- phase B: tile UB, survivors, compaction into the fast-path slots
        double ub = warp_min_d(full ? Dhi : INF_D);
        if (lane == 0) S.red[w] = ub;
        __syncthreads();
        ub = S.red[0];
#pragma unroll
        for (int q = 1; q < NW; ++q) ub = fmin(ub, S.red[q]);
        const bool surv = have && Dlo <= ub;
        const unsigned bal = __ballot_sync(0xffffffffu, surv);
        if (lane == 0) S.wc[w] = __popc(bal);
        __syncthreads();
        int off = 0, nsurv = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < w ? S.wc[q] : 0;
            nsurv += S.wc[q];
        }
        const bool fast_now = fast && nsurv <= SCAP;
        const int pos = off + __popc(bal & ((1u << lane) - 1u));
        // exact mode processes survivors in windows of SCAP
        for (int sb = 0; sb < nsurv; sb += SCAP) {
            const int cnt = min(SCAP, nsurv - sb);
            if (surv && pos >= sb && pos < sb + SCAP) {
                const int p = pos - sb;
                S.id[p] = id;
                S.c[p][0] = cx;
                S.c[p][1] = cy;
                S.c[p][2] = cz;
                S.c[p][3] = tsq;
                S.c[p][4] = cv;
                S.has[p] = chas;
                S.cvf[p] = (float)cv;
                S.wvf[p] = (useval && chas) ? (float)a.wv : 0.0f;
                // fp32 tables (+inf outside the box-test interval)
                for (int i = 0; i < TX; ++i) {
                    float e = INF_F;
                    if (i >= xa && i <= xb) {
                        const double d = DSUB(cx, S.x[i]);
                        e = to_f(DMUL(d, d));
                    }
                    S.dx2[p][i] = e;
                }
                for (int j = 0; j < TY; ++j) {
                    float e = INF_F;
                    if (j >= ya && j <= yb) {
                        const double d = DSUB(cy, S.y[j]);
                        e = to_f(DMUL(d, d));
                    }
                    S.dy2[p][j] = e;
                }
                for (int k = 0; k < TZ; ++k) {
                    float e = INF_F;
                    if (k >= za && k <= zb) {
                        const double d = DSUB(cz, S.z[k]);
                        e = to_f(DADD(DMUL(d, d), tsq));
                    }
                    S.dz2[p][k] = e;
                }
            }
            if (fast_now)
                for (int i = tid; i < cnt * 11; i += NT) (&S.acc[0][0])[i] = 0ull;
            __syncthreads();

            if (fast_now) {
                nsurv_fast = cnt;
                // ---- warp culling over the 4x4x4 brick (fp32 bounds from the tables)
                const float fwd = (float)a.wd;
                const float vwl = (float)wvlo, vwh = (float)wvhi;
                float cvmax = 0.0f;
                unsigned long long keep = 0ull;    // survivors kept by this warp (<= 64)
                float ubw = INF_F;
                float dl_mine[2] = {INF_F, INF_F};
                for (int r = 0; r < 2; ++r) {
                    const int s = lane + 32 * r;
                    if (s < cnt) {
                        float xmn = INF_F, xmx = 0.f, ymn = INF_F, ymx = 0.f, zmn = INF_F, zmx = 0.f;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int ix = bx + q, iy = by + q;
                            if (ix < X.len) {
                                xmn = fminf(xmn, S.dx2[s][ix]);
                                xmx = fmaxf(xmx, S.dx2[s][ix]);
                            }
                            if (iy < Y.len) {
                                ymn = fminf(ymn, S.dy2[s][iy]);
                                ymx = fmaxf(ymx, S.dy2[s][iy]);
                            }
                            if (q < Z.len) {
                                zmn = fminf(zmn, S.dz2[s][q]);
                                zmx = fmaxf(zmx, S.dz2[s][q]);
                            }
                        }
                        const float cvs = S.cvf[s], wvs = S.wvf[s];
                        const float pl = vwl - cvs, ph = vwh - cvs;
                        const float amin = (pl <= 0.f && ph >= 0.f) ? 0.f : fminf(fabsf(pl), fabsf(ph));
                        const float amax = fmaxf(fabsf(pl), fabsf(ph));
                        const float vtl = wvs > 0.f ? wvs * amin : 0.f;   // no 0 * inf
                        const float vth = wvs > 0.f ? wvs * amax : 0.f;
                        const float dl = fmaf(fwd, sqrt_approx((xmn + ymn) + zmn), vtl);
                        const float dh = fmaf(fwd, sqrt_approx((xmx + ymx) + zmx), vth);
                        dl_mine[r] = dl;                        // inf when no valid sample
                        ubw = fminf(ubw, dh);                   // inf unless valid on the whole brick
                        cvmax = fmaxf(cvmax, wvs > 0.f ? fabsf(cvs) : 0.f);
                    }
                }
                ubw = warp_min_f(ubw);
                cvmax = warp_max_f(cvmax);
                const float slack = 3e-13f * (float)(a.wd + a.wv);   // fp32 underflow of tiny terms
                const float Wb = (useval ? (float)a.wv * (fmaxf(fabsf(vwl), fabsf(vwh)) + cvmax) : 0.f) +
                                 slack;
                const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) / (1.f - KCULL);
                for (int r = 0; r < 2; ++r) {
                    const bool k = (lane + 32 * r) < cnt && (dl_mine[r] <= thr || (a.debug & 1));
                    keep |= (unsigned long long)__ballot_sync(0xffffffffu, k) << (32 * r);
                }
                // ---- per-sample fp32 screen over the kept survivors
                const float fv0 = (float)v0, fv1 = (float)v1;
                float b1a = INF_F, b2a = INF_F, b1b = INF_F, b2b = INF_F;
                int i1a = -1, i1b = -1;
                unsigned long long it = keep;
                while (it) {
                    const int s = __ffsll((long long)it) - 1;
                    it &= it - 1;
                    const float axy = S.dx2[s][lx] + S.dy2[s][ly];
                    const float cvs = S.cvf[s], wvs = S.wvf[s];
                    const float da = fmaf(fwd, sqrt_approx(axy + S.dz2[s][lz0]), wvs * fabsf(fv0 - cvs));
                    const float db = fmaf(fwd, sqrt_approx(axy + S.dz2[s][lz0 + 2]), wvs * fabsf(fv1 - cvs));
                    if (da < b1a) { b2a = b1a; b1a = da; i1a = s; } else { b2a = fminf(b2a, da); }
                    if (db < b1b) { b2b = b1b; b1b = db; i1b = s; } else { b2b = fminf(b2b, db); }
                }
                // ---- certify or resolve exactly
                const float Wa = (useval ? (float)a.wv * (fabsf(fv0) + cvmax) : 0.f) + slack;
                const float Wq = (useval ? (float)a.wv * (fabsf(fv1) + cvmax) : 0.f) + slack;
                const bool oka = b2a * (1.f - KSCR) > b1a * (1.f + KSCR) + 2.f * KSCR * Wa && b1a < INF_F &&
                                 !(a.debug & 2);
                const bool okb = b2b * (1.f - KSCR) > b1b * (1.f + KSCR) + 2.f * KSCR * Wq && b1b < INF_F &&
                                 !(a.debug & 2);
                sl0 = oka ? i1a : -1;
                sl1 = okb ? i1b : -1;
                const double px = S.x[lx < TX ? lx : 0], py = S.y[ly < TY ? ly : 0];
                if ((live0 && !oka) || (live1 && !okb)) {
                    // every survivor within the margin (or any valid one when the
                    // screen overflowed) is evaluated in exact fp64
                    const float ta = b1a < INF_F ? (b1a * (1.f + KSCR) + 2.f * KSCR * Wa) / (1.f - KSCR) : INF_F;
                    const float tb = b1b < INF_F ? (b1b * (1.f + KSCR) + 2.f * KSCR * Wq) / (1.f - KSCR) : INF_F;
                    double eDa = INF_D, eDb = INF_D;
                    int eIa = INT_MAX, eIb = INT_MAX, eSa = -1, eSb = -1;
                    for (int s = 0; s < cnt; ++s) {
                        const bool vx = S.dx2[s][lx < TX ? lx : 0] != INF_F && S.dy2[s][ly < TY ? ly : 0] != INF_F;
                        const float axy = S.dx2[s][lx < TX ? lx : 0] + S.dy2[s][ly < TY ? ly : 0];
                        const float cvs = S.cvf[s], wvs = S.wvf[s];
                        const int cid = S.id[s];
                        if (live0 && !oka && vx && S.dz2[s][lz0] != INF_F) {
                            const float d = fmaf(fwd, sqrt_approx(axy + S.dz2[s][lz0]), wvs * fabsf(fv0 - cvs));
                            if (!(d > ta)) {
                                const double D = exact_D(S.c[s], px, py, S.z[lz0], v0, S.has[s], a.wv, a.wd);
                                if (better(D, cid, eDa, eIa)) { eDa = D; eIa = cid; eSa = s; }
                            }
                        }
                        if (live1 && !okb && vx && S.dz2[s][lz0 + 2] != INF_F) {
                            const float d = fmaf(fwd, sqrt_approx(axy + S.dz2[s][lz0 + 2]), wvs * fabsf(fv1 - cvs));
                            if (!(d > tb)) {
                                const double D = exact_D(S.c[s], px, py, S.z[lz0 + 2], v1, S.has[s], a.wv, a.wd);
                                if (better(D, cid, eDb, eIb)) { eDb = D; eIb = cid; eSb = s; }
                            }
                        }
                    }
                    if (live0 && !oka) sl0 = eSa;
                    if (live1 && !okb) sl1 = eSb;
                }
                lab0 = (live0 && sl0 >= 0) ? S.id[sl0] : -1;
                lab1 = (live1 && sl1 >= 0) ? S.id[sl1] : -1;
                if (!live0) sl0 = -1;
                if (!live1) sl1 = -1;
            } else {
                // ---- exact mode (crowded bins): every valid survivor in fp64
                const double px = S.x[lx < TX ? lx : 0], py = S.y[ly < TY ? ly : 0];
                for (int s = 0; s < cnt; ++s) {
                    const int cid = S.id[s];
                    const bool vx = S.dx2[s][lx < TX ? lx : 0] != INF_F && S.dy2[s][ly < TY ? ly : 0] != INF_F;
                    if (live0 && vx && S.dz2[s][lz0] != INF_F) {
                        const double D = exact_D(S.c[s], px, py, S.z[lz0], v0, S.has[s], a.wv, a.wd);
                        if (better(D, cid, bD0, bI0)) { bD0 = D; bI0 = cid; }
                    }
                    if (live1 && vx && S.dz2[s][lz0 + 2] != INF_F) {
                        const double D = exact_D(S.c[s], px, py, S.z[lz0 + 2], v1, S.has[s], a.wv, a.wd);
                        if (better(D, cid, bD1, bI1)) { bD1 = D; bI1 = cid; }
                    }
                }
            }
            __syncthreads();   // slots are rewritten by the next window
            if (fast_now) break;
        }
        if (fast_now) break;   // the fast path consumed the single candidate chunk
    }
    if (nsurv_fast == 0) {   // exact mode (or no candidates at all: stranded)
        lab0 = (live0 && bI0 != INT_MAX) ? bI0 : -1;
        lab1 = (live1 && bI1 != INT_MAX) ? bI1 : -1;
        sl0 = sl1 = -1;
    }
    // ---- labels + stranded list
    if (live0) {
        a.labels[f0] = lab0;
        if (lab0 < 0) {
            const unsigned long long p = atomicAdd(a.n_stranded, 1ull);
            if ((long long)p < a.stranded_cap) a.stranded[p] = f0;
        }
    }
    if (live1) {
        a.labels[f1] = lab1;
        if (lab1 < 0) {
            const unsigned long long p = atomicAdd(a.n_stranded, 1ull);
            if ((long long)p < a.stranded_cap) a.stranded[p] = f1;
        }
    }
    if (!a.accumulate) {
        if (ovf_local) *a.overflow = 1;
        return;
    }
    // ---- exact accumulation
    if (nsurv_fast > 0) {
        unsigned long long vl0 = 0, vl1 = 0;
        long long vh0 = 0, vh1 = 0;
        if (sl0 >= 0) d2fix(v0, vl0, vh0, &ovf_local);
        if (sl1 >= 0) d2fix(v1, vl1, vh1, &ovf_local);
        unsigned p0 = __ballot_sync(0xffffffffu, sl0 >= 0), p1 = __ballot_sync(0xffffffffu, sl1 >= 0);
        while (p0 | p1) {
            const int L = p0 ? __shfl_sync(0xffffffffu, sl0, __ffs(p0) - 1)
                             : __shfl_sync(0xffffffffu, sl1, __ffs(p1) - 1);
            const unsigned m0 = __ballot_sync(0xffffffffu, sl0 == L);
            const unsigned m1 = __ballot_sync(0xffffffffu, sl1 == L);
            unsigned long long lo = 0;
            long long hi = 0;
            if (sl0 == L) add128(lo, hi, vl0, vh0);
            if (sl1 == L) add128(lo, hi, vl1, vh1);
            warp_sum128(lo, hi);
            unsigned long long *acc = S.acc[L];
            // marginal counts x per-axis fixed-point coordinates (lanes 0..12)
            if (lane < 4) {
                const unsigned M = 0x11111111u << lane;
                const unsigned c = __popc(m0 & M) + __popc(m1 & M);
                if (c) {
                    const __int128 v = ((__int128)(long long)S.xf[bx + lane][1] << 64 |
                                        (__int128)S.xf[bx + lane][0]) * (__int128)c;
                    smem_add128(acc + 0, (unsigned long long)v, (long long)(v >> 64));
                }
            } else if (lane < 8) {
                const int q = lane - 4;
                const unsigned M = 0x000F000Fu << (4 * q);
                const unsigned c = __popc(m0 & M) + __popc(m1 & M);
                if (c) {
                    const __int128 v = ((__int128)(long long)S.yf[by + q][1] << 64 |
                                        (__int128)S.yf[by + q][0]) * (__int128)c;
                    smem_add128(acc + 2, (unsigned long long)v, (long long)(v >> 64));
                }
            } else if (lane < 12) {
                const int q = lane - 8;
                const unsigned mm = q < 2 ? m0 : m1;
                const unsigned c = __popc((q & 1) ? (mm >> 16) : (mm & 0xFFFFu));
                if (c) {
                    const __int128 v = ((__int128)(long long)S.zf[q][1] << 64 |
                                        (__int128)S.zf[q][0]) * (__int128)c;
                    smem_add128(acc + 4, (unsigned long long)v, (long long)(v >> 64));
                }
            } else if (lane == 12) {
                const unsigned c = __popc(m0) + __popc(m1);
                const __int128 v = ((__int128)(long long)S.tf[1] << 64 | (__int128)S.tf[0]) * (__int128)c;
                smem_add128(acc + 6, (unsigned long long)v, (long long)(v >> 64));
                atomicAdd(acc + 10, (unsigned long long)c);
            } else if (lane == 13) {
                smem_add128(acc + 8, lo, hi);
            }
            p0 &= ~m0;
            p1 &= ~m1;
        }
        __syncthreads();
        // ---- flush the tile's per-survivor sums: one global atomic per word
        for (int i = tid; i < nsurv_fast * 6; i += NT) {
            const int s = i / 6, wd = i % 6;
            const unsigned long long *src = S.acc[s];
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            if (src[10] == 0) continue;
            if (wd < 4) {
                atomic_add_fix(dst + 2 * wd, src[2 * wd], (long long)src[2 * wd + 1]);
            } else if (wd == 4) {
                atomic_add_fix(dst + 10, src[8], (long long)src[9]);   // field-value sum
            } else {
                atomicAdd(dst + 13, src[10]);                          // n_fields
            }
        }
    } else {
        // exact-mode tile: per-sample fixed point straight to the global sums
        const double px = S.x[lx < TX ? lx : 0], py = S.y[ly < TY ? ly : 0];
        const int labs[2] = {lab0, lab1};
        const double vs[2] = {v0, v1};
        for (int r = 0; r < 2; ++r) {
            const int L = labs[r];
            if (L < 0) continue;
            unsigned long long *dst = a.acc + (size_t)L * MFSEG_ACC_WORDS;
            atomic_add_double_fix(dst + 0, px, &ovf_local);
            atomic_add_double_fix(dst + 2, py, &ovf_local);
            atomic_add_double_fix(dst + 4, S.z[lz0 + 2 * r], &ovf_local);
            atomic_add_double_fix(dst + 6, tm, &ovf_local);
            atomic_add_double_fix(dst + 10, vs[r], &ovf_local);
            atomicAdd(dst + 13, 1ull);
        }
    }
    if (ovf_local) *a.overflow = 1;
}

}  // namespace mfseg

namespace mfseg {
int launch_field_assign_v2(const FieldArgs &a, long long ntiles, cudaStream_t st) {
    if (ntiles <= 0) return 0;
    if (ntiles > 0x7fffffffll) {
        set_error("field tile grid too large");
        return 3;
    }
    ::mfseg::count_launch();
    k_field_assign2<<<(unsigned)ntiles, NT, 0, st>>>(a);
    MFSEG_LAUNCH("k_field_assign2");
    return 0;
}
}  // namespace mfseg
