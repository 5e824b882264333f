// k_field_assign — windowed exact assignment of field samples (v3).
//
// Same result as the reference's _assign_chunk / _metric (engine.py:137-192)
// for every field sample: argmin over valid candidates of the fp64 D computed
// in the reference's operation order, lowest id on ties.  What changes is how
// few (sample, centre) pairs are evaluated in fp64:
//
//  1. tile level (16x8x4 voxels of one timestep inside one sample bin): for
//     each candidate of the bin's neighbour list, exact fp64 lower/upper bounds
//     of D over the tile (every fp64 op is monotone under round-to-nearest, so
//     the reference formula on extreme per-axis distances bounds every sample);
//     candidates whose lower bound exceeds the best whole-tile upper bound are
//     dropped (typically ~52 -> ~12).
//  2. per survivor, fp32 tables of the per-axis squared distances over the
//     tile (dx^2[16], dy^2[8], dz^2+dt^2[4], each computed in fp64 and rounded
//     once; +inf where the box test |c - s| <= C fails), built by all threads.
//  3. warp level (4x4x4 sub-brick): fp32 bounds from the tables, culled with
//     a relative margin 2^-16 (>> the 2^-19 error bound of the fp32 path).
//  4. per sample: fp32 screen d32 with |d32 - D| <= 2^-19 (D + W),
//     W = w_v (|v| + max|c_v|), tracking best and second best.  If
//     d2 (1-k) > d1 (1+k) + 2 k W (k = 2^-18) the best is provably the exact
//     argmin; otherwise every candidate inside that margin is re-evaluated in
//     exact fp64 (near-ties only: ~1e-3 of the warps).
//  5. accumulation: per warp and label one record without atomics — x/y/z/t
//     sums as (per-row counts from ballots) x (128-bit fixed-point coordinate
//     tables), the value sum as a fixed-order fp64 butterfly; per tile the
//     records are combined per (slot, word) and added to the 128-bit global
//     sums with one integer atomic each.  Tiles are canonical (never split
//     across GPUs) and integer addition is order-free, so the sums are
//     deterministic and independent of the GPU count.
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();
constexpr float FLT_BIG = 3.4028234663852886e38f;

constexpr int TX = 16, TY = 8, TZ = 4;
constexpr int NT = 256, NW = 8;
constexpr int SCAP = 64;            // survivors handled by the fast path
constexpr int TENT = TX + TY + TZ;  // table entries per survivor
constexpr int RMAX = 12;            // warp records kept in shared memory
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

// fp32 sqrt approximation; subnormal inputs flush to 0 (absolute error covered
// by the slack term of the screen margin)
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float to_f(double x) {   // round once, saturate finite values
    return fminf(__double2float_rn(x), FLT_BIG);
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

__device__ __forceinline__ void add128(unsigned long long &lo, long long &hi,
                                       unsigned long long blo, long long bhi) {
    unsigned long long n = lo + blo;
    hi = hi + bhi + (n < lo ? 1 : 0);
    lo = n;
}

// exact fp64 D of one (sample, survivor) pair; the box test must already hold
__device__ __forceinline__ double exact_D(const double *c, double px, double py, double pz,
                                          double v, bool has, double wv, double wd) {
    double dx = DSUB(c[0], px), dy = DSUB(c[1], py), dz = DSUB(c[2], pz);
    double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    return metric_tail(q, c[3], v, c[4], has, wv, wd);
}

struct Rec {                       // one (warp, label) partial sum
    int slot, n;
    unsigned long long f[4][2];    // x, y, z, t in 128-bit fixed point
    double v;                      // value sum (fixed-order fp64 butterfly)
};

struct Smem {
    double x[TX], y[TY], z[TZ];
    unsigned long long xf[TX][2], yf[TY][2], zf[TZ][2], tf[2];
    int id[SCAP];
    double c[SCAP][5];              // cx, cy, cz, tsq, cv (0 when absent)
    unsigned box[SCAP];             // xa | xb<<5 | ya<<10 | yb<<15 | za<<20 | zb<<25
    unsigned char has[SCAP];
    float cvf[SCAP], wvf[SCAP];
    float tab[SCAP][TENT];          // dx^2[16] | dy^2[8] | dz^2+dt^2[4]
    Rec rec[NW][RMAX];
    int nrec[NW];
    double red[2 * NW];
    int wc[NW];
};

__device__ __forceinline__ bool in_box(unsigned b, int sh, int i) {
    return i >= (int)((b >> sh) & 31u) && i <= (int)((b >> (sh + 5)) & 31u);
}

}  // namespace

__global__ void __launch_bounds__(NT, 3) k_field_assign3(FieldArgs a) {
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
    // tile coordinates (fp64, exact reference formula) + 128-bit fixed-point copies
    if (tid < TENT + 1) {
        double cv;
        unsigned long long *dst;
        if (tid < TX) {
            cv = cell_coord(a.ox, a.sx, X.start + tid);
            S.x[tid] = cv;
            dst = S.xf[tid];
        } else if (tid < TX + TY) {
            cv = cell_coord(a.oy, a.sy, Y.start + tid - TX);
            S.y[tid - TX] = cv;
            dst = S.yf[tid - TX];
        } else if (tid < TENT) {
            cv = cell_coord(a.oz, a.sz, Z.start + tid - TX - TY);
            S.z[tid - TX - TY] = cv;
            dst = S.zf[tid - TX - TY];
        } else {
            cv = tm;
            dst = S.tf;
        }
        long long hi;
        d2fix(cv, dst[0], hi, &ovf_local);
        dst[1] = (unsigned long long)hi;
    }
    const int sbin = ((a.tbin[m] * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;

    // ---- this lane's two samples: (lx, ly, lz0) and (lx, ly, lz0 + 2) of warp w's 4x4x4 brick
    const int bx = (w & 3) * 4, by = (w >> 2) * 4;
    const int lx = bx + (lane & 3), ly = by + ((lane >> 2) & 3), lz0 = lane >> 4;
    const bool rowok = lx < X.len && ly < Y.len;
    const bool live0 = rowok && lz0 < Z.len, live1 = rowok && lz0 + 2 < Z.len;
    const long long plane = (long long)a.ny * a.nx;
    const long long f0 = (((long long)m * a.nz + Z.start + lz0) * a.ny + (Y.start + ly)) * (long long)a.nx +
                         (X.start + lx);
    const long long f1 = f0 + 2 * plane;
    const double v0 = live0 ? __ldg(a.values + f0) : 0.0;
    const double v1 = live1 ? __ldg(a.values + f1) : 0.0;
    const bool useval = a.wv > 0.0;
    // warp value range (warp culling) and tile value range (phase A bounds)
    double wvlo = 0.0, wvhi = 0.0;
    if (useval) {
        double lo = INF_D, hi = -INF_D;
        if (live0) { lo = v0; hi = v0; }
        if (live1) { lo = fmin(lo, v1); hi = fmax(hi, v1); }
        wvlo = warp_min_d(lo);
        wvhi = warp_max_d(hi);
        if (lane == 0) {
            S.red[w] = wvlo;
            S.red[NW + w] = wvhi;
        }
    }
    __syncthreads();
    double tvlo = 0.0, tvhi = 0.0;
    if (useval) {
        tvlo = S.red[0];
        tvhi = S.red[NW];
#pragma unroll
        for (int q = 1; q < NW; ++q) {
            tvlo = fmin(tvlo, S.red[q]);
            tvhi = fmax(tvhi, S.red[NW + q]);
        }
    }

    int sl0 = -1, sl1 = -1;            // fast path: survivor slots of the two samples
    double bD0 = INF_D, bD1 = INF_D;   // exact mode: running best
    int bI0 = INT_MAX, bI1 = INT_MAX;
    int nfast = 0;                     // > 0: labels are fast-path slots
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    const bool single_chunk = (L1 - L0) <= NT;
    const double px = S.x[lx], py = S.y[ly], pz0 = S.z[lz0], pz1 = S.z[lz0 + 2];

    for (int cb = L0; cb < L1; cb += NT) {
        // ---- phase A: exact fp64 tile bounds, one candidate per thread
        const int ci = cb + tid;
        bool have = ci < L1;
        int id = 0;
        double cx = 0, cy = 0, cz = 0, cv = 0, tsq = 0, Dlo = INF_D, Dhi = INF_D;
        bool chas = false, full = false;
        unsigned box = 0;
        if (have) {
            id = a.g.cand_ids[ci];
            const int4 b0 = a.g.vbox[2 * id], b1 = a.g.vbox[2 * id + 1];
            const int xa = max(b0.x - X.start, 0), xb = min(b0.y - X.start, X.len - 1);
            const int ya = max(b0.z - Y.start, 0), yb = min(b0.w - Y.start, Y.len - 1);
            const int za = max(b1.x - Z.start, 0), zb = min(b1.y - Z.start, Z.len - 1);
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
                box = (unsigned)xa | ((unsigned)xb << 5) | ((unsigned)ya << 10) |
                      ((unsigned)yb << 15) | ((unsigned)za << 20) | ((unsigned)zb << 25);
            }
        }
        // ---- phase B: tile UB, survivor count and positions
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
        const bool fast = single_chunk && nsurv <= SCAP;
        const int pos = off + __popc(bal & ((1u << lane) - 1u));
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
                S.box[p] = box;
                S.has[p] = chas;
                S.cvf[p] = (float)cv;
                S.wvf[p] = (useval && chas) ? (float)a.wv : 0.0f;
            }
            __syncthreads();
            // fp32 distance tables, all threads (+inf outside the box-test interval)
            for (int e = tid; e < cnt * TENT; e += NT) {
                const int p = e / TENT, j = e - p * TENT;
                const unsigned b = S.box[p];
                float val = INF_F;
                if (j < TX) {
                    if (in_box(b, 0, j)) {
                        const double d = DSUB(S.c[p][0], S.x[j]);
                        val = to_f(DMUL(d, d));
                    }
                } else if (j < TX + TY) {
                    if (in_box(b, 10, j - TX)) {
                        const double d = DSUB(S.c[p][1], S.y[j - TX]);
                        val = to_f(DMUL(d, d));
                    }
                } else if (in_box(b, 20, j - TX - TY)) {
                    const double d = DSUB(S.c[p][2], S.z[j - TX - TY]);
                    val = to_f(DADD(DMUL(d, d), S.c[p][3]));
                }
                S.tab[p][j] = val;
            }
            __syncthreads();

            if (fast) {
                nfast = cnt;
                // ---- warp culling over the 4x4x4 brick (fp32 bounds from the tables)
                const float fwd = (float)a.wd;
                const float vwl = (float)wvlo, vwh = (float)wvhi;
                const float slack = 3e-13f * (float)(a.wd + a.wv);   // fp32 underflow of tiny terms
                float cvmax = 0.0f, ubw = INF_F;
                float dl_r[2] = {INF_F, INF_F};
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int s = lane + 32 * r;
                    if (s < cnt) {
                        const float *T = S.tab[s];
                        float xmn = INF_F, xmx = 0.f, ymn = INF_F, ymx = 0.f, zmn = INF_F, zmx = 0.f;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (bx + q < X.len) {
                                const float e = T[bx + q];
                                xmn = fminf(xmn, e);
                                xmx = fmaxf(xmx, e);
                            }
                            if (by + q < Y.len) {
                                const float e = T[TX + by + q];
                                ymn = fminf(ymn, e);
                                ymx = fmaxf(ymx, e);
                            }
                            if (q < Z.len) {
                                const float e = T[TX + TY + q];
                                zmn = fminf(zmn, e);
                                zmx = fmaxf(zmx, e);
                            }
                        }
                        const float wvs = S.wvf[s];
                        float vtl = 0.f, vth = 0.f;
                        if (wvs > 0.f) {   // no 0 * inf on lanes without live samples
                            const float cvs = S.cvf[s];
                            const float pl = vwl - cvs, ph = vwh - cvs;
                            vtl = wvs * ((pl <= 0.f && ph >= 0.f) ? 0.f : fminf(fabsf(pl), fabsf(ph)));
                            vth = wvs * fmaxf(fabsf(pl), fabsf(ph));
                            cvmax = fmaxf(cvmax, fabsf(cvs));
                        }
                        dl_r[r] = fmaf(fwd, sqrt_approx((xmn + ymn) + zmn), vtl);  // inf: no valid sample
                        ubw = fminf(ubw, fmaf(fwd, sqrt_approx((xmx + ymx) + zmx), vth));  // inf unless full
                    }
                }
                ubw = warp_min_f(ubw);
                cvmax = warp_max_f(cvmax);
                const float Wb = (useval ? (float)a.wv * (fmaxf(fabsf(vwl), fabsf(vwh)) + cvmax) : 0.f) +
                                 slack;
                const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) / (1.f - KCULL);
                unsigned keep0 = __ballot_sync(0xffffffffu, lane < cnt && (dl_r[0] <= thr || (a.debug & 1)));
                unsigned keep1 = __ballot_sync(0xffffffffu, lane + 32 < cnt && (dl_r[1] <= thr || (a.debug & 1)));
                // ---- per-sample fp32 screen over the kept survivors
                const float fv0 = (float)v0, fv1 = (float)v1;
                float b1a = INF_F, b2a = INF_F, b1b = INF_F, b2b = INF_F;
                int i1a = -1, i1b = -1;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    unsigned it = half ? keep1 : keep0;
                    while (it) {
                        const int s = __ffs(it) - 1 + 32 * half;
                        it &= it - 1;
                        const float *T = S.tab[s];
                        const float axy = T[lx] + T[TX + ly];
                        const float cvs = S.cvf[s], wvs = S.wvf[s];
                        const float da = fmaf(fwd, sqrt_approx(axy + T[TX + TY + lz0]), wvs * fabsf(fv0 - cvs));
                        const float db = fmaf(fwd, sqrt_approx(axy + T[TX + TY + lz0 + 2]), wvs * fabsf(fv1 - cvs));
                        if (da < b1a) { b2a = b1a; b1a = da; i1a = s; } else { b2a = fminf(b2a, da); }
                        if (db < b1b) { b2b = b1b; b1b = db; i1b = s; } else { b2b = fminf(b2b, db); }
                    }
                }
                // ---- certify or resolve exactly
                const float Wa = (useval ? (float)a.wv * (fabsf(fv0) + cvmax) : 0.f) + slack;
                const float Wq = (useval ? (float)a.wv * (fabsf(fv1) + cvmax) : 0.f) + slack;
                const bool oka = !(a.debug & 2) && b1a < INF_F &&
                                 b2a * (1.f - KSCR) > b1a * (1.f + KSCR) + 2.f * KSCR * Wa;
                const bool okb = !(a.debug & 2) && b1b < INF_F &&
                                 b2b * (1.f - KSCR) > b1b * (1.f + KSCR) + 2.f * KSCR * Wq;
                sl0 = oka ? i1a : -1;
                sl1 = okb ? i1b : -1;
                const bool need0 = live0 && !oka, need1 = live1 && !okb;
                if (__any_sync(0xffffffffu, need0 || need1)) {
                    // every survivor within the margin (or any valid one when the
                    // screen overflowed) is evaluated in exact fp64
                    const float ta = b1a < INF_F ? (b1a * (1.f + KSCR) + 2.f * KSCR * Wa) / (1.f - KSCR) : INF_F;
                    const float tb = b1b < INF_F ? (b1b * (1.f + KSCR) + 2.f * KSCR * Wq) / (1.f - KSCR) : INF_F;
                    double eDa = INF_D, eDb = INF_D;
                    int eIa = INT_MAX, eIb = INT_MAX, eSa = -1, eSb = -1;
                    if (need0 || need1) {
                        for (int s = 0; s < cnt; ++s) {
                            const float *T = S.tab[s];
                            const bool vxy = T[lx] != INF_F && T[TX + ly] != INF_F;
                            const float axy = T[lx] + T[TX + ly];
                            const float cvs = S.cvf[s], wvs = S.wvf[s];
                            const int cid = S.id[s];
                            if (need0 && vxy && T[TX + TY + lz0] != INF_F) {
                                const float d = fmaf(fwd, sqrt_approx(axy + T[TX + TY + lz0]), wvs * fabsf(fv0 - cvs));
                                if (!(d > ta)) {
                                    const double D = exact_D(S.c[s], px, py, pz0, v0, S.has[s], a.wv, a.wd);
                                    if (better(D, cid, eDa, eIa)) { eDa = D; eIa = cid; eSa = s; }
                                }
                            }
                            if (need1 && vxy && T[TX + TY + lz0 + 2] != INF_F) {
                                const float d = fmaf(fwd, sqrt_approx(axy + T[TX + TY + lz0 + 2]), wvs * fabsf(fv1 - cvs));
                                if (!(d > tb)) {
                                    const double D = exact_D(S.c[s], px, py, pz1, v1, S.has[s], a.wv, a.wd);
                                    if (better(D, cid, eDb, eIb)) { eDb = D; eIb = cid; eSb = s; }
                                }
                            }
                        }
                    }
                    if (need0) sl0 = eSa;
                    if (need1) sl1 = eSb;
                }
                if (!live0) sl0 = -1;
                if (!live1) sl1 = -1;
                break;   // the fast path consumed the single window
            }
            // ---- exact mode (crowded bins): every valid survivor of the window in fp64
            for (int s = 0; s < cnt; ++s) {
                const float *T = S.tab[s];
                const int cid = S.id[s];
                const bool vxy = T[lx] != INF_F && T[TX + ly] != INF_F;
                if (live0 && vxy && T[TX + TY + lz0] != INF_F) {
                    const double D = exact_D(S.c[s], px, py, pz0, v0, S.has[s], a.wv, a.wd);
                    if (better(D, cid, bD0, bI0)) { bD0 = D; bI0 = cid; }
                }
                if (live1 && vxy && T[TX + TY + lz0 + 2] != INF_F) {
                    const double D = exact_D(S.c[s], px, py, pz1, v1, S.has[s], a.wv, a.wd);
                    if (better(D, cid, bD1, bI1)) { bD1 = D; bI1 = cid; }
                }
            }
            __syncthreads();   // slots are rewritten by the next window
        }
        if (fast) break;
    }

    // ---- labels + stranded list
    const int lab0 = !live0 ? -1 : nfast ? (sl0 >= 0 ? S.id[sl0] : -1) : (bI0 != INT_MAX ? bI0 : -1);
    const int lab1 = !live1 ? -1 : nfast ? (sl1 >= 0 ? S.id[sl1] : -1) : (bI1 != INT_MAX ? bI1 : -1);
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
    if (a.accumulate && nfast) {
        // ---- per-warp records: counts x fixed coordinates, fp64 value butterfly
        int nrec = 0;
        unsigned p0 = __ballot_sync(0xffffffffu, sl0 >= 0), p1 = __ballot_sync(0xffffffffu, sl1 >= 0);
        while (p0 | p1) {
            const int L = p0 ? __shfl_sync(0xffffffffu, sl0, __ffs(p0) - 1)
                             : __shfl_sync(0xffffffffu, sl1, __ffs(p1) - 1);
            const unsigned m0 = __ballot_sync(0xffffffffu, sl0 == L);
            const unsigned m1 = __ballot_sync(0xffffffffu, sl1 == L);
            p0 &= ~m0;
            p1 &= ~m1;
            double sv = 0.0;
            if (sl0 == L) sv = v0;
            if (sl1 == L) sv = DADD(sv, v1);
            sv = warp_sum_d(sv);
            // lanes 0-3: x rows, 4-7: y rows, 8-11: z planes, 12: t; within each
            // group of 4 lanes reduce count * fixed coordinate exactly
            unsigned c = 0;
            const unsigned long long *fx = S.tf;
            const int q = lane & 3;
            if (lane < 4) {
                const unsigned M = 0x11111111u << q;
                c = __popc(m0 & M) + __popc(m1 & M);
                fx = S.xf[bx + q];
            } else if (lane < 8) {
                const unsigned M = 0x000F000Fu << (4 * q);
                c = __popc(m0 & M) + __popc(m1 & M);
                fx = S.yf[by + q];
            } else if (lane < 12) {
                const unsigned mm = q < 2 ? m0 : m1;
                c = __popc((q & 1) ? (mm >> 16) : (mm & 0xFFFFu));
                fx = S.zf[q];
            } else if (lane == 12) {
                c = __popc(m0) + __popc(m1);
            }
            const __int128 prod = c ? (((__int128)(long long)fx[1] << 64) | (__int128)fx[0]) * (__int128)c
                                    : (__int128)0;
            unsigned long long lo = (unsigned long long)prod;
            long long hi = (long long)(prod >> 64);
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const unsigned long long ol = __shfl_xor_sync(0xffffffffu, lo, o);
                const long long oh = __shfl_xor_sync(0xffffffffu, hi, o);
                add128(lo, hi, ol, oh);
            }
            if (nrec < RMAX) {
                Rec &R = S.rec[w][nrec];
                if ((lane & 3) == 0 && lane < 16) {
                    const int ax = lane >> 2;    // 0 x, 1 y, 2 z, 3 t
                    R.f[ax][0] = lo;
                    R.f[ax][1] = (unsigned long long)hi;
                }
                if (lane == 0) {
                    R.slot = L;
                    R.n = __popc(m0) + __popc(m1);
                    R.v = sv;
                }
            } else {
                // record overflow (pathological label mix): straight to the global sums
                unsigned long long *dst = a.acc + (size_t)S.id[L] * MFSEG_ACC_WORDS;
                if ((lane & 3) == 0 && lane < 16) atomic_add_fix(dst + 2 * (lane >> 2), lo, hi);
                if (lane == 0) {
                    atomic_add_double_fix(dst + 10, sv, &ovf_local);
                    atomicAdd(dst + 13, (unsigned long long)(__popc(m0) + __popc(m1)));
                }
            }
            ++nrec;
        }
        if (lane == 0) S.nrec[w] = min(nrec, RMAX);
        __syncthreads();
        // ---- tile combine per (slot, word) + one global atomic each
        for (int i = tid; i < nfast * 6; i += NT) {
            const int s = i / 6, wd = i - s * 6;
            unsigned long long lo = 0;
            long long hi = 0, n = 0;
            double vs = 0.0;
            bool any = false;
            for (int q = 0; q < NW; ++q) {
                const int nr = S.nrec[q];
                for (int r = 0; r < nr; ++r) {
                    const Rec &R = S.rec[q][r];
                    if (R.slot != s) continue;
                    any = true;
                    if (wd < 4) add128(lo, hi, R.f[wd][0], (long long)R.f[wd][1]);
                    else if (wd == 4) vs = DADD(vs, R.v);
                    else n += R.n;
                }
            }
            if (!any) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            if (wd < 4) atomic_add_fix(dst + 2 * wd, lo, hi);
            else if (wd == 4) atomic_add_double_fix(dst + 10, vs, &ovf_local);   // field-value sum
            else atomicAdd(dst + 13, (unsigned long long)n);                      // n_fields
        }
    } else if (a.accumulate) {
        // exact-mode tile (crowded bins): per-sample fixed point into the global sums
        const int labs[2] = {lab0, lab1};
        const double vs[2] = {v0, v1}, zs[2] = {pz0, pz1};
        for (int r = 0; r < 2; ++r) {
            if (labs[r] < 0) continue;
            unsigned long long *dst = a.acc + (size_t)labs[r] * MFSEG_ACC_WORDS;
            atomic_add_double_fix(dst + 0, px, &ovf_local);
            atomic_add_double_fix(dst + 2, py, &ovf_local);
            atomic_add_double_fix(dst + 4, zs[r], &ovf_local);
            atomic_add_double_fix(dst + 6, tm, &ovf_local);
            atomic_add_double_fix(dst + 10, vs[r], &ovf_local);
            atomicAdd(dst + 13, 1ull);
        }
    }
    if (ovf_local) *a.overflow = 1;
}

namespace {

// ============================================================== v4: multi-timestep tiles
constexpr int TT = 4;                       // timesteps per tile (one t-bin)
constexpr int TENT4 = TX + TY + TZ * TT;    // dx^2[16] | dy^2[8] | (dz^2 + (cf dt)^2)[4][4]
constexpr int NS = 2 * TT;                  // samples per lane
constexpr int RMAX4 = 8;

struct Rec4 {
    int slot, n;
    unsigned long long x[4][2], y[4][2], z[4][2], t[2];
    double v;
};

struct Smem4 {
    double x[TX], y[TY], z[TZ], t[TT];
    unsigned long long xf[TX][2], yf[TY][2], zf[TZ][2], tf[TT][2];
    int id[SCAP];
    double c[SCAP][5];              // cx, cy, cz, ct (raw), cv (0 when absent)
    unsigned box[SCAP];             // x 4+4 | y 3+3 | z 2+2 | t 2+2 bits
    unsigned char has[SCAP];
    float cvf[SCAP], wvf[SCAP];
    float tab[SCAP][TENT4];
    Rec4 rec[NW][RMAX4];
    int nrec[NW];
    double red[2 * NW];
    int wc[NW];
};

__device__ __forceinline__ void put128(unsigned long long *dst, __int128 v) {
    dst[0] = (unsigned long long)v;
    dst[1] = (unsigned long long)(v >> 64);
}
__device__ __forceinline__ __int128 get128(const unsigned long long *p) {
    return (__int128)(((unsigned __int128)p[1] << 64) | (unsigned __int128)p[0]);
}

}  // namespace

__global__ void __launch_bounds__(NT, 3) k_field_assign4(FieldArgs a) {
    __shared__ Smem4 S;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    long long tile = blockIdx.x;
    const int txi = (int)(tile % a.ntx);
    tile /= a.ntx;
    const int tyi = (int)(tile % a.nty);
    tile /= a.nty;
    const int tzi = (int)(tile % a.ntz);
    const int tti = (int)(tile / a.ntz);
    const AxisTile X = a.xt[txi], Y = a.yt[tyi], Z = a.zt[tzi], Tm = a.tt[tti];
    int ovf_local = 0;
    if (tid < TENT) {   // 28 spatial coordinates
        double cv;
        unsigned long long *dst;
        if (tid < TX) {
            cv = cell_coord(a.ox, a.sx, X.start + tid);
            S.x[tid] = cv;
            dst = S.xf[tid];
        } else if (tid < TX + TY) {
            cv = cell_coord(a.oy, a.sy, Y.start + tid - TX);
            S.y[tid - TX] = cv;
            dst = S.yf[tid - TX];
        } else {
            cv = cell_coord(a.oz, a.sz, Z.start + tid - TX - TY);
            S.z[tid - TX - TY] = cv;
            dst = S.zf[tid - TX - TY];
        }
        long long hi;
        d2fix(cv, dst[0], hi, &ovf_local);
        dst[1] = (unsigned long long)hi;
    } else if (tid < TENT + TT) {
        const int q = tid - TENT;
        const double tv = a.times[Tm.start + (q < Tm.len ? q : 0)];
        S.t[q] = tv;
        long long hi;
        d2fix(tv, S.tf[q][0], hi, &ovf_local);
        S.tf[q][1] = (unsigned long long)hi;
    }
    const int sbin = ((Tm.bin * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;

    // ---- this lane's samples: k = q*TT + tt at (lx, ly, lz0 + 2q, timestep tt)
    const int bx = (w & 3) * 4, by = (w >> 2) * 4;
    const int lx = bx + (lane & 3), ly = by + ((lane >> 2) & 3), lz0 = lane >> 4;
    const bool rowok = lx < X.len && ly < Y.len;
    const long long plane = (long long)a.ny * a.nx, vol = plane * a.nz;
    const long long fbase = (((long long)Tm.start * a.nz + Z.start + lz0) * a.ny + (Y.start + ly)) *
                                (long long)a.nx + (X.start + lx);
    unsigned livem = 0;   // bit k: sample k exists
    double v[NS];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int t = 0; t < TT; ++t) {
            const int k = q * TT + t;
            const bool lv = rowok && lz0 + 2 * q < Z.len && t < Tm.len;
            if (lv) livem |= 1u << k;
            v[k] = lv ? __ldg(a.values + fbase + 2 * q * plane + t * vol) : 0.0;
        }
    const bool useval = a.wv > 0.0;
    double wvlo = 0.0, wvhi = 0.0;
    if (useval) {
        double lo = INF_D, hi = -INF_D;
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (livem >> k & 1) {
                lo = fmin(lo, v[k]);
                hi = fmax(hi, v[k]);
            }
        wvlo = warp_min_d(lo);
        wvhi = warp_max_d(hi);
        if (lane == 0) {
            S.red[w] = wvlo;
            S.red[NW + w] = wvhi;
        }
    }
    __syncthreads();
    double tvlo = 0.0, tvhi = 0.0;
    if (useval) {
        tvlo = S.red[0];
        tvhi = S.red[NW];
#pragma unroll
        for (int q = 1; q < NW; ++q) {
            tvlo = fmin(tvlo, S.red[q]);
            tvhi = fmax(tvhi, S.red[NW + q]);
        }
    }

    int sl[NS];                        // survivor slot per sample (-1: stranded)
#pragma unroll
    for (int k = 0; k < NS; ++k) sl[k] = -1;
    int nfast = 0;
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    // crowded candidate lists are deferred whole to k_deferred (exact, per sample)
    bool deferred = (L1 - L0) > NT;
    const double px = S.x[lx], py = S.y[ly];

    if (!deferred && L1 > L0) {
        // ---- phase A: exact fp64 bounds over the 4D tile, one candidate per thread
        const int ci = L0 + tid;
        bool have = ci < L1;
        int id = 0;
        double cx = 0, cy = 0, cz = 0, ctr = 0, cv = 0, Dlo = INF_D, Dhi = INF_D;
        bool chas = false, full = false;
        unsigned box = 0;
        if (have) {
            id = a.g.cand_ids[ci];
            const int4 b0 = a.g.vbox[2 * id], b1 = a.g.vbox[2 * id + 1];
            const int xa = max(b0.x - X.start, 0), xb = min(b0.y - X.start, X.len - 1);
            const int ya = max(b0.z - Y.start, 0), yb = min(b0.w - Y.start, Y.len - 1);
            const int za = max(b1.x - Z.start, 0), zb = min(b1.y - Z.start, Z.len - 1);
            const int ta = max(b1.z - Tm.start, 0), tb = min(b1.w - Tm.start, Tm.len - 1);
            have = xa <= xb && ya <= yb && za <= zb && ta <= tb;
            if (have) {
                cx = a.c.x[id];
                cy = a.c.y[id];
                cz = a.c.z[id];
                ctr = a.c.t[id];
                chas = a.chas[id] != 0;
                cv = chas ? a.cval[id] : 0.0;
                full = xa == 0 && xb == X.len - 1 && ya == 0 && yb == Y.len - 1 && za == 0 &&
                       zb == Z.len - 1 && ta == 0 && tb == Tm.len - 1;
                double dxl, dxh, dyl, dyh, dzl, dzh, dtl, dth;
                axis_range(cx, S.x[xa], S.x[xb], dxl, dxh);
                axis_range(cy, S.y[ya], S.y[yb], dyl, dyh);
                axis_range(cz, S.z[za], S.z[zb], dzl, dzh);
                axis_range(ctr, S.t[ta], S.t[tb], dtl, dth);
                const double ctl = DMUL(a.cf, dtl), cth = DMUL(a.cf, dth);
                double vtl = 0.0, vth = 0.0;
                if (useval && chas) {
                    const double p = DSUB(tvlo, cv), q = DSUB(tvhi, cv);
                    const double fp = fabs(p), fq = fabs(q);
                    vtl = DMUL(a.wv, (p <= 0.0 && q >= 0.0) ? 0.0 : fmin(fp, fq));
                    vth = DMUL(a.wv, fmax(fp, fq));
                }
                Dlo = bound_D(dxl, dyl, dzl, DMUL(ctl, ctl), vtl, a.wd);
                Dhi = bound_D(dxh, dyh, dzh, DMUL(cth, cth), vth, a.wd);
                box = (unsigned)xa | ((unsigned)xb << 4) | ((unsigned)ya << 8) | ((unsigned)yb << 11) |
                      ((unsigned)za << 14) | ((unsigned)zb << 16) | ((unsigned)ta << 18) |
                      ((unsigned)tb << 20);
            }
        }
        // ---- phase B: tile UB, survivor count and positions
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
        deferred = nsurv > SCAP;
        const int pos = off + __popc(bal & ((1u << lane) - 1u));
        if (!deferred && nsurv > 0) {
            const int cnt = nsurv;
            if (surv) {
                const int p = pos;
                S.id[p] = id;
                S.c[p][0] = cx;
                S.c[p][1] = cy;
                S.c[p][2] = cz;
                S.c[p][3] = ctr;
                S.c[p][4] = cv;
                S.box[p] = box;
                S.has[p] = chas;
                S.cvf[p] = (float)cv;
                S.wvf[p] = (useval && chas) ? (float)a.wv : 0.0f;
            }
            __syncthreads();
            for (int e = tid; e < cnt * TENT4; e += NT) {
                const int p = e / TENT4, j = e - p * TENT4;
                const unsigned b = S.box[p];
                float val = INF_F;
                if (j < TX) {
                    if (j >= (int)(b & 15u) && j <= (int)((b >> 4) & 15u)) {
                        const double d = DSUB(S.c[p][0], S.x[j]);
                        val = to_f(DMUL(d, d));
                    }
                } else if (j < TX + TY) {
                    const int i = j - TX;
                    if (i >= (int)((b >> 8) & 7u) && i <= (int)((b >> 11) & 7u)) {
                        const double d = DSUB(S.c[p][1], S.y[i]);
                        val = to_f(DMUL(d, d));
                    }
                } else {
                    const int i = j - TX - TY, zi = i / TT, ti = i - zi * TT;
                    if (zi >= (int)((b >> 14) & 3u) && zi <= (int)((b >> 16) & 3u) &&
                        ti >= (int)((b >> 18) & 3u) && ti <= (int)((b >> 20) & 3u)) {
                        const double d = DSUB(S.c[p][2], S.z[zi]);
                        const double ct = DMUL(a.cf, DSUB(S.c[p][3], S.t[ti]));
                        val = to_f(DADD(DMUL(d, d), DMUL(ct, ct)));
                    }
                }
                S.tab[p][j] = val;
            }
            __syncthreads();

            {
                nfast = cnt;
                const float fwd = (float)a.wd;
                const float vwl = (float)wvlo, vwh = (float)wvhi;
                const float slack = 3e-13f * (float)(a.wd + a.wv);
                // ---- warp culling over the 4x4x4 x TT brick
                float cvmax = 0.0f, ubw = INF_F;
                float dl_r[2] = {INF_F, INF_F};
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int s = lane + 32 * r;
                    if (s < cnt) {
                        const float *T = S.tab[s];
                        float xmn = INF_F, xmx = 0.f, ymn = INF_F, ymx = 0.f, zmn = INF_F, zmx = 0.f;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (bx + q < X.len) {
                                const float e = T[bx + q];
                                xmn = fminf(xmn, e);
                                xmx = fmaxf(xmx, e);
                            }
                            if (by + q < Y.len) {
                                const float e = T[TX + by + q];
                                ymn = fminf(ymn, e);
                                ymx = fmaxf(ymx, e);
                            }
                        }
#pragma unroll
                        for (int q = 0; q < TZ * TT; ++q) {
                            if ((q / TT) < Z.len && (q % TT) < Tm.len) {
                                const float e = T[TX + TY + q];
                                zmn = fminf(zmn, e);
                                zmx = fmaxf(zmx, e);
                            }
                        }
                        const float wvs = S.wvf[s];
                        float vtl = 0.f, vth = 0.f;
                        if (wvs > 0.f) {
                            const float cvs = S.cvf[s];
                            const float pl = vwl - cvs, ph = vwh - cvs;
                            vtl = wvs * ((pl <= 0.f && ph >= 0.f) ? 0.f : fminf(fabsf(pl), fabsf(ph)));
                            vth = wvs * fmaxf(fabsf(pl), fabsf(ph));
                            cvmax = fmaxf(cvmax, fabsf(cvs));
                        }
                        dl_r[r] = fmaf(fwd, sqrt_approx((xmn + ymn) + zmn), vtl);
                        ubw = fminf(ubw, fmaf(fwd, sqrt_approx((xmx + ymx) + zmx), vth));
                    }
                }
                ubw = warp_min_f(ubw);
                cvmax = warp_max_f(cvmax);
                const float Wb = (useval ? (float)a.wv * (fmaxf(fabsf(vwl), fabsf(vwh)) + cvmax) : 0.f) +
                                 slack;
                const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) * (1.f + 0x1.0p-15f);   // >= /(1-KCULL)
                const unsigned keep0 = __ballot_sync(0xffffffffu, lane < cnt && (dl_r[0] <= thr || (a.debug & 1)));
                const unsigned keep1 =
                    __ballot_sync(0xffffffffu, lane + 32 < cnt && (dl_r[1] <= thr || (a.debug & 1)));
                // ---- per-sample fp32 screen
                float fv[NS], b1[NS], b2[NS];
                int i1[NS];
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    fv[k] = (float)v[k];
                    b1[k] = INF_F;
                    b2[k] = INF_F;
                    i1[k] = -1;
                }
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    unsigned it = half ? keep1 : keep0;
                    while (it) {
                        const int s = __ffs(it) - 1 + 32 * half;
                        it &= it - 1;
                        const float *T = S.tab[s];
                        const float axy = T[lx] + T[TX + ly];
                        const float cvs = S.cvf[s], wvs = S.wvf[s];
                        const float *Tz = T + TX + TY + lz0 * TT;
#pragma unroll
                        for (int k = 0; k < NS; ++k) {
                            const float az = Tz[(k / TT) * 2 * TT + (k % TT)];
                            const float d = fmaf(fwd, sqrt_approx(axy + az), wvs * fabsf(fv[k] - cvs));
                            if (d < b1[k]) {
                                b2[k] = b1[k];
                                b1[k] = d;
                                i1[k] = s;
                            } else {
                                b2[k] = fminf(b2[k], d);
                            }
                        }
                    }
                }
                // ---- certify or resolve exactly
                unsigned need = 0;
                const float wvf = useval ? (float)a.wv : 0.f;
#pragma unroll
                for (int k = 0; k < NS; ++k) {
                    const float W = fmaf(wvf, fabsf(fv[k]) + cvmax, slack);
                    const bool ok = !(a.debug & 2) && b1[k] < INF_F &&
                                    b2[k] * (1.f - KSCR) > b1[k] * (1.f + KSCR) + 2.f * KSCR * W;
                    sl[k] = ok ? i1[k] : -1;
                    if (!ok && (livem >> k & 1)) need |= 1u << k;
                }
                if (__any_sync(0xffffffffu, need != 0)) {
                    if (need) {
#pragma unroll
                        for (int k = 0; k < NS; ++k) {
                            if (!(need >> k & 1)) continue;
                            const int zi = lz0 + 2 * (k / TT), ti = k % TT;
                            const float W = fmaf(wvf, fabsf(fv[k]) + cvmax, slack);
                            // (b1 (1+k) + 2 k W) / (1-k) <= that * (1 + 2^-17)
                            const float thrk = b1[k] < INF_F
                                                   ? (b1[k] * (1.f + KSCR) + 2.f * KSCR * W) * (1.f + 0x1.0p-17f)
                                                   : INF_F;
                            double eD = INF_D;
                            int eI = INT_MAX, eS = -1;
                            for (int s = 0; s < cnt; ++s) {
                                const float *T = S.tab[s];
                                const float az = T[TX + TY + zi * TT + ti];
                                if (T[lx] == INF_F || T[TX + ly] == INF_F || az == INF_F) continue;
                                const float d = fmaf(fwd, sqrt_approx(T[lx] + T[TX + ly] + az),
                                                     S.wvf[s] * fabsf(fv[k] - S.cvf[s]));
                                if (d > thrk) continue;
                                const double dx = DSUB(S.c[s][0], px), dy = DSUB(S.c[s][1], py),
                                             dz = DSUB(S.c[s][2], S.z[zi]);
                                const double ct = DMUL(a.cf, DSUB(S.c[s][3], S.t[ti]));
                                const double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
                                const double D = metric_tail(qq, DMUL(ct, ct), v[k], S.c[s][4], S.has[s],
                                                             a.wv, a.wd);
                                if (better(D, S.id[s], eD, eI)) {
                                    eD = D;
                                    eI = S.id[s];
                                    eS = s;
                                }
                            }
                            sl[k] = eS;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < NS; ++k)
                    if (!(livem >> k & 1)) sl[k] = -1;
            }
        }
    }

    // ---- labels + stranded list
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if (!(livem >> k & 1)) continue;
        const long long f = fbase + 2 * (k / TT) * plane + (k % TT) * vol;
        if (deferred) {
            a.labels[f] = -2;
            const unsigned long long p = atomicAdd(a.n_deferred, 1ull);
            if ((long long)p < a.deferred_cap) a.deferred[p] = f;
        } else {
            const int lab = sl[k] >= 0 ? S.id[sl[k]] : -1;
            a.labels[f] = lab;
            if (lab < 0) {
                const unsigned long long p = atomicAdd(a.n_stranded, 1ull);
                if ((long long)p < a.stranded_cap) a.stranded[p] = f;
            }
        }
    }
    if (a.accumulate && nfast && !deferred) {
        // ---- per-warp records from __reduce_add_sync count marginals
        const unsigned MX = 0x11111111u << (lane & 3);
        const unsigned MY = 0x000F000Fu << (4 * ((lane >> 2) & 3));
        const unsigned MZ = lz0 ? 0xFFFF0000u : 0x0000FFFFu;
        unsigned todo = 0;
#pragma unroll
        for (int k = 0; k < NS; ++k)
            if (sl[k] >= 0) todo |= 1u << k;
        int nrec = 0;
        while (true) {
            int mine = -1;
#pragma unroll
            for (int k = NS - 1; k >= 0; --k)
                if (todo >> k & 1) mine = sl[k];
            const unsigned act = __ballot_sync(0xffffffffu, mine >= 0);
            if (!act) break;
            const int L = __shfl_sync(0xffffffffu, mine, __ffs(act) - 1);
            unsigned c = 0, cz0 = 0, cz1 = 0, ct[TT];
            double vs = 0.0;
#pragma unroll
            for (int t = 0; t < TT; ++t) ct[t] = 0;
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                if ((todo >> k & 1) && sl[k] == L) {
                    todo &= ~(1u << k);
                    ++c;
                    if (k < TT) ++cz0; else ++cz1;
                    ct[k % TT] += 1;
                    vs = DADD(vs, v[k]);
                }
            }
            const unsigned sx = __reduce_add_sync(MX, c);
            const unsigned sy = __reduce_add_sync(MY, c);
            const unsigned sz0 = __reduce_add_sync(MZ, cz0), sz1 = __reduce_add_sync(MZ, cz1);
            unsigned st[TT];
#pragma unroll
            for (int t = 0; t < TT; ++t) st[t] = __reduce_add_sync(0xffffffffu, ct[t]);
            const unsigned n = __reduce_add_sync(0xffffffffu, c);
            vs = warp_sum_d(vs);
            if (nrec < RMAX4) {
                Rec4 &R = S.rec[w][nrec];
                if (lane < 4) put128(R.x[lane], get128(S.xf[bx + lane]) * (__int128)sx);
                if (lane >= 16 && (lane & 3) == 0) {
                    const int j = (lane >> 2) & 3;
                    put128(R.y[j], get128(S.yf[by + j]) * (__int128)sy);
                }
                if (lane == 4 || lane == 20) {   // lz0 = 0 / 1: planes lz0 and lz0 + 2
                    put128(R.z[lz0], get128(S.zf[lz0]) * (__int128)sz0);
                    put128(R.z[lz0 + 2], get128(S.zf[lz0 + 2]) * (__int128)sz1);
                }
                if (lane == 8) {
                    __int128 tsum = 0;
#pragma unroll
                    for (int t = 0; t < TT; ++t) tsum += get128(S.tf[t]) * (__int128)st[t];
                    put128(R.t, tsum);
                }
                if (lane == 0) {
                    R.slot = L;
                    R.n = (int)n;
                    R.v = vs;
                }
            } else {
                unsigned long long *dst = a.acc + (size_t)S.id[L] * MFSEG_ACC_WORDS;
                if (lane < 4) {
                    const __int128 x = get128(S.xf[bx + lane]) * (__int128)sx;
                    atomic_add_fix(dst + 0, (unsigned long long)x, (long long)(x >> 64));
                }
                if (lane >= 16 && (lane & 3) == 0) {
                    const int j = (lane >> 2) & 3;
                    const __int128 y = get128(S.yf[by + j]) * (__int128)sy;
                    atomic_add_fix(dst + 2, (unsigned long long)y, (long long)(y >> 64));
                }
                if (lane == 4 || lane == 20) {
                    const __int128 z = get128(S.zf[lz0]) * (__int128)sz0 + get128(S.zf[lz0 + 2]) * (__int128)sz1;
                    atomic_add_fix(dst + 4, (unsigned long long)z, (long long)(z >> 64));
                }
                if (lane == 8) {
                    __int128 tsum = 0;
#pragma unroll
                    for (int t = 0; t < TT; ++t) tsum += get128(S.tf[t]) * (__int128)st[t];
                    atomic_add_fix(dst + 6, (unsigned long long)tsum, (long long)(tsum >> 64));
                }
                if (lane == 0) {
                    atomic_add_double_fix(dst + 10, vs, &ovf_local);
                    atomicAdd(dst + 13, (unsigned long long)n);
                }
            }
            ++nrec;
        }
        if (lane == 0) S.nrec[w] = min(nrec, RMAX4);
        __syncthreads();
        for (int i = tid; i < nfast * 6; i += NT) {
            const int s = i / 6, wd = i - s * 6;
            __int128 acc = 0;
            long long n = 0;
            double vs = 0.0;
            bool any = false;
            for (int q = 0; q < NW; ++q) {
                const int nr = S.nrec[q];
                for (int r = 0; r < nr; ++r) {
                    const Rec4 &R = S.rec[q][r];
                    if (R.slot != s) continue;
                    any = true;
                    if (wd == 0) {
                        for (int j = 0; j < 4; ++j) acc += get128(R.x[j]);
                    } else if (wd == 1) {
                        for (int j = 0; j < 4; ++j) acc += get128(R.y[j]);
                    } else if (wd == 2) {
                        for (int j = 0; j < 4; ++j) acc += get128(R.z[j]);
                    } else if (wd == 3) {
                        acc += get128(R.t);
                    } else if (wd == 4) {
                        vs = DADD(vs, R.v);
                    } else {
                        n += R.n;
                    }
                }
            }
            if (!any) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            if (wd < 4) atomic_add_fix(dst + 2 * wd, (unsigned long long)acc, (long long)(acc >> 64));
            else if (wd == 4) atomic_add_double_fix(dst + 10, vs, &ovf_local);
            else atomicAdd(dst + 13, (unsigned long long)n);
        }
    }
    if (ovf_local) *a.overflow = 1;
}

int launch_field_assign_v2(const FieldArgs &a, long long ntiles, cudaStream_t st) {
    if (ntiles <= 0) return 0;
    if (getenv("MFSEG_FIELD_V3")) {
        if (ntiles > 0x7fffffffll) {
            set_error("field tile grid too large");
            return 3;
        }
        ::mfseg::count_launch();
        k_field_assign3<<<(unsigned)ntiles, NT, 0, st>>>(a);
        MFSEG_LAUNCH("k_field_assign3");
        return 0;
    }
    const long long n4 = (long long)a.ntx * a.nty * a.ntz * a.ntt;
    if (n4 > 0x7fffffffll) {
        set_error("field tile grid too large");
        return 3;
    }
    ::mfseg::count_launch();
    k_field_assign4<<<(unsigned)n4, NT, 0, st>>>(a);
    MFSEG_LAUNCH("k_field_assign4");
    return 0;
}

}  // namespace mfseg
