// k_point_assign — windowed exact assignment of point samples (v3).
//
// Same contract as k_field_assign3 (exact reference labels, lowest id on ties)
// for unstructured samples.  Points are pre-sorted once per run by (sample
// bin, 4^4 sub-cell inside the bin) and cut into tiles of <= 256 points of one
// bin, so a tile shares one candidate list and a warp's 64 points are
// spatially compact.  Multi-GPU time slabs are whole t-bins, so tiles never
// straddle ranks (bit-identical sums for any number of GPUs).
//
//  1. tile level: exact fp64 bounds of D over the tile's bounding box per
//     candidate (none / partial / full box-test classes), cull against the best
//     full upper bound.
//  2. survivors get tile-relative fp32 coordinates rc = fl32(fl64(c - o)) (o =
//     tile minimum corner, t scaled by c_f); points get rp likewise.  Then
//     |(rc - rp)_d - (c - s)_d| <= 2^-22 (E_d + C_d) =: delta_d / 2 (E = tile
//     extent), so the fp32 distance is within Delta = ||delta|| of the exact
//     one: |d32 - D| <= 2^-19 (D + W) + w_d Delta.
//  3. warp level: fp32 bounds over the warp's 64-point box, cull with margin.
//  4. per point: fp32 screen (box test in fp32 with a +-delta guard band and an
//     exact fp64 test inside the band), best/second best, certification with
//     margin 2^-18 relative + 2 w_d Delta absolute, exact fp64 otherwise.
//  5. accumulation: per-warp records (fixed-order fp64 butterflies of x, y, z,
//     t, v), per-tile combine per (slot, word), 128-bit integer atomics.
#include <climits>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();

constexpr int NT = 128, NW = 4;
static_assert(2 * NT == POINT_TILE, "k_point_assign3 covers POINT_TILE points per tile");
constexpr int SCAP = 128;
constexpr int RMAX = 16;
constexpr float KSCR = 0x1.0p-18f;
constexpr float KCULL = 0x1.0p-16f;

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
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
__device__ __forceinline__ double bound_D(double dx, double dy, double dz, double tsq, double vt,
                                          double wd) {
    double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    return DADD(vt, DMUL(wd, DSQRT(DADD(q, tsq))));
}

struct PRec {
    int slot, n;
    double s[5];    // x, y, z, t, v
};

struct PSmem {
    int id[SCAP];
    double c[SCAP][5];          // cx, cy, cz, ct (raw), cv
    float rc[SCAP][4];          // tile-relative fp32 coordinates (t scaled by c_f)
    float cvf[SCAP], wvf[SCAP];
    unsigned char has[SCAP], full[SCAP];
    PRec rec[NW][RMAX];
    int nrec[NW];
    double red[8 * NW];
    int wc[NW];
    double o[4];                // tile origin
    float delta[4], Cf[4];      // guard bands, fp32 box half-widths (t scaled by c_f)
    float Aabs;                 // absolute error allowance of the fp32 distance
};

// exact reference box test + metric of one pair (engine.py:137-149, 179-181)
__device__ __forceinline__ bool exact_pair(const double *c, double x, double y, double z, double t,
                                           double v, bool has, double cf, double wv, double wd,
                                           const double *C, double &D) {
    const double dx = DSUB(c[0], x), dy = DSUB(c[1], y), dz = DSUB(c[2], z), dt = DSUB(c[3], t);
    if (!(fabs(dx) <= C[0] && fabs(dy) <= C[1] && fabs(dz) <= C[2] && fabs(dt) <= C[3])) return false;
    const double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    const double ct = DMUL(cf, dt);
    D = metric_tail(q, DMUL(ct, ct), v, c[4], has, wv, wd);
    return true;
}

}  // namespace

__global__ void __launch_bounds__(NT, 4) k_point_assign3(PointArgs a) {
    __shared__ PSmem S;
    if ((int)blockIdx.x >= *a.n_tiles) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int4 T = a.tiles[blockIdx.x];
    const int sbin = T.x;
    const double Cd[4] = {a.Cx, a.Cy, a.Cz, a.Ct};
    // ---- this lane's two points (warp w: tile positions 64w + lane, 64w + 32 + lane)
    const long long p0 = (long long)T.y + 64 * w + lane, p1 = p0 + 32;
    const bool live0 = 64 * w + lane < T.z, live1 = 64 * w + 32 + lane < T.z;
    double P0[5] = {0, 0, 0, 0, 0}, P1[5] = {0, 0, 0, 0, 0};   // x, y, z, t, v
    if (live0) {
        P0[0] = a.x[p0]; P0[1] = a.y[p0]; P0[2] = a.z[p0]; P0[3] = a.t[p0]; P0[4] = a.v[p0];
    }
    if (live1) {
        P1[0] = a.x[p1]; P1[1] = a.y[p1]; P1[2] = a.z[p1]; P1[3] = a.t[p1]; P1[4] = a.v[p1];
    }
    // ---- tile box (exact min/max) and value range, via warp + block reduction
    double lo[5], hi[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        double l = INF_D, h = -INF_D;
        if (live0) { l = P0[d]; h = P0[d]; }
        if (live1) { l = fmin(l, P1[d]); h = fmax(h, P1[d]); }
        l = wmin_d(l);
        h = wmax_d(h);
        lo[d] = l;
        hi[d] = h;
        if (lane == 0) {
            S.red[d * NW + w] = l;
        }
    }
    // (5 mins in red[0..5*NW), maxes need a second buffer)
    __shared__ double s_hi[5 * NW];
    if (lane == 0)
        for (int d = 0; d < 5; ++d) s_hi[d * NW + w] = hi[d];
    __syncthreads();
    double tlo[5], thi[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        tlo[d] = S.red[d * NW];
        thi[d] = s_hi[d * NW];
#pragma unroll
        for (int q = 1; q < NW; ++q) {
            tlo[d] = fmin(tlo[d], S.red[d * NW + q]);
            thi[d] = fmax(thi[d], s_hi[d * NW + q]);
        }
    }
    const bool useval = a.wv > 0.0;
    if (tid < 4) {   // per-tile constants, shared
        const int d = tid;
        const double sc = d == 3 ? a.cf : 1.0;
        S.o[d] = tlo[d];
        S.delta[d] = (float)(DMUL(DMUL(DADD(DSUB(thi[d], tlo[d]), Cd[d]), sc), 0x1.0p-21));   // 2x the 2^-22 bound
        S.Cf[d] = (float)DMUL(Cd[d], sc);
    }
    __syncthreads();
    if (tid == 0) {
        const float D0 = S.delta[0], D1 = S.delta[1], D2 = S.delta[2], D3 = S.delta[3];
        S.Aabs = 1.1f * (float)a.wd * sqrtf(D0 * D0 + D1 * D1 + D2 * D2 + D3 * D3) +
                 3e-13f * (float)(a.wd + a.wv);
    }
    float rp0[4], rp1[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        const double sc = d == 3 ? a.cf : 1.0;
        rp0[d] = (float)DMUL(DSUB(P0[d], S.o[d]), sc);
        rp1[d] = (float)DMUL(DSUB(P1[d], S.o[d]), sc);
    }
    const float fwd = (float)a.wd;

    int sl0 = -1, sl1 = -1;
    int nfast = 0;
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    bool deferred = (L1 - L0) > NT;     // crowded candidate lists -> k_deferred
    __syncthreads();                    // S.Aabs
    const float Aabs = S.Aabs;

    if (!deferred && L1 > L0) {
        // ---- phase A: exact fp64 classification + bounds over the tile box
        const int ci = L0 + tid;
        bool have = ci < L1;
        int id = 0;
        double c4[4] = {0, 0, 0, 0}, cv = 0, Dlo = INF_D, Dhi = INF_D;
        bool chas = false, full = false;
        if (have) {
            id = a.g.cand_ids[ci];
            c4[0] = a.c.x[id];
            c4[1] = a.c.y[id];
            c4[2] = a.c.z[id];
            c4[3] = a.c.t[id];
            double dl[4], dh[4];
            full = true;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const double da = DSUB(c4[d], tlo[d]), db = DSUB(c4[d], thi[d]);   // da >= db
                if (da < -Cd[d] || db > Cd[d]) have = false;                        // nobody passes
                if (!(da <= Cd[d] && db >= -Cd[d])) full = false;                   // not everybody
                const double ea = fmin(da, Cd[d]), eb = fmax(db, -Cd[d]);
                const double fa = fabs(ea), fb = fabs(eb);
                dh[d] = fmax(fa, fb);
                dl[d] = (eb <= 0.0 && ea >= 0.0) ? 0.0 : fmin(fa, fb);
            }
            if (have) {
                chas = a.chas[id] != 0;
                cv = chas ? a.cval[id] : 0.0;
                const double tl = DMUL(a.cf, dl[3]), th = DMUL(a.cf, dh[3]);
                double vtl = 0.0, vth = 0.0;
                if (useval && chas) {
                    const double p = DSUB(tlo[4], cv), q = DSUB(thi[4], cv);
                    const double fp = fabs(p), fq = fabs(q);
                    vtl = DMUL(a.wv, (p <= 0.0 && q >= 0.0) ? 0.0 : fmin(fp, fq));
                    vth = DMUL(a.wv, fmax(fp, fq));
                }
                Dlo = bound_D(dl[0], dl[1], dl[2], DMUL(tl, tl), vtl, a.wd);
                Dhi = bound_D(dh[0], dh[1], dh[2], DMUL(th, th), vth, a.wd);
            } else {
                full = false;
            }
        }
        double ub = wmin_d(full ? Dhi : INF_D);
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
                S.c[p][0] = c4[0];
                S.c[p][1] = c4[1];
                S.c[p][2] = c4[2];
                S.c[p][3] = c4[3];
                S.c[p][4] = cv;
#pragma unroll
                for (int d = 0; d < 4; ++d)
                    S.rc[p][d] = (float)DMUL(DSUB(c4[d], S.o[d]), d == 3 ? a.cf : 1.0);
                S.cvf[p] = (float)cv;
                S.wvf[p] = (useval && chas) ? (float)a.wv : 0.f;
                S.has[p] = chas;
                S.full[p] = full;
            }
            __syncthreads();
            {
                nfast = cnt;
                const float delta[4] = {S.delta[0], S.delta[1], S.delta[2], S.delta[3]};
                const float Cf[4] = {S.Cf[0], S.Cf[1], S.Cf[2], S.Cf[3]};
                // ---- warp culling over the warp's point box (fp32, relative)
                float wl[4], wh[4];
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    float l = INF_F, h = -INF_F;
                    if (live0) { l = rp0[d]; h = rp0[d]; }
                    if (live1) { l = fminf(l, rp1[d]); h = fmaxf(h, rp1[d]); }
                    wl[d] = wmin_f(l);
                    wh[d] = wmax_f(h);
                }
                float vl = 0.f, vh = 0.f;
                if (useval) {
                    vl = (float)lo[4];
                    vh = (float)hi[4];
                }
                float ubw = INF_F, cvmax = 0.f;
                float dl_r[SCAP / 32];
#pragma unroll
                for (int r = 0; r < SCAP / 32; ++r) dl_r[r] = INF_F;
#pragma unroll
                for (int r = 0; r < SCAP / 32; ++r) {
                    const int s = lane + 32 * r;
                    if (s < cnt) {
                        float ql = 0.f, qh = 0.f;
                        bool wfull = true, none = false;
#pragma unroll
                        for (int d = 0; d < 4; ++d) {
                            const float a1 = S.rc[s][d] - wl[d], b1 = S.rc[s][d] - wh[d];   // a1 >= b1
                            if (a1 < -(Cf[d] + delta[d]) || b1 > Cf[d] + delta[d]) none = true;
                            if (!(a1 <= Cf[d] - delta[d] && b1 >= -(Cf[d] - delta[d]))) wfull = false;
                            const float e1 = fminf(a1, Cf[d] + delta[d]), e2 = fmaxf(b1, -(Cf[d] + delta[d]));
                            const float mx = fmaxf(fabsf(e1), fabsf(e2));
                            const float mn = (e2 <= 0.f && e1 >= 0.f) ? 0.f : fminf(fabsf(e1), fabsf(e2));
                            ql = fmaf(mn, mn, ql);
                            qh = fmaf(mx, mx, qh);
                        }
                        const float wvs = S.wvf[s];
                        float vtl = 0.f, vth = 0.f;
                        if (wvs > 0.f) {
                            const float cvs = S.cvf[s];
                            const float pl = vl - cvs, ph = vh - cvs;
                            vtl = wvs * ((pl <= 0.f && ph >= 0.f) ? 0.f : fminf(fabsf(pl), fabsf(ph)));
                            vth = wvs * fmaxf(fabsf(pl), fabsf(ph));
                            cvmax = fmaxf(cvmax, fabsf(cvs));
                        }
                        if (!none) dl_r[r] = fmaf(fwd, sqrt_approx(ql), vtl);
                        if (wfull && !none) ubw = fminf(ubw, fmaf(fwd, sqrt_approx(qh), vth));
                    }
                }
                ubw = wmin_f(ubw);
                cvmax = wmax_f(cvmax);
                const float Wb = useval ? (float)a.wv * (fmaxf(fabsf(vl), fabsf(vh)) + cvmax) : 0.f;
                const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb + 2.f * Aabs) * (1.f + 0x1.0p-15f);
                unsigned keep[SCAP / 32];
#pragma unroll
                for (int r = 0; r < SCAP / 32; ++r)
                    keep[r] = __ballot_sync(0xffffffffu, lane + 32 * r < cnt && (dl_r[r] <= thr || (a.debug & 1)));
                // ---- per-point fp32 screen
                const float fv0 = (float)P0[4], fv1 = (float)P1[4];
                float b1a = INF_F, b2a = INF_F, b1b = INF_F, b2b = INF_F;
                int i1a = -1, i1b = -1;
                bool unsure_a = false, unsure_b = false;   // box test inside the guard band
#pragma unroll
                for (int half = 0; half < SCAP / 32; ++half) {
                    unsigned it = keep[half];
                    while (it) {
                        const int s = __ffs(it) - 1 + 32 * half;
                        it &= it - 1;
                        const float r0 = S.rc[s][0], r1 = S.rc[s][1], r2 = S.rc[s][2], r3 = S.rc[s][3];
                        const float cvs = S.cvf[s], wvs = S.wvf[s];
                        const bool fl = S.full[s];
                        {
                            const float dx = r0 - rp0[0], dy = r1 - rp0[1], dz = r2 - rp0[2], dt = r3 - rp0[3];
                            bool ok = true;
                            if (!fl) {
                                const float m0 = fabsf(dx) - Cf[0], m1 = fabsf(dy) - Cf[1],
                                            m2 = fabsf(dz) - Cf[2], m3 = fabsf(dt) - Cf[3];
                                const bool out = m0 > delta[0] || m1 > delta[1] || m2 > delta[2] || m3 > delta[3];
                                const bool in = m0 < -delta[0] && m1 < -delta[1] && m2 < -delta[2] && m3 < -delta[3];
                                ok = !out;
                                if (!out && !in) unsure_a = true;
                            }
                            if (ok) {
                                const float q = fmaf(dt, dt, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
                                const float d = fmaf(fwd, sqrt_approx(q), wvs * fabsf(fv0 - cvs));
                                if (d < b1a) { b2a = b1a; b1a = d; i1a = s; } else { b2a = fminf(b2a, d); }
                            }
                        }
                        {
                            const float dx = r0 - rp1[0], dy = r1 - rp1[1], dz = r2 - rp1[2], dt = r3 - rp1[3];
                            bool ok = true;
                            if (!fl) {
                                const float m0 = fabsf(dx) - Cf[0], m1 = fabsf(dy) - Cf[1],
                                            m2 = fabsf(dz) - Cf[2], m3 = fabsf(dt) - Cf[3];
                                const bool out = m0 > delta[0] || m1 > delta[1] || m2 > delta[2] || m3 > delta[3];
                                const bool in = m0 < -delta[0] && m1 < -delta[1] && m2 < -delta[2] && m3 < -delta[3];
                                ok = !out;
                                if (!out && !in) unsure_b = true;
                            }
                            if (ok) {
                                const float q = fmaf(dt, dt, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
                                const float d = fmaf(fwd, sqrt_approx(q), wvs * fabsf(fv1 - cvs));
                                if (d < b1b) { b2b = b1b; b1b = d; i1b = s; } else { b2b = fminf(b2b, d); }
                            }
                        }
                    }
                }
                const float Wa = (useval ? (float)a.wv * (fabsf(fv0) + cvmax) : 0.f);
                const float Wq = (useval ? (float)a.wv * (fabsf(fv1) + cvmax) : 0.f);
                const bool oka = !(a.debug & 2) && !unsure_a && b1a < INF_F &&
                                 b2a * (1.f - KSCR) > b1a * (1.f + KSCR) + 2.f * KSCR * Wa + 2.f * Aabs;
                const bool okb = !(a.debug & 2) && !unsure_b && b1b < INF_F &&
                                 b2b * (1.f - KSCR) > b1b * (1.f + KSCR) + 2.f * KSCR * Wq + 2.f * Aabs;
                sl0 = oka ? i1a : -1;
                sl1 = okb ? i1b : -1;
                const bool need0 = live0 && !oka, need1 = live1 && !okb;
                if (__any_sync(0xffffffffu, need0 || need1)) {
                    // exact fp64 over every survivor inside the margin (all of them
                    // when the screen was unsure about a box test or overflowed)
                    const float ta = (b1a < INF_F && !unsure_a)
                                         ? (b1a * (1.f + KSCR) + 2.f * KSCR * Wa + 2.f * Aabs) * (1.f + 0x1.0p-17f)
                                         : INF_F;
                    const float tb = (b1b < INF_F && !unsure_b)
                                         ? (b1b * (1.f + KSCR) + 2.f * KSCR * Wq + 2.f * Aabs) * (1.f + 0x1.0p-17f)
                                         : INF_F;
                    double eDa = INF_D, eDb = INF_D;
                    int eIa = INT_MAX, eIb = INT_MAX, eSa = -1, eSb = -1;
                    if (need0 || need1) {
                        for (int s = 0; s < cnt; ++s) {
                            const int cid = S.id[s];
                            const float cvs = S.cvf[s], wvs = S.wvf[s];
                            if (need0) {
                                const float dx = S.rc[s][0] - rp0[0], dy = S.rc[s][1] - rp0[1],
                                            dz = S.rc[s][2] - rp0[2], dt = S.rc[s][3] - rp0[3];
                                const float q = fmaf(dt, dt, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
                                const float d = fmaf(fwd, sqrt_approx(q), wvs * fabsf(fv0 - cvs));
                                double D;
                                if (!(d > ta) && exact_pair(S.c[s], P0[0], P0[1], P0[2], P0[3], P0[4],
                                                            S.has[s], a.cf, a.wv, a.wd, Cd, D) &&
                                    better(D, cid, eDa, eIa)) {
                                    eDa = D; eIa = cid; eSa = s;
                                }
                            }
                            if (need1) {
                                const float dx = S.rc[s][0] - rp1[0], dy = S.rc[s][1] - rp1[1],
                                            dz = S.rc[s][2] - rp1[2], dt = S.rc[s][3] - rp1[3];
                                const float q = fmaf(dt, dt, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
                                const float d = fmaf(fwd, sqrt_approx(q), wvs * fabsf(fv1 - cvs));
                                double D;
                                if (!(d > tb) && exact_pair(S.c[s], P1[0], P1[1], P1[2], P1[3], P1[4],
                                                            S.has[s], a.cf, a.wv, a.wd, Cd, D) &&
                                    better(D, cid, eDb, eIb)) {
                                    eDb = D; eIb = cid; eSb = s;
                                }
                            }
                        }
                    }
                    if (need0) sl0 = eSa;
                    if (need1) sl1 = eSb;
                }
                if (!live0) sl0 = -1;
                if (!live1) sl1 = -1;
            }
        }
    }

    const int lab0 = (live0 && sl0 >= 0) ? S.id[sl0] : -1;
    const int lab1 = (live1 && sl1 >= 0) ? S.id[sl1] : -1;
    if (live0) {
        if (deferred) {
            a.labels[p0] = -2;
            const unsigned long long q = atomicAdd(a.n_deferred, 1ull);
            if ((long long)q < a.deferred_cap) a.deferred[q] = p0;
        } else {
            a.labels[p0] = lab0;
            if (lab0 < 0) {
                const unsigned long long q = atomicAdd(a.n_stranded, 1ull);
                if ((long long)q < a.stranded_cap) a.stranded[q] = p0;
            }
        }
    }
    if (live1) {
        if (deferred) {
            a.labels[p1] = -2;
            const unsigned long long q = atomicAdd(a.n_deferred, 1ull);
            if ((long long)q < a.deferred_cap) a.deferred[q] = p1;
        } else {
            a.labels[p1] = lab1;
            if (lab1 < 0) {
                const unsigned long long q = atomicAdd(a.n_stranded, 1ull);
                if ((long long)q < a.stranded_cap) a.stranded[q] = p1;
            }
        }
    }
    int ovf_local = 0;
    if (a.accumulate && nfast && !deferred) {
        int nrec = 0;
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
            if (nrec < RMAX) {
                if (lane == 0) {
                    PRec &R = S.rec[w][nrec];
                    R.slot = L;
                    R.n = __popc(g0) + __popc(g1);
#pragma unroll
                    for (int d = 0; d < 5; ++d) R.s[d] = s5[d];
                }
            } else if (lane == 0) {
                unsigned long long *dst = a.acc + (size_t)S.id[L] * MFSEG_ACC_WORDS;
                for (int d = 0; d < 4; ++d) atomic_add_double_fix(dst + 2 * d, s5[d], &ovf_local);
                atomic_add_double_fix(dst + 8, s5[4], &ovf_local);
                atomicAdd(dst + 12, (unsigned long long)(__popc(g0) + __popc(g1)));
            }
            ++nrec;
        }
        if (lane == 0) S.nrec[w] = min(nrec, RMAX);
        __syncthreads();
        for (int i = tid; i < nfast * 6; i += NT) {
            const int s = i / 6, wd = i - s * 6;
            double acc = 0.0;
            long long n = 0;
            bool any = false;
            for (int q = 0; q < NW; ++q)
                for (int r = 0; r < S.nrec[q]; ++r) {
                    const PRec &R = S.rec[q][r];
                    if (R.slot != s) continue;
                    any = true;
                    if (wd < 5) acc = DADD(acc, R.s[wd]);
                    else n += R.n;
                }
            if (!any) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            if (wd < 4) atomic_add_double_fix(dst + 2 * wd, acc, &ovf_local);
            else if (wd == 4) atomic_add_double_fix(dst + 8, acc, &ovf_local);   // point-value sum
            else atomicAdd(dst + 12, (unsigned long long)n);                     // n_points
        }
    }
    if (ovf_local) *a.overflow = 1;
}

int launch_point_assign_v3(const PointArgs &a, long long max_tiles, cudaStream_t st) {
    if (max_tiles <= 0) return 0;
    ::mfseg::count_launch();
    k_point_assign3<<<(unsigned)max_tiles, NT, 0, st>>>(a);
    MFSEG_LAUNCH("k_point_assign3");
    return 0;
}

}  // namespace mfseg
