// Windowed assignment with fused exact accumulation (the hot path).
//
// Reference: engine._assign_chunk / _metric / _fallback_assign / accumulate
// (engine.py:137-263).  For every sample the label is
//     argmin_(D, id) { D(s, c) : c in cand(bin(s)), |c - s| <= C per axis }
// with D computed in the reference's fp64 operation order; if the set is empty
// the sample is "stranded" and takes the doubling-window fallback over all K
// centres.  This is an exact predicate per (sample, centre) pair, so the
// tiling below changes only WHICH pairs get evaluated, never the result.
//
// Field tiles (k_field_assign): a CTA owns a TX x TY x TZ brick of one
// timestep lying inside ONE sample bin, so the tile shares one candidate list.
// For every candidate it derives exact lower/upper bounds of the fp64 D over
// the tile (all fp64 ops are monotone under round-to-nearest, so evaluating
// the reference formula on the extreme per-axis distances bounds every
// sample's computed D).  Candidates whose lower bound exceeds the smallest
// upper bound of a candidate valid on the whole tile can never win and are
// culled before the per-sample loop.  Typical survivors: a handful of ~50.
//
// Accumulation: per warp, a butterfly sum per distinct label (fixed lane
// order), per tile a fixed-order combine of the warp records, then one
// conversion to 128-bit fixed point and integer atomics.  Tiles are canonical
// (independent of the GPU count) and integer addition is associative, so the
// sums are deterministic and shard-count independent.
#include <climits>
#include <cstdlib>

#include "kernels.cuh"

namespace mfseg {



namespace {

constexpr double INF = __builtin_huge_val();

// |fl(c - s)| over s in [lo, hi] (both valid samples): min and max
__device__ __forceinline__ void axis_range(double c, double lo, double hi, double &dmin,
                                           double &dmax) {
    double a = DSUB(c, lo), b = DSUB(c, hi);   // a >= b
    double fa = fabs(a), fb = fabs(b);
    dmax = fmax(fa, fb);
    dmin = (b <= 0.0 && a >= 0.0) ? 0.0 : fmin(fa, fb);
}

__device__ __forceinline__ double bound_D(double dx, double dy, double dz, double tsq, double vt,
                                          double wd) {
    double q = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
    return DADD(vt, DMUL(wd, DSQRT(DADD(q, tsq))));
}

template <int NW>
__device__ double block_min(double v, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double r = red[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) r = fmin(r, red[i]);
    return r;
}

template <int NW>
__device__ double block_max(double v, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double r = red[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) r = fmax(r, red[i]);
    return r;
}

// value-term bounds over v in [vlo, vhi]
__device__ __forceinline__ void value_bounds(double vlo, double vhi, double cv, bool chas,
                                             double wv, double &lo, double &hi) {
    if (wv > 0.0 && chas) {
        double a = DSUB(vlo, cv), b = DSUB(vhi, cv);
        double fa = fabs(a), fb = fabs(b);
        double amin = (a <= 0.0 && b >= 0.0) ? 0.0 : fmin(fa, fb);
        lo = DMUL(wv, amin);
        hi = DMUL(wv, fmax(fa, fb));
    } else {
        lo = hi = 0.0;
    }
}

// Per-tile, per-label exact accumulation.  Each warp reduces its lanes' samples
// per distinct label (butterfly, fixed lane order) into records; the block
// combines records of equal label in (warp, record) order and adds the
// 128-bit fixed-point result to acc with integer atomics.
template <int NW, int RCAP>
struct Records {
    int lab[NW][RCAP];
    int cnt[NW][RCAP];
    double val[NW][RCAP][4];   // x, y, z, v  (t is added exactly as count * t or summed)
    double tsum[NW][RCAP];
    int nrec[NW];
};

template <int NW, int RCAP>
__device__ void warp_records(Records<NW, RCAP> &R, int lab, double x, double y, double z,
                             double t, double v, int &nrec) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned pend = __ballot_sync(0xffffffffu, lab >= 0);
    while (pend) {
        int leader = __ffs(pend) - 1;
        int L = __shfl_sync(0xffffffffu, lab, leader);
        bool mine = lab == L;
        unsigned msk = __ballot_sync(0xffffffffu, mine);
        double sx = warp_sum_d(mine ? x : 0.0);
        double sy = warp_sum_d(mine ? y : 0.0);
        double sz = warp_sum_d(mine ? z : 0.0);
        double st = warp_sum_d(mine ? t : 0.0);
        double sv = warp_sum_d(mine ? v : 0.0);
        if (lane == 0 && nrec < RCAP) {
            R.lab[w][nrec] = L;
            R.cnt[w][nrec] = __popc(msk);
            R.val[w][nrec][0] = sx;
            R.val[w][nrec][1] = sy;
            R.val[w][nrec][2] = sz;
            R.val[w][nrec][3] = sv;
            R.tsum[w][nrec] = st;
        }
        ++nrec;
        pend &= ~msk;
    }
}

// word offsets inside one cluster's MFSEG_ACC_WORDS accumulator
constexpr int ACC_X = 0, ACC_PV = 8, ACC_FV = 10, ACC_NP = 12, ACC_NF = 13;

template <int NW, int RCAP, int NT>
__device__ void flush_records(Records<NW, RCAP> &R, unsigned long long *acc, bool field_kind,
                              int *overflow) {
    __syncthreads();
    int total = 0;
    int base[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        base[w] = total;
        total += min(R.nrec[w], RCAP);
    }
    for (int r = threadIdx.x; r < total; r += NT) {
        int w = 0;
#pragma unroll
        for (int q = 1; q < NW; ++q)
            if (r >= base[q]) w = q;
        int i = r - base[w];
        int L = R.lab[w][i];
        bool first = true;
        for (int q = 0; q < NW && first; ++q) {
            int n = min(R.nrec[q], RCAP);
            for (int j = 0; j < n; ++j) {
                if (q == w && j == i) break;
                if (R.lab[q][j] == L) {
                    first = false;
                    break;
                }
            }
            if (q == w) break;
        }
        if (!first) continue;
        double sx = 0.0, sy = 0.0, sz = 0.0, sv = 0.0, stt = 0.0;
        long long n = 0;
        for (int q = w; q < NW; ++q) {
            int m = min(R.nrec[q], RCAP);
            for (int j = (q == w ? i : 0); j < m; ++j) {
                if (R.lab[q][j] != L) continue;
                sx = DADD(sx, R.val[q][j][0]);
                sy = DADD(sy, R.val[q][j][1]);
                sz = DADD(sz, R.val[q][j][2]);
                sv = DADD(sv, R.val[q][j][3]);
                stt = DADD(stt, R.tsum[q][j]);
                n += R.cnt[q][j];
            }
        }
        unsigned long long *a = acc + (size_t)L * MFSEG_ACC_WORDS;
        atomic_add_double_fix(a + ACC_X + 0, sx, overflow);
        atomic_add_double_fix(a + ACC_X + 2, sy, overflow);
        atomic_add_double_fix(a + ACC_X + 4, sz, overflow);
        atomic_add_double_fix(a + ACC_X + 6, stt, overflow);
        atomic_add_double_fix(a + (field_kind ? ACC_FV : ACC_PV), sv, overflow);
        atomicAdd(a + (field_kind ? ACC_NF : ACC_NP), (unsigned long long)n);
    }
    for (int w = 0; w < NW; ++w)
        if (R.nrec[w] > RCAP && threadIdx.x == 0) *overflow = 2;   // cannot happen: RCAP = 32 * SPT
}

}  // namespace

// ====================================================================== fields
template <int TX, int TY, int TZ, int NT>
__global__ void __launch_bounds__(NT) k_field_assign(FieldArgs a) {
    constexpr int NS = TX * TY * TZ, SPT = NS / NT, NW = NT / 32, CAP = NT;
    constexpr int RCAP = 32 * SPT;
    static_assert(NS % NT == 0, "tile must be a multiple of the block");
    __shared__ double s_x[TX], s_y[TY], s_z[TZ];
    __shared__ int s_id[CAP];
    __shared__ double s_cx[CAP], s_cy[CAP], s_cz[CAP], s_tsq[CAP], s_cv[CAP];
    __shared__ unsigned s_box[CAP];
    __shared__ unsigned char s_has[CAP];
    __shared__ double s_red[NW];
    __shared__ int s_wc[NW];
    __shared__ Records<NW, RCAP> R;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    long long tile = blockIdx.x;
    const int txi = (int)(tile % a.ntx);
    tile /= a.ntx;
    const int tyi = (int)(tile % a.nty);
    tile /= a.nty;
    const int tzi = (int)(tile % a.ntz);
    const int m = (int)(tile / a.ntz);
    const AxisTile X = a.xt[txi], Y = a.yt[tyi], Z = a.zt[tzi];
    if (tid < X.len) s_x[tid] = cell_coord(a.ox, a.sx, X.start + tid);
    if (tid < Y.len) s_y[tid] = cell_coord(a.oy, a.sy, Y.start + tid);
    if (tid < Z.len) s_z[tid] = cell_coord(a.oz, a.sz, Z.start + tid);
    const double tm = a.times[m];
    const int sbin = ((a.tbin[m] * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;

    int lx[SPT], ly[SPT], lz[SPT];
    bool live[SPT];
    double v[SPT];
    long long flat[SPT];
    double vlo = INF, vhi = -INF;
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        int li = tid + s * NT;
        lx[s] = li % TX;
        ly[s] = (li / TX) % TY;
        lz[s] = li / (TX * TY);
        live[s] = lx[s] < X.len && ly[s] < Y.len && lz[s] < Z.len;
        flat[s] = (((long long)m * a.nz + (Z.start + lz[s])) * a.ny + (Y.start + ly[s])) *
                      (long long)a.nx + (X.start + lx[s]);
        v[s] = live[s] ? __ldg(a.values + flat[s]) : 0.0;
        if (live[s]) {
            vlo = fmin(vlo, v[s]);
            vhi = fmax(vhi, v[s]);
        }
    }
    if (a.wv > 0.0) {
        vlo = block_min<NW>(vlo, s_red);
        vhi = block_max<NW>(vhi, s_red);
    }
    __syncthreads();
    double px[SPT], py[SPT], pz[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        px[s] = live[s] ? s_x[lx[s]] : 0.0;
        py[s] = live[s] ? s_y[ly[s]] : 0.0;
        pz[s] = live[s] ? s_z[lz[s]] : 0.0;
    }

    double bestD[SPT];
    int bestI[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        bestD[s] = INF;
        bestI[s] = INT_MAX;
    }

    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    for (int cb = L0; cb < L1; cb += CAP) {
        // ---- phase A: one candidate per thread -> exact D bounds over the tile
        int ci = cb + tid;
        bool have = ci < L1;
        int id = 0;
        double cx = 0, cy = 0, cz = 0, cv = 0, tsq = 0, Dlo = INF, Dhi = INF;
        bool chas = false, full = false;
        unsigned box = 0;
        if (have) {
            id = a.g.cand_ids[ci];
            int4 b0 = a.g.vbox[2 * id], b1 = a.g.vbox[2 * id + 1];
            int xa = max(b0.x - X.start, 0), xb = min(b0.y - X.start, X.len - 1);
            int ya = max(b0.z - Y.start, 0), yb = min(b0.w - Y.start, Y.len - 1);
            int za = max(b1.x - Z.start, 0), zb = min(b1.y - Z.start, Z.len - 1);
            have = m >= b1.z && m <= b1.w && xa <= xb && ya <= yb && za <= zb;
            if (have) {
                cx = a.c.x[id];
                cy = a.c.y[id];
                cz = a.c.z[id];
                double ct = DMUL(a.cf, DSUB(a.c.t[id], tm));
                tsq = DMUL(ct, ct);
                chas = a.chas[id] != 0;
                cv = chas ? a.cval[id] : 0.0;
                full = xa == 0 && xb == X.len - 1 && ya == 0 && yb == Y.len - 1 && za == 0 &&
                       zb == Z.len - 1;
                double dxl, dxh, dyl, dyh, dzl, dzh, vl, vh;
                axis_range(cx, s_x[xa], s_x[xb], dxl, dxh);
                axis_range(cy, s_y[ya], s_y[yb], dyl, dyh);
                axis_range(cz, s_z[za], s_z[zb], dzl, dzh);
                value_bounds(vlo, vhi, cv, chas, a.wv, vl, vh);
                Dlo = bound_D(dxl, dyl, dzl, tsq, vl, a.wd);
                Dhi = bound_D(dxh, dyh, dzh, tsq, vh, a.wd);
                box = (unsigned)xa | ((unsigned)xb << 5) | ((unsigned)ya << 10) |
                      ((unsigned)yb << 15) | ((unsigned)za << 20) | ((unsigned)zb << 25) |
                      (full ? 0x80000000u : 0u);
            }
        }
        // ---- phase B: cull against the best whole-tile upper bound, compact
        double ub = block_min<NW>(full ? Dhi : INF, s_red);
        bool surv = have && Dlo <= ub;
        unsigned bal = __ballot_sync(0xffffffffu, surv);
        if (lane == 0) s_wc[w] = __popc(bal);
        __syncthreads();
        int off = 0, nsurv = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < w ? s_wc[q] : 0;
            nsurv += s_wc[q];
        }
        if (surv) {
            int pos = off + __popc(bal & ((1u << lane) - 1u));
            s_id[pos] = id;
            s_cx[pos] = cx;
            s_cy[pos] = cy;
            s_cz[pos] = cz;
            s_tsq[pos] = tsq;
            s_cv[pos] = cv;
            s_has[pos] = chas;
            s_box[pos] = box;
        }
        __syncthreads();
        // ---- phase C: exact per-sample evaluation over the survivors
        for (int q = 0; q < nsurv; ++q) {
            const unsigned bx = s_box[q];
            const int cid = s_id[q];
            const double qx = s_cx[q], qy = s_cy[q], qz = s_cz[q], qt = s_tsq[q], qv = s_cv[q];
            const bool qh = s_has[q] != 0;
            const bool qfull = (bx >> 31) != 0;
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                if (!live[s]) continue;
                if (!qfull) {
                    int x0 = bx & 31, x1 = (bx >> 5) & 31, y0 = (bx >> 10) & 31,
                        y1 = (bx >> 15) & 31, z0 = (bx >> 20) & 31, z1 = (bx >> 25) & 31;
                    if (lx[s] < x0 || lx[s] > x1 || ly[s] < y0 || ly[s] > y1 || lz[s] < z0 ||
                        lz[s] > z1)
                        continue;
                }
                double dx = DSUB(qx, px[s]), dy = DSUB(qy, py[s]), dz = DSUB(qz, pz[s]);
                double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
                double D = metric_tail(qq, qt, v[s], qv, qh, a.wv, a.wd);
                if (better(D, cid, bestD[s], bestI[s])) {
                    bestD[s] = D;
                    bestI[s] = cid;
                }
            }
        }
        __syncthreads();
    }

    // ---- labels, stranded list
    int lab[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        lab[s] = (live[s] && bestI[s] != INT_MAX) ? bestI[s] : -1;
        if (live[s]) {
            a.labels[flat[s]] = lab[s];
            if (lab[s] < 0) {
                unsigned long long p = atomicAdd(a.n_stranded, 1ull);
                if ((long long)p < a.stranded_cap) a.stranded[p] = flat[s];
            }
        }
    }
    if (!a.accumulate) return;
    // ---- fused exact accumulation
    int nrec = 0;
#pragma unroll
    for (int s = 0; s < SPT; ++s)
        warp_records<NW, RCAP>(R, lab[s], px[s], py[s], pz[s], tm, v[s], nrec);
    if (lane == 0) R.nrec[w] = nrec;
    flush_records<NW, RCAP, NT>(R, a.acc, true, a.overflow);
}

// ====================================================================== points
template <int NT, int SPT>
__global__ void __launch_bounds__(NT) k_point_assign(PointArgs a) {
    constexpr int NW = NT / 32, CAP = NT, RCAP = 32 * SPT;
    __shared__ int s_id[CAP];
    __shared__ double s_cx[CAP], s_cy[CAP], s_cz[CAP], s_ct[CAP], s_cv[CAP];
    __shared__ unsigned char s_flags[CAP];   // bit0 has, bit1 full
    __shared__ double s_red[NW];
    __shared__ int s_wc[NW];
    __shared__ Records<NW, RCAP> R;

    if ((int)blockIdx.x >= *a.n_tiles) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int4 T = a.tiles[blockIdx.x];
    const int sbin = T.x;
    double px[SPT], py[SPT], pz[SPT], pt[SPT], v[SPT];
    bool live[SPT];
    long long pos[SPT];
    double lo[4] = {INF, INF, INF, INF}, hi[4] = {-INF, -INF, -INF, -INF};
    double vlo = INF, vhi = -INF;
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        int li = tid + s * NT;
        live[s] = li < T.z;
        pos[s] = (long long)T.y + li;
        if (live[s]) {
            px[s] = a.x[pos[s]];
            py[s] = a.y[pos[s]];
            pz[s] = a.z[pos[s]];
            pt[s] = a.t[pos[s]];
            v[s] = a.v[pos[s]];
            lo[0] = fmin(lo[0], px[s]);
            hi[0] = fmax(hi[0], px[s]);
            lo[1] = fmin(lo[1], py[s]);
            hi[1] = fmax(hi[1], py[s]);
            lo[2] = fmin(lo[2], pz[s]);
            hi[2] = fmax(hi[2], pz[s]);
            lo[3] = fmin(lo[3], pt[s]);
            hi[3] = fmax(hi[3], pt[s]);
            vlo = fmin(vlo, v[s]);
            vhi = fmax(vhi, v[s]);
        } else {
            px[s] = py[s] = pz[s] = pt[s] = v[s] = 0.0;
        }
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        lo[d] = block_min<NW>(lo[d], s_red);
        hi[d] = block_max<NW>(hi[d], s_red);
    }
    if (a.wv > 0.0) {
        vlo = block_min<NW>(vlo, s_red);
        vhi = block_max<NW>(vhi, s_red);
    }
    const double Cd[4] = {a.Cx, a.Cy, a.Cz, a.Ct};

    double bestD[SPT];
    int bestI[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        bestD[s] = INF;
        bestI[s] = INT_MAX;
    }
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    for (int cb = L0; cb < L1; cb += CAP) {
        int ci = cb + tid;
        bool have = ci < L1;
        int id = 0;
        double c4[4] = {0, 0, 0, 0}, cv = 0, Dlo = INF, Dhi = INF;
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
                double da = DSUB(c4[d], lo[d]), db = DSUB(c4[d], hi[d]);   // da >= db
                if (da < -Cd[d] || db > Cd[d]) have = false;                // no sample passes
                if (!(da <= Cd[d] && db >= -Cd[d])) full = false;           // not all pass
                double ea = fmin(da, Cd[d]), eb = fmax(db, -Cd[d]);         // passing range
                double fa = fabs(ea), fb = fabs(eb);
                dh[d] = fmax(fa, fb);
                dl[d] = (eb <= 0.0 && ea >= 0.0) ? 0.0 : fmin(fa, fb);
            }
            if (have) {
                chas = a.chas[id] != 0;
                cv = chas ? a.cval[id] : 0.0;
                double tl = DMUL(a.cf, dl[3]), th = DMUL(a.cf, dh[3]);
                double vl, vh;
                value_bounds(vlo, vhi, cv, chas, a.wv, vl, vh);
                Dlo = bound_D(dl[0], dl[1], dl[2], DMUL(tl, tl), vl, a.wd);
                Dhi = bound_D(dh[0], dh[1], dh[2], DMUL(th, th), vh, a.wd);
            } else {
                full = false;
            }
        }
        double ub = block_min<NW>(full ? Dhi : INF, s_red);
        bool surv = have && Dlo <= ub;
        unsigned bal = __ballot_sync(0xffffffffu, surv);
        if (lane == 0) s_wc[w] = __popc(bal);
        __syncthreads();
        int off = 0, nsurv = 0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            off += q < w ? s_wc[q] : 0;
            nsurv += s_wc[q];
        }
        if (surv) {
            int p = off + __popc(bal & ((1u << lane) - 1u));
            s_id[p] = id;
            s_cx[p] = c4[0];
            s_cy[p] = c4[1];
            s_cz[p] = c4[2];
            s_ct[p] = c4[3];
            s_cv[p] = cv;
            s_flags[p] = (chas ? 1 : 0) | (full ? 2 : 0);
        }
        __syncthreads();
        for (int q = 0; q < nsurv; ++q) {
            const int cid = s_id[q];
            const double qx = s_cx[q], qy = s_cy[q], qz = s_cz[q], qt = s_ct[q], qv = s_cv[q];
            const unsigned fl = s_flags[q];
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                if (!live[s]) continue;
                double dx = DSUB(qx, px[s]), dy = DSUB(qy, py[s]), dz = DSUB(qz, pz[s]),
                       dt = DSUB(qt, pt[s]);
                if (!(fl & 2u)) {
                    if (!(fabs(dx) <= a.Cx && fabs(dy) <= a.Cy && fabs(dz) <= a.Cz &&
                          fabs(dt) <= a.Ct))
                        continue;
                }
                double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
                double ct = DMUL(a.cf, dt);
                double D = metric_tail(qq, DMUL(ct, ct), v[s], qv, (fl & 1u) != 0, a.wv, a.wd);
                if (better(D, cid, bestD[s], bestI[s])) {
                    bestD[s] = D;
                    bestI[s] = cid;
                }
            }
        }
        __syncthreads();
    }
    int lab[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        lab[s] = (live[s] && bestI[s] != INT_MAX) ? bestI[s] : -1;
        if (live[s]) {
            a.labels[pos[s]] = lab[s];
            if (lab[s] < 0) {
                unsigned long long p = atomicAdd(a.n_stranded, 1ull);
                if ((long long)p < a.stranded_cap) a.stranded[p] = pos[s];
            }
        }
    }
    if (!a.accumulate) return;
    int nrec = 0;
#pragma unroll
    for (int s = 0; s < SPT; ++s)
        warp_records<NW, RCAP>(R, lab[s], px[s], py[s], pz[s], pt[s], v[s], nrec);
    if (lane == 0) R.nrec[w] = nrec;
    flush_records<NW, RCAP, NT>(R, a.acc, false, a.overflow);
}

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
        s0 = cell_coord(a.ox, a.sx, i);
        s1 = cell_coord(a.oy, a.sy, j);
        s2 = cell_coord(a.oz, a.sz, k);
        s3 = a.times[m];
        v = a.values[idx];
    } else {
        s0 = a.px[idx];
        s1 = a.py[idx];
        s2 = a.pz[idx];
        s3 = a.pt[idx];
        v = a.pv[idx];
    }
    double mult = 2.0;
    int best = INT_MAX;
    for (int guard = 0; guard < 1100 && best == INT_MAX; ++guard, mult = DMUL(mult, 2.0)) {
        double b0 = DMUL(mult, a.C[0]), b1 = DMUL(mult, a.C[1]), b2 = DMUL(mult, a.C[2]),
               b3 = DMUL(mult, a.C[3]);
        double bD = INF;
        int bI = INT_MAX;
        for (int c = lane; c < a.K; c += 32) {
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
};

__device__ void deferred_one(const FallbackArgs &a, const DeferredGeo &G, long long idx) {
    const int lane = threadIdx.x & 31;
    double s0, s1, s2, s3, v;
    int bt;
    if (a.kind == 1) {
        long long r = idx;
        const int i = (int)(r % a.nx);
        r /= a.nx;
        const int j = (int)(r % a.ny);
        r /= a.ny;
        const int k = (int)(r % a.nz);
        const int m = (int)(r / a.nz);
        s0 = cell_coord(a.ox, a.sx, i);
        s1 = cell_coord(a.oy, a.sy, j);
        s2 = cell_coord(a.oz, a.sz, k);
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
    const int sbin = ((bt * G.k.z + bz) * G.k.y + by) * G.k.x + bx;
    double bD = INF;
    int bI = INT_MAX;
    for (int p = G.g.cand_start[sbin] + lane; p < G.g.cand_start[sbin + 1]; p += 32) {
        const int c = G.g.cand_ids[p];
        const double dx = DSUB(a.c.x[c], s0), dy = DSUB(a.c.y[c], s1), dz = DSUB(a.c.z[c], s2),
                     dt = DSUB(a.c.t[c], s3);
        if (!(fabs(dx) <= a.C[0] && fabs(dy) <= a.C[1] && fabs(dz) <= a.C[2] && fabs(dt) <= a.C[3]))
            continue;
        const double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
        const double ct = DMUL(a.cf, dt);
        const bool h = a.chas[c] != 0;
        const double D = metric_tail(qq, DMUL(ct, ct), v, h ? a.cval[c] : 0.0, h, a.wv, a.wd);
        if (better(D, c, bD, bI)) {
            bD = D;
            bI = c;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double oD = __shfl_xor_sync(0xffffffffu, bD, o);
        const int oI = __shfl_xor_sync(0xffffffffu, bI, o);
        if (better(oD, oI, bD, bI)) {
            bD = oD;
            bI = oI;
        }
    }
    if (lane != 0) return;
    if (bI == INT_MAX) {   // stranded: the fallback kernel runs next
        a.labels[idx] = -1;
        const unsigned long long q = atomicAdd((unsigned long long *)a.n_stranded, 1ull);
        if ((long long)q < a.cap) ((long long *)a.stranded)[q] = idx;
        return;
    }
    a.labels[idx] = bI;
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

__global__ void k_deferred(FallbackArgs a, DeferredGeo G) {
    const long long n = (long long)*G.count;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n <= G.cap) {
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
                                   double oz, double sx, double sy, double sz,
                                   const double *times, const double *values, const int *labels,
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
        atomic_add_double_fix(p + ACC_X + 0, cell_coord(ox, sx, i), overflow);
        atomic_add_double_fix(p + ACC_X + 2, cell_coord(oy, sy, j), overflow);
        atomic_add_double_fix(p + ACC_X + 4, cell_coord(oz, sz, k), overflow);
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
constexpr int FTX = 16, FTY = 8, FTZ = 4, FNT = 256;
constexpr int PNT = 128, PSPT = 2;   // tile = 256 points for v1 and v3 (k_point_assign3: 128 thr x 2)

// field kernel generation: 5 (default), or 4 / 3 / 1 for comparisons
int field_version() {
    if (getenv("MFSEG_FIELD_V1")) return 1;
    if (getenv("MFSEG_FIELD_V3")) return 3;
    if (getenv("MFSEG_FIELD_V4")) return 4;
    return 5;
}

int field_tile_dims(int *tx, int *ty, int *tz) {
    const bool v5 = field_version() == 5;
    *tx = FTX;
    *ty = v5 ? 16 : FTY;
    *tz = v5 ? 16 : FTZ;
    return 0;
}
static_assert(PNT * PSPT == POINT_TILE, "v1 point tile size");
// point kernel generation: 4 (default), or 3 / 1 for comparisons
int point_version() {
    if (getenv("MFSEG_POINT_V1")) return 1;
    if (getenv("MFSEG_POINT_V3")) return 3;
    return 4;
}
int point_tile_size() { return point_version() == 4 ? POINT_CHUNK : POINT_TILE; }

int launch_field_assign_v2(const FieldArgs &a, long long ntiles, cudaStream_t st);
int launch_field_assign_v5(const FieldArgs &a, cudaStream_t st);

int launch_field_assign(const FieldArgs &a, long long ntiles, cudaStream_t st) {
    const int ver = field_version();
    if (ver == 5) return launch_field_assign_v5(a, st);
    if (ver != 1) return launch_field_assign_v2(a, ntiles, st);
    if (ntiles <= 0) return 0;
    if (ntiles > 0x7fffffffll) {
        set_error("field tile grid too large");
        return 3;
    }
    ::mfseg::count_launch();
    k_field_assign<FTX, FTY, FTZ, FNT><<<(unsigned)ntiles, FNT, 0, st>>>(a);
    MFSEG_LAUNCH("k_field_assign");
    return 0;
}

int launch_point_assign_v3(const PointArgs &a, long long max_tiles, cudaStream_t st);
int launch_point_assign_v4(const PointArgs &a, long long max_tiles, cudaStream_t st);

int launch_point_assign(const PointArgs &a, long long max_tiles, cudaStream_t st) {
    const int ver = point_version();
    if (ver == 4) return launch_point_assign_v4(a, max_tiles, st);
    if (ver == 3) return launch_point_assign_v3(a, max_tiles, st);
    if (max_tiles <= 0) return 0;
    ::mfseg::count_launch();
    k_point_assign<PNT, PSPT><<<(unsigned)max_tiles, PNT, 0, st>>>(a);
    MFSEG_LAUNCH("k_point_assign");
    return 0;
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
    ::mfseg::count_launch();
    k_deferred<<<148 * 4, 256, 0, st>>>(a, G);
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
                                                f->spacing[1], f->spacing[2], f->times,
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
