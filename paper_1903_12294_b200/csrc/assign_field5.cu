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
//  * each warp walks 8 bricks of 4x4x4 voxels x 4 timesteps (8 samples per
//    lane).  Warp culling uses the quad tables (O(1) per candidate and brick);
//  * the fp32 screen tracks best/second best as packed 32-bit keys
//    (float bits of d with the low 7 mantissa bits replaced by the slot), so
//    the top-2 update is three integer min/max;
//  * partial sums: per slot 16-bit count marginals in shared memory (x, y, z,
//    t indices; shared-memory integer atomics), value sums as per-warp fp64
//    running sums in the warp's fixed brick order; once per block the
//    marginals x 128-bit fixed-point coordinates and the warp value sums
//    (converted exactly) go to the global 128-bit sums.
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

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();
constexpr float FLT_BIG = 3.4028234663852886e38f;
constexpr unsigned INF_BITS = 0x7F800000u;

constexpr int BX = 16, BY = 16, BZ = 16, BT = 4;   // block = one bin's 16^3 x 4 samples (at most)
constexpr int NT = 256, NW = 8;
constexpr int CAP = 128;                           // candidates per block (more: deferred)
constexpr unsigned SLOT_MASK = 127u;               // 7 slot bits in the packed keys
constexpr int TE = BX + BY + BZ + BT;              // 52 table entries per candidate
constexpr int OZ = BX + BY, OT = BX + BY + BZ;     // table offsets of z and t
constexpr int NQ = 13;                             // quads: x 4, y 4, z 4, t 1
constexpr int HW = 27;                             // histogram words: x 8, y 8, z 8, t 2, n 1
constexpr float KSCR = 0x1.0p-18f;
constexpr float KCULL = 0x1.0p-16f;

struct __align__(16) Smem5 {
    float tab[CAP][TE];             // 16-byte aligned rows (52 floats)
    float2 qmm[CAP][NQ];            // (min, max) of each quad of table entries
    double c[CAP][5];               // cx, cy, cz, ct, cv (0 when absent)
    double wsum[NW][CAP];           // per-warp fp64 value sums (fixed brick order)
    unsigned hist[CAP][HW];         // 16-bit count marginals, two per word
    unsigned long long xf[BX][2], yf[BY][2], zf[BZ][2], tf[BT][2];
    double x[BX], y[BY], z[BZ], t[BT];
    int id[CAP];
    unsigned box[CAP];              // x 4+4 | y 4+4 | z 4+4 | t 2+2 bits
    float cvf[CAP], wvf[CAP];
    unsigned char has[CAP];
    int wc[NW];
    float red[NW];
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

template <bool USEVAL>
__global__ void __launch_bounds__(NT, 3) k_field_assign5(FieldArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem5 &S = *reinterpret_cast<Smem5 *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    unsigned tile = blockIdx.x;
    const int txi = (int)(tile % (unsigned)a.ntx);
    tile /= (unsigned)a.ntx;
    const int tyi = (int)(tile % (unsigned)a.nty);
    tile /= (unsigned)a.nty;
    const int tzi = (int)(tile % (unsigned)a.ntz);
    const int tti = (int)(tile / (unsigned)a.ntz);
    const AxisTile X = a.xt[txi], Y = a.yt[tyi], Z = a.zt[tzi], Tm = a.tt[tti];
    int ovf_local = 0;

    // ---- block coordinates (reference formula) + 128-bit fixed-point copies
    if (tid < TE) {
        double cv;
        unsigned long long *dst;
        if (tid < BX) {
            cv = cell_coord(a.ox, a.sx, X.start + min(tid, X.len - 1));
            S.x[tid] = cv;
            dst = S.xf[tid];
        } else if (tid < OZ) {
            const int i = tid - BX;
            cv = cell_coord(a.oy, a.sy, Y.start + min(i, Y.len - 1));
            S.y[i] = cv;
            dst = S.yf[i];
        } else if (tid < OT) {
            const int i = tid - OZ;
            cv = cell_coord(a.oz, a.sz, Z.start + min(i, Z.len - 1));
            S.z[i] = cv;
            dst = S.zf[i];
        } else {
            const int i = tid - OT;
            cv = a.times[Tm.start + min(i, Tm.len - 1)];
            S.t[i] = cv;
            dst = S.tf[i];
        }
        long long hi;
        d2fix(cv, dst[0], hi, &ovf_local);
        dst[1] = (unsigned long long)hi;
    }
    const int sbin = ((Tm.bin * a.kz + Z.bin) * a.ky + Y.bin) * a.kx + X.bin;
    const int L0 = a.g.cand_start[sbin], L1 = a.g.cand_start[sbin + 1];
    bool deferred = (L1 - L0) > NT;
    int cnt = 0;
    float cvmax = 0.0f;
    if (!deferred) {
        // ---- candidates whose validity box meets the block, compacted to slots
        const int ci = L0 + tid;
        bool have = ci < L1;
        int id = 0;
        unsigned box = 0;
        if (have) {
            id = a.g.cand_ids[ci];
            const int4 b0 = a.g.vbox[2 * id], b1 = a.g.vbox[2 * id + 1];
            const int xa = max(b0.x - X.start, 0), xb = min(b0.y - X.start, X.len - 1);
            const int ya = max(b0.z - Y.start, 0), yb = min(b0.w - Y.start, Y.len - 1);
            const int za = max(b1.x - Z.start, 0), zb = min(b1.y - Z.start, Z.len - 1);
            const int ta = max(b1.z - Tm.start, 0), tb = min(b1.w - Tm.start, Tm.len - 1);
            have = xa <= xb && ya <= yb && za <= zb && ta <= tb;
            box = (unsigned)xa | ((unsigned)xb << 4) | ((unsigned)ya << 8) | ((unsigned)yb << 12) |
                  ((unsigned)za << 16) | ((unsigned)zb << 20) | ((unsigned)ta << 24) |
                  ((unsigned)tb << 26);
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
            const bool chas = a.chas[id] != 0;
            const double cv = chas ? a.cval[id] : 0.0;
            S.id[p] = id;
            S.c[p][0] = a.c.x[id];
            S.c[p][1] = a.c.y[id];
            S.c[p][2] = a.c.z[id];
            S.c[p][3] = a.c.t[id];
            S.c[p][4] = cv;
            S.box[p] = box;
            S.has[p] = chas;
            S.cvf[p] = (float)cv;
            S.wvf[p] = (USEVAL && chas) ? (float)a.wv : 0.0f;
            if (USEVAL && chas) mycv = fabsf((float)cv);
        }
        if (USEVAL) {
            mycv = warp_max_f(mycv);
            if (lane == 0) S.red[w] = mycv;
        }
        __syncthreads();
        if (USEVAL) {
#pragma unroll
            for (int q = 0; q < NW; ++q) cvmax = fmaxf(cvmax, S.red[q]);
        }
    }

    if (!deferred && cnt > 0) {
        // ---- fp32 tables (fp64 differences and squares as the reference, rounded once)
        for (int e = tid; e < cnt * TE; e += NT) {
            const int p = e / TE, j = e - p * TE;
            const unsigned b = S.box[p];
            float val = INF_F;
            if (j < BX) {
                if (j >= (int)(b & 15u) && j <= (int)((b >> 4) & 15u)) {
                    const double d = DSUB(S.c[p][0], S.x[j]);
                    val = to_f(DMUL(d, d));
                }
            } else if (j < OZ) {
                const int i = j - BX;
                if (i >= (int)((b >> 8) & 15u) && i <= (int)((b >> 12) & 15u)) {
                    const double d = DSUB(S.c[p][1], S.y[i]);
                    val = to_f(DMUL(d, d));
                }
            } else if (j < OT) {
                const int i = j - OZ;
                if (i >= (int)((b >> 16) & 15u) && i <= (int)((b >> 20) & 15u)) {
                    const double d = DSUB(S.c[p][2], S.z[i]);
                    val = to_f(DMUL(d, d));
                }
            } else {
                const int i = j - OT;
                if (i >= (int)((b >> 24) & 3u) && i <= (int)((b >> 26) & 3u)) {
                    const double ct = DMUL(a.cf, DSUB(S.c[p][3], S.t[i]));
                    val = to_f(DMUL(ct, ct));
                }
            }
            S.tab[p][j] = val;
        }
        if (a.accumulate) {
            for (int e = tid; e < cnt * HW; e += NT) (&S.hist[0][0])[e] = 0u;
            for (int e = tid; e < NW * CAP; e += NT) (&S.wsum[0][0])[e] = 0.0;
        }
        __syncthreads();
        // quad (min, max) over the entries that exist in this block
        for (int e = tid; e < cnt * NQ; e += NT) {
            const int p = e / NQ, q = e - p * NQ;
            int base, lo, n;
            if (q < 4) {
                base = 4 * q;
                lo = base;
                n = X.len;
            } else if (q < 8) {
                base = BX + 4 * (q - 4);
                lo = 4 * (q - 4);
                n = Y.len;
            } else if (q < 12) {
                base = OZ + 4 * (q - 8);
                lo = 4 * (q - 8);
                n = Z.len;
            } else {
                base = OT;
                lo = 0;
                n = Tm.len;
            }
            float mn = INF_F, mx = 0.0f;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (lo + r < n) {
                    const float v = S.tab[p][base + r];
                    mn = fminf(mn, v);
                    mx = fmaxf(mx, v);
                }
            S.qmm[p][q] = make_float2(mn, mx);
        }
        __syncthreads();
    }

    // ---- bricks: warp w takes bricks w, w + 8, ..., 4x4x4 voxels x 4 timesteps each
    const long long plane = (long long)a.ny * a.nx, vol = plane * a.nz;
    const float fwd = (float)a.wd;
    const float wvf = USEVAL ? (float)a.wv : 0.0f;
    const float slack = 3e-13f * (float)(a.wd + a.wv);
    const int nrounds = (cnt + 31) >> 5;
    for (int bi = w; bi < 64; bi += NW) {
        const int bx = bi & 3, by = (bi >> 2) & 3, bz = bi >> 4;
        if (4 * bx >= X.len || 4 * by >= Y.len || 4 * bz >= Z.len) continue;   // warp-uniform
        const int lx = 4 * bx + (lane & 3), ly = 4 * by + ((lane >> 2) & 3);
        const int lz0 = 4 * bz + (lane >> 4);
        const bool rowok = lx < X.len && ly < Y.len;
        const long long fbase = (((long long)Tm.start * a.nz + Z.start + lz0) * a.ny + (Y.start + ly)) *
                                    (long long)a.nx + (X.start + lx);
        unsigned livem = 0;   // bit k: sample k = q*4 + t at (lx, ly, lz0 + 2q, t) exists
        double v[8];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int t = 0; t < BT; ++t) {
                const int k = q * BT + t;
                const bool lv = rowok && lz0 + 2 * q < Z.len && t < Tm.len;
                if (lv) livem |= 1u << k;
                v[k] = lv ? __ldg(a.values + fbase + 2 * q * plane + t * vol) : 0.0;
            }

        int sl[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) sl[k] = -1;
        if (!deferred && cnt > 0) {
            float fv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) fv[k] = (livem >> k & 1) ? (float)v[k] : __int_as_float(0x7fffffff);
            // brick value range: min/max of fl(v) = fl(min/max of v) (rounding is monotone)
            float vwl = 0.0f, vwh = 0.0f;
            if (USEVAL) {
                float lo = INF_F, hi = -INF_F;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    lo = fminf(lo, fv[k]);   // NaN (dead sample) ignored
                    hi = fmaxf(hi, fv[k]);
                }
                vwl = warp_min_f(lo);
                vwh = warp_max_f(hi);
            }
            // ---- warp culling from the quad tables
            float dl[4];
            float ubw = INF_F;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                dl[r] = INF_F;
                const int s = lane + 32 * r;
                if (r < nrounds && s < cnt) {
                    const float2 qx = S.qmm[s][bx], qy = S.qmm[s][4 + by], qz = S.qmm[s][8 + bz],
                                 qt = S.qmm[s][12];
                    float vtl = 0.0f, vth = 0.0f;
                    if (USEVAL) {
                        const float wvs = S.wvf[s];
                        if (wvs > 0.0f) {
                            const float cvs = S.cvf[s];
                            const float pl = vwl - cvs, ph = vwh - cvs;
                            vtl = wvs * ((pl <= 0.f && ph >= 0.f) ? 0.f : fminf(fabsf(pl), fabsf(ph)));
                            vth = wvs * fmaxf(fabsf(pl), fabsf(ph));
                        }
                    }
                    dl[r] = fmaf(fwd, sqrt_approx((qx.x + qy.x) + (qz.x + qt.x)), vtl);
                    ubw = fminf(ubw, fmaf(fwd, sqrt_approx((qx.y + qy.y) + (qz.y + qt.y)), vth));
                }
            }
            ubw = warp_min_f(ubw);
            const float Wb = (USEVAL ? wvf * (fmaxf(fabsf(vwl), fabsf(vwh)) + cvmax) : 0.f) + slack;
            const float thr = (ubw * (1.f + KCULL) + 2.f * KCULL * Wb) * (1.f + 0x1.0p-15f);
            unsigned keep[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                keep[r] = __ballot_sync(0xffffffffu,
                                        dl[r] < INF_F && (dl[r] <= thr || (a.debug & 1)));

            // ---- per-sample fp32 screen with packed (d, slot) keys
            unsigned b1[8], b2[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                b1[k] = 0xFFFFFFFFu;
                b2[k] = 0xFFFFFFFFu;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                unsigned it = keep[r];
                while (it) {
                    const int s = __ffs(it) - 1 + 32 * r;
                    it &= it - 1;
                    const float *T = S.tab[s];
                    const float axy = T[lx] + T[BX + ly];
                    const float a0 = axy + T[OZ + lz0], a1 = axy + T[OZ + lz0 + 2];
                    const float4 tt = *reinterpret_cast<const float4 *>(T + OT);
                    const float ta[4] = {tt.x, tt.y, tt.z, tt.w};
                    float cvs = 0.0f, wvs = 0.0f;
                    if (USEVAL) {
                        cvs = S.cvf[s];
                        wvs = S.wvf[s];
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float sq = (k < 4 ? a0 : a1) + ta[k & 3];
                        const float d = USEVAL ? fmaf(fwd, sqrt_approx(sq), wvs * fabsf(fv[k] - cvs))
                                               : fwd * sqrt_approx(sq);
                        const unsigned key = (__float_as_uint(d) & ~SLOT_MASK) | (unsigned)s;
                        b2[k] = min(b2[k], max(b1[k], key));
                        b1[k] = min(b1[k], key);
                    }
                }
            }
            // ---- certify, or resolve exactly
            unsigned need = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float t1 = __uint_as_float(min(b1[k] & ~SLOT_MASK, INF_BITS));
                const float t2 = __uint_as_float(min(b2[k] & ~SLOT_MASK, INF_BITS));
                const float u1 = t1 * (1.f + 0x1.0p-15f);
                const float W = USEVAL ? fmaf(wvf, fabsf(fv[k]) + cvmax, slack) : slack;
                const bool ok = !(a.debug & 2) && b1[k] < INF_BITS &&
                                t2 * (1.f - KSCR) > u1 * (1.f + KSCR) + 2.f * KSCR * W;
                sl[k] = ok ? (int)(b1[k] & SLOT_MASK) : -1;
                if (!ok && (livem >> k & 1)) need |= 1u << k;
            }
            if (__any_sync(0xffffffffu, need != 0) && need) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!(need >> k & 1)) continue;
                    const int zi = lz0 + 2 * (k >> 2), ti = k & 3;
                    const float W = USEVAL ? fmaf(wvf, fabsf(fv[k]) + cvmax, slack) : slack;
                    const float u1 = __uint_as_float(b1[k] & ~SLOT_MASK) * (1.f + 0x1.0p-15f);
                    const float thrk = b1[k] < INF_BITS
                                           ? (u1 * (1.f + KSCR) + 2.f * KSCR * W) * (1.f + 0x1.0p-17f)
                                           : INF_F;
                    const double px = S.x[lx], py = S.y[ly], pz = S.z[zi];
                    double eD = INF_D;
                    int eI = INT_MAX, eS = -1;
#pragma unroll 1
                    for (int r = 0; r < 4; ++r) {
                        unsigned it = r == 0 ? keep[0] : r == 1 ? keep[1] : r == 2 ? keep[2] : keep[3];
                        while (it) {
                            const int s = __ffs(it) - 1 + 32 * r;
                            it &= it - 1;
                            const float *T = S.tab[s];
                            const float ex = T[lx], ey = T[BX + ly], ez = T[OZ + zi], et = T[OT + ti];
                            if (ex == INF_F || ey == INF_F || ez == INF_F || et == INF_F) continue;
                            const float sq = ((ex + ey) + ez) + et;
                            const float d = USEVAL ? fmaf(fwd, sqrt_approx(sq), S.wvf[s] * fabsf(fv[k] - S.cvf[s]))
                                                   : fwd * sqrt_approx(sq);
                            if (d > thrk) continue;
                            const double dx = DSUB(S.c[s][0], px), dy = DSUB(S.c[s][1], py),
                                         dz = DSUB(S.c[s][2], pz);
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
                    }
                    sl[k] = eS;
                }
            }
        }

        // ---- labels; deferred / stranded samples to their lists (warp-aggregated)
        int nlist = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (!(livem >> k & 1)) continue;
            const long long f = fbase + 2 * (k >> 2) * plane + (k & 3) * vol;
            const int lab = deferred ? -2 : (sl[k] >= 0 ? S.id[sl[k]] : -1);
            a.labels[f] = lab;
            if (lab < 0) ++nlist;
        }
        if (__any_sync(0xffffffffu, nlist > 0)) {
            unsigned long long *ctr = deferred ? a.n_deferred : a.n_stranded;
            long long *lst = deferred ? a.deferred : a.stranded;
            const long long cap = deferred ? a.deferred_cap : a.stranded_cap;
            long long p = warp_reserve(ctr, nlist);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (!(livem >> k & 1)) continue;
                if (!deferred && sl[k] >= 0) continue;
                if (p < cap) lst[p] = fbase + 2 * (k >> 2) * plane + (k & 3) * vol;
                ++p;
            }
        }

        // ---- partial sums: count marginals (shared atomics) + per-warp value sums
        if (a.accumulate && !deferred && cnt > 0) {
            unsigned todo = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (sl[k] >= 0 && (livem >> k & 1)) todo |= 1u << k;
            const unsigned MX = 0x11111111u << (lane & 3);
            const unsigned MY = 0x000F000Fu << (4 * ((lane >> 2) & 3));
            while (true) {
                int mine = -1;
#pragma unroll
                for (int k = 7; k >= 0; --k)
                    if (todo >> k & 1) mine = sl[k];
                const unsigned act = __ballot_sync(0xffffffffu, mine >= 0);
                if (!act) break;
                const int L = __shfl_sync(0xffffffffu, mine, __ffs(act) - 1);
                unsigned c = 0, czp = 0, ctp = 0;   // count; z pair (16|16); t counts (8 bits each)
                double vs = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if ((todo >> k & 1) && sl[k] == L) {
                        todo &= ~(1u << k);
                        ++c;
                        czp += (k < 4) ? 1u : 0x10000u;
                        ctp += 1u << (8 * (k & 3));
                        vs = DADD(vs, v[k]);
                    }
                }
                const unsigned sx = __reduce_add_sync(MX, c);
                const unsigned sy = __reduce_add_sync(MY, c);
                const unsigned sz = __reduce_add_sync(lane < 16 ? 0x0000FFFFu : 0xFFFF0000u, czp);
                const unsigned st = __reduce_add_sync(0xffffffffu, ctp);
                vs = warp_sum_d(vs);
                unsigned *h = S.hist[L];
                if (lane < 4) {
                    const int i = 4 * bx + lane;
                    if (sx) atomicAdd(&h[i >> 1], sx << (16 * (i & 1)));
                }
                if (lane < 16 && (lane & 3) == 0) {
                    const int i = 4 * by + (lane >> 2);
                    if (sy) atomicAdd(&h[8 + (i >> 1)], sy << (16 * (i & 1)));
                }
                if (lane == 0 || lane == 16) {   // z = lz0 (low half) and lz0 + 2 (high half)
                    const int i0 = lz0, i1 = lz0 + 2;
                    if (sz & 0xFFFFu) atomicAdd(&h[16 + (i0 >> 1)], (sz & 0xFFFFu) << (16 * (i0 & 1)));
                    if (sz >> 16) atomicAdd(&h[16 + (i1 >> 1)], (sz >> 16) << (16 * (i1 & 1)));
                }
                if (lane == 0) {
                    const unsigned t0 = st & 0xFFu, t1 = (st >> 8) & 0xFFu, t2 = (st >> 16) & 0xFFu,
                                   t3 = st >> 24;
                    atomicAdd(&h[24], t0 | (t1 << 16));
                    atomicAdd(&h[25], t2 | (t3 << 16));
                    atomicAdd(&h[26], t0 + t1 + t2 + t3);
                    S.wsum[w][L] = DADD(S.wsum[w][L], vs);
                }
            }
        }
    }

    // ---- once per block: marginals x fixed-point coordinates -> global 128-bit sums
    if (a.accumulate && !deferred && cnt > 0) {
        __syncthreads();
        for (int e = tid; e < cnt * 6; e += NT) {
            const int s = e / 6, wd = e - s * 6;
            const unsigned *h = S.hist[s];
            const int n = (int)h[26];
            if (n == 0) continue;
            unsigned long long *dst = a.acc + (size_t)S.id[s] * MFSEG_ACC_WORDS;
            __int128 acc = 0;
            if (wd == 0) {
#pragma unroll
                for (int i = 0; i < BX; ++i) acc += get128(S.xf[i]) * (__int128)hget(h, i);
            } else if (wd == 1) {
#pragma unroll
                for (int i = 0; i < BY; ++i) acc += get128(S.yf[i]) * (__int128)hget(h + 8, i);
            } else if (wd == 2) {
#pragma unroll
                for (int i = 0; i < BZ; ++i) acc += get128(S.zf[i]) * (__int128)hget(h + 16, i);
            } else if (wd == 3) {
#pragma unroll
                for (int i = 0; i < BT; ++i) acc += get128(S.tf[i]) * (__int128)hget(h + 24, i);
            } else if (wd == 4) {
#pragma unroll
                for (int q = 0; q < NW; ++q) {
                    unsigned long long lo;
                    long long hi;
                    d2fix(S.wsum[q][s], lo, hi, &ovf_local);
                    acc += (__int128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
                }
            } else {
                atomicAdd(dst + 13, (unsigned long long)n);
                continue;
            }
            atomic_add_fix(dst + (wd < 4 ? 2 * wd : 10), (unsigned long long)acc, (long long)(acc >> 64));
        }
    }
    if (ovf_local) *a.overflow = 1;
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
        MFSEG_CUDA(cudaFuncSetAttribute(k_field_assign5<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MFSEG_CUDA(cudaFuncSetAttribute(k_field_assign5<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = true;
    }
    ::mfseg::count_launch();
    if (a.wv > 0.0)
        k_field_assign5<true><<<(unsigned)n, NT, smem, st>>>(a);
    else
        k_field_assign5<false><<<(unsigned)n, NT, smem, st>>>(a);
    MFSEG_LAUNCH("k_field_assign5");
    return 0;
}

}  // namespace mfseg
