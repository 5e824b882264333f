// k_field_screen — per-sample resolution of the field bricks that
// k_field_assign5 left with several candidates (cell boundaries and value
// edges run through them).  One warp per brick, candidates by global id.
//
// Every number here is computed exactly as in k_field_assign5: the fp32
// per-axis entries fl32((c - s)^2) (fp64 difference and square, one rounding,
// +inf outside the validity window), d32 = fwd sqrt(((Tx + Ty) + Tz) + Tt)
// + w_v |fl(v) - fl(cv)|, packed (d | candidate) keys, the certification
// t2 (1-K) > u1 (1+K) + 2 K W and the exact fp64 re-evaluation within the
// margin (error analysis: assign_field5.cu header).  W uses the largest |cv|
// among the kept candidates, the only ones compared.
//
// Partial sums: per (brick, cluster) record, x / y / z / t sums as count
// marginals x 128-bit fixed-point coordinates (exact), reduced over the warp
// in 128-bit integer arithmetic; the value sum as the fixed-order fp64 warp sum
// converted exactly; one 128-bit integer atomic per word.  Integer sums are
// order-free, so the result does not depend on which warp takes which brick.
#include <climits>

#include "kernels.cuh"

namespace mfseg {
namespace {

constexpr double INF_D = __builtin_huge_val();
constexpr float INF_F = __builtin_huge_valf();
constexpr float FLT_BIG = 3.4028234663852886e38f;
constexpr unsigned INF_BITS = 0x7F800000u;
constexpr unsigned KEY_MASK = 127u;   // same key truncation as k_field_assign5
constexpr float KSCR = 0x1.0p-18f;
constexpr int ACC_FV = 10, ACC_NF = 13;   // accumulator words (assign.cu)
#ifndef MFSEG_SCREEN_MINB
#define MFSEG_SCREEN_MINB 4
#endif
constexpr int SCREEN_MINB = MFSEG_SCREEN_MINB;

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float to_f(double x) { return fminf(__double2float_rn(x), FLT_BIG); }

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

struct ScreenCand {            // one warp's kept candidates, staged in shared memory
    double c[4][MULTI_MAX];
    double cv[MULTI_MAX];
    int4 b0[MULTI_MAX], b1[MULTI_MAX];
    float cvf[MULTI_MAX], wvf[MULTI_MAX];
    int id[MULTI_MAX], has[MULTI_MAX];
    double v[8][32];          // the brick's samples (k, lane)
    double pz[4], pt[2];      // its z-plane and timestep coordinates
    float tab[MULTI_MAX][18]; // per candidate: the brick's fp32 table entries x[8] y[4] z[4] t[2]
};

template <bool USEVAL>
__global__ void __launch_bounds__(256, SCREEN_MINB) k_field_screen(FieldArgs a) {
    __shared__ ScreenCand SC[8];
    const int lane = threadIdx.x & 31;
    ScreenCand &Q = SC[threadIdx.x >> 5];
    const long long n_items = min((long long)*a.n_multi, a.multi_cap);
    const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
    int ovf_local = 0;
    const long long plane = (long long)a.ny * a.nx, vol = plane * a.nz;
    const float fwd = (float)a.wd;
    const float wvf = USEVAL ? (float)a.wv : 0.0f;
    const float slack = 3e-13f * (float)(a.wd + a.wv);
    for (long long item = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; item < n_items;
         item += nwarps) {
        const MultiItem &it = a.multi[item];
        const int meta = it.meta, nk = meta & 0xFF;
        const int ex = (meta >> 8) & 15, ey = (meta >> 12) & 15, ez = (meta >> 16) & 15,
                  et = (meta >> 20) & 15;
        const int lxr = lane & 7, lyr = lane >> 3;
        const int gx = it.x0 + lxr, gy = it.y0 + lyr, gz0 = it.z0, gt0 = it.t0;
        const long long fbase = (((long long)gt0 * a.nz + gz0) * a.ny + gy) * (long long)a.nx + gx;
        unsigned livem = 0;
        if (lxr < ex && lyr < ey) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if ((k & 3) < ez && (k >> 2) < et) livem |= 1u << k;
        }
        // samples to shared memory (dead samples: 0, their keys are never used);
        // fp32 copies stay in registers for the screen
        __syncwarp();
        float fv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double vk = (livem >> k & 1) ? __ldg(a.values + fbase + (k & 3) * plane + (k >> 2) * vol) : 0.0;
            Q.v[k][lane] = vk;
            fv[k] = (float)vk;
        }
        // sample coordinates (reference formula); index clamped for dead lanes
        const double px = cell_coord(a.ox, a.sx, a.x0 + it.x0 + min(lxr, ex - 1));
        const double py = cell_coord(a.oy, a.sy, a.y0 + it.y0 + min(lyr, ey - 1));
        if (lane < 4)
            Q.pz[lane] = a.swap_zt ? a.times[gz0 + min(lane, ez - 1)]
                                   : cell_coord(a.oz, a.sz, a.z0 + gz0 + min(lane, ez - 1));
        else if (lane < 6)
            Q.pt[lane - 4] = a.swap_zt ? cell_coord(a.oz, a.sz, a.z0 + gt0 + min(lane - 4, et - 1))
                                       : a.times[gt0 + min(lane - 4, et - 1)];
        const double *pz = Q.pz, *pt = Q.pt;
        // stage the kept candidates; largest |cv| among them (certification's W)
        float cvmax = 0.f;
        __syncwarp();
        if (lane < nk) {
            const int id = it.id[lane];
            const bool has = a.chas[id] != 0;
            const double cv = has ? a.cval[id] : 0.0;
            Q.id[lane] = id;
            Q.has[lane] = has;
            Q.cv[lane] = cv;
            Q.cvf[lane] = (float)cv;
            Q.wvf[lane] = (USEVAL && has) ? (float)a.wv : 0.f;
            Q.c[0][lane] = a.c.x[id];
            Q.c[1][lane] = a.c.y[id];
            Q.c[2][lane] = a.c.z[id];
            Q.c[3][lane] = a.c.t[id];
            Q.b0[lane] = a.g.vbox[2 * id];
            const int4 br = a.g.vbox[2 * id + 1];
            Q.b1[lane] = a.swap_zt ? make_int4(br.z, br.w, br.x, br.y) : br;   // kernel (z, t) ranges
            if (USEVAL && has) cvmax = fabsf((float)cv);
        }
        __syncwarp();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cvmax = fmaxf(cvmax, __shfl_xor_sync(0xffffffffu, cvmax, o));
        // the candidates' table entries over the brick (as the block tables: an fp64
        // difference and square rounded once, +inf outside the validity box; c_f on
        // the time axis), computed once per item by the warp instead of per lane
        for (int e = lane; e < nk * 18; e += 32) {
            const int j = e / 18, q = e - 18 * j;
            const int4 b0 = Q.b0[j], bb = Q.b1[j];
            float val = INF_F;
            if (q < 8) {
                if (it.x0 + q >= b0.x && it.x0 + q <= b0.y) {
                    const double d = DSUB(Q.c[0][j], cell_coord(a.ox, a.sx, a.x0 + it.x0 + min(q, ex - 1)));
                    val = to_f(DMUL(d, d));
                }
            } else if (q < 12) {
                const int r = q - 8;
                if (it.y0 + r >= b0.z && it.y0 + r <= b0.w) {
                    const double d = DSUB(Q.c[1][j], cell_coord(a.oy, a.sy, a.y0 + it.y0 + min(r, ey - 1)));
                    val = to_f(DMUL(d, d));
                }
            } else if (q < 16) {
                const int r = q - 12;
                if (gz0 + r >= bb.x && gz0 + r <= bb.y) {
                    double d = DSUB(Q.c[2][j], Q.pz[r]);
                    if (a.swap_zt) d = DMUL(a.cf, d);   // the kernel's z axis is time
                    val = to_f(DMUL(d, d));
                }
            } else {
                const int r = q - 16;
                if (gt0 + r >= bb.z && gt0 + r <= bb.w) {
                    double d = DSUB(Q.c[3][j], Q.pt[r]);
                    if (!a.swap_zt) d = DMUL(a.cf, d);
                    val = to_f(DMUL(d, d));
                }
            }
            Q.tab[j][q] = val;
        }
        __syncwarp();

        // ---- screen over the kept candidates
        unsigned b1[8], b2[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            b1[k] = 0xFFFFFFFFu;
            b2[k] = 0xFFFFFFFFu;
        }
#pragma unroll 1
        for (int j = 0; j < nk; ++j) {
            const float *tb = Q.tab[j];
            const float tx = tb[lxr], ty = tb[8 + lyr];
            const float tz[4] = {tb[12], tb[13], tb[14], tb[15]}, tt[2] = {tb[16], tb[17]};
            const float cvs = USEVAL ? Q.cvf[j] : 0.f, wvs = USEVAL ? Q.wvf[j] : 0.f;
            const float axy = tx + ty;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float sq = (axy + tz[k & 3]) + tt[k >> 2];
                const float d = USEVAL ? fmaf(fwd, sqrt_approx(sq), wvs * fabsf(fv[k] - cvs))
                                       : fwd * sqrt_approx(sq);
                const unsigned key = (__float_as_uint(d) & ~KEY_MASK) | (unsigned)j;
                b2[k] = min(b2[k], max(b1[k], key));
                b1[k] = min(b1[k], key);
            }
        }
        // ---- certify, or resolve exactly
        int sl[8];
        unsigned need = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float t1 = __uint_as_float(min(b1[k] & ~KEY_MASK, INF_BITS));
            const float t2 = __uint_as_float(min(b2[k] & ~KEY_MASK, INF_BITS));
            const float u1 = t1 * (1.f + 0x1.0p-15f);
            const float W = USEVAL ? fmaf(wvf, fabsf(fv[k]) + cvmax, slack) : slack;
            const bool ok = !(a.debug & 2) && b1[k] < INF_BITS &&
                            t2 * (1.f - KSCR) > u1 * (1.f + KSCR) + 2.f * KSCR * W;
            sl[k] = ok ? (int)(b1[k] & KEY_MASK) : -1;
            if (!ok && (livem >> k & 1)) need |= 1u << k;
        }
        if (DEVICE_STATS(a) && a.stats) {   // counters[33]: items, [34]: exact samples
            if (lane == 0) atomicAdd(a.stats + 25, 1ull);
            if (need) atomicAdd(a.stats + 26, (unsigned long long)__popc(need));
        }
        if (need) {
#pragma unroll 1
            for (int k = 0; k < 8; ++k) {
                if (!(need >> k & 1)) continue;
                const double vk = Q.v[k][lane], pzk = pz[k & 3], ptk = pt[k >> 2];
                unsigned b1k = b1[0];
#pragma unroll
                for (int q = 1; q < 8; ++q)
                    if (q == k) {
                        b1k = b1[q];
                    }
                const float fvk = (float)vk;
                const float W = USEVAL ? fmaf(wvf, fabsf(fvk) + cvmax, slack) : slack;
                const float u1 = __uint_as_float(b1k & ~KEY_MASK) * (1.f + 0x1.0p-15f);
                const float thrk = b1k < INF_BITS
                                       ? (u1 * (1.f + KSCR) + 2.f * KSCR * W) * (1.f + 0x1.0p-17f)
                                       : INF_F;
                const int gz = gz0 + (k & 3), gt = gt0 + (k >> 2);
                double eD = INF_D;
                int eI = INT_MAX, eJ = -1;
                for (int j = 0; j < nk; ++j) {
                    const int id = Q.id[j];
                    const int4 b0 = Q.b0[j], bb = Q.b1[j];
                    if (!(gx >= b0.x && gx <= b0.y && gy >= b0.z && gy <= b0.w && gz >= bb.x &&
                          gz <= bb.y && gt >= bb.z && gt <= bb.w))
                        continue;
                    const double cx = Q.c[0][j], cy = Q.c[1][j], cz = Q.c[2][j], ct = Q.c[3][j];
                    // (real z and t differences: the kernel's z axis is time when swapped)
                    const double dkz = DSUB(cz, pzk), dkt = DSUB(ct, ptk);
                    const double dx = DSUB(cx, px), dy = DSUB(cy, py), dz = a.swap_zt ? dkt : dkz;
                    const double dt = DMUL(a.cf, a.swap_zt ? dkz : dkt);
                    // fp32 screen value of this pair (prune outside the margin)
                    const float sq = ((to_f(DMUL(dx, dx)) + to_f(DMUL(dy, dy))) + to_f(DMUL(dz, dz))) +
                                     to_f(DMUL(dt, dt));
                    const bool has = Q.has[j] != 0;
                    const float cvs = Q.cvf[j];
                    const float wvs = USEVAL ? Q.wvf[j] : 0.f;
                    const float d = USEVAL ? fmaf(fwd, sqrt_approx(sq), wvs * fabsf(fvk - cvs))
                                           : fwd * sqrt_approx(sq);
                    if (d > thrk) continue;
                    const double qq = DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz));
                    const double D = metric_tail(qq, DMUL(dt, dt), vk, Q.cv[j], has,
                                                 a.wv, a.wd);
                    if (better(D, id, eD, eI)) {
                        eD = D;
                        eI = id;
                        eJ = j;
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q == k) sl[q] = eJ;
            }
        }

        // ---- labels; stranded samples (no kept candidate valid) to the fallback list
        int nout = 0;
        int *lab_base = a.labels + fbase;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (!(livem >> k & 1)) continue;
            const int lab = sl[k] >= 0 ? Q.id[sl[k]] : -1;
            lab_base[(k & 3) * plane + (k >> 2) * vol] = lab;
            if (lab < 0) ++nout;
        }
        if (__any_sync(0xffffffffu, nout > 0)) {
            long long p = warp_reserve(a.n_stranded, nout);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (!(livem >> k & 1) || sl[k] >= 0) continue;
                if (p < a.stranded_cap) a.stranded[p] = fbase + (k & 3) * plane + (k >> 2) * vol;
                ++p;
            }
        }

        // ---- partial sums: one record per cluster present in the brick.  Group
        // lanes hold one fixed-point coordinate each: x columns on lanes 0-7, y rows
        // on 8-11, z planes on 16-19, timesteps on 24-25 (others 0); per record the
        // count-weighted products are summed inside each 8-lane group.
        if (a.accumulate) {
            const int grp = lane >> 3, gi = lane & 7;
            double gc = 0.0;
            {
                const double pyr = __shfl_sync(0xffffffffu, py, (gi & 3) << 3);
                const double pzq = pz[gi & 3];
                gc = grp == 0 ? px : grp == 1 ? pyr : grp == 2 ? pzq : (gi & 1) ? pt[1] : pt[0];
            }
            const bool gl = grp == 0 || gi < (grp == 3 ? 2 : 4);
            unsigned long long flo = 0;
            long long fhi = 0;
            if (gl) d2fix(gc, flo, fhi, &ovf_local);
            unsigned todo = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (sl[k] >= 0 && (livem >> k & 1)) todo |= 1u << k;
            while (true) {
                int mine = -1;
#pragma unroll
                for (int k = 7; k >= 0; --k)
                    if (todo >> k & 1) mine = sl[k];
                const unsigned act = __ballot_sync(0xffffffffu, mine >= 0);
                if (!act) break;
                const int L = __shfl_sync(0xffffffffu, mine, __ffs(act) - 1);
                unsigned c = 0, zp = 0, tp = 0;
                double vs = 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if ((todo >> k & 1) && sl[k] == L) {
                        todo &= ~(1u << k);
                        ++c;
                        zp += 1u << (8 * (k & 3));
                        tp += 1u << (16 * (k >> 2));
                        vs = DADD(vs, Q.v[k][lane]);
                    }
                }
                unsigned sx = c + __shfl_xor_sync(0xffffffffu, c, 8);   // column sums
                sx += __shfl_xor_sync(0xffffffffu, sx, 16);
                unsigned sy = c + __shfl_xor_sync(0xffffffffu, c, 1);    // row sums
                sy += __shfl_xor_sync(0xffffffffu, sy, 2);
                sy += __shfl_xor_sync(0xffffffffu, sy, 4);
                const unsigned sz = __reduce_add_sync(0xffffffffu, zp);
                const unsigned st = __reduce_add_sync(0xffffffffu, tp);
                vs = warp_sum_d(vs);
                const unsigned syr = __shfl_sync(0xffffffffu, sy, (gi & 3) << 3);
                unsigned cnt = grp == 0 ? sx : grp == 1 ? syr
                             : grp == 2 ? (sz >> (8 * (gi & 3))) & 0xFFu
                                        : (st >> (16 * (gi & 1))) & 0xFFFFu;
                if (!gl) cnt = 0;
                // 128-bit (flo, fhi) * cnt, then the sum over the 8 lanes of the group
                unsigned long long lo = flo * cnt;
                long long hi = fhi * (long long)cnt + (long long)__umul64hi(flo, cnt);
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
                    const long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
                    const unsigned long long n = lo + l2;
                    hi = hi + h2 + (n < lo ? 1 : 0);
                    lo = n;
                }
                unsigned long long *dst = a.acc + (size_t)Q.id[L] * MFSEG_ACC_WORDS;
                if (lane == 1) d2fix(vs, lo, hi, &ovf_local);
                const int word = lane == 1 ? ACC_FV : 2 * (a.swap_zt && grp >= 2 ? 5 - grp : grp);   // real axis
                if (gi == 0 || lane == 1) atomic_add_fix(dst + word, lo, hi);
                if (lane == 2) atomicAdd(dst + ACC_NF, (unsigned long long)((st & 0xFFFFu) + (st >> 16)));
            }
        }
    }
    if (ovf_local) *a.overflow = 1;
}

int launch_field_screen(const FieldArgs &a, cudaStream_t st) {
    if (!a.multi) return 0;
    ::mfseg::count_launch();
#ifndef MFSEG_SCREEN_CTAS
#define MFSEG_SCREEN_CTAS (148 * 32)   // 8 waves of the 4 resident CTAs per SM: even tails
#endif
    if (a.wv > 0.0)
        k_field_screen<true><<<MFSEG_SCREEN_CTAS, 256, 0, st>>>(a);
    else
        k_field_screen<false><<<MFSEG_SCREEN_CTAS, 256, 0, st>>>(a);
    MFSEG_LAUNCH("k_field_screen");
    return 0;
}

}  // namespace mfseg
