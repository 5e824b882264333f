// Internal helpers shared by the sm_100a segmentation kernels.
//
// Exactness rules (labels must equal the reference bit for bit):
//   * every fp64 operation is an explicit IEEE round-to-nearest intrinsic
//     (__dadd_rn / __dmul_rn / ...) in the reference's operation order, and
//     the library is compiled with -fmad=false so nothing is contracted to FMA;
//   * sample coordinates are re-derived from indices with the reference's own
//     two roundings: x = origin + (i + 0.5) * spacing  (model.py:137-142).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/mfseg_sm100.h"

namespace mfseg {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
int fail(const char *where, cudaError_t e);

#define MFSEG_CUDA(call)                                              \
    do {                                                              \
        cudaError_t e__ = (call);                                     \
        if (e__ != cudaSuccess) return ::mfseg::fail(#call, e__);     \
    } while (0)

#define MFSEG_LAUNCH(where)                                           \
    do {                                                              \
        cudaError_t e__ = cudaGetLastError();                         \
        if (e__ != cudaSuccess) return ::mfseg::fail(where, e__);     \
    } while (0)

#define MFSEG_TRY(call)                  \
    do {                                 \
        int r__ = (call);                \
        if (r__ != 0) return r__;        \
    } while (0)

// ------------------------------------------------------------------ instrumentation
// every kernel launch site calls count_launch(); bench.py reads the counter
// around its timed region (mfseg_launch_count) to report gpu_launches.
void count_launch();

// ------------------------------------------------------------------ workspace carving
struct Carver {
    char *base;
    size_t off, cap;
    explicit Carver(void *b = nullptr, size_t c = 0) : base((char *)b), off(0), cap(c) {}
    // every carving is 256-byte aligned in absolute address (the caller's
    // workspace pointer need not be aligned: the size queries include 256 B of slack)
    template <class T>
    T *take(size_t n) {
        const size_t b = (size_t)(uintptr_t)base;
        size_t a = ((b + off + 255) & ~size_t(255)) - b;
        off = a + sizeof(T) * (n > 0 ? n : 1);
        return base ? (T *)(base + a) : nullptr;
    }
    bool ok() const { return base == nullptr || off <= cap; }
};

// ------------------------------------------------------------------ exact fp64
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DSQRT(a) __dsqrt_rn(a)

// cell centre along one axis: origin + (i + 0.5) * spacing   (model.py:137-142)
__host__ __device__ __forceinline__ double cell_coord(double origin, double spacing, long long i) {
#ifdef __CUDA_ARCH__
    return DADD(origin, DMUL((double)i + 0.5, spacing));
#else
    volatile double p = ((double)i + 0.5) * spacing;
    return origin + p;
#endif
}

// clip(floor((x - min) / C), 0, k-1)   (engine.py:111-113)
__host__ __device__ __forceinline__ int bin_coord(double x, double mn, double C, int k) {
#ifdef __CUDA_ARCH__
    double q = floor(DDIV(DSUB(x, mn), C));
#else
    volatile double dq = x - mn;
    double q = floor(dq / C);
#endif
    if (!(q >= 0.0)) return 0;            // also NaN-safe
    if (q >= (double)(k - 1)) return k - 1;
    return (int)q;
}

// D = vterm + wd * sqrt(((dx^2 + dy^2) + dz^2) + (cf*dt)^2)   (engine.py:137-149)
// vterm = wv * |v - cval| when the centre has this kind's value, else 0.
__device__ __forceinline__ double metric_tail(double q_xyz, double tsq, double v, double cval,
                                              bool chas, double wv, double wd) {
    double sst = DSQRT(DADD(q_xyz, tsq));
    double vt = (wv > 0.0 && chas) ? DMUL(wv, fabs(DSUB(v, cval))) : 0.0;
    return DADD(vt, DMUL(wd, sst));
}

__device__ __forceinline__ bool better(double D, int id, double bD, int bid) {
    return D < bD || (D == bD && id < bid);
}

// ------------------------------------------------------------------ 128-bit fixed point
// value * 2^64 as a signed 128-bit integer (lo, hi); |value| < 2^62 required.
// Rounds toward zero below 2^-64 (irrelevant at fp64 resolution of the sums).
__device__ __forceinline__ void d2fix(double x, unsigned long long &lo, long long &hi,
                                      int *overflow) {
    unsigned long long bits = (unsigned long long)__double_as_longlong(x);
    int e = (int)((bits >> 52) & 0x7ff);
    unsigned long long m = bits & ((1ull << 52) - 1);
    if (e == 0x7ff) {
        if (overflow) *overflow = 1;
        lo = 0;
        hi = 0;
        return;
    }
    if (e == 0) e = 1; else m |= (1ull << 52);
    const int sh = e - 1011;   // m * 2^(e-1075) * 2^64
    unsigned long long ul, uh;  // |x| * 2^64 (64-bit shifts: no 128-bit shift sequences)
    if (sh > 73) {
        if (overflow) *overflow = 1;
        ul = uh = 0;
    } else if (sh >= 64) {
        ul = 0;
        uh = m << (sh - 64);
    } else if (sh > 0) {
        ul = m << sh;
        uh = m >> (64 - sh);
    } else if (sh > -64) {
        ul = m >> (-sh);
        uh = 0;
    } else {
        ul = uh = 0;
    }
    if (bits >> 63) {   // two's complement negation of (uh, ul)
        lo = 0ull - ul;
        hi = (long long)(~uh + (ul == 0 ? 1ull : 0ull));
    } else {
        lo = ul;
        hi = (long long)uh;
    }
}

// correctly rounded (nearest-even) double of the 128-bit fixed value * 2^-64
__device__ __forceinline__ double fix2d(unsigned long long lo, long long hi) {
    __int128 s = (((__int128)hi) << 64) | (__int128)lo;
    if (s == 0) return 0.0;
    bool neg = s < 0;
    unsigned __int128 u = neg ? (unsigned __int128)(-s) : (unsigned __int128)s;
    unsigned long long uh = (unsigned long long)(u >> 64), ul = (unsigned long long)u;
    int msb = uh ? 127 - __clzll((long long)uh) : 63 - __clzll((long long)ul);
    double r;
    if (msb <= 52) {
        r = (double)ul;   // exact
        r = ldexp(r, -64);
    } else {
        int drop = msb - 52;
        unsigned __int128 mant = u >> drop;
        unsigned __int128 rem = u - (mant << drop);
        unsigned __int128 half = ((unsigned __int128)1) << (drop - 1);
        if (rem > half || (rem == half && (mant & 1))) mant += 1;
        r = ldexp((double)(unsigned long long)mant, drop - 64);
    }
    return neg ? -r : r;
}

__device__ __forceinline__ void atomic_add_fix(unsigned long long *p, unsigned long long lo,
                                               long long hi) {
    unsigned long long old = atomicAdd(p, lo);
    unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
    unsigned long long h = (unsigned long long)hi + carry;
    if (h) atomicAdd(p + 1, h);
}

__device__ __forceinline__ void atomic_add_double_fix(unsigned long long *p, double x, int *ovf) {
    unsigned long long lo;
    long long hi;
    d2fix(x, lo, hi, ovf);
    atomic_add_fix(p, lo, hi);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = DADD(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------------ device views
struct CentersView {      // read-only centre state for the assign kernels
    const double *x, *y, *z, *t, *pval, *fval;
    const uint8_t *has_p, *has_f;
};

struct Grid {             // CenterGrid (engine.py:89-134), rebuilt every pass
    int K;                // centres
    int NB;               // bins = k1*k2*k3*k4
    int *cbin;            // [K] flat bin of every centre
    int *bin_start;       // [K+1] CSR of centres by bin
    int *bin_ids;         // [K]
    int *cand_start;      // [K+1] per sample bin: centres in the 3^4 neighbour bins
    int *cand_ids;        // [<= 81 K]
    int4 *vbox;           // [K][2]: (ilo, ihi, jlo, jhi), (klo, khi, mlo, mhi) box test per field axis
};

struct AxisTile {         // field tile along one axis: index range inside one sample bin
    int start, len, bin, pad;
};

// 256 bytes of device scratch (plus a pinned host mirror) per host thread and
// device, allocated once: the small flag / min-max buffers of the synchronous
// ABI calls.  (cudaMallocAsync/cudaFreeAsync on the default pool took up to a
// second per call next to the caching allocator's multi-GB blocks.)
int tiny_scratch(void **dev, void **host);

// host-side internal entry points shared between translation units
int scan_exclusive_i32(const int *in, int *out, long long n, void *tmp, size_t tmp_bytes,
                       cudaStream_t st);
int scan_exclusive_i64(const long long *in, long long *out, long long n, void *tmp,
                       size_t tmp_bytes, cudaStream_t st);
size_t scan_tmp_bytes(long long n);
size_t radix_tmp_bytes(long long n);
int radix_sort_pairs(const unsigned *keys_in, const unsigned *vals_in, unsigned *keys_out,
                     unsigned *vals_out, long long n, int key_bits, void *tmp, size_t tmp_bytes,
                     cudaStream_t st);
int radix_sort_pairs64(const unsigned long long *keys_in, const unsigned *vals_in,
                       unsigned long long *keys_out, unsigned *vals_out, long long n,
                       int key_bits, void *tmp, size_t tmp_bytes, cudaStream_t st);

}  // namespace mfseg
