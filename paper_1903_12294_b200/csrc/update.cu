// update_centers + has_converged + max_center_delta (engine.py:266-320), and
// the conversions of the exact 128-bit accumulators.
#include <cstring>

#include "kernels.cuh"

namespace mfseg {

namespace {

constexpr double DELTA = 1e-12;   // model.py:16

__device__ __forceinline__ double rel_change(double o, double n) {
    return DDIV(fabs(DSUB(n, o)), DADD(fabs(o), DELTA));
}

struct Flags {              // reduced on the device, read back once per pass
    int any_active;
    int not_converged;
    unsigned long long delta_bits;   // max of non-negative doubles, as bits
};

__global__ void k_update(int K, const unsigned long long *acc, mfseg_centers o, mfseg_centers n,
                         double eps_c, Flags *fl) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    int active = 0, notconv = 0;
    double dmax = 0.0;
    bool have_delta = false;
    if (c < K) {
        const unsigned long long *a = acc + (size_t)c * MFSEG_ACC_WORDS;
        long long np = (long long)a[12], nf = (long long)a[13];
        long long tot = np + nf;
        double ox = o.loc[c], oy = o.loc[K + c], oz = o.loc[2 * K + c], ot = o.loc[3 * K + c];
        bool ohp = o.has_p[c], ohf = o.has_f[c];
        double opv = o.pval[c], ofv = o.fval[c];
        double nl[4];
        bool nhp, nhf;
        double npv, nfv;
        if (tot > 0) {
            double dt = (double)tot;
            for (int d = 0; d < 4; ++d)
                nl[d] = DDIV(fix2d(a[2 * d], (long long)a[2 * d + 1]), dt);
            nhp = np > 0;
            nhf = nf > 0;
            npv = nhp ? DDIV(fix2d(a[8], (long long)a[9]), (double)np) : __longlong_as_double(0x7ff8000000000000ll);
            nfv = nhf ? DDIV(fix2d(a[10], (long long)a[11]), (double)nf) : __longlong_as_double(0x7ff8000000000000ll);
        } else {   // empty: freeze location, values and has-flags; go dormant
            nl[0] = ox;
            nl[1] = oy;
            nl[2] = oz;
            nl[3] = ot;
            nhp = ohp;
            nhf = ohf;
            npv = opv;
            nfv = ofv;
        }
        n.loc[c] = nl[0];
        n.loc[K + c] = nl[1];
        n.loc[2 * K + c] = nl[2];
        n.loc[3 * K + c] = nl[3];
        n.pval[c] = npv;
        n.fval[c] = nfv;
        n.has_p[c] = nhp;
        n.has_f[c] = nhf;
        n.dormant[c] = tot == 0;
        n.n_points[c] = np;
        n.n_fields[c] = nf;
        if (tot > 0) {   // active (non-dormant) centre
            active = 1;
            double ol[4] = {ox, oy, oz, ot};
            for (int d = 0; d < 4; ++d) {
                double r = rel_change(ol[d], nl[d]);
                if (r >= eps_c) notconv = 1;
                dmax = have_delta ? fmax(dmax, r) : r;
                have_delta = true;
            }
            if (ohp != nhp || ohf != nhf) notconv = 1;
            if (ohp && nhp) {
                double r = rel_change(opv, npv);
                if (r >= eps_c) notconv = 1;
                dmax = fmax(dmax, r);
            }
            if (ohf && nhf) {
                double r = rel_change(ofv, nfv);
                if (r >= eps_c) notconv = 1;
                dmax = fmax(dmax, r);
            }
        }
    }
    // block reduce then one atomic per block
    __shared__ int s_a[32], s_n[32];
    __shared__ double s_d[32];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int off = 16; off > 0; off >>= 1) {
        active |= __shfl_xor_sync(0xffffffffu, active, off);
        notconv |= __shfl_xor_sync(0xffffffffu, notconv, off);
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    }
    if (lane == 0) {
        s_a[w] = active;
        s_n[w] = notconv;
        s_d[w] = dmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            active |= s_a[i];
            notconv |= s_n[i];
            dmax = fmax(dmax, s_d[i]);
        }
        if (active) atomicOr(&fl->any_active, 1);
        if (notconv) atomicOr(&fl->not_converged, 1);
        atomicMax(&fl->delta_bits, (unsigned long long)__double_as_longlong(dmax));
    }
}

// update_centers from fp64 sums (the reference's own signature, engine.py:266-286)
__global__ void k_update_f64(int K, const double *sums, const double *psum, const double *fsum,
                             const long long *n_p, const long long *n_f, mfseg_centers o,
                             mfseg_centers n) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    long long np = n_p[c], nf = n_f[c], tot = np + nf;
    double nan = __longlong_as_double(0x7ff8000000000000ll);
    if (tot > 0) {
        for (int d = 0; d < 4; ++d) n.loc[(size_t)d * K + c] = DDIV(sums[4 * c + d], (double)tot);
        n.has_p[c] = np > 0;
        n.has_f[c] = nf > 0;
        n.pval[c] = np > 0 ? DDIV(psum[c], (double)np) : nan;
        n.fval[c] = nf > 0 ? DDIV(fsum[c], (double)nf) : nan;
    } else {
        for (int d = 0; d < 4; ++d) n.loc[(size_t)d * K + c] = o.loc[(size_t)d * K + c];
        n.has_p[c] = o.has_p[c];
        n.has_f[c] = o.has_f[c];
        n.pval[c] = o.pval[c];
        n.fval[c] = o.fval[c];
    }
    n.dormant[c] = tot == 0;
    n.n_points[c] = np;
    n.n_fields[c] = nf;
}

// has_converged + max_center_delta of two states (engine.py:289-320)
__global__ void k_compare(int K, mfseg_centers o, mfseg_centers n, double eps_c, Flags *fl) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    int active = 0, notconv = 0;
    double dmax = 0.0;
    if (c < K && !n.dormant[c]) {
        active = 1;
        for (int d = 0; d < 4; ++d) {
            double r = rel_change(o.loc[(size_t)d * K + c], n.loc[(size_t)d * K + c]);
            if (r >= eps_c) notconv = 1;
            dmax = fmax(dmax, r);
        }
        bool ohp = o.has_p[c], nhp = n.has_p[c], ohf = o.has_f[c], nhf = n.has_f[c];
        if (ohp != nhp || ohf != nhf) notconv = 1;
        if (ohp && nhp) {
            double r = rel_change(o.pval[c], n.pval[c]);
            if (r >= eps_c) notconv = 1;
            dmax = fmax(dmax, r);
        }
        if (ohf && nhf) {
            double r = rel_change(o.fval[c], n.fval[c]);
            if (r >= eps_c) notconv = 1;
            dmax = fmax(dmax, r);
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        active |= __shfl_xor_sync(0xffffffffu, active, off);
        notconv |= __shfl_xor_sync(0xffffffffu, notconv, off);
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
    }
    if ((threadIdx.x & 31) == 0) {
        if (active) atomicOr(&fl->any_active, 1);
        if (notconv) atomicOr(&fl->not_converged, 1);
        atomicMax(&fl->delta_bits, (unsigned long long)__double_as_longlong(dmax));
    }
}

__global__ void k_acc_to_double(int K, const unsigned long long *acc, double *sums, double *psum,
                                double *fsum, long long *n_p, long long *n_f) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= K) return;
    const unsigned long long *a = acc + (size_t)c * MFSEG_ACC_WORDS;
    for (int d = 0; d < 4; ++d) sums[4 * c + d] = fix2d(a[2 * d], (long long)a[2 * d + 1]);
    psum[c] = fix2d(a[8], (long long)a[9]);
    fsum[c] = fix2d(a[10], (long long)a[11]);
    n_p[c] = (long long)a[12];
    n_f[c] = (long long)a[13];
}

// 128-bit (lo, hi) <-> three 42-bit limbs (sign in the top limb).  Counts are
// stored as pairs too (hi = 0), so one code path covers every word.
__global__ void k_to_limbs(long long npairs, const unsigned long long *acc, long long *limbs) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    __int128 s = (((__int128)(long long)acc[2 * i + 1]) << 64) | (__int128)acc[2 * i];
    const long long M = (1ll << 42) - 1;
    limbs[3 * i] = (long long)(s & M);
    limbs[3 * i + 1] = (long long)((s >> 42) & M);
    limbs[3 * i + 2] = (long long)(s >> 84);
}

__global__ void k_from_limbs(long long npairs, const long long *limbs, unsigned long long *acc) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= npairs) return;
    __int128 s = (__int128)limbs[3 * i] + (((__int128)limbs[3 * i + 1]) << 42) +
                 (((__int128)limbs[3 * i + 2]) << 84);
    acc[2 * i] = (unsigned long long)s;
    acc[2 * i + 1] = (unsigned long long)(s >> 64);
}

}  // namespace

size_t update_flags_bytes() { return sizeof(Flags); }

int launch_update(int K, const unsigned long long *acc, mfseg_centers o, mfseg_centers n,
                  double eps_c, void *flags_dev, cudaStream_t st) {
    MFSEG_CUDA(cudaMemsetAsync(flags_dev, 0, sizeof(Flags), st));
    ::mfseg::count_launch();
    k_update<<<(K + 255) / 256, 256, 0, st>>>(K, acc, o, n, eps_c, (Flags *)flags_dev);
    MFSEG_LAUNCH("k_update");
    return 0;
}

// decode the flags copied to the host: returns converged, delta (engine.py:293-320)
void decode_flags(const void *flags_host, int *converged, double *delta) {
    const Flags *f = (const Flags *)flags_host;
    if (!f->any_active) {
        *converged = 1;
        *delta = 0.0;
        return;
    }
    *converged = f->not_converged ? 0 : 1;
    long long b = (long long)f->delta_bits;
    double d;
    memcpy(&d, &b, sizeof d);
    *delta = d;
}

int launch_acc_to_double(int K, const unsigned long long *acc, double *sums, double *psum,
                         double *fsum, long long *n_p, long long *n_f, cudaStream_t st) {
    if (K <= 0) return 0;
    ::mfseg::count_launch();
    k_acc_to_double<<<(K + 255) / 256, 256, 0, st>>>(K, acc, sums, psum, fsum, n_p, n_f);
    MFSEG_LAUNCH("k_acc_to_double");
    return 0;
}

int launch_to_limbs(long long npairs, const unsigned long long *acc, long long *limbs,
                    cudaStream_t st) {
    if (npairs <= 0) return 0;
    ::mfseg::count_launch();
    k_to_limbs<<<(unsigned)((npairs + 255) / 256), 256, 0, st>>>(npairs, acc, limbs);
    MFSEG_LAUNCH("k_to_limbs");
    return 0;
}

int launch_from_limbs(long long npairs, const long long *limbs, unsigned long long *acc,
                      cudaStream_t st) {
    if (npairs <= 0) return 0;
    ::mfseg::count_launch();
    k_from_limbs<<<(unsigned)((npairs + 255) / 256), 256, 0, st>>>(npairs, limbs, acc);
    MFSEG_LAUNCH("k_from_limbs");
    return 0;
}

}  // namespace mfseg

using namespace mfseg;

extern "C" {

int mfseg_update_centers_f64(int32_t K, const double *sums, const double *psum, const double *fsum,
                             const int64_t *n_p, const int64_t *n_f, mfseg_centers old_state,
                             mfseg_centers new_state, void *stream) {
    if (K <= 0) return 0;
    ::mfseg::count_launch();
    k_update_f64<<<(K + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        K, sums, psum, fsum, (const long long *)n_p, (const long long *)n_f, old_state, new_state);
    MFSEG_LAUNCH("k_update_f64");
    return 0;
}

int mfseg_compare_centers(int32_t K, mfseg_centers old_state, mfseg_centers new_state,
                          double eps_c, int32_t *conv_host, double *delta_host, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Flags *fl = nullptr, *hf = nullptr;
    static_assert(sizeof(Flags) <= 256, "tiny scratch");
    MFSEG_TRY(tiny_scratch((void **)&fl, (void **)&hf));
    MFSEG_CUDA(cudaMemsetAsync(fl, 0, sizeof(Flags), st));
    if (K > 0) {
        ::mfseg::count_launch();
        k_compare<<<(K + 255) / 256, 256, 0, st>>>(K, old_state, new_state, eps_c, fl);
    }
    MFSEG_LAUNCH("k_compare");
    MFSEG_CUDA(cudaMemcpyAsync(hf, fl, sizeof(Flags), cudaMemcpyDeviceToHost, st));
    MFSEG_CUDA(cudaStreamSynchronize(st));
    int conv;
    double delta;
    decode_flags(hf, &conv, &delta);
    if (conv_host) *conv_host = conv;
    if (delta_host) *delta_host = delta;
    return 0;
}

}  // extern "C"
