// Counter-based synthetic inputs for the benchmark configurations.
//
// Same spirit as the reference's generator (drifting blobs over a background
// plus noise, ingest.py:341-544) but every value is a pure function of
// (seed, index), so a GPU can generate 5e8 voxels in milliseconds and the
// numpy mirror (oracle/synth.py) reproduces any sub-block bit for bit.  Only
// exactly-rounded IEEE ops are used (+ - * / floor, no transcendental).
#include "kernels.cuh"

namespace mfseg {
namespace {

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ unsigned long long h3(unsigned long long seed,
                                                          unsigned long long a,
                                                          unsigned long long b) {
    return mix64(mix64(seed ^ mix64(a)) + b);
}
__host__ __device__ __forceinline__ double u01(unsigned long long h) {
    return (double)(h >> 11) * 0x1.0p-53;
}

constexpr int MAXB = 16;
struct Blob {
    double cx, cy, cz, rx, ry, rz, vx, vy, vz, fv, pv;
};
struct Blobs {
    int n;
    Blob b[MAXB];
};

// blob b of a dataset (dims in cell units, spacing 1, origin 0)
Blobs make_blobs(const mfseg_synth *s) {
    Blobs B;
    B.n = s->n_blobs < MAXB ? s->n_blobs : MAXB;
    double nx = s->nx, ny = s->ny, nz = s->nz, nt = s->nt > 1 ? s->nt - 1 : 1;
    for (int b = 0; b < B.n; ++b) {
        volatile double u[9];
        for (int q = 0; q < 9; ++q) u[q] = u01(h3(s->seed, 1000 + b, q));
        Blob &o = B.b[b];
        volatile double t;
        t = 0.6 * u[0]; o.cx = nx * (0.2 + t);
        t = 0.6 * u[1]; o.cy = ny * (0.2 + t);
        t = 0.6 * u[2]; o.cz = nz * (0.2 + t);
        t = 0.08 * u[3]; o.rx = nx * (0.06 + t);
        t = 0.08 * u[4]; o.ry = ny * (0.06 + t);
        t = 0.08 * u[5]; o.rz = nz * (0.06 + t);
        t = nx * (u[6] - 0.5); o.vx = (t * 0.3) / nt;
        t = ny * (u[7] - 0.5); o.vy = (t * 0.3) / nt;
        t = nz * (u[8] - 0.5); o.vz = (t * 0.3) / nt;
        o.fv = (double)(b + 1) / (double)(B.n + 1);
        o.pv = 1.0 - o.fv;
    }
    return B;
}

__device__ int blob_at(const Blobs &B, double x, double y, double z, double m) {
    for (int b = 0; b < B.n; ++b) {
        const Blob &o = B.b[b];
        double dx = DDIV(DSUB(x, DADD(o.cx, DMUL(o.vx, m))), o.rx);
        double dy = DDIV(DSUB(y, DADD(o.cy, DMUL(o.vy, m))), o.ry);
        double dz = DDIV(DSUB(z, DADD(o.cz, DMUL(o.vz, m))), o.rz);
        if (DADD(DADD(DMUL(dx, dx), DMUL(dy, dy)), DMUL(dz, dz)) <= 1.0) return b;
    }
    return -1;
}

__device__ double noisy(double base, unsigned long long seed, unsigned long long idx,
                        double noise, int dyadic) {
    double u = DADD(DADD(DADD(u01(h3(seed, idx, 1)), u01(h3(seed, idx, 2))), u01(h3(seed, idx, 3))),
                    u01(h3(seed, idx, 4)));
    double v = DADD(base, DMUL(noise, DSUB(u, 2.0)));
    if (dyadic) {
        v = DDIV(floor(DMUL(v, 1048576.0)), 1048576.0);
        v = fmin(fmax(v, 0.0), 1.0);
    }
    return v;
}

// window [m0, m0 + wt) x [z0, z0 + wz) of the dataset's timesteps x z-planes;
// every value depends only on its GLOBAL flat index q
__global__ void k_synth_field(mfseg_synth s, Blobs B, int m0, int wt, int z0, int wz, double *values) {
    const long long plane = (long long)s.nx * s.ny, ncell = plane * s.nz;
    const long long n = plane * wz * wt;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < n;
         w += (long long)gridDim.x * blockDim.x) {
        long long r = w;
        int i = (int)(r % s.nx);
        r /= s.nx;
        int j = (int)(r % s.ny);
        r /= s.ny;
        int k = z0 + (int)(r % wz);
        int m = m0 + (int)(r / wz);
        const long long q = (long long)m * ncell + ((long long)k * s.ny + j) * s.nx + i;
        int b = blob_at(B, (double)i + 0.5, (double)j + 0.5, (double)k + 0.5, (double)m);
        double v = noisy(b >= 0 ? B.b[b].fv : 0.0, s.seed, (unsigned long long)q, s.noise, s.dyadic);
        if (s.dyadic && q < 2) v = (double)q;   // pin min 0 / max 1: normalization is the identity
        values[w] = v;
    }
}

// trajectories [p0, p0 + wp) x timesteps [m0, m0 + wt), trajectory-major; every
// sample depends only on its GLOBAL record index q = p * nt + m
__global__ void k_synth_points(mfseg_synth s, Blobs B, long long p0, long long wp, int m0, int wt,
                               long long *traj_id, double *t, double *xyz, double *value) {
    long long n = wp * wt;
    double ex = s.nx, ey = s.ny, ez = s.nz;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < n;
         w += (long long)gridDim.x * blockDim.x) {
        long long p = p0 + w / wt;
        int m = m0 + (int)(w % wt);
        const long long q = p * s.nt + m;
        unsigned long long sp = s.seed ^ 0x5bd1e995ull;
        double x0 = DMUL(ex, u01(h3(sp, p, 11))), y0 = DMUL(ey, u01(h3(sp, p, 12))),
               z0 = DMUL(ez, u01(h3(sp, p, 13)));
        double vx = DSUB(DMUL(2.0, u01(h3(sp, p, 14))), 1.0);
        double vy = DSUB(DMUL(2.0, u01(h3(sp, p, 15))), 1.0);
        double vz = DSUB(DMUL(2.0, u01(h3(sp, p, 16))), 1.0);
        double mm = (double)m;
        double x = DADD(x0, DMUL(vx, mm)), y = DADD(y0, DMUL(vy, mm)), z = DADD(z0, DMUL(vz, mm));
        // keep inside [0, n) (clip; exact)
        x = fmin(fmax(x, 0.0), DSUB(ex, 0x1.0p-16));
        y = fmin(fmax(y, 0.0), DSUB(ey, 0x1.0p-16));
        z = fmin(fmax(z, 0.0), DSUB(ez, 0x1.0p-16));
        if (s.dyadic) {
            x = DDIV(floor(DMUL(x, 65536.0)), 65536.0);
            y = DDIV(floor(DMUL(y, 65536.0)), 65536.0);
            z = DDIV(floor(DMUL(z, 65536.0)), 65536.0);
        }
        int b = blob_at(B, x, y, z, mm);
        double v = noisy(b >= 0 ? B.b[b].pv : 0.0, sp, (unsigned long long)q, s.noise, s.dyadic);
        if (s.dyadic && q < 2) v = (double)q;
        traj_id[w] = p;
        t[w] = mm;
        xyz[3 * w] = x;
        xyz[3 * w + 1] = y;
        xyz[3 * w + 2] = z;
        value[w] = v;
    }
}

// Taxi-like 2D+t trajectories (configs[3]): `steps` consecutive samples from a
// uniform random start step; a fraction `skew` of the trajectories drive along
// one of the road rows / columns (a fraction `road_frac` of them, evenly
// spread), the rest move freely.  z is the single layer's centre 0.5 * nz.
__global__ void k_synth_taxi(mfseg_synth s, Blobs B, int steps, double skew, int n_rows, int n_cols,
                             long long p0, long long wp, long long *traj_id, double *t, double *xyz,
                             double *value) {
    const long long n = wp * steps;
    const double ex = s.nx, ey = s.ny;
    const double z = DMUL(0.5, (double)s.nz);
    const int span = s.nt - steps + 1 > 1 ? s.nt - steps + 1 : 1;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < n;
         w += (long long)gridDim.x * blockDim.x) {
        const long long p = p0 + w / steps;
        const int j = (int)(w % steps);
        const unsigned long long sp = s.seed ^ 0x7a3c5e91ull;
        const int s0 = min((int)(u01(h3(sp, p, 21)) * span), span - 1);
        const int m = s0 + j;
        double x0 = DMUL(ex, u01(h3(sp, p, 22))), y0 = DMUL(ey, u01(h3(sp, p, 23)));
        double vx = DSUB(DMUL(2.0, u01(h3(sp, p, 24))), 1.0);
        double vy = DSUB(DMUL(2.0, u01(h3(sp, p, 25))), 1.0);
        if (u01(h3(sp, p, 26)) < skew) {
            const double r = u01(h3(sp, p, 27));
            if (u01(h3(sp, p, 28)) < 0.5) {   // along a road row
                const int q = min((int)(r * n_rows), n_rows - 1);
                y0 = DADD(floor(DDIV(DMUL((double)q + 0.5, ey), (double)n_rows)), 0.5);
                vy = 0.0;
                vx = DMUL(vx, 3.0);
            } else {                           // along a road column
                const int q = min((int)(r * n_cols), n_cols - 1);
                x0 = DADD(floor(DDIV(DMUL((double)q + 0.5, ex), (double)n_cols)), 0.5);
                vx = 0.0;
                vy = DMUL(vy, 3.0);
            }
        }
        const double mm = (double)j;
        double x = DADD(x0, DMUL(vx, mm)), y = DADD(y0, DMUL(vy, mm));
        x = fmin(fmax(x, 0.0), DSUB(ex, 0x1.0p-16));
        y = fmin(fmax(y, 0.0), DSUB(ey, 0x1.0p-16));
        const int b = blob_at(B, x, y, z, (double)m);
        const double v = noisy(b >= 0 ? B.b[b].pv : 0.0, sp, (unsigned long long)(p * steps + j),
                               s.noise, 0);
        traj_id[w] = p;
        t[w] = (double)m;
        xyz[3 * w] = x;
        xyz[3 * w + 1] = y;
        xyz[3 * w + 2] = z;
        value[w] = v;
    }
}

}  // namespace
}  // namespace mfseg

using namespace mfseg;

extern "C" {

int mfseg_synth_field_window(const mfseg_synth *s, int32_t m0, int32_t m1, int32_t z0, int32_t z1,
                             double *values, void *stream) {
    if (m0 < 0 || m1 > s->nt || m0 > m1 || z0 < 0 || z1 > s->nz || z0 > z1) {
        set_error("synth_field_window: window outside the dataset");
        return 2;
    }
    if (m1 == m0 || z1 == z0) return 0;
    Blobs B = make_blobs(s);
    ::mfseg::count_launch();
    k_synth_field<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(*s, B, m0, m1 - m0, z0, z1 - z0, values);
    MFSEG_LAUNCH("k_synth_field");
    return 0;
}

int mfseg_synth_field(const mfseg_synth *s, double *values, void *stream) {
    return mfseg_synth_field_window(s, 0, s->nt, 0, s->nz, values, stream);
}

int mfseg_synth_points_window(const mfseg_synth *s, int64_t p0, int64_t p1, int32_t m0, int32_t m1,
                              int64_t *traj_id, double *t, double *xyz, double *value, void *stream) {
    if (p0 < 0 || p1 > s->n_traj || p0 > p1 || m0 < 0 || m1 > s->nt || m0 > m1) {
        set_error("synth_points_window: window outside the dataset");
        return 2;
    }
    if (p1 == p0 || m1 == m0) return 0;
    Blobs B = make_blobs(s);
    ::mfseg::count_launch();
    k_synth_points<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(*s, B, p0, p1 - p0, m0, m1 - m0,
                                                               (long long *)traj_id, t, xyz, value);
    MFSEG_LAUNCH("k_synth_points");
    return 0;
}

int mfseg_synth_points(const mfseg_synth *s, int64_t *traj_id, double *t, double *xyz,
                       double *value, void *stream) {
    return mfseg_synth_points_window(s, 0, s->n_traj, 0, s->nt, traj_id, t, xyz, value, stream);
}

int mfseg_synth_taxi_points(const mfseg_synth *s, int32_t steps, double skew, double road_frac,
                            int64_t p0, int64_t p1, int64_t *traj_id, double *t, double *xyz,
                            double *value, void *stream) {
    if (p0 < 0 || p1 > s->n_traj || p0 > p1 || steps < 1 || steps > s->nt) {
        set_error("synth_taxi_points: bad trajectory window or steps");
        return 2;
    }
    if (p1 == p0) return 0;
    Blobs B = make_blobs(s);
    const int n_rows = (int)(road_frac * s->ny) > 1 ? (int)(road_frac * s->ny) : 1;
    const int n_cols = (int)(road_frac * s->nx) > 1 ? (int)(road_frac * s->nx) : 1;
    ::mfseg::count_launch();
    k_synth_taxi<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(*s, B, steps, skew, n_rows, n_cols, p0,
                                                             p1 - p0, (long long *)traj_id, t, xyz,
                                                             value);
    MFSEG_LAUNCH("k_synth_taxi");
    return 0;
}

}  // extern "C"
