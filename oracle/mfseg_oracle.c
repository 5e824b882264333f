/*
 * CPU ORACLE (C restatement) for the segmentation hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm (arXiv 1903.12294, `mfseg`
 * package, /root/reference/pkg/src/mfseg/engine.py) used by tests/ and by the
 * CPU-baseline leg of bench.py to CHECK and to TIME-AGAINST the CUDA product.
 * The product library (paper_1903_12294_b200/csrc) never links or calls this.
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, IEEE double on
 * SSE2), so every floating-point operation below rounds exactly like numpy's.
 *
 *   oracle_assign   engine._assign_chunk + _fallback_assign  (engine.py:164-205)
 *   oracle_assign_field  the same for field cells given by the grid geometry
 *   oracle_run      engine.run incl. np.bincount's sequential
 *                   sums (engine.py:244-263) and update/converge (266-320)
 *   oracle_run_grid engine.run with field locations derived from the geometry
 *                   (model.py:137-150) instead of a materialised loc4 array
 *
 * Pinned against the reference's own outputs by tests/test_oracle_golden.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int K;
    const double *cloc; /* K x 4 row-major (x, y, z, t) */
    const double *cval; /* K */
    const uint8_t *chas;
    double mins[4], C[4];
    int k[4];
    int *bin_start; /* nbins + 1 */
    int *bin_ids;   /* K, ascending id inside each bin */
} grid_t;

static long long flat4(const int b[4], const int k[4]) {
    return (((long long)b[3] * k[2] + b[2]) * k[1] + b[1]) * k[0] + b[0];
}

/* clip(floor((x - min) / C), 0, k-1)   engine.py:111-113 */
static void bin_of(const double *loc, const double *mins, const double *C, const int *k, int b[4]) {
    for (int d = 0; d < 4; ++d) {
        double q = floor((loc[d] - mins[d]) / C[d]);
        long long v = (long long)q;
        if (q < 0) v = 0;
        if (v > k[d] - 1) v = k[d] - 1;
        b[d] = (int)v;
    }
}

static int grid_build(grid_t *g) {
    long long nb = (long long)g->k[0] * g->k[1] * g->k[2] * g->k[3];
    g->bin_start = (int *)calloc((size_t)nb + 1, sizeof(int));
    g->bin_ids = (int *)malloc(sizeof(int) * (size_t)(g->K > 0 ? g->K : 1));
    long long *key = (long long *)malloc(sizeof(long long) * (size_t)(g->K > 0 ? g->K : 1));
    if (!g->bin_start || !g->bin_ids || !key) return -1;
    for (int c = 0; c < g->K; ++c) {
        int b[4];
        bin_of(g->cloc + 4 * (size_t)c, g->mins, g->C, g->k, b);
        key[c] = flat4(b, g->k);
        g->bin_start[key[c] + 1]++;
    }
    for (long long i = 0; i < nb; ++i) g->bin_start[i + 1] += g->bin_start[i];
    int *cur = (int *)malloc(sizeof(int) * (size_t)nb);
    if (!cur) return -1;
    memcpy(cur, g->bin_start, sizeof(int) * (size_t)nb);
    for (int c = 0; c < g->K; ++c) g->bin_ids[cur[key[c]]++] = c; /* ascending id */
    free(cur);
    free(key);
    return 0;
}

static void grid_free(grid_t *g) {
    free(g->bin_start);
    free(g->bin_ids);
}

/* D = vterm + wd * sqrt(((dx*dx + dy*dy) + dz*dz) + (cf*dt)*(cf*dt))   engine.py:137-149 */
static double metric(const double *s, double v, const double *c, double cv, int has,
                     double wv, double wd, double cf) {
    double dx = c[0] - s[0], dy = c[1] - s[1], dz = c[2] - s[2], dt = c[3] - s[3];
    double ct = cf * dt;
    double q = dx * dx + dy * dy;
    q = q + dz * dz;
    q = q + ct * ct;
    double sst = sqrt(q);
    double vt = 0.0;
    if (wv > 0) {
        double a = fabs(v - (has ? cv : 0.0));
        vt = wv * (has ? a : 0.0);
    }
    return vt + wd * sst;
}

static int assign_one(const grid_t *g, const double *s, double v, double wv, double wd, double cf) {
    int b[4];
    bin_of(s, g->mins, g->C, g->k, b);
    double best = INFINITY;
    int arg = -1;
    for (int o = 0; o < 81; ++o) {
        int nb[4], oo = o, ok = 1;
        for (int d = 0; d < 4; ++d) {
            nb[d] = b[d] + (oo % 3) - 1;
            oo /= 3;
            if (nb[d] < 0 || nb[d] >= g->k[d]) ok = 0;
        }
        if (!ok) continue;
        long long key = flat4(nb, g->k);
        for (int p = g->bin_start[key]; p < g->bin_start[key + 1]; ++p) {
            int c = g->bin_ids[p];
            const double *cl = g->cloc + 4 * (size_t)c;
            if (fabs(cl[0] - s[0]) <= g->C[0] && fabs(cl[1] - s[1]) <= g->C[1] &&
                fabs(cl[2] - s[2]) <= g->C[2] && fabs(cl[3] - s[3]) <= g->C[3]) {
                double D = metric(s, v, cl, g->cval[c], g->chas[c], wv, wd, cf);
                if (D < best || (D == best && c < arg)) {
                    best = D;
                    arg = c;
                }
            }
        }
    }
    if (arg >= 0) return arg;
    /* stranded: doubling window over ALL centres   engine.py:195-205 */
    for (double mult = 2.0;; mult *= 2.0) {
        for (int c = 0; c < g->K; ++c) {
            const double *cl = g->cloc + 4 * (size_t)c;
            if (fabs(cl[0] - s[0]) <= mult * g->C[0] && fabs(cl[1] - s[1]) <= mult * g->C[1] &&
                fabs(cl[2] - s[2]) <= mult * g->C[2] && fabs(cl[3] - s[3]) <= mult * g->C[3]) {
                double D = metric(s, v, cl, g->cval[c], g->chas[c], wv, wd, cf);
                if (arg < 0 || D < best) { /* ascending ids: first minimum wins */
                    best = D;
                    arg = c;
                }
            }
        }
        if (arg >= 0) return arg;
        if (!(mult < 1e300)) return -1;
    }
}

/* Samples: either an n x 4 location array, or field cells whose locations are
 * derived from the grid geometry exactly as FieldSet.cell_centers / loc4 do
 * (model.py:137-150: origin + (i + 0.5) * spacing, two roundings; timestep-major,
 * x fastest), optionally restricted to a list of flat indices. */
typedef struct {
    const double *loc;    /* n x 4, or NULL: field geometry below */
    const double *val;    /* per sample (loc mode) or the whole field (geometry mode) */
    int nx, ny, nz;
    long long ncell;
    double origin[3], spacing[3];
    const double *times;
    const int64_t *idx;   /* geometry mode: flat indices of the samples, or NULL = all */
} src_t;

static void src_sample(const src_t *s, long long i, double out[4], double *v) {
    if (s->loc) {
        memcpy(out, s->loc + 4 * i, 4 * sizeof(double));
        *v = s->val[i];
        return;
    }
    long long q = s->idx ? s->idx[i] : i;
    long long m = q / s->ncell, r = q % s->ncell;
    long long ii = r % s->nx, jj = (r / s->nx) % s->ny, kk = r / ((long long)s->nx * s->ny);
    out[0] = s->origin[0] + ((double)ii + 0.5) * s->spacing[0];
    out[1] = s->origin[1] + ((double)jj + 0.5) * s->spacing[1];
    out[2] = s->origin[2] + ((double)kk + 0.5) * s->spacing[2];
    out[3] = s->times[m];
    *v = s->val[q];
}

static src_t loc_src(const double *loc, const double *val) {
    src_t s;
    memset(&s, 0, sizeof s);
    s.loc = loc;
    s.val = val;
    return s;
}

static src_t grid_src(const int *dims, const double *origin, const double *spacing,
                      const double *times, const double *values, const int64_t *idx) {
    src_t s;
    memset(&s, 0, sizeof s);
    s.val = values;
    s.nx = dims[0];
    s.ny = dims[1];
    s.nz = dims[2];
    s.ncell = (long long)dims[0] * dims[1] * dims[2];
    for (int d = 0; d < 3; ++d) {
        s.origin[d] = origin[d];
        s.spacing[d] = spacing[d];
    }
    s.times = times;
    s.idx = idx;
    return s;
}

typedef struct {
    const grid_t *g;
    const src_t *src;
    int64_t *out;
    long long lo, hi;
    double wv, wd, cf;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    double s[4], v;
    for (long long i = j->lo; i < j->hi; ++i) {
        src_sample(j->src, i, s, &v);
        j->out[i] = assign_one(j->g, s, v, j->wv, j->wd, j->cf);
    }
    return NULL;
}

static void assign_all(const grid_t *g, long long n, const src_t *src,
                       double wv, double wd, double cf, int64_t *out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (n < 4096) threads = 1;
    pthread_t th[256];
    job_t jobs[256];
    long long per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        long long lo = per * t, hi = lo + per < n ? lo + per : n;
        if (lo > n) lo = n;
        jobs[t] = (job_t){g, src, out, lo, hi, wv, wd, cf};
        if (threads == 1) worker(&jobs[t]);
        else pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* One windowed assignment of n samples given the centres.  loc is n x 4. */
int oracle_assign(long long n, const double *loc, const double *val, int K, const double *cloc,
                  const double *cval, const uint8_t *chas, const double *mins, const double *C,
                  const int *k, double wv, double wd, double cf, int64_t *out, int threads) {
    grid_t g = {K, cloc, cval, chas, {0}, {0}, {0}, NULL, NULL};
    for (int d = 0; d < 4; ++d) {
        g.mins[d] = mins[d];
        g.C[d] = C[d];
        g.k[d] = k[d];
    }
    if (grid_build(&g)) return -1;
    src_t s = loc_src(loc, val);
    assign_all(&g, n, &s, wv, wd, cf, out, threads);
    grid_free(&g);
    return 0;
}

/* The same for field cells given by the grid geometry: the samples are the
 * flat indices idx[0..n) (or all nt * ncell cells when idx is NULL). */
int oracle_assign_field(long long n, const int64_t *idx, const int *dims, const double *origin,
                        const double *spacing, const double *times, const double *values, int K,
                        const double *cloc, const double *cval, const uint8_t *chas,
                        const double *mins, const double *C, const int *k, double wv, double wd,
                        double cf, int64_t *out, int threads) {
    grid_t g = {K, cloc, cval, chas, {0}, {0}, {0}, NULL, NULL};
    for (int d = 0; d < 4; ++d) {
        g.mins[d] = mins[d];
        g.C[d] = C[d];
        g.k[d] = k[d];
    }
    if (grid_build(&g)) return -1;
    src_t s = grid_src(dims, origin, spacing, times, values, idx);
    assign_all(&g, n, &s, wv, wd, cf, out, threads);
    grid_free(&g);
    return 0;
}

/* Sequential per-cluster sums in sample-index order (np.bincount)  engine.py:244-263 */
static void accumulate(int K, long long np_, const src_t *ps, const int64_t *pl, long long nf,
                       const src_t *fs, const int64_t *fl, double *sums, double *psum,
                       double *fsum, int64_t *n_p, int64_t *n_f) {
    double s[4], v;
    double *P = (double *)calloc((size_t)K * 4, sizeof(double));
    double *F = (double *)calloc((size_t)K * 4, sizeof(double));
    memset(psum, 0, sizeof(double) * K);
    memset(fsum, 0, sizeof(double) * K);
    memset(n_p, 0, sizeof(int64_t) * K);
    memset(n_f, 0, sizeof(int64_t) * K);
    for (long long i = 0; i < np_; ++i) {
        int64_t c = pl[i];
        src_sample(ps, i, s, &v);
        for (int d = 0; d < 4; ++d) P[4 * c + d] += s[d];
        psum[c] += v;
        n_p[c]++;
    }
    for (long long i = 0; i < nf; ++i) {
        int64_t c = fl[i];
        src_sample(fs, i, s, &v);
        for (int d = 0; d < 4; ++d) F[4 * c + d] += s[d];
        fsum[c] += v;
        n_f[c]++;
    }
    for (long long j = 0; j < 4LL * K; ++j) sums[j] = (0.0 + P[j]) + F[j];
    free(P);
    free(F);
}

static double rel(double o, double n) { return fabs(n - o) / (fabs(o) + 1e-12); }

/*
 * engine.run (engine.py:323-381) on already-normalized samples.
 * ploc: np x 4, floc: nf x 4 (field sample locations, timestep-major).
 * State arrays (cloc K x 4, pval, fval, has_p, has_f, n_points, n_fields, dormant)
 * are outputs; progress_delta[max_iter] receives the per-iteration max delta.
 * Returns iterations_used, converged via pointers.
 */
static int run_impl(long long np_, const src_t *ps, long long nf, const src_t *fs,
                    const double *mins, const double *maxs, const int *k, double cf, double wd,
                    double wp, double wf, double eps_c, int max_iter, int threads,
                    int32_t *pl_out, int32_t *fl_out, double *cloc, double *cpv, double *cfv,
                    uint8_t *has_p, uint8_t *has_f, int64_t *n_points, int64_t *n_fields,
                    uint8_t *dormant, int *iters_used, int *converged, double *progress_delta) {
    double C[4];
    for (int d = 0; d < 4; ++d) C[d] = (maxs[d] - mins[d]) / k[d];
    int K = k[0] * k[1] * k[2] * k[3];
    /* seeds engine.py:31-45 */
    int id = 0;
    for (int it = 0; it < k[3]; ++it)
        for (int iz = 0; iz < k[2]; ++iz)
            for (int iy = 0; iy < k[1]; ++iy)
                for (int ix = 0; ix < k[0]; ++ix, ++id) {
                    cloc[4 * id + 0] = mins[0] + (ix + 0.5) * C[0];
                    cloc[4 * id + 1] = mins[1] + (iy + 0.5) * C[1];
                    cloc[4 * id + 2] = mins[2] + (iz + 0.5) * C[2];
                    cloc[4 * id + 3] = mins[3] + (it + 0.5) * C[3];
                }
    for (int c = 0; c < K; ++c) {
        cpv[c] = NAN;
        cfv[c] = NAN;
        has_p[c] = has_f[c] = dormant[c] = 0;
        n_points[c] = n_fields[c] = 0;
    }
    int64_t *pl = (int64_t *)malloc(sizeof(int64_t) * (size_t)(np_ > 0 ? np_ : 1));
    int64_t *fl = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf > 0 ? nf : 1));
    double *sums = (double *)malloc(sizeof(double) * 4 * K);
    double *psum = (double *)malloc(sizeof(double) * K), *fsum = (double *)malloc(sizeof(double) * K);
    int64_t *cnp = (int64_t *)malloc(sizeof(int64_t) * K), *cnf = (int64_t *)malloc(sizeof(int64_t) * K);
    double *oloc = (double *)malloc(sizeof(double) * 4 * K);
    double *opv = (double *)malloc(sizeof(double) * K), *ofv = (double *)malloc(sizeof(double) * K);
    uint8_t *ohp = (uint8_t *)malloc(K), *ohf = (uint8_t *)malloc(K);
    *iters_used = 0;
    *converged = 0;
    for (int pass = 0; pass <= max_iter; ++pass) {
        double pw = pass == 0 ? 0.0 : wp, fw = pass == 0 ? 0.0 : wf, dw = pass == 0 ? 1.0 : wd;
        grid_t g = {K, cloc, cpv, has_p, {0}, {0}, {0}, NULL, NULL};
        for (int d = 0; d < 4; ++d) {
            g.mins[d] = mins[d];
            g.C[d] = C[d];
            g.k[d] = k[d];
        }
        if (grid_build(&g)) return -1;
        assign_all(&g, np_, ps, pw, dw, cf, pl, threads);
        g.cval = cfv;
        g.chas = has_f;
        assign_all(&g, nf, fs, fw, dw, cf, fl, threads);
        grid_free(&g);
        accumulate(K, np_, ps, pl, nf, fs, fl, sums, psum, fsum, cnp, cnf);
        memcpy(oloc, cloc, sizeof(double) * 4 * K);
        memcpy(opv, cpv, sizeof(double) * K);
        memcpy(ofv, cfv, sizeof(double) * K);
        memcpy(ohp, has_p, K);
        memcpy(ohf, has_f, K);
        /* update_centers  engine.py:266-286 */
        for (int c = 0; c < K; ++c) {
            int64_t tot = cnp[c] + cnf[c];
            if (tot > 0) {
                for (int d = 0; d < 4; ++d) cloc[4 * c + d] = sums[4 * c + d] / (double)tot;
                has_p[c] = cnp[c] > 0;
                has_f[c] = cnf[c] > 0;
                cpv[c] = has_p[c] ? psum[c] / (double)(cnp[c] > 1 ? cnp[c] : 1) : NAN;
                cfv[c] = has_f[c] ? fsum[c] / (double)(cnf[c] > 1 ? cnf[c] : 1) : NAN;
                dormant[c] = 0;
            } else {
                dormant[c] = 1; /* loc, values and has-flags frozen */
            }
            n_points[c] = cnp[c];
            n_fields[c] = cnf[c];
        }
        if (pass == 0) continue;
        /* max_center_delta + has_converged  engine.py:289-320 */
        int any_active = 0, conv = 1;
        double delta = 0.0;
        int have_p = 0, have_f = 0;
        double dp = 0.0, df = 0.0, dl = 0.0;
        int first = 1;
        for (int c = 0; c < K; ++c) {
            if (dormant[c]) continue;
            any_active = 1;
            for (int d = 0; d < 4; ++d) {
                double r = rel(oloc[4 * c + d], cloc[4 * c + d]);
                if (first || r > dl) dl = r;
                first = 0;
                if (r >= eps_c) conv = 0;
            }
            if (ohp[c] != has_p[c] || ohf[c] != has_f[c]) conv = 0;
            if (ohp[c] && has_p[c]) {
                double r = rel(opv[c], cpv[c]);
                if (!have_p || r > dp) dp = r;
                have_p = 1;
                if (r >= eps_c) conv = 0;
            }
            if (ohf[c] && has_f[c]) {
                double r = rel(ofv[c], cfv[c]);
                if (!have_f || r > df) df = r;
                have_f = 1;
                if (r >= eps_c) conv = 0;
            }
        }
        if (!any_active) {
            conv = 1;
            delta = 0.0;
        } else {
            delta = dl;
            if (have_p && dp > delta) delta = dp;
            if (have_f && df > delta) delta = df;
        }
        progress_delta[pass - 1] = delta;
        *iters_used = pass;
        *converged = conv;
        if (conv) break;
    }
    for (long long i = 0; i < np_; ++i) pl_out[i] = (int32_t)pl[i];
    for (long long i = 0; i < nf; ++i) fl_out[i] = (int32_t)fl[i];
    free(pl); free(fl); free(sums); free(psum); free(fsum); free(cnp); free(cnf);
    free(oloc); free(opv); free(ofv); free(ohp); free(ohf);
    return 0;
}

int oracle_run(long long np_, const double *ploc, const double *pval, long long nf,
               const double *floc, const double *fval, const double *mins, const double *maxs,
               const int *k, double cf, double wd, double wp, double wf, double eps_c,
               int max_iter, int threads, int32_t *pl_out, int32_t *fl_out, double *cloc,
               double *cpv, double *cfv, uint8_t *has_p, uint8_t *has_f, int64_t *n_points,
               int64_t *n_fields, uint8_t *dormant, int *iters_used, int *converged,
               double *progress_delta) {
    src_t ps = loc_src(ploc, pval), fs = loc_src(floc, fval);
    return run_impl(np_, &ps, nf, &fs, mins, maxs, k, cf, wd, wp, wf, eps_c, max_iter, threads,
                    pl_out, fl_out, cloc, cpv, cfv, has_p, has_f, n_points, n_fields, dormant,
                    iters_used, converged, progress_delta);
}

/* engine.run with the field given by its grid geometry (dims, origin, spacing,
 * times, values [nt][ncell]): field locations are derived per cell (model.py:137-150)
 * instead of a materialised loc4 array, so bench-scale fields fit in host memory. */
int oracle_run_grid(long long np_, const double *ploc, const double *pval, int nt,
                    const int *dims, const double *origin, const double *spacing,
                    const double *times, const double *fval, const double *mins,
                    const double *maxs, const int *k, double cf, double wd, double wp, double wf,
                    double eps_c, int max_iter, int threads, int32_t *pl_out, int32_t *fl_out,
                    double *cloc, double *cpv, double *cfv, uint8_t *has_p, uint8_t *has_f,
                    int64_t *n_points, int64_t *n_fields, uint8_t *dormant, int *iters_used,
                    int *converged, double *progress_delta) {
    src_t ps = loc_src(ploc, pval);
    src_t fs = grid_src(dims, origin, spacing, times, fval, NULL);
    long long nf = nt > 0 ? (long long)nt * fs.ncell : 0;
    return run_impl(np_, &ps, nf, &fs, mins, maxs, k, cf, wd, wp, wf, eps_c, max_iter, threads,
                    pl_out, fl_out, cloc, cpv, cfv, has_p, has_f, n_points, n_fields, dormant,
                    iters_used, converged, progress_delta);
}
