/*
 * mlb_oracle.c -- plain-C restatement of the reference NFFT spread / gather
 * (TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs may load it; the product never does).
 *
 * Reference: /root/reference/pkg/src/multilap/fastsum.py
 *   _kb_window        fastsum.py:158-167  (three branches: sinh / sin / b/pi)
 *   _make_binding     fastsum.py:333-372  (per axis u = floor(ng*x) + o,
 *                                          o = -m..m, weight phi(ng*x - u),
 *                                          index u mod ng, row-major flat
 *                                          index with axis 0 slowest)
 *   bind_points       fastsum.py:375-386  (x * 1/sqrt(d) onto the torus)
 *   _spread_real      fastsum.py:389-391  (g[c] += w v_i)
 *   _gather           fastsum.py:400-406  (y_i = sum_c w g[c])
 *
 * It is the chunked oracle of SURVEY 8(c) without the binding arrays: the
 * tensor-product weights of a point are formed on the fly (the reference
 * binding would need 16 (2m+1)^d bytes per point: 213 GB at config 4), the
 * arithmetic per weight is the reference's (product of the d axis windows in
 * axis order, then times v), and only the summation order differs: every
 * host thread (pthreads) spreads a contiguous point range into a private grid and the grids
 * are summed in thread order.  nv vectors share one pass over the points.
 * The FFT stage (rfftn * fused * irfftn, fastsum.py:492-495) stays in
 * numpy/scipy (oracle/c_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MLBO_MAXS 32  /* 2m+1 <= 31 */

/* phi(t), fastsum.py:158-167: z = m^2 - t^2 */
double mlbo_window(double t, int m, double b) {
    const double z = (double)m * (double)m - t * t;
    if (z > 0.0) {
        const double s = sqrt(z);
        return sinh(b * s) / s / M_PI;
    }
    if (z < 0.0) {
        const double s = sqrt(-z);
        return sin(b * s) / s / M_PI;
    }
    return b / M_PI;
}

/* per axis: flat index part (u mod ng) and window weight for the 2m+1 offsets */
static void axis_weights(double x, double scale, int ng, int m, double b, int32_t* idx, double* w) {
    const double tx = (double)ng * (x * scale);
    const int64_t u0 = (int64_t)floor(tx);
    for (int o = -m; o <= m; ++o) {
        const int64_t u = u0 + o;
        w[o + m] = mlbo_window(tx - (double)u, m, b);
        int64_t r = u % ng;
        if (r < 0) r += ng;
        idx[o + m] = (int32_t)r;
    }
}

/* ---- host threads: a static partition of [0, n) (results independent of timing) */
typedef struct {
    int d, ng, m, nv, tid, nt;
    double b, scale;
    const double* pts;
    int64_t n, G;
    const double* in;   /* spread: v (nv x n); gather: grid (nv x G) */
    double* out;        /* spread: private grid of this thread; gather: y (nv x n) */
} job_t;

static int default_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c < 1 ? 1 : (int)c;
}

static void* spread_job(void* arg) {
    const job_t* J = (const job_t*)arg;
    const int d = J->d, ng = J->ng, m = J->m, nv = J->nv, S = 2 * m + 1;
    const int64_t n = J->n, G = J->G;
    const int64_t i0 = n * J->tid / J->nt, i1 = n * (J->tid + 1) / J->nt;
    const double* v = J->in;
    double* g = J->out;
    int32_t idx[3][MLBO_MAXS];
    double w[3][MLBO_MAXS];
    for (int64_t i = i0; i < i1; ++i) {
        for (int a = 0; a < d; ++a) axis_weights(J->pts[i * d + a], J->scale, ng, m, J->b, idx[a], w[a]);
        if (d == 1) {
            for (int p = 0; p < S; ++p)
                for (int k = 0; k < nv; ++k) g[k * G + idx[0][p]] += w[0][p] * v[k * n + i];
        } else if (d == 2) {
            for (int p = 0; p < S; ++p)
                for (int q = 0; q < S; ++q) {
                    const int64_t c = (int64_t)idx[0][p] * ng + idx[1][q];
                    const double wt = w[0][p] * w[1][q];
                    for (int k = 0; k < nv; ++k) g[k * G + c] += wt * v[k * n + i];
                }
        } else {
            for (int p = 0; p < S; ++p)
                for (int q = 0; q < S; ++q) {
                    const int64_t c01 = ((int64_t)idx[0][p] * ng + idx[1][q]) * ng;
                    const double w01 = w[0][p] * w[1][q];
                    for (int r = 0; r < S; ++r) {
                        const int64_t c = c01 + idx[2][r];
                        const double wt = w01 * w[2][r];
                        for (int k = 0; k < nv; ++k) g[k * G + c] += wt * v[k * n + i];
                    }
                }
        }
    }
    return NULL;
}

static void* gather_job(void* arg) {
    const job_t* J = (const job_t*)arg;
    const int d = J->d, ng = J->ng, m = J->m, nv = J->nv, S = 2 * m + 1;
    const int64_t n = J->n, G = J->G;
    const int64_t i0 = n * J->tid / J->nt, i1 = n * (J->tid + 1) / J->nt;
    const double* grid = J->in;
    int32_t idx[3][MLBO_MAXS];
    double w[3][MLBO_MAXS];
    for (int64_t i = i0; i < i1; ++i) {
        double acc[16];
        for (int k = 0; k < nv; ++k) acc[k] = 0.0;
        for (int a = 0; a < d; ++a) axis_weights(J->pts[i * d + a], J->scale, ng, m, J->b, idx[a], w[a]);
        if (d == 1) {
            for (int p = 0; p < S; ++p)
                for (int k = 0; k < nv; ++k) acc[k] += w[0][p] * grid[k * G + idx[0][p]];
        } else if (d == 2) {
            for (int p = 0; p < S; ++p)
                for (int q = 0; q < S; ++q) {
                    const int64_t c = (int64_t)idx[0][p] * ng + idx[1][q];
                    const double wt = w[0][p] * w[1][q];
                    for (int k = 0; k < nv; ++k) acc[k] += wt * grid[k * G + c];
                }
        } else {
            for (int p = 0; p < S; ++p)
                for (int q = 0; q < S; ++q) {
                    const int64_t c01 = ((int64_t)idx[0][p] * ng + idx[1][q]) * ng;
                    const double w01 = w[0][p] * w[1][q];
                    for (int r = 0; r < S; ++r) {
                        const double wt = w01 * w[2][r];
                        const int64_t c = c01 + idx[2][r];
                        for (int k = 0; k < nv; ++k) acc[k] += wt * grid[k * G + c];
                    }
                }
        }
        for (int k = 0; k < nv; ++k) J->out[k * n + i] = acc[k];
    }
    return NULL;
}

static int run_jobs(job_t* jobs, int nt, void* (*fn)(void*)) {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
    if (!th) return 2;
    int started = 0, rc = 0;
    for (int t = 1; t < nt; ++t) {
        if (pthread_create(&th[t], NULL, fn, &jobs[t]) != 0) {
            rc = 3;
            break;
        }
        started = t;
    }
    if (rc == 0) fn(&jobs[0]);
    for (int t = 1; t <= started; ++t) pthread_join(th[t], NULL);
    free(th);
    return rc;
}

static int64_t grid_size(int d, int ng) {
    int64_t G = 1;
    for (int a = 0; a < d; ++a) G *= ng;
    return G;
}

/* grid[k * G + c] = sum over points of w * v[k * n + i]  (nv vectors, G = ng^d) */
int mlbo_spread(int d, int ng, int m, double b, double scale, const double* pts, int64_t n, const double* v, int nv,
                double* grid, int threads) {
    if (d < 1 || d > 3 || 2 * m + 1 > MLBO_MAXS || nv < 1) return 1;
    const int64_t G = grid_size(d, ng);
    const int nt = threads < 1 ? default_threads() : threads;
    double* priv = (double*)calloc((size_t)nt * nv * G, sizeof(double));
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nt);
    if (!priv || !jobs) {
        free(priv);
        free(jobs);
        return 2;
    }
    for (int t = 0; t < nt; ++t)
        jobs[t] = (job_t){d, ng, m, nv, t, nt, b, scale, pts, n, G, v, priv + (size_t)t * nv * G};
    int rc = run_jobs(jobs, nt, spread_job);
    /* the private grids summed in thread order */
    if (rc == 0)
        for (int64_t c = 0; c < (int64_t)nv * G; ++c) {
            double acc = priv[c];
            for (int t = 1; t < nt; ++t) acc += priv[(size_t)t * nv * G + c];
            grid[c] = acc;
        }
    free(priv);
    free(jobs);
    return rc;
}

/* y[k * n + i] = sum over the point's stencil of w * grid[k * G + c] */
int mlbo_gather(int d, int ng, int m, double b, double scale, const double* pts, int64_t n, const double* grid, int nv,
                double* y, int threads) {
    if (d < 1 || d > 3 || 2 * m + 1 > MLBO_MAXS || nv < 1 || nv > 16) return 1;
    const int64_t G = grid_size(d, ng);
    const int nt = threads < 1 ? default_threads() : threads;
    job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nt);
    if (!jobs) return 2;
    for (int t = 0; t < nt; ++t) jobs[t] = (job_t){d, ng, m, nv, t, nt, b, scale, pts, n, G, grid, y};
    int rc = run_jobs(jobs, nt, gather_job);
    free(jobs);
    return rc;
}
