/*
 * sb_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the reference stencil sweeps
 * (arxiv 1004.1741 / package `stencilbench`).  Nothing in the product path
 * (paper_1004_1741_b200/, libsb200.so) links or calls this file; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg load it, as the checker or as the timed CPU baseline.
 *
 * Parity is pinned: tests/test_oracle.py checks every function below
 * bit-for-bit against the tests/golden fixtures, which tests/golden/make_golden.py
 * produced by running the reference package itself (numba kernels).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: the reference kernels
 * are strict IEEE, no FMA contraction -- SURVEY.md finding 2).
 *
 * Layout (reference pkg/src/stencilbench/grid.py:61-91): a grid is
 * (nk+2) x (nj+2) x (ni+2) doubles, i unit stride; interior (k,j,i) lives at
 * padded (k+1, j+1, i+1).  Halo cells hold Dirichlet values, never written.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { SBO_JACOBI = 0, SBO_GS_NAIVE = 1, SBO_GS_INTERLEAVED = 2 };

/* Plane-window kernels.  km/kc/kp: padded planes k-1, k, k+1 with row pitch
 * nip = ni+2; rows [jp0, jp1) in padded j coordinates; the i loop covers
 * the full interior.                                                      */

/* reference kernels.py:125-134 (_jacobi_window_nb) / :61-70 (numpy).
 * dst = a*c + b*(((((W+E)+S)+N)+D)+U), left to right. */
void sbo_jacobi_window(double *dst, const double *km, const double *kc,
                       const double *kp, int64_t nip, double a, double b,
                       int64_t jp0, int64_t jp1)
{
    for (int64_t j = jp0; j < jp1; ++j) {
        const double *c = kc + j * nip, *s = c - nip, *n = c + nip;
        const double *d = km + j * nip, *u = kp + j * nip;
        double *o = dst + j * nip;
        for (int64_t i = 1; i < nip - 1; ++i) {
            double acc = c[i - 1] + c[i + 1];
            acc = acc + s[i];
            acc = acc + n[i];
            acc = acc + d[i];
            acc = acc + u[i];
            o[i] = a * c[i] + b * acc;
        }
    }
}

/* reference kernels.py:154-163 (_gs_window_nb): in place, i ascending. */
void sbo_gs_window(const double *km, double *kc, const double *kp,
                   int64_t nip, double b, int64_t jp0, int64_t jp1)
{
    for (int64_t j = jp0; j < jp1; ++j) {
        double *c = kc + j * nip;
        const double *s = c - nip, *n = c + nip;
        const double *d = km + j * nip, *u = kp + j * nip;
        for (int64_t i = 1; i < nip - 1; ++i) {
            double acc = c[i - 1] + c[i + 1];
            acc = acc + s[i];
            acc = acc + n[i];
            acc = acc + d[i];
            acc = acc + u[i];
            c[i] = b * acc;
        }
    }
}

/* reference kernels.py:165-187 (_gs_window_interleaved_nb): the five
 * non-recursive terms of cell i+1 are summed one cell ahead
 * (tmp = (((E+S)+N)+D)+U) and x_i = b*(W + tmp).  ni < 2 -> naive. */
void sbo_gs_window_interleaved(const double *km, double *kc, const double *kp,
                               int64_t nip, double b, int64_t jp0, int64_t jp1)
{
    if (nip - 2 < 2) {
        sbo_gs_window(km, kc, kp, nip, b, jp0, jp1);
        return;
    }
    for (int64_t j = jp0; j < jp1; ++j) {
        double *c = kc + j * nip;
        const double *s = c - nip, *n = c + nip;
        const double *d = km + j * nip, *u = kp + j * nip;
        double tmp1 = (((c[2] + s[1]) + n[1]) + d[1]) + u[1];
        double tmp2 = 0.0;
        for (int64_t i = 1; i < nip - 1; ++i) {
            if (i + 1 < nip - 1)
                tmp2 = (((c[i + 2] + s[i + 1]) + n[i + 1]) + d[i + 1]) + u[i + 1];
            c[i] = b * (c[i - 1] + tmp1);
            tmp1 = tmp2;
        }
    }
}

static void gs_win(int kernel, const double *km, double *kc, const double *kp,
                   int64_t nip, double b, int64_t jp0, int64_t jp1)
{
    if (kernel == SBO_GS_INTERLEAVED)
        sbo_gs_window_interleaved(km, kc, kp, nip, b, jp0, jp1);
    else
        sbo_gs_window(km, kc, kp, nip, b, jp0, jp1);
}

/* reference sweeps/serial.py:8-42.  Jacobi ping-pongs g and scratch (the
 * scratch is initialised here as a full copy of g, like g.copy(), so the
 * Dirichlet halo persists in both).  Returns 1 when the final field lives
 * in `scratch` (odd Jacobi iteration counts), else 0.  GS runs in place. */
int sbo_run_serial(int kernel, double *g, double *scratch, int64_t ni,
                   int64_t nj, int64_t nk, int64_t iters, double a, double b)
{
    const int64_t nip = ni + 2, njp = nj + 2, plane = nip * njp;
    if (iters == 0)
        return 0;
    if (kernel == SBO_JACOBI) {
        memcpy(scratch, g, (size_t)(plane * (nk + 2)) * sizeof(double));
        double *src = g, *dst = scratch;
        for (int64_t s = 0; s < iters; ++s) {
            for (int64_t k = 0; k < nk; ++k)
                sbo_jacobi_window(dst + (k + 1) * plane, src + k * plane,
                                  src + (k + 1) * plane, src + (k + 2) * plane,
                                  nip, a, b, 1, njp - 1);
            double *t = src; src = dst; dst = t;
        }
        return src == scratch;
    }
    for (int64_t s = 0; s < iters; ++s)
        for (int64_t k = 0; k < nk; ++k)
            gs_win(kernel, g + k * plane, g + (k + 1) * plane, g + (k + 2) * plane,
                   nip, b, 1, njp - 1);
    return 0;
}

/* reference sweeps/plan.py:106-120: contiguous, sizes differ by <= 1,
 * larger blocks first. */
static void partition(int64_t extent, int count, int idx, int64_t *lo, int64_t *hi)
{
    int64_t base = extent / count, rem = extent % count;
    *lo = idx * base + (idx < rem ? idx : rem);
    *hi = *lo + base + (idx < rem ? 1 : 0);
}

typedef struct {
    int kernel, rank, p;
    double *bufs[2];
    int64_t ni, nj, nk, iters;
    double a, b;
    pthread_barrier_t *bar;
} team_arg;

/* reference sweeps/threaded.py:28-59: k-slabs per thread, one barrier per
 * sweep, ping-pong. */
static void *jacobi_worker(void *vp)
{
    team_arg *t = vp;
    const int64_t nip = t->ni + 2, njp = t->nj + 2, plane = nip * njp;
    int64_t k_lo, k_hi;
    partition(t->nk, t->p, t->rank, &k_lo, &k_hi);
    for (int64_t s = 0; s < t->iters; ++s) {
        const double *sd = t->bufs[s & 1];
        double *dd = t->bufs[(s + 1) & 1];
        for (int64_t k = k_lo; k < k_hi; ++k)
            sbo_jacobi_window(dd + (k + 1) * plane, sd + k * plane,
                              sd + (k + 1) * plane, sd + (k + 2) * plane,
                              nip, t->a, t->b, 1, njp - 1);
        pthread_barrier_wait(t->bar);
    }
    return NULL;
}

/* reference sweeps/threaded.py:62-96: j-blocks per thread; at stage s the
 * thread of rank p updates plane s-p; nk+P-1 stages per sweep, a barrier
 * after every stage: the exact serial lexicographic order. */
static void *pipeline_worker(void *vp)
{
    team_arg *t = vp;
    const int64_t nip = t->ni + 2, plane = nip * (t->nj + 2);
    int64_t j_lo, j_hi;
    partition(t->nj, t->p, t->rank, &j_lo, &j_hi);
    double *d = t->bufs[0];
    const int64_t stages = t->nk + t->p - 1;
    for (int64_t s = 0; s < t->iters; ++s) {
        for (int64_t st = 0; st < stages; ++st) {
            int64_t k = st - t->rank;
            if (k >= 0 && k < t->nk)
                gs_win(t->kernel, d + k * plane, d + (k + 1) * plane,
                       d + (k + 2) * plane, nip, t->b, j_lo + 1, j_hi + 1);
            pthread_barrier_wait(t->bar);
        }
    }
    return NULL;
}

static int run_team(void *(*fn)(void *), int kernel, double *g, double *scratch,
                    int64_t ni, int64_t nj, int64_t nk, int64_t iters,
                    double a, double b, int p)
{
    pthread_t *th = calloc((size_t)p, sizeof(pthread_t));
    team_arg *args = calloc((size_t)p, sizeof(team_arg));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)p);
    for (int r = 0; r < p; ++r) {
        args[r] = (team_arg){kernel, r, p, {g, scratch}, ni, nj, nk, iters, a, b, &bar};
        if (r > 0)
            pthread_create(&th[r], NULL, fn, &args[r]);
    }
    fn(&args[0]);
    for (int r = 1; r < p; ++r)
        pthread_join(th[r], NULL);
    pthread_barrier_destroy(&bar);
    free(th);
    free(args);
    return 0;
}

/* Returns 1 when the result is in scratch, 0 when in g, -1 on a partition
 * error (p > nk), mirroring run_threaded_jacobi's PartitionError. */
int sbo_run_threaded_jacobi(double *g, double *scratch, int64_t ni, int64_t nj,
                            int64_t nk, int64_t iters, double a, double b, int p)
{
    if (p < 1 || p > nk)
        return -1;
    if (iters == 0)
        return 0;
    memcpy(scratch, g, (size_t)((ni + 2) * (nj + 2) * (nk + 2)) * sizeof(double));
    run_team(jacobi_worker, SBO_JACOBI, g, scratch, ni, nj, nk, iters, a, b, p);
    return (int)(iters & 1);
}

int sbo_run_pipeline_gs(int kernel, double *g, int64_t ni, int64_t nj, int64_t nk,
                        int64_t iters, double b, int p)
{
    if (p < 1 || p > nj)
        return -1;
    if (iters == 0)
        return 0;
    run_team(pipeline_worker, kernel, g, NULL, ni, nj, nk, iters, 0.0, b, p);
    return 0;
}
