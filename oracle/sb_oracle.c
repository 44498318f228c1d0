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

/* ------------------------------------------------------------------------
 * Wavefront temporal blocking (reference sweeps/wavefront.py:127-376): the
 * paper's shared-cache wavefront engines, restated schedule for schedule so
 * they can be timed as the reference's best CPU variant (bench.py's CPU
 * baseline) -- n groups of t threads, one barrier per plane phase, B
 * j-blocks walked round robin, parallelogram-skewed windows; Jacobi with a
 * 2t-plane ring per group and interface lines carried between blocks.
 * Bitwise equal to run_serial (the reference pins that in its own tests;
 * tests/test_oracle.py pins this port against the serial oracle). */

/* reference kernels.py:136-152: row jp0 takes its j-1 neighbour from ov */
static void jacobi_window_jlow(double *dst, const double *km, const double *kc,
                               const double *kp, const double *ov, int64_t nip,
                               double a, double b, int64_t jp0, int64_t jp1)
{
    if (jp1 <= jp0)
        return;
    const double *c = kc + jp0 * nip, *n = c + nip;
    const double *d = km + jp0 * nip, *u = kp + jp0 * nip;
    double *o = dst + jp0 * nip;
    for (int64_t i = 1; i < nip - 1; ++i) {
        double acc = c[i - 1] + c[i + 1];
        acc = acc + ov[i];
        acc = acc + n[i];
        acc = acc + d[i];
        acc = acc + u[i];
        o[i] = a * c[i] + b * acc;
    }
    sbo_jacobi_window(dst, km, kc, kp, nip, a, b, jp0 + 1, jp1);
}

typedef struct {
    int kernel, t, n, nblocks, steps, writers, rows, spw;
    int64_t ni, nj, nk, nip, njp, plane, length, span, phases, delta;
    int64_t *blk;           /* nblocks x (start, end) */
    double *g, a, b;
    double *rings;          /* n x 2t planes */
    double *bounds;         /* n x writers x 2 x rows x nk x nip */
    pthread_barrier_t *bar;
} wf_ctx;

typedef struct {
    wf_ctx *c;
    int idx;
} wf_arg;

static void wf_window(int64_t start, int64_t end, int64_t shift, int64_t nj, int64_t *w0, int64_t *w1)
{
    *w0 = start - shift > 0 ? start - shift : 0;
    *w1 = end - shift < nj ? end - shift : nj;
}

static double *wf_slot(wf_ctx *c, int gid, int writer, int64_t k)
{
    return c->rings + ((int64_t)gid * 2 * c->t + writer * c->spw + k % c->spw) * c->plane;
}

/* boundary line (group, writer, parity, row, plane k) */
static double *wf_bline(wf_ctx *c, int group, int writer, int parity, int row, int64_t k)
{
    int64_t off = ((((int64_t)group * c->writers + writer) * 2 + parity) * c->rows + row) * c->nk + k;
    return c->bounds + off * c->nip;
}

static double *wf_outgoing(wf_ctx *c, int gid, int w, int64_t q, int row, int64_t k)
{
    return wf_bline(c, gid, w, (int)((q / c->n) % 2), row, k);
}

static double *wf_incoming(wf_ctx *c, int64_t q, int w, int row, int64_t k)
{
    return wf_bline(c, (int)((q - 1) % c->n), w, (int)(((q - 1) / c->n) % 2), row, k);
}

static void wf_jacobi_even(wf_ctx *c, int gid, int r, int64_t q, int64_t k, int64_t start, int64_t end)
{
    int64_t w0, w1, cw0, cw1;
    const int64_t nip = c->nip, njp = c->njp, nj = c->nj;
    wf_window(start, end, r, nj, &w0, &w1);
    wf_window(start, end, r + 1, nj, &cw0, &cw1);
    if (w1 <= w0 && cw1 <= cw0)
        return;
    const int w = r / 2;
    double *slot = wf_slot(c, gid, w, k);
    const double *sd = c->g, *srcp = sd + (k + 1) * c->plane;
    memcpy(slot, srcp, nip * sizeof(double));
    memcpy(slot + (njp - 1) * nip, srcp + (njp - 1) * nip, nip * sizeof(double));
    if (q >= 1) {
        const int64_t rows[2] = {start - r - 2, start - r - 1};
        for (int bi = 0; bi < 2; ++bi)
            if (rows[bi] >= 0 && rows[bi] < nj)
                memcpy(slot + (rows[bi] + 1) * nip, wf_incoming(c, q, w, bi, k), nip * sizeof(double));
    }
    for (int64_t j = cw0 + 1; j < cw1 + 1; ++j) {
        slot[j * nip] = srcp[j * nip];
        slot[j * nip + nip - 1] = srcp[j * nip + nip - 1];
    }
    if (w1 > w0)
        sbo_jacobi_window(slot, sd + k * c->plane, srcp, sd + (k + 2) * c->plane, nip, c->a, c->b,
                          w0 + 1, w1 + 1);
    const int64_t rows[2] = {end - r - 2, end - r - 1};
    for (int bi = 0; bi < 2; ++bi)
        if (rows[bi] >= 0 && rows[bi] < nj) {
            const double *from = (w0 <= rows[bi] && rows[bi] < w1)
                                      ? slot + (rows[bi] + 1) * nip
                                      : wf_incoming(c, q, w, 1, k); /* width-1 block */
            memcpy(wf_outgoing(c, gid, w, q, bi, k), from, nip * sizeof(double));
        }
}

static void wf_jacobi_odd(wf_ctx *c, int gid, int r, int64_t k, int64_t start, int64_t end)
{
    int64_t w0, w1;
    wf_window(start, end, r, c->nj, &w0, &w1);
    if (w1 <= w0)
        return;
    const int w = (r - 1) / 2;
    double *sd = c->g;
    const double *rd[3];
    for (int d = 0; d < 3; ++d) {
        int64_t kq = k - 1 + d;
        rd[d] = (kq >= 0 && kq < c->nk) ? wf_slot(c, gid, w, kq) : sd + (kq + 1) * c->plane;
    }
    sbo_jacobi_window(sd + (k + 1) * c->plane, rd[0], rd[1], rd[2], c->nip, c->a, c->b, w0 + 1, w1 + 1);
}

static void wf_jacobi_t1(wf_ctx *c, int gid, int64_t q, int64_t pi, int64_t start, int64_t end)
{
    double *sd = c->g;
    const int64_t nip = c->nip, plane = c->plane;
    if (pi < c->nk) {
        const int64_t k = pi;
        double *slot = wf_slot(c, gid, 0, k);
        if (q >= 1)
            jacobi_window_jlow(slot, sd + k * plane, sd + (k + 1) * plane, sd + (k + 2) * plane,
                               wf_incoming(c, q, 0, 0, k), nip, c->a, c->b, start + 1, end + 1);
        else
            sbo_jacobi_window(slot, sd + k * plane, sd + (k + 1) * plane, sd + (k + 2) * plane, nip,
                              c->a, c->b, start + 1, end + 1);
    }
    const int64_t kk = pi - 1;
    if (kk >= 0 && kk < c->nk) {
        /* save the pre-update top line, then retire the plane in place */
        memcpy(wf_outgoing(c, gid, 0, q, 0, kk), sd + (kk + 1) * plane + end * nip, nip * sizeof(double));
        const double *slot = wf_slot(c, gid, 0, kk);
        for (int64_t j = start + 1; j < end + 1; ++j)
            memcpy(sd + (kk + 1) * plane + j * nip + 1, slot + j * nip + 1, (nip - 2) * sizeof(double));
    }
}

static void *wf_worker(void *vp)
{
    wf_arg *arg = vp;
    wf_ctx *c = arg->c;
    const int gid = arg->idx / c->t, r = arg->idx % c->t;
    const int64_t my_delay = c->delta * gid;
    for (int64_t phi = 0; phi < c->phases; ++phi) {
        const int64_t local = phi - my_delay;
        if (local >= 0 && local < c->span) {
            const int64_t sg = local / c->length, pi = local % c->length;
            const int64_t q = (sg % c->steps) * c->n + gid;
            if (q < c->nblocks) {
                const int64_t start = c->blk[2 * q], end = c->blk[2 * q + 1];
                const int64_t k = pi - 2 * r;
                if (c->kernel == SBO_JACOBI) {
                    if (c->t == 1)
                        wf_jacobi_t1(c, gid, q, pi, start, end);
                    else if (k >= 0 && k < c->nk) {
                        if (r % 2 == 0)
                            wf_jacobi_even(c, gid, r, q, k, start, end);
                        else
                            wf_jacobi_odd(c, gid, r, k, start, end);
                    }
                } else if (k >= 0 && k < c->nk) {
                    int64_t w0, w1;
                    wf_window(start, end, r, c->nj, &w0, &w1);
                    if (w1 > w0)
                        gs_win(c->kernel, c->g + k * c->plane, c->g + (k + 1) * c->plane,
                               c->g + (k + 2) * c->plane, c->nip, c->b, w0 + 1, w1 + 1);
                }
            }
        }
        pthread_barrier_wait(c->bar);
    }
    return NULL;
}

/* reference sweeps/wavefront.py:160-376 (run_wavefront): n groups x t
 * threads, B j-blocks.  Returns the number of barrier phases (the
 * reference's stats["barrier_phases"]), or -1 on a plan error (iters % t,
 * odd t > 1 for Jacobi, B < 1 or B > nj). */
int64_t sbo_run_wavefront(int kernel, double *g, int64_t ni, int64_t nj, int64_t nk,
                          int64_t iters, double a, double b, int n, int t, int B)
{
    if (n < 1 || t < 1 || B < 1 || B > nj || iters % t != 0)
        return -1;
    if (kernel == SBO_JACOBI && t > 1 && t % 2)
        return -1;
    if (iters == 0)
        return 0;
    wf_ctx c;
    memset(&c, 0, sizeof c);
    c.kernel = kernel;
    c.t = t;
    c.n = n;
    c.ni = ni;
    c.nj = nj;
    c.nk = nk;
    c.nip = ni + 2;
    c.njp = nj + 2;
    c.plane = c.nip * c.njp;
    c.g = g;
    c.a = a;
    c.b = b;
    c.nblocks = B + (t >= 2 ? 1 : 0); /* + drain pseudo-block */
    c.blk = malloc(sizeof(int64_t) * 2 * (size_t)c.nblocks);
    for (int q = 0; q < B; ++q)
        partition(nj, B, q, &c.blk[2 * q], &c.blk[2 * q + 1]);
    if (t >= 2) {
        c.blk[2 * B] = nj;
        c.blk[2 * B + 1] = nj + t - 1;
    }
    c.steps = (c.nblocks + n - 1) / n;
    const int64_t rounds = iters / t;
    if (kernel == SBO_JACOBI) {
        c.delta = 2;
        c.length = t >= 2 ? nk + 2 * (t - 1) : nk + 1;
    } else {
        c.delta = 1;
        c.length = nk + 2 * (t - 1);
    }
    if (n > 1 && c.length < c.delta * (n - 1) + 2)
        c.length = c.delta * (n - 1) + 2;
    c.span = rounds * c.steps * c.length;
    c.phases = c.span + c.delta * (n - 1);
    if (kernel == SBO_JACOBI) {
        c.writers = t / 2 > 1 ? t / 2 : 1;
        c.rows = t >= 2 ? 2 : 1;
        c.spw = t >= 2 ? 4 : 2;
        c.rings = calloc((size_t)n * 2 * t * c.plane, sizeof(double));
        c.bounds = calloc((size_t)n * c.writers * 2 * c.rows * nk * c.nip, sizeof(double));
    }
    const int p = n * t;
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)p);
    c.bar = &bar;
    pthread_t *th = calloc((size_t)p, sizeof(pthread_t));
    wf_arg *args = calloc((size_t)p, sizeof(wf_arg));
    for (int i = 0; i < p; ++i) {
        args[i].c = &c;
        args[i].idx = i;
        if (i > 0)
            pthread_create(&th[i], NULL, wf_worker, &args[i]);
    }
    wf_worker(&args[0]);
    for (int i = 1; i < p; ++i)
        pthread_join(th[i], NULL);
    pthread_barrier_destroy(&bar);
    free(th);
    free(args);
    free(c.rings);
    free(c.bounds);
    free(c.blk);
    return c.phases;
}
