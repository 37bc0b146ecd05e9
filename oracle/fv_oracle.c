/*
 * fv_oracle.c -- CPU restatement of the reference's batched Rusanov FV step.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (libfvb.so) never
 * links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement byte-for-byte
 * against (a) golden fixtures produced by importing the reference itself
 * (oracle/gen_golden.py -> tests/golden/) and (b) the SHA-256 golden table of
 * SURVEY.md Appendix B, and (c) the reference's frozen LCG first-cell KAT
 * (pkg/tests/test_bench.py:46-69).
 *
 * It restates the SEQUENTIAL golden executor literally (run_sequential,
 * pkg/src/patchbench/executors.py:219-270): per patch, the steps
 * copy, flux_0..d-1, lambda_0..d-1, acc_0..d-1, reduce run in order over
 * their per-step ranges (kernelgraph.py:134-182), with every face flux
 * evaluated twice (once from each adjacent cell, microkernels.py:157-184),
 * exactly as the reference does.  Expression trees follow
 * equations.py:60-107 and microkernels.py:157-193 operator for operator;
 * build with -ffp-contract=off (no FMA contraction) so every binary op is
 * rounded once like numpy / Python floats.
 *
 * Layout of the batch arrays handled here: SoA over cells
 * (patchdata.py:163-165): value(k, patch, lin) at k*T*M + patch*M + lin,
 * M = m^d, m = p+2 (haloed input) or p (interior output), coordinate 0
 * fastest (patchdata.py:122-129).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* equations.py:60-74 */
static inline double ref_pressure(const double *q, int d, double gamma) {
    double ke = q[1] * q[1] + q[2] * q[2];
    if (d == 3) ke = ke + q[3] * q[3];
    return (gamma - 1.0) * (q[d + 1] - ke / (2.0 * q[0]));
}

/* equations.py:77-95 */
static inline void ref_flux(const double *q, int d, int axis, double gamma, double *f) {
    double p = ref_pressure(q, d, gamma);
    double rho = q[0];
    double energy = q[d + 1];
    double un = q[1 + axis] / rho;
    f[0] = q[1 + axis];
    for (int i = 0; i < d; ++i) f[1 + i] = (i == axis) ? q[1 + i] * un + p : q[1 + i] * un;
    f[d + 1] = un * (energy + p);
}

/* equations.py:98-107 */
static inline double ref_lambda(const double *q, int d, int axis, double gamma) {
    double p = ref_pressure(q, d, gamma);
    double rho = q[0];
    return fabs(q[1 + axis] / rho) + sqrt(gamma * p / rho);
}

/* Python builtin max(a, b): returns a unless b > a. */
static inline double py_max(double a, double b) { return (b > a) ? b : a; }

static inline int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}

/* Linearisation, coordinate 0 fastest (patchdata.py:122-129). */
static inline int64_t lin_of(const int *c, int d, int m, int shift) {
    int64_t lin = 0;
    for (int k = d - 1; k >= 0; --k) lin = lin * m + (c[k] + shift);
    return lin;
}

/* Advance the d-dim cell counter over a box [lo_k, hi_k), coordinate 0 fastest. */
static inline int next_cell(int *c, const int *lo, const int *hi, int d) {
    for (int k = 0; k < d; ++k) {
        if (++c[k] < hi[k]) return 1;
        c[k] = lo[k];
    }
    return 0;
}

/*
 * One patch, SoA batch arrays.  tmpF: d*n*M doubles, tmpL: d*M doubles
 * (full haloed cube per axis, like ScratchArrays, microkernels.py:70-77).
 * Returns the patch's max eigenvalue of the updated solution (neutral 0).
 */
static double patch_step(int d, int p, int64_t T, int64_t patch, const double *qin, double *qout,
                         double dt, double h, double gamma, int with_reduction, double *tmpF,
                         double *tmpL) {
    const int n = d + 2, m = p + 2;
    const int64_t M = ipow(m, d), Mi = ipow(p, d);
    const int64_t sin = T * M, sout = T * Mi;
    const double *qi = qin + patch * M;
    double *qo = qout + patch * Mi;
    int c[3], lo[3], hi[3];
    double q[5], f[5];

    /* COPY over [0,p)^d  (microkernels.py:124-126) */
    for (int k = 0; k < d; ++k) lo[k] = 0, hi[k] = p, c[k] = 0;
    do {
        int64_t lh = lin_of(c, d, m, 1), li = lin_of(c, d, p, 0);
        for (int k = 0; k < n; ++k) qo[k * sout + li] = qi[k * sin + lh];
    } while (next_cell(c, lo, hi, d));

    /* FLUX_a over c_a in [-1,p], others [0,p)  (microkernels.py:129-141) */
    for (int a = 0; a < d; ++a) {
        for (int k = 0; k < d; ++k) lo[k] = (k == a) ? -1 : 0, hi[k] = (k == a) ? p + 1 : p, c[k] = lo[k];
        do {
            int64_t lh = lin_of(c, d, m, 1);
            for (int k = 0; k < n; ++k) q[k] = qi[k * sin + lh];
            ref_flux(q, d, a, gamma, f);
            for (int k = 0; k < n; ++k) tmpF[((int64_t)a * n + k) * M + lh] = f[k];
        } while (next_cell(c, lo, hi, d));
    }
    /* EIGENVALUE_a (microkernels.py:144-154) */
    for (int a = 0; a < d; ++a) {
        for (int k = 0; k < d; ++k) lo[k] = (k == a) ? -1 : 0, hi[k] = (k == a) ? p + 1 : p, c[k] = lo[k];
        do {
            int64_t lh = lin_of(c, d, m, 1);
            for (int k = 0; k < n; ++k) q[k] = qi[k * sin + lh];
            tmpL[(int64_t)a * M + lh] = ref_lambda(q, d, a, gamma);
        } while (next_cell(c, lo, hi, d));
    }
    /* ACCUMULATE_a over [0,p)^d, a = 0..d-1 in order (microkernels.py:157-184) */
    const double scale = dt / h;
    for (int a = 0; a < d; ++a) {
        const int64_t stride = ipow(m, a);
        for (int k = 0; k < d; ++k) lo[k] = 0, hi[k] = p, c[k] = 0;
        do {
            int64_t lv = lin_of(c, d, m, 1), ll = lv - stride, lr = lv + stride;
            int64_t li = lin_of(c, d, p, 0);
            const double *F = tmpF + (int64_t)a * n * M;
            const double *L = tmpL + (int64_t)a * M;
            double lam_v = L[lv];
            double w_l = py_max(L[ll], lam_v);
            double w_r = py_max(lam_v, L[lr]);
            for (int k = 0; k < n; ++k) {
                double q_v = qi[k * sin + lv];
                double f_v = F[k * M + lv];
                double f_face_l = 0.5 * (F[k * M + ll] + f_v) - 0.5 * w_l * (q_v - qi[k * sin + ll]);
                double f_face_r = 0.5 * (f_v + F[k * M + lr]) - 0.5 * w_r * (qi[k * sin + lr] - q_v);
                qo[k * sout + li] = qo[k * sout + li] + scale * (f_face_l - f_face_r);
            }
        } while (next_cell(c, lo, hi, d));
    }
    /* REDUCE (microkernels.py:187-193, executors.py:263-269) */
    double red = 0.0;
    if (with_reduction) {
        for (int k = 0; k < d; ++k) lo[k] = 0, hi[k] = p, c[k] = 0;
        do {
            int64_t li = lin_of(c, d, p, 0);
            for (int k = 0; k < n; ++k) q[k] = qo[k * sout + li];
            double value = ref_lambda(q, d, 0, gamma);
            for (int a = 1; a < d; ++a) value = py_max(value, ref_lambda(q, d, a, gamma));
            if (value > red) red = value;
        } while (next_cell(c, lo, hi, d));
    }
    return red;
}

/*
 * Whole batch.  Returns the reduced eigenvalue (0.0 when with_reduction == 0,
 * the caller maps that to None).  lam_patch (optional, T doubles) receives
 * the per-patch maxima.  threads <= 0 uses the OpenMP default.
 */
double fvo_step_soa(int d, int p, int64_t T, const double *q_in, double *q_out, double dt, double h,
                    double gamma, int with_reduction, double *lam_patch, int threads) {
    const int n = d + 2;
    const int64_t M = ipow(p + 2, d);
    double red = 0.0;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    threads = 1;
#endif
#pragma omp parallel num_threads(threads) reduction(max : red)
    {
        double *tmpF = (double *)malloc(sizeof(double) * (size_t)(d * n * M));
        double *tmpL = (double *)malloc(sizeof(double) * (size_t)(d * M));
#pragma omp for schedule(static)
        for (int64_t patch = 0; patch < T; ++patch) {
            double r = patch_step(d, p, T, patch, q_in, q_out, dt, h, gamma, with_reduction, tmpF, tmpL);
            if (lam_patch) lam_patch[patch] = r;
            if (r > red) red = r;
        }
        free(tmpF);
        free(tmpL);
    }
    return red;
}

/* ---------------------------------------------------------------------
 * Seeded field (bench.py:89-133): 64-bit LCG, MMIX constants, one draw
 * sequence over patches -> haloed cells (canonical order) -> rho, u_0..u_{d-1}, p.
 * fvo_init_field_soa fills patches [p0, p0+count) of a T-patch SoA batch,
 * jumping the generator ahead to the first draw of patch p0, so shards and
 * threads reproduce the single-stream bits.
 * --------------------------------------------------------------------- */
#define LCG_A 6364136223846793005ULL
#define LCG_C 1442695040888963407ULL

/* State after `steps` applications of s -> a*s + c (mod 2^64). */
uint64_t fvo_lcg_jump(uint64_t state, uint64_t steps) {
    uint64_t acc_a = 1, acc_c = 0, a = LCG_A, c = LCG_C;
    while (steps) {
        if (steps & 1) {
            acc_a = acc_a * a;
            acc_c = acc_c * a + c;
        }
        c = (a + 1) * c;
        a = a * a;
        steps >>= 1;
    }
    return acc_a * state + acc_c;
}

static inline double lcg_uniform(uint64_t *s, double lo, double hi) {
    *s = *s * LCG_A + LCG_C;
    return lo + (hi - lo) * ((double)(*s >> 11) * 0x1p-53);
}

void fvo_init_field_soa(int d, int p, int64_t T, uint64_t seed, double gamma, double *q_in,
                        int64_t p0, int64_t count, int threads) {
    const int n = d + 2;
    const int64_t M = ipow(p + 2, d);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    threads = 1;
#endif
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t patch = p0; patch < p0 + count; ++patch) {
        uint64_t s = fvo_lcg_jump(seed, (uint64_t)(patch * M * n));
        for (int64_t lin = 0; lin < M; ++lin) {
            double rho = lcg_uniform(&s, 0.5, 2.0);
            double u[3] = {0.0, 0.0, 0.0};
            for (int i = 0; i < d; ++i) u[i] = lcg_uniform(&s, -0.5, 0.5);
            double pr = lcg_uniform(&s, 0.5, 2.0);
            double ke = u[0] * u[0] + u[1] * u[1];
            if (d == 3) ke = ke + u[2] * u[2];
            int64_t at = patch * M + lin;
            q_in[at] = rho;
            for (int i = 0; i < d; ++i) q_in[(int64_t)(1 + i) * T * M + at] = rho * u[i];
            q_in[(int64_t)(d + 1) * T * M + at] = pr / (gamma - 1.0) + 0.5 * rho * ke;
        }
    }
}

int fvo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
