/*
 * nlse_oracle.c -- TEST INFRASTRUCTURE ONLY (see nlse_oracle.h).
 *
 * The plain serial CPU oracle for the NLSEmagic hot path (RK4 + CD/2SHOC,
 * Dirichlet/MSD, fp32/fp64), the functional twin of the paper's serial C MEX
 * integrators.  Build (done by __graft_entry__.build()):
 *   gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o liboracle.so nlse_oracle.c -lm
 * x86-64 SSE2 arithmetic: every float / double operation is one IEEE-754
 * round-to-nearest operation in its own precision.
 */
#include <math.h>
#include <stdlib.h>
#include "nlse_oracle.h"

/* Built twice: liboracle.so (serial, the reference for every test) and, with -fopenmp,
 * liboracle_omp.so (the same sweeps split over the host cores for the all-cores CPU baseline;
 * per-point arithmetic unchanged, so the same bits -- tests/test_oracle_pins.py checks it). */
#ifdef _OPENMP
#define ORC_PARFOR _Pragma("omp parallel for schedule(static)")
#else
#define ORC_PARFOR
#endif

static int oracle_check(const oracle_problem *p)
{
    if (!p || p->ndim < 1 || p->ndim > 3) return -1;
    for (int d = 0; d < 3; d++) {
        if (d < p->ndim) { if (p->n[d] < 3) return -1; }
        else if (p->n[d] != 1) return -1;
    }
    if (!(p->h > 0) || !(p->a > 0) || !isfinite(p->s)) return -1;
    if (p->bc != 0 && p->bc != 1 && p->bc != 2) return -1;
    if (p->order != 2 && p->order != 4) return -1;
    return 0;
}

#define REAL double
#define SUF f64
#include "nlse_oracle_impl.h"
#undef REAL
#undef SUF

#define REAL float
#define SUF f32
#include "nlse_oracle_impl.h"
#undef REAL
#undef SUF

/* Kahan-compensated running sum (fp64). */
typedef struct { double s, c; } kahan;
static void kahan_add(kahan *k, double x)
{
    double y = x - k->c;
    double t = k->s + y;
    k->c = (t - k->s) - y;
    k->s = t;
}

/* Diagnostics (reading R-DIAG; the paper itself reports none):
 *   M = h^d sum_p |Psi_p|^2
 *   H = h^d sum_p [ a sum_axes |Psi_{p+e} - Psi_p|^2 / h^2   (pairs inside the grid)
 *                   + V_p |Psi_p|^2 - (s/2) |Psi_p|^4 ]
 * H is the functional whose variation gives (NLSE): i Psi_t = dH/dPsi*. */
int oracle_diag_f64(const oracle_problem *p, const double *V, const double *re, const double *im,
                    double *mass, double *ham)
{
    if (oracle_check(p) || !mass || !ham) return -1;
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    const long st[3] = {1, nx, nx * ny};
    const long nn[3] = {nx, ny, nz};
    kahan km = {0, 0}, kh = {0, 0};
    for (long k = 0; k < nz; k++)
        for (long j = 0; j < ny; j++)
            for (long i = 0; i < nx; i++) {
                const long q = (k * ny + j) * nx + i;
                const long idx[3] = {i, j, k};
                double rho = re[q] * re[q] + im[q] * im[q];
                kahan_add(&km, rho);
                double grad = 0;
                for (int d = 0; d < p->ndim; d++) {
                    if (idx[d] + 1 >= nn[d]) continue;
                    double dr = re[q + st[d]] - re[q], di = im[q + st[d]] - im[q];
                    grad += dr * dr + di * di;
                }
                double e = p->a * grad / (p->h * p->h) - 0.5 * p->s * rho * rho;
                if (V) e += V[q] * rho;
                kahan_add(&kh, e);
            }
    double hd = p->h;
    for (int d = 1; d < p->ndim; d++) hd *= p->h;
    *mass = hd * km.s;
    *ham = hd * kh.s;
    return 0;
}
