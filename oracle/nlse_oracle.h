/*
 * nlse_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, serial CPU oracle for the RK4 + CD / 2SHOC time step of the
 * cubic NLSE / GPE  i Psi_t + a Lap(Psi) - V Psi + s|Psi|^2 Psi = 0
 * (PAPER.md (NLSE) P:76-80), written directly from the paper.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_1203_1263_b200/) never links, imports or calls it, and it shares no
 * code, header, table or constant with the CUDA path.
 *
 * Layout: split real / imaginary arrays (the paper's serial MEX layout,
 * (fsplit) P:423-429), x fastest: offset(i,j,k) = (k*ny + j)*nx + i.
 *
 * All functions return 0 on success, a negative value on a bad argument.
 */
#ifndef NLSE_ORACLE_H
#define NLSE_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int ndim;       /* 1, 2 or 3 */
    long n[3];      /* nx, ny, nz (unused dims = 1) */
    double h;       /* grid spacing, same in every direction */
    double a;       /* dispersion coefficient, a > 0 */
    double s;       /* nonlinearity coefficient */
    int bc;         /* 0 = Dirichlet, 1 = MSD, 2 = L0 */
    int order;      /* 2 = CD, 4 = 2SHOC */
} oracle_problem;

/* nsteps RK4 steps in place, literal (RK4) schedule P:164-180. V may be NULL (V = 0). */
int oracle_step_f64(const oracle_problem *p, const double *V, double *re, double *im,
                    double k, long nsteps);
int oracle_step_f32(const oracle_problem *p, const float *V, float *re, float *im,
                    double k, long nsteps);

/* F(Y) at every grid point (interior: (fsplit); boundary: time-derivative BC form). */
int oracle_rhs_f64(const oracle_problem *p, const double *V, const double *yr, const double *yi,
                   double *fr, double *fi);
int oracle_rhs_f32(const oracle_problem *p, const float *V, const float *yr, const float *yi,
                   float *fr, float *fi);

/* The Laplacian pieces: D (step 1, interior; 2SHOC: boundary faces from the Laplacian-form
 * BC, NaN on domain edges/corners where the scheme never needs it; CD: NaN on the whole
 * boundary) and L (interior only; boundary entries set to NaN). */
int oracle_lap_f64(const oracle_problem *p, const double *V, const double *yr, const double *yi,
                   double *dr, double *di, double *lr, double *li);
int oracle_lap_f32(const oracle_problem *p, const float *V, const float *yr, const float *yi,
                   float *dr, float *di, float *lr, float *li);

/* Mass M = h^d sum |Psi|^2 and Hamiltonian H (reading R-DIAG), fp64 Kahan sums. */
int oracle_diag_f64(const oracle_problem *p, const double *V, const double *re, const double *im,
                    double *mass, double *ham);

#ifdef __cplusplus
}
#endif
#endif
