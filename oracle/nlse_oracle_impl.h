/*
 * nlse_oracle_impl.h -- TEST INFRASTRUCTURE ONLY (see nlse_oracle.h).
 *
 * Included twice by nlse_oracle.c, with REAL = double / SUF = f64 and
 * REAL = float / SUF = f32: a run in single precision is single precision
 * throughout, as the paper's single-precision integrators.
 *
 * Every arithmetic expression below is written in the association order
 * DESIGN.md section "Readings" fixes (R-ASSOC); the paper gives the formulas
 * but not the association.  Compiled with -O2 -ffp-contract=off (no FMA
 * contraction), no fast-math, SSE2 (no x87 extended precision), no FTZ/DAZ.
 */

#define ORC_CAT2(a, b) a##_##b
#define ORC_CAT(a, b) ORC_CAT2(a, b)
#define FN(name) ORC_CAT(name, SUF)
/* ORC_PARFOR (nlse_oracle.c): "omp parallel for" on the outermost loop of each sweep when the
 * oracle is built with -fopenmp (liboracle_omp.so, the all-cores CPU baseline of SURVEY §8(d)),
 * nothing otherwise.  Every point's arithmetic is the same either way (the sweeps write each
 * point once from values of the previous sweep), so both builds give the same bits. */

/* Constants: evaluated in double from the user's double parameters, then
 * rounded once to REAL (reading R-CONST). */
typedef struct {
    REAL ih2;    /* 1/h^2                 (2shoc1d) P:197 */
    REAL c76;    /* 7/6                   (2shoc1d2) P:198 */
    REAL c112;   /* 1/12 */
    REAL c16h2;  /* 1/(6 h^2) */
    REAL a;      /* a                     (NLSE) P:78 */
    REAL s;      /* s                     (NLSE) P:78 */
    REAL inv_a;  /* 1/a                   (BCDlap) P:322, (BCMSDlap) P:338 */
    REAL eps2;   /* MSD division guard    reading R-MSD-GUARD */
} FN(oracle_consts);

/* Fused multiply-add, one IEEE rounding (C99 fma / fmaf): the canonical DAG contracts a
 * product into a following add at the positions listed in DESIGN.md reading R-ASSOC
 * (the CUDA side uses the same explicit fused operations, so both stay bit-identical). */
static REAL FN(fmar)(REAL a, REAL b, REAL c)
{
    return sizeof(REAL) == 8 ? (REAL)fma((double)a, (double)b, (double)c) : (REAL)fmaf((float)a, (float)b, (float)c);
}

static FN(oracle_consts) FN(make_consts)(const oracle_problem *p)
{
    FN(oracle_consts) c;
    c.ih2 = (REAL)(1.0 / (p->h * p->h));
    c.c76 = (REAL)(7.0 / 6.0);
    c.c112 = (REAL)(1.0 / 12.0);
    c.c16h2 = (REAL)(1.0 / (6.0 * p->h * p->h));
    c.a = (REAL)p->a;
    c.s = (REAL)p->s;
    c.inv_a = (REAL)(1.0 / p->a);
    c.eps2 = (sizeof(REAL) == 8) ? (REAL)1e-24 : (REAL)1e-12;
    return c;
}

/* ---------------------------------------------------------------------------
 * 2SHOC step 1 / CD: D = Delta_2 Y / h^2 at interior points, one component.
 *   1D (2shoc1d) P:197; 2D (2d2shocs1) P:202-210; 3D (3d2shocs) P:232-253;
 *   "The standard second-order central differencing ... is simply given by
 *   step one" P:301.
 * Written per axis in difference form ((Y_- + Y_+) - 2Y), axes in x, y, z
 * order (reading R-ASSOC).
 * ------------------------------------------------------------------------- */
static void FN(d_interior)(const oracle_problem *p, const FN(oracle_consts) *c,
                           const REAL *y, REAL *d)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    const long sx = 1, sy = nx, sz = nx * ny;
    if (p->ndim == 1) {
        ORC_PARFOR
        for (long i = 1; i < nx - 1; i++) {
            REAL y2 = y[i] + y[i];
            d[i] = ((y[i - sx] + y[i + sx]) - y2) * c->ih2;
        }
    } else if (p->ndim == 2) {
        ORC_PARFOR
        for (long j = 1; j < ny - 1; j++)
            for (long i = 1; i < nx - 1; i++) {
                long q = j * sy + i;
                REAL y2 = y[q] + y[q];
                d[q] = (((y[q - sx] + y[q + sx]) - y2) + ((y[q - sy] + y[q + sy]) - y2)) * c->ih2;
            }
    } else {
        ORC_PARFOR
        for (long k = 1; k < nz - 1; k++)
            for (long j = 1; j < ny - 1; j++)
                for (long i = 1; i < nx - 1; i++) {
                    long q = k * sz + j * sy + i;
                    REAL y2 = y[q] + y[q];
                    d[q] = ((((y[q - sx] + y[q + sx]) - y2) + ((y[q - sy] + y[q + sy]) - y2))
                            + ((y[q - sz] + y[q + sz]) - y2)) * c->ih2;
                }
    }
}

/* Is (i,j,k) on the domain boundary ("b represents a boundary point", P:314;
 * reading R-BND: any active index equal to 0 or n-1)? Returns the number of
 * active axes on which it is a boundary index. */
static int FN(n_bnd_axes)(const oracle_problem *p, long i, long j, long k)
{
    int m = 0;
    if (i == 0 || i == p->n[0] - 1) m++;
    if (p->ndim >= 2 && (j == 0 || j == p->n[1] - 1)) m++;
    if (p->ndim >= 3 && (k == 0 || k == p->n[2] - 1)) m++;
    return m;
}

/* Step one index inward along every boundary axis (MSD "b-1"; at
 * domain edges/corners the diagonal inward neighbour, reading R-MSD-NBR). */
static long FN(inward)(const oracle_problem *p, long i, long j, long k)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    if (i == 0) i = 1; else if (i == nx - 1) i = nx - 2;
    if (p->ndim >= 2) { if (j == 0) j = 1; else if (j == ny - 1) j = ny - 2; }
    if (p->ndim >= 3) { if (k == 0) k = 1; else if (k == nz - 1) k = nz - 2; }
    return (k * ny + j) * nx + i;
}

/* N = s|Y|^2 - V  ((nbnb1) P:341-344). */
static REAL FN(nlin)(const FN(oracle_consts) *c, const REAL *V, long q, REAL yr, REAL yi)
{
    REAL rho = (yr * yr) + (yi * yi);
    REAL n = c->s * rho;
    if (V) n = n - V[q];
    return n;
}

/* ---------------------------------------------------------------------------
 * Boundary values of D for 2SHOC step 2 -- the Laplacian form of the BC
 * ("they additionally need to be expressed in terms of the Laplacian in order
 * to compute proper boundaries in the first step of the 2SHOC").
 *   Dirichlet (BCDlap) P:320-323:  Lap Psi_b = -(1/a)(s|Psi_b|^2 - V_b) Psi_b
 *   MSD      (BCMSDlap) P:336-344: Lap Psi_b = [Im(i Lap Psi_{b-1}/Psi_{b-1})
 *                                     + (N_{b-1} - N_b)/a] Psi_b
 *     with Im(i z) = Re z (reading R-MSD-LAP), and Lap Psi_{b-1} = D_{b-1}.
 *   L0       (BCL0lap) P:352-355:  Lap Psi_b = 0 ("by definition").
 * Only boundary points with exactly one boundary axis (faces) are reachable
 * from 2SHOC step 2 at an interior point; edges and corners are set to NaN so
 * that any use poisons the result (reading R-DFACE).
 * ------------------------------------------------------------------------- */
static void FN(d_boundary)(const oracle_problem *p, const FN(oracle_consts) *c, const REAL *V,
                           const REAL *yr, const REAL *yi, REAL *dr, REAL *di)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    ORC_PARFOR
    for (long k = 0; k < nz; k++)
        for (long j = 0; j < ny; j++)
            for (long i = 0; i < nx; i++) {
                int m = FN(n_bnd_axes)(p, i, j, k);
                if (m == 0) continue;
                long q = (k * ny + j) * nx + i;
                if (m > 1) { dr[q] = (REAL)NAN; di[q] = (REAL)NAN; continue; }
                if (p->bc == 2) { dr[q] = 0; di[q] = 0; continue; }
                REAL nb = FN(nlin)(c, V, q, yr[q], yi[q]);
                if (p->bc == 0) {
                    REAL t = c->inv_a * nb;
                    dr[q] = -(t * yr[q]);
                    di[q] = -(t * yi[q]);
                } else {
                    long b1 = FN(inward)(p, i, j, k);   /* the face's inward normal neighbour */
                    REAL rho1 = (yr[b1] * yr[b1]) + (yi[b1] * yi[b1]);
                    REAL re_q = 0;
                    if (!(rho1 < c->eps2))
                        re_q = ((dr[b1] * yr[b1]) + (di[b1] * yi[b1])) / rho1;
                    REAL n1 = FN(nlin)(c, V, b1, yr[b1], yi[b1]);
                    REAL g = re_q + ((n1 - nb) * c->inv_a);
                    dr[q] = g * yr[q];
                    di[q] = g * yi[q];
                }
            }
}

/* ---------------------------------------------------------------------------
 * 2SHOC step 2 at interior points, one component (CD: L = D).
 *   1D (2shoc1d2) P:198:  L = (7/6) D_i - (1/12)(D_{i+1} + D_{i-1})
 *   2D (2d2shocs2) P:214-228:
 *       L = -(1/12)[sum of 4 face-neighbour D - 12 D] + 1/(6h^2)[4 corner Y - 4 Y]
 *   3D (3d2shocs2) P:257-299:
 *       L = -(1/12)[sum of 6 face-neighbour D - 10 D] + 1/(6h^2)[12 edge Y - 12 Y]
 *       (the 12 edge points are the diagonal neighbours in the xy, xz and yz
 *       planes; the 8 cube corners are not used)
 * The Y cross term is grouped per coordinate plane, each plane's four
 * diagonal neighbours summed in pairs minus 4Y (reading R-ASSOC).
 * ------------------------------------------------------------------------- */
static void FN(l_interior)(const oracle_problem *p, const FN(oracle_consts) *c,
                           const REAL *y, const REAL *d, REAL *l)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    const long sx = 1, sy = nx, sz = nx * ny;
    const REAL four = 4, ten = 10, twelve = 12;
    if (p->ndim == 1) {
        ORC_PARFOR
        for (long i = 1; i < nx - 1; i++)
            l[i] = (p->order == 2) ? d[i]
                 : FN(fmar)(c->c76, d[i], -(c->c112 * (d[i - sx] + d[i + sx])));
    } else if (p->ndim == 2) {
        ORC_PARFOR
        for (long j = 1; j < ny - 1; j++)
            for (long i = 1; i < nx - 1; i++) {
                long q = j * sy + i;
                if (p->order == 2) { l[q] = d[q]; continue; }
                REAL y4 = four * y[q];
                REAL cxy = ((y[q - sx - sy] + y[q + sx - sy]) + (y[q - sx + sy] + y[q + sx + sy])) - y4;
                REAL td = FN(fmar)(-twelve, d[q], (d[q - sx] + d[q + sx]) + (d[q - sy] + d[q + sy]));
                l[q] = FN(fmar)(c->c16h2, cxy, -(c->c112 * td));
            }
    } else {
        ORC_PARFOR
        for (long k = 1; k < nz - 1; k++)
            for (long j = 1; j < ny - 1; j++)
                for (long i = 1; i < nx - 1; i++) {
                    long q = k * sz + j * sy + i;
                    if (p->order == 2) { l[q] = d[q]; continue; }
                    REAL y4 = four * y[q];
                    REAL exy = ((y[q - sx - sy] + y[q + sx - sy]) + (y[q - sx + sy] + y[q + sx + sy])) - y4;
                    REAL exz = ((y[q - sx - sz] + y[q + sx - sz]) + (y[q - sx + sz] + y[q + sx + sz])) - y4;
                    REAL eyz = ((y[q - sy - sz] + y[q + sy - sz]) + (y[q - sy + sz] + y[q + sy + sz])) - y4;
                    REAL e = (exy + exz) + eyz;
                    REAL td = FN(fmar)(-ten, d[q], ((d[q - sx] + d[q + sx]) + (d[q - sy] + d[q + sy]))
                                                   + (d[q - sz] + d[q + sz]));
                    l[q] = FN(fmar)(c->c16h2, e, -(c->c112 * td));
                }
    }
}

/* F(Psi) = i[a Lap Psi + (s|Psi|^2 - V) Psi] in split form, (fsplit) P:424-428:
 *   F^R = -a Lap Psi^I - s(Psi^R^2 + Psi^I^2) Psi^I + V Psi^I
 *   F^I =  a Lap Psi^R + s(Psi^R^2 + Psi^I^2) Psi^R - V Psi^R
 * (with V absent the V terms are omitted, reading R-V0). */
static void FN(f_point)(const FN(oracle_consts) *c, REAL yr, REAL yi, REAL lr, REAL li,
                        const REAL *V, long q, REAL *fr, REAL *fi)
{
    REAL rho = (yr * yr) + (yi * yi);
    REAL sr = c->s * rho;
    REAL r = FN(fmar)(-c->a, li, -(sr * yi));
    REAL m = FN(fmar)(c->a, lr, sr * yr);
    if (V) {
        r = FN(fmar)(V[q], yi, r);
        m = FN(fmar)(-V[q], yr, m);
    }
    *fr = r;
    *fi = m;
}

/* F at boundary points, time-derivative BC form.
 *   Dirichlet (BCDdt) P:315-318: dPsi_b/dt = 0
 *   MSD (msd) P:331-335: dPsi_b/dt = i Im[(1/Psi_{b-1}) dPsi_{b-1}/dt] Psi_b,
 *     dPsi_{b-1}/dt "precomputed using the internal finite-difference scheme"
 *     -- so this runs after the interior F.
 *   Im[F/Y] = (F^I Y^R - F^R Y^I)/|Y|^2.
 *   L0 (BCL0dt) P:347-350: dPsi_b/dt = i(s|Psi_b|^2 - V_b) Psi_b, evaluated as
 *     (fsplit) with Lap Psi_b = 0 ((BCL0lap) P:352-355; reading R-L0). */
static void FN(f_boundary)(const oracle_problem *p, const FN(oracle_consts) *c, const REAL *V,
                           const REAL *yr, const REAL *yi, REAL *fr, REAL *fi)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    ORC_PARFOR
    for (long k = 0; k < nz; k++)
        for (long j = 0; j < ny; j++)
            for (long i = 0; i < nx; i++) {
                if (FN(n_bnd_axes)(p, i, j, k) == 0) continue;
                long q = (k * ny + j) * nx + i;
                if (p->bc == 0) { fr[q] = 0; fi[q] = 0; continue; }
                if (p->bc == 2) { FN(f_point)(c, yr[q], yi[q], 0, 0, V, q, &fr[q], &fi[q]); continue; }
                long b1 = FN(inward)(p, i, j, k);
                REAL rho1 = (yr[b1] * yr[b1]) + (yi[b1] * yi[b1]);
                REAL m = 0;
                if (!(rho1 < c->eps2))
                    m = ((fi[b1] * yr[b1]) - (fr[b1] * yi[b1])) / rho1;
                fr[q] = -(m * yi[q]);
                fi[q] = m * yr[q];
            }
}

/* Laplacian pieces; D and L sized like the grid. */
static void FN(laplacian)(const oracle_problem *p, const FN(oracle_consts) *c, const REAL *V,
                          const REAL *yr, const REAL *yi, REAL *dr, REAL *di, REAL *lr, REAL *li)
{
    long n = p->n[0] * p->n[1] * p->n[2];
    ORC_PARFOR
    for (long q = 0; q < n; q++) { dr[q] = di[q] = lr[q] = li[q] = (REAL)NAN; }
    FN(d_interior)(p, c, yr, dr);
    FN(d_interior)(p, c, yi, di);
    if (p->order == 4) FN(d_boundary)(p, c, V, yr, yi, dr, di);
    FN(l_interior)(p, c, yr, dr, lr);
    FN(l_interior)(p, c, yi, di, li);
}

/* F(Y) over the whole grid: interior by (fsplit), then the boundary by the
 * time-derivative BC.  Scratch: dr, di, lr, li. */
static void FN(rhs)(const oracle_problem *p, const FN(oracle_consts) *c, const REAL *V,
                    const REAL *yr, const REAL *yi, REAL *fr, REAL *fi,
                    REAL *dr, REAL *di, REAL *lr, REAL *li)
{
    const long nx = p->n[0], ny = p->n[1], nz = p->n[2];
    FN(laplacian)(p, c, V, yr, yi, dr, di, lr, li);
    ORC_PARFOR
    for (long k = 0; k < nz; k++)
        for (long j = 0; j < ny; j++)
            for (long i = 0; i < nx; i++) {
                if (FN(n_bnd_axes)(p, i, j, k) != 0) continue;
                long q = (k * ny + j) * nx + i;
                FN(f_point)(c, yr[q], yi[q], lr[q], li[q], V, q, &fr[q], &fi[q]);
            }
    FN(f_boundary)(p, c, V, yr, yi, fr, fi);
}

int FN(oracle_rhs)(const oracle_problem *p, const REAL *V, const REAL *yr, const REAL *yi,
                   REAL *fr, REAL *fi)
{
    if (oracle_check(p)) return -1;
    long n = p->n[0] * p->n[1] * p->n[2];
    REAL *w = (REAL *)malloc(sizeof(REAL) * 4 * (size_t)n);
    if (!w) return -2;
    FN(oracle_consts) c = FN(make_consts)(p);
    FN(rhs)(p, &c, V, yr, yi, fr, fi, w, w + n, w + 2 * n, w + 3 * n);
    free(w);
    return 0;
}

int FN(oracle_lap)(const oracle_problem *p, const REAL *V, const REAL *yr, const REAL *yi,
                   REAL *dr, REAL *di, REAL *lr, REAL *li)
{
    if (oracle_check(p)) return -1;
    FN(oracle_consts) c = FN(make_consts)(p);
    FN(laplacian)(p, &c, V, yr, yi, dr, di, lr, li);
    return 0;
}

/* ---------------------------------------------------------------------------
 * nsteps steps of the classic RK4 in the paper's 10-step algorithmic form,
 * (RK4) P:164-180, with F evaluated as above:
 *   1) Ktot = F(Psi^n)              6) Ktmp = F(Psi_tmp)
 *   2) Psi_tmp = Psi^n + k/2 Ktot   7) Ktot = Ktot + 2 Ktmp
 *   3) Ktmp = F(Psi_tmp)            8) Psi_tmp = Psi^n + k Ktmp
 *   4) Ktot = Ktot + 2 Ktmp         9) Ktmp = F(Psi_tmp)
 *   5) Psi_tmp = Psi^n + k/2 Ktmp  10) Psi^{n+1} = Psi^n + k/6 (Ktot + Ktmp)
 * ------------------------------------------------------------------------- */
int FN(oracle_step)(const oracle_problem *p, const REAL *V, REAL *re, REAL *im,
                    double k, long nsteps)
{
    if (oracle_check(p) || !(k > 0) || nsteps < 0) return -1;
    const long n = p->n[0] * p->n[1] * p->n[2];
    REAL *w = (REAL *)malloc(sizeof(REAL) * 10 * (size_t)n);
    if (!w) return -2;
    REAL *ktr = w, *kti = w + n, *kmr = w + 2 * n, *kmi = w + 3 * n;
    REAL *ptr = w + 4 * n, *pti = w + 5 * n;
    REAL *dr = w + 6 * n, *di = w + 7 * n, *lr = w + 8 * n, *li = w + 9 * n;
    FN(oracle_consts) c = FN(make_consts)(p);
    const REAL k2 = (REAL)(k / 2.0), k1 = (REAL)k, k6 = (REAL)(k / 6.0), two = 2;

    for (long step = 0; step < nsteps; step++) {
        /* 1) */ FN(rhs)(p, &c, V, re, im, ktr, kti, dr, di, lr, li);
        ORC_PARFOR
        /* 2) */ for (long q = 0; q < n; q++) { ptr[q] = FN(fmar)(k2, ktr[q], re[q]); pti[q] = FN(fmar)(k2, kti[q], im[q]); }
        /* 3) */ FN(rhs)(p, &c, V, ptr, pti, kmr, kmi, dr, di, lr, li);
        ORC_PARFOR
        /* 4) */ for (long q = 0; q < n; q++) { ktr[q] = FN(fmar)(two, kmr[q], ktr[q]); kti[q] = FN(fmar)(two, kmi[q], kti[q]); }
        ORC_PARFOR
        /* 5) */ for (long q = 0; q < n; q++) { ptr[q] = FN(fmar)(k2, kmr[q], re[q]); pti[q] = FN(fmar)(k2, kmi[q], im[q]); }
        /* 6) */ FN(rhs)(p, &c, V, ptr, pti, kmr, kmi, dr, di, lr, li);
        ORC_PARFOR
        /* 7) */ for (long q = 0; q < n; q++) { ktr[q] = FN(fmar)(two, kmr[q], ktr[q]); kti[q] = FN(fmar)(two, kmi[q], kti[q]); }
        ORC_PARFOR
        /* 8) */ for (long q = 0; q < n; q++) { ptr[q] = FN(fmar)(k1, kmr[q], re[q]); pti[q] = FN(fmar)(k1, kmi[q], im[q]); }
        /* 9) */ FN(rhs)(p, &c, V, ptr, pti, kmr, kmi, dr, di, lr, li);
        ORC_PARFOR
        /* 10) */ for (long q = 0; q < n; q++) {
            re[q] = FN(fmar)(k6, ktr[q] + kmr[q], re[q]);
            im[q] = FN(fmar)(k6, kti[q] + kmi[q], im[q]);
        }
    }
    free(w);
    return 0;
}

#undef FN
#undef ORC_CAT
#undef ORC_CAT2
