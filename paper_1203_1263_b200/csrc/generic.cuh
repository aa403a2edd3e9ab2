// generic.cuh -- one-thread-per-point evaluation of F(Y) at any grid point,
// reading the stage input straight from global memory (through L1/L2).
//
// It serves two roles:
//   * the boundary path of every kernel family: F at boundary points (BC time
//     derivative form, which needs F at the inward neighbour b', recomputed
//     here locally instead of the paper's intra-block sync), and
//   * a complete second GPU implementation (NLSE_FLAG_GENERIC_KERNELS), the
//     paper's kernel structure without shared-memory tiling.
// Expression graph: DESIGN.md §3.1 (reading R-ASSOC), term by term.
#pragma once
#include "common.cuh"

namespace nlse {

template <typename T, int DIM, int ORDER, int BC>
struct PointEval {
    using C = cplx<T>;
    const C *Y;
    const T *V;
    Grid g;
    Consts<T> c;

    __device__ __forceinline__ C y(int64_t q) const { return ldg_c(Y + q); }
    __device__ __forceinline__ T v(int64_t q) const { return __ldg(V + q); }

    __device__ __forceinline__ int n_bnd(int64_t i, int64_t j, int64_t k) const {
        int m = x_face<DIM>(g, i);
        if (DIM >= 2) m += y_face<DIM>(g, j);
        if (DIM >= 3) m += is_zface(g, k);
        return m;
    }
    // Inward neighbour: one step in along every boundary axis (R-MSD-NBR).
    __device__ __forceinline__ void inward(int64_t &i, int64_t &j, int64_t &k) const {
        if (DIM == 1) i = (g.zf_lo && i == 0) ? 1 : ((g.zf_hi && i == g.nx - 1) ? g.nx - 2 : i);
        else i = (i == 0) ? 1 : (i == g.nx - 1 ? g.nx - 2 : i);
        if (DIM == 3) j = (j == 0) ? 1 : (j == g.ny - 1 ? g.ny - 2 : j);
        if (DIM == 2) j = (g.zf_lo && j == 0) ? 1 : ((g.zf_hi && j == g.ny - 1) ? g.ny - 2 : j);
        if (DIM >= 3) k = (g.zf_lo && k == 0) ? 1 : ((g.zf_hi && k == g.nz - 1) ? g.nz - 2 : k);
    }
    __device__ __forceinline__ int64_t idx(int64_t i, int64_t j, int64_t k) const {
        return k * g.sz + j * g.sy + i;
    }

    // 2SHOC step 1 / CD at an interior point: D = (((Px-Y2)+(Py-Y2))+(Pz-Y2))*ih2.
    __device__ __forceinline__ C D_int(int64_t q) const {
        C y0 = y(q);
        C y2 = cadd(y0, y0);
        C acc = csub(cadd(y(q - 1), y(q + 1)), y2);
        if (DIM >= 2) acc = cadd(acc, csub(cadd(y(q - g.sy), y(q + g.sy)), y2));
        if (DIM >= 3) acc = cadd(acc, csub(cadd(y(q - g.sz), y(q + g.sz)), y2));
        return cscale(c.ih2, acc);
    }

    // N = s|Y|^2 - V ((nbnb1) P:341-344)
    __device__ __forceinline__ T nlin(int64_t q, C yq) const {
        T rho = (yq.x * yq.x) + (yq.y * yq.y);
        T n = c.s * rho;
        if (V) n = n - v(q);
        return n;
    }

    // Boundary D on a face point (2SHOC), Laplacian-form BC: (BCDlap) P:320-323,
    // (BCMSDlap) P:336-344 with b' the inward normal neighbour (R-DFACE, R-MSD-LAP).
    __device__ __forceinline__ C D_face(int64_t i, int64_t j, int64_t k) const {
        const int64_t q = idx(i, j, k);
        const C yb = y(q);
        if (BC == BC_L0) { C z; z.x = T(0); z.y = T(0); return z; }   // (BCL0lap) P:352-355
        const T nb = nlin(q, yb);
        if (BC == BC_DIRICHLET) {
            T t = c.inv_a * nb;
            C r; r.x = -(t * yb.x); r.y = -(t * yb.y);
            return r;
        } else {
            int64_t i1 = i, j1 = j, k1 = k;
            inward(i1, j1, k1);
            const int64_t q1 = idx(i1, j1, k1);
            const C y1 = y(q1);
            const C d1 = D_int(q1);
            T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T re = T(0);
            if (!(rho1 < c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
            T n1 = nlin(q1, y1);
            T gg = re + ((n1 - nb) * c.inv_a);
            return cscale(gg, yb);
        }
    }

    // D at a point that is interior or a face point.
    __device__ __forceinline__ C D_any(int64_t i, int64_t j, int64_t k) const {
        if (n_bnd(i, j, k) == 0) return D_int(idx(i, j, k));
        return D_face(i, j, k);
    }

    // L at an interior point (CD: L = D; 2SHOC step 2 otherwise).
    __device__ __forceinline__ C L_int(int64_t i, int64_t j, int64_t k) const {
        const int64_t q = idx(i, j, k);
        if (ORDER == ORDER_CD) return D_int(q);
        const C d0 = D_int(q);
        if (DIM == 1) {
            C dm = D_any(i - 1, j, k), dp = D_any(i + 1, j, k);
            return cfma(c.c76, d0, cneg(cscale(c.c112, cadd(dm, dp))));
        }
        const C y4 = cscale(T(4), y(q));
        if (DIM == 2) {
            C cxy = csub(cadd(cadd(y(q - 1 - g.sy), y(q + 1 - g.sy)), cadd(y(q - 1 + g.sy), y(q + 1 + g.sy))), y4);
            C sd = cadd(cadd(D_any(i - 1, j, k), D_any(i + 1, j, k)), cadd(D_any(i, j - 1, k), D_any(i, j + 1, k)));
            C td = cfma(T(-12), d0, sd);
            return cfma(c.c16h2, cxy, cneg(cscale(c.c112, td)));
        }
        C exy = csub(cadd(cadd(y(q - 1 - g.sy), y(q + 1 - g.sy)), cadd(y(q - 1 + g.sy), y(q + 1 + g.sy))), y4);
        C exz = csub(cadd(cadd(y(q - 1 - g.sz), y(q + 1 - g.sz)), cadd(y(q - 1 + g.sz), y(q + 1 + g.sz))), y4);
        C eyz = csub(cadd(cadd(y(q - g.sy - g.sz), y(q + g.sy - g.sz)), cadd(y(q - g.sy + g.sz), y(q + g.sy + g.sz))), y4);
        C e = cadd(cadd(exy, exz), eyz);
        C sd = cadd(cadd(cadd(D_any(i - 1, j, k), D_any(i + 1, j, k)), cadd(D_any(i, j - 1, k), D_any(i, j + 1, k))),
                    cadd(D_any(i, j, k - 1), D_any(i, j, k + 1)));
        C td = cfma(T(-10), d0, sd);
        return cfma(c.c16h2, e, cneg(cscale(c.c112, td)));
    }

    // Interior F, (fsplit) P:424-428.
    __device__ __forceinline__ C F_from(int64_t q, C yq, C L) const {
        T rho = (yq.x * yq.x) + (yq.y * yq.y);
        T sr = c.s * rho;
        T r = tfma(-c.a, L.y, -(sr * yq.y));
        T m = tfma(c.a, L.x, sr * yq.x);
        if (V) {
            T vq = v(q);
            r = tfma(vq, yq.y, r);
            m = tfma(-vq, yq.x, m);
        }
        C f; f.x = r; f.y = m;
        return f;
    }
    __device__ __forceinline__ C F_int(int64_t i, int64_t j, int64_t k) const {
        const int64_t q = idx(i, j, k);
        return F_from(q, y(q), L_int(i, j, k));
    }

    // F at a boundary point: (BCDdt) P:315-318 / (msd) P:331-335 / (BCL0dt) P:347-350
    // evaluated as (fsplit) with Lap Psi_b = 0 (reading R-L0).
    __device__ __forceinline__ C F_bnd(int64_t i, int64_t j, int64_t k) const {
        C f;
        if (BC == BC_DIRICHLET) { f.x = T(0); f.y = T(0); return f; }
        if (BC == BC_L0) {
            const int64_t qb = idx(i, j, k);
            C zero; zero.x = T(0); zero.y = T(0);
            return F_from(qb, y(qb), zero);
        }
        int64_t i1 = i, j1 = j, k1 = k;
        inward(i1, j1, k1);
        const int64_t q1 = idx(i1, j1, k1);
        const C y1 = y(q1);
        const C f1 = F_int(i1, j1, k1);
        T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
        T m = T(0);
        if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
        const C yb = y(idx(i, j, k));
        f.x = -(m * yb.y);
        f.y = m * yb.x;
        return f;
    }

    __device__ __forceinline__ C F_any(int64_t i, int64_t j, int64_t k) const {
        if (n_bnd(i, j, k) == 0) return F_int(i, j, k);
        return F_bnd(i, j, k);
    }
};

// The slab-axis index of (j, k): the plane in 3D, the row in 2D (neighbour stores, store_out).
template <int DIM>
__device__ __forceinline__ int64_t slab_index(int64_t i, int64_t j, int64_t k) { return DIM == 3 ? k : (DIM == 2 ? j : i); }

// One thread per grid point over the whole grid.
template <typename T, int DIM, int ORDER, int BC, int STAGE>
__global__ void __launch_bounds__(256) stage_generic(StageArgs<T> A) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= A.g.n) return;
    const int64_t i = t % A.g.nx;
    const int64_t j = (t / A.g.nx) % A.g.ny;
    const int64_t k = t / (A.g.nx * A.g.ny);
    PointEval<T, DIM, ORDER, BC> ev{A.Y, A.V, A.g, A.c};
    const int64_t q = ev.idx(i, j, k);
    cplx<T> F = ev.F_any(i, j, k);
    cplx<T> psi = (STAGE == 1) ? ev.y(q) : A.Psi[q];
    rk_combine<STAGE, T>(A, q, slab_index<DIM>(i, j, k), F, psi);
}

// Boundary points only: a flat index over the boundary surface, mapped to (i,j,k).
// 1D: 2 points; 2D: the global y-face rows this slab owns (row 0 if zf_lo, row ny-1 if
// zf_hi; both on one GPU), then the two x-face points of every other owned row (the
// 2(nx + ny) - 4 perimeter on one GPU); 3D: the global z faces this grid
// owns (plane 0 if zf_lo, plane nz-1 if zf_hi), then the perimeter of every other
// owned plane.
// rows_only (3D): the interior planes contribute their two y-face rows only (the x-face
// points of those planes are finished elsewhere: StageArgs::xfuse).
template <int DIM>
__device__ __forceinline__ bool bnd_point(const Grid &g, int64_t t64, int64_t &i, int64_t &j, int64_t &k,
                                          bool rows_only = false) {
    // 32-bit index arithmetic (64-bit division is a long software sequence on the GPU); the
    // launch checks that the boundary count and a face fit in 31 bits
    const unsigned nx = unsigned(g.nx), ny = unsigned(g.ny);
    unsigned t = unsigned(t64);
    if (DIM == 1) {                    // the x faces this slab holds
        if (t >= unsigned(g.zf_lo + g.zf_hi)) return false;
        i = (g.zf_lo && t == 0) ? 0 : g.nx - 1; j = 0; k = 0;
        return true;
    }
    const unsigned per = 2u * nx + (rows_only ? 0u : 2u * (ny - 2u));   // perimeter of one xy plane
    auto perim = [&](unsigned u, int64_t &ii, int64_t &jj) {
        if (u < nx) { ii = u; jj = 0; }
        else if (u < 2u * nx) { ii = u - nx; jj = ny - 1u; }
        else { const unsigned v = u - 2u * nx; ii = (v & 1u) ? nx - 1u : 0; jj = 1u + (v >> 1); }
    };
    if (DIM == 2) {
        const unsigned nf = unsigned(g.zf_lo + g.zf_hi);
        k = 0;
        if (t < nf * nx) {
            j = (g.zf_lo && t < nx) ? 0 : ny - 1u;
            i = (t < nx) ? t : t - nx;
            return true;
        }
        const unsigned v = t - nf * nx;
        if (v >= 2u * (ny - nf)) return false;
        i = (v & 1u) ? nx - 1u : 0;
        j = unsigned(g.zf_lo) + (v >> 1);
        return true;
    }
    const unsigned face = nx * ny;
    const unsigned nf = unsigned(g.zf_lo + g.zf_hi);
    if (t < nf * face) {
        k = (g.zf_lo && t < face) ? 0 : g.nz - 1;
        const unsigned u = (t < face) ? t : t - face;
        const unsigned jj = u / nx;
        i = u - jj * nx; j = jj;
        return true;
    }
    t -= nf * face;
    const unsigned kk = t / per;
    if (kk >= unsigned(g.nz) - nf) return false;
    k = int64_t(g.zf_lo) + kk;
    perim(t - kk * per, i, j);
    return true;
}

template <int DIM>
__host__ __device__ inline int64_t n_boundary_points(const Grid &g, bool rows_only = false) {
    if (DIM == 1) return g.zf_lo + g.zf_hi;
    if (DIM == 2) return (g.zf_lo + g.zf_hi) * g.nx + 2 * (g.ny - g.zf_lo - g.zf_hi);
    const int64_t per = 2 * g.nx + (rows_only ? 0 : 2 * (g.ny - 2));
    const int nf = g.zf_lo + g.zf_hi;
    return nf * g.nx * g.ny + per * (g.nz - nf);
}

template <typename T, int DIM, int ORDER, int BC, int STAGE>
__global__ void __launch_bounds__(256) stage_boundary(StageArgs<T> A) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t i, j, k;
    if (!bnd_point<DIM>(A.g, t, i, j, k)) return;
    PointEval<T, DIM, ORDER, BC> ev{A.Y, A.V, A.g, A.c};
    const int64_t q = ev.idx(i, j, k);
    cplx<T> F = ev.F_bnd(i, j, k);
    cplx<T> psi = (STAGE == 1) ? ev.y(q) : A.Psi[q];
    rk_combine<STAGE, T>(A, q, slab_index<DIM>(i, j, k), F, psi);
}

// 3D MSD boundary points with F(b') taken from what the interior kernel stored (A.fz /
// A.fp), instead of recomputing the two-step Laplacian at b': (msd) P:331-335,
// F_b = i Im(F_b'/Y_b') Y_b, same arithmetic as PointEval::F_bnd.
template <typename T, int STAGE>
__global__ void __launch_bounds__(256) stage_boundary_msd_fb(StageArgs<T> A) {
    using C = cplx<T>;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t i, j, k;
    if (!bnd_point<3>(A.g, t, i, j, k, A.xfuse != 0)) return;
    const int nx = int(A.g.nx), ny = int(A.g.ny);
    const int i1 = i == 0 ? 1 : (i == nx - 1 ? nx - 2 : int(i));
    const int j1 = j == 0 ? 1 : (j == ny - 1 ? ny - 2 : int(j));
    const bool zlo = A.g.zf_lo && k == 0, zhi = A.g.zf_hi && k == A.g.nz - 1;
    const int64_t k1 = zlo ? 1 : (zhi ? A.g.nz - 2 : k);
    C f1;
    if (zlo) f1 = A.fz[int64_t(j1) * nx + i1];
    else if (zhi) f1 = A.fz[int64_t(nx) * ny + int64_t(j1) * nx + i1];
    else f1 = A.fp[k * A.per2 + shell_u(i1, j1, nx, ny)];
    const int64_t q = k * A.g.sz + j * A.g.sy + i;
    const C y1 = A.Y[k1 * A.g.sz + int64_t(j1) * A.g.sy + i1];
    const C yb = A.Y[q];
    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
    T m = T(0);
    if (!(rho1 < A.c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
    C F;
    F.x = -(m * yb.y);
    F.y = m * yb.x;
    const C psi = (STAGE == 1) ? yb : A.Psi[q];
    rk_combine<STAGE, T>(A, q, k, F, psi);
}

}  // namespace nlse

namespace nlse {

// Interior points only, one thread per point (flat index over the interior box).
template <typename T, int DIM, int ORDER, int BC, int STAGE>
__global__ void __launch_bounds__(256) stage_interior_generic(StageArgs<T> A) {
    const int64_t k0 = DIM >= 3 ? A.g.zf_lo : 0;
    const int64_t j0 = DIM == 2 ? A.g.zf_lo : 1;                  // 2D: first owned interior row
    const int64_t i0 = DIM == 1 ? A.g.zf_lo : 1;                  // 1D: first owned interior point
    const int64_t mx = DIM == 1 ? A.g.nx - A.g.zf_lo - A.g.zf_hi : A.g.nx - 2;
    const int64_t my = DIM == 3 ? A.g.ny - 2 : (DIM == 2 ? A.g.ny - A.g.zf_lo - A.g.zf_hi : 1);
    const int64_t mz = DIM >= 3 ? A.g.nz - A.g.zf_lo - A.g.zf_hi : 1;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= mx * my * mz) return;
    const int64_t i = i0 + t % mx;
    const int64_t j = DIM >= 2 ? j0 + (t / mx) % my : 0;
    const int64_t k = DIM >= 3 ? k0 + t / (mx * my) : 0;
    PointEval<T, DIM, ORDER, BC> ev{A.Y, A.V, A.g, A.c};
    const int64_t q = ev.idx(i, j, k);
    cplx<T> F = ev.F_int(i, j, k);
    cplx<T> psi = (STAGE == 1) ? ev.y(q) : A.Psi[q];
    rk_combine<STAGE, T>(A, q, slab_index<DIM>(i, j, k), F, psi);
}

}  // namespace nlse
