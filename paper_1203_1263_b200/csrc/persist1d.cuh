// persist1d.cuh -- 1D grids: all RK4 steps of one nlse_step call in ONE CTA, with the
// whole state (Psi, K_tot, Psi_tmp, Psi_out and V) resident in shared memory.
//
// The 1D configurations (1025-2001 points) are latency-bound:
// per stage there are only ~2000 points of work, so eight kernel launches per step would
// cost far more than the arithmetic.  Here a stage is ONE block-wide phase (round 2; it was
// three, separated by barriers): every thread evaluates, for each of its points, 2SHOC step 1
// D = Delta_2 Y / h^2 ((2shoc1d) P:197) at the point and its two neighbours itself (boundary
// points by the Laplacian form of the BC, (BCDlap) P:320-323, (BCMSDlap) P:336-344, (BCL0lap)
// P:352-355), step 2 ((2shoc1d2) P:198; CD: L = D), F (fsplit) P:424-428 and the RK4 stage
// combine (RK4_GPU) P:495-519; the two boundary points recompute F at b' themselves ((BCDdt)
// P:315-318, (msd) P:331-335, (BCL0dt) P:347-350).  One __syncthreads per stage.
// Every value follows the DAG of DESIGN.md §3.1 (the same expressions as generic.cuh),
// so the result is bit-identical to the oracle and to the per-stage kernels.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"

namespace nlse {

constexpr int P1_THREADS = 1024;
#ifndef NLSE_P1_MSD2
#define NLSE_P1_MSD2 1
#endif

template <typename T>
struct Persist1DArgs {
    cplx<T> *psi;          // global Psi (read at entry, written at exit)
    const T *V;            // nullptr => V = 0
    int n;
    Consts<T> c[4];        // per stage: kc = k/2, k/2, k, k/6
    int64_t nsteps;
    int *diverged;
    const int *step_base;
};

template <typename T>
inline size_t persist1d_smem(int n, bool hasV, bool shoc) {
    (void)shoc;                          // (round 2: no D / F arrays, one phase per stage)
    // Psi, K_tot, Psi_tmp, Psi_out, F at points 1 and n - 2 (MSD), V
    return size_t(n) * sizeof(cplx<T>) * 4 + 2 * sizeof(cplx<T>) + (hasV ? size_t(n) * sizeof(T) : 0);
}

template <typename T, int ORDER, int BC>
__global__ void __launch_bounds__(P1_THREADS, 1) rk4_1d_persistent(Persist1DArgs<T> P) {
    using C = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = P.n;
    C *Ps = reinterpret_cast<C *>(smem_raw);
    C *Ks = Ps + n, *As = Ks + n, *Bs = As + n;
    C *Fb = Bs + n;                                            // MSD: F at points 1, n - 2
    T *Vs = reinterpret_cast<T *>(Fb + 2);
    const bool hasV = P.V != nullptr;
    for (int i = threadIdx.x; i < n; i += P1_THREADS) {
        Ps[i] = P.psi[i];
        if (hasV) Vs[i] = P.V[i];
    }
    __syncthreads();

    auto nlin = [&](const Consts<T> &c, int i, C y) -> T {
        T rho = (y.x * y.x) + (y.y * y.y);
        T r = c.s * rho;
        if (hasV) r = r - Vs[i];
        return r;
    };
    auto d_int = [&](const Consts<T> &c, const C *Y, int i) -> C {
        const C y2 = cadd(Y[i], Y[i]);
        return cscale(c.ih2, csub(cadd(Y[i - 1], Y[i + 1]), y2));
    };
    auto f_of = [&](const Consts<T> &c, int i, C y, C L) -> C {
        const T rho = (y.x * y.x) + (y.y * y.y);
        const T sr = c.s * rho;
        T fr = tfma(-c.a, L.y, -(sr * y.y));
        T fi = tfma(c.a, L.x, sr * y.x);
        if (hasV) { fr = tfma(Vs[i], y.y, fr); fi = tfma(-Vs[i], y.x, fi); }
        C F; F.x = fr; F.y = fi;
        return F;
    };

    for (int64_t step = 0; step < P.nsteps; step++) {
#pragma unroll 1
        for (int stage = 1; stage <= 4; stage++) {
            const Consts<T> &c = P.c[stage - 1];
            const C *Y = stage == 1 ? Ps : (stage == 3 ? Bs : As);
            C *Out = stage == 1 ? As : (stage == 2 ? Bs : (stage == 3 ? As : Ps));
            auto combine = [&](int i, C F) {
                if (stage == 1) {
                    Ks[i] = F;
                    Out[i] = cfma(c.kc, F, Y[i]);
                } else if (stage == 4) {
                    const C r = cfma(c.kc, cadd(Ks[i], F), Ps[i]);
                    Out[i] = r;
                    if (!(isfinite(r.x) && isfinite(r.y))) atomicMin(P.diverged, *P.step_base + int(step));
                } else {
                    Ks[i] = cfma(T(2), F, Ks[i]);
                    Out[i] = cfma(c.kc, F, Ps[i]);
                }
            };
            // D at point j: 2SHOC step 1 at interior points, the Laplacian form of the BC at the two
            // boundary points (with D_int and Y at b')
            auto d_any = [&](int j) -> C {
                if (j > 0 && j < n - 1) return d_int(c, Y, j);
                C d;
                if (BC == BC_L0) {
                    d.x = T(0); d.y = T(0);
                    return d;
                }
                const C yb = Y[j];
                const T nb = nlin(c, j, yb);
                if (BC == BC_DIRICHLET) {
                    const T t = c.inv_a * nb;
                    d.x = -(t * yb.x); d.y = -(t * yb.y);
                } else {
                    const int j1 = j == 0 ? 1 : n - 2;
                    const C y1 = Y[j1], d1 = d_int(c, Y, j1);
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T re = T(0);
                    if (!(rho1 < c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
                    const T n1 = nlin(c, j1, y1);
                    const T g = re + ((n1 - nb) * c.inv_a);
                    d = cscale(g, yb);
                }
                return d;
            };
            // F at interior point j: L ((2shoc1d2) P:198 from D at j-1, j, j+1, each evaluated here;
            // CD: L = D), (fsplit) P:424-428
            auto f_int = [&](int j) -> C {
                C L;
                if (ORDER == ORDER_CD) L = d_int(c, Y, j);
                else L = cfma(c.c76, d_any(j), cneg(cscale(c.c112, cadd(d_any(j - 1), d_any(j + 1)))));
                return f_of(c, j, Y[j], L);
            };
            // One phase per stage: every point of this thread, the boundary points with F(b')
            // recomputed locally ((BCDdt) P:315-318, (msd) P:331-335, (BCL0dt) P:347-350), so the
            // only barrier is the one before the next stage reads this stage's output.  (D is
            // evaluated up to three times per point instead of once through shared memory: the
            // same expressions, so the same bits, and two block barriers fewer per stage.)
            // MSD (NLSE_P1_MSD2, default): the two boundary points take F(b') from the threads of
            // points 1 and n - 2 through shared memory after a second barrier, instead of
            // recomputing it (two dependent divisions on one thread's critical path)
            constexpr bool MSD2 = BC == BC_MSD && NLSE_P1_MSD2;
            for (int i = threadIdx.x; i < n; i += P1_THREADS) {
                C F;
                if (i > 0 && i < n - 1) {
                    F = f_int(i);
                    if (MSD2) {
                        if (i == 1) Fb[0] = F;
                        if (i == n - 2) Fb[1] = F;
                    }
                } else if (MSD2) {
                    continue;
                } else if (BC == BC_DIRICHLET) {
                    F.x = T(0); F.y = T(0);
                } else if (BC == BC_L0) {
                    C z; z.x = T(0); z.y = T(0);
                    F = f_of(c, i, Y[i], z);
                } else {
                    const int i1 = i == 0 ? 1 : n - 2;
                    const C y1 = Y[i1], f1 = f_int(i1), yb = Y[i];
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T m = T(0);
                    if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                    F.x = -(m * yb.y);
                    F.y = m * yb.x;
                }
                combine(i, F);
            }
            if (MSD2) {
                __syncthreads();
                if (threadIdx.x < 2) {
                    const int i = threadIdx.x == 0 ? 0 : n - 1, i1 = i == 0 ? 1 : n - 2;
                    const C y1 = Y[i1], f1 = Fb[threadIdx.x], yb = Y[i];
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T m = T(0);
                    if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                    C F;
                    F.x = -(m * yb.y);
                    F.y = m * yb.x;
                    combine(i, F);
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += P1_THREADS) P.psi[i] = Ps[i];
}

// ------------------------------------------------------------------ thread-block cluster variant
// The single-CTA kernel above runs on ONE SM, and on configs[0] (1025 points, ~1 point per thread)
// its stage is bound by that SM's fp64 issue rate and the latency chain of one point.  Here the
// grid is split into NC contiguous segments, one per CTA of a thread-block cluster (NC <= 8
// SMs): each CTA keeps its segment of Psi, K_tot, Psi_tmp, Psi_out and V in its own shared
// memory, reads the <= 2 points beyond its segment ends from the neighbouring CTAs' shared memory
// (distributed shared memory), and a cluster barrier ends each stage.  Per point the same
// expressions as rk4_1d_persistent (one phase per stage, MSD boundary F(b') through a second CTA
// barrier in the first / last CTA), so the same bits.
template <typename T>
inline size_t cluster1d_smem(int n, int nc, bool hasV) {
    const size_t m = size_t((n + nc - 1) / nc);              // the longest segment
    return m * sizeof(cplx<T>) * 4 + 2 * sizeof(cplx<T>) + (hasV ? m * sizeof(T) : 0);
}

template <typename T, int ORDER, int BC>
__global__ void __launch_bounds__(1024, 1) rk4_1d_cluster(Persist1DArgs<T> P) {
    using C = cplx<T>;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int nc = int(cl.num_blocks()), rk = int(cl.block_rank());
    const int n = P.n, nt = int(blockDim.x), tid = int(threadIdx.x);
    auto seg0 = [&](int r) { return int((int64_t(n) * r) / nc); };
    const int a = seg0(rk), b = seg0(rk + 1), mmax = (n + nc - 1) / nc;
    const int al = rk > 0 ? seg0(rk - 1) : 0;                 // global start of the left segment
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Ps = reinterpret_cast<C *>(smem_raw);
    C *Ks = Ps + mmax, *As = Ks + mmax, *Bs = As + mmax;
    C *Fb = Bs + mmax;                                         // MSD: F at points 1, n - 2
    T *Vs = reinterpret_cast<T *>(Fb + 2);
    const bool hasV = P.V != nullptr;
    for (int i = tid; i < b - a; i += nt) {
        Ps[i] = P.psi[a + i];
        if (hasV) Vs[i] = P.V[a + i];
    }
    cl.sync();
    // Y at global point j (own segment, or the left / right neighbour's copy of the same buffer)
    auto yat = [&](const C *Y, int j) -> C {
        if (j >= a && j < b) return Y[j - a];
        if (j < a) return cl.map_shared_rank(const_cast<C *>(Y), rk - 1)[j - al];
        return cl.map_shared_rank(const_cast<C *>(Y), rk + 1)[j - b];
    };
    auto nlin = [&](const Consts<T> &c, int j, C y) -> T {   // (V at the first / last CTA's points)
        T rho = (y.x * y.x) + (y.y * y.y);
        T r = c.s * rho;
        if (hasV) r = r - Vs[j - a];
        return r;
    };
    auto d_int = [&](const Consts<T> &c, const C *Y, int j) -> C {
        const C yj = yat(Y, j);
        const C y2 = cadd(yj, yj);
        return cscale(c.ih2, csub(cadd(yat(Y, j - 1), yat(Y, j + 1)), y2));
    };
    auto f_of = [&](const Consts<T> &c, int j, C y, C L) -> C {
        const T rho = (y.x * y.x) + (y.y * y.y);
        const T sr = c.s * rho;
        T fr = tfma(-c.a, L.y, -(sr * y.y));
        T fi = tfma(c.a, L.x, sr * y.x);
        if (hasV) { fr = tfma(Vs[j - a], y.y, fr); fi = tfma(-Vs[j - a], y.x, fi); }
        C F; F.x = fr; F.y = fi;
        return F;
    };
    for (int64_t step = 0; step < P.nsteps; step++) {
#pragma unroll 1
        for (int stage = 1; stage <= 4; stage++) {
            const Consts<T> &c = P.c[stage - 1];
            const C *Y = stage == 1 ? Ps : (stage == 3 ? Bs : As);
            C *Out = stage == 1 ? As : (stage == 2 ? Bs : (stage == 3 ? As : Ps));
            auto combine = [&](int i, C F) {
                const int li = i - a;
                if (stage == 1) {
                    Ks[li] = F;
                    Out[li] = cfma(c.kc, F, Y[li]);
                } else if (stage == 4) {
                    const C r = cfma(c.kc, cadd(Ks[li], F), Ps[li]);
                    Out[li] = r;
                    if (!(isfinite(r.x) && isfinite(r.y))) atomicMin(P.diverged, *P.step_base + int(step));
                } else {
                    Ks[li] = cfma(T(2), F, Ks[li]);
                    Out[li] = cfma(c.kc, F, Ps[li]);
                }
            };
            auto d_any = [&](int j) -> C {
                if (j > 0 && j < n - 1) return d_int(c, Y, j);
                C d;
                if (BC == BC_L0) { d.x = T(0); d.y = T(0); return d; }
                const C yb = yat(Y, j);
                const T nb = nlin(c, j, yb);
                if (BC == BC_DIRICHLET) {
                    const T t = c.inv_a * nb;
                    d.x = -(t * yb.x); d.y = -(t * yb.y);
                } else {
                    const int j1 = j == 0 ? 1 : n - 2;
                    const C y1 = yat(Y, j1), d1 = d_int(c, Y, j1);
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T re = T(0);
                    if (!(rho1 < c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
                    const T n1 = nlin(c, j1, y1);
                    const T g = re + ((n1 - nb) * c.inv_a);
                    d = cscale(g, yb);
                }
                return d;
            };
            auto f_int = [&](int j) -> C {
                C L;
                if (ORDER == ORDER_CD) L = d_int(c, Y, j);
                else L = cfma(c.c76, d_any(j), cneg(cscale(c.c112, cadd(d_any(j - 1), d_any(j + 1)))));
                return f_of(c, j, yat(Y, j), L);
            };
            constexpr bool MSD2 = BC == BC_MSD && NLSE_P1_MSD2;
            for (int i = a + tid; i < b; i += nt) {
                C F;
                if (i > 0 && i < n - 1) {
                    F = f_int(i);
                    if (MSD2) {
                        if (i == 1) Fb[0] = F;
                        if (i == n - 2) Fb[1] = F;
                    }
                } else if (MSD2) {
                    continue;
                } else if (BC == BC_DIRICHLET) {
                    F.x = T(0); F.y = T(0);
                } else if (BC == BC_L0) {
                    C z; z.x = T(0); z.y = T(0);
                    F = f_of(c, i, yat(Y, i), z);
                } else {
                    const int i1 = i == 0 ? 1 : n - 2;
                    const C y1 = yat(Y, i1), f1 = f_int(i1), yb = yat(Y, i);
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T m = T(0);
                    if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                    F.x = -(m * yb.y);
                    F.y = m * yb.x;
                }
                combine(i, F);
            }
            if (MSD2) {
                __syncthreads();                               // Fb of this CTA written
                const bool lo = rk == 0 && tid == 0, hi = rk == nc - 1 && tid == (nc == 1 ? 1 : 0);
                if (lo || hi) {
                    const int i = lo ? 0 : n - 1, i1 = lo ? 1 : n - 2;
                    const C y1 = yat(Y, i1), f1 = Fb[lo ? 0 : 1], yb = yat(Y, i);
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T m = T(0);
                    if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                    C F;
                    F.x = -(m * yb.y);
                    F.y = m * yb.x;
                    combine(i, F);
                }
            }
            cl.sync();                                         // stage outputs visible cluster-wide
        }
    }
    for (int i = tid; i < b - a; i += nt) P.psi[a + i] = Ps[i];
}

}  // namespace nlse
