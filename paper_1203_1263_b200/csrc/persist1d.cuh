// persist1d.cuh -- 1D grids: all RK4 steps of one nlse_step call in ONE CTA, with the
// whole state (Psi, K_tot, Psi_tmp, Psi_out, D, F and V) resident in shared memory.
//
// The 1D configurations (1025-2001 points) are latency-bound:
// per stage there are only ~2000 points of work, so eight kernel launches per step would
// cost far more than the arithmetic.  Here a stage is three block-wide phases separated
// by __syncthreads:
//   (1) 2SHOC step 1, D = Delta_2 Y / h^2 ((2shoc1d) P:197) at every point, boundary
//       points by the Laplacian form of the BC ((BCDlap) P:320-323, (BCMSDlap) P:336-344,
//       (BCL0lap) P:352-355);
//   (2) interior points: L ((2shoc1d2) P:198, or L = D for CD), F (fsplit) P:424-428, F
//       kept in shared memory, and the RK4 stage combine (RK4_GPU) P:495-519;
//   (3) the two boundary points: F from the time-derivative BC ((BCDdt) P:315-318,
//       (msd) P:331-335 with F at b' from phase 2, (BCL0dt) P:347-350) and the combine.
// Every value follows the DAG of DESIGN.md §3.1 (the same expressions as generic.cuh),
// so the result is bit-identical to the oracle and to the per-stage kernels.
#pragma once
#include "common.cuh"

namespace nlse {

constexpr int P1_THREADS = 1024;

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
    return size_t(n) * (sizeof(cplx<T>) * (5 + (shoc ? 1 : 0)) + (hasV ? sizeof(T) : 0));
}

template <typename T, int ORDER, int BC>
__global__ void __launch_bounds__(P1_THREADS, 1) rk4_1d_persistent(Persist1DArgs<T> P) {
    using C = cplx<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = P.n;
    C *Ps = reinterpret_cast<C *>(smem_raw);
    C *Ks = Ps + n, *As = Ks + n, *Bs = As + n, *Fs = Bs + n;
    C *Ds = Fs + n;                                            // 2SHOC only
    T *Vs = reinterpret_cast<T *>(Ds + (ORDER == ORDER_2SHOC ? n : 0));
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
            // (1) 2SHOC step 1 with boundary D from the Laplacian form of the BC
            if (ORDER == ORDER_2SHOC) {
                for (int i = threadIdx.x; i < n; i += P1_THREADS) {
                    C d;
                    if (i > 0 && i < n - 1) {
                        d = d_int(c, Y, i);
                    } else if (BC == BC_L0) {
                        d.x = T(0); d.y = T(0);
                    } else {
                        const C yb = Y[i];
                        const T nb = nlin(c, i, yb);
                        if (BC == BC_DIRICHLET) {
                            const T t = c.inv_a * nb;
                            d.x = -(t * yb.x); d.y = -(t * yb.y);
                        } else {
                            const int i1 = i == 0 ? 1 : n - 2;
                            const C y1 = Y[i1], d1 = d_int(c, Y, i1);
                            const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                            T re = T(0);
                            if (!(rho1 < c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
                            const T n1 = nlin(c, i1, y1);
                            const T g = re + ((n1 - nb) * c.inv_a);
                            d = cscale(g, yb);
                        }
                    }
                    Ds[i] = d;
                }
                __syncthreads();
            }
            // (2) interior: L, F, combine
            for (int i = 1 + threadIdx.x; i < n - 1; i += P1_THREADS) {
                C L;
                if (ORDER == ORDER_CD) L = d_int(c, Y, i);
                else L = cfma(c.c76, Ds[i], cneg(cscale(c.c112, cadd(Ds[i - 1], Ds[i + 1]))));
                const C F = f_of(c, i, Y[i], L);
                Fs[i] = F;
                combine(i, F);
            }
            __syncthreads();
            // (3) boundary points
            if (threadIdx.x < 2) {
                const int i = threadIdx.x == 0 ? 0 : n - 1;
                C F;
                if (BC == BC_DIRICHLET) {
                    F.x = T(0); F.y = T(0);
                } else if (BC == BC_L0) {
                    C z; z.x = T(0); z.y = T(0);
                    F = f_of(c, i, Y[i], z);
                } else {
                    const int i1 = i == 0 ? 1 : n - 2;
                    const C y1 = Y[i1], f1 = Fs[i1], yb = Y[i];
                    const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                    T m = T(0);
                    if (!(rho1 < c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                    F.x = -(m * yb.y);
                    F.y = m * yb.x;
                }
                combine(i, F);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += P1_THREADS) P.psi[i] = Ps[i];
}

}  // namespace nlse
