// tile2d.cuh -- 2D interior stage kernel (§8(a) rows a1-a5, a7 for 2D grids).
//
// CTA = 256 threads owns a TX x TY = 32 x 16 tile of output points (each thread two
// rows, ty and ty + 8).  The stage input Y is staged once per stage in shared memory
// as a (TX+2H) x (TY+2H) tile with an H = w wide halo (coalesced 16-byte loads, one
// warp per tile row); for 2SHOC, step 1 (D = Delta_2 Y / h^2, (2d2shocs1) P:202-210)
// is evaluated once per tile point plus a one-point ring into a shared D tile (faces:
// the Laplacian form of the BC; D never touches HBM); step 2
// ((2d2shocs2) P:214-228), F (fsplit) and the RK4 stage combine then run per owned
// point with Psi, K_tot, V read once from HBM.  The grid working set of the 2D configs
// (1024^2 fp64 + V: 75 MB) is L2-resident on B200, so the halo re-reads are L2 hits.
// Domain-boundary outputs come from stage_boundary.  DAG: DESIGN.md §3.1 (bitwise =
// oracle).
#pragma once
#include "generic.cuh"

namespace nlse {

#ifndef NLSE_T2_TY
#define NLSE_T2_TY 16
#endif
constexpr int T2_TX = 32, T2_TY = NLSE_T2_TY, T2_NT = 256;
constexpr int T2_RPT = T2_TY / 8;          // rows per thread (8 warps)

// cp.async (Ampere-style asynchronous copies, global -> shared without a register round
// trip): every load of the tile and of the owned Psi / K_tot / V is in flight at once
template <int BYTES>
__device__ __forceinline__ void t2_cp(void *sdst, const void *gsrc, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    const int n = valid ? BYTES : 0;                  // src-size 0: zero fill
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gsrc), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(sa), "l"(gsrc), "n"(BYTES), "r"(n)
                     : "memory");
}
__device__ __forceinline__ void t2_cp_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Shared memory of one 2D tile (sized for stages 2-4; stage 1 leaves Psi / K_tot unused).
template <typename T, int ORDER>
struct T2Smem {
    using C = cplx<T>;
    static constexpr int H = (ORDER == ORDER_2SHOC) ? 2 : 1;
    static constexpr int PX = T2_TX + 2 * H, PY = T2_TY + 2 * H;
    static constexpr int DPX = T2_TX + 2, DPY = T2_TY + 2;
    C ys[PY * PX];
    C ds[(ORDER == ORDER_2SHOC) ? DPY * DPX : 1];
    C ps[T2_RPT * T2_NT], ks[T2_RPT * T2_NT];
    T vs[T2_RPT * T2_NT];
};

// One 32 x T2_TY tile at (x0, y0) of one stage (the whole body of stage2d_tile; the persistent
// 2D kernel runs it for many tiles and stages).
template <typename T, int ORDER, int BC, int STAGE>
__device__ __forceinline__ void t2_tile(const StageArgs<T> &A, T2Smem<T, ORDER> &S, int x0, int y0) {
    using C = cplx<T>;
    constexpr int H = T2Smem<T, ORDER>::H, PX = T2Smem<T, ORDER>::PX;
    constexpr int DPX = T2Smem<T, ORDER>::DPX, DPY = T2Smem<T, ORDER>::DPY;
    C *ys = S.ys, *ds = S.ds, *ps = S.ps, *ks = S.ks;
    T *vs = S.vs;
    const int nx = int(A.g.nx), ny = int(A.g.ny);
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    // y-slab mode (§8(e)): rows [ymlo, ymhi) are in memory (ghost rows of the neighbours below /
    // above); rows [olo, ohi] are this slab's output rows; y faces only where the slab holds them
    const bool flo = A.g.zf_lo != 0, fhi = A.g.zf_hi != 0;
    const int ymlo = flo ? 0 : -A.g.zghost, ymhi = fhi ? ny : ny + A.g.zghost;
    const int olo = flo ? 1 : 0, ohi = fhi ? ny - 2 : ny - 1;

    // (1) Y tile with halo (zero outside the grid; those values are never used), and Psi,
    // K_tot, V of the owned points, all as asynchronous copies
    for (int ly = ty - H; ly < T2_TY + H; ly += T2_NT / 32) {
        const int gy = y0 + ly;
        for (int lx = tx - H; lx < T2_TX + H; lx += 32) {
            const int gx = x0 + lx;
            const bool in = gx >= 0 && gx < nx && gy >= ymlo && gy < ymhi;
            t2_cp<int(sizeof(C))>(&ys[(ly + H) * PX + (lx + H)], A.Y + (in ? int64_t(gy) * A.g.sy + gx : 0), in);
        }
    }
#pragma unroll
    for (int r = 0; r < T2_RPT; r++) {
        const int gx = x0 + tx, gy = y0 + ty + 8 * r;
        if (gx >= 1 && gx <= nx - 2 && gy >= olo && gy <= ohi) {
            const int64_t q = int64_t(gy) * A.g.sy + gx;
            if (STAGE != 1) {
                t2_cp<int(sizeof(C))>(&ps[r * T2_NT + tid], A.Psi + q, true);
                t2_cp<int(sizeof(C))>(&ks[r * T2_NT + tid], A.K + q, true);
            }
            if (A.V) t2_cp<int(sizeof(T))>(&vs[r * T2_NT + tid], A.V + q, true);
        }
    }
    t2_cp_wait_all();
    __syncthreads();
    auto Ys = [&](int lx, int ly) -> C { return ys[(ly + H) * PX + (lx + H)]; };
    auto D_int = [&](int lx, int ly) -> C {
        const C yc = Ys(lx, ly);
        const C y2 = cadd(yc, yc);
        C acc = csub(cadd(Ys(lx - 1, ly), Ys(lx + 1, ly)), y2);
        acc = cadd(acc, csub(cadd(Ys(lx, ly - 1), Ys(lx, ly + 1)), y2));
        return cscale(A.c.ih2, acc);
    };
    auto nlin = [&](int gx, int gy, C yq) -> T {
        T rho = (yq.x * yq.x) + (yq.y * yq.y);
        T n = A.c.s * rho;
        if (A.V) n = n - __ldg(A.V + int64_t(gy) * A.g.sy + gx);
        return n;
    };

    // (2) 2SHOC step 1 over the tile + ring.  Tiles whose ring is in-grid interior (the
    // bulk of a large grid) take the stencil everywhere, without per-point face tests.
    const bool inner = x0 >= 2 && x0 + T2_TX <= nx - 2 && y0 - H >= ymlo && y0 + T2_TY + H <= ymhi &&
                       (!flo || y0 >= 2) && (!fhi || y0 + T2_TY <= ny - 2);
    if (ORDER == ORDER_2SHOC && inner) {
        for (int e = tid; e < DPX * DPY; e += T2_NT) {
            const int lx = e % DPX - 1, ly = e / DPX - 1;
            ds[e] = D_int(lx, ly);
        }
        __syncthreads();
    } else if (ORDER == ORDER_2SHOC) {
        for (int e = tid; e < DPX * DPY; e += T2_NT) {
            const int lx = e % DPX - 1, ly = e / DPX - 1;
            const int gx = x0 + lx, gy = y0 + ly;
            C d; d.x = T(NAN); d.y = T(NAN);
            // (ring points beyond the rows in memory or x faces of ghost rows are never used)
            const bool ghost_row = gy < 0 || gy >= ny;
            if (gx >= 0 && gx < nx && gy >= (flo ? 0 : ymlo + 1) && gy < (fhi ? ny : ymhi - 1)) {
                const bool fx = (gx == 0 || gx == nx - 1), fy = (flo && gy == 0) || (fhi && gy == ny - 1);
                if (fx && ghost_row) {
                } else if (!fx && !fy) {
                    d = D_int(lx, ly);
                } else if (BC == BC_L0 && !(fx && fy)) {
                    d.x = T(0); d.y = T(0);                       // (BCL0lap) P:352-355
                } else if (!(fx && fy)) {
                    // face: Laplacian form of the BC with b' the in-plane inward neighbour
                    const C yb = Ys(lx, ly);
                    const T nb = nlin(gx, gy, yb);
                    if (BC == BC_DIRICHLET) {
                        const T t = A.c.inv_a * nb;
                        d.x = -(t * yb.x); d.y = -(t * yb.y);
                    } else {
                        int lx1 = lx, ly1 = ly;
                        if (gx == 0) lx1 = lx + 1; else if (gx == nx - 1) lx1 = lx - 1;
                        else if (gy == 0) ly1 = ly + 1; else ly1 = ly - 1;
                        const C y1 = Ys(lx1, ly1), d1 = D_int(lx1, ly1);
                        const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                        T re = T(0);
                        if (!(rho1 < A.c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
                        const T n1 = nlin(x0 + lx1, y0 + ly1, y1);
                        const T gg = re + ((n1 - nb) * A.c.inv_a);
                        d = cscale(gg, yb);
                    }
                }
            }
            ds[e] = d;
        }
        __syncthreads();
    }

    // (3) step 2, F, RK4 stage combine at the owned interior points
#pragma unroll
    for (int r = 0; r < T2_RPT; r++) {
        const int lx = tx, ly = ty + 8 * r;
        const int gx = x0 + lx, gy = y0 + ly;
        if (gx < 1 || gx > nx - 2 || gy < olo || gy > ohi) continue;
        const int64_t q = int64_t(gy) * A.g.sy + gx;
        const C yc = Ys(lx, ly);
        C L;
        if (ORDER == ORDER_CD) {
            L = D_int(lx, ly);
        } else {
            const C y4 = cscale(T(4), yc);
            const C pxa = cadd(Ys(lx - 1, ly - 1), Ys(lx + 1, ly - 1));
            const C pxb = cadd(Ys(lx - 1, ly + 1), Ys(lx + 1, ly + 1));
            const C cxy = csub(cadd(pxa, pxb), y4);
            const C *Dp = ds + (ly + 1) * DPX + (lx + 1);
            const C sd = cadd(cadd(Dp[-1], Dp[1]), cadd(Dp[-DPX], Dp[DPX]));
            const C td = cfma(T(-12), Dp[0], sd);
            L = cfma(A.c.c16h2, cxy, cneg(cscale(A.c.c112, td)));
        }
        // F (fsplit) P:424-428
        const T rho = (yc.x * yc.x) + (yc.y * yc.y);
        const T sr = A.c.s * rho;
        C F = f_lin(A.c.a, L, sr, yc);
        if (A.V) F = f_addv(F, vs[r * T2_NT + tid], yc);
        // RK4 stage combine (RK4_GPU) P:495-519, as rk_combine with Psi, K_tot staged
        if (STAGE == 1) {
            A.K[q] = F;
            store_out(A, q, gy, cfma(A.c.kc, F, yc));
        } else if (STAGE == 4) {
            const C o = cfma(A.c.kc, cadd(ks[r * T2_NT + tid], F), ps[r * T2_NT + tid]);
            store_out(A, q, gy, o);
            if (!(isfinite(o.x) && isfinite(o.y))) atomicMin(A.diverged, *A.step_base + A.step);
        } else {
            A.K[q] = cfma(T(2), F, ks[r * T2_NT + tid]);
            store_out(A, q, gy, cfma(A.c.kc, F, ps[r * T2_NT + tid]));
        }
    }
}

#ifndef NLSE_T2_MINB
#define NLSE_T2_MINB 1
#endif
template <typename T, int ORDER, int BC, int STAGE>
__global__ void __launch_bounds__(T2_NT, NLSE_T2_MINB) stage2d_tile(StageArgs<T> A) {
    __shared__ __align__(16) T2Smem<T, ORDER> S;
    t2_tile<T, ORDER, BC, STAGE>(A, S, int(blockIdx.x) * T2_TX, int(blockIdx.y) * T2_TY);
}

// ------------------------------------------------------------------ persistent 2D stepper
// L2-scale 2D grids (configs[2], 1024^2: ~1 M points, a stage is ~20 us of launch-bound work)
// run every stage of every step of an nlse_step call in ONE cooperative launch: the co-resident
// CTAs loop over the tiles of a stage (t2_tile) and over its boundary points (F by the BC
// time-derivative form, as stage_boundary), then meet at a grid-wide barrier before the next
// stage reads what this one wrote.  Same per-point operations as the per-stage kernels.
template <typename T>
struct Persist2DArgs {
    StageArgs<T> A[4];           // stage operands (stage s + 1), step field set per step
    int64_t nsteps;
    unsigned *bar_count;         // grid barrier: arrivals of the current generation
    unsigned *bar_gen;           // grid barrier: generation
};

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Sense-counting grid barrier over the co-resident CTAs of a cooperative launch.
__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_gpu_u32(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            st_release_gpu_u32(gen, g + 1);
        } else {
            while (ld_acquire_gpu_u32(gen) == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename T, int ORDER, int BC, int STAGE>
__device__ __forceinline__ void p2_stage(const StageArgs<T> &A, T2Smem<T, ORDER> &S, int ntx, int ntiles) {
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        t2_tile<T, ORDER, BC, STAGE>(A, S, (t % ntx) * T2_TX, (t / ntx) * T2_TY);
        __syncthreads();                 // the tile's shared arrays are reused by the next tile
    }
    const int64_t nb = n_boundary_points<2>(A.g);
    PointEval<T, 2, ORDER, BC> ev{A.Y, A.V, A.g, A.c};
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nb; b += int64_t(gridDim.x) * blockDim.x) {
        int64_t i, j, k;
        bnd_point<2>(A.g, b, i, j, k);
        const int64_t q = ev.idx(i, j, k);
        const cplx<T> F = ev.F_bnd(i, j, k);
        const cplx<T> psi = (STAGE == 1) ? ev.y(q) : A.Psi[q];
        rk_combine<STAGE, T>(A, q, j, F, psi);
    }
}

template <typename T, int ORDER, int BC>
__global__ void __launch_bounds__(T2_NT) rk4_2d_persistent(const __grid_constant__ Persist2DArgs<T> P) {
    __shared__ __align__(16) T2Smem<T, ORDER> S;
    const int ntx = int((P.A[0].g.nx + T2_TX - 1) / T2_TX), nty = int((P.A[0].g.ny + T2_TY - 1) / T2_TY);
    const int ntiles = ntx * nty;
    for (int64_t n = 0; n < P.nsteps; n++) {
        StageArgs<T> A;
        A = P.A[0]; A.step = int(n); p2_stage<T, ORDER, BC, 1>(A, S, ntx, ntiles); grid_barrier(P.bar_count, P.bar_gen);
        A = P.A[1]; A.step = int(n); p2_stage<T, ORDER, BC, 2>(A, S, ntx, ntiles); grid_barrier(P.bar_count, P.bar_gen);
        A = P.A[2]; A.step = int(n); p2_stage<T, ORDER, BC, 3>(A, S, ntx, ntiles); grid_barrier(P.bar_count, P.bar_gen);
        A = P.A[3]; A.step = int(n); p2_stage<T, ORDER, BC, 4>(A, S, ntx, ntiles); grid_barrier(P.bar_count, P.bar_gen);
    }
}

template <typename T, int ORDER, int BC, int STAGE>
void launch_tile2d(const StageArgs<T> &A, cudaStream_t st) {
    const dim3 grid(unsigned((A.g.nx + T2_TX - 1) / T2_TX), unsigned((A.g.ny + T2_TY - 1) / T2_TY));
    stage2d_tile<T, ORDER, BC, STAGE><<<grid, T2_NT, 0, st>>>(A);
}

// 1D grids above the persistent single-CTA limit (the paper's Table 1 runs 1D up to 3e6 points,
// P:664-686): one CTA per tile of T1_N = 256 x T1_R points.  The stage input Y is staged once
// in shared memory with an H = w wide halo (coalesced loads), 2SHOC step 1 ((2shoc1d) P:197)
// is evaluated once per tile point plus a one-point ring into a shared D tile (the face point
// x = 0 / nx - 1 by the Laplacian form of the BC, (BCDlap) P:320-323, (BCMSDlap) P:336-344,
// (BCL0lap) P:352-355), then step 2 ((2shoc1d2) P:198), F (fsplit) P:424-428 and the RK4 stage
// combine (RK4_GPU) P:495-519 run per owned interior point with Psi, K_tot, V read once.
// The two boundary points are finished by the CTAs owning their inward neighbours b' = 1 and
// nx - 2 (F_b from F(b') in registers: (BCDdt) P:315-318, (msd) P:331-335, (BCL0dt) P:347-350),
// so a stage is one launch.  DAG: DESIGN.md §3.1 (bitwise = oracle).
constexpr int T1_NT = 256;

// T1_R points per thread: 4 on long grids (fewer halo loads), 1 below 2^20 points (more CTAs
// in flight: 1e4-1e5-point grids are latency-bound)
template <typename T, int ORDER, int BC, int STAGE, int T1_R>
__global__ void __launch_bounds__(T1_NT) stage1d_tile(StageArgs<T> A) {
    using C = cplx<T>;
    constexpr int T1_N = T1_NT * T1_R;
    constexpr int H = (ORDER == ORDER_2SHOC) ? 2 : 1;
    __shared__ __align__(16) C ys[T1_N + 2 * H];
    __shared__ __align__(16) C ds[(ORDER == ORDER_2SHOC) ? T1_N + 2 : 1];
    pdl_trigger();                       // (launched with programmatic dependent launch, launch_tile1d)
    pdl_wait();
    const int64_t nx = A.g.nx;
    const int64_t x0 = int64_t(blockIdx.x) * T1_N;
    const int tid = threadIdx.x;
    // x-slab mode (§8(e)): points [xmlo, xmhi) are in memory (ghosts of the neighbours); x faces
    // only where the slab holds them; output points [olo, ohi]
    const bool flo = A.g.zf_lo != 0, fhi = A.g.zf_hi != 0;
    const int64_t xmlo = flo ? 0 : -A.g.zghost, xmhi = fhi ? nx : nx + A.g.zghost;
    const int64_t olo = flo ? 1 : 0, ohi = fhi ? nx - 2 : nx - 1;
    // (1) Y tile with halo (zero outside the grid: never used)
    for (int e = tid; e < T1_N + 2 * H; e += T1_NT) {
        const int64_t gx = x0 - H + e;
        C v; v.x = T(0); v.y = T(0);
        if (gx >= xmlo && gx < xmhi) v = A.Y[gx];
        ys[e] = v;
    }
    __syncthreads();
    auto Yl = [&](int lx) -> C { return ys[lx + H]; };       // local x in [-H, T1_N + H)
    auto d_int = [&](int lx) -> C {
        const C yc = Yl(lx);
        const C y2 = cadd(yc, yc);
        return cscale(A.c.ih2, csub(cadd(Yl(lx - 1), Yl(lx + 1)), y2));
    };
    // (2) 2SHOC step 1 on the tile + one-point ring; faces by the Laplacian form of the BC
    if (ORDER == ORDER_2SHOC) {
        for (int e = tid; e < T1_N + 2; e += T1_NT) {
            const int lx = e - 1;
            const int64_t gx = x0 + lx;
            C d; d.x = T(NAN); d.y = T(NAN);
            const bool face = (flo && gx == 0) || (fhi && gx == nx - 1);
            if (!face && gx > xmlo && gx < xmhi - 1) {
                d = d_int(lx);
            } else if (face) {
                if (BC == BC_L0) {
                    d.x = T(0); d.y = T(0);
                } else {
                    const C yb = Yl(lx);
                    T nb = A.c.s * ((yb.x * yb.x) + (yb.y * yb.y));
                    if (A.V) nb = nb - __ldg(A.V + gx);
                    if (BC == BC_DIRICHLET) {
                        const T t = A.c.inv_a * nb;
                        d.x = -(t * yb.x); d.y = -(t * yb.y);
                    } else {
                        const int lx1 = gx == 0 ? lx + 1 : lx - 1;
                        const C y1 = Yl(lx1), d1 = d_int(lx1);
                        const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                        T re = T(0);
                        if (!(rho1 < A.c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
                        T n1 = A.c.s * rho1;
                        if (A.V) n1 = n1 - __ldg(A.V + (x0 + lx1));
                        const T gg = re + ((n1 - nb) * A.c.inv_a);
                        d = cscale(gg, yb);
                    }
                }
            }
            ds[e] = d;
        }
        __syncthreads();
    }
    // (3) step 2, F, RK4 stage combine at the owned interior points (coalesced: thread t owns
    // points t, t + 256, ...)
#pragma unroll
    for (int r = 0; r < T1_R; r++) {
        const int lx = tid + r * T1_NT;
        const int64_t q = x0 + lx;
        if (q < olo || q > ohi) continue;
        const C yc = Yl(lx);
        C L;
        if (ORDER == ORDER_CD) L = d_int(lx);
        else L = cfma(A.c.c76, ds[lx + 1], cneg(cscale(A.c.c112, cadd(ds[lx], ds[lx + 2]))));
        const T rho = (yc.x * yc.x) + (yc.y * yc.y);
        const T sr = A.c.s * rho;
        C F = f_lin(A.c.a, L, sr, yc);
        if (A.V) F = f_addv(F, __ldg(A.V + q), yc);
        const C psi = STAGE == 1 ? yc : A.Psi[q];
        rk_combine<STAGE, T>(A, q, q, F, psi);
        // the boundary point whose b' is q (nx = 3: q = 1 is b' of both); held faces only
        for (int side = 0; side < 2; side++) {
            const int64_t qb = side == 0 ? 0 : nx - 1;
            if (!(side == 0 ? flo : fhi) || q != (side == 0 ? 1 : nx - 2)) continue;
            const C yb = Yl(int(qb - x0));
            C Fb;
            if (BC == BC_DIRICHLET) {
                Fb.x = T(0); Fb.y = T(0);
            } else if (BC == BC_L0) {
                const T rb = (yb.x * yb.x) + (yb.y * yb.y);
                const T srb = A.c.s * rb;
                T gr = tfma(-A.c.a, T(0), -(srb * yb.y));
                T gi = tfma(A.c.a, T(0), srb * yb.x);
                if (A.V) {
                    const T vb = __ldg(A.V + qb);
                    gr = tfma(vb, yb.y, gr);
                    gi = tfma(-vb, yb.x, gi);
                }
                Fb.x = gr; Fb.y = gi;
            } else {
                T m = T(0);
                if (!(rho < A.c.eps2)) m = ((F.y * yc.x) - (F.x * yc.y)) / rho;
                Fb.x = -(m * yb.y);
                Fb.y = m * yb.x;
            }
            const C psib = STAGE == 1 ? yb : A.Psi[qb];
            rk_combine<STAGE, T>(A, qb, qb, Fb, psib);
        }
    }
}

// Programmatic dependent launch (NLSE_PDL=0: off) for grids of at most 148 CTAs: the ~10^4-point
// grids of the paper's Table 1 are launch-latency bound (10^4 points 9.8 vs 10.8 us/step; at 10^5
// points, 391 CTAs, it measured slower: 12.9 vs 11.3, r02 pdl_c).
template <typename T, int ORDER, int BC, int STAGE>
void launch_tile1d(const StageArgs<T> &A, cudaStream_t st) {
    const bool big = A.g.nx >= (int64_t(1) << 20);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(big ? (A.g.nx + 4 * T1_NT - 1) / (4 * T1_NT) : (A.g.nx + T1_NT - 1) / T1_NT), 1, 1);
    cfg.blockDim = dim3(T1_NT, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    const char *e = getenv("NLSE_PDL");
    cfg.attrs = at;
    cfg.numAttrs = ((e && e[0] == '0') || cfg.gridDim.x > 148) ? 0 : 1;
    if (big) cudaLaunchKernelEx(&cfg, stage1d_tile<T, ORDER, BC, STAGE, 4>, A);
    else cudaLaunchKernelEx(&cfg, stage1d_tile<T, ORDER, BC, STAGE, 1>, A);
}

}  // namespace nlse
