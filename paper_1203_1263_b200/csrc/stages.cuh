// stages.cuh -- stage launches (§8(a) row a8): one RK4 stage = the interior kernel of the
// context's family + the boundary kernel, with the per-stage operands of (RK4_GPU)
// P:495-519.  Included only by the instantiation units inst_*.cu; each defines, through
// NLSE_DEFINE_STAGES(_BC), the enqueue entry points of one (precision, dimension, order)
// family for one or all three BCs (declared in runtime.cuh, called by nlse_api.cu).
#pragma once
#include <algorithm>
#include "runtime.cuh"
#include "generic.cuh"
#include "persist1d.cuh"
#include "stage3d_tma.cuh"
#include "stream3d.cuh"
#include "tile2d.cuh"
#include "fused3d.cuh"
#include "strip2d.cuh"

namespace nlse_rt {

// The stage kernel finishes the x-face boundary points itself (StageArgs::xfuse) when every
// tile that owns x-face points runs the lean face-aware loop (t3_lean_ok in stage3d_tma.cuh:
// no face point on a tile's ring, no x face on lane 0 of a tile past x = 0).
inline bool xfuse_mode(const nlse_ctx *c) {
    if (!c->tma || !c->fp || c->order != NLSE_2SHOC4) return false;
    const char *fe = getenv("NLSE_FORCE_EDGE");
    if (fe && fe[0] == '2') return false;
    const char *ex = getenv("NLSE_XFUSE");
    if (ex && ex[0] == '0') return false;
    const int64_t nx = c->g.nx, ny = c->g.ny;
    if ((nx - 1) % 32 == 0 || (ny - 1) % c->tma_ty == 0) return false;
    // worth it where the light pass is bandwidth-bound on the scattered x-face points (1024^3:
    // 2.1M of them, -0.6 % step time); on small grids the edge tiles are the critical path
    // (87x87x203: 161 vs 150 us/step with it), so only from 2^18 x-face points on (or =1)
    if (ex && ex[0] == '1') return true;
    return 2 * (ny - 2) * (c->g.nz - c->g.zf_lo - c->g.zf_hi) >= (int64_t(1) << 18);
}

template <typename T, int ORDER, int BC, int STAGE, int TYV>
void launch_tma3d_ty(nlse_ctx *c, const StageArgs<T> &A) {
    constexpr int PS = STAGE == 1 ? TMA_P1 : TMA_P;
    using Cfg = T3Cfg<T, ORDER, PS, TYV, STAGE != 1>;
    auto kern = stage3d_tma<T, ORDER, BC, STAGE, PS, TYV>;
    const int64_t nx = A.g.nx, ny = A.g.ny;
    const int64_t mz = A.g.nz - A.g.zf_lo - A.g.zf_hi;
    const unsigned gx = unsigned((nx + Cfg::TX - 1) / Cfg::TX);
    const unsigned gy = unsigned((ny + Cfg::TY - 1) / Cfg::TY);
    // z chunks: at most 128 planes (L2 locality of neighbouring tiles, r01e), and the
    // chunk count that minimises (waves of resident CTAs) x (planes per chunk + the ~4-plane
    // prologue), so that small grids fill the GPU in whole waves
    const int64_t cols = int64_t(gx) * gy;
    static PerDevice per_sm_cache;
    int per_sm = per_sm_cache.get(c->device);
    if (!per_sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::NT, Cfg::SMEM);
        if (per_sm < 1) per_sm = 1;
        per_sm_cache.set(c->device, per_sm);
    }
    const int64_t resident = int64_t(c->nsm) * per_sm;
    int64_t zchunk = mz, best = -1;
    for (int64_t nzc = (mz + 127) / 128; nzc <= mz; nzc++) {
        const int64_t ch = (mz + nzc - 1) / nzc;
        const int64_t waves = (cols * nzc + resident - 1) / resident;
        const int64_t cost = waves * (ch + 4);
        if (best < 0 || cost < best) { best = cost; zchunk = ch; }
        if (ch <= 4) break;
    }
    const char *ezc = getenv("NLSE_ZCHUNK");               // (read per launch: tests vary it)
    const int64_t env_chunk = ezc ? std::atoll(ezc) : int64_t(0);
    if (env_chunk > 0) zchunk = env_chunk;
    if (zchunk > mz) zchunk = mz;
    const unsigned gz = unsigned((mz + zchunk - 1) / zchunk);
    const int64_t items = int64_t(gx) * gy * gz;
    // tile order (stage3d_tma): bands of 4 tile rows walked column by column where there are at
    // least 8 tile rows (1024^3: 78.8 vs 80.6 DRAM bytes per point-stage, -0.6 % step time, r02
    // band); NLSE_TILE_BAND=0 row-major, =B bands of B rows
    const char *eband = getenv("NLSE_TILE_BAND");
    const int band = eband ? std::atoi(eband) : (gy >= 8 ? 4 : 0);
    // debug / measurement / tests: NLSE_FORCE_EDGE=1 runs every tile on the face-aware lean
    // loop, =2 every tile on the per-point face path (t3_run, EDGE)
    const char *fe = getenv("NLSE_FORCE_EDGE");
    int force_edge = (fe && (fe[0] == '0' || fe[0] == '1' || fe[0] == '2')) ? fe[0] - '0' : -1;
    if (force_edge < 0) {
        // grids where most tiles touch a face (87x87: 14 of 18) run every tile on the face-aware
        // lean loop: one hot code path for the instruction cache instead of two (r02 ring_ab:
        // 87x87x203 144.8 vs 150.8 us/step fp64, 96.5 vs 99.9 fp32); large grids keep the
        // branch-free interior loop on their interior tiles
        auto inner = [](int64_t n, int64_t t) {          // tiles with 2 <= x0 and x0 + t <= n - 2
            int64_t c = 0;
            for (int64_t x0 = 0; x0 < n; x0 += t) c += (x0 >= 2 && x0 + t <= n - 2);
            return c;
        };
        force_edge = (2 * inner(nx, Cfg::TX) * inner(ny, Cfg::TY) < cols) ? 1 : 0;
    }
    kern<<<unsigned(items), Cfg::NT, Cfg::SMEM, c->stream>>>(c->maps.y[ybuf_of_stage(STAGE)], c->maps.psi, c->maps.k,
                                                          c->maps.v, A, int(zchunk), int(gx), int(gy), force_edge, band);
}

template <typename T, int ORDER, int BC, int STAGE>
void launch_tma3d(nlse_ctx *c, const StageArgs<T> &A) {
    if (c->tma_ty == 16) launch_tma3d_ty<T, ORDER, BC, STAGE, 16>(c, A);
    else launch_tma3d_ty<T, ORDER, BC, STAGE, 8>(c, A);
}

// One stage: interior kernel family + boundary kernel (or the generic kernel over the
// whole owned grid).
template <typename T, int DIM, int ORDER, int BC, int STAGE>
void launch_stage(nlse_ctx *c, const StageArgs<T> &A) {
    if (c->interior_kind == KK_GENERIC) {
        LaunchTimer lt(c, KK_GENERIC, c->g.n);
        stage_generic<T, DIM, ORDER, BC, STAGE><<<blocks_for(c->g.n, 256), 256, 0, c->stream>>>(A);
        return;
    }
    if constexpr (DIM == 2) {
        if (c->interior_kind == KK_STRIP2D) {          // boundary included: one launch per stage
            LaunchTimer lt(c, KK_STRIP2D, c->g.n);
            launch_strip2d<T, ORDER, BC, STAGE>(A, c->nsm, c->stream);
            return;
        }
    }
    // 2D/3D: the boundary kernel (disjoint outputs, same inputs: it recomputes what it needs at
    // b') runs concurrently on a side stream, forked from and joined back into the context
    // stream (not in timing mode, so that per-kernel shares stay attributable).  The 3D MSD
    // light pass (c->fp: F(b') stored by the interior kernel) must follow the interior kernel.
    const bool side = DIM >= 2 && !c->timing && c->side_stream && !c->fp;
    if (side) {
        const int64_t nb = n_boundary_points<DIM>(c->g);
        cudaEventRecord(c->ev_fork, c->stream);
        cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0);
        stage_boundary<T, DIM, ORDER, BC, STAGE><<<blocks_for(nb, 256), 256, 0, c->side_stream>>>(A);
        cudaEventRecord(c->ev_join, c->side_stream);
    }
    {
        const int64_t ni = (c->g.nx - 2) * (DIM >= 2 ? c->g.ny - 2 : 1) *
                           (DIM >= 3 ? c->g.nz - c->g.zf_lo - c->g.zf_hi : 1);
        LaunchTimer lt(c, c->interior_kind, ni);
        if constexpr (DIM == 3) {
            if (c->interior_kind == KK_TMA3D) launch_tma3d<T, ORDER, BC, STAGE>(c, A);
            else launch_stream3d<T, ORDER, BC, STAGE>(A, c->stream);
        } else if constexpr (DIM == 2) {
            launch_tile2d<T, ORDER, BC, STAGE>(A, c->stream);
        } else {
            launch_tile1d<T, ORDER, BC, STAGE>(A, c->stream);
        }
    }
    if (DIM == 1) return;               // stage1d_tile finishes the two boundary points itself
    if (side) {
        cudaStreamWaitEvent(c->stream, c->ev_join, 0);
    } else if (DIM == 3 && BC == BC_MSD && A.fp) {
        // F(b') was stored by the interior kernel: a light pass after it
        const int64_t nb = n_boundary_points<DIM>(c->g, A.xfuse != 0);
        LaunchTimer lt(c, KK_BOUNDARY, nb);
        stage_boundary_msd_fb<T, STAGE><<<blocks_for(nb, 256), 256, 0, c->stream>>>(A);
    } else {
        const int64_t nb = n_boundary_points<DIM>(c->g);
        LaunchTimer lt(c, KK_BOUNDARY, nb);
        stage_boundary<T, DIM, ORDER, BC, STAGE><<<blocks_for(nb, 256), 256, 0, c->stream>>>(A);
    }
}

// neighbour base pointers: peer_lo[q] / peer_hi[q] address the neighbour's copy of local q
template <typename T>
void peer_ptrs(const nlse_ctx *c, int b, cplx<T> *&lo, cplx<T> *&hi) {
    lo = hi = nullptr;
    if (!c->dist || !c->connected) return;
    const int64_t su = c->g.su;
    // (the peer's plane / row 0 is ghost_off bytes into its allocation, as here)
    if (c->peer_alloc[b][0]) lo = (cplx<T> *)((char *)c->peer_alloc[b][0] + c->ghost_off) + c->peer_nloc[0] * su;
    if (c->peer_alloc[b][1]) hi = (cplx<T> *)((char *)c->peer_alloc[b][1] + c->ghost_off) - c->g.ns * su;
}

template <typename T, int DIM, int ORDER, int BC>
void enqueue_stage_t(nlse_ctx *c, int stage, double k, int step) {
    using C = cplx<T>;
    const double kc = stage == 3 ? k : (stage == 4 ? k / 6.0 : k / 2.0);
    StageArgs<T> A{};
    A.Y = (const C *)c->buf[ybuf_of_stage(stage)];
    A.Psi = (const C *)c->buf[BUF_PSI];
    A.K = (C *)c->K;
    A.out = (C *)c->buf[obuf_of_stage(stage)];
    A.V = (const T *)c->V;
    A.g = c->g;
    A.c = make_consts<T>(c, kc);
    A.diverged = c->d_div;
    A.step_base = c->d_steps;
    A.step = step;
    peer_ptrs<T>(c, obuf_of_stage(stage), A.peer_lo, A.peer_hi);
    A.wsend = halo_w(c);
    {
        static const int env_hints = [] {
            const char *e = getenv("NLSE_L2_HINTS");
            return e ? std::atoi(e) : -1;
        }();
        A.stream_hints = env_hints >= 0 ? env_hints : 0;   // r01y: evict-first hints were slower
        static const int env_rot = [] {
            const char *e = getenv("NLSE_RING_ROT");
            return e ? std::atoi(e) : 1;
        }();
        A.ring_rot = env_rot;
    }
    A.fz = (C *)c->fz;
    A.fp = (C *)c->fp;
    A.per2 = c->per2;
    A.xfuse = xfuse_mode(c) ? 1 : 0;
    // (RK4_GPU) P:495-519: stages {1-3}, {4-6}, {7-9}, {10-11}
    switch (stage) {
        case 1: launch_stage<T, DIM, ORDER, BC, 1>(c, A); break;
        case 2: launch_stage<T, DIM, ORDER, BC, 2>(c, A); break;
        case 3: launch_stage<T, DIM, ORDER, BC, 3>(c, A); break;
        default: launch_stage<T, DIM, ORDER, BC, 4>(c, A); break;
    }
}

// 1D: all nsteps in one persistent CTA when the state fits in shared memory.
template <typename T, int ORDER, int BC>
void launch_persist1d(nlse_ctx *c, double k, int64_t nsteps) {
    Persist1DArgs<T> P{};
    P.psi = (cplx<T> *)c->buf[BUF_PSI];
    P.V = (const T *)c->V;
    P.n = int(c->g.nx);
    P.c[0] = make_consts<T>(c, k / 2.0);
    P.c[1] = make_consts<T>(c, k / 2.0);
    P.c[2] = make_consts<T>(c, k);
    P.c[3] = make_consts<T>(c, k / 6.0);
    P.nsteps = nsteps;
    P.diverged = c->d_div;
    P.step_base = c->d_steps;
    const size_t smem = persist1d_smem<T>(P.n, c->hasV, ORDER == ORDER_2SHOC);
    static PerDevice attr;
    if (!attr.get(c->device)) {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
        cudaFuncSetAttribute(rk4_1d_persistent<T, ORDER, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
        attr.set(c->device, 1);
    }
    LaunchTimer lt(c, KK_TILE1D, c->g.n * nsteps);
    if (c->cluster1d > 1) {
        // thread-block cluster of c->cluster1d CTAs, one grid segment each (rk4_1d_cluster)
        const int nc = c->cluster1d;
        const int m = (P.n + nc - 1) / nc;
        const int nt = std::min(1024, (m + 31) / 32 * 32);
        const size_t csm = cluster1d_smem<T>(P.n, nc, c->hasV);
        auto kern = rk4_1d_cluster<T, ORDER, BC>;
        static PerDevice cattr;
        if (!cattr.get(c->device)) {
            int optin = 0;
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
            cattr.set(c->device, 1);
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(nc), 1, 1);
        cfg.blockDim = dim3(unsigned(nt), 1, 1);
        cfg.dynamicSmemBytes = csm;
        cfg.stream = c->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = unsigned(nc);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, P);
        return;
    }
    rk4_1d_persistent<T, ORDER, BC><<<1, P1_THREADS, smem, c->stream>>>(P);
}

// ------------------------------------------------------------------ fused two-stage passes
// One RK4 step in fused mode (§8(f) rank 2, fused3d.cuh): pass 1 = S1+S2, pass 2 = S3+S4, each
// followed by the boundary kernel of its second stage; Psi_new goes to the second Psi buffer and
// the two Psi buffers are swapped.
template <typename T, int BC, int PAIR, int TYV>
void launch_fused_pass(nlse_ctx *c, double k, int step) {
    using C = cplx<T>;
    using Cfg = F3Cfg<T, TYV, PAIR>;
    constexpr int STAGE_B = PAIR == 1 ? 2 : 4;
    auto kern = fused3d_cd<T, BC, PAIR, TYV>;
    StageArgs<T> A{};
    A.Y = (const C *)c->buf[BUF_TMP];                 // stage-B input at face / b' points (boundary pass)
    A.Psi = (const C *)c->buf[BUF_PSI];
    A.K = (C *)c->K;
    A.out = (C *)c->buf[PAIR == 1 ? BUF_OUT : BUF_PSI2];
    A.V = (const T *)c->V;
    A.g = c->g;
    A.c = make_consts<T>(c, PAIR == 1 ? k / 2.0 : k / 6.0);
    A.diverged = c->d_div;
    A.step_base = c->d_steps;
    A.step = step;
    A.wsend = 1;
    A.fz = (C *)c->fz;
    A.fp = (C *)c->fp;
    A.per2 = c->per2;
    A.xfuse = 0;
    FusedArgs<T> FA{};
    FA.cA = T(PAIR == 1 ? k / 2.0 : k);
    FA.ztmp = (C *)c->buf[BUF_TMP];
    const int64_t nx = c->g.nx, ny = c->g.ny, mz = c->g.nz - 2;
    const unsigned gx = unsigned((nx + Cfg::TX - 1) / Cfg::TX), gy = unsigned((ny + Cfg::TY - 1) / Cfg::TY);
    static PerDevice attr;
    if (!attr.get(c->device)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        attr.set(c->device, 1);
    }
    // z chunks as launch_tma3d_ty: <= 128 planes, whole waves of one CTA per SM
    const int64_t cols = int64_t(gx) * gy;
    int64_t zchunk = mz, best = -1;
    for (int64_t nzc = (mz + 127) / 128; nzc <= mz; nzc++) {
        const int64_t ch = (mz + nzc - 1) / nzc;
        const int64_t waves = (cols * nzc + c->nsm - 1) / c->nsm;
        const int64_t cost = waves * (ch + 4);
        if (best < 0 || cost < best) { best = cost; zchunk = ch; }
        if (ch <= 4) break;
    }
    const unsigned gz = unsigned((mz + zchunk - 1) / zchunk);
    const CUtensorMap &mY = c->fmaps.y[PAIR == 1 ? BUF_PSI : BUF_OUT];
    {
        LaunchTimer lt(c, KK_FUSED3D, (nx - 2) * (ny - 2) * mz);
        kern<<<unsigned(cols * gz), Cfg::NT, Cfg::SMEM, c->stream>>>(mY, c->fmaps.base[BUF_PSI], c->fmaps.k,
                                                                     c->fmaps.v, A, FA, int(zchunk), int(gx), int(gy));
    }
    // stage-B outputs at the domain boundary
    if (BC == BC_MSD) {
        const int64_t nb = n_boundary_points<3>(c->g, false);
        LaunchTimer lt(c, KK_BOUNDARY, nb);
        stage_boundary_msd_fb<T, STAGE_B><<<blocks_for(nb, 256), 256, 0, c->stream>>>(A);
    } else {
        const int64_t nb = n_boundary_points<3>(c->g);
        LaunchTimer lt(c, KK_BOUNDARY, nb);
        stage_boundary<T, 3, ORDER_CD, BC, STAGE_B><<<blocks_for(nb, 256), 256, 0, c->stream>>>(A);
    }
}

template <typename T, int BC>
void fused_step_t(nlse_ctx *c, double k, int step) {
    if (c->fused_ty == 8) {
        launch_fused_pass<T, BC, 1, 8>(c, k, step);
        launch_fused_pass<T, BC, 2, 8>(c, k, step);
    } else {
        launch_fused_pass<T, BC, 1, 16>(c, k, step);
        launch_fused_pass<T, BC, 2, 16>(c, k, step);
    }
    swap_psi(c);
}

// 2D L2-scale grids: every stage of nsteps steps in one cooperative launch (tile2d.cuh).
template <typename T, int ORDER, int BC>
void launch_persist2d(nlse_ctx *c, double k, int64_t nsteps) {
    using C = cplx<T>;
    Persist2DArgs<T> P{};
    for (int s = 1; s <= 4; s++) {
        StageArgs<T> &A = P.A[s - 1];
        const double kc = s == 3 ? k : (s == 4 ? k / 6.0 : k / 2.0);
        A.Y = (const C *)c->buf[ybuf_of_stage(s)];
        A.Psi = (const C *)c->buf[BUF_PSI];
        A.K = (C *)c->K;
        A.out = (C *)c->buf[obuf_of_stage(s)];
        A.V = (const T *)c->V;
        A.g = c->g;
        A.c = make_consts<T>(c, kc);
        A.diverged = c->d_div;
        A.step_base = c->d_steps;
        A.wsend = halo_w(c);
    }
    P.nsteps = nsteps;
    P.bar_count = c->d_bar;
    P.bar_gen = c->d_bar + 1;
    auto kern = rk4_2d_persistent<T, ORDER, BC>;
    static PerDevice per_sm_cache;
    int per_sm = per_sm_cache.get(c->device);
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T2_NT, 0);
        if (per_sm < 1) per_sm = 1;
        per_sm_cache.set(c->device, per_sm);
    }
    const int64_t ntiles = ((c->g.nx + T2_TX - 1) / T2_TX) * ((c->g.ny + T2_TY - 1) / T2_TY);
    const unsigned grid = unsigned(std::min<int64_t>(ntiles, int64_t(c->nsm) * per_sm));
    void *args[] = {&P};
    // a fresh barrier per launch (an aborted earlier launch cannot leave it mid-generation)
    cudaMemsetAsync(c->d_bar, 0, 2 * sizeof(unsigned), c->stream);
    LaunchTimer lt(c, KK_TILE2D, c->g.n * nsteps * 4);
    cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(T2_NT), args, 0, c->stream);
}

template <typename T, int ORDER>
void persist2d_family(nlse_ctx *c, double k, int64_t nsteps) {
    if (c->bc == NLSE_BC_MSD) launch_persist2d<T, ORDER, BC_MSD>(c, k, nsteps);
    else if (c->bc == NLSE_BC_L0) launch_persist2d<T, ORDER, BC_L0>(c, k, nsteps);
    else launch_persist2d<T, ORDER, BC_DIRICHLET>(c, k, nsteps);
}

template <typename T, int ORDER>
void persist1d_family(nlse_ctx *c, double k, int64_t nsteps) {
    if (c->bc == NLSE_BC_MSD) launch_persist1d<T, ORDER, BC_MSD>(c, k, nsteps);
    else if (c->bc == NLSE_BC_L0) launch_persist1d<T, ORDER, BC_L0>(c, k, nsteps);
    else launch_persist1d<T, ORDER, BC_DIRICHLET>(c, k, nsteps);
}

}  // namespace nlse_rt

#define NLSE_ORDER_cd nlse::ORDER_CD
#define NLSE_ORDER_shoc nlse::ORDER_2SHOC
#define NLSE_REAL_f64 double
#define NLSE_REAL_f32 float
#define NLSE_BC_dirichlet nlse::BC_DIRICHLET
#define NLSE_BC_msd nlse::BC_MSD
#define NLSE_BC_l0 nlse::BC_L0
// Define the stage entry point of one family and BC (and, for 1D, its persistent-CTA launcher).
#define NLSE_DEFINE_STAGES_BC(P, D, O, B)                                                       \
    void nlse_rt::enqueue_stage_##P##_##D##d_##O##_##B(nlse_ctx *c, int stage, double k, int step) { \
        nlse_rt::enqueue_stage_t<NLSE_REAL_##P, D, NLSE_ORDER_##O, NLSE_BC_##B>(c, stage, k, step); \
    }
#define NLSE_DEFINE_STAGES(P, D, O)                                                             \
    NLSE_DEFINE_STAGES_BC(P, D, O, dirichlet) NLSE_DEFINE_STAGES_BC(P, D, O, msd) NLSE_DEFINE_STAGES_BC(P, D, O, l0)
#define NLSE_DEFINE_PERSIST1D(P, O)                                                             \
    void nlse_rt::persist1d_##P##_##O(nlse_ctx *c, double k, int64_t nsteps) {                  \
        nlse_rt::persist1d_family<NLSE_REAL_##P, NLSE_ORDER_##O>(c, k, nsteps);                 \
    }
#define NLSE_DEFINE_PERSIST2D(P, O)                                                             \
    void nlse_rt::persist2d_##P##_##O(nlse_ctx *c, double k, int64_t nsteps) {                  \
        nlse_rt::persist2d_family<NLSE_REAL_##P, NLSE_ORDER_##O>(c, k, nsteps);                 \
    }
#define NLSE_DEFINE_FUSED(P, B)                                                                 \
    void nlse_rt::fused_step_##P##_##B(nlse_ctx *c, double k, int step) {                       \
        nlse_rt::fused_step_t<NLSE_REAL_##P, NLSE_BC_##B>(c, k, step);                           \
    }
