// nlse_api.cu -- the C ABI (include/nlse.h) and the runtime behind it: context,
// device buffers, TMA descriptors, constants, validation, stage sequencing (a8),
// slab mode (a9: ghost planes, peer mapping, per-stage neighbour barriers),
// divergence flag, diagnostics (a10) and per-kernel timing.
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/nlse.h"
#include "comm.cuh"
#include "common.cuh"
#include "diag.cuh"
#include "generic.cuh"
#include "persist1d.cuh"
#include "stage3d_tma.cuh"
#include "stream3d.cuh"
#include "tile2d.cuh"

using namespace nlse;

static_assert(NLSE_MAX_RANKS == MAX_RANKS, "rank limits of nlse.h and comm.cuh differ");

namespace {

thread_local std::string g_create_error;

enum KernelKind { KK_GENERIC = 0, KK_STREAM3D, KK_TMA3D, KK_TILE2D, KK_TILE1D, KK_BOUNDARY, KK_DIAG, KK_COMM, KK_COUNT };
const char *kKindName[KK_COUNT] = {"stage_generic", "stage3d_stream", "stage3d_tma", "stage2d_tile",
                                   "stage1d_tile", "stage_boundary", "diag", "peer_barrier"};
static_assert(KK_COUNT <= NLSE_MAX_KINDS, "too many kernel kinds");

struct TimedLaunch { int kind; cudaEvent_t a, b; int64_t points; };

#ifndef NLSE_TMA_P
#define NLSE_TMA_P 3
#endif
#ifndef NLSE_TMA_P1
#define NLSE_TMA_P1 3
#endif
constexpr int TMA_P1 = NLSE_TMA_P1;  // ... for stage 1 (Y and V only: a deeper Y ring fits)
constexpr int TMA_P = NLSE_TMA_P;  // TMA ring prefetch depth of the Y planes (planes ahead; 2 and 4 measured slower, r01 ab1)
constexpr int GRAPH_STEPS = 8;  // RK4 steps per captured CUDA graph

enum { BUF_PSI = 0, BUF_TMP = 1, BUF_OUT = 2 };

struct DistBlob {               // what nlse_dist_export writes (NLSE_DIST_HANDLE_BYTES)
    uint32_t magic, version;
    int32_t rank, nranks;
    int64_t nloc;
    int32_t pid, device;
    cudaIpcMemHandle_t h[4];    // Psi, Psi_tmp, Psi_out allocations, comm block
};
static_assert(sizeof(DistBlob) <= NLSE_DIST_HANDLE_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0x4e4c5345u;  // "NLSE"

}  // namespace

struct StreamHolder {
    cudaStream_t s = nullptr;
    ~StreamHolder() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } }
};

struct nlse_ctx {
    int ndim = 0;
    int64_t dims[3] = {1, 1, 1};    // global grid
    double h = 0, a = 0, s = 0;
    nlse_bc bc = NLSE_BC_DIRICHLET;
    nlse_order order = NLSE_CD2;
    nlse_precision prec = NLSE_FP64;
    uint32_t flags = 0;
    Grid g{};                        // owned grid (the slab in slab mode)
    int eb = 8;                      // sizeof(real)
    bool hasV = false;
    // halo'd buffers: allocation base (plane -zghost) and plane-0 pointer
    void *alloc[3] = {nullptr, nullptr, nullptr};
    void *buf[3] = {nullptr, nullptr, nullptr};
    void *K = nullptr, *V = nullptr;
    void *fz = nullptr, *fp = nullptr;   // MSD 3D TMA path: stored F(b') (see StageArgs)
    int per2 = 0;
    int *d_div = nullptr;
    int *h_div = nullptr;            // pinned
    int *d_steps = nullptr;          // device counter of completed steps (divergence report)
    // CUDA graph of GRAPH_STEPS steps for the current k (nlse_step with many steps)
    cudaGraphExec_t graph_exec = nullptr;
    double graph_k = 0;
    double *d_partial = nullptr, *d_result = nullptr, *h_result = nullptr;
    int diag_blocks = 0;
    cudaStream_t stream = nullptr;
    std::shared_ptr<StreamHolder> stream_ref;   // virtual ranks of one group share one stream
    cudaStream_t side_stream = nullptr;          // 2D/3D boundary kernel, forked / joined per stage
    cudaStream_t io_stream = nullptr;            // nlse_run_frames downloads
    void *snap[2] = {nullptr, nullptr};          // nlse_run_frames: double2 snapshots of Psi
    cudaEvent_t ev_snap[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int device = 0;
    int64_t steps_done = 0;
    int64_t device_bytes = 0;
    std::string err;
    bool sticky = false;
    bool timing = false;
    std::vector<TimedLaunch> pending;
    std::vector<cudaEvent_t> event_pool;
    double kind_ms[KK_COUNT] = {0};
    int64_t kind_launches[KK_COUNT] = {0};
    int64_t kind_points[KK_COUNT] = {0};
    int interior_kind = KK_GENERIC;
    bool tma = false;
    int tma_ty = 8;                  // TMA kernel tile height (8: 256 threads, 16: 512 threads)
    Tma3Maps maps{};
    // slab mode
    bool dist = false;
    int rank = 0, nranks = 1;
    int64_t z0 = 0;
    CommBlock *comm = nullptr;
    bool connected = false;
    void *peer_alloc[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};  // [buf][lo, hi]
    int64_t peer_nloc[2] = {0, 0};
    CommBlock *peer_comm[MAX_RANKS] = {nullptr};
    std::vector<void *> ipc_opened;
    bool ghost_stale = false;
    bool virtual_group = false;      // connected by nlse_dist_connect_local: _group calls only
    bool persist1d = false;          // 1D: one persistent CTA per nlse_step call
};

namespace {

nlse_status fail(nlse_ctx *c, nlse_status st, const std::string &msg) {
    if (c) {
        c->err = msg;
        if (st == NLSE_ERR_CUDA) c->sticky = true;
    } else {
        g_create_error = msg;
    }
    return st;
}

#define CUDA_TRY(ctx, expr)                                                                      \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? NLSE_ERR_OOM : NLSE_ERR_CUDA,     \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                     \
    } while (0)

cudaEvent_t take_event(nlse_ctx *c) {
    if (!c->event_pool.empty()) { cudaEvent_t e = c->event_pool.back(); c->event_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct LaunchTimer {
    nlse_ctx *c; int kind; int64_t pts; cudaEvent_t a = nullptr;
    LaunchTimer(nlse_ctx *c_, int kind_, int64_t pts_) : c(c_), kind(kind_), pts(pts_) {
        if (c->timing) { a = take_event(c); cudaEventRecord(a, c->stream); }
    }
    ~LaunchTimer() {
        if (c->timing) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, c->stream);
            c->pending.push_back({kind, a, b, pts});
        }
    }
};

void collect_timing(nlse_ctx *c) {
    for (auto &t : c->pending) {
        float ms = 0;
        cudaEventElapsedTime(&ms, t.a, t.b);
        c->kind_ms[t.kind] += ms;
        c->kind_launches[t.kind] += 1;
        c->kind_points[t.kind] += t.points;
        c->event_pool.push_back(t.a);
        c->event_pool.push_back(t.b);
    }
    c->pending.clear();
}

template <typename T>
Consts<T> make_consts(const nlse_ctx *c, double kc) {
    Consts<T> k;
    k.ih2 = T(1.0 / (c->h * c->h));
    k.c76 = T(7.0 / 6.0);
    k.c112 = T(1.0 / 12.0);
    k.c16h2 = T(1.0 / (6.0 * c->h * c->h));
    k.a = T(c->a);
    k.s = T(c->s);
    k.inv_a = T(1.0 / c->a);
    k.eps2 = sizeof(T) == 8 ? T(1e-24) : T(1e-12);
    k.kc = T(kc);
    return k;
}

inline unsigned blocks_for(int64_t n, int threads) { return unsigned((n + threads - 1) / threads); }
inline int halo_w(const nlse_ctx *c) { return c->order == NLSE_2SHOC4 ? 2 : 1; }

// ------------------------------------------------------------------ TMA descriptors

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 3D map over [d2][d1][d0] elements of T (d0 fastest), box {b0, b1, 1}.
bool make_map(CUtensorMap *m, void *base, int eb, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * uint64_t(eb), d0 * d1 * uint64_t(eb)};
    cuuint32_t box[3] = {b0, b1, 1}, estr[3] = {1, 1, 1};
    if (strides[0] % 16 || strides[1] % 16) return false;
    // L2 promotion of the TMA reads: NLSE_TMA_L2PROMO = 0 (none) / 64 / 128 / 256 (default) bytes
    static const CUtensorMapL2promotion promo = [] {
        const char *e = getenv("NLSE_TMA_L2PROMO");
        const int v = e ? std::atoi(e) : 256;
        return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                      : (v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                 : (v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B));
    }();
    CUresult r = enc(m, eb == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The stage kernel finishes the x-face boundary points itself (StageArgs::xfuse) when every
// tile that owns x-face points runs the lean face-aware loop (t3_lean_ok in stage3d_tma.cuh:
// no face point on a tile's ring, no x face on lane 0 of a tile past x = 0).
bool xfuse_mode(const nlse_ctx *c) {
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

template <typename T, int ORDER, int TYV>
bool build_maps(nlse_ctx *c) {
    using Cfg = T3Cfg<T, ORDER, TMA_P, TYV>;
    const uint64_t nx = c->g.nx, ny = c->g.ny, nz = c->g.nz, nza = nz + 2 * c->g.zghost;
    const int eb = int(sizeof(T));
    bool ok = true;
    for (int b = 0; b < 3; b++)
        ok = ok && make_map(&c->maps.y[b], c->alloc[b], eb, 2 * nx, ny, nza, Cfg::BOX_Y_X, Cfg::BOX_Y_Y);
    ok = ok && make_map(&c->maps.psi, c->alloc[BUF_PSI], eb, 2 * nx, ny, nza, Cfg::BOX_C_X, Cfg::BOX_O_Y);
    ok = ok && make_map(&c->maps.k, c->K, eb, 2 * nx, ny, nz, Cfg::BOX_C_X, Cfg::BOX_O_Y);
    if (c->V) ok = ok && make_map(&c->maps.v, c->V, eb, nx, ny, nz, Cfg::BOX_R_X, Cfg::BOX_O_Y);
    else c->maps.v = c->maps.k;   // never dereferenced without a V array
    return ok;
}

// ------------------------------------------------------------------ stage launches

int ybuf_of_stage(int stage) { return stage == 1 ? BUF_PSI : (stage == 3 ? BUF_OUT : BUF_TMP); }
int obuf_of_stage(int stage) { return stage == 1 ? BUF_TMP : (stage == 2 ? BUF_OUT : (stage == 3 ? BUF_TMP : BUF_PSI)); }

template <typename T, int ORDER, int BC, int STAGE, int TYV>
void launch_tma3d_ty(nlse_ctx *c, const StageArgs<T> &A) {
    constexpr int PS = STAGE == 1 ? TMA_P1 : TMA_P;
    using Cfg = T3Cfg<T, ORDER, PS, TYV, STAGE != 1>;
    const int64_t nx = A.g.nx, ny = A.g.ny;
    const int64_t mz = A.g.nz - A.g.zf_lo - A.g.zf_hi;
    const unsigned gx = unsigned((nx + Cfg::TX - 1) / Cfg::TX);
    const unsigned gy = unsigned((ny + Cfg::TY - 1) / Cfg::TY);
    // z chunks: at most 128 planes (L2 locality of neighbouring tiles, r01e), and the
    // chunk count that minimises (waves of resident CTAs) x (planes per chunk + the ~4-plane
    // prologue), so that small grids fill the GPU in whole waves
    const int64_t cols = int64_t(gx) * gy;
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(stage3d_tma<T, ORDER, BC, STAGE, PS, TYV>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage3d_tma<T, ORDER, BC, STAGE, PS, TYV>,
                                                      Cfg::NT, Cfg::SMEM);
        if (per_sm < 1) per_sm = 1;
    }
    static int nsm = 0;
    if (!nsm && cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess) nsm = 148;
    const int64_t resident = int64_t(nsm) * per_sm;
    int64_t zchunk = mz, best = -1;
    for (int64_t nzc = (mz + 127) / 128; nzc <= mz; nzc++) {
        const int64_t ch = (mz + nzc - 1) / nzc;
        const int64_t waves = (cols * nzc + resident - 1) / resident;
        const int64_t cost = waves * (ch + 4);
        if (best < 0 || cost < best) { best = cost; zchunk = ch; }
        if (ch <= 4) break;
    }
    static const int64_t env_chunk = [] {
        const char *e = getenv("NLSE_ZCHUNK");
        return e ? std::atoll(e) : int64_t(0);
    }();
    if (env_chunk > 0) zchunk = env_chunk;
    if (zchunk > mz) zchunk = mz;
    const unsigned gz = unsigned((mz + zchunk - 1) / zchunk);
    const int64_t items = int64_t(gx) * gy * gz;
    // debug / measurement / tests: NLSE_FORCE_EDGE=1 runs every tile on the face-aware lean
    // loop, =2 every tile on the per-point face path (t3_run, EDGE)
    const char *fe = getenv("NLSE_FORCE_EDGE");
    const int force_edge = (fe && (fe[0] == '1' || fe[0] == '2')) ? fe[0] - '0' : 0;
    stage3d_tma<T, ORDER, BC, STAGE, PS, TYV><<<unsigned(items), Cfg::NT, Cfg::SMEM, c->stream>>>(
        c->maps.y[ybuf_of_stage(STAGE)], c->maps.psi, c->maps.k, c->maps.v, A, int(zchunk), int(gx), int(gy),
        force_edge);
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
        if (DIM == 3) {
            if (c->interior_kind == KK_TMA3D) launch_tma3d<T, ORDER, BC, STAGE>(c, A);
            else launch_stream3d<T, ORDER, BC, STAGE>(A, c->stream);
        } else if (DIM == 2) {
            launch_tile2d<T, ORDER, BC, STAGE>(A, c->stream);
        } else {
            launch_tile1d<T, ORDER, BC, STAGE>(A, c->stream);
        }
    }
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
    const int64_t sz = c->g.sz, zg = c->g.zghost;
    if (c->peer_alloc[b][0]) lo = (cplx<T> *)c->peer_alloc[b][0] + (zg + c->peer_nloc[0]) * sz;
    if (c->peer_alloc[b][1]) hi = (cplx<T> *)c->peer_alloc[b][1] + (zg - c->g.nz) * sz;
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
        const int64_t state_bytes = c->g.n * int64_t(4 * 2 * c->eb + (c->hasV ? c->eb : 0));
        A.stream_hints = env_hints >= 0 ? env_hints : 0;   // r01y: evict-first hints were slower
        (void)state_bytes;
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

template <typename F>
auto dispatch(nlse_ctx *c, F &&f) {
    auto by_bc = [&](auto T, auto DIM, auto ORD) {
        if (c->bc == NLSE_BC_MSD) return f(T, DIM, ORD, std::integral_constant<int, BC_MSD>());
        if (c->bc == NLSE_BC_L0) return f(T, DIM, ORD, std::integral_constant<int, BC_L0>());
        return f(T, DIM, ORD, std::integral_constant<int, BC_DIRICHLET>());
    };
    auto by_order = [&](auto T, auto DIM) {
        if (c->order == NLSE_2SHOC4) return by_bc(T, DIM, std::integral_constant<int, ORDER_2SHOC>());
        return by_bc(T, DIM, std::integral_constant<int, ORDER_CD>());
    };
    auto by_dim = [&](auto T) {
        if (c->ndim == 1) return by_order(T, std::integral_constant<int, 1>());
        if (c->ndim == 2) return by_order(T, std::integral_constant<int, 2>());
        return by_order(T, std::integral_constant<int, 3>());
    };
    if (c->prec == NLSE_FP64) return by_dim(double());
    return by_dim(float());
}

void enqueue_stage(nlse_ctx *c, int stage, double k, int step) {
    dispatch(c, [&](auto T, auto DIM, auto ORD, auto BCK) {
        enqueue_stage_t<decltype(T), decltype(DIM)::value, decltype(ORD)::value, decltype(BCK)::value>(c, stage, k,
                                                                                                     step);
        return 0;
    });
}

// ------------------------------------------------------------------ slab-mode plumbing

// Barrier with the z neighbours (full = false) or with every rank (full = true).
// mode 3 = signal + wait (one kernel); the group calls enqueue mode 1 for every rank,
// then mode 2 (same epoch: pass bump = false for the wait half).
void enqueue_barrier(nlse_ctx *c, bool full, int mode = 3) {
    if (!c->dist) return;
    BarrierArgs b{};
    b.own = c->comm;
    b.me = c->rank;
    for (int j = 0; j < c->nranks; j++) {
        if (j == c->rank) continue;
        if (!full && j != c->rank - 1 && j != c->rank + 1) continue;
        b.sig[b.nsig++] = c->peer_comm[j];
        b.wait_rank[b.nwait++] = j;
    }
    if (b.nsig == 0) return;
    LaunchTimer lt(c, KK_COMM, 0);
    peer_barrier<<<1, 32, 0, c->stream>>>(b, mode);
}

// Copy the first / last w owned planes of Psi into the neighbours' ghost planes (after
// nlse_set_psi*), then barrier (mode as enqueue_barrier).
nlse_status enqueue_halo_refresh(nlse_ctx *c, int mode = 3) {
    if (!c->dist || !c->ghost_stale) return NLSE_OK;
    const int w = halo_w(c);
    const size_t cb = size_t(2 * c->eb), plane = size_t(c->g.sz) * cb;
    if (c->peer_alloc[BUF_PSI][0]) {
        char *dst = (char *)c->peer_alloc[BUF_PSI][0] + (c->g.zghost + c->peer_nloc[0]) * plane;
        CUDA_TRY(c, cudaMemcpyAsync(dst, c->buf[BUF_PSI], w * plane, cudaMemcpyDefault, c->stream));
    }
    if (c->peer_alloc[BUF_PSI][1]) {
        char *dst = (char *)c->peer_alloc[BUF_PSI][1] + (c->g.zghost - w) * plane;
        const char *src = (const char *)c->buf[BUF_PSI] + (c->g.nz - w) * plane;
        CUDA_TRY(c, cudaMemcpyAsync(dst, src, w * plane, cudaMemcpyDefault, c->stream));
    }
    enqueue_barrier(c, false, mode);
    c->ghost_stale = false;
    return NLSE_OK;
}

nlse_status check_ctx(nlse_ctx *c) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (c->sticky) return NLSE_ERR_CUDA;
    if (c->dist && !c->connected) return fail(c, NLSE_ERR_COMM, "slab-mode context used before nlse_dist_connect");
    return NLSE_OK;
}

nlse_status check_step_args(nlse_ctx *c, double k, int64_t nsteps) {
    if (!std::isfinite(k) || !(k > 0)) return fail(c, NLSE_ERR_ARG, "k must be finite and > 0");
    if (nsteps < 0) return fail(c, NLSE_ERR_ARG, "nsteps must be >= 0");
    double kmax = c->h * c->h / (double(c->ndim) * std::sqrt(2.0) * c->a);
    if (c->order == NLSE_2SHOC4) kmax *= 0.75;
    if (k > kmax && !(c->flags & NLSE_FLAG_FORCE_DT)) {
        char buf[160];
        snprintf(buf, sizeof buf, "k = %.9g exceeds the linear stability bound %.9g (P:363-372); use NLSE_FLAG_FORCE_DT",
                 k, kmax);
        return fail(c, NLSE_ERR_UNSTABLE, buf);
    }
    return NLSE_OK;
}

// Enqueue one RK4 stage of step n of the current launch sequence, followed (slab mode)
// by the neighbour barrier (mode as enqueue_barrier).
void enqueue_step_stage(nlse_ctx *c, int stage, double k, int64_t n, int mode = 3) {
    enqueue_stage(c, stage, k, int(std::min<int64_t>(n, INT32_MAX / 2)));
    enqueue_barrier(c, false, mode);
}

void enqueue_add_steps(nlse_ctx *c, int64_t n) {
    add_steps<<<1, 1, 0, c->stream>>>(c->d_steps, int(n));
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
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(rk4_1d_persistent<T, ORDER, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        attr = true;
    }
    LaunchTimer lt(c, KK_TILE1D, c->g.n * nsteps);
    rk4_1d_persistent<T, ORDER, BC><<<1, P1_THREADS, smem, c->stream>>>(P);
}

bool use_persist1d(const nlse_ctx *c) {
    if (c->ndim != 1 || c->interior_kind == KK_GENERIC) return false;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const size_t need = c->prec == NLSE_FP64 ? persist1d_smem<double>(int(c->g.nx), c->hasV, c->order == NLSE_2SHOC4)
                                             : persist1d_smem<float>(int(c->g.nx), c->hasV, c->order == NLSE_2SHOC4);
    return c->g.nx <= (int64_t(1) << 30) && need <= size_t(optin);
}

void drop_graph(nlse_ctx *c) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
}

// Capture GRAPH_STEPS steps (all launches, barriers and the step-counter update) once
// per k; false if capture is unavailable (then the caller launches directly).
bool ensure_graph(nlse_ctx *c, double k) {
    if (c->graph_exec && c->graph_k == k) return true;
    drop_graph(c);
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    for (int n = 0; n < GRAPH_STEPS; n++)
        for (int s = 1; s <= 4; s++) enqueue_step_stage(c, s, k, n);
    enqueue_add_steps(c, GRAPH_STEPS);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->graph_exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c->graph_exec = nullptr;
        return false;
    }
    c->graph_k = k;
    return true;
}

bool graphs_enabled(const nlse_ctx *c, int64_t nsteps) {
    static const bool env_off = [] {
        const char *e = getenv("NLSE_GRAPHS");
        return e && e[0] == '0';
    }();
    return !env_off && !c->timing && !c->virtual_group && nsteps >= 2 * GRAPH_STEPS;
}

nlse_status finish_steps(nlse_ctx *c, int64_t nsteps) {
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->h_div, c->d_div, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->timing) collect_timing(c);
    c->steps_done += nsteps;
    if (*c->h_div != INT32_MAX) {
        char buf[128];
        snprintf(buf, sizeof buf, "Psi became non-finite at step %d (0-based, counted from context creation)", *c->h_div);
        return fail(c, NLSE_ERR_DIVERGED, buf);
    }
    return NLSE_OK;
}

// diagnostics, local part: partial sums over the owned points (unscaled in slab mode)
void enqueue_diag_local(nlse_ctx *c, double hd) {
    const double ih2 = 1.0 / (c->h * c->h);
    LaunchTimer lt(c, KK_DIAG, c->g.n);
    auto go = [&](auto T, auto DIM) {
        using TT = decltype(T);
        diag_partial<TT, decltype(DIM)::value><<<c->diag_blocks, DIAG_THREADS, 0, c->stream>>>(
            (const cplx<TT> *)c->buf[BUF_PSI], (const TT *)c->V, c->g, c->a, c->s, ih2, c->d_partial);
    };
    if (c->prec == NLSE_FP64) {
        if (c->ndim == 1) go(double(), std::integral_constant<int, 1>());
        else if (c->ndim == 2) go(double(), std::integral_constant<int, 2>());
        else go(double(), std::integral_constant<int, 3>());
    } else {
        if (c->ndim == 1) go(float(), std::integral_constant<int, 1>());
        else if (c->ndim == 2) go(float(), std::integral_constant<int, 2>());
        else go(float(), std::integral_constant<int, 3>());
    }
    diag_final<<<1, DIAG_THREADS, 0, c->stream>>>(c->d_partial, c->diag_blocks, c->dist ? 1.0 : hd, c->d_result);
}

void enqueue_diag_push(nlse_ctx *c) {
    PushArgs a{};
    a.me = c->rank;
    for (int j = 0; j < c->nranks; j++) a.dst[a.n++] = j == c->rank ? c->comm : c->peer_comm[j];
    diag_push<<<1, 32, 0, c->stream>>>(c->d_result, a);
}

double hd_of(const nlse_ctx *c) {
    double hd = c->h;
    for (int d = 1; d < c->ndim; d++) hd *= c->h;
    return hd;
}

nlse_status finish_diag(nlse_ctx *c, double *mass, double *ham) {
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->d_result, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->timing) collect_timing(c);
    *mass = c->h_result[0];
    *ham = c->h_result[1];
    return NLSE_OK;
}

template <typename T>
__global__ void widen_psi(const cplx<T> *src, double2 *dst, int64_t n) {
    int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n) { cplx<T> v = src[q]; dst[q] = make_double2(double(v.x), double(v.y)); }
}
template <typename T>
__global__ void narrow_psi(const double2 *src, cplx<T> *dst, int64_t n) {
    int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n) { double2 v = src[q]; cplx<T> r; r.x = T(v.x); r.y = T(v.y); dst[q] = r; }
}
template <typename T>
__global__ void narrow_real(const double *src, T *dst, int64_t n) {
    int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n) dst[q] = T(src[q]);
}

double linear_bound(int ndim, double a, double h, nlse_order order) {
    double k = h * h / (double(ndim) * std::sqrt(2.0) * a);
    return order == NLSE_2SHOC4 ? 0.75 * k : k;
}

// Host double (re, im) -> device working precision, staged through Psi_out (scratch
// between calls) for fp32.
nlse_status upload_complex(nlse_ctx *c, const double *host, void *dev) {
    const size_t n = size_t(c->g.n);
    if (c->prec == NLSE_FP64) {
        CUDA_TRY(c, cudaMemcpyAsync(dev, host, n * 16, cudaMemcpyHostToDevice, c->stream));
    } else {
        const size_t chunk = n / 2 > 0 ? n / 2 : 1;  // outb holds n float2 = n/2 double2
        double2 *scratch = (double2 *)c->buf[BUF_OUT];
        for (size_t off = 0; off < n; off += chunk) {
            size_t m = std::min(chunk, n - off);
            CUDA_TRY(c, cudaMemcpyAsync(scratch, host + 2 * off, m * 16, cudaMemcpyHostToDevice, c->stream));
            narrow_psi<float><<<blocks_for(m, 256), 256, 0, c->stream>>>(scratch, (float2 *)dev + off, int64_t(m));
            CUDA_TRY(c, cudaGetLastError());
        }
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

nlse_status download_complex(nlse_ctx *c, const void *dev, double *host) {
    const size_t n = size_t(c->g.n);
    if (c->prec == NLSE_FP64) {
        CUDA_TRY(c, cudaMemcpyAsync(host, dev, n * 16, cudaMemcpyDeviceToHost, c->stream));
    } else {
        const size_t chunk = n / 2 > 0 ? n / 2 : 1;
        double2 *scratch = (double2 *)c->buf[BUF_OUT];
        for (size_t off = 0; off < n; off += chunk) {
            size_t m = std::min(chunk, n - off);
            widen_psi<float><<<blocks_for(m, 256), 256, 0, c->stream>>>((const float2 *)dev + off, scratch, int64_t(m));
            CUDA_TRY(c, cudaGetLastError());
            CUDA_TRY(c, cudaMemcpyAsync(host + 2 * off, scratch, m * 16, cudaMemcpyDeviceToHost, c->stream));
        }
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

const char *env_kernel() {
    const char *e = getenv("NLSE_3D_KERNEL");
    return e ? e : "";
}

nlse_status create_common(int ndim, const int64_t dims[3], double h, double a, double s, const double *V,
                          nlse_bc bc, nlse_order order, nlse_precision prec, uint32_t flags, int rank, int nranks,
                          bool dist, nlse_ctx **out) {
    if (!out) return fail(nullptr, NLSE_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (ndim < 1 || ndim > 3) return fail(nullptr, NLSE_ERR_ARG, "ndim must be 1, 2 or 3");
    if (!dims) return fail(nullptr, NLSE_ERR_ARG, "dims is NULL");
    for (int d = 0; d < 3; d++) {
        if (d < ndim && dims[d] < 3) return fail(nullptr, NLSE_ERR_ARG, "every active dimension needs >= 3 points");
        if (d >= ndim && dims[d] != 1) return fail(nullptr, NLSE_ERR_ARG, "inactive dimensions must be 1");
    }
    if (!(h > 0) || !std::isfinite(h)) return fail(nullptr, NLSE_ERR_ARG, "h must be finite and > 0");
    if (!(a > 0) || !std::isfinite(a)) return fail(nullptr, NLSE_ERR_ARG, "a must be finite and > 0");
    if (!std::isfinite(s)) return fail(nullptr, NLSE_ERR_ARG, "s must be finite");
    if (bc != NLSE_BC_DIRICHLET && bc != NLSE_BC_MSD && bc != NLSE_BC_L0) return fail(nullptr, NLSE_ERR_ARG, "unknown bc");
    if (order != NLSE_CD2 && order != NLSE_2SHOC4) return fail(nullptr, NLSE_ERR_ARG, "unknown order");
    if (prec != NLSE_FP32 && prec != NLSE_FP64) return fail(nullptr, NLSE_ERR_ARG, "unknown precision");
    if (dims[0] * dims[1] >= (int64_t(1) << 31) || dims[2] >= (int64_t(1) << 31))
        return fail(nullptr, NLSE_ERR_ARG, "an xy plane must have fewer than 2^31 points (32-bit in-plane indexing)");
    const int w = order == NLSE_2SHOC4 ? 2 : 1;
    int64_t z0 = 0, nloc = dims[2];
    if (dist) {
        if (ndim != 3) return fail(nullptr, NLSE_ERR_ARG, "slab mode partitions 3D grids only (1D/2D run as replicas)");
        if (nranks < 1 || nranks > NLSE_MAX_RANKS || rank < 0 || rank >= nranks)
            return fail(nullptr, NLSE_ERR_ARG, "rank / nranks out of range");
        nlse_slab_range(dims[2], nranks, rank, &z0, &nloc);
        if (nloc < 2 * w) return fail(nullptr, NLSE_ERR_ARG, "every slab needs at least 2w planes (w = 1 CD, 2 2SHOC)");
    }
    const int64_t n = dims[0] * dims[1] * nloc;
    if (V) {
        for (int64_t q = 0; q < n; q++)
            if (!std::isfinite(V[q])) return fail(nullptr, NLSE_ERR_ARG, "V must be finite");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, NLSE_ERR_CUDA, "no CUDA device (there is no CPU fallback)");

    nlse_ctx *c = new nlse_ctx();
    c->ndim = ndim;
    for (int d = 0; d < 3; d++) c->dims[d] = dims[d];
    c->h = h; c->a = a; c->s = s; c->bc = bc; c->order = order; c->prec = prec; c->flags = flags;
    c->dist = dist; c->rank = rank; c->nranks = nranks; c->z0 = z0;
    c->g.nx = dims[0]; c->g.ny = dims[1]; c->g.nz = nloc;
    c->g.sy = dims[0]; c->g.sz = dims[0] * dims[1]; c->g.n = n;
    c->g.zf_lo = (!dist || rank == 0) ? 1 : 0;
    c->g.zf_hi = (!dist || rank == nranks - 1) ? 1 : 0;
    c->g.zghost = dist ? w : 0;
    c->eb = prec == NLSE_FP64 ? 8 : 4;
    c->hasV = V != nullptr;
    cudaGetDevice(&c->device);
    if (flags & NLSE_FLAG_GENERIC_KERNELS) c->interior_kind = KK_GENERIC;
    else c->interior_kind = ndim == 3 ? KK_TMA3D : (ndim == 2 ? KK_TILE2D : KK_TILE1D);

    auto bail = [&](nlse_status st) { g_create_error = c->err; nlse_destroy(c); return st; };
#define CREATE_TRY(expr)                                                                         \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) {                                                                 \
            fail(c, e_ == cudaErrorMemoryAllocation ? NLSE_ERR_OOM : NLSE_ERR_CUDA,              \
                 std::string(#expr) + ": " + cudaGetErrorString(e_));                            \
            return bail(e_ == cudaErrorMemoryAllocation ? NLSE_ERR_OOM : NLSE_ERR_CUDA);         \
        }                                                                                        \
    } while (0)

    c->stream_ref = std::make_shared<StreamHolder>();
    CREATE_TRY(cudaStreamCreateWithFlags(&c->stream_ref->s, cudaStreamNonBlocking));
    c->stream = c->stream_ref->s;
    if (ndim >= 2) {
        CREATE_TRY(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
        CREATE_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CREATE_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    const size_t cb = size_t(2 * c->eb), plane = size_t(c->g.sz) * cb;
    const size_t halo_bytes = size_t(n) * cb + 2 * size_t(c->g.zghost) * plane;
    for (int b = 0; b < 3; b++) {
        CREATE_TRY(cudaMalloc(&c->alloc[b], halo_bytes));
        CREATE_TRY(cudaMemsetAsync(c->alloc[b], 0, halo_bytes, c->stream));
        c->buf[b] = (char *)c->alloc[b] + size_t(c->g.zghost) * plane;
    }
    CREATE_TRY(cudaMalloc(&c->K, size_t(n) * cb));
    c->device_bytes = int64_t(3 * halo_bytes + size_t(n) * cb);
    if (V) {
        CREATE_TRY(cudaMalloc(&c->V, size_t(n) * c->eb));
        c->device_bytes += int64_t(size_t(n) * c->eb);
        if (prec == NLSE_FP64) {
            CREATE_TRY(cudaMemcpyAsync(c->V, V, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
        } else {
            // stage the double V through K (n complex floats = n doubles) and round once on the device
            CREATE_TRY(cudaMemcpyAsync(c->K, V, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
            narrow_real<float><<<blocks_for(n, 256), 256, 0, c->stream>>>((const double *)c->K, (float *)c->V, n);
            CREATE_TRY(cudaGetLastError());
        }
    }
    if (dist) {
        CREATE_TRY(cudaMalloc(&c->comm, sizeof(CommBlock)));
        CREATE_TRY(cudaMemsetAsync(c->comm, 0, sizeof(CommBlock), c->stream));
    }
    CREATE_TRY(cudaMalloc(&c->d_steps, sizeof(int)));
    CREATE_TRY(cudaMemsetAsync(c->d_steps, 0, sizeof(int), c->stream));
    CREATE_TRY(cudaMalloc(&c->d_div, sizeof(int)));
    CREATE_TRY(cudaMallocHost(&c->h_div, sizeof(int)));
    int big = INT32_MAX;
    CREATE_TRY(cudaMemcpyAsync(c->d_div, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    c->diag_blocks = nsm * 8;
    CREATE_TRY(cudaMalloc(&c->d_partial, sizeof(double) * 2 * c->diag_blocks));
    CREATE_TRY(cudaMalloc(&c->d_result, sizeof(double) * 2));
    CREATE_TRY(cudaMallocHost(&c->h_result, sizeof(double) * 2));
    CREATE_TRY(cudaStreamSynchronize(c->stream));
    if (c->interior_kind == KK_TMA3D) {
        const std::string ek = env_kernel();
        bool ok = ek != "v1";
        const char *ety = getenv("NLSE_TMA_TY");
        c->tma_ty = (ety && std::atoi(ety) == 8) ? 8 : 16;   // 16 measured faster (r01f, r01j)
        if (ok) {
            auto bm = [&](auto TYc) {
                constexpr int TYV = decltype(TYc)::value;
                if (prec == NLSE_FP64)
                    return order == NLSE_2SHOC4 ? build_maps<double, ORDER_2SHOC, TYV>(c) : build_maps<double, ORDER_CD, TYV>(c);
                return order == NLSE_2SHOC4 ? build_maps<float, ORDER_2SHOC, TYV>(c) : build_maps<float, ORDER_CD, TYV>(c);
            };
            ok = c->tma_ty == 16 ? bm(std::integral_constant<int, 16>()) : bm(std::integral_constant<int, 8>());
        }
        // TMA needs 16-byte row strides (complex rows: nx even for fp32; V rows: nx*sizeof(T) % 16)
        if (!ok) c->interior_kind = KK_STREAM3D;
        c->tma = ok;
        // MSD: the interior kernel stores F(b') and a light pass after it forms the boundary
        // outputs.  Recomputing the two-step Laplacian at b' instead costs ~0.8 ms per stage at
        // 1024^3, and even at 87x87x203, where that kernel could run concurrently on the side
        // stream, it is slower (17.5 us on the few SMs the interior kernel leaves free vs the
        // serial 8.3 us light pass: 194 vs 150 us/step, r01 probe2).  NLSE_MSD_FB=0: recompute.
        const char *efb = getenv("NLSE_MSD_FB");
        const bool want_fb = !(efb && efb[0] == '0');
        if (ok && want_fb && bc == NLSE_BC_MSD && c->g.nx >= 5 && c->g.ny >= 5) {
            c->per2 = int(2 * (c->g.nx - 2) + 2 * (c->g.ny - 4));
            const size_t fzb = size_t(2) * size_t(c->g.sz) * cb, fpb = size_t(c->g.nz) * size_t(c->per2) * cb;
            CREATE_TRY(cudaMalloc(&c->fz, fzb));
            CREATE_TRY(cudaMalloc(&c->fp, fpb));
            c->device_bytes += int64_t(fzb + fpb);
        }
    }
#undef CREATE_TRY
    c->persist1d = use_persist1d(c);
    c->connected = !dist;
    *out = c;
    return NLSE_OK;
}

// nsteps RK4 steps on the context stream: the persistent 1D kernel, or replays of the CUDA
// graph of GRAPH_STEPS steps plus direct launches for the remainder.
nlse_status enqueue_steps(nlse_ctx *c, double k, int64_t nsteps) {
    if (c->persist1d) {
        dispatch(c, [&](auto T, auto DIM, auto ORD, auto BCK) {
            if constexpr (decltype(DIM)::value == 1)
                launch_persist1d<decltype(T), decltype(ORD)::value, decltype(BCK)::value>(c, k, nsteps);
            return 0;
        });
        enqueue_add_steps(c, nsteps);
        return NLSE_OK;
    }
    int64_t done = 0;
    if (graphs_enabled(c, nsteps) && ensure_graph(c, k)) {
        for (; done + GRAPH_STEPS <= nsteps; done += GRAPH_STEPS)
            CUDA_TRY(c, cudaGraphLaunch(c->graph_exec, c->stream));
    }
    if (done < nsteps) {
        for (int64_t n = 0; n < nsteps - done; n++)
            for (int s = 1; s <= 4; s++) enqueue_step_stage(c, s, k, n);
        enqueue_add_steps(c, nsteps - done);
    }
    return NLSE_OK;
}

}  // namespace

extern "C" {

const char *nlse_status_string(nlse_status st) {
    switch (st) {
        case NLSE_OK: return "NLSE_OK";
        case NLSE_ERR_ARG: return "NLSE_ERR_ARG";
        case NLSE_ERR_UNSTABLE: return "NLSE_ERR_UNSTABLE";
        case NLSE_ERR_OOM: return "NLSE_ERR_OOM";
        case NLSE_ERR_CUDA: return "NLSE_ERR_CUDA";
        case NLSE_ERR_COMM: return "NLSE_ERR_COMM";
        case NLSE_ERR_DIVERGED: return "NLSE_ERR_DIVERGED";
    }
    return "NLSE_ERR_UNKNOWN";
}

const char *nlse_last_error(const nlse_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

nlse_status nlse_stability_bound(int ndim, double a, double h, nlse_order order, double *k_max, double *k_rec) {
    if (ndim < 1 || ndim > 3) return fail(nullptr, NLSE_ERR_ARG, "ndim must be 1, 2 or 3");
    if (!(a > 0) || !std::isfinite(a)) return fail(nullptr, NLSE_ERR_ARG, "a must be finite and > 0");
    if (!(h > 0) || !std::isfinite(h)) return fail(nullptr, NLSE_ERR_ARG, "h must be finite and > 0");
    if (order != NLSE_CD2 && order != NLSE_2SHOC4) return fail(nullptr, NLSE_ERR_ARG, "unknown order");
    double k = linear_bound(ndim, a, h, order);
    if (k_max) *k_max = k;
    if (k_rec) *k_rec = 0.8 * k;
    return NLSE_OK;
}

nlse_status nlse_slab_range(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *nloc) {
    if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z0 || !nloc)
        return fail(nullptr, NLSE_ERR_ARG, "nlse_slab_range: bad arguments");
    const int64_t base = nz / nranks, rem = nz % nranks;
    *nloc = base + (rank < rem ? 1 : 0);
    *z0 = int64_t(rank) * base + std::min<int64_t>(rank, rem);
    return NLSE_OK;
}

void nlse_destroy(nlse_ctx *c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto &t : c->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    for (void *p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    for (int b = 0; b < 3; b++) cudaFree(c->alloc[b]);
    cudaFree(c->K); cudaFree(c->V); cudaFree(c->comm); cudaFree(c->fz); cudaFree(c->fp);
    drop_graph(c);
    cudaFree(c->d_div); cudaFree(c->d_steps); cudaFree(c->d_partial); cudaFree(c->d_result);
    if (c->h_div) cudaFreeHost(c->h_div);
    if (c->h_result) cudaFreeHost(c->h_result);
    if (c->side_stream) { cudaStreamSynchronize(c->side_stream); cudaStreamDestroy(c->side_stream); }
    if (c->io_stream) { cudaStreamSynchronize(c->io_stream); cudaStreamDestroy(c->io_stream); }
    for (int b = 0; b < 2; b++) {
        cudaFree(c->snap[b]);
        if (c->ev_snap[b]) cudaEventDestroy(c->ev_snap[b]);
        if (c->ev_copied[b]) cudaEventDestroy(c->ev_copied[b]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    c->stream_ref.reset();    // destroys the stream with its last user
    delete c;
}

nlse_status nlse_create(int ndim, const int64_t dims[3], double h, double a, double s, const double *V,
                        nlse_bc bc, nlse_order order, nlse_precision prec, uint32_t flags, nlse_ctx **out) {
    return create_common(ndim, dims, h, a, s, V, bc, order, prec, flags, 0, 1, false, out);
}

nlse_status nlse_create_dist(int ndim, const int64_t dims[3], double h, double a, double s, const double *V_local,
                             nlse_bc bc, nlse_order order, nlse_precision prec, uint32_t flags, int rank, int nranks,
                             nlse_ctx **out) {
    return create_common(ndim, dims, h, a, s, V_local, bc, order, prec, flags, rank, nranks, true, out);
}

nlse_status nlse_dist_export(nlse_ctx *c, void *handle) {
    if (!c || !handle) return fail(c, NLSE_ERR_ARG, "ctx / handle is NULL");
    if (!c->dist) return fail(c, NLSE_ERR_ARG, "not a slab-mode context");
    DistBlob b{};
    b.magic = kBlobMagic; b.version = NLSE_ABI_VERSION;
    b.rank = c->rank; b.nranks = c->nranks; b.nloc = c->g.nz;
    b.pid = int32_t(getpid()); b.device = c->device;
    for (int i = 0; i < 3; i++) CUDA_TRY(c, cudaIpcGetMemHandle(&b.h[i], c->alloc[i]));
    CUDA_TRY(c, cudaIpcGetMemHandle(&b.h[3], c->comm));
    memset(handle, 0, NLSE_DIST_HANDLE_BYTES);
    memcpy(handle, &b, sizeof b);
    return NLSE_OK;
}

nlse_status nlse_dist_connect(nlse_ctx *c, const void *handles) {
    if (!c || !handles) return fail(c, NLSE_ERR_ARG, "ctx / handles is NULL");
    if (!c->dist) return fail(c, NLSE_ERR_ARG, "not a slab-mode context");
    if (c->connected) return fail(c, NLSE_ERR_ARG, "already connected");
    const char *hb = (const char *)handles;
    for (int j = 0; j < c->nranks; j++) {
        DistBlob b;
        memcpy(&b, hb + size_t(j) * NLSE_DIST_HANDLE_BYTES, sizeof b);
        if (b.magic != kBlobMagic || b.rank != j || b.nranks != c->nranks)
            return fail(c, NLSE_ERR_COMM, "handle " + std::to_string(j) + " is not rank " + std::to_string(j) + "'s export");
        if (j == c->rank) continue;
        if (b.pid == int32_t(getpid()))
            return fail(c, NLSE_ERR_COMM, "peer handles from the same process: use nlse_dist_connect_local");
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, b.h[3], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(c, NLSE_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        c->ipc_opened.push_back(p);
        c->peer_comm[j] = (CommBlock *)p;
        const int side = j == c->rank - 1 ? 0 : (j == c->rank + 1 ? 1 : -1);
        if (side < 0) continue;
        c->peer_nloc[side] = b.nloc;
        for (int i = 0; i < 3; i++) {
            e = cudaIpcOpenMemHandle(&p, b.h[i], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return fail(c, NLSE_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
            c->ipc_opened.push_back(p);
            c->peer_alloc[i][side] = p;
        }
    }
    c->peer_comm[c->rank] = c->comm;
    c->connected = true;
    c->ghost_stale = true;
    return NLSE_OK;
}

nlse_status nlse_dist_connect_local(nlse_ctx *const *ctxs, int n) {
    if (!ctxs || n < 1) return fail(nullptr, NLSE_ERR_ARG, "ctxs is NULL or n < 1");
    for (int j = 0; j < n; j++) {
        nlse_ctx *c = ctxs[j];
        if (!c || !c->dist || c->rank != j || c->nranks != n || c->connected)
            return fail(nullptr, NLSE_ERR_ARG, "ctxs must be the unconnected slab contexts of ranks 0..n-1 in order");
        if (c->device != ctxs[0]->device)
            return fail(nullptr, NLSE_ERR_ARG, "virtual ranks must share one device");
    }
    // one stream for the whole group: stream order then sequences the ranks' stages, and
    // every signal is enqueued before the waits that depend on it
    for (int j = 0; j < n; j++) cudaStreamSynchronize(ctxs[j]->stream);
    for (int j = 1; j < n; j++) {
        ctxs[j]->stream_ref = ctxs[0]->stream_ref;
        ctxs[j]->stream = ctxs[0]->stream;
    }
    for (int j = 0; j < n; j++) {
        nlse_ctx *c = ctxs[j];
        for (int i = 0; i < n; i++) c->peer_comm[i] = ctxs[i]->comm;
        for (int side = 0; side < 2; side++) {
            const int nb = side == 0 ? j - 1 : j + 1;
            if (nb < 0 || nb >= n) continue;
            c->peer_nloc[side] = ctxs[nb]->g.nz;
            for (int i = 0; i < 3; i++) c->peer_alloc[i][side] = ctxs[nb]->alloc[i];
        }
        c->connected = true;
        c->ghost_stale = true;
        c->virtual_group = n > 1;
    }
    return NLSE_OK;
}

nlse_status nlse_set_psi(nlse_ctx *c, const double *psi) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!psi) return fail(c, NLSE_ERR_ARG, "psi is NULL");
    st = upload_complex(c, psi, c->buf[BUF_PSI]);
    c->ghost_stale = c->dist;
    return st;
}

nlse_status nlse_get_psi(nlse_ctx *c, double *psi) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!psi) return fail(c, NLSE_ERR_ARG, "psi_out is NULL");
    return download_complex(c, c->buf[BUF_PSI], psi);
}

nlse_status nlse_set_psi_device(nlse_ctx *c, const void *d) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!d) return fail(c, NLSE_ERR_ARG, "d_psi is NULL");
    CUDA_TRY(c, cudaMemcpyAsync(c->buf[BUF_PSI], d, size_t(c->g.n) * 2 * c->eb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->ghost_stale = c->dist;
    return NLSE_OK;
}

nlse_status nlse_get_psi_device(nlse_ctx *c, void *d) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!d) return fail(c, NLSE_ERR_ARG, "d_psi is NULL");
    CUDA_TRY(c, cudaMemcpyAsync(d, c->buf[BUF_PSI], size_t(c->g.n) * 2 * c->eb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

nlse_status nlse_step(nlse_ctx *c, double k, int64_t nsteps) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (c->virtual_group) return fail(c, NLSE_ERR_ARG, "virtual ranks step together: use nlse_step_group");
    if ((st = check_step_args(c, k, nsteps))) return st;
    if (nsteps == 0) return NLSE_OK;
    if ((st = enqueue_halo_refresh(c))) return st;
    if ((st = enqueue_steps(c, k, nsteps))) return st;
    return finish_steps(c, nsteps);
}

nlse_status nlse_run_frames(nlse_ctx *c, double k, int64_t chunk, int nframes, double *frames) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (c->virtual_group) return fail(c, NLSE_ERR_ARG, "virtual ranks: nlse_run_frames is per process");
    if (chunk < 1 || nframes < 1 || !frames) return fail(c, NLSE_ERR_ARG, "chunk >= 1, nframes >= 1 and frames != NULL");
    if ((st = check_step_args(c, k, chunk))) return st;
    const size_t n = size_t(c->g.n), fb = n * sizeof(double2);
    if (!c->io_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->io_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
        if (!c->snap[b]) {
            CUDA_TRY(c, cudaMalloc(&c->snap[b], fb));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_snap[b], cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
            c->device_bytes += int64_t(fb);
        }
    }
    if ((st = enqueue_halo_refresh(c))) return st;
    for (int f = 0; f < nframes; f++) {
        if ((st = enqueue_steps(c, k, chunk))) return st;
        const int b = f & 1;
        // snapshot b is free once the download of frame f-2 has finished
        if (f >= 2) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));
        double2 *snap = (double2 *)c->snap[b];
        if (c->prec == NLSE_FP64) {
            CUDA_TRY(c, cudaMemcpyAsync(snap, c->buf[BUF_PSI], fb, cudaMemcpyDeviceToDevice, c->stream));
        } else {
            widen_psi<float><<<blocks_for(int64_t(n), 256), 256, 0, c->stream>>>((const float2 *)c->buf[BUF_PSI],
                                                                                snap, int64_t(n));
            CUDA_TRY(c, cudaGetLastError());
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_snap[b], c->stream));
        // the download overlaps the next chunk's compute
        CUDA_TRY(c, cudaStreamWaitEvent(c->io_stream, c->ev_snap[b], 0));
        CUDA_TRY(c, cudaMemcpyAsync(frames + 2 * n * size_t(f), snap, fb, cudaMemcpyDeviceToHost, c->io_stream));
        CUDA_TRY(c, cudaEventRecord(c->ev_copied[b], c->io_stream));
    }
    st = finish_steps(c, chunk * nframes);
    CUDA_TRY(c, cudaStreamSynchronize(c->io_stream));
    return st;
}

nlse_status nlse_step_group(nlse_ctx *const *ctxs, int n, double k, int64_t nsteps) {
    if (!ctxs || n < 1) return fail(nullptr, NLSE_ERR_ARG, "ctxs is NULL or n < 1");
    for (int j = 0; j < n; j++) {
        nlse_status st = check_ctx(ctxs[j]);
        if (st) return st;
        if ((st = check_step_args(ctxs[j], k, nsteps))) return st;
    }
    if (nsteps == 0) return NLSE_OK;
    for (int j = 0; j < n; j++) {
        nlse_status st = enqueue_halo_refresh(ctxs[j], 1);
        if (st) return st;
    }
    for (int j = 0; j < n; j++) enqueue_barrier(ctxs[j], false, 2);
    // per stage: every rank's stage kernels and barrier signal, then every rank's wait
    for (int64_t t = 0; t < nsteps; t++)
        for (int s = 1; s <= 4; s++) {
            for (int j = 0; j < n; j++) enqueue_step_stage(ctxs[j], s, k, t, 1);
            for (int j = 0; j < n; j++) enqueue_barrier(ctxs[j], false, 2);
        }
    for (int j = 0; j < n; j++) enqueue_add_steps(ctxs[j], nsteps);
    nlse_status first = NLSE_OK;
    for (int j = 0; j < n; j++) {
        nlse_status st = finish_steps(ctxs[j], nsteps);
        if (st && !first) first = st;
    }
    return first;
}

nlse_status nlse_diagnostics(nlse_ctx *c, double *mass, double *ham) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!mass || !ham) return fail(c, NLSE_ERR_ARG, "mass / hamiltonian pointer is NULL");
    if (c->virtual_group) return fail(c, NLSE_ERR_ARG, "virtual ranks: use nlse_diagnostics_group");
    if ((st = enqueue_halo_refresh(c))) return st;
    enqueue_diag_local(c, hd_of(c));
    if (c->dist) {
        enqueue_diag_push(c);
        enqueue_barrier(c, true);
        diag_sum<<<1, 32, 0, c->stream>>>(c->comm, c->nranks, hd_of(c), c->d_result);
    }
    return finish_diag(c, mass, ham);
}

nlse_status nlse_diagnostics_group(nlse_ctx *const *ctxs, int n, double *mass, double *ham) {
    if (!ctxs || n < 1 || !mass || !ham) return fail(nullptr, NLSE_ERR_ARG, "bad arguments");
    for (int j = 0; j < n; j++) {
        nlse_status st = check_ctx(ctxs[j]);
        if (st) return st;
    }
    for (int j = 0; j < n; j++) {
        nlse_status st = enqueue_halo_refresh(ctxs[j], 1);
        if (st) return st;
    }
    for (int j = 0; j < n; j++) enqueue_barrier(ctxs[j], false, 2);
    for (int j = 0; j < n; j++) enqueue_diag_local(ctxs[j], hd_of(ctxs[j]));
    for (int j = 0; j < n; j++) {
        nlse_ctx *c = ctxs[j];
        if (!c->dist) continue;
        enqueue_diag_push(c);
    }
    for (int j = 0; j < n; j++) enqueue_barrier(ctxs[j], true, 1);
    for (int j = 0; j < n; j++) enqueue_barrier(ctxs[j], true, 2);
    for (int j = 0; j < n; j++) {
        nlse_ctx *c = ctxs[j];
        if (c->dist) diag_sum<<<1, 32, 0, c->stream>>>(c->comm, c->nranks, hd_of(c), c->d_result);
    }
    for (int j = 0; j < n; j++) {
        nlse_status st = finish_diag(ctxs[j], &mass[j], &ham[j]);
        if (st) return st;
    }
    return NLSE_OK;
}

nlse_status nlse_get_stream(nlse_ctx *c, void **stream) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (!stream) return fail(c, NLSE_ERR_ARG, "stream is NULL");
    *stream = (void *)c->stream;
    return NLSE_OK;
}

nlse_status nlse_set_timing(nlse_ctx *c, int enable) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    c->timing = enable != 0;
    return NLSE_OK;
}

nlse_status nlse_reset_timing(nlse_ctx *c) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    for (int i = 0; i < KK_COUNT; i++) { c->kind_ms[i] = 0; c->kind_launches[i] = 0; c->kind_points[i] = 0; }
    return NLSE_OK;
}

nlse_status nlse_get_timing(nlse_ctx *c, nlse_timing *out) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (!out) return fail(c, NLSE_ERR_ARG, "out is NULL");
    memset(out, 0, sizeof *out);
    out->n_kinds = KK_COUNT;
    for (int i = 0; i < KK_COUNT; i++) {
        snprintf(out->name[i], sizeof out->name[i], "%s", kKindName[i]);
        out->ms[i] = c->kind_ms[i];
        out->launches[i] = c->kind_launches[i];
        out->points[i] = c->kind_points[i];
    }
    return NLSE_OK;
}

nlse_status nlse_get_info(nlse_ctx *c, nlse_info *out) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (!out) return fail(c, NLSE_ERR_ARG, "out is NULL");
    memset(out, 0, sizeof *out);
    out->points = c->g.n;
    int per_stage = c->interior_kind == KK_GENERIC ? 1 : 2;
    if (c->dist && c->nranks > 1) per_stage += 1;
    out->launches_per_step = c->persist1d ? 0 : 4 * per_stage;   // 0: one launch per nlse_step call
    const int64_t cbytes = 2 * c->eb, rv = c->hasV ? c->eb : 0;
    out->min_bytes_per_step = (16 * cbytes + 4 * rv) * c->g.n;
    out->device_bytes = c->device_bytes;
    out->elem_bytes = c->eb;
    snprintf(out->variant, sizeof out->variant, "%s", c->persist1d ? "rk4_1d_persistent" : kKindName[c->interior_kind]);
    out->rank = c->rank;
    out->nranks = c->nranks;
    out->z0 = c->z0;
    out->nz_local = c->g.nz;
    return NLSE_OK;
}

}  // extern "C"
