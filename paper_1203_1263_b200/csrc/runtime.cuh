// runtime.cuh -- the context (struct nlse_ctx) and the host-side helpers shared by the
// translation units of libnlse_b200.so: nlse_api.cu (the C ABI, include/nlse.h) and the
// stage-instantiation units inst_<precision>_<dim>d_<order>.cu (one per kernel family, so
// that nvcc compiles them in parallel; see stages.cuh).
#pragma once
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/nlse.h"
#include "comm.cuh"
#include "common.cuh"

enum KernelKind { KK_GENERIC = 0, KK_STREAM3D, KK_TMA3D, KK_TILE2D, KK_TILE1D, KK_BOUNDARY, KK_DIAG, KK_COMM,
                  KK_FUSED3D, KK_STRIP2D, KK_COUNT };
static_assert(KK_COUNT <= NLSE_MAX_KINDS, "too many kernel kinds");

struct TimedLaunch { int kind; cudaEvent_t a, b; int64_t points; };

// The TMA descriptors of one context: Y maps of the three halo'd buffers (Psi, Psi_tmp,
// Psi_out; halo box), and Psi, K_tot, V over the owned box.  z coordinate of local
// plane p is p + zghost for the halo'd buffers, p for K_tot and V.
struct Tma3Maps {
    CUtensorMap y[3];
    CUtensorMap psi, k, v;
};

// TMA descriptors of the fused two-stage kernel (fused3d.cuh): the Y_A box over every halo'd
// buffer (index = buffer, 3 = the second Psi buffer), the ring-R base box over the two Psi
// buffers, K over the owned box, V over the ring-R box.
struct FusedMaps {
    CUtensorMap y[4];
    CUtensorMap base[4];
    CUtensorMap k, v;
};

struct StreamHolder {
    cudaStream_t s = nullptr;
    ~StreamHolder() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } }
};

enum { BUF_PSI = 0, BUF_TMP = 1, BUF_OUT = 2, BUF_PSI2 = 3 };   // BUF_PSI2: fused mode's Psi ping-pong

struct nlse_ctx {
    int ndim = 0;
    int64_t dims[3] = {1, 1, 1};    // global grid
    double h = 0, a = 0, s = 0;
    nlse_bc bc = NLSE_BC_DIRICHLET;
    nlse_order order = NLSE_CD2;
    nlse_precision prec = NLSE_FP64;
    uint32_t flags = 0;
    nlse::Grid g{};                  // owned grid (the slab in slab mode)
    int eb = 8;                      // sizeof(real)
    bool hasV = false;
    bool pitched = false;            // rows padded to g.sy > nx points (16-byte TMA strides)
    size_t ghost_off = 0;            // bytes from a halo'd allocation to its plane / row 0 (>= the
                                     // lower ghosts, rounded up to 256 B so that buf is aligned)
    // halo'd buffers: allocation base (plane -zghost) and plane-0 pointer
    void *alloc[4] = {nullptr, nullptr, nullptr, nullptr};
    void *buf[4] = {nullptr, nullptr, nullptr, nullptr};
    void *K = nullptr, *V = nullptr;
    void *fz = nullptr, *fp = nullptr;   // MSD 3D TMA path: stored F(b') (see StageArgs)
    int per2 = 0;
    int *d_div = nullptr;
    int *h_div = nullptr;            // pinned
    int *d_steps = nullptr;          // device counter of completed steps (divergence report)
    // CUDA graph of GRAPH_STEPS steps for the current k (nlse_step with many steps)
    cudaGraphExec_t graph_exec = nullptr;
    double graph_k = 0;
    bool graphs = true;              // NLSE_GRAPHS=0 at creation: direct launches only
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
    int nsm = 148;
    int64_t steps_done = 0;
    int64_t device_bytes = 0;
    std::string err;
    bool sticky = false;
    bool sticky_comm = false;        // slab mode: a barrier timed out / was aborted (NLSE_ERR_COMM)
    unsigned long long barrier_timeout_ns = 60000000000ull;
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
    // temporal blocking (§8(f) rank 2, fused3d.cuh): two RK4 stages per HBM pass, 3D CD, one GPU
    bool fused = false;
    int fused_ty = 16;
    FusedMaps fmaps{};
    int swap_parity = 0;             // Psi buffers swapped an odd number of times (fused mode)
    int graph_parity = 0;            // swap_parity when the CUDA graph was captured
    // slab mode
    bool dist = false;
    int rank = 0, nranks = 1;
    int64_t z0 = 0;
    nlse::CommBlock *comm = nullptr;
    bool connected = false;
    void *peer_alloc[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};  // [buf][lo, hi]
    int64_t peer_nloc[2] = {0, 0};
    nlse::CommBlock *peer_comm[nlse::MAX_RANKS] = {nullptr};
    std::vector<void *> ipc_opened;
    bool ghost_stale = false;
    bool virtual_group = false;      // connected by nlse_dist_connect_local: _group calls only
    bool persist1d = false;          // 1D: one persistent CTA per nlse_step call
    int cluster1d = 0;               // ... or a cluster of this many CTAs (> 1; rk4_1d_cluster)
    bool persist2d = false;          // 2D L2-scale grids: one cooperative launch per nlse_step call
    unsigned *d_bar = nullptr;       // its grid barrier (count, generation)
};

namespace nlse_rt {

using namespace nlse;

extern thread_local std::string g_create_error;   // defined in nlse_api.cu

inline nlse_status fail(nlse_ctx *c, nlse_status st, const std::string &msg) {
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
            return nlse_rt::fail(ctx, e_ == cudaErrorMemoryAllocation ? NLSE_ERR_OOM : NLSE_ERR_CUDA, \
                                 std::string(#expr) + ": " + cudaGetErrorString(e_));            \
    } while (0)

inline cudaEvent_t take_event(nlse_ctx *c) {
    if (!c->event_pool.empty()) { cudaEvent_t e = c->event_pool.back(); c->event_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Per-launch CUDA events on the context stream (timing mode only).
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

#ifndef NLSE_TMA_P
#define NLSE_TMA_P 3
#endif
#ifndef NLSE_TMA_P1
#define NLSE_TMA_P1 3
#endif
constexpr int TMA_P = NLSE_TMA_P;    // TMA ring prefetch depth of the Y planes (planes ahead; 2 and 4 measured slower, r01 ab1)
constexpr int TMA_P1 = NLSE_TMA_P1;  // ... for stage 1 (Y and V only: a deeper Y ring fits)
constexpr int GRAPH_STEPS = 8;       // RK4 steps per captured CUDA graph

inline unsigned blocks_for(int64_t n, int threads) { return unsigned((n + threads - 1) / threads); }
inline int halo_w(const nlse_ctx *c) { return c->order == NLSE_2SHOC4 ? 2 : 1; }
inline int ybuf_of_stage(int stage) { return stage == 1 ? BUF_PSI : (stage == 3 ? BUF_OUT : BUF_TMP); }
inline int obuf_of_stage(int stage) { return stage == 1 ? BUF_TMP : (stage == 2 ? BUF_OUT : (stage == 3 ? BUF_TMP : BUF_PSI)); }

// Per-device cache of a launch property (an occupancy figure, a shared-memory opt-in done):
// kernel attributes are per device, so one process driving contexts on several GPUs needs one
// entry per device (0 = not yet set).  Races are benign: every writer stores the same value.
constexpr int MAX_DEVICES = 64;
struct PerDevice {
    std::atomic<int> v[MAX_DEVICES];
    int get(int dev) const { return (dev >= 0 && dev < MAX_DEVICES) ? v[dev].load(std::memory_order_relaxed) : 0; }
    void set(int dev, int x) { if (dev >= 0 && dev < MAX_DEVICES) v[dev].store(x, std::memory_order_relaxed); }
};

// The stage enqueue entry point of one (precision, dimension, order) family, defined in its
// instantiation unit (stages.cuh, NLSE_DEFINE_STAGES): enqueue stage `stage` (1-4) of step
// `step` of the current launch sequence for the context's BC.
using EnqueueStageFn = void (*)(nlse_ctx *, int stage, double k, int step);
// 1D: all nsteps in one persistent CTA (persist1d.cuh)
using Persist1DFn = void (*)(nlse_ctx *, double k, int64_t nsteps);
using Persist1DSmemFn = size_t (*)(const nlse_ctx *);
// fused mode: one RK4 step (two fused passes + their boundary passes), then the Psi swap
using FusedStepFn = void (*)(nlse_ctx *, double k, int step);
void fused_step_f64_dirichlet(nlse_ctx *, double, int);
void fused_step_f64_msd(nlse_ctx *, double, int);
void fused_step_f64_l0(nlse_ctx *, double, int);
void fused_step_f32_dirichlet(nlse_ctx *, double, int);
void fused_step_f32_msd(nlse_ctx *, double, int);
void fused_step_f32_l0(nlse_ctx *, double, int);
// Swap the two Psi buffers (fused mode, after each step's second pass).
inline void swap_psi(nlse_ctx *c) {
    std::swap(c->alloc[BUF_PSI], c->alloc[BUF_PSI2]);
    std::swap(c->buf[BUF_PSI], c->buf[BUF_PSI2]);
    std::swap(c->fmaps.y[BUF_PSI], c->fmaps.y[BUF_PSI2]);
    std::swap(c->fmaps.base[BUF_PSI], c->fmaps.base[BUF_PSI2]);
    c->swap_parity ^= 1;
}

#define NLSE_FAMILIES(X)                                                                        \
    X(f64, 1, cd) X(f64, 1, shoc) X(f64, 2, cd) X(f64, 2, shoc) X(f64, 3, cd) X(f64, 3, shoc)  \
    X(f32, 1, cd) X(f32, 1, shoc) X(f32, 2, cd) X(f32, 2, shoc) X(f32, 3, cd) X(f32, 3, shoc)
// one entry point per family and BC (dirichlet, msd, l0)
#define NLSE_DECLARE_FAMILY(P, D, O)                                                            \
    void enqueue_stage_##P##_##D##d_##O##_dirichlet(nlse_ctx *, int, double, int);              \
    void enqueue_stage_##P##_##D##d_##O##_msd(nlse_ctx *, int, double, int);                    \
    void enqueue_stage_##P##_##D##d_##O##_l0(nlse_ctx *, int, double, int);
NLSE_FAMILIES(NLSE_DECLARE_FAMILY)
#undef NLSE_DECLARE_FAMILY
void persist2d_f64_cd(nlse_ctx *, double, int64_t);
void persist2d_f64_shoc(nlse_ctx *, double, int64_t);
void persist2d_f32_cd(nlse_ctx *, double, int64_t);
void persist2d_f32_shoc(nlse_ctx *, double, int64_t);
void persist1d_f64_cd(nlse_ctx *, double, int64_t);
void persist1d_f64_shoc(nlse_ctx *, double, int64_t);
void persist1d_f32_cd(nlse_ctx *, double, int64_t);
void persist1d_f32_shoc(nlse_ctx *, double, int64_t);

}  // namespace nlse_rt
