// nlse_api.cu -- the C ABI (include/nlse.h) and the runtime behind it: context,
// device buffers, TMA descriptors, constants, validation, stage sequencing (a8),
// slab mode (a9: ghost planes, peer mapping, per-stage neighbour barriers),
// divergence flag, diagnostics (a10) and per-kernel timing.
#include <unistd.h>

#include <cudaTypedefs.h>

#include "runtime.cuh"
#include "diag.cuh"
#include "generic.cuh"
#include "persist1d.cuh"
#include "stage3d_tma.cuh"
#include "fused3d.cuh"

using namespace nlse;
using namespace nlse_rt;

static_assert(NLSE_MAX_RANKS == MAX_RANKS, "rank limits of nlse.h and comm.cuh differ");

thread_local std::string nlse_rt::g_create_error;

namespace {

const char *kKindName[KK_COUNT] = {"stage_generic", "stage3d_stream", "stage3d_tma", "stage2d_tile",
                                   "stage1d_tile", "stage_boundary", "diag", "peer_barrier", "fused3d_cd",
                                   "stage2d_strip"};

struct DistBlob {               // what nlse_dist_export writes (NLSE_DIST_HANDLE_BYTES)
    uint32_t magic, version;
    int32_t rank, nranks;
    int64_t nloc;
    int32_t pid, device;
    cudaIpcMemHandle_t h[4];    // Psi, Psi_tmp, Psi_out allocations, comm block
};
static_assert(sizeof(DistBlob) <= NLSE_DIST_HANDLE_BYTES, "blob too large");
constexpr uint32_t kBlobMagic = 0x4e4c5345u;  // "NLSE"

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

// 3D map over [d2][d1][d0] elements of T (d0 fastest; rows of p0 >= d0 elements in memory),
// box {b0, b1, 1}.  TMA needs 16-byte multiples for the row and plane strides (pitched rows,
// nlse_ctx::pitched, make every grid qualify).
bool make_map(CUtensorMap *m, void *base, int eb, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t p0, uint32_t b0,
              uint32_t b1) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {p0 * uint64_t(eb), p0 * d1 * uint64_t(eb)};
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

// Fused mode (fused3d.cuh): Y_A box maps over all four halo'd buffers, the ring-R base box over
// the Psi buffers, K over the owned box, V over the ring-R box (16-byte-aligned x origin).
template <typename T, int TYV>
bool build_fused_maps(nlse_ctx *c) {
    using Cfg = F3Cfg<T, TYV>;
    const uint64_t nx = c->g.nx, ny = c->g.ny, nz = c->g.nz, sy = c->g.sy;
    const int eb = int(sizeof(T));
    bool ok = true;
    for (int b = 0; b < 4; b++) {
        ok = ok && make_map(&c->fmaps.y[b], c->buf[b], eb, 2 * nx, ny, nz, 2 * sy, Cfg::BOX_Y_X, Cfg::BOX_Y_Y);
        ok = ok && make_map(&c->fmaps.base[b], c->buf[b], eb, 2 * nx, ny, nz, 2 * sy, Cfg::BOX_B_X, Cfg::BOX_B_Y);
    }
    ok = ok && make_map(&c->fmaps.k, c->K, eb, 2 * nx, ny, nz, 2 * sy, Cfg::BOX_K_X, Cfg::BOX_K_Y);
    if (c->V) ok = ok && make_map(&c->fmaps.v, c->V, eb, nx, ny, nz, sy, Cfg::BOX_V_X, Cfg::BOX_V_Y);
    else c->fmaps.v = c->fmaps.k;   // never dereferenced without a V array
    return ok;
}

// First lower ghost plane of halo'd buffer b (the TMA maps address planes from there)
void *ghost_base(const nlse_ctx *c, int b) {
    return (char *)c->buf[b] - size_t(c->g.zghost) * size_t(c->g.su) * size_t(2 * c->eb);
}

template <typename T, int ORDER, int TYV>
bool build_maps(nlse_ctx *c) {
    using Cfg = T3Cfg<T, ORDER, TMA_P, TYV>;
    const uint64_t nx = c->g.nx, ny = c->g.ny, nz = c->g.nz, nza = nz + 2 * c->g.zghost, sy = c->g.sy;
    const int eb = int(sizeof(T));
    bool ok = true;
    for (int b = 0; b < 3; b++)
        ok = ok && make_map(&c->maps.y[b], ghost_base(c, b), eb, 2 * nx, ny, nza, 2 * sy, Cfg::BOX_Y_X, Cfg::BOX_Y_Y);
    ok = ok && make_map(&c->maps.psi, ghost_base(c, BUF_PSI), eb, 2 * nx, ny, nza, 2 * sy, Cfg::BOX_C_X, Cfg::BOX_O_Y);
    ok = ok && make_map(&c->maps.k, c->K, eb, 2 * nx, ny, nz, 2 * sy, Cfg::BOX_C_X, Cfg::BOX_O_Y);
    if (c->V) ok = ok && make_map(&c->maps.v, c->V, eb, nx, ny, nz, sy, Cfg::BOX_R_X, Cfg::BOX_O_Y);
    else c->maps.v = c->maps.k;   // never dereferenced without a V array
    return ok;
}


// The stage entry point of the context's (precision, dimension, order, BC) family (inst_*.cu).
EnqueueStageFn stage_fn(const nlse_ctx *c) {
    const bool f64 = c->prec == NLSE_FP64, shoc = c->order == NLSE_2SHOC4;
    const int bc = c->bc == NLSE_BC_MSD ? 1 : (c->bc == NLSE_BC_L0 ? 2 : 0);
#define NLSE_PICK(P, D, O)                                                                        \
    if (f64 == (std::string(#P) == "f64") && c->ndim == D && shoc == (std::string(#O) == "shoc")) { \
        const EnqueueStageFn fns[3] = {&enqueue_stage_##P##_##D##d_##O##_dirichlet,                   \
                                       &enqueue_stage_##P##_##D##d_##O##_msd,                         \
                                       &enqueue_stage_##P##_##D##d_##O##_l0};                         \
        return fns[bc];                                                                           \
    }
    NLSE_FAMILIES(NLSE_PICK)
#undef NLSE_PICK
    return nullptr;
}

void enqueue_stage(nlse_ctx *c, int stage, double k, int step) { stage_fn(c)(c, stage, k, step); }

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
    b.timeout_ns = c->barrier_timeout_ns;
    LaunchTimer lt(c, KK_COMM, 0);
    peer_barrier<<<1, 32, 0, c->stream>>>(b, mode);
}

// Copy the first / last w owned planes of Psi into the neighbours' ghost planes (after
// nlse_set_psi*), then barrier (mode as enqueue_barrier).
nlse_status enqueue_halo_refresh(nlse_ctx *c, int mode = 3) {
    if (!c->dist || !c->ghost_stale) return NLSE_OK;
    const int w = halo_w(c);
    const size_t cb = size_t(2 * c->eb), plane = size_t(c->g.su) * cb;
    if (c->peer_alloc[BUF_PSI][0]) {
        char *dst = (char *)c->peer_alloc[BUF_PSI][0] + c->ghost_off + c->peer_nloc[0] * plane;
        CUDA_TRY(c, cudaMemcpyAsync(dst, c->buf[BUF_PSI], w * plane, cudaMemcpyDefault, c->stream));
    }
    if (c->peer_alloc[BUF_PSI][1]) {
        char *dst = (char *)c->peer_alloc[BUF_PSI][1] + c->ghost_off - w * plane;
        const char *src = (const char *)c->buf[BUF_PSI] + (c->g.ns - w) * plane;
        CUDA_TRY(c, cudaMemcpyAsync(dst, src, w * plane, cudaMemcpyDefault, c->stream));
    }
    enqueue_barrier(c, false, mode);
    c->ghost_stale = false;
    return NLSE_OK;
}

// The divergence flag (first step index with a non-finite Psi, INT32_MAX = none) stays set
// until Psi is replaced by nlse_set_psi / nlse_set_psi_device.
nlse_status reset_divergence(nlse_ctx *c) {
    static const int big = INT32_MAX;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_div, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    return NLSE_OK;
}

nlse_status check_ctx(nlse_ctx *c) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (c->sticky) return NLSE_ERR_CUDA;
    if (c->sticky_comm) return NLSE_ERR_COMM;
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

FusedStepFn fused_fn(const nlse_ctx *c) {
    const bool f64 = c->prec == NLSE_FP64;
    if (c->bc == NLSE_BC_MSD) return f64 ? &fused_step_f64_msd : &fused_step_f32_msd;
    if (c->bc == NLSE_BC_L0) return f64 ? &fused_step_f64_l0 : &fused_step_f32_l0;
    return f64 ? &fused_step_f64_dirichlet : &fused_step_f32_dirichlet;
}

// Enqueue one RK4 stage of step n of the current launch sequence, followed (slab mode)
// by the neighbour barrier (mode as enqueue_barrier).
void enqueue_step_stage(nlse_ctx *c, int stage, double k, int64_t n, int mode = 3) {
    enqueue_stage(c, stage, k, int(std::min<int64_t>(n, INT32_MAX / 2)));
    enqueue_barrier(c, false, mode);
}

// One RK4 step: four stage launches, or (fused mode) two fused two-stage passes.
void enqueue_one_step(nlse_ctx *c, double k, int64_t n) {
    if (c->fused) {
        fused_fn(c)(c, k, int(std::min<int64_t>(n, INT32_MAX / 2)));
        return;
    }
    for (int s = 1; s <= 4; s++) enqueue_step_stage(c, s, k, n);
}

void enqueue_add_steps(nlse_ctx *c, int64_t n) {
    add_steps<<<1, 1, 0, c->stream>>>(c->d_steps, int(n));
}

bool use_persist1d(const nlse_ctx *c) {
    if (c->ndim != 1 || c->interior_kind == KK_GENERIC || c->dist) return false;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const size_t need = c->prec == NLSE_FP64 ? persist1d_smem<double>(int(c->g.nx), c->hasV, c->order == NLSE_2SHOC4)
                                             : persist1d_smem<float>(int(c->g.nx), c->hasV, c->order == NLSE_2SHOC4);
    return c->g.nx <= (int64_t(1) << 30) && need <= size_t(optin);
}

// 1D persistent kernel on a thread-block cluster: NLSE_1D_CLUSTER=N forces N CTAs (0 / 1: the
// single-CTA kernel); default 8 CTAs (a portable cluster) for fp64 and 512 <= n <= 3200 (configs[0] 1025
// points: 3.8 vs 4.1 us/step, 1001-point MSD 5.4 vs 5.7; at 10^4 points the tiled kernels are
// faster, 9.2 vs 10.4 us/step, r02 c1d2), when every segment holds >= 4 points and fits the CTA.
int choose_cluster1d(const nlse_ctx *c) {
    if (c->ndim != 1 || c->interior_kind == KK_GENERIC || c->dist) return 0;
    const int64_t n = c->g.nx;
    const char *e = getenv("NLSE_1D_CLUSTER");
    // (fp32: the single CTA is faster -- configs[1] fp32 3.87 vs 4.83 us/step, r02fin2 / r02fin3)
    int64_t nc = e ? std::atoll(e) : ((c->prec == NLSE_FP64 && n >= 512 && n <= 3200) ? 8 : 0);
    if (nc > 8) nc = 8;
    if (nc < 2 || n < 4 * nc) return 0;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const size_t need = c->prec == NLSE_FP64 ? cluster1d_smem<double>(int(n), int(nc), c->hasV)
                                             : cluster1d_smem<float>(int(n), int(nc), c->hasV);
    return need <= size_t(optin) ? int(nc) : 0;
}

void drop_graph(nlse_ctx *c) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
}

// Capture GRAPH_STEPS steps (all launches, barriers and the step-counter update) once
// per k; false if capture is unavailable (then the caller launches directly).
bool ensure_graph(nlse_ctx *c, double k) {
    if (c->graph_exec && c->graph_k == k && c->graph_parity == c->swap_parity) return true;
    drop_graph(c);
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int parity0 = c->swap_parity;
    for (int n = 0; n < GRAPH_STEPS; n++) enqueue_one_step(c, k, n);
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
    c->graph_parity = parity0;     // GRAPH_STEPS is even: replaying it leaves the Psi buffers in place
    return true;
}

bool graphs_enabled(const nlse_ctx *c, int64_t nsteps) {
    return c->graphs && !c->timing && !c->virtual_group && nsteps >= 2 * GRAPH_STEPS;
}

// Slab mode: a neighbour barrier that timed out or saw an abort (comm.cuh peer_barrier) makes
// the context unusable (sticky NLSE_ERR_COMM): the halo data of that stage may be incomplete.
nlse_status check_comm(nlse_ctx *c) {
    if (!c->dist || !c->comm) return NLSE_OK;
    unsigned st = 0;
    CUDA_TRY(c, cudaMemcpy(&st, &c->comm->status, sizeof st, cudaMemcpyDeviceToHost));
    if (st) {
        c->sticky_comm = true;
        return fail(c, NLSE_ERR_COMM, st == 2 ? "a rank aborted (nlse_dist_abort) while this rank waited at a "
                                                 "neighbour barrier"
                                              : "a neighbour barrier timed out (NLSE_BARRIER_TIMEOUT_S): a peer "
                                                "rank is late, stopped or failed");
    }
    return NLSE_OK;
}

nlse_status finish_steps(nlse_ctx *c, int64_t nsteps) {
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->h_div, c->d_div, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->timing) collect_timing(c);
    c->steps_done += nsteps;
    if (nlse_status st = check_comm(c)) return st;
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
    if (nlse_status st = check_comm(c)) return st;
    *mass = c->h_result[0];
    *ham = c->h_result[1];
    return NLSE_OK;
}

// Element offset of logical point q (x fastest, rows of nx points) in a buffer with rows of
// sy >= nx elements (pitched rows, nlse_ctx::pitched).
__device__ __forceinline__ int64_t pitched_at(int64_t q, int64_t nx, int64_t sy) {
    if (nx == sy) return q;
    const int64_t r = q / nx;
    return r * sy + (q - r * nx);
}
// Conversions between the host layout (double, logical) and the device buffers (working
// precision, pitched): logical points q0 .. q0 + m - 1; the logical side is indexed from q0.
template <typename T>
__global__ void widen_psi(const cplx<T> *src, double2 *dst, int64_t q0, int64_t m, int64_t nx, int64_t sy) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) { cplx<T> v = src[pitched_at(q0 + t, nx, sy)]; dst[t] = make_double2(double(v.x), double(v.y)); }
}
template <typename T>
__global__ void narrow_psi(const double2 *src, cplx<T> *dst, int64_t q0, int64_t m, int64_t nx, int64_t sy) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) { double2 v = src[t]; cplx<T> r; r.x = T(v.x); r.y = T(v.y); dst[pitched_at(q0 + t, nx, sy)] = r; }
}
template <typename T>
__global__ void narrow_real(const double *src, T *dst, int64_t m, int64_t nx, int64_t sy) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < m) dst[pitched_at(t, nx, sy)] = T(src[t]);
}

double linear_bound(int ndim, double a, double h, nlse_order order) {
    double k = h * h / (double(ndim) * std::sqrt(2.0) * a);
    return order == NLSE_2SHOC4 ? 0.75 * k : k;
}

// Host double (re, im) -> device working precision, staged through Psi_out (scratch
// between calls) for fp32.
nlse_status upload_complex(nlse_ctx *c, const double *host, void *dev) {
    const size_t n = size_t(c->g.n), nx = size_t(c->g.nx), sy = size_t(c->g.sy);
    if (c->prec == NLSE_FP64) {
        CUDA_TRY(c, cudaMemcpy2DAsync(dev, sy * 16, host, nx * 16, nx * 16, n / nx, cudaMemcpyHostToDevice, c->stream));
    } else {
        const size_t chunk = n / 2 > 0 ? n / 2 : 1;  // outb holds >= n float2 = n/2 double2
        double2 *scratch = (double2 *)c->buf[BUF_OUT];
        for (size_t off = 0; off < n; off += chunk) {
            size_t m = std::min(chunk, n - off);
            CUDA_TRY(c, cudaMemcpyAsync(scratch, host + 2 * off, m * 16, cudaMemcpyHostToDevice, c->stream));
            narrow_psi<float><<<blocks_for(m, 256), 256, 0, c->stream>>>(scratch, (float2 *)dev, int64_t(off),
                                                                          int64_t(m), int64_t(nx), int64_t(sy));
            CUDA_TRY(c, cudaGetLastError());
        }
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

nlse_status download_complex(nlse_ctx *c, const void *dev, double *host) {
    const size_t n = size_t(c->g.n), nx = size_t(c->g.nx), sy = size_t(c->g.sy);
    if (c->prec == NLSE_FP64) {
        CUDA_TRY(c, cudaMemcpy2DAsync(host, nx * 16, dev, sy * 16, nx * 16, n / nx, cudaMemcpyDeviceToHost, c->stream));
    } else {
        const size_t chunk = n / 2 > 0 ? n / 2 : 1;
        double2 *scratch = (double2 *)c->buf[BUF_OUT];
        for (size_t off = 0; off < n; off += chunk) {
            size_t m = std::min(chunk, n - off);
            widen_psi<float><<<blocks_for(m, 256), 256, 0, c->stream>>>((const float2 *)dev, scratch, int64_t(off),
                                                                         int64_t(m), int64_t(nx), int64_t(sy));
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
    // slab axis (§8(e)): z in 3D, y in 2D, x in 1D; nloc = its owned length
    const int sax = ndim - 1;
    int64_t z0 = 0, nloc = dims[sax];
    if (dist) {
        if (nranks < 1 || nranks > NLSE_MAX_RANKS || rank < 0 || rank >= nranks)
            return fail(nullptr, NLSE_ERR_ARG, "rank / nranks out of range");
        nlse_slab_range(dims[sax], nranks, rank, &z0, &nloc);
        if (nloc < 2 * w) return fail(nullptr, NLSE_ERR_ARG, "every slab needs at least 2w planes / rows / points (w = 1 CD, 2 2SHOC)");
    }
    const int64_t nx_own = ndim == 1 ? nloc : dims[0];
    const int64_t ny_own = ndim == 2 ? nloc : dims[1], nz_own = ndim == 3 ? nloc : 1;
    const int64_t n = nx_own * ny_own * nz_own;
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
    c->g.nx = nx_own; c->g.ny = ny_own; c->g.nz = nz_own;
    c->g.sy = nx_own; c->g.sz = nx_own * ny_own; c->g.n = n;
    c->eb = prec == NLSE_FP64 ? 8 : 4;
    // Pitched rows: the 3D TMA kernels need 16-byte row strides in every array (complex rows
    // 2*nx*eb, V rows nx*eb bytes); the paper pads rows the same way (cudaMallocPitch).
    // Rows are padded to sy points only where they would not qualify (e.g. fp32 with odd nx:
    // the paper's 87x87x203 ring); padding is zero, never read (TMA boxes stop at nx) or written.
    if (ndim == 3 && !(flags & NLSE_FLAG_GENERIC_KERNELS) && std::string(env_kernel()) != "v1") {
        const int64_t per16 = 16 / c->eb;                       // points per 16 bytes of a real row
        const bool bad = (2 * dims[0] * c->eb) % 16 != 0 || (V && (dims[0] * c->eb) % 16 != 0);
        if (bad) {
            c->g.sy = (dims[0] + per16 - 1) / per16 * per16;
            c->g.sz = c->g.sy * dims[1];
            c->pitched = true;
        }
    }
    c->g.zf_lo = (!dist || rank == 0) ? 1 : 0;
    c->g.zf_hi = (!dist || rank == nranks - 1) ? 1 : 0;
    c->g.zghost = dist ? w : 0;
    c->g.ns = ndim == 3 ? c->g.nz : (ndim == 2 ? c->g.ny : c->g.nx);
    c->g.su = ndim == 3 ? c->g.sz : (ndim == 2 ? c->g.sy : 1);
    c->hasV = V != nullptr;
    cudaGetDevice(&c->device);
    if (flags & NLSE_FLAG_GENERIC_KERNELS) c->interior_kind = KK_GENERIC;
    else c->interior_kind = ndim == 3 ? KK_TMA3D : (ndim == 2 ? KK_STRIP2D : KK_TILE1D);
    // 2D: the warp-strip kernel (strip2d.cuh, boundary included, one launch per stage) by default;
    // NLSE_2D_KERNEL=tile selects the round-1 shared-tile kernel + boundary kernel
    if (c->interior_kind == KK_STRIP2D) {
        const char *e2 = getenv("NLSE_2D_KERNEL");
        const char *ep2 = getenv("NLSE_PERSIST2D");    // (the persistent stepper runs the tile body)
        // (the strip kernel addresses rows by 32-bit element offsets)
        const bool fits = (c->g.ny + 2 * int64_t(c->g.zghost) + 1) * c->g.sy < (int64_t(1) << 31);
        if ((e2 && std::string(e2) == "tile") || (ep2 && ep2[0] == '1') || !fits) c->interior_kind = KK_TILE2D;
    }

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
    // one slab-axis unit (a plane in 3D, a row in 2D); the halo'd buffers carry zghost units of
    // ghosts below and above the owned ones
    const size_t cb = size_t(2 * c->eb), plane = size_t(c->g.su) * cb;
    // the owned planes start 256-byte aligned (a row-sized 2D ghost unit need not be a 16-byte
    // multiple); all ranks of a slab job use the same offset, so peers address each other's
    // planes from their allocation bases
    c->ghost_off = (size_t(c->g.zghost) * plane + 255) / 256 * 256;
    const size_t halo_bytes = c->ghost_off + (size_t(c->g.ns) + size_t(c->g.zghost)) * plane;
    const size_t cells = size_t(c->g.ns) * size_t(c->g.su);    // allocated points (>= n with pitched rows)
    for (int b = 0; b < 3; b++) {
        CREATE_TRY(cudaMalloc(&c->alloc[b], halo_bytes));
        CREATE_TRY(cudaMemsetAsync(c->alloc[b], 0, halo_bytes, c->stream));
        c->buf[b] = (char *)c->alloc[b] + c->ghost_off;
    }
    CREATE_TRY(cudaMalloc(&c->K, cells * cb));
    CREATE_TRY(cudaMemsetAsync(c->K, 0, cells * cb, c->stream));
    c->device_bytes = int64_t(3 * halo_bytes + cells * cb);
    if (V) {
        CREATE_TRY(cudaMalloc(&c->V, cells * c->eb));
        CREATE_TRY(cudaMemsetAsync(c->V, 0, cells * c->eb, c->stream));
        c->device_bytes += int64_t(cells * c->eb);
        const size_t nx = size_t(c->g.nx), sy = size_t(c->g.sy);
        if (prec == NLSE_FP64) {
            CREATE_TRY(cudaMemcpy2DAsync(c->V, sy * 8, V, nx * 8, nx * 8, size_t(n) / nx, cudaMemcpyHostToDevice,
                                         c->stream));
        } else {
            // stage the double V through K (>= n complex floats = n doubles) and round once on the device
            CREATE_TRY(cudaMemcpyAsync(c->K, V, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
            narrow_real<float><<<blocks_for(n, 256), 256, 0, c->stream>>>((const double *)c->K, (float *)c->V, n,
                                                                           int64_t(nx), int64_t(sy));
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
    cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, c->device);
    c->diag_blocks = c->nsm * 8;
    {
        const char *e = getenv("NLSE_GRAPHS");
        c->graphs = !(e && e[0] == '0');
        const char *t = getenv("NLSE_BARRIER_TIMEOUT_S");
        const double ts = t ? std::atof(t) : 60.0;
        c->barrier_timeout_ns = ts > 0 ? (unsigned long long)(ts * 1e9) : 60000000000ull;
    }
    CREATE_TRY(cudaMalloc(&c->d_partial, sizeof(double) * 2 * c->diag_blocks));
    CREATE_TRY(cudaMalloc(&c->d_result, sizeof(double) * 2));
    CREATE_TRY(cudaMallocHost(&c->h_result, sizeof(double) * 2));
    CREATE_TRY(cudaStreamSynchronize(c->stream));
    if (c->interior_kind == KK_TMA3D) {
        const std::string ek = env_kernel();
        bool ok = ek != "v1";
        const char *ety = getenv("NLSE_TMA_TY");
        // fp64: 16-row tiles (512 threads, 1 CTA/SM, <= 128 registers) measured faster (r01f, r01j);
        // fp32: 8-row tiles (256 threads, 3 CTAs/SM, 80 registers, spill-free) measured faster than
        // 16 rows at 1 CTA/SM (no spills) or 2 CTAs/SM (64 registers, spills): r02b
        const int ty_default = prec == NLSE_FP32 ? 8 : 16;
        c->tma_ty = ety ? (std::atoi(ety) == 8 ? 8 : 16) : ty_default;
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
        // temporal blocking (§8(f) rank 2, fused3d.cuh): S1+S2 and S3+S4 in one HBM pass each; 3D
        // CD on one GPU; MSD needs the stored-F(b') boundary pass.  Default: fp64 grids of >= 2^26
        // points, where it measured faster (r02f: 1024^3 46.3 vs 54.6 ms/step); the L2-scale and
        // fp32 grids stay on the single-stage kernel.  NLSE_FUSED=1 / 0 forces it on / off.
        const char *efu = getenv("NLSE_FUSED");
        const bool want_fused = efu ? efu[0] == '1' : (prec == NLSE_FP64 && n >= (int64_t(1) << 26));
        if (ok && want_fused && order == NLSE_CD2 && !dist && (bc != NLSE_BC_MSD || c->fp)) {
            CREATE_TRY(cudaMalloc(&c->alloc[BUF_PSI2], halo_bytes));
            CREATE_TRY(cudaMemsetAsync(c->alloc[BUF_PSI2], 0, halo_bytes, c->stream));
            c->buf[BUF_PSI2] = (char *)c->alloc[BUF_PSI2] + c->ghost_off;
            c->device_bytes += int64_t(halo_bytes);
            const char *fty = getenv("NLSE_FUSED_TY");
            c->fused_ty = (fty && std::atoi(fty) == 8) ? 8 : 16;
            bool fok;
            if (prec == NLSE_FP64)
                fok = c->fused_ty == 16 ? build_fused_maps<double, 16>(c) : build_fused_maps<double, 8>(c);
            else
                fok = c->fused_ty == 16 ? build_fused_maps<float, 16>(c) : build_fused_maps<float, 8>(c);
            c->fused = fok;
        }
    }
    // 2D: all stages of an nlse_step call in one cooperative launch (tile2d.cuh rk4_2d_persistent)
    if (ndim == 2 && !dist && c->interior_kind == KK_TILE2D) {
        const char *ep = getenv("NLSE_PERSIST2D");
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device);
        // measured slower than the per-stage kernels (1024^2: 115.7 vs 77.8 us/step, r02r: tiles run
        // one after another inside a CTA and 4 grid barriers per step serialise ~600 CTAs), so off
        // by default; NLSE_PERSIST2D=1 selects it
        const bool want = ep && ep[0] == '1';
        if (want && coop) {
            CREATE_TRY(cudaMalloc(&c->d_bar, 2 * sizeof(unsigned)));
            CREATE_TRY(cudaMemsetAsync(c->d_bar, 0, 2 * sizeof(unsigned), c->stream));
            CREATE_TRY(cudaStreamSynchronize(c->stream));
            c->persist2d = true;
        }
    }
#undef CREATE_TRY
    c->cluster1d = choose_cluster1d(c);
    c->persist1d = c->cluster1d > 1 || use_persist1d(c);
    c->connected = !dist;
    *out = c;
    return NLSE_OK;
}

// nsteps RK4 steps on the context stream: the persistent 1D kernel, or replays of the CUDA
// graph of GRAPH_STEPS steps plus direct launches for the remainder.
nlse_status enqueue_steps(nlse_ctx *c, double k, int64_t nsteps) {
    if (c->persist1d) {
        const bool f64 = c->prec == NLSE_FP64, shoc = c->order == NLSE_2SHOC4;
        (f64 ? (shoc ? persist1d_f64_shoc : persist1d_f64_cd) : (shoc ? persist1d_f32_shoc : persist1d_f32_cd))(
            c, k, nsteps);
        CUDA_TRY(c, cudaGetLastError());               // (e.g. a cluster launch the device refuses)
        enqueue_add_steps(c, nsteps);
        return NLSE_OK;
    }
    if (c->persist2d) {
        const bool f64 = c->prec == NLSE_FP64, shoc = c->order == NLSE_2SHOC4;
        (f64 ? (shoc ? persist2d_f64_shoc : persist2d_f64_cd) : (shoc ? persist2d_f32_shoc : persist2d_f32_cd))(
            c, k, nsteps);
        CUDA_TRY(c, cudaGetLastError());
        enqueue_add_steps(c, nsteps);
        return NLSE_OK;
    }
    int64_t done = 0;
    if (graphs_enabled(c, nsteps) && ensure_graph(c, k)) {
        for (; done + GRAPH_STEPS <= nsteps; done += GRAPH_STEPS)
            CUDA_TRY(c, cudaGraphLaunch(c->graph_exec, c->stream));
    }
    if (done < nsteps) {
        for (int64_t n = 0; n < nsteps - done; n++) enqueue_one_step(c, k, n);
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
    for (int b = 0; b < 4; b++) cudaFree(c->alloc[b]);
    cudaFree(c->K); cudaFree(c->V); cudaFree(c->comm); cudaFree(c->fz); cudaFree(c->fp);
    drop_graph(c);
    cudaFree(c->d_div); cudaFree(c->d_steps); cudaFree(c->d_partial); cudaFree(c->d_result); cudaFree(c->d_bar);
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
    b.rank = c->rank; b.nranks = c->nranks; b.nloc = c->g.ns;
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
            c->peer_nloc[side] = ctxs[nb]->g.ns;
            for (int i = 0; i < 3; i++) c->peer_alloc[i][side] = ctxs[nb]->alloc[i];
        }
        c->connected = true;
        c->ghost_stale = true;
        c->virtual_group = n > 1;
    }
    return NLSE_OK;
}

nlse_status nlse_dist_abort(nlse_ctx *c) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (!c->dist || !c->comm) return fail(c, NLSE_ERR_ARG, "not a slab-mode context");
    // on a separate stream: the context stream may be blocked behind a waiting barrier kernel
    cudaStream_t s = nullptr;
    CUDA_TRY(c, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    static const unsigned one = 1;
    cudaError_t e = cudaSuccess;
    for (int j = 0; j < c->nranks && e == cudaSuccess; j++) {
        CommBlock *cb = j == c->rank ? c->comm : c->peer_comm[j];
        if (cb) e = cudaMemcpyAsync(&cb->abort, &one, sizeof one, cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e != cudaSuccess) return fail(c, NLSE_ERR_CUDA, std::string("nlse_dist_abort: ") + cudaGetErrorString(e));
    c->sticky_comm = true;
    c->err = "aborted by nlse_dist_abort";
    return NLSE_OK;
}

nlse_status nlse_set_psi(nlse_ctx *c, const double *psi) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!psi) return fail(c, NLSE_ERR_ARG, "psi is NULL");
    if ((st = reset_divergence(c))) return st;
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
    if ((st = reset_divergence(c))) return st;
    const size_t row = size_t(c->g.nx) * 2 * c->eb;
    CUDA_TRY(c, cudaMemcpy2DAsync(c->buf[BUF_PSI], size_t(c->g.sy) * 2 * c->eb, d, row, row, size_t(c->g.n / c->g.nx),
                                  cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->ghost_stale = c->dist;
    return NLSE_OK;
}

nlse_status nlse_get_psi_device(nlse_ctx *c, void *d) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!d) return fail(c, NLSE_ERR_ARG, "d_psi is NULL");
    const size_t row = size_t(c->g.nx) * 2 * c->eb;
    CUDA_TRY(c, cudaMemcpy2DAsync(d, row, c->buf[BUF_PSI], size_t(c->g.sy) * 2 * c->eb, row, size_t(c->g.n / c->g.nx),
                                  cudaMemcpyDeviceToDevice, c->stream));
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
            CUDA_TRY(c, cudaMemcpy2DAsync(snap, size_t(c->g.nx) * 16, c->buf[BUF_PSI], size_t(c->g.sy) * 16,
                                          size_t(c->g.nx) * 16, n / size_t(c->g.nx), cudaMemcpyDeviceToDevice,
                                          c->stream));
        } else {
            widen_psi<float><<<blocks_for(int64_t(n), 256), 256, 0, c->stream>>>(
                (const float2 *)c->buf[BUF_PSI], snap, 0, int64_t(n), c->g.nx, c->g.sy);
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
    int per_stage = (c->interior_kind == KK_GENERIC || c->interior_kind == KK_TILE1D || c->interior_kind == KK_STRIP2D) ? 1 : 2;
    if (c->dist && c->nranks > 1) per_stage += 1;
    out->launches_per_step = (c->persist1d || c->persist2d) ? 0 : (c->fused ? 4 : 4 * per_stage);   // 0: one launch per nlse_step call
    const int64_t cbytes = 2 * c->eb, rv = c->hasV ? c->eb : 0;
    out->min_bytes_per_step = (16 * cbytes + 4 * rv) * c->g.n;
    out->device_bytes = c->device_bytes;
    out->elem_bytes = c->eb;
    snprintf(out->variant, sizeof out->variant, "%s",
             c->persist1d ? (c->cluster1d > 1 ? "rk4_1d_cluster" : "rk4_1d_persistent")
                          : (c->persist2d ? "rk4_2d_persistent"
                                          : (c->fused ? kKindName[KK_FUSED3D] : kKindName[c->interior_kind])));
    out->rank = c->rank;
    out->nranks = c->nranks;
    out->z0 = c->z0;
    out->nz_local = c->g.ns;
    return NLSE_OK;
}

}  // extern "C"
