// nlse_api.cu -- the C ABI (include/nlse.h) and the runtime behind it: context,
// device buffers, constants, validation, stage sequencing (a8), divergence flag,
// diagnostics launch and per-kernel timing.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nlse.h"
#include "common.cuh"
#include "diag.cuh"
#include "generic.cuh"
#include "stream3d.cuh"
#include "tile2d.cuh"

using namespace nlse;

namespace {

thread_local std::string g_create_error;

enum KernelKind { KK_GENERIC = 0, KK_STREAM3D, KK_TILE2D, KK_TILE1D, KK_BOUNDARY, KK_DIAG, KK_COUNT };
const char *kKindName[KK_COUNT] = {"stage_generic", "stage3d_stream", "stage2d_tile", "stage1d_tile",
                                   "stage_boundary", "diag"};

struct TimedLaunch { int kind; cudaEvent_t a, b; int64_t points; };

}  // namespace

struct nlse_ctx {
    int ndim = 0;
    int64_t dims[3] = {1, 1, 1};
    double h = 0, a = 0, s = 0;
    nlse_bc bc = NLSE_BC_DIRICHLET;
    nlse_order order = NLSE_CD2;
    nlse_precision prec = NLSE_FP64;
    uint32_t flags = 0;
    Grid g{};
    int eb = 8;                // sizeof(real)
    bool hasV = false;
    void *psi = nullptr, *K = nullptr, *tmp = nullptr, *outb = nullptr, *V = nullptr;
    int *d_div = nullptr;
    int *h_div = nullptr;      // pinned
    double *d_partial = nullptr, *d_result = nullptr, *h_result = nullptr;
    int diag_blocks = 0;
    cudaStream_t stream = nullptr;
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

// One stage of one step: interior kernel family + boundary kernel (or the generic
// kernel over the whole grid).
template <typename T, int DIM, int ORDER, int BC, int STAGE>
void launch_stage(nlse_ctx *c, const StageArgs<T> &A) {
    if (c->interior_kind == KK_GENERIC) {
        LaunchTimer lt(c, KK_GENERIC, c->g.n);
        stage_generic<T, DIM, ORDER, BC, STAGE><<<blocks_for(c->g.n, 256), 256, 0, c->stream>>>(A);
        return;
    }
    {
        const int64_t ni = (c->g.nx - 2) * (DIM >= 2 ? c->g.ny - 2 : 1) * (DIM >= 3 ? c->g.nz - 2 : 1);
        LaunchTimer lt(c, c->interior_kind, ni);
        if (DIM == 3) launch_stream3d<T, ORDER, BC, STAGE>(A, c->stream);
        else if (DIM == 2) launch_tile2d<T, ORDER, BC, STAGE>(A, c->stream);
        else launch_tile1d<T, ORDER, BC, STAGE>(A, c->stream);
    }
    {
        const int64_t nb = n_boundary_points<DIM>(c->g);
        LaunchTimer lt(c, KK_BOUNDARY, nb);
        stage_boundary<T, DIM, ORDER, BC, STAGE><<<blocks_for(nb, 256), 256, 0, c->stream>>>(A);
    }
}

template <typename T, int DIM, int ORDER, int BC>
nlse_status run_steps(nlse_ctx *c, double k, int64_t nsteps) {
    using C = cplx<T>;
    C *psi = (C *)c->psi, *K = (C *)c->K, *tmp = (C *)c->tmp, *outb = (C *)c->outb;
    const T *V = (const T *)c->V;
    const Consts<T> c2 = make_consts<T>(c, k / 2.0), c1 = make_consts<T>(c, k), c6 = make_consts<T>(c, k / 6.0);
    for (int64_t n = 0; n < nsteps; n++) {
        const int step = int(std::min<int64_t>(c->steps_done + n, INT32_MAX - 1));
        // (RK4_GPU) P:495-519: 1-3, 4-6, 7-9, 10-11
        launch_stage<T, DIM, ORDER, BC, 1>(c, StageArgs<T>{psi, psi, K, tmp, V, c->g, c2, c->d_div, step});
        launch_stage<T, DIM, ORDER, BC, 2>(c, StageArgs<T>{tmp, psi, K, outb, V, c->g, c2, c->d_div, step});
        launch_stage<T, DIM, ORDER, BC, 3>(c, StageArgs<T>{outb, psi, K, tmp, V, c->g, c1, c->d_div, step});
        launch_stage<T, DIM, ORDER, BC, 4>(c, StageArgs<T>{tmp, psi, K, psi, V, c->g, c6, c->d_div, step});
    }
    CUDA_TRY(c, cudaGetLastError());
    return NLSE_OK;
}

template <typename F>
nlse_status dispatch(nlse_ctx *c, F &&f) {
    auto by_bc = [&](auto T, auto DIM, auto ORD) -> nlse_status {
        if (c->bc == NLSE_BC_MSD) return f(T, DIM, ORD, std::integral_constant<int, BC_MSD>());
        return f(T, DIM, ORD, std::integral_constant<int, BC_DIRICHLET>());
    };
    auto by_order = [&](auto T, auto DIM) -> nlse_status {
        if (c->order == NLSE_2SHOC4) return by_bc(T, DIM, std::integral_constant<int, ORDER_2SHOC>());
        return by_bc(T, DIM, std::integral_constant<int, ORDER_CD>());
    };
    auto by_dim = [&](auto T) -> nlse_status {
        if (c->ndim == 1) return by_order(T, std::integral_constant<int, 1>());
        if (c->ndim == 2) return by_order(T, std::integral_constant<int, 2>());
        return by_order(T, std::integral_constant<int, 3>());
    };
    if (c->prec == NLSE_FP64) return by_dim(double());
    return by_dim(float());
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

nlse_status check_ctx(nlse_ctx *c) {
    if (!c) return fail(nullptr, NLSE_ERR_ARG, "ctx is NULL");
    if (c->sticky) return NLSE_ERR_CUDA;
    return NLSE_OK;
}

// Host double (re, im) -> device working precision, staged through a device double buffer.
nlse_status upload_complex(nlse_ctx *c, const double *host, void *dev) {
    const size_t n = size_t(c->g.n);
    if (c->prec == NLSE_FP64) {
        CUDA_TRY(c, cudaMemcpyAsync(dev, host, n * 16, cudaMemcpyHostToDevice, c->stream));
    } else {
        // stage through Psi_out (unused between steps) reinterpreted as double2 scratch in chunks
        const size_t chunk = size_t(c->g.n) / 2 > 0 ? size_t(c->g.n) / 2 : 1;  // outb holds n float2 = n/2 double2
        double2 *scratch = (double2 *)c->outb;
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
        const size_t chunk = size_t(c->g.n) / 2 > 0 ? size_t(c->g.n) / 2 : 1;
        double2 *scratch = (double2 *)c->outb;
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

void nlse_destroy(nlse_ctx *c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto &t : c->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    cudaFree(c->psi); cudaFree(c->K); cudaFree(c->tmp); cudaFree(c->outb); cudaFree(c->V);
    cudaFree(c->d_div); cudaFree(c->d_partial); cudaFree(c->d_result);
    if (c->h_div) cudaFreeHost(c->h_div);
    if (c->h_result) cudaFreeHost(c->h_result);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

nlse_status nlse_create(int ndim, const int64_t dims[3], double h, double a, double s, const double *V,
                        nlse_bc bc, nlse_order order, nlse_precision prec, uint32_t flags, nlse_ctx **out) {
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
    if (bc != NLSE_BC_DIRICHLET && bc != NLSE_BC_MSD) return fail(nullptr, NLSE_ERR_ARG, "unknown bc");
    if (order != NLSE_CD2 && order != NLSE_2SHOC4) return fail(nullptr, NLSE_ERR_ARG, "unknown order");
    if (prec != NLSE_FP32 && prec != NLSE_FP64) return fail(nullptr, NLSE_ERR_ARG, "unknown precision");
    const int64_t n = dims[0] * dims[1] * dims[2];
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
    c->g.nx = dims[0]; c->g.ny = dims[1]; c->g.nz = dims[2];
    c->g.sy = dims[0]; c->g.sz = dims[0] * dims[1]; c->g.n = n;
    c->eb = prec == NLSE_FP64 ? 8 : 4;
    c->hasV = V != nullptr;
    if (flags & NLSE_FLAG_GENERIC_KERNELS) c->interior_kind = KK_GENERIC;
    else c->interior_kind = ndim == 3 ? KK_STREAM3D : (ndim == 2 ? KK_TILE2D : KK_TILE1D);

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

    CREATE_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    const size_t cb = size_t(n) * 2 * c->eb;
    CREATE_TRY(cudaMalloc(&c->psi, cb));
    CREATE_TRY(cudaMalloc(&c->K, cb));
    CREATE_TRY(cudaMalloc(&c->tmp, cb));
    CREATE_TRY(cudaMalloc(&c->outb, cb));
    c->device_bytes = int64_t(4 * cb);
    CREATE_TRY(cudaMemsetAsync(c->psi, 0, cb, c->stream));
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
    CREATE_TRY(cudaMalloc(&c->d_div, sizeof(int)));
    CREATE_TRY(cudaMallocHost(&c->h_div, sizeof(int)));
    int big = INT32_MAX;
    CREATE_TRY(cudaMemcpyAsync(c->d_div, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    c->diag_blocks = nsm * 8;
    CREATE_TRY(cudaMalloc(&c->d_partial, sizeof(double) * 2 * c->diag_blocks));
    CREATE_TRY(cudaMalloc(&c->d_result, sizeof(double) * 2));
    CREATE_TRY(cudaMallocHost(&c->h_result, sizeof(double) * 2));
    CREATE_TRY(cudaStreamSynchronize(c->stream));
#undef CREATE_TRY
    *out = c;
    return NLSE_OK;
}

nlse_status nlse_set_psi(nlse_ctx *c, const double *psi) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!psi) return fail(c, NLSE_ERR_ARG, "psi is NULL");
    return upload_complex(c, psi, c->psi);
}

nlse_status nlse_get_psi(nlse_ctx *c, double *psi) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!psi) return fail(c, NLSE_ERR_ARG, "psi_out is NULL");
    return download_complex(c, c->psi, psi);
}

nlse_status nlse_set_psi_device(nlse_ctx *c, const void *d) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!d) return fail(c, NLSE_ERR_ARG, "d_psi is NULL");
    CUDA_TRY(c, cudaMemcpyAsync(c->psi, d, size_t(c->g.n) * 2 * c->eb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

nlse_status nlse_get_psi_device(nlse_ctx *c, void *d) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!d) return fail(c, NLSE_ERR_ARG, "d_psi is NULL");
    CUDA_TRY(c, cudaMemcpyAsync(d, c->psi, size_t(c->g.n) * 2 * c->eb, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return NLSE_OK;
}

nlse_status nlse_step(nlse_ctx *c, double k, int64_t nsteps) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!std::isfinite(k) || !(k > 0)) return fail(c, NLSE_ERR_ARG, "k must be finite and > 0");
    if (nsteps < 0) return fail(c, NLSE_ERR_ARG, "nsteps must be >= 0");
    if (nsteps == 0) return NLSE_OK;
    const double kmax = linear_bound(c->ndim, c->a, c->h, c->order);
    if (k > kmax && !(c->flags & NLSE_FLAG_FORCE_DT)) {
        char buf[160];
        snprintf(buf, sizeof buf, "k = %.9g exceeds the linear stability bound %.9g (P:363-372); use NLSE_FLAG_FORCE_DT", k, kmax);
        return fail(c, NLSE_ERR_UNSTABLE, buf);
    }
    st = dispatch(c, [&](auto T, auto DIM, auto ORD, auto BCK) -> nlse_status {
        return run_steps<decltype(T), decltype(DIM)::value, decltype(ORD)::value, decltype(BCK)::value>(c, k, nsteps);
    });
    if (st) return st;
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

nlse_status nlse_diagnostics(nlse_ctx *c, double *mass, double *ham) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!mass || !ham) return fail(c, NLSE_ERR_ARG, "mass / hamiltonian pointer is NULL");
    double hd = c->h;
    for (int d = 1; d < c->ndim; d++) hd *= c->h;
    const double ih2 = 1.0 / (c->h * c->h);
    {
        LaunchTimer lt(c, KK_DIAG, c->g.n);
        auto go = [&](auto T, auto DIM) {
            using TT = decltype(T);
            diag_partial<TT, decltype(DIM)::value><<<c->diag_blocks, DIAG_THREADS, 0, c->stream>>>(
                (const cplx<TT> *)c->psi, (const TT *)c->V, c->g, c->a, c->s, ih2, c->d_partial);
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
        diag_final<<<1, DIAG_THREADS, 0, c->stream>>>(c->d_partial, c->diag_blocks, hd, c->d_result);
    }
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->h_result, c->d_result, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->timing) collect_timing(c);
    *mass = c->h_result[0];
    *ham = c->h_result[1];
    return NLSE_OK;
}

nlse_status nlse_get_stream(nlse_ctx *c, void **stream) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!stream) return fail(c, NLSE_ERR_ARG, "stream is NULL");
    *stream = (void *)c->stream;
    return NLSE_OK;
}

nlse_status nlse_set_timing(nlse_ctx *c, int enable) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    c->timing = enable != 0;
    return NLSE_OK;
}

nlse_status nlse_reset_timing(nlse_ctx *c) {
    nlse_status st = check_ctx(c);
    if (st) return st;
    for (int i = 0; i < KK_COUNT; i++) { c->kind_ms[i] = 0; c->kind_launches[i] = 0; c->kind_points[i] = 0; }
    return NLSE_OK;
}

nlse_status nlse_get_timing(nlse_ctx *c, nlse_timing *out) {
    nlse_status st = check_ctx(c);
    if (st) return st;
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
    nlse_status st = check_ctx(c);
    if (st) return st;
    if (!out) return fail(c, NLSE_ERR_ARG, "out is NULL");
    memset(out, 0, sizeof *out);
    out->points = c->g.n;
    out->launches_per_step = c->interior_kind == KK_GENERIC ? 4 : 8;
    const int64_t cbytes = 2 * c->eb, rv = c->hasV ? c->eb : 0;
    out->min_bytes_per_step = (16 * cbytes + 4 * rv) * c->g.n;
    out->device_bytes = c->device_bytes;
    out->elem_bytes = c->eb;
    snprintf(out->variant, sizeof out->variant, "%s", kKindName[c->interior_kind]);
    return NLSE_OK;
}

}  // extern "C"
