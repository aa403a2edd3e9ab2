// common.cuh -- shared device-side definitions for the NLSE stage kernels.
//
// All kernels are compiled with -fmad=false (no FMA contraction), IEEE division
// and no FTZ, and evaluate the per-point expression graph fixed in DESIGN.md
// §3.1 (reading R-ASSOC) term by term, so that each output is bit-identical to
// the CPU oracle.  This file holds only CUDA-side code; nothing here is shared
// with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nlse {

enum BcKind { BC_DIRICHLET = 0, BC_MSD = 1, BC_L0 = 2 };
enum OrderKind { ORDER_CD = 2, ORDER_2SHOC = 4 };

template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <typename T> using cplx = typename Vec2<T>::type;

// Programmatic dependent launch (kernels launched with the programmatic-stream-serialization
// attribute): pdl_trigger lets the next kernel on the stream be scheduled while this one runs (its
// CTAs then wait in pdl_wait); pdl_wait blocks until the previous kernel on the stream has completed
// and its memory is visible -- every global access of a kernel comes after it.  Both are no-ops for
// kernels launched without the attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Componentwise helpers: each is exactly one IEEE operation per component.
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { C r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { C r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename C, typename T> __device__ __forceinline__ C cscale(T s, C a) { C r; r.x = s * a.x; r.y = s * a.y; return r; }

template <typename C> __device__ __forceinline__ C ldg_c(const C *p) { return __ldg(p); }

// Fused multiply-add with one IEEE rounding, at the positions DESIGN.md §3.1 (R-ASSOC)
// fixes (the oracle uses C99 fma / fmaf at the same positions).
__device__ __forceinline__ double tfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float tfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <typename C, typename T> __device__ __forceinline__ C cfma(T s, C a, C b) {
    C r; r.x = tfma(s, a.x, b.x); r.y = tfma(s, a.y, b.y); return r;
}
template <typename C> __device__ __forceinline__ C cneg(C a) { C r; r.x = -a.x; r.y = -a.y; return r; }

// fp32: the componentwise complex operations as sm_100 packed-fp32 instructions (FADD2 / FMUL2 /
// FFMA2: add / mul / fma .rn.f32x2).  Each lane is one IEEE round-to-nearest fp32 operation, no
// FTZ, exactly as the scalar pair it replaces -- same bits, half the FP instructions (the fp32
// stage kernels are bound by their instruction stream).  Non-template overloads: preferred over
// the templates above for float2 arguments.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    float2 r;
    asm("{\n.reg .b64 ra, rb, rr;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nadd.rn.f32x2 rr, ra, rb;\n"
        "mov.b64 {%0, %1}, rr;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    float2 r;
    asm("{\n.reg .b64 ra, rb, rr;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nsub.rn.f32x2 rr, ra, rb;\n"
        "mov.b64 {%0, %1}, rr;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 cscale(float s, float2 a) {
    float2 r;
    asm("{\n.reg .b64 rs, ra, rr;\nmov.b64 rs, {%2, %2};\nmov.b64 ra, {%3, %4};\nmul.rn.f32x2 rr, rs, ra;\n"
        "mov.b64 {%0, %1}, rr;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(s), "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 cfma(float s, float2 a, float2 b) {
    float2 r;
    asm("{\n.reg .b64 rs, ra, rb, rr;\nmov.b64 rs, {%2, %2};\nmov.b64 ra, {%3, %4};\nmov.b64 rb, {%5, %6};\n"
        "fma.rn.f32x2 rr, rs, ra, rb;\nmov.b64 {%0, %1}, rr;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(s), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

// F (fsplit) P:424-428 at one point, split as the kernels evaluate it (R-ASSOC):
//   f_lin:  (fma(-a, L_I, -(sr Y_I)), fma(a, L_R, sr Y_R))      sr = s |Y|^2
//   f_addv: (fma(V, Y_I, F_R), fma(-V, Y_R, F_I))                 (with a V array)
// fp32: one FMUL2 + one FFMA2 (lane swap and per-lane negation are operand modifiers), one
// FFMA2 for the V term -- the same IEEE operations per lane as the scalar forms.
template <typename T> __device__ __forceinline__ cplx<T> f_lin(T a, cplx<T> L, T sr, cplx<T> y) {
    cplx<T> F;
    F.x = tfma(-a, L.y, -(sr * y.y));
    F.y = tfma(a, L.x, sr * y.x);
    return F;
}
template <typename T> __device__ __forceinline__ cplx<T> f_addv(cplx<T> F, T v, cplx<T> y) {
    cplx<T> r;
    r.x = tfma(v, y.y, F.x);
    r.y = tfma(-v, y.x, F.y);
    return r;
}
__device__ __forceinline__ float2 f_lin(float a, float2 L, float sr, float2 y) {
    float2 r;
    asm("{\n.reg .b64 rs, ry, rt, ra, rl, rn;\n.reg .f32 t0, t1, n1, na;\n"
        "mov.b64 rs, {%2, %2};\nmov.b64 ry, {%3, %4};\nmul.rn.f32x2 rt, rs, ry;\n"
        "mov.b64 {t0, t1}, rt;\nneg.f32 n1, t1;\nmov.b64 rn, {n1, t0};\n"
        "neg.f32 na, %7;\nmov.b64 ra, {na, %7};\nmov.b64 rl, {%6, %5};\n"
        "fma.rn.f32x2 rt, ra, rl, rn;\nmov.b64 {%0, %1}, rt;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(sr), "f"(y.x), "f"(y.y), "f"(L.x), "f"(L.y), "f"(a));
    return r;
}
__device__ __forceinline__ float2 f_addv(float2 F, float v, float2 y) {
    float2 r;
    asm("{\n.reg .b64 rv, ry, rf, rr;\n.reg .f32 nv;\nneg.f32 nv, %2;\nmov.b64 rv, {%2, nv};\n"
        "mov.b64 ry, {%4, %3};\nmov.b64 rf, {%5, %6};\nfma.rn.f32x2 rr, rv, ry, rf;\nmov.b64 {%0, %1}, rr;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(v), "f"(y.x), "f"(y.y), "f"(F.x), "f"(F.y));
    return r;
}

// Per-run constants, evaluated in double on the host from the user's doubles and
// rounded once to T (reading R-CONST).
template <typename T> struct Consts {
    T ih2;    // 1/h^2                (2shoc1d) P:197
    T c76;    // 7/6                  (2shoc1d2) P:198
    T c112;   // 1/12
    T c16h2;  // 1/(6 h^2)
    T a;      // a                    (NLSE) P:78
    T s;      // s
    T inv_a;  // 1/a                  (BCDlap) P:322, (BCMSDlap) P:338
    T eps2;   // MSD guard (R-MSD-GUARD)
    T kc;     // stage coefficient: k/2 (S1, S2), k (S3), k/6 (S4)   (RK4_GPU) P:495-519
};

// The grid a context owns.  Single GPU: the whole grid.  Slab mode (§8(e)): the z
// planes [z0, z0 + nz) of the global grid; the buffers read with a halo carry zghost
// planes below plane 0 and above plane nz - 1, filled by the neighbours.
// Slab mode partitions the slowest axis (the "slab axis": z in 3D, y in 2D, x in 1D): ns = its
// owned length (nz, ny, nx), su = the stride of one slab-axis step (sz, sy, 1); zf_lo / zf_hi /
// zghost refer to that axis.
struct Grid {
    int64_t nx, ny, nz;   // points per axis (unused = 1); 3D: nz = owned planes, 2D: ny = owned rows
    int64_t sy, sz;       // strides: sy = nx (or the pitched row), sz = sy*ny
    int64_t n;            // owned points
    int zf_lo, zf_hi;     // 1 if local slab-axis index 0 / ns - 1 is a global face (always 1 on one GPU)
    int zghost;           // ghost planes (3D) / rows (2D) on each side of the halo'd buffers (0 on one GPU)
    int64_t ns, su;       // slab axis: owned length and stride (3D: nz, sz; 2D: ny, sy; 1D: nx, 1)
};

// 2D y-slab / 1D x-slab face tests (other axes keep 0 / n - 1 as faces): the low / high end of
// the owned points along the slab axis is a domain face only where the slab holds the global
// face (zf_lo / zf_hi)
template <int DIM>
__host__ __device__ __forceinline__ bool y_face(const Grid &g, int64_t j) {
    if (DIM == 2) return (g.zf_lo && j == 0) || (g.zf_hi && j == g.ny - 1);
    return j == 0 || j == g.ny - 1;
}
template <int DIM>
__host__ __device__ __forceinline__ bool x_face(const Grid &g, int64_t i) {
    if (DIM == 1) return (g.zf_lo && i == 0) || (g.zf_hi && i == g.nx - 1);
    return i == 0 || i == g.nx - 1;
}

// global z-face test for a local plane index (DIM == 3)
__host__ __device__ __forceinline__ bool is_zface(const Grid &g, int64_t k) {
    return (g.zf_lo && k == 0) || (g.zf_hi && k == g.nz - 1);
}

// Stage operands (RK4_GPU) P:495-519.  stage 1: Y = Psi, out = Psi_tmp;
// stage 2: Y = Psi_tmp, out = Psi_out; stage 3: Y = Psi_out, out = Psi_tmp;
// stage 4: Y = Psi_tmp, out = Psi (in place; Psi is read only at the owned point).
template <typename T> struct StageArgs {
    const cplx<T> *Y;
    const cplx<T> *Psi;
    cplx<T> *K;
    cplx<T> *out;
    const T *V;           // nullptr => V = 0 (reading R-V0)
    Grid g;
    Consts<T> c;
    int *diverged;        // stage 4: atomicMin(step index) when a non-finite value is produced
    const int *step_base; // device counter of the steps completed before this launch sequence
    int step;             // step index within the launch sequence (absolute = *step_base + step;
                          // read only when a non-finite value appears, so CUDA graphs can replay)
    // Slab mode: the stage output of the first / last `wsend` owned planes is also stored
    // into the lower / upper neighbour's ghost planes (remote stores over NVLink, the halo
    // exchange a9 fused into the producing kernel).  peer_lo[q] / peer_hi[q] address the
    // neighbour's copy of local point q; nullptr on a global face or on one GPU.
    cplx<T> *peer_lo, *peer_hi;
    int wsend;
    // MSD, 3D TMA path: the interior kernel also stores F at the points b' that the boundary
    // points take their time derivative from ((msd) P:331-335): fz = planes 1 and nz-2
    // (2 x nx*ny), fp = the ring of points one in from the x/y faces of every owned plane
    // (nz x per2, indexed by shell_u).  nullptr: the boundary kernel recomputes F(b').
    cplx<T> *fz, *fp;
    int per2;
    int stream_hints;     // 1: L2 evict-first hints on the once-per-stage streams (measured slower, off)
    int ring_rot;         // 1: rotate the 3D ring-D duty over the warps plane by plane
    int xfuse;            // 3D MSD light-pass mode: the x-face points with 1 <= j <= ny-2 of the
                          // interior planes are finished by the stage kernel (F(b') by a lane
                          // shuffle); the light pass covers the z faces and the y-face rows only
};

// Index of an in-plane point one step in from the x/y faces (nx, ny >= 5), in the order:
// row j = 1, row j = ny-2, then columns i = 1 / i = nx-2 for j = 2 .. ny-3.
__host__ __device__ __forceinline__ int shell_u(int i, int j, int nx, int ny) {
    if (j == 1) return i - 1;
    if (j == ny - 2) return (nx - 2) + (i - 1);
    return 2 * (nx - 2) + 2 * (j - 2) + (i == nx - 2 ? 1 : 0);
}

// Store one stage output value at local point q, slab-axis index k (plane in 3D, row in 2D),
// and into the neighbours' ghosts.
template <typename T>
__device__ __forceinline__ void store_out(const StageArgs<T> &A, int64_t q, int64_t k, cplx<T> v) {
    A.out[q] = v;
    if (A.peer_lo && k < A.wsend) A.peer_lo[q] = v;
    if (A.peer_hi && k >= A.g.ns - A.wsend) A.peer_hi[q] = v;
}

// RK4 stage combine at one point, (RK4_GPU) P:495-519 / (RK4) P:164-180 (fused
// multiply-adds, R-ASSOC):
//   S1: K = F;            out = fma(k/2, F, Psi)
//   S2: K = fma(2, F, K); out = fma(k/2, F, Psi)
//   S3: K = fma(2, F, K); out = fma(k, F, Psi)
//   S4:                   out = fma(k/6, K + F, Psi)
// kz = slab-axis index of q (plane in 3D, row in 2D; for the neighbour stores; 0 in 1D).
template <int STAGE, typename T>
__device__ __forceinline__ void rk_combine(const StageArgs<T> &A, int64_t q, int64_t kz, cplx<T> F, cplx<T> psi) {
    using C = cplx<T>;
    const T two = T(2);
    if (STAGE == 1) {
        A.K[q] = F;
        store_out(A, q, kz, cfma(A.c.kc, F, psi));
    } else if (STAGE == 2 || STAGE == 3) {
        C k = A.K[q];
        A.K[q] = cfma(two, F, k);
        store_out(A, q, kz, cfma(A.c.kc, F, psi));
    } else {
        C k = A.K[q];
        C r = cfma(A.c.kc, cadd(k, F), psi);
        store_out(A, q, kz, r);
        if (!(isfinite(r.x) && isfinite(r.y))) atomicMin(A.diverged, *A.step_base + A.step);
    }
}

}  // namespace nlse
