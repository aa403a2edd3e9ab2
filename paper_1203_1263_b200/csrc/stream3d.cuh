// stream3d.cuh -- the 3D interior stage kernel: one fused HBM pass per RK4 stage
// (§8(a) rows a1-a5, a7), 2.5D z-streaming.
//
// Each CTA owns a TX x TY column tile of interior output points (TX = 32 = one warp
// along x, TY = 8*RY; every thread owns RY consecutive y rows of one x column) and
// streams it along z through a z-chunk:
//   * the stage input Y arrives plane by plane in shared memory through cp.async
//     (LDGSTS, L2-only .cg), as a (TX+2H) x (TY+2H) tile with an H = w wide halo
//     (w = 1 CD, 2 2SHOC), in a ring of NB plane buffers, up to three planes ahead;
//   * Psi, K_tot and V are read once, at the owned points, straight into registers
//     at the top of the plane iteration (in flight while D is computed);
//   * 2SHOC step 1 (D = Delta_2 Y / h^2) for plane z+1 is computed over
//     the tile plus a one-point ring and kept in shared memory (two plane buffers);
//     D never touches HBM.  D at the owned column of planes z-1, z, z+1 and the pair
//     sums Px = Y[-x]+Y[+x], Py = Y[-y]+Y[+y] of planes z-1, z, z+1 live in registers
//     (a register queue along z): the 2SHOC edge cross term of step 2 is
//     exactly sums of those pair sums, 9 adds per component;
//   * boundary-face D values a 2SHOC interior point needs come from the Laplacian
//     form of the BC, evaluated in place;
//   * step 2, F (fsplit) and the RK4 stage combine run in registers; K_tot and the
//     stage output are stored once.
// Domain-boundary outputs (the BC time-derivative form) are written by
// stage_boundary (generic.cuh).  Every value follows the DAG of DESIGN.md §3.1, so
// the output is bit-identical to the oracle.
#pragma once
#include <cstdlib>
#include "generic.cuh"

namespace nlse {

__device__ __forceinline__ void cp_async16(unsigned saddr, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(unsigned saddr, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <typename T> __device__ __forceinline__ cplx<T> cnan() {
    cplx<T> r; r.x = T(NAN); r.y = T(NAN); return r;
}

constexpr int S3_TX = 32;
constexpr int S3_THREADS = 256;
constexpr int S3_TYT = S3_THREADS / S3_TX;  // 8 thread rows

template <typename T, int ORDER, int RY>
struct S3Cfg {
    static constexpr int H = (ORDER == ORDER_2SHOC) ? 2 : 1;
    static constexpr int TX = S3_TX;
    static constexpr int TY = S3_TYT * RY;
    static constexpr int PX = TX + 2 * H;          // Y tile pitch (elements)
    static constexpr int PY = TY + 2 * H;
    static constexpr int PLANE = PX * PY;
    static constexpr int NB = (ORDER == ORDER_2SHOC) ? 5 : 4;   // Y plane buffers
    static constexpr int DPX = TX + 2, DPY = TY + 2, DPLANE = DPX * DPY;
    static constexpr int ND = (ORDER == ORDER_2SHOC) ? 2 : 0;   // D plane buffers
    static constexpr int RING = 2 * TX + 2 * TY;
    static constexpr size_t smem_bytes() {
        return sizeof(cplx<T>) * (size_t(NB) * PLANE + size_t(ND) * DPLANE);
    }
};

template <typename T, int ORDER, int BC, int RY>
struct S3 {
    using C = cplx<T>;
    using Cfg = S3Cfg<T, ORDER, RY>;
    static constexpr int H = Cfg::H, TX = Cfg::TX, TY = Cfg::TY, PX = Cfg::PX, NB = Cfg::NB;
    static constexpr int DPX = Cfg::DPX;

    const StageArgs<T> &A;
    C *ys;                 // NB Y plane buffers
    C *ds;                 // 2 D plane buffers
    int x0, y0;            // global coords of local (0, 0)

    __device__ __forceinline__ S3(const StageArgs<T> &a, C *smem, int x0_, int y0_)
        : A(a), ys(smem), ds(smem + NB * Cfg::PLANE), x0(x0_), y0(y0_) {}

    // element offset of local (lx, ly) inside a Y plane buffer; lx in [-H, TX+H)
    static __device__ __forceinline__ int yo(int lx, int ly) { return (ly + H) * PX + (lx + H); }
    __device__ __forceinline__ C Ys(int slot, int lx, int ly) const { return ys[slot * Cfg::PLANE + yo(lx, ly)]; }
    __device__ __forceinline__ C &Ds(int dslot, int lx, int ly) const {
        return ds[dslot * Cfg::DPLANE + (ly + 1) * DPX + (lx + 1)];
    }

    // cp.async of plane p into buffer `slot` (in-grid points of the halo tile only).
    __device__ __forceinline__ void load_plane(int64_t p, int slot) const {
        const C *src = A.Y + p * A.g.sz;
        const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(ys + slot * Cfg::PLANE));
        for (int e = threadIdx.x; e < Cfg::PLANE; e += S3_THREADS) {
            const int ly = e / PX - H, lx = e % PX - H;
            const int gx = x0 + lx, gy = y0 + ly;
            if (gx >= 0 && gx < A.g.nx && gy >= 0 && gy < A.g.ny) {
                if (sizeof(C) == 16) cp_async16(sbase + e * 16, src + int64_t(gy) * A.g.sy + gx);
                else cp_async8(sbase + e * 8, src + int64_t(gy) * A.g.sy + gx);
            }
        }
    }

    // D at an interior point from shared memory (slots of planes p-1, p, p+1).
    __device__ __forceinline__ C D_int_s(int sm, int s0, int sp, int lx, int ly) const {
        const C y0v = Ys(s0, lx, ly);
        const C y2 = cadd(y0v, y0v);
        C acc = csub(cadd(Ys(s0, lx - 1, ly), Ys(s0, lx + 1, ly)), y2);
        acc = cadd(acc, csub(cadd(Ys(s0, lx, ly - 1), Ys(s0, lx, ly + 1)), y2));
        acc = cadd(acc, csub(cadd(Ys(sm, lx, ly), Ys(sp, lx, ly)), y2));
        return cscale(A.c.ih2, acc);
    }

    __device__ __forceinline__ T nlin(int64_t q, C yq) const {
        T rho = (yq.x * yq.x) + (yq.y * yq.y);
        T n = A.c.s * rho;
        if (A.V) n = n - __ldg(A.V + q);
        return n;
    }

    // Boundary D on a face point b (Laplacian-form BC, (BCDlap) P:320-323 / (BCMSDlap)
    // P:336-344), given Y_b, Y_b' and D_b' (b' = inward normal neighbour).
    __device__ __forceinline__ C D_face_val(int64_t qb, C yb, int64_t qb1, C y1, C d1) const {
        if (BC == BC_L0) { C z; z.x = T(0); z.y = T(0); return z; }   // (BCL0lap) P:352-355
        const T nb = nlin(qb, yb);
        if (BC == BC_DIRICHLET) {
            T t = A.c.inv_a * nb;
            C r; r.x = -(t * yb.x); r.y = -(t * yb.y);
            return r;
        } else {
            T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T re = T(0);
            if (!(rho1 < A.c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
            T n1 = nlin(qb1, y1);
            T gg = re + ((n1 - nb) * A.c.inv_a);
            return cscale(gg, yb);
        }
    }

    // D at (lx, ly) of an INTERIOR plane p (slots sm, s0, sp): interior point -> stencil,
    // x / y face -> BC form with D at the in-plane inward neighbour recomputed here,
    // edge or outside -> NaN (never used, R-DFACE).
    __device__ C D_plane_s(int64_t p, int sm, int s0, int sp, int lx, int ly) const {
        const int gx = x0 + lx, gy = y0 + ly;
        if (gx < 0 || gx >= A.g.nx || gy < 0 || gy >= A.g.ny) return cnan<T>();
        const bool fx = (gx == 0 || gx == A.g.nx - 1), fy = (gy == 0 || gy == A.g.ny - 1);
        if (!fx && !fy) return D_int_s(sm, s0, sp, lx, ly);
        if (fx && fy) return cnan<T>();
        int lx1 = lx, ly1 = ly;
        if (gx == 0) lx1 = lx + 1; else if (gx == A.g.nx - 1) lx1 = lx - 1;
        else if (gy == 0) ly1 = ly + 1; else ly1 = ly - 1;
        const C d1 = D_int_s(sm, s0, sp, lx1, ly1);
        const int64_t qb = p * A.g.sz + int64_t(gy) * A.g.sy + gx;
        const int64_t qb1 = p * A.g.sz + int64_t(y0 + ly1) * A.g.sy + (x0 + lx1);
        return D_face_val(qb, Ys(s0, lx, ly), qb1, Ys(s0, lx1, ly1), d1);
    }

    __device__ __forceinline__ void ring_xy(int t, int &lx, int &ly) const {
        if (t < TX) { lx = t; ly = -1; }
        else if (t < 2 * TX) { lx = t - TX; ly = TY; }
        else if (t < 2 * TX + TY) { lx = -1; ly = t - 2 * TX; }
        else { lx = TX; ly = t - 2 * TX - TY; }
    }
};

// F (fsplit) P:424-428 and the RK4 stage combine (RK4_GPU) P:495-519 at one point.
template <typename T, int STAGE>
__device__ __forceinline__ void finish_point(const StageArgs<T> &A, int64_t q, int z, cplx<T> yc, cplx<T> L,
                                             cplx<T> psi, cplx<T> kt, T v) {
    using C = cplx<T>;
    T rho = (yc.x * yc.x) + (yc.y * yc.y);
    T sr = A.c.s * rho;
    T fr = tfma(-A.c.a, L.y, -(sr * yc.y));
    T fi = tfma(A.c.a, L.x, sr * yc.x);
    if (A.V) { fr = tfma(v, yc.y, fr); fi = tfma(-v, yc.x, fi); }
    C F; F.x = fr; F.y = fi;
    if (STAGE == 1) {
        A.K[q] = F;
        store_out(A, q, z, cfma(A.c.kc, F, yc));
    } else if (STAGE == 4) {
        C r4 = cfma(A.c.kc, cadd(kt, F), psi);
        store_out(A, q, z, r4);
        if (!(isfinite(r4.x) && isfinite(r4.y))) atomicMin(A.diverged, *A.step_base + A.step);
    } else {
        A.K[q] = cfma(T(2), F, kt);
        store_out(A, q, z, cfma(A.c.kc, F, psi));
    }
}

template <typename T, int ORDER, int BC, int STAGE, int RY>
__global__ void __launch_bounds__(S3_THREADS, (sizeof(T) == 8 ? 2 : 3))
stage3d_stream(StageArgs<T> A, int zchunk) {
    using C = cplx<T>;
    using Cfg = S3Cfg<T, ORDER, RY>;
    using K = S3<T, ORDER, BC, RY>;
    constexpr int NB = Cfg::NB;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const int tx = threadIdx.x % S3_TX, ty = threadIdx.x / S3_TX;
    const int x0 = 1 + blockIdx.x * Cfg::TX;
    const int y0 = 1 + blockIdx.y * Cfg::TY;
    // output planes: the owned planes that are not global z faces, split in z chunks
    const int zlo = A.g.zf_lo ? 1 : 0, zhi = int(A.g.nz) - (A.g.zf_hi ? 1 : 0);
    const int zmem_lo = A.g.zf_lo ? 0 : -A.g.zghost;               // planes present in memory
    const int zmem_hi = int(A.g.nz) + (A.g.zf_hi ? 0 : A.g.zghost);
    const int zs = zlo + blockIdx.z * zchunk;
    const int ze = min(zs + zchunk, zhi);   // outputs [zs, ze)
    if (zs >= ze) return;
    const K k(A, reinterpret_cast<C *>(smem_raw), x0, y0);
    const Grid &g = A.g;
    const int gx = x0 + tx;
    const int ly0 = ty * RY;
    int64_t qrow[RY];             // global offset of (gx, gy[r]) in plane 0
    bool row_in[RY], out_ok[RY];
#pragma unroll
    for (int r = 0; r < RY; r++) {
        const int gy = y0 + ly0 + r;
        qrow[r] = int64_t(gy) * g.sy + gx;
        row_in[r] = gx < g.nx && gy < g.ny;
        out_ok[r] = gx <= g.nx - 2 && gy <= g.ny - 2;
    }

    if (ORDER == ORDER_CD) {
        // ------------------------------------------------------------------ CD: L = D
        int sm = (zs - 1 + NB) % NB, s0 = zs % NB, sp = (zs + 1) % NB;
        k.load_plane(zs - 1, sm);
        k.load_plane(zs, s0);
        k.load_plane(zs + 1, sp);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        C ym[RY], yc[RY];
#pragma unroll
        for (int r = 0; r < RY; r++) { ym[r] = k.Ys(sm, tx, ly0 + r); yc[r] = k.Ys(s0, tx, ly0 + r); }
        for (int z = zs; z < ze; z++) {
            const int sn = (sp + 1 == NB) ? 0 : sp + 1;
            if (z + 1 < ze) k.load_plane(z + 2, sn);
            cp_async_commit();
            const int64_t zo = int64_t(z) * g.sz;
            C psi[RY], kt[RY];
            T v[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) {
                if (out_ok[r]) {
                    if (STAGE != 1) psi[r] = ldg_c(A.Psi + zo + qrow[r]);
                    if (STAGE != 1) kt[r] = A.K[zo + qrow[r]];
                    if (A.V) v[r] = __ldg(A.V + zo + qrow[r]);
                }
            }
            C yp[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) yp[r] = k.Ys(sp, tx, ly0 + r);
#pragma unroll
            for (int r = 0; r < RY; r++) {
                if (!out_ok[r]) continue;
                const int ly = ly0 + r;
                const C y2 = cadd(yc[r], yc[r]);
                const C ya = (r > 0) ? yc[r - 1] : k.Ys(s0, tx, ly - 1);
                const C yb = (r < RY - 1) ? yc[r + 1] : k.Ys(s0, tx, ly + 1);
                C acc = csub(cadd(k.Ys(s0, tx - 1, ly), k.Ys(s0, tx + 1, ly)), y2);
                acc = cadd(acc, csub(cadd(ya, yb), y2));
                acc = cadd(acc, csub(cadd(ym[r], yp[r]), y2));
                const C L = cscale(A.c.ih2, acc);
                finish_point<T, STAGE>(A, zo + qrow[r], z, yc[r], L, psi[r], kt[r], v[r]);
            }
#pragma unroll
            for (int r = 0; r < RY; r++) { ym[r] = yc[r]; yc[r] = yp[r]; }
            sm = s0; s0 = sp; sp = sn;
            cp_async_wait_all();
            __syncthreads();
        }
        return;
    }

    // ---------------------------------------------------------------------- 2SHOC
    // slots of planes z-1, z, z+1, z+2 (and z-2 in the prologue)
    int s_m1 = (zs - 1 + NB) % NB, s_0 = zs % NB, s_1 = (zs + 1) % NB, s_2 = (zs + 2) % NB;
    const int s_m2 = (zs + NB - 2) % NB;
    if (zs - 2 >= zmem_lo) k.load_plane(zs - 2, s_m2);
    k.load_plane(zs - 1, s_m1);
    k.load_plane(zs, s_0);
    k.load_plane(zs + 1, s_1);
    if (zs + 2 < zmem_hi) k.load_plane(zs + 2, s_2);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();

    C yq0[RY], yq1[RY];                 // Y center at z, z+1
    C dm[RY], d0[RY];                   // D center at z-1, z
    C pxm[RY], pym[RY], px0[RY], py0[RY];   // pair sums at z-1, z
    int dsl = zs & 1;                   // D slot of plane z
    // D(zs) over the owned columns + ring; pair sums at zs and zs-1
#pragma unroll
    for (int r = 0; r < RY; r++) {
        const int ly = ly0 + r;
        yq0[r] = k.Ys(s_0, tx, ly);
        yq1[r] = k.Ys(s_1, tx, ly);
        px0[r] = cadd(k.Ys(s_0, tx - 1, ly), k.Ys(s_0, tx + 1, ly));
        py0[r] = cadd(k.Ys(s_0, tx, ly - 1), k.Ys(s_0, tx, ly + 1));
        pxm[r] = cadd(k.Ys(s_m1, tx - 1, ly), k.Ys(s_m1, tx + 1, ly));
        pym[r] = cadd(k.Ys(s_m1, tx, ly - 1), k.Ys(s_m1, tx, ly + 1));
        d0[r] = row_in[r] ? k.D_plane_s(zs, s_m1, s_0, s_1, tx, ly) : cnan<T>();
        k.Ds(dsl, tx, ly) = d0[r];
    }
    for (int t = threadIdx.x; t < Cfg::RING; t += S3_THREADS) {
        int lx, ly;
        k.ring_xy(t, lx, ly);
        k.Ds(dsl, lx, ly) = k.D_plane_s(zs, s_m1, s_0, s_1, lx, ly);
    }
#pragma unroll
    for (int r = 0; r < RY; r++) {
        const int ly = ly0 + r;
        if (!out_ok[r]) { dm[r] = cnan<T>(); continue; }
        if (g.zf_lo && zs - 1 == 0) {
            // z face: BC form with b' = (x, y, 1), whose D was computed above
            dm[r] = k.D_face_val(qrow[r], k.Ys(s_m1, tx, ly), qrow[r] + g.sz, yq0[r], d0[r]);
        } else {
            dm[r] = k.D_int_s(s_m2, s_m1, s_0, tx, ly);
        }
    }
    __syncthreads();

    for (int z = zs; z < ze; z++) {
        // (1) Y plane z+3 (into the slot of plane z-2) and this plane's Psi, K, V
        const int s_3 = (s_2 + 1 == NB) ? 0 : s_2 + 1;
        if (z + 1 < ze && z + 3 < zmem_hi) k.load_plane(z + 3, s_3);
        cp_async_commit();
        const int64_t zo = int64_t(z) * g.sz;
        C psi[RY], kt[RY];
        T v[RY];
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (out_ok[r]) {
                if (STAGE != 1) psi[r] = ldg_c(A.Psi + zo + qrow[r]);
                if (STAGE != 1) kt[r] = A.K[zo + qrow[r]];
                if (A.V) v[r] = __ldg(A.V + zo + qrow[r]);
            }
        }

        // (2) D(z+1) at the owned columns, pair sums at z+1
        const int zp = z + 1;
        const bool zface = g.zf_hi && (zp == g.nz - 1);
        const int dsn = dsl ^ 1;
        C dn[RY], px1[RY], py1[RY], yq2[RY];
#pragma unroll
        for (int r = 0; r < RY; r++) {
            const int ly = ly0 + r;
            px1[r] = cadd(k.Ys(s_1, tx - 1, ly), k.Ys(s_1, tx + 1, ly));
            const C ya = (r > 0) ? yq1[r - 1] : k.Ys(s_1, tx, ly - 1);
            const C yb = (r < RY - 1) ? yq1[r + 1] : k.Ys(s_1, tx, ly + 1);
            py1[r] = cadd(ya, yb);
            yq2[r] = k.Ys(s_2, tx, ly);           // garbage on the last plane (unused there)
        }
#pragma unroll
        for (int r = 0; r < RY; r++) {
            const int ly = ly0 + r;
            if (out_ok[r]) {
                if (zface) {
                    dn[r] = k.D_face_val(zo + g.sz + qrow[r], yq1[r], zo + qrow[r], yq0[r], d0[r]);
                } else {
                    const C y2 = cadd(yq1[r], yq1[r]);
                    C acc = csub(px1[r], y2);
                    acc = cadd(acc, csub(py1[r], y2));
                    acc = cadd(acc, csub(cadd(yq0[r], yq2[r]), y2));
                    dn[r] = cscale(A.c.ih2, acc);
                }
            } else if (row_in[r] && !zface) {
                dn[r] = k.D_plane_s(zp, s_0, s_1, s_2, tx, ly);   // x / y face column inside the tile
            } else {
                dn[r] = cnan<T>();
            }
            k.Ds(dsn, tx, ly) = dn[r];
        }
        if (!zface) {
            for (int t = threadIdx.x; t < Cfg::RING; t += S3_THREADS) {
                int lx, ly;
                k.ring_xy(t, lx, ly);
                k.Ds(dsn, lx, ly) = k.D_plane_s(zp, s_0, s_1, s_2, lx, ly);
            }
        }
        __syncthreads();

        // (3) 2SHOC step 2 at (x, y, z), F, RK4 stage combine
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (!out_ok[r]) continue;
            const int ly = ly0 + r;
            const C yc = yq0[r];
            const C y4 = cscale(T(4), yc);
            // edge cross term E (grouping of DESIGN.md §3.1)
            const C pxa = (r > 0) ? px0[r - 1] : cadd(k.Ys(s_0, tx - 1, ly - 1), k.Ys(s_0, tx + 1, ly - 1));
            const C pxb = (r < RY - 1) ? px0[r + 1] : cadd(k.Ys(s_0, tx - 1, ly + 1), k.Ys(s_0, tx + 1, ly + 1));
            const C exy = csub(cadd(pxa, pxb), y4);
            const C exz = csub(cadd(pxm[r], px1[r]), y4);
            const C eyz = csub(cadd(pym[r], py1[r]), y4);
            const C E = cadd(cadd(exy, exz), eyz);
            // D terms
            const C dya = (r > 0) ? d0[r - 1] : k.Ds(dsl, tx, ly - 1);
            const C dyb = (r < RY - 1) ? d0[r + 1] : k.Ds(dsl, tx, ly + 1);
            const C sd = cadd(cadd(cadd(k.Ds(dsl, tx - 1, ly), k.Ds(dsl, tx + 1, ly)), cadd(dya, dyb)),
                              cadd(dm[r], dn[r]));
            const C td = cfma(T(-10), d0[r], sd);
            const C L = cfma(A.c.c16h2, E, cneg(cscale(A.c.c112, td)));
            finish_point<T, STAGE>(A, zo + qrow[r], z, yc, L, psi[r], kt[r], v[r]);
        }
        // (4) rotate the register queues and the slots
#pragma unroll
        for (int r = 0; r < RY; r++) {
            dm[r] = d0[r]; d0[r] = dn[r];
            pxm[r] = px0[r]; px0[r] = px1[r];
            pym[r] = py0[r]; py0[r] = py1[r];
            yq0[r] = yq1[r]; yq1[r] = yq2[r];
        }
        s_m1 = s_0; s_0 = s_1; s_1 = s_2; s_2 = s_3;
        dsl = dsn;
        cp_async_wait_all();
        __syncthreads();
    }
}

template <typename T, int ORDER, int BC, int STAGE, int RY>
void launch_stream3d_ry(const StageArgs<T> &A, cudaStream_t st) {
    using Cfg = S3Cfg<T, ORDER, RY>;
    const int64_t mx = A.g.nx - 2, my = A.g.ny - 2, mz = A.g.nz - A.g.zf_lo - A.g.zf_hi;
    const unsigned gx = unsigned((mx + Cfg::TX - 1) / Cfg::TX);
    const unsigned gy = unsigned((my + Cfg::TY - 1) / Cfg::TY);
    // z chunks: enough CTAs for ~4 waves of resident CTAs, chunks >= 32 planes
    const int64_t cols = int64_t(gx) * gy;
    int64_t want = (148 * 2 * 4 + cols - 1) / cols;
    int64_t zchunk = (mz + want - 1) / want;
    if (zchunk < 32) zchunk = 32;
    if (zchunk > mz) zchunk = mz;
    const unsigned gz = unsigned((mz + zchunk - 1) / zchunk);
    const size_t smem = Cfg::smem_bytes();
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(stage3d_stream<T, ORDER, BC, STAGE, RY>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        attr_set = true;
    }
    stage3d_stream<T, ORDER, BC, STAGE, RY><<<dim3(gx, gy, gz), S3_THREADS, smem, st>>>(A, int(zchunk));
}

inline int s3_ry_choice() {
    static int ry = [] {
        const char *e = getenv("NLSE_S3_RY");
        return (e && e[0] == '2') ? 2 : 1;
    }();
    return ry;
}

template <typename T, int ORDER, int BC, int STAGE>
void launch_stream3d(const StageArgs<T> &A, cudaStream_t st) {
    if (s3_ry_choice() == 2) launch_stream3d_ry<T, ORDER, BC, STAGE, 2>(A, st);
    else launch_stream3d_ry<T, ORDER, BC, STAGE, 1>(A, st);
}

}  // namespace nlse
