// stream3d.cuh -- the 3D interior stage kernel: one fused HBM pass per RK4 stage
// (§8(a) rows a1-a5, a7), 2.5D z-streaming.
//
// Each CTA owns a TX x TY column tile of interior output points (TX = 32 = one warp
// along x, TY = 8*RY; every thread owns RY consecutive y rows of one x column) and
// streams it along z through a z-chunk:
//   * the stage input Y arrives plane by plane in shared memory through cp.async
//     (LDGSTS, L2-only .cg), as a (TX+2H) x (TY+2H) tile with an H = w wide halo
//     (w = 1 CD, 2 2SHOC), in a ring of NB plane buffers three planes ahead;
//   * Psi, K_tot and V for the output plane are prefetched one plane ahead into
//     registers (they are read once, at the owned point only);
//   * 2SHOC step 1 (D = Delta_2 Y / h^2) for plane z+1 is computed over
//     the tile plus a one-point ring and kept in shared memory (two plane buffers);
//     D never touches HBM.  D at the owned column of planes z-1, z, z+1 and the pair
//     sums Px = Y[-x]+Y[+x], Py = Y[-y]+Y[+y] of planes z-1, z, z+1 live in registers
//     (register queue along z): the 2SHOC edge cross term of step 2 is
//     exactly sums of those pair sums, so it costs 9 adds/component;
//   * boundary-face D values a 2SHOC interior point needs come from the Laplacian
//     form of the BC, evaluated in place;
//   * step 2, F (fsplit) and the RK4 stage combine run in registers and K_tot and the
//     stage output are stored once.
// Domain-boundary outputs (the BC time-derivative form) are written by
// stage_boundary (generic.cuh).  Every value follows the DAG of DESIGN.md §3.1, so
// the output is bit-identical to the oracle.
#pragma once
#include "generic.cuh"

namespace nlse {

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <typename C>
__device__ __forceinline__ void cp_async_c(C *smem, const C *gmem) {
    if (sizeof(C) == 16) cp_async16(smem, gmem);
    else cp_async8(smem, gmem);
}

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

template <typename T, int ORDER, int BC, int STAGE, int RY>
struct Stream3D {
    using C = cplx<T>;
    using Cfg = S3Cfg<T, ORDER, RY>;
    static constexpr int H = Cfg::H, TX = Cfg::TX, TY = Cfg::TY, PX = Cfg::PX, NB = Cfg::NB;
    static constexpr int DPX = Cfg::DPX;

    const StageArgs<T> &A;
    C *ys;      // NB plane buffers
    C *ds;      // 2 D plane buffers (2SHOC)
    int64_t x0, y0;

    __device__ Stream3D(const StageArgs<T> &a, C *smem, int64_t x0_, int64_t y0_)
        : A(a), ys(smem), ds(smem + size_t(NB) * Cfg::PLANE), x0(x0_), y0(y0_) {}

    // local coords: lx in [-H, TX+H), ly in [-H, TY+H)
    __device__ __forceinline__ C &Y(int64_t p, int lx, int ly) const {
        return ys[size_t(p % NB) * Cfg::PLANE + (ly + H) * PX + (lx + H)];
    }
    __device__ __forceinline__ C &Dl(int64_t p, int lx, int ly) const {
        return ds[size_t(p & 1) * Cfg::DPLANE + (ly + 1) * DPX + (lx + 1)];
    }

    // Issue the cp.async copies of plane p of Y (in-grid points of the halo tile).
    __device__ __forceinline__ void load_plane(int64_t p) const {
        const C *src = A.Y + p * A.g.sz;
        for (int e = threadIdx.x; e < Cfg::PLANE; e += S3_THREADS) {
            const int ly = e / PX - H, lx = e % PX - H;
            const int64_t gx = x0 + lx, gy = y0 + ly;
            if (gx >= 0 && gx < A.g.nx && gy >= 0 && gy < A.g.ny)
                cp_async_c(&Y(p, lx, ly), src + gy * A.g.sy + gx);
        }
    }

    __device__ __forceinline__ int nbnd(int64_t gx, int64_t gy, int64_t p) const {
        return (gx == 0 || gx == A.g.nx - 1) + (gy == 0 || gy == A.g.ny - 1) + (p == 0 || p == A.g.nz - 1);
    }

    // D at an interior point from shared memory (planes p-1, p, p+1 resident).
    __device__ __forceinline__ C D_int_s(int64_t p, int lx, int ly) const {
        const C y0v = Y(p, lx, ly);
        const C y2 = cadd(y0v, y0v);
        C acc = csub(cadd(Y(p, lx - 1, ly), Y(p, lx + 1, ly)), y2);
        acc = cadd(acc, csub(cadd(Y(p, lx, ly - 1), Y(p, lx, ly + 1)), y2));
        acc = cadd(acc, csub(cadd(Y(p - 1, lx, ly), Y(p + 1, lx, ly)), y2));
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

    // D at any needed point (lx, ly) of plane p from shared memory: interior -> stencil,
    // face -> BC form (D at the inward neighbour recomputed here), edge/corner -> unused.
    // Requires planes p-1..p+1 resident (p-2..p+2 for a z face: its b' stencil).
    __device__ C D_any_s(int64_t p, int lx, int ly) const {
        const int64_t gx = x0 + lx, gy = y0 + ly;
        if (gx < 0 || gx >= A.g.nx || gy < 0 || gy >= A.g.ny) return cnan<T>();
        const int nb = nbnd(gx, gy, p);
        if (nb == 0) return D_int_s(p, lx, ly);
        if (nb > 1) return cnan<T>();
        int lx1 = lx, ly1 = ly;
        int64_t p1 = p;
        if (gx == 0) lx1 = lx + 1; else if (gx == A.g.nx - 1) lx1 = lx - 1;
        else if (gy == 0) ly1 = ly + 1; else if (gy == A.g.ny - 1) ly1 = ly - 1;
        else if (p == 0) p1 = 1; else p1 = p - 1;
        const C d1 = D_int_s(p1, lx1, ly1);
        const int64_t qb = p * A.g.sz + gy * A.g.sy + gx;
        const int64_t qb1 = p1 * A.g.sz + (y0 + ly1) * A.g.sy + (x0 + lx1);
        return D_face_val(qb, Y(p, lx, ly), qb1, Y(p1, lx1, ly1), d1);
    }

    // Ring point t (0 <= t < RING) -> local coords.
    __device__ __forceinline__ void ring_xy(int t, int &lx, int &ly) const {
        if (t < TX) { lx = t; ly = -1; }
        else if (t < 2 * TX) { lx = t - TX; ly = TY; }
        else if (t < 2 * TX + TY) { lx = -1; ly = t - 2 * TX; }
        else { lx = TX; ly = t - 2 * TX - TY; }
    }
};

// z face below the first output plane: is (gx, gy) an interior column?
__device__ __forceinline__ bool nbnd_ok(int64_t gx, int64_t gy, const Grid &g) {
    return gx >= 1 && gx <= g.nx - 2 && gy >= 1 && gy <= g.ny - 2;
}

template <typename T, int ORDER, int BC, int STAGE, int RY>
__global__ void __launch_bounds__(S3_THREADS, (sizeof(T) == 8 ? 2 : 3))
stage3d_stream(StageArgs<T> A, int zchunk) {
    using C = cplx<T>;
    using Cfg = S3Cfg<T, ORDER, RY>;
    using K = Stream3D<T, ORDER, BC, STAGE, RY>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *smem = reinterpret_cast<C *>(smem_raw);

    const int tx = threadIdx.x % S3_TX, ty = threadIdx.x / S3_TX;
    const int64_t x0 = 1 + int64_t(blockIdx.x) * Cfg::TX;
    const int64_t y0 = 1 + int64_t(blockIdx.y) * Cfg::TY;
    const int64_t zs = 1 + int64_t(blockIdx.z) * zchunk;
    const int64_t ze = min(zs + zchunk, A.g.nz - 1);   // outputs [zs, ze)
    if (zs >= ze) return;
    K k(A, smem, x0, y0);
    const Grid &g = A.g;
    const int64_t gx = x0 + tx;
    const bool col_in = gx < g.nx;                       // column inside the grid
    const bool col_int = gx <= g.nx - 2;                 // interior column (x)
    int64_t gy[RY];
    bool row_in[RY], out_ok[RY];
#pragma unroll
    for (int r = 0; r < RY; r++) {
        gy[r] = y0 + ty * RY + r;
        row_in[r] = col_in && gy[r] < g.ny;
        out_ok[r] = col_int && gy[r] <= g.ny - 2;
    }
    const int ly0 = ty * RY;

    // register prefetch of Psi, K_tot, V at the owned points of one plane
    C pre_psi[RY], pre_k[RY];
    T pre_v[RY];
    auto prefetch = [&](int64_t z) {
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (out_ok[r]) {
                const int64_t q = z * g.sz + gy[r] * g.sy + gx;
                if (STAGE != 1) pre_psi[r] = ldg_c(A.Psi + q);
                if (STAGE != 1) pre_k[r] = A.K[q];
                if (A.V) pre_v[r] = __ldg(A.V + q);
            }
        }
    };

    if (ORDER == ORDER_CD) {
        // ------------------------------------------------------------------ CD: L = D
        // prologue: planes zs-1, zs, zs+1
        for (int64_t p = zs - 1; p <= zs + 1; p++) k.load_plane(p);
        cp_async_commit();
        prefetch(zs);
        cp_async_wait_all();
        __syncthreads();
        C ym[RY], y0v[RY];
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (row_in[r]) { ym[r] = k.Y(zs - 1, tx, ly0 + r); y0v[r] = k.Y(zs, tx, ly0 + r); }
        }
        for (int64_t z = zs; z < ze; z++) {
            if (z + 1 < ze && z + 2 <= g.nz - 1) k.load_plane(z + 2);
            cp_async_commit();
            C cur_psi[RY], cur_k[RY];
            T cur_v[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) { cur_psi[r] = pre_psi[r]; cur_k[r] = pre_k[r]; cur_v[r] = pre_v[r]; }
            if (z + 1 < ze) prefetch(z + 1);
            C yp[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) {
                if (!row_in[r]) continue;
                yp[r] = k.Y(z + 1, tx, ly0 + r);
                if (!out_ok[r]) continue;
                const C yc = y0v[r];
                const C y2 = cadd(yc, yc);
                const C yym = (r > 0) ? y0v[r - 1] : k.Y(z, tx, ly0 + r - 1);
                const C yyp = (r < RY - 1) ? y0v[r + 1] : k.Y(z, tx, ly0 + r + 1);
                C acc = csub(cadd(k.Y(z, tx - 1, ly0 + r), k.Y(z, tx + 1, ly0 + r)), y2);
                acc = cadd(acc, csub(cadd(yym, yyp), y2));
                acc = cadd(acc, csub(cadd(ym[r], yp[r]), y2));
                const C L = cscale(A.c.ih2, acc);
                // (fsplit) P:424-428
                T rho = (yc.x * yc.x) + (yc.y * yc.y);
                T sr = A.c.s * rho;
                T fr = (-(A.c.a * L.y)) - (sr * yc.y);
                T fi = (A.c.a * L.x) + (sr * yc.x);
                if (A.V) { fr = fr + (cur_v[r] * yc.y); fi = fi - (cur_v[r] * yc.x); }
                C F; F.x = fr; F.y = fi;
                const int64_t q = z * g.sz + gy[r] * g.sy + gx;
                const C psi = (STAGE == 1) ? yc : cur_psi[r];
                if (STAGE == 1) {
                    A.K[q] = F;
                    A.out[q] = cadd(psi, cscale(A.c.kc, F));
                } else if (STAGE == 4) {
                    C r4 = cadd(psi, cscale(A.c.kc, cadd(cur_k[r], F)));
                    A.out[q] = r4;
                    if (!(isfinite(r4.x) && isfinite(r4.y))) atomicMin(A.diverged, A.step);
                } else {
                    A.K[q] = cadd(cur_k[r], cscale(T(2), F));
                    A.out[q] = cadd(psi, cscale(A.c.kc, F));
                }
            }
#pragma unroll
            for (int r = 0; r < RY; r++) if (row_in[r]) { ym[r] = y0v[r]; y0v[r] = yp[r]; }
            cp_async_wait_all();
            __syncthreads();
        }
        return;
    } else {
        // ------------------------------------------------------------------ 2SHOC
        // prologue: planes zs-2 .. zs+2 (clipped to the grid)
        for (int64_t p = zs - 2; p <= zs + 2; p++)
            if (p >= 0 && p <= g.nz - 1) k.load_plane(p);
        cp_async_commit();
        prefetch(zs);
        cp_async_wait_all();
        __syncthreads();

        C yq0[RY], yq1[RY];             // Y center at z, z+1
        C dm[RY], d0[RY];               // D center at z-1, z
        C pxm[RY], pym[RY], px0[RY], py0[RY];   // pair sums at z-1, z
        // D(zs) over the tile (owned columns) + ring, pair sums at zs and zs-1
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (!row_in[r]) continue;
            const int ly = ly0 + r;
            yq0[r] = k.Y(zs, tx, ly);
            yq1[r] = k.Y(zs + 1, tx, ly);
            px0[r] = cadd(k.Y(zs, tx - 1, ly), k.Y(zs, tx + 1, ly));
            py0[r] = cadd(k.Y(zs, tx, ly - 1), k.Y(zs, tx, ly + 1));
            pxm[r] = cadd(k.Y(zs - 1, tx - 1, ly), k.Y(zs - 1, tx + 1, ly));
            pym[r] = cadd(k.Y(zs - 1, tx, ly - 1), k.Y(zs - 1, tx, ly + 1));
            d0[r] = k.D_any_s(zs, tx, ly);
            k.Dl(zs, tx, ly) = d0[r];
        }
        for (int t = threadIdx.x; t < Cfg::RING; t += S3_THREADS) {
            int lx, ly;
            k.ring_xy(t, lx, ly);
            k.Dl(zs, lx, ly) = k.D_any_s(zs, lx, ly);
        }
#pragma unroll
        for (int r = 0; r < RY; r++) {
            if (!row_in[r]) continue;
            const int ly = ly0 + r;
            if (zs - 1 == 0) {
                // z face: BC form with b' = (x, y, 1) = D(zs) computed above
                const int64_t qb = gy[r] * g.sy + gx;
                dm[r] = (nbnd_ok(gx, gy[r], g)) ? k.D_face_val(qb, k.Y(0, tx, ly), qb + g.sz, yq0[r], d0[r]) : cnan<T>();
            } else {
                dm[r] = k.D_any_s(zs - 1, tx, ly);
            }
        }
        __syncthreads();

        for (int64_t z = zs; z < ze; z++) {
            // (1) next Y plane (three ahead) and next output plane's Psi, K, V
            if (z + 1 < ze && z + 3 <= g.nz - 1) k.load_plane(z + 3);
            cp_async_commit();
            C cur_psi[RY], cur_k[RY];
            T cur_v[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) { cur_psi[r] = pre_psi[r]; cur_k[r] = pre_k[r]; cur_v[r] = pre_v[r]; }
            if (z + 1 < ze) prefetch(z + 1);

            // (2) D(z+1) at the owned columns, pair sums at z+1
            const int64_t zp = z + 1;
            const bool zface = (zp == g.nz - 1);
            C yq2[RY], dn[RY], px1[RY], py1[RY];
#pragma unroll
            for (int r = 0; r < RY; r++) {
                if (!row_in[r]) continue;
                const int ly = ly0 + r;
                px1[r] = cadd(k.Y(zp, tx - 1, ly), k.Y(zp, tx + 1, ly));
                const C ya = (r > 0) ? yq1[r - 1] : k.Y(zp, tx, ly - 1);
                const C yb = (r < RY - 1) ? yq1[r + 1] : k.Y(zp, tx, ly + 1);
                py1[r] = cadd(ya, yb);
                if (!zface) yq2[r] = k.Y(zp + 1, tx, ly);
                const int nb = (col_int && gy[r] <= g.ny - 2) ? 0 : 1;
                if (zface) {
                    const int64_t qb = zp * g.sz + gy[r] * g.sy + gx;
                    dn[r] = nb == 0 ? k.D_face_val(qb, yq1[r], qb - g.sz, yq0[r], d0[r]) : cnan<T>();
                } else if (nb == 0) {
                    const C y2 = cadd(yq1[r], yq1[r]);
                    C acc = csub(px1[r], y2);
                    acc = cadd(acc, csub(py1[r], y2));
                    acc = cadd(acc, csub(cadd(yq0[r], yq2[r]), y2));
                    dn[r] = cscale(A.c.ih2, acc);
                } else {
                    dn[r] = k.D_any_s(zp, tx, ly);     // x / y face column inside the tile
                }
                k.Dl(zp, tx, ly) = dn[r];
            }
            // ring D(z+1) (not needed on the last plane: a z face has no in-plane D neighbours used)
            if (!zface) {
                for (int t = threadIdx.x; t < Cfg::RING; t += S3_THREADS) {
                    int lx, ly;
                    k.ring_xy(t, lx, ly);
                    k.Dl(zp, lx, ly) = k.D_any_s(zp, lx, ly);
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
                const C pxa = (r > 0) ? px0[r - 1] : cadd(k.Y(z, tx - 1, ly - 1), k.Y(z, tx + 1, ly - 1));
                const C pxb = (r < RY - 1) ? px0[r + 1] : cadd(k.Y(z, tx - 1, ly + 1), k.Y(z, tx + 1, ly + 1));
                const C exy = csub(cadd(pxa, pxb), y4);
                const C exz = csub(cadd(pxm[r], px1[r]), y4);
                const C eyz = csub(cadd(pym[r], py1[r]), y4);
                const C E = cadd(cadd(exy, exz), eyz);
                // D terms
                const C dya = (r > 0) ? d0[r - 1] : k.Dl(z, tx, ly - 1);
                const C dyb = (r < RY - 1) ? d0[r + 1] : k.Dl(z, tx, ly + 1);
                const C sd = cadd(cadd(cadd(k.Dl(z, tx - 1, ly), k.Dl(z, tx + 1, ly)), cadd(dya, dyb)),
                                  cadd(dm[r], dn[r]));
                const C td = csub(sd, cscale(T(10), d0[r]));
                const C L = csub(cscale(A.c.c16h2, E), cscale(A.c.c112, td));
                // (fsplit) P:424-428
                T rho = (yc.x * yc.x) + (yc.y * yc.y);
                T sr = A.c.s * rho;
                T fr = (-(A.c.a * L.y)) - (sr * yc.y);
                T fi = (A.c.a * L.x) + (sr * yc.x);
                if (A.V) { fr = fr + (cur_v[r] * yc.y); fi = fi - (cur_v[r] * yc.x); }
                C F; F.x = fr; F.y = fi;
                // (RK4_GPU) P:495-519
                const int64_t q = z * g.sz + gy[r] * g.sy + gx;
                const C psi = (STAGE == 1) ? yc : cur_psi[r];
                if (STAGE == 1) {
                    A.K[q] = F;
                    A.out[q] = cadd(psi, cscale(A.c.kc, F));
                } else if (STAGE == 4) {
                    C r4 = cadd(psi, cscale(A.c.kc, cadd(cur_k[r], F)));
                    A.out[q] = r4;
                    if (!(isfinite(r4.x) && isfinite(r4.y))) atomicMin(A.diverged, A.step);
                } else {
                    A.K[q] = cadd(cur_k[r], cscale(T(2), F));
                    A.out[q] = cadd(psi, cscale(A.c.kc, F));
                }
            }
            // (4) rotate the register queues
#pragma unroll
            for (int r = 0; r < RY; r++) {
                if (!row_in[r]) continue;
                dm[r] = d0[r]; d0[r] = dn[r];
                pxm[r] = px0[r]; px0[r] = px1[r];
                pym[r] = py0[r]; py0[r] = py1[r];
                yq0[r] = yq1[r];
                if (!zface) yq1[r] = yq2[r];
            }
            cp_async_wait_all();
            __syncthreads();
        }
    }
}

template <typename T, int ORDER, int BC, int STAGE>
void launch_stream3d(const StageArgs<T> &A, cudaStream_t st) {
    constexpr int RY = 2;
    using Cfg = S3Cfg<T, ORDER, RY>;
    const int64_t mx = A.g.nx - 2, my = A.g.ny - 2, mz = A.g.nz - 2;
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

}  // namespace nlse
