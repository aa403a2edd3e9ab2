// stage3d_tma.cuh -- 3D interior stage kernel, v2: one fused HBM pass per RK4 stage
// (§8(a) rows a1-a5, a7; a9's send side in slab mode), 2.5D z-streaming with TMA.
//
// CTA = 256 threads = 8 warps owns a TX x TY = 32 x 8 column of output points (lane =
// x, warp = y) and streams it along a z chunk.  Per plane, one elected thread issues
// TMA (cp.async.bulk.tensor) loads into mbarrier-tracked shared-memory rings, P planes
// ahead of use:
//   * the stage input Y as a (TX+2H) x (TY+2H) tile (H = w: 1 CD, 2 2SHOC) -- ring of
//     NS = P+4 planes (the planes in use, P in flight, one that laggard warps may still
//     read, one free);
//   * Psi, K_tot (stages 2-4) and V at the owned points -- ring of NP = P+2 planes.
// There is no per-element address arithmetic: out-of-grid parts of a box are zero-
// filled by TMA and never used.  Compute per plane z (2SHOC):
//   1. D(z+1) = Delta_2 Y / h^2 (2SHOC step 1) at the owned point and, by
//      warps 0-2, on the one-point ring around the tile, into a shared D plane (3-plane
//      ring, so one __syncthreads per plane suffices).  D never touches HBM.  Face
//      points take the Laplacian form of the BC.
//   2. 2SHOC step 2 from D(z) in shared memory and the register queue
//      D(z-1), D(z), D(z+1), pair sums Px, Py of planes z-1, z, z+1 (the edge cross
//      term is sums of pair sums); F (fsplit) P:424-428; the RK4 stage
//      combine (RK4_GPU) P:495-519; K_tot and the stage output stored once (STG.128,
//      one warp = 512 contiguous bytes).
// Tiles whose ring touches an x/y face or lies partly outside the grid run the same
// loop with per-point face handling (EDGE = true); all others run branch-free.
// Domain-boundary outputs are written by stage_boundary (generic.cuh).  Every value
// follows the DAG of DESIGN.md §3.1, so the output is bit-identical to the oracle.
#pragma once
#include <cuda.h>
#include <type_traits>
#include "generic.cuh"

namespace nlse {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
#ifdef NLSE_MBAR_HINT
// try_wait with a suspend-time hint (ns): the thread sleeps until the phase completes or the
// hint expires instead of re-polling at the system-dependent default interval (A/B knob)
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "n"(NLSE_MBAR_HINT)
        : "memory");
}
#else
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
#endif
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// TMA load with an L2 cache policy (createpolicy): used with evict_first for the streams
// read once per stage (Psi, K_tot, V) so that they do not push out the Y halo lines the
// neighbouring tiles re-read
__device__ __forceinline__ void tma_load_3d_hint(unsigned dst, const CUtensorMap *map, int c0, int c1, int c2,
                                                 unsigned bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_inval(unsigned bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

// ------------------------------------------------------------------ configuration
// PK: Psi and K_tot are staged (stages 2-4); stage 1 streams only Y and V, and spends the
// shared memory on a deeper Y ring instead (P = TMA_P1 for stage 1)
template <typename T, int ORDER, int P, int TYV = 8, bool PK = true>
struct T3Cfg {
    static constexpr int H = (ORDER == ORDER_2SHOC) ? 2 : 1;
    // x halo of the staged tile: a TMA box must start on a 16-byte boundary, so fp32 tiles
    // carry a 2-point x halo even for CD (x0 is a multiple of 32)
    static constexpr int HX = (sizeof(T) == 4) ? 2 : H;
    static constexpr int TX = 32, TY = TYV, NT = TX * TY;   // lane = x, warp = y
    static constexpr int PX = TX + 2 * HX, PY = TY + 2 * H;
    static constexpr int CB = 2 * int(sizeof(T));                   // bytes per complex value
    // Psi/K/V prefetch depth (planes ahead); Y uses P.  A slot is refilled only once every
    // thread has finished the plane two planes back (see the barrier protocol in t3_run),
    // hence ring sizes P + 4 (Y: the planes in use reach two ahead) and PP + 2.
    // PP = 3 for fp64 measured 1.5 % faster than 2 (r01 ab1: 68.7 vs 69.8 ms/step at 1024^3,
    // 222 KB of shared memory per CTA at TY = 16); NLSE_TMA_PP64 overrides (A/B builds)
#ifndef NLSE_TMA_PP64
#define NLSE_TMA_PP64 3
#endif
#ifndef NLSE_TMA_PP32
#define NLSE_TMA_PP32 3
#endif
    static constexpr int PP = (sizeof(T) == 8) ? NLSE_TMA_PP64 : NLSE_TMA_PP32;
    static constexpr int NS = P + 4, NP = PP + 2, ND = (ORDER == ORDER_2SHOC) ? 4 : 0;
    static constexpr int DPX = TX + 2, DPY = TY + 2;
    static constexpr int up128(int b) { return (b + 127) / 128 * 128; }
    static constexpr int YBYTES = PX * PY * CB;
    static constexpr int YSLOT = up128(YBYTES);
    static constexpr int OWN_C = NT * CB, OWN_R = NT * int(sizeof(T));
    static constexpr int VOFF = PK ? 2 * OWN_C : 0;                    // V after Psi | K_tot
    static constexpr int PKVSLOT = up128(VOFF + OWN_R);                // [Psi | K_tot |] V
    static constexpr int DSLOT = up128(DPX * DPY * CB);
    static constexpr int OFF_PKV = NS * YSLOT;
    static constexpr int OFF_D = OFF_PKV + NP * PKVSLOT;
    static constexpr int OFF_BAR = OFF_D + ND * DSLOT;
    static constexpr int SMEM = OFF_BAR + (NS + NP + 2) * 8;   // + two CTA barriers
    // box dimensions (in T elements along x) of the four tensor maps
    static constexpr int BOX_Y_X = 2 * PX, BOX_Y_Y = PY;
    static constexpr int BOX_C_X = 2 * TX, BOX_R_X = TX, BOX_O_Y = TY;
};

template <typename T, int ORDER, int BC, int STAGE, int P, int TYV, bool EDGE>
struct T3Body {
    using C = cplx<T>;
    using Cfg = T3Cfg<T, ORDER, P, TYV, STAGE != 1>;
    static constexpr int H = Cfg::H, HX = Cfg::HX, TX = Cfg::TX, TY = Cfg::TY, PX = Cfg::PX, NS = Cfg::NS;
    static constexpr int NP = Cfg::NP, DPX = Cfg::DPX;

    const StageArgs<T> &A;
    unsigned char *sm;
    int x0, y0;

    __device__ __forceinline__ C *yslot(int s) const { return reinterpret_cast<C *>(sm + s * Cfg::YSLOT) + H * PX + HX; }
    __device__ __forceinline__ C *dslot(int s) const {
        return reinterpret_cast<C *>(sm + Cfg::OFF_D + s * Cfg::DSLOT) + DPX + 1;
    }
    __device__ __forceinline__ unsigned char *pkvslot(int s) const { return sm + Cfg::OFF_PKV + s * Cfg::PKVSLOT; }

    __device__ __forceinline__ T nlin(int64_t q, C yq) const {
        T rho = (yq.x * yq.x) + (yq.y * yq.y);
        T n = A.c.s * rho;
        if (A.V) n = n - __ldg(A.V + q);
        return n;
    }
    __device__ __forceinline__ int64_t gq(int p, int lx, int ly) const {
        return int64_t(p) * A.g.sz + int64_t(y0 + ly) * A.g.sy + (x0 + lx);
    }
    // Boundary D at a face point b (Laplacian form of the BC, (BCDlap) P:320-323 /
    // (BCMSDlap) P:336-344), given Y_b, and Y, D at the inward normal neighbour b'.
    __device__ __forceinline__ C D_bc(int64_t qb, C yb, int64_t qb1, C y1, C d1) const {
        if (BC == BC_L0) { C z; z.x = T(0); z.y = T(0); return z; }   // (BCL0lap) P:352-355
        const T nb = nlin(qb, yb);
        if (BC == BC_DIRICHLET) {
            const T t = A.c.inv_a * nb;
            C r; r.x = -(t * yb.x); r.y = -(t * yb.y);
            return r;
        } else {
            const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T re = T(0);
            if (!(rho1 < A.c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
            const T n1 = nlin(qb1, y1);
            const T gg = re + ((n1 - nb) * A.c.inv_a);
            return cscale(gg, yb);
        }
    }
    // 2SHOC step 1 / CD at an in-plane-interior point: (((Px-Y2)+(Py-Y2))+(Pz-Y2))*ih2
    __device__ __forceinline__ C D_int(const C *ym, const C *y0p, const C *yp) const {
        const C yc = y0p[0];
        const C y2 = cadd(yc, yc);
        C acc = csub(cadd(y0p[-1], y0p[1]), y2);
        acc = cadd(acc, csub(cadd(y0p[-PX], y0p[PX]), y2));
        acc = cadd(acc, csub(cadd(ym[0], yp[0]), y2));
        return cscale(A.c.ih2, acc);
    }
    // D(p) at local (lx, ly) of plane p with full face handling (edge tiles and z-face
    // planes).  sm_, s0, sp: Y slots of planes p-1, p, p+1 (sp unused when p is a z face);
    // dprev: D slot of plane p-1 (the inward neighbour of a z-face plane p = nz-1).
    __device__ C D_gen(int p, int smm, int s0, int sp, int dprev, int lx, int ly) const {
        const int gx = x0 + lx, gy = y0 + ly;
        const int nx = int(A.g.nx), ny = int(A.g.ny);
        C nanv; nanv.x = T(NAN); nanv.y = T(NAN);
        if (gx < 0 || gx >= nx || gy < 0 || gy >= ny) return nanv;
        const bool fx = (gx == 0 || gx == nx - 1), fy = (gy == 0 || gy == ny - 1);
        const bool fz = A.g.zf_hi && (p == int(A.g.nz) - 1);   // plane p is never the lower z face
        if (int(fx) + int(fy) + int(fz) >= 2) return nanv;      // edge / corner: never used (R-DFACE)
        const int o = ly * PX + lx;
        if (fz) {
            const int od = ly * DPX + lx;
            return D_bc(gq(p, lx, ly), yslot(s0)[o], gq(p - 1, lx, ly), yslot(smm)[o], dslot(dprev)[od]);
        }
        if (!fx && !fy) return D_int(yslot(smm) + o, yslot(s0) + o, yslot(sp) + o);
        int lx1 = lx, ly1 = ly;
        if (gx == 0) lx1 = lx + 1; else if (gx == nx - 1) lx1 = lx - 1;
        else if (gy == 0) ly1 = ly + 1; else ly1 = ly - 1;
        const int o1 = ly1 * PX + lx1;
        const C d1 = D_int(yslot(smm) + o1, yslot(s0) + o1, yslot(sp) + o1);
        return D_bc(gq(p, lx, ly), yslot(s0)[o], gq(p, lx1, ly1), yslot(s0)[o1], d1);
    }
};

// The per-run constants the inner loop uses, read once into registers.
template <typename T>
struct HotC {
    T ih2, c16h2, c112, a, s, kc;
    __device__ __forceinline__ explicit HotC(const Consts<T> &c)
        : ih2(c.ih2), c16h2(c.c16h2), c112(c.c112), a(c.a), s(c.s), kc(c.kc) {}
};

// F (fsplit) P:424-428 and the RK4 stage combine (RK4_GPU) P:495-519 at one point.
template <typename T, int STAGE>
__device__ __forceinline__ void t3_finish(const StageArgs<T> &A, const HotC<T> &hc, int64_t q, int z, int gx, int gy,
                                          cplx<T> yc, cplx<T> L, cplx<T> psi, cplx<T> kt, T v) {
    using C = cplx<T>;
    const T rho = (yc.x * yc.x) + (yc.y * yc.y);
    const T sr = hc.s * rho;
    C F = f_lin(hc.a, L, sr, yc);
    if (A.V) F = f_addv(F, v, yc);
    if (A.fp) {
        const int nx = int(A.g.nx), ny = int(A.g.ny), nz = int(A.g.nz);
        if (A.g.zf_lo && z == 1) A.fz[gy * nx + gx] = F;
        if (A.g.zf_hi && z == nz - 2) A.fz[int64_t(nx) * ny + gy * nx + gx] = F;
        if (gx == 1 || gx == nx - 2 || gy == 1 || gy == ny - 2)
            A.fp[int64_t(z) * A.per2 + shell_u(gx, gy, nx, ny)] = F;
    }
    // K_tot is re-read only by the next stage: a streaming store when the grid exceeds L2
    auto store_k = [&](C kv) { if (A.stream_hints) __stcs(A.K + q, kv); else A.K[q] = kv; };
    if (STAGE == 1) {
        store_k(F);
        store_out(A, q, z, cfma(hc.kc, F, yc));
    } else if (STAGE == 4) {
        const C r4 = cfma(hc.kc, cadd(kt, F), psi);
        store_out(A, q, z, r4);
        if (!(isfinite(r4.x) && isfinite(r4.y))) atomicMin(A.diverged, *A.step_base + A.step);
    } else {
        store_k(cfma(T(2), F, kt));
        store_out(A, q, z, cfma(hc.kc, F, psi));
    }
}

template <typename T, int ORDER, int BC, int STAGE, int P, int TYV, bool EDGE>
__device__ __forceinline__ void t3_run(const CUtensorMap *mY, const CUtensorMap *mP, const CUtensorMap *mK,
                                       const CUtensorMap *mV, const StageArgs<T> &A, unsigned char *sm, int x0,
                                       int y0, int zs, int ze) {
    using C = cplx<T>;
    using Cfg = T3Cfg<T, ORDER, P, TYV, STAGE != 1>;
    using B = T3Body<T, ORDER, BC, STAGE, P, TYV, EDGE>;
    constexpr int H = Cfg::H, TX = Cfg::TX, PX = Cfg::PX, NS = Cfg::NS, NP = Cfg::NP, DPX = Cfg::DPX;
    const B b{A, sm, x0, y0};
    const HotC<T> hc(A.c);
    const Grid &g = A.g;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int nz = int(g.nz);
    const int zmem_lo = g.zf_lo ? 0 : -g.zghost, zmem_hi = nz + (g.zf_hi ? 0 : g.zghost);
    const int zl_lo = max(zs - H, zmem_lo), zl_hi = min(ze + H - 1, zmem_hi - 1);  // Y planes loaded
    const int zbase = zs - H;
    const unsigned bar0 = smem_u32(sm + Cfg::OFF_BAR);   // NS Y barriers, then NP PKV barriers
    const unsigned pkv_bytes = (STAGE != 1 ? 2u * Cfg::OWN_C : 0u) + (A.V ? unsigned(Cfg::OWN_R) : 0u);

    auto issue_y = [&](int p) {
        if (p > zl_hi) return;                        // past the last plane: never waited on
        const int s = (p - zbase) % NS;
        const unsigned bar = bar0 + 8 * s;
        if (p < zl_lo) {                              // not in memory (below a z face): complete
            mbar_arrive(bar);                         // the phase anyway so parities stay in step
            return;
        }
        mbar_expect_tx(bar, Cfg::YBYTES);
        tma_load_3d(smem_u32(sm + s * Cfg::YSLOT), mY, 2 * (x0 - Cfg::HX), y0 - H, p + g.zghost, bar);
    };
    auto issue_pkv = [&](int p) {
        if (p >= ze || pkv_bytes == 0) return;
        const int s = (p - zs) % NP;
        const unsigned bar = bar0 + 8 * (NS + s);
        unsigned char *dst = sm + Cfg::OFF_PKV + s * Cfg::PKVSLOT;
        mbar_expect_tx(bar, pkv_bytes);
        if (A.stream_hints) {
            const uint64_t pol = policy_evict_first();
            if (STAGE != 1) {
                tma_load_3d_hint(smem_u32(dst), mP, 2 * x0, y0, p + g.zghost, bar, pol);
                tma_load_3d_hint(smem_u32(dst + Cfg::OWN_C), mK, 2 * x0, y0, p, bar, pol);
            }
            if (A.V) tma_load_3d_hint(smem_u32(dst + Cfg::VOFF), mV, x0, y0, p, bar, pol);
            return;
        }
        if (STAGE != 1) {
            tma_load_3d(smem_u32(dst), mP, 2 * x0, y0, p + g.zghost, bar);
            tma_load_3d(smem_u32(dst + Cfg::OWN_C), mK, 2 * x0, y0, p, bar);
        }
        if (A.V) tma_load_3d(smem_u32(dst + Cfg::VOFF), mV, x0, y0, p, bar);
    };
    // the TMA issuer: lane 0 of the last warp (no ring work there)
    const bool issuer = (tid == Cfg::NT - 32);
    const unsigned cbar0 = bar0 + 8 * (NS + NP);      // two CTA barriers (2SHOC)

    if (tid == 0) {
        for (int i = 0; i < NS + NP; i++) mbar_init(bar0 + 8 * i, 1);
        mbar_init(cbar0, Cfg::NT);
        mbar_init(cbar0 + 8, Cfg::NT);
        fence_proxy_async();
    }
    __syncthreads();
    if (issuer) {
        for (int p = zbase; p <= zs + H + P - 1; p++) issue_y(p);
        for (int p = zs; p <= zs + Cfg::PP - 1; p++) issue_pkv(p);
    }

    const int gx = x0 + tx, gy = y0 + ty;
    const int nx = int(g.nx), ny = int(g.ny);
    const bool out_ok = !EDGE || (gx >= 1 && gx <= nx - 2 && gy >= 1 && gy <= ny - 2);
    const int own = ty * PX + tx;                      // offset of the owned point in a Y tile
    const int downo = ty * DPX + tx;                   // ... in a D tile
    const int pown = ty * TX + tx;                     // ... in an owned-box (Psi/K/V) tile
    const int64_t qrow = int64_t(gy) * g.sy + gx;     // global offset in plane 0
    // ring duty (2SHOC): role 0 = row -1, role 1 = row TY, role 2 = columns -1 and TX; in
    // iteration j the roles go to warps j, j+1, j+2 (mod TY), so the extra D evaluations
    // rotate over all warps instead of always slowing the same three
    auto ring_pos = [&](int jj, int &rx, int &ry) -> bool {
        const int role = A.ring_rot ? (ty + Cfg::TY - (jj % Cfg::TY)) % Cfg::TY : ty;
        if (role == 0) { rx = tx; ry = -1; return true; }
        if (role == 1) { rx = tx; ry = Cfg::TY; return true; }
        if (role == 2 && tx < 2 * Cfg::TY) { rx = tx < Cfg::TY ? -1 : TX; ry = tx % Cfg::TY; return true; }
        rx = 0; ry = 0;
        return false;
    };
    int rlx = 0, rly = 0;
    bool ring = ORDER == ORDER_2SHOC && ring_pos(0, rlx, rly);
    int ro = rly * PX + rlx, rdo = rly * DPX + rlx;

    // PKV ring position of plane z
    int ps = 0; unsigned pp = 0;
    auto pkv_wait = [&]() { if (pkv_bytes) mbar_wait(bar0 + 8 * (NS + ps), pp); };
    auto pkv_next = [&]() { if (++ps == NP) { ps = 0; pp ^= 1u; } };
    auto load_own = [&](C &psi, C &kt, T &v) {
        const unsigned char *src = b.pkvslot(ps);
        if (STAGE != 1) {
            psi = reinterpret_cast<const C *>(src)[pown];
            kt = reinterpret_cast<const C *>(src + Cfg::OWN_C)[pown];
        }
        if (A.V) v = reinterpret_cast<const T *>(src + Cfg::VOFF)[pown];
    };

    if (ORDER == ORDER_CD) {
        // ------------------------------------------------------------ CD: L = D
        // slots of planes z-1, z, z+1 (relative index p - zbase: 0, 1, 2 at z = zs)
        int sm1 = 0, s0 = 1, s1 = 2;
        unsigned par1 = 0;                            // parity of plane z+1's slot use
        mbar_wait(bar0 + 8 * sm1, 0);                // (arrive-only when below a z face)
        mbar_wait(bar0 + 8 * s0, 0);
        C ym = b.yslot(sm1)[own], yc = b.yslot(s0)[own];
        for (int z = zs; z < ze; z++) {
            if (issuer) { issue_y(z + H + P); issue_pkv(z + Cfg::PP); }
            mbar_wait(bar0 + 8 * s1, par1);
            const C *Y0 = b.yslot(s0) + own;
            const C yp = b.yslot(s1)[own];
            C psi, kt; T v;
            pkv_wait();
            load_own(psi, kt, v);
            if (out_ok) {
                const C y2 = cadd(yc, yc);
                C acc = csub(cadd(Y0[-1], Y0[1]), y2);
                acc = cadd(acc, csub(cadd(Y0[-PX], Y0[PX]), y2));
                acc = cadd(acc, csub(cadd(ym, yp), y2));
                const C L = cscale(hc.ih2, acc);
                t3_finish<T, STAGE>(A, hc, int64_t(z) * g.sz + qrow, z, gx, gy, yc, L, psi, kt, v);
            }
            ym = yc; yc = yp;
            sm1 = s0; s0 = s1;
            if (++s1 == NS) { s1 = 0; par1 ^= 1u; }
            pkv_next();
            __syncthreads();
        }
        return;
    }

    // ---------------------------------------------------------------- 2SHOC
    // Barrier protocol (no __syncthreads in the loop): phase j = "every thread has written
    // D(zs + j) to shared memory"; it completes on CTA barrier cbar[j & 1] (arrival count
    // NT) as that barrier's (j >> 1)-th phase, so a waiter can never see its barrier two
    // phases ahead.  In iteration z = zs + j a thread writes D(z+1), arrives on phase j+1,
    // then waits for phase j before reading D(z) of its neighbours.  Passing phase j means
    // every thread has finished iteration z-2, so right after that wait the issuer refills
    // the Y and Psi/K/V slots of plane z-2; D(z+1) (written before the wait, when only
    // phase j-1 is known) goes into the slot of D(z-3) (4 D slots).
    // Register queues: yq = Y centre at (z, z+1, z+2), dq = D at (z-1, z, z+1), pxq / pyq =
    // pair sums at (z-1, z, z+1), stored with period 3; the z loop is unrolled by 3 so the
    // queue rotation is pure register renaming.
    int sm1 = 1, s0 = 2, s1 = 3, s2 = 4;              // Y slots of planes z-1 .. z+2 at z = zs
    unsigned par2 = 0;                                // parity of plane z+2's slot use
    mbar_wait(bar0 + 0, 0);                           // (arrive-only when below a z face)
    mbar_wait(bar0 + 8 * sm1, 0);
    mbar_wait(bar0 + 8 * s0, 0);
    mbar_wait(bar0 + 8 * s1, 0);
    int d0s = 0;                                      // D slot of plane z (4-plane ring)
    C yq[3], dq[3], pxq[3], pyq[3];
    yq[0] = b.yslot(s0)[own];
    yq[1] = b.yslot(s1)[own];
    {
        const C *Y0 = b.yslot(s0) + own, *Ym = b.yslot(sm1) + own;
        pxq[1] = cadd(Y0[-1], Y0[1]);
        pyq[1] = cadd(Y0[-PX], Y0[PX]);
        pxq[0] = cadd(Ym[-1], Ym[1]);
        pyq[0] = cadd(Ym[-PX], Ym[PX]);
        // D(zs) at the owned point and the ring (zs is never a z face)
        if (EDGE) dq[1] = b.D_gen(zs, sm1, s0, s1, 0, tx, ty);
        else dq[1] = b.D_int(Ym, Y0, b.yslot(s1) + own);
        b.dslot(d0s)[downo] = dq[1];
        if (ring) {
            C dr;
            if (EDGE) dr = b.D_gen(zs, sm1, s0, s1, 0, rlx, rly);
            else dr = b.D_int(b.yslot(sm1) + ro, b.yslot(s0) + ro, b.yslot(s1) + ro);
            b.dslot(d0s)[rdo] = dr;
        }
        // D(zs - 1) at the owned point (used only there): BC form on the lower z face,
        // else the stencil
        dq[0] = dq[1];
        if (!out_ok) {
        } else if (g.zf_lo && zs - 1 == 0) {
            dq[0] = b.D_bc(int64_t(qrow), Ym[0], int64_t(g.sz) + qrow, yq[0], dq[1]);
        } else {
            const C *Ymm = b.yslot(0) + own;
            const C y2 = cadd(Ym[0], Ym[0]);
            C acc = csub(pxq[0], y2);
            acc = cadd(acc, csub(pyq[0], y2));
            acc = cadd(acc, csub(cadd(Ymm[0], yq[0]), y2));
            dq[0] = cscale(A.c.ih2, acc);
        }
    }
    mbar_arrive(cbar0);                               // phase 0: D(zs) written
    int j = 0;                                        // z - zs

    auto body = [&](auto phase, int z) {
        constexpr int PH = decltype(phase)::value;
        constexpr int I0 = PH, I1 = (PH + 1) % 3, I2 = (PH + 2) % 3;
        const bool zf1 = g.zf_hi && (z + 1 == nz - 1);       // D(z+1) by the BC form
        const int d1s = (d0s + 1) & 3;
        if (!zf1) mbar_wait(bar0 + 8 * s2, par2);
        const C *Y0 = b.yslot(s0) + own, *Y1 = b.yslot(s1) + own;
        const C px1 = cadd(Y1[-1], Y1[1]);
        const C py1 = cadd(Y1[-PX], Y1[PX]);
        C yz2 = yq[I1], dn;
        if (EDGE) {
            dn = b.D_gen(z + 1, s0, s1, s2, d0s, tx, ty);
            if (!zf1) yz2 = b.yslot(s2)[own];
        } else if (zf1) {
            dn = b.D_bc(int64_t(z + 1) * g.sz + qrow, yq[I1], int64_t(z) * g.sz + qrow, yq[I0], dq[I1]);
        } else {
            yz2 = b.yslot(s2)[own];
            const C y2 = cadd(yq[I1], yq[I1]);
            C acc = csub(px1, y2);
            acc = cadd(acc, csub(py1, y2));
            acc = cadd(acc, csub(cadd(yq[I0], yz2), y2));
            dn = cscale(hc.ih2, acc);
        }
        b.dslot(d1s)[downo] = dn;
        ring = ring_pos(j + 1, rlx, rly);
        ro = rly * PX + rlx;
        rdo = rly * DPX + rlx;
        // on the upper z face the ring D(z+1) needs D(z) at the same ring point, written in the
        // previous iteration by the warp that had this ring role then: wait for phase j first
        if (ring && zf1) mbar_wait(cbar0 + 8 * (j & 1), unsigned(j >> 1) & 1u);
        if (ring) {
            C dr;
            if (EDGE) {
                dr = b.D_gen(z + 1, s0, s1, s2, d0s, rlx, rly);
            } else if (zf1) {
                dr = b.D_bc(b.gq(z + 1, rlx, rly), b.yslot(s1)[ro], b.gq(z, rlx, rly), b.yslot(s0)[ro],
                            b.dslot(d0s)[rdo]);
            } else {
                dr = b.D_int(b.yslot(s0) + ro, b.yslot(s1) + ro, b.yslot(s2) + ro);
            }
            b.dslot(d1s)[rdo] = dr;
        }
        mbar_arrive(cbar0 + 8 * ((j + 1) & 1));            // phase j+1: D(z+1) written
        // 2SHOC step 2, grouping of DESIGN.md §3.1: the parts that need no
        // neighbour D first, then wait for phase j (D(z) of the whole tile + ring)
        const C y2c = cadd(yq[I0], yq[I0]);
        const C y4 = cadd(y2c, y2c);                        // = 4 Y exactly (powers of two)
        const C pxa = cadd(Y0[-PX - 1], Y0[-PX + 1]);
        const C pxb = cadd(Y0[PX - 1], Y0[PX + 1]);
        const C exy = csub(cadd(pxa, pxb), y4);
        const C exz = csub(cadd(pxq[I0], px1), y4);
        const C eyz = csub(cadd(pyq[I0], py1), y4);
        const C E = cadd(cadd(exy, exz), eyz);
        mbar_wait(cbar0 + 8 * (j & 1), unsigned(j >> 1) & 1u);
        // the issuer rotates with the plane too (a warp without ring duty this plane)
        if (tx == 0 && ty == (A.ring_rot ? (j + 3) % Cfg::TY : Cfg::TY - 1)) {
            issue_y(z + H + P);
            issue_pkv(z + Cfg::PP);
        }
        C psi, kt; T v;
        pkv_wait();
        load_own(psi, kt, v);
        if (out_ok) {
            const C *Dz = b.dslot(d0s) + downo;
            const C sd = cadd(cadd(cadd(Dz[-1], Dz[1]), cadd(Dz[-DPX], Dz[DPX])), cadd(dq[I0], dn));
            const C td = cfma(T(-10), dq[I1], sd);
            const C L = cfma(hc.c16h2, E, cneg(cscale(hc.c112, td)));
            t3_finish<T, STAGE>(A, hc, int64_t(z) * g.sz + qrow, z, gx, gy, yq[I0], L, psi, kt, v);
        }
        // queue update (the slots of plane z-1 become those of plane z+2) and ring rotation
        dq[I2] = dn; pxq[I2] = px1; pyq[I2] = py1; yq[I2] = yz2;
        sm1 = s0; s0 = s1; s1 = s2;
        if (++s2 == NS) { s2 = 0; par2 ^= 1u; }
        d0s = d1s;
        pkv_next();
        ++j;
    };
    int z = zs;
    for (; z + 3 <= ze; z += 3) {
        body(std::integral_constant<int, 0>(), z);
        body(std::integral_constant<int, 1>(), z + 1);
        body(std::integral_constant<int, 2>(), z + 2);
    }
    if (z < ze) body(std::integral_constant<int, 0>(), z++);
    if (z < ze) body(std::integral_constant<int, 1>(), z++);
}

// Shared-memory access by 32-bit shared-window address (the fast path keeps one base
// register instead of re-deriving the window base of the dynamic shared memory per access).
__device__ __forceinline__ double2 lds_c(unsigned a, double) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds_c(unsigned a, float) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_r(unsigned a, double) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_r(unsigned a, float) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_c(unsigned a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void sts_c(unsigned a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
// a value the compiler must keep (it cannot re-derive it from the shared-window base)
__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
    unsigned r;
    asm volatile("mov.u32 %0, %1;\n" : "=r"(r) : "r"(x));
    return r;
}

#ifndef NLSE_PKV_EARLY
#define NLSE_PKV_EARLY 1
#endif
#ifndef NLSE_HOIST
#define NLSE_HOIST 1
#endif

// v2.3: the 2SHOC loop of t3_run for interior tiles (EDGE = false) with the per-plane
// control work cut down (ncu source counters, r01 ncus: the v2.2 loop issued ~275 warp
// instructions per point-stage, ~85 of them fp64): shared memory by 32-bit addresses from
// one base register, ring offsets by arithmetic on the role, output / K_tot pointers
// advanced by one plane stride, the rare per-plane cases (F at the b' planes, neighbour
// stores) behind one uniform test each, and the one iteration that can meet the upper z
// face peeled out of the unrolled loop.  Same rings, barrier protocol and per-point DAG as
// t3_run, so the same bits.
// EDGE = true: a tile whose owned points touch an x/y face or leave the grid, but whose ring
// has no face point (x0 + TX != nx - 1, y0 + TY != ny - 1; t3_lean_ok).  Every point takes the
// stencil D; face points then replace it by the Laplacian form of the BC ((BCDlap) P:320-323,
// (BCMSDlap) P:336-344) from Y_b, Y_b', D_b' (x faces: D_b' by a lane shuffle; y faces: the
// stencil at b' again) and V_b, V_b' prefetched one plane ahead into registers.  Edge, corner
// and out-of-grid points keep the stencil value, which no output reads (R-DFACE); only
// interior points are stored.
template <typename T, int BC, int STAGE, int P, int TYV, bool EDGE>
__device__ __forceinline__ void t3_fast(const CUtensorMap *mY, const CUtensorMap *mP, const CUtensorMap *mK,
                                        const CUtensorMap *mV, const StageArgs<T> &A, unsigned char *sm, int x0,
                                        int y0, int zs, int ze) {
    using C = cplx<T>;
    using Cfg = T3Cfg<T, ORDER_2SHOC, P, TYV, STAGE != 1>;
    using B = T3Body<T, ORDER_2SHOC, BC, STAGE, P, TYV, false>;
    constexpr int H = Cfg::H, TX = Cfg::TX, TY = Cfg::TY, PX = Cfg::PX, NS = Cfg::NS, NP = Cfg::NP, DPX = Cfg::DPX;
    constexpr int CB = Cfg::CB;
    constexpr unsigned YS = Cfg::YSLOT, DS = Cfg::DSLOT, PS = Cfg::PKVSLOT;
    static_assert((TY & (TY - 1)) == 0 && TY >= 4, "ring roles by mask need a power-of-two TY");
    const B b{A, sm, x0, y0};
    const HotC<T> hc(A.c);
    const Grid &g = A.g;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int nz = int(g.nz);
    const int zmem_lo = g.zf_lo ? 0 : -g.zghost, zmem_hi = nz + (g.zf_hi ? 0 : g.zghost);
    const int zl_lo = max(zs - H, zmem_lo), zl_hi = min(ze + H - 1, zmem_hi - 1);
    const int zbase = zs - H;
    const unsigned sb = opaque_u32(smem_u32(sm));
    const unsigned bar0 = sb + Cfg::OFF_BAR;
    const bool hasV = A.V != nullptr;
    const unsigned pkv_bytes = (STAGE != 1 ? 2u * Cfg::OWN_C : 0u) + (hasV ? unsigned(Cfg::OWN_R) : 0u);

    auto issue_y = [&](int p) {
        if (p > zl_hi) return;
        const int s = (p - zbase) % NS;
        const unsigned bar = bar0 + 8 * s;
        if (p < zl_lo) { mbar_arrive(bar); return; }
        mbar_expect_tx(bar, Cfg::YBYTES);
        tma_load_3d(sb + s * YS, mY, 2 * (x0 - Cfg::HX), y0 - H, p + g.zghost, bar);
    };
    auto issue_pkv = [&](int p) {
        if (p >= ze || pkv_bytes == 0) return;
        const int s = (p - zs) % NP;
        const unsigned bar = bar0 + 8 * (NS + s);
        const unsigned dst = sb + Cfg::OFF_PKV + s * PS;
        mbar_expect_tx(bar, pkv_bytes);
        if (STAGE != 1) {
            tma_load_3d(dst, mP, 2 * x0, y0, p + g.zghost, bar);
            tma_load_3d(dst + Cfg::OWN_C, mK, 2 * x0, y0, p, bar);
        }
        if (hasV) tma_load_3d(dst + Cfg::VOFF, mV, x0, y0, p, bar);
    };
    const unsigned cbar0 = bar0 + 8 * (NS + NP);
    if (tid == 0) {
        for (int i = 0; i < NS + NP; i++) mbar_init(bar0 + 8 * i, 1);
        mbar_init(cbar0, Cfg::NT);
        mbar_init(cbar0 + 8, Cfg::NT);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == Cfg::NT - 32) {
        for (int p = zbase; p <= zs + H + P - 1; p++) issue_y(p);
        for (int p = zs; p <= zs + Cfg::PP - 1; p++) issue_pkv(p);
    }

    const int gx = x0 + tx, gy = y0 + ty;
    const int nx = int(g.nx), ny = int(g.ny);
    // point classes (fixed along z): ok = in-plane interior (an output point); xf / yf = on
    // exactly one x / y face (D by the BC); everything else (edges, corners, outside) unused
    const bool ing = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    const bool fxp = gx == 0 || gx == nx - 1, fyp = gy == 0 || gy == ny - 1;
    const bool ok = !EDGE || (ing && !fxp && !fyp);
    const bool xf = EDGE && ing && fxp && !fyp, yf = EDGE && ing && fyp && !fxp;
    const int srcl = (gx == 0) ? tx + 1 : tx - 1;        // lane of b' for an x-face point
    const int dyb = (gy == 0) ? 1 : -1;                   // row step to b' for a y-face point
    const int64_t qb1off = xf ? (gx == 0 ? 1 : -1) : (yf ? int64_t(dyb) * g.sy : 0);
    // in-plane ring of points one in from the x/y faces: F(b') for the MSD boundary pass
    const bool shell = EDGE && ok && A.fp != nullptr && (gx == 1 || gx == nx - 2 || gy == 1 || gy == ny - 2);
    const int shell_i = shell ? shell_u(gx, gy, nx, ny) : 0;
    // shared addresses of this thread's point in Y slot 0, D slot 0 and Psi/K/V slot 0
    const unsigned ownY = sb + unsigned(((ty + H) * PX + tx + Cfg::HX) * CB);
    const unsigned ownD = sb + unsigned(Cfg::OFF_D + ((ty + 1) * DPX + tx + 1) * CB);
    const unsigned ownP = sb + unsigned(Cfg::OFF_PKV + (ty * TX + tx) * CB);
    const unsigned ownV = sb + unsigned(Cfg::OFF_PKV + Cfg::VOFF + (ty * TX + tx) * int(sizeof(T)));
    auto ldY = [&](unsigned slotB, int d) -> C { return lds_c(ownY + slotB + unsigned(d * CB), T()); };
    // ring duty: role 0 = row -1, 1 = row TY, 2 = columns -1 and TX (2 TY lanes), 3 = none;
    // role of warp ty in iteration jj = (ty - jj) mod TY with rotation, ty without
    const bool rot = A.ring_rot != 0;
    auto ring_role = [&](int jj) {
        const int r = rot ? ((ty - jj) & (TY - 1)) : ty;
        return (r > 2 || (r == 2 && tx >= 2 * TY)) ? 3 : r;
    };
    // (lx, ly) of a role's ring point -> offsets inside a Y slot / a D slot (bytes)
    auto ring_xy = [&](int role, int &rx, int &ry) {
        rx = role == 2 ? (tx < TY ? -1 : TX) : tx;
        ry = role == 0 ? -1 : (role == 1 ? TY : (tx & (TY - 1)));
    };
    // global pointers of the owned point at plane zs, advanced by one plane per iteration
    const int64_t sz = g.sz;
    const int64_t qrow = int64_t(gy) * g.sy + gx;
    C *outp = A.out + (int64_t(zs) * sz + qrow);
    C *kp = A.K + (int64_t(zs) * sz + qrow);
    const int zf1_at = g.zf_hi ? nz - 2 : INT32_MIN;              // z + 1 is the upper z face
    const bool fpz = A.fp != nullptr;
    const int fz_lo = (fpz && g.zf_lo) ? 1 : INT32_MIN, fz_hi = (fpz && g.zf_hi) ? nz - 2 : INT32_MIN;
    const bool peers = A.peer_lo != nullptr || A.peer_hi != nullptr;
    const bool xfuse = BC == BC_MSD && A.xfuse != 0;
    // face points: V at b and b' of a plane (global, read one plane ahead; planes outside
    // [0, nz) have no V and their face D is never read)
    const bool vface = (xf || yf) && hasV && BC != BC_L0;
    auto ld_vface = [&](int p, T &vb, T &vb1) {
        if (vface && p >= 0 && p < nz) {
            const int64_t q = int64_t(p) * sz + qrow;
            vb = __ldg(A.V + q);
            vb1 = __ldg(A.V + q + qb1off);
        }
    };
    // the BC form of D at a face point from Y_b, Y_b', D_b' (the same operations as
    // T3Body::D_bc, with V passed in)
    auto dface = [&](C yb, T vb, C y1, T vb1, C d1) -> C {
        if (BC == BC_L0) { C zr; zr.x = T(0); zr.y = T(0); return zr; }
        T nb = A.c.s * ((yb.x * yb.x) + (yb.y * yb.y));
        if (hasV) nb = nb - vb;
        if (BC == BC_DIRICHLET) {
            const T t = A.c.inv_a * nb;
            C r; r.x = -(t * yb.x); r.y = -(t * yb.y);
            return r;
        } else {
            const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T re = T(0);
            if (!(rho1 < A.c.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
            T n1 = A.c.s * rho1;
            if (hasV) n1 = n1 - vb1;
            const T gg = re + ((n1 - nb) * A.c.inv_a);
            return cscale(gg, yb);
        }
    };
    // stencil D at the point d bytes away from the own point, planes (m, 0, p) = Y slots
    auto dstencil = [&](unsigned yBm, unsigned yBc, unsigned yBp, int d) -> C {
        const unsigned a0 = ownY + unsigned(d);
        const C yc = lds_c(a0 + yBc, T());
        const C y2 = cadd(yc, yc);
        C acc = csub(cadd(lds_c(a0 + yBc - CB, T()), lds_c(a0 + yBc + CB, T())), y2);
        acc = cadd(acc, csub(cadd(lds_c(a0 + yBc - PX * CB, T()), lds_c(a0 + yBc + PX * CB, T())), y2));
        acc = cadd(acc, csub(cadd(lds_c(a0 + yBm, T()), lds_c(a0 + yBp, T())), y2));
        return cscale(A.c.ih2, acc);
    };
    // replace the stencil value dst (own point, centre slot yBc) by the face BC form
    auto face_fix = [&](C &dst, unsigned yBm, unsigned yBc, unsigned yBp, C yb, T vb, T vb1) {
        const unsigned full = 0xffffffffu;
        C d1x;
        d1x.x = __shfl_sync(full, dst.x, srcl);
        d1x.y = __shfl_sync(full, dst.y, srcl);
        if (xf || yf) {
            const int d = xf ? (gx == 0 ? CB : -CB) : dyb * PX * CB;
            const C y1 = lds_c(ownY + yBc + unsigned(d), T());
            const C d1 = xf ? d1x : dstencil(yBm, yBc, yBp, d);
            dst = dface(yb, vb, y1, vb1, d1);
        }
    };
    T vb_n = T(0), vb1_n = T(0);                        // V at b, b' of the plane z + 1

    // ---------------------------------------------------------------- prologue (t3_run)
    int s2 = 4;
    unsigned par2 = 0;
    unsigned yB0 = 2 * YS, yB1 = 3 * YS, yB2 = 4 * YS;          // Y slots of planes z, z+1, z+2
    mbar_wait(bar0 + 0, 0);
    mbar_wait(bar0 + 8 * 1, 0);
    mbar_wait(bar0 + 8 * 2, 0);
    mbar_wait(bar0 + 8 * 3, 0);
    unsigned dB0 = 0;                                   // D slot (byte offset) of plane z
    C yq[3], dq[3], pxq[3], pyq[3];
    dq[0].x = T(0); dq[0].y = T(0);
    {
        const unsigned yBm = 1 * YS, yBmm = 0;
        yq[0] = ldY(yB0, 0);
        yq[1] = ldY(yB1, 0);
        pxq[1] = cadd(ldY(yB0, -1), ldY(yB0, 1));
        pyq[1] = cadd(ldY(yB0, -PX), ldY(yB0, PX));
        pxq[0] = cadd(ldY(yBm, -1), ldY(yBm, 1));
        pyq[0] = cadd(ldY(yBm, -PX), ldY(yBm, PX));
        {
            const C y2 = cadd(yq[0], yq[0]);
            C acc = csub(pxq[1], y2);
            acc = cadd(acc, csub(pyq[1], y2));
            acc = cadd(acc, csub(cadd(ldY(yBm, 0), yq[1]), y2));
            dq[1] = cscale(A.c.ih2, acc);
        }
        if (EDGE) {
            T vb = T(0), vb1 = T(0);
            ld_vface(zs, vb, vb1);
            face_fix(dq[1], yBm, yB0, yB1, yq[0], vb, vb1);
            ld_vface(zs + 1, vb_n, vb1_n);
        }
        sts_c(ownD + dB0, dq[1]);
        const int role = ring_role(0);
        if (role < 3) {
            int rx, ry;
            ring_xy(role, rx, ry);
            const int oy = ((ry - ty) * PX + (rx - tx)) * CB, od = ((ry - ty) * DPX + (rx - tx)) * CB;
            const unsigned a0 = ownY + unsigned(oy);
            const C yc = lds_c(a0 + yB0, T());
            const C y2 = cadd(yc, yc);
            C acc = csub(cadd(lds_c(a0 + yB0 - CB, T()), lds_c(a0 + yB0 + CB, T())), y2);
            acc = cadd(acc, csub(cadd(lds_c(a0 + yB0 - PX * CB, T()), lds_c(a0 + yB0 + PX * CB, T())), y2));
            acc = cadd(acc, csub(cadd(lds_c(a0 + yBm, T()), lds_c(a0 + yB1, T())), y2));
            sts_c(ownD + dB0 + unsigned(od), cscale(A.c.ih2, acc));
        }
        const C ym = ldY(yBm, 0);
        if (g.zf_lo && zs - 1 == 0) {
            if (ok) dq[0] = b.D_bc(qrow, ym, sz + qrow, yq[0], dq[1]);
        } else {
            const C y2 = cadd(ym, ym);
            C acc = csub(pxq[0], y2);
            acc = cadd(acc, csub(pyq[0], y2));
            acc = cadd(acc, csub(cadd(ldY(yBmm, 0), yq[0]), y2));
            dq[0] = cscale(A.c.ih2, acc);
        }
    }
    mbar_arrive(cbar0);
    int j = 0;
    unsigned pB = 0, pp = 0;                            // Psi/K/V slot (byte offset) of plane z, parity
    int ps = 0;

    // one plane; ZF: this iteration may be the one whose z + 1 is the upper z face
    auto body = [&](auto phase, auto zfc, int z) {
        constexpr int PH = decltype(phase)::value;
        constexpr bool ZF = decltype(zfc)::value;
        constexpr int I0 = PH, I1 = (PH + 1) % 3, I2 = (PH + 2) % 3;
        const bool zf1 = ZF && (z == zf1_at);
        const unsigned dB1 = (dB0 + DS == 4 * DS) ? 0u : dB0 + DS;
        // plane z+1 has been in shared memory since the previous plane: its loads go before the
        // wait for plane z+2 (NLSE_HOIST >= 1), and with NLSE_HOIST >= 2 so do the plane-z loads
        // of the edge cross terms
#if NLSE_HOIST >= 1
        const C px1 = cadd(ldY(yB1, -1), ldY(yB1, 1));
        const C py1 = cadd(ldY(yB1, -PX), ldY(yB1, PX));
#endif
#if NLSE_HOIST >= 2
        const C pxa = cadd(ldY(yB0, -PX - 1), ldY(yB0, -PX + 1));
        const C pxb = cadd(ldY(yB0, PX - 1), ldY(yB0, PX + 1));
#endif
        if (!zf1) mbar_wait(bar0 + 8 * s2, par2);
#if NLSE_HOIST < 1
        const C px1 = cadd(ldY(yB1, -1), ldY(yB1, 1));
        const C py1 = cadd(ldY(yB1, -PX), ldY(yB1, PX));
#endif
        C yz2 = yq[I1], dn;
        if (zf1) {
            if (ok) dn = b.D_bc(int64_t(z + 1) * sz + qrow, yq[I1], int64_t(z) * sz + qrow, yq[I0], dq[I1]);
            else dn = dq[I1];                           // edge / outside: never read
        } else {
            yz2 = ldY(yB2, 0);
            const C y2 = cadd(yq[I1], yq[I1]);
            C acc = csub(px1, y2);
            acc = cadd(acc, csub(py1, y2));
            acc = cadd(acc, csub(cadd(yq[I0], yz2), y2));
            dn = cscale(hc.ih2, acc);
        }
        if (EDGE && !zf1) {
            face_fix(dn, yB0, yB1, yB2, yq[I1], vb_n, vb1_n);
            ld_vface(z + 2, vb_n, vb1_n);
        }
        sts_c(ownD + dB1, dn);
        const int role = ring_role(j + 1);
        if (role < 3) {
            int rx, ry;
            ring_xy(role, rx, ry);
            const int oy = ((ry - ty) * PX + (rx - tx)) * CB, od = ((ry - ty) * DPX + (rx - tx)) * CB;
            const unsigned a0 = ownY + unsigned(oy);
            C dr;
            if (zf1) {
                // D(z) at this ring point was written by the warp that had this role in the
                // previous iteration: wait for phase j first
                mbar_wait(cbar0 + 8 * (j & 1), unsigned(j >> 1) & 1u);
                const int rgx = x0 + rx, rgy = y0 + ry;
                if (!EDGE || (rgx >= 1 && rgx <= nx - 2 && rgy >= 1 && rgy <= ny - 2))
                    dr = b.D_bc(b.gq(z + 1, rx, ry), lds_c(a0 + yB1, T()), b.gq(z, rx, ry), lds_c(a0 + yB0, T()),
                                lds_c(ownD + dB0 + unsigned(od), T()));
                else
                    dr = lds_c(ownD + dB0 + unsigned(od), T());   // edge / outside: never read
            } else {
                const C yc = lds_c(a0 + yB1, T());
                const C y2 = cadd(yc, yc);
                C acc = csub(cadd(lds_c(a0 + yB1 - CB, T()), lds_c(a0 + yB1 + CB, T())), y2);
                acc = cadd(acc, csub(cadd(lds_c(a0 + yB1 - PX * CB, T()), lds_c(a0 + yB1 + PX * CB, T())), y2));
                acc = cadd(acc, csub(cadd(lds_c(a0 + yB0, T()), lds_c(a0 + yB2, T())), y2));
                dr = cscale(hc.ih2, acc);
            }
            sts_c(ownD + dB1 + unsigned(od), dr);
        }
        mbar_arrive(cbar0 + 8 * ((j + 1) & 1));
        const C y2c = cadd(yq[I0], yq[I0]);
        const C y4 = cadd(y2c, y2c);
#if NLSE_HOIST < 2
        const C pxa = cadd(ldY(yB0, -PX - 1), ldY(yB0, -PX + 1));
        const C pxb = cadd(ldY(yB0, PX - 1), ldY(yB0, PX + 1));
#endif
        const C exy = csub(cadd(pxa, pxb), y4);
        const C exz = csub(cadd(pxq[I0], px1), y4);
        const C eyz = csub(cadd(pyq[I0], py1), y4);
        const C E = cadd(cadd(exy, exz), eyz);
        C psi, kt; T v;
#if NLSE_PKV_EARLY
        // Psi / K_tot / V of plane z do not depend on the CTA barrier: load them before it, so
        // their shared-memory latency overlaps the barrier wait (the slot of plane z is refilled
        // only two planes later, after every thread has passed the barrier of plane z + 2)
        if (pkv_bytes) mbar_wait(bar0 + 8 * (NS + ps), pp);
        if (STAGE != 1) {
            psi = lds_c(ownP + pB, T());
            kt = lds_c(ownP + pB + Cfg::OWN_C, T());
        }
        if (hasV) v = lds_r(ownV + pB, T());
#endif
        mbar_wait(cbar0 + 8 * (j & 1), unsigned(j >> 1) & 1u);
        if (tx == 0 && ty == (rot ? ((j + 3) & (TY - 1)) : TY - 1)) {
            issue_y(z + H + P);
            issue_pkv(z + Cfg::PP);
        }
#if !NLSE_PKV_EARLY
        if (pkv_bytes) mbar_wait(bar0 + 8 * (NS + ps), pp);
        if (STAGE != 1) {
            psi = lds_c(ownP + pB, T());
            kt = lds_c(ownP + pB + Cfg::OWN_C, T());
        }
        if (hasV) v = lds_r(ownV + pB, T());
#endif
        const unsigned ad = ownD + dB0;
        const C sd = cadd(cadd(cadd(lds_c(ad - CB, T()), lds_c(ad + CB, T())),
                               cadd(lds_c(ad - DPX * CB, T()), lds_c(ad + DPX * CB, T()))),
                          cadd(dq[I0], dn));
        const C td = cfma(T(-10), dq[I1], sd);
        const C L = cfma(hc.c16h2, E, cneg(cscale(hc.c112, td)));
        // F (fsplit) P:424-428 and the stage combine (RK4_GPU) P:495-519 (as t3_finish)
        const C yc = yq[I0];
        const T rho = (yc.x * yc.x) + (yc.y * yc.y);
        const T sr = hc.s * rho;
        C F = f_lin(hc.a, L, sr, yc);
        if (hasV) F = f_addv(F, v, yc);
        if (shell) A.fp[int64_t(z) * A.per2 + shell_i] = F;
        if (ok && (z == fz_lo || z == fz_hi)) {
            if (z == fz_lo) A.fz[gy * nx + gx] = F;
            if (z == fz_hi) A.fz[int64_t(nx) * g.ny + gy * nx + gx] = F;
        }
        if (EDGE && xfuse) {
            // x-face points of this plane, (msd) P:331-335: F_b = i Im(F_b'/Y_b') Y_b with b' the
            // neighbouring lane (same arithmetic as stage_boundary_msd_fb)
            const unsigned full = 0xffffffffu;
            C f1, y1;
            f1.x = __shfl_sync(full, F.x, srcl);
            f1.y = __shfl_sync(full, F.y, srcl);
            y1.x = __shfl_sync(full, yc.x, srcl);
            y1.y = __shfl_sync(full, yc.y, srcl);
            if (xf) {
                const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
                T m = T(0);
                if (!(rho1 < A.c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
                F.x = -(m * yc.y);
                F.y = m * yc.x;
            }
        }
        C o;
        const bool okw = ok || (EDGE && xfuse && xf);   // points this thread writes
        if (STAGE == 1) {
            if (okw) *kp = F;
            o = cfma(hc.kc, F, yc);
        } else if (STAGE == 4) {
            o = cfma(hc.kc, cadd(kt, F), psi);
        } else {
            if (okw) *kp = cfma(T(2), F, kt);
            o = cfma(hc.kc, F, psi);
        }
        if (okw) *outp = o;
        if (peers && okw) {                                    // slab mode: the neighbours' ghost planes
            const int64_t q = outp - A.out;
            if (A.peer_lo && z < A.wsend) A.peer_lo[q] = o;
            if (A.peer_hi && z >= nz - A.wsend) A.peer_hi[q] = o;
        }
        if (STAGE == 4 && okw && !(isfinite(o.x) && isfinite(o.y))) atomicMin(A.diverged, *A.step_base + A.step);
        outp += sz;
        kp += sz;
        // queue update and slot rotation
        dq[I2] = dn; pxq[I2] = px1; pyq[I2] = py1; yq[I2] = yz2;
        yB0 = yB1; yB1 = yB2;
        if (++s2 == NS) { s2 = 0; par2 ^= 1u; }
        yB2 = s2 * YS;
        dB0 = dB1;
        if (++ps == NP) { ps = 0; pp ^= 1u; }
        pB = ps * PS;
        ++j;
    };
    using F0 = std::false_type;
    using F1 = std::true_type;
    using P0 = std::integral_constant<int, 0>;
    using P1 = std::integral_constant<int, 1>;
    using P2 = std::integral_constant<int, 2>;
    int z = zs;
    const int zlast = ze - 1;                           // the only iteration that can meet the upper face
    for (; z + 3 <= zlast; z += 3) {
        body(P0(), F0(), z);
        body(P1(), F0(), z + 1);
        body(P2(), F0(), z + 2);
    }
    const int rem = zlast - z;                          // 0, 1 or 2 iterations before zlast
    if (rem == 0) {
        body(P0(), F1(), z);
    } else if (rem == 1) {
        body(P0(), F0(), z);
        body(P1(), F1(), z + 1);
    } else {
        body(P0(), F0(), z);
        body(P1(), F0(), z + 1);
        body(P2(), F1(), z + 2);
    }
}

// One CTA per work item (tile, z chunk); blockIdx.x enumerates the items z-chunk-major,
// then tile row, then tile column, so the CTAs resident at any time cover whole bands of
// consecutive tiles of one z chunk (their shared halo rows and columns are L2 hits).
// Measured alternatives (r01g-j: a persistent grid drawing items from a counter, banded
// tile orders) were not faster.
// Resident CTAs per SM the register allocation is sized for (__launch_bounds__): fp64 TY=16 one
// CTA (<= 128 registers); fp32 TY=16 NLSE_F32_MINB CTAs (2: <= 64 registers, which spills the
// 2SHOC loop; 1: <= 128 registers, no spills, half the resident warps).
#ifndef NLSE_F32_MINB
#define NLSE_F32_MINB 1
#endif
#ifndef NLSE_F32_MINB8
#define NLSE_F32_MINB8 3
#endif
#ifndef NLSE_F32_MINB8_DIR
#define NLSE_F32_MINB8_DIR NLSE_F32_MINB8
#endif
template <typename T, int TYV, int BC = BC_MSD>
constexpr int t3_min_blocks() {
    return TYV == 8 ? (sizeof(T) == 8 ? 2 : (BC == BC_DIRICHLET ? NLSE_F32_MINB8_DIR : NLSE_F32_MINB8))
                    : (sizeof(T) == 8 ? 1 : NLSE_F32_MINB);
}
template <typename T, int ORDER, int BC, int STAGE, int P, int TYV>
__global__ void __launch_bounds__(32 * TYV, t3_min_blocks<T, TYV, BC>())
stage3d_tma(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mP,
            const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV,
            const __grid_constant__ StageArgs<T> A, int zchunk, int ntx, int nty, int force_edge, int band) {
    using Cfg = T3Cfg<T, ORDER, P, TYV, STAGE != 1>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int ntiles = ntx * nty;
    const int w = blockIdx.x;
    const int c = w / ntiles, t = w - c * ntiles;
    // tile order within a z chunk: row-major (band = 0), or bands of `band` tile rows walked column
    // by column, so that the tiles sharing a y halo start within a few CTAs of each other (their
    // halo planes are then L2 hits; row-major puts a tile's y neighbour a whole tile row, ~30 planes
    // of progress, ahead)
    int tx_, ty_;
    if (band > 1) {
        const int b = t / (band * ntx), u = t - b * band * ntx;
        const int rows = min(band, nty - b * band);
        tx_ = u / rows;
        ty_ = b * band + (u - tx_ * rows);
    } else {
        tx_ = t % ntx;
        ty_ = t / ntx;
    }
    const int x0 = tx_ * Cfg::TX, y0 = ty_ * Cfg::TY;
    const int nz = int(A.g.nz);
    const int zlo = A.g.zf_lo ? 1 : 0, zhi = nz - (A.g.zf_hi ? 1 : 0);
    const int zs = zlo + c * zchunk;
    const int ze = min(zs + zchunk, zhi);
    if (zs >= ze) return;
    const int nx = int(A.g.nx), ny = int(A.g.ny);
    // every owned and ring point in-plane interior -> branch-free path
    const bool edge = force_edge || !(x0 >= 2 && x0 + Cfg::TX <= nx - 2 && y0 >= 2 && y0 + Cfg::TY <= ny - 2);
    // edge tiles without a face point on their ring run the lean loop with face handling;
    // force_edge == 2 keeps them on the per-point face path (measurement / tests)
    // (x0 == nx - 1: the x-face point's b' is on the previous tile, out of shuffle reach)
    const bool lean_edge = force_edge != 2 && x0 + Cfg::TX != nx - 1 && y0 + Cfg::TY != ny - 1 && x0 != nx - 1;
    if constexpr (ORDER == ORDER_2SHOC) {
        if (!edge) t3_fast<T, BC, STAGE, P, TYV, false>(&mY, &mP, &mK, &mV, A, smem_raw, x0, y0, zs, ze);
        else if (lean_edge) t3_fast<T, BC, STAGE, P, TYV, true>(&mY, &mP, &mK, &mV, A, smem_raw, x0, y0, zs, ze);
        else t3_run<T, ORDER, BC, STAGE, P, TYV, true>(&mY, &mP, &mK, &mV, A, smem_raw, x0, y0, zs, ze);
    } else {
        if (edge) t3_run<T, ORDER, BC, STAGE, P, TYV, true>(&mY, &mP, &mK, &mV, A, smem_raw, x0, y0, zs, ze);
        else t3_run<T, ORDER, BC, STAGE, P, TYV, false>(&mY, &mP, &mK, &mV, A, smem_raw, x0, y0, zs, ze);
    }
}

}  // namespace nlse
