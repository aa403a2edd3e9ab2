// strip2d.cuh -- 2D stage kernel, round 2 (§8(a) rows a1-a7 for 2D grids, boundary included):
// one WARP (one warp per CTA) streams a 32-column strip along y, with no CTA barrier; the only
// shared memory is the warp's own cp.async staging ring.
//
// The shared-tile kernel of round 1 (tile2d.cuh: load tile -> barrier -> D tile -> barrier ->
// combine, one tile per CTA, plus a boundary kernel) was latency-bound on configs[2] (1024^2
// fp64 + V: 23 us per stage, r02s).  (That grid's 72 MB of state does not make it L2-bound: on
// B200 the L2 delivers about the HBM rate at that size, profiles/r02_l2_bandwidth.json.)
// Here the 2.5D z-streaming design of stage3d_tma is taken one dimension down, where a "plane"
// is one row of a strip, so that a warp alone holds everything it needs:
//   * lane l holds column gx = xs + l, xs = 1 + s W - H (H = w: 1 CD, 2 2SHOC); lanes
//     [H, H + W) (W = 32 - 2H) are the strip's interior output columns, the lanes around them its
//     halo; x-neighbours come from warp shuffles (Y(x +- 1) for the x pair sums and D(x +- 1)
//     for 2SHOC step 2), y-neighbours from register queues along y (Y, D and the x pair sums Px
//     of rows y - 1, y, y + 1), exactly as the z queues of the 3D kernel;
//   * the loads of a row (Y two rows ahead, Psi / K_tot / V of the row) are staged S2_NSL - 1 rows
//     ahead by cp.async into a per-warp shared-memory ring (each lane its own column);
//   * the two edge strips (x faces: the face arithmetic makes their rows ~1.6x as long) run in
//     row chunks 8x shorter than the interior strips, so the single wave does not wait for them;
//   * per row y: D(y + 1) (2SHOC step 1, (2d2shocs1) P:202-210; faces: the Laplacian form of
//     the BC, (BCDlap) P:320-323, (BCMSDlap) P:336-344, (BCL0lap) P:352-355), step 2 at row y
//     ((2d2shocs2) P:214-228), F (fsplit) P:424-428 and the RK4 stage combine (RK4_GPU)
//     P:495-519; CD: L = D;
//   * the domain boundary is finished in the same pass: the x-face points x = 0 / nx - 1 by the
//     lane next to the strip's first / last output lane (F(b'), Y(b') by a shuffle from the
//     inward lane), the y-face rows 0 / ny - 1 after the row loop from F(b'), Y(b') of rows 1 /
//     ny - 2 kept in registers (corners take b' = (clamp x, clamp y), R-MSD-NBR):
//     (BCDdt) P:315-318, (msd) P:331-335, (BCL0dt) P:347-350.  One launch per stage.
// y-slab mode (§8(e)): rows [-zghost, 0) and [ny, ny + zghost) are the neighbours' ghost rows,
// y faces only where the slab holds them, outputs of the first / last wsend rows also go to the
// neighbours (store_out).  Every value follows the DAG of DESIGN.md §3.1 (bitwise = oracle).
#pragma once
#include <algorithm>
#include <utility>
#include "generic.cuh"

namespace nlse {

#ifndef NLSE_S2_WARPS
#define NLSE_S2_WARPS 1
#endif
// warps per CTA: 1 keeps every loop bound and branch of the row loop derived from blockIdx (provably
// warp-uniform), so the shuffles compile without the divergent-collective fallback (WARPSYNC loops)
constexpr int S2_WARPS = NLSE_S2_WARPS, S2_NT = 32 * S2_WARPS;
// the unroll factor of the row loop = the period of the register queues (3: Y, D and the pair sums
// of rows y - 1, y, y + 1), so that the queue rotation is register renaming
constexpr int S2_PF = 3;

template <typename T>
__device__ __forceinline__ cplx<T> s2_up(cplx<T> v) {      // the value of lane - 1
    cplx<T> r;
    r.x = __shfl_up_sync(0xffffffffu, v.x, 1);
    r.y = __shfl_up_sync(0xffffffffu, v.y, 1);
    return r;
}
template <typename T>
__device__ __forceinline__ cplx<T> s2_dn(cplx<T> v) {      // the value of lane + 1
    cplx<T> r;
    r.x = __shfl_down_sync(0xffffffffu, v.x, 1);
    r.y = __shfl_down_sync(0xffffffffu, v.y, 1);
    return r;
}

// Rows [ys, ye) in order, the loop unrolled by S2_PF: row r runs with phase (r - ys) % S2_PF as a
// compile-time index (queue positions).  One copy of the body per phase (the kernel's hot code must
// stay within the instruction cache: "no instruction" stalls dominated a version with 14 copies).
template <typename B>
__device__ __forceinline__ void s2_rows(int ys, int ye, B &body) {
    static_assert(S2_PF == 3, "phases");
    for (int y = ys; y < ye; y += 3) {
        body(std::integral_constant<int, 0>(), y);
        if (y + 1 >= ye) break;
        body(std::integral_constant<int, 1>(), y + 1);
        if (y + 2 >= ye) break;
        body(std::integral_constant<int, 2>(), y + 2);
    }
}

// The loads of row r: Y(r + H) (the new stencil row), V(r + H - 1) (2SHOC: the row of the D
// computed at r; CD: row r), Psi(r), K_tot(r) -- staged by asynchronous copies (cp.async, global ->
// shared without registers) into a per-warp shared-memory ring of S2_NSL row slots, S2_NSL - 1 rows
// ahead of the row computed: deep memory-level parallelism at no register cost (the 2D grids are
// L2-scale, so the latency to cover is that of L2 hits and misses, not DRAM streaming alone).
#ifndef NLSE_S2_NSL
#define NLSE_S2_NSL 6
#endif
constexpr int S2_NSL = NLSE_S2_NSL;
template <typename T>
struct S2Slot {
    static constexpr int CB = 2 * int(sizeof(T));
    static constexpr int YOFF = 0, POFF = 32 * CB, KOFF = 64 * CB, VOFF = 96 * CB;
    static constexpr int BYTES = 96 * CB + 32 * int(sizeof(T));
    static constexpr int SMEM = S2_WARPS * S2_NSL * BYTES;      // per CTA
};
template <typename T>
struct S2In {
    cplx<T> y, psi, k;
    T v;
};
template <int BYTES>
__device__ __forceinline__ void s2_cp(unsigned sdst, const void *gsrc) {
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sdst), "l"(gsrc), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void s2_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void s2_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// One warp, strip s, rows [ys, ye).  EDGE: the strip holds an x face (strips 0 and nstrips - 1).
template <typename T, int ORDER, int BC, int STAGE, bool EDGE>
__device__ __forceinline__ void s2_strip(const StageArgs<T> &A, int s, int ys, int ye) {
    using C = cplx<T>;
    constexpr int H = (ORDER == ORDER_2SHOC) ? 2 : 1;
    constexpr int W = 32 - 2 * H;
    const int lane = threadIdx.x & 31;
    const Grid &g = A.g;
    const int nx = int(g.nx), ny = int(g.ny);
    const bool flo = g.zf_lo != 0, fhi = g.zf_hi != 0;
    const int ymlo = flo ? 0 : -g.zghost, ymhi = fhi ? ny : ny + g.zghost;   // rows in memory
    const int sy = int(g.sy);                                  // 32-bit offsets (checked at launch)

    const int gx = 1 + s * W - H + lane;
    // lanes outside the grid read column 0 / nx - 1 instead (values no output uses)
    const int gxc = gx < 0 ? 0 : (gx > nx - 1 ? nx - 1 : gx);
    const bool xin = lane >= H && lane < H + W && (!EDGE || gx <= nx - 2);   // interior output column
    const bool xf_lo = EDGE && gx == 0;                                        // (strip 0, lane H - 1)
    const bool xf_hi = EDGE && gx == nx - 1 && s == (nx - 3) / W;              // owner: strip of nx - 2
    const bool xf = xf_lo || xf_hi;
    const bool own = xin || xf;                                                // this lane writes its column
    const bool hasV = A.V != nullptr;
    const bool peers = A.peer_lo != nullptr || A.peer_hi != nullptr;
    const Consts<T> &hc = A.c;             // (constant-bank operands, not registers)
    const int srcl = xf_lo ? lane + 1 : (lane > 0 ? lane - 1 : 0);   // lane of b' for an x-face lane

    // addresses: the parameter-space base pointer + a 32-bit element offset (no pointer registers)
    auto ldY = [&](int r) -> C { return __ldg(A.Y + (gxc + (r < ymlo ? ymlo : (r < ymhi ? r : ymhi - 1)) * sy)); };
    auto ldV = [&](int r) -> T { return hasV ? __ldg(A.V + (gxc + (r < ny ? r : ny - 1) * sy)) : T(0); };
    // Y(b') of an x-face lane from the x-neighbour shuffles (lane + 1 at x = 0, lane - 1 at nx - 1);
    // other values at b' by one shuffle from srcl
    auto pick = [&](C up, C dn) -> C { return xf_lo ? dn : up; };
    auto fromb1 = [&](C v) -> C {
        C r;
        r.x = __shfl_sync(0xffffffffu, v.x, srcl);
        r.y = __shfl_sync(0xffffffffu, v.y, srcl);
        return r;
    };
    // the Laplacian form of the BC at a face point b from Y_b, V_b and Y, V, D at b' (as dface in
    // stage3d_tma.cuh / PointEval::D_face)
    auto dface = [&](C yb, T vb, C y1, T vb1, C d1) -> C {
        if (BC == BC_L0) { C zr; zr.x = T(0); zr.y = T(0); return zr; }
        T nb = hc.s * ((yb.x * yb.x) + (yb.y * yb.y));
        if (hasV) nb = nb - vb;
        if (BC == BC_DIRICHLET) {
            const T t = hc.inv_a * nb;
            C r; r.x = -(t * yb.x); r.y = -(t * yb.y);
            return r;
        } else {
            const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T re = T(0);
            if (!(rho1 < hc.eps2)) re = ((d1.x * y1.x) + (d1.y * y1.y)) / rho1;
            T n1 = hc.s * rho1;
            if (hasV) n1 = n1 - vb1;
            const T gg = re + ((n1 - nb) * hc.inv_a);
            return cscale(gg, yb);
        }
    };
    // F at a boundary point b: (BCDdt) P:315-318, (msd) P:331-335 from F, Y at b', (BCL0dt)
    // P:347-350 as (fsplit) with Lap Psi_b = 0 (as PointEval::F_bnd)
    auto fbnd = [&](C yb, T vb, C f1, C y1) -> C {
        C f;
        if (BC == BC_DIRICHLET) { f.x = T(0); f.y = T(0); return f; }
        if (BC == BC_L0) {
            C zero; zero.x = T(0); zero.y = T(0);
            const T sr = hc.s * ((yb.x * yb.x) + (yb.y * yb.y));
            f = f_lin(hc.a, zero, sr, yb);
            if (hasV) f = f_addv(f, vb, yb);
            return f;
        }
        const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
        T m = T(0);
        if (!(rho1 < hc.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
        f.x = -(m * yb.y);
        f.y = m * yb.x;
        return f;
    };
    // interior F (fsplit) P:424-428
    auto fint = [&](C yc, C L, T v) -> C {
        const T sr = hc.s * ((yc.x * yc.x) + (yc.y * yc.y));
        C F = f_lin(hc.a, L, sr, yc);
        if (hasV) F = f_addv(F, v, yc);
        return F;
    };
    // RK4 stage combine (RK4_GPU) P:495-519 at local row r (as rk_combine, Psi / K_tot given);
    // stores predicated on `w` (no branch around them)
    auto combine = [&](int r, C F, C yc, C psi, C kt, bool w) {
        const int o_ = gxc + r * sy;
        C o;
        if (STAGE == 1) {
            if (w) A.K[o_] = F;
            o = cfma(hc.kc, F, yc);
        } else if (STAGE == 4) {
            o = cfma(hc.kc, cadd(kt, F), psi);
        } else {
            const C kn = cfma(T(2), F, kt);
            if (w) A.K[o_] = kn;
            o = cfma(hc.kc, F, psi);
        }
        if (w) A.out[o_] = o;
        if (peers) {                                      // slab mode: the neighbours' ghost rows
            if (w && A.peer_lo && r < A.wsend) A.peer_lo[o_] = o;
            if (w && A.peer_hi && r >= ny - A.wsend) A.peer_hi[o_] = o;
        }
        if (STAGE == 4 && w && !(isfinite(o.x) && isfinite(o.y))) atomicMin(A.diverged, *A.step_base + A.step);
    };
    // a y-face row rf (0 or ny - 1): F_b from F, Y at b' = (clamp x, inward row) = (f1, y1)
    auto face_row = [&](int rf, C yb, T vb, C f1, C y1) {
        if (!own) return;
        C psi = yb, kt = yb;
        if (STAGE != 1) { psi = A.Psi[gxc + rf * sy]; kt = A.K[gxc + rf * sy]; }
        combine(rf, fbnd(yb, vb, f1, y1), yb, psi, kt, true);
    };

    // F, Y at b' of the y-face rows (row 1 -> row 0, row ny - 2 -> row ny - 1), kept from the row
    // iterations; the face rows themselves are finished after the loop (cold code out of it)
    C lo_f1, lo_y1, hi_f1, hi_y1;
    auto finish_faces = [&]() {
        if (flo && ys == 1) face_row(0, ldY(0), ldV(0), lo_f1, lo_y1);
        if (fhi && ye == ny - 1) face_row(ny - 1, ldY(ny - 1), ldV(ny - 1), hi_f1, hi_y1);
    };

    // the warp's shared-memory ring (S2Slot): row r in slot (r - ys) % S2_NSL; each lane copies
    // and reads back only its own column, so no synchronisation beyond cp.async.wait_group
    using SL = S2Slot<T>;
    extern __shared__ __align__(16) unsigned char s2_smem[];
    unsigned char *wring = s2_smem + (threadIdx.x >> 5) * (S2_NSL * SL::BYTES);
    const unsigned wbase = static_cast<unsigned>(__cvta_generic_to_shared(wring));
    const unsigned lc = unsigned(lane * SL::CB), lr = unsigned(lane * int(sizeof(T)));
    auto issue = [&](int r, int slot) {                   // one commit group per row (maybe empty)
        if (r < ye) {
            const unsigned d = wbase + unsigned(slot * SL::BYTES);
            const int ry = r + H;
            s2_cp<SL::CB>(d + SL::YOFF + lc, A.Y + (gxc + (ry < ymhi ? ry : ymhi - 1) * sy));
            if (hasV) {
                const int rv = r + H - 1;
                s2_cp<int(sizeof(T))>(d + SL::VOFF + lr, A.V + (gxc + (rv < ny ? rv : ny - 1) * sy));
            }
            if (STAGE != 1 && own) {
                s2_cp<SL::CB>(d + SL::POFF + lc, A.Psi + (gxc + r * sy));
                s2_cp<SL::CB>(d + SL::KOFF + lc, A.K + (gxc + r * sy));
            }
        }
        s2_commit();
    };
#pragma unroll
    for (int i = 0; i < S2_NSL - 1; i++) issue(ys + i, i);
    int slot = 0;
    // the inputs of row y (its copies have landed once at most S2_NSL - 2 younger groups are
    // pending), then the copies of row y + S2_NSL - 1 into the slot row y - 1 used
    auto fetch = [&](int y) -> S2In<T> {
        s2_wait<S2_NSL - 2>();
        const unsigned char *p = wring + slot * SL::BYTES;
        S2In<T> c;
        c.y = reinterpret_cast<const C *>(p + SL::YOFF)[lane];
        c.v = hasV ? reinterpret_cast<const T *>(p + SL::VOFF)[lane] : T(0);
        if (STAGE != 1) {
            c.psi = reinterpret_cast<const C *>(p + SL::POFF)[lane];
            c.k = reinterpret_cast<const C *>(p + SL::KOFF)[lane];
        }
        issue(y + S2_NSL - 1, slot == 0 ? S2_NSL - 1 : slot - 1);
        slot = (slot + 1 == S2_NSL) ? 0 : slot + 1;
        return c;
    };

    if constexpr (ORDER == ORDER_CD) {
        // ---------------------------------------------------------------- CD: L = D
        // queue yq: Y(y-1), Y(y), Y(y+1) at positions P, P+1, P+2 (mod 3) in phase P
        C yq[3];
        yq[0] = ldY(ys - 1);
        yq[1] = ldY(ys);
        auto body = [&](auto ph, int y) {
            constexpr int P = decltype(ph)::value, I0 = P, I1 = (P + 1) % 3, I2 = (P + 2) % 3;
            const S2In<T> cur = fetch(y);
            const C ym = yq[I0], yc = yq[I1], yp = cur.y;
            const C yl = s2_up<T>(yc), yr = s2_dn<T>(yc);
            const C y2 = cadd(yc, yc);
            C acc = csub(cadd(yl, yr), y2);
            acc = cadd(acc, csub(cadd(ym, yp), y2));
            const C L = cscale(hc.ih2, acc);
            const C F = fint(yc, L, cur.v);
            C Fo = F, f1 = F, y1 = yc;
            if (EDGE) {
                // F, Y at b': own values on interior columns, the inward lane's on x faces
                const C fsh = fromb1(F), ysh = pick(yl, yr);
                if (xf) { Fo = fbnd(yc, cur.v, fsh, ysh); f1 = fsh; y1 = ysh; }
            }
            combine(y, Fo, yc, cur.psi, cur.k, own);
            if (flo && y == 1) { lo_f1 = f1; lo_y1 = y1; }       // the y-face rows: after the loop
            if (fhi && y == ny - 2) { hi_f1 = f1; hi_y1 = y1; }
            yq[I2] = yp;
        };
        s2_rows(ys, ye, body);
        finish_faces();
        return;
    }

    // -------------------------------------------------------------------- 2SHOC
    // queues (phase P: rows y-1, y, y+1 at positions P, P+1, P+2 mod 3): yq = Y, pq = x pair sums
    // Px, dq = D, vq = V, bq = Y(b') of x-face lanes
    C yq[3], pq[3], dq[3], bq[3];
    T vq[3];
    const C ymm = ldY(ys - 2);
    yq[0] = ldY(ys - 1);
    yq[1] = ldY(ys);
    yq[2] = ldY(ys + 1);
    vq[1] = ldV(ys);
    {
        const C ylm = s2_up<T>(yq[0]), yrm = s2_dn<T>(yq[0]);
        const C ylc = s2_up<T>(yq[1]), yrc = s2_dn<T>(yq[1]);
        pq[0] = cadd(ylm, yrm);
        pq[1] = cadd(ylc, yrc);
        bq[1] = pick(ylc, yrc);
        // D(ys): ys is never a y face; x faces by the BC form from the inward lane
        {
            const C y2 = cadd(yq[1], yq[1]);
            C acc = csub(pq[1], y2);
            acc = cadd(acc, csub(cadd(yq[0], yq[2]), y2));
            dq[1] = cscale(hc.ih2, acc);
            if (EDGE) {
                const C dsh = fromb1(dq[1]);
                const T vsh = __shfl_sync(0xffffffffu, vq[1], srcl);
                if (xf) dq[1] = dface(yq[1], vq[1], bq[1], vsh, dsh);
            }
        }
        // D(ys - 1): the lower y face (b' = (x, 1): own lane) or the stencil (ghost rows included);
        // its x-face values are never read
        if (flo && ys == 1) {
            dq[0] = dface(yq[0], ldV(0), yq[1], vq[1], dq[1]);
        } else {
            const C y2 = cadd(yq[0], yq[0]);
            C acc = csub(pq[0], y2);
            acc = cadd(acc, csub(cadd(ymm, yq[1]), y2));
            dq[0] = cscale(hc.ih2, acc);
        }
    }
    auto body = [&](auto ph, int y) {
        constexpr int P = decltype(ph)::value, I0 = P, I1 = (P + 1) % 3, I2 = (P + 2) % 3;
        const S2In<T> cur = fetch(y);
        const C ym = yq[I0], yc = yq[I1], yp = yq[I2];
        const T vc = vq[I1], vn = cur.v;                      // V(y), V(y + 1)
        const C ylp = s2_up<T>(yp), yrp = s2_dn<T>(yp);
        const C pxp = cadd(ylp, yrp);
        const C ybp = pick(ylp, yrp);
        // D(y + 1): the upper y face by the BC form (b' = (x, y): own lane), else the stencil
        // with x faces from the inward lane
        C dp;
        if (fhi && y + 1 == ny - 1) {
            dp = dface(yp, vn, yc, vc, dq[I1]);
        } else {
            const C y2 = cadd(yp, yp);
            C acc = csub(pxp, y2);
            acc = cadd(acc, csub(cadd(yc, cur.y), y2));
            dp = cscale(hc.ih2, acc);
            if (EDGE) {
                const C dsh = fromb1(dp);
                const T vsh = __shfl_sync(0xffffffffu, vn, srcl);
                if (xf) dp = dface(yp, vn, ybp, vsh, dsh);
            }
        }
        // 2SHOC step 2 (2d2shocs2) P:214-228 at row y (DAG of DESIGN.md §3.1)
        const C dc = dq[I1];
        const C dl = s2_up<T>(dc), dr = s2_dn<T>(dc);
        const C y4 = cscale(T(4), yc);
        const C cxy = csub(cadd(pq[I0], pxp), y4);
        const C sd = cadd(cadd(dl, dr), cadd(dq[I0], dp));
        const C td = cfma(T(-12), dc, sd);
        const C L = cfma(hc.c16h2, cxy, cneg(cscale(hc.c112, td)));
        const C F = fint(yc, L, vc);
        C Fo = F, f1 = F, y1 = yc;
        if (EDGE) {
            const C fsh = fromb1(F);
            if (xf) { Fo = fbnd(yc, vc, fsh, bq[I1]); f1 = fsh; y1 = bq[I1]; }
        }
        combine(y, Fo, yc, cur.psi, cur.k, own);
        if (flo && y == 1) { lo_f1 = f1; lo_y1 = y1; }           // the y-face rows: after the loop
        if (fhi && y == ny - 2) { hi_f1 = f1; hi_y1 = y1; }
        // the queue positions of row y - 1 take row y + 2 (rotation = renaming across phases)
        yq[I0] = cur.y;
        pq[I2] = pxp;
        dq[I2] = dp;
        vq[I2] = vn;
        bq[I2] = ybp;
    };
    s2_rows(ys, ye, body);
    finish_faces();
}

template <typename T, int ORDER, int BC, int STAGE>
#ifndef NLSE_S2_MINB
#define NLSE_S2_MINB (16 / NLSE_S2_WARPS)     // 16 resident warps per SM (<= 128 registers)
#endif
__global__ void __launch_bounds__(S2_NT, NLSE_S2_MINB) stage2d_strip(const __grid_constant__ StageArgs<T> A, int nstrips, int rows,
                                                                     int rows_e) {
    // items: the interior strips 1 .. nstrips - 2 in chunks of `rows` rows, then the two edge strips
    // (x faces: the face arithmetic makes a row ~1.6x as long) in shorter chunks of `rows_e` rows, so
    // that edge warps end with the others (a single wave otherwise waits for them: ncu showed the
    // SMs active only 57 % of the launch with equal chunks)
    const int item = int(blockIdx.x) * S2_WARPS + int(threadIdx.x >> 5);
    const int r_lo = A.g.zf_lo ? 1 : 0, r_hi = A.g.zf_hi ? int(A.g.ny) - 1 : int(A.g.ny);  // rows computed
    const int ni = nstrips > 2 ? nstrips - 2 : 0;
    const int nch = (r_hi - r_lo + rows - 1) / rows;
    int s, ys, ye;
    if (item < ni * nch) {
        const int chunk = item / ni;
        s = 1 + (item - chunk * ni);
        ys = r_lo + chunk * rows;                          // (face rows ride along with rows 1, ny - 2)
        ye = min(ys + rows, r_hi);
    } else {
        const int ne = nstrips > 1 ? 2 : 1, e = item - ni * nch;
        const int chunk = e / ne;
        s = (e - chunk * ne) == 0 ? 0 : nstrips - 1;
        ys = r_lo + chunk * rows_e;
        ye = min(ys + rows_e, r_hi);
    }
    pdl_trigger();
    if (ys >= r_hi) return;                                  // (whole warp: no CTA-wide sync here)
    pdl_wait();                                              // (before any global access)
    if (s == 0 || s == nstrips - 1) s2_strip<T, ORDER, BC, STAGE, true>(A, s, ys, ye);
    else s2_strip<T, ORDER, BC, STAGE, false>(A, s, ys, ye);
}

// Strips of W interior columns; chunks of `rows` rows per warp.
template <typename T, int ORDER, int BC, int STAGE>
void launch_strip2d(const StageArgs<T> &A, int nsm, cudaStream_t st) {
    constexpr int W = 32 - 2 * ((ORDER == ORDER_2SHOC) ? 2 : 1);
    const int64_t nstrips = (A.g.nx - 2 + W - 1) / W;
    const int64_t nrows = (A.g.zf_hi ? A.g.ny - 1 : A.g.ny) - (A.g.zf_lo ? 1 : 0);
    const char *erows = getenv("NLSE_STRIP_ROWS");    // (read per launch: tests vary it)
    const int env_rows = erows ? std::atoi(erows) : 0;
    int64_t rows;
    if (env_rows > 0) {
        rows = env_rows;
    } else {
        // about 16 resident warps per SM over the whole GPU, chunks of 12 to 32 rows (longer chunks
        // spread the concurrently resident warps over more distant rows: 4096^2 measured 309 us per
        // stage at 256 rows vs 239 us at 32, r02 s2d_e)
        const int64_t target = int64_t(nsm) * 16;                 // warps
        int64_t nch = target / nstrips;
        if (nch > nrows / 12) nch = nrows / 12;
        if (nch < 1) nch = 1;
        rows = (nrows + nch - 1) / nch;
        if (rows > 32) rows = 32;
    }
    // edge-strip chunks of rows / div rows: div = 8 measured best (1024^2: 56.2 us/step vs 68.7 at
    // div 2 and 69.5 at 1; 4096^2 flat, r02 s2d_h / s2d_i)
    const char *ediv = getenv("NLSE_STRIP_EDGE_DIV");
    const int64_t div = ediv ? std::max(1, std::atoi(ediv)) : 8;
    const int64_t rows_e = std::max<int64_t>(1, (rows + div - 1) / div);
    const int64_t nchunks = (nrows + rows - 1) / rows, nchunks_e = (nrows + rows_e - 1) / rows_e;
    const int64_t items = (nstrips > 2 ? nstrips - 2 : 0) * nchunks + (nstrips > 1 ? 2 : 1) * nchunks_e;
    auto kern = stage2d_strip<T, ORDER, BC, STAGE>;
    if (S2Slot<T>::SMEM > 48 * 1024)      // (idempotent, per device of the calling thread)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S2Slot<T>::SMEM);
    // programmatic dependent launch (NLSE_PDL=0: off): this launch's CTAs may be scheduled while the
    // previous stage's tail runs and wait in pdl_wait, overlapping one launch's ramp with the other's
    // tail
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((items + S2_WARPS - 1) / S2_WARPS), 1, 1);
    cfg.blockDim = dim3(S2_NT, 1, 1);
    cfg.dynamicSmemBytes = S2Slot<T>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    const char *epdl = getenv("NLSE_PDL");
    cfg.attrs = at;
    cfg.numAttrs = (epdl && epdl[0] == '0') ? 0 : 1;
    cudaLaunchKernelEx(&cfg, kern, A, int(nstrips), int(rows), int(rows_e));
}

}  // namespace nlse
