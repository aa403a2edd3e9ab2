// fused3d.cuh -- temporal blocking of the RK4 stages ("the more
// computations a single kernel call performs, the better"): ONE HBM pass computes
// two consecutive stages, S1+S2 (PAIR 1) or S3+S4 (PAIR 2), for the 3D CD scheme.
//
// Per CTA: a 32 x TY column tile streamed along a z chunk, as stage3d_tma.  Stage A (S1 or S3)
// is evaluated on the tile plus a one-point ring R (34 x (TY+2) points), one plane ahead of
// stage B (S2 or S4), so its output Z (Psi_tmp) never leaves shared memory:
//   A(p):  F_A = F(Y_A) on R of plane p (CD: L = D, (fsplit) P:424-428; faces by the BC time-
//          derivative form, (BCDdt) P:315-318, (msd) P:331-335, (BCL0dt) P:347-350, with F_A at
//          b' from the same pass); Z = base + c_A F_A  (S1: base = Y_A = Psi, c_A = k/2;
//          S3: base = Psi, c_A = k; (RK4_GPU) P:495-519)
//   B(z):  F_B = F(Z) at the owned interior points of plane z; S2: K = 2 F_B + F_A,
//          Psi_out = Psi + (k/2) F_B;  S4: Psi_new = Psi + (k/6)((2 F_A + K) + F_B)
// HBM traffic per point and step (fp64 + V): pair 1 reads Psi, V and writes K, Psi_out
// (56 B); pair 2 reads Psi_out, Psi, K, V and writes Psi_new (72 B): 128 B instead of the
// 304 B of four single-stage passes.  Psi_new goes to a second Psi buffer (ping-pong): pair 2
// reads Psi on the ring R, so it cannot be updated in place.
//
// Domain-boundary outputs of stage B come from the existing boundary kernels run after this
// one (stage_boundary / stage_boundary_msd_fb): this kernel leaves them what they read --
// Z at face points and at their inward neighbours b' (planes 1, nz-2 and the in-plane shell)
// in the Psi_tmp buffer, K after stage A at face points, and (MSD) F_B at b' in fz / fp.
// Every value follows the DAG of DESIGN.md §3.1 term by term, so results are bit-identical to
// the oracle's four separate stages.  Single GPU (no slab mode), 3D, CD.
#pragma once
#include "stage3d_tma.cuh"

namespace nlse {

#ifndef NLSE_FUSED_P
#define NLSE_FUSED_P 2
#endif
#ifndef NLSE_FUSED_MINB
#define NLSE_FUSED_MINB 1
#endif
template <typename T, int TYV, int PAIR = 2>
struct F3Cfg {
    static constexpr int TX = 32, TY = TYV;
    static constexpr int RX = TX + 2, RY = TY + 2, RS = RX * RY;    // region R (stage A outputs)
    static constexpr int NT = (RS + 31) / 32 * 32;                  // one thread per point of R
    static constexpr int YX = TX + 4, YY = TY + 4;                  // Y_A box, origin (x0-2, y0-2)
    static constexpr int BX = TX + 4, BY = RY;                      // base box (complex), origin (x0-2, y0-1)
    static constexpr int VXO = sizeof(T) == 4 ? 4 : 2;              // V box origin x0 - VXO (16-byte aligned)
    static constexpr int VX = TX + 2 * VXO, VY = RY;
    static constexpr int CB = 2 * int(sizeof(T));
    // ring sizes: a slot is refilled one plane after its last reader (single barrier per plane)
    static constexpr int P = NLSE_FUSED_P;                          // planes of prefetch
    static constexpr int NSY = P + 3;                               // Y_A ring (planes p-1, p, p+1 + P)
    static constexpr int NSV = P + 2;                               // V / base ring (planes z, p + P)
    static constexpr int NSK = P + 1;                               // K ring (plane z + P)
    static constexpr int NZ = 4;                                    // Z ring (planes z-1, z, z+1 + one being written)
    static constexpr int up128(int b) { return (b + 127) / 128 * 128; }
    static constexpr int YSLOT = up128(YX * YY * CB);
    static constexpr int VSLOT = up128(VX * VY * int(sizeof(T)));
    static constexpr int BSLOT = up128(BX * BY * CB);
    static constexpr int KSLOT = up128(TX * TY * CB);
    static constexpr int RSLOT = up128(RS * CB);
    static constexpr int OFF_V = NSY * YSLOT;
    static constexpr int OFF_B = OFF_V + NSV * VSLOT;
    static constexpr int OFF_K = OFF_B + (PAIR == 2 ? NSV * BSLOT : 0);   // base and K: pair 2 only
    static constexpr int OFF_Z = OFF_K + (PAIR == 2 ? NSK * KSLOT : 0);
    static constexpr int OFF_BAR = OFF_Z + NZ * RSLOT;
    static constexpr int SMEM = OFF_BAR + (NSY + NSV + NSK) * 8;
    // box dimensions in T elements (x) and rows
    static constexpr int BOX_Y_X = 2 * YX, BOX_Y_Y = YY;
    static constexpr int BOX_B_X = 2 * BX, BOX_B_Y = BY;
    static constexpr int BOX_V_X = VX, BOX_V_Y = VY;
    static constexpr int BOX_K_X = 2 * TX, BOX_K_Y = TY;
};

// Arguments of one fused launch (in addition to the StageArgs of stage B, A.c.kc = c_B).
template <typename T>
struct FusedArgs {
    T cA;                 // stage A coefficient: k/2 (S1) or k (S3)
    cplx<T> *ztmp;        // Psi_tmp buffer: Z at face / b' points for the boundary pass
};

// One fused pass.  PAIR 1: Y_A = base = Psi (mY), out = Psi_out, K written.  PAIR 2: Y_A = Psi_out
// (mY), base = Psi (mB), K read (mK), out = the other Psi buffer.
template <typename T, int BC, int PAIR, int TYV>
__global__ void __launch_bounds__(F3Cfg<T, TYV>::NT, NLSE_FUSED_MINB)
fused3d_cd(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mB,
           const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV,
           const __grid_constant__ StageArgs<T> A, const __grid_constant__ FusedArgs<T> FA, int zchunk, int ntx,
           int nty) {
    using C = cplx<T>;
    using Cfg = F3Cfg<T, TYV, PAIR>;
    constexpr int TX = Cfg::TX, TY = Cfg::TY, RX = Cfg::RX, RS = Cfg::RS;
    constexpr int YX = Cfg::YX, BX = Cfg::BX, VX = Cfg::VX, VXO = Cfg::VXO;
    constexpr int NSY = Cfg::NSY, NSV = Cfg::NSV, NSK = Cfg::NSK, P = Cfg::P;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw;
    const Grid &g = A.g;
    const int ntiles = ntx * nty;
    const int w = blockIdx.x;
    const int cidx = w / ntiles, t = w - cidx * ntiles;
    const int x0 = (t % ntx) * TX, y0 = (t / ntx) * TY;
    const int nx = int(g.nx), ny = int(g.ny), nz = int(g.nz);
    const int zs = 1 + cidx * zchunk;
    const int ze = min(zs + zchunk, nz - 1);
    if (zs >= ze) return;
    const int tid = threadIdx.x;
    const bool hasV = A.V != nullptr;
    const unsigned sb = smem_u32(sm);
    const unsigned barY = sb + Cfg::OFF_BAR, barV = barY + 8 * NSY, barK = barV + 8 * NSV;

    // ---- TMA issue (one elected thread) ----
    const int ylo = zs - 2, yhi = min(ze + 1, nz - 1);        // Y_A planes needed (clipped to the grid)
    const int vlo = zs - 1, vhi = ze;                        // V / base planes (A on zs-1 .. ze)
    auto issue_y = [&](int p) {
        if (p > yhi) return;
        const int s = (p - ylo) % NSY;
        const unsigned bar = barY + 8 * s;
        if (p < 0) { mbar_arrive(bar); return; }            // below the grid: never read
        mbar_expect_tx(bar, Cfg::YX * Cfg::YY * Cfg::CB);
        tma_load_3d(sb + s * Cfg::YSLOT, &mY, 2 * (x0 - 2), y0 - 2, p, bar);
    };
    const unsigned vbytes = (hasV ? unsigned(VX * Cfg::VY * sizeof(T)) : 0u) +
                            (PAIR == 2 ? unsigned(BX * Cfg::BY * Cfg::CB) : 0u);
    auto issue_v = [&](int p) {
        if (p > vhi || vbytes == 0) return;
        const int s = (p - vlo) % NSV;
        const unsigned bar = barV + 8 * s;
        mbar_expect_tx(bar, vbytes);
        if (hasV) tma_load_3d(sb + Cfg::OFF_V + s * Cfg::VSLOT, &mV, x0 - VXO, y0 - 1, p, bar);
        if (PAIR == 2) tma_load_3d(sb + Cfg::OFF_B + s * Cfg::BSLOT, &mB, 2 * (x0 - 2), y0 - 1, p, bar);
    };
    auto issue_k = [&](int z) {
        if (PAIR != 2 || z >= ze) return;
        const int s = (z - zs) % NSK;
        const unsigned bar = barK + 8 * s;
        mbar_expect_tx(bar, TX * TY * Cfg::CB);
        tma_load_3d(sb + Cfg::OFF_K + s * Cfg::KSLOT, &mK, 2 * x0, y0, z, bar);
    };
    if (tid == 0) {
        for (int i = 0; i < NSY + NSV + NSK; i++) mbar_init(barY + 8 * i, 1);
        fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0) {
        for (int p = ylo; p < ylo + NSY; p++) issue_y(p);
        for (int p = vlo; p < vlo + NSV; p++) issue_v(p);
        for (int z = zs; z < zs + NSK; z++) issue_k(z);
    }
    auto wait_y = [&](int p) {
        if (p > yhi) return;
        const int u = p - ylo;
        mbar_wait(barY + 8 * (u % NSY), unsigned(u / NSY) & 1u);
    };
    auto wait_v = [&](int p) {
        if (vbytes == 0) return;
        const int u = p - vlo;
        mbar_wait(barV + 8 * (u % NSV), unsigned(u / NSV) & 1u);
    };
    auto wait_k = [&](int z) {
        if (PAIR != 2) return;
        const int u = z - zs;
        mbar_wait(barK + 8 * (u % NSK), unsigned(u / NSK) & 1u);
    };
    // ---- shared-memory views: local coordinates (lx, ly) relative to (x0, y0) ----
    auto Yp = [&](int p) -> const C * {                      // Y_A at (lx, ly): [(ly+2)*YX + lx+2]
        return reinterpret_cast<const C *>(sm + ((p - ylo) % NSY) * Cfg::YSLOT) + 2 * YX + 2;
    };
    auto Vp = [&](int p) -> const T * {                      // V at (lx, ly): [(ly+1)*VX + lx+VXO]
        return reinterpret_cast<const T *>(sm + Cfg::OFF_V + ((p - vlo) % NSV) * Cfg::VSLOT) + VX + VXO;
    };
    auto Bp = [&](int p) -> const C * {                      // base at (lx, ly): [(ly+1)*BX + lx+2]
        return reinterpret_cast<const C *>(sm + Cfg::OFF_B + ((p - vlo) % NSV) * Cfg::BSLOT) + BX + 2;
    };
    auto Kp = [&](int z) -> const C * {                      // K at owned (lx, ly): [ly*TX + lx]
        return reinterpret_cast<const C *>(sm + Cfg::OFF_K + ((z - zs) % NSK) * Cfg::KSLOT);
    };
    // the same views by ring slot index (the loop advances the slot indices incrementally)
    auto Ys = [&](int sl) -> const C * { return reinterpret_cast<const C *>(sm + sl * Cfg::YSLOT) + 2 * YX + 2; };
    auto Vs = [&](int sl) -> const T * {
        return reinterpret_cast<const T *>(sm + Cfg::OFF_V + sl * Cfg::VSLOT) + VX + VXO;
    };
    auto Bs = [&](int sl) -> const C * {
        return reinterpret_cast<const C *>(sm + Cfg::OFF_B + sl * Cfg::BSLOT) + BX + 2;
    };
    auto Zsl = [&](int sl) -> C * { return reinterpret_cast<C *>(sm + Cfg::OFF_Z + sl * Cfg::RSLOT) + RX + 1; };
    const T s_ = A.c.s, a_ = A.c.a, ih2 = A.c.ih2;
    // F (fsplit) P:424-428 at one point, R-ASSOC
    auto fsplit = [&](C y, C L, T v) -> C {
        const T rho = (y.x * y.x) + (y.y * y.y);
        const T sr = s_ * rho;
        C F = f_lin(a_, L, sr, y);
        if (hasV) F = f_addv(F, v, y);
        return F;
    };
    // CD: L = D = (((Px - Y2) + (Py - Y2)) + (Pz - Y2)) * ih2 from a plane view with row pitch W
    auto cd = [&](const C *ym, const C *y0p, const C *yp, int o, int W) -> C {
        const C yc = y0p[o];
        const C y2 = cadd(yc, yc);
        C acc = csub(cadd(y0p[o - 1], y0p[o + 1]), y2);
        acc = cadd(acc, csub(cadd(y0p[o - W], y0p[o + W]), y2));
        acc = cadd(acc, csub(cadd(ym[o], yp[o]), y2));
        return cscale(ih2, acc);
    };
    auto vat = [&](int p, int lx, int ly) -> T { return hasV ? Vp(p)[ly * VX + lx] : T(0); };
    auto zface = [&](int p) { return (g.zf_lo && p == 0) || (g.zf_hi && p == nz - 1); };

    // Thread t owns point t of the ring region R (local (lx, ly) = (t % RX - 1, t / RX - 1)) in
    // stage A and, when that point is one of the tile's own interior points, in stage B too, so
    // F_A of its point stays in a register from A(z) to B(z).
    const int lx = tid % RX - 1, ly = tid / RX - 1;
    const int gx = x0 + lx, gy = y0 + ly;
    const bool in_r = tid < RS && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
    const bool fx = gx == 0 || gx == nx - 1, fy = gy == 0 || gy == ny - 1;
    const bool interior = in_r && !fx && !fy;
    const bool owned = in_r && lx >= 0 && lx < TX && ly >= 0 && ly < TY;
    const bool outpt = owned && interior;                          // a stage-B output point
    const int lx1 = gx == 0 ? lx + 1 : (gx == nx - 1 ? lx - 1 : lx);  // b': one step inward
    const int ly1 = gy == 0 ? ly + 1 : (gy == ny - 1 ? ly - 1 : ly);  //     along every face axis
    const int oy = ly * YX + lx, oy1 = ly1 * YX + lx1, orr = ly * RX + lx;
    const int64_t qrow = int64_t(gy) * g.sy + gx;
    const bool shell_xy = gx == 1 || gx == nx - 2 || gy == 1 || gy == ny - 2;
    // F_A at an in-plane interior point (CD, (fsplit)) of plane p, Y-box offset o, V offset (x, y)
    auto f_int = [&](int p, int o, int vx, int vy) -> C {
        return fsplit(Yp(p)[o], cd(Yp(p - 1), Yp(p), Yp(p + 1), o, YX), vat(p, vx, vy));
    };
    // Stage A at this thread's point of plane p: F_A (faces by the BC time-derivative form with
    // F_A(b') recomputed here, b' on plane pb), Z = base + c_A F_A into the Z slot of plane p,
    // and the boundary data of the stage-B boundary kernel at this CTA's own points.
    // ym, yc, yp: Y_A slots of planes p-1, p, p+1; vc: V slot of p (or null); bc_: base slot of p;
    // zo: Z slot of plane p
    auto stage_a = [&](int p, const C *ym, const C *yc, const C *yp, const T *vc, const C *bc_, C *zo) -> C {
        C f; f.x = T(0); f.y = T(0);
        if (!in_r) return f;
        const bool zf = zface(p);
        const C y = yc[oy];
        const bool face = zf || fx || fy;
        if (!face) {
            f = fsplit(y, cd(ym, yc, yp, oy, YX), hasV ? vc[ly * VX + lx] : T(0));
        } else if (BC == BC_L0) {
            C zr; zr.x = T(0); zr.y = T(0);
            f = fsplit(y, zr, vat(p, lx, ly));                        // (BCL0dt) P:347-350, R-L0
        } else if (BC == BC_MSD) {                                    // (msd) P:331-335
            const int pb = zf ? (p == 0 ? 1 : nz - 2) : p;
            const C y1 = Yp(pb)[oy1];
            const C f1 = f_int(pb, oy1, lx1, ly1);
            const T rho1 = (y1.x * y1.x) + (y1.y * y1.y);
            T m = T(0);
            if (!(rho1 < A.c.eps2)) m = ((f1.y * y1.x) - (f1.x * y1.y)) / rho1;
            f.x = -(m * y.y);
            f.y = m * y.x;
        }                                                             // Dirichlet: 0 (BCDdt) P:315-318
        const C base = PAIR == 1 ? y : bc_[ly * BX + lx];
        const C z = cfma(FA.cA, f, base);
        zo[orr] = z;
        if (owned && ((p >= zs && p < ze) || zf)) {
            const int64_t q = int64_t(p) * g.sz + qrow;
            const bool shell = !face && (shell_xy || (g.zf_lo && p == 1) || (g.zf_hi && p == nz - 2));
            if (face || shell) FA.ztmp[q] = z;
            if (face) A.K[q] = PAIR == 1 ? f : cfma(T(2), f, __ldg(A.K + q));
        }
        return f;
    };
    // Stage B at this thread's own interior point of plane z (F_A of that point given)
    // zm, zc, zp: Z slots of planes z-1, z, z+1; yz: Y_A slot of z; vz, bz: V / base slots of z
    auto stage_b = [&](int z, C fa, const C *zm, const C *zc, const C *zp, const C *yz, const T *vz, const C *bz) {
        const C y = zc[orr];
        const C fb = fsplit(y, cd(zm, zc, zp, orr, RX), hasV ? vz[ly * VX + lx] : T(0));
        const int64_t q = int64_t(z) * g.sz + qrow;
        if (PAIR == 1) {
            const C psi = yz[oy];
            A.K[q] = cfma(T(2), fb, fa);                              // S2: K = 2 F_B + F_A (S1: K = F_A)
            A.out[q] = cfma(A.c.kc, fb, psi);                         // Psi_out = Psi + (k/2) F_B
        } else {
            const C psi = bz[ly * BX + lx];
            const C kt = cfma(T(2), fa, Kp(z)[ly * TX + lx]);        // S3: K = 2 F_A + K
            const C o = cfma(A.c.kc, cadd(kt, fb), psi);              // S4: Psi + (k/6)(K + F_B)
            A.out[q] = o;
            if (!(isfinite(o.x) && isfinite(o.y))) atomicMin(A.diverged, *A.step_base + A.step);
        }
        if (A.fp) {                                                   // F_B at b' for the MSD light pass
            if (g.zf_lo && z == 1) A.fz[gy * nx + gx] = fb;
            if (g.zf_hi && z == nz - 2) A.fz[int64_t(nx) * ny + gy * nx + gx] = fb;
            if (shell_xy) A.fp[int64_t(z) * A.per2 + shell_u(gx, gy, nx, ny)] = fb;
        }
    };

    // ---- prologue: stage A on planes zs-1 (a z face when zs == 1) and zs ----
    wait_y(zs - 2); wait_y(zs - 1); wait_y(zs); wait_y(zs + 1);
    wait_v(zs - 1); wait_v(zs);
    // Z ring: planes z-1, z, z+1 in slots zm1, z0s, zp1; zfr is written next (plane z+2)
    int zm1 = 0, z0s = 1, zp1 = 2, zfr = 3;
    stage_a(zs - 1, Yp(zs - 2), Yp(zs - 1), Yp(zs), hasV ? Vp(zs - 1) : nullptr, Bp(zs - 1), Zsl(zm1));
    C fa = stage_a(zs, Yp(zs - 1), Yp(zs), Yp(zs + 1), hasV ? Vp(zs) : nullptr, Bp(zs), Zsl(z0s));
    __syncthreads();
    if (tid == 0) {                     // the prologue-only planes zs-2 (Y_A) and zs-1 (V / base) are free
        issue_y(zs - 2 + NSY);
        issue_v(zs - 1 + NSV);
    }
    // ring slots of plane z (Y_A, V / base) and of Z planes z-1, z, z+1, advanced per plane
    int sy0 = (zs - ylo) % NSY, sv0 = (zs - vlo) % NSV;
    auto nxt = [](int sl, int n) { return sl + 1 == n ? 0 : sl + 1; };
    for (int z = zs; z < ze; z++) {
        const int p = z + 1;
        if (!zface(p)) wait_y(p + 1);
        wait_v(p);
        wait_k(z);
        const int sy1 = nxt(sy0, NSY), sy2 = nxt(sy1, NSY), sv1 = nxt(sv0, NSV);
        // top z face: b' on plane p - 1 = z (its Y / V slots are intact)
        const C fa_next = stage_a(p, Ys(sy0), Ys(sy1), Ys(sy2), hasV ? Vs(sv1) : nullptr, Bs(sv1), Zsl(zp1));
        // the one barrier per plane: Z(z+1) is complete, and every thread has finished iteration
        // z-1, so the slots whose last reader was B(z-1) / A(z) are free: Y_A(z-1), V / base(z-1),
        // K(z-1) (the Z slot written next iteration held plane z-2, read last by B(z-1))
        __syncthreads();
        if (tid == 0) {
            issue_y(z - 1 + NSY);
            if (z > zs) issue_v(z - 1 + NSV);   // (V / base(zs-1) was refilled after the prologue;
            if (z > zs) issue_k(z - 1 + NSK);   //  K has no plane zs-1)
        }
        if (outpt) stage_b(z, fa, Zsl(zm1), Zsl(z0s), Zsl(zp1), Ys(sy0), hasV ? Vs(sv0) : nullptr, Bs(sv0));
        fa = fa_next;
        sy0 = sy1; sv0 = sv1;
        { const int t = zm1; zm1 = z0s; z0s = zp1; zp1 = zfr; zfr = t; }
    }
}

}  // namespace nlse
