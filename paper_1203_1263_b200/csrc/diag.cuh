// diag.cuh -- mass and Hamiltonian (north_star (c); reading R-DIAG):
//   M = h^d sum_p |Psi_p|^2
//   H = h^d sum_p [ a sum_axes |Psi_{p+e} - Psi_p|^2 / h^2 + V_p |Psi_p|^2 - (s/2)|Psi_p|^4 ]
// Per-point terms in fp64 (Psi widened exactly), per-thread fp64 partial sums,
// warp-shuffle then block reduction, one partial pair per block, and a fixed-order
// single-block final pass: deterministic for a given grid and launch shape.
#pragma once
#include "common.cuh"

namespace nlse {

constexpr int DIAG_THREADS = 256;

__device__ __forceinline__ void block_reduce2(double &m, double &e, double *smem) {
    for (int o = 16; o > 0; o >>= 1) {
        m += __shfl_down_sync(0xffffffffu, m, o);
        e += __shfl_down_sync(0xffffffffu, e, o);
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { smem[2 * w] = m; smem[2 * w + 1] = e; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        m = lane < nw ? smem[2 * lane] : 0.0;
        e = lane < nw ? smem[2 * lane + 1] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            m += __shfl_down_sync(0xffffffffu, m, o);
            e += __shfl_down_sync(0xffffffffu, e, o);
        }
    }
}

template <typename T, int DIM>
__global__ void __launch_bounds__(DIAG_THREADS)
diag_partial(const cplx<T> *__restrict__ Psi, const T *__restrict__ V, Grid g, double a, double s,
             double ih2, double *__restrict__ partial) {
    __shared__ double smem[2 * (DIAG_THREADS / 32)];
    double m = 0.0, e = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < g.n; t += stride) {
        // logical point t -> (i, row), element q of the (possibly pitched, g.sy >= nx) buffer
        const int64_t row = t / g.nx, i = t - row * g.nx;
        const int64_t q = row * g.sy + i;
        const cplx<T> p = Psi[q];
        const double pr = p.x, pi = p.y;
        const double rho = pr * pr + pi * pi;
        double grad = 0.0;
        // x pairs (1D x-slabs: also across to the upper neighbour's first point, a ghost)
        if (i + 1 < g.nx + ((DIM == 1 && !g.zf_hi) ? 1 : 0)) {
            const cplx<T> u = Psi[q + 1];
            const double dr = double(u.x) - pr, di = double(u.y) - pi;
            grad += dr * dr + di * di;
        }
        // y pairs (2D y-slabs: also across to the upper neighbour's first row, a ghost row)
        if (DIM >= 2 && (row % g.ny) + 1 < g.ny + ((DIM == 2 && !g.zf_hi) ? 1 : 0)) {
            const cplx<T> u = Psi[q + g.sy];
            const double dr = double(u.x) - pr, di = double(u.y) - pi;
            grad += dr * dr + di * di;
        }
        // z pairs: inside the slab, or across to the upper neighbour's first plane (ghost)
        if (DIM >= 3 && (row / g.ny) + 1 < g.nz + (g.zf_hi ? 0 : 1)) {
            const cplx<T> u = Psi[q + g.sz];
            const double dr = double(u.x) - pr, di = double(u.y) - pi;
            grad += dr * dr + di * di;
        }
        double en = a * grad * ih2 - 0.5 * s * rho * rho;
        if (V) en += double(V[q]) * rho;
        m += rho;
        e += en;
    }
    block_reduce2(m, e, smem);
    if (threadIdx.x == 0) { partial[2 * blockIdx.x] = m; partial[2 * blockIdx.x + 1] = e; }
}

__global__ void __launch_bounds__(DIAG_THREADS)
diag_final(const double *__restrict__ partial, int nblocks, double hd, double *__restrict__ result) {
    __shared__ double smem[2 * (DIAG_THREADS / 32)];
    double m = 0.0, e = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) { m += partial[2 * b]; e += partial[2 * b + 1]; }
    block_reduce2(m, e, smem);
    if (threadIdx.x == 0) { result[0] = hd * m; result[1] = hd * e; }
}

}  // namespace nlse
