// stream3d.cuh -- 3D interior stage kernel (placeholder: interior-only generic evaluation).
#pragma once
#include "generic.cuh"

namespace nlse {

template <typename T, int DIM, int ORDER, int BC, int STAGE>
__global__ void __launch_bounds__(256) stage_interior_generic(StageArgs<T> A) {
    // interior points only, flat index over the (nx-2)(ny-2)(nz-2) box
    const int64_t mx = A.g.nx - 2, my = DIM >= 2 ? A.g.ny - 2 : 1, mz = DIM >= 3 ? A.g.nz - 2 : 1;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= mx * my * mz) return;
    const int64_t i = 1 + t % mx;
    const int64_t j = DIM >= 2 ? 1 + (t / mx) % my : 0;
    const int64_t k = DIM >= 3 ? 1 + t / (mx * my) : 0;
    PointEval<T, DIM, ORDER, BC> ev{A.Y, A.V, A.g, A.c};
    const int64_t q = ev.idx(i, j, k);
    cplx<T> F = ev.F_int(i, j, k);
    cplx<T> psi = (STAGE == 1) ? ev.y(q) : A.Psi[q];
    rk_combine<STAGE, T>(A, q, F, psi);
}

template <typename T, int ORDER, int BC, int STAGE>
void launch_stream3d(const StageArgs<T> &A, cudaStream_t st) {
    const int64_t m = (A.g.nx - 2) * (A.g.ny - 2) * (A.g.nz - 2);
    stage_interior_generic<T, 3, ORDER, BC, STAGE><<<unsigned((m + 255) / 256), 256, 0, st>>>(A);
}

}  // namespace nlse
