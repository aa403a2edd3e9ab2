// tile2d.cuh -- 1D / 2D interior stage kernels (placeholder: interior-only generic evaluation).
#pragma once
#include "stream3d.cuh"

namespace nlse {

template <typename T, int ORDER, int BC, int STAGE>
void launch_tile2d(const StageArgs<T> &A, cudaStream_t st) {
    const int64_t m = (A.g.nx - 2) * (A.g.ny - 2);
    stage_interior_generic<T, 2, ORDER, BC, STAGE><<<unsigned((m + 255) / 256), 256, 0, st>>>(A);
}
template <typename T, int ORDER, int BC, int STAGE>
void launch_tile1d(const StageArgs<T> &A, cudaStream_t st) {
    const int64_t m = A.g.nx - 2;
    stage_interior_generic<T, 1, ORDER, BC, STAGE><<<unsigned((m + 255) / 256), 256, 0, st>>>(A);
}

}  // namespace nlse
