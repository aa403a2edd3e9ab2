// Stage kernels of one family (precision f32, 3D, CD): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f32, 3, cd)
NLSE_DEFINE_FUSED(f32, dirichlet)
NLSE_DEFINE_FUSED(f32, msd)
NLSE_DEFINE_FUSED(f32, l0)
