// Stage kernels of one family (precision f64, 3D, CD): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f64, 3, cd)
NLSE_DEFINE_FUSED(f64, dirichlet)
NLSE_DEFINE_FUSED(f64, msd)
NLSE_DEFINE_FUSED(f64, l0)
