// Stage kernels of one family (precision f32, 1D, CD): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f32, 1, cd)
NLSE_DEFINE_PERSIST1D(f32, cd)
