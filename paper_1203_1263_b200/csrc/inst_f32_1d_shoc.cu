// Stage kernels of one family (precision f32, 1D, 2SHOC): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f32, 1, shoc)
NLSE_DEFINE_PERSIST1D(f32, shoc)
