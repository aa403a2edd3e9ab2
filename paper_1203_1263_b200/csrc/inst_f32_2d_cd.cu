// Stage kernels of one family (precision f32, 2D, CD): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f32, 2, cd)
NLSE_DEFINE_PERSIST2D(f32, cd)
