// Stage kernels of one family (precision f64, 1D, 2SHOC): a separate translation unit so
// that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES(f64, 1, shoc)
NLSE_DEFINE_PERSIST1D(f64, shoc)
