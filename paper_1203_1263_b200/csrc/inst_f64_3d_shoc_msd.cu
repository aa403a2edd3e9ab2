// Stage kernels of one family (precision f64, 3D, 2SHOC, BC msd): a separate translation unit
// so that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES_BC(f64, 3, shoc, msd)
