// Stage kernels of one family (precision f32, 3D, 2SHOC, BC l0): a separate translation unit
// so that nvcc compiles the families in parallel (stages.cuh).
#include "stages.cuh"

NLSE_DEFINE_STAGES_BC(f32, 3, shoc, l0)
