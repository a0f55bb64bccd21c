// Row-kernel instantiations for the OpsSigmoid pattern (see fmm_kernels.cuh).
#include "fmm_dispatch.cuh"
FMM_DEFINE_STATIC_LAUNCH(launch_sigmoid, OpsSigmoid)
