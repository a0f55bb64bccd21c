// Row-kernel instantiations for the OpsTdist pattern (see fmm_kernels.cuh).
#include "fmm_dispatch.cuh"
FMM_DEFINE_STATIC_LAUNCH(launch_tdist, OpsTdist)
