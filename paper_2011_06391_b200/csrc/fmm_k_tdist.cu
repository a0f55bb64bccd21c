// Row-kernel instantiations for the OpsTdist pattern (see fmm_kernels.cuh), and
// the persistent pipelined variant (fmm_sched.cuh).
#include "fmm_dispatch.cuh"
#include "fmm_sched.cuh"
FMM_DEFINE_STATIC_LAUNCH(launch_tdist, OpsTdist)
namespace fmm {
bool launch_sched_tdist(const SchedParams& p, int d, int variant, int num_sms, cudaStream_t s) {
    return launch_sched<OpsTdist>(p, OpsTdist{}, d, variant, num_sms, s);
}
}  // namespace fmm
