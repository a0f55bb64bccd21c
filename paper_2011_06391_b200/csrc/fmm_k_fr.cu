// Row-kernel instantiations for the OpsFr pattern (see fmm_kernels.cuh), and
// the persistent pipelined variant (fmm_sched.cuh).
#include "fmm_dispatch.cuh"
#include "fmm_sched.cuh"
FMM_DEFINE_STATIC_LAUNCH(launch_fr, OpsFr)
namespace fmm {
bool launch_sched_fr(const SchedParams& p, int d, int variant, int num_sms, cudaStream_t s) {
    return launch_sched<OpsFr>(p, OpsFr{}, d, variant, num_sms, s);
}
}  // namespace fmm
