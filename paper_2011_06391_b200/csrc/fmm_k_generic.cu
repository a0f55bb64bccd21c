// Row-kernel instantiations with run-time op codes: every non-USER slot
// combination of ops.hpp:14-18 plus the device extensions, any d <= 1024.
#include "fmm_dispatch.cuh"
namespace fmm {
bool launch_generic(const KParams& p, int d, bool exact, bool vectorised, cudaStream_t s) {
    const DOps ops{p.vop, p.rop, p.sop, p.mop, p.aop};
    if (vectorised)
        return exact ? launch_aligned<DOps, true>(p, ops, d, s) : launch_aligned<DOps, false>(p, ops, d, s);
    return exact ? launch_masked<DOps, true>(p, ops, d, s) : launch_masked<DOps, false>(p, ops, d, s);
}
}  // namespace fmm
