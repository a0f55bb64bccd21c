// Row-kernel instantiations with run-time op codes: every non-USER slot
// combination of ops.hpp:14-18 plus the device extensions, any d <= 1024.
// One compact shape per d (no tuning variants) keeps this unit's code size
// bounded: the op switch is resolved per element at run time.
#include "fmm_dispatch.cuh"
namespace fmm {

template <bool EXACT>
static bool generic_aligned(const KParams& p, const DOps& ops, int d, cudaStream_t s) {
    switch (d) {
        case 1: launch_one<DOps, 1, 1, 1, 8, EXACT, false>(p, ops, s); return true;
        case 2: launch_one<DOps, 1, 2, 1, 8, EXACT, false>(p, ops, s); return true;
        case 4: launch_one<DOps, 1, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 8: launch_one<DOps, 2, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 16: launch_one<DOps, 4, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 32: launch_one<DOps, 8, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 64: launch_one<DOps, 16, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 128: launch_one<DOps, 32, 4, 1, 4, EXACT, false>(p, ops, s); return true;
        case 256: launch_one<DOps, 32, 4, 2, 2, EXACT, false>(p, ops, s); return true;
        case 512: launch_one<DOps, 32, 4, 4, 1, EXACT, false>(p, ops, s); return true;
        default: return false;
    }
}

template <bool EXACT>
static bool generic_masked(const KParams& p, const DOps& ops, int d, cudaStream_t s) {
    const int nv = (d + 31) / 32;
    if (nv <= 1) { launch_one<DOps, 32, 1, 1, 4, EXACT, true>(p, ops, s); return true; }
    if (nv <= 2) { launch_one<DOps, 32, 1, 2, 4, EXACT, true>(p, ops, s); return true; }
    if (nv <= 4) { launch_one<DOps, 32, 1, 4, 2, EXACT, true>(p, ops, s); return true; }
    if (nv <= 8) { launch_one<DOps, 32, 1, 8, 1, EXACT, true>(p, ops, s); return true; }
    if (nv <= 16) { launch_one<DOps, 32, 1, 16, 1, EXACT, true>(p, ops, s); return true; }
    if (nv <= 32) { launch_one<DOps, 32, 1, 32, 1, EXACT, true>(p, ops, s); return true; }
    return false;
}

bool launch_generic(const KParams& p, int d, bool exact, bool vectorised, cudaStream_t s) {
    const DOps ops{p.vop, p.rop, p.sop, p.mop, p.aop, p.mlp_wx, p.mlp_wy, p.mlp_b};
    if (vectorised)
        return exact ? generic_aligned<true>(p, ops, d, s) : generic_aligned<false>(p, ops, d, s);
    return exact ? generic_masked<true>(p, ops, d, s) : generic_masked<false>(p, ops, d, s);
}
}  // namespace fmm
