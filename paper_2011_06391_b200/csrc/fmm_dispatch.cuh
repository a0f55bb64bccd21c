// fmm_dispatch.cuh — maps (d, alignment) to a row-kernel instantiation.
// Included by one translation unit per op kind so the instantiations compile
// in parallel.
#pragma once

#include "fmm_kernels.cuh"

namespace fmm {

template <class Ops, int LPR, int VEC, int NV, int UNROLL, bool EXACT, bool MASKED>
inline void launch_one(const KParams& p, const Ops& ops, cudaStream_t stream) {
    constexpr int kThreads = 256;
    constexpr int groups_per_block = kThreads / LPR;
    const int64_t total = p.n_chunk_items + p.n_row_items;
    if (total <= 0) return;
    const int64_t blocks = (total + groups_per_block - 1) / groups_per_block;
    fmm_rows_kernel<Ops, LPR, VEC, NV, UNROLL, EXACT, MASKED>
        <<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(p, ops);
}

// Vectorised shapes: d = LPR * VEC * NV exactly, rows VEC*4-byte aligned.
template <class Ops, bool EXACT>
inline bool launch_aligned(const KParams& p, const Ops& ops, int d, cudaStream_t s) {
    switch (d) {
        case 1: launch_one<Ops, 1, 1, 1, 8, EXACT, false>(p, ops, s); return true;
        case 2: launch_one<Ops, 1, 2, 1, 8, EXACT, false>(p, ops, s); return true;
        case 4: launch_one<Ops, 1, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 8: launch_one<Ops, 2, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 16: launch_one<Ops, 4, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 32: launch_one<Ops, 8, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 64: launch_one<Ops, 16, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 128: launch_one<Ops, 32, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 256: launch_one<Ops, 32, 4, 2, 4, EXACT, false>(p, ops, s); return true;
        case 512: launch_one<Ops, 32, 4, 4, 2, EXACT, false>(p, ops, s); return true;
        default: return false;
    }
}

// Masked scalar-load shapes for any d <= 1024.
template <class Ops, bool EXACT>
inline bool launch_masked(const KParams& p, const Ops& ops, int d, cudaStream_t s) {
    const int nv = (d + 31) / 32;
    if (nv <= 1) { launch_one<Ops, 32, 1, 1, 8, EXACT, true>(p, ops, s); return true; }
    if (nv <= 2) { launch_one<Ops, 32, 1, 2, 8, EXACT, true>(p, ops, s); return true; }
    if (nv <= 4) { launch_one<Ops, 32, 1, 4, 4, EXACT, true>(p, ops, s); return true; }
    if (nv <= 8) { launch_one<Ops, 32, 1, 8, 2, EXACT, true>(p, ops, s); return true; }
    if (nv <= 16) { launch_one<Ops, 32, 1, 16, 1, EXACT, true>(p, ops, s); return true; }
    if (nv <= 32) { launch_one<Ops, 32, 1, 32, 1, EXACT, true>(p, ops, s); return true; }
    return false;
}

// True when d has a vectorised shape and the row alignment permits it.
inline bool aligned_shape(int d, bool aligned16, bool aligned8) {
    switch (d) {
        case 1: return true;
        case 2: return aligned8;
        case 4: case 8: case 16: case 32: case 64: case 128: case 256: case 512:
            return aligned16;
        default: return false;
    }
}

bool launch_sigmoid(const KParams& p, int d, bool exact, cudaStream_t s);
bool launch_gcn(const KParams& p, int d, bool exact, cudaStream_t s);
bool launch_fr(const KParams& p, int d, bool exact, cudaStream_t s);
bool launch_tdist(const KParams& p, int d, bool exact, cudaStream_t s);
bool launch_frattr(const KParams& p, int d, bool exact, cudaStream_t s);
bool launch_generic(const KParams& p, int d, bool exact, bool vectorised, cudaStream_t s);

}  // namespace fmm

#define FMM_DEFINE_STATIC_LAUNCH(NAME, OPS)                                        \
    namespace fmm {                                                                \
    bool NAME(const KParams& p, int d, bool exact, cudaStream_t s) {               \
        const OPS ops{};                                                           \
        return exact ? launch_aligned<OPS, true>(p, ops, d, s)                     \
                     : launch_aligned<OPS, false>(p, ops, d, s);                   \
    }                                                                              \
    }
