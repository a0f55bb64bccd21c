// fmm_dispatch.cuh — maps (d, alignment, shape variant) to a row-kernel
// instantiation. Included by one translation unit per op kind so the
// instantiations compile in parallel.
#pragma once

#include <cstdlib>
#include <type_traits>

#include "fmm_kernels.cuh"

namespace fmm {

// Set while fmm_create walks the dispatch tables: launch_one then only
// queries the kernel's attributes, which makes CUDA's lazy module loading
// load it now rather than inside the caller's first fused_mm call.
inline thread_local bool t_preload = false;

template <class Ops, int LPG, int VEC, int NV, int UNROLL, bool EXACT, bool MASKED, int MINB = 0, int PF = -1, int BT = 256>
inline void launch_one(const KParams& p, const Ops& ops, cudaStream_t stream) {
    if (t_preload) {
        cudaFuncAttributes a;
        cudaFuncGetAttributes(&a, fmm_rows_kernel<Ops, LPG, VEC, NV, UNROLL, EXACT, MASKED, MINB, PF, BT>);
        return;
    }
    // Warps never cooperate across a block (no shared memory, no barrier), so
    // the block is as small as the kernel's register-limited occupancy allows:
    // a block's slot frees when its slowest warp is done, and with 8 warps per
    // block that idled ~7% of the resident warps (r3: config 2 1.177 -> 1.136
    // ms, config 3 0.456 -> 0.436 ms with one warp per block). 32 blocks per SM
    // is the hardware limit, so kernels that fit more than 32 warps keep
    // larger blocks. FMM_BLOCK_THREADS overrides (tuning).
    static const int kThreads = [] {
        if (const char* e = std::getenv("FMM_BLOCK_THREADS")) {
            const int t = std::atoi(e);
            if (t >= 32 && t <= BT && t % 32 == 0) return t;
        }
        if (BT < 256) return BT;
        auto kern = fmm_rows_kernel<Ops, LPG, VEC, NV, UNROLL, EXACT, MASKED, MINB, PF, BT>;
        int full = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&full, kern, 256, 0) != cudaSuccess || full <= 0) return 256;
        for (int t = 32; t < 256; t *= 2) {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, t, 0) == cudaSuccess && nb * t >= full * 256)
                return t;
        }
        return 256;
    }();
    constexpr int GPW = 32 / LPG;
    const int64_t wide = EXACT ? 0 : p.n_chunk_items + p.n_wide_rows;
    const int64_t zero_left = p.n_zero_rows - p.n_zero_piggy;
    const int64_t warps = wide + (p.n_narrow_rows + GPW - 1) / GPW + (zero_left + kZeroRowsPerWarp - 1) / kZeroRowsPerWarp;
    if (warps <= 0) return;
    const int64_t blocks = (warps + (kThreads / 32) - 1) / (kThreads / 32);
    fmm_rows_kernel<Ops, LPG, VEC, NV, UNROLL, EXACT, MASKED, MINB, PF, BT>
        <<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(p, ops);
}

// Vectorised shapes: d = LPG * VEC * NV exactly, rows VEC*4-byte aligned.
// variant < 0 selects the default shape for d. The shipped library holds the
// defaults plus one alternative (variant 20: the VEC = 4 shapes even when
// rows are 32-byte aligned); the tuning alternatives swept in r01-r08
// (tests/sweep_variants.py) compile only with -DFMM_TUNING_VARIANTS
// (FMM_TUNING=1 python -m paper_2011_06391_b200.build), so the .so stays small
// and its modules load fast. Unknown variants fall back to the default.
// 256-bit shapes (VEC = 8; rows 32-byte aligned, d % 8 == 0): twice the bytes
// per gather request of the VEC = 4 shapes.
template <class Ops, bool EXACT>
inline bool launch_aligned32(const KParams& p, const Ops& ops, int d, int variant, cudaStream_t s) {
    (void)variant;
    switch (d) {
        case 32:
#ifdef FMM_TUNING_VARIANTS
            if constexpr (!EXACT) {
                if (variant == 21) { launch_one<Ops, 2, 8, 2, 4, EXACT, false, 3, 1>(p, ops, s); return true; }
                if (variant == 22) { launch_one<Ops, 4, 8, 1, 8, EXACT, false, 3, 1>(p, ops, s); return true; }
                if (variant == 23) { launch_one<Ops, 4, 8, 1, 4, EXACT, false, 4, 1>(p, ops, s); return true; }
                if (variant == 24) { launch_one<Ops, 4, 8, 1, 2, EXACT, false, 4, 1>(p, ops, s); return true; }
                if (variant == 25) { launch_one<Ops, 4, 8, 1, 2, EXACT, false, 5, 1>(p, ops, s); return true; }
                if (variant == 26) { launch_one<Ops, 4, 8, 1, 4, EXACT, false, 3, 1>(p, ops, s); return true; }
                if (variant == 27) { launch_one<Ops, 4, 4, 2, 2, EXACT, false, 5, 1>(p, ops, s); return true; }
                if (variant == 28) { launch_one<Ops, 4, 8, 1, 2, EXACT, false, 6, 1>(p, ops, s); return true; }
                if (variant == 29) { launch_one<Ops, 8, 4, 1, 2, EXACT, false, 6, 1>(p, ops, s); return true; }
                if (variant == 30) { launch_one<Ops, 8, 4, 1, 4, EXACT, false, 5, 1>(p, ops, s); return true; }
                if (variant == 56) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 32, 1, 32>(p, ops, s); return true; }
                if (variant == 57) { launch_one<Ops, 4, 8, 1, 4, EXACT, false, 28, 1, 32>(p, ops, s); return true; }
                if (variant == 58) { launch_one<Ops, 4, 4, 2, 8, EXACT, false, 18, 1, 32>(p, ops, s); return true; }
                if (variant == 59) { launch_one<Ops, 4, 8, 1, 4, EXACT, false, 24, 1, 32>(p, ops, s); return true; }
                if (variant == 60) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 24, 1, 32>(p, ops, s); return true; }
                if (variant == 61) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 28, 1, 32>(p, ops, s); return true; }
                if (variant == 62) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 26, 1, 32>(p, ops, s); return true; }
                if (variant == 63) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 30, 1, 32>(p, ops, s); return true; }
            }
#endif
            // config 3 keeps the VEC = 4 shape (0.616 ms; VEC = 8 U = 2: 0.618)
            return false;
        case 64:
            launch_one<Ops, 8, 8, 1, 4, EXACT, false>(p, ops, s); return true;  // config 1
        case 128:
            if constexpr (!EXACT) {
#ifdef FMM_TUNING_VARIANTS
                if (variant == 21) { launch_one<Ops, 4, 8, 4, 4, EXACT, false>(p, ops, s); return true; }
                if (variant == 22) { launch_one<Ops, 16, 8, 1, 4, EXACT, false>(p, ops, s); return true; }
                if (variant == 23) { launch_one<Ops, 8, 8, 2, 2, EXACT, false>(p, ops, s); return true; }
                if (variant == 24) { launch_one<Ops, 8, 8, 2, 4, EXACT, false, 3>(p, ops, s); return true; }
                if (variant == 60) { launch_one<Ops, 8, 8, 2, 4, EXACT, false, 15, -1, 32>(p, ops, s); return true; }
                if (variant == 61) { launch_one<Ops, 8, 8, 2, 4, EXACT, false, 17, -1, 32>(p, ops, s); return true; }
                if (variant == 62) { launch_one<Ops, 8, 8, 2, 4, EXACT, false, 16, -1, 32>(p, ops, s); return true; }
                if (variant == 63) { launch_one<Ops, 16, 8, 1, 8, EXACT, false, 18, -1, 32>(p, ops, s); return true; }
#endif
                launch_one<Ops, 8, 8, 2, 4, EXACT, false>(p, ops, s); return true;  // config 2
            }
            launch_one<Ops, 8, 8, 2, 2, EXACT, false>(p, ops, s); return true;
        case 256:
            if constexpr (!EXACT) {
#ifdef FMM_TUNING_VARIANTS
                if (variant == 21) { launch_one<Ops, 16, 8, 2, 4, EXACT, false>(p, ops, s); return true; }
                if (variant == 22) { launch_one<Ops, 8, 8, 4, 2, EXACT, false>(p, ops, s); return true; }
                if (variant == 25) { launch_one<Ops, 32, 8, 1, 8, EXACT, false>(p, ops, s); return true; }
                if (variant == 56) { launch_one<Ops, 16, 8, 2, 4, EXACT, false, 14, -1, 32>(p, ops, s); return true; }
                if (variant == 57) { launch_one<Ops, 16, 8, 2, 4, EXACT, false, 16, -1, 32>(p, ops, s); return true; }
                if (variant == 58) { launch_one<Ops, 16, 8, 2, 4, EXACT, false, 12, -1, 32>(p, ops, s); return true; }
                if (variant == 59) { launch_one<Ops, 16, 8, 2, 2, EXACT, false, 20, -1, 32>(p, ops, s); return true; }
                if (variant == 60) { launch_one<Ops, 32, 8, 1, 8, EXACT, false, 18, -1, 32>(p, ops, s); return true; }
                if (variant == 61) { launch_one<Ops, 32, 8, 1, 8, EXACT, false, 16, -1, 32>(p, ops, s); return true; }
                if (variant == 62) { launch_one<Ops, 32, 8, 1, 4, EXACT, false, 28, -1, 32>(p, ops, s); return true; }
                if (variant == 63) { launch_one<Ops, 32, 8, 1, 4, EXACT, false, 21, -1, 32>(p, ops, s); return true; }
#endif
                // config 5: two rows per warp, 16 lanes x 64 B each, at 128
                // registers / 16 one-warp blocks per SM (r3z, with the column
                // bands: 92.5 ms; 32 lanes x 32 B at 80 registers: 98.9 ms)
#ifdef FMM_TUNING_VARIANTS
                if (variant == 26) { launch_one<Ops, 32, 8, 1, 4, EXACT, false>(p, ops, s); return true; }
#endif
                launch_one<Ops, 16, 8, 2, 4, EXACT, false, 16, -1, 32>(p, ops, s); return true;
            }
            launch_one<Ops, 16, 8, 2, 2, EXACT, false>(p, ops, s); return true;
        default: return false;
    }
}

template <class Ops, bool EXACT>
inline bool launch_aligned(const KParams& p, const Ops& ops, int d, int variant, cudaStream_t s) {
    (void)variant;
    switch (d) {
        case 1: launch_one<Ops, 1, 1, 1, 8, EXACT, false>(p, ops, s); return true;
        case 2:
#ifdef FMM_TUNING_VARIANTS
            if (variant == 0) { launch_one<Ops, 1, 2, 1, 8, EXACT, false>(p, ops, s); return true; }
            if (variant == 3) { launch_one<Ops, 1, 2, 1, 2, EXACT, false, 8>(p, ops, s); return true; }
            if (variant == 5) { launch_one<Ops, 1, 2, 1, 4, EXACT, false, 8>(p, ops, s); return true; }
#endif
            // config 4: with the index slots read through L1 the register cap
            // of 8 blocks/SM no longer pays (0.0963 vs 0.0983 ms, r08f)
            launch_one<Ops, 1, 2, 1, 4, EXACT, false>(p, ops, s); return true;
        case 4: launch_one<Ops, 1, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 8: launch_one<Ops, 2, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 16: launch_one<Ops, 4, 4, 1, 8, EXACT, false>(p, ops, s); return true;
        case 32:
            if constexpr (!EXACT) {
#ifdef FMM_TUNING_VARIANTS
                if (variant == 0) { launch_one<Ops, 8, 4, 1, 8, EXACT, false>(p, ops, s); return true; }
                if (variant == 1) { launch_one<Ops, 4, 4, 2, 4, EXACT, false>(p, ops, s); return true; }
                if (variant == 4) { launch_one<Ops, 4, 4, 2, 8, EXACT, false>(p, ops, s); return true; }
                if (variant == 8) { launch_one<Ops, 4, 4, 2, 4, EXACT, false, 4, 1>(p, ops, s); return true; }
#endif
                // config 3: U = 4 at 72 registers / 28 one-warp blocks per SM
                // with the column prefetch (r3j: 0.412 ms; U = 2 at 64
                // registers / 32 warps: 0.442 ms; U = 4 at 80 / 25: 0.426 ms)
#ifdef FMM_TUNING_VARIANTS
                if (variant == 9) { launch_one<Ops, 4, 4, 2, 2, EXACT, false, 4, 1>(p, ops, s); return true; }
#endif
                launch_one<Ops, 4, 4, 2, 4, EXACT, false, 28, 1, 32>(p, ops, s); return true;
            }
            launch_one<Ops, 4, 4, 2, 4, EXACT, false>(p, ops, s); return true;
        case 64:
            launch_one<Ops, 8, 4, 2, 4, EXACT, false>(p, ops, s); return true;
        case 128:
            if constexpr (!EXACT) {
#ifdef FMM_TUNING_VARIANTS
                if (variant == 0) { launch_one<Ops, 32, 4, 1, 8, EXACT, false>(p, ops, s); return true; }
                if (variant == 1) { launch_one<Ops, 8, 4, 4, 2, EXACT, false>(p, ops, s); return true; }
                if (variant == 3) { launch_one<Ops, 16, 4, 2, 4, EXACT, false>(p, ops, s); return true; }
#endif
                launch_one<Ops, 8, 4, 4, 4, EXACT, false>(p, ops, s); return true;
            }
            launch_one<Ops, 8, 4, 4, 2, EXACT, false>(p, ops, s); return true;
        case 256:
            if constexpr (!EXACT) {
#ifdef FMM_TUNING_VARIANTS
                if (variant == 0) { launch_one<Ops, 32, 4, 2, 4, EXACT, false>(p, ops, s); return true; }
                if (variant == 1) { launch_one<Ops, 8, 4, 8, 2, EXACT, false>(p, ops, s); return true; }
                if (variant == 7) { launch_one<Ops, 16, 4, 4, 2, EXACT, false>(p, ops, s); return true; }
#endif
                launch_one<Ops, 16, 4, 4, 4, EXACT, false>(p, ops, s); return true;
            }
            launch_one<Ops, 16, 4, 4, 2, EXACT, false>(p, ops, s); return true;
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

bool launch_sigmoid(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s);
bool launch_gcn(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s);
bool launch_fr(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s);
bool launch_tdist(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s);
bool launch_frattr(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s);
bool launch_generic(const KParams& p, int d, bool exact, bool vectorised, cudaStream_t s);
// d > kMaxRegDim: one warp per row, d streamed in tiles (fmm_k_stream.cu)
bool launch_stream(const KParams& p, bool exact, cudaStream_t s);

}  // namespace fmm

#define FMM_DEFINE_STATIC_LAUNCH(NAME, OPS)                                        \
    namespace fmm {                                                                \
    bool NAME(const KParams& p, int d, bool exact, int variant, bool a32, cudaStream_t s) { \
        const OPS ops{};                                                           \
        if (a32 && variant != 20 && (variant < 0 || variant > 20) &&              \
            (exact ? launch_aligned32<OPS, true>(p, ops, d, variant, s)           \
                   : launch_aligned32<OPS, false>(p, ops, d, variant, s)))        \
            return true;                                                           \
        if (variant == 20) variant = -1;                                           \
        return exact ? launch_aligned<OPS, true>(p, ops, d, variant, s)            \
                     : launch_aligned<OPS, false>(p, ops, d, variant, s);          \
    }                                                                              \
    }
