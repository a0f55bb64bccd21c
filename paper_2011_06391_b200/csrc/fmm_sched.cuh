// fmm_sched.cuh — persistent, cp.async-pipelined FusedMM row kernel
// (fast scheme, d in {32, 64, 128, 256}).
//
// The row kernel of fmm_kernels.cuh holds its in-flight gathers in
// registers, which caps occupancy (~14 warps/SM at d=128) and leaves each
// warp idle while it computes: the profile is latency-bound
// (long_scoreboard). Here every warp is persistent (one 8-warp block per SM)
// and streams a precomputed list of work items per lane group; neighbour rows
// y_v (and x_u at the first step of an item) are copied global->shared with
// cp.async (LDGSTS, no registers held in flight) S-1 steps ahead of the step
// being consumed, so the memory system always has ~(S-1)*U*GPW rows per warp
// in flight while the warp computes. Each lane copies and later reads back
// only its own 16-byte pieces of every row, so no cross-lane shared-memory
// synchronisation is needed (cp.async.wait_group per thread suffices).
//
// Items are whole rows (degree <= the plan's chunk size) or fixed-size chunks of
// heavy rows, assigned to lane groups longest-first by the host
// (fmm_plan.cpp build_group_schedule); per item the group folds its edges in
// storage order exactly like update_u (kernel.hpp:92-106). Empty rows are
// written with the AOP identity in a prologue.
#pragma once

#include "fmm_kernels.cuh"

namespace fmm {

struct SchedParams {
    const int32_t* col;               // shard-local edge columns
    const float* val;                 // a_uv or nullptr
    const float* X;                   // x_u = X + (row0 + r) * d
    const float* Y;
    float* Z;                         // z_r = Z + r * d
    float* partial;                   // chunk partials
    const int32_t* group_item_begin;  // per lane group, G+1
    const int4* items;                // {row or slot, e_begin, n, chunk ? row+1 : 0}
    const int32_t* warp_steps;        // steps per warp
    const int32_t* empty_rows;
    int64_t n_empty;
    int64_t row0;
    int d;
    int vop, rop, sop, mop, aop;
    float alpha, k;
};

enum : int { kMetaFirst = 1, kMetaLast = 2, kMetaChunk = 4, kMetaIdle = 8 };

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    const int n = valid ? 16 : 0;  // src-size 0: zero-fill, no global read
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int LPG, int NV, int U, int S>
struct SchedShape {
    static constexpr int GPW = 32 / LPG;
    static constexpr int RF = LPG * NV;          // float4 per row
    static constexpr int kWarps = 8;
    static constexpr int ring_f4 = S * GPW * (U + 1) * RF;  // per warp (slot U = x row)
    static constexpr size_t smem_bytes =
        static_cast<size_t>(kWarps) * (ring_f4 * 16 + S * 32 * 16 + S * 32 * 4);
};

template <class Ops, int LPG, int NV, int U, int S>
__global__ void __launch_bounds__(256, 1)
fmm_sched_kernel(const SchedParams p, const Ops ops) {
    using Sh = SchedShape<LPG, NV, U, S>;
    constexpr int GPW = Sh::GPW;
    constexpr int RF = Sh::RF;
    constexpr int NE = NV * 4;
    constexpr int d = LPG * NV * 4;
    static_assert(U <= LPG, "one column per lane per step");

    extern __shared__ float4 smem[];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPG - 1);
    const int g = lane / LPG;
    const int gbase = lane & ~(LPG - 1);
    const int W = gridDim.x * Sh::kWarps;
    const int w = blockIdx.x * Sh::kWarps + wib;

    float4* ring = smem + wib * Sh::ring_f4;  // [S][GPW][U+1][RF]
    int4* rmeta = reinterpret_cast<int4*>(smem + Sh::kWarps * Sh::ring_f4) + wib * S * 32;
    float* rval = reinterpret_cast<float*>(reinterpret_cast<int4*>(smem + Sh::kWarps * Sh::ring_f4) +
                                           Sh::kWarps * S * 32) + wib * S * 32;

    const float ident = aop_identity(ops);
    const bool need_x = ops.vop() != FMM_VOP_SEL2ND;
    const bool has_val = p.val != nullptr;

    // ---- empty rows: z = AOP identity (update_u with no neighbours)
    for (int64_t i = static_cast<int64_t>(w) * GPW + g; i < p.n_empty; i += static_cast<int64_t>(W) * GPW) {
        float* out = p.Z + static_cast<int64_t>(p.empty_rows[i]) * d;
#pragma unroll
        for (int i4 = 0; i4 < NV; ++i4)
            reinterpret_cast<float4*>(out)[i4 * LPG + gl] = make_float4(ident, ident, ident, ident);
    }

    const int T = p.warp_steps[w];
    if (T == 0) return;

    // ---- issue cursor (identical in every lane of a group)
    const int G = w * GPW + g;
    int it = p.group_item_begin[G];
    const int it_end = p.group_item_begin[G + 1];
    // item descriptors are read through L1 (8 per 128-byte line, the next line
    // prefetched) so advancing to the next item never waits on L2
    auto fetch_item = [&](int i) {
        return i < it_end ? __ldg(p.items + i) : make_int4(-1, 0, 0, 0);
    };
    int4 cur = fetch_item(it);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p.items + it + 8));
    int pos = 0;
    // columns (and a_uv) of the step about to be issued, one per lane gl < U
    int c_pend = -1;
    float a_pend = 1.0f;
    auto load_cols = [&]() {
        c_pend = -1;
        a_pend = 1.0f;
        if (cur.x >= 0 && gl < U && pos + gl < cur.z) {
            // L1-allocating: the next steps of the item read the same line
            c_pend = __ldg(p.col + cur.y + pos + gl);
            if (has_val) a_pend = __ldg(p.val + cur.y + pos + gl);
        }
    };
    load_cols();

    auto issue = [&](int s) {
        const int slot = s % S;
        float4* base = ring + (slot * GPW + g) * (U + 1) * RF;
        int flags = kMetaIdle, valid = 0, ref = 0;
        // shuffles stay outside the per-group branch (all 32 lanes converge)
        int vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) vv[u] = __shfl_sync(0xffffffffu, c_pend, gbase + u);
        if (s < T && cur.x >= 0) {
            flags = (pos == 0 ? kMetaFirst : 0) | (pos + U >= cur.z ? kMetaLast : 0) | (cur.w ? kMetaChunk : 0);
            ref = cur.x;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = vv[u];
                const bool ok = v >= 0;
                valid |= ok ? (1 << u) : 0;
                const float4* src = reinterpret_cast<const float4*>(p.Y + static_cast<int64_t>(ok ? v : 0) * d);
#pragma unroll
                for (int i4 = 0; i4 < NV; ++i4)
                    cp_async16(base + u * RF + i4 * LPG + gl, src + i4 * LPG + gl, ok);
            }
            if (pos == 0 && need_x) {
                // rows carry their id in .x; chunks carry the partial slot in .x
                // and their row + 1 in .w
                const int64_t xrow = cur.w ? cur.w - 1 : cur.x;
                const float4* xs = reinterpret_cast<const float4*>(p.X + (p.row0 + xrow) * d);
#pragma unroll
                for (int i4 = 0; i4 < NV; ++i4) cp_async16(base + U * RF + i4 * LPG + gl, xs + i4 * LPG + gl, true);
            }
            rval[slot * 32 + lane] = a_pend;
            // advance the cursor by one step
            pos += U;
            if (pos >= cur.z) {
                ++it;
                cur = fetch_item(it);
                pos = 0;
                if ((it & 7) == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.items + it + 8));
            }
        }
        rmeta[slot * 32 + lane] = make_int4(ref, flags, valid, 0);
        cp_async_commit();
        load_cols();
    };

#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) issue(s);

    float x[NE], z[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) { x[e] = 0.0f; z[e] = ident; }
    bool elem_ok[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) elem_ok[i] = true;

#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        issue(t + S - 1);
        cp_async_wait<S - 1>();
        const int slot = t % S;
        const int4 meta = rmeta[slot * 32 + lane];
        const float4* base = ring + (slot * GPW + g) * (U + 1) * RF;
        if (meta.y & kMetaFirst) {
#pragma unroll
            for (int e = 0; e < NE; ++e) z[e] = ident;
            if (need_x) {
#pragma unroll
                for (int i4 = 0; i4 < NV; ++i4) {
                    const float4 v = base[U * RF + i4 * LPG + gl];
                    x[i4 * 4 + 0] = v.x; x[i4 * 4 + 1] = v.y; x[i4 * 4 + 2] = v.z; x[i4 * 4 + 3] = v.w;
                }
            }
        }
        float y[U][NE];
        float a[U];
        bool ok[U];
        const float av = rval[slot * 32 + lane];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int i4 = 0; i4 < NV; ++i4) {
                const float4 v = base[u * RF + i4 * LPG + gl];
                y[u][i4 * 4 + 0] = v.x; y[u][i4 * 4 + 1] = v.y; y[u][i4 * 4 + 2] = v.z; y[u][i4 * 4 + 3] = v.w;
            }
            a[u] = has_val ? __shfl_sync(0xffffffffu, av, gbase + u) : 1.0f;
            ok[u] = (meta.z >> u) & 1;
        }
        KParams kp{};
        kp.alpha = p.alpha;
        kp.k = p.k;
        consume_edges<Ops, LPG, 4, NV, U, false, false>(ops, kp, x, z, y, a, ok, elem_ok);
        if ((meta.y & kMetaLast) && !(meta.y & kMetaIdle)) {
            float* out = (meta.y & kMetaChunk) ? p.partial + static_cast<int64_t>(meta.x) * d
                                               : p.Z + static_cast<int64_t>(meta.x) * d;
#pragma unroll
            for (int i4 = 0; i4 < NV; ++i4)
                reinterpret_cast<float4*>(out)[i4 * LPG + gl] =
                    make_float4(z[i4 * 4 + 0], z[i4 * 4 + 1], z[i4 * 4 + 2], z[i4 * 4 + 3]);
        }
    }
    cp_async_wait<0>();
}

// Launch one instantiation persistently: gridDim = #SMs, 8 warps per block.
template <class Ops, int LPG, int NV, int U, int S>
inline bool launch_sched_one(const SchedParams& p, const Ops& ops, int num_sms, cudaStream_t s) {
    using Sh = SchedShape<LPG, NV, U, S>;
    static bool configured = false;
    if (!configured) {
        if (cudaFuncSetAttribute(fmm_sched_kernel<Ops, LPG, NV, U, S>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Sh::smem_bytes)) != cudaSuccess)
            return false;
        configured = true;
    }
    fmm_sched_kernel<Ops, LPG, NV, U, S><<<num_sms, 256, Sh::smem_bytes, s>>>(p, ops);
    return true;
}

// Shape per d: (LPG, NV, U, S). Mirrored on the host by sched_shape_for().
// variant 0 is the default shape; variant 1 an alternative (tuning).
template <class Ops>
inline bool launch_sched(const SchedParams& p, const Ops& ops, int d, int variant, int num_sms, cudaStream_t s) {
    switch (d) {
        case 32: return variant == 1 ? launch_sched_one<Ops, 4, 2, 4, 2>(p, ops, num_sms, s)
                                     : launch_sched_one<Ops, 4, 2, 4, 4>(p, ops, num_sms, s);
        case 64: return launch_sched_one<Ops, 8, 2, 4, 4>(p, ops, num_sms, s);
        case 128: return variant == 1 ? launch_sched_one<Ops, 8, 4, 4, 2>(p, ops, num_sms, s)
                                      : launch_sched_one<Ops, 8, 4, 2, 4>(p, ops, num_sms, s);
        case 256: return launch_sched_one<Ops, 16, 4, 2, 4>(p, ops, num_sms, s);
        default: return false;
    }
}

// Host mirror of launch_sched's shapes: lane groups per warp and U.
inline bool sched_shape_for(int d, int variant, int* gpw, int* u) {
    switch (d) {
        case 32: *gpw = 8; *u = 4; return true;
        case 64: *gpw = 4; *u = 4; return true;
        case 128: *gpw = 4; *u = variant == 1 ? 4 : 2; return true;
        case 256: *gpw = 2; *u = 2; return true;
        default: return false;
    }
}

bool launch_sched_sigmoid(const SchedParams& p, int d, int variant, int num_sms, cudaStream_t s);
bool launch_sched_tdist(const SchedParams& p, int d, int variant, int num_sms, cudaStream_t s);
bool launch_sched_fr(const SchedParams& p, int d, int variant, int num_sms, cudaStream_t s);

}  // namespace fmm
