// fmm_k_stream.cu — rows with d > kMaxRegDim (1024): the d dimension is
// streamed in tiles instead of held in registers.
//
// The reference runs any d: the blocked kernels cover the first
// kBlockedDimLimit columns and a second sweep over the row's neighbours
// streams the rest (row_tail_streamed, kernel.hpp:192-225); the generic path
// (update_u, kernel.hpp:81-107) keeps 2d scratch. Here one warp owns one row:
//   scalar message (ROP != NOOP): pass A folds, per edge in storage order,
//     s = ROP over all d of VOP(x_u, y_v) (lane-strided partials + butterfly),
//     h = SOP(s), written to a per-edge scratch (hbuf, one float per edge of
//     the shard); pass B walks z_u in tiles of 32 x 8 columns held in
//     registers and, per tile, folds every edge in storage order with the
//     same MOP/AOP arithmetic as the row kernels (consume_edges);
//   vector message (ROP == NOOP): pass B alone (t = SOP(VOP(x, y))
//     elementwise), so the exact scheme stays bit-identical to update_u
//     (per element: sequential storage-order fold, no contraction).
// Rows come heavy-first from the shard's item list; split rows are not used.
#include "fmm_dispatch.cuh"

namespace fmm {
namespace {

constexpr int kTile = 8;  // columns per lane per tile (32 x 8 = 256 per warp)
constexpr int kUE = 4;    // edges in flight per warp

// z (+)= w with the row kernels' fused forms on the fast scheme
template <bool EXACT>
__device__ __forceinline__ float fold_edge(const DOps& ops, const KParams& p, float z, float x, float y, float a,
                                           float h, bool scalar) {
    if (ops.aop() == FMM_AOP_ASUM && ops.mop() != FMM_MOP_SEL2ND) {
        if (scalar) {
            if (ops.mop() == FMM_MOP_MUL_VOP) {
                const float t = vop_apply<EXACT>(ops, x, y);
                if constexpr (!EXACT) return fmaf(a * h, t, z);
                return fadd<EXACT>(z, fmul<EXACT>(a, fmul<EXACT>(h, t)));
            }
            return fmac<EXACT>(z, h, y);
        }
        float t = vop_apply<EXACT>(ops, x, y);
        t = sop_apply<EXACT>(ops, t, p.alpha, p.k, p.kinv);
        return fmac<EXACT>(z, a, t);
    }
    float w;
    if (ops.mop() == FMM_MOP_SEL2ND) {
        w = y;
    } else if (scalar) {
        w = ops.mop() == FMM_MOP_MUL_VOP ? fmul<EXACT>(a, fmul<EXACT>(h, vop_apply<EXACT>(ops, x, y)))
                                         : fmul<EXACT>(h, y);
    } else {
        float t = vop_apply<EXACT>(ops, x, y);
        t = sop_apply<EXACT>(ops, t, p.alpha, p.k, p.kinv);
        w = fmul<EXACT>(a, t);
    }
    return aop_apply<EXACT>(ops, z, w);
}

template <bool EXACT>
__global__ void __launch_bounds__(256) fmm_stream_kernel(const KParams p, const DOps ops) {
    const int lane = threadIdx.x & 31;
    const int64_t wi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (wi >= p.n_narrow_rows) return;
    const int4 it = __ldg(p.items + wi);
    const int64_t r = it.x;
    const int64_t e0 = static_cast<int64_t>(static_cast<uint32_t>(it.y)) | (static_cast<int64_t>(it.z) << 32);
    const int64_t n = it.w;
    const int d = p.d;
    const float* xr = p.X + (p.row0 + r) * static_cast<int64_t>(d);
    const bool scalar = ops.rop() != FMM_ROP_NOOP;
    const bool need_x = ops.vop() != FMM_VOP_SEL2ND;
    const bool has_val = p.val != nullptr;

    if (scalar && n > 0) {
        // pass A: h of every edge of the row
        const bool prod = ops.rop() == FMM_ROP_RMUL;
        for (int64_t k0 = 0; k0 < n; k0 += kUE) {
            const float* yr[kUE];
            float acc[kUE];
#pragma unroll
            for (int u = 0; u < kUE; ++u) {
                const int64_t k = min(k0 + u, n - 1);
                yr[u] = p.Y + static_cast<int64_t>(__ldg(p.col + e0 + k)) * d;
                acc[u] = prod ? 1.0f : 0.0f;
            }
            for (int j = lane; j < d; j += 32) {
                const float x = need_x ? __ldg(xr + j) : 0.0f;
#pragma unroll
                for (int u = 0; u < kUE; ++u) acc[u] = vop_rop_step<EXACT>(ops, acc[u], x, __ldg(yr[u] + j));
            }
#pragma unroll
            for (int u = 0; u < kUE; ++u) {
                float s = prod ? group_prod<32>(acc[u]) : group_sum<32>(acc[u]);
                if (ops.rop() == FMM_ROP_NORM) s = sqrtf(s);
                const float h = sop_apply<EXACT>(ops, s, p.alpha, p.k, p.kinv);
                if (lane == 0 && k0 + u < n) p.hbuf[e0 + k0 + u] = h;
            }
        }
        __syncwarp();  // lane 0's h stores are visible to the warp
    }

    // pass B: z_u in tiles of 32 x kTile columns, edges folded in storage order
    const float ident = aop_identity(ops);
    float* zr = p.Z + r * static_cast<int64_t>(d);
    const unsigned pm = p.n_peer > 0 ? peer_bits(p.peer_mask, r) : 0u;
    for (int t0 = 0; t0 < d; t0 += 32 * kTile) {
        float z[kTile], x[kTile];
#pragma unroll
        for (int i = 0; i < kTile; ++i) {
            const int j = t0 + i * 32 + lane;
            z[i] = ident;
            x[i] = (need_x && j < d) ? __ldg(xr + j) : 0.0f;
        }
        for (int64_t k0 = 0; k0 < n; k0 += kUE) {
            float y[kUE][kTile];
            float a[kUE], h[kUE];
#pragma unroll
            for (int u = 0; u < kUE; ++u) {
                const int64_t k = min(k0 + u, n - 1);
                const int64_t e = e0 + k;
                const float* yr = p.Y + static_cast<int64_t>(__ldg(p.col + e)) * d;
                a[u] = has_val ? __ldg(p.val + e) : 1.0f;
                h[u] = scalar ? p.hbuf[e] : 0.0f;
#pragma unroll
                for (int i = 0; i < kTile; ++i) {
                    const int j = t0 + i * 32 + lane;
                    y[u][i] = j < d ? __ldg(yr + j) : 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < kUE; ++u) {
                if (k0 + u >= n) break;
#pragma unroll
                for (int i = 0; i < kTile; ++i) z[i] = fold_edge<EXACT>(ops, p, z[i], x[i], y[u][i], a[u], h[u], scalar);
            }
        }
#pragma unroll
        for (int i = 0; i < kTile; ++i) {
            const int j = t0 + i * 32 + lane;
            if (j < d) {
                zr[j] = z[i];
                for (int q = 0; q < p.n_peer; ++q)
                    if ((pm >> q) & 1u) p.zpeer[q][r * static_cast<int64_t>(d) + j] = z[i];
            }
        }
    }
}

}  // namespace

bool launch_stream(const KParams& p, bool exact, cudaStream_t s) {
    if (t_preload) {
        cudaFuncAttributes a;
        cudaFuncGetAttributes(&a, exact ? fmm_stream_kernel<true> : fmm_stream_kernel<false>);
        return true;
    }
    if (p.rop != FMM_ROP_NOOP && p.hbuf == nullptr && p.n_narrow_rows > 0) return false;
    const DOps ops{p.vop, p.rop, p.sop, p.mop, p.aop, p.mlp_wx, p.mlp_wy, p.mlp_b};
    if (p.n_narrow_rows <= 0) return true;
    const int64_t blocks = (p.n_narrow_rows + 7) / 8;  // 8 warps (rows) per 256-thread block
    if (exact)
        fmm_stream_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, ops);
    else
        fmm_stream_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, ops);
    return true;
}

}  // namespace fmm
