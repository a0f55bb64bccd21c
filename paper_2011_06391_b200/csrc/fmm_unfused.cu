// fmm_unfused.cu — the UNFUSED GPU pipeline, the baseline the fused kernel is
// measured against.
//
// Restates the reference's two-phase path on the device:
//   sddmm  (reference.hpp:41-123): materialise the per-edge messages H —
//          one scalar per edge when ROP is active, a d-vector per edge
//          otherwise (vop, then sop elementwise);
//   spmm   (reference.hpp:127-155): z_u = AOP over edges of MOP(h_e, y_v, a_uv)
//          — for scalar messages MUL gives h*y_v, i.e. a weighted SpMM with
//          the weights H; for vector messages a_uv*H[e] rows are summed.
// The SpMM phase reuses the row kernels (weights = H, or Y = H with
// column e for vector messages), so the comparison isolates the fusion.
#include "fmm_dispatch.cuh"
#include "fmm_unfused.h"

namespace fmm {

// Edge-parallel: lane group g owns edges [g*kEPG, (g+1)*kEPG) of the CSR
// (balanced whatever the degrees), finds its first row by binary search on
// row_ptr and walks rows as it crosses their ends; each message is written
// once.
constexpr int kEPG = 32;

template <class Ops, int LPG, int NV>
__global__ void __launch_bounds__(256)
fmm_sddmm_kernel(const SddmmParams p, const Ops ops) {
    constexpr int NE = NV * 4;
    constexpr int d = LPG * NE;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPG - 1);
    const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / LPG;
    const int64_t nnz = p.nnz;
    const int64_t e0 = gid * kEPG;
    const bool active = e0 < nnz;
    if (__all_sync(0xffffffffu, !active)) return;
    const int64_t e1 = active ? min(nnz, e0 + kEPG) : e0;
    // r = last row with row_ptr[r] <= e0
    int64_t lo = 0, hi = p.n_rows;
    while (active && hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (p.row_ptr[mid] <= e0) lo = mid; else hi = mid;
    }
    int64_t r = lo;
    int64_t rend = active ? p.row_ptr[r + 1] : 0;
    float x[NE];
    auto load_x = [&]() {
        if (ops.vop() != FMM_VOP_SEL2ND)
#pragma unroll
            for (int i = 0; i < NV; ++i) load_vec<4>(&x[i * 4], p.X + (p.row0 + r) * d + (i * LPG + gl) * 4);
    };
#pragma unroll
    for (int i = 0; i < NE; ++i) x[i] = 0.f;
    if (active) load_x();
    const int n = static_cast<int>(e1 - e0);
    const int nmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
    const bool scalar = ops.rop() != FMM_ROP_NOOP;
    for (int k = 0; k < nmax; ++k) {
        const bool ok = k < n;
        if (ok) {
            bool moved = false;
            while (e0 + k >= rend) {  // skip to the row that owns this edge
                ++r;
                rend = p.row_ptr[r + 1];
                moved = true;
            }
            if (moved) load_x();
        }
        float y[NE];
        const int v = ok ? __ldg(p.col + e0 + k) : 0;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (ok) load_vec<4>(&y[i * 4], p.Y + static_cast<int64_t>(v) * d + (i * LPG + gl) * 4);
            else y[i * 4] = y[i * 4 + 1] = y[i * 4 + 2] = y[i * 4 + 3] = 0.f;
        }
        if (scalar) {
            const bool prod = rop_is_product(ops.rop());
            float acc = prod ? 1.f : 0.f;
#pragma unroll
            for (int e = 0; e < NE; ++e) acc = vop_rop_step<false>(ops, acc, x[e], y[e]);
            acc = prod ? group_prod<LPG>(acc) : group_sum<LPG>(acc);
            if (ops.rop() == FMM_ROP_NORM) acc = sqrtf(acc);
            const float h = sop_apply<false>(ops, acc, p.alpha, p.k);
            if (ok && gl == 0) p.H[e0 + k] = h;
        } else {
            float t[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) t[e] = sop_apply<false>(ops, vop_apply<false>(ops, x[e], y[e]), p.alpha, p.k);
            if (ok)
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    store_vec<4>(p.H + (e0 + k) * d + (i * LPG + gl) * 4, &t[i * 4]);
        }
    }
}

__global__ void fmm_iota_kernel(int32_t* out, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<int32_t>(i);
}

template <class Ops>
bool launch_sddmm_ops(const SddmmParams& p, const Ops& ops, cudaStream_t s) {
    if (p.nnz == 0) return true;
    const int64_t groups = (p.nnz + kEPG - 1) / kEPG;
    auto go = [&](auto kernel, int lpg) {
        const int64_t blocks = (groups * lpg + 255) / 256;
        kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(p, ops);
        return true;
    };
    switch (p.d) {
        case 32: return go(fmm_sddmm_kernel<Ops, 8, 1>, 8);
        case 64: return go(fmm_sddmm_kernel<Ops, 16, 1>, 16);
        case 128: return go(fmm_sddmm_kernel<Ops, 32, 1>, 32);
        case 256: return go(fmm_sddmm_kernel<Ops, 32, 2>, 32);
        default: return false;
    }
}

bool launch_sddmm(const SddmmParams& p, int vop, int rop, int sop, int mop, int aop, cudaStream_t s) {
    if (vop == FMM_VOP_MUL && rop == FMM_ROP_RSUM && sop == FMM_SOP_SIGMOID)
        return launch_sddmm_ops(p, OpsSigmoid{}, s);
    const DOps ops{vop, rop, sop, mop, aop, 0.f, 0.f, 0.f};
    return launch_sddmm_ops(p, ops, s);
}

void launch_iota(int32_t* out, int64_t n, cudaStream_t s) {
    if (n > 0) fmm_iota_kernel<<<148 * 8, 256, 0, s>>>(out, n);
}

}  // namespace fmm
