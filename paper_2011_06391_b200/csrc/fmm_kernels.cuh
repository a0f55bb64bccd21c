// fmm_kernels.cuh — sm_100a FusedMM row kernels.
//
// One lane group of LPR lanes owns one work item (a whole CSR row, or a
// fixed-size chunk of a heavy row). The group keeps x_u and the z_u
// accumulator in registers, streams the row's column indices with one
// coalesced load per lane and broadcasts them with shuffles, gathers the
// neighbour rows y_v with 128-bit loads (UNROLL rows in flight per group),
// reduces the per-edge VOP output across the group with xor-butterflies, and
// stores z_u once. This is the device restatement of
//   fusedmm::update_u            kernel.hpp:81-107  (generic five-slot loop)
//   detail::row_sigmoid_embed    kernel.hpp:118-143
//   detail::row_spmm_gcn         kernel.hpp:145-158
//   detail::row_fr_layout        kernel.hpp:160-190
// with the per-slot arithmetic of ops.hpp:53-187.
//
// Numerics schemes (template flag EXACT):
//   EXACT=true  — no FMA contraction (__fmul_rn/__fadd_rn, the reference is
//                 built with -ffp-contract=off, CMakeLists.txt:25), neighbour
//                 order strictly sequential per row (rows never split), lane-
//                 local reductions in element order. Bit-identical to the
//                 reference whenever the d-reduction is lane-local (LPR == 1)
//                 or absent (SPMM_GCN) — configs 1 and 4.
//   EXACT=false — FMA, heavy rows split into chunks combined in fixed chunk
//                 order (deterministic, independent of the shard count).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fusedmm_cuda.h"

namespace fmm {

constexpr int kMaxPeers = 7;  // 8 GPUs per NVSwitch domain in one process
// Largest d the register-resident row kernels hold (masked shapes: 32 lanes
// x 32 values); beyond it the streamed kernel (fmm_k_stream.cu) tiles d.
constexpr int kMaxRegDim = 1024;
// empty rows one dedicated warp (or, at most, one wide warp) fills
constexpr int kZeroRowsPerWarp = 64;
constexpr int kZeroPerWideMax = 32;

struct PeerOut {
    float* p[kMaxPeers];
    int n;
    const uint8_t* mask;  // per shard-local row: bit q -> peer q reads the row (nullptr: all)
};

// Peers that receive row r (bit q = zpeer[q]); all of them without a mask.
__device__ __forceinline__ unsigned peer_bits(const uint8_t* mask, int64_t r) {
    return mask ? static_cast<unsigned>(__ldg(mask + r)) : 0xffu;
}

struct KParams {
    const int64_t* row_ptr;  // shard-local, rebased to 0, rows+1 entries
    const int32_t* col;      // shard-local edge columns (narrowed to int32)
    const float* val;        // a_uv per edge, or nullptr (all ones)
    const float* X;          // x_u = X + (row0 + r) * d
    const float* Y;          // y_v = Y + v * d
    float* Z;                // z_r = Z + r * d   (r shard-local)
    float* partial;          // chunk partial rows: partial + slot * d
    const int32_t* order;    // rows, heavy first: wide rows then narrow rows
    const int4* items;       // per order slot {row, e0 lo, e0 hi, degree}: one
                             // load replaces order[i] -> row_ptr[r], row_ptr[r+1]
    const int4* chunks;      // chunk items {split-row index, first edge (row-relative), edges, slot}, band-major
    // in-kernel chunk fold: the warp finishing a split row's last chunk
    // (ticket from split_count) folds the row's partials in chunk order
    const int4* split_rows;  // {row, first slot, nchunks, 0}
    unsigned* split_count;   // per split row, zero between launches; nullptr: fold kernel
    int fold_max;            // AOP is AMAX
    int64_t n_chunk_items;
    int64_t n_wide_rows;     // rows a whole warp folds (edges over its groups)
    int64_t n_narrow_rows;   // rows one lane group folds (non-empty ones)
    // empty rows (order slots after the narrow rows) only receive the AOP
    // identity: wide warp w writes slots [w*zero_per_wide, (w+1)*zero_per_wide)
    // of the first n_zero_piggy while it waits for its own x_u / column
    // loads; the rest go to dedicated warps at the end of the grid, each
    // writing kZeroRowsPerWarp rows
    int64_t n_zero_rows;
    int64_t n_zero_piggy;
    int zero_per_wide;
    int64_t row0;
    int chunk;               // edges per chunk (fast scheme)
    int d;
    // dynamic op codes (used by DOps only)
    int vop, rop, sop, mop, aop;
    float alpha, k;
    float kinv;  // 1/k when k is a power of two (exact), else 0
    float mlp_wx, mlp_wy, mlp_b;
    // fused exchange: every final z row is also stored to zpeer[q] + r*d —
    // the other shards' next-iterate buffers, reached over NVLink (P2P) — so
    // the per-iteration all-gather rides on the kernel's own stores
    float* zpeer[kMaxPeers];
    int n_peer;
    // halo exchange: per shard-local row, bit q set iff peer q reads the row
    // (one of its edges points at it); nullptr stores every row to every peer
    const uint8_t* peer_mask;
    // split-row fold may use float4 loads/stores: d % 4 == 0 and Z, partial
    // and every zpeer 16-byte aligned
    int fold_vec4;
    // d > kMaxRegDim, scalar message: one h per edge (streamed kernel)
    float* hbuf;
};

// ---------------------------------------------------------------- op kinds
template <int V, int R, int S, int M, int A>
struct SOps {
    __device__ __forceinline__ int vop() const { return V; }
    __device__ __forceinline__ int rop() const { return R; }
    __device__ __forceinline__ int sop() const { return S; }
    __device__ __forceinline__ int mop() const { return M; }
    __device__ __forceinline__ int aop() const { return A; }
    __device__ __forceinline__ float3 mlp() const { return make_float3(0.f, 0.f, 0.f); }
};
struct DOps {
    int v, r, s, m, a;
    float wx, wy, wb;  // FMM_VOP_MLP weights / bias
    __device__ __forceinline__ int vop() const { return v; }
    __device__ __forceinline__ int rop() const { return r; }
    __device__ __forceinline__ int sop() const { return s; }
    __device__ __forceinline__ int mop() const { return m; }
    __device__ __forceinline__ int aop() const { return a; }
    __device__ __forceinline__ float3 mlp() const { return make_float3(wx, wy, wb); }
};

using OpsSigmoid = SOps<FMM_VOP_MUL, FMM_ROP_RSUM, FMM_SOP_SIGMOID, FMM_MOP_MUL, FMM_AOP_ASUM>;
using OpsGcn = SOps<FMM_VOP_SEL2ND, FMM_ROP_NOOP, FMM_SOP_NOOP, FMM_MOP_MUL, FMM_AOP_ASUM>;
using OpsFr = SOps<FMM_VOP_ADD, FMM_ROP_NORM, FMM_SOP_SCAL, FMM_MOP_MUL, FMM_AOP_ASUM>;
using OpsTdist = SOps<FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_TDIST, FMM_MOP_MUL_VOP, FMM_AOP_ASUM>;
using OpsFrAttr = SOps<FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_SQK, FMM_MOP_MUL_VOP, FMM_AOP_ASUM>;

// ------------------------------------------------------------- arithmetic
template <bool EXACT>
__device__ __forceinline__ float fmul(float a, float b) {
    if constexpr (EXACT) return __fmul_rn(a, b);
    else return a * b;
}
template <bool EXACT>
__device__ __forceinline__ float fadd(float a, float b) {
    if constexpr (EXACT) return __fadd_rn(a, b);
    else return a + b;
}
template <bool EXACT>
__device__ __forceinline__ float fsub(float a, float b) {
    if constexpr (EXACT) return __fsub_rn(a, b);
    else return a - b;
}
// acc + a*b : separate roundings when EXACT (reference: acc += a*b without FMA)
template <bool EXACT>
__device__ __forceinline__ float fmac(float acc, float a, float b) {
    if constexpr (EXACT) return __fadd_rn(acc, __fmul_rn(a, b));
    else return fmaf(a, b, acc);
}

// 1/x for x >= 1 (x may be +inf): rcp.approx refined by one Newton step,
// branch-free, within 1 ulp of the IEEE quotient.
__device__ __forceinline__ float recip_ge1(float x) {
    x = fminf(x, 3.0e38f);  // 1/inf -> 0 without a NaN from the Newton step
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}

template <bool EXACT>
__device__ __forceinline__ float sigmoid_f(float s) {
    if constexpr (EXACT) return 1.0f / (1.0f + expf(-s));
    else return recip_ge1(1.0f + expf(-s));
}

// ops.hpp:58-80, plus the toy MLP hook of apps.hpp:58-64 as FMM_VOP_MLP:
// sigmoid(w_x*x + w_y*y + bias), evaluated left to right without contraction
// on the exact scheme
template <bool EXACT, class Ops>
__device__ __forceinline__ float vop_apply(const Ops& ops, float x, float y) {
    switch (ops.vop()) {
        case FMM_VOP_ADD: return fadd<EXACT>(x, y);
        case FMM_VOP_MUL: return fmul<EXACT>(x, y);
        case FMM_VOP_SEL2ND: return y;
        case FMM_VOP_MLP: {
            const float3 w = ops.mlp();
            return sigmoid_f<EXACT>(fadd<EXACT>(fadd<EXACT>(fmul<EXACT>(w.x, x), fmul<EXACT>(w.y, y)), w.z));
        }
        default: return fsub<EXACT>(x, y);  // FMM_VOP_SUB
    }
}

__device__ __forceinline__ bool rop_is_product(int rop) { return rop == FMM_ROP_RMUL; }

// lane-local step of ops.hpp:82-106 (RSUM / RMUL / NORM / SQNORM)
template <bool EXACT, class Ops>
__device__ __forceinline__ float rop_step(const Ops& ops, float acc, float t) {
    switch (ops.rop()) {
        case FMM_ROP_RMUL: return fmul<EXACT>(acc, t);
        case FMM_ROP_NORM:
        case FMM_ROP_SQNORM: return fmac<EXACT>(acc, t, t);
        default: return fadd<EXACT>(acc, t);  // RSUM
    }
}

// Fused "t = vop(x,y); acc = rop_step(acc, t)" — lets the fast scheme emit one
// FMA per element for the MUL/RSUM dot product.
template <bool EXACT, class Ops>
__device__ __forceinline__ float vop_rop_step(const Ops& ops, float acc, float x, float y) {
    if (ops.vop() == FMM_VOP_MUL && ops.rop() == FMM_ROP_RSUM) return fmac<EXACT>(acc, x, y);
    return rop_step<EXACT>(ops, acc, vop_apply<EXACT>(ops, x, y));
}

// ops.hpp:53-56, 108-121 plus the device extensions TDIST / SQK. Sigmoid is
// 1/(1+exp(-s)) with CUDA's accurate expf (no LUT, no clamp);
// the exact scheme divides with IEEE rounding, the fast one uses recip_ge1.
template <bool EXACT, class Ops>
__device__ __forceinline__ float sop_apply(const Ops& ops, float s, float alpha, float k, float kinv = 0.0f) {
    switch (ops.sop()) {
        case FMM_SOP_SIGMOID: return sigmoid_f<EXACT>(s);
        case FMM_SOP_SCAL: return __fmul_rn(alpha, s);
        case FMM_SOP_TDIST:
            // s >= 0 after a squared / plain norm, so 1+s >= 1
            if (!EXACT && (ops.rop() == FMM_ROP_SQNORM || ops.rop() == FMM_ROP_NORM)) return recip_ge1(1.0f + s);
            return 1.0f / (1.0f + s);
        // s / k; for k a power of two (kinv = 1/k exact and normal) the
        // product s * kinv is the same correctly rounded value in one FMUL
        case FMM_SOP_SQK: return kinv != 0.0f ? __fmul_rn(s, kinv) : __fdiv_rn(s, k);
        default: return s;  // NOOP
    }
}

// ops.hpp:166-182 (AMAX mirrors std::max(acc, w) == (acc < w ? w : acc))
template <bool EXACT, class Ops>
__device__ __forceinline__ float aop_apply(const Ops& ops, float acc, float w) {
    if (ops.aop() == FMM_AOP_AMAX) return (acc < w) ? w : acc;
    return fadd<EXACT>(acc, w);
}

template <class Ops>
__device__ __forceinline__ float aop_identity(const Ops& ops) {
    return ops.aop() == FMM_AOP_AMAX ? -__int_as_float(0x7f800000) : 0.0f;
}

// ------------------------------------------------------------ memory ops
// 32-byte vector (sm_100a 256-bit LDG/STG: LDG.E.ENL2.256). Random row
// gathers served from L2 deliver ~1.7x more bytes per SM with 256-bit than
// with 128-bit requests (profiles/r03_probe_ldg256.log: 19.0 vs 11.2 TB/s).
struct alignas(32) float8v {
    float v[8];
};
template <int VEC> struct VecT;
template <> struct VecT<8> { using T = float8v; };
template <> struct VecT<4> { using T = float4; };
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<1> { using T = float; };

template <int VEC>
__device__ __forceinline__ void load_vec(float* dst, const float* src) {
    if constexpr (VEC == 8) {
        asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(dst[0]), "=f"(dst[1]), "=f"(dst[2]), "=f"(dst[3]), "=f"(dst[4]), "=f"(dst[5]),
                       "=f"(dst[6]), "=f"(dst[7])
                     : "l"(src));
    } else if constexpr (VEC == 4) {
        float4 v = __ldg(reinterpret_cast<const float4*>(src));
        dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;
    } else if constexpr (VEC == 2) {
        float2 v = __ldg(reinterpret_cast<const float2*>(src));
        dst[0] = v.x; dst[1] = v.y;
    } else {
        dst[0] = __ldg(src);
    }
}
template <int VEC>
__device__ __forceinline__ void store_vec(float* dst, const float* src) {
    if constexpr (VEC == 8) {
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "f"(src[0]), "f"(src[1]),
                     "f"(src[2]), "f"(src[3]), "f"(src[4]), "f"(src[5]), "f"(src[6]), "f"(src[7])
                     : "memory");
    } else if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(dst) = make_float4(src[0], src[1], src[2], src[3]);
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<float2*>(dst) = make_float2(src[0], src[1]);
    } else {
        dst[0] = src[0];
    }
}
__device__ __forceinline__ int ld_stream_i32(const int32_t* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

// xor-butterfly over the LPR lanes of a group; every lane ends with the same
// bits (a+b == b+a in IEEE arithmetic), so all lanes agree on h.
template <int LPR>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
template <int LPR>
__device__ __forceinline__ float group_prod(float v) {
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Transposed group reduction of U values over the LPG lanes of a group
// (U <= LPG, both powers of two): stage k (xor offset LPG >> (k+1)) keeps the
// lower or upper half of the values a lane carries, by its lane bit, and adds
// the partner's other half; after log2(U) stages every lane holds the full
// sum of one value, the remaining stages are a plain butterfly. Lane l ends
// with value transposed_value(l); every lane holding it has the same bits.
template <int LPG, int U>
__device__ __forceinline__ float transposed_sum(const float (&s)[U]) {
    const int lane = threadIdx.x & 31;
    float v[U];
#pragma unroll
    for (int i = 0; i < U; ++i) v[i] = s[i];
#pragma unroll
    for (int n = U, o = LPG / 2; o >= 1; o >>= 1) {
        if (n > 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < n / 2; ++i) {
                const float keep = up ? v[i + n / 2] : v[i];
                const float send = up ? v[i] : v[i + n / 2];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
            n /= 2;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
    return v[0];
}
// Lane offset (within the group) that holds value u after transposed_sum.
template <int LPG, int U>
__device__ __forceinline__ constexpr int transposed_lane(int u) {
    int off = 0;
    for (int w = U / 2, o = LPG / 2; w >= 1; w >>= 1, o >>= 1)
        if (u & w) off += o;
    return off;
}

// --------------------------------------------------------------- the kernel
// Per-edge work for U gathered neighbour rows: ROP across the group, SOP,
// MOP, AOP into z (update_u's loop body, kernel.hpp:92-106).
template <class Ops, int LPG, int VEC, int NV, int U, bool EXACT, bool MASKED>
__device__ __forceinline__ void consume_edges(const Ops& ops, const KParams& p, const float (&x)[NV * VEC],
                                              float (&z)[NV * VEC], const float (&y)[U][NV * VEC],
                                              const float (&a)[U], const bool (&ok)[U],
                                              const bool (&elem_ok)[NV]) {
    constexpr int NE = NV * VEC;
    // ASUM accumulations may run predicated (an invalid edge adds +0);
    // AMAX and the exact scheme skip invalid edges explicitly.
    const bool predicated = !EXACT && ops.aop() == FMM_AOP_ASUM;
    if constexpr (VEC % 2 == 0 && !MASKED) {
        // Packed f32x2 path (Blackwell FFMA2/FADD2/FMUL2: two lanes of math per
        // instruction), fast scheme only: scalar messages with ASUM. (The
        // exact scheme stays scalar: ptxas may contract packed mul+add.)
        if (!EXACT && ops.aop() == FMM_AOP_ASUM && ops.rop() != FMM_ROP_NOOP &&
            ops.rop() != FMM_ROP_RMUL && ops.mop() != FMM_MOP_SEL2ND && ops.vop() != FMM_VOP_MLP) {
            float s[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int e = 0; e < NE; e += 2) {
                    const float2 xv = make_float2(x[e], x[e + 1]);
                    const float2 yv = make_float2(y[u][e], y[u][e + 1]);
                    float2& acc = ((e >> 1) & 1) ? acc1 : acc0;
                    if (ops.vop() == FMM_VOP_MUL && ops.rop() == FMM_ROP_RSUM) {
                        acc = __ffma2_rn(xv, yv, acc);
                    } else {
                        float2 t;
                        switch (ops.vop()) {
                            case FMM_VOP_ADD: t = __fadd2_rn(xv, yv); break;
                            case FMM_VOP_MUL: t = __fmul2_rn(xv, yv); break;
                            case FMM_VOP_SEL2ND: t = yv; break;
                            default: t = __ffma2_rn(yv, make_float2(-1.f, -1.f), xv); break;  // x - y
                        }
                        if (ops.rop() == FMM_ROP_RSUM) acc = __fadd2_rn(acc, t);
                        else acc = __ffma2_rn(t, t, acc);  // NORM / SQNORM
                    }
                }
                s[u] = (acc0.x + acc0.y) + (acc1.x + acc1.y);
            }
            // h of every edge: with U <= LPG the U partial dots are reduced
            // "transposed" (each stage halves the values a lane carries, so
            // U-1 + log2(LPG/U) shuffles instead of U*log2(LPG)), each lane
            // evaluates the scalar op for one edge, and the U results are
            // broadcast back; otherwise a butterfly per edge.
            float hv[U];
            if constexpr (LPG >= U && U >= 2 && (U & (U - 1)) == 0) {
                float t = transposed_sum<LPG, U>(s);
                if (ops.rop() == FMM_ROP_NORM) t = sqrtf(t);
                const float hl = sop_apply<EXACT>(ops, t, p.alpha, p.k, p.kinv);
                const int gbase = (threadIdx.x & 31) & ~(LPG - 1);
#pragma unroll
                for (int u = 0; u < U; ++u) hv[u] = __shfl_sync(0xffffffffu, hl, gbase + transposed_lane<LPG, U>(u));
            } else {
                if (LPG > 1) {
#pragma unroll
                    for (int u = 0; u < U; ++u) s[u] = group_sum<LPG>(s[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    float sv = s[u];
                    if (ops.rop() == FMM_ROP_NORM) sv = sqrtf(sv);
                    hv[u] = sop_apply<EXACT>(ops, sv, p.alpha, p.k, p.kinv);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float h = ok[u] ? hv[u] : 0.0f;
                if (ops.mop() == FMM_MOP_MUL_VOP) h *= a[u];
                const float2 h2 = make_float2(h, h);
#pragma unroll
                for (int e = 0; e < NE; e += 2) {
                    const float2 yv = make_float2(y[u][e], y[u][e + 1]);
                    float2 zv = make_float2(z[e], z[e + 1]);
                    if (ops.mop() == FMM_MOP_MUL_VOP) {
                        const float2 xv = make_float2(x[e], x[e + 1]);
                        float2 t;
                        switch (ops.vop()) {
                            case FMM_VOP_ADD: t = __fadd2_rn(xv, yv); break;
                            case FMM_VOP_MUL: t = __fmul2_rn(xv, yv); break;
                            case FMM_VOP_SEL2ND: t = yv; break;
                            default: t = __ffma2_rn(yv, make_float2(-1.f, -1.f), xv); break;
                        }
                        zv = __ffma2_rn(h2, t, zv);
                    } else {
                        zv = __ffma2_rn(h2, yv, zv);
                    }
                    z[e] = zv.x;
                    z[e + 1] = zv.y;
                }
            }
            return;
        }
    }
    if (ops.rop() != FMM_ROP_NOOP) {
        const bool prod = rop_is_product(ops.rop());
        float s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float acc = prod ? 1.0f : 0.0f;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                if (!elem_ok[i]) continue;
#pragma unroll
                for (int c = 0; c < VEC; ++c)
                    acc = vop_rop_step<EXACT>(ops, acc, x[i * VEC + c], y[u][i * VEC + c]);
            }
            s[u] = acc;
        }
        if (LPG > 1) {
#pragma unroll
            for (int u = 0; u < U; ++u) s[u] = prod ? group_prod<LPG>(s[u]) : group_sum<LPG>(s[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float sv = s[u];
            if (ops.rop() == FMM_ROP_NORM) sv = sqrtf(sv);
            float h = sop_apply<EXACT>(ops, sv, p.alpha, p.k, p.kinv);
            if (predicated) {
                h = ok[u] ? h : 0.0f;
            } else if (!ok[u]) {
                continue;
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                float w;
                if (ops.mop() == FMM_MOP_SEL2ND) {
                    w = y[u][e];
                } else if (ops.mop() == FMM_MOP_MUL_VOP) {
                    const float t = vop_apply<EXACT>(ops, x[e], y[u][e]);
                    if (ops.aop() == FMM_AOP_ASUM && !EXACT) {
                        z[e] = fmaf(a[u] * h, t, z[e]);
                        continue;
                    }
                    w = fmul<EXACT>(a[u], fmul<EXACT>(h, t));
                } else {  // MUL: h * y_v, a_uv ignored (ops.hpp:131-137)
                    if (ops.aop() == FMM_AOP_ASUM) {
                        z[e] = fmac<EXACT>(z[e], h, y[u][e]);
                        continue;
                    }
                    w = fmul<EXACT>(h, y[u][e]);
                }
                z[e] = aop_apply<EXACT>(ops, z[e], w);
            }
        }
    } else {
        // vector message: SOP elementwise, MOP with a_uv (ops.hpp:123-127, 150-156)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                float t = vop_apply<EXACT>(ops, x[e], y[u][e]);
                t = sop_apply<EXACT>(ops, t, p.alpha, p.k, p.kinv);
                float w;
                if (ops.mop() == FMM_MOP_SEL2ND) {
                    w = y[u][e];
                } else {
                    if (ops.aop() == FMM_AOP_ASUM) {
                        z[e] = fmac<EXACT>(z[e], a[u], t);
                        continue;
                    }
                    w = fmul<EXACT>(a[u], t);
                }
                z[e] = aop_apply<EXACT>(ops, z[e], w);
            }
        }
    }
}

template <int LPG, int VEC, int NV, int U, bool MASKED>
__device__ __forceinline__ void gather_rows(const float* __restrict__ Y, int d, const int (&v)[U],
                                            const bool (&ok)[U], const bool (&elem_ok)[NV], int gl,
                                            float (&y)[U][NV * VEC]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const float* yr = Y + static_cast<int64_t>(v[u]) * d;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            if (ok[u] && elem_ok[i]) {
                load_vec<VEC>(&y[u][i * VEC], yr + (i * LPG + gl) * VEC);
            } else {
#pragma unroll
                for (int c = 0; c < VEC; ++c) y[u][i * VEC + c] = 0.0f;
            }
        }
    }
}

// AOP identity into the empty rows at order slots [zs, zs + zn) (relative to
// the first empty slot, which follows the narrow rows): lane l fetches row id
// zs + l, the lane groups then store GPW rows per step, to Z and to every
// peer that reads the row.
template <class Ops, int LPG, int VEC, int NV, bool MASKED>
__device__ __forceinline__ void fill_identity_rows(const KParams& p, const Ops& ops, int64_t zs, int zn) {
    constexpr int GPW = 32 / LPG;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPG - 1);
    const int g = lane / LPG;
    const int d = MASKED ? p.d : LPG * VEC * NV;
    const int32_t* zorder = p.order + p.n_wide_rows + p.n_narrow_rows + zs;
    float idv[VEC];
#pragma unroll
    for (int c = 0; c < VEC; ++c) idv[c] = aop_identity(ops);
    for (int b0 = 0; b0 < zn; b0 += 32) {
        const int rid = (b0 + lane < zn) ? __ldg(zorder + b0 + lane) : 0;
        const int lim = min(32, zn - b0);  // warp-uniform
        for (int j = 0; j < lim; j += GPW) {
            const int zr = __shfl_sync(0xffffffffu, rid, j + g);
            if (j + g < lim) {
                const unsigned zpm = p.n_peer > 0 ? peer_bits(p.peer_mask, zr) : 0u;
                float* zo = p.Z + static_cast<int64_t>(zr) * d;
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    if (!MASKED || (i * LPG + gl) * VEC < d) {
                        store_vec<VEC>(zo + (i * LPG + gl) * VEC, idv);
                        for (int q = 0; q < p.n_peer; ++q)
                            if ((zpm >> q) & 1u)
                                store_vec<VEC>(p.zpeer[q] + static_cast<int64_t>(zr) * d + (i * LPG + gl) * VEC, idv);
                    }
            }
        }
    }
}

// Work items, in launch order (heaviest first, LPT-like):
//   [0, n_chunk_items)                 piece of a split row  -> wide warp
//                                      (band-major when the plan cut the heavy
//                                      rows at column-band boundaries)
//   [.., + n_wide_rows)                row order[i]          -> wide warp
//   then narrow rows, GPW = 32/LPG per warp, one per lane group,
//   then warps that only write the AOP identity to empty rows
//   (kZeroRowsPerWarp each; the wide warps take the first n_zero_piggy).
// One warp per block wherever the occupancy allows (launch_one).
// A wide warp spreads its item's edges over the GPW groups round-robin
// (edge k -> group k % GPW), each group folds its edges in storage order,
// and the GPW partial z are combined by an xor-butterfly in fixed order.
// Lane layout: element j = (i*LPG + lane_in_group)*VEC + c.
// MINB = 0 leaves the register budget to ptxas (as __launch_bounds__(256));
// MINB > 0 asks for that many resident blocks of BT threads per SM. Warps are
// independent, so BT = 32 with MINB = w sets the register budget for w warps
// per SM in steps of one warp (d = 32: 72 registers, 28 warps).
template <class Ops, int LPG, int VEC, int NV, int UNROLL, bool EXACT, bool MASKED, int MINB = 0, int PF = -1, int BT = 256>
__global__ void __launch_bounds__(BT, MINB)
fmm_rows_kernel(const KParams p, const Ops ops) {
    constexpr int NE = NV * VEC;
    constexpr int GPW = 32 / LPG;
    constexpr int U = UNROLL;
    static_assert(32 % LPG == 0, "group shape");
    // Fetch column indices one batch ahead on the wide-row fast shapes
    // (config 2: -5%, config 5: -1.5%); for short rows / small d the extra
    // registers cost more than the hidden index latency (measured).
    // PF: -1 = this rule, 0 / 1 = forced (tuning variants)
    constexpr bool kPrefetchCols = PF >= 0 ? (PF == 1) : (!EXACT && !MASKED && (LPG * VEC * NV >= 128));

    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPG - 1);
    const int g = lane / LPG;
    const int gbase = lane & ~(LPG - 1);
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_wide_items = EXACT ? 0 : p.n_chunk_items + p.n_wide_rows;
    const bool wide = warp < n_wide_items;  // warp-uniform
    {
        // warps past the narrow rows only write the AOP identity to empty rows
        const int64_t zw = warp - n_wide_items - (p.n_narrow_rows + GPW - 1) / GPW;
        if (zw >= 0) {
            const int64_t zs = p.n_zero_piggy + zw * kZeroRowsPerWarp;
            if (zs < p.n_zero_rows)
                fill_identity_rows<Ops, LPG, VEC, NV, MASKED>(
                    p, ops, zs, static_cast<int>(min(static_cast<int64_t>(kZeroRowsPerWarp), p.n_zero_rows - zs)));
            return;
        }
    }

    int64_t r = 0, e0 = 0, e1 = 0;
    float* out = nullptr;
    bool active;
    if (wide) {
        active = true;
        if (warp < p.n_chunk_items) {
            const int4 c = __ldg(p.chunks + warp);  // {split-row index, first edge, edges, slot}
            r = __ldg(p.split_rows + c.x).x;
            e0 = p.row_ptr[r] + c.y;
            e1 = e0 + c.z;
            out = p.partial + static_cast<int64_t>(c.w) * (MASKED ? p.d : LPG * VEC * NV);
        } else {
            const int4 it = __ldg(p.items + (warp - p.n_chunk_items));
            r = it.x;
            e0 = static_cast<int64_t>(static_cast<uint32_t>(it.y)) | (static_cast<int64_t>(it.z) << 32);
            e1 = e0 + it.w;
            out = p.Z + r * (MASKED ? p.d : LPG * VEC * NV);
        }
    } else {
        const int64_t idx = (warp - n_wide_items) * GPW + g;
        active = idx < p.n_narrow_rows;
        if (__all_sync(0xffffffffu, !active)) return;
        if (active) {
            const int4 it = __ldg(p.items + (p.n_wide_rows + idx));
            r = it.x;
            e0 = static_cast<int64_t>(static_cast<uint32_t>(it.y)) | (static_cast<int64_t>(it.z) << 32);
            e1 = e0 + it.w;
            out = p.Z + r * (MASKED ? p.d : LPG * VEC * NV);
        }
    }

    const int d = MASKED ? p.d : LPG * VEC * NV;
    const bool need_x = ops.vop() != FMM_VOP_SEL2ND;
    const bool has_val = p.val != nullptr;

    float x[NE], z[NE];
    const float ident = aop_identity(ops);
#pragma unroll
    for (int i = 0; i < NE; ++i) { x[i] = 0.0f; z[i] = ident; }
    bool elem_ok[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) elem_ok[i] = !MASKED || ((i * LPG + gl) * VEC < d);
    // empty rows (38-50% of the R-MAT configs' rows) never read x_u
    if (active && need_x && e1 > e0) {
        const float* xr = p.X + (p.row0 + r) * d;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (elem_ok[i]) load_vec<VEC>(&x[i * VEC], xr + (i * LPG + gl) * VEC);
    }

    if (wide) {
        // ---- one item per warp; edge k of the item goes to group k % GPW
        constexpr int SB = GPW * U;                   // edges per sub-batch
        constexpr int B = SB > 32 ? SB : 32;          // edges per column batch
        constexpr int KPL = B / 32;                   // column slots per lane
        static_assert(SB <= 32 ? (32 % SB == 0) : (SB % 32 == 0), "sub-batch shape");
        const int n = static_cast<int>(e1 - e0);
        int cnext[KPL];
        float anext[KPL];
        auto fetch = [&](int bb) {  // one batch ahead, as in the narrow loop
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int eb = bb + q * 32 + lane;
                cnext[q] = 0;
                anext[q] = 1.0f;
                if (eb < n) {
                    cnext[q] = ld_stream_i32(p.col + e0 + eb);
                    if (has_val) anext[q] = ld_stream_f32(p.val + e0 + eb);
                }
            }
        };
        if constexpr (kPrefetchCols) fetch(0);
        // this warp's share of the empty rows, written while x_u and the first
        // column batch are on their way
        if (p.zero_per_wide > 0) {
            const int64_t zs = warp * p.zero_per_wide;
            if (zs < p.n_zero_piggy)
                fill_identity_rows<Ops, LPG, VEC, NV, MASKED>(
                    p, ops, zs, static_cast<int>(min(static_cast<int64_t>(p.zero_per_wide), p.n_zero_piggy - zs)));
        }
        for (int base = 0; base < n; base += B) {
            if constexpr (!kPrefetchCols) fetch(base);
            int cidx[KPL];
            float aval[KPL];
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                cidx[q] = cnext[q];
                aval[q] = anext[q];
            }
            if constexpr (kPrefetchCols)
                if (base + B < n) fetch(base + B);
            const int cnt = min(B, n - base);
            // SB >= 32: a single sub-batch per column batch (static slots);
            // SB < 32: KPL == 1 and the sub-batch offset s is a run-time value.
#pragma unroll 1
            for (int s = 0; s < B; s += SB) {
                if (s >= cnt) break;
                int v[U];
                float a[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int bq = s + u * GPW;
                    const int slot = KPL == 1 ? 0 : (u * GPW) / 32;
                    const int src = (bq % 32) + g;
                    v[u] = __shfl_sync(0xffffffffu, cidx[slot], src);
                    a[u] = has_val ? __shfl_sync(0xffffffffu, aval[slot], src) : 1.0f;
                    ok[u] = (base + bq + g) < n;
                }
                float y[U][NE];
                gather_rows<LPG, VEC, NV, U, MASKED>(p.Y, d, v, ok, elem_ok, gl, y);
                consume_edges<Ops, LPG, VEC, NV, U, EXACT, MASKED>(ops, p, x, z, y, a, ok, elem_ok);
            }
        }
        // fold the GPW group partials (fixed butterfly order -> deterministic)
        if (GPW > 1) {
            const bool is_max = ops.aop() == FMM_AOP_AMAX;
#pragma unroll
            for (int off = LPG; off < 32; off <<= 1) {
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const float o = __shfl_xor_sync(0xffffffffu, z[e], off);
                    z[e] = is_max ? ((z[e] < o) ? o : z[e]) : z[e] + o;
                }
            }
        }
        // group gg stores vectors i with i % GPW == gg; final rows (not chunk
        // partials) also go straight into the peers' next-iterate buffers
        const bool is_chunk = warp < p.n_chunk_items;  // a split row's partial, not a final row
        const bool to_peers = !is_chunk && p.n_peer > 0;
        const unsigned pm = to_peers ? peer_bits(p.peer_mask, r) : 0u;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if ((i % GPW) == g && elem_ok[i]) {
                store_vec<VEC>(out + (i * LPG + gl) * VEC, &z[i * VEC]);
                if (to_peers)
                    for (int q = 0; q < p.n_peer; ++q)
                        if ((pm >> q) & 1u)
                            store_vec<VEC>(p.zpeer[q] + r * d + (i * LPG + gl) * VEC, &z[i * VEC]);
            }
        if (is_chunk && p.split_count != nullptr) {
            // last chunk of the row to finish folds all its partials, in
            // chunk order per element (deterministic, shard-independent)
            const int si = __ldg(p.chunks + warp).x;
            const int4 sr = p.split_rows[si];
            __threadfence();  // this warp's partial is visible device-wide
            __syncwarp();     // ... every lane's, before lane 0 takes the ticket
            unsigned ticket = 0;
            if (lane == 0) ticket = atomicAdd(p.split_count + si, 1u);
            ticket = __shfl_sync(0xffffffffu, ticket, 0);
            if (ticket + 1 == static_cast<unsigned>(sr.z)) {
                __threadfence();  // acquire: every partial of the row is visible
                const float* base = p.partial + static_cast<int64_t>(sr.y) * d;
                float* zr = p.Z + static_cast<int64_t>(sr.x) * d;
                const float id = aop_identity(ops);
                const bool mx = p.fold_max != 0;
                const unsigned fpm = p.n_peer > 0 ? peer_bits(p.peer_mask, sr.x) : 0u;
                auto f1 = [&](float a, float v) { return mx ? (a < v ? v : a) : __fadd_rn(a, v); };
                if (p.fold_vec4) {
                    // float4 per lane, 8 chunks in flight; per element the
                    // chunks fold in order
                    const int d4 = d >> 2;
                    for (int j4 = lane; j4 < d4; j4 += 32) {
                        float4 acc = make_float4(id, id, id, id);
                        int k = 0;
                        for (; k + 8 <= sr.z; k += 8) {
                            float4 v[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                v[q] = __ldcg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(k + q) * d) + j4);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                acc.x = f1(acc.x, v[q].x); acc.y = f1(acc.y, v[q].y);
                                acc.z = f1(acc.z, v[q].z); acc.w = f1(acc.w, v[q].w);
                            }
                        }
                        for (; k < sr.z; ++k) {
                            const float4 v = __ldcg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(k) * d) + j4);
                            acc.x = f1(acc.x, v.x); acc.y = f1(acc.y, v.y);
                            acc.z = f1(acc.z, v.z); acc.w = f1(acc.w, v.w);
                        }
                        reinterpret_cast<float4*>(zr)[j4] = acc;
                        for (int q = 0; q < p.n_peer; ++q)
                            if ((fpm >> q) & 1u)
                                reinterpret_cast<float4*>(p.zpeer[q] + static_cast<int64_t>(sr.x) * d)[j4] = acc;
                    }
                } else {
                    for (int j = lane; j < d; j += 32) {
                        float acc = id;
                        for (int k = 0; k < sr.z; ++k) acc = f1(acc, __ldcg(base + static_cast<int64_t>(k) * d + j));
                        zr[j] = acc;
                        for (int q = 0; q < p.n_peer; ++q)
                            if ((fpm >> q) & 1u) p.zpeer[q][static_cast<int64_t>(sr.x) * d + j] = acc;
                    }
                }
                if (lane == 0) p.split_count[si] = 0;  // ready for the next launch
            }
        }
        return;
    }

    // ---- narrow: one row per lane group
    {
        constexpr int B = (LPG > U) ? LPG : U;  // edges per column batch
        constexpr int KPL = B / LPG;            // column slots per lane
        const int n = static_cast<int>(e1 - e0);
        const int nmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(n)));
        // column indices are fetched one batch ahead, so the index load of
        // batch k+1 overlaps the gathers of batch k instead of preceding them
        int cnext[KPL];
        float anext[KPL];
        auto fetch = [&](int bb) {
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                const int eb = bb + q * LPG + gl;
                cnext[q] = 0;
                anext[q] = 1.0f;
                if (eb < n) {
                    // a group's index window rarely fills whole sectors and
                    // the next batch (or, with KPL > 1, the lane's next slot)
                    // reads the rest: keep the sectors in L1 so each is
                    // fetched from L2 once (config 4: L2->SM 1.18 -> 0.69 GB)
                    cnext[q] = __ldg(p.col + e0 + eb);
                    if (has_val) anext[q] = __ldg(p.val + e0 + eb);
                }
            }
        };
        if constexpr (kPrefetchCols) fetch(0);
        for (int base = 0; base < nmax; base += B) {
            if constexpr (!kPrefetchCols) fetch(base);
            int cidx[KPL];
            float aval[KPL];
#pragma unroll
            for (int q = 0; q < KPL; ++q) {
                cidx[q] = cnext[q];
                aval[q] = anext[q];
            }
            if constexpr (kPrefetchCols)
                if (base + B < nmax) fetch(base + B);
            const int cnt = min(B, nmax - base);  // warp-uniform
#pragma unroll 1
            for (int u0 = 0; u0 < B; u0 += U) {
                if (u0 >= cnt) break;
                int v[U];
                float a[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int b = u0 + u;
                    v[u] = __shfl_sync(0xffffffffu, cidx[KPL == 1 ? 0 : b / LPG], gbase + (b % LPG));
                    a[u] = has_val ? __shfl_sync(0xffffffffu, aval[KPL == 1 ? 0 : b / LPG], gbase + (b % LPG)) : 1.0f;
                    ok[u] = (base + b) < n;
                }
                float y[U][NE];
                gather_rows<LPG, VEC, NV, U, MASKED>(p.Y, d, v, ok, elem_ok, gl, y);
                consume_edges<Ops, LPG, VEC, NV, U, EXACT, MASKED>(ops, p, x, z, y, a, ok, elem_ok);
            }
        }
        if (active) {
            const unsigned pm = p.n_peer > 0 ? peer_bits(p.peer_mask, r) : 0u;
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if (elem_ok[i]) {
                    store_vec<VEC>(out + (i * LPG + gl) * VEC, &z[i * VEC]);
                    for (int q = 0; q < p.n_peer; ++q)
                        if ((pm >> q) & 1u)
                            store_vec<VEC>(p.zpeer[q] + r * d + (i * LPG + gl) * VEC, &z[i * VEC]);
                }
        }
    }
}

#ifdef FMM_AUX_KERNELS
// Fold chunk partials of split rows into Z in chunk order (deterministic).
// split = {row, first slot, nchunks, 0}. Q chunk lanes per element each fold
// a contiguous chunk range, then lane 0 folds the Q results in order.
__global__ void __launch_bounds__(256)
fmm_combine_kernel(const int4* __restrict__ split, const float* __restrict__ partial,
                   float* __restrict__ Z, int d, int is_max, const PeerOut peers) {
    __shared__ float red[256];
    const int4 s = split[blockIdx.x];
    const int K = s.z;
    const float* base = partial + static_cast<int64_t>(s.y) * d;
    float* zr = Z + static_cast<int64_t>(s.x) * d;
    const float ident = is_max ? -__int_as_float(0x7f800000) : 0.0f;
    if (d >= 256) {
        for (int j = threadIdx.x; j < d; j += 256) {
            float acc = ident;
            int k = 0;
            for (; k + 4 <= K; k += 4) {
                const float v0 = base[(int64_t)(k + 0) * d + j];
                const float v1 = base[(int64_t)(k + 1) * d + j];
                const float v2 = base[(int64_t)(k + 2) * d + j];
                const float v3 = base[(int64_t)(k + 3) * d + j];
                if (is_max) {
                    acc = acc < v0 ? v0 : acc; acc = acc < v1 ? v1 : acc;
                    acc = acc < v2 ? v2 : acc; acc = acc < v3 ? v3 : acc;
                } else {
                    acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v0), v1), v2), v3);
                }
            }
            for (; k < K; ++k) {
                const float v = base[(int64_t)k * d + j];
                acc = is_max ? (acc < v ? v : acc) : __fadd_rn(acc, v);
            }
            zr[j] = acc;
            const unsigned pm = peers.n > 0 ? peer_bits(peers.mask, s.x) : 0u;
            for (int q = 0; q < peers.n; ++q)
                if ((pm >> q) & 1u) peers.p[q][static_cast<int64_t>(s.x) * d + j] = acc;
        }
        return;
    }
    const int Q = 256 / d;
    const int q = threadIdx.x / d;
    const int j = threadIdx.x % d;
    if (q < Q) {
        const int k0 = static_cast<int>((static_cast<int64_t>(K) * q) / Q);
        const int k1 = static_cast<int>((static_cast<int64_t>(K) * (q + 1)) / Q);
        float acc = ident;
        int k = k0;
        for (; k + 4 <= k1; k += 4) {
            const float v0 = base[(int64_t)(k + 0) * d + j];
            const float v1 = base[(int64_t)(k + 1) * d + j];
            const float v2 = base[(int64_t)(k + 2) * d + j];
            const float v3 = base[(int64_t)(k + 3) * d + j];
            if (is_max) {
                acc = acc < v0 ? v0 : acc; acc = acc < v1 ? v1 : acc;
                acc = acc < v2 ? v2 : acc; acc = acc < v3 ? v3 : acc;
            } else {
                acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v0), v1), v2), v3);
            }
        }
        for (; k < k1; ++k) {
            const float v = base[(int64_t)k * d + j];
            acc = is_max ? (acc < v ? v : acc) : __fadd_rn(acc, v);
        }
        red[threadIdx.x] = acc;
    }
    __syncthreads();
    if (q == 0) {
        float acc = red[j];
        for (int qq = 1; qq < Q; ++qq) {
            const float v = red[qq * d + j];
            acc = is_max ? (acc < v ? v : acc) : __fadd_rn(acc, v);
        }
        zr[j] = acc;
        const unsigned pm = peers.n > 0 ? peer_bits(peers.mask, s.x) : 0u;
        for (int qq = 0; qq < peers.n; ++qq)
            if ((pm >> qq) & 1u) peers.p[qq][static_cast<int64_t>(s.x) * d + j] = acc;
    }
}

// Narrow int64 columns to int32 while validating 0 <= c < n; tracks max col.
__global__ void fmm_narrow_cols_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                                       int64_t count, int64_t n, int* __restrict__ bad,
                                       int* __restrict__ max_col) {
    int local_max = -1;
    bool local_bad = false;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = src[i];
        if (c < 0 || c >= n) {
            local_bad = true;
            dst[i] = 0;
        } else {
            dst[i] = static_cast<int32_t>(c);
            local_max = max(local_max, static_cast<int>(c));
        }
    }
    local_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(local_max + 1))) - 1;
    if ((threadIdx.x & 31) == 0 && local_max >= 0) atomicMax(max_col, local_max);
    if (local_bad) atomicExch(bad, 1);
}

// need[c] = 1 for every column an edge points at (halo masks).
__global__ void fmm_mark_cols_kernel(const int32_t* __restrict__ col, int64_t count, uint8_t* __restrict__ need) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        need[col[i]] = 1;
}

#endif  // FMM_AUX_KERNELS

// Launch descriptor shared by the dispatch translation units.
struct LaunchCfg {
    int pattern;   // FMM_PATTERN_*
    int d;
    bool exact;
    bool aligned;  // X/Y/Z 16-byte aligned rows
};

// Defined in fmm_dispatch_*.cu; returns false if no instantiation fits.
bool launch_rows(const KParams& p, const LaunchCfg& cfg, cudaStream_t stream);

}  // namespace fmm
