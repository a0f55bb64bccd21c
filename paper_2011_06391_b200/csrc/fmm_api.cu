// fmm_api.cu — the C ABI of libfusedmm_cuda (include/fusedmm_cuda.h).
//
// Replaces the reference driver fusedmm::fused_mm (kernel.hpp:297-353): where
// the reference validates dims (check_dims, kernel.hpp:269-282), plans a 1D
// nnz-balanced partition (part1d, kernel.hpp:24-49) and spawns t std::thread
// workers over it (kernel.hpp:335-345), this library uploads the CSR once,
// partitions it with the same part1d rule across `ngpu` shards (one CUDA
// stream each), and launches the row kernels of fmm_kernels.cuh per shard.
#define FMM_AUX_KERNELS
#include "fmm_kernels.cuh"
#include "fmm_dispatch.cuh"
#include "fmm_plan.h"
#include "fmm_unfused.h"

#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
};

struct Shard {
    int dev = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t ext = nullptr;
    bool use_ext = false;  // ext may legitimately be the legacy NULL stream
    DevBuf X, Y, Z, Xb, partial;
    DevBuf H, iota;  // unfused baseline: materialised messages, edge ids
    DevBuf hs;       // d > 1024 streamed kernel: per-edge scalar h
    cudaEvent_t ev_start = nullptr, ev_k0 = nullptr, ev_k1 = nullptr, ev_end = nullptr,
                ev_copy = nullptr;
    // Launches that use this shard's scratch (chunk partials, fold tickets,
    // unfused messages) are ordered after the previous one even when the
    // caller moved to another stream (fmm_set_stream + FMM_ASYNC): the next
    // launch waits on ev_last when its stream differs from last_stream.
    cudaEvent_t ev_last = nullptr;
    cudaStream_t last_stream = nullptr;
    bool has_last = false;
    // host-pointer FMM_ASYNC pipeline: two buffer slots, copy-in / compute /
    // copy-out on three streams, so call k's Z download overlaps call k+1's
    // X upload (PCIe is full duplex) and the kernels
    cudaStream_t s_in = nullptr, s_out = nullptr;
    DevBuf aX[2], aY[2], aZ[2];
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
    int aslot = 0;
    cudaStream_t stream() const { return use_ext ? ext : own; }
};

}  // namespace

struct fmm_ctx {
    std::vector<Shard> shards;
    // Lifetime: graphs keep their context's shard table alive. fmm_destroy
    // releases the device resources at once but deletes the struct only when
    // the last graph of the context is freed, so fmm_graph_free is safe in
    // either order (Python finalisers and C++ destructors run in arbitrary
    // order at shutdown). Guarded by life_mu().
    int graphs = 0;
    bool destroyed = false;
    int variant = -1;  // kernel shape variant (FMM_VARIANT env, tuning only)
    double row_weight = 0.0;  // shard partition: 0 = part1d, > 0 = part1d_weighted
    bool p2p_ok = true;  // every pair of distinct shard devices has peer access
    std::string err;
    std::mutex mu;
};

namespace {

struct GShard {
    int shard = 0;
    int chunk = 256;  // edges per chunk of a split row (fast scheme)
    int64_t edge_begin = 0;  // first edge of the shard in the uploaded CSR
    int64_t row_begin = 0, row_end = 0, nnz = 0;
    int64_t n_split_rows = 0, n_wide_rows = 0, n_chunks = 0, n_slots = 0, nonempty = 0, max_degree = 0;
    int64_t n_wide_at[fmm::kWideLevels] = {};  // unsplit rows with degree >= 64 << k
    int64_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    float* val = nullptr;
    int32_t* order = nullptr;
    int4* items = nullptr;
    int4* chunks = nullptr;
    int4* split_rows = nullptr;
    unsigned* split_count = nullptr;  // in-kernel fold tickets (zero between launches)
    uint8_t* peer_mask = nullptr;     // per shard-local row: bit q = peer slot q reads it
    int64_t exchange_rows = 0;        // sum of popcount(peer_mask) (rows sent per exchange)
    int64_t exchange_rows_all = 0;    // rows * peers (every row to every peer)
};

}  // namespace

struct fmm_graph {
    fmm_ctx* ctx = nullptr;
    int64_t m = 0, n = 0, nnz = 0, row_begin = 0, row_end = 0;
    int64_t max_col = -1;
    bool has_values = false;
    bool iter_masks = false;  // fmm_iterate's halo masks were built
    std::vector<GShard> shards;
};

namespace {

fmm_status set_err(fmm_ctx* ctx, fmm_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

fmm_status cuda_err(fmm_ctx* ctx, cudaError_t e, const char* what) {
    const fmm_status st = (e == cudaErrorMemoryAllocation) ? FMM_E_OOM : FMM_E_CUDA;
    return set_err(ctx, st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define FMM_CK(ctx, call)                                            \
    do {                                                             \
        cudaError_t e_ = (call);                                     \
        if (e_ != cudaSuccess) return cuda_err((ctx), e_, #call);    \
    } while (0)

std::mutex& life_mu() {
    static std::mutex mu;
    return mu;
}

// Scratch-using launches on a shard: wait for the previous one if it ran on
// another stream, then (after the launch) remember this one.
fmm_status order_scratch(fmm_ctx* ctx, Shard& sh, cudaStream_t s) {
    if (sh.has_last && sh.last_stream != s) FMM_CK(ctx, cudaStreamWaitEvent(s, sh.ev_last, 0));
    return FMM_OK;
}
fmm_status mark_scratch(fmm_ctx* ctx, Shard& sh, cudaStream_t s) {
    FMM_CK(ctx, cudaEventRecord(sh.ev_last, s));
    sh.last_stream = s;
    sh.has_last = true;
    return FMM_OK;
}

fmm_status ensure(fmm_ctx* ctx, const Shard& sh, DevBuf& b, size_t bytes) {
    if (bytes <= b.cap) return FMM_OK;
    FMM_CK(ctx, cudaSetDevice(sh.dev));
    if (b.ptr) {
        FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
        FMM_CK(ctx, cudaFree(b.ptr));
        b.ptr = nullptr;
        b.cap = 0;
    }
    FMM_CK(ctx, cudaMalloc(&b.ptr, bytes));
    b.cap = bytes;
    return FMM_OK;
}

template <class T>
fmm_status upload_vec(fmm_ctx* ctx, const std::vector<T>& v, T** dst) {
    *dst = nullptr;
    if (v.empty()) return FMM_OK;
    FMM_CK(ctx, cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T)));
    FMM_CK(ctx, cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return FMM_OK;
}

bool is_user(const fmm_opspec& s) {
    return s.vop == FMM_VOP_USER || s.rop == FMM_ROP_USER || s.sop == FMM_SOP_USER ||
           s.mop == FMM_MOP_USER || s.aop == FMM_AOP_USER;
}

bool valid_codes(const fmm_opspec& s) {
    const bool v = (s.vop >= FMM_VOP_ADD && s.vop <= FMM_VOP_USER) || s.vop == FMM_VOP_MLP;
    const bool r = (s.rop >= FMM_ROP_NOOP && s.rop <= FMM_ROP_USER) || s.rop == FMM_ROP_SQNORM;
    const bool so = (s.sop >= FMM_SOP_NOOP && s.sop <= FMM_SOP_USER) || s.sop == FMM_SOP_TDIST ||
                    s.sop == FMM_SOP_SQK;
    const bool mo = (s.mop >= FMM_MOP_MUL && s.mop <= FMM_MOP_USER) || s.mop == FMM_MOP_MUL_VOP;
    const bool a = s.aop >= FMM_AOP_ASUM && s.aop <= FMM_AOP_USER;
    return v && r && so && mo && a;
}

// ops.hpp:189-203 plus the two device-only patterns.
int pattern_of(const fmm_opspec& s) {
    if (is_user(s)) return FMM_PATTERN_GENERIC;
    auto is = [&](int v, int r, int so, int mo, int a) {
        return s.vop == v && s.rop == r && s.sop == so && s.mop == mo && s.aop == a;
    };
    if (is(FMM_VOP_MUL, FMM_ROP_RSUM, FMM_SOP_SIGMOID, FMM_MOP_MUL, FMM_AOP_ASUM))
        return FMM_PATTERN_SIGMOID_EMBED;
    if (is(FMM_VOP_SEL2ND, FMM_ROP_NOOP, FMM_SOP_NOOP, FMM_MOP_MUL, FMM_AOP_ASUM))
        return FMM_PATTERN_SPMM_GCN;
    if (is(FMM_VOP_ADD, FMM_ROP_NORM, FMM_SOP_SCAL, FMM_MOP_MUL, FMM_AOP_ASUM))
        return FMM_PATTERN_FR_LAYOUT;
    if (is(FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_TDIST, FMM_MOP_MUL_VOP, FMM_AOP_ASUM))
        return FMM_PATTERN_TDIST;
    if (is(FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_SQK, FMM_MOP_MUL_VOP, FMM_AOP_ASUM))
        return FMM_PATTERN_FR_ATTRACT;
    return FMM_PATTERN_GENERIC;
}

// Default numerics scheme per pattern: bit-exact where the reference order is
// reproducible without serialising rows (configs 1 and 4).
bool default_exact(int pattern, int64_t d) {
    if (pattern == FMM_PATTERN_SPMM_GCN) return true;
    if (pattern == FMM_PATTERN_FR_ATTRACT && d <= 4) return true;
    return false;
}

// 1/k when k is a power of two whose reciprocal is a normal float (then
// s * (1/k) rounds exactly like s / k: both round the same exact value), else 0.
float exact_reciprocal(float k) {
    uint32_t b;
    std::memcpy(&b, &k, sizeof(b));
    const uint32_t ex = (b >> 23) & 0xffu;
    if ((b & 0x7fffffu) != 0 || ex == 0 || ex == 0xffu) return 0.0f;  // not a normal power of two
    const float inv = 1.0f / k;
    uint32_t bi;
    std::memcpy(&bi, &inv, sizeof(bi));
    const uint32_t exi = (bi >> 23) & 0xffu;
    return (exi == 0 || exi == 0xffu) ? 0.0f : inv;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

bool launch_rows(const fmm::KParams& p, int pattern, int d, bool exact, bool a32, bool a16, bool a8,
                 int variant, cudaStream_t s) {
    const bool vec = fmm::aligned_shape(d, a16, a8);
    if (vec) {
        switch (pattern) {
            case FMM_PATTERN_SIGMOID_EMBED: return fmm::launch_sigmoid(p, d, exact, variant, a32, s);
            case FMM_PATTERN_SPMM_GCN: return fmm::launch_gcn(p, d, exact, variant, a32, s);
            case FMM_PATTERN_FR_LAYOUT: return fmm::launch_fr(p, d, exact, variant, a32, s);
            case FMM_PATTERN_TDIST: return fmm::launch_tdist(p, d, exact, variant, a32, s);
            case FMM_PATTERN_FR_ATTRACT: return fmm::launch_frattr(p, d, exact, variant, a32, s);
            default: break;
        }
    }
    return fmm::launch_generic(p, d, exact, vec, s);
}

// need[c] = 1 for the columns shard gs's edges point at (empty vector when
// the shard has no edges). Caller holds ctx->mu.
fmm_status shard_column_use(fmm_ctx* ctx, const GShard& gs, int64_t n, std::vector<uint8_t>& need) {
    need.clear();
    if (gs.nnz == 0 || n <= 0) return FMM_OK;
    const Shard& sh = ctx->shards[gs.shard];
    FMM_CK(ctx, cudaSetDevice(sh.dev));
    uint8_t* dn = nullptr;
    FMM_CK(ctx, cudaMalloc(&dn, static_cast<size_t>(n)));
    cudaError_t e = cudaMemset(dn, 0, static_cast<size_t>(n));
    if (e == cudaSuccess) {
        const int blocks = static_cast<int>(std::min<int64_t>((gs.nnz + 255) / 256, 148 * 16));
        fmm::fmm_mark_cols_kernel<<<blocks, 256>>>(gs.col, gs.nnz, dn);
        e = cudaGetLastError();
    }
    need.resize(static_cast<size_t>(n));
    if (e == cudaSuccess) e = cudaMemcpy(need.data(), dn, static_cast<size_t>(n), cudaMemcpyDeviceToHost);
    cudaFree(dn);
    if (e != cudaSuccess) return cuda_err(ctx, e, "column use");
    return FMM_OK;
}

// Halo masks of a multi-shard graph for fmm_iterate's fused exchange: bit
// slot(q) of shard s's row r is set iff shard q's edges point at it, slot(q)
// = q for q < s and q-1 above (the order of the kernel's zpeer list).
fmm_status build_iterate_masks(fmm_ctx* ctx, fmm_graph* g) {
    const int S = static_cast<int>(g->shards.size());
    std::vector<std::vector<uint8_t>> need(S);
    for (int q = 0; q < S; ++q) {
        fmm_status st = shard_column_use(ctx, g->shards[q], g->n, need[q]);
        if (st != FMM_OK) return st;
    }
    for (int s = 0; s < S; ++s) {
        GShard& gs = g->shards[s];
        const int64_t rows = gs.row_end - gs.row_begin;
        std::vector<uint8_t> m(static_cast<size_t>(std::max<int64_t>(rows, 1)), 0);
        gs.exchange_rows = 0;
        for (int q = 0; q < S; ++q) {
            if (q == s || need[q].empty()) continue;
            const uint8_t bit = static_cast<uint8_t>(1u << (q < s ? q : q - 1));
            const uint8_t* nq = need[q].data() + gs.row_begin;
            for (int64_t r = 0; r < rows; ++r)
                if (nq[r]) m[r] |= bit;
        }
        for (int64_t r = 0; r < rows; ++r) gs.exchange_rows += __builtin_popcount(m[r]);
        gs.exchange_rows_all = rows * (S - 1);
        FMM_CK(ctx, cudaSetDevice(ctx->shards[gs.shard].dev));
        if (gs.peer_mask) {
            cudaFree(gs.peer_mask);
            gs.peer_mask = nullptr;
        }
        fmm_status st = upload_vec(ctx, m, &gs.peer_mask);
        if (st != FMM_OK) return st;
    }
    g->iter_masks = true;
    return FMM_OK;
}

// d > kMaxRegDim with a scalar message: the streamed kernel keeps one h per
// edge of the shard (fmm_k_stream.cu). nullptr when not needed.
float* hscratch(fmm_ctx* ctx, Shard& sh, const GShard& gs, int64_t d, const fmm_opspec& spec) {
    if (d <= fmm::kMaxRegDim || spec.rop == FMM_ROP_NOOP || gs.nnz == 0) return nullptr;
    if (ensure(ctx, sh, sh.hs, static_cast<size_t>(gs.nnz) * sizeof(float)) != FMM_OK) return nullptr;
    return static_cast<float*>(sh.hs.ptr);
}

int launch_shard(GShard& gs, const fmm_opspec& spec, int pattern, int64_t d, bool exact,
                 const float* X, int64_t row0, const float* Y, float* Z, float* partial,
                 const float* val, int variant, cudaStream_t stream,
                 const fmm::PeerOut* peers = nullptr, float* hs = nullptr, bool use_mask = true) {
    fmm::KParams p{};
    fmm::PeerOut po{};
    if (peers) {
        po = *peers;
        for (int q = 0; q < po.n; ++q) p.zpeer[q] = po.p[q];
        p.n_peer = po.n;
        // halo exchange: only rows some peer reads are stored to it
        if (use_mask && po.n > 0 && gs.peer_mask) p.peer_mask = gs.peer_mask;
        po.mask = p.peer_mask;
    }
    p.hbuf = hs;
    p.row_ptr = gs.row_ptr;
    p.col = gs.col;
    p.val = val;
    p.X = X;
    p.Y = Y;
    p.Z = Z;
    p.partial = partial;
    p.row0 = row0;
    p.chunk = gs.chunk;
    p.d = static_cast<int>(d);
    p.vop = spec.vop; p.rop = spec.rop; p.sop = spec.sop; p.mop = spec.mop; p.aop = spec.aop;
    p.alpha = spec.alpha;
    p.k = spec.k;
    p.kinv = exact_reciprocal(spec.k);
    p.mlp_wx = spec.mlp_wx;
    p.mlp_wy = spec.mlp_wy;
    p.mlp_b = spec.mlp_b;
    const int64_t rows = gs.row_end - gs.row_begin;
    const bool split = !exact && gs.n_chunks > 0;
    if (!exact) {
        // fast scheme: chunks of split rows, then wide rows, then narrow rows
        p.chunks = gs.chunks;
        p.n_chunk_items = gs.n_chunks;
        p.order = gs.order + gs.n_split_rows;
        p.items = gs.items + gs.n_split_rows;
        // rows a whole warp folds: the threshold depends on d (fmm_plan.h)
        p.n_wide_rows = gs.n_wide_at[fmm::wide_level_for(gs.chunk, static_cast<int>(d))];
        p.n_narrow_rows = rows - gs.n_split_rows - p.n_wide_rows;
    } else {
        // exact scheme: every row folded by one lane group, storage order
        p.chunks = nullptr;
        p.n_chunk_items = 0;
        p.order = gs.order;
        p.items = gs.items;
        p.n_wide_rows = 0;
        p.n_narrow_rows = rows;
    }
    if (p.n_chunk_items + p.n_wide_rows + p.n_narrow_rows == 0) return 0;
    if (d <= fmm::kMaxRegDim) {
        // empty rows sort last: they leave the narrow list and only get the
        // AOP identity, from the wide warps' prologues (up to kZeroPerWideMax
        // rows each) and from dedicated warps for the remainder
        static const bool zero_narrow = std::getenv("FMM_ZERO_NARROW") != nullptr;  // tuning: the old path
        if (!zero_narrow) {
            p.n_zero_rows = rows - gs.nonempty;
            p.n_narrow_rows -= p.n_zero_rows;
            const int64_t wide_warps = p.n_chunk_items + p.n_wide_rows;
            if (wide_warps > 0 && p.n_zero_rows > 0) {
                const int64_t per = std::min<int64_t>((p.n_zero_rows + wide_warps - 1) / wide_warps, fmm::kZeroPerWideMax);
                p.zero_per_wide = static_cast<int>(per);
                p.n_zero_piggy = std::min<int64_t>(p.n_zero_rows, per * wide_warps);
            }
        }
    }
    if (d > fmm::kMaxRegDim) {
        // any d past the register-resident shapes: the streamed kernel tiles
        // d (reference: the d > 256 second sweep, kernel.hpp:192-225); rows
        // are never split, each folded by one warp in storage order
        p.chunks = nullptr;
        p.n_chunk_items = 0;
        p.order = gs.order;
        p.items = gs.items;
        p.n_wide_rows = 0;
        p.n_narrow_rows = rows;
        return fmm::launch_stream(p, exact, stream) ? 1 : -1;
    }
    const size_t a = static_cast<size_t>(d) * sizeof(float);
    bool a16 = (d % 4 == 0) && aligned(X, 16) && aligned(Y, 16) && aligned(Z, 16) &&
               (partial == nullptr || aligned(partial, 16)) && (a % 16 == 0);
    bool a8 = (d % 2 == 0) && aligned(X, 8) && aligned(Y, 8) && aligned(Z, 8) &&
              (partial == nullptr || aligned(partial, 8));
    bool a32 = (d % 8 == 0) && aligned(X, 32) && aligned(Y, 32) && aligned(Z, 32) &&
               (partial == nullptr || aligned(partial, 32));
    bool fold4 = (d % 4 == 0) && aligned(Z, 16) && (partial == nullptr || aligned(partial, 16));
    // the vector shapes also store z rows to the peers with the same width
    for (int q = 0; q < po.n; ++q) {
        a32 = a32 && aligned(po.p[q], 32);
        a16 = a16 && aligned(po.p[q], 16);
        a8 = a8 && aligned(po.p[q], 8);
        fold4 = fold4 && aligned(po.p[q], 16);
    }
    p.fold_vec4 = fold4 ? 1 : 0;
    if (variant < -1) variant = -1;
    // split rows fold inside the row kernel (the last chunk's warp) unless
    // FMM_FOLD_KERNEL selects the separate combine kernel
    static const bool fold_kernel = std::getenv("FMM_FOLD_KERNEL") != nullptr;
    const bool inline_fold = split && gs.split_count != nullptr && !fold_kernel;
    if (inline_fold) {
        p.split_rows = gs.split_rows;
        p.split_count = gs.split_count;
        p.fold_max = spec.aop == FMM_AOP_AMAX ? 1 : 0;
    }
    if (!launch_rows(p, pattern, static_cast<int>(d), exact, a32, a16, a8, variant, stream)) return -1;
    int launches = 1;
    if (split && gs.n_split_rows > 0 && !inline_fold) {
        fmm::fmm_combine_kernel<<<static_cast<unsigned>(gs.n_split_rows), 256, 0, stream>>>(
            gs.split_rows, partial, Z, static_cast<int>(d), spec.aop == FMM_AOP_AMAX ? 1 : 0, po);
        ++launches;
    }
    return launches;
}

// Walk the dispatch tables with launch_one in attribute-query mode.
void preload_kernels() {
    fmm::KParams p{};
    const int pats[] = {FMM_PATTERN_SIGMOID_EMBED, FMM_PATTERN_SPMM_GCN, FMM_PATTERN_FR_LAYOUT, FMM_PATTERN_TDIST,
                        FMM_PATTERN_FR_ATTRACT, FMM_PATTERN_GENERIC};
    const int dims[] = {1, 2, 4, 8, 16, 32, 64, 128, 256, 512};
    fmm::t_preload = true;
    for (int pat : pats)
        for (int d : dims)
            for (int ex = 0; ex < 2; ++ex)
                for (int a32 = 0; a32 < 2; ++a32) launch_rows(p, pat, d, ex != 0, a32 != 0, true, true, -1, nullptr);
    for (int ex = 0; ex < 2; ++ex) {
        for (int d : {32, 64, 96, 128, 256, 512, 1024}) fmm::launch_generic(p, d, ex != 0, false, nullptr);
        fmm::launch_stream(p, ex != 0, nullptr);
    }
    fmm::t_preload = false;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0.f;
    return ms;
}

fmm_status check_spec(fmm_ctx* ctx, const fmm_opspec* spec, int64_t d) {
    if (!spec) return set_err(ctx, FMM_E_INVAL, "fused_mm: spec is NULL");
    if (!valid_codes(*spec)) return set_err(ctx, FMM_E_INVAL, "fused_mm: unknown op code");
    if (is_user(*spec))
        return set_err(ctx, FMM_E_UNSUPPORTED,
                       "fused_mm: USER slot has no device kernel (no CPU fallback)");
    if (d < 1) return set_err(ctx, FMM_E_INVAL, "fused_mm: d must be >= 1");
    if (d > (int64_t(1) << 24)) return set_err(ctx, FMM_E_UNSUPPORTED, "fused_mm: d > 2^24 not supported");
    return FMM_OK;
}

// fmm_run with host pointers and FMM_ASYNC: enqueue upload / fused kernels /
// download on the shard's copy-in, compute and copy-out streams using buffer
// slot (call index % 2), then return. The caller keeps X, Y, Z valid (pinned
// for true overlap) until fmm_sync.
fmm_status run_host_async(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec& spec, int pattern,
                          bool exact, int64_t d, const float* X, int64_t ny, const float* Y, float* Z,
                          fmm_stats* stats) {
    const size_t row_bytes = static_cast<size_t>(d) * sizeof(float);
    const bool alias = (X == Y) && (ny == g->m);
    int launches = 0;
    size_t aux = 0;
    fmm_status st;
    for (size_t s = 0; s < g->shards.size(); ++s) {
        const GShard& gs = g->shards[s];
        Shard& sh = ctx->shards[gs.shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        if (!sh.s_in) {
            FMM_CK(ctx, cudaStreamCreateWithFlags(&sh.s_in, cudaStreamNonBlocking));
            FMM_CK(ctx, cudaStreamCreateWithFlags(&sh.s_out, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                FMM_CK(ctx, cudaEventCreateWithFlags(&sh.ev_in[i], cudaEventDisableTiming));
                FMM_CK(ctx, cudaEventCreateWithFlags(&sh.ev_comp[i], cudaEventDisableTiming));
                FMM_CK(ctx, cudaEventCreateWithFlags(&sh.ev_out[i], cudaEventDisableTiming));
                // recorded once so the first waits on them are satisfied
                FMM_CK(ctx, cudaEventRecord(sh.ev_comp[i], sh.s_in));
                FMM_CK(ctx, cudaEventRecord(sh.ev_out[i], sh.s_out));
            }
        }
        const int k = sh.aslot;
        sh.aslot ^= 1;
        const int64_t srows = gs.row_end - gs.row_begin;
        // buffers of slot k (a reallocation waits for every stream)
        const size_t ybytes = std::max<size_t>(1, ny * row_bytes);
        const size_t xbytes = std::max<size_t>(1, srows * row_bytes);
        if (sh.aY[k].cap < ybytes || (!alias && sh.aX[k].cap < xbytes) || sh.aZ[k].cap < xbytes) {
            for (cudaStream_t q : {sh.s_in, sh.s_out, sh.stream()}) FMM_CK(ctx, cudaStreamSynchronize(q));
        }
        if ((st = ensure(ctx, sh, sh.aY[k], ybytes)) != FMM_OK) return st;
        if (!alias && (st = ensure(ctx, sh, sh.aX[k], xbytes)) != FMM_OK) return st;
        if ((st = ensure(ctx, sh, sh.aZ[k], xbytes)) != FMM_OK) return st;
        float* part = nullptr;
        if (!exact && gs.n_slots > 0) {
            const size_t pb = static_cast<size_t>(gs.n_slots) * row_bytes;
            if (sh.partial.cap < pb) FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
            if ((st = ensure(ctx, sh, sh.partial, pb)) != FMM_OK) return st;
            part = static_cast<float*>(sh.partial.ptr);
            aux = std::max(aux, pb);
        }
        // upload into slot k once the kernels of call k-2 stopped reading it
        FMM_CK(ctx, cudaStreamWaitEvent(sh.s_in, sh.ev_comp[k], 0));
        if (ny > 0) FMM_CK(ctx, cudaMemcpyAsync(sh.aY[k].ptr, Y, ny * row_bytes, cudaMemcpyHostToDevice, sh.s_in));
        if (!alias && srows > 0)
            FMM_CK(ctx, cudaMemcpyAsync(sh.aX[k].ptr, X + gs.row_begin * d, srows * row_bytes,
                                        cudaMemcpyHostToDevice, sh.s_in));
        FMM_CK(ctx, cudaEventRecord(sh.ev_in[k], sh.s_in));
        // compute once uploaded and once call k-2's download released Z slot k
        cudaStream_t cs = sh.stream();
        FMM_CK(ctx, cudaStreamWaitEvent(cs, sh.ev_in[k], 0));
        FMM_CK(ctx, cudaStreamWaitEvent(cs, sh.ev_out[k], 0));
        const float* yd = static_cast<const float*>(sh.aY[k].ptr);
        const float* xd = alias ? yd : static_cast<const float*>(sh.aX[k].ptr);
        const int64_t row0 = alias ? gs.row_begin : 0;
        float* zd = static_cast<float*>(sh.aZ[k].ptr);
        float* hs = hscratch(ctx, sh, gs, d, spec);
        if ((part || hs) && (st = order_scratch(ctx, sh, cs)) != FMM_OK) return st;
        const int l = launch_shard(const_cast<GShard&>(gs), spec, pattern, d, exact, xd, row0, yd, zd, part,
                                   gs.val, ctx->variant, cs, nullptr, hs);
        if (l < 0) return set_err(ctx, FMM_E_UNSUPPORTED, "fused_mm: no kernel for this d / alignment");
        if ((part || hs) && (st = mark_scratch(ctx, sh, cs)) != FMM_OK) return st;
        launches += l;
        FMM_CK(ctx, cudaGetLastError());
        FMM_CK(ctx, cudaEventRecord(sh.ev_comp[k], cs));
        // download after the kernels
        FMM_CK(ctx, cudaStreamWaitEvent(sh.s_out, sh.ev_comp[k], 0));
        if (srows > 0)
            FMM_CK(ctx, cudaMemcpyAsync(Z + (gs.row_begin - g->row_begin) * d, zd, srows * row_bytes,
                                        cudaMemcpyDeviceToHost, sh.s_out));
        FMM_CK(ctx, cudaEventRecord(sh.ev_out[k], sh.s_out));
    }
    if (stats) {
        *stats = fmm_stats{};
        stats->aux_bytes = aux;
        stats->threads = static_cast<int32_t>(g->shards.size());
        stats->pattern = pattern;
        stats->exact = exact ? 1 : 0;
        stats->launches = launches;
    }
    return FMM_OK;
}

}  // namespace

extern "C" {

fmm_status fmm_host_alloc(void** ptr, size_t bytes) {
    if (!ptr) return FMM_E_INVAL;
    *ptr = nullptr;
    const cudaError_t e = cudaHostAlloc(ptr, std::max<size_t>(bytes, 1), cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? FMM_E_OOM : FMM_E_CUDA;
    }
    return FMM_OK;
}

fmm_status fmm_host_free(void* ptr) {
    if (!ptr) return FMM_OK;
    return cudaFreeHost(ptr) == cudaSuccess ? FMM_OK : FMM_E_CUDA;
}

fmm_status fmm_sync(fmm_ctx* ctx) {
    if (!ctx) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    for (Shard& sh : ctx->shards) {
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        if (sh.s_in) FMM_CK(ctx, cudaStreamSynchronize(sh.s_in));
        FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
        if (sh.s_out) FMM_CK(ctx, cudaStreamSynchronize(sh.s_out));
    }
    return FMM_OK;
}

const char* fmm_version(void) { return "libfusedmm_cuda 0.1 (sm_100a)"; }

const char* fmm_status_string(fmm_status s) {
    switch (s) {
        case FMM_OK: return "ok";
        case FMM_E_INVAL: return "invalid argument";
        case FMM_E_UNSUPPORTED: return "unsupported";
        case FMM_E_CUDA: return "cuda error";
        case FMM_E_NCCL: return "nccl error";
        case FMM_E_OOM: return "out of memory";
        case FMM_E_LOGIC: return "logic error";
    }
    return "unknown status";
}

int fmm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

fmm_status fmm_create(int ngpu, const int* devs, fmm_ctx** out) {
    if (!out) return FMM_E_INVAL;
    *out = nullptr;
    if (ngpu < 1) return FMM_E_INVAL;  // kernel.hpp:303: t must be >= 1
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FMM_E_CUDA;
    fmm_ctx* ctx = new (std::nothrow) fmm_ctx();
    if (!ctx) return FMM_E_OOM;
    ctx->shards.resize(ngpu);
    if (const char* v = std::getenv("FMM_VARIANT")) ctx->variant = std::atoi(v);
    for (int i = 0; i < ngpu; ++i) {
        const int dev = devs ? devs[i] : (i % ndev);
        if (dev < 0 || dev >= ndev) {
            delete ctx;
            return FMM_E_INVAL;
        }
        Shard& sh = ctx->shards[i];
        sh.dev = dev;
        cudaDeviceGetAttribute(&sh.num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaSetDevice(dev) != cudaSuccess ||
            cudaStreamCreateWithFlags(&sh.own, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreate(&sh.ev_start) != cudaSuccess || cudaEventCreate(&sh.ev_k0) != cudaSuccess ||
            cudaEventCreate(&sh.ev_k1) != cudaSuccess || cudaEventCreate(&sh.ev_end) != cudaSuccess ||
            cudaEventCreateWithFlags(&sh.ev_copy, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sh.ev_last, cudaEventDisableTiming) != cudaSuccess) {
            fmm_destroy(ctx);
            return FMM_E_CUDA;
        }
    }
    // load every shipped row kernel now (CUDA loads modules lazily, ~10 ms
    // per op kind on the first launch otherwise: the drop-in's first
    // fused_mm call would pay it); FMM_NO_PRELOAD=1 skips
    if (!std::getenv("FMM_NO_PRELOAD")) {
        std::vector<int> seen;
        for (int i = 0; i < ngpu; ++i) {
            const int dev = ctx->shards[i].dev;
            if (std::find(seen.begin(), seen.end(), dev) != seen.end()) continue;
            seen.push_back(dev);
            cudaSetDevice(dev);
            preload_kernels();
        }
        cudaGetLastError();
    }
    // peer access between distinct devices (NVLink / NVSwitch)
    for (int i = 0; i < ngpu; ++i)
        for (int j = 0; j < ngpu; ++j) {
            const int a = ctx->shards[i].dev, b = ctx->shards[j].dev;
            if (a == b) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, a, b);
            if (can) {
                cudaSetDevice(a);
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) ctx->p2p_ok = false;
            } else {
                ctx->p2p_ok = false;  // kernels cannot store into that peer
            }
        }
    *out = ctx;
    return FMM_OK;
}

fmm_status fmm_destroy(fmm_ctx* ctx) {
    if (!ctx) return FMM_E_INVAL;
    std::lock_guard<std::mutex> life(life_mu());
    if (ctx->destroyed) return FMM_E_INVAL;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (Shard& sh : ctx->shards) {
            cudaSetDevice(sh.dev);
            if (sh.own) cudaStreamSynchronize(sh.own);
            if (sh.use_ext) cudaStreamSynchronize(sh.ext);
            for (cudaStream_t st : {sh.s_in, sh.s_out})
                if (st) cudaStreamSynchronize(st);
            for (DevBuf* b : {&sh.X, &sh.Y, &sh.Z, &sh.Xb, &sh.partial, &sh.H, &sh.iota, &sh.hs, &sh.aX[0],
                              &sh.aX[1], &sh.aY[0], &sh.aY[1], &sh.aZ[0], &sh.aZ[1]})
                if (b->ptr) {
                    cudaFree(b->ptr);
                    b->ptr = nullptr;
                    b->cap = 0;
                }
            for (cudaEvent_t* e : {&sh.ev_start, &sh.ev_k0, &sh.ev_k1, &sh.ev_end, &sh.ev_copy, &sh.ev_last,
                                   &sh.ev_in[0], &sh.ev_in[1], &sh.ev_comp[0], &sh.ev_comp[1], &sh.ev_out[0],
                                   &sh.ev_out[1]})
                if (*e) {
                    cudaEventDestroy(*e);
                    *e = nullptr;
                }
            for (cudaStream_t* st : {&sh.own, &sh.s_in, &sh.s_out})
                if (*st) {
                    cudaStreamDestroy(*st);
                    *st = nullptr;
                }
            sh.use_ext = false;
            sh.has_last = false;
        }
        ctx->destroyed = true;
    }
    // graphs still alive keep the (now resource-free) shard table until the
    // last of them is freed
    if (ctx->graphs == 0) delete ctx;
    return FMM_OK;
}

const char* fmm_last_error(const fmm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fmm_status fmm_set_stream(fmm_ctx* ctx, int shard, void* stream) {
    if (!ctx || shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    ctx->shards[shard].ext = static_cast<cudaStream_t>(stream);
    ctx->shards[shard].use_ext = true;
    return FMM_OK;
}

fmm_status fmm_set_variant(fmm_ctx* ctx, int variant) {
    if (!ctx || variant < -6 || variant > 63) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    ctx->variant = variant;
    return FMM_OK;
}

int fmm_get_variant(const fmm_ctx* ctx) { return ctx ? ctx->variant : -1; }

fmm_status fmm_reset_stream(fmm_ctx* ctx, int shard) {
    if (!ctx || shard < 0 || shard >= static_cast<int>(ctx->shards.size())) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    ctx->shards[shard].ext = nullptr;
    ctx->shards[shard].use_ext = false;
    return FMM_OK;
}

fmm_status fmm_pattern_of(const fmm_opspec* spec, int32_t* pattern) {
    if (!spec || !pattern) return FMM_E_INVAL;
    *pattern = pattern_of(*spec);
    return FMM_OK;
}

fmm_status fmm_part1d_weighted(int64_t m, const int64_t* row_ptr, int t, double row_weight,
                               int64_t* boundaries) {
    if (m < 0 || !row_ptr || !boundaries || t < 1 || !(row_weight >= 0.0)) return FMM_E_INVAL;
    try {
        const auto b = fmm::part1d_weighted(m, row_ptr, t, row_weight);
        std::memcpy(boundaries, b.data(), b.size() * sizeof(int64_t));
    } catch (const std::exception&) {
        return FMM_E_INVAL;
    }
    return FMM_OK;
}

fmm_status fmm_plan_pieces(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           int64_t row_begin, int64_t row_end, int64_t* chunk_edges,
                           int64_t* n_split_rows, int64_t* n_banded_rows, int64_t* n_pieces,
                           int64_t* pieces, int64_t cap) {
    if (m < 0 || n < 0 || !row_ptr || row_begin < 0 || row_end > m || row_begin > row_end) return FMM_E_INVAL;
    if (!fmm::validate_row_ptr(m, row_ptr).empty()) return FMM_E_INVAL;
    try {
        const int chunk = fmm::choose_chunk_edges(row_ptr[m] - row_ptr[0]);
        const fmm::BandParams bands = fmm::choose_bands(n);
        const fmm::ShardPlan P = fmm::build_shard_plan(row_ptr, row_begin, row_end, chunk, col_idx, bands);
        if (chunk_edges) *chunk_edges = chunk;
        if (n_split_rows) *n_split_rows = P.n_split_rows;
        if (n_banded_rows) *n_banded_rows = P.n_banded_rows;
        if (n_pieces) *n_pieces = static_cast<int64_t>(P.chunks.size());
        if (pieces) {
            const int64_t cnt = std::min<int64_t>(cap, static_cast<int64_t>(P.chunks.size()));
            for (int64_t i = 0; i < cnt; ++i) {
                const fmm::Int4& c = P.chunks[static_cast<size_t>(i)];
                const int64_t row = P.split_rows[static_cast<size_t>(c.x)].x;  // shard-local
                pieces[4 * i + 0] = row_begin + row;
                pieces[4 * i + 1] = c.y;
                pieces[4 * i + 2] = c.z;
                int64_t band = 0;
                if (bands.band_cols > 0 && col_idx)
                    band = std::max<int64_t>(col_idx[row_ptr[row_begin + row] + c.y], 0) / bands.band_cols;
                pieces[4 * i + 3] = band;
            }
        }
    } catch (const std::exception&) {
        return FMM_E_UNSUPPORTED;
    }
    return FMM_OK;
}

fmm_status fmm_set_row_weight(fmm_ctx* ctx, double row_weight) {
    if (!ctx || !(row_weight >= 0.0)) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    ctx->row_weight = row_weight;
    return FMM_OK;
}

fmm_status fmm_part1d(int64_t m, const int64_t* row_ptr, int t, int64_t* boundaries) {
    if (m < 0 || !row_ptr || !boundaries || t < 1) return FMM_E_INVAL;
    try {
        const auto b = fmm::part1d(m, row_ptr, t);
        std::memcpy(boundaries, b.data(), b.size() * sizeof(int64_t));
    } catch (const std::exception&) {
        return FMM_E_INVAL;
    }
    return FMM_OK;
}

fmm_status fmm_graph_upload(fmm_ctx* ctx, int64_t m, int64_t n, const int64_t* row_ptr,
                            const int64_t* col_idx, const float* values, int64_t row_begin,
                            int64_t row_end, fmm_graph** out) {
    if (!ctx || !out) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    *out = nullptr;
    if (m < 0 || n < 0 || !row_ptr) return set_err(ctx, FMM_E_INVAL, "graph_upload: bad sizes");
    if (n > INT32_MAX) return set_err(ctx, FMM_E_UNSUPPORTED, "graph_upload: n >= 2^31");
    if (row_begin < 0 || row_end > m || row_begin > row_end)
        return set_err(ctx, FMM_E_INVAL, "graph_upload: bad row range");
    const std::string bad = fmm::validate_row_ptr(m, row_ptr);
    if (!bad.empty()) return set_err(ctx, FMM_E_INVAL, "graph_upload: " + bad);
    if (row_ptr[m] > 0 && !col_idx) return set_err(ctx, FMM_E_INVAL, "graph_upload: col_idx NULL");

    fmm_graph* g = new (std::nothrow) fmm_graph();
    if (!g) return FMM_E_OOM;
    g->ctx = ctx;
    {
        std::lock_guard<std::mutex> life(life_mu());
        ++ctx->graphs;  // fmm_graph_free (also on the error paths below) releases it
    }
    g->m = m;
    g->n = n;
    g->row_begin = row_begin;
    g->row_end = row_end;
    g->nnz = row_ptr[row_end] - row_ptr[row_begin];
    g->has_values = values != nullptr;

    const int S = static_cast<int>(ctx->shards.size());
    // part1d over the requested row range (kernel.hpp:24-49)
    std::vector<int64_t> bounds;
    try {
        bounds = fmm::part1d_weighted(row_end - row_begin, row_ptr + row_begin, S, ctx->row_weight);
    } catch (const std::exception& e) {
        delete g;
        return set_err(ctx, FMM_E_INVAL, e.what());
    }
    g->shards.resize(S);
    // chunk size from the whole matrix (never the uploaded range or a shard):
    // per-rank uploads of one graph must split rows identically
    const int chunk = fmm::choose_chunk_edges(row_ptr[m] - row_ptr[0]);
    // column bands for the heavy rows of graphs far larger than the L2 (also a
    // function of the whole matrix only)
    const fmm::BandParams bands = fmm::choose_bands(n);
    fmm_status st = FMM_OK;
    for (int s = 0; s < S && st == FMM_OK; ++s) {
        GShard& gs = g->shards[s];
        const Shard& sh = ctx->shards[s];
        gs.shard = s;
        gs.row_begin = row_begin + bounds[s];
        gs.row_end = row_begin + bounds[s + 1];
        fmm::ShardPlan P;
        try {
            P = fmm::build_shard_plan(row_ptr, gs.row_begin, gs.row_end, chunk, col_idx, bands);
        } catch (const std::exception& e) {
            st = set_err(ctx, FMM_E_UNSUPPORTED, e.what());
            break;
        }
        gs.nnz = P.nnz;
        gs.chunk = P.chunk;
        gs.edge_begin = P.edge_begin;
        gs.n_split_rows = P.n_split_rows;
        gs.n_wide_rows = P.n_wide_rows;
        for (int k = 0; k < fmm::kWideLevels; ++k) gs.n_wide_at[k] = P.n_wide_at[k];
        gs.n_chunks = static_cast<int64_t>(P.chunks.size());
        gs.n_slots = P.n_slots;
        gs.nonempty = P.nonempty_rows;
        gs.max_degree = P.max_degree;
        if (cudaSetDevice(sh.dev) != cudaSuccess) { st = set_err(ctx, FMM_E_CUDA, "cudaSetDevice"); break; }
        if ((st = upload_vec(ctx, P.local_row_ptr, &gs.row_ptr)) != FMM_OK) break;
        if ((st = upload_vec(ctx, P.order, &gs.order)) != FMM_OK) break;
        static_assert(sizeof(fmm::Int4) == sizeof(int4), "int4 layout");
        std::vector<int4> ch(P.chunks.size()), sr(P.split_rows.size()), it(P.items.size());
        std::memcpy(ch.data(), P.chunks.data(), ch.size() * sizeof(int4));
        std::memcpy(it.data(), P.items.data(), it.size() * sizeof(int4));
        if ((st = upload_vec(ctx, it, &gs.items)) != FMM_OK) break;
        std::memcpy(sr.data(), P.split_rows.data(), sr.size() * sizeof(int4));
        if ((st = upload_vec(ctx, ch, &gs.chunks)) != FMM_OK) break;
        if ((st = upload_vec(ctx, sr, &gs.split_rows)) != FMM_OK) break;
        if (!sr.empty()) {
            cudaError_t e = cudaMalloc(&gs.split_count, sr.size() * sizeof(unsigned));
            if (e == cudaSuccess) e = cudaMemset(gs.split_count, 0, sr.size() * sizeof(unsigned));
            if (e != cudaSuccess) { st = cuda_err(ctx, e, "split counters"); break; }
        }
        if (gs.nnz > 0) {
            // narrow + validate columns in staged slices
            auto fail = [&](cudaError_t e, const char* w) { st = cuda_err(ctx, e, w); };
            cudaError_t e;
            if ((e = cudaMalloc(&gs.col, gs.nnz * sizeof(int32_t))) != cudaSuccess) { fail(e, "cudaMalloc col"); break; }
            const int64_t stage = std::min<int64_t>(gs.nnz, int64_t(1) << 24);
            int64_t* tmp = nullptr;
            int* flags = nullptr;
            if ((e = cudaMalloc(&tmp, stage * sizeof(int64_t))) != cudaSuccess) { fail(e, "cudaMalloc stage"); break; }
            if ((e = cudaMalloc(&flags, 2 * sizeof(int))) != cudaSuccess) { cudaFree(tmp); fail(e, "cudaMalloc flags"); break; }
            int init[2] = {0, -1};
            cudaMemcpy(flags, init, sizeof(init), cudaMemcpyHostToDevice);
            for (int64_t off = 0; off < gs.nnz && st == FMM_OK; off += stage) {
                const int64_t cnt = std::min(stage, gs.nnz - off);
                e = cudaMemcpy(tmp, col_idx + P.edge_begin + off, cnt * sizeof(int64_t), cudaMemcpyHostToDevice);
                if (e != cudaSuccess) { fail(e, "cudaMemcpy cols"); break; }
                const int blocks = static_cast<int>(std::min<int64_t>((cnt + 255) / 256, 148 * 16));
                fmm::fmm_narrow_cols_kernel<<<blocks, 256>>>(tmp, gs.col + off, cnt, n, flags, flags + 1);
                if ((e = cudaGetLastError()) != cudaSuccess) { fail(e, "narrow kernel"); break; }
            }
            int res[2] = {0, -1};
            if (st == FMM_OK) {
                if ((e = cudaMemcpy(res, flags, sizeof(res), cudaMemcpyDeviceToHost)) != cudaSuccess) fail(e, "cudaMemcpy flags");
            }
            cudaFree(tmp);
            cudaFree(flags);
            if (st != FMM_OK) break;
            if (res[0]) { st = set_err(ctx, FMM_E_INVAL, "graph_upload: column index out of range"); break; }
            g->max_col = std::max<int64_t>(g->max_col, res[1]);
            if (values) {
                if ((e = cudaMalloc(&gs.val, gs.nnz * sizeof(float))) != cudaSuccess) { fail(e, "cudaMalloc val"); break; }
                if ((e = cudaMemcpy(gs.val, values + P.edge_begin, gs.nnz * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess) { fail(e, "cudaMemcpy val"); break; }
            }
        }
    }
    if (st != FMM_OK) {
        fmm_graph_free(g);
        return st;
    }
    *out = g;
    return FMM_OK;
}

fmm_status fmm_graph_column_use(const fmm_graph* g, uint8_t* need) {
    if (!g || !need) return FMM_E_INVAL;
    fmm_ctx* ctx = g->ctx;
    if (ctx->destroyed) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    std::memset(need, 0, static_cast<size_t>(std::max<int64_t>(g->n, 0)));
    std::vector<uint8_t> part;
    for (const GShard& gs : g->shards) {
        fmm_status st = shard_column_use(ctx, gs, g->n, part);
        if (st != FMM_OK) return st;
        if (!part.empty())
            for (int64_t c = 0; c < g->n; ++c) need[c] |= part[c];
    }
    return FMM_OK;
}

fmm_status fmm_graph_set_peer_mask(fmm_graph* g, const uint8_t* mask, int npeer) {
    if (!g || npeer < 0 || npeer > fmm::kMaxPeers) return FMM_E_INVAL;
    fmm_ctx* ctx = g->ctx;
    if (ctx->destroyed) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (g->shards.size() != 1) return set_err(ctx, FMM_E_INVAL, "set_peer_mask: single-shard graphs only");
    GShard& gs = g->shards[0];
    FMM_CK(ctx, cudaSetDevice(ctx->shards[gs.shard].dev));
    if (gs.peer_mask) {
        FMM_CK(ctx, cudaDeviceSynchronize());  // a launch may still read it
        cudaFree(gs.peer_mask);
        gs.peer_mask = nullptr;
    }
    gs.exchange_rows = gs.exchange_rows_all = 0;
    if (!mask) return FMM_OK;  // cleared: every row to every peer
    const int64_t rows = gs.row_end - gs.row_begin;
    const unsigned keep = npeer >= 8 ? 0xffu : ((1u << npeer) - 1u);
    std::vector<uint8_t> m(static_cast<size_t>(std::max<int64_t>(rows, 1)), 0);
    for (int64_t r = 0; r < rows; ++r) {
        m[r] = static_cast<uint8_t>(mask[r] & keep);
        gs.exchange_rows += __builtin_popcount(m[r]);
    }
    gs.exchange_rows_all = rows * npeer;
    fmm_status st = upload_vec(ctx, m, &gs.peer_mask);
    return st;
}

fmm_status fmm_graph_free(fmm_graph* g) {
    if (!g) return FMM_E_INVAL;
    fmm_ctx* ctx = g->ctx;
    for (GShard& gs : g->shards) {
        cudaSetDevice(ctx->shards[gs.shard].dev);
        for (void* p : {static_cast<void*>(gs.row_ptr), static_cast<void*>(gs.col), static_cast<void*>(gs.val),
                        static_cast<void*>(gs.order), static_cast<void*>(gs.items), static_cast<void*>(gs.chunks),
                        static_cast<void*>(gs.split_count), static_cast<void*>(gs.split_rows),
                        static_cast<void*>(gs.peer_mask)})
            if (p) cudaFree(p);
    }
    delete g;
    std::lock_guard<std::mutex> life(life_mu());
    if (--ctx->graphs == 0 && ctx->destroyed) delete ctx;
    return FMM_OK;
}

fmm_status fmm_graph_update_values(fmm_graph* g, const float* values) {
    if (!g) return FMM_E_INVAL;
    fmm_ctx* ctx = g->ctx;
    if (ctx->destroyed) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    for (GShard& gs : g->shards) {
        Shard& sh = ctx->shards[gs.shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        // a launch still in flight may read the old values
        FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
        if (!values) {
            if (gs.val) cudaFree(gs.val);
            gs.val = nullptr;
            continue;
        }
        if (gs.nnz == 0) continue;
        if (!gs.val) FMM_CK(ctx, cudaMalloc(&gs.val, gs.nnz * sizeof(float)));
        FMM_CK(ctx, cudaMemcpy(gs.val, values + gs.edge_begin, gs.nnz * sizeof(float), cudaMemcpyHostToDevice));
    }
    g->has_values = values != nullptr;
    return FMM_OK;
}

uint64_t fmm_fingerprint(const void* data, size_t bytes) {
    if (!data || bytes == 0) return 0x9e3779b97f4a7c15ull ^ bytes;
    const unsigned char* b = static_cast<const unsigned char*>(data);
    constexpr size_t kChunk = size_t(1) << 22;  // 4 MiB per task, combined in order
    const size_t nchunk = (bytes + kChunk - 1) / kChunk;
    std::vector<uint64_t> h(nchunk);
    auto hash_chunk = [&](size_t c) {
        const size_t lo = c * kChunk, hi = std::min(bytes, lo + kChunk);
        uint64_t a = 0x243f6a8885a308d3ull ^ lo, z = 0x13198a2e03707344ull;
        size_t i = lo;
        for (; i + 16 <= hi; i += 16) {
            uint64_t w0, w1;
            std::memcpy(&w0, b + i, 8);
            std::memcpy(&w1, b + i + 8, 8);
            a = (a ^ w0) * 0x9fb21c651e98df25ull;
            z = (z ^ w1) * 0xc2b2ae3d27d4eb4full;
            a ^= a >> 29;
            z ^= z >> 31;
        }
        for (; i < hi; ++i) a = (a ^ b[i]) * 0x100000001b3ull;
        h[c] = a * 0xff51afd7ed558ccdull ^ z;
    };
    const unsigned nt = std::max(1u, std::min<unsigned>(static_cast<unsigned>(nchunk),
                                                        std::thread::hardware_concurrency()));
    if (nt == 1) {
        for (size_t c = 0; c < nchunk; ++c) hash_chunk(c);
    } else {
        std::atomic<size_t> next{0};
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&] {
                for (size_t c; (c = next.fetch_add(1)) < nchunk;) hash_chunk(c);
            });
        for (auto& x : th) x.join();
    }
    uint64_t out = 0xcbf29ce484222325ull ^ bytes;
    for (uint64_t v : h) {
        out = (out ^ v) * 0x9e3779b97f4a7c15ull;
        out ^= out >> 32;
    }
    return out;
}

fmm_status fmm_graph_get_info(const fmm_graph* g, fmm_graph_info* out) {
    if (!g || !out) return FMM_E_INVAL;
    fmm_graph_info I{};
    I.m = g->m;
    I.n = g->n;
    I.nnz = g->nnz;
    I.row_begin = g->row_begin;
    I.row_end = g->row_end;
    I.shards = static_cast<int32_t>(g->shards.size());
    I.has_values = g->has_values ? 1 : 0;
    for (const GShard& gs : g->shards) {
        I.exchange_rows += gs.exchange_rows;
        I.exchange_rows_all += gs.exchange_rows_all;
        I.nonempty_rows += gs.nonempty;
        I.max_degree = std::max(I.max_degree, gs.max_degree);
        I.split_rows += gs.n_split_rows;
        I.split_chunks += gs.n_chunks;
    }
    *out = I;
    return FMM_OK;
}

fmm_status fmm_graph_shard_bounds(const fmm_graph* g, int64_t* bounds) {
    if (!g || !bounds) return FMM_E_INVAL;
    for (size_t s = 0; s < g->shards.size(); ++s) bounds[s] = g->shards[s].row_begin;
    bounds[g->shards.size()] = g->row_end;
    return FMM_OK;
}

}  // extern "C"

namespace {

// fmm_run's body; peers (device pointers, single shard) receive every final
// z row as well (the fused exchange of fmm_run_peers).
fmm_status run_impl(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec, int64_t d, const float* X,
                    int64_t ny, const float* Y, float* Z, uint32_t flags, fmm_stats* stats,
                    const fmm::PeerOut* peers) {
    if (!ctx || !g || g->ctx != ctx) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    fmm_status st = check_spec(ctx, spec, d);
    if (st != FMM_OK) return st;
    const int64_t rows = g->row_end - g->row_begin;
    if (ny < 0) return set_err(ctx, FMM_E_INVAL, "fused_mm: negative Y rows");
    // kernel.hpp:278-281: Y must cover every referenced column
    if (g->nnz > 0 && ny < g->max_col + 1) return set_err(ctx, FMM_E_INVAL, "fused_mm: Y has too few rows");
    if (rows > 0 && (!X || !Z)) return set_err(ctx, FMM_E_INVAL, "fused_mm: NULL X or Z");
    if (g->nnz > 0 && !Y) return set_err(ctx, FMM_E_INVAL, "fused_mm: NULL Y");
    const bool dev_ptrs = (flags & FMM_DEVICE_PTRS) != 0;
    const bool async = dev_ptrs && (flags & FMM_ASYNC) != 0;
    if (dev_ptrs && ctx->shards.size() != 1)
        return set_err(ctx, FMM_E_INVAL, "fused_mm: device pointers need a single-shard context");
    const int pattern = pattern_of(*spec);
    bool exact = default_exact(pattern, d);
    if (flags & FMM_EXACT) exact = true;
    if (flags & FMM_FAST) exact = false;
    if (!dev_ptrs && (flags & FMM_ASYNC))
        return run_host_async(ctx, g, *spec, pattern, exact, d, X, ny, Y, Z, stats);
    const size_t row_bytes = static_cast<size_t>(d) * sizeof(float);
    const bool alias = (X == Y) && (ny == g->m);
    int launches = 0;
    size_t aux = 0;
    const bool timed = stats != nullptr && !async;

    for (size_t s = 0; s < g->shards.size(); ++s) {
        const GShard& gs = g->shards[s];
        Shard& sh = ctx->shards[gs.shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        cudaStream_t stream = sh.stream();
        const int64_t srows = gs.row_end - gs.row_begin;
        const float* xd;
        const float* yd;
        float* zd;
        int64_t row0;
        if (timed) FMM_CK(ctx, cudaEventRecord(sh.ev_start, stream));
        if (dev_ptrs) {
            xd = X;
            yd = Y;
            zd = Z + (gs.row_begin - g->row_begin) * d;
            row0 = gs.row_begin;
        } else {
            if ((st = ensure(ctx, sh, sh.Y, std::max<size_t>(1, ny * row_bytes))) != FMM_OK) return st;
            if (ny > 0)
                FMM_CK(ctx, cudaMemcpyAsync(sh.Y.ptr, Y, ny * row_bytes, cudaMemcpyHostToDevice, stream));
            yd = static_cast<const float*>(sh.Y.ptr);
            if (alias) {
                xd = yd;
                row0 = gs.row_begin;
            } else {
                if ((st = ensure(ctx, sh, sh.X, std::max<size_t>(1, srows * row_bytes))) != FMM_OK) return st;
                if (srows > 0)
                    FMM_CK(ctx, cudaMemcpyAsync(sh.X.ptr, X + gs.row_begin * d, srows * row_bytes,
                                                cudaMemcpyHostToDevice, stream));
                xd = static_cast<const float*>(sh.X.ptr);
                row0 = 0;
            }
            if ((st = ensure(ctx, sh, sh.Z, std::max<size_t>(1, srows * row_bytes))) != FMM_OK) return st;
            zd = static_cast<float*>(sh.Z.ptr);
        }
        float* part = nullptr;
        if (!exact && gs.n_slots > 0) {
            const size_t pb = static_cast<size_t>(gs.n_slots) * row_bytes;
            if ((st = ensure(ctx, sh, sh.partial, pb)) != FMM_OK) return st;
            part = static_cast<float*>(sh.partial.ptr);
            aux = std::max(aux, pb);
        }
        if (timed) FMM_CK(ctx, cudaEventRecord(sh.ev_k0, stream));
        float* hs = hscratch(ctx, sh, gs, d, *spec);
        if ((part || hs) && (st = order_scratch(ctx, sh, stream)) != FMM_OK) return st;
        const int l = launch_shard(const_cast<GShard&>(gs), *spec, pattern, d, exact, xd, row0, yd, zd, part,
                                   gs.val, ctx->variant, stream, dev_ptrs ? peers : nullptr, hs,
                                   (flags & FMM_PEERS_ALL) == 0);
        if (l < 0) return set_err(ctx, FMM_E_UNSUPPORTED, "fused_mm: no kernel for this d / alignment");
        if ((part || hs) && (st = mark_scratch(ctx, sh, stream)) != FMM_OK) return st;
        launches += l;
        FMM_CK(ctx, cudaGetLastError());
        if (timed) FMM_CK(ctx, cudaEventRecord(sh.ev_k1, stream));
        if (!dev_ptrs && srows > 0)
            FMM_CK(ctx, cudaMemcpyAsync(Z + (gs.row_begin - g->row_begin) * d, zd, srows * row_bytes,
                                        cudaMemcpyDeviceToHost, stream));
        if (timed) FMM_CK(ctx, cudaEventRecord(sh.ev_end, stream));
    }
    float kms = 0.f, tms = 0.f;
    if (!async) {
        for (const GShard& gs : g->shards) {
            Shard& sh = ctx->shards[gs.shard];
            FMM_CK(ctx, cudaSetDevice(sh.dev));
            FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
            if (timed) {
                kms = std::max(kms, elapsed(sh.ev_k0, sh.ev_k1));
                tms = std::max(tms, elapsed(sh.ev_start, sh.ev_end));
            }
        }
    }
    if (stats) {
        stats->aux_bytes = aux;
        stats->threads = static_cast<int32_t>(g->shards.size());
        stats->pattern = pattern;
        stats->exact = exact ? 1 : 0;
        stats->launches = launches;
        stats->kernel_ms = kms;
        stats->total_ms = tms;
    }
    (void)rows;
    return FMM_OK;
}

}  // namespace

extern "C" {

fmm_status fmm_run(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec, int64_t d,
                   const float* X, int64_t ny, const float* Y, float* Z, uint32_t flags,
                   fmm_stats* stats) {
    return run_impl(ctx, g, spec, d, X, ny, Y, Z, flags, stats, nullptr);
}

fmm_status fmm_run_peers(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec, int64_t d,
                         const float* X, int64_t ny, const float* Y, float* Z, float* const* peers,
                         int npeer, uint32_t flags, fmm_stats* stats) {
    if (!ctx || !g || g->ctx != ctx) return FMM_E_INVAL;
    if (!(flags & FMM_DEVICE_PTRS) || ctx->shards.size() != 1)
        return set_err(ctx, FMM_E_INVAL, "run_peers: device pointers on a single-shard context");
    if (npeer < 0 || npeer > fmm::kMaxPeers || (npeer > 0 && !peers))
        return set_err(ctx, FMM_E_INVAL, "run_peers: 0..7 peer buffers");
    fmm::PeerOut po{};
    for (int q = 0; q < npeer; ++q) {
        if (!peers[q]) return set_err(ctx, FMM_E_INVAL, "run_peers: NULL peer buffer");
        po.p[po.n++] = peers[q];
    }
    return run_impl(ctx, g, spec, d, X, ny, Y, Z, flags, stats, &po);
}

fmm_status fmm_ipc_handle(const void* dptr, void* handle, uint64_t* offset) {
    if (!dptr || !handle || !offset) return FMM_E_INVAL;
    // The handle names the whole allocation dptr lies in (a caching
    // allocator sub-allocates); report dptr's offset from its base.
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            cudaGetLastError();
            return FMM_E_CUDA;
        }
        get_range = reinterpret_cast<GetRange>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS) return FMM_E_CUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
        cudaGetLastError();
        return FMM_E_CUDA;
    }
    static_assert(sizeof(h) == FMM_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    *offset = reinterpret_cast<uint64_t>(dptr) - static_cast<uint64_t>(base);
    return FMM_OK;
}

fmm_status fmm_ipc_open(const void* handle, int device, void** dptr) {
    if (!handle || !dptr) return FMM_E_INVAL;
    *dptr = nullptr;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return FMM_E_CUDA;
    }
    return FMM_OK;
}

fmm_status fmm_ipc_close(void* dptr) {
    if (!dptr) return FMM_E_INVAL;
    if (cudaIpcCloseMemHandle(dptr) != cudaSuccess) {
        cudaGetLastError();
        return FMM_E_CUDA;
    }
    return FMM_OK;
}

fmm_status fmm_run_unfused(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec, int64_t d,
                           const float* X, int64_t ny, const float* Y, float* Z, uint32_t flags,
                           fmm_stats* stats) {
    if (!ctx || !g || g->ctx != ctx) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    fmm_status st = check_spec(ctx, spec, d);
    if (st != FMM_OK) return st;
    if (!(flags & FMM_DEVICE_PTRS) || ctx->shards.size() != 1)
        return set_err(ctx, FMM_E_INVAL, "unfused: device pointers on a single-shard context");
    if (spec->mop == FMM_MOP_MUL_VOP || spec->vop == FMM_VOP_MLP)
        return set_err(ctx, FMM_E_UNSUPPORTED, "unfused: op not in the reference's unfused pipeline");
    if (d != 32 && d != 64 && d != 128 && d != 256)
        return set_err(ctx, FMM_E_UNSUPPORTED, "unfused: d must be 32, 64, 128 or 256");
    if (g->nnz > 0 && ny < g->max_col + 1) return set_err(ctx, FMM_E_INVAL, "fused_mm: Y has too few rows");
    const GShard& gs = g->shards[0];
    Shard& sh = ctx->shards[gs.shard];
    FMM_CK(ctx, cudaSetDevice(sh.dev));
    cudaStream_t stream = sh.stream();
    const bool scalar = spec->rop != FMM_ROP_NOOP;
    const int64_t rows = gs.row_end - gs.row_begin;
    const size_t hbytes = std::max<size_t>(1, static_cast<size_t>(gs.nnz) * (scalar ? 1 : d) * sizeof(float));
    if ((st = ensure(ctx, sh, sh.H, hbytes)) != FMM_OK) return st;
    size_t aux = hbytes;
    const bool timed = stats != nullptr && !(flags & FMM_ASYNC);
    if ((st = order_scratch(ctx, sh, stream)) != FMM_OK) return st;
    if (timed) FMM_CK(ctx, cudaEventRecord(sh.ev_k0, stream));
    // phase 1: SDDMM, H materialised in HBM
    fmm::SddmmParams sp{};
    sp.row_ptr = gs.row_ptr;
    sp.col = gs.col;
    sp.val = gs.val;
    sp.X = X;
    sp.Y = Y;
    sp.H = static_cast<float*>(sh.H.ptr);
    sp.order = gs.order;
    sp.n_rows = rows;
    sp.nnz = gs.nnz;
    sp.row0 = gs.row_begin;
    sp.d = static_cast<int>(d);
    sp.alpha = spec->alpha;
    sp.k = spec->k;
    if (!fmm::launch_sddmm(sp, spec->vop, spec->rop, spec->sop, spec->mop, spec->aop, stream))
        return set_err(ctx, FMM_E_UNSUPPORTED, "unfused: no SDDMM kernel");
    FMM_CK(ctx, cudaGetLastError());
    int launches = 1;
    // phase 2: SpMM over the materialised messages with the row kernels
    fmm_opspec sp2{FMM_VOP_SEL2ND, FMM_ROP_NOOP, FMM_SOP_NOOP, FMM_MOP_MUL, spec->aop, 1.f, 1.f, 0.f, 0.f, 0.f};
    GShard g2 = gs;  // shallow: same device arrays, possibly other columns
    const float* vals = gs.val;
    const float* Ysrc = Y;
    if (spec->mop == FMM_MOP_SEL2ND) {
        vals = nullptr;  // w = y_v
    } else if (scalar) {
        vals = static_cast<const float*>(sh.H.ptr);  // w = h_e * y_v
    } else {
        // w = a_uv * H[e]: gather H rows by edge id
        const size_t ib = std::max<size_t>(1, static_cast<size_t>(gs.nnz) * sizeof(int32_t));
        if ((st = ensure(ctx, sh, sh.iota, ib)) != FMM_OK) return st;
        fmm::launch_iota(static_cast<int32_t*>(sh.iota.ptr), gs.nnz, stream);
        ++launches;
        g2.col = static_cast<int32_t*>(sh.iota.ptr);
        Ysrc = static_cast<const float*>(sh.H.ptr);
        aux += ib;
    }
    float* part = nullptr;
    if (gs.n_slots > 0) {
        const size_t pb = static_cast<size_t>(gs.n_slots) * d * sizeof(float);
        if ((st = ensure(ctx, sh, sh.partial, pb)) != FMM_OK) return st;
        part = static_cast<float*>(sh.partial.ptr);
    }
    const int l = launch_shard(g2, sp2, pattern_of(sp2), d, /*exact=*/false, X, gs.row_begin, Ysrc, Z, part,
                               vals, ctx->variant, stream);
    if (l < 0) return set_err(ctx, FMM_E_UNSUPPORTED, "unfused: no SpMM kernel");
    if ((st = mark_scratch(ctx, sh, stream)) != FMM_OK) return st;
    launches += l;
    FMM_CK(ctx, cudaGetLastError());
    float kms = 0.f;
    if (timed) {
        FMM_CK(ctx, cudaEventRecord(sh.ev_k1, stream));
        FMM_CK(ctx, cudaStreamSynchronize(stream));
        kms = elapsed(sh.ev_k0, sh.ev_k1);
    } else if (!(flags & FMM_ASYNC)) {
        FMM_CK(ctx, cudaStreamSynchronize(stream));
    }
    if (stats) {
        *stats = fmm_stats{};
        stats->aux_bytes = aux;
        stats->threads = 1;
        stats->pattern = pattern_of(*spec);
        stats->exact = 0;
        stats->launches = launches;
        stats->kernel_ms = kms;
        stats->total_ms = kms;
    }
    return FMM_OK;
}

fmm_status fmm_iterate(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec, int64_t d,
                       float* X, int iters, uint32_t flags, fmm_stats* stats) {
    if (!ctx || !g || g->ctx != ctx) return FMM_E_INVAL;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->destroyed) return set_err(ctx, FMM_E_INVAL, "context was destroyed");
    fmm_status st = check_spec(ctx, spec, d);
    if (st != FMM_OK) return st;
    if (iters < 0) return set_err(ctx, FMM_E_INVAL, "iterate: iters must be >= 0");
    if (g->m != g->n || g->row_begin != 0 || g->row_end != g->m)
        return set_err(ctx, FMM_E_INVAL, "iterate: needs a square graph uploaded over all rows");
    if (flags & FMM_DEVICE_PTRS) return set_err(ctx, FMM_E_INVAL, "iterate: host pointers only");
    if (g->m > 0 && !X) return set_err(ctx, FMM_E_INVAL, "iterate: NULL X");
    const int pattern = pattern_of(*spec);
    bool exact = default_exact(pattern, d);
    if (flags & FMM_EXACT) exact = true;
    if (flags & FMM_FAST) exact = false;
    const int64_t m = g->m;
    const size_t row_bytes = static_cast<size_t>(d) * sizeof(float);
    const size_t full = std::max<size_t>(1, m * row_bytes);
    const int S = static_cast<int>(g->shards.size());
    int launches = 0;
    size_t aux = 0;
    // buffers + upload of X0 into every shard's current buffer
    for (int s = 0; s < S; ++s) {
        Shard& sh = ctx->shards[g->shards[s].shard];
        if ((st = ensure(ctx, sh, sh.Y, full)) != FMM_OK) return st;
        if ((st = ensure(ctx, sh, sh.Xb, full)) != FMM_OK) return st;
        const GShard& gs = g->shards[s];
        if (!exact && gs.n_slots > 0) {
            const size_t pb = static_cast<size_t>(gs.n_slots) * row_bytes;
            if ((st = ensure(ctx, sh, sh.partial, pb)) != FMM_OK) return st;
            aux = std::max(aux, pb);
        }
    }
    for (int s = 0; s < S; ++s) {
        Shard& sh = ctx->shards[g->shards[s].shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        FMM_CK(ctx, cudaEventRecord(sh.ev_start, sh.stream()));
        if (m > 0) FMM_CK(ctx, cudaMemcpyAsync(sh.Y.ptr, X, m * row_bytes, cudaMemcpyHostToDevice, sh.stream()));
        FMM_CK(ctx, cudaEventRecord(sh.ev_k0, sh.stream()));
    }
    // Fused exchange (default): each shard's kernels store every finished z
    // row into its own next buffer AND into every peer's (P2P over NVLink, or
    // plain stores for shards sharing a device), so the all-gather overlaps
    // the compute; kernel completion (events) orders the next iteration.
    // FMM_EXCHANGE_COPIES: post-kernel cudaMemcpyPeerAsync slices instead.
    const bool fused = S > 1 && S - 1 <= fmm::kMaxPeers && ctx->p2p_ok && !(flags & FMM_EXCHANGE_COPIES);
    // halo exchange: rows no other shard reads are never sent (R-MAT
    // configs: every empty row, plus rows referenced only locally)
    if (fused && iters > 1 && !g->iter_masks && (st = build_iterate_masks(ctx, const_cast<fmm_graph*>(g))) != FMM_OK)
        return st;
    int cur = 0;  // 0: Y holds the iterate, 1: Xb holds it
    for (int it = 0; it < iters; ++it) {
        const bool exchange = it + 1 < iters && S > 1;
        for (int s = 0; s < S; ++s) {
            const GShard& gs = g->shards[s];
            Shard& sh = ctx->shards[gs.shard];
            FMM_CK(ctx, cudaSetDevice(sh.dev));
            if (it > 0)
                for (int q = 0; q < S; ++q)
                    if (q != s) FMM_CK(ctx, cudaStreamWaitEvent(sh.stream(), ctx->shards[g->shards[q].shard].ev_copy, 0));
            float* xc = static_cast<float*>(cur == 0 ? sh.Y.ptr : sh.Xb.ptr);
            float* xn = static_cast<float*>(cur == 0 ? sh.Xb.ptr : sh.Y.ptr);
            fmm::PeerOut po{};
            if (fused && exchange)
                for (int q = 0; q < S; ++q) {
                    if (q == s) continue;
                    Shard& sq = ctx->shards[g->shards[q].shard];
                    po.p[po.n++] = static_cast<float*>(cur == 0 ? sq.Xb.ptr : sq.Y.ptr) + gs.row_begin * d;
                }
            float* part = static_cast<float*>(sh.partial.ptr);
            float* hs = hscratch(ctx, sh, gs, d, *spec);
            if ((part || hs) && (st = order_scratch(ctx, sh, sh.stream())) != FMM_OK) return st;
            const int l = launch_shard(const_cast<GShard&>(gs), *spec, pattern, d, exact, xc, gs.row_begin, xc,
                                       xn + gs.row_begin * d, part, gs.val, ctx->variant, sh.stream(),
                                       &po, hs, !(flags & FMM_PEERS_ALL));
            if (l < 0) return set_err(ctx, FMM_E_UNSUPPORTED, "iterate: no kernel for this d / alignment");
            if ((part || hs) && (st = mark_scratch(ctx, sh, sh.stream())) != FMM_OK) return st;
            launches += l;
            FMM_CK(ctx, cudaGetLastError());
        }
        // ev_copy of every shard is recorded only after all shards' kernels
        // of this iteration were enqueued: a record inside the launch loop
        // would make shard s's kernel wait for shard q < s's kernel of the
        // SAME iteration (the wait takes the most recent record) and
        // serialise the shards
        if (fused && exchange)
            for (int s = 0; s < S; ++s) {
                Shard& sh = ctx->shards[g->shards[s].shard];
                FMM_CK(ctx, cudaSetDevice(sh.dev));
                FMM_CK(ctx, cudaEventRecord(sh.ev_copy, sh.stream()));
            }
        if (exchange && !fused) {
            // exchange: every shard pushes its fresh Z slice into every peer's next buffer
            for (int s = 0; s < S; ++s) {
                const GShard& gs = g->shards[s];
                Shard& sh = ctx->shards[gs.shard];
                FMM_CK(ctx, cudaSetDevice(sh.dev));
                const float* src = static_cast<const float*>(cur == 0 ? sh.Xb.ptr : sh.Y.ptr) + gs.row_begin * d;
                const size_t bytes = (gs.row_end - gs.row_begin) * row_bytes;
                for (int q = 0; q < S && bytes > 0; ++q) {
                    if (q == s) continue;
                    Shard& sq = ctx->shards[g->shards[q].shard];
                    float* dst = static_cast<float*>(cur == 0 ? sq.Xb.ptr : sq.Y.ptr) + gs.row_begin * d;
                    FMM_CK(ctx, cudaMemcpyPeerAsync(dst, sq.dev, src, sh.dev, bytes, sh.stream()));
                }
                FMM_CK(ctx, cudaEventRecord(sh.ev_copy, sh.stream()));
            }
        }
        cur ^= 1;
    }
    for (int s = 0; s < S; ++s) {
        const GShard& gs = g->shards[s];
        Shard& sh = ctx->shards[gs.shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        FMM_CK(ctx, cudaEventRecord(sh.ev_k1, sh.stream()));
        const float* src = static_cast<const float*>(cur == 0 ? sh.Y.ptr : sh.Xb.ptr) + gs.row_begin * d;
        const size_t bytes = (gs.row_end - gs.row_begin) * row_bytes;
        if (bytes > 0)
            FMM_CK(ctx, cudaMemcpyAsync(X + gs.row_begin * d, src, bytes, cudaMemcpyDeviceToHost, sh.stream()));
        FMM_CK(ctx, cudaEventRecord(sh.ev_end, sh.stream()));
    }
    float kms = 0.f, tms = 0.f;
    for (int s = 0; s < S; ++s) {
        Shard& sh = ctx->shards[g->shards[s].shard];
        FMM_CK(ctx, cudaSetDevice(sh.dev));
        FMM_CK(ctx, cudaStreamSynchronize(sh.stream()));
        kms = std::max(kms, elapsed(sh.ev_k0, sh.ev_k1));
        tms = std::max(tms, elapsed(sh.ev_start, sh.ev_end));
    }
    if (stats) {
        stats->aux_bytes = aux;
        stats->threads = S;
        stats->pattern = pattern;
        stats->exact = exact ? 1 : 0;
        stats->launches = launches;
        stats->kernel_ms = kms;
        stats->total_ms = tms;
    }
    return FMM_OK;
}

}  // extern "C"
