// fusedmm_cuda.hpp — header-only C++ wrapper over libfusedmm_cuda's C ABI
// with the reference driver's signature and exception behaviour:
//
//   reference:  fusedmm::fused_mm(A, X, Y, spec, t, stats, opts)
//               (/root/reference/proj/include/fusedmm/kernel.hpp:297-353)
//   here:       fusedmm::cuda::fused_mm(A, X, Y, spec, t, stats, opts)
//
// The wrapper is generic over the container types: it works with the
// reference's own fusedmm::CsrMatrix<float> / DenseMatrix<float> /
// OpSpec<float> / KernelStats / KernelOptions (so existing host code switches
// by changing the namespace), and with the minimal mirrors in
// fusedmm::cuda::types for code that does not include the reference.
//
// Errors: dimension mismatch and t < 1 throw std::invalid_argument exactly
// where kernel.hpp:269-282,303 does; a USER slot (a std::function the device
// cannot run) throws fusedmm::cuda::unsupported — there is no CPU fallback.
// t is the number of GPU shards (devices 0..n-1 round-robin), the analogue of
// the reference's worker threads; the result is bitwise independent of t.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "fusedmm_cuda.h"

namespace fusedmm {
namespace cuda {

struct unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void throw_status(fmm_status st, const fmm_ctx* ctx = nullptr) {
    if (st == FMM_OK) return;
    std::string msg = ctx ? fmm_last_error(ctx) : "";
    if (msg.empty()) msg = fmm_status_string(st);
    switch (st) {
        case FMM_E_INVAL: throw std::invalid_argument(msg);
        case FMM_E_LOGIC: throw std::logic_error(msg);
        case FMM_E_UNSUPPORTED: throw unsupported(msg);
        case FMM_E_OOM: throw std::bad_alloc();
        default: throw device_error(msg);
    }
}

// Minimal containers with the reference field names (matrix.hpp:18-68,
// ops.hpp:22-51, kernel.hpp:51-55,286-288) for users without the reference.
namespace types {
enum class Vop { ADD, MUL, SEL2ND, SUB, USER };
enum class Rop { NOOP, RSUM, RMUL, NORM, USER };
enum class Sop { NOOP, SIGMOID, SCAL, USER };
enum class Mop { MUL, SEL2ND, USER };
enum class Aop { ASUM, AMAX, USER };
enum class KnownPattern { SIGMOID_EMBED, SPMM_GCN, FR_LAYOUT, GENERIC };

struct DenseMatrix {
    int64_t nrows = 0, dim = 0;
    std::vector<float> data;
    DenseMatrix() = default;
    DenseMatrix(int64_t rows, int64_t d, float fill = 0.f)
        : nrows(rows), dim(d), data(static_cast<size_t>(rows * d), fill) {}
};
struct CsrMatrix {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> row_ptr{0}, col_idx;
    std::vector<float> values;
    int64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
};
struct OpSpec {
    Vop vop = Vop::MUL;
    Rop rop = Rop::RSUM;
    Sop sop = Sop::NOOP;
    Mop mop = Mop::MUL;
    Aop aop = Aop::ASUM;
    float alpha = 1.f;
};
struct KernelStats {
    std::size_t aux_bytes = 0;
    int threads = 0;
    KnownPattern pattern = KnownPattern::GENERIC;
};
struct KernelOptions {
    int lane_width = 8;
};
}  // namespace types

// Device-only op descriptor for the patterns the reference can only express
// through a USER VOP lambda (configs 3 and 4).
inline fmm_opspec tdist_ops() {
    return fmm_opspec{FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_TDIST, FMM_MOP_MUL_VOP, FMM_AOP_ASUM, 1.f, 1.f};
}
inline fmm_opspec fr_attract_ops(float k) {
    return fmm_opspec{FMM_VOP_SUB, FMM_ROP_SQNORM, FMM_SOP_SQK, FMM_MOP_MUL_VOP, FMM_AOP_ASUM, 1.f, k};
}

// One context per shard count, one uploaded graph cached per context. The
// cache is keyed on the CONTENTS of A (fmm_fingerprint of row_ptr, col_idx
// and values), never on its addresses: the reference reads A afresh on
// every call (kernel.hpp:297-353), so a CSR rebuilt at the same addresses or
// edited in place is re-uploaded (values-only changes are re-sent in place).
// Every call on a context holds its mutex (graph lookup + run), so two host
// threads sharing a shard count cannot free each other's graph.
class Context {
public:
    explicit Context(int t) : t_(t) {
        const int ndev = fmm_device_count();
        if (ndev < 1) throw device_error("fusedmm::cuda: no CUDA device (no CPU fallback)");
        std::vector<int> devs(static_cast<size_t>(t));
        for (int i = 0; i < t; ++i) devs[i] = i % ndev;
        throw_status(fmm_create(t, devs.data(), &ctx_));
    }
    ~Context() {
        if (graph_) fmm_graph_free(graph_);
        if (ctx_) fmm_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    static Context& for_shards(int t) {
        static std::mutex mu;
        static std::vector<std::unique_ptr<Context>> pool;
        std::lock_guard<std::mutex> lk(mu);
        for (auto& c : pool)
            if (c->t_ == t) return *c;
        pool.emplace_back(new Context(t));
        return *pool.back();
    }

    // The device copy of A, uploaded (or its values refreshed) when A's
    // contents differ from the cached graph's. Caller holds mutex().
    template <class Csr>
    fmm_graph* graph_for(const Csr& A) {
        const uint64_t rp = fmm_fingerprint(A.row_ptr.data(), A.row_ptr.size() * sizeof(A.row_ptr[0]));
        const uint64_t ci = fmm_fingerprint(A.col_idx.data(), A.col_idx.size() * sizeof(A.col_idx[0]));
        const uint64_t va = fmm_fingerprint(A.values.data(), A.values.size() * sizeof(float));
        const int64_t shape[3] = {static_cast<int64_t>(A.nrows), static_cast<int64_t>(A.ncols),
                                  static_cast<int64_t>(A.nnz())};
        const bool same_structure = graph_ && rp == rp_ && ci == ci_ && std::memcmp(shape, shape_, sizeof(shape)) == 0;
        if (same_structure) {
            if (va != va_) {
                throw_status(fmm_graph_update_values(graph_, A.values.empty() ? nullptr : A.values.data()), ctx_);
                va_ = va;
            }
            return graph_;
        }
        if (graph_) fmm_graph_free(graph_);
        graph_ = nullptr;
        throw_status(fmm_graph_upload(ctx_, A.nrows, A.ncols, A.row_ptr.data(),
                                      A.col_idx.empty() ? nullptr : A.col_idx.data(),
                                      A.values.empty() ? nullptr : A.values.data(), 0, A.nrows,
                                      &graph_),
                     ctx_);
        rp_ = rp;
        ci_ = ci;
        va_ = va;
        std::memcpy(shape_, shape, sizeof(shape));
        return graph_;
    }
    fmm_ctx* get() const { return ctx_; }
    std::mutex& mutex() { return mu_; }

private:
    fmm_ctx* ctx_ = nullptr;
    fmm_graph* graph_ = nullptr;
    uint64_t rp_ = 0, ci_ = 0, va_ = 0;
    int64_t shape_[3] = {-1, -1, -1};
    int t_ = 0;
    std::mutex mu_;
};

// KernelOptions::lane_width (kernel.hpp:286-288) on the device: 4 selects
// the 128-bit-gather shapes (variant 20), 8 and 16 the default 256-bit
// shapes. tune_lane_width below times them.
inline int variant_for_lane_width(int w) { return w == 4 ? 20 : -1; }

namespace detail {

// kernel.hpp:269-282, same conditions and messages
template <class Csr, class Dense>
void check_dims(const Csr& A, const Dense& X, const Dense& Y) {
    if (X.nrows != A.nrows) throw std::invalid_argument("fused_mm: X.nrows != A.nrows");
    if (X.dim != Y.dim) throw std::invalid_argument("fused_mm: X.dim != Y.dim");
    if (Y.nrows < A.ncols) {
        int64_t max_col = -1;
        for (auto c : A.col_idx) max_col = std::max<int64_t>(max_col, c);
        if (Y.nrows < max_col + 1) throw std::invalid_argument("fused_mm: Y has too few rows");
    }
}

template <class Spec>
fmm_opspec to_c(const Spec& s) {
    return fmm_opspec{static_cast<int32_t>(s.vop), static_cast<int32_t>(s.rop),
                      static_cast<int32_t>(s.sop), static_cast<int32_t>(s.mop),
                      static_cast<int32_t>(s.aop), static_cast<float>(s.alpha), 1.f};
}

template <class Csr, class Dense, class Stats>
Dense run(const Csr& A, const Dense& X, const Dense& Y, const fmm_opspec& c, int t, Stats* stats,
          int lane_width = 8) {
    check_dims(A, X, Y);
    if (t < 1) throw std::invalid_argument("fused_mm: t must be >= 1");
    if (lane_width != 4 && lane_width != 8 && lane_width != 16)
        throw std::invalid_argument("KernelOptions.lane_width must be 4, 8 or 16");
    Dense Z(A.nrows, X.dim);
    fmm_stats st{};
    if (A.nrows > 0) {
        Context& ctx = Context::for_shards(t);
        std::lock_guard<std::mutex> lk(ctx.mutex());
        fmm_graph* g = ctx.graph_for(A);
        const float* y = (&X == &Y) ? X.data.data() : Y.data.data();
        const int prev = fmm_get_variant(ctx.get());
        fmm_set_variant(ctx.get(), variant_for_lane_width(lane_width));
        const fmm_status rs = fmm_run(ctx.get(), g, &c, X.dim, X.data.data(), Y.nrows, y, Z.data.data(),
                                      FMM_HOST_PTRS, &st);
        fmm_set_variant(ctx.get(), prev);
        throw_status(rs, ctx.get());
    } else {
        int32_t pat = FMM_PATTERN_GENERIC;
        fmm_pattern_of(&c, &pat);
        st.pattern = pat;
        st.threads = t;
    }
    if (stats) {
        stats->aux_bytes = static_cast<decltype(stats->aux_bytes)>(st.aux_bytes);
        stats->threads = st.threads;
        // device-only patterns are GENERIC in the reference's enum
        const int p = st.pattern <= FMM_PATTERN_GENERIC ? st.pattern : FMM_PATTERN_GENERIC;
        stats->pattern = static_cast<decltype(stats->pattern)>(p);
    }
    return Z;
}

struct NoStats {
    std::size_t aux_bytes;
    int threads;
    int pattern;
};

}  // namespace detail

// Drop-in for fusedmm::fused_mm<float> (kernel.hpp:297-353).
template <class Csr, class Dense, class Spec, class Stats = detail::NoStats,
          class Opts = types::KernelOptions>
Dense fused_mm(const Csr& A, const Dense& X, const Dense& Y, const Spec& spec, int t,
               Stats* stats = nullptr, const Opts& opts = {}) {
    const bool user = static_cast<int>(spec.vop) == FMM_VOP_USER ||
                      static_cast<int>(spec.rop) == FMM_ROP_USER ||
                      static_cast<int>(spec.sop) == FMM_SOP_USER ||
                      static_cast<int>(spec.mop) == FMM_MOP_USER ||
                      static_cast<int>(spec.aop) == FMM_AOP_USER;
    if (user) {
        detail::check_dims(A, X, Y);
        throw unsupported("fused_mm: USER slot has no device kernel (use a device op descriptor)");
    }
    return detail::run(A, X, Y, detail::to_c(spec), t, stats, opts.lane_width);
}

// Overload taking the device op descriptor (configs 3/4: tdist_ops(),
// fr_attract_ops(k)), since a std::function cannot be introspected.
template <class Csr, class Dense, class Stats = detail::NoStats>
Dense fused_mm(const Csr& A, const Dense& X, const Dense& Y, const fmm_opspec& ops, int t,
               Stats* stats = nullptr) {
    return detail::run(A, X, Y, ops, t, stats);
}

// update_u (kernel.hpp:81-107): one vertex update, z_u = fold over the
// stored neighbours (cols, vals) of the five slots, on the device. Spans are
// any contiguous ranges with data()/size(); scratch is accepted for
// signature parity (the device keeps x_u and z_u in registers). Runs as a
// one-row fused call (graph uploaded per call), so it is for single-vertex
// use, not for loops over every row — fused_mm is.
template <class ColSpan, class ValSpan, class XSpan, class Dense, class Spec, class ZSpan, class Scratch>
void update_u(const ColSpan& cols, const ValSpan& vals, const XSpan& x_u, const Dense& Y, const Spec& spec,
              ZSpan&& z_u, Scratch&& scratch) {
    (void)scratch;
    const int64_t d = static_cast<int64_t>(x_u.size());
    const int64_t k = static_cast<int64_t>(cols.size());
    if (static_cast<int64_t>(z_u.size()) != d || static_cast<int64_t>(Y.dim) != d)
        throw std::invalid_argument("update_u: length mismatch");
    if (static_cast<int64_t>(vals.size()) != k) throw std::invalid_argument("update_u: cols / vals differ in length");
    types::CsrMatrix A;
    A.nrows = 1;
    A.ncols = static_cast<int64_t>(Y.nrows);
    A.row_ptr = {0, k};
    A.col_idx.assign(cols.data(), cols.data() + k);
    A.values.assign(vals.data(), vals.data() + k);
    types::DenseMatrix X(1, d), Yc(static_cast<int64_t>(Y.nrows), d);
    std::copy(x_u.data(), x_u.data() + d, X.data.begin());
    std::copy(Y.data.data(), Y.data.data() + Yc.data.size(), Yc.data.begin());
    const types::DenseMatrix Z = fused_mm(A, X, Yc, spec, 1);
    std::copy(Z.data.begin(), Z.data.end(), z_u.data());
}

// fused_mm_specialized (kernel.hpp:356-378): direct entry to a fast path;
// GENERIC (or any other value) throws std::invalid_argument as there.
template <class Pattern, class Csr, class Dense, class T, class Opts = types::KernelOptions>
Dense fused_mm_specialized(Pattern pattern, const Csr& A, const Dense& X, const Dense& Y, T alpha, int t,
                           const Opts& opts = {}) {
    fmm_opspec c{};
    switch (static_cast<int>(pattern)) {
        case FMM_PATTERN_SIGMOID_EMBED:
            c = fmm_opspec{FMM_VOP_MUL, FMM_ROP_RSUM, FMM_SOP_SIGMOID, FMM_MOP_MUL, FMM_AOP_ASUM, 1.f, 1.f};
            break;
        case FMM_PATTERN_SPMM_GCN:
            c = fmm_opspec{FMM_VOP_SEL2ND, FMM_ROP_NOOP, FMM_SOP_NOOP, FMM_MOP_MUL, FMM_AOP_ASUM, 1.f, 1.f};
            break;
        case FMM_PATTERN_FR_LAYOUT:
            c = fmm_opspec{FMM_VOP_ADD, FMM_ROP_NORM, FMM_SOP_SCAL, FMM_MOP_MUL, FMM_AOP_ASUM,
                           static_cast<float>(alpha), 1.f};
            break;
        default:
            throw std::invalid_argument("fused_mm_specialized: pattern has no fast path");
    }
    return detail::run(A, X, Y, c, t, static_cast<detail::NoStats*>(nullptr), opts.lane_width);
}

// tune_lane_width (kernel.hpp:382-402): times the device shape families the
// lane widths select (4: 128-bit gathers, 8: the default 256-bit shapes;
// 16 selects the same shapes as 8) and returns the fastest width.
template <class Csr, class Dense, class Spec>
int tune_lane_width(const Csr& A, const Dense& X, const Dense& Y, const Spec& spec, int t, int repeats = 3) {
    int best_w = 8;
    double best = 1e300;
    for (int w : {4, 8}) {
        types::KernelOptions opts{w};
        (void)fused_mm(A, X, Y, spec, t, static_cast<detail::NoStats*>(nullptr), opts);  // warm-up
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < repeats; ++r)
            (void)fused_mm(A, X, Y, spec, t, static_cast<detail::NoStats*>(nullptr), opts);
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (secs < best) {
            best = secs;
            best_w = w;
        }
    }
    return best_w;
}

// csr_from_coo on the GPU (matrix.hpp:87-140): same signature shape as the
// reference (entries with .row/.col/.value, m, n), same result, same
// std::invalid_argument for an out-of-bounds entry. Csr is the caller's CSR
// type (the reference's CsrMatrix<float> or types::CsrMatrix).
template <class Csr, class Entry>
Csr csr_from_coo(const std::vector<Entry>& entries, int64_t m, int64_t n, int device = 0) {
    const size_t cnt = entries.size();
    std::vector<int64_t> rows(cnt), cols(cnt);
    std::vector<float> vals(cnt);
    for (size_t i = 0; i < cnt; ++i) {
        rows[i] = entries[i].row;
        cols[i] = entries[i].col;
        vals[i] = static_cast<float>(entries[i].value);
    }
    Csr A;
    A.nrows = m;
    A.ncols = n;
    A.row_ptr.assign(static_cast<size_t>(m) + 1, 0);
    A.col_idx.assign(cnt, 0);
    A.values.assign(cnt, 0.f);
    int64_t nnz = 0;
    const fmm_status st = fmm_csr_from_coo(device, m, n, static_cast<int64_t>(cnt), rows.data(), cols.data(),
                                           vals.data(), A.row_ptr.data(), A.col_idx.data(), A.values.data(), &nnz);
    if (st == FMM_E_INVAL) throw std::invalid_argument("csr_from_coo: entry out of bounds");
    throw_status(st);
    A.col_idx.resize(static_cast<size_t>(nnz));
    A.values.resize(static_cast<size_t>(nnz));
    return A;
}

}  // namespace cuda
}  // namespace fusedmm
