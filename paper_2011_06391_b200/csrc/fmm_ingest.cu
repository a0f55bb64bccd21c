// fmm_ingest.cu — device-side graph construction.
//
//   fmm_csr_from_coo   the reference's csr_from_coo (matrix.hpp:87-140) on the
//                      GPU: bounds check, duplicate (row, col) entries summed in
//                      insertion order into the first occurrence, per-row
//                      storage order = first-occurrence order. Applied to the
//                      R-MAT insertion stream it is rmat_generate (rmat.hpp:
//                      24-61: self-loops kept, duplicates summed).
//   fmm_csr_sym_unique the BASELINE.json graph recipe for configs 2, 3, 5:
//                      drop self-loops, add (u,v) and (v,u), sort, unique,
//                      a_uv = 1 (sorted columns per row).
//
// Both run as stable LSD radix sorts (CUB) over packed 64-bit keys
// (row << 32 | col, then row << 32 | first-occurrence index for the storage
// order), a segmented fold of duplicate groups (one thread per group, values
// added left to right in insertion order, so the sums are bit-identical to the
// reference's sequential `+=`), and a per-row count + scan for row_ptr.
// Host arrays in, host arrays out, like the reference's value-returning API.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fmm_mt64.h"
#include "fusedmm_cuda.h"

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n) {
    return static_cast<int>(std::min<int64_t>(std::max<int64_t>((n + kThreads - 1) / kThreads, 1), 148 * 32));
}

inline int bits_for(uint64_t v) {  // bits needed to represent values < v (v >= 1)
    int b = 0;
    while (b < 64 && (uint64_t(1) << b) < v) ++b;
    return std::max(b, 1);
}

__global__ void coo_keys_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols, int64_t count,
                                int64_t m, int64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                                int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        if (r < 0 || r >= m || c < 0 || c >= n) {
            atomicExch(bad, 1);
            keys[i] = 0;
        } else {
            keys[i] = (static_cast<uint64_t>(r) << 32) | static_cast<uint64_t>(c);
        }
        idx[i] = static_cast<uint32_t>(i);
    }
}

__global__ void heads_kernel(const uint64_t* __restrict__ keys, int64_t count, uint32_t* __restrict__ head) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// One thread per duplicate group (its head): the group's entries sit in
// insertion order after the stable sort; fold their values left to right.
__global__ void fold_groups_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ sidx,
                                   const uint32_t* __restrict__ head, const uint32_t* __restrict__ uid,
                                   int64_t count, const float* __restrict__ vals, uint64_t* __restrict__ key2,
                                   uint32_t* __restrict__ uorder, int32_t* __restrict__ ucol,
                                   float* __restrict__ uval) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!head[i]) continue;
        const uint32_t u = uid[i];
        const uint32_t first = sidx[i];
        float sum = vals ? vals[first] : 1.0f;
        for (int64_t j = i + 1; j < count && !head[j]; ++j) sum = __fadd_rn(sum, vals ? vals[sidx[j]] : 1.0f);
        const uint64_t row = keys[i] >> 32;
        key2[u] = (row << 32) | first;
        uorder[u] = u;
        ucol[u] = static_cast<int32_t>(keys[i] & 0xffffffffu);
        uval[u] = sum;
    }
}

__global__ void emit_kernel(const uint64_t* __restrict__ key2, const uint32_t* __restrict__ ord,
                            const int32_t* __restrict__ ucol, const float* __restrict__ uval, int64_t U,
                            int64_t* __restrict__ col_out, float* __restrict__ val_out,
                            unsigned long long* __restrict__ counts) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < U;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t u = ord[i];
        col_out[i] = ucol[u];
        if (val_out) val_out[i] = uval[u];
        atomicAdd(counts + (key2[i] >> 32) + 1, 1ull);
    }
}

// Sorted-unique symmetric recipe: keys of (u,v) and (v,u) for u != v.
__global__ void sym_keys_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols, int64_t count,
                                int64_t n, int drop_self, int symmetrize, uint64_t* __restrict__ keys,
                                int* __restrict__ bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        const uint64_t none = ~uint64_t(0);  // sorts last, dropped
        uint64_t k0 = none, k1 = none;
        if (r < 0 || r >= n || c < 0 || c >= n) {
            atomicExch(bad, 1);
        } else if (!(drop_self && r == c)) {
            k0 = (static_cast<uint64_t>(r) << 32) | static_cast<uint64_t>(c);
            if (symmetrize) k1 = (static_cast<uint64_t>(c) << 32) | static_cast<uint64_t>(r);
        }
        keys[2 * i] = k0;
        keys[2 * i + 1] = k1;
    }
}

__global__ void unique_emit_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ head,
                                   const uint32_t* __restrict__ uid, int64_t count, int64_t* __restrict__ col_out,
                                   unsigned long long* __restrict__ counts) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!head[i] || keys[i] == ~uint64_t(0)) continue;
        col_out[uid[i]] = static_cast<int64_t>(keys[i] & 0xffffffffu);
        atomicAdd(counts + (keys[i] >> 32) + 1, 1ull);
    }
}

// RAII device allocations for one call.
struct Scratch {
    std::vector<void*> ptrs;
    ~Scratch() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        *p = nullptr;
        const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
};

fmm_status status_of(cudaError_t e) {
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? FMM_E_OOM : FMM_E_CUDA;
}

#define ING_CK(call)                                \
    do {                                            \
        const cudaError_t e_ = (call);              \
        if (e_ != cudaSuccess) return status_of(e_); \
    } while (0)

// row_ptr[0..m] = exclusive scan of the per-row counts (counts[r + 1] = degree of r).
fmm_status counts_to_row_ptr(Scratch& S, unsigned long long* counts, int64_t m, int64_t* row_ptr_host,
                             cudaStream_t st) {
    unsigned long long* scanned;
    ING_CK(S.alloc(&scanned, m + 1));
    size_t tmp = 0;
    ING_CK(cub::DeviceScan::InclusiveSum(nullptr, tmp, counts, scanned, m + 1, st));
    void* t;
    ING_CK(S.alloc(reinterpret_cast<char**>(&t), tmp));
    ING_CK(cub::DeviceScan::InclusiveSum(t, tmp, counts, scanned, m + 1, st));
    static_assert(sizeof(unsigned long long) == sizeof(int64_t), "row_ptr width");
    ING_CK(cudaMemcpyAsync(row_ptr_host, scanned, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    return FMM_OK;
}

// ---- the R-MAT insertion stream on the device (rmat.hpp:32-58) ----------
// One warp per sub-stream of E edges (E*scale words, a multiple of 312): the
// sub-stream's mt19937_64 window comes from the host jump-ahead
// (fmm_mt64.cpp); the warp twists 312 words at a time (two phases: words
// 0..155 depend only on the old window, 156..311 also on the new 0..155),
// tempers them, and descends `scale` quadrant levels per edge from its
// consecutive words. u01 < t is evaluated exactly as (r >> 11) < ceil(t*2^53)
// (u01 = (r >> 11) * 2^-53 is exact in double), so the stream is bitwise the
// reference's sequential one.
constexpr int kMtN = 312, kMtM = 156;
constexpr int kGenWarps = 4;

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}
__device__ __forceinline__ uint64_t mt_next(uint64_t x0, uint64_t x1, uint64_t xm) {
    const uint64_t y = (x0 & 0xFFFFFFFF80000000ull) | (x1 & 0x7FFFFFFFull);
    return xm ^ (y >> 1) ^ ((x1 & 1) ? 0xB5026F5AA96619E9ull : 0ull);
}

__global__ void __launch_bounds__(32 * kGenWarps)
rmat_stream_kernel(const uint64_t* __restrict__ windows, int64_t nstreams, int64_t edges_per_stream, int64_t nedges,
                   int scale, uint64_t ta, uint64_t tab, uint64_t tabc, int64_t* __restrict__ rows,
                   int64_t* __restrict__ cols) {
    __shared__ uint64_t raw[kGenWarps][2][kMtN];   // window, next window
    __shared__ uint64_t tmp[kGenWarps][2][kMtN];   // tempered words of the last two chunks
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t sid = static_cast<int64_t>(blockIdx.x) * kGenWarps + wl;
    if (sid >= nstreams) return;
    const int64_t e_begin = sid * edges_per_stream;
    const int64_t e_end = min(nedges, e_begin + edges_per_stream);
    for (int i = lane; i < kMtN; i += 32) raw[wl][0][i] = windows[sid * kMtN + i];
    __syncwarp();
    int cur = 0;
    int64_t chunk = 0, e = e_begin;
    while (e < e_end) {
        const uint64_t* o = raw[wl][cur];
        uint64_t* nw = raw[wl][cur ^ 1];
        for (int i = lane; i < kMtM; i += 32) nw[i] = mt_next(o[i], o[i + 1], o[i + kMtM]);
        __syncwarp();
        for (int i = kMtM + lane; i < kMtN; i += 32)
            nw[i] = mt_next(o[i], i + 1 < kMtN ? o[i + 1] : nw[0], nw[i - kMtM]);
        __syncwarp();
        uint64_t* tw = tmp[wl][chunk & 1];
        for (int i = lane; i < kMtN; i += 32) tw[i] = mt_temper(nw[i]);
        __syncwarp();
        cur ^= 1;
        // edges whose words all lie in chunks <= this one
        const int64_t words_avail = (chunk + 1) * kMtN;
        const int64_t e_lim = min(e_end, e_begin + words_avail / scale);
        for (int64_t eb = e; eb < e_lim; eb += 32) {
            const int64_t ee = eb + lane;
            if (ee < e_lim) {
                int64_t w = (ee - e_begin) * scale;
                uint64_t row = 0, col = 0;
                for (int level = 0; level < scale; ++level, ++w) {
                    const uint64_t k = tmp[wl][(w / kMtN) & 1][w % kMtN] >> 11;
                    row <<= 1;
                    col <<= 1;
                    if (k < ta) {
                    } else if (k < tab) {
                        col |= 1;
                    } else if (k < tabc) {
                        row |= 1;
                    } else {
                        row |= 1;
                        col |= 1;
                    }
                }
                rows[ee] = static_cast<int64_t>(row);
                cols[ee] = static_cast<int64_t>(col);
            }
        }
        e = e_lim;
        ++chunk;
        __syncwarp();
    }
}

// rows/cols[0..nedges) = the stream of rmat_generate(scale, nedges/2^scale,
// a, b, c, seed) (device arrays)
fmm_status rmat_stream_dev(cudaStream_t st, Scratch& S, int scale, int64_t nedges, double a, double b, double c,
                           uint64_t seed, int64_t* d_rows, int64_t* d_cols) {
    if (nedges == 0) return FMM_OK;
    // sub-stream length: E edges, E*scale a multiple of 312 words
    int64_t unit = kMtN / std::gcd<int64_t>(kMtN, scale);
    const int64_t target = std::max<int64_t>(1, nedges / 2048);
    const int64_t E = ((target + unit - 1) / unit) * unit;
    const int64_t nstreams = (nedges + E - 1) / E;
    const std::vector<uint64_t> win = fmm::mt64::windows(seed, static_cast<uint64_t>(E * scale), nstreams);
    uint64_t* d_win;
    ING_CK(S.alloc(&d_win, win.size()));
    ING_CK(cudaMemcpyAsync(d_win, win.data(), win.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    auto thr = [](double t) { return static_cast<uint64_t>(std::ceil(t * 0x1.0p53)); };
    const uint64_t ta = thr(a), tab = thr(a + b), tabc = thr(a + b + c);
    const unsigned blocks = static_cast<unsigned>((nstreams + kGenWarps - 1) / kGenWarps);
    rmat_stream_kernel<<<blocks, 32 * kGenWarps, 0, st>>>(d_win, nstreams, E, nedges, scale, ta, tab, tabc, d_rows,
                                                           d_cols);
    ING_CK(cudaGetLastError());
    ING_CK(cudaStreamSynchronize(st));  // win (host vector) is released on return
    return FMM_OK;
}

// csr_from_coo over device arrays d_rows / d_cols / d_vals (nullable),
// results copied to the host arrays. Caller set the device.
fmm_status csr_from_coo_dev(cudaStream_t st, Scratch& S, int64_t m, int64_t n, int64_t count, const int64_t* d_rows,
                            const int64_t* d_cols, const float* d_vals, int64_t* row_ptr, int64_t* col_idx,
                            float* values, int64_t* nnz_out) {
    uint64_t *keys, *keys_s;
    uint32_t *idx, *idx_s;
    int* bad;
    ING_CK(S.alloc(&keys, count));
    ING_CK(S.alloc(&keys_s, count));
    ING_CK(S.alloc(&idx, count));
    ING_CK(S.alloc(&idx_s, count));
    ING_CK(S.alloc(&bad, 1));
    ING_CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    if (count > 0) {
        coo_keys_kernel<<<grid_for(count), kThreads, 0, st>>>(d_rows, d_cols, count, m, n, keys, idx, bad);
        ING_CK(cudaGetLastError());
    }
    int h_bad = 0;
    ING_CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    ING_CK(cudaStreamSynchronize(st));
    if (h_bad) return FMM_E_INVAL;  // matrix.hpp:89-95: entry out of bounds
    unsigned long long* counts;
    ING_CK(S.alloc(&counts, m + 1));
    ING_CK(cudaMemsetAsync(counts, 0, (m + 1) * sizeof(unsigned long long), st));
    int64_t U = 0;
    if (count > 0) {
        // 1) stable sort by (row, col): duplicate groups in insertion order
        const int end_bit = 32 + bits_for(static_cast<uint64_t>(m));
        size_t tmp = 0;
        ING_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys_s, idx, idx_s, count, 0, end_bit, st));
        char* t;
        ING_CK(S.alloc(&t, tmp));
        ING_CK(cub::DeviceRadixSort::SortPairs(t, tmp, keys, keys_s, idx, idx_s, count, 0, end_bit, st));
        // 2) group heads, unique ids
        uint32_t *head, *uid;
        ING_CK(S.alloc(&head, count));
        ING_CK(S.alloc(&uid, count));
        heads_kernel<<<grid_for(count), kThreads, 0, st>>>(keys_s, count, head);
        size_t tmp2 = 0;
        ING_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, head, uid, count, st));
        char* t2;
        ING_CK(S.alloc(&t2, tmp2));
        ING_CK(cub::DeviceScan::ExclusiveSum(t2, tmp2, head, uid, count, st));
        uint32_t last_uid = 0, last_head = 0;
        ING_CK(cudaMemcpyAsync(&last_uid, uid + count - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaMemcpyAsync(&last_head, head + count - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaStreamSynchronize(st));
        U = static_cast<int64_t>(last_uid) + last_head;
        // 3) fold each group; key2 = (row, first occurrence)
        uint64_t *key2, *key2_s;
        uint32_t *uord, *uord_s;
        int32_t* ucol;
        float* uval;
        ING_CK(S.alloc(&key2, U));
        ING_CK(S.alloc(&key2_s, U));
        ING_CK(S.alloc(&uord, U));
        ING_CK(S.alloc(&uord_s, U));
        ING_CK(S.alloc(&ucol, U));
        ING_CK(S.alloc(&uval, U));
        fold_groups_kernel<<<grid_for(count), kThreads, 0, st>>>(keys_s, idx_s, head, uid, count, d_vals, key2,
                                                                  uord, ucol, uval);
        ING_CK(cudaGetLastError());
        // 4) storage order: sort by (row, first occurrence)
        size_t tmp3 = 0;
        ING_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp3, key2, key2_s, uord, uord_s, U, 0, end_bit, st));
        char* t3;
        ING_CK(S.alloc(&t3, tmp3));
        ING_CK(cub::DeviceRadixSort::SortPairs(t3, tmp3, key2, key2_s, uord, uord_s, U, 0, end_bit, st));
        // 5) emit columns / values, per-row counts
        int64_t* d_col_out;
        float* d_val_out = nullptr;
        ING_CK(S.alloc(&d_col_out, U));
        if (values) ING_CK(S.alloc(&d_val_out, U));
        emit_kernel<<<grid_for(U), kThreads, 0, st>>>(key2_s, uord_s, ucol, uval, U, d_col_out, d_val_out, counts);
        ING_CK(cudaGetLastError());
        ING_CK(cudaMemcpyAsync(col_idx, d_col_out, U * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        if (values) ING_CK(cudaMemcpyAsync(values, d_val_out, U * sizeof(float), cudaMemcpyDeviceToHost, st));
    }
    fmm_status s = counts_to_row_ptr(S, counts, m, row_ptr, st);
    if (s != FMM_OK) return s;
    ING_CK(cudaStreamSynchronize(st));
    *nnz_out = U;
    return FMM_OK;
}

// the BASELINE recipe over device arrays (see fmm_csr_sym_unique)
fmm_status sym_unique_dev(cudaStream_t st, Scratch& S, int64_t n, int64_t count, const int64_t* d_rows,
                          const int64_t* d_cols, int drop_self, int symmetrize, int64_t* row_ptr, int64_t* col_idx,
                          int64_t* nnz_out) {
    const int64_t nk = 2 * count;
    uint64_t *keys, *keys_s;
    int* bad;
    ING_CK(S.alloc(&keys, nk));
    ING_CK(S.alloc(&keys_s, nk));
    ING_CK(S.alloc(&bad, 1));
    ING_CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    if (count > 0) {
        sym_keys_kernel<<<grid_for(count), kThreads, 0, st>>>(d_rows, d_cols, count, n, drop_self, symmetrize, keys,
                                                               bad);
        ING_CK(cudaGetLastError());
    }
    int h_bad = 0;
    ING_CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    ING_CK(cudaStreamSynchronize(st));
    if (h_bad) return FMM_E_INVAL;
    unsigned long long* counts;
    ING_CK(S.alloc(&counts, n + 1));
    ING_CK(cudaMemsetAsync(counts, 0, (n + 1) * sizeof(unsigned long long), st));
    int64_t U = 0;
    if (count > 0) {
        size_t tmp = 0;
        ING_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, keys_s, nk, 0, 64, st));
        char* t;
        ING_CK(S.alloc(&t, tmp));
        ING_CK(cub::DeviceRadixSort::SortKeys(t, tmp, keys, keys_s, nk, 0, 64, st));
        uint32_t *head, *uid;
        ING_CK(S.alloc(&head, nk));
        ING_CK(S.alloc(&uid, nk));
        heads_kernel<<<grid_for(nk), kThreads, 0, st>>>(keys_s, nk, head);
        size_t tmp2 = 0;
        ING_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, head, uid, nk, st));
        char* t2;
        ING_CK(S.alloc(&t2, tmp2));
        ING_CK(cub::DeviceScan::ExclusiveSum(t2, tmp2, head, uid, nk, st));
        // unique count excluding the dropped-entry sentinel group (sorts last)
        uint32_t last_uid = 0, last_head = 0;
        uint64_t last_key = 0;
        ING_CK(cudaMemcpyAsync(&last_uid, uid + nk - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaMemcpyAsync(&last_head, head + nk - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaMemcpyAsync(&last_key, keys_s + nk - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaStreamSynchronize(st));
        U = static_cast<int64_t>(last_uid) + last_head - (last_key == ~uint64_t(0) ? 1 : 0);
        int64_t* d_col_out;
        ING_CK(S.alloc(&d_col_out, U));
        unique_emit_kernel<<<grid_for(nk), kThreads, 0, st>>>(keys_s, head, uid, nk, d_col_out, counts);
        ING_CK(cudaGetLastError());
        ING_CK(cudaMemcpyAsync(col_idx, d_col_out, U * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    }
    fmm_status s = counts_to_row_ptr(S, counts, n, row_ptr, st);
    if (s != FMM_OK) return s;
    ING_CK(cudaStreamSynchronize(st));
    *nnz_out = U;
    return FMM_OK;
}

struct StreamGuard {
    cudaStream_t s = nullptr;
    ~StreamGuard() {
        if (s) cudaStreamDestroy(s);
    }
};

}  // namespace

extern "C" {

fmm_status fmm_csr_from_coo(int device, int64_t m, int64_t n, int64_t count, const int64_t* rows,
                            const int64_t* cols, const float* vals, int64_t* row_ptr, int64_t* col_idx,
                            float* values, int64_t* nnz_out) {
    if (m < 0 || n < 0 || count < 0 || !row_ptr || !nnz_out) return FMM_E_INVAL;
    if (count > 0 && (!rows || !cols || !col_idx)) return FMM_E_INVAL;
    if (m >= (int64_t(1) << 32) || n > INT32_MAX || count > UINT32_MAX) return FMM_E_UNSUPPORTED;
    *nnz_out = 0;
    if (cudaSetDevice(device) != cudaSuccess) return status_of(cudaErrorInvalidDevice);
    StreamGuard g;
    ING_CK(cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking));
    Scratch S;
    int64_t *d_rows, *d_cols;
    float* d_vals = nullptr;
    ING_CK(S.alloc(&d_rows, count));
    ING_CK(S.alloc(&d_cols, count));
    if (count > 0) {
        ING_CK(cudaMemcpyAsync(d_rows, rows, count * sizeof(int64_t), cudaMemcpyHostToDevice, g.s));
        ING_CK(cudaMemcpyAsync(d_cols, cols, count * sizeof(int64_t), cudaMemcpyHostToDevice, g.s));
        if (vals) {
            ING_CK(S.alloc(&d_vals, count));
            ING_CK(cudaMemcpyAsync(d_vals, vals, count * sizeof(float), cudaMemcpyHostToDevice, g.s));
        }
    }
    return csr_from_coo_dev(g.s, S, m, n, count, d_rows, d_cols, d_vals, row_ptr, col_idx, values, nnz_out);
}

fmm_status fmm_csr_sym_unique(int device, int64_t n, int64_t count, const int64_t* rows, const int64_t* cols,
                              int drop_self, int symmetrize, int64_t* row_ptr, int64_t* col_idx,
                              int64_t* nnz_out) {
    if (n < 0 || count < 0 || !row_ptr || !nnz_out) return FMM_E_INVAL;
    if (count > 0 && (!rows || !cols || !col_idx)) return FMM_E_INVAL;
    if (n > INT32_MAX || 2 * count > static_cast<int64_t>(UINT32_MAX)) return FMM_E_UNSUPPORTED;
    *nnz_out = 0;
    if (cudaSetDevice(device) != cudaSuccess) return status_of(cudaErrorInvalidDevice);
    StreamGuard g;
    ING_CK(cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking));
    Scratch S;
    int64_t *d_rows, *d_cols;
    ING_CK(S.alloc(&d_rows, count));
    ING_CK(S.alloc(&d_cols, count));
    if (count > 0) {
        ING_CK(cudaMemcpyAsync(d_rows, rows, count * sizeof(int64_t), cudaMemcpyHostToDevice, g.s));
        ING_CK(cudaMemcpyAsync(d_cols, cols, count * sizeof(int64_t), cudaMemcpyHostToDevice, g.s));
    }
    return sym_unique_dev(g.s, S, n, count, d_rows, d_cols, drop_self, symmetrize, row_ptr, col_idx, nnz_out);
}

fmm_status fmm_rmat_device(int device, int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                           int recipe, int64_t* row_ptr, int64_t* col_idx, float* values, int64_t* rows_out,
                           int64_t* cols_out, int64_t* nnz_out) {
    if (scale < 1 || scale > 30 || edge_factor < 0 || !nnz_out || recipe < 0 || recipe > 2) return FMM_E_INVAL;
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0 + 1e-12)) return FMM_E_INVAL;
    const int64_t nverts = int64_t(1) << scale;
    const int64_t nedges = static_cast<int64_t>(edge_factor) * nverts;
    if (recipe != 2 && (!row_ptr || (nedges > 0 && !col_idx))) return FMM_E_INVAL;
    if (recipe == 2 && (!rows_out || !cols_out)) return FMM_E_INVAL;
    if (nedges > static_cast<int64_t>(UINT32_MAX) / 2) return FMM_E_UNSUPPORTED;
    *nnz_out = 0;
    if (cudaSetDevice(device) != cudaSuccess) return status_of(cudaErrorInvalidDevice);
    StreamGuard g;
    ING_CK(cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking));
    Scratch S;
    int64_t *d_rows, *d_cols;
    ING_CK(S.alloc(&d_rows, nedges));
    ING_CK(S.alloc(&d_cols, nedges));
    const fmm_status gs = rmat_stream_dev(g.s, S, scale, nedges, a, b, c, seed, d_rows, d_cols);
    if (gs != FMM_OK) return gs;
    if (recipe == 2) {  // the raw insertion stream
        ING_CK(cudaMemcpyAsync(rows_out, d_rows, nedges * sizeof(int64_t), cudaMemcpyDeviceToHost, g.s));
        ING_CK(cudaMemcpyAsync(cols_out, d_cols, nedges * sizeof(int64_t), cudaMemcpyDeviceToHost, g.s));
        ING_CK(cudaStreamSynchronize(g.s));
        *nnz_out = nedges;
        return FMM_OK;
    }
    if (recipe == 0)  // rmat_generate: csr_from_coo of the stream, unit values summed
        return csr_from_coo_dev(g.s, S, nverts, nverts, nedges, d_rows, d_cols, nullptr, row_ptr, col_idx, values,
                                nnz_out);
    return sym_unique_dev(g.s, S, nverts, nedges, d_rows, d_cols, 1, 1, row_ptr, col_idx, nnz_out);
}

}  // extern "C"
