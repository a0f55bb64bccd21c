/*
 * fusedmm_cuda.h — C ABI of libfusedmm_cuda, the sm_100a (B200) FusedMM path.
 *
 * Drop-in boundary for the reference's header-only kernel
 *   template<class T> DenseMatrix<T> fusedmm::fused_mm(A, X, Y, spec, t, stats, opts)
 *   (/root/reference/proj/include/fusedmm/kernel.hpp:297-353)
 * and its five-slot operator interface OpSpec<T>{vop,rop,sop,mop,aop,alpha,...}
 *   (/root/reference/proj/include/fusedmm/ops.hpp:12-51).
 *
 * Everything here is plain C: pointers, sizes, status codes. No torch / C++
 * types cross this boundary. The C++ wrapper with the reference's exact
 * signature and exception types is include/fusedmm_cuda.hpp; the Python mirror
 * is paper_2011_06391_b200/fusedmm.py. Bindings a maintainer would add are in
 * INTEGRATION.md.
 *
 * Semantics: Z[u,:] = AOP-fold over v in N(u), in CSR storage order, of
 *   VOP(x_u, y_v) -> [ROP -> SOP(s, a_uv) -> MOP(h, y_v)]   (scalar message)
 *                 -> [SOP elementwise -> MOP(t, y_v, a_uv)]  (vector message)
 * exactly as fusedmm::update_u (kernel.hpp:81-107). There is no CPU fallback:
 * a slot this library cannot run on the device returns FMM_E_UNSUPPORTED.
 */
#ifndef FUSEDMM_CUDA_H
#define FUSEDMM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMM_ABI_VERSION 2

/* Status codes. FMM_E_INVAL maps to std::invalid_argument and FMM_E_LOGIC to
 * std::logic_error in the C++ wrapper (kernel.hpp:272-281,303; ops.hpp:102-103). */
typedef enum fmm_status {
    FMM_OK = 0,
    FMM_E_INVAL = 1,       /* bad argument / dimension mismatch / bad CSR   */
    FMM_E_UNSUPPORTED = 2, /* USER slot or shape with no device kernel      */
    FMM_E_CUDA = 3,        /* CUDA runtime error (message in last_error)    */
    FMM_E_NCCL = 4,        /* reserved for the collective layer             */
    FMM_E_OOM = 5,         /* device or pinned-host allocation failed       */
    FMM_E_LOGIC = 6        /* contract violation inside the call            */
} fmm_status;

/* Slot codes keep the reference enum order (ops.hpp:14-18). Device-only
 * extensions sit above the USER values; they express the "scale the VOP
 * output" step (the paper's VSC) that the reference can only reach through a
 * USER VOP lambda (SURVEY.md §8(a) "Oracle op definitions"). */
enum {
    FMM_VOP_ADD = 0, FMM_VOP_MUL = 1, FMM_VOP_SEL2ND = 2, FMM_VOP_SUB = 3,
    FMM_VOP_USER = 4,
    FMM_VOP_MLP = 16 /* t_j = sigmoid(mlp_wx*x_j + mlp_wy*y_j + mlp_b): the
                        reference's toy single-layer MLP hook for GNN_MLP
                        (apps.hpp:58-64) as a device op                    */
};
enum {
    FMM_ROP_NOOP = 0, FMM_ROP_RSUM = 1, FMM_ROP_RMUL = 2, FMM_ROP_NORM = 3,
    FMM_ROP_USER = 4,
    FMM_ROP_SQNORM = 16 /* s = sum_j t_j*t_j (no sqrt)                     */
};
enum {
    FMM_SOP_NOOP = 0, FMM_SOP_SIGMOID = 1, FMM_SOP_SCAL = 2, FMM_SOP_USER = 3,
    FMM_SOP_TDIST = 16, /* h = 1/(1+s)         (t-distribution kernel)      */
    FMM_SOP_SQK = 17    /* h = s/k             (FR attractive, k = spec.k)  */
};
enum {
    FMM_MOP_MUL = 0, FMM_MOP_SEL2ND = 1, FMM_MOP_USER = 2,
    FMM_MOP_MUL_VOP = 16 /* w_j = a_uv*(h*t_j): scale the VOP output t     */
};
enum { FMM_AOP_ASUM = 0, FMM_AOP_AMAX = 1, FMM_AOP_USER = 2 };

/* KnownPattern (ops.hpp:20) plus the two device-only patterns. */
enum {
    FMM_PATTERN_SIGMOID_EMBED = 0,
    FMM_PATTERN_SPMM_GCN = 1,
    FMM_PATTERN_FR_LAYOUT = 2,
    FMM_PATTERN_GENERIC = 3,
    FMM_PATTERN_TDIST = 16,      /* SUB,SQNORM,TDIST,MUL_VOP,ASUM (config 3) */
    FMM_PATTERN_FR_ATTRACT = 17  /* SUB,SQNORM,SQK,MUL_VOP,ASUM   (config 4) */
};

/* POD mirror of OpSpec<float> without the std::function hooks. */
typedef struct fmm_opspec {
    int32_t vop, rop, sop, mop, aop;
    float alpha; /* SCAL factor (ops.hpp:49)                  */
    float k;     /* SQK divisor; ignored by the other ops      */
    float mlp_wx, mlp_wy, mlp_b; /* FMM_VOP_MLP weights and bias   */
} fmm_opspec;

/* fmm_run / fmm_iterate flags. */
enum {
    FMM_HOST_PTRS = 0,         /* X, Y, Z are host pointers (default)       */
    FMM_DEVICE_PTRS = 1u << 0, /* X, Y, Z are device pointers on shard 0's
                                  device; single-shard contexts only        */
    FMM_ASYNC = 1u << 1,       /* do not synchronize. Device pointers: the
                                  kernels are enqueued on the shard stream.
                                  Host pointers: upload / kernels / download
                                  are pipelined on three streams over two
                                  device buffer slots (call k's download
                                  overlaps call k+1's upload); host buffers
                                  must stay valid (pinned for overlap) until
                                  fmm_sync                                  */
    FMM_EXACT = 1u << 2,       /* force bit-exact scheme    */
    FMM_FAST = 1u << 3,        /* force reassociating scheme (FMA, splits)  */
    FMM_EXCHANGE_COPIES = 1u << 4, /* fmm_iterate: exchange Z slices with
                                  peer copies after the kernels instead of
                                  the fused P2P-store epilogue (default)    */
    FMM_PEERS_ALL = 1u << 5    /* fmm_run_peers / fmm_iterate: store every
                                  row to every peer, ignoring the halo mask
                                  (e.g. the last iteration, when the caller
                                  wants the iterate fully replicated)       */
};

/* Mirrors KernelStats (kernel.hpp:51-55) plus device-side evidence. */
typedef struct fmm_stats {
    uint64_t aux_bytes;   /* device scratch held for the call (partials)    */
    int32_t threads;      /* number of shards (GPUs) that ran                */
    int32_t pattern;      /* FMM_PATTERN_*                                   */
    int32_t exact;        /* 1 if the bit-exact scheme ran                   */
    int32_t launches;     /* kernels launched by this call                   */
    float kernel_ms;      /* device time of the fused kernels (shard max),
                             measured with events on the launch stream; 0
                             under FMM_ASYNC                                 */
    float total_ms;       /* device time including host<->device copies     */
} fmm_stats;

/* Graph summary after upload (for tests and the bench's byte model). */
typedef struct fmm_graph_info {
    int64_t m, n, nnz;
    int64_t row_begin, row_end; /* rows this graph object covers          */
    int64_t nonempty_rows;
    int64_t max_degree;
    int64_t split_rows;         /* rows cut into chunks on the fast path  */
    int64_t split_chunks;
    int32_t shards;
    int32_t has_values;
    /* Halo exchange (iterative workloads): rows stored to peers per
     * exchange with the per-row peer masks (sum over shards of popcount),
     * and without them (every row to every peer). 0 / 0 before masks exist. */
    int64_t exchange_rows;
    int64_t exchange_rows_all;
} fmm_graph_info;

typedef struct fmm_ctx fmm_ctx;
typedef struct fmm_graph fmm_graph;

const char* fmm_version(void);
const char* fmm_status_string(fmm_status s);

/* Context: one shard per entry of devs (duplicates allowed; they become
 * independent shards on the same GPU, which is how the multi-shard exchange
 * is exercised on one device). ngpu >= 1 mirrors `t >= 1` (kernel.hpp:303). */
fmm_status fmm_create(int ngpu, const int* devs, fmm_ctx** out);
fmm_status fmm_destroy(fmm_ctx* ctx);
const char* fmm_last_error(const fmm_ctx* ctx);
int fmm_device_count(void);

/* Run shard i's kernels on an external stream (e.g. torch's current stream)
 * instead of the context's own. stream is a cudaStream_t; NULL means the
 * legacy default stream. fmm_reset_stream restores the context's own. */
fmm_status fmm_set_stream(fmm_ctx* ctx, int shard, void* stream);

/* Kernel shape variant of this context (the device analogue of the
 * reference's KernelOptions::lane_width, kernel.hpp:286-288): -1 = the
 * default shape for d, other values select tuning alternatives (lane-group
 * width, vector width, unroll, occupancy; unknown values fall back to the
 * default). fmm_get_variant returns the current one. Initialised from the
 * FMM_VARIANT environment variable. */
fmm_status fmm_set_variant(fmm_ctx* ctx, int variant);
int fmm_get_variant(const fmm_ctx* ctx);
fmm_status fmm_reset_stream(fmm_ctx* ctx, int shard);

/* Host-side helpers, no device work. */
fmm_status fmm_pattern_of(const fmm_opspec* spec, int32_t* pattern);
/* part1d (kernel.hpp:24-49): boundaries[0..t], same greedy rule. */
fmm_status fmm_part1d(int64_t m, const int64_t* row_ptr, int t,
                      int64_t* boundaries);

/* Cost-balanced row partition for GPU shards: boundary i is the smallest row
 * r with (row_ptr[r] + w*r) * t >= i * (nnz + w*m) — each row also costs w
 * edge-equivalents of per-row kernel work; w = 0 is exactly fmm_part1d. The
 * result is bitwise independent of the partition (rows are never split). */
fmm_status fmm_part1d_weighted(int64_t m, const int64_t* row_ptr, int t,
                               double row_weight, int64_t* boundaries);
/* Host only (no GPU): the split-row work list fmm_graph_upload would build
 * for rows [row_begin, row_end) of this matrix — the rows cut into pieces
 * (longer than the chunk size, or, on graphs far larger than L2, of 4096+
 * edges cut at column-band boundaries) in launch order. pieces (may be NULL)
 * receives up to cap entries of 4 values {row, first edge relative to the
 * row, edges, band of the first column}. A diagnostic / test aid: the cuts
 * depend on the row's own columns and on (n, total nnz) only, never on the
 * row range, which is what keeps results bitwise independent of the shard
 * count. */
fmm_status fmm_plan_pieces(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           int64_t row_begin, int64_t row_end, int64_t* chunk_edges,
                           int64_t* n_split_rows, int64_t* n_banded_rows, int64_t* n_pieces,
                           int64_t* pieces, int64_t cap);

/* Row weight fmm_graph_upload uses to split a multi-shard context's rows
 * (default 0: the reference's part1d). */
fmm_status fmm_set_row_weight(fmm_ctx* ctx, double row_weight);

/* Upload A (CSR, host arrays, int64 indices as in matrix.hpp:48-68).
 * Only rows [row_begin, row_end) are uploaded (pass 0, m for all rows); a
 * multi-shard context further splits that range with part1d. values may be
 * NULL (all a_uv = 1). Validates row_ptr monotone / col in [0, n). */
fmm_status fmm_graph_upload(fmm_ctx* ctx, int64_t m, int64_t n,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const float* values, int64_t row_begin,
                            int64_t row_end, fmm_graph** out);
fmm_status fmm_graph_free(fmm_graph* g);
/* Replace the edge values a_uv of an uploaded graph in place (values: the
 * full host array of the m-row CSR the graph was uploaded from, NULL = all
 * ones); the structure is kept. For callers that change A.values between
 * calls (the reference reads A afresh on every fused_mm). */
fmm_status fmm_graph_update_values(fmm_graph* g, const float* values);
/* 64-bit content fingerprint of a host buffer (multi-threaded, ~memory
 * bandwidth): the wrappers key their uploaded-graph caches on the contents
 * of row_ptr / col_idx / values, not on their addresses. */
uint64_t fmm_fingerprint(const void* data, size_t bytes);
fmm_status fmm_graph_get_info(const fmm_graph* g, fmm_graph_info* out);
/* Boundaries of the shards (length shards+1, absolute row ids). */
fmm_status fmm_graph_shard_bounds(const fmm_graph* g, int64_t* bounds);

/* One fused call. X: m x d (rows indexed by absolute row id), Y: ny x d,
 * Z: (row_end-row_begin) x d output for this graph's rows. Host pointers
 * unless FMM_DEVICE_PTRS. stats may be NULL. */
fmm_status fmm_run(fmm_ctx* ctx, const fmm_graph* g, const fmm_opspec* spec,
                   int64_t d, const float* X, int64_t ny, const float* Y,
                   float* Z, uint32_t flags, fmm_stats* stats);

/* iters fused calls with X <- Z between them (square A, Y = X), the Z slices
 * exchanged between shards on the device. X is the host m x d input and
 * receives the final iterate. */
/* The UNFUSED baseline of the same call (reference.hpp:41-155 on the
 * device): an SDDMM kernel materialises the per-edge messages H (nnz
 * scalars, or nnz*d values for vector messages) in HBM, then an SpMM pass
 * aggregates them. Device pointers, single-shard context, d in
 * {32, 64, 128, 256}; stats->aux_bytes = bytes of H. For measuring what the
 * fusion saves, not for production use. */
fmm_status fmm_run_unfused(fmm_ctx* ctx, const fmm_graph* g,
                           const fmm_opspec* spec, int64_t d, const float* X,
                           int64_t ny, const float* Y, float* Z,
                           uint32_t flags, fmm_stats* stats);

/* Wait for every call enqueued with FMM_ASYNC on this context. */
fmm_status fmm_sync(fmm_ctx* ctx);

/* Page-locked (pinned, portable) host buffers for FMM_ASYNC host calls. */
fmm_status fmm_host_alloc(void** ptr, size_t bytes);
fmm_status fmm_host_free(void* ptr);

fmm_status fmm_iterate(fmm_ctx* ctx, const fmm_graph* g,
                       const fmm_opspec* spec, int64_t d, float* X, int iters,
                       uint32_t flags, fmm_stats* stats);

/* ---- one process per GPU: the fused exchange across processes ---------
 * fmm_run with every final z row also stored into `npeer` (<= 7) peer
 * buffers: device pointers (FMM_DEVICE_PTRS, single-shard context), each at
 * the peer's copy of this shard's first row — the next-iterate buffers of
 * the other ranks, opened with fmm_ipc_open. The slice all-gather of the
 * iterative workloads then rides on the kernel's own stores (NVLink P2P);
 * the caller orders the next iteration after every rank's kernel (e.g. a
 * stream-ordered NCCL barrier). */
fmm_status fmm_run_peers(fmm_ctx* ctx, const fmm_graph* g,
                         const fmm_opspec* spec, int64_t d, const float* X,
                         int64_t ny, const float* Y, float* Z,
                         float* const* peers, int npeer, uint32_t flags,
                         fmm_stats* stats);

/* Halo masks for the one-process-per-GPU exchange. need[c] (n bytes) is
 * set to 1 for every column c some edge of g points at (0 elsewhere): the
 * rows this graph's shard READS. A rank gathers every peer's need array and
 * passes mask[r] (row_end-row_begin bytes, bit q = peer slot q reads row
 * row_begin+r; slots in the order of fmm_run_peers' peers array) to
 * fmm_graph_set_peer_mask; fmm_run_peers then stores row r only to the
 * peers whose bit is set (FMM_PEERS_ALL overrides). Results are unchanged:
 * a peer never reads a row it does not reference. fmm_iterate builds the
 * same masks for its own shards. */
fmm_status fmm_graph_column_use(const fmm_graph* g, uint8_t* need);
fmm_status fmm_graph_set_peer_mask(fmm_graph* g, const uint8_t* mask, int npeer);

#define FMM_IPC_HANDLE_BYTES 64
/* CUDA IPC: export the allocation dptr lies in (handle: FMM_IPC_HANDLE_BYTES
 * bytes; *offset = dptr - allocation base), map another process's allocation
 * on `device` (the peer adds the offset), unmap it. */
fmm_status fmm_ipc_handle(const void* dptr, void* handle, uint64_t* offset);
fmm_status fmm_ipc_open(const void* handle, int device, void** dptr);
fmm_status fmm_ipc_close(void* dptr);

/* ---- device-side graph construction ----------- */

/* csr_from_coo on GPU `device` (replaces fusedmm::csr_from_coo,
 * matrix.hpp:87-140): entries (rows[i], cols[i], vals[i]) in insertion
 * order; duplicates summed left to right into the first occurrence; per-row
 * storage order is first-occurrence order. vals NULL means every value is 1.
 * Host arrays: row_ptr[m+1]; col_idx / values (NULL to skip) with room for
 * `count` entries; *nnz_out = entries written. FMM_E_INVAL for an entry out of
 * bounds (the reference throws std::invalid_argument). Applied to the R-MAT
 * insertion stream this is rmat_generate (rmat.hpp:24-61). */
fmm_status fmm_csr_from_coo(int device, int64_t m, int64_t n, int64_t count,
                            const int64_t* rows, const int64_t* cols,
                            const float* vals, int64_t* row_ptr,
                            int64_t* col_idx, float* values, int64_t* nnz_out);

/* read_matrix_market (mmio.hpp:23-84): coordinate real|integer|pattern,
 * general|symmetric, 1-based; pattern values 1, symmetric files mirrored;
 * parsed on the host with the reference's rules, folded by fmm_csr_from_coo
 * on GPU `device`. Outputs are malloc'd (release with fmm_free). Parse errors
 * return FMM_E_INVAL with "<path>:<line>: <what>" in err (the reference's
 * MmParseError message). */
fmm_status fmm_read_matrix_market(const char* path, int device, int64_t* m,
                                  int64_t* n, int64_t* nnz, int64_t** row_ptr,
                                  int64_t** col_idx, float** values,
                                  char* err, size_t err_cap);
/* write_matrix_market (mmio.hpp:87-99): coordinate real general, 1-based,
 * 17 significant digits. */
fmm_status fmm_write_matrix_market(const char* path, int64_t m, int64_t n,
                                   const int64_t* row_ptr,
                                   const int64_t* col_idx,
                                   const float* values);
void fmm_free(void* p);

/* The BASELINE.json graph recipe on GPU `device`: an n x n edge list with
 * self-loops dropped (drop_self), both directions added (symmetrize), sorted
 * and deduplicated; unweighted (a_uv = 1). Host arrays: row_ptr[n+1], col_idx
 * with room for 2*count entries. */
fmm_status fmm_csr_sym_unique(int device, int64_t n, int64_t count,
                              const int64_t* rows, const int64_t* cols,
                              int drop_self, int symmetrize, int64_t* row_ptr,
                              int64_t* col_idx, int64_t* nnz_out);

/* rmat_generate (rmat.hpp:24-61) on GPU `device`: the seeded insertion
 * stream (scale levels of quadrant descent per edge from one mt19937_64)
 * generated on the device by independent sub-streams whose generator states
 * come from a jump-ahead (fmm_mt64_window), bitwise the reference's sequential
 * stream; then
 *   recipe 0: csr_from_coo of the stream (= rmat_generate: self-loops kept,
 *             duplicates summed into values; col_idx / values with room for
 *             edge_factor << scale entries),
 *   recipe 1: the BASELINE.json recipe (fmm_csr_sym_unique: self-loops
 *             dropped, symmetrised, sorted, unique; col_idx with room for
 *             2 * edge_factor << scale; values unused),
 *   recipe 2: the raw stream into rows_out / cols_out (edge_factor << scale).
 * row_ptr has scale-sized n + 1 entries; *nnz_out = entries written. */
fmm_status fmm_rmat_device(int device, int scale, int edge_factor, double a,
                           double b, double c, uint64_t seed, int recipe,
                           int64_t* row_ptr, int64_t* col_idx, float* values,
                           int64_t* rows_out, int64_t* cols_out,
                           int64_t* nnz_out);
/* The 312-word window (x_p .. x_{p+311}) of std::mt19937_64(seed)'s word
 * recurrence: its next outputs are temper(x_{p+312}), ... i.e. outputs
 * p, p+1, ... of the generator (host; polynomial jump-ahead). */
fmm_status fmm_mt64_window(uint64_t seed, uint64_t position, uint64_t* window);

#ifdef __cplusplus
}
#endif
#endif /* FUSEDMM_CUDA_H */
