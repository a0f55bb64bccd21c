// probe_gather4.cu — random-row gather throughput: per-lane 128-bit LDG versus
// the sm_100a TMA row gather (cp.async.bulk.tensor.2d...tile::gather4: four
// rows of a 2-D tensor map into shared memory per instruction, completion on
// an mbarrier). Decides whether a TMA-gather pipeline (no registers held per
// in-flight row) beats the register-bound LDG row kernel on latency-bound
// gathers (config 3: 128-byte rows, ~70% L2 hits).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_gather4 probe_gather4.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));    \
            exit(1);                                                                               \
        }                                                                                          \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int col, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

// LDG baseline: LPG lanes x 16 B per row, U rows in flight per group.
template <int LPG, int U>
__global__ void __launch_bounds__(256) ldg_kernel(const float4* __restrict__ Y, const int* __restrict__ idx,
                                                  int64_t n_idx, float* out) {
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPG;
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPG;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPG;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t e = gid; e < n_idx; e += ng * U) {
        int v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = e + u * ng < n_idx ? __ldg(idx + e + u * ng) : 0;
        float4 val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = __ldg(Y + (int64_t)v[u] * LPG + gl);
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += val[u].x; acc.y += val[u].y; acc.z += val[u].z; acc.w += val[u].w; }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
}

// 256-bit per-lane loads (sm_100a LDG.E.ENL2.256): LPG lanes x 32 B per row.
struct F8 { float v[8]; };
__device__ __forceinline__ F8 ld256(const float* p) {
    F8 r;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
    return r;
}
template <int LPG, int U>
__global__ void __launch_bounds__(256) ldg256_kernel(const float* __restrict__ Y, const int* __restrict__ idx,
                                                     int64_t n_idx, float* out) {
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPG;
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPG;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPG;
    float acc = 0.f;
    for (int64_t e = gid; e < n_idx; e += ng * U) {
        int v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = e + u * ng < n_idx ? __ldg(idx + e + u * ng) : 0;
        F8 val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = ld256(Y + ((int64_t)v[u] * LPG + gl) * 8);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc += val[u].v[c];
    }
    if (acc == 12345.f) out[0] = acc;
}

// TMA gather4: each warp streams its contiguous slice of idx through S
// stages of K gather4 (4K rows of ROWB bytes) in shared memory; lane 0
// issues, every lane consumes (sums) the landed rows.
template <int ROWB, int S, int K>
__global__ void __launch_bounds__(256) g4_kernel(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx,
                                                 int64_t n_idx, float* out) {
    constexpr int STAGE = 4 * K * ROWB;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    unsigned char* buf = smem + (size_t)warp * S * STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwarps * S * STAGE) + warp * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
    const int64_t nw = (int64_t)gridDim.x * nwarps;
    const int64_t per = (n_idx / (4 * K) + nw - 1) / nw;  // batches per warp
    const int64_t b0 = gw * per;
    const int64_t b1 = min(b0 + per, n_idx / (4 * K));
    auto issue = [&](int64_t b, int s) {
        if (lane == 0) {
            mbar_expect_tx(&bars[s], STAGE);
            const int* ip = idx + b * 4 * K;
#pragma unroll
            for (int k = 0; k < K; ++k)
                tma_gather4(buf + s * STAGE + k * 4 * ROWB, &map, &bars[s], 0, ip[4 * k], ip[4 * k + 1], ip[4 * k + 2],
                            ip[4 * k + 3]);
        }
    };
    for (int s = 0; s < S && b0 + s < b1; ++s) issue(b0 + s, s);
    float acc = 0.f;
    uint32_t phase = 0;
    int s = 0;
    for (int64_t b = b0; b < b1; ++b) {
        mbar_wait(&bars[s], phase);
        const float4* p = reinterpret_cast<const float4*>(buf + s * STAGE);
#pragma unroll
        for (int i = lane; i < STAGE / 16; i += 32) {
            const float4 v = p[i];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (b + S < b1) issue(b + S, s);
        if (++s == S) { s = 0; phase ^= 1; }
    }
    if (acc == 12345.f) out[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) { fprintf(stderr, "no cuTensorMapEncodeTiled\n"); exit(1); }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static float time_ms(void (*launch)(void*), void* arg) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        CK(cudaEventRecord(a));
        launch(arg);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    return best;
}

struct Args {
    const float* Y;
    const int* idx;
    int64_t n;
    float* out;
    CUtensorMap map;
    int grid, threads;
    size_t smem;
};

template <int LPG, int U>
static void launch_ldg(void* a_) {
    Args* a = static_cast<Args*>(a_);
    ldg_kernel<LPG, U><<<a->grid, 256>>>(reinterpret_cast<const float4*>(a->Y), a->idx, a->n, a->out);
}
template <int LPG, int U>
static void launch_ldg256(void* a_) {
    Args* a = static_cast<Args*>(a_);
    ldg256_kernel<LPG, U><<<a->grid, 256>>>(a->Y, a->idx, a->n, a->out);
}
template <int ROWB, int S, int K>
static void launch_g4(void* a_) {
    Args* a = static_cast<Args*>(a_);
    g4_kernel<ROWB, S, K><<<a->grid, a->threads, a->smem>>>(a->map, a->idx, a->n, a->out);
}

template <int ROWB, int S, int K>
static void run_g4(Args& a, int nsm, int warps_per_cta, const char* tag) {
    a.threads = 32 * warps_per_cta;
    a.smem = (size_t)warps_per_cta * S * 4 * K * ROWB + warps_per_cta * S * 8;
    CK(cudaFuncSetAttribute(g4_kernel<ROWB, S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, g4_kernel<ROWB, S, K>, a.threads, a.smem));
    a.grid = nsm * bps;
    const float ms = time_ms(launch_g4<ROWB, S, K>, &a);
    printf("%-6s g4   row=%dB S=%d K=%d warps/cta=%d ctas/sm=%d (warps/sm %2d, %3zu KB smem/sm): %.3f ms %.2f TB/s\n", tag,
           ROWB, S, K, warps_per_cta, bps, bps * warps_per_cta, bps * a.smem / 1024, ms,
           (double)a.n * ROWB / (ms * 1e-3) / 1e12);
}

// File mode: gather 512-byte rows in the order of an int32 index file (e.g.
// the config 2 CSR column stream written by tools/gather_pattern.py).
static int file_mode(const char* path, int64_t rows, int rowb, int nsm) {
    FILE* f = fopen(path, "rb");
    if (!f) { perror(path); return 1; }
    fseek(f, 0, SEEK_END);
    const int64_t n = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int> h(n);
    if (fread(h.data(), 4, n, f) != (size_t)n) { fprintf(stderr, "short read\n"); return 1; }
    fclose(f);
    Args a{};
    float *Y, *out;
    int* idx;
    CK(cudaMalloc(&Y, rows * rowb));
    CK(cudaMemset(Y, 0, rows * rowb));
    CK(cudaMalloc(&idx, n * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
    a.Y = Y; a.idx = idx; a.n = n; a.out = out;
    for (int ctas : {2, 4, 8}) {
        a.grid = nsm * ctas;
        float ms1, ms2;
        if (rowb == 512) {
            ms1 = time_ms(launch_ldg<32, 4>, &a);
            ms2 = time_ms(launch_ldg256<16, 4>, &a);
        } else if (rowb == 128) {
            ms1 = time_ms(launch_ldg<8, 4>, &a);
            ms2 = time_ms(launch_ldg256<4, 4>, &a);
        } else {
            fprintf(stderr, "row bytes must be 128 or 512\n");
            return 1;
        }
        printf("%s row=%dB ldg128 warps/sm %2d: %.3f ms %.2f TB/s\n", path, rowb, ctas * 8, ms1,
               (double)n * rowb / (ms1 * 1e-3) / 1e12);
        printf("%s row=%dB ldg256 warps/sm %2d: %.3f ms %.2f TB/s\n", path, rowb, ctas * 8, ms2,
               (double)n * rowb / (ms2 * 1e-3) / 1e12);
    }
    return 0;
}

int main(int argc, char** argv) {
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    if (argc > 2) return file_mode(argv[1], atoll(argv[2]), argc > 3 ? atoi(argv[3]) : 512, nsm);
    const int64_t n_idx = 32 << 20;
    const int64_t y_bytes = 1ll << 30;
    float* Y;
    int *idx_hot, *idx_cold;
    float* out;
    CK(cudaMalloc(&Y, y_bytes));
    CK(cudaMemset(Y, 0, y_bytes));
    CK(cudaMalloc(&idx_hot, n_idx * 4));
    CK(cudaMalloc(&idx_cold, n_idx * 4));
    CK(cudaMalloc(&out, 4));
    std::vector<int> h(n_idx);
    uint64_t st = 88172645463325252ull;
    auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
    auto encode = encode_fn();

    constexpr int ROWB = 128;
    const int64_t rows = y_bytes / ROWB;
    const int64_t hot_rows = (32ll << 20) / ROWB;
    for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % hot_rows);
    CK(cudaMemcpy(idx_hot, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % rows);
    CK(cudaMemcpy(idx_cold, h.data(), n_idx * 4, cudaMemcpyHostToDevice));

    Args a{};
    a.Y = Y;
    a.out = out;
    a.n = n_idx;
    {
        cuuint64_t gdim[2] = {ROWB / 4, (cuuint64_t)rows};
        cuuint64_t gstride[1] = {ROWB};
        cuuint32_t box[2] = {ROWB / 4, 1};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, gdim, gstride, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); return 1; }
    }
    for (int pass = 0; pass < 2; ++pass) {
        a.idx = pass == 0 ? idx_cold : idx_hot;
        const char* tag = pass == 0 ? "DRAM" : "L2";
        for (int ctas : {4, 8}) {
            a.grid = nsm * ctas;
            const float ms = time_ms(launch_ldg<8, 4>, &a);
            printf("%-6s ldg  row=%dB LPG=8 U=4 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ROWB, ctas * 8, ms,
                   (double)n_idx * ROWB / (ms * 1e-3) / 1e12);
        }
        for (int ctas : {4, 8}) {
            a.grid = nsm * ctas;
            float ms = time_ms(launch_ldg256<4, 4>, &a);
            printf("%-6s ldg256 row=%dB LPG=4 U=4 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ROWB, ctas * 8, ms,
                   (double)n_idx * ROWB / (ms * 1e-3) / 1e12);
            ms = time_ms(launch_ldg256<4, 8>, &a);
            printf("%-6s ldg256 row=%dB LPG=4 U=8 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ROWB, ctas * 8, ms,
                   (double)n_idx * ROWB / (ms * 1e-3) / 1e12);
            ms = time_ms(launch_ldg<8, 8>, &a);
            printf("%-6s ldg  row=%dB LPG=8 U=8 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ROWB, ctas * 8, ms,
                   (double)n_idx * ROWB / (ms * 1e-3) / 1e12);
        }
        run_g4<ROWB, 4, 2>(a, nsm, 4, tag);
        run_g4<ROWB, 4, 4>(a, nsm, 4, tag);
        run_g4<ROWB, 8, 4>(a, nsm, 4, tag);
        run_g4<ROWB, 4, 8>(a, nsm, 4, tag);
        run_g4<ROWB, 8, 8>(a, nsm, 2, tag);
        run_g4<ROWB, 2, 8>(a, nsm, 8, tag);
        run_g4<ROWB, 4, 4>(a, nsm, 8, tag);
    }
    // 512-byte rows (config 2): 128-bit vs 256-bit loads, L2-resident and DRAM-random
    {
        const int64_t rows512 = y_bytes / 512, hot512 = (32ll << 20) / 512;
        for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % hot512);
        CK(cudaMemcpy(idx_hot, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
        for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % rows512);
        CK(cudaMemcpy(idx_cold, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
        a.n = n_idx / 4;
        for (int pass = 0; pass < 2; ++pass) {
            a.idx = pass == 0 ? idx_cold : idx_hot;
            const char* tag = pass == 0 ? "DRAM" : "L2";
            for (int ctas : {2, 4, 8}) {
                a.grid = nsm * ctas;
                float ms = time_ms(launch_ldg<32, 4>, &a);
                printf("%-6s ldg  row=512B LPG=32 U=4 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ctas * 8, ms,
                       (double)a.n * 512 / (ms * 1e-3) / 1e12);
                ms = time_ms(launch_ldg256<16, 4>, &a);
                printf("%-6s ldg256 row=512B LPG=16 U=4 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ctas * 8, ms,
                       (double)a.n * 512 / (ms * 1e-3) / 1e12);
                ms = time_ms(launch_ldg256<16, 2>, &a);
                printf("%-6s ldg256 row=512B LPG=16 U=2 warps/sm %d: %.3f ms %.2f TB/s\n", tag, ctas * 8, ms,
                       (double)a.n * 512 / (ms * 1e-3) / 1e12);
            }
        }
    }
    printf("done\n");
    return 0;
}
