// probe_fabric.cu — microbenchmark for the delivery ceilings that bound the
// FusedMM gathers: random row gathers served from L2 (hot set < L2), from
// distributed shared memory of a thread-block cluster (DSMEM), and a mix.
// Decides whether a cluster-wide hub-row cache can add bandwidth beyond the
// L2->SM fabric (profiles/README.md: every gather-bound config sits at
// ~11 TB/s of L2->SM delivery).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_fabric probe_fabric.cu
//   ./probe_fabric
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

// MODE 0: all gathers from global (ld.global.nc, Y + idx*ROW)
// MODE 1: all gathers from the cluster's smem (rank idx % csize, slot (idx / csize) % H), ld.shared::cluster
// MODE 2: idx < split -> cluster smem, else global
// MODE 3: all gathers from the CTA's own smem (slot idx % H), ld.shared
// MODE 4: idx < split -> own smem, else global
// H is a power of two, csize a power of two.
__device__ __forceinline__ float4 ld_nc4(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ float4 ld_smem4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

template <int LPG, int U, int MODE>
__global__ void __launch_bounds__(512, 1) gather_kernel(const float4* __restrict__ Y, const int* __restrict__ idx,
                                                        int64_t n_idx, int logH, int split, float* out) {
    extern __shared__ float4 cache[];  // H rows of LPG float4
    constexpr int ROW = LPG;           // float4 per row
    cg::cluster_group cluster = cg::this_cluster();
    const int csize = cluster.num_blocks();
    const int logc = 31 - __clz(csize);
    const int crank = cluster.block_rank();
    const int H = 1 << logH;
    if (MODE != 0) {
        for (int i = threadIdx.x; i < H * ROW; i += blockDim.x) {
            const int s = i / ROW, c = i % ROW;
            cache[i] = Y[(int64_t)(s * csize + crank) * ROW + c];
        }
    }
    cluster.sync();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(cache);
    uint32_t rbase[16];
    if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int r = 0; r < 16; ++r) rbase[r] = r < csize ? mapa(sbase, r) : 0;
    }
    const int lane = threadIdx.x & 31;
    const int gl = lane % LPG;
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPG;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / LPG;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t e = gid; e < n_idx; e += ng * U) {
        int v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t ee = e + u * ng;
            v[u] = ee < n_idx ? __ldg(idx + ee) : 0;
        }
        float4 val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (MODE == 0 || ((MODE == 2 || MODE == 4) && v[u] >= split)) {
                val[u] = ld_nc4(Y + (int64_t)v[u] * ROW + gl);
            } else if (MODE == 3 || MODE == 4) {
                val[u] = ld_smem4(sbase + (((v[u] & (H - 1)) * ROW + gl) << 4));
            } else {
                const int r = v[u] & (csize - 1);
                const int s = (v[u] >> logc) & (H - 1);
                uint32_t b = rbase[0];
#pragma unroll
                for (int q = 1; q < 16; ++q) b = (r == q) ? rbase[q] : b;
                val[u] = ld_dsmem4(b + ((s * ROW + gl) << 4));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc.x += val[u].x; acc.y += val[u].y; acc.z += val[u].z; acc.w += val[u].w;
        }
    }
    cluster.sync();  // remote smem must stay alive until every reader is done
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
}

template <int LPG, int U, int MODE>
double run(const float4* Y, const int* idx, int64_t n_idx, int H, int split, int csize, int ctas_per_sm,
           int nthreads, float* out, int nsm) {
    const int mode = MODE;
    auto k = gather_kernel<LPG, U, MODE>;
    const int logH = 31 - __builtin_clz(H);
    const size_t smem = (mode == 0) ? 0 : (size_t)H * LPG * 16;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (csize > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    int grid = nsm * ctas_per_sm;
    grid = (grid / csize) * csize;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(nthreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg) != cudaSuccess) nclusters = -1;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        CK(cudaEventRecord(a));
        CK(cudaLaunchKernelEx(&cfg, k, Y, idx, n_idx, logH, split, out));
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    const double bytes = (double)n_idx * LPG * 16;
    const double tbs = bytes / (best * 1e-3) / 1e12;
    printf("row=%4dB U=%d mode=%d csize=%2d grid=%4d thr=%d H=%5d smem=%6zu activeClusters=%3d : %.3f ms  %.2f TB/s\n",
           LPG * 16, U, mode, csize, grid, nthreads, H, smem, nclusters, best, tbs);
    return tbs;
}

int main() {
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int64_t n_idx = 32 << 20;  // 32M gathers
    const int64_t y_bytes = 1ll << 30;
    float4* Y;
    int* idx_hot;
    int* idx_cold;
    float* out;
    CK(cudaMalloc(&Y, y_bytes));
    CK(cudaMemset(Y, 0, y_bytes));
    CK(cudaMalloc(&idx_hot, n_idx * 4));
    CK(cudaMalloc(&idx_cold, n_idx * 4));
    CK(cudaMalloc(&out, 4));
    std::vector<int> h(n_idx);
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };

    for (int rowb : {128, 512}) {
        const int64_t hot_rows = (32ll << 20) / rowb;  // 32 MB hot set: L2-resident
        const int64_t all_rows = y_bytes / rowb;
        for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % hot_rows);
        CK(cudaMemcpy(idx_hot, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
        for (int64_t i = 0; i < n_idx; ++i) h[i] = (int)(rnd() % all_rows);
        CK(cudaMemcpy(idx_cold, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
        const int H = (rowb == 128) ? 1024 : 256;  // 128 KB of rows per CTA
        printf("--- row %d B\n", rowb);
        if (rowb == 128) {
            run<8, 4, 0>(Y, idx_cold, n_idx, H, 0, 1, 2, 512, out, nsm);   // DRAM random
            run<8, 4, 0>(Y, idx_hot, n_idx, H, 0, 1, 2, 512, out, nsm);    // L2 random
            run<8, 8, 0>(Y, idx_hot, n_idx, H, 0, 1, 2, 512, out, nsm);
            run<8, 4, 0>(Y, idx_hot, n_idx, H, 0, 1, 4, 256, out, nsm);
            run<8, 4, 3>(Y, idx_hot, n_idx, H, 0, 1, 1, 512, out, nsm);    // own smem
            for (int f : {10, 25, 50}) run<8, 4, 4>(Y, idx_hot, n_idx, H, (int)(hot_rows * f / 100), 1, 1, 512, out, nsm);
            for (int f : {10, 25, 50}) run<8, 4, 4>(Y, idx_cold, n_idx, H, (int)((1ll << 30) / 128 * f / 100), 1, 1, 512, out, nsm);
            for (int cs : {1, 2, 4, 8, 16}) run<8, 4, 1>(Y, idx_hot, n_idx, H, 0, cs, 1, 512, out, nsm);
            run<8, 8, 1>(Y, idx_hot, n_idx, H, 0, 8, 1, 512, out, nsm);
            for (int f : {25, 50}) {
                const int split = (int)(hot_rows * f / 100);
                run<8, 4, 2>(Y, idx_hot, n_idx, H, split, 8, 1, 512, out, nsm);
                run<8, 8, 2>(Y, idx_hot, n_idx, H, split, 8, 1, 512, out, nsm);
                run<8, 4, 2>(Y, idx_hot, n_idx, H, split, 4, 1, 512, out, nsm);
            }
        } else {
            run<32, 4, 0>(Y, idx_cold, n_idx, H, 0, 1, 2, 512, out, nsm);
            run<32, 4, 0>(Y, idx_hot, n_idx, H, 0, 1, 2, 512, out, nsm);
            run<32, 4, 3>(Y, idx_hot, n_idx, H, 0, 1, 1, 512, out, nsm);
            for (int f : {10, 25, 50}) run<32, 4, 4>(Y, idx_hot, n_idx, H, (int)(hot_rows * f / 100), 1, 1, 512, out, nsm);
            for (int cs : {1, 2, 4, 8, 16}) run<32, 4, 1>(Y, idx_hot, n_idx, H, 0, cs, 1, 512, out, nsm);
            for (int f : {25, 50}) {
                const int split = (int)(hot_rows * f / 100);
                run<32, 4, 2>(Y, idx_hot, n_idx, H, split, 8, 1, 512, out, nsm);
                run<32, 4, 2>(Y, idx_hot, n_idx, H, split, 16, 1, 512, out, nsm);
            }
        }
    }
    printf("done\n");
    return 0;
}
