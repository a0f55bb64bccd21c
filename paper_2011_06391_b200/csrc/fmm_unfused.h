// fmm_unfused.h — launch interface of the unfused SDDMM -> SpMM baseline
// (fmm_unfused.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fmm {

struct SddmmParams {
    const int64_t* row_ptr;
    const int32_t* col;
    const float* val;
    const float* X;
    const float* Y;
    float* H;               // nnz (scalar) or nnz*d (vector) messages
    const int32_t* order;   // rows (shard-local)
    int64_t n_rows;
    int64_t nnz;
    int64_t row0;
    int d;
    float alpha, k;
};

bool launch_sddmm(const SddmmParams& p, int vop, int rop, int sop, int mop, int aop, cudaStream_t s);
void launch_iota(int32_t* out, int64_t n, cudaStream_t s);

}  // namespace fmm
