// Compile check: include/fusedmm_cuda.hpp used from reference host code with
// the reference's OWN types (proj/include/fusedmm), as INTEGRATION.md tells
// a maintainer to do — switching namespace fusedmm:: -> fusedmm::cuda:: for
// fused_mm (kernel.hpp:297-353), update_u (kernel.hpp:81-84),
// fused_mm_specialized (kernel.hpp:356-378) and tune_lane_width
// (kernel.hpp:382-402). Built by tests/test_abi.py (-fsyntax-only: no GPU,
// no link); the same calls run on the GPU through wrapper_demo.cpp.
#include <vector>

#include "fusedmm/kernel.hpp"
#include "fusedmm/ops.hpp"
#include "fusedmm_cuda.hpp"

int dropin(const fusedmm::CsrMatrix<float>& A, const fusedmm::DenseMatrix<float>& X) {
    fusedmm::OpSpec<float> spec;  // reference defaults: MUL, RSUM, NOOP, MUL, ASUM
    spec.sop = fusedmm::Sop::SIGMOID;
    fusedmm::KernelStats stats;
    fusedmm::KernelOptions opts;
    fusedmm::DenseMatrix<float> Z = fusedmm::cuda::fused_mm(A, X, X, spec, 2, &stats, opts);
    fusedmm::DenseMatrix<float> Zs =
        fusedmm::cuda::fused_mm_specialized(fusedmm::KnownPattern::FR_LAYOUT, A, X, X, 0.5f, 1, opts);
    fusedmm::DenseMatrix<float> Zt = fusedmm::cuda::fused_mm(A, X, X, fusedmm::cuda::tdist_ops(), 1, &stats);
    std::vector<float> scratch(2 * X.dim), z(X.dim);
    fusedmm::cuda::update_u(A.row_cols(0), A.row_vals(0), X.row(0), X, spec, std::span<float>(z),
                            std::span<float>(scratch));
    const int w = fusedmm::cuda::tune_lane_width(A, X, X, spec, 1);
    return static_cast<int>(Z.nrows + Zs.nrows + Zt.nrows) + w + static_cast<int>(stats.pattern);
}
