// Exercise include/fusedmm_cuda.hpp the way reference host code would:
// the reference's own KATs (proj/tests/test_kernel.cpp:110-144) through the
// drop-in fusedmm::cuda::fused_mm. Built on any box; run on a GPU box.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "fusedmm_cuda.hpp"

using namespace fusedmm::cuda::types;
namespace fc = fusedmm::cuda;

static int failures = 0;
#define CHECK(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++failures; } } while (0)

int main() {
    // GCN tiny case: {5,5,6,6} (test_kernel.cpp:110-116)
    CsrMatrix A;
    A.nrows = 2; A.ncols = 2;
    A.row_ptr = {0, 2, 3};
    A.col_idx = {0, 1, 1};
    A.values = {1.f, 2.f, 3.f};
    DenseMatrix Y(2, 2);
    Y.data = {1, 1, 2, 2};
    DenseMatrix X(2, 2);
    OpSpec gcn{Vop::SEL2ND, Rop::NOOP, Sop::NOOP, Mop::MUL, Aop::ASUM};
    KernelStats st;
    DenseMatrix Z = fc::fused_mm(A, X, Y, gcn, 2, &st);
    CHECK(Z.data == (std::vector<float>{5, 5, 6, 6}));
    CHECK(st.threads == 2 && st.pattern == KnownPattern::SPMM_GCN);

    // sigmoid 2-cycle: 1.0 and 0.5 (test_kernel.cpp:118-125)
    CsrMatrix C;
    C.nrows = 2; C.ncols = 2;
    C.row_ptr = {0, 1, 2};
    C.col_idx = {1, 0};
    C.values = {1.f, 1.f};
    DenseMatrix X1(2, 1), Y1(2, 1);
    Y1.data = {1, 2};
    OpSpec emb{Vop::MUL, Rop::RSUM, Sop::SIGMOID, Mop::MUL, Aop::ASUM};
    DenseMatrix Z1 = fc::fused_mm(C, X1, Y1, emb, 1);
    CHECK(std::fabs(Z1.data[0] - 1.f) < 1e-6f && std::fabs(Z1.data[1] - 0.5f) < 1e-6f);

    // dimension mismatch throws std::invalid_argument (test_kernel.cpp:134-144)
    DenseMatrix Xbad(1, 2);
    bool threw = false;
    try { fc::fused_mm(A, Xbad, Y, gcn, 1); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    threw = false;
    try { fc::fused_mm(A, X, Y, gcn, 0); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // USER slot: no device kernel, no CPU fallback
    OpSpec user = emb;
    user.vop = Vop::USER;
    threw = false;
    try { fc::fused_mm(A, X, Y, user, 1); } catch (const fc::unsupported&) { threw = true; }
    CHECK(threw);
    // t-distribution through the device op descriptor: t=(-2,-2), h=1/9
    CsrMatrix E;
    E.nrows = 1; E.ncols = 1;
    E.row_ptr = {0, 1};
    E.col_idx = {0};
    DenseMatrix Xe(1, 2), Ye(1, 2);
    Xe.data = {1, 2};
    Ye.data = {3, 4};
    DenseMatrix Ze = fc::fused_mm(E, Xe, Ye, fc::tdist_ops(), 1);
    CHECK(std::fabs(Ze.data[0] + 2.f / 9.f) < 1e-6f);
    // csr_from_coo on the device: duplicates summed into the first
    // occurrence, first-occurrence order (matrix.hpp:87-140)
    struct Coo { int64_t row, col; float value; };
    std::vector<Coo> ent = {{1, 2, 1.f}, {0, 1, 2.f}, {1, 0, 3.f}, {1, 2, 4.f}, {0, 1, 0.5f}};
    CsrMatrix Cc = fc::csr_from_coo<CsrMatrix>(ent, 2, 3);
    CHECK(Cc.row_ptr == (std::vector<int64_t>{0, 1, 3}));
    CHECK(Cc.col_idx == (std::vector<int64_t>{1, 2, 0}));
    CHECK(Cc.values == (std::vector<float>{2.5f, 5.f, 3.f}));
    threw = false;
    try { fc::csr_from_coo<CsrMatrix>(std::vector<Coo>{{2, 0, 1.f}}, 2, 3); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // the reference reads A afresh every call: values edited in place, then
    // the whole CSR rewritten at the same addresses, are both seen
    A.values[0] = 10.f;  // row 0: 10*y0 + 2*y1 = {14, 14}
    DenseMatrix Zv = fc::fused_mm(A, X, Y, gcn, 1);
    CHECK(Zv.data == (std::vector<float>{14, 14, 6, 6}));
    A.col_idx[0] = 1;    // row 0: 10*y1 + 2*y1 = {24, 24}
    DenseMatrix Zc = fc::fused_mm(A, X, Y, gcn, 1);
    CHECK(Zc.data == (std::vector<float>{24, 24, 6, 6}));
    A.col_idx[0] = 0;
    A.values[0] = 1.f;
    // update_u (kernel.hpp:81-107): GCN row [5,5] (test_kernel.cpp:89-96)
    std::vector<int64_t> ucols{0, 1};
    std::vector<float> uvals{1.f, 2.f}, xu(2, 0.f), zu(2, -1.f), scratch(4);
    fc::update_u(ucols, uvals, xu, Y, gcn, zu, scratch);
    CHECK(zu == (std::vector<float>{5, 5}));
    // fused_mm_specialized (kernel.hpp:356-378) and its GENERIC rejection
    DenseMatrix Zs = fc::fused_mm_specialized(KnownPattern::SPMM_GCN, A, X, Y, 1.f, 1);
    CHECK(Zs.data == (std::vector<float>{5, 5, 6, 6}));
    threw = false;
    try { fc::fused_mm_specialized(KnownPattern::GENERIC, A, X, Y, 1.f, 1); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    // lane widths: 4 / 8 / 16 run, others throw; tune_lane_width picks one
    for (int w : {4, 8, 16}) {
        KernelOptions o{w};
        CHECK(fc::fused_mm(A, X, Y, gcn, 1, &st, o).data == (std::vector<float>{5, 5, 6, 6}));
    }
    threw = false;
    try { fc::fused_mm(A, X, Y, gcn, 1, &st, KernelOptions{3}); } catch (const std::invalid_argument&) { threw = true; }
    CHECK(threw);
    const int tw = fc::tune_lane_width(A, X, Y, gcn, 1, 1);
    CHECK(tw == 4 || tw == 8);
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "wrapper ok", failures);
    return failures ? 1 : 0;
}
