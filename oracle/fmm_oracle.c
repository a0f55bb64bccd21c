/*
 * fmm_oracle.c — CPU ORACLE for the FusedMM hot path. TEST INFRASTRUCTURE.
 *
 * A plain-C restatement of the reference algorithm, used only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * It is never linked into, called by, or used as a fallback for the product
 * library (paper_2011_06391_b200/, libfusedmm_cuda.so).
 *
 * It follows, function by function:
 *   fused_mm                 /root/reference/proj/include/fusedmm/kernel.hpp:297-353
 *   update_u                 kernel.hpp:81-107
 *   row_sigmoid_embed<W>     kernel.hpp:118-143
 *   row_spmm_gcn<W>          kernel.hpp:145-158
 *   row_fr_layout<W>         kernel.hpp:160-190
 *   row_tail_streamed        kernel.hpp:194-225
 *   part1d                   kernel.hpp:24-49
 *   sigmoid / apply_*        ops.hpp:53-187,   pattern_of ops.hpp:189-203
 * Built with -ffp-contract=off like the reference (CMakeLists.txt:19-26), so
 * its float results are bitwise those of fusedmm::fused_mm<float>; this is
 * pinned in tests/test_oracle.py against (a) the reference's own known-answer
 * tests, (b) golden vectors produced by the reference itself
 * (tests/golden/make_golden.py via oracle/_ref) and (c) oracle/_ref directly
 * when it is built.
 *
 * Device-only op extensions (SQNORM, TDIST, SQK, MUL_VOP) are restated as the
 * USER-VOP lambda route the reference needs for configs 3 and 4
 * (SURVEY.md §8(a) "Oracle op definitions").
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_VOP_ADD = 0, OR_VOP_MUL = 1, OR_VOP_SEL2ND = 2, OR_VOP_SUB = 3, OR_VOP_USER = 4,
       OR_VOP_MLP = 16 };
enum { OR_ROP_NOOP = 0, OR_ROP_RSUM = 1, OR_ROP_RMUL = 2, OR_ROP_NORM = 3, OR_ROP_USER = 4,
       OR_ROP_SQNORM = 16 };
enum { OR_SOP_NOOP = 0, OR_SOP_SIGMOID = 1, OR_SOP_SCAL = 2, OR_SOP_USER = 3, OR_SOP_TDIST = 16,
       OR_SOP_SQK = 17 };
enum { OR_MOP_MUL = 0, OR_MOP_SEL2ND = 1, OR_MOP_USER = 2, OR_MOP_MUL_VOP = 16 };
enum { OR_AOP_ASUM = 0, OR_AOP_AMAX = 1, OR_AOP_USER = 2 };
enum { OR_PATTERN_SIGMOID_EMBED = 0, OR_PATTERN_SPMM_GCN = 1, OR_PATTERN_FR_LAYOUT = 2,
       OR_PATTERN_GENERIC = 3 };

/* kernel.hpp:61-70 */
#define OR_WORKSPACE_PANEL 512
#define OR_BLOCKED_DIM_LIMIT 256
#define OR_SPECIALIZE_DIM_MIN 32

typedef struct {
    int32_t vop, rop, sop, mop, aop;
    double alpha;
    double k;
    double mlp_wx, mlp_wy, mlp_b; /* OR_VOP_MLP: apps.hpp:58-64 toy hook */
} or_spec;

typedef struct {
    int64_t m, n, d;
    const int64_t* row_ptr;
    const int64_t* col;
    or_spec spec;
    int lane_width;      /* KernelOptions.lane_width: 4, 8 or 16 */
    int threads;
    const int64_t* rows; /* optional row selection */
    int64_t nrows_sel;
} or_job;

/* ops.hpp:189-203; the extension ops never match a known pattern, so they
 * take the generic update_u path exactly like a USER slot (ops.hpp:191). */
static int or_pattern_of(const or_spec* s) {
    if (s->rop == OR_ROP_SQNORM || s->sop == OR_SOP_TDIST || s->sop == OR_SOP_SQK ||
        s->mop == OR_MOP_MUL_VOP)
        return OR_PATTERN_GENERIC;
    if (s->vop == OR_VOP_MUL && s->rop == OR_ROP_RSUM && s->sop == OR_SOP_SIGMOID &&
        s->mop == OR_MOP_MUL && s->aop == OR_AOP_ASUM)
        return OR_PATTERN_SIGMOID_EMBED;
    if (s->vop == OR_VOP_SEL2ND && s->rop == OR_ROP_NOOP && s->sop == OR_SOP_NOOP &&
        s->mop == OR_MOP_MUL && s->aop == OR_AOP_ASUM)
        return OR_PATTERN_SPMM_GCN;
    if (s->vop == OR_VOP_ADD && s->rop == OR_ROP_NORM && s->sop == OR_SOP_SCAL &&
        s->mop == OR_MOP_MUL && s->aop == OR_AOP_ASUM)
        return OR_PATTERN_FR_LAYOUT;
    return OR_PATTERN_GENERIC;
}

#define REAL float
#define SFX(name) name##_f32
#define EXPF expf
#define SQRTF sqrtf
#include "fmm_oracle_impl.h"
#undef REAL
#undef SFX
#undef EXPF
#undef SQRTF

#define REAL double
#define SFX(name) name##_f64
#define EXPF exp
#define SQRTF sqrt
#include "fmm_oracle_impl.h"
#undef REAL
#undef SFX
#undef EXPF
#undef SQRTF

static int check(const or_job* J, int64_t ny) {
    int64_t i, max_col = -1;
    const int64_t nnz = J->m > 0 ? J->row_ptr[J->m] : 0;
    if (J->d < 1 || J->m < 0) return 1;
    if (J->lane_width != 4 && J->lane_width != 8 && J->lane_width != 16) return 1;
    if (J->spec.vop == OR_VOP_USER || J->spec.rop == OR_ROP_USER || J->spec.sop == OR_SOP_USER ||
        J->spec.mop == OR_MOP_USER || J->spec.aop == OR_AOP_USER)
        return 2;
    for (i = 0; i < nnz; ++i)
        if (J->col[i] > max_col) max_col = J->col[i];
    if (ny < max_col + 1) return 1; /* kernel.hpp:278-281 */
    return 0;
}

/* Returns 0 on success, 1 on bad arguments, 2 for USER slots. */
int fmm_oracle_fused_mm_f32(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col,
                            const float* val, int64_t d, const float* X, int64_t ny,
                            const float* Y, const or_spec* spec, int lane_width, int threads,
                            const int64_t* rows, int64_t nrows_sel, float* Z) {
    or_job J;
    int rc;
    J.m = m; J.n = n; J.d = d; J.row_ptr = row_ptr; J.col = col; J.spec = *spec;
    J.lane_width = lane_width; J.threads = threads; J.rows = rows; J.nrows_sel = nrows_sel;
    if ((rc = check(&J, ny)) != 0) return rc;
    return run_f32(&J, val, X, Y, Z);
}

int fmm_oracle_fused_mm_f64(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col,
                            const double* val, int64_t d, const double* X, int64_t ny,
                            const double* Y, const or_spec* spec, int lane_width, int threads,
                            const int64_t* rows, int64_t nrows_sel, double* Z) {
    or_job J;
    int rc;
    J.m = m; J.n = n; J.d = d; J.row_ptr = row_ptr; J.col = col; J.spec = *spec;
    J.lane_width = lane_width; J.threads = threads; J.rows = rows; J.nrows_sel = nrows_sel;
    if ((rc = check(&J, ny)) != 0) return rc;
    return run_f64(&J, val, X, Y, Z);
}

/* part1d, kernel.hpp:24-49 */
int fmm_oracle_part1d(int64_t m, const int64_t* row_ptr, int t, int64_t* b) {
    int64_t nnz, row = 0;
    int i;
    if (t < 1) return 1;
    nnz = row_ptr[m];
    b[0] = 0;
    b[t] = m;
    if (nnz == 0) {
        for (i = 1; i < t; ++i) b[i] = m * i / t;
        return 0;
    }
    for (i = 1; i < t; ++i) {
        while (row < m && row_ptr[row] * (int64_t)t < (int64_t)i * nnz) ++row;
        b[i] = row;
    }
    return 0;
}

int fmm_oracle_pattern_of(const or_spec* s) { return or_pattern_of(s); }
