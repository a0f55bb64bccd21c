/*
 * fmm_oracle_impl.h — body of the CPU oracle, included twice by fmm_oracle.c
 * with REAL = float (SFX f32) and REAL = double (SFX f64).
 *
 * TEST INFRASTRUCTURE ONLY (see fmm_oracle.c header).
 */

/* ops.hpp:53-56 — exact sigmoid, no LUT, no clamp */
static REAL SFX(sigmoid)(REAL s) { return (REAL)1 / ((REAL)1 + EXPF(-s)); }

/* ops.hpp:58-80; OR_VOP_MLP is make_toy_mlp_vop (apps.hpp:58-64):
 * sigmoid(w_x*x + w_y*y + bias), left to right */
static void SFX(apply_vop)(const or_spec* sp, const REAL* x, const REAL* y, REAL* out, int64_t d) {
    int64_t i;
    switch (sp->vop) {
        case OR_VOP_MLP:
            for (i = 0; i < d; ++i)
                out[i] = SFX(sigmoid)((REAL)sp->mlp_wx * x[i] + (REAL)sp->mlp_wy * y[i] + (REAL)sp->mlp_b);
            break;
        case OR_VOP_ADD: for (i = 0; i < d; ++i) out[i] = x[i] + y[i]; break;
        case OR_VOP_MUL: for (i = 0; i < d; ++i) out[i] = x[i] * y[i]; break;
        case OR_VOP_SEL2ND: for (i = 0; i < d; ++i) out[i] = y[i]; break;
        default: for (i = 0; i < d; ++i) out[i] = x[i] - y[i]; break; /* SUB */
    }
}

/* ops.hpp:82-106, plus SQNORM = NORM without the square root (the sq loop of
 * the t-distribution / FR-attractive USER-VOP lambdas) */
static REAL SFX(apply_rop)(int rop, const REAL* t, int64_t d) {
    REAL s;
    int64_t i;
    switch (rop) {
        case OR_ROP_RSUM: s = 0; for (i = 0; i < d; ++i) s += t[i]; return s;
        case OR_ROP_RMUL: s = 1; for (i = 0; i < d; ++i) s *= t[i]; return s;
        case OR_ROP_NORM: s = 0; for (i = 0; i < d; ++i) s += t[i] * t[i]; return SQRTF(s);
        default: s = 0; for (i = 0; i < d; ++i) s += t[i] * t[i]; return s; /* SQNORM */
    }
}

/* ops.hpp:108-121 plus TDIST 1/(1+s) and SQK s/k */
static REAL SFX(apply_sop)(const or_spec* sp, REAL s) {
    switch (sp->sop) {
        case OR_SOP_SIGMOID: return SFX(sigmoid)(s);
        case OR_SOP_SCAL: return (REAL)sp->alpha * s;
        case OR_SOP_TDIST: return (REAL)1 / ((REAL)1 + s);
        case OR_SOP_SQK: return s / (REAL)sp->k;
        default: return s;
    }
}

/* ops.hpp:166-182 */
static void SFX(apply_aop)(int aop, REAL* acc, const REAL* w, int64_t d) {
    int64_t i;
    if (aop == OR_AOP_AMAX) {
        for (i = 0; i < d; ++i) acc[i] = (acc[i] < w[i]) ? w[i] : acc[i];
    } else {
        for (i = 0; i < d; ++i) acc[i] += w[i];
    }
}

/* update_u, kernel.hpp:81-107. The MUL_VOP extension follows the USER-VOP
 * lambda route the reference needs for configs 3/4: the "VOP output" is
 * out_j = h * t_j with h = sop(rop(t)), the message is a vector, SOP is NOOP
 * and MOP=MUL gives w_j = a_uv * out_j (ops.hpp:150-156). With ROP=NOOP there
 * is no scalar to scale by and MUL_VOP acts as the vector-message MUL. */
static void SFX(update_u)(const int64_t* cols, const REAL* vals, int64_t nk, const REAL* x_u,
                          const REAL* Y, int64_t d, const or_spec* sp, REAL* z_u, REAL* tmp,
                          REAL* w) {
    const REAL identity = sp->aop == OR_AOP_AMAX ? -(REAL)INFINITY : (REAL)0;
    int64_t j, k;
    for (j = 0; j < d; ++j) z_u[j] = identity;
    for (k = 0; k < nk; ++k) {
        const REAL* y_v = Y + cols[k] * d;
        const REAL a = vals ? vals[k] : (REAL)1;
        if (sp->mop == OR_MOP_MUL_VOP && sp->rop != OR_ROP_NOOP) {
            REAL s, h;
            SFX(apply_vop)(sp, x_u, y_v, tmp, d);
            s = SFX(apply_rop)(sp->rop, tmp, d);
            h = SFX(apply_sop)(sp, s);
            for (j = 0; j < d; ++j) tmp[j] = h * tmp[j];
            for (j = 0; j < d; ++j) w[j] = a * tmp[j];
        } else if (sp->rop != OR_ROP_NOOP) { /* scalar message, ops.hpp:45 */
            REAL s, h;
            SFX(apply_vop)(sp, x_u, y_v, tmp, d);
            s = SFX(apply_rop)(sp->rop, tmp, d);
            h = SFX(apply_sop)(sp, s);
            if (sp->mop == OR_MOP_SEL2ND) for (j = 0; j < d; ++j) w[j] = y_v[j];
            else for (j = 0; j < d; ++j) w[j] = h * y_v[j]; /* a_uv ignored, ops.hpp:131-137 */
        } else { /* vector message */
            SFX(apply_vop)(sp, x_u, y_v, tmp, d);
            if (sp->sop != OR_SOP_NOOP)
                for (j = 0; j < d; ++j) tmp[j] = SFX(apply_sop)(sp, tmp[j]);
            if (sp->mop == OR_MOP_SEL2ND) for (j = 0; j < d; ++j) w[j] = y_v[j];
            else for (j = 0; j < d; ++j) w[j] = a * tmp[j];
        }
        SFX(apply_aop)(sp->aop, z_u, w, d);
    }
}

/* row_sigmoid_embed<W> (kernel.hpp:118-143), row_spmm_gcn<W> (145-158),
 * row_fr_layout<W> (160-190) and the d > 256 second sweep
 * row_tail_streamed (194-225), for one row, written into z_row. */
static void SFX(blocked_row)(int pattern, int W, const int64_t* cols, const REAL* vals, int64_t nk,
                             const REAL* xu, const REAL* Y, int64_t d, REAL alpha, REAL* z_acc,
                             REAL* z_row) {
    const int64_t db = d < OR_BLOCKED_DIM_LIMIT ? d : OR_BLOCKED_DIM_LIMIT;
    const int64_t full = db - db % W;
    int64_t j, b, k;
    int l;
    REAL acc[16];
    for (j = 0; j < db; ++j) z_acc[j] = 0;
    for (k = 0; k < nk; ++k) {
        const REAL* yv = Y + cols[k] * d;
        REAL h;
        if (pattern == OR_PATTERN_SPMM_GCN) {
            const REAL a = vals ? vals[k] : (REAL)1;
            for (b = 0; b < full; b += W)
                for (l = 0; l < W; ++l) z_acc[b + l] += a * yv[b + l];
            for (j = full; j < db; ++j) z_acc[j] += a * yv[j];
            continue;
        }
        for (l = 0; l < W; ++l) acc[l] = 0;
        if (pattern == OR_PATTERN_SIGMOID_EMBED) {
            REAL dot = 0;
            for (b = 0; b < full; b += W)
                for (l = 0; l < W; ++l) acc[l] += xu[b + l] * yv[b + l];
            for (l = 0; l < W; ++l) dot += acc[l];
            for (j = full; j < d; ++j) dot += xu[j] * yv[j];
            h = SFX(sigmoid)(dot);
        } else { /* FR_LAYOUT */
            REAL sq = 0;
            for (b = 0; b < full; b += W)
                for (l = 0; l < W; ++l) {
                    const REAL e = xu[b + l] + yv[b + l];
                    acc[l] += e * e;
                }
            for (l = 0; l < W; ++l) sq += acc[l];
            for (j = full; j < d; ++j) {
                const REAL e = xu[j] + yv[j];
                sq += e * e;
            }
            h = alpha * SQRTF(sq);
        }
        for (b = 0; b < full; b += W)
            for (l = 0; l < W; ++l) z_acc[b + l] += h * yv[b + l];
        for (j = full; j < db; ++j) z_acc[j] += h * yv[j];
    }
    for (j = 0; j < db; ++j) z_row[j] = z_acc[j];
    if (d > OR_BLOCKED_DIM_LIMIT) {
        for (j = OR_BLOCKED_DIM_LIMIT; j < d; ++j) z_row[j] = 0;
        for (k = 0; k < nk; ++k) {
            const REAL* y_v = Y + cols[k] * d;
            REAL h;
            if (pattern == OR_PATTERN_SIGMOID_EMBED) {
                REAL dot = 0;
                for (j = 0; j < d; ++j) dot += xu[j] * y_v[j];
                h = SFX(sigmoid)(dot);
            } else if (pattern == OR_PATTERN_FR_LAYOUT) {
                REAL sq = 0;
                for (j = 0; j < d; ++j) {
                    const REAL e = xu[j] + y_v[j];
                    sq += e * e;
                }
                h = alpha * SQRTF(sq);
            } else {
                h = vals ? vals[k] : (REAL)1;
            }
            for (j = OR_BLOCKED_DIM_LIMIT; j < d; ++j) z_row[j] += h * y_v[j];
        }
    }
}

typedef struct {
    const or_job* job;
    const REAL* vals;
    const REAL* X;
    const REAL* Y;
    REAL* Z;
    int64_t lo, hi; /* range of selected-row indices */
    int pattern;
} SFX(or_work);

static void* SFX(worker)(void* arg) {
    const SFX(or_work)* w = (const SFX(or_work)*)arg;
    const or_job* J = w->job;
    const int64_t d = J->d;
    const int64_t ws = 2 * d > OR_WORKSPACE_PANEL ? 2 * d : OR_WORKSPACE_PANEL;
    REAL* scratch = (REAL*)malloc(sizeof(REAL) * (size_t)(ws + 2 * d));
    int64_t i;
    const int blocked = w->pattern != OR_PATTERN_GENERIC && d >= OR_SPECIALIZE_DIM_MIN;
    for (i = w->lo; i < w->hi; ++i) {
        const int64_t u = J->rows ? J->rows[i] : i;
        const int64_t b = J->row_ptr[u], e = J->row_ptr[u + 1];
        const REAL* vals = w->vals ? w->vals + b : NULL;
        REAL* z = w->Z + i * d;
        if (blocked)
            SFX(blocked_row)(w->pattern, J->lane_width, J->col + b, vals, e - b, w->X + u * d, w->Y,
                             d, (REAL)J->spec.alpha, scratch, z);
        else
            SFX(update_u)(J->col + b, vals, e - b, w->X + u * d, w->Y, d, &J->spec, z, scratch,
                          scratch + d);
    }
    free(scratch);
    return NULL;
}

/* fused_mm (kernel.hpp:297-353) over the selected rows (all rows when
 * job->rows == NULL), t workers over part1d-style contiguous ranges. Output
 * row i of Z is selected row i. The worker split never changes results
 * (kernel.hpp:290-295). */
static int SFX(run)(const or_job* J, const REAL* vals, const REAL* X, const REAL* Y, REAL* Z) {
    const int pattern = or_pattern_of(&J->spec);
    const int64_t nsel = J->rows ? J->nrows_sel : J->m;
    int t = J->threads < 1 ? 1 : J->threads;
    int i;
    SFX(or_work) work[256];
    pthread_t th[256];
    if (t > 256) t = 256;
    if ((int64_t)t > nsel) t = nsel > 0 ? (int)nsel : 1;
    for (i = 0; i < t; ++i) {
        work[i].job = J;
        work[i].vals = vals;
        work[i].X = X;
        work[i].Y = Y;
        work[i].Z = Z;
        work[i].lo = nsel * i / t;
        work[i].hi = nsel * (i + 1) / t;
        work[i].pattern = pattern;
    }
    if (t == 1) {
        SFX(worker)(&work[0]);
        return 0;
    }
    for (i = 0; i < t; ++i) pthread_create(&th[i], NULL, SFX(worker), &work[i]);
    for (i = 0; i < t; ++i) pthread_join(th[i], NULL);
    return 0;
}
