/*
 * oracle/oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of the vector-Jacobian
 * products (vjp) of scan, reduce, reduce_by_index and scatter, written from
 * PAPER.md (arXiv 2202.10297, Schenck et al., "AD for an Array Language with
 * Nested Parallelism").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no
 * code, header, constant or helper with the CUDA path under
 * paper_2202_10297_b200/; the enum values below are re-declared from
 * DESIGN.md, not included from include/vjp.h.
 *
 * Arithmetic: every intermediate is `long double` (x87 80-bit on x86-64,
 * u ~ 5.4e-20); each output is rounded once to its storage dtype.  The rules
 * are followed literally, in the paper's order, with no blocking, fusion or
 * reordering:
 *
 *   scan            P:1143-1158 (sec 5.2): forward loop rs[i] = rs[i-1] (.) as[i],
 *                   then the reversed loop applying Eq. 3 to every
 *                   unrolled statement.  NOT the lin_o scan (that is the GPU's
 *                   algorithm); this is the O(n) sequential definition.
 *   reduce          ADD: P:1034-1038.  MUL: the paper's GENERAL rule
 *                   P:1000-1011 (exclusive scan ls, reversed exclusive scan rs,
 *                   a_i += d(l_i*a_i*r_i)/da_i * ybar = l_i*r_i*ybar), deliberately
 *                   NOT the (p, z) special case of P:1040-1061 that the GPU uses.
 *                   MIN/MAX: P:1063-1074, argmin with the FIRST index (strict
 *                   compare in a left-to-right loop).
 *   reduce_by_index P:1098-1106 forward semantics (the literal loop), return
 *                   sweep P:1120-1126 (ybar replaced by hs_bar[inds[i]]); MUL per
 *                   bin again through the general l_i*r_i rule (per-bin running
 *                   products forward and backward).
 *   scatter         P:1274-1275: vs_bar += gather is ys_bar;
 *                   xs_bar = scatter ys_bar is (replicate m 0).
 *   kmeans          SURVEY 8f row f3 / P:1663-1720: f(C) = sum_p min_j ||p - c_j||^2
 *                   (reading R15: squared distance), its vjp (reduce(+) adjoint,
 *                   the min-reduce sparse adjoint with the FIRST index, the map's
 *                   vjp 2(c - p) accumulated per center) and the jvp of that vjp
 *                   in the all-ones direction (the Hessian diagonal),
 *                   all by the literal per-point loop.
 *
 * Readings of the paper where it is silent or garbled:
 *   R1 MAT2 scan order R_i = R_{i-1} . A_i (P:1137 semantics of scan).
 *   R2 LINREC element (d, c), (d1,c1) (.) (d2,c2) = (d2 + c2*d1, c2*c1) = lin_o
 *       used as a primal operator.
 *   R3 MIN/MAX scan subgradient: pick left (the carry) on ties.
 *   R4 out-of-range bins / scatter targets are skipped, adjoint 0.
 *   R5 duplicate scatter targets: precondition; reported as 5.
 *   R6 default overwrite; flags&1 (ACCUMULATE) gives the paper's +=.
 *   R7 n = 0: no-op; reduce result is the neutral element; empty bin has no
 *      winner (-1).
 *   R8 reduce(MUL) one-zero case uses the product of the NONZERO elements
 *      (P:1051 literally says y*ybar but y = 0 there); the general rule used
 *      here reaches that value without special-casing it.
 *
 * Parity pins (tests/test_oracle_pins.py) check every function here against
 * exact rational forward-mode (dual-number) Jacobians of the primal
 * definitions, central finite differences (exact for multilinear ops), the
 * paper's/SPEC's worked examples (tests/golden/) and closed forms.  No
 * function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef long double LD;

/* Re-declared (not shared) tags; values documented in DESIGN.md. */
enum { O_F32 = 1, O_F64 = 2 };
enum { O_I32 = 1, O_I64 = 2 };
enum { O_ADD = 1, O_MUL = 2, O_MIN = 3, O_MAX = 4, O_LINREC = 5, O_MAT2 = 6 };
enum { O_OK = 0, O_EINVAL = 1, O_EUNSUPPORTED = 2, O_EDUPINDEX = 5 };
enum { O_ACCUMULATE = 1u };

/* scalars per element of a scan operand */
static int width_of(int op) {
    switch (op) {
    case O_ADD: case O_MUL: case O_MIN: case O_MAX: return 1;
    case O_LINREC: return 2;
    case O_MAT2: return 4;
    }
    return 0;
}

static LD ld_get(int dtype, const void *p, int64_t k) {
    return dtype == O_F32 ? (LD)((const float *)p)[k] : (LD)((const double *)p)[k];
}
/* store one value, rounding once to the storage dtype; ACCUMULATE adds to
 * the existing value first (still one rounding of the long-double sum). */
static void ld_put(int dtype, void *p, int64_t k, LD v, unsigned flags) {
    if (dtype == O_F32) {
        float *q = (float *)p;
        q[k] = (flags & O_ACCUMULATE) ? (float)((LD)q[k] + v) : (float)v;
    } else {
        double *q = (double *)p;
        q[k] = (flags & O_ACCUMULATE) ? (double)((LD)q[k] + v) : (double)v;
    }
}
static int64_t idx_get(int itype, const void *p, int64_t k) {
    return itype == O_I32 ? (int64_t)((const int32_t *)p)[k] : ((const int64_t *)p)[k];
}

/* ------------------------------------------------------------------ */
/* The primal operator (.) of each scan tag, on long-double elements.  */
/* ------------------------------------------------------------------ */
static void op_apply(int op, const LD *r, const LD *a, LD *out) {
    switch (op) {
    case O_ADD: out[0] = r[0] + a[0]; break;
    case O_MUL: out[0] = r[0] * a[0]; break;
    case O_MIN: out[0] = (r[0] <= a[0]) ? r[0] : a[0]; break;   /* R3: pick left on tie */
    case O_MAX: out[0] = (r[0] >= a[0]) ? r[0] : a[0]; break;
    case O_LINREC: /* R2: (D, C) (.) (d, c) = (d + c*D, c*C) */
        out[0] = a[0] + a[1] * r[0];
        out[1] = a[1] * r[1];
        break;
    case O_MAT2: /* R1: R . A, 2x2 row-major */
        out[0] = r[0] * a[0] + r[1] * a[2];
        out[1] = r[0] * a[1] + r[1] * a[3];
        out[2] = r[2] * a[0] + r[3] * a[2];
        out[3] = r[2] * a[1] + r[3] * a[3];
        break;
    }
}

/*
 * Eq. 3 for v = r (.) a, written out per tag:
 *   abar += (dv/da)^T vbar      (written to ga)
 *   rbar += (dv/dr)^T vbar      (added into gr)
 * These are the partial derivatives of op_apply above, entry by entry.
 */
static void op_vjp(int op, const LD *r, const LD *a, const LD *vbar, LD *ga, LD *gr) {
    switch (op) {
    case O_ADD:
        ga[0] = vbar[0];
        gr[0] += vbar[0];
        break;
    case O_MUL:
        ga[0] = r[0] * vbar[0];
        gr[0] += a[0] * vbar[0];
        break;
    case O_MIN: {
        int left = (r[0] <= a[0]);
        ga[0] = left ? 0.0L : vbar[0];
        gr[0] += left ? vbar[0] : 0.0L;
        break;
    }
    case O_MAX: {
        int left = (r[0] >= a[0]);
        ga[0] = left ? 0.0L : vbar[0];
        gr[0] += left ? vbar[0] : 0.0L;
        break;
    }
    case O_LINREC:
        /* v0 = a0 + a1*r0 ; v1 = a1*r1 */
        ga[0] = vbar[0];                          /* dv0/da0 = 1, dv1/da0 = 0 */
        ga[1] = r[0] * vbar[0] + r[1] * vbar[1];  /* dv0/da1 = r0, dv1/da1 = r1 */
        gr[0] += a[1] * vbar[0];                  /* dv0/dr0 = a1 */
        gr[1] += a[1] * vbar[1];                  /* dv1/dr1 = a1 */
        break;
    case O_MAT2:
        /* v = r . a :  dv_ij/da_kj = r_ik  ->  abar = r^T vbar ;
         *              dv_ij/dr_ik = a_kj  ->  rbar += vbar a^T   */
        ga[0] = r[0] * vbar[0] + r[2] * vbar[2];
        ga[1] = r[0] * vbar[1] + r[2] * vbar[3];
        ga[2] = r[1] * vbar[0] + r[3] * vbar[2];
        ga[3] = r[1] * vbar[1] + r[3] * vbar[3];
        gr[0] += vbar[0] * a[0] + vbar[1] * a[1];
        gr[1] += vbar[0] * a[2] + vbar[1] * a[3];
        gr[2] += vbar[2] * a[0] + vbar[3] * a[1];
        gr[3] += vbar[2] * a[2] + vbar[3] * a[3];
        break;
    }
}

/*
 * vjp of  ys = scan (.) e as, as the paper derives it
 * (P:1143-1158):
 *     rs[0] = as[0];  rs[i] = rs[i-1] (.) as[i]                 (forward)
 *     rbar = copy ysbar
 *     for i = n-1 .. 1:
 *         rbar[i-1] += d(rs[i-1] (.) as[i])/d rs[i-1] * rbar[i]
 *         asbar[i]  += d(rs[i-1] (.) as[i])/d as[i]   * rbar[i]
 *     asbar[0] += rbar[0]
 * `as` may be NULL for ADD (the derivative does not read it).  ys (nullable)
 * receives the primal scan.
 *
 * cond (nullable, n*W doubles): the condition scale of each adjoint entry,
 * sum_terms |term| (SURVEY 8c reading A22), for comparing signed data where
 * an adjoint entry is a cancelling sum.  Every adjoint entry of the loop above
 * is a sum of products of entries of ysbar, as and rs; cond runs the SAME loop
 * on |ysbar|, |as| and rs recomputed from |as|, so each product becomes its
 * absolute value and the sum becomes sum |term| exactly (up to rounding: all
 * addends are >= 0).  ADD, MUL, LINREC and MAT2 are polynomials with +1
 * coefficients in these entries (op_apply / op_vjp above), so this is the
 * literal sum of |monomials|.  MIN / MAX select by comparing the REAL rs and
 * as (the branch taken is part of the derivative, not a term), so their
 * selections use the real values and only ysbar is replaced by |ysbar|.
 */
static void scan_cond(int op, int dtype, int64_t n, const void *as, const void *ys_bar, double *cond);

int oracle_vjp_scan(int op, int dtype, int64_t n, const void *as, const void *ys_bar,
                    void *as_bar, void *ys, double *cond, unsigned flags) {
    int w = width_of(op);
    if (w == 0 || (dtype != O_F32 && dtype != O_F64) || n < 0) return O_EINVAL;
    if (n == 0) return O_OK;
    if (!ys_bar || !as_bar || (!as && op != O_ADD) || (!as && ys)) return O_EINVAL;

    LD *rs = NULL;
    if (as) {
        rs = (LD *)malloc(sizeof(LD) * (size_t)n * w);
        if (!rs) return O_EINVAL;
        for (int k = 0; k < w; ++k) rs[k] = ld_get(dtype, as, k);
        for (int64_t i = 1; i < n; ++i) {
            LD a[4];
            for (int k = 0; k < w; ++k) a[k] = ld_get(dtype, as, i * w + k);
            op_apply(op, &rs[(i - 1) * w], a, &rs[i * w]);
        }
        if (ys)
            for (int64_t i = 0; i < n * w; ++i) ld_put(dtype, ys, i, rs[i], 0);
    }

    LD *rbar = (LD *)malloc(sizeof(LD) * (size_t)n * w);
    if (!rbar) { free(rs); return O_EINVAL; }
    for (int64_t i = 0; i < n * w; ++i) rbar[i] = ld_get(dtype, ys_bar, i);

    LD one[4] = {0, 0, 0, 0};   /* ADD ignores operand values */
    for (int64_t i = n - 1; i >= 1; --i) {
        LD a[4], ga[4];
        const LD *r = rs ? &rs[(i - 1) * w] : one;
        if (as) for (int k = 0; k < w; ++k) a[k] = ld_get(dtype, as, i * w + k);
        else    for (int k = 0; k < w; ++k) a[k] = 0.0L;
        op_vjp(op, r, a, &rbar[i * w], ga, &rbar[(i - 1) * w]);
        for (int k = 0; k < w; ++k) ld_put(dtype, as_bar, i * w + k, ga[k], flags);
    }
    for (int k = 0; k < w; ++k) ld_put(dtype, as_bar, k, rbar[k], flags);

    free(rbar);
    free(rs);
    if (cond) scan_cond(op, dtype, n, as, ys_bar, cond);
    return O_OK;
}

/* the loop of oracle_vjp_scan on absolute values (see its comment) */
static void scan_cond(int op, int dtype, int64_t n, const void *as, const void *ys_bar, double *cond) {
    const int w = width_of(op);
    const int sel = (op == O_MIN || op == O_MAX);
    LD *rs = NULL;
    if (as) {
        rs = (LD *)malloc(sizeof(LD) * (size_t)n * w);
        if (!rs) return;
        for (int k = 0; k < w; ++k) rs[k] = sel ? ld_get(dtype, as, k) : fabsl(ld_get(dtype, as, k));
        for (int64_t i = 1; i < n; ++i) {
            LD a[4];
            for (int k = 0; k < w; ++k) {
                a[k] = ld_get(dtype, as, i * w + k);
                if (!sel) a[k] = fabsl(a[k]);
            }
            op_apply(op, &rs[(i - 1) * w], a, &rs[i * w]);
        }
    }
    LD *rbar = (LD *)malloc(sizeof(LD) * (size_t)n * w);
    if (!rbar) { free(rs); return; }
    for (int64_t i = 0; i < n * w; ++i) rbar[i] = fabsl(ld_get(dtype, ys_bar, i));
    LD zero[4] = {0, 0, 0, 0};
    for (int64_t i = n - 1; i >= 1; --i) {
        LD a[4], ga[4];
        const LD *r = rs ? &rs[(i - 1) * w] : zero;
        for (int k = 0; k < w; ++k) {
            a[k] = as ? ld_get(dtype, as, i * w + k) : 0.0L;
            if (!sel) a[k] = fabsl(a[k]);
        }
        op_vjp(op, r, a, &rbar[i * w], ga, &rbar[(i - 1) * w]);
        for (int k = 0; k < w; ++k) cond[i * w + k] = (double)ga[k];
    }
    for (int k = 0; k < w; ++k) cond[k] = (double)rbar[k];
    free(rbar);
    free(rs);
}

/*
 * vjp of  y = reduce (.) e as.
 *   ADD      : y = sum; asbar_i += ybar.
 *   MUL      : general rule P:1006-1011 with (.) = *:
 *                ls = scan^exc (*) 1 as ; rs = reverse (scan^exc (*) 1 (reverse as))
 *                asbar_i += ls_i * rs_i * ybar
 *              `arg` receives the first zero index (-1 if none), `zeros` the
 *              number of zeros (IEEE: -0.0 == 0.0 counts), for comparison with
 *              the GPU's (p, z, i0) forward state of P:1055-1058.
 *   MIN/MAX  : (y, i_y) = argmin with the first index on ties;
 *              asbar[i_y] += ybar.  Dense (overwrite) mode
 *              writes 0 everywhere else; ACCUMULATE touches only i_y.
 * y_bar is a host pointer to one element of dtype; y (nullable) receives y.
 */
/*
 * The paper's GENERAL reduce rule for an operator with no
 * special case (here the d-vector operators LINREC and MAT2):
 *     ls = scan^exc (.) e as
 *     rs = reverse as |> scan^exc (\x y -> y (.) x) e |> reverse     (A18)
 *     asbar_i += d(l_i (.) a_i (.) r_i)/da_i . ybar
 * The last line is Eq. 3 applied to v = x (.) r_i with x = l_i (.) a_i:
 * xbar = dv/dx^T ybar, then abar = d(l_i (.) a_i)/da_i^T xbar (op_vjp twice).
 * y_bar holds one element (W scalars); y receives the reduction.
 */
static int reduce_general(int op, int dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                          void *y, int64_t *arg, int64_t *zeros, unsigned flags) {
    const int W = width_of(op);
    if (!y_bar || (n > 0 && (!as || !as_bar))) return O_EINVAL;
    LD ybar[4], e[4];
    for (int k = 0; k < W; ++k) ybar[k] = ld_get(dtype, y_bar, k);
    /* neutral element: LINREC (0, 1), MAT2 I */
    if (op == O_LINREC) { e[0] = 0.0L; e[1] = 1.0L; }
    else { e[0] = 1.0L; e[1] = 0.0L; e[2] = 0.0L; e[3] = 1.0L; }
    LD *ls = (LD *)malloc(sizeof(LD) * (size_t)(n > 0 ? n : 1) * W);
    LD *rs = (LD *)malloc(sizeof(LD) * (size_t)(n > 0 ? n : 1) * W);
    if (!ls || !rs) { free(ls); free(rs); return O_EINVAL; }
    LD acc[4], a[4], t[4];
    for (int k = 0; k < W; ++k) acc[k] = e[k];
    for (int64_t i = 0; i < n; ++i) {   /* ls: exclusive forward scan */
        for (int k = 0; k < W; ++k) { ls[i * W + k] = acc[k]; a[k] = ld_get(dtype, as, i * W + k); }
        op_apply(op, acc, a, t);
        for (int k = 0; k < W; ++k) acc[k] = t[k];
    }
    if (y) for (int k = 0; k < W; ++k) ld_put(dtype, y, k, acc[k], 0);
    for (int k = 0; k < W; ++k) acc[k] = e[k];
    for (int64_t i = n - 1; i >= 0; --i) {  /* rs: exclusive scan of the reversed array, flipped (.) */
        for (int k = 0; k < W; ++k) { rs[i * W + k] = acc[k]; a[k] = ld_get(dtype, as, i * W + k); }
        op_apply(op, a, acc, t);  /* (\x y -> y (.) x) acc a = a (.) acc */
        for (int k = 0; k < W; ++k) acc[k] = t[k];
    }
    for (int64_t i = 0; i < n; ++i) {
        LD x[4], xbar[4], gr_unused[4], ga[4], ga_r[4];
        for (int k = 0; k < W; ++k) a[k] = ld_get(dtype, as, i * W + k);
        op_apply(op, ls + i * W, a, x);                     /* x = l_i (.) a_i */
        for (int k = 0; k < W; ++k) xbar[k] = 0.0L;
        op_vjp(op, x, rs + i * W, ybar, ga_r, xbar);        /* xbar = d(x (.) r_i)/dx^T ybar */
        for (int k = 0; k < W; ++k) gr_unused[k] = 0.0L;
        op_vjp(op, ls + i * W, a, xbar, ga, gr_unused);     /* abar_i = d(l_i (.) a_i)/da_i^T xbar */
        for (int k = 0; k < W; ++k) ld_put(dtype, as_bar, i * W + k, ga[k], flags);
    }
    free(ls);
    free(rs);
    if (arg) *arg = -1;
    if (zeros) *zeros = 0;
    return O_OK;
}

int oracle_vjp_reduce(int op, int dtype, int64_t n, const void *as, const void *y_bar,
                      void *as_bar, void *y, int64_t *arg, int64_t *zeros, unsigned flags) {
    if ((dtype != O_F32 && dtype != O_F64) || n < 0) return O_EINVAL;
    if (op == O_LINREC || op == O_MAT2)
        return reduce_general(op, dtype, n, as, y_bar, as_bar, y, arg, zeros, flags);
    if (op != O_ADD && op != O_MUL && op != O_MIN && op != O_MAX) return O_EUNSUPPORTED;
    if (!y_bar || (n > 0 && (!as || !as_bar))) return O_EINVAL;
    LD ybar = ld_get(dtype, y_bar, 0);

    if (op == O_ADD) {
        LD s = 0.0L;
        for (int64_t i = 0; i < n; ++i) s += ld_get(dtype, as, i);
        for (int64_t i = 0; i < n; ++i) ld_put(dtype, as_bar, i, ybar, flags);
        if (y) ld_put(dtype, y, 0, s, 0);
        if (arg) *arg = -1;
        if (zeros) *zeros = 0;
        return O_OK;
    }
    if (op == O_MUL) {
        int64_t z = 0, i0 = -1;
        for (int64_t i = 0; i < n; ++i)
            if (ld_get(dtype, as, i) == 0.0L) { if (i0 < 0) i0 = i; ++z; }
        /* ls: exclusive forward scan of (*), neutral 1 */
        LD *ls = (LD *)malloc(sizeof(LD) * (size_t)(n > 0 ? n : 1));
        if (!ls) return O_EINVAL;
        LD acc = 1.0L;
        for (int64_t i = 0; i < n; ++i) { ls[i] = acc; acc = acc * ld_get(dtype, as, i); }
        if (y) ld_put(dtype, y, 0, acc, 0);
        /* rs: exclusive scan of the reversed array, reversed back; the flipped
         * operator (\x y -> y (.) x) of P:1009 equals (*) since * commutes.
         * Consumed on the fly in the same backward order. */
        LD racc = 1.0L;
        for (int64_t i = n - 1; i >= 0; --i) {
            ld_put(dtype, as_bar, i, ls[i] * racc * ybar, flags);
            racc = ld_get(dtype, as, i) * racc;
        }
        free(ls);
        if (arg) *arg = i0;
        if (zeros) *zeros = z;
        return O_OK;
    }
    /* MIN / MAX */
    if (n == 0) {
        if (y) ld_put(dtype, y, 0, op == O_MIN ? (LD)INFINITY : -(LD)INFINITY, 0);
        if (arg) *arg = -1;
        if (zeros) *zeros = 0;
        return O_OK;
    }
    LD best = ld_get(dtype, as, 0);
    int64_t bi = 0;
    for (int64_t i = 1; i < n; ++i) {
        LD v = ld_get(dtype, as, i);
        if (op == O_MIN ? (v < best) : (v > best)) { best = v; bi = i; }
    }
    if (flags & O_ACCUMULATE) {
        ld_put(dtype, as_bar, bi, ybar, flags);
    } else {
        for (int64_t i = 0; i < n; ++i) ld_put(dtype, as_bar, i, i == bi ? ybar : 0.0L, 0);
    }
    if (y) ld_put(dtype, y, 0, best, 0);
    if (arg) *arg = bi;
    if (zeros) *zeros = 0;
    return O_OK;
}

/*
 * vjp of  hs = reduce_by_index (.) e m inds as:
 *     hs = replicate m e ; for i in 0..n-1: hs[inds[i]] (.)= as[i]
 * (bins outside [0, m) are skipped, reading R4).  Return sweep P:1120-1126:
 * the reduce rule with ybar replaced by hs_bar[inds[i]]:
 *   ADD      asbar_i += hs_bar[b_i]
 *   MUL      asbar_i += hs_bar[b_i] * l_i * r_i, l_i / r_i the products of the
 *            elements of bin b_i before / after i (general rule per bin)
 *   MIN/MAX  asbar_i += hs_bar[b_i] iff i is the first index reaching the bin's
 *            extremum (winners[b], -1 for an empty bin)
 * hs (nullable) receives the primal histogram, zeros (nullable) the per-bin
 * zero count (MUL), winners (nullable) the per-bin winner (MIN/MAX).
 */
int oracle_vjp_reduce_by_index(int op, int dtype, int itype, int64_t n, int64_t m,
                               const void *inds, const void *as, const void *hs_bar,
                               void *as_bar, void *hs, int64_t *winners, int64_t *zeros,
                               unsigned flags) {
    if ((dtype != O_F32 && dtype != O_F64) || (itype != O_I32 && itype != O_I64)) return O_EINVAL;
    if (n < 0 || m < 1) return O_EINVAL;
    if (op != O_ADD && op != O_MUL && op != O_MIN && op != O_MAX) return O_EUNSUPPORTED;
    if (n > 0 && (!inds || !hs_bar || !as_bar || (!as && op != O_ADD))) return O_EINVAL;

    if (op == O_ADD) {
        if (hs) {
            LD *h = (LD *)calloc((size_t)m, sizeof(LD));
            if (!h) return O_EINVAL;
            for (int64_t i = 0; i < n; ++i) {
                int64_t b = idx_get(itype, inds, i);
                if (b >= 0 && b < m) h[b] = h[b] + ld_get(dtype, as, i);
            }
            for (int64_t b = 0; b < m; ++b) ld_put(dtype, hs, b, h[b], 0);
            free(h);
        }
        for (int64_t i = 0; i < n; ++i) {
            int64_t b = idx_get(itype, inds, i);
            ld_put(dtype, as_bar, i, (b >= 0 && b < m) ? ld_get(dtype, hs_bar, b) : 0.0L, flags);
        }
        return O_OK;
    }
    if (op == O_MUL) {
        LD *run = (LD *)malloc(sizeof(LD) * (size_t)m);
        LD *ls = (LD *)malloc(sizeof(LD) * (size_t)(n > 0 ? n : 1));
        int64_t *z = (int64_t *)calloc((size_t)m, sizeof(int64_t));
        if (!run || !ls || !z) { free(run); free(ls); free(z); return O_EINVAL; }
        /* forward: per-bin running product; ls_i = product of the bin's earlier elements */
        for (int64_t b = 0; b < m; ++b) run[b] = 1.0L;
        for (int64_t i = 0; i < n; ++i) {
            int64_t b = idx_get(itype, inds, i);
            if (b < 0 || b >= m) { ls[i] = 0.0L; continue; }
            LD a = ld_get(dtype, as, i);
            ls[i] = run[b];
            run[b] = run[b] * a;
            if (a == 0.0L) z[b] += 1;
        }
        if (hs) for (int64_t b = 0; b < m; ++b) ld_put(dtype, hs, b, run[b], 0);
        if (zeros) for (int64_t b = 0; b < m; ++b) zeros[b] = z[b];
        /* backward: per-bin running product of the later elements */
        for (int64_t b = 0; b < m; ++b) run[b] = 1.0L;
        for (int64_t i = n - 1; i >= 0; --i) {
            int64_t b = idx_get(itype, inds, i);
            if (b < 0 || b >= m) { ld_put(dtype, as_bar, i, 0.0L, flags); continue; }
            ld_put(dtype, as_bar, i, ld_get(dtype, hs_bar, b) * ls[i] * run[b], flags);
            run[b] = ld_get(dtype, as, i) * run[b];
        }
        free(run); free(ls); free(z);
        return O_OK;
    }
    /* MIN / MAX: the extended operator (value, first index), sequential */
    LD *best = (LD *)malloc(sizeof(LD) * (size_t)m);
    int64_t *win = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    if (!best || !win) { free(best); free(win); return O_EINVAL; }
    for (int64_t b = 0; b < m; ++b) { best[b] = op == O_MIN ? (LD)INFINITY : -(LD)INFINITY; win[b] = -1; }
    for (int64_t i = 0; i < n; ++i) {
        int64_t b = idx_get(itype, inds, i);
        if (b < 0 || b >= m) continue;
        LD v = ld_get(dtype, as, i);
        if (win[b] < 0 || (op == O_MIN ? (v < best[b]) : (v > best[b]))) { best[b] = v; win[b] = i; }
    }
    if (flags & O_ACCUMULATE) {
        for (int64_t b = 0; b < m; ++b)
            if (win[b] >= 0) ld_put(dtype, as_bar, win[b], ld_get(dtype, hs_bar, b), flags);
    } else {
        for (int64_t i = 0; i < n; ++i) {
            int64_t b = idx_get(itype, inds, i);
            int won = (b >= 0 && b < m && win[b] == i);
            ld_put(dtype, as_bar, i, won ? ld_get(dtype, hs_bar, b) : 0.0L, 0);
        }
    }
    if (hs) for (int64_t b = 0; b < m; ++b) ld_put(dtype, hs, b, best[b], 0);
    if (winners) for (int64_t b = 0; b < m; ++b) winners[b] = win[b];
    free(best); free(win);
    return O_OK;
}

/*
 * vjp of  ys = scatter xs is vs with the return sweep of
 * P:1274-1275:
 *     vs_bar += gather is ys_bar            (vs_bar[j] += ys_bar[is[j]])
 *     xs_bar  = scatter ys_bar is (replicate m 0)
 * `width` scalars per element (1 on the hot path).  Out-of-range targets are
 * skipped (R4) and their vs_bar contribution is 0.  Duplicate in-range targets
 * violate the precondition of P:1247 and return O_EDUPINDEX (outputs then
 * unspecified).  xs_bar may alias ys_bar.
 */
int oracle_vjp_scatter(int dtype, int itype, int64_t n, int64_t m, int64_t width,
                       const void *is, const void *ys_bar, void *xs_bar, void *vs_bar,
                       unsigned flags) {
    if ((dtype != O_F32 && dtype != O_F64) || (itype != O_I32 && itype != O_I64)) return O_EINVAL;
    if (n < 0 || m < 0 || width < 1) return O_EINVAL;
    if ((m > 0 && (!is || !vs_bar)) || (n > 0 && (!ys_bar || !xs_bar))) return O_EINVAL;
    unsigned char *seen = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!seen) return O_EINVAL;
    int dup = 0;
    for (int64_t j = 0; j < m; ++j) {
        int64_t t = idx_get(itype, is, j);
        if (t < 0 || t >= n) continue;
        if (seen[t]) dup = 1;
        seen[t] = 1;
    }
    /* gather first (reads ys_bar before any zeroing, so aliasing is safe) */
    for (int64_t j = 0; j < m; ++j) {
        int64_t t = idx_get(itype, is, j);
        for (int64_t k = 0; k < width; ++k) {
            LD g = (t >= 0 && t < n) ? ld_get(dtype, ys_bar, t * width + k) : 0.0L;
            ld_put(dtype, vs_bar, j * width + k, g, flags);
        }
    }
    if (xs_bar != ys_bar)
        for (int64_t i = 0; i < n * width; ++i) ld_put(dtype, xs_bar, i, ld_get(dtype, ys_bar, i), 0);
    for (int64_t j = 0; j < m; ++j) {
        int64_t t = idx_get(itype, is, j);
        if (t < 0 || t >= n) continue;
        for (int64_t k = 0; k < width; ++k) ld_put(dtype, xs_bar, t * width + k, 0.0L, 0);
    }
    free(seen);
    return dup ? O_EDUPINDEX : O_OK;
}

/*
 * k-means cost and its derivatives.
 *
 *   f(C) = sum_p min_j dist(p, j),  dist(p, j) = sum_t (p_t - c_jt)^2
 *
 * (P:1687 writes ||p - c||; reading R15 takes the SQUARED distance, the only
 * reading with the diagonal Hessian the paper relies on.)
 * Forward, literally: for every point the distance to every center, then the
 * min-reduce with the FIRST index among equal minima (strict '<' in a
 * left-to-right loop), then the +-reduce over points.
 * Return sweep with cost_bar = ybar, Eq. 3 applied statement by statement:
 *   y_p bar = ybar (reduce(+));
 *   dist(p, j) bar = y_p bar if j == a(p), else 0 (reduce(min));
 *   c_jt bar += dist(p, j) bar * 2 (c_jt - p_t)  (the map's vjp; accumulated
 *   over p in index order).
 * jvp of that vjp in the direction cdot = 1 (all ones; ybar, P fixed): the
 * tangent of c_jt bar is sum_p dist(p, j) bar * 2 * cdot_jt = 2 ybar cnt_j,
 * which is the Hessian diagonal since the Hessian is diagonal.
 * Outputs (nullable except Cbar): Cbar, H [k x d]; assign int32 [n];
 * counts int64 [k]; cost [1].  Arrays are row-major [rows x d].
 */
int oracle_kmeans(int dtype, int64_t n, int64_t k, int64_t d, const void *P, const void *C,
                  const void *cost_bar, void *Cbar, void *H, int32_t *assign, int64_t *counts,
                  void *cost) {
    if ((dtype != O_F32 && dtype != O_F64) || n < 0 || k < 1 || d < 1) return O_EINVAL;
    if ((n > 0 && !P) || !C || !cost_bar || !Cbar) return O_EINVAL;
    const LD ybar = ld_get(dtype, cost_bar, 0);
    LD *g = (LD *)calloc((size_t)(k * d), sizeof(LD));
    int64_t *cnt = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    if (!g || !cnt) { free(g); free(cnt); return O_EINVAL; }
    LD total = 0.0L;
    for (int64_t p = 0; p < n; ++p) {
        /* forward: distances and the first-index argmin */
        int64_t a = -1;
        LD best = 0.0L;
        for (int64_t j = 0; j < k; ++j) {
            LD dist = 0.0L;
            for (int64_t t = 0; t < d; ++t) {
                LD diff = ld_get(dtype, P, p * d + t) - ld_get(dtype, C, j * d + t);
                dist += diff * diff;
            }
            if (a < 0 || dist < best) { best = dist; a = j; }
        }
        total += best;
        if (assign) assign[p] = (int32_t)a;
        cnt[a] += 1;
        /* return sweep of this point: only the argmin center receives an adjoint */
        for (int64_t t = 0; t < d; ++t)
            g[a * d + t] += ybar * 2.0L * (ld_get(dtype, C, a * d + t) - ld_get(dtype, P, p * d + t));
    }
    for (int64_t j = 0; j < k; ++j) {
        for (int64_t t = 0; t < d; ++t) {
            ld_put(dtype, Cbar, j * d + t, g[j * d + t], 0);
            if (H) ld_put(dtype, H, j * d + t, 2.0L * ybar * (LD)cnt[j], 0);
        }
        if (counts) counts[j] = cnt[j];
    }
    if (cost) ld_put(dtype, cost, 0, total, 0);
    free(g);
    free(cnt);
    return O_OK;
}
