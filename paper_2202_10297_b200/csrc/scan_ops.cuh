// scan_ops.cuh — per-operator algebra of the scan adjoint (sec 5.2).
//
// For ys = scan (.) as with rs_i = rs_{i-1} (.) a_i, the
// return sweep of P:1153-1158 is the backward linear recurrence
//     rbar_{i-1} = ybar_{i-1} + J_L(rs_{i-1}, a_i)^T rbar_i
//     abar_i     = J_R(rs_{i-1}, a_i)^T rbar_i,  abar_0 = rbar_0
// with J_L = d(r (.) a)/dr and J_R = d(r (.) a)/da.  The paper solves the
// recurrence with a scan whose operator is composition of the affine maps
// X -> d + c.X (lin_o), generalised to d-vectors with c a Jacobian
// and neutral (0, I).
//
// We group each element's map so that it uses only that element's own data
// (DESIGN.md "Differences from the paper"): with H_i = J_L(rs_{i-1},a_i)^T rbar_i
// (the contribution element i passes to the left),
//     rbar_i = ybar_i + H_{i+1},   H_i = M_i(H_{i+1}),   M_i(X) = J_L^T (ybar_i + X)
// M_i is affine, X -> D + C.X with D = J_L^T ybar_i, C = J_L^T; the M_i are
// composed right to left (the same lin_o composition, re-associated), so no
// tile needs its right neighbour's element (no halo).
//
// Each op provides (all arithmetic in double, even for f32 data, reading R9):
//   Val  (primal element / prefix, W doubles)   fwd_id(), fwd(l, r) = l (.) r
//   Map  (affine map on W-vector adjoints)      map_id(), compose(outer, inner),
//        apply(M, X), constant(V) (C = 0: X -> V)
//   make_map(rs_prev, a, ybar) = M_i ;  out(rs_prev, a, g) = J_R^T g
//   pass_left(rs_prev, a, g) = J_L^T g ;  extend(T, rs_prev, a, ybar) = M_i o T
#pragma once
#include <math.h>

namespace vjpk {

#define HD __host__ __device__ __forceinline__

template <int W>
struct Vec {
    double x[W];
};

// ------------------------------------------------------------------ ADD
// r (.) a = r + a;  J_L = J_R = 1 (P:1233-1236 closed form).
struct OpAdd {
    static constexpr int W = 1;
    static constexpr bool kRevNeedsRs = false;
    static constexpr bool kFirstSpecial = false;
    using Val = Vec<1>;
    struct Map { double D; };  // X -> D + X
    static constexpr int kMapD = 1;
    HD static Val fwd_id() { return {{0.0}}; }
    HD static Val fwd(const Val &l, const Val &r) { return {{l.x[0] + r.x[0]}}; }
    HD static Map map_id() { return {0.0}; }
    HD static Map compose(const Map &o, const Map &i) { return {o.D + i.D}; }
    HD static Val apply(const Map &m, const Val &X) { return {{m.D + X.x[0]}}; }
    HD static Map constant(const Val &v) { return {v.x[0]}; }
    HD static Map make_map(const Val &, const Val &, const Val &yb) { return {yb.x[0]}; }
    HD static Val out(const Val &, const Val &, const Val &g) { return g; }
    // pass_left = J_L^T g (the contribution to the carry); extend(T) = make_map o T
    HD static Val pass_left(const Val &, const Val &, const Val &g) { return g; }
    HD static Map extend(const Map &T, const Val &, const Val &, const Val &yb) { return {yb.x[0] + T.D}; }
};

// ------------------------------------------------------------------ MUL
// r (.) a = r*a;  J_L = a, J_R = r.
struct OpMul {
    static constexpr int W = 1;
    static constexpr bool kRevNeedsRs = false;
    static constexpr bool kFirstSpecial = false;
    using Val = Vec<1>;
    struct Map { double D, C; };  // X -> D + C X
    static constexpr int kMapD = 2;
    HD static Val fwd_id() { return {{1.0}}; }
    HD static Val fwd(const Val &l, const Val &r) { return {{l.x[0] * r.x[0]}}; }
    HD static Map map_id() { return {0.0, 1.0}; }
    HD static Map compose(const Map &o, const Map &i) { return {o.D + o.C * i.D, o.C * i.C}; }
    HD static Val apply(const Map &m, const Val &X) { return {{m.D + m.C * X.x[0]}}; }
    HD static Map constant(const Val &v) { return {v.x[0], 0.0}; }
    HD static Map make_map(const Val &, const Val &a, const Val &yb) { return {a.x[0] * yb.x[0], a.x[0]}; }
    HD static Val out(const Val &rp, const Val &, const Val &g) { return {{rp.x[0] * g.x[0]}}; }
    HD static Val pass_left(const Val &, const Val &a, const Val &g) { return {{a.x[0] * g.x[0]}}; }
    HD static Map extend(const Map &T, const Val &, const Val &a, const Val &yb) {
        return {a.x[0] * (yb.x[0] + T.D), a.x[0] * T.C};
    }
};

// ------------------------------------------------------------ MIN / MAX
// r (.) a = pick-left extremum (reading R3); J_L = [left], J_R = 1 - J_L.
template <bool IsMax>
struct OpExt {
    static constexpr int W = 1;
    static constexpr bool kRevNeedsRs = true;
    static constexpr bool kFirstSpecial = true;  // abar_0 = rbar_0 even if a_0 = +-inf
    using Val = Vec<1>;
    struct Map { double D, C; };
    static constexpr int kMapD = 2;
    HD static bool left(double r, double a) { return IsMax ? (r >= a) : (r <= a); }
    HD static Val fwd_id() { return {{IsMax ? -INFINITY : INFINITY}}; }
    HD static Val fwd(const Val &l, const Val &r) { return left(l.x[0], r.x[0]) ? l : r; }
    HD static Map map_id() { return {0.0, 1.0}; }
    HD static Map compose(const Map &o, const Map &i) { return {o.D + o.C * i.D, o.C * i.C}; }
    HD static Val apply(const Map &m, const Val &X) { return {{m.D + m.C * X.x[0]}}; }
    HD static Map constant(const Val &v) { return {v.x[0], 0.0}; }
    HD static Map make_map(const Val &rp, const Val &a, const Val &yb) {
        double jl = left(rp.x[0], a.x[0]) ? 1.0 : 0.0;
        return {jl * yb.x[0], jl};
    }
    HD static Val out(const Val &rp, const Val &a, const Val &g) {
        return {{left(rp.x[0], a.x[0]) ? 0.0 : g.x[0]}};
    }
    HD static Val pass_left(const Val &rp, const Val &a, const Val &g) {
        return {{left(rp.x[0], a.x[0]) ? g.x[0] : 0.0}};
    }
    HD static Map extend(const Map &T, const Val &rp, const Val &a, const Val &yb) {
        double jl = left(rp.x[0], a.x[0]) ? 1.0 : 0.0;
        return {jl * (yb.x[0] + T.D), jl * T.C};
    }
};
using OpMin = OpExt<false>;
using OpMax = OpExt<true>;

// --------------------------------------------------------------- LINREC
// (D, C) (.) (d, c) = (d + c D, c C)  (lin_o; reading R2).
// J_L = c I;  J_R^T (gD, gC) = (gD, gD D + gC C).
struct OpLinrec {
    static constexpr int W = 2;
    static constexpr bool kRevNeedsRs = false;
    static constexpr bool kFirstSpecial = false;
    using Val = Vec<2>;
    struct Map { double D0, D1, C; };  // X -> D + C X (X a 2-vector, C scalar)
    static constexpr int kMapD = 3;
    HD static Val fwd_id() { return {{0.0, 1.0}}; }
    HD static Val fwd(const Val &l, const Val &r) { return {{r.x[0] + r.x[1] * l.x[0], r.x[1] * l.x[1]}}; }
    HD static Map map_id() { return {0.0, 0.0, 1.0}; }
    HD static Map compose(const Map &o, const Map &i) {
        return {o.D0 + o.C * i.D0, o.D1 + o.C * i.D1, o.C * i.C};
    }
    HD static Val apply(const Map &m, const Val &X) { return {{m.D0 + m.C * X.x[0], m.D1 + m.C * X.x[1]}}; }
    HD static Map constant(const Val &v) { return {v.x[0], v.x[1], 0.0}; }
    HD static Map make_map(const Val &, const Val &a, const Val &yb) {
        double c = a.x[1];
        return {c * yb.x[0], c * yb.x[1], c};
    }
    HD static Val out(const Val &rp, const Val &, const Val &g) {
        return {{g.x[0], g.x[0] * rp.x[0] + g.x[1] * rp.x[1]}};
    }
    HD static Val pass_left(const Val &, const Val &a, const Val &g) { return {{a.x[1] * g.x[0], a.x[1] * g.x[1]}}; }
    HD static Map extend(const Map &T, const Val &, const Val &a, const Val &yb) {
        double c = a.x[1];
        return {c * (yb.x[0] + T.D0), c * (yb.x[1] + T.D1), c * T.C};
    }
};

// ----------------------------------------------------------------- MAT2
// R (.) A = R . A (2x2, row-major, reading R1).
// J_L^T G = G A^T ;  J_R^T G = R^T G.   Maps act by right multiplication:
// X -> D + X C with D = ybar A^T, C = A^T; compose(o, i) = (D_o + D_i C_o, C_i C_o).
struct OpMat2 {
    static constexpr int W = 4;
    static constexpr bool kRevNeedsRs = false;
    static constexpr bool kFirstSpecial = false;
    using Val = Vec<4>;
    struct Map { double D[4], C[4]; };
    static constexpr int kMapD = 8;
    HD static Val mm(const Val &a, const Val &b) {  // a . b
        return {{a.x[0] * b.x[0] + a.x[1] * b.x[2], a.x[0] * b.x[1] + a.x[1] * b.x[3],
                 a.x[2] * b.x[0] + a.x[3] * b.x[2], a.x[2] * b.x[1] + a.x[3] * b.x[3]}};
    }
    HD static Val fwd_id() { return {{1.0, 0.0, 0.0, 1.0}}; }
    HD static Val fwd(const Val &l, const Val &r) { return mm(l, r); }
    HD static Map map_id() { return {{0.0, 0.0, 0.0, 0.0}, {1.0, 0.0, 0.0, 1.0}}; }
    HD static Map compose(const Map &o, const Map &i) {
        Val Do{{o.D[0], o.D[1], o.D[2], o.D[3]}}, Co{{o.C[0], o.C[1], o.C[2], o.C[3]}};
        Val Di{{i.D[0], i.D[1], i.D[2], i.D[3]}}, Ci{{i.C[0], i.C[1], i.C[2], i.C[3]}};
        Val DC = mm(Di, Co), CC = mm(Ci, Co);
        return {{Do.x[0] + DC.x[0], Do.x[1] + DC.x[1], Do.x[2] + DC.x[2], Do.x[3] + DC.x[3]},
                {CC.x[0], CC.x[1], CC.x[2], CC.x[3]}};
    }
    HD static Val apply(const Map &m, const Val &X) {
        Val C{{m.C[0], m.C[1], m.C[2], m.C[3]}};
        Val XC = mm(X, C);
        return {{m.D[0] + XC.x[0], m.D[1] + XC.x[1], m.D[2] + XC.x[2], m.D[3] + XC.x[3]}};
    }
    HD static Map constant(const Val &v) { return {{v.x[0], v.x[1], v.x[2], v.x[3]}, {0.0, 0.0, 0.0, 0.0}}; }
    HD static Map make_map(const Val &, const Val &a, const Val &yb) {
        Val At{{a.x[0], a.x[2], a.x[1], a.x[3]}};
        Val D = mm(yb, At);
        return {{D.x[0], D.x[1], D.x[2], D.x[3]}, {At.x[0], At.x[1], At.x[2], At.x[3]}};
    }
    HD static Val out(const Val &rp, const Val &, const Val &g) {
        Val Rt{{rp.x[0], rp.x[2], rp.x[1], rp.x[3]}};
        return mm(Rt, g);
    }
    HD static Val pass_left(const Val &, const Val &a, const Val &g) {  // g A^T
        Val At{{a.x[0], a.x[2], a.x[1], a.x[3]}};
        return mm(g, At);
    }
    HD static Map extend(const Map &T, const Val &, const Val &a, const Val &yb) {
        // (X -> (yb + D + X C) A^T): D' = (yb + D) A^T, C' = C A^T
        Val At{{a.x[0], a.x[2], a.x[1], a.x[3]}};
        Val s{{yb.x[0] + T.D[0], yb.x[1] + T.D[1], yb.x[2] + T.D[2], yb.x[3] + T.D[3]}};
        Val C{{T.C[0], T.C[1], T.C[2], T.C[3]}};
        Val D2 = mm(s, At), C2 = mm(C, At);
        return {{D2.x[0], D2.x[1], D2.x[2], D2.x[3]}, {C2.x[0], C2.x[1], C2.x[2], C2.x[3]}};
    }
};

// Map <-> flat doubles (workspace records, shuffles)
template <class Op>
HD void map_to(const typename Op::Map &m, double *d) {
    const double *s = reinterpret_cast<const double *>(&m);
#pragma unroll
    for (int k = 0; k < Op::kMapD; ++k) d[k] = s[k];
}
template <class Op>
HD typename Op::Map map_from(const double *d) {
    typename Op::Map m;
    double *s = reinterpret_cast<double *>(&m);
#pragma unroll
    for (int k = 0; k < Op::kMapD; ++k) s[k] = d[k];
    return m;
}

// Shard carries for the multi-GPU finish: record r = [fwd aggregate
// (W doubles) | reverse map aggregate (kMapD doubles)].  The forward carry of
// rank r is rec_0.F (.) ... (.) rec_{r-1}.F; the reverse carry entering its last
// element is (rec_{r+1}.M o ... o rec_{world-1}.M)(0).
template <class Op>
HD void shard_carries(const double *gathered, int rank, int world, typename Op::Val &F,
                      typename Op::Val &Hin) {
    constexpr int R = Op::W + Op::kMapD;
    F = Op::fwd_id();
    for (int q = 0; q < rank; ++q) {
        typename Op::Val v;
        for (int k = 0; k < Op::W; ++k) v.x[k] = gathered[q * R + k];
        F = Op::fwd(F, v);
    }
    typename Op::Map M = Op::map_id();
    for (int q = rank + 1; q < world; ++q) M = Op::compose(M, map_from<Op>(gathered + q * R + Op::W));
    typename Op::Val z;
    for (int k = 0; k < Op::W; ++k) z.x[k] = 0.0;
    Hin = Op::apply(M, z);
}

#undef HD
}  // namespace vjpk
