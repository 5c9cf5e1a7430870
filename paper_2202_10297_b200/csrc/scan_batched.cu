// scan_batched.cu — vjp of a VECTORISED scan:
//
//     ys = scan (map (.)) (replicate w e) xs,   xs [n][w] (w components per element)
//
// The paper turns it into a regular-segmented scan by the transpose rule
// (transpose |> map (scan (.) e) |> transpose): w independent
// scans along n.  Here the transpose is a thread mapping, not a data movement:
// a thread owns one COLUMN j of a chunk of rows and walks its rows in
// registers (a warp reads 32 consecutive columns of a row: coalesced), so the
// column-wise scan needs no cross-thread combining inside a chunk.
//
//   K_R  scan_bat_reduce : per (chunk, column) the forward aggregate F (the
//        re-executed primal) and the composed reverse map M (the
//        lin_o composition of P:1196-1198 with the per-element grouping of
//        scan_ops.cuh), one ascending pass; also every tile's exclusive
//        forward prefix inside the chunk.
//   K_S  scan_bat_carries : per column, a block-wide scan over the chunk
//        records -> forward prefix entering each chunk and reverse carry
//        entering it from the right.
//   K_C  scan_bat_apply : per (chunk, column), tiles right to left: registers
//        hold the tile's rows, the primal is re-executed from the tile prefix
//        (tape-free), outputs run right to left:
//        rbar_i = ybar_i + H, abar_i = J_R^T rbar_i, H = J_L^T rbar_i.
// ADD, MUL, LINREC, MAT2 (carry-independent reverse maps) and MIN/MAX, whose
// reverse maps need the forward carry: forward records, forward prefixes,
// maps rebuilt with the true rs (scan_bat_maps_rs), then the carries.
#include <cstdint>
#include <type_traits>

#include "scan_kernels.cuh"

namespace vjpk {

constexpr int kBatThreads = 128;

template <class Op>
struct BatGeo {
    static constexpr int TR = 16 / Op::W;  // rows per register tile (16 scalars of each array)
};

struct BatParams {
    int64_t n, w;
    int64_t C, TPC;  // chunks, tiles per chunk (chunk = TPC * TR rows)
    int32_t CW, CPB; // columns per column group (power of two), chunk slots per CTA
    const void *as;
    const void *ys_bar;
    void *as_bar;
    double *rec;     // [w][C][W + MD] (a column's chunk records contiguous for scan_bat_carries)
    double *tileP;   // [C * TPC][w][W] exclusive forward prefix of each tile inside its chunk
    double *carry;   // [w][C][2W]  {forward prefix entering the chunk, reverse carry entering it}
    int32_t acc;
};

template <class T, int W>
__device__ __forceinline__ Vec<W> bat_ld(const T *p) {
    Vec<W> v;
#pragma unroll
    for (int k = 0; k < W; ++k) v.x[k] = (double)p[k];
    return v;
}

// thread -> (chunk, column); false if out of range
__device__ __forceinline__ bool bat_coord(const BatParams &p, int64_t &c, int64_t &j) {
    const int t = threadIdx.x;
    j = (int64_t)blockIdx.x * p.CW + (t % p.CW);
    c = (int64_t)blockIdx.y * p.CPB + (t / p.CW);
    return j < p.w && c < p.C;
}

template <class Op, class T, bool FWD, bool MAPS = true>
__global__ void __launch_bounds__(kBatThreads) scan_bat_reduce(const BatParams p) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD, TR = BatGeo<Op>::TR;
    int64_t c, j;
    if (!bat_coord(p, c, j)) return;
    const T *as = static_cast<const T *>(p.as);
    const T *yb = static_cast<const T *>(p.ys_bar);
    const int64_t r0 = c * p.TPC * TR;
    V F = Op::fwd_id();
    M Mc = Op::map_id();
    for (int64_t k = 0; k < p.TPC; ++k) {
        const int64_t rt = r0 + k * TR;
        if (FWD) {
#pragma unroll
            for (int q = 0; q < W; ++q) p.tileP[((c * p.TPC + k) * p.w + j) * W + q] = F.x[q];
        }
        V a[TR], y[TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            const bool in = rt + r < p.n;
            const int64_t e = ((rt + r) * p.w + j) * W;
            a[r] = (FWD && in) ? bat_ld<T, W>(as + e) : Op::fwd_id();
            if (in) {
                y[r] = bat_ld<T, W>(yb + e);
            } else {
#pragma unroll
                for (int q = 0; q < W; ++q) y[r].x[q] = 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            if (rt + r < p.n) {
                if (FWD) F = Op::fwd(F, a[r]);
                if (MAPS) Mc = Op::compose(Mc, Op::make_map(Op::fwd_id(), a[r], y[r]));
            }
        }
    }
    double rec[W + MD];
#pragma unroll
    for (int q = 0; q < W; ++q) rec[q] = F.x[q];
    map_to<Op>(Mc, rec + W);
    double *dst = p.rec + (j * p.C + c) * (W + MD);  // column-major: a column's chunk records contiguous
#pragma unroll
    for (int q = 0; q < W + MD; ++q) dst[q] = rec[q];
}

// rs-dependent operators (MIN/MAX): the chunk's reverse map with the TRUE rs,
// walking the rows from the chunk's forward prefix (carry[..][0..W), written
// by a first scan_bat_carries); only the M part of the record is rewritten
template <class Op, class T>
__global__ void __launch_bounds__(kBatThreads) scan_bat_maps_rs(const BatParams p) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD, TR = BatGeo<Op>::TR;
    int64_t c, j;
    if (!bat_coord(p, c, j)) return;
    const T *as = static_cast<const T *>(p.as);
    const T *yb = static_cast<const T *>(p.ys_bar);
    const double *cr = p.carry + (j * p.C + c) * 2 * W;
    V rs;
#pragma unroll
    for (int q = 0; q < W; ++q) rs.x[q] = cr[q];
    M Mc = Op::map_id();
    const int64_t r0 = c * p.TPC * TR, r1 = r0 + p.TPC * TR < p.n ? r0 + p.TPC * TR : p.n;
    for (int64_t rt = r0; rt < r1; rt += TR) {
        V a[TR], y[TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            if (rt + r < r1) {
                const int64_t e = ((rt + r) * p.w + j) * W;
                a[r] = bat_ld<T, W>(as + e);
                y[r] = bat_ld<T, W>(yb + e);
            }
        }
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            if (rt + r < r1) {
                Mc = Op::compose(Mc, Op::make_map(rs, a[r], y[r]));
                rs = Op::fwd(rs, a[r]);
            }
        }
    }
    double rec[MD];
    map_to<Op>(Mc, rec);
    double *dst = p.rec + (j * p.C + c) * (W + MD) + W;
#pragma unroll
    for (int q = 0; q < MD; ++q) dst[q] = rec[q];
}

// one CTA of 1024 threads per column: exclusive scans over the C chunk
// records (~SMs x 2048 / w of them: 1024 threads keep each thread's serial
// walk short — 256 threads left it latency bound: 96 us for LINREC w = 32)
constexpr int kBatCarryThreads = 1024;
template <class Op>
__global__ void __launch_bounds__(kBatCarryThreads) scan_bat_carries(const BatParams p) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD, R = W + MD, NW = kBatCarryThreads / 32;
    __shared__ V vs[NW + 1];
    __shared__ M ms[NW + 1];
    const int64_t j = blockIdx.x;
    const int t = threadIdx.x;
    const int64_t per = (p.C + kBatCarryThreads - 1) / kBatCarryThreads, c0 = t * per,
                  c1 = c0 + per < p.C ? c0 + per : p.C;
    V f = Op::fwd_id();
    M m = Op::map_id();
    for (int64_t c = c0; c < c1; ++c) {
        const double *r = p.rec + (j * p.C + c) * R;
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = r[q];
        f = Op::fwd(f, v);
        m = Op::compose(m, map_from<Op>(r + W));
    }
    V ftot;
    M mtot;
    V fpre = block_excl_fwd<Op, NW>(f, vs, ftot);   // chunks before this thread's range
    M mpost = block_excl_rev<Op, NW>(m, ms, mtot);  // chunks after it
    V x;
#pragma unroll
    for (int q = 0; q < W; ++q) x.x[q] = 0.0;
    x = Op::apply(mpost, x);  // reverse carry entering the thread's last chunk from the right
    // forward prefixes ascending, reverse carries descending
    for (int64_t c = c0; c < c1; ++c) {
        double *cr = p.carry + (j * p.C + c) * 2 * W;
#pragma unroll
        for (int q = 0; q < W; ++q) cr[q] = fpre.x[q];
        const double *r = p.rec + (j * p.C + c) * R;
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = r[q];
        fpre = Op::fwd(fpre, v);
    }
    for (int64_t c = c1 - 1; c >= c0; --c) {
        double *cr = p.carry + (j * p.C + c) * 2 * W;
#pragma unroll
        for (int q = 0; q < W; ++q) cr[W + q] = x.x[q];
        x = Op::apply(map_from<Op>(p.rec + (j * p.C + c) * R + W), x);
    }
}

template <class Op, class T, bool FWD, bool ACC>
__global__ void __launch_bounds__(kBatThreads) scan_bat_apply(const BatParams p) {
    using V = typename Op::Val;
    constexpr int W = Op::W, TR = BatGeo<Op>::TR;
    int64_t c, j;
    if (!bat_coord(p, c, j)) return;
    const T *as = static_cast<const T *>(p.as);
    const T *yb = static_cast<const T *>(p.ys_bar);
    T *ab = static_cast<T *>(p.as_bar);
    const double *cr = p.carry + (j * p.C + c) * 2 * W;
    V F0, X;
#pragma unroll
    for (int q = 0; q < W; ++q) {
        F0.x[q] = cr[q];
        X.x[q] = cr[W + q];
    }
    const int64_t r0 = c * p.TPC * TR;
    for (int64_t k = p.TPC - 1; k >= 0; --k) {
        const int64_t rt = r0 + k * TR;
        if (rt >= p.n) continue;
        V a[TR], y[TR], rsp[TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
            const bool in = rt + r < p.n;
            const int64_t e = ((rt + r) * p.w + j) * W;
            a[r] = (FWD && in) ? bat_ld<T, W>(as + e) : Op::fwd_id();
            if (in) {
                y[r] = bat_ld<T, W>(yb + e);
            } else {
#pragma unroll
                for (int q = 0; q < W; ++q) y[r].x[q] = 0.0;
            }
        }
        if (FWD) {
            V rs = F0;
            V tp;
#pragma unroll
            for (int q = 0; q < W; ++q) tp.x[q] = p.tileP[((c * p.TPC + k) * p.w + j) * W + q];
            rs = Op::fwd(rs, tp);
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                rsp[r] = rs;
                rs = Op::fwd(rs, a[r]);
            }
        } else {
#pragma unroll
            for (int r = 0; r < TR; ++r) rsp[r] = Op::fwd_id();
        }
#pragma unroll
        for (int r = TR - 1; r >= 0; --r) {
            if (rt + r >= p.n) continue;
            V g;
#pragma unroll
            for (int q = 0; q < W; ++q) g.x[q] = y[r].x[q] + X.x[q];  // rbar_i = ybar_i + H_{i+1}
            V o = Op::out(rsp[r], a[r], g);
            if (Op::kFirstSpecial && rt + r == 0) o = g;  // abar_0 = rbar_0, whatever a_0 is
            X = Op::pass_left(rsp[r], a[r], g);
            T *dst = ab + ((rt + r) * p.w + j) * W;
#pragma unroll
            for (int q = 0; q < W; ++q) dst[q] = ACC ? (T)((double)dst[q] + o.x[q]) : (T)o.x[q];
        }
    }
}

}  // namespace vjpk

namespace {
using namespace vjph;

struct BatLayout {
    int64_t C, TPC;
    int32_t CW, CPB;
    size_t rec, tileP, carry, total;
};

template <class Op>
BatLayout bat_layout(int64_t n, int64_t w) {
    constexpr int W = Op::W, MD = Op::kMapD, TR = vjpk::BatGeo<Op>::TR;
    BatLayout L{};
    const int64_t tiles = n > 0 ? (n + TR - 1) / TR : 0;
    // enough (chunk, column) threads to fill the GPU: ~ SMs x 2048
    const int64_t want = (int64_t)sm_count() * 2048;
    int64_t C = (want + w - 1) / w;
    if (C > tiles) C = tiles;
    if (C < 1) C = 1;
    L.TPC = tiles > 0 ? (tiles + C - 1) / C : 1;
    L.C = tiles > 0 ? (tiles + L.TPC - 1) / L.TPC : 1;
    int cw = 1;
    while (cw < w && cw < vjpk::kBatThreads) cw <<= 1;
    L.CW = cw;
    L.CPB = vjpk::kBatThreads / cw;
    size_t off = 0;
    L.rec = off; off += align256((size_t)L.C * w * (W + MD) * 8);
    L.tileP = off; off += align256((size_t)L.C * L.TPC * w * W * 8);
    L.carry = off; off += align256((size_t)L.C * w * 2 * W * 8);
    L.total = off;
    return L;
}

template <class Op, class T>
vjp_status bat_run(int64_t n, int64_t w, const void *as, const void *yb, void *ab, void *ws, cudaStream_t s,
                   unsigned flags) {
    BatLayout L = bat_layout<Op>(n, w);
    vjpk::BatParams p{};
    p.n = n;
    p.w = w;
    p.C = L.C;
    p.TPC = L.TPC;
    p.CW = L.CW;
    p.CPB = L.CPB;
    p.as = as;
    p.ys_bar = yb;
    p.as_bar = ab;
    unsigned char *b = static_cast<unsigned char *>(ws);
    p.rec = reinterpret_cast<double *>(b + L.rec);
    p.tileP = reinterpret_cast<double *>(b + L.tileP);
    p.carry = reinterpret_cast<double *>(b + L.carry);
    p.acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    constexpr bool FWD = !std::is_same<Op, vjpk::OpAdd>::value;
    const dim3 grid((unsigned)((w + L.CW - 1) / L.CW), (unsigned)((L.C + L.CPB - 1) / L.CPB));
    if (grid.y > 65535u) return VJP_EUNSUPPORTED;
    if constexpr (Op::kRevNeedsRs) {
        // MIN/MAX: forward records -> forward prefixes -> maps with the true rs
        // -> carries again (forward prefixes recomputed identically, reverse now valid)
        vjpk::scan_bat_reduce<Op, T, true, false><<<grid, vjpk::kBatThreads, 0, s>>>(p);
        vjpk::scan_bat_carries<Op><<<(unsigned)w, vjpk::kBatCarryThreads, 0, s>>>(p);
        vjpk::scan_bat_maps_rs<Op, T><<<grid, vjpk::kBatThreads, 0, s>>>(p);
        count_launch(2);
    } else {
        vjpk::scan_bat_reduce<Op, T, FWD><<<grid, vjpk::kBatThreads, 0, s>>>(p);
    }
    vjpk::scan_bat_carries<Op><<<(unsigned)w, vjpk::kBatCarryThreads, 0, s>>>(p);
    if (p.acc)
        vjpk::scan_bat_apply<Op, T, FWD, true><<<grid, vjpk::kBatThreads, 0, s>>>(p);
    else
        vjpk::scan_bat_apply<Op, T, FWD, false><<<grid, vjpk::kBatThreads, 0, s>>>(p);
    count_launch(3);
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class Op>
size_t bat_ws(int64_t n, int64_t w) { return bat_layout<Op>(n, w).total; }
}  // namespace

extern "C" {

size_t vjp_scan_batched_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t width) {
    if ((dtype != VJP_F32 && dtype != VJP_F64) || n < 0 || width < 1) return 0;
    switch (op) {
    case VJP_ADD: return bat_ws<vjpk::OpAdd>(n, width);
    case VJP_MUL: return bat_ws<vjpk::OpMul>(n, width);
    case VJP_LINREC: return bat_ws<vjpk::OpLinrec>(n, width);
    case VJP_MAT2: return bat_ws<vjpk::OpMat2>(n, width);
    case VJP_MIN: return bat_ws<vjpk::OpMin>(n, width);
    case VJP_MAX: return bat_ws<vjpk::OpMax>(n, width);
    default: return 0;
    }
}

vjp_status vjp_scan_batched(vjp_op op, vjp_dtype dtype, int64_t n, int64_t width, const void *as,
                            const void *ys_bar, void *as_bar, void *ws, size_t ws_bytes, vjp_stream_t stream,
                            unsigned flags) {
    VJP_NVTX("vjp_scan_batched");
    if ((dtype != VJP_F32 && dtype != VJP_F64) || n < 0 || width < 1) return VJP_EINVAL;
    if (op < VJP_ADD || op > VJP_MAT2) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    if (!ys_bar || !as_bar || (op != VJP_ADD && !as)) return VJP_EINVAL;
    if (as_bar == ys_bar || (as && as_bar == as)) return VJP_EINVAL;
    const size_t es = dtype == VJP_F64 ? 8 : 4;
    const void *al[] = {as, ys_bar, as_bar};
    for (const void *q : al)
        if (q && (reinterpret_cast<uintptr_t>(q) % es) != 0) return VJP_EALIGN;
    const size_t need = vjp_scan_batched_workspace_bytes(op, dtype, n, width);
    if (ws_bytes < need || !ws || !aligned16(ws)) return VJP_EWORKSPACE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const bool f64 = dtype == VJP_F64;
    switch (op) {
    case VJP_ADD:
        return f64 ? bat_run<vjpk::OpAdd, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpAdd, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    case VJP_MUL:
        return f64 ? bat_run<vjpk::OpMul, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpMul, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    case VJP_LINREC:
        return f64 ? bat_run<vjpk::OpLinrec, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpLinrec, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    case VJP_MIN:
        return f64 ? bat_run<vjpk::OpMin, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpMin, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    case VJP_MAX:
        return f64 ? bat_run<vjpk::OpMax, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpMax, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    default:
        return f64 ? bat_run<vjpk::OpMat2, double>(n, width, as, ys_bar, as_bar, ws, s, flags)
                   : bat_run<vjpk::OpMat2, float>(n, width, as, ys_bar, as_bar, ws, s, flags);
    }
}

}  // extern "C"
