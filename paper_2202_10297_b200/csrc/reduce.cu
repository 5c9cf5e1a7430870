// reduce.cu — vjp_reduce (sec 5.1) for sm_100a.
//
// Forward sweep (P:1055-1058 for *, P:1067-1071 for min/max): one streaming
// map-reduce kernel (grid-stride, 128-bit loads, warp-shuffle + shared-memory
// block reduction, per-CTA partials, the last CTA combines the partials in
// CTA order -> deterministic) producing a 32-byte record:
//   ADD      {sum}
//   MUL      {p = product of the NONZERO elements (f64), z = #zeros, i0 = first zero}
//   MIN/MAX  {y, i_y = FIRST index reaching the extremum}
// Return sweep: one streaming map kernel writing as_bar by the special-case
// rules.  Multi-GPU: the records of
// all shards are combined in rank order in the return kernel's prologue.
#include <cfloat>

#include "common.cuh"

namespace vjph {  // scan_abi.cu: the general reduce rule through the chunked scan kernels
size_t reduce_general_ws(vjp_op op, vjp_dtype dtype, int64_t n);
vjp_status reduce_general(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                          void *y, void *ws, size_t ws_bytes, cudaStream_t stream, unsigned flags);
}  // namespace vjph

namespace vjpk {

struct RRec {     // 32 bytes, also the multi-GPU exchange record
    double a;     // sum | p | extremum
    int64_t b;    // - | z | index
    int64_t c;    // - | i0 | -
    int64_t pad;
};

constexpr int kRThreads = 256;
constexpr int64_t kNoIdx = INT64_MAX;

template <int OP>
__host__ __device__ __forceinline__ RRec rrec_id() {
    RRec r{};
    if (OP == VJP_ADD) { r.a = 0.0; }
    if (OP == VJP_MUL) { r.a = 1.0; r.b = 0; r.c = kNoIdx; }
    if (OP == VJP_MIN) { r.a = INFINITY; r.b = kNoIdx; }
    if (OP == VJP_MAX) { r.a = -INFINITY; r.b = kNoIdx; }
    return r;
}

// combine two partial states.  MIN/MAX: IEEE compare (-0.0 ties +0.0), ties go
// to the LOWER index ("(first) index") — commutative and associative.
template <int OP>
__host__ __device__ __forceinline__ RRec rrec_combine(const RRec &x, const RRec &y) {
    RRec r = x;
    if (OP == VJP_ADD) r.a = x.a + y.a;
    if (OP == VJP_MUL) {
        r.a = x.a * y.a;
        r.b = x.b + y.b;
        r.c = x.c < y.c ? x.c : y.c;
    }
    if (OP == VJP_MIN || OP == VJP_MAX) {
        bool take_y = (OP == VJP_MIN) ? (y.a < x.a) : (y.a > x.a);
        if (y.a == x.a) take_y = y.b < x.b;
        if (take_y) r = y;
    }
    return r;
}

template <int OP>
__global__ void reduce_id_record(RRec *r) {
    if (threadIdx.x == 0) *r = rrec_id<OP>();
}

template <int OP>
__device__ __forceinline__ void rrec_add(RRec &r, double x, int64_t idx) {
    if (OP == VJP_ADD) r.a += x;
    if (OP == VJP_MUL) {
        if (x == 0.0) {  // -0.0 counts as a zero
            r.b += 1;
            if (idx < r.c) r.c = idx;
        } else {
            r.a *= x;
        }
    }
    if (OP == VJP_MIN || OP == VJP_MAX) {
        bool take = (OP == VJP_MIN) ? (x < r.a) : (x > r.a);
        if (x == r.a && idx < r.b) take = true;
        if (take) { r.a = x; r.b = idx; }
    }
}

template <int OP>
__device__ __forceinline__ RRec rrec_shfl_xor(const RRec &r, int m) {
    RRec o;
    o.a = __shfl_xor_sync(0xffffffffu, r.a, m);
    o.b = __shfl_xor_sync(0xffffffffu, r.b, m);
    o.c = __shfl_xor_sync(0xffffffffu, r.c, m);
    o.pad = 0;
    return o;
}

template <int OP>
__device__ __forceinline__ RRec block_rrec(RRec r, RRec *scr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) r = rrec_combine<OP>(r, rrec_shfl_xor<OP>(r, m));
    if (lane == 0) scr[warp] = r;
    __syncthreads();
    RRec t = scr[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = rrec_combine<OP>(t, scr[w]);
    __syncthreads();
    return t;
}

template <class T>
struct Vec16;
template <>
struct Vec16<float> {
    static constexpr int N = 4;
    using V = float4;
    __device__ static __forceinline__ void get(const V &v, double *o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
    __device__ static __forceinline__ V make(const double *o) {
        return make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
    }
};
template <>
struct Vec16<double> {
    static constexpr int N = 2;
    using V = double2;
    __device__ static __forceinline__ void get(const V &v, double *o) { o[0] = v.x; o[1] = v.y; }
    __device__ static __forceinline__ V make(const double *o) { return make_double2(o[0], o[1]); }
};

// ---------------------------------------------------------------- forward
template <class T, int OP>
__global__ void __launch_bounds__(kRThreads) reduce_fwd(const T *__restrict__ as, int64_t n, int64_t goff,
                                                        RRec *partials, uint32_t *counter, RRec *out) {
    using VV = Vec16<T>;
    __shared__ RRec scr[kRThreads / 32];
    __shared__ int is_last;
    RRec r = rrec_id<OP>();
    const int64_t nv = n / VV::N;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const typename VV::V *av = reinterpret_cast<const typename VV::V *>(as);
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // 4 independent 16-byte loads in flight per thread, 4 independent
    // accumulators (no serial dependency chain across the vectors)
    {
        RRec ru[4] = {rrec_id<OP>(), rrec_id<OP>(), rrec_id<OP>(), rrec_id<OP>()};
        for (; j + 3 * stride < nv; j += 4 * stride) {
            typename VV::V v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(av + j + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double x[VV::N];
                VV::get(v[u], x);
#pragma unroll
                for (int q = 0; q < VV::N; ++q) rrec_add<OP>(ru[u], x[q], goff + (j + u * stride) * VV::N + q);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) r = rrec_combine<OP>(r, ru[u]);
    }
    for (; j < nv; j += stride) {
        double x[VV::N];
        VV::get(__ldcs(av + j), x);
#pragma unroll
        for (int q = 0; q < VV::N; ++q) rrec_add<OP>(r, x[q], goff + j * VV::N + q);
    }
    if (blockIdx.x == 0) {  // scalar tail
        for (int64_t e = nv * VV::N + threadIdx.x; e < n; e += blockDim.x) rrec_add<OP>(r, (double)as[e], goff + e);
    }
    RRec b = block_rrec<OP>(r, scr);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = b;
        __threadfence();
        is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        // fixed-order combination of the per-CTA partials (deterministic)
        RRec t = rrec_id<OP>();
        for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
            RRec q;
            q.a = __ldcg(&partials[k].a);
            q.b = __ldcg(reinterpret_cast<const long long *>(&partials[k].b));
            q.c = __ldcg(reinterpret_cast<const long long *>(&partials[k].c));
            q.pad = 0;
            t = rrec_combine<OP>(t, q);
        }
        t = block_rrec<OP>(t, scr);
        if (threadIdx.x == 0) {
            *out = t;
            *counter = 0u;
        }
    }
}

// ----------------------------------------------------------------- return
struct RBwd {
    int64_t n, goff;
    int32_t world, acc;
    const RRec *recs;  // world records, rank order
    const void *ybar;  // device scalar of T
    void *y;           // nullable
    int64_t *arg;      // nullable
};

template <int OP>
__device__ __forceinline__ RRec combine_recs(const RRec *recs, int world) {
    if (!recs) return rrec_id<OP>();  // ADD without a forward sweep
    RRec t = recs[0];
    for (int k = 1; k < world; ++k) t = rrec_combine<OP>(t, recs[k]);
    return t;
}

template <class T, int OP>
__global__ void __launch_bounds__(kRThreads) reduce_bwd(const T *__restrict__ as, T *__restrict__ ab, RBwd p) {
    using VV = Vec16<T>;
    const RRec st = combine_recs<OP>(p.recs, p.world);
    const double yb = (double)*static_cast<const T *>(p.ybar);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (p.y) {
            double y = st.a;
            if (OP == VJP_MUL && st.b > 0) y = 0.0;
            *static_cast<T *>(p.y) = (T)y;
        }
        if (p.arg) {
            int64_t a = -1;
            if (OP == VJP_MUL) a = st.b > 0 ? st.c : -1;
            if (OP == VJP_MIN || OP == VJP_MAX) a = st.b == kNoIdx ? -1 : st.b;
            *p.arg = a;
        }
    }
    // single-point updates: MIN/MAX, and MUL with exactly one zero
    int64_t point = -1;
    double pval = 0.0;
    if (OP == VJP_MIN || OP == VJP_MAX) { point = st.b; pval = yb; }
    if (OP == VJP_MUL && st.b == 1) { point = st.c; pval = yb * st.a; }  // reading R8: product of the nonzeros
    const bool sparse = (OP == VJP_MIN || OP == VJP_MAX || (OP == VJP_MUL && st.b >= 1));
    if (p.acc && sparse) {
        // ACCUMULATE: touch only the documented element
        if (blockIdx.x == 0 && threadIdx.x == 0 && point != kNoIdx && point >= p.goff && point < p.goff + p.n &&
            !(OP == VJP_MUL && st.b >= 2)) {
            T *d = ab + (point - p.goff);
            *d = (T)((double)*d + pval);
        }
        return;
    }
    const double q = yb * st.a;  // MUL, z = 0: ybar * p / a_i  (P:1043-1046 with y/a_i = p/a_i)
    const int64_t nv = p.n / VV::N;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const typename VV::V *av = reinterpret_cast<const typename VV::V *>(as);
    typename VV::V *bv = reinterpret_cast<typename VV::V *>(ab);
    auto value = [&](double a, int64_t gi, double old) -> double {
        double v;
        if (OP == VJP_ADD) v = yb;
        else if (OP == VJP_MUL) v = (st.b == 0) ? q / a : (gi == point && st.b == 1 ? pval : 0.0);
        else v = (gi == point) ? pval : 0.0;
        return p.acc ? old + v : v;
    };
    const bool need_a = (OP == VJP_MUL && st.b == 0);
    if (!p.acc) {
        // overwrite mode: 4 independent 16-byte vectors per thread per iteration
        int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        // f32 data: the quotient is rounded to f32 anyway, so divide in f32 when
        // q = ybar * p is a normal f32 (one extra f32 rounding: <= 1.5 ulp f32,
        // far inside 1e-4); the f64 division made this loop compute bound
        const bool f32div = sizeof(T) == 4 && fabs(q) < 1e37 && fabs(q) > 1e-37;
        if (need_a && f32div) {
            const float qf = (float)q;
            for (; j + 3 * stride < nv; j += 4 * stride) {
                typename VV::V v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcs(av + j + u * stride);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    double a[VV::N], r[VV::N];
                    VV::get(v[u], a);
#pragma unroll
                    for (int q2 = 0; q2 < VV::N; ++q2) r[q2] = (double)(qf / (float)a[q2]);
                    __stcs(bv + j + u * stride, VV::make(r));
                }
            }
        } else if (need_a) {  // MUL, no zero: as_bar_i = ybar * p / a_i
            for (; j + 3 * stride < nv; j += 4 * stride) {
                typename VV::V v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcs(av + j + u * stride);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    double a[VV::N], r[VV::N];
                    VV::get(v[u], a);
#pragma unroll
                    for (int q2 = 0; q2 < VV::N; ++q2) r[q2] = q / a[q2];
                    __stcs(bv + j + u * stride, VV::make(r));
                }
            }
        } else {  // ADD broadcast, or zeros with at most one point value (sparse cases)
            const int64_t pv = (point != kNoIdx && point >= p.goff && point < p.goff + p.n) ? (point - p.goff) / VV::N : -1;
            double fill = (OP == VJP_ADD) ? yb : 0.0;
            double f[VV::N];
#pragma unroll
            for (int q2 = 0; q2 < VV::N; ++q2) f[q2] = fill;
            const typename VV::V fv = VV::make(f);
            for (; j + 3 * stride < nv; j += 4 * stride) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t jj = j + u * stride;
                    if (jj == pv) {
                        double r[VV::N];
#pragma unroll
                        for (int q2 = 0; q2 < VV::N; ++q2) r[q2] = value(0.0, p.goff + jj * VV::N + q2, 0.0);
                        __stcs(bv + jj, VV::make(r));
                    } else {
                        __stcs(bv + jj, fv);
                    }
                }
            }
        }
        // remainder vectors: generic path below
        for (; j < nv; j += stride) {
            double a[VV::N] = {}, r[VV::N];
            if (need_a) VV::get(__ldcs(av + j), a);
#pragma unroll
            for (int q2 = 0; q2 < VV::N; ++q2) r[q2] = value(a[q2], p.goff + j * VV::N + q2, 0.0);
            __stcs(bv + j, VV::make(r));
        }
        if (blockIdx.x == 0) {
            for (int64_t e = nv * VV::N + threadIdx.x; e < p.n; e += blockDim.x) {
                double a = need_a ? (double)as[e] : 0.0;
                ab[e] = (T)value(a, p.goff + e, 0.0);
            }
        }
        return;
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += stride) {
        double a[VV::N] = {}, o[VV::N] = {}, r[VV::N];
        if (need_a) VV::get(__ldcs(av + j), a);
        if (p.acc) VV::get(bv[j], o);
#pragma unroll
        for (int q2 = 0; q2 < VV::N; ++q2) r[q2] = value(a[q2], p.goff + j * VV::N + q2, o[q2]);
        __stcs(bv + j, VV::make(r));
    }
    if (blockIdx.x == 0) {
        for (int64_t e = nv * VV::N + threadIdx.x; e < p.n; e += blockDim.x) {
            double a = need_a ? (double)as[e] : 0.0;
            double o = p.acc ? (double)ab[e] : 0.0;
            ab[e] = (T)value(a, p.goff + e, o);
        }
    }
}

}  // namespace vjpk

// =============================================================================
// host side
// =============================================================================
namespace {
using namespace vjpk;

int reduce_grid() { return vjph::sm_count() * 4; }

struct RLayout {
    size_t partials, counter, final_rec, total;
};
RLayout rlayout() {
    RLayout L{};
    size_t off = 0;
    L.partials = off; off += vjph::align256(sizeof(RRec) * 4096);
    L.counter = off; off += 256;
    L.final_rec = off; off += 256;
    L.total = off;
    return L;
}

bool op_ok(vjp_op op) { return op == VJP_ADD || op == VJP_MUL || op == VJP_MIN || op == VJP_MAX; }
bool dt_ok(vjp_dtype d) { return d == VJP_F32 || d == VJP_F64; }

template <class T, int OP>
vjp_status fwd_launch(const void *as, int64_t n, int64_t goff, void *ws, RRec *out, cudaStream_t s) {
    RLayout L = rlayout();
    unsigned char *w = static_cast<unsigned char *>(ws);
    uint32_t *counter = reinterpret_cast<uint32_t *>(w + L.counter);
    if (cudaMemsetAsync(counter, 0, 4, s) != cudaSuccess) return VJP_ECUDA;
    int64_t nv = n / Vec16<T>::N;
    int64_t g = (nv + kRThreads - 1) / kRThreads;
    int grid = (int)(g < 1 ? 1 : (g < reduce_grid() ? g : reduce_grid()));
    reduce_fwd<T, OP><<<grid, kRThreads, 0, s>>>(static_cast<const T *>(as), n, goff,
                                                 reinterpret_cast<RRec *>(w + L.partials), counter, out);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class T, int OP>
vjp_status bwd_launch(const void *as, void *ab, const RBwd &p, cudaStream_t s) {
    int64_t nv = p.n / Vec16<T>::N;
    int64_t g = (nv + kRThreads - 1) / kRThreads;
    int grid = (int)(g < 1 ? 1 : (g < reduce_grid() * 2 ? g : reduce_grid() * 2));
    reduce_bwd<T, OP><<<grid, kRThreads, 0, s>>>(static_cast<const T *>(as), static_cast<T *>(ab), p);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class T>
vjp_status fwd_dispatch(vjp_op op, const void *as, int64_t n, int64_t goff, void *ws, RRec *out, cudaStream_t s) {
    switch (op) {
    case VJP_ADD: return fwd_launch<T, VJP_ADD>(as, n, goff, ws, out, s);
    case VJP_MUL: return fwd_launch<T, VJP_MUL>(as, n, goff, ws, out, s);
    case VJP_MIN: return fwd_launch<T, VJP_MIN>(as, n, goff, ws, out, s);
    case VJP_MAX: return fwd_launch<T, VJP_MAX>(as, n, goff, ws, out, s);
    default: return VJP_EINVAL;
    }
}
template <class T>
vjp_status bwd_dispatch(vjp_op op, const void *as, void *ab, const RBwd &p, cudaStream_t s) {
    switch (op) {
    case VJP_ADD: return bwd_launch<T, VJP_ADD>(as, ab, p, s);
    case VJP_MUL: return bwd_launch<T, VJP_MUL>(as, ab, p, s);
    case VJP_MIN: return bwd_launch<T, VJP_MIN>(as, ab, p, s);
    case VJP_MAX: return bwd_launch<T, VJP_MAX>(as, ab, p, s);
    default: return VJP_EINVAL;
    }
}

vjp_status check(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, void *ws, size_t ws_bytes) {
    if (!op_ok(op) || !dt_ok(dtype) || n < 0) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    if (!as) return VJP_EINVAL;
    if (!vjph::aligned16(as)) return VJP_EALIGN;
    if (!ws || ws_bytes < rlayout().total) return VJP_EWORKSPACE;
    if (!vjph::aligned16(ws)) return VJP_EALIGN;
    return VJP_OK;
}

vjp_status run_fwd(vjp_op op, vjp_dtype dtype, const void *as, int64_t n, int64_t goff, void *ws, RRec *out,
                   cudaStream_t s) {
    return dtype == VJP_F64 ? fwd_dispatch<double>(op, as, n, goff, ws, out, s)
                            : fwd_dispatch<float>(op, as, n, goff, ws, out, s);
}
vjp_status run_bwd(vjp_op op, vjp_dtype dtype, const void *as, void *ab, const RBwd &p, cudaStream_t s) {
    return dtype == VJP_F64 ? bwd_dispatch<double>(op, as, ab, p, s) : bwd_dispatch<float>(op, as, ab, p, s);
}
}  // namespace

extern "C" {

size_t vjp_reduce_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n) {
    if (op == VJP_LINREC || op == VJP_MAT2) return vjph::reduce_general_ws(op, dtype, n);
    if (!op_ok(op) || !dt_ok(dtype) || n < 0) return 0;
    return rlayout().total;
}

size_t vjp_reduce_partial_bytes(void) { return sizeof(RRec); }

vjp_status vjp_reduce(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                      void *y, int64_t *arg, void *ws, size_t ws_bytes, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_reduce");
    if (op == VJP_LINREC || op == VJP_MAT2) {  // the paper's general rule
        if (arg && n > 0 && cudaMemsetAsync(arg, 0xff, 8, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
            return VJP_ECUDA;  // -1: no index for the general rule
        return vjph::reduce_general(op, dtype, n, as, y_bar, as_bar, y, ws, ws_bytes,
                                    reinterpret_cast<cudaStream_t>(stream), flags);
    }
    vjp_status st = check(op, dtype, n, as, ws, ws_bytes);
    if (st != VJP_OK) return st;
    if (n == 0) return VJP_OK;
    if (!y_bar || !as_bar) return VJP_EINVAL;
    if (!vjph::aligned16(as_bar)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    RLayout L = rlayout();
    RRec *fin = reinterpret_cast<RRec *>(static_cast<unsigned char *>(ws) + L.final_rec);
    const bool need_fwd = op != VJP_ADD || y != nullptr;
    if (need_fwd) {
        st = run_fwd(op, dtype, as, n, 0, ws, fin, s);
        if (st != VJP_OK) return st;
    }
    RBwd p{};
    p.n = n;
    p.goff = 0;
    p.world = 1;
    p.acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    p.recs = need_fwd ? fin : nullptr;  // ADD without y: a broadcast of ybar
    p.ybar = y_bar;
    p.y = y;
    p.arg = arg;
    return run_bwd(op, dtype, as, as_bar, p, s);
}

vjp_status vjp_reduce_partial(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, void *ws, size_t ws_bytes,
                              const vjp_shard *shard, void *partial, vjp_stream_t stream) {
    VJP_NVTX("vjp_reduce_partial");
    if (!shard || !partial || n < 0) return VJP_EINVAL;
    vjp_status st = check(op, dtype, n, as, ws, ws_bytes);
    if (st != VJP_OK) return st;
    if (!vjph::aligned16(partial)) return VJP_EALIGN;
    if (n == 0) {  // empty shard: the neutral record
        RRec *r = static_cast<RRec *>(partial);
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        switch (op) {
        case VJP_ADD: reduce_id_record<VJP_ADD><<<1, 32, 0, s>>>(r); break;
        case VJP_MUL: reduce_id_record<VJP_MUL><<<1, 32, 0, s>>>(r); break;
        case VJP_MIN: reduce_id_record<VJP_MIN><<<1, 32, 0, s>>>(r); break;
        default: reduce_id_record<VJP_MAX><<<1, 32, 0, s>>>(r); break;
        }
        vjph::count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    return run_fwd(op, dtype, as, n, shard->global_offset, ws, static_cast<RRec *>(partial),
                   reinterpret_cast<cudaStream_t>(stream));
}

vjp_status vjp_reduce_finish(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                             void *y, int64_t *arg, void *ws, size_t ws_bytes, const vjp_shard *shard,
                             const void *gathered, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_reduce_finish");
    if (!shard || !gathered || n < 0 || shard->world < 1) return VJP_EINVAL;
    vjp_status st = check(op, dtype, n, as, ws, ws_bytes);
    if (st != VJP_OK) return st;
    if (!y_bar || (n > 0 && !as_bar)) return VJP_EINVAL;
    if (n > 0 && !vjph::aligned16(as_bar)) return VJP_EALIGN;
    if (n == 0 && !y && !arg) return VJP_OK;  // empty shard, no primal outputs requested
    RBwd p{};
    p.n = n;
    p.goff = shard->global_offset;
    p.world = shard->world;
    p.acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    p.recs = static_cast<const RRec *>(gathered);
    p.ybar = y_bar;
    // every rank combines the same records in the same order: y / arg are
    // identical everywhere, so every rank writes them
    p.y = y;
    p.arg = arg;
    return run_bwd(op, dtype, as, as_bar, p, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
