// scatter.cu — vjp_scatter (sec 5.3) for sm_100a.
//
// Return sweep:
//     vs_bar += gather is ys_bar          (vs_bar[j] = ys_bar[is[j]])
//     xs_bar  = scatter ys_bar is (replicate m 0)
// One thread per (target, component): gather then zero, in that order, in the
// same thread, so the in-place form (xs_bar aliasing ys_bar) is race free given
// distinct targets (the precondition of P:1247-1248) and costs O(m) — nothing
// proportional to n is touched.  Out-of-range targets are
// skipped and their vs_bar is 0 (reading R4).  vjp_scatter_forward /
// vjp_scatter_restore are the in-place update's forward save and
// the return sweep's step (3), O(m) as well.  VJP_ACCUMULATE applies to
// vs_bar (the paper's +=); xs_bar is the assignment of P:1275.
#include "common.cuh"

namespace vjpk {

template <class T, class I>
__global__ void scatter_vjp(const I *__restrict__ is, const T *ys_bar, T *xs_bar, T *__restrict__ vs_bar, int64_t n,
                            int64_t m, int64_t width, int acc, int64_t goff) {
    const int64_t total = m * width;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = k / width, c = k - j * width;
        const int64_t t = (int64_t)is[j] - goff;  // goff: first global target this shard owns
        const bool in = t >= 0 && t < n;
        const T g = in ? ys_bar[t * width + c] : (T)0;
        vs_bar[k] = acc ? (T)((double)vs_bar[k] + (double)g) : g;
        if (in) xs_bar[t * width + c] = (T)0;  // after the gather (aliasing-safe)
    }
}

// Forward save + in-place update: saved[j] = xs[is[j]] before
// xs[is[j]] = vs[j], in the same thread.  RESTORE=true is the return sweep's
// step (3): ys[is[j]] = saved[j].  Distinct targets make every
// (target, component) owned by one thread.
template <class T, class I, bool RESTORE>
__global__ void scatter_save(const I *__restrict__ is, const T *__restrict__ vs, T *xs, T *__restrict__ saved,
                             int64_t n, int64_t m, int64_t width) {
    const int64_t total = m * width;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = k / width, c = k - j * width;
        const int64_t t = (int64_t)is[j];
        const bool in = t >= 0 && t < n;
        if (RESTORE) {
            if (in) xs[t * width + c] = saved[k];
        } else {
            saved[k] = in ? xs[t * width + c] : (T)0;
            if (in) xs[t * width + c] = vs[k];
        }
    }
}

// VJP_CHECK_INDICES: count out-of-range and duplicate targets with a bitmap
template <class I>
__global__ void scatter_check(const I *__restrict__ is, int64_t n, int64_t m, uint32_t *bitmap, unsigned long long *cnt) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = (int64_t)is[j];
        if (t < 0 || t >= n) {
            atomicAdd(&cnt[0], 1ull);
            continue;
        }
        const uint32_t bit = 1u << (t & 31);
        if (atomicOr(&bitmap[t >> 5], bit) & bit) atomicAdd(&cnt[1], 1ull);
    }
}

}  // namespace vjpk

namespace {
using namespace vjpk;

size_t check_bytes(int64_t n) { return 256 + vjph::align256((size_t)((n + 31) / 32) * 4); }

template <class T, class I>
vjp_status run(int64_t n, int64_t m, int64_t width, const void *is, const void *ysb, void *xsb, void *vsb,
               cudaStream_t s, int acc, int64_t goff = 0) {
    const int64_t total = m * width;
    int64_t g = (total + 255) / 256;
    const int64_t cap = (int64_t)vjph::sm_count() * 16;
    int grid = (int)(g < 1 ? 1 : (g > cap ? cap : g));
    scatter_vjp<T, I><<<grid, 256, 0, s>>>(static_cast<const I *>(is), static_cast<const T *>(ysb),
                                          static_cast<T *>(xsb), static_cast<T *>(vsb), n, m, width, acc, goff);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class T, class I, bool RESTORE>
vjp_status run_save(int64_t n, int64_t m, int64_t width, const void *is, const void *vs, void *xs, void *saved,
                    cudaStream_t s) {
    const int64_t total = m * width;
    int64_t g = (total + 255) / 256;
    const int64_t cap = (int64_t)vjph::sm_count() * 16;
    int grid = (int)(g < 1 ? 1 : (g > cap ? cap : g));
    scatter_save<T, I, RESTORE><<<grid, 256, 0, s>>>(static_cast<const I *>(is), static_cast<const T *>(vs),
                                                     static_cast<T *>(xs), static_cast<T *>(saved), n, m, width);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <bool RESTORE>
vjp_status dispatch_save(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width, const void *is,
                         const void *vs, void *xs, void *saved, cudaStream_t s) {
    if (dtype == VJP_F64)
        return itype == VJP_I32 ? run_save<double, int32_t, RESTORE>(n, m, width, is, vs, xs, saved, s)
                                : run_save<double, int64_t, RESTORE>(n, m, width, is, vs, xs, saved, s);
    return itype == VJP_I32 ? run_save<float, int32_t, RESTORE>(n, m, width, is, vs, xs, saved, s)
                            : run_save<float, int64_t, RESTORE>(n, m, width, is, vs, xs, saved, s);
}

template <class I>
vjp_status check(int64_t n, int64_t m, const void *is, void *ws, cudaStream_t s) {
    unsigned char *w = static_cast<unsigned char *>(ws);
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(w);
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(w + 256);
    if (cudaMemsetAsync(ws, 0, check_bytes(n), s) != cudaSuccess) return VJP_ECUDA;
    int64_t g = (m + 255) / 256;
    int grid = (int)(g < 1 ? 1 : (g > 4096 ? 4096 : g));
    if (m > 0) {
        scatter_check<I><<<grid, 256, 0, s>>>(static_cast<const I *>(is), n, m, bitmap, cnt);
        vjph::count_launch();
    }
    unsigned long long h[2] = {0, 0};
    if (cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess) return VJP_ECUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) return VJP_ECUDA;
    if (h[0]) return VJP_EOOB;
    if (h[1]) return VJP_EDUPINDEX;
    return VJP_OK;
}
}  // namespace

extern "C" {

size_t vjp_scatter_workspace_bytes(vjp_dtype dtype, int64_t n, int64_t m) {
    (void)dtype;
    (void)m;
    return n < 0 ? 0 : check_bytes(n);  // only used with VJP_CHECK_INDICES
}

vjp_status vjp_scatter(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width, const void *is,
                       const void *ys_bar, void *xs_bar, void *vs_bar, void *ws, size_t ws_bytes, vjp_stream_t stream,
                       unsigned flags) {
    VJP_NVTX("vjp_scatter");
    if ((dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (n < 0 || m < 0 || width < 1) return VJP_EINVAL;
    if ((m > 0 && (!is || !vs_bar)) || (n > 0 && (!ys_bar || !xs_bar))) return VJP_EINVAL;
    const void *ps[4] = {is, ys_bar, xs_bar, vs_bar};
    for (const void *p : ps)
        if (p && !vjph::aligned16(p)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (flags & VJP_CHECK_INDICES) {
        if (!ws || ws_bytes < check_bytes(n)) return VJP_EWORKSPACE;
        vjp_status st = itype == VJP_I32 ? check<int32_t>(n, m, is, ws, s) : check<int64_t>(n, m, is, ws, s);
        if (st != VJP_OK) return st;
    }
    if (n > 0 && xs_bar != ys_bar) {
        const size_t es = dtype == VJP_F64 ? 8 : 4;
        if (cudaMemcpyAsync(xs_bar, ys_bar, (size_t)n * (size_t)width * es, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return VJP_ECUDA;
    }
    if (m == 0) return VJP_OK;
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    if (dtype == VJP_F64)
        return itype == VJP_I32 ? run<double, int32_t>(n, m, width, is, ys_bar, xs_bar, vs_bar, s, acc)
                                : run<double, int64_t>(n, m, width, is, ys_bar, xs_bar, vs_bar, s, acc);
    return itype == VJP_I32 ? run<float, int32_t>(n, m, width, is, ys_bar, xs_bar, vs_bar, s, acc)
                            : run<float, int64_t>(n, m, width, is, ys_bar, xs_bar, vs_bar, s, acc);
}

vjp_status vjp_scatter_shard(vjp_dtype dtype, vjp_itype itype, int64_t n_local, int64_t m, int64_t width,
                             const void *is, const void *ys_bar, void *xs_bar, void *vs_bar_partial,
                             const vjp_shard *shard, vjp_stream_t stream) {
    VJP_NVTX("vjp_scatter_shard");
    if (!shard || shard->world < 1 || shard->global_offset < 0 || n_local < 0 ||
        shard->global_offset + n_local > shard->global_n)
        return VJP_EINVAL;
    if ((dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (m < 0 || width < 1) return VJP_EINVAL;
    if ((m > 0 && (!is || !vs_bar_partial)) || (n_local > 0 && (!ys_bar || !xs_bar))) return VJP_EINVAL;
    const void *ps[4] = {is, ys_bar, xs_bar, vs_bar_partial};
    for (const void *p : ps)
        if (p && !vjph::aligned16(p)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n_local > 0 && xs_bar != ys_bar) {
        const size_t es = dtype == VJP_F64 ? 8 : 4;
        if (cudaMemcpyAsync(xs_bar, ys_bar, (size_t)n_local * (size_t)width * es, cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess)
            return VJP_ECUDA;
    }
    if (m == 0) return VJP_OK;
    const int64_t g = shard->global_offset;
    if (dtype == VJP_F64)
        return itype == VJP_I32 ? run<double, int32_t>(n_local, m, width, is, ys_bar, xs_bar, vs_bar_partial, s, 0, g)
                                : run<double, int64_t>(n_local, m, width, is, ys_bar, xs_bar, vs_bar_partial, s, 0, g);
    return itype == VJP_I32 ? run<float, int32_t>(n_local, m, width, is, ys_bar, xs_bar, vs_bar_partial, s, 0, g)
                            : run<float, int64_t>(n_local, m, width, is, ys_bar, xs_bar, vs_bar_partial, s, 0, g);
}

vjp_status vjp_scatter_forward(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *is, const void *vs, void *xs, void *xs_saved, void *ws, size_t ws_bytes,
                               vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_scatter_forward");
    if ((dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (n < 0 || m < 0 || width < 1 || (flags & ~(unsigned)VJP_CHECK_INDICES)) return VJP_EINVAL;
    if (m > 0 && (!is || !vs || !xs_saved || (n > 0 && !xs))) return VJP_EINVAL;
    const void *ps[4] = {is, vs, xs, xs_saved};
    for (const void *p : ps)
        if (p && !vjph::aligned16(p)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (flags & VJP_CHECK_INDICES) {
        if (!ws || ws_bytes < check_bytes(n)) return VJP_EWORKSPACE;
        vjp_status st = itype == VJP_I32 ? check<int32_t>(n, m, is, ws, s) : check<int64_t>(n, m, is, ws, s);
        if (st != VJP_OK) return st;
    }
    if (m == 0) return VJP_OK;
    return dispatch_save<false>(dtype, itype, n, m, width, is, vs, xs, xs_saved, s);
}

vjp_status vjp_scatter_restore(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *is, const void *xs_saved, void *ys, vjp_stream_t stream) {
    VJP_NVTX("vjp_scatter_restore");
    if ((dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (n < 0 || m < 0 || width < 1) return VJP_EINVAL;
    if (m > 0 && (!is || !xs_saved || (n > 0 && !ys))) return VJP_EINVAL;
    const void *ps[3] = {is, xs_saved, ys};
    for (const void *p : ps)
        if (p && !vjph::aligned16(p)) return VJP_EALIGN;
    if (m == 0) return VJP_OK;
    return dispatch_save<true>(dtype, itype, n, m, width, is, nullptr, ys, const_cast<void *>(xs_saved),
                               reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
