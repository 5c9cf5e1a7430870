// rbi_general.cu — reduce_by_index(×) by the paper's GENERAL rule (sec 5.1.2,
// P:1107-1119, with the reduce rule of P:986-1013 applied per bin), for sm_100a.
//
// The paper sketches it as "radix sort + segmented scans" and leaves it "work
// in progress".  Per bin b the general reduce rule gives
//     as_bar_i += hs_bar[b] * l_i * r_i,
// l_i / r_i = product of the bin's other elements before / after i.  Here:
//   rg_count   per-bin element counts (global 64-bit reductions)
//   rg_offsets exclusive scan of the counts (one CTA) -> bin segments
//   rg_place   bucket the values into their bin's segment and record each
//              element's slot pos_of[i] (counting sort;
//              the order inside a segment is the atomic order — l_i * r_i is
//              the product of the OTHER elements whatever the order, so only
//              rounding depends on it)
//   rg_bins    one warp per bin: forward exclusive product scan (l, stored),
//              backward exclusive product scan (r), res = hbar * l * r in
//              segment order
//   rg_gather  as_bar[i] = res[pos_of[i]] in index order
// Small m (<= 8192 bins, n / m long segments): per-chunk shared-memory
// histograms + a column scan give each (chunk, bin) its output range, the
// placement uses shared-memory cursors (runs of a bin are contiguous), and
// one 32-warp CTA per bin scans the segment in 32 parts.
// No zero-count special case: a zero in the bin makes l or r zero exactly as
// the definition does.  Domain: the partial products l_i, r_i stay finite and
// normal (the special-case path, `vjp_reduce_by_index`, tracks exponents in
// the log domain instead; reading R13).  Out-of-range bins: as_bar 0 (R4).
#include "common.cuh"

namespace vjpk {

template <class I>
__global__ void rg_count(const I *__restrict__ inds, int64_t n, int64_t m, unsigned long long *cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = (int64_t)inds[i];
        if (b >= 0 && b < m) atomicAdd(cnt + b, 1ull);
    }
}

// exclusive scan of m counts by one CTA of 1024 threads, 1024 bins per step
__global__ void rg_offsets(const unsigned long long *__restrict__ cnt, int64_t m, unsigned long long *off,
                           unsigned long long *cursor) {
    __shared__ unsigned long long part[32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < m; base += blockDim.x) {
        const int64_t b = base + threadIdx.x;
        const unsigned long long c = b < m ? cnt[b] : 0ull;
        unsigned long long x = c;  // inclusive warp scan
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) part[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned long long p = lane < (int)(blockDim.x >> 5) ? part[lane] : 0ull;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, p, d);
                if (lane >= d) p += y;
            }
            part[lane] = p;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long excl = carry + (wid ? part[wid - 1] : 0ull) + x - c;
        if (b < m) { off[b] = excl; cursor[b] = excl; }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + c;
        __syncthreads();
    }
}

template <class T, class I>
__global__ void rg_place(const I *__restrict__ inds, const T *__restrict__ as, int64_t n, int64_t m,
                         unsigned long long *cursor, int64_t *pos_of, double *val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = (int64_t)inds[i];
        int64_t pos = -1;  // out-of-range bin: no contribution (reading R4)
        if (b >= 0 && b < m) {
            pos = (int64_t)atomicAdd(cursor + b, 1ull);
            val[pos] = (double)as[i];
        }
        pos_of[i] = pos;
    }
}

// product scans over one warp-sized chunk: inclusive (left to right) and the
// exclusive value of each lane
__device__ __forceinline__ double warp_excl_prod(double v, int lane, double *total) {
    double x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x *= y;
    }
    *total = __shfl_sync(0xffffffffu, x, 31);
    const double e = __shfl_up_sync(0xffffffffu, x, 1);
    return lane == 0 ? 1.0 : e;
}
__device__ __forceinline__ double warp_excl_prod_rev(double v, int lane, double *total) {
    double x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_down_sync(0xffffffffu, x, d);
        if (lane + d < 32) x *= y;
    }
    *total = __shfl_sync(0xffffffffu, x, 0);
    const double e = __shfl_down_sync(0xffffffffu, x, 1);
    return lane == 31 ? 1.0 : e;
}

template <class T>
__global__ void rg_bins(const unsigned long long *__restrict__ off, const unsigned long long *__restrict__ cnt,
                        int64_t m, const double *__restrict__ val, double *lbuf, const T *__restrict__ hs_bar) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = gw; b < m; b += nw) {
        const int64_t s0 = (int64_t)off[b], len = (int64_t)cnt[b];
        if (len == 0) continue;
        const double hb = (double)hs_bar[b];
        // forward: l = product of the segment's elements before this one
        double carry = 1.0;
        for (int64_t c = 0; c < len; c += 32) {
            const int64_t k = c + lane;
            const double v = k < len ? val[s0 + k] : 1.0;
            double tot;
            const double e = warp_excl_prod(v, lane, &tot);
            if (k < len) lbuf[s0 + k] = carry * e;
            carry *= tot;
        }
        // backward: r = product after; write the adjoint
        carry = 1.0;
        const int64_t last = ((len - 1) / 32) * 32;
        for (int64_t c = last; c >= 0; c -= 32) {
            const int64_t k = c + lane;
            const double v = k < len ? val[s0 + k] : 1.0;
            double tot;
            const double e = warp_excl_prod_rev(v, lane, &tot);
            if (k < len) {
                lbuf[s0 + k] = hb * (lbuf[s0 + k] * (e * carry));  // the adjoint, in segment order
            }
            carry *= tot;
        }
    }
}

// ---- small m (<= kGenSmallM bins): per-chunk shared-memory histograms and
// placement, and one CTA per bin for the scans (a warp per bin would walk
// n / m elements serially)
constexpr int64_t kGenSmallM = 8192;
constexpr int64_t kGenChunk = 1 << 18;  // elements per placement CTA

template <class I>
__global__ void rg_hist_small(const I *__restrict__ inds, int64_t n, int64_t m, unsigned *__restrict__ H,
                              unsigned long long *cnt) {
    extern __shared__ unsigned hs_[];
    for (int64_t b = threadIdx.x; b < m; b += blockDim.x) hs_[b] = 0u;
    __syncthreads();
    const int64_t e0 = (int64_t)blockIdx.x * kGenChunk, e1 = min(n, e0 + kGenChunk);
    for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
        const int64_t b = (int64_t)inds[i];
        if (b >= 0 && b < m) atomicAdd(hs_ + b, 1u);
    }
    __syncthreads();
    for (int64_t b = threadIdx.x; b < m; b += blockDim.x) {
        H[(int64_t)blockIdx.x * m + b] = hs_[b];
        if (hs_[b]) atomicAdd(cnt + b, (unsigned long long)hs_[b]);
    }
}

// base[c][b] = off[b] + sum_{c' < c} H[c'][b] (one thread per bin, chunks in order)
__global__ void rg_colscan_small(const unsigned *__restrict__ H, int64_t nchunks, int64_t m,
                                 const unsigned long long *__restrict__ off, unsigned long long *base) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m) return;
    unsigned long long run = off[b];
    for (int64_t c = 0; c < nchunks; ++c) {
        base[c * m + b] = run;
        run += H[c * m + b];
    }
}

template <class T, class I>
__global__ void rg_place_small(const I *__restrict__ inds, const T *__restrict__ as, int64_t n, int64_t m,
                               const unsigned long long *__restrict__ base, int64_t *pos_of, double *val) {
    extern __shared__ __align__(16) unsigned char sm_[];
    unsigned long long *bs = reinterpret_cast<unsigned long long *>(sm_);
    unsigned *lc = reinterpret_cast<unsigned *>(bs + m);
    for (int64_t b = threadIdx.x; b < m; b += blockDim.x) { bs[b] = base[(int64_t)blockIdx.x * m + b]; lc[b] = 0u; }
    __syncthreads();
    const int64_t e0 = (int64_t)blockIdx.x * kGenChunk, e1 = min(n, e0 + kGenChunk);
    for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
        const int64_t b = (int64_t)inds[i];
        int64_t pos = -1;
        if (b >= 0 && b < m) {
            pos = (int64_t)(bs[b] + atomicAdd(lc + b, 1u));
            val[pos] = (double)as[i];
        }
        pos_of[i] = pos;
    }
}

// one CTA (32 warps) per bin: the segment is cut into 32 contiguous parts;
// part products -> exclusive scans over the parts -> each warp scans its part
template <class T>
__global__ void __launch_bounds__(1024) rg_bins_cta(const unsigned long long *__restrict__ off,
                                                    const unsigned long long *__restrict__ cnt, int64_t m,
                                                    const double *__restrict__ val, double *lbuf,
                                                    const T *__restrict__ hs_bar) {
    __shared__ double part[32], pre[32], suf[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
        const int64_t s0 = (int64_t)off[b], len = (int64_t)cnt[b];
        if (len == 0) continue;  // uniform across the CTA
        const double hb = (double)hs_bar[b];
        const int64_t per = (len + 31) / 32;
        const int64_t p0 = min(len, (int64_t)w * per), p1 = min(len, p0 + per);
        double pr = 1.0;
        for (int64_t k = p0 + lane; k < p1; k += 32) pr *= val[s0 + k];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) pr *= __shfl_xor_sync(0xffffffffu, pr, d);
        if (lane == 0) part[w] = pr;
        __syncthreads();
        if (threadIdx.x == 0) {
            double r = 1.0;
            for (int j = 0; j < 32; ++j) { pre[j] = r; r *= part[j]; }
            r = 1.0;
            for (int j = 31; j >= 0; --j) { suf[j] = r; r *= part[j]; }
        }
        __syncthreads();
        double carry = pre[w];
        for (int64_t c = p0; c < p1; c += 32) {
            const int64_t k = c + lane;
            const double v = k < p1 ? val[s0 + k] : 1.0;
            double tot;
            const double e = warp_excl_prod(v, lane, &tot);
            if (k < p1) lbuf[s0 + k] = carry * e;
            carry *= tot;
        }
        carry = suf[w];
        if (p1 > p0) {
            for (int64_t c = p0 + ((p1 - p0 - 1) / 32) * 32; c >= p0; c -= 32) {
                const int64_t k = c + lane;
                const double v = k < p1 ? val[s0 + k] : 1.0;
                double tot;
                const double e = warp_excl_prod_rev(v, lane, &tot);
                if (k < p1) {
                    lbuf[s0 + k] = hb * (lbuf[s0 + k] * (e * carry));
                }
                carry *= tot;
            }
        }
        __syncthreads();  // part / pre / suf reused by the next bin
    }
}

// write-back in index order: as_bar[i] (+)= res[pos_of[i]] (coalesced stores,
// random 8-byte reads, instead of a random read-modify-write scatter)
template <class T>
__global__ void rg_gather(const int64_t *__restrict__ pos_of, const double *__restrict__ res, int64_t n, T *as_bar,
                          int acc) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = pos_of[i];
        const double g = p >= 0 ? res[p] : 0.0;
        as_bar[i] = acc ? (T)((double)as_bar[i] + g) : (T)g;
    }
}

}  // namespace vjpk

namespace {

struct GLayout {
    size_t cnt, off, cur, pos, val, lbuf, H, base, total;
};
GLayout glayout(int64_t n, int64_t m) {
    GLayout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += vjph::align256(bytes); return r; };
    L.cnt = take(8 * (size_t)m);
    L.off = take(8 * (size_t)m);
    L.cur = take(8 * (size_t)m);
    L.pos = take(8 * (size_t)n);
    L.val = take(8 * (size_t)n);
    L.lbuf = take(8 * (size_t)n);
    if (m <= vjpk::kGenSmallM) {
        const size_t nch = (size_t)((n + vjpk::kGenChunk - 1) / vjpk::kGenChunk);
        L.H = take(4 * nch * (size_t)m);
        L.base = take(8 * nch * (size_t)m);
    }
    L.total = o;
    return L;
}

template <class T, class I>
vjp_status run_general(int64_t n, int64_t m, const void *inds_, const void *as_, const void *hsb_, void *ab_, void *ws,
                       cudaStream_t s, int acc) {
    using namespace vjpk;
    const I *inds = static_cast<const I *>(inds_);
    const T *as = static_cast<const T *>(as_);
    const T *hsb = static_cast<const T *>(hsb_);
    T *ab = static_cast<T *>(ab_);
    GLayout L = glayout(n, m);
    unsigned char *w = static_cast<unsigned char *>(ws);
    auto *cnt = reinterpret_cast<unsigned long long *>(w + L.cnt);
    auto *off = reinterpret_cast<unsigned long long *>(w + L.off);
    auto *cur = reinterpret_cast<unsigned long long *>(w + L.cur);
    auto *pos_of = reinterpret_cast<int64_t *>(w + L.pos);
    auto *val = reinterpret_cast<double *>(w + L.val);
    auto *lbuf = reinterpret_cast<double *>(w + L.lbuf);
    if (cudaMemsetAsync(cnt, 0, 8 * (size_t)m, s) != cudaSuccess) return VJP_ECUDA;
    const int64_t cap = (int64_t)vjph::sm_count() * 8;
    int64_t g = (n + 255) / 256;
    const int grid = (int)(g < 1 ? 1 : (g > cap ? cap : g));
    if (m <= kGenSmallM) {
        auto *H = reinterpret_cast<unsigned *>(w + L.H);
        auto *base = reinterpret_cast<unsigned long long *>(w + L.base);
        const int64_t nch = (n + kGenChunk - 1) / kGenChunk;
        const size_t smh = 4 * (size_t)m, smp = 12 * (size_t)m;
        cudaFuncSetAttribute(rg_hist_small<I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smh);
        cudaFuncSetAttribute(rg_place_small<T, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smp);
        rg_hist_small<I><<<(unsigned)nch, 1024, smh, s>>>(inds, n, m, H, cnt);
        rg_offsets<<<1, 1024, 0, s>>>(cnt, m, off, cur);
        rg_colscan_small<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(H, nch, m, off, base);
        rg_place_small<T, I><<<(unsigned)nch, 1024, smp, s>>>(inds, as, n, m, base, pos_of, val);
        const int64_t gcap = (int64_t)vjph::sm_count() * 2;
        rg_bins_cta<T><<<(unsigned)(m < gcap ? m : gcap), 1024, 0, s>>>(off, cnt, m, val, lbuf, hsb);
        vjph::count_launch(5);
    } else {
        rg_count<I><<<grid, 256, 0, s>>>(inds, n, m, cnt);
        rg_offsets<<<1, 1024, 0, s>>>(cnt, m, off, cur);
        rg_place<T, I><<<grid, 256, 0, s>>>(inds, as, n, m, cur, pos_of, val);
        int64_t gb = (m * 32 + 255) / 256;
        const int gridb = (int)(gb < 1 ? 1 : (gb > cap ? cap : gb));
        rg_bins<T><<<gridb, 256, 0, s>>>(off, cnt, m, val, lbuf, hsb);
        vjph::count_launch(4);
    }
    rg_gather<T><<<grid, 256, 0, s>>>(pos_of, lbuf, n, ab, acc);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

}  // namespace

extern "C" {

size_t vjp_reduce_by_index_general_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m) {
    (void)dtype;
    if (op != VJP_MUL || n < 0 || m < 1) return 0;
    return glayout(n, m).total;
}

vjp_status vjp_reduce_by_index_general(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m,
                                       const void *inds, const void *as, const void *hs_bar, void *as_bar, void *ws,
                                       size_t ws_bytes, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_reduce_by_index_general");
    if (op == VJP_LINREC || op == VJP_MAT2) return VJP_EUNSUPPORTED;
    if (op != VJP_MUL) return VJP_EUNSUPPORTED;  // ADD / MIN / MAX: the special cases are the rule
    if ((dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (n < 0 || m < 1 || (flags & ~(unsigned)VJP_ACCUMULATE)) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    if (!inds || !as || !hs_bar || !as_bar) return VJP_EINVAL;
    const void *ps[4] = {inds, as, hs_bar, as_bar};
    for (const void *p : ps)
        if (!vjph::aligned16(p)) return VJP_EALIGN;
    const size_t need = glayout(n, m).total;
    if (!ws || ws_bytes < need) return VJP_EWORKSPACE;
    if (!vjph::aligned16(ws)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    if (dtype == VJP_F64)
        return itype == VJP_I32 ? run_general<double, int32_t>(n, m, inds, as, hs_bar, as_bar, ws, s, acc)
                                : run_general<double, int64_t>(n, m, inds, as, hs_bar, as_bar, ws, s, acc);
    return itype == VJP_I32 ? run_general<float, int32_t>(n, m, inds, as, hs_bar, as_bar, ws, s, acc)
                            : run_general<float, int64_t>(n, m, inds, as, hs_bar, as_bar, ws, s, acc);
}

}  // extern "C"
