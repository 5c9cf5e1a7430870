// binsort.cuh — deterministic reduce_by_index(+) accumulation of width-w rows
// (P:1120-1126 forward; the AD accumulator of P:1705-1712): a STABLE counting
// sort of the elements by bin, then one CTA per bin sums its (index-ordered)
// segment in a fixed order — no floating-point atomics, so the result does
// not depend on scheduling.  Used by vjp_reduce_by_index(+)'s primal
// histogram (width >= 1, small m) and by vjp_kmeans's center accumulator.
//
//   bs_hist      per block of B elements, per-bin counts (32-bit shared atomics);
//                bins outside [0, m) go to the extra bin m (skipped, R4)
//   bs_colscan   per bin, exclusive scan over the blocks (in place) + totals
//   bs_startscan exclusive scan of the totals -> segment starts (start[m+1])
//   bs_order     stable ranks (warp match_any per 32 elements, in index order)
//                -> order[] = element indices grouped by bin, increasing
//   bs_segsum    per bin b (one CTA): out[b][t] = scale * sum_{i in b} x_i[t]
//                with x_i = as[i] or, given a per-bin offset row off[b],
//                x_i = off[b] - as[i] (the k-means map fused in); each warp a
//                contiguous quarter of the segment, added in warp order.
#pragma once

#include "common.cuh"

namespace vjpk {

constexpr int kBsSegW = 4;   // warps per bin in bs_segsum
constexpr int kBsRows = 16;  // rows gathered per batch in bs_segsum

template <class I>
__device__ __forceinline__ int32_t bs_bin(const I *inds, int64_t i, int64_t m) {
    const int64_t b = (int64_t)inds[i];
    return (b >= 0 && b < m) ? (int32_t)b : (int32_t)m;
}

template <class I>
__global__ void bs_hist(const I *__restrict__ inds, int64_t n, int64_t m, int64_t B, int32_t *__restrict__ hist) {
    extern __shared__ int32_t h[];
    const int64_t mb = m + 1;
    for (int64_t j = threadIdx.x; j < mb; j += blockDim.x) h[j] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * B;
    for (int64_t i = b0 + threadIdx.x; i < b0 + B && i < n; i += blockDim.x) atomicAdd(h + bs_bin(inds, i, m), 1);
    __syncthreads();
    for (int64_t j = threadIdx.x; j < mb; j += blockDim.x) hist[(int64_t)blockIdx.x * mb + j] = h[j];
}

// per bin (column): exclusive scan over the blocks in place, column total.
// CTA = 32 bins (x, coalesced) x 32 block segments (y)
static __global__ void __launch_bounds__(1024) bs_colscan(int32_t *__restrict__ hist, int64_t nb, int64_t mb,
                                                   int32_t *__restrict__ colsum) {
    __shared__ int32_t seg[32][33];
    const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + x;
    const int64_t per = (nb + 31) / 32, b0 = y * per, b1 = b0 + per < nb ? b0 + per : nb;
    int32_t s = 0;
    if (j < mb) {
#pragma unroll 8
        for (int64_t b = b0; b < b1; ++b) s += hist[b * mb + j];
    }
    seg[y][x] = s;
    __syncthreads();
    if (y == 0) {
        int32_t run = 0;
        for (int q = 0; q < 32; ++q) {
            const int32_t v = seg[q][x];
            seg[q][x] = run;
            run += v;
        }
        if (j < mb) colsum[j] = run;
    }
    __syncthreads();
    if (j < mb) {
        int32_t run = seg[y][x];
        for (int64_t b = b0; b < b1; ++b) {
            const int32_t v = hist[b * mb + j];
            hist[b * mb + j] = run;
            run += v;
        }
    }
}

// exclusive scan of the column totals (one CTA of 1024 threads): start[j],
// start[mb] = n; counts (nullable) = the per-bin totals of the m real bins
static __global__ void __launch_bounds__(1024) bs_startscan(const int32_t *__restrict__ colsum, int64_t mb,
                                                     int32_t *__restrict__ start, int64_t *__restrict__ counts,
                                                     int acc_counts) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < mb; base += 1024) {
        const int64_t j = base + t;
        const int32_t v = j < mb ? colsum[j] : 0;
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const int32_t excl = carry + (w ? wsum[w - 1] : 0) + x - v;
        if (j < mb) {
            start[j] = excl;
            if (counts && j < mb - 1) counts[j] = (acc_counts ? counts[j] : 0) + v;
        }
        __syncthreads();
        if (t == 1023) carry = excl + v;
        __syncthreads();
    }
    if (t == 0) start[mb] = carry;
}

// stable counting-sort scatter: one warp per block of B elements, in index order
template <class I>
__global__ void bs_order(const I *__restrict__ inds, int64_t n, int64_t m, int64_t B,
                         const int32_t *__restrict__ hist, const int32_t *__restrict__ start,
                         int32_t *__restrict__ order, int64_t nb) {
    extern __shared__ int32_t cnt[];  // [warps][m + 1]
    const int64_t mb = m + 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * nw + w;
    int32_t *c = cnt + (int64_t)w * mb;
    for (int64_t j = lane; j < mb; j += 32) c[j] = 0;
    __syncwarp();
    if (b >= nb) return;
    const int64_t b0 = b * B;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t b1 = b0 + B < n ? b0 + B : n;
    int32_t an = (b0 + lane < b1) ? bs_bin(inds, b0 + lane, m) : -1;
    for (int64_t i0 = b0; i0 < b1; i0 += 32) {
        const int64_t i = i0 + lane;
        const bool in = i < b1;
        const int32_t a = an;
        an = (i + 32 < b1) ? bs_bin(inds, i + 32, m) : -1;  // next round in flight
        const unsigned act = __ballot_sync(0xffffffffu, in);
        const unsigned peers = __match_any_sync(0xffffffffu, a) & act;
        int32_t base = 0;
        if (in) base = c[a];
        __syncwarp();
        if (in) {
            const int32_t r = base + __popc(peers & lt);
            order[start[a] + hist[b * mb + a] + r] = (int32_t)i;
            if ((peers & lt) == 0) c[a] = base + __popc(peers);  // group leader
        }
        __syncwarp();
    }
}

// one CTA of kBsSegW warps per bin: warp w sums its contiguous quarter of the
// bin's (index-ordered) segment, kBsRows rows in flight; the partials are
// added in warp order — a fixed order, so the result is deterministic.
// out[b][t] = scale * sum x_i[t] (+ out[b][t] with acc), scale = scale_mul *
// (*scale_dev if given: a device scalar such as k-means' cost_bar); cnt_out (nullable):
// cnt_out[b][t] = scale * count_b (+=) — the k-means Hessian diagonal.
template <class T, int RMAX>
__global__ void __launch_bounds__(32 * kBsSegW) bs_segsum(const T *__restrict__ as, const T *__restrict__ off,
                                                          const int32_t *__restrict__ order,
                                                          const int32_t *__restrict__ start, int64_t w,
                                                          double scale_mul, const T *__restrict__ scale_dev,
                                                          T *__restrict__ out, T *__restrict__ cnt_out, int acc) {
    __shared__ double part[kBsSegW][32 * RMAX];
    const double scale = scale_mul * (scale_dev ? (double)*scale_dev : 1.0);
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int64_t j = blockIdx.x;
    const int32_t s0 = start[j], s1 = start[j + 1];
    const int32_t len = s1 - s0, per = (len + kBsSegW - 1) / kBsSegW;
    const int32_t w0 = s0 + min(len, wp * per), w1 = s0 + min(len, (wp + 1) * per);
    for (int64_t dc = 0; dc < w; dc += 32 * RMAX) {
        double oj[RMAX], g[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
            const int64_t t = dc + lane + 32 * r;
            oj[r] = (off && t < w) ? (double)off[j * w + t] : 0.0;
            g[r] = 0.0;
        }
        for (int32_t s = w0; s < w1; s += kBsRows) {
            int32_t pi[kBsRows];
#pragma unroll
            for (int u = 0; u < kBsRows; ++u) pi[u] = (s + u < w1) ? __ldg(order + s + u) : -1;
            double v[kBsRows][RMAX];
#pragma unroll
            for (int u = 0; u < kBsRows; ++u)
#pragma unroll
                for (int r = 0; r < RMAX; ++r) {
                    const int64_t t = dc + lane + 32 * r;
                    v[u][r] = (pi[u] >= 0 && t < w) ? (double)__ldg(as + (int64_t)pi[u] * w + t) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < kBsRows; ++u)
                if (pi[u] >= 0) {
#pragma unroll
                    for (int r = 0; r < RMAX; ++r) g[r] += off ? oj[r] - v[u][r] : v[u][r];
                }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RMAX; ++r) part[wp][lane + 32 * r] = g[r];
        __syncthreads();
        if (wp == 0) {
            const double h = scale * (double)len;
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
                const int64_t t = dc + lane + 32 * r;
                double tot = part[0][lane + 32 * r];
#pragma unroll
                for (int q = 1; q < kBsSegW; ++q) tot += part[q][lane + 32 * r];
                if (t < w) {
                    const double cb = scale * tot;
                    out[j * w + t] = acc ? (T)((double)out[j * w + t] + cb) : (T)cb;
                    if (cnt_out) cnt_out[j * w + t] = acc ? (T)((double)cnt_out[j * w + t] + h) : (T)h;
                }
            }
        }
    }
}

}  // namespace vjpk

namespace vjph {

// workspace of the bin sort: block size, block count and the layout
struct BsLayout {
    int64_t B, nb;
    size_t hist, colsum, start, order, total;
};
inline BsLayout bs_layout(int64_t n, int64_t m, int64_t Bmin = 1024) {
    BsLayout L{};
    const int64_t mb = m + 1;
    // block size: >= Bmin, and the per-block histograms (nb x (m+1) ints)
    // kept within 2^26 entries (256 MB) for large n x m
    int64_t B = Bmin;
    while (n > 0 && ((n + B - 1) / B) * mb > ((int64_t)1 << 26)) B *= 2;
    L.B = B;
    L.nb = n > 0 ? (n + B - 1) / B : 0;
    size_t off = 0;
    L.hist = off; off += align256((size_t)(L.nb > 0 ? L.nb : 1) * (size_t)mb * 4);
    L.colsum = off; off += align256((size_t)mb * 4);
    L.start = off; off += align256((size_t)(mb + 1) * 4);
    L.order = off; off += align256((size_t)(n > 0 ? n : 1) * 4);
    L.total = off;
    return L;
}
constexpr int64_t kBsMaxBins = 12287;  // (m + 1) per-block / per-warp tables in shared memory

// stable counting sort of n elements by bin (m + 1 bins; out of range -> m):
// fills start[0..m+1] and order[0..n) of the layout; counts (nullable) gets
// the per-bin sizes of the m real bins (acc: added)
template <class I>
inline int bs_sort(const I *inds, int64_t n, int64_t m, const BsLayout &L, unsigned char *ws, int64_t *counts,
                   int acc_counts, cudaStream_t s) {
    int32_t *hist = reinterpret_cast<int32_t *>(ws + L.hist);
    int32_t *colsum = reinterpret_cast<int32_t *>(ws + L.colsum);
    int32_t *start = reinterpret_cast<int32_t *>(ws + L.start);
    int32_t *order = reinterpret_cast<int32_t *>(ws + L.order);
    const int64_t mb = m + 1;
    int launches = 0;
    if (n > 0) {
        const size_t hsm = (size_t)mb * 4;
        cudaFuncSetAttribute(vjpk::bs_hist<I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
        vjpk::bs_hist<I><<<(unsigned)L.nb, 256, hsm, s>>>(inds, n, m, L.B, hist);
        ++launches;
    }
    vjpk::bs_colscan<<<(unsigned)((mb + 31) / 32), 1024, 0, s>>>(hist, L.nb, mb, colsum);
    vjpk::bs_startscan<<<1, 1024, 0, s>>>(colsum, mb, start, counts, acc_counts);
    launches += 2;
    if (n > 0) {
        const int wpb = 4;
        const size_t osm = (size_t)wpb * (size_t)mb * 4;
        cudaFuncSetAttribute(vjpk::bs_order<I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osm);
        vjpk::bs_order<I><<<(unsigned)((L.nb + wpb - 1) / wpb), 32 * wpb, osm, s>>>(inds, n, m, L.B, hist, start,
                                                                                  order, L.nb);
        ++launches;
    }
    return launches;
}

// per-bin row sums over the sorted segments (bins 0..m-1; the extra bin m of
// out-of-range elements is not written)
template <class T>
inline int bs_rowsum(const T *as, const T *off, int64_t m, int64_t w, double scale_mul, const T *scale_dev,
                     const BsLayout &L, unsigned char *ws, T *out, T *cnt_out, int acc, cudaStream_t s) {
    const int32_t *start = reinterpret_cast<const int32_t *>(ws + L.start);
    const int32_t *order = reinterpret_cast<const int32_t *>(ws + L.order);
    auto k = w <= 32 ? vjpk::bs_segsum<T, 1> : (w <= 64 ? vjpk::bs_segsum<T, 2> : vjpk::bs_segsum<T, 4>);
    k<<<(unsigned)m, 32 * vjpk::kBsSegW, 0, s>>>(as, off, order, start, w, scale_mul, scale_dev, out, cnt_out, acc);
    return 1;
}

}  // namespace vjph
