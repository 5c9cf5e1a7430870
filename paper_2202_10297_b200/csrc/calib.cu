// calib.cu — calibration kernels for the reduce_by_index rooflines (not part
// of any vjp): the L2 ceilings of random 8-byte accesses into an L2-resident
// table, measured the same way the m = 10^6 histogram kernels access their
// per-bin state (bins streamed by 128-bit loads with an L2 evict-first hint,
// 4 per lane, one 32-byte sector per access).
//   vjp_calib_l2_gather: out[w] = sum over the warp-lane's elements of
//                        table[idx[i]]  (gathers; one store per thread)
//   vjp_calib_l2_red:    red.add.f64 table[idx[i]] += 1  (fire-and-forget
//                        L2 reductions, as the x histogram's codes)
#include "common.cuh"

namespace vjpk {

__device__ __forceinline__ uint64_t calib_pol() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int4 calib_ld4(const int32_t *p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

__global__ void __launch_bounds__(256) calib_gather(const double *__restrict__ table, const int32_t *__restrict__ idx,
                                                    int64_t n, double *__restrict__ out) {
    const uint64_t pol = calib_pol();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // 16 independent gathers in flight per thread (four 128-bit bin loads
    // issued together), the sums kept in four independent chains
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int64_t e = t * 4;
    for (; e + 12 * stride + 3 < n; e += stride * 16) {
        const int4 b0 = calib_ld4(idx + e, pol), b1 = calib_ld4(idx + e + 4 * stride, pol);
        const int4 b2 = calib_ld4(idx + e + 8 * stride, pol), b3 = calib_ld4(idx + e + 12 * stride, pol);
        const double v0 = __ldg(table + b0.x), v1 = __ldg(table + b0.y), v2 = __ldg(table + b0.z), v3 = __ldg(table + b0.w);
        const double w0 = __ldg(table + b1.x), w1 = __ldg(table + b1.y), w2 = __ldg(table + b1.z), w3 = __ldg(table + b1.w);
        const double x0 = __ldg(table + b2.x), x1 = __ldg(table + b2.y), x2 = __ldg(table + b2.z), x3 = __ldg(table + b2.w);
        const double y0 = __ldg(table + b3.x), y1 = __ldg(table + b3.y), y2 = __ldg(table + b3.z), y3 = __ldg(table + b3.w);
        acc0 += (v0 + v1) + (v2 + v3);
        acc1 += (w0 + w1) + (w2 + w3);
        acc2 += (x0 + x1) + (x2 + x3);
        acc3 += (y0 + y1) + (y2 + y3);
    }
    for (; e + 3 < n; e += stride * 4) {
        const int4 b = calib_ld4(idx + e, pol);
        acc0 += __ldg(table + b.x) + __ldg(table + b.y) + __ldg(table + b.z) + __ldg(table + b.w);
    }
    out[t] = (acc0 + acc1) + (acc2 + acc3);
}

__global__ void __launch_bounds__(256) calib_red(double *__restrict__ table, const int32_t *__restrict__ idx,
                                                 int64_t n) {
    const uint64_t pol = calib_pol();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = t * 4; e + 3 < n; e += stride * 4) {
        const int4 b = calib_ld4(idx + e, pol);
        atomicAdd(table + b.x, 1.0);
        atomicAdd(table + b.y, 1.0);
        atomicAdd(table + b.z, 1.0);
        atomicAdd(table + b.w, 1.0);
    }
}

}  // namespace vjpk

namespace {
int calib_grid() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, vjpk::calib_gather, 256, 0);
    return vjph::sm_count() * (occ > 0 ? occ : 1);
}
}  // namespace

extern "C" {

vjp_status vjp_calib_l2_gather(const double *table, const int32_t *idx, int64_t n, double *out, int64_t out_len,
                               vjp_stream_t stream) {
    if (!table || !idx || !out || n < 0 || (n % 4) || !vjph::aligned16(idx)) return VJP_EINVAL;
    const int g = calib_grid();
    if (out_len < (int64_t)g * 256) return VJP_EINVAL;
    vjpk::calib_gather<<<g, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(table, idx, n, out);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

vjp_status vjp_calib_l2_red(double *table, const int32_t *idx, int64_t n, vjp_stream_t stream) {
    if (!table || !idx || n < 0 || (n % 4) || !vjph::aligned16(idx)) return VJP_EINVAL;
    vjpk::calib_red<<<calib_grid(), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(table, idx, n);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

int64_t vjp_calib_out_len(void) { return (int64_t)calib_grid() * 256; }

}  // extern "C"
