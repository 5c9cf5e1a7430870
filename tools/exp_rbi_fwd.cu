// exp_rbi_fwd.cu — bottleneck experiment for the small-m reduce_by_index(x)
// forward histogram (rbi.cu rbi_fwd_smem_log): n = 2^28 f64 factors, int32
// bins in [0, 1000).  Variants (template V):
//   0  the library's code path (table log2, F2I rounding, 2 shared atomics)
//   1  integer abs / sign / zero tests, rounding by a magic-number FMA
//   2  as 1 with one shared atomic per element (timing only: wrong sums)
//   3  as 1 with no atomics (codes xor-folded into a register)
//   4  atomics only (the factor's raw bits as the code)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2202_10297_b200/csrc \
//        -o exp_rbi_fwd tools/exp_rbi_fwd.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "log2_table.cuh"

using namespace vjpk;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
struct Log2Tab {
    double inv[128], hi[128], lo[128];
};

template <int V>
__device__ __forceinline__ unsigned long long code_of(double x, uint32_t tb) {
    if (V == 4) return (unsigned long long)__double_as_longlong(x);
    long long b = __double_as_longlong(x) & 0x7fffffffffffffffll;
    int e = (int)(b >> 52);
    if (e == 0) {
        b = __double_as_longlong(__longlong_as_double(b) * 0x1p54);
        e = (int)(b >> 52) - 54;
    }
    e -= 1023;
    const uint32_t k8 = (uint32_t)(b >> 42) & (127u << 3);
    const double m = __longlong_as_double((b & 0x000fffffffffffffll) | 0x3ff0000000000000ll);
    const double r = fma(m, lds_f64(tb + k8), -1.0);
    const double r2 = r * r;
    double P = fma(-1.0 / 6.0, r, 1.0 / 5.0);
    P = fma(P, r, -0.25);
    P = fma(P, r, 1.0 / 3.0);
    P = fma(P, r, -0.5);
    const double u = r2 * P;
    const double K_hi = 1.4426950408889634, K_lo = 2.0355273740931033e-17;
    const double s_hi = r * K_hi;
    double s_lo = fma(r, K_hi, -s_hi);
    s_lo = fma(r, K_lo, s_lo);
    s_lo = fma(u, K_hi, s_lo);
    const double L = lds_f64(tb + 1024 + k8) + (s_hi + (s_lo + lds_f64(tb + 2048 + k8)));
    long long q;
    if (V == 0) {
        q = ((long long)e << 51) + __double2ll_rn(L * 0x1p51);
        return (unsigned long long)q + (x < 0.0 ? 0x8000000000000000ull : 0ull);
    }
    // 1.5 * 2^52: fma(L, 2^51, M) = M + rne(L * 2^51) exactly (0 <= L * 2^51 <= 2^51)
    const double t = fma(L, 0x1p51, 0x1.8p52);
    q = ((long long)e << 51) + (__double_as_longlong(t) - 0x4338000000000000ll);
    return (unsigned long long)q + ((unsigned long long)__double_as_longlong(x) & 0x8000000000000000ull);
}

template <int V>
__global__ void __launch_bounds__(256, 4) fwd(const int *__restrict__ inds, const double *__restrict__ as, int64_t n,
                                             int m, unsigned long long *out, unsigned *zout) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Log2Tab tb;
    for (int k = threadIdx.x; k < 128; k += blockDim.x) {
        tb.inv[k] = kLog2Tab[k][0];
        tb.hi[k] = kLog2Tab[k][1];
        tb.lo[k] = kLog2Tab[k][2];
    }
    unsigned *lo = reinterpret_cast<unsigned *>(smem);
    unsigned *hi = lo + m;
    unsigned *zc = hi + m;
    for (int b = threadIdx.x; b < m; b += blockDim.x) { lo[b] = 0u; hi[b] = 0u; zc[b] = 0u; }
    __syncthreads();
    const uint32_t a_lo = smem_u32(lo), a_hi = smem_u32(hi), a_zc = smem_u32(zc), a_tb = smem_u32(&tb);
    unsigned long long fold = 0;
    auto visit = [&](int b, double x) {
        if ((unsigned)b >= (unsigned)m) return;
        const uint32_t o = (uint32_t)b * 4u;
        const bool zero = V == 0 ? (x == 0.0) : ((__double_as_longlong(x) << 1) == 0);
        if (zero) {
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a_zc + o) : "memory");
        } else {
            const unsigned long long q = code_of<V>(x, a_tb);
            if (V == 3) {
                fold ^= q;
            } else if (V == 2) {
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a_lo + o), "r"((unsigned)q) : "memory");
            } else {
                const unsigned ql = (unsigned)q;
                unsigned old;
                asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a_lo + o), "r"(ql) : "memory");
                const unsigned qh = (unsigned)(q >> 32) + (old + ql < old ? 1u : 0u);
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a_hi + o), "r"(qh) : "memory");
            }
        }
    };
    const int64_t ns = n / 128;
    const int lane = threadIdx.x & 31;
    const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int4 ba, bb;
    double4 xa, xb;
    if (sl < ns) {
        ba = __ldg(reinterpret_cast<const int4 *>(inds + sl * 128 + lane * 4));
        xa = *reinterpret_cast<const double4 *>(as + sl * 128 + lane * 4);
    }
    for (; sl < ns; sl += 2 * ws) {
        const int64_t s1 = sl + ws, s2 = sl + 2 * ws;
        if (s1 < ns) {
            bb = __ldg(reinterpret_cast<const int4 *>(inds + s1 * 128 + lane * 4));
            xb = *reinterpret_cast<const double4 *>(as + s1 * 128 + lane * 4);
        }
        visit(ba.x, xa.x); visit(ba.y, xa.y); visit(ba.z, xa.z); visit(ba.w, xa.w);
        if (s1 >= ns) break;
        if (s2 < ns) {
            ba = __ldg(reinterpret_cast<const int4 *>(inds + s2 * 128 + lane * 4));
            xa = *reinterpret_cast<const double4 *>(as + s2 * 128 + lane * 4);
        }
        visit(bb.x, xb.x); visit(bb.y, xb.y); visit(bb.z, xb.z); visit(bb.w, xb.w);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < m; b += blockDim.x) {
        const unsigned long long t = ((unsigned long long)hi[b] << 32) | lo[b];
        if (t) atomicAdd(out + b, t);
        if (zc[b]) atomicAdd(zout + b, zc[b]);
    }
    if (V == 3 && fold == 0x1234567ull) out[0] = fold;
}

__global__ void gen(int *inds, double *as, int64_t n, int m) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
        inds[i] = (int)((h & 0xffffffffull) % (unsigned)m);
        const double u = (double)((h >> 11) & ((1ull << 40) - 1)) * 0x1p-40;
        double v = exp2((u - 0.5) * 8.0);
        if ((h >> 60) & 1) v = -v;
        if (((h >> 52) & 1023) == 7) v = 0.0;
        as[i] = v;
    }
}

template <int V>
float run(const int *inds, const double *as, int64_t n, int m, unsigned long long *out, unsigned *z, int grid) {
    const size_t sm = 3 * 4 * (size_t)m;
    cudaFuncSetAttribute(fwd<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaMemset(out, 0, 8 * m);
        cudaMemset(z, 0, 4 * m);
        cudaEventRecord(e0);
        fwd<V><<<grid, 256, sm>>>(inds, as, n, m, out, z);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return best;
}

int main() {
    const int64_t n = 1ll << 28;
    const int m = 1000;
    int *inds;
    double *as;
    unsigned long long *out, *out0;
    unsigned *z;
    cudaMalloc(&inds, n * 4);
    cudaMalloc(&as, n * 8);
    cudaMalloc(&out, 8 * m);
    cudaMalloc(&out0, 8 * m);
    cudaMalloc(&z, 4 * m);
    gen<<<4096, 256>>>(inds, as, n, m);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {3, 4}) {
        const int grid = nsm * per;
        float t0 = run<0>(inds, as, n, m, out, z, grid);
        cudaMemcpy(out0, out, 8 * m, cudaMemcpyDeviceToDevice);
        float t1 = run<1>(inds, as, n, m, out, z, grid);
        unsigned long long h0[1000], h1[1000];
        cudaMemcpy(h0, out0, 8 * m, cudaMemcpyDeviceToHost);
        cudaMemcpy(h1, out, 8 * m, cudaMemcpyDeviceToHost);
        int diff = 0;
        for (int b = 0; b < m; ++b) diff += h0[b] != h1[b];
        float t2 = run<2>(inds, as, n, m, out, z, grid);
        float t3 = run<3>(inds, as, n, m, out, z, grid);
        float t4 = run<4>(inds, as, n, m, out, z, grid);
        printf("{\"ctas_per_sm\": %d, \"v0_ms\": %.4f, \"v1_ms\": %.4f, \"v1_bins_differing_from_v0\": %d, "
               "\"v2_one_atomic_ms\": %.4f, \"v3_no_atomics_ms\": %.4f, \"v4_atomics_only_ms\": %.4f, "
               "\"stream_bound_ms\": %.4f}\n",
               per, t0, t1, diff, t2, t3, t4, (double)n * 12 / 6.45e12 * 1e3);
    }
    return cudaGetLastError() != cudaSuccess;
}
