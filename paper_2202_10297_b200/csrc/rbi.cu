// rbi.cu — vjp_reduce_by_index (sec 5.1.2) for sm_100a.
//
// Forward sweep = the histogram with the operator extended as for reduce
// (P:1120-1124); return sweep = the reduce rule with ybar replaced by
// hs_bar[inds[i]].  Bins outside [0, m) are skipped (reading R4).
//
//   ADD      return sweep only: as_bar_i = hs_bar[b_i] — a streaming gather
//            (hs_bar is L2 resident: 8 KB at m = 10^3, 8 MB at m = 10^6).
//   MUL      forward: per-bin (p_b = product of the nonzeros, z_b = #zeros),
//            accumulated in the log domain (sum log2|a| with f64 reductions,
//            zero and negative-factor counts; p_b = +-exp2(sum) per bin):
//            small m in a per-CTA shared-memory table, large m in L2.
//            return: per-bin q_b = hs_bar_b * p_b packed with z_b (one 16-byte
//            gather per element), then the three cases of P:1043-1053.
//   MIN/MAX  forward: per-bin winner = (extremum, LOWEST index) as
//            {orderable value key, ~index}: phase A red.max of the value keys
//            behind a monotone filter plus a per-warp candidate list, phase B
//            red.max of ~index over the candidates equal to the final key.
//            The dense return is a memset plus a scatter of hs_bar[b] to the
//            m winners.
#include <cstdlib>

#include "common.cuh"
#include "log2_table.cuh"
#include "binsort.cuh"

namespace vjpk {

constexpr int kBThreads = 256;
// shared-memory histogram kernels (MIN/MAX phase A, small-m MUL): <= 64
// registers -> 4 CTAs (32 warps) per SM to hide the load latency (78 registers
// gave 3 CTAs, long-scoreboard bound): MAX m=1e3 1.21 -> 1.11 ms.  Measured
// slower for the gather / L2-reduction kernels, which keep their registers.
#ifndef VJP_RBI_MINB
#define VJP_RBI_MINB 4
#endif
constexpr int kBMinBlocks = VJP_RBI_MINB;
constexpr int64_t kSmallM = 16384;  // per-bin tables that stay in L1 / shared memory

template <class I>
struct IdxVec;
template <>
struct IdxVec<int32_t> {
    static constexpr int N = 4;
    using V = int4;
    __device__ static __forceinline__ void get(const V &v, int64_t *o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct IdxVec<int64_t> {
    static constexpr int N = 2;
    using V = longlong2;
    __device__ static __forceinline__ void get(const V &v, int64_t *o) { o[0] = v.x; o[1] = v.y; }
};

// ------------------------------------------------------------ key helpers
// orderable 64-bit key of a double (total order = IEEE order on non-NaN,
// -0.0 canonicalised to +0.0 so that the two tie, reading A9/R-tie)
__device__ __forceinline__ uint64_t ord_key(double x, bool is_min) {
    if (x == 0.0) x = 0.0;
    uint64_t u = (uint64_t)__double_as_longlong(x);
    u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    return is_min ? ~u : u;  // min-reduction: larger key = smaller value
}
__device__ __forceinline__ double key_val(uint64_t k, bool is_min) {
    uint64_t u = is_min ? ~k : k;
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)u);
}

struct alignas(16) Win {
    uint64_t key;  // 0 = empty bin
    uint64_t inv;  // ~index (larger = lower index)
};

__device__ __forceinline__ bool win_better(uint64_t k, uint64_t i, uint64_t ck, uint64_t ci) {
    return k > ck || (k == ck && i > ci);
}

struct RbiParams {
    int64_t n, m, goff;
    int32_t acc, zero_fill;
    int32_t v256, pad;  // value arrays 32-byte aligned: 256-bit accesses
    double *p;        // MUL: [m] product of nonzeros
    unsigned long long *z;  // MUL: [m] zero count
    Win *win;         // MIN/MAX: [m] {value key (max), ~index (max)}
    unsigned long long *code;   // MUL: [m] sum of the factors' codes (mod 2^64), aliases p
    int32_t log_domain, pad2;   // MUL: p holds the codes until rbi_log_finalize
    unsigned long long *cand;   // MIN/MAX: candidate list [cap][3] = {key, global index, bin}
    unsigned long long *ncand;  // candidate counter
    int64_t cap;
};

// ------------------------------------------------------------ init
template <int OP>
__global__ void rbi_init(RbiParams P) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.ncand) *P.ncand = 0ull;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < P.m; b += (int64_t)gridDim.x * blockDim.x) {
        if (OP == VJP_MUL) {
            P.code[b] = 0ull;
            P.z[b] = 0ull;
        }
        else { P.win[b].key = 0ull; P.win[b].inv = 0ull; }
    }
}

// ------------------------------------------------------------ element I/O
// A lane owns 4 consecutive elements per "slab" (a warp covers 128): bins by
// one 16-byte (int32) or two 16-byte (int64) loads, values by one (f32) or two
// (f64) 16-byte loads, zero-fill by 16-byte stores — lane-contiguous and
// read-only cached, so every DRAM sector is fetched once.
// streamed arrays are touched once: L2 evict_first so they do not push the
// per-bin state / hs_bar (re-used, L2 resident) out of L2
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void ld_bins4(const int32_t *p, int64_t e, int64_t *b, uint64_t pol) {
    int x, y, z, w;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "l"(p + e), "l"(pol));
    b[0] = x; b[1] = y; b[2] = z; b[3] = w;
}
__device__ __forceinline__ void ld_bins4(const int64_t *p, int64_t e, int64_t *b, uint64_t pol) {
    long long x, y, z, w;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s64 {%0,%1}, [%2], %3;"
                 : "=l"(x), "=l"(y) : "l"(p + e), "l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s64 {%0,%1}, [%2], %3;"
                 : "=l"(z), "=l"(w) : "l"(p + e + 2), "l"(pol));
    b[0] = x; b[1] = y; b[2] = z; b[3] = w;
}
// f64: one 256-bit access per lane (a whole 32-byte sector); requires 32-byte
// aligned arrays (checked on the host, else two 128-bit accesses)
__device__ __forceinline__ void ld_vals4(const double *p, int64_t e, double *x, uint64_t pol, bool v256) {
    if (v256) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(p + e), "l"(pol));
    } else {
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(x[0]), "=d"(x[1]) : "l"(p + e), "l"(pol));
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(x[2]), "=d"(x[3]) : "l"(p + e + 2), "l"(pol));
    }
}
__device__ __forceinline__ void ld_vals4(const float *p, int64_t e, double *x, uint64_t pol, bool) {
    float a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(p + e), "l"(pol));
    x[0] = a; x[1] = b; x[2] = c; x[3] = d;
}
__device__ __forceinline__ void st_vals4(double *p, int64_t e, const double *x, uint64_t pol, bool v256) {
    if (v256) {
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;"
                     ::"l"(p + e), "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3]), "l"(pol) : "memory");
    } else {
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p + e), "d"(x[0]), "d"(x[1]), "l"(pol) : "memory");
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p + e + 2), "d"(x[2]), "d"(x[3]), "l"(pol) : "memory");
    }
}
__device__ __forceinline__ void st_vals4(float *p, int64_t e, const double *x, uint64_t pol, bool) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 ::"l"(p + e), "f"((float)x[0]), "f"((float)x[1]), "f"((float)x[2]), "f"((float)x[3]), "l"(pol) : "memory");
}
// plain (cached) loads of the accumulate input
__device__ __forceinline__ void ld_acc4(const double *p, int64_t e, double *x) {
    double2 v0 = reinterpret_cast<const double2 *>(p + e)[0], v1 = reinterpret_cast<const double2 *>(p + e)[1];
    x[0] = v0.x; x[1] = v0.y; x[2] = v1.x; x[3] = v1.y;
}
__device__ __forceinline__ void ld_acc4(const float *p, int64_t e, double *x) {
    float4 v = *reinterpret_cast<const float4 *>(p + e);
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
}

// ------------------------------------------------------------ forward
// Every element is visited once; `visit(b, x, gi, ok)` is called by all 32
// lanes of a warp together (warp-uniform trip counts), ok = in-range bin.
template <class T, class I, class F>
__device__ __forceinline__ void rbi_stream(const I *__restrict__ inds, const T *__restrict__ as, T *__restrict__ ab,
                                           const RbiParams &P, F visit) {
    const int64_t ns = P.n / 128;  // full slabs
    const int lane = threadIdx.x & 31;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = policy_evict_first();
    // register double-buffering: the next slab's loads are in flight while
    // the current slab's bins are being updated
    int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t b[4], bn[4];
    double x[4], xn[4];
    if (sl < ns) {
        ld_bins4(inds, sl * 128 + lane * 4, b, pol);
        ld_vals4(as, sl * 128 + lane * 4, x, pol, P.v256);
    }
    for (; sl < ns; sl += wstride) {
        const int64_t e = sl * 128 + lane * 4;
        const int64_t sn = sl + wstride;
        if (sn < ns) {
            ld_bins4(inds, sn * 128 + lane * 4, bn, pol);
            ld_vals4(as, sn * 128 + lane * 4, xn, pol, P.v256);
        }
        if (P.zero_fill) {
            const double z[4] = {0.0, 0.0, 0.0, 0.0};
            st_vals4(ab, e, z, pol, P.v256);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) visit(b[q], x[q], P.goff + e + q, b[q] >= 0 && b[q] < P.m);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[q] = bn[q];
            x[q] = xn[q];
        }
    }
    // tail (< 128 elements): warp 0 of block 0, warp-uniform rounds
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        for (int64_t e0 = ns * 128; e0 < P.n; e0 += 32) {
            const int64_t e = e0 + lane;
            const bool in = e < P.n;
            const int64_t bb = in ? (int64_t)inds[e] : -1;
            const double xx = in ? (double)as[e] : 0.0;
            if (in && P.zero_fill) ab[e] = (T)0;
            visit(bb, xx, P.goff + e, in && bb >= 0 && bb < P.m);
        }
    }
}

// The MUL histograms accumulate, per bin, ONE 64-bit integer code per
// nonzero factor a (reading R13b, DESIGN 7.4):
//     code(a) = round(log2|a| * 2^51)  +  (a < 0 ? 2^63 : 0)      (mod 2^64)
// Sums of codes are taken mod 2^64 with integer adds, so they are EXACT and
// independent of the order of the additions (deterministic, and the
// multi-GPU exchange is an integer SUM).  Decoding a bin's total T: the log
// sum L = T sign-extended from 63 bits (|L| < 2^62 because |sum log2|a|| <
// 2048 in the domain where p stays finite and normal, reading R13), the sign
// parity = bit 63 of (T - L); p = (-1)^parity * 2^(L / 2^51).  Quantisation
// error 2^-52 per factor on log2, i.e. <= 0.7 * 2^-52 * n_b relative on p
// (n_b = factors in the bin): 4e-11 at n_b = 2.7e5 (config 4, m = 10^3).
// The code's log2 by table + short series (no division, ~13 FP64 ops): x =
// m * 2^e, m in [1, 2); k = top 7 bits of m's fraction; inv_k ~ 1/c_k and
// T_k = -log2(inv_k) exactly (hi + lo) from log2_table.cuh (staged in shared
// memory: divergent lookups); m * inv_k = 1 + r, |r| < 2^-7.9, r from one FMA
// (error <= 2^-61); log2(1 + r) = (r + r^2 P(r)) / ln 2, P the ln(1+r)
// series to r^6 (truncation < 2^-58); the products by 1/ln 2 carry an error
// term, so the code is within ~2^-52 of log2|x| * 2^51 rounded.
struct Log2Tab {
    double inv[128], hi[128], lo[128];
};
__device__ __forceinline__ void log2tab_load(Log2Tab &t) {
    for (int k = threadIdx.x; k < 128; k += blockDim.x) {
        t.inv[k] = kLog2Tab[k][0];
        t.hi[k] = kLog2Tab[k][1];
        t.lo[k] = kLog2Tab[k][2];
    }
}
__device__ __constant__ double kLn1pP[5] = {-1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -1.0 / 2.0};
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// the same code with the table addressed through a 32-bit shared-window
// address computed once per thread (the hot loop of the small-m histogram)
__device__ __forceinline__ unsigned long long mul_code_s(double x, uint32_t tb) {
    // |x| by integer ops on the high word (not a DADD on the FP64 pipe)
    long long b = ((long long)(__double2hiint(x) & 0x7fffffff) << 32) | (unsigned)__double2loint(x);
    int e = (int)(b >> 52);
    if (e == 0) {  // subnormal
        b = __double_as_longlong(__longlong_as_double(b) * 0x1p54);
        e = (int)(b >> 52) - 54;
    }
    e -= 1023;
    const uint32_t k8 = (uint32_t)(b >> 42) & (127u << 3);  // 8 * (top 7 fraction bits)
    const double m = __longlong_as_double((b & 0x000fffffffffffffll) | 0x3ff0000000000000ll);
    const double r = fma(m, lds_f64(tb + k8), -1.0);
    const double r2 = r * r;
    double P = fma(-1.0 / 6.0, r, 1.0 / 5.0);
    P = fma(P, r, -0.25);
    P = fma(P, r, 1.0 / 3.0);
    P = fma(P, r, -0.5);
    const double u = r2 * P;  // ln(1 + r) = r + u
    const double K_hi = 1.4426950408889634, K_lo = 2.0355273740931033e-17;  // 1 / ln 2
    const double s_hi = r * K_hi;
    double s_lo = fma(r, K_hi, -s_hi);
    s_lo = fma(r, K_lo, s_lo);
    s_lo = fma(u, K_hi, s_lo);
    const double L = lds_f64(tb + 1024 + k8) + (s_hi + (s_lo + lds_f64(tb + 2048 + k8)));
    // rne(L * 2^51) by one FMA: 0 <= L * 2^51 <= 2^51, so L * 2^51 + 1.5 * 2^52
    // lies in a binade of unit ulp and its low mantissa bits are the rounded
    // integer (the same value as __double2ll_rn, without the F2I.F64 pipe)
    const double t = fma(L, 0x1p51, 0x1.8p52);
    const long long q = ((long long)e << 51) + (__double_as_longlong(t) - 0x4338000000000000ll);
    return (unsigned long long)q + ((unsigned long long)__double_as_longlong(x) & 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned long long mul_code(double x, const Log2Tab &tb) {
    // |x| by integer ops on the high word (not a DADD on the FP64 pipe)
    long long b = ((long long)(__double2hiint(x) & 0x7fffffff) << 32) | (unsigned)__double2loint(x);
    int e = (int)(b >> 52);
    if (e == 0) {  // subnormal
        b = __double_as_longlong(__longlong_as_double(b) * 0x1p54);
        e = (int)(b >> 52) - 54;
    }
    e -= 1023;
    const int k = (int)((b >> 45) & 127);
    const double m = __longlong_as_double((b & 0x000fffffffffffffll) | 0x3ff0000000000000ll);
    const double r = fma(m, tb.inv[k], -1.0);
    const double r2 = r * r;
    double P = fma(kLn1pP[0], r, kLn1pP[1]);
    P = fma(P, r, kLn1pP[2]);
    P = fma(P, r, kLn1pP[3]);
    P = fma(P, r, kLn1pP[4]);
    const double u = r2 * P;  // ln(1 + r) = r + u
    const double K_hi = 1.4426950408889634, K_lo = 2.0355273740931033e-17;  // 1 / ln 2
    const double s_hi = r * K_hi;
    double s_lo = fma(r, K_hi, -s_hi);
    s_lo = fma(r, K_lo, s_lo);
    s_lo = fma(u, K_hi, s_lo);
    const double L = tb.hi[k] + (s_hi + (s_lo + tb.lo[k]));  // log2 m in [0, 1]
    // rne(L * 2^51) by one FMA: 0 <= L * 2^51 <= 2^51, so L * 2^51 + 1.5 * 2^52
    // lies in a binade of unit ulp and its low mantissa bits are the rounded
    // integer (the same value as __double2ll_rn, without the F2I.F64 pipe)
    const double t = fma(L, 0x1p51, 0x1.8p52);
    const long long q = ((long long)e << 51) + (__double_as_longlong(t) - 0x4338000000000000ll);
    return (unsigned long long)q + ((unsigned long long)__double_as_longlong(x) & 0x8000000000000000ull);
}
__device__ __forceinline__ double mul_decode(unsigned long long T) {
    const long long L = ((long long)(T << 1)) >> 1;  // sign-extend 63 bits
    const bool neg = (((T - (unsigned long long)L) >> 63) & 1ull) != 0;
    const long long E = L >> 51;                      // floor(L / 2^51)
    const double f = (double)(L & ((1ll << 51) - 1)) * 0x1p-51;  // [0, 1), exact
    double v = exp2(f);
    v = (E > 2100) ? INFINITY : (E < -2100 ? 0.0 : ldexp(v, (int)E));
    return neg ? -v : v;
}

// test hook: the factor codes of n values (tests compare them with exact codes)
__global__ void rbi_code_probe(const double *x, unsigned long long *y, int64_t n) {
    __shared__ Log2Tab tb;
    log2tab_load(tb);
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = mul_code(x[i], tb);
}

// MUL, large m: every element must contribute, and a CAS-multiply costs two
// dependent L2 round trips per element.  Instead add each factor's 64-bit
// code (above) into the bin with a fire-and-forget integer red.add (native
// RED.ADD.64 in L2) and count zeros.
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbi_fwd_log(const I *__restrict__ inds, const T *__restrict__ as,
                                                         RbiParams P) {
    __shared__ Log2Tab tb;
    log2tab_load(tb);
    __syncthreads();
    rbi_stream<T, I>(inds, as, nullptr, P, [&](int64_t b, double x, int64_t, bool ok) {
        if (!ok) return;
        if ((__double_as_longlong(x) << 1) == 0) atomicAdd(P.z + b, 1ull);  // +-0 (integer test)
        else atomicAdd(P.code + b, mul_code(x, tb));
    });
}
// ---- cp.async ring for the streamed (inds, as) slabs ----------------------
// The register double-buffer (rbi_stream) keeps ONE slab (1.5 KB per warp) in
// flight; ncu of the small-m x histogram shows a third of its warp samples on
// the long scoreboard.  Here each lane stages its own 16-byte granules of the
// next S slabs in shared memory with cp.async (no registers held) and reads
// back only what it copied itself — its own cp.async.wait_group is the only
// synchronisation.  Granule g of thread t in stage s sits at s * kStage +
// g * 4 KB + t * 16 B (conflict-free 128-bit accesses).  Measured at n = 2^28,
// m = 10^3: forward 856 -> 804 us.  Used by the x histogram only: in the x
// return map (992 -> 1131 us at depth 2 or 4) and in MIN/MAX phase A (whole
// call 1.09 -> 1.20 ms) it measured slower (DESIGN 7.6).
#ifndef VJP_RING_FWD
#define VJP_RING_FWD 3
#endif
constexpr int kRingFwd = VJP_RING_FWD > 0 ? VJP_RING_FWD : 1;  // forward histogram (0: register path)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
template <class T, class I, int S>
struct SlabRing {
    static constexpr int GI = (int)sizeof(I) / 4, GV = (int)sizeof(T) / 4;  // 16-byte granules per lane
    static constexpr int kGran = kBThreads * 16;
    static constexpr int kStage = (GI + GV) * kGran;
    static constexpr int kBytes = S * kStage;
    __device__ static __forceinline__ void issue(uint32_t sb, int st, const I *inds, const T *as, int64_t e,
                                                 uint64_t pol) {
        const uint32_t d = sb + st * kStage + threadIdx.x * 16;
#pragma unroll
        for (int g = 0; g < GI; ++g) cp_async16(d + g * kGran, reinterpret_cast<const char *>(inds + e) + 16 * g, pol);
#pragma unroll
        for (int g = 0; g < GV; ++g)
            cp_async16(d + (GI + g) * kGran, reinterpret_cast<const char *>(as + e) + 16 * g, pol);
    }
    __device__ static __forceinline__ void read(uint32_t sb, int st, int64_t *b, double *x) {
        const uint32_t d = sb + st * kStage + threadIdx.x * 16;
        if (GI == 1) {
            const uint4 v = lds128(d);
            b[0] = (int32_t)v.x; b[1] = (int32_t)v.y; b[2] = (int32_t)v.z; b[3] = (int32_t)v.w;
        } else {
            const uint4 v = lds128(d), w = lds128(d + kGran);
            b[0] = (int64_t)(((uint64_t)v.y << 32) | v.x); b[1] = (int64_t)(((uint64_t)v.w << 32) | v.z);
            b[2] = (int64_t)(((uint64_t)w.y << 32) | w.x); b[3] = (int64_t)(((uint64_t)w.w << 32) | w.z);
        }
        const uint32_t dv = d + GI * kGran;
        if (GV == 1) {
            const uint4 v = lds128(dv);
            x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y); x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
        } else {
            const uint4 v = lds128(dv), w = lds128(dv + kGran);
            x[0] = __hiloint2double((int)v.y, (int)v.x); x[1] = __hiloint2double((int)v.w, (int)v.z);
            x[2] = __hiloint2double((int)w.y, (int)w.x); x[3] = __hiloint2double((int)w.w, (int)w.z);
        }
    }
};
// small m: one shared-memory table per CTA.  Shared-memory atomics are native
// only for 32-bit integer add on sm_100a (f64 and 64-bit adds compile to
// ATOMS.CAST.SPIN.64 CAS loops, profiles/r01_ncu_full_rbi_fwd_smem_log_m1e3.txt),
// so each 64-bit code is added as two 32-bit words: the low word with
// ATOMS.ADD returning the old value (a wrap is a carry into the high word),
// the high word with ATOMS.ADD — exact mod 2^64.  Zero counts: 32-bit adds.
// Merged into the global codes with RED.ADD.64.
template <class T, class I, bool RING>
__global__ void __launch_bounds__(kBThreads, kBMinBlocks) rbi_fwd_smem_log(const I *__restrict__ inds, const T *__restrict__ as,
                                                              RbiParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Log2Tab tb;
    log2tab_load(tb);
    unsigned *lo = reinterpret_cast<unsigned *>(smem);
    unsigned *hi = lo + P.m;
    unsigned *zc = hi + P.m;
    for (int64_t b = threadIdx.x; b < P.m; b += blockDim.x) { lo[b] = 0u; hi[b] = 0u; zc[b] = 0u; }
    __syncthreads();
    const uint64_t m = (uint64_t)P.m;
    // 32-bit shared-window addresses, computed once (the generic-pointer
    // atomics re-derived the window base for every element)
    const uint32_t a_lo = smem_u32(lo), a_hi = smem_u32(hi), a_zc = smem_u32(zc), a_tb = smem_u32(&tb);
    auto visit = [&](int64_t b, double x) {
        if ((uint64_t)b >= m) return;  // out-of-range bins (negative ones wrap): skipped (R4)
        const uint32_t o = (uint32_t)b * 4u;
        if ((__double_as_longlong(x) << 1) == 0) {  // +-0 (integer test, no FP64 compare)
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a_zc + o) : "memory");
        } else {
            const unsigned long long q = mul_code_s(x, a_tb);
            const unsigned ql = (unsigned)q;
            unsigned old;
            asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a_lo + o), "r"(ql) : "memory");
            const unsigned qh = (unsigned)(q >> 32) + (old + ql < old ? 1u : 0u);
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a_hi + o), "r"(qh) : "memory");
        }
    };
    if constexpr (RING) {  // cp.async-staged slabs after the table (16-byte aligned streams)
        using R = SlabRing<T, I, kRingFwd>;
        const uint32_t sb = smem_u32(smem) + (((uint32_t)P.m * 12u + 15u) & ~15u);
        const int64_t ns = P.n / 128;
        const int lane = threadIdx.x & 31;
        const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
        const uint64_t pol = policy_evict_first();
        const int64_t sl0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
        for (int k = 0; k < kRingFwd; ++k) {
            const int64_t s = sl0 + k * ws;
            if (s < ns) R::issue(sb, k, inds, as, s * 128 + lane * 4, pol);
            cp_async_commit();
        }
        int st = 0;
        for (int64_t sl = sl0; sl < ns; sl += ws) {
            cp_async_wait<kRingFwd - 1>();
            int64_t b[4];
            double x[4];
            R::read(sb, st, b, x);
#pragma unroll
            for (int q = 0; q < 4; ++q) visit(b[q], x[q]);
            const int64_t sn = sl + kRingFwd * ws;  // refill after the values were consumed
            if (sn < ns) R::issue(sb, st, inds, as, sn * 128 + lane * 4, pol);
            cp_async_commit();
            st = (st + 1 == kRingFwd) ? 0 : st + 1;
        }
        cp_async_wait<0>();
        if (blockIdx.x == 0 && threadIdx.x < 32) {  // tail (< 128 elements)
            for (int64_t e = ns * 128 + lane; e < P.n; e += 32) visit((int64_t)inds[e], (double)as[e]);
        }
    } else {  // slab loop unrolled by two (ping-pong register buffers: no copies)
        const int64_t ns = P.n / 128;
        const int lane = threadIdx.x & 31;
        const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
        const uint64_t pol = policy_evict_first();
        int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        int64_t ba[4], bb[4];
        double xa[4], xb[4];
        if (sl < ns) {
            ld_bins4(inds, sl * 128 + lane * 4, ba, pol);
            ld_vals4(as, sl * 128 + lane * 4, xa, pol, P.v256);
        }
        for (; sl < ns; sl += 2 * ws) {
            const int64_t s1 = sl + ws, s2 = sl + 2 * ws;
            if (s1 < ns) {
                ld_bins4(inds, s1 * 128 + lane * 4, bb, pol);
                ld_vals4(as, s1 * 128 + lane * 4, xb, pol, P.v256);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) visit(ba[q], xa[q]);
            if (s1 >= ns) break;
            if (s2 < ns) {
                ld_bins4(inds, s2 * 128 + lane * 4, ba, pol);
                ld_vals4(as, s2 * 128 + lane * 4, xa, pol, P.v256);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) visit(bb[q], xb[q]);
        }
        if (blockIdx.x == 0 && threadIdx.x < 32) {  // tail (< 128 elements)
            for (int64_t e = ns * 128 + lane; e < P.n; e += 32) visit((int64_t)inds[e], (double)as[e]);
        }
    }
    __syncthreads();
    for (int64_t b = threadIdx.x; b < P.m; b += blockDim.x) {
        const unsigned long long t = ((unsigned long long)hi[b] << 32) | lo[b];
        if (t) atomicAdd(P.code + b, t);
        if (zc[b]) atomicAdd(P.z + b, (unsigned long long)zc[b]);
    }
}

// p_b from the bin's code (in place: P.p aliases P.code)
__global__ void rbi_log_finalize(RbiParams P) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < P.m; b += (int64_t)gridDim.x * blockDim.x)
        P.p[b] = mul_decode(P.code[b]);
}

__device__ __forceinline__ void red_max_u64(unsigned long long *a, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

__device__ __forceinline__ void red_max_u64_shared(unsigned long long *a, unsigned long long v) {
    asm volatile("red.relaxed.cta.shared::cta.max.u64 [%0], %1;" ::"r"(smem_u32(a)), "l"(v) : "memory");
}

// MIN/MAX phase A: per-bin extremum of the value key.  The stored key only
// grows, so an element whose key is below a stored key can never win: skip
// it; otherwise fire-and-forget red.max (no round trip, no divergent wait)
// and append it to the warp's own region of the candidate list (no shared
// counter).  Every eventual winner passes the filter (its key >= any stored
// key).  SMEM (small m): the filter is a per-CTA shared-memory table merged
// into the global keys at the end; large m: the global keys in L2.
template <class T, class I, int OP, bool SMEM>
__global__ void __launch_bounds__(kBThreads, kBMinBlocks) rbi_ext_a(const I *__restrict__ inds, const T *__restrict__ as,
                                                       T *__restrict__ ab, RbiParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long *hk = reinterpret_cast<unsigned long long *>(smem);
    const bool is_min = OP == VJP_MIN;
    const int lane = threadIdx.x & 31;
    if (SMEM) {
        for (int64_t b = threadIdx.x; b < P.m; b += blockDim.x) hk[b] = 0ull;
        __syncthreads();
    }
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t R = P.cap / nw;  // this warp's region of the candidate list
    unsigned long long *reg = P.cand + 3 * gw * R;
    int64_t cnt = 0;
    auto visit = [&](int64_t b, double x, int64_t gi, bool ok) {
        uint64_t k = 0;
        bool cand = false;
        if (ok) {
            k = ord_key(x, is_min);
            unsigned long long *slot = SMEM ? hk + b : reinterpret_cast<unsigned long long *>(&P.win[b].key);
            const uint64_t ck = SMEM ? *reinterpret_cast<volatile unsigned long long *>(slot) : __ldcg(slot);
            cand = k >= ck;
            if (k > ck) {
                if (SMEM) red_max_u64_shared(slot, k);
                else red_max_u64(slot, k);
            }
        }
        const unsigned msk = __ballot_sync(0xffffffffu, cand);
        if (cand) {
            const int64_t q = cnt + __popc(msk & ((1u << lane) - 1u));
            if (q < R) {
                unsigned long long *c = reg + 3 * q;
                c[0] = k;
                c[1] = (unsigned long long)gi;
                c[2] = (unsigned long long)b;
            }
        }
        cnt += __popc(msk);
    };
    rbi_stream<T, I>(inds, as, ab, P, visit);
    if (lane == 0) {
        P.ncand[1 + gw] = (unsigned long long)cnt;
        if (cnt > R) atomicOr(P.ncand, 1ull);  // overflow: phase B re-reads the inputs
    }
    if (SMEM) {
        __syncthreads();
        for (int64_t b = threadIdx.x; b < P.m; b += blockDim.x)
            if (hk[b]) red_max_u64(reinterpret_cast<unsigned long long *>(&P.win[b].key), hk[b]);
    }
}

// MIN/MAX phase B: among the elements whose key equals the final per-bin key,
// the LOWEST global index wins (red.max of ~index).  Walks the candidate list,
// or (if it overflowed) re-reads the inputs.
template <class T, class I, int OP>
__global__ void __launch_bounds__(kBThreads) rbi_ext_b(const I *__restrict__ inds, const T *__restrict__ as,
                                                       RbiParams P, int64_t nwa) {
    const bool is_min = OP == VJP_MIN;
    if (__ldcg(P.ncand) == 0ull) {
        // walk every phase-A warp's region (nwa warps, R entries each)
        const int64_t R = P.cap / nwa;
        const int64_t total = nwa * R;
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
             c += (int64_t)gridDim.x * blockDim.x) {
            const int64_t w = c / R, q = c - w * R;
            if (q >= (int64_t)__ldcg(P.ncand + 1 + w)) continue;
            const unsigned long long *e = P.cand + 3 * c;
            const int64_t b = (int64_t)e[2];
            if (e[0] == __ldcg(reinterpret_cast<const unsigned long long *>(&P.win[b].key)))
                red_max_u64(reinterpret_cast<unsigned long long *>(&P.win[b].inv), ~e[1]);
        }
        return;
    }
    RbiParams Q = P;
    Q.zero_fill = 0;  // the fallback only re-reads
    rbi_stream<T, I>(inds, as, nullptr, Q, [&](int64_t b, double x, int64_t gi, bool ok) {
        if (ok && ord_key(x, is_min) == __ldcg(reinterpret_cast<const unsigned long long *>(&P.win[b].key)))
            red_max_u64(reinterpret_cast<unsigned long long *>(&P.win[b].inv), ~(uint64_t)gi);
    });
}

// ADD primal histogram (only when hs is requested; atomic adds, order-dependent rounding)
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbi_add_hist(const I *__restrict__ inds, const T *__restrict__ as, T *hs,
                                                          RbiParams P) {
    rbi_stream<T, I>(inds, as, nullptr, P, [&](int64_t b, double x, int64_t, bool ok) {
        if (ok) atomicAdd(hs + b, (T)x);
    });
}

// ------------------------------------------------------------ return
template <class T>
struct alignas(16) MulPack {
    double q;   // hs_bar_b * p_b
    int64_t z;  // zero count
};

template <class T>
__global__ void rbi_mul_prep(const T *__restrict__ hs_bar, const double *__restrict__ p,
                             const unsigned long long *__restrict__ z, MulPack<T> *pk, int64_t m, T *hs,
                             int64_t *winners) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m; b += (int64_t)gridDim.x * blockDim.x) {
        const double pb = p[b];
        const int64_t zb = (int64_t)z[b];
        pk[b].q = (double)hs_bar[b] * pb;
        pk[b].z = zb;
        if (hs) hs[b] = (T)(zb ? 0.0 : pb);
        if (winners) winners[b] = zb;
    }
}

// ADD (gather) and MUL (three cases) return map; lane-contiguous 4-element
// groups, two slabs per iteration for 8 independent gathers in flight per lane
template <class T, class I, int OP>
__device__ __forceinline__ void rbi_bwd_map_body(const I *__restrict__ inds, const T *__restrict__ as,
                                                         const T *__restrict__ hs_bar, const MulPack<T> *__restrict__ pk,
                                                         T *__restrict__ ab, int64_t n, int64_t m, int acc, int v256) {
    const uint64_t pol = policy_evict_first();
    auto val = [&](int64_t b, double a, bool &touch) -> double {
        touch = false;
        if (b < 0 || b >= m) return 0.0;
        if (OP == VJP_ADD) {
            touch = true;
            return (double)__ldg(hs_bar + b);
        }
        const double2 k = __ldg(reinterpret_cast<const double2 *>(pk + b));
        const int64_t z = (int64_t)__double_as_longlong(k.y);
        if (z == 0) {
            touch = true;
            return k.x / a;  // hs_bar_b * y_b / a_i
        }
        touch = (z == 1 && a == 0.0);  // P:1048-1053 per bin
        return touch ? k.x : 0.0;
    };
    const int lane = threadIdx.x & 31;
    const int64_t ns = n / 128;
    const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t b[4], bn[4];
    double a[4] = {0, 0, 0, 0}, an[4] = {0, 0, 0, 0};
    if (sl < ns) {
        ld_bins4(inds, sl * 128 + lane * 4, b, pol);
        if (OP != VJP_ADD) ld_vals4(as, sl * 128 + lane * 4, a, pol, v256);
    }
    for (; sl < ns; sl += wstride) {
        const int64_t e = sl * 128 + lane * 4;
        const int64_t sn = sl + wstride;
        if (sn < ns) {  // next slab's loads in flight during this slab's gathers
            ld_bins4(inds, sn * 128 + lane * 4, bn, pol);
            if (OP != VJP_ADD) ld_vals4(as, sn * 128 + lane * 4, an, pol, v256);
        }
        double o[4] = {0, 0, 0, 0}, r[4];
        if (acc) ld_acc4(ab, e, o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            bool touch;
            const double v = val(b[q], a[q], touch);
            r[q] = acc ? (touch ? o[q] + v : o[q]) : v;
        }
        st_vals4(ab, e, r, pol, v256);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[q] = bn[q];
            a[q] = an[q];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        for (int64_t e = ns * 128 + lane; e < n; e += 32) {
            bool touch;
            const double v = val((int64_t)inds[e], OP == VJP_ADD ? 0.0 : (double)as[e], touch);
            if (acc) {
                if (touch) ab[e] = (T)((double)ab[e] + v);
            } else {
                ab[e] = (T)v;
            }
        }
    }
}
template <class T, class I, int OP>
__global__ void __launch_bounds__(kBThreads) rbi_bwd_map(const I *__restrict__ inds, const T *__restrict__ as,
                                                         const T *__restrict__ hs_bar, const MulPack<T> *__restrict__ pk,
                                                         T *__restrict__ ab, int64_t n, int64_t m, int acc, int v256) {
    rbi_bwd_map_body<T, I, OP>(inds, as, hs_bar, pk, ab, n, m, acc, v256);
}
// small per-bin tables (L1 hits): capped at 64 registers -> 4 CTAs/SM (MUL m = 1e3)
template <class T, class I, int OP>
__global__ void __launch_bounds__(kBThreads, kBMinBlocks) rbi_bwd_map_small(const I *__restrict__ inds, const T *__restrict__ as,
                                                         const T *__restrict__ hs_bar, const MulPack<T> *__restrict__ pk,
                                                         T *__restrict__ ab, int64_t n, int64_t m, int acc, int v256) {
    rbi_bwd_map_body<T, I, OP>(inds, as, hs_bar, pk, ab, n, m, acc, v256);
}

// MIN/MAX return: scatter hs_bar[b] to the winner of every bin (as_bar was
// zero-filled by the forward kernel in dense mode)
template <class T, int OP>
__global__ void rbi_ext_scatter(const Win *__restrict__ win, const T *__restrict__ hs_bar, T *__restrict__ ab,
                                int64_t m, int64_t goff, int64_t n, int acc, T *hs, int64_t *winners) {
    const bool is_min = OP == VJP_MIN;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m; b += (int64_t)gridDim.x * blockDim.x) {
        const Win w = win[b];
        const int64_t gi = w.key ? (int64_t)~w.inv : -1;
        if (winners) winners[b] = gi;
        if (hs) hs[b] = (T)(w.key ? key_val(w.key, is_min) : (is_min ? INFINITY : -INFINITY));
        if (gi >= goff && gi < goff + n) {
            T *d = ab + (gi - goff);
            *d = acc ? (T)((double)*d + (double)hs_bar[b]) : hs_bar[b];
        }
    }
}

// multi-GPU helpers -------------------------------------------------------
template <int OP>
__global__ void rbi_export(const RbiParams P, double *bin_val, int64_t *bin_aux) {
    const bool is_min = OP == VJP_MIN;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < P.m; b += (int64_t)gridDim.x * blockDim.x) {
        if (OP == VJP_MUL) {  // the bin's code sum (int64 bits; combined by integer SUM) and zero count
            reinterpret_cast<unsigned long long *>(bin_val)[b] = P.code[b];
            bin_aux[b] = (int64_t)P.z[b];
        } else {
            const Win w = P.win[b];
            bin_val[b] = w.key ? key_val(w.key, is_min) : (is_min ? INFINITY : -INFINITY);
            bin_aux[b] = w.key ? (int64_t)~w.inv : INT64_MAX;
        }
    }
}
__global__ void rbi_select(int64_t m, const double *gval, const double *lval, int64_t *aux) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m; b += (int64_t)gridDim.x * blockDim.x)
        if (!(lval[b] == gval[b])) aux[b] = INT64_MAX;  // IEEE ==: -0.0 ties +0.0
}
template <class T>
__global__ void rbi_mul_prep_ext(const T *__restrict__ hs_bar, const double *__restrict__ bin_val,
                                 const int64_t *__restrict__ bin_aux, MulPack<T> *pk, int64_t m) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m; b += (int64_t)gridDim.x * blockDim.x) {
        const double pb = mul_decode(reinterpret_cast<const unsigned long long *>(bin_val)[b]);
        pk[b].q = (double)hs_bar[b] * pb;
        pk[b].z = bin_aux[b];
    }
}
// dense MIN/MAX finish over a shard: as_bar_i = hs_bar[b_i] iff i is the bin's global winner
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbi_ext_gather(const I *__restrict__ inds, const T *__restrict__ hs_bar,
                                                            const int64_t *__restrict__ bin_aux, T *__restrict__ ab,
                                                            int64_t n, int64_t m, int64_t goff, int acc) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = (int64_t)inds[e];
        const bool won = b >= 0 && b < m && bin_aux[b] == goff + e;
        if (acc) {
            if (won) ab[e] = (T)((double)ab[e] + (double)hs_bar[b]);
        } else {
            ab[e] = won ? hs_bar[b] : (T)0;
        }
    }
}


// =============================================================================
// width > 1: vectorised operators ("elementwise"; reading A24):
// element i is the row as[i][0..w), bin b the row hs[b][0..w), and the rules
// apply per component j — (bin, component) (b, j) is an independent scalar
// bin with its own (p, z) for MUL and its own lowest-index winner for MIN/MAX.
// Rows are handled by groups of GW = min(32, pow2 >= w) lanes (no division:
// the group loops over rows, its lanes over the row's components), so a row
// of w >= 32 components is read and written coalesced.  Per-(bin, component)
// state lives in the same workspace arrays as width 1, indexed b * w + j.
// =============================================================================
struct WideGeo {
    int64_t n, m, w;
    int32_t gw, pad;  // lanes per row group
};
__device__ __forceinline__ void wide_start(const WideGeo &g, int64_t &row, int64_t &rstride, int &lane) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    row = t / g.gw;
    lane = (int)(t % g.gw);
    rstride = ((int64_t)gridDim.x * blockDim.x) / g.gw;
}

template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbiw_add_bwd(const I *__restrict__ inds, const T *__restrict__ hs_bar,
                                                          T *__restrict__ ab, WideGeo g, int acc) {
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        const bool ok = b >= 0 && b < g.m;
        for (int64_t j = lane; j < g.w; j += g.gw) {
            const double v = ok ? (double)__ldg(hs_bar + b * g.w + j) : 0.0;
            T *d = ab + i * g.w + j;
            if (acc) { if (ok) *d = (T)((double)*d + v); }
            else *d = (T)v;
        }
    }
}
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbiw_add_hist(const I *__restrict__ inds, const T *__restrict__ as,
                                                           T *__restrict__ hs, WideGeo g) {
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        if (b < 0 || b >= g.m) continue;
        for (int64_t j = lane; j < g.w; j += g.gw) atomicAdd(hs + b * g.w + j, __ldg(as + i * g.w + j));
    }
}
// MUL forward: per (bin, component) code sums and zero counts (L2 reductions)
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbiw_mul_fwd(const I *__restrict__ inds, const T *__restrict__ as,
                                                          RbiParams P, WideGeo g) {
    __shared__ Log2Tab tb;
    log2tab_load(tb);
    __syncthreads();
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        if (b < 0 || b >= g.m) continue;
        for (int64_t j = lane; j < g.w; j += g.gw) {
            const double x = (double)__ldg(as + i * g.w + j);
            if (x == 0.0) atomicAdd(P.z + b * g.w + j, 1ull);
            else atomicAdd(P.code + b * g.w + j, mul_code(x, tb));
        }
    }
}
template <class T, class I>
__global__ void __launch_bounds__(kBThreads) rbiw_mul_bwd(const I *__restrict__ inds, const T *__restrict__ as,
                                                          const MulPack<T> *__restrict__ pk, T *__restrict__ ab,
                                                          WideGeo g, int acc) {
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        const bool ok = b >= 0 && b < g.m;
        for (int64_t j = lane; j < g.w; j += g.gw) {
            const double a = (double)__ldg(as + i * g.w + j);
            double v = 0.0;
            bool touch = false;
            if (ok) {
                const double2 k = __ldg(reinterpret_cast<const double2 *>(pk + b * g.w + j));
                const int64_t z = (int64_t)__double_as_longlong(k.y);
                if (z == 0) { touch = true; v = k.x / a; }              // P:1043-1046 per (bin, component)
                else if (z == 1 && a == 0.0) { touch = true; v = k.x; }
            }
            T *d = ab + i * g.w + j;
            if (acc) { if (touch) *d = (T)((double)*d + v); }
            else *d = (T)v;
        }
    }
}
// MIN/MAX: phase A (value keys, red.max behind the monotone filter), phase B
// (lowest ELEMENT index among the elements reaching the final key), scatter
template <class T, class I, int OP>
__global__ void __launch_bounds__(kBThreads) rbiw_ext_a(const I *__restrict__ inds, const T *__restrict__ as,
                                                        RbiParams P, WideGeo g) {
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        if (b < 0 || b >= g.m) continue;
        for (int64_t j = lane; j < g.w; j += g.gw) {
            const uint64_t k = ord_key((double)__ldg(as + i * g.w + j), OP == VJP_MIN);
            unsigned long long *slot = reinterpret_cast<unsigned long long *>(&P.win[b * g.w + j].key);
            if (k > __ldcg(slot)) red_max_u64(slot, k);
        }
    }
}
template <class T, class I, int OP>
__global__ void __launch_bounds__(kBThreads) rbiw_ext_b(const I *__restrict__ inds, const T *__restrict__ as,
                                                        RbiParams P, WideGeo g) {
    int64_t i, rs;
    int lane;
    wide_start(g, i, rs, lane);
    for (; i < g.n; i += rs) {
        const int64_t b = (int64_t)__ldg(inds + i);
        if (b < 0 || b >= g.m) continue;
        for (int64_t j = lane; j < g.w; j += g.gw) {
            const uint64_t k = ord_key((double)__ldg(as + i * g.w + j), OP == VJP_MIN);
            Win *wb = P.win + b * g.w + j;
            if (k == __ldcg(reinterpret_cast<const unsigned long long *>(&wb->key)))
                red_max_u64(reinterpret_cast<unsigned long long *>(&wb->inv), ~(uint64_t)i);
        }
    }
}
template <class T, int OP>
__global__ void rbiw_ext_scatter(const Win *__restrict__ win, const T *__restrict__ hs_bar, T *__restrict__ ab,
                                 WideGeo g, int acc, T *hs, int64_t *winners) {
    const bool is_min = OP == VJP_MIN;
    const int64_t mw = g.m * g.w;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < mw; q += (int64_t)gridDim.x * blockDim.x) {
        const Win w = win[q];
        const int64_t i = w.key ? (int64_t)~w.inv : -1;  // winning element (row) of (b, j)
        if (winners) winners[q] = i;
        if (hs) hs[q] = (T)(w.key ? key_val(w.key, is_min) : (is_min ? INFINITY : -INFINITY));
        if (i >= 0) {
            T *d = ab + i * g.w + (q % g.w);
            *d = acc ? (T)((double)*d + (double)hs_bar[q]) : hs_bar[q];
        }
    }
}

}  // namespace vjpk

// =============================================================================
// host side
// =============================================================================
namespace {
using namespace vjpk;

constexpr size_t kSmemCap = 200 * 1024;
constexpr int64_t kMaxWarpsA = 65536;  // phase-A warps (per-warp candidate counts)

bool op_ok(vjp_op op) { return op == VJP_ADD || op == VJP_MUL || op == VJP_MIN || op == VJP_MAX; }

struct BLayout {
    size_t p, z, win, pk, ncand, cand, total;
    int64_t cap;
};
// candidate list capacity for MIN/MAX: ~(H(n/m) + ties) per bin are expected;
// overflow is handled (phase B re-reads the inputs)
int64_t cand_cap(int64_t n, int64_t m) {
    int64_t c = n / 16;
    if (c < 16 * m) c = 16 * m;
    if (c < (1 << 16)) c = 1 << 16;
    return c;
}
BLayout blayout(int64_t m, int64_t n = 0, bool ext = false) {
    BLayout L{};
    size_t off = 0;
    L.p = off; off += vjph::align256(sizeof(double) * (size_t)m);
    L.z = off; off += vjph::align256(sizeof(unsigned long long) * (size_t)m);
    L.win = off; off += vjph::align256(sizeof(Win) * (size_t)m);
    L.pk = off; off += vjph::align256(16 * (size_t)m);
    L.ncand = off; off += vjph::align256(8 * (1 + kMaxWarpsA));
    L.cap = ext ? cand_cap(n, m) : 0;
    L.cand = off; off += vjph::align256((size_t)L.cap * 24);
    L.total = off;
    return L;
}

int grid_for(int64_t work, int per_sm) {
    int64_t g = (work + kBThreads - 1) / kBThreads;
    int64_t cap = (int64_t)vjph::sm_count() * per_sm;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}
// persistent grid: exactly the CTAs that fit at once (one wave, no tail)
template <class K>
int grid_resident(K kernel, int64_t work, size_t smem = 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kBThreads, smem) != cudaSuccess || occ < 1) occ = 1;
    return grid_for(work, occ);
}

bool a32(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

RbiParams params(int64_t n, int64_t m, int64_t goff, void *ws, unsigned flags, int zero_fill, bool ext = false) {
    BLayout L = blayout(m, n, ext);
    unsigned char *w = static_cast<unsigned char *>(ws);
    RbiParams P{};
    P.n = n;
    P.m = m;
    P.goff = goff;
    P.acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    P.zero_fill = zero_fill;
    P.p = reinterpret_cast<double *>(w + L.p);
    P.z = reinterpret_cast<unsigned long long *>(w + L.z);
    P.win = reinterpret_cast<Win *>(w + L.win);
    P.code = reinterpret_cast<unsigned long long *>(w + L.p);  // the codes, decoded in place into p
    P.ncand = reinterpret_cast<unsigned long long *>(w + L.ncand);
    P.cand = reinterpret_cast<unsigned long long *>(w + L.cand);
    P.cap = L.cap;
    P.v256 = 0;
    return P;
}

// forward histogram (MUL / MIN / MAX), init included
template <class T, class I, int OP>
vjp_status forward(const I *inds, const T *as, T *ab, RbiParams P, cudaStream_t s, bool finalize = true) {
    const size_t sm_log = (size_t)P.m * 12;  // low word, high word, zero count
    P.log_domain = (OP == VJP_MUL) ? 1 : 0;
    rbi_init<OP><<<grid_for(P.m, 4), kBThreads, 0, s>>>(P);
    vjph::count_launch();
    const int nvec = (int)(16 / sizeof(I));
    const int64_t work = P.n / nvec + 1;
    if (OP == VJP_MUL) {
        if (sm_log <= kSmemCap) {  // small m: per-CTA shared-memory table
            const size_t sm_ring = ((sm_log + 15) & ~size_t(15)) + SlabRing<T, I, kRingFwd>::kBytes;
            int occ_ring = 0, occ_plain = 0;  // the ring only where it keeps the occupancy
            cudaFuncSetAttribute(rbi_fwd_smem_log<T, I, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sm_ring <= kSmemCap ? sm_ring : sm_log));
            cudaFuncSetAttribute(rbi_fwd_smem_log<T, I, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_log);
            if (sm_ring <= kSmemCap)
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_ring, rbi_fwd_smem_log<T, I, true>, kBThreads, sm_ring);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_plain, rbi_fwd_smem_log<T, I, false>, kBThreads, sm_log);
            if (VJP_RING_FWD > 0 && vjph::aligned16(inds) && vjph::aligned16(as) && sm_ring <= kSmemCap &&
                occ_ring >= occ_plain) {
                auto k = rbi_fwd_smem_log<T, I, true>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ring);
                k<<<grid_resident(k, work, sm_ring), kBThreads, sm_ring, s>>>(inds, as, P);
            } else {
                auto k = rbi_fwd_smem_log<T, I, false>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_log);
                k<<<grid_resident(k, work, sm_log), kBThreads, sm_log, s>>>(inds, as, P);
            }
        } else {  // large m: global reductions (L2)
            rbi_fwd_log<T, I><<<grid_resident(rbi_fwd_log<T, I>, work), kBThreads, 0, s>>>(inds, as, P);
        }
        vjph::count_launch();
        if (!finalize) return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;  // partial: export the codes
        rbi_log_finalize<<<grid_for(P.m, 4), kBThreads, 0, s>>>(P);
    } else {
        const size_t smk = sizeof(unsigned long long) * (size_t)P.m;
        int ga;
        if (smk <= 128 * 1024) {  // (the cp.async ring measured slower here: 1.09 -> 1.20 ms, DESIGN 7.6)
            auto k = rbi_ext_a<T, I, OP, true>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smk);
            ga = grid_resident(k, work, smk);
            if ((int64_t)ga * (kBThreads / 32) > kMaxWarpsA) ga = (int)(kMaxWarpsA / (kBThreads / 32));
            k<<<ga, kBThreads, smk, s>>>(inds, as, ab, P);
        } else {
            auto k = rbi_ext_a<T, I, OP, false>;
            ga = grid_resident(k, work);
            if ((int64_t)ga * (kBThreads / 32) > kMaxWarpsA) ga = (int)(kMaxWarpsA / (kBThreads / 32));
            k<<<ga, kBThreads, 0, s>>>(inds, as, ab, P);
        }
        vjph::count_launch();
        rbi_ext_b<T, I, OP><<<grid_resident(rbi_ext_b<T, I, OP>, work), kBThreads, 0, s>>>(inds, as, P,
                                                                                           (int64_t)ga * (kBThreads / 32));
    }
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

// deterministic primal sum of the rows (ADD with hs requested): the bin sort
// + in-order segmented sums of binsort.cuh, when the caller's workspace holds
// it (vjp_reduce_by_index_hs_workspace_bytes); else atomic adds
bool add_sorted_ok(int64_t n, int64_t m, size_t ws_bytes) {
    return m <= vjph::kBsMaxBins && n < ((int64_t)1 << 31) && ws_bytes >= vjph::bs_layout(n, m).total;
}
template <class T, class I>
int add_hist_sorted(const I *inds, const T *as, int64_t n, int64_t m, int64_t w, T *hs, void *ws, cudaStream_t s) {
    const vjph::BsLayout L = vjph::bs_layout(n, m);
    unsigned char *wb = static_cast<unsigned char *>(ws);
    int k = vjph::bs_sort<I>(inds, n, m, L, wb, nullptr, 0, s);
    k += vjph::bs_rowsum<T>(as, nullptr, m, w, 1.0, nullptr, L, wb, hs, nullptr, 0, s);
    return k;
}

template <class T, class I>
vjp_status run_full(vjp_op op, int64_t n, int64_t m, const void *inds_, const void *as_, const void *hsb_, void *ab_,
                    void *hs_, int64_t *winners, void *ws, size_t ws_bytes, cudaStream_t s, unsigned flags) {
    const I *inds = static_cast<const I *>(inds_);
    const T *as = static_cast<const T *>(as_);
    const T *hsb = static_cast<const T *>(hsb_);
    T *ab = static_cast<T *>(ab_);
    T *hs = static_cast<T *>(hs_);
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    const int nvec = (int)(16 / sizeof(I));
    if (op == VJP_ADD) {
        if (hs && add_sorted_ok(n, m, ws_bytes)) {
            vjph::count_launch(add_hist_sorted<T, I>(inds, as, n, m, 1, hs, ws, s));
        } else if (hs) {
            // primal histogram on request, atomic adds (order-dependent rounding)
            if (cudaMemsetAsync(hs, 0, sizeof(T) * (size_t)m, s) != cudaSuccess) return VJP_ECUDA;
            RbiParams P = params(n, m, 0, ws, 0, 0);
            P.v256 = a32(as);
            rbi_add_hist<T, I><<<grid_for(n / nvec + 1, 8), kBThreads, 0, s>>>(inds, as, hs, P);
            vjph::count_launch();
        }
        rbi_bwd_map<T, I, VJP_ADD><<<grid_resident(rbi_bwd_map<T, I, VJP_ADD>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, nullptr, ab, n, m, acc, (int)((!as || a32(as)) && a32(ab)));
        vjph::count_launch();
        if (cudaGetLastError() != cudaSuccess) return VJP_ECUDA;
        if (winners && cudaMemsetAsync(winners, 0xff, sizeof(int64_t) * (size_t)m, s) != cudaSuccess) return VJP_ECUDA;
        return VJP_OK;
    }
    // dense MIN/MAX: as_bar = 0 except the winners; the scatter below
    // overwrites the m winners.  Small m (shared-memory filter, latency bound):
    // a plain memset first (fusing the stores slowed phase A, DESIGN 7.6);
    // large m (L2 bound): phase A stores the zeros while it streams the bins
    const bool fuse_zero = op != VJP_MUL && !acc && (size_t)m * 8 > 128 * 1024;
    if (op != VJP_MUL && !acc && !fuse_zero && cudaMemsetAsync(ab, 0, sizeof(T) * (size_t)n, s) != cudaSuccess)
        return VJP_ECUDA;
    RbiParams P = params(n, m, 0, ws, flags, fuse_zero ? 1 : 0, op != VJP_MUL);
    P.v256 = a32(as) && a32(ab);
    vjp_status st = VJP_OK;
    if (op == VJP_MUL) st = forward<T, I, VJP_MUL>(inds, as, ab, P, s);
    if (op == VJP_MIN) st = forward<T, I, VJP_MIN>(inds, as, ab, P, s);
    if (op == VJP_MAX) st = forward<T, I, VJP_MAX>(inds, as, ab, P, s);
    if (st != VJP_OK) return st;
    BLayout L = blayout(m);
    if (op == VJP_MUL) {
        MulPack<T> *pk = reinterpret_cast<MulPack<T> *>(static_cast<unsigned char *>(ws) + L.pk);
        rbi_mul_prep<T><<<grid_for(m, 4), kBThreads, 0, s>>>(hsb, P.p, P.z, pk, m, hs, winners);
        if (m <= kSmallM)  // small table (L1 hits): 4 CTAs/SM hide the stream latency
            rbi_bwd_map_small<T, I, VJP_MUL><<<grid_resident(rbi_bwd_map_small<T, I, VJP_MUL>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, pk, ab, n, m, acc, (int)(a32(as) && a32(ab)));
        else
            rbi_bwd_map<T, I, VJP_MUL><<<grid_resident(rbi_bwd_map<T, I, VJP_MUL>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, pk, ab, n, m, acc, (int)(a32(as) && a32(ab)));
        vjph::count_launch(2);
    } else if (op == VJP_MIN) {
        rbi_ext_scatter<T, VJP_MIN><<<grid_for(m, 4), kBThreads, 0, s>>>(P.win, hsb, ab, m, 0, n, acc, hs, winners);
        vjph::count_launch();
    } else {
        rbi_ext_scatter<T, VJP_MAX><<<grid_for(m, 4), kBThreads, 0, s>>>(P.win, hsb, ab, m, 0, n, acc, hs, winners);
        vjph::count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class T, class I>
vjp_status run_partial(vjp_op op, int64_t n, int64_t m, int64_t goff, const void *inds, const void *as, void *ws,
                       double *bin_val, int64_t *bin_aux, cudaStream_t s) {
    RbiParams P = params(n, m, goff, ws, 0, 0, op != VJP_MUL);
    P.v256 = a32(as);
    vjp_status st = VJP_OK;
    const I *ix = static_cast<const I *>(inds);
    const T *a = static_cast<const T *>(as);
    if (op == VJP_MUL) st = forward<T, I, VJP_MUL>(ix, a, nullptr, P, s, false);
    if (op == VJP_MIN) st = forward<T, I, VJP_MIN>(ix, a, nullptr, P, s);
    if (op == VJP_MAX) st = forward<T, I, VJP_MAX>(ix, a, nullptr, P, s);
    if (st != VJP_OK) return st;
    if (op == VJP_MUL) rbi_export<VJP_MUL><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux);
    if (op == VJP_MIN) rbi_export<VJP_MIN><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux);
    if (op == VJP_MAX) rbi_export<VJP_MAX><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

template <class T, class I>
vjp_status run_finish(vjp_op op, int64_t n, int64_t m, int64_t goff, const void *inds_, const void *as_,
                      const void *hsb_, void *ab_, const double *bin_val, const int64_t *bin_aux, void *ws,
                      cudaStream_t s, unsigned flags) {
    const I *inds = static_cast<const I *>(inds_);
    const T *as = static_cast<const T *>(as_);
    const T *hsb = static_cast<const T *>(hsb_);
    T *ab = static_cast<T *>(ab_);
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    const int nvec = (int)(16 / sizeof(I));
    if (op == VJP_ADD) {
        rbi_bwd_map<T, I, VJP_ADD><<<grid_resident(rbi_bwd_map<T, I, VJP_ADD>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, nullptr, ab, n, m, acc, (int)((!as || a32(as)) && a32(ab)));
    } else if (op == VJP_MUL) {
        BLayout L = blayout(m, n, false);
        MulPack<T> *pk = reinterpret_cast<MulPack<T> *>(static_cast<unsigned char *>(ws) + L.pk);
        rbi_mul_prep_ext<T><<<grid_for(m, 4), kBThreads, 0, s>>>(hsb, bin_val, bin_aux, pk, m);
        vjph::count_launch();
        if (m <= kSmallM)  // small table (L1 hits): 4 CTAs/SM hide the stream latency
            rbi_bwd_map_small<T, I, VJP_MUL><<<grid_resident(rbi_bwd_map_small<T, I, VJP_MUL>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, pk, ab, n, m, acc, (int)(a32(as) && a32(ab)));
        else
            rbi_bwd_map<T, I, VJP_MUL><<<grid_resident(rbi_bwd_map<T, I, VJP_MUL>, n / 4 + 1), kBThreads, 0, s>>>(inds, as, hsb, pk, ab, n, m, acc, (int)(a32(as) && a32(ab)));
    } else {
        rbi_ext_gather<T, I><<<grid_for(n, 8), kBThreads, 0, s>>>(inds, hsb, bin_aux, ab, n, m, goff, acc);
    }
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}


// width > 1 (vectorised operators, reading A24): per-(bin, component) state
// in the width-1 workspace layout with m * width bins
WideGeo wide_geo(int64_t n, int64_t m, int64_t w) {
    WideGeo g{};
    g.n = n;
    g.m = m;
    g.w = w;
    int gw = 1;
    while (gw < w && gw < 32) gw <<= 1;
    g.gw = gw;
    return g;
}
int grid_wide(const WideGeo &g) {
    int64_t rows_per_cta = kBThreads / g.gw;
    int64_t b = (g.n + rows_per_cta - 1) / rows_per_cta;
    int64_t cap = (int64_t)vjph::sm_count() * 8;
    if (b > cap) b = cap;
    return (int)(b < 1 ? 1 : b);
}
template <class T, class I>
vjp_status run_wide(vjp_op op, int64_t n, int64_t m, int64_t w, const void *inds_, const void *as_,
                    const void *hsb_, void *ab_, void *hs_, int64_t *winners, void *ws, size_t ws_bytes,
                    cudaStream_t s, unsigned flags) {
    const I *inds = static_cast<const I *>(inds_);
    const T *as = static_cast<const T *>(as_);
    const T *hsb = static_cast<const T *>(hsb_);
    T *ab = static_cast<T *>(ab_);
    T *hs = static_cast<T *>(hs_);
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    const WideGeo g = wide_geo(n, m, w);
    const int grid = grid_wide(g);
    const int64_t mw = m * w;
    if (op == VJP_ADD) {
        if (hs && add_sorted_ok(n, m, ws_bytes)) {
            vjph::count_launch(add_hist_sorted<T, I>(inds, as, n, m, w, hs, ws, s));
        } else if (hs) {
            if (cudaMemsetAsync(hs, 0, sizeof(T) * (size_t)mw, s) != cudaSuccess) return VJP_ECUDA;
            rbiw_add_hist<T, I><<<grid, kBThreads, 0, s>>>(inds, as, hs, g);
            vjph::count_launch();
        }
        rbiw_add_bwd<T, I><<<grid, kBThreads, 0, s>>>(inds, hsb, ab, g, acc);
        vjph::count_launch();
        if (winners && cudaMemsetAsync(winners, 0xff, sizeof(int64_t) * (size_t)mw, s) != cudaSuccess) return VJP_ECUDA;
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    RbiParams P = params(n, mw, 0, ws, flags, 0, false);
    const int gm = grid_for(mw, 4);
    if (op == VJP_MUL) {
        P.log_domain = 1;
        rbi_init<VJP_MUL><<<gm, kBThreads, 0, s>>>(P);
        rbiw_mul_fwd<T, I><<<grid, kBThreads, 0, s>>>(inds, as, P, g);
        rbi_log_finalize<<<gm, kBThreads, 0, s>>>(P);
        BLayout L = blayout(mw);
        MulPack<T> *pk = reinterpret_cast<MulPack<T> *>(static_cast<unsigned char *>(ws) + L.pk);
        rbi_mul_prep<T><<<gm, kBThreads, 0, s>>>(hsb, P.p, P.z, pk, mw, hs, winners);
        rbiw_mul_bwd<T, I><<<grid, kBThreads, 0, s>>>(inds, as, pk, ab, g, acc);
        vjph::count_launch(5);
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    if (!acc && cudaMemsetAsync(ab, 0, sizeof(T) * (size_t)(n * w), s) != cudaSuccess) return VJP_ECUDA;
    if (op == VJP_MIN) {
        rbi_init<VJP_MIN><<<gm, kBThreads, 0, s>>>(P);
        rbiw_ext_a<T, I, VJP_MIN><<<grid, kBThreads, 0, s>>>(inds, as, P, g);
        rbiw_ext_b<T, I, VJP_MIN><<<grid, kBThreads, 0, s>>>(inds, as, P, g);
        rbiw_ext_scatter<T, VJP_MIN><<<gm, kBThreads, 0, s>>>(P.win, hsb, ab, g, acc, hs, winners);
    } else {
        rbi_init<VJP_MAX><<<gm, kBThreads, 0, s>>>(P);
        rbiw_ext_a<T, I, VJP_MAX><<<grid, kBThreads, 0, s>>>(inds, as, P, g);
        rbiw_ext_b<T, I, VJP_MAX><<<grid, kBThreads, 0, s>>>(inds, as, P, g);
        rbiw_ext_scatter<T, VJP_MAX><<<gm, kBThreads, 0, s>>>(P.win, hsb, ab, g, acc, hs, winners);
    }
    vjph::count_launch(4);
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

vjp_status common_check(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, const void *inds,
                        const void *as, const void *hs_bar) {
    if (op == VJP_LINREC || op == VJP_MAT2) return VJP_EUNSUPPORTED;  // no rule in the paper
    if (!op_ok(op) || (dtype != VJP_F32 && dtype != VJP_F64) || (itype != VJP_I32 && itype != VJP_I64)) return VJP_EINVAL;
    if (n < 0 || m < 1) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    if (!inds || !hs_bar || (!as && op != VJP_ADD)) return VJP_EINVAL;
    const void *ps[3] = {inds, as, hs_bar};
    for (const void *p : ps)
        if (p && !vjph::aligned16(p)) return VJP_EALIGN;
    return VJP_OK;
}

#define RBI_DISPATCH(FN, ...)                                                                        \
    (dtype == VJP_F64 ? (itype == VJP_I32 ? FN<double, int32_t>(__VA_ARGS__) : FN<double, int64_t>(__VA_ARGS__)) \
                      : (itype == VJP_I32 ? FN<float, int32_t>(__VA_ARGS__) : FN<float, int64_t>(__VA_ARGS__)))
}  // namespace

extern "C" {

// test hook for the MUL codes: code[i] = code(x[i]) by the kernels' routine
vjp_status vjp_debug_mul_code(const double *x, int64_t *code, int64_t n, vjp_stream_t stream) {
    if (n < 0 || (n > 0 && (!x || !code))) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    vjpk::rbi_code_probe<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        x, reinterpret_cast<unsigned long long *>(code), n);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}


size_t vjp_reduce_by_index_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m, int64_t width) {
    (void)dtype;
    if (!op_ok(op) || m < 1 || n < 0 || width < 1) return 0;
    if (op == VJP_ADD) return 0;
    if (width > 1) return blayout(m * width, 0, false).total;
    return blayout(m, n, op != VJP_MUL).total;
}

size_t vjp_reduce_by_index_hs_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m, int64_t width) {
    const size_t base = vjp_reduce_by_index_workspace_bytes(op, dtype, n, m, width);
    if (op != VJP_ADD || m < 1 || n < 0 || width < 1 || m > vjph::kBsMaxBins || n >= ((int64_t)1 << 31)) return base;
    const size_t srt = vjph::bs_layout(n, m).total;
    return srt > base ? srt : base;
}

vjp_status vjp_reduce_by_index(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *inds, const void *as, const void *hs_bar, void *as_bar, void *hs,
                               int64_t *winners, void *ws, size_t ws_bytes, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_reduce_by_index");
    if (width < 1) return VJP_EINVAL;
    vjp_status st = common_check(op, dtype, itype, n, m, inds, as, hs_bar);
    if (st != VJP_OK || n == 0) return st;
    if (!as_bar) return VJP_EINVAL;
    if (!vjph::aligned16(as_bar)) return VJP_EALIGN;
    if (op == VJP_ADD && hs && !as) return VJP_EINVAL;  // the primal sum needs `as`
    const size_t need = vjp_reduce_by_index_workspace_bytes(op, dtype, n, m, width);
    if (ws_bytes < need || (need && !ws)) return VJP_EWORKSPACE;
    if (ws && !vjph::aligned16(ws)) return VJP_EALIGN;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (width > 1)
        return RBI_DISPATCH(run_wide, op, n, m, width, inds, as, hs_bar, as_bar, hs, winners, ws, ws_bytes, s, flags);
    return RBI_DISPATCH(run_full, op, n, m, inds, as, hs_bar, as_bar, hs, winners, ws, ws_bytes, s, flags);
}

vjp_status vjp_reduce_by_index_partial(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m,
                                       const void *inds, const void *as, void *ws, size_t ws_bytes,
                                       const vjp_shard *shard, double *bin_val, int64_t *bin_aux,
                                       vjp_stream_t stream) {
    VJP_NVTX("vjp_reduce_by_index_partial");
    if (!shard) return VJP_EINVAL;
    if (op == VJP_ADD) return op_ok(op) ? VJP_OK : VJP_EINVAL;
    vjp_status st = common_check(op, dtype, itype, n, m, inds, as, inds);
    if (st != VJP_OK) return st;
    if (!bin_val || !bin_aux) return VJP_EINVAL;
    if (ws_bytes < blayout(m, n, op != VJP_MUL).total || !ws) return VJP_EWORKSPACE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n == 0) {
        // empty shard: neutral per-bin state
        RbiParams P = params(0, m, shard->global_offset, ws, 0, 0, op != VJP_MUL);
        if (op == VJP_MUL) { rbi_init<VJP_MUL><<<grid_for(m, 4), kBThreads, 0, s>>>(P); rbi_export<VJP_MUL><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux); }
        if (op == VJP_MIN) { rbi_init<VJP_MIN><<<grid_for(m, 4), kBThreads, 0, s>>>(P); rbi_export<VJP_MIN><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux); }
        if (op == VJP_MAX) { rbi_init<VJP_MAX><<<grid_for(m, 4), kBThreads, 0, s>>>(P); rbi_export<VJP_MAX><<<grid_for(m, 4), kBThreads, 0, s>>>(P, bin_val, bin_aux); }
        vjph::count_launch(2);
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    return RBI_DISPATCH(run_partial, op, n, m, shard->global_offset, inds, as, ws, bin_val, bin_aux, s);
}

vjp_status vjp_reduce_by_index_select(vjp_op op, int64_t m, const double *bin_val_global, const double *bin_val_local,
                                      int64_t *bin_aux, vjp_stream_t stream) {
    if ((op != VJP_MIN && op != VJP_MAX) || m < 1 || !bin_val_global || !bin_val_local || !bin_aux) return VJP_EINVAL;
    rbi_select<<<grid_for(m, 4), kBThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(m, bin_val_global,
                                                                                         bin_val_local, bin_aux);
    vjph::count_launch();
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

vjp_status vjp_reduce_by_index_finish(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m,
                                      const void *inds, const void *as, const void *hs_bar, void *as_bar,
                                      const double *bin_val, const int64_t *bin_aux, void *ws, size_t ws_bytes,
                                      const vjp_shard *shard, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_reduce_by_index_finish");
    if (!shard) return VJP_EINVAL;
    vjp_status st = common_check(op, dtype, itype, n, m, inds, as, hs_bar);
    if (st != VJP_OK || n == 0) return st;
    if (!as_bar) return VJP_EINVAL;
    if (!vjph::aligned16(as_bar)) return VJP_EALIGN;
    if (op != VJP_ADD && (!bin_val || !bin_aux)) return VJP_EINVAL;
    const size_t need = vjp_reduce_by_index_workspace_bytes(op, dtype, n, m, 1);
    if (ws_bytes < need || (need && !ws)) return VJP_EWORKSPACE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return RBI_DISPATCH(run_finish, op, n, m, shard->global_offset, inds, as, hs_bar, as_bar, bin_val, bin_aux, ws,
                        s, flags);
}

}  // extern "C"
