// kmeans.cu — composite k-means cost gradient (BASELINE
// config 5) for sm_100a.
//
//   f(C) = sum_p min_j ||p - c_j||^2        (reading R15: squared distance)
//
// Forward (compute bound, FP64 FMA):
//   km_cnorm   ||c_j||^2
//   km_assign  register-tiled distance expansion ||c_j||^2 - 2 p.c_j per point
//              and center (128 points x 64 centers per CTA, 8 x 8 per thread,
//              smem tiles of 32 dimensions), the FIRST-index argmin per point
//               and the per-point minimum distance (cost).
// Return sweep with cost_bar = ybar (vjp; P:1034-1038 for the sum over points,
// P:1071-1087 for the min's sparse adjoint — only dist(p, a(p)) gets ybar —
// and the map's vjp 2 (c_a - p)), its accumulation per center being a
// reduce_by_index(+) of width d into k bins: realised as a
// STABLE counting sort of the points by center followed by an in-order
// segmented sum, so the result is deterministic (no floating-point atomics):
//   km_hist      per block of 4096 points, per-center counts (smem 32-bit atomics)
//   km_colscan   per center, exclusive scan over the blocks (column of the table)
//   km_startscan exclusive scan of the per-center totals -> segment starts
//   km_order     stable ranks (warp match_any per 32 points, in index order)
//                -> order[] = point indices grouped by center, increasing
//   km_segsum    one CTA per center: C_bar_j = 2 ybar sum_{p in j} (c_j - p),
//                each warp a contiguous quarter of the index-ordered segment
//                (rows gathered 16 at a time, coalesced per row), partials
//                added in warp order (deterministic);
//                Hessian diagonal (jvp of the vjp, all-ones direction,
//                P:1696-1700) H_j = 2 ybar cnt_j.
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "binsort.cuh"

namespace vjpk {

constexpr int KM_BP = 128;   // points per assign CTA
constexpr int KM_BC = 64;    // centers per tile
constexpr int KM_KD = 32;    // dimensions per smem stage
constexpr int KM_NT = 128;   // assign threads (16 x 8 grid of 8 x 8 tiles)
constexpr int KM_BH = 1024;  // points per histogram / ordering block
constexpr int KM_SEGB = 16;  // rows gathered per batch in km_segsum

// position of point pp (0..127) / center cc (0..63) in the swizzled smem rows:
// thread tp owns points tp*8 .. tp*8+7 and reads them as 4 x 16 B at
// q*32 + tp*2 (conflict free); thread tc owns centers tc*8 .. tc*8+7 at q*16 + tc*2
__device__ __forceinline__ int km_ppos(int pp) { return ((pp & 7) >> 1) * 32 + (pp >> 3) * 2 + (pp & 1); }
__device__ __forceinline__ int km_cpos(int cc) { return ((cc & 7) >> 1) * 16 + (cc >> 3) * 2 + (cc & 1); }

template <class T>
__global__ void km_cnorm(const T *__restrict__ C, int64_t k, int64_t d, double *__restrict__ cn) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    double s = 0.0;
    for (int64_t t = 0; t < d; ++t) {
        const double v = (double)C[j * d + t];
        s = fma(v, v, s);
    }
    cn[j] = s;
}

// one element of a stage: f64 by an 8-byte cp.async (zero-filled when out of
// range), f32 through a register (converted to f64)
__device__ __forceinline__ void km_stage(double *dst, const double *src, bool ok) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(ok ? src : nullptr), "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void km_stage(double *dst, const float *src, bool ok) { *dst = ok ? (double)*src : 0.0; }
// two f64 elements by one 16-byte cp.async.cg (even d, 16-byte aligned rows)
__device__ __forceinline__ void km_stage16(double *dst, const double *src, bool ok) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(ok ? src : nullptr), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void km_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void km_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Dynamic shared memory: Ps [DP][128] point tile (dim-major, swizzled), resident
// for the whole CTA when d <= 64 (DP = d rounded up to 32), else one 32-dim
// chunk re-staged per stage; Cs [2][32][64] double-buffered center chunks.
// Stage s = (center tile s / nd, dim chunk s % nd), prefetched one ahead.
template <class T, bool RES>
__global__ void __launch_bounds__(KM_NT, 2) km_assign(const T *__restrict__ P, const T *__restrict__ C,
                                                      const double *__restrict__ cn, int64_t n, int64_t k,
                                                      int64_t d, int32_t *__restrict__ assign,
                                                      double *__restrict__ cost_part) {
    extern __shared__ __align__(16) double km_smem[];
    const int nd = (int)((d + KM_KD - 1) / KM_KD);
    const int DP = RES ? nd * KM_KD : 2 * KM_KD;        // rows of Ps
    double *Ps = km_smem;                                // [DP][KM_BP]
    double *Cs = km_smem + (size_t)DP * KM_BP;           // [2][KM_KD][KM_BC]
    const int t = threadIdx.x, tp = t & 15, tc = t >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * KM_BP;
    const int nct = (int)((k + KM_BC - 1) / KM_BC), nst = nct * nd;

    auto stage = [&](int st) {
        const int ct = st / nd, dc = st % nd, buf = st & 1;
        const int64_t c0 = (int64_t)ct * KM_BC, d0 = (int64_t)dc * KM_KD;
        double *cs = Cs + (size_t)buf * KM_KD * KM_BC;
#pragma unroll 4
        for (int idx = t; idx < KM_BC * KM_KD; idx += KM_NT) {
            const int cc = idx / KM_KD, kk = idx % KM_KD;
            const int64_t gc = c0 + cc, gd = d0 + kk;
            const bool ok = gc < k && gd < d;
            km_stage(cs + kk * KM_BC + km_cpos(cc), C + (ok ? gc * d + gd : 0), ok);
        }
        if (!RES) {
            double *ps = Ps + (size_t)buf * KM_KD * KM_BP;
#pragma unroll 4
            for (int idx = t; idx < KM_BP * KM_KD; idx += KM_NT) {
                const int pp = idx / KM_KD, kk = idx % KM_KD;
                const int64_t gp = p0 + pp, gd = d0 + kk;
                const bool ok = gp < n && gd < d;
                km_stage(ps + kk * KM_BP + km_ppos(pp), P + (ok ? gp * d + gd : 0), ok);
            }
        }
        km_commit();
    };

    if (RES) {  // the whole point tile, once
#pragma unroll 4
        for (int idx = t; idx < KM_BP * DP; idx += KM_NT) {
            const int pp = idx / DP, kk = idx % DP;
            const int64_t gp = p0 + pp;
            const bool ok = gp < n && kk < d;
            km_stage(Ps + kk * KM_BP + km_ppos(pp), P + (ok ? gp * d + kk : 0), ok);
        }
    }
    stage(0);  // (commits the resident tile with it)

    double bv[8];
    int32_t bj[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        bv[i] = INFINITY;
        bj[i] = 0x7fffffff;
    }
    double pnorm = 0.0;  // ||p_{p0+t}||^2, accumulated during center tile 0
    double acc[8][8];
    for (int st = 0; st < nst; ++st) {
        const int ct = st / nd, dc = st % nd;
        if (dc == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
        }
        if (st + 1 < nst) {
            __syncthreads();  // buffer (st+1)&1 was consumed at stage st-1
            stage(st + 1);
            km_wait<1>();
        } else {
            km_wait<0>();
        }
        __syncthreads();
        const double *ps = RES ? Ps + (size_t)dc * KM_KD * KM_BP : Ps + (size_t)(st & 1) * KM_KD * KM_BP;
        const double *cs = Cs + (size_t)(st & 1) * KM_KD * KM_BC;
        if (ct == 0) {
#pragma unroll 8
            for (int kk = 0; kk < KM_KD; ++kk) {
                const double v = ps[kk * KM_BP + km_ppos(t)];
                pnorm = fma(v, v, pnorm);
            }
        }
#pragma unroll 2
        for (int kk = 0; kk < KM_KD; ++kk) {
            double a[8], b[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double2 va = *reinterpret_cast<const double2 *>(ps + kk * KM_BP + q * 32 + tp * 2);
                const double2 vb = *reinterpret_cast<const double2 *>(cs + kk * KM_BC + q * 16 + tc * 2);
                a[2 * q] = va.x;
                a[2 * q + 1] = va.y;
                b[2 * q] = vb.x;
                b[2 * q + 1] = vb.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (dc == nd - 1) {
            // candidates: ||c_j||^2 - 2 p.c_j (||p||^2 is common to a point's candidates)
            const int64_t c0 = (int64_t)ct * KM_BC;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t gc = c0 + tc * 8 + j;
                if (gc < k) {
                    const double cnj = cn[gc];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const double v = fma(-2.0, acc[i][j], cnj);
                        if (v < bv[i] || (v == bv[i] && (int32_t)gc < bj[i])) {
                            bv[i] = v;
                            bj[i] = (int32_t)gc;
                        }
                    }
                }
            }
        }
    }
    // combine the 8 center columns of each point (first index on ties);
    // the epilogue scratch reuses the center buffers
    __syncthreads();
    double *rv = Cs;                                        // [8][128]
    int32_t *rj = reinterpret_cast<int32_t *>(Cs + 8 * KM_BP);  // [8][128]
    double *pn = Cs + 12 * KM_BP;                           // [128]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        rv[tc * KM_BP + tp * 8 + i] = bv[i];
        rj[tc * KM_BP + tp * 8 + i] = bj[i];
    }
    pn[t] = pnorm;
    __syncthreads();
    double md = 0.0;
    {
        const int pp = t;  // one point per thread
        double v = rv[pp];
        int32_t j = rj[pp];
#pragma unroll
        for (int c = 1; c < 8; ++c) {
            const double w = rv[c * KM_BP + pp];
            const int32_t jw = rj[c * KM_BP + pp];
            if (w < v || (w == v && jw < j)) {
                v = w;
                j = jw;
            }
        }
        const int64_t gp = p0 + pp;
        // no candidate compared smaller (NaN coordinates, or every distance
        // +inf): the first center, as the oracle's strict-compare loop keeps it
        // (the assignment indexes the per-center tables: never out of range)
        if (j < 0 || j >= k) j = 0;
        if (gp < n) {
            assign[gp] = j;
            md = fmax(pn[pp] + v, 0.0);
        }
    }
    // per-CTA cost partial, fixed order (deterministic)
    for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
    __syncthreads();
    if ((t & 31) == 0) rv[t >> 5] = md;
    __syncthreads();
    if (t == 0) cost_part[blockIdx.x] = ((rv[0] + rv[1]) + rv[2]) + rv[3];
}

// ---------------------------------------------------------------------------
// DMMA variant (mma.sync m8n8k4 f64, FP64 tensor cores): CTA = 128 points x
// 64 centers, warp w = points [32w, 32w + 32) x 64 centers = 4 x 8 tiles of
// 8 x 8; row-major smem tiles with a row stride = 4 (mod 16) doubles so the
// A/B fragment loads (8 rows x 4 consecutive doubles) are conflict free.
// Same candidate rule (||c||^2 - 2 p.c, first index on ties) as km_assign.
constexpr int KM_PS_PAD = 4;
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int KM_MMA_NT = 256;  // 8 warps: 4 point groups x 2 center halves

template <class T, bool RES, bool V16 = false>
__global__ void __launch_bounds__(KM_MMA_NT, 2) km_assign_mma(const T *__restrict__ P, const T *__restrict__ C,
                                                              const double *__restrict__ cn, int64_t n, int64_t k,
                                                              int64_t d, int32_t *__restrict__ assign,
                                                              double *__restrict__ cost_part) {
    extern __shared__ __align__(16) double km_smem[];
    const int nd = (int)((d + KM_KD - 1) / KM_KD);
    const int PW = (RES ? nd * KM_KD : KM_KD) + KM_PS_PAD;  // P row stride (doubles)
    constexpr int CW = KM_KD + KM_PS_PAD;                    // C row stride
    double *Ps = km_smem;                                    // RES: [128][PW]; else [2][128][PW]
    double *Cs = km_smem + (size_t)(RES ? 1 : 2) * KM_BP * PW;  // [2][64][CW]
    const int t = threadIdx.x, lane = t & 31, w = t >> 5, g = lane >> 2, tig = lane & 3;
    const int pg = w >> 1, ch = w & 1;  // warp: points [32 pg, 32 pg + 32) x centers [32 ch, 32 ch + 32) of the tile
    const int64_t p0 = (int64_t)blockIdx.x * KM_BP;
    const int nct = (int)((k + KM_BC - 1) / KM_BC), nst = nct * nd;

    auto stage = [&](int st) {
        const int ct = st / nd, dc = st % nd, buf = st & 1;
        const int64_t c0 = (int64_t)ct * KM_BC, d0 = (int64_t)dc * KM_KD;
        double *cs = Cs + (size_t)buf * KM_BC * CW;
        if constexpr (V16) {
#pragma unroll 2
            for (int idx = t; idx < KM_BC * KM_KD / 2; idx += KM_MMA_NT) {
                const int cc = idx / (KM_KD / 2), kk = 2 * (idx % (KM_KD / 2));
                const int64_t gc = c0 + cc, gd = d0 + kk;
                const bool ok = gc < k && gd < d;
                km_stage16(cs + cc * CW + kk, reinterpret_cast<const double *>(C) + (ok ? gc * d + gd : 0), ok);
            }
        } else {
#pragma unroll 2
            for (int idx = t; idx < KM_BC * KM_KD; idx += KM_MMA_NT) {
                const int cc = idx / KM_KD, kk = idx % KM_KD;
                const int64_t gc = c0 + cc, gd = d0 + kk;
                const bool ok = gc < k && gd < d;
                km_stage(cs + cc * CW + kk, C + (ok ? gc * d + gd : 0), ok);
            }
        }
        if (!RES) {
            double *ps = Ps + (size_t)buf * KM_BP * PW;
#pragma unroll 2
            for (int idx = t; idx < KM_BP * KM_KD; idx += KM_MMA_NT) {
                const int pp = idx / KM_KD, kk = idx % KM_KD;
                const int64_t gp = p0 + pp, gd = d0 + kk;
                const bool ok = gp < n && gd < d;
                km_stage(ps + pp * PW + kk, P + (ok ? gp * d + gd : 0), ok);
            }
        }
        km_commit();
    };
    if (RES) {
        const int DP = nd * KM_KD;
        if constexpr (V16) {
#pragma unroll 4
            for (int idx = t; idx < KM_BP * DP / 2; idx += KM_MMA_NT) {
                const int pp = idx / (DP / 2), kk = 2 * (idx % (DP / 2));
                const int64_t gp = p0 + pp;
                const bool ok = gp < n && kk < d;
                km_stage16(Ps + pp * PW + kk, reinterpret_cast<const double *>(P) + (ok ? gp * d + kk : 0), ok);
            }
        } else {
#pragma unroll 4
            for (int idx = t; idx < KM_BP * DP; idx += KM_MMA_NT) {
                const int pp = idx / DP, kk = idx % DP;
                const int64_t gp = p0 + pp;
                const bool ok = gp < n && kk < d;
                km_stage(Ps + pp * PW + kk, P + (ok ? gp * d + kk : 0), ok);
            }
        }
    }
    stage(0);

    double bv[4];
    int32_t bj[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        bv[i] = INFINITY;
        bj[i] = 0x7fffffff;
    }
    double pnorm = 0.0;  // threads t < 128: ||p_{p0 + t}||^2
    double acc[4][4][2];
    for (int st = 0; st < nst; ++st) {
        const int ct = st / nd, dc = st % nd;
        if (dc == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        }
        if (st + 1 < nst) {
            __syncthreads();
            stage(st + 1);
            km_wait<1>();
        } else {
            km_wait<0>();
        }
        __syncthreads();
        const double *ps = RES ? Ps + dc * KM_KD : Ps + (size_t)(st & 1) * KM_BP * PW;
        const double *cs = Cs + (size_t)(st & 1) * KM_BC * CW;
        if (ct == 0 && t < KM_BP) {
#pragma unroll 8
            for (int kk = 0; kk < KM_KD; ++kk) {
                const double v = ps[t * PW + kk];
                pnorm = fma(v, v, pnorm);
            }
        }
#pragma unroll 4
        for (int k4 = 0; k4 < KM_KD; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = ps[(pg * 32 + mi * 8 + g) * PW + k4 + tig];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = cs[(ch * 32 + ni * 8 + g) * CW + k4 + tig];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        if (dc == nd - 1) {
            const int64_t c0 = (int64_t)ct * KM_BC + ch * 32;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t gc = c0 + ni * 8 + tig * 2 + e;
                    if (gc < k) {
                        const double cnj = cn[gc];
#pragma unroll
                        for (int mi = 0; mi < 4; ++mi) {
                            const double v = fma(-2.0, acc[mi][ni][e], cnj);
                            if (v < bv[mi] || (v == bv[mi] && (int32_t)gc < bj[mi])) {
                                bv[mi] = v;
                                bj[mi] = (int32_t)gc;
                            }
                        }
                    }
                }
        }
    }
    // the 4 threads of a group share their points: combine (first index on ties)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv[mi], o);
            const int32_t oj = __shfl_xor_sync(0xffffffffu, bj[mi], o);
            if (ov < bv[mi] || (ov == bv[mi] && oj < bj[mi])) {
                bv[mi] = ov;
                bj[mi] = oj;
            }
        }
    __syncthreads();
    double *pn = Cs;                                                    // [128]
    double *hv = Cs + KM_BP;                                            // [2][128] per center half
    int32_t *hj = reinterpret_cast<int32_t *>(Cs + 3 * KM_BP);          // [2][128]
    if (t < KM_BP) pn[t] = pnorm;
    if (tig == 0) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int pp = pg * 32 + mi * 8 + g;
            hv[ch * KM_BP + pp] = bv[mi];
            hj[ch * KM_BP + pp] = bj[mi];
        }
    }
    __syncthreads();
    double md = 0.0;
    if (t < KM_BP) {
        double v = hv[t];
        int32_t j = hj[t];
        const double v1 = hv[KM_BP + t];
        const int32_t j1 = hj[KM_BP + t];
        if (v1 < v || (v1 == v && j1 < j)) {
            v = v1;
            j = j1;
        }
        if (j < 0 || j >= k) j = 0;  // no candidate compared smaller (see km_assign)
        if (p0 + t < n) {
            assign[p0 + t] = j;
            md = fmax(pn[t] + v, 0.0);
        }
    }
    for (int o = 16; o > 0; o >>= 1) md += __shfl_down_sync(0xffffffffu, md, o);
    __syncthreads();
    if (lane == 0 && w < 4) hv[w] = md;
    __syncthreads();
    if (t == 0) cost_part[blockIdx.x] = ((hv[0] + hv[1]) + hv[2]) + hv[3];
}

template <class T>
__global__ void km_cost_final(const double *__restrict__ part, int64_t np, T *__restrict__ cost, int acc) {
    __shared__ double s[256];
    double x = 0.0;
    const int64_t per = (np + 255) / 256;
    for (int64_t i = threadIdx.x * per; i < (threadIdx.x + 1) * per && i < np; ++i) x += part[i];
    s[threadIdx.x] = x;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *cost = acc ? (T)((double)*cost + s[0]) : (T)s[0];
}

}  // namespace vjpk

namespace {
using namespace vjph;

struct KmLayout {
    size_t cn, part, assign, sort, total;
    int64_t nbA;
    BsLayout bs;  // the center accumulator's bin sort (binsort.cuh)
};
KmLayout km_layout(int64_t n, int64_t k) {
    KmLayout L{};
    L.nbA = (n + vjpk::KM_BP - 1) / vjpk::KM_BP;
    L.bs = bs_layout(n, k);
    size_t off = 0;
    L.cn = off; off += align256((size_t)k * 8);
    L.part = off; off += align256((size_t)(L.nbA > 0 ? L.nbA : 1) * 8);
    L.assign = off; off += align256((size_t)(n > 0 ? n : 1) * 4);
    L.sort = off; off += L.bs.total;
    L.total = off;
    return L;
}

template <class T>
vjp_status km_run(int64_t n, int64_t k, int64_t d, const void *P, const void *C, const void *cost_bar, void *Cbar,
                  void *H, int32_t *assign, int64_t *counts, void *cost, void *ws, cudaStream_t s, unsigned flags) {
    KmLayout L = km_layout(n, k);
    unsigned char *w = static_cast<unsigned char *>(ws);
    double *cn = reinterpret_cast<double *>(w + L.cn);
    double *part = reinterpret_cast<double *>(w + L.part);
    int32_t *asg = assign ? assign : reinterpret_cast<int32_t *>(w + L.assign);
    const T *Pt = static_cast<const T *>(P);
    const T *Ct = static_cast<const T *>(C);
    const int acc = (flags & VJP_ACCUMULATE) ? 1 : 0;
    int launches = 0;
    vjpk::km_cnorm<T><<<(unsigned)((k + 127) / 128), 128, 0, s>>>(Ct, k, d, cn);
    ++launches;
    if (n > 0) {
        const int64_t nd = (d + vjpk::KM_KD - 1) / vjpk::KM_KD;
        const bool res = nd <= 2;
        const size_t asm_ = ((size_t)(res ? nd * vjpk::KM_KD : 2 * vjpk::KM_KD) * vjpk::KM_BP +
                             (size_t)2 * vjpk::KM_KD * vjpk::KM_BC) * 8;
        static const int use_mma = [] {
            const char *e = std::getenv("VJP_KMEANS_FFMA");
            return (e && *e == '1') ? 0 : 1;
        }();
        if (use_mma) {
            const int PW = (res ? (int)nd * vjpk::KM_KD : vjpk::KM_KD) + vjpk::KM_PS_PAD;
            const size_t msm = ((size_t)(res ? 1 : 2) * vjpk::KM_BP * PW +
                                (size_t)2 * vjpk::KM_BC * (vjpk::KM_KD + vjpk::KM_PS_PAD)) * 8;
            // 16-byte staging copies for f64 with even d (rows 16-byte aligned)
            const bool v16 = sizeof(T) == 8 && (d % 2) == 0 && (reinterpret_cast<uintptr_t>(Pt) % 16) == 0 &&
                             (reinterpret_cast<uintptr_t>(Ct) % 16) == 0;
            auto km = res ? (v16 ? vjpk::km_assign_mma<T, true, true> : vjpk::km_assign_mma<T, true, false>)
                          : (v16 ? vjpk::km_assign_mma<T, false, true> : vjpk::km_assign_mma<T, false, false>);
            cudaFuncSetAttribute(km, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm);
            km<<<(unsigned)L.nbA, vjpk::KM_MMA_NT, msm, s>>>(Pt, Ct, cn, n, k, d, asg, part);
        } else {
            auto ka = res ? vjpk::km_assign<T, true> : vjpk::km_assign<T, false>;
            cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asm_);
            ka<<<(unsigned)L.nbA, vjpk::KM_NT, asm_, s>>>(Pt, Ct, cn, n, k, d, asg, part);
        }
        ++launches;
    }
    // the return sweep's accumulator: C_bar_j = 2 ybar sum_{p: a(p) = j} (c_j - p)
    // and H_j = 2 ybar cnt_j — a width-d reduce_by_index(+) of the rows
    // (c_{a(p)} - p) into k bins, done by the
    // library's deterministic bin sort + segmented row sums (binsort.cuh),
    // the same routine as vjp_reduce_by_index(+)'s primal histogram
    launches += bs_sort<int32_t>(asg, n, k, L.bs, w + L.sort, counts, acc, s);
    launches += bs_rowsum<T>(Pt, Ct, k, d, 2.0, static_cast<const T *>(cost_bar), L.bs, w + L.sort,
                             static_cast<T *>(Cbar), static_cast<T *>(H), acc, s);
    if (cost) {
        if (n > 0) {
            vjpk::km_cost_final<T><<<1, 256, 0, s>>>(part, L.nbA, static_cast<T *>(cost), acc);
            ++launches;
        } else if (!acc && cudaMemsetAsync(cost, 0, sizeof(T), s) != cudaSuccess) {
            return VJP_ECUDA;
        }
    }
    count_launch(launches);
    return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
}

constexpr int64_t kKmMaxK = 12288;  // per-block histograms and order counters live in shared memory
}  // namespace

extern "C" {

size_t vjp_kmeans_workspace_bytes(vjp_dtype dtype, int64_t n, int64_t k, int64_t d) {
    if ((dtype != VJP_F32 && dtype != VJP_F64) || n < 0 || k < 1 || d < 1) return 0;
    return km_layout(n, k).total;
}

vjp_status vjp_kmeans(vjp_dtype dtype, int64_t n, int64_t k, int64_t d, const void *points, const void *centers,
                      const void *cost_bar, void *centers_bar, void *hess_diag, int32_t *assign, int64_t *counts,
                      void *cost, void *ws, size_t ws_bytes, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_kmeans");
    if (dtype != VJP_F32 && dtype != VJP_F64) return VJP_EINVAL;
    if (n < 0 || k < 1 || d < 1 || n >= ((int64_t)1 << 31) || k > kKmMaxK) return k > kKmMaxK ? VJP_EUNSUPPORTED : VJP_EINVAL;
    if ((n > 0 && !points) || !centers || !cost_bar || !centers_bar) return VJP_EINVAL;
    const size_t es = dtype == VJP_F64 ? 8 : 4;
    const void *al[] = {points, centers, cost_bar, centers_bar, hess_diag, assign, counts, cost};
    for (const void *p : al)
        if (p && (reinterpret_cast<uintptr_t>(p) % es) != 0) return VJP_EALIGN;
    if (ws_bytes < km_layout(n, k).total || !ws || !aligned16(ws)) return VJP_EWORKSPACE;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dtype == VJP_F64
               ? km_run<double>(n, k, d, points, centers, cost_bar, centers_bar, hess_diag, assign, counts, cost, ws, s,
                                flags)
               : km_run<float>(n, k, d, points, centers, cost_bar, centers_bar, hess_diag, assign, counts, cost, ws, s,
                               flags);
}

}  // extern "C"
