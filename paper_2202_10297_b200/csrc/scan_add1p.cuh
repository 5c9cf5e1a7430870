// scan_add1p.cuh — scan(+) closed form (as_bar = reverse (scan
// (+) (reverse ys_bar)), `as` not read) as ONE pass with a TWO-LEVEL
// decoupled look-back: ys_bar read once, as_bar written once (16 B/elem f64,
// 8 B f32: the method bytes).  The default for scan(+) on one GPU without
// ys / ACCUMULATE (DESIGN 7.1d).
//
// Tiles of 768 rows x 128 B (96 KB) staged in shared memory by TMA (2 CTAs per SM).  CTAs
// take tickets in start order; ticket k is the k-th tile from the RIGHT (the
// return sweep runs right to left).  A tile publishes its
// aggregate (AGG record, one 16-byte store = flag + value) as soon as it has
// summed its data, and a dedicated look-back warp, running while the data
// streams in, forms the sum of everything to its right:
//   level 1: the 97..128 tickets just below k (4 records per lane, issued
//            at once) — the tiles still in flight — down to a group
//            boundary; the nearest INCL record found there terminates it;
//   level 2: whole groups of 32 tickets below: each group's sum (GRP record,
//            published by the group's last tile to arrive) and the INCL
//            record of the group's last ticket (= the inclusive sum through
//            that group), a window of 32 groups (1024 tiles) per round trip.
// The look-back only ever waits for AGG / GRP records (published right after
// a tile's load), never for a chain of inclusive sums: with ~450-900 tiles
// in flight the single-level window of round 1 walked ~20 windows of AGGs
// per tile (DESIGN 7.6); here it is one round trip after the nearest
// predecessor's data has landed.  Then INCL = exclusive + AGG is published
// and the tile writes its outputs (f64 sums; R9 for f32).
#pragma once

#include "common.cuh"

namespace vjpk {

// (no timeouts: every wait is on a record of an earlier ticket, i.e. of a CTA
// that started before this one and is running: dynamic tickets make the
// look-back deadlock-free)

struct Add1pParams {
    int64_t n;
    int64_t ntiles;
    const void *ys_bar;
    void *as_bar;
    uint32_t *ticket;       // [1]
    uint32_t *gcount;       // [ngroups] tiles of the group that published AGG
    double2 *agg;           // [ntiles] {flag (1), tile sum}
    double2 *inc;           // [ntiles] {flag (2), inclusive sum: the tile and everything right of it}
    double2 *grp;           // [ngroups] {flag (1), group sum}
};

__device__ __forceinline__ void st_rec16(double2 *p, double flag, double v) {
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(flag), "d"(v) : "memory");
}
__device__ __forceinline__ double2 ld_rec16(const double2 *p) {
    double2 r;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p) : "memory");
    return r;
}

// 16-byte chunk <-> 2 f64 / 4 f32 elements, by value (no address of a
// register array: that would put the row in local memory)
__device__ __forceinline__ void unpack16(const double2 &w, double *v) { v[0] = w.x; v[1] = w.y; }
__device__ __forceinline__ void unpack16(const double2 &w, float *v) {
    const unsigned long long a = (unsigned long long)__double_as_longlong(w.x);
    const unsigned long long b = (unsigned long long)__double_as_longlong(w.y);
    v[0] = __uint_as_float((unsigned)a);
    v[1] = __uint_as_float((unsigned)(a >> 32));
    v[2] = __uint_as_float((unsigned)b);
    v[3] = __uint_as_float((unsigned)(b >> 32));
}
__device__ __forceinline__ double2 pack16(const double *v) { return make_double2(v[0], v[1]); }
__device__ __forceinline__ double2 pack16(const float *v) {
    const unsigned long long a = (unsigned long long)__float_as_uint(v[0]) | ((unsigned long long)__float_as_uint(v[1]) << 32);
    const unsigned long long b = (unsigned long long)__float_as_uint(v[2]) | ((unsigned long long)__float_as_uint(v[3]) << 32);
    return make_double2(__longlong_as_double((long long)a), __longlong_as_double((long long)b));
}

// exclusive sum of everything right of ticket k (one warp; result in every
// lane).  Level 1 covers the D (97..128) tickets just below k, down to a
// group boundary 32 G0, reading their records DIRECTLY (4 per lane, all
// issued at once): these are the tiles still in flight, so no group record
// stands between their loads and this look-back; the nearest inclusive
// record found there terminates it.  Level 2 continues over whole groups
// G0-1, G0-2, ... (their group records and group-last inclusive records,
// windows of 32 groups) — old enough that both are normally published.
constexpr int k1pM = 4;  // level-1 tickets per lane
__device__ __forceinline__ double add1p_lookback(const Add1pParams &P, int64_t k, int lane) {
    const int64_t G0 = k >= 97 ? (k - 97) >> 5 : 0;
    const int D = (int)(k - (G0 << 5));  // 1 .. 128
    double2 q[k1pM], a[k1pM];
#pragma unroll
    for (int m = 0; m < k1pM; ++m) {
        const int d = lane + 1 + 32 * m;
        q[m] = make_double2(0.0, 0.0);
        a[m] = make_double2(0.0, 0.0);
        if (d <= D) {
            q[m] = ld_rec16(P.inc + (k - d));
            if (k - d != 0) a[m] = ld_rec16(P.agg + (k - d));
        }
    }
    // group records of the first level-2 window, issued with level 1
    const int64_t g2 = G0 - 1 - lane;
    double2 q2 = make_double2(0.0, 0.0), r2 = make_double2(0.0, 0.0);
    if (g2 >= 0) {
        q2 = ld_rec16(P.inc + (g2 << 5) + 31);
        r2 = ld_rec16(P.grp + g2);
    }
    // ---- level 1: nearest inclusive record (ticket 0 always becomes one)
    int dstar = 0;  // 0: none
#pragma unroll
    for (int m = k1pM - 1; m >= 0; --m) {
        const int d = lane + 1 + 32 * m;
        if (d <= D && k - d == 0)
            while (q[m].x == 0.0) q[m] = ld_rec16(P.inc);
        const unsigned mk = __ballot_sync(0xffffffffu, d <= D && q[m].x != 0.0);
        if (mk) dstar = 32 * m + __ffs(mk);
    }
    double x = 0.0;
#pragma unroll
    for (int m = 0; m < k1pM; ++m) {
        const int d = lane + 1 + 32 * m;
        if (d > D) continue;
        if (dstar && d == dstar) {
            x += q[m].y;
        } else if (!dstar || d < dstar) {
            while (a[m].x == 0.0) a[m] = ld_rec16(P.agg + (k - d));
            x += a[m].y;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (dstar || G0 == 0) return x;
    double sum = x;
    // ---- level 2: windows of 32 groups below G0
    for (int64_t gb = G0 - 1; gb >= 0; gb -= 32) {
        const int64_t gl = gb - lane;
        if (gb != G0 - 1 && gl >= 0) {
            q2 = ld_rec16(P.inc + (gl << 5) + 31);
            r2 = ld_rec16(P.grp + gl);
        }
        const unsigned incm = __ballot_sync(0xffffffffu, gl >= 0 && q2.x != 0.0);
        const int lim = incm ? __ffs(incm) - 1 : 32;  // nearest group whose last ticket is inclusive
        double y = 0.0;
        if (gl >= 0 && lane < lim) {
            while (r2.x == 0.0) r2 = ld_rec16(P.grp + gl);
            y = r2.y;
        } else if (lane == lim) {
            y = q2.y;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        sum += y;
        if (incm) break;
    }
    return sum;
}

__device__ __forceinline__ uint32_t atom_add_release_gpu(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// named barrier WITHOUT .aligned (bar.sync is barrier.sync.aligned, which
// requires the whole warp converged at the instruction — the look-back warp
// arrives from per-lane polling loops; compute-sanitizer synccheck flags it)
__device__ __forceinline__ void bar_named(int id, int count) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// 8 data warps + 1 look-back warp that computes the exclusive sum WHILE the
// tile streams in.  The tile (256 threads x RPT rows of 128 B; RPT = 3: 96 KB)
// moves global -> shared -> global by 2-D TMA with the 128B swizzle (one box
// of 256 rows per TMA instruction, mbarrier completion), so a CTA holds no
// tile data in registers while its look-back runs; thread t owns rows
// RPT t .. RPT t + RPT - 1 and reads / writes them conflict-free (swz).
constexpr int k1pData = 256;
template <class T, int RPT>
__global__ void __launch_bounds__(k1pData + 32, 2) scan_add_1p(const __grid_constant__ CUtensorMap tm_in,
                                                             const __grid_constant__ CUtensorMap tm_out,
                                                             const Add1pParams P) {
    constexpr int E = 128 / (int)sizeof(T);  // elements per row
    constexpr int NW = k1pData / 32;
    constexpr int TB = k1pData * RPT * 128;  // tile bytes
    constexpr int TE = TB / (int)sizeof(T);  // tile elements
    constexpr int EPC = 16 / (int)sizeof(T); // elements per 16-byte chunk
    extern __shared__ __align__(1024) unsigned char s_raw[];
    unsigned char *s_tile = smem_align1024(s_raw);
    __shared__ int64_t s_tick;
    __shared__ double s_wsum[NW];
    __shared__ double s_excl;
    __shared__ uint64_t s_bar;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        const int64_t k0 = (int64_t)atomicAdd(P.ticket, 1u);
        s_tick = k0;
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const int64_t tile0 = P.ntiles - 1 - k0;
        if ((tile0 + 1) * (int64_t)TE <= P.n) {  // full tile: TMA in (128B-swizzled rows, 256 per box)
            mbar_arrive_expect_tx(&s_bar, TB);
#pragma unroll
            for (int b = 0; b < RPT; ++b)
                tma_load_2d(s_tile + b * 256 * 128, &tm_in, &s_bar, 0, (int)(tile0 * 256 * RPT + b * 256));
        } else {
            mbar_arrive(&s_bar);
        }
    }
    __syncthreads();
    const int64_t k = s_tick;
    if (warp == NW) {
        // ---------------- look-back warp
        const double ex = k > 0 ? add1p_lookback(P, k, lane) : 0.0;
        if (lane == 0) s_excl = ex;
        bar_named(1, k1pData + 32);  // excl ready / the data warps' sums ready
        if (lane == 0 && k > 0) {
            double tile_sum = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) tile_sum += s_wsum[w];
            st_rec16(P.inc + k, 2.0, ex + tile_sum);
        }
        return;
    }
    // ---------------- data warps
    const int64_t tile = P.ntiles - 1 - k;
    const bool full = (tile + 1) * (int64_t)TE <= P.n;
    const int64_t te0 = tile * (int64_t)TE;
    if (!full) {  // the partial rightmost tile: element-wise into the swizzled rows (zero padded)
        const T *src = static_cast<const T *>(P.ys_bar);
        for (int e = t; e < TE; e += k1pData) {
            const int r = e / E, q = e % E;
            T *d = reinterpret_cast<T *>(s_tile + swz(r, q / EPC)) + q % EPC;
            *d = (te0 + e < P.n) ? src[te0 + e] : (T)0;
        }
        bar_named(2, k1pData);
    }
    mbar_wait(&s_bar, 0);
    // pass 1: the thread's sum over its RPT rows (8 independent chunk sums per
    // row, added as a tree: short dependent chains)
    double rs = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = RPT * t + i;
        double cs[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            T v[EPC];
            unpack16(*reinterpret_cast<const double2 *>(s_tile + swz(r, c)), v);
            cs[c] = 0.0;
#pragma unroll
            for (int q = 0; q < EPC; ++q) cs[c] += (double)v[q];
        }
        rs += ((cs[0] + cs[1]) + (cs[2] + cs[3])) + ((cs[4] + cs[5]) + (cs[6] + cs[7]));
    }
    double sw = rs;  // inclusive suffix over the warp (lanes to the right = higher elements)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_down_sync(0xffffffffu, sw, o);
        if (lane + o < 32) sw += u;
    }
    if (lane == 0) s_wsum[warp] = sw;
    bar_named(2, k1pData);
    double tile_sum = 0.0, right_warps = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        tile_sum += s_wsum[w];
        if (w > warp) right_warps += s_wsum[w];
    }
    if (warp == 0) {
        uint32_t arrived = 0;
        const int64_t g = k >> 5;
        if (lane == 0) {
            if (k == 0) st_rec16(P.inc, 2.0, tile_sum);
            else st_rec16(P.agg + k, 1.0, tile_sum);
            arrived = atom_add_release_gpu(P.gcount + g, 1u) + 1u;
        }
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        if (arrived == 32u) {
            fence_acq_rel_gpu();
            const int64_t j = (g << 5) + lane;
            double2 r;
            if (j == 0) {
                do { r = ld_rec16(P.inc); } while (r.x == 0.0);
            } else {
                do { r = ld_rec16(P.agg + j); } while (r.x == 0.0);
            }
            double x = r.y;
#pragma unroll
            for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == 0) st_rec16(P.grp + g, 1.0, x);
        }
    }
    bar_named(1, k1pData + 32);
    double carry = s_excl + right_warps + (sw - rs);
    // pass 2: rows right to left; per row the 8 chunk sums first, then the
    // suffix over the chunks, then inside each chunk (dependent chain 8 + EPC
    // instead of E); results written back in place
#pragma unroll
    for (int i = RPT - 1; i >= 0; --i) {
        const int r = RPT * t + i;
        T v[E];
        double cs[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            unpack16(*reinterpret_cast<const double2 *>(s_tile + swz(r, c)), v + c * EPC);
            cs[c] = 0.0;
#pragma unroll
            for (int q = 0; q < EPC; ++q) cs[c] += (double)v[c * EPC + q];
        }
        double suf = carry;  // entering chunk c from the right
#pragma unroll
        for (int c = 7; c >= 0; --c) {
            double run = suf;
#pragma unroll
            for (int q = EPC - 1; q >= 0; --q) {
                run += (double)v[c * EPC + q];
                v[c * EPC + q] = (T)run;
            }
            suf += cs[c];
        }
        carry = suf;
#pragma unroll
        for (int c = 0; c < 8; ++c) *reinterpret_cast<double2 *>(s_tile + swz(r, c)) = pack16(v + c * EPC);
    }
    if (full) {
        fence_proxy_async_smem();
        bar_named(2, k1pData);
        if (t == 0) {
#pragma unroll
            for (int b = 0; b < RPT; ++b)
                tma_store_2d(&tm_out, s_tile + b * 256 * 128, 0, (int)(tile * 256 * RPT + b * 256));
            tma_store_commit();
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else {
        bar_named(2, k1pData);
        T *dst = static_cast<T *>(P.as_bar);
        for (int e = t; e < TE; e += k1pData) {
            const int r = e / E, q = e % E;
            if (te0 + e < P.n) dst[te0 + e] = *(reinterpret_cast<const T *>(s_tile + swz(r, q / EPC)) + q % EPC);
        }
    }
}

}  // namespace vjpk
