// scan_chunked.cuh — chunked reduce-then-scan vjp_scan kernels (the default
// path for ADD, MUL, LINREC and MAT2).
//
// Why: the single-pass decoupled look-back (scan_kernels.cuh) serialises every
// tile behind an L2 round-trip chain while its CTA holds a 64 KB tile; on B200
// that left HBM at ~25% (profiles/).  Here every CTA is persistent over one
// contiguous CHUNK of tiles and streams it through an S-stage TMA ring
// (mbarrier full barriers, bulk async-group stores), and CTAs never wait on
// each other:
//
//   K_R  scan_reduce : per tile, forward aggregate F_t (the re-executed primal
//        scan) and reverse-map aggregate M_t (the composed affine maps of
//        the return sweep, grouped per element as in
//        scan_ops.cuh); writes F_t per tile and (F, M) per chunk.
//   K_C  scan_apply  : prologue combines the chunk records (ordered, on the
//        device) into this chunk's forward prefix and the reverse carry entering
//        its right end, then walks its tiles right to left: re-executes the
//        primal scan in registers from the tile's prefix (tape-free), builds
//        and reverse-scans the maps, applies the carry, writes as_bar (and ys).
//
// Inside a tile every thread owns one 128-byte row (a few elements) and folds
// it serially; the per-row aggregates go to shared memory and ONE warp scans
// each direction (warp 0 forward, warp 1 reverse: serial over NT/32 rows per
// lane, then a 5-level shuffle scan), instead of every thread running a
// shuffle tree of 2x2-map compositions.
//
// The return sweep therefore reads `as` and `ys_bar` twice (K_R, K_C) — the
// same traffic the contiguous multi-GPU partition pays — in
// exchange for pure streaming kernels.  For world > 1 the chunk records are
// reduced once more into the shard record exchanged by all_gather.
#pragma once

#include "scan_kernels.cuh"

namespace vjpk {

// Tile-data accesses of K_R / K_C: 1 = through a generic pointer (LD/ST), 0 =
// shared-typed (LDS/STS).  The row scratch is always shared-typed.  Measured
// (tools/time_variants.py, config 2 at 2^26 f64): MAT2 1.77 ms with shared-
// typed tiles vs 1.68 ms generic (the generic loads are scheduled less
// eagerly: fewer live registers around the row loops); LINREC unchanged.
#ifndef VJP_APPLY_TILE
#define VJP_APPLY_TILE 1
#endif
#ifndef VJP_REDUCE_TILE
#define VJP_REDUCE_TILE 1
#endif
template <int GENERIC>
__device__ __forceinline__ unsigned char *tile_base(unsigned char *sbase) {
    if (GENERIC) {  // opaque to the address-space inference
        unsigned long long r;
        asm("mov.b64 %0, %1;" : "=l"(r) : "l"(reinterpret_cast<unsigned long long>(sbase)));
        return reinterpret_cast<unsigned char *>(r);
    }
    return sbase;
}

#ifndef VJP_REDUCE_FUSEDROW
#define VJP_REDUCE_FUSEDROW 1  // K_R: one right-to-left pass per row for both aggregates
#endif
#ifndef VJP_APPLY_FUSEDROW
#define VJP_APPLY_FUSEDROW 1   // K_C phase 1: the same (MAT2)
#endif
struct ChunkParams {
    int64_t n;
    int64_t full_rows;
    int32_t tail_bytes;
    int32_t ntiles;
    int32_t nchunks;
    int32_t pad0;
    const void *as;
    const void *ys_bar;
    void *as_bar;
    void *ys;
    double *tileF;     // [ntiles][W] forward tile aggregates
    double *tileP;     // [ntiles][W] forward exclusive prefixes (K_C prologue)
    double *chunkRec;  // [nchunks][W + kMapD]
    double *partial;   // shard record (world > 1) or nullptr
    uint32_t *counter; // last-block counter for the shard record
    const double *gathered;
    int32_t rank, world;
    int32_t global_first;
    const void *ylast;  // YL kernels (general reduce rule): ys_bar = ylast at element n-1, 0 elsewhere
};

// per-CTA shared scratch beside the TMA stages (sized on the host with sizeof).
// Row aggregates are stored component-major with one pad slot per 16 entries
// (spos) so that both the per-thread writes (entry = thread) and the scan
// warp's reads (lane l reads entries l*K .. l*K+K-1) are bank-conflict free.
template <int NT>
struct RowArr {
    static constexpr int kStride = NT + NT / 16;
    __device__ static __forceinline__ int spos(int e) { return e + (e >> 4); }
};
template <class Op, int NT, int S>
struct ReduceSmem {
    uint64_t bar[S];
    int last;
    double rv[Op::W * RowArr<NT>::kStride];      // row forward aggregates
    double rm[Op::kMapD * RowArr<NT>::kStride];  // row reverse maps
    typename Op::Val vs[NT / 32 + 1];
    typename Op::Map ms[NT / 32 + 1];
};
template <class Op, int NT, int S>
struct ApplySmem {
    uint64_t bar[S];
    double rv[Op::W * RowArr<NT>::kStride];      // row forward aggregates -> rs entering each row
    double rm[Op::kMapD * RowArr<NT>::kStride];  // row reverse maps; reused for H entering each row
    typename Op::Val vs[NT / 32 + 1];
    typename Op::Map ms[NT / 32 + 1];
};

template <int NT, int D>
__device__ __forceinline__ void row_put(double *a, int e, const double *v) {
#pragma unroll
    for (int k = 0; k < D; ++k) a[k * RowArr<NT>::kStride + RowArr<NT>::spos(e)] = v[k];
}
template <int NT, int D>
__device__ __forceinline__ void row_get(const double *a, int e, double *v) {
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = a[k * RowArr<NT>::kStride + RowArr<NT>::spos(e)];
}
template <class Op, int NT>
__device__ __forceinline__ void put_v(double *a, int e, const typename Op::Val &v) { row_put<NT, Op::W>(a, e, v.x); }
template <class Op, int NT>
__device__ __forceinline__ typename Op::Val get_v(const double *a, int e) {
    typename Op::Val v;
    row_get<NT, Op::W>(a, e, v.x);
    return v;
}
template <class Op, int NT>
__device__ __forceinline__ void put_m(double *a, int e, const typename Op::Map &m) {
    row_put<NT, Op::kMapD>(a, e, reinterpret_cast<const double *>(&m));
}
template <class Op, int NT>
__device__ __forceinline__ typename Op::Map get_m(const double *a, int e) {
    typename Op::Map m;
    row_get<NT, Op::kMapD>(a, e, reinterpret_cast<double *>(&m));
    return m;
}

__device__ __forceinline__ int64_t chunk_begin(const ChunkParams &p, int64_t c) {
    return c * (int64_t)p.ntiles / p.nchunks;
}

template <int NT>
__device__ __forceinline__ int chunk_tile_rows(const ChunkParams &p, int64_t tile) {
    int64_t r = p.full_rows - tile * NT;
    return r <= 0 ? 0 : (r >= NT ? NT : (int)r);
}

// thread 0: start the TMA loads of `tile` into a stage (NB buffers of NT rows)
template <int NT, int NB>
__device__ __forceinline__ void issue_tile(const ChunkParams &p, int64_t tile, uint64_t *bar, unsigned char *stage,
                                           const CUtensorMap *m0, const CUtensorMap *m1, const CUtensorMap *m2) {
    const int rows = chunk_tile_rows<NT>(p, tile);
    if (rows > 0) {
        mbar_arrive_expect_tx(bar, NB * NT * kRowBytes);
        const CUtensorMap *ms[3] = {m0, m1, m2};
#pragma unroll
        for (int b = 0; b < NB; ++b) tma_load_2d(stage + b * NT * kRowBytes, ms[b], bar, 0, (int)(tile * NT));
    } else {
        mbar_arrive(bar);  // keeps the stage's phase sequence when a tile has no full row
    }
}

// ordered reduction of chunk records [lo, hi) over the block: forward part
// F_lo (.) ... (.) F_{hi-1} and reverse part M_lo o ... o M_{hi-1}.
template <class Op, int NT>
__device__ __forceinline__ void range_reduce(const double *recs, int64_t lo, int64_t hi, typename Op::Val *vs,
                                             typename Op::Map *ms, typename Op::Val &F, typename Op::Map &M) {
    constexpr int W = Op::W, R = Op::W + Op::kMapD, NW = NT / 32;
    const int t = threadIdx.x;
    const int64_t cnt = hi > lo ? hi - lo : 0;
    const int64_t per = (cnt + NT - 1) / NT;
    typename Op::Val f = Op::fwd_id();
    typename Op::Map m = Op::map_id();
    for (int64_t j = lo + t * per; j < lo + (t + 1) * per && j < hi; ++j) {
        double d[R];
        ld_rec<R>(recs + j * R, d);
        typename Op::Val v;
#pragma unroll
        for (int k = 0; k < W; ++k) v.x[k] = d[k];
        f = Op::fwd(f, v);
        m = Op::compose(m, map_from<Op>(d + W));
    }
    F = block_reduce_fwd<Op, NW>(f, vs);
    M = block_reduce_rev<Op, NW>(m, ms);
}

// ---- one thread's row: forward product and composed reverse map -----------
template <class Op, class T, bool FWD>
__device__ __forceinline__ typename Op::Val row_fwd(const unsigned char *sA, int t, int64_t e0, bool mask, int64_t n) {
    using G = Geo<Op, T>;
    typename Op::Val F = Op::fwd_id();
    if constexpr (FWD) {
#pragma unroll
        for (int g = 0; g < G::NG; ++g) {
            uint32_t w[G::GB / 4];
            lds_group<G::GB>(sA, t, g, w);
#pragma unroll
            for (int e = 0; e < G::EG; ++e) {
                typename Op::Val a = dec<T, Op::W>(w + e * (G::ES / 4));
                if (!mask || e0 + g * G::EG + e < n) F = Op::fwd(F, a);
            }
        }
    }
    return F;
}

// M_e0 o ... o M_{e0+EPR-1}; rs-independent operators only (chunked path).
// YL: ys_bar is virtual — *yl at element n-1, zero elsewhere (general reduce).
template <class Op, class T, bool FWD, bool YL = false>
__device__ __forceinline__ typename Op::Map row_map(const unsigned char *sA, const unsigned char *sY, int t,
                                                    int64_t e0, bool mask, int64_t n,
                                                    const typename Op::Val *yl = nullptr) {
    using G = Geo<Op, T>;
    if constexpr (std::is_same<Op, OpAdd>::value && !YL && sizeof(T) == 8) {
        // + maps commute: one partial sum per access group (independent
        // chains instead of 16 dependent adds per row), then a tree.  f64
        // only: measured 3.73 -> 3.69 ms for the f64 sweep at 2^30, while the
        // f32 chunked reduce got slower (2.19 -> 2.34 ms)
        double part[G::NG];
#pragma unroll
        for (int g = 0; g < G::NG; ++g) {
            uint32_t wy[G::GB / 4];
            lds_group<G::GB>(sY, t, g, wy);
            part[g] = 0.0;
#pragma unroll
            for (int e = 0; e < G::EG; ++e)
                if (!mask || e0 + g * G::EG + e < n) part[g] += dec<T, 1>(wy + e * (G::ES / 4)).x[0];
        }
#pragma unroll
        for (int w = 1; w < G::NG; w <<= 1)
#pragma unroll
            for (int g = 0; g + w < G::NG; g += 2 * w) part[g] += part[g + w];
        return {part[0]};
    }
    typename Op::Map Tm = Op::map_id();
#pragma unroll
    for (int g = G::NG - 1; g >= 0; --g) {
        uint32_t wa[G::GB / 4], wy[G::GB / 4];
        if (FWD) lds_group<G::GB>(sA, t, g, wa);
        if (!YL) lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
        for (int e = G::EG - 1; e >= 0; --e) {
            typename Op::Val a = FWD ? dec<T, Op::W>(wa + e * (G::ES / 4)) : Op::fwd_id();
            typename Op::Val y;
            if (YL) {
#pragma unroll
                for (int q = 0; q < Op::W; ++q) y.x[q] = (e0 + g * G::EG + e == n - 1) ? yl->x[q] : 0.0;
            } else {
                y = dec<T, Op::W>(wy + e * (G::ES / 4));
            }
            if (!mask || e0 + g * G::EG + e < n) Tm = Op::extend(Tm, Op::fwd_id(), a, y);
        }
    }
    return Tm;
}

// the virtual ys_bar element of YL kernels (every thread keeps a copy)
template <class Op, class T>
__device__ __forceinline__ typename Op::Val load_ylast(const void *p) {
    typename Op::Val v;
#pragma unroll
    for (int q = 0; q < Op::W; ++q) v.x[q] = p ? (double)static_cast<const T *>(p)[q] : 0.0;
    return v;
}

// rs-DEPENDENT operators (MIN/MAX: the Jacobians pick a side by comparing
// rs_{i-1} with a_i): re-execute the primal over the row from `rs` (the prefix
// entering the row), then compose the maps right to left with the true rs.
template <class Op, class T>
__device__ __forceinline__ typename Op::Map row_map_rs(const unsigned char *sA, const unsigned char *sY, int t,
                                                       int64_t e0, bool mask, int64_t n, typename Op::Val rs) {
    using G = Geo<Op, T>;
    typename Op::Val rsp[G::EPR];
#pragma unroll
    for (int g = 0; g < G::NG; ++g) {
        uint32_t wa[G::GB / 4];
        lds_group<G::GB>(sA, t, g, wa);
#pragma unroll
        for (int e = 0; e < G::EG; ++e) {
            const int q = g * G::EG + e;
            rsp[q] = rs;
            if (!mask || e0 + q < n) rs = Op::fwd(rs, dec<T, Op::W>(wa + e * (G::ES / 4)));
        }
    }
    typename Op::Map Tm = Op::map_id();
#pragma unroll
    for (int g = G::NG - 1; g >= 0; --g) {
        uint32_t wa[G::GB / 4], wy[G::GB / 4];
        lds_group<G::GB>(sA, t, g, wa);
        lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
        for (int e = G::EG - 1; e >= 0; --e) {
            const int q = g * G::EG + e;
            if (!mask || e0 + q < n)
                Tm = Op::extend(Tm, rsp[q], dec<T, Op::W>(wa + e * (G::ES / 4)), dec<T, Op::W>(wy + e * (G::ES / 4)));
        }
    }
    return Tm;
}

// both row aggregates in ONE right-to-left pass over the row (K_R with FWD and
// REV): the forward product accumulated from the right, F <- a (.) F
// (associativity), so each element's words are read from shared memory once
template <class Op, class T, bool YL>
__device__ __forceinline__ void row_fwd_map(const unsigned char *sA, const unsigned char *sY, int t, int64_t e0,
                                            bool mask, int64_t n, const typename Op::Val *yl,
                                            typename Op::Val &F, typename Op::Map &Tm) {
    using G = Geo<Op, T>;
    F = Op::fwd_id();
    Tm = Op::map_id();
#pragma unroll
    for (int g = G::NG - 1; g >= 0; --g) {
        uint32_t wa[G::GB / 4], wy[G::GB / 4];
        lds_group<G::GB>(sA, t, g, wa);
        if (!YL) lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
        for (int e = G::EG - 1; e >= 0; --e) {
            const typename Op::Val a = dec<T, Op::W>(wa + e * (G::ES / 4));
            typename Op::Val y;
            if (YL) {
#pragma unroll
                for (int q = 0; q < Op::W; ++q) y.x[q] = (e0 + g * G::EG + e == n - 1) ? yl->x[q] : 0.0;
            } else {
                y = dec<T, Op::W>(wy + e * (G::ES / 4));
            }
            if (!mask || e0 + g * G::EG + e < n) {
                Tm = Op::extend(Tm, Op::fwd_id(), a, y);
                F = Op::fwd(a, F);
            }
        }
    }
}

// ---- warp-level scans over the NT row aggregates in shared memory ----------
// (executed by one full warp; lane l owns rows [l*K, l*K + K), K = NT/32)

// reduce: returns v_0 (.) ... (.) v_{NT-1} in every lane
template <class Op, int NT>
__device__ __forceinline__ typename Op::Val warp_reduce_fwd_rows(const double *v) {
    constexpr int K = NT / 32;
    const int lane = threadIdx.x & 31;
    typename Op::Val a = get_v<Op, NT>(v, lane * K);
#pragma unroll
    for (int j = 1; j < K; ++j) a = Op::fwd(a, get_v<Op, NT>(v, lane * K + j));
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        typename Op::Val o = shfl_down_v(a, s);
        if (lane + s < 32) a = Op::fwd(a, o);
    }
    return shfl_idx_v(a, 0);
}
template <class Op, int NT>
__device__ __forceinline__ typename Op::Map warp_reduce_rev_rows(const double *m) {
    constexpr int K = NT / 32;
    const int lane = threadIdx.x & 31;
    typename Op::Map a = get_m<Op, NT>(m, lane * K);
#pragma unroll
    for (int j = 1; j < K; ++j) a = Op::compose(a, get_m<Op, NT>(m, lane * K + j));
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        typename Op::Map o = shfl_down_m<Op>(a, s);
        if (lane + s < 32) a = Op::compose(a, o);
    }
    return shfl_idx_m<Op>(a, 0);
}

// exclusive forward scan, seeded with `pre`; overwrites v[r] with
// pre (.) v_0 (.) ... (.) v_{r-1}
template <class Op, int NT>
__device__ __forceinline__ void warp_excl_fwd_rows(double *v, typename Op::Val pre) {
    using V = typename Op::Val;
    constexpr int K = NT / 32;
    const int lane = threadIdx.x & 31;
    V e[K];
#pragma unroll
    for (int j = 0; j < K; ++j) e[j] = get_v<Op, NT>(v, lane * K + j);
    V loc = e[0];
#pragma unroll
    for (int j = 1; j < K; ++j) loc = Op::fwd(loc, e[j]);
    V inc = loc;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        V o = shfl_up_v(inc, s);
        if (lane >= s) inc = Op::fwd(o, inc);
    }
    V ex = shfl_up_v(inc, 1);
    V r = lane == 0 ? pre : Op::fwd(pre, ex);
#pragma unroll
    for (int j = 0; j < K; ++j) {
        put_v<Op, NT>(v, lane * K + j, r);
        r = Op::fwd(r, e[j]);
    }
}

// reverse: given the maps m[r] of the rows and the carry X entering the tile
// from the right, overwrites row r with (m_{r+1} o ... o m_{NT-1})(X) (the H
// entering row r from the right, as a Val) and returns (m_0 o ... o m_{NT-1})(X) (the carry for
// the next tile to the left) in every lane.
template <class Op, int NT>
__device__ __forceinline__ typename Op::Val warp_excl_rev_rows(double *m, typename Op::Val X) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int K = NT / 32;
    const int lane = threadIdx.x & 31;
    M e[K];
#pragma unroll
    for (int j = 0; j < K; ++j) e[j] = get_m<Op, NT>(m, lane * K + j);
    __syncwarp();  // the H values overwrite the maps in place
    M loc = e[K - 1];
#pragma unroll
    for (int j = K - 2; j >= 0; --j) loc = Op::compose(e[j], loc);
    M inc = loc;  // lanes l..31
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        M o = shfl_down_m<Op>(inc, s);
        if (lane + s < 32) inc = Op::compose(inc, o);
    }
    M ex = shfl_down_m<Op>(inc, 1);
    V h = lane == 31 ? X : Op::apply(ex, X);
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
        put_v<Op, NT>(m, lane * K + j, h);
        h = Op::apply(e[j], h);
    }
    return shfl_idx_v(h, 0);
}

// =============================================================================
// K_R: per-tile / per-chunk aggregates
// =============================================================================
template <class Op, class T, int NT, int S, bool FWD, bool REV, bool YL = false>
__global__ void __launch_bounds__(NT, 1) scan_reduce(const __grid_constant__ CUtensorMap tm_as,
                                                     const __grid_constant__ CUtensorMap tm_yb,
                                                     const ChunkParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, NW = NT / 32, R = Op::W + Op::kMapD;
    constexpr int NB = (FWD ? 1 : 0) + ((REV && !YL) ? 1 : 0);
    constexpr int BUF = NT * kRowBytes, STG = NB * BUF;
    static_assert(NW >= 2, "needs a forward and a reverse scan warp");

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *const sbase = smem_align1024(smem_raw);
    ReduceSmem<Op, NT, S> &sm = *reinterpret_cast<ReduceSmem<Op, NT, S> *>(sbase + S * STG);
    unsigned char *base = tile_base<VJP_REDUCE_TILE>(sbase);
    const V yl = YL ? load_ylast<Op, T>(p.ylast) : Op::fwd_id();

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    const CUtensorMap *m0 = FWD ? &tm_as : &tm_yb;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < S && s < k; ++s) issue_tile<NT, NB>(p, t0 + s, &sm.bar[s], base + s * STG, m0, &tm_yb, &tm_yb);
    }
    __syncthreads();

    V Fc = Op::fwd_id();  // chunk aggregates, kept by warp 0 / warp 1
    M Mc = Op::map_id();
    for (int64_t i = 0; i < k; ++i) {
        const int64_t tile = t0 + i;
        const int s = (int)(i % S);
        mbar_wait(&sm.bar[s], (uint32_t)((i / S) & 1));
        unsigned char *sA = base + s * STG;
        unsigned char *sY = sA + (FWD ? BUF : 0);
        const bool last = (tile == p.ntiles - 1);
        if (last && p.tail_bytes) {
            if (t == (int)(p.full_rows - tile * NT)) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                if (REV && !YL) load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
            }
            __syncthreads();
        }
        const int64_t e0 = (tile * NT + t) * G::EPR;
        V rowF;
        M rowM;
        if constexpr (FWD && REV && (VJP_REDUCE_FUSEDROW != 0) && !std::is_same<Op, OpAdd>::value) {
            row_fwd_map<Op, T, YL>(sA, sY, t, e0, last, p.n, &yl, rowF, rowM);
        } else {
            rowF = row_fwd<Op, T, FWD>(sA, t, e0, last, p.n);
            rowM = REV ? row_map<Op, T, FWD, YL>(sA, sY, t, e0, last, p.n, &yl) : Op::map_id();
        }
        __syncthreads();  // every row read its data (stage s is free) and the scan warps are done with the scratch
        if (t == 0 && i + S < k) issue_tile<NT, NB>(p, tile + S, &sm.bar[s], sA, m0, &tm_yb, &tm_yb);
        if (FWD) put_v<Op, NT>(sm.rv, t, rowF);
        if (REV) put_m<Op, NT>(sm.rm, t, rowM);
        __syncthreads();
        if (FWD && warp == 0) {
            V Ft = warp_reduce_fwd_rows<Op, NT>(sm.rv);
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < W; ++q) st_cg(p.tileF + tile * W + q, Ft.x[q]);
            }
            Fc = Op::fwd(Fc, Ft);
        }
        if (REV && warp == 1) Mc = Op::compose(Mc, warp_reduce_rev_rows<Op, NT>(sm.rm));
    }
    // chunk record [F | M]: F from warp 0, M from warp 1
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < W; ++q) st_cg(p.chunkRec + c * R + q, Fc.x[q]);
    }
    if (t == 32) {
        double rec[Op::kMapD];
        map_to<Op>(Mc, rec);
        st_rec<Op::kMapD>(p.chunkRec + c * R + W, rec);
    }
    if (p.partial) {
        // last-block pattern: the CTA that finishes last reduces all chunk
        // records, in chunk order (deterministic), into the shard record.
        __threadfence();
        __syncthreads();
        if (t == 0) sm.last = (atomicAdd(p.counter, 1u) == (unsigned)(p.nchunks - 1));
        __syncthreads();
        if (sm.last) {
            __threadfence();
            V F;
            M Mm;
            range_reduce<Op, NT>(p.chunkRec, 0, p.nchunks, sm.vs, sm.ms, F, Mm);
            if (t == 0) {
                double rec[R];
#pragma unroll
                for (int q = 0; q < W; ++q) rec[q] = F.x[q];
                map_to<Op>(Mm, rec + W);
                for (int q = 0; q < R; ++q) p.partial[q] = rec[q];
                *p.counter = 0u;  // self-cleaning for the next call
            }
        }
    }
}

// =============================================================================
// K_R' (rs-dependent operators): per chunk the composed reverse map with the
// TRUE rs — the forward prefix entering every tile (tileP, from the forward
// pre-pass K_F + scan_tile_prefix) and a warp-0 row scan give rs entering each
// row; the maps are then built as for the other operators.
// =============================================================================
template <class Op, class T, int NT, int S>
__global__ void __launch_bounds__(NT, 1) scan_reduce_rs(const __grid_constant__ CUtensorMap tm_as,
                                                        const __grid_constant__ CUtensorMap tm_yb,
                                                        const ChunkParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, NW = NT / 32, R = Op::W + Op::kMapD;
    constexpr int NB = 2;
    constexpr int BUF = NT * kRowBytes, STG = NB * BUF;
    static_assert(NW >= 2, "needs a forward and a reverse scan warp");

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = smem_align1024(smem_raw);
    ReduceSmem<Op, NT, S> &sm = *reinterpret_cast<ReduceSmem<Op, NT, S> *>(base + S * STG);

    const int t = threadIdx.x, warp = t >> 5;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < S && s < k; ++s) issue_tile<NT, NB>(p, t0 + s, &sm.bar[s], base + s * STG, &tm_as, &tm_yb, &tm_yb);
    }
    __syncthreads();

    M Mc = Op::map_id();  // kept by warp 1
    for (int64_t i = 0; i < k; ++i) {
        const int64_t tile = t0 + i;
        const int s = (int)(i % S);
        V Ftile = Op::fwd_id();
        if (warp == 0) {
#pragma unroll
            for (int q = 0; q < W; ++q) Ftile.x[q] = ld_cg(p.tileP + tile * W + q);
        }
        mbar_wait(&sm.bar[s], (uint32_t)((i / S) & 1));
        unsigned char *sA = base + s * STG;
        unsigned char *sY = sA + BUF;
        const bool last = (tile == p.ntiles - 1);
        if (last && p.tail_bytes) {
            if (t == (int)(p.full_rows - tile * NT)) {
                load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
            }
            __syncthreads();
        }
        const int64_t e0 = (tile * NT + t) * G::EPR;
        put_v<Op, NT>(sm.rv, t, row_fwd<Op, T, true>(sA, t, e0, last, p.n));
        __syncthreads();  // (also: warp 1 is done with the previous tile's maps)
        if (warp == 0) warp_excl_fwd_rows<Op, NT>(sm.rv, Ftile);
        __syncthreads();
        M rowM = row_map_rs<Op, T>(sA, sY, t, e0, last, p.n, get_v<Op, NT>(sm.rv, t));
        __syncthreads();  // stage s consumed
        if (t == 0 && i + S < k) issue_tile<NT, NB>(p, tile + S, &sm.bar[s], sA, &tm_as, &tm_yb, &tm_yb);
        put_m<Op, NT>(sm.rm, t, rowM);
        __syncthreads();
        if (warp == 1) Mc = Op::compose(Mc, warp_reduce_rev_rows<Op, NT>(sm.rm));
    }
    if (t == 32) {
        double rec[R];
        const V id = Op::fwd_id();
#pragma unroll
        for (int q = 0; q < W; ++q) rec[q] = id.x[q];
        map_to<Op>(Mc, rec + W);
        st_rec<R>(p.chunkRec + c * R, rec);
    }
    if (p.partial) {
        // multi-GPU (second exchange): the last CTA composes the chunk maps, in
        // chunk order, into the shard record [identity | M_shard]
        __threadfence();
        __syncthreads();
        if (t == 0) sm.last = (atomicAdd(p.counter, 1u) == (unsigned)(p.nchunks - 1));
        __syncthreads();
        if (sm.last) {
            __threadfence();
            V F;
            M Mm;
            range_reduce<Op, NT>(p.chunkRec, 0, p.nchunks, sm.vs, sm.ms, F, Mm);
            if (t == 0) {
                double rec[R];
                const V id = Op::fwd_id();
#pragma unroll
                for (int q = 0; q < W; ++q) rec[q] = id.x[q];
                map_to<Op>(Mm, rec + W);
                for (int q = 0; q < R; ++q) p.partial[q] = rec[q];
                *p.counter = 0u;
            }
        }
    }
}

// =============================================================================
// K_C: return sweep over the chunk, right to left
// =============================================================================
template <class Op, class T, int NT, int S, bool FWD, bool ACC, bool YS, bool YL = false, bool RS = false>
__global__ void __launch_bounds__(NT, 1) scan_apply(const __grid_constant__ CUtensorMap tm_as,
                                                    const __grid_constant__ CUtensorMap tm_yb,
                                                    const __grid_constant__ CUtensorMap tm_ab,
                                                    const __grid_constant__ CUtensorMap tm_ys,
                                                    const ChunkParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, NW = NT / 32;
    // loaded buffers: [A][Y][C] (output written over Y); YL: [A][C] plus an
    // output-only buffer O after them
    constexpr int NB = YL ? (FWD ? 1 : 0) + (ACC ? 1 : 0) : (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
    constexpr int NBA = YL ? NB + 1 : NB;
    constexpr int BUF = NT * kRowBytes, STG = NBA * BUF;
    static_assert(NW >= 2, "needs a forward and a reverse scan warp");

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *const sbase = smem_align1024(smem_raw);
    ApplySmem<Op, NT, S> &sm = *reinterpret_cast<ApplySmem<Op, NT, S> *>(sbase + S * STG);
    unsigned char *base = tile_base<VJP_APPLY_TILE>(sbase);
    const V yl = YL ? load_ylast<Op, T>(p.ylast) : Op::fwd_id();

    const int t = threadIdx.x, warp = t >> 5;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    const CUtensorMap *m0 = YL ? (FWD ? &tm_as : &tm_ab) : (FWD ? &tm_as : &tm_yb);
    const CUtensorMap *m1 = YL ? &tm_ab : (FWD ? &tm_yb : &tm_ab);
    const CUtensorMap *m2 = &tm_ab;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < S && s < k; ++s) issue_tile<NT, NB>(p, t1 - 1 - s, &sm.bar[s], base + s * STG, m0, m1, m2);
    }

    // ---- carries: shard level (multi-GPU) then chunk level ----
    V Fsh = Op::fwd_id();
    V Hin;
#pragma unroll
    for (int q = 0; q < W; ++q) Hin.x[q] = 0.0;
    if (p.world > 1) shard_carries<Op>(p.gathered, p.rank, p.world, Fsh, Hin);
    V X;  // H entering the current tile from the right (used by warp 1)
    {
        V Fpre, Fdummy;
        M Mdummy, Mpost;
        range_reduce<Op, NT>(p.chunkRec, 0, c, sm.vs, sm.ms, Fpre, Mdummy);
        range_reduce<Op, NT>(p.chunkRec, c + 1, p.nchunks, sm.vs, sm.ms, Fdummy, Mpost);
        X = Op::apply(Mpost, Hin);
        if constexpr (FWD && !RS) {  // (RS: tileP comes from the forward pre-pass)
            // forward exclusive prefix of every tile of the chunk -> tileP
            V Fch = Op::fwd(Fsh, Fpre);
            const int64_t per = (k + NT - 1) / NT;
            V f = Op::fwd_id();
            for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
                V v;
#pragma unroll
                for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
                f = Op::fwd(f, v);
            }
            V tot;
            V ex = block_excl_fwd<Op, NW>(f, sm.vs, tot);
            V r = Op::fwd(Fch, ex);
            for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
#pragma unroll
                for (int q = 0; q < W; ++q) st_cg(p.tileP + j * W + q, r.x[q]);
                V v;
#pragma unroll
                for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
                r = Op::fwd(r, v);
            }
            __threadfence_block();
        }
    }
    __syncthreads();

    for (int64_t i = 0; i < k; ++i) {
        const int64_t tile = t1 - 1 - i;
        const int s = (int)(i % S);
        V Ftile = Op::fwd_id();
        if (FWD && warp == 0) {
#pragma unroll
            for (int q = 0; q < W; ++q) Ftile.x[q] = ld_cg(p.tileP + tile * W + q);
        }
        mbar_wait(&sm.bar[s], (uint32_t)((i / S) & 1));
        unsigned char *sA = base + s * STG;
        unsigned char *sY = sA + (FWD ? BUF : 0);                                  // not YL
        unsigned char *sC = YL ? sA + (FWD ? BUF : 0) : sY + BUF;
        unsigned char *sO = YL ? sA + (size_t)NB * BUF : sY;                       // output tile
        const bool last = (tile == p.ntiles - 1);
        const int prow = (int)(p.full_rows - tile * NT);
        const bool has_partial = last && p.tail_bytes && t == prow;
        if (last && p.tail_bytes) {
            if (has_partial) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                if (!YL) load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
                if (ACC) load_partial_row(sC, t, p.as_bar, p.full_rows, p.tail_bytes);
            }
            __syncthreads();
        }
        const int64_t e0 = (tile * NT + t) * G::EPR;

        if constexpr (RS) {
            // rs-dependent maps: forward row scan first, then maps with the true rs
            put_v<Op, NT>(sm.rv, t, row_fwd<Op, T, true>(sA, t, e0, last, p.n));
            __syncthreads();
            if (warp == 0) warp_excl_fwd_rows<Op, NT>(sm.rv, Ftile);
            __syncthreads();
            put_m<Op, NT>(sm.rm, t, row_map_rs<Op, T>(sA, sY, t, e0, last, p.n, get_v<Op, NT>(sm.rv, t)));
            __syncthreads();
            if (warp == 1) X = warp_excl_rev_rows<Op, NT>(sm.rm, X);
            __syncthreads();
        } else {
            // phase 1: row aggregates -> shared memory
            // (MAT2 only: 1.668 -> 1.634 ms per call; LINREC measured 0.005 ms slower)
            if constexpr (FWD && (VJP_APPLY_FUSEDROW != 0) && std::is_same<Op, OpMat2>::value) {
                V rf;
                M rmap;
                row_fwd_map<Op, T, YL>(sA, sY, t, e0, last, p.n, &yl, rf, rmap);
                put_v<Op, NT>(sm.rv, t, rf);
                put_m<Op, NT>(sm.rm, t, rmap);
            } else {
                if (FWD) put_v<Op, NT>(sm.rv, t, row_fwd<Op, T, FWD>(sA, t, e0, last, p.n));
                put_m<Op, NT>(sm.rm, t, row_map<Op, T, FWD, YL>(sA, sY, t, e0, last, p.n, &yl));
            }
            __syncthreads();
            // block scans: warp 0 forward (rs entering each row), warp 1 reverse (H entering each row)
            if (FWD && warp == 0) warp_excl_fwd_rows<Op, NT>(sm.rv, Ftile);
            if (warp == 1) X = warp_excl_rev_rows<Op, NT>(sm.rm, X);
            __syncthreads();
        }

        // phase 2: re-execute the primal scan over the row, then outputs right to left
        V rsp[G::EPR];
        if constexpr (FWD) {
            V r = get_v<Op, NT>(sm.rv, t);
#pragma unroll
            for (int g = 0; g < G::NG; ++g) {
                uint32_t w[G::GB / 4];
                lds_group<G::GB>(sA, t, g, w);
#pragma unroll
                for (int e = 0; e < G::EG; ++e) {
                    V a = dec<T, W>(w + e * (G::ES / 4));
                    rsp[g * G::EG + e] = r;
                    r = Op::fwd(r, a);
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < G::EPR; ++q) rsp[q] = Op::fwd_id();
        }
        V Xr = get_v<Op, NT>(sm.rm, t);
#pragma unroll
        for (int g = G::NG - 1; g >= 0; --g) {
            uint32_t wa[G::GB / 4], wy[G::GB / 4], wc[G::GB / 4], wo[G::GB / 4], wz[G::GB / 4];
            if (FWD) lds_group<G::GB>(sA, t, g, wa);
            if (!YL) lds_group<G::GB>(sY, t, g, wy);
            if (ACC) lds_group<G::GB>(sC, t, g, wc);
#pragma unroll
            for (int e = G::EG - 1; e >= 0; --e) {
                const int q = g * G::EG + e;
                V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
                V y;
                if (YL) {
#pragma unroll
                    for (int z = 0; z < W; ++z) y.x[z] = (e0 + q == p.n - 1) ? yl.x[z] : 0.0;
                } else {
                    y = dec<T, W>(wy + e * (G::ES / 4));
                }
                V gv;
#pragma unroll
                for (int z = 0; z < W; ++z) gv.x[z] = y.x[z] + Xr.x[z];  // rbar_i = ybar_i + H_{i+1}
                V o = Op::out(rsp[q], a, gv);
                if (Op::kFirstSpecial && p.global_first && e0 + q == 0) o = gv;
                if (ACC) {
                    V cc = dec<T, W>(wc + e * (G::ES / 4));
#pragma unroll
                    for (int z = 0; z < W; ++z) o.x[z] += cc.x[z];
                }
                enc<T, W>(o, wo + e * (G::ES / 4));
                if (YS) enc<T, W>(Op::fwd(rsp[q], a), wz + e * (G::ES / 4));
                if (!last || e0 + q < p.n) Xr = Op::pass_left(rsp[q], a, gv);  // H_i = J_L^T rbar_i
            }
            sts_group<G::GB>(sO, t, g, wo);
            if (YS) sts_group<G::GB>(sA, t, g, wz);
        }
        if (has_partial) {
            store_partial_row(sO, t, p.as_bar, p.full_rows, p.tail_bytes);
            if (YS) store_partial_row(sA, t, p.ys, p.full_rows, p.tail_bytes);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (t == 0) {
            if (chunk_tile_rows<NT>(p, tile) > 0) {
                tma_store_2d(&tm_ab, sO, 0, (int)(tile * NT));
                if (YS) tma_store_2d(&tm_ys, sA, 0, (int)(tile * NT));
            }
            tma_store_commit();
            // refill the PREVIOUS tile's stage (its store has had a whole tile to drain)
            if (i >= 1 && i - 1 + S < k) {
                tma_store_wait_read1();
                const int sp = (int)((i - 1) % S);
                issue_tile<NT, NB>(p, t1 - 1 - (i - 1 + S), &sm.bar[sp], base + sp * STG, m0, m1, m2);
            }
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the record of an EMPTY shard (multi-GPU split with n_local = 0): the neutral
// forward element and the identity reverse map, so the carry combination of
// the other ranks passes straight through it
template <class Op>
__global__ void scan_identity_record(double *rec) {
    if (threadIdx.x == 0) {
        const typename Op::Val e = Op::fwd_id();
#pragma unroll
        for (int q = 0; q < Op::W; ++q) rec[q] = e.x[q];
        map_to<Op>(Op::map_id(), rec + Op::W);
    }
}

// ordered combination of the chunk records' forward parts (the primal
// reduction of the general reduce rule), one CTA
template <class Op, class T, int NT>
__global__ void __launch_bounds__(NT) scan_chunks_total(const ChunkParams p, T *y) {
    __shared__ typename Op::Val vs[NT / 32 + 1];
    __shared__ typename Op::Map ms[NT / 32 + 1];
    typename Op::Val F;
    typename Op::Map M;
    range_reduce<Op, NT>(p.chunkRec, 0, p.nchunks, vs, ms, F, M);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < Op::W; ++q) y[q] = (T)F.x[q];
    }
}

}  // namespace vjpk
