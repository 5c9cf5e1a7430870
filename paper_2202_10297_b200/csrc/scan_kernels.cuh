// scan_kernels.cuh — the vjp_scan kernels (sec 5.2) for sm_100a.
//
// Two kernels, each a single sweep with decoupled look-back over tiles:
//   pass 1 (forward re-execution, "the forward sweep is the original
//           scan"): per-tile aggregate of `as` under (.) and its inclusive
//           prefix by forward look-back.  rs is NOT stored (tape-free,
//           P:127-149); only one W-vector per tile is written.  With REV (multi-
//           GPU) it also reads ys_bar and carries the reverse-map aggregate so
//           the shard's record can be exchanged.
//   pass 2 (return sweep): re-executes the primal scan inside the
//           tile from the pass-1 prefix (registers only), builds the per-element
//           affine maps, reverse-scans them (thread -> warp -> block -> look-back
//           to the right) and writes as_bar (and optionally ys).
// For ADD without ys, pass 1 is skipped (closed form P:1233-1236: a single
// reverse suffix-sum sweep that never reads `as`).
//
// Tiles: 256 threads x 128-byte rows per array (32 KB), moved by TMA with the
// 128B swizzle so that thread t reads its own row with conflict-free 16-byte
// shared loads.  The partial last row (n*ES not a multiple of 128) is moved by
// plain loads/stores of its owner thread.
#pragma once

#include "common.cuh"
#include "scan_ops.cuh"

namespace vjpk {

struct ScanParams {
    int64_t n;           // local elements
    int64_t full_rows;   // 128-byte rows fully inside the array (TMA-covered)
    int32_t ntiles;
    int32_t tail_bytes;  // bytes of the partial row (0..127)
    const void *as;
    const void *ys_bar;
    void *as_bar;
    void *ys;
    uint32_t *counters;  // [0] pass-1 ticket, [1] pass-2 ticket
    uint32_t *flags1;
    uint32_t *flags2;
    double *p1_agg;   // [ntiles][R1]  R1 = W (+ kMapD with REV)
    double *p1_inc;
    double *p2_agg;   // [ntiles][kMapD]
    double *p2_inc;
    double *partial;          // pass 1: this shard's record (W + kMapD doubles)
    const double *gathered;   // pass 2: world records (NULL when world == 1)
    int32_t rank, world;
    int32_t global_first;     // this shard holds global element 0
};

template <class Op, class T>
struct Geo {
    static constexpr int W = Op::W;
    static constexpr int ES = W * (int)sizeof(T);  // element bytes
    static constexpr int EPR = kRowBytes / ES;     // elements per row / thread
    static constexpr int TILE_E = EPR * kThreads;  // elements per tile
    static constexpr int GB = ES >= 16 ? ES : 16;  // bytes per access group
    static constexpr int NG = kRowBytes / GB;      // groups per row
    static constexpr int EG = GB / ES;             // elements per group
};

// ---- element <-> words ---------------------------------------------------
template <class T, int W>
__device__ __forceinline__ Vec<W> dec(const uint32_t *w) {
    Vec<W> v;
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int s = 0; s < W; ++s) v.x[s] = __hiloint2double((int)w[2 * s + 1], (int)w[2 * s]);
    } else {
#pragma unroll
        for (int s = 0; s < W; ++s) v.x[s] = (double)__uint_as_float(w[s]);
    }
    return v;
}
template <class T, int W>
__device__ __forceinline__ void enc(const Vec<W> &v, uint32_t *w) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int s = 0; s < W; ++s) {
            w[2 * s] = (uint32_t)__double2loint(v.x[s]);
            w[2 * s + 1] = (uint32_t)__double2hiint(v.x[s]);
        }
    } else {
#pragma unroll
        for (int s = 0; s < W; ++s) w[s] = __float_as_uint((float)v.x[s]);
    }
}

// load / store one access group (GB bytes = GB/16 swizzled chunks) of row t
template <int GB>
__device__ __forceinline__ void lds_group(const unsigned char *buf, int t, int g, uint32_t (&w)[GB / 4]) {
#pragma unroll
    for (int q = 0; q < GB / 16; ++q) {
        uint4 v = *reinterpret_cast<const uint4 *>(buf + swz(t, g * (GB / 16) + q));
        w[4 * q + 0] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
}
template <int GB>
__device__ __forceinline__ void sts_group(unsigned char *buf, int t, int g, const uint32_t (&w)[GB / 4]) {
#pragma unroll
    for (int q = 0; q < GB / 16; ++q)
        *reinterpret_cast<uint4 *>(buf + swz(t, g * (GB / 16) + q)) =
            make_uint4(w[4 * q + 0], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// ---- shuffles of Val / Map -------------------------------------------------
template <int W>
__device__ __forceinline__ Vec<W> shfl_up_v(const Vec<W> &v, int s) {
    Vec<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) r.x[k] = shfl_up_t(v.x[k], s);
    return r;
}
template <int W>
__device__ __forceinline__ Vec<W> shfl_down_v(const Vec<W> &v, int s) {
    Vec<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) r.x[k] = shfl_down_t(v.x[k], s);
    return r;
}
template <int W>
__device__ __forceinline__ Vec<W> shfl_idx_v(const Vec<W> &v, int l) {
    Vec<W> r;
#pragma unroll
    for (int k = 0; k < W; ++k) r.x[k] = shfl_idx_t(v.x[k], l);
    return r;
}
template <class Op>
__device__ __forceinline__ typename Op::Map shfl_down_m(const typename Op::Map &m, int s) {
    typename Op::Map r;
    const double *a = reinterpret_cast<const double *>(&m);
    double *b = reinterpret_cast<double *>(&r);
#pragma unroll
    for (int k = 0; k < Op::kMapD; ++k) b[k] = shfl_down_t(a[k], s);
    return r;
}
template <class Op>
__device__ __forceinline__ typename Op::Map shfl_up_m(const typename Op::Map &m, int s) {
    typename Op::Map r;
    const double *a = reinterpret_cast<const double *>(&m);
    double *b = reinterpret_cast<double *>(&r);
#pragma unroll
    for (int k = 0; k < Op::kMapD; ++k) b[k] = shfl_up_t(a[k], s);
    return r;
}
template <class Op>
__device__ __forceinline__ typename Op::Map shfl_idx_m(const typename Op::Map &m, int l) {
    typename Op::Map r;
    const double *a = reinterpret_cast<const double *>(&m);
    double *b = reinterpret_cast<double *>(&r);
#pragma unroll
    for (int k = 0; k < Op::kMapD; ++k) b[k] = shfl_idx_t(a[k], l);
    return r;
}

// ---- block-wide primitives (256 threads, 8 warps) --------------------------
// exclusive forward scan of Val under fwd(); returns the thread's exclusive
// prefix; `total` receives the block aggregate.  Uses scratch of 9 Vals.
template <class Op, int NW = kThreads / 32>
__device__ __forceinline__ typename Op::Val block_excl_fwd(typename Op::Val v, typename Op::Val *scr,
                                                           typename Op::Val &total) {
    using V = typename Op::Val;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    V inc = v;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        V o = shfl_up_v(inc, s);
        if (lane >= s) inc = Op::fwd(o, inc);
    }
    if (lane == 31) scr[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        V w = lane < NW ? scr[lane] : Op::fwd_id();
        V wi = w;
#pragma unroll
        for (int s = 1; s < NW; s <<= 1) {
            V o = shfl_up_v(wi, s);
            if (lane >= s) wi = Op::fwd(o, wi);
        }
        V we = shfl_up_v(wi, 1);
        if (lane == 0) we = Op::fwd_id();
        if (lane < NW) scr[lane] = we;
        if (lane == NW - 1) scr[NW] = wi;
    }
    __syncthreads();
    V ex = shfl_up_v(inc, 1);
    if (lane == 0) ex = Op::fwd_id();
    V r = Op::fwd(scr[warp], ex);
    total = scr[NW];
    return r;
}

// ordered block reduce (fwd); result valid in all threads.
template <class Op, int NW = kThreads / 32>
__device__ __forceinline__ typename Op::Val block_reduce_fwd(typename Op::Val v, typename Op::Val *scr) {
    using V = typename Op::Val;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        V o = shfl_down_v(v, s);
        if (lane + s < 32) v = Op::fwd(v, o);
    }
    if (lane == 0) scr[warp] = v;
    __syncthreads();
    V r = scr[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) r = Op::fwd(r, scr[w]);
    __syncthreads();
    return r;
}

// exclusive REVERSE scan of maps: thread t gets M_{t+1} o ... o M_255 (identity
// for t = 255); `total` = M_0 o ... o M_255.  Scratch of 9 Maps.
template <class Op, int NW = kThreads / 32>
__device__ __forceinline__ typename Op::Map block_excl_rev(typename Op::Map m, typename Op::Map *scr,
                                                           typename Op::Map &total) {
    using M = typename Op::Map;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    M inc = m;  // becomes M_lane o ... o M_31 (within warp)
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        M o = shfl_down_m<Op>(inc, s);
        if (lane + s < 32) inc = Op::compose(inc, o);
    }
    if (lane == 0) scr[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        M w = lane < NW ? scr[lane] : Op::map_id();
        M wi = w;  // W_lane o ... o W_{NW-1}
#pragma unroll
        for (int s = 1; s < NW; s <<= 1) {
            M o = shfl_down_m<Op>(wi, s);
            if (lane + s < NW) wi = Op::compose(wi, o);
        }
        M we = shfl_down_m<Op>(wi, 1);
        if (lane == NW - 1) we = Op::map_id();
        if (lane < NW) scr[lane] = we;
        if (lane == 0) scr[NW] = wi;
    }
    __syncthreads();
    M ex = shfl_down_m<Op>(inc, 1);
    if (lane == 31) ex = Op::map_id();
    M r = Op::compose(ex, scr[warp]);
    total = scr[NW];
    return r;
}

// ordered block reduce of maps (M_0 o ... o M_255), valid in all threads.
template <class Op, int NW = kThreads / 32>
__device__ __forceinline__ typename Op::Map block_reduce_rev(typename Op::Map m, typename Op::Map *scr) {
    using M = typename Op::Map;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        M o = shfl_down_m<Op>(m, s);
        if (lane + s < 32) m = Op::compose(m, o);
    }
    if (lane == 0) scr[warp] = m;
    __syncthreads();
    M r = scr[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) r = Op::compose(r, scr[w]);
    __syncthreads();
    return r;
}

// ---- record I/O (L2-only) ---------------------------------------------------
template <int K>
__device__ __forceinline__ void st_rec(double *dst, const double *src) {
#pragma unroll
    for (int k = 0; k < K; ++k) st_cg(dst + k, src[k]);
}
template <int K>
__device__ __forceinline__ void ld_rec(const double *src, double *dst) {
#pragma unroll
    for (int k = 0; k < K; ++k) dst[k] = ld_cg(src + k);
}

// ---- TMA tile issue helper --------------------------------------------------
__device__ __forceinline__ int tile_full_rows(const ScanParams &p, int tile) {
    int64_t r = p.full_rows - (int64_t)tile * kThreads;
    return r <= 0 ? 0 : (r >= kThreads ? kThreads : (int)r);
}

// Partial row (bytes past full_rows*128): its owner thread copies it with
// plain accesses into the swizzled tile (after TMA zero-filled that row).
__device__ __forceinline__ void load_partial_row(unsigned char *buf, int t, const void *src,
                                                 int64_t row, int bytes) {
    const uint32_t *s = reinterpret_cast<const uint32_t *>(static_cast<const unsigned char *>(src) + row * kRowBytes);
    for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
        for (int q = 0; q < 4; ++q) {
            int b = c * 16 + q * 4;
            w[q] = b < bytes ? s[b / 4] : 0u;
        }
        *reinterpret_cast<uint4 *>(buf + swz(t, c)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}
__device__ __forceinline__ void store_partial_row(const unsigned char *buf, int t, void *dst, int64_t row,
                                                  int bytes) {
    uint32_t *d = reinterpret_cast<uint32_t *>(static_cast<unsigned char *>(dst) + row * kRowBytes);
    for (int c = 0; c < 8; ++c) {
        uint4 v = *reinterpret_cast<const uint4 *>(buf + swz(t, c));
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
        for (int q = 0; q < 4; ++q) {
            int b = c * 16 + q * 4;
            if (b < bytes) d[b / 4] = w[q];
        }
    }
}

// =============================================================================
// PASS 1: forward tile aggregates + forward decoupled look-back.
// =============================================================================
template <class Op, class T, bool FWD, bool REV>
__global__ void __launch_bounds__(kThreads) scan_pass1(const __grid_constant__ CUtensorMap tm_as,
                                                       const __grid_constant__ CUtensorMap tm_yb,
                                                       const ScanParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W;
    constexpr int R1 = (FWD ? W : 0) + (REV ? Op::kMapD : 0);
    constexpr int NB = (FWD ? 1 : 0) + (REV ? 1 : 0);

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = smem_align1024(smem_raw);
    unsigned char *sA = base;
    unsigned char *sY = base + (FWD ? kTileBytes : 0);
    struct Small {
        uint64_t bar;
        int tile;
        V vs[9];
        M ms[9];
    };
    Small &sm = *reinterpret_cast<Small *>(base + NB * kTileBytes);

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        int tile = (int)atomicAdd(&p.counters[0], 1u);
        sm.tile = tile;
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
        int rows = tile_full_rows(p, tile);
        if (rows > 0) {
            mbar_arrive_expect_tx(&sm.bar, NB * kTileBytes);
            if (FWD) tma_load_2d(sA, &tm_as, &sm.bar, 0, tile * kThreads);
            if (REV) tma_load_2d(sY, &tm_yb, &sm.bar, 0, tile * kThreads);
        }
    }
    __syncthreads();
    const int tile = sm.tile;
    const int rows = tile_full_rows(p, tile);
    if (rows > 0) mbar_wait(&sm.bar, 0);
    const int64_t prow = p.full_rows - (int64_t)tile * kThreads;  // local row of the partial row
    if (p.tail_bytes && prow == t) {
        if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
        if (REV) load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
    }
    __syncthreads();

    const int64_t e0 = ((int64_t)tile * kThreads + t) * G::EPR;  // first element of this row
    const bool tail_tile = (tile == p.ntiles - 1);

    // thread aggregates
    V F = Op::fwd_id();
    M Mt = Op::map_id();
    if constexpr (FWD) {
#pragma unroll
        for (int g = 0; g < G::NG; ++g) {
            uint32_t w[G::GB / 4];
            lds_group<G::GB>(sA, t, g, w);
#pragma unroll
            for (int e = 0; e < G::EG; ++e) {
                V a = dec<T, W>(w + e * (G::ES / 4));
                if (!tail_tile || e0 + g * G::EG + e < p.n) F = Op::fwd(F, a);
            }
        }
    }
    if constexpr (REV) {
#pragma unroll
        for (int g = G::NG - 1; g >= 0; --g) {
            uint32_t wa[G::GB / 4], wy[G::GB / 4];
            if (FWD) lds_group<G::GB>(sA, t, g, wa);
            lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
            for (int e = G::EG - 1; e >= 0; --e) {
                V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
                V y = dec<T, W>(wy + e * (G::ES / 4));
                if (!tail_tile || e0 + g * G::EG + e < p.n) Mt = Op::compose(Op::make_map(Op::fwd_id(), a, y), Mt);
            }
        }
    }
    V Ft = FWD ? block_reduce_fwd<Op>(F, sm.vs) : F;
    M Mtile = REV ? block_reduce_rev<Op>(Mt, sm.ms) : Mt;

    // forward decoupled look-back (warp 0): inclusive_t = inclusive_{t-1} (+) agg_t
    if (warp == 0) {
        double rec[R1 > 0 ? R1 : 1];
        auto pack = [&](const V &f, const M &m, double *d) {
            int o = 0;
            if (FWD) for (int k = 0; k < W; ++k) d[o++] = f.x[k];
            if (REV) map_to<Op>(m, d + o);
        };
        V incF = Ft;
        M incM = Mtile;
        if (tile > 0) {
            if (lane == 0) {
                pack(Ft, Mtile, rec);
                st_rec<R1>(p.p1_agg + (size_t)tile * R1, rec);
                st_flag_release(&p.flags1[tile], 1u);
            }
            V runF = Op::fwd_id();  // prefix of the tiles before `tile`
            M runM = Op::map_id();
            int j0 = tile - 1;
            while (true) {
                int idx = j0 - lane;
                uint32_t f;
                do {
                    f = idx >= 0 ? ld_flag(&p.flags1[idx]) : 2u;
                } while (!__all_sync(0xffffffffu, f != 0u));
                fence_acq_rel_gpu();
                unsigned incl = __ballot_sync(0xffffffffu, f == 2u);
                int L = incl ? (__ffs(incl) - 1) : 32;
                V lf = Op::fwd_id();
                M lm = Op::map_id();
                if (lane <= L && idx >= 0) {
                    double d[R1 > 0 ? R1 : 1];
                    ld_rec<R1>((lane == L ? p.p1_inc : p.p1_agg) + (size_t)idx * R1, d);
                    int o = 0;
                    if (FWD) for (int k = 0; k < W; ++k) lf.x[k] = d[o++];
                    if (REV) lm = map_from<Op>(d + o);
                }
                // lane j holds tile j0-j; combine farther (left) tiles on the left
#pragma unroll
                for (int s = 1; s < 32; s <<= 1) {
                    V of = shfl_down_v(lf, s);
                    M om = shfl_down_m<Op>(lm, s);
                    if (lane + s < 32) {
                        if (FWD) lf = Op::fwd(of, lf);
                        if (REV) lm = Op::compose(om, lm);
                    }
                }
                lf = shfl_idx_v(lf, 0);
                lm = shfl_idx_m<Op>(lm, 0);
                if (FWD) runF = Op::fwd(lf, runF);
                if (REV) runM = Op::compose(lm, runM);
                if (L < 32) break;
                j0 -= 32;
            }
            if (FWD) incF = Op::fwd(runF, Ft);
            if (REV) incM = Op::compose(runM, Mtile);
        }
        if (lane == 0) {
            pack(incF, incM, rec);
            st_rec<R1>(p.p1_inc + (size_t)tile * R1, rec);
            st_flag_release(&p.flags1[tile], 2u);
            if (tile == p.ntiles - 1 && p.partial) {
                // shard record: [fwd aggregate (W) | reverse map aggregate (kMapD)]
                V f = FWD ? incF : Op::fwd_id();
                M m = REV ? incM : Op::map_id();
                for (int k = 0; k < W; ++k) p.partial[k] = f.x[k];
                map_to<Op>(m, p.partial + W);
            }
        }
    }
}

// =============================================================================
// PASS 2: return sweep.
// =============================================================================
template <class Op, class T, bool FWD, bool ACC, bool YS>
__global__ void __launch_bounds__(kThreads, 2) scan_pass2(const __grid_constant__ CUtensorMap tm_as,
                                                          const __grid_constant__ CUtensorMap tm_yb,
                                                          const __grid_constant__ CUtensorMap tm_ab,
                                                          const __grid_constant__ CUtensorMap tm_ys,
                                                          const ScanParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W;
    constexpr int NB = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = smem_align1024(smem_raw);
    unsigned char *sA = base;
    unsigned char *sY = base + (FWD ? kTileBytes : 0);
    unsigned char *sC = sY + kTileBytes;
    struct Small {
        uint64_t bar;
        int tile;
        V ftile;
        V xin;
        V vs[9];
        M ms[9];
    };
    Small &sm = *reinterpret_cast<Small *>(base + NB * kTileBytes);

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        int tile = p.ntiles - 1 - (int)atomicAdd(&p.counters[1], 1u);
        sm.tile = tile;
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
        int rows = tile_full_rows(p, tile);
        if (rows > 0) {
            mbar_arrive_expect_tx(&sm.bar, NB * kTileBytes);
            if (FWD) tma_load_2d(sA, &tm_as, &sm.bar, 0, tile * kThreads);
            tma_load_2d(sY, &tm_yb, &sm.bar, 0, tile * kThreads);
            if (ACC) tma_load_2d(sC, &tm_ab, &sm.bar, 0, tile * kThreads);
        }
    }
    __syncthreads();
    const int tile = sm.tile;
    const int rows = tile_full_rows(p, tile);

    // shard-level carries (multi-GPU) and this tile's forward prefix
    V Hin;
    for (int k = 0; k < W; ++k) Hin.x[k] = 0.0;
    V Fsh = Op::fwd_id();
    if (p.world > 1) shard_carries<Op>(p.gathered, p.rank, p.world, Fsh, Hin);
    if constexpr (FWD) {
        if (t == 0) {
            V f = Fsh;
            if (tile > 0) {
                V pre;
                const int R1s = p.world > 1 ? (W + Op::kMapD) : W;
                for (int k = 0; k < W; ++k) pre.x[k] = ld_cg(p.p1_inc + (size_t)(tile - 1) * R1s + k);
                f = Op::fwd(Fsh, pre);
            }
            sm.ftile = f;
        }
    }
    if (rows > 0) mbar_wait(&sm.bar, 0);
    const int64_t prow = p.full_rows - (int64_t)tile * kThreads;
    const bool has_partial = p.tail_bytes && prow == t;
    if (has_partial) {
        if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
        load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
        if (ACC) load_partial_row(sC, t, p.as_bar, p.full_rows, p.tail_bytes);
    }
    __syncthreads();

    const int64_t e0 = ((int64_t)tile * kThreads + t) * G::EPR;
    const bool tail_tile = (tile == p.ntiles - 1);

    // ---- forward re-execution inside the tile (registers only) ----
    V rsp[G::EPR];  // rs_{i-1} for each element of this row
    if constexpr (FWD) {
        V F = Op::fwd_id();
#pragma unroll
        for (int g = 0; g < G::NG; ++g) {
            uint32_t w[G::GB / 4];
            lds_group<G::GB>(sA, t, g, w);
#pragma unroll
            for (int e = 0; e < G::EG; ++e) {
                V a = dec<T, W>(w + e * (G::ES / 4));
                if (!tail_tile || e0 + g * G::EG + e < p.n) F = Op::fwd(F, a);
            }
        }
        V tot;
        V ex = block_excl_fwd<Op>(F, sm.vs, tot);
        V r = Op::fwd(sm.ftile, ex);
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
        for (int k = 0; k < G::EPR; ++k) rsp[k] = Op::fwd_id();
    }

    // ---- thread map: M_e0 o M_e0+1 o ... o M_e0+EPR-1 ----
    M Tm = Op::map_id();
#pragma unroll
    for (int g = G::NG - 1; g >= 0; --g) {
        uint32_t wa[G::GB / 4], wy[G::GB / 4];
        if (FWD) lds_group<G::GB>(sA, t, g, wa);
        lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
        for (int e = G::EG - 1; e >= 0; --e) {
            V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
            V y = dec<T, W>(wy + e * (G::ES / 4));
            if (!tail_tile || e0 + g * G::EG + e < p.n)
                Tm = Op::compose(Op::make_map(rsp[g * G::EG + e], a, y), Tm);
        }
    }
    M Agg;
    M Nt = block_excl_rev<Op>(Tm, sm.ms, Agg);

    // ---- reverse decoupled look-back (warp 0) ----
    if (warp == 0) {
        constexpr int MD = Op::kMapD;
        V xin = Hin;
        if (tile < p.ntiles - 1) {
            if (lane == 0) {
                double rec[MD];
                map_to<Op>(Agg, rec);
                st_rec<MD>(p.p2_agg + (size_t)tile * MD, rec);
                st_flag_release(&p.flags2[tile], 1u);
            }
            M run = Op::map_id();
            int j0 = tile + 1;
            while (true) {
                int idx = j0 + lane;
                uint32_t f;
                do {
                    f = idx < p.ntiles ? ld_flag(&p.flags2[idx]) : 2u;
                } while (!__all_sync(0xffffffffu, f != 0u));
                fence_acq_rel_gpu();
                unsigned incl = __ballot_sync(0xffffffffu, f == 2u);
                int L = incl ? (__ffs(incl) - 1) : 32;
                M lm = Op::map_id();
                if (lane <= L && idx < p.ntiles) {
                    double d[MD];
                    ld_rec<MD>((lane == L ? p.p2_inc : p.p2_agg) + (size_t)idx * MD, d);
                    lm = map_from<Op>(d);
                }
#pragma unroll
                for (int s = 1; s < 32; s <<= 1) {
                    M o = shfl_down_m<Op>(lm, s);
                    if (lane + s < 32) lm = Op::compose(lm, o);
                }
                lm = shfl_idx_m<Op>(lm, 0);
                run = Op::compose(run, lm);
                if (L < 32) break;
                j0 += 32;
            }
            V z;
            for (int k = 0; k < W; ++k) z.x[k] = 0.0;
            xin = Op::apply(run, z);
        }
        if (lane == 0) {
            double rec[MD];
            map_to<Op>(Op::constant(Op::apply(Agg, xin)), rec);
            st_rec<MD>(p.p2_inc + (size_t)tile * MD, rec);
            st_flag_release(&p.flags2[tile], 2u);
            sm.xin = xin;
        }
    }
    __syncthreads();

    // ---- outputs, right to left ----
    V X = Op::apply(Nt, sm.xin);  // H entering this row from the right
#pragma unroll
    for (int g = G::NG - 1; g >= 0; --g) {
        uint32_t wa[G::GB / 4], wy[G::GB / 4], wc[G::GB / 4], wo[G::GB / 4], ws[G::GB / 4];
        if (FWD) lds_group<G::GB>(sA, t, g, wa);
        lds_group<G::GB>(sY, t, g, wy);
        if (ACC) lds_group<G::GB>(sC, t, g, wc);
#pragma unroll
        for (int e = G::EG - 1; e >= 0; --e) {
            const int k = g * G::EG + e;
            V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
            V y = dec<T, W>(wy + e * (G::ES / 4));
            const bool valid = !tail_tile || e0 + k < p.n;
            V gv;
#pragma unroll
            for (int s = 0; s < W; ++s) gv.x[s] = y.x[s] + X.x[s];  // rbar_i = ybar_i + H_{i+1}
            V o = Op::out(rsp[k], a, gv);
            if (Op::kFirstSpecial && p.global_first && e0 + k == 0) o = gv;
            if (ACC) {
                V c = dec<T, W>(wc + e * (G::ES / 4));
#pragma unroll
                for (int s = 0; s < W; ++s) o.x[s] += c.x[s];
            }
            enc<T, W>(o, wo + e * (G::ES / 4));
            if (YS) enc<T, W>(Op::fwd(rsp[k], a), ws + e * (G::ES / 4));
            if (valid) X = Op::apply(Op::make_map(rsp[k], a, y), X);
        }
        sts_group<G::GB>(sY, t, g, wo);
        if (YS) sts_group<G::GB>(sA, t, g, ws);
    }
    if (has_partial) {
        store_partial_row(sY, t, p.as_bar, p.full_rows, p.tail_bytes);
        if (YS) store_partial_row(sA, t, p.ys, p.full_rows, p.tail_bytes);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (t == 0 && rows > 0) {
        tma_store_2d(&tm_ab, sY, 0, tile * kThreads);
        if (YS) tma_store_2d(&tm_ys, sA, 0, tile * kThreads);
        tma_store_commit();
        tma_store_wait_read0();
    }
}

}  // namespace vjpk
