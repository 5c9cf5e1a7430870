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
// The return sweep therefore reads `as` and `ys_bar` twice (K_R, K_C) — the
// same traffic the contiguous multi-GPU partition pays — in
// exchange for pure streaming kernels.  For world > 1 the chunk records are
// reduced once more into the shard record exchanged by all_gather.
#pragma once

#include "scan_kernels.cuh"

namespace vjpk {

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
};

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

// =============================================================================
// K_R: per-tile / per-chunk aggregates
// =============================================================================
template <class Op, class T, int NT, int S, bool FWD, bool REV>
__global__ void __launch_bounds__(NT, 1) scan_reduce(const __grid_constant__ CUtensorMap tm_as,
                                                     const __grid_constant__ CUtensorMap tm_yb,
                                                     const ChunkParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, NW = NT / 32, R = Op::W + Op::kMapD;
    constexpr int NB = (FWD ? 1 : 0) + (REV ? 1 : 0);
    constexpr int BUF = NT * kRowBytes, STG = NB * BUF;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    struct Small {
        uint64_t bar[S];
        int last;
        V vs[NW + 1];
        M ms[NW + 1];
    };
    Small &sm = *reinterpret_cast<Small *>(base + S * STG);

    const int t = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    const CUtensorMap *m0 = FWD ? &tm_as : &tm_yb;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < S && s < k; ++s) issue_tile<NT, NB>(p, t0 + s, &sm.bar[s], base + s * STG, m0, &tm_yb, &tm_yb);
    }
    __syncthreads();

    V Fc = Op::fwd_id();
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
                if (REV) load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
            }
            __syncthreads();
        }
        const int64_t e0 = (tile * NT + t) * G::EPR;
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
                    if (!last || e0 + g * G::EG + e < p.n) F = Op::fwd(F, a);
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
                    if (!last || e0 + g * G::EG + e < p.n) Mt = Op::compose(Op::make_map(Op::fwd_id(), a, y), Mt);
                }
            }
        }
        V Ft = FWD ? block_reduce_fwd<Op, NW>(F, sm.vs) : F;
        M Mtile = REV ? block_reduce_rev<Op, NW>(Mt, sm.ms) : Mt;
        // the block reductions end in __syncthreads: stage s is free again
        if (t == 0) {
            if (FWD) {
#pragma unroll
                for (int q = 0; q < W; ++q) st_cg(p.tileF + tile * W + q, Ft.x[q]);
            }
            if (i + S < k) issue_tile<NT, NB>(p, tile + S, &sm.bar[s], sA, m0, &tm_yb, &tm_yb);
        }
        if (FWD) Fc = Op::fwd(Fc, Ft);
        if (REV) Mc = Op::compose(Mc, Mtile);
    }
    if (t == 0) {
        double rec[R];
#pragma unroll
        for (int q = 0; q < W; ++q) rec[q] = Fc.x[q];
        map_to<Op>(Mc, rec + W);
        st_rec<R>(p.chunkRec + c * R, rec);
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
// K_C: return sweep over the chunk, right to left
// =============================================================================
template <class Op, class T, int NT, int S, bool FWD, bool ACC, bool YS>
__global__ void __launch_bounds__(NT, 1) scan_apply(const __grid_constant__ CUtensorMap tm_as,
                                                    const __grid_constant__ CUtensorMap tm_yb,
                                                    const __grid_constant__ CUtensorMap tm_ab,
                                                    const __grid_constant__ CUtensorMap tm_ys,
                                                    const ChunkParams p) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, NW = NT / 32;
    constexpr int NB = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
    constexpr int BUF = NT * kRowBytes, STG = NB * BUF;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    struct Small {
        uint64_t bar[S];
        V vs[NW + 1];
        M ms[NW + 1];
    };
    Small &sm = *reinterpret_cast<Small *>(base + S * STG);

    const int t = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    // stage buffer order: [A][Y][C]
    const CUtensorMap *m0 = FWD ? &tm_as : &tm_yb;
    const CUtensorMap *m1 = FWD ? &tm_yb : &tm_ab;
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
    V X;  // H entering the current tile from the right
    {
        V Fpre, Fdummy;
        M Mdummy, Mpost;
        range_reduce<Op, NT>(p.chunkRec, 0, c, sm.vs, sm.ms, Fpre, Mdummy);
        range_reduce<Op, NT>(p.chunkRec, c + 1, p.nchunks, sm.vs, sm.ms, Fdummy, Mpost);
        X = Op::apply(Mpost, Hin);
        if constexpr (FWD) {
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
        if constexpr (FWD) {
#pragma unroll
            for (int q = 0; q < W; ++q) Ftile.x[q] = ld_cg(p.tileP + tile * W + q);
        }
        mbar_wait(&sm.bar[s], (uint32_t)((i / S) & 1));
        unsigned char *sA = base + s * STG;
        unsigned char *sY = sA + (FWD ? BUF : 0);
        unsigned char *sC = sY + BUF;
        const bool last = (tile == p.ntiles - 1);
        const int prow = (int)(p.full_rows - tile * NT);
        const bool has_partial = last && p.tail_bytes && t == prow;
        if (last && p.tail_bytes) {
            if (has_partial) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
                if (ACC) load_partial_row(sC, t, p.as_bar, p.full_rows, p.tail_bytes);
            }
            __syncthreads();
        }
        const int64_t e0 = (tile * NT + t) * G::EPR;

        // forward re-execution inside the tile (registers only)
        V rsp[G::EPR];
        if constexpr (FWD) {
            V F = Op::fwd_id();
#pragma unroll
            for (int g = 0; g < G::NG; ++g) {
                uint32_t w[G::GB / 4];
                lds_group<G::GB>(sA, t, g, w);
#pragma unroll
                for (int e = 0; e < G::EG; ++e) {
                    V a = dec<T, W>(w + e * (G::ES / 4));
                    if (!last || e0 + g * G::EG + e < p.n) F = Op::fwd(F, a);
                }
            }
            V tot;
            V ex = block_excl_fwd<Op, NW>(F, sm.vs, tot);
            V r = Op::fwd(Ftile, ex);
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

        // thread map and its block-wide reverse exclusive scan
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
                if (!last || e0 + g * G::EG + e < p.n) Tm = Op::compose(Op::make_map(rsp[g * G::EG + e], a, y), Tm);
            }
        }
        M Agg;
        M Nt = block_excl_rev<Op, NW>(Tm, sm.ms, Agg);
        V Xr = Op::apply(Nt, X);   // H entering this thread's row from the right
        X = Op::apply(Agg, X);     // carry for the next tile (to the left)

        // outputs, right to left
#pragma unroll
        for (int g = G::NG - 1; g >= 0; --g) {
            uint32_t wa[G::GB / 4], wy[G::GB / 4], wc[G::GB / 4], wo[G::GB / 4], wz[G::GB / 4];
            if (FWD) lds_group<G::GB>(sA, t, g, wa);
            lds_group<G::GB>(sY, t, g, wy);
            if (ACC) lds_group<G::GB>(sC, t, g, wc);
#pragma unroll
            for (int e = G::EG - 1; e >= 0; --e) {
                const int q = g * G::EG + e;
                V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
                V y = dec<T, W>(wy + e * (G::ES / 4));
                const bool valid = !last || e0 + q < p.n;
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
                if (valid) Xr = Op::apply(Op::make_map(rsp[q], a, y), Xr);
            }
            sts_group<G::GB>(sY, t, g, wo);
            if (YS) sts_group<G::GB>(sA, t, g, wz);
        }
        if (has_partial) {
            store_partial_row(sY, t, p.as_bar, p.full_rows, p.tail_bytes);
            if (YS) store_partial_row(sA, t, p.ys, p.full_rows, p.tail_bytes);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (t == 0) {
            if (chunk_tile_rows<NT>(p, tile) > 0) {
                tma_store_2d(&tm_ab, sY, 0, (int)(tile * NT));
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

}  // namespace vjpk
