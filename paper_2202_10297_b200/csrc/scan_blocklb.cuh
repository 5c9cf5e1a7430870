// scan_blocklb.cuh — one-read return sweep of vjp_scan by decoupled look-back
// over L2-resident BLOCKS of tiles (single GPU; sec 5.2).
//
// The return sweep is a reverse scan of the composed affine maps M_i (lin_o,
// P:1196, grouped per element as in scan_ops.cuh) followed by the output map
// (P:1200-1202).  The chunked kernels (scan_chunked.cuh) read `as` and
// `ys_bar` twice (K_R for the chunk maps, K_C for the outputs); this kernel
// reads them from HBM ONCE:
//
//   * blocks of B consecutive tiles are handed out right to left by an atomic
//     ticket (ticket j = block nblocks-1-j), so every block's right
//     neighbours were started before it;
//   * R phase (4 compute warps): the block's tiles stream in from HBM (TMA
//     ring).  Per tile, the rows' forward aggregates and reverse maps, warp 0
//     the forward row scan (rs entering every row, from the K_F tile prefix),
//     warp 1 the reverse row scan AS MAPS: S_r = M_{r+1} o ... o M_last (the
//     map taking the carry entering the tile from the right to the H entering
//     row r) and the tile map T.  rs_r and S_r do not depend on the carry, so
//     they are parked, component-major, in the tile's own as_bar rows (which
//     the A phase overwrites with the outputs; the partial last tile uses a
//     workspace slot).  M_blk = T_first o ... o T_last is published with an
//     AGGREGATE flag as soon as the phase ends;
//   * look-back (warp 4, concurrent with the R phase): walks the descriptors of
//     the blocks to the right, 32 per step, composing their maps until one
//     carries an INCLUSIVE value, giving the carry X_blk entering the block
//     from the right; then publishes the block's inclusive value M_blk(X_blk);
//   * A phase (compute warps): the block's tiles stream in AGAIN — L2 hits, the
//     block was read a few microseconds earlier and the blocks in flight hold
//     ~G*B*tile bytes << L2 — and every thread works alone: H_r = S_r(X_tile),
//     the primal scan re-executed over its row from rs_r (tape-free),
//     rbar_i = ybar_i + H_{i+1}, abar_i = J_R^T rbar_i; X_tile moves one tile
//     left by the tile map T.  No warp scans and no look-back in this phase.
//
// The forward prefix of every tile (tileP) comes from the `as`-only pre-pass
// (K_F = scan_reduce<FWD> + scan_tile_prefix), so HBM sees the method's bytes
// and nothing else: LINREC 16 + 48, MAT2 32 + 96 B per element (K_F + this
// kernel), scan(+) 16 B (no pre-pass), MIN/MAX 8 + 24 (f64).  The parked rs /
// S_r lines are written and re-read in L2 and finally overwritten by the
// outputs.
//
// The TMA load sequence of a CTA is [R tiles of block k][A tiles of block k]
// [R tiles of block k+1]...; tickets are taken when the producer (thread 0)
// reaches a block, so the next block's HBM reads are in flight during this
// block's A phase.  Deadlock freedom: a block waits only for smaller tickets,
// and every CTA processes its tickets in increasing order.  A look-back that
// waits longer than ~4 s traps (a kernel error, never a hang).
//
// Not for VJP_ACCUMULATE (as_bar holds the caller's values; the chunked
// kernels serve that case).
#pragma once

#include "scan_sweep.cuh"

namespace vjpk {

constexpr int kLbBMax = 16;      // tiles per block (tile maps of two blocks kept in shared memory)
constexpr int kLbCompute = 128;  // compute threads (4 warps); warp 4 looks back

struct LbParams {
    ChunkParams c;     // geometry, arrays, tileP (forward prefix of every tile)
    int32_t B;         // tiles per block
    int32_t nblocks;
    uint32_t *ticket;  // [1] block ticket counter (zeroed before the launch)
    uint32_t *flags;   // [nblocks] per ticket: 0 empty, 1 aggregate, 2 inclusive (zeroed)
    double *agg;       // [nblocks][kMapD] block maps
    double *inc;       // [nblocks][W] inclusive values (carry leaving the block to the left)
    double *tailpark;  // [NT][W + kMapD] parking of the last tile (not a full as_bar tile)
    unsigned long long *trace;  // tuning only (nullptr): per ticket 8 timestamps / counters
};

template <class Op, int NT, int S>
struct LbSmem {
    uint64_t bar[S];
    int32_t tick[4];           // tickets of the blocks between producer and consumers
    volatile int32_t tickseq[4];  // block number whose ticket is in tick[] (look-back warp handshake)
    volatile int32_t aggseq;   // last block whose M_blk is in mblk
    volatile int32_t xseq;     // last block whose carry is in xv
    double mblk[2][Op::kMapD];
    double xv[2][Op::W];
    double tileT[2][kLbBMax * Op::kMapD];  // tile maps of the two blocks in flight
    double rv[Op::W * RowArr<NT>::kStride];
    double rm[Op::kMapD * RowArr<NT>::kStride];
};

// (globaltimer_ns: scan_sweep.cuh)
// barrier of the 4 compute warps only (the look-back warp never joins)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kLbCompute) : "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// spin (with back-off) until *p >= want; traps after ~4 s
__device__ __forceinline__ void spin_ge(const volatile int32_t *p, int32_t want) {
    const uint64_t t0 = globaltimer_ns();
    int spins = 0;
    while (*p < want) {
        if (++spins > 8) __nanosleep(32);
        if ((spins & 4095) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
    }
}
// spin (with back-off) until *p == want; traps after ~4 s
__device__ __forceinline__ void spin_eq(const volatile int32_t *p, int32_t want) {
    const uint64_t t0 = globaltimer_ns();
    int spins = 0;
    while (*p != want) {
        if (++spins > 8) __nanosleep(64);
        if ((spins & 4095) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
    }
}

// reverse row scan AS MAPS (one warp): overwrites row r of `m` with
// S_r = m_{r+1} o ... o m_{NT-1} (identity for the last row) and returns the
// tile map m_0 o ... o m_{NT-1} in every lane
template <class Op, int NT>
__device__ __forceinline__ typename Op::Map warp_excl_rev_rows_maps(double *m) {
    using M = typename Op::Map;
    constexpr int K = NT / 32;
    const int lane = threadIdx.x & 31;
    M e[K];
#pragma unroll
    for (int j = 0; j < K; ++j) e[j] = get_m<Op, NT>(m, lane * K + j);
    __syncwarp();
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
    M sfx = lane == 31 ? Op::map_id() : ex;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
        put_m<Op, NT>(m, lane * K + j, sfx);
        sfx = Op::compose(e[j], sfx);
    }
    return shfl_idx_m<Op>(inc, 0);
}

// the look-back warp: carry entering block `tk` from the right, from the
// descriptors of the blocks to its right (every lane returns it)
template <class Op>
__device__ __forceinline__ typename Op::Val lb_prefix(const LbParams &P, int32_t tk) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD;
    const int lane = threadIdx.x & 31;
    V X;
#pragma unroll
    for (int q = 0; q < W; ++q) X.x[q] = 0.0;  // single GPU: nothing enters the last element
    if (tk == 0) return X;
    // windows of 32 lanes x KL descriptors; lane l holds the KL consecutive
    // blocks pos - l*KL, ..., pos - l*KL - KL + 1 (nearest first), so one
    // window covers the ~G blocks in flight with all loads issued at once
    constexpr int KL = 8;
    M acc = Op::map_id();
    int64_t pos = tk - 1;
    const uint64_t t0 = globaltimer_ns();
    while (true) {
        const int64_t base = pos - (int64_t)lane * KL;
        uint32_t f[KL];
#pragma unroll
        for (int j = 0; j < KL; ++j) f[j] = (base - j >= 0) ? ld_flag(P.flags + base - j) : 2u;
        int spins = 0;
        while (true) {  // every descriptor of the lane published (aggregate or inclusive)
            bool ready = true;
#pragma unroll
            for (int j = 0; j < KL; ++j)
                if (f[j] == 0u) {
                    f[j] = ld_flag(P.flags + base - j);
                    ready &= f[j] != 0u;
                }
            if (ready) break;
            if (++spins > 4) __nanosleep(32);
            if ((spins & 4095) == 0 && globaltimer_ns() - t0 > 4000000000ull) __trap();
        }
        __syncwarp();
        fence_acq_rel_gpu();
        int jinc = KL;  // the lane's nearest inclusive descriptor
#pragma unroll
        for (int j = KL - 1; j >= 0; --j)
            if (f[j] == 2u) jinc = j;
        // the lane's maps before it, nearest outermost: loads in batches of 4
        // issued together (independent L2 round trips), then composed
        M ml = Op::map_id();
#pragma unroll
        for (int j0 = 0; j0 < KL; j0 += 4) {
            double d[4][MD];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t idx = base - (j0 + j);
                const double *src = P.agg + (idx >= 0 ? idx : 0) * MD;
#pragma unroll
                for (int q = 0; q < MD; ++q) d[j][q] = ld_cg(src + q);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j0 + j < jinc && base - (j0 + j) >= 0) ml = Op::compose(ml, map_from<Op>(d[j]));
        }
        const unsigned incm = __ballot_sync(0xffffffffu, jinc < KL);
        const int k = incm ? __ffs(incm) - 1 : 32;
        V vl = X;
        if (lane == k && base - jinc >= 0) ld_rec<W>(P.inc + (base - jinc) * W, vl.x);
        if (lane > k) ml = Op::map_id();
        // lanes 0..k in order: lane 0 (the nearest blocks) outermost
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            M o = shfl_down_m<Op>(ml, s);
            if (lane + s < 32) ml = Op::compose(ml, o);
        }
        acc = Op::compose(acc, shfl_idx_m<Op>(ml, 0));
        if (k < 32) {
            X = Op::apply(acc, shfl_idx_v(vl, k));
            break;
        }
        pos -= 32 * KL;
        if (P.trace && lane == 0) P.trace[(int64_t)tk * 8 + 7] += 1;
    }
    return X;
}

template <class Op, class T, int NT, int S, bool FWD, bool YS, bool RS>
__global__ void __launch_bounds__(kLbCompute + 32, 1) scan_blocklb(const __grid_constant__ CUtensorMap tm_as,
                                                                   const __grid_constant__ CUtensorMap tm_yb,
                                                                   const __grid_constant__ CUtensorMap tm_ab,
                                                                   const __grid_constant__ CUtensorMap tm_ys,
                                                                   const LbParams P) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD, PK = (FWD ? W : 0) + MD;  // parked doubles per row
    constexpr int NB = (FWD ? 1 : 0) + 1;  // [A][Y], outputs over Y
    constexpr int BUF = NT * kRowBytes, STG = NB * BUF;
    static_assert(NT == kLbCompute, "one row per compute thread");
    static_assert(!RS || FWD, "rs-dependent maps need `as`");
    static_assert(PK * 8 <= kRowBytes, "the parked row must fit in the row's as_bar bytes");

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = smem_align1024(smem_raw);
    LbSmem<Op, NT, S> &sm = *reinterpret_cast<LbSmem<Op, NT, S> *>(base + S * STG);
    const ChunkParams &p = P.c;
    const int t = threadIdx.x, warp = t >> 5;
    if (t == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.bar[s], 1);
        fence_mbar_init();
        for (int q = 0; q < 4; ++q) sm.tickseq[q] = -1;
        sm.aggseq = -1;
        sm.xseq = -1;
    }
    __syncthreads();
    auto blk_tiles = [&](int32_t tk, int64_t &t0, int64_t &t1) {
        const int64_t b = (int64_t)P.nblocks - 1 - tk;
        t0 = b * P.B;
        t1 = t0 + P.B < p.ntiles ? t0 + P.B : p.ntiles;
    };

    // ======================================================== look-back warp
    if (warp == kLbCompute / 32) {
        for (int32_t k = 0;; ++k) {
            spin_eq(&sm.tickseq[k & 3], k);
            const int32_t tk = sm.tick[k & 3];
            if (tk >= P.nblocks) break;
            if (P.trace && (t & 31) == 0) P.trace[(int64_t)tk * 8 + 0] = globaltimer_ns();
            const V X = lb_prefix<Op>(P, tk);
            if (P.trace && (t & 31) == 0) P.trace[(int64_t)tk * 8 + 1] = globaltimer_ns();
            spin_ge(&sm.aggseq, k);
            M Mb;
#pragma unroll
            for (int q = 0; q < MD; ++q) reinterpret_cast<double *>(&Mb)[q] = sm.mblk[k & 1][q];
            if ((t & 31) == 0) {
                const V incv = Op::apply(Mb, X);
                st_rec<W>(P.inc + (int64_t)tk * W, incv.x);
                st_flag_release(P.flags + tk, 2u);
#pragma unroll
                for (int q = 0; q < W; ++q) sm.xv[k & 1][q] = X.x[q];
                __threadfence_block();
                sm.xseq = k;
            }
            __syncwarp();
        }
        return;
    }

    // ======================================================== compute warps
    // Two blocks in flight per CTA: the order is R(0), R(1), A(0), R(2), A(1),
    // ..., so block k's look-back has the whole R phase of block k+1 to land.
    uint64_t pol_last, pol_first;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    const CUtensorMap *m0 = FWD ? &tm_as : &tm_yb;

    // ---- producer state (thread 0): the CTA's load sequence ----
    int32_t ik = 0, iph = 0, ii = 0;  // phase 0: R(ik); phase 1: A(ik - 1)
    bool inoR = false, idone = false;
    int64_t iL = 0;  // loads issued
    auto issue_next = [&]() {
        while (!idone) {
            if (iph == 0) {
                if (ii == 0) {  // entering R(ik): take its ticket
                    const int32_t tk = (int32_t)atomicAdd(P.ticket, 1u);
                    sm.tick[ik & 3] = tk;
                    __threadfence_block();
                    sm.tickseq[ik & 3] = ik;
                    if (tk >= P.nblocks) {
                        inoR = true;
                        if (ik == 0) {
                            idone = true;
                            return;
                        }
                        iph = 1;  // only A(ik - 1) is left
                        continue;
                    }
                }
                int64_t t0, t1;
                blk_tiles(sm.tick[ik & 3], t0, t1);
                const int64_t tile = t1 - 1 - ii;
                const int s = (int)(iL % S);
                if (chunk_tile_rows<NT>(p, tile) > 0) {  // R loads: keep the block in L2 until its A phase
                    mbar_arrive_expect_tx(&sm.bar[s], NB * NT * kRowBytes);
                    tma_load_2d_hint(base + s * STG, m0, &sm.bar[s], 0, (int)(tile * NT), pol_last);
                    if (FWD) tma_load_2d_hint(base + s * STG + BUF, &tm_yb, &sm.bar[s], 0, (int)(tile * NT), pol_last);
                } else {
                    mbar_arrive(&sm.bar[s]);
                }
                ++iL;
                if (++ii == (int)(t1 - t0)) {
                    ii = 0;
                    if (ik == 0) ik = 1;  // no A(-1)
                    else iph = 1;
                }
                return;
            } else {
                int64_t t0, t1;
                blk_tiles(sm.tick[(ik - 1) & 3], t0, t1);
                const int64_t tile = t1 - 1 - ii;
                const int s = (int)(iL % S);
                if (chunk_tile_rows<NT>(p, tile) > 0) {  // A loads: last use
                    mbar_arrive_expect_tx(&sm.bar[s], NB * NT * kRowBytes);
                    tma_load_2d_hint(base + s * STG, m0, &sm.bar[s], 0, (int)(tile * NT), pol_first);
                    if (FWD) tma_load_2d_hint(base + s * STG + BUF, &tm_yb, &sm.bar[s], 0, (int)(tile * NT), pol_first);
                } else {
                    mbar_arrive(&sm.bar[s]);
                }
                ++iL;
                if (++ii == (int)(t1 - t0)) {
                    ii = 0;
                    if (inoR) idone = true;
                    else {
                        iph = 0;
                        ++ik;
                    }
                }
                return;
            }
        }
    };
    if (t == 0)
        for (int s = 0; s < S; ++s) issue_next();

    int64_t L = 0;  // loads consumed
    // after consuming load L: commit this iteration's store group and refill
    // the stage of load L-1 (its store, if any, has had a whole tile to drain)
    auto retire = [&]() {
        if (t == 0) {
            tma_store_commit();
            if (L >= 1) {
                tma_store_wait_read1();
                issue_next();
            }
        }
        ++L;
    };
    // parking of row t of `tile`: component-major in the tile's as_bar bytes
    auto park_of = [&](int64_t tile) -> double * {
        if (tile == p.ntiles - 1) return P.tailpark;
        return reinterpret_cast<double *>(static_cast<unsigned char *>(p.as_bar) + tile * NT * kRowBytes);
    };

    // ---------------------------------------------------- R phase of block k
    auto r_phase = [&](int32_t k, int32_t tk) {
        int64_t t0, t1;
        blk_tiles(tk, t0, t1);
        const int nt = (int)(t1 - t0);
        if (P.trace && t == 0) P.trace[(int64_t)tk * 8 + 2] = globaltimer_ns();
        double *tT = sm.tileT[k & 1];
        M Mblk = Op::map_id();  // kept by warp 1
        for (int i = 0; i < nt; ++i) {
            const int64_t tile = t1 - 1 - i;
            const int s = (int)(L % S);
            V Ftile = Op::fwd_id();
            if (FWD && warp == 0) {
#pragma unroll
                for (int q = 0; q < W; ++q) Ftile.x[q] = ld_cg(p.tileP + tile * W + q);
            }
            mbar_wait(&sm.bar[s], (uint32_t)((L / S) & 1));
            unsigned char *sA = base + s * STG;
            unsigned char *sY = sA + (FWD ? BUF : 0);
            const bool last = (tile == p.ntiles - 1);
            if (last && p.tail_bytes && t == (int)(p.full_rows - tile * NT)) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
            }
            const int64_t e0 = (tile * NT + t) * G::EPR;
            if constexpr (RS) {
                put_v<Op, NT>(sm.rv, t, row_fwd<Op, T, true>(sA, t, e0, last, p.n));
                csync();
                if (warp == 0) warp_excl_fwd_rows<Op, NT>(sm.rv, Ftile);
                csync();
                put_m<Op, NT>(sm.rm, t, row_map_rs<Op, T>(sA, sY, t, e0, last, p.n, get_v<Op, NT>(sm.rv, t)));
                csync();
            } else {
                if (FWD) put_v<Op, NT>(sm.rv, t, row_fwd<Op, T, true>(sA, t, e0, last, p.n));
                put_m<Op, NT>(sm.rm, t, row_map<Op, T, FWD>(sA, sY, t, e0, last, p.n));
                csync();
                if (FWD && warp == 0) warp_excl_fwd_rows<Op, NT>(sm.rv, Ftile);
            }
            if (warp == 1) {
                const M Tt = warp_excl_rev_rows_maps<Op, NT>(sm.rm);
                Mblk = Op::compose(Tt, Mblk);
                if ((t & 31) == 0) {
#pragma unroll
                    for (int q = 0; q < MD; ++q) tT[i * MD + q] = reinterpret_cast<const double *>(&Tt)[q];
                }
            }
            csync();
            // park rs entering row t and S_t (coalesced: component-major)
            {
                double *pk = park_of(tile);
                if constexpr (FWD) {
#pragma unroll
                    for (int q = 0; q < W; ++q)
                        __stcg(pk + q * NT + t, sm.rv[q * RowArr<NT>::kStride + RowArr<NT>::spos(t)]);
                }
#pragma unroll
                for (int q = 0; q < MD; ++q)
                    __stcg(pk + ((FWD ? W : 0) + q) * NT + t, sm.rm[q * RowArr<NT>::kStride + RowArr<NT>::spos(t)]);
            }
            retire();
        }
        if (warp == 1 && (t & 31) == 0) {
            // publish the block's aggregate at once, and hand it to the look-back warp
            double d[MD];
            map_to<Op>(Mblk, d);
            if (tk > 0) {
                st_rec<MD>(P.agg + (int64_t)tk * MD, d);
                st_flag_release(P.flags + tk, 1u);
            }
#pragma unroll
            for (int q = 0; q < MD; ++q) sm.mblk[k & 1][q] = d[q];
            __threadfence_block();
            sm.aggseq = k;
        }
        if (P.trace && t == 0) P.trace[(int64_t)tk * 8 + 3] = globaltimer_ns();
    };

    // ---------------------------------------------------- A phase of block k
    auto a_phase = [&](int32_t k, int32_t tk) {
        int64_t t0, t1;
        blk_tiles(tk, t0, t1);
        const int nt = (int)(t1 - t0);
        if (t == 0) spin_ge(&sm.xseq, k);
        if (P.trace && t == 0) P.trace[(int64_t)tk * 8 + 4] = globaltimer_ns();
        csync();
        const double *tT = sm.tileT[k & 1];
        V X;  // carry entering the current tile from the right
#pragma unroll
        for (int q = 0; q < W; ++q) X.x[q] = sm.xv[k & 1][q];
        for (int i = 0; i < nt; ++i) {
            const int64_t tile = t1 - 1 - i;
            const int s = (int)(L % S);
            // the parked rs / S_t of this row (L2), before waiting for the stage
            const double *pk = park_of(tile);
            V rs0 = Op::fwd_id();
            if constexpr (FWD) {
#pragma unroll
                for (int q = 0; q < W; ++q) rs0.x[q] = __ldcg(pk + q * NT + t);
            }
            double sd[MD];
#pragma unroll
            for (int q = 0; q < MD; ++q) sd[q] = __ldcg(pk + ((FWD ? W : 0) + q) * NT + t);
            M Tt;
#pragma unroll
            for (int q = 0; q < MD; ++q) reinterpret_cast<double *>(&Tt)[q] = tT[i * MD + q];
            mbar_wait(&sm.bar[s], (uint32_t)((L / S) & 1));
            unsigned char *sA = base + s * STG;
            unsigned char *sY = sA + (FWD ? BUF : 0);
            unsigned char *sO = sY;
            const bool last = (tile == p.ntiles - 1);
            const bool has_partial = last && p.tail_bytes && t == (int)(p.full_rows - tile * NT);
            if (has_partial) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
            }
            const int64_t e0 = (tile * NT + t) * G::EPR;
            // re-execute the primal scan over the row from rs_t, then outputs right to left
            V rsp[G::EPR];
            if constexpr (FWD) {
                V r = rs0;
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
            V Xr = Op::apply(map_from<Op>(sd), X);  // H entering row t from the right
#pragma unroll
            for (int g = G::NG - 1; g >= 0; --g) {
                uint32_t wa[G::GB / 4], wy[G::GB / 4], wo[G::GB / 4], wz[G::GB / 4];
                if (FWD) lds_group<G::GB>(sA, t, g, wa);
                lds_group<G::GB>(sY, t, g, wy);
#pragma unroll
                for (int e = G::EG - 1; e >= 0; --e) {
                    const int q = g * G::EG + e;
                    V a = FWD ? dec<T, W>(wa + e * (G::ES / 4)) : Op::fwd_id();
                    V y = dec<T, W>(wy + e * (G::ES / 4));
                    V gv;
#pragma unroll
                    for (int z = 0; z < W; ++z) gv.x[z] = y.x[z] + Xr.x[z];  // rbar_i = ybar_i + H_{i+1}
                    V o = Op::out(rsp[q], a, gv);
                    if (Op::kFirstSpecial && p.global_first && e0 + q == 0) o = gv;
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
            X = Op::apply(Tt, X);  // the carry entering the next tile to the left
            fence_proxy_async_smem();
            fence_proxy_async_global();  // the parked rows were read (generic proxy) before the TMA store overwrites them
            csync();
            if (t == 0 && chunk_tile_rows<NT>(p, tile) > 0) {
                tma_store_2d_hint(&tm_ab, sO, 0, (int)(tile * NT), pol_first);
                if (YS) tma_store_2d(&tm_ys, sA, 0, (int)(tile * NT));
            }
            retire();
        }
        if (P.trace && t == 0) {
            P.trace[(int64_t)tk * 8 + 5] = globaltimer_ns();
            P.trace[(int64_t)tk * 8 + 6] = blockIdx.x;
        }
    };

    csync();  // sm.tick[0] was written before the first load was issued
    int32_t tkprev = sm.tick[0];
    if (tkprev < P.nblocks) {
        r_phase(0, tkprev);
        for (int32_t k = 1;; ++k) {
            csync();  // sm.tick[k & 3] was written before block k's first load (or the end)
            const int32_t tk = sm.tick[k & 3];
            const bool more = tk < P.nblocks;
            if (more) r_phase(k, tk);
            a_phase(k - 1, tkprev);
            if (!more) break;
            tkprev = tk;
        }
    }
    if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace vjpk
