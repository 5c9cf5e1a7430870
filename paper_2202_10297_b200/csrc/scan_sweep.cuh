// scan_sweep.cuh — single-read L2-round return sweep of vjp_scan (the default
// single-GPU path for ADD, MUL, LINREC and MAT2).
//
// The chunked kernels (scan_chunked.cuh) read `as`/`ys_bar` twice from HBM:
// once in K_R for the chunk aggregates, once in K_C.  Here the two passes are
// interleaved in ONE persistent (cooperatively launched) kernel over ROUNDS of
// G*K tiles taken from the right end of the array (the return sweep runs right
// to left):
//
//   round r, CTA c owns the K consecutive tiles  q in [(rG+c)K, (rG+c+1)K)
//   counted from the right (tile = ntiles-1-q); CTA 0 is the rightmost.
//
//   job sequence of the tile warps:  R(0) R(1) A(0) R(2) A(1) ... R(R-1) A(R-2) A(R-1)
//     R(r): stream its sub-chunk of round r from HBM and compose the tiles'
//           reverse maps (the lin_o composition of P:1196-1198, grouped per
//           element as in scan_ops.cuh) into the sub-chunk map M_{r,c};
//     A(r): re-read the sub-chunk — now an L2 hit, since it was loaded one
//           segment ago — and run the K_C tile body (forward re-execution in
//           registers from tileP, row maps, warp scans, outputs, TMA store)
//           from the carry entering the sub-chunk.
//   The four tile warps work on their own 32 rows: shuffle scans of the row
//   maps (no single-warp bottleneck), one named barrier per apply tile to
//   exchange the four warp aggregates, per-warp TMA stores; a reduce tile needs
//   no barrier at all.  A PRODUCER warp feeds an S-stage TMA ring with
//   full/empty mbarriers, and a CARRY warp, off the tiles' critical path, per
//   round r: publishes
//   M_{r,c} (global record + release-add on arrive[r]), waits arrive[r] == G,
//   loads the round's G records and composes the carry entering this sub-chunk
//   (M_{r,c-1} o ... o M_{r,0})(Xin_r) and the next round's Xin_{r+1}; it
//   talks to the tile warps through shared memory + mbarriers (two slots each,
//   which the job order makes sufficient).
//
// HBM therefore sees each input once (ADD 16 B/elem, LINREC 48 + the
// forward pre-pass 16, MAT2 96 + 32: the method bytes of SURVEY 8d).  The round
// size is chosen so that about three rounds of traffic fit in L2.  For the
// forward operators tileP (forward exclusive prefix per tile) comes from the
// pre-pass K_F = scan_reduce<FWD only> and scan_tile_prefix.
#pragma once

#include <type_traits>

#include "scan_chunked.cuh"

namespace vjpk {

constexpr int kSweepNT = 128;  // tile threads (+ one carry warp)

constexpr int kCycMax = 8;  // ranks of one NVSwitch domain (block-cyclic mode)

struct SweepParams {
    ChunkParams c;      // geometry, arrays, tileP (tileF/chunkRec unused here)
    int32_t G;          // CTAs (all co-resident: cooperative launch)
    int32_t K;          // tiles per CTA per round
    int32_t R;          // rounds
    int32_t D;          // reduce look-ahead in rounds (1 or 2)
    double *roundRec;   // [R][G][kMapD] sub-chunk reverse maps
    uint32_t *arrive;   // [R] arrival counters, zeroed before the launch
    // ---- block-cyclic multi-GPU partition; cyc == 0: one GPU.
    // The global array is cut into superblocks (SB) of tps tiles; SB J is owned
    // by rank J % cw and is this rank's local SB J / cw (local arrays are the
    // owned SBs in order).  Round r = local SB l = R - 1 - r (right to left).
    // The carry entering SB J comes from SB J + 1 on the NEXT rank: look-back
    // over the SB status words every rank pushes to every rank's status
    // buffer (peer-mapped device memory over NVLink), see cyc_carry.
    int32_t cyc, cw, cr;  // mode, world, rank
    uint32_t epoch;       // status words read (epoch << 2) | 1 once the SB's map (AGG) is in
    int32_t tps;          // tiles per superblock
    int32_t nsb;          // global superblocks
    uint32_t *shdr[kCycMax];   // every rank's status header: [0] error word, [1 + q] epoch rank q entered
    uint32_t *sflag[kCycMax];  // every rank's status words [nsb] (peer pointers)
    double *spay[kCycMax];     // every rank's payloads [nsb][kMapD]: the superblocks' reverse maps
    uint32_t *err;             // local: a look-back wait timed out (results invalid)
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t make_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// TMA load with an L2 cache-policy hint
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                 uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap *map, const void *src, int c0, int c1,
                                                  uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
                 ::"l"(map), "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol) : "memory");
}

// ---- job sequence -------------------------------------------------------------
// segments s = 0 .. D + 2R - 1:  R(0) .. R(D-1), then pairs (R(k + D), A(k)),
// k = 0 .. R-1 (R(k + D) empty once k + D >= R).
struct SweepSeg {
    bool apply;
    int32_t round;
};
__device__ __forceinline__ SweepSeg sweep_seg(int s, int D) {
    if (s < D) return {false, s};
    const int i = s - D;
    return (i & 1) ? SweepSeg{true, i >> 1} : SweepSeg{false, (i >> 1) + D};
}
// round r spans tiles [sweep_begin, sweep_end); CTA c owns the K tiles
// counted from the round's right end: tile = end - 1 - (cK + j)
__device__ __forceinline__ int64_t sweep_end(const SweepParams &p, int r) {
    if (p.cyc) {
        const int64_t e = (int64_t)(p.R - r) * p.tps;
        return e < p.c.ntiles ? e : p.c.ntiles;
    }
    return (int64_t)p.c.ntiles - (int64_t)r * p.G * p.K;
}
__device__ __forceinline__ int64_t sweep_begin(const SweepParams &p, int r) {
    if (p.cyc) return (int64_t)(p.R - 1 - r) * p.tps;
    const int64_t b = (int64_t)p.c.ntiles - (int64_t)(r + 1) * p.G * p.K;
    return b > 0 ? b : 0;
}
__device__ __forceinline__ int64_t sweep_tile(const SweepParams &p, int r, int j) {
    return sweep_end(p, r) - 1 - ((int64_t)blockIdx.x * p.K + j);
}
__device__ __forceinline__ int sweep_nseg(const SweepParams &p) { return p.D + 2 * p.R; }
__device__ __forceinline__ int sweep_count(const SweepParams &p, int r) {
    if (r >= p.R) return 0;
    const int64_t left = sweep_end(p, r) - sweep_begin(p, r) - (int64_t)blockIdx.x * p.K;
    return left <= 0 ? 0 : (left >= p.K ? p.K : (int)left);
}

// producer-side iterator over the non-empty jobs
struct SweepIt {
    int s, j;
    bool done;
};
__device__ __forceinline__ void sweep_norm(const SweepParams &p, SweepIt &it) {
    while (!it.done && it.j >= sweep_count(p, sweep_seg(it.s, p.D).round)) {
        ++it.s;
        it.j = 0;
        if (it.s >= sweep_nseg(p)) it.done = true;
    }
}

// exclusive forward prefix of every tile (tileP) from the K_F records: one CTA
// per K_F chunk (the forward part of the K_C prologue).
template <class Op, int NT>
__global__ void __launch_bounds__(NT) scan_tile_prefix(const ChunkParams p) {
    using V = typename Op::Val;
    constexpr int W = Op::W, R = Op::W + Op::kMapD, NW = NT / 32;
    __shared__ V vs[NW + 1];
    const int t = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int64_t t0 = chunk_begin(p, c), t1 = chunk_begin(p, c + 1), k = t1 - t0;
    // forward aggregate of chunks [0, c)
    V f = Op::fwd_id();
    {
        const int64_t per = (c + NT - 1) / NT;
        for (int64_t j = t * per; j < (t + 1) * per && j < c; ++j) {
            V v;
#pragma unroll
            for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.chunkRec + j * R + q);
            f = Op::fwd(f, v);
        }
    }
    V Fpre = block_reduce_fwd<Op, NW>(f, vs);
    if (p.world > 1 && p.gathered) {  // multi-GPU (MIN/MAX split): the shards to the left come first
        V Fsh, Hunused;
        shard_carries<Op>(p.gathered, p.rank, p.world, Fsh, Hunused);
        Fpre = Op::fwd(Fsh, Fpre);
    }
    const int64_t per = (k + NT - 1) / NT;
    f = Op::fwd_id();
    for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
        f = Op::fwd(f, v);
    }
    V tot;
    V ex = block_excl_fwd<Op, NW>(f, vs, tot);
    V r = Op::fwd(Fpre, ex);
    for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
#pragma unroll
        for (int q = 0; q < W; ++q) st_cg(p.tileP + j * W + q, r.x[q]);
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
        r = Op::fwd(r, v);
    }
}

// ---- block-cyclic forward re-execution (f1; "the forward sweep is
// the original scan") --------------------------------------------------------
// one CTA per local superblock l: its forward aggregate (ordered fold of the
// K_F tile aggregates tileF over the SB's tiles) -> sbagg[l][W]
template <class Op, int NT>
__global__ void __launch_bounds__(NT) scan_cyc_sbagg(const ChunkParams p, int32_t tps, double *__restrict__ sbagg) {
    using V = typename Op::Val;
    constexpr int W = Op::W, NW = NT / 32;
    __shared__ V vs[NW + 1];
    const int t = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * tps;
    const int64_t t1 = t0 + tps < p.ntiles ? t0 + tps : p.ntiles;
    const int64_t k = t1 - t0, per = (k + NT - 1) / NT;
    V f = Op::fwd_id();
    for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
        f = Op::fwd(f, v);
    }
    const V tot = block_reduce_fwd<Op, NW>(f, vs);
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < W; ++q) sbagg[(int64_t)blockIdx.x * W + q] = tot.x[q];
    }
}
// one CTA per local SB l (global J = l * cw + cr): forward prefix entering the
// SB = ordered fold of every rank's SB aggregates J' < J from the gathered
// table [cw][nloc_max][W] (SB J' is rank J' % cw's local SB J' / cw), then the
// exclusive prefixes of the SB's tiles -> tileP
template <class Op, int NT>
__global__ void __launch_bounds__(NT) scan_cyc_tileprefix(const ChunkParams p, int32_t tps, int32_t cw, int32_t cr,
                                                          int32_t nloc_max, const double *__restrict__ gathered) {
    using V = typename Op::Val;
    constexpr int W = Op::W, NW = NT / 32;
    __shared__ V vs[NW + 1];
    const int t = threadIdx.x;
    const int64_t J = (int64_t)blockIdx.x * cw + cr;
    V f = Op::fwd_id();
    {
        const int64_t per = (J + NT - 1) / NT;
        for (int64_t j = t * per; j < (t + 1) * per && j < J; ++j) {
            const double *g = gathered + ((j % cw) * (int64_t)nloc_max + j / cw) * W;
            V v;
#pragma unroll
            for (int q = 0; q < W; ++q) v.x[q] = g[q];
            f = Op::fwd(f, v);
        }
    }
    const V Fpre = block_reduce_fwd<Op, NW>(f, vs);
    const int64_t t0 = (int64_t)blockIdx.x * tps;
    const int64_t t1 = t0 + tps < p.ntiles ? t0 + tps : p.ntiles;
    const int64_t k = t1 - t0, per = (k + NT - 1) / NT;
    f = Op::fwd_id();
    for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
        f = Op::fwd(f, v);
    }
    V tot;
    const V ex = block_excl_fwd<Op, NW>(f, vs, tot);
    V r = Op::fwd(Fpre, ex);
    for (int64_t j = t0 + t * per; j < t0 + (t + 1) * per && j < t1; ++j) {
#pragma unroll
        for (int q = 0; q < W; ++q) st_cg(p.tileP + j * W + q, r.x[q]);
        V v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.x[q] = ld_cg(p.tileF + j * W + q);
        r = Op::fwd(r, v);
    }
}

// =============================================================================
// the sweep
// =============================================================================
constexpr int kSweepKMax = 8;
constexpr int kSweepSlots = 4;  // rounds in flight between tile warps and carry warp (D <= 2)
constexpr long long kSweepPollCycles = 2000;  // tiles per CTA per round (reduce aggregates kept in smem)

template <class Op, int S>
struct SweepSmem {
    uint64_t full[S], empty[S];
    uint64_t recbar[kSweepSlots];    // tile warps -> carry warp: M_{r,c} in rec[r % slots]
    uint64_t carrybar[kSweepSlots];  // carry warp -> tile warps: X_{r,c} in carry[r % slots]
    typename Op::Map rec[kSweepSlots];
    typename Op::Val carry[kSweepSlots];
    typename Op::Map aggM[2][4];  // apply: warp aggregates (reverse maps), by job parity
    typename Op::Val aggF[2][4];  // apply: warp aggregates (forward), by job parity
    typename Op::Map ragg[2][kSweepKMax][4];  // reduce: per tile, per warp, by round parity
};

__device__ __forceinline__ void bar_tiles() { asm volatile("bar.sync 1, %0;" ::"n"(kSweepNT) : "memory"); }

__device__ __forceinline__ void red_release_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void tma_store_wait_read0_() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// suffix composition over the warp: lane l gets m_l o m_{l+1} o ... o m_31
template <class Op>
__device__ __forceinline__ typename Op::Map warp_suffix_maps(typename Op::Map m, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        typename Op::Map u = shfl_down_m<Op>(m, o);
        if (lane + o < 32) m = Op::compose(m, u);
    }
    return m;
}
// prefix of forward values over the warp: lane l gets v_0 (.) ... (.) v_l
template <class Op>
__device__ __forceinline__ typename Op::Val warp_prefix_vals(typename Op::Val v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        typename Op::Val u = shfl_up_v(v, o);
        if (lane >= o) v = Op::fwd(u, v);
    }
    return v;
}
// lane-parallel ordered composition: lane k holds E_k (E_{k+1} sits LEFT of E_k);
// returns E_31 o ... o E_0 in every lane
template <class Op>
__device__ __forceinline__ typename Op::Map warp_compose_leftward(typename Op::Map m, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        typename Op::Map u = shfl_down_m<Op>(m, o);
        if (lane + o < 32) m = Op::compose(u, m);
    }
    return shfl_idx_m<Op>(m, 0);
}

// producer warp (lane 0): all jobs of this CTA, in order, through the ring
template <int NT, int S, int NBR, int NBA, bool HINT>
__device__ __forceinline__ void sweep_producer(const SweepParams &sp, uint64_t *full, uint64_t *empty,
                                               unsigned char *base, int STG, const CUtensorMap *m0,
                                               const CUtensorMap *m1, const CUtensorMap *m2) {
    const uint64_t pol = HINT ? make_policy_evict_first() : 0ull;
    SweepIt it{0, 0, false};
    sweep_norm(sp, it);
    for (int64_t j = 0; !it.done; ++j) {
        const int s = (int)(j % S);
        if (j >= S) mbar_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
        const SweepSeg sg = sweep_seg(it.s, sp.D);
        const int64_t tile = sweep_tile(sp, sg.round, it.j);
        const int rows = chunk_tile_rows<NT>(sp.c, tile);
        const int nb = sg.apply ? NBA : NBR;
        unsigned char *stage = base + s * STG;
        if (rows > 0) {
            mbar_arrive_expect_tx(&full[s], nb * NT * kRowBytes);
            const CUtensorMap *ms[3] = {m0, m1, m2};
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                if (b < nb) {
                    if (HINT && sg.apply)
                        tma_load_2d_hint(stage + b * NT * kRowBytes, ms[b], &full[s], 0, (int)(tile * NT), pol);
                    else
                        tma_load_2d(stage + b * NT * kRowBytes, ms[b], &full[s], 0, (int)(tile * NT));
                }
            }
        } else {
            mbar_arrive(&full[s]);
        }
        ++it.j;
        sweep_norm(sp, it);
    }
}

// ---- block-cyclic look-back (f1) ------------------------------------------
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_f64(double *p, double v) {
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double *p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
constexpr uint64_t kCycTimeoutNs = 4000000000ull;  // a wait this long means a missing peer: flag and go on

// wait until the status word of SB j (in this rank's buffer) carries this
// epoch; returns the state (1 = AGG; 0 after a timeout)
__device__ __forceinline__ uint32_t cyc_wait(const SweepParams &sp, int64_t j) {
    const uint32_t *f = sp.sflag[sp.cr] + j;
    uint64_t t0 = 0;
    for (int it = 0;; ++it) {
        const uint32_t v = ld_acquire_sys_u32(f);
        if ((v >> 2) == sp.epoch && (v & 3u)) return v & 3u;
        if ((it & 63) == 63) {
            const uint64_t t = globaltimer_ns();
            if (!t0) t0 = t;
            else if (t - t0 > kCycTimeoutNs || ld_flag(sp.err)) {  // after one timeout: no more waiting
                atomicOr(sp.err, 1u);
                return 0;
            }
        }
        __nanosleep(64);
    }
}
// push (state, payload) of SB J to every rank's status buffer: payload
// stores (row J of width PR, NP doubles at column off), one sys-scope
// acq_rel fence, then the status words — a release pattern at sys scope
template <int PR, int NP>
__device__ __forceinline__ void cyc_publish(const SweepParams &sp, int64_t J, int off, const double *d,
                                            uint32_t state) {
    for (int q = 0; q < sp.cw; ++q)
#pragma unroll
        for (int k = 0; k < NP; ++k) st_relaxed_sys_f64(sp.spay[q] + J * PR + off + k, d[k]);
    fence_acq_rel_sys();
    for (int q = 0; q < sp.cw; ++q) st_relaxed_sys_u32(sp.sflag[q] + J, (sp.epoch << 2) | state);
}

// Round r of a rank = its superblock J = (R - 1 - r) cw + cr.  The carry
// entering SB J from the right is X_J = M_{J+1} o M_{J+2} o ... o M_{J+cw-1}
// (E_{J+cw}): the maps of the cw - 1 superblocks between J and this rank's
// previous superblock J + cw (owned by the OTHER ranks), applied to the carry
// E_{J+cw} leaving that previous superblock — which every CTA of this rank
// already holds (it applied that SB).  So the look-back only ever waits for
// other ranks' AGG words (published right after their reduce phase: no
// chain of inclusive values across ranks), and its terminator is local.  In
// the first round (this rank's rightmost SB) it runs to the right end, where
// the carry is 0 (the return sweep's zero carry).
//
// CTA 0's carry warp, lane 0, first: the entry barrier (r == 0) and the AGG
// word of SB J (its map la) pushed to every rank.
template <class Op>
__device__ void cyc_publish_agg(const SweepParams &sp, int r, const typename Op::Map &la) {
    constexpr int MD = Op::kMapD;
    const int64_t J = (int64_t)(sp.R - 1 - r) * sp.cw + sp.cr;
    if (r == 0) {
        // entry barrier: this call writes status words into every rank's
        // buffer, so first every rank that owns a superblock must have entered
        // this epoch — i.e. finished the previous call (stream order) and with
        // it every read of the previous call's words.  Epochs increase.
        for (int q = 0; q < sp.cw; ++q) st_relaxed_sys_u32(sp.shdr[q] + 1 + sp.cr, sp.epoch);
        for (int q = 0; q < sp.cw && q < sp.nsb; ++q) {
            uint64_t t0 = 0;
            for (int it = 0; ld_acquire_sys_u32(sp.shdr[sp.cr] + 1 + q) < sp.epoch; ++it) {
                __nanosleep(64);
                if ((it & 63) == 63) {
                    const uint64_t t = globaltimer_ns();
                    if (!t0) t0 = t;
                    else if (t - t0 > kCycTimeoutNs || ld_flag(sp.err)) { atomicOr(sp.err, 1u); break; }
                }
            }
        }
    }
    double d[MD];
    map_to<Op>(la, d);
    cyc_publish<MD, MD>(sp, J, 0, d, 1u);
}
// every CTA's carry warp, lane 0: X_J from Xprev = E_{J+cw} (r > 0) or 0
template <class Op>
__device__ typename Op::Val cyc_carry(const SweepParams &sp, int r, typename Op::Val Xprev) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD;
    const int64_t J = (int64_t)(sp.R - 1 - r) * sp.cw + sp.cr;
    int64_t jend = J + sp.cw;  // this rank's previous superblock (its exit carry is Xprev)
    if (r == 0) {
        jend = sp.nsb;  // rightmost SB of this rank: look back to the array's end
#pragma unroll
        for (int q = 0; q < W; ++q) Xprev.x[q] = 0.0;
    }
    if (jend > sp.nsb) jend = sp.nsb;
    M acc = Op::map_id();
    const double *pay = sp.spay[sp.cr];
    for (int64_t j = J + 1; j < jend; ++j) {
        (void)cyc_wait(sp, j);
        double md[MD];
#pragma unroll
        for (int q = 0; q < MD; ++q) md[q] = ld_relaxed_sys_f64(pay + j * MD + q);
        acc = Op::compose(acc, map_from<Op>(md));  // acc o M_j
    }
    return Op::apply(acc, Xprev);
}

// carry warp (lane-parallel record loads, 8 in flight per lane)
template <class Op, int S>
__device__ __forceinline__ void sweep_carry_warp(const SweepParams &sp, SweepSmem<Op, S> &sm) {
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W, MD = Op::kMapD, U = 8;
    const int lane = threadIdx.x & 31, c = blockIdx.x;
    V Xin;
#pragma unroll
    for (int q = 0; q < W; ++q) Xin.x[q] = 0.0;
    const int per = (sp.G + 31) / 32;
    // this CTA's M_{r,c}: global record + release-add on arrive[r]
    auto publish = [&](int r) {
        if (r >= sp.R) return;
        mbar_wait(&sm.recbar[r % kSweepSlots], (uint32_t)((r / kSweepSlots) & 1));
        if (lane == 0) {
            double rec[MD];
            map_to<Op>(sm.rec[r % kSweepSlots], rec);
            st_rec<MD>(sp.roundRec + ((int64_t)r * sp.G + c) * MD, rec);
            red_release_add(sp.arrive + r, 1u);
        }
    };
    // the tile warps finish R(r + D) before they need carry(r)
    for (int r = 0; r <= sp.D; ++r) publish(r);
    for (int r = 0; r < sp.R; ++r) {
        const int slot = r % kSweepSlots;
        if (r > 0) publish(r + sp.D);
        // wait for the round, then compose its records (record j sits LEFT of j-1)
        // relaxed polling with back-off (every CTA polls this one counter), then
        // one acquire before the record loads
        while (ld_flag(sp.arrive + r) < (uint32_t)sp.G) {
            const long long t0 = clock64();  // ~1 us between polls (nanosleep alone wakes early)
            do {
                __nanosleep(256);
            } while (clock64() - t0 < kSweepPollCycles);
        }
        (void)ld_acquire_u32(sp.arrive + r);
        M la = Op::map_id(), lp = Op::map_id();
        const int j0 = lane * per, j1 = min(j0 + per, sp.G);
        for (int jb = j0; jb < j1; jb += U) {
            double d[U][MD];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (jb + u < j1) ld_rec<MD>(sp.roundRec + ((int64_t)r * sp.G + jb + u) * MD, d[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (jb + u < j1) {
                    M mj = map_from<Op>(d[u]);
                    la = Op::compose(mj, la);
                    if (jb + u < c) lp = Op::compose(mj, lp);
                }
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            M ua = shfl_down_m<Op>(la, o);
            M up = shfl_down_m<Op>(lp, o);
            if (lane + o < 32) {
                la = Op::compose(ua, la);
                lp = Op::compose(up, lp);
            }
        }
        if (sp.cyc) {
            // block-cyclic: the carry entering this SB, Xin = E of this rank's previous SB
            if (lane == 0) {
                const M lat = la;
                if (c == 0) cyc_publish_agg<Op>(sp, r, lat);
                const V X = cyc_carry<Op>(sp, r, Xin);
                sm.carry[slot] = Op::apply(lp, X);
                mbar_arrive(&sm.carrybar[slot]);
                Xin = Op::apply(lat, X);  // E_J: the next round's terminator
            }
            continue;
        }
        if (lane == 0) {
            sm.carry[slot] = Op::apply(lp, Xin);
            mbar_arrive(&sm.carrybar[slot]);
        }
        Xin = Op::apply(shfl_idx_m<Op>(la, 0), Xin);
    }
}

template <class Op, class T, int NT, int S, bool FWD, bool ACC, bool YS, bool HINT>
__global__ void __launch_bounds__(NT + 64, (FWD || ACC) ? 2 : 3) scan_sweep(const __grid_constant__ CUtensorMap tm_as,
                                                         const __grid_constant__ CUtensorMap tm_yb,
                                                         const __grid_constant__ CUtensorMap tm_ab,
                                                         const __grid_constant__ CUtensorMap tm_ab32,
                                                         const __grid_constant__ CUtensorMap tm_ys32,
                                                         const SweepParams sp) {
    using G = Geo<Op, T>;
    using V = typename Op::Val;
    using M = typename Op::Map;
    constexpr int W = Op::W;
    constexpr int NBR = (FWD ? 1 : 0) + 1;
    constexpr int NBA = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
    constexpr int BUF = NT * kRowBytes, STG = NBA * BUF;
    constexpr int NWT = NT / 32;
    static_assert(NT == kSweepNT && NWT == 4, "four tile warps, counted by the named barrier");
    const ChunkParams &p = sp.c;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = smem_align1024(smem_raw);
    SweepSmem<Op, S> &ss = *reinterpret_cast<SweepSmem<Op, S> *>(base + S * STG);

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&ss.full[s], 1);
            mbar_init(&ss.empty[s], NWT);
        }
        for (int s = 0; s < kSweepSlots; ++s) {
            mbar_init(&ss.recbar[s], 1);
            mbar_init(&ss.carrybar[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NWT) {  // producer
        if (lane == 0)
            sweep_producer<NT, S, NBR, NBA, HINT>(sp, ss.full, ss.empty, base, STG, FWD ? &tm_as : &tm_yb,
                                                  FWD ? &tm_yb : &tm_ab, &tm_ab);
        return;
    }
    if (warp == NWT + 1) {
        sweep_carry_warp<Op, S>(sp, ss);
        return;
    }

    const uint64_t pol = HINT ? make_policy_evict_first() : 0ull;
    V X;              // reverse carry entering the current tile from the right (every warp)
    int64_t job = 0;
    // ADD: the reverse maps X -> D + X commute, so a reduce segment needs no
    // per-tile ordering: every thread sums its rows over the segment's tiles
    constexpr bool kComm = std::is_same<Op, OpAdd>::value;
    M mthr = Op::map_id();
    int pend = -1;    // stage whose empty-arrive waits for this warp's TMA store to read it

    for (int s = 0; s < sweep_nseg(sp); ++s) {
        const SweepSeg sg = sweep_seg(s, sp.D);
        if (!sg.apply && sg.round >= sp.R) continue;
        const int cnt = sweep_count(sp, sg.round);
        const int slot = sg.round % kSweepSlots;
        const uint32_t par = (uint32_t)((sg.round / kSweepSlots) & 1);
        const int rslot = sg.round & 1;
        if (!sg.apply) {
            // ------------------------------------------------ R(r): no block barrier per tile
            for (int i = 0; i < cnt; ++i, ++job) {
                const int64_t tile = sweep_tile(sp, sg.round, i);
                const int st = (int)(job % S);
                mbar_wait(&ss.full[st], (uint32_t)((job / S) & 1));
                unsigned char *sA = base + st * STG;
                unsigned char *sY = sA + (FWD ? BUF : 0);
                const bool last = (tile == p.ntiles - 1);
                if (last && p.tail_bytes && t == (int)(p.full_rows - tile * NT)) {
                    if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                    load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
                }
                const int64_t e0 = (tile * NT + t) * G::EPR;
                M m = row_map<Op, T, FWD>(sA, sY, t, e0, last, p.n);
                __syncwarp();
                if (lane == 0) {
                    if (pend >= 0) {  // the previous job's store must have read its stage
                        tma_store_wait_read0_();
                        mbar_arrive(&ss.empty[pend]);
                        pend = -1;
                    }
                    mbar_arrive(&ss.empty[st]);
                }
                if constexpr (kComm) {
                    mthr = Op::compose(m, mthr);  // commutative maps: per-thread sum over the tiles
                } else {
                    m = warp_suffix_maps<Op>(m, lane);
                    if (lane == 0 && i < kSweepKMax) ss.ragg[rslot][i][warp] = m;
                }
            }
            if constexpr (kComm) {  // one warp reduction per segment instead of one per tile
                mthr = warp_suffix_maps<Op>(mthr, lane);
                if (lane == 0) ss.ragg[rslot][0][warp] = mthr;
                mthr = Op::map_id();
            }
            bar_tiles();
            if (kComm && warp == 1) {
                if (lane == 0) {
                    M seg = Op::map_id();
#pragma unroll
                    for (int w2 = 0; w2 < NWT; ++w2) seg = Op::compose(ss.ragg[rslot][0][w2], seg);
                    ss.rec[slot] = seg;
                    mbar_arrive(&ss.recbar[slot]);
                }
            } else if (warp == 1) {
                // E_k, k = 4i + (3 - w): tiles right to left, warps right to left within a tile
                M seg = Op::map_id();
                for (int b = 0; b < cnt * NWT; b += 32) {
                    const int k = b + lane;
                    M e = Op::map_id();
                    if (k < cnt * NWT) e = ss.ragg[rslot][k >> 2][3 - (k & 3)];
                    seg = Op::compose(warp_compose_leftward<Op>(e, lane), seg);
                }
                if (lane == 0) {
                    ss.rec[slot] = seg;
                    mbar_arrive(&ss.recbar[slot]);
                }
            }
            continue;
        }
        // ---------------------------------------------------- A(r)
        mbar_wait(&ss.carrybar[slot], par);
        X = ss.carry[slot];
        for (int i = 0; i < cnt; ++i, ++job) {
            const int64_t tile = sweep_tile(sp, sg.round, i);
            const int st = (int)(job % S);
            const int jp = (int)(job & 1);
            V Ftile = Op::fwd_id();
            if (FWD) {
#pragma unroll
                for (int q = 0; q < W; ++q) Ftile.x[q] = ld_cg(p.tileP + tile * W + q);
            }
            mbar_wait(&ss.full[st], (uint32_t)((job / S) & 1));
            unsigned char *sA = base + st * STG;
            unsigned char *sY = sA + (FWD ? BUF : 0);
            unsigned char *sC = sY + BUF;
            const bool last = (tile == p.ntiles - 1);
            const bool has_partial = last && p.tail_bytes && t == (int)(p.full_rows - tile * NT);
            if (has_partial) {
                if (FWD) load_partial_row(sA, t, p.as, p.full_rows, p.tail_bytes);
                load_partial_row(sY, t, p.ys_bar, p.full_rows, p.tail_bytes);
                if (ACC) load_partial_row(sC, t, p.as_bar, p.full_rows, p.tail_bytes);
            }
            const int64_t e0 = (tile * NT + t) * G::EPR;

            // row aggregates -> warp scans -> warp aggregates (one barrier)
            V fin = Op::fwd_id();
            if (FWD) {
                fin = warp_prefix_vals<Op>(row_fwd<Op, T, FWD>(sA, t, e0, last, p.n), lane);
                if (lane == 31) ss.aggF[jp][warp] = fin;
            }
            M sfx = warp_suffix_maps<Op>(row_map<Op, T, FWD>(sA, sY, t, e0, last, p.n), lane);
            if (lane == 0) ss.aggM[jp][warp] = sfx;
            bar_tiles();

            // rs entering this row: Ftile (.) warps to the left (.) lanes to the left
            V rin = Ftile;
            if (FWD) {
#pragma unroll
                for (int k = 0; k < NWT - 1; ++k)
                    if (k < warp) rin = Op::fwd(rin, ss.aggF[jp][k]);
                V fex = shfl_up_v(fin, 1);
                if (lane > 0) rin = Op::fwd(rin, fex);
            }
            // H entering this row from the right: lanes to the right o warps to the right (X)
            V xw = X;
#pragma unroll
            for (int k = NWT - 1; k > 0; --k)
                if (k > warp) xw = Op::apply(ss.aggM[jp][k], xw);
            M sex = shfl_down_m<Op>(sfx, 1);
            V Xr = (lane == 31) ? xw : Op::apply(sex, xw);
            // carry for the next tile (identical in every warp)
            {
                V xn = X;
#pragma unroll
                for (int k = NWT - 1; k >= 0; --k) xn = Op::apply(ss.aggM[jp][k], xn);
                X = xn;
            }

            V rsp[G::EPR];
            if constexpr (FWD) {
                V r = rin;
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
            if constexpr (std::is_same<Op, OpAdd>::value && !FWD && sizeof(T) == 8) {
                // + (f64): group sums first, then the suffix over the groups,
                // then inside each group — dependent chain NG + EG instead of EPR
                double yv[G::EPR], gs[G::NG], gsuf[G::NG];
#pragma unroll
                for (int g = 0; g < G::NG; ++g) {
                    uint32_t wy[G::GB / 4];
                    lds_group<G::GB>(sY, t, g, wy);
                    gs[g] = 0.0;
#pragma unroll
                    for (int e = 0; e < G::EG; ++e) {
                        const int q = g * G::EG + e;
                        yv[q] = (!last || e0 + q < p.n) ? dec<T, 1>(wy + e * (G::ES / 4)).x[0] : 0.0;
                        gs[g] += yv[q];
                    }
                }
                gsuf[G::NG - 1] = Xr.x[0];
#pragma unroll
                for (int g = G::NG - 2; g >= 0; --g) gsuf[g] = gsuf[g + 1] + gs[g + 1];
#pragma unroll
                for (int g = G::NG - 1; g >= 0; --g) {
                    uint32_t wc[G::GB / 4], wo[G::GB / 4];
                    if (ACC) lds_group<G::GB>(sC, t, g, wc);
                    double run = gsuf[g];
#pragma unroll
                    for (int e = G::EG - 1; e >= 0; --e) {
                        const int q = g * G::EG + e;
                        run = yv[q] + run;
                        V o;
                        o.x[0] = run;
                        if (ACC) o.x[0] += dec<T, 1>(wc + e * (G::ES / 4)).x[0];
                        enc<T, 1>(o, wo + e * (G::ES / 4));
                    }
                    sts_group<G::GB>(sY, t, g, wo);
                }
                Xr.x[0] = gsuf[0] + gs[0];
            } else {
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
                    V gv;
#pragma unroll
                    for (int z = 0; z < W; ++z) gv.x[z] = y.x[z] + Xr.x[z];
                    V o = Op::out(rsp[q], a, gv);
                    if (Op::kFirstSpecial && p.global_first && e0 + q == 0) o = gv;
                    if (ACC) {
                        V cc = dec<T, W>(wc + e * (G::ES / 4));
#pragma unroll
                        for (int z = 0; z < W; ++z) o.x[z] += cc.x[z];
                    }
                    enc<T, W>(o, wo + e * (G::ES / 4));
                    if (YS) enc<T, W>(Op::fwd(rsp[q], a), wz + e * (G::ES / 4));
                    if (!last || e0 + q < p.n) Xr = Op::pass_left(rsp[q], a, gv);
                }
                sts_group<G::GB>(sY, t, g, wo);
                if (YS) sts_group<G::GB>(sA, t, g, wz);
            }
            }
            if (has_partial) {
                store_partial_row(sY, t, p.as_bar, p.full_rows, p.tail_bytes);
                if (YS) store_partial_row(sA, t, p.ys, p.full_rows, p.tail_bytes);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                const int rows = chunk_tile_rows<NT>(p, tile);
                if (rows > 32 * warp) {
                    const int row0 = (int)(tile * NT) + 32 * warp;
                    if (HINT) {
                        tma_store_2d_hint(&tm_ab32, sY + 32 * warp * kRowBytes, 0, row0, pol);
                        if (YS) tma_store_2d_hint(&tm_ys32, sA + 32 * warp * kRowBytes, 0, row0, pol);
                    } else {
                        tma_store_2d(&tm_ab32, sY + 32 * warp * kRowBytes, 0, row0);
                        if (YS) tma_store_2d(&tm_ys32, sA + 32 * warp * kRowBytes, 0, row0);
                    }
                }
                tma_store_commit();
                if (pend >= 0) {
                    tma_store_wait_read1();
                    mbar_arrive(&ss.empty[pend]);
                }
                pend = st;
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace vjpk
