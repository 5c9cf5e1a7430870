// scan_impl.cuh — host driver of the vjp_scan kernels (validation is done by
// the C-ABI layer in scan_abi.cu; this file owns workspace layout and launches).
#pragma once

#include <mutex>
#include <type_traits>

#include <cstdio>
#include <cstdlib>

#include "scan_blocklb.cuh"
#include "scan_add1p.cuh"
#include "scan_ext1p.cuh"

namespace vjph {

// Tuning knobs of the scan paths, read ONCE per process (first use) from the
// environment — never per call, so a call's behaviour depends only on its
// arguments and on these process-wide constants (documented in vjp.h):
//   VJP_LB_L2_MB      block look-back: L2 bytes held by the blocks in flight (MB)
//   VJP_LB_VARIANT    block look-back TMA stages (0: 3, 1: 2)
//   VJP_SWEEP_K / VJP_SWEEP_D / VJP_SWEEP_ROUND_MB   one-read sweep geometry
struct ScanTune {
    int lb_l2_mb, lb_variant, sweep_k, sweep_d, sweep_round_mb;
};
inline int tune_env(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}
inline const ScanTune &scan_tune() {
    static const ScanTune t{tune_env("VJP_LB_L2_MB", 40), tune_env("VJP_LB_VARIANT", 0), tune_env("VJP_SWEEP_K", 0),
                            tune_env("VJP_SWEEP_D", 1),
                            tune_env("VJP_SWEEP_ROUND_MB", 32)};
    return t;
}

// tuning only: a device buffer for per-block timestamps of the block look-back
// (set by vjp_debug_lb_trace; nullptr = off)
unsigned long long *&lb_trace_ptr();

struct ScanCall {
    vjp_op op;
    vjp_dtype dtype;
    int64_t n;
    const void *as;
    const void *ys_bar;
    void *as_bar;
    void *ys;
    void *ws;
    size_t ws_bytes;
    cudaStream_t stream;
    unsigned flags;
    int32_t rank, world;
    int64_t global_offset;
    void *partial;         // partial phase: record output (device)
    const void *gathered;  // finish phase: world records (device)
    const vjp_cyclic *cyc; // block-cyclic multi-GPU call (f1), else nullptr
};

enum ScanPhase { kScanWs = 0, kScanPartial = 1, kScanFinish = 2, kScanPartialBytes = 3, kReduceGeneral = 4,
                 kScanPartial2 = 5, kScanIdentity = 6, kCycForward = 7, kCycFinish = 8, kCycSbTiles = 9 };

template <class Op, class T>
struct ScanImpl {
    using G = vjpk::Geo<Op, T>;
    static constexpr int W = Op::W;
    static constexpr int MD = Op::kMapD;
    static constexpr int R1MAX = W + MD;

    // chunked path geometry (scan_chunked.cuh)
    static constexpr int NTC = 128;  // rows (threads) per tile
    static constexpr int SC = 3;     // TMA ring stages
    static constexpr int kMaxChunks = 4096;
    static constexpr int64_t TILE_C = (int64_t)G::EPR * NTC;

    struct Layout {
        int64_t ntiles;
        size_t counters, flags1, flags2, memset_bytes, p1agg, p1inc, p2agg, p2inc, partial;
        int64_t ntiles_c;
        size_t tileF, tileP, chunkRec, counter_c, roundRec, arrive, lbFlags, lbAgg, lbInc, lbTileF, lbTileP, lbPark,
            p1Ctr, p1Agg, p1Inc, p1Grp, p1End, pxCtr, pxAgg, pxInc, pxGrp, pxEnd, total;
        int64_t p1Tiles;
    };
    static Layout layout(int64_t n) {
        Layout L{};
        L.ntiles = n > 0 ? (n + G::TILE_E - 1) / G::TILE_E : 0;
        size_t off = 0;
        L.counters = off; off += 256;
        L.flags1 = off; off += align256((size_t)L.ntiles * 4);
        L.flags2 = off; off += align256((size_t)L.ntiles * 4);
        L.memset_bytes = off;
        L.p1agg = off; off += align256((size_t)L.ntiles * R1MAX * 8);
        L.p1inc = off; off += align256((size_t)L.ntiles * R1MAX * 8);
        L.p2agg = off; off += align256((size_t)L.ntiles * MD * 8);
        L.p2inc = off; off += align256((size_t)L.ntiles * MD * 8);
        L.partial = off; off += align256((size_t)R1MAX * 8);
        L.ntiles_c = n > 0 ? (n + TILE_C - 1) / TILE_C : 0;
        L.tileF = off; off += align256((size_t)L.ntiles_c * W * 8);
        L.tileP = off; off += align256((size_t)L.ntiles_c * W * 8);
        L.chunkRec = off; off += align256((size_t)kMaxChunks * R1MAX * 8);
        L.counter_c = off; off += 256;
        // sweep: R*G <= ntiles_c/K + G <= ntiles_c + kMaxChunks records; R <= ntiles_c
        L.roundRec = off; off += align256((size_t)(L.ntiles_c + kMaxChunks) * MD * 8);
        L.arrive = off; off += align256((size_t)(L.ntiles_c + 1) * 4);
        // block look-back: [ticket | pad to 256 B | flags per block], maps and
        // inclusive values per block (at most one block per tile)
        const int64_t ntl = ntiles_of(n, NTL_MIN);
        L.lbFlags = off; off += 256 + align256((size_t)ntl * 4);
        L.lbAgg = off; off += align256((size_t)ntl * MD * 8);
        L.lbInc = off; off += align256((size_t)ntl * W * 8);
        L.lbTileF = off; off += align256((size_t)ntl * W * 8);
        L.lbTileP = off; off += align256((size_t)ntl * W * 8);
        L.lbPark = off; off += align256((size_t)NTL_MIN * (W + MD) * 8);  // the last tile's parked rows
        // one-pass scan(+) (scan_add1p.cuh): ticket + group counters | records
        L.p1Tiles = n > 0 ? (n + P1_TE - 1) / P1_TE : 0;
        const int64_t p1g = (L.p1Tiles + 31) / 32;
        L.p1Ctr = off; off += align256(256 + (size_t)p1g * 4);
        L.p1Agg = off; off += align256((size_t)L.p1Tiles * 16);
        L.p1Inc = off; off += align256((size_t)L.p1Tiles * 16);
        L.p1Grp = off; off += align256((size_t)p1g * 16);
        L.p1End = off;
        // one-pass MIN/MAX return (scan_ext1p.cuh): records per 256-row tile
        {
            const int64_t xg = (L.ntiles + 31) / 32;
            L.pxCtr = off; off += align256(256 + (size_t)xg * 4);
            L.pxAgg = off; off += align256((size_t)L.ntiles * 16);
            L.pxInc = off; off += align256((size_t)L.ntiles * 16);
            L.pxGrp = off; off += align256((size_t)xg * 16);
            L.pxEnd = off;
        }
        L.total = off;
        return L;
    }

    static vjpk::ScanParams params(const ScanCall &c, const Layout &L) {
        vjpk::ScanParams p{};
        const int64_t bytes = c.n * (int64_t)G::ES;
        p.n = c.n;
        p.full_rows = bytes / vjpk::kRowBytes;
        p.tail_bytes = (int32_t)(bytes % vjpk::kRowBytes);
        p.ntiles = (int32_t)L.ntiles;
        p.as = c.as;
        p.ys_bar = c.ys_bar;
        p.as_bar = c.as_bar;
        p.ys = c.ys;
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        p.counters = reinterpret_cast<uint32_t *>(ws + L.counters);
        p.flags1 = reinterpret_cast<uint32_t *>(ws + L.flags1);
        p.flags2 = reinterpret_cast<uint32_t *>(ws + L.flags2);
        p.p1_agg = reinterpret_cast<double *>(ws + L.p1agg);
        p.p1_inc = reinterpret_cast<double *>(ws + L.p1inc);
        p.p2_agg = reinterpret_cast<double *>(ws + L.p2agg);
        p.p2_inc = reinterpret_cast<double *>(ws + L.p2inc);
        p.partial = c.partial ? static_cast<double *>(c.partial) : reinterpret_cast<double *>(ws + L.partial);
        p.gathered = static_cast<const double *>(c.gathered);
        p.rank = c.rank;
        p.world = c.world;
        p.global_first = (c.global_offset == 0) ? 1 : 0;
        return p;
    }

    static size_t smem_bytes(int nb) { return 1024 + (size_t)nb * vjpk::kTileBytes + 2048; }

    template <class K>
    static void set_smem(K kernel, size_t bytes) {
        // idempotent and cheap; done on every launch so multi-device use works
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    }

    static bool maps(const ScanCall &c, int64_t rows, CUtensorMap *m_as, CUtensorMap *m_yb, CUtensorMap *m_ab,
                     CUtensorMap *m_ys) {
        const bool f64 = sizeof(T) == 8;
        bool ok = true;
        ok &= c.as ? make_row_tmap(m_as, c.as, rows, f64) : make_row_tmap(m_as, nullptr, 0, f64);
        ok &= make_row_tmap(m_yb, c.ys_bar, rows, f64);
        ok &= c.as_bar ? make_row_tmap(m_ab, c.as_bar, rows, f64) : make_row_tmap(m_ab, nullptr, 0, f64);
        ok &= c.ys ? make_row_tmap(m_ys, c.ys, rows, f64) : make_row_tmap(m_ys, nullptr, 0, f64);
        return ok;
    }

    template <bool FWD, bool REV>
    static vjp_status launch_pass1(const ScanCall &c, const vjpk::ScanParams &p, const CUtensorMap &ma,
                                   const CUtensorMap &my) {
        constexpr int NB = (FWD ? 1 : 0) + (REV ? 1 : 0);
        auto k = vjpk::scan_pass1<Op, T, FWD, REV>;
        size_t sm = smem_bytes(NB);
        set_smem(k, sm);
        k<<<(unsigned)p.ntiles, vjpk::kThreads, sm, c.stream>>>(ma, my, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    template <bool FWD, bool ACC, bool YS>
    static vjp_status launch_pass2(const ScanCall &c, const vjpk::ScanParams &p, const CUtensorMap &ma,
                                   const CUtensorMap &my, const CUtensorMap &mab, const CUtensorMap &mys) {
        constexpr int NB = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
        auto k = vjpk::scan_pass2<Op, T, FWD, ACC, YS>;
        size_t sm = smem_bytes(NB);
        set_smem(k, sm);
        k<<<(unsigned)p.ntiles, vjpk::kThreads, sm, c.stream>>>(ma, my, mab, mys, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    // ---------------- chunked reduce-then-scan path ----------------
    static size_t smem_r(int nb) {
        return 1024 + (size_t)SC * nb * NTC * vjpk::kRowBytes + sizeof(vjpk::ReduceSmem<Op, NTC, SC>);
    }
    static size_t smem_a(int nb) {
        return 1024 + (size_t)SC * nb * NTC * vjpk::kRowBytes + sizeof(vjpk::ApplySmem<Op, NTC, SC>);
    }

    static vjpk::ChunkParams cparams(const ScanCall &c, const Layout &L, int nchunks) {
        vjpk::ChunkParams p{};
        const int64_t bytes = c.n * (int64_t)G::ES;
        p.n = c.n;
        p.full_rows = bytes / vjpk::kRowBytes;
        p.tail_bytes = (int32_t)(bytes % vjpk::kRowBytes);
        p.ntiles = (int32_t)L.ntiles_c;
        p.nchunks = nchunks;
        p.as = c.as;
        p.ys_bar = c.ys_bar;
        p.as_bar = c.as_bar;
        p.ys = c.ys;
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        p.tileF = reinterpret_cast<double *>(ws + L.tileF);
        p.tileP = reinterpret_cast<double *>(ws + L.tileP);
        p.chunkRec = reinterpret_cast<double *>(ws + L.chunkRec);
        p.counter = reinterpret_cast<uint32_t *>(ws + L.counter_c);
        p.partial = (c.world > 1) ? static_cast<double *>(c.partial) : nullptr;
        p.gathered = static_cast<const double *>(c.gathered);
        p.rank = c.rank;
        p.world = c.world;
        p.global_first = (c.global_offset == 0) ? 1 : 0;
        return p;
    }

    template <class K>
    static int occupancy(K kernel, size_t smem) {
        set_smem(kernel, smem);
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, NTC, smem) != cudaSuccess || nb < 1) nb = 1;
        return nb;
    }

    // one chunk per co-resident CTA of the heavier kernel (identical for both phases)
    static int nchunks_for(const Layout &L, bool fwd, bool acc) {
        constexpr int nbR = 2;
        int occR = fwd ? occupancy(vjpk::scan_reduce<Op, T, NTC, SC, true, true>, smem_r(nbR))
                       : occupancy(vjpk::scan_reduce<Op, T, NTC, SC, false, true>, smem_r(1));
        int nbC = (fwd ? 1 : 0) + 1 + (acc ? 1 : 0);
        int occC = fwd ? occupancy(vjpk::scan_apply<Op, T, NTC, SC, true, false, false>, smem_a(nbC))
                       : occupancy(vjpk::scan_apply<Op, T, NTC, SC, false, false, false>, smem_a(nbC));
        int per = occR < occC ? occR : occC;
        int64_t g = (int64_t)sm_count() * per;
        if (g > kMaxChunks) g = kMaxChunks;
        if (g > L.ntiles_c) g = L.ntiles_c;
        return (int)(g < 1 ? 1 : g);
    }

    static bool maps_c(const ScanCall &c, int64_t rows, CUtensorMap *m_as, CUtensorMap *m_yb, CUtensorMap *m_ab,
                       CUtensorMap *m_ys) {
        const bool f64 = sizeof(T) == 8;
        bool ok = true;
        ok &= make_row_tmap(m_as, c.as, c.as ? rows : 0, f64, NTC);
        ok &= make_row_tmap(m_yb, c.ys_bar, rows, f64, NTC);
        ok &= make_row_tmap(m_ab, c.as_bar, c.as_bar ? rows : 0, f64, NTC);
        ok &= make_row_tmap(m_ys, c.ys, c.ys ? rows : 0, f64, NTC);
        return ok;
    }

    template <bool FWD>
    static vjp_status launch_reduce(const ScanCall &c, const vjpk::ChunkParams &p, const CUtensorMap &ma,
                                    const CUtensorMap &my) {
        constexpr int NB = (FWD ? 1 : 0) + 1;
        auto k = vjpk::scan_reduce<Op, T, NTC, SC, FWD, true>;
        size_t sm = smem_r(NB);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    template <bool FWD, bool ACC, bool YS>
    static vjp_status launch_apply(const ScanCall &c, const vjpk::ChunkParams &p, const CUtensorMap &ma,
                                   const CUtensorMap &my, const CUtensorMap &mab, const CUtensorMap &mys) {
        constexpr int NB = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
        auto k = vjpk::scan_apply<Op, T, NTC, SC, FWD, ACC, YS>;
        size_t sm = smem_a(NB);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, mab, mys, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    static bool use_chunked(const ScanCall &c) {
        return !Op::kRevNeedsRs && !(c.flags & VJP_SCAN_LOOKBACK);
    }

    static vjp_status partial_c(const ScanCall &c) {
        Layout L = layout(c.n);
        const bool fwd = need_fwd(c);
        const int G = nchunks_for(L, fwd, (c.flags & VJP_ACCUMULATE) != 0);
        vjpk::ChunkParams p = cparams(c, L, G);
        if (c.world > 1 && cudaMemsetAsync(p.counter, 0, 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        if constexpr (std::is_same<Op, vjpk::OpAdd>::value) {
            if (!fwd) return launch_reduce<false>(c, p, ma, my);
        }
        return launch_reduce<true>(c, p, ma, my);
    }

    static vjp_status finish_c(const ScanCall &c) {
        Layout L = layout(c.n);
        const bool fwd = need_fwd(c);
        const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
        const int G = nchunks_for(L, fwd, acc);
        vjpk::ChunkParams p = cparams(c, L, G);
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const bool ys = c.ys != nullptr;
        if constexpr (std::is_same<Op, vjpk::OpAdd>::value) {
            if (!ys)
                return acc ? launch_apply<false, true, false>(c, p, ma, my, mab, mys)
                           : launch_apply<false, false, false>(c, p, ma, my, mab, mys);
        }
        if (acc) return ys ? launch_apply<true, true, true>(c, p, ma, my, mab, mys)
                           : launch_apply<true, true, false>(c, p, ma, my, mab, mys);
        return ys ? launch_apply<true, false, true>(c, p, ma, my, mab, mys)
                  : launch_apply<true, false, false>(c, p, ma, my, mab, mys);
    }

    static bool need_fwd(const ScanCall &c) {
        return !std::is_same<Op, vjpk::OpAdd>::value || c.ys != nullptr;
    }

    // ---------------- single-read L2-round sweep (world == 1) ----------------
    static constexpr int SW_S_1 = 4;  // TMA stages when a stage is one 16 KB buffer
    static constexpr int SW_S_2 = 3;  // ... two or three buffers

    // the one-read sweep is the default for f64 scan(+) without ys on one GPU
    // (its reverse maps commute: 3.73 vs 4.14 ms at 2^30 f64; for f32 the
    // chunked kernels are faster, 2.20 vs 2.78 ms at 2^30); the other operators
    // take it only on request (their shuffle scans of d-vector maps make it
    // slower than the chunked kernels)
    static bool use_sweep(const ScanCall &c) {
        if (c.world != 1 || (c.flags & (VJP_SCAN_LOOKBACK | VJP_SCAN_CHUNKED | VJP_SCAN_BLOCKLB))) return false;
        if (c.ys) return false;  // the sweep does not write the primal ys (the other paths do)
        if (c.flags & VJP_SCAN_SWEEP) return true;
        return std::is_same<Op, vjpk::OpAdd>::value && sizeof(T) == 8 && c.ys == nullptr;
    }

    template <bool FWD, bool ACC, bool YS>
    static constexpr int sw_stages() { return ((FWD ? 1 : 0) + 1 + (ACC ? 1 : 0)) == 1 ? SW_S_1 : SW_S_2; }

    template <bool FWD, bool ACC, bool YS>
    static size_t smem_sw() {
        constexpr int S = sw_stages<FWD, ACC, YS>();
        constexpr int NBA = (FWD ? 1 : 0) + 1 + (ACC ? 1 : 0);
        return 1024 + (size_t)S * NBA * NTC * vjpk::kRowBytes + sizeof(vjpk::SweepSmem<Op, S>);
    }

    // K_F chunking (forward aggregates only) shared by partial and finish
    static int nchunks_fwd(const Layout &L) {
        int occ = occupancy(vjpk::scan_reduce<Op, T, NTC, SC, true, false>, smem_r(1));
        int64_t g = (int64_t)sm_count() * occ;
        if (g > kMaxChunks) g = kMaxChunks;
        if (g > L.ntiles_c) g = L.ntiles_c;
        return (int)(g < 1 ? 1 : g);
    }

    static vjp_status partial_sw(const ScanCall &c) {
        if (!need_fwd(c)) return VJP_OK;  // ADD closed form: nothing before the sweep
        Layout L = layout(c.n);
        vjpk::ChunkParams p = cparams(c, L, nchunks_fwd(L));
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        auto k = vjpk::scan_reduce<Op, T, NTC, SC, true, false>;
        size_t sm = smem_r(1);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    template <bool FWD, bool ACC, bool YS>
    static vjp_status launch_sweep(const ScanCall &c, const Layout &L) {
        constexpr int S = sw_stages<FWD, ACC, YS>();
        constexpr int NBR = (FWD ? 1 : 0) + 1;
        constexpr int NTH = NTC + 64;  // four tile warps + producer + carry
        auto k = vjpk::scan_sweep<Op, T, NTC, S, FWD, ACC, YS, true>;
        const size_t sm = smem_sw<FWD, ACC, YS>();
        set_smem(k, sm);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTH, sm) != cudaSuccess || occ < 1) occ = 1;
        vjpk::SweepParams sp{};
        sp.c = cparams(c, L, 1);
        int64_t G = (int64_t)sm_count() * occ;
        if (G > kMaxChunks) G = kMaxChunks;
        // tiles per CTA per round: about `round_mb` MB of HBM-read input per round
        const int64_t round_bytes = (int64_t)scan_tune().sweep_round_mb << 20;
        int64_t K = round_bytes / (G * NBR * NTC * vjpk::kRowBytes);
        if (std::is_same<Op, vjpk::OpAdd>::value) K = 4;  // measured best for scan(+) at 2^26..2^30 (DESIGN 7.6)
        if (scan_tune().sweep_k > 0) K = scan_tune().sweep_k;
        if (K < 1) K = 1;
        if (K > vjpk::kSweepKMax) K = vjpk::kSweepKMax;
        if (G * K > L.ntiles_c) {  // small inputs: fewer, fuller CTAs
            K = 1;
            if (G > L.ntiles_c) G = L.ntiles_c;
        }
        sp.G = (int32_t)G;
        sp.K = (int32_t)K;
        sp.R = (int32_t)((L.ntiles_c + G * K - 1) / (G * K));
        sp.D = scan_tune().sweep_d >= 2 ? 2 : 1;
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        sp.roundRec = reinterpret_cast<double *>(ws + L.roundRec);
        sp.arrive = reinterpret_cast<uint32_t *>(ws + L.arrive);
        if (cudaMemsetAsync(sp.arrive, 0, (size_t)sp.R * 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        CUtensorMap ma, my, mab, mys, mab32, mys32;
        if (!maps_c(c, sp.c.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const bool f64 = sizeof(T) == 8;
        if (!make_row_tmap(&mab32, c.as_bar, sp.c.full_rows, f64, 32)) return VJP_ECUDA;
        if (!make_row_tmap(&mys32, c.ys, c.ys ? sp.c.full_rows : 0, f64, 32)) return VJP_ECUDA;
        void *args[] = {&ma, &my, &mab, &mab32, &mys32, &sp};
        cudaError_t e = cudaLaunchCooperativeKernel((const void *)k, dim3((unsigned)G), dim3(NTH), args, sm, c.stream);
        if (e == cudaErrorCooperativeLaunchTooLarge) {
            // the GPU cannot hold all CTAs at once right now (e.g. another kernel is
            // resident): the sweep's round synchronisation would not be safe, so
            // the call takes the chunked kernels instead (same results)
            (void)cudaGetLastError();
            return VJP_EUNSUPPORTED;
        }
        count_launch();
        return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    static vjp_status finish_sw(const ScanCall &c) {
        Layout L = layout(c.n);
        const bool fwd = need_fwd(c);
        const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
        const bool ys = c.ys != nullptr;
        if (fwd) {
            vjpk::ChunkParams p = cparams(c, L, nchunks_fwd(L));
            vjpk::scan_tile_prefix<Op, NTC><<<(unsigned)p.nchunks, NTC, 0, c.stream>>>(p);
            count_launch();
            if (cudaGetLastError() != cudaSuccess) return VJP_ECUDA;
        }
        vjp_status st;
        if (std::is_same<Op, vjpk::OpAdd>::value && !ys)
            st = acc ? launch_sweep<false, true, false>(c, L) : launch_sweep<false, false, false>(c, L);
        else if (acc)
            st = ys ? launch_sweep<true, true, true>(c, L) : launch_sweep<true, true, false>(c, L);
        else
            st = ys ? launch_sweep<true, false, true>(c, L) : launch_sweep<true, false, false>(c, L);
        if (st == VJP_EUNSUPPORTED) {  // cooperative launch refused: the chunked kernels
            vjp_status s2 = partial_c(c);
            return s2 == VJP_OK ? finish_c(c) : s2;
        }
        return st;
    }

    // ---------------- one-pass scan(+) with two-level look-back (scan_add1p.cuh) ----------------
    static constexpr int P1_RPT = 3;  // rows per thread: 96 KB tiles
    static constexpr int64_t P1_TE = (int64_t)vjpk::k1pData * P1_RPT * 128 / (int64_t)sizeof(T);
    static bool use_1p(const ScanCall &c) {
        if constexpr (!std::is_same<Op, vjpk::OpAdd>::value) {
            return false;
        } else {
            if (c.world != 1 || c.ys || c.cyc) return false;
            if (c.flags & (VJP_SCAN_LOOKBACK | VJP_SCAN_CHUNKED | VJP_SCAN_SWEEP | VJP_SCAN_BLOCKLB | VJP_ACCUMULATE))
                return false;  // ACCUMULATE (as_bar read as well) keeps the sweep / chunked kernels
            // 1-D bulk copies: 16-byte aligned arrays (the ABI's requirement)
            return true;
        }
    }
    static vjp_status launch_1p(const ScanCall &c) {
        Layout L = layout(c.n);
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        if (cudaMemsetAsync(ws + L.p1Ctr, 0, L.p1End - L.p1Ctr, c.stream) != cudaSuccess) return VJP_ECUDA;
        vjpk::Add1pParams P{};
        P.n = c.n;
        P.ntiles = L.p1Tiles;
        P.ys_bar = c.ys_bar;
        P.as_bar = c.as_bar;
        P.ticket = reinterpret_cast<uint32_t *>(ws + L.p1Ctr);
        P.gcount = reinterpret_cast<uint32_t *>(ws + L.p1Ctr + 256);
        P.agg = reinterpret_cast<double2 *>(ws + L.p1Agg);
        P.inc = reinterpret_cast<double2 *>(ws + L.p1Inc);
        P.grp = reinterpret_cast<double2 *>(ws + L.p1Grp);
        const int64_t rows = c.n * (int64_t)sizeof(T) / vjpk::kRowBytes;  // full 128-byte rows
        CUtensorMap mi, mo;
        if (!make_row_tmap(&mi, c.ys_bar, rows, sizeof(T) == 8, 256) ||
            !make_row_tmap(&mo, c.as_bar, rows, sizeof(T) == 8, 256))
            return VJP_ECUDA;
        constexpr size_t sm = 1024 + (size_t)vjpk::k1pData * P1_RPT * 128;
        auto k = vjpk::scan_add_1p<T, P1_RPT>;
        set_smem(k, sm);
        vjpk::Add1pParams Q = P;
        Q.ntiles = (c.n + P1_TE - 1) / P1_TE;
        k<<<(unsigned)Q.ntiles, vjpk::k1pData + 32, sm, c.stream>>>(mi, mo, Q);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }

    // ---------------- block-cyclic multi-GPU sweep (scan_sweep.cuh) ----------------
    // geometry shared by every rank: tiles per superblock (the SB size is the
    // caller's, identical on all ranks), this rank's local SBs, CTAs
    static int64_t cyc_tps(const vjp_cyclic &cy) { return cy.sb_elems / TILE_C; }
    static int64_t cyc_nsb(const vjp_cyclic &cy) { return (cy.global_n + cy.sb_elems - 1) / cy.sb_elems; }
    static int64_t cyc_nloc(const vjp_cyclic &cy, int rank) {
        const int64_t nsb = cyc_nsb(cy);
        return nsb > rank ? (nsb - 1 - rank) / cy.world + 1 : 0;
    }
    template <bool FWD, bool ACC, bool YS>
    static int cyc_occupancy() {
        constexpr int S = sw_stages<FWD, ACC, YS>();
        auto k = vjpk::scan_sweep<Op, T, NTC, S, FWD, ACC, YS, true>;
        const size_t sm = smem_sw<FWD, ACC, YS>();
        set_smem(k, sm);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTC + 64, sm) != cudaSuccess || occ < 1) occ = 1;
        return occ;
    }
    // forward pass (FWD operators): K_F tile aggregates, then per local SB its aggregate -> c.partial [nloc][W]
    static vjp_status cyc_forward(const ScanCall &c) {
        if (!need_fwd(c)) return VJP_OK;
        const vjp_cyclic &cy = *c.cyc;
        Layout L = layout(c.n);
        vjpk::ChunkParams p = cparams(c, L, nchunks_fwd(L));
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        auto k = vjpk::scan_reduce<Op, T, NTC, SC, true, false>;
        const size_t sm = smem_r(1);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, p);
        const int64_t nloc = cyc_nloc(cy, cy.rank);
        vjpk::scan_cyc_sbagg<Op, NTC><<<(unsigned)nloc, NTC, 0, c.stream>>>(p, (int32_t)cyc_tps(cy),
                                                                           static_cast<double *>(c.partial));
        count_launch(2);
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    template <bool FWD, bool ACC, bool YS>
    static vjp_status cyc_launch(const ScanCall &c, const Layout &L) {
        constexpr int S = sw_stages<FWD, ACC, YS>();
        constexpr int NTH = NTC + 64;
        const vjp_cyclic &cy = *c.cyc;
        auto k = vjpk::scan_sweep<Op, T, NTC, S, FWD, ACC, YS, true>;
        const size_t sm = smem_sw<FWD, ACC, YS>();
        set_smem(k, sm);
        int64_t G = cy.grid_ctas > 0 ? cy.grid_ctas : (int64_t)sm_count() * cyc_occupancy<FWD, ACC, YS>();
        if (G > kMaxChunks) G = kMaxChunks;
        const int64_t tps = cyc_tps(cy);
        if (G > tps) G = tps;  // a CTA per tile at most (keeps R * G records within the workspace)
        int64_t K = (tps + G - 1) / G;
        if (K > vjpk::kSweepKMax) return VJP_EINVAL;  // superblock too large for this grid
        vjpk::SweepParams sp{};
        sp.c = cparams(c, L, 1);
        sp.c.global_first = cy.rank == 0 ? 1 : 0;
        sp.G = (int32_t)G;
        sp.K = (int32_t)K;
        sp.R = (int32_t)cyc_nloc(cy, cy.rank);
        sp.D = 1;
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        sp.roundRec = reinterpret_cast<double *>(ws + L.roundRec);
        sp.arrive = reinterpret_cast<uint32_t *>(ws + L.arrive);
        sp.cyc = 1;
        sp.cw = cy.world;
        sp.cr = cy.rank;
        sp.epoch = cy.epoch;
        sp.tps = (int32_t)tps;
        sp.nsb = (int32_t)cyc_nsb(cy);
        for (int q = 0; q < cy.world; ++q) {
            unsigned char *b = static_cast<unsigned char *>(cy.status[q]);
            sp.shdr[q] = reinterpret_cast<uint32_t *>(b);
            sp.sflag[q] = reinterpret_cast<uint32_t *>(b + 256);
            sp.spay[q] = reinterpret_cast<double *>(b + 256 + align256((size_t)sp.nsb * 4));
        }
        sp.err = static_cast<uint32_t *>(cy.status[cy.rank]);  // word 0 of this rank's status buffer
        if (cudaMemsetAsync(sp.arrive, 0, (size_t)sp.R * 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        CUtensorMap ma, my, mab, mys, mab32, mys32;
        if (!maps_c(c, sp.c.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const bool f64 = sizeof(T) == 8;
        if (!make_row_tmap(&mab32, c.as_bar, sp.c.full_rows, f64, 32)) return VJP_ECUDA;
        if (!make_row_tmap(&mys32, c.ys, c.ys ? sp.c.full_rows : 0, f64, 32)) return VJP_ECUDA;
        if (cy.grid_ctas > 0) {
            // virtual ranks sharing one device: plain launch of a grid the caller
            // sized so that every rank's CTAs are resident together
            k<<<(unsigned)G, NTH, sm, c.stream>>>(ma, my, mab, mab32, mys32, sp);
            count_launch();
            return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
        }
        void *args[] = {&ma, &my, &mab, &mab32, &mys32, &sp};
        cudaError_t e = cudaLaunchCooperativeKernel((const void *)k, dim3((unsigned)G), dim3(NTH), args, sm, c.stream);
        count_launch();
        return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    static vjp_status cyc_finish(const ScanCall &c) {
        const vjp_cyclic &cy = *c.cyc;
        Layout L = layout(c.n);
        const bool fwd = need_fwd(c);
        const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
        const bool ys = c.ys != nullptr;
        if (fwd) {
            vjpk::ChunkParams p = cparams(c, L, 1);
            const int64_t nloc = cyc_nloc(cy, cy.rank);
            const int64_t nloc_max = cyc_nloc(cy, 0);
            vjpk::scan_cyc_tileprefix<Op, NTC><<<(unsigned)nloc, NTC, 0, c.stream>>>(
                p, (int32_t)cyc_tps(cy), cy.world, cy.rank, (int32_t)nloc_max, static_cast<const double *>(c.gathered));
            count_launch();
            if (cudaGetLastError() != cudaSuccess) return VJP_ECUDA;
        }
        if (std::is_same<Op, vjpk::OpAdd>::value && !ys)
            return acc ? cyc_launch<false, true, false>(c, L) : cyc_launch<false, false, false>(c, L);
        if (acc) return ys ? cyc_launch<true, true, true>(c, L) : cyc_launch<true, true, false>(c, L);
        return ys ? cyc_launch<true, false, true>(c, L) : cyc_launch<true, false, false>(c, L);
    }
    // tiles per superblock the sweep geometry of this device suggests (K = 4
    // tiles per CTA, the measured best round for scan(+), DESIGN 7.6)
    static int64_t cyc_default_sb_tiles() {
        return (int64_t)sm_count() * cyc_occupancy<!std::is_same<Op, vjpk::OpAdd>::value, false, false>() * 4;
    }

    // ---------------- one-read block look-back (world == 1; scan_blocklb.cuh) ----------------
    static bool use_lb(const ScanCall &c) {
        if (c.world != 1 || (c.flags & VJP_ACCUMULATE)) return false;  // ACCUMULATE: as_bar holds inputs
        if (c.flags & VJP_SCAN_BLOCKLB) return true;
        if (c.flags & (VJP_SCAN_LOOKBACK | VJP_SCAN_CHUNKED | VJP_SCAN_SWEEP)) return false;
        return false;  // opt-in until measured faster (DESIGN 7.1c)
    }
    // geometry of the block look-back: NTL = 128 rows (one per compute thread)
    // per tile, SL TMA stages; the forward pre-pass (K_F + tile prefix) runs on
    // the same tiles.  Variants (scan_tune().lb_variant): 0 = 3 stages, 1 = 2.
    static constexpr int NTL_MIN = 128;
    static int64_t ntiles_of(int64_t n, int nt) { return n > 0 ? (n + (int64_t)G::EPR * nt - 1) / ((int64_t)G::EPR * nt) : 0; }
    template <int NTL>
    static vjpk::ChunkParams lb_cparams(const ScanCall &c, const Layout &L, int nchunks) {
        vjpk::ChunkParams p = cparams(c, L, nchunks);
        p.ntiles = (int32_t)ntiles_of(c.n, NTL);
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        p.tileF = reinterpret_cast<double *>(ws + L.lbTileF);
        p.tileP = reinterpret_cast<double *>(ws + L.lbTileP);
        return p;
    }
    template <int NTL>
    static bool lb_maps(const ScanCall &c, int64_t rows, CUtensorMap *m_as, CUtensorMap *m_yb, CUtensorMap *m_ab,
                        CUtensorMap *m_ys) {
        const bool f64 = sizeof(T) == 8;
        bool ok = true;
        ok &= make_row_tmap(m_as, c.as, c.as ? rows : 0, f64, NTL);
        ok &= make_row_tmap(m_yb, c.ys_bar, rows, f64, NTL);
        ok &= make_row_tmap(m_ab, c.as_bar, c.as_bar ? rows : 0, f64, NTL);
        ok &= make_row_tmap(m_ys, c.ys, c.ys ? rows : 0, f64, NTL);
        return ok;
    }
    // K_F on NTL-row tiles: forward tile aggregates (tileF) + per-chunk records
    template <int NTL>
    static vjp_status lb_forward(const ScanCall &c, const Layout &L) {
        auto k = vjpk::scan_reduce<Op, T, NTL, SC, true, false>;
        const size_t sm = 1024 + (size_t)SC * NTL * vjpk::kRowBytes + sizeof(vjpk::ReduceSmem<Op, NTL, SC>);
        int occ = 0;
        set_smem(k, sm);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTL, sm) != cudaSuccess || occ < 1) occ = 1;
        int64_t g = (int64_t)sm_count() * occ;
        const int64_t nt = ntiles_of(c.n, NTL);
        if (g > kMaxChunks) g = kMaxChunks;
        if (g > nt) g = nt;
        vjpk::ChunkParams p = lb_cparams<NTL>(c, L, (int)(g < 1 ? 1 : g));
        CUtensorMap ma, my, mab, mys;
        if (!lb_maps<NTL>(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        k<<<(unsigned)p.nchunks, NTL, sm, c.stream>>>(ma, my, p);
        vjpk::scan_tile_prefix<Op, NTL><<<(unsigned)p.nchunks, NTL, 0, c.stream>>>(p);
        count_launch(2);
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    template <int NTL, int SL, bool FWD, bool YS, bool RS>
    static vjp_status launch_lb(const ScanCall &c, const Layout &L) {
        auto k = vjpk::scan_blocklb<Op, T, NTL, SL, FWD, YS, RS>;
        constexpr int NB = (FWD ? 1 : 0) + 1;
        constexpr int NTH = vjpk::kLbCompute + 32;  // 4 compute warps + the look-back warp
        const size_t sm = 1024 + (size_t)SL * NB * NTL * vjpk::kRowBytes + sizeof(vjpk::LbSmem<Op, NTL, SL>);
        set_smem(k, sm);
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTH, sm) != cudaSuccess || occ < 1) occ = 1;
        vjpk::LbParams P{};
        P.c = lb_cparams<NTL>(c, L, 1);
        const int64_t nt = P.c.ntiles;
        int64_t G = (int64_t)sm_count() * occ;
        // tiles per block: the blocks in flight (two per CTA, between their R
        // and A phases) hold ~2 * G * B * NB tiles in L2
        int64_t B = ((int64_t)scan_tune().lb_l2_mb << 20) / (2 * G * NB * NTL * vjpk::kRowBytes);
        if (B < 1) B = 1;
        if (B > vjpk::kLbBMax) B = vjpk::kLbBMax;
        if (B * G > nt) {  // small inputs: more, smaller blocks keep every CTA busy
            B = nt / G;
            if (B < 1) B = 1;
        }
        P.B = (int32_t)B;
        P.nblocks = (int32_t)((nt + B - 1) / B);
        unsigned char *ws = static_cast<unsigned char *>(c.ws);
        P.ticket = reinterpret_cast<uint32_t *>(ws + L.lbFlags);
        P.flags = reinterpret_cast<uint32_t *>(ws + L.lbFlags + 256);
        P.agg = reinterpret_cast<double *>(ws + L.lbAgg);
        P.inc = reinterpret_cast<double *>(ws + L.lbInc);
        P.tailpark = reinterpret_cast<double *>(ws + L.lbPark);
        P.trace = lb_trace_ptr();
        if (cudaMemsetAsync(ws + L.lbFlags, 0, 256 + (size_t)P.nblocks * 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        CUtensorMap ma, my, mab, mys;
        if (!lb_maps<NTL>(c, P.c.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const int64_t grid = G < P.nblocks ? G : P.nblocks;
        k<<<(unsigned)grid, NTH, sm, c.stream>>>(ma, my, mab, mys, P);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    template <int NTL, int SL>
    static vjp_status run_lb(const ScanCall &c, bool fwd_phase) {
        Layout L = layout(c.n);
        const bool fwd = need_fwd(c);
        if (fwd_phase) return fwd ? lb_forward<NTL>(c, L) : VJP_OK;
        const bool ys = c.ys != nullptr;
        constexpr bool RS = Op::kRevNeedsRs;
        if constexpr (std::is_same<Op, vjpk::OpAdd>::value) {
            if (!ys) return launch_lb<NTL, SL, false, false, false>(c, L);
        }
        return ys ? launch_lb<NTL, SL, true, true, RS>(c, L) : launch_lb<NTL, SL, true, false, RS>(c, L);
    }
    static vjp_status phase_lb(const ScanCall &c, bool fwd_phase) {
        switch (scan_tune().lb_variant) {
        case 1: return run_lb<128, 2>(c, fwd_phase);
        default: return run_lb<128, 3>(c, fwd_phase);
        }
    }

    // ---------------- general reduce rule, LINREC / MAT2 ----------------
    // vjp of y = reduce (.) e as equals the scan's return sweep seeded only at
    // the last element (scan-last == reduce): the chunked kernels run
    // with a VIRTUAL ys_bar (c.ys_bar -> the W scalars of y_bar at element
    // n-1, zero elsewhere; YL) — nothing of ys_bar is read from memory, so the
    // sweep moves `as` twice and writes as_bar once (MAT2 96 B/elem, against
    // the >= 5 accesses per element of the paper's two-scans-and-a-map).
    static vjp_status reduce_general(const ScanCall &c) {
        if constexpr (Op::kRevNeedsRs || std::is_same<Op, vjpk::OpAdd>::value) {
            return VJP_EUNSUPPORTED;
        } else {
            Layout L = layout(c.n);
            const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
            const int G = nchunks_for(L, true, acc);
            vjpk::ChunkParams p = cparams(c, L, G);
            p.ylast = c.ys_bar;
            p.ys_bar = nullptr;
            p.ys = nullptr;
            CUtensorMap ma, my, mab, mys;
            const bool f64 = sizeof(T) == 8;
            if (!make_row_tmap(&ma, c.as, p.full_rows, f64, NTC) || !make_row_tmap(&my, nullptr, 0, f64, NTC) ||
                !make_row_tmap(&mab, c.as_bar, p.full_rows, f64, NTC) || !make_row_tmap(&mys, nullptr, 0, f64, NTC))
                return VJP_ECUDA;
            auto kr = vjpk::scan_reduce<Op, T, NTC, SC, true, true, true>;
            const size_t smr = smem_r(1);
            set_smem(kr, smr);
            kr<<<(unsigned)p.nchunks, NTC, smr, c.stream>>>(ma, my, p);
            auto kc = acc ? vjpk::scan_apply<Op, T, NTC, SC, true, true, false, true>
                          : vjpk::scan_apply<Op, T, NTC, SC, true, false, false, true>;
            const size_t sma = smem_a(acc ? 3 : 2);
            set_smem(kc, sma);
            kc<<<(unsigned)p.nchunks, NTC, sma, c.stream>>>(ma, my, mab, mys, p);
            int launches = 2;
            if (c.ys) {  // the primal reduction: ordered combination of the chunk records
                vjpk::scan_chunks_total<Op, T, NTC><<<1, NTC, 0, c.stream>>>(p, static_cast<T *>(c.ys));
                ++launches;
            }
            count_launch(launches);
            return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
        }
    }

    // ---------------- chunked path for rs-dependent operators (MIN / MAX) ----------------
    // K_F (forward aggregates, reads as) -> scan_tile_prefix (tileP) -> K_R'
    // (reverse-map chunk records with the true rs, reads as + ys_bar) -> K_C (RS
    // variant).  Three streaming passes (f64: 8 + 16 + 24 B/elem) instead of the
    // latency-bound single-sweep look-back.  Single GPU.
    static bool use_rs_chunked(const ScanCall &c) {
        return Op::kRevNeedsRs && (c.world > 1 || !(c.flags & VJP_SCAN_LOOKBACK));
    }
    static vjp_status partial_rs(const ScanCall &c) {
        Layout L = layout(c.n);
        vjpk::ChunkParams p = cparams(c, L, nchunks_fwd(L));
        if (c.world > 1) {  // first exchange: the shard's forward aggregate
            p.partial = static_cast<double *>(c.partial);
            if (cudaMemsetAsync(p.counter, 0, 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        }
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        auto k = vjpk::scan_reduce<Op, T, NTC, SC, true, false>;
        size_t sm = smem_r(1);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    // tile prefixes (with the shard forward carry from `gathered` when world > 1)
    // and K_R' (-> chunk records; world > 1: the shard record for exchange 2)
    static vjp_status reverse_records_rs(const ScanCall &c, bool acc) {
        Layout L = layout(c.n);
        {
            vjpk::ChunkParams pf = cparams(c, L, nchunks_fwd(L));
            pf.gathered = static_cast<const double *>(c.gathered);
            vjpk::scan_tile_prefix<Op, NTC><<<(unsigned)pf.nchunks, NTC, 0, c.stream>>>(pf);
            count_launch();
        }
        const int G = nchunks_for(L, true, acc);
        vjpk::ChunkParams p = cparams(c, L, G);
        if (c.world > 1) {
            p.partial = static_cast<double *>(c.partial);
            if (cudaMemsetAsync(p.counter, 0, 4, c.stream) != cudaSuccess) return VJP_ECUDA;
        }
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        auto kr = vjpk::scan_reduce_rs<Op, T, NTC, SC>;
        const size_t smr = smem_r(2);
        set_smem(kr, smr);
        kr<<<(unsigned)p.nchunks, NTC, smr, c.stream>>>(ma, my, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    static vjp_status partial2(const ScanCall &c) {
        if constexpr (!Op::kRevNeedsRs) {
            return VJP_EUNSUPPORTED;  // one exchange suffices for these operators
        } else {
            return reverse_records_rs(c, (c.flags & VJP_ACCUMULATE) != 0);
        }
    }
    template <bool ACC, bool YS>
    static vjp_status launch_apply_rs(const ScanCall &c, const vjpk::ChunkParams &p, const CUtensorMap &ma,
                                      const CUtensorMap &my, const CUtensorMap &mab, const CUtensorMap &mys) {
        constexpr int NB = 2 + (ACC ? 1 : 0);
        auto k = vjpk::scan_apply<Op, T, NTC, SC, true, ACC, YS, false, true>;
        size_t sm = smem_a(NB);
        set_smem(k, sm);
        k<<<(unsigned)p.nchunks, NTC, sm, c.stream>>>(ma, my, mab, mys, p);
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    static vjp_status finish_rs(const ScanCall &c) {
        Layout L = layout(c.n);
        const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
        const bool ys = c.ys != nullptr;
        if (c.world == 1) {
            vjp_status st = reverse_records_rs(c, acc);
            if (st != VJP_OK) return st;
        }  // world > 1: done by vjp_scan_partial2 before the second exchange
        const int G = nchunks_for(L, true, acc);
        vjpk::ChunkParams p = cparams(c, L, G);
        CUtensorMap ma, my, mab, mys;
        if (!maps_c(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        if (acc) return ys ? launch_apply_rs<true, true>(c, p, ma, my, mab, mys)
                           : launch_apply_rs<true, false>(c, p, ma, my, mab, mys);
        return ys ? launch_apply_rs<false, true>(c, p, ma, my, mab, mys)
                  : launch_apply_rs<false, false>(c, p, ma, my, mab, mys);
    }

    // ---------------- MIN/MAX: K_F + one return pass with look-back (scan_ext1p.cuh) ----------------
    static bool use_ext1p(const ScanCall &c) {
        if constexpr (!Op::kRevNeedsRs) {
            return false;
        } else {
            if (c.world != 1 || c.ys || c.cyc) return false;
            return !(c.flags & (VJP_SCAN_LOOKBACK | VJP_SCAN_CHUNKED | VJP_ACCUMULATE));
        }
    }
    static vjp_status finish_ext1p(const ScanCall &c) {
        if constexpr (!Op::kRevNeedsRs) {
            return VJP_EUNSUPPORTED;
        } else {
            Layout L = layout(c.n);
            vjpk::ChunkParams pf = cparams(c, L, nchunks_fwd(L));
            vjpk::scan_tile_prefix<Op, NTC><<<(unsigned)pf.nchunks, NTC, 0, c.stream>>>(pf);
            unsigned char *ws = static_cast<unsigned char *>(c.ws);
            if (cudaMemsetAsync(ws + L.pxCtr, 0, L.pxEnd - L.pxCtr, c.stream) != cudaSuccess) return VJP_ECUDA;
            vjpk::Ext1pParams X{};
            X.r.n = c.n;
            X.r.ntiles = L.ntiles;
            X.r.ys_bar = c.ys_bar;
            X.r.as_bar = c.as_bar;
            X.r.ticket = reinterpret_cast<uint32_t *>(ws + L.pxCtr);
            X.r.gcount = reinterpret_cast<uint32_t *>(ws + L.pxCtr + 256);
            X.r.agg = reinterpret_cast<double2 *>(ws + L.pxAgg);
            X.r.inc = reinterpret_cast<double2 *>(ws + L.pxInc);
            X.r.grp = reinterpret_cast<double2 *>(ws + L.pxGrp);
            X.as = c.as;
            X.tileP = pf.tileP;
            X.global_first = c.global_offset == 0 ? 1 : 0;
            const int64_t rows = c.n * (int64_t)sizeof(T) / vjpk::kRowBytes;
            CUtensorMap ma, my, mo;
            const bool f64 = sizeof(T) == 8;
            if (!make_row_tmap(&ma, c.as, rows, f64, 256) || !make_row_tmap(&my, c.ys_bar, rows, f64, 256) ||
                !make_row_tmap(&mo, c.as_bar, rows, f64, 256))
                return VJP_ECUDA;
            constexpr size_t sm = 1024 + (size_t)2 * vjpk::k1pData * 128;
            auto k = vjpk::scan_ext_1p<Op, T>;
            set_smem(k, sm);
            k<<<(unsigned)L.ntiles, vjpk::k1pData + 32, sm, c.stream>>>(ma, my, mo, X);
            count_launch(2);
            return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
        }
    }

    static vjp_status partial(const ScanCall &c) {
        if (use_1p(c)) return VJP_OK;             // one pass, in finish
        if (use_ext1p(c)) return partial_rs(c);   // K_F: forward tile aggregates of `as`
        if (use_lb(c)) return phase_lb(c, true);  // the `as`-only forward pre-pass K_F (nothing for scan(+))
        if constexpr (Op::kRevNeedsRs) {
            if (use_rs_chunked(c)) return partial_rs(c);
        }
        if constexpr (!Op::kRevNeedsRs) {
            if (use_sweep(c)) return partial_sw(c);
            if (use_chunked(c)) return partial_c(c);
        }
        Layout L = layout(c.n);
        vjpk::ScanParams p = params(c, L);
        if (cudaMemsetAsync(c.ws, 0, L.memset_bytes, c.stream) != cudaSuccess) return VJP_ECUDA;
        CUtensorMap ma, my, mab, mys;
        if (!maps(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const bool fwd = need_fwd(c);
        if (c.world > 1) {
            if constexpr (std::is_same<Op, vjpk::OpAdd>::value) {
                if (!fwd) return launch_pass1<false, true>(c, p, ma, my);
            }
            if constexpr (!Op::kRevNeedsRs) return launch_pass1<true, true>(c, p, ma, my);
            return VJP_EUNSUPPORTED;
        }
        if (!fwd) return VJP_OK;  // ADD closed form: no forward sweep
        return launch_pass1<true, false>(c, p, ma, my);
    }

    static vjp_status finish(const ScanCall &c) {
        if (use_1p(c)) return launch_1p(c);
        if (use_ext1p(c)) return finish_ext1p(c);
        if (use_lb(c)) return phase_lb(c, false);
        if constexpr (Op::kRevNeedsRs) {
            if (use_rs_chunked(c)) return finish_rs(c);
        }
        if constexpr (!Op::kRevNeedsRs) {
            if (use_sweep(c)) return finish_sw(c);
            if (use_chunked(c)) return finish_c(c);
        }
        Layout L = layout(c.n);
        vjpk::ScanParams p = params(c, L);
        CUtensorMap ma, my, mab, mys;
        if (!maps(c, p.full_rows, &ma, &my, &mab, &mys)) return VJP_ECUDA;
        const bool acc = (c.flags & VJP_ACCUMULATE) != 0;
        const bool ys = c.ys != nullptr;
        if constexpr (std::is_same<Op, vjpk::OpAdd>::value) {
            if (!ys)
                return acc ? launch_pass2<false, true, false>(c, p, ma, my, mab, mys)
                           : launch_pass2<false, false, false>(c, p, ma, my, mab, mys);
        }
        if (acc) return ys ? launch_pass2<true, true, true>(c, p, ma, my, mab, mys)
                           : launch_pass2<true, true, false>(c, p, ma, my, mab, mys);
        return ys ? launch_pass2<true, false, true>(c, p, ma, my, mab, mys)
                  : launch_pass2<true, false, false>(c, p, ma, my, mab, mys);
    }
};

// carries of the multi-GPU finish, evaluated on the host (tests)
template <class Op>
void carries_host(const double *gathered, int rank, int world, double *fwd, double *rev) {
    typename Op::Val F, H;
    vjpk::shard_carries<Op>(gathered, rank, world, F, H);
    for (int k = 0; k < Op::W; ++k) {
        fwd[k] = F.x[k];
        rev[k] = H.x[k];
    }
}

template <class Op>
vjp_status scan_dispatch(int phase, const ScanCall &c, size_t *out) {
    if (phase == kScanPartialBytes) {
        *out = (size_t)(Op::W + Op::kMapD) * 8;
        return VJP_OK;
    }
    if (phase == kScanIdentity) {  // an empty shard's record: neutral element, identity map
        vjpk::scan_identity_record<Op><<<1, 32, 0, c.stream>>>(static_cast<double *>(c.partial));
        count_launch();
        return cudaGetLastError() == cudaSuccess ? VJP_OK : VJP_ECUDA;
    }
    if (phase == kCycSbTiles) {
        if constexpr (Op::kRevNeedsRs) {
            *out = 0;
            return VJP_EUNSUPPORTED;
        } else {
            *out = (size_t)(c.dtype == VJP_F64 ? ScanImpl<Op, double>::cyc_default_sb_tiles()
                                               : ScanImpl<Op, float>::cyc_default_sb_tiles()) *
                   (size_t)(c.dtype == VJP_F64 ? ScanImpl<Op, double>::TILE_C : ScanImpl<Op, float>::TILE_C);
            return VJP_OK;
        }
    }
    if (phase == kCycForward || phase == kCycFinish) {
        if constexpr (Op::kRevNeedsRs) {
            return VJP_EUNSUPPORTED;  // MIN/MAX: reverse maps depend on the forward carry (two exchanges)
        } else {
            if (c.dtype == VJP_F64)
                return phase == kCycForward ? ScanImpl<Op, double>::cyc_forward(c) : ScanImpl<Op, double>::cyc_finish(c);
            return phase == kCycForward ? ScanImpl<Op, float>::cyc_forward(c) : ScanImpl<Op, float>::cyc_finish(c);
        }
    }
    if (c.dtype == VJP_F64) {
        using I = ScanImpl<Op, double>;
        if (phase == kScanWs) { *out = I::layout(c.n).total; return VJP_OK; }
        if (phase == kReduceGeneral) return I::reduce_general(c);
        if (phase == kScanPartial2) return I::partial2(c);
        return phase == kScanPartial ? I::partial(c) : I::finish(c);
    }
    using I = ScanImpl<Op, float>;
    if (phase == kScanWs) { *out = I::layout(c.n).total; return VJP_OK; }
    if (phase == kReduceGeneral) return I::reduce_general(c);
    if (phase == kScanPartial2) return I::partial2(c);
    return phase == kScanPartial ? I::partial(c) : I::finish(c);
}

vjp_status scan_dispatch_add(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_mul(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_min(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_max(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_linrec(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_mat2(int, const ScanCall &, size_t *);

// general reduce rule for LINREC / MAT2 (reduce.cu routes vjp_reduce here)
size_t reduce_general_ws(vjp_op op, vjp_dtype dtype, int64_t n);
vjp_status reduce_general(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                          void *y, void *ws, size_t ws_bytes, cudaStream_t stream, unsigned flags);

}  // namespace vjph
