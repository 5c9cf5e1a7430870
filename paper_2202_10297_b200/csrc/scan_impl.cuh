// scan_impl.cuh — host driver of the vjp_scan kernels (validation is done by
// the C-ABI layer in scan_abi.cu; this file owns workspace layout and launches).
#pragma once

#include <mutex>
#include <type_traits>

#include "scan_kernels.cuh"

namespace vjph {

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
};

enum ScanPhase { kScanWs = 0, kScanPartial = 1, kScanFinish = 2, kScanPartialBytes = 3 };

template <class Op, class T>
struct ScanImpl {
    using G = vjpk::Geo<Op, T>;
    static constexpr int W = Op::W;
    static constexpr int MD = Op::kMapD;
    static constexpr int R1MAX = W + MD;

    struct Layout {
        int64_t ntiles;
        size_t counters, flags1, flags2, memset_bytes, p1agg, p1inc, p2agg, p2inc, partial, total;
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

    static bool need_fwd(const ScanCall &c) {
        return !std::is_same<Op, vjpk::OpAdd>::value || c.ys != nullptr;
    }

    static vjp_status partial(const ScanCall &c) {
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
    if (c.dtype == VJP_F64) {
        using I = ScanImpl<Op, double>;
        if (phase == kScanWs) { *out = I::layout(c.n).total; return VJP_OK; }
        return phase == kScanPartial ? I::partial(c) : I::finish(c);
    }
    using I = ScanImpl<Op, float>;
    if (phase == kScanWs) { *out = I::layout(c.n).total; return VJP_OK; }
    return phase == kScanPartial ? I::partial(c) : I::finish(c);
}

vjp_status scan_dispatch_add(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_mul(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_min(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_max(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_linrec(int, const ScanCall &, size_t *);
vjp_status scan_dispatch_mat2(int, const ScanCall &, size_t *);

}  // namespace vjph
