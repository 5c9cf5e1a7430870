// scan_ext1p.cuh — vjp of scan(min) / scan(max) (pick-left subgradient,
// reading R3) as a forward pre-pass + ONE return pass with the two-level
// decoupled look-back of scan_add1p.cuh.
//
// With rs the primal running extremum, the per-element reverse map is
// X -> jl_i (ybar_i + X), jl_i = [rs_{i-1} wins against a_i] in {0, 1}
// (scan_ops.cuh OpExt): the carry accumulates ybar leftwards and is reset at
// every "record" (jl = 0, a_i strictly better than everything left of it),
// where as_bar_i takes the accumulated sum (P:1143-1158 with the min/max
// Jacobians).  A tile's composed map is (D, C) with C in {0, 1} (C = no record
// in the tile), so a look-back record is {flag, D} — one 16-byte store, the
// flag carrying C (1: AGG with C = 0, 3: AGG with C = 1, 2: INCL) — and the
// composition along the look-back is a SUM of D's up to the nearest
// terminator: an INCL record or a tile (group) with a record (C = 0), whose D
// is then exact.
//
// Pre-pass (scan_impl.cuh): K_F over `as` (forward tile aggregates) and
// scan_tile_prefix -> the running extremum entering every 128-row tile.  The
// return pass reads `as` and ys_bar once (TMA, 32 KB each per tile of 256
// rows, 128B swizzle), writes as_bar once: 8 + 24 B/elem f64 moved for 24 B of
// method bytes (round 1's chunked path: 8 + 16 + 24).
#pragma once

#include "scan_add1p.cuh"
#include "scan_ops.cuh"

namespace vjpk {

struct Ext1pParams {
    Add1pParams r;          // records / tickets (as in scan_add1p) + n, ntiles, ys_bar, as_bar
    const void *as;
    const double *tileP;    // [128-row K_F tiles]: running extremum entering each (K_F + scan_tile_prefix)
    int32_t global_first;   // this array holds global element 0 (kFirstSpecial)
    int32_t pad;
};

__device__ __forceinline__ double ext_flag(bool C) { return C ? 3.0 : 1.0; }

// X_k = the carry entering ticket k from the right: sum of the D's of the
// tickets below k up to the nearest terminator (INCL, or a tile / group with
// C = 0), plus the terminator's value.  Level 1 reads the 97..128 tickets
// below k directly; level 2 walks whole groups.
__device__ __forceinline__ double ext1p_lookback(const Add1pParams &P, int64_t k, int lane) {
    const int64_t G0 = k >= 97 ? (k - 97) >> 5 : 0;
    const int D = (int)(k - (G0 << 5));
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
    // level 1: a terminator is an INCL record or an AGG with C = 0; records not
    // yet published are polled until the nearest terminator is known
    int dstar = 0;
    for (;;) {
        int best = 0;
#pragma unroll
        for (int m = k1pM - 1; m >= 0; --m) {
            const int d = lane + 1 + 32 * m;
            const bool term = d <= D && (q[m].x == 2.0 || a[m].x == 1.0);
            const unsigned mk = __ballot_sync(0xffffffffu, term);
            if (mk) best = 32 * m + __ffs(mk);
        }
        // every ticket nearer than the best terminator must have its AGG in
        bool missing = false;
#pragma unroll
        for (int m = 0; m < k1pM; ++m) {
            const int d = lane + 1 + 32 * m;
            if (d <= D && (best == 0 || d <= best) && q[m].x == 0.0 && a[m].x == 0.0) missing = true;
        }
        if (!__any_sync(0xffffffffu, missing)) {
            dstar = best;
            break;
        }
#pragma unroll
        for (int m = 0; m < k1pM; ++m) {
            const int d = lane + 1 + 32 * m;
            if (d <= D && (best == 0 || d <= best) && q[m].x == 0.0 && a[m].x == 0.0) {
                q[m] = ld_rec16(P.inc + (k - d));
                if (k - d != 0) a[m] = ld_rec16(P.agg + (k - d));
            }
        }
    }
    double x = 0.0;
#pragma unroll
    for (int m = 0; m < k1pM; ++m) {
        const int d = lane + 1 + 32 * m;
        if (d > D || (dstar && d > dstar)) continue;
        if (dstar && d == dstar) x += (q[m].x == 2.0) ? q[m].y : a[m].y;  // INCL value, or the record tile's D
        else x += (q[m].x == 2.0) ? q[m].y : a[m].y;                       // C = 1 maps: their D (an INCL nearer
                                                                            // than dstar would be the terminator)
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (dstar || G0 == 0) return x;
    double sum = x;
    for (int64_t gb = G0 - 1; gb >= 0; gb -= 32) {
        const int64_t gl = gb - lane;
        double2 q2 = make_double2(0.0, 0.0), r2 = make_double2(0.0, 0.0);
        if (gl >= 0) {
            q2 = ld_rec16(P.inc + (gl << 5) + 31);
            r2 = ld_rec16(P.grp + gl);
        }
        int lim;
        for (;;) {
            const unsigned tm = __ballot_sync(0xffffffffu, gl >= 0 && (q2.x == 2.0 || r2.x == 1.0));
            lim = tm ? __ffs(tm) - 1 : 32;
            const bool missing = gl >= 0 && lane <= lim && q2.x == 0.0 && r2.x == 0.0;
            if (!__any_sync(0xffffffffu, missing)) break;
            if (missing) {
                q2 = ld_rec16(P.inc + (gl << 5) + 31);
                r2 = ld_rec16(P.grp + gl);
            }
        }
        double y = 0.0;
        if (gl >= 0 && lane <= lim) y = (q2.x == 2.0) ? q2.y : r2.y;
#pragma unroll
        for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        sum += y;
        if (lim < 32) break;
    }
    return sum;
}

// (D, C) maps: o after i (i applied first)
struct ExtMap {
    double D;
    bool C;
};
__device__ __forceinline__ ExtMap ext_compose(const ExtMap &o, const ExtMap &i) {
    return {o.D + (o.C ? i.D : 0.0), o.C && i.C};
}

template <class Op, class T>
__global__ void __launch_bounds__(k1pData + 32, 3) scan_ext_1p(const __grid_constant__ CUtensorMap tm_as,
                                                             const __grid_constant__ CUtensorMap tm_yb,
                                                             const __grid_constant__ CUtensorMap tm_out,
                                                             const Ext1pParams X) {
    constexpr int E = 128 / (int)sizeof(T);
    constexpr int NW = k1pData / 32;
    constexpr int TB = k1pData * 128;  // one row per thread: 32 KB per array
    constexpr int TE = TB / (int)sizeof(T);
    constexpr int EPC = 16 / (int)sizeof(T);
    const Add1pParams &P = X.r;
    extern __shared__ __align__(1024) unsigned char s_raw[];
    unsigned char *sA = smem_align1024(s_raw);
    unsigned char *sY = sA + TB;
    __shared__ int64_t s_tick;
    __shared__ double s_f[NW];     // warp forward aggregates
    __shared__ ExtMap s_m[NW];     // warp map aggregates
    __shared__ double s_excl;
    __shared__ uint64_t s_bar;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        const int64_t k0 = (int64_t)atomicAdd(P.ticket, 1u);
        s_tick = k0;
        mbar_init(&s_bar, 1);
        fence_mbar_init();
        const int64_t tile0 = P.ntiles - 1 - k0;
        if ((tile0 + 1) * (int64_t)TE <= P.n) {
            mbar_arrive_expect_tx(&s_bar, 2 * TB);
            tma_load_2d(sA, &tm_as, &s_bar, 0, (int)(tile0 * 256));
            tma_load_2d(sY, &tm_yb, &s_bar, 0, (int)(tile0 * 256));
        } else {
            mbar_arrive(&s_bar);
        }
    }
    __syncthreads();
    const int64_t k = s_tick;
    if (warp == NW) {
        // ---------------- look-back warp
        const double ex = k > 0 ? ext1p_lookback(P, k, lane) : 0.0;
        if (lane == 0) s_excl = ex;
        bar_named(1, k1pData + 32);
        if (lane == 0 && k > 0) {
            // INCL = M_tile(ex): the tile map from the warp aggregates
            ExtMap Mt = {0.0, true};
            for (int w = NW - 1; w >= 0; --w) Mt = ext_compose(s_m[w], Mt);  // warp 7 (rightmost) applied first
            st_rec16(P.inc + k, 2.0, Mt.D + (Mt.C ? ex : 0.0));
        }
        return;
    }
    // ---------------- data warps: thread t owns row t (E elements)
    const int64_t tile = P.ntiles - 1 - k;
    const bool full = (tile + 1) * (int64_t)TE <= P.n;
    const int64_t te0 = tile * (int64_t)TE;
    if (!full) {  // partial rightmost tile: padding as = neutral element, ybar = 0 (no effect)
        const T *ga = static_cast<const T *>(X.as);
        const T *gy = static_cast<const T *>(P.ys_bar);
        const T neutral = (T)Op::fwd_id().x[0];
        for (int e = t; e < TE; e += k1pData) {
            const int r = e / E, q = e % E;
            const bool in = te0 + e < P.n;
            *(reinterpret_cast<T *>(sA + swz(r, q / EPC)) + q % EPC) = in ? ga[te0 + e] : neutral;
            *(reinterpret_cast<T *>(sY + swz(r, q / EPC)) + q % EPC) = in ? gy[te0 + e] : (T)0;
        }
        bar_named(2, k1pData);
    }
    mbar_wait(&s_bar, 0);
    // 1. forward: the row's extremum, the block's exclusive scan over rows,
    //    then the pick-left bits jl (bit q: rs_{q-1} wins against a_q)
    uint32_t jl = 0;
    {
        T av[E];
#pragma unroll
        for (int c = 0; c < 8; ++c) unpack16(*reinterpret_cast<const double2 *>(sA + swz(t, c)), av + c * EPC);
        double f = Op::fwd_id().x[0];
#pragma unroll
        for (int q = 0; q < E; ++q) f = Op::left(f, (double)av[q]) ? f : (double)av[q];
        double inc = f;  // ordered inclusive scan over the lanes (left = lower lane)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc = Op::left(u, inc) ? u : inc;
        }
        if (lane == 31) s_f[warp] = inc;
        bar_named(2, k1pData);
        double rs = X.tileP[2 * tile];  // entering the tile (K_F tiles are 128 rows)
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if (w < warp) rs = Op::left(rs, s_f[w]) ? rs : s_f[w];
        const double ex = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane > 0) rs = Op::left(rs, ex) ? rs : ex;
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const bool l = Op::left(rs, (double)av[q]);
            jl |= (l ? 1u : 0u) << q;
            rs = l ? rs : (double)av[q];
        }
    }
    // 2. the row's reverse map, the warp's inclusive suffix of maps, the tile map
    T yv[E];
#pragma unroll
    for (int c = 0; c < 8; ++c) unpack16(*reinterpret_cast<const double2 *>(sY + swz(t, c)), yv + c * EPC);
    ExtMap m = {0.0, true};
#pragma unroll
    for (int q = E - 1; q >= 0; --q) m = ((jl >> q) & 1u) ? ExtMap{(double)yv[q] + m.D, m.C} : ExtMap{0.0, false};
    ExtMap sfx = m;  // M_lane o M_{lane+1} o ... o M_31
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        ExtMap u;
        u.D = __shfl_down_sync(0xffffffffu, sfx.D, o);
        u.C = __shfl_down_sync(0xffffffffu, (int)sfx.C, o) != 0;
        if (lane + o < 32) sfx = ext_compose(sfx, u);
    }
    if (lane == 0) s_m[warp] = sfx;
    bar_named(2, k1pData);
    if (warp == 0) {
        ExtMap Mt = {0.0, true};
        for (int w = NW - 1; w >= 0; --w) Mt = ext_compose(s_m[w], Mt);
        uint32_t arrived = 0;
        const int64_t g = k >> 5;
        if (lane == 0) {
            if (k == 0) st_rec16(P.inc, 2.0, Mt.D);  // the rightmost tile: its carry out is M(0)
            else st_rec16(P.agg + k, ext_flag(Mt.C), Mt.D);
            arrived = atom_add_release_gpu(P.gcount + g, 1u) + 1u;
        }
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        if (arrived == 32u) {
            // the group's map M_{32g+31} o ... o M_{32g} (ticket 0: its INCL is a constant map)
            fence_acq_rel_gpu();
            const int64_t j = (g << 5) + lane;
            double2 rr;
            ExtMap x;
            if (j == 0) {
                do { rr = ld_rec16(P.inc); } while (rr.x == 0.0);
                x = {rr.y, false};
            } else {
                do { rr = ld_rec16(P.agg + j); } while (rr.x == 0.0);
                x = {rr.y, rr.x == 3.0};
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                ExtMap u;
                u.D = __shfl_down_sync(0xffffffffu, x.D, o);
                u.C = __shfl_down_sync(0xffffffffu, (int)x.C, o) != 0;
                if (lane + o < 32) x = ext_compose(u, x);  // higher tickets lie to the left: applied later
            }
            if (lane == 0) st_rec16(P.grp + g, ext_flag(x.C), x.D);
        }
    }
    bar_named(1, k1pData + 32);
    // 3. outputs: the carry entering this row = (maps right of it in the tile)(X_k)
    double H = s_excl;
#pragma unroll
    for (int w = NW - 1; w >= 0; --w)
        if (w > warp) H = s_m[w].D + (s_m[w].C ? H : 0.0);
    {
        ExtMap r;  // lanes to the right within the warp: exclusive suffix
        r.D = __shfl_down_sync(0xffffffffu, sfx.D, 1);
        r.C = __shfl_down_sync(0xffffffffu, (int)sfx.C, 1) != 0;
        if (lane < 31) H = r.D + (r.C ? H : 0.0);
    }
    const int64_t re0 = te0 + (int64_t)t * E;
#pragma unroll
    for (int q = E - 1; q >= 0; --q) {
        const double gq = (double)yv[q] + H;
        const bool l = (jl >> q) & 1u;
        double o = l ? 0.0 : gq;
        if (X.global_first && re0 + q == 0) o = gq;  // as_bar_0 = rbar_0
        H = l ? gq : 0.0;
        yv[q] = (T)o;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) *reinterpret_cast<double2 *>(sY + swz(t, c)) = pack16(yv + c * EPC);
    if (full) {
        fence_proxy_async_smem();
        bar_named(2, k1pData);
        if (t == 0) {
            tma_store_2d(&tm_out, sY, 0, (int)(tile * 256));
            tma_store_commit();
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    } else {
        bar_named(2, k1pData);
        T *dst = static_cast<T *>(P.as_bar);
        for (int e = t; e < TE; e += k1pData) {
            const int r = e / E, q = e % E;
            if (te0 + e < P.n) dst[te0 + e] = *(reinterpret_cast<const T *>(sY + swz(r, q / EPC)) + q % EPC);
        }
    }
}

}  // namespace vjpk
