// scan_abi.cu — extern "C" vjp_scan* entry points (include/vjp.h):
// argument validation, then dispatch to the per-operator drivers.
#include "scan_impl.cuh"

namespace {
using namespace vjph;

typedef vjp_status (*Disp)(int, const ScanCall &, size_t *);

Disp disp_for(vjp_op op) {
    switch (op) {
    case VJP_ADD: return scan_dispatch_add;
    case VJP_MUL: return scan_dispatch_mul;
    case VJP_MIN: return scan_dispatch_min;
    case VJP_MAX: return scan_dispatch_max;
    case VJP_LINREC: return scan_dispatch_linrec;
    case VJP_MAT2: return scan_dispatch_mat2;
    }
    return nullptr;
}

bool dtype_ok(vjp_dtype d) { return d == VJP_F32 || d == VJP_F64; }

bool shard_ok(const vjp_shard *s, int64_t n) {
    if (!s) return true;
    return s->world >= 1 && s->rank >= 0 && s->rank < s->world && s->global_offset >= 0 &&
           s->global_n >= s->global_offset + n;
}

ScanCall make_call(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *ys_bar, void *as_bar,
                   void *ys, void *ws, size_t ws_bytes, vjp_stream_t stream, unsigned flags,
                   const vjp_shard *shard) {
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    c.n = n;
    c.as = as;
    c.ys_bar = ys_bar;
    c.as_bar = as_bar;
    c.ys = ys;
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = reinterpret_cast<cudaStream_t>(stream);
    c.flags = flags;
    c.rank = shard ? shard->rank : 0;
    c.world = shard ? shard->world : 1;
    c.global_offset = shard ? shard->global_offset : 0;
    return c;
}

// common checks; `need_out` = as_bar required (finish / full call)
vjp_status check(const ScanCall &c, bool need_out) {
    if (!disp_for(c.op) || !dtype_ok(c.dtype) || c.n < 0) return VJP_EINVAL;
    if (c.n == 0) return VJP_OK;
    if (!c.ys_bar) return VJP_EINVAL;
    if (need_out && !c.as_bar) return VJP_EINVAL;
    if (!c.as && (c.op != VJP_ADD || c.ys)) return VJP_EINVAL;
    const void *ptrs[4] = {c.as, c.ys_bar, c.as_bar, c.ys};
    for (const void *p : ptrs)
        if (p && !aligned16(p)) return VJP_EALIGN;
    if (need_out && (c.as_bar == c.ys_bar || (c.as && c.as_bar == c.as))) return VJP_EINVAL;
    size_t need = 0;
    disp_for(c.op)(kScanWs, c, &need);
    if (c.ws_bytes < need || (need && !c.ws)) return VJP_EWORKSPACE;
    if (!aligned16(c.ws)) return VJP_EALIGN;
    // tile count must fit the kernels' 32-bit tile ids
    if (c.n / 1024 > (int64_t)1 << 30) return VJP_EINVAL;
    return VJP_OK;
}
}  // namespace

namespace vjph {
size_t reduce_general_ws(vjp_op op, vjp_dtype dtype, int64_t n) {
    Disp d = disp_for(op);
    if (!d || (op != VJP_LINREC && op != VJP_MAT2) || !dtype_ok(dtype) || n < 0) return 0;
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    c.n = n;
    size_t out = 0;
    d(kScanWs, c, &out);
    return out;
}
vjp_status reduce_general(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *y_bar, void *as_bar,
                          void *y, void *ws, size_t ws_bytes, cudaStream_t stream, unsigned flags) {
    if ((op != VJP_LINREC && op != VJP_MAT2) || !dtype_ok(dtype) || n < 0) return VJP_EINVAL;
    if (n == 0) return VJP_OK;
    if (!as || !y_bar || !as_bar) return VJP_EINVAL;
    const void *ptrs[3] = {as, as_bar, y};
    for (const void *p : ptrs)
        if (p && !aligned16(p)) return VJP_EALIGN;
    if (as_bar == as) return VJP_EINVAL;
    if (ws_bytes < reduce_general_ws(op, dtype, n) || !ws) return VJP_EWORKSPACE;
    if (!aligned16(ws)) return VJP_EALIGN;
    if (n / 1024 > (int64_t)1 << 30) return VJP_EINVAL;
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    c.n = n;
    c.as = as;
    c.ys_bar = y_bar;  // the W scalars of the reduce's output adjoint
    c.as_bar = as_bar;
    c.ys = y;          // the primal reduction (nullable)
    c.ws = ws;
    c.ws_bytes = ws_bytes;
    c.stream = stream;
    c.flags = flags;
    c.world = 1;
    return disp_for(op)(kReduceGeneral, c, nullptr);
}
}  // namespace vjph

namespace vjph {
unsigned long long *&lb_trace_ptr() {
    static unsigned long long *p = nullptr;
    return p;
}
}  // namespace vjph

extern "C" {

size_t vjp_scan_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n) {
    Disp d = disp_for(op);
    if (!d || !dtype_ok(dtype) || n < 0) return 0;
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    c.n = n;
    size_t out = 0;
    d(kScanWs, c, &out);
    return out;
}

size_t vjp_scan_partial_bytes(vjp_op op, vjp_dtype dtype) {
    Disp d = disp_for(op);
    if (!d || !dtype_ok(dtype)) return 0;
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    size_t out = 0;
    d(kScanPartialBytes, c, &out);
    return out;
}

vjp_status vjp_scan(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *ys_bar, void *as_bar,
                    void *ys, void *ws, size_t ws_bytes, vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_scan");
    ScanCall c = make_call(op, dtype, n, as, ys_bar, as_bar, ys, ws, ws_bytes, stream, flags, nullptr);
    vjp_status s = check(c, true);
    if (s != VJP_OK || n == 0) return s;
    Disp d = disp_for(op);
    s = d(kScanPartial, c, nullptr);
    if (s != VJP_OK) return s;
    return d(kScanFinish, c, nullptr);
}

vjp_status vjp_scan_partial(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *ys_bar, void *ws,
                            size_t ws_bytes, const vjp_shard *shard, void *partial, vjp_stream_t stream,
                            unsigned flags) {
    VJP_NVTX("vjp_scan_partial");
    if (!shard_ok(shard, n)) return VJP_EINVAL;
    ScanCall c = make_call(op, dtype, n, as, ys_bar, nullptr, nullptr, ws, ws_bytes, stream, flags, shard);
    c.partial = partial;
    vjp_status s = check(c, false);
    if (s != VJP_OK) return s;
    if (partial && !aligned16(partial)) return VJP_EALIGN;
    if (n == 0) {
        // empty shard (global_n < world, or an uneven split): identity record
        // (neutral forward element, identity map); nothing else to do
        if (!partial) return VJP_OK;
        return disp_for(op)(kScanIdentity, c, nullptr);
    }
    return disp_for(op)(kScanPartial, c, nullptr);
}

vjp_status vjp_scan_partial2(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *ys_bar, void *ws,
                             size_t ws_bytes, const vjp_shard *shard, const void *gathered1, void *partial2,
                             vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_scan_partial2");
    if (op != VJP_MIN && op != VJP_MAX) return VJP_EUNSUPPORTED;
    if (!shard_ok(shard, n) || !shard || shard->world < 2) return VJP_EINVAL;
    ScanCall c = make_call(op, dtype, n, as, ys_bar, nullptr, nullptr, ws, ws_bytes, stream, flags, shard);
    c.partial = partial2;
    c.gathered = gathered1;
    vjp_status s = check(c, false);
    if (s != VJP_OK) return s;
    if (!partial2 || !aligned16(partial2) || !gathered1 || !aligned16(gathered1)) return VJP_EINVAL;
    if (n == 0) return disp_for(op)(kScanIdentity, c, nullptr);  // empty shard: identity record
    return disp_for(op)(kScanPartial2, c, nullptr);
}

vjp_status vjp_scan_finish(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, const void *ys_bar, void *as_bar,
                           void *ys, void *ws, size_t ws_bytes, const vjp_shard *shard, const void *gathered,
                           vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_scan_finish");
    if (!shard_ok(shard, n)) return VJP_EINVAL;
    ScanCall c = make_call(op, dtype, n, as, ys_bar, as_bar, ys, ws, ws_bytes, stream, flags, shard);
    c.gathered = gathered;
    vjp_status s = check(c, true);
    if (s != VJP_OK || n == 0) return s;
    if (c.world > 1 && (!gathered || !aligned16(gathered))) return VJP_EINVAL;
    return disp_for(op)(kScanFinish, c, nullptr);
}

vjp_status vjp_scan_carries_host(vjp_op op, vjp_dtype dtype, int32_t rank, int32_t world, const void *gathered,
                                 double *fwd_carry, double *rev_carry) {
    if (!dtype_ok(dtype) || world < 1 || rank < 0 || rank >= world || !gathered || !fwd_carry || !rev_carry)
        return VJP_EINVAL;
    const double *g = static_cast<const double *>(gathered);
    switch (op) {
    case VJP_ADD: carries_host<vjpk::OpAdd>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    case VJP_MUL: carries_host<vjpk::OpMul>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    case VJP_LINREC: carries_host<vjpk::OpLinrec>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    case VJP_MAT2: carries_host<vjpk::OpMat2>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    // MIN/MAX (two exchanges): call with the first gathered array for the
    // forward carry and with the second one for the reverse carry
    case VJP_MIN: carries_host<vjpk::OpMin>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    case VJP_MAX: carries_host<vjpk::OpMax>(g, rank, world, fwd_carry, rev_carry); return VJP_OK;
    }
    return VJP_EINVAL;
}

// ---------------- block-cyclic multi-GPU vjp_scan ----------------
// geometry of the descriptor (what the size queries need)
static bool cyc_geo_ok(vjp_op op, vjp_dtype dtype, const vjp_cyclic *cy) {
    if (!cy || !dtype_ok(dtype) || !disp_for(op)) return false;
    if (cy->world < 1 || cy->world > VJP_CYCLIC_MAX_RANKS || cy->rank < 0 || cy->rank >= cy->world) return false;
    if (cy->global_n < 0 || cy->sb_elems <= 0 || cy->grid_ctas < 0) return false;
    const int64_t te = vjp_scan_cyclic_tile_elems(op, dtype);
    return te > 0 && cy->sb_elems % te == 0;
}
// ... plus what a call needs
static bool cyc_ok(vjp_op op, vjp_dtype dtype, const vjp_cyclic *cy) {
    if (!cyc_geo_ok(op, dtype, cy)) return false;
    if (cy->epoch == 0 || cy->epoch >= (1u << 30)) return false;
    for (int q = 0; q < cy->world; ++q)
        if (!cy->status[q] || !aligned16(cy->status[q])) return false;
    return true;
}

int64_t vjp_scan_cyclic_tile_elems(vjp_op op, vjp_dtype dtype) {
    if (!dtype_ok(dtype) || !disp_for(op)) return 0;
    const int w = op == VJP_LINREC ? 2 : (op == VJP_MAT2 ? 4 : 1);
    const int es = w * (dtype == VJP_F64 ? 8 : 4);
    return (int64_t)(vjpk::kRowBytes / es) * 128;  // one 128-row TMA tile of the chunked / sweep kernels
}

int64_t vjp_scan_cyclic_sb_elems(vjp_op op, vjp_dtype dtype) {
    Disp d = disp_for(op);
    if (!d || !dtype_ok(dtype)) return 0;
    ScanCall c{};
    c.op = op;
    c.dtype = dtype;
    size_t out = 0;
    if (d(kCycSbTiles, c, &out) != VJP_OK) return 0;
    return (int64_t)out;
}

int64_t vjp_scan_cyclic_local_n(const vjp_cyclic *cy) {
    if (!cy || cy->world < 1 || cy->rank < 0 || cy->rank >= cy->world || cy->sb_elems <= 0 || cy->global_n < 0)
        return -1;
    const int64_t nsb = (cy->global_n + cy->sb_elems - 1) / cy->sb_elems;
    int64_t n = 0;
    for (int64_t J = cy->rank; J < nsb; J += cy->world) {
        const int64_t e = (J + 1) * cy->sb_elems < cy->global_n ? (J + 1) * cy->sb_elems : cy->global_n;
        n += e - J * cy->sb_elems;
    }
    return n;
}

size_t vjp_scan_cyclic_status_bytes(vjp_op op, int64_t global_n, int64_t sb_elems) {
    if (!disp_for(op) || global_n < 0 || sb_elems <= 0) return 0;
    const int64_t nsb = (global_n + sb_elems - 1) / sb_elems;
    const int w = op == VJP_LINREC ? 2 : (op == VJP_MAT2 ? 4 : 1);
    const int md = op == VJP_MAT2 ? 8 : (op == VJP_LINREC ? 3 : (op == VJP_MUL ? 2 : 1));
    (void)w;
    return 256 + align256((size_t)nsb * 4) + align256((size_t)nsb * md * 8);
}

size_t vjp_scan_cyclic_fwd_bytes(vjp_op op, vjp_dtype dtype, const vjp_cyclic *cy) {
    if (!cyc_geo_ok(op, dtype, cy)) return 0;
    const int w = op == VJP_LINREC ? 2 : (op == VJP_MAT2 ? 4 : 1);
    const int64_t nsb = (cy->global_n + cy->sb_elems - 1) / cy->sb_elems;
    const int64_t nloc_max = nsb > 0 ? (nsb - 1) / cy->world + 1 : 0;
    return (size_t)(nloc_max > 0 ? nloc_max : 1) * w * 8;
}

vjp_status vjp_scan_cyclic_forward(vjp_op op, vjp_dtype dtype, int64_t n_local, const void *as, void *ws,
                                   size_t ws_bytes, const vjp_cyclic *cy, void *sbagg, vjp_stream_t stream) {
    VJP_NVTX("vjp_scan_cyclic_forward");
    if (!cyc_ok(op, dtype, cy)) return VJP_EINVAL;
    if (op == VJP_MIN || op == VJP_MAX) return VJP_EUNSUPPORTED;
    if (n_local != vjp_scan_cyclic_local_n(cy)) return VJP_EINVAL;
    if (op == VJP_ADD || n_local == 0) return VJP_OK;  // closed form / nothing owned: no forward pass
    if (!as || !sbagg || !aligned16(as) || !aligned16(sbagg)) return VJP_EINVAL;
    ScanCall c = make_call(op, dtype, n_local, as, as, nullptr, nullptr, ws, ws_bytes, stream, 0, nullptr);
    c.cyc = cy;
    c.partial = sbagg;
    size_t need = 0;
    disp_for(op)(kScanWs, c, &need);
    if (ws_bytes < need || !ws || !aligned16(ws)) return VJP_EWORKSPACE;
    return disp_for(op)(kCycForward, c, nullptr);
}

vjp_status vjp_scan_cyclic(vjp_op op, vjp_dtype dtype, int64_t n_local, const void *as, const void *ys_bar,
                           void *as_bar, void *ws, size_t ws_bytes, const vjp_cyclic *cy, const void *gathered,
                           vjp_stream_t stream, unsigned flags) {
    VJP_NVTX("vjp_scan_cyclic");
    if (!cyc_ok(op, dtype, cy)) return VJP_EINVAL;
    if (op == VJP_MIN || op == VJP_MAX) return VJP_EUNSUPPORTED;
    if (n_local != vjp_scan_cyclic_local_n(cy)) return VJP_EINVAL;
    if (flags & ~(unsigned)VJP_ACCUMULATE) return VJP_EINVAL;
    ScanCall c = make_call(op, dtype, n_local, as, ys_bar, as_bar, nullptr, ws, ws_bytes, stream, flags, nullptr);
    c.cyc = cy;
    c.gathered = gathered;
    c.world = 1;  // the chunked shard logic is not used: the sweep's look-back does the exchange
    if (n_local == 0) return VJP_OK;  // (a rank owning no superblock publishes nothing: no SB waits on it)
    vjp_status s = check(c, true);
    if (s != VJP_OK) return s;
    if (op != VJP_ADD && (!gathered || !aligned16(gathered))) return VJP_EINVAL;
    return disp_for(op)(kCycFinish, c, nullptr);
}

// tuning hook: per-block timestamps of the block look-back (DEVICE buffer of
// 8 u64 per block, zeroed by the caller; nullptr turns it off)
vjp_status vjp_debug_lb_trace(unsigned long long *buf) {
    vjph::lb_trace_ptr() = buf;
    return VJP_OK;
}

}  // extern "C"
