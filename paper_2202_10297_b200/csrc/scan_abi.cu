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

// tuning hook: per-block timestamps of the block look-back (DEVICE buffer of
// 8 u64 per block, zeroed by the caller; nullptr turns it off)
vjp_status vjp_debug_lb_trace(unsigned long long *buf) {
    vjph::lb_trace_ptr() = buf;
    return VJP_OK;
}

}  // extern "C"
