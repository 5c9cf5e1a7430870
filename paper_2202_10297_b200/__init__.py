"""paper_2202_10297_b200 — B200 (sm_100a) vjp return sweeps of scan, reduce,
reduce_by_index and scatter (arXiv 2202.10297, sec 5).

Thin Python binding over the C ABI of ``_lib/libvjp_b200.so``
(``include/vjp.h``): argument marshalling only — every step of the path runs in
the library's CUDA kernels.  PyTorch supplies device memory, streams and (in
``dist``) process groups.  There is no CPU fallback: if the library is missing
or the tensors are not on a CUDA device the calls raise.

Host (CPU) tensors are accepted for the end-to-end path: they are copied to the
current CUDA device, the call runs there, and the results are copied back.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libvjp_b200.so")

F32, F64 = 1, 2
I32, I64 = 1, 2
ADD, MUL, MIN, MAX, LINREC, MAT2 = 1, 2, 3, 4, 5, 6
OPS = {"add": ADD, "mul": MUL, "min": MIN, "max": MAX, "linrec": LINREC, "mat2": MAT2}
WIDTH = {ADD: 1, MUL: 1, MIN: 1, MAX: 1, LINREC: 2, MAT2: 4}
ACCUMULATE = 1
CHECK_INDICES = 2
SCAN_LOOKBACK = 1 << 16
SCAN_SWEEP = 1 << 17
SCAN_CHUNKED = 1 << 18
SCAN_BLOCKLB = 1 << 19
STATUS = {0: "VJP_OK", 1: "VJP_EINVAL", 2: "VJP_EUNSUPPORTED", 3: "VJP_EWORKSPACE", 4: "VJP_ECUDA",
          5: "VJP_EDUPINDEX", 6: "VJP_EOOB", 7: "VJP_EALIGN"}

_lib = None


class VjpError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = lib().vjp_status_string(code).decode()
        super().__init__(f"{where}: {msg}")


class VjpShard(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("global_offset", ctypes.c_int64),
                ("global_n", ctypes.c_int64)]


CYCLIC_MAX_RANKS = 8


class VjpCyclic(ctypes.Structure):
    """vjp_cyclic (include/vjp.h): block-cyclic multi-GPU scan descriptor."""
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("global_n", ctypes.c_int64),
                ("sb_elems", ctypes.c_int64), ("epoch", ctypes.c_uint32), ("grid_ctas", ctypes.c_int32),
                ("status", ctypes.c_void_p * CYCLIC_MAX_RANKS)]


def lib():
    """Load libvjp_b200.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2202_10297_b200._build)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, sz, u32, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_uint, ctypes.c_int
        sp = ctypes.POINTER(VjpShard)
        cy = ctypes.POINTER(VjpCyclic)
        sig = {
            "vjp_status_string": ([ci], ctypes.c_char_p),
            "vjp_launch_count": ([], ctypes.c_uint64),
            "vjp_scan_workspace_bytes": ([ci, ci, i64], sz),
            "vjp_scan": ([ci, ci, i64, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_scan_partial_bytes": ([ci, ci], sz),
            "vjp_scan_partial": ([ci, ci, i64, vp, vp, vp, sz, sp, vp, vp, u32], ci),
            "vjp_scan_finish": ([ci, ci, i64, vp, vp, vp, vp, vp, sz, sp, vp, vp, u32], ci),
            "vjp_scan_partial2": ([ci, ci, i64, vp, vp, vp, sz, sp, vp, vp, vp, u32], ci),
            "vjp_scan_carries_host": ([ci, ci, ctypes.c_int32, ctypes.c_int32, vp, vp, vp], ci),
            "vjp_reduce_workspace_bytes": ([ci, ci, i64], sz),
            "vjp_reduce": ([ci, ci, i64, vp, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_reduce_partial_bytes": ([], sz),
            "vjp_reduce_partial": ([ci, ci, i64, vp, vp, sz, sp, vp, vp], ci),
            "vjp_reduce_finish": ([ci, ci, i64, vp, vp, vp, vp, vp, vp, sz, sp, vp, vp, u32], ci),
            "vjp_reduce_by_index_workspace_bytes": ([ci, ci, i64, i64, i64], sz),
            "vjp_reduce_by_index_hs_workspace_bytes": ([ci, ci, i64, i64, i64], sz),
            "vjp_reduce_by_index": ([ci, ci, ci, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_reduce_by_index_partial": ([ci, ci, ci, i64, i64, vp, vp, vp, sz, sp, vp, vp, vp], ci),
            "vjp_reduce_by_index_select": ([ci, i64, vp, vp, vp, vp], ci),
            "vjp_reduce_by_index_finish": ([ci, ci, ci, i64, i64, vp, vp, vp, vp, vp, vp, vp, sz, sp, vp, u32], ci),
            "vjp_scatter_workspace_bytes": ([ci, i64, i64], sz),
            "vjp_scatter": ([ci, ci, i64, i64, i64, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_reduce_by_index_general_workspace_bytes": ([ci, ci, i64, i64], sz),
            "vjp_reduce_by_index_general": ([ci, ci, ci, i64, i64, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_scatter_shard": ([ci, ci, i64, i64, i64, vp, vp, vp, vp, sp, vp], ci),
            "vjp_scatter_forward": ([ci, ci, i64, i64, i64, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_scatter_restore": ([ci, ci, i64, i64, i64, vp, vp, vp, vp], ci),
            "vjp_kmeans_workspace_bytes": ([ci, i64, i64, i64], sz),
            "vjp_scan_batched_workspace_bytes": ([ci, ci, i64, i64], sz),
            "vjp_debug_mul_code": ([vp, vp, i64, vp], ci),
            "vjp_scan_batched": ([ci, ci, i64, i64, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_kmeans": ([ci, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, u32], ci),
            "vjp_calib_out_len": ([], i64),
            "vjp_calib_l2_gather": ([vp, vp, i64, vp, i64, vp], ci),
            "vjp_calib_l2_red": ([vp, vp, i64, vp], ci),
            "vjp_scan_cyclic_tile_elems": ([ci, ci], i64),
            "vjp_scan_cyclic_sb_elems": ([ci, ci], i64),
            "vjp_scan_cyclic_local_n": ([cy], i64),
            "vjp_scan_cyclic_status_bytes": ([ci, i64, i64], sz),
            "vjp_scan_cyclic_fwd_bytes": ([ci, ci, cy], sz),
            "vjp_scan_cyclic_forward": ([ci, ci, i64, vp, vp, sz, cy, vp, vp], ci),
            "vjp_scan_cyclic": ([ci, ci, i64, vp, vp, vp, vp, sz, cy, vp, vp, u32], ci),
        }
        for name, (args, res) in sig.items():
            if not hasattr(L, name):
                continue  # reported by tests/test_abi_cpu.py::test_exports
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def launch_count() -> int:
    """Kernels launched by the library in this process (bench gpu_launches)."""
    return int(lib().vjp_launch_count())


# ----------------------------------------------------------------- helpers

def _op(op) -> int:
    o = OPS[op] if isinstance(op, str) else int(op)
    if o not in WIDTH:
        raise ValueError(f"unknown operator {op!r}")
    return o


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.float64:
        return F64
    raise TypeError(f"vjp: value tensors must be float32/float64, got {t.dtype}")


def _it(t: torch.Tensor) -> int:
    if t.dtype == torch.int32:
        return I32
    if t.dtype == torch.int64:
        return I64
    raise TypeError(f"vjp: index tensors must be int32/int64, got {t.dtype}")


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check(code: int, where: str):
    if code != 0:
        raise VjpError(code, where)


def _dev_of(*ts):
    for t in ts:
        if t is not None and t.is_cuda:
            return t.device
    if not torch.cuda.is_available():
        raise RuntimeError("vjp: no CUDA device (this library has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _to(t, dev):
    if t is None:
        return None
    if t.is_cuda:
        return t.contiguous()
    src = t.contiguous()
    if not src.is_pinned():
        src = src.pin_memory()
    return src.to(dev, non_blocking=True)


def _check_out(out, numel: int, dtype, dev, what: str = "out"):
    """the kernels write numel * sizeof(dtype) bytes through out's data pointer:
    refuse anything that is not exactly that (size, dtype, device, layout)."""
    if out.numel() != numel:
        raise ValueError(f"vjp: {what} has {out.numel()} elements, expected {numel}")
    if out.dtype != dtype:
        raise TypeError(f"vjp: {what} is {out.dtype}, expected {dtype}")
    if out.is_cuda and out.device != torch.device(dev):
        raise ValueError(f"vjp: {what} is on {out.device}, the call runs on {dev}")
    if not out.is_contiguous():
        raise ValueError(f"vjp: {what} must be contiguous")


def _out_buf(out, like, dev, accumulate):
    """device buffer for an output: `out` itself if on the device; for a host
    `out`, a device temporary (pre-loaded only when accumulating).  With
    accumulate=True the caller must pass the adjoint to add into."""
    if out is None:
        if accumulate:
            raise ValueError("vjp: accumulate=True adds into `out`: pass the existing adjoint")
        return torch.empty_like(like, device=dev)
    _check_out(out, like.numel(), like.dtype, dev)
    if out.is_cuda:
        return out
    return _to(out, dev) if accumulate else torch.empty(out.shape, dtype=out.dtype, device=dev)


def workspace(nbytes: int, dev) -> torch.Tensor | None:
    if nbytes == 0:
        return None
    return torch.empty(nbytes, dtype=torch.uint8, device=dev)


def _host_out(t: torch.Tensor, like_host: bool):
    if not like_host:
        return t
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out


# ------------------------------------------------- asynchronous host path
_XSTREAMS: dict = {}


def _xstreams(dev):
    """(copy-in, compute, copy-out) streams of a device for the async host path"""
    k = str(dev)
    if k not in _XSTREAMS:
        _XSTREAMS[k] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _XSTREAMS[k]


class Pending:
    """an in-flight asynchronous host-buffer call; .wait() returns its output"""

    def __init__(self, done: torch.cuda.Event, out: torch.Tensor, keep):
        self.done, self.out, self._keep = done, out, keep

    def wait(self) -> torch.Tensor:
        self.done.synchronize()
        self._keep = None
        return self.out


def _scan_host_async(o: int, ys_bar: torch.Tensor, as_, out, accumulate: bool) -> Pending:
    if out is None or out.is_cuda or not out.is_pinned() or not ys_bar.is_pinned() or \
            (as_ is not None and not as_.is_pinned()):
        raise ValueError("scan(sync=False): pinned host ys_bar / as_ / out are required")
    if accumulate:
        raise ValueError("scan(sync=False): accumulate is not supported on the host path")
    dev = torch.device("cuda", torch.cuda.current_device())
    _check_out(out, ys_bar.numel(), ys_bar.dtype, dev)
    w = WIDTH[o]
    n = ys_bar.numel() // w
    s_in, s_c, s_out = _xstreams(dev)
    s_in.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s_in):
        yb = ys_bar.to(dev, non_blocking=True)
        a = None if as_ is None else as_.to(dev, non_blocking=True)
    s_c.wait_stream(s_in)
    L = lib()
    with torch.cuda.stream(s_c):
        ab = torch.empty_like(yb)
        ws = workspace(L.vjp_scan_workspace_bytes(o, _dt(yb), n), dev)
        _check(L.vjp_scan(o, _dt(yb), n, _p(a), _p(yb), _p(ab), None, _p(ws), 0 if ws is None else ws.numel(),
                          ctypes.c_void_p(s_c.cuda_stream), 0), "vjp_scan")
    s_out.wait_stream(s_c)
    with torch.cuda.stream(s_out):
        out.copy_(ab, non_blocking=True)
        done = torch.cuda.Event()
        done.record(s_out)
    # keep the device buffers alive until the copy-out has run (tensors were
    # allocated on s_in / s_c and are used on later streams)
    for t in (yb, a, ab, ws):
        if t is not None:
            t.record_stream(s_out)
    return Pending(done, out, (yb, a, ab, ws))


# ----------------------------------------------------------------- calls

def scan(op, ys_bar: torch.Tensor, as_: torch.Tensor | None = None, *, out: torch.Tensor | None = None,
         want_ys: bool = False, accumulate: bool = False, lookback: bool = False, sweep: bool = False, chunked: bool = False,
         blocklb: bool = False, sync: bool = True):
    """as_bar of ``ys = scan op as_`` with output adjoint ``ys_bar`` (sec 5.2).

    Tensors hold n elements of the operator's width (LINREC: (d, c) pairs,
    MAT2: row-major 2x2), any shape with that many scalars.  Returns as_bar
    (same shape as ys_bar), or (as_bar, ys) if want_ys.  lookback=True selects
    the single-sweep decoupled look-back kernels, sweep=True the one-read
    L2-round sweep, chunked=True the two chunked kernels, blocklb=True the
    one-read block look-back (tuning/testing; the default on one GPU is the
    chunked pair, and the L2-round sweep for f64 scan(+) without ys).

    HOST tensors (the end-to-end path): inputs are copied to the device, the
    result back.  With ``sync=False`` and a pinned host ``out`` the call
    returns a Pending at once: its host->device copies, kernels and
    device->host copy run on three per-device streams (copy-in, compute,
    copy-out) ordered by events, so consecutive calls overlap one call's
    copy-out with the next one's copy-in (PCIe is full duplex) and the
    kernels; ``Pending.wait()`` (or torch.cuda.synchronize()) completes it."""
    o = _op(op)
    if not sync and not ys_bar.is_cuda:
        return _scan_host_async(o, ys_bar, as_, out, accumulate)
    host = not ys_bar.is_cuda
    dev = _dev_of(ys_bar, as_, out)
    yb = _to(ys_bar, dev)
    a = _to(as_, dev)
    w = WIDTH[o]
    if yb.numel() % w:
        raise ValueError(f"ys_bar has {yb.numel()} scalars, not a multiple of width {w}")
    n = yb.numel() // w
    if a is not None and (a.numel() != yb.numel() or a.dtype != yb.dtype):
        raise ValueError("as_ must match ys_bar in size and dtype")
    ab = _out_buf(out, yb, dev, accumulate)
    ys = torch.empty_like(yb) if want_ys else None
    L = lib()
    ws = workspace(L.vjp_scan_workspace_bytes(o, _dt(yb), n), dev)
    _check(L.vjp_scan(o, _dt(yb), n, _p(a), _p(yb), _p(ab), _p(ys), _p(ws),
                      0 if ws is None else ws.numel(), _stream(dev),
                      (ACCUMULATE if accumulate else 0) | (SCAN_LOOKBACK if lookback else 0)
                      | (SCAN_SWEEP if sweep else 0) | (SCAN_CHUNKED if chunked else 0)
                      | (SCAN_BLOCKLB if blocklb else 0)),
           "vjp_scan")
    if out is not None and not out.is_cuda:
        out.copy_(ab, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        ab = out
    else:
        ab = _host_out(ab, host)
    if want_ys:
        return ab, _host_out(ys, host)
    return ab


def reduce(op, as_: torch.Tensor, y_bar, *, out: torch.Tensor | None = None, want_y: bool = False,
           accumulate: bool = False):
    """as_bar of ``y = reduce op as_`` (sec 5.1).  y_bar: python float or a
    tensor of one element (W scalars for LINREC / MAT2, whose vjp is the
    paper's general rule).  Returns as_bar, or (as_bar, y, arg) if
    want_y (arg = argmin/argmax for MIN/MAX, first zero index or -1 for MUL,
    -1 for ADD / LINREC / MAT2)."""
    o = _op(op)
    w = WIDTH[o]
    host = not as_.is_cuda
    dev = _dev_of(as_, out)
    a = _to(as_, dev)
    if a.numel() % w:
        raise ValueError(f"as_ has {a.numel()} scalars, not a multiple of width {w}")
    n = a.numel() // w
    if isinstance(y_bar, torch.Tensor):
        yb = _to(y_bar.reshape(-1).to(a.dtype), dev)
    else:
        yb = torch.tensor([float(v) for v in (y_bar if hasattr(y_bar, "__len__") else [y_bar])],
                          dtype=a.dtype).to(dev)
    if yb.numel() != w:
        raise ValueError(f"y_bar must hold {w} scalars")
    ab = _out_buf(out, a, dev, accumulate)
    y = torch.empty(w, dtype=a.dtype, device=dev) if want_y else None
    arg = torch.empty(1, dtype=torch.int64, device=dev) if want_y else None
    L = lib()
    ws = workspace(L.vjp_reduce_workspace_bytes(o, _dt(a), n), dev)
    _check(L.vjp_reduce(o, _dt(a), n, _p(a), _p(yb), _p(ab), _p(y), _p(arg), _p(ws),
                        0 if ws is None else ws.numel(), _stream(dev), ACCUMULATE if accumulate else 0),
           "vjp_reduce")
    if out is not None and not out.is_cuda:
        out.copy_(ab, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        ab = out
    else:
        ab = _host_out(ab, host)
    if want_y:
        return ab, _host_out(y, host), _host_out(arg, host)
    return ab


def reduce_by_index(op, inds: torch.Tensor, as_: torch.Tensor | None, hs_bar: torch.Tensor, *,
                    out: torch.Tensor | None = None, want_hs: bool = False, accumulate: bool = False,
                    general: bool = False, width: int = 1):
    """as_bar of ``hs = reduce_by_index op m inds as_`` with m = len(hs_bar) / width
    (sec 5.1.2).  Returns as_bar, or (as_bar, hs, winners) if want_hs
    (winners: MIN/MAX per-bin winner index, -1 for an empty bin; MUL: zero count).
    width > 1: vectorised operator, as_ is [n x width] and
    hs_bar [m x width] (flat or 2-D), rules per component (reading A24).
    general=True (MUL, width 1): the paper's general rule, counting sort +
    per-bin exclusive product scans (vjp_reduce_by_index_general)."""
    o = _op(op)
    host = not inds.is_cuda
    dev = _dev_of(inds, as_, hs_bar, out)
    ix = _to(inds, dev)
    a = _to(as_, dev)
    hb = _to(hs_bar, dev)
    if width < 1 or hb.numel() % width:
        raise ValueError("width must be >= 1 and divide hs_bar's size")
    n, m = ix.numel(), hb.numel() // width
    if a is not None and (a.dtype != hb.dtype or a.numel() != n * width):
        raise ValueError("as_ must have len(inds) * width elements of hs_bar's dtype")
    ab = _out_buf(out, torch.empty(n * width, dtype=hb.dtype, device=dev), dev, accumulate)
    hs = torch.empty(m * width, dtype=hb.dtype, device=dev) if want_hs else None
    win = torch.empty(m * width, dtype=torch.int64, device=dev) if want_hs else None
    L = lib()
    if general:
        if width != 1:
            raise ValueError("general=True supports width 1")
        if want_hs:
            raise ValueError("general=True returns the adjoint only")
        ws = workspace(L.vjp_reduce_by_index_general_workspace_bytes(o, _dt(hb), n, m), dev)
        _check(L.vjp_reduce_by_index_general(o, _dt(hb), _it(ix), n, m, _p(ix), _p(a), _p(hb), _p(ab), _p(ws),
                                             0 if ws is None else ws.numel(), _stream(dev),
                                             ACCUMULATE if accumulate else 0), "vjp_reduce_by_index_general")
        if out is not None and not out.is_cuda:
            out.copy_(ab, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            return out
        return _host_out(ab, host)
    wsq = L.vjp_reduce_by_index_hs_workspace_bytes if want_hs else L.vjp_reduce_by_index_workspace_bytes
    ws = workspace(wsq(o, _dt(hb), n, m, width), dev)
    _check(L.vjp_reduce_by_index(o, _dt(hb), _it(ix), n, m, width, _p(ix), _p(a), _p(hb), _p(ab), _p(hs), _p(win),
                                 _p(ws), 0 if ws is None else ws.numel(), _stream(dev),
                                 ACCUMULATE if accumulate else 0),
           "vjp_reduce_by_index")
    if out is not None and not out.is_cuda:
        out.copy_(ab, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        ab = out
    else:
        ab = _host_out(ab, host)
    if want_hs:
        return ab, _host_out(hs, host), _host_out(win, host)
    return ab


def scatter(is_: torch.Tensor, ys_bar: torch.Tensor, *, width: int = 1, in_place: bool = False,
            vs_out: torch.Tensor | None = None, accumulate: bool = False, check: bool = False):
    """Adjoints of ``ys = scatter xs is vs`` (sec 5.3): returns (xs_bar, vs_bar).
    in_place=True reuses ys_bar's storage for xs_bar (O(m) work)."""
    host = not ys_bar.is_cuda
    dev = _dev_of(is_, ys_bar, vs_out)
    ix = _to(is_, dev)
    yb = _to(ys_bar, dev)
    if in_place and host:
        raise ValueError("in_place scatter needs device tensors")
    n, m = yb.numel() // width, ix.numel()
    xb = yb if in_place else torch.empty_like(yb)
    if vs_out is not None:
        _check_out(vs_out, m * width, yb.dtype, dev, "vs_out")
    elif accumulate:
        raise ValueError("vjp: accumulate=True adds into `vs_out`: pass the existing adjoint")
    vb = _to(vs_out, dev) if vs_out is not None else torch.empty(m * width, dtype=yb.dtype, device=dev)
    flags = (ACCUMULATE if accumulate else 0) | (CHECK_INDICES if check else 0)
    L = lib()
    ws = workspace(L.vjp_scatter_workspace_bytes(_dt(yb), n, m), dev) if check else None
    _check(L.vjp_scatter(_dt(yb), _it(ix), n, m, width, _p(ix), _p(yb), _p(xb), _p(vb), _p(ws),
                         0 if ws is None else ws.numel(), _stream(dev), flags), "vjp_scatter")
    return _host_out(xb, host), _host_out(vb, host)


def scatter_forward(xs: torch.Tensor, is_: torch.Tensor, vs: torch.Tensor, *, width: int = 1,
                    saved_out: torch.Tensor | None = None, check: bool = False) -> torch.Tensor:
    """Forward sweep of the in-place ``let xs = scatter xs is vs``:
    returns xs_saved = gather xs is and updates the DEVICE tensor xs in place
    (it becomes ys).  O(m)."""
    if not xs.is_cuda:
        raise ValueError("scatter_forward updates xs in place: it must be a device tensor")
    dev = xs.device
    ix, v = _to(is_, dev), _to(vs, dev)
    n, m = xs.numel() // width, ix.numel()
    if v.numel() != m * width or v.dtype != xs.dtype:
        raise ValueError("vs must be [m x width] of xs's dtype")
    if saved_out is not None:
        _check_out(saved_out, m * width, xs.dtype, dev, "saved_out")
    saved = saved_out if saved_out is not None else torch.empty(m * width, dtype=xs.dtype, device=dev)
    L = lib()
    ws = workspace(L.vjp_scatter_workspace_bytes(_dt(xs), n, m), dev) if check else None
    _check(L.vjp_scatter_forward(_dt(xs), _it(ix), n, m, width, _p(ix), _p(v), _p(xs), _p(saved), _p(ws),
                                 0 if ws is None else ws.numel(), _stream(dev), CHECK_INDICES if check else 0),
           "vjp_scatter_forward")
    return saved


def scatter_restore(ys: torch.Tensor, is_: torch.Tensor, xs_saved: torch.Tensor, *, width: int = 1) -> torch.Tensor:
    """Return sweep step (3): ``xs = scatter ys is xs_saved`` on the
    DEVICE tensor ys, in place; returns it.  O(m)."""
    if not ys.is_cuda:
        raise ValueError("scatter_restore updates ys in place: it must be a device tensor")
    dev = ys.device
    ix, sv = _to(is_, dev), _to(xs_saved, dev)
    n, m = ys.numel() // width, ix.numel()
    if sv.numel() != m * width or sv.dtype != ys.dtype:
        raise ValueError("xs_saved must be [m x width] of ys's dtype")
    _check(lib().vjp_scatter_restore(_dt(ys), _it(ix), n, m, width, _p(ix), _p(sv), _p(ys), _stream(dev)),
           "vjp_scatter_restore")
    return ys


def kmeans(points: torch.Tensor, centers: torch.Tensor, cost_bar=1.0, *, hess: bool = True,
           accumulate: bool = False, out: dict | None = None):
    """Composite k-means gradient (BASELINE config 5;
    P:1663-1720): for f(C) = sum_p min_j ||p - c_j||^2, returns a dict with
    ``cbar`` (vjp of f at C with cost_bar), ``hdiag`` (jvp of that vjp in the
    all-ones direction = the Hessian diagonal 2 cost_bar cnt_j; if hess),
    ``assign`` (int32 first-index argmin per point), ``counts`` (int64 [k]) and
    ``cost`` (0-d tensor).  points [n x d], centers [k x d], f32 or f64 (the
    arithmetic is f64).  ``out`` may hold preallocated device tensors under the
    same keys (accumulate adds into cbar / hdiag / counts / cost)."""
    dev = _dev_of(points, centers)
    P = _to(points, dev)
    C = _to(centers, dev)
    if P.dim() != 2 or C.dim() != 2 or P.shape[1] != C.shape[1] or P.dtype != C.dtype:
        raise ValueError("kmeans: points [n x d] and centers [k x d] of one dtype")
    n, d = P.shape
    k = C.shape[0]
    if not torch.is_tensor(cost_bar):
        cost_bar = torch.tensor([float(cost_bar)], dtype=C.dtype)
    yb = _to(cost_bar.reshape(1).to(C.dtype), dev)
    o = dict(out or {})
    cbar = o.get("cbar")
    if cbar is None:
        cbar = torch.empty_like(C) if not accumulate else torch.zeros_like(C)
    hd = o.get("hdiag")
    if hess and hd is None:
        hd = torch.empty_like(C) if not accumulate else torch.zeros_like(C)
    asg = o.get("assign")
    if asg is None or asg.numel() != n:
        asg = torch.empty(n, dtype=torch.int32, device=dev)
    for key, t, numel in (("cbar", cbar, k * d), ("hdiag", hd, k * d), ("counts", o.get("counts"), k)):
        if t is not None and t.numel() != numel:
            raise ValueError(f"kmeans: out[{key!r}] has {t.numel()} elements, expected {numel}")
    cnt = o.get("counts")
    if cnt is None:
        cnt = torch.zeros(k, dtype=torch.int64, device=dev)
    cost = o.get("cost")
    if cost is None:
        cost = torch.zeros((), dtype=C.dtype, device=dev)
    L = lib()
    ws = workspace(L.vjp_kmeans_workspace_bytes(_dt(C), n, k, d), dev)
    _check(L.vjp_kmeans(_dt(C), n, k, d, _p(P), _p(C), _p(yb), _p(cbar), _p(hd), _p(asg), _p(cnt), _p(cost),
                        _p(ws), 0 if ws is None else ws.numel(), _stream(dev), ACCUMULATE if accumulate else 0),
           "vjp_kmeans")
    return {"cbar": cbar, "hdiag": hd, "assign": asg, "counts": cnt, "cost": cost}


def scan_batched(op, ys_bar: torch.Tensor, as_: torch.Tensor | None = None, *, width: int,
                 out: torch.Tensor | None = None, accumulate: bool = False):
    """as_bar of the VECTORISED scan ys = scan (map op) e as_:
    `width` independent scans along the leading dimension, element i component
    j at [i][j] (op width W scalars each).  Tensors hold n * width * W scalars."""
    o = _op(op)
    host = not ys_bar.is_cuda
    dev = _dev_of(ys_bar, as_, out)
    yb = _to(ys_bar, dev)
    a = _to(as_, dev)
    w = WIDTH[o]
    if yb.numel() % (w * width):
        raise ValueError(f"ys_bar has {yb.numel()} scalars, not a multiple of width*{w}")
    n = yb.numel() // (w * width)
    if a is not None and (a.numel() != yb.numel() or a.dtype != yb.dtype):
        raise ValueError("as_ must match ys_bar in size and dtype")
    ab = _out_buf(out, yb, dev, accumulate)
    L = lib()
    ws = workspace(L.vjp_scan_batched_workspace_bytes(o, _dt(yb), n, width), dev)
    _check(L.vjp_scan_batched(o, _dt(yb), n, width, _p(a), _p(yb), _p(ab), _p(ws), 0 if ws is None else ws.numel(),
                              _stream(dev), ACCUMULATE if accumulate else 0), "vjp_scan_batched")
    if out is not None and not out.is_cuda:
        out.copy_(ab, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return out
    return _host_out(ab, host)
