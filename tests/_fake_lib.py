"""CPU stand-in for the multi-GPU kernel entry points of libvjp_b200.so, so
that world-size-2 gloo tests can drive paper_2202_10297_b200.dist.* itself (its
sequencing, buffers, dtype views and collectives) without a GPU.

TEST INFRASTRUCTURE ONLY.  Each fake implements the entry point's documented
contract (include/vjp.h) on host pointers; per-shard states come from the
oracle (plain CPU definitions) where one exists, the MUL exchange code from
its definition in vjp.h: code(a) = round(log2|a| 2^51) + [a < 0] 2^63 mod 2^64."""
from __future__ import annotations

import ctypes
import math

import numpy as np

import oracle

I64MAX = np.iinfo(np.int64).max
_DT = {1: np.float32, 2: np.float64}
_IT = {1: np.int32, 2: np.int64}
_OPN = {1: "add", 2: "mul", 3: "min", 4: "max"}


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    ptr = ptr.value if isinstance(ptr, ctypes.c_void_p) else ptr
    return np.ctypeslib.as_array((np.ctypeslib.as_ctypes_type(np.dtype(dtype)) * n).from_address(ptr))


def _code(a: float) -> int:
    q = round(math.log2(abs(a)) * (1 << 51))
    return (q + ((1 << 63) if a < 0 else 0)) & ((1 << 64) - 1)


def _decode(t: int) -> float:
    L = t & ((1 << 63) - 1)
    if L >= 1 << 62:
        L -= 1 << 63
    neg = ((t - L) >> 63) & 1
    v = 2.0 ** (L / float(1 << 51))
    return -v if neg else v


class FakeLib:
    def vjp_reduce_by_index_workspace_bytes(self, o, dt, n, m, w):
        return 0

    def vjp_reduce_by_index_partial(self, o, dt, it, n, m, inds, as_, ws, nb, sh, bin_val, bin_aux, s):
        sh = sh._obj if hasattr(sh, "_obj") else sh
        ix = _arr(inds, n, _IT[it])
        a = _arr(as_, n, _DT[dt])
        bv = _arr(bin_val, m, np.float64)
        ba = _arr(bin_aux, m, np.int64)
        if o == 2:
            codes = np.zeros(m, dtype=np.uint64)
            z = np.zeros(m, dtype=np.int64)
            for b, x in zip(ix, a):
                if 0 <= b < m:
                    if x == 0:
                        z[b] += 1
                    else:
                        codes[b] = np.uint64((int(codes[b]) + _code(float(x))) & ((1 << 64) - 1))
            bv.view(np.uint64)[:] = codes
            ba[:] = z
        else:
            _, hs, win, _ = oracle.vjp_reduce_by_index(_OPN[o], ix, a, np.zeros(m, _DT[dt]))
            bv[:] = np.where(win >= 0, hs, np.inf if o == 3 else -np.inf)
            ba[:] = np.where(win >= 0, win + sh.global_offset, I64MAX)
        return 0

    def vjp_reduce_by_index_select(self, o, m, gval, lval, aux, s):
        g, l, x = _arr(gval, m, np.float64), _arr(lval, m, np.float64), _arr(aux, m, np.int64)
        x[~(l == g)] = I64MAX
        return 0

    def vjp_reduce_by_index_finish(self, o, dt, it, n, m, inds, as_, hs_bar, as_bar, bin_val, bin_aux, ws, nb, sh,
                                   s, flags):
        sh = sh._obj if hasattr(sh, "_obj") else sh
        ix = _arr(inds, n, _IT[it])
        hb = _arr(hs_bar, m, _DT[dt])
        ab = _arr(as_bar, n, _DT[dt])
        if o == 1:
            ab[:] = [hb[b] if 0 <= b < m else 0 for b in ix]
            return 0
        aux = _arr(bin_aux, m, np.int64)
        if o == 2:
            a = _arr(as_, n, _DT[dt])
            codes = _arr(bin_val, m, np.float64).view(np.uint64)
            for i, (b, x) in enumerate(zip(ix, a)):
                v = 0.0
                if 0 <= b < m:
                    p = _decode(int(codes[b]))
                    if aux[b] == 0:
                        v = hb[b] * p / x
                    elif aux[b] == 1 and x == 0:
                        v = hb[b] * p
                ab[i] = v
            return 0
        for i, b in enumerate(ix):
            ab[i] = hb[b] if (0 <= b < m and aux[b] == sh.global_offset + i) else 0
        return 0

    def vjp_scatter_shard(self, dt, it, n, m, width, is_, ys_bar, xs_bar, vs_part, sh, s):
        sh = sh._obj if hasattr(sh, "_obj") else sh
        t = _arr(is_, m, _IT[it])
        y = _arr(ys_bar, n * width, _DT[dt])
        x = _arr(xs_bar, n * width, _DT[dt])
        v = _arr(vs_part, m * width, _DT[dt])
        if x.ctypes.data != y.ctypes.data:
            x[:] = y
        for j, g in enumerate(t):
            loc = int(g) - sh.global_offset
            if 0 <= loc < n:
                v[j * width:(j + 1) * width] = y[loc * width:(loc + 1) * width]
                x[loc * width:(loc + 1) * width] = 0
            else:
                v[j * width:(j + 1) * width] = 0
        return 0
