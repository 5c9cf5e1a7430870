"""The multi-GPU split API (partial -> exchange -> finish) on ONE GPU: every
"rank" is a shard of the same array, the exchange (all_gather / all_reduce)
is emulated by torch ops on the device.  Checks the device-side carry
combination end to end against the oracle on the whole array, for 2..5
shards with ragged sizes (gpurun gives one GPU; the real NCCL run is the
same calls with dist.all_gather_into_tensor / all_reduce)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from _parity import assert_close

pytestmark = pytest.mark.gpu
vjp = pytest.importorskip("paper_2202_10297_b200")
from paper_2202_10297_b200 import VjpShard, dist as vdist  # noqa: E402

DEV = "cuda"


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def shards(N, world):
    return [vdist.shard_bounds(N, world, r) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_scan_split_emulated(op, world):
    L = vjp.lib()
    o = vjp.OPS[op]
    w = vjp.WIDTH[o]
    N = 200_003
    if op == "add":
        a, yb = None, synth.scan_add_seed(N)
    elif op == "mul":
        a = 1.0 + (synth.uniform(N, 7) - 0.5) * 2.0 ** -6
        yb = synth.uniform(N, 8)
    elif op == "linrec":
        a, yb = synth.linrec_inputs(N)
    else:
        a, yb = synth.mat2_inputs(N)
    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy())
    rec = L.vjp_scan_partial_bytes(o, 2) // 8
    parts, state = [], []
    for r, (off, n) in enumerate(shards(N, world)):
        a_r = None if a is None else a[off * w:(off + n) * w].clone().to(DEV)
        y_r = yb[off * w:(off + n) * w].clone().to(DEV)
        ws = torch.empty(L.vjp_scan_workspace_bytes(o, 2, n), dtype=torch.uint8, device=DEV)
        part = torch.empty(rec, dtype=torch.float64, device=DEV)
        sh = VjpShard(r, world, off, N)
        assert L.vjp_scan_partial(o, 2, n, _p(a_r), _p(y_r), _p(ws), ws.numel(), sh, _p(part), _s(), 0) == 0
        parts.append(part)
        state.append((a_r, y_r, ws, sh, n))
    gathered = torch.cat(parts)  # the all_gather, in rank order
    outs = []
    for a_r, y_r, ws, sh, n in state:
        ab = torch.empty_like(y_r)
        assert L.vjp_scan_finish(o, 2, n, _p(a_r), _p(y_r), _p(ab), None, _p(ws), ws.numel(), sh, _p(gathered),
                                 _s(), 0) == 0
        outs.append(ab)
    got = torch.cat(outs).cpu().numpy()
    assert_close(got, ref, np.float64, what=f"split {op} world={world}")


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("op", ["min", "max"])
def test_scan_minmax_two_exchanges_emulated(op, world):
    """MIN/MAX scans across shards: partial (forward aggregates) -> gather ->
    partial2 (reverse aggregates with the shard forward carry) -> gather ->
    finish; many exact ties (pick-left) so the forward carry decides sides."""
    L = vjp.lib()
    o = vjp.OPS[op]
    N = 200_003
    k = synth.integers(N, 9, 0, 63)
    a = k.to(torch.float64) / 64.0
    yb = synth.uniform(N, 10)
    ref = oracle.vjp_scan(op, yb.numpy(), a.numpy())
    rec = L.vjp_scan_partial_bytes(o, 2) // 8
    state, parts = [], []
    for r, (off, n) in enumerate(shards(N, world)):
        a_r = a[off:off + n].clone().to(DEV)
        y_r = yb[off:off + n].clone().to(DEV)
        ws = torch.empty(L.vjp_scan_workspace_bytes(o, 2, n), dtype=torch.uint8, device=DEV)
        part = torch.empty(rec, dtype=torch.float64, device=DEV)
        sh = VjpShard(r, world, off, N)
        assert L.vjp_scan_partial(o, 2, n, _p(a_r), _p(y_r), _p(ws), ws.numel(), sh, _p(part), _s(), 0) == 0
        parts.append(part)
        state.append((a_r, y_r, ws, sh, n))
    g1 = torch.cat(parts)
    parts2 = []
    for a_r, y_r, ws, sh, n in state:
        part2 = torch.empty(rec, dtype=torch.float64, device=DEV)
        assert L.vjp_scan_partial2(o, 2, n, _p(a_r), _p(y_r), _p(ws), ws.numel(), sh, _p(g1), _p(part2), _s(), 0) == 0
        parts2.append(part2)
    g2 = torch.cat(parts2)
    outs = []
    for a_r, y_r, ws, sh, n in state:
        ab = torch.empty_like(y_r)
        assert L.vjp_scan_finish(o, 2, n, _p(a_r), _p(y_r), _p(ab), None, _p(ws), ws.numel(), sh, _p(g2), _s(), 0) == 0
        outs.append(ab)
    assert_close(torch.cat(outs).cpu().numpy(), ref, np.float64, what=f"split {op} world={world}")


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("op,zeros", [("add", "none"), ("mul", "none"), ("mul", "one"), ("mul", "two"),
                                      ("min", None), ("max", None)])
def test_reduce_split_emulated(op, zeros, world):
    L = vjp.lib()
    o = vjp.OPS[op]
    N = 300_007
    a = (synth.mul_inputs(N, zeros=zeros, dtype=torch.float64) if op == "mul"
         else synth.min_inputs(N, dtype=torch.float64) * (-1 if op == "max" else 1) if op in ("min", "max")
         else synth.uniform(N, 3))
    ref_ab, ref_y, ref_arg, ref_z = oracle.vjp_reduce(op, a.numpy(), 2.0)
    recb = L.vjp_reduce_partial_bytes()
    parts, state = [], []
    for r, (off, n) in enumerate(shards(N, world)):
        a_r = a[off:off + n].clone().to(DEV)
        ws = torch.empty(L.vjp_reduce_workspace_bytes(o, 2, n), dtype=torch.uint8, device=DEV)
        part = torch.empty(recb, dtype=torch.uint8, device=DEV)
        sh = VjpShard(r, world, off, N)
        assert L.vjp_reduce_partial(o, 2, n, _p(a_r), _p(ws), ws.numel(), sh, _p(part), _s()) == 0
        parts.append(part)
        state.append((a_r, ws, sh, n))
    gathered = torch.cat(parts)
    yb = torch.tensor([2.0], dtype=torch.float64, device=DEV)
    outs = []
    y = torch.empty(1, dtype=torch.float64, device=DEV)
    arg = torch.empty(1, dtype=torch.int64, device=DEV)
    for a_r, ws, sh, n in state:
        ab = torch.empty_like(a_r)
        assert L.vjp_reduce_finish(o, 2, n, _p(a_r), _p(yb), _p(ab), _p(y), _p(arg), _p(ws), ws.numel(), sh,
                                   _p(gathered), _s(), 0) == 0
        outs.append(ab)
    got = torch.cat(outs).cpu().numpy()
    if op in ("min", "max"):
        assert int(arg.item()) == ref_arg and np.array_equal(got, ref_ab)
    else:
        assert_close(got, ref_ab, np.float64, what=f"split reduce {op}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("op,m", [("add", 1000), ("mul", 1000), ("mul", 100_000), ("max", 1000),
                                  ("max", 100_000), ("min", 5000)])
def test_rbi_split_emulated(op, m, world):
    """per-bin state all-reduced (integer SUM of the 64-bit factor codes and of
    the zero counts for *, MAX/MIN then MIN of the candidate indices for
    max/min), then the finish per shard."""
    L = vjp.lib()
    o = vjp.OPS[op]
    N = 400_009
    inds, a, hb = synth.rbi_inputs(N, m, op)
    ref = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy())[0]
    hb_d = hb.to(DEV)
    vals, auxs, state = [], [], []
    for r, (off, n) in enumerate(shards(N, world)):
        i_r = inds[off:off + n].clone().to(DEV)
        a_r = a[off:off + n].clone().to(DEV)
        ws_n = L.vjp_reduce_by_index_workspace_bytes(o, 2, n, m, 1)
        ws = torch.empty(max(ws_n, 1), dtype=torch.uint8, device=DEV)
        bv = torch.empty(m, dtype=torch.float64, device=DEV)
        ba = torch.empty(m, dtype=torch.int64, device=DEV)
        sh = VjpShard(r, world, off, N)
        assert L.vjp_reduce_by_index_partial(o, 2, 1, n, m, _p(i_r), _p(a_r), _p(ws), ws_n, sh, _p(bv), _p(ba),
                                             _s()) == 0
        vals.append(bv)
        auxs.append(ba)
        state.append((i_r, a_r, ws, ws_n, sh, n))
    if op == "mul":
        # codes add mod 2^64 (int64 two's complement wrap-around, as NCCL's SUM)
        gv = torch.stack([v.view(torch.int64) for v in vals]).sum(0).view(torch.float64)
        ga = torch.stack(auxs).sum(0)
        gvs, gas = [gv] * world, [ga] * world
    elif op in ("max", "min"):
        gv = torch.stack(vals).amax(0) if op == "max" else torch.stack(vals).amin(0)
        for r in range(world):
            assert L.vjp_reduce_by_index_select(o, m, _p(gv), _p(vals[r]), _p(auxs[r]), _s()) == 0
        ga = torch.stack(auxs).amin(0)
        gvs, gas = [gv] * world, [ga] * world
    else:
        gvs, gas = vals, auxs
    outs = []
    for r, (i_r, a_r, ws, ws_n, sh, n) in enumerate(state):
        ab = torch.empty(n, dtype=torch.float64, device=DEV)
        assert L.vjp_reduce_by_index_finish(o, 2, 1, n, m, _p(i_r), _p(a_r), _p(hb_d), _p(ab), _p(gvs[r]), _p(gas[r]),
                                            _p(ws), ws_n, sh, _s(), 0) == 0
        outs.append(ab)
    got = torch.cat(outs).cpu().numpy()
    if op == "mul":
        assert_close(got, ref, np.float64, what=f"split rbi mul m={m}")
    else:
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("it", [torch.int32, torch.int64], ids=["i32", "i64"])
def test_scatter_split_emulated(world, it):
    """vjp_scatter_shard per shard (ragged contiguous split of ys_bar, global
    targets replicated), the all_reduce SUM of the partial vs_bar emulated:
    bit-exact against the oracle on the whole array (one owner per target)."""
    L = vjp.lib()
    N, M, width = 70_001, 20_000, 2
    is_, yb = synth.scatter_inputs(N, M, itype=it, oob=4)
    yb = yb.repeat_interleave(width)
    rx, rv, _ = oracle.vjp_scatter(is_.numpy(), yb.numpy(), width=width)
    ix = is_.to(DEV)
    vsum = torch.zeros(M * width, dtype=torch.float64, device=DEV)
    xparts = []
    for r, (off, n) in enumerate(shards(N, world)):
        ys_loc = yb[off * width:(off + n) * width].clone().to(DEV)
        vpart = torch.empty(M * width, dtype=torch.float64, device=DEV)
        sh = VjpShard(r, world, off, N)
        rc = L.vjp_scatter_shard(2, 1 if it == torch.int32 else 2, n, M, width, _p(ix), _p(ys_loc), _p(ys_loc),
                                 _p(vpart), sh, _s())
        assert rc == 0
        vsum += vpart
        xparts.append(ys_loc.cpu().numpy())
    assert np.array_equal(np.concatenate(xparts), rx)
    assert np.array_equal(vsum.cpu().numpy(), rv)
