"""GPU parity of the BLOCK-CYCLIC multi-GPU vjp_scan (SURVEY 8f row f1,
vjp_scan_cyclic: superblocks dealt round-robin to the ranks, one persistent
sweep per rank, cross-rank decoupled look-back over status words every rank
pushes to every rank's status buffer).

gpurun has one GPU, so W ranks run as W VIRTUAL ranks on one device: each rank
has its own local arrays, workspace, status buffer and CUDA stream, and its own
kernel launch with grid_ctas = (SMs / W) CTAs, so all ranks' CTAs are resident
together and their sweeps really run concurrently, exchanging status words
through device memory exactly as peer-mapped buffers are used across GPUs.
The forward all_gather (MUL / LINREC / MAT2) is a torch.stack here.  Every
result is compared with the oracle on the whole array."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from _parity import assert_close

pytestmark = pytest.mark.gpu
vjp = pytest.importorskip("paper_2202_10297_b200")
from paper_2202_10297_b200 import dist as vdist  # noqa: E402

DEV = "cuda"
TD = {np.float64: torch.float64, np.float32: torch.float32}


def make(op, n, dt):
    td = TD[dt]
    if op == "add":
        return None, synth.scan_add_seed(n, dtype=td)
    if op == "mul":
        a = (1.0 + (synth.uniform(n, 7, dtype=torch.float64) - 0.5) * 2.0 ** -6).to(td)
        return a, synth.uniform(n, 8, dtype=td)
    if op == "linrec":
        return synth.linrec_inputs(n, dtype=td)
    return synth.mat2_inputs(n, dtype=td)


def run_cyclic(op, N, W, sb_tiles, dt=np.float64, epochs=(1,), accumulate=False, a=None, yb=None):
    L = vjp.lib()
    o = vjp.OPS[op]
    d = 2 if dt == np.float64 else 1
    w = vjp.WIDTH[o]
    if yb is None:
        a, yb = make(op, N, dt)
    sb = L.vjp_scan_cyclic_tile_elems(o, d) * sb_tiles
    sbytes = L.vjp_scan_cyclic_status_bytes(o, N, sb)
    status = [torch.zeros(sbytes, dtype=torch.uint8, device=DEV) for _ in range(W)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    grid = max(1, sms // W)
    ranks = []
    for r in range(W):
        cy = vjp.VjpCyclic()
        cy.rank, cy.world, cy.global_n, cy.sb_elems, cy.grid_ctas = r, W, N, sb, grid
        for q in range(W):
            cy.status[q] = status[q].data_ptr()
        spans = vdist.cyclic_layout(N, sb, W, r)
        n_loc = sum(ln for _, ln in spans)
        assert n_loc == L.vjp_scan_cyclic_local_n(cy)
        idx = np.concatenate([np.arange(g0, g0 + ln) for g0, ln in spans]) if spans else np.zeros(0, np.int64)
        def loc(t):
            return None if t is None else t.view(N, -1)[torch.from_numpy(idx)].reshape(-1).contiguous().to(DEV)
        ab0 = synth.uniform(n_loc * w, 77 + r, dtype=TD[dt]).to(DEV) if accumulate else None
        ranks.append(dict(cy=cy, idx=idx, n=n_loc, a=loc(a), yb=loc(yb), ab=(ab0.clone() if accumulate else
                     torch.empty(n_loc * w, dtype=TD[dt], device=DEV)), ab0=ab0,
                     ws=vjp.workspace(L.vjp_scan_workspace_bytes(o, d, n_loc), DEV),
                     stream=torch.cuda.Stream()))
    fwd_b = L.vjp_scan_cyclic_fwd_bytes(o, d, ranks[0]["cy"])
    results = []
    for ep in epochs:
        gathered = None
        if op != "add":
            parts = []
            for rk in ranks:
                rk["cy"].epoch = ep
                sbagg = torch.zeros(fwd_b // 8, dtype=torch.float64, device=DEV)
                ws = rk["ws"]
                rc = L.vjp_scan_cyclic_forward(o, d, rk["n"], vjp._p(rk["a"]), vjp._p(ws),
                                               0 if ws is None else ws.numel(), rk["cy"], vjp._p(sbagg),
                                               vjp._stream(torch.device(DEV)))
                assert rc == 0, rc
                parts.append(sbagg)
            gathered = torch.cat(parts)  # the all_gather, rank order
        torch.cuda.synchronize()
        for rk in ranks:  # every rank's sweep on its own stream: they run concurrently
            rk["cy"].epoch = ep
            if accumulate:
                rk["ab"].copy_(rk["ab0"])
            torch.cuda.synchronize()
        for rk in ranks:
            ws = rk["ws"]
            rc = L.vjp_scan_cyclic(o, d, rk["n"], vjp._p(rk["a"]), vjp._p(rk["yb"]), vjp._p(rk["ab"]), vjp._p(ws),
                                   0 if ws is None else ws.numel(), rk["cy"], vjp._p(gathered),
                                   ctypes_stream(rk["stream"]), vjp.ACCUMULATE if accumulate else 0)
            assert rc == 0, rc
        torch.cuda.synchronize()
        for q in range(W):
            assert int(status[q][:4].view(torch.int32).item()) == 0, f"rank {q}: look-back timed out"
        got = np.zeros((N, w), dtype=dt)
        for rk in ranks:
            got[rk["idx"]] = rk["ab"].view(-1, w).cpu().numpy()
        results.append(got.reshape(-1))
    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy())
    if accumulate:
        base = np.zeros((N, w), dtype=dt)
        for rk in ranks:
            base[rk["idx"]] = rk["ab0"].view(-1, w).cpu().numpy()
        ref = ref + base.reshape(-1)
    return results, ref


def ctypes_stream(s):
    import ctypes
    return ctypes.c_void_p(s.cuda_stream)


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_cyclic_parity(op, W):
    """ragged global size (the last superblock partial, its last tile partial),
    several superblocks per rank, every rank count 1..8; f64"""
    te = vjp.lib().vjp_scan_cyclic_tile_elems(vjp.OPS[op], 2)
    N = te * 4 * 23 + 777  # 24 superblocks of 4 tiles (last ragged)
    res, ref = run_cyclic(op, N, W, 4)
    if op == "add":
        assert_close(res[0], ref, np.float64, what=f"cyclic {op} W={W}")
    else:
        assert_close(res[0], ref, np.float64, what=f"cyclic {op} W={W}")


@pytest.mark.parametrize("op", ["add", "linrec"])
def test_cyclic_integer_seeds_bit_exact_and_epochs(op):
    """integer seeds (|.| <= 8) make every summation order exact: bit-exact
    against the oracle, over three consecutive calls (epochs) on the same
    status buffers — stale status words of the previous call are never read"""
    N = vjp.lib().vjp_scan_cyclic_tile_elems(vjp.OPS[op], 2) * 8 * 11 + 5
    a, yb = make(op, N, np.float64)
    yb = synth.integers(yb.numel(), 31, -8, 8).to(torch.float64)
    if op == "linrec":  # integer d and c = 1: every carry, prefix and product is an exact integer
        a = a.view(N, 2).clone()
        a[:, 0] = synth.integers(N, 32, -8, 8).to(torch.float64)
        a[:, 1] = 1.0
        a = a.reshape(-1)
    res, ref = run_cyclic(op, N, 4, 8, epochs=(5, 6, 7), a=a, yb=yb)
    for g in res:
        assert np.array_equal(g, ref)


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_cyclic_accumulate_and_f32(dt):
    op = "mat2"
    N = vjp.lib().vjp_scan_cyclic_tile_elems(vjp.OPS[op], 2 if dt == np.float64 else 1) * 3 * 9 + 3
    res, ref = run_cyclic(op, N, 3, 3, dt=dt, accumulate=True)
    assert_close(res[0], ref, dt, what="cyclic accumulate")


def test_cyclic_small_and_single_superblock():
    for op in ("add", "mat2"):
        for N in (1, 5, 1000):
            res, ref = run_cyclic(op, N, 4, 2)  # fewer superblocks than ranks: ranks that own none
            assert_close(res[0], ref, np.float64, what=f"cyclic tiny {op} N={N}")


@pytest.mark.slow
def test_cyclic_scan_add_2p28():
    """scan(+) f64 at 2^28 over 4 virtual ranks, default superblock size"""
    L = vjp.lib()
    N = 1 << 28
    sb_tiles = max(1, L.vjp_scan_cyclic_sb_elems(1, 2) // L.vjp_scan_cyclic_tile_elems(1, 2) // 8)
    res, ref = run_cyclic("add", N, 4, sb_tiles)
    assert_close(res[0], ref, np.float64, what="cyclic 2^28")
