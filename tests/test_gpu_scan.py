"""GPU parity of vjp_scan (CUDA path through the C ABI) against the oracle.

Sizes span several tiles and ragged tails for every operator and dtype
(tile = 256 rows x 128 B: e.g. 4096 f64 ADD elements, 1024 f64 MAT2 elements),
plus config 1 (n = 10^4) and config 2 (n = 2^26 LINREC and MAT2, f64) at full
size.  Tolerances: north_star (f64 rel 1e-10, f32 rel 1e-4); integer seeds are
compared bit-exactly.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from _parity import assert_close

pytestmark = pytest.mark.gpu

vjp = pytest.importorskip("paper_2202_10297_b200")

DEV = "cuda"
SIZES = [1, 2, 3, 5, 31, 32, 33, 255, 256, 257, 1023, 1024, 1025, 4095, 4096, 4097, 8191, 8193,
         3 * 8192 + 17, 10_000, 100_003, 1_000_001]
WIDTH = {"add": 1, "mul": 1, "min": 1, "max": 1, "linrec": 2, "mat2": 4}
TD = {np.float64: torch.float64, np.float32: torch.float32}


def make(op, n, dt, device="cpu"):
    td = TD[dt]
    w = WIDTH[op]
    if op == "add":
        return None, synth.scan_add_seed(n, dtype=td, device=device)
    if op == "mul":
        a = (1.0 + (synth.uniform(n, 7, dtype=torch.float64, device=device) - 0.5) * 2.0 ** -6).to(td)
        return a, synth.uniform(n, 8, dtype=td, device=device)
    if op in ("min", "max"):
        k = synth.integers(n, 9, 0, 63, device=device)
        a = (k.to(torch.float64) / 64.0).to(td)  # many exact ties: pick-left rule matters
        return a, synth.uniform(n, 10, dtype=td, device=device)
    if op == "linrec":
        return synth.linrec_inputs(n, dtype=td, device=device)
    if op == "mat2":
        return synth.mat2_inputs(n, dtype=td, device=device)
    raise ValueError(op)


def run_both(op, n, dt, lookback=False, sweep=False, **kw):
    a, yb = make(op, n, dt)
    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy())
    got = vjp.scan(op, yb.to(DEV), None if a is None else a.to(DEV), lookback=lookback, sweep=sweep, **kw)
    torch.cuda.synchronize()
    return got.cpu().numpy(), ref


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "min", "max", "linrec", "mat2"])
def test_scan_parity_sizes(op, dt):
    """default path (chunked reduce-then-scan; MIN/MAX: look-back)"""
    for n in SIZES:
        got, ref = run_both(op, n, dt)
        assert_close(got, ref, dt, what=f"{op} n={n}")


@pytest.mark.parametrize("op", ["add", "mul", "min", "max", "linrec", "mat2"])
def test_scan_parity_lookback_path(op):
    """the single-sweep decoupled look-back kernels (VJP_SCAN_LOOKBACK)"""
    for n in (1, 33, 1023, 4097, 100_003, 1_000_001):
        got, ref = run_both(op, n, np.float64, lookback=True)
        assert_close(got, ref, np.float64, what=f"lookback {op} n={n}")


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "linrec", "mat2"])
def test_scan_parity_sweep_path(op, dt):
    """the one-read L2-round sweep (VJP_SCAN_SWEEP): rounds of G*K tiles,
    producer / carry warps, per-warp TMA stores; sizes from one partial tile to
    many rounds (1 tile per CTA per round at these sizes)."""
    for n in (1, 33, 1023, 4097, 100_003, 1_000_001, 3_000_017):
        got, ref = run_both(op, n, dt, sweep=True)
        assert_close(got, ref, dt, what=f"sweep {op} n={n}")


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["add", "mul", "min", "max", "linrec", "mat2"])
def test_scan_parity_blocklb_path(op, dt):
    """the one-read block look-back (VJP_SCAN_BLOCKLB; scan_blocklb.cuh):
    one partial tile, one block, many blocks with several look-back windows of
    32 descriptors, ragged last tiles."""
    for n in (1, 33, 1023, 4097, 100_003, 1_000_001, 3_000_017, 9_000_011):
        got, ref = run_both(op, n, dt, blocklb=True)
        assert_close(got, ref, dt, what=f"blocklb {op} n={n}")


@pytest.mark.parametrize("path", ["sweep", "blocklb"])
@pytest.mark.parametrize("op", ["add", "linrec", "mat2", "min"])
def test_scan_one_read_paths_accumulate_ys(op, path):
    """the one-read paths with ACCUMULATE and with ys."""
    if op == "min" and path == "sweep":
        pytest.skip("the sweep handles rs-independent maps only")
    n = 2_000_003
    a, yb = make(op, n, np.float64)
    if a is None:
        a = synth.uniform(n, 11, dtype=torch.float64)
    base = synth.uniform(n * WIDTH[op], 12, dtype=torch.float64)
    ref_acc = oracle.vjp_scan(op, yb.numpy(), a.numpy(), out=base.numpy().copy(), accumulate=True)
    ref, ref_ys = oracle.vjp_scan(op, yb.numpy(), a.numpy(), want_ys=True)
    kw = {path: True}
    out = base.to(DEV)
    vjp.scan(op, yb.to(DEV), a.to(DEV), out=out, accumulate=True, **kw)
    assert_close(out.cpu().numpy(), ref_acc, np.float64, what=f"{path} acc {op}")
    got, ys = vjp.scan(op, yb.to(DEV), a.to(DEV), want_ys=True, **kw)
    assert_close(got.cpu().numpy(), ref, np.float64, what=f"{path} {op}")
    # (LINREC's C = prod c underflows towards 0 at this length: absolute scale 1e-290 there)
    assert_close(ys.cpu().numpy(), ref_ys, np.float64, scale=np.full(ref_ys.size, 1e-290), what=f"{path} ys {op}")


def test_scan_tuning_knobs_subprocess():
    """the process-wide tuning knobs (read once at first use, vjp.h): several
    sweep tiles per CTA per round, a 2-round look-ahead, and block look-back
    blocks of 1 tile (many look-back windows) still match the oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "import numpy as np, torch, oracle, synth, paper_2202_10297_b200 as vjp\n"
        "from _parity import assert_close\n"
        "for op in ('add', 'linrec'):\n"
        "    n = 2_000_003\n"
        "    a, yb = (None, synth.scan_add_seed(n)) if op == 'add' else synth.linrec_inputs(n)\n"
        "    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy())\n"
        "    for kw in ({'sweep': True}, {'blocklb': True}):\n"
        "        got = vjp.scan(op, yb.cuda(), None if a is None else a.cuda(), **kw).cpu().numpy()\n"
        "        assert_close(got, ref, np.float64, what=f'{op} {kw}')\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"VJP_SWEEP_K": "3", "VJP_SWEEP_D": "1", "VJP_LB_L2_MB": "1"},
                {"VJP_SWEEP_K": "8", "VJP_SWEEP_D": "2", "VJP_LB_L2_MB": "400"}):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env},
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("dt", [np.float64, np.float32], ids=["f64", "f32"])
def test_scan_add_integer_seeds_bit_exact(dt):
    """integer seeds in [-8, 8]: every summation order is exact."""
    for n in (10_000, 1 << 20, (1 << 20) + 3, 5_000_011):
        yb = synth.scan_add_seed(n, kind="int", dtype=TD[dt])
        ref = oracle.vjp_scan("add", yb.numpy(), None)
        for kw in ({}, {"lookback": True}, {"sweep": True}, {"chunked": True}, {"blocklb": True}):
            got = vjp.scan("add", yb.to(DEV), **kw).cpu().numpy()
            assert np.array_equal(got, ref), kw


def test_scan_add_config1_closed_form():
    """config 1: n = 10^4 f64, U(0,1) seeds: oracle parity + closed form
    as_bar_i = n - i for ones."""
    n = 10_000
    got, ref = run_both("add", n, np.float64)
    assert_close(got, ref, np.float64, what="config1")
    ones = torch.ones(n, dtype=torch.float64, device=DEV)
    assert torch.equal(vjp.scan("add", ones).cpu(), torch.arange(n, 0, -1, dtype=torch.float64))


@pytest.mark.parametrize("op", ["add", "mul", "min", "linrec", "mat2"])
def test_scan_want_ys(op):
    """the primal scan recomputed in the return sweep (ys) matches the oracle."""
    for n in (1, 1000, 70_001):
        a, yb = make(op, n, np.float64)
        if a is None:
            a = synth.uniform(n, 11, dtype=torch.float64)
        if op == "linrec":  # keep prod(c) away from underflow so ys_C is comparable elementwise
            a = a.reshape(n, 2).clone()
            a[:, 1] = 1.0 + (synth.uniform(n, 13, dtype=torch.float64) - 0.5) / 64
            a = a.reshape(-1)
        ref, ref_ys = oracle.vjp_scan(op, yb.numpy(), a.numpy(), want_ys=True)
        got, ys = vjp.scan(op, yb.to(DEV), a.to(DEV), want_ys=True)
        assert_close(got.cpu().numpy(), ref, np.float64, what=f"{op} as_bar n={n}")
        assert_close(ys.cpu().numpy(), ref_ys, np.float64, what=f"{op} ys n={n}")


@pytest.mark.parametrize("op", ["add", "mat2", "max"])
def test_scan_accumulate(op):
    n = 50_001
    a, yb = make(op, n, np.float64)
    base = synth.uniform(n * WIDTH[op], 12, dtype=torch.float64)
    ref = oracle.vjp_scan(op, yb.numpy(), None if a is None else a.numpy(), out=base.numpy().copy(),
                          accumulate=True)
    out = base.to(DEV)
    vjp.scan(op, yb.to(DEV), None if a is None else a.to(DEV), out=out, accumulate=True)
    assert_close(out.cpu().numpy(), ref, np.float64, what="accumulate")


def test_scan_host_buffers_e2e():
    """the public API with host tensors (copies inside the call)."""
    a, yb = make("linrec", 12345, np.float64)
    got = vjp.scan("linrec", yb, a)
    assert not got.is_cuda
    assert_close(got.numpy(), oracle.vjp_scan("linrec", yb.numpy(), a.numpy()), np.float64)


def test_scan_errors():
    yb = torch.ones(16, dtype=torch.float64, device=DEV)
    with pytest.raises(vjp.VjpError) as e:
        vjp.scan("mat2", yb, None)  # MAT2 needs `as`
    assert e.value.code == 1
    big = torch.ones(17, dtype=torch.float64, device=DEV)
    with pytest.raises(vjp.VjpError) as e:
        vjp.scan("add", big[1:])  # 8-byte offset: not 16-byte aligned
    assert e.value.code == 7
    assert vjp.scan("add", torch.ones(0, dtype=torch.float64, device=DEV)).numel() == 0


@pytest.mark.slow
@pytest.mark.parametrize("op", ["linrec", "mat2"])
def test_config2_full_size(op):
    """config 2: n = 2^26 f64 on one B200, the launch configuration bench.py times."""
    n = 1 << 26
    a, yb = make(op, n, np.float64, device=DEV)
    got = vjp.scan(op, yb, a).cpu().numpy()
    ref = oracle.vjp_scan(op, yb.cpu().numpy(), a.cpu().numpy())
    assert_close(got, ref, np.float64, what=f"config2 {op}")


@pytest.mark.slow
def test_scan_add_2pow30_sampled():
    """target size n = 2^30 f64: integer seeds -> the closed form is exact, so
    the reversed cumulative sum (torch, int64) is the oracle's value exactly."""
    n = 1 << 30
    yb = synth.scan_add_seed(n, kind="int", device=DEV)
    got = vjp.scan("add", yb)
    exact = torch.flip(torch.cumsum(torch.flip(yb.to(torch.int64), [0]), 0), [0])
    assert torch.equal(got.to(torch.int64), exact)
    got_ch = vjp.scan("add", yb, chunked=True)  # (the default above is the one-pass look-back kernel)
    assert torch.equal(got_ch.to(torch.int64), exact)
    del got_ch
    # sampled comparison against the oracle on a slice near the end (independent of the prefix)
    tail = yb[-100_000:].cpu().numpy()
    ref_tail = oracle.vjp_scan("add", tail, None)
    assert np.array_equal(got[-100_000:].cpu().numpy(), ref_tail)


@pytest.mark.parametrize("op", ["min", "max"])
def test_scan_minmax_special_values(op):
    """MIN/MAX scans (chunked rs-dependent path): +-inf at the start (the first
    element's adjoint is rbar_0 whatever a_0 is), long runs of ties
    (pick-left), -0.0 vs +0.0, a tail spanning tiles; both paths vs the oracle."""
    n = 300_007
    k = synth.integers(n, 21, 0, 3)
    a = (k.to(torch.float64) - 1.5)
    a[0] = float("inf") if op == "min" else float("-inf")
    a[1000:1100] = -0.0
    a[1100:1200] = 0.0
    yb = synth.uniform(n, 22)
    ref = oracle.vjp_scan(op, yb.numpy(), a.numpy())
    for kw in ({}, {"lookback": True}):
        got = vjp.scan(op, yb.to(DEV), a.to(DEV), **kw).cpu().numpy()
        assert_close(got, ref, np.float64, what=f"{op} special {kw}")


def test_scan_host_async_pipeline():
    """the asynchronous host-buffer path (sync=False): several calls in flight
    on the copy-in / compute / copy-out streams give the synchronous results"""
    outs, refs = [], []
    for k, op in enumerate(["linrec", "mat2", "add", "linrec"]):
        n = 100_003 + 1000 * k
        a, yb = make(op, n, np.float64)
        a = None if a is None else a.pin_memory()
        yb = yb.pin_memory()
        out = torch.empty(yb.shape, dtype=yb.dtype, pin_memory=True)
        outs.append((vjp.scan(op, yb, a, out=out, sync=False), out))
        refs.append(vjp.scan(op, yb.to(DEV), None if a is None else a.to(DEV)).cpu())
    for (p, out), ref in zip(outs, refs):
        got = p.wait()
        assert got.data_ptr() == out.data_ptr()
        assert torch.equal(got, ref)


@pytest.mark.parametrize("op", ["linrec", "mat2"])
def test_bench_sequence_dist_scan_world1(op):
    """the exact call sequence bench.py times for config 2 (dist.scan at
    world = 1: vjp_scan_partial + vjp_scan_finish on a whole-array 'shard',
    events around the finish, a preallocated out) against the oracle, at a
    tile-spanning ragged size and twice in a row on the same buffers"""
    from paper_2202_10297_b200 import dist as vdist
    n = 3 * (1 << 16) + 123
    a, yb = make(op, n, np.float64)
    ref = oracle.vjp_scan(op, yb.numpy(), a.numpy())
    ad, ybd = a.to(DEV), yb.to(DEV)
    ab = torch.empty_like(ybd)
    for _ in range(2):
        ev = {"finish_start": torch.cuda.Event(enable_timing=True), "finish_end": torch.cuda.Event(enable_timing=True)}
        vdist.scan(op, ybd, ad, offset=0, global_n=n, out=ab, events=ev)
        torch.cuda.synchronize()
        assert ev["finish_start"].elapsed_time(ev["finish_end"]) > 0
        assert_close(ab.cpu().numpy(), ref, np.float64, what=f"bench sequence {op}")


def test_scan_add_f32_2pow30_one_pass():
    """target size n = 2^30 f32 on the default one-pass kernel: integer seeds
    (|.| <= 8), accumulated in f64 (R9) exactly, rounded once to f32 — the
    same single rounding of the exact suffix sum the oracle performs, so the
    result equals the exact int64 suffix sum cast to f32 bit for bit."""
    n = 1 << 30
    yb = synth.scan_add_seed(n, kind="int", device=DEV).to(torch.float32)
    got = vjp.scan("add", yb)
    exact = torch.flip(torch.cumsum(torch.flip(yb.to(torch.int64), [0]), 0), [0])
    assert torch.equal(got, exact.to(torch.float64).to(torch.float32))


@pytest.mark.parametrize("op", ["min", "max"])
def test_scan_minmax_one_pass_large(op):
    """MIN/MAX one-pass return (K_F + look-back) at 2^26 f64 with many ties
    and records spread over the array: against the chunked rs path (an
    independent kernel chain) exactly, and against the oracle on a sampled
    tail slice (its carry from the right is zero at the end)"""
    n = 1 << 26
    a = synth.min_inputs(n, dtype=torch.float64, device=DEV)
    if op == "max":
        a = -a
    yb = synth.scan_add_seed(n, kind="int", device=DEV)  # integer seeds: every order exact
    got = vjp.scan(op, yb, a)
    ref = vjp.scan(op, yb, a, chunked=True)
    assert torch.equal(got, ref)
    m = 200_000
    # the oracle on the whole array would be slow: compare the head (records
    # entering from the left are exactly those of the prefix)
    head_ref = oracle.vjp_scan(op, yb[:m].cpu().numpy(), a[:m].cpu().numpy())
    # the head's outputs also depend on the carry from the right: only where a
    # record lies at or after the head's end does the carry vanish, so compare
    # the positions before the last record of the head
    rec = np.nonzero(head_ref != 0)[0]
    if len(rec) > 1:
        last = rec[-1]
        assert np.array_equal(got[:last].cpu().numpy(), head_ref[:last])
