"""Multi-process (world_size 2, gloo, CPU) checks of the host-side logic of
the multi-GPU path: contiguous shard bounds, the rank-ordered all_gather of
per-shard scan records feeding the carry combination (vjp_scan_carries_host,
the same __host__ __device__ code the finish kernel runs), the two-exchange
protocol of the MIN/MAX scans, and the
reduce_by_index max/min winner protocol (all_reduce MAX of values, candidate
selection, all_reduce MIN of global indices) — each against the oracle on the
unsharded array."""
from __future__ import annotations

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mat2_record(A, Y):
    """[fwd product | D | C] of a shard, from the definitions (P:1137 and the
    per-element grouping H_i = (ybar_i + H_{i+1}) A_i^T of P:1180)."""
    P = np.eye(2)
    for a in A:
        P = P @ a
    D, C = np.zeros((2, 2)), np.eye(2)
    for a, y in zip(A[::-1], Y[::-1]):
        D = (y + D) @ a.T
        C = C @ a.T
    return np.concatenate([P.ravel(), D.ravel(), C.ravel()])


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import oracle
        import synth
        import paper_2202_10297_b200 as vjp
        from paper_2202_10297_b200.dist import shard_bounds

        L = vjp.lib()
        # ---- scan MAT2: records -> all_gather -> carries -----------------
        N = 37
        a, y = synth.mat2_inputs(N)
        A, Y = a.numpy().reshape(N, 2, 2), y.numpy().reshape(N, 2, 2)
        off, n = shard_bounds(N, world, rank)
        rec = torch.from_numpy(_mat2_record(A[off:off + n], Y[off:off + n]))
        bufs = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(bufs, rec)
        gathered = torch.cat(bufs).contiguous().numpy()
        fwd, rev = np.zeros(4), np.zeros(4)
        rc = L.vjp_scan_carries_host(6, 2, rank, world, gathered.ctypes.data_as(ctypes.c_void_p),
                                     fwd.ctypes.data_as(ctypes.c_void_p), rev.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        _, ys = oracle.vjp_scan("mat2", y.numpy(), a.numpy(), want_ys=True)
        exp_fwd = ys.reshape(N, 4)[off - 1] if off > 0 else np.eye(2).ravel()
        np.testing.assert_allclose(fwd, exp_fwd, rtol=1e-13)
        H = np.zeros((2, 2))
        for j in range(N - 1, off + n - 1, -1):
            H = (Y[j] + H) @ A[j].T
        np.testing.assert_allclose(rev, H.ravel(), rtol=1e-12, atol=1e-300)

        # ---- scan MIN across ranks: the two-exchange protocol -------------
        # exchange 1: forward aggregates; exchange 2: the reverse-map aggregates
        # built with the forward carry (pick-left Jacobians need rs); then each
        # rank's return sweep from the combined carries equals the oracle slice
        N = 41
        a = (synth.integers(N, 9, 0, 5).to(torch.float64) / 4.0).numpy()
        yv = synth.uniform(N, 10).numpy()
        off, n = shard_bounds(N, world, rank)
        F = float("inf")
        for v in a[off:off + n]:
            F = F if F <= v else v
        r1 = torch.tensor([F, 0.0, 1.0], dtype=torch.float64)
        b1 = [torch.empty_like(r1) for _ in range(world)]
        dist.all_gather(b1, r1)
        g1 = torch.cat(b1).contiguous().numpy()
        fwd, rev = np.zeros(1), np.zeros(1)
        assert L.vjp_scan_carries_host(3, 2, rank, world, g1.ctypes.data_as(ctypes.c_void_p),
                                       fwd.ctypes.data_as(ctypes.c_void_p), rev.ctypes.data_as(ctypes.c_void_p)) == 0
        exp_f = float("inf")
        for v in a[:off]:
            exp_f = exp_f if exp_f <= v else v
        assert fwd[0] == exp_f
        rs = fwd[0]  # maps with the true rs: M_i(X) = [rs_{i-1} <= a_i] (ybar_i + X), composed right to left
        Dm, Cm = 0.0, 1.0
        jl = []
        for v in a[off:off + n]:
            jl.append(1.0 if rs <= v else 0.0)
            rs = rs if rs <= v else v
        for i in range(n - 1, -1, -1):  # M = M_lo o ... o M_hi
            Dm, Cm = jl[i] * (yv[off + i] + Dm), jl[i] * Cm
        r2 = torch.tensor([float("inf"), Dm, Cm], dtype=torch.float64)
        b2 = [torch.empty_like(r2) for _ in range(world)]
        dist.all_gather(b2, r2)
        g2 = torch.cat(b2).contiguous().numpy()
        assert L.vjp_scan_carries_host(3, 2, rank, world, g2.ctypes.data_as(ctypes.c_void_p),
                                       fwd.ctypes.data_as(ctypes.c_void_p), rev.ctypes.data_as(ctypes.c_void_p)) == 0
        H = rev[0]
        out = np.zeros(n)
        for i in range(n - 1, -1, -1):
            g = yv[off + i] + H
            out[i] = g if off + i == 0 else (1.0 - jl[i]) * g
            H = jl[i] * g
        ref = oracle.vjp_scan("min", yv, a)
        np.testing.assert_allclose(out, ref[off:off + n], rtol=1e-14, atol=0)

        # ---- reduce_by_index and scatter THROUGH dist.* (the module's own
        # sequencing, buffers and gloo collectives), with the kernels replaced by
        # CPU fakes of their documented contracts (tests/_fake_lib.py) ----------
        import paper_2202_10297_b200.dist as vdist
        from _fake_lib import FakeLib
        real_lib, real_stream = vdist.lib, vdist._stream
        vdist.lib = lambda: FakeLib()
        vdist._stream = lambda dev: None
        try:
            for op, M, NN in (("max", 50, 2000), ("min", 37, 1500), ("mul", 40, 1200), ("add", 30, 900)):
                inds, av, hb = synth.rbi_inputs(NN, M, op)
                if op == "mul":  # signed factors: the exchange must carry the sign parity
                    av = torch.where(synth.uniform(NN, 55) < 0.3, -av, av)
                off, n = shard_bounds(NN, world, rank)
                got = vdist.reduce_by_index(op, inds[off:off + n].clone(), av[off:off + n].clone(), hb.clone(),
                                            offset=off, global_n=NN)
                ref = oracle.vjp_reduce_by_index(op, inds.numpy(), av.numpy(), hb.numpy())[0][off:off + n]
                if op == "mul":
                    np.testing.assert_allclose(got.numpy(), ref, rtol=1e-10, atol=0)
                else:
                    assert np.array_equal(got.numpy(), ref), op
            NS, MS = 5_021, 900
            is_, ybs = synth.scatter_inputs(NS, MS, oob=3)
            off, n = shard_bounds(NS, world, rank)
            xb, vb = vdist.scatter(is_, ybs[off:off + n].clone(), offset=off, global_n=NS)
            rx, rv, _ = oracle.vjp_scatter(is_.numpy(), ybs.numpy())
            assert np.array_equal(vb.numpy(), rv)
            assert np.array_equal(xb.numpy(), rx[off:off + n])
        finally:
            vdist.lib, vdist._stream = real_lib, real_stream
        # ---- block-cyclic layout (f1): the ranks' superblocks tile [0, N) once,
        # and the library's local-size query agrees with the Python layout ------
        for NN, sb in ((100_000, 4096), (4096 * 7, 4096), (5, 4096), (0, 4096)):
            spans = vdist.cyclic_layout(NN, sb, world, rank)
            cy = vjp.VjpCyclic()
            cy.rank, cy.world, cy.global_n, cy.sb_elems = rank, world, NN, sb
            assert L.vjp_scan_cyclic_local_n(cy) == sum(ln for _, ln in spans)
            mine = torch.zeros(NN, dtype=torch.int64)
            for g0, ln in spans:
                assert (g0 // sb) % world == rank
                mine[g0:g0 + ln] += 1
            dist.all_reduce(mine)
            assert bool((mine == 1).all())
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_dist_protocols_gloo(world):
    from paper_2202_10297_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]


def test_shard_bounds_cover():
    from paper_2202_10297_b200.dist import shard_bounds
    for N in (0, 1, 7, 1000, 10**6 + 3):
        for W in (1, 2, 3, 8):
            bs = [shard_bounds(N, W, r) for r in range(W)]
            assert bs[0][0] == 0
            for (o1, n1), (o2, _) in zip(bs, bs[1:]):
                assert o1 + n1 == o2
            assert sum(n for _, n in bs) == N
            assert max(n for _, n in bs) - min(n for _, n in bs) <= 1
