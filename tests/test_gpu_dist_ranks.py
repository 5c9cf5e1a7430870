"""The multi-GPU module (paper_2202_10297_b200.dist) with REAL process groups:
world_size 2 processes, both on cuda:0 (gpurun exposes one GPU), gloo backend
for the tiny exchanges (dist routes them through host memory; with NCCL on an
8-GPU box the same calls use all_gather_into_tensor / all_reduce on device).
The NCCL data plane itself (device all_gather_into_tensor / all_reduce) runs
in `test_dist_nccl_world1`: one rank, backend "nccl" (NCCL rejects two ranks
on one device), the same calls and checks.
Every rank computes its contiguous shard; rank 0 assembles and checks against
the oracle on the whole array."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, backend="gloo"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(0)
        dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2202_10297_b200 import dist as vdist
        from _parity import assert_close
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        results = {}
        # scan LINREC / MAT2 / ADD over a global array split in contiguous shards
        for op, gen, w in (("linrec", synth.linrec_inputs, 2), ("mat2", synth.mat2_inputs, 4),
                           ("add", None, 1), ("min", "min", 1)):
            N = 300_007
            off, n = vdist.shard_bounds(N, world, rank)
            if gen is None:
                a_l, y_l = None, synth.scan_add_seed(n, offset=off, device=dev)
            elif gen == "min":  # two exchanges (rs-dependent reverse maps)
                a_l = synth.integers(n, 9, 0, 63, offset=off, device=dev).to(torch.float64) / 64.0
                y_l = synth.uniform(n, 10, offset=off, device=dev)
            else:
                a_l, y_l = gen(n, offset=off, device=dev)
            ab = vdist.scan(op, y_l, a_l, offset=off, global_n=N)
            parts = [None] * world
            dist.all_gather_object(parts, ab.cpu().numpy())  # shards differ in size by one element
            if rank == 0:
                if gen is None:
                    a, y = None, synth.scan_add_seed(N)
                elif gen == "min":
                    a, y = synth.integers(N, 9, 0, 63).to(torch.float64) / 64.0, synth.uniform(N, 10)
                else:
                    a, y = gen(N)
                ref = oracle.vjp_scan(op, y.numpy(), None if a is None else a.numpy())
                assert_close(np.concatenate(parts), ref, np.float64, what=f"2-rank scan {op}")
        # reduce(min) and reduce(*) with one zero
        for op in ("min", "mul"):
            N = 1_000_003
            off, n = vdist.shard_bounds(N, world, rank)
            full = synth.min_inputs(N, dtype=torch.float64) if op == "min" else \
                synth.mul_inputs(N, zeros="one", dtype=torch.float64)
            ab, y, arg = vdist.reduce(op, full[off:off + n].clone().to(dev), 1.5, offset=off, global_n=N, want_y=True)
            parts = [None] * world
            dist.all_gather_object(parts, ab.cpu().numpy())
            if rank == 0:
                ref, ry, rarg, _ = oracle.vjp_reduce(op, full.numpy(), 1.5)
                got = np.concatenate(parts)
                assert int(arg.item()) == rarg
                assert_close(got, ref, np.float64, what=f"2-rank reduce {op}")
        # reduce_by_index (+, *, max)
        for op, m in (("add", 1000), ("mul", 1000), ("max", 20_000)):
            N = 500_009
            off, n = vdist.shard_bounds(N, world, rank)
            inds, a, hb = synth.rbi_inputs(N, m, op)
            ab = vdist.reduce_by_index(op, inds[off:off + n].clone().to(dev), a[off:off + n].clone().to(dev),
                                       hb.to(dev), offset=off, global_n=N)
            parts = [None] * world
            dist.all_gather_object(parts, ab.cpu().numpy())
            if rank == 0:
                ref = oracle.vjp_reduce_by_index(op, inds.numpy(), a.numpy(), hb.numpy())[0]
                assert_close(np.concatenate(parts), ref, np.float64, what=f"2-rank rbi {op}")
        # scatter: ys_bar partitioned, global targets replicated, vs_bar all_reduced
        for width in (1, 3):
            N, M = 100_003, 30_000
            off, n = vdist.shard_bounds(N, world, rank)
            is_, yb = synth.scatter_inputs(N, M, oob=2)
            yb = yb.repeat_interleave(width) if width > 1 else yb
            xb, vb = vdist.scatter(is_.to(dev), yb[off * width:(off + n) * width].clone().to(dev), offset=off,
                                   global_n=N, width=width, in_place=(width == 1))
            parts = [None] * world
            dist.all_gather_object(parts, xb.cpu().numpy())
            if rank == 0:
                rx, rv, _ = oracle.vjp_scatter(is_.numpy(), yb.numpy(), width=width)
                assert np.array_equal(np.concatenate(parts), rx), "2-rank scatter xs_bar"
                assert np.array_equal(vb.cpu().numpy(), rv), "2-rank scatter vs_bar"
        # config-5 k-means gradient: points split by rank, all_reduce of partials
        N, K, D = 40_003, 96, 24
        P, C = synth.kmeans_inputs(N, K, D)
        off, n = vdist.shard_bounds(N, world, rank)
        r = vdist.kmeans(P[off:off + n].to(dev), C.to(dev), 0.5)
        if rank == 0:
            ref = oracle.kmeans(P.numpy(), C.numpy(), cost_bar=0.5)
            assert np.array_equal(r["counts"].cpu().numpy(), ref["counts"])
            assert np.array_equal(r["hdiag"].cpu().numpy(), ref["hdiag"])
            a = ref["assign"]
            scale = np.zeros((K, D))
            np.add.at(scale, a, np.abs(C.numpy()[a] - P.numpy()))  # condition scaling (reading A22)
            assert_close(r["cbar"].cpu().numpy().ravel(), ref["cbar"].ravel(), np.float64,
                         scale=(2 * 0.5 * scale).ravel(), what="2-rank kmeans")
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))


def test_dist_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]


def test_dist_nccl_world1():
    """the same sequence with backend "nccl" at world size 1: every exchange of
    dist.py goes through NCCL's device collectives"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(0, 1, _free_port(), q, "nccl"))
    p.start()
    rank, res = q.get(timeout=600)
    p.join(timeout=60)
    assert res == "ok", res
