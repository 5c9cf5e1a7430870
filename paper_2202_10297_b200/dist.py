"""Multi-GPU vjp over torch.distributed (NCCL over NVLink), one process per GPU.

Contiguous partition: rank r owns elements
[offset_r, offset_r + n_r) of the global problem.  The path shards with ONE tiny
exchange step:

  scan            partial (forward re-execution + reverse-map aggregate of the
                  shard) -> all_gather of the per-shard records (40 B LINREC,
                  96 B MAT2) -> finish (return sweep with the combined carries).
                  MIN/MAX: two exchanges (forward aggregates, then reverse
                  aggregates built with the forward carry: partial2).
  reduce          partial record (p, z, i0) / (value, index) / sum -> all_gather
                  -> finish (deterministic rank-order combine on the device).
  reduce_by_index per-bin state -> all_reduce (integer SUM of the 64-bit factor
                  codes and of the zero counts for *, MAX/MIN then
                  MIN of candidate indices for max/min) -> finish; ADD needs no
                  exchange (hs_bar is replicated).
  scatter         ys_bar partitioned, targets replicated: each rank zeroes its
                  own targets and gathers them into a partial vs_bar (0 for
                  targets it does not own) -> all_reduce SUM (m * width
                  scalars; exactly one owner per target, so the sum is exact).
  kmeans          (config 5) points partitioned by rank, centers replicated:
                  every output is a sum over points, so the per-rank partials
                  (centers_bar, Hessian diagonal, counts, cost) are all_reduced
                  (SUM, k*d*8 B twice + k*8 B).

All arithmetic runs in libvjp_b200.so; this module only sequences the calls and
the collectives on the current stream.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (ACCUMULATE, ADD, MAX, MIN, WIDTH, VjpCyclic, VjpShard, _check, _dt, _it, _op, _p, _stream, lib,
               workspace)


def _all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather of a small device record; NCCL directly, gloo (CPU testing
    of the multi-rank path, e.g. several ranks on one GPU) through host memory."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    parts = [torch.empty_like(inp, device="cpu") for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, inp.cpu(), group=group)
    out.copy_(torch.cat(parts).to(out.device))


def _all_reduce(t: torch.Tensor, op, group=None):
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=op, group=group)
        return
    h = t.cpu()
    dist.all_reduce(h, op=op, group=group)
    t.copy_(h.to(t.device))


def cyclic_layout(global_n: int, sb_elems: int, world: int, rank: int) -> list[tuple[int, int]]:
    """block-cyclic partition (vjp_scan_cyclic): superblock J
    = global elements [J sb, min((J + 1) sb, global_n)) belongs to rank J %
    world; a rank's local array is its superblocks in increasing J.  Returns
    [(global_start, length), ...] in local order."""
    nsb = -(-global_n // sb_elems) if global_n > 0 else 0
    return [(J * sb_elems, min((J + 1) * sb_elems, global_n) - J * sb_elems) for J in range(rank, nsb, world)]


def shard_bounds(global_n: int, world: int, rank: int) -> tuple[int, int]:
    """contiguous, balanced split; rank r gets [off, off + n)."""
    base, rem = divmod(global_n, world)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def _shard(offset: int, n: int, global_n: int, group) -> VjpShard:
    if not (dist.is_available() and dist.is_initialized()):
        return VjpShard(0, 1, offset, global_n)
    return VjpShard(dist.get_rank(group), dist.get_world_size(group), offset, global_n)


def scan(op, ys_bar: torch.Tensor, as_: torch.Tensor | None, *, offset: int, global_n: int, group=None,
         out: torch.Tensor | None = None, want_ys: bool = False, accumulate: bool = False,
         events: dict | None = None):
    """vjp_scan over this rank's contiguous shard of a global scan.

    `events`, if given, maps "finish_start"/"finish_end" to torch.cuda.Event
    objects recorded around the return-sweep kernel (bench roofline)."""
    o = _op(op)
    dev = ys_bar.device
    w = WIDTH[o]
    n = ys_bar.numel() // w
    dt = _dt(ys_bar)
    L = lib()
    sh = _shard(offset, n, global_n, group)
    world = sh.world
    ab = out if out is not None else torch.empty_like(ys_bar)
    ys = torch.empty_like(ys_bar) if want_ys else None
    ws = workspace(L.vjp_scan_workspace_bytes(o, dt, n), dev)
    nbytes = 0 if ws is None else ws.numel()
    rec = L.vjp_scan_partial_bytes(o, dt) // 8
    part = torch.empty(rec, dtype=torch.float64, device=dev)
    s = _stream(dev)
    flags = ACCUMULATE if accumulate else 0
    _check(L.vjp_scan_partial(o, dt, n, _p(as_), _p(ys_bar), _p(ws), nbytes, sh, _p(part), s, flags),
           "vjp_scan_partial")
    gathered = None
    if world > 1:
        gathered = torch.empty(world * rec, dtype=torch.float64, device=dev)
        _all_gather_into(gathered, part, group)
        if o in (MIN, MAX):  # rs-dependent maps: a second exchange of reverse aggregates
            part2 = torch.empty(rec, dtype=torch.float64, device=dev)
            _check(L.vjp_scan_partial2(o, dt, n, _p(as_), _p(ys_bar), _p(ws), nbytes, sh, _p(gathered), _p(part2), s,
                                       flags), "vjp_scan_partial2")
            gathered = torch.empty(world * rec, dtype=torch.float64, device=dev)
            _all_gather_into(gathered, part2, group)
    if events:
        events["finish_start"].record()
    _check(L.vjp_scan_finish(o, dt, n, _p(as_), _p(ys_bar), _p(ab), _p(ys), _p(ws), nbytes, sh, _p(gathered), s,
                             flags), "vjp_scan_finish")
    if events:
        events["finish_end"].record()
    return (ab, ys) if want_ys else ab


_CYC: dict = {}


def _cyclic_status(o: int, global_n: int, sb_elems: int, group, dev):
    """this rank's status buffer and every rank's (peer-mapped) pointer to its
    buffer, allocated once per (group, op, sizes) and kept with an epoch
    counter: torch symmetric memory (NVLink peer mappings) for world > 1."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    key = (id(group), o, global_n, sb_elems, str(dev))
    st = _CYC.get(key)
    if st is None:
        nbytes = lib().vjp_scan_cyclic_status_bytes(o, global_n, sb_elems)
        if world == 1:
            buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
            st = {"buf": buf, "ptrs": [buf.data_ptr()], "epoch": 0}
        else:
            if dist.get_backend(group) != "nccl":
                raise RuntimeError("scan_cyclic: the status buffers are peer-mapped device memory (NCCL group, "
                                   "torch symmetric memory); gloo groups use dist.scan")
            import torch.distributed._symmetric_memory as symm
            buf = symm.empty(nbytes, dtype=torch.uint8, device=dev)
            buf.zero_()
            h = symm.rendezvous(buf, group)
            torch.cuda.synchronize(dev)
            h.barrier()
            st = {"buf": buf, "ptrs": list(h.buffer_ptrs), "epoch": 0, "handle": h}
        _CYC[key] = st
    return st


def scan_cyclic(op, ys_bar: torch.Tensor, as_: torch.Tensor | None, *, global_n: int, sb_elems: int | None = None,
                group=None, out: torch.Tensor | None = None, accumulate: bool = False, events: dict | None = None):
    """vjp_scan over this rank's BLOCK-CYCLIC share of a global scan (SURVEY 8f
    row f1; include/vjp.h vjp_scan_cyclic): ys_bar / as_ hold the superblocks
    cyclic_layout(global_n, sb_elems, world, rank) lists, concatenated.  The
    reverse carries cross ranks inside the kernel (NVLink status words, no
    collective); MUL / LINREC / MAT2 all-gather the per-superblock forward
    aggregates first (the forward re-execution's prefix, 8-32 B per superblock)."""
    o = _op(op)
    dev = ys_bar.device
    w = WIDTH[o]
    n = ys_bar.numel() // w
    dt = _dt(ys_bar)
    L = lib()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if sb_elems is None:
        sb_elems = L.vjp_scan_cyclic_sb_elems(o, dt)
    st = _cyclic_status(o, global_n, sb_elems, group, dev)
    st["epoch"] += 1
    cy = VjpCyclic()
    cy.rank, cy.world, cy.global_n, cy.sb_elems, cy.epoch, cy.grid_ctas = rank, world, global_n, sb_elems, st["epoch"], 0
    for q, ptr in enumerate(st["ptrs"]):
        cy.status[q] = ptr
    if n != L.vjp_scan_cyclic_local_n(cy):
        raise ValueError(f"scan_cyclic: rank {rank} holds {n} elements, the layout gives "
                         f"{L.vjp_scan_cyclic_local_n(cy)} (dist.cyclic_layout)")
    ws = workspace(L.vjp_scan_workspace_bytes(o, dt, n), dev)
    nbytes = 0 if ws is None else ws.numel()
    s = _stream(dev)
    gathered = None
    if o != ADD:
        fb = L.vjp_scan_cyclic_fwd_bytes(o, dt, cy) // 8
        sbagg = torch.zeros(fb, dtype=torch.float64, device=dev)
        _check(L.vjp_scan_cyclic_forward(o, dt, n, _p(as_), _p(ws), nbytes, cy, _p(sbagg), s),
               "vjp_scan_cyclic_forward")
        gathered = torch.empty(world * fb, dtype=torch.float64, device=dev)
        if world > 1:
            _all_gather_into(gathered, sbagg, group)
        else:
            gathered.copy_(sbagg)
    ab = out if out is not None else torch.empty_like(ys_bar)
    if events:
        events["finish_start"].record()
    _check(L.vjp_scan_cyclic(o, dt, n, _p(as_), _p(ys_bar), _p(ab), _p(ws), nbytes, cy, _p(gathered), s,
                             ACCUMULATE if accumulate else 0), "vjp_scan_cyclic")
    if events:
        events["finish_end"].record()
    return ab


def scan_cyclic_error(global_n: int, op, sb_elems: int, group=None, dev=None) -> int:
    """word 0 of this rank's status buffer: non-zero if a look-back wait of a
    previous scan_cyclic call timed out (synchronises)."""
    st = _CYC.get((id(group), _op(op), global_n, sb_elems, str(dev)))
    if st is None:
        return 0
    return int(st["buf"][:4].view(torch.int32).item())


def reduce(op, as_: torch.Tensor, y_bar, *, offset: int, global_n: int, group=None, out=None, want_y=False,
           accumulate=False):
    o = _op(op)
    dev = as_.device
    n = as_.numel()
    dt = _dt(as_)
    L = lib()
    sh = _shard(offset, n, global_n, group)
    yb = y_bar.reshape(1).to(device=dev, dtype=as_.dtype) if isinstance(y_bar, torch.Tensor) else torch.full(
        (1,), float(y_bar), dtype=as_.dtype, device=dev)
    ab = out if out is not None else torch.empty_like(as_)
    y = torch.empty(1, dtype=as_.dtype, device=dev) if want_y else None
    arg = torch.empty(1, dtype=torch.int64, device=dev) if want_y else None
    ws = workspace(L.vjp_reduce_workspace_bytes(o, dt, n), dev)
    nbytes = 0 if ws is None else ws.numel()
    rec = L.vjp_reduce_partial_bytes()
    part = torch.empty(rec, dtype=torch.uint8, device=dev)
    s = _stream(dev)
    _check(L.vjp_reduce_partial(o, dt, n, _p(as_), _p(ws), nbytes, sh, _p(part), s), "vjp_reduce_partial")
    gathered = torch.empty(sh.world * rec, dtype=torch.uint8, device=dev)
    if sh.world > 1:
        _all_gather_into(gathered, part, group)
    else:
        gathered.copy_(part)
    _check(L.vjp_reduce_finish(o, dt, n, _p(as_), _p(yb), _p(ab), _p(y), _p(arg), _p(ws), nbytes, sh, _p(gathered),
                               s, ACCUMULATE if accumulate else 0), "vjp_reduce_finish")
    return (ab, y, arg) if want_y else ab


def reduce_by_index(op, inds: torch.Tensor, as_: torch.Tensor | None, hs_bar: torch.Tensor, *, offset: int,
                    global_n: int, group=None, out=None, accumulate=False):
    o = _op(op)
    dev = inds.device
    n, m = inds.numel(), hs_bar.numel()
    dt = _dt(hs_bar)
    it = _it(inds)
    L = lib()
    sh = _shard(offset, n, global_n, group)
    ab = out if out is not None else torch.empty(n, dtype=hs_bar.dtype, device=dev)
    s = _stream(dev)
    bin_val = torch.empty(m, dtype=torch.float64, device=dev)
    bin_aux = torch.empty(m, dtype=torch.int64, device=dev)
    ws = workspace(L.vjp_reduce_by_index_workspace_bytes(o, dt, n, m, 1), dev)
    nbytes = 0 if ws is None else ws.numel()
    if o != 1:  # ADD needs no exchange: hs_bar is replicated
        _check(L.vjp_reduce_by_index_partial(o, dt, it, n, m, _p(inds), _p(as_), _p(ws), nbytes, sh, _p(bin_val),
                                             _p(bin_aux), s), "vjp_reduce_by_index_partial")
        if sh.world > 1:
            if o == 2:  # MUL: the bins' 64-bit code sums (log2|a| fixed point + sign, mod 2^64) and zero counts
                codes = bin_val.view(torch.int64)
                _all_reduce(codes, dist.ReduceOp.SUM, group)
                _all_reduce(bin_aux, dist.ReduceOp.SUM, group)
            else:
                local = bin_val.clone()
                _all_reduce(bin_val, dist.ReduceOp.MAX if o == 4 else dist.ReduceOp.MIN, group)
                _check(L.vjp_reduce_by_index_select(o, m, _p(bin_val), _p(local), _p(bin_aux), s),
                       "vjp_reduce_by_index_select")
                _all_reduce(bin_aux, dist.ReduceOp.MIN, group)
    _check(L.vjp_reduce_by_index_finish(o, dt, it, n, m, _p(inds), _p(as_), _p(hs_bar), _p(ab), _p(bin_val),
                                        _p(bin_aux), _p(ws), nbytes, sh, s, ACCUMULATE if accumulate else 0),
           "vjp_reduce_by_index_finish")
    return ab


def scatter(is_: torch.Tensor, ys_bar: torch.Tensor, *, offset: int, global_n: int, width: int = 1,
            in_place: bool = False, group=None):
    """Adjoints of ys = scatter xs is vs with ys_bar partitioned by rank (this
    rank: global elements [offset, offset + len(ys_bar) / width)); `is_` holds
    the GLOBAL targets on every rank.  Returns (xs_bar_local, vs_bar) with
    vs_bar complete on every rank."""
    dev = ys_bar.device
    ix = is_.to(dev)
    n, m = ys_bar.numel() // width, ix.numel()
    xb = ys_bar if in_place else torch.empty_like(ys_bar)
    vb = torch.empty(m * width, dtype=ys_bar.dtype, device=dev)
    sh = _shard(offset, n, global_n, group)
    _check(lib().vjp_scatter_shard(_dt(ys_bar), _it(ix), n, m, width, _p(ix), _p(ys_bar), _p(xb), _p(vb), sh,
                                   _stream(dev)), "vjp_scatter_shard")
    if sh.world > 1:
        _all_reduce(vb, dist.ReduceOp.SUM, group)
    return xb, vb


def kmeans(points: torch.Tensor, centers: torch.Tensor, cost_bar=1.0, *, group=None, hess: bool = True):
    """config 5 over the ranks: this rank's points (any contiguous slice of the
    global point set), replicated centers; returns the GLOBAL cbar / hdiag /
    counts / cost (all_reduce SUM of the per-rank partials) and this rank's
    assignment."""
    from . import kmeans as _kmeans
    r = _kmeans(points, centers, cost_bar, hess=hess)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        for key in ("cbar", "hdiag", "counts"):
            if r[key] is not None:
                _all_reduce(r[key], dist.ReduceOp.SUM, group)
        c = r["cost"].reshape(1)
        _all_reduce(c, dist.ReduceOp.SUM, group)
    return r
