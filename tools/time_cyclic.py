"""Timing helper for the block-cyclic scan (f1, vjp_scan_cyclic) on ONE GPU:
W virtual ranks (own arrays / workspace / status buffer / stream, grid =
SMs*occ/W CTAs each) run concurrently; the time is the device span from one
start event to the last rank's end (CUDA events), median of 10 after 3
warm-ups.  W = 1 also runs dist.scan_cyclic (one rank, the whole device,
cooperative launch) and the default single-GPU vjp_scan for reference.
  python tools/time_cyclic.py [op] [log2 n] [Ws] [sb_tiles]"""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2202_10297_b200 as vjp
from paper_2202_10297_b200 import dist as vdist

op = sys.argv[1] if len(sys.argv) > 1 else "add"
N = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 30)
Ws = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4,8").split(",")]
L = vjp.lib()
o = vjp.OPS[op]
w = vjp.WIDTH[o]
te = L.vjp_scan_cyclic_tile_elems(o, 2)
sb_default = L.vjp_scan_cyclic_sb_elems(o, 2)
NB = {"add": 16, "mul": 32, "linrec": 64, "mat2": 128}[op]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6543.4
dev = torch.device("cuda")
if op == "add":
    a, yb = None, synth.scan_add_seed(N, device=dev)
elif op == "linrec":
    a, yb = synth.linrec_inputs(N, device=dev)
elif op == "mat2":
    a, yb = synth.mat2_inputs(N, device=dev)
else:
    a, yb = (1.0 + (synth.uniform(N, 7, device=dev) - 0.5) * 2.0 ** -6), synth.uniform(N, 8, device=dev)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = torch.empty_like(yb)
t = timed(lambda: vjp.scan(op, yb, a, out=out))
print(json.dumps({"path": "vjp_scan default (1 GPU)", "op": op, "n": N, "ms": round(t, 4),
                  "frac": round(NB * N / (t * 1e-3) / 1e9 / peak, 3)}), flush=True)
t = timed(lambda: vdist.scan_cyclic(op, yb, a, global_n=N, out=out))
print(json.dumps({"path": "scan_cyclic world=1 (whole device)", "op": op, "n": N, "sb_elems": sb_default,
                  "ms": round(t, 4), "frac": round(NB * N / (t * 1e-3) / 1e9 / peak, 3)}), flush=True)
del out
sms = torch.cuda.get_device_properties(0).multi_processor_count
for W in Ws:
    if W == 1:
        continue
    occ = 3 if op == "add" else 2
    grid = max(1, sms * occ // W)
    tiles = min(8 * grid, max(1, sb_default // te // W))
    sb = te * tiles
    sbytes = L.vjp_scan_cyclic_status_bytes(o, N, sb)
    status = [torch.zeros(sbytes, dtype=torch.uint8, device=dev) for _ in range(W)]
    ranks = []
    for r in range(W):
        spans = vdist.cyclic_layout(N, sb, W, r)
        idx = torch.cat([torch.arange(g0, g0 + ln, device=dev) for g0, ln in spans])
        cy = vjp.VjpCyclic()
        cy.rank, cy.world, cy.global_n, cy.sb_elems, cy.grid_ctas = r, W, N, sb, grid
        for q in range(W):
            cy.status[q] = status[q].data_ptr()
        n_loc = idx.numel()
        rk = dict(cy=cy, n=n_loc, yb=yb.view(N, -1)[idx].reshape(-1).contiguous(),
                  a=None if a is None else a.view(N, -1)[idx].reshape(-1).contiguous(),
                  ab=torch.empty(n_loc * w, dtype=torch.float64, device=dev),
                  ws=vjp.workspace(L.vjp_scan_workspace_bytes(o, 2, n_loc), dev), s=torch.cuda.Stream())
        del idx
        ranks.append(rk)
    fb = L.vjp_scan_cyclic_fwd_bytes(o, 2, ranks[0]["cy"]) // 8
    ep = [0]

    def step():
        ep[0] += 1
        cur = torch.cuda.current_stream()
        gathered = None
        if op != "add":
            parts = []
            for rk in ranks:
                rk["cy"].epoch = ep[0]
                sbagg = torch.zeros(fb, dtype=torch.float64, device=dev)
                assert L.vjp_scan_cyclic_forward(o, 2, rk["n"], vjp._p(rk["a"]), vjp._p(rk["ws"]), rk["ws"].numel(),
                                                 rk["cy"], vjp._p(sbagg), vjp._stream(dev)) == 0
                parts.append(sbagg)
            gathered = torch.cat(parts)
        for rk in ranks:
            rk["cy"].epoch = ep[0]
            rk["s"].wait_stream(cur)
        for rk in ranks:
            assert L.vjp_scan_cyclic(o, 2, rk["n"], vjp._p(rk["a"]), vjp._p(rk["yb"]), vjp._p(rk["ab"]),
                                     vjp._p(rk["ws"]), rk["ws"].numel(), rk["cy"], vjp._p(gathered),
                                     ctypes.c_void_p(rk["s"].cuda_stream), 0) == 0
        for rk in ranks:
            cur.wait_stream(rk["s"])

    t = timed(step)
    errs = [int(s_[:4].view(torch.int32).item()) for s_ in status]
    print(json.dumps({"path": f"scan_cyclic {W} virtual ranks on one GPU", "op": op, "n": N, "sb_elems": sb,
                      "grid_per_rank": grid, "ms": round(t, 4), "frac": round(NB * N / (t * 1e-3) / 1e9 / peak, 3),
                      "timeouts": errs}), flush=True)
    del ranks, status
    torch.cuda.empty_cache()
