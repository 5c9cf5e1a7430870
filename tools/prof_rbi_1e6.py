"""Profiling helper: one call each of vjp_reduce_by_index +, x, max at config 4
(n = 2^28 f64, m = 10^6, uniform int32 bins) plus the L2 calibration kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
import bench
dev = torch.device("cuda")
for op in ("add", "mul", "max"):
    inds, a, hb = synth.rbi_inputs(1 << 28, 1_000_000, op, device=dev)
    o = torch.empty(1 << 28, dtype=torch.float64, device=dev)
    vjp.reduce_by_index(op, inds, a, hb, out=o)
    torch.cuda.synchronize()
    if op == "add":
        bench.l2_ceilings(inds, 1_000_000, dev)
    del inds, a, hb, o
