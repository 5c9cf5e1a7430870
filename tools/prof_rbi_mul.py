"""Profiling helper: two calls of vjp_reduce_by_index(*) at config 4 (n = 2^28, m = 10^3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2202_10297_b200 as vjp
inds, a, hb = synth.rbi_inputs(1 << 28, 1000, "mul", itype=torch.int32, device="cuda")
for _ in range(2):
    vjp.reduce_by_index("mul", inds, a, hb)
torch.cuda.synchronize()
