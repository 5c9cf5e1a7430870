"""Profiling helper: one vjp_scan(MIN) f64 call at n = 2^26 (chunked rs-dependent path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

n = 1 << 26
a = synth.min_inputs(n, dtype=torch.float64, device="cuda")
y = synth.uniform(n, 10, device="cuda")
vjp.scan("min", y, a)
torch.cuda.synchronize()
