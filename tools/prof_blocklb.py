"""Profiling helper: one block look-back vjp_scan call per operator at n = 2^26
f64 (argv: operators, default linrec mat2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

n = 1 << 26
for op in sys.argv[1:] or ["linrec", "mat2"]:
    a, yb = (synth.linrec_inputs if op == "linrec" else synth.mat2_inputs)(n, device="cuda")
    vjp.scan(op, yb, a, blocklb=True)
    torch.cuda.synchronize()
    del a, yb
