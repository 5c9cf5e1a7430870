"""Profiling helper: one vjp_reduce_by_index_general(MUL) call at n = 2^28, m = argv[1]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

inds, a, hb = synth.rbi_inputs(1 << 28, int(sys.argv[1]), "mul", device="cuda")
vjp.reduce_by_index("mul", inds, a, hb, general=True)
torch.cuda.synchronize()
