"""Tuning helper: per-block timeline of the block look-back (vjp_debug_lb_trace)
for one call at n = 2^26 f64.  Prints the distribution of the R phase, the
look-back walk, the wait for the carry and the A phase (microseconds)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "mat2"
n = 1 << 26
a, yb = (synth.linrec_inputs if op == "linrec" else synth.mat2_inputs)(n, device="cuda")
L = vjp.lib()
L.vjp_debug_lb_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros(8 * 200000, dtype=torch.int64, device="cuda")
for _ in range(2):
    vjp.scan(op, yb, a, blocklb=True)
buf.zero_()
L.vjp_debug_lb_trace(ctypes.c_void_p(buf.data_ptr()))
vjp.scan(op, yb, a, blocklb=True)
torch.cuda.synchronize()
L.vjp_debug_lb_trace(None)
tr = buf.cpu().numpy().reshape(-1, 8)
tr = tr[tr[:, 5] > 0]
t0 = tr[:, 2].min()
lb0, lb1, r0, r1, a0, a1 = [(tr[:, i] - t0) / 1e3 for i in (0, 1, 2, 3, 4, 5)]
q = lambda x: f"p10 {np.percentile(x, 10):7.2f} p50 {np.percentile(x, 50):7.2f} p90 {np.percentile(x, 90):7.2f}"
print(f"{op}: blocks {len(tr)}, span {(a1.max()):.1f} us")
print("R phase        ", q(r1 - r0))
print("look-back walk ", q(lb1 - lb0), " windows", q(tr[:, 7].astype(float)))
print("walk start-R0  ", q(lb0 - r0))
print("walk end - R end", q(lb1 - r1))
print("wait for X     ", q(a0 - r1))
print("A phase        ", q(a1 - a0))
print("block total    ", q(a1 - r0))
# per-CTA gap between blocks
order = np.lexsort((r0, tr[:, 6]))
cta, rs, ae = tr[order, 6], r0[order], a1[order]
same = cta[1:] == cta[:-1]
print("gap A end->next R start", q((rs[1:] - ae[:-1])[same]))
