"""Tuning helper: config-2 operators (LINREC, MAT2 at 2^26 f64) and the other
scan operators on the block look-back vs the chunked kernels (CUDA events,
median of 10 after 3 warm-ups).  Usage: python tools/time_blocklb.py [ops...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_10297_b200 as vjp  # noqa: E402
import synth  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


ops = sys.argv[1:] or ["linrec", "mat2"]
n = 1 << 26
tag = os.environ.get("VJP_LB_L2_MB", "40")
for op in ops:
    if op == "linrec":
        a, yb = synth.linrec_inputs(n, device="cuda")
    elif op == "mat2":
        a, yb = synth.mat2_inputs(n, device="cuda")
    elif op == "add32":
        a, yb = None, synth.scan_add_seed(1 << 30, device="cuda").float()
    elif op == "add64":
        a, yb = None, synth.scan_add_seed(1 << 30, device="cuda")
    elif op in ("min", "mul"):
        a = synth.min_inputs(n, dtype=torch.float64, device="cuda") if op == "min" else \
            synth.mul_inputs(n, dtype=torch.float64, device="cuda")
        yb = synth.uniform(n, 10, device="cuda")
    out = torch.empty_like(yb)
    o = op[:3] if op.startswith("add") else op
    for label, kw in (("blocklb", {"blocklb": True}), ("chunked", {"chunked": True})):
        ms = timeit(lambda: vjp.scan(o, yb, a, out=out, **kw))
        print(f"{op:7s} {label:8s} L2MB={tag:4s} {ms:.3f} ms", flush=True)
    del a, yb, out
