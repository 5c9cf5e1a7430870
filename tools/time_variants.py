"""Time the config-2 kernels (vjp_scan LINREC and MAT2, n = 2^26 f64) and
reduce_by_index(x) m = 10^3 under each library build given on the command
line (default build = "default"), one subprocess per build; CUDA events,
median of 10 after 3 warm-ups.   python tools/time_variants.py default var_a ..."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    import paper_2202_10297_b200 as vjp
    import synth
    name = sys.argv[2]
    if name != "default":
        vjp.LIB_PATH = os.path.join(ROOT, "paper_2202_10297_b200", "_lib", name + ".so")

    def med(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    n = 1 << 26
    res = {"build": name}
    if os.environ.get("TV_SCAN_ADD"):
        for dt in (torch.float64, torch.float32):
            yb = synth.scan_add_seed(1 << 30, device="cuda").to(dt)
            ob = torch.empty_like(yb)
            res[f"scan_add_2p30_{str(dt)[-7:]}_ms"] = med(lambda: vjp.scan("add", yb, out=ob))
            del yb, ob
    a1, y1 = synth.linrec_inputs(n, device="cuda")
    o1 = torch.empty_like(y1)
    res["linrec_ms"] = med(lambda: vjp.scan("linrec", y1, a1, out=o1))
    del a1, y1, o1
    a2, y2 = synth.mat2_inputs(n, device="cuda")
    o2 = torch.empty_like(y2)
    res["mat2_ms"] = med(lambda: vjp.scan("mat2", y2, a2, out=o2))
    del a2, y2, o2
    am = synth.min_inputs(n, dtype=torch.float64, device="cuda")
    ym = synth.uniform(n, 10, device="cuda")
    om = torch.empty_like(ym)
    for op in ("min", "max"):
        res[f"scan_{op}_2p26_ms"] = med(lambda: vjp.scan(op, ym, am, out=om))
    del am, ym, om
    o = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
    for op in ("mul", "max"):
        inds, a, hb = synth.rbi_inputs(1 << 28, 1000, op, device="cuda")
        res[f"rbi_{op}_1e3_ms"] = med(lambda: vjp.reduce_by_index(op, inds, a, hb, out=o))
        del inds, a, hb
    print(json.dumps(res), flush=True)
else:
    for name in sys.argv[1:] or ["default"]:
        subprocess.run([sys.executable, __file__, "--child", name], check=False)
