#!/usr/bin/env python
"""bench.py — vjp elements/s and achieved HBM GB/s on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[1], the config the metric is quoted on
for one GPU): the vjp of scan with the 2x2 linear-recurrence (LINREC) and the
2x2 matrix-multiply (MAT2) operators, n = 2^26 elements per operator, f64.  One
STEP = one whole pass of the hot path over one batch: vjp_scan(LINREC) then
vjp_scan(MAT2) (forward re-execution + return sweep each).  With N GPUs each
rank owns a contiguous 2^26-element shard of each scan (weak scaling) and the
shards exchange their per-shard Jacobian aggregates by all_gather (the path's
one real exchange step).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                  [--workload config2|scan_add|reduce|rbi]

Prints ONE JSON line (rank 0).  Inputs (>= 1 GiB per array) are far larger than
the 126 MB L2, so no flush is needed between steps.  --impl reference times the
oracle (the plain CPU definition, oracle/) on bounded samples of the same
workload.  Other --workload values print extra lines for DESIGN.md, not the
headline.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "vjp elements/s (scan LINREC+MAT2 n=2^26 f64 per GPU)"
UNIT = "elements/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    (in-process, every 2 ms, so even a ~50 ms region gets many samples), else
    an nvidia-smi -lms subprocess started (and waited for) before the region."""

    NAMES = {"hw_slowdown": "HwSlowdown", "hw_thermal_slowdown": "HwThermalSlowdown",
             "sw_thermal_slowdown": "SwThermalSlowdown", "sw_power_cap": "SwPowerCap",
             "hw_power_brake_slowdown": "HwPowerBrakeSlowdown"}
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []  # (sm_mhz, max_mhz, set of reason names)
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.src = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = (pynvml, h)
            self.src = "nvml"
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.src = "nvidia-smi"
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._smi_read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10:  # first sample before the region starts
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _nvml_loop(self):
        pynvml, h = self.nvml
        while not self.stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                act = {k for k, v in self.NAMES.items() if r & getattr(pynvml, "nvmlClocksEventReason" + v, 0)}
                self.rows.append((float(sm), float(mx), act))
            except Exception:
                pass
            self.stop.wait(0.002)

    def _smi_read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                act = {names[i] for i in range(4) if len(r) > 3 + i and r[3 + i].lower().startswith("active")}
                self.rows.append((float(r[0]), float(r[1]), act))
            except ValueError:
                pass

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "source": self.src}
        sm = [r[0] for r in self.rows]
        reasons = sorted(set().union(*[r[2] for r in self.rows]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": self.src}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info():
    """the box's host CPU (lscpu model name) and core count, for cpu_baseline"""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    if model is None:
        try:
            for ln in open("/proc/cpuinfo"):
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
        except Exception:
            pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_oracle_sample(n: int, reps: int = 1):
    """oracle (plain CPU definition, one thread) on LINREC+MAT2 samples of n
    elements, the calling thread pinned to one core (sched_setaffinity, the
    in-process equivalent of taskset -c) and timed with a monotonic clock
    (time.perf_counter, like std::chrono::steady_clock)."""
    import oracle
    import synth
    a1, y1 = synth.linrec_inputs(n)
    a2, y2 = synth.mat2_inputs(n)
    a1, y1, a2, y2 = a1.numpy(), y1.numpy(), a2.numpy(), y2.numpy()
    old = None
    try:
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(old)})
    except Exception:
        old = None
    try:
        t0 = time.perf_counter()
        for _ in range(reps):
            oracle.vjp_scan("linrec", y1, a1)
            oracle.vjp_scan("mat2", y2, a2)
        dt = (time.perf_counter() - t0) / reps
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return 2 * n / dt, dt


# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    n = 1 << 22  # bounded sample per step: 2 x 2^22 elements (~1.6 s of one core)
    times = []
    for i in range(args.warmup + args.steps):
        v, dt = cpu_oracle_sample(n)
        if i >= args.warmup:
            times.append(dt)
    mean = statistics.mean(times)
    val = 2 * n / mean
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seed 2202)",
        "config": {"workload": "configs[1]: vjp_scan LINREC + MAT2, n = 2^26 elements per op per GPU, f64",
                   "ops": ["linrec", "mat2"], "parallelism": "1 CPU thread (the oracle)",
                   "sample": f"bounded: each step runs n = 2^22 elements per op ({n} of the 2^26), "
                             "the metric is per element so it is comparable"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"LINREC+MAT2 n=2^22 each per step, {args.steps} steps, one thread pinned to "
                                   "one core", **host_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def measure_targets(args, dev, peak):
    """The north_star target kernels (BASELINE.json: vjp_scan + and the 2x2
    linear recurrence at 2^30 f64, vjp_reduce_by_index +/x/max at n = 2^28 with
    m = 10^3 and 10^6), each timed alone on one GPU: CUDA events around each
    call on the launching stream, median over `steps` calls after `warmup`,
    NVML clocks sampled during that target's own timed region.  Method bytes
    per element: scan(+) 16, LINREC 64 (forward re-execution reads
    `as` once more), rbi + 12, x 32, max 20.  Inputs >= 2 GiB per array (no L2
    flush needed); each target's arrays are freed before the next."""
    import torch

    import paper_2202_10297_b200 as vjp
    import synth

    steps = max(5, min(args.steps, 10))
    out = []

    def one(name, workload, n, nbytes, fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        with ClockSampler(dev.index) as clk:
            for e0, e1 in ev:
                e0.record()
                fn()
                e1.record()
            torch.cuda.synchronize()
        ts = [a.elapsed_time(b) for a, b in ev]
        ms = statistics.median(ts)
        gbs = nbytes / (ms * 1e-3) / 1e9
        out.append({"name": name, "workload": workload, "n": n, "ms": ms, "mean_ms": statistics.mean(ts),
                    "min_ms": min(ts), "steps": steps, "elements_per_s": n / (ms * 1e-3),
                    "method_bytes": nbytes, "alg_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
                    "clocks": clk.summary()})

    N30, N28 = 1 << 30, 1 << 28
    yb = synth.scan_add_seed(N30, device=dev)
    ab = torch.empty_like(yb)
    one("scan(+) f64 2^30", "vjp_scan ADD, n = 2^30 f64 (config 1 at the target size)", N30, 16 * N30,
        lambda: vjp.scan("add", yb, out=ab))
    del yb, ab
    a, yb = synth.linrec_inputs(N30, device=dev)
    ab = torch.empty_like(yb)
    one("LINREC f64 2^30", "vjp_scan LINREC, n = 2^30 f64", N30, 64 * N30,
        lambda: vjp.scan("linrec", yb, a, out=ab))
    del a, yb, ab
    l2 = None
    for m in (1000, 1_000_000):
        for op, nb in (("add", 12), ("mul", 32), ("max", 20)):
            inds, a, hb = synth.rbi_inputs(N28, m, op, device=dev)
            o = torch.empty(N28, dtype=torch.float64, device=dev)
            if m == 1_000_000 and l2 is None:
                l2 = l2_ceilings(inds, m, dev)
            one(f"rbi {op} m={m}", f"vjp_reduce_by_index {op.upper()}, n = 2^28 f64, int32 bins, m = {m} "
                "(config 4, uniform bins)", N28, nb * N28,
                lambda op=op, inds=inds, a=a, hb=hb, o=o: vjp.reduce_by_index(op, inds, a, hb, out=o))
            if m == 1_000_000:
                # L2-bound (every access a random 32-byte sector in an 8-16 MB
                # table): the L2 budget of the call at the CALIBRATED rates —
                # random gathers and f64 reductions as timed by vjp_calib_* (each
                # including its 4 B bin stream), plus the other streamed bytes
                # as 32-byte sectors at the calibrated sector rate.  Per element:
                # +: 1 gather, 8 B more (as_bar); x: 1 reduction (forward) + 1
                # gather (return), 24 B more (as twice, as_bar); max: 1 gather
                # (the filter read; its reductions are rare), 16 B more (as,
                # the fused zero-fill of as_bar).
                g, r, extra = {"add": (1, 0, 8), "mul": (1, 1, 24), "max": (1, 0, 16)}[op]
                bound = g * l2["gather_ms"] + r * l2["red_ms"] + (extra / 32) * N28 / l2["sectors_per_ms"]
                out[-1]["l2_bound_ms"] = bound
                out[-1]["frac_l2"] = bound / out[-1]["ms"]
            del inds, a, hb, o
    out.append({"name": "L2 ceilings (calibration)", **l2})
    torch.cuda.empty_cache()
    return out


def l2_ceilings(inds, m, dev):
    """calibration (vjp_calib_*): 2^28 random 8-byte gathers / f64 red.adds
    into an m-entry (8 MB at m = 10^6) L2-resident table, bins streamed as in
    the histogram kernels; CUDA events, median of 5 after 2 warm-ups."""
    import torch

    import paper_2202_10297_b200 as vjp

    L = vjp.lib()
    n = inds.numel() - inds.numel() % 4
    table = torch.ones(m, dtype=torch.float64, device=dev)
    olen = L.vjp_calib_out_len()
    outb = torch.empty(olen, dtype=torch.float64, device=dev)
    res = {}
    for name, fn in (("gather_ms", lambda: L.vjp_calib_l2_gather(vjp._p(table), vjp._p(inds), n, vjp._p(outb), olen,
                                                                 vjp._stream(dev))),
                     ("red_ms", lambda: L.vjp_calib_l2_red(vjp._p(table), vjp._p(inds), n, vjp._stream(dev)))):
        for _ in range(2):
            assert fn() == 0
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert fn() == 0
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = statistics.median(ts)
    res.update({"n": n, "m": m, "gathers_per_s": n / (res["gather_ms"] * 1e-3),
                "reds_per_s": n / (res["red_ms"] * 1e-3),
                # algorithmic L2 sectors of the gather calibration: one per
                # gather + its 4 B bin (1/8 sector)
                "sectors_per_ms": 1.125 * n / res["gather_ms"],
                "ncu_note": "ncu (profiles/r02_rbi1e6_launches.csv): the gather calibration runs at 80.4 % of "
                            "lts__throughput, the reduction one at 78.7 %"})
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2202_10297_b200 as vjp
    from paper_2202_10297_b200 import dist as vdist
    import synth

    world, rank, local = dist_env()
    assert world == args.gpus or world == 1, "--gpus must match WORLD_SIZE"
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    backend = os.environ.get("VJP_DIST_BACKEND", "nccl")  # gloo: test several ranks on one GPU
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    vjp.lib()

    n = args.n or (1 << 26)
    gN = n * world
    off = rank * n
    ops = ["linrec", "mat2"]
    gens = {"linrec": synth.linrec_inputs, "mat2": synth.mat2_inputs}
    data = {}
    for op in ops:
        a, yb = gens[op](n, offset=off, device=dev)
        data[op] = (a, yb, torch.empty_like(yb))
    torch.cuda.synchronize()

    def mk():
        return {op: {"finish_start": torch.cuda.Event(enable_timing=True),
                     "finish_end": torch.cuda.Event(enable_timing=True)} for op in ops}

    def step(evs=None):
        for op in ops:
            a, yb, ab = data[op]
            vdist.scan(op, yb, a, offset=off, global_n=gN, out=ab, events=evs[op] if evs else None)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # --- timed region (device time, CUDA events on the launching stream) ---
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kev = [mk() for _ in range(args.steps)]
    launches0 = vjp.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local % ndev) as clk:
        for i in range(args.steps):
            starts[i].record()
            step(kev[i])
            ends[i].record()
        torch.cuda.synchronize()
    k_mat2 = [e["mat2"]["finish_start"].elapsed_time(e["mat2"]["finish_end"]) for e in kev]
    k_lin = [e["linrec"]["finish_start"].elapsed_time(e["linrec"]["finish_end"]) for e in kev]
    launches = vjp.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    mean_ms = statistics.mean(step_ms)
    t = torch.tensor([mean_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    mean_ms = float(t.item())

    # --- end to end through the public API with host buffers ---
    e2e = None
    if not args.no_e2e:
        host = {}
        for op in ops:
            a, yb, ab = data[op]
            host[op] = (a.cpu().pin_memory(), yb.cpu().pin_memory(), torch.empty(ab.shape, dtype=ab.dtype,
                                                                                  pin_memory=True))
        h2d = sum(h[0].numel() * h[0].element_size() + h[1].numel() * h[1].element_size() for h in host.values())
        d2h = sum(h[2].numel() * h[2].element_size() for h in host.values())
        e2e_steps = max(1, min(16, args.steps))  # steady state: fill / drain amortised
        for op in ops:  # warm
            vjp.scan(op, host[op][1], host[op][0], out=host[op][2])
            if world == 1:
                vjp.scan(op, host[op][1], host[op][0], out=host[op][2], sync=False).wait()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pend = []
        for _ in range(e2e_steps):
            for op in ops:
                if world > 1:
                    a_d = host[op][0].to(dev, non_blocking=True)
                    y_d = host[op][1].to(dev, non_blocking=True)
                    ab_d = vdist.scan(op, y_d, a_d, offset=off, global_n=gN)
                    host[op][2].copy_(ab_d, non_blocking=True)
                    torch.cuda.synchronize()
                else:
                    # the public API's asynchronous host-buffer call: copy-in,
                    # kernels and copy-out on their own streams, so one call's
                    # copy-out overlaps the next call's copy-in (full-duplex PCIe)
                    pend.append(vjp.scan(op, host[op][1], host[op][0], out=host[op][2], sync=False))
                    if len(pend) > 4:  # a bounded window of calls in flight (device memory stays bounded)
                        pend.pop(0).wait()
        for p_ in pend:
            p_.wait()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = float(te.item())
        e2e = {"value": 2 * gN / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
               "path": "vjp.scan on pinned host buffers" + (", sync=False: copy-in / kernels / copy-out on three "
                                                           "streams, consecutive calls overlapped" if world == 1
                                                           else " via dist.scan, synchronous")}

    if rank == 0:
        peak, peak_src = peaks()
        kmat2 = statistics.mean(k_mat2)
        alg_bytes = 96 * n  # MAT2 return sweep: read A 32 B + ybar 32 B, write abar 32 B per element
        achieved = alg_bytes / (kmat2 * 1e-3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("scan_apply_mat2_f64_n2^26") if n == (1 << 26) else None
            except Exception:
                traffic = None
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, dt = cpu_oracle_sample(1 << 23)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                   "sample": "LINREC + MAT2, n = 2^23 each, one pass of the oracle (one host thread pinned "
                             "to one core)", **host_info()}
        line = {
            "metric": METRIC, "value": 2 * gN / (mean_ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seed 2202)",
            "config": {"workload": "configs[1]: vjp_scan LINREC + MAT2, n = 2^26 elements per op per GPU, f64",
                       "n_per_op_per_gpu": n, "global_n_per_op": gN, "ops": ops,
                       "parallelism": f"contiguous shards x{world}, all_gather of shard aggregates"
                                      + ("" if world == 1 else f" ({backend})"),
                       "l2": "no flush: every array >= 1 GiB >> 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "scan_apply<OpMat2,f64> (MAT2 return sweep, chunked)",
                         "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": kmat2,
                         "peak_source": peak_src,
                         "peak_note": "the peak is a 1:1 read:write copy (MEASURED_PEAKS.json); this kernel reads "
                                      "2 bytes per byte written, a mix the HBM serves faster, so frac can exceed 1",
                         "linrec_apply_ms": statistics.mean(k_lin),
                         "linrec_apply_gbs": 48 * n / (statistics.mean(k_lin) * 1e-3) / 1e9,
                         "step_alg_gbs": (64 + 128) * n / (mean_ms * 1e-3) / 1e9},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_targets:
            for op in ops:  # free the headline arrays first
                data[op] = None
            torch.cuda.empty_cache()
            line["targets"] = measure_targets(args, dev, peak)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_extra(args):
    """Extra lines for DESIGN.md/BASELINE.md (not the headline): each vjp call of
    configs 1-4 timed alone with CUDA events (median over steps)."""
    import torch

    import paper_2202_10297_b200 as vjp
    import synth

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    vjp.lib()
    peak, peak_src = peaks()
    def run_case(name, n, nbytes, fn):
        # each case runs as soon as it is defined, so its inputs can be freed
        # before the next case allocates
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(json.dumps({"extra": name, "n": n, "ms": ms, "elements_per_s": n / (ms * 1e-3),
                          "alg_bytes": nbytes, "alg_gbs": nbytes / (ms * 1e-3) / 1e9,
                          "frac_of_peak": nbytes / (ms * 1e-3) / 1e9 / peak, "peak": peak,
                          "min_ms": min(ts)}), flush=True)

    class _Cases:
        def append(self, case):
            run_case(*case)

    cases = _Cases()
    N30, N28, N26 = 1 << 30, 1 << 28, 1 << 26
    w = args.workload
    if w in ("scan_add", "all"):
        yb = synth.scan_add_seed(N30, device=dev)
        out = torch.empty_like(yb)
        cases.append(("scan ADD f64 n=2^30 (target; default = one pass, two-level look-back)", N30, 16 * N30,
                      lambda yb=yb, out=out: vjp.scan("add", yb, out=out)))
        cases.append(("scan ADD f64 n=2^30 chunked kernels (24 B moved)", N30, 16 * N30,
                      lambda yb=yb, out=out: vjp.scan("add", yb, out=out, chunked=True)))
        cases.append(("scan ADD f64 n=2^30 look-back kernels", N30, 16 * N30,
                      lambda yb=yb, out=out: vjp.scan("add", yb, out=out, lookback=True)))
        yb = out = None
        yf = synth.scan_add_seed(N30, device=dev).float()
        of = torch.empty_like(yf)
        cases.append(("scan ADD f32 n=2^30 (8 B/elem)", N30, 8 * N30,
                      lambda yf=yf, of=of: vjp.scan("add", yf, out=of)))
        yf = of = None
    yb = out = None
    if w in ("scan_linrec30", "all"):
        a, yb2 = synth.linrec_inputs(N30, device=dev)
        out2 = torch.empty_like(yb2)
        cases.append(("scan LINREC f64 n=2^30", N30, 64 * N30,
                      lambda yb2=yb2, a=a, out2=out2: vjp.scan("linrec", yb2, a, out=out2)))
    a = yb2 = out2 = None
    if w in ("reduce", "all"):
        for z in ("none", "one", "two", "sparse"):
            a = synth.mul_inputs(N30, zeros=z, dtype=torch.float32, device=dev)
            o = torch.empty_like(a)
            nb = (12 if z == "none" else 8) * N30
            cases.append((f"reduce MUL f32 n=2^30 zeros={z}", N30, nb,
                          (lambda a=a, o=o: vjp.reduce("mul", a, 1.0, out=o))))
        a = synth.min_inputs(N30, dtype=torch.float32, device=dev)
        o = torch.empty_like(a)
        cases.append(("reduce MIN f32 n=2^30 dense", N30, 8 * N30,
                      lambda a=a, o=o: vjp.reduce("min", a, 1.5, out=o)))
        cases.append(("reduce MIN f32 n=2^30 accumulate", N30, 4 * N30,
                      lambda a=a, o=o: vjp.reduce("min", a, 1.5, out=o, accumulate=True)))
        cases.append(("reduce ADD f32 n=2^30 (broadcast of ybar, 4 B/elem)", N30, 4 * N30,
                      lambda a=a, o=o: vjp.reduce("add", a, 1.5, out=o)))
        del a
        # scatter (a14): m = 2^24 distinct targets into n = 2^28 f64, in place (O(m):
        # gather 8 B + zero 8 B + index 8 B + vs_bar 8 B per target)
        is_, ybs = synth.scatter_inputs(N28, 1 << 24, device=dev)
        vs = torch.empty(1 << 24, dtype=torch.float64, device=dev)
        cases.append(("scatter in place f64 n=2^28 m=2^24 (32 B/target)", 1 << 24, 32 * (1 << 24),
                      lambda is_=is_, ybs=ybs, vs=vs: vjp.scatter(is_, ybs, in_place=True, vs_out=vs)))
        # the in-place update's forward save + restore: per target
        # index 8 B, xs read 8 B, xs_saved 8 B written, vs 8 B read, xs 8 B written;
        # then restore: index 8 B, xs_saved 8 B, xs 8 B
        saved = torch.empty(1 << 24, dtype=torch.float64, device=dev)
        cases.append(("scatter forward save + restore f64 n=2^28 m=2^24 (64 B/target)", 1 << 24, 64 * (1 << 24),
                      lambda is_=is_, ybs=ybs, vs=vs, saved=saved: vjp.scatter_restore(
                          ybs, is_, vjp.scatter_forward(ybs, is_, vs, saved_out=saved))))
        # MIN scan (pick-left subgradient; the reverse maps need rs: K_F + K_R' + K_C)
        am = synth.min_inputs(N26, dtype=torch.float64, device=dev)
        ym = synth.uniform(N26, 10, device=dev)
        omn = torch.empty_like(ym)
        cases.append(("scan MIN f64 n=2^26 (chunked rs-dependent path, 24 B/elem method)", N26, 24 * N26,
                      lambda am=am, ym=ym, omn=omn: vjp.scan("min", ym, am, out=omn)))
    o = am = ym = omn = is_ = ybs = vs = None
    if w in ("rbi", "all"):
        for skew in (False, True):  # bins uniform over m, or skewed (floor(m u^2): a heavy head)
            for m in (1000, 1_000_000):
                for op, nb in (("add", 12), ("mul", 32), ("max", 20)):
                    inds = a = hb = None
                    inds, a, hb = synth.rbi_inputs(N28, m, op, device=dev, skew=skew)
                    o = torch.empty(N28, dtype=torch.float64, device=dev)
                    cases.append((f"rbi {op.upper()} f64 n=2^28 m={m}{' skewed bins' if skew else ''}", N28, nb * N28,
                                  (lambda op=op, inds=inds, a=a, hb=hb, o=o: vjp.reduce_by_index(op, inds, a, hb, out=o))))
            # the general rule: counting sort + per-bin product scans
            if not skew:
                for m in (1000, 1_000_000):
                    inds = a = hb = None
                    inds, a, hb = synth.rbi_inputs(N28, m, "mul", device=dev)
                    o = torch.empty(N28, dtype=torch.float64, device=dev)
                    cases.append((f"rbi MUL f64 n=2^28 m={m} general rule (sort + segmented scans)", N28, 32 * N28,
                                  (lambda inds=inds, a=a, hb=hb, o=o: vjp.reduce_by_index("mul", inds, a, hb, out=o,
                                                                                          general=True))))
        inds = a = hb = o = None
    if w in ("batched", "all"):
        # vectorised scans: ADD 2^20 x 64, LINREC 2^20 x 32 (f64)
        ya = synth.scan_add_seed((1 << 20) * 64, device=dev)
        oa = torch.empty_like(ya)
        cases.append(("batched scan ADD f64 n=2^20 w=64", (1 << 20) * 64, 16 * (1 << 20) * 64,
                      lambda ya=ya, oa=oa: vjp.scan_batched("add", ya, width=64, out=oa)))
        al, yl = synth.linrec_inputs((1 << 20) * 32, device=dev)
        ol = torch.empty_like(yl)
        cases.append(("batched scan LINREC f64 n=2^20 w=32", (1 << 20) * 32, 64 * (1 << 20) * 32,
                      lambda al=al, yl=yl, ol=ol: vjp.scan_batched("linrec", yl, al, width=32, out=ol)))
        # general reduce rule: MAT2 reduce, n = 2^26 f64 (as read twice + as_bar: 96 B/elem)
        am, _ = synth.mat2_inputs(N26, device=dev)
        om = torch.empty_like(am)
        ybm = torch.tensor([1.0, 0.5, -0.5, 2.0], dtype=torch.float64, device=dev)
        cases.append(("general reduce MAT2 f64 n=2^26", N26, 96 * N26,
                      lambda am=am, om=om, ybm=ybm: vjp.reduce("mat2", am, ybm, out=om)))
    if w == "call":
        # one vjp call from the flags (method bytes as in SURVEY 8d / DESIGN 7)
        n = args.n or (1 << 28)
        td = torch.float64 if args.dtype == "f64" else torch.float32
        es = 8 if args.dtype == "f64" else 4
        width = {"linrec": 2, "mat2": 4}.get(args.op, 1)
        if args.kind == "scan":
            gen = {"linrec": synth.linrec_inputs, "mat2": synth.mat2_inputs}
            if args.op in gen:
                a, yb = gen[args.op](n, dtype=td, device=dev)
            elif args.op == "add":
                a, yb = None, synth.scan_add_seed(n, dtype=td, device=dev)
            elif args.op in ("min", "max"):
                a, yb = synth.min_inputs(n, dtype=td, device=dev), synth.uniform(n, 10, dtype=td, device=dev)
            else:
                a = (1.0 + (synth.uniform(n, 7, device=dev) - 0.5) * 2.0 ** -6).to(td)
                yb = synth.uniform(n, 8, dtype=td, device=dev)
            out = torch.empty_like(yb)
            # method bytes: ADD 2 arrays; MUL/LINREC/MAT2 4 (as read by the forward
            # re-execution and the return sweep); MIN/MAX 3 (as the round-1 lines count them)
            nb = (2 if args.op == "add" else (3 if args.op in ("min", "max") else 4)) * width * es
            cases.append((f"scan {args.op.upper()} {args.dtype} n={n}", n, nb * n,
                          lambda: vjp.scan(args.op, yb, a, out=out)))
        elif args.kind == "reduce":
            if args.op == "mul":
                a = synth.mul_inputs(n, dtype=td, device=dev)
            elif args.op in ("min", "max"):
                a = synth.min_inputs(n, dtype=td, device=dev)
            else:
                a = synth.uniform(n * width, 5, dtype=td, device=dev)
            out = torch.empty_like(a)
            nb = {"add": 1, "mul": 3, "min": 2, "max": 2}.get(args.op, 3) * width * es
            ybar = 1.0 if width == 1 else torch.ones(width, dtype=td, device=dev)
            cases.append((f"reduce {args.op.upper()} {args.dtype} n={n}", n, nb * n,
                          lambda: vjp.reduce(args.op, a, ybar, out=out)))
        else:
            inds, a, hb = synth.rbi_inputs(n, args.m, args.op, dtype=td, device=dev)
            out = torch.empty(n, dtype=td, device=dev)
            nb = {"add": 4 + es, "mul": 4 + 3 * es, "max": 4 + 2 * es, "min": 4 + 2 * es}[args.op]
            cases.append((f"rbi {args.op.upper()} {args.dtype} n={n} m={args.m}", n, nb * n,
                          lambda: vjp.reduce_by_index(args.op, inds, a, hb, out=out)))
    if w in ("kmeans", "all"):
        # config 5: n = 10^6 points, d = 64, k = 1024, f64 (one call: forward
        # distance/argmin on the FP64 tensor pipe + the return sweep)
        nk, kk, dk = 1_000_000, 1024, 64
        P, C = synth.kmeans_inputs(nk, kk, dk, device=dev)
        out = vjp.kmeans(P, C, 1.0)
        cases.append((f"kmeans grad n=1e6 k=1024 d=64 f64 (flops {2 * nk * kk * dk:.3g})", nk,
                      nk * dk * 8 * 2, lambda P=P, C=C, out=out: vjp.kmeans(P, C, 1.0, out=out)))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override elements per op per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-targets", action="store_true", help="skip the north_star target kernels (1 GPU)")
    ap.add_argument("--workload", default="config2",
                    choices=["config2", "scan_add", "scan_linrec30", "reduce", "rbi", "kmeans", "batched", "call",
                             "all"],
                    help="config2 = the headline line; the others print per-call extra lines; call = one vjp "
                         "call chosen by --kind/--op/--dtype/--n/--m")
    ap.add_argument("--kind", default="scan", choices=["scan", "reduce", "rbi"], help="--workload call: combinator")
    ap.add_argument("--op", default="add", choices=["add", "mul", "min", "max", "linrec", "mat2"],
                    help="--workload call: operator")
    ap.add_argument("--dtype", default="f64", choices=["f32", "f64"], help="--workload call: value dtype")
    ap.add_argument("--m", type=int, default=1000, help="--workload call, rbi: bins")
    ap.add_argument("--seed", type=int, default=2202, help="synthetic-input seed (synth.set_seed)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.seed != 2202:
        import synth
        synth.set_seed(args.seed)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "config2":
        return run_extra(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
