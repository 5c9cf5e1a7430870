"""Host<->device copy bandwidth of this box (pinned memory, CUDA events).

The bound of bench.py's `e2e` leg: every config-2 step copies 6.44 GB in and
3.22 GB out over PCIe.  Prints one JSON line per case:
  h2d alone, d2h alone, h2d + d2h concurrently on two streams (full duplex),
  h2d split in 4 pieces on one stream (per-copy overhead).
"""
import json

import torch


def main():
    dev = torch.device("cuda", 0)
    nb = 2 << 30
    h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    h_in.fill_(1)
    d_a = torch.empty(nb, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nb, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn, reps=3):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best

    def h2d():
        d_a.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_b, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream(dev)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    def h2d4():
        q = nb // 4
        for i in range(4):
            d_a[i * q:(i + 1) * q].copy_(h_in[i * q:(i + 1) * q], non_blocking=True)

    def h2d_2s():  # two halves on two streams (two copy engines?)
        cur = torch.cuda.current_stream(dev)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        q = nb // 2
        with torch.cuda.stream(s1):
            d_a[:q].copy_(h_in[:q], non_blocking=True)
        with torch.cuda.stream(s2):
            d_a[q:].copy_(h_in[q:], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for name, fn, bytes_ in (("h2d", h2d, nb), ("d2h", d2h, nb), ("h2d+d2h concurrent", both, 2 * nb),
                             ("h2d 4 pieces", h2d4, nb), ("h2d 2 streams", h2d_2s, nb)):
        ms = timed(fn)
        print(json.dumps({"case": name, "bytes": bytes_, "ms": ms, "GB/s": bytes_ / ms / 1e6}))


if __name__ == "__main__":
    main()
