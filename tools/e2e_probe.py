#!/usr/bin/env python3
"""Where does the end-to-end C4 step time go?  Runs K pipelined host steps (the bench's e2e
loop) and prints: wall ms/step, the host time spent inside each API call, and the device
time per step between compute-stream events; then the same loop with device-resident inputs
and outputs (no copies) for comparison."""
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import F16, Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    sc = Scenario("C4")
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    p = 1.0 / (2.0 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    nb = 4
    host = [sc.batch(b) for b in range(nb)]
    pinned = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()) for x, y in host]
    devb = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in host]
    outs = [torch.empty((R, C), dtype=torch.uint8).pin_memory() for _ in range(2)]
    ldev = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp = Mapper(D, 0, l, sc.bounds)
    calls = {"enc": 0.0, "dec": 0.0, "ent": 0.0, "wait": 0.0}
    hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
    use_enc_stream = len(sys.argv) > 2 and sys.argv[2] == "pipe"
    torch.cuda.set_stream(hi)
    if use_enc_stream:
        mp.set_encode_stream(lo)

    mode = sys.argv[3] if len(sys.argv) > 3 else "both"   # both | up (no download) | down (no upload)

    def step_async(k):
        t0 = time.perf_counter()
        if mode == "down":
            mp.encode_bundle(*devb[k % nb])
        else:
            mp.encode_bundle_host_async(*pinned[k % nb])
        t1 = time.perf_counter()
        mp.decode(0.0, 0.0, res, R, C, 0, R, h, precision=F16)
        t2 = time.perf_counter()
        if mode == "up":
            mp.entropy(h, h, tau, -tau, 0, None, ldev)
            t = None
        else:
            t = mp.entropy_host_async(h, h, tau, -tau, 0, None, outs[k % 2])
        t3 = time.perf_counter()
        calls["enc"] += t1 - t0
        calls["dec"] += t2 - t1
        calls["ent"] += t3 - t2
        return t

    def wait(t):
        if t is None:
            torch.cuda.current_stream().synchronize()
        else:
            mp.wait(t)

    for k in range(3):
        wait(step_async(k))
    for key in calls:
        calls[key] = 0.0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(hi)
    prev = None
    for k in range(K):
        t = step_async(k)
        if prev is not None or (mode == "up" and k):
            tw = time.perf_counter()
            if mode != "up":
                wait(prev)
            calls["wait"] += time.perf_counter() - tw
        prev = t
    wait(prev)
    e1.record(hi)
    wall = (time.perf_counter() - t0) * 1e3 / K
    torch.cuda.synchronize()
    print(f"pipelined host: wall {wall:.4f} ms/step, compute stream {e0.elapsed_time(e1) / K:.4f} ms/step; "
          + ", ".join(f"{a} {b * 1e3 / K:.4f}" for a, b in calls.items()))

    for k in range(3):
        mp.encode_bundle(*devb[k % nb])
        mp.decode(0.0, 0.0, res, R, C, 0, R, h, precision=F16)
        mp.entropy(h, h, tau, -tau, 0, None, ldev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(hi)
    for k in range(K):
        mp.encode_bundle(*devb[k % nb])
        mp.decode(0.0, 0.0, res, R, C, 0, R, h, precision=F16)
        mp.entropy(h, h, tau, -tau, 0, None, ldev)
    e1.record(hi)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / K
    print(f"device-resident, no per-step sync: wall {wall:.4f} ms/step, compute stream {e0.elapsed_time(e1) / K:.4f}")
    assert mp.sync() == 0


if __name__ == "__main__":
    main()
