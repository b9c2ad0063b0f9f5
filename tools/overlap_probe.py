#!/usr/bin/env python3
"""Streaming C4 steps on one B200, serial vs pipelined (vsaogm_set_encode_stream: the encode
of batch k+1 runs on a low-priority stream beside the GEMM + entropy of batch k on a
high-priority stream).  Device time over K steps with CUDA events, no L2 flush (the step's
working set exceeds L2).  Checks that both schedules give the same labels and memories."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import F16, Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def run(K, pipelined, dev, L, sc, tau):
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    mp = Mapper(D, 0, l, sc.bounds)
    hi = torch.cuda.Stream(priority=-1)
    lo = torch.cuda.Stream(priority=0)
    with torch.cuda.stream(hi):
        if pipelined:
            mp.set_encode_stream(lo)

        def step(k):
            mp.encode_bundle(*dev[k % len(dev)])
            mp.decode(0.0, 0.0, res, R, C, 0, R, h, precision=F16)
            mp.entropy(h, h, tau, -tau, 0, None, L)

        for k in range(3):
            step(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(hi)
        for k in range(K):
            step(3 + k)
        e1.record(hi)
        torch.cuda.synchronize()
        mp.profile_read()
        mp.profile_enable(True)
        for k in range(K):
            step(3 + K + k)
        prof = mp.profile_read()
        mp.profile_enable(False)
        print("   per-kernel wall ms (events on each kernel's stream):",
              {k: round(v[0] / max(1, K), 4) for k, v in prof.items() if v[0]})
        assert mp.sync() == 0
        mem = mp.get_memory()
    mp.close()
    return e0.elapsed_time(e1) / K, mem


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    sc = Scenario("C4")
    D = sc.cfg["D"]
    p = 1.0 / (2.0 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in (sc.batch(b) for b in range(4))]
    Ls, Lp = (torch.empty((sc.cfg["rows"], sc.cfg["cols"]), dtype=torch.uint8, device="cuda") for _ in range(2))
    for _ in range(2):
        ts, ms = run(K, False, dev, Ls, sc, tau)
        tp, mpm = run(K, True, dev, Lp, sc, tau)
        print(f"serial {ts:.4f} ms/step   pipelined {tp:.4f} ms/step")
    assert np.array_equal(ms[0], mpm[0]) and list(ms[1]) == list(mpm[1])
    assert torch.equal(Ls, Lp)
    print("memories and last labels identical")


if __name__ == "__main__":
    main()
