#!/usr/bin/env python3
"""Does the C4 encode overlap with the C4 decode on one B200?  Two independent contexts:
A bundles batches on stream s2, B (fixed memories) decodes + entropies the 2000x2000 grid on
stream s1.  Times K iterations serially (one stream) and concurrently (two streams) with
CUDA events; prints ms per iteration for both."""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    sc = Scenario("C4")
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    p = 1.0 / (2.0 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    batches = [sc.batch(b) for b in range(4)]
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in batches]
    A = Mapper(D, 0, l, sc.bounds)
    B = Mapper(D, 0, l, sc.bounds)
    B.encode_bundle(*dev[0])
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)   # decode stream high priority

    def enc(k, s):
        with torch.cuda.stream(s):
            A.encode_bundle(*dev[k % len(dev)])

    def dec(s):
        with torch.cuda.stream(s):
            B.decode(0.0, 0.0, res, R, C, 0, R, h)
            B.entropy(h, h, tau, -tau, 0, None, L)

    for mode in ("serial", "concurrent", "serial", "concurrent"):
        for k in range(3):
            enc(k, s1 if mode == "serial" else s2)
            dec(s1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        for k in range(K):
            enc(k, s1 if mode == "serial" else s2)
            dec(s1)
        done2 = torch.cuda.Event()
        done2.record(s2)
        s1.wait_event(done2)
        e1.record(s1)
        torch.cuda.synchronize()
        print(f"{mode:10s} {e0.elapsed_time(e1) / K:.4f} ms per (encode + decode + entropy)")
    assert A.sync() == 0 and B.sync() == 0


if __name__ == "__main__":
    main()
