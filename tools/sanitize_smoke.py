#!/usr/bin/env python3
"""Small end-to-end exercise of every kernel path for compute-sanitizer (memcheck / racecheck):
packed and scalar encodes, delta = 2 sorted runs, split-K decode band, box / fixed / generic /
histogram entropy, the encode stream, the pipelined host I/O, export / import.
  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def tau_of(D):
    p = 1.0 / (2.0 * D)
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


def main():
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    xy, lab = xy[:20000], lab[:20000]
    xg, lg = torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(np.ascontiguousarray(lab)).cuda()
    R, C, res = 120, 203, 0.25
    for D, delta, x2 in ((2048, 1, "2"), (2048, 1, "0"), (2048, 2, "2"), (512, 1, "2")):
        os.environ["VSAOGM_ENC_X2"] = x2
        mp = Mapper(D, 0, 0.25, sc.bounds, delta=delta)
        mp.encode_bundle(xg, lg)
        q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
        mp.decode(0.0, 0.0, res, R, C, 0, R, 3, q_out=q)
        S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
        L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
        t = tau_of(D)
        for h, disk in ((2, 0), (3, 1), (1, 0)):
            mp.entropy(h, h, t, -t, disk, S, L)
        mp.entropy(2, 3, t, -t, 0, S, L)          # unequal radii: generic kernel
        mp.decode(0.0, 0.0, res, R, C, 40, 70, 3)   # band (split-K)
        Sb = torch.empty((3, 30, C), dtype=torch.float32, device="cuda")
        mp.entropy(3, 3, t, -t, 0, Sb, None)
        mp.set_estimator(1)
        mp.decode(0.0, 0.0, res, R, C, 0, R, 2)
        mp.entropy(2, 2, 0.5, 0.5, 0, S, L)
        mp.set_estimator(0)
        blob = mp.export()
        mp.fuse(blob)
        assert mp.sync() == 0
        mp.close()
    os.environ["VSAOGM_ENC_X2"] = "2"
    lo = torch.cuda.Stream()
    mp = Mapper(2048, 0, 0.25, sc.bounds)
    mp.set_encode_stream(lo)
    pinned = (torch.from_numpy(np.ascontiguousarray(xy)).pin_memory(),
              torch.from_numpy(np.ascontiguousarray(lab)).pin_memory())
    out = [torch.empty((R, C), dtype=torch.uint8).pin_memory() for _ in range(2)]
    tickets = []
    for k in range(3):
        mp.encode_bundle_host_async(*pinned)
        mp.decode(0.0, 0.0, res, R, C, 0, R, 2)
        tickets.append(mp.entropy_host_async(2, 2, tau_of(2048), -tau_of(2048), 0, None, out[k % 2]))
        if k:
            assert mp.wait(tickets[k - 1]) == 0
    assert mp.wait(tickets[-1]) == 0
    assert mp.sync() == 0
    mp.close()
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
