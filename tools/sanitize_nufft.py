#!/usr/bin/env python3
"""Small exercise of the NUFFT encode / decode, the dependent-launch chain and the column-walk
entropy kernel for compute-sanitizer:
  compute-sanitizer --tool memcheck python tools/sanitize_nufft.py
  compute-sanitizer --tool racecheck python tools/sanitize_nufft.py"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    xy, lab = xy[:6000], lab[:6000]
    xg, lg = torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(np.ascontiguousarray(lab)).cuda()
    D, l = 2048, 0.25
    p = 1.0 / (2 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
    with torch.cuda.stream(hi):
        mp = Mapper(D, 0, l, sc.bounds)
        mp.set_tuning("enc_method", 1)
        mp.set_tuning("dec_method", 1)
        mp.set_encode_stream(lo)
        # transform sizes 256 (LOGN 8), 512 (9: the skipped radix-2 pass), 1024 on the two axes; ragged columns
        for (R, C, res, h) in ((120, 203, 0.1, 2), (75, 130, 0.1, 1), (300, 400, 0.1, 3)):
            for (r0, r1) in ((0, R), (R // 3, 2 * R // 3)):
                mp.encode_bundle(xg, lg)
                q = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
                mp.decode(0.0, 0.0, res, R, C, r0, r1, h, q_out=q)
                L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
                mp.entropy(h, h, tau, -tau, 0, None, L)          # column-walk kernel
                mp.decode(0.0, 0.0, res, R, C, r0, r1, h)         # lean row pass (no q)
                mp.set_tuning("entropy_kernel", 2)
                mp.entropy(h, h, tau, -tau, 0, None, L)          # TMA-streamed kernel
                mp.set_tuning("entropy_kernel", 0)
        assert mp.sync() == 0
        mp.close()
    print("sanitize_nufft: done")


if __name__ == "__main__":
    main()
