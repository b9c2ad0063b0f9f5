#!/usr/bin/env python3
"""One C5 step (10M points, D = 16384, 4000^2 grid, 7x7) for an ncu launch list:
  ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file out.csv python tools/c5_kernels.py"""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402

sc = Scenario("C5")
cfg = sc.cfg
xy, lab = sc.all_points()
D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
p = 1.0 / (2 * D)
tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
xg, lg = torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda()
mp = Mapper(D, 0, l, sc.bounds)
L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
for _ in range(3):
    mp.reset()
    mp.encode_bundle(xg, lg)
    mp.decode(0.0, 0.0, res, R, C, 0, R, h)
    mp.entropy(h, h, tau, -tau, 0, None, L)
assert mp.sync() == 0
mp.close()
