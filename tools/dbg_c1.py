"""Debug helper: one C1 pass through the library, synchronising after each call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_09066_b200 import Mapper
from synth.lidar import Scenario
sc = Scenario("C1"); cfg = sc.cfg
xy, lab = sc.all_points()
mp = Mapper(cfg["D"], 0, cfg["l"], sc.bounds)
mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda()); print("encode", mp.sync(), flush=True)
R, C = cfg["rows"], cfg["cols"]
mp.decode(0, 0, cfg["res"], R, C, 0, R, 1); print("decode", mp.sync(), flush=True)
L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
mp.entropy(1, 1, 0.001, -0.001, 0, None, L); print("entropy", mp.sync(), flush=True)
