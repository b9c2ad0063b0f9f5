"""Entropy-stencil microbenchmark at C4 (or CFG=C5: 7x7): one decode, then the entropy kernel
repeated (library CUDA events), per variant given as tuning specs, with the achieved
algorithmic bandwidth (8 B read + 1 B written per cell).
  python tools/ent_bench.py "" "entropy_kernel=1" ...
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    sc = Scenario(os.environ.get("CFG", "C4"))
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    xy, lab = sc.batch(0) if cfg["batch_scans"] else sc.scans(0, 100)
    p = 1.0 / (2 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    mp = Mapper(D, 0, l, sc.bounds)
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    mp.decode(0.0, 0.0, res, R, C, 0, R, h)
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for spec in sys.argv[1:] or [""]:
        for kv in [x for x in spec.split(",") if x]:
            k, v = kv.split("=")
            mp.set_tuning(k, int(v))
        for _ in range(3):
            mp.entropy(h, h, tau, -tau, 0, None, L)
        for flushed in (False, True):
            mp.sync()
            mp.profile_read()
            mp.profile_enable(True)
            for _ in range(30):
                if flushed:
                    flush.zero_()
                mp.entropy(h, h, tau, -tau, 0, None, L)
            prof = mp.profile_read()
            mp.profile_enable(False)
            us = 1e3 * prof["entropy"][0] / prof["entropy"][1]
            print(json.dumps({"spec": spec, "l2_flushed": flushed, "entropy_us": round(us, 2),
                              "gbs": round(9 * R * C / (us * 1e-6) / 1e9, 1)}), flush=True)
        mp.set_tuning("entropy_kernel", 0)
        mp.set_tuning("entropy_rw", 0)
    mp.close()


if __name__ == "__main__":
    main()
