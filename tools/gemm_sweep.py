"""Decode-GEMM sweep at one config's shape (default C3: A 2000 x 8192, B 1000 x 8192, fp16): the
library decode with pinned tile width / split-K / kernel variant, GEMM time from the library's
CUDA events (L2 flushed before each decode), TFLOP/s and fraction of the measured burst peak.
  CFG=C3 python tools/gemm_sweep.py "" "gemm_bn=128" "gemm_splits=2" ...
"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    sc = Scenario(os.environ.get("CFG", "C3"))
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    xy, lab = sc.scans(0, 20)
    mp = Mapper(D, 0, l, sc.bounds)
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    Dp = (D + 31) // 32 * 32
    flops = 2.0 * 2 * R * C * 2 * Dp
    for spec in sys.argv[1:] or [""]:
        saved = {}
        for kv in [x for x in spec.split(",") if x]:
            k, v = kv.split("=")
            saved[k] = mp.get_tuning(k)
            mp.set_tuning(k, int(v))
        for _ in range(3):
            mp.decode(0.0, 0.0, res, R, C, 0, R, h)
        mp.sync()
        mp.profile_read()
        mp.profile_enable(True)
        for _ in range(20):
            flush.zero_()
            mp.decode(0.0, 0.0, res, R, C, 0, R, h)
        prof = mp.profile_read()
        mp.profile_enable(False)
        ms = prof["decode_gemm"][0] / prof["decode_gemm"][1]
        tf = flops / (ms * 1e-3) / 1e12
        print(json.dumps({"cfg": sc.name, "spec": spec, "gemm_us": round(1e3 * ms, 2), "tflops": round(tf, 1),
                          "frac_burst": round(tf / pk["bf16_tflops"], 4),
                          "table_A_us": round(1e3 * prof["table_A"][0] / prof["table_A"][1], 2) if prof["table_A"][1] else 0.0}),
              flush=True)
        for k, v in saved.items():
            mp.set_tuning(k, v)
    mp.close()


if __name__ == "__main__":
    main()
