#!/usr/bin/env python3
"""Per-config throughput on one B200 (C1..C5): encode (points bundled/s, fraction of the
MUFU roofline) and decode (cells/s, GEMM TFLOP/s, fraction of tensor peak), from the
library's in-stream CUDA events.  C5 runs one row band of 8 (its per-GPU share) with its
full 10M-point encode.  Writes profiles/<tag>_configs.json.
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2408_09066_b200 import Mapper  # noqa: E402
from paper_2408_09066_b200.parallel import decoded_rows, row_band  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def tau_of(D):
    p = 1.0 / (2.0 * D)
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


def bench_config(name, reps, pk, points=None, band=None, delta=1, dec_method=-1):
    sc = Scenario(name)
    cfg = sc.cfg
    xy, lab = points if points is not None else sc.all_points()
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    r0, r1 = band if band else (0, R)
    tau = tau_of(D)
    mp = Mapper(D, 0, l, sc.bounds, delta=delta)
    mp.set_tuning("dec_method", dec_method)
    xg, lg = torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda()
    L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def once():
        mp.reset()
        mp.encode_bundle(xg, lg)
        mp.decode(0.0, 0.0, res, R, C, r0, r1, h)
        mp.entropy(h, h, tau, -tau, 0, None, L)

    for _ in range(2):
        once()
    torch.cuda.synchronize()
    mp.profile_read()
    mp.profile_enable(True)
    for _ in range(reps):
        flush.zero_()
        once()
    prof = mp.profile_read()
    mp.profile_enable(False)
    assert mp.sync() == 0
    mp.close()
    per = {k: v[0] / reps for k, v in prof.items()}
    n = len(lab)
    Dp = (D + 31) // 32 * 32
    ra, rb = decoded_rows(R, r0, r1, h)
    flops = 2.0 * 2 * (rb - ra) * C * 2 * Dp
    enc_ms = per["encode"] + per["reduce"]
    nd_ms = per.get("nd_spread", 0.0) + per.get("nd_colfft", 0.0) + per.get("nd_rowfft", 0.0)
    dec_ms = per["norms"] + per["table_A"] + per["decode_gemm"] + nd_ms
    gemm_tf = flops / (per["decode_gemm"] * 1e-3) / 1e12 if per["decode_gemm"] > 0 else None
    sfu_peak = 148 * 8 * pk["sm_max_mhz"] * 1e6   # one point at a time: 2 MUFU per phasor
    out = {
        "config": name, "delta": delta, "points": n, "D": D, "grid": f"{R}x{C}", "band_rows": [r0, r1],
        "decode_method": "nufft" if nd_ms > 0 else "gemm",
        "kernel_ms": {k: round(v, 5) for k, v in per.items()},
        "points_bundled_per_s": n / (enc_ms * 1e-3),
        "encode_frac_mufu_roofline": n * D / (per["encode"] * 1e-3) / sfu_peak,
        "cells_decoded_per_s": (r1 - r0) * C / (dec_ms * 1e-3),
        "gemm_tflops": gemm_tf,
        "gemm_frac_sustained": gemm_tf / pk["bf16_tflops_sustained"] if gemm_tf else None,
        "gemm_frac_burst": gemm_tf / pk["bf16_tflops"] if gemm_tf else None,
        "dense_equivalent_tflops": flops / (dec_ms * 1e-3) / 1e12,
        "entropy_GBps": (r1 - r0) * C * 9 / (per["entropy"] * 1e-3) / 1e9,
        "step_ms": sum(per.values()),
    }
    print(json.dumps(out), flush=True)
    return out


def main(tag):
    torch.cuda.set_device(0)
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"sm_max_mhz": 1965.0, "bf16_tflops_sustained": 1400.0,
                                                        "bf16_tflops": 1600.0}
    res = [bench_config("C1", 50, pk), bench_config("C2", 20, pk), bench_config("C3", 5, pk),
           bench_config("C3", 5, pk, dec_method=0), bench_config("C2", 20, pk, dec_method=1),
           bench_config("C4", 10, pk, points=Scenario("C4").batch(0)),
           bench_config("C4", 10, pk, points=Scenario("C4").batch(0), dec_method=0)]
    sc5 = Scenario("C5")
    res.append(bench_config("C5", 2, pk, points=sc5.all_points(), band=row_band(4000, 0, 8)))
    # quadrant memories (NEXT #1): the C4 step with delta = 2 and 4
    for dl in (2, 4):
        res.append(bench_config("C4", 10, pk, points=Scenario("C4").batch(0), delta=dl))
    path = os.path.join(ROOT, "gpurun_out", f"{tag}_configs.json")   # copied to profiles/ by hand
    json.dump(res, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
