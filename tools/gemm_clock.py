"""Sustained-loop comparison at the C4 decode shape: the library decode GEMM (k_decode_gemm2,
fused H_b epilogue) back to back for ~2 s vs torch.matmul (cuBLAS) on the same M x N x K for
~2 s, each with NVML SM-clock samples (median) and power-cap reasons.  Tells whether a gap
to cuBLAS is the clock (power) or the kernel.  One JSON line per arm."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def timed(fn, seconds=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 0
    with ClockSampler(0) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        while time.perf_counter() - t0 < seconds:
            for _ in range(20):
                fn()
            n += 20
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, clk.summary()


def main():
    sc = Scenario(os.environ.get("CFG", "C4"))
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    Dp = (D + 31) // 32 * 32
    xy, lab = sc.scans(0, 20)
    mp = Mapper(D, 0, l, sc.bounds)
    for kv in [x for x in (sys.argv[1] if len(sys.argv) > 1 else "").split(",") if x]:
        k, v = kv.split("=")
        mp.set_tuning(k, int(v))
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    mp.decode(0.0, 0.0, res, R, C, 0, R, h)
    mp.sync()
    flops = 2.0 * 2 * (R + 2 * h) * C * 2 * Dp
    mp.profile_read()
    mp.profile_enable(True)
    ms_step, clk = timed(lambda: mp.decode(0.0, 0.0, res, R, C, 0, R, h))
    prof = mp.profile_read()
    gemm_ms = prof["decode_gemm"][0] / prof["decode_gemm"][1]
    print(json.dumps({"arm": "k_decode_gemm2", "cfg": sc.name, "gemm_ms": round(gemm_ms, 4),
                      "tflops": round(flops / gemm_ms / 1e9, 1), "decode_ms_per_call": round(ms_step, 4),
                      "clocks": clk}), flush=True)
    mp.close()
    M, N, K = 2 * (R + 2 * h), C, 2 * Dp
    for dt in (torch.float16, torch.bfloat16):
        a = torch.randn(M, K, device="cuda", dtype=dt)
        b = torch.randn(N, K, device="cuda", dtype=dt)
        ms, clk = timed(lambda: torch.matmul(a, b.t()))
        print(json.dumps({"arm": "cublas", "dtype": str(dt).split(".")[-1], "M": M, "N": N, "K": K,
                          "ms": round(ms, 4), "tflops": round(2.0 * M * N * K / ms / 1e9, 1), "clocks": clk}), flush=True)


if __name__ == "__main__":
    main()
