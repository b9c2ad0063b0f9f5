"""cuBLAS (torch.matmul) on the decode GEMM's exact shapes, for context beside k_decode_gemm2:
M = 2 (rows + halo) class rows, N = cols, K = 2 Dp, f16 / bf16 operands, fp32 accumulate
(output f16 as torch returns; the decode kernel instead writes H_b / q in its epilogue).
Prints one JSON line per shape: best-of-20 and median ms, TFLOP/s."""
import json
import sys

import torch

SHAPES = {"C3": (2 * 1006, 1000, 2 * 4096), "C4": (2 * 2006, 2000, 2 * 8192), "C5_band": (2 * 506, 4000, 2 * 16384),
          "cube8192": (8192, 8192, 8192)}


def main():
    dev = torch.device("cuda:0")
    for name, (M, N, K) in SHAPES.items():
        for dt in (torch.float16, torch.bfloat16):
            a = torch.randn(M, K, device=dev, dtype=dt)
            b = torch.randn(N, K, device=dev, dtype=dt)
            for _ in range(3):
                torch.matmul(a, b.t())
            torch.cuda.synchronize()
            ts = []
            for _ in range(20):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b.t())
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            fl = 2.0 * M * N * K
            print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "dtype": str(dt).split(".")[-1],
                              "best_ms": round(ts[0], 4), "median_ms": round(ts[len(ts) // 2], 4),
                              "best_tflops": round(fl / ts[0] / 1e9, 1),
                              "median_tflops": round(fl / ts[len(ts) // 2] / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
