#!/usr/bin/env python3
"""Library baseline for the NUFFT decode's transforms: cuFFT (through torch.fft) on the same batches,
unpruned and unfused -- context for DESIGN.md section 6b, not part of the product path.
  python tools/cufft_compare.py"""
import json

import torch


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1e3   # us


def main():
    torch.cuda.set_device(0)
    out = {}
    for name, batch, n in (("row pass (C4): 2000 transforms of 4096", 2000, 4096),
                           ("column pass (C4): 697 transforms of 4096", 697, 4096),
                           ("row pass (C5): 4006 transforms of 8192", 4006, 8192),
                           ("encode row pass (C4): 764 transforms of 2048", 764, 2048)):
        x = torch.randn(batch, n, dtype=torch.complex64, device="cuda")
        out[name] = {"cufft_c2c_us": round(timeit(lambda: torch.fft.ifft(x, dim=1, norm="backward")), 2)}
    # the whole 2-D transform of the C4 decode as a library call: zero-padded 4096 x 4096
    g = torch.zeros(4096, 4096, dtype=torch.complex64, device="cuda")
    out["2-D 4096 x 4096 (the unpruned C4 decode grid)"] = {"cufft_c2c_us": round(timeit(lambda: torch.fft.ifft2(g), reps=20), 2)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
