#!/usr/bin/env python3
"""bench.py -- VSA-OGM hot path on B200: one JSON line per run (driver contract).

A step is one pass of the whole hot path over one
batch of the streaming config C4 (BASELINE.json configs[3], the config the
metric "... at D=8192" is quoted on): bundle one 100-scan batch (~204k
labelled points) into the persistent D=8192 memories, [all-reduce + commit
across ranks], decode the 2000 x 2000 grid (0.05 m, 100 m x 100 m) on the
tensor cores, and compute the 5x5 local-entropy map and labels.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL): points of each batch
are sharded (contiguous ranges) with one all-reduce of the pending memories
(Alg. 3), and grid rows are sharded into bands with halo rows; `value` is the
whole-job throughput (cells of the full grid per second).  --impl reference
times the fp64 CPU oracle (the only reference that exists for this tier) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid cells decoded/sec and points bundled/sec at D=8192; decode % tensor peak"
CONFIG = "C4"
N_DISTINCT_BATCHES = 8


def label_tau(D: int) -> float:
    """Harness label band (L14): tau = H_b(1/(2D))."""
    p = 1.0 / (2.0 * D)
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks (NVML, sampled in a thread)
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self._t = threading.Thread(target=self._run, args=(period_s,), daemon=True)

    def _run(self, period):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(period)

    def __enter__(self):
        if self.ok:
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_config(sc, n_pts_mean, world):
    cfg = sc.cfg
    return {
        "workload": "C4 streaming step: bundle one 100-scan lidar batch into persistent D=8192 FHRR memories, "
                    "decode the 2000x2000 grid (0.05 m) on tcgen05, 5x5 local entropy + 3-way labels",
        "D": cfg["D"], "length_scale_m": cfg["l"], "grid": f"{cfg['rows']}x{cfg['cols']}@{cfg['res']}m",
        "points_per_step": int(round(n_pts_mean)), "cells_per_step": cfg["rows"] * cfg["cols"],
        "window": f"{2 * cfg['half'] + 1}x{2 * cfg['half'] + 1} box",
        "decode_operands": "f16 (fp32 accumulate in TMEM)",
        "l2": "pipelined value and e2e: inputs larger than L2 (per-step working set: table A 131 MB written + "
              "read, table B 65 MB, H_b 32 MB > 126 MB L2); serial sub-line: flushed between steps (256 MiB write)",
        "parallelism": "single GPU" if world == 1 else f"points sharded x{world} + NCCL all-reduce of memories; "
                                                      f"grid row bands x{world} with halo",
        "distinct_batches": N_DISTINCT_BATCHES,
    }


def load_ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------------ native arm
def run_native(args):
    import torch
    import torch.distributed as dist

    from paper_2408_09066_b200 import F16, Mapper
    from paper_2408_09066_b200.parallel import fuse_and_commit, point_shard, row_band
    from synth.lidar import Scenario

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    sc = Scenario(CONFIG)
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    tau = label_tau(D)
    nb = min(N_DISTINCT_BATCHES, args.steps + args.warmup)
    host_batches, dev_batches, pinned = [], [], []
    n_total = []
    for b in range(nb):
        xy, lab = sc.batch(b)
        n_total.append(len(lab))
        lo, hi = point_shard(len(lab), rank, world)
        xy, lab = np.ascontiguousarray(xy[lo:hi]), np.ascontiguousarray(lab[lo:hi])
        host_batches.append((xy, lab))
        dev_batches.append((torch.from_numpy(xy).to(dev), torch.from_numpy(lab).to(dev)))
        pinned.append((torch.from_numpy(xy).pin_memory(), torch.from_numpy(lab).pin_memory()))
    r0, r1 = row_band(R, rank, world)
    band = r1 - r0
    labels_dev = torch.empty((band, C), dtype=torch.uint8, device=dev)
    labels_host = torch.empty((band, C), dtype=torch.uint8).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    mp = Mapper(D, 0, l, sc.bounds)

    def step(b, host=False):
        if host:
            xy, lab = pinned[b % nb]
            mp.encode_bundle_host(xy, lab)
        else:
            xy, lab = dev_batches[b % nb]
            mp.encode_bundle(xy, lab)
        if world > 1:
            fuse_and_commit(mp)
        mp.decode(0.0, 0.0, res, R, C, r0, r1, h, precision=F16)
        if host:
            mp.entropy_host(h, h, tau, -tau, 0, None, labels_host)
        else:
            mp.entropy(h, h, tau, -tau, 0, None, labels_dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (untimed)
    for b in range(args.warmup):
        step(b)
    barrier()
    if mp.sync() != 0:
        raise RuntimeError("deferred device error during warm-up")

    # Two timed regions of K steps each (barrier + synchronize on both sides, max over ranks),
    # NVML clocks sampled through both:
    # (1) serial: one stream, per-step CUDA events, L2 flushed between steps (outside the
    #     events) -- the per-kernel times, shares and rooflines come from here;
    # (2) pipelined streaming (the headline `value`): vsaogm_set_encode_stream puts the encodes
    #     on a low-priority stream, where the encode of batch k+1 overlaps the GEMM + entropy of
    #     batch k (high-priority stream); CUDA events around the K steps; no flush -- the step's
    #     working set (tables A 131 MB + B 65 MB, H_b 32 MB) exceeds the 126 MB L2.
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mp.profile_read()              # clear
    mp.profile_enable(True)
    with ClockSampler(dev.index) as clk:
        barrier()
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            step(args.warmup + k)
            evs[k][1].record(stream)
        barrier()
        prof = mp.profile_read()
        mp.profile_enable(False)

        hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
        with torch.cuda.stream(hi):
            mp.set_encode_stream(lo)
            for b in range(args.warmup):           # fill the pipeline (untimed)
                step(b)
            barrier()
            if mp.sync() != 0:
                raise RuntimeError("deferred device error during pipelined warm-up")
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            launches0 = mp.launch_count()
            barrier()
            p0.record(hi)
            for k in range(args.steps):
                step(args.warmup + k)
            p1.record(hi)                          # the last decode waited for the last encode
            barrier()
            launches = mp.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = torch.tensor([sum(step_ms), p0.elapsed_time(p1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    serial_ms_per_step = t_ms[0].item() / args.steps
    ms_per_step = t_ms[1].item() / args.steps

    # end-to-end through the public pipelined host API: every step uploads its batch from pinned
    # host memory (upload stream), bundles, decodes, and downloads the labels to pinned host
    # memory (download stream); step k's copies overlap the kernels of steps k-1 / k+1.  Wall
    # clock over all K steps, including the final wait; max over ranks.
    labels_pipe = [torch.empty((band, C), dtype=torch.uint8).pin_memory() for _ in range(3)]

    def step_async(b, slot):
        xy, lab = pinned[b % nb]
        mp.encode_bundle_host_async(xy, lab)
        if world > 1:
            fuse_and_commit(mp)
        mp.decode(0.0, 0.0, res, R, C, r0, r1, h, precision=F16)
        return mp.entropy_host_async(h, h, tau, -tau, 0, None, labels_pipe[slot])

    def run_e2e(first, count):
        """`count` pipelined steps, two in flight (the library's three I/O slots); returns (total
        wall ms, per-step wall ms between ticket waits)."""
        t0 = time.perf_counter()
        tickets, marks = [], []
        for k in range(count):
            tickets.append(step_async(first + k, k % 3))
            if k >= 2 and mp.wait(tickets[k - 2]) != 0:
                raise RuntimeError("deferred device error (e2e)")
            marks.append(time.perf_counter())
        for t in tickets[-2:]:
            if mp.wait(t) != 0:
                raise RuntimeError("deferred device error (e2e)")
        t1 = time.perf_counter()
        return (t1 - t0) * 1e3, [(b - a) * 1e3 for a, b in zip(marks, marks[1:])]

    with torch.cuda.stream(hi):                    # encode stream still set: the same pipeline
        run_e2e(0, max(3, args.warmup, nb))        # untimed: every distinct batch once (sizes the slots)
        barrier()
        e2e_total, e2e_steps = run_e2e(args.warmup, args.steps)
        e2e_t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        mp.set_encode_stream(None)
    e2e_median = statistics.median(e2e_steps) if e2e_steps else None
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_ms_step = e2e_t.item() / args.steps
    if mp.sync() != 0:
        raise RuntimeError("deferred device error")

    cells = R * C
    n_mean = float(np.mean([n_total[(args.warmup + k) % nb] for k in range(args.steps)]))
    value = cells / (ms_per_step * 1e-3)
    pk, pk_kind = peaks()

    # per-kernel averages (this rank) and rooflines
    def avg(name):
        ms, n = prof[name]
        return ms / n if n else float("nan")
    enc_ms, gemm_ms = avg("encode"), avg("decode_gemm")
    shares = {k: round(v[0] / max(1e-12, sum(x[0] for x in prof.values())), 4) for k, v in prof.items()}
    # encode (dominant): SFU-bound; algorithmic work = D phasors (1 MUFU sin + 1 MUFU cos) per point
    my_pts = float(np.mean([len(host_batches[(args.warmup + k) % nb][1]) for k in range(args.steps)]))
    phasors = my_pts * D
    sm_max = pk.get("sm_max_mhz", 1965.0)
    sfu_peak = 148 * 16 / 2 * sm_max * 1e6          # MUFU-only: 16 MUFU/clk/SM, 2 MUFU per phasor
    # combined MUFU + FMA-pipe ceiling of the packed encode, per SM per
    # clock from the guide's unit counts: 16 MUFU, 128 FMA-pipe lanes.  A MUFU phasor costs
    # 2 MUFU + 5 FMA lanes (angle 2, FMUL.RZ 1, accumulate 2); a polynomial phasor 16 FMA
    # lanes (angle 2, sincos_fma2_lite 12, accumulate 2).  max m + p s.t. 2m <= 16,
    # 5m + 16p <= 128 -> m = 8, p = 88/16 (the ALU pipe, 3 ops per polynomial phasor, and the
    # issue slots, 5 and 11 per phasor, are not binding there).
    per_clk = 8 + (128 - 5 * 8) / 16
    alu_peak = 148 * per_clk * sm_max * 1e6
    enc_rate = phasors / (enc_ms * 1e-3)
    clocks = clk.summary()
    # decode GEMM: 2 M N K flops with M = 2 (band + halo rows), N = C, K = 2 Dp
    from paper_2408_09066_b200.parallel import decoded_rows
    ra, rb = decoded_rows(R, r0, r1, h)
    Dp = (D + 31) // 32 * 32
    flops = 2.0 * (2 * (rb - ra)) * C * (2 * Dp)
    gemm_tf = flops / (gemm_ms * 1e-3) / 1e12
    traffic = load_ncu_traffic()
    enc_share = shares.get("encode", 0)
    dominant = "encode" if enc_share >= shares.get("decode_gemm", 0) else "decode_gemm"
    if dominant == "encode":
        roofline = {"kernel": "k_encode_bundle_x2", "bound": "alu", "achieved": round(enc_rate / 1e9, 2),
                    "peak": round(alu_peak / 1e9, 2), "unit": "Gphasor/s", "frac": round(enc_rate / alu_peak, 4),
                    "traffic": traffic.get("encode"),
                    "peak_basis": f"combined MUFU+FMA-pipe ceiling {per_clk:.2f} phasors/clk/SM x 148 SM x "
                                  f"{sm_max:.0f} MHz (guide unit counts: 16 MUFU + 128 FMA lanes/clk/SM; "
                                  "DESIGN.md sec. 6)",
                    "mufu_only_peak": round(sfu_peak / 1e9, 2),
                    "frac_of_mufu_only": round(enc_rate / sfu_peak, 4),
                    "frac_at_measured_clock": (round(enc_rate / (148 * per_clk * clocks["sm_mhz"] * 1e6), 4)
                                               if clocks.get("sm_mhz") else None)}
    else:
        roofline = None
    gemm_roof = {"kernel": "k_decode_gemm", "bound": "tensor", "achieved": round(gemm_tf, 1),
                 "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                 "frac": round(gemm_tf / pk["bf16_tflops_sustained"], 4),
                 "frac_of_burst": round(gemm_tf / pk["bf16_tflops"], 4), "traffic": traffic.get("decode_gemm"),
                 "peak_basis": f"MEASURED_PEAKS.json ({pk_kind}) bf16 sustained; fp16 dense = bf16 dense"}
    if roofline is None:
        roofline = gemm_roof

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 (decode MMA operands f16, fp32 accumulate)",
        "data": "synthetic", "config": workload_config(sc, n_mean, world),
        "points_bundled_per_s": round(n_mean / (ms_per_step * 1e-3), 1),
        "decode_cells_per_s_gemm_only": round(cells / (gemm_ms * 1e-3), 1),
        "decode_pct_tensor_peak": round(100 * gemm_tf / pk["bf16_tflops_sustained"], 2),
        "roofline": roofline, "decode_roofline": gemm_roof,
        "schedule": "pipelined: encode of batch k+1 (low-priority stream) overlaps the GEMM + entropy of batch k",
        "serial": {"ms_per_step": round(serial_ms_per_step, 4), "value": round(cells / (serial_ms_per_step * 1e-3), 1),
                   "note": "one stream, L2 flushed between steps; kernel_ms_per_step and the rooflines are from here"},
        "kernel_ms_per_step": {k: round(v[0] / args.steps, 5) for k, v in prof.items()},
        "kernel_time_share": shares,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": round(cells / (e2e_ms_step * 1e-3), 1), "unit": "cells/s",
                "ms_per_step": round(e2e_ms_step, 4),
                "ms_per_step_median": round(e2e_median, 4) if e2e_median else None,
                "h2d_bytes_per_step": int(round(my_pts * 9)),
                "d2h_bytes_per_step": int(band * C)},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(sc, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    mp.close()
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ oracle (CPU) timing
_ORACLE_INPUTS = {}


def oracle_step_estimate(sc, budget_s, seed=0):
    """Time the fp64 oracle on a bounded sample of the C4 step and extrapolate
    linearly to one full step.  Returns (seconds per step, sample description, threads)."""
    import oracle
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    nthreads = oracle.default_threads()
    if "batch0" not in _ORACLE_INPUTS:
        _ORACLE_INPUTS["batch0"] = sc.batch(0)
        _ORACLE_INPUTS["theta"] = oracle.theta(0, D)
    xy, lab = _ORACLE_INPUTS["batch0"]
    tx, ty = _ORACLE_INPUTS["theta"]
    rng = np.random.default_rng(seed)
    # probe the per-item cost, then size each sample to ~budget/2 seconds
    t0 = time.perf_counter()
    oracle.encode(tx, ty, l, xy[:2000], lab[:2000], nthreads=nthreads)
    per_pt = (time.perf_counter() - t0) / 2000
    n_enc = int(min(len(lab), max(2000, budget_s / 2 / per_pt)))
    t0 = time.perf_counter()
    m, _, _ = oracle.encode(tx, ty, l, xy[:n_enc], lab[:n_enc], nthreads=nthreads)
    t_enc = time.perf_counter() - t0
    # decode: sampled cells with their entropy windows ((2h+1)^2 cells each) -> per-cell cost
    per_cell = per_pt   # same D sincos per item
    n_win = max(4, int(budget_s / 2 / per_cell / (2 * h + 1) ** 2))
    cells = rng.integers(h, [R - h, C - h], size=(n_win, 2))
    t0 = time.perf_counter()
    tau = label_tau(D)
    w = 2 * h + 1
    du, dv = np.meshgrid(np.arange(-h, h + 1), np.arange(-h, h + 1), indexing="ij")
    rows = (cells[:, 0, None] + du.ravel()[None, :]).ravel()
    cols = (cells[:, 1, None] + dv.ravel()[None, :]).ravel()
    q_all = oracle.decode_cells(tx, ty, l, m, 0, 0, res, rows, cols, nthreads=nthreads).reshape(2, n_win, w, w)
    for e, (r, c) in enumerate(cells):
        oracle.entropy_cells(R, C, r - h, r + h + 1, c - h, c + h + 1, q_all[:, e], h, h, 0, tau, -tau, [r], [c])
    t_dec = time.perf_counter() - t0
    n_dec_cells = n_win * (2 * h + 1) ** 2
    step_s = t_enc * (len(lab) / n_enc) + t_dec * (R * C / n_dec_cells)
    sample = (f"oracle on C4 batch 0: encode {n_enc} of {len(lab)} points ({t_enc:.1f} s), decode+entropy "
              f"of {n_win} cells via their {2 * h + 1}x{2 * h + 1} windows = {n_dec_cells} decoded cells "
              f"({t_dec:.1f} s); extrapolated linearly to one full step ({len(lab)} points + {R * C} cells)")
    return step_s, sample, nthreads, len(lab)


def cpu_baseline(sc, budget_s=20.0):
    cfg = sc.cfg
    step_s, sample, nthreads, _ = oracle_step_estimate(sc, budget_s)
    return {"value": round(cfg["rows"] * cfg["cols"] / step_s, 1), "unit": "cells/s", "cores": nthreads,
            "kind": "oracle", "sample": sample}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from synth.lidar import Scenario
    sc = Scenario(CONFIG)
    cfg = sc.cfg
    cells = cfg["rows"] * cfg["cols"]
    # the whole --steps K --warmup W run is bounded to ~3 x cpu_seconds of CPU time
    budget = max(0.3, 3 * args.cpu_seconds / max(1, args.steps + args.warmup))
    times = []
    for k in range(args.warmup + args.steps):
        step_s, sample, nthreads, n_pts = oracle_step_estimate(sc, budget, seed=k)
        if k >= args.warmup:
            times.append(step_s)
    ms = 1e3 * float(np.mean(times))
    value = cells / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "cells/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": workload_config(sc, n_pts, 1),
        "cpu_baseline": {"value": round(value, 2), "unit": "cells/s", "cores": nthreads, "kind": "oracle",
                         "sample": sample + " (each step a bounded sample)"},
        "e2e": {"value": round(value, 2), "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
