#!/usr/bin/env python3
"""Summarise an ncu capture (--set full .ncu-rep) and a launch list (.csv) into profiles/.

  python tools/ncu_summary.py <tag>        reads gpurun_out/prof_<tag>.ncu-rep, gpurun_out/launches_<tag>.csv
                                           writes profiles/<tag>_ncu_summary.md, profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
SHORT = {"k_nu_": None, "k_nd_": None, "k_encode_pairs": "encode", "k_encode_bundle": "encode", "k_decode_gemm": "decode_gemm",
         "k_entropy": "entropy",
         "k_table<__half2, 1>": "table_A", "k_table<__nv_bfloat162, 1>": "table_A",
         "k_table<__half2, 0>": "table_B", "k_table<__nv_bfloat162, 0>": "table_B",
         "k_reduce_partials": "reduce", "k_commit_norms": "norms", "k_commit": "commit",
         "k_nu_spread_tiles": "nu_spread", "k_nu_rowfft": "nu_rowfft", "k_nu_colfft": "nu_colfft",
         "k_nu_interp": "nu_interp", "k_nu_bin": "nu_bin", "k_nu_scan": "nu_scan", "k_nu_place": "nu_place",
         "k_nd_spread": "nd_spread", "k_nd_strength": "nd_strength", "k_nd_colfft": "nd_colfft",
         "k_nd_rowfft": "nd_rowfft"}


def short(name):
    for k, v in SHORT.items():
        if v is not None and k in name:
            return v
    return name[:60]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val) * mult


def main(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary `{tag}` (`--set full --clock-control none`, one capture per kernel; cold-cache, serialised)",
             "", "| kernel | " + " | ".join(m[1] for m in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    traffic = {}
    stats = {}
    for r in data:
        name = short(r[col["Kernel Name"]])
        vals = []
        for m, _ in METRICS:
            i = col.get(m)
            vals.append(f"{r[i]} {units[i]}".strip() if i is not None else "n/a")
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        rd = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        traffic.setdefault(name, rd + wr)

        def num(metric):
            i = col.get(metric)
            try:
                return float(r[i].replace(",", "")) if i is not None else None
            except ValueError:
                return None
        stats.setdefault(name, {"tag": tag, "duration_us": num("gpu__time_duration.sum"),
                                "issue_active_pct": num("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
                                "warp_instructions": num("smsp__inst_executed.sum"),
                                "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                                "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
                                "registers": num("launch__registers_per_thread")})
    launches = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(launches):
        txt = open(launches).read()
        start = txt.find('"ID"')
        lrows = list(csv.reader(io.StringIO(txt[start:])))
        h = lrows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in lrows[1:]:
            if len(r) <= vi:
                continue
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
            v = float(r[vi].replace(",", "")) * scale
            tot[short(r[ki])] += v
            cnt[short(r[ki])] += 1
        s = sum(tot.values())
        lines += ["", "## Launch list (every launch of the profiled bench command, `gpu__time_duration.sum`)", "",
                  "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for k in sorted(tot, key=lambda k: -tot[k]):
            lines.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {tot[k] / s:.3f} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md")
    open(out, "w").write("\n".join(lines) + "\n")
    # merge: kernels not in this capture keep the figure (and the tag) of the capture they came from
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tags = old.get("tags", {k: old.get("tag", "?") for k in old if k not in ("tag", "tags")})
    merged = {k: v for k, v in old.items() if k not in ("tag", "tags") and not k.startswith(("<unnamed>", "void "))}
    for k, v in traffic.items():
        merged[k] = v
        tags[k] = tag
    tags = {k: t for k, t in tags.items() if k in merged}
    json.dump({"tag": tag, "tags": tags, **merged}, open(tpath, "w"), indent=1)
    spath = os.path.join(ROOT, "profiles", "ncu_kernel_stats.json")
    old_stats = json.load(open(spath)) if os.path.exists(spath) else {}
    old_stats.update(stats)
    json.dump(old_stats, open(spath, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
