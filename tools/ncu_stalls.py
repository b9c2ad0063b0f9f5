#!/usr/bin/env python3
"""Print the headline metrics and the top stall reasons of every kernel in an ncu report:
   python tools/ncu_stalls.py gpurun_out/prof_<tag>.ncu-rep"""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sector_hit_rate.pct", "sm__cycles_active.avg"]
stalls = [h for h in hdr if "warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")]
for r in data:
    print("=====", r[col["Kernel Name"]][:90])
    for w in want:
        if w in col:
            print(f"  {w}: {r[col[w]]} {units[col[w]]}")
    st = sorted([(float(r[col[s]].replace(",", "")), s) for s in stalls if r[col[s]] not in ("", "n/a")], reverse=True)[:7]
    for v, s in st:
        print(f"    stall {s.split('issue_stalled_')[1][:40]}: {v:.2f}")
