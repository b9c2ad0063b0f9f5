#!/usr/bin/env python3
"""Quick C4-step timing for quadrant memories: python tools/delta_bench.py <delta> [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, torch
from synth.lidar import Scenario
from tools.config_bench import bench_config
pk = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {"sm_max_mhz": 1965.0, "bf16_tflops_sustained": 1400.0}
torch.cuda.set_device(0)
bench_config("C4", int(sys.argv[2]) if len(sys.argv) > 2 else 5, pk, points=Scenario("C4").batch(0), delta=int(sys.argv[1]))
