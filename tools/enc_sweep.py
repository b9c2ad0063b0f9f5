"""Encode variant sweep on C4 batches (one GPU): per-variant encode kernel time (library CUDA
events), phasors/s, and the memory error vs the fp64 oracle on batch 0.
  python tools/enc_sweep.py "enc_x2=2,enc_x2_npoly=4" "enc_x2=4,enc_x2_npoly=4,enc_x2_minb=3" ...
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2408_09066_b200 import Mapper  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def main():
    sc = Scenario(os.environ.get("CFG", "C4"))
    cfg = sc.cfg
    D, l = cfg["D"], cfg["l"]
    xy, lab = sc.batch(0) if cfg["batch_scans"] else sc.all_points()
    dxy, dlab = torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda()
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode(tx, ty, l, xy, lab)
    out = []
    for spec in sys.argv[1:]:
        mp = Mapper(D, 0, l, sc.bounds)
        knobs = dict(kv.split("=") for kv in spec.split(",") if kv)
        for k, v in knobs.items():
            mp.set_tuning(k, int(v))
        mp.encode_bundle(dxy, dlab)
        mg, cg = mp.get_memory()
        err = max(np.linalg.norm(mg[c] - mo[c]) / np.linalg.norm(mo[c]) for c in (0, 1))
        for _ in range(3):
            mp.encode_bundle(dxy, dlab)
        mp.sync()
        mp.profile_read()
        mp.profile_enable(True)
        for _ in range(20):
            mp.encode_bundle(dxy, dlab)
        prof = mp.profile_read()
        ms = prof["encode"][0] / prof["encode"][1]
        red = prof["reduce"][0] / max(1, prof["reduce"][1])
        rec = {"spec": spec, "encode_ms": round(ms, 4), "reduce_ms": round(red, 4),
               "gphasor_s": round(len(lab) * D / ms / 1e6, 1), "mem_err": float(f"{err:.3e}"),
               "counts_ok": list(cg) == list(co)}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        mp.close()


if __name__ == "__main__":
    main()
