#!/usr/bin/env python3
"""Dimensionality ablation on the paper's circle dataset (sec. IV-B-1):
AUC of the global entropy map at the 10 % validation points vs D, on the GPU, with the fp64
oracle's AUC beside it for D <= 4096.  l = 0.2 m, r(psi=1) = r(psi=0) = 2 (disk), as in the
paper.  D complex phasors ~ the paper's d = 2D real dimensions.  Writes profiles/<tag>_ablation.json.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GRID = dict(x0=-0.1, y0=-0.1, res=0.1, rows=82, cols=82)
L, H = 0.2, 2


def gpu_auc(D, xy, lab, tr, va, estimator=0):
    from paper_2408_09066_b200 import Mapper
    from paper_2408_09066_b200.evaluate import evaluate
    from synth.circle import BOUNDS
    mp = Mapper(D, 0, L, BOUNDS)
    mp.set_estimator(estimator)
    t0 = time.perf_counter()
    mp.encode_bundle(torch.from_numpy(xy[tr]).cuda(), torch.from_numpy(lab[tr]).cuda())
    g = GRID
    mp.decode(g["x0"], g["y0"], g["res"], g["rows"], g["cols"], 0, g["rows"], H)
    S = torch.empty((3, g["rows"], g["cols"]), dtype=torch.float32, device="cuda")
    mp.entropy(H, H, 0.0, 0.0, 1, S, None)
    assert mp.sync() == 0
    ms = (time.perf_counter() - t0) * 1e3
    mp.close()
    r = evaluate(S[2].cpu().numpy().astype(np.float64), xy[va], lab[va], g["x0"], g["y0"], g["res"])
    r["wall_ms"] = ms
    return r


def oracle_auc(D, xy, lab, tr, va):
    import oracle
    from paper_2408_09066_b200.evaluate import evaluate
    g = GRID
    tx, ty = oracle.theta(0, D)
    m, _, _ = oracle.encode(tx, ty, L, xy[tr], lab[tr])
    q = oracle.decode_grid(tx, ty, L, m, g["x0"], g["y0"], g["res"], 0, g["rows"], 0, g["cols"])
    S, _ = oracle.entropy_grid(q, H, H, 1, 0.0, 0.0)
    return evaluate(S[2], xy[va], lab[va], g["x0"], g["y0"], g["res"])


def main(tag):
    from synth.circle import gen_circle_dataset, split_train_val
    torch.cuda.set_device(0)
    xy, lab = gen_circle_dataset(0)
    tr, va = split_train_val(len(lab), 0.9, 0)
    out = []
    for e in range(1, 15):
        D = 2 ** e
        row = {"D": D, "paper_d_equiv": 2 * D, "gpu": gpu_auc(D, xy, lab, tr, va),
               "gpu_histogram_estimator": gpu_auc(D, xy, lab, tr, va, estimator=1)}
        if D <= 4096:
            row["oracle"] = oracle_auc(D, xy, lab, tr, va)
        print(json.dumps(row), flush=True)
        out.append(row)
    path = os.path.join(ROOT, "profiles", f"{tag}_ablation.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
