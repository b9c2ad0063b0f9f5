#!/usr/bin/env python3
"""Measured GPU-vs-oracle parity numbers for every BASELINE config (writes profiles/<tag>_parity.json).

Full grids for C1 and C2; sampled windows for C3, C4 (one batch) and C5 (one row band of 8,
first 150 scans).  Reports, per config and operand precision: memory relative error,
peak-normalised max |dq| per class, absolute max |dq|, label agreement.
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2408_09066_b200 import Mapper  # noqa: E402
from paper_2408_09066_b200.parallel import row_band  # noqa: E402
from synth.lidar import Scenario  # noqa: E402


def tau_of(D):
    p = 1.0 / (2.0 * D)
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


def run(name, full, points=None, band=None, n_samples=150):
    sc = Scenario(name)
    cfg = sc.cfg
    xy, lab = points if points is not None else sc.all_points()
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    r0, r1 = band if band else (0, R)
    tau = tau_of(D)
    mp = Mapper(D, 0, l, sc.bounds)
    t0 = time.time()
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    res_out = {"config": name, "points": int(len(lab)), "D": D, "grid": f"{R}x{C}", "band": [r0, r1]}
    gpu = {}
    for prec in (0, 1):
        q = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
        mp.decode(0.0, 0.0, res, R, C, r0, r1, h, precision=prec, q_out=q)
        L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
        mp.entropy(h, h, tau, -tau, 0, None, L)
        assert mp.sync() == 0
        gpu[prec] = (q.cpu().numpy().astype(np.float64), L.cpu().numpy())
    mg, cg = mp.get_memory()
    mp.close()
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode(tx, ty, l, xy, lab)
    res_out["counts_equal"] = bool(list(cg) == list(co))
    res_out["memory_rel_err"] = max(float(np.linalg.norm(mg[c] - mo[c]) / np.linalg.norm(mo[c])) for c in (0, 1))
    if full:
        qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, r0, r1, 0, C)
        _, Lo = oracle.entropy_grid(qo, h, h, 0, tau, -tau)
        for prec, tag in ((0, "f16"), (1, "bf16")):
            qg, Lg = gpu[prec]
            res_out[tag] = {
                "q_peak_norm_max_err": [float(np.abs(qg[c] - qo[c]).max() / np.abs(qo[c]).max()) for c in (0, 1)],
                "q_abs_max_err": float(np.abs(qg - qo).max()),
                "label_agreement": float((Lg == Lo).mean()), "cells_compared": int(Lo.size)}
    else:
        rng = np.random.default_rng(0)
        cells = [tuple(v) for v in np.stack([rng.integers(r0, r1, n_samples), rng.integers(0, C, n_samples)], 1)]
        near = [i for i in rng.choice(len(lab), 4 * n_samples, replace=False) if r0 <= xy[i, 1] / res < r1][:n_samples]
        cells += [(min(r1 - 1, int(xy[i, 1] / res)), min(C - 1, int(xy[i, 0] / res))) for i in near]
        for prec, tag in ((0, "f16"), (1, "bf16")):
            qg, Lg = gpu[prec]
            peak = np.abs(qg).reshape(2, -1).max(axis=1)
            errs, abs_err, agree = [], 0.0, []
            for (r, c) in cells:
                ra, rb, ca, cb = max(0, r - h), min(R, r + h + 1), max(0, c - h), min(C, c + h + 1)
                qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, ra, rb, ca, cb)
                ga, gb = max(ra, r0), min(rb, r1)
                d = np.abs(qg[:, ga - r0:gb - r0, ca:cb] - qo[:, ga - ra:gb - ra])
                errs.append([float(d[k].max() / peak[k]) for k in (0, 1)])
                abs_err = max(abs_err, float(d.max()))
                _, lo = oracle.entropy_cells(R, C, ra, rb, ca, cb, qo, h, h, 0, tau, -tau, [r], [c])
                agree.append(lo[0] == Lg[r - r0, c])
            e = np.array(errs)
            res_out[tag] = {"q_peak_norm_max_err": [float(e[:, 0].max()), float(e[:, 1].max())],
                            "q_abs_max_err": abs_err, "label_agreement": float(np.mean(agree)),
                            "cells_compared": len(cells), "sampled": True}
        res_out["f16_vs_bf16_label_agreement"] = float((gpu[0][1] == gpu[1][1]).mean())
    res_out["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(res_out), flush=True)
    return res_out


def main(tag):
    torch.cuda.set_device(0)
    out = [run("C1", True), run("C2", True), run("C3", False)]
    sc4 = Scenario("C4")
    out.append(run("C4", False, points=sc4.batch(0)))
    sc5 = Scenario("C5")
    out.append(run("C5", False, points=sc5.scans(0, 150), band=row_band(4000, 3, 8)))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", f"{tag}_parity.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
