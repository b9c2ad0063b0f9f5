"""Multi-rank host logic on CPU (gloo, world size 2): point shards + all-reduce of the
pending memories reproduce the one-shot memories (Alg. 3 fusion),
and decoding row bands with halos then stitching reproduces the full-grid entropy
labels (no communication in the decode).  The arithmetic per rank is the oracle's
(CPU stand-in for the device memories); the sharding and the collective are the
product code of paper_2408_09066_b200/parallel.py."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import oracle
    from paper_2408_09066_b200.parallel import allreduce_pending, decoded_rows, point_shard, row_band
    from synth.lidar import Scenario
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scenario("C1")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    tx, ty = oracle.theta(0, D)
    lo, hi = point_shard(len(lab), rank, world)
    m, cnt, _ = oracle.encode(tx, ty, l, xy[lo:hi], lab[lo:hi], nthreads=2)
    # the library's packed pending layout: memories [2][D][2], then the counts as doubles
    buf = torch.from_numpy(np.concatenate([np.stack([m.real, m.imag], axis=-1).ravel(), cnt.astype(np.float64)]))
    allreduce_pending(buf)
    pend = buf[: 4 * D].view(2, D, 2)
    cnts = buf[4 * D:].to(torch.int64)
    mfull = pend[..., 0].numpy() + 1j * pend[..., 1].numpy()
    r0, r1 = row_band(R, rank, world)
    ra, rb = decoded_rows(R, r0, r1, h)
    q = oracle.decode_grid(tx, ty, l, mfull, 0, 0, res, ra, rb, 0, C, nthreads=2)
    rr, cc = np.meshgrid(np.arange(r0, r1), np.arange(C), indexing="ij")
    S, labels = oracle.entropy_cells(R, C, ra, rb, 0, C, q, h, h, 0, 0.001, -0.001, rr.ravel(), cc.ravel())
    out[rank] = (mfull, cnts.numpy(), labels.reshape(r1 - r0, C))
    dist.destroy_process_group()


def test_two_rank_shards_allreduce_and_bands():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    import oracle
    from synth.lidar import Scenario
    sc = Scenario("C1")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    tx, ty = oracle.theta(0, cfg["D"])
    m1, c1, _ = oracle.encode(tx, ty, cfg["l"], xy, lab)
    q = oracle.decode_grid(tx, ty, cfg["l"], m1, 0, 0, cfg["res"], 0, cfg["rows"], 0, cfg["cols"])
    _, L = oracle.entropy_grid(q, cfg["half"], cfg["half"], 0, 0.001, -0.001)
    for r in range(world):
        m, c, _ = out[r]
        np.testing.assert_allclose(m, m1, atol=1e-9)
        assert list(c) == list(c1)
    stitched = np.concatenate([out[r][2] for r in range(world)], axis=0)
    assert np.array_equal(stitched, L)


def test_shard_helpers_cover_exactly():
    from paper_2408_09066_b200.parallel import decoded_rows, point_shard, row_band
    for n, G in ((10_000_000, 8), (7, 3), (1, 2)):
        rs = [point_shard(n, g, G) for g in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
    bands = [row_band(4000, g, 8) for g in range(8)]
    assert bands[3] == (1500, 2000)
    assert decoded_rows(4000, 0, 500, 3) == (0, 503)
    assert decoded_rows(4000, 3500, 4000, 3) == (3497, 4000)
