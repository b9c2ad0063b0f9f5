"""GPU parity: the sm_100a path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (north_star):
  heatmap   max|q_gpu - q_orc| / max|q_orc| <= 1e-3 (fp16 operands, fp32 accumulate), <= 2e-2 (bf16)
  labels    agreement >= 99.9 % of compared cells
  memories  ||m_gpu - m_orc|| / ||m_orc|| <= 1e-4   (fp32 phase + MUFU sincos, derived in DESIGN.md)
  theta     bit-exact (two independent splitmix64 implementations)
"""
import math

import numpy as np
import pytest
import torch

import oracle
from conftest import label_tau
from synth.lidar import Scenario

pytestmark = pytest.mark.gpu

Q_TOL = {0: 1e-3, 1: 2e-2}
M_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _mapper(D, l, bounds, seed=0):
    from paper_2408_09066_b200 import Mapper
    return Mapper(D, seed, l, bounds)


def _cuda(xy, lab):
    return torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(np.ascontiguousarray(lab)).cuda()


def _qerr(qg, qo):
    return max(np.abs(qg[c] - qo[c]).max() / max(np.abs(qo[c]).max(), 1e-300) for c in (0, 1))


def _mem_err(mg, mo):
    return max(np.linalg.norm(mg[c] - mo[c]) / max(np.linalg.norm(mo[c]), 1e-300) for c in (0, 1))


# ------------------------------------------------------------------ building blocks

def test_theta_bit_exact():
    for D, seed in ((512, 0), (100, 7), (16384, 12345)):
        mp = _mapper(D, 0.3, (0, 0, 1, 1), seed)
        gx, gy = mp.get_phases()
        ox, oy = oracle.theta(seed, D)
        assert np.array_equal(gx, ox) and np.array_equal(gy, oy)
        mp.close()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 128), (1000, 777, 640), (4000, 2000, 1024),
                                   (257, 33, 192)])
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_gemm_vs_torch_fp32(M, N, K, prec, kernel):
    from paper_2408_09066_b200 import test_gemm
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    dt = torch.float16 if prec == 0 else torch.bfloat16
    A = torch.randn(M, K, device="cuda", generator=g).to(dt)
    B = torch.randn(N, K, device="cuda", generator=g).to(dt)
    C = test_gemm(A, B, prec, kernel)
    ref = A.float() @ B.float().T
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-4, err


@pytest.mark.parametrize("splits", [2, 3, 7])
@pytest.mark.parametrize("M,N,K", [(300, 500, 1024), (508, 2000, 4096)])
@pytest.mark.parametrize("kernel", [0, 2])
def test_gemm_split_k(splits, M, N, K, kernel):
    from paper_2408_09066_b200 import test_gemm
    g = torch.Generator(device="cuda").manual_seed(splits + M)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    B = torch.randn(N, K, device="cuda", generator=g).half()
    C = test_gemm(A, B, 0, kernel, splits=splits)
    ref = A.float() @ B.float().T
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-4


def test_decode_band_split_k_matches_unsplit():
    """A narrow row band (one rank of 8 at C4 scale) picks split-K automatically; its q and
    labels equal the forced unsplit decode up to fp32 summation order."""
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    D, l, h, R, C, res = 2048, 0.25, 2, 2000, 2000, 0.02
    mp = _mapper(D, l, sc.bounds)
    mp.set_tuning("dec_method", 0)   # the GEMM's split-K (the NUFFT decode has no split)
    mp.encode_bundle(*_cuda(xy, lab))
    out = []
    for s in (None, "1"):
        if s:
            mp.set_tuning("gemm_splits", int(s))
        q = torch.empty((2, 250, C), dtype=torch.float32, device="cuda")
        mp.decode(0, 0, res, R, C, 750, 1000, h, q_out=q)
        L = torch.empty((250, C), dtype=torch.uint8, device="cuda")
        mp.entropy(h, h, 0.001, -0.001, 0, None, L)
        out.append((q, L))
    assert mp.sync() == 0
    assert (out[0][0] - out[1][0]).abs().max().item() <= 1e-5 * out[1][0].abs().max().item() + 1e-7
    assert (out[0][1] == out[1][1]).float().mean().item() >= 0.9999
    mp.close()


@pytest.mark.parametrize("bn", [256, 224, 192, 160, 128])
@pytest.mark.parametrize("kernel", [0, 2])
def test_gemm_pair_tile_widths(bn, kernel):
    from paper_2408_09066_b200 import test_gemm
    g = torch.Generator(device="cuda").manual_seed(bn)
    A = torch.randn(600, 320, device="cuda", generator=g).half()
    B = torch.randn(1000, 320, device="cuda", generator=g).half()
    C = test_gemm(A, B, 0, kernel, bn=bn)
    ref = A.float() @ B.float().T
    assert (C - ref).abs().max().item() / ref.abs().max().item() < 1e-4


# ------------------------------------------------------------------ end-to-end configs

def _run_full(name, prec=0, q_out=True):
    sc = Scenario(name)
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, h = cfg["D"], cfg["l"], cfg["half"]
    R, C, res = cfg["rows"], cfg["cols"], cfg["res"]
    tau = label_tau(D)
    mp = _mapper(D, l, sc.bounds)
    mp.encode_bundle(*_cuda(xy, lab))
    q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0.0, 0.0, res, R, C, 0, R, h, precision=prec, q_out=q)
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, tau, -tau, 0, S, L)
    assert mp.sync() == 0
    mg, cg = mp.get_memory()
    mp.close()
    return sc, xy, lab, mg, cg, q.cpu().numpy().astype(np.float64), S.cpu().numpy(), L.cpu().numpy()


@pytest.fixture(scope="module")
def c1_oracle():
    sc = Scenario("C1")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    tx, ty = oracle.theta(0, cfg["D"])
    m, cnt, _ = oracle.encode(tx, ty, cfg["l"], xy, lab)
    q = oracle.decode_grid(tx, ty, cfg["l"], m, 0, 0, cfg["res"], 0, cfg["rows"], 0, cfg["cols"])
    return tx, ty, m, cnt, q


def test_c1_memory_heatmap_labels(c1_oracle):
    tx, ty, mo, co, qo = c1_oracle
    sc, xy, lab, mg, cg, qg, Sg, Lg = _run_full("C1")
    assert list(cg) == list(co)
    assert _mem_err(mg, mo) <= M_TOL
    assert _qerr(qg, qo) <= Q_TOL[0]
    h, D = sc.cfg["half"], sc.cfg["D"]
    tau = label_tau(D)
    So, Lo = oracle.entropy_grid(qo, h, h, 0, tau, -tau)
    assert (Lg == Lo).mean() >= 0.999
    assert np.abs(Sg - So).max() <= 1e-3 * np.abs(So).max() + 1e-6


def test_c1_bf16(c1_oracle):
    _, _, _, _, qo = c1_oracle
    *_, qg, _, _ = _run_full("C1", prec=1)
    assert _qerr(qg, qo) <= Q_TOL[1]


def test_c2_full_grid():
    sc, xy, lab, mg, cg, qg, Sg, Lg = _run_full("C2")
    cfg = sc.cfg
    tx, ty = oracle.theta(0, cfg["D"])
    mo, co, _ = oracle.encode(tx, ty, cfg["l"], xy, lab)
    assert list(cg) == list(co)
    assert _mem_err(mg, mo) <= M_TOL
    qo = oracle.decode_grid(tx, ty, cfg["l"], mo, 0, 0, cfg["res"], 0, cfg["rows"], 0, cfg["cols"])
    assert _qerr(qg, qo) <= Q_TOL[0]
    tau = label_tau(cfg["D"])
    So, Lo = oracle.entropy_grid(qo, cfg["half"], cfg["half"], 0, tau, -tau)
    assert (Lg == Lo).mean() >= 0.999


# C3 / C4 (streamed, bench schedule) / C5 at full size: tests/test_gpu_parity_large.py


def test_nccl_fuse_and_commit_single_rank():
    """The multi-rank step's collective path on a 1-rank NCCL group: the library's pending
    buffer wrapped as a torch tensor, all-reduced in place, committed."""
    import os
    import torch.distributed as dist
    from paper_2408_09066_b200.parallel import fuse_and_commit
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sc = Scenario("C1")
        xy, lab = sc.all_points()
        D, l = sc.cfg["D"], sc.cfg["l"]
        mp = _mapper(D, l, sc.bounds)
        mp.encode_bundle(*_cuda(xy, lab))
        pend = mp.pending()
        assert pend.shape == (2, mp.Dp, 2) and pend.dtype == torch.float64
        dist.all_reduce(pend)          # world of 1: identity, exercised on library-owned memory
        fuse_and_commit(mp)
        mg, cg = mp.get_memory()
        tx, ty = oracle.theta(0, D)
        mo, co, _ = oracle.encode(tx, ty, l, xy, lab)
        assert list(cg) == list(co)
        assert _mem_err(mg, mo) <= M_TOL
        mp.decode(0, 0, 0.1, 100, 100)   # committed: multi-rank decode is allowed
        mp.close()
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ properties and edge cases

def test_single_point_self_similarity_and_empty_class():
    D, l, res = 1024, 0.25, 0.1
    mp = _mapper(D, l, (0, 0, 5, 5))
    r, c = 17, 23
    pt = np.array([[(c + 0.5) * res, (r + 0.5) * res]], np.float32)
    mp.encode_bundle(*_cuda(pt, np.array([1], np.uint8)))
    q = torch.empty((2, 50, 50), dtype=torch.float32, device="cuda")
    mp.decode(0.0, 0.0, res, 50, 50, 0, 50, 1, q_out=q)
    mp.entropy(1, 1, 0.0, 0.0)
    assert mp.sync() == 0
    qn = q.cpu().numpy()
    assert abs(qn[1, r, c] - 1.0) < 2e-3
    assert np.all(qn[0] == 0.0)                  # empty class decodes to 0 (L8)
    assert np.abs(qn[1]).max() <= 1.0 + 2e-3
    mp.close()


def test_ragged_dims_and_band_stitching():
    # D not a multiple of 32, grid not a multiple of the tiles, 3 row bands with halo == full grid
    D, l, res, R, C, h = 100, 0.3, 0.07, 77, 300, 2
    rng = np.random.default_rng(1)
    xy = rng.uniform(0, [C * res, R * res], size=(5000, 2)).astype(np.float32)
    lab = (rng.random(5000) < 0.3).astype(np.uint8)
    mp = _mapper(D, l, (0, 0, C * res, R * res))
    # the GEMM decode: its row bands are bit-identical to the full grid (the NUFFT decode centres each
    # band on its own rows, so its bands agree to ~1e-6: tests/test_gpu_nudecode.py)
    mp.set_tuning("dec_method", 0)
    mp.encode_bundle(*_cuda(xy, lab))
    qf = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, res, R, C, 0, R, h, q_out=qf)
    Lf = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    Sf = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    mp.entropy(h, h, 0.001, -0.001, 0, Sf, Lf)
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
    assert _qerr(qf.cpu().numpy(), qo) <= Q_TOL[0]
    from paper_2408_09066_b200.parallel import row_band
    for g in range(3):
        r0, r1 = row_band(R, g, 3)
        qb = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
        mp.decode(0, 0, res, R, C, r0, r1, h, q_out=qb)
        Sb = torch.empty((3, r1 - r0, C), dtype=torch.float32, device="cuda")
        Lb = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
        mp.entropy(h, h, 0.001, -0.001, 0, Sb, Lb)
        assert torch.equal(qb, qf[:, r0:r1])
        assert torch.equal(Lb, Lf[r0:r1])
        assert torch.allclose(Sb, Sf[:, r0:r1], atol=1e-6)
    assert mp.sync() == 0
    mp.close()


@pytest.mark.parametrize("disk", [0, 1])
def test_entropy_disk_and_per_class_radii(disk):
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    cfg = sc.cfg
    D, l, R, C, res = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"]
    h1, h0 = 3, 2
    mp = _mapper(D, l, sc.bounds)
    mp.encode_bundle(*_cuda(xy, lab))
    q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, res, R, C, 0, R, 3, q_out=q)
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h1, h0, 0.002, -0.002, disk, S, L)
    assert mp.sync() == 0
    # oracle entropy on the GPU's own q (isolates the stencil): fp32 vs fp64 sums only
    So, Lo = oracle.entropy_grid(q.cpu().numpy().astype(np.float64), h1, h0, disk, 0.002, -0.002)
    assert np.abs(S.cpu().numpy() - So).max() <= 2e-5
    assert (L.cpu().numpy() == Lo).mean() >= 0.9999
    mp.close()


@pytest.mark.parametrize("disk", [0, 1])
@pytest.mark.parametrize("h", [1, 3, 7])
def test_entropy_equal_radii_fast_path(disk, h):
    """The compile-time-window kernel (equal radii, h <= 8) vs the oracle stencil on the
    GPU's own q, on a ragged grid (cols not a multiple of 4 or of the 128-column tile)."""
    D, l, res, R, C = 256, 0.3, 0.07, 71, 203
    rng = np.random.default_rng(h + 10 * disk)
    xy = rng.uniform(0, [C * res, R * res], size=(3000, 2)).astype(np.float32)
    lab = (rng.random(3000) < 0.4).astype(np.uint8)
    mp = _mapper(D, l, (0, 0, C * res, R * res))
    mp.encode_bundle(*_cuda(xy, lab))
    q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, res, R, C, 0, R, h, q_out=q)
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, 0.001, -0.001, disk, S, L)
    assert mp.sync() == 0
    So, Lo = oracle.entropy_grid(q.cpu().numpy().astype(np.float64), h, h, disk, 0.001, -0.001)
    assert np.abs(S.cpu().numpy() - So).max() <= 2e-5
    assert (L.cpu().numpy() == Lo).mean() >= 0.9999
    # band with halo: same rows as the full grid
    r0, r1 = 20, 50
    mp.decode(0, 0, res, R, C, r0, r1, h)
    Sb = torch.empty((3, r1 - r0, C), dtype=torch.float32, device="cuda")
    mp.entropy(h, h, 0.001, -0.001, disk, Sb, None)
    assert torch.allclose(Sb, S[:, r0:r1], atol=1e-6)
    mp.close()



@pytest.mark.parametrize("h", [1, 2, 3, 4])
@pytest.mark.parametrize("R,C,rw", [(75, 203, 0), (75, 203, 3), (300, 1000, 0), (300, 1000, 5), (64, 2000, 7)])
def test_entropy_stream_kernel(h, R, C, rw):
    """k_entropy_cols (the default: a thread walks 4 columns down a chunk of rows) and k_entropy_stream
    (TMA-streamed warps) -- box windows h <= 4, labels only, running vertical sums of the class
    difference -- against the generic staged kernel and the oracle: on ragged
    grids (203 and 1000 columns: partial strips, C not a multiple of 8), on bands with halo
    rows, and with short work items (rw) so that warps stream several items through their
    stage rings and the work queue wraps; S from the generic kernel is within 2e-5 of the
    oracle, the labels of both kernels agree with each other and with the oracle."""
    D, l, res = 256, 0.3, 0.07
    rng = np.random.default_rng(100 + h)
    xy = rng.uniform(0, [C * res, R * res], size=(3000, 2)).astype(np.float32)
    lab = (rng.random(3000) < 0.4).astype(np.uint8)
    mp = _mapper(D, l, (0, 0, C * res, R * res))
    mp.encode_bundle(*_cuda(xy, lab))
    q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.set_tuning("entropy_rw", rw)
    outs = {}
    for kernel in (0, 2, 1):   # both labels-only box kernels (0 column walk, 2 TMA-streamed), then the generic one
        mp.set_tuning("entropy_kernel", kernel)
        outs[kernel] = []
        for (r0, r1) in ((0, R), (21, 58), (R - 17, R)):
            mp.decode(0, 0, res, R, C, r0, r1, h, q_out=q if (r0, r1) == (0, R) else None)
            L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
            mp.entropy(h, h, 0.001, -0.001, 0, None, L)
            outs[kernel].append(L.cpu())
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, res, R, C, 0, R, h)
    mp.entropy(h, h, 0.001, -0.001, 0, S, None)          # S maps: the generic kernel
    assert mp.sync() == 0
    So, Lo = oracle.entropy_grid(q.cpu().numpy().astype(np.float64), h, h, 0, 0.001, -0.001)
    assert np.abs(S.cpu().numpy() - So).max() <= 2e-5
    for fast in (0, 2):
        for a, b in zip(outs[fast], outs[1]):
            assert (a == b).float().mean().item() >= 0.9999
        assert (outs[fast][0].numpy() == Lo).mean() >= 0.9999
        assert torch.equal(outs[fast][1], outs[fast][0][21:58]) and torch.equal(outs[fast][2], outs[fast][0][R - 17:])
    mp.close()


def test_streaming_equals_one_shot_and_reset():
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    D, l = sc.cfg["D"], sc.cfg["l"]
    mp = _mapper(D, l, sc.bounds)
    half = len(lab) // 2
    mp.encode_bundle(*_cuda(xy[:half], lab[:half]))
    mp.commit()
    mp.encode_bundle(*_cuda(xy[half:], lab[half:]))
    m2, c2 = mp.get_memory()
    mp.reset()
    m0, c0 = mp.get_memory()
    assert np.all(m0 == 0) and list(c0) == [0, 0]
    mp.encode_bundle(*_cuda(xy, lab))
    m1, c1 = mp.get_memory()
    assert list(c1) == list(c2)
    assert _mem_err(m2, m1) <= 1e-5
    mp.close()


def test_errors_and_deferred_errors():
    from paper_2408_09066_b200.vsaogm import EEMPTY, ELABEL, ENONFINITE, ESTATE, VsaogmError
    D, l = 256, 0.3
    mp = _mapper(D, l, (0, 0, 4, 4))
    xy = np.array([[1, 1], [2, 2], [np.nan, 1], [3, 3]], np.float32)
    lab = np.array([1, 7, 0, 0], np.uint8)
    mp.encode_bundle(*_cuda(xy, lab))
    assert mp.sync() == ELABEL
    assert mp.sync() == 0                     # cleared after being reported
    mg, cg = mp.get_memory()
    tx, ty = oracle.theta(0, D)
    mo, co, bad = oracle.encode(tx, ty, l, xy, lab)
    assert bad == 2 and list(cg) == list(co) == [1, 1]
    assert _mem_err(mg, mo) <= M_TOL
    mp.encode_bundle(*_cuda(np.array([[np.inf, 0]], np.float32), np.array([0], np.uint8)))
    assert mp.sync() == ENONFINITE
    with pytest.raises(VsaogmError) as e:
        mp.encode_bundle(torch.empty((0, 2), device="cuda"), torch.empty(0, dtype=torch.uint8, device="cuda"))
    assert e.value.code == EEMPTY
    with pytest.raises(VsaogmError) as e:
        mp.entropy(1, 1, 0.0, 0.0)            # no decode yet
    assert e.value.code == ESTATE
    # multi-rank mode: decode refuses uncommitted pending work
    mp.pending()
    mp.encode_bundle(*_cuda(xy[:1], lab[:1]))
    with pytest.raises(VsaogmError) as e:
        mp.decode(0, 0, 0.1, 10, 10)
    assert e.value.code == ESTATE
    mp.commit()
    mp.decode(0, 0, 0.1, 10, 10)
    mp.entropy(3, 3, 0.0, 0.0)                # whole grid: no neighbouring band, any window is fine
    mp.decode(0, 0, 0.1, 10, 10, 0, 5, 2)
    mp.entropy(2, 2, 0.0, 0.0)
    with pytest.raises(VsaogmError):
        mp.entropy(3, 3, 0.0, 0.0)            # wider than the decode halo of a band
    mp.close()


def test_multi_rank_emulated_on_one_gpu():
    """G point shards in G contexts, pending summed on the device (the all-reduce),
    committed: equals the 1-shot memory; decode identical up to rounding."""
    from paper_2408_09066_b200.parallel import point_shard
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    D, l = sc.cfg["D"], sc.cfg["l"]
    G = 4
    ms = [_mapper(D, l, sc.bounds) for _ in range(G)]
    for g, mp in enumerate(ms):
        lo, hi = point_shard(len(lab), g, G)
        mp.encode_bundle(*_cuda(xy[lo:hi], lab[lo:hi]))
    pend = [mp.pending() for mp in ms]
    cnts = [mp.pending_counts() for mp in ms]
    torch.cuda.synchronize()
    tot = sum(p.clone() for p in pend)
    totc = sum(c.clone() for c in cnts)
    for mp, p, c in zip(ms, pend, cnts):
        p.copy_(tot)
        c.copy_(totc)
        mp.commit()
    one = _mapper(D, l, sc.bounds)
    one.encode_bundle(*_cuda(xy, lab))
    m1, c1 = one.get_memory()
    for mp in ms:
        mg, cg = mp.get_memory()
        assert list(cg) == list(c1)
        assert _mem_err(mg, m1) <= 1e-6
    for mp in ms + [one]:
        mp.close()


def test_pipelined_host_steps_match_synchronous():
    """vsaogm_encode_bundle_host_async / vsaogm_entropy_host_async / vsaogm_wait: a pipelined run
    of several streaming steps (copies on the upload / download streams, four slots each)
    returns, per step, the same labels and S as the synchronous host path."""
    import math
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    p = 1.0 / (2.0 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    xy, lab = sc.all_points()
    chunks = np.array_split(np.arange(len(lab)), 5)
    batches = [(torch.from_numpy(np.ascontiguousarray(xy[c])).pin_memory(),
                torch.from_numpy(np.ascontiguousarray(lab[c])).pin_memory()) for c in chunks]
    ref = []
    mp = Mapper(D, 0, l, sc.bounds)
    for bx, bl in batches:
        L = torch.empty((R, C), dtype=torch.uint8).pin_memory()
        S = torch.empty((3, R, C), dtype=torch.float32).pin_memory()
        mp.encode_bundle_host(bx, bl)
        mp.decode(0.0, 0.0, res, R, C, 0, R, h)
        mp.entropy_host(h, h, tau, -tau, 0, S, L)
        ref.append((L.clone(), S.clone()))
    mp.close()
    mp = Mapper(D, 0, l, sc.bounds)
    outs = [(torch.empty((R, C), dtype=torch.uint8).pin_memory(), torch.empty((3, R, C), dtype=torch.float32).pin_memory())
            for _ in batches]
    tickets = []
    for k, (bx, bl) in enumerate(batches):
        mp.encode_bundle_host_async(bx, bl)
        mp.decode(0.0, 0.0, res, R, C, 0, R, h)
        tickets.append(mp.entropy_host_async(h, h, tau, -tau, 0, outs[k][1], outs[k][0]))
        if k >= 1:
            assert mp.wait(tickets[k - 1]) == 0
            assert torch.equal(outs[k - 1][0], ref[k - 1][0])
            assert torch.equal(outs[k - 1][1], ref[k - 1][1])
    assert mp.wait(tickets[-1]) == 0
    assert torch.equal(outs[-1][0], ref[-1][0]) and torch.equal(outs[-1][1], ref[-1][1])
    with pytest.raises(Exception):
        mp.wait(len(batches) + 3)
    mp.close()


def test_encode_stream_pipeline_matches_serial():
    """vsaogm_set_encode_stream: encodes on a second (low-priority) stream overlapping the previous
    decode give, step for step, the labels and S of the one-stream schedule, and the same
    memories; commit / reset / pending / the async host path keep their call order."""
    import math
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], cfg["cols"], cfg["res"]
    p = 1.0 / (2.0 * D)
    tau = -p * math.log2(p) - (1 - p) * math.log2(1 - p)
    xy, lab = sc.all_points()
    chunks = np.array_split(np.arange(len(lab)), 6)
    dev = [_cuda(np.ascontiguousarray(xy[c]), np.ascontiguousarray(lab[c])) for c in chunks]
    pinned = [(torch.from_numpy(np.ascontiguousarray(xy[c])).pin_memory(),
               torch.from_numpy(np.ascontiguousarray(lab[c])).pin_memory()) for c in chunks]

    def schedule(pipelined):
        hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
        outs = []
        with torch.cuda.stream(hi):
            mp = Mapper(D, 0, l, sc.bounds)
            if pipelined:
                mp.set_encode_stream(lo)
            for k in range(4):
                if k == 2:
                    mp.encode_bundle_host(*pinned[k])   # library-owned staging buffers
                else:
                    mp.encode_bundle(*dev[k])
                if k == 1:
                    mp.encode_bundle_host(*pinned[4])   # two encodes before one decode, the second
                    mp.encode_bundle_host(*pinned[3])   # and third reusing the staging buffers
                mp.decode(0.0, 0.0, res, R, C, 0, R, h)
                S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
                L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
                mp.entropy(h, h, tau, -tau, 0, S, L)
                outs.append((S, L))
            mp.encode_bundle(*dev[5])
            mp.commit()                            # explicit commit, then reset and start again
            m_commit = mp.get_memory()
            mp.reset()
            mp.encode_bundle(*dev[0])
            pend = mp.pending().clone()            # pending view after the encode
            mp.commit()
            labs = torch.empty((R, C), dtype=torch.uint8).pin_memory()
            mp.encode_bundle_host_async(*pinned[1])
            mp.commit()                            # multi-rank mode since pending(): explicit commit
            mp.decode(0.0, 0.0, res, R, C, 0, R, h)
            t = mp.entropy_host_async(h, h, tau, -tau, 0, None, labs)
            assert mp.wait(t) == 0
            torch.cuda.synchronize()
            mem = mp.get_memory()
            assert mp.sync() == 0
            mp.close()
        return outs, m_commit, pend, labs, mem

    a, b = schedule(False), schedule(True)
    for (Sa, La), (Sb, Lb) in zip(a[0], b[0]):
        assert torch.equal(Sa, Sb) and torch.equal(La, Lb)
    assert np.array_equal(a[1][0], b[1][0]) and list(a[1][1]) == list(b[1][1])
    assert torch.equal(a[2], b[2])
    assert torch.equal(a[3], b[3])
    assert np.array_equal(a[4][0], b[4][0]) and list(a[4][1]) == list(b[4][1])


@pytest.mark.parametrize("delta,prec", [(1, 0), (1, 1), (2, 0)])
def test_gemm_phasor_tiles_on_the_fly(delta, prec):
    """gemm_agen = 1: the decode GEMM generates its A phasor tiles in shared memory (row
    recurrence, no table A).  q equals the table-A decode within the 16-bit operand rounding
    (1e-3 of peak fp16, 2e-2 bf16) and the oracle within the north_star bounds, on a full grid
    with a class boundary inside an A tile, on a row band with halo rows (split-K), and with
    quadrant memories (grouped GEMM); labels agree."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    cfg = sc.cfg
    D, l, h, R, C, res = cfg["D"], cfg["l"], cfg["half"], cfg["rows"], 333, cfg["res"]
    tau = label_tau(D)
    mp = Mapper(D, 0, l, sc.bounds, delta=delta)
    mp.set_tuning("dec_method", 0)   # both variants of the GEMM decode
    mp.encode_bundle(*_cuda(xy, lab))
    outs = {}
    for agen in (0, 1):
        mp.set_tuning("gemm_agen", agen)
        for (r0, r1) in ((0, R), (150, 250)):
            q = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
            mp.decode(0.0, 0.0, res, R, C, r0, r1, h, precision=prec, q_out=q)
            L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
            mp.entropy(h, h, tau, -tau, 0, None, L)
            outs[(agen, r0)] = (q.cpu().numpy().astype(np.float64), L.cpu().numpy())
    assert mp.sync() == 0
    mp.close()
    tol = Q_TOL[prec]
    for r0 in (0, 150):
        qa, La = outs[(0, r0)]
        qb, Lb = outs[(1, r0)]
        assert _qerr(qb, qa) <= tol, _qerr(qb, qa)
        assert (La == Lb).mean() >= 0.999
    if delta == 1:
        tx, ty = oracle.theta(0, D)
        mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
        qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
        assert _qerr(outs[(1, 0)][0], qo) <= tol


@pytest.mark.parametrize("cfg", ["C2", "C4"])
def test_encode_methods_agree_and_nufft_reproducible(cfg):
    """The type-3 NUFFT encode (enc_method 1) and the direct pair kernel (0) give the same
    memories within their fp32 error (each is within ~1.5e-5 of the fp64 oracle, the NUFFT within
    ~1e-6), the same counts; two NUFFT encodes of the same points are bit-identical (fixed-point
    spreading, fixed-order reductions)."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario(cfg)
    xy, lab = sc.batch(0) if sc.cfg["batch_scans"] else sc.all_points()
    D, l = sc.cfg["D"], sc.cfg["l"]
    mems = {}
    for method in (0, 1):
        mp = Mapper(D, 0, l, sc.bounds)
        mp.set_tuning("enc_method", method)
        mp.encode_bundle(*_cuda(xy, lab))
        mems[method] = mp.get_memory()
        if method == 1:
            mp.reset()
            mp.encode_bundle(*_cuda(xy, lab))
            again = mp.get_memory()
            assert np.array_equal(again[0], mems[1][0]) and list(again[1]) == list(mems[1][1])
        mp.close()
    assert list(mems[0][1]) == list(mems[1][1])
    assert _mem_err(mems[1][0], mems[0][0]) <= 5e-5
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode(tx, ty, l, xy, lab)
    assert _mem_err(mems[1][0], mo) <= 1e-5


def test_nufft_outliers_and_single_class():
    """Points off the NUFFT grid (far outside the world bounds: the direct fallback) and a batch
    with one class only: memories equal the oracle's, the empty class stays exactly zero."""
    from paper_2408_09066_b200 import Mapper
    rng = np.random.default_rng(7)
    D, l, W = 4096, 0.3, 40.0
    xy = rng.uniform(0, W, size=(60000, 2)).astype(np.float32)
    xy[:500] = rng.uniform(-3 * W, 4 * W, size=(500, 2)).astype(np.float32)   # outliers
    lab = (rng.random(60000) < 0.3).astype(np.uint8)
    tx, ty = oracle.theta(0, D)
    for labels in (lab, np.ones_like(lab)):
        mp = Mapper(D, 0, l, (0.0, 0.0, W, W))
        mp.set_tuning("enc_method", 1)
        mp.encode_bundle(*_cuda(xy, labels))
        assert mp.sync() == 0
        mg, cg = mp.get_memory()
        mp.close()
        mo, co, _ = oracle.encode(tx, ty, l, xy, labels)
        assert list(cg) == list(co)
        for c in (0, 1):
            if co[c]:
                assert np.linalg.norm(mg[c] - mo[c]) <= 1e-5 * np.linalg.norm(mo[c])
            else:
                assert not np.any(mg[c])


@pytest.mark.parametrize("W", [9.6, 23.0, 50.0, 105.0, 215.0, 432.0])
def test_nufft_transform_sizes(W):
    """The NUFFT encode at every transform size (l = 0.3: N = 256 ... 8192 as the world grows,
    odd and even log2 N, fewer values than threads per stage at the small end) equals the oracle
    within 1e-5; the counts are exact."""
    from paper_2408_09066_b200 import Mapper
    rng = np.random.default_rng(int(W * 10))
    D, l = 2048, 0.3
    xy = rng.uniform(0, W, size=(20000, 2)).astype(np.float32)
    lab = (rng.random(20000) < 0.25).astype(np.uint8)
    mp = Mapper(D, 0, l, (0.0, 0.0, W, W))
    mp.set_tuning("enc_method", 1)
    for _ in range(2):   # the second encode checks that the row pass left the grid clean
        mp.reset()
        mp.encode_bundle(*_cuda(xy, lab))
        assert mp.sync() == 0
        mg, cg = mp.get_memory()
    mp.close()
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode(tx, ty, l, xy, lab)
    assert list(cg) == list(co)
    assert _mem_err(mg, mo) <= 1e-5
