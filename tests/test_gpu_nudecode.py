"""GPU parity of the type-1 NUFFT decode (csrc/nudecode.cu) against the fp64
oracle's direct evaluation of Eq. 11 (oracle.decode_grid: every cell summed over k, no factorisation).

Tolerances: heatmap max|q_gpu - q_orc| / max|q_orc| <= 5e-5 (Gaussian gridding
with msp = 5 and fp32 transforms: ~1e-6; plus the fp32 encode's memory error), i.e. 20x inside the
north_star's 1e-3 bar; labels >= 99.9 %; reruns bit-identical (fixed-order gather, no atomics).
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import label_tau
from synth.lidar import Scenario

pytestmark = pytest.mark.gpu

Q_NU = 5e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _qerr(qg, qo):
    return max(np.abs(qg[c] - qo[c]).max() / max(np.abs(qo[c]).max(), 1e-300) for c in (0, 1))


def _decode(mp, x0, y0, res, R, C, r0, r1, halo, method):
    mp.set_tuning("dec_method", method)
    mp.profile_enable(True)
    q = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
    mp.decode(x0, y0, res, R, C, r0, r1, halo, q_out=q)
    assert mp.sync() == 0
    prof = mp.profile_read()
    mp.profile_enable(False)
    return q.cpu().numpy().astype(np.float64), prof


@pytest.mark.parametrize("method", [0, 1])
def test_c2_full_grid_both_methods(method):
    """C2 end to end with each decode method: q vs the oracle (NUFFT: 5e-5; GEMM: 1e-3), labels
    >= 99.9 %; the NUFFT decode is the one that ran (its profile id), and a rerun is bit-identical."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, R, C, res, h = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"], cfg["half"]
    mp = Mapper(D, 0, l, sc.bounds)
    mp.encode_bundle(_cuda(xy), _cuda(lab))
    qg, prof = _decode(mp, 0, 0, res, R, C, 0, R, 0, method)
    ran = "nd_rowfft" if method == 1 else "decode_gemm"
    assert prof[ran][1] >= 1
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    tau = label_tau(D)
    mp.entropy(h, h, tau, -tau, 0, S, L)
    q2, _ = _decode(mp, 0, 0, res, R, C, 0, R, 0, method)
    assert np.array_equal(q2, qg)
    mp.close()
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
    assert _qerr(qg, qo) <= (Q_NU if method == 1 else 1e-3)
    So, Lo = oracle.entropy_grid(qo, h, h, 0, tau, -tau)
    assert (L.cpu().numpy() == Lo).mean() >= 0.999
    assert np.abs(S.cpu().numpy() - So).max() <= 1e-4 * np.abs(So).max() + 1e-6


# (D, l, res, R, C, r0, r1, halo, x0, y0): transform sizes 256 .. 8192 on both axes, odd and ragged
# sizes, one-row bands, bands with clipped and interior halos, grids off the bounds centre
GEOMS = [
    (512, 0.3, 0.05, 1, 1, 0, 1, 0, 3.0, 4.0),           # one cell (M = 256 both axes)
    (1024, 0.3, 0.05, 37, 53, 0, 37, 0, -1.3, 2.7),      # ragged, odd
    (2048, 0.25, 0.1, 400, 400, 150, 151, 2, 0.0, 0.0),  # one-row band with halo
    (2048, 0.3, 0.05, 4000, 9, 1000, 1100, 3, 0.0, 0.0), # tall: logy from the band (r_ext 106)
    (2048, 0.3, 0.05, 300, 4000, 0, 300, 0, 0.0, 0.0),   # wide: logx = 13
    (1024, 0.3, 0.07, 3000, 64, 0, 3000, 0, 0.0, 0.0),   # logy = 13
    (4096, 0.3, 0.1, 1000, 1000, 0, 1000, 0, 0.0, 0.0),  # C3 geometry
    (2048, 0.3, 0.05, 600, 700, 590, 600, 4, 12.0, -7.0),  # band at the last rows, clipped halo
]


@pytest.mark.parametrize("geom", GEOMS)
def test_nudecode_geometries(geom):
    """The NUFFT decode at every transform size and shape vs the oracle on the decoded band
    (all cells when the oracle finishes in seconds, else a seeded sample of rows); the halo rows
    enter through the entropy of the band, which must equal the full-grid entropy rows."""
    from paper_2408_09066_b200 import Mapper
    D, l, res, R, C, r0, r1, halo, x0, y0 = geom
    rng = np.random.default_rng(D + R + C)
    W = max(R, C) * res
    bounds = (x0, y0, x0 + C * res, y0 + R * res)
    n = 20000
    xy = np.stack([rng.uniform(x0 - 1, x0 + C * res + 1, n), rng.uniform(y0 - 1, y0 + R * res + 1, n)], 1)
    xy = xy.astype(np.float32)
    lab = (rng.random(n) < 0.35).astype(np.uint8)
    mp = Mapper(D, 0, l, bounds)
    mp.encode_bundle(_cuda(xy), _cuda(lab))
    qg, prof = _decode(mp, x0, y0, res, R, C, r0, r1, halo, 1)
    assert prof["nd_rowfft"][1] >= 1
    mp.close()
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    rows = np.arange(r0, r1)
    if len(rows) * C * D > 1e9:
        rows = np.sort(rng.choice(rows, size=max(1, int(1e9 // (C * D))), replace=False))
    qo = np.concatenate([oracle.decode_grid(tx, ty, l, mo, x0, y0, res, r, r + 1, 0, C) for r in rows], axis=1)
    assert _qerr(qg[:, rows - r0], qo) <= Q_NU, W


def test_nudecode_band_entropy_equals_full_grid():
    """Row bands with halos decoded by the NUFFT stitch to the full-grid labels exactly."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, R, C, res, h = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"], cfg["half"]
    tau = label_tau(D)
    mp = Mapper(D, 0, l, sc.bounds)
    mp.set_tuning("dec_method", 1)
    mp.encode_bundle(_cuda(xy), _cuda(lab))
    mp.decode(0, 0, res, R, C, 0, R, h)
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, tau, -tau, 0, None, L)
    full = L.clone()
    for b0, b1 in ((0, 97), (97, 250), (250, 400)):
        mp.decode(0, 0, res, R, C, b0, b1, h)
        Lb = torch.empty((b1 - b0, C), dtype=torch.uint8, device="cuda")
        mp.entropy(h, h, tau, -tau, 0, None, Lb)
        assert mp.sync() == 0
        assert torch.equal(Lb, full[b0:b1])
    mp.close()


def test_nudecode_empty_class_and_single_point():
    """One occupied point, no empty points: q_0 is exactly 0 everywhere (L8), q_1 peaks at 1 at
    the point's own cell centre (self-similarity D / (sqrt(D) ||m||) = 1) within 1e-5."""
    from paper_2408_09066_b200 import Mapper
    D, l, res, R, C = 4096, 0.3, 0.05, 200, 300
    x0, y0 = 0.0, 0.0
    pt = np.array([[x0 + (121 + 0.5) * res, y0 + (77 + 0.5) * res]], dtype=np.float32)
    mp = Mapper(D, 0, l, (x0, y0, x0 + C * res, y0 + R * res))
    mp.encode_bundle(_cuda(pt), _cuda(np.ones(1, np.uint8)))
    qg, _ = _decode(mp, x0, y0, res, R, C, 0, R, 0, 1)
    mp.close()
    assert not np.any(qg[0])
    assert abs(qg[1, 77, 121] - 1.0) <= 1e-5
    assert np.unravel_index(np.argmax(qg[1]), qg[1].shape) == (77, 121)


def test_nudecode_c1_falls_back_to_gemm():
    """C1's grid spacing is l / 2: the NUFFT band would fill the zero-padded half, so dec_method 1
    falls back to the GEMM (its profile id), still within the 1e-3 bar."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C1")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, R, C, res = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"]
    mp = Mapper(D, 0, l, sc.bounds)
    mp.encode_bundle(_cuda(xy), _cuda(lab))
    qg, prof = _decode(mp, 0, 0, res, R, C, 0, R, 0, 1)
    mp.close()
    assert prof["decode_gemm"][1] >= 1 and prof["nd_rowfft"][1] == 0
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
    assert _qerr(qg, qo) <= 1e-3


def test_nudecode_histogram_estimator():
    """The 8-bit code epilogue of the NUFFT decode: codes equal the kernel-precision decision on
    the NUFFT's own q (fp32 p, fp32 code), and labels agree with the GEMM path's on >= 99 %."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, R, C, res, h = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"], cfg["half"]
    labs = {}
    for method in (0, 1):
        mp = Mapper(D, 0, l, sc.bounds)
        mp.set_estimator(1)
        mp.set_tuning("dec_method", method)
        mp.encode_bundle(_cuda(xy), _cuda(lab))
        q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
        mp.decode(0, 0, res, R, C, 0, R, h, q_out=q)
        L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
        S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
        mp.entropy(h, h, 0.1, -0.1, 0, S, L)
        assert mp.sync() == 0
        labs[method] = L.cpu().numpy()
        if method == 1:
            q32 = q.cpu().numpy().astype(np.float32)
            p = np.minimum(q32 * q32, np.float32(1)).astype(np.float64)
            So, Lo = oracle.entropy_hist_grid(p, h, h, 0, 0.1, -0.1)
            assert np.abs(S.cpu().numpy() - So).max() <= 2e-5
            assert (labs[1] == Lo).mean() >= 0.9999
        mp.close()
    assert (labs[0] == labs[1]).mean() >= 0.99


def test_dependent_launches_bit_identical():
    """Programmatic dependent launch (tuning knob pdl) only changes when a
    kernel's blocks are scheduled, never what they read: with the NUFFT encode and decode forced
    (the whole chain of dependent kernels), streamed steps on one stream and on the pipelined
    schedule give bit-identical memories, q and labels with pdl = 1 and pdl = 0."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D, l, R, C, res, h = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"], cfg["half"]
    tau = label_tau(D)
    chunks = np.array_split(np.arange(len(lab)), 4)
    dev = [(_cuda(xy[c]), _cuda(lab[c])) for c in chunks]

    def run(pdl, pipelined):
        hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
        outs = []
        with torch.cuda.stream(hi):
            mp = Mapper(D, 0, l, sc.bounds)
            mp.set_tuning("pdl", pdl)
            mp.set_tuning("enc_method", 1)
            mp.set_tuning("dec_method", 1)
            if pipelined:
                mp.set_encode_stream(lo)
            for x, y in dev:
                mp.encode_bundle(x, y)
                q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
                L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
                mp.decode(0, 0, res, R, C, 0, R, h, q_out=q)
                mp.entropy(h, h, tau, -tau, 0, None, L)
                outs.append((q, L))
            assert mp.sync() == 0
            mem = mp.get_memory()
            mp.close()
        return outs, mem

    ref = run(0, False)
    for pdl, pipelined in ((1, False), (1, True), (0, True)):
        got = run(pdl, pipelined)
        for (qa, La), (qb, Lb) in zip(ref[0], got[0]):
            assert torch.equal(qa, qb) and torch.equal(La, Lb)
        assert np.array_equal(ref[1][0], got[1][0]) and list(ref[1][1]) == list(got[1][1])
    # and the result is the oracle's
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
    assert _qerr(ref[0][-1][0].cpu().numpy().astype(np.float64), qo) <= Q_NU
