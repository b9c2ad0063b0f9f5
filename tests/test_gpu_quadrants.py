"""GPU parity for quadrant memories (delta > 1; sec. III-B-4, Alg. 1)
against the fp64 oracle (oracle.encode_quadrants / decode_cells_quadrants).  SURVEY.md 8(f) NEXT #1."""
import numpy as np
import pytest
import torch

import oracle
from conftest import label_tau
from synth.lidar import Scenario

pytestmark = pytest.mark.gpu

Q_TOL = 1e-3
M_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _cuda(xy, lab):
    return torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(np.ascontiguousarray(lab)).cuda()


def _run(name, delta, grid=None, D=None, halo=None, band=None):
    from paper_2408_09066_b200 import Mapper
    sc = Scenario(name)
    cfg = sc.cfg
    xy, lab = sc.all_points()
    D = D or cfg["D"]
    l, h = cfg["l"], cfg["half"] if halo is None else halo
    x0, y0, res, R, C = grid or (0.0, 0.0, cfg["res"], cfg["rows"], cfg["cols"])
    r0, r1 = band or (0, R)
    tau = label_tau(D)
    mp = Mapper(D, 0, l, sc.bounds, delta=delta)
    mp.encode_bundle(*_cuda(xy, lab))
    q = torch.empty((2, r1 - r0, C), dtype=torch.float32, device="cuda")
    mp.decode(x0, y0, res, R, C, r0, r1, h, q_out=q)
    L = torch.empty((r1 - r0, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, tau, -tau, 0, None, L)
    assert mp.sync() == 0
    mg, cg = mp.get_memory()
    mp.close()
    return sc, xy, lab, D, l, h, tau, mg, cg, q.cpu().numpy().astype(np.float64), L.cpu().numpy()


@pytest.mark.parametrize("delta", [2, 3, 6])
def test_c1_quadrants_memory_heatmap_labels(delta):
    sc, xy, lab, D, l, h, tau, mg, cg, qg, Lg = _run("C1", delta)
    cfg = sc.cfg
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode_quadrants(tx, ty, l, sc.bounds, delta, xy, lab)
    assert list(cg) == list(co)
    for s in range(2 * delta * delta):
        if co[s]:
            assert np.linalg.norm(mg[s] - mo[s]) <= M_TOL * np.linalg.norm(mo[s])
        else:
            assert np.all(mg[s] == 0)
    qo, _ = oracle.decode_grid_quadrants(tx, ty, l, mo, sc.bounds, delta, 0, 0, cfg["res"], 0, cfg["rows"], 0,
                                        cfg["cols"])
    for c in (0, 1):
        assert np.abs(qg[c] - qo[c]).max() <= Q_TOL * np.abs(qo[c]).max()
    _, Lo = oracle.entropy_grid(qo, h, h, 0, tau, -tau)
    assert (Lg == Lo).mean() >= 0.999


def test_c2_delta2_full_grid():
    sc, xy, lab, D, l, h, tau, mg, cg, qg, Lg = _run("C2", 2)
    cfg = sc.cfg
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode_quadrants(tx, ty, l, sc.bounds, 2, xy, lab)
    assert list(cg) == list(co)
    qo, _ = oracle.decode_grid_quadrants(tx, ty, l, mo, sc.bounds, 2, 0, 0, cfg["res"], 0, cfg["rows"], 0,
                                        cfg["cols"])
    for c in (0, 1):
        assert np.abs(qg[c] - qo[c]).max() <= Q_TOL * np.abs(qo[c]).max()
    _, Lo = oracle.entropy_grid(qo, h, h, 0, tau, -tau)
    assert (Lg == Lo).mean() >= 0.999


def test_misaligned_grid_band_and_halo():
    """Cell boundaries that do not align with quadrant boundaries, an offset grid origin
    that puts cells outside the bounds, and a row band with halo (delta = 3)."""
    grid = (-0.33, 0.21, 0.07, 150, 160)
    full = _run("C1", 3, grid=grid, D=384, halo=2)
    band = _run("C1", 3, grid=grid, D=384, halo=2, band=(40, 95))
    sc, xy, lab, D, l, h, tau = full[:7]
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode_quadrants(tx, ty, l, sc.bounds, 3, xy, lab)
    qo, beta = oracle.decode_grid_quadrants(tx, ty, l, mo, sc.bounds, 3, *grid[:3], 0, grid[3], 0, grid[4])
    assert len(np.unique(beta)) == 9
    qg = full[9]
    for c in (0, 1):
        assert np.abs(qg[c] - qo[c]).max() <= Q_TOL * np.abs(qo[c]).max()
    assert np.array_equal(band[9], qg[:, 40:95])
    assert np.array_equal(band[10], full[10][40:95])


def test_delta1_create_quadrants_equals_create():
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    outs = []
    for delta in (None, 1):
        mp = Mapper(512, 0, 0.2, sc.bounds) if delta is None else Mapper(512, 0, 0.2, sc.bounds, delta=delta)
        mp.encode_bundle(*_cuda(xy, lab))
        q = torch.empty((2, 100, 100), dtype=torch.float32, device="cuda")
        mp.decode(0, 0, 0.1, 100, 100, 0, 100, 1, q_out=q)
        outs.append((mp.get_memory(), q.cpu()))
        mp.close()
    assert np.array_equal(outs[0][0][0], outs[1][0][0])
    assert torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("delta", [1, 2])
def test_encode_paths_agree(monkeypatch, delta):
    """The three encode paths (0: counting sort by slot + equal runs, the default for delta > 1;
    1: label-split blocks for delta = 1 / slot-filtered for delta > 1; 2: slot-filtered blocks)
    give the same memories up to fp32 rounding, and the same counts.  The pair (half-angle)
    kernels pair consecutive points of a slot within their tile or run, so different paths
    pair some points differently and round those terms differently: each path is within
    ~1.5e-5 of the fp64 oracle, two paths within 5e-5 of each other."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    mems = []
    for knob in ("0", "1", "2"):
        mp = Mapper(2048, 0, 0.25, sc.bounds, delta=delta)
        mp.set_tuning("enc_path", int(knob))
        mp.encode_bundle(*_cuda(xy, lab))
        mems.append(mp.get_memory())
        mp.close()
    for other in mems[1:]:
        assert list(mems[0][1]) == list(other[1])
        for s in range(2 * delta * delta):
            if mems[0][1][s]:
                assert np.linalg.norm(mems[0][0][s] - other[0][s]) <= 5e-5 * np.linalg.norm(mems[0][0][s])


@pytest.mark.parametrize("delta", [1, 2])
def test_encode_packed_variants_agree(monkeypatch, delta):
    """The packed fp32x2 encode kernels (enc_x2 = 1: uniform 4-warp blocks; 2: all-MUFU warps
    beside 4-polynomial warps; 3: 1- beside 5-polynomial warps; 4: the pair (half-angle)
    kernels, the default) agree with the scalar kernel (0) up to fp32 rounding: the
    polynomial phasors (sincos_fma2_lite, max error 1e-6), the pairing and the chunking
    differ (each within ~1.5e-5 of the oracle), the counts are exact."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    mems = []
    for knob in ("0", "1", "2", "3", "4"):
        mp = Mapper(4096, 3, 0.25, sc.bounds, delta=delta)
        mp.set_tuning("enc_x2", int(knob))
        mp.encode_bundle(*_cuda(xy, lab))
        mems.append(mp.get_memory())
        mp.close()
    for other in mems[1:]:
        assert list(mems[0][1]) == list(other[1])
        for s in range(2 * delta * delta):
            if mems[0][1][s]:
                assert np.linalg.norm(mems[0][0][s] - other[0][s]) <= 5e-5 * np.linalg.norm(mems[0][0][s])
