"""Pins that tie the fp64 oracle to the paper and to mathematics (-m "not gpu").

Each pin checks the oracle against something other than itself: a published
test vector, hand-derived closed forms (tests/golden), a library routine
(numpy.fft, scipy.ndimage, scipy.stats), a textbook limit (sinc), or a brute
force with a different formulation.  Chosen so that a dropped term, a wrong
sign / index or a transposed operand in oracle.c fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import ndimage, stats

import oracle
from conftest import label_tau


def _grid_cells(rows, cols):
    rr, cc = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    return rr.ravel(), cc.ravel()


# ---------------------------------------------------------------- theta (Eq. 3, L2)

def test_splitmix64_published_vector(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "splitmix64.json")))
    out = oracle.splitmix64_stream(g["seed"], len(g["outputs_hex"]))
    assert [f"{int(v):016x}" for v in out] == g["outputs_hex"]


def test_theta_from_stream_definition():
    # theta = pi (1 - 2 u), u = (z >> 11) 2^-53; x-axis draws first, then y (L2)
    D = 37
    z = oracle.splitmix64_stream(123, 2 * D)
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    tx, ty = oracle.theta(123, D)
    np.testing.assert_array_equal(tx, math.pi * (1 - 2 * u[:D]))
    np.testing.assert_array_equal(ty, math.pi * (1 - 2 * u[D:]))


def test_theta_uniform_and_deterministic():
    tx, ty = oracle.theta(0, 16384)
    tx2, ty2 = oracle.theta(0, 16384)
    np.testing.assert_array_equal(tx, tx2)
    np.testing.assert_array_equal(ty, ty2)
    for t in (tx, ty):
        assert np.all(t > -math.pi) and np.all(t <= math.pi)
        # KS test against U(-pi, pi] ("uniformly distributed")
        assert stats.kstest(t, stats.uniform(loc=-math.pi, scale=2 * math.pi).cdf).pvalue > 1e-3
    assert not np.array_equal(oracle.theta(1, 64)[0], oracle.theta(0, 64)[0])


# ---------------------------------------------------------------- hand-derived golden case

def test_golden_hand_case(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "hand_D2.json")))
    ev = {"0": 0.0, "pi/2": math.pi / 2, "pi": math.pi}
    tx = np.array([ev[s] for s in g["theta_x"]])
    ty = np.array([ev[s] for s in g["theta_y"]])
    xy = np.array(g["points"], dtype=np.float32)
    lab = np.array(g["labels"], dtype=np.uint8)
    m, cnt, bad = oracle.encode(tx, ty, g["l"], xy, lab)
    assert bad == 0 and list(cnt) == [1, 2]
    np.testing.assert_allclose(m.real, g["m_re"], atol=1e-15)
    np.testing.assert_allclose(m.imag, g["m_im"], atol=1e-15)
    np.testing.assert_allclose(oracle.norms(m), g["norms"], rtol=1e-15)
    gr = g["grid"]
    q = oracle.decode_grid(tx, ty, g["l"], m, gr["x0"], gr["y0"], gr["res"], 0, gr["rows"], 0, gr["cols"])
    np.testing.assert_allclose(q[0], g["q_empty"], atol=1e-15)
    np.testing.assert_allclose(q[1], g["q_occupied"], atol=1e-15)
    S, labels = oracle.entropy_grid(q, g["half"], g["half"], 0, 0.09, 0.09)
    np.testing.assert_allclose(S[0], g["S_occ"], atol=1e-15)
    np.testing.assert_allclose(S[1], g["S_emp"], atol=1e-15)
    np.testing.assert_allclose(S[2], g["S"], atol=1e-15)
    assert np.all(labels == 1)
    _, labels = oracle.entropy_grid(q, g["half"], g["half"], 0, 0.1, 0.1)
    assert np.all(labels == 0)


# ---------------------------------------------------------------- encode / decode closed forms

@pytest.fixture(scope="module")
def small_setup():
    D = 256
    tx, ty = oracle.theta(7, D)
    return D, tx, ty


def test_unit_modulus_single_point(small_setup):
    # |F{phi}_k| = 1: one encoded point is a vector of unit phasors
    D, tx, ty = small_setup
    m, cnt, _ = oracle.encode(tx, ty, 0.3, np.array([[3.7, -1.2]], np.float32), np.array([1], np.uint8))
    np.testing.assert_allclose(np.abs(m[1]), 1.0, atol=1e-13)
    assert np.all(m[0] == 0) and list(cnt) == [0, 1]
    np.testing.assert_allclose(oracle.norms(m), [0.0, math.sqrt(D)], rtol=1e-13)


def test_self_similarity_and_empty_class(small_setup):
    # one point at a cell centre: H = D there, q = 1; empty class -> 0 (L8)
    D, tx, ty = small_setup
    x0, y0, res = -2.0, 1.0, 0.1
    r, c = 13, 21
    px, py = x0 + (c + 0.5) * res, y0 + (r + 0.5) * res
    m, _, _ = oracle.encode(tx, ty, 0.25, np.array([[px, py]], np.float32), np.array([1], np.uint8))
    q = oracle.decode_cells(tx, ty, 0.25, m, x0, y0, res, [r], [c])
    # the point is stored as float32: evaluate at its exact float32 coordinates
    fx, fy = float(np.float32(px)), float(np.float32(py))
    assert abs(fx - px) < 1e-6 and abs(fy - py) < 1e-6
    q_exact = oracle.decode_cells(tx, ty, 0.25, m, fx - (c + 0.5) * res, fy - (r + 0.5) * res, res, [r], [c])
    assert abs(q_exact[1, 0] - 1.0) < 1e-12
    assert q[1, 0] > 0.999
    assert q[0, 0] == 0.0


def test_single_point_closed_form_and_shift_invariance(small_setup):
    # H(Delta) = sum_k cos((thx_k dx + thy_k dy)/l): depends only on the offset
    D, tx, ty = small_setup
    l, res = 0.3, 0.05
    pt = np.array([[0.25, 0.75]], np.float32)   # exactly representable
    m, _, _ = oracle.encode(tx, ty, l, pt, np.array([1], np.uint8))
    rows, cols = _grid_cells(9, 11)
    q = oracle.decode_cells(tx, ty, l, m, 0.0, 0.0, res, rows, cols)
    dx = (cols + 0.5) * res - 0.25
    dy = (rows + 0.5) * res - 0.75
    H = np.cos((np.outer(dx, tx) + np.outer(dy, ty)) / l).sum(axis=1)
    np.testing.assert_allclose(q[1] * math.sqrt(D) * math.sqrt(D), H, atol=1e-10)
    # translate point and grid origin by whole cells: identical heatmap
    pt2 = np.array([[0.25 + 8 * 0.125, 0.75 - 4 * 0.125]], np.float32)
    m2, _, _ = oracle.encode(tx, ty, l, pt2, np.array([1], np.uint8))
    q2 = oracle.decode_cells(tx, ty, l, m2, 8 * 0.125, -4 * 0.125, res, rows, cols)
    np.testing.assert_allclose(q2[1], q[1], atol=1e-11)


def test_bundling_linearity(small_setup):
    # Eq. 5 / Alg. 3: m(A u B) = m(A) + m(B); H is linear in m before normalisation
    D, tx, ty = small_setup
    rng = np.random.default_rng(1)
    xy = rng.uniform(0, 5, size=(300, 2)).astype(np.float32)
    lab = rng.integers(0, 2, size=300).astype(np.uint8)
    mA, cA, _ = oracle.encode(tx, ty, 0.3, xy[:120], lab[:120])
    mB, cB, _ = oracle.encode(tx, ty, 0.3, xy[120:], lab[120:])
    mAB, cAB, _ = oracle.encode(tx, ty, 0.3, xy, lab)
    np.testing.assert_allclose(mAB, mA + mB, atol=1e-10)
    assert list(cAB) == list(cA + cB)
    # streaming form: add B on top of A
    mS, cS, _ = oracle.encode(tx, ty, 0.3, xy[120:], lab[120:], m=mA, counts=cA)
    np.testing.assert_allclose(mS, mAB, atol=1e-10)
    rows, cols = _grid_cells(5, 6)

    def H(m):
        return oracle.decode_cells(tx, ty, 0.3, m, 0, 0, 0.7, rows, cols) * (math.sqrt(D) * oracle.norms(m))[:, None]
    np.testing.assert_allclose(H(mAB), H(mA) + H(mB), atol=1e-9)


def test_kernel_sum_bruteforce():
    # H_c(x) = sum_{i: psi_i=c} sum_k cos((thx_k (x-x_i) + thy_k (y-y_i))/l): brute force
    # without the memory vector
    D = 64
    tx, ty = oracle.theta(3, D)
    rng = np.random.default_rng(2)
    xy = rng.uniform(0, 2, size=(9, 2)).astype(np.float32)
    lab = np.array([0, 1, 1, 0, 1, 0, 0, 1, 1], np.uint8)
    l = 0.2
    m, _, _ = oracle.encode(tx, ty, l, xy, lab)
    rows, cols = _grid_cells(6, 7)
    x0, y0, res = 0.1, -0.2, 0.3
    q = oracle.decode_cells(tx, ty, l, m, x0, y0, res, rows, cols)
    n = oracle.norms(m)
    cx = x0 + (cols + 0.5) * res
    cy = y0 + (rows + 0.5) * res
    pts = xy.astype(np.float64)
    for c in (0, 1):
        sel = pts[lab == c]
        Hb = np.zeros(len(rows))
        for (px, py) in sel:
            Hb += np.cos((np.outer(cx - px, tx) + np.outer(cy - py, ty)) / l).sum(axis=1)
        np.testing.assert_allclose(q[c] * math.sqrt(D) * n[c], Hb, atol=1e-10)


def test_parseval_norm():
    # n_c^2 = sum_{i,j} sum_k cos(theta_k . (p_i - p_j) / l)
    D = 128
    tx, ty = oracle.theta(5, D)
    rng = np.random.default_rng(3)
    xy = rng.uniform(-3, 3, size=(11, 2)).astype(np.float32)
    lab = np.ones(11, np.uint8)
    m, _, _ = oracle.encode(tx, ty, 0.5, xy, lab)
    p = xy.astype(np.float64)
    dx = p[:, None, 0] - p[None, :, 0]
    dy = p[:, None, 1] - p[None, :, 1]
    n2 = np.cos((dx[..., None] * tx + dy[..., None] * ty) / 0.5).sum()
    assert abs(oracle.norms(m)[1] ** 2 - n2) < 1e-9 * n2


def test_fft_library_special_case():
    # SPEC's real-vector FHRR is the special case of a
    # conjugate-symmetric theta with D = d: H/d equals the time-domain dot
    # product <sum_i phi_i, phi_loc> with vectors from numpy.fft.ifft (Eq. 3, Eq. 9)
    d = 64
    rng = np.random.default_rng(4)

    def sym(rng):
        th = np.zeros(d)
        free = rng.uniform(-math.pi, math.pi, size=d // 2 - 1)
        th[1:d // 2] = free
        th[d // 2 + 1:] = -free[::-1]
        return th
    tx, ty = sym(rng), sym(rng)
    l = 0.4
    xy = rng.uniform(0, 3, size=(20, 2)).astype(np.float32)
    lab = np.ones(20, np.uint8)
    m, _, _ = oracle.encode(tx, ty, l, xy, lab)

    def phi(x, y):
        v = np.fft.ifft(np.exp(1j * tx * x / l) * np.exp(1j * ty * y / l))
        assert np.max(np.abs(v.imag)) < 1e-12
        return v.real
    mt = sum(phi(float(x), float(y)) for x, y in xy.astype(np.float64))
    rows, cols = _grid_cells(4, 5)
    x0, y0, res = 0.2, 0.1, 0.5
    q = oracle.decode_cells(tx, ty, l, m, x0, y0, res, rows, cols)
    H = q[1] * math.sqrt(d) * oracle.norms(m)[1]
    for e in range(len(rows)):
        dot = float(np.dot(mt, phi(x0 + (cols[e] + 0.5) * res, y0 + (rows[e] + 0.5) * res)))
        assert abs(H[e] / d - dot) < 1e-12


def test_sinc_limit():
    # P:231 / Fig. 1B: the similarity tends to sinc(dx/l) sinc(dy/l) as D grows; |err| <= 5/sqrt(2D)
    D = 16384
    tx, ty = oracle.theta(0, D)
    l = 1.0
    m, _, _ = oracle.encode(tx, ty, l, np.array([[0.0, 0.0]], np.float32), np.array([1], np.uint8))
    offs = [(0.0, 0.0), (0.5, 0.0), (1.0, 0.0), (1.5, 0.0), (3.5, 0.0), (0.5, 0.5), (2.5, 1.5)]
    for (a, b) in offs:
        q = oracle.decode_cells(tx, ty, l, m, a - 0.5, b - 0.5, 1.0, [0], [0])[1, 0]
        ref = np.sinc(a) * np.sinc(b)
        assert abs(q - ref) <= 5 / math.sqrt(2 * D), (a, b, q, ref)
    q35 = oracle.decode_cells(tx, ty, l, m, 3.0, -0.5, 1.0, [0], [0])[1, 0]
    assert abs(q35 - (-0.0909)) < 0.05            # S:60 example


def test_range_on_lidar_data():
    from synth.lidar import Scenario
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    D = 512
    tx, ty = oracle.theta(0, D)
    m, cnt, bad = oracle.encode(tx, ty, 0.2, xy, lab)
    assert bad == 0 and cnt.sum() == len(lab)
    rows, cols = _grid_cells(100, 100)
    q = oracle.decode_cells(tx, ty, 0.2, m, 0, 0, 0.1, rows[::7], cols[::7])   # asserts |q| <= 1
    assert np.all(np.abs(q) <= 1 + 1e-12)


def test_invalid_points_skipped():
    tx, ty = oracle.theta(0, 16)
    xy = np.array([[1, 1], [np.nan, 0], [2, 2], [0, np.inf]], np.float32)
    lab = np.array([1, 1, 2, 0], np.uint8)
    m, cnt, bad = oracle.encode(tx, ty, 0.3, xy, lab)
    assert bad == 3 and list(cnt) == [0, 1]


# ---------------------------------------------------------------- entropy / labels (Alg. 2, Eq. 12)

def test_hb_textbook_values():
    assert oracle.hb(0.0) == 0.0 and oracle.hb(1.0) == 0.0
    assert oracle.hb(0.5) == 1.0
    assert abs(oracle.hb(0.25) - (2 - 0.75 * math.log2(3))) < 1e-15


def test_entropy_constant_grids():
    R, C = 9, 12
    for disk in (0, 1):
        q = np.full((2, R, C), math.sqrt(0.5))
        S, lab = oracle.entropy_grid(q, 2, 3, disk, 0.0, 0.0)
        np.testing.assert_allclose(S[0], 1.0, atol=1e-15)
        np.testing.assert_allclose(S[1], 1.0, atol=1e-15)
        np.testing.assert_allclose(S[2], 0.0, atol=1e-15)
        q = np.random.default_rng(0).integers(0, 2, size=(2, R, C)).astype(np.float64)
        S, _ = oracle.entropy_grid(q, 2, 3, disk, 0.0, 0.0)
        assert np.all(S == 0.0)


def _hb_np(p):
    with np.errstate(divide="ignore", invalid="ignore"):
        a = np.where(p > 0, -p * np.log2(np.where(p > 0, p, 1)), 0.0)
        b = np.where(p < 1, -(1 - p) * np.log2(np.where(p < 1, 1 - p, 1)), 0.0)
    return a + b


@pytest.mark.parametrize("disk", [0, 1])
@pytest.mark.parametrize("h", [1, 2, 3, 4])
def test_entropy_vs_scipy_correlate(disk, h):
    # window mean clipped at the grid border = correlate(hb, mask, 0-pad) / correlate(1, mask, 0-pad)
    rng = np.random.default_rng(10 * h + disk)
    R, C = 16, 19
    q = rng.uniform(-1, 1, size=(2, R, C))
    u = np.arange(-h, h + 1)
    mask = (np.abs(u[:, None]) <= h) & (np.abs(u[None, :]) <= h)
    if disk:
        mask = u[:, None] ** 2 + u[None, :] ** 2 <= h * h
    mask = mask.astype(np.float64)
    h_emp = max(1, h - 1)
    u2 = np.arange(-h_emp, h_emp + 1)
    mask2 = (u2[:, None] ** 2 + u2[None, :] ** 2 <= h_emp ** 2) if disk else np.ones((2 * h_emp + 1,) * 2, bool)
    mask2 = mask2.astype(np.float64)
    S, lab = oracle.entropy_grid(q, h, h_emp, disk, 0.05, -0.05)
    ones = np.ones((R, C))
    s1 = ndimage.correlate(_hb_np(q[1] ** 2), mask, mode="constant") / ndimage.correlate(ones, mask, mode="constant")
    s0 = ndimage.correlate(_hb_np(q[0] ** 2), mask2, mode="constant") / ndimage.correlate(ones, mask2, mode="constant")
    np.testing.assert_allclose(S[0], s1, atol=1e-12)
    np.testing.assert_allclose(S[1], s0, atol=1e-12)
    np.testing.assert_allclose(S[2], s1 - s0, atol=1e-12)
    ref = np.where(s1 - s0 >= 0.05, 1, np.where(s1 - s0 < -0.05, 0, 2))
    assert np.array_equal(lab, ref)


def test_disk_counts(golden_dir):
    # one cell with hb = 1 (p = 1/2) in an otherwise zero grid: S at that cell = 1 / |disk|
    g = json.load(open(os.path.join(golden_dir, "disk_counts.json")))
    for r, cnt in zip(g["r"], g["count"]):
        R = 2 * r + 5
        q = np.zeros((2, R, R))
        q[1, R // 2, R // 2] = math.sqrt(0.5)
        S, _ = oracle.entropy_cells(R, R, 0, R, 0, R, q, r, r, 1, 0, 0, [R // 2], [R // 2])
        assert abs(1.0 / S[0, 0] - cnt) < 1e-9
        Sb, _ = oracle.entropy_cells(R, R, 0, R, 0, R, q, r, r, 0, 0, 0, [R // 2], [R // 2])
        assert abs(1.0 / Sb[0, 0] - (2 * r + 1) ** 2) < 1e-9


def test_global_antisymmetry_and_threshold_rules():
    rng = np.random.default_rng(5)
    q = rng.uniform(-1, 1, size=(2, 10, 13))
    S, _ = oracle.entropy_grid(q, 2, 2, 0, 0, 0)
    Sw, _ = oracle.entropy_grid(q[::-1].copy(), 2, 2, 0, 0, 0)
    np.testing.assert_allclose(Sw[2], -S[2], atol=1e-15)
    _, lab = oracle.entropy_grid(q, 2, 2, 0, -2.0, -2.0)
    assert np.all(lab == 1)            # rho below range: all occupied
    _, lab = oracle.entropy_grid(q, 2, 2, 0, 2.0, 2.0)
    assert np.all(lab == 0)            # rho above range: all empty
    prev = None
    for rho in np.linspace(-0.5, 0.5, 21):
        _, lab = oracle.entropy_grid(q, 2, 2, 0, rho, rho)
        occ = lab == 1
        assert np.all(lab != 2)        # rho_emp = rho_occ reduces to Eq. 12 (binary)
        if prev is not None:
            assert not np.any(occ & ~prev)     # occupied set non-increasing in rho
        prev = occ
    # unknown band between rho_emp and rho_occ
    tau = label_tau(512)
    _, lab = oracle.entropy_grid(q, 2, 2, 0, tau, -tau)
    s = S[2]
    assert np.array_equal(lab == 2, (s < tau) & (s >= -tau))
