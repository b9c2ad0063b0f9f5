"""Pins for the oracle's quadrant memories (delta > 1; sec. III-B-4, Alg. 1
P:260-285; SPEC memory module S:192-274).  SURVEY.md 8(f) NEXT #1."""
import math

import numpy as np
import pytest

import oracle


def test_centers_spec_examples():
    cx, cy = oracle.quadrant_centers((0, 0, 10, 10), 1)
    assert list(zip(cx, cy)) == [(5.0, 5.0)]
    cx, cy = oracle.quadrant_centers((0, 0, 10, 10), 2)
    assert list(zip(cx, cy)) == [(2.5, 2.5), (7.5, 2.5), (2.5, 7.5), (7.5, 7.5)]
    cx, cy = oracle.quadrant_centers((0, 0, 8, 8), 6)            # 36 centres spaced 8/6
    assert len(cx) == 36
    np.testing.assert_allclose(np.diff(np.unique(cx)), 8 / 6, rtol=1e-12)
    np.testing.assert_allclose(np.diff(np.unique(cy)), 8 / 6, rtol=1e-12)


def test_assignment_examples_and_property():
    b = (0, 0, 10, 10)
    beta = oracle.assign_quadrants(b, 2, [1.0, 5.0, 9.0, 1.0, -5.0, 100.0, 7.5],
                                   [1.0, 5.0, 1.0, 9.0, -5.0, 1.0, 7.5])
    # S:222 (1,1) -> 0; S:223 (5,5) equidistant to all four -> 0 (tie to lowest); out-of-bounds
    # points go to the nearest centre
    assert list(beta) == [0, 0, 1, 2, 0, 1, 3]
    rng = np.random.default_rng(0)
    for delta in (2, 3, 6):
        x = rng.uniform(-2, 12, 2000)
        y = rng.uniform(-2, 12, 2000)
        # include exact quadrant boundaries (ties)
        x[:40] = np.round(x[:40] * delta / 10) * 10 / delta
        beta = oracle.assign_quadrants(b, delta, x, y)
        cx, cy = oracle.quadrant_centers(b, delta)
        d = (x[:, None] - cx[None, :]) ** 2 + (y[:, None] - cy[None, :]) ** 2
        dmin = d.min(axis=1)
        assert np.all(d[np.arange(len(x)), beta] == dmin)                 # nearest
        first = np.argmax(d == dmin[:, None], axis=1)
        assert np.array_equal(beta, first)                                # lowest index among ties


@pytest.fixture(scope="module")
def setup():
    from synth.lidar import Scenario
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    D = 256
    tx, ty = oracle.theta(11, D)
    return sc.bounds, xy, lab, tx, ty


def test_delta1_equals_plain_encode(setup):
    b, xy, lab, tx, ty = setup
    m1, c1, _ = oracle.encode(tx, ty, 0.2, xy, lab)
    mq, cq, _ = oracle.encode_quadrants(tx, ty, 0.2, b, 1, xy, lab)
    np.testing.assert_allclose(mq, m1, atol=1e-10)
    assert list(cq) == list(c1)


@pytest.mark.parametrize("delta", [2, 3, 6])
def test_partition_invariant(setup, delta):
    # every point lands in exactly one slot 2 beta + psi: the quadrant memories of a
    # class sum to the delta = 1 memory of that class (Eq. 5 additivity), counts likewise
    b, xy, lab, tx, ty = setup
    m1, c1, _ = oracle.encode(tx, ty, 0.2, xy, lab)
    mq, cq, _ = oracle.encode_quadrants(tx, ty, 0.2, b, delta, xy, lab)
    assert mq.shape == (2 * delta * delta, 256)
    for c in (0, 1):
        np.testing.assert_allclose(mq[c::2].sum(axis=0), m1[c], atol=1e-9)
        assert cq[c::2].sum() == c1[c]
    beta = oracle.assign_quadrants(b, delta, xy[:, 0].astype(np.float64), xy[:, 1].astype(np.float64))
    for s in range(2 * delta * delta):
        assert cq[s] == np.sum((2 * beta + lab) == s)


def test_single_point_in_quadrant(setup):
    # one occupied point in quadrant 0 of a fresh bank -> slot 1 = its location vector, others 0
    b, _, _, tx, ty = setup
    m, cnt, _ = oracle.encode_quadrants(tx, ty, 0.2, b, 2, np.array([[1.0, 1.0]], np.float32),
                                        np.array([1], np.uint8))
    assert list(cnt) == [0, 1] + [0] * 6
    np.testing.assert_allclose(np.abs(m[1]), 1.0, atol=1e-13)
    assert np.all(m[[0, 2, 3, 4, 5, 6, 7]] == 0)


@pytest.mark.parametrize("delta", [2, 3])
def test_decode_uses_the_cells_own_quadrant(setup, delta):
    # a cell in quadrant beta decodes exactly like the (pinned) delta = 1 decode of memories 2 beta, 2 beta + 1
    b, xy, lab, tx, ty = setup
    mq, _, _ = oracle.encode_quadrants(tx, ty, 0.2, b, delta, xy, lab)
    rng = np.random.default_rng(delta)
    rows = rng.integers(0, 100, 300)
    cols = rng.integers(0, 100, 300)
    q, beta = oracle.decode_cells_quadrants(tx, ty, 0.2, mq, b, delta, 0.0, 0.0, 0.1, rows, cols)
    cxs = (cols + 0.5) * 0.1
    cys = (rows + 0.5) * 0.1
    assert np.array_equal(beta, oracle.assign_quadrants(b, delta, cxs, cys))
    for bq in np.unique(beta):
        sel = beta == bq
        qq = oracle.decode_cells(tx, ty, 0.2, mq[2 * bq:2 * bq + 2], 0.0, 0.0, 0.1, rows[sel], cols[sel])
        np.testing.assert_allclose(q[:, sel], qq, atol=1e-12)
