"""Pins for the oracle's histogram ("rank") local-entropy estimator (
PAPER.md:311, :318, Alg. 2 :330-356): Shannon entropy in bits of the 8-bit
grey-level histogram of p inside the clipped footprint."""
import math

import numpy as np
import pytest
from scipy import stats

import oracle


def _codes(p):
    return np.clip(np.floor(p.astype(np.float32) * np.float32(255) + np.float32(0.5)), 0, 255).astype(int)


def test_constant_and_distinct_windows():
    R = C = 9
    p = np.full((2, R, C), 0.3)
    S, _ = oracle.entropy_hist_grid(p, 2, 2, 0, 0, 0)
    assert np.all(S == 0)                                      # one grey level -> 0 bits
    # all 25 cells of a 5x5 window distinct -> log2(25) at an interior cell
    p = np.zeros((2, R, C))
    p[0] = (np.arange(R * C).reshape(R, C) % 200) / 255.0
    p[1] = p[0]
    S, _ = oracle.entropy_hist_cells(R, C, 0, R, 0, C, p, 2, 2, 0, 0, 0, [4], [4])
    assert abs(S[0, 0] - math.log2(25)) < 1e-12 and abs(S[2, 0]) < 1e-15
    # two grey levels half / half in a 1x2 clipped footprint -> 1 bit
    p = np.zeros((2, 1, 2))
    p[1, 0, 1] = 1.0
    S, _ = oracle.entropy_hist_cells(1, 2, 0, 1, 0, 2, p, 1, 1, 0, 0, 0, [0], [0])
    assert abs(S[0, 0] - 1.0) < 1e-15 and S[1, 0] == 0.0


@pytest.mark.parametrize("disk", [0, 1])
@pytest.mark.parametrize("h", [1, 2, 3])
def test_vs_scipy_entropy_of_bincount(disk, h):
    rng = np.random.default_rng(h + 7 * disk)
    R, C = 12, 14
    # few grey levels so that histograms have repeats
    p = rng.integers(0, 6, size=(2, R, C)) / 255.0 * 40
    S, lab = oracle.entropy_hist_grid(p, h, h, disk, 0.01, -0.01)
    codes = _codes(p)
    u = np.arange(-h, h + 1)
    mask = (u[:, None] ** 2 + u[None, :] ** 2 <= h * h) if disk else np.ones((2 * h + 1,) * 2, bool)
    for cls, si in ((1, 0), (0, 1)):
        for r in range(R):
            for c in range(C):
                vals = [codes[cls, r + a, c + b] for a in u for b in u
                        if mask[a + h, b + h] and 0 <= r + a < R and 0 <= c + b < C]
                ref = stats.entropy(np.bincount(vals), base=2)
                assert abs(S[si, r, c] - ref) < 1e-12
    g = S[0] - S[1]
    assert np.array_equal(lab, np.where(g >= 0.01, 1, np.where(g < -0.01, 0, 2)))


def test_quantisation_rule():
    # floor(255 p + 1/2) in fp32, clipped: p = 1 -> 255, p = 0 -> 0, p = 0.5/255 -> 1 (half up)
    assert list(_codes(np.array([0.0, 1.0, 0.5 / 255, 1.49 / 255]))) == [0, 255, 1, 1]
