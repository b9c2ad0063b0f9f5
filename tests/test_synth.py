"""Host-side checks of the shared seeded input generator (synth/lidar.py)."""
import numpy as np

from synth.lidar import Scenario


def test_c1_counts_and_determinism():
    a = Scenario("C1").all_points()
    b = Scenario("C1").all_points()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    xy, lab = a
    # 360 beams, walls guarantee a hit within 7.07 m < 8 m range, 4 free samples each
    assert len(lab) == 1800 and int(lab.sum()) == 360
    assert xy.dtype == np.float32 and lab.dtype == np.uint8
    assert np.all((xy >= -1e-4) & (xy <= 10 + 1e-4))
    # order per beam: hit then its free samples
    assert np.all(lab.reshape(360, 5)[:, 0] == 1) and np.all(lab.reshape(360, 5)[:, 1:] == 0)


def test_c2_shape():
    xy, lab = Scenario("C2").all_points()
    assert 60_000 < len(lab) <= 20 * 1081 * 3
    assert abs(lab.mean() - 1 / 3) < 0.02


def test_c4_batches_independent_and_deterministic():
    sc = Scenario("C4")
    b1 = sc.batch(1)
    b1b = Scenario("C4").batch(1)
    assert np.array_equal(b1[0], b1b[0])
    assert 150_000 < len(b1[1]) <= 100 * 1081 * 2
    b0 = sc.batch(0)
    assert not np.array_equal(b0[0][:100], b1[0][:100])
