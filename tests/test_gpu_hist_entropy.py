"""GPU parity of the histogram (8-bit grey-level) local-entropy estimator."""
import numpy as np
import pytest
import torch

import oracle
from synth.lidar import Scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _p32(q):
    q = q.astype(np.float32)
    return np.minimum(q * q, np.float32(1)).astype(np.float64)


@pytest.mark.parametrize("disk", [0, 1])
@pytest.mark.parametrize("h1,h0", [(2, 2), (3, 1), (1, 4)])
def test_hist_entropy_vs_oracle_on_gpu_q(disk, h1, h0):
    """Stencil isolated: the oracle estimator on the GPU's own p (same fp32 p, same fp32 codes)."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    R, C = 100, 100
    mp = Mapper(512, 0, 0.2, sc.bounds)
    mp.set_estimator(1)
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    q = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, 0.1, R, C, 0, R, 4, q_out=q)
    S = torch.empty((3, R, C), dtype=torch.float32, device="cuda")
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h1, h0, 0.05, -0.05, disk, S, L)
    assert mp.sync() == 0
    So, Lo = oracle.entropy_hist_grid(_p32(q.cpu().numpy()), h1, h0, disk, 0.05, -0.05)
    assert np.abs(S.cpu().numpy() - So).max() <= 2e-5
    assert (L.cpu().numpy() == Lo).mean() >= 0.9999
    mp.close()


def _codes32(q):
    """The kernel's decision in the kernel's precision: p = min(q^2, 1)
    and code = floor(255 p + 1/2), each operation rounded to fp32."""
    p = _p32(q).astype(np.float32)
    return np.floor(np.float32(255) * p + np.float32(0.5)).astype(np.int32)


def test_hist_entropy_end_to_end_c2_and_band():
    """End to end against the oracle's own q on C2.  The estimator quantises p to 8-bit codes, an
    integer decision taken in fp32 on both sides; where the GPU's q (fp16 operands, |dq| ~ 1e-5)
    and the oracle's (fp64) straddle a code boundary the code differs, and so may the window's
    entropy.  So: on every cell whose whole footprint has identical codes on both sides, the
    labels agree (>= 99.99 %: only S ties at a threshold can differ); the fraction of windows that
    contain a flipped code is small (measured ~1e-3; bound 1 %); overall agreement >= 99 %.
    A row band equals the full grid."""
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    cfg = sc.cfg
    D, l, R, C, res, h = cfg["D"], cfg["l"], cfg["rows"], cfg["cols"], cfg["res"], cfg["half"]
    mp = Mapper(D, 0, l, sc.bounds)
    mp.set_estimator(1)
    mp.encode_bundle(torch.from_numpy(xy).cuda(), torch.from_numpy(lab).cuda())
    qg = torch.empty((2, R, C), dtype=torch.float32, device="cuda")
    mp.decode(0, 0, res, R, C, 0, R, h, q_out=qg)
    L = torch.empty((R, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, 0.1, -0.1, 0, None, L)
    mp.decode(0, 0, res, R, C, 100, 250, h)
    Lb = torch.empty((150, C), dtype=torch.uint8, device="cuda")
    mp.entropy(h, h, 0.1, -0.1, 0, None, Lb)
    assert mp.sync() == 0
    assert torch.equal(Lb, L[100:250])
    tx, ty = oracle.theta(0, D)
    mo, _, _ = oracle.encode(tx, ty, l, xy, lab)
    qo = oracle.decode_grid(tx, ty, l, mo, 0, 0, res, 0, R, 0, C)
    _, Lo = oracle.entropy_hist_grid(_p32(qo), h, h, 0, 0.1, -0.1)
    Lg = L.cpu().numpy()
    flip = (_codes32(qg.cpu().numpy()) != _codes32(qo)).any(axis=0).astype(np.int32)
    # windows (2h+1)^2, clipped, that contain a flipped code in either class
    from scipy.ndimage import maximum_filter
    win_flip = maximum_filter(flip, size=2 * h + 1, mode="constant", cval=0) > 0
    same = ~win_flip
    print(f"hist end to end: cells with a code flip {flip.mean():.2e}, windows touched {win_flip.mean():.2e}, "
          f"agreement on untouched windows {(Lg[same] == Lo[same]).mean():.6f}, overall {(Lg == Lo).mean():.5f}")
    assert win_flip.mean() <= 0.01
    assert (Lg[same] == Lo[same]).mean() >= 0.9999
    assert (Lg == Lo).mean() >= 0.99
    # switching estimators requires a new decode
    from paper_2408_09066_b200.vsaogm import ESTATE, VsaogmError
    mp.set_estimator(0)
    with pytest.raises(VsaogmError) as e:
        mp.entropy(h, h, 0.1, -0.1)
    assert e.value.code == ESTATE
    mp.close()
