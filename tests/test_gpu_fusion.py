"""Multi-agent fusion (Alg. 3): export / import /
fuse of memory states, preconditions, and additivity against the fp64 oracle.  SURVEY.md 8(f) NEXT #3."""
import struct

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


def _cuda(xy, lab):
    return torch.from_numpy(np.ascontiguousarray(xy)).cuda(), torch.from_numpy(np.ascontiguousarray(lab)).cuda()


def _parse(blob):
    assert blob[:8] == b"VSAOGM1\x00"
    end = blob.index(b"\n\n", 8)
    hdr = dict(line.split("=", 1) for line in blob[8:end].decode().split("\n"))
    S, D = int(hdr["slots"]), int(hdr["D"])
    off = end + 2
    counts = np.frombuffer(blob, dtype="<i8", count=S, offset=off)
    mem = np.frombuffer(blob, dtype="<f8", count=2 * S * D, offset=off + 8 * S).reshape(S, D, 2)
    return hdr, counts, mem[..., 0] + 1j * mem[..., 1]


@pytest.mark.parametrize("delta", [1, 2])
def test_two_agents_fuse_equals_union(delta):
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C2")
    xy, lab = sc.all_points()
    D, l = 2048, 0.25
    half = len(lab) // 2
    a = Mapper(D, 0, l, sc.bounds, delta=delta)
    b = Mapper(D, 0, l, sc.bounds, delta=delta)
    a.encode_bundle(*_cuda(xy[:half], lab[:half]))
    b.encode_bundle(*_cuda(xy[half:], lab[half:]))
    blob_b = b.export()
    hdr, cnt_b, mem_b = _parse(blob_b)
    mg, cg = b.get_memory()
    assert int(hdr["D"]) == D and int(hdr["delta"]) == delta and int(hdr["seed"]) == 0
    assert np.array_equal(cnt_b, cg) and np.array_equal(mem_b, mg)
    a.fuse(blob_b)                         # Alg. 3: same-index memories bundled
    mf, cf = a.get_memory()
    tx, ty = oracle.theta(0, D)
    mo, co, _ = oracle.encode_quadrants(tx, ty, l, sc.bounds, delta, xy, lab)
    assert list(cf) == list(co)
    for s in range(2 * delta * delta):
        if co[s]:
            assert np.linalg.norm(mf[s] - mo[s]) <= 1e-4 * np.linalg.norm(mo[s])
    # decode of the fused map equals the decode of a single agent trained on the union
    u = Mapper(D, 0, l, sc.bounds, delta=delta)
    u.encode_bundle(*_cuda(xy, lab))
    qs = []
    for mp in (a, u):
        q = torch.empty((2, 400, 400), dtype=torch.float32, device="cuda")
        mp.decode(0, 0, 0.1, 400, 400, 0, 400, 2, q_out=q)
        qs.append(q)
    assert (qs[0] - qs[1]).abs().max().item() <= 1e-5
    for mp in (a, b, u):
        mp.close()


def test_load_restores_state_and_fuse_is_additive():
    from paper_2408_09066_b200 import Mapper
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    a = Mapper(512, 7, 0.2, sc.bounds)
    a.encode_bundle(*_cuda(xy, lab))
    blob = a.export()
    c = Mapper(512, 7, 0.2, sc.bounds)
    c.load(blob)
    ma, ca = a.get_memory()
    mc, cc = c.get_memory()
    assert list(ca) == list(cc)
    np.testing.assert_allclose(mc, ma, rtol=0, atol=1e-10 * np.abs(ma).max())
    c.fuse(blob)                           # adding the same state twice doubles it
    m2, c2 = c.get_memory()
    assert list(c2) == [2 * v for v in ca]
    np.testing.assert_allclose(m2, 2 * ma, rtol=0, atol=1e-9 * np.abs(ma).max())
    a.close()
    c.close()


def test_fusion_preconditions():
    from paper_2408_09066_b200 import Mapper
    from paper_2408_09066_b200.vsaogm import EINVAL_ARG, EPRECOND, VsaogmError
    sc = Scenario("C1")
    xy, lab = sc.all_points()
    base = Mapper(256, 1, 0.2, sc.bounds)
    base.encode_bundle(*_cuda(xy, lab))
    blob = base.export()
    others = [Mapper(256, 2, 0.2, sc.bounds),                      # different axis vectors (seed)
              Mapper(256, 1, 0.3, sc.bounds),                      # different length scale
              Mapper(256, 1, 0.2, sc.bounds, delta=2),             # different delta
              Mapper(256, 1, 0.2, (0, 0, 10, 11)),                 # different bounds
              Mapper(128, 1, 0.2, sc.bounds)]                      # different D
    for o in others:
        with pytest.raises(VsaogmError) as e:
            o.fuse(blob)
        assert e.value.code == EPRECOND
        assert np.all(o.get_memory()[0] == 0)                     # nothing changed
        o.close()
    with pytest.raises(VsaogmError) as e:
        base.fuse(b"NOTVSAOGM" + blob[9:])
    assert e.value.code == EINVAL_ARG
    with pytest.raises(VsaogmError) as e:
        base.fuse(blob[:len(blob) // 2])                           # truncated
    assert e.value.code == EINVAL_ARG
    base.close()
