"""Accuracy harness on the GPU: AUC of the GPU map at the circle dataset's
validation points equals the fp64 oracle pipeline's AUC, and improves with D."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def test_auc_matches_oracle_and_grows_with_D():
    from synth.circle import gen_circle_dataset, split_train_val
    from tools.ablation import gpu_auc, oracle_auc
    xy, lab = gen_circle_dataset(0)
    tr, va = split_train_val(len(lab), 0.9, 0)
    aucs = []
    for D in (4, 64, 1024):
        g = gpu_auc(D, xy, lab, tr, va)
        o = oracle_auc(D, xy, lab, tr, va)
        assert abs(g["auc"] - o["auc"]) <= 2e-3, (D, g, o)
        aucs.append(g["auc"])
    assert aucs[0] < aucs[1] < aucs[2]
    assert aucs[2] > 0.9
