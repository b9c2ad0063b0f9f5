"""Host-side pins of the accuracy harness."""
import math

import numpy as np
from sklearn.metrics import roc_auc_score

from paper_2408_09066_b200.evaluate import confusion_metrics, roc_auc, select_threshold
from synth.circle import gen_circle_dataset, split_train_val


def test_auc_closed_forms_and_library():
    assert roc_auc([0.9, 0.8, 0.2, 0.1], [1, 1, 0, 0]) == 1.0
    assert roc_auc([0.1, 0.2, 0.8, 0.9], [1, 1, 0, 0]) == 0.0
    rng = np.random.default_rng(0)
    s = np.round(rng.normal(size=300), 1)            # ties on purpose
    y = rng.integers(0, 2, 300)
    pos, neg = s[y == 1], s[y == 0]
    brute = (np.sum(pos[:, None] > neg[None, :]) + 0.5 * np.sum(pos[:, None] == neg[None, :])) / (len(pos) * len(neg))
    assert abs(roc_auc(s, y) - brute) < 1e-12
    assert abs(roc_auc(s, y) - roc_auc_score(y, s)) < 1e-12
    assert abs(roc_auc(s ** 3 + 2 * s, y) - roc_auc(s, y)) < 1e-12      # invariant under increasing maps
    s2 = rng.normal(size=300)
    assert abs(roc_auc(s2, y) + roc_auc(-s2, y) - 1.0) < 1e-12


def test_youden_threshold_and_confusion():
    # perfect separation -> lowest threshold achieving TPR - FPR = 1 is 0.8
    assert select_threshold([0.9, 0.8, 0.2, 0.1], [1, 1, 0, 0]) == 0.8
    rng = np.random.default_rng(1)
    s = rng.normal(size=200)
    y = (s + rng.normal(size=200) > 0).astype(int)
    rho = select_threshold(s, y)
    best = max((np.mean(s[y == 1] >= c) - np.mean(s[y == 0] >= c), -c) for c in np.unique(s))
    assert abs(rho - (-best[1])) < 1e-15                 # O(n^2) exhaustive scan
    assert confusion_metrics([0.9, 0.8, 0.2, 0.1], [1, 1, 0, 0], 0.5) == (1.0, 1.0, 1.0)
    assert confusion_metrics([0.9, 0.8], [1, 0], 2.0) == (0.0, 0.0, 0.0)


def test_circle_dataset_and_split():
    xy, lab = gen_circle_dataset(0)
    assert len(lab) == 10000 and lab.sum() == 5000
    d = np.hypot(xy[:, 0].astype(np.float64) - 4, xy[:, 1].astype(np.float64) - 4)
    assert np.all(np.abs(d[lab == 1] - 4) < 1e-5)        # float32 storage of points on r = 4
    assert np.all(d[lab == 0] < 4 + 1e-5)
    assert abs(d[lab == 0].mean() - 8 / 3) < 0.05        # uniform disk: E[r] = 2R/3
    tr, va = split_train_val(10000, 0.9, 0)
    assert len(tr) == 9000 and len(va) == 1000 and len(np.intersect1d(tr, va)) == 0
    tr2, va2 = split_train_val(10000, 0.9, 0)
    assert np.array_equal(tr, tr2) and np.array_equal(va, va2)
    assert 0 < lab[va].sum() < len(va)
