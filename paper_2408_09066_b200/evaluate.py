"""Accuracy harness: ROC-AUC of the global entropy map at labelled
validation points ("mapping accuracy is measured as the area under the receiver
operating characteristic curve"), the TPR - FPR threshold (Fig. 7 caption), and
confusion metrics (Table III).  Host-side numpy on the maps the library produced.

Readings: scores are S sampled at the grid cell containing each
validation point (nearest cell centre; cells outside the grid are an error); AUC is the
Mann-Whitney statistic with average ranks for ties; rho maximises TPR - FPR over the distinct
score cut-points, ties to the lowest threshold; zero-denominator metrics are 0.
"""
from __future__ import annotations

import numpy as np
from scipy.stats import rankdata


def roc_auc(scores, labels) -> float:
    s = np.asarray(scores, dtype=np.float64).reshape(-1)
    y = np.asarray(labels).reshape(-1).astype(bool)
    n1, n0 = int(y.sum()), int((~y).sum())
    if n1 == 0 or n0 == 0:
        raise ValueError("roc_auc needs both classes")
    ranks = rankdata(s)                               # average ranks for ties
    return float((ranks[y].sum() - n1 * (n1 + 1) / 2.0) / (n1 * n0))


def select_threshold(scores, labels) -> float:
    """rho maximising TPR - FPR (Youden) over the distinct scores as cut-points (score >= rho
    predicts occupied); ties broken by the lowest threshold."""
    s = np.asarray(scores, dtype=np.float64).reshape(-1)
    y = np.asarray(labels).reshape(-1).astype(bool)
    n1, n0 = int(y.sum()), int((~y).sum())
    if n1 == 0 or n0 == 0:
        raise ValueError("select_threshold needs both classes")
    cuts = np.unique(s)
    order = np.argsort(s, kind="stable")
    ss, yy = s[order], y[order]
    idx = np.searchsorted(ss, cuts, side="left")      # first sorted position with score >= cut
    cum1 = np.concatenate([[0], np.cumsum(yy)])
    cum0 = np.concatenate([[0], np.cumsum(~yy)])
    tp = n1 - cum1[idx]                               # positives with score >= cut
    fp = n0 - cum0[idx]
    j = tp / n1 - fp / n0
    best = np.max(j)
    return float(cuts[np.flatnonzero(j == best)[0]])


def confusion_metrics(scores, labels, rho):
    s = np.asarray(scores, dtype=np.float64).reshape(-1)
    y = np.asarray(labels).reshape(-1).astype(bool)
    pred = s >= rho
    tp = int(np.sum(pred & y))
    fp = int(np.sum(pred & ~y))
    fn = int(np.sum(~pred & y))
    precision = tp / (tp + fp) if tp + fp else 0.0
    recall = tp / (tp + fn) if tp + fn else 0.0
    f1 = 2 * precision * recall / (precision + recall) if precision + recall else 0.0
    return precision, recall, f1


def cell_of(xy, x0, y0, res, rows, cols):
    """(row, col) of the grid cell containing each point (the nearest cell centre)."""
    xy = np.asarray(xy, dtype=np.float64)
    c = np.floor((xy[:, 0] - x0) / res).astype(np.int64)
    r = np.floor((xy[:, 1] - y0) / res).astype(np.int64)
    if np.any((r < 0) | (r >= rows) | (c < 0) | (c >= cols)):
        raise ValueError("a validation point lies outside the grid")
    return r, c


def evaluate(S_map, xy_val, labels_val, x0, y0, res):
    """AUC, rho, precision, recall, f1 of the global entropy map S at the validation points."""
    rows, cols = S_map.shape
    r, c = cell_of(xy_val, x0, y0, res, rows, cols)
    scores = np.asarray(S_map)[r, c]
    auc = roc_auc(scores, labels_val)
    rho = select_threshold(scores, labels_val)
    p, rc, f1 = confusion_metrics(scores, labels_val, rho)
    return {"auc": auc, "rho": rho, "precision": p, "recall": rc, "f1": f1, "n_val": int(len(scores))}
