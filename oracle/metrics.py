"""oracle.metrics — TEST INFRASTRUCTURE ONLY (detection evaluation utility).

Precision / recall / F-measure as printed in the paper's Results
and SPEC's greedy one-to-one matching.  Used by tests to score
detections against the synthetic ground truth; not part of the hot path
(out of the hot path).
"""
from __future__ import annotations

import numpy as np


def prf(tp: int, fp: int, fn: int):
    """P = TP/(TP+FP), R = TP/(TP+FN), F = 2PR/(P+R); 0 when undefined."""
    p = tp / (tp + fp) if tp + fp else 0.0
    r = tp / (tp + fn) if tp + fn else 0.0
    f = 2 * p * r / (p + r) if p + r else 0.0
    return p, r, f


def f_measure(p: float, r: float) -> float:
    return 2 * p * r / (p + r) if p + r else 0.0


def match_detections(dets: np.ndarray, truth: np.ndarray, tau: float):
    """sort all (det, truth) pairs by distance (ties by (det, truth) index),
    accept a pair if both unmatched and distance <= tau."""
    dets = np.asarray(dets, float).reshape(-1, 3)
    truth = np.asarray(truth, float).reshape(-1, 3)
    pairs = []
    for i, d in enumerate(dets):
        dist = np.linalg.norm(truth - d, axis=1)
        for j in np.nonzero(dist <= tau)[0]:
            pairs.append((dist[j], i, int(j)))
    pairs.sort()
    used_d, used_t, matches = set(), set(), []
    for dist, i, j in pairs:
        if i not in used_d and j not in used_t:
            used_d.add(i)
            used_t.add(j)
            matches.append((i, j, dist))
    tp = len(matches)
    return {"tp": tp, "fp": len(dets) - tp, "fn": len(truth) - tp,
            "prf": prf(tp, len(dets) - tp, len(truth) - tp), "matches": matches}
