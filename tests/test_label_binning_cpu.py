"""The binned evaluation of the oracle's O7 rule used by the full-size GPU
label checks (tests/test_gpu_parity_scale.py) equals the oracle's own label
map over all detections (2D and 3D, overlapping balls, ties by index)."""
import numpy as np

import oracle
from test_gpu_parity_scale import oracle_labels_binned


def test_binned_labels_equal_oracle_map():
    rng = np.random.default_rng(5)
    for dim, n, k in [(3, (150, 140, 70), 400), (2, (300, 260, 1), 300)]:
        c = (rng.uniform(0, 1, (k, 3)) * np.array(n)).astype(np.float32)
        if dim == 2:
            c[:, 2] = 0
        R = rng.uniform(3, 14, k).astype(np.float32)
        c[1] = c[0]
        R[1] = R[0]   # an exact tie: the smaller index wins
        full = oracle.label(n, dim, c, R)
        if dim == 3:
            z, y, x = np.meshgrid(np.arange(n[2]), np.arange(n[1]), np.arange(n[0]), indexing="ij")
        else:
            z = np.zeros((1, n[1], n[0]), np.int64)
            y, x = np.meshgrid(np.arange(n[1]), np.arange(n[0]), indexing="ij")
            y, x = y[None], x[None]
        pts = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
        got = oracle_labels_binned(dim, pts, c, R, bin_=32)
        assert np.array_equal(got, full.ravel())
        assert (full > 0).mean() > 0.05
