"""Pins of the oracle's d-linear lookup (reading G17:
trilinear interpolation S:179, clamp-to-edge S:395), through oracle.interp —
independent of the evolution that uses it.

* Multilinear functions (a x + b y + c z + d, and x y z) are reproduced exactly
  by d-linear interpolation at any interior point: a dropped term, a swapped
  axis, a wrong fraction or a nearest-neighbour lookup all fail.
* scipy.ndimage.map_coordinates(order=1, mode='nearest') is the textbook
  trilinear interpolation with edge replication: element-wise equal, including
  points past the edges and exactly on the last voxel (the i0 = min(floor(k),
  n - 2) rule).
"""
import numpy as np
import pytest
from scipy import ndimage

import oracle


def _affine(shape, coef):
    z, y, x = np.indices(shape, dtype=np.int64)
    a, b, c, d = coef
    return (a * x + b * y + c * z + d).astype(np.uint16)


@pytest.mark.parametrize("shape,coef", [((7, 9, 11), (3, 17, 101, 40)), ((5, 13, 6), (250, 1, 7, 9)),
                                        ((12, 4, 9), (0, 0, 1000, 5))])
def test_interp_exact_on_affine_volumes(shape, coef):
    vol = _affine(shape, coef)
    rng = np.random.default_rng(sum(shape))
    n = np.array([shape[2], shape[1], shape[0]], np.float64)
    pts = rng.uniform(0.0, 1.0, size=(4000, 3)) * (n - 1)
    got, halo = oracle.interp(vol, pts)
    a, b, c, d = coef
    exp = a * pts[:, 0] + b * pts[:, 1] + c * pts[:, 2] + d
    assert not halo.any()
    np.testing.assert_allclose(got, exp, rtol=1e-13, atol=1e-9)
    # iscale multiplies the interpolated value (G6)
    g2, _ = oracle.interp(vol, pts[:50], iscale=1.0 / 257.0)
    np.testing.assert_allclose(g2, exp[:50] / 257.0, rtol=1e-13, atol=1e-11)


def test_interp_exact_on_trilinear_product():
    shape = (9, 8, 10)
    z, y, x = np.indices(shape)
    vol = (x * y * z + 3 * x * y + 2 * y * z + x + 7).astype(np.uint16)
    rng = np.random.default_rng(4)
    n = np.array([shape[2], shape[1], shape[0]], np.float64)
    p = rng.uniform(0.0, 1.0, size=(3000, 3)) * (n - 1)
    got, _ = oracle.interp(vol, p)
    X, Y, Z = p[:, 0], p[:, 1], p[:, 2]
    np.testing.assert_allclose(got, X * Y * Z + 3 * X * Y + 2 * Y * Z + X + 7, rtol=1e-13, atol=1e-9)


@pytest.mark.parametrize("shape", [(6, 7, 8), (2, 2, 2), (3, 17, 5)])
def test_interp_equals_scipy_map_coordinates(shape):
    rng = np.random.default_rng(len(shape) + shape[0])
    vol = rng.integers(0, 65536, size=shape, dtype=np.uint16)
    n = np.array([shape[2], shape[1], shape[0]], np.float64)
    pts = rng.uniform(-3.0, 1.0, size=(5000, 3)) * (n + 5) + np.array([0.0, 0.0, 0.0])
    pts = np.concatenate([pts, rng.uniform(0, 1, size=(2000, 3)) * (n - 1)])
    # exactly on voxel centres, on the last voxel (i0 = n - 2, f = 1) and past it
    last = np.array([[n[0] - 1, n[1] - 1, n[2] - 1], [n[0] - 1, 0, 0], [0, n[1] - 1, n[2] - 1],
                     [n[0] - 1 + 1e-9, n[1] - 1, 0.5], [n[0] + 2.5, -0.75, n[2] - 1]])
    pts = np.concatenate([pts, last, np.floor(pts[:300])])
    got, halo = oracle.interp(vol, pts)
    exp = ndimage.map_coordinates(vol.astype(np.float64), [pts[:, 2], pts[:, 1], pts[:, 0]], order=1,
                                  mode="nearest", prefilter=False)
    assert not halo.any()
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-9)
    # the last voxel exactly
    v_last, _ = oracle.interp(vol, last[:1])
    assert v_last[0] == float(vol[-1, -1, -1])


def test_interp_2d_bilinear_and_anisotropic():
    rng = np.random.default_rng(9)
    img = rng.integers(0, 65536, size=(1, 23, 31), dtype=np.uint16)
    pts = np.stack([rng.uniform(-2, 33, 3000), rng.uniform(-2, 25, 3000), np.zeros(3000)], axis=1)
    got, _ = oracle.interp(img, pts, dim=2)
    exp = ndimage.map_coordinates(img[0].astype(np.float64), [pts[:, 1], pts[:, 0]], order=1, mode="nearest")
    np.testing.assert_allclose(got, exp, rtol=0, atol=1e-9)
    # physical coordinates on a (1, 1, 2) grid (G28): the raw grid is read at k / scale
    vol = rng.integers(0, 65536, size=(8, 9, 10), dtype=np.uint16)
    k = rng.uniform(0, 1, size=(2000, 3)) * np.array([9.0, 8.0, 14.0])
    g2, _ = oracle.interp(vol, k, scale=(1.0, 1.0, 2.0))
    e2 = ndimage.map_coordinates(vol.astype(np.float64), [k[:, 2] / 2.0, k[:, 1], k[:, 0]], order=1,
                                 mode="nearest")
    np.testing.assert_allclose(g2, e2, rtol=0, atol=1e-9)


def test_interp_crop_matches_full_volume_and_flags_halo():
    rng = np.random.default_rng(2)
    vol = rng.integers(0, 65536, size=(20, 18, 16), dtype=np.uint16)
    org = np.array([3, 4, 5])
    crop = vol[5:15, 4:14, 3:13]
    pts = rng.uniform(0, 1, size=(1000, 3)) * 8.5 + org + 0.2   # inside the crop's interior
    full, h0 = oracle.interp(vol, pts)
    part, h1 = oracle.interp(crop, pts, org=org, n_global=(16, 18, 20))
    assert not h0.any() and not h1.any()
    assert np.array_equal(full, part)
    _, h2 = oracle.interp(crop, [[1.0, 1.0, 1.0]], org=org, n_global=(16, 18, 20))
    assert h2.all()
