"""Pins for the oracle's integer volume passes and seed lists.

Blur taps are pinned by the table SURVEY A13 computed independently; the
passes by scipy.ndimage.correlate1d (an independent convolution routine) and by
invariants (constants and linear ramps pass through unchanged); resampling by
S:365's example and exactness on ramps; lattice seeds by the C1 example and the
spacing rule; maxima seeds by scipy.ndimage.maximum_filter on a lexicographic
(value, -index) key (an independent formulation of the definition).
"""
import math

import numpy as np
import pytest
from scipy import ndimage

from conftest import golden_rows, golden_value

# ---------------------------------------------------------------- Q14 taps (A13)


def test_q14_taps_tables(ora):
    for row in golden_rows("q14_taps.txt"):     # tests/golden/q14_taps.txt (A13)
        assert ora.q14_taps(float(row[0])).tolist() == [int(x) for x in row[1:]]
    t2 = ora.q14_taps(2.0)
    assert len(t2) == 17 and t2[8] == 3270 and t2.sum() == 16384
    assert ora.q14_taps(0.0).tolist() == [16384]
    for s in (0.7, 1.3, 2.5, 3.0):
        t = ora.q14_taps(s)
        assert t.sum() == 16384 and len(t) == 2 * math.ceil(4 * s) + 1
        assert np.array_equal(t, t[::-1])


# ---------------------------------------------------------------- blur (O2)


def _scipy_blur(vol, dim, sigma, taps):
    cur = vol.astype(np.int64)
    axes = [2, 1, 0] if dim == 3 else [2, 1]   # x, y, z  (array axes z, y, x)
    for ax in axes:
        acc = ndimage.correlate1d(cur, taps.astype(np.int64), axis=ax, mode="nearest")
        cur = (acc + 8192) >> 14
    return cur.astype(np.uint16)


@pytest.mark.parametrize("dim,shape,sigma", [(3, (9, 13, 17), 1.0), (3, (5, 6, 31), 2.0),
                                             (2, (1, 40, 33), 1.0), (3, (20, 3, 4), 0.5)])
def test_blur_matches_scipy(ora, dim, shape, sigma):
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 65536, size=shape, dtype=np.uint16)
    got = ora.blur(vol, dim, sigma)
    assert np.array_equal(got, _scipy_blur(vol, dim, sigma, ora.q14_taps(sigma)))


def test_blur_invariants(ora):
    vol = np.full((10, 11, 12), 40000, np.uint16)
    assert np.array_equal(ora.blur(vol, 3, 1.0), vol)          # sum w = 16384
    z, y, x = np.meshgrid(np.arange(20), np.arange(20), np.arange(20), indexing="ij")
    ramp = (1000 + 50 * x + 70 * y + 90 * z).astype(np.uint16)
    out = ora.blur(ramp, 3, 1.0)
    assert np.array_equal(out[4:-4, 4:-4, 4:-4], ramp[4:-4, 4:-4, 4:-4])   # symmetric taps
    assert np.array_equal(ora.blur(ramp, 3, 0.0), ramp)        # sigma = 0 identity
    imp = np.zeros((9, 9, 9), np.uint16)
    imp[4, 4, 4] = 16384
    out = ora.blur(imp, 3, 1.0)
    # centre = product of per-axis centre taps (with per-pass Q14 rounding)
    c1 = 6536
    c2 = (c1 * 6536 + 8192) >> 14
    c3 = (c2 * 6536 + 8192) >> 14
    assert out[4, 4, 4] == c3


# ---------------------------------------------------------------- gradmag (O3)


def test_gradmag_brute(ora):
    rng = np.random.default_rng(4)
    for dim, shape in [(3, (6, 7, 8)), (2, (1, 9, 10))]:
        B = rng.integers(0, 65536, size=shape, dtype=np.uint16)
        got = ora.gradmag(B, dim)
        P = np.pad(B.astype(np.int64), 1, mode="edge")
        gx = P[1:-1, 1:-1, 2:] - P[1:-1, 1:-1, :-2]
        gy = P[1:-1, 2:, 1:-1] - P[1:-1, :-2, 1:-1]
        gz = (P[2:, 1:-1, 1:-1] - P[:-2, 1:-1, 1:-1]) if dim == 3 else 0 * gx
        s = gx * gx + gy * gy + gz * gz
        exp = np.vectorize(lambda v: (math.isqrt(int(v)) + 1) >> 1)(s)
        assert np.array_equal(got, exp.astype(np.uint16))
    # extreme: maximal step in all three axes still fits u16
    B = np.zeros((3, 3, 3), np.uint16)
    B[2:, 2:, 2:] = 65535
    assert ora.gradmag(B, 3).max() == (math.isqrt(3 * 65535 ** 2) + 1) >> 1


# ---------------------------------------------------------------- resample (O1)


def test_resample_dims_and_identity(ora):
    assert ora.resample_dims((4, 4, 4), (0.5, 0.5, 1.0)).tolist() == [4, 4, 8]
    assert ora.resample_dims((512, 512, 128), (1, 1, 2)).tolist() == [512, 512, 256]
    vol = np.arange(60, dtype=np.uint16).reshape(3, 4, 5)
    assert np.array_equal(ora.resample(vol, (1, 1, 1)), vol)


def test_resample_ramp_and_weights(ora):
    """Linear interpolation is exact on linear functions; C3 weights are
    {12288, 4096} (ratio 1/2)."""
    z = np.arange(16)
    vol = np.broadcast_to((1000 + 1600 * z)[:, None, None], (16, 3, 4)).astype(np.uint16).copy()
    out = ora.resample(vol, (1.0, 1.0, 2.0))
    assert out.shape == (32, 3, 4)
    k = np.arange(32)
    src = np.clip((k + 0.5) * 0.5 - 0.5, 0, 15)
    assert np.array_equal(out[:, 0, 0], np.floor(1000 + 1600 * src + 0.5).astype(np.uint16))
    assert np.all(out == out[:, :1, :1])
    const = np.full((6, 5, 4), 777, np.uint16)
    assert np.all(ora.resample(const, (1.0, 1.0, 2.0)) == 777)
    assert np.all(ora.resample(const, (3.0, 1.5, 1.0)) == 777)


# ---------------------------------------------------------------- lattice seeds (O4)


def test_lattice_c1_example(ora):
    st, s = ora.seeds_lattice((64, 64, 64), 3, 10.0, 2.0)
    assert st == 0 and len(s) == 64
    first = golden_value("lattice_c1_first_centre")
    assert s[0].tolist() == pytest.approx([first] * 3, abs=1e-4)
    # nearest-neighbour spacing sqrt(1.5) R0; footprints inside
    sp = math.sqrt(1.5) * 10
    assert s[1, 0] - s[0, 0] == pytest.approx(sp, abs=1e-5)
    assert s[4, 1] - s[0, 1] == pytest.approx(sp, abs=1e-5)
    assert s[16, 2] - s[0, 2] == pytest.approx(sp, abs=1e-5)
    assert s.min() >= 11.0 and s.max() <= 63 - 11.0
    # centred: symmetric margins
    assert s[:, 0].min() - 11 == pytest.approx(63 - 11 - s[:, 0].max(), abs=1e-4)


def test_lattice_counts_and_empty(ora):
    # extent 100, R0 = 15 -> centres in [16, 83] spaced 18.37 apart -> 4 per axis
    st, s = ora.seeds_lattice((100, 100, 100), 3, 15.0, 2.0)
    assert st == 0 and len(s) == 64
    st, s = ora.seeds_lattice((2048, 2048, 1), 2, 25.0, 2.0)
    assert st == 0 and np.all(s[:, 2] == 0) and len(s) == 66 * 66
    st, s = ora.seeds_lattice((20, 64, 64), 3, 10.0, 2.0)     # domain smaller than a footprint
    assert st == 1 and len(s) == 0


# ---------------------------------------------------------------- maxima seeds (O4)


def _maxima_scipy(B, dim, w, thr):
    nz, ny, nx = B.shape
    lin = np.arange(B.size, dtype=np.int64).reshape(B.shape)
    # lexicographic (B, -lin) packed so that it stays exact in float64 (scipy filters in double)
    key = B.astype(np.int64) * B.size + (B.size - 1 - lin)
    assert key.max() < 2 ** 52
    size = (2 * w + 1, 2 * w + 1, 2 * w + 1) if dim == 3 else (1, 2 * w + 1, 2 * w + 1)
    mx = ndimage.maximum_filter(key, size=size, mode="constant", cval=-1)
    sel = (key == mx) & (B >= thr)
    zz, yy, xx = np.nonzero(sel)
    return np.stack([xx, yy, zz], axis=1).astype(np.float32)   # nonzero is in C (linear) order


@pytest.mark.parametrize("dim,shape,w,levels", [(3, (12, 13, 14), 2, 6), (3, (9, 9, 9), 3, 65536),
                                                (2, (1, 30, 31), 3, 4), (3, (7, 20, 6), 1, 3)])
def test_maxima_matches_lexicographic_maximum_filter(ora, dim, shape, w, levels):
    rng = np.random.default_rng(5)
    B = (rng.integers(0, levels, size=shape) * (65535 // max(levels - 1, 1))).astype(np.uint16)
    thr = int(np.median(B))
    got = ora.seeds_maxima(B, dim, w, thr)
    exp = _maxima_scipy(B, dim, w, thr)
    assert np.array_equal(got, exp)
    for x, y, z in got.astype(int):
        assert ora.is_maxima_seed(B, dim, w, thr, x, y, z)


def test_maxima_plateau_single_seed(ora):
    B = np.zeros((8, 8, 8), np.uint16)
    B[2:6, 2:6, 2:6] = 30000        # flat plateau: lowest linear index wins
    s = ora.seeds_maxima(B, 3, 4, 20000)
    assert s.tolist() == [[2.0, 2.0, 2.0]]


def test_maxima_on_crop_equals_full(ora):
    """A crop with a w-margin gives the full volume's seeds in its interior (§8(e))."""
    rng = np.random.default_rng(11)
    B = (rng.integers(0, 8, size=(20, 22, 24)) * 9000).astype(np.uint16)
    w, thr = 2, 20000
    full = ora.seeds_maxima(B, 3, w, thr)
    org = np.array([3, 4, 5])
    crop = B[5:17, 4:20, 3:21]                     # (z, y, x) = org + [0, nb)
    n = (24, 22, 20)
    lo, hi = org + w, org + np.array([18, 16, 12]) - 1 - w
    got = ora.seeds_maxima(crop, 3, w, thr, org=org, n_global=n, lo=lo, hi=hi)
    sel = np.all((full >= lo) & (full <= hi), axis=1)
    assert np.array_equal(got, full[sel])


def test_ingest_u8_pins(ora):
    """O0 against facts independent of its formula: the byte-doubling identity
    257 v = (v << 8) | v for every 8-bit value, the end points 0 -> 0 and
    255 -> 65535 (the full u16 range), exact division back to the 8-bit value
    (reading G6: intensity_scale 1/257), order preserved."""
    v = np.arange(256, dtype=np.uint8)
    out = ora.ingest_u8(v)
    assert out.dtype == np.uint16
    assert np.array_equal(out, (v.astype(np.uint16) << 8) | v.astype(np.uint16))
    assert out[0] == 0 and out[255] == 65535
    assert np.array_equal(out.astype(np.int64) % 257, np.zeros(256)) and np.array_equal(out // 257, v)
    assert np.all(np.diff(out.astype(np.int64)) == 257)


def test_resample_half_ratio_rounds_half_up(ora):
    """O1 on C3's ratio 1/2 against the exact weights: output plane 2m + 1 samples
    src = m + 1/4 and 2m samples m - 1/4 (S:365 centre-aligned), so the values are
    (3 v[m] + v[m+1]) / 4 and (v[m-1] + 3 v[m]) / 4 rounded half up —
    (x + 2) >> 2 on the integer x — with the end planes clamped.
    Random values (odd differences) make truncation or round-half-even fail."""
    rng = np.random.default_rng(5)
    v = rng.integers(0, 65536, size=(9, 3, 4)).astype(np.int64)
    out = ora.resample(v.astype(np.uint16), (1.0, 1.0, 2.0)).astype(np.int64)
    assert out.shape == (18, 3, 4)
    exp = np.empty_like(out)
    n = v.shape[0]
    for k in range(18):
        m = k // 2
        if k == 0:
            exp[k] = v[0]
        elif k == 17:
            exp[k] = v[n - 1]
        elif k % 2:
            exp[k] = (3 * v[m] + v[m + 1] + 2) >> 2
        else:
            exp[k] = (v[m - 1] + 3 * v[m] + 2) >> 2
    assert np.array_equal(out, exp)
