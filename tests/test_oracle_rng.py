"""Pins for the oracle's sampler (readings G10-G12).

Philox4x32-10 is pinned to the Random123 known-answer vectors; the ball/disk
laws are pinned by the volume/area-uniformity facts SPEC S:219, S:228, S:233
state (they fail for a wrong radial exponent, a wrong direction law or a
dropped factor of 2 in phi)."""
import numpy as np
import pytest
from scipy import stats


from conftest import golden_rows

# Random123 philox4x32_10 KAT vectors (tests/golden/philox4x32_10_kat.txt, with its citation)
KAT = [([int(x, 16) for x in r[0:4]], [int(x, 16) for x in r[5:7]], [int(x, 16) for x in r[8:12]])
       for r in golden_rows("philox4x32_10_kat.txt")]
assert len(KAT) == 3


@pytest.mark.parametrize("ctr,key,expect", KAT)
def test_philox_kat(ora, ctr, key, expect):
    assert [int(x) for x in ora.philox4x32_10(ctr, key)] == expect


def _draw(ora, dim, n, rho_s=1.0, cell_id=7, it=3, seed=1804063040):
    pts = np.empty((n, 3))
    ts = np.empty(n)
    for j in range(n):
        om, t = ora.sample(dim, j, it, cell_id, seed, rho_s)
        pts[j] = om * t
        ts[j] = t
    return pts, ts


def test_sample_is_keyed_and_deterministic(ora):
    a = ora.sample(3, 5, 9, 123, 42, 2.0)
    b = ora.sample(3, 5, 9, 123, 42, 2.0)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    # every key component changes the draw (cell, iteration, sample, seed)
    for args in [(3, 6, 9, 123, 42), (3, 5, 10, 123, 42), (3, 5, 9, 124, 42), (3, 5, 9, 123, 43),
                 (3, 5, 9, 123 + (1 << 32), 42)]:
        c = ora.sample(*args, 2.0)
        assert c[1] != a[1]


def test_ball_uniformity(ora):
    """fraction with |x| <= rho_s / cbrt(2) is 0.5 +- 0.005 (10^5 draws)."""
    pts, ts = _draw(ora, 3, 100_000, rho_s=3.0)
    r = np.linalg.norm(pts, axis=1)
    assert np.all(r <= 3.0 + 1e-12)
    assert np.allclose(r, ts)   # omega is a unit vector
    frac = np.mean(r <= 3.0 / 2 ** (1 / 3))
    assert abs(frac - 0.5) < 0.005
    # chi-square over 8 equal-volume radial shells
    edges = 3.0 * (np.arange(9) / 8) ** (1 / 3)
    counts, _ = np.histogram(r, edges)
    assert stats.chisquare(counts).pvalue > 0.01
    # mean -> 0 within 3 standard errors; isotropy: E[x_a^2] = rho_s^2 / 5
    se = pts.std(axis=0) / np.sqrt(len(pts))
    assert np.all(np.abs(pts.mean(axis=0)) < 3 * se)
    m2 = (pts ** 2).mean(axis=0)
    assert np.allclose(m2, 9.0 / 5.0, rtol=0.02)


def test_disk_uniformity(ora):
    """2D fraction with |x| <= rho_s / sqrt(2) is 0.5 +- 0.005."""
    pts, ts = _draw(ora, 2, 100_000, rho_s=2.0)
    assert np.all(pts[:, 2] == 0.0)
    r = np.linalg.norm(pts, axis=1)
    assert abs(np.mean(r <= 2.0 / np.sqrt(2.0)) - 0.5) < 0.005
    edges = 2.0 * np.sqrt(np.arange(9) / 8)
    counts, _ = np.histogram(r, edges)
    assert stats.chisquare(counts).pvalue > 0.01
    # angle uniform on [0, 2 pi)
    ang = np.arctan2(pts[:, 1], pts[:, 0])
    counts, _ = np.histogram(ang, np.linspace(-np.pi, np.pi, 17))
    assert stats.chisquare(counts).pvalue > 0.01


def test_direction_hatbox(ora):
    """G10: Archimedes - z = omega_z uniform on [-1, 1], azimuth uniform."""
    om = np.array([ora.sample(3, j, 1, 0, 5, 1.0)[0] for j in range(50_000)])
    assert np.allclose(np.linalg.norm(om, axis=1), 1.0, atol=1e-12)
    counts, _ = np.histogram(om[:, 2], np.linspace(-1, 1, 17))
    assert stats.chisquare(counts).pvalue > 0.01
    az = np.arctan2(om[:, 1], om[:, 0])
    counts, _ = np.histogram(az, np.linspace(-np.pi, np.pi, 17))
    assert stats.chisquare(counts).pvalue > 0.01


@pytest.mark.parametrize("dim", [3, 2])
def test_word_stream_layout(ora, dim):
    """G11: the samples of one cell-iteration consume the Philox word stream in
    order, each word once (3D: 3 words per sample, 4 samples per 3 blocks; 2D: 2
    words per sample).  The uniforms are recovered from the sample itself."""
    it, cid, seed, rho_s = 11, (5 << 32) + 9, 1804063040, 2.5
    key = [seed & 0xFFFFFFFF, seed >> 32]
    words = []
    for b in range(8):
        words += [int(x) for x in ora.philox4x32_10([b, it, cid & 0xFFFFFFFF, cid >> 32], key)]
    u = [(w >> 9) * 2.0 ** -23 for w in words]
    k = 3 if dim == 3 else 2
    for j in range(10):
        om, t = ora.sample(dim, j, it, cid, seed, rho_s)
        got_u1 = (np.arctan2(om[1], om[0]) / (2 * np.pi)) % 1.0
        if dim == 3:
            assert abs((1.0 - om[2]) / 2.0 - u[3 * j]) < 1e-12
            assert abs((t / rho_s) ** 3 - u[3 * j + 2]) < 1e-12
            exp_u1 = u[3 * j + 1]
        else:
            assert abs((t / rho_s) ** 2 - u[2 * j + 1]) < 1e-12
            exp_u1 = u[2 * j]
        d = abs(got_u1 - exp_u1)
        assert min(d, 1.0 - d) < 1e-12, (j, got_u1, exp_u1)
    assert k * 10 <= len(words)
