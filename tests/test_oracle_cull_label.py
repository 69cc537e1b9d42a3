"""Pins for the oracle's culling (O6) and label map (O7, G19).

Culling is pinned by the two properties that characterise the greedy result
uniquely (the lexicographically-first maximal independent set in (E, id)
order), checked with exact rational arithmetic: no two survivors overlap, and
every removed candidate overlaps a survivor of higher priority.  Labels are
pinned by exact rational checks of ball membership and nearest-key winners.
"""
from fractions import Fraction

import numpy as np
import pytest

RHO3 = 0.7937005259840998
RHO2_3D = 0.6299605249474366
COLLAPSED, RMAX = 2, 4


def _overlap_exact(ci, cj, Ri, Rj, rho):
    d2 = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(ci, cj))
    t = Fraction(rho) * Fraction(float(max(Ri, Rj)))
    return d2 < t * t


def _random_set(rng, k):
    c = rng.uniform(0, 40, (k, 3)).astype(np.float32)
    R = rng.uniform(4, 12, k).astype(np.float32)
    E = rng.uniform(-10, 0, k).astype(np.float32)
    flags = np.zeros(k, np.uint32)
    ids = rng.permutation(1000)[:k].astype(np.int64)
    return c, R, E, flags, ids


def test_cull_characterisation(ora):
    rng = np.random.default_rng(6)
    for _ in range(100):
        c, R, E, flags, ids = _random_set(rng, 20)
        flags[rng.integers(0, 20, 2)] = rng.choice([COLLAPSED, RMAX])
        keep = ora.cull(c, R, E, flags, ids, 3, -3.0)
        cand = [i for i in range(20) if E[i] <= -3.0 and not (flags[i] & (COLLAPSED | RMAX))]
        order = sorted(cand, key=lambda i: (E[i], ids[i]))
        assert list(keep) == [i for i in order if i in set(keep)]      # output in (E, id) order
        ks = set(int(i) for i in keep)
        for a in ks:
            for b in ks:
                if a < b:
                    assert not _overlap_exact(c[a], c[b], R[a], R[b], RHO3)
        for i in cand:
            if i in ks:
                continue
            pri = order.index(i)
            assert any(_overlap_exact(c[i], c[a], R[i], R[a], RHO3) and order.index(a) < pri
                       for a in ks)


def test_cull_simple_cases(ora):
    # S:297 two identical snakes -> exactly one survives (the lower id on equal E)
    c = np.array([[10, 10, 10], [10, 10, 10]], np.float32)
    R = np.array([8, 8], np.float32)
    E = np.array([-5, -5], np.float32)
    keep = ora.cull(c, R, E, np.zeros(2, np.uint32), np.array([7, 3]), 3, -3.0)
    assert keep.tolist() == [1]
    # S:298 centres 2R apart -> both survive; S:299 chain -5 < -4 < -3 all mutually overlapping
    c = np.array([[0, 0, 0], [16, 0, 0]], np.float32)
    assert len(ora.cull(c, R, E, np.zeros(2, np.uint32), np.array([0, 1]), 3, -3.0)) == 2
    c = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], np.float32)
    keep = ora.cull(c, np.full(3, 8, np.float32), np.array([-4, -5, -3], np.float32),
                    np.zeros(3, np.uint32), np.arange(3), 3, -3.0)
    assert keep.tolist() == [1]
    # E0 filter ("energy greater than a threshold E0 are removed")
    keep = ora.cull(c[:1], R[:1], np.array([-2.9], np.float32), np.zeros(1, np.uint32),
                    np.arange(1), 3, -3.0)
    assert len(keep) == 0
    # boundary of the overlap test: distance exactly rho * R survives
    R1 = np.array([8, 8], np.float32)
    d = np.float32(RHO3 * 8)
    c = np.array([[0, 0, 0], [d, 0, 0]], np.float32)
    exp = 2 if float(d) ** 2 >= (RHO3 * 8.0) ** 2 else 1
    assert len(ora.cull(c, R1, np.array([-5, -4], np.float32), np.zeros(2, np.uint32),
                        np.arange(2), 3, -3.0)) == exp


def test_label_exact_properties(ora):
    rng = np.random.default_rng(7)
    n = (24, 20, 16)
    k = 12
    c = rng.uniform(0, 20, (k, 3)).astype(np.float32)
    R = rng.uniform(2, 8, k).astype(np.float32)
    lab = ora.label(n, 3, c, R)
    assert lab.shape == (16, 20, 24)
    thr = [Fraction(float(r)) * Fraction(float(r)) * Fraction(RHO2_3D) for r in R]
    for z in range(0, 16, 3):
        for y in range(0, 20, 2):
            for x in range(24):
                keys = []
                for i in range(k):
                    d2 = sum((Fraction(v) - Fraction(float(ci))) ** 2 for v, ci in zip((x, y, z), c[i]))
                    if d2 <= thr[i]:
                        keys.append((d2 / thr[i], i))
                got = int(lab[z, y, x])
                if not keys:
                    assert got == 0
                else:
                    best = min(keys)
                    if got != best[1] + 1:   # only a rounding near-tie may differ
                        other = [kk for kk, i in keys if i == got - 1]
                        assert other and abs(float(other[0] - best[0])) < 1e-12


def test_label_points_and_2d(ora):
    rng = np.random.default_rng(8)
    c = rng.uniform(0, 30, (6, 3)).astype(np.float32)
    c[:, 2] = 0
    R = rng.uniform(3, 9, 6).astype(np.float32)
    lab = ora.label((32, 32, 1), 2, c, R)
    pts = np.array([[x, y, 0] for y in range(32) for x in range(32)])
    assert np.array_equal(ora.label_points(2, pts, c, R), lab.reshape(-1))
    # 2D inner disk radius R / sqrt(2): the centre voxel of an isolated detection
    c1 = np.array([[10, 10, 0]], np.float32)
    lab1 = ora.label((21, 21, 1), 2, c1, np.array([4.0], np.float32))
    assert lab1[0, 10, 10] == 1 and lab1[0, 10, 12] == 1 and lab1[0, 10, 13] == 0  # 2 <= 2.83 < 3


def test_label_equal_keys_go_to_the_smaller_index(ora):
    """O7's tie rule (reading G19): an exact duplicate detection never wins, and a
    voxel on the bisecting plane of two equal balls (equal keys exactly) takes
    the smaller index."""
    n = (24, 20, 18)
    c = np.array([[8.0, 9.0, 9.0], [8.0, 9.0, 9.0], [14.0, 9.0, 9.0]], np.float32)
    R = np.array([6.0, 6.0, 6.0], np.float32)
    lab = ora.label(n, 3, c, R)
    assert not (lab == 2).any()                       # the duplicate of detection 0
    assert (lab == 1).any() and (lab == 3).any()
    # x = 11 is equidistant from x = 8 and x = 14: inside both inner balls -> index 0
    plane = lab[:, :, 11]
    inside = plane > 0
    assert inside.any() and np.all(plane[inside] == 1)
    # swapping the order of the two distinct balls swaps the winner on the plane
    lab2 = ora.label(n, 3, c[[2, 1, 0]], R)
    assert np.all(lab2[:, :, 11][lab2[:, :, 11] > 0] == 1)   # now index 0 is the ball at x = 14
    assert lab2[9, 9, 13] == 1 and lab[9, 9, 13] == 3
