"""Pins for the oracle's contour evolution (O5; Eqs. 11-14) and the
end-to-end pipeline.

The equilibrium radii are pinned by 1D quadrature of the closed-form
Gaussian-blurred ball / disk profiles (computed here with scipy, independent of
the oracle's volume code); the ellipsoid radius by a brute-force argmin of the
supersampled energy; the touching-sphere case, stationarity on a uniform image
 and SPEC's offset-phantom example by their stated outcomes.
"""
import math

import numpy as np
import pytest
from scipy import integrate, optimize, special

import synth
from conftest import golden_value


def blurred_ball(r, r0, sigma, A):
    """Closed form of a ball of radius r0 (value A) convolved with a 3D Gaussian."""
    s2 = math.sqrt(2) * sigma
    a = 0.5 * A * (special.erf((r0 - r) / s2) + special.erf((r0 + r) / s2))
    b = A * sigma / (r * math.sqrt(2 * math.pi)) * (np.exp(-(r - r0) ** 2 / (2 * sigma ** 2))
                                                    - np.exp(-(r + r0) ** 2 / (2 * sigma ** 2)))
    return a - b


def blurred_disk(r, r0, sigma, A):
    """A disk of radius r0 convolved with a 2D Gaussian (radial integral, i0e-stable)."""
    f = lambda p: p / sigma ** 2 * np.exp(-(r - p) ** 2 / (2 * sigma ** 2)) * special.i0e(r * p / sigma ** 2)
    return A * integrate.quad(f, 0.0, r0, limit=200)[0]


def radial_argmin(ora, prof, dim, dR=2.0, lo=None, hi=None):
    area = 4 * math.pi if dim == 3 else 2 * math.pi

    def e(R):
        rho = 2 ** (-1 / dim)
        pts = [rho * (R - dR / 2), rho * (R + dR / 2), R - dR / 2]
        val = integrate.quad(lambda r: ora.weight(r, R, dR, dim)[0] * prof(r) * r ** (dim - 1),
                             1e-9, R + dR / 2, points=pts, limit=200)[0]
        return area * val * (2 * R) ** (-dim)

    return optimize.minimize_scalar(e, bounds=(lo, hi), method="bounded",
                                    options={"xatol": 1e-5}).x


def _ball_volume(n, c, r0, amp=100.0, dim=3, ora=None, sigma=1.0):
    shape = (n, n, n) if dim == 3 else (n, n, 1)
    v = synth.sphere_volume(shape, c, r0, amp=amp, scale=257.0, supersample=6)
    return ora.blur(v, dim, sigma)


@pytest.mark.parametrize("mode", [0, 2, 3])
def test_equilibrium_radius_3d(ora, mode):
    """r0 = 10, dR = 2, sigma = 1: R* = 12.8493, then the oracle's
    evolution of centred snakes converges to within 0.1 of it — plain MC (0),
    with the control variate (2) and with the stratified ray march (3)."""
    rstar = radial_argmin(ora, lambda r: blurred_ball(r, 10.0, 1.0, 100.0), 3, lo=11, hi=14)
    assert rstar == pytest.approx(golden_value("equilibrium_radius_3d"), abs=2e-3)
    vol = _ball_volume(48, (24.0, 24.0, 24.0), 10.0, ora=ora)
    p = ora.Params(r0=10.0, n_samples=1024, dim=3, mode=mode)
    seeds = np.array([[25.0, 23.0, 24.5]] * 8, np.float32)
    cells = ora.evolve(vol, p, seeds, ids=np.arange(8) * 1000 + 17)
    assert abs(cells["R"].mean() - rstar) < 0.1
    assert np.all(np.abs(cells["c"] - 24.0).max(axis=1) < 0.2)
    assert np.all(cells["E"] < -3)


def test_equilibrium_radius_2d(ora):
    """2D mode: blurred disk r0 = 15, A = 100, sigma = 1: R* = 21.3630
    (hard-edge theory sqrt(2) r0 = 21.2132)."""
    rstar = radial_argmin(ora, lambda r: blurred_disk(r, 15.0, 1.0, 100.0), 2, lo=19, hi=23)
    assert rstar == pytest.approx(golden_value("equilibrium_radius_2d"), abs=2e-3)
    v = synth.sphere_volume((72, 72, 1), (36.0, 36.0, 0.0), 15.0, amp=100.0, supersample=6)
    vol = ora.blur(v, 2, 1.0)
    p = ora.Params(r0=25.0, n_samples=1024, dim=2)
    seeds = np.array([[34.0, 37.5, 0.0]] * 8, np.float32)
    cells = ora.evolve(vol, p, seeds, ids=np.arange(8) + 5)
    assert abs(cells["R"].mean() - rstar) < 0.1
    assert np.all(np.abs(cells["c"][:, :2] - 36.0).max(axis=1) < 0.15)
    assert np.all(cells["c"][:, 2] == 0.0)


def test_offset_phantom_spec_example(ora):
    """snake 3 voxels off a phantom sphere (r0 = 10, R0 = 15): final centre
    within 1 voxel, final R within 10% of cbrt(2) r0."""
    vol = _ball_volume(56, (28.0, 28.0, 28.0), 10.0, ora=ora)
    p = ora.Params(r0=15.0, n_samples=1024, dim=3)
    cells = ora.evolve(vol, p, np.array([[31.0, 28.0, 28.0]], np.float32), ids=np.array([3]))
    assert np.max(np.abs(cells["c"][0] - 28.0)) < 1.0
    assert abs(cells["R"][0] - 10 * 2 ** (1 / 3)) < 0.1 * 10 * 2 ** (1 / 3)


def test_first_step_size(ora):
    """G7: eps0 = 0.5 gives a ~0.47 voxel first step of the state (c, R) on SPEC's
    canonical offset-3 phantom (r0 = 10, R0 = 15), toward the blob."""
    vol = _ball_volume(56, (28.0, 28.0, 28.0), 10.0, ora=ora)
    p = ora.Params(r0=15.0, n_samples=4096, dim=3, max_iters=1)
    cells = ora.evolve(vol, p, np.array([[31.0, 28.0, 28.0]] * 4, np.float32), ids=np.arange(4))
    dc = cells["c"] - np.array([31.0, 28.0, 28.0])
    dR = cells["R"] - 15.0
    step = np.sqrt((dc ** 2).sum(axis=1) + dR ** 2).mean()
    assert 0.3 < step < 0.7
    assert np.all(dc[:, 0] < 0) and np.all(dR < 0)    # toward the blob, shrinking


def test_ellipsoid_radius_matches_energy_argmin(ora):
    """north_star: an ellipsoid converges to its known radius — the argmin over R
    of the supersampled energy at the true centre (brute force)."""
    n = 44
    z, y, x = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    inside = ((x - 22) / 10.5) ** 2 + ((y - 22) / 9.0) ** 2 + ((z - 22) / 8.0) ** 2 < 1
    vol = ora.blur((inside * 100 * 257).astype(np.uint16), 3, 1.0)
    p = ora.Params(r0=11.0, n_samples=1024, dim=3)
    Rs = np.arange(10.5, 14.01, 0.25)
    es = [ora.energy_ss(vol, p, (22.0, 22.0, 22.0), R, q=3) for R in Rs]
    i = int(np.argmin(es))
    a, b, c = np.polyfit(Rs[i - 2:i + 3], es[i - 2:i + 3], 2)
    r_best = -b / (2 * a)
    cells = ora.evolve(vol, p, np.array([[22.5, 21.5, 22.0]] * 6, np.float32), ids=np.arange(6))
    assert abs(cells["R"].mean() - r_best) < 0.15
    assert np.all(np.abs(cells["c"] - 22.0).max(axis=1) < 0.3)


def test_two_touching_spheres(ora):
    """Image-mediated 'repulsion': r0 = 9, centres 18 apart.
    Each snake settles outward of its own nucleus, mirror-symmetrically, and both
    survive the overlap competition."""
    n = (60, 40, 40)
    v1 = synth.sphere_volume(n, (21.0, 20.0, 20.0), 9.0, amp=100.0, supersample=4)
    v2 = synth.sphere_volume(n, (39.0, 20.0, 20.0), 9.0, amp=100.0, supersample=4)
    vol = ora.blur(np.maximum(v1, v2), 3, 1.0)
    p = ora.Params(r0=11.0, n_samples=1024, dim=3)
    k = 8
    seeds = np.array([[21.0, 20.0, 20.0]] * k + [[39.0, 20.0, 20.0]] * k, np.float32)
    cells = ora.evolve(vol, p, seeds, ids=np.arange(2 * k))
    left = cells["c"][:k, 0].mean() - 21.0
    right = cells["c"][k:, 0].mean() - 39.0
    assert left < -0.05 and right > 0.05           # outward
    assert abs(left + right) < 0.1                  # mirror symmetric
    assert abs(left) < 0.4 and abs(right) < 0.4
    pair = cells[[0, k]]
    keep = ora.cull(pair["c"].astype(np.float32), pair["R"].astype(np.float32),
                    pair["E"].astype(np.float32), pair["flags"], pair["id"], 3, -3.0)
    assert len(keep) == 2


def test_uniform_image_grid_mode_stationary(ora):
    """P:93 / S:279 / AC4: on a constant image the grid-mode snake moves < 0.1 voxel
    in 400 iterations (reading G21: asserted in grid mode only)."""
    vol = np.full((40, 40, 40), 60 * 257, np.uint16)
    p = ora.Params(r0=10.0, dim=3, mode=1)
    cells = ora.evolve(vol, p, np.array([[20.3, 19.7, 20.1]], np.float32))
    assert np.max(np.abs(cells["c"][0] - [20.3, 19.7, 20.1])) < 0.1


def test_safeguards(ora):
    vol = _ball_volume(48, (24.0, 24.0, 24.0), 10.0, ora=ora)
    # leash (G8): |c - seed| <= leash per component
    p = ora.Params(r0=10.0, n_samples=256, dim=3, leash=0.5, max_iters=60)
    c = ora.evolve(vol, p, np.array([[28.0, 24.0, 24.0]], np.float32))
    assert abs(c["c"][0][0] - 28.0) <= 0.5 + 1e-12 and c["flags"][0] & ora.LEASHED
    # max_step bounds the total displacement
    p = ora.Params(r0=10.0, n_samples=256, dim=3, max_step=1e-3, max_iters=10)
    c = ora.evolve(vol, p, np.array([[28.0, 24.0, 24.0]], np.float32))
    assert np.max(np.abs(c["c"][0] - [28, 24, 24])) <= 1e-2 + 1e-12
    assert abs(c["R"][0] - 10.0) <= 1e-2 + 1e-12
    # domain clamp keeps the footprint inside
    p = ora.Params(r0=10.0, n_samples=256, dim=3, max_iters=5)
    c = ora.evolve(vol, p, np.array([[2.0, 24.0, 24.0]], np.float32))
    assert c["c"][0][0] >= c["R"][0] + 1.0 - 1e-9
    # dark image: the contour collapses to r_min and is flagged (never a detection)
    dark = np.zeros((48, 48, 48), np.uint16)
    p = ora.Params(r0=10.0, n_samples=64, dim=3, max_iters=40, eps0=0.5)
    c = ora.evolve(dark, p, np.array([[24.0, 24.0, 24.0]], np.float32))
    assert c["E"][0] == 0.0


def test_determinism_across_thread_counts(ora):
    vol = _ball_volume(40, (20.0, 20.0, 20.0), 8.0, ora=ora)
    p = ora.Params(r0=9.0, n_samples=128, dim=3, max_iters=50)
    seeds = np.random.default_rng(9).uniform(15, 25, (12, 3)).astype(np.float32)
    nt = ora.num_threads()
    try:
        ora.set_num_threads(1)
        a = ora.evolve(vol, p, seeds)
        ora.set_num_threads(max(nt, 4))
        b = ora.evolve(vol, p, seeds)
    finally:
        ora.set_num_threads(nt)
    assert a.tobytes() == b.tobytes()


def test_c1_end_to_end(ora):
    """SURVEY A9 / SPEC AC6 on C1: 64 lattice snakes -> one detection per nucleus."""
    cfg = synth.CONFIGS["C1"]
    raw = synth.generate(cfg)
    p = ora.Params(r0=cfg.r0, n_samples=cfg.n_samples, dim=3, seed=cfg.philox_seed)
    res = ora.run_pipeline(raw, p, seed_mode="lattice")
    truth = synth.nuclei(cfg)
    assert len(res.seeds) == 64
    det = res.cells[res.keep]
    assert len(det) == len(truth) == 8
    d = np.linalg.norm(det["c"][:, None, :] - truth["c"][None, :, :], axis=2)
    assert sorted(np.argmin(d, axis=1).tolist()) == list(range(8))   # one per nucleus
    assert d.min(axis=1).max() < 2.0
    # label map: every detection's centre voxel carries its label
    for i, cc in enumerate(det["c"]):
        x, y, z = np.round(cc).astype(int)
        assert res.labels[z, y, x] == i + 1


def test_crop_and_slab_equal_full_volume(ora):
    """T4 on the CPU: evolving on a crop / z-slab holding every voxel a cell can
    reach (leash + r_max + dR/2 + 1) gives bit-identical cells (§8(e))."""
    vol = _ball_volume(48, (24.0, 22.0, 25.0), 8.0, ora=ora)
    p = ora.Params(r0=9.0, n_samples=128, dim=3, max_iters=60, leash=3.0, r_max=11.0)
    seeds = np.array([[23.5, 22.5, 24.0], [26.0, 20.0, 25.5]], np.float32)
    full = ora.evolve(vol, p, seeds, ids=np.array([5, 9]))
    reach = int(np.ceil(3.0 + 11.0 + 1.0 + 1.0))
    lo = np.floor(seeds.min(0)).astype(int) - reach
    hi = np.ceil(seeds.max(0)).astype(int) + reach
    lo, hi = np.maximum(lo, 0), np.minimum(hi, 47)
    crop = vol[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
    got = ora.evolve(crop, p, seeds, ids=np.array([5, 9]), org=lo, n_global=(48, 48, 48))
    assert got.tobytes() == full.tobytes()
    slab = vol[lo[2]:hi[2] + 1]
    got = ora.evolve(slab, p, seeds, ids=np.array([5, 9]), z_lo=int(lo[2]), n_global=(48, 48, 48))
    assert got.tobytes() == full.tobytes()
    assert not np.any(full["flags"] & ora.HALO)
    # a crop that is too small is detected (HALO flag), never silently wrong
    small = ora.evolve(vol[20:30], p, seeds, ids=np.array([5, 9]), z_lo=20, n_global=(48, 48, 48))
    assert np.all(small["flags"] & ora.HALO)


# ---------------------------------------------------------------- periodic culling


def test_segments_resume_exactly(ora):
    """Evolution in segments [1,a], [a+1,b], ..., [., T+1] from the records is the
    same computation as one run (the record is the whole state)."""
    vol = _ball_volume(40, (20.0, 20.0, 20.0), 8.0, ora=ora)
    p = ora.Params(r0=9.0, n_samples=128, dim=3, max_iters=50)
    seeds = np.random.default_rng(3).uniform(15, 25, (6, 3)).astype(np.float32)
    one = ora.evolve(vol, p, seeds, ids=np.arange(10, 16))
    assert ora.checkpoints(50, 20) == [(1, 20), (21, 40), (41, 51)]
    assert ora.checkpoints(50, 0) == [(1, 51)] and ora.checkpoints(50, 50) == [(1, 51)]
    cells = ora.init_cells(p, seeds, ids=np.arange(10, 16))
    for a, b in [(1, 7), (8, 8), (9, 33), (34, 51)]:
        cells = ora.evolve_range(vol, p, cells, a, b)
    assert cells.tobytes() == one.tobytes()
    # grid mode too
    pg = ora.Params(r0=9.0, dim=3, max_iters=20, mode=1)
    one = ora.evolve(vol, pg, seeds[:2])
    cells = ora.evolve_range(vol, pg, ora.evolve_range(vol, pg, ora.init_cells(pg, seeds[:2]), 1, 11), 12, 21)
    assert cells.tobytes() == one.tobytes()


def test_periodic_culling_blank_volume(ora):
    """A uniform image has no blob: the MC energy stays above E0 = -3 (|E| <= 2.4,
    SURVEY A10), so the first checkpoint culls every cell."""
    vol = np.full((48, 48, 48), 60 * 257, np.uint16)
    p = ora.Params(r0=10.0, n_samples=256, dim=3, max_iters=60)
    st, seeds = ora.seeds_lattice((48, 48, 48), 3, 10.0)
    live = ora.evolve_periodic(vol, p, seeds, 20)
    assert len(seeds) == 27 and len(live) == 0


def test_periodic_culling_c1_same_detections(ora):
    """On C1 (64 lattice snakes, 8 nuclei) culling every 50 iterations still finds
    one detection per nucleus (A9 / AC6); cells never interact during evolution,
    so every detection's record is bit-identical to the same cell's record in the
    run without periodic culling (only WHICH cells survive may change: an early
    overlap competition can pick a different snake of the same nucleus); and
    every removed cell violated E0 or lost an overlap competition at its
    checkpoint."""
    cfg = synth.CONFIGS["C1"]
    raw = synth.generate(cfg)
    p = ora.Params(r0=cfg.r0, n_samples=cfg.n_samples, dim=3, seed=cfg.philox_seed)
    B = ora.blur(raw, 3, 1.0)
    st, seeds = ora.seeds_lattice(cfg.n, 3, cfg.r0)
    full = ora.evolve(B, p, seeds)
    det_full = full[ora.cull(full["c"].astype(np.float32), full["R"].astype(np.float32),
                             full["E"].astype(np.float32), full["flags"], full["id"], 3, p.e0)]
    live = ora.evolve_periodic(B, p, seeds, 50)
    assert 8 <= len(live) < 64
    det = live[ora.cull(live["c"].astype(np.float32), live["R"].astype(np.float32),
                        live["E"].astype(np.float32), live["flags"], live["id"], 3, p.e0)]
    assert len(det) == 8 and len(det_full) == 8
    truth = synth.nuclei(cfg)
    d = np.linalg.norm(det["c"][:, None, :] - truth["c"][None, :, :], axis=2)
    assert sorted(np.argmin(d, axis=1).tolist()) == list(range(8)) and d.min(axis=1).max() < 2.0
    assert det.tobytes() == full[det["id"]].tobytes()
    # the survivors of the checkpoint are exactly the O6 survivors of the records there
    cells = ora.evolve_range(B, p, ora.init_cells(p, seeds), 1, 50)
    keep = ora.cull(cells["c"].astype(np.float32), cells["R"].astype(np.float32),
                    cells["E"].astype(np.float32), cells["flags"], cells["id"], 3, p.e0)
    dropped = np.setdiff1d(np.arange(64), keep)
    c32, R32 = cells["c"].astype(np.float32).astype(np.float64), cells["R"].astype(np.float32).astype(np.float64)
    rho = 2.0 ** (-1.0 / 3.0)
    for i in dropped:
        bad_e = np.float32(cells["E"][i]) > p.e0 or cells["flags"][i] & (ora.COLLAPSED | ora.RMAX)
        lost = any(np.sum((c32[i] - c32[a]) ** 2) < (rho * max(R32[i], R32[a])) ** 2
                   and (np.float32(cells["E"][a]), a) < (np.float32(cells["E"][i]), i) for a in keep)
        assert bad_e or lost, f"cell {i} dropped without a reason"
