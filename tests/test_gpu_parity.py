"""GPU (libsnk, sm_100a) vs the fp64 CPU oracle, element by element.

Contract: integer volume passes, seeds, culling and labels
bit-exact; per-cell R and c within 1e-3 voxel and E within 1e-3 max(1, |E|)
(fp32 vs fp64, same Philox samples); evolution bit-identical across
warps-per-cell schedules.  Oracle inputs are always computed by the oracle
from the raw synthetic volume — never taken from the CUDA path.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_RC = 1e-3


def _t(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _ora_params(cfg, **kw):
    d = dict(r0=cfg.r0, n_samples=cfg.n_samples, max_iters=cfg.max_iters, dim=cfg.dim,
             seed=cfg.philox_seed)
    d.update(kw)
    return oracle.Params(**d)


def _assert_cells_close(g, o, ctx=""):
    """GPU snk_cell records vs oracle cells (same order)."""
    assert len(g) == len(o), ctx
    dR = np.abs(g["R"].astype(np.float64) - o["R"])
    dc = np.abs(g["c"].astype(np.float64) - o["c"]).max(axis=1)
    dE = np.abs(g["energy"].astype(np.float64) - o["E"]) / np.maximum(1.0, np.abs(o["E"]))
    assert np.array_equal(g["id"], o["id"]), ctx
    assert np.array_equal(g["seed"].astype(np.float64), o["seed"]), ctx
    bad = np.nonzero((dR > TOL_RC) | (dc > TOL_RC) | (dE > 1e-3))[0]
    assert len(bad) == 0, (f"{ctx}: {len(bad)}/{len(g)} cells out of tolerance; worst dR={dR.max():.3g} "
                           f"dc={dc.max():.3g} dE={dE.max():.3g}; first {bad[:5]}")
    return dR.max(), dc.max(), dE.max()


# ---------------------------------------------------------------- a1-a3 volume passes


@pytest.mark.parametrize("dim,shape,sigma", [(3, (37, 45, 67), 1.0), (3, (2, 17, 9), 1.0),
                                             (3, (21, 33, 70), 2.0), (3, (12, 13, 14), 0.0),
                                             (2, (1, 129, 257), 1.0), (3, (9, 5, 300), 0.5),
                                             # x extent % 8 == 0: the vectorised passes
                                             (3, (19, 23, 64), 1.0), (3, (10, 12, 136), 2.0),
                                             (3, (7, 9, 8), 1.0), (3, (33, 17, 48), 0.5),
                                             (2, (1, 100, 256), 1.0), (2, (1, 31, 8), 2.0),
                                             # nz > 32: the column-streamed z pass, ragged last chunk
                                             (3, (70, 9, 16), 1.0), (3, (41, 6, 24), 2.0), (3, (33, 7, 8), 0.5),
                                             # the TMA blur: several x / y tiles, z chunks of 64 + ragged
                                             (3, (130, 70, 136), 1.0), (3, (67, 33, 64), 2.0),
                                             (3, (3, 100, 200), 1.0), (2, (1, 97, 520), 1.0),
                                             # odd radii (h = 3, 1): TMA stages padded to 128 bytes
                                             (3, (40, 37, 72), 0.75), (3, (20, 50, 64), 0.25)])
def test_blur_gradmag_bitexact(gpu, dim, shape, sigma):
    torch, snk, _ = gpu
    rng = np.random.default_rng(hash(shape) % 2 ** 32)
    vol = rng.integers(0, 65536, size=shape, dtype=np.uint16)
    n = (shape[2], shape[1], shape[0])
    g = snk.make_grid(dim, n)
    p = snk.make_params(10.0, sigma=sigma)
    d_in = _t(torch, vol)
    sm, gm = torch.empty_like(d_in), torch.empty_like(d_in)
    ws = torch.empty(snk.snk_workspace_bytes(g, p, 16), dtype=torch.uint8, device="cuda")
    snk.snk_preprocess(g, p, d_in, sm, gm, ws)
    torch.cuda.synchronize()
    B = oracle.blur(vol, dim, sigma)
    assert np.array_equal(sm.cpu().numpy(), B)
    assert np.array_equal(gm.cpu().numpy(), oracle.gradmag(B, dim))


@pytest.mark.parametrize("dim,shape", [(3, (6, 10, 64)), (3, (5, 7, 67)), (2, (1, 20, 32))])
def test_gradmag_extreme_bitexact(gpu, dim, shape):
    """a3 at the largest gradients (0 / 65535 checkerboards, v up to 3 * 65535^2):
    the float-estimated isqrt must still be exact."""
    torch, snk, _ = gpu
    z, y, x = np.indices(shape)
    vol = (((x + y + z) % 2) * 65535).astype(np.uint16)
    vol[:, :, ::3] = 65535 - vol[:, :, ::3]
    n = (shape[2], shape[1], shape[0])
    g = snk.make_grid(dim, n)
    p = snk.make_params(10.0, sigma=0.0)
    d_in = _t(torch, vol)
    sm, gm = torch.empty_like(d_in), torch.empty_like(d_in)
    ws = torch.empty(snk.snk_workspace_bytes(g, p, 16), dtype=torch.uint8, device="cuda")
    snk.snk_preprocess(g, p, d_in, sm, gm, ws)
    torch.cuda.synchronize()
    assert np.array_equal(sm.cpu().numpy(), vol)
    assert np.array_equal(gm.cpu().numpy(), oracle.gradmag(vol, dim))


@pytest.mark.parametrize("dim,shape,w", [(3, (30, 26, 64), 3), (3, (21, 19, 40), 0), (3, (40, 36, 32), 8),
                                         (3, (25, 22, 45), 5), (2, (1, 90, 128), 6), (2, (1, 70, 75), 4),
                                         # nz > 32: the column-streamed z fold
                                         (3, (75, 20, 24), 5), (3, (33, 10, 16), 1), (3, (97, 6, 8), 2),
                                         (3, (140, 70, 136), 5), (3, (66, 100, 72), 4)])
def test_seeds_maxima_plateaus_bitexact(gpu, dim, shape, w):
    """a4 MAXIMA on quantised random volumes (many equal values: the tie rule
    decides), vectorised (x % 8 == 0) and fallback paths, w in {0, .., 8}."""
    torch, snk, _ = gpu
    rng = np.random.default_rng(sum(shape) + w)
    vol = (rng.integers(0, 12, size=shape) * 5000).astype(np.uint16)
    n = (shape[2], shape[1], shape[0])
    g = snk.make_grid(dim, n)
    p = snk.make_params(10.0, seed_mode=snk.SEED_MAXIMA, seed_window=w, seed_threshold=20000)
    cap = int(np.prod(shape)) + 16
    seeds = torch.empty((cap, 3), dtype=torch.float32, device="cuda")
    ws = torch.empty(max(snk.snk_workspace_bytes(g, p, 16), 16), dtype=torch.uint8, device="cuda")
    cnt, _ = snk.snk_seeds(g, p, _t(torch, vol), seeds, cap, ws)
    exp = oracle.seeds_maxima(vol, dim, w, 20000)
    assert cnt == len(exp) > 0
    assert np.array_equal(seeds[:cnt].cpu().numpy(), exp)


@pytest.mark.parametrize("shape,w", [((75, 20, 24), 5), ((40, 36, 32), 8), ((140, 70, 136), 5),
                                     ((50, 33, 80), 7), ((30, 40, 16), 2), ((66, 100, 72), 4)])
def test_seeds_maxima_tma_path(gpu, monkeypatch, shape, w):
    """The one-pass TMA MAXIMA kernel (SNK_TMA_MAXIMA=1: several x / y tiles, z
    chunks, ragged edges): bit-exact like the default box-max passes."""
    torch, snk, _ = gpu
    monkeypatch.setenv("SNK_TMA_MAXIMA", "1")
    rng = np.random.default_rng(sum(shape) + w)
    vol = (rng.integers(0, 12, size=shape) * 5000).astype(np.uint16)
    g = snk.make_grid(3, (shape[2], shape[1], shape[0]))
    p = snk.make_params(10.0, seed_mode=snk.SEED_MAXIMA, seed_window=w, seed_threshold=20000)
    cap = int(np.prod(shape)) + 16
    seeds = torch.empty((cap, 3), dtype=torch.float32, device="cuda")
    ws = torch.empty(max(snk.snk_workspace_bytes(g, p, 16), 16), dtype=torch.uint8, device="cuda")
    cnt, _ = snk.snk_seeds(g, p, _t(torch, vol), seeds, cap, ws)
    exp = oracle.seeds_maxima(vol, 3, w, 20000)
    assert cnt == len(exp) > 0
    assert np.array_equal(seeds[:cnt].cpu().numpy(), exp)


@pytest.mark.parametrize("n,spacing", [((40, 36, 20), (1.0, 1.0, 2.0)), ((23, 17, 11), (3.0, 1.5, 1.0)),
                                       ((16, 16, 9), (1.0, 1.0, 2.7))])
def test_resample_bitexact(gpu, n, spacing):
    torch, snk, _ = gpu
    rng = np.random.default_rng(7)
    raw = rng.integers(0, 65536, size=(n[2], n[1], n[0]), dtype=np.uint16)
    no = snk.snk_resample_dims(3, n, spacing)
    out = torch.empty((no[2], no[1], no[0]), dtype=torch.uint16, device="cuda")
    ws = torch.empty(4 * no[0] * no[1] * no[2] * 2 + 4096, dtype=torch.uint8, device="cuda")
    snk.snk_resample(3, n, spacing, 0, n[2], _t(torch, raw), 0, no[2], out, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.resample(raw, spacing, 3))


def test_resample_c3_full(gpu):
    torch, snk, _ = gpu
    cfg = synth.CONFIGS["C3"]
    raw = synth.generate(cfg)
    no = snk.snk_resample_dims(3, cfg.n, cfg.spacing)
    out = torch.empty((no[2], no[1], no[0]), dtype=torch.uint16, device="cuda")
    snk.snk_resample(3, cfg.n, cfg.spacing, 0, cfg.n[2], _t(torch, raw), 0, no[2], out, None)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.resample(raw, cfg.spacing, 3))


# ---------------------------------------------------------------- a4 seeds


def test_seeds_lattice_bitexact(gpu):
    torch, snk, _ = gpu
    for dim, n, r0 in [(3, (64, 64, 64), 10.0), (3, (100, 77, 51), 9.0), (2, (2048, 2048, 1), 25.0)]:
        g = snk.make_grid(dim, n)
        p = snk.make_params(r0, seed_mode=snk.SEED_LATTICE)
        seeds = torch.empty((100_000, 3), dtype=torch.float32, device="cuda")
        cnt, first = snk.snk_seeds(g, p, None, seeds, 100_000, None)
        st, exp = oracle.seeds_lattice(n, dim, r0)
        assert st == 0 and first == 0
        assert np.array_equal(seeds[:cnt].cpu().numpy(), exp)
    g = snk.make_grid(3, (20, 64, 64))
    with pytest.raises(snk.SNKError) as e:
        snk.snk_seeds(g, snk.make_params(10.0, seed_mode=snk.SEED_LATTICE), None, seeds, 10, None)
    assert e.value.status == snk.EMPTY_DOMAIN


def _gpu_smooth_seeds(torch, snk, pipeline, cfg, **over):
    p = pipeline.params_for(cfg, **over)
    P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing)
    raw = synth.generate(cfg)
    P.upload(raw)
    P.preprocess()
    P.seed()
    torch.cuda.synchronize()
    return P, raw, p


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_seeds_maxima_bitexact_full(gpu, name):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS[name]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg, seed_mode=snk.SEED_MAXIMA)
    vol = raw if cfg.dim == 3 else raw
    B = oracle.blur(vol, cfg.dim, 1.0)
    assert np.array_equal(P.smooth.cpu().numpy().reshape(B.shape), B)
    exp = oracle.seeds_maxima(B, cfg.dim, cfg.window, cfg.seed_threshold)
    assert P.n_seeds == len(exp) > 0
    assert np.array_equal(P.seeds_np(), exp)


def _crop(lo, hi):
    return tuple(slice(int(lo[a]), int(hi[a]) + 1) for a in (2, 1, 0))


def _oracle_smooth_crop(raw_iso, lo, hi, n):
    """Oracle blur of raw[lo-4 .. hi+4] (clipped); returns (org, crop) whose voxels
    lo..hi are exact (clamp-to-edge only acts at the true volume boundary)."""
    m = 4
    a = np.maximum(np.asarray(lo) - m, 0)
    b = np.minimum(np.asarray(hi) + m, np.asarray(n) - 1)
    B = oracle.blur(raw_iso[_crop(a, b)], 3, 1.0)
    return a, B


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_size_sampled_parity(gpu, name):
    """Full BASELINE sizes in the bench's launch configuration (auto kernel choice):
    sampled crops of the smoothed volume and the seed list are bit-exact; sampled
    cells evolve within tolerance; the full-launch results for those cells are
    bit-identical to a separate launch of just them."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS[name]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    n = P.n_iso
    raw_iso = oracle.resample(raw, cfg.spacing, 3) if P.resample else raw
    if P.resample:   # resampled volume: sampled planes bit-exact
        for z in [0, 1, n[2] // 2, n[2] - 1]:
            assert np.array_equal(P.iso[z].cpu().numpy(), raw_iso[z])
    rng = np.random.default_rng(12)
    gseeds = P.seeds_np()
    w = cfg.window
    test_seeds = []
    for k in range(3):
        size = np.array([96, 96, 64])
        lo = np.array([rng.integers(0, n[a] - size[a]) for a in range(3)])
        hi = lo + size - 1
        org, B = _oracle_smooth_crop(raw_iso, lo, hi, n)
        gs = P.smooth[_crop(lo, hi)].cpu().numpy()
        assert np.array_equal(gs, B[_crop(lo - org, hi - org)])
        ilo, ihi = lo + w, hi - w
        exp = oracle.seeds_maxima(B, 3, w, cfg.seed_threshold, org=org, n_global=n, lo=ilo, hi=ihi)
        sel = np.all((gseeds >= ilo) & (gseeds <= ihi), axis=1)
        assert np.array_equal(gseeds[sel], exp)
        test_seeds.append(exp[rng.permutation(len(exp))[:8]])
    seeds = np.concatenate(test_seeds).astype(np.float32)
    ids = rng.permutation(1 << 20)[:len(seeds)].astype(np.int64) + 12345
    # GPU: the bench's kernel configuration (auto: brick kernel), explicit seeds and ids
    p1 = pipeline.params_for(cfg)
    cells = torch.empty(len(seeds) * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_evolve(P.grid, p1, P.smooth, _t(torch, seeds), _t(torch, ids), 0, len(seeds), cells, None)
    torch.cuda.synchronize()
    g = pipeline.as_cells(cells, len(seeds))
    # oracle: each cell on an oracle-smoothed crop covering everything it can reach
    op = _ora_params(cfg)
    reach = int(np.ceil(2 * cfg.r0 + 2 * cfg.r0 + 1.0 + 2))
    outs = []
    for s, i in zip(seeds, ids):
        lo = np.maximum(np.floor(s).astype(int) - reach, 0)
        hi = np.minimum(np.ceil(s).astype(int) + reach, np.asarray(n) - 1)
        org, B = _oracle_smooth_crop(raw_iso, lo, hi, n)
        outs.append(oracle.evolve(B, op, s[None], ids=np.array([i]), org=org, n_global=n)[0])
    o = np.array(outs, dtype=oracle.CELL_DTYPE)
    assert not np.any(o["flags"] & oracle.HALO)
    _assert_cells_close(g, o, name)
    # the full launch (all seeds, as bench.py times it) gives bit-identical cells
    P.params = p1
    P.evolve()
    torch.cuda.synchronize()
    allc = P.cells_np()
    idx = [int(np.nonzero(np.all(gseeds == s, axis=1))[0][0]) for s in seeds]
    full = allc[idx]
    # same cells with the pipeline's ids in a separate small launch: identical bytes
    snk.snk_evolve(P.grid, p1, P.smooth, _t(torch, seeds), _t(torch, full["id"].copy()), 0,
                   len(seeds), cells, None)
    torch.cuda.synchronize()
    again = pipeline.as_cells(cells, len(seeds))
    assert again.tobytes() == full.tobytes()


# ---------------------------------------------------------------- a5-a6 evolution


def test_evolve_c1_parity_and_schedules(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    B = oracle.blur(raw, 3, 1.0)
    st, oseeds = oracle.seeds_lattice(cfg.n, 3, cfg.r0)
    assert np.array_equal(P.seeds_np(), oseeds)
    ref = None
    # warp kernel (global gathers) at W = 1..8 and brick kernel (TMA + smem) at W = 4, 8
    for variant, W in ((1, 1), (1, 2), (1, 4), (1, 8), (2, 4), (2, 8), (0, 0)):
        P.params = pipeline.params_for(cfg, cta_warps=W, kernel_variant=variant)
        P.evolve()
        torch.cuda.synchronize()
        c = P.cells_np()
        if ref is None:
            ref = c
        assert c.tobytes() == ref.tobytes(), f"variant={variant} cta_warps={W} differs"
    o = oracle.evolve(B, _ora_params(cfg), oseeds, ids=np.arange(len(oseeds)))
    _assert_cells_close(ref, o, "C1")
    fmask = oracle.COLLAPSED | oracle.RMAX
    assert np.array_equal(ref["flags"] & fmask, o["flags"] & fmask)


@pytest.mark.parametrize("r0", [14.0, 18.0])
def test_brick_reload_and_global_fallback(gpu, r0):
    """Large contours whose sampled ball does not always fit the 32^3 brick take
    the global-gather path for those iterations; lattice snakes far from nuclei
    move and force brick re-centring.  Both kernels agree bit for bit and with
    the oracle."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(r0=r0, max_iters=120, n_samples=256)
    n = (72, 72, 72)
    raw = synth.generate(synth.CONFIGS["C1"].with_(n=n))
    p = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE)
    P = pipeline.Pipeline(3, n, p)
    P.upload(raw)
    P.preprocess()
    P.seed()
    out = []
    for variant in (1, 2):
        P.params = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE, kernel_variant=variant,
                                       cta_warps=4 if variant == 2 else 0)
        P.evolve()
        torch.cuda.synchronize()
        out.append(P.cells_np())
    assert out[0].tobytes() == out[1].tobytes()
    B = oracle.blur(raw, 3, 1.0)
    o = oracle.evolve(B, _ora_params(cfg), P.seeds_np(), ids=np.arange(P.n_seeds))
    _assert_cells_close(out[1], o, f"r0={r0}")


@pytest.mark.parametrize("N", [32, 64, 256, 4096])
def test_evolve_sample_counts(gpu, N):
    """C5's N sweep: every per-thread block size (B = 1 .. 128) matches the oracle."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(n_samples=N, max_iters=60)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    B = oracle.blur(raw, 3, 1.0)
    for W in ((1, 8) if N >= 256 else (1,)):
        P.params = pipeline.params_for(cfg, cta_warps=W)   # N >= 256: W=8 takes the brick kernel
        P.evolve(n=16)
        torch.cuda.synchronize()
        g = P.cells_np()[:16]
        o = oracle.evolve(B, _ora_params(cfg), P.seeds_np()[:16], ids=np.arange(16))
        _assert_cells_close(g, o, f"N={N} W={W}")


def test_evolve_2d_parity(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C2"]
    raw = synth.generate(cfg)[0]
    sub = np.ascontiguousarray(raw[:300, :400])
    c2 = cfg.with_(n=(400, 300, 1), max_iters=400)
    p = pipeline.params_for(c2)
    P = pipeline.Pipeline(2, c2.n, p)
    P.upload(sub[None])
    P.preprocess()
    P.seed()
    torch.cuda.synchronize()
    B = oracle.blur(sub[None], 2, 1.0)
    assert np.array_equal(P.smooth.cpu().numpy(), B)
    exp = oracle.seeds_maxima(B, 2, c2.window, c2.seed_threshold)
    assert np.array_equal(P.seeds_np(), exp) and len(exp) > 5
    P.evolve()
    torch.cuda.synchronize()
    o = oracle.evolve(B, _ora_params(c2), exp, ids=np.arange(len(exp)))
    _assert_cells_close(P.cells_np(), o, "2D")
    assert np.all(P.cells_np()["c"][:, 2] == 0)


def test_evolve_slab_buffer_bit_identical(gpu):
    """T4 on one GPU: a z-slab buffer (with halo) gives the same cells as the whole volume."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.evolve()
    torch.cuda.synchronize()
    full = P.cells_np()
    sel = np.nonzero(P.seeds_np()[:, 2] < 20)[0]
    z1 = 20 + int(np.ceil(2 * cfg.r0 + 2 * cfg.r0 + 2 + 2))
    g = snk.make_grid(3, (64, 64, 64), z_lo=0, nz_buf=z1, own=(0, 20))
    cells = torch.empty(len(sel) * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_evolve(g, p, P.smooth[:z1].contiguous(), P.seeds[sel].contiguous(),
                   _t(torch, sel.astype(np.int64)), 0, len(sel), cells, None)
    torch.cuda.synchronize()
    got = pipeline.as_cells(cells, len(sel))
    assert got.tobytes() == full[sel].tobytes()


# ---------------------------------------------------------------- grid estimator (Eq. 5)


@pytest.mark.parametrize("r0,T", [(10.0, 400), (14.0, 150), (18.0, 80)])
def test_evolve_grid_parity(gpu, r0, T):
    """SNK_EST_GRID: the paper's uniform integration (Eq. 5 over the voxels of
    the ball) vs the oracle's grid mode, fp32 vs fp64.  r0 = 14 and 18 move the
    brick and take the global path (balls larger than the brick)."""
    torch, snk, pipeline = gpu
    n = (64, 64, 64) if r0 == 10.0 else (72, 72, 72)
    cfg = synth.CONFIGS["C1"].with_(r0=r0, max_iters=T, n=n)
    raw = synth.generate(synth.CONFIGS["C1"].with_(n=n))
    p = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE, estimator=snk.EST_GRID)
    P = pipeline.Pipeline(3, n, p)
    P.upload(raw)
    P.preprocess()
    P.seed()
    P.evolve()
    torch.cuda.synchronize()
    g = P.cells_np()
    P.evolve()
    torch.cuda.synchronize()
    assert P.cells_np().tobytes() == g.tobytes(), "grid evolution is not deterministic"
    B = oracle.blur(raw, 3, 1.0)
    o = oracle.evolve(B, _ora_params(cfg, mode=1), P.seeds_np(), ids=np.arange(P.n_seeds))
    _assert_cells_close(g, o, f"grid r0={r0}")
    fmask = oracle.COLLAPSED | oracle.RMAX
    assert np.array_equal(g["flags"] & fmask, o["flags"] & fmask)


def test_evolve_grid_2d_and_slab(gpu):
    """Grid estimator in 2D (C2 crop) and on a z-slab buffer (bit-identical to the whole volume)."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C2"]
    sub = np.ascontiguousarray(synth.generate(cfg)[0][:200, :256])
    c2 = cfg.with_(n=(256, 200, 1), max_iters=200)
    p = pipeline.params_for(c2, estimator=snk.EST_GRID)
    P = pipeline.Pipeline(2, c2.n, p)
    P.upload(sub[None])
    P.preprocess()
    P.seed()
    P.evolve()
    torch.cuda.synchronize()
    B = oracle.blur(sub[None], 2, 1.0)
    o = oracle.evolve(B, _ora_params(c2, mode=1), P.seeds_np(), ids=np.arange(P.n_seeds))
    assert P.n_seeds > 3
    _assert_cells_close(P.cells_np(), o, "grid 2D")
    # 3D slab
    cfg = synth.CONFIGS["C1"].with_(max_iters=100)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    p = pipeline.params_for(cfg, estimator=snk.EST_GRID)
    P.params = p
    P.evolve()
    torch.cuda.synchronize()
    full = P.cells_np()
    sel = np.nonzero(P.seeds_np()[:, 2] < 20)[0]
    z1 = 20 + int(np.ceil(2 * cfg.r0 + 2 * cfg.r0 + 2 + 2))
    g = snk.make_grid(3, (64, 64, 64), z_lo=0, nz_buf=z1, own=(0, 20))
    cells = torch.empty(len(sel) * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_evolve(g, p, P.smooth[:z1].contiguous(), P.seeds[sel].contiguous(),
                   _t(torch, sel.astype(np.int64)), 0, len(sel), cells, None)
    torch.cuda.synchronize()
    assert pipeline.as_cells(cells, len(sel)).tobytes() == full[sel].tobytes()


# ---------------------------------------------------------------- CV and ray-march estimators (§8(f) 3-4)


@pytest.mark.parametrize("est,mode,W,N", [("EST_MC_CV", 2, 4, 1024), ("EST_RAY", 3, 4, 1024),
                                         ("EST_RAY", 3, 8, 2048)])
def test_evolve_estimator_variants(gpu, est, mode, W, N):
    """Control-variate MC (G21) and the stratified ray march (G27) vs the
    oracle's modes 2 and 3 (same Philox words, fp32 vs fp64); a z-slab buffer
    gives bit-identical cells; the 2D mode on a C2 crop."""
    torch, snk, pipeline = gpu
    e = getattr(snk, est)
    cfg = synth.CONFIGS["C1"].with_(n_samples=N, max_iters=200)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg, estimator=e, cta_warps=W)
    P.evolve()
    torch.cuda.synchronize()
    g = P.cells_np()
    B = oracle.blur(raw, 3, 1.0)
    o = oracle.evolve(B, _ora_params(cfg, mode=mode), P.seeds_np(), ids=np.arange(P.n_seeds))
    _assert_cells_close(g, o, est)
    sel = np.nonzero(P.seeds_np()[:, 2] < 20)[0]
    z1 = 20 + int(np.ceil(2 * cfg.r0 + 2 * cfg.r0 + 2 + 2))
    gs = snk.make_grid(3, (64, 64, 64), z_lo=0, nz_buf=z1, own=(0, 20))
    cells = torch.empty(len(sel) * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_evolve(gs, p, P.smooth[:z1].contiguous(), P.seeds[sel].contiguous(),
                   _t(torch, sel.astype(np.int64)), 0, len(sel), cells, None)
    torch.cuda.synchronize()
    assert pipeline.as_cells(cells, len(sel)).tobytes() == g[sel].tobytes()
    if W == 4:
        c2 = synth.CONFIGS["C2"]
        sub = np.ascontiguousarray(synth.generate(c2)[0][:200, :256])
        c2 = c2.with_(n=(256, 200, 1), max_iters=150, n_samples=N)
        P = pipeline.Pipeline(2, c2.n, pipeline.params_for(c2, estimator=e))
        P.upload(sub[None])
        P.preprocess()
        P.seed()
        P.evolve()
        torch.cuda.synchronize()
        o = oracle.evolve(oracle.blur(sub[None], 2, 1.0), _ora_params(c2, mode=mode), P.seeds_np(),
                          ids=np.arange(P.n_seeds))
        assert P.n_seeds > 3
        _assert_cells_close(P.cells_np(), o, est + " 2D")


def test_estimator_variant_config_errors(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.params = pipeline.params_for(cfg, estimator=snk.EST_RAY)   # N = 256: not 256 * warps
    with pytest.raises(snk.SNKError) as ei:
        P.evolve()
    assert ei.value.status == snk.CONFIG


# ---------------------------------------------------------------- periodic culling


def test_evolve_range_resumes_bit_exactly(gpu):
    """Segments 1..a, a+1..b, ..., ..T+1 of snk_evolve_range from the records give
    records bit-identical to one snk_evolve, for the brick, warp and grid kernels."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(max_iters=90)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    n = P.n_seeds
    for kw in (dict(), dict(kernel_variant=1, cta_warps=2), dict(estimator=snk.EST_GRID)):
        p = pipeline.params_for(cfg, **kw)
        P.params = p
        P.evolve()
        torch.cuda.synchronize()
        one = P.cells_np()
        cells = torch.empty(n * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
        snk.snk_cells_init(p, P.seeds, None, 0, n, cells)
        for a, b in [(1, 1), (2, 40), (41, 90), (91, 91)]:
            snk.snk_evolve_range(P.grid, p, P.smooth, cells, n, a, b, None)
        torch.cuda.synchronize()
        assert pipeline.as_cells(cells, n).tobytes() == one.tobytes(), kw


def test_periodic_culling_c1_vs_oracle(gpu):
    """cull_every = 50 on C1: the GPU (pipeline and snk_run) keeps the same cells
    at every checkpoint as the oracle (E, c, R within tolerance), and the final
    detections match; every checkpoint cull is bit-exact given the GPU records."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"]
    k = 50
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg, cull_every=k)
    B = oracle.blur(raw, 3, 1.0)
    op = _ora_params(cfg)
    seeds = P.seeds_np()
    # stage by stage: GPU segments, oracle cull of the GPU records == GPU cull
    n = P.n_seeds
    cur = torch.empty(n * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    nxt = torch.empty(n * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_cells_init(p, P.seeds, None, 0, n, cur)
    ocells = oracle.init_cells(op, seeds)
    live = n
    for i, (a, b) in enumerate(snk.checkpoints(cfg.max_iters, k)):
        snk.snk_evolve_range(P.grid, p, P.smooth, cur, live, a, b, None)
        ocells = oracle.evolve_range(B, op, ocells, a, b)
        torch.cuda.synchronize()
        g = pipeline.as_cells(cur, live)
        o = ocells[np.argsort(ocells["id"])]
        gs = g[np.argsort(g["id"])]
        _assert_cells_close(gs, o, f"segment {a}..{b}")
        if b > cfg.max_iters:
            break
        live = snk.snk_cull(P.grid, p, cur, live, nxt, n, P.ws)
        keep = oracle.cull(g["c"], g["R"], g["energy"], g["flags"], g["id"], 3, op.e0)
        assert pipeline.as_cells(nxt, live).tobytes() == g[keep].tobytes(), f"checkpoint {b}"
        okeep = oracle.cull(ocells["c"].astype(np.float32), ocells["R"].astype(np.float32),
                            ocells["E"].astype(np.float32), ocells["flags"], ocells["id"], 3, op.e0)
        assert np.array_equal(np.sort(ocells["id"][okeep]), np.sort(g["id"][keep])), f"checkpoint {b}"
        ocells = ocells[np.sort(okeep)]
        cur, nxt = nxt, cur
    # the pipeline's periodic path and the end-to-end host call agree bit for bit
    P.evolve()
    P.cull()
    torch.cuda.synchronize()
    dets = P.dets_np()
    o = oracle.evolve_periodic(B, op, seeds, k)
    okeep = oracle.cull(o["c"].astype(np.float32), o["R"].astype(np.float32), o["E"].astype(np.float32),
                        o["flags"], o["id"], 3, op.e0)
    assert np.array_equal(dets["id"], o["id"][okeep]) and len(dets) == 8
    _assert_cells_close(dets, o[okeep], "periodic detections")
    hr = pipeline.HostRunner(3, cfg.n, p)
    h_raw = torch.from_numpy(raw).pin_memory()
    nd = hr.run(h_raw)
    assert nd == len(dets) and hr.dets_np(nd).tobytes() == dets.tobytes()


# ---------------------------------------------------------------- a7-a8, stage-isolated and end to end


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_cull_and_label_stage_isolated(gpu, name):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS[name]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.evolve()
    P.cull()
    P.label()
    torch.cuda.synchronize()
    cells = P.cells_np()
    keep = oracle.cull(cells["c"], cells["R"], cells["energy"], cells["flags"], cells["id"], cfg.dim,
                       -3.0)
    dets = P.dets_np()
    assert dets.tobytes() == cells[keep].tobytes()
    n = P.n_iso
    if name == "C1":
        lab = oracle.label(n, 3, dets["c"], dets["R"])
        assert np.array_equal(P.labels.cpu().numpy(), lab)
    else:
        rng = np.random.default_rng(3)
        pts = np.stack([rng.integers(0, n[a], 200_000) for a in range(3)], axis=1)
        # plus every detection's centre neighbourhood (where labels are dense)
        cen = np.round(dets["c"][:2000]).astype(np.int64)
        pts = np.concatenate([pts, cen, np.clip(cen + 3, 0, np.asarray(n) - 1)])
        exp = oracle.label_points(3, pts, dets["c"], dets["R"])
        got = P.labels.cpu().numpy()[pts[:, 2], pts[:, 1], pts[:, 0]]
        assert np.array_equal(got, exp)
    assert (P.labels.cpu().numpy() > 0).any()


def _crafted_dets(snk, rng, n, dim, k):
    """Detections built to exercise every rule of O7: heavily overlapping inner
    balls (second-ball keys), exact duplicates (equal keys: the smaller index
    wins), integer centres with radii whose inner ball passes through voxel
    centres (d2 == thr up to rounding: the fp32 filter's band), balls cut by the
    volume faces."""
    d = np.zeros(k, snk.CELL_DTYPE)
    c = rng.uniform(-3, np.asarray(n, np.float64) + 3, (k, 3)).astype(np.float32)
    R = rng.uniform(2.0, 9.0, k).astype(np.float32)
    h = k // 4
    c[h:2 * h] = c[:h] + rng.uniform(-2, 2, (h, 3)).astype(np.float32)   # overlapping partners
    c[2 * h:2 * h + h // 2] = c[:h // 2]                                  # exact duplicates
    R[2 * h:2 * h + h // 2] = R[:h // 2]
    c[3 * h:] = np.round(c[3 * h:])                                       # boundary-band radii
    rho = 2.0 ** (-1.0 / dim)
    R[3 * h:] = (np.sqrt(rng.integers(4, 60, k - 3 * h)) / rho).astype(np.float32)
    if dim == 2:
        c[:, 2] = 0.0
    d["c"], d["R"] = c, R
    return d


@pytest.mark.parametrize("dim,n,k,scale", [(3, (70, 45, 40), 400, (1.0, 1.0, 1.0)),
                                           (3, (64, 40, 33), 300, (1.0, 1.0, 2.0)),
                                           (2, (150, 110, 1), 500, (1.0, 1.0, 1.0))])
def test_label_crafted_bitexact(gpu, dim, n, k, scale):
    """a8 alone on crafted detection lists: the whole label map equals the
    oracle's fp64 definition (O7, G19) bit for bit."""
    torch, snk, _ = gpu
    rng = np.random.default_rng(k + dim)
    dets = _crafted_dets(snk, rng, n, dim, k)
    g = snk.make_grid(dim, n, scale=scale)
    p = snk.make_params(10.0)
    d_dets = torch.from_numpy(dets.view(np.uint8)).cuda()
    lab = torch.empty((n[2], n[1], n[0]), dtype=torch.int32, device="cuda")
    ws = torch.empty(snk.snk_workspace_bytes(g, p, k), dtype=torch.uint8, device="cuda")
    snk.snk_label(g, p, d_dets, k, lab, ws)
    torch.cuda.synchronize()
    exp = oracle.label(n, dim, dets["c"], dets["R"], scale=scale)
    got = lab.cpu().numpy()
    assert (exp > 0).mean() > 0.2
    assert np.array_equal(got, exp), f"{int((got != exp).sum())} voxels differ"


@pytest.mark.parametrize("n,off", [(1 << 20, 0), (100_003, 0), (4099, 3)])
def test_ingest_u8_bitexact(gpu, n, off):
    """a0: snk_ingest_u8 = O0 (257 v), vectorised (16-byte aligned) and scalar
    (unaligned) kernels, ragged lengths."""
    torch, snk, _ = gpu
    rng = np.random.default_rng(n)
    v = rng.integers(0, 256, n, dtype=np.uint8)
    d_in = torch.empty(n + 16, dtype=torch.uint8, device="cuda")
    d_in[off:off + n] = _t(torch, v)
    d_out = torch.empty(n + 16, dtype=torch.int16, device="cuda")
    snk.snk_ingest_u8(d_in.data_ptr() + off, d_out.data_ptr() + 2 * off, n)
    torch.cuda.synchronize()
    got = d_out.cpu().numpy().view(np.uint16)[off:off + n]
    assert np.array_equal(got, oracle.ingest_u8(v))


def test_run_u8_equals_run(gpu):
    """snk_run_u8 (8-bit host volume, promoted on the device) gives the
    detections and label map of snk_run on the u16 volume O0 makes of it."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(max_iters=80)
    raw8 = (synth.generate(cfg) // 257).astype(np.uint8)
    p = pipeline.params_for(cfg)
    H = pipeline.HostRunner(cfg.dim, cfg.n, p)
    n8 = H.run(torch.from_numpy(raw8).pin_memory())
    d8, l8 = H.dets_np(n8), H.h_labels.numpy().copy()
    n16 = H.run(torch.from_numpy(oracle.ingest_u8(raw8)).pin_memory())
    assert n8 == n16 > 0
    assert H.dets_np(n16).tobytes() == d8.tobytes()
    assert np.array_equal(H.h_labels.numpy(), l8)


def test_end_to_end_c1_and_host_call(gpu):
    """C1 through the device pipeline and through snk_run (host buffers) against
    the oracle's own end-to-end run."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.evolve()
    P.cull()
    P.label()
    torch.cuda.synchronize()
    res = oracle.run_pipeline(raw, _ora_params(cfg), seed_mode="lattice")
    odets = res.cells[res.keep]
    gdets = P.dets_np()
    assert len(gdets) == len(odets) == 8
    assert np.array_equal(gdets["id"], odets["id"])
    assert np.abs(gdets["c"] - odets["c"]).max() < TOL_RC
    assert np.array_equal(P.labels.cpu().numpy(), res.labels)
    H = pipeline.HostRunner(3, cfg.n, p)
    h_raw = torch.from_numpy(raw).pin_memory()
    nd = H.run(h_raw)
    assert nd == len(gdets)
    assert H.dets_np(nd).tobytes() == gdets.tobytes()
    assert np.array_equal(H.h_labels.numpy(), P.labels.cpu().numpy())


def test_host_call_resampled_c3(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C3"]
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.evolve()
    P.cull()
    P.label()
    torch.cuda.synchronize()
    H = pipeline.HostRunner(3, cfg.n, p, spacing=cfg.spacing, max_cells=P.max_cells)
    nd = H.run(torch.from_numpy(raw).pin_memory())
    assert nd == P.n_dets > 1000
    assert H.dets_np(nd).tobytes() == P.dets_np().tobytes()
    assert np.array_equal(H.h_labels.numpy(), P.labels.cpu().numpy())


# ---------------------------------------------------------------- edge cases


def test_edge_cases(gpu):
    torch, snk, pipeline = gpu
    # blank volume: no maxima above threshold -> 0 seeds, 0 detections, empty label map
    cfg = synth.CONFIGS["C1"]
    p = pipeline.params_for(cfg, seed_mode=snk.SEED_MAXIMA, seed_window=4)
    P = pipeline.Pipeline(3, (40, 30, 20), p)
    P.upload(np.full((20, 30, 40), 1000, np.uint16))
    r = P.step()
    assert (r.n_seeds, r.n_dets) == (0, 0)
    assert int(P.labels.abs().sum()) == 0
    # capacity: the required count is reported
    P2 = pipeline.Pipeline(3, cfg.n, pipeline.params_for(cfg), max_cells=10)
    P2.upload(synth.generate(cfg))
    P2.preprocess()
    with pytest.raises(snk.SNKError) as e:
        P2.seed()
    assert e.value.status == snk.CAPACITY
    # minimal 3D volume 2x2x2 and n = 0 evolve are fine
    g = snk.make_grid(3, (2, 2, 2))
    pp = snk.make_params(0.5, r_min=0.1, seed_mode=snk.SEED_MAXIMA, seed_window=1, seed_threshold=0)
    d = _t(torch, (np.arange(8, dtype=np.uint16) * 1000).reshape(2, 2, 2))
    sm = torch.empty_like(d)
    ws = torch.empty(snk.snk_workspace_bytes(g, pp, 8), dtype=torch.uint8, device="cuda")
    snk.snk_preprocess(g, pp, d, sm, None, ws)
    seeds = torch.empty((8, 3), dtype=torch.float32, device="cuda")
    n, _ = snk.snk_seeds(g, pp, sm, seeds, 8, ws)
    B = oracle.blur(d.cpu().numpy(), 3, 1.0)
    assert np.array_equal(sm.cpu().numpy(), B)
    assert np.array_equal(seeds[:n].cpu().numpy(), oracle.seeds_maxima(B, 3, 1, 0))
    snk.snk_evolve(g, pp, sm, seeds, None, 0, 0, torch.empty(snk.CELL_BYTES, dtype=torch.uint8, device="cuda"), None)
    assert snk.snk_cull(g, pp, torch.empty(snk.CELL_BYTES, dtype=torch.uint8, device="cuda"), 0,
                        torch.empty(snk.CELL_BYTES, dtype=torch.uint8, device="cuda"), 1, ws) == 0


# ---------------------------------------------------------------- anisotropic grids without resampling (§8(f) 4, G28)


def test_anisotropic_physical_pipeline_c3_crop(gpu):
    """C3's raw (1, 1, 2)-spaced volume used without resampling: per-axis blur
    (sigma_z = 0.5 voxel) and MAXIMA windows (w_z = round(w / 2)) bit-exact,
    physical seeds, evolution in physical coordinates within tolerance (MC, CV,
    ray), and the cull + label map (physical voxel positions) bit-exact given
    the GPU cells; a z-slab buffer gives bit-identical cells."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C3"]
    raw = np.ascontiguousarray(synth.generate(cfg)[40:88, 100:228, 64:192])   # 48 x 128 x 128 raw
    n = (128, 128, 48)
    sc = (1.0, 1.0, 2.0)
    c3 = cfg.with_(n=n, max_iters=120)
    p = pipeline.params_for(c3)
    P = pipeline.Pipeline(3, n, p, spacing=cfg.spacing, physical=True)
    assert P.scale == sc and P.n_iso == n
    P.upload(raw)
    P.preprocess()
    P.seed()
    torch.cuda.synchronize()
    B = oracle.blur(raw, 3, (1.0, 1.0, 0.5))
    assert np.array_equal(P.smooth.cpu().numpy(), B)
    w = c3.window
    w3 = (w, w, int(np.floor(w / 2 + 0.5)))
    exp = oracle.seeds_maxima(B, 3, w3, c3.seed_threshold, scale=sc)
    assert len(exp) > 20 and np.array_equal(P.seeds_np(), exp)
    for est, mode in (("EST_MC", 0), ("EST_MC_CV", 2), ("EST_RAY", 3)):
        P.params = pipeline.params_for(c3, estimator=getattr(snk, est))
        P.evolve(n=24)
        torch.cuda.synchronize()
        g = P.cells_np()
        o = oracle.evolve(B, _ora_params(c3, mode=mode, scale=sc), exp[:24], ids=np.arange(24))
        _assert_cells_close(g, o, "aniso " + est)
    P.params = p
    P.evolve()
    torch.cuda.synchronize()
    cells = P.cells_np()
    nd = P.cull()
    torch.cuda.synchronize()
    keep = oracle.cull(cells["c"], cells["R"], cells["energy"], cells["flags"], cells["id"], 3, -3.0)
    assert nd == len(keep) > 5 and P.dets_np().tobytes() == cells[keep].tobytes()
    P.label()
    torch.cuda.synchronize()
    dets = P.dets_np()
    lab = oracle.label(n, 3, dets["c"], dets["R"], scale=sc)
    assert np.array_equal(P.labels.cpu().numpy(), lab)
    # z-slab buffer, physical z planes [0, 20) owned
    sel = np.nonzero(P.seeds_np()[:, 2] < 20.0)[0][:16]
    g = snk.make_grid(3, n, z_lo=0, nz_buf=40, own=(0, 20), scale=sc)
    out = torch.empty(len(sel) * snk.CELL_BYTES, dtype=torch.uint8, device="cuda")
    snk.snk_evolve(g, p, P.smooth[:40].contiguous(), P.seeds[sel].contiguous(),
                   _t(torch, sel.astype(np.int64)), 0, len(sel), out, None)
    torch.cuda.synchronize()
    got = pipeline.as_cells(out, len(sel))
    ok = (got["flags"] & snk.F_HALO) == 0
    assert ok.sum() > 0 and got[ok].tobytes() == cells[sel][ok].tobytes()


def test_anisotropic_lattice_and_config_errors(gpu):
    torch, snk, pipeline = gpu
    n = (64, 60, 32)
    g = snk.make_grid(3, n, scale=(1.0, 1.0, 2.0))
    p = snk.make_params(10.0, seed_mode=snk.SEED_LATTICE)
    seeds = torch.empty((4096, 3), dtype=torch.float32, device="cuda")
    cnt, _ = snk.snk_seeds(g, p, None, seeds, 4096, None)
    st, exp = oracle.seeds_lattice(n, 3, 10.0, scale=(1.0, 1.0, 2.0))
    assert cnt == len(exp) > 1 and np.array_equal(seeds[:cnt].cpu().numpy(), exp)
    vol = torch.zeros((32, 60, 64), dtype=torch.uint16, device="cuda")
    cells = torch.empty(snk.CELL_BYTES * 4, dtype=torch.uint8, device="cuda")
    with pytest.raises(snk.SNKError):   # grid estimator is isotropic only
        snk.snk_evolve(g, snk.make_params(10.0, estimator=snk.EST_GRID), vol, seeds, None, 0, 2, cells, None)
    with pytest.raises(snk.SNKError):   # N must be 1024 (4 warps x 8 samples)
        snk.snk_evolve(g, snk.make_params(10.0, n_samples=256), vol, seeds, None, 0, 2, cells, None)


@pytest.mark.parametrize("N", [64, 128, 256, 512])   # 64: the warp kernel (faster there)
def test_small_n_small_brick_kernel(gpu, N):
    """C5's small-N regime (r0 <= 9.5, N < 1024, auto warps): the 27^3-brick
    kernel with 1-2 warps per cell matches the oracle and is bit-identical to
    the warp kernel (same canonical tree)."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(r0=9.0, n_samples=N, max_iters=120)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg, seed_mode=snk.SEED_LATTICE)
    P.evolve()
    torch.cuda.synchronize()
    g = P.cells_np()
    P.params = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE, kernel_variant=1, cta_warps=1)
    P.evolve()
    torch.cuda.synchronize()
    assert P.cells_np().tobytes() == g.tobytes()
    B = oracle.blur(raw, 3, 1.0)
    o = oracle.evolve(B, _ora_params(cfg), P.seeds_np(), ids=np.arange(P.n_seeds))
    _assert_cells_close(g, o, f"small N={N}")


@pytest.mark.parametrize("N,B", [(64, 4), (64, 16), (128, 8), (128, 32), (256, 16), (256, 32)])
def test_group_kernel_bit_identical_to_warp_kernel(gpu, monkeypatch, N, B):
    """The group kernel (N / B lanes per cell, several cells per warp; the
    default for N <= 256) takes the same canonical tree as the warp kernel:
    byte-identical records, lattice cells near the volume faces included (the
    clamped and the unclamped gathers mix inside a warp's iterations)."""
    torch, snk, pipeline = gpu
    monkeypatch.setenv("SNK_GROUP_B", str(B))
    cfg = synth.CONFIGS["C1"].with_(r0=9.0, n_samples=N, max_iters=60)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg, seed_mode=snk.SEED_LATTICE, kernel_variant=3)
    P.evolve()
    torch.cuda.synchronize()
    g = P.cells_np()
    P.params = pipeline.params_for(cfg, seed_mode=snk.SEED_LATTICE, kernel_variant=1, cta_warps=1)
    P.evolve()
    torch.cuda.synchronize()
    assert P.cells_np().tobytes() == g.tobytes()


@pytest.mark.parametrize("N,W", [(1024, 4), (2048, 8), (1024, 1)])
def test_brick_fast_path_bit_identical_to_warp_kernel(gpu, N, W):
    """The default launch (brick kernel, f32x2 fast path, 8 samples per thread)
    against the warp kernel (scalar, global gathers): the same canonical tree
    and per-sample arithmetic, so the records are identical bytes."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(n_samples=N, max_iters=150)
    P, raw, p = _gpu_smooth_seeds(torch, snk, pipeline, cfg)
    P.evolve()
    torch.cuda.synchronize()
    a = P.cells_np()
    P.params = pipeline.params_for(cfg, kernel_variant=1, cta_warps=W)
    P.evolve()
    torch.cuda.synchronize()
    assert P.cells_np().tobytes() == a.tobytes()


def test_run_batch_equals_run(gpu):
    """snk_run_batch (uploads / downloads overlapped with the kernels on internal
    streams, double-buffered) gives, volume by volume, the bytes of snk_run."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C1"].with_(max_iters=80)
    p = pipeline.params_for(cfg)
    raws = [torch.from_numpy(synth.generate(cfg.with_(gen_seed=cfg.gen_seed + i))).pin_memory() for i in range(3)]
    hr = pipeline.HostRunner(3, cfg.n, p)
    exp = []
    for r in raws:
        nd = hr.run(r)
        exp.append((hr.dets_np(nd).tobytes(), hr.h_labels.numpy().copy()))
    br = pipeline.BatchRunner(3, cfg.n, p, max_cells=hr.max_cells)
    seq = [raws[0], raws[1], raws[2], raws[1]]
    nds = br.run(seq)
    assert len(nds) == 4
    # slots alternate: volume 2 -> slot 0, volume 3 (= raws[1]) -> slot 1
    assert br.dets_np(0, nds[2]).tobytes() == exp[2][0] and np.array_equal(br.h_labels[0].numpy(), exp[2][1])
    assert br.dets_np(1, nds[3]).tobytes() == exp[1][0] and np.array_equal(br.h_labels[1].numpy(), exp[1][1])
    assert nds[0] == len(exp[0][0]) // snk.CELL_BYTES and nds[1] == len(exp[1][0]) // snk.CELL_BYTES


def test_run_batch_resampled_and_periodic(gpu):
    """snk_run_batch with an anisotropic (resampled) volume and periodic culling:
    the raw buffer is recycled only after a1/a2 consumed it; results equal snk_run."""
    torch, snk, pipeline = gpu
    c3 = synth.CONFIGS["C3"]
    base = synth.generate(c3)
    raws = [torch.from_numpy(np.ascontiguousarray(base[8 * i:8 * i + 24, 100:164, 64:128])).pin_memory()
            for i in range(3)]
    n = (64, 64, 24)
    cfg = c3.with_(n=n, max_iters=60)
    p = pipeline.params_for(cfg, cull_every=20)
    hr = pipeline.HostRunner(3, n, p, spacing=c3.spacing)
    exp = []
    for r in raws:
        nd = hr.run(r)
        exp.append((hr.dets_np(nd).tobytes(), hr.h_labels.numpy().copy()))
    br = pipeline.BatchRunner(3, n, p, spacing=c3.spacing, max_cells=hr.max_cells)
    nds = br.run(raws)
    # the last two volumes are still in the two result slots
    assert br.dets_np(0, nds[2]).tobytes() == exp[2][0] and np.array_equal(br.h_labels[0].numpy(), exp[2][1])
    assert br.dets_np(1, nds[1]).tobytes() == exp[1][0] and np.array_equal(br.h_labels[1].numpy(), exp[1][1])
    assert nds[0] * snk.CELL_BYTES == len(exp[0][0])
