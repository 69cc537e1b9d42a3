"""Parity at BASELINE sizes (VERDICT r1 "next" 1b-1d): the CUDA path against
the fp64 oracle on C4 (2048x2048x512, 359k cells), C3 and C2 in full, in the
launch configuration bench.py times.

* C4 stage by stage: the whole blurred volume and the whole seed list
  bit-exact; the id = 0 mod 100 subset evolved by the oracle
  within the north_star tolerance; the oracle's cull of all 359k GPU records
  bit-exact; labels bit-exact on 16 full 64^3 boxes, 10^5 random voxels and
  a neighbourhood voxel of every detection.
* C3 (resampled) and C2 (2D) end to end against the oracle's own run: every
  cell within tolerance, and every differing detection / label voxel counted
  and attributed to a near-tie (SURVEY §8(c) parity contract, a7-a8 end to
  end).  A C4 crop (256x256x128) end to end likewise.

Label checks at this size evaluate the oracle's O7 rule per spatial bin with
the detections whose inner ball can reach the bin: a detection that cannot
contain a voxel has d^2 > thr there and can never be its label (O7), so the
result is the oracle's over all detections.  10^5 random voxels are also
checked against the oracle with every detection, unbinned.
"""
import numpy as np
import pytest
from scipy.spatial import cKDTree

import oracle
import synth



TOL = 1e-3
RHO = {3: 2.0 ** (-1.0 / 3.0), 2: 2.0 ** (-0.5)}


def _t(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _ora_params(cfg, **kw):
    d = dict(r0=cfg.r0, n_samples=cfg.n_samples, max_iters=cfg.max_iters, dim=cfg.dim, seed=cfg.philox_seed)
    d.update(kw)
    return oracle.Params(**d)


def _close(g, o, ctx):
    """GPU records vs oracle cells (same order): ids, seeds equal; c, R within
    TOL voxel, E within TOL max(1, |E|).  Returns (max dR, max dc)."""
    assert len(g) == len(o), ctx
    assert np.array_equal(g["id"], o["id"]), ctx
    assert np.array_equal(g["seed"].astype(np.float64), o["seed"]), ctx
    dR = np.abs(g["R"].astype(np.float64) - o["R"])
    dc = np.abs(g["c"].astype(np.float64) - o["c"]).max(axis=1)
    dE = np.abs(g["energy"].astype(np.float64) - o["E"]) / np.maximum(1.0, np.abs(o["E"]))
    bad = np.nonzero((dR > TOL) | (dc > TOL) | (dE > TOL))[0]
    assert len(bad) == 0, (f"{ctx}: {len(bad)}/{len(g)} cells out of tolerance; worst dR={dR.max():.3g} "
                           f"dc={dc.max():.3g} dE={dE.max():.3g}")
    dEa = np.abs(g["energy"].astype(np.float64) - o["E"])
    print(f"{ctx}: {len(g)} cells, max|dR|={dR.max():.2e} max|dc|={dc.max():.2e} max|dE|rel={dE.max():.2e}")
    return float(dR.max()), float(dc.max()), float(dEa.max())


def oracle_labels_binned(dim, pts, c, R, bin_=64):
    """O7 labels (index + 1 into c/R, or 0) at integer points (x, y, z)."""
    pts = np.ascontiguousarray(pts, np.int64).reshape(-1, 3)
    c = np.ascontiguousarray(c, np.float32).reshape(-1, 3)
    R = np.ascontiguousarray(R, np.float32)
    out = np.zeros(len(pts), np.int32)
    if len(R) == 0 or len(pts) == 0:
        return out
    ext = RHO[dim] * R.astype(np.float64) * (1 + 1e-6) + 1.0
    assert ext.max() < bin_
    lo = np.floor((c - ext[:, None]) / bin_).astype(np.int64)
    hi = np.floor((c + ext[:, None]) / bin_).astype(np.int64)
    off = 1 << 20

    def key(b):
        return ((b[:, 2] + 2) * off + (b[:, 1] + 2)) * off + (b[:, 0] + 2)

    # (bin key, detection index) for every bin a detection's inner ball can reach (<= 2 per axis)
    pairs = []
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                b = lo + np.array([dx, dy, dz])
                ok = np.all(b <= hi, axis=1)
                idx = np.nonzero(ok)[0]
                pairs.append(np.stack([key(b[idx]), idx], axis=1))
    pairs = np.concatenate(pairs)
    pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
    pk = key(pts // bin_)
    order = np.argsort(pk, kind="stable")
    ukeys, starts = np.unique(pk[order], return_index=True)
    ends = np.append(starts[1:], len(order))
    dstart = np.searchsorted(pairs[:, 0], ukeys, side="left")
    dend = np.searchsorted(pairs[:, 0], ukeys, side="right")
    for k in range(len(ukeys)):
        sel = pairs[dstart[k]:dend[k], 1]          # ascending detection index (tie rule order kept)
        if len(sel) == 0:
            continue
        pi = order[starts[k]:ends[k]]
        lab = oracle.label_points(dim, pts[pi], c[sel], R[sel])
        out[pi] = np.where(lab > 0, sel[np.maximum(lab - 1, 0)] + 1, 0)
    return out


def gpu_labels_at(torch, labels, pts):
    p = torch.from_numpy(np.ascontiguousarray(pts, np.int64)).cuda()
    if labels.dim() == 3:
        return labels[p[:, 2], p[:, 1], p[:, 0]].cpu().numpy()
    return labels[p[:, 1], p[:, 0]].cpu().numpy()


def neighbourhood_points(dets, n, dim, rng):
    """Per detection: the voxel nearest its centre and one just inside / outside
    its inner ball along a random axis direction."""
    c = dets["c"].astype(np.float64)
    r = RHO[dim] * dets["R"].astype(np.float64)
    ax = rng.integers(0, dim, len(c))
    sgn = rng.choice([-1.0, 1.0], len(c))
    pts = [np.rint(c)]
    for dr in (-0.6, 0.4):
        q = c.copy()
        q[np.arange(len(c)), ax] += sgn * (r + dr)
        pts.append(np.rint(q))
    pts = np.concatenate(pts).astype(np.int64)
    hi = np.asarray(n, np.int64) - 1
    return np.clip(pts, 0, hi)


def attribute_detections(g, o, gkeep, okeep, dim, e0, delta, etol):
    """Every id kept by exactly one side must be explained by a near-tie
    (SURVEY §8(c)): |E - E0| < etol on either side; or a competitor overlapping
    it (within delta) whose energy is within etol of its own; or (cascade) it
    overlaps another differing cell that is explained.  etol = max(1e-3, twice
    the observed |E_gpu - E_oracle|): E is compared to 1e-3 max(1, |E|), so two
    energies can swap order within that band.  Returns (n_diff, unexplained ids)."""
    ids = g["id"]
    assert np.array_equal(ids, o["id"])
    gk = np.zeros(len(g), bool)
    gk[gkeep] = True
    ok_ = np.zeros(len(o), bool)
    ok_[okeep] = True
    diff = np.nonzero(gk != ok_)[0]
    if len(diff) == 0:
        return 0, []
    Eg, Eo = g["energy"].astype(np.float64), o["E"]
    c = g["c"].astype(np.float64)
    R = np.maximum(g["R"].astype(np.float64), o["R"])
    tree = cKDTree(c)
    rmax = RHO[dim] * R.max() + delta + 1e-6
    expl = {}
    for i in diff:
        if abs(Eg[i] - e0) < etol or abs(Eo[i] - e0) < etol:
            expl[i] = "E0"
    nb = {i: [j for j in tree.query_ball_point(c[i], rmax) if j != i and
              np.linalg.norm(c[i] - c[j]) <= RHO[dim] * max(R[i], R[j]) + delta] for i in diff}
    for i in diff:
        if i in expl:
            continue
        for j in nb[i]:
            if abs(Eg[i] - Eg[j]) < etol or abs(Eo[i] - Eo[j]) < etol:
                expl[i] = "E tie"
                break
    changed = True
    dset = set(diff.tolist())
    while changed:
        changed = False
        for i in diff:
            if i not in expl and any(j in expl and j in dset for j in nb[i]):
                expl[i] = "cascade"
                changed = True
    un = [int(ids[i]) for i in diff if i not in expl]
    kinds = {k: sum(1 for v in expl.values() if v == k) for k in ("E0", "E tie", "cascade")}
    print(f"detection differences: {len(diff)} ({kinds}), unexplained {len(un)}")
    return len(diff), un


def attribute_labels(pts, lg, lo, gd, od, dim, delta):
    """Every voxel whose GPU label differs from the oracle's end-to-end label
    must lie within delta of an inner-ball boundary of a detection of either
    run, or inside a detection kept by only one run (G19, O7)."""
    bad = np.nonzero(lg != lo)[0]
    if len(bad) == 0:
        return 0, 0
    gset = set(gd["id"].tolist())
    oset = set(od["id"].tolist())
    cen = np.concatenate([gd["c"].astype(np.float64), od["c"].astype(np.float64)])
    rad = RHO[dim] * np.concatenate([gd["R"].astype(np.float64), od["R"].astype(np.float64)])
    only = np.array([i not in oset for i in gd["id"]] + [i not in gset for i in od["id"]])
    tree = cKDTree(cen)
    un = 0
    for k in bad:
        x = pts[k].astype(np.float64)
        js = tree.query_ball_point(x, rad.max() + delta + 1.0)
        ok = False
        for j in js:
            d = np.linalg.norm(x - cen[j])
            if abs(d - rad[j]) <= delta or (only[j] and d <= rad[j] + delta):
                ok = True
                break
        un += not ok
    print(f"label differences: {len(bad)} of {len(pts)} voxels, unexplained {un}")
    return len(bad), un


def _delta(dR, dc, dim):
    # the observed per-cell discrepancy, as a distance: centre offset + rho dR (+ rounding)
    return float(np.sqrt(dim) * dc + RHO[dim] * dR + 1e-6)


def _run_gpu(torch, pipeline, cfg, raw, **over):
    p = pipeline.params_for(cfg, **over)
    P = pipeline.Pipeline(cfg.dim, cfg.n, p, spacing=cfg.spacing)
    P.upload(raw)
    r = P.step()
    torch.cuda.synchronize()
    return P, r


# ---------------------------------------------------------------------------- C4


@pytest.mark.gpu
def test_c4_full_size_stagewise(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C4"]
    raw = synth.generate(cfg)
    P, r = _run_gpu(torch, pipeline, cfg, raw)
    n = P.n_iso
    # a2: the whole 2048 x 2048 x 512 smoothed volume
    B = oracle.blur(raw, 3, 1.0)
    assert np.array_equal(P.smooth.cpu().numpy(), B)
    # a4: the whole seed list (359k maxima, linear-index order)
    exp = oracle.seeds_maxima(B, 3, cfg.window, cfg.seed_threshold)
    assert P.n_seeds == len(exp) > 300_000
    assert np.array_equal(P.seeds_np(), exp)
    del raw
    # a5/a6: the 1% subset id = 0 mod 100, evolved by the oracle on the full volume
    cells = P.cells_np()
    assert len(cells) == P.n_seeds and np.array_equal(cells["id"], np.arange(P.n_seeds))
    sub = np.nonzero(cells["id"] % 100 == 0)[0]
    o = oracle.evolve(B, _ora_params(cfg), exp[sub], ids=cells["id"][sub])
    _close(cells[sub], o, "C4 1% subset")
    del B
    # a7: the oracle's cull of every GPU record
    keep = oracle.cull(cells["c"], cells["R"], cells["energy"], cells["flags"], cells["id"], 3, -3.0)
    dets = P.dets_np()
    assert len(dets) == len(keep) > 150_000
    assert dets.tobytes() == cells[keep].tobytes()
    # a8: 16 whole 64^3 boxes, 10^5 random voxels, 3 neighbourhood voxels per detection
    rng = np.random.default_rng(44)
    boxes = []
    for _ in range(16):
        o0 = np.array([rng.integers(0, n[a] - 64) for a in range(3)])
        z, y, x = np.meshgrid(*(np.arange(o0[a], o0[a] + 64) for a in (2, 1, 0)), indexing="ij")
        boxes.append(np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1))
    pts = np.concatenate(boxes + [neighbourhood_points(dets, n, 3, rng)])
    got = gpu_labels_at(torch, P.labels, pts)
    exp_l = oracle_labels_binned(3, pts, dets["c"], dets["R"])
    assert np.array_equal(got, exp_l), f"{int((got != exp_l).sum())} label voxels differ"
    assert (got > 0).mean() > 0.1
    rnd = np.stack([rng.integers(0, n[a], 100_000) for a in range(3)], axis=1)
    assert np.array_equal(gpu_labels_at(torch, P.labels, rnd),
                          oracle.label_points(3, rnd, dets["c"], dets["R"]))


@pytest.mark.gpu
def test_c4_crop_end_to_end(gpu):
    """A 256 x 256 x 128 crop of C4 as a volume of its own, GPU vs the oracle's
    own end-to-end run, differences attributed."""
    torch, snk, pipeline = gpu
    full = synth.CONFIGS["C4"]
    raw = np.ascontiguousarray(synth.generate(full, 200, 328)[:, 900:1156, 700:956])
    cfg = full.with_(n=(256, 256, 128))
    P, r = _run_gpu(torch, pipeline, cfg, raw)
    _end_to_end(torch, P, cfg, raw, "C4 crop")


# ---------------------------------------------------------------------------- C3, C2


@pytest.mark.gpu
def test_c3_end_to_end(gpu):
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C3"]
    raw = synth.generate(cfg)
    P, r = _run_gpu(torch, pipeline, cfg, raw)
    _end_to_end(torch, P, cfg, raw, "C3")


@pytest.mark.gpu
def test_c2_full_size(gpu):
    """C2 (2D 2048^2) in full: every cell within tolerance, the cull and the whole
    label map bit-exact given the GPU cells, and end to end with attribution."""
    torch, snk, pipeline = gpu
    cfg = synth.CONFIGS["C2"]
    raw = synth.generate(cfg)
    P, r = _run_gpu(torch, pipeline, cfg, raw)
    cells = P.cells_np()
    keep = oracle.cull(cells["c"], cells["R"], cells["energy"], cells["flags"], cells["id"], 2, -3.0)
    dets = P.dets_np()
    assert dets.tobytes() == cells[keep].tobytes()
    lab = oracle.label(P.n_iso, 2, dets["c"], dets["R"])
    assert np.array_equal(P.labels.cpu().numpy().reshape(lab.shape), lab)
    _end_to_end(torch, P, cfg, raw, "C2")


def _end_to_end(torch, P, cfg, raw, ctx):
    dim = cfg.dim
    vol = raw if raw.ndim == 3 else raw[None]
    iso = oracle.resample(vol, cfg.spacing, 3) if P.resample else vol
    if P.resample:
        assert np.array_equal(P.iso.cpu().numpy(), iso)
    B = oracle.blur(iso, dim, 1.0)
    assert np.array_equal(P.smooth.cpu().numpy().reshape(B.shape), B)
    seeds = oracle.seeds_maxima(B, dim, cfg.window, cfg.seed_threshold)
    assert np.array_equal(P.seeds_np(), seeds) and len(seeds) > 100
    o = oracle.evolve(B, _ora_params(cfg), seeds)
    g = P.cells_np()
    dR, dc, dE = _close(g, o, ctx)
    okeep = oracle.cull(o["c"].astype(np.float32), o["R"].astype(np.float32), o["E"].astype(np.float32),
                        o["flags"], o["id"], dim, -3.0)
    gkeep = oracle.cull(g["c"], g["R"], g["energy"], g["flags"], g["id"], dim, -3.0)
    gd = P.dets_np()
    assert gd.tobytes() == g[gkeep].tobytes()
    delta = _delta(dR, dc, dim)
    nd, un = attribute_detections(g, o, gkeep, okeep, dim, -3.0, delta, max(1e-3, 2 * dE))
    assert not un, f"{ctx}: unexplained detection differences {un[:10]}"
    # labels: the whole map (binned oracle) against the oracle's detections
    n = P.n_iso
    if dim == 3:
        z, y, x = np.meshgrid(np.arange(n[2]), np.arange(n[1]), np.arange(n[0]), indexing="ij")
        pts = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)
    else:
        y, x = np.meshgrid(np.arange(n[1]), np.arange(n[0]), indexing="ij")
        pts = np.stack([x.ravel(), y.ravel(), np.zeros(x.size, np.int64)], axis=1)
    od = o[okeep]
    lo = oracle_labels_binned(dim, pts, od["c"].astype(np.float32), od["R"].astype(np.float32))
    lg = P.labels.cpu().numpy().ravel()
    # GPU label indices -> ids, oracle indices -> ids (the two detection lists may differ)
    gid = np.where(lg > 0, gd["id"][np.maximum(lg - 1, 0)], -1)
    oid = np.where(lo > 0, od["id"][np.maximum(lo - 1, 0)], -1)
    nl, unl = attribute_labels(pts, gid, oid, gd, od, dim, delta)
    assert unl == 0, f"{ctx}: {unl} unexplained label differences"
    print(f"{ctx} end to end: {len(gd)} GPU / {len(od)} oracle detections, {nd} differ (all near-ties); "
          f"{nl} of {len(pts)} label voxels differ (all within delta = {delta:.2e} of a boundary)")
