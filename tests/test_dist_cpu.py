"""Multi-rank z-slab decomposition (paper_1804_06304_b200.dist) on CPU with gloo,
world_size 2 and 3: the driver's partition, halo exchange (N1), id prefix (N2)
and candidate all_gather (N3) give seeds, cells, detections and labels that
are bit-identical to a single-process run.  The per-stage
compute is the CPU oracle here (test-only backend); on GPUs it is libsnk."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1804_06304_b200 import dist as D

REC = np.dtype([("c", "<f4", 3), ("R", "<f4"), ("seed", "<f4", 3), ("energy", "<f4"),
                ("flags", "<u4"), ("iters", "<i4"), ("id", "<i8"), ("disp", "<f4", 3), ("reserved", "<u4")])
CFG = synth.Config(name="slab", dim=3, n=(48, 40, 150), count=(2, 2, 6), pitch=(24.0, 20.0, 25.0),
                   jitter=2.0, rbar=(5.0, 6.5), bg_wavelength=64.0, r0=7.0, n_samples=64,
                   max_iters=40, seed_window=3, gen_seed=77, philox_seed=991)


class P:   # the fields the planner reads (mirrors snk_params)
    leash, r_max, delta_R, sigma, seed_window = 5.0, 10.0, 2.0, 1.0, 3


def _to_rec(cells):
    r = np.zeros(len(cells), REC)
    r["c"], r["R"], r["seed"] = cells["c"], cells["R"], cells["seed"]
    r["energy"], r["flags"], r["iters"], r["id"] = cells["E"], cells["flags"], cells["iters"], cells["id"]
    r["disp"] = (cells["c"] - cells["seed"]).astype(np.float32)
    return r


def _params():
    return oracle.Params(r0=CFG.r0, n_samples=CFG.n_samples, max_iters=CFG.max_iters, leash=P.leash,
                         r_max=P.r_max, seed=CFG.philox_seed)


class OracleBackend:
    """Test-only stage implementation on the CPU oracle (numpy <-> torch bytes)."""

    def preprocess(self, pl, local):
        return oracle.blur(local.numpy(), 3, 1.0)

    def seeds(self, pl, B):
        n = pl.n
        s = oracle.seeds_maxima(B, 3, P.seed_window, CFG.seed_threshold, org=(0, 0, pl.buf[0]),
                                n_global=n, lo=(0, 0, pl.own[0]), hi=(n[0] - 1, n[1] - 1, pl.own[1] - 1))
        return s, len(s)

    def evolve(self, pl, B, seeds, n, id_base):
        cells = oracle.evolve(B, _params(), seeds, ids=id_base + np.arange(n), org=(0, 0, pl.buf[0]),
                              n_global=pl.n)
        return torch.from_numpy(_to_rec(cells).view(np.uint8).copy())

    def init_cells(self, pl, seeds, n, id_base):
        return torch.from_numpy(_to_rec(oracle.init_cells(_params(), seeds, ids=id_base + np.arange(n)))
                                .view(np.uint8).copy())

    def evolve_range(self, pl, B, cells, n, it0, it1):
        r = cells.numpy().view(REC)[:n]
        o = np.zeros(n, oracle.CELL_DTYPE)
        o["c"], o["R"], o["E"], o["seed"] = r["c"], r["R"], r["energy"], r["seed"]
        o["flags"], o["iters"], o["id"] = r["flags"], r["iters"], r["id"]
        o = oracle.evolve_range(B, _params(), o, it0, it1, org=(0, 0, pl.buf[0]), n_global=pl.n)
        return torch.from_numpy(_to_rec(o).view(np.uint8).copy())

    def select_ids(self, recs, n, lo, hi):
        r = recs.numpy().view(REC)[:n]
        keep = r[(r["id"] >= lo) & (r["id"] < hi)]
        return torch.from_numpy(keep.view(np.uint8).copy()), len(keep)

    def compact(self, cells, n):
        r = cells.numpy().view(REC)[:n]
        keep = r[(r["energy"] <= -3.0) & ((r["flags"] & (oracle.COLLAPSED | oracle.RMAX)) == 0)]
        return torch.from_numpy(keep.view(np.uint8).copy()), len(keep)

    def cull(self, pl, allc, ntot):
        r = allc.numpy().view(REC)[:ntot]
        k = oracle.cull(r["c"], r["R"], r["energy"], r["flags"], r["id"], 3, -3.0)
        return torch.from_numpy(r[k].view(np.uint8).copy()), len(k)

    def label(self, pl, dets, nd):
        r = dets.numpy().view(REC)[:nd]
        return oracle.label(pl.n, 3, r["c"], r["R"], z0=pl.own[0], nz=pl.own[1] - pl.own[0])


def _worker(rank, world, port, q, k=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        raw = synth.generate(CFG)
        plan = D.plan_slabs(CFG.n, world, rank, P)
        own = torch.from_numpy(raw[plan.own[0]:plan.own[1]].copy())
        out = D.SlabRun(plan, OracleBackend(), torch.device("cpu"), cull_every=k,
                        max_iters=CFG.max_iters).step(own)
        # the halo exchange reproduced exactly the planes of the full volume
        local = D.exchange_halo(plan, own)
        assert np.array_equal(local.numpy(), raw[plan.buf[0]:plan.buf[1]])
        q.put((rank, out["seeds"], out["cells"].numpy()[: out["n_live"] * 64].copy(),
               out["dets"].numpy()[: out["n_dets"] * 64].copy(), out["labels"], out["id_base"]))
    finally:
        tdist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_slabs_bit_identical_to_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process reference
    raw = synth.generate(CFG)
    B = oracle.blur(raw, 3, 1.0)
    seeds = oracle.seeds_maxima(B, 3, P.seed_window, CFG.seed_threshold)
    cells = _to_rec(oracle.evolve(B, _params(), seeds))
    cand = cells[(cells["energy"] <= -3.0) & ((cells["flags"] & (oracle.COLLAPSED | oracle.RMAX)) == 0)]
    k = oracle.cull(cand["c"], cand["R"], cand["energy"], cand["flags"], cand["id"], 3, -3.0)
    dets = cand[k]
    labels = oracle.label(CFG.n, 3, dets["c"], dets["R"])
    assert len(seeds) > 10 and len(dets) > 5
    assert np.array_equal(np.concatenate([r[1] for r in res]), seeds)
    assert np.concatenate([r[2] for r in res]).tobytes() == cells.tobytes()
    for r in res:
        assert r[3].tobytes() == dets.tobytes()          # every rank has the same detections
    assert np.array_equal(np.concatenate([r[4] for r in res]), labels)
    assert [r[5] for r in res] == list(np.cumsum([0] + [len(r[1]) for r in res[:-1]]))


def test_plan_covers_reach():
    for world in (1, 2, 4, 8):
        for r in range(world):
            pl = D.plan_slabs((2048, 2048, 512), world, r, type("p", (), dict(
                leash=26.0, r_max=26.0, delta_R=2.0, sigma=1.0, seed_window=5))())
            z0, z1 = pl.own
            assert pl.halo == 55 and pl.blur == 4
            assert pl.buf[0] == max(z0 - 59, 0) and pl.buf[1] == min(z1 + 59, 512)
    assert sum(D.slab_bounds(512, 8, r)[1] - D.slab_bounds(512, 8, r)[0] for r in range(8)) == 512
    assert [D.slab_bounds(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]


def test_slabs_periodic_culling_bit_identical():
    """Periodic culling (G25) on 2 ranks: the N6 checkpoint exchange + the same
    deterministic cull on every rank + ownership by id range give the live cells,
    detections and labels of a single-process run of the same segments."""
    k, world = 15, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, k)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    raw = synth.generate(CFG)
    B = oracle.blur(raw, 3, 1.0)
    seeds = oracle.seeds_maxima(B, 3, P.seed_window, CFG.seed_threshold)
    be, pl = OracleBackend(), D.plan_slabs(CFG.n, 1, 0, P)
    cells, live = be.init_cells(pl, seeds, len(seeds), 0), len(seeds)
    segs = D.checkpoints(CFG.max_iters, k)
    assert segs == [(1, 15), (16, 30), (31, 41)]
    for i, (a, b) in enumerate(segs):
        cells = be.evolve_range(pl, B, cells, live, a, b)
        if i + 1 < len(segs):
            cand, nc = be.compact(cells, live)
            cells, live = be.cull(pl, cand, nc)
    cells = cells.numpy().view(REC)[:live]
    cells = cells[np.argsort(cells["id"], kind="stable")]
    cand = cells[(cells["energy"] <= -3.0) & ((cells["flags"] & (oracle.COLLAPSED | oracle.RMAX)) == 0)]
    kk = oracle.cull(cand["c"], cand["R"], cand["energy"], cand["flags"], cand["id"], 3, -3.0)
    dets = cand[kk]
    labels = oracle.label(CFG.n, 3, dets["c"], dets["R"])
    assert len(seeds) > live > 5 and len(dets) > 5
    got = np.concatenate([r[2] for r in res]).view(REC)
    got = got[np.argsort(got["id"], kind="stable")]
    assert got.tobytes() == cells.tobytes()
    for r in res:
        assert r[3].tobytes() == dets.tobytes()
    assert np.array_equal(np.concatenate([r[4] for r in res]), labels)
