"""The z-slab driver (paper_1804_06304_b200.dist) with the real kernels: world
sizes 2 and 3 as processes sharing one GPU (gloo, host-staged exchanges — the
round's GPU box has one device; NCCL runs the same code on 8).  Seeds, cells,
detections and the label map must be bit-identical to the single-GPU pipeline
(DESIGN.md §7)."""
import json
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

CFG = synth.Config(name="slab", dim=3, n=(48, 40, 150), count=(2, 2, 6), pitch=(24.0, 20.0, 25.0),
                   jitter=2.0, rbar=(5.0, 6.5), bg_wavelength=64.0, r0=7.0, n_samples=128,
                   max_iters=40, seed_window=3, gen_seed=77, philox_seed=991)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, k=0):
    import torch
    import torch.distributed as tdist
    from paper_1804_06304_b200 import dist as D, pipeline, snk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = pipeline.params_for(CFG, image_term=snk.IMAGE_INTENSITY, cull_every=k)
        plan = D.plan_slabs(CFG.n, world, rank, p)
        raw = synth.generate(CFG)
        own = torch.from_numpy(raw[plan.own[0]:plan.own[1]].copy()).cuda()
        be = D.CudaBackend(plan, p, max_cells=4096)
        r = D.SlabRun(plan, be, torch.device("cuda", 0), cull_every=k, max_iters=CFG.max_iters).step(own)
        torch.cuda.synchronize()
        ns, nd, nl = r["n_seeds"], r["n_dets"], r["n_live"]
        q.put((rank, {"seeds": r["seeds"][:ns].cpu().numpy(), "cells": r["cells"][:nl * 64].cpu().numpy(),
                      "dets": r["dets"][:nd * 64].cpu().numpy(), "labels": r["labels"].cpu().numpy(),
                      "id_base": r["id_base"], "n_total": r["n_total"]}))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        tdist.destroy_process_group()


@pytest.fixture(scope="module")
def single(gpu):
    torch, snk, pipeline = gpu
    p = pipeline.params_for(CFG, image_term=snk.IMAGE_INTENSITY)
    P = pipeline.Pipeline(3, CFG.n, p, gradmag=False)
    P.upload(synth.generate(CFG))
    res = P.step()
    torch.cuda.synchronize()
    return {"seeds": P.seeds[:res.n_seeds].cpu().numpy(), "cells": P.cells[:res.n_seeds * 64].cpu().numpy(),
            "dets": P.dets[:res.n_dets * 64].cpu().numpy(), "labels": P.labels.cpu().numpy()}


@pytest.mark.parametrize("world", [2, 3])
def test_slabs_match_single_gpu(single, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    assert out[0]["n_total"] == len(single["seeds"])
    assert np.array_equal(np.concatenate([out[r]["seeds"] for r in range(world)]), single["seeds"])
    assert np.array_equal(np.concatenate([out[r]["cells"] for r in range(world)]), single["cells"])
    for r in range(world):
        assert np.array_equal(out[r]["dets"], single["dets"])
    assert np.array_equal(np.concatenate([out[r]["labels"] for r in range(world)]), single["labels"])


@pytest.fixture(scope="module")
def single_periodic(gpu):
    torch, snk, pipeline = gpu
    p = pipeline.params_for(CFG, image_term=snk.IMAGE_INTENSITY, cull_every=15)
    P = pipeline.Pipeline(3, CFG.n, p, gradmag=False)
    P.upload(synth.generate(CFG))
    res = P.step()
    torch.cuda.synchronize()
    return {"cells": P.cells_np(), "dets": P.dets[:res.n_dets * 64].cpu().numpy(),
            "labels": P.labels.cpu().numpy(), "n_seeds": res.n_seeds}


def test_slabs_periodic_culling_match_single_gpu(single_periodic):
    """Periodic culling (G25) with the N6 checkpoint exchange on 2 ranks: the
    live cells (as a set), the detections and the label map equal one GPU's."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, 15)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for pr in procs:
        pr.join(timeout=120)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    from paper_1804_06304_b200 import snk
    got = np.concatenate([out[r]["cells"] for r in range(world)]).view(snk.CELL_DTYPE)
    exp = single_periodic["cells"]
    assert len(exp) < single_periodic["n_seeds"]
    assert got[np.argsort(got["id"])].tobytes() == exp[np.argsort(exp["id"])].tobytes()
    for r in range(world):
        assert np.array_equal(out[r]["dets"], single_periodic["dets"])
    assert np.array_equal(np.concatenate([out[r]["labels"] for r in range(world)]), single_periodic["labels"])


def _nccl_world1(q):
    import torch
    import torch.distributed as tdist
    from paper_1804_06304_b200 import dist as D, pipeline, snk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), NCCL_DEBUG="INFO",
                      NCCL_DEBUG_SUBSYS="INIT")
    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = pipeline.params_for(CFG, image_term=snk.IMAGE_INTENSITY)
        plan = D.plan_slabs(CFG.n, 1, 0, p)
        own = torch.from_numpy(synth.generate(CFG)).cuda()
        be = D.CudaBackend(plan, p, max_cells=4096, gradmag=False)
        r = D.SlabRun(plan, be, torch.device("cuda", 0), max_iters=CFG.max_iters).step(own)
        torch.cuda.synchronize()
        ns, nd = r["n_seeds"], r["n_dets"]
        q.put({"backend": tdist.get_backend(), "seeds": r["seeds"][:ns].cpu().numpy(),
               "cells": r["cells"][:ns * 64].cpu().numpy(), "dets": r["dets"][:nd * 64].cpu().numpy(),
               "labels": r["labels"].cpu().numpy()})
    except Exception as e:
        q.put(repr(e))
        raise
    finally:
        tdist.destroy_process_group()


def test_nccl_world_of_one_matches_single_gpu(single):
    """The driver's NCCL branch (the N2 / N3 all_gathers through NCCL on device
    buffers) on the one GPU of this box: bit-identical to the pipeline."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_world1, args=(q,))
    pr.start()
    out = q.get(timeout=600)
    pr.join(timeout=120)
    assert not isinstance(out, str), out
    assert out["backend"] == "nccl"
    for k in ("seeds", "cells", "dets", "labels"):
        assert np.array_equal(out[k], single[k]), k


def _bench(args, env=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                       env=e, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line), r.stdout, r.stderr


def test_bench_launches_ranks_itself(gpu):
    """`bench.py --gpus 2` without a launcher starts two ranks (torch.distributed.run);
    here they share the box's one GPU (gloo, host-staged exchanges) and find the
    same cells and detections as one GPU; `--dist` runs the driver's NCCL branch
    at N = 1."""
    common = ["--config", "C1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"]
    one, _, _ = _bench(common + ["--no-e2e"])
    two, _, _ = _bench(["--gpus", "2"] + common, {"SNK_DIST_BACKEND": "gloo"})
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["cells"] == one["cells"]
    assert two["detections"] == one["detections"]
    nc, out, err = _bench(["--dist"] + common)
    assert nc["n_gpus"] == 1 and nc["backend"] == "nccl"
    assert nc["detections"] == one["detections"]
    # NCCL's communicator lines are kept, on stderr: stdout is the one JSON line
    assert "NCCL INFO" in err
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1 and json.loads(lines[0]) == nc, out[-2000:]
