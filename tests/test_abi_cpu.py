"""The C-ABI library builds, loads and exports every symbol include/snk.h
declares; host-only validation and sizing behave as documented.  No device
work is issued (these run on CPU-only machines)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def snk():
    from paper_1804_06304_b200 import build
    build.build()
    from paper_1804_06304_b200 import snk as mod
    return mod


def test_exports_every_declared_symbol(snk):
    declared = snk.declared_symbols()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", snk.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(snk, s), f"binding lacks {s}"


def test_library_is_sm100a_only(snk):
    out = subprocess.run(["cuobjdump", "--list-elf", snk.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_struct_layouts(snk):
    assert C.sizeof(snk.snk_cell) == 64
    assert C.sizeof(snk.snk_grid) == 88                 # static_assert-ed in abi.cu too
    assert C.sizeof(snk.snk_params) == 136
    assert snk.snk_abi_version() == 5
    assert snk.status_string(0) == "ok" and snk.status_string(6) == "capacity exceeded"


def test_validation_errors(snk):
    g = snk.make_grid(3, (64, 64, 64))
    p = snk.make_params(10.0)
    assert snk.snk_validate(g, p) == snk.OK
    bad = snk.make_params(10.0, e0=1.0)                   # e0 <= 0
    assert snk.snk_validate(g, bad) == snk.CONFIG and "e0" in snk.snk_last_error()
    assert snk.snk_validate(g, snk.make_params(10.0, n_samples=1000)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, max_iters=0)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, r_min=20.0)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, cta_warps=3)) == snk.CONFIG
    assert snk.snk_validate(snk.make_grid(3, (64, 64, 1)), p) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(2, (64, 64, 2)), p) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(3, (64, 64, 64), z_lo=10, nz_buf=60), p) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(3, (64, 64, 64), own=(0, 70)), p) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(2, (64, 64, 1)), p) == snk.OK


def test_validation_of_round_one_features(snk):
    """Estimators, periodic culling and anisotropic grids (G25-G28): host-side checks."""
    g = snk.make_grid(3, (64, 64, 64))
    for e in (snk.EST_MC, snk.EST_GRID, snk.EST_MC_CV, snk.EST_RAY):
        assert snk.snk_validate(g, snk.make_params(10.0, estimator=e)) == snk.OK
    assert snk.snk_validate(g, snk.make_params(10.0, estimator=4)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, estimator=snk.EST_GRID, kernel_variant=1)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, cull_every=-1)) == snk.CONFIG
    assert snk.snk_validate(g, snk.make_params(10.0, cull_every=50)) == snk.OK
    ga = snk.make_grid(3, (64, 64, 32), scale=(1.0, 1.0, 2.0))
    assert snk.snk_validate(ga, snk.make_params(10.0)) == snk.OK
    assert snk.snk_validate(ga, snk.make_params(10.0, estimator=snk.EST_GRID)) == snk.CONFIG
    assert snk.snk_validate(ga, snk.make_params(10.0, image_term=snk.IMAGE_GRADMAG)) == snk.CONFIG
    assert snk.snk_validate(snk.make_grid(3, (60, 64, 32), scale=(1.0, 1.0, 2.0)), snk.make_params(10.0)) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(3, (64, 64, 32), scale=(1.0, -1.0, 2.0)), snk.make_params(10.0)) == snk.SHAPE
    assert snk.snk_validate(snk.make_grid(3, (60, 64, 32), scale=(0.0, 0.0, 0.0)), snk.make_params(10.0)) == snk.OK
    # the periodic-culling segments: the binding's list equals the driver's
    from paper_1804_06304_b200 import dist
    def c_loop(T, k):   # transcription of snk_run's segment loop (abi.cu), computed on the fly
        if not (0 < k < T):
            return [(1, T + 1)]
        out, a = [], 1
        while a <= T + 1:
            e = a + k - 1 if a + k - 1 < T else T + 1
            out.append((a, e))
            a = e + 1
        return out

    for T, k in ((400, 50), (400, 0), (400, 400), (40, 15), (7, 3), (1, 1), (5000, 1), (9000, 2)):
        assert snk.checkpoints(T, k) == dist.checkpoints(T, k) == c_loop(T, k)
        segs = snk.checkpoints(T, k)
        assert segs[0][0] == 1 and segs[-1][1] == T + 1
        assert all(b + 1 == a for (_, b), (a, _) in zip(segs, segs[1:]))


def test_workspace_and_resample_dims(snk):
    import oracle
    for n, sp in [((512, 512, 128), (1, 1, 2)), ((4, 4, 4), (0.5, 0.5, 1.0)), ((30, 20, 10), (3, 1.5, 1)),
                  ((64, 64, 64), (1, 1, 1))]:
        assert tuple(snk.snk_resample_dims(3, n, sp)) == tuple(oracle.resample_dims(n, sp, 3))
    g = snk.make_grid(3, (512, 512, 256))
    p = snk.make_params(11.0, seed_window=4)
    ws = snk.snk_workspace_bytes(g, p, 100_000)
    assert ws >= 2 * 512 * 512 * 256 * 2          # box-max ping-pong volumes
    assert snk.snk_run_workspace_bytes(3, (512, 512, 128), (1, 1, 2), p, 100_000) > ws


def test_product_path_has_no_oracle_dependency():
    """The CUDA package never imports or loads the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_1804_06304_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f
