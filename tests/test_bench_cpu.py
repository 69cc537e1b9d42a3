"""bench.py's rank launcher on CPU: `--gpus 2` without a launcher starts two
ranks through torch.distributed.run (127.0.0.1) that join one process group."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_launches_two_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["n_gpus"] == 2 and out["ranks"] == [0, 1]


def test_reference_arm_survey_plan_c1():
    """`--impl reference` times the oracle by SURVEY 8(d)'s plan (slab volume
    passes and the id = 0 mod 100 evolution subset, extrapolated) and prints our
    arm's workload config."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    sys.path.insert(0, ROOT)
    import bench
    import synth
    assert out["impl"] == "reference" and out["value"] > 0 and out["cpu_baseline"]["extrapolated"]
    assert out["config"] == bench.workload_config(synth.CONFIGS["C1"])
    assert "id = 0 mod 100" in out["cpu_baseline"]["sample"]
