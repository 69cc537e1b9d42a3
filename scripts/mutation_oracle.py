"""Mutation check of the oracle's pins (a nearest-neighbour mutant of
Image::interp passed every pin).  Each mutant of oracle/oracle.cpp is built in
a scratch copy of {oracle, synth, tests} and the CPU pins are run against it;
a mutant must make at least one pin fail.

    python scripts/mutation_oracle.py            # all mutants
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) — each original must occur exactly once
MUTANTS = [
    ("interp: nearest neighbour",
     "      f[a] = kc - (double)i0[a];\n",
     "      f[a] = std::floor(kc - (double)i0[a] + 0.5);\n"),
    ("interp: y lerp uses the x fraction",
     "    const double c0 = lerp(c00, c10, f[1]);\n",
     "    const double c0 = lerp(c00, c10, f[0]);\n"),
    ("interp: no i0 <= n - 2 rule",
     "      i0[a] = std::min((int64_t)std::floor(kc), n[a] - 2);\n",
     "      i0[a] = (int64_t)std::floor(kc);\n"),
    ("interp: no clamp to [0, n - 1]",
     "      const double kc = clampd(k[a], 0.0, (double)(n[a] - 1));\n",
     "      const double kc = k[a];\n"),
    ("interp: z lerp swapped operands",
     "    return iscale * lerp(c0, c1, f[2]);\n",
     "    return iscale * lerp(c1, c0, f[2]);\n"),
]

PINS = ["tests/test_oracle_interp.py", "tests/test_oracle_energy.py", "tests/test_oracle_evolve.py",
        "tests/test_oracle_aniso.py"]


def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    ok = True
    for name, a, b in MUTANTS:
        assert src.count(a) == 1, name
        with tempfile.TemporaryDirectory() as d:
            for sub in ("oracle", "synth", "tests"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("liboracle.so", "__pycache__"))
            shutil.copy(os.path.join(ROOT, "pytest.ini"), d)
            open(os.path.join(d, "oracle", "oracle.cpp"), "w").write(src.replace(a, b))
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                                *PINS], cwd=d, capture_output=True, text=True)
            tail = [l for l in r.stdout.splitlines() if l.strip()][-1:]
            killed = r.returncode != 0
            ok &= killed
            print(f"{'KILLED' if killed else 'SURVIVED'}  {name}: {tail[0] if tail else ''}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
