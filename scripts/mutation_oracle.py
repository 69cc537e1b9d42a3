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
    # round 2: mutants across the rest of the oracle
    ("philox: 9 rounds", "for (int round = 0; round < 10; ++round)", "for (int round = 0; round < 9; ++round)"),
    ("philox: multiplier typo", "M1 = 0xCD9E8D57u", "M1 = 0xCD9E8D55u"),
    ("philox: key words swapped", "const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;",
     "const uint32_t n0 = hi1 ^ c1 ^ k1, n1 = lo1, n2 = hi0 ^ c3 ^ k0, n3 = lo0;"),
    ("sampler: sin(theta) without its factor 2", "    const double st = 2.0 * std::sqrt(u0 * (1.0 - u0));\n    omega[0]",
     "    const double st = std::sqrt(u0 * (1.0 - u0));\n    omega[0]"),
    ("sampler: 3D radius law sqrt instead of cbrt", "*t = rho_s * std::cbrt(u2);", "*t = rho_s * std::sqrt(u2);"),
    ("weight: inner ramp gain 1 instead of 2", "*S = (1.0 - s3(tau_o)) - 2.0 * (1.0 - s3(tau_i));",
     "*S = (1.0 - s3(tau_o)) - 1.0 * (1.0 - s3(tau_i));"),
    ("weight: S_r sign of the outer term", "*S_r = -ds3(tau_o) / dR + 2.0 * ds3(tau_i) / (rho * dR);",
     "*S_r = ds3(tau_o) / dR + 2.0 * ds3(tau_i) / (rho * dR);"),
    ("weight: S_R inner term over rho dR", "*S_R = ds3(tau_o) / dR - 2.0 * ds3(tau_i) / dR;",
     "*S_R = ds3(tau_o) / dR - 2.0 * ds3(tau_i) / (rho * dR);"),
    ("step: eps0 / n instead of eps0 / sqrt(n)", "const double eps = p->eps0 / std::sqrt((double)it);",
     "const double eps = p->eps0 / (double)it;"),
    ("step: eps instead of eps / 2 on c", "clampd(-(eps / 2.0) * eo.gc[a]", "clampd(-(eps) * eo.gc[a]"),
    ("leash: asymmetric", "clampd(c[a], s[a] - p->leash, s[a] + p->leash)", "clampd(c[a], s[a] - 2.0 * p->leash, s[a] + p->leash)"),
    ("domain: ball may leave the volume", "else cd = clampd(c[a], m, L - m);", "else cd = clampd(c[a], 0.0, L);"),
    ("cull: E descending", "if (E[a] != E[b]) return E[a] < E[b];", "if (E[a] != E[b]) return E[a] > E[b];"),
    ("cull: id tie descending", "    return ids[a] < ids[b];\n", "    return ids[a] > ids[b];\n"),
    ("label: ties to the larger index", "if (best < 0 || key < best_key) { best = i; best_key = key; }",
     "if (best < 0 || key <= best_key) { best = i; best_key = key; }"),
    ("label: threshold 1% large", "const double thr = ((double)R[i] * (double)R[i]) * rho2;",
     "const double thr = ((double)R[i] * (double)R[i]) * rho2 * 1.01;"),
    ("blur: rounding constant 8191", "nxt[x + y * stride[1] + z * stride[2]] = (uint16_t)((acc + 8192) >> 14);",
     "nxt[x + y * stride[1] + z * stride[2]] = (uint16_t)((acc + 8191) >> 14);"),
    ("maxima: ties to the later voxel", "if (u == v && (zz * ny + yy) * nx + xx < lin) return false;",
     "if (u == v && (zz * ny + yy) * nx + xx > lin) return false;"),
    ("lattice: spacing sqrt(2) r0", "const double s = std::sqrt(1.5) * r0;", "const double s = std::sqrt(2.0) * r0;"),
    ("resample: truncation instead of rounding", "(v0 * (16384 - w1[k]) + v1 * w1[k] + 8192) >> 14",
     "(v0 * (16384 - w1[k]) + v1 * w1[k]) >> 14"),
    ("gradmag: isqrt off by one", "  while ((r + 1) * (r + 1) <= v) ++r;\n  return r;", "  while ((r + 1) * (r + 1) <= v) ++r;\n  return r + (v > 4 ? 1 : 0);"),
]


PINS = ["tests/test_oracle_interp.py", "tests/test_oracle_energy.py", "tests/test_oracle_evolve.py",
        "tests/test_oracle_aniso.py", "tests/test_oracle_rng.py", "tests/test_oracle_weight.py",
        "tests/test_oracle_volume.py", "tests/test_oracle_cull_label.py"]


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
            if os.path.exists(os.path.join(ROOT, "tests", "golden")):
                pass   # copied with tests/
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
