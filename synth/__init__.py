"""synth — seeded synthetic inputs for configs C1..C5.

This module generates INPUTS only (u16 volumes of DAPI-like ellipsoidal nuclei
plus their ground truth) and the per-config run parameters.  It contains none
of the method's arithmetic, and is shared by the oracle tests and the CUDA
path.  The heavy lifting is C++ (synth/gen.cpp, OpenMP); any z-range of a
volume can be generated independently, which the z-slab driver relies on.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.cpp")
_LIB = os.path.join(_HERE, "libsynth.so")


def build(force: bool = False) -> str:
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    subprocess.check_call(["g++", "-O3", "-std=c++17", "-fopenmp", "-shared", "-fPIC",
                           "-o", _LIB + ".tmp", _SRC])
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class synth_spec(C.Structure):
    _fields_ = [("dim", C.c_int32), ("_pad", C.c_int32), ("n", C.c_int64 * 3),
                ("spacing", C.c_double * 3), ("count", C.c_int64 * 3), ("pitch", C.c_double * 3),
                ("origin", C.c_double * 3), ("jitter", C.c_double), ("rbar_lo", C.c_double),
                ("rbar_hi", C.c_double), ("axis_var", C.c_double), ("amp", C.c_double),
                ("amp_cv", C.c_double), ("edge", C.c_double), ("bg", C.c_double),
                ("bg_mod", C.c_double), ("bg_wavelength", C.c_double), ("noise", C.c_double),
                ("seed", C.c_uint64)]


NUCLEUS_DTYPE = np.dtype([("c", "<f8", 3), ("axes", "<f8", 3), ("rot", "<f8", 9),
                          ("amp", "<f8"), ("rbar", "<f8")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.synth_generate.restype = C.c_int
        _lib.synth_generate.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        _lib.synth_num_nuclei.restype = C.c_int64
        _lib.synth_num_nuclei.argtypes = [C.c_void_p]
        _lib.synth_nuclei.restype = None
        _lib.synth_nuclei.argtypes = [C.c_void_p, C.c_void_p]
        _lib.synth_num_threads.restype = C.c_int
    return _lib


@dataclass
class Config:
    """One workload: the synthetic volume recipe and the run parameters."""
    name: str
    dim: int
    n: tuple                      # raw dims (x, y, z)
    spacing: tuple = (1.0, 1.0, 1.0)
    count: tuple = (1, 1, 1)      # nuclei per axis
    pitch: tuple = (1.0, 1.0, 1.0)
    origin: tuple | None = None   # None: lattice centred in the isotropic volume
    jitter: float = 0.0
    rbar: tuple = (10.0, 10.0)
    axis_var: float = 0.2
    amp: float = 100.0
    amp_cv: float = 0.1
    edge: float = 0.5
    bg: float = 20.0
    bg_mod: float = 5.0
    bg_wavelength: float = 128.0
    noise: float = 10.0
    gen_seed: int = 0x5EED0001
    # run parameters (SURVEY §8 defaults)
    r0: float = 10.0
    n_samples: int = 1024
    max_iters: int = 400
    seed_mode: str = "maxima"     # "lattice" | "maxima"
    seed_threshold: int = 70 * 257
    seed_window: int | None = None  # default round(rho r0 / 2)
    philox_seed: int = 1804063040
    extra: dict = field(default_factory=dict)

    @property
    def iso_n(self):
        sp = self.spacing[:self.dim]
        smin = min(sp)
        out = list(self.n)
        for a in range(self.dim):
            if self.spacing[a] > smin:
                out[a] = int(round(self.n[a] * self.spacing[a] / smin))
        return tuple(out)

    @property
    def window(self):
        if self.seed_window is not None:
            return self.seed_window
        rho = 2.0 ** (-1.0 / self.dim)
        return int(math.floor(rho * self.r0 / 2.0 + 0.5))

    def spec(self) -> synth_spec:
        s = synth_spec()
        s.dim = self.dim
        s.n[:] = list(self.n)
        s.spacing[:] = list(self.spacing)
        s.count[:] = list(self.count)
        s.pitch[:] = list(self.pitch)
        if self.origin is None:
            iso = self.iso_n
            org = [(iso[a] - self.count[a] * self.pitch[a]) / 2.0 + self.pitch[a] / 2.0
                   if a < self.dim else 0.0 for a in range(3)]
        else:
            org = list(self.origin)
        s.origin[:] = org
        s.jitter = self.jitter
        s.rbar_lo, s.rbar_hi = self.rbar
        s.axis_var, s.amp, s.amp_cv, s.edge = self.axis_var, self.amp, self.amp_cv, self.edge
        s.bg, s.bg_mod, s.bg_wavelength, s.noise = self.bg, self.bg_mod, self.bg_wavelength, self.noise
        s.seed = self.gen_seed
        return s

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


def _c3_like(name, pitch, count, rbar, r0, idx, **kw):
    return Config(name=name, dim=3, n=(512, 512, 128), spacing=(1.0, 1.0, 2.0), count=count,
                  pitch=pitch, jitter=0.15 * min(pitch), rbar=(rbar, rbar), r0=r0,
                  gen_seed=0x5EED0000 + idx, philox_seed=1804063040 + idx, **kw)


CONFIGS = {
    # C1: 64^3, 8 well separated nuclei on a 2x2x2 lattice at 16/48 +- 2, rbar in [6, 9]
    "C1": Config(name="C1", dim=3, n=(64, 64, 64), count=(2, 2, 2), pitch=(32.0, 32.0, 32.0),
                 origin=(16.0, 16.0, 16.0), jitter=2.0, rbar=(6.0, 9.0), bg_wavelength=64.0,
                 r0=10.0, n_samples=256, seed_mode="lattice", gen_seed=0x5EED0001,
                 philox_seed=1804063041),
    # C2: 2D 2048^2, ~2025 densely packed ellipses (paper's 2D mode)
    "C2": Config(name="C2", dim=2, n=(2048, 2048, 1), count=(45, 45, 1), pitch=(45.0, 45.0, 1.0),
                 jitter=0.15 * 45.0, rbar=(18.0, 18.0), bg_wavelength=256.0, r0=25.0,
                 n_samples=1024, gen_seed=0x5EED0002, philox_seed=1804063042),
    # C3: 512x512x128 raw, spacing (1,1,2) -> 512x512x256, ~10.2k touching nuclei
    "C3": _c3_like("C3", (17.8, 17.8, 19.0), (28, 28, 13), 9.0, 11.0, 3, n_samples=1024),
    # C4: 2048x2048x512 brain-like, 198,927 touching nuclei (z-slabs on 1/2/4/8 GPUs)
    "C4": Config(name="C4", dim=3, n=(2048, 2048, 512), count=(93, 93, 23),
                 pitch=(22.0, 22.0, 22.0), jitter=0.15 * 22.0, rbar=(10.0, 10.0),
                 bg_wavelength=256.0, r0=13.0, n_samples=1024, gen_seed=0x5EED0004,
                 philox_seed=1804063044),
}
# C5: C3's volume at four densities (r-bar 7, R0 9), swept over N in 64..4096
for _i, (_a, _k) in enumerate([(29.0, (17, 17, 8)), (23.0, (22, 22, 11)), (18.3, (27, 27, 13)),
                               (14.6, (35, 35, 17))]):
    CONFIGS[f"C5_{_i}"] = _c3_like(f"C5_{_i}", (_a, _a, _a), _k, 7.0, 9.0, 5, n_samples=1024)


def get(cfg) -> Config:
    return CONFIGS[cfg] if isinstance(cfg, str) else cfg


def generate(cfg, z0: int = 0, z1: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Raw u16 planes [z0, z1) of the config's volume, shaped (nz, ny, nx)."""
    cfg = get(cfg)
    z1 = cfg.n[2] if z1 is None else z1
    shape = (z1 - z0, cfg.n[1], cfg.n[0])
    if out is None:
        out = np.empty(shape, np.uint16)
    assert out.shape == shape and out.dtype == np.uint16 and out.flags.c_contiguous
    s = cfg.spec()
    lib().synth_generate(C.byref(s), z0, z1, out.ctypes.data_as(C.c_void_p))
    return out


def generate_into_ptr(cfg, ptr: int, z0: int = 0, z1: int | None = None) -> None:
    """Write raw planes [z0, z1) to host memory at ``ptr`` (e.g. a pinned tensor)."""
    cfg = get(cfg)
    z1 = cfg.n[2] if z1 is None else z1
    s = cfg.spec()
    lib().synth_generate(C.byref(s), z0, z1, C.c_void_p(ptr))


def nuclei(cfg) -> np.ndarray:
    """Ground truth: one NUCLEUS_DTYPE record per nucleus (isotropic voxel units)."""
    cfg = get(cfg)
    s = cfg.spec()
    k = lib().synth_num_nuclei(C.byref(s))
    out = np.zeros(k, NUCLEUS_DTYPE)
    lib().synth_nuclei(C.byref(s), out.ctypes.data_as(C.c_void_p))
    return out


def sphere_volume(n_xyz, centre, r0, amp=100.0, bg=0.0, scale=257.0, supersample=4):
    """Voxelised sphere phantom (P:94 blob model I = 1 + sign(r0 - r), scaled):
    each voxel gets bg + amp * (fraction of its q^3 sub-points inside the sphere),
    times ``scale``, rounded to u16.  Used by the analytic oracle pins."""
    nx, ny, nz = n_xyz
    q = supersample
    off = (np.arange(q) + 0.5) / q - 0.5
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    frac = np.zeros((nz, ny, nx))
    for dz in (off if nz > 1 else [0.0]):
        for dy in off:
            for dx in off:
                r2 = (x + dx - centre[0]) ** 2 + (y + dy - centre[1]) ** 2
                if nz > 1:
                    r2 = r2 + (z + dz - centre[2]) ** 2
                frac += r2 < r0 * r0
    frac /= q ** (3 if nz > 1 else 2)
    v = np.floor((bg + amp * frac) * scale + 0.5)
    return np.clip(v, 0, 65535).astype(np.uint16)
