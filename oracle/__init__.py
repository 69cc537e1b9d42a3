"""oracle — TEST INFRASTRUCTURE ONLY.

A plain fp64 CPU oracle for the hot path of arXiv 1804.06304, written from
PAPER.md (see oracle/oracle.cpp for the per-function citations).  It checks the
CUDA path; it is not part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with
``paper_1804_06304_b200`` and never imports it.

Volumes are numpy arrays shaped ``(nz, ny, nx)`` (x fastest);
2D images use ``nz == 1``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

# Cell flags — SURVEY §8(b); the CUDA path defines its own copy in include/snk.h.
CONVERGED, COLLAPSED, RMAX, DOMAIN, LEASHED, CULLED_E0, CULLED_OVERLAP, HALO = (
    1, 2, 4, 8, 16, 32, 64, 128)
OK, EMPTY, CONFIG, SHAPE, CAPACITY = 0, 1, 2, 3, 6


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (fp64, no FMA contraction, OpenMP)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC]
    subprocess.check_call(cmd)
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


class ora_params(C.Structure):
    _fields_ = [("r0", C.c_double), ("delta_R", C.c_double), ("eps0", C.c_double),
                ("e0", C.c_double), ("iscale", C.c_double), ("max_step", C.c_double),
                ("r_min", C.c_double), ("r_max", C.c_double), ("leash", C.c_double),
                ("conv_tol", C.c_double), ("max_iters", C.c_int32), ("n_samples", C.c_int32),
                ("dim", C.c_int32), ("mode", C.c_int32), ("seed", C.c_uint64),
                ("scale", C.c_double * 3)]


class ora_cell(C.Structure):
    _fields_ = [("c", C.c_double * 3), ("R", C.c_double), ("E", C.c_double),
                ("seed", C.c_double * 3), ("flags", C.c_uint32), ("iters", C.c_int32),
                ("id", C.c_int64)]


CELL_DTYPE = np.dtype([("c", "<f8", 3), ("R", "<f8"), ("E", "<f8"), ("seed", "<f8", 3),
                       ("flags", "<u4"), ("iters", "<i4"), ("id", "<i8")])
assert CELL_DTYPE.itemsize == C.sizeof(ora_cell)


@dataclass
class Params:
    """Evolution parameters; defaults are SURVEY §8's table (readings G2-G9)."""
    r0: float = 10.0
    delta_R: float = 2.0           # G2: fixed voxels ("remain unchanged")
    eps0: float = 0.5              # G7
    e0: float = -3.0
    iscale: float = 1.0 / 257.0    # G6
    max_step: float = 1.0          # G8
    r_min: float = 1.0
    r_max: float | None = None     # default 2 r0
    leash: float | None = None     # default 2 r0
    conv_tol: float = 1e-3
    max_iters: int = 400
    n_samples: int = 1024
    dim: int = 3
    mode: int = 0                  # 0 MC, 1 grid (Eq. 5, isotropic only), 2 MC + CV, 3 ray march
    seed: int = 1804063040
    scale: tuple = (1.0, 1.0, 1.0)  # physical voxel size per axis (G28): anisotropic sampling

    def c(self) -> ora_params:
        return ora_params(self.r0, self.delta_R, self.eps0, self.e0, self.iscale,
                          self.max_step, self.r_min,
                          2 * self.r0 if self.r_max is None else self.r_max,
                          2 * self.r0 if self.leash is None else self.leash,
                          self.conv_tol, self.max_iters, self.n_samples, self.dim, self.mode,
                          self.seed & 0xFFFFFFFFFFFFFFFF, (C.c_double * 3)(*self.scale))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _declare(L):
    vp, i64, i32, u32, u64, d = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32, C.c_uint64, C.c_double
    sig = {
        "ora_philox4x32_10": (None, [vp, vp, vp]),
        "ora_sample": (None, [i32, u32, u32, i64, u64, d, vp, vp]),
        "ora_weight": (None, [d, d, d, i32, vp]),
        "ora_q14_taps": (i32, [d, vp, i32]),
        "ora_blur": (i32, [vp, vp, i32, d, vp]),
        "ora_blur3": (i32, [vp, vp, i32, vp, vp]),
        "ora_seeds_lattice3": (i32, [vp, i32, d, d, vp, vp, i64, vp]),
        "ora_seeds_maxima3": (i32, [vp, vp, vp, vp, vp, vp, i32, vp, vp, u32, vp, i64, vp]),
        "ora_label3": (i32, [vp, i32, i64, i64, vp, vp, vp, i64, vp]),
        "ora_gradmag": (i32, [vp, vp, i32, vp]),
        "ora_resample_dims": (None, [vp, vp, i32, vp]),
        "ora_resample": (i32, [vp, vp, vp, i32, vp]),
        "ora_seeds_lattice": (i32, [vp, i32, d, d, vp, i64, vp]),
        "ora_is_maxima_seed": (i32, [vp, vp, vp, vp, i32, i32, u32, i64, i64, i64]),
        "ora_seeds_maxima": (i32, [vp, vp, vp, vp, vp, vp, i32, i32, u32, vp, i64, vp]),
        "ora_energy_mc": (None, [vp, vp, vp, vp, vp, vp, d, u32, i64, vp]),
        "ora_evolve_range": (None, [vp, vp, vp, vp, vp, vp, i64, i32, i32]),
        "ora_energy_grid": (None, [vp, vp, vp, vp, vp, vp, d, vp]),
        "ora_interp": (None, [vp, vp, vp, vp, vp, vp, i64, vp, vp]),
        "ora_energy_ss": (d, [vp, vp, vp, vp, d, i32]),
        "ora_evolve": (None, [vp, vp, vp, vp, vp, vp, vp, i64, vp]),
        "ora_cull": (i32, [vp, vp, vp, vp, vp, i64, i32, d, vp, vp]),
        "ora_label": (i32, [vp, i32, i64, i64, vp, vp, i64, vp]),
        "ora_label_points": (i32, [i32, vp, i64, vp, vp, i64, vp]),
        "ora_constants": (None, [vp]),
        "ora_num_threads": (i32, []),
        "ora_set_num_threads": (None, [i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _dims(vol):
    vol = np.asarray(vol)
    if vol.ndim == 2:
        return np.array([vol.shape[1], vol.shape[0], 1], np.int64)
    return np.array([vol.shape[2], vol.shape[1], vol.shape[0]], np.int64)


def _u16(vol):
    return np.ascontiguousarray(vol, dtype=np.uint16)


# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().ora_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def sample(dim, j, it, cell_id, seed, rho_s):
    om = np.zeros(3)
    t = C.c_double()
    lib().ora_sample(dim, j, it, cell_id, seed & 0xFFFFFFFFFFFFFFFF, rho_s, _p(om), C.byref(t))
    return om, t.value


def weight(r, R, dR, dim=3):
    out = np.zeros(3)
    lib().ora_weight(r, R, dR, dim, _p(out))
    return out


def q14_taps(sigma):
    taps = np.zeros(257, np.int32)
    h = lib().ora_q14_taps(sigma, _p(taps), 257)
    if h < 0:
        raise ValueError("sigma too large")
    return taps[:2 * h + 1].copy()


def ingest_u8(vol):
    """O0 (SPEC S:348-356 loads u8 samples "without rescaling", S:402
    dtype "u8"): an 8-bit sample v becomes the u16 sample 257 v, so that the path's
    intensity scale 1/257 (reading G6) gives back v in 8-bit units exactly."""
    v = np.asarray(vol)
    assert v.dtype == np.uint8
    return (v.astype(np.int64) * 257).astype(np.uint16)


def blur(vol, dim=3, sigma=1.0):
    """O2; sigma may be a per-axis triple (anisotropic grid, G28: sigma / scale_a)."""
    v = _u16(vol)
    out = np.empty_like(v)
    if np.ndim(sigma) == 0:
        st = lib().ora_blur(_p(v), _p(_dims(v)), dim, float(sigma), _p(out))
    else:
        s3 = np.asarray(sigma, np.float64).copy()
        st = lib().ora_blur3(_p(v), _p(_dims(v)), dim, _p(s3), _p(out))
    assert st == OK
    return out


def gradmag(vol, dim=3):
    v = _u16(vol)
    out = np.empty_like(v)
    lib().ora_gradmag(_p(v), _p(_dims(v)), dim, _p(out))
    return out


def resample_dims(n_xyz, spacing, dim=3):
    n = np.asarray(n_xyz, np.int64).copy()
    s = np.asarray(spacing, np.float64).copy()
    out = np.zeros(3, np.int64)
    lib().ora_resample_dims(_p(n), _p(s), dim, _p(out))
    return out


def resample(vol, spacing, dim=3):
    v = _u16(vol)
    n = _dims(v)
    s = np.asarray(spacing, np.float64).copy()
    no = resample_dims(n, s, dim)
    out = np.empty((no[2], no[1], no[0]), np.uint16)
    lib().ora_resample(_p(v), _p(n), _p(s), dim, _p(out))
    return out if vol.ndim == 3 else out[0]


def seeds_lattice(n_xyz, dim, r0, dR=2.0, scale=(1.0, 1.0, 1.0)):
    """O4 LATTICE; on an anisotropic grid (G28) in physical coordinates."""
    n = np.asarray(n_xyz, np.int64).copy()
    sc = np.asarray(scale, np.float64).copy()
    cnt = C.c_int64()
    lib().ora_seeds_lattice3(_p(n), dim, r0, dR, _p(sc), None, 0, C.byref(cnt))
    cap = max(int(cnt.value), 1)
    out = np.zeros((cap, 3), np.float32)
    st = lib().ora_seeds_lattice3(_p(n), dim, r0, dR, _p(sc), _p(out), cap, C.byref(cnt))
    return st, out[:cnt.value] if st == OK else out[:0]


def _box(v, org, n_global, z_lo=0):
    """(global dims, box origin, box dims) as int64 arrays for a buffer v."""
    nb = _dims(v)
    org = np.array([0, 0, z_lo] if org is None else org, np.int64)
    n = (org + nb) if n_global is None else np.asarray(n_global, np.int64).copy()
    if n_global is None and tuple(org) != (0, 0, 0):
        raise ValueError("n_global is required for a crop")
    return n, org, nb


def is_maxima_seed(vol, dim, w, thr, x, y, z, org=None, n_global=None):
    v = _u16(vol)
    n, o, nb = _box(v, org, n_global)
    r = lib().ora_is_maxima_seed(_p(v), _p(n), _p(o), _p(nb), dim, w, thr, x, y, z)
    if r < 0:
        raise ValueError("window outside the buffer")
    return bool(r)


def seeds_maxima(vol, dim, w, thr, org=None, n_global=None, lo=None, hi=None, scale=(1.0, 1.0, 1.0)):
    """Seeds of the (global) box lo..hi (inclusive; default: the whole buffer).
    w may be a per-axis triple; seeds come out in physical coordinates (index x scale, G28)."""
    v = _u16(vol)
    n, o, nb = _box(v, org, n_global)
    lo = o.copy() if lo is None else np.asarray(lo, np.int64).copy()
    hi = (o + nb - 1) if hi is None else np.asarray(hi, np.int64).copy()
    w3 = np.asarray([w, w, w] if np.ndim(w) == 0 else w, np.int32).copy()
    sc = np.asarray(scale, np.float64).copy()
    cnt = C.c_int64()
    cap = 1 << 16
    while True:
        out = np.zeros((cap, 3), np.float32)
        st = lib().ora_seeds_maxima3(_p(v), _p(n), _p(o), _p(nb), _p(lo), _p(hi), dim, _p(w3), _p(sc), thr,
                                     _p(out), cap, C.byref(cnt))
        if st == CAPACITY:
            cap = int(cnt.value)
            continue
        if st != OK:
            raise ValueError(f"ora_seeds_maxima status {st}")
        return out[:cnt.value]


def energy_mc(vol, params: Params, c, R, it, cell_id, org=None, n_global=None):
    v = _u16(vol)
    n, o, nb = _box(v, org, n_global)
    cc = np.asarray(c, np.float64).copy()
    out = np.zeros(6)
    pc = params.c()
    lib().ora_energy_mc(_p(v), _p(n), _p(o), _p(nb), C.byref(pc), _p(cc), R, it, cell_id, _p(out))
    return out


def interp(vol, pts_xyz, dim=3, iscale=1.0, scale=(1.0, 1.0, 1.0), org=None, n_global=None):
    """O5 step 4 (G17): d-linear lookup of the u16 volume at physical points
    (x, y, z) — clamp to [0, n-1], i0 = min(floor(k), n-2), x then y then z —
    times iscale.  Returns (values, halo flags)."""
    v = _u16(vol)
    n, o, nb = _box(v, org, n_global)
    pc = Params(dim=dim, iscale=iscale, scale=tuple(scale)).c()
    k = np.ascontiguousarray(pts_xyz, np.float64).reshape(-1, 3)
    out = np.zeros(len(k))
    halo = np.zeros(len(k), np.int32)
    lib().ora_interp(_p(v), _p(n), _p(o), _p(nb), C.byref(pc), _p(k), len(k), _p(out), _p(halo))
    return out, halo.astype(bool)


def energy_grid(vol, params: Params, c, R):
    v = _u16(vol)
    n = _dims(v)
    cc = np.asarray(c, np.float64).copy()
    out = np.zeros(6)
    pc = params.c()
    o = np.zeros(3, np.int64)
    lib().ora_energy_grid(_p(v), _p(n), _p(o), _p(n), C.byref(pc), _p(cc), R, _p(out))
    return out


def energy_ss(vol, params: Params, c, R, q=6):
    v = _u16(vol)
    cc = np.asarray(c, np.float64).copy()
    pc = params.c()
    return lib().ora_energy_ss(_p(v), _p(_dims(v)), C.byref(pc), _p(cc), R, q)


def evolve(vol, params: Params, seeds, ids=None, org=None, n_global=None, z_lo=0):
    """O5 for every seed; returns a CELL_DTYPE record array.  ``vol`` may be a
    crop/slab at ``org`` (or planes from ``z_lo``) of a volume of dims ``n_global``."""
    v = _u16(vol)
    if org is None and z_lo:
        org = (0, 0, z_lo)
    n, o, nb = _box(v, org, n_global)
    s = np.ascontiguousarray(seeds, np.float32).reshape(-1, 3)
    ids = (np.arange(len(s), dtype=np.int64) if ids is None
           else np.ascontiguousarray(ids, np.int64))
    out = np.zeros(len(s), CELL_DTYPE)
    pc = params.c()
    lib().ora_evolve(_p(v), _p(n), _p(o), _p(nb), C.byref(pc), _p(s), _p(ids), len(s), _p(out))
    return out


def evolve_range(vol, params: Params, cells, it0: int, it1: int, org=None, n_global=None):
    """Continue the records ``cells`` (CELL_DTYPE; c, R, E, seed, flags, id are
    the state) through iterations it0..it1; returns the new records."""
    v = _u16(vol)
    n, o, nb = _box(v, org, n_global)
    out = np.ascontiguousarray(cells, CELL_DTYPE).copy()
    pc = params.c()
    lib().ora_evolve_range(_p(v), _p(n), _p(o), _p(nb), C.byref(pc), _p(out), len(out), int(it0), int(it1))
    return out


def init_cells(params: Params, seeds, ids=None):
    """Records at the start of evolution: c = seed, R = r0 (O5)."""
    s = np.ascontiguousarray(seeds, np.float32).reshape(-1, 3).astype(np.float64)
    out = np.zeros(len(s), CELL_DTYPE)
    out["c"] = s
    out["seed"] = s
    out["R"] = params.r0
    out["id"] = np.arange(len(s), dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    return out


def checkpoints(T: int, k: int):
    """Periodic-culling segments (reading G25): [1, k], [k+1, 2k], ..., the last
    one ending at T + 1 (E_final); a cull after every segment but the last."""
    if k <= 0 or k >= T:
        return [(1, T + 1)]
    ends = list(range(k, T, k)) + [T + 1]
    starts = [1] + [e + 1 for e in ends[:-1]]
    return list(zip(starts, ends))


def evolve_periodic(vol, params: Params, seeds, k: int, ids=None, org=None, n_global=None):
    """Evolution with periodic culling every k iterations (SURVEY §8(f) 2
    "dynamic culling"; reading G25): after segment [a, b] (b < T + 1) the live
    records — state after iteration b, E of iteration b — go through O6 (E0,
    then the greedy overlap competition on fp32 values); the survivors continue.
    Returns the live records after iteration T + 1 (cull them with ``cull`` for
    the detections)."""
    cells = init_cells(params, seeds, ids)
    for a, b in checkpoints(params.max_iters, k):
        cells = evolve_range(vol, params, cells, a, b, org=org, n_global=n_global)
        if b <= params.max_iters:
            keep = cull(cells["c"].astype(np.float32), cells["R"].astype(np.float32),
                        cells["E"].astype(np.float32), cells["flags"], cells["id"], params.dim, params.e0)
            cells = cells[np.sort(keep)]
    return cells


def cull(c, R, E, flags, ids, dim, e0):
    """O6; returns input indices of the survivors in (E, id) order."""
    c = np.ascontiguousarray(c, np.float32).reshape(-1, 3)
    R = np.ascontiguousarray(R, np.float32)
    E = np.ascontiguousarray(E, np.float32)
    flags = np.ascontiguousarray(flags, np.uint32)
    ids = np.ascontiguousarray(ids, np.int64)
    keep = np.zeros(max(len(R), 1), np.int64)
    nk = C.c_int64()
    lib().ora_cull(_p(c), _p(R), _p(E), _p(flags), _p(ids), len(R), dim, e0, _p(keep), C.byref(nk))
    return keep[:nk.value].copy()


def label(n_xyz, dim, c, R, z0=0, nz=None, scale=(1.0, 1.0, 1.0)):
    """O7; voxel (x, y, z) at the physical point (x, y, z) * scale (G28)."""
    n = np.asarray(n_xyz, np.int64).copy()
    nz = int(n[2]) - z0 if nz is None else nz
    c = np.ascontiguousarray(c, np.float32).reshape(-1, 3)
    R = np.ascontiguousarray(R, np.float32)
    sc = np.asarray(scale, np.float64).copy()
    out = np.zeros((nz, n[1], n[0]), np.int32)
    lib().ora_label3(_p(n), dim, z0, nz, _p(sc), _p(c), _p(R), len(R), _p(out))
    return out


def label_points(dim, pts_xyz, c, R):
    pts = np.ascontiguousarray(pts_xyz, np.int64).reshape(-1, 3)
    c = np.ascontiguousarray(c, np.float32).reshape(-1, 3)
    R = np.ascontiguousarray(R, np.float32)
    out = np.zeros(len(pts), np.int32)
    lib().ora_label_points(dim, _p(pts), len(pts), _p(c), _p(R), len(R), _p(out))
    return out


def constants():
    out = np.zeros(4)
    lib().ora_constants(_p(out))
    return {"rho3": out[0], "rho2": out[1], "rho2_3d": out[2], "rho2_2d": out[3]}


def num_threads():
    return lib().ora_num_threads()


def set_num_threads(t):
    lib().ora_set_num_threads(t)


@dataclass
class Result:
    """End-to-end oracle pipeline output."""
    seeds: np.ndarray
    cells: np.ndarray
    keep: np.ndarray
    labels: np.ndarray | None = None
    extra: dict = field(default_factory=dict)


def run_pipeline(raw, params: Params, *, spacing=(1.0, 1.0, 1.0), sigma=1.0, seed_mode="lattice",
                 seed_window=None, seed_threshold=None, image_term="intensity", with_labels=True):
    """a1..a8 on the CPU: resample -> blur (+gradmag) -> seeds -> evolve -> cull -> label."""
    dim = params.dim
    vol = raw if raw.ndim == 3 else raw[None]
    if any(s != spacing[0] for s in spacing[:dim]):
        vol = resample(vol, spacing, dim)
    B = blur(vol, dim, sigma)
    img = gradmag(B, dim) if image_term == "gradmag" else B
    n = _dims(B)
    if seed_mode == "lattice":
        st, seeds = seeds_lattice(n, dim, params.r0, params.delta_R)
    else:
        seeds = seeds_maxima(B, dim, seed_window, seed_threshold)
    cells = evolve(img, params, seeds)
    c32 = cells["c"].astype(np.float32)
    R32 = cells["R"].astype(np.float32)
    E32 = cells["E"].astype(np.float32)
    keep = cull(c32, R32, E32, cells["flags"], cells["id"], dim, params.e0)
    labels = label(n, dim, c32[keep], R32[keep]) if with_labels else None
    return Result(seeds=seeds, cells=cells, keep=keep, labels=labels, extra={"smooth": B})
