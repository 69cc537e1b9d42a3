"""Thin ctypes binding of libsnk.so (include/snk.h): the same names, argument
marshalling only.  Every step of the hot path runs in the CUDA kernels behind
these calls; there is no CPU fallback — if libsnk.so is missing, importing
this module raises.

Pointers may be passed as torch tensors (``.data_ptr()`` is used), numpy
arrays (host), or plain integers.  Streams are ``torch.cuda.Stream`` objects,
raw ``cudaStream_t`` integers, or None (the legacy default stream).
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SNK_LIB: an alternative build (tuning experiments, scripts/); default the in-tree libsnk.so
LIB_PATH = os.environ.get("SNK_LIB") or os.path.join(HERE, "libsnk.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "snk.h")

OK, EMPTY_DOMAIN, CONFIG, SHAPE, INTERNAL, CUDA, CAPACITY = 0, 1, 2, 3, 4, 5, 6
F_CONVERGED, F_COLLAPSED, F_RMAX, F_DOMAIN, F_LEASHED, F_CULLED_E0, F_CULLED_OVERLAP, F_HALO = (
    1, 2, 4, 8, 16, 32, 64, 128)
SEED_LATTICE, SEED_MAXIMA, SEED_GIVEN = 0, 1, 2
IMAGE_INTENSITY, IMAGE_GRADMAG = 0, 1
EST_MC, EST_GRID, EST_MC_CV, EST_RAY = 0, 1, 2, 3


class SNKError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status} ({status_string(status)}): {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1804_06304_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)


class snk_grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("_pad0", C.c_int32), ("n", C.c_int64 * 3),
                ("z_lo", C.c_int64), ("nz_buf", C.c_int64), ("own_z0", C.c_int64),
                ("own_z1", C.c_int64), ("scale", C.c_double * 3)]


class snk_params(C.Structure):
    _fields_ = [("r0", C.c_double), ("delta_R", C.c_double), ("eps0", C.c_double),
                ("e0", C.c_double), ("sigma", C.c_double), ("intensity_scale", C.c_double),
                ("max_step", C.c_double), ("r_min", C.c_double), ("r_max", C.c_double),
                ("leash", C.c_double), ("conv_tol", C.c_double), ("max_iters", C.c_int32),
                ("n_samples", C.c_int32), ("seed_mode", C.c_int32), ("seed_window", C.c_int32),
                ("image_term", C.c_int32), ("cta_warps", C.c_int32), ("seed_threshold", C.c_uint32),
                ("kernel_variant", C.c_uint32), ("estimator", C.c_int32), ("cull_every", C.c_int32),
                ("seed", C.c_uint64)]


class snk_cell(C.Structure):
    _fields_ = [("c", C.c_float * 3), ("R", C.c_float), ("seed", C.c_float * 3),
                ("energy", C.c_float), ("flags", C.c_uint32), ("iters", C.c_int32),
                ("id", C.c_int64), ("disp", C.c_float * 3), ("reserved", C.c_uint32)]


CELL_DTYPE = np.dtype([("c", "<f4", 3), ("R", "<f4"), ("seed", "<f4", 3), ("energy", "<f4"),
                       ("flags", "<u4"), ("iters", "<i4"), ("id", "<i8"), ("disp", "<f4", 3),
                       ("reserved", "<u4")])
CELL_BYTES = 64   # sizeof(snk_cell), include/snk.h
assert CELL_DTYPE.itemsize == C.sizeof(snk_cell) == CELL_BYTES

_vp, _i32, _i64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
_P = C.POINTER
_SIGS = {
    "snk_abi_version": (_i32, []),
    "snk_last_error": (C.c_char_p, []),
    "snk_status_string": (C.c_char_p, [_i32]),
    "snk_validate": (_i32, [_P(snk_grid), _P(snk_params)]),
    "snk_workspace_bytes": (_i32, [_P(snk_grid), _P(snk_params), _i64, _P(_sz)]),
    "snk_resample_dims": (_i32, [_i32, _vp, _vp, _vp]),
    "snk_resample": (_i32, [_i32, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "snk_preprocess": (_i32, [_P(snk_grid), _P(snk_params), _vp, _vp, _vp, _vp, _sz, _vp]),
    "snk_seeds": (_i32, [_P(snk_grid), _P(snk_params), _vp, _vp, _i64, _P(_i64), _P(_i64), _vp, _sz,
                         _vp]),
    "snk_evolve": (_i32, [_P(snk_grid), _P(snk_params), _vp, _vp, _vp, _i64, _i64, _vp, _vp, _sz,
                          _vp]),
    "snk_cells_init": (_i32, [_P(snk_params), _vp, _vp, _i64, _i64, _vp, _vp]),
    "snk_evolve_range": (_i32, [_P(snk_grid), _P(snk_params), _vp, _vp, _i64, _i32, _i32, _vp, _sz, _vp]),
    "snk_compact_candidates": (_i32, [_P(snk_params), _vp, _i64, _vp, _i64, _P(_i64), _vp, _sz, _vp]),
    "snk_select_ids": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _P(_i64), _vp, _sz, _vp]),
    "snk_cull": (_i32, [_P(snk_grid), _P(snk_params), _vp, _i64, _vp, _i64, _P(_i64), _vp, _sz, _vp]),
    "snk_label": (_i32, [_P(snk_grid), _P(snk_params), _vp, _i64, _vp, _vp, _sz, _vp]),
    "snk_run_workspace_bytes": (_i32, [_i32, _vp, _vp, _P(snk_params), _i64, _P(_sz)]),
    "snk_ingest_u8": (_i32, [_vp, _vp, _i64, _vp]),
    "snk_run_u8": (_i32, [_i32, _vp, _vp, _P(snk_params), _vp, _vp, _i64, _P(_i64), _vp, _i64, _vp, _sz, _vp]),
    "snk_run": (_i32, [_i32, _vp, _vp, _P(snk_params), _vp, _vp, _i64, _P(_i64), _vp, _i64, _vp, _sz,
                       _vp]),
    "snk_run_batch_workspace_bytes": (_i32, [_i32, _vp, _vp, _P(snk_params), _i64, _P(_sz)]),
    "snk_run_batch": (_i32, [_i32, _vp, _vp, _P(snk_params), _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _sz,
                             _vp]),
    "snk_launch_count": (_i64, []),
    "snk_evolve_stats": (_i32, [_vp, _i32]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def declared_symbols() -> list[str]:
    """Functions declared in include/snk.h (used by the ABI test)."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(snk_\w+)\(", txt, re.M)))


# ---------------------------------------------------------------- marshalling
def _ptr(x) -> C.c_void_p:
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        return x.ctypes.data_as(C.c_void_p)
    raise TypeError(f"cannot pass {type(x)} as a pointer")


def _stream(s) -> C.c_void_p:
    if s is None:
        return None
    if isinstance(s, int):
        return C.c_void_p(s)
    return C.c_void_p(s.cuda_stream)


def _nbytes(x) -> int:
    if x is None:
        return 0
    if hasattr(x, "untyped_storage"):
        return x.numel() * x.element_size()
    return int(x)


def _check(status: int, where: str):
    if status != OK:
        raise SNKError(status, where, snk_last_error())


def _i64x3(v):
    return (C.c_int64 * 3)(*[int(a) for a in v])


def _f64x3(v):
    return (C.c_double * 3)(*[float(a) for a in v])


# ---------------------------------------------------------------- the C ABI, same names
def snk_abi_version() -> int:
    return _lib.snk_abi_version()


def snk_last_error() -> str:
    return (_lib.snk_last_error() or b"").decode()


def status_string(s: int) -> str:
    return (_lib.snk_status_string(s) or b"").decode()


snk_status_string = status_string


def snk_launch_count() -> int:
    return _lib.snk_launch_count()


def snk_evolve_stats(reset: bool = False) -> dict:
    out = np.zeros(4, np.int64)
    _check(_lib.snk_evolve_stats(out.ctypes.data_as(C.c_void_p), int(reset)), "snk_evolve_stats")
    return {"brick_loads": int(out[0]), "global_iterations": int(out[1])}


def snk_validate(g: snk_grid, p: snk_params) -> int:
    return _lib.snk_validate(C.byref(g), C.byref(p))


def snk_workspace_bytes(g: snk_grid, p: snk_params, max_cells: int) -> int:
    out = C.c_size_t()
    _check(_lib.snk_workspace_bytes(C.byref(g), C.byref(p), max_cells, C.byref(out)),
           "snk_workspace_bytes")
    return out.value


def snk_resample_dims(dim: int, n_raw, spacing) -> tuple:
    out = (C.c_int64 * 3)()
    _check(_lib.snk_resample_dims(dim, _i64x3(n_raw), _f64x3(spacing), out), "snk_resample_dims")
    return tuple(out)


def snk_resample(dim, n_raw, spacing, zr_lo, nzr, d_raw, z_lo, nz_out, d_out, d_ws, stream=None):
    _check(_lib.snk_resample(dim, _i64x3(n_raw), _f64x3(spacing), zr_lo, nzr, _ptr(d_raw), z_lo,
                             nz_out, _ptr(d_out), _ptr(d_ws), _nbytes(d_ws) if d_ws is not None else 0,
                             _stream(stream)), "snk_resample")


def snk_preprocess(g, p, d_in, d_smooth, d_gradmag, d_ws, stream=None):
    _check(_lib.snk_preprocess(C.byref(g), C.byref(p), _ptr(d_in), _ptr(d_smooth), _ptr(d_gradmag),
                               _ptr(d_ws), _nbytes(d_ws), _stream(stream)), "snk_preprocess")


def snk_seeds(g, p, d_smooth, d_seeds, cap, d_ws, stream=None) -> tuple[int, int]:
    n = C.c_int64()
    first = C.c_int64()
    _check(_lib.snk_seeds(C.byref(g), C.byref(p), _ptr(d_smooth), _ptr(d_seeds), cap, C.byref(n),
                          C.byref(first), _ptr(d_ws), _nbytes(d_ws), _stream(stream)), "snk_seeds")
    return n.value, first.value


def snk_evolve(g, p, d_image, d_seeds, d_ids, id_base, n, d_cells, d_ws, stream=None):
    _check(_lib.snk_evolve(C.byref(g), C.byref(p), _ptr(d_image), _ptr(d_seeds), _ptr(d_ids), id_base,
                           n, _ptr(d_cells), _ptr(d_ws), _nbytes(d_ws) if d_ws is not None else 0,
                           _stream(stream)), "snk_evolve")


def snk_cells_init(p, d_seeds, d_ids, id_base, n, d_cells, stream=None):
    _check(_lib.snk_cells_init(C.byref(p), _ptr(d_seeds), _ptr(d_ids), id_base, n, _ptr(d_cells),
                               _stream(stream)), "snk_cells_init")


def snk_evolve_range(g, p, d_image, d_cells, n, it0, it1, d_ws, stream=None):
    _check(_lib.snk_evolve_range(C.byref(g), C.byref(p), _ptr(d_image), _ptr(d_cells), n, it0, it1,
                                 _ptr(d_ws), _nbytes(d_ws) if d_ws is not None else 0, _stream(stream)),
           "snk_evolve_range")


def checkpoints(T: int, k: int):
    """Periodic-culling segments (G25; the library's own list in snk_run): [1, k],
    [k+1, 2k], ..., the last ending at T + 1; a cull after each but the last."""
    if k <= 0 or k >= T:
        return [(1, T + 1)]
    ends = list(range(k, T, k)) + [T + 1]
    return list(zip([1] + [e + 1 for e in ends[:-1]], ends))


def snk_compact_candidates(p, d_cells, n, d_out, cap, d_ws, stream=None) -> int:
    out = C.c_int64()
    _check(_lib.snk_compact_candidates(C.byref(p), _ptr(d_cells), n, _ptr(d_out), cap, C.byref(out),
                                       _ptr(d_ws), _nbytes(d_ws), _stream(stream)),
           "snk_compact_candidates")
    return out.value


def snk_select_ids(d_cells, n, id_lo, id_hi, d_out, cap, d_ws, stream=None) -> int:
    out = C.c_int64()
    _check(_lib.snk_select_ids(_ptr(d_cells), n, id_lo, id_hi, _ptr(d_out), cap, C.byref(out), _ptr(d_ws),
                               _nbytes(d_ws), _stream(stream)), "snk_select_ids")
    return out.value


def snk_cull(g, p, d_cells, n, d_dets, cap, d_ws, stream=None) -> int:
    out = C.c_int64()
    _check(_lib.snk_cull(C.byref(g), C.byref(p), _ptr(d_cells), n, _ptr(d_dets), cap, C.byref(out),
                         _ptr(d_ws), _nbytes(d_ws), _stream(stream)), "snk_cull")
    return out.value


def snk_label(g, p, d_dets, n, d_labels, d_ws, stream=None):
    _check(_lib.snk_label(C.byref(g), C.byref(p), _ptr(d_dets), n, _ptr(d_labels), _ptr(d_ws),
                          _nbytes(d_ws), _stream(stream)), "snk_label")


def snk_run_workspace_bytes(dim, n_raw, spacing, p, max_cells) -> int:
    out = C.c_size_t()
    _check(_lib.snk_run_workspace_bytes(dim, _i64x3(n_raw), _f64x3(spacing), C.byref(p), max_cells,
                                        C.byref(out)), "snk_run_workspace_bytes")
    return out.value


def snk_ingest_u8(d_in, d_out, n, stream=None):
    _check(_lib.snk_ingest_u8(_ptr(d_in), _ptr(d_out), n, _stream(stream)), "snk_ingest_u8")


def snk_run_u8(dim, n_raw, spacing, p, h_raw, h_dets, det_cap, h_labels, max_cells, d_ws,
               stream=None) -> int:
    nd = C.c_int64()
    _check(_lib.snk_run_u8(dim, _i64x3(n_raw), _f64x3(spacing), C.byref(p), _ptr(h_raw), _ptr(h_dets),
                           det_cap, C.byref(nd), _ptr(h_labels), max_cells, _ptr(d_ws), _nbytes(d_ws),
                           _stream(stream)), "snk_run_u8")
    return nd.value


def snk_run(dim, n_raw, spacing, p, h_raw, h_dets, det_cap, h_labels, max_cells, d_ws,
            stream=None) -> int:
    nd = C.c_int64()
    _check(_lib.snk_run(dim, _i64x3(n_raw), _f64x3(spacing), C.byref(p), _ptr(h_raw), _ptr(h_dets),
                        det_cap, C.byref(nd), _ptr(h_labels), max_cells, _ptr(d_ws), _nbytes(d_ws),
                        _stream(stream)), "snk_run")
    return nd.value


def snk_run_batch_workspace_bytes(dim, n_raw, spacing, p, max_cells) -> int:
    n = (C.c_int64 * 3)(*[int(a) for a in n_raw])
    sp = (C.c_double * 3)(*[float(a) for a in spacing])
    out = C.c_size_t()
    _check(_lib.snk_run_batch_workspace_bytes(dim, n, sp, C.byref(p), max_cells, C.byref(out)),
           "snk_run_batch_workspace_bytes")
    return out.value


def snk_run_batch(dim, n_raw, spacing, p, h_raws, h_dets, det_cap, h_labels, max_cells, d_ws, stream=None):
    """h_raws / h_dets / h_labels: sequences of host buffers (one per volume; the
    same buffer may repeat); returns the detection counts."""
    k = len(h_raws)
    n = (C.c_int64 * 3)(*[int(a) for a in n_raw])
    sp = (C.c_double * 3)(*[float(a) for a in spacing])
    raws = (C.c_void_p * k)(*[_ptr(b) for b in h_raws])
    dets = (C.c_void_p * k)(*[_ptr(b) for b in h_dets])
    labs = (C.c_void_p * k)(*[_ptr(b) for b in h_labels]) if h_labels is not None else None
    nd = (C.c_int64 * max(k, 1))()
    _check(_lib.snk_run_batch(dim, n, sp, C.byref(p), k, raws, dets, det_cap, nd, labs, max_cells, _ptr(d_ws),
                              _nbytes(d_ws), _stream(stream)), "snk_run_batch")
    return [int(nd[i]) for i in range(k)]


# ---------------------------------------------------------------- struct helpers
def make_grid(dim: int, n, z_lo: int = 0, nz_buf: int | None = None, own=None,
              scale=(1.0, 1.0, 1.0)) -> snk_grid:
    """scale: physical voxel size per axis (anisotropic sampling without resampling, G28)."""
    g = snk_grid()
    g.scale[:] = [float(a) for a in scale]
    g.dim = dim
    g.n[:] = [int(a) for a in n]
    g.z_lo = z_lo
    g.nz_buf = int(n[2]) - z_lo if nz_buf is None else nz_buf
    own = (g.z_lo, g.z_lo + g.nz_buf) if own is None else own
    g.own_z0, g.own_z1 = int(own[0]), int(own[1])
    return g


def make_params(r0=10.0, *, delta_R=2.0, eps0=0.5, e0=-3.0, sigma=1.0, intensity_scale=1.0 / 257.0,
                max_step=1.0, r_min=1.0, r_max=None, leash=None, conv_tol=1e-3, max_iters=400,
                n_samples=1024, seed_mode=SEED_MAXIMA, seed_window=4, image_term=IMAGE_INTENSITY,
                cta_warps=0, seed_threshold=70 * 257, seed=1804063040,
                kernel_variant=0, estimator=EST_MC, cull_every=0) -> snk_params:
    """Defaults: DESIGN.md §3 (readings G2-G9, G18, G20)."""
    p = snk_params()
    p.r0, p.delta_R, p.eps0, p.e0, p.sigma = r0, delta_R, eps0, e0, sigma
    p.intensity_scale, p.max_step, p.r_min = intensity_scale, max_step, r_min
    p.r_max = 2 * r0 if r_max is None else r_max
    p.leash = 2 * r0 if leash is None else leash
    p.conv_tol, p.max_iters, p.n_samples = conv_tol, max_iters, n_samples
    p.seed_mode, p.seed_window, p.image_term, p.cta_warps = seed_mode, seed_window, image_term, cta_warps
    p.seed_threshold = seed_threshold
    p.kernel_variant = kernel_variant
    p.estimator = estimator
    p.cull_every = cull_every
    p.seed = seed & 0xFFFFFFFFFFFFFFFF
    return p
