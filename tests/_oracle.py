"""ctypes wrapper of oracle/build/liboracle.so -- the CPU restatement of the
reference executor (TEST INFRASTRUCTURE: the checker, never the product).
Builds the library with `make -C oracle` on first use if it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "oracle", "build", "liboracle.so")

CANONICAL, SPACE, TIME, REMAINDER = 0, 1, 2, 3
OK, EINVAL, EILLEGAL, ESLOTS = 0, 1, 2, 3


class or_term(C.Structure):
    _fields_ = [("coeff", C.c_float), ("dt", C.c_int), ("off", C.c_int * 3)]


class or_spec(C.Structure):
    _fields_ = [("ndims", C.c_int), ("model", C.c_int), ("nterms", C.c_int), ("terms", C.POINTER(or_term))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
        L = C.CDLL(LIB)
        I64P, FP, SP = C.POINTER(C.c_int64), C.POINTER(C.c_float), C.POINTER(or_spec)
        sig = {
            "or_time_depth": (C.c_int, [SP]),
            "or_radius": (C.c_int, [SP, C.c_int]),
            "or_flops_per_point": (C.c_int64, [SP]),
            "or_validate": (C.c_int, [SP]),
            "or_plane": (C.c_int64, [SP, I64P]),
            "or_init_reference": (None, [SP, I64P, FP, C.c_int64, C.c_uint64]),
            "or_init_unit": (None, [SP, I64P, FP, C.c_int64, C.c_uint64]),
            "or_init_gaussian": (None, [SP, I64P, FP, C.c_int64, C.c_double, I64P]),
            "or_mfield_layered": (None, [C.c_int, I64P, FP, C.c_double, C.c_double, C.c_int64, C.c_double, C.c_double]),
            "or_mfield_random_smoothed": (None, [C.c_int, I64P, FP, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double]),
            "or_lcg_reference": (None, [C.c_uint64, C.c_int64, FP]),
            "or_check_legality": (C.c_int, [SP, C.c_int, C.POINTER(C.c_int)]),
            "or_execute": (C.c_int, [SP, I64P, FP, C.c_int64, C.c_int64, C.c_int64, FP, C.c_int, C.c_int, C.c_int64,
                                     I64P, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
            "or_verify_bitwise": (C.c_int, [SP, I64P, FP, C.c_int64, FP, C.c_int64, C.c_int64, C.c_int64]),
            "or_max_rel_err": (C.c_double, [SP, I64P, FP, C.c_int64, FP, C.c_int64, C.c_int64, C.c_int64]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _fp(a: Optional[np.ndarray]):
    if a is None:
        return C.cast(C.c_void_p(0), C.POINTER(C.c_float))
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i64(vals: Sequence[int]):
    a = (C.c_int64 * 3)(1, 1, 1)
    for i, v in enumerate(vals):
        a[i] = int(v)
    return a


class Spec:
    """Terms: list of (coeff, dt, offsets)."""

    def __init__(self, ndims: int, terms, model: int = 0):
        self.ndims, self.model = ndims, model
        self._terms = (or_term * len(terms))()
        for k, (c, dt, off) in enumerate(terms):
            self._terms[k].coeff = float(c)
            self._terms[k].dt = int(dt)
            for i, o in enumerate(off):
                self._terms[k].off[i] = int(o)
        self.s = or_spec(ndims, model, len(terms), self._terms)
        self.terms = list(terms)

    @property
    def ref(self):
        return C.byref(self.s)

    @property
    def time_depth(self) -> int:
        return lib().or_time_depth(self.ref)

    def radius(self, d: int) -> int:
        return lib().or_radius(self.ref, d)

    def flops(self) -> int:
        return lib().or_flops_per_point(self.ref)

    def plane(self, extents) -> int:
        return lib().or_plane(self.ref, _i64(extents))

    def padded(self, extents) -> Tuple[int, ...]:
        return tuple(int(e) + 2 * self.radius(i) for i, e in enumerate(extents))


def new_grid(spec: Spec, extents, slots: int) -> np.ndarray:
    return np.zeros(slots * spec.plane(extents), dtype=np.float32)


def init_reference(spec, extents, slots, seed) -> np.ndarray:
    g = new_grid(spec, extents, slots)
    lib().or_init_reference(spec.ref, _i64(extents), _fp(g), slots, seed)
    return g


def init_unit(spec, extents, slots, seed) -> np.ndarray:
    g = new_grid(spec, extents, slots)
    lib().or_init_unit(spec.ref, _i64(extents), _fp(g), slots, seed)
    return g


def init_gaussian(spec, extents, slots, sigma, centre) -> np.ndarray:
    g = new_grid(spec, extents, slots)
    lib().or_init_gaussian(spec.ref, _i64(extents), _fp(g), slots, sigma, _i64(centre))
    return g


def mfield_layered(extents, v_top, v_bottom, split, dt, h) -> np.ndarray:
    m = np.zeros(int(np.prod(extents)), dtype=np.float32)
    lib().or_mfield_layered(len(extents), _i64(extents), _fp(m), v_top, v_bottom, split, dt, h)
    return m


def mfield_random(extents, seed, vmin, vmax, dt, h) -> np.ndarray:
    m = np.zeros(int(np.prod(extents)), dtype=np.float32)
    lib().or_mfield_random_smoothed(len(extents), _i64(extents), _fp(m), seed, vmin, vmax, dt, h)
    return m


def lcg_reference(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.float32)
    lib().or_lcg_reference(seed, n, _fp(out))
    return out


def execute(spec, extents, grid, slots, t_begin, t_end, mfield=None, schedule=CANONICAL, skew=0,
            time_tile=1, tiles=None, reverse_parallel=False, nthreads=1):
    """Returns (status, wall_seconds, points)."""
    secs = C.c_double()
    pts = C.c_int64()
    tl = _i64(tiles) if tiles is not None else None
    rc = lib().or_execute(spec.ref, _i64(extents), _fp(grid), slots, t_begin, t_end, _fp(mfield), schedule, skew,
                          time_tile, tl, 1 if reverse_parallel else 0, nthreads, C.byref(secs), C.byref(pts))
    return rc, secs.value, pts.value


def verify_bitwise(spec, extents, a, sa, b, sb, last_level, levels) -> int:
    return lib().or_verify_bitwise(spec.ref, _i64(extents), _fp(a), sa, _fp(b), sb, last_level, levels)


def max_rel_err(spec, extents, a, sa, b, sb, last_level, levels) -> float:
    return lib().or_max_rel_err(spec.ref, _i64(extents), _fp(a), sa, _fp(b), sb, last_level, levels)


def uniform_halo(spec, extents, grid, slots) -> np.ndarray:
    """Copy slot 0's halo cells into every other slot (interiors untouched),
    so that results do not depend on the slot count (see DESIGN.md ledger)."""
    P = spec.padded(extents)
    v = grid.reshape((slots,) + P)
    R = [spec.radius(i) for i in range(spec.ndims)]
    mask = np.ones(P, dtype=bool)
    mask[tuple(slice(r, r + e) for r, e in zip(R, extents))] = False
    for s in range(1, slots):
        v[s][mask] = v[0][mask]
    return grid
