"""Arithmetic-intensity estimators and the roofline model
(/root/reference/proj/include/tiler/analysis.hpp:1-84).

Pure host functions over a StencilSpec-like object (``ndims``, ``radii``,
``time_depth``, ``terms``), an IterationSpace-like object (``extents``) and a
TilePlan-like object (``time_tile``, ``space_tiles``).  Units follow the
reference: estimator internals in float32 elements, AI in flops/byte, 4 bytes
per element.

The GPU side of the same question -- how many DRAM bytes does one
point-update of *our* realisation move -- is ``traffic.py``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Sequence

ELEM_BYTES = 4


def _radii(spec) -> List[int]:
    r = spec.radii
    return list(r() if callable(r) else r)


def _flops(spec) -> int:
    # flops_per_point (stencil.hpp:107): k multiplies and k-1 adds
    terms = spec.terms() if callable(spec.terms) else spec.terms
    return 2 * len(terms) - 1


@dataclasses.dataclass
class MachineProfile:
    """stencil.hpp:65-70."""
    peak_gflops: float
    bandwidth_gbs: float
    cache_elems: int = 1
    elem_bytes: int = ELEM_BYTES


def bytes_per_point(spec) -> float:
    """Compulsory traffic per point-update: delta_t levels read + 1 written
    (analysis.hpp:31-32)."""
    return float((spec.time_depth + 1) * ELEM_BYTES)


def ai_spatial(spec) -> float:
    """analysis.hpp:38: flops_per_point / ((delta_t + 1) * 4)."""
    return _flops(spec) / bytes_per_point(spec)


def naive_from_spatial(ai: float, time_tile: int) -> float:
    return ai * time_tile


def ai_naive_tt(spec, time_tile: int) -> float:
    """analysis.hpp:41: the spatial estimate scaled by the time tile."""
    if time_tile < 1:
        raise ValueError("time_tile < 1")
    return naive_from_spatial(ai_spatial(spec), time_tile)


def face_sizes(spec, extents: Sequence[int], time_tile: int, tiles: Sequence[int]) -> List[int]:
    """analysis.hpp:47-49: F_i = t_t * 2 * (prod_{j<i} t_j) * delta_i *
    (prod_{k>i} D_k) elements, loop order d_1 outer .. d_n inner."""
    r = _radii(spec)
    n = len(extents)
    out = []
    for i in range(n):
        f = time_tile * 2 * r[i]
        for j in range(i):
            f *= tiles[j]
        for k in range(i + 1, n):
            f *= extents[k]
        out.append(int(f))
    return out


def boundary_fracs(spec, extents: Sequence[int], tiles: Sequence[int]) -> List[float]:
    """analysis.hpp:51-53: frac_i = min(1, 2 * (delta_i / D_i) * floor(D_i / t_i))."""
    r = _radii(spec)
    return [min(1.0, 2.0 * (r[i] / extents[i]) * (extents[i] // tiles[i])) for i in range(len(extents))]


def union_frac(fracs: Sequence[float]) -> float:
    """analysis.hpp:55-58: 1 - prod(1 - f_j) (pairwise inclusion-exclusion for two)."""
    p = 1.0
    for f in fracs:
        p *= 1.0 - f
    return 1.0 - p


@dataclasses.dataclass
class IntensityEstimate:
    flops_per_point: int
    bytes_per_point: float
    ai_spatial: float
    ai_naive_tt: float
    ai_tight_tt: float
    divisor: float


@dataclasses.dataclass
class FaceAnalysis:
    face_sizes: List[int]
    boundary_fracs: List[float]
    union_frac: float
    bcase: str           # "empty" | "f1_only" | "multi"
    critical_dim: int    # i* (1-based), 0 when no face reaches the cache size


def tight_bound(spec, extents: Sequence[int], time_tile: int, tiles: Sequence[int], cache_elems: int):
    """analysis.hpp:60-70 / SPEC.md:470-478.  i* = the largest i with
    F_i >= cache_elems.  None: the tight estimate equals the naive one.
    i* = 1: |B| = (F_1 - cache_elems) * floor(D_1 / t_1).  i* >= 2:
    B = B_1 u .. u B_{i*-1}.  The naive estimate is divided by 1 + |B|/prod(D)."""
    if cache_elems < 1:
        raise ValueError("cache_elems < 1")
    F = face_sizes(spec, extents, time_tile, tiles)
    fr = boundary_fracs(spec, extents, tiles)
    istar = 0
    for i, f in enumerate(F, start=1):
        if f >= cache_elems:
            istar = i
    if istar == 0:
        u, case = 0.0, "empty"
    elif istar == 1:
        vol = math.prod(extents)
        u, case = min(1.0, (F[0] - cache_elems) * (extents[0] // tiles[0]) / vol), "f1_only"
    else:
        u, case = union_frac(fr[: istar - 1]), "multi"
    naive = ai_naive_tt(spec, time_tile)
    est = IntensityEstimate(_flops(spec), bytes_per_point(spec), ai_spatial(spec), naive, naive / (1.0 + u), 1.0 + u)
    return est, FaceAnalysis(F, fr, u, case, istar)


def roofline_bound(profile: MachineProfile, ai: float) -> float:
    """analysis.hpp:77-79: min(peak, bandwidth * ai) in GFlop/s."""
    if ai <= 0:
        raise ValueError("ai <= 0")
    return min(profile.peak_gflops, profile.bandwidth_gbs * ai)


def ridge_point(profile: MachineProfile) -> float:
    """analysis.hpp:81-82: peak / bandwidth."""
    if profile.bandwidth_gbs <= 0:
        raise ValueError("bandwidth <= 0")
    return profile.peak_gflops / profile.bandwidth_gbs
