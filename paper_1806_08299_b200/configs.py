"""The five BASELINE.json configurations, fixed once.

Axis mapping (ledger A.1): reference d_1 = z (slowest, sharded), d_2 = y,
d_3 = x (contiguous).  Coefficients are folded in double and cast once
(A.2); term order is centre, then per axis d_1..d_n: -1, +1, -2, +2, ...
The wave model (A.3) is u' = (2u - u_prev) + m * lap with m = (c dt / h)^2.
Seeds are chosen here and recorded (BASELINE.json leaves them open).
"""
from __future__ import annotations

import dataclasses
from fractions import Fraction
from math import factorial
from typing import List, Optional, Sequence, Tuple

import numpy as np

SEED_FIELD = 1806       # interior [0,1) LCG seed (heat configs)
SEED_VELOCITY = 8299    # config 4 velocity LCG seed
H = 10.0                # grid spacing, m


def star_terms(ndims: int, centre: float, weights: Sequence[float]) -> List[Tuple[float, int, Tuple[int, ...]]]:
    """Canonical star order: centre, then per axis d_1..d_n, -k before +k."""
    terms = [(float(np.float32(centre)), 1, (0,) * ndims)]
    for a in range(ndims):
        for k, w in enumerate(weights, start=1):
            for sgn in (-1, 1):
                off = [0] * ndims
                off[a] = sgn * k
                terms.append((float(np.float32(w)), 1, tuple(off)))
    return terms


def fd2_weights(order: int) -> List[Fraction]:
    """Central 2nd-derivative weights w_0..w_r, r = order/2 (exact):
    w_k = 2(-1)^{k+1} (r!)^2 / (k^2 (r-k)! (r+k)!), w_0 = -2 sum w_k."""
    r = order // 2
    w = [Fraction(2 * (-1) ** (k + 1) * factorial(r) ** 2, k * k * factorial(r - k) * factorial(r + k))
         for k in range(1, r + 1)]
    return [-2 * sum(w)] + w


@dataclasses.dataclass
class Config:
    index: int
    name: str
    ndims: int
    model: int              # 0 = terms (heat), 1 = wave
    extents: Tuple[int, ...]
    steps: int
    terms: List[Tuple[float, int, Tuple[int, ...]]]
    radius: int
    skew: int
    time_tiles: Tuple[int, ...]
    space_tiles: Tuple[int, ...]
    init: str               # "unit" | "gaussian"
    field: Optional[str] = None   # None | "layered" | "random"
    dt: float = 0.0
    v_top: float = 0.0
    v_bottom: float = 0.0
    vmin: float = 0.0
    vmax: float = 0.0
    sigma: float = 5.0
    bytes_per_point: int = 8
    sharded: bool = False

    def scaled(self, extents: Sequence[int], steps: int) -> "Config":
        """Same stencil / init rules on a smaller (parity-test) grid."""
        return dataclasses.replace(self, extents=tuple(int(e) for e in extents), steps=int(steps))


def heat2d_so2() -> Config:
    # folded centre 1 - 4*0.2 in double, cast once (ledger A.2)
    return Config(1, "heat2d_so2", 2, 0, (1024, 1024), 100, star_terms(2, 1.0 - 4 * 0.2, [0.2]), 1, 1,
                  (8,), (64, 64), "unit")


def heat3d_so4() -> Config:
    a = 0.1
    centre = 1.0 + a * 3 * (-5.0 / 2.0)
    w = [a * 4.0 / 3.0, a * (-1.0 / 12.0)]
    return Config(2, "heat3d_so4", 3, 0, (256, 256, 256), 64, star_terms(3, centre, w), 2, 2,
                  (1, 4, 8, 16), (0, 32, 64), "unit")


def wave3d(order: int, n: int = 512) -> Config:
    w = fd2_weights(order)
    centre = 3 * float(w[0])
    terms = star_terms(3, centre, [float(x) for x in w[1:]])
    r = order // 2
    return terms, r


def wave3d_so8() -> Config:
    terms, r = wave3d(8)
    dt = 0.4 * H / 3000.0
    return Config(3, "wave3d_so8", 3, 1, (512, 512, 512), 200, terms, r, r, (1, 2, 4), (0, 32, 64), "gaussian",
                  field="layered", dt=dt, v_top=1500.0, v_bottom=3000.0, bytes_per_point=16)


def wave3d_so16() -> Config:
    terms, r = wave3d(16)
    dt = 0.4 * H / 4500.0
    return Config(4, "wave3d_so16", 3, 1, (512, 512, 512), 100, terms, r, r, (1, 2), (0, 32, 32), "gaussian",
                  field="random", dt=dt, vmin=1500.0, vmax=4500.0, bytes_per_point=16)


def wave3d_so8_weak(G: int = 1) -> Config:
    terms, r = wave3d(8)
    dt = 0.4 * H / 3000.0
    return Config(5, "wave3d_so8_weak", 3, 1, (512 * G, 1024, 1024), 200, terms, r, r, (1, 2, 4), (0, 32, 64),
                  "gaussian", field="layered", dt=dt, v_top=1500.0, v_bottom=3000.0, bytes_per_point=16,
                  sharded=True)


def heat3d_so2() -> Config:
    # Study workload beyond BASELINE's five configs (same operator family as
    # configs 1-2: the 7-point 3-D Laplacian smoother, kappa*dt/h^2 = 0.15,
    # stable below 1/6): the radius at which the on-chip fused realisation
    # pays most.  bench.py --config 6.
    a = 0.15
    return Config(6, "heat3d_so2", 3, 0, (512, 512, 512), 48, star_terms(3, 1.0 - 6 * a, [a]), 1, 1,
                  (1, 3), (0, 24, 0), "unit")


def wave3d_so2() -> Config:
    # Study workload beyond BASELINE's five configs: config 3's leapfrog
    # (layered velocity, Gaussian pulse, dt at CFL 0.4) at space order 2 --
    # the radius at which the fused wave realisation pays.
    terms, r = wave3d(2)
    dt = 0.4 * H / 3000.0
    return Config(7, "wave3d_so2", 3, 1, (512, 512, 512), 48, terms, r, r, (1, 3), (0, 16, 0), "gaussian",
                  field="layered", dt=dt, v_top=1500.0, v_bottom=3000.0, bytes_per_point=16)


CONFIGS = {1: heat2d_so2, 2: heat3d_so4, 3: wave3d_so8, 4: wave3d_so16, 5: wave3d_so8_weak, 6: heat3d_so2,
           7: wave3d_so2}


def get(index: int, **kw) -> Config:
    return CONFIGS[index](**kw)


# Tuned executor plans per config (B200; scratch sweeps + autotune.py, see
# DESIGN.md section 5).  bench.py runs these; tests/test_gpu_fullsize.py checks
# every FAST plan here against the 1e-5 tolerance at full size.
#  * config 2: one skewed wavefront over 32 levels, z-chunks longer than the
#    skewed extent (nz + 2*31 = 318 -> one chunk per level), 32-row tiles.
#    FAST is within tolerance over the full run (diffusion damps rounding).
#  * wave configs: FAST stays within 1e-5 over the full runs -- so16 with paired
#    symmetric taps (5.2e-6), so8 with the ordered hybrid (4.5e-6; pairing its
#    taps drifted 1.29e-5) -- so the bench runs them FAST and times the
#    bit-exact mode beside it ("bit_exact" in the JSON line).
BENCH_PLANS = {
    1: dict(time_tile=4, mode="reference", schedule="time", fused=16),  # SM-resident 2-D tiles, 16 levels per exchange
    # FAST: 32-row V4 tile; bit-exact (--mode reference): 24-row V8, 12 warps x 2 rows
    2: dict(time_tile=32, mode="fast", schedule="time", tiles=(320, 32, 0), tiles_reference=(320, 24, 0)),
    3: dict(time_tile=8, mode="fast", schedule="time", tiles=(512, 24, 0)),   # 24-row tile (12 warps x 2 rows), m as 1-byte codes
    4: dict(time_tile=4, mode="fast", schedule="time", tiles=(512, 12, 0)),   # 12 warps x 1 row
    5: dict(time_tile=4, mode="reference", schedule="canonical"),
    # study (not in BASELINE): 3 levels per pass on-chip, 24-row output tiles
    6: dict(time_tile=3, mode="fast", schedule="time", tiles=(0, 24, 0), fused=3, tiles_reference=(0, 0, 0)),
    # study (not in BASELINE): the so2 leapfrog, 3 levels per pass on-chip, bit-exact
    7: dict(time_tile=3, mode="reference", schedule="time", tiles=(0, 16, 0), fused=3),
}


# Plans of the z-slab (sharded) runs: one wavefront launch per time tile over
# the trapezoid of slab ranges, ghost depth r*T per side exchanged per tile.
# T trades exchange count against redundant ghost compute (~r(T-1)/2 planes
# per side per level).  z-chunk 4096 = one chunk per level (clipped).
DIST_PLANS = {
    2: dict(time_tile=8, mode="fast", schedule="time", tiles=(4096, 32, 0)),
    # 24-row tile (12 warps x 2 rows).  FAST is DRAM-bound at full clock: z-chunks of 256 planes keep
    # y-neighbour tiles (8 tickets apart on 1024-wide rows) within a few planes of each other, so the shared
    # halo rows come from L2 (415 -> 478 GPts/s at full clock); bit-exact is compute-bound: whole-depth items
    5: dict(time_tile=4, mode="fast", schedule="time", tiles=(256, 24, 0), tiles_reference=(4096, 24, 0)),
}


def sharded(index: int, world: int) -> "Config":
    """The weak-scaled global problem of `world` z-slabs: config 5 as defined
    (512 planes per GPU); any other config stacks `world` copies of its grid
    along d_1 (z-slabs of the single-GPU extent)."""
    if index == 5:
        return wave3d_so8_weak(world)
    c = get(index)
    return dataclasses.replace(c, extents=(c.extents[0] * world,) + tuple(c.extents[1:]), sharded=True)
