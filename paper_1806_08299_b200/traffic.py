"""DRAM bytes per point-update of the B200 realisations -- the GPU analogue of
the reference's traffic models (analysis.hpp:47-75 tight_bound: re-loaded
tile faces; cache_sim.hpp:28-34: an LRU replay), SURVEY.md 8(f)3.

A point-update of level L reads its input levels and writes one level.  On
the B200 three things move the DRAM bytes away from that compulsory count:

* tile faces (the halo of the TMA box: ``halo_factor``) -- re-read from DRAM
  when the neighbouring tile's lines have left L2 in between.  KAPPA is the
  fraction of face bytes that miss; one constant for every realisation,
  fitted to the star-kernel measurements in profiles/traffic.json (0.17 to
  0.46 observed);
* reuse of level L's output by level L+1 through L2 (the wavefront): the
  data written between a plane's write and its read by the next level is
  ``lag_bytes`` = (items of one level / CTA slots) x one item's z-stream x
  every slot's tile-plane bytes; the reuse fraction is exp(-lag / L2),
  an LRU-like decay in the reuse distance;
* on-chip levels (fused passes, the SM-resident grid): F levels per pass
  over memory.

``predict`` returns the point estimate; tests/test_traffic_model.py checks it
against every ncu measurement recorded in profiles/traffic.json.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

ELEM = 4
KAPPA = 0.4                 # fraction of tile-face (halo) bytes re-read from DRAM
L2_BYTES = 126 * 2 ** 20    # B200 L2 (cudaDevAttrL2CacheSize)
TX = 128                    # every compiled tile is 128 x (rows)


@dataclasses.dataclass
class Plan:
    """What the model needs of a realisation."""
    kind: str                 # "sweep" | "wavefront" | "fused" | "resident"
    extents: tuple            # (nz, ny, nx) (3-D) or (nz, nx) (2-D)
    radius: int
    wave: bool                # leapfrog: reads u^n and u^{n-1} (+ m), writes u^{n+1}
    rows: int = 16            # CTA tile rows (TY)
    m_bytes: int = 4          # wave coefficient field: 4 (float) or 1 (palette codes)
    levels_per_pass: int = 1  # fused F / resident levels per launch
    time_tile: int = 1        # wavefront T
    slots: int = 148          # resident CTAs (SMs x CTAs per SM)
    cz: Optional[int] = None  # wavefront z-chunk (None = whole depth)


def halo_factor(p: Plan) -> float:
    """TMA box / output tile of one plane (x halo rounded up to float4s)."""
    r = p.radius
    xh = (r + 3) // 4 * 4
    if p.kind == "fused":
        F = p.levels_per_pass
        hx = (r * (F - 1) + 3) // 4 * 4
        bw, bh = TX + 2 * hx + 2 * xh, p.rows + 2 * r * (F - 1) + 2 * r
    else:
        bw, bh = TX + 2 * xh, p.rows + 2 * r
    return bw * bh / (TX * p.rows)


def compute_grid_factor(p: Plan) -> float:
    """Fused wave passes read u^{n-1} and m over the level-1 compute grid."""
    if p.kind != "fused":
        return 1.0
    F, r = p.levels_per_pass, p.radius
    hx = (r * (F - 1) + 3) // 4 * 4
    return (TX + 2 * hx) * (p.rows + 2 * r * (F - 1)) / (TX * p.rows)


def lag_bytes(p: Plan) -> float:
    """L2 bytes written between level L's write of a plane and level L+1's
    read of it (wavefront ticket order: one level's items, then the next)."""
    nz = p.extents[0]
    plane_pts = math.prod(p.extents[1:])
    items = math.ceil(plane_pts / (TX * p.rows))
    cz = min(nz, p.cz) if p.cz else nz
    busy = min(p.slots, items * p.time_tile)
    # the next level's item for a column starts items/slots item-durations
    # later; meanwhile every busy slot streams tile planes (read + write)
    planes_between = cz * items / p.slots
    return planes_between * busy * TX * p.rows * ELEM * 2


def reuse_fraction(p: Plan) -> float:
    if p.kind != "wavefront" or p.time_tile <= 1:
        return 0.0
    return math.exp(-lag_bytes(p) / L2_BYTES)


def predict(p: Plan) -> float:
    """DRAM bytes per point-update."""
    if p.kind == "resident":
        # the grid lives in shared memory for the whole run: the input level
        # is read once per launch of p.levels_per_pass levels; the output
        # level (4 MiB for config 1) is still in the write-back L2 when the
        # launch ends, so DRAM sees it only later
        return ELEM / p.levels_per_pass
    h = 1.0 + KAPPA * (halo_factor(p) - 1.0)
    if p.kind == "fused":
        F = p.levels_per_pass
        g = 1.0 + KAPPA * (compute_grid_factor(p) - 1.0)
        reads = ELEM * h + ((ELEM + p.m_bytes) * g if p.wave else 0.0)
        writes = ELEM * (2 if p.wave and F > 1 else 1)
        return (reads + writes) / F
    rho = reuse_fraction(p)
    reads = ELEM * h + ((ELEM + p.m_bytes) if p.wave else 0.0)
    return ELEM + reads * (1.0 - rho)
