"""GPU autotuner for the executor's runtime tile parameters.

Restates the reference autotune module for the B200:
``tune(spec, space, search, cost)`` evaluates every plan of a Cartesian
``SearchSpace``; the wall_time cost of a plan is the minimum over R trials
("the reported figure will be the minimum"), here device
time measured with CUDA events by ``st_apply``; ties go to the
lexicographically smallest plan.  The skew is not searched (the paper found
the minimum legal skew best).

The searched parameters are exactly the ones the executor takes at run
time: schedule (untiled sweep or time-tiled wavefront), time tile T, the
d_1 tile (z-chunk planes of the wavefront), the d_2 tile (CTA tile height,
selecting one of the compiled tile shapes) and, with --fused, the on-chip
realisations of the time tile (st_plan.fused_levels: F levels per pass in
3-D, levels per halo exchange of the SM-resident 2-D kernel).

  python -m paper_1806_08299_b200.autotune --config 2 [--trials 3] [--quick]
"""
from __future__ import annotations

import argparse
import dataclasses
import itertools
import json
import sys
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import configs as CF
from . import tiler as P


@dataclasses.dataclass(frozen=True)
class Candidate:
    schedule: str          # "canonical" | "time"
    time_tile: int
    cz: int                # d_1 tile (planes per wavefront chunk); 0 = auto
    ty: int                # d_2 tile (CTA tile rows); 0 = default
    mode: int = P.MODE_REFERENCE
    fused: int = 0         # st_plan.fused_levels (0 = wavefront)

    def key(self) -> Tuple:
        return (self.schedule != "canonical", self.fused, self.time_tile, self.cz, self.ty, self.mode)


@dataclasses.dataclass
class SearchSpace:
    time_tiles: Sequence[int] = (1, 2, 4, 8, 16, 32)
    chunks: Sequence[int] = (64, 128, 256, 384)
    tile_rows: Sequence[int] = (8, 16, 24, 32)
    include_canonical: bool = True
    modes: Sequence[int] = (P.MODE_REFERENCE,)
    trials: int = 3
    fused_levels: Sequence[int] = ()   # on-chip realisations to try besides the wavefront

    def candidates(self, steps: int) -> List[Candidate]:
        out = []
        for m in self.modes:
            if self.include_canonical:
                for ty in self.tile_rows:
                    out.append(Candidate("canonical", 1, 0, ty, m))
            for T, cz, ty in itertools.product(self.time_tiles, self.chunks, self.tile_rows):
                if T <= steps:
                    out.append(Candidate("time", T, cz, ty, m))
            for F, ty in itertools.product(self.fused_levels, self.tile_rows):
                if 1 <= F <= steps:   # the fused pass needs no z-chunk; T = F sizes the slots
                    out.append(Candidate("time", F, 0, ty, m, F))
        return out


@dataclasses.dataclass
class TuneResult:
    best: Candidate
    best_cost: float
    table: List[Tuple[Candidate, float]]

    def to_json(self):
        return {"best": dataclasses.asdict(self.best), "best_cost_s": self.best_cost,
                "table": [dict(dataclasses.asdict(c), cost_s=v) for c, v in self.table]}


def _nest(spec: P.StencilSpec, radius: int, c: Candidate, ndims: int) -> P.LoopNest:
    canon = P.build_canonical_nest(spec, None)
    tiles = (c.cz, c.ty, 0)[:ndims] if ndims == 3 else (c.cz,) + (0,) * (ndims - 1)
    if c.schedule == "canonical":
        return P.LoopNest(P.SCHED_CANONICAL, P.TilePlan(0, 1, tiles))
    return P.tile_time(canon, spec, None, P.TilePlan(radius, c.time_tile, tiles, fused_levels=c.fused))


def tune(dg: P.DeviceGrid, spec: P.StencilSpec, radius: int, ndims: int, steps: int, last_level: int,
         search: SearchSpace, flush_l2: bool = True) -> TuneResult:
    """wall_time cost: every candidate runs `steps` levels
    continuing the device grid (the cost of a plan does not depend on the
    data), min over `trials` of the device time, L2 overwritten before each
    trial so no plan is timed on its predecessor's resident data."""
    table = []
    t = last_level - spec.time_depth + 1
    for c in search.candidates(steps):
        nest = _nest(spec, radius, c, ndims)
        dg.apply(t, t + steps, nest, c.mode)      # warm-up (module load, tensor maps)
        t += steps
        best = float("inf")
        for _ in range(max(1, search.trials)):
            if flush_l2:
                dg.ctx.flush_l2()
            rep = dg.apply(t, t + steps, nest, c.mode)
            t += steps
            best = min(best, rep.device_seconds)
        table.append((c, best))
    best_c, best_v = min(table, key=lambda cv: (cv[1], cv[0].key()))
    return TuneResult(best_c, best_v, table)


# ---------------------------------------------- sim_traffic (host-only) ---
@dataclasses.dataclass
class HostSearchSpace:
    """SearchSpace of SPEC.md:531-534: time tiles {1,2,4,8,16} within [1, D_t];
    per dimension the powers of two in [2, D_i], plus D_i itself for the
    innermost; skew fixed at min_skew_factor."""
    time_tiles: Sequence[int] = (1, 2, 4, 8, 16)
    space_tiles: Optional[Sequence[Sequence[int]]] = None   # per dim; None = the SPEC default

    def plans(self, spec: P.StencilSpec, space: P.IterationSpace) -> List[P.TilePlan]:
        D = list(space.extents)
        tts = [t for t in self.time_tiles if 1 <= t <= space.time_steps]
        if self.space_tiles is not None:
            per = [list(v) for v in self.space_tiles]
        else:
            per = []
            for i, d in enumerate(D):
                v = [1 << k for k in range(1, 64) if (1 << k) <= d]
                if i == len(D) - 1 and d not in v:
                    v.append(d)
                per.append(v or [d])
        if not tts or any(not v for v in per):
            raise P.Error("empty search space")
        s = P.min_skew_factor(spec)
        return [P.TilePlan(s, tt, tuple(ts)) for tt in tts for ts in itertools.product(*per)]


def plan_key(plan: P.TilePlan) -> Tuple:
    """Lexicographic tie order (t_t, t_1, ..., t_n)."""
    return (plan.time_tile,) + tuple(plan.space_tiles)


def tune_sim(spec: P.StencilSpec, space: P.IterationSpace, search: HostSearchSpace,
             cache: P.CacheConfig) -> Tuple[P.TilePlan, int, List[Tuple[P.TilePlan, int]]]:
    """tune(spec, space, search, sim_traffic): every plan of
    the Cartesian space as a time-tiled nest, cost = simulated bytes (one
    deterministic evaluation), argmin with lexicographic ties.  Returns
    (best plan, best bytes, table)."""
    canon = P.build_canonical_nest(spec, space)
    table = []
    for plan in search.plans(spec, space):
        rep = P.simulate(P.tile_time(canon, spec, space, plan), spec, space, cache)
        table.append((plan, rep.bytes))
    best, cost = min(table, key=lambda pc: (pc[1], plan_key(pc[0])))
    return best, cost, table


def _search(args) -> SearchSpace:
    fused = tuple(int(f) for f in args.fused_levels.split(",")) if args.fused_levels else ()
    if args.quick:
        return SearchSpace(time_tiles=(4, 16, 32), chunks=(128, 384), tile_rows=(16, 24, 32), trials=args.trials,
                           fused_levels=fused)
    return SearchSpace(trials=args.trials, fused_levels=fused)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--trials", type=int, default=3)
    ap.add_argument("--quick", action="store_true", help="small search space")
    ap.add_argument("--fast", action="store_true", help="also search FAST mode")
    ap.add_argument("--fused-levels", type=str, default="",
                    help="comma list of st_plan.fused_levels to search besides the wavefront, e.g. 2,3")
    args = ap.parse_args(argv)
    cfg = CF.get(args.config)
    spec = P.StencilSpec.make(cfg.name, cfg.ndims, [P.StencilTerm(c, dt, o) for c, dt, o in cfg.terms], model=cfg.model)
    ctx = P.Context(0)
    search = _search(args)
    slots = spec.time_depth + max(list(search.time_tiles) + list(search.fused_levels))   # deepest required_slots
    space = P.IterationSpace(cfg.steps, cfg.extents)
    grid = (P.init_unit(spec, space, CF.SEED_FIELD, slots) if cfg.init == "unit"
            else P.init_gaussian(spec, space, slots, cfg.sigma, [e // 2 for e in cfg.extents]))
    dg = P.DeviceGrid(ctx, spec, cfg.extents, slots)
    dg.upload(grid.data, spec.time_depth - 1, uniform_halo=True)
    if cfg.field:
        m = np.empty(int(np.prod(cfg.extents)), np.float32)
        lib = P._lib()
        ext = P.N.i64array(cfg.extents)
        if cfg.field == "layered":
            lib.st_field_layered(3, ext, P._fptr(m), cfg.v_top, cfg.v_bottom, cfg.extents[0] // 2, cfg.dt, CF.H, 0)
        else:
            lib.st_field_random_smoothed(3, ext, P._fptr(m), CF.SEED_VELOCITY, cfg.vmin, cfg.vmax, cfg.dt, CF.H)
        dg.set_field(m)
    if args.fast and cfg.model == 0:
        search.modes = (P.MODE_REFERENCE, P.MODE_FAST)
    res = tune(dg, spec, cfg.radius, cfg.ndims, cfg.steps, spec.time_depth - 1, search)
    pts = cfg.steps * int(np.prod(cfg.extents))
    out = res.to_json()
    out["config"] = cfg.index
    out["best_gpts"] = pts / res.best_cost / 1e9
    for row in out["table"]:
        row["gpts"] = pts / row["cost_s"] / 1e9
    print(json.dumps(out))
    dg.close()
    ctx.close()


if __name__ == "__main__":
    sys.exit(main())
