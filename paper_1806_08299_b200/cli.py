"""Command-line front end over the B200 executor (the
reference's `cli` module), for the subcommands on the executor path:

  python -m paper_1806_08299_b200.cli run    <spec> --mode M [--tiles a,b,c] [--time-tile k] [--skew s] [--seed S]
  python -m paper_1806_08299_b200.cli verify <spec> --mode M [...]          -> {"bitwise_equal": bool}
  python -m paper_1806_08299_b200.cli tune   <spec> [--cost time|traffic] [--trials R] [--cache-elems W]
                                             [--fused-levels 2,4]
  python -m paper_1806_08299_b200.cli transform <spec> --mode M [...] [-o out.c]   (C99, codegen.py)
  python -m paper_1806_08299_b200.cli analyze  <spec> --tiles a,b --time-tile k [--cache-elems W]
                                             [--profile peak,bw]
  python -m paper_1806_08299_b200.cli simulate <spec> --mode M [...] [--cache-elems W] [--line-elems L]

M in {none, space, space-remainder, time}.  Executor extensions: --arith
{reference,fast} (st_mode) and --fused F (st_plan.fused_levels).  Every JSON
output is one object on stdout; diagnostics go to stderr.  Exit codes as the
reference: 2 on parse / flag / legality errors, 1 on a verification
failure, 0 on success.  `transform` emits the nest as C99 (codegen.py,
SPEC.md:574-609).  `analyze` (analysis.py: the reference's AI estimators and
roofline) and `simulate` (st_simulate: the LRU cache model over the nest's
access stream) are host-only models; `tune --cost traffic` searches the
reference's plan space with the simulated bytes (deterministic), `--cost
time` times the B200 realisations (min over trials, L2 flushed).
Default cache size: 5 242 880 elements (the thesis machine's 20 MB L3,
SPEC.md cli ledger).

The spec file format is the reference's, parsed by
st_stencil_parse (stencil.hpp:87-97).  Grids are initialised with the
reference init_grid (executor.hpp:87-90).
"""
from __future__ import annotations

import argparse
import json
import sys
from typing import List, Optional

from . import tiler as P

MODES = ("none", "space", "space-remainder", "time")
EXECUTOR_SUBCOMMANDS = ("run", "verify", "tune", "transform", "analyze", "simulate")
DEFAULT_CACHE_ELEMS = 5_242_880


class UsageError(Exception):
    pass


def _ints(text: Optional[str]) -> List[int]:
    if not text:
        return []
    try:
        return [int(t) for t in text.split(",")]
    except ValueError:
        raise UsageError(f"bad integer list {text!r}")


def build_nest(spec: P.StencilSpec, space: P.IterationSpace, mode: str, tiles: List[int], time_tile: int,
               skew: Optional[int], fused: int) -> P.LoopNest:
    """The nest of `--mode`: the legality gate of tile_time
    raises P.Error with ST_ERR_ILLEGAL_PLAN (exit 2)."""
    canon = P.build_canonical_nest(spec, space)
    n = len(space.extents)
    if tiles and len(tiles) != n:
        raise UsageError(f"--tiles needs {n} extents")
    t = tuple(tiles) if tiles else tuple(0 for _ in range(n))
    if mode == "none":
        return canon
    if mode in ("space", "space-remainder"):
        # the min/max nest subsumes the remainder group (execute_group ==
        # canonical, DESIGN.md section 1 row a12)
        return P.tile_space_minmax(canon, t)
    s = P.min_skew_factor(spec) if skew is None else skew   # default skew (SPEC.md cli ledger)
    return P.tile_time(canon, spec, space, P.TilePlan(s, time_tile, t, fused_levels=fused))


def _report_json(rep: P.ExecReport, nest: P.LoopNest) -> dict:
    return {"points_updated": rep.points_updated, "flops": rep.flops, "wall_seconds": rep.wall_seconds,
            "device_seconds": rep.device_seconds, "time_tile_used": rep.time_tile_used,
            "kernel_launches": rep.kernel_launches, "tile": list(rep.tile), "mode_used": rep.mode_used,
            "kernel_kind": rep.kernel_kind, "schedule": nest.schedule,
            "plan": None if nest.plan is None else {"skew": nest.plan.skew, "time_tile": nest.plan.time_tile,
                                                    "space_tiles": list(nest.plan.space_tiles),
                                                    "fused_levels": nest.plan.fused_levels}}


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1806_08299_b200.cli", add_help=True)
    ap.add_argument("command")
    ap.add_argument("spec")
    ap.add_argument("--mode", choices=MODES, default="none")
    ap.add_argument("--tiles", default="")
    ap.add_argument("--time-tile", type=int, default=1)
    ap.add_argument("--skew", type=int, default=None)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--arith", choices=("reference", "fast"), default="reference")
    ap.add_argument("--fused", type=int, default=0)
    ap.add_argument("--trials", type=int, default=3)
    ap.add_argument("--fused-levels", default="")
    ap.add_argument("--cost", choices=("time", "traffic"), default="time")
    ap.add_argument("--cache-elems", type=int, default=DEFAULT_CACHE_ELEMS)
    ap.add_argument("--line-elems", type=int, default=16)
    ap.add_argument("--profile", default="")
    ap.add_argument("-o", "--output", default=None)
    return ap


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def main(argv: Optional[List[str]] = None) -> int:
    ap = _parser()
    ap.__class__ = _ArgParser
    try:
        args = ap.parse_args(argv)
        if args.command not in EXECUTOR_SUBCOMMANDS:
            raise UsageError(f"unknown subcommand {args.command!r}")
        try:
            with open(args.spec) as f:
                text = f.read()
        except OSError as e:
            raise UsageError(f"cannot read {args.spec}: {e}")
        spec, space = P.parse_spec(text)
        if args.command == "tune":
            return _tune_traffic(spec, space, args) if args.cost == "traffic" else _tune(spec, space, args)
        if args.command == "analyze":
            return _analyze(spec, space, args)
        nest = build_nest(spec, space, args.mode, _ints(args.tiles), args.time_tile, args.skew, args.fused)
        if args.command == "transform":
            return _transform(spec, space, nest, args)
        if args.command == "simulate":
            rep = P.simulate(nest, spec, space, P.CacheConfig(args.cache_elems, args.line_elems))
            print(json.dumps(dataclasses_asdict(rep)))
            return 0
    except P.ParseError as e:
        print(f"parse error (line {e.line()}): {e}", file=sys.stderr)
        return 2
    except (UsageError, P.Error) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2

    arith = P.MODE_FAST if args.arith == "fast" else P.MODE_REFERENCE
    if args.command == "run":
        grid = P.init_grid(spec, space, args.seed, P.required_slots(nest, spec))
        rep = P.execute(nest, spec, space, grid, arith)
        print(json.dumps(_report_json(rep, nest)))
        return 0
    # verify: canonical and transformed on grids of the same slot count, so
    # that the literal per-slot halos (DESIGN.md ledger 5) cannot differ
    canon = P.build_canonical_nest(spec, space)
    slots = max(P.required_slots(nest, spec), P.required_slots(canon, spec))
    a = P.init_grid(spec, space, args.seed, slots)
    b = P.init_grid(spec, space, args.seed, slots)
    P.execute(canon, spec, space, a, P.MODE_REFERENCE)
    P.execute(nest, spec, space, b, arith)
    equal = P.verify_bitwise(a, b, spec.time_depth)
    print(json.dumps({"bitwise_equal": bool(equal)}))
    return 0 if equal else 1


def _transform(spec: P.StencilSpec, space: P.IterationSpace, nest: P.LoopNest, args) -> int:
    from . import codegen
    if spec.model != P.MODEL_TERMS:
        raise UsageError("transform emits the terms model only (the wave field is an executor extension)")
    sched = {P.SCHED_CANONICAL: "canonical", P.SCHED_SPACE: "space", P.SCHED_TIME: "time"}[nest.schedule]
    plan = nest.plan
    n = len(space.extents)
    tiles = None
    if sched != "canonical":
        tiles = [t if t > 0 else e for t, e in zip(plan.space_tiles, space.extents)]   # 0 = whole extent
    try:
        src = codegen.emit_c(n, [(t.coeff, t.dt, tuple(t.offsets)) for t in spec.terms], space.extents,
                             space.time_steps, P.required_slots(nest, spec), sched,
                             skew=plan.skew if plan else 0, time_tile=plan.time_tile if plan else 1, tiles=tiles,
                             seed=args.seed)
    except ValueError as e:
        raise UsageError(str(e))
    if args.output:
        with open(args.output, "w") as f:
            f.write(src)
    else:
        sys.stdout.write(src)
    return 0


def dataclasses_asdict(x) -> dict:
    import dataclasses
    return dataclasses.asdict(x)


def _analyze(spec: P.StencilSpec, space: P.IterationSpace, args) -> int:
    """IntensityEstimate + FaceAnalysis + roofline bound."""
    from . import analysis as A
    n = len(space.extents)
    tiles = _ints(args.tiles) or list(space.extents)
    if len(tiles) != n or any(t < 1 for t in tiles):
        raise UsageError(f"--tiles needs {n} positive extents")
    if args.time_tile < 1 or args.cache_elems < 1:
        raise UsageError("--time-tile and --cache-elems must be >= 1")
    est, faces = A.tight_bound(spec, space.extents, args.time_tile, tiles, args.cache_elems)
    out = {"estimate": dataclasses_asdict(est), "faces": dataclasses_asdict(faces),
           "tiles": tiles, "time_tile": args.time_tile, "cache_elems": args.cache_elems}
    if args.profile:
        try:
            peak, bw = (float(v) for v in args.profile.split(","))
        except ValueError:
            raise UsageError("--profile needs peak_gflops,bandwidth_gbs")
        prof = A.MachineProfile(peak, bw, args.cache_elems)
        out["ridge_point"] = A.ridge_point(prof)
        out["roofline_bound"] = {k: A.roofline_bound(prof, getattr(est, k)) for k in
                                 ("ai_spatial", "ai_naive_tt", "ai_tight_tt")}
    print(json.dumps(out))
    return 0


def _tune_traffic(spec: P.StencilSpec, space: P.IterationSpace, args) -> int:
    """tune --cost traffic: the reference's plan space with
    the simulated bytes as cost; byte-identical output across runs."""
    from . import autotune as A
    cache = P.CacheConfig(args.cache_elems, args.line_elems)
    best, cost, table = A.tune_sim(spec, space, A.HostSearchSpace(), cache)
    plan = lambda p: {"skew": p.skew, "time_tile": p.time_tile, "space_tiles": list(p.space_tiles)}  # noqa: E731
    print(json.dumps({"best": plan(best), "best_cost_bytes": cost,
                      "table": [dict(plan(p), cost_bytes=c) for p, c in table]}))
    return 0


def _tune(spec: P.StencilSpec, space: P.IterationSpace, args) -> int:
    from . import autotune as A
    fused = tuple(_ints(args.fused_levels))
    search = A.SearchSpace(trials=args.trials, fused_levels=fused)
    if args.arith == "fast":
        search.modes = (P.MODE_REFERENCE, P.MODE_FAST)
    slots = spec.time_depth + max(list(search.time_tiles) + list(fused))
    ctx = P.default_context()
    grid = P.init_grid(spec, space, args.seed, slots)
    dg = P.DeviceGrid(ctx, spec, space.extents, slots)
    try:
        dg.upload(grid.data, grid.last_level)
        radius = max(spec.radii)
        res = A.tune(dg, spec, radius, len(space.extents), space.time_steps, grid.last_level, search)
    finally:
        dg.close()
    print(json.dumps(res.to_json()))
    return 0


if __name__ == "__main__":
    sys.exit(main())
