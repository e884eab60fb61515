"""Plan sweep on one resident grid (B200): each plan runs the config's full
time range through st_apply, device time from the report (CUDA events).

  python profiles/tools/sweep_wf.py CONFIG PLAN [PLAN ...] [--mode reference|fast]
         [--reps N] [--sustain SECONDS] [--steps K] [--extents z,y,x] [--check]

PLAN = "T,cz,ty[@ENV=VAL[@ENV=VAL...]]": time tile, z-chunk planes, tile rows
(d_2 space tile), then environment knobs of the executor for that plan only
(e.g. ST_WF_YSKEW=4@ST_WF_CY_ROWS=64).  T = 0 runs the canonical schedule.
--reps: best of N after one warm-up (short runs: full clocks).  --sustain S:
repeat for S seconds first and report the mean of the following N runs (the
board sits at its power cap, as in bench.py).  --check compares every plan's
result bitwise with the first plan's.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
import paper_1806_08299_b200 as P  # noqa: E402
from paper_1806_08299_b200 import configs as CF  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("plans", nargs="+")
    ap.add_argument("--mode", default="reference")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--sustain", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--extents", type=str, default=None)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    cfg = CF.get(a.config)
    if a.extents or a.steps:
        ext = tuple(int(v) for v in a.extents.split(",")) if a.extents else cfg.extents
        cfg = cfg.scaled(ext, a.steps or cfg.steps)
    mode = P.MODE_FAST if a.mode == "fast" else P.MODE_REFERENCE
    spec = B.make_spec(cfg)
    dtd = 2 if cfg.model else 1
    Tmax = max(int(pl.split("@")[0].split(",")[0]) for pl in a.plans)
    slots = dtd + max(1, Tmax)
    host, m = B.host_inputs(cfg, slots, spec, pinned=False)
    ctx = P.Context(0)
    dg = P.DeviceGrid(ctx, spec, cfg.extents, slots)
    if m is not None:
        dg.set_field(m)
    updates = cfg.steps * int(np.prod(cfg.extents))
    first = None
    for pl in a.plans:
        parts = pl.split("@")
        T, cz, ty = (int(v) for v in parts[0].split(","))
        envs = dict(kv.split("=", 1) for kv in parts[1:])
        for k, v in envs.items():
            os.environ[k] = v
        canon = P.build_canonical_nest(spec, None)
        nest = canon if T == 0 else P.tile_time(canon, spec, None, P.TilePlan(cfg.radius, T, (cz, ty, 0)))

        def once():
            dg.upload(host, dtd - 1)
            ctx.flush_l2()
            return dg.apply(0, cfg.steps, nest, mode).device_seconds

        try:
            once()
            if a.sustain > 0:
                t0 = time.time()
                while time.time() - t0 < a.sustain:
                    once()
                ts = [once() for _ in range(a.reps)]
                sec = sum(ts) / len(ts)
            else:
                sec = min(once() for _ in range(a.reps))
            line = f"{pl:60s} {updates / sec / 1e9:8.1f} GPts/s  {sec * 1e3:9.3f} ms"
            if a.check:
                out = host.copy()
                dg.download(out)
                if first is None:
                    first = out
                    line += "  (check base)"
                else:
                    line += "  bitwise" if np.array_equal(out, first) else "  DIFFERS"
        except P.Error as e:
            line = f"{pl:60s} failed: {e}"
        print(line, flush=True)
        for k in envs:
            del os.environ[k]
    dg.close()


if __name__ == "__main__":
    main()
