"""What the z-slab path costs per GPU beside the N = 1 persistent launch: the
G-slab weak-scaled config 5 run as G loopback slabs on ONE B200 (the slabs'
kernels run back to back on the one device; the ghost exchange is a device
copy on the side stream), i.e. the per-time-tile launches, the boundary
cones, the redundant ghost planes and the launch tails -- everything of the
N > 1 path except NVLink.  Throughput per slab / N = 1 throughput is an upper
bound on the weak-scaling efficiency the same plan can reach.

  python profiles/tools/slab_overhead.py [G] [--mode fast|reference] [--planes 512] [--tiles 256,24,0] [--T 4]
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
    ap.add_argument("G", type=int, nargs="?", default=2)
    ap.add_argument("--mode", default=None)
    ap.add_argument("--planes", type=int, default=512)
    ap.add_argument("--tiles", default=None)
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    plan = CF.DIST_PLANS[5]
    mode_s = a.mode or plan["mode"]
    mode = P.MODE_FAST if mode_s == "fast" else P.MODE_REFERENCE
    T = a.T or plan["time_tile"]
    tiles = (tuple(int(v) for v in a.tiles.split(",")) if a.tiles
             else tuple(plan.get("tiles_reference" if mode == P.MODE_REFERENCE else "tiles", plan["tiles"])))
    cfg1 = CF.get(5)
    ext_g = (a.planes * a.G,) + tuple(cfg1.extents[1:])
    cfg = cfg1.scaled(ext_g, cfg1.steps)
    spec = B.make_spec(cfg)
    r, dtd = cfg.radius, spec.time_depth
    slots = dtd + T
    nest = P.LoopNest(P.SCHED_TIME, P.TilePlan(r, T, tiles))
    ctx = P.Context(0)
    lib = P._native.load()

    def build(G):
        members, grids = [], []
        ghost = r * T if G > 1 else 0
        ext = (a.planes * G,) + tuple(cfg1.extents[1:])
        for rank in range(G):
            z0, nzs, glo, ghi = P.dist_partition(ext[0], G, rank, ghost)
            lext = (nzs + glo + ghi,) + tuple(ext[1:])
            grid = P.init_gaussian(spec, P.IterationSpace(cfg.steps, lext), slots, cfg.sigma, [e // 2 for e in ext],
                                   z_begin=z0 - glo)
            m = np.empty(int(np.prod(lext)), dtype=np.float32)
            P.tiler._check(lib.st_field_layered(3, P._native.i64array(lext), P.tiler._fptr(m), cfg.v_top, cfg.v_bottom,
                                                ext[0] // 2, cfg.dt, CF.H, z0 - glo))
            dg = P.DeviceGrid(ctx, spec, lext, slots)
            dg.upload(grid.data, dtd - 1, uniform_halo=True)
            dg.set_field(m)
            del grid, m
            grids.append(dg)
            members.append(P.Dist(dg, rank, G, glo, ghi))
        if G > 1:
            P.Dist.link_loopback(members)
        return members, grids

    res = {}
    for G in (1, a.G):
        members, grids = build(G)
        t = 0
        best = None
        for i in range(1 + a.reps):
            ctx.flush_l2()
            w0 = time.perf_counter()
            rep = members[0].apply(t, t + cfg.steps, nest, mode)   # returns after the last launch's event
            wall = time.perf_counter() - w0
            t += cfg.steps
            if i > 0:   # wall clock: launch gaps and host-side waits between the per-tile launches count
                best = wall if best is None else min(best, wall)
        pts = cfg.steps * a.planes * G * cfg1.extents[1] * cfg1.extents[2]
        res[G] = pts / best / 1e9
        print(f"G = {G}: {rep.kernel_launches} launches per run, {best * 1e3:.1f} ms wall (device sum {rep.device_seconds * 1e3:.1f}), "
              f"{res[G]:.1f} GPts/s on one GPU ({mode_s}, T = {T}, tiles {tiles})", flush=True)
        for m_ in members:
            m_.close()
        for g in grids:
            g.close()
    print(f"slab path / persistent launch = {res[a.G] / res[1]:.3f} "
          f"(per-tile launches, cones, ghost planes; no NVLink in this number)")


if __name__ == "__main__":
    main()
