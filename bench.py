#!/usr/bin/env python
"""Benchmark: grid-point updates per second (GPts/s) of the stencil executor.

One *step* = one apply() of the configured run (e.g. config 2: 64 time steps
of the 3D heat so4 stencil over 256^3) through the C-ABI, inputs resident in
HBM.  `value` is device time (CUDA events on the launching stream, summed
over K timed steps, L2 flushed between them, max over ranks); `e2e` is the
same metric through the public API with host buffers (H2D of the inputs +
apply + D2H of the retained levels, per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
                  [--impl ours|reference] [--time-tile T] [--mode reference|fast]

--impl reference times the reference's CPU path on the host cores: the
compiled oracle restatement (the reference itself has no definitions to
compile), all host threads, on the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_1806_08299_b200 as P  # noqa: E402
from paper_1806_08299_b200 import configs as CF  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")

# Per-config executor plans (tuned on B200): configs.BENCH_PLANS.
DEFAULTS = CF.BENCH_PLANS

# What "fast" means per config: the arithmetic is chosen so the full run stays
# within the 1e-5 contract (max|gpu - reference| / max|reference|); measured
# by tests/test_gpu_fullsize.py and tests/test_gpu_fullrun.py.
FAST_NOTE = {
    0: "<= 1e-5 of max|u| after the full run (BASELINE north_star), tests/test_gpu_fullsize.py",
    3: "<= 1e-5 of max|u| after the full run: 4.5e-6 measured (ordered hybrid: reference summation order, "
       "products of the taps at distance >= 2 fused), tests/test_gpu_fullrun.py",
    4: "<= 1e-5 of max|u| after the full run: 5.2e-6 measured (symmetric taps paired + FMA), tests/test_gpu_fullsize.py",
    5: "<= 1e-5 of max|u| after the full run: 4.5e-6 measured on the same pulse (config 3's box; ordered hybrid: "
       "reference summation order, products of the taps at distance >= 2 fused), tests/test_gpu_fullrun.py",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- inputs ---
def host_inputs(cfg: CF.Config, slots: int, spec: P.StencilSpec, pinned: bool = True):
    """Reference-layout host grid (+ wave m field) built by the product's own
    initialisers (st_init_* in the C-ABI), in pinned memory when torch is
    available."""
    lay = P.GridLayout.make(spec, P.IterationSpace(cfg.steps, cfg.extents), slots)
    n = lay.total_elems()
    buf = None
    if pinned:
        try:
            import torch
            buf = torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
        except Exception:
            buf = None
    if buf is None:
        buf = np.empty(n, dtype=np.float32)
    lib = P._native.load()
    ext = P._native.i64array(cfg.extents)
    fptr = P.tiler._fptr(buf)
    if cfg.init == "unit":
        rc = lib.st_init_unit(spec.handle, ext, fptr, slots, CF.SEED_FIELD)
    else:
        rc = lib.st_init_gaussian(spec.handle, ext, fptr, slots, cfg.sigma,
                                  P._native.i64array([e // 2 for e in cfg.extents]))
    P.tiler._check(rc)
    m = None
    if cfg.field:
        m = np.empty(int(np.prod(cfg.extents)), dtype=np.float32)
        if cfg.field == "layered":
            rc = lib.st_field_layered(cfg.ndims, ext, P.tiler._fptr(m), cfg.v_top, cfg.v_bottom, cfg.extents[0] // 2,
                                      cfg.dt, CF.H, 0)
        else:
            rc = lib.st_field_random_smoothed(cfg.ndims, ext, P.tiler._fptr(m), CF.SEED_VELOCITY, cfg.vmin, cfg.vmax,
                                              cfg.dt, CF.H)
        P.tiler._check(rc)
    return buf, m


def make_spec(cfg: CF.Config) -> P.StencilSpec:
    return P.StencilSpec.make(cfg.name, cfg.ndims, [P.StencilTerm(c, dt, off) for c, dt, off in cfg.terms],
                              model=cfg.model)


# ---------------------------------------------------------------- clocks ---
class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.watts = [], set(), None, []
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log(f"[bench] NVML unavailable: {e}")
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.watts.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.002)   # the config 2 timed region is ~10 ms

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w": round(statistics.median(self.watts), 1) if self.watts else None}


# ---------------------------------------------------------- CPU baseline ---
def cpu_run(cfg: CF.Config, steps: int, threads: int, schedule: int, T: int, tiles):
    """The oracle (CPU restatement of the reference executor) on `steps`
    steps of `cfg`, grid init excluded; returns (GPts/s, seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O  # test infrastructure: the CPU baseline leg only
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    dtd = spec.time_depth
    slots = dtd + (T if schedule == O.TIME else 1)
    ext = cfg.extents
    if cfg.init == "unit":
        g = O.init_unit(spec, ext, slots, CF.SEED_FIELD)
    else:
        g = O.init_gaussian(spec, ext, slots, cfg.sigma, [e // 2 for e in ext])
    m = None
    if cfg.field == "layered":
        m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H)
    elif cfg.field == "random":
        m = O.mfield_random(ext, CF.SEED_VELOCITY, cfg.vmin, cfg.vmax, cfg.dt, CF.H)
    rc, secs, pts = O.execute(spec, ext, g, slots, 0, steps, mfield=m, schedule=schedule,
                              skew=max(spec.radius(i) for i in range(spec.ndims)), time_tile=T, tiles=tiles,
                              nthreads=threads)
    assert rc == 0, rc
    return pts / secs / 1e9, secs


def cpu_tiles(cfg):
    # spatial tiles of the CPU nests: full innermost extent (the paper's
    # auto-tuner always chose it, PAPER.md via SPEC.md:559), 8 rows / planes
    if cfg.ndims == 3:
        return (8, 8, cfg.extents[2])
    if cfg.ndims == 2:
        return (32, cfg.extents[1])
    return (cfg.extents[0],)


def cpu_baseline(cfg: CF.Config, budget_s: float = 20.0):
    """Bounded sample: the space-tiled (S) and time-tiled (T) CPU nests on all
    host cores, min of 3 trials each, steps scaled to ~budget_s total."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    tiles = cpu_tiles(cfg)
    # calibrate with 1 step
    rate, _ = cpu_run(cfg, 1, threads, O.SPACE, 1, tiles)
    pts_step = int(np.prod(cfg.extents))
    steps = max(1, min(cfg.steps, int(budget_s / 6 * rate * 1e9 / pts_step)))
    res = {}
    for name, sched, T in (("space", O.SPACE, 1), ("time", O.TIME, min(4, steps))):
        best = 0.0
        for _ in range(3):
            r, _ = cpu_run(cfg, steps, threads, sched, T, tiles)
            best = max(best, r)
        res[name] = best
    kind = "port"
    best_name = max(res, key=res.get)
    return {
        "value": round(res[best_name], 4), "unit": "GPts/s", "cores": threads, "kind": kind,
        "sample": f"{cfg.name} {'x'.join(map(str, cfg.extents))}, {steps} of {cfg.steps} steps, "
                  f"oracle {best_name}-tiled nest (S {res['space']:.3f} / T {res['time']:.3f} GPts/s), "
                  f"tiles {tiles}, T=4, min of 3 trials, init excluded",
        "space_tiled": round(res["space"], 4), "time_tiled": round(res["time"], 4),
    }


# ------------------------------------------------------------ reference ---
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    full = cfg
    # a grid of > 2^28 points (config 5 weak-scaled: 4 Gi points at N = 8, tens
    # of GB of host memory per level set) is sampled as a 64-plane z-slab of
    # the same rows: the CPU rate per point does not depend on depth
    zsample = int(np.prod(cfg.extents)) > (1 << 28)
    if zsample:
        cfg = cfg.scaled((min(cfg.extents[0], 64),) + tuple(cfg.extents[1:]), cfg.steps)
    tiles = cpu_tiles(cfg)
    # the faster of the reference's CPU nests (space-tiled: 8.2 vs 1.6 GPts/s
    # time-tiled on config 2, 16 cores) -- the conservative baseline
    rate, _ = cpu_run(cfg, 1, threads, O.SPACE, 1, tiles)
    pts_step = int(np.prod(cfg.extents))
    # each step: a bounded sample of the run so W + K steps take ~2-3 min
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    steps = max(1, min(cfg.steps, int(per_step_budget * rate * 1e9 / pts_step)))
    for _ in range(args.warmup):
        cpu_run(cfg, steps, threads, O.SPACE, 1, tiles)
    secs_total, pts_total = 0.0, 0
    for _ in range(args.steps):
        r, s = cpu_run(cfg, steps, threads, O.SPACE, 1, tiles)
        secs_total += s
        pts_total += steps * pts_step
    value = pts_total / secs_total / 1e9
    line = {
        "metric": "grid-point updates/sec (GPts/s)", "value": round(value, 4), "unit": "GPts/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs_total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
        "config": dict(workload(full, args, 1, "space-tiled oracle"), mode="reference (oracle, bit-exact)"),
        "cpu_baseline": {"value": round(value, 4), "unit": "GPts/s", "cores": threads, "kind": "port",
                         "sample": (f"z-sample {'x'.join(map(str, cfg.extents))} of the grid, " if zsample else "") +
                                   f"{steps} of {cfg.steps} time steps per bench step, space-tiled oracle nest "
                                   f"(tiles {tiles}, the faster of the reference's CPU nests); the reference "
                                   f"ships no definitions, the oracle restates its executor (SURVEY.md 0, 8c)"},
        "e2e": {"value": round(value, 4), "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- helpers ---
def workload(cfg, args, T, sched):
    return {
        "workload": f"config{cfg.index} {cfg.name} {'x'.join(map(str, cfg.extents))} x {cfg.steps} steps",
        "stencil": cfg.name, "extents": list(cfg.extents), "time_steps": cfg.steps, "radius": cfg.radius,
        "schedule": sched, "time_tile": T, "mode": args.mode or DEFAULTS[cfg.index]["mode"],
        "l2": "flushed between timed steps (256 MiB write)", "seed": CF.SEED_FIELD,
    }


def flush_l2(buf):
    buf.fill_(1.0)


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------- e2e (N=1) ---
def e2e_lanes(cfg, spec, extents, slots, nest, mode, host, m, local, steps, dtd):
    """End to end through the public host-grid API (st_execute_host: upload
    the input levels from page-locked memory, run the step, write the newest
    delta_t levels back), the m field re-sent from page-locked memory every
    step.  ST_E2E_INFLIGHT independent problems are in flight (one device
    grid / context / host thread each: one problem's copies overlap another's
    kernels, the throughput a server sees); the single-call latency is
    reported beside it."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    nflight = int(os.environ.get("ST_E2E_INFLIGHT", "4"))   # config 5: 4 x 12 GB of device grids, 4 x 13 GB page-locked
    per_lane = max(1, min(steps, int(os.environ.get("ST_E2E_PER_LANE", "4"))))   # steady state: the fill / drain of the lanes amortised

    def pinned_copy(a):
        try:
            b = torch.empty(a.size, dtype=torch.float32, pin_memory=True).numpy()
        except Exception:
            b = np.empty_like(a)
        b[:] = a
        return b

    mp = pinned_copy(m) if m is not None else None
    lanes = []
    for _ in range(nflight):
        c = P.Context(local)
        g = P.DeviceGrid(c, spec, extents, slots)
        lanes.append((c, g, pinned_copy(host)))

    def run_lane(lane, n):
        _, g, buf = lane
        torch.cuda.set_device(local)
        for _ in range(n):
            if mp is not None:
                g.set_field(mp)
            g.execute_host(buf, 0, cfg.steps, nest, mode, uniform_halo=True)

    def timed(fn):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return time.perf_counter() - w0

    with ThreadPoolExecutor(nflight) as ex:
        list(ex.map(lambda l: run_lane(l, 1), lanes))            # warm-up
        single = timed(lambda: run_lane(lanes[0], 1))
        secs = timed(lambda: list(ex.map(lambda l: run_lane(l, per_lane), lanes)))
    for c, g, _ in lanes:
        g.close()
        c.close()
    pts = cfg.steps * int(np.prod(extents))
    padded = int(np.prod([e + 2 * cfg.radius for e in extents]))
    interior = int(np.prod(extents))
    n = nflight * per_lane
    return {"value": round(n * pts / secs / 1e9, 3), "unit": "GPts/s",
            "h2d_bytes_per_step": int(dtd * padded * 4 + (m.size * 4 if m is not None else 0)),
            "d2h_bytes_per_step": int(dtd * interior * 4), "steps": n, "ms_per_step": round(secs / n * 1e3, 3),
            "api": f"st_grid_set_field + st_execute_host from page-locked memory, {nflight} problems in flight "
                   f"({nflight} device grids / contexts, 1 host thread each)",
            "single_call_ms": round(single * 1e3, 3), "single_call_value": round(pts / single / 1e9, 3)}


# --------------------------------------------------------- sharded (5) ---
def run_dist(args, cfg, rank, world, local, dist):
    """z-slabs along d_1, one per GPU (weak scaling): ghost depth r*T exchanged
    with NCCL send/recv once per time tile (st_dist_*), one wavefront launch
    per time tile over the trapezoid of slab ranges."""
    import torch
    cidx = cfg.index
    plan = CF.DIST_PLANS.get(cidx, DEFAULTS[cidx])
    mode = {"reference": P.MODE_REFERENCE, "fast": P.MODE_FAST}[args.mode or plan["mode"]]
    T = args.time_tile or plan["time_tile"]
    sched = args.schedule or plan["schedule"]
    tiles = (tuple(int(x) for x in args.tiles.split(",")) if args.tiles
             else tuple(plan.get("tiles_reference" if mode == P.MODE_REFERENCE and world == 1 else "tiles",
                                 plan.get("tiles", tuple(0 for _ in cfg.extents)))))
    # (whole-depth items suit the bit-exact mode only inside the N = 1 persistent launch: with one launch
    # per time tile the shorter z-chunks leave a smaller tail, profiles/r02b_slab_overhead.log)
    r = cfg.radius
    ghost = r * T if world > 1 else 0
    z0, nzs, glo, ghi = P.dist_partition(cfg.extents[0], world, rank, ghost)
    lext = (nzs + glo + ghi,) + tuple(cfg.extents[1:])
    spec = make_spec(cfg)
    dtd = spec.time_depth
    nest = (P.LoopNest(P.SCHED_TIME, P.TilePlan(r, T, tiles)) if sched == "time"
            else P.LoopNest(P.SCHED_CANONICAL, P.TilePlan(r, T, ())))
    slots = dtd + (T if sched == "time" else 1)
    space = P.IterationSpace(cfg.steps, lext)
    if cfg.init == "unit":
        # per-slab seeded interiors: the first exchange overwrites the ghosts
        # with the neighbours' planes, so every slab is consistent
        grid = P.init_unit(spec, space, CF.SEED_FIELD + rank, slots)
    else:
        centre = [e // 2 for e in cfg.extents]
        grid = P.init_gaussian(spec, space, slots, cfg.sigma, centre, z_begin=z0 - glo)
    m = None
    if cfg.field == "layered":
        m = np.empty(int(np.prod(lext)), dtype=np.float32)
        P.tiler._check(P._native.load().st_field_layered(3, P._native.i64array(lext), P.tiler._fptr(m), cfg.v_top,
                                                         cfg.v_bottom, cfg.extents[0] // 2, cfg.dt, CF.H, z0 - glo))
    torch.cuda.set_device(local)
    ctx = P.Context(local)
    dg = P.DeviceGrid(ctx, spec, lext, slots)
    dg.upload(grid.data, dtd - 1, uniform_halo=True)
    if m is not None:
        dg.set_field(m)
    nid = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(P.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tolist())
    d = P.Dist(dg, rank, world, glo, ghi, nid)
    stream = torch.cuda.ExternalStream(ctx.stream)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    pts_rank = cfg.steps * nzs * lext[1] * lext[2]
    t = 0
    for _ in range(args.warmup):
        d.apply(t, t + cfg.steps, nest, mode)
        t += cfg.steps
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    total, launches, reps = 0.0, 0, []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(l2)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = d.apply(t, t + cfg.steps, nest, mode)
            e1.record(stream)
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1) * 1e-3
            t += cfg.steps
            launches += rep.kernel_launches
            reps.append(rep)
    if dist:
        tt = torch.tensor([total], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    value = world * args.steps * pts_rank / total / 1e9

    # ---- the same plan in reference mode (bitwise equal to the oracle), timed
    # beside a FAST headline so both arithmetics are on record (N = 1)
    bit_exact = None
    if mode == P.MODE_FAST and world == 1 and not args.no_bit_exact:
        nb = max(1, min(args.steps, 3))
        rt = tuple(plan.get("tiles_reference", tiles)) if not args.tiles else tiles
        rnest = (P.LoopNest(P.SCHED_TIME, P.TilePlan(r, T, rt)) if sched == "time" else nest)
        d.apply(t, t + cfg.steps, rnest, P.MODE_REFERENCE)
        t += cfg.steps
        torch.cuda.synchronize()
        tb = 0.0
        for _ in range(nb):
            flush_l2(l2)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d.apply(t, t + cfg.steps, rnest, P.MODE_REFERENCE)
            e1.record(stream)
            torch.cuda.synchronize()
            tb += e0.elapsed_time(e1) * 1e-3
            t += cfg.steps
        bit_exact = {"value": round(nb * pts_rank / tb / 1e9, 3), "unit": "GPts/s", "steps": nb,
                     "ms_per_step": round(tb / nb * 1e3, 3), "tiles": list(rt),
                     "mode": "reference (bitwise equal to the oracle)"}

    # ---- end to end through the public API with host buffers: every step
    # each rank uploads its slab's input levels (and the m field) from
    # page-locked memory, runs the sharded step (NCCL ghost exchanges
    # included) and downloads its newest levels; wall clock, max over ranks
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = e2e_lanes(cfg, spec, lext, slots, nest, mode, grid.data, m, local, args.steps, dtd)
    elif not args.no_e2e:
        if world == 1:
            def pinned():
                try:
                    return torch.empty(grid.data.size, dtype=torch.float32, pin_memory=True).numpy()
                except Exception:
                    return np.empty_like(grid.data)
            host_in, host_out = pinned(), pinned()   # inputs stay intact, results land apart
            host_in[:] = grid.data
        else:
            # N ranks on one host: a slab's reference grid is ~14 GB at T = 4;
            # pinning two copies per rank would lock ~28 GB x N of host memory.
            # Pageable buffers (staged copies), the output lazily zero-filled.
            host_in, host_out = grid.data, np.zeros_like(grid.data)
        n_e2e = max(1, min(args.steps, 3))

        def e2e_step():
            dg.upload(host_in, dtd - 1, uniform_halo=True)
            if m is not None:
                dg.set_field(m)
            d.apply(0, cfg.steps, nest, mode)
            dg.download(host_out)

        e2e_step()                                   # warm-up
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        torch.cuda.synchronize()
        secs = time.perf_counter() - w0
        if dist:
            tt = torch.tensor([secs], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            secs = float(tt.item())
        padded = int(np.prod([e + 2 * r for e in lext]))
        e2e = {"value": round(world * n_e2e * pts_rank / secs / 1e9, 3), "unit": "GPts/s",
               "h2d_bytes_per_step": int(dtd * padded * 4 + (m.size * 4 if m is not None else 0)),
               "d2h_bytes_per_step": int((dtd + 1) * padded * 4), "steps": n_e2e,   # the retained levels
               "ms_per_step": round(secs / n_e2e * 1e3, 3),
               "api": "per rank: st_grid_upload + st_dist_apply + st_grid_download (staged), wall clock, max over ranks"}

    peaks = load_json(PEAKS_FILE) or {}
    peak = peaks.get("hbm_gbs") or 6650.0
    # algorithmic bytes of the slab's updates per device second (max over ranks)
    achieved = cfg.bytes_per_point * args.steps * pts_rank / (total / 1.0) / 1e9
    # ncu DRAM bytes per launch of this plan (profiles/traffic.json; one GPU)
    mkey = "fast" if mode == P.MODE_FAST else "reference"
    tkey = f"config{cidx}:slab{world}:{sched}:T{T}:{mkey}" + (f":F{reps[0].time_tile_used}" if reps[0].kernel_kind >= 2 else "")
    traffic = (load_json(TRAFFIC_FILE) or {}).get(tkey, {}).get("dram_bytes_per_launch")
    line = {
        "metric": "grid-point updates/sec (GPts/s)", "value": round(value, 3), "unit": "GPts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Gaussian pulse, layered velocity; SURVEY.md App. A)",
        "config": {"workload": f"config{cidx} {cfg.name} {'x'.join(map(str, cfg.extents))} x {cfg.steps} steps"
                               f" ({world} z-slab{'s' if world > 1 else ''} of {cfg.extents[0] // world} planes)",
                   "slab": [z0, nzs], "ghost": [glo, ghi], "exchange_every": T, "schedule": sched, "tiles": list(tiles),
                   "mode": args.mode or plan["mode"],
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"z-slabs x{world} (NCCL send/recv)" if world > 1 else "1gpu"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "note": f"{cfg.bytes_per_point} B/point-update x slab updates / device time (max over ranks)"},
        "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(), "updates_per_step": world * pts_rank,
    }
    if mode == P.MODE_FAST:
        line["config"]["tolerance"] = FAST_NOTE.get(cidx, FAST_NOTE[0])
    if bit_exact:
        bit_exact["frac"] = round(cfg.bytes_per_point * bit_exact["value"] / peak, 4)
        line["bit_exact"] = bit_exact
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg.scaled((64,) + tuple(cfg.extents[1:]), cfg.steps)
                                                if cidx == 5 else cfg)
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    d.close()
    dg.close()
    ctx.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------- launch ---
def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_launch(gpus: int, env, argv) -> dict:
    """How `bench.py --gpus N` runs its ranks.

    * under torchrun (WORLD_SIZE set): this process is one rank; WORLD_SIZE
      must equal N ("error" otherwise -- never a silent single rank);
    * N = 1 without torchrun: this process is the only rank ("single");
    * N > 1 without torchrun: re-launch this script under
      torch.distributed.run with N processes on 127.0.0.1 ("spawn")."""
    if gpus < 1:
        return {"mode": "error", "error": f"--gpus {gpus}: need at least 1"}
    ws = env.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus:
            return {"mode": "error", "error": f"--gpus {gpus} but WORLD_SIZE={ws} (torchrun rank count)"}
        return {"mode": "rank", "world": int(ws), "rank": int(env.get("RANK", "0"))}
    if gpus == 1:
        return {"mode": "single", "world": 1, "rank": 0}
    port = _free_port()
    rest = [a for a in argv if a != "--dry-run"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + rest
    return {"mode": "spawn", "world": gpus, "argv": cmd}


# ----------------------------------------------------------------- main ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=None)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--time-tile", type=int, default=None)
    ap.add_argument("--schedule", choices=["time", "space", "canonical"], default=None)
    ap.add_argument("--tiles", type=str, default=None, help="z,y,x tile extents (0 = auto)")
    ap.add_argument("--mode", choices=["reference", "fast"], default=None)
    ap.add_argument("--fused", type=int, default=None,
                    help="levels advanced on-chip per pass (st_plan.fused_levels; 0 = wavefront)")
    ap.add_argument("--extents", type=str, default=None, help="override the config's extents (z,y,x), for studies")
    ap.add_argument("--time-steps", type=int, default=None, help="override the config's step count, for studies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-bit-exact", action="store_true",
                    help="skip the reference-mode timing that accompanies a FAST headline")
    ap.add_argument("--slab-path", action="store_true", help="run the z-slab (sharded) path even at N = 1")
    ap.add_argument("--dry-run", action="store_true",
                    help="print the rank launch (torchrun command or single process) as JSON and exit")
    args = ap.parse_args()

    # --gpus N without a torchrun environment: launch N ranks ourselves (one
    # process per GPU, torch.distributed.run on 127.0.0.1), never silently
    # fewer.  Under torchrun WORLD_SIZE must equal --gpus.
    launch = rank_launch(args.gpus, os.environ, sys.argv[1:])
    if args.dry_run:
        print(json.dumps(launch), flush=True)
        return
    if launch["mode"] == "spawn":
        import subprocess
        sys.exit(subprocess.call(launch["argv"]))
    if launch["mode"] == "error":
        log(f"[bench] {launch['error']}")
        sys.exit(2)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BASELINE's metric is quoted at 1/2/4/8 B200 on the weak-scaled config 5
    # (z-slabs of 512 planes per GPU), so config 5 is the headline
    # at every N, N = 1 included (the same slab path with no neighbours);
    # configs 1-4 are single-GPU (`--config C`).  `--config C --gpus N`
    # shards any config as z-slabs of its single-GPU grid.
    cidx = args.config or 5
    if world > 1:
        import torch
        if torch.cuda.is_available() and torch.cuda.device_count() < world:
            log(f"[bench] --gpus {world}: only {torch.cuda.device_count()} visible GPU(s)")
            sys.exit(2)
    cfg = CF.sharded(cidx, world) if (world > 1 or cidx == 5 or args.slab_path) else CF.get(cidx)
    if args.extents or args.time_steps:
        cfg = cfg.scaled(tuple(int(x) for x in args.extents.split(",")) if args.extents else cfg.extents,
                         args.time_steps or cfg.steps)

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    if cfg.sharded:
        run_dist(args, cfg, rank, world, local, dist)
        return

    mode = {"reference": P.MODE_REFERENCE, "fast": P.MODE_FAST}[args.mode or DEFAULTS[cidx]["mode"]]
    T = args.time_tile or DEFAULTS[cidx]["time_tile"]
    sched = args.schedule or DEFAULTS[cidx]["schedule"]
    tiles = (tuple(int(x) for x in args.tiles.split(",")) if args.tiles
             else tuple(DEFAULTS[cidx].get("tiles_reference" if mode == P.MODE_REFERENCE else "tiles",
                                           DEFAULTS[cidx].get("tiles", tuple(0 for _ in cfg.extents)))))

    torch.cuda.set_device(local)
    ctx = P.Context(local)
    spec = make_spec(cfg)
    dtd = spec.time_depth
    F = args.fused if args.fused is not None else DEFAULTS[cidx].get("fused", 0)
    plan = P.TilePlan(cfg.radius, T, tiles, fused_levels=F if sched == "time" else 0)
    canon = P.build_canonical_nest(spec, None)
    nest = {"time": lambda: P.tile_time(canon, spec, None, plan),
            "space": lambda: P.tile_space_minmax(canon, tiles),
            "canonical": lambda: canon}[sched]()
    slots = P.required_slots(nest, spec)
    host, m = host_inputs(cfg, slots, spec)
    dg = P.DeviceGrid(ctx, spec, cfg.extents, slots)
    dg.upload(host, dtd - 1, uniform_halo=True)
    if m is not None:
        dg.set_field(m)
    pts_step = cfg.steps * int(np.prod(cfg.extents))
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")

    t = 0
    for _ in range(args.warmup):
        dg.apply(t, t + cfg.steps, nest, mode)
        t += cfg.steps

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_times, launches, reps = [], 0, []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(l2)
            torch.cuda.synchronize()
            rep = dg.apply(t, t + cfg.steps, nest, mode)
            t += cfg.steps
            dev_times.append(rep.device_seconds)
            launches += rep.kernel_launches
            reps.append(rep)
    torch.cuda.synchronize()
    total = sum(dev_times)
    if dist:
        tt = torch.tensor([total], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
        dist.barrier()
    value = world * args.steps * pts_step / total / 1e9
    ms = total / args.steps * 1e3

    # ---- the same plan in reference mode (bitwise equal to the oracle), timed
    # beside a FAST headline so both arithmetics are on record
    bit_exact = None
    if mode == P.MODE_FAST and world == 1 and not args.no_bit_exact and not args.tiles:
        rt = tuple(DEFAULTS[cidx].get("tiles_reference", tiles))
        rplan = P.TilePlan(cfg.radius, T, rt, fused_levels=F if sched == "time" else 0)
        rnest = {"time": lambda: P.tile_time(canon, spec, None, rplan),
                 "space": lambda: P.tile_space_minmax(canon, rt), "canonical": lambda: canon}[sched]()
        nb = max(1, min(args.steps, 3))
        dg.apply(t, t + cfg.steps, rnest, P.MODE_REFERENCE)
        t += cfg.steps
        tb = 0.0
        for _ in range(nb):
            flush_l2(l2)
            torch.cuda.synchronize()
            tb += dg.apply(t, t + cfg.steps, rnest, P.MODE_REFERENCE).device_seconds
            t += cfg.steps
        bit_exact = {"value": round(nb * pts_step / tb / 1e9, 3), "unit": "GPts/s", "steps": nb,
                     "ms_per_step": round(tb / nb * 1e3, 4), "tiles": list(rt),
                     "mode": "reference (bitwise equal to the oracle)"}

    # ---- end to end through the public API with host buffers (e2e_lanes:
    # st_execute_host from page-locked memory, several problems in flight,
    # the single-call latency beside it)
    e2e = None
    if not args.no_e2e:
        os.environ.setdefault("ST_E2E_INFLIGHT", "4")
        e2e = e2e_lanes(cfg, spec, cfg.extents, slots, nest, mode, host, m, local, args.steps, dtd)

    # ---- roofline of the dominant kernel (the stencil kernel)
    peaks = load_json(PEAKS_FILE) or {}
    peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json)"
    if not peak:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    per_launch = [r.device_seconds / max(1, r.kernel_launches) for r in reps]
    avg_launch = sum(per_launch) / len(per_launch)
    pts_launch = pts_step / max(1, reps[0].kernel_launches)
    alg_bytes = cfg.bytes_per_point * pts_launch
    achieved = alg_bytes / avg_launch / 1e9
    traffic = None
    tr = load_json(TRAFFIC_FILE) or {}
    key = f"config{cidx}:{sched}:T{T if sched == 'time' else 1}:{'fast' if mode else 'reference'}"
    if reps[0].kernel_kind >= 2:
        key += f":F{reps[0].time_tile_used}"
    if key in tr:
        traffic = tr[key].get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "note": f"algorithmic {cfg.bytes_per_point} B/point-update (untiled sweep) x {int(pts_launch)} "
                    f"updates per launch / mean launch time; peak {peak_src}; frac > 1 = temporal reuse"}

    clocks = clk.summary()
    line = {
        "metric": "grid-point updates/sec (GPts/s)", "value": round(value, 3), "unit": "GPts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded LCG / Gaussian, SURVEY.md App. A)",
        "config": dict(workload(cfg, args, T, sched), tile=list(reps[0].tile),
                       fused_levels=reps[0].time_tile_used if reps[0].kernel_kind >= 2 else 0,
                       kernel={3: "resident", 2: "fused", 1: "star", 0: "generic"}[reps[0].kernel_kind],
                       parallelism=f"replicas{world}" if world > 1 else "1gpu"),
        "roofline": roof, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        "updates_per_step": pts_step,
    }
    if mode == P.MODE_FAST:
        line["config"]["tolerance"] = FAST_NOTE.get(cidx, FAST_NOTE[0])
    if bit_exact:
        bit_exact["frac"] = round(cfg.bytes_per_point * bit_exact["value"] / peak, 4)
        line["bit_exact"] = bit_exact
    if rank == 0 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as e:  # the GPU number stands on its own
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    dg.close()
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
