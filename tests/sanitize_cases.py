"""Small cases of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck), each checked bitwise against the oracle so a run that
silently skipped work fails:

  compute-sanitizer --tool racecheck python tests/sanitize_cases.py

Covers the star kernel (per-level sweep and the cross-CTA wavefront, heat
r = 2 and wave r = 4 with palette-coded m), the generic kernel, the fused
on-chip levels (heat r = 2, leapfrog r = 1), the SM-resident 2-D kernel, and
the z-slab path with the overlapped exchange (loopback, G = 2).  Test
infrastructure (imports the oracle); not a pytest module.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import _oracle as O  # noqa: E402
import paper_1806_08299_b200 as P  # noqa: E402
from paper_1806_08299_b200 import configs as CF  # noqa: E402
from _common import config_inputs, gpu_run, product_spec  # noqa: E402


def check(name, spec, ext, ref, got, slots, last, levels):
    ok = O.verify_bitwise(spec, ext, ref, slots, got, slots, last, levels) == 1
    print(f"{'ok ' if ok else 'BAD'} {name}", flush=True)
    if not ok:
        sys.exit(1)


def star_cases():
    for cidx, ext, steps in ((2, (20, 37, 140), 6), (3, (26, 34, 136), 5)):
        cfg = CF.get(cidx).scaled(ext, steps)
        dtd = 2 if cfg.model else 1
        for sched, T, tiles, band in (("canonical", 1, (0, 0, 0), 0), ("time", 3, (0, 16, 0), 0),
                                      ("time", 4, (9, 8, 0), 0), ("time", 3, (0, 24, 0), 0),     # 12 warps x 2 rows
                                      ("time", 4, (0, 24, 0), 24), ("time", 3, (11, 16, 0), 16)):  # row-skewed y-bands
            slots = dtd + T
            spec, base, m = config_inputs(cfg, slots)
            ref = base.copy()
            assert O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)[0] == 0
            ps = product_spec(spec)
            canon = P.build_canonical_nest(ps, None)
            nest = canon if sched == "canonical" else P.tile_time(
                canon, ps, None, P.TilePlan(cfg.radius, T, tiles, band_rows=band, band_skew=cfg.radius if band else 0))
            got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, P.MODE_REFERENCE, m, pspec=ps)
            check(f"star config{cidx} {sched} T={T} tiles={tiles} band={band} kind={rep.kernel_kind} "
                  f"tile={tuple(rep.tile)}", spec, ext, ref, got, slots, dtd - 1 + steps, dtd)


def generic_case():
    spec = O.Spec(3, [(0.5, 1, (0, 0, 0)), (0.2, 1, (1, -1, 0)), (0.2, 1, (0, 2, -1)), (0.1, 2, (-1, 0, 1))])
    ext, steps, slots = (12, 17, 45), 5, 2 + 3
    base = O.init_reference(spec, ext, slots, 3)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=8)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(2, 3, (0, 0, 0)))
    got, rep = gpu_run(spec, ext, base, slots, 1, 0, steps, nest, pspec=ps)
    check(f"generic time T=3 kind={rep.kernel_kind}", spec, ext, ref, got, slots, 1 + steps, 2)


def fused_and_resident_cases():
    for cidx, ext, steps, F in ((2, (18, 30, 70), 7, 2), (7, (16, 28, 66), 7, 3), (1, (90, 130), 13, 4)):
        cfg = CF.get(cidx).scaled(ext, steps)
        dtd = 2 if cfg.model else 1
        slots = dtd + F
        spec, base, m = config_inputs(cfg, slots)
        ref = base.copy()
        assert O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)[0] == 0
        ps = product_spec(spec)
        nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None,
                           P.TilePlan(cfg.radius, F, tuple(0 for _ in ext), fused_levels=F))
        got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, P.MODE_REFERENCE, m, pspec=ps)
        assert rep.kernel_kind in (2, 3)
        check(f"on-chip config{cidx} F={F} kind={rep.kernel_kind}", spec, ext, ref, got, slots, dtd - 1 + steps, dtd)


def slab_case():
    from test_gpu_dist import _slab_run
    cfg = CF.get(3).scaled((96, 24, 40), 9)
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    T, G = 2, 2
    slots = 2 + T
    rng = np.random.default_rng(11)
    base = O.new_grid(spec, cfg.extents, slots)
    v = base.reshape((slots,) + spec.padded(cfg.extents))
    R = cfg.radius
    ext = cfg.extents
    for lv in range(2):
        v[lv][R:R + ext[0], R:R + ext[1], R:R + ext[2]] = rng.random(ext, dtype=np.float32)
    m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H)
    ref = base.copy()
    O.execute(spec, ext, ref, slots, 0, cfg.steps, mfield=m, nthreads=8)
    got, rep = _slab_run(spec, product_spec(spec), ext, base, slots, cfg.steps, G, T, 1, m, sched="time")
    check(f"z-slabs G={G} T={T} overlapped exchange, {rep.kernel_launches} launches", spec, ext, ref, got, slots,
          1 + cfg.steps, 2)


if __name__ == "__main__":
    star_cases()
    generic_case()
    fused_and_resident_cases()
    slab_case()
    print("sanitize cases done", flush=True)
