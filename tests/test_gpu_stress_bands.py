"""Randomized stress of the round-2b paths of the star wavefront (GPU): the
radius-4 leapfrog and the radius-2 / radius-8 stencils on random ragged
extents, every compiled tile height (8 / 12 / 16 / 24 / 32 rows), random
time tiles, z-chunks and row-skewed y-bands (st_plan.band_rows / band_skew),
runs split into resumed segments -- each bitwise equal to the oracle in
reference mode; in FAST mode bitwise equal to the unbanded whole-depth FAST
run of the same grid (same arithmetic, another order of items).

ST_STRESS_CASES=<n> widens the corpus for scratch runs (default 40).
"""
import os
import random

import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import config_inputs, gpu_run, product_spec

pytestmark = pytest.mark.gpu
NCASES = int(os.environ.get("ST_STRESS_CASES", "40"))


@pytest.mark.parametrize("case", range(NCASES))
def test_random_plans_star_wavefront(case):
    rng = random.Random(52000 + case)
    cidx = rng.choice([3, 3, 3, 2, 2, 4])
    ext = (rng.randint(3, 44), rng.randint(5, 130), rng.randint(8, 300))
    steps = rng.randint(1, 12)
    cfg = CF.get(cidx).scaled(ext, steps)
    R = cfg.radius
    dtd = 2 if cfg.model else 1
    T = rng.choice([1, 2, 3, 4, 5, 8])
    slots = dtd + T
    spec, base, m = config_inputs(cfg, slots)
    nrng = np.random.default_rng(52000 + case)
    v = base.reshape((slots,) + spec.padded(ext))
    inner = tuple(slice(R, R + e) for e in ext)
    for lv in range(dtd):   # random interiors: boundaries and band edges carry signal
        v[lv][inner] = nrng.random(ext, dtype=np.float32)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)[0] == 0
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)

    def plan():
        ty = rng.choice([0, 8, 12, 16, 24, 32])
        cz = rng.choice([0, 4096, rng.randint(1, ext[0] + 6)])
        band = rng.choice([0, 0, rng.randint(8, 140)])
        skew = rng.choice([0, R, rng.randint(1, 24)])
        return P.TilePlan(R, T, (cz, ty, 0), band_rows=band, band_skew=skew if band else 0)

    cuts = sorted(rng.sample(range(1, steps), min(steps - 1, rng.randint(0, 2)))) if steps > 1 else []
    segs = list(zip([0] + cuts, cuts + [steps]))
    last = dtd - 1 + steps
    ctx = P.default_context()

    def run(mode, plans):
        dg = P.DeviceGrid(ctx, ps, ext, slots)
        try:
            dg.upload(base, dtd - 1)
            if m is not None:
                dg.set_field(m)
            for (a, b), pl in zip(segs, plans):
                rep = dg.apply(a, b, P.tile_time(canon, ps, None, pl), mode)
                assert rep.kernel_kind == 1 and rep.points_updated == (b - a) * int(np.prod(ext))
            out = base.copy()
            assert dg.download(out) == last
        finally:
            dg.close()
        return out

    plans = [plan() for _ in segs]
    got = run(P.MODE_REFERENCE, plans)
    assert O.verify_bitwise(spec, ext, ref, slots, got, slots, last, dtd) == 1, \
        (case, cidx, ext, steps, T, plans, O.max_rel_err(spec, ext, ref, slots, got, slots, last, dtd))
    if case % 3 == 0:   # FAST: the plan must not change a bit either
        fast = run(P.MODE_FAST, plans)
        plain = run(P.MODE_FAST, [P.TilePlan(R, T, (4096, 0, 0)) for _ in segs])
        assert np.array_equal(fast, plain), (case, cidx, ext, steps, T, plans)
