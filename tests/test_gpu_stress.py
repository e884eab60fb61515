"""Randomized end-to-end stress of the executor (GPU): random term sets and
canonical stars (1-3 dims), random extents and step counts, every schedule
(canonical / space-tiled / wavefront / on-chip fused levels) chained over 1-3
resumed segments, device-grid and host-grid (st_execute_host) entry points,
uniform and per-slot (reference init) halos, both arithmetic modes -- each
against the oracle: bitwise in reference mode, <= 1e-5 in FAST mode."""
import random

import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from _common import product_spec, random_spec
from test_gpu_fused import _random_star

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", range(40))
def test_random_schedules_segments_entry_points(case):
    rng = random.Random(31000 + case)
    nrng = np.random.default_rng(31000 + case)
    if case % 3 == 0:
        spec = random_spec(rng)
    else:
        nd = rng.choice([2, 3])
        R = rng.choice([1, 2]) if nd == 3 else rng.choice([1, 2, 4])
        spec = _random_star(nrng, nd, R, bool(case % 2))
    n = spec.ndims
    ext = tuple(rng.randint(1, {1: 300, 2: 90, 3: 30}[n]) for _ in range(n))
    steps = rng.randint(1, 14)
    dtd = spec.time_depth
    smin = max(spec.radius(i) for i in range(n))
    T = rng.choice([1, 2, 3, 4])
    slots = dtd + T
    uniform = rng.random() < 0.6
    base = O.init_reference(spec, ext, slots, 9 + case)
    if uniform:
        base = O.uniform_halo(spec, ext, base, slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=8)[0] == 0
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)

    def pick():
        kind = rng.choice(["canonical", "space", "time", "fused"])
        tiles = tuple(rng.choice([0, rng.randint(1, e + 3)]) for e in ext)
        if kind == "canonical":
            return canon
        if kind == "space":
            return P.tile_space_minmax(canon, tiles)
        F = min(rng.choice([1, 2, 3, 4]), T) if kind == "fused" else 0
        return P.tile_time(canon, ps, None, P.TilePlan(smin, T, tiles, fused_levels=F))

    mode = P.MODE_FAST if (rng.random() < 0.3 and spec.model == 0) else P.MODE_REFERENCE
    cuts = sorted(rng.sample(range(1, steps), min(steps - 1, rng.randint(0, 2)))) if steps > 1 else []
    segs = list(zip([0] + cuts, cuts + [steps]))
    dg = P.DeviceGrid(P.default_context(), ps, ext, slots)
    try:
        if rng.random() < 0.4:
            import torch
            got = torch.empty(base.size, dtype=torch.float32, pin_memory=True).numpy()
            got[:] = base
            for a, b in segs:
                dg.execute_host(got, a, b, pick(), mode, uniform_halo=uniform)
        else:
            dg.upload(base, dtd - 1)
            for a, b in segs:
                dg.apply(a, b, pick(), mode)
            got = base.copy()
            dg.download(got)
    finally:
        dg.close()
    last = dtd - 1 + steps
    if mode == P.MODE_REFERENCE:
        assert O.verify_bitwise(spec, ext, ref, slots, got, slots, last, dtd) == 1, (ext, steps, segs)
    else:
        assert O.max_rel_err(spec, ext, ref, slots, got, slots, last, dtd) <= 1e-5
