"""GPU parity of st_execute_host: execute (executor.hpp:92-98) on a HOST grid
(copy-engine upload blocks converted on the GPU, pitched 2D download).

The host grid's newest delta_t levels must equal the oracle bitwise, every
other slot must be untouched, and two grids driven concurrently from two
threads (overlapping one another's copies and kernels) must both be exact.
"""
import numpy as np
import pytest
import torch

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import config_inputs, gpu_run, product_spec

pytestmark = pytest.mark.gpu


_PINNED = []   # keeps the page-locked allocations alive for the module


def pinned_copy(a: np.ndarray) -> np.ndarray:
    t = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
    _PINNED.append(t)
    out = t.numpy()
    out[:] = a.reshape(-1)
    return out


def exec_host(spec, ext, host, t_begin, t_end, nest, mode=P.MODE_REFERENCE, m=None, slots=None, ctx=None):
    ps = product_spec(spec)
    dg = P.DeviceGrid(ctx or P.default_context(), ps, ext, slots)
    try:
        if m is not None:
            dg.set_field(m)
        rep = dg.execute_host(host, t_begin, t_end, nest, mode, uniform_halo=True)
        assert dg.last_level() == t_end + ps.time_depth - 1
    finally:
        dg.close()
    return rep


def _nests(ps, radius):
    canon = P.build_canonical_nest(ps, None)
    return {
        "canonical": canon,
        "time4": P.tile_time(canon, ps, None, P.TilePlan(radius, 4, (0, 0, 0))),
        "time8_long": P.tile_time(canon, ps, None, P.TilePlan(radius, 8, (4096, 32, 0))),
        "time3_chunks": P.tile_time(canon, ps, None, P.TilePlan(radius + 1, 3, (9, 16, 0))),
    }


@pytest.mark.parametrize("cidx,ext,steps", [
    (2, (37, 70, 150), 13),      # heat so4, delta_t = 1
    (3, (30, 41, 136), 9),       # wave so8, delta_t = 2 (+ m field)
])
@pytest.mark.parametrize("mode", [P.MODE_REFERENCE, P.MODE_FAST])
def test_execute_host_matches_oracle(cidx, ext, steps, mode):
    cfg = CF.get(cidx).scaled(ext, steps)
    dtd = 2 if cfg.model else 1
    slots = dtd + 8
    spec, base, m = config_inputs(cfg, slots)
    ref = base.copy()
    rc, _, _ = O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=16)
    assert rc == 0
    ps = product_spec(spec)
    last = dtd - 1 + steps
    out_slots = {(steps + i) % slots for i in range(dtd)}
    for name, nest in _nests(ps, cfg.radius).items():
        host = pinned_copy(base)
        rep = exec_host(spec, ext, host, 0, steps, nest, mode, m, slots)
        assert rep.points_updated == steps * int(np.prod(ext))
        if mode == P.MODE_REFERENCE:
            assert O.verify_bitwise(spec, ext, ref, slots, host, slots, last, dtd) == 1, name
        else:
            err = O.max_rel_err(spec, ext, ref, slots, host, slots, last, dtd)
            assert err <= (1e-5 if cidx == 2 else 1e-4), (name, err)
        hv = host.reshape((slots, -1))
        bv = base.reshape((slots, -1))
        for s in range(slots):
            if s not in out_slots:
                assert np.array_equal(hv[s].view(np.uint32), bv[s].view(np.uint32)), (name, s)
        if mode == P.MODE_REFERENCE:   # whole output slots, halos included, equal the oracle's
            rv = ref.reshape((slots, -1))
            for s in out_slots:
                assert np.array_equal(hv[s].view(np.uint32), rv[s].view(np.uint32)), (name, s)


def test_execute_host_pageable_and_resume():
    """Pageable host memory takes the staged path; two chained calls equal
    one call (continuation through the host grid)."""
    cfg = CF.get(2).scaled((24, 33, 70), 10)
    slots = 1 + 4
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    rc, _, _ = O.execute(spec, cfg.extents, ref, slots, 0, 10, nthreads=16)
    assert rc == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(2, 4, (0, 0, 0)))
    pageable = base.copy()
    exec_host(spec, cfg.extents, pageable, 0, 10, nest, slots=slots)   # staged fallback
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, pageable, slots, 10, 1) == 1
    host = pinned_copy(base)
    exec_host(spec, cfg.extents, host, 0, 4, nest, slots=slots)
    exec_host(spec, cfg.extents, host, 4, 10, nest, slots=slots)
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, host, slots, 10, 1) == 1


def test_execute_host_full_size_bench_plan():
    """Config 2 at full size with the bench plan: the host execute equals
    st_apply + download bitwise (FAST mode, as benchmarked), also with two
    grids running concurrently."""
    cfg = CF.get(2)
    bp = CF.BENCH_PLANS[2]
    slots = 1 + bp["time_tile"]
    spec, base, _ = config_inputs(cfg, slots)
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(cfg.radius, bp["time_tile"], bp["tiles"]))
    want, _ = gpu_run(spec, cfg.extents, base, slots, 0, 0, cfg.steps, nest, P.MODE_FAST, pspec=ps)
    # two grids on two contexts, driven concurrently from two threads, twice
    from concurrent.futures import ThreadPoolExecutor
    ctxs = [P.default_context(), P.Context(0)]
    hosts = [pinned_copy(base), pinned_copy(base)]
    try:
        with ThreadPoolExecutor(2) as ex:
            for _ in range(2):
                list(ex.map(lambda i: exec_host(spec, cfg.extents, hosts[i], 0, cfg.steps, nest, P.MODE_FAST,
                                                slots=slots, ctx=ctxs[i]), range(2)))
                for h in hosts:
                    assert O.verify_bitwise(spec, cfg.extents, want, slots, h, slots, cfg.steps, 1) == 1
                    h[:] = base.reshape(-1)
    finally:
        ctxs[1].close()
