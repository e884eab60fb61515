"""GPU parity of the fused-level kernel (on-chip time tile, st_fused.cuh):
F levels per pass over memory with overlapped x/y tiles and trapezoidal z
ranges.  Reference mode is bitwise equal to the oracle; FAST mode is bitwise
equal to the star kernel's FAST mode (same per-point arithmetic) and within
the 1e-5 tolerance of the oracle."""
import dataclasses

import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import config_inputs, gpu_run, product_spec

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-5
KIND_FUSED = 2


def uniform_halo_reference_init(spec, ext, slots, seed):
    """The reference init_grid (LCG values in the halo too), with every slot
    given slot 0's halo: non-zero frozen halos the fused kernel must keep."""
    return O.uniform_halo(spec, ext, O.init_reference(spec, ext, slots, seed), slots)


def fused_nest(ps, F, ty=0, T=4):
    return P.tile_time(P.build_canonical_nest(ps, None), ps, None,
                       P.TilePlan(2, T, (0, ty, 0), fused_levels=F))


@pytest.mark.parametrize("ext,steps", [
    ((19, 75, 260), 9),      # ragged: several row tiles, three x tiles, odd step count
    ((21, 37, 70), 13),
    ((9, 5, 7), 5),          # smaller than one tile in every axis
    ((40, 32, 128), 8),      # exact tiles
    ((3, 130, 129), 4),      # fewer planes than the z trapezoid
])
@pytest.mark.parametrize("F,ty", [(2, 16), (2, 24), (3, 8)])
def test_fused_bitwise_vs_oracle(ext, steps, F, ty):
    cfg = CF.get(2).scaled(ext, steps)
    slots = 1 + 4
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=16)[0] == 0
    ps = product_spec(spec)
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, fused_nest(ps, F, ty), P.MODE_REFERENCE, pspec=ps)
    assert rep.kernel_kind == KIND_FUSED and rep.time_tile_used == F
    assert rep.tile[1] == ty
    assert rep.kernel_launches == -(-steps // F)
    assert O.verify_bitwise(spec, ext, ref, slots, got, slots, steps, 1) == 1, \
        O.max_rel_err(spec, ext, ref, slots, got, slots, steps, 1)


@pytest.mark.parametrize("F", [2, 3])
def test_fused_nonzero_frozen_halo(F):
    """LCG values in the (uniform) halo: every level keeps them frozen."""
    cfg = CF.get(2).scaled((17, 41, 133), 7)
    spec = O.Spec(3, cfg.terms, cfg.model)
    ext = cfg.extents
    slots = 5
    base = uniform_halo_reference_init(spec, ext, slots, 11)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, 7, nthreads=16)[0] == 0
    ps = product_spec(spec)
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, 7, fused_nest(ps, F), P.MODE_REFERENCE, pspec=ps)
    assert rep.kernel_kind == KIND_FUSED
    assert O.verify_bitwise(spec, ext, ref, slots, got, slots, 7, 1) == 1


@pytest.mark.parametrize("F", [2, 3])
def test_fused_fast_equals_star_fast(F):
    cfg = CF.get(2).scaled((23, 70, 200), 10)
    slots = 5
    spec, base, _ = config_inputs(cfg, slots)
    ps = product_spec(spec)
    star_nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(2, 4, (0, 0, 0)))
    a, ra = gpu_run(spec, cfg.extents, base, slots, 0, 0, 10, star_nest, P.MODE_FAST, pspec=ps)
    b, rb = gpu_run(spec, cfg.extents, base, slots, 0, 0, 10, fused_nest(ps, F), P.MODE_FAST, pspec=ps)
    assert ra.kernel_kind == 1 and rb.kernel_kind == KIND_FUSED
    assert ra.mode_used == rb.mode_used == P.MODE_FAST
    assert O.verify_bitwise(spec, cfg.extents, a, slots, b, slots, 10, 1) == 1
    ref = base.copy()
    O.execute(spec, cfg.extents, ref, slots, 0, 10, nthreads=16)
    assert O.max_rel_err(spec, cfg.extents, ref, slots, b, slots, 10, 1) <= FAST_TOL


def test_fused_resume_and_mixed_schedules():
    """[0,5) fused + [5,9) wavefront + [9,14) fused == one canonical run."""
    cfg = CF.get(2).scaled((16, 24, 140), 14)
    slots = 5
    spec, base, _ = config_inputs(cfg, slots)
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)
    one, _ = gpu_run(spec, cfg.extents, base, slots, 0, 0, 14, canon, pspec=ps)
    dg = P.DeviceGrid(P.default_context(), ps, cfg.extents, slots)
    dg.upload(base, 0)
    assert dg.apply(0, 5, fused_nest(ps, 2)).kernel_kind == KIND_FUSED
    assert dg.apply(5, 9, P.tile_time(canon, ps, None, P.TilePlan(2, 4, (0, 0, 0)))).kernel_kind == 1
    assert dg.apply(9, 14, fused_nest(ps, 3)).kernel_kind == KIND_FUSED
    two = base.copy()
    assert dg.download(two) == 14
    dg.close()
    assert O.verify_bitwise(spec, cfg.extents, one, slots, two, slots, 14, 1) == 1


def test_fused_full_config2():
    """Config 2 at full size and step count (256^3 x 64), F = 2: bitwise."""
    cfg = CF.get(2)
    slots = 5
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, cfg.extents, ref, slots, 0, cfg.steps, nthreads=32)[0] == 0
    ps = product_spec(spec)
    got, rep = gpu_run(spec, cfg.extents, base, slots, 0, 0, cfg.steps, fused_nest(ps, 2), P.MODE_REFERENCE,
                       pspec=ps)
    assert rep.kernel_kind == KIND_FUSED
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, got, slots, cfg.steps, 1) == 1


def test_fused_execute_host():
    """st_execute_host (host grid, overlapped copies) with a fused plan."""
    cfg = CF.get(2).scaled((30, 50, 260), 9)
    slots = 5
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    O.execute(spec, cfg.extents, ref, slots, 0, 9, nthreads=16)
    ps = product_spec(spec)
    import torch
    host = torch.empty(base.size, dtype=torch.float32, pin_memory=True).numpy()
    host[:] = base
    dg = P.DeviceGrid(P.default_context(), ps, cfg.extents, slots)
    for _ in range(2):   # twice: the spare buffer exists (and must be refreshed) the second time
        host[:] = base
        rep = dg.execute_host(host, 0, 9, fused_nest(ps, 2), P.MODE_REFERENCE, uniform_halo=True)
        assert rep.kernel_kind == KIND_FUSED
        assert O.verify_bitwise(spec, cfg.extents, ref, slots, host, slots, 9, 1) == 1
    dg.close()


def test_fused_falls_back_without_uniform_halo():
    """Per-slot halos (the literal reference init) need the halo bank: the
    plan runs on the wavefront instead, still bitwise."""
    cfg = CF.get(2).scaled((12, 20, 40), 6)
    spec = O.Spec(3, cfg.terms, cfg.model)
    slots = 5
    base = O.init_reference(spec, cfg.extents, slots, 3)
    ref = base.copy()
    O.execute(spec, cfg.extents, ref, slots, 0, 6, nthreads=16)
    ps = product_spec(spec)
    got, rep = gpu_run(spec, cfg.extents, base, slots, 0, 0, 6, fused_nest(ps, 2), pspec=ps)
    assert rep.kernel_kind == 1
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, got, slots, 6, 1) == 1


# ---------------------------------------------------------------- 2-D ------
KIND_RESIDENT = 3


def heat2d(R):
    """2-D heat star of radius R (config 1 for R = 1; stable weights otherwise)."""
    if R == 1:
        return CF.get(1)
    w = {2: [0.08, -0.005], 4: [0.05, -0.01, 0.004, -0.001]}[R]
    centre = 1.0 - 4 * sum(w)
    return dataclasses.replace(CF.get(1), terms=CF.star_terms(2, centre, w), radius=R)


@pytest.mark.parametrize("R,ext,steps,F", [
    (1, (67, 131), 21, 4),
    (1, (67, 131), 21, 1),
    (1, (5, 7), 9, 3),             # fewer rows than CTAs
    (1, (300, 1030), 17, 8),       # ragged x (not a multiple of 4), several exchanges
    (2, (150, 200), 13, 5),
    (4, (90, 64), 7, 2),
    (2, (40, 400), 11, 8),         # halo ring deeper than a tile: several owners per side
])
@pytest.mark.parametrize("mode", [P.MODE_REFERENCE, P.MODE_FAST])
@pytest.mark.parametrize("gx", [0, 1, 3, 16])
def test_resident2d_vs_oracle(R, ext, steps, F, mode, gx, monkeypatch):
    """SM-resident 2-D kernel vs the oracle; gx forces the column tiles
    (ST_RES_GX; 0 = the cost model's choice, 1 = row strips)."""
    nx4 = (ext[1] + 3) // 4
    if gx:
        monkeypatch.setenv("ST_RES_GX", str(min(gx, nx4, 16)))
    cfg = heat2d(R).scaled(ext, steps)
    slots = 1 + F
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=16)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(R, F, (0, 0), fused_levels=F))
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, mode, pspec=ps)
    assert rep.kernel_kind == KIND_RESIDENT and rep.kernel_launches == 1
    if gx:
        assert rep.tile[2] == 4 * -(-nx4 // min(gx, nx4, 16))
    if mode == P.MODE_REFERENCE:
        assert O.verify_bitwise(spec, ext, ref, slots, got, slots, steps, 1) == 1, \
            O.max_rel_err(spec, ext, ref, slots, got, slots, steps, 1)
    else:
        assert O.max_rel_err(spec, ext, ref, slots, got, slots, steps, 1) <= FAST_TOL


@pytest.mark.parametrize("R,ext,F,gx", [
    (4, (248, 137), 15, 0),    # the planner's own choice: a middle tile reaches the grid edge
    (2, (1106, 371), 21, 0),
    (1, (64, 64), 4, 9),       # forced narrow column tiles: halo ring wider than a tile
    (4, (300, 200), 24, 13),
    (4, (97, 61), 30, 16),
    (2, (500, 90), 40, 11),
])
def test_resident2d_smem_sizing_regressions(R, ext, F, gx, monkeypatch):
    """Tiles that are neither first nor last yet reach the grid edge take the
    whole frozen halo (st_resident.cuh lcs/lce): the plan must reserve the
    shared memory the kernel indexes (the kernel traps if not)."""
    if gx:
        monkeypatch.setenv("ST_RES_GX", str(min(gx, (ext[1] + 3) // 4)))
    steps = F + 3
    cfg = heat2d(R).scaled(ext, steps)
    slots = 1 + F
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=16)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(R, F, (0, 0), fused_levels=F))
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, P.MODE_REFERENCE, pspec=ps)
    assert rep.kernel_kind == KIND_RESIDENT
    assert O.verify_bitwise(spec, ext, ref, slots, got, slots, steps, 1) == 1


def test_resident2d_full_config1_and_halo():
    """Config 1 at full size (1024^2 x 100, F = 8) bitwise; then LCG values in
    a uniform halo stay frozen."""
    cfg = CF.get(1)
    slots = 9
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, cfg.extents, ref, slots, 0, cfg.steps, nthreads=32)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(1, 8, (0, 0), fused_levels=8))
    got, rep = gpu_run(spec, cfg.extents, base, slots, 0, 0, cfg.steps, nest, pspec=ps)
    assert rep.kernel_kind == KIND_RESIDENT
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, got, slots, cfg.steps, 1) == 1
    ext = (200, 77)
    base = uniform_halo_reference_init(spec, ext, slots, 5)
    ref = base.copy()
    O.execute(spec, ext, ref, slots, 0, 30, nthreads=16)
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, 30, nest, pspec=ps)
    assert rep.kernel_kind == KIND_RESIDENT
    assert O.verify_bitwise(spec, ext, ref, slots, got, slots, 30, 1) == 1


def test_resident2d_resume_and_execute_host():
    cfg = CF.get(1).scaled((130, 260), 20)
    slots = 5
    spec, base, _ = config_inputs(cfg, slots)
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)
    one, _ = gpu_run(spec, cfg.extents, base, slots, 0, 0, 20, canon, pspec=ps)
    nest = P.tile_time(canon, ps, None, P.TilePlan(1, 4, (0, 0), fused_levels=4))
    dg = P.DeviceGrid(P.default_context(), ps, cfg.extents, slots)
    dg.upload(base, 0)
    assert dg.apply(0, 7, nest).kernel_kind == KIND_RESIDENT
    assert dg.apply(7, 11, canon).kernel_kind == 1
    assert dg.apply(11, 20, nest).kernel_kind == KIND_RESIDENT
    two = base.copy()
    assert dg.download(two) == 20
    assert O.verify_bitwise(spec, cfg.extents, one, slots, two, slots, 20, 1) == 1
    import torch
    host = torch.empty(base.size, dtype=torch.float32, pin_memory=True).numpy()
    host[:] = base
    rep = dg.execute_host(host, 0, 20, nest, P.MODE_REFERENCE, uniform_halo=True)
    assert rep.kernel_kind == KIND_RESIDENT
    assert O.verify_bitwise(spec, cfg.extents, one, slots, host, slots, 20, 1) == 1
    dg.close()


# ------------------------------------------------------- randomized --------
def _random_star(rng, ndims, R, symmetric):
    """A stable random heat-model star of radius R in canonical term order."""
    w = [float(np.float32(rng.uniform(0.01, 0.08) / k)) for k in range(1, R + 1)]
    terms = [(0.0, 1, (0,) * ndims)]
    total = 0.0
    for a in range(ndims):
        for k in range(1, R + 1):
            for sgn in (-1, 1):
                c = w[k - 1] if symmetric else float(np.float32(w[k - 1] * rng.uniform(0.8, 1.2)))
                off = [0] * ndims
                off[a] = sgn * k
                terms.append((c, 1, tuple(off)))
                total += c
    terms[0] = (float(np.float32(1.0 - total)), 1, (0,) * ndims)
    return O.Spec(ndims, terms)


@pytest.mark.parametrize("case", range(14))
def test_fused_random_extents_and_stencils(case):
    """Random extents (smaller and larger than a tile in every axis), step
    counts, F, tile heights and coefficient sets, random uniform halos:
    bitwise vs the oracle; FAST (symmetric sets only) within 1e-5.  Radius 2
    (F = 2, 3; tile heights 16 / 24 / 8) and radius 1 (F = 2, 3, 4)."""
    rng = np.random.default_rng(5000 + case)
    ext = (int(rng.integers(1, 40)), int(rng.integers(1, 90)), int(rng.integers(1, 300)))
    steps = int(rng.integers(1, 12))
    R, F, ty = [(2, 2, 16), (2, 2, 24), (2, 3, 8), (1, 2, 0), (1, 3, 0), (1, 4, 0), (2, 2, 0)][case % 7]
    sym = bool(case % 2)
    spec = _random_star(rng, 3, R, sym)
    slots = 1 + F
    base = O.uniform_halo(spec, ext, O.init_reference(spec, ext, slots, 77 + case), slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=16)[0] == 0
    ps = product_spec(spec)
    for mode in ((P.MODE_REFERENCE, P.MODE_FAST) if sym else (P.MODE_REFERENCE,)):
        nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(R, F, (0, ty, 0), fused_levels=F))
        got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, mode, pspec=ps)
        assert rep.kernel_kind == KIND_FUSED, (ext, steps, F)
        if mode == P.MODE_REFERENCE:
            assert O.verify_bitwise(spec, ext, ref, slots, got, slots, steps, 1) == 1, (ext, steps, F, ty)
        else:
            assert O.max_rel_err(spec, ext, ref, slots, got, slots, steps, 1) <= FAST_TOL


@pytest.mark.parametrize("case", range(16))
def test_resident2d_random_extents_and_stencils(case, monkeypatch):
    """Random extents, radii, F and stencils; every other case forces a
    random column-tile count (2-D tiles instead of the model's choice)."""
    rng = np.random.default_rng(6000 + case)
    R = [1, 2, 4][case % 3]
    ext = (int(rng.integers(1, 400)), int(rng.integers(1, 1200)))
    steps = int(rng.integers(1, 30))
    F = int(rng.integers(1, 9))
    gx = int(rng.integers(1, 17))
    if case % 2 == 0:
        monkeypatch.setenv("ST_RES_GX", str(min(gx, (ext[1] + 3) // 4)))
    sym = bool(case % 2)
    spec = _random_star(rng, 2, R, sym)
    slots = 1 + F
    base = O.uniform_halo(spec, ext, O.init_reference(spec, ext, slots, 91 + case), slots)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, nthreads=16)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(R, F, (0, 0), fused_levels=F))
    for mode in ((P.MODE_REFERENCE, P.MODE_FAST) if sym else (P.MODE_REFERENCE,)):
        got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, mode, pspec=ps)
        assert rep.kernel_kind == KIND_RESIDENT, (ext, steps, F, R)
        if mode == P.MODE_REFERENCE:
            assert O.verify_bitwise(spec, ext, ref, slots, got, slots, steps, 1) == 1, (ext, steps, F, R)
        else:
            assert O.max_rel_err(spec, ext, ref, slots, got, slots, steps, 1) <= FAST_TOL


def test_fused_study_config6_full_size():
    """The study workload beyond BASELINE's configs (3-D heat so2, 512^3 x 48)
    at full size under its bench plan (3 levels per pass on-chip, 24-row
    tiles): bitwise in reference mode, within 1e-5 in FAST mode."""
    cfg = CF.get(6)
    bp = CF.BENCH_PLANS[6]
    slots = 1 + bp["time_tile"]
    spec, base, _ = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, cfg.extents, ref, slots, 0, cfg.steps, nthreads=32)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None,
                       P.TilePlan(1, bp["time_tile"], bp["tiles"], fused_levels=bp["fused"]))
    got, rep = gpu_run(spec, cfg.extents, base, slots, 0, 0, cfg.steps, nest, P.MODE_REFERENCE, pspec=ps)
    assert rep.kernel_kind == KIND_FUSED and rep.time_tile_used == 3 and rep.tile[1] == 24
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, got, slots, cfg.steps, 1) == 1
    fast, rep = gpu_run(spec, cfg.extents, base, slots, 0, 0, cfg.steps, nest, P.MODE_FAST, pspec=ps)
    assert rep.mode_used == P.MODE_FAST
    assert O.max_rel_err(spec, cfg.extents, ref, slots, fast, slots, cfg.steps, 1) <= FAST_TOL


# ------------------------------------------------------------ wave ---------
def wave_cfg(order, ext, steps, field="layered"):
    """The config 3 leapfrog (layered or random m field) at space order 2 / 4:
    the radii the fused wave kernel is built for."""
    terms, r = CF.wave3d(order)
    base = CF.get(3) if field == "layered" else CF.get(4)
    return dataclasses.replace(base, terms=terms, radius=r, skew=r, extents=tuple(ext), steps=steps)


@pytest.mark.parametrize("order,F", [(2, 1), (2, 2), (2, 3), (4, 1), (4, 2), (8, 2)])
@pytest.mark.parametrize("ext,steps,field", [((20, 37, 70), 9, "layered"), ((9, 5, 7), 5, "random"),
                                            ((33, 41, 260), 7, "random")])
def test_fused_wave_bitwise(order, F, ext, steps, field):
    """Fused levels for the leapfrog: two input levels, two output levels per
    pass; u^{n-1} and m tiles ride in the TMA ring.  Random interiors in both
    starting levels (waves reach the boundary): bitwise vs the oracle."""
    cfg = wave_cfg(order, ext, steps, field)
    slots = 2 + F
    spec, base, m = config_inputs(cfg, slots)
    rng = np.random.default_rng(order * 10 + F)
    v = base.reshape((slots,) + spec.padded(ext))
    inner = tuple(slice(cfg.radius, cfg.radius + e) for e in ext)
    for lv in range(2):
        v[lv][inner] = rng.random(ext, dtype=np.float32)
    ref = base.copy()
    assert O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=16)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None,
                       P.TilePlan(cfg.radius, F, (0, 0, 0), fused_levels=F))
    for mode in (P.MODE_REFERENCE, P.MODE_FAST):
        got, rep = gpu_run(spec, ext, base, slots, 1, 0, steps, nest, mode, m, pspec=ps)
        assert rep.kernel_kind == KIND_FUSED and rep.time_tile_used == F
        if mode == P.MODE_REFERENCE:
            assert O.verify_bitwise(spec, ext, ref, slots, got, slots, 1 + steps, 2) == 1, \
                O.max_rel_err(spec, ext, ref, slots, got, slots, 1 + steps, 2)
        else:
            assert O.max_rel_err(spec, ext, ref, slots, got, slots, 1 + steps, 2) <= FAST_TOL


def test_fused_wave_resume_and_mixed():
    """[0,4) fused F=2 + [4,7) wavefront + [7,12) fused F=3 (so2 wave)."""
    cfg = wave_cfg(2, (24, 30, 140), 12)
    slots = 5
    spec, base, m = config_inputs(cfg, slots)
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)
    one, _ = gpu_run(spec, cfg.extents, base, slots, 1, 0, 12, canon, P.MODE_REFERENCE, m, pspec=ps)
    dg = P.DeviceGrid(P.default_context(), ps, cfg.extents, slots)
    dg.upload(base, 1)
    dg.set_field(m)
    assert dg.apply(0, 4, P.tile_time(canon, ps, None, P.TilePlan(1, 2, (0, 0, 0), fused_levels=2))).kernel_kind == 2
    assert dg.apply(4, 7, P.tile_time(canon, ps, None, P.TilePlan(1, 3, (0, 0, 0)))).kernel_kind == 1
    assert dg.apply(7, 12, P.tile_time(canon, ps, None, P.TilePlan(1, 3, (0, 0, 0), fused_levels=3))).kernel_kind == 2
    two = base.copy()
    assert dg.download(two) == 13
    dg.close()
    assert O.verify_bitwise(spec, cfg.extents, one, slots, two, slots, 13, 2) == 1


def test_fused_study_config7_full_size():
    """Study workload 7 (the config 3 leapfrog at space order 2, 512^3 x 48)
    at full size under its bench plan (fused F = 3): bitwise."""
    cfg = CF.get(7)
    bp = CF.BENCH_PLANS[7]
    slots = 2 + bp["time_tile"]
    spec, base, m = config_inputs(cfg, slots)
    ref = base.copy()
    assert O.execute(spec, cfg.extents, ref, slots, 0, cfg.steps, mfield=m, nthreads=32)[0] == 0
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None,
                       P.TilePlan(1, bp["time_tile"], bp["tiles"], fused_levels=bp["fused"]))
    got, rep = gpu_run(spec, cfg.extents, base, slots, 1, 0, cfg.steps, nest, P.MODE_REFERENCE, m, pspec=ps)
    assert rep.kernel_kind == KIND_FUSED and rep.time_tile_used == 3
    assert O.verify_bitwise(spec, cfg.extents, ref, slots, got, slots, 1 + cfg.steps, 2) == 1
