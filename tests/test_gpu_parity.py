"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle
on the same seeded inputs.  Bitwise in reference mode; <= 1e-5 relative to
the field's max magnitude in fast mode (BASELINE.json north_star tolerance).
"""
import random

import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import config_inputs, gpu_run, product_spec, random_spec

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-5


def oracle_run(spec, ext, grid, slots, t0, t1, m=None, nthreads=16):
    g = grid.copy()
    rc, _, _ = O.execute(spec, ext, g, slots, t0, t1, mfield=m, nthreads=nthreads)
    assert rc == 0
    return g


def nests(spec_p, ext, radius, tiles=None, Ts=(1, 2, 4, 8)):
    n = len(ext)
    tiles = tiles or tuple(max(1, e // 2) for e in ext)
    out = [("canonical", P.build_canonical_nest(spec_p, None)),
           ("space", P.tile_space_minmax(P.build_canonical_nest(spec_p, None), tiles))]
    for T in Ts:
        out.append((f"time{T}", P.tile_time(P.build_canonical_nest(spec_p, None), spec_p, None,
                                            P.TilePlan(radius, T, tiles))))
    return out


def check(spec, ext, got, gs, ref, rs, last, levels, tol=0.0):
    if tol == 0.0:
        assert O.verify_bitwise(spec, ext, ref, rs, got, gs, last, levels) == 1, \
            f"max rel err {O.max_rel_err(spec, ext, ref, rs, got, gs, last, levels)}"
    else:
        err = O.max_rel_err(spec, ext, ref, rs, got, gs, last, levels)
        assert err <= tol, err


@pytest.mark.parametrize("cfg_idx,ext,steps", [
    (1, (67, 131), 21),          # heat 2D so2, non-dividing extents
    (2, (21, 37, 70), 13),       # heat 3D so4
    (3, (24, 33, 70), 11),       # wave so8
    (4, (20, 35, 40), 7),        # wave so16
])
@pytest.mark.parametrize("mode", [P.MODE_REFERENCE, P.MODE_FAST])
@pytest.mark.parametrize("per_level", [False, True])
def test_config_stencils_all_schedules(cfg_idx, ext, steps, mode, per_level, monkeypatch):
    """Every config stencil under canonical, space and time schedules; 3-D
    canonical / space run as one persistent level-major launch by default,
    per_level = True forces one launch per level (ST_CANON_SWEEP=1)."""
    if per_level:
        monkeypatch.setenv("ST_CANON_SWEEP", "1")
    cfg = CF.get(cfg_idx).scaled(ext, steps)
    dtd = 2 if cfg.model else 1
    slots = dtd + 8
    spec, base, m = config_inputs(cfg, slots)
    if cfg.init == "gaussian":  # small grids: make the boundary matter too
        rng = np.random.default_rng(cfg_idx)
        v = base.reshape((slots,) + spec.padded(ext))
        inner = tuple(slice(r, r + e) for r, e in zip([cfg.radius] * 3, ext))
        for lv in range(dtd):
            v[lv][inner] = rng.random(ext, dtype=np.float32)
    ref = oracle_run(spec, ext, base, slots, 0, steps, m)
    last = dtd - 1 + steps
    ps = product_spec(spec)
    for name, nest in nests(ps, ext, cfg.radius):
        got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, mode, m, pspec=ps)
        assert rep.kernel_kind == 1, name                  # the star kernel ran
        if nest.schedule != P.SCHED_TIME:
            persistent = cfg.ndims == 3 and not per_level
            assert (rep.kernel_launches == 1) == persistent, (name, rep.kernel_launches)
        if mode == P.MODE_REFERENCE:
            assert rep.mode_used == P.MODE_REFERENCE
            check(spec, ext, got, slots, ref, slots, last, dtd)
        else:
            check(spec, ext, got, slots, ref, slots, last, dtd, FAST_TOL)
        assert rep.points_updated == steps * int(np.prod(ext))


@pytest.mark.parametrize("case", range(20))
def test_random_corpus_reference_init(case):
    """SPEC.md:656 corpus (1-3 dims, radius <= 4, delta_t <= 2, k <= 9) with
    the reference init_grid (LCG incl. halo, per-slot halos): GPU == oracle
    bitwise for the same slot count, for every schedule."""
    rng = random.Random(900 + case)
    spec = random_spec(rng)
    ext = tuple(rng.randint(1, {1: 200, 2: 40, 3: 20}[spec.ndims]) for _ in range(spec.ndims))
    steps = rng.randint(1, 9)
    dtd = spec.time_depth
    smin = max(spec.radius(i) for i in range(spec.ndims))
    ps = product_spec(spec)
    for T in (1, 2, 4):
        slots = dtd + T
        base = O.init_reference(spec, ext, slots, 31 + case)
        ref = oracle_run(spec, ext, base, slots, 0, steps)
        tiles = tuple(rng.randint(1, e + 3) for e in ext)
        for nest in (P.build_canonical_nest(ps, None), P.tile_space_minmax(P.build_canonical_nest(ps, None), tiles),
                     P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(smin, T, tiles))):
            got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, pspec=ps)
            check(spec, ext, got, slots, ref, slots, dtd - 1 + steps, dtd)


def test_resume_equals_single_run():
    cfg = CF.get(2).scaled((16, 24, 40), 12)
    spec, base, _ = config_inputs(cfg, 5)
    ps = product_spec(spec)
    ctx = P.default_context()
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(2, 4, (0, 0, 0)))
    one, _ = gpu_run(spec, cfg.extents, base, 5, 0, 0, 12, nest, pspec=ps)
    dg = P.DeviceGrid(ctx, ps, cfg.extents, 5)
    dg.upload(base, 0)
    dg.apply(0, 5, nest)
    dg.apply(5, 12, nest)
    two = base.copy()
    assert dg.download(two) == 12
    dg.close()
    assert O.verify_bitwise(spec, cfg.extents, one, 5, two, 5, 12, 1) == 1


def test_errors_mirror_reference():
    spec = O.Spec(2, [(0.5, 1, (0, 0)), (0.25, 1, (1, 0)), (0.25, 1, (-1, 0))])
    ps = product_spec(spec)
    with pytest.raises(P.Error) as e:
        P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(0, 2, (4, 4)))
    assert e.value.code == 2
    ctx = P.default_context()
    dg = P.DeviceGrid(ctx, ps, (8, 8), 2)
    base = O.init_reference(spec, (8, 8), 2, 1)
    dg.upload(base, 0)
    nest = P.LoopNest(P.SCHED_TIME, P.TilePlan(1, 4, (4, 4)))
    with pytest.raises(P.Error) as e:          # 2 slots < delta_t + t_t = 5
        dg.apply(0, 4, nest)
    assert e.value.code == 3
    with pytest.raises(P.Error) as e:          # does not continue last_level
        dg.apply(3, 4, P.build_canonical_nest(ps, None))
    assert e.value.code == 3
    dg.close()


def test_execute_reference_api_roundtrip():
    """The reference call sequence (SPEC.md:620-622 / SURVEY 3.1) end to end."""
    spec_p, space = P.parse_spec("stencil lap\ndims 2\nextent 33 47\nsteps 9\n"
                                 "term 0.6 1 0 0\nterm 0.1 1 -1 0\nterm 0.1 1 1 0\nterm 0.1 1 0 -1\nterm 0.1 1 0 1\n")
    nest = P.build_canonical_nest(spec_p, space)
    tt = P.tile_time(nest, spec_p, space, P.TilePlan(P.min_skew_factor(spec_p), 4, (8, 8)))
    a = P.init_grid(spec_p, space, 7, P.required_slots(nest, spec_p))
    b = P.init_grid(spec_p, space, 7, P.required_slots(tt, spec_p))
    # uniform halos so the slot counts are comparable (DESIGN.md ledger)
    for g in (a, b):
        v = g.view()
        for s in range(1, g.layout.slots):
            m = np.ones(g.layout.padded, bool)
            m[1:-1, 1:-1] = False
            v[s][m] = v[0][m]
    ra = P.execute(nest, spec_p, space, a)
    rb = P.execute(tt, spec_p, space, b)
    assert ra.points_updated == rb.points_updated == 9 * 33 * 47
    assert ra.flops == ra.points_updated * P.flops_per_point(spec_p)
    assert P.verify_bitwise(a, b, spec_p.time_depth)
    # and both equal the oracle
    ospec = O.Spec(2, [(t.coeff, t.dt, t.offsets) for t in spec_p.terms])
    c = P.init_grid(spec_p, space, 7, 2)
    v = c.view()
    m = np.ones(c.layout.padded, bool)
    m[1:-1, 1:-1] = False
    v[1][m] = v[0][m]
    ref = c.data.copy()
    O.execute(ospec, (33, 47), ref, 2, 0, 9)
    assert O.verify_bitwise(ospec, (33, 47), ref, 2, a.data, a.layout.slots, 9, 1) == 1


@pytest.mark.parametrize("cfg_idx,ext,steps", [
    (2, (19, 75, 260), 9),       # heat so4: several 8/16/32-row tiles and two x tiles, ragged
    (3, (18, 41, 136), 6),       # wave so8
    (4, (14, 41, 136), 4),       # wave so16: 8-row (V0) and 12-row (V7) shapes
])
@pytest.mark.parametrize("ty", [8, 16, 24, 32, 0])
def test_every_tile_shape(cfg_idx, ext, steps, ty):
    """The d_2 space tile selects the compiled CTA tile shape (8 / 16 / 32
    rows: variants V2, V0, V4 for r = 2; 8 / 16 / 24 rows for the r = 4 wave:
    V2, V0, V11 or V8 (m as codes or floats); 8 / 12 rows for r = 8); every one of them, in the sweep and in the wavefront, is bitwise
    equal to the oracle."""
    cfg = CF.get(cfg_idx).scaled(ext, steps)
    dtd = 2 if cfg.model else 1
    slots = dtd + 4
    spec, base, m = config_inputs(cfg, slots)
    ref = oracle_run(spec, ext, base, slots, 0, steps, m)
    ps = product_spec(spec)
    canon = P.build_canonical_nest(ps, None)
    for nest in (P.tile_space_minmax(canon, (0, ty, 0)),
                 P.tile_time(canon, ps, None, P.TilePlan(cfg.radius, 4, (7, ty, 0))),
                 P.tile_time(canon, ps, None, P.TilePlan(cfg.radius, 3, (0, ty, 0)))):
        for mode in (P.MODE_REFERENCE, P.MODE_FAST):
            got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, mode, m, pspec=ps)
            assert rep.kernel_kind == 1
            if ty and cfg.radius == 8:
                assert rep.tile[1] == (8 if ty <= 8 else 12), (ty, tuple(rep.tile))
            elif ty and cfg.radius == 4:   # wave so8: 8 / 16 rows, 24 (12 warps x 2 rows) above
                assert rep.tile[1] == (8 if ty <= 8 else 16 if ty <= 16 else 24), (ty, tuple(rep.tile))
            elif ty:
                assert rep.tile[1] == max(ty, 8) or rep.tile[1] == 16 or (ty == 24 and rep.tile[1] == 32), \
                    (ty, tuple(rep.tile))
            check(spec, ext, got, slots, ref, slots, dtd - 1 + steps, dtd, 0.0 if mode == P.MODE_REFERENCE else FAST_TOL)


@pytest.mark.parametrize("cfg_idx,ext,steps", [(2, (12, 20, 40), 6), (2, (6, 8, 8), 3), (1, (20, 30), 5)])
@pytest.mark.parametrize("T", [2, 4])
def test_star_wavefront_per_slot_halos(cfg_idx, ext, steps, T):
    """Star stencils under the wavefront with the literal reference init (LCG
    halos in slot 0 only, S = 1 + T slots): each level's z halo below plane 0
    is refreshed from its slot when that level stores plane 0, and the next
    level's producer must wait for it (regression: it loaded those planes
    without waiting)."""
    cfg = CF.get(cfg_idx).scaled(ext, steps)
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    slots = 1 + T
    base = O.init_reference(spec, ext, slots, 3)
    ref = oracle_run(spec, ext, base, slots, 0, steps)
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(cfg.radius, T, tuple(0 for _ in ext)))
    got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, pspec=ps)
    assert rep.kernel_kind == 1
    check(spec, ext, got, slots, ref, slots, steps, 1)


def test_cli_run_and_verify(capsys):
    """SPEC.md cli example: `verify lap1.stencil --mode time --time-tile 4
    --skew 1 --seed 7` -> {"bitwise_equal": true}, exit 0; run prints one
    ExecReport JSON object."""
    import json
    import os
    from paper_1806_08299_b200 import cli
    data = os.path.join(os.path.dirname(__file__), "data")
    for f, extra in (("lap1.stencil", ["--fused", "0"]), ("lap1.stencil", ["--fused", "3"]),
                     ("heat3d.stencil", ["--fused", "2"])):
        rc = cli.main(["verify", os.path.join(data, f), "--mode", "time", "--time-tile", "4", "--skew", "1",
                       "--seed", "7"] + extra)
        out, _ = capsys.readouterr()
        assert rc == 0 and json.loads(out) == {"bitwise_equal": True}, (f, extra, out)
    rc = cli.main(["run", os.path.join(data, "heat3d.stencil"), "--mode", "space", "--tiles", "8,8,32"])
    out, _ = capsys.readouterr()
    rep = json.loads(out)
    assert rc == 0 and rep["points_updated"] == 6 * 20 * 24 * 70 and rep["kernel_kind"] == 1


@pytest.mark.parametrize("R,ty", [(4, 0), (4, 32), (8, 0)])
def test_star_heat_big_radius_time_tiles(R, ty):
    """3-D heat stars of radius 4 / 8 under the wavefront with the default or
    32-row tile (regression: the 32-row r = 4 shape asked for more than the
    227 KB of shared memory and the launch failed; the stale error then also
    failed the next call).  Bitwise vs the oracle."""
    from test_gpu_fused import _random_star
    rng = np.random.default_rng(400 + R + ty)
    spec = _random_star(rng, 3, R, True)
    ext = (13, 37, 70)
    steps = 5
    T = 2
    slots = 1 + T
    base = O.uniform_halo(spec, ext, O.init_reference(spec, ext, slots, 3), slots)
    ref = oracle_run(spec, ext, base, slots, 0, steps)
    ps = product_spec(spec)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(R, T, (0, ty, 0)))
    for mode in (P.MODE_REFERENCE, P.MODE_FAST):
        got, rep = gpu_run(spec, ext, base, slots, 0, 0, steps, nest, mode, pspec=ps)
        assert rep.kernel_kind == 1
        check(spec, ext, got, slots, ref, slots, steps, 1, 0.0 if mode == P.MODE_REFERENCE else FAST_TOL)


def test_palettized_m_field_bitwise(monkeypatch):
    """The layered m field (2 distinct values) is read as 1-byte palette codes
    (the default) or as floats (ST_MCODES=0); both bitwise.  A field with
    > 256 values (config 4's smoothed random velocity) is not palettized and
    still runs."""
    for cidx, ext, steps in ((3, (24, 33, 70), 9), (4, (20, 35, 40), 5)):
        cfg = CF.get(cidx).scaled(ext, steps)
        slots = 3
        spec, base, m = config_inputs(cfg, slots)
        rng = np.random.default_rng(cidx)
        v = base.reshape((slots,) + spec.padded(ext))
        inner = tuple(slice(cfg.radius, cfg.radius + e) for e in ext)
        for lv in range(2):
            v[lv][inner] = rng.random(ext, dtype=np.float32)
        ref = oracle_run(spec, ext, base, slots, 0, steps, m)
        ps = product_spec(spec)
        for mc in ("1", "0"):
            monkeypatch.setenv("ST_MCODES", mc)
            got, rep = gpu_run(spec, ext, base, slots, 1, 0, steps, P.build_canonical_nest(ps, None),
                               P.MODE_REFERENCE, m, pspec=ps)
            assert rep.kernel_kind == 1
            check(spec, ext, got, slots, ref, slots, 1 + steps, 2)
        monkeypatch.delenv("ST_MCODES")
