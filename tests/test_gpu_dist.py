"""Z-slab decomposition (config 5 path) on ONE GPU through the in-process
loopback backend: G slab grids (slab + ghosts of depth r*T) exchange ghost
planes every time tile with device copies instead of NCCL, then compute the
shrinking valid ranges.  The gathered slabs must equal the single-grid run
bit for bit.  Random interiors, so every slab interface carries signal
(SURVEY.md 4.4)."""
import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import gpu_run, product_spec

pytestmark = pytest.mark.gpu


def _slab_run(spec, ps, ext, base, slots, steps, G, T, ghost_mult, m=None, mode=P.MODE_REFERENCE, sched="canonical",
              tiles=(0, 0, 0), band_rows=0, band_skew=0):
    """Run the global grid `base` (reference layout) as G loopback slabs."""
    r = spec.radius(0)
    dtd = spec.time_depth
    Pg = spec.padded(ext)
    gv = base.reshape((slots,) + Pg)
    ctx = P.default_context()
    members, grids, parts = [], [], []
    ghost = r * T * ghost_mult
    for rank in range(G):
        z0, nzs, glo, ghi = P.dist_partition(ext[0], G, rank, ghost)
        lext = (nzs + glo + ghi,) + tuple(ext[1:])
        Pl = spec.padded(lext)
        loc = np.zeros((slots,) + Pl, np.float32)
        # local grid = global planes [z0 - glo - r, z0 + nzs + ghi + r) (padded coords)
        loc[:] = gv[:, z0 - glo: z0 - glo + Pl[0]]
        dg = P.DeviceGrid(ctx, ps, lext, slots)
        dg.upload(np.ascontiguousarray(loc.reshape(-1)), dtd - 1)
        if m is not None:
            mv = m.reshape(ext)[z0 - glo: z0 + nzs + ghi]
            dg.set_field(np.ascontiguousarray(mv))
        grids.append((dg, loc, z0, nzs, glo, ghi, lext))
        members.append(P.Dist(dg, rank, G, glo, ghi))
    P.Dist.link_loopback(members)
    canon = P.build_canonical_nest(ps, None)
    if sched == "time":   # one wavefront launch per time tile over the trapezoid of z ranges
        nest = P.LoopNest(P.SCHED_TIME, P.TilePlan(r, T, tiles, band_rows=band_rows, band_skew=band_skew))
    else:
        nest = P.LoopNest(P.SCHED_CANONICAL, P.TilePlan(r, T, ()))
    rep = members[0].apply(0, steps, nest, mode)
    out = base.copy().reshape((slots,) + Pg)
    last = dtd - 1 + steps
    for dg, loc, z0, nzs, glo, ghi, lext in grids:
        flat = np.ascontiguousarray(loc.reshape(-1))
        dg.download(flat)
        lv = flat.reshape(loc.shape)
        for lvl in range(last - dtd + 1, last + 1):
            s = lvl % slots
            out[s, r + z0: r + z0 + nzs] = lv[s, r + glo: r + glo + nzs]
    for mbr in members:
        mbr.close()
    for g in grids:
        g[0].close()
    return out.reshape(-1), rep


@pytest.mark.parametrize("sched,tiles", [("canonical", (0, 0, 0)), ("time", (0, 0, 0)), ("time", (7, 16, 0)),
                                         ("time", (9, 24, 0))])   # z-chunks shorter than a slab, 24-row shapes
@pytest.mark.parametrize("cidx,ext,steps,G,T,gm", [
    (2, (40, 24, 70), 9, 2, 2, 1),
    (2, (41, 20, 33), 7, 3, 1, 1),
    (2, (64, 16, 40), 10, 4, 3, 2),
    (2, (70, 40, 140), 12, 2, 6, 1),
    (3, (48, 20, 40), 9, 2, 2, 1),
    (3, (61, 17, 35), 8, 3, 4, 1),
])
def test_loopback_slabs_bitwise_equal_single_grid(cidx, ext, steps, G, T, gm, sched, tiles):
    cfg = CF.get(cidx).scaled(ext, steps)
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    dtd = spec.time_depth
    slots = dtd + (T if sched == "time" else 1)   # required_slots of the plan
    rng = np.random.default_rng(cidx * 100 + G)
    base = O.new_grid(spec, ext, slots)
    v = base.reshape((slots,) + spec.padded(ext))
    R = cfg.radius
    for lv in range(dtd):
        v[lv][R:R + ext[0], R:R + ext[1], R:R + ext[2]] = rng.random(ext, dtype=np.float32)
    m = None
    if cfg.model:
        m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H)
    ps = product_spec(spec)
    single, _ = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, P.build_canonical_nest(ps, None), mfield=m,
                        pspec=ps)
    slabs, rep = _slab_run(spec, ps, ext, base, slots, steps, G, T, gm, m, sched=sched, tiles=tiles)
    if sched == "time":   # >= one wavefront launch per time tile per slab (split tiles: stripes + interior)
        assert rep.kernel_launches >= -(-steps // T) * G
    assert rep.points_updated == steps * int(np.prod(ext))
    assert O.verify_bitwise(spec, ext, single, slots, slabs, slots, dtd - 1 + steps, dtd) == 1
    # and against the oracle
    ref = base.copy()
    O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)
    assert O.verify_bitwise(spec, ext, ref, slots, slabs, slots, dtd - 1 + steps, dtd) == 1


@pytest.mark.parametrize("cidx,ext,steps,G,T", [
    (3, (96, 40, 72), 13, 2, 2),
    (3, (240, 33, 40), 12, 3, 3),
    (2, (120, 30, 50), 17, 4, 2),
])
def test_overlapped_exchange_equals_serial_and_oracle(cidx, ext, steps, G, T, monkeypatch):
    """The overlapped exchange (boundary cones first, the next tile's ghosts on
    a side stream while the interior runs) is bitwise the serial schedule
    (ST_DIST_SERIAL=1: exchange, then one launch per tile) and the oracle."""
    cfg = CF.get(cidx).scaled(ext, steps)
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    dtd = spec.time_depth
    slots = dtd + T
    rng = np.random.default_rng(7 + cidx * 10 + G)
    base = O.new_grid(spec, ext, slots)
    v = base.reshape((slots,) + spec.padded(ext))
    R = cfg.radius
    for lv in range(dtd):
        v[lv][R:R + ext[0], R:R + ext[1], R:R + ext[2]] = rng.random(ext, dtype=np.float32)
    m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H) if cfg.model else None
    ps = product_spec(spec)
    over, rep_o = _slab_run(spec, ps, ext, base, slots, steps, G, T, 1, m, sched="time")
    monkeypatch.setenv("ST_DIST_SERIAL", "1")
    ser, rep_s = _slab_run(spec, ps, ext, base, slots, steps, G, T, 1, m, sched="time")
    tiles = -(-steps // T)
    assert rep_s.kernel_launches == tiles * G
    # split tiles: stripes (one per neighbour) + interior; the last tile is whole
    nb = 2 * (G - 1)
    assert rep_o.kernel_launches == (tiles - 1) * (G + nb) + G
    last = dtd - 1 + steps
    assert O.verify_bitwise(spec, ext, ser, slots, over, slots, last, dtd) == 1
    ref = base.copy()
    O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)
    assert O.verify_bitwise(spec, ext, ref, slots, over, slots, last, dtd) == 1


@pytest.mark.parametrize("cidx,ext,steps,G,T,tiles,band", [
    (3, (70, 100, 140), 10, 2, 4, (4096, 24, 0), 48),    # so8 wave, 24-row shape, whole-depth items
    (3, (90, 70, 128), 9, 3, 3, (16, 16, 0), 32),        # short z-chunks, 16-row shape
    (2, (60, 90, 130), 11, 2, 4, (4096, 16, 0), 32),     # heat so4
])
def test_loopback_slabs_with_row_skewed_bands(cidx, ext, steps, G, T, tiles, band):
    """The d_2 time tile (st_plan.band_rows / band_skew) inside the z-slab
    path: the trapezoid of z ranges, the cones-first split and the row-skewed
    y-bands together, bitwise equal to the oracle."""
    cfg = CF.get(cidx).scaled(ext, steps)
    spec = O.Spec(cfg.ndims, cfg.terms, cfg.model)
    dtd = spec.time_depth
    slots = dtd + T
    rng = np.random.default_rng(31 * cidx + G)
    base = O.new_grid(spec, ext, slots)
    v = base.reshape((slots,) + spec.padded(ext))
    R = cfg.radius
    for lv in range(dtd):
        v[lv][R:R + ext[0], R:R + ext[1], R:R + ext[2]] = rng.random(ext, dtype=np.float32)
    m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H) if cfg.model else None
    ps = product_spec(spec)
    slabs, rep = _slab_run(spec, ps, ext, base, slots, steps, G, T, 1, m, sched="time", tiles=tiles, band_rows=band,
                           band_skew=R)
    ref = base.copy()
    O.execute(spec, ext, ref, slots, 0, steps, mfield=m, nthreads=8)
    assert O.verify_bitwise(spec, ext, ref, slots, slabs, slots, dtd - 1 + steps, dtd) == 1
