"""Row-skewed y-bands (the L2 time tile of the star wavefront): the level
with index lt in its time tile runs on the tile grid shifted by -ysk*lt
rows, bands of cy tiles advance T levels back to back (tile_time applied to
d_2 with the minimum skew, transforms.hpp:53-59).  Every
plan must be bitwise equal to the oracle's canonical run.
"""
import numpy as np
import pytest

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF
from _common import config_inputs, gpu_run, product_spec

pytestmark = pytest.mark.gpu


def _inputs(cidx, ext, steps, slots, seed):
    cfg = CF.get(cidx).scaled(ext, steps)
    dtd = 2 if cfg.model else 1
    spec, base, m = config_inputs(cfg, slots)
    rng = np.random.default_rng(seed)
    v = base.reshape((slots,) + spec.padded(ext))
    inner = tuple(slice(cfg.radius, cfg.radius + e) for e in ext)
    for lv in range(dtd):   # random interiors: every band boundary carries signal
        v[lv][inner] = rng.random(ext, dtype=np.float32)
    return cfg, dtd, spec, base, m


def _oracle(spec, ext, base, slots, steps, m):
    g = base.copy()
    rc, _, _ = O.execute(spec, ext, g, slots, 0, steps, mfield=m, nthreads=16)
    assert rc == 0
    return g


@pytest.mark.parametrize("cidx,ext,steps,ty", [
    (3, (22, 90, 140), 11, 16),     # wave so8 (radius 4), 16-row tiles, ragged x
    (3, (19, 70, 128), 9, 8),       # ... 8-row tiles (2r = ty)
    (3, (17, 100, 128), 9, 24),     # ... 24-row tiles (12 warps x 2 rows, m as 1-byte codes)
    (2, (21, 100, 130), 13, 16),    # heat so4 (radius 2), 16-row tiles
    (2, (21, 100, 70), 10, 32),     # ... 32-row tiles
    (4, (20, 50, 40), 6, 12),       # wave so16 (radius 8): 2r > ty, the plan falls back (still exact)
])
@pytest.mark.parametrize("T,ysk,band", [
    (2, 0, 32), (4, 4, 16), (4, 4, 32), (8, 4, 48), (8, 6, 32), (3, 9, 16), (8, 16, 64), (5, 20, 32),
])
def test_row_skewed_bands_bitwise(cidx, ext, steps, ty, T, ysk, band, monkeypatch):
    slots = 3 if cidx != 2 else 2
    cfg, dtd, spec, base, m = _inputs(cidx, ext, steps, slots + T, 7 * cidx + T)
    slots += T
    ref = _oracle(spec, ext, base, slots, steps, m)
    ps = product_spec(spec)
    if (T + band) % 2:   # through the study knobs of the environment ...
        monkeypatch.setenv("ST_WF_YSKEW", str(max(ysk, 1)))   # clamped up to the radius by the planner
        monkeypatch.setenv("ST_WF_CY_ROWS", str(band))
        plan = P.TilePlan(cfg.radius, T, (4096, ty, 0))
    else:                # ... and through the plan (st_plan.band_rows / band_skew)
        plan = P.TilePlan(cfg.radius, T, (4096, ty, 0), band_rows=band, band_skew=ysk)
    nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, plan)
    for mode in (P.MODE_REFERENCE,):
        got, rep = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, mode, m, pspec=ps)
        assert rep.kernel_kind == 1
        assert O.verify_bitwise(spec, ext, ref, slots, got, slots, dtd - 1 + steps, dtd) == 1, \
            O.max_rel_err(spec, ext, ref, slots, got, slots, dtd - 1 + steps, dtd)


def test_row_skewed_bands_short_chunks_and_resume(monkeypatch):
    """z-chunks shorter than the grid, a resumed run, and FAST mode equal to
    the unbanded FAST run bit for bit (same arithmetic, another order of
    items)."""
    cidx, ext, steps, T = 3, (40, 80, 128), 12, 4
    slots = 3 + T
    cfg, dtd, spec, base, m = _inputs(cidx, ext, steps, slots, 5)
    ref = _oracle(spec, ext, base, slots, steps, m)
    ps = product_spec(spec)
    ctx = P.default_context()
    for cz in (8, 16, 4096):
        nest = P.tile_time(P.build_canonical_nest(ps, None), ps, None, P.TilePlan(cfg.radius, T, (cz, 16, 0)))
        outs = {}
        for banded in (True, False):
            if banded:
                monkeypatch.setenv("ST_WF_YSKEW", "4")
                monkeypatch.setenv("ST_WF_CY_ROWS", "32")
            else:
                monkeypatch.delenv("ST_WF_YSKEW")
                monkeypatch.delenv("ST_WF_CY_ROWS")
            dg = P.DeviceGrid(ctx, ps, ext, slots)
            dg.upload(base, dtd - 1)
            dg.set_field(m)
            dg.apply(0, 5, nest)
            dg.apply(5, steps, nest)
            out = base.copy()
            dg.download(out)
            dg.close()
            assert O.verify_bitwise(spec, ext, ref, slots, out, slots, dtd - 1 + steps, dtd) == 1, (cz, banded)
            got, _ = gpu_run(spec, ext, base, slots, dtd - 1, 0, steps, nest, P.MODE_FAST, m, pspec=ps)
            outs[banded] = got
        assert np.array_equal(outs[True], outs[False])
