"""Helpers shared by the parity tests: random corpus specs,
oracle <-> product spec conversion, and a GPU run through the C-ABI."""
from __future__ import annotations

import random
from typing import List, Sequence, Tuple

import numpy as np

import _oracle as O
import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import configs as CF


def product_spec(spec: O.Spec, name="t") -> P.StencilSpec:
    return P.StencilSpec.make(name, spec.ndims, [P.StencilTerm(c, dt, tuple(off)) for c, dt, off in spec.terms],
                              model=spec.model)


def random_spec(rng: random.Random, ndims=None, radius_max=4, dt_max=2, k_max=9) -> O.Spec:
    """Acceptance-criterion-1 corpus: 1-3 dims, radii <= 4, delta_t <= 2,
    k <= 9 terms, |coeff| summing <= 1."""
    n = ndims or rng.randint(1, 3)
    k = rng.randint(1, k_max)
    raw = [rng.uniform(-1, 1) for _ in range(k)]
    s = sum(abs(x) for x in raw) or 1.0
    terms = []
    for c in raw:
        off = tuple(rng.randint(-radius_max, radius_max) for _ in range(n))
        terms.append((float(np.float32(c / s)), rng.randint(1, dt_max), off))
    return O.Spec(n, terms)


def config_spec(cfg: CF.Config) -> O.Spec:
    return O.Spec(cfg.ndims, cfg.terms, cfg.model)


def config_inputs(cfg: CF.Config, slots: int, seed: int = CF.SEED_FIELD):
    """Oracle-side inputs for a (possibly scaled) config: grid + m field."""
    spec = config_spec(cfg)
    ext = cfg.extents
    if cfg.init == "unit":
        g = O.init_unit(spec, ext, slots, seed)
    else:
        g = O.init_gaussian(spec, ext, slots, cfg.sigma, [e // 2 for e in ext])
    m = None
    if cfg.field == "layered":
        m = O.mfield_layered(ext, cfg.v_top, cfg.v_bottom, ext[0] // 2, cfg.dt, CF.H)
    elif cfg.field == "random":
        m = O.mfield_random(ext, CF.SEED_VELOCITY, cfg.vmin, cfg.vmax, cfg.dt, CF.H)
    return spec, g, m


def gpu_run(spec: O.Spec, extents, grid: np.ndarray, slots: int, last_level: int, t_begin: int, t_end: int,
            nest: P.LoopNest, mode: int = P.MODE_REFERENCE, mfield=None, ctx=None, pspec=None):
    """Upload -> st_apply -> download through the C-ABI; returns (grid, report)."""
    ctx = ctx or P.default_context()
    pspec = pspec or product_spec(spec)
    dg = P.DeviceGrid(ctx, pspec, extents, slots)
    try:
        dg.upload(grid, last_level)
        if mfield is not None:
            dg.set_field(mfield)
        rep = dg.apply(t_begin, t_end, nest, mode)
        out = grid.copy()
        ll = dg.download(out)
        assert ll == last_level + (t_end - t_begin)
    finally:
        dg.close()
    return out, rep
