"""C emitter: the emitted program, compiled with
-ffp-contract=off and run, writes final levels bitwise equal to the oracle
running the same nest from the same reference init_grid."""
import random
import shutil
import subprocess

import numpy as np
import pytest

import _oracle as O
from _common import random_spec
from paper_1806_08299_b200 import codegen as CG

pytestmark = pytest.mark.skipif(shutil.which("gcc") is None, reason="needs a C compiler")


def run_emitted(src, tmp_path, name):
    c = tmp_path / f"{name}.c"
    exe = tmp_path / name
    c.write_text(src)
    subprocess.run(["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off", "-o", str(exe), str(c)], check=True)
    return np.frombuffer(subprocess.run([str(exe)], check=True, capture_output=True).stdout, dtype=np.float32)


@pytest.mark.parametrize("case", range(8))
def test_emitted_nests_equal_oracle(case, tmp_path):
    rng = random.Random(700 + case)
    spec = random_spec(rng, radius_max=2, dt_max=2, k_max=7)
    n = spec.ndims
    ext = tuple(rng.randint(1, {1: 60, 2: 14, 3: 7}[n]) for _ in range(n))
    steps = rng.randint(1, 6)
    dtd = spec.time_depth
    smin = max(spec.radius(i) for i in range(n))
    T = rng.choice([1, 2, 3])
    slots = dtd + T
    tiles = tuple(rng.randint(1, e + 2) for e in ext)
    oracle_sched = {"canonical": O.CANONICAL, "space": O.SPACE, "time": O.TIME}
    for sched in ("canonical", "space", "time"):
        src = CG.emit_c(n, spec.terms, ext, steps, slots, sched, skew=smin, time_tile=T,
                        tiles=None if sched == "canonical" else tiles, seed=11 + case)
        got = run_emitted(src, tmp_path, f"{sched}{case}")
        grid = O.init_reference(spec, ext, slots, 11 + case)
        kw = {} if sched == "canonical" else {"tiles": tiles}
        if sched == "time":
            kw.update(skew=smin, time_tile=T)
        assert O.execute(spec, ext, grid, slots, 0, steps, schedule=oracle_sched[sched], **kw)[0] == 0
        plane = spec.plane(ext)
        want = np.concatenate([grid[(lv % slots) * plane:(lv % slots + 1) * plane]
                               for lv in range(steps, steps + dtd)])
        assert got.tobytes() == want.tobytes(), (sched, ext, steps)


def test_emitted_bounds_and_pragmas():
    """SPEC.md:588-590 examples: MAX/MIN in the incremental bounds of a
    time-tiled nest, the pragma above the incremental x loop and not above
    x_blk or any t loop; emission is deterministic; illegal skew raises."""
    terms = [(0.5, 1, (0,)), (0.25, 1, (-1,)), (0.25, 1, (1,))]
    src = CG.emit_c(1, terms, (32,), 8, 5, "time", skew=1, time_tile=4, tiles=(8,))
    lines = src.splitlines()
    inc = [i for i, l in enumerate(lines) if "for (int64_t x1 = MAX(" in l]
    assert inc and "MIN(" in lines[inc[0]]
    assert "#pragma omp parallel for" in lines[inc[0] - 1]
    assert sum("#pragma omp parallel for" in l for l in lines) == 1
    assert src == CG.emit_c(1, terms, (32,), 8, 5, "time", skew=1, time_tile=4, tiles=(8,))
    with pytest.raises(ValueError):
        CG.emit_c(1, terms, (32,), 8, 5, "time", skew=0, time_tile=4, tiles=(8,))
