"""Cache simulator and the sim_traffic autotuner (host-only; SPEC.md:354-400,
526-572; acceptance criteria 6, 7, 10)."""
import itertools

import pytest

import paper_1806_08299_b200 as P
from paper_1806_08299_b200 import analysis as A
from paper_1806_08299_b200 import autotune as T


def lap(ndims, c=0.1, dt=1):
    terms = [P.StencilTerm(1 - 2 * ndims * c, 1, (0,) * ndims)]
    for i in range(ndims):
        for s in (-1, 1):
            off = [0] * ndims
            off[i] = s
            terms.append(P.StencilTerm(c, dt, tuple(off)))
    return P.StencilSpec.make("lap", ndims, terms)


def test_simulate_known_answers():
    ident = P.StencilSpec.make("id", 1, [P.StencilTerm(1.0, 1, (0,))])
    sp = P.IterationSpace(1, (4,))
    r = P.simulate(P.build_canonical_nest(ident, sp), ident, sp, P.CacheConfig(1 << 20, 1))
    assert (r.lines_loaded, r.lines_written_back, r.bytes, r.flops) == (4, 4, 32, 4)
    assert P.measured_ai_elems(r) == pytest.approx(0.125)
    s3 = lap(1)
    canon = P.build_canonical_nest(s3, sp)
    one = P.simulate(canon, s3, sp, P.CacheConfig(1, 1))
    assert one.lines_loaded >= 3 * 4 - 2          # every point reloads its neighbourhood
    prev = None
    for omega in (1, 2, 4, 8, 64):                 # LRU: more capacity never misses more
        r = P.simulate(canon, s3, sp, P.CacheConfig(omega, 1))
        assert prev is None or r.lines_loaded <= prev
        prev = r.lines_loaded
    # compulsory floor with an ideal cache: every distinct element once
    big = P.simulate(canon, s3, sp, P.CacheConfig(1 << 20, 1))
    assert big.lines_loaded == 4 + 2 and big.lines_written_back == 4
    with pytest.raises(P.Error):
        P.simulate(canon, s3, P.IterationSpace(10, (100,)), P.CacheConfig(64, 1), cap=50)
    with pytest.raises(P.Error):
        P.simulate(canon, s3, sp, P.CacheConfig(10, 4))   # capacity not a multiple of the line


def test_simulate_trace_is_schedule_invariant_with_ideal_cache():
    """Every schedule traces the same multiset of points (equal flops); with
    an unbounded L = 1 cache the canonical and space-tiled nests (same slot
    count) move identical compulsory traffic, the time-tiled one touches its
    delta_t + t_t slots."""
    s = lap(2)
    sp = P.IterationSpace(6, (20, 13))
    canon = P.build_canonical_nest(s, sp)
    nests = [canon, P.tile_space_minmax(canon, (4, 8)), P.tile_time(canon, s, sp, P.TilePlan(1, 3, (5, 4)))]
    reps = [P.simulate(n, s, sp, P.CacheConfig(1 << 22, 1)) for n in nests]
    assert len({r.flops for r in reps}) == 1
    assert (reps[0].lines_loaded, reps[0].lines_written_back) == (reps[1].lines_loaded, reps[1].lines_written_back)
    plane = 22 * 15
    assert reps[2].lines_written_back == 4 * plane - 4 * (plane - 20 * 13)   # 4 slots' interiors written
    assert reps[0].lines_written_back == 2 * 20 * 13


@pytest.mark.parametrize("ndims,ext,steps,tt,tiles", [
    (2, (200, 200), 4, 2, (8, 200)),
    (2, (192, 256), 4, 4, (16, 256)),
    (2, (256, 160), 3, 2, (32, 160)),
    (1, (40000,), 4, 4, (512,)),
    (2, (181, 200), 4, 2, (4, 64)),
])
def test_estimators_overestimate_measured_ai(ndims, ext, steps, tt, tiles):
    """SPEC.md:388 / criterion 6: with a per-level footprint >= 8 Omega the
    simulated (L = 1) AI is at most the tight estimate, which is at most the
    naive one."""
    omega = 4096
    s = lap(ndims)
    sp = P.IterationSpace(steps, ext)
    foot = 1
    for d, r in zip(ext, s.radii):
        foot *= d + 2 * r
    assert foot >= 8 * omega
    plan = P.TilePlan(1, tt, tiles)
    rep = P.simulate(P.tile_time(P.build_canonical_nest(s, sp), s, sp, plan), s, sp, P.CacheConfig(omega, 1))
    est, _ = A.tight_bound(s, ext, tt, tiles, omega)
    assert rep.measured_ai <= est.ai_tight_tt + 1e-12 <= est.ai_naive_tt + 1e-12


def test_tuned_time_tiling_moves_fewer_bytes_than_tuned_space_tiling():
    """Criterion 7: desk-scale analogue of the paper's 20-45% runtime
    decrease -- simulated bytes of the tuned time-tiled nest < those of the
    tuned space-tiled nest."""
    s = lap(2)
    sp = P.IterationSpace(8, (96, 96))
    cache = P.CacheConfig(2048, 1)
    canon = P.build_canonical_nest(s, sp)
    space_best = min(P.simulate(P.tile_space_minmax(canon, (a, b)), s, sp, cache).bytes
                     for a in (4, 8, 16, 32) for b in (16, 32, 96))
    _, time_best, _ = T.tune_sim(s, sp, T.HostSearchSpace(time_tiles=(1, 2, 4, 8), space_tiles=((4, 8, 16, 32),
                                                                                               (16, 32, 96))), cache)
    assert time_best < space_best
    print(f"time-tiled {time_best} B vs space-tiled {space_best} B: {100 * (1 - time_best / space_best):.1f}% less")


def test_tune_sim_equals_independent_bruteforce_argmin():
    """Criterion 10: a 1-D space, <= 12 plans, sim_traffic cost: tune's result
    is the independently coded exhaustive argmin (lexicographic ties), and
    deterministic over 3 runs."""
    s = lap(1)
    sp = P.IterationSpace(8, (24,))
    cache = P.CacheConfig(12, 1)
    search = T.HostSearchSpace(time_tiles=(1, 2, 4, 8), space_tiles=((4, 8, 24),))
    results = [T.tune_sim(s, sp, search, cache) for _ in range(3)]
    assert len(results[0][2]) == 12
    assert all((r[0].time_tile, tuple(r[0].space_tiles), r[1]) ==
               (results[0][0].time_tile, tuple(results[0][0].space_tiles), results[0][1]) for r in results)
    # independent exhaustive loop
    canon = P.build_canonical_nest(s, sp)
    best = None
    for tt, t1 in itertools.product((1, 2, 4, 8), (4, 8, 24)):
        nb = P.simulate(P.tile_time(canon, s, sp, P.TilePlan(1, tt, (t1,))), s, sp, cache).bytes
        if best is None or nb < best[0] or (nb == best[0] and (tt, t1) < best[1]):
            best = (nb, (tt, t1))
    got = results[0]
    assert (got[1], (got[0].time_tile, got[0].space_tiles[0])) == best
    # best_cost <= the all-ones plan (t_t = 1, t_i = D_i) of the same table
    ones = [c for p, c in got[2] if p.time_tile == 1 and p.space_tiles[0] == 24]
    assert got[1] <= ones[0]


def test_host_search_space_defaults():
    s = lap(2)
    plans = T.HostSearchSpace().plans(s, P.IterationSpace(5, (8, 12)))
    tts = sorted({p.time_tile for p in plans})
    assert tts == [1, 2, 4]                       # {1,2,4,8,16} within [1, D_t = 5]
    inner = sorted({p.space_tiles[1] for p in plans})
    assert inner == [2, 4, 8, 12]                 # powers of two in [2, 12] plus D_2 itself
    outer = sorted({p.space_tiles[0] for p in plans})
    assert outer == [2, 4, 8]
    assert all(p.skew == 1 for p in plans)
