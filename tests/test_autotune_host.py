"""Autotuner search space (host logic, no GPU): SPEC.md:526-572 semantics --
a Cartesian product of the runtime parameters, plans beyond the step count
dropped, ties broken by the lexicographic plan key."""
from paper_1806_08299_b200 import autotune as A


def test_candidates_cartesian_and_fused():
    s = A.SearchSpace(time_tiles=(1, 4, 64), chunks=(64, 128), tile_rows=(16, 32), fused_levels=(2, 3, 99))
    c = s.candidates(steps=10)
    canon = [x for x in c if x.schedule == "canonical"]
    wave = [x for x in c if x.schedule == "time" and x.fused == 0]
    fused = [x for x in c if x.fused]
    assert len(canon) == 2
    assert len(wave) == 2 * 2 * 2          # T = 64 > 10 steps is dropped
    assert sorted({(x.fused, x.time_tile) for x in fused}) == [(2, 2), (3, 3)]
    assert all(x.cz == 0 for x in fused)
    keys = [x.key() for x in c]
    assert len(set(keys)) == len(keys)


def test_tie_break_is_lexicographic():
    a = A.Candidate("time", 4, 64, 16)
    b = A.Candidate("time", 4, 64, 16, fused=2)
    table = [(b, 1.0), (a, 1.0)]
    best = min(table, key=lambda cv: (cv[1], cv[0].key()))[0]
    assert best == a
