"""The GPU traffic predictor (paper_1806_08299_b200/traffic.py, SURVEY.md
8(f)3) against every ncu DRAM measurement recorded in profiles/traffic.json
(host-only: reads the committed measurements)."""
import json
import os

import pytest

from paper_1806_08299_b200.traffic import Plan, predict, reuse_fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRAFFIC = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))

# traffic.json key -> (plan the measurement ran, updates per launch, tolerance)
CASES = {
    "config2:canonical:T1:reference": (Plan("sweep", (256, 256, 256), 2, False, rows=32), 256 ** 3, 0.15),
    "config2:time:T32:fast": (Plan("wavefront", (256, 256, 256), 2, False, rows=32, time_tile=32), 64 * 256 ** 3,
                              0.15),
    "config3:time:T8:reference": (Plan("wavefront", (512, 512, 512), 4, True, rows=24, m_bytes=1, time_tile=8),
                                  200 * 512 ** 3, 0.15),
    "config4:time:T4:reference": (Plan("wavefront", (512, 512, 512), 8, True, rows=8, time_tile=4),
                                  100 * 512 ** 3, 0.15),
    "config4:time:T4:fast": (Plan("wavefront", (512, 512, 512), 8, True, rows=12, time_tile=4),
                             100 * 512 ** 3, 0.15),
    # round 2b plans: 24-row tiles (12 warps x 2 rows), one persistent launch per run
    "config5:slab1:time:T4:reference": (Plan("wavefront", (512, 1024, 1024), 4, True, rows=24, m_bytes=1,
                                             time_tile=4), 200 * 512 * 1024 ** 2, 0.15),
    "config5:slab1:time:T4:fast": (Plan("wavefront", (512, 1024, 1024), 4, True, rows=24, m_bytes=1,
                                        time_tile=4, cz=256), 200 * 512 * 1024 ** 2, 0.15),
    "config3:time:T8:fast": (Plan("wavefront", (512, 512, 512), 4, True, rows=24, m_bytes=1, time_tile=8),
                             200 * 512 ** 3, 0.15),
    # bit-exact config 2 on the 24-row tile: the slower arithmetic keeps the levels closer together than the
    # model's lag estimate (5.25 measured, 6.9 predicted)
    "config2:time:T32:reference": (Plan("wavefront", (256, 256, 256), 2, False, rows=24, time_tile=32),
                                   64 * 256 ** 3, 0.35),
    # fused passes: the model under-predicts by 23-30%: the
    # halo reads of neighbouring overlapped tiles miss L2 more than KAPPA says
    "config2:time:T32:fast:F2": (Plan("fused", (256, 256, 256), 2, False, rows=16, levels_per_pass=2),
                                 2 * 256 ** 3, 0.35),
    "config6:time:T3:fast:F3": (Plan("fused", (512, 512, 512), 1, False, rows=24, levels_per_pass=3),
                                3 * 512 ** 3, 0.35),
    "config7:time:T3:reference:F3": (Plan("fused", (512, 512, 512), 1, True, rows=16, levels_per_pass=3),
                                     3 * 512 ** 3, 0.35),
    "config1:time:T4:reference:F16": (Plan("resident", (1024, 1024), 1, False, levels_per_pass=100),
                                      100 * 1024 ** 2, 0.15),
}


@pytest.mark.parametrize("key", sorted(CASES))
def test_prediction_matches_ncu(key):
    plan, updates, tol = CASES[key]
    measured = TRAFFIC[key]["dram_bytes_per_launch"] / updates
    pred = predict(plan)
    assert abs(pred - measured) <= tol * measured, (key, pred, measured)


def test_wavefront_reuse_decays_with_the_level_lag():
    """Config 2's 256^2 planes: the next level re-reads through L2 (reuse
    > 0); config 3/5's 512^2 / 1024^2 planes: one level's items exceed the
    CTA slots, the lag dwarfs L2, no reuse (SURVEY.md 7 hard part 3)."""
    small = Plan("wavefront", (256, 256, 256), 2, False, rows=32, time_tile=32)
    big = Plan("wavefront", (512, 1024, 1024), 4, True, rows=16, m_bytes=1, time_tile=4)
    assert reuse_fraction(small) > 0.2 and reuse_fraction(big) < 0.01
    assert predict(Plan("wavefront", (256, 256, 256), 2, False, rows=32, time_tile=1)) > predict(small)
