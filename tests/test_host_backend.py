"""Host-side problem tables (paper_2604_00510_b200.backend) vs reference fixtures."""

import time

import pytest

from golden_io import load
from paper_2604_00510_b200 import backend as B
from paper_2604_00510_b200.backend import Difficulty

MIX = (0.6, 0.25, 0.15)


def _check(specs, recs):
    assert len(specs) == len(recs)
    table = B.problem_table(specs)
    for s, rec, row in zip(specs, recs, table):
        assert s.problem_id == rec["problem_id"]
        assert s.seed == rec["seed"]
        assert s.difficulty.value == rec["difficulty"]
        assert s.base_depth == rec["base_depth"]
        assert row.base_depth == rec["base_depth"]
        if rec["golden_path"] is None:
            assert s.golden_path is None and row.golden_len == -1
        else:
            assert list(s.golden_path) == rec["golden_path"]
            assert list(B.golden_step_rewards(s)) == rec["golden_rewards"]
            assert list(row.golden_rewards[: row.golden_len]) == rec["golden_rewards"]


def test_make_workload_c1():
    D = {d: (7, 7) for d in Difficulty}
    _check(B.make_workload(64, MIX, 0, branching=4, depth_ranges=D), load("workloads")["c1"])


def test_make_workload_cli_default():
    _check(B.make_workload(500, MIX, 20260810), load("workloads")["cli_default"])


def test_make_workload_mixed():
    D = {Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)}
    _check(B.make_workload(97, (0.5, 0.3, 0.2), 77, branching=3, depth_ranges=D, accept_threshold=0.35),
           load("workloads")["mixed_b3"])


def test_make_workload_c2_full_and_fast():
    D = {d: (15, 15) for d in Difficulty}
    t = time.time()
    specs = B.make_workload(4096, MIX, 0, branching=4, depth_ranges=D)
    assert time.time() - t < 20
    _check(specs, load("workloads")["c2"])


def test_stagnation_profile_problems():
    recs = load("workloads")["c4_stagnation"]
    from paper_2604_00510_b200 import keyed
    specs = [B.make_problem(f"s{i:04d}", keyed.mix(0, 8, i), Difficulty.HARD_SOLVABLE, (31, 31), 8,
                            B.stagnation_profile()) for i in range(len(recs))]
    _check(specs, recs)


def test_make_workload_validation():
    with pytest.raises(ValueError):
        B.make_workload(0, MIX, 0)
    with pytest.raises(ValueError):
        B.make_workload(5, (0.5, 0.5, 0.5), 0)


def test_serving_arrival_steps_match_reference_generator():
    """backend.serving_arrival_steps (config 5: 65,536 Poisson arrivals) equals
    the reference generator's cumulative exponential times quantised to waves
    (simulator.py:193-200; fixture from tests/golden/make_golden.py gen_arrivals)."""
    from paper_2604_00510_b200 import keyed

    for name, case in load("arrivals").items():
        got = B.serving_arrival_steps(case["n"], case["rate"], case["seed"], case["steps_per_unit"])
        assert got == case["steps"], name
        t = 0.0
        for i, want in enumerate(case["times_head"]):
            t += keyed.exponential_draw(case["rate"], case["seed"], B.TAG_ARRIVAL, i)
            assert t == want, (name, i)
