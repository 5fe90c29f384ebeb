"""The rest of the reference's public surface (treeserve/__init__.py):
generate_steps on the device (csrc/steps.cu) against the reference's
generate_steps fixtures, the cost model, aggregate/classify helpers, and the
workload replay format (bytes from the reference's workload_to_json)."""

from __future__ import annotations

import random

import pytest

from golden_io import load, problem_from_record


def test_aggregate_and_classify_reference_cases():
    """test_scoring.py TestAggregate / TestClassifyLeaf."""
    from paper_2604_00510_b200.scoring import (AggregationScheme, FutilityBound, LeafClass, ScoringConfig,
                                               UnsupportedSchemeError, aggregate_trajectory, classify_leaf)

    P, MIN = AggregationScheme.CUMULATIVE_PRODUCT, AggregationScheme.MINIMUM
    assert aggregate_trajectory([0.9, 0.8, 0.5], P) == pytest.approx(0.36)
    for s in AggregationScheme:
        assert aggregate_trajectory([0.7], s) == pytest.approx(0.7)
    assert aggregate_trajectory([0.9, 0.8, 0.5], MIN) == 0.5
    assert aggregate_trajectory([0.5, 0.5, 0.5], AggregationScheme.CUMULATIVE_SUM) == 1.5
    assert aggregate_trajectory([0.2, 0.4], AggregationScheme.AVERAGE) == pytest.approx(0.3)
    assert aggregate_trajectory([0.1] * 10, AggregationScheme.CUMULATIVE_SUM) == 1.0  # CPython 3.12 sum()
    with pytest.raises(ValueError):
        aggregate_trajectory([], P)
    rnd = random.Random(5)
    for _ in range(300):
        r = [rnd.random() for _ in range(rnd.randrange(1, 8))]
        assert aggregate_trajectory(r, MIN) >= aggregate_trajectory(r, P)
    cfg = ScoringConfig()
    assert classify_leaf(0.2, 1.0, cfg) is LeafClass.FUTILE
    assert classify_leaf(0.3, 1.0, cfg) is LeafClass.VIABLE
    pre = ScoringConfig(futility_bound=FutilityBound.PREFIX_AGGREGATE)
    assert classify_leaf(0.9, 0.25, pre) is LeafClass.FUTILE and classify_leaf(0.9, 0.25, cfg) is LeafClass.VIABLE
    for s in (AggregationScheme.CUMULATIVE_SUM, AggregationScheme.AVERAGE):
        with pytest.raises(UnsupportedSchemeError):
            classify_leaf(0.2, 1.0, ScoringConfig(scheme=s))


def test_cost_model_reference_cases():
    """test_backend.py TestCostModel."""
    from paper_2604_00510_b200.backend import CostModel, service_time

    m = CostModel(per_token_latency=0.002, engine_capacity=32)
    assert service_time(100, m, 10) == pytest.approx(0.200)
    assert service_time(100, m, 64) == pytest.approx(0.400)
    assert service_time(1, m, 0) == pytest.approx(0.002)
    d = CostModel()
    ts = [service_time(t, d, 0) for t in range(1, 200, 7)]
    assert all(a <= b for a, b in zip(ts, ts[1:]))
    ls = [service_time(80, d, x) for x in range(0, 200, 5)]
    assert all(a <= b for a, b in zip(ls, ls[1:]))
    with pytest.raises(ValueError):
        service_time(0, d, 0)
    with pytest.raises(ValueError):
        service_time(10, d, -1)
    with pytest.raises(ValueError):
        CostModel(per_token_latency=0.0)


def test_workload_json_is_byte_identical_to_reference():
    from paper_2604_00510_b200 import backend as B

    D7 = {d: (7, 7) for d in B.Difficulty}
    a = B.workload_to_json(B.make_workload(64, (0.6, 0.25, 0.15), 0, branching=4, depth_ranges=D7))
    assert a == load("workload_json")["c1"]
    assert B.workload_to_json(B.make_workload(40, (0.6, 0.25, 0.15), 20260810)) == load("workload_json")["cli_default"]
    back = B.workload_from_json(load("workload_json")["c1"])
    assert B.workload_to_json(back) == a
    assert [s.base_depth for s in back] == [s.base_depth for s in B.make_workload(64, (0.6, 0.25, 0.15), 0,
                                                                                    branching=4, depth_ranges=D7)]


def test_package_exports_the_reference_names():
    import paper_2604_00510_b200 as t

    for name in ("CostModel", "Difficulty", "StepCandidate", "SyntheticProblemSpec", "generate_steps",
                 "make_workload", "service_time", "BeamConfig", "beam_step", "run_beam_search", "RequestRecord",
                 "SummaryStats", "percentile", "records_to_csv", "summarize", "Job", "SchedulerConfig",
                 "SchedulerState", "AggregationScheme", "ExitDecision", "ExitKind", "ScoringConfig",
                 "aggregate_trajectory", "check_negative_exit", "check_positive_exit", "classify_leaf",
                 "decide_exit", "SearchOutcome", "run_tree_search", "SelectionParams"):
        assert hasattr(t, name), name


@pytest.mark.gpu
def test_device_generate_steps_matches_reference_kats():
    from paper_2604_00510_b200.backend import generate_steps_many

    kats = load("steps_kats")
    by_width = {}
    for k in kats:
        by_width.setdefault(k["width"], []).append(k)
    for width, ks in by_width.items():
        got = generate_steps_many([problem_from_record(k["problem"]) for k in ks], [k["path"] for k in ks], width)
        for k, cands in zip(ks, got):
            assert [[c.step_ref, c.token_count, c.prior, c.prm_reward, int(c.is_terminal)] for c in cands] == \
                k["candidates"], (k["path"], width)


@pytest.mark.gpu
def test_device_generate_steps_errors_like_reference():
    from paper_2604_00510_b200.backend import generate_steps

    rec = load("workloads")["c1"][0]
    p = problem_from_record(rec)
    golden = rec["golden_path"]
    if golden is not None:
        with pytest.raises(ValueError):
            generate_steps(p, golden, 4)  # the full golden path is terminal
    with pytest.raises(ValueError):
        generate_steps(p, [0] * (rec["base_depth"] + 2), 4)  # deeper than max_depth
    with pytest.raises(ValueError):
        generate_steps(p, [], 0)
    assert len(generate_steps(p, [], 7)) == 7  # width above branching repeats children
