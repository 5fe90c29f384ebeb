"""Request records, CSV and summaries in the reference's formats (metrics.py),
against bytes produced by the reference's own metrics module
(tests/golden/metrics.json.gz)."""

from __future__ import annotations

from types import SimpleNamespace

import pytest

from golden_io import config_from_case, load, table
from paper_2604_00510_b200.metrics import percentile, records_from_outcomes, records_to_csv, summarize
from paper_2604_00510_b200.scoring import ExitKind


def _case(name):
    return next(c for c in load("waves") if c["name"] == name)


def test_percentile_nearest_rank():
    assert percentile([5.0, 1.0, 3.0, 2.0, 4.0], 50.0) == 3.0
    assert percentile([5.0, 1.0, 3.0, 2.0, 4.0], 99.0) == 5.0
    assert percentile([1.0] * 100 + [9.0], 99.0) == 1.0
    with pytest.raises(ValueError):
        percentile([], 50.0)
    with pytest.raises(ValueError):
        percentile([1.0], 0.0)


def test_records_reproduce_reference_bytes_from_fixture_outcomes():
    for m in load("metrics"):
        case = _case(m["case"])
        outs = [SimpleNamespace(exit_kind=ExitKind(o["exit_kind"]), exit_step=o["exit_step"],
                                rollouts_completed=o["rollouts_completed"], cancelled=o["cancelled"],
                                tokens_generated=o["tokens_generated"], best_score=o["best_score"],
                                solved=o["solved"], best_path=tuple(o["best_path"]))
                for o in case["outcomes"]]
        recs = records_from_outcomes(outs, [o["problem_id"] for o in case["outcomes"]], case["arrival_steps"],
                                     m["dt"])
        assert records_to_csv(recs) == m["csv"]
        assert summarize(recs).to_json() == m["summary"]


@pytest.mark.gpu
def test_engine_serving_run_reproduces_reference_csv():
    from paper_2604_00510_b200.engine import Engine

    for m in load("metrics"):
        case = _case(m["case"])
        recs_in = load("workloads")[case["workload"]][: len(case["outcomes"])]
        with Engine(config_from_case(case), 0) as eng:
            eng.load(table(recs_in, case["arrival_steps"]))
            eng.run()
            outs = eng.outcomes()
        recs = records_from_outcomes(outs, [r["problem_id"] for r in recs_in], case["arrival_steps"], m["dt"])
        assert records_to_csv(recs) == m["csv"]
        assert summarize(recs).to_json() == m["summary"]


@pytest.mark.gpu
def test_engine_tree_json_is_byte_identical_to_reference():
    """Engine.tree_json vs SearchTree.to_json() of the same serial search (tests/golden/tree_json)."""
    from golden_io import scoring_from_record
    from paper_2604_00510_b200.config import serial_config
    from paper_2604_00510_b200.engine import Engine

    for case in load("tree_json"):
        rec = load("workloads")[case["workload"]][case["index"]]
        cfg = serial_config(scoring_from_record(case["scoring"]), rollout_budget=case["budget"],
                            depth_cap=case["depth_cap"], expand_width=case["expand_width"],
                            positive_exit=case["positive_exit"], negative_exit=case["negative_exit"])
        with Engine(cfg, 0) as eng:
            eng.load(table([rec]))
            eng.run()
            assert eng.tree_json(0) == case["json"]


def test_trace_assembly_reproduces_reference_trace():
    """Host half of the trace (metrics.trace_entries/trace_to_jsonl) on CPU:
    rows taken from the reference trace's own allocation records and the wave
    fixture's exit steps rebuild the reference JSONL byte for byte."""
    import json
    from types import SimpleNamespace

    import numpy as np

    from paper_2604_00510_b200.metrics import trace_entries, trace_to_jsonl

    for case in load("trace"):
        wave = next(c for c in load("waves") if c["name"] == case["wave_case"])
        entries = [json.loads(x) for x in case["jsonl"].splitlines()]
        alloc = [e for e in entries if e["kind"] == "allocation"]
        dt = np.dtype([("step", "<i4"), ("job", "<i4"), ("target", "<i4"), ("active", "<i4"), ("score", "<f8")])
        rows = np.array([(round(e["time"] / case["dt"]), e["job"], e["target"], e["active"], e["score"])
                         for e in alloc], dtype=dt)[::-1]
        code = {"positive": 1, "negative": 2, "budget_exhausted": 3}
        outs = [SimpleNamespace(exit_kind=code[o["exit_kind"]], exit_step=o["exit_step"]) for o in wave["outcomes"]]
        rows = rows[np.lexsort((rows["job"], rows["step"]))]
        assert trace_to_jsonl(trace_entries(rows, outs, case["dt"])) == case["jsonl"], case["name"]
