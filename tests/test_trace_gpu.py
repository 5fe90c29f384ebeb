"""The per-pass trace: allocation / action / job_finished
records of a wave run, byte-identical to the trace a wave run composed only of
reference calls writes (tests/golden/wave_ref.py with ``trace=``:
``parallelism_score`` and ``reconcile`` of scheduler.py, the record shapes of
simulator.py:240-249, 314-341, the JSONL text of cli.py:263-265).

The engine writes one row per running search per pass on the device
(``ts_engine_set_trace`` / ``k_trace``), through both the CUDA-graph loop
(``ts_run``) and the host-driven step API (``ts_step_*``)."""

import pytest

from golden_io import config_from_case, load, table

pytestmark = pytest.mark.gpu

CASES = [c["name"] for c in load("trace")]


def _wave_case(name):
    return next(c for c in load("waves") if c["name"] == name)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("path", ["graph", "steps"])
def test_trace_matches_reference(name, path):
    import torch

    from paper_2604_00510_b200.engine import Engine
    from paper_2604_00510_b200.metrics import trace_entries, trace_to_jsonl

    want = next(c for c in load("trace") if c["name"] == name)
    case = _wave_case(want["wave_case"])
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    n = len(recs)
    with Engine(config_from_case(case), 0) as eng:
        eng.set_trace(64 * n * case["budget"])
        eng.load(table(recs, case["arrival_steps"]))
        if path == "graph":
            eng.run()
        else:
            counts = torch.zeros(3, dtype=torch.int64, device="cuda")
            records = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
            for step in range(case["steps"]):
                eng.step_counts(step, counts.data_ptr())
                eng.step_admit(step, counts.data_ptr(), 1, 0)
                eng.step_records(step, records.data_ptr())
                eng.step_targets(step, records.data_ptr())
                eng.step_wave(step)
        text = trace_to_jsonl(trace_entries(eng.trace_rows(), eng.outcomes(), want["dt"]))
    assert text == want["jsonl"]


def test_trace_overflow_is_reported():
    from paper_2604_00510_b200.engine import Engine
    from paper_2604_00510_b200.tree import AccountingError

    case = _wave_case("c1_M256")
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    with Engine(config_from_case(case), 0) as eng:
        eng.set_trace(8)
        eng.load(table(recs, case["arrival_steps"]))
        eng.run()
        with pytest.raises(AccountingError):
            eng.trace_rows()
        eng.set_trace(0)
        eng.load(table(recs, case["arrival_steps"]))
        eng.run()
        assert len(eng.trace_rows()) == 0
