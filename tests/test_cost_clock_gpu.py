"""The cost model's wave clock (ts_engine_set_cost_model) on the
device vs the reference-composed wave clock (tests/golden/cost.json.gz, made by
wave_ref.run_waves(cost=CostModel(...)) from the reference's service_time) and
vs the pinned C oracle at config-5 size, every simulated time bit for bit; then
the paper's ablation directions on that clock (test_acceptance.py:231-269,
criteria 6-8)."""

import pytest

from golden_io import cost_case_config, load, table
from oracle import oracle

pytestmark = pytest.mark.gpu

CASES = [c["name"] for c in load("cost")]


def _run(case_cfg, tab, cost, path="graph", steps=None):
    import torch

    from paper_2604_00510_b200.engine import Engine

    eng = Engine(case_cfg, 0)
    eng.set_cost_model(cost)
    eng.load(tab)
    if path == "graph":
        eng.run()
    else:
        n = len(tab)
        counts = torch.zeros(3, dtype=torch.int64, device="cuda")
        records = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
        for step in range(steps):
            eng.step_counts(step, counts.data_ptr())
            eng.step_admit(step, counts.data_ptr(), 1, 0)
            eng.step_records(step, records.data_ptr())
            eng.step_targets(step, records.data_ptr())
            eng.step_wave(step)
    return eng


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("path", ["graph", "steps"])
def test_wave_clock_matches_reference(name, path):
    case = next(c for c in load("cost") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: case["n"]]
    eng = _run(cost_case_config(case), table(recs, case["arrival_steps"]), tuple(case["cost"]), path,
               case["steps"])
    done, arr = eng.sim_times()
    assert [o.tokens_generated for o in eng.outcomes()] == case["tokens"]
    assert done.tolist() == case["sim_completion"]
    assert arr.tolist() == case["sim_arrival"]
    eng.close()


@pytest.mark.parametrize("arm", ["pe", "pe_ne_boost"])
def test_wave_clock_config5_vs_oracle(arm):
    """65,536 Poisson arrivals at M = 4096 (config 5), default CostModel."""
    from test_configs_gpu import THREADS, config_case

    specs, t, cfg = config_case("c5_" + arm)
    cost = (0.002, 32, 0.01)
    ref = oracle.OracleRun(t, cfg.to_c(), threads=THREADS, cost=cost)
    eng = _run(cfg, t, cost)
    done, arr = eng.sim_times()
    rdone, rarr = ref.sim_times()
    assert (done == rdone).all() and (arr == rarr).all()
    eng.close()
    ref.close()


def test_ablation_directions_on_the_wave_clock():
    """Criteria 6-8 (test_acceptance.py:231-269) on the CLI workload (500
    requests, Poisson arrivals at rate 5 quantised to 20 steps per second,
    M = 16, default CostModel), tree-search presets on the device wave clock
    and the beam arms' tokens from the beam kernel."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.beam import BeamConfig, run_beam_searches
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.metrics import records_from_sim_times, summarize
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    specs = B.make_workload(500, (0.6, 0.25, 0.15), 20260810)
    arrivals = B.serving_arrival_steps(500, 5.0, 20260810, 20.0)
    tab = B.problem_table(specs, arrivals)
    stats = {}
    for preset, pe, ne, boost in (("vanilla", False, False, False), ("pe", True, False, False),
                                  ("pe_ne", True, True, False), ("pe_ne_boost", True, True, True)):
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=16, boosting_enabled=boost), rollout_budget=32,
                           depth_cap=16, expand_width=4, positive_exit=pe, negative_exit=ne)
        eng = _run(cfg, tab, (0.002, 32, 0.01))
        done, arr = eng.sim_times()
        recs = records_from_sim_times(eng.outcomes(), [s.problem_id for s in specs], done, arr)
        assert len(recs) == 500
        stats[preset] = summarize(recs)
        eng.close()
    p99 = {k: v.p99_latency for k, v in stats.items()}
    assert p99["pe"] < p99["vanilla"]                 # criterion 6
    assert p99["pe_ne"] <= p99["pe"]
    assert p99["pe_ne_boost"] <= p99["pe_ne"]
    thr = {k: v.throughput for k, v in stats.items()}
    assert thr["pe"] > thr["vanilla"]                 # criterion 8
    assert thr["pe_ne"] >= thr["pe"]
    tok = {k: v.total_tokens for k, v in stats.items()}
    beam = sum(r.tokens_generated for r in run_beam_searches(specs, BeamConfig()))
    beam_no_pe = sum(r.tokens_generated for r in run_beam_searches(specs, BeamConfig(positive_exit_enabled=False)))
    assert tok["vanilla"] < beam_no_pe                # criterion 7
    assert tok["pe"] < beam
    assert 1.0 - tok["pe"] / tok["vanilla"] > 1.0 - beam / beam_no_pe
