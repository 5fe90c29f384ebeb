"""Pin the C oracle (oracle/ts_oracle.c) against the reference's own outputs.

Every expected value comes from tests/golden/*.json.gz, produced by
tests/golden/make_golden.py from the UNMODIFIED reference.  Equality is exact
(floats compared bit-for-bit).  CPU only.
"""

import ctypes

import pytest

from golden_io import (WAVE_KEYS, assert_tree_equal, config_from_case, load, outcome_dict,
                       problem_from_record, table)
from oracle import oracle


def test_rng_kats():
    for kat in load("rng_kats"):
        keys = kat["keys"]
        assert oracle.mix(keys) == kat["mix"]
        assert oracle.uniform(keys) == kat["uniform"]
        lo, hi, v = kat["uniform_in"]
        assert oracle.uniform_in(lo, hi, keys) == v
        lo, hi, v = kat["randint"]
        assert oracle.randint_in(lo, hi, keys) == v
        rate, v = kat["exponential"]
        assert oracle.exponential(rate, keys) == v


@pytest.mark.parametrize("name", ["c1", "cli_default", "mixed_b3", "c4_stagnation", "c2"])
def test_problem_table_fill(name):
    recs = load("workloads")[name]
    if name == "c2":
        recs = recs[::16]
    for rec in recs:
        p = oracle.fill_problem(rec["seed"], rec["golden_path"] is not None, rec["depth_range"],
                                rec["branching"], rec["profile"])
        assert p.base_depth == rec["base_depth"]
        if rec["golden_path"] is None:
            assert p.golden_len == -1
        else:
            assert list(p.golden_path[: p.golden_len]) == rec["golden_path"]
            assert list(p.golden_rewards[: p.golden_len]) == rec["golden_rewards"]


def test_generate_steps_kats():
    for kat in load("steps_kats"):
        p = problem_from_record(kat["problem"])
        got = oracle.generate_steps(p, kat["path"], kat["width"])
        want = [(c[0], c[1], c[2], c[3], bool(c[4])) for c in kat["candidates"]]
        assert got == want


def test_generate_steps_rejects_terminal_context():
    kat = load("steps_kats")[0]
    p = problem_from_record(kat["problem"])
    deep = [0] * (p.base_depth + 2)
    with pytest.raises(ValueError):
        oracle.generate_steps(p, deep, 2)


@pytest.mark.parametrize("case_idx", range(6))
def test_serial_run_tree_search(case_idx):
    case = load("serial")[case_idx]
    recs = load("workloads")[case["workload"]]
    cfg = config_from_case(case).to_c()
    for rec, want in zip(recs, case["outcomes"]):
        o = oracle.run_tree_search(problem_from_record(rec), cfg)
        got = outcome_dict(o)
        w = dict(want)
        w.pop("problem_id")
        assert got == w, rec["problem_id"]


@pytest.mark.parametrize("case_idx", range(6))
def test_serial_trees_via_waves(case_idx):
    """Boosting off ⇒ waves of one rollout ⇒ run_tree_search trees, node by node."""
    case = load("serial")[case_idx]
    recs = load("workloads")[case["workload"]]
    cfg = config_from_case(case).to_c()
    run = oracle.OracleRun(table(recs), cfg, threads=4)
    for i, want in enumerate(case["outcomes"]):
        w = dict(want)
        w.pop("problem_id")
        assert outcome_dict(run.outcomes[i]) == w
    for idx, tree in case["trees"].items():
        assert_tree_equal(run.tree(int(idx)), tree, f"{case['name']}[{idx}]")
    run.close()


def test_deep_trees():
    for case in load("deep_trees"):
        rec = load("workloads")[case["workload"]][case["index"]]
        cfg = config_from_case(case).to_c()
        run = oracle.OracleRun(table([rec]), cfg)
        assert_tree_equal(run.tree(0), case["tree"], case["name"])
        run.close()


@pytest.mark.parametrize("name", [c["name"] for c in load("waves")])
def test_wave_oracle(name):
    case = next(c for c in load("waves") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case).to_c()
    trace_cap = sum(len(t) for t in case["targets_trace"])
    run = oracle.OracleRun(table(recs, case["arrival_steps"]), cfg, threads=4, trace_cap=trace_cap)
    assert run.steps == case["steps"]
    flat = [t for step in case["targets_trace"] for t in step]
    assert run.targets_trace() == flat
    for i, want in enumerate(case["outcomes"]):
        got = outcome_dict(run.outcomes[i])
        for k in got:
            assert got[k] == want[k], (name, i, k)
        for k in WAVE_KEYS:
            assert getattr(run.outcomes[i], k) == want[k], (name, i, k)
    for idx, tree in case["trees"].items():
        assert_tree_equal(run.tree(int(idx)), tree, f"{name}[{idx}]")
    run.close()


def test_compute_targets_kats():
    from paper_2604_00510_b200._abi import TsConfig

    for kat in load("targets_kats"):
        cfg = TsConfig()
        cfg.max_concurrency = kat["M"]
        cfg.beta = kat["beta"]
        cfg.proximity = kat["proximity"]
        cfg.obs_threshold = kat["obs_threshold"]
        cfg.boosting_enabled = int(kat["boosting"])
        cfg.positive_exit_threshold = kat["theta_pos"]
        arr = [j[0] for j in kat["jobs"]]
        comp = [j[1] for j in kat["jobs"]]
        best = [j[2] for j in kat["jobs"]]
        assert oracle.compute_targets(cfg, kat["now_step"], arr, comp, best) == kat["targets"]


@pytest.mark.parametrize("name", [c["name"] for c in load("cost")])
def test_wave_clock_matches_reference(name):
    """The oracle's wave clock of the cost model (or_run_waves_cost) equals the
    reference-composed wave run charging service_time/reward_latency
    (wave_ref.run_waves(cost=...)), every simulated time bit for bit."""
    from golden_io import cost_case_config

    case = next(c for c in load("cost") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: case["n"]]
    r = oracle.OracleRun(table(recs, case["arrival_steps"]), cost_case_config(case).to_c(), threads=4,
                         cost=case["cost"])
    done, arr = r.sim_times()
    assert r.steps == case["steps"]
    assert [o.tokens_generated for o in r.outcomes[: case["n"]]] == case["tokens"]
    assert done.tolist() == case["sim_completion"]
    assert arr.tolist() == case["sim_arrival"]
    r.close()
