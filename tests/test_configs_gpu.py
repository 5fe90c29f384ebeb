"""Every BASELINE.json config at its STATED size vs the pinned C oracle (needs a B200).

The oracle (oracle/ts_oracle.c, pinned to the unmodified reference by
tests/test_oracle.py and the fixtures of tests/golden/) replays each whole
batch on the host cores; the engine runs it through its timed path (ts_run's
CUDA-graph loop) with the invariant kernels on (ts_engine_set_checks), so the
same run is compared with the oracle — every outcome field, the step count,
the run totals and whole trees of sampled searches — AND checked against the
reference's run-time invariants on the device state of every wave:

* capacity: at most M rollouts in flight per wave, |running| <= M
  (simulator.py:258-260, test_acceptance.py:167-187);
* serial gate: a search below obs_threshold runs one rollout (same test);
* rollout conservation: launched == completed + cancelled per search, and no
  rollout in flight (O == 0 on every node) when a wave ends
  (simulator.py:252-255, test_simulator.py:58-64);
* root N == completed_rollouts;
* negative exit on every unsolvable request when negative exit is on
  (test_acceptance.py:291-304).

Sizes: C2 4096 x 128 (with and without exits), C3 32,768 searches with M =
4 x 32,768 (P = 4) as one engine and as 8 block-sharded engines exchanging
through the step API, C4 1024 x 1024 rollouts at depth 32 (b = 8), C5 65,536
Poisson arrivals at M = 4096 for the `pe` and `pe_ne_boost` arms.
"""

import os

import pytest

from golden_io import assert_tree_equal
from oracle import oracle

pytestmark = pytest.mark.gpu

MIX = (0.6, 0.25, 0.15)
THREADS = os.cpu_count() or 1
OUT_KEYS = ("exit_kind", "rollouts_completed", "tokens_generated", "best_score", "best_len", "solved",
            "exit_step", "admit_step", "launched", "cancelled", "nodes", "status")


def cfg_of(M, budget, cap, width, pe=True, ne=True, boost=True):
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    return SearchConfig(scheduler=SchedulerConfig(max_concurrency=M, boosting_enabled=boost), rollout_budget=budget,
                        depth_cap=cap, expand_width=width, positive_exit=pe, negative_exit=ne)


def config_case(name):
    """(specs, table, SearchConfig) of a BASELINE config at its stated size."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200 import keyed

    D15 = {d: (15, 15) for d in B.Difficulty}
    if name == "c1":
        specs = B.make_workload(64, MIX, 0, branching=4, depth_ranges={d: (7, 7) for d in B.Difficulty})
        return specs, B.problem_table(specs), cfg_of(64, 32, 8, 4)
    if name in ("c2", "c2off"):
        ex = name == "c2"
        specs = B.make_workload(4096, MIX, 0, branching=4, depth_ranges=D15)
        return specs, B.problem_table(specs), cfg_of(4096, 128, 16, 4, ex, ex)
    if name in ("c3", "c3off"):
        ex = name == "c3"
        specs = B.make_workload(32768, MIX, 0, branching=4, depth_ranges=D15)
        return specs, B.problem_table(specs), cfg_of(4 * 32768, 128, 16, 4, ex, ex)
    if name == "c4":
        specs = [B.make_problem(f"s{i:04d}", keyed.mix(0, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                                B.stagnation_profile()) for i in range(1024)]
        return specs, B.problem_table(specs), cfg_of(1024, 1024, 32, 8)
    if name in ("c5_pe", "c5_pe_ne_boost"):
        n = 65536
        specs = B.make_workload(n, MIX, 20260810)
        arrivals = B.serving_arrival_steps(n, 1.0, 20260810, 1.0 / 2800.0)
        boost = name == "c5_pe_ne_boost"
        return specs, B.problem_table(specs, arrivals), cfg_of(4096, 32, 16, 4, True, boost, boost)
    raise KeyError(name)


_ORACLE = {}


def oracle_run(name):
    """One oracle run per config per session (the big ones take tens of seconds)."""
    if name not in _ORACLE:
        specs, t, cfg = config_case(name)
        _ORACLE[name] = oracle.OracleRun(t, cfg.to_c(), threads=THREADS)
    return _ORACLE[name]


def cmp_outcomes(got, want, label):
    assert len(got) == len(want)
    for i, (a, b) in enumerate(zip(got, want)):
        for k in OUT_KEYS:
            assert getattr(a, k) == getattr(b, k), f"{label}[{i}].{k}: {getattr(a, k)!r} != {getattr(b, k)!r}"
        assert bytes(a.best_path[: a.best_len]) == bytes(b.best_path[: b.best_len]), f"{label}[{i}] best_path"


def assert_invariants(inv, M, label):
    assert inv["waves"] > 0, label
    for k in ("capacity_violations", "gate_violations", "inflight_nodes", "conservation_violations",
              "root_mismatches"):
        assert inv[k] == 0, f"{label}: {k} = {inv[k]} ({inv})"
    assert inv["max_wave_launched"] <= M and inv["max_running"] <= M, (label, inv)


def assert_negative_exit_on_unsolvable(specs, outs, cfg, label):
    """Criterion 10 (test_acceptance.py:291-304) where negative exit is on."""
    if not cfg.negative_exit:
        return
    from paper_2604_00510_b200 import backend as B

    unsolvable = [i for i, s in enumerate(specs) if s.difficulty is B.Difficulty.UNSOLVABLE]
    if not unsolvable:  # config 4 is all HARD_SOLVABLE (stagnation profile)
        return
    bad = [i for i in unsolvable if outs[i].exit_kind != 2]
    assert not bad, f"{label}: unsolvable searches without a negative exit: {bad[:10]}"


def sample_ids(n):
    return sorted({0, 1, n // 3, n // 2, n - 1})


@pytest.mark.parametrize("name", ["c1", "c2", "c2off", "c3", "c3off", "c4", "c5_pe", "c5_pe_ne_boost"])
def test_config_at_stated_size_vs_oracle(name):
    from paper_2604_00510_b200.engine import Engine

    specs, t, cfg = config_case(name)
    ref = oracle_run(name)
    n = len(specs)
    with Engine(cfg, 0) as eng:
        eng.set_checks(True)
        eng.load(t)
        st = eng.run()
        outs = eng.outcomes()
        cmp_outcomes(outs, ref.outcomes[:n], name)
        assert st.steps == ref.steps, name
        assert st.rollouts == ref.stats.rollouts and st.launched == ref.stats.launched, name
        assert st.nodes + n == ref.stats.nodes and st.tokens == ref.stats.tokens, name
        assert_invariants(eng.invariants(), cfg.scheduler.max_concurrency, name)
        assert_negative_exit_on_unsolvable(specs, outs, cfg, name)
        for i in sample_ids(n):
            assert_tree_equal(eng.tree(i), ref.tree(i), f"{name}[{i}]")


@pytest.mark.parametrize("name", ["c3off", "c3"])
def test_config3_as_eight_sharded_engines(name):
    """Config 3 as 8 ranks of 4096 searches on one GPU: block-sharded engines
    (ts_load_problems(global_offset, n_global)) exchanging counts and scheduler
    records through the step API every wave (device copies standing in for the
    NCCL all-gathers); the 32,768-record scheduler step runs on many CTAs."""
    import torch

    from paper_2604_00510_b200.engine import Engine

    specs, t, cfg = config_case(name)
    ref = oracle_run(name)
    world, n = 8, len(specs)
    per = n // world
    engines = []
    for r in range(world):
        e = Engine(cfg, 0)
        e.set_checks(True)
        e.load(t[r * per:(r + 1) * per], global_offset=r * per, n_global=n)
        engines.append(e)
    counts = [torch.zeros(3, dtype=torch.int64, device="cuda") for _ in engines]
    recs = [torch.zeros(per * 16, dtype=torch.uint8, device="cuda") for _ in engines]
    steps = 0
    for step in range(1 << 20):
        for e, c in zip(engines, counts):
            e.step_counts(step, c.data_ptr())
        allc = torch.cat(counts)
        if int(allc.view(world, 3)[:, 2].sum()) == 0:
            steps = step
            break
        for r, e in enumerate(engines):
            e.step_admit(step, allc.data_ptr(), world, r)
        for e, b in zip(engines, recs):
            e.step_records(step, b.data_ptr())
        allr = torch.cat(recs)
        for e in engines:
            e.step_targets(step, allr.data_ptr())
            e.step_wave(step)
    assert steps == ref.steps
    outs = [o for e in engines for o in e.outcomes()]
    cmp_outcomes(outs, ref.outcomes[:n], f"{name}-sharded")
    for r, e in enumerate(engines):
        inv = e.invariants()
        assert inv["capacity_violations"] == inv["gate_violations"] == inv["inflight_nodes"] == 0, (r, inv)
        assert inv["conservation_violations"] == inv["root_mismatches"] == 0, (r, inv)
    for i in (0, per - 1, 5 * per + 7):
        r, j = divmod(i, per)
        assert_tree_equal(engines[r].tree(j), ref.tree(i), f"{name}-sharded[{i}]")
    for e in engines:
        e.close()
