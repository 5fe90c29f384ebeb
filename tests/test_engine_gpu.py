"""Parity of the CUDA engine with the reference, through the C-ABI (needs a B200).

Expected values are the committed fixtures made by the UNMODIFIED reference
(tests/golden/make_golden.py) and, for larger or random cases, the C oracle
(oracle/ts_oracle.c, itself pinned to those fixtures by tests/test_oracle.py).
Everything integer/index is compared exactly; floats are compared bit-for-bit
(the north star's 1e-12 Q tolerance is not needed: W accumulates in the
reference's order).
"""

import ctypes
import math
import random

import numpy as np
import pytest

from golden_io import WAVE_KEYS, assert_tree_equal, config_from_case, load, outcome_dict, table
from oracle import oracle

pytestmark = pytest.mark.gpu


def _engine(cfg):
    from paper_2604_00510_b200.engine import Engine

    return Engine(cfg, 0)


OUT_KEYS = ("exit_kind", "rollouts_completed", "tokens_generated", "best_score", "best_len", "solved",
            "exit_step", "admit_step", "launched", "cancelled", "nodes", "status")


def _cmp_outcomes(got, want, label):
    for i, (a, b) in enumerate(zip(got, want)):
        for k in OUT_KEYS:
            assert getattr(a, k) == getattr(b, k), f"{label}[{i}].{k}: {getattr(a, k)!r} != {getattr(b, k)!r}"
        assert list(a.best_path[: a.best_len]) == list(b.best_path[: b.best_len]), f"{label}[{i}] best_path"


@pytest.mark.parametrize("case_idx", range(6))
def test_serial_goldens(case_idx):
    """run_tree_search per request (search.py:79) == waves of one rollout."""
    case = load("serial")[case_idx]
    recs = load("workloads")[case["workload"]]
    cfg = config_from_case(case)
    with _engine(cfg) as eng:
        eng.load(table(recs))
        eng.run()
        outs = eng.outcomes()
        for o, want in zip(outs, case["outcomes"]):
            w = dict(want)
            pid = w.pop("problem_id")
            assert outcome_dict(o) == w, pid
        for idx, tree in case["trees"].items():
            assert_tree_equal(eng.tree(int(idx)), tree, f"{case['name']}[{idx}]")


def test_deep_tree_goldens():
    for case in load("deep_trees"):
        rec = load("workloads")[case["workload"]][case["index"]]
        with _engine(config_from_case(case)) as eng:
            eng.load(table([rec]))
            eng.run()
            assert_tree_equal(eng.tree(0), case["tree"], case["name"])


@pytest.mark.parametrize("name", [c["name"] for c in load("waves")])
def test_wave_goldens(name):
    """Boosted virtual-loss waves vs the reference-composed wave oracle, step by step."""
    case = next(c for c in load("waves") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case)
    import torch

    n = len(recs)
    with _engine(cfg) as eng:
        eng.load(table(recs, case["arrival_steps"]))
        counts = torch.zeros(3, dtype=torch.int64, device="cuda")
        records = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
        trace = []
        for step in range(case["steps"]):
            eng.step_counts(step, counts.data_ptr())
            eng.step_admit(step, counts.data_ptr(), 1, 0)
            eng.step_records(step, records.data_ptr())
            eng.step_targets(step, records.data_ptr())
            t = eng.read_targets()
            run = [x for x in t if x > 0]
            if run:
                trace.append(run)
            eng.step_wave(step)
        assert trace == case["targets_trace"]
        st = eng.stats()
        assert st.steps == case["steps"]
        outs = eng.outcomes()
        for i, want in enumerate(case["outcomes"]):
            got = outcome_dict(outs[i])
            for k in got:
                assert got[k] == want[k], (name, i, k)
            for k in WAVE_KEYS:
                assert getattr(outs[i], k) == want[k], (name, i, k)
        for idx, tree in case["trees"].items():
            assert_tree_equal(eng.tree(int(idx)), tree, f"{name}[{idx}]")
    # the one-call run path (the CUDA-graph loop the bench times) agrees with
    # the reference on every per-wave field and on the trees too
    with _engine(cfg) as eng:
        eng.load(table(recs, case["arrival_steps"]))
        st = eng.run()
        assert st.steps == case["steps"]
        outs = eng.outcomes()
        for i, want in enumerate(case["outcomes"]):
            assert outcome_dict(outs[i]) == {k: want[k] for k in outcome_dict(outs[i])}
            for k in WAVE_KEYS:
                assert getattr(outs[i], k) == want[k], (name, "graph", i, k)
        for idx, tree in case["trees"].items():
            assert_tree_equal(eng.tree(int(idx)), tree, f"{name}[{idx}] graph")


def test_compute_targets_kats():
    """Device compute_targets (k_targets) vs the reference's KATs, fed raw records."""
    import torch

    from paper_2604_00510_b200._abi import TsSchedRecord
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig
    from paper_2604_00510_b200.scoring import ScoringConfig

    dummy = load("workloads")["c1"][0]
    for kat in load("targets_kats"):
        n = len(kat["jobs"])
        sch = SchedulerConfig(max_concurrency=kat["M"], beta=kat["beta"], proximity=kat["proximity"],
                              obs_threshold=kat["obs_threshold"], boosting_enabled=kat["boosting"])
        cfg = SearchConfig(scoring=ScoringConfig(positive_exit_threshold=kat["theta_pos"]), scheduler=sch)
        recs = (TsSchedRecord * n)()
        for i, (arr, comp, best) in enumerate(kat["jobs"]):
            ratio = best / kat["theta_pos"]
            boosted = ratio > kat["proximity"]
            recs[i].score = math.log1p(kat["now_step"] - arr) + (kat["beta"] if boosted else 0.0)
            recs[i].flags = 1 | (2 if comp >= kat["obs_threshold"] else 0) | (4 if boosted else 0)
        dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
        with _engine(cfg) as eng:
            eng.load(table([dummy] * n))
            eng.step_targets(kat["now_step"], dev.data_ptr())
            assert eng.read_targets() == kat["targets"], kat


def _random_targets_case(rng, n, lockstep):
    M = n + rng.randint(0, 6 * n)
    now = rng.randint(0, 60)
    rows, arr = [], 0
    for _ in range(n):
        if not lockstep and rng.random() < 0.3:
            arr = min(now, arr + rng.randint(0, 3))
        rows.append((0 if lockstep else arr, rng.randint(0, 4), rng.choice([0.0, 0.46, 0.44, rng.random() * 0.6])))
    return M, now, rows


@pytest.mark.parametrize("n", [1, 7, 300, 1025, 5000, 20000, 70000, 140000])
def test_compute_targets_random_vs_oracle(n):
    """Larger pools (multi-chunk scans, long runs, lock-step ties) vs the oracle's
    literal sorted loop (scheduler.py:143-187 restated in oracle/ts_oracle.c).
    Above 65,536 records the cooperative k_mt_all keeps its run-block offsets
    in global memory (the phase-7 path)."""
    import torch

    from paper_2604_00510_b200._abi import TsConfig, TsSchedRecord
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    rng = random.Random(n)
    dummy = load("workloads")["c1"][0]
    for trial in range(4):
        M, now, rows = _random_targets_case(rng, n, lockstep=trial % 2 == 0)
        sch = SchedulerConfig(max_concurrency=M, obs_threshold=rng.choice([1, 2, 3]))
        cfg = SearchConfig(scheduler=sch)
        c = cfg.to_c()
        want = oracle.compute_targets(c, now, [r[0] for r in rows], [r[1] for r in rows], [r[2] for r in rows])
        recs = (TsSchedRecord * n)()
        for i, (arr, comp, best) in enumerate(rows):
            boosted = best / 0.5 > sch.proximity
            recs[i].score = math.log1p(now - arr) + (sch.beta if boosted else 0.0)
            recs[i].flags = 1 | (2 if comp >= sch.obs_threshold else 0) | (4 if boosted else 0)
        dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
        with _engine(cfg) as eng:
            eng.load(table([dummy] * n))
            eng.step_targets(now, dev.data_ptr())
            assert eng.read_targets() == want, (n, trial)


@pytest.mark.parametrize("name,multi_cta", [("c1_M48_admission", False), ("c1_M48_admission", True),
                                             ("cli_serving_pe_ne_boost", False), ("cli_serving_pe_ne_boost", True),
                                             ("c2_s512_M2048", True), ("c2_s512_M2048", "nocoop")])
def test_sharded_engines_match_single(name, multi_cta, monkeypatch):
    """Block sharding of the run queue over 3 engines (one 'rank' each) with the
    exchanges done by device copies == one engine: the multi-GPU step contract
    (FIFO admission across ranks, Poisson arrivals, the boosting exchange),
    with the one-CTA or the many-CTA scheduler step."""
    import torch

    if multi_cta:
        monkeypatch.setenv("TS_MT_MIN", "0")
    if multi_cta == "nocoop":  # the many-CTA step as separate kernels instead of one cooperative launch
        monkeypatch.setenv("TS_MT_COOP", "0")
    case = next(c for c in load("waves") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case)
    n = len(recs)
    bounds = [0, n // 3, (2 * n) // 3 + 1, n]
    arr = case.get("arrival_steps")
    engines = []
    for r in range(3):
        e = _engine(cfg)
        lo, hi = bounds[r], bounds[r + 1]
        e.load(table(recs[lo:hi], arr[lo:hi] if arr else None), global_offset=lo, n_global=n)
        engines.append(e)
    counts = [torch.zeros(3, dtype=torch.int64, device="cuda") for _ in engines]
    recbufs = [torch.zeros((bounds[r + 1] - bounds[r]) * 16, dtype=torch.uint8, device="cuda") for r in range(3)]
    for step in range(case["steps"]):
        for e, c in zip(engines, counts):
            e.step_counts(step, c.data_ptr())
        allc = torch.cat(counts)
        for r, e in enumerate(engines):
            e.step_admit(step, allc.data_ptr(), 3, r)
        for e, b in zip(engines, recbufs):
            e.step_records(step, b.data_ptr())
        allr = torch.cat(recbufs)
        for e in engines:
            e.step_targets(step, allr.data_ptr())
            e.step_wave(step)
    got = [o for e in engines for o in e.outcomes()]
    for i, want in enumerate(case["outcomes"]):
        g = outcome_dict(got[i])
        for k in g:
            assert g[k] == want[k], (i, k)
        for k in WAVE_KEYS:
            assert getattr(got[i], k) == want[k], (i, k)
    for e in engines:
        e.close()


@pytest.mark.parametrize("preset", ["c2_exits_off_P1", "c2_full", "c4_stagnation"])
def test_random_batches_vs_oracle(preset):
    """Bigger batches vs the C oracle: trees node by node for a sample."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    if preset == "c2_exits_off_P1":
        specs = B.make_workload(256, (0.6, 0.25, 0.15), 3, branching=4,
                                depth_ranges={d: (15, 15) for d in B.Difficulty})
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=1 << 30, boosting_enabled=False),
                           rollout_budget=32, depth_cap=16, expand_width=4, positive_exit=False,
                           negative_exit=False)
    elif preset == "c2_full":
        specs = B.make_workload(1024, (0.6, 0.25, 0.15), 11, branching=4,
                                depth_ranges={d: (15, 15) for d in B.Difficulty})
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=2048), rollout_budget=128, depth_cap=16,
                           expand_width=4)
    else:
        from paper_2604_00510_b200 import keyed
        specs = [B.make_problem(f"s{i}", keyed.mix(5, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                                B.stagnation_profile()) for i in range(16)]
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=64), rollout_budget=64, depth_cap=32,
                           expand_width=8)
    t = B.problem_table(specs)
    ref = oracle.OracleRun(t, cfg.to_c(), threads=8)
    with _engine(cfg) as eng:
        eng.load(t)
        st = eng.run()
        _cmp_outcomes(eng.outcomes(), ref.outcomes, preset)
        assert st.steps == ref.steps
        assert st.rollouts == ref.stats.rollouts and st.nodes + len(specs) == ref.stats.nodes
        for i in (0, 1, len(specs) - 1):
            assert_tree_equal(eng.tree(i), ref.tree(i), f"{preset}[{i}]")
    ref.close()


def test_host_end_to_end_call():
    """ts_run_batch_host: host problems in, host outcomes out, one C call."""
    case = load("serial")[0]
    recs = load("workloads")[case["workload"]]
    with _engine(config_from_case(case)) as eng:
        outs, st = eng.run_batch_host(table(recs))
        for o, want in zip(outs, case["outcomes"]):
            w = dict(want)
            w.pop("problem_id")
            assert outcome_dict(o) == w


def test_dropin_run_tree_search_matches_reference_outcomes():
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.search import run_tree_search, run_tree_searches

    D7 = {d: (7, 7) for d in B.Difficulty}
    specs = B.make_workload(64, (0.6, 0.25, 0.15), 0, branching=4, depth_ranges=D7)
    case = load("serial")[0]
    outs = run_tree_searches(specs, rollout_budget=32, depth_cap=8, expand_width=4)
    for o, want in zip(outs, case["outcomes"]):
        assert o.problem_id == want["problem_id"]
        assert o.exit_kind.value == want["exit_kind"]
        assert o.best_score == want["best_score"] and list(o.best_path) == want["best_path"]
        assert (o.rollouts_completed, o.tokens_generated, o.solved) == (
            want["rollouts_completed"], want["tokens_generated"], want["solved"])
    one = run_tree_search(specs[5], rollout_budget=32, depth_cap=8, expand_width=4)
    assert one == outs[5]


def test_invalid_config_raises():
    from paper_2604_00510_b200._abi import TsConfig
    from paper_2604_00510_b200.engine import Engine

    c = TsConfig()
    with pytest.raises(ValueError):
        Engine(c, 0)


@pytest.mark.parametrize("seed,M,budget,cap,b,base,scheme", [
    (0, 256, 32, 8, 4, 7, "cumulative_product"), (5, 4096, 128, 16, 4, 15, "cumulative_product"),
    (9, 512, 64, 12, 8, 11, "cumulative_product"), (3, 1024, 48, 6, 2, 7, "cumulative_product"),
    (11, 512, 64, 24, 4, 23, "cumulative_product"), (13, 512, 64, 12, 4, 11, "minimum"),
    (17, 256, 48, 10, 3, 9, "average")])
def test_pipelined_mode_matches_single_warp_mode(seed, M, budget, cap, b, base, scheme, monkeypatch):
    """Searches with many rollouts per wave run in the pipelined CTA mode
    (selector warp + simulator warps, in-order commits); the result must equal
    the single-warp mode bit for bit — outcomes and whole trees (all fold
    layouts, widths 2-8, and the product / minimum / average aggregations)."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig
    from paper_2604_00510_b200.scoring import AggregationScheme, ScoringConfig

    n = M // 4
    specs = B.make_workload(n, (0.5, 0.3, 0.2), seed, branching=b,
                            depth_ranges={d: (base, base) for d in B.Difficulty})
    t = B.problem_table(specs)
    sc = AggregationScheme(scheme)
    cfg = SearchConfig(scoring=ScoringConfig(scheme=sc), scheduler=SchedulerConfig(max_concurrency=M),
                       rollout_budget=budget, depth_cap=cap, expand_width=b,
                       negative_exit=sc in (AggregationScheme.CUMULATIVE_PRODUCT, AggregationScheme.MINIMUM))
    res = {}
    # "sync": the pipelined mode with every rollout committed before the next selection
    for mode in ("0", "1", "sync") if seed in (0, 13) else ("0", "1"):
        monkeypatch.setenv("TS_NO_PIPELINE", "0" if mode == "sync" else mode)
        monkeypatch.setenv("TS_PIPELINE_SYNC", "1" if mode == "sync" else "0")
        with _engine(cfg) as eng:
            eng.load(t)
            st = eng.run()
            outs = eng.outcomes()
            trees = [eng.tree(i) for i in range(0, n, max(1, n // 16))]
            res[mode] = (st.steps, st.rollouts, st.launched, st.nodes, outs, trees)
    c = res["1"]
    for mode, a in res.items():
        if mode == "1":
            continue
        assert a[:4] == c[:4]
        _cmp_outcomes(a[4], c[4], f"pipelined[{seed}/{mode}]")
        for x, y in zip(a[5], c[5]):
            assert_tree_equal(x, {k: v.tolist() for k, v in y.items()}, f"pipelined tree ({mode})")


def test_sum_scheme_q_out_of_range_raises_like_reference():
    """CUMULATIVE_SUM scores exceed 1, so W/N > 1 and wu_puct_score raises
    ValueError("q_value out of range") (tree.py:227-229) once a visited child is
    scored; the engine reports it per search and the drop-in raises it."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.scoring import AggregationScheme, ScoringConfig
    from paper_2604_00510_b200.search import run_tree_search

    p = B.make_workload(8, (1.0, 0.0, 0.0), 4, branching=2, depth_ranges={d: (4, 4) for d in B.Difficulty})[0]
    with pytest.raises(ValueError):
        run_tree_search(p, ScoringConfig(scheme=AggregationScheme.CUMULATIVE_SUM), rollout_budget=32,
                        depth_cap=8, expand_width=2, positive_exit=False, negative_exit=False)


def test_minimum_scheme_and_prefix_bound_trees_vs_oracle():
    """MINIMUM aggregation with the PREFIX_AGGREGATE futility bound under boosting."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig
    from paper_2604_00510_b200.scoring import AggregationScheme, FutilityBound, ScoringConfig

    specs = B.make_workload(300, (0.4, 0.3, 0.3), 21, branching=3,
                            depth_ranges={d: (5, 9) for d in B.Difficulty})
    t = B.problem_table(specs)
    cfg = SearchConfig(scoring=ScoringConfig(scheme=AggregationScheme.MINIMUM, futility_bound=FutilityBound.PREFIX_AGGREGATE,
                                             strict_negative_exit=True, positive_exit_threshold=0.6),
                       scheduler=SchedulerConfig(max_concurrency=900, obs_threshold=1), rollout_budget=40,
                       depth_cap=7, expand_width=3)
    ref = oracle.OracleRun(t, cfg.to_c(), threads=8)
    with _engine(cfg) as eng:
        eng.load(t)
        st = eng.run()
        _cmp_outcomes(eng.outcomes(), ref.outcomes, "min-prefix")
        assert st.steps == ref.steps
        for i in (0, 7, 150, 299):
            assert_tree_equal(eng.tree(i), ref.tree(i), f"min-prefix[{i}]")
    ref.close()


@pytest.mark.parametrize("boost", [True, False])
def test_serving_arrivals_vs_oracle(boost):
    """Config-5 shape: Poisson arrivals (reference generator, step-quantised),
    FIFO admission under M, PE(+NE+boost); the windowed scheduler vs the oracle."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    n = 6000
    specs = B.make_workload(n, (0.6, 0.25, 0.15), 20260810)
    arrivals = B.serving_arrival_steps(n, 1.0, 20260810, 1.0 / 700.0)
    t = B.problem_table(specs, arrivals)
    cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=1024, boosting_enabled=boost), rollout_budget=32,
                       depth_cap=16, expand_width=4, negative_exit=boost)
    ref = oracle.OracleRun(t, cfg.to_c(), threads=8)
    with _engine(cfg) as eng:
        eng.load(t)
        st = eng.run()
        _cmp_outcomes(eng.outcomes(), ref.outcomes, f"serving[{boost}]")
        assert st.steps == ref.steps
        for i in (0, 1234, n - 1):
            assert_tree_equal(eng.tree(i), ref.tree(i), f"serving[{i}]")
    ref.close()


def test_external_scheduler_targets():
    """ts_step_set_targets: the targets k_targets computes, replayed into a second
    engine through the external-scheduler hook, give the same batch bit for bit;
    all-ones targets give run_tree_search per problem (the serial fixtures)."""
    import torch

    case = next(c for c in load("waves") if c["name"] == "c1_M256")
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case)
    n = len(recs)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    records = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    with _engine(cfg) as a, _engine(cfg) as b:
        a.load(table(recs))
        b.load(table(recs))
        for step in range(case["steps"]):
            for e in (a, b):
                e.step_counts(step, counts.data_ptr())
                e.step_admit(step, counts.data_ptr(), 1, 0)
                e.step_records(step, records.data_ptr())
            a.step_targets(step, records.data_ptr())
            t = torch.tensor(a.read_targets(), dtype=torch.int32, device="cuda")
            b.step_set_targets(step, t.data_ptr())
            a.step_wave(step)
            b.step_wave(step)
        for i in range(n):
            assert outcome_dict(a.outcomes()[i]) == outcome_dict(b.outcomes()[i]), i
        for i in (0, 7, 33):
            assert_tree_equal(b.tree(i), {k: v.tolist() for k, v in a.tree(i).items()}, f"external[{i}]")
    serial = next(c for c in load("serial") if c["name"] == "c1_default")
    srecs = load("workloads")[serial["workload"]]
    scfg = config_from_case(serial)
    ones = torch.ones(len(srecs), dtype=torch.int32, device="cuda")
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    records = torch.zeros(len(srecs) * 16, dtype=torch.uint8, device="cuda")
    with _engine(scfg) as e:
        e.load(table(srecs))
        for step in range(serial["budget"] + 2):
            e.step_counts(step, counts.data_ptr())
            e.step_admit(step, counts.data_ptr(), 1, 0)
            e.step_records(step, records.data_ptr())
            e.step_set_targets(step, ones.data_ptr())
            e.step_wave(step)
        outs = e.outcomes()
    for i, want in enumerate(serial["outcomes"]):
        got = outcome_dict(outs[i])
        assert {k: got[k] for k in want if k in got} == {k: want[k] for k in want if k in got}, i


@pytest.mark.parametrize("name", ["c1_M256", "mixed_M200_obs3", "c2_s512_M2048"])
def test_policy_operator_drives_the_engine(name):
    """The standalone compute_targets operator (csrc/policy.cu, any run-queue
    order, device log1p) as the engine's external scheduler: fed the engine's
    own job state every wave, it reproduces the reference-composed wave oracle."""
    import torch

    from paper_2604_00510_b200.policy import compute_targets_arrays

    case = next(c for c in load("waves") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case)
    sched = cfg.scheduler
    n = len(recs)
    arrivals = case.get("arrival_steps") or [0] * n
    arr_t = torch.tensor(arrivals, dtype=torch.float64, device="cuda")
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    records = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    with _engine(cfg) as e:
        e.load(table(recs, case.get("arrival_steps")))
        for step in range(case["steps"]):
            e.step_counts(step, counts.data_ptr())
            e.step_admit(step, counts.data_ptr(), 1, 0)
            e.step_records(step, records.data_ptr())
            running, completed, best = e.read_jobs()
            idx = torch.nonzero(running, as_tuple=False).flatten()  # run queue = index order
            targets = torch.zeros(n, dtype=torch.int32, device="cuda")
            if idx.numel():
                t, _ = compute_targets_arrays(arr_t[idx], best[idx], completed[idx], ids[idx], float(step), sched,
                                              cfg.scoring.positive_exit_threshold)
                targets[idx] = t
            e.step_set_targets(step, targets.data_ptr())
            e.step_wave(step)
        outs = e.outcomes()
    for i, want in enumerate(case["outcomes"]):
        got = outcome_dict(outs[i])
        for k in got:
            assert got[k] == want[k], (name, i, k)


@pytest.mark.parametrize("unroll,no_graph", [(1, False), (2, False), (4, False), (3, True)])
def test_graph_loop_variants_match_oracle(unroll, no_graph, monkeypatch):
    """The graph loop with 1-4 passes per while-loop iteration (a batch that
    ends mid-body runs empty passes) and host-driven stepping give the oracle's
    outcomes; the batch mixes the P = 1 fast path (no free slot) with boosted
    passes (slots freed by exits) and a second batch reuses the instantiated graph."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    monkeypatch.setenv("TS_GRAPH_UNROLL", str(unroll))
    if no_graph:
        monkeypatch.setenv("TS_NO_GRAPH", "1")
    specs = B.make_workload(512, (0.6, 0.25, 0.15), 17, branching=4, depth_ranges={d: (11, 11) for d in B.Difficulty})
    cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=512), rollout_budget=64, depth_cap=12,
                       expand_width=4)
    t = B.problem_table(specs)
    ref = oracle.OracleRun(t, cfg.to_c(), threads=8)
    with _engine(cfg) as eng:
        for rep in range(2):
            eng.load(t)
            st = eng.run()
            _cmp_outcomes(eng.outcomes(), ref.outcomes, f"unroll{unroll}{'-nograph' if no_graph else ''}#{rep}")
            assert st.steps == ref.steps and st.rollouts == ref.stats.rollouts
    ref.close()


@pytest.mark.parametrize("case", ["boost_on_full_queue", "boost_off_arrivals"])
def test_free_running_waves(case, monkeypatch):
    """Free-running waves (k_sched: every search admitted, no exit before the
    budget, the next passes can only give P = 1) == the same batch with a
    scheduler pass per wave (TS_NO_FREE=1) == the C oracle: every outcome field
    (exit_step and admit_step included), the wave count, and trees node by node."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    n = 512
    specs = B.make_workload(n, (0.6, 0.25, 0.15), 17, branching=4, depth_ranges={d: (15, 15) for d in B.Difficulty})
    if case == "boost_on_full_queue":  # M = run queue: no free slot, every search advances in lockstep
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=n), rollout_budget=64, depth_cap=16,
                           expand_width=4, positive_exit=False, negative_exit=False)
        t = B.problem_table(specs)
    else:  # boosting off, staggered arrivals: free once the last search is admitted, unequal remaining budgets
        cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=4 * n, boosting_enabled=False),
                           rollout_budget=48, depth_cap=16, expand_width=4, positive_exit=False,
                           negative_exit=False)
        t = B.problem_table(specs)
        for i in range(n):
            t[i].arrival_step = (i * 20) // n
    runs = {}
    # k_wave_free (single-rollout kernel), the same waves inside k_wave, host-driven passes, one pass per wave
    envs = {"free": {}, "free_in_k_wave": {"TS_NO_FREE_KERNEL": "1"}, "host_driven": {"TS_NO_GRAPH": "1"},
            "per_wave": {"TS_NO_FREE": "1"}}
    for mode, env in envs.items():
        for k in ("TS_NO_FREE_KERNEL", "TS_NO_GRAPH", "TS_NO_FREE"):
            monkeypatch.delenv(k, raising=False)
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        with _engine(cfg) as eng:
            eng.load(t)
            st = eng.run()
            runs[mode] = (st, eng.outcomes(), [eng.tree(i) for i in (0, n // 2, n - 1)])
    sf, of, tf = runs["free"]
    sw = runs["per_wave"][0]
    assert sf.kernel_launches * 2 < sw.kernel_launches  # the free-running path was taken
    for mode in ("free_in_k_wave", "host_driven", "per_wave"):
        so, oo, to = runs[mode]
        assert (sf.steps, sf.rollouts, sf.nodes, sf.tokens) == (so.steps, so.rollouts, so.nodes, so.tokens), mode
        _cmp_outcomes(of, oo, f"{case}/{mode}")
        for a, b in zip(tf, to):
            assert_tree_equal(a, b, f"{case}/{mode}")
    ref = oracle.OracleRun(t, cfg.to_c(), threads=8)
    _cmp_outcomes(of, ref.outcomes, case)
    assert sf.steps == ref.steps
    assert_tree_equal(tf[1], ref.tree(n // 2), case)
    ref.close()
