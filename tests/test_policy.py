"""Standalone policy operators (csrc/policy.cu) behind the reference's scheduler
and exit-policy entry points (scheduler.py:118-233, scoring.py:153-207).

CPU tests pin the C oracle's general-run-queue and forest checkers to the
reference fixtures (tests/golden/policy_kats.json.gz, made by
tests/golden/make_golden.py from the unmodified reference) and cover the host
bookkeeping; the GPU tests run the kernels against the same fixtures, the
reference's own unit-test cases, and the oracle at larger sizes.
"""

from __future__ import annotations

import math
import random
from collections import deque
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import pytest

from golden_io import load
from oracle import oracle
from paper_2604_00510_b200._abi import TsConfig
from paper_2604_00510_b200.policy import flatten_trees
from paper_2604_00510_b200.scheduler import (
    InflightRollout,
    Job,
    JobState,
    LaunchAction,
    PreemptAction,
    SchedulerConfig,
    SchedulerState,
    admit_jobs,
    choose_preemption_victims,
    on_rollout_complete,
    reconcile,
)
from paper_2604_00510_b200.scoring import (
    AggregationScheme,
    ExitDecision,
    ExitKind,
    FutilityBound,
    ScoringConfig,
    UnsupportedSchemeError,
)

THETA_POS = 0.5
KIND_CODE = {"continue": 0, "positive": 1, "negative": 2, "budget_exhausted": 3}


# ---- a minimal reference-shaped SearchTree (duck type of tree.py:117-181) --------
@dataclass
class Node:
    node_id: int
    parent_id: Optional[int]
    prm_reward: float
    depth: int
    is_terminal: bool = False
    children: list = field(default_factory=list)


@dataclass(frozen=True)
class Traj:
    node_path: tuple
    aggregate_score: float
    rollout_index: int = 0


class MiniTree:
    def __init__(self, rollout_budget=32):
        self.rollout_budget = rollout_budget
        self.nodes = {0: Node(0, None, 1.0, 0)}
        self.root_id = 0
        self.completed_rollouts = 0
        self.best_trajectory = None

    @property
    def root(self):
        return self.nodes[0]

    def expand(self, leaf, rewards, terminal=None):
        ids = []
        for i, r in enumerate(rewards):
            nid = len(self.nodes)
            self.nodes[nid] = Node(nid, leaf, r, self.nodes[leaf].depth + 1,
                                   bool(terminal[i]) if terminal else False)
            self.nodes[leaf].children.append(nid)
            ids.append(nid)
        return ids


def tree_with_leaf_rewards(firsts, leaves):
    t = MiniTree()
    fs = t.expand(0, firsts)
    for b, lr in zip(fs, leaves):
        if lr:
            t.expand(b, lr)
    return t


def scoring_from(rec) -> ScoringConfig:
    return ScoringConfig(scheme=AggregationScheme(rec["scheme"]), accept_threshold=rec["accept_threshold"],
                         positive_exit_threshold=rec["positive_exit_threshold"],
                         first_step_threshold=rec["first_step_threshold"],
                         strict_negative_exit=rec["strict_negative_exit"],
                         futility_bound=FutilityBound(rec["futility_bound"]))


def ts_cfg(kat) -> TsConfig:
    c = TsConfig()
    c.max_concurrency = kat["M"]
    c.beta = kat["beta"]
    c.proximity = kat["proximity"]
    c.obs_threshold = kat["obs_threshold"]
    c.boosting_enabled = int(kat["boosting"])
    c.positive_exit_threshold = kat["theta_pos"]
    return c


def sched_cfg(kat) -> SchedulerConfig:
    return SchedulerConfig(max_concurrency=kat["M"], beta=kat["beta"], proximity=kat["proximity"],
                           obs_threshold=kat["obs_threshold"], boosting_enabled=kat["boosting"])


def cols(kat):
    j = kat["jobs"]
    return ([r[0] for r in j], [r[1] for r in j], [r[2] for r in j], [r[3] for r in j])


# ================================ CPU: the checker and the host glue ====================
def test_golden_log1p_is_this_hosts_libm():
    for x, y in load("policy_kats")["log1p"]:
        assert math.log1p(x) == y


def test_oracle_general_targets_match_reference():
    for kat in load("policy_kats")["targets"]:
        arr, comp, best, ids = cols(kat)
        assert oracle.compute_targets_general(ts_cfg(kat), kat["now"], arr, comp, best, ids) == kat["targets"]


def test_oracle_target_errors_match_reference():
    for case in load("policy_kats")["target_errors"]:
        c = TsConfig()
        c.max_concurrency = 20
        c.beta, c.proximity, c.obs_threshold, c.positive_exit_threshold = 2.0, 0.9, 2, 0.5
        c.boosting_enabled = int(case["boosting"])
        args = (c, 3.0, [0.0, 1.0, 4.5, 2.0, 7.0], [0] * 5, [0.0] * 5, list(range(5)))
        if "error" in case:
            with pytest.raises(ValueError, match="precedes arrival=4.5"):
                oracle.compute_targets_general(*args)
        else:
            assert oracle.compute_targets_general(*args) == case["targets"]


def _forest_answers(fixture):
    trees = fixture["trees"]
    flat = flatten_trees(trees)
    flat_ex = flatten_trees(trees, [True] * len(trees))
    return trees, flat, flat_ex


def _expected(tree, ci, pe, ne, ex):
    v = tree["answers"][ci][f"{int(pe)}{int(ne)}{int(ex)}"]
    return -5 if v == "unsupported" else KIND_CODE[v[0]]


def test_oracle_forest_policy_matches_reference():
    from paper_2604_00510_b200.config import scoring_to_c

    fx = load("policy_kats")
    trees, flat, flat_ex = _forest_answers(fx)
    fields = ("offsets", "parent", "reward", "depth", "flags", "best_score", "has_best", "completed", "budget",
              "exhausted")
    for ci, sc in enumerate(fx["scoring"]):
        s = scoring_from(sc)
        for pe in (True, False):
            for ne in (True, False):
                for ex in (False, True):
                    f = flat_ex if ex else flat
                    kinds, nes = oracle.forest_policy(scoring_to_c(s, pe, ne), *[f[k] for k in fields])
                    for t, tree in enumerate(trees):
                        assert kinds[t] == _expected(tree, ci, pe, ne, ex), (ci, t, pe, ne, ex)
                        want_ne = tree["answers"][ci]["ne"]
                        assert nes[t] == (2 if want_ne == "unsupported" else int(want_ne))


def test_flatten_accepts_tree_objects_and_dumps():
    t = tree_with_leaf_rewards([0.05, 0.5], [[0.50], [0.25]])
    t.best_trajectory = Traj((1,), 0.4)
    t.completed_rollouts = 3
    a = flatten_trees([t])
    assert a["offsets"].tolist() == [0, 5]
    assert a["parent"].tolist() == [-1, 0, 0, 1, 2]
    assert a["flags"].tolist() == [2, 2, 2, 0, 0]
    assert a["best_score"].tolist() == [0.4] and a["has_best"].tolist() == [1]
    d = {"root": 0, "nodes": [{"id": n.node_id, "parent": n.parent_id, "reward": n.prm_reward, "depth": n.depth,
                               "terminal": n.is_terminal} for n in t.nodes.values()]}
    b = flatten_trees([d, t])
    assert b["offsets"].tolist() == [0, 5, 10]
    assert b["parent"][5:].tolist() == [-1, 5, 5, 6, 7]


def make_job(job_id, arrival=0.0, completed=5, best=0.0, state=JobState.RUNNING):
    job = Job(job_id=job_id, arrival_time=arrival, tree=MiniTree(32))
    job.completed_rollouts = completed
    job.best_score = best
    job.state = state
    return job


def running_state(jobs, now=0.0):
    return SchedulerState(pending_queue=deque(), run_queue=list(jobs), now=now)


def test_admission_fifo_up_to_capacity():
    """test_scheduler.py TestAdmission."""
    pending = deque(make_job(i, state=JobState.PENDING) for i in range(20))
    state = SchedulerState(pending_queue=pending, run_queue=[], now=0.0)
    admit_jobs(state, SchedulerConfig(max_concurrency=16))
    assert [j.job_id for j in state.run_queue] == list(range(16))
    assert [j.job_id for j in state.pending_queue] == [16, 17, 18, 19]
    assert all(j.state is JobState.RUNNING and j.target_parallelism == 1 for j in state.run_queue)
    full = SchedulerState(pending_queue=deque([make_job(99, state=JobState.PENDING)]),
                          run_queue=[make_job(i) for i in range(4)])
    admit_jobs(full, SchedulerConfig(max_concurrency=4))
    assert len(full.run_queue) == 4 and full.pending_queue[0].job_id == 99


@pytest.mark.gpu
def test_reconcile_and_victims():
    """test_scheduler.py TestReconcile, on the device operator (ts_reconcile)."""
    def with_active(scores):
        job = make_job(0)
        job.active_rollouts = [InflightRollout(i, s) for i, s in enumerate(scores)]
        return job

    acts = reconcile(running_state([with_active([0.9, 0.2, 0.5, 0.1])]), {0: 2})
    assert {a.rollout_id for a in acts if isinstance(a, PreemptAction)} == {1, 3}
    assert reconcile(running_state([with_active([0.9])]), {0: 3}) == [LaunchAction(0, 2)]
    assert reconcile(running_state([with_active([0.9, 0.5])]), {0: 2}) == []
    rnd = random.Random(21)
    for _ in range(100):
        scores = [round(rnd.uniform(0, 1), 3) for _ in range(rnd.randrange(1, 10))]
        rollouts = [InflightRollout(i, s) for i, s in enumerate(scores)]
        k = rnd.randrange(0, len(rollouts) + 1)
        assert choose_preemption_victims(rollouts, k) == sorted(rollouts, key=lambda r: (r.prefix_score,
                                                                                            r.rollout_id))[:k]


def test_on_rollout_complete():
    """test_scheduler.py TestOnRolloutComplete (host bookkeeping)."""
    job = make_job(0)
    job.active_rollouts = [InflightRollout(i, 0.5) for i in range(3)]
    state = running_state([job])
    acts = on_rollout_complete(state, job, ExitDecision(ExitKind.POSITIVE_EXIT, 0.9))
    assert len(acts) == 3 and job.state is JobState.FINISHED and job.finished_kind is ExitKind.POSITIVE_EXIT
    assert job not in state.run_queue
    job = make_job(0)
    state = running_state([job])
    assert on_rollout_complete(state, job, ExitDecision(ExitKind.CONTINUE, 0.1)) == []
    assert job.state is JobState.RUNNING
    job = make_job(0)
    job.tree.best_trajectory = Traj((1,), 0.42)
    job.tree.completed_rollouts = 7
    on_rollout_complete(running_state([job]), job, ExitDecision(ExitKind.CONTINUE, 0.42))
    assert job.best_score == 0.42 and job.completed_rollouts == 7


def test_policy_ops_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_00510_b200.scheduler import compute_targets
    from paper_2604_00510_b200.scoring import check_negative_exit

    with pytest.raises(RuntimeError):
        compute_targets(running_state([make_job(0)]), SchedulerConfig(), THETA_POS)
    with pytest.raises(RuntimeError):
        check_negative_exit(tree_with_leaf_rewards([0.5], [[0.25]]), ScoringConfig())


# ================================ GPU: the kernels ========================================
@pytest.mark.gpu
def test_device_log1p_matches_libm():
    from paper_2604_00510_b200.policy import parallelism_scores_arrays

    xs = [x for x, _ in load("policy_kats")["log1p"] if x < 1e300]
    want = [y for x, y in load("policy_kats")["log1p"] if x < 1e300]
    # arrival 0, best 0: the score is log1p(now - 0) exactly; one call per value of now
    # would be slow, so use now = 0 and arrival = -x (waited = 0 - (-x) = x exactly)
    got = parallelism_scores_arrays([-x for x in xs], [0.0] * len(xs), 0.0, 0.5, SchedulerConfig()).cpu().tolist()
    assert got == want
    rnd = random.Random(5)
    more = [rnd.uniform(0, 1e4) * rnd.choice([1.0, 1e-3, 1e-9]) for _ in range(200000)]
    got = parallelism_scores_arrays(np.negative(more), np.zeros(len(more)), 0.0, 0.5, SchedulerConfig()).cpu()
    assert got.tolist() == [math.log1p(x) for x in more]


@pytest.mark.gpu
def test_device_targets_match_reference_kats():
    from paper_2604_00510_b200.policy import compute_targets_arrays, parallelism_scores_arrays

    for kat in load("policy_kats")["targets"]:
        arr, comp, best, ids = cols(kat)
        out, info = compute_targets_arrays(arr, best, comp, ids, kat["now"], sched_cfg(kat), kat["theta_pos"])
        assert out.cpu().tolist() == kat["targets"], kat
        if kat["scores"] is not None:
            s = parallelism_scores_arrays(arr, best, kat["now"], kat["theta_pos"], sched_cfg(kat))
            assert s.cpu().tolist() == kat["scores"]


@pytest.mark.gpu
def test_device_targets_errors_like_reference():
    from paper_2604_00510_b200.scheduler import compute_targets

    for case in load("policy_kats")["target_errors"]:
        state = SchedulerState(now=3.0)
        for i, a in enumerate([0.0, 1.0, 4.5, 2.0, 7.0]):
            state.run_queue.append(make_job(i, arrival=a, completed=0))
        cfg = SchedulerConfig(max_concurrency=20, boosting_enabled=case["boosting"])
        if "error" in case:
            with pytest.raises(ValueError, match=r"now=3\.0 precedes arrival=4\.5"):
                compute_targets(state, cfg, 0.5)
        else:
            assert compute_targets(state, cfg, 0.5) == dict(enumerate(case["targets"]))
    with pytest.raises(ValueError, match="no running jobs"):
        compute_targets(SchedulerState(), SchedulerConfig(), 0.5)


@pytest.mark.gpu
def test_reference_scheduler_unit_cases_on_device():
    """test_scheduler.py TestParallelismScore / TestComputeTargets through the drop-in API."""
    from paper_2604_00510_b200.scheduler import compute_targets, parallelism_score

    cfg = SchedulerConfig(beta=2.0)
    assert parallelism_score(make_job(0, arrival=5.0, best=0.25), 5.0, THETA_POS, cfg) == 0.0
    assert parallelism_score(make_job(0, best=0.475), math.e - 1, THETA_POS, cfg) == pytest.approx(3.0)
    assert parallelism_score(make_job(0, best=0.45), math.e - 1, THETA_POS, cfg) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        parallelism_score(make_job(0, arrival=10.0), 9.0, THETA_POS, cfg)

    def scored(scores):
        return [make_job(i, arrival=-math.expm1(s), completed=10) for i, s in enumerate(scores)]

    assert compute_targets(running_state(scored([3.0, 1.0])), SchedulerConfig(max_concurrency=16), 0.5) == {0: 12, 1: 4}
    assert compute_targets(running_state(scored([2.0, 1.0])), SchedulerConfig(max_concurrency=10), 0.5) == {0: 7, 1: 3}
    jobs = scored([3.0, 1.0])
    jobs[0].completed_rollouts = 0
    t = compute_targets(running_state(jobs), SchedulerConfig(max_concurrency=16), 0.5)
    assert t[0] == 1 and t[1] >= 1
    t = compute_targets(running_state([make_job(i, arrival=10.0, completed=10) for i in range(3)], 10.0),
                        SchedulerConfig(max_concurrency=5), 0.5)
    assert sum(t.values()) == 5 and t[0] >= t[1] >= t[2]
    assert compute_targets(running_state(scored([3.0, 1.0])),
                           SchedulerConfig(max_concurrency=16, boosting_enabled=False), 0.5) == {0: 1, 1: 1}
    t = compute_targets(running_state(scored([6.5, 0.001, 0.001])), SchedulerConfig(max_concurrency=16), 0.5)
    assert sum(t.values()) <= 16 and min(t.values()) >= 1
    rnd = random.Random(3)
    for _ in range(100):
        jobs = [make_job(i, arrival=500.0 - rnd.uniform(0, 200), completed=rnd.choice([0, 1, 5, 9]),
                         best=rnd.uniform(0, 0.5)) for i in range(rnd.randrange(1, 10))]
        c = SchedulerConfig(max_concurrency=16)
        t = compute_targets(running_state(jobs, 500.0), c, 0.5)
        assert sum(t.values()) <= 16 and all(v >= 1 for v in t.values())
        assert all(t[j.job_id] == 1 for j in jobs if j.completed_rollouts < c.obs_threshold)
        if any(j.completed_rollouts >= c.obs_threshold for j in jobs):
            assert sum(t.values()) == 16


@pytest.mark.gpu
@pytest.mark.parametrize("n,kind", [(1, 0), (1023, 0), (1025, 1), (4096, 2), (50000, 0), (200000, 1), (70000, 3)])
def test_device_targets_vs_oracle_large(n, kind):
    """General run queues at sizes the fixtures do not reach: unsorted
    fractional arrivals, integer ties, a lock-step pool, and tiny waits whose
    log1p has bits below 2^-64 (the sequential-sum fallback)."""
    from paper_2604_00510_b200.policy import compute_targets_arrays

    rng = np.random.default_rng(n + kind)
    now = 1000.0
    if kind == 0:
        arr = rng.uniform(0, now, n)
    elif kind == 1:
        arr = rng.integers(0, 1000, n).astype(np.float64)
    elif kind == 2:
        arr = np.zeros(n)
    else:
        arr = now - rng.uniform(0, 1e-12, n)
    comp = rng.integers(0, 5, n).astype(np.int32)
    best = rng.choice([0.0, 0.3, 0.46, 0.44, 0.6], n)
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    for M in (n, n + 3, 4 * n + 7):
        cfg = SchedulerConfig(max_concurrency=M, obs_threshold=2)
        c = TsConfig()
        c.max_concurrency, c.beta, c.proximity, c.obs_threshold, c.boosting_enabled = M, 2.0, 0.9, 2, 1
        c.positive_exit_threshold = 0.5
        want = oracle.compute_targets_general(c, now, arr, comp, best, ids)
        got, info = compute_targets_arrays(arr, best, comp, ids, now, cfg, 0.5)
        assert got.cpu().tolist() == want
        if kind == 3:
            assert info.sum_fallback == 1


@pytest.mark.gpu
def test_device_exit_policy_matches_reference_trees():
    from paper_2604_00510_b200.policy import Forest, exit_policy

    fx = load("policy_kats")
    trees = fx["trees"]
    forests = {False: Forest(trees), True: Forest(trees, [True] * len(trees))}
    for ci, sc in enumerate(fx["scoring"]):
        s = scoring_from(sc)
        for pe in (True, False):
            for ne in (True, False):
                for ex in (False, True):
                    kinds, nes = exit_policy(forests[ex], s, pe, ne)
                    for t, tree in enumerate(trees):
                        assert kinds[t] == _expected(tree, ci, pe, ne, ex), (ci, t, pe, ne, ex)
                        want_ne = tree["answers"][ci]["ne"]
                        assert nes[t] == (2 if want_ne == "unsupported" else int(want_ne))


@pytest.mark.gpu
def test_reference_scoring_unit_cases_on_device():
    """test_scoring.py TestNegativeExit / TestPositiveExit / TestDecideExit."""
    from paper_2604_00510_b200.scoring import check_negative_exit, check_positive_exit, decide_exit, decide_exits

    strict = ScoringConfig(strict_negative_exit=True)
    assert check_negative_exit(tree_with_leaf_rewards([0.5], [[0.25, 0.28]]), strict)
    assert not check_negative_exit(tree_with_leaf_rewards([0.5], [[0.25, 0.50]]), strict)
    t = tree_with_leaf_rewards([0.05, 0.5], [[0.50], [0.25]])
    assert check_negative_exit(t, ScoringConfig(first_step_threshold=0.1))
    assert not check_negative_exit(t, strict)
    assert not check_negative_exit(MiniTree(4), ScoringConfig())
    rnd = random.Random(11)
    trees = []
    for _ in range(200):
        firsts = [rnd.random() for _ in range(rnd.randrange(1, 4))]
        trees.append(tree_with_leaf_rewards(firsts, [[rnd.random() for _ in range(rnd.randrange(0, 3))]
                                                     for _ in firsts]))
    from paper_2604_00510_b200.scoring import check_negative_exit_many

    s_many = check_negative_exit_many(trees, strict)
    sel_many = check_negative_exit_many(trees, ScoringConfig())
    assert all(b for a, b in zip(s_many, sel_many) if a)

    def with_best(score):
        t = MiniTree(4)
        t.best_trajectory = Traj((1,), score)
        return t

    assert check_positive_exit(with_best(0.95), ScoringConfig(positive_exit_threshold=0.9))
    assert not check_positive_exit(MiniTree(4), ScoringConfig())
    assert check_positive_exit(with_best(0.9), ScoringConfig(positive_exit_threshold=0.9))
    t = tree_with_leaf_rewards([0.5], [[0.25, 0.28]])
    t.best_trajectory = Traj((1,), 0.95)
    d = decide_exit(t, ScoringConfig())
    assert d.kind is ExitKind.POSITIVE_EXIT and d.best_score == 0.95
    assert decide_exit(t, ScoringConfig(), False, False).kind is ExitKind.CONTINUE
    t = tree_with_leaf_rewards([0.5], [[0.45, 0.50]])
    t.best_trajectory = Traj((1,), 0.45)
    t.completed_rollouts = t.rollout_budget
    assert decide_exit(t, ScoringConfig()).kind is ExitKind.BUDGET_EXHAUSTED
    t.completed_rollouts = 1
    assert decide_exit(t, ScoringConfig()).kind is ExitKind.CONTINUE
    t = MiniTree(8)
    t.expand(0, [0.9], terminal=[True])
    assert decide_exit(t, ScoringConfig(), False, False, True).kind is ExitKind.BUDGET_EXHAUSTED
    with pytest.raises(UnsupportedSchemeError):
        check_negative_exit(tree_with_leaf_rewards([0.5], [[0.25]]), ScoringConfig(scheme=AggregationScheme.AVERAGE))
    # no leaf survives the selective filter: fires without raising (scoring.py:164-175)
    assert check_negative_exit(tree_with_leaf_rewards([0.05], [[0.25]]),
                               ScoringConfig(scheme=AggregationScheme.AVERAGE))
    assert len(decide_exits([], ScoringConfig())) == 0


@pytest.mark.gpu
def test_device_exit_policy_on_engine_trees_vs_oracle():
    """Deep engine-built trees (config-4 shape, prefix bound) through the forest
    kernels vs the oracle's forest checker."""
    from golden_io import table
    from paper_2604_00510_b200.config import SearchConfig, scoring_to_c
    from paper_2604_00510_b200.engine import Engine
    from paper_2604_00510_b200.policy import Forest, exit_policy

    recs = load("workloads")["c4_stagnation"][:6]
    cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=64), rollout_budget=48, depth_cap=32,
                       expand_width=8, positive_exit=False, negative_exit=False)
    with Engine(cfg, 0) as eng:
        eng.load(table(recs))
        eng.run()
        trees = []
        for i, o in enumerate(eng.outcomes()):
            d = eng.tree(i)
            d["best_score"] = o.best_score if o.best_len > 0 else None
            trees.append(d)
    fields = ("offsets", "parent", "reward", "depth", "flags", "best_score", "has_best", "completed", "budget",
              "exhausted")
    flat = flatten_trees(trees)
    for sc in (ScoringConfig(futility_bound=FutilityBound.PREFIX_AGGREGATE, accept_threshold=0.05),
               ScoringConfig(scheme=AggregationScheme.MINIMUM, futility_bound=FutilityBound.PREFIX_AGGREGATE,
                             accept_threshold=0.4),
               ScoringConfig(strict_negative_exit=True, accept_threshold=0.9)):
        want_k, want_ne = oracle.forest_policy(scoring_to_c(sc, True, True), *[flat[k] for k in fields])
        kinds, nes = exit_policy(Forest(trees), sc, True, True)
        assert kinds.tolist() == want_k.tolist()
        assert nes.tolist() == want_ne.tolist()


@pytest.mark.gpu
def test_engine_exit_decisions_agree_with_forest_policy():
    """The engine decides negative exit with an incremental viable-leaf count;
    the forest kernels of the standalone policy do the reference's full scan.
    On the engine's final trees (an exit happens after every expansion of its
    wave) both must give the engine's exit kind for every search."""
    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.engine import Engine
    from paper_2604_00510_b200.scheduler import SchedulerConfig
    from paper_2604_00510_b200.scoring import decide_exits

    kinds = {1: ExitKind.POSITIVE_EXIT, 2: ExitKind.NEGATIVE_EXIT, 3: ExitKind.BUDGET_EXHAUSTED}
    for scoring, b, depth, budget in ((ScoringConfig(), 4, 9, 48),
                                      (ScoringConfig(futility_bound=FutilityBound.PREFIX_AGGREGATE,
                                                     accept_threshold=0.35), 3, 7, 40),
                                      (ScoringConfig(scheme=AggregationScheme.MINIMUM, strict_negative_exit=True,
                                                     accept_threshold=0.4), 2, 6, 32)):
        specs = B.make_workload(256, (0.5, 0.3, 0.2), 21, branching=b, depth_ranges={d: (depth, depth)
                                                                                    for d in B.Difficulty})
        cfg = SearchConfig(scoring=scoring, scheduler=SchedulerConfig(max_concurrency=512), rollout_budget=budget,
                           depth_cap=depth + 1, expand_width=b)
        with Engine(cfg, 0) as eng:
            eng.load(B.problem_table(specs))
            eng.run()
            outs = eng.outcomes()
            trees = []
            for i, o in enumerate(outs):
                d = eng.tree(i)
                d["best_score"] = o.best_score if o.best_len > 0 else None
                d["completed_rollouts"] = o.rollouts_completed
                d["rollout_budget"] = budget
                trees.append(d)
        exhausted = [o.exit_kind == 3 and o.rollouts_completed < budget for o in outs]
        got = decide_exits(trees, scoring, True, True, exhausted)
        assert [g.kind for g in got] == [kinds[o.exit_kind] for o in outs]


@pytest.mark.gpu
def test_preemption_victims_criterion_4():
    """test_acceptance.py criterion 4: 200 seeded scenarios, victims == the
    lowest-prefix-reward sort (ties to the earlier launch), on the device."""
    rnd = random.Random(20260810 + 4)
    for _ in range(200):
        count = rnd.randrange(1, 12)
        rollouts = [InflightRollout(rollout_id=i, prefix_score=round(rnd.uniform(0, 1), 3)) for i in range(count)]
        rnd.shuffle(rollouts)
        victims = rnd.randrange(0, count + 1)
        assert choose_preemption_victims(rollouts, victims) == sorted(
            rollouts, key=lambda r: (r.prefix_score, r.rollout_id))[:victims]


@pytest.mark.gpu
def test_reconcile_large_run_queue_vs_sort():
    """ts_reconcile over 20,000 jobs (0-300 in-flight rollouts each, ties in the
    scores, targets above and below): every action equals the reference
    definition (scheduler.py:190-214) restated with sorted()."""
    import numpy as np

    from paper_2604_00510_b200.policy import reconcile_arrays

    rng = np.random.default_rng(7)
    n = 20000
    active = rng.integers(0, 300, n)
    active[rng.random(n) < 0.3] = 0
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(active)
    m = int(off[-1])
    scores = rng.choice([0.0, -0.0, 0.25, 0.5, 0.9], m) + (rng.random(m) < 0.5) * rng.random(m)
    ids = rng.permutation(m).astype(np.int64)
    targets = np.maximum(0, active + rng.integers(-320, 40, n)).astype(np.int32)
    running = (rng.random(n) < 0.9).astype(np.int32)
    launch, rank = reconcile_arrays(targets, off, scores, ids, running)
    launch, rank = launch.cpu().numpy(), rank.cpu().numpy()
    for j in range(n):
        a, b = int(off[j]), int(off[j + 1])
        gap = int(targets[j]) - (b - a) if running[j] else 0
        assert launch[j] == max(gap, 0), j
        want = [-1] * (b - a)
        if gap < 0:
            order = sorted(range(a, b), key=lambda r: (scores[r], ids[r]))
            for pos, r in enumerate(order[:-gap]):
                want[r - a] = pos
        assert rank[a:b].tolist() == want, j
