"""Helpers to read the committed golden fixtures (tests/golden/*.json.gz)."""

from __future__ import annotations

import functools
import gzip
import json
import os

from paper_2604_00510_b200._abi import TsProblem
from paper_2604_00510_b200.config import SearchConfig
from paper_2604_00510_b200.scheduler import SchedulerConfig
from paper_2604_00510_b200.scoring import AggregationScheme, FutilityBound, ScoringConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name: str):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt", encoding="utf-8") as f:
        return json.load(f)


def problem_from_record(rec, arrival_step: int = 0) -> TsProblem:
    p = TsProblem()
    prof = rec["profile"]
    p.seed = rec["seed"]
    p.branching = rec["branching"]
    p.base_depth = rec["base_depth"]
    p.hidden_until_depth = prof["hidden_until_depth"]
    p.has_shared = 1 if prof["shared_range"] else 0
    p.arrival_step = arrival_step
    p.off_lo, p.off_hi = prof["off_path_range"]
    if prof["shared_range"]:
        p.shared_lo, p.shared_hi = prof["shared_range"]
    if rec["golden_path"] is None:
        p.golden_len = -1
    else:
        p.golden_len = len(rec["golden_path"])
        for d, (s, r) in enumerate(zip(rec["golden_path"], rec["golden_rewards"])):
            p.golden_path[d] = s
            p.golden_rewards[d] = r
    return p


def table(records, arrival_steps=None):
    arr = (TsProblem * len(records))()
    for i, rec in enumerate(records):
        arr[i] = problem_from_record(rec, arrival_steps[i] if arrival_steps else 0)
    return arr


def scoring_from_record(s) -> ScoringConfig:
    return ScoringConfig(
        scheme=AggregationScheme(s["scheme"]),
        accept_threshold=s["accept_threshold"],
        positive_exit_threshold=s["positive_exit_threshold"],
        first_step_threshold=s["first_step_threshold"],
        strict_negative_exit=s["strict_negative_exit"],
        futility_bound=FutilityBound(s["futility_bound"]),
    )


def config_from_case(case) -> SearchConfig:
    sched = case.get("sched")
    sc = SchedulerConfig(**sched) if sched else SchedulerConfig(max_concurrency=1 << 30, boosting_enabled=False)
    return SearchConfig(
        scoring=scoring_from_record(case["scoring"]) if "scoring" in case else ScoringConfig(),
        scheduler=sc,
        rollout_budget=case["budget"],
        depth_cap=case["depth_cap"],
        expand_width=case["expand_width"],
        positive_exit=case["positive_exit"],
        negative_exit=case["negative_exit"],
    )


EXIT_NAMES = {0: None, 1: "positive", 2: "negative", 3: "budget_exhausted"}


def outcome_dict(o) -> dict:
    return {
        "exit_kind": EXIT_NAMES[o.exit_kind],
        "best_score": o.best_score,
        "best_path": list(o.best_path[: o.best_len]),
        "rollouts_completed": o.rollouts_completed,
        "tokens_generated": o.tokens_generated,
        "solved": bool(o.solved),
    }


WAVE_KEYS = ("exit_step", "admit_step", "launched", "cancelled", "nodes")


def assert_tree_equal(got: dict, want: dict, label: str = ""):
    import numpy as np

    n = len(want["parent"])
    assert len(got["parent"]) == n, f"{label}: node count {len(got['parent'])} != {n}"
    for k in ("parent", "reward", "prior", "N", "O", "W", "terminal", "depth", "step_ref"):
        g = np.asarray(got[k])
        w = np.asarray(want[k], dtype=g.dtype)
        bad = np.nonzero(g != w)[0]
        assert bad.size == 0, f"{label}: field {k} differs at node {bad[0]}: {g[bad[0]]!r} != {w[bad[0]]!r}"


def cost_case_config(case) -> SearchConfig:
    """SearchConfig of a tests/golden/cost.json.gz case (default scoring/selection)."""
    return SearchConfig(
        scheduler=SchedulerConfig(max_concurrency=case["max_concurrency"], boosting_enabled=case["boosting_enabled"]),
        rollout_budget=case["budget"], depth_cap=case["depth_cap"], expand_width=case["expand_width"],
        positive_exit=case["positive_exit"], negative_exit=case["negative_exit"])
