"""Drop-in search driver: the reference's ``run_tree_search`` (search.py:79-119)
and its batched, boosted generalisation, both executed by the CUDA engine.

* :func:`run_tree_search` — same signature and ``SearchOutcome`` as the
  reference; one request, serial rollouts.
* :func:`run_tree_searches` — the same for a whole batch: every request is an
  independent tree advanced one rollout per wave, so outcomes equal
  ``[run_tree_search(p, ...) for p in problems]``.
* :func:`run_waves` — adaptive parallel MCTS: FIFO admission under the
  concurrency budget M (admit_jobs), per-wave targets from the boosting
  scheduler (compute_targets), virtual-loss waves of P_i rollouts per search,
  exit checks after every backup with cancel-on-exit.

All three accept reference ``SyntheticProblemSpec`` objects or ours (duck-typed).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

from .backend import problem_table
from .config import SearchConfig
from .engine import Engine
from .scheduler import SchedulerConfig
from .scoring import EXIT_FROM_CODE, ExitKind, ScoringConfig
from .tree import DEFAULT_DEPTH_CAP, SelectionParams

__all__ = ["SearchOutcome", "run_tree_search", "run_tree_searches", "run_waves", "WaveOutcome"]


@dataclass(frozen=True)
class SearchOutcome:
    """Result of one complete tree search (search.py:32-42)."""

    problem_id: str
    exit_kind: ExitKind
    best_score: float
    best_path: tuple[int, ...]
    rollouts_completed: int
    tokens_generated: int
    solved: bool


@dataclass(frozen=True)
class WaveOutcome(SearchOutcome):
    """SearchOutcome plus the wave bookkeeping of the batched engine."""

    exit_step: int = -1
    admit_step: int = -1
    launched: int = 0
    cancelled: int = 0
    nodes: int = 0


def _raise_search_error(o, pid: str) -> None:
    from ._abi import raise_for_status

    raise_for_status(o.status, f"search {pid}")


def _outcome(o, pid: str, cls=SearchOutcome):
    if o.status:
        _raise_search_error(o, pid)
    base = dict(
        problem_id=pid,
        exit_kind=EXIT_FROM_CODE[o.exit_kind],
        best_score=o.best_score,
        best_path=tuple(o.best_path[: o.best_len]),
        rollouts_completed=o.rollouts_completed,
        tokens_generated=o.tokens_generated,
        solved=bool(o.solved),
    )
    if cls is WaveOutcome:
        base.update(exit_step=o.exit_step, admit_step=o.admit_step, launched=o.launched,
                    cancelled=o.cancelled, nodes=o.nodes)
    return cls(**base)


def run_tree_searches(
    problems: Sequence,
    scoring: Optional[ScoringConfig] = None,
    selection: Optional[SelectionParams] = None,
    rollout_budget: int = 32,
    depth_cap: int = DEFAULT_DEPTH_CAP,
    expand_width: int = 4,
    positive_exit: bool = True,
    negative_exit: bool = True,
    device: int = 0,
) -> list[SearchOutcome]:
    """``run_tree_search`` for every problem, all advanced concurrently."""
    cfg = SearchConfig(
        scoring=scoring or ScoringConfig(),
        selection=selection or SelectionParams(),
        scheduler=SchedulerConfig(max_concurrency=max(1, len(problems)), boosting_enabled=False),
        rollout_budget=rollout_budget,
        depth_cap=depth_cap,
        expand_width=expand_width,
        positive_exit=positive_exit,
        negative_exit=negative_exit,
    )
    with Engine(cfg, device) as eng:
        eng.load(problem_table(problems))
        eng.run()
        outs = eng.outcomes()
    return [_outcome(o, p.problem_id) for o, p in zip(outs, problems)]


def run_tree_search(
    problem,
    scoring: Optional[ScoringConfig] = None,
    selection: Optional[SelectionParams] = None,
    rollout_budget: int = 32,
    depth_cap: int = DEFAULT_DEPTH_CAP,
    expand_width: int = 4,
    positive_exit: bool = True,
    negative_exit: bool = True,
) -> SearchOutcome:
    """Reference-signature serial search (search.py:79-88).

    One deviation: with negative exit on, a CUMULATIVE_SUM or AVERAGE scheme
    raises ``UnsupportedSchemeError`` up front (SearchConfig), where the
    reference raises lazily inside ``classify_leaf`` (scoring.py:119-127) and
    so returns normally for a search whose tree never holds a check-relevant
    expandable leaf when an exit check runs (e.g. every depth-1 step below
    ``first_step_threshold``, or a positive exit at the first rollout)."""
    return run_tree_searches([problem], scoring, selection, rollout_budget, depth_cap, expand_width,
                             positive_exit, negative_exit)[0]


def run_waves(
    problems: Sequence,
    scoring: Optional[ScoringConfig] = None,
    selection: Optional[SelectionParams] = None,
    sched: Optional[SchedulerConfig] = None,
    rollout_budget: int = 32,
    depth_cap: int = DEFAULT_DEPTH_CAP,
    expand_width: int = 4,
    positive_exit: bool = True,
    negative_exit: bool = True,
    arrival_steps: Optional[Sequence[int]] = None,
    max_steps: int = (1 << 31) - 1,
    device: int = 0,
):
    """Adaptive parallel MCTS over a batch (or a step-quantised arrival stream).

    Returns ``(outcomes, stats)`` with one :class:`WaveOutcome` per problem.
    """
    cfg = SearchConfig(
        scoring=scoring or ScoringConfig(),
        selection=selection or SelectionParams(),
        scheduler=sched or SchedulerConfig(),
        rollout_budget=rollout_budget,
        depth_cap=depth_cap,
        expand_width=expand_width,
        positive_exit=positive_exit,
        negative_exit=negative_exit,
    )
    with Engine(cfg, device) as eng:
        eng.load(problem_table(problems, arrival_steps))
        stats = eng.run(max_steps)
        outs = eng.outcomes()
    return [_outcome(o, p.problem_id, WaveOutcome) for o, p in zip(outs, problems)], stats
