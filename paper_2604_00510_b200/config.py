"""Flatten the reference's frozen config dataclasses into the POD ts_config."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from ._abi import TS_MAX_DEPTH, TsConfig
from .scheduler import SchedulerConfig
from .scoring import SCHEME_CODE, FutilityBound, ScoringConfig, check_scheme_for_pruning
from .tree import DEFAULT_DEPTH_CAP, SelectionParams


@dataclass(frozen=True)
class SearchConfig:
    """Everything one batch of searches needs besides the problems: the
    reference's run_tree_search knobs (search.py:79-88) plus the three config
    dataclasses (scoring.py:76, tree.py:92, scheduler.py:77)."""

    scoring: ScoringConfig = field(default_factory=ScoringConfig)
    selection: SelectionParams = field(default_factory=SelectionParams)
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    rollout_budget: int = 32
    depth_cap: int = DEFAULT_DEPTH_CAP
    expand_width: int = 4
    positive_exit: bool = True
    negative_exit: bool = True

    def __post_init__(self) -> None:
        if self.rollout_budget < 1:
            raise ValueError("rollout_budget must be positive")
        if self.depth_cap < 1 or self.expand_width < 1:
            raise ValueError("depth cap and expand width must be positive")
        if self.negative_exit:
            check_scheme_for_pruning(self.scoring)

    def to_c(self) -> TsConfig:
        c = TsConfig()
        s, sel, sch = self.scoring, self.selection, self.scheduler
        c.scheme = SCHEME_CODE[s.scheme]
        c.futility_bound = 0 if s.futility_bound is FutilityBound.LEAF_REWARD else 1
        c.strict_negative_exit = int(s.strict_negative_exit)
        c.positive_exit = int(self.positive_exit)
        c.negative_exit = int(self.negative_exit)
        c.rollout_budget = self.rollout_budget
        c.depth_cap = min(self.depth_cap, 1 << 30)
        c.expand_width = self.expand_width
        c.max_concurrency = sch.max_concurrency
        c.obs_threshold = sch.obs_threshold
        c.boosting_enabled = int(sch.boosting_enabled)
        c.accept_threshold = s.accept_threshold
        c.positive_exit_threshold = s.positive_exit_threshold
        c.first_step_threshold = s.first_step_threshold
        c.c_puct = sel.c_puct
        c.beta = sch.beta
        c.proximity = sch.proximity
        return c


def serial_config(
    scoring: Optional[ScoringConfig] = None,
    selection: Optional[SelectionParams] = None,
    rollout_budget: int = 32,
    depth_cap: int = DEFAULT_DEPTH_CAP,
    expand_width: int = 4,
    positive_exit: bool = True,
    negative_exit: bool = True,
    max_concurrency: int = 1 << 30,
) -> SearchConfig:
    """run_tree_search semantics: boosting off, every request admitted at once."""
    return SearchConfig(
        scoring=scoring or ScoringConfig(),
        selection=selection or SelectionParams(),
        scheduler=SchedulerConfig(max_concurrency=max_concurrency, boosting_enabled=False),
        rollout_budget=rollout_budget,
        depth_cap=depth_cap,
        expand_width=expand_width,
        positive_exit=positive_exit,
        negative_exit=negative_exit,
    )


MAX_NODE_DEPTH = TS_MAX_DEPTH


def scoring_to_c(scoring: ScoringConfig, positive_exit: bool = True, negative_exit: bool = True) -> TsConfig:
    """The ScoringConfig part of ts_config (for the standalone exit policy)."""
    c = TsConfig()
    c.scheme = SCHEME_CODE[scoring.scheme]
    c.futility_bound = 0 if scoring.futility_bound is FutilityBound.LEAF_REWARD else 1
    c.strict_negative_exit = int(scoring.strict_negative_exit)
    c.positive_exit = int(positive_exit)
    c.negative_exit = int(negative_exit)
    c.accept_threshold = scoring.accept_threshold
    c.positive_exit_threshold = scoring.positive_exit_threshold
    c.first_step_threshold = scoring.first_step_threshold
    return c
