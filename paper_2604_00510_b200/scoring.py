"""Scoring/exit-policy configuration (reference scoring.py:38-103).

The exit tests themselves run on the device after every backup (csrc/engine.cu:
``decide_exit`` with an incremental viable-leaf counter in place of the
reference's full-tree scan, scoring.py:153-175).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass


class UnsupportedSchemeError(Exception):
    """A scheme without the leaf upper bound was used for pruning (scoring.py:38)."""


class AggregationScheme(enum.Enum):
    MINIMUM = "minimum"
    CUMULATIVE_PRODUCT = "cumulative_product"
    CUMULATIVE_SUM = "cumulative_sum"
    AVERAGE = "average"


_PRUNABLE_SCHEMES = (AggregationScheme.MINIMUM, AggregationScheme.CUMULATIVE_PRODUCT)
SCHEME_CODE = {
    AggregationScheme.MINIMUM: 0,
    AggregationScheme.CUMULATIVE_PRODUCT: 1,
    AggregationScheme.CUMULATIVE_SUM: 2,
    AggregationScheme.AVERAGE: 3,
}


class FutilityBound(enum.Enum):
    LEAF_REWARD = "leaf_reward"
    PREFIX_AGGREGATE = "prefix_aggregate"


class ExitKind(enum.Enum):
    CONTINUE = "continue"
    POSITIVE_EXIT = "positive"
    NEGATIVE_EXIT = "negative"
    BUDGET_EXHAUSTED = "budget_exhausted"


EXIT_FROM_CODE = {
    0: ExitKind.CONTINUE,
    1: ExitKind.POSITIVE_EXIT,
    2: ExitKind.NEGATIVE_EXIT,
    3: ExitKind.BUDGET_EXHAUSTED,
}


@dataclass(frozen=True)
class ExitDecision:
    kind: ExitKind
    best_score: float


@dataclass(frozen=True)
class ScoringConfig:
    """Aggregation scheme plus exit thresholds (scoring.py:76-103)."""

    scheme: AggregationScheme = AggregationScheme.CUMULATIVE_PRODUCT
    accept_threshold: float = 0.3
    positive_exit_threshold: float = 0.5
    first_step_threshold: float = 0.1
    strict_negative_exit: bool = False
    futility_bound: FutilityBound = FutilityBound.LEAF_REWARD

    def __post_init__(self) -> None:
        if not 0.0 < self.accept_threshold < 1.0:
            raise ValueError(f"accept_threshold out of (0,1): {self.accept_threshold}")
        if not 0.0 < self.positive_exit_threshold < 1.0:
            raise ValueError(f"positive_exit_threshold out of (0,1): {self.positive_exit_threshold}")
        if not 0.0 <= self.first_step_threshold < 1.0:
            raise ValueError(f"first_step_threshold out of [0,1): {self.first_step_threshold}")


def check_scheme_for_pruning(config: ScoringConfig) -> None:
    """classify_leaf's scheme check (scoring.py:124-127), raised up front the
    way SimulationConfig.__post_init__ does (simulator.py:106-110)."""
    if config.scheme not in _PRUNABLE_SCHEMES:
        raise UnsupportedSchemeError(
            f"negative exit is unsound under {config.scheme.value} aggregation"
        )
