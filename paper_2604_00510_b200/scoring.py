"""Scoring and exit policy (reference scoring.py), drop-in names.

Inside the engine the exit tests run on the device after every backup
(csrc/engine.cu: ``decide_exit`` with an incremental viable-leaf counter in
place of the reference's full-tree scan, scoring.py:153-175).  For callers
that hold their own trees, ``check_negative_exit``, ``check_positive_exit``
and ``decide_exit`` (and the batched ``decide_exits``) take reference-style
``SearchTree`` objects (or their ``to_dict()`` dumps) and run the standalone
forest kernels of csrc/policy.cu: one thread per node classifies the
expandable leaves, one per tree decides.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import Optional, Sequence


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


class LeafClass(enum.Enum):
    VIABLE = "viable"
    FUTILE = "futile"


def aggregate_trajectory(rewards, scheme: AggregationScheme) -> float:
    """One trajectory score from per-step rewards (scoring.py:106-116): min,
    left-to-right product, CPython float sum, or that sum over the length.
    (The engine computes the same incrementally on the device, `Agg`.)"""
    values = list(rewards)
    if len(values) == 0:
        raise ValueError("rewards must be non-empty")
    table = {
        AggregationScheme.MINIMUM: lambda v: min(v),
        AggregationScheme.CUMULATIVE_PRODUCT: lambda v: math.prod(v),
        AggregationScheme.CUMULATIVE_SUM: lambda v: sum(v),
    }
    if scheme in table:
        return table[scheme](values)
    return sum(values) / len(values)


def classify_leaf(leaf_reward: float, prefix_aggregate: float, config: ScoringConfig) -> LeafClass:
    """FUTILE iff the futility bound is below the acceptance threshold
    (scoring.py:119-134); only the minimum and product schemes admit a bound."""
    check_scheme_for_pruning(config)
    if config.futility_bound is FutilityBound.LEAF_REWARD:
        bound = leaf_reward
    else:
        bound = min(leaf_reward, prefix_aggregate)
    return LeafClass.FUTILE if bound < config.accept_threshold else LeafClass.VIABLE


_KIND_OF_CODE = EXIT_FROM_CODE


def _decisions(trees: Sequence, config: ScoringConfig, positive_enabled: bool, negative_enabled: bool,
               tree_exhausted: Optional[Sequence[bool]], device: int):
    from .policy import Forest, exit_policy

    forest = Forest(trees, tree_exhausted, device)
    kinds, ne = exit_policy(forest, config, positive_enabled, negative_enabled)
    return forest, kinds, ne


def _unsupported(config: ScoringConfig) -> UnsupportedSchemeError:
    return UnsupportedSchemeError(f"negative exit is unsound under {config.scheme.value} aggregation")


def decide_exits(trees: Sequence, config: ScoringConfig, positive_enabled: bool = True,
                 negative_enabled: bool = True, tree_exhausted: Optional[Sequence[bool]] = None,
                 device: int = 0) -> list:
    """decide_exit (scoring.py:184-207) for many trees in one pass on the device."""
    forest, kinds, _ = _decisions(trees, config, positive_enabled, negative_enabled, tree_exhausted, device)
    out = []
    for t, k in enumerate(kinds.tolist()):
        if k < 0:
            raise _unsupported(config)
        out.append(ExitDecision(_KIND_OF_CODE[k], float(forest.best[t]) if forest.has_best[t] else 0.0))
    return out


def decide_exit(tree, config: ScoringConfig, positive_enabled: bool = True, negative_enabled: bool = True,
                tree_exhausted: bool = False) -> ExitDecision:
    """Combine the exit checks after a completed rollout (scoring.py:184-207)."""
    return decide_exits([tree], config, positive_enabled, negative_enabled, [tree_exhausted])[0]


def check_negative_exit_many(trees: Sequence, config: ScoringConfig, device: int = 0) -> list:
    """check_negative_exit (scoring.py:153-175) for many trees on the device."""
    _, _, ne = _decisions(trees, config, False, True, None, device)
    res = []
    for v in ne.tolist():
        if v == 2:
            raise _unsupported(config)
        res.append(v == 1)
    return res


def check_negative_exit(tree, config: ScoringConfig) -> bool:
    """True when no check-relevant leaf can still reach the acceptance threshold."""
    return check_negative_exit_many([tree], config)[0]


def check_positive_exit(tree, config: ScoringConfig) -> bool:
    """True once the best completed trajectory meets the exit threshold (scoring.py:178-181)."""
    _, kinds, _ = _decisions([tree], config, True, False, None, 0)
    return int(kinds[0]) == 1
