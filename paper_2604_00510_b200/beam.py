"""Beam-search baseline (reference beam.py), drop-in names, run on the device.

``run_beam_search`` / ``run_beam_searches`` execute the whole
expansion-pruning loop of beam.py:143-176 for every problem in the sm_100a
kernel of csrc/beam.cu (one warp per problem), against the same replayed
synthetic backend the tree search uses.  Results come back as the
reference's ``BeamResult`` / ``Beam`` dataclasses.  No CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _abi
from ._abi import TsBeamConfig, TsBeamResult, load_library, raise_for_status
from .scoring import SCHEME_CODE, ScoringConfig

__all__ = ["Beam", "BeamConfig", "BeamResult", "run_beam_search", "run_beam_searches"]


@dataclass(frozen=True)
class BeamConfig:
    beam_width: int = 8
    candidates_per_beam: int = 4
    max_depth: int = 16
    positive_exit_enabled: bool = True

    def __post_init__(self) -> None:
        if self.beam_width < 1 or self.candidates_per_beam < 1 or self.max_depth < 1:
            raise ValueError("beam parameters must be positive")


@dataclass(frozen=True)
class Beam:
    """A partial (or finished) trajectory: child-index path plus its rewards."""

    index_path: tuple
    rewards: tuple
    score: float
    is_terminal: bool = False


@dataclass(frozen=True)
class BeamResult:
    problem_id: str
    best: Optional[Beam]
    complete: bool
    steps: int
    tokens_generated: int


def to_c(config: BeamConfig, scoring: ScoringConfig) -> TsBeamConfig:
    return TsBeamConfig(config.beam_width, config.candidates_per_beam, config.max_depth,
                        1 if config.positive_exit_enabled else 0, SCHEME_CODE[scoring.scheme], 0,
                        scoring.positive_exit_threshold)


def _table(problems):
    from .backend import problem_table

    if isinstance(problems, ctypes.Array):
        return problems
    if problems and isinstance(problems[0], _abi.TsProblem):
        arr = (_abi.TsProblem * len(problems))()
        for i, p in enumerate(problems):
            arr[i] = p
        return arr
    return problem_table(list(problems))


def run_beam_searches_raw(problems, cfg: TsBeamConfig, stream=None) -> list:
    """ts_beam_search_host over a problem table (ts_problem rows or specs)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the beam kernel runs on the CUDA device; no CUDA device is available")
    lib = load_library()
    table = _table(problems)
    n = len(table)
    out = (TsBeamResult * max(1, n))()
    s = int(torch.cuda.current_stream().cuda_stream) if stream is None else int(getattr(stream, "cuda_stream", stream))
    rc = lib.ts_beam_search_host(ctypes.byref(cfg), table if n else None, n, out, s)
    if rc == _abi.TS_INVALID_ARGUMENT:
        raise ValueError("beam search: invalid configuration (beam_width * candidates_per_beam must be <= "
                         f"{_abi.TS_BEAM_MAX_CANDIDATES})")
    raise_for_status(rc, "ts_beam_search_host")
    return list(out[:n])


def _result(spec, r: TsBeamResult) -> BeamResult:
    best = None
    if r.has_best:
        best = Beam(tuple(r.best_path[: r.best_len]), tuple(r.best_rewards[: r.best_len]), r.best_score,
                    bool(r.is_terminal))
    pid = getattr(spec, "problem_id", "")
    return BeamResult(pid, best, bool(r.complete), r.steps, r.tokens_generated)


def run_beam_searches(problems: Sequence, config: Optional[BeamConfig] = None,
                      scoring: Optional[ScoringConfig] = None) -> list:
    """run_beam_search (beam.py:143-176) for every problem in one kernel launch."""
    config = config or BeamConfig()
    scoring = scoring or ScoringConfig()
    raw = run_beam_searches_raw(problems, to_c(config, scoring))
    return [_result(p, r) for p, r in zip(problems, raw)]


def run_beam_search(problem, config: Optional[BeamConfig] = None,
                    scoring: Optional[ScoringConfig] = None) -> BeamResult:
    """Iterate expansion and pruning until the depth limit, beam exhaustion,
    or a finished trajectory meets the positive-exit threshold."""
    return run_beam_searches([problem], config, scoring)[0]
