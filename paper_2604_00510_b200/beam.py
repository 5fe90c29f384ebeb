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

__all__ = ["Beam", "BeamCandidate", "BeamConfig", "BeamResult", "BeamStep", "beam_step", "expand_beams",
           "prune_candidates", "run_beam_search", "run_beam_searches"]


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
class BeamCandidate:
    beam: Beam
    order: int  # candidate index within the step (tie-break)
    token_count: int


@dataclass(frozen=True)
class BeamStep:
    survivors: list
    finished: list
    tokens_generated: int


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


# ---- step-level operators (beam.py:76-131) on the device ---------------------------

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the beam kernels run on the CUDA device; no CUDA device is available")
    return torch


def _expand_raw(beams: Sequence[Beam], config: BeamConfig, scoring: ScoringConfig, problem):
    """ts_beam_expand for one problem: candidates (beam-major) with prune ranks."""
    from ._abi import TS_BEAM_MAX_CANDIDATES, TsBeam, TsBeamCandidate

    torch = _torch()
    nb = len(beams)
    if nb * config.candidates_per_beam > TS_BEAM_MAX_CANDIDATES:
        raise ValueError(f"{nb} beams x {config.candidates_per_beam} candidates exceed "
                         f"{TS_BEAM_MAX_CANDIDATES} per problem on this engine")
    arr = (TsBeam * TS_BEAM_MAX_CANDIDATES)()
    for i, b in enumerate(beams):
        if len(b.index_path) >= _abi.TS_MAX_DEPTH:
            raise ValueError(f"context {tuple(b.index_path)} is terminal")
        arr[i].len = len(b.index_path)
        arr[i].is_terminal = int(b.is_terminal)
        arr[i].score = b.score
        for d, (ref, r) in enumerate(zip(b.index_path, b.rewards)):
            arr[i].path[d] = int(ref)
            arr[i].rewards[d] = float(r)
    table = _table([problem])
    dev = lambda raw: torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()  # noqa: E731
    dprob, dbeams = dev(bytes(table)), dev(bytes(arr))
    dcount = torch.tensor([nb], dtype=torch.int32, device="cuda")
    dcand = torch.zeros(ctypes.sizeof(TsBeamCandidate) * TS_BEAM_MAX_CANDIDATES, dtype=torch.uint8, device="cuda")
    dstat = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib = load_library()
    cfg = to_c(config, scoring)
    rc = lib.ts_beam_expand(ctypes.byref(cfg), ctypes.c_void_p(dprob.data_ptr()), 1,
                            ctypes.c_void_p(dbeams.data_ptr()), ctypes.c_void_p(dcount.data_ptr()),
                            ctypes.c_void_p(dcand.data_ptr()), ctypes.c_void_p(dstat.data_ptr()),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    raise_for_status(rc, "ts_beam_expand")
    if int(dstat.item()) != 0:
        raise ValueError("context is terminal for the problem")
    cands = (TsBeamCandidate * TS_BEAM_MAX_CANDIDATES).from_buffer_copy(dcand.cpu().numpy().tobytes())
    return list(cands[: nb * config.candidates_per_beam])


def _candidate(beams, c) -> BeamCandidate:
    parent = beams[c.beam]
    return BeamCandidate(Beam(tuple(parent.index_path) + (c.step_ref,), tuple(parent.rewards) + (c.prm_reward,),
                              c.score, bool(c.is_terminal)), c.order, c.token_count)


def expand_beams(beams: Sequence[Beam], config: BeamConfig, scoring: ScoringConfig, problem) -> list:
    """``candidates_per_beam`` sampled extensions of every beam, beam-major (beam.py:76-104)."""
    if not beams:
        return []
    return [_candidate(beams, c) for c in _expand_raw(beams, config, scoring, problem)]


def prune_candidates(candidates: Sequence[BeamCandidate], beam_width: int) -> tuple:
    """Terminal candidates retire; the top ``beam_width`` of the rest by
    (-score, order) survive (beam.py:107-117).  Ranks computed on the device."""
    from ._abi import TsBeamCandidate

    torch = _torch()
    n = len(candidates)
    finished = [c.beam for c in candidates if c.beam.is_terminal]
    if n == 0:
        return [], finished
    if n > 1024:
        raise ValueError("prune_candidates: at most 1024 candidates per call on this engine")
    arr = (TsBeamCandidate * n)()
    for i, c in enumerate(candidates):
        arr[i].order = c.order
        arr[i].score = c.beam.score
        arr[i].is_terminal = int(c.beam.is_terminal)
    dev = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).cuda()
    rc = load_library().ts_beam_prune(ctypes.c_void_p(dev.data_ptr()), n, max(1, beam_width),
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    raise_for_status(rc, "ts_beam_prune")
    out = (TsBeamCandidate * n).from_buffer_copy(dev.cpu().numpy().tobytes())
    slots = sorted((c.rank, i) for i, c in enumerate(out) if c.rank >= 0)
    survivors = [candidates[i].beam for _, i in slots] if beam_width > 0 else []
    return survivors, finished


def beam_step(beams: Sequence[Beam], config: BeamConfig, scoring: ScoringConfig, problem) -> BeamStep:
    """One expansion-pruning round (beam.py:120-131): one kernel for both."""
    if not 1 <= len(beams) <= config.beam_width:
        raise ValueError(f"beam count {len(beams)} out of [1, {config.beam_width}]")
    raw = _expand_raw(beams, config, scoring, problem)
    cands = [_candidate(beams, c) for c in raw]
    slots = sorted((c.rank, i) for i, c in enumerate(raw) if c.rank >= 0)
    return BeamStep(survivors=[cands[i].beam for _, i in slots],
                    finished=[cands[i].beam for i, c in enumerate(raw) if c.is_terminal],
                    tokens_generated=sum(c.token_count for c in raw))
