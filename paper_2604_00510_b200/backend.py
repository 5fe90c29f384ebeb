"""Synthetic problem specs and the device problem table.

The reference generates every step on demand from ``(seed, path)``
(backend.py:230-269); here the per-request constants are computed ONCE on the
host and uploaded as a ``ts_problem`` table: seed, branching, base depth
(backend.py:135-137), golden path (140-141), the LIFTED golden rewards
(golden_step_rewards, 201-215 — uses ``pow`` so it stays on the host) and the
reward ranges.  Everything per-step (priors, rewards, tokens, terminal flags)
is replayed on the device from the same keyed splitmix64 draws.

Public names mirror the reference (Difficulty, RewardProfile,
SyntheticProblemSpec, default_profile, make_problem, make_workload,
golden_step_rewards) so a caller can switch imports; reference spec objects
are also accepted by :func:`problem_table` (duck-typed).
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import keyed
from ._abi import TS_MAX_DEPTH, TsProblem

# key tags of the reference's stateless rng (backend.py:49-57, simulator.py:55)
TAG_REWARD, TAG_PRIOR, TAG_TOKENS, TAG_DEPTH, TAG_GOLD, TAG_EXTEND, TAG_SHUFFLE, TAG_PROBLEM_SEED = 1, 2, 3, 4, 5, 6, 7, 8
TAG_ARRIVAL = 21
TOKENS_PER_STEP = (40, 120)


class Difficulty(enum.Enum):
    EASY = "easy"
    HARD_SOLVABLE = "hard_solvable"
    UNSOLVABLE = "unsolvable"


@dataclass(frozen=True)
class RewardProfile:
    """Per-step reward distribution of one difficulty class (backend.py:79-93)."""

    golden_range: tuple[float, float]
    off_path_range: tuple[float, float]
    hidden_until_depth: int = 0
    shared_range: Optional[tuple[float, float]] = None
    target_aggregate: float = 0.55


def default_profile(difficulty: Difficulty, accept_threshold: float = 0.3) -> RewardProfile:
    """The reference's three class profiles (backend.py:96-110)."""
    if difficulty is Difficulty.EASY:
        return RewardProfile((0.90, 0.99), (0.30, 0.70))
    if difficulty is Difficulty.HARD_SOLVABLE:
        return RewardProfile((0.75, 0.90), (0.20, 0.60), 2, (0.70, 0.95))
    return RewardProfile((0.0, 0.0), (0.05, accept_threshold - 0.02), target_aggregate=0.0)


def stagnation_profile() -> RewardProfile:
    """Config-4 "heavy-tailed stagnation" profile (BASELINE.json configs[3]).

    Not in the reference; defined once here (and identically in
    tests/golden/make_golden.py) and pinned by oracle goldens: off-path rewards
    straddle the acceptance threshold, the golden branch hides among shared
    rewards down to depth 6.
    """
    return RewardProfile((0.93, 0.99), (0.22, 0.75), 6, (0.80, 0.97), 0.55)


@dataclass(frozen=True)
class SyntheticProblemSpec:
    """One synthetic reasoning request (backend.py:113-132)."""

    problem_id: str
    seed: int
    difficulty: Difficulty
    depth_range: tuple[int, int]
    branching: int
    reward_profile: RewardProfile
    golden_path: Optional[tuple[int, ...]] = None
    _base: int = field(default=-1, repr=False, compare=False)

    @property
    def base_depth(self) -> int:
        if self._base >= 0:
            return self._base
        lo, hi = self.depth_range
        return lo + keyed.mix(self.seed, TAG_DEPTH) % (hi - lo + 1)

    @property
    def max_depth(self) -> int:
        return self.base_depth + 1


def _base_depths(seeds: np.ndarray, lo: int, hi: int) -> np.ndarray:
    h = keyed.fold_columns(seeds, np.uint64(TAG_DEPTH))
    return (lo + (h % np.uint64(hi - lo + 1))).astype(np.int64)


def _golden_paths(seeds: np.ndarray, depth: int, branching: int) -> np.ndarray:
    """randint_in(0, b-1, seed, TAG_GOLD, d) for d < depth, all seeds at once."""
    if depth == 0:
        return np.zeros((len(seeds), 0), dtype=np.int64)
    d = np.arange(depth, dtype=np.uint64)[None, :]
    h = keyed.fold_columns(seeds[:, None], np.uint64(TAG_GOLD), d)
    return (h % np.uint64(branching)).astype(np.int64)


def make_problem(
    problem_id: str,
    seed: int,
    difficulty: Difficulty,
    depth_range: tuple[int, int],
    branching: int = 2,
    profile: Optional[RewardProfile] = None,
) -> SyntheticProblemSpec:
    """backend.py:144-166."""
    return _make_many([problem_id], np.array([seed], dtype=np.uint64), difficulty, depth_range,
                      branching, profile or default_profile(difficulty))[0]


def _make_many(ids, seeds, difficulty, depth_range, branching, profile):
    lo, hi = depth_range
    bases = _base_depths(seeds, lo, hi)
    out = []
    gold_by_base = {}
    if difficulty is not Difficulty.UNSOLVABLE:
        for b in np.unique(bases):
            sel = np.nonzero(bases == b)[0]
            gold_by_base[int(b)] = (sel, _golden_paths(seeds[sel], int(b), branching))
    golden = [None] * len(ids)
    for b, (sel, paths) in gold_by_base.items():
        for k, i in enumerate(sel.tolist()):
            golden[i] = tuple(int(x) for x in paths[k])
    for i, pid in enumerate(ids):
        out.append(SyntheticProblemSpec(pid, int(seeds[i]), difficulty, tuple(depth_range), branching,
                                        profile, golden[i], int(bases[i])))
    return out


def _raw_golden_rewards(spec) -> list[float]:
    prof = spec.reward_profile
    g = spec.golden_path
    seed = np.uint64(spec.seed)
    out = []
    for d in range(1, len(g) + 1):
        if prof.shared_range is not None and d <= prof.hidden_until_depth:
            lo, hi = prof.shared_range
        else:
            lo, hi = prof.golden_range
        h = keyed.fold_columns(seed, np.uint64(TAG_REWARD), np.uint64(d), *[np.uint64(x) for x in g[:d]])
        out.append(lo + (hi - lo) * float(keyed.to_unit(h)))
    return out


def golden_step_rewards(spec) -> tuple[float, ...]:
    """Golden-path rewards after the target-aggregate lift (backend.py:201-215):
    at most four rounds of ``r*lift*1.001`` capped at 0.99, with
    ``lift = (target/prod)**(1/depth)``, ``prod`` the left-to-right product."""
    if spec.golden_path is None:
        raise ValueError(f"{spec.problem_id} has no golden path")
    depth = len(spec.golden_path)
    rewards = _raw_golden_rewards(spec)
    target = spec.reward_profile.target_aggregate
    for _ in range(4):
        prod = 1.0
        for r in rewards:
            prod *= r
        if prod >= target:
            break
        lift = (target / prod) ** (1.0 / depth)
        rewards = [min(0.99, r * lift * 1.001) for r in rewards]
    return tuple(rewards)


def make_workload(
    count: int,
    mixture: tuple[float, float, float],
    seed: int,
    branching: int = 2,
    depth_ranges: Optional[dict] = None,
    accept_threshold: float = 0.3,
) -> list[SyntheticProblemSpec]:
    """Deterministic mixed-difficulty workload (backend.py:314-356), built with
    vectorised folds: problem seeds mix(seed, 8, i), difficulty order shuffled
    with tag 7, counts rounded with the remainder on the largest fraction."""
    if count < 1:
        raise ValueError("count must be >= 1")
    if abs(sum(mixture) - 1.0) > 1e-9:
        raise ValueError(f"mixture fractions must sum to 1, got {sum(mixture)}")
    if depth_ranges is None:
        depth_ranges = {Difficulty.EASY: (2, 4), Difficulty.HARD_SOLVABLE: (3, 5), Difficulty.UNSOLVABLE: (2, 4)}
    order = [Difficulty.EASY, Difficulty.HARD_SOLVABLE, Difficulty.UNSOLVABLE]
    counts = [round(f * count) for f in mixture]
    counts[max(range(3), key=lambda i: mixture[i])] += count - sum(counts)
    labels: list[Difficulty] = []
    for d, n in zip(order, counts):
        labels.extend([d] * n)
    labels = keyed.keyed_permutation(labels, seed, TAG_SHUFFLE)
    seeds = keyed.fold_columns(np.uint64(seed & 0xFFFFFFFFFFFFFFFF), np.uint64(TAG_PROBLEM_SEED),
                               np.arange(count, dtype=np.uint64))
    specs: list[Optional[SyntheticProblemSpec]] = [None] * count
    for d in order:
        idx = [i for i, lab in enumerate(labels) if lab is d]
        if not idx:
            continue
        made = _make_many([f"p{i:04d}" for i in idx], seeds[idx], d, tuple(depth_ranges[d]), branching,
                          default_profile(d, accept_threshold))
        for i, s in zip(idx, made):
            specs[i] = s
    return specs  # type: ignore[return-value]


def serving_arrival_steps(count: int, rate: float, seed: int, steps_per_unit: float) -> list[int]:
    """Config-5 arrivals: the reference's Poisson generator (cumulative
    ``exponential(rate, seed, 21, i)``, simulator.py:193-200) quantised to
    waves: ``int(t_i * steps_per_unit)``."""
    t = 0.0
    out = []
    for i in range(count):
        t += keyed.exponential_draw(rate, seed, TAG_ARRIVAL, i)
        out.append(int(t * steps_per_unit))
    return out


def problem_table(specs: Sequence, arrival_steps: Optional[Sequence[int]] = None) -> ctypes.Array:
    """Pack specs (ours or the reference's, duck-typed) into a ts_problem array."""
    n = len(specs)
    arr = (TsProblem * n)()
    for i, s in enumerate(specs):
        p = arr[i]
        prof = s.reward_profile
        p.seed = int(s.seed) & 0xFFFFFFFFFFFFFFFF
        p.branching = int(s.branching)
        p.base_depth = int(s.base_depth)
        p.hidden_until_depth = int(prof.hidden_until_depth)
        p.has_shared = 1 if prof.shared_range is not None else 0
        p.arrival_step = int(arrival_steps[i]) if arrival_steps is not None else 0
        p.off_lo, p.off_hi = float(prof.off_path_range[0]), float(prof.off_path_range[1])
        if prof.shared_range is not None:
            p.shared_lo, p.shared_hi = float(prof.shared_range[0]), float(prof.shared_range[1])
        if s.golden_path is None:
            p.golden_len = -1
        else:
            g = tuple(s.golden_path)
            if len(g) > TS_MAX_DEPTH:
                raise ValueError(f"golden path deeper than {TS_MAX_DEPTH}")
            p.golden_len = len(g)
            rewards = golden_step_rewards(s)
            for d, (step, r) in enumerate(zip(g, rewards)):
                p.golden_path[d] = int(step)
                p.golden_rewards[d] = float(r)
    return arr


# ---- generate_steps and the cost model (backend.py:62-70, 230-311) -------------------

@dataclass(frozen=True)
class StepCandidate:
    """One generated reasoning step with its verifier reward (backend.py:62-70)."""

    step_ref: int
    token_count: int
    prior: float
    prm_reward: float
    is_terminal: bool


def generate_steps_many(problems: Sequence, context_paths: Sequence[Sequence[int]], width: int) -> list:
    """generate_steps for many (problem, context path) pairs in one kernel
    (csrc/steps.cu).  Returns one candidate list per pair; raises ValueError
    (like the reference) if any context is terminal or too deep."""
    import torch

    from ._abi import TS_MAX_WIDTH, TsStepCandidate, load_library, raise_for_status

    if width < 1:
        raise ValueError("width must be >= 1")
    if width > TS_MAX_WIDTH:
        raise ValueError(f"width above {TS_MAX_WIDTH} is not supported by this engine")
    if not torch.cuda.is_available():
        raise RuntimeError("generate_steps runs on the CUDA device; no CUDA device is available")
    n = len(problems)
    if n == 0:
        return []
    paths = np.zeros((n, TS_MAX_DEPTH), np.uint8)
    lens = np.zeros(n, np.int32)
    for i, cp in enumerate(context_paths):
        cp = tuple(cp)
        if len(cp) >= TS_MAX_DEPTH:
            raise ValueError(f"context {cp} is terminal")
        paths[i, : len(cp)] = cp
        lens[i] = len(cp)
    if isinstance(problems, ctypes.Array):
        table = problems
    elif isinstance(problems[0], TsProblem):  # ts_problem rows already
        table = (TsProblem * n)(*problems)
    else:
        table = problem_table(list(problems))
    dev = torch.device("cuda")
    dprob = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).to(dev)
    dpath = torch.from_numpy(paths).to(dev)
    dlen = torch.from_numpy(lens).to(dev)
    dout = torch.zeros(n * width * ctypes.sizeof(TsStepCandidate), dtype=torch.uint8, device=dev)
    dstat = torch.zeros(n, dtype=torch.int32, device=dev)
    rc = load_library().ts_generate_steps(ctypes.c_void_p(dprob.data_ptr()), n, ctypes.c_void_p(dpath.data_ptr()),
                                          ctypes.c_void_p(dlen.data_ptr()), width, ctypes.c_void_p(dout.data_ptr()),
                                          ctypes.c_void_p(dstat.data_ptr()),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    raise_for_status(rc, "ts_generate_steps")
    bad = dstat.cpu().numpy()
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise ValueError(f"context {tuple(context_paths[i])} is terminal")
    raw = (TsStepCandidate * (n * width)).from_buffer_copy(dout.cpu().numpy().tobytes())
    return [[StepCandidate(c.step_ref, c.token_count, c.prior, c.prm_reward, bool(c.is_terminal))
             for c in raw[i * width:(i + 1) * width]] for i in range(n)]


def generate_steps(problem, context_path: Sequence[int], width: int) -> list:
    """``width`` child steps below ``context_path`` (backend.py:230-269), on the device."""
    return generate_steps_many([problem], [tuple(context_path)], width)[0]


@dataclass(frozen=True)
class CostModel:
    """Token-latency model with a concurrency knee (backend.py:287-300)."""

    per_token_latency: float = 0.002
    engine_capacity: int = 32
    reward_latency: float = 0.01

    def __post_init__(self) -> None:
        if not (self.per_token_latency > 0 and self.engine_capacity >= 1 and self.reward_latency >= 0):
            raise ValueError("cost model parameters must be positive")


def service_time(token_count: int, model: CostModel, inflight_load: int) -> float:
    """Generation latency of one request under load (backend.py:303-311): the
    per-token latency stretched by the overload ratio past engine_capacity."""
    if token_count < 1:
        raise ValueError("token_count must be >= 1")
    if inflight_load < 0:
        raise ValueError("inflight_load must be >= 0")
    stretch = max(1.0, inflight_load / model.engine_capacity)
    return token_count * model.per_token_latency * stretch


# ---- workload replay files (backend.py:359-410) ----------------------------------------

def _spec_doc(spec) -> dict:
    prof = spec.reward_profile
    shared = prof.shared_range
    return {
        "branching": spec.branching,
        "depth_range": [int(x) for x in spec.depth_range],
        "difficulty": spec.difficulty.value,
        "golden_path": [int(x) for x in spec.golden_path] if spec.golden_path else None,
        "problem_id": spec.problem_id,
        "reward_profile": {
            "golden_range": [float(x) for x in prof.golden_range],
            "hidden_until_depth": prof.hidden_until_depth,
            "off_path_range": [float(x) for x in prof.off_path_range],
            "shared_range": [float(x) for x in shared] if shared else None,
            "target_aggregate": prof.target_aggregate,
        },
        "seed": int(spec.seed),
    }


def workload_to_json(specs: Sequence) -> str:
    """The reference's workload replay format: sorted keys, indent 2 (byte-identical)."""
    import json

    return json.dumps([_spec_doc(s) for s in specs], indent=2, sort_keys=True)


def workload_from_json(text: str) -> list:
    """Specs back from :func:`workload_to_json` (or the reference's file)."""
    import json

    out = []
    for doc in json.loads(text):
        p = doc["reward_profile"]
        prof = RewardProfile(tuple(p["golden_range"]), tuple(p["off_path_range"]), p["hidden_until_depth"],
                             tuple(p["shared_range"]) if p["shared_range"] else None, p["target_aggregate"])
        golden = tuple(doc["golden_path"]) if doc["golden_path"] else None
        out.append(SyntheticProblemSpec(doc["problem_id"], doc["seed"], Difficulty(doc["difficulty"]),
                                        tuple(doc["depth_range"]), doc["branching"], prof, golden))
    return out
