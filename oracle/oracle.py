"""ctypes binding of the CPU ORACLE (oracle/ts_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the timed
CPU baseline — never on the product path.  Parity of the oracle with the
reference is pinned by tests/test_oracle.py against tests/golden/.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from paper_2604_00510_b200._abi import TsConfig, TsOutcome, TsProblem, TsRunStats

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "lib", "libts_oracle.so")


class OrCandidate(ctypes.Structure):
    _fields_ = [
        ("step_ref", ctypes.c_int32),
        ("token_count", ctypes.c_int32),
        ("prior", ctypes.c_double),
        ("prm_reward", ctypes.c_double),
        ("is_terminal", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "CC=gcc"], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        u64p = P(ctypes.c_uint64)
        i32 = ctypes.c_int32
        L.or_mix.restype = ctypes.c_uint64
        L.or_mix.argtypes = [u64p, i32]
        L.or_uniform.restype = ctypes.c_double
        L.or_uniform.argtypes = [u64p, i32]
        L.or_uniform_in.restype = ctypes.c_double
        L.or_uniform_in.argtypes = [ctypes.c_double, ctypes.c_double, u64p, i32]
        L.or_randint_in.restype = ctypes.c_int64
        L.or_randint_in.argtypes = [ctypes.c_int64, ctypes.c_int64, u64p, i32]
        L.or_exponential.restype = ctypes.c_double
        L.or_exponential.argtypes = [ctypes.c_double, u64p, i32]
        L.or_fill_problem.restype = i32
        L.or_fill_problem.argtypes = [ctypes.c_uint64, i32, i32, i32, i32, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, i32, i32, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, P(TsProblem)]
        L.or_generate_steps.restype = i32
        L.or_generate_steps.argtypes = [P(TsProblem), P(i32), i32, i32, P(OrCandidate)]
        L.or_compute_targets.restype = i32
        L.or_compute_targets.argtypes = [P(TsConfig), i32, i32, P(i32), P(i32), P(ctypes.c_double), P(i32)]
        L.or_compute_targets_general.restype = i32
        L.or_compute_targets_general.argtypes = [P(TsConfig), ctypes.c_double, i32] + [ctypes.c_void_p] * 5
        L.or_forest_policy.restype = None
        L.or_forest_policy.argtypes = [P(TsConfig), i32] + [ctypes.c_void_p] * 12
        L.or_beam_search.restype = i32
        L.or_beam_search.argtypes = [P(TsProblem), ctypes.c_void_p, ctypes.c_void_p]
        L.or_run_waves.restype = ctypes.c_void_p
        L.or_run_waves.argtypes = [P(TsProblem), i32, P(TsConfig), i32, i32, P(i32), ctypes.c_int64,
                                   P(ctypes.c_int64)]
        L.or_run_waves_cost.restype = ctypes.c_void_p
        L.or_run_waves_cost.argtypes = [P(TsProblem), i32, P(TsConfig), i32, i32, ctypes.c_double, i32,
                                        ctypes.c_double]
        L.or_run_sim_times.restype = None
        L.or_run_sim_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.or_run_steps.restype = i32
        L.or_run_steps.argtypes = [ctypes.c_void_p]
        L.or_run_outcomes.restype = None
        L.or_run_outcomes.argtypes = [ctypes.c_void_p, P(TsOutcome)]
        L.or_run_stats.restype = None
        L.or_run_stats.argtypes = [ctypes.c_void_p, P(TsRunStats)]
        L.or_tree_size.restype = i32
        L.or_tree_size.argtypes = [ctypes.c_void_p, i32]
        L.or_tree_dump.restype = None
        L.or_tree_dump.argtypes = [ctypes.c_void_p, i32] + [ctypes.c_void_p] * 9
        L.or_run_latencies.restype = None
        L.or_run_latencies.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.or_run_free.restype = None
        L.or_run_free.argtypes = [ctypes.c_void_p]
        L.or_run_tree_search.restype = i32
        L.or_run_tree_search.argtypes = [P(TsProblem), P(TsConfig), P(TsOutcome)]
        for f in ("or_sizeof_problem", "or_sizeof_config", "or_sizeof_outcome"):
            getattr(L, f).restype = i32
        assert L.or_sizeof_problem() == ctypes.sizeof(TsProblem)
        assert L.or_sizeof_config() == ctypes.sizeof(TsConfig)
        assert L.or_sizeof_outcome() == ctypes.sizeof(TsOutcome)
        _lib = L
    return _lib


def _keys(keys):
    arr = (ctypes.c_uint64 * max(1, len(keys)))(*[int(k) & 0xFFFFFFFFFFFFFFFF for k in keys])
    return arr, len(keys)


def mix(keys):
    a, n = _keys(keys)
    return lib().or_mix(a, n)


def uniform(keys):
    a, n = _keys(keys)
    return lib().or_uniform(a, n)


def uniform_in(lo, hi, keys):
    a, n = _keys(keys)
    return lib().or_uniform_in(lo, hi, a, n)


def randint_in(lo, hi, keys):
    a, n = _keys(keys)
    return lib().or_randint_in(lo, hi, a, n)


def exponential(rate, keys):
    a, n = _keys(keys)
    return lib().or_exponential(rate, a, n)


def fill_problem(seed, solvable, depth_range, branching, profile) -> TsProblem:
    p = TsProblem()
    sh = profile["shared_range"]
    rc = lib().or_fill_problem(
        seed, int(solvable), depth_range[0], depth_range[1], branching, profile["golden_range"][0],
        profile["golden_range"][1], profile["off_path_range"][0], profile["off_path_range"][1],
        profile["hidden_until_depth"], 1 if sh else 0, sh[0] if sh else 0.0, sh[1] if sh else 0.0,
        profile["target_aggregate"], ctypes.byref(p))
    if rc:
        raise ValueError("fill_problem failed")
    return p


def generate_steps(problem: TsProblem, path, width):
    buf = (OrCandidate * max(1, width))()
    parr = (ctypes.c_int32 * max(1, len(path)))(*path)
    rc = lib().or_generate_steps(ctypes.byref(problem), parr, len(path), width, buf)
    if rc:
        raise ValueError(f"context {tuple(path)} is terminal")
    return [(c.step_ref, c.token_count, c.prior, c.prm_reward, bool(c.is_terminal)) for c in buf[:width]]


def compute_targets(cfg: TsConfig, now_step, arrival, completed, best):
    n = len(arrival)
    A = (ctypes.c_int32 * n)(*arrival)
    C = (ctypes.c_int32 * n)(*completed)
    B = (ctypes.c_double * n)(*best)
    T = (ctypes.c_int32 * n)()
    rc = lib().or_compute_targets(ctypes.byref(cfg), now_step, n, A, C, B, T)
    if rc:
        raise ValueError("run queue holds no running jobs")
    return list(T)


def compute_targets_general(cfg: TsConfig, now, arrival, completed, best, ids):
    """compute_targets on a general run queue; raises ValueError like the reference."""
    import numpy as np

    n = len(arrival)
    A = np.ascontiguousarray(arrival, np.float64)
    C = np.ascontiguousarray(completed, np.int32)
    B = np.ascontiguousarray(best, np.float64)
    I = np.ascontiguousarray(ids, np.int64)  # noqa: E741
    T = np.zeros(max(1, n), np.int32)
    rc = lib().or_compute_targets_general(ctypes.byref(cfg), float(now), n, A.ctypes.data, C.ctypes.data,
                                          B.ctypes.data, I.ctypes.data, T.ctypes.data)
    if rc < 0:
        raise ValueError(f"now={now} precedes arrival={A[-rc - 1]}")
    if rc:
        raise ValueError("run queue holds no running jobs")
    return T[:n].tolist()


def forest_policy(cfg: TsConfig, off, parent, reward, depth, flags, best, has_best, completed, budget, exhausted):
    """(kinds, ne) of every tree of a flat forest (see or_forest_policy)."""
    import numpy as np

    arrs = [np.ascontiguousarray(a, dt) for a, dt in
            ((off, np.int32), (parent, np.int32), (reward, np.float64), (depth, np.int32), (flags, np.uint8),
             (best, np.float64), (has_best, np.uint8), (completed, np.int32), (budget, np.int32),
             (exhausted, np.uint8))]
    nt = len(off) - 1
    kind = np.zeros(max(1, nt), np.int32)
    ne = np.zeros(max(1, nt), np.uint8)
    lib().or_forest_policy(ctypes.byref(cfg), nt, *[a.ctypes.data for a in arrs], kind.ctypes.data, ne.ctypes.data)
    return kind[:nt], ne[:nt]


def beam_search(problem: TsProblem, cfg, out=None):
    """run_beam_search of one problem; cfg is an _abi.TsBeamConfig."""
    from paper_2604_00510_b200._abi import TsBeamResult

    r = TsBeamResult() if out is None else out
    rc = lib().or_beam_search(ctypes.byref(problem), ctypes.addressof(cfg), ctypes.addressof(r))
    if rc:
        raise ValueError("beam search: bad arguments")
    return r


class OracleRun:
    """Result of or_run_waves; owns the C trees until closed."""

    def __init__(self, table, cfg: TsConfig, threads: int = 1, max_steps: int = 1 << 30, trace_cap: int = 0,
                 cost=None):
        """``cost``: (per_token_latency, engine_capacity, reward_latency) runs
        the wave clock of the cost model (or_run_waves_cost)."""
        self.n = len(table)
        self._trace = (ctypes.c_int32 * max(1, trace_cap))()
        tl = ctypes.c_int64(0)
        if cost is not None:
            pt, cap, rl = cost
            self._h = lib().or_run_waves_cost(table, self.n, ctypes.byref(cfg), threads, max_steps, float(pt),
                                              int(cap), float(rl))
        else:
            self._h = lib().or_run_waves(table, self.n, ctypes.byref(cfg), threads, max_steps,
                                         self._trace if trace_cap else None, trace_cap, ctypes.byref(tl))
        self.trace_len = tl.value
        self.steps = lib().or_run_steps(self._h)
        self.outcomes = (TsOutcome * max(1, self.n))()
        lib().or_run_outcomes(self._h, self.outcomes)
        st = TsRunStats()
        lib().or_run_stats(self._h, ctypes.byref(st))
        self.stats = st

    def targets_trace(self):
        return list(self._trace[: min(self.trace_len, len(self._trace))])

    def tree(self, i: int) -> dict:
        import numpy as np

        n = lib().or_tree_size(self._h, i)
        out = {
            "parent": np.zeros(n, np.int32), "reward": np.zeros(n, np.float64), "prior": np.zeros(n, np.float64),
            "N": np.zeros(n, np.int32), "O": np.zeros(n, np.int32), "W": np.zeros(n, np.float64),
            "terminal": np.zeros(n, np.uint8), "depth": np.zeros(n, np.int32), "step_ref": np.zeros(n, np.int32),
        }
        order = ["parent", "reward", "prior", "N", "O", "W", "terminal", "depth", "step_ref"]
        lib().or_tree_dump(self._h, i, *[out[k].ctypes.data_as(ctypes.c_void_p) for k in order])
        return out

    def sim_times(self):
        """(completion, arrival) on the wave clock of the cost model, per job."""
        import numpy as np

        c = np.zeros(max(1, self.n), np.float64)
        a = np.zeros(max(1, self.n), np.float64)
        lib().or_run_sim_times(self._h, c.ctypes.data_as(ctypes.c_void_p), a.ctypes.data_as(ctypes.c_void_p))
        return c[: self.n], a[: self.n]

    def latencies_s(self):
        import numpy as np

        out = np.zeros(max(1, self.n), np.float64)
        lib().or_run_latencies(self._h, out.ctypes.data_as(ctypes.c_void_p))
        return out[: self.n]

    def close(self):
        if self._h:
            lib().or_run_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_tree_search(problem: TsProblem, cfg: TsConfig) -> TsOutcome:
    o = TsOutcome()
    rc = lib().or_run_tree_search(ctypes.byref(problem), ctypes.byref(cfg), ctypes.byref(o))
    if rc:
        raise RuntimeError(f"oracle run_tree_search status {rc}")
    return o
