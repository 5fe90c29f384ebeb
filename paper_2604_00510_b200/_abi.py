"""ctypes mirror of include/treeserve_b200.h and the status → exception map.

The shared library is built in-tree by ``__graft_entry__.build()`` into
``paper_2604_00510_b200/lib/libtreeserve_b200.so``.  There is no fallback:
if the library is missing, :func:`load_library` raises.
"""

from __future__ import annotations

import ctypes
import os

TS_MAX_DEPTH = 32
TS_MAX_WIDTH = 32
TS_ABI_VERSION = 6

TS_OK = 0
TS_INVALID_ARGUMENT = 1
TS_TREE_STRUCTURE = 2
TS_EXHAUSTED = 3
TS_ACCOUNTING = 4
TS_UNSUPPORTED_SCHEME = 5
TS_POOL_OVERFLOW = 6
TS_CUDA = 7

EXIT_NONE, EXIT_POSITIVE, EXIT_NEGATIVE, EXIT_BUDGET = 0, 1, 2, 3

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.path.join(LIB_DIR, "libtreeserve_b200.so")


class TsProblem(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("branching", ctypes.c_int32),
        ("base_depth", ctypes.c_int32),
        ("golden_len", ctypes.c_int32),
        ("hidden_until_depth", ctypes.c_int32),
        ("has_shared", ctypes.c_int32),
        ("arrival_step", ctypes.c_int32),
        ("off_lo", ctypes.c_double),
        ("off_hi", ctypes.c_double),
        ("shared_lo", ctypes.c_double),
        ("shared_hi", ctypes.c_double),
        ("golden_path", ctypes.c_uint8 * TS_MAX_DEPTH),
        ("golden_rewards", ctypes.c_double * TS_MAX_DEPTH),
    ]


class TsConfig(ctypes.Structure):
    _fields_ = [
        ("scheme", ctypes.c_int32),
        ("futility_bound", ctypes.c_int32),
        ("strict_negative_exit", ctypes.c_int32),
        ("positive_exit", ctypes.c_int32),
        ("negative_exit", ctypes.c_int32),
        ("rollout_budget", ctypes.c_int32),
        ("depth_cap", ctypes.c_int32),
        ("expand_width", ctypes.c_int32),
        ("max_concurrency", ctypes.c_int32),
        ("obs_threshold", ctypes.c_int32),
        ("boosting_enabled", ctypes.c_int32),
        ("_pad0", ctypes.c_int32),
        ("accept_threshold", ctypes.c_double),
        ("positive_exit_threshold", ctypes.c_double),
        ("first_step_threshold", ctypes.c_double),
        ("c_puct", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("proximity", ctypes.c_double),
    ]


class TsOutcome(ctypes.Structure):
    _fields_ = [
        ("exit_kind", ctypes.c_int32),
        ("rollouts_completed", ctypes.c_int32),
        ("tokens_generated", ctypes.c_int64),
        ("best_score", ctypes.c_double),
        ("best_len", ctypes.c_int32),
        ("solved", ctypes.c_int32),
        ("exit_step", ctypes.c_int32),
        ("admit_step", ctypes.c_int32),
        ("launched", ctypes.c_int32),
        ("cancelled", ctypes.c_int32),
        ("nodes", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("best_path", ctypes.c_uint8 * TS_MAX_DEPTH),
    ]


class TsSchedRecord(ctypes.Structure):
    _fields_ = [("score", ctypes.c_double), ("flags", ctypes.c_uint32), ("_pad", ctypes.c_uint32)]


class TsRunStats(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int32),
        ("finished", ctypes.c_int32),
        ("rollouts", ctypes.c_int64),
        ("launched", ctypes.c_int64),
        ("nodes", ctypes.c_int64),
        ("tokens", ctypes.c_int64),
        ("children_scored", ctypes.c_int64),
        ("select_levels", ctypes.c_int64),
        ("path_nodes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("wave_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class TsInvariants(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "waves", "capacity_violations", "gate_violations", "inflight_nodes", "conservation_violations",
        "root_mismatches", "max_wave_launched", "max_running")]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class TsTraceRow(ctypes.Structure):
    """ts_trace_row: one "allocation" record of a scheduler pass (simulator.py:314-330)."""
    _fields_ = [("step", ctypes.c_int32), ("job", ctypes.c_int32), ("target", ctypes.c_int32),
                ("active", ctypes.c_int32), ("score", ctypes.c_double)]


# Every symbol include/treeserve_b200.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "ts_engine_create", "ts_engine_destroy", "ts_last_error", "ts_abi_version",
    "ts_load_problems", "ts_step_counts", "ts_step_admit", "ts_step_records", "ts_step_targets",
    "ts_step_set_targets", "ts_read_jobs", "ts_step_wave", "ts_run", "ts_read_outcomes", "ts_read_stats", "ts_read_targets",
    "ts_read_step_times", "ts_read_latencies", "ts_run_batch_host", "ts_tree_size", "ts_dump_tree", "ts_fill_problem",
    "ts_policy_last_error", "ts_parallelism_scores", "ts_compute_targets", "ts_exit_policy",
    "ts_beam_search", "ts_beam_search_host", "ts_beam_expand", "ts_beam_prune",
    "ts_generate_steps", "ts_engine_set_checks", "ts_read_invariants", "ts_engine_set_trace", "ts_read_trace",
    "ts_reconcile", "ts_engine_set_cost_model", "ts_read_sim_times",
    "ts_xchg_bytes", "ts_xchg_create", "ts_xchg_connect", "ts_run_sharded", "ts_read_px_times",
)
TS_MAX_PEERS = 8
TS_IPC_HANDLE_BYTES = 64


class TsSchedParams(ctypes.Structure):
    _fields_ = [
        ("max_concurrency", ctypes.c_int64),
        ("beta", ctypes.c_double),
        ("proximity", ctypes.c_double),
        ("obs_threshold", ctypes.c_int32),
        ("boosting_enabled", ctypes.c_int32),
        ("positive_exit_threshold", ctypes.c_double),
    ]


class TsTargetsInfo(ctypes.Structure):
    _fields_ = [
        ("total_score", ctypes.c_double),
        ("ungated", ctypes.c_int64),
        ("first_bad", ctypes.c_int32),
        ("sum_fallback", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


TS_NODE_TERMINAL = 1
TS_NODE_HAS_CHILDREN = 2


class TsForest(ctypes.Structure):
    _fields_ = [("n_trees", ctypes.c_int32), ("n_nodes", ctypes.c_int32)] + [
        (name, ctypes.c_void_p)
        for name in ("offsets", "tree_of", "parent", "reward", "depth", "flags", "best_score", "has_best",
                     "completed", "budget", "exhausted")
    ]


TS_BEAM_MAX_CANDIDATES = 32


class TsBeamConfig(ctypes.Structure):
    _fields_ = [
        ("beam_width", ctypes.c_int32),
        ("candidates_per_beam", ctypes.c_int32),
        ("max_depth", ctypes.c_int32),
        ("positive_exit_enabled", ctypes.c_int32),
        ("scheme", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("positive_exit_threshold", ctypes.c_double),
    ]


class TsBeamResult(ctypes.Structure):
    _fields_ = [
        ("complete", ctypes.c_int32),
        ("has_best", ctypes.c_int32),
        ("is_terminal", ctypes.c_int32),
        ("best_len", ctypes.c_int32),
        ("steps", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("tokens_generated", ctypes.c_int64),
        ("best_score", ctypes.c_double),
        ("best_path", ctypes.c_uint8 * TS_MAX_DEPTH),
        ("best_rewards", ctypes.c_double * TS_MAX_DEPTH),
    ]


class TsBeam(ctypes.Structure):
    _fields_ = [
        ("len", ctypes.c_int32),
        ("is_terminal", ctypes.c_int32),
        ("score", ctypes.c_double),
        ("path", ctypes.c_uint8 * TS_MAX_DEPTH),
        ("rewards", ctypes.c_double * TS_MAX_DEPTH),
    ]


class TsBeamCandidate(ctypes.Structure):
    _fields_ = [
        ("beam", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("step_ref", ctypes.c_int32),
        ("token_count", ctypes.c_int32),
        ("prm_reward", ctypes.c_double),
        ("score", ctypes.c_double),
        ("is_terminal", ctypes.c_int32),
        ("rank", ctypes.c_int32),
    ]


class TsStepCandidate(ctypes.Structure):
    _fields_ = [
        ("step_ref", ctypes.c_int32),
        ("token_count", ctypes.c_int32),
        ("prior", ctypes.c_double),
        ("prm_reward", ctypes.c_double),
        ("is_terminal", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
    ]


_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load the in-tree CUDA extension; raises if it has not been built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("TS_LIB_PATH") or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} is missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(p)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    i32 = ctypes.c_int32
    sig = {
        "ts_engine_create": (ctypes.c_int, [P(TsConfig), i32, P(vp)]),
        "ts_engine_destroy": (ctypes.c_int, [vp]),
        "ts_last_error": (ctypes.c_char_p, [vp]),
        "ts_abi_version": (ctypes.c_int, []),
        "ts_load_problems": (ctypes.c_int, [vp, P(TsProblem), i32, i32, i32, vp]),
        "ts_step_counts": (ctypes.c_int, [vp, i32, vp, vp]),
        "ts_step_admit": (ctypes.c_int, [vp, i32, vp, i32, i32, vp]),
        "ts_step_records": (ctypes.c_int, [vp, i32, vp, vp]),
        "ts_step_targets": (ctypes.c_int, [vp, i32, vp, vp]),
        "ts_step_set_targets": (ctypes.c_int, [vp, i32, vp, vp]),
        "ts_read_jobs": (ctypes.c_int, [vp, vp, vp, vp, vp]),
        "ts_step_wave": (ctypes.c_int, [vp, i32, vp]),
        "ts_run": (ctypes.c_int, [vp, i32, P(TsRunStats), vp]),
        "ts_read_outcomes": (ctypes.c_int, [vp, P(TsOutcome), i32, vp]),
        "ts_read_stats": (ctypes.c_int, [vp, P(TsRunStats), vp]),
        "ts_read_targets": (ctypes.c_int, [vp, P(i32), i32, vp]),
        "ts_read_step_times": (ctypes.c_int, [vp, P(ctypes.c_uint64), i32, vp]),
        "ts_read_latencies": (ctypes.c_int, [vp, P(ctypes.c_uint64), i32, vp]),
        "ts_run_batch_host": (ctypes.c_int, [vp, P(TsProblem), i32, i32, P(TsOutcome), P(TsRunStats), vp]),
        "ts_tree_size": (ctypes.c_int, [vp, i32, P(i32)]),
        "ts_dump_tree": (ctypes.c_int, [vp, i32] + [vp] * 9),
        "ts_policy_last_error": (ctypes.c_char_p, []),
        "ts_parallelism_scores": (ctypes.c_int, [ctypes.c_double] * 4 + [vp, vp, i32, vp, P(i32), vp]),
        "ts_compute_targets": (ctypes.c_int, [P(TsSchedParams), ctypes.c_double, vp, vp, vp, vp, i32, vp,
                                              P(TsTargetsInfo), vp]),
        "ts_exit_policy": (ctypes.c_int, [P(TsConfig), P(TsForest), vp, vp, vp]),
        "ts_beam_search": (ctypes.c_int, [P(TsBeamConfig), vp, i32, vp, vp]),
        "ts_beam_search_host": (ctypes.c_int, [P(TsBeamConfig), vp, i32, vp, vp]),
        "ts_beam_expand": (ctypes.c_int, [P(TsBeamConfig), vp, i32, vp, vp, vp, vp, vp]),
        "ts_beam_prune": (ctypes.c_int, [vp, i32, i32, vp]),
        "ts_generate_steps": (ctypes.c_int, [vp, i32, vp, vp, i32, vp, vp, vp]),
        "ts_engine_set_checks": (ctypes.c_int, [vp, i32]),
        "ts_read_invariants": (ctypes.c_int, [vp, P(TsInvariants), vp]),
        "ts_engine_set_trace": (ctypes.c_int, [vp, ctypes.c_int64]),
        "ts_reconcile": (ctypes.c_int, [vp, vp, vp, vp, vp, i32, vp, vp, vp]),
        "ts_engine_set_cost_model": (ctypes.c_int, [vp, ctypes.c_double, i32, ctypes.c_double]),
        "ts_read_sim_times": (ctypes.c_int, [vp, vp, vp, i32, vp]),
        "ts_read_trace": (ctypes.c_int, [vp, vp, ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int64), vp]),
        "ts_xchg_bytes": (ctypes.c_int64, [i32]),
        "ts_xchg_create": (ctypes.c_int, [vp, i32, i32, P(vp), vp]),
        "ts_xchg_connect": (ctypes.c_int, [vp, vp, vp]),
        "ts_run_sharded": (ctypes.c_int, [vp, i32, i32, P(TsRunStats), vp]),
        "ts_read_px_times": (ctypes.c_int, [vp, P(ctypes.c_uint64), i32, vp]),
        "ts_fill_problem": (ctypes.c_int, [ctypes.c_uint64, i32, i32, i32, i32, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double, i32, i32,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double, P(TsProblem)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ts_abi_version() != TS_ABI_VERSION:
        raise ImportError("treeserve_b200 ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def raise_for_status(code: int, where: str, detail: str = "") -> None:
    """Map a ts_status to the reference's exception classes."""
    if code == TS_OK:
        return
    from .scoring import UnsupportedSchemeError
    from .tree import AccountingError, NoExpandableLeafError, TreeStructureError

    msg = f"{where}: {detail}" if detail else where
    if code == TS_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == TS_TREE_STRUCTURE:
        raise TreeStructureError(msg)
    if code == TS_EXHAUSTED:
        raise NoExpandableLeafError(msg)
    if code == TS_ACCOUNTING:
        raise AccountingError(msg)
    if code == TS_UNSUPPORTED_SCHEME:
        raise UnsupportedSchemeError(msg)
    if code == TS_POOL_OVERFLOW:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error in {msg}")
