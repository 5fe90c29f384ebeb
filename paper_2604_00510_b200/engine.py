"""Python handle on the CUDA engine (include/treeserve_b200.h through ctypes).

One :class:`Engine` owns one GPU's node pool and search table.  Everything
per step runs in the sm_100a kernels of ``csrc/engine.cu``; this class only
moves problem tables in and outcomes out.  There is no CPU fallback: without
the built library or a CUDA device the constructor raises.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _abi
from ._abi import TsConfig, TsInvariants, TsOutcome, TsProblem, TsRunStats, load_library, raise_for_status
from .config import SearchConfig


def _stream_handle(stream) -> int:
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return int(torch.cuda.current_stream().cuda_stream)
        except Exception:  # pragma: no cover - torch missing
            pass
        return 0
    if hasattr(stream, "cuda_stream"):
        return int(stream.cuda_stream)
    return int(stream)


class Engine:
    """One GPU's batch of concurrent searches (SearchTree + ProblemBackend +
    SchedulerState for every request, tree.py:120, backend.py:275, scheduler.py:96)."""

    def __init__(self, config: SearchConfig, device: int = 0, stream=None):
        self.lib = load_library()
        self.config = config
        self.device = device
        self._cfg = config.to_c() if isinstance(config, SearchConfig) else config
        self._h = ctypes.c_void_p()
        self._stream = stream
        rc = self.lib.ts_engine_create(ctypes.byref(self._cfg), device, ctypes.byref(self._h))
        if rc != _abi.TS_OK:
            msg = self.last_error()
            self.lib.ts_engine_destroy(self._h)
            self._h = ctypes.c_void_p()
            raise_for_status(rc, "ts_engine_create", msg)
        self.n = 0

    # ---- plumbing ---------------------------------------------------------
    @property
    def stream(self) -> int:
        return _stream_handle(self._stream)

    def last_error(self) -> str:
        e = self.lib.ts_last_error(self._h)
        return e.decode() if e else ""

    def _check(self, rc: int, where: str) -> None:
        if rc != _abi.TS_OK:
            raise_for_status(rc, where, self.last_error())

    def close(self) -> None:
        if self._h:
            self.lib.ts_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- batch API --------------------------------------------------------
    def load(self, table, global_offset: int = 0, n_global: Optional[int] = None) -> None:
        """Upload a ts_problem array and reset every tree to a bare root."""
        n = len(table)
        if not isinstance(table, ctypes.Array):
            arr = (TsProblem * n)()
            for i, p in enumerate(table):
                arr[i] = p
            table = arr
        self._table = table
        self.n = n
        self._check(self.lib.ts_load_problems(self._h, table, n, global_offset,
                                              n if n_global is None else n_global, self.stream),
                    "ts_load_problems")

    def run(self, max_steps: int = (1 << 31) - 1) -> TsRunStats:
        st = TsRunStats()
        self._check(self.lib.ts_run(self._h, max_steps, ctypes.byref(st), self.stream), "ts_run")
        return st

    def stats(self) -> TsRunStats:
        st = TsRunStats()
        self._check(self.lib.ts_read_stats(self._h, ctypes.byref(st), self.stream), "ts_read_stats")
        return st

    def set_checks(self, enable: bool = True) -> None:
        """Run the invariant kernels around every wave (ts_engine_set_checks)."""
        self._check(self.lib.ts_engine_set_checks(self._h, 1 if enable else 0), "ts_engine_set_checks")

    def invariants(self) -> dict:
        """Violation counts of the checked mode since the last load (ts_read_invariants)."""
        inv = TsInvariants()
        self._check(self.lib.ts_read_invariants(self._h, ctypes.byref(inv), self.stream), "ts_read_invariants")
        return inv.as_dict()

    def set_cost_model(self, cost=None) -> None:
        """Run the wave clock of a cost model (ts_engine_set_cost_model): a
        ``CostModel``-like object (per_token_latency, engine_capacity,
        reward_latency) or a 3-tuple; None turns it off."""
        if cost is None:
            pt, cap, rl = 0.0, 0, 0.0
        elif isinstance(cost, tuple):
            pt, cap, rl = cost
        else:
            pt, cap, rl = cost.per_token_latency, cost.engine_capacity, cost.reward_latency
        self._check(self.lib.ts_engine_set_cost_model(self._h, float(pt), int(cap), float(rl)),
                    "ts_engine_set_cost_model")

    def sim_times(self, n: Optional[int] = None):
        """(completion, arrival) of the local searches on the cost model's wave clock."""
        n = self.n if n is None else n
        c = np.zeros(max(1, n), np.float64)
        a = np.zeros(max(1, n), np.float64)
        self._check(self.lib.ts_read_sim_times(self._h, c.ctypes.data_as(ctypes.c_void_p),
                                               a.ctypes.data_as(ctypes.c_void_p), n, self.stream),
                    "ts_read_sim_times")
        return c[:n], a[:n]

    def set_trace(self, capacity: int) -> None:
        """Keep the per-pass allocation rows of the next runs (ts_engine_set_trace);
        0 turns the trace off."""
        self._check(self.lib.ts_engine_set_trace(self._h, int(capacity)), "ts_engine_set_trace")

    def trace_rows(self) -> np.ndarray:
        """The allocation rows since the last load, in run-queue order per step
        (a structured array: step, job, target, active, score)."""
        n, dropped = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.ts_read_trace(self._h, None, 0, ctypes.byref(n), ctypes.byref(dropped), self.stream),
                    "ts_read_trace")
        if dropped.value:
            from .tree import AccountingError

            raise AccountingError(f"trace buffer too small: {dropped.value} rows dropped")
        rows = (_abi.TsTraceRow * max(1, n.value))()
        self._check(self.lib.ts_read_trace(self._h, rows, n.value, ctypes.byref(n), None, self.stream),
                    "ts_read_trace")
        dt = np.dtype([("step", "<i4"), ("job", "<i4"), ("target", "<i4"), ("active", "<i4"), ("score", "<f8")])
        arr = np.frombuffer(bytes(rows)[: n.value * dt.itemsize], dtype=dt).copy()
        return arr[np.lexsort((arr["job"], arr["step"]))]

    def outcomes(self, n: Optional[int] = None):
        n = self.n if n is None else n
        out = (TsOutcome * max(1, n))()
        self._check(self.lib.ts_read_outcomes(self._h, out, n, self.stream), "ts_read_outcomes")
        return out[:n]

    def tree(self, i: int) -> dict:
        """SearchTree.to_dict() of search i as numpy columns (tree.py:183-203)."""
        n = ctypes.c_int32()
        self._check(self.lib.ts_tree_size(self._h, i, ctypes.byref(n)), "ts_tree_size")
        n = n.value
        out = {
            "parent": np.zeros(n, np.int32), "reward": np.zeros(n, np.float64), "prior": np.zeros(n, np.float64),
            "N": np.zeros(n, np.int32), "O": np.zeros(n, np.int32), "W": np.zeros(n, np.float64),
            "terminal": np.zeros(n, np.uint8), "depth": np.zeros(n, np.int32), "step_ref": np.zeros(n, np.int32),
        }
        order = ["parent", "reward", "prior", "N", "O", "W", "terminal", "depth", "step_ref"]
        self._check(self.lib.ts_dump_tree(self._h, i, *[out[k].ctypes.data_as(ctypes.c_void_p) for k in order]),
                    "ts_dump_tree")
        return out

    def tree_dict(self, i: int) -> dict:
        """Search i in the SearchTree.to_dict() schema (tree.py:183-203)."""
        t = self.tree(i)
        o = self.outcomes(i + 1)[i]
        nodes = [
            {"id": k, "parent": None if int(p) < 0 else int(p), "reward": float(r), "prior": float(pr),
             "N": int(n), "O": int(inf), "W": float(w), "terminal": bool(term), "depth": int(d)}
            for k, (p, r, pr, n, inf, w, term, d) in enumerate(zip(t["parent"], t["reward"], t["prior"], t["N"],
                                                                   t["O"], t["W"], t["terminal"], t["depth"]))
        ]
        return {"root": 0, "completed_rollouts": int(o.rollouts_completed),
                "rollout_budget": int(self._cfg.rollout_budget), "nodes": nodes}

    def tree_json(self, i: int) -> str:
        """SearchTree.to_json() (tree.py:205-206): byte-comparable with the reference's dump."""
        import json

        return json.dumps(self.tree_dict(i), sort_keys=True)

    # ---- step API (multi-GPU drivers, tests) -----------------------------
    def step_counts(self, step: int, dev_counts: int) -> None:
        self._check(self.lib.ts_step_counts(self._h, step, ctypes.c_void_p(dev_counts), self.stream),
                    "ts_step_counts")

    def step_admit(self, step: int, dev_all_counts: int, world: int, rank: int) -> None:
        self._check(self.lib.ts_step_admit(self._h, step, ctypes.c_void_p(dev_all_counts), world, rank,
                                           self.stream), "ts_step_admit")

    def step_records(self, step: int, dev_records: int) -> None:
        self._check(self.lib.ts_step_records(self._h, step, ctypes.c_void_p(dev_records), self.stream),
                    "ts_step_records")

    def step_targets(self, step: int, dev_all_records: int) -> None:
        self._check(self.lib.ts_step_targets(self._h, step, ctypes.c_void_p(dev_all_records), self.stream),
                    "ts_step_targets")

    def step_set_targets(self, step: int, dev_targets: int) -> None:
        """Targets from an external scheduler (int32 device array, one per local search)."""
        self._check(self.lib.ts_step_set_targets(self._h, step, ctypes.c_void_p(dev_targets), self.stream),
                    "ts_step_set_targets")

    def read_jobs(self):
        """(running int32, completed int32, best float64) device tensors of the
        local searches: the Job fields an external scheduler works on."""
        import torch

        n = max(1, self.n)
        dev = torch.device("cuda", self.device)
        running = torch.empty(n, dtype=torch.int32, device=dev)
        completed = torch.empty(n, dtype=torch.int32, device=dev)
        best = torch.empty(n, dtype=torch.float64, device=dev)
        self._check(self.lib.ts_read_jobs(self._h, ctypes.c_void_p(running.data_ptr()),
                                          ctypes.c_void_p(completed.data_ptr()), ctypes.c_void_p(best.data_ptr()),
                                          self.stream), "ts_read_jobs")
        return running[: self.n], completed[: self.n], best[: self.n]

    def step_wave(self, step: int) -> None:
        self._check(self.lib.ts_step_wave(self._h, step, self.stream), "ts_step_wave")

    # ---- the sharded batch over peer memory (multi-GPU) -----
    def xchg_create(self, world: int, rank: int, ipc: bool = True):
        """Allocate this rank's exchange buffer (after :meth:`load`); returns
        (device pointer, 64-byte CUDA IPC handle or None)."""
        from ._abi import TS_IPC_HANDLE_BYTES

        ptr = ctypes.c_void_p()
        handle = (ctypes.c_uint8 * TS_IPC_HANDLE_BYTES)() if ipc else None
        self._check(self.lib.ts_xchg_create(self._h, world, rank, ctypes.byref(ptr), handle), "ts_xchg_create")
        return int(ptr.value or 0), (bytes(handle) if ipc else None)

    def xchg_connect(self, handles=None, dev_ptrs=None) -> None:
        """Map every rank's buffer: ``handles`` (list of 64-byte IPC handles,
        other processes) or ``dev_ptrs`` (device pointers, ranks in this process)."""
        h = None
        if handles is not None:
            h = (ctypes.c_uint8 * (64 * len(handles))).from_buffer_copy(b"".join(handles))
        d = None
        if dev_ptrs is not None:
            d = (ctypes.c_void_p * len(dev_ptrs))(*[ctypes.c_void_p(x) for x in dev_ptrs])
        self._check(self.lib.ts_xchg_connect(self._h, h, d), "ts_xchg_connect")

    def px_times(self, n: int) -> np.ndarray:
        """[n, 3] ns stamps per wave of the last run_sharded: counts phase start,
        all records in, compute_targets done."""
        buf = np.zeros((max(1, n), 3), np.uint64)
        self._check(self.lib.ts_read_px_times(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n,
                                              self.stream), "ts_read_px_times")
        return buf[:n]

    def run_sharded(self, max_steps: int = (1 << 31) - 1, last_arrival: int = 0) -> TsRunStats:
        """The whole sharded batch as one device-driven graph loop (a collective
        over the connected ranks); ``last_arrival`` = the largest arrival step
        of the global run queue."""
        st = TsRunStats()
        self._check(self.lib.ts_run_sharded(self._h, max_steps, last_arrival, ctypes.byref(st), self.stream),
                    "ts_run_sharded")
        return st

    def read_targets(self, n: Optional[int] = None) -> list:
        n = self.n if n is None else n
        buf = (ctypes.c_int32 * max(1, n))()
        self._check(self.lib.ts_read_targets(self._h, buf, n, self.stream), "ts_read_targets")
        return list(buf[:n])

    def latencies_ns(self, n: Optional[int] = None) -> np.ndarray:
        """Per-search admission→exit latency in ns (device %globaltimer)."""
        n = self.n if n is None else n
        buf = np.zeros(max(1, n), np.uint64)
        self._check(self.lib.ts_read_latencies(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n,
                                               self.stream), "ts_read_latencies")
        return buf[:n]

    def step_times(self, n: int) -> np.ndarray:
        buf = np.zeros(max(1, n), np.uint64)
        self._check(self.lib.ts_read_step_times(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n,
                                                self.stream), "ts_read_step_times")
        return buf[:n]

    def run_batch_host(self, table, max_steps: int = (1 << 31) - 1, out=None):
        """End to end through one C-ABI call: host table in, host outcomes out
        (pinned buffers from :func:`pinned_array` are copied by DMA directly)."""
        n = len(table)
        out = (TsOutcome * n)() if out is None else out
        st = TsRunStats()
        self._check(self.lib.ts_run_batch_host(self._h, table, n, max_steps, out, ctypes.byref(st), self.stream),
                    "ts_run_batch_host")
        self.n = n
        return out, st


def fill_problem(seed: int, solvable: bool, depth_range, branching: int, profile) -> TsProblem:
    """ts_fill_problem: make_problem + golden_step_rewards in the library (backend.py:144-215)."""
    lib = load_library()
    p = TsProblem()
    sh = profile.shared_range
    rc = lib.ts_fill_problem(int(seed) & 0xFFFFFFFFFFFFFFFF, int(solvable), depth_range[0], depth_range[1], branching,
                             profile.golden_range[0], profile.golden_range[1], profile.off_path_range[0],
                             profile.off_path_range[1], profile.hidden_until_depth, 1 if sh else 0,
                             sh[0] if sh else 0.0, sh[1] if sh else 0.0, profile.target_aggregate, ctypes.byref(p))
    raise_for_status(rc, "ts_fill_problem")
    return p


def pinned_array(ctype, n: int, init=None):
    """A ctypes array of ``n`` ``ctype`` in page-locked host memory (kept alive
    by the returned array's ``_owner``), optionally filled from ``init``."""
    import torch

    buf = torch.empty(ctypes.sizeof(ctype) * max(1, n), dtype=torch.uint8, pin_memory=True)
    arr = (ctype * n).from_address(buf.data_ptr())
    arr._owner = buf
    if init is not None:
        ctypes.memmove(arr, init, ctypes.sizeof(ctype) * n)
    return arr
