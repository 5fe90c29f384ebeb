"""Device plumbing of the standalone policy operators (csrc/policy.cu).

The reference's scheduler and exit-policy entry points take Python state —
a ``SchedulerState`` run queue, ``SearchTree`` objects.  These helpers flatten
that state into device arrays, call the C-ABI (``ts_compute_targets``,
``ts_parallelism_scores``, ``ts_exit_policy``) and map the status codes back
to the reference's exceptions.  The arithmetic (scores, the ordered score
sum, the (-S, arrival, id) ordering, the allocation, leaf classification and
the exit decision) runs in the kernels; nothing here computes a policy value.
There is no CPU path: without a CUDA device these raise.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _abi
from ._abi import TsForest, TsSchedParams, TsTargetsInfo, load_library, raise_for_status


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the policy operators run on the CUDA device; no CUDA device is available")
    return torch


def _stream(stream) -> int:
    torch = _torch()
    if stream is None:
        return int(torch.cuda.current_stream().cuda_stream)
    return int(getattr(stream, "cuda_stream", stream))


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _err() -> str:
    return (load_library().ts_policy_last_error() or b"").decode()


def sched_params(config, positive_exit_threshold: float) -> TsSchedParams:
    return TsSchedParams(int(config.max_concurrency), float(config.beta), float(config.proximity),
                         int(config.obs_threshold), 1 if config.boosting_enabled else 0,
                         float(positive_exit_threshold))


def _torch_stream(stream, device):
    """The torch stream object for a caller's stream argument (None: current)."""
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(getattr(stream, "cuda_stream", stream)), device=device)


def _dev(a, dtype, torch, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).pin_memory().to(device, non_blocking=True)


def compute_targets_arrays(arrival, best, completed, job_id, now: float, config, positive_exit_threshold: float,
                           device: int = 0, stream=None):
    """compute_targets over a run queue given as arrays (numpy or device
    tensors) in run-queue order.  Returns (targets int32 device tensor,
    TsTargetsInfo).  Raises ValueError like the reference."""
    torch = _torch()
    lib = load_library()
    dev = torch.device("cuda", device)
    # the H2D copies and the output live on the stream the kernels run on
    with torch.cuda.device(dev), torch.cuda.stream(_torch_stream(stream, dev)):
        arr = _dev(arrival, torch.float64, torch, dev)
        bst = _dev(best, torch.float64, torch, dev)
        cmp = _dev(completed, torch.int32, torch, dev)
        ids = _dev(job_id, torch.int64, torch, dev)
        n = int(arr.numel())
        out = torch.empty(max(1, n), dtype=torch.int32, device=dev)
        info = TsTargetsInfo()
        p = sched_params(config, positive_exit_threshold)
        rc = lib.ts_compute_targets(ctypes.byref(p), float(now), _ptr(arr), _ptr(bst), _ptr(cmp), _ptr(ids), n,
                                    _ptr(out), ctypes.byref(info), _stream(stream))
    if rc != _abi.TS_OK:
        if rc == _abi.TS_INVALID_ARGUMENT and n and info.first_bad < n:
            a = float(arr[info.first_bad].item())
            raise ValueError(f"now={now} precedes arrival={a}")
        raise_for_status(rc, "compute_targets", _err())
    return out[:n], info


def parallelism_scores_arrays(arrival, best, now: float, positive_exit_threshold: float, config,
                              device: int = 0, stream=None):
    """parallelism_score for many jobs (device tensor of float64)."""
    torch = _torch()
    lib = load_library()
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev), torch.cuda.stream(_torch_stream(stream, dev)):
        arr = _dev(arrival, torch.float64, torch, dev)
        bst = _dev(best, torch.float64, torch, dev)
        n = int(arr.numel())
        out = torch.empty(max(1, n), dtype=torch.float64, device=dev)
        bad = ctypes.c_int32(n)
        rc = lib.ts_parallelism_scores(float(now), float(positive_exit_threshold), float(config.beta),
                                       float(config.proximity), _ptr(arr), _ptr(bst), n, _ptr(out),
                                       ctypes.byref(bad), _stream(stream))
    if rc != _abi.TS_OK:
        if rc == _abi.TS_INVALID_ARGUMENT and bad.value < n:
            raise ValueError(f"now={now} precedes arrival={float(arr[bad.value].item())}")
        raise_for_status(rc, "parallelism_score", _err())
    return out[:n]


def reconcile_arrays(targets, offsets, prefix_score, rollout_id, running=None, device: int = 0, stream=None):
    """reconcile + choose_preemption_victims (scheduler.py:190-214) over a run
    queue as arrays: job j's in-flight rollouts are [offsets[j], offsets[j+1])
    of ``prefix_score``/``rollout_id``.  Returns (launch int32[n_jobs],
    victim_rank int32[n_rollouts]) device tensors (see ts_reconcile)."""
    torch = _torch()
    lib = load_library()
    dev = torch.device("cuda", device)
    with torch.cuda.device(dev), torch.cuda.stream(_torch_stream(stream, dev)):
        tgt = _dev(targets, torch.int32, torch, dev)
        off = _dev(offsets, torch.int64, torch, dev)
        sc = _dev(prefix_score, torch.float64, torch, dev)
        ids = _dev(rollout_id, torch.int64, torch, dev)
        run = None if running is None else _dev(running, torch.int32, torch, dev)
        n = int(tgt.numel())
        if int(off.numel()) != n + 1 or int(sc.numel()) != int(ids.numel()):
            raise ValueError("reconcile: offsets must have n_jobs + 1 entries, scores and ids one per rollout")
        launch = torch.empty(max(1, n), dtype=torch.int32, device=dev)
        rank = torch.empty(max(1, int(sc.numel())), dtype=torch.int32, device=dev)
        rc = lib.ts_reconcile(_ptr(run), _ptr(tgt), _ptr(off), _ptr(sc), _ptr(ids), n, _ptr(launch), _ptr(rank),
                              _stream(stream))
    if rc != _abi.TS_OK:
        raise_for_status(rc, "reconcile", _err())
    return launch[:n], rank[: int(sc.numel())]


# ---- forests of SearchTrees ------------------------------------------------------

def _tree_columns(tree):
    """(parent local index, reward, depth, terminal, has_children, best, completed, budget)
    of one tree: a reference-style SearchTree (``nodes`` dict of StepNodes,
    ``root_id``), its ``to_dict()`` dump, or an Engine.tree() column dict."""
    if isinstance(tree, dict) and "parent" in tree and not isinstance(tree.get("nodes"), list):
        parent = np.asarray(tree["parent"], np.int32)
        n = parent.size
        has_kids = np.zeros(n, bool)
        has_kids[parent[parent >= 0]] = True
        best = tree.get("best_score")
        return (parent, np.asarray(tree["reward"], np.float64), np.asarray(tree["depth"], np.int32),
                np.asarray(tree["terminal"], bool), has_kids, best, tree.get("completed_rollouts"),
                tree.get("rollout_budget"))
    if isinstance(tree, dict):  # SearchTree.to_dict() (tree.py:183-203)
        nodes = tree["nodes"]
        root = tree["root"]
        order = [root] + [r["id"] for r in nodes if r["id"] != root]
        pos = {nid: i for i, nid in enumerate(order)}
        by_id = {r["id"]: r for r in nodes}
        recs = [by_id[i] for i in order]
        parent = np.array([-1 if r["parent"] is None else pos[r["parent"]] for r in recs], np.int32)
        has_kids = np.zeros(len(recs), bool)
        has_kids[parent[parent >= 0]] = True
        return (parent, np.array([r["reward"] for r in recs], np.float64),
                np.array([r["depth"] for r in recs], np.int32), np.array([r["terminal"] for r in recs], bool),
                has_kids, tree.get("best_score"), tree.get("completed_rollouts"), tree.get("rollout_budget"))
    nodes = tree.nodes
    root = tree.root_id
    order = [root] + [nid for nid in nodes if nid != root]
    pos = {nid: i for i, nid in enumerate(order)}
    recs = [nodes[i] for i in order]
    parent = np.array([-1 if n.parent_id is None else pos[n.parent_id] for n in recs], np.int32)
    best_t = getattr(tree, "best_trajectory", None)
    return (parent, np.array([n.prm_reward for n in recs], np.float64), np.array([n.depth for n in recs], np.int32),
            np.array([n.is_terminal for n in recs], bool), np.array([bool(n.children) for n in recs], bool),
            None if best_t is None else best_t.aggregate_score, getattr(tree, "completed_rollouts", None),
            getattr(tree, "rollout_budget", None))


FOREST_FIELDS = ("offsets", "tree_of", "parent", "reward", "depth", "flags", "best_score", "has_best", "completed",
                 "budget", "exhausted")


def flatten_trees(trees: Sequence, tree_exhausted: Optional[Sequence[bool]] = None) -> dict:
    """Host numpy columns of a forest (the ts_forest layout)."""
    cols = [_tree_columns(t) for t in trees]
    sizes = np.array([c[0].size for c in cols], np.int64)
    off = np.zeros(len(cols) + 1, np.int64)
    np.cumsum(sizes, out=off[1:])
    if off[-1] >= 2**31:
        raise ValueError("forest too large")
    parent = np.concatenate([np.where(c[0] >= 0, c[0] + o, -1) for c, o in zip(cols, off[:-1])]) \
        if cols else np.zeros(0, np.int32)
    cat = (lambda i, dt: np.concatenate([c[i] for c in cols]).astype(dt) if cols else np.zeros(0, dt))  # noqa: E731
    flags = (cat(3, np.uint8) * _abi.TS_NODE_TERMINAL) | (cat(4, np.uint8) * _abi.TS_NODE_HAS_CHILDREN)
    return {
        "offsets": off.astype(np.int32),
        "tree_of": np.repeat(np.arange(len(cols), dtype=np.int32), sizes),
        "parent": parent.astype(np.int32),
        "reward": cat(1, np.float64),
        "depth": cat(2, np.int32),
        "flags": flags.astype(np.uint8),
        "best_score": np.array([0.0 if c[5] is None else c[5] for c in cols], np.float64),
        "has_best": np.array([c[5] is not None for c in cols], np.uint8),
        "completed": np.array([-1 if c[6] is None else c[6] for c in cols], np.int32),
        "budget": np.array([(1 << 31) - 1 if c[7] is None else c[7] for c in cols], np.int32),
        "exhausted": np.zeros(len(cols), np.uint8) if tree_exhausted is None else
        np.asarray(tree_exhausted, np.uint8),
    }


class Forest:
    """A forest of trees in device memory (ts_forest)."""

    def __init__(self, trees: Sequence, tree_exhausted: Optional[Sequence[bool]] = None, device: int = 0):
        torch = _torch()
        host = flatten_trees(trees, tree_exhausted)
        dev = torch.device("cuda", device)
        self.device = device
        self._keep = {k: torch.as_tensor(v).to(dev) for k, v in host.items()}
        self.n_trees = len(host["offsets"]) - 1
        self.n_nodes = int(host["offsets"][-1])
        self.c = TsForest(self.n_trees, self.n_nodes, *[self._keep[k].data_ptr() for k in FOREST_FIELDS])
        self.best = host["best_score"]
        self.has_best = host["has_best"]


def exit_policy(forest: Forest, scoring, positive_enabled: bool, negative_enabled: bool, stream=None):
    """(kinds int32[n], ne uint8[n]) host arrays from one ts_exit_policy call."""
    torch = _torch()
    from .config import scoring_to_c

    lib = load_library()
    cfg = scoring_to_c(scoring, positive_enabled, negative_enabled)
    dev = torch.device("cuda", forest.device)
    n = max(1, forest.n_trees)
    with torch.cuda.device(dev):
        kind = torch.empty(n, dtype=torch.int32, device=dev)
        ne = torch.empty(n, dtype=torch.uint8, device=dev)
        rc = lib.ts_exit_policy(ctypes.byref(cfg), ctypes.byref(forest.c), _ptr(kind), _ptr(ne), _stream(stream))
        raise_for_status(rc, "ts_exit_policy", _err())
        return kind[: forest.n_trees].cpu().numpy(), ne[: forest.n_trees].cpu().numpy()
