"""The multi-rank wave driver (paper_2604_00510_b200/distributed.py) on CPU:
world_size 2 over gloo with a host-side mock of the engine's step API.

The mock reproduces the step contract the kernels implement (k_counts,
k_admit's global FIFO, per-search records in run-queue order, one rollout per
running search per wave) so the test checks the exchange logic: counts and
records are gathered in global run-queue order, admission is one FIFO over
ranks, and a sharded run decides exactly like a single-rank run.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_00510_b200.distributed import RECORD_BYTES, run_sharded, shard_bounds

N_TOTAL = 24
M = 5


def _workload():
    rng = np.random.RandomState(3)
    arrivals = np.cumsum(rng.randint(0, 3, size=N_TOTAL)).tolist()
    lifetimes = rng.randint(1, 6, size=N_TOTAL).tolist()
    return arrivals, lifetimes


class MockEngine:
    def __init__(self, arrivals, lifetimes, goff):
        self.arr, self.life, self.goff = arrivals, lifetimes, goff
        n = len(arrivals)
        self.state = [0] * n  # 0 pending, 1 running, 2 finished
        self.done = [0] * n
        self.admit = [-1] * n
        self.exit = [-1] * n
        self.head = 0
        self.running = 0
        self.targets = [0] * n

    def step_counts(self, step, ptr):
        arrived = sum(1 for a in self.arr if a <= step)
        fin = sum(1 for s in self.state if s == 2)
        vals = (ctypes.c_int64 * 3)(self.running, arrived - self.head, len(self.arr) - fin)
        ctypes.memmove(ptr, vals, 24)

    def step_admit(self, step, ptr, world, rank):
        allc = np.frombuffer((ctypes.c_int64 * (3 * world)).from_address(ptr), dtype=np.int64).reshape(world, 3)
        run_g, pend_g = int(allc[:, 0].sum()), int(allc[:, 1].sum())
        before = int(allc[:rank, 1].sum())
        a = max(0, min(M - run_g, pend_g))
        q = max(0, min(a - before, int(allc[rank, 1])))
        for i in range(self.head, self.head + q):
            self.state[i] = 1
            self.admit[i] = step
        self.head += q
        self.running += q

    def step_records(self, step, ptr):
        buf = np.zeros(len(self.arr) * 2, dtype=np.float64)
        flags = buf.view(np.uint32)
        for i, st in enumerate(self.state):
            if st == 1:
                buf[2 * i] = float(self.goff + i)
                flags[4 * i + 2] = 1
        ctypes.memmove(ptr, buf.ctypes.data, buf.nbytes)

    def step_targets(self, step, ptr):
        n = N_TOTAL
        recs = np.frombuffer((ctypes.c_uint8 * (n * RECORD_BYTES)).from_address(ptr), dtype=np.uint8).copy()
        scores = recs.view(np.float64)[0::2]
        flags = recs.view(np.uint32)[2::4]
        for g in range(n):  # records arrive in global run-queue order
            if flags[g] & 1:
                assert scores[g] == float(g)
        for i in range(len(self.arr)):
            self.targets[i] = 1 if self.state[i] == 1 else 0

    def step_wave(self, step):
        for i, st in enumerate(self.state):
            if st == 1 and self.targets[i]:
                self.done[i] += 1
                if self.done[i] >= self.life[i]:
                    self.state[i] = 2
                    self.exit[i] = step
                    self.running -= 1


def _worker(rank, world, port, out, batch=False):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    arrivals, lifetimes = _workload()
    if batch:  # all requests at step 0, budget for all: the loop skips the counts exchange
        global M
        M = N_TOTAL
        arrivals = [0] * N_TOTAL
    lo, hi = shard_bounds(N_TOTAL, world, rank)
    eng = MockEngine(arrivals[lo:hi], lifetimes[lo:hi], lo)
    if batch:
        eng._cfg = type("Cfg", (), {"max_concurrency": M})()
        eng._table = [type("P", (), {"arrival_step": a})() for a in arrivals[lo:hi]]
    steps = run_sharded(eng, dist, hi - lo, N_TOTAL, "cpu", check_every=1)
    out[rank] = (steps, eng.admit, eng.exit)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, batch=False):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, batch), nprocs=world, join=True)
    steps = {out[r][0] for r in range(world)}
    assert len(steps) == 1
    admit = [a for r in range(world) for a in out[r][1]]
    exit_ = [e for r in range(world) for e in out[r][2]]
    return steps.pop(), admit, exit_


def test_shard_bounds_cover_queue():
    for n in (1, 7, 4096, 32768):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_gloo_world2_matches_single_rank():
    s1, a1, e1 = _run(1)
    s2, a2, e2 = _run(2)
    assert (s1, a1, e1) == (s2, a2, e2)
    # global FIFO under M: never more than M running at once
    for step in range(s1):
        running = sum(1 for a, e in zip(a1, e1) if a <= step <= e and a >= 0)
        assert running <= M


def test_gloo_world2_batch_mode_skips_counts_exchange():
    """M >= the run queue and every request at step 0: after the first wave the
    loop skips the counts exchange and stops on the gathered running flags,
    with the same decisions as one rank and no extra (empty) waves."""
    s1, a1, e1 = _run(1, batch=True)
    s2, a2, e2 = _run(2, batch=True)
    assert (s1, a1, e1) == (s2, a2, e2)
    assert all(a == 0 for a in a1)
    assert s1 == max(e1) + 1
