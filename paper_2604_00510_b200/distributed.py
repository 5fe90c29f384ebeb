"""Multi-GPU driver: one process per GPU, searches block-sharded over ranks.

Searches are independent trees and the synthetic backend is stateless keyed
RNG, so each rank owns a contiguous block of the global run queue
(``Engine.load(table, global_offset, n_global)``).  The only data crossing
GPUs per wave are the boosting scheduler's global terms:

* 3 int64 counts per rank {running, arrived-but-pending, unfinished} — the
  global FIFO admission (admit_jobs, scheduler.py:131-140) and the loop test;
* one 16-byte ``ts_sched_record`` per search {S(i,t), flags} — the ordered
  score sum and the merge ranks of compute_targets (scheduler.py:143-187).

Both are all-gathered (NCCL over NVLink on GPUs; any torch.distributed
backend works) in rank order, which is global run-queue order, and every rank
then runs the scheduler kernel on the same global records and keeps its slice.
"""

from __future__ import annotations

from typing import Optional

RECORD_BYTES = 16
COUNT_WORDS = 3


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of the global run queue owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class ShardedRun:
    """The per-wave exchange loop of one rank.

    ``engine`` exposes the step API of :class:`paper_2604_00510_b200.engine.Engine`
    (step_counts/step_admit/step_records/step_targets/step_wave taking device
    pointers); ``dist`` is ``torch.distributed`` with an initialised group.
    """

    def __init__(self, engine, dist, n_local: int, n_total: int, device, group=None, check_every: int = 8,
                 host_staging: bool = False):
        import torch

        self.engine = engine
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # host_staging: exchange through host memory (a backend without device
        # tensors, e.g. gloo with several ranks on one GPU in tests)
        self.host = host_staging
        xdev = "cpu" if host_staging else device
        if self.world > 1 and any(s != n_local for s in self._all_sizes(n_local, xdev)):
            raise ValueError("all-gather needs equal shard sizes; pad the run queue")
        self.n_local = n_local
        self.n_total = n_total
        self.check_every = max(1, check_every)
        self.counts = torch.zeros(COUNT_WORDS, dtype=torch.int64, device=device)
        self.all_counts = torch.zeros(COUNT_WORDS * self.world, dtype=torch.int64, device=device)
        self.records = torch.zeros(n_local * RECORD_BYTES, dtype=torch.uint8, device=device)
        self.all_records = torch.zeros(n_total * RECORD_BYTES, dtype=torch.uint8, device=device)

    def _all_sizes(self, n_local, device):
        import torch

        t = torch.tensor([n_local], dtype=torch.int64, device=device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]

    def _gather(self, out, inp):
        if self.host:
            o = out.new_empty(out.shape, device="cpu")
            parts = list(o.chunk(self.world))
            self.dist.all_gather(parts, inp.cpu(), group=self.group)
            out.copy_(o if parts[0].data_ptr() == o.data_ptr() else __import__("torch").cat(parts))
            return
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        parts = list(out.chunk(self.world))
        self.dist.all_gather(parts, inp, group=self.group)
        if parts[0].data_ptr() != out.data_ptr():  # backend returned fresh tensors
            out.copy_(__import__("torch").cat(parts))

    def _global_max(self, x: int) -> int:
        import torch

        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device="cpu" if self.host else self.counts.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def run(self, max_steps: int = 1 << 30, wave_events: Optional[list] = None) -> int:
        """Advance waves until every search of every rank has exited; returns
        the number of waves (the reference loop's ``steps``).  ``wave_events``
        collects (start, stop) CUDA events around every wave launch.

        Admission needs the counts exchange only while a search can still be
        waiting: with M >= the whole run queue, after the last arrival step
        nothing is ever pending, so those waves skip it (admit_jobs with no
        pending search admits nothing) and the loop test reads the running
        flags of the records every wave instead; otherwise the counts are
        exchanged and tested every wave.  Either test is read back after the
        wave is queued (a finished run costs one empty wave, never a wrong
        step count).  ``check_every`` is kept for API compatibility."""
        import torch

        eng = self.engine
        table = getattr(eng, "_table", None)
        local_max = max((int(p.arrival_step) for p in table), default=0) if table is not None else 1 << 30
        last_arrival = self._global_max(local_max)
        cfg = getattr(eng, "_cfg", None)
        capacity = int(cfg.max_concurrency) if cfg is not None else 0  # unknown: always exchange counts
        no_pending = torch.zeros(COUNT_WORDS * self.world, dtype=torch.int64, device=self.counts.device)
        on_gpu = self.counts.device.type == "cuda"
        self._flag_host = torch.zeros(1, dtype=torch.int32, pin_memory=on_gpu)
        self._flag_event = torch.cuda.Event() if on_gpu else _HostEvent()
        for step in range(max_steps):
            admission = capacity < self.n_total or step <= last_arrival
            if admission:
                eng.step_counts(step, self.counts.data_ptr())
                self._gather(self.all_counts, self.counts)
                # the loop test (no unfinished search on any rank) is read back
                # after this wave is queued, like the running flags below: the
                # returned step count is exact and the GPU never idles on it
                unfinished = self.all_counts.view(-1, COUNT_WORDS)[:, 2].sum()
                self._flag_host.copy_((unfinished > 0).to(torch.int32).view(1), non_blocking=True)
                self._flag_event.record()
                eng.step_admit(step, self.all_counts.data_ptr(), self.world, self.rank)
            else:
                eng.step_admit(step, no_pending.data_ptr(), self.world, self.rank)
            eng.step_records(step, self.records.data_ptr())
            self._gather(self.all_records, self.records)
            if not admission:
                # the loop test reads this wave's running flags, but only after
                # the wave is queued: the GPU never idles on the host's check
                # (a finished job costs one empty scheduler step instead)
                flags = self.all_records.view(-1, RECORD_BYTES)[:, 8]
                self._flag_host.copy_((flags & 1).any().to(torch.int32).view(1), non_blocking=True)
                self._flag_event.record()
            eng.step_targets(step, self.all_records.data_ptr())
            if wave_events is None:
                eng.step_wave(step)
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                eng.step_wave(step)
                e1.record()
                wave_events.append((e0, e1))
            self._flag_event.synchronize()
            if int(self._flag_host[0]) == 0:
                return step
        return max_steps


class PeerShardedRun:
    """The sharded batch of one rank as one device-driven graph loop
    (``ts_run_sharded``): per wave every rank writes its admission counts and
    scheduler records straight into every rank's exchange buffer over NVLink
    (CUDA IPC mappings) and waits on flags in its own buffer — no collective
    call and no host round trip per wave.  ``dist`` is used once, at set-up,
    to exchange the 64-byte IPC handles and the last arrival step.  Shards may
    differ in size."""

    def __init__(self, engine, dist, group=None):
        import torch

        self.engine = engine
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        ptr, handle = engine.xchg_create(self.world, self.rank, ipc=self.world > 1)
        handles = [handle]
        # host-side collectives once at set-up (NCCL needs device tensors)
        dev = torch.device("cuda", torch.cuda.current_device()) if (
            self.world > 1 and dist.get_backend(group) == "nccl") else torch.device("cpu")
        if self.world > 1:
            mine = torch.tensor(list(handle), dtype=torch.uint8, device=dev)
            out = [torch.zeros_like(mine) for _ in range(self.world)]
            dist.all_gather(out, mine, group=group)
            handles = [bytes(t.cpu().tolist()) for t in out]
        engine.xchg_connect(handles=handles if self.world > 1 else None,
                            dev_ptrs=None if self.world > 1 else [ptr])
        table = getattr(engine, "_table", None)
        local_max = max((int(p.arrival_step) for p in table), default=0) if table is not None else 0
        t = torch.tensor([local_max], dtype=torch.int64, device=dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            dist.barrier(group=group)  # every buffer is zeroed and mapped before any peer writes
        self.last_arrival = int(t.item())

    def run(self, max_steps: int = (1 << 31) - 1):
        return self.engine.run_sharded(max_steps, self.last_arrival)


def connect_in_process(engines) -> list:
    """Ranks emulated in one process (one GPU): connect the engines' exchange
    buffers by device pointer; returns the pointers."""
    world = len(engines)
    ptrs = []
    for r, e in enumerate(engines):
        p, _ = e.xchg_create(world, r, ipc=False)
        ptrs.append(p)
    for e in engines:
        e.xchg_connect(dev_ptrs=ptrs)
    return ptrs


def last_arrival_of(tables) -> int:
    return max((int(p.arrival_step) for t in tables for p in t), default=0)


class _HostEvent:
    """Stand-in for a CUDA event when the exchange runs on CPU tensors."""

    def record(self):
        pass

    def synchronize(self):
        pass


def run_sharded(engine, dist, n_local: int, n_total: int, device, group=None,
                max_steps: int = 1 << 30, check_every: int = 8, host_staging: bool = False) -> int:
    return ShardedRun(engine, dist, n_local, n_total, device, group, check_every, host_staging).run(max_steps)
