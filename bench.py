"""Benchmark: MCTS rollouts/s and p99 per-search latency (BASELINE.json metric).

Workload (N=1, BASELINE.json configs[1]): 4096 concurrent searches, branching 4,
depth 16 (base depth 15 + 1), rollout budget 128, positive + negative early
exit and adaptive boosting on, M = 4096, workload seed 0 — synthetic problems
from the reference's seeded generator (make_workload).  One bench "step" is
one whole batch: every search admitted at wave 0 and advanced wave by wave
until all have exited.  Under torchrun (N>1) every rank runs its own block of
4096 searches of one 4096*N-request run queue (weak scaling; M = 4096*N) and
the scheduler records are all-gathered over NCCL each wave.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PER_GPU = 4096
BUDGET, DEPTH_CAP, WIDTH, BRANCH, BASE = 128, 16, 4, 4, 15
METRIC = "MCTS rollouts/sec (p99 per-search latency alongside)"
UNIT = "rollouts/s"
# algorithmic bytes: per WU-PUCT child scored, per
# selection level, per node created, per path node of a backup/cancel
B_SCORED, B_LEVEL, B_NODE, B_PATH = 28, 28, 44, 48


def workload(n_total: int):
    from paper_2604_00510_b200 import backend as B

    D = {d: (BASE, BASE) for d in B.Difficulty}
    return B.make_workload(n_total, (0.6, 0.25, 0.15), 0, branching=BRANCH, depth_ranges=D)


def config_dict(n_total: int, n_gpus: int) -> dict:
    """The workload description, identical in both arms (--impl ours|reference)."""
    return {"workload": f"c2: {PER_GPU}/GPU searches, b={BRANCH}, depth {BASE + 1}, budget {BUDGET}, "
                        f"PE+NE+boost, M={n_total}",
            "searches": n_total, "branching": BRANCH, "depth": BASE + 1, "rollout_budget": BUDGET,
            "max_concurrency": n_total, "parallelism": f"search-sharded x{n_gpus}",
            "l2": "flushed (512 MiB write) before every timed step; node pool > L2"}


def search_config(M: int, exits: bool = True):
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    return SearchConfig(scheduler=SchedulerConfig(max_concurrency=M), rollout_budget=BUDGET, depth_cap=DEPTH_CAP,
                        expand_width=WIDTH, positive_exit=exits, negative_exit=exits)


def percentile(values, pct: float) -> float:
    """Nearest-rank percentile, as metrics.percentile (metrics.py:86-94)."""
    vals = sorted(values)
    if not vals:
        return 0.0
    import math

    k = max(1, math.ceil(pct / 100.0 * len(vals)))
    return vals[k - 1]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock and throttle reasons sampled every ~2 ms during the timed region
    (NVML in a background thread; nvidia-smi as a fallback)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.err = [], set(), None, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv, self.err = None, str(e)
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        while not self._stop.is_set():
            if self.nv is not None:
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    try:
                        r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    except AttributeError:
                        r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                    for bit, name in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception as e:  # pragma: no cover
                    self.err = str(e)
            time.sleep(0.002)

    def stop(self) -> dict:
        self._stop.set()
        self.t.join()
        busy = [x for x in self.samples if x > 0]
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(busy), "source": "nvml" if self.nv else self.err}


def flush_l2(buf):
    buf.add_(1)  # writes 512 MiB > the 126 MB L2


# --------------------------------------------------------------------------- ours
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = "nccl"

    def init(self):
        import torch

        # TS_BENCH_BACKEND=gloo runs the N>1 path with several ranks on one GPU
        # (validation of the sharded driver only; the measured path is NCCL)
        self.backend = os.environ.get("TS_BENCH_BACKEND", "nccl")
        if self.backend == "nccl" and self.world > torch.cuda.device_count():
            raise SystemExit(f"bench.py: {self.world} ranks over NCCL need {self.world} GPUs, this node has "
                             f"{torch.cuda.device_count()} (TS_BENCH_BACKEND=gloo validates N ranks on one GPU)")
        if self.backend != "nccl":
            self.local = self.local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.local)
        if self.world > 1:
            import torch.distributed as dist

            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        self.pg.all_reduce(t)
        return float(t.item())


def algorithmic_bytes(st) -> int:
    return (B_SCORED * st.children_scored + B_LEVEL * st.select_levels + B_NODE * st.nodes
            + B_PATH * st.path_nodes)


def issue_roofline(rollouts_per_s: float, rollouts: int):
    """The throughput regime's real bound: warp-instruction issue.  Instructions
    per rollout from the newest ncu capture of the exits-off batch's
    free-running kernel (one launch = the whole batch); peak = 4 schedulers x
    SMs x the SM clock, one warp-instruction each per cycle."""
    import torch

    for rnd in ("r02",):
        path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_full_captures.json")
        try:
            with open(path) as f:
                cap = json.load(f)["k_wave_free_exits_off"]["metrics"]
        except Exception:
            continue
        instr = float(cap["Executed Instructions"].split()[0].replace(",", ""))
        per = instr / 524288.0  # the captured launch ran the whole 4096 x 128-rollout batch
        props = torch.cuda.get_device_properties(torch.cuda.current_device())
        clk = float(cap["SM Frequency"].split()[0]) * 1e9
        peak = 4.0 * props.multi_processor_count * clk
        achieved = per * rollouts_per_s
        return {"bound": "issue", "instr_per_rollout": per, "achieved_warp_instr_per_s": achieved,
                "peak_warp_instr_per_s": peak, "frac": achieved / peak,
                "ceiling_rollouts_per_s": peak / per,
                "source": f"{os.path.relpath(path, ROOT)} (ncu --set full, k_wave_free, "
                          f"issue slots busy {cap.get('Issue Slots Busy')})"}
    return None


def peer_exchange(eng, table, lo, n_total, d: Dist):
    """The sharded loop over peer memory (PeerShardedRun: one device-driven
    graph per batch, scheduler inputs written straight into every rank's
    buffer over NVLink).  Validated with one batch; if any rank cannot set it
    up (no CUDA IPC / peer access), every rank falls back to ShardedRun's
    NCCL all-gathers together."""
    import sys

    from paper_2604_00510_b200.distributed import PeerShardedRun

    peer, ok = None, 1.0
    try:
        eng.load(table, lo, n_total)
        peer = PeerShardedRun(eng, d.pg)
        peer.run()
    except Exception as ex:  # reported; the whole job switches transport together
        print(f"bench.py rank {d.rank}: peer exchange unavailable ({ex}); NCCL all-gather loop", file=sys.stderr)
        ok = 0.0
    if -d.max(-ok) < 1.0:
        return None
    return peer


def profile_waves(eng, table, lo, n_total, d: Dist, sharded=None):
    """Σ wave-kernel time (CUDA events on the launch stream) and algorithmic
    bytes of one batch; for N ranks the bytes of all ranks over the slowest
    rank's wave time."""
    import torch

    if d.world > 1:
        eng.load(table, lo, n_total)
        evs = []
        torch.cuda.synchronize()
        d.barrier()
        sharded.run(wave_events=evs)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        return d.max(ms), int(d.sum(algorithmic_bytes(eng.stats())))
    n = len(table)
    eng.load(table, lo, n_total)
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    recs = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    evs = []
    step = 0
    while True:
        eng.step_counts(step, counts.data_ptr())
        if step % 4 == 0:
            torch.cuda.synchronize()
            if int(counts[2].item()) == 0:
                break
        eng.step_admit(step, counts.data_ptr(), 1, 0)
        eng.step_records(step, recs.data_ptr())
        eng.step_targets(step, recs.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step_wave(step)
        e1.record()
        evs.append((e0, e1))
        step += 1
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    return ms, algorithmic_bytes(eng.stats())


def bench_ours(args, d: Dist):
    import torch

    from paper_2604_00510_b200.backend import problem_table
    from paper_2604_00510_b200.engine import Engine

    N = d.world
    n_total = PER_GPU * N
    specs = workload(n_total)
    lo = d.rank * PER_GPU
    table = problem_table(specs[lo: lo + PER_GPU])
    cfg = search_config(n_total)
    eng = Engine(cfg, d.local)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    sharded, peer = None, None
    if N > 1:
        from paper_2604_00510_b200.distributed import ShardedRun

        sharded = ShardedRun(eng, d.pg, PER_GPU, n_total, torch.device("cuda", d.local),
                             host_staging=d.backend != "nccl")
        peer = peer_exchange(eng, table, lo, n_total, d)

    def one_step():
        if N == 1:
            eng.run()
        elif peer is not None:
            peer.run()
        else:
            sharded.run()

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        eng.load(table, lo, n_total)
        one_step()
    torch.cuda.synchronize()
    d.barrier()
    clocks = Clocks(d.local) if d.rank == 0 else None
    total_ms, rollouts, launches, lat, stats = 0.0, 0, 0, [], None
    for _ in range(args.steps):
        eng.load(table, lo, n_total)  # H2D of the problem table + tree reset: outside the timed region
        flush_l2(flush)
        torch.cuda.synchronize()
        d.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = d.max(e0.elapsed_time(e1))
        total_ms += ms
        stats = eng.stats()
        rollouts += stats.rollouts
        launches += stats.kernel_launches
        lat.extend((eng.latencies_ns() / 1e6).tolist())
    clk = clocks.stop() if clocks else None
    rollouts_all = d.sum(rollouts)
    value = rollouts_all / (total_ms / 1e3)
    outs = eng.outcomes()
    exits = {k: sum(1 for o in outs if o.exit_kind == k) for k in (1, 2, 3)}

    # roofline: one extra batch through the step API with CUDA events around
    # every k_wave launch on the launch stream (the graph path above has no
    # per-kernel events); algorithmic bytes from the engine counters
    wave_ms, byte_total = profile_waves(eng, table, lo, n_total, d, sharded)

    # e2e: host problem table in → host outcomes out through the public API
    e2e = None
    if N > 1:
        from paper_2604_00510_b200._abi import TsOutcome, TsProblem

        ts, ro = [], 0
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            d.barrier()
            t0 = time.perf_counter()
            eng.load(table, lo, n_total)  # H2D of this rank's problem table
            one_step()
            eng.outcomes()  # D2H of this rank's outcomes
            ts.append(d.max(time.perf_counter() - t0))
            ro = d.sum(eng.stats().rollouts)
        e2e = {"value": ro / statistics.median(ts), "unit": UNIT,
               "h2d_bytes_per_step": ctypes.sizeof(TsProblem) * n_total,
               "d2h_bytes_per_step": ctypes.sizeof(TsOutcome) * n_total,
               "ms_per_step": 1e3 * statistics.median(ts),
               "api": "Engine.load + " + ("PeerShardedRun.run" if peer is not None else "ShardedRun.run")
                      + " + Engine.outcomes"}
    if N == 1:
        from paper_2604_00510_b200._abi import TsOutcome, TsProblem
        from paper_2604_00510_b200.engine import pinned_array

        # inputs and results live in pinned host memory (the e2e contract)
        ptable = pinned_array(TsProblem, len(table), table)
        pout = pinned_array(TsOutcome, len(table))
        ts = []
        ro = 0
        for _ in range(max(3, min(args.steps, 10))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, st = eng.run_batch_host(ptable, out=pout)
            t1 = time.perf_counter()
            ts.append(t1 - t0)
            ro = st.rollouts

        e2e = {"value": ro / statistics.median(ts), "unit": UNIT,
               "h2d_bytes_per_step": ctypes.sizeof(TsProblem) * PER_GPU,
               "d2h_bytes_per_step": ctypes.sizeof(TsOutcome) * PER_GPU,
               "ms_per_step": 1e3 * statistics.median(ts), "api": "ts_run_batch_host"}

    # exits-off throughput variant on the same seeds (every search runs its budget)
    variant = None
    if N == 1:
        eng2 = Engine(search_config(n_total, exits=False), d.local)
        eng2.load(table)
        eng2.run()
        eng2.load(table)
        flush_l2(flush)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st2 = eng2.run()
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1)
        wms2, b2 = profile_waves(eng2, table, 0, n_total, d)
        hbm, _ = peaks()
        variant = {"workload": "same 4096 searches, exits off (every search runs 128 rollouts)",
                   "value": st2.rollouts / (ms2 / 1e3), "unit": UNIT, "ms": ms2, "waves": st2.steps,
                   "wave_ms": wms2, "wave_kernel_GBs": b2 / (wms2 / 1e3) / 1e9,
                   "wave_frac": b2 / (wms2 / 1e3) / 1e9 / hbm,
                   "issue_roofline": issue_roofline(st2.rollouts / (ms2 / 1e3), st2.rollouts)}
        eng2.close()

    c3 = c3_rollout_step(table, lo, n_total, d, flush, args)
    extra = other_paths(table, flush, args) if N == 1 else {}

    cpu = cpu_baseline(n_total, args.steps, args.warmup) if (d.rank == 0 and N == 1 and not args.no_cpu) else None
    if d.rank != 0:
        eng.close()
        return None
    hbm, src = peaks()
    achieved = byte_total / (wave_ms / 1e3) / 1e9 if wave_ms > 0 else 0.0
    traffic, traffic_src = None, None
    for rnd in ("r02", "r01"):  # DRAM bytes of the same wave kernels over one batch, newest ncu capture
        path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_dram_c2_full.json")
        try:
            with open(path) as f:
                kk = json.load(f)["kernels"]
            traffic = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kk.values())
            traffic_src = os.path.relpath(path, ROOT)
            break
        except Exception:
            continue
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+u64", "data": "synthetic (reference make_workload generator, seed 0)",
        "config": config_dict(n_total, N),
        "p99_search_latency_ms": percentile(lat, 99), "p50_search_latency_ms": percentile(lat, 50),
        "rollouts_per_step": rollouts_all / args.steps, "exits": exits,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "k_wave + k_heavy (the wave phase of one batch)",
                     "peak_source": src, "algorithmic_bytes": byte_total, "wave_ms": wave_ms,
                     "traffic_note": f"ncu dram__bytes_read+write of every k_wave/k_heavy launch of one batch "
                                     f"({traffic_src}, tools/profile_round.sh on the benchmarked build), per batch "
                                     "like algorithmic_bytes; "
                                     "below the algorithmic bytes because the trees stay L2-resident",
                     "regime": "latency-bound: the boosted tail wave is sequential per search by definition"},
        "cpu_baseline": cpu, "clocks": clk, "variants": {"exits_off": variant, "c3_rollout_step": c3, **extra},
    }
    if N > 1:
        line["exchange"] = ("peer memory: ts_run_sharded (one device-driven graph per batch, counts and group "
                            "tables written into every rank's buffer over NVLink)" if peer is not None else
                            "NCCL all-gathers of counts and records per wave (ShardedRun, host-driven)")
    eng.close()
    return line


def c3_rollout_step(table, lo, n_total, d: Dist, flush, args) -> dict:
    """Config 3's shape on N GPUs: 4096 searches per GPU of a 4096*N run queue,
    M = 4 * 4096 * N (4 parallel rollouts per ungated search with virtual
    loss), exits off so every wave advances every search; `ms_per_wave` is the
    north star's "one rollout step" (max over ranks, device-timed)."""
    import torch

    from paper_2604_00510_b200.engine import Engine

    N = d.world
    eng = Engine(search_config(4 * n_total, exits=False), d.local)
    sharded, peer = None, None
    if N > 1:
        from paper_2604_00510_b200.distributed import ShardedRun

        sharded = ShardedRun(eng, d.pg, PER_GPU, n_total, torch.device("cuda", d.local),
                             host_staging=d.backend != "nccl")
        peer = peer_exchange(eng, table, lo, n_total, d)
    if N == 1:
        run = lambda: eng.run()  # noqa: E731
    elif peer is not None:
        run = lambda: peer.run().steps  # noqa: E731
    else:
        run = lambda: sharded.run()  # noqa: E731
    eng.load(table, lo, n_total)
    run()
    stream = torch.cuda.current_stream()
    ts, waves, ro = [], 0, 0
    for _ in range(max(3, min(args.steps, 5))):
        eng.load(table, lo, n_total)
        flush_l2(flush)
        torch.cuda.synchronize()
        d.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        w = run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(d.max(e0.elapsed_time(e1)))
        st = eng.stats()
        waves = st.steps if N == 1 else w
        ro = d.sum(st.rollouts)
    eng.close()
    ms = statistics.median(ts)
    return {"workload": f"c3 shape: {PER_GPU}/GPU searches of {n_total}, M={4 * n_total} (P=4), exits off",
            "value": ro / (ms / 1e3), "unit": UNIT, "ms_per_batch": ms, "waves": waves,
            "ms_per_wave": ms / max(1, waves), "rollouts_per_batch": ro}


def other_paths(table, flush, args) -> dict:
    """The other device paths of the boundary on the same 4096 problems: the
    beam-search baseline (beam.py:143-176, default BeamConfig) and the
    standalone compute_targets operator on a 32768-job run queue."""
    import numpy as np
    import torch

    from paper_2604_00510_b200._abi import TsBeamConfig, TsBeamResult, load_library
    from paper_2604_00510_b200.policy import compute_targets_arrays
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    lib = load_library()
    out = {}
    n = len(table)
    stream = torch.cuda.current_stream()
    dprob = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).cuda()
    dres = torch.empty(n * ctypes.sizeof(TsBeamResult), dtype=torch.uint8, device="cuda")
    cfg = TsBeamConfig(8, 4, 16, 1, 1, 0, 0.5)
    launch = lambda: lib.ts_beam_search(ctypes.byref(cfg), ctypes.c_void_p(dprob.data_ptr()), n,  # noqa: E731
                                        ctypes.c_void_p(dres.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
    for _ in range(3):
        launch()
    ts = []
    for _ in range(max(5, args.steps // 5)):
        flush_l2(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res = (TsBeamResult * n).from_buffer_copy(dres.cpu().numpy().tobytes())
    steps = sum(r.steps for r in res)
    ms = statistics.median(ts)
    out["beam_baseline"] = {"workload": f"beam.py run_beam_search, BeamConfig() (8 beams x 4 samples, max depth 16), "
                                        f"{n} c2 problems", "value": n / (ms / 1e3), "unit": "searches/s",
                            "ms": ms, "beam_steps": steps, "kernel": "k_beam (one warp per problem)"}
    # standalone compute_targets on a 32768-job run queue (unsorted fractional arrivals)
    m = 32768
    rng = np.random.default_rng(0)
    arr = torch.tensor(rng.uniform(0, 100, m), device="cuda")
    best = torch.tensor(rng.choice([0.0, 0.3, 0.46, 0.6], m), device="cuda")
    comp = torch.tensor(rng.integers(0, 5, m), dtype=torch.int32, device="cuda")
    ids = torch.arange(m, dtype=torch.int64, device="cuda")
    sc = SchedulerConfig(max_concurrency=4 * m)
    for _ in range(3):
        compute_targets_arrays(arr, best, comp, ids, 100.0, sc, 0.5)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, info = compute_targets_arrays(arr, best, comp, ids, 100.0, sc, 0.5)
        ts.append(time.perf_counter() - t0)
    out["compute_targets_standalone"] = {"workload": f"compute_targets on {m} running jobs, M={4 * m}",
                                         "value": 1e3 * statistics.median(ts), "unit": "ms per call (host-timed, "
                                         "includes the status read-back)", "kernel_launches": info.kernel_launches}
    return out


# --------------------------------------------------------------------------- CPU
def oracle_batches(n_total: int, steps: int, warmup: int, threads: int):
    """The reference algorithm (the C restatement in oracle/, test
    infrastructure) over the whole n_total-search batch on `threads` host
    threads: `warmup` untimed batches, then `steps` timed ones.  Both arms
    time the CPU this way (same batch, warm-up and repetitions; median)."""
    from oracle import oracle
    from paper_2604_00510_b200.backend import problem_table

    oracle.build()
    t = problem_table(workload(n_total))
    cfg = search_config(n_total).to_c()
    for _ in range(warmup):
        oracle.OracleRun(t, cfg, threads=threads).close()
    times, ro, lat = [], 0, []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = oracle.OracleRun(t, cfg, threads=threads)
        times.append(time.perf_counter() - t0)
        ro = r.stats.rollouts
        lat.extend((r.latencies_s() * 1e3).tolist())
        r.close()
    med = statistics.median(times)
    return {"value": ro / med, "ms_per_step": 1e3 * med, "rollouts_per_step": ro,
            "p99_search_latency_ms": percentile(lat, 99)}


def python_reference_sample(n: int = 64):
    """The UNMODIFIED Python reference (treeserve, installed into baseline/_ref)
    on the first n searches of the same workload, composed into waves only of
    reference calls (tests/golden/wave_ref.py); one host core.  None when the
    reference is not importable on this machine."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    try:
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import wave_ref
        from treeserve.backend import Difficulty, make_workload
        from treeserve.scheduler import SchedulerConfig as RefSched
    except Exception as e:  # pragma: no cover - reference absent
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.pop(0)
    specs = make_workload(PER_GPU, (0.6, 0.25, 0.15), 0, branching=BRANCH,
                          depth_ranges={d: (BASE, BASE) for d in Difficulty})[:n]
    t0 = time.perf_counter()
    recs, info = wave_ref.run_waves(specs, sched=RefSched(max_concurrency=n), rollout_budget=BUDGET,
                                    depth_cap=DEPTH_CAP, expand_width=WIDTH)
    dt = time.perf_counter() - t0
    ro = sum(r["rollouts_completed"] for r in recs)
    return {"value": ro / dt, "unit": UNIT, "cores": 1, "rollouts": ro, "s": dt,
            "sample": f"first {n} searches of the same workload, M={n}, unmodified Python reference"}


def cpu_baseline(n_total: int, steps: int, warmup: int):
    """The CPU oracle timed like the reference arm, plus one-core and
    Python-reference samples for context."""
    threads = os.cpu_count() or 1
    full = oracle_batches(n_total, steps, warmup, threads)
    one = oracle_batches(n_total, max(1, min(steps, 3)), 1, 1)
    return {"value": full["value"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"the whole {n_total}-search batch per step, {warmup} warm-up + {steps} timed batches, "
                      f"median ({full['ms_per_step']:.1f} ms per batch)",
            "p99_search_latency_ms": full["p99_search_latency_ms"],
            "single_core_value": one["value"],
            "python_reference": python_reference_sample()}


def bench_reference(args):
    """--impl reference: the reference algorithm on the host cores (oracle port;
    the reference is pure Python and is not what a CPU deployment of this path
    would time) over the same batch as our arm, all host threads."""
    N = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    n_total = PER_GPU * N
    threads = os.cpu_count() or 1
    r = oracle_batches(n_total, args.steps, args.warmup, threads)
    return {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64",
        "data": "synthetic (reference make_workload generator, seed 0)",
        "config": config_dict(n_total, N),
        "p99_search_latency_ms": r["p99_search_latency_ms"], "rollouts_per_step": r["rollouts_per_step"],
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"the whole {n_total}-search batch per step, median of {args.steps}"},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: re-exec this script
    as N ranks (one process per GPU) on 127.0.0.1 and pass rank 0's line on."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        print(json.dumps(bench_reference(args)))
        return
    if world is None and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch N ranks for --gpus N")
    import __graft_entry__

    __graft_entry__.build()
    d = Dist()
    d.init()
    line = bench_ours(args, d)
    if line is not None:
        print(json.dumps(line))
    if d.pg:
        d.pg.destroy_process_group()


if __name__ == "__main__":
    main()
