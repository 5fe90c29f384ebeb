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

    sharded = None
    if N > 1:
        from paper_2604_00510_b200.distributed import ShardedRun

        sharded = ShardedRun(eng, d.pg, PER_GPU, n_total, torch.device("cuda", d.local),
                             host_staging=d.backend != "nccl")

    def one_step():
        if N == 1:
            eng.run()
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
            sharded.run()
            eng.outcomes()  # D2H of this rank's outcomes
            ts.append(d.max(time.perf_counter() - t0))
            ro = d.sum(eng.stats().rollouts)
        e2e = {"value": ro / statistics.median(ts), "unit": UNIT,
               "h2d_bytes_per_step": ctypes.sizeof(TsProblem) * n_total,
               "d2h_bytes_per_step": ctypes.sizeof(TsOutcome) * n_total,
               "ms_per_step": 1e3 * statistics.median(ts), "api": "Engine.load + ShardedRun.run + Engine.outcomes"}
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
                   "wave_frac": b2 / (wms2 / 1e3) / 1e9 / hbm}
        eng2.close()

    extra = other_paths(table, flush, args) if N == 1 else {}

    cpu = cpu_baseline(PER_GPU, n_total) if (d.rank == 0 and N == 1 and not args.no_cpu) else None
    if d.rank != 0:
        eng.close()
        return None
    hbm, src = peaks()
    achieved = byte_total / (wave_ms / 1e3) / 1e9 if wave_ms > 0 else 0.0
    traffic = None
    try:  # DRAM bytes of the same wave kernels over one batch, from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "r01_ncu_dram_c2_full.json")) as f:
            kk = json.load(f)["kernels"]
        traffic = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in kk.values())
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+u64", "data": "synthetic (reference make_workload generator, seed 0)",
        "config": {"workload": f"c2: {PER_GPU}/GPU searches, b={BRANCH}, depth {BASE + 1}, budget {BUDGET}, "
                               f"PE+NE+boost, M={n_total}",
                   "searches": n_total, "branching": BRANCH, "depth": BASE + 1, "rollout_budget": BUDGET,
                   "max_concurrency": n_total, "parallelism": f"search-sharded x{N}",
                   "l2": "flushed (512 MiB write) before every timed step; node pool > L2"},
        "p99_search_latency_ms": percentile(lat, 99), "p50_search_latency_ms": percentile(lat, 50),
        "rollouts_per_step": rollouts_all / args.steps, "exits": exits,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "k_wave + k_heavy (the wave phase of one batch)",
                     "peak_source": src, "algorithmic_bytes": byte_total, "wave_ms": wave_ms,
                     "traffic_note": "ncu dram__bytes_read+write of every k_wave/k_heavy launch of one batch "
                                     "(profiles/r01_ncu_dram_c2_full.json), per batch like algorithmic_bytes; "
                                     "below the algorithmic bytes because the trees stay L2-resident",
                     "regime": "latency-bound: the boosted tail wave is sequential per search by definition"},
        "cpu_baseline": cpu, "clocks": clk, "variants": {"exits_off": variant, **extra},
    }
    eng.close()
    return line


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
def cpu_baseline(per_gpu: int, n_total: int, target_s: float = 12.0):
    """The C oracle (a restatement of the reference, oracle/) on the host cores:
    a bounded sample of the same workload (the first S searches, M scaled)."""
    from oracle import oracle
    from paper_2604_00510_b200.backend import problem_table

    threads = os.cpu_count() or 1
    specs = workload(n_total)
    sample = 256
    while True:
        t = problem_table(specs[:sample])
        cfg = search_config(sample).to_c()
        t0 = time.perf_counter()
        r = oracle.OracleRun(t, cfg, threads=threads)
        dt = time.perf_counter() - t0
        ro = r.stats.rollouts
        lat = (r.latencies_s() * 1e3).tolist()
        r.close()
        if dt > target_s / 4 or sample >= per_gpu:
            break
        sample = min(per_gpu, sample * 4)
    # one host core on the same sample (single core and all cores)
    t1 = time.perf_counter()
    r1 = oracle.OracleRun(t, cfg, threads=1)
    dt1 = time.perf_counter() - t1
    ro1 = r1.stats.rollouts
    r1.close()
    return {"value": ro / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {sample} of the {per_gpu} searches, M={sample}, same budget/exits/boosting; "
                      f"{ro} rollouts in {dt:.2f} s",
            "p99_search_latency_ms": percentile(lat, 99),
            "single_core_value": ro1 / dt1}


def bench_reference(args):
    """--impl reference: the reference algorithm on the host cores (oracle port;
    the Python reference itself is not present on the GPU box)."""
    from oracle import oracle
    from paper_2604_00510_b200.backend import problem_table

    oracle.build()
    threads = os.cpu_count() or 1
    specs = workload(PER_GPU)
    sample = PER_GPU  # the whole config-2 batch: ~30 ms per step on 16 host threads
    t = problem_table(specs[:sample])
    cfg = search_config(sample).to_c()
    for _ in range(args.warmup):
        oracle.OracleRun(t, cfg, threads=threads).close()
    times, ro, lat = [], 0, []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle.OracleRun(t, cfg, threads=threads)
        times.append(time.perf_counter() - t0)
        ro += r.stats.rollouts
        lat.extend((r.latencies_s() * 1e3).tolist())
        r.close()
    value = ro / sum(times)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": f"c2: {PER_GPU}/GPU searches, b={BRANCH}, depth {BASE + 1}, budget {BUDGET}, "
                               f"PE+NE+boost, M={PER_GPU}", "searches": sample},
        "p99_search_latency_ms": percentile(lat, 99),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"the full batch of {sample} searches per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        print(json.dumps(bench_reference(args)))
        return
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
