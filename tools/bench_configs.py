"""All five BASELINE.json configs on one B200, each with the CPU oracle timed
beside it on a bounded sample.  Writes one JSON object per config.

    python tools/bench_configs.py [--out profiles/rNN_configs.json] [--only c1,c2,...]

c1  reference CPU demo: 64 searches, b=4, depth 8, 32 rollouts, PE+NE+boost, M=64
c2  4096 searches, b=4, depth 16, 128 rollouts, PE+NE+boost, M=4096 (also exits off)
c3  one GPU's shard of config 3: 4096 searches, M = 4x4096 (4 parallel rollouts per
    ungated search with virtual loss), exits off so every search runs its budget
c4  deep-tree stress: 1024 searches, b=8, depth 32, 1024 rollouts, stagnation profile
c5  serving: 65536 Poisson arrivals (reference generator, step-quantised), M=4096,
    arms pe (positive exit only, no boosting) vs pe_ne_boost; p99 arrival→exit latency
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2604_00510_b200 import backend as B  # noqa: E402
from paper_2604_00510_b200 import keyed  # noqa: E402
from paper_2604_00510_b200.config import SearchConfig  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402
from paper_2604_00510_b200.scheduler import SchedulerConfig  # noqa: E402

MIX = (0.6, 0.25, 0.15)
THREADS = os.cpu_count() or 1


def pct(vals, p):
    v = sorted(vals)
    if not v:
        return 0.0
    return v[max(1, math.ceil(p / 100 * len(v))) - 1]


def gpu_run(table, cfg, arrivals=None, reps=3):
    """Timed ts_run (CUDA events) of a loaded batch; best of `reps`."""
    eng = Engine(cfg, 0)
    best = None
    for _ in range(reps + 1):
        eng.load(table)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = eng.run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if best is None or ms < best[0]:
            outs = eng.outcomes()
            lat = eng.latencies_ns() / 1e6
            if arrivals is not None:
                times = eng.step_times(st.steps + 2).astype("float64") / 1e6
                adm = [o.admit_step for o in outs]
                lat = [l + (times[a] - times[arr]) for l, a, arr in zip(lat.tolist(), adm, arrivals)]
            else:
                lat = lat.tolist()
            best = (ms, st, outs, lat)
    eng.close()
    ms, st, outs, lat = best
    return {"ms": ms, "rollouts": st.rollouts, "launched": st.launched, "waves": st.steps, "nodes": st.nodes,
            "rollouts_per_s": st.rollouts / (ms / 1e3), "p50_latency_ms": pct(lat, 50),
            "p99_latency_ms": pct(lat, 99),
            "exits": {k: sum(1 for o in outs if o.exit_kind == c) for k, c in
                      (("positive", 1), ("negative", 2), ("budget", 3))}}, outs


def cpu_run(table, cfg, arrivals=None):
    t0 = time.perf_counter()
    r = oracle.OracleRun(table, cfg.to_c(), threads=THREADS)
    dt = time.perf_counter() - t0
    lat = (r.latencies_s() * 1e3).tolist()
    res = {"s": dt, "rollouts": r.stats.rollouts, "rollouts_per_s": r.stats.rollouts / dt, "threads": THREADS,
           "p99_latency_ms": pct(lat, 99), "waves": r.steps}
    outs = list(r.outcomes)
    r.close()
    return res, outs


def parity(g, c, n):
    keys = ("exit_kind", "rollouts_completed", "tokens_generated", "best_score", "exit_step", "launched", "nodes")
    return all(getattr(g[i], k) == getattr(c[i], k) for i in range(n) for k in keys)


def cfg_of(M, budget, cap, width, pe=True, ne=True, boost=True):
    return SearchConfig(scheduler=SchedulerConfig(max_concurrency=M, boosting_enabled=boost), rollout_budget=budget,
                        depth_cap=cap, expand_width=width, positive_exit=pe, negative_exit=ne)


def c1():
    specs = B.make_workload(64, MIX, 0, branching=4, depth_ranges={d: (7, 7) for d in B.Difficulty})
    t = B.problem_table(specs)
    cfg = cfg_of(64, 32, 8, 4)
    g, go = gpu_run(t, cfg)
    c, co = cpu_run(t, cfg)
    return {"gpu": g, "cpu": c, "cpu_sample": "all 64", "parity_vs_oracle": parity(go, co, 64)}


def c2(exits=True):
    specs = B.make_workload(4096, MIX, 0, branching=4, depth_ranges={d: (15, 15) for d in B.Difficulty})
    t = B.problem_table(specs)
    cfg = cfg_of(4096, 128, 16, 4, exits, exits)
    g, go = gpu_run(t, cfg)
    n = 4096 if exits else 512
    cs = B.problem_table(specs[:n])
    c, co = cpu_run(cs, cfg_of(n, 128, 16, 4, exits, exits))
    return {"gpu": g, "cpu": c, "cpu_sample": f"first {n} searches, M={n}",
            "parity_vs_oracle": parity(go, co, n) if n == 4096 else None}


def c3():
    specs = B.make_workload(4096, MIX, 0, branching=4, depth_ranges={d: (15, 15) for d in B.Difficulty})
    t = B.problem_table(specs)
    g, go = gpu_run(t, cfg_of(4 * 4096, 128, 16, 4, False, False))
    cs = B.problem_table(specs[:256])
    c, co = cpu_run(cs, cfg_of(4 * 256, 128, 16, 4, False, False))
    return {"gpu": g, "cpu": c, "cpu_sample": "first 256 searches, M=1024", "note": "one GPU's shard of config 3"}


def c4(n=1024):
    specs = [B.make_problem(f"s{i:04d}", keyed.mix(0, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                            B.stagnation_profile()) for i in range(n)]
    t = B.problem_table(specs)
    g, go = gpu_run(t, cfg_of(n, 1024, 32, 8), reps=1)
    cs = B.problem_table(specs[:16])
    c, co = cpu_run(cs, cfg_of(16, 1024, 32, 8))
    return {"gpu": g, "cpu": c, "cpu_sample": "first 16 searches, M=16"}


def c5(n=65536, per_wave=2800.0, M=4096):
    specs = B.make_workload(n, MIX, 20260810)
    arrivals = B.serving_arrival_steps(n, 1.0, 20260810, 1.0 / per_wave)
    t = B.problem_table(specs, arrivals)
    out = {"arrivals_per_wave": per_wave, "M": M, "arrival_waves": arrivals[-1] + 1}
    for arm, pe, ne, boost in (("pe", True, False, False), ("pe_ne_boost", True, True, True)):
        cfg = cfg_of(M, 32, 16, 4, pe, ne, boost)
        g, go = gpu_run(t, cfg, arrivals, reps=1)
        ns = 8192
        cs = B.problem_table(specs[:ns], arrivals[:ns])
        c, co = cpu_run(cs, cfg)
        out[arm] = {"gpu": g, "cpu": c, "cpu_sample": f"first {ns} arrivals, same M",
                    "parity_vs_oracle_first_8192": None}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="c1,c2,c2off,c3,c4,c5")
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "cpu_threads": THREADS}
    for name in args.only.split(","):
        t0 = time.time()
        if name == "c2off":
            res[name] = c2(False)
        else:
            res[name] = globals()[name]()
        res[name]["wall_s"] = round(time.time() - t0, 1)
        print(name, json.dumps(res[name]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
