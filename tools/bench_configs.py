"""Every BASELINE.json config at its STATED size on one B200, with the CPU
oracle run over the same whole batch on all host threads: the oracle run is
both the parity check (every outcome field and best path, bit for bit) and the
CPU baseline.  Writes one JSON object per config.

    python tools/bench_configs.py [--out profiles/rNN_configs.json] [--only c1,c2,...]

c1      reference CPU demo: 64 searches, b=4, depth 8, 32 rollouts, PE+NE+boost, M=64
c2      4096 searches, b=4, depth 16, 128 rollouts, PE+NE+boost, M=4096
c2off   the same, exits off (every search runs its budget)
c3      32,768 searches, M = 4 x 32,768 (P = 4 per ungated search, virtual loss), PE+NE+boost
c3off   the same, exits off
c4      deep-tree stress: 1024 searches, b=8, depth 32, 1024 rollouts, stagnation profile
c5_*    serving: 65,536 Poisson arrivals (reference generator, step-quantised), M=4096,
        arms pe (positive exit only, no boosting) and pe_ne_boost; p99 arrival→exit latency
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
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402

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


OUT_KEYS = ("exit_kind", "rollouts_completed", "tokens_generated", "best_score", "best_len", "solved",
            "exit_step", "admit_step", "launched", "cancelled", "nodes", "status")


def parity(g, c, n):
    """Every outcome field and best path of all n searches, bit for bit."""
    return all(getattr(g[i], k) == getattr(c[i], k) for i in range(n) for k in OUT_KEYS) and all(
        bytes(g[i].best_path[: g[i].best_len]) == bytes(c[i].best_path[: c[i].best_len]) for i in range(n))


def run_config(name, reps=3):
    """A BASELINE config at its stated size (tests/test_configs_gpu.config_case):
    the engine's timed batch, and the oracle over the WHOLE batch on all host
    threads, which is both the parity check and the CPU baseline."""
    from test_configs_gpu import config_case

    specs, t, cfg = config_case(name)
    arrivals = [int(p.arrival_step) for p in t] if name.startswith("c5") else None
    g, go = gpu_run(t, cfg, arrivals, reps=reps)
    c, co = cpu_run(t, cfg)
    n = len(specs)
    return {"searches": n, "M": cfg.scheduler.max_concurrency, "gpu": g, "cpu": c,
            "cpu_sample": f"the whole batch ({n} searches) on {THREADS} threads",
            "parity_vs_oracle": parity(go, co, n), "waves_match": g["waves"] == c["waves"],
            "speedup": c["s"] * 1e3 / g["ms"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="c1,c2,c2off,c3,c3off,c4,c5_pe,c5_pe_ne_boost")
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "cpu_threads": THREADS}
    for name in args.only.split(","):
        t0 = time.time()
        res[name] = run_config(name, reps=1 if name in ("c3", "c3off", "c4") else 3)
        res[name]["wall_s"] = round(time.time() - t0, 1)
        print(name, json.dumps(res[name]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
