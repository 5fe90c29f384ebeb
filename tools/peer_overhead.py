"""Per-wave cost of the sharded loop over peer memory (ts_run_sharded) with W
ranks emulated on one GPU (one engine, stream and host thread per rank).

    python tools/peer_overhead.py [W=8] [per_rank=4096] [mt_min]

Workload: config 3's shape, per_rank searches per rank of a W*per_rank run
queue, M = 4 * W * per_rank (P = 4 per ungated search), exits off.  For rank 0
it prints, per wave, from device %globaltimer stamps: the exchange (counts
phase start -> every rank's records in) and compute_targets (records in ->
targets done), i.e. the work between the previous wave's kernels and this
wave's.  All ranks share the GPU, so a rank's records can arrive late because
the other ranks' waves hold the SMs; the "exchange" column is therefore an
upper bound of what one rank per GPU sees.  The W=1 line is the same loop with
a one-rank run queue (no peer), for comparison."""
import os
import statistics
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.distributed import connect_in_process  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402


def run(W, per, reps=3):
    n = W * per
    specs = bench.workload(n)
    cfg = bench.search_config(4 * n, exits=False)
    engines = []
    for r in range(W):
        e = Engine(cfg, 0, stream=torch.cuda.Stream())
        e.load(problem_table(specs[r * per:(r + 1) * per]), r * per, n)
        engines.append(e)
    torch.cuda.synchronize()
    connect_in_process(engines)
    rows = []
    for rep in range(reps):
        if rep:
            for r, e in enumerate(engines):
                e.load(problem_table(specs[r * per:(r + 1) * per]), r * per, n)
            torch.cuda.synchronize()
        stats = [None] * W
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()

        def go(r):
            stats[r] = engines[r].run_sharded()

        th = [threading.Thread(target=go, args=(r,)) for r in range(W)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        t1.record()
        torch.cuda.synchronize()
        waves = stats[0].steps
        st = engines[0].px_times(waves).astype(np.int64)
        xch = (st[:, 1] - st[:, 0]) / 1e3
        sch = (st[:, 2] - st[:, 1]) / 1e3
        period = np.diff(st[:, 0]) / 1e3
        rows.append({"waves": waves, "rollouts": sum(s.rollouts for s in stats),
                     "exchange_us": float(np.median(xch)), "targets_us": float(np.median(sch)),
                     "period_us": float(np.median(period)) if len(period) else 0.0})
    for e in engines:
        e.close()
    r = rows[-1]
    print(f"W={W} per_rank={per} n_global={n}: waves {r['waves']}, rank-0 medians per wave: "
          f"exchange {r['exchange_us']:.1f} us, compute_targets {r['targets_us']:.1f} us, "
          f"wave period {r['period_us']:.1f} us (all {W} ranks' waves share this GPU)", flush=True)
    return r


if __name__ == "__main__":
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    per = int(sys.argv[2]) if len(sys.argv) > 2 else bench.PER_GPU
    if len(sys.argv) > 3:
        os.environ["TS_MT_MIN"] = sys.argv[3]
    run(1, per)
    run(W, per)
