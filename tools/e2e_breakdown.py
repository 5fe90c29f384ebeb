"""Where the end-to-end batch time (bench.py's e2e: ts_run_batch_host from
pinned host buffers, host clock) goes beyond the device batch: host-timed
load (H2D + k_init + sync), run (graph + outcome counters + sync), the whole
call, and a device-event bracket of the call."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200._abi import TsOutcome, TsProblem  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine, pinned_array  # noqa: E402

table = problem_table(bench.workload(bench.PER_GPU))
eng = Engine(bench.search_config(bench.PER_GPU), 0)
ptable = pinned_array(TsProblem, len(table), table)
pout = pinned_array(TsOutcome, len(table))
res = {k: [] for k in ("call", "call_dev", "load", "run", "load_run")}
for it in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run_batch_host(ptable, out=pout)
    res["call"].append(time.perf_counter() - t0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    eng.run_batch_host(ptable, out=pout)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    res["call_dev"].append(e0.elapsed_time(e1) / 1e3)
    t0 = time.perf_counter()
    eng.load(ptable)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng.run()
    t2 = time.perf_counter()
    res["load"].append(t1 - t0)
    res["run"].append(t2 - t1)
    res["load_run"].append(t2 - t0)
print({k: round(1e3 * statistics.median(v[5:]), 4) for k, v in res.items()}, "ms (median)")
