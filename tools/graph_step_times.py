"""Per-step device timestamps of the CUDA-graph step loop (ts_run) for the
headline batch: the duration of each step (k_sched + the wave kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402

table = problem_table(bench.workload(bench.PER_GPU))
eng = Engine(bench.search_config(bench.PER_GPU), 0)
tot = []
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
for rep in range(12):
    eng.load(table)
    if flush is not None:  # as bench.py: L2 flushed before every timed batch
        bench.flush_l2(flush)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = eng.run()
    e1.record()
    torch.cuda.synchronize()
    tot.append(e0.elapsed_time(e1))
tot = sorted(tot[2:])
print(os.path.basename(os.environ.get("TS_LIB_PATH", "default")), "batch ms min %.4f median %.4f" % (tot[0], tot[len(tot) // 2]))
t = eng.step_times(st.steps + 1).astype("int64")
d = [(t[i + 1] - t[i]) / 1e3 for i in range(st.steps - 1 + 1) if t[i + 1] > 0]
print("total ms", e0.elapsed_time(e1), "steps", st.steps, "step durations us", [round(x, 1) for x in d])
lat = eng.latencies_ns()
print("max latency us", lat.max() / 1e3)
