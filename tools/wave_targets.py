"""Per-wave target distribution of the headline batch (how many searches run
in the pipelined mode, their P): diagnostics for the heavy waves."""
import collections
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
n = bench.PER_GPU
eng.load(table)
counts = torch.zeros(3, dtype=torch.int64, device="cuda")
recs = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
for step in range(6):
    eng.step_counts(step, counts.data_ptr())
    eng.step_admit(step, counts.data_ptr(), 1, 0)
    eng.step_records(step, recs.data_ptr())
    eng.step_targets(step, recs.data_ptr())
    t = [x for x in eng.read_targets() if x > 0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step_wave(step)
    e1.record()
    torch.cuda.synchronize()
    if not t:
        break
    h = collections.Counter(min(x, 200) for x in t)
    print(f"wave {step}: running {len(t)}, P>=8: {sum(1 for x in t if x >= 8)}, max P {max(t)}, "
          f"sum P {sum(t)}, {e0.elapsed_time(e1) * 1e3:.0f} us, P histogram {sorted(h.items())[:12]}", flush=True)
