"""Per-step device time of a graph-mode batch (from the %globaltimer stamps
k_sched writes at the start of every step).  Diagnostic."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402

for exits in (True, False):
    table = problem_table(bench.workload(bench.PER_GPU))
    eng = Engine(bench.search_config(bench.PER_GPU, exits=exits), 0)
    for rep in range(3):
        eng.load(table)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = eng.run()
        e1.record()
        torch.cuda.synchronize()
    t = eng.step_times(st.steps + 2).astype("int64")
    d = [(t[i + 1] - t[i]) / 1e3 for i in range(min(st.steps + 1, 12))]
    print("exits" if exits else "exits_off", f"total {e0.elapsed_time(e1):.3f} ms, steps {st.steps}, "
          f"first-stamp-to-last {(t[st.steps] - t[0]) / 1e6:.3f} ms; step us:", [round(x, 1) for x in d])
    eng.close()
