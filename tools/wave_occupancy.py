"""Exits-off wave throughput of c2 / c3-shard / c4 for the library in
TS_LIB_PATH (occupancy experiments; best of 3 ts_run, CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2604_00510_b200 import backend as B  # noqa: E402
from paper_2604_00510_b200.config import SearchConfig  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402
from paper_2604_00510_b200.scheduler import SchedulerConfig  # noqa: E402

MIX = (0.6, 0.25, 0.15)


def run(table, cfg):
    eng = Engine(cfg, 0)
    best = None
    for _ in range(4):
        eng.load(table)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = eng.run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    r = st.rollouts
    eng.close()
    return best, r


D15 = {d: (15, 15) for d in B.Difficulty}
c2 = B.problem_table(B.make_workload(4096, MIX, 0, branching=4, depth_ranges=D15))
for name, cfg in [
    ("c2 exits off", SearchConfig(scheduler=SchedulerConfig(max_concurrency=4096), rollout_budget=128, depth_cap=16,
                                  expand_width=4, positive_exit=False, negative_exit=False)),
    ("c3 shard P=4", SearchConfig(scheduler=SchedulerConfig(max_concurrency=4 * 4096), rollout_budget=128,
                                  depth_cap=16, expand_width=4, positive_exit=False, negative_exit=False)),
    ("c2 full", SearchConfig(scheduler=SchedulerConfig(max_concurrency=4096), rollout_budget=128, depth_cap=16,
                             expand_width=4)),
]:
    ms, r = run(c2, cfg)
    print(f"{os.path.basename(os.environ.get('TS_LIB_PATH', 'default'))} {name}: {ms:.3f} ms, {r / ms / 1e3:.1f} M rollouts/s",
          flush=True)
specs = [B.make_problem(f"s{i}", B.keyed.mix(0, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                        B.stagnation_profile()) for i in range(1024)]
c4 = B.problem_table(specs)
ms, r = run(c4, SearchConfig(scheduler=SchedulerConfig(max_concurrency=1024), rollout_budget=256, depth_cap=32,
                             expand_width=8))
print(f"{os.path.basename(os.environ.get('TS_LIB_PATH', 'default'))} c4 (budget 256): {ms:.3f} ms, {r / ms / 1e3:.1f} M rollouts/s", flush=True)
