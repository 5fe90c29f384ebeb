"""Config-4 (deep stress) batch through the step API for ncu captures (never a bench number)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2604_00510_b200 import backend as B  # noqa: E402
from paper_2604_00510_b200.config import SearchConfig  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402
from paper_2604_00510_b200.scheduler import SchedulerConfig  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 120
specs = [B.make_problem(f"s{i}", B.keyed.mix(0, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                        B.stagnation_profile()) for i in range(1024)]
eng = Engine(SearchConfig(scheduler=SchedulerConfig(max_concurrency=1024), rollout_budget=1024, depth_cap=32,
                          expand_width=8), 0)
eng.load(B.problem_table(specs))
counts = torch.zeros(3, dtype=torch.int64, device="cuda")
recs = torch.zeros(1024 * 16, dtype=torch.uint8, device="cuda")
for step in range(steps):
    eng.step_counts(step, counts.data_ptr())
    eng.step_admit(step, counts.data_ptr(), 1, 0)
    eng.step_records(step, recs.data_ptr())
    eng.step_targets(step, recs.data_ptr())
    eng.step_wave(step)
torch.cuda.synchronize()
print("c4 steps", steps, "rollouts", eng.stats().rollouts)
