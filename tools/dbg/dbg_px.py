import sys, os, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
from paper_2604_00510_b200 import backend as B
from paper_2604_00510_b200.config import SearchConfig
from paper_2604_00510_b200.engine import Engine
from paper_2604_00510_b200.scheduler import SchedulerConfig
from paper_2604_00510_b200.distributed import connect_in_process
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
specs = B.make_workload(n, (0.6, 0.25, 0.15), 11, branching=4, depth_ranges={d: (7, 7) for d in B.Difficulty})
cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=2 * n), rollout_budget=16, depth_cap=8, expand_width=4)
tab = B.problem_table(specs)
e = Engine(cfg, 0, stream=torch.cuda.Stream())
e.load(tab)
torch.cuda.synchronize()
connect_in_process([e])
print("connected", flush=True)
t = time.time()
st = e.run_sharded(max_steps=int(sys.argv[2]) if len(sys.argv) > 2 else 50)
print("steps", st.steps, "rollouts", st.rollouts, "t", time.time() - t, flush=True)
print(e.px_times(min(st.steps, 8)))
c = e.stats()
print("finished", c.finished)
