import sys, os
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_2604_00510_b200.backend import problem_table
from paper_2604_00510_b200.engine import Engine
t = problem_table(bench.workload(4096))
e = Engine(bench.search_config(4096), 0)
for i in range(3):
    e.load(t)
    st = e.run()
    print("steps", st.steps, "launches", st.kernel_launches, flush=True)
