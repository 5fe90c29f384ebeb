"""Short single-GPU driver for ncu captures (never a bench number).

    python tools/prof_driver.py full|exits_off|both [graph]

Default drives the waves through the step API (one kernel launch per
scheduler phase and per wave, so ncu sees every k_wave); "graph" uses ts_run.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402


def stepwise(eng, n):
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    recs = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    step = 0
    while True:
        eng.step_counts(step, counts.data_ptr())
        torch.cuda.synchronize()
        if int(counts[2].item()) == 0:
            return
        eng.step_admit(step, counts.data_ptr(), 1, 0)
        eng.step_records(step, recs.data_ptr())
        eng.step_targets(step, recs.data_ptr())
        eng.step_wave(step)
        step += 1


def main(mode, graph):
    table = problem_table(bench.workload(bench.PER_GPU))
    modes = ["full", "exits_off"] if mode == "both" else [mode]
    for m in modes:
        eng = Engine(bench.search_config(bench.PER_GPU, exits=(m == "full")), 0)
        eng.load(table)
        if graph:
            eng.run()
        else:
            stepwise(eng, len(table))
        st = eng.stats()
        print(m, "waves", st.steps, "rollouts", st.rollouts, "launches", st.kernel_launches, flush=True)
        eng.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "both", len(sys.argv) > 2 and sys.argv[2] == "graph")
