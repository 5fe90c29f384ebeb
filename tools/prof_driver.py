"""Short single-GPU driver for ncu captures (never a bench number).

    python tools/prof_driver.py full|exits_off|both
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402


def main(mode):
    table = problem_table(bench.workload(bench.PER_GPU))
    modes = ["full", "exits_off"] if mode == "both" else [mode]
    for m in modes:
        eng = Engine(bench.search_config(bench.PER_GPU, exits=(m == "full")), 0)
        eng.load(table)
        st = eng.run()
        print(m, "waves", st.steps, "rollouts", st.rollouts, "wave_ms", round(st.wave_ms, 3), "launches",
              st.kernel_launches, flush=True)
        eng.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "both")
