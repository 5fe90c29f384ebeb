"""Warm per-kernel timings of one batch, step by step (CUDA events on the
launch stream).  Diagnostic only.   python tools/step_timing.py full|exits_off"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402


def main(mode):
    table = problem_table(bench.workload(bench.PER_GPU))
    eng = Engine(bench.search_config(bench.PER_GPU, exits=(mode == "full")), 0)
    n = bench.PER_GPU
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    recs = torch.zeros(n * 16, dtype=torch.uint8, device="cuda")
    for rep in range(2):
        eng.load(table)
        torch.cuda.synchronize()
        names = ["counts", "admit", "records", "targets", "wave"]
        tot = {k: 0.0 for k in names}
        ev = []
        step = 0
        while True:
            es = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            es[0].record()
            eng.step_counts(step, counts.data_ptr()); es[1].record()
            eng.step_admit(step, counts.data_ptr(), 1, 0); es[2].record()
            eng.step_records(step, recs.data_ptr()); es[3].record()
            eng.step_targets(step, recs.data_ptr()); es[4].record()
            eng.step_wave(step); es[5].record()
            ev.append(es)
            if rep == 1 and mode == "full" and step < 6:
                torch.cuda.synchronize()
                st = eng.stats()
                print(f"  after wave {step}: launched={st.launched} rollouts={st.rollouts} nodes={st.nodes} "
                      f"levels={st.select_levels} scored={st.children_scored} path={st.path_nodes}")
            step += 1
            if step % 8 == 0:
                torch.cuda.synchronize()
                if int(counts[2].item()) == 0:
                    break
        torch.cuda.synchronize()
        per_wave = []
        for es in ev:
            for i, k in enumerate(names):
                tot[k] += es[i].elapsed_time(es[i + 1])
            per_wave.append(es[4].elapsed_time(es[5]))
        span = ev[0][0].elapsed_time(ev[-1][5])
        st = eng.stats()
        print(mode, "rep", rep, "steps", step, "waves", st.steps, "rollouts", st.rollouts, f"span {span:.3f} ms",
              " ".join(f"{k}={v:.3f}" for k, v in tot.items()))
        if mode == "full":
            print("  per-wave ms:", [round(x, 3) for x in per_wave[:8]])
        else:
            print("  wave ms first/mid/last:", round(per_wave[0], 4), round(per_wave[len(per_wave) // 2], 4),
                  round(per_wave[st.steps - 1], 4))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "full")
