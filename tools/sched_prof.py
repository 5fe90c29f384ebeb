"""Where the per-wave time of the CUDA-graph loop goes (diagnostics build
lib/libtreeserve_b200_sprof.so, -DTS_SCHED_PROF; %globaltimer stamps in
k_sched, targets_block and the wave kernels).

    nvcc <build() flags> -DTS_SCHED_PROF -o paper_2604_00510_b200/lib/libtreeserve_b200_sprof.so <srcs>
    python tools/sched_prof.py [exits_off | c4]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TS_LIB_PATH", os.path.join(ROOT, "paper_2604_00510_b200", "lib", "libtreeserve_b200_sprof.so"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "full"
exits_off = mode == "exits_off"
cfg = bench.search_config(bench.PER_GPU, exits=not exits_off)
table = problem_table(bench.workload(bench.PER_GPU))
if mode == "c4":  # tools/bench_configs.py c4: 1024 deep searches, budget 1024, M = 1024
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_configs as bc  # noqa: E402
    from paper_2604_00510_b200 import backend as B  # noqa: E402
    specs = [B.make_problem(f"s{i:04d}", bc.keyed.mix(0, 8, i), B.Difficulty.HARD_SOLVABLE, (31, 31), 8,
                            B.stagnation_profile()) for i in range(1024)]
    table = problem_table(specs)
    cfg = bc.cfg_of(1024, 1024, 32, 8)
eng = Engine(cfg, 0)
eng.lib.ts_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for rep in range(3):
    eng.load(table)
    st = eng.run()
    torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 32)()
eng.lib.ts_debug_prof(eng._h, buf)
p = list(buf)
n = max(1, p[10])
names = ["wave end -> k_sched start", "wave span (first CTA start -> last CTA end)",
         "k_sched end -> first wave CTA start", "k_sched: loop test + admission", "k_sched: records",
         "targets: counts + exact sum", "targets: runs", "targets: want per run", "targets: per-search targets",
         "targets: work lists (or the P = 1 fast path)"]
print(f"{ {'full': 'PE+NE+boost', 'exits_off': 'exits off', 'c4': 'config 4'}[mode]}: {n} scheduler passes, {st.steps} waves")
for i, nm in enumerate(names):
    print(f"  {nm:48s} {p[i] / n / 1000.0:8.2f} us/pass")
