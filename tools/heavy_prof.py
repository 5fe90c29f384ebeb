"""Phase counters of the pipelined CTA mode (diagnostics build
lib/libtreeserve_b200_prof.so, -DTS_HEAVY_PROF).   TS_LIB_PATH=... python tools/heavy_prof.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TS_LIB_PATH", os.path.join(ROOT, "paper_2604_00510_b200", "lib", "libtreeserve_b200_prof.so"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402

table = problem_table(bench.workload(bench.PER_GPU))
eng = Engine(bench.search_config(bench.PER_GPU), 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
for rep in range(2):
    eng.load(table)
    if flush is not None:  # as bench.py: L2 flushed before every batch
        bench.flush_l2(flush)
    st = eng.run()
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 32)()
eng.lib.ts_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
eng.lib.ts_debug_prof(eng._h, buf)
p = list(buf)
jobs = max(1, p[5])
print("jobs", jobs, "rollouts", st.rollouts)
print("selector cycles/job: total %.0f risky-wait %.0f inflight-wait %.0f ring-wait %.0f | drain total %.0f" %
      (p[0] / jobs, p[1] / jobs, p[2] / jobs, p[3] / jobs, p[4]))
print("selector per job: prologue %.0f descent %.0f epilogue %.0f (levels/job %.2f)" % (p[6] / jobs, p[7] / jobs, p[2] / jobs, p[12] / jobs))
print("max over searches: selector loop %d drain %d finish %d cycles" % (p[13], p[14], p[15]))
print("simulator cycles/job: wait-issue %.0f compute %.0f wait-commit %.0f commit %.0f" %
      (p[8] / jobs, p[9] / jobs, p[10] / jobs, p[11] / jobs))
r = max(1, p[21])
print("two-level rounds %d (%.2f/job): per round l1-load %.0f l2(shfl+load) %.0f math %.0f ballots+argmax %.0f take1 %.0f level2 %.0f" %
      (p[21], p[21] / jobs, p[16] / r, p[17] / r, p[22] / r, p[18] / r, p[19] / r, p[20] / r))
print("selector epilogue per job: ring writes %.0f release %.0f registration %.0f" % (p[23] / jobs, p[24] / jobs, p[25] / jobs))
rr = max(1, p[28])
print("root rounds %d: l1-load %.0f l2 %.0f per root round; other rounds: l1 %.0f l2 %.0f" % (
    p[28], p[26] / rr, p[27] / rr, (p[16] - p[26]) / max(1, p[21] - p[28]), (p[17] - p[27]) / max(1, p[21] - p[28])))
