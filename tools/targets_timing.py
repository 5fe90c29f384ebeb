"""Device time of the engine's k_targets (ts_step_targets) vs run-queue size
(the multi-GPU path runs it over all n_global records every wave)."""
import math
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from golden_io import load, table  # noqa: E402
from paper_2604_00510_b200._abi import TsSchedRecord  # noqa: E402
from paper_2604_00510_b200.config import SearchConfig  # noqa: E402
from paper_2604_00510_b200.engine import Engine  # noqa: E402
from paper_2604_00510_b200.scheduler import SchedulerConfig  # noqa: E402

rng = random.Random(0)
dummy = load("workloads")["c1"][0]
for n in [int(x) for x in os.environ.get("TT_SIZES", "4096,16384,32768,65536").split(",")]:
    M = 4 * n
    now = 30
    sch = SchedulerConfig(max_concurrency=M)
    recs = (TsSchedRecord * n)()
    arr = 0
    for i in range(n):
        if rng.random() < 0.3:
            arr = min(now, arr + rng.randint(0, 3))
        best = rng.choice([0.0, 0.46, 0.44, rng.random() * 0.6])
        boosted = best / 0.5 > sch.proximity
        recs[i].score = math.log1p(now - arr) + (sch.beta if boosted else 0.0)
        recs[i].flags = 1 | (2 if rng.randint(0, 4) >= 2 else 0) | (4 if boosted else 0)
    dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
    eng = Engine(SearchConfig(scheduler=sch), 0)
    eng.load(table([dummy] * n))
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step_targets(now, dev.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"n={n}: k_targets {1e3 * min(ts[1:]):.1f} us", flush=True)
    eng.close()
if os.environ.get("TS_LIB_PATH", "").endswith("_sprof.so"):
    # -DTS_SCHED_PROF build: %globaltimer at each grid barrier of k_mt_all (CTA 0)
    import ctypes
    n = int(os.environ.get("TT_PROF_N", "32768"))
    eng = Engine(SearchConfig(scheduler=SchedulerConfig(max_concurrency=4 * n)), 0)
    eng.load(table([dummy] * n))
    recs = (TsSchedRecord * n)()
    for i in range(n):
        recs[i].score = math.log1p(30 - (i * 31) // n)
        recs[i].flags = 3
    dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
    for r in range(10):
        eng.step_targets(30, dev.data_ptr())
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * 32)()
    eng.lib.ts_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    eng.lib.ts_debug_prof(eng._h, buf)
    calls = max(1, buf[11])
    print(f"k_mt_all n={n}, {calls} calls: us since kernel start at grid barriers 1-6 and at the end:",
          [round(buf[i] / calls / 1e3, 2) for i in range(12, 19)])
elif os.environ.get("TS_LIB_PATH", "").endswith("_prof.so"):
    import ctypes
    eng = Engine(SearchConfig(scheduler=SchedulerConfig(max_concurrency=4 * 32768)), 0)
    buf = (ctypes.c_uint64 * 32)()
    eng.lib.ts_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    # counters accumulate per engine; re-run the 32768 case on a fresh engine
    n = 32768
    eng.load(table([dummy] * n))
    recs = (TsSchedRecord * n)()
    for i in range(n):
        recs[i].score = math.log1p(30 - (i * 31) // n)
        recs[i].flags = 3
    dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
    for r in range(10):
        eng.step_targets(30, dev.data_ptr())
    torch.cuda.synchronize()
    eng.lib.ts_debug_prof(eng._h, buf)
    print("k_mt_all cumulative cycles at each grid sync (per call):", [round(buf[i] / 10) for i in range(23, 32)])
