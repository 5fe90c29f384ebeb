"""Short driver for ncu captures of the beam kernel (never a bench number)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_00510_b200._abi import TsBeamConfig, TsBeamResult, load_library  # noqa: E402
from paper_2604_00510_b200.backend import problem_table  # noqa: E402

table = problem_table(bench.workload(bench.PER_GPU))
n = len(table)
lib = load_library()
dprob = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).cuda()
dres = torch.empty(n * ctypes.sizeof(TsBeamResult), dtype=torch.uint8, device="cuda")
cfg = TsBeamConfig(8, 4, 16, 1, 1, 0, 0.5)
for _ in range(2):
    rc = lib.ts_beam_search(ctypes.byref(cfg), ctypes.c_void_p(dprob.data_ptr()), n, ctypes.c_void_p(dres.data_ptr()),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
torch.cuda.synchronize()
print("beam ok", n)
