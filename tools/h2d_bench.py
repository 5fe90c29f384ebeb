"""H2D of the config-2 problem table (4096 rows of 352 B, pinned): one
contiguous copy vs pitched copies of only the bytes the engine reads (the
96-byte header + golden_rewards[:max_glen]).  CUDA events, median of 50."""
import ctypes
import os
import statistics

import nvidia.cuda_runtime
import torch

rt = ctypes.CDLL(os.path.join(os.path.dirname(nvidia.cuda_runtime.__file__), "lib", "libcudart.so.12"))
N, ROW = 4096, 352
src = torch.empty(N * ROW, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(N * ROW, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
H2D = 1


def c2d(w, off=0):
    rt.cudaMemcpy2DAsync(ctypes.c_void_p(dst.data_ptr() + off), ctypes.c_size_t(ROW), ctypes.c_void_p(src.data_ptr() + off),
                         ctypes.c_size_t(ROW), ctypes.c_size_t(w), ctypes.c_size_t(N), H2D, ctypes.c_void_p(st.cuda_stream))


cases = {
    "contiguous 1.44 MB": lambda: dst.copy_(src, non_blocking=True),
    "2D width 216 (header + 15 rewards)": lambda: c2d(216),
    "2D width 224": lambda: c2d(224),
    "2D width 256": lambda: c2d(256),
    "2D 96 + 2D 120": lambda: (c2d(96), c2d(120, 96)),
}
for name, f in cases.items():
    ts = []
    for _ in range(60):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name}: {statistics.median(ts[10:]):.1f} us")
