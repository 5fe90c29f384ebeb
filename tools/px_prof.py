"""Phase times of the fused sharded step k_px_step (diagnostics build with
-DTS_PX_PROF, lib/libtreeserve_b200_pxprof.so):  python tools/px_prof.py [W] [per_rank]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("TS_LIB_PATH", os.path.join(ROOT, "paper_2604_00510_b200", "lib", "libtreeserve_b200_pxprof.so"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import peer_overhead  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1
per = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
import paper_2604_00510_b200.engine as E  # noqa: E402

captured = []
orig_close = E.Engine.close


def close(self):
    if not captured:
        buf = (ctypes.c_uint64 * 32)()
        self.lib.ts_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        self.lib.ts_debug_prof(self._h, buf)
        captured.append(list(buf))
    orig_close(self)


E.Engine.close = close
r = peer_overhead.run(W, per, reps=1)
p = captured[0]
waves = r["waves"]
names = ["admission", "load jobs", "segment scan", "entries", "publish+wait", "read headers+stage", "merge scan",
         "runs+sum", "tables (to targets)", "per-job targets", "work lists", "(warp) headers", "(warp) entry loads",
         "(warp) seg scan", "(warp) merged+scores", "(warp) sums+want", "(warp) run bases"]
for i, nm in enumerate(names):
    if i < 12:
        print(f"{nm:20s} {p[i] / max(1, waves) / 1e3:8.2f} us/wave")
    else:  # the one-warp sub-phases are clock64 cycles
        print(f"{nm:20s} {p[i] / max(1, waves):8.0f} cycles/wave")
