import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2604_00510_b200.policy import compute_targets_arrays
from paper_2604_00510_b200.scheduler import SchedulerConfig
m = 32768
rng = np.random.default_rng(0)
arr = torch.tensor(rng.uniform(0, 100, m), device="cuda")
best = torch.tensor(rng.choice([0.0, 0.3, 0.46, 0.6], m), device="cuda")
comp = torch.tensor(rng.integers(0, 5, m), dtype=torch.int32, device="cuda")
ids = torch.arange(m, dtype=torch.int64, device="cuda")
sc = SchedulerConfig(max_concurrency=4 * m)
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, info = compute_targets_arrays(arr, best, comp, ids, 100.0, sc, 0.5)
    print(i, (time.perf_counter() - t0) * 1e3, "ms fallback", info.sum_fallback, "T", info.total_score, flush=True)
