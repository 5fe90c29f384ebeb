"""The sharded batch over peer memory (ts_run_sharded) == one
engine over the whole run queue.

Ranks are emulated in one process on one GPU: every rank is an engine with
its own stream and host thread, and the exchange buffers are connected by
device pointer (the same kernels write into another GPU's buffer through a
CUDA IPC mapping on a multi-GPU node; tests/test_multiprocess_gpu.py covers
the IPC path with two processes).  Shards are deliberately unequal."""

import threading

import pytest

from golden_io import WAVE_KEYS, config_from_case, load, outcome_dict, table

pytestmark = pytest.mark.gpu


def _run_ranks(cfg, tables_with_offsets, n_global, env=None):
    import torch

    from paper_2604_00510_b200.distributed import connect_in_process, last_arrival_of
    from paper_2604_00510_b200.engine import Engine

    engines, streams = [], []
    for tab, off in tables_with_offsets:
        st = torch.cuda.Stream()
        e = Engine(cfg, 0, stream=st)
        e.load(tab, global_offset=off, n_global=n_global)
        engines.append(e)
        streams.append(st)
    torch.cuda.synchronize()
    connect_in_process(engines)
    last = last_arrival_of([t for t, _ in tables_with_offsets])
    return engines, _launch(engines, last)


def _launch(engines, last):
    """ts_run_sharded on every rank at once (one host thread per rank: each
    call returns when the global loop has ended)."""
    import torch

    stats, errors = [None] * len(engines), []

    def go(r):
        try:
            stats[r] = engines[r].run_sharded(last_arrival=last)
        except Exception as ex:  # surfaced below
            errors.append(ex)

    th = [threading.Thread(target=go, args=(r,)) for r in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    return stats


def _bounds(n, parts):
    # unequal blocks: 40 %, 15 %, the rest
    b = [0, (2 * n) // 5, (2 * n) // 5 + max(1, (3 * n) // 20), n]
    return b[: parts + 1] if parts == 3 else [0, n]


MODES = ["fused", "fused_block_tables", "two_kernels"]


def _mode_env(monkeypatch, mode):
    if mode == "fused_block_tables":  # k_px_step with the block-wide table path even for small tables
        monkeypatch.setenv("TS_PX_GWARP", "0")
    if mode == "two_kernels":  # k_px_groups + k_px_sched
        monkeypatch.setenv("TS_PX_TWO_KERNELS", "1")


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", ["c1_M48_admission", "cli_serving_pe_ne_boost", "c2_s512_M2048"])
def test_peer_sharded_matches_reference_waves(name, mode, monkeypatch):
    """3 unequal ranks over peer memory reproduce the reference-composed wave
    oracle (FIFO admission across ranks, Poisson arrivals, boosting) with each
    scheduler variant of the graph loop."""
    _mode_env(monkeypatch, mode)
    case = next(c for c in load("waves") if c["name"] == name)
    recs = load("workloads")[case["workload"]][: len(case["outcomes"])]
    cfg = config_from_case(case)
    n = len(recs)
    b = _bounds(n, 3)
    arr = case.get("arrival_steps")
    parts = [(table(recs[b[r]:b[r + 1]], arr[b[r]:b[r + 1]] if arr else None), b[r]) for r in range(3)]
    engines, stats = _run_ranks(cfg, parts, n)
    assert len({s.steps for s in stats}) == 1  # one global loop
    assert stats[0].steps == case["steps"]
    got = [o for e in engines for o in e.outcomes()]
    for i, want in enumerate(case["outcomes"]):
        g = outcome_dict(got[i])
        for k in g:
            assert g[k] == want[k], (i, k)
        for k in WAVE_KEYS:
            assert getattr(got[i], k) == want[k], (i, k)
    for e in engines:
        e.close()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("world", [1, 2, 5])
def test_peer_sharded_matches_single_engine(world, mode, monkeypatch):
    """C2-shape batch (boosting, exits) sharded over `world` unequal ranks ==
    ts_run on one engine: every outcome field and the global wave count."""
    import torch

    _mode_env(monkeypatch, mode)

    from paper_2604_00510_b200 import backend as B
    from paper_2604_00510_b200.config import SearchConfig
    from paper_2604_00510_b200.engine import Engine
    from paper_2604_00510_b200.scheduler import SchedulerConfig

    specs = B.make_workload(600, (0.6, 0.25, 0.15), 11, branching=4,
                            depth_ranges={d: (15, 15) for d in B.Difficulty})
    cfg = SearchConfig(scheduler=SchedulerConfig(max_concurrency=1200), rollout_budget=48, depth_cap=16,
                       expand_width=4)
    tab = B.problem_table(specs)
    with Engine(cfg, 0) as one:
        one.load(tab)
        st1 = one.run()
        want = one.outcomes()
    n = len(specs)
    cuts = [0] + sorted({(n * (k * k)) // (world * world) for k in range(1, world)}) + [n]
    parts = [(B.problem_table(specs[cuts[r]:cuts[r + 1]]), cuts[r]) for r in range(len(cuts) - 1)]
    engines, stats = _run_ranks(cfg, parts, n)
    got = [o for e in engines for o in e.outcomes()]
    keys = ("exit_kind", "rollouts_completed", "tokens_generated", "best_score", "best_len", "solved", "exit_step",
            "launched", "cancelled", "nodes", "status")
    for i in range(n):
        for k in keys:
            assert getattr(got[i], k) == getattr(want[i], k), (i, k)
    assert stats[0].steps == st1.steps
    assert sum(s.rollouts for s in stats) == st1.rollouts
    # a second batch over the same connection (the flags' next generation)
    for e, (tb, off) in zip(engines, parts):
        e.load(tb, global_offset=off, n_global=n)
    torch.cuda.synchronize()
    stats2 = _launch(engines, 0)
    got2 = [o for e in engines for o in e.outcomes()]
    for i in range(n):
        for k in keys:
            assert getattr(got2[i], k) == getattr(want[i], k), (i, k)
    assert stats2[0].steps == st1.steps
    for e in engines:
        e.close()
