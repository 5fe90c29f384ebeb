"""The multi-rank path end to end on one GPU: 2 processes (one engine each,
both on cuda:0) run either paper_2604_00510_b200.distributed.ShardedRun with a
gloo group and host-staged all-gathers, or PeerShardedRun (ts_run_sharded:
each process maps the other's exchange buffer through a CUDA IPC handle and
writes into it from its kernels — the multi-GPU path, with the peer on the
same device); the outcomes must equal the reference wave oracle's."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASE = "c1_M48_admission"


def _worker(rank, world, port, out, mode):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist

    from golden_io import config_from_case, load, table
    from paper_2604_00510_b200.distributed import PeerShardedRun, ShardedRun, shard_bounds
    from paper_2604_00510_b200.engine import Engine

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    case = next(c for c in load("waves") if c["name"] == CASE)
    recs = load("workloads")[case["workload"]]
    lo, hi = shard_bounds(len(recs), world, rank)
    eng = Engine(config_from_case(case), 0)
    eng.load(table(recs[lo:hi]), lo, len(recs))
    if mode == "peer":
        steps = PeerShardedRun(eng, dist).run().steps
    else:
        run = ShardedRun(eng, dist, hi - lo, len(recs), torch.device("cuda", 0), check_every=1, host_staging=True)
        steps = run.run()
    o = eng.outcomes()
    out[rank] = (steps, [(x.exit_kind, x.rollouts_completed, x.tokens_generated, x.best_score, x.exit_step,
                          x.admit_step, x.launched, x.cancelled, x.nodes) for x in o])
    eng.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["host_staged", "peer"])
def test_two_ranks_one_gpu_match_wave_oracle(mode):
    from golden_io import load

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out, mode), nprocs=2, join=True)
    case = next(c for c in load("waves") if c["name"] == CASE)
    got = out[0][1] + out[1][1]
    assert out[0][0] == out[1][0] == case["steps"]
    names = {None: 0, "positive": 1, "negative": 2, "budget_exhausted": 3}
    for g, w in zip(got, case["outcomes"]):
        assert g == (names[w["exit_kind"]], w["rollouts_completed"], w["tokens_generated"], w["best_score"],
                     w["exit_step"], w["admit_step"], w["launched"], w["cancelled"], w["nodes"])
