"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every value written here comes from reference calls (``/root/reference/pkg/src``)
or from ``wave_ref.run_waves``, which is composed only of reference calls.  The
fixtures pin the C oracle (``oracle/``) and, through it and directly, the CUDA
engine.  Floats are stored with ``repr`` (shortest round-trip), so equality
checks against them are bit-exact.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import wave_ref  # noqa: E402  (puts the reference on sys.path)
from treeserve import rng  # noqa: E402
from treeserve.backend import (  # noqa: E402
    Difficulty,
    RewardProfile,
    generate_steps,
    golden_step_rewards,
    make_problem,
    make_workload,
)
from treeserve.scheduler import Job, SchedulerConfig, SchedulerState, JobState, compute_targets  # noqa: E402
from treeserve.scoring import AggregationScheme, FutilityBound, ScoringConfig  # noqa: E402
from treeserve.search import run_tree_search  # noqa: E402
from treeserve.tree import SearchTree  # noqa: E402

SEED = 0
MIX = (0.6, 0.25, 0.15)

# Config-4 "heavy-tailed stagnation" profile (BASELINE.json configs[3]); the
# reference has no such profile, so it is defined here and in
# paper_2604_00510_b200/backend.py (stagnation_profile) with identical values.
STAGNATION = RewardProfile(
    golden_range=(0.93, 0.99),
    off_path_range=(0.22, 0.75),
    hidden_until_depth=6,
    shared_range=(0.80, 0.97),
    target_aggregate=0.55,
)


def dump(name, obj):
    path = os.path.join(HERE, name + ".json.gz")
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def problem_record(p):
    prof = p.reward_profile
    return {
        "problem_id": p.problem_id,
        "seed": p.seed,
        "difficulty": p.difficulty.value,
        "depth_range": list(p.depth_range),
        "branching": p.branching,
        "base_depth": p.base_depth,
        "golden_path": list(p.golden_path) if p.golden_path is not None else None,
        "golden_rewards": list(golden_step_rewards(p)) if p.golden_path is not None else None,
        "profile": {
            "golden_range": list(prof.golden_range),
            "off_path_range": list(prof.off_path_range),
            "hidden_until_depth": prof.hidden_until_depth,
            "shared_range": list(prof.shared_range) if prof.shared_range else None,
            "target_aggregate": prof.target_aggregate,
        },
    }


def tree_record(tree: SearchTree):
    d = tree.to_dict()
    # children order is creation order (ids ascending); keep the dump compact
    return {
        "completed_rollouts": d["completed_rollouts"],
        "rollout_budget": d["rollout_budget"],
        "parent": [n["parent"] if n["parent"] is not None else -1 for n in d["nodes"]],
        "reward": [n["reward"] for n in d["nodes"]],
        "prior": [n["prior"] for n in d["nodes"]],
        "N": [n["N"] for n in d["nodes"]],
        "O": [n["O"] for n in d["nodes"]],
        "W": [n["W"] for n in d["nodes"]],
        "terminal": [int(n["terminal"]) for n in d["nodes"]],
        "depth": [n["depth"] for n in d["nodes"]],
        "step_ref": [tree.nodes[n["id"]].step_ref if n["parent"] is not None else -1 for n in d["nodes"]],
    }


def outcome_record(o):
    return {
        "problem_id": o.problem_id,
        "exit_kind": o.exit_kind.value,
        "best_score": o.best_score,
        "best_path": list(o.best_path),
        "rollouts_completed": o.rollouts_completed,
        "tokens_generated": o.tokens_generated,
        "solved": o.solved,
    }


def scoring_record(s: ScoringConfig):
    return {
        "scheme": s.scheme.value,
        "accept_threshold": s.accept_threshold,
        "positive_exit_threshold": s.positive_exit_threshold,
        "first_step_threshold": s.first_step_threshold,
        "strict_negative_exit": s.strict_negative_exit,
        "futility_bound": s.futility_bound.value,
    }


def serial_tree(problem, scoring, budget, cap, width, pe, ne):
    """run_tree_search, but keeping the tree (same loop as search.py:79-119)."""
    out, _ = wave_ref.run_waves(
        [problem], scoring=scoring, sched=SchedulerConfig(max_concurrency=1, boosting_enabled=False),
        rollout_budget=budget, depth_cap=cap, expand_width=width, positive_exit=pe,
        negative_exit=ne, keep_trees=True,
    )
    return out[0]["tree"]


def gen_rng():
    r = random.Random(1234)
    kats = []
    for _ in range(300):
        n = r.randint(0, 36)
        keys = [r.choice([r.randint(0, 40), r.getrandbits(64), r.getrandbits(20)]) for _ in range(n)]
        lo = r.randint(0, 100)
        hi = lo + r.randint(0, 200)
        kats.append({
            "keys": keys,
            "mix": rng.mix(*keys),
            "uniform": rng.uniform(*keys),
            "uniform_in": [0.05, 0.28, rng.uniform_in(0.05, 0.28, *keys)],
            "randint": [lo, hi, rng.randint_in(lo, hi, *keys)],
            "exponential": [2.5, rng.exponential(2.5, *keys)],
        })
    dump("rng_kats", kats)


def gen_workloads():
    D7 = {d: (7, 7) for d in Difficulty}
    D15 = {d: (15, 15) for d in Difficulty}
    wl = {
        "c1": [problem_record(p) for p in make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)],
        "c2": [problem_record(p) for p in make_workload(4096, MIX, SEED, branching=4, depth_ranges=D15)],
        "cli_default": [problem_record(p) for p in make_workload(500, MIX, 20260810)],
        "mixed_b3": [problem_record(p) for p in make_workload(
            97, (0.5, 0.3, 0.2), 77, branching=3,
            depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
            accept_threshold=0.35)],
        "c4_stagnation": [problem_record(make_problem(f"s{i:04d}", rng.mix(SEED, 8, i), Difficulty.HARD_SOLVABLE,
                                                      (31, 31), 8, STAGNATION)) for i in range(16)],
    }
    dump("workloads", wl)


def gen_steps():
    r = random.Random(99)
    kats = []
    specs = list(make_workload(40, MIX, 5, branching=4, depth_ranges={d: (3, 12) for d in Difficulty}))
    specs += [make_problem(f"s{i}", rng.mix(3, 8, i), Difficulty.HARD_SOLVABLE, (31, 31), 8, STAGNATION) for i in range(4)]
    for p in specs:
        for _ in range(12):
            # random non-terminal context: walk down random children until terminal
            path = []
            depth_target = r.randint(0, p.max_depth)
            while len(path) < depth_target:
                cands = generate_steps(p, path, p.branching)
                j = r.randrange(len(cands))
                if cands[j].is_terminal:
                    break
                path.append(cands[j].step_ref)
            width = r.randint(1, p.branching)
            cands = generate_steps(p, path, width)
            kats.append({
                "problem": problem_record(p),
                "path": path,
                "width": width,
                "candidates": [[c.step_ref, c.token_count, c.prior, c.prm_reward, int(c.is_terminal)] for c in cands],
            })
    dump("steps_kats", kats)


def gen_serial():
    """run_tree_search outcomes (search.py:79) for several scoring variants + tree dumps."""
    D7 = {d: (7, 7) for d in Difficulty}
    c1 = make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)
    mixed = make_workload(97, (0.5, 0.3, 0.2), 77, branching=3,
                          depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
                          accept_threshold=0.35)
    cases = []
    variants = [
        ("c1_default", c1, ScoringConfig(), 32, 8, 4, True, True),
        ("c1_exits_off", c1, ScoringConfig(), 32, 8, 4, False, False),
        ("c1_pe_only", c1, ScoringConfig(), 32, 8, 4, True, False),
        ("mixed_strict_prefix", mixed, ScoringConfig(strict_negative_exit=True, futility_bound=FutilityBound.PREFIX_AGGREGATE, accept_threshold=0.35), 48, 7, 3, True, True),
        ("mixed_min_scheme", mixed, ScoringConfig(scheme=AggregationScheme.MINIMUM, positive_exit_threshold=0.6, first_step_threshold=0.3), 40, 12, 2, True, True),
        ("mixed_cap5", mixed, ScoringConfig(), 24, 5, 3, True, True),
    ]
    for name, wl, sc, budget, cap, width, pe, ne in variants:
        outs = [outcome_record(run_tree_search(p, sc, None, budget, cap, width, pe, ne)) for p in wl]
        trees = {}
        for idx in (0, 1, 2, 5, 11, 40):
            if idx < len(wl):
                trees[str(idx)] = tree_record(serial_tree(wl[idx], sc, budget, cap, width, pe, ne))
        cases.append({
            "name": name, "workload": "c1" if wl is c1 else "mixed_b3", "scoring": scoring_record(sc),
            "budget": budget, "depth_cap": cap, "expand_width": width, "positive_exit": pe,
            "negative_exit": ne, "outcomes": outs, "trees": trees,
        })
    dump("serial", cases)


def gen_deep():
    """Exits-off deep trees (C2 shape, budget 128) and config-4 stagnation shape."""
    D15 = {d: (15, 15) for d in Difficulty}
    c2 = make_workload(4096, MIX, SEED, branching=4, depth_ranges=D15)
    cases = []
    for idx in (0, 3):
        t0 = time.time()
        tree = serial_tree(c2[idx], ScoringConfig(), 128, 16, 4, False, False)
        cases.append({"name": f"c2_exits_off_{idx}", "workload": "c2", "index": idx, "budget": 128,
                      "depth_cap": 16, "expand_width": 4, "positive_exit": False, "negative_exit": False,
                      "tree": tree_record(tree)})
        print("deep", idx, len(tree.nodes), time.time() - t0)
    s = make_problem("s0000", rng.mix(SEED, 8, 0), Difficulty.HARD_SOLVABLE, (31, 31), 8, STAGNATION)
    tree = serial_tree(s, ScoringConfig(), 48, 32, 8, False, False)
    cases.append({"name": "c4_exits_off_0", "workload": "c4_stagnation", "index": 0, "budget": 48,
                  "depth_cap": 32, "expand_width": 8, "positive_exit": False, "negative_exit": False,
                  "tree": tree_record(tree)})
    print("deep c4", len(tree.nodes))
    dump("deep_trees", cases)


def wave_case(name, wl_name, problems, sched, budget, cap, width, pe, ne, scoring=None,
              arrival_steps=None, tree_idx=()):
    t0 = time.time()
    out, info = wave_ref.run_waves(problems, scoring=scoring, sched=sched, rollout_budget=budget,
                                   depth_cap=cap, expand_width=width, positive_exit=pe,
                                   negative_exit=ne, arrival_steps=arrival_steps,
                                   keep_trees=bool(tree_idx))
    trees = {str(i): tree_record(out[i]["tree"]) for i in tree_idx}
    for o in out:
        o.pop("tree", None)
    print(name, "steps", info["steps"], "rollouts", sum(o["rollouts_completed"] for o in out),
          f"{time.time() - t0:.1f}s")
    return {
        "name": name, "workload": wl_name, "scoring": scoring_record(scoring or ScoringConfig()),
        "sched": {"max_concurrency": sched.max_concurrency, "beta": sched.beta, "proximity": sched.proximity,
                  "obs_threshold": sched.obs_threshold, "boosting_enabled": sched.boosting_enabled},
        "budget": budget, "depth_cap": cap, "expand_width": width, "positive_exit": pe,
        "negative_exit": ne, "arrival_steps": arrival_steps, "steps": info["steps"],
        "targets_trace": info["targets_trace"], "outcomes": out, "trees": trees,
    }


def serving_arrivals(n, rate, seed, steps_per_unit):
    """Config-5 arrivals: the reference generator (simulator.py:193-200) quantised to steps."""
    t = 0.0
    steps = []
    for i in range(n):
        t += rng.exponential(rate, seed, 21, i)
        steps.append(int(t * steps_per_unit))
    return steps


def gen_waves():
    D7 = {d: (7, 7) for d in Difficulty}
    D15 = {d: (15, 15) for d in Difficulty}
    c1 = make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)
    c2 = make_workload(4096, MIX, SEED, branching=4, depth_ranges=D15)
    cli = make_workload(500, MIX, 20260810)
    mixed = make_workload(97, (0.5, 0.3, 0.2), 77, branching=3,
                          depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
                          accept_threshold=0.35)
    cases = [
        wave_case("c1_M64", "c1", c1, SchedulerConfig(max_concurrency=64), 32, 8, 4, True, True, tree_idx=(0, 7)),
        wave_case("c1_M256", "c1", c1, SchedulerConfig(max_concurrency=256), 32, 8, 4, True, True, tree_idx=(0, 7)),
        wave_case("c1_M256_pe", "c1", c1, SchedulerConfig(max_concurrency=256), 32, 8, 4, True, False),
        wave_case("c1_M48_admission", "c1", c1, SchedulerConfig(max_concurrency=48), 32, 8, 4, True, True),
        wave_case("mixed_M200_obs3", "mixed_b3", mixed,
                  SchedulerConfig(max_concurrency=200, beta=1.5, proximity=0.8, obs_threshold=3), 40, 9, 3, True, True,
                  scoring=ScoringConfig(accept_threshold=0.35), tree_idx=(4,)),
        wave_case("c2_M4096", "c2", c2, SchedulerConfig(max_concurrency=4096), 128, 16, 4, True, True, tree_idx=(1, 2)),
        wave_case("c2_s512_M2048", "c2", c2[:512], SchedulerConfig(max_concurrency=2048), 128, 16, 4, True, True),
        wave_case("c3_s256_M1024_exits_off", "c2", c2[:256], SchedulerConfig(max_concurrency=1024), 24, 16, 4, False, False,
                  tree_idx=(0,)),
        wave_case("cli_serving_pe_ne_boost", "cli_default", cli, SchedulerConfig(max_concurrency=16), 32, 16, 4, True, True,
                  arrival_steps=serving_arrivals(500, 5.0, 20260810, 20.0)),
        wave_case("cli_serving_pe", "cli_default", cli, SchedulerConfig(max_concurrency=16, boosting_enabled=False), 32, 16, 4,
                  True, False, arrival_steps=serving_arrivals(500, 5.0, 20260810, 20.0)),
    ]
    dump("waves", cases)


def gen_trace():
    """The per-pass trace (simulator.py:314-341 allocation/action records, plus
    job_finished events) of wave runs, as the JSONL text cli.py:263-265 writes."""
    import json as _json

    D7 = {d: (7, 7) for d in Difficulty}
    c1 = make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)
    cli = make_workload(500, MIX, 20260810)
    mixed = make_workload(97, (0.5, 0.3, 0.2), 77, branching=3,
                          depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
                          accept_threshold=0.35)
    cases = []
    for name, wl, probs, sch, budget, cap, width, pe, ne, scoring, arr, dt in (
        ("c1_M256", "c1", c1, SchedulerConfig(max_concurrency=256), 32, 8, 4, True, True, None, None, 1.0),
        ("c1_M48_admission", "c1", c1, SchedulerConfig(max_concurrency=48), 32, 8, 4, True, True, None, None, 1.0),
        ("mixed_M200_obs3", "mixed_b3", mixed, SchedulerConfig(max_concurrency=200, beta=1.5, proximity=0.8, obs_threshold=3),
         40, 9, 3, True, True, ScoringConfig(accept_threshold=0.35), None, 1.0),
        ("cli_serving_pe_ne_boost", "cli_default", cli, SchedulerConfig(max_concurrency=16), 32, 16, 4, True, True, None,
         serving_arrivals(500, 5.0, 20260810, 20.0), 1.0),
    ):
        tr = []
        wave_ref.run_waves(probs, scoring=scoring, sched=sch, rollout_budget=budget, depth_cap=cap, expand_width=width,
                           positive_exit=pe, negative_exit=ne, arrival_steps=arr, dt=dt, trace=tr)
        jsonl = "".join(_json.dumps(e, sort_keys=True) + "\n" for e in tr)
        print("trace", name, len(tr))
        cases.append({"name": name, "wave_case": name, "dt": dt, "jsonl": jsonl})
    dump("trace", cases)


def gen_cost():
    """The wave clock of the reference cost model (wave_ref.run_waves(cost=...):
    service_time and CostModel of backend.py:287-311, charged as
    simulator.py:443-463) on the CLI serving workload, four presets."""
    from treeserve.backend import CostModel

    cli = make_workload(500, MIX, 20260810)
    arr = serving_arrivals(500, 5.0, 20260810, 20.0)
    mixed = make_workload(97, (0.5, 0.3, 0.2), 77, branching=3,
                          depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
                          accept_threshold=0.35)
    cases = []
    for name, wl, probs, arrivals, M, pe, ne, boost, cost in (
        ("cli_vanilla", "cli_default", cli, arr, 16, False, False, False, CostModel()),
        ("cli_pe", "cli_default", cli, arr, 16, True, False, False, CostModel()),
        ("cli_pe_ne", "cli_default", cli, arr, 16, True, True, False, CostModel()),
        ("cli_pe_ne_boost", "cli_default", cli, arr, 16, True, True, True, CostModel()),
        ("mixed_M200_cost", "mixed_b3", mixed, None, 200, True, True, True,
         CostModel(per_token_latency=0.0031, engine_capacity=7, reward_latency=0.02)),
    ):
        sch = SchedulerConfig(max_concurrency=M, boosting_enabled=boost)
        out, info = wave_ref.run_waves(probs, sched=sch, rollout_budget=32, depth_cap=16, expand_width=4,
                                       positive_exit=pe, negative_exit=ne, arrival_steps=arrivals, cost=cost)
        cases.append({"name": name, "workload": wl, "n": len(probs), "arrival_steps": arrivals,
                      "max_concurrency": M, "positive_exit": pe, "negative_exit": ne, "boosting_enabled": boost,
                      "budget": 32, "depth_cap": 16, "expand_width": 4,
                      "cost": [cost.per_token_latency, cost.engine_capacity, cost.reward_latency],
                      "steps": info["steps"],
                      "sim_arrival": [o["sim_arrival"] for o in out],
                      "sim_completion": [o["sim_completion"] for o in out],
                      "tokens": [o["tokens_generated"] for o in out]})
        print("cost", name, info["steps"])
    dump("cost", cases)


def gen_targets():
    """compute_targets (scheduler.py:143-187) on random pools, incl. equal-score lock-step pools."""
    r = random.Random(7)
    kats = []
    for t in range(400):
        n = r.randint(1, 60) if t % 4 else r.randint(100, 700)
        M = n + r.randint(0, 5 * n)
        cfg = SchedulerConfig(max_concurrency=M, beta=r.choice([2.0, 1.0, 0.5]), proximity=r.choice([0.9, 0.5]),
                              obs_threshold=r.choice([1, 2, 3]), boosting_enabled=r.random() > 0.05)
        lockstep = t % 3 == 0
        now_step = r.randint(0, 40)
        state = SchedulerState(now=float(now_step))
        rows = []
        arr = 0
        for i in range(n):
            if not lockstep:
                arr = min(now_step, arr + (r.randint(0, 2) if r.random() < 0.5 else 0))
            job = Job(job_id=i, arrival_time=float(0 if lockstep else arr), tree=SearchTree(8))
            job.completed_rollouts = r.randint(0, 5)
            job.best_score = r.choice([0.0, r.random(), 0.46, 0.44, 0.5 * 0.9, r.random() * 0.6])
            job.state = JobState.RUNNING
            state.run_queue.append(job)
            rows.append([int(job.arrival_time), job.completed_rollouts, job.best_score])
        targets = compute_targets(state, cfg, 0.5)
        kats.append({"now_step": now_step, "M": M, "beta": cfg.beta, "proximity": cfg.proximity,
                     "obs_threshold": cfg.obs_threshold, "boosting": cfg.boosting_enabled,
                     "theta_pos": 0.5, "jobs": rows, "targets": [targets[i] for i in range(n)]})
    dump("targets_kats", kats)


def _policy_tree_record(tree: SearchTree, configs):
    """to_dict() plus best score and, per scoring config, the reference's
    check_negative_exit / decide_exit answers (or the exception it raises)."""
    from treeserve.scoring import UnsupportedSchemeError, check_negative_exit, decide_exit

    rec = tree.to_dict()
    rec["nodes"] = [{k: nd[k] for k in ("id", "parent", "reward", "terminal", "depth")} for nd in rec["nodes"]]
    best = tree.best_trajectory
    rec["best_score"] = None if best is None else best.aggregate_score
    answers = []
    for sc in configs:
        row = {}
        try:
            row["ne"] = check_negative_exit(tree, sc)
        except UnsupportedSchemeError:
            row["ne"] = "unsupported"
        for pe in (True, False):
            for ne in (True, False):
                for ex in (False, True):
                    key = f"{int(pe)}{int(ne)}{int(ex)}"
                    try:
                        d = decide_exit(tree, sc, pe, ne, ex)
                        row[key] = [d.kind.value, d.best_score]
                    except UnsupportedSchemeError:
                        row[key] = "unsupported"
        answers.append(row)
    rec["answers"] = answers
    return rec


def gen_policy():
    """Standalone policy operators (csrc/policy.cu): compute_targets on general
    run queues (unsorted fractional arrivals, shuffled ids), parallelism_score
    errors, math.log1p values, and check_negative_exit / decide_exit on trees
    taken mid-search from reference runs and on hand-built deep trees."""
    import math

    from treeserve.backend import ProblemBackend
    from treeserve.scheduler import parallelism_score
    from treeserve.search import finish_rollout
    from treeserve.tree import (NoExpandableLeafError, SelectionParams, expand, select_leaf,
                                simulate_to_terminal)

    r = random.Random(11)
    out = {}
    # log1p KATs (wait times: non-negative)
    xs = [0.0, 1e-300, 5e-324, 1e-17, 2.0**-29, 2.0**-28, 1e-5, 0.1, 0.2928, 0.2929, 0.41421, 0.4142135623730950,
          0.5, 1.0, 2.0, 3.0, 10.0, 1e6, 2.0**53, 1e300, 1.7976931348623157e308]
    for e in range(-40, 40):
        for _ in range(25):
            xs.append(math.ldexp(r.random() + 0.5, e))
    xs += [r.uniform(0, 50) for _ in range(2000)] + [float(k) for k in range(200)]
    out["log1p"] = [[x, math.log1p(x)] for x in xs]
    # general compute_targets
    kats = []
    for t in range(300):
        n = r.randint(1, 40) if t % 5 else r.randint(200, 3000)
        M = n + r.choice([0, r.randint(0, n), r.randint(0, 6 * n)])
        cfg = SchedulerConfig(max_concurrency=M, beta=r.choice([2.0, 1.0, 0.5, 3.7]), proximity=r.choice([0.9, 0.5, 0.75]),
                              obs_threshold=r.choice([1, 2, 3]), boosting_enabled=r.random() > 0.05)
        theta = r.choice([0.5, 0.6, 0.35])
        now = r.choice([r.uniform(0, 100), float(r.randint(0, 50))])
        kind = t % 4
        ids = r.sample(range(10 * n + 10), n)
        rows = []
        state = SchedulerState(now=now)
        for i in range(n):
            if kind == 0:
                arr = r.uniform(0, now)                      # unsorted fractional arrivals
            elif kind == 1:
                arr = float(r.randint(0, int(now)))          # integer arrivals, many ties
            elif kind == 2:
                arr = 0.0                                    # lock-step pool (all equal scores)
            else:
                arr = r.choice([0.0, now, now / 2, r.uniform(0, now)])
            job = Job(job_id=ids[i], arrival_time=arr, tree=SearchTree(8))
            job.completed_rollouts = r.randint(0, 5)
            job.best_score = r.choice([0.0, r.random(), theta * cfg.proximity, theta * 0.95, r.random() * theta * 1.2])
            job.state = JobState.RUNNING
            state.run_queue.append(job)
            rows.append([arr, job.completed_rollouts, job.best_score, ids[i]])
        targets = compute_targets(state, cfg, theta)
        scores = None if not cfg.boosting_enabled else [parallelism_score(j, now, theta, cfg) for j in state.run_queue]
        kats.append({"now": now, "M": M, "beta": cfg.beta, "proximity": cfg.proximity, "obs_threshold": cfg.obs_threshold,
                     "boosting": cfg.boosting_enabled, "theta_pos": theta, "jobs": rows,
                     "targets": [targets[j[3]] for j in rows], "scores": scores})
    out["targets"] = kats
    # error cases: a job arriving after now
    errs = []
    for boosting in (True, False):
        state = SchedulerState(now=3.0)
        for i, arr in enumerate([0.0, 1.0, 4.5, 2.0, 7.0]):
            job = Job(job_id=i, arrival_time=arr, tree=SearchTree(8))
            job.state = JobState.RUNNING
            state.run_queue.append(job)
        cfg = SchedulerConfig(max_concurrency=20, boosting_enabled=boosting)
        try:
            res = compute_targets(state, cfg, 0.5)
            errs.append({"boosting": boosting, "targets": [res[i] for i in range(5)]})
        except ValueError as e:
            errs.append({"boosting": boosting, "error": str(e)})
    out["target_errors"] = errs
    # trees for the exit policy
    configs = [ScoringConfig(), ScoringConfig(strict_negative_exit=True),
               ScoringConfig(futility_bound=FutilityBound.PREFIX_AGGREGATE),
               ScoringConfig(scheme=AggregationScheme.MINIMUM, futility_bound=FutilityBound.PREFIX_AGGREGATE),
               ScoringConfig(scheme=AggregationScheme.MINIMUM, strict_negative_exit=True, accept_threshold=0.5),
               ScoringConfig(accept_threshold=0.6, first_step_threshold=0.5, positive_exit_threshold=0.7),
               ScoringConfig(scheme=AggregationScheme.AVERAGE), ScoringConfig(scheme=AggregationScheme.CUMULATIVE_SUM)]
    out["scoring"] = [scoring_record(c) for c in configs]
    trees = []
    wl = make_workload(32, MIX, 3, branching=3, depth_ranges={d: (3, 6) for d in Difficulty})
    wl2 = make_workload(8, MIX, 4, branching=4, depth_ranges={d: (8, 10) for d in Difficulty})
    for pi, problem in enumerate(list(wl) + list(wl2)):
        tree = SearchTree(40)
        backend = ProblemBackend(problem, 4)
        stops = sorted(r.sample(range(0, 40), 3))
        k = 0
        for stop in stops:
            while k < stop:
                try:
                    leaf = select_leaf(tree, SelectionParams())
                except NoExpandableLeafError:
                    break
                term = simulate_to_terminal(tree, leaf, backend, 12)
                finish_rollout(tree, term, ScoringConfig())
                k += 1
            trees.append(_policy_tree_record(tree, configs))
    # a bare root, a root with only terminal children, and a chain deeper than 64
    trees.append(_policy_tree_record(SearchTree(4), configs))

    class _C:
        def __init__(self, ref, reward, term):
            self.step_ref, self.prior, self.prm_reward, self.is_terminal = ref, 0.5, reward, term

    t = SearchTree(4)
    expand(t, t.root_id, [_C(0, 0.9, True), _C(1, 0.2, True)])
    trees.append(_policy_tree_record(t, configs))
    for chain_rewards in ([0.99] * 90, [0.999] * 70 + [0.2], [0.95] * 80):
        t = SearchTree(4)
        node = t.root_id
        for d, rw in enumerate(chain_rewards):
            kids = expand(t, node, [_C(0, rw, False), _C(1, r.uniform(0.0, 0.6), d % 3 == 0)])
            node = kids[0]
        trees.append(_policy_tree_record(t, configs))
    out["trees"] = trees
    dump("policy_kats", out)


def gen_beam():
    """run_beam_search (beam.py:143-176) on committed workloads under several
    BeamConfigs and schemes; problems are referenced by (workload, index)."""
    from treeserve.beam import BeamConfig, run_beam_search

    D7 = {d: (7, 7) for d in Difficulty}
    D15 = {d: (15, 15) for d in Difficulty}
    wls = {
        "c1": list(make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)),
        "c2": list(make_workload(4096, MIX, SEED, branching=4, depth_ranges=D15))[:256],
        "cli_default": list(make_workload(500, MIX, 20260810)),
        "mixed_b3": list(make_workload(
            97, (0.5, 0.3, 0.2), 77, branching=3,
            depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
            accept_threshold=0.35)),
        "c4_stagnation": [make_problem(f"s{i:04d}", rng.mix(SEED, 8, i), Difficulty.HARD_SOLVABLE, (31, 31), 8,
                                       STAGNATION) for i in range(16)],
    }
    cases = [
        ("c1", BeamConfig(), ScoringConfig()),
        ("c1", BeamConfig(beam_width=2, candidates_per_beam=4, max_depth=5), ScoringConfig()),
        ("c1", BeamConfig(positive_exit_enabled=False), ScoringConfig()),
        ("c2", BeamConfig(), ScoringConfig()),
        ("c2", BeamConfig(beam_width=4, candidates_per_beam=8, max_depth=20, positive_exit_enabled=False),
         ScoringConfig()),
        ("cli_default", BeamConfig(), ScoringConfig()),
        ("cli_default", BeamConfig(beam_width=1, candidates_per_beam=1), ScoringConfig()),
        ("cli_default", BeamConfig(beam_width=3, candidates_per_beam=4), ScoringConfig(scheme=AggregationScheme.MINIMUM)),
        ("mixed_b3", BeamConfig(beam_width=16, candidates_per_beam=2), ScoringConfig(scheme=AggregationScheme.AVERAGE)),
        ("mixed_b3", BeamConfig(beam_width=5, candidates_per_beam=6),
         ScoringConfig(scheme=AggregationScheme.CUMULATIVE_SUM, positive_exit_threshold=0.9)),
        ("mixed_b3", BeamConfig(beam_width=32, candidates_per_beam=1, max_depth=3), ScoringConfig()),
        ("c4_stagnation", BeamConfig(max_depth=40), ScoringConfig()),
        ("c4_stagnation", BeamConfig(beam_width=2, candidates_per_beam=16, max_depth=40, positive_exit_enabled=False),
         ScoringConfig(scheme=AggregationScheme.MINIMUM)),
    ]
    out = []
    for wl, bc, sc in cases:
        results = []
        for p in wls[wl]:
            r = run_beam_search(p, bc, sc)
            b = r.best
            results.append({
                "complete": r.complete, "steps": r.steps, "tokens": r.tokens_generated,
                "best": None if b is None else {"path": list(b.index_path), "rewards": list(b.rewards),
                                                "score": b.score, "terminal": b.is_terminal},
            })
        out.append({"workload": wl, "beam_width": bc.beam_width, "candidates_per_beam": bc.candidates_per_beam,
                    "max_depth": bc.max_depth, "positive_exit_enabled": bc.positive_exit_enabled,
                    "scoring": scoring_record(sc), "results": results})
    dump("beam", out)


def gen_metrics():
    """records_to_csv / summarize (metrics.py:62-128) of the serving wave
    cases on the wave clock (arrival = arrival_step * dt, completion =
    (exit_step + 1) * dt), computed by the reference's metrics module."""
    import gzip as _gz

    from treeserve.metrics import RecordExitKind, RequestRecord, records_to_csv, summarize

    with _gz.open(os.path.join(HERE, "waves.json.gz"), "rt", encoding="utf-8") as f:
        cases = json.load(f)
    out = []
    for c in cases:
        if not c.get("arrival_steps"):
            continue
        for dt in (1.0, 0.05):
            recs = [RequestRecord(o["problem_id"], a * dt, (o["exit_step"] + 1) * dt, o["rollouts_completed"],
                                  o["cancelled"], o["tokens_generated"], RecordExitKind(o["exit_kind"]), o["best_score"],
                                  o["solved"], tuple(o["best_path"]))
                    for o, a in zip(c["outcomes"], c["arrival_steps"]) if o["exit_kind"] != "continue"]
            out.append({"case": c["name"], "dt": dt, "csv": records_to_csv(recs), "summary": summarize(recs).to_json()})
    dump("metrics", out)


def gen_tree_json():
    """SearchTree.to_json() (tree.py:183-206) of finished serial searches: the
    byte-level dump format the engine's Engine.tree_json reproduces."""
    D7 = {d: (7, 7) for d in Difficulty}
    c1 = make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)
    mixed = make_workload(97, (0.5, 0.3, 0.2), 77, branching=3,
                          depth_ranges={Difficulty.EASY: (3, 9), Difficulty.HARD_SOLVABLE: (4, 10), Difficulty.UNSOLVABLE: (2, 6)},
                          accept_threshold=0.35)
    out = []
    for wl_name, wl, sc, budget, cap, width, pe, ne in [
        ("c1", c1, ScoringConfig(), 32, 8, 4, True, True),
        ("c1", c1, ScoringConfig(), 32, 8, 4, False, False),
        ("mixed_b3", mixed, ScoringConfig(scheme=AggregationScheme.MINIMUM, positive_exit_threshold=0.6,
                                          first_step_threshold=0.3), 40, 12, 2, True, True),
    ]:
        for idx in (0, 3, 7):
            tree = serial_tree(wl[idx], sc, budget, cap, width, pe, ne)
            out.append({"workload": wl_name, "index": idx, "scoring": scoring_record(sc), "budget": budget,
                        "depth_cap": cap, "expand_width": width, "positive_exit": pe, "negative_exit": ne,
                        "json": tree.to_json()})
    dump("tree_json", out)


def gen_beam_steps():
    """beam_step / expand_beams / prune_candidates (beam.py:76-131) on beams taken
    from reference beam searches mid-run."""
    from treeserve.beam import Beam, BeamConfig, beam_step, expand_beams, prune_candidates

    def brec(b):
        return {"path": list(b.index_path), "rewards": list(b.rewards), "score": b.score, "terminal": b.is_terminal}

    wl = list(make_workload(24, MIX, 5, branching=3, depth_ranges={d: (4, 9) for d in Difficulty}))
    wl2 = list(make_workload(8, MIX, 6, branching=2, depth_ranges={d: (3, 5) for d in Difficulty}))
    out = []
    for pi, problem in enumerate(wl + wl2):
        for bc, sc in [(BeamConfig(beam_width=8, candidates_per_beam=4), ScoringConfig()),
                       (BeamConfig(beam_width=3, candidates_per_beam=4), ScoringConfig(scheme=AggregationScheme.MINIMUM)),
                       (BeamConfig(beam_width=5, candidates_per_beam=6), ScoringConfig(scheme=AggregationScheme.AVERAGE))]:
            active = [Beam(index_path=(), rewards=(), score=0.0)]
            steps = []
            for _ in range(4):
                if not active:
                    break
                cands = expand_beams(active, bc, sc, problem)
                res = beam_step(active, bc, sc, problem)
                surv, fin = prune_candidates(cands, bc.beam_width)
                steps.append({"beams": [brec(b) for b in active],
                              "candidates": [{"beam": brec(c.beam), "order": c.order, "tokens": c.token_count}
                                             for c in cands],
                              "survivors": [brec(b) for b in res.survivors], "finished": [brec(b) for b in res.finished],
                              "tokens": res.tokens_generated, "prune_survivors": [brec(b) for b in surv],
                              "prune_finished": [brec(b) for b in fin]})
                active = res.survivors
            out.append({"workload": "w5" if pi < len(wl) else "w6", "index": pi if pi < len(wl) else pi - len(wl),
                        "beam_width": bc.beam_width, "candidates_per_beam": bc.candidates_per_beam,
                        "max_depth": bc.max_depth, "positive_exit_enabled": bc.positive_exit_enabled,
                        "scoring": scoring_record(sc), "problem": problem_record(problem), "steps": steps})
    dump("beam_steps", out)


def gen_workload_json():
    """workload_to_json (backend.py:359-384) of two workloads: the replay-file bytes."""
    from treeserve.backend import workload_to_json

    D7 = {d: (7, 7) for d in Difficulty}
    out = {"c1": workload_to_json(make_workload(64, MIX, SEED, branching=4, depth_ranges=D7)),
           "cli_default": workload_to_json(make_workload(40, MIX, 20260810))}
    dump("workload_json", out)


def gen_arrivals():
    """Config-5 arrival steps at full size (65,536 Poisson arrivals, simulator.py:193-200):
    the reference generator's cumulative times t_i (``rng.exponential(rate, seed, 21, i)``)
    quantised to waves as int(t_i * steps_per_unit); the first 256 times are stored too."""
    out = {}
    for name, n, rate, seed, spu in (("c5", 65536, 1.0, 20260810, 1.0 / 2800.0), ("cli_500", 500, 5.0, 20260810, 20.0)):
        t, times, steps = 0.0, [], []
        for i in range(n):
            t += rng.exponential(rate, seed, 21, i)
            times.append(t)
            steps.append(int(t * spu))
        out[name] = {"n": n, "rate": rate, "seed": seed, "steps_per_unit": spu, "times_head": times[:256],
                     "steps": steps}
    dump("arrivals", out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "workloads", "steps", "serial", "deep", "waves", "targets", "policy", "beam", "metrics", "tree_json", "beam_steps", "workload_json", "arrivals", "trace", "cost"]
    for w in which:
        globals()["gen_" + w]()
