"""Wave oracle composed ONLY of reference calls (fixture generation, this container only).

This module imports the UNMODIFIED reference from ``/root/reference/pkg/src`` and
defines the step-synchronous "wave" semantics the B200 engine implements
(SURVEY.md §8(c)).  It is test infrastructure: it is run here to produce the
committed fixtures under ``tests/golden/``; nothing on the GPU box imports it.

One step (wave), for every running job in run-queue order:

* ``state.now = step * dt``; ``admit_jobs`` (FIFO, arrivals with
  ``arrival_step <= step``); ``compute_targets`` (scheduler.py:143-187) gives P_i.
* launch clamp ``n = min(P_i, budget - completed)`` (simulator.py:373-375);
  for k < n: ``select_leaf`` (tree.py:264) -> ``simulate_to_terminal``
  (tree.py:322).  ``NoExpandableLeafError`` at k == 0 ends the job with
  ``decide_exit(tree_exhausted=True)`` (search.py:96-102, simulator.py:376-388);
  at k > 0 it stops launching for this wave.
* in launch order: ``finish_rollout`` (search.py:63) -> ``decide_exit``
  (scoring.py:184) -> ``on_rollout_complete`` (scheduler.py:217); a non-CONTINUE
  decision cancels the wave's remaining rollouts with ``cancel_inflight``
  (tree.py:374) on their root..terminal paths (simulator.py:495-497).

With boosting off (targets all 1) this is exactly ``run_tree_search`` per job.
"""

from __future__ import annotations

import sys
from collections import deque

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from treeserve.backend import ProblemBackend, service_time  # noqa: E402
from treeserve.scheduler import (  # noqa: E402
    Job,
    JobState,
    SchedulerConfig,
    SchedulerState,
    admit_jobs,
    compute_targets,
    on_rollout_complete,
    parallelism_score,
    reconcile,
)
from treeserve.scheduler import LaunchAction  # noqa: E402
from treeserve.scoring import ExitKind, ScoringConfig, decide_exit  # noqa: E402
from treeserve.search import _CountingBackend, finish_rollout, trajectory_index_path  # noqa: E402
from treeserve.tree import (  # noqa: E402
    NoExpandableLeafError,
    SearchTree,
    SelectionParams,
    cancel_inflight,
    select_leaf,
    simulate_to_terminal,
)


def run_waves(
    problems,
    scoring: ScoringConfig | None = None,
    selection: SelectionParams | None = None,
    sched: SchedulerConfig | None = None,
    rollout_budget: int = 32,
    depth_cap: int = 16,
    expand_width: int = 4,
    positive_exit: bool = True,
    negative_exit: bool = True,
    arrival_steps=None,
    dt: float = 1.0,
    max_steps: int = 1_000_000,
    keep_trees: bool = False,
    trace=None,
    cost=None,
):
    """``trace``: a list that receives the per-pass records of the reference's
    trace (simulator.py:314-341: "allocation" per running job, then the
    "action" records of ``reconcile``), plus a "job_finished" record when a
    job exits (the event record of simulator.py:240-249 without the heap's
    ``seq``).

    ``cost``: a reference ``CostModel`` (backend.py:287-311) drives the WAVE
    CLOCK: each launched rollout's generation requests (its expansions, in
    order) take ``max(service_time(c.token_count, cost, load) for c) +
    cost.reward_latency`` each (simulator.py:443-463), accumulated onto the
    wave's start clock like the reference's event times; ``load`` is the
    wave's in-flight candidate count, sum over the wave's launched rollouts of
    the expansion width; a job's wave ends with its last rollout, the clock
    advances to the latest job's end (idle steps take no time).  A job's
    simulated arrival is the clock at its arrival step, its completion the end
    of its exit wave."""
    scoring = scoring or ScoringConfig()
    selection = selection or SelectionParams()
    sched = sched or SchedulerConfig()
    n = len(problems)
    if arrival_steps is None:
        arrival_steps = [0] * n
    state = SchedulerState()
    jobs = [
        Job(job_id=i, arrival_time=arrival_steps[i] * dt, tree=SearchTree(rollout_budget))
        for i in range(n)
    ]
    backends = [_CountingBackend(ProblemBackend(p, expand_width)) for p in problems]
    exit_step = [-1] * n
    admit_step = [-1] * n
    decisions = [None] * n
    launched_total = [0] * n
    cancelled_total = [0] * n
    targets_trace = []
    next_arrival = 0
    step = 0
    clock = 0.0
    clock_at = []
    sim_done = [None] * n
    rec_toks = None  # per launched rollout of the current job: max token count of each expansion

    if cost is not None:
        class _Rec:
            def __init__(self, inner):
                self.inner = inner

            def candidates_for(self, tree, node_id):
                cands = self.inner.candidates_for(tree, node_id)
                rec_toks[-1].append([c.token_count for c in cands])
                return cands

        backends = [_Rec(b) for b in backends]
    while step < max_steps:
        while next_arrival < n and arrival_steps[next_arrival] <= step:
            state.pending_queue.append(jobs[next_arrival])
            next_arrival += 1
        if next_arrival >= n and not state.pending_queue and not state.run_queue:
            break
        clock_at.append(clock)
        state.now = step * dt
        for job in admit_jobs(state, sched):
            admit_step[job.job_id] = step
        running = [j for j in state.run_queue if j.state is JobState.RUNNING]
        if not running:
            step += 1
            continue
        targets = compute_targets(state, sched, scoring.positive_exit_threshold)
        targets_trace.append([targets[j.job_id] for j in running])
        if trace is not None:
            now = state.now
            for job in running:
                trace.append({"time": round(now, 9), "kind": "allocation", "job": job.job_id,
                              "score": round(parallelism_score(job, now, scoring.positive_exit_threshold, sched), 9),
                              "target": targets[job.job_id], "active": len(job.active_rollouts)})
            for action in reconcile(state, targets):
                entry = ({"action": "launch", "count": action.count} if isinstance(action, LaunchAction)
                         else {"action": "preempt", "rollout": action.rollout_id})
                trace.append({"time": round(now, 9), "kind": "action", "job": action.job_id, **entry})
        wave_rollouts = {}  # job -> [[token counts of each expansion] per launched rollout]
        finished_now = []
        for job in list(running):
            i = job.job_id
            tree = job.tree
            backend = backends[i]
            rec_toks = wave_rollouts.setdefault(i, [])
            P = targets[i]
            count = min(P, tree.rollout_budget - tree.completed_rollouts)
            terms = []
            finished = False
            for k in range(count):
                try:
                    leaf = select_leaf(tree, selection)
                except NoExpandableLeafError:
                    if k == 0:
                        d = decide_exit(tree, scoring, positive_exit, negative_exit, tree_exhausted=True)
                        on_rollout_complete(state, job, d)
                        decisions[i] = d
                        exit_step[i] = step
                        finished = True
                        finished_now.append(i)
                        if trace is not None:
                            trace.append({"time": round(state.now, 9), "kind": "job_finished", "job": i,
                                          "rollout": None})
                    break
                if cost is not None:
                    rec_toks.append([])
                terms.append(simulate_to_terminal(tree, leaf, backend, depth_cap))
            launched_total[i] += len(terms)
            if finished:
                continue
            for idx, term in enumerate(terms):
                finish_rollout(tree, term, scoring)
                d = decide_exit(tree, scoring, positive_exit, negative_exit)
                on_rollout_complete(state, job, d)
                if d.kind is not ExitKind.CONTINUE:
                    for t2 in terms[idx + 1:]:
                        cancel_inflight(tree, tree.path_to_root(t2))
                        cancelled_total[i] += 1
                    decisions[i] = d
                    exit_step[i] = step
                    finished_now.append(i)
                    if trace is not None:
                        trace.append({"time": round(state.now, 9), "kind": "job_finished", "job": i,
                                      "rollout": None})
                    break
        if cost is not None:
            load = sum(min(expand_width, problems[i].branching) * len(r) for i, r in wave_rollouts.items())
            latest = clock
            for i, rolls in wave_rollouts.items():
                end = clock
                for exps in rolls:
                    t = clock
                    for toks in exps:
                        t = t + (max(service_time(tc, cost, load) for tc in toks) + cost.reward_latency)
                    end = max(end, t)
                if i in finished_now:
                    sim_done[i] = end
                latest = max(latest, end)
            clock = latest
        step += 1
    out = []
    for i, (job, problem) in enumerate(zip(jobs, problems)):
        tree = job.tree
        best = tree.best_trajectory
        best_path = trajectory_index_path(tree, best) if best else ()
        rec = {
            "problem_id": problem.problem_id,
            "exit_kind": decisions[i].kind.value if decisions[i] else None,
            "best_score": best.aggregate_score if best else 0.0,
            "best_path": list(best_path),
            "rollouts_completed": tree.completed_rollouts,
            "tokens_generated": getattr(backends[i], "inner", backends[i]).tokens,
            "solved": problem.golden_path is not None and tuple(best_path) == problem.golden_path,
            "exit_step": exit_step[i],
            "admit_step": admit_step[i],
            "launched": launched_total[i],
            "cancelled": cancelled_total[i],
            "nodes": len(tree.nodes),
        }
        if keep_trees:
            rec["tree"] = tree
        if cost is not None:
            rec["sim_arrival"] = clock_at[arrival_steps[i]]
            rec["sim_completion"] = sim_done[i]
        out.append(rec)
    return out, {"steps": step, "targets_trace": targets_trace}
