/*
 * treeserve_b200.h — C-ABI of the B200-native adaptive parallel MCTS engine.
 *
 * The reference (arXiv 2604.00510, /root/reference/pkg) exposes no FFI: its
 * seams are Python functions.  This header is the boundary
 * those Python entry points bind through ctypes; every entry
 * point below names the reference interface it replaces.  Plain pointers and
 * sizes only: no torch types.  All calls return a ts_status; no exception ever
 * crosses the ABI.  One engine = one GPU = one host thread (the reference's
 * single-owner model, tree.py:12-13).
 *
 * Time unit: one wave ("step").  A request's arrival is an integer step, the
 * scheduler's clock is now = step (SchedulerState.now, scheduler.py:100).
 */
#ifndef TREESERVE_B200_H
#define TREESERVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 6
#define TS_MAX_DEPTH 32 /* golden path / reward table length; base_depth <= 31 */
#define TS_MAX_WIDTH 32 /* branching <= one warp                                */
#define TS_MAX_PEERS 8  /* ranks of one node in ts_run_sharded                    */
#define TS_IPC_HANDLE_BYTES 64

/* Status codes, mapped to the reference's exception classes by the shim. */
typedef enum ts_status {
  TS_OK = 0,
  TS_INVALID_ARGUMENT = 1,   /* ValueError                                    */
  TS_TREE_STRUCTURE = 2,     /* TreeStructureError (tree.py:42)               */
  TS_EXHAUSTED = 3,          /* NoExpandableLeafError — per-search, never a call failure */
  TS_ACCOUNTING = 4,         /* AccountingError (tree.py:50)                  */
  TS_UNSUPPORTED_SCHEME = 5, /* UnsupportedSchemeError (scoring.py:38)        */
  TS_POOL_OVERFLOW = 6,      /* node arena exhausted (engine bug signal)      */
  TS_CUDA = 7                /* CUDA runtime failure                          */
} ts_status;

/* AggregationScheme (scoring.py:42-46) */
enum { TS_SCHEME_MINIMUM = 0, TS_SCHEME_PRODUCT = 1, TS_SCHEME_SUM = 2, TS_SCHEME_AVERAGE = 3 };
/* FutilityBound (scoring.py:53-55) */
enum { TS_BOUND_LEAF_REWARD = 0, TS_BOUND_PREFIX_AGGREGATE = 1 };
/* ExitKind (scoring.py:63-67); TS_EXIT_NONE = CONTINUE / still running */
enum { TS_EXIT_NONE = 0, TS_EXIT_POSITIVE = 1, TS_EXIT_NEGATIVE = 2, TS_EXIT_BUDGET = 3 };

/*
 * One search request: the host-precomputed problem-table row.
 * Mirrors SyntheticProblemSpec (backend.py:113-132) plus derived constants:
 * base_depth (backend.py:135-137), golden path (140-141) and the LIFTED golden
 * rewards golden_step_rewards() (201-215, uses pow → computed on the host).
 */
typedef struct ts_problem {
  uint64_t seed;
  int32_t branching;
  int32_t base_depth;          /* max_depth = base_depth + 1 (backend.py:129-132) */
  int32_t golden_len;          /* len(golden_path), or -1 when golden_path is None */
  int32_t hidden_until_depth;  /* RewardProfile.hidden_until_depth */
  int32_t has_shared;          /* RewardProfile.shared_range is not None */
  int32_t arrival_step;        /* serving: step at which the request arrives (0 = batch);
                                  non-decreasing in request order (simulator.py:193-200) */
  double off_lo, off_hi;       /* RewardProfile.off_path_range */
  double shared_lo, shared_hi; /* RewardProfile.shared_range */
  uint8_t golden_path[TS_MAX_DEPTH];
  double golden_rewards[TS_MAX_DEPTH];
} ts_problem;

/*
 * Flattened ScoringConfig (scoring.py:76-103) + SelectionParams (tree.py:92-100)
 * + SchedulerConfig (scheduler.py:77-93) + run_tree_search knobs (search.py:79-88).
 */
typedef struct ts_config {
  int32_t scheme;
  int32_t futility_bound;
  int32_t strict_negative_exit;
  int32_t positive_exit;     /* enable flags (decide_exit, scoring.py:184-190) */
  int32_t negative_exit;
  int32_t rollout_budget;
  int32_t depth_cap;
  int32_t expand_width;
  int32_t max_concurrency;   /* M: caps admitted jobs and in-flight rollouts */
  int32_t obs_threshold;
  int32_t boosting_enabled;
  int32_t _pad0;
  double accept_threshold;
  double positive_exit_threshold;
  double first_step_threshold;
  double c_puct;
  double beta;
  double proximity;
} ts_config;

/* SearchOutcome (search.py:32-42) + wave bookkeeping. */
typedef struct ts_outcome {
  int32_t exit_kind;
  int32_t rollouts_completed;
  int64_t tokens_generated;
  double best_score;
  int32_t best_len;
  int32_t solved;
  int32_t exit_step;  /* wave index of the exit decision, -1 if none */
  int32_t admit_step; /* wave index of admission (admit_jobs), -1 if never */
  int32_t launched;   /* rollouts launched (completed + cancelled) */
  int32_t cancelled;  /* rollouts cancelled by an exit mid-wave (cancel_inflight) */
  int32_t nodes;      /* len(tree.nodes) */
  int32_t status;     /* per-search ts_status (TS_OK, or the error it hit) */
  uint8_t best_path[TS_MAX_DEPTH];
} ts_outcome;

/* Counters of one engine since its last ts_load_problems. */
typedef struct ts_run_stats {
  int32_t steps;          /* waves executed (1 + last exit step for ts_run) */
  int32_t finished;       /* searches with an exit decision */
  int64_t rollouts;       /* completed (backpropagated) rollouts */
  int64_t launched;       /* launched rollouts */
  int64_t nodes;          /* nodes created (roots excluded) */
  int64_t tokens;
  int64_t children_scored;/* selection work (WU-PUCT evaluations) */
  int64_t select_levels;  /* selection descent levels */
  int64_t path_nodes;     /* Σ (trajectory length + 1) over completed+cancelled rollouts */
  int64_t kernel_launches;/* engine kernels launched since ts_load_problems (host count) */
  double wave_ms;         /* Σ device time of the wave kernels (CUDA events on the launch stream) */
} ts_run_stats;

/* One scheduler record per search, all-gathered across ranks in global
 * run-queue order before ts_step_targets. */
typedef struct ts_sched_record {
  double score;           /* parallelism_score S(i,t), scheduler.py:118-128 */
  uint32_t flags;         /* bit0 running, bit1 ungated (completed >= obs), bit2 boosted */
  uint32_t _pad;
} ts_sched_record;

typedef struct ts_engine ts_engine;

/* ---- engine lifetime ---------------------------------------------------- */
/* Replaces constructing SearchTree/ProblemBackend/SchedulerState per request
 * (tree.py:120, backend.py:275, scheduler.py:96).  Validates the config the
 * way the reference's frozen dataclasses do (__post_init__). */
int ts_engine_create(const ts_config* cfg, int32_t device, ts_engine** out);
int ts_engine_destroy(ts_engine* eng);
const char* ts_last_error(const ts_engine* eng);
int ts_abi_version(void);

/* Upload a batch of requests (host array) and reset every tree to a bare root
 * (SearchTree.__init__, tree.py:120-128).  The n_local searches are the
 * contiguous block [global_offset, global_offset + n_local) of an n_global
 * run queue sharded over ranks (n_global = n_local on one GPU).  Sizes the
 * SoA node pool from rollout_budget × width × min(depth_cap, base_depth+1). */
int ts_load_problems(ts_engine* eng, const ts_problem* host_problems, int32_t n_local,
                     int32_t global_offset, int32_t n_global, void* stream);

/* ---- one step (wave), in call order; ts_run composes them on one GPU ----- */
/* Local counts before admission: dev_counts[0..2] = {running, arrived-but-
 * pending (arrival_step <= step), unfinished}.  For multi-GPU, all-gather
 * these (world × 3 int64) before ts_step_admit. */
int ts_step_counts(ts_engine* eng, int32_t step, int64_t* dev_counts, void* stream);
/* admit_jobs (scheduler.py:131-140) as one global FIFO over ranks. */
int ts_step_admit(ts_engine* eng, int32_t step, const int64_t* dev_all_counts, int32_t world,
                  int32_t rank, void* stream);
/* parallelism_score per local search (scheduler.py:118-128) → n_local records. */
int ts_step_records(ts_engine* eng, int32_t step, ts_sched_record* dev_records, void* stream);
/* compute_targets (scheduler.py:143-187) over all n_global records (global
 * run-queue order); keeps this rank's P_i and builds the wave's work list. */
int ts_step_targets(ts_engine* eng, int32_t step, const ts_sched_record* dev_all_records,
                    void* stream);
/* An external scheduler's targets instead of ts_step_targets: dev_targets[i]
 * = P_i for local search i (call after ts_step_records, which marks this
 * step's admissions as running); running searches get max(1, P_i). */
int ts_step_set_targets(ts_engine* eng, int32_t step, const int32_t* dev_targets, void* stream);
/* The Job fields an external scheduler needs (scheduler.py:63-74), per local
 * search, into device arrays (any may be NULL): running (1/0),
 * completed_rollouts, best_score.  Call after ts_step_records. */
int ts_read_jobs(ts_engine* eng, int32_t* dev_running, int32_t* dev_completed, double* dev_best, void* stream);
/* One wave for every running search with its target P_i: select_leaf →
 * simulate_to_terminal ×min(P_i, budget-completed), then finish_rollout →
 * decide_exit per rollout in launch order, cancel_inflight on exit
 * (search.py:95-107, simulator.py:367-501). */
int ts_step_wave(ts_engine* eng, int32_t step, void* stream);

/* Whole batch on one GPU: the five calls above per step until every search
 * has exited (or max_steps).  stats_out may be NULL. */
int ts_run(ts_engine* eng, int32_t max_steps, ts_run_stats* stats_out, void* stream);

/* ---- multi-GPU: the sharded batch over peer memory ---------
 * Replaces the per-wave all-gathers of ts_step_counts / ts_step_records plus
 * a host round trip.  Each rank owns an exchange buffer (ts_xchg_bytes: a
 * 512-byte header of flags and counts, then n_global scheduler records);
 * every rank writes its counts and records straight into every rank's buffer
 * (NVLink stores through CUDA IPC mappings, or device stores when several
 * ranks share a device in one process) and raises a flag there, and waits on
 * the flags in its own buffer.  Unequal shards are fine (each rank writes at
 * its global offset).  Call order on every rank: ts_load_problems →
 * ts_xchg_create (allocates and zeroes this rank's buffer; ipc_handle_out,
 * TS_IPC_HANDLE_BYTES, may be NULL for in-process ranks) → exchange the
 * handles (any host collective) and a barrier → ts_xchg_connect (ipc_handles:
 * world × TS_IPC_HANDLE_BYTES, or dev_ptrs: world device pointers for ranks
 * in this process; entry rank is ignored) → ts_run_sharded per batch (a
 * collective: every rank the same number of times, with the same
 * last_arrival_global = the largest arrival_step of the whole run queue).
 * ts_run_sharded is ts_run's device-driven graph loop with the exchange
 * inside; stats_out->steps is the global wave count.  A peer that stops
 * signalling for 20 s fails the call with TS_CUDA instead of hanging.
 * Checked mode, the trace and the cost-model clock are ts_run features
 * (TS_INVALID_ARGUMENT here). */
int64_t ts_xchg_bytes(int32_t n_global);
int ts_xchg_create(ts_engine* eng, int32_t world, int32_t rank, void** dev_ptr_out, uint8_t* ipc_handle_out);
int ts_xchg_connect(ts_engine* eng, const uint8_t* ipc_handles, void* const* dev_ptrs);
int ts_run_sharded(ts_engine* eng, int32_t max_steps, int32_t last_arrival_global, ts_run_stats* stats_out,
                   void* stream);
/* Per wave of the last ts_run_sharded (first n waves, n <= 65536): three
 * %globaltimer stamps (ns) — the counts phase starts (the previous wave's
 * kernels are done), every rank's records are in, compute_targets is done. */
int ts_read_px_times(ts_engine* eng, uint64_t* host_out, int32_t n, void* stream);

/* ---- run-time invariants (checked mode) ---------------------------------- */
/* The reference asserts these while it runs (Engine._check_capacity and the
 * conservation check, simulator.py:252-260; test_acceptance.py:167-187,
 * test_simulator.py:58-64).  With checks enabled, two extra kernels bracket
 * every wave (ts_run's graph loop and ts_step_wave alike) and count
 * violations on the device; ts_read_invariants reads the counts since the
 * last ts_load_problems.  All *_violations / inflight_nodes / root_mismatches
 * are 0 on a correct run. */
typedef struct ts_invariants {
  int64_t waves;                   /* waves checked */
  int64_t capacity_violations;     /* waves with Σ min(P_i, budget-completed_i) > M, or |running| > M */
  int64_t gate_violations;         /* searches below obs_threshold given P_i > 1 */
  int64_t inflight_nodes;          /* nodes with O != 0 after a wave (every launch backed up or cancelled) */
  int64_t conservation_violations; /* searches with launched != completed + cancelled after a wave */
  int64_t root_mismatches;         /* searches whose root N != completed_rollouts after a wave */
  int64_t max_wave_launched;       /* largest number of rollouts in flight in one wave */
  int64_t max_running;             /* largest run queue */
} ts_invariants;
int ts_engine_set_checks(ts_engine* eng, int32_t enable);
int ts_read_invariants(ts_engine* eng, ts_invariants* host_out, void* stream);

/* ---- allocation trace ------------------------------------------------------
 * Replaces the reference's per-pass trace records (simulator.py:314-341,
 * written to <preset>_<rate>_trace.jsonl by cli.py:263-265): with a trace
 * buffer set, one row per running search per scheduler pass is written between
 * the pass and its wave (ts_run's graph loop and ts_step_wave alike).  The
 * row holds the "allocation" record's fields; the "action" record follows
 * from them (reconcile, scheduler.py:199-214: every wave starts with no rollout
 * in flight, so the action is launch(target)).  Rows are in completion order
 * of the writing threads; sort by (step, job) for run-queue order. */
typedef struct ts_trace_row {
  int32_t step;   /* the pass's step (now = step * dt) */
  int32_t job;    /* global run-queue index (job_id) */
  int32_t target; /* compute_targets(...)[job] */
  int32_t active; /* len(job.active_rollouts) at the pass: 0 in the wave model */
  double score;   /* parallelism_score(job, now, θ_pos, config) (scheduler.py:118-128) */
} ts_trace_row;
/* ---- wave clock of the cost model ------------------------------
 * The reference's simulated time (CostModel / service_time, backend.py:287-311,
 * charged per generation request, simulator.py:443-463) restated on waves:
 * every expansion of a launched rollout takes
 *   ((max candidate token_count * per_token_latency) * contention) + reward_latency,
 * contention = max(1, load / engine_capacity), load = the wave's in-flight
 * candidates (sum over the wave's launched rollouts of the expansion width),
 * accumulated onto the wave's start clock in expansion order; a search's wave
 * ends with its last rollout and the clock advances to the latest end (idle
 * steps take no time).  engine_capacity = 0 turns it off; otherwise the
 * parameters are validated like CostModel (ValueError).  One engine only (the
 * load is the whole run queue's). */
int ts_engine_set_cost_model(ts_engine* eng, double per_token_latency, int32_t engine_capacity,
                             double reward_latency);
/* Per local search [0, n): simulated completion (the end of its exit wave, 0
 * if not exited) and simulated arrival (the clock at its arrival step). */
int ts_read_sim_times(ts_engine* eng, double* host_completion, double* host_arrival, int32_t n, void* stream);

/* capacity = rows kept per run (0 frees the buffer and disables the trace);
 * rows past it are counted as dropped. */
int ts_engine_set_trace(ts_engine* eng, int64_t capacity);
/* Rows of the run since the last ts_load_problems: copies min(n, cap) rows,
 * *n_out = rows held, *dropped = rows lost to a full buffer (may be NULL). */
int ts_read_trace(ts_engine* eng, ts_trace_row* host_out, int64_t cap, int64_t* n_out, int64_t* dropped,
                  void* stream);

/* ---- readout ------------------------------------------------------------ */
/* Device→host SearchOutcome records for local searches [0, n). */
int ts_read_outcomes(ts_engine* eng, ts_outcome* host_out, int32_t n, void* stream);
int ts_read_stats(ts_engine* eng, ts_run_stats* host_out, void* stream);
/* Targets P_i of the last ts_step_targets for local searches [0, n) (0 = not
 * running); call between ts_step_targets and ts_step_wave. */
int ts_read_targets(ts_engine* eng, int32_t* host_out, int32_t n, void* stream);
/* Per-search latency in ns (device %globaltimer): exit decision time minus the
 * start of the admission step; 0 for searches that have not exited. */
int ts_read_latencies(ts_engine* eng, uint64_t* host_ns, int32_t n, void* stream);
/* Device timestamps (ns, %globaltimer) at the start of each step [0, n). */
int ts_read_step_times(ts_engine* eng, uint64_t* host_out, int32_t n, void* stream);

/* End-to-end: host problems in, host outcomes out (H2D, run, D2H). */
int ts_run_batch_host(ts_engine* eng, const ts_problem* host_problems, int32_t n,
                      int32_t max_steps, ts_outcome* host_out, ts_run_stats* stats_out, void* stream);

/* Tree dump in the SearchTree.to_dict schema (tree.py:183-203); arrays sized
 * by ts_tree_size.  Any pointer may be NULL to skip that field.  step_ref of
 * the root is -1. */
int ts_tree_size(ts_engine* eng, int32_t search, int32_t* nodes_out);
int ts_dump_tree(ts_engine* eng, int32_t search, int32_t* parent, double* reward, double* prior,
                 int32_t* visits, int32_t* inflight, double* value_sum, uint8_t* terminal,
                 int32_t* depth, int32_t* step_ref);

/* Host-side problem-table builder (make_problem + golden_step_rewards,
 * backend.py:144-215): fills *out from the spec fields. */
int ts_fill_problem(uint64_t seed, int32_t solvable, int32_t depth_lo, int32_t depth_hi,
                    int32_t branching, double golden_lo, double golden_hi, double off_lo,
                    double off_hi, int32_t hidden_until_depth, int32_t has_shared,
                    double shared_lo, double shared_hi, double target_aggregate,
                    ts_problem* out);

/* ---- standalone batched policy operators (csrc/policy.cu) ------------------
 * The reference's scheduler and exit-policy entry points applied to state the
 * caller owns (its own run queue or trees), for callers that do not run whole
 * searches in an engine.  No engine handle: errors are reported by the return
 * code and ts_policy_last_error().  Every device pointer is read on `stream`;
 * the calls that return a ValueError condition synchronise the stream. */
const char* ts_policy_last_error(void);

/* SchedulerConfig (scheduler.py:77-93) + positive_exit_threshold. */
typedef struct ts_sched_params {
  int64_t max_concurrency;
  double beta;
  double proximity;
  int32_t obs_threshold;
  int32_t boosting_enabled;
  double positive_exit_threshold;
} ts_sched_params;

/* Diagnostics of one ts_compute_targets call. */
typedef struct ts_targets_info {
  double total_score;      /* Σ S over the run queue (CPython sum semantics) */
  int64_t ungated;         /* jobs past the observation gate */
  int32_t first_bad;       /* lowest index with now < arrival (n if none) */
  int32_t sum_fallback;    /* 1 if Σ S needed the sequential loop */
  int32_t kernel_launches;
  int32_t _pad;
} ts_targets_info;

/* parallelism_score (scheduler.py:118-128) for n jobs: scores[i] =
 * log1p(now - arrival[i]) + (beta if best[i]/θ_pos > proximity else 0), log1p
 * bit-identical to the host libm.  TS_INVALID_ARGUMENT (ValueError) when some
 * now < arrival[i]; *host_first_bad = the lowest such i (n if none). */
int ts_parallelism_scores(double now, double positive_exit_threshold, double beta, double proximity,
                          const double* dev_arrival, const double* dev_best, int32_t n, double* dev_scores,
                          int32_t* host_first_bad, void* stream);

/* compute_targets (scheduler.py:143-187) for a run queue of n RUNNING jobs in
 * run-queue order (device arrays; job ids unique): dev_targets[i] = the
 * target parallelism of job i.  Any arrival order is accepted (the ungated
 * jobs are sorted on the device by (-S, arrival, id)).  Errors as the
 * reference: n == 0 → "run queue holds no running jobs", now < arrival →
 * ValueError (only when boosting is enabled, like the reference). */
int ts_compute_targets(const ts_sched_params* params, double now, const double* dev_arrival,
                       const double* dev_best, const int32_t* dev_completed, const int64_t* dev_job_id,
                       int32_t n, int32_t* dev_targets, ts_targets_info* host_info, void* stream);

/* reconcile (scheduler.py:199-214) with choose_preemption_victims (190-196)
 * over a run queue of n_jobs jobs in run-queue order: job j's in-flight
 * rollouts (Job.active_rollouts) are entries [offsets[j], offsets[j+1]) of
 * prefix_score / rollout_id (InflightRollout, scheduler.py:59-62).  Outputs:
 * launch[j] = target - active when a running job is below its target
 * (LaunchAction), else 0; victim_rank[r] = the rank of rollout r among its
 * job's in-flight rollouts by (prefix_score, rollout_id) when it is one of
 * the active - target victims of a running job above its target
 * (PreemptAction, emitted in rank order), else -1.  dev_running may be NULL
 * (every job running; the reference skips jobs whose state is not RUNNING). */
int ts_reconcile(const int32_t* dev_running, const int32_t* dev_targets, const int64_t* dev_offsets,
                 const double* dev_prefix_score, const int64_t* dev_rollout_id, int32_t n_jobs, int32_t* dev_launch,
                 int32_t* dev_victim_rank, void* stream);

/* A forest of SearchTrees (tree.py:117-181) in flat device arrays: tree t owns
 * nodes [offsets[t], offsets[t+1]), its root first; parent[] holds forest
 * indices (-1 for a root); per-tree fields feed decide_exit and may be NULL
 * (no best trajectory / not exhausted / no budget check). */
enum { TS_NODE_TERMINAL = 1, TS_NODE_HAS_CHILDREN = 2 };
typedef struct ts_forest {
  int32_t n_trees, n_nodes;
  const int32_t* offsets;    /* n_trees + 1 */
  const int32_t* tree_of;    /* n_nodes: owning tree */
  const int32_t* parent;     /* n_nodes */
  const double* reward;      /* n_nodes: prm_reward */
  const int32_t* depth;      /* n_nodes: StepNode.depth */
  const uint8_t* flags;      /* n_nodes: TS_NODE_* */
  const double* best_score;  /* n_trees: best_trajectory.aggregate_score */
  const uint8_t* has_best;   /* n_trees: best_trajectory is not None */
  const int32_t* completed;  /* n_trees: completed_rollouts */
  const int32_t* budget;     /* n_trees: rollout_budget */
  const uint8_t* exhausted;  /* n_trees: decide_exit(tree_exhausted=...) */
} ts_forest;

/* check_negative_exit (scoring.py:153-175) and decide_exit (184-207) for every
 * tree of the forest under one ScoringConfig + enable flags (cfg->scheme,
 * futility_bound, strict_negative_exit, accept_threshold, first_step_threshold,
 * positive_exit_threshold, positive_exit, negative_exit; other fields unused).
 * dev_ne[t] (may be NULL) = 1 if check_negative_exit fires, 0 if not, 2 if it
 * would raise UnsupportedSchemeError (a check-relevant leaf under SUM/AVERAGE).
 * dev_kind[t] (may be NULL) = the ExitKind (TS_EXIT_*; NONE = CONTINUE), or
 * -TS_UNSUPPORTED_SCHEME where decide_exit raises. */
int ts_exit_policy(const ts_config* cfg, const ts_forest* forest, int32_t* dev_kind, uint8_t* dev_ne,
                   void* stream);

/* ---- beam-search baseline (csrc/beam.cu) ---------------
 * run_beam_search (beam.py:143-176) for many problems at once, one warp per
 * problem: every step expands each surviving beam into candidates_per_beam
 * sampled steps (expand_beams, beam.py:76-104), retires terminal candidates,
 * keeps the top beam_width of the rest by (-score, candidate order)
 * (prune_candidates, 107-117), and stops at max_depth, on an empty beam, or
 * (when enabled) once the best finished score reaches positive_exit_threshold.
 * This engine runs beam_width * candidates_per_beam <= TS_BEAM_MAX_CANDIDATES. */
#define TS_BEAM_MAX_CANDIDATES 32
/* BeamConfig (beam.py:30-41) + the ScoringConfig fields the beam reads. */
typedef struct ts_beam_config {
  int32_t beam_width;
  int32_t candidates_per_beam;
  int32_t max_depth;
  int32_t positive_exit_enabled;
  int32_t scheme;                  /* AggregationScheme of the accumulated score */
  int32_t _pad;
  double positive_exit_threshold;
} ts_beam_config;
/* BeamResult (beam.py:62-68): best finished beam, or the best surviving partial
 * (complete = 0), or none (has_best = 0). */
typedef struct ts_beam_result {
  int32_t complete;
  int32_t has_best;
  int32_t is_terminal;             /* Beam.is_terminal of the best beam */
  int32_t best_len;                /* len(index_path) */
  int32_t steps;
  int32_t status;                  /* ts_status of this problem */
  int64_t tokens_generated;
  double best_score;
  uint8_t best_path[TS_MAX_DEPTH];
  double best_rewards[TS_MAX_DEPTH];
} ts_beam_result;
int ts_beam_search(const ts_beam_config* cfg, const ts_problem* dev_problems, int32_t n,
                   ts_beam_result* dev_results, void* stream);
/* End to end: host problems in, host results out (H2D, kernel, D2H). */
int ts_beam_search_host(const ts_beam_config* cfg, const ts_problem* host_problems, int32_t n,
                        ts_beam_result* host_results, void* stream);

/* Step-level beam operators (beam.py:44-131) for callers that drive the loop
 * themselves: expand_beams + prune_candidates for many problems at once. */
typedef struct ts_beam {          /* Beam (beam.py:44-51) */
  int32_t len;                    /* len(index_path) */
  int32_t is_terminal;
  double score;
  uint8_t path[TS_MAX_DEPTH];
  double rewards[TS_MAX_DEPTH];
} ts_beam;
typedef struct ts_beam_candidate { /* BeamCandidate (beam.py:54-59) + the pruning result */
  int32_t beam;                   /* index of the extended input beam */
  int32_t order;                  /* candidate index within the step (tie-break) */
  int32_t step_ref;
  int32_t token_count;
  double prm_reward;
  double score;                   /* aggregate_trajectory of the extended rewards */
  int32_t is_terminal;
  int32_t rank;                   /* prune_candidates: survivor slot, -1 pruned, -2 finished */
} ts_beam_candidate;
/* expand_beams (beam.py:76-104) then prune_candidates (107-117) for problem i:
 * input beams dev_beams[i * TS_BEAM_MAX_CANDIDATES + b], b < dev_counts[i]
 * (counts * candidates_per_beam <= TS_BEAM_MAX_CANDIDATES); candidates out in
 * dev_cands[i * TS_BEAM_MAX_CANDIDATES + j], beam-major, each with its rank
 * among the non-terminal candidates under (-score, order) (rank < beam_width
 * survives).  Per-problem status (ValueError on a terminal or too-deep
 * context, generate_steps backend.py:244-246) in dev_status[i]. */
int ts_beam_expand(const ts_beam_config* cfg, const ts_problem* dev_problems, int32_t n, const ts_beam* dev_beams,
                   const int32_t* dev_counts, ts_beam_candidate* dev_cands, int32_t* dev_status, void* stream);
/* prune_candidates (beam.py:107-117) over caller candidates (score, order,
 * is_terminal used; rank written): n <= 1024 candidates of one problem. */
int ts_beam_prune(ts_beam_candidate* dev_cands, int32_t n, int32_t beam_width, void* stream);

/* ---- the synthetic backend as an operator (csrc/steps.cu) -------------------
 * generate_steps (backend.py:230-269) for n (problem, context path) pairs:
 * candidate j of pair i in dev_out[i * width + j].  dev_paths holds
 * TS_MAX_DEPTH bytes per pair, dev_lens the context lengths; dev_status[i] =
 * TS_INVALID_ARGUMENT where the reference raises ValueError (terminal or
 * too-deep context).  width <= TS_MAX_WIDTH. */
typedef struct ts_step_candidate { /* StepCandidate (backend.py:62-70) */
  int32_t step_ref;
  int32_t token_count;
  double prior;
  double prm_reward;
  int32_t is_terminal;
  int32_t _pad;
} ts_step_candidate;
int ts_generate_steps(const ts_problem* dev_problems, int32_t n, const uint8_t* dev_paths, const int32_t* dev_lens,
                      int32_t width, ts_step_candidate* dev_out, int32_t* dev_status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TREESERVE_B200_H */
