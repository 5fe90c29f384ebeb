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
 */
#ifndef TREESERVE_B200_H
#define TREESERVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 1
#define TS_MAX_DEPTH 32 /* deepest node any search may create            */
#define TS_MAX_WIDTH 32 /* min(expand_width, branching) ≤ one warp       */

/* Status codes, mapped to the reference's exception classes by the shim. */
typedef enum ts_status {
  TS_OK = 0,
  TS_INVALID_ARGUMENT = 1, /* ValueError                       */
  TS_TREE_STRUCTURE = 2,   /* TreeStructureError (tree.py:42)  */
  TS_EXHAUSTED = 3,        /* NoExpandableLeafError — per-search flag, never a call failure */
  TS_ACCOUNTING = 4,       /* AccountingError (tree.py:50)     */
  TS_UNSUPPORTED_SCHEME = 5, /* UnsupportedSchemeError (scoring.py:38) */
  TS_POOL_OVERFLOW = 6,    /* node arena exhausted (engine bug signal) */
  TS_CUDA = 7              /* CUDA runtime failure              */
} ts_status;

/* AggregationScheme (scoring.py:42-46) */
enum { TS_SCHEME_MINIMUM = 0, TS_SCHEME_PRODUCT = 1, TS_SCHEME_SUM = 2, TS_SCHEME_AVERAGE = 3 };
/* FutilityBound (scoring.py:53-55) */
enum { TS_BOUND_LEAF_REWARD = 0, TS_BOUND_PREFIX_AGGREGATE = 1 };
/* ExitKind (scoring.py:63-67); TS_EXIT_NONE = still running */
enum { TS_EXIT_NONE = 0, TS_EXIT_POSITIVE = 1, TS_EXIT_NEGATIVE = 2, TS_EXIT_BUDGET = 3 };

/*
 * One search request: the host-precomputed problem table row.
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
  int32_t arrival_step;        /* serving: step at which the request arrives (0 = batch) */
  double off_lo, off_hi;       /* RewardProfile.off_path_range */
  double shared_lo, shared_hi; /* RewardProfile.shared_range */
  uint8_t golden_path[TS_MAX_DEPTH];
  double golden_rewards[TS_MAX_DEPTH];
} ts_problem;

/*
 * Flattened ScoringConfig (scoring.py:76-103) + SelectionParams (tree.py:92-100)
 * + SchedulerConfig (scheduler.py:77-93) + run_tree_search knobs (search.py:79-88).
 * Time unit: one wave (step).  now = step, arrival = arrival_step.
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

/* Per-run statistics of one batch (ts_run). */
typedef struct ts_run_stats {
  int32_t steps;          /* waves executed */
  int32_t finished;       /* searches with an exit decision */
  int64_t rollouts;       /* completed (backpropagated) rollouts */
  int64_t launched;       /* launched rollouts */
  int64_t nodes;          /* nodes created */
  int64_t tokens;
  int64_t children_scored;/* selection work (WU-PUCT evaluations) */
  int64_t select_levels;  /* selection descent levels */
  int64_t path_nodes;     /* Σ (trajectory length + 1) over completed+cancelled rollouts */
} ts_run_stats;

typedef struct ts_engine ts_engine;

/* ---- engine lifetime ---------------------------------------------------- */
/* Replaces constructing SearchTree/ProblemBackend/SchedulerState per request
 * (tree.py:120, backend.py:275, scheduler.py:96).  capacity = max searches. */
int ts_engine_create(const ts_config* cfg, int32_t device, int32_t capacity, ts_engine** out);
int ts_engine_destroy(ts_engine* eng);
const char* ts_last_error(const ts_engine* eng);
int ts_abi_version(void);

/* Upload a batch of problems (host array) and reset every tree to a bare root
 * (SearchTree.__init__, tree.py:120-128).  Searches get local ids 0..n-1.
 * global_offset/global_stride place them in the global run queue when the
 * batch is sharded over ranks (global id = global_offset + i*global_stride). */
int ts_load_problems(ts_engine* eng, const ts_problem* host_problems, int32_t n,
                     int32_t global_offset, int32_t global_stride, void* stream);

/* One wave for every running search with its current target P_i:
 * select_leaf → simulate_to_terminal (×min(P_i, budget-completed)), then
 * finish_rollout → decide_exit per rollout in launch order, cancel_inflight on
 * exit (search.py:95-107, simulator.py:367-501).            */
int ts_wave(ts_engine* eng, int32_t step, void* stream);

/* Scheduler, local half: admission (admit_jobs, scheduler.py:131-140) is
 * global; this writes the per-search record {S_i, flags} (parallelism_score,
 * scheduler.py:118-128) into dev_records[local] (2 doubles each).          */
int ts_sched_records(ts_engine* eng, int32_t step, double* dev_records, void* stream);

/* Scheduler, global half: compute_targets (scheduler.py:143-187) over the
 * gathered records of all ranks (world_size blocks of n_local_max records,
 * rank-major), writing this rank's P_i.  Single GPU: world_size = 1.     */
int ts_sched_targets(ts_engine* eng, int32_t step, const double* dev_all_records,
                     int32_t world_size, int32_t n_local_max, int32_t rank, void* stream);

/* Admission (admit_jobs) for the serving loop: admit queued arrivals while the
 * GLOBAL running count < M.  dev_counts = {global running, global admitted}. */
int ts_admit(ts_engine* eng, int32_t step, const int64_t* dev_global_counts, void* stream);
int ts_local_counts(ts_engine* eng, int64_t* dev_counts_out, void* stream);

/* Whole batch on one GPU: admission + targets + waves until every search has
 * exited (or max_steps).  Equivalent to ts_admit, ts_sched_records, ts_sched_targets, ts_wave per step. */
int ts_run(ts_engine* eng, int32_t max_steps, ts_run_stats* stats_out, void* stream);

/* Device→host readout of SearchOutcome records for searches [0, n). */
int ts_read_outcomes(ts_engine* eng, ts_outcome* host_out, int32_t n, void* stream);
int ts_read_stats(ts_engine* eng, ts_run_stats* host_out, void* stream);

/* End-to-end: host problems in, host outcomes out (H2D, run, D2H). */
int ts_run_batch_host(ts_engine* eng, const ts_problem* host_problems, int32_t n,
                      int32_t max_steps, ts_outcome* host_out, ts_run_stats* stats_out, void* stream);

/* Tree dump in the SearchTree.to_dict schema (tree.py:183-203); arrays sized
 * by ts_tree_size.  Any pointer may be NULL to skip that field. */
int ts_tree_size(ts_engine* eng, int32_t search, int32_t* nodes_out);
int ts_dump_tree(ts_engine* eng, int32_t search, int32_t* parent, double* reward, double* prior,
                 int32_t* visits, int32_t* inflight, double* value_sum, uint8_t* terminal,
                 int32_t* depth, int32_t* step_ref);

/* Host-side problem-table builder (make_problem + golden_step_rewards,
 * backend.py:144-215): fills derived fields of *out from the spec fields. */
int ts_fill_problem(uint64_t seed, int32_t solvable, int32_t depth_lo, int32_t depth_hi,
                    int32_t branching, double golden_lo, double golden_hi, double off_lo,
                    double off_hi, int32_t hidden_until_depth, int32_t has_shared,
                    double shared_lo, double shared_hi, double target_aggregate,
                    ts_problem* out);

#ifdef __cplusplus
}
#endif
#endif /* TREESERVE_B200_H */
