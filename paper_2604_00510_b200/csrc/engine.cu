// engine.cu — B200-native (sm_100a) engine for the data-parallel core of the
// adaptive parallel MCTS of arXiv 2604.00510 (reference: /root/reference/pkg,
// "treeserve").  One warp owns one search; thousands of searches advance one
// wave per step.  See DESIGN.md for layout, kernels and rooflines.
//
// Numerics: compiled with -fmad=false; every floating-point expression keeps
// the reference's evaluation order, so results are
// bit-identical to the CPU reference.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/treeserve_b200.h"
#include "exact.cuh"
#include "rng.cuh"

namespace {
using tsx::u128;
using tsx::to_fixed;
using tsx::fixed_to_double;
using tsx::MIX_INIT;
using tsx::sm64;
using tsx::u53;
using tsx::Agg;

constexpr unsigned FULL = 0xffffffffu;

// ---- node meta word (one u32 per node) -------------------------------------
constexpr uint32_t M_DEPTH = 0x3Fu;       // bits 0-5: depth (root 0, <= 32)
constexpr int SH_REF = 6;                 // bits 6-10: step_ref (child index)
constexpr uint32_t M_TERM = 1u << 11;     // is_terminal
constexpr uint32_t M_FORCED = 1u << 12;   // force_terminated (tree.py:340-343)
constexpr uint32_t M_KIDS = 1u << 13;     // has children
constexpr int SH_NEXP = 16;               // bits 16-21: # expandable children
constexpr uint32_t NEXP_ONE = 1u << SH_NEXP;
constexpr uint64_t O_ONE = 1ull << 32;    // no word: N in low 32, O (in-flight) in high 32

__host__ __device__ inline uint64_t mk_mf(int fc, uint32_t meta) {
  return ((uint64_t)(uint32_t)fc << 32) | (uint64_t)meta;
}
__host__ __device__ inline int meta_nexp(uint32_t m) { return (int)((m >> SH_NEXP) & 0x3Fu); }
// _expandable (tree.py:175-181), maintained incrementally: a non-terminal
// node is expandable iff it is a leaf or one of its children is.
__host__ __device__ inline bool meta_expandable(uint32_t m) {
  // bitwise, so that no branch is emitted on the selection chain
  return ((m & M_TERM) == 0) & (((m & M_KIDS) == 0) | ((m & (0x3Fu << SH_NEXP)) != 0));
}

enum { ST_PENDING = 0, ST_RUNNING = 1, ST_FINISHED = 2 };

// Per-search state (SoA would split one warp's scalar reads over many lines;
// a search's row is touched only by its owning warp and the scheduler).
struct __align__(16) SearchState {
  // the scheduler's inputs share the first 16 bytes (one vector load in k_sched)
  int32_t state, completed;
  double job_best;  // Job.best_score (scheduler.py:71, refreshed by on_rollout_complete)
  int32_t launched, cancelled;
  int32_t nodes, viable, best_term, exit_kind;
  int32_t exit_step, admit_step, status, _pad;
  int64_t tokens;
  double best;      // best trajectory score, valid iff best_term >= 0
  unsigned long long t_exit;  // %globaltimer at the exit decision
};
static_assert(sizeof(SearchState) == 80, "SearchState layout");

struct Counters {
  long long running, head, finished, last_exit_step;
  long long step, max_steps;  // device-side step counter of ts_run's graph loop
  long long win_lo;           // lowest admitted search that may still be running (k_sched window)
  int cur_step, _pad;
  long long admit_lo, admit_hi;
  int work_count, work_next;
  int heavy_count, heavy_next;  // searches with >= HEAVY_P rollouts this wave (pipelined CTA mode)
  int heavy_next2, _pad_h;      // k_heavy's claims beyond the first round
  int sum_fallbacks, sched_error;
  unsigned long long rollouts, launched, nodes, tokens, scored, levels, path_nodes, cancelled;
  unsigned long long prof[32];  // TS_HEAVY_PROF diagnostics (cycles), zero otherwise
  // invariant checks (ts_engine_set_checks): ts_invariants in order, and the
  // current wave's Σ launched rollouts
  long long inv[8];
  long long inv_wave;
  // ts_engine_set_trace: rows written / rows dropped (buffer full)
  unsigned long long trace_n, trace_drop;
  // ts_engine_set_cost_model: the wave clock (s) at the current wave's start,
  // the latest end of a search's wave so far (bits of a double >= 0), and the
  // wave's in-flight candidate count
  double clock;
  unsigned long long clock_max;
  long long cost_load;
  long long clock_step1;  // 1 + the last step whose start clock was recorded (0: none)
  // ts_run_sharded: the batch has ended (every later kernel of the graph body
  // returns at once), (unused), a peer timed out (1) or the score sum needs the sequential loop (2)
  int px_done, px_blocks, px_err, px_gen;  // px_gen: the batch generation (epochs of the flags)
  int px_last_arrival, _pad4;              // the run queue's last arrival step (admission exchange)
  // free-running waves (see k_sched): on for this pass, its first step, the
  // waves it covers, the next (search, chunk) item; scheduler passes so far
  int free_run, free_t0, free_rem, _pad5;
  unsigned long long free_next;
  long long passes;
};

// Kernel-side view of one engine.
struct View {
  // SoA node pool; search s owns nodes [s*cap, (s+1)*cap), ids in creation order
  uint64_t* no;      // N | O << 32
  double* W;         // value_sum
  double* Q;         // mean value W/N, valid when N > 0 (rewritten at every backup)
  double* prior;
  double* reward;    // prm_reward
  uint64_t* mf;      // meta (low 32) | first child (high 32, -1 for leaves; children are
                     // contiguous): one 8-byte word, so a reader sees both old or both new
  int32_t* parent;
  long long cap;
  SearchState* st;
  const ts_problem* prob;
  const int32_t* arrival;  // local arrival steps (non-decreasing)
  Counters* ctr;
  int32_t* work;           // this wave's running local searches (single-warp mode)
  int32_t* work_heavy;     // this wave's searches for the pipelined CTA mode
  int32_t* tgt;            // P_i of this wave per local search (compute_targets)
  ts_sched_record* nrec;   // next wave's scheduler record per search, written by the wave (see k_sched)
  int32_t heavy_on;        // pipelined mode available (uniform width 2/4/8)
  int32_t heavy_sync;      // diagnostics: commit every job before the next selection
  int32_t max_arrival;     // last arrival step of the loaded requests
  int32_t* sp;             // scratch paths of a multi-rollout wave [n_local][budget][32]
  double* ss;              // scratch scores
  int32_t* sl;             // scratch lengths
  const double* log1p_tab; // log1p(k) computed by the host libm, k < log1p_n
  int32_t log1p_n;
  int32_t checks;          // ts_engine_set_checks: invariant kernels around every wave
  int32_t free_ok;         // free-running waves allowed (k_sched decides per pass); see k_sched
  int32_t free_kernel;     // the graph runs them in k_wave_free (else k_wave does)
  int32_t* fdone;          // free-running: chunks of a search's rollouts done
  ts_trace_row* trace;     // ts_engine_set_trace: allocation rows of every pass (null: off)
  long long trace_cap;
  // ts_engine_set_cost_model (cost_cap 0: off)
  double cost_pt, cost_rl;
  int32_t cost_cap;
  int2* cost_snap;         // (nodes, launched) of every search at its wave's start
  double* sim_done;        // simulated completion time of every exited search
  double* clock_at;        // wave clock at the start of every step (step_times_cap entries)
  int32_t n_local, goff, n_global;
  unsigned long long* step_times;
  int32_t step_times_cap;
  // targets-kernel scratch (global fallback when runs exceed shared memory)
  // ts_run_sharded: every rank's exchange buffer (this process's mapping, px[prank]
  // is this rank's own), the batch generation, and whether admission needs
  // the counts exchange (capacity below the run queue) or up to which step
  unsigned char* px[TS_MAX_PEERS];
  int32_t pworld, prank, padm_all;
  unsigned long long* pstamp;  // per wave: counts phase start, every group table in, scheduler done (%globaltimer)
  unsigned char* pscr;         // group scheduler scratch (px_scratch_bytes)
  int32_t pgwarp;              // k_px_step: one-warp scheduler up to this many table entries (<= 32)
  double* g_runS;
  int32_t* g_runStart;
  long long* g_runWant;
  long long* g_runPW;
  ts_config cfg;
};

// ---- warp helpers ------------------------------------------------------------
// argmax with strict '>' and the lowest index winning ties (tree.py:258, 316);
// lanes >= wp2 (a power of two >= width) must be invalid.
// The double is mapped to an order-preserving u64 key (-0.0 folded into +0.0,
// so equal values tie) and reduced with two REDUX steps; the lowest winning
// lane is the first child among equals.  Invalid lanes never win.
__device__ __forceinline__ int warp_argmax(double v, bool valid, int /*wp2*/) {
  const uint64_t b = (uint64_t)__double_as_longlong(v + 0.0);
  const uint64_t key = (b >> 63) ? ~b : (b | (1ull << 63));
  const unsigned hi = valid ? (unsigned)(key >> 32) : 0u;
  const unsigned lo = valid ? (unsigned)key : 0u;
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  const unsigned win = __ballot_sync(FULL, valid && hi == mh && lo == ml);
  return __ffs(win) - 1;
}

// warp_argmax for values that are never -0.0 (WU-PUCT scores: q >= +0 and the
// exploration term >= +0), without the fold of -0.0 into +0.0.
__device__ __forceinline__ int warp_argmax_nonneg(double v, bool valid) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint64_t key = (b >> 63) ? ~b : (b | (1ull << 63));
  const unsigned hi = valid ? (unsigned)(key >> 32) : 0u;
  const unsigned lo = valid ? (unsigned)key : 0u;
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  const unsigned win = __ballot_sync(FULL, valid && hi == mh && lo == ml);
  return __ffs(win) - 1;
}

// Running splitmix64 folds: for every expansion depth d a rollout can reach,
// the lanes hold fold(seed, TAG, len, path[0:depth]) for the four key tags of
// generate_steps (backend.py:230-269): prior (2, d), reward (1, d+1), tokens
// (3, d+1), extend (6, d+1).  Each descent step absorbs the chosen step_ref
// into all of them in parallel, so an expansion at depth d costs O(1) hashes
// on the critical path instead of the reference's O(d) fold per draw.
// NSLOT states per lane; 4 tags x (8*NSLOT) depths = 32*NSLOT states.
template <int NSLOT>
__device__ __forceinline__ void slot_header(int lane, int k, uint64_t& tag, uint64_t& len) {
  constexpr int GS = 8 * NSLOT;
  const int g = lane / GS, d = lane % GS;
  const int t = g * NSLOT + k;
  tag = t == 0 ? 2u : t == 1 ? 1u : t == 2 ? 3u : 6u;
  len = (uint64_t)(t == 0 ? d : d + 1);
}
template <int NSLOT, int T>
__device__ __forceinline__ uint64_t state_at(const uint64_t (&h)[NSLOT], int d) {
  constexpr int GS = 8 * NSLOT;
  return __shfl_sync(FULL, h[T % NSLOT], (T / NSLOT) * GS + d);
}
// The simulation keeps, per depth d it expands, the fold states of that depth:
// lanes with lane % GS == d copy their slots at level d (`snap`).  The prior
// (tag 2, len d) and token (tag 3, len d+1) draws of the w children are not on
// greedy_child's critical path, so they are made in the lane-parallel
// expansion batch instead (lane l = depth l), from these snapshots.
template <int NSLOT>
__device__ __forceinline__ void snap_take(uint64_t (&snap)[NSLOT], const uint64_t (&h)[NSLOT], int d) {
  constexpr int GS = 8 * NSLOT;
  if (((threadIdx.x & 31) % GS) == d) {
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) snap[k] = h[k];
  }
}
template <int NSLOT>
__device__ __forceinline__ void snap_prior_tokens(const uint64_t (&snap)[NSLOT], uint64_t& hp, uint64_t& hk) {
  constexpr int GS = 8 * NSLOT;
  const int l = (threadIdx.x & 31) % GS;
  hp = __shfl_sync(FULL, snap[0 % NSLOT], (0 / NSLOT) * GS + l);
  hk = __shfl_sync(FULL, snap[2 % NSLOT], ((2 / NSLOT) * GS + l) & 31);
}
template <int WT>
__device__ __forceinline__ double pick_raw(const double (&rv)[WT ? WT : 1], const double* rawl, int i) {
  if constexpr (WT > 0) return rv[i];
  else return rawl[i];
}
// generate_steps (backend.py:248-263) for child j of a node whose prior/token
// prefix folds are hp/hk: the raw prior 0.5 + uniform and the token count.
__device__ __forceinline__ double draw_raw_prior(uint64_t hp, int j) { return 0.5 + u53(sm64(hp ^ (uint64_t)j)); }
__device__ __forceinline__ long long draw_tokens(uint64_t hk, int j) {
  return 40 + (long long)(sm64(hk ^ (uint64_t)j) % 81ull);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// TS_SCHED_PROF (diagnostics build): %globaltimer phase stamps of the graph
// loop in Counters::prof, read by tools/sched_prof.py.  Slots: 0 wave end ->
// k_sched start, 1 wave span, 2 k_sched end -> first wave CTA, 3-9 k_sched
// phases, 10 passes, 20/21/22 the current wave's last end / first start and
// the last k_sched end, 30 the batch has ended.
#ifdef TS_SCHED_PROF
#define SP_MARK(slot, t0)                                                       \
  do {                                                                          \
    if (threadIdx.x == 0) {                                                     \
      const unsigned long long t_ = globaltimer();                              \
      atomicAdd(&v.ctr->prof[slot], t_ - (t0));                                 \
      (t0) = t_;                                                                \
    }                                                                           \
  } while (0)
#else
#define SP_MARK(slot, t0) do { } while (0)
#endif

// ---- kernels -------------------------------------------------------------------

// The record of search s for the scheduler pass of step+1, written by the
// search's own wave: the fields k_sched would otherwise gather from the
// SearchState, the arrival and the log1p table (parallelism_score,
// scheduler.py:118-128, the same expressions as the gather).  Bits 8..31 of
// flags tag the step the record is for; NREC_FINAL (an exited search) is valid
// at every later step, NREC_NONE at none.
constexpr uint32_t NREC_FINAL = 0xFFFFFFu, NREC_NONE = 0xFFFFFEu;
__device__ __forceinline__ void write_next_record(const View& v, int s, int step, bool finished, int completed,
                                                  double job_best) {
  ts_sched_record r;
  r.score = 0.0;
  r._pad = 0;
  r.flags = NREC_NONE << 8;
  const int ns = step + 1;
  if (finished) {
    r.flags = NREC_FINAL << 8;
  } else if (ns < v.log1p_n) {
    const ts_config& cf = v.cfg;
    const bool boosted = job_best / cf.positive_exit_threshold > cf.proximity;
    r.score = v.log1p_tab[ns - v.arrival[s]] + (boosted ? cf.beta : 0.0);
    r.flags = 1u | (completed >= cf.obs_threshold ? 2u : 0u) | (boosted ? 4u : 0u) | ((uint32_t)ns << 8);
    r._pad = (uint32_t)completed;
  }
  v.nrec[s] = r;
}

// SearchTree.__init__ (tree.py:120-128): bare root, reward 1.0, prior 1.0.
__global__ void k_init(View v) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) {  // the run's counters (nothing reads them before the next kernel)
    memset(v.ctr, 0, sizeof(Counters));
    v.ctr->last_exit_step = -1;
  }
  if (s >= v.n_local) return;
  size_t r = (size_t)s * (size_t)v.cap;
  v.no[r] = 0;
  v.W[r] = 0.0;
  v.Q[r] = 0.0;
  v.prior[r] = 1.0;
  v.reward[r] = 1.0;
  v.mf[r] = mk_mf(-1, 0);
  v.parent[r] = -1;
  const_cast<int32_t*>(v.arrival)[s] = v.prob[s].arrival_step;  // the run queue's arrival column
  SearchState z;
  z.state = ST_PENDING;
  z.completed = z.launched = z.cancelled = 0;
  z.nodes = 1;
  z.viable = 0;
  z.best_term = -1;
  z.exit_kind = TS_EXIT_NONE;
  z.exit_step = -1;
  z.admit_step = -1;
  z.status = TS_OK;
  z._pad = 0;
  v.tgt[s] = 0;
  ts_sched_record nr0;
  nr0.score = 0.0;
  nr0._pad = 0;
  nr0.flags = NREC_NONE << 8;
  v.nrec[s] = nr0;
  z.tokens = 0;
  z.best = 0.0;
  z.job_best = 0.0;
  z.t_exit = 0;
  v.st[s] = z;
  if (v.sim_done) v.sim_done[s] = 0.0;
}


__global__ void k_set_max_steps(Counters* c, int max_steps) { c->max_steps = max_steps; }

// Local counts before admission: {running, arrived-but-pending, unfinished}.
__global__ void k_counts(View v, int step, long long* out) {
  // arrivals are non-decreasing: upper_bound(arrival, step)
  int lo = 0, hi = v.n_local;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (v.arrival[mid] <= step) lo = mid + 1;
    else hi = mid;
  }
  Counters* c = v.ctr;
  out[0] = c->running;
  out[1] = (long long)lo - c->head;
  out[2] = (long long)v.n_local - c->finished;
}

// admit_jobs (scheduler.py:131-140): one FIFO over the global run queue.
__global__ void k_admit(View v, const long long* all, int world, int rank) {
  long long run_g = 0, pend_g = 0, before = 0;
  for (int r = 0; r < world; ++r) {
    run_g += all[3 * r];
    pend_g += all[3 * r + 1];
    if (r < rank) before += all[3 * r + 1];
  }
  long long A = (long long)v.cfg.max_concurrency - run_g;
  if (A > pend_g) A = pend_g;
  if (A < 0) A = 0;
  long long mine = all[3 * rank + 1];
  long long q = A - before;
  if (q > mine) q = mine;
  if (q < 0) q = 0;
  Counters* c = v.ctr;
  c->admit_lo = c->head;
  c->admit_hi = c->head + q;
  c->head += q;
  c->running += q;
}

// parallelism_score (scheduler.py:118-128) → one record per local search.
__global__ void k_records(View v, int step, ts_sched_record* rec) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.n_local) return;
  SearchState* s = v.st + i;
  const Counters* c = v.ctr;
  int state = s->state;
  if (i >= c->admit_lo && i < c->admit_hi) {
    state = ST_RUNNING;
    s->state = ST_RUNNING;
    s->admit_step = step;
  }
  ts_sched_record r;
  r.score = 0.0;
  r.flags = 0;
  r._pad = 0;
  if (state == ST_RUNNING) {
    const ts_config& cf = v.cfg;
    int waited = step - v.arrival[i];
    double ratio = s->job_best / cf.positive_exit_threshold;
    double boost = ratio > cf.proximity ? cf.beta : 0.0;
    r.score = v.log1p_tab[waited] + boost;
    r.flags = 1u | (s->completed >= cf.obs_threshold ? 2u : 0u) | (ratio > cf.proximity ? 4u : 0u);
    r._pad = (uint32_t)s->completed;
  }
  rec[i] = r;
}

// ---- compute_targets (scheduler.py:143-187) in one CTA ------------------------
constexpr int TT = 1024;
// k_sched and k_targets (targets_block): one CTA whose time is the instruction
// issue of one SM, dominated by the block scans every warp performs, so fewer
// warps with more records each
constexpr int SCHED_T = 1024, SCHED_W = SCHED_T / 32;
constexpr int HEAVY_P = 8;  // rollouts in one wave from which a search runs in pipelined CTA mode
constexpr int HBITS_WORDS = 2048;  // run-queue slots with a pipelined-mode flag bit (65536)
constexpr int SREC_MAX = 4096;     // k_sched keeps the records of up to this many searches in shared memory
constexpr int RUNCAP = 1536;  // runs per list kept in shared memory
constexpr size_t TGT_SCR = (96 + 96 + 32 + 64) * 8;  // targets_block scan scratch (bytes)

// Four exclusive (+) scans in one pass; totals in tot[4].  All threads must call.
__device__ void block_scan_add4(long long (&x)[4], long long (&tot)[4], long long* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    incl[q] = x[q];
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(FULL, incl[q], o);
      if (lane >= o) incl[q] += y;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < 4; ++q) sh[q * 32 + wid] = incl[q];
  }
  __syncthreads();
  if (wid < 4) {
    long long w = sh[wid * 32 + lane];
    long long wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += y;
    }
    sh[128 + wid * 32 + lane] = wi - w;
    if (lane == 31) sh[256 + wid] = wi;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long base = sh[128 + q * 32 + wid];
    tot[q] = sh[256 + q];
    x[q] = base + incl[q] - x[q];
  }
  __syncthreads();
}

// Exclusive min-scan of doubles (identity +inf).
__device__ double block_scan_min(double x, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl = fmin(incl, y);
  }
  double excl = __shfl_up_sync(FULL, incl, 1);
  if (lane == 0) excl = INFINITY;
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    double w = sh[lane];
    double wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi = fmin(wi, y);
    }
    double we = __shfl_up_sync(FULL, wi, 1);
    if (lane == 0) we = INFINITY;
    sh[32 + lane] = we;
  }
  __syncthreads();
  double res = fmin(sh[32 + wid], excl);
  __syncthreads();
  return res;
}

// First run (runs strictly decreasing in S) with runS <= s.
__device__ __forceinline__ int runs_lower(const double* runS, int nr, double s) {
  int lo = 0, hi = nr;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (runS[mid] > s) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// compute_targets over the global run queue (records in global id order).
// The reference sorts ungated jobs by (-S, arrival, id).  Because arrivals
// are non-decreasing in run-queue order and S = log1p(now - arrival) + boost,
// the unboosted and the boosted jobs each form a list already sorted by
// (-S, id) in run-queue order; the sorted order is their merge.  Within a
// list, equal scores form runs with one `want` each; a job's sorted position
// and the Σ(want-1) before it follow from run prefix sums plus a binary
// search in the other list.  The clamp loop (scheduler.py:169-180) then has
// the closed form extra_k = clamp(R - Σ_{j<k}(want_j-1), 0, want_k-1), and the
// round-robin leftover gives floor(R'/U) + [pos < R' mod U] (181-186).
// The score sum Σ S (scheduler.py:165, CPython's Neumaier sum) equals the
// correctly rounded exact sum when all compensation terms are exact (checked
// below); it is computed exactly in 128-bit fixed point.
// rec holds n records in global run-queue order; records [glo, ghi) are this
// engine's searches base + (i - glo).
// Exclusive (+) scans of N values per thread with ONE barrier: lane 31 of each
// warp publishes the warp's inclusive totals, then every warp rescans the 32
// warp totals itself instead of waiting for one warp to publish offsets.  `sh`
// (32*N long longs) may be reused two calls later: the intervening call's
// barrier orders every read of this one before the next write.
template <int N, typename T>
__device__ __forceinline__ void scan1_add(T (&x)[N], T (&tot)[N], T* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    inc[q] = x[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(FULL, inc[q], o);
      if (lane >= o) inc[q] += y;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < N; ++q) sh[q * 32 + wid] = inc[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const T w = lane < (int)(blockDim.x >> 5) ? sh[q * 32 + lane] : (T)0;
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += y;
    }
    tot[q] = __shfl_sync(FULL, wi, 31);
    x[q] = __shfl_sync(FULL, wi - w, wid) + inc[q] - x[q];
  }
}

// compute_targets over the global run queue (records in global id order).
// The reference sorts ungated jobs by (-S, arrival, id).  Because arrivals
// are non-decreasing in run-queue order and S = log1p(now - arrival) + boost,
// the unboosted and the boosted jobs each form a list already sorted by
// (-S, id) in run-queue order; the sorted order is their merge.  Within a
// list, equal scores form runs with one `want` each; a job's sorted position
// and the Σ(want-1) before it follow from run prefix sums plus a binary
// search in the other list.  The clamp loop (scheduler.py:169-180) then has
// the closed form extra_k = clamp(R - Σ_{j<k}(want_j-1), 0, want_k-1), and the
// round-robin leftover gives floor(R'/U) + [pos < R' mod U] (181-186).
// The score sum Σ S (scheduler.py:165, CPython's Neumaier sum) equals the
// correctly rounded exact sum when all compensation terms are exact (checked
// below); it is computed exactly in 128-bit fixed point.
// rec holds n records in global run-queue order; records [glo, ghi) are this
// engine's searches base + (i - glo).  Thread t owns records
// [t*ceil(n/TT), ...) in every pass, so a caller that wrote them with the same
// partition needs no barrier before the call.  Six barriers in all: the
// counts/sum/min scan, the run-count scan, the run table, the want-prefix
// scan, the run prefixes, the work-list scan.
// cid: the records are a compacted run queue (running searches only, in
// run-queue order) and record i's search is base + (flags >> 8)
__device__ void targets_block(const View& v, int step, const ts_sched_record* rec, int n, int glo, int ghi,
                              int base, bool cid = false) {
  extern __shared__ __align__(16) unsigned char smem[];
  long long* shA = (long long*)smem;                  // 96: scan scratch (even calls)
  long long* shB = shA + 96;                          // 96: scan scratch (odd calls)
  long long* shF = shB + 96;                          // 32: per-warp fallback flags
  int* shA32 = (int*)shA;                             // 32-bit views of the scan scratch
  int* shB32 = (int*)shB;
  double* shD = (double*)(shF + 32);                  // 64: per-warp list minima
  u128* shq = (u128*)(smem + TGT_SCR);                // 32: per-warp partial sums
  uint32_t* hbits = (uint32_t*)(smem + TGT_SCR + 32 * 16);  // pipelined-mode flag per run-queue slot
  double* s_runS = (double*)(smem + TGT_SCR + 32 * 16 + HBITS_WORDS * 4);
  int32_t* s_runStart = (int32_t*)(s_runS + 2 * RUNCAP);
  long long* s_runWant = (long long*)(s_runStart + 2 * RUNCAP);
  long long* s_runPW = s_runWant + 2 * RUNCAP;
  __shared__ double sT;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const ts_config& cf = v.cfg;
  if (tid == 0 && step < v.step_times_cap) v.step_times[step] = globaltimer();
#ifdef TS_SCHED_PROF
  unsigned long long sp_t = globaltimer();
#endif
  const int per = (n + SCHED_T - 1) / SCHED_T;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  for (int w = tid; w < (ghi - glo + 31) / 32 && w < HBITS_WORDS; w += SCHED_T) hbits[w] = 0u;

  // phase 1: counts, exact score sum, list positions, list minima before each
  // thread (the lists are non-increasing, so the last score before a thread's
  // range is the minimum over the threads before it)
  u128 fx = 0;
  bool bad = false;
  int c3[3] = {0, 0, 0};  // running, gated-in unboosted (list 0), boosted (list 1)
  double min0 = INFINITY, min1 = INFINITY;
  for (int i = lo; i < hi; ++i) {
    const ts_sched_record r = rec[i];
    if (!(r.flags & 1u)) continue;
    ++c3[0];
    u128 q;
    if (to_fixed(r.score, q)) fx += q;
    else bad = true;
    if (r.flags & 2u) {
      if (r.flags & 4u) { ++c3[2]; min1 = fmin(min1, r.score); }
      else { ++c3[1]; min0 = fmin(min0, r.score); }
    }
  }
  int t3[3];
  double prev0, prev1;
  u128 fsum;
  bool anybad;
  {
    int inc[3];
    double m0 = min0, m1 = min1;
#pragma unroll
    for (int q = 0; q < 3; ++q) inc[q] = c3[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int y = __shfl_up_sync(FULL, inc[q], o);
        if (lane >= o) inc[q] += y;
      }
      const double y0 = __shfl_up_sync(FULL, m0, o), y1 = __shfl_up_sync(FULL, m1, o);
      if (lane >= o) { m0 = fmin(m0, y0); m1 = fmin(m1, y1); }
    }
    double e0 = __shfl_up_sync(FULL, m0, 1), e1 = __shfl_up_sync(FULL, m1, 1);
    if (lane == 0) e0 = e1 = INFINITY;
    u128 x = fx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t h = __shfl_xor_sync(FULL, (uint64_t)(x >> 64), o);
      const uint64_t l = __shfl_xor_sync(FULL, (uint64_t)x, o);
      x += ((u128)h << 64) | l;
    }
    const bool wbad = __any_sync(FULL, bad);
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < 3; ++q) shA32[q * 32 + wid] = inc[q];
      shD[wid] = m0;
      shD[32 + wid] = m1;
    }
    if (lane == 0) {
      shq[wid] = x;
      shF[wid] = wbad;
    }
    __syncthreads();
    // every warp: scans of the warp totals, the block sum, the fallback flag
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int w = lane < SCHED_W ? shA32[q * 32 + lane] : 0;
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, wi, o);
        if (lane >= o) wi += y;
      }
      t3[q] = __shfl_sync(FULL, wi, 31);
      c3[q] = __shfl_sync(FULL, wi - w, wid) + inc[q] - c3[q];
    }
    double w0 = lane < SCHED_W ? shD[lane] : INFINITY, w1 = lane < SCHED_W ? shD[32 + lane] : INFINITY;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y0 = __shfl_up_sync(FULL, w0, o), y1 = __shfl_up_sync(FULL, w1, o);
      if (lane >= o) { w0 = fmin(w0, y0); w1 = fmin(w1, y1); }
    }
    const double b0 = __shfl_sync(FULL, w0, (wid + 31) & 31), b1 = __shfl_sync(FULL, w1, (wid + 31) & 31);
    prev0 = wid == 0 ? e0 : fmin(b0, e0);
    prev1 = wid == 0 ? e1 : fmin(b1, e1);
    fsum = lane < SCHED_W ? shq[lane] : (u128)0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t h = __shfl_xor_sync(FULL, (uint64_t)(fsum >> 64), o);
      const uint64_t l = __shfl_xor_sync(FULL, (uint64_t)fsum, o);
      fsum += ((u128)h << 64) | l;
    }
    anybad = __any_sync(FULL, lane < SCHED_W && shF[lane] != 0);
  }
  const long long tot_run = t3[0], len0 = t3[1], len1 = t3[2];
  const int pos0 = c3[1], pos1 = c3[2];
  double T = 0.0;
  bool fallback = anybad;
  if (!fallback) {
    T = fixed_to_double(fsum);
    // compensation exactness: n * ulp(2T) < 2^-10
    const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
    if ((double)tot_run * u2 >= 0x1p-10) fallback = true;
  }
  if (fallback) {  // block-uniform: sequential Neumaier sum in run-queue order
    if (tid == 0) {
      double f = 0.0, c = 0.0;
      bool first = true;
      for (int i = 0; i < n; ++i) {
        const ts_sched_record r = rec[i];
        if (!(r.flags & 1u)) continue;
        const double x2 = r.score;
        if (first) { f = x2; first = false; continue; }
        const double t = f + x2;
        if (fabs(f) >= fabs(x2)) c += (f - t) + x2;
        else c += (x2 - t) + f;
        f = t;
      }
      if (c != 0.0 && isfinite(c)) f += c;
      sT = f;
      atomicAdd(&v.ctr->sum_fallbacks, 1);
    }
    __syncthreads();
    T = sT;
  }
  SP_MARK(5, sp_t);
  const long long M = cf.max_concurrency;
  const long long R = M - tot_run;
  // no free slot or nobody past the observation gate: every running job gets 1
  const bool boost_on = cf.boosting_enabled != 0 && tot_run > 0 && R > 0 && len0 + len1 > 0;

  // phase 2: runs of equal score in each list (lists are non-increasing)
  int rid[2] = {0, 0}, nrr[2] = {0, 0};
  if (boost_on) {
    double p0 = prev0, p1 = prev1;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = rec[i];
      if ((r.flags & 3u) != 3u) continue;
      if (r.flags & 4u) { if (r.score != p1) ++rid[1]; if (r.score > p1) v.ctr->sched_error = 1; p1 = r.score; }
      else { if (r.score != p0) ++rid[0]; if (r.score > p0) v.ctr->sched_error = 1; p0 = r.score; }
    }
    scan1_add<2>(rid, nrr, shB32);
  }
  const int nr0 = nrr[0], nr1 = nrr[1];
  const bool in_smem = nr0 <= RUNCAP && nr1 <= RUNCAP;
  double* runS = in_smem ? s_runS : v.g_runS;
  int32_t* runStart = in_smem ? s_runStart : v.g_runStart;
  long long* runWant = in_smem ? s_runWant : v.g_runWant;
  long long* runPW = in_smem ? s_runPW : v.g_runPW;
  const int stride = in_smem ? RUNCAP : v.n_global;  // list 1 offset
  long long tw0 = 0, tw1 = 0;
  if (boost_on) {
    {
      double p0 = prev0, p1 = prev1;
      int q0 = pos0, q1 = pos1, k0 = rid[0], k1 = rid[1];
      for (int i = lo; i < hi; ++i) {
        const ts_sched_record r = rec[i];
        if ((r.flags & 3u) != 3u) continue;
        if (r.flags & 4u) {
          if (r.score != p1) { runS[stride + k1] = r.score; runStart[stride + k1] = (int)q1; ++k1; }
          p1 = r.score;
          ++q1;
        } else {
          if (r.score != p0) { runS[k0] = r.score; runStart[k0] = (int)q0; ++k0; }
          p0 = r.score;
          ++q0;
        }
      }
    }
    __syncthreads();
    SP_MARK(6, sp_t);
    // phase 3: want per run, prefix Σ cnt*(want-1) over runs (both lists in one scan)
    long long pre[2] = {0, 0}, tw[2];
    int a0[2], a1[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int nr = b ? nr1 : nr0;
      const int len = (int)(b ? len1 : len0);
      const int off = b ? stride : 0;
      const int per2 = (nr + SCHED_T - 1) / SCHED_T;
      a0[b] = min(tid * per2, nr);
      a1[b] = min(a0[b] + per2, nr);
      for (int k = a0[b]; k < a1[b]; ++k) {
        const double sc = runS[off + k];
        long long want = 1;
        if (T > 0.0) {
          const double f = floor(sc / T * (double)M);
          want = f > 1.0 ? (long long)f : 1;
        }
        const int cnt = (k + 1 < nr ? runStart[off + k + 1] : len) - runStart[off + k];
        runWant[off + k] = want;
        pre[b] += cnt * (want - 1);
      }
    }
    scan1_add<2>(pre, tw, shA);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int nr = b ? nr1 : nr0;
      const int len = (int)(b ? len1 : len0);
      const int off = b ? stride : 0;
      long long q = pre[b];
      for (int k = a0[b]; k < a1[b]; ++k) {
        runPW[off + k] = q;
        const int cnt = (k + 1 < nr ? runStart[off + k + 1] : len) - runStart[off + k];
        q += cnt * (runWant[off + k] - 1);
      }
    }
    tw0 = tw[0];
    tw1 = tw[1];
    __syncthreads();
  }
  SP_MARK(7, sp_t);
  // phase 4: targets; each thread counts its local searches per work list
  const long long U = len0 + len1;
  long long Rp = R - (tw0 + tw1);
  if (Rp < 0) Rp = 0;
  const long long rr_q = U > 0 ? Rp / U : 0, rr_r = U > 0 ? Rp % U : 0;
  int nl2[2] = {0, 0};  // pipelined-mode, single-warp
  {
    int q0 = pos0, q1 = pos1, k0 = rid[0] - 1, k1 = rid[1] - 1;
    double p0 = prev0, p1 = prev1;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = rec[i];
      const bool local = i >= glo && i < ghi;
      if (!(r.flags & 1u)) {
        if (local) v.tgt[cid ? base + (int)(r.flags >> 8) : base + i - glo] = 0;
        continue;
      }
      long long tgt = 1;
      if ((r.flags & 2u) && boost_on) {
        const int b = (r.flags & 4u) ? 1 : 0;
        int pos, k;
        if (b) { if (r.score != p1) ++k1; p1 = r.score; pos = q1++; k = k1; }
        else { if (r.score != p0) ++k0; p0 = r.score; pos = q0++; k = k0; }
        const int off = b ? stride : 0, oo = b ? 0 : stride;
        const long long want = runWant[off + k];
        long long before = runPW[off + k] + (long long)(pos - runStart[off + k]) * (want - 1);
        // cross list: elements with S' > S, or S' == S and smaller id
        const int nro = b ? nr0 : nr1, leno = (int)(b ? len0 : len1);
        const long long two = b ? tw0 : tw1;
        const int obefore = b ? q0 : q1;  // other-list elements with id < i
        const int kk = runs_lower(runS + oo, nro, r.score);
        int c;
        long long cw;
        if (kk < nro && runS[oo + kk] == r.score) {
          const int st0 = runStart[oo + kk];
          const int cntk = (kk + 1 < nro ? runStart[oo + kk + 1] : leno) - st0;
          int part = obefore - st0;
          if (part < 0) part = 0;
          if (part > cntk) part = cntk;
          c = st0 + part;
          cw = runPW[oo + kk] + (long long)part * (runWant[oo + kk] - 1);
        } else if (kk < nro) {
          c = runStart[oo + kk];
          cw = runPW[oo + kk];
        } else {
          c = leno;
          cw = two;
        }
        const int spos = pos + c;
        before += cw;
        long long extra = R - before;
        if (extra < 0) extra = 0;
        if (extra > want - 1) extra = want - 1;
        tgt = 1 + extra + rr_q + (spos < rr_r ? 1 : 0);
      }
      if (local) {
        v.tgt[cid ? base + (int)(r.flags >> 8) : base + i - glo] = (int)tgt;
        // rollouts this wave = min(P_i, budget - completed); `_pad` carries completed
        if (v.heavy_on && min(tgt, (long long)(cf.rollout_budget - (int)r._pad)) >= HEAVY_P) {
          atomicOr(&hbits[(i - glo) >> 5], 1u << ((i - glo) & 31));
          ++nl2[0];
        } else {
          ++nl2[1];
        }
      }
    }
  }
  SP_MARK(8, sp_t);
  // phase 5: the local running searches split into the single-warp and the
  // pipelined (many rollouts this wave) work lists, in run-queue order.  A
  // thread reads back only the flag bits it set itself.
  int tl2[2];
  scan1_add<2>(nl2, tl2, shB32);
  {
    int ph = nl2[0], pl = nl2[1];
    const int loc_lo = max(lo, glo) - glo, loc_hi = max(loc_lo, min(hi, ghi) - glo);
    for (int i = loc_lo; i < loc_hi; ++i) {
      const uint32_t fl = rec[i + glo].flags;
      if (!(fl & 1u)) continue;
      const int id = cid ? base + (int)(fl >> 8) : base + i;
      if ((hbits[i >> 5] >> (i & 31)) & 1u) v.work_heavy[ph++] = id;
      else v.work[pl++] = id;
    }
  }
  if (tid == 0) {
    v.ctr->work_count = (int)tl2[1];
    v.ctr->work_next = 0;
    v.ctr->heavy_count = (int)tl2[0];
    v.ctr->heavy_next = v.ctr->heavy_next2 = 0;
    v.ctr->cur_step = step;
  }
  SP_MARK(9, sp_t);
}

__device__ __forceinline__ size_t targets_smem_dev() {
  return TGT_SCR + 32 * 16 + HBITS_WORDS * 4 + (size_t)2 * RUNCAP * (8 + 4 + 8 + 8);
}

__global__ void __launch_bounds__(SCHED_T) k_targets(View v, int step, const ts_sched_record* rec) {
  targets_block(v, step, rec, v.n_global, v.goff, v.goff + v.n_local, 0);
}

// ---- the sharded wave loop over peer memory (ts_run_sharded) ----------------------
//
// Every rank owns an exchange buffer; a peer writes its scheduler inputs
// straight into every other rank's buffer (NVLink stores through CUDA IPC
// mappings; plain device stores when the ranks are emulated on one GPU) and
// then sets its flag there to the wave's epoch.  A rank waits on the flags in
// its own buffer, so each exchange is one round of peer stores plus one flag
// wait — no collective library call, no host round trip — and the whole
// sharded batch is one device-driven graph loop like ts_run's.
struct XHdr {
  unsigned long long fa[TS_MAX_PEERS];  // counts phase: epoch written by peer p
  unsigned long long fb[TS_MAX_PEERS];  // groups phase
  long long cnt[TS_MAX_PEERS][4];       // peer p: {running, arrived-but-pending, unfinished, -} before admission
  long long unf[TS_MAX_PEERS];          // peer p: unfinished searches when its groups were written
  long long nent[TS_MAX_PEERS];         // peer p: entries of its group table
  long long goff[TS_MAX_PEERS];         // peer p: its global offset (its table starts at entry goff)
};
constexpr size_t XHDR_BYTES = 1024;
// One entry per distinct arrival step among a rank's running searches: the
// running and the ungated (completed >= obs_threshold) counts of the
// unboosted (0) and boosted (1) lists.  parallelism_score depends only on
// (arrival, boosted) (scheduler.py:118-128), so these counts carry everything
// compute_targets needs from the other ranks.
struct PxEnt {
  int a, nr0, nu0, nr1, nu1, _p0, _p1, _p2;
};
static_assert(sizeof(PxEnt) == 32, "group entry");
constexpr int PX_MAX_WAVES = 1 << 20;  // the log1p table ts_xchg_connect sizes for the sharded loop
constexpr int PX_STAMP_WAVES = 1 << 16;  // waves with timestamps (ts_read_px_times)
__device__ __forceinline__ void px_stamp(const View& v, int step, int k) {
  if (step < PX_STAMP_WAVES) v.pstamp[3 * step + k] = globaltimer();
}
static_assert(sizeof(XHdr) <= XHDR_BYTES, "exchange header");
__host__ __device__ inline size_t xchg_bytes(long long n_global) {
  return XHDR_BYTES + (size_t)n_global * sizeof(PxEnt);
}
__device__ __forceinline__ PxEnt* xent(const View& v, int p) { return (PxEnt*)(v.px[p] + XHDR_BYTES); }
__device__ __forceinline__ XHdr* xh(const View& v, int p) { return (XHdr*)v.px[p]; }
__device__ __forceinline__ unsigned long long px_epoch(const View& v, int step) {
  return ((unsigned long long)(uint32_t)v.ctr->px_gen << 32) | (unsigned long long)(uint32_t)(step + 1);
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long x) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long x;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return x;
}
// wait until every peer's flag in this rank's buffer reached `epoch`; a peer
// that stays silent for TS_PX_TIMEOUT_NS ends the batch with an error
#ifndef TS_PX_TIMEOUT_NS
#define TS_PX_TIMEOUT_NS 20000000000ull
#endif
__device__ bool px_wait(const View& v, const unsigned long long* flags, unsigned long long epoch) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < (unsigned)v.pworld) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(flags + threadIdx.x) < epoch) {
      if (globaltimer() - t0 > TS_PX_TIMEOUT_NS) {
        s_ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  return s_ok != 0;
}
__device__ __forceinline__ bool px_adm_active(const View& v, int step) {
  return v.padm_all || step <= v.ctr->px_last_arrival;
}
// the batch ends: every later kernel of the graph returns at once and the
// waves find empty work lists
__device__ void px_finish(const View& v, cudaGraphConditionalHandle cond, int err) {
  Counters* c = v.ctr;
  c->px_done = 1;
  if (err) c->px_err = err;
  c->work_count = 0;
  c->work_next = 0;
  c->heavy_count = 0;
  c->heavy_next = c->heavy_next2 = 0;
  cudaGraphSetConditional(cond, 0);
}

__global__ void k_px_reset(Counters* c, int gen, int last_arrival) {
  c->px_done = 0;
  c->px_blocks = 0;
  c->px_err = 0;
  c->px_gen = gen;
  c->px_last_arrival = last_arrival;
}

// counts phase: this rank's {running, pending, unfinished} into every peer's buffer
__global__ void k_px_counts(View v) {
  Counters* c = v.ctr;
  if (c->px_done) return;
  const int step = (int)c->step;
  if (threadIdx.x == 0) px_stamp(v, step, 0);
  if (!px_adm_active(v, step)) return;
  int lo = 0, hi = v.n_local;  // arrivals are non-decreasing: upper_bound(arrival, step)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v.arrival[mid] <= step) lo = mid + 1;
    else hi = mid;
  }
  const long long run = c->running, pend = (long long)lo - c->head, unf = (long long)v.n_local - c->finished;
  const int p = threadIdx.x;
  if (p < v.pworld) {
    long long* d = xh(v, p)->cnt[v.prank];
    d[0] = run;
    d[1] = pend;
    d[2] = unf;
    __threadfence_system();
    st_release_sys(&xh(v, p)->fa[v.prank], px_epoch(v, step));
  }
}

// admit_jobs (scheduler.py:131-140) over the global FIFO from every rank's
// counts, and the loop test (no unfinished search on any rank)
__global__ void k_px_admit(View v, cudaGraphConditionalHandle cond, int max_steps) {
  Counters* c = v.ctr;
  if (c->px_done) return;
  const int step = (int)c->step;
  if (step >= max_steps || step >= v.log1p_n) {
    if (threadIdx.x == 0) px_finish(v, cond, 0);
    return;
  }
  if (!px_adm_active(v, step)) {
    if (threadIdx.x == 0) c->admit_lo = c->admit_hi = c->head;  // nobody can be pending
    return;
  }
  const XHdr* x = xh(v, v.prank);
  if (!px_wait(v, x->fa, px_epoch(v, step))) {
    if (threadIdx.x == 0) px_finish(v, cond, 1);
    return;
  }
  if (threadIdx.x != 0) return;
  long long run_g = 0, pend_g = 0, before = 0, unf_g = 0;
  for (int r = 0; r < v.pworld; ++r) {
    const long long c0 = __ldcg(&x->cnt[r][0]), c1 = __ldcg(&x->cnt[r][1]), c2 = __ldcg(&x->cnt[r][2]);
    run_g += c0;
    pend_g += c1;
    unf_g += c2;
    if (r < v.prank) before += c1;
  }
  if (unf_g == 0) {
    px_finish(v, cond, 0);
    return;
  }
  long long A = (long long)v.cfg.max_concurrency - run_g;
  if (A > pend_g) A = pend_g;
  if (A < 0) A = 0;
  long long q = A - before;
  if (q > __ldcg(&x->cnt[v.prank][1])) q = __ldcg(&x->cnt[v.prank][1]);
  if (q < 0) q = 0;
  c->admit_lo = c->head;
  c->admit_hi = c->head + q;
  c->head += q;
  c->running += q;
}

// scratch of the group scheduler (k_px_groups / k_px_sched), carved from one buffer
struct PxScr {
  // per local search
  unsigned char *code, *heavy;  // code: segment start | running << 1 | ungated << 2 | list << 3
  int *segid, *jpre;            // arrival segment; exclusive prefix of the ungated of its list
  int4* jq;                     // (entry, position among the ungated of its (entry, list) here, code, completed)
  // per local arrival segment
  int4 *segb, *sege;            // exclusive prefix (run0, ung0, run1, ung1) at its first job / inclusive at its last
  int *sega, *segent;           // arrival; entry (-1: no running search)
  // per entry of the concatenated global table, per merged entry, per run of each list
  int* gm;                      // merged entry
  int4* gp;                     // exclusive prefix (nr0, nu0, nr1, nu1) over the concatenated table
  int* mfirst;                  // first concatenated entry of a merged entry
  int2* mrun;                   // its run in list 0 / list 1 (-1: none)
  double* rS[2];                // run score (non-increasing), arrival, ungated count, want, prefix U, prefix W
  int *rA[2], *rC[2];
  long long *rWant[2], *rU[2], *rW[2];
};
__host__ __device__ inline PxScr px_scr(unsigned char* base, long long nl, long long ng, size_t* bytes) {
  PxScr X;
  size_t o = 0;
  auto take = [&](size_t b) -> unsigned char* {
    unsigned char* q = base ? base + o : nullptr;
    o += (b + 15) & ~(size_t)15;
    return q;
  };
  X.code = take(nl);
  X.heavy = take(nl);
  X.segid = (int*)take(4 * nl);
  X.jpre = (int*)take(4 * nl);
  X.jq = (int4*)take(16 * nl);
  X.segb = (int4*)take(16 * nl);
  X.sege = (int4*)take(16 * nl);
  X.sega = (int*)take(4 * nl);
  X.segent = (int*)take(4 * nl);
  X.gm = (int*)take(4 * ng);
  X.gp = (int4*)take(16 * ng);
  X.mfirst = (int*)take(4 * ng);
  X.mrun = (int2*)take(8 * ng);
  for (int b = 0; b < 2; ++b) {
    X.rS[b] = (double*)take(8 * ng);
    X.rA[b] = (int*)take(4 * ng);
    X.rC[b] = (int*)take(4 * ng);
    X.rWant[b] = (long long*)take(8 * ng);
    X.rU[b] = (long long*)take(8 * ng);
    X.rW[b] = (long long*)take(8 * ng);
  }
  if (bytes) *bytes = o;
  return X;
}

constexpr int PXT = 1024;  // k_px_groups / k_px_sched block size
constexpr int PXS = 512;   // k_px_step block size (128 registers per thread)

// The groups phase: admission state (admit_jobs), then this rank's group
// table — one PxEnt per distinct arrival among its running searches, in
// arrival order — into every rank's buffer at this rank's global offset, and
// each running search's entry and position within it for k_px_sched.
__global__ void __launch_bounds__(PXT) k_px_groups(View v) {
  Counters* c = v.ctr;
  if (c->px_done) return;
  const int step = (int)c->step;
  const int tid = threadIdx.x;
  __shared__ int sh[5 * 32];
  const ts_config& cf = v.cfg;
  const bool fold = cf.beta == 0.0;  // the boosted flag does not change the score: one list
  const int n = v.n_local;
  const PxScr X = px_scr(v.pscr, n, v.n_global, nullptr);
  const int per = (n + PXT - 1) / PXT, lo = min(n, tid * per), hi = min(n, lo + per);
  const long long alo = c->admit_lo, ahi = c->admit_hi;
  int cnt[5] = {0, 0, 0, 0, 0};  // segment starts, run0, ung0, run1, ung1
  for (int i = lo; i < hi; ++i) {
    SearchState* st = v.st + i;
    int state = st->state;
    if (i >= alo && i < ahi) {
      state = ST_RUNNING;
      st->state = ST_RUNNING;
      st->admit_step = step;
    }
    const int a = v.arrival[i];
    const int ap = i > 0 ? v.arrival[i - 1] : a;
    if (a < ap) c->sched_error = 1;
    const bool start = i == 0 || a != ap;
    unsigned code = start ? 1u : 0u;
    int comp = 0;
    if (state == ST_RUNNING) {
      comp = st->completed;
      const bool boosted = st->job_best / cf.positive_exit_threshold > cf.proximity;  // scheduler.py:126
      const bool ung = comp >= cf.obs_threshold;
      const int b = (boosted && !fold) ? 1 : 0;
      code |= 2u | (ung ? 4u : 0u) | ((unsigned)b << 3);
      cnt[1 + 2 * b] += 1;
      if (ung) cnt[2 + 2 * b] += 1;
    }
    cnt[0] += start ? 1 : 0;
    X.code[i] = (unsigned char)code;
    X.jq[i] = make_int4(0, 0, 0, comp);
  }
  int tot[5];
  scan1_add<5>(cnt, tot, sh);
  {
    int q[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) q[k] = cnt[k];
    for (int i = lo; i < hi; ++i) {
      const unsigned code = X.code[i];
      if (code & 1u) {
        X.segb[q[0]] = make_int4(q[1], q[2], q[3], q[4]);
        X.sega[q[0]] = v.arrival[i];
        ++q[0];
      }
      const int sg = q[0] - 1;
      const int b = (code >> 3) & 1;
      X.segid[i] = sg;
      X.jpre[i] = q[2 + 2 * b];
      if (code & 2u) {
        q[1 + 2 * b] += 1;
        if (code & 4u) q[2 + 2 * b] += 1;
      }
      if (i == n - 1 || v.arrival[i + 1] != v.arrival[i]) X.sege[sg] = make_int4(q[1], q[2], q[3], q[4]);
    }
  }
  const int nseg = tot[0];
  __syncthreads();
  const int per2 = (nseg + PXT - 1) / PXT, s0 = min(nseg, tid * per2), s1 = min(nseg, s0 + per2);
  int hr[1] = {0}, hrt[1];
  for (int sg = s0; sg < s1; ++sg) {
    const int4 b0 = X.segb[sg], b1 = X.sege[sg];
    if (b1.x - b0.x + b1.z - b0.z > 0) ++hr[0];
  }
  scan1_add<1>(hr, hrt, sh);
  {
    int id = hr[0];
    for (int sg = s0; sg < s1; ++sg) {
      const int4 b0 = X.segb[sg], b1 = X.sege[sg];
      if (b1.x - b0.x + b1.z - b0.z > 0) {
        PxEnt en;
        en.a = X.sega[sg];
        en.nr0 = b1.x - b0.x;
        en.nu0 = b1.y - b0.y;
        en.nr1 = b1.z - b0.z;
        en.nu1 = b1.w - b0.w;
        en._p0 = en._p1 = en._p2 = 0;
        for (int p = 0; p < v.pworld; ++p) xent(v, p)[v.goff + id] = en;
        X.segent[sg] = id++;
      } else {
        X.segent[sg] = -1;
      }
    }
  }
  const int nent = hrt[0];
  __syncthreads();
  for (int i = lo; i < hi; ++i) {
    const unsigned code = X.code[i];
    int4 q = X.jq[i];
    if (code & 2u) {
      const int sg = X.segid[i];
      const int4 sb = X.segb[sg];
      q.x = X.segent[sg];
      q.y = X.jpre[i] - ((code & 8u) ? sb.w : sb.y);
    } else {
      q.x = -1;
      q.y = 0;
    }
    q.z = (int)code;
    X.jq[i] = q;
  }
  __threadfence_system();
  __syncthreads();
  const int p = tid;
  if (p < v.pworld) {
    XHdr* h = xh(v, p);
    h->nent[v.prank] = nent;
    h->goff[v.prank] = v.goff;
    h->unf[v.prank] = (long long)n - c->finished;
    __threadfence_system();
    st_release_sys(&h->fb[v.prank], px_epoch(v, step));
  }
}

__device__ u128 block_sum_u128(u128 x, bool& bad) {
  __shared__ u128 sq[32];
  __shared__ int sb[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t h = __shfl_xor_sync(FULL, (uint64_t)(x >> 64), o);
    const uint64_t l = __shfl_xor_sync(FULL, (uint64_t)x, o);
    x += ((u128)h << 64) | l;
  }
  const bool wb = __any_sync(FULL, bad);
  if (lane == 0) {
    sq[wid] = x;
    sb[wid] = wb;
  }
  __syncthreads();
  u128 t = lane < (int)(blockDim.x >> 5) ? sq[lane] : (u128)0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t h = __shfl_xor_sync(FULL, (uint64_t)(t >> 64), o);
    const uint64_t l = __shfl_xor_sync(FULL, (uint64_t)t, o);
    t += ((u128)h << 64) | l;
  }
  bad = __any_sync(FULL, lane < (int)(blockDim.x >> 5) && sb[lane] != 0);
  return t;
}

// compute_targets (scheduler.py:143-187) from every rank's group table.  The
// reference sorts the ungated jobs by (-S, arrival, id); S depends only on
// (arrival, boosted), and arrivals are non-decreasing in run-queue order, so
// the sorted order is the merge of the unboosted and the boosted list, each a
// sequence of runs = entries of one arrival (S non-increasing along it),
// ordered inside a run by id.  A job's sorted position and the Σ(want-1)
// before it are run prefix sums, its position inside its run (the run's
// count on lower ranks plus its rank-local position), and a binary search in
// the other list (equal scores there: the earlier arrival first).  The score
// sum is the exact fixed-point sum of count × S (equal to CPython's Neumaier
// sum under the check targets_block documents).  Then the closed forms of the
// clamp and the round robin, and the two work lists, as targets_block.
__global__ void __launch_bounds__(PXT) k_px_sched(View v, cudaGraphConditionalHandle cond) {
  Counters* c = v.ctr;
  if (c->px_done) return;
  const int step = (int)c->step;
  const int tid = threadIdx.x;
  const XHdr* x = xh(v, v.prank);
  if (!px_wait(v, x->fb, px_epoch(v, step))) {
    if (tid == 0) px_finish(v, cond, 1);
    return;
  }
  if (tid == 0) px_stamp(v, step, 1);
  __shared__ int shi[5 * 32];
  __shared__ long long shl[4 * 32];
  const ts_config& cf = v.cfg;
  const int W = v.pworld;
  int off[TS_MAX_PEERS + 1];
  long long gof[TS_MAX_PEERS];
  long long unf_g = 0;
  off[0] = 0;
  for (int r = 0; r < W; ++r) {
    unf_g += __ldcg(&x->unf[r]);
    off[r + 1] = off[r] + (int)__ldcg(&x->nent[r]);
    gof[r] = __ldcg(&x->goff[r]);
  }
  if (unf_g == 0) {
    if (tid == 0) px_finish(v, cond, 0);
    return;
  }
  const int G = off[W];
  const PxEnt* tab = xent(v, v.prank);
  // entries written by peers: read from L2 (ld.global.cg), never a stale L1 line
  auto ent = [&](int g) -> PxEnt {
    int r = 0;
    while (r + 1 < W && off[r + 1] <= g) ++r;
    const int4* e4 = (const int4*)(tab + gof[r] + (g - off[r]));
    const int4 u = __ldcg(e4), w = __ldcg(e4 + 1);
    PxEnt e;
    e.a = u.x;
    e.nr0 = u.y;
    e.nu0 = u.z;
    e.nr1 = u.w;
    e.nu1 = w.x;
    e._p0 = e._p1 = e._p2 = 0;
    return e;
  };
  const PxScr X = px_scr(v.pscr, v.n_local, v.n_global, nullptr);
  // 1. merged entries (equal arrivals at rank boundaries) and the exclusive
  //    prefix of the counts over the concatenated table
  const int pg = (G + PXT - 1) / PXT, g0 = min(G, tid * pg), g1 = min(G, g0 + pg);
  int cg[5] = {0, 0, 0, 0, 0}, tg[5];
  for (int g = g0; g < g1; ++g) {
    const PxEnt e = ent(g);
    cg[0] += (g == 0 || e.a != ent(g - 1).a) ? 1 : 0;
    cg[1] += e.nr0;
    cg[2] += e.nu0;
    cg[3] += e.nr1;
    cg[4] += e.nu1;
  }
  scan1_add<5>(cg, tg, shi);
  for (int g = g0; g < g1; ++g) {
    const PxEnt e = ent(g);
    if (g == 0 || e.a != ent(g - 1).a) X.mfirst[cg[0]++] = g;
    X.gm[g] = cg[0] - 1;
    X.gp[g] = make_int4(cg[1], cg[2], cg[3], cg[4]);
    cg[1] += e.nr0;
    cg[2] += e.nu0;
    cg[3] += e.nr1;
    cg[4] += e.nu1;
  }
  const int Gm = tg[0];
  const long long tot_run = (long long)tg[1] + tg[3], len0 = tg[2], len1 = tg[4];
  const int4 ptot = make_int4(tg[1], tg[2], tg[3], tg[4]);
  __syncthreads();
  // 2. per merged entry: its counts and scores, the exact score sum, runs per list
  const int pm = (Gm + PXT - 1) / PXT, m0 = min(Gm, tid * pm), m1 = min(Gm, m0 + pm);
  auto mcounts = [&](int m, int& a, int4& k) {
    const int ga = X.mfirst[m], gb = m + 1 < Gm ? X.mfirst[m + 1] : G;
    const int4 pa = X.gp[ga], pb = gb < G ? X.gp[gb] : ptot;
    k = make_int4(pb.x - pa.x, pb.y - pa.y, pb.z - pa.z, pb.w - pa.w);
    a = ent(ga).a;
  };
  u128 fx = 0;
  bool bad = false;
  int cr[2] = {0, 0}, tr[2];
  for (int m = m0; m < m1; ++m) {
    int a;
    int4 k;
    mcounts(m, a, k);
    // parallelism_score as the records phase writes it: log1p(waited) + boost
    const double S0 = v.log1p_tab[step - a] + 0.0, S1 = v.log1p_tab[step - a] + cf.beta;
    u128 q;
    if (k.x > 0) {
      if (to_fixed(S0, q)) fx += q * (u128)(unsigned)k.x;
      else bad = true;
    }
    if (k.z > 0) {
      if (to_fixed(S1, q)) fx += q * (u128)(unsigned)k.z;
      else bad = true;
    }
    cr[0] += k.y > 0 ? 1 : 0;
    cr[1] += k.w > 0 ? 1 : 0;
  }
  scan1_add<2>(cr, tr, shi);
  const u128 fsum = block_sum_u128(fx, bad);
  for (int m = m0; m < m1; ++m) {
    int a;
    int4 k;
    mcounts(m, a, k);
    const double S0 = v.log1p_tab[step - a] + 0.0, S1 = v.log1p_tab[step - a] + cf.beta;
    int2 mr = make_int2(-1, -1);
    if (k.y > 0) {
      X.rS[0][cr[0]] = S0;
      X.rA[0][cr[0]] = a;
      X.rC[0][cr[0]] = k.y;
      mr.x = cr[0]++;
    }
    if (k.w > 0) {
      X.rS[1][cr[1]] = S1;
      X.rA[1][cr[1]] = a;
      X.rC[1][cr[1]] = k.w;
      mr.y = cr[1]++;
    }
    X.mrun[m] = mr;
  }
  const int nrun[2] = {tr[0], tr[1]};
  double T = fixed_to_double(fsum);
  {
    const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
    if (bad || (double)tot_run * u2 >= 0x1p-10) {  // would need the sequential sum (targets_block)
      if (tid == 0) px_finish(v, cond, 2);
      return;
    }
  }
  __syncthreads();
  // 3. want per run, exclusive prefixes U (count) and W (count * (want-1)) per list
  const long long M = cf.max_concurrency;
  const long long R = M - tot_run;
  const bool boost_on = cf.boosting_enabled != 0 && tot_run > 0 && R > 0 && len0 + len1 > 0;
  long long tw[2] = {0, 0}, lenl[2] = {len0, len1};
  if (boost_on) {
    long long pre[4] = {0, 0, 0, 0}, tot4[4];
    int a0[2], a1[2];
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int pr = (nrun[b] + PXT - 1) / PXT;
      a0[b] = min(nrun[b], tid * pr);
      a1[b] = min(nrun[b], a0[b] + pr);
      for (int k = a0[b]; k < a1[b]; ++k) {
        long long want = 1;
        if (T > 0.0) {
          const double f = floor(X.rS[b][k] / T * (double)M);  // scheduler.py:173-175
          want = f > 1.0 ? (long long)f : 1;
        }
        X.rWant[b][k] = want;
        pre[2 * b] += X.rC[b][k];
        pre[2 * b + 1] += (long long)X.rC[b][k] * (want - 1);
      }
    }
    scan1_add<4>(pre, tot4, shl);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      long long u = pre[2 * b], w = pre[2 * b + 1];
      for (int k = a0[b]; k < a1[b]; ++k) {
        X.rU[b][k] = u;
        X.rW[b][k] = w;
        u += X.rC[b][k];
        w += (long long)X.rC[b][k] * (X.rWant[b][k] - 1);
      }
    }
    tw[0] = tot4[1];
    tw[1] = tot4[3];
    __syncthreads();
  }
  // 4. targets of this rank's searches, and the two work lists in run-queue order
  const long long U = len0 + len1;
  long long Rp = R - (tw[0] + tw[1]);
  if (Rp < 0) Rp = 0;
  const long long rr_q = U > 0 ? Rp / U : 0, rr_r = U > 0 ? Rp % U : 0;
  const int n = v.n_local, me = v.prank;
  const int per = (n + PXT - 1) / PXT, lo = min(n, tid * per), hi = min(n, lo + per);
  int nl2[2] = {0, 0}, tl2[2];
  for (int i = lo; i < hi; ++i) {
    const int4 q = X.jq[i];
    const unsigned code = (unsigned)q.z;
    unsigned char hv = 0;
    if (!(code & 2u)) {
      v.tgt[i] = 0;
      X.heavy[i] = 2;  // not running
      continue;
    }
    long long tgt = 1;
    if ((code & 4u) && boost_on) {
      const int b = (code >> 3) & 1, o = 1 - b;
      const int g = off[me] + q.x, m = X.gm[g];
      const int k = b ? X.mrun[m].y : X.mrun[m].x;
      const int4 pg0 = X.gp[X.mfirst[m]], pgg = X.gp[g];
      const long long qt = (long long)q.y + (b ? pgg.w - pg0.w : pgg.y - pg0.y);
      const long long want = X.rWant[b][k];
      const double S = X.rS[b][k];
      const int a = X.rA[b][k];
      long long pos = X.rU[b][k] + qt;
      long long before = X.rW[b][k] + qt * (want - 1);
      int kk = runs_lower(X.rS[o], nrun[o], S);  // other-list runs with a higher score
      if (kk < nrun[o] && X.rS[o][kk] == S && X.rA[o][kk] < a) ++kk;  // equal score: earlier arrival first
      pos += kk < nrun[o] ? X.rU[o][kk] : lenl[o];
      before += kk < nrun[o] ? X.rW[o][kk] : tw[o];
      long long extra = R - before;
      if (extra < 0) extra = 0;
      if (extra > want - 1) extra = want - 1;
      tgt = 1 + extra + rr_q + (pos < rr_r ? 1 : 0);
    }
    v.tgt[i] = (int)tgt;
    if (v.heavy_on && min(tgt, (long long)(cf.rollout_budget - q.w)) >= HEAVY_P) hv = 1;
    X.heavy[i] = hv;
    ++nl2[hv ? 0 : 1];
  }
  scan1_add<2>(nl2, tl2, shi);
  {
    int ph = nl2[0], pl = nl2[1];
    for (int i = lo; i < hi; ++i) {
      const unsigned char hv = X.heavy[i];
      if (hv == 2) continue;
      if (hv) v.work_heavy[ph++] = i;
      else v.work[pl++] = i;
    }
  }
  if (tid == 0) {
    c->work_count = tl2[1];
    c->work_next = 0;
    c->heavy_count = tl2[0];
    c->heavy_next = c->heavy_next2 = 0;
    c->cur_step = step;
    c->step = step + 1;
    px_stamp(v, step, 2);
  }
}

// ---- the fused sharded step (k_px_step): one CTA per rank per wave ----------------
//
// Admission (when a search can be pending), the group table, its exchange and
// compute_targets in ONE kernel: jobs are processed in rounds of PXT (thread t
// holds job r*PXT + t of round r, state in registers), arrival segments come
// from a block-wide segmented scan, and the merged group tables live in shared
// memory.  Rank shards up to PXT * 8 searches; larger shards use
// k_px_groups + k_px_sched.
constexpr int PX_GCAP = 768;  // concatenated group entries staged in shared memory
struct PxTabs {
  int *a, *gm, *mfirst;
  unsigned long long *c0, *c1, *p0, *p1;  // counts (run | ungated << 32) of list 0/1; exclusive prefixes
  int2* mrun;
  double* rS[2];
  int *rA[2], *rC[2];
  long long *rWant[2], *rU[2], *rW[2];
  int *l0, *l1;                   // per concatenated entry: ungated of list 0/1 earlier in its merged entry
  long long *bp[2], *bb[2], *wn[2];  // per merged entry: its run's first sorted position, Σ(want-1) before, want
};
__host__ __device__ inline PxTabs px_tabs(unsigned char* base, long long cap, size_t* bytes) {
  PxTabs t;
  size_t o = 0;
  auto take = [&](size_t b) -> unsigned char* {
    unsigned char* q = base ? base + o : nullptr;
    o += (b + 15) & ~(size_t)15;
    return q;
  };
  t.a = (int*)take(4 * cap);
  t.gm = (int*)take(4 * cap);
  t.mfirst = (int*)take(4 * cap);
  t.c0 = (unsigned long long*)take(8 * cap);
  t.c1 = (unsigned long long*)take(8 * cap);
  t.p0 = (unsigned long long*)take(8 * cap);
  t.p1 = (unsigned long long*)take(8 * cap);
  t.mrun = (int2*)take(8 * cap);
  for (int b = 0; b < 2; ++b) {
    t.rS[b] = (double*)take(8 * cap);
    t.rA[b] = (int*)take(4 * cap);
    t.rC[b] = (int*)take(4 * cap);
    t.rWant[b] = (long long*)take(8 * cap);
    t.rU[b] = (long long*)take(8 * cap);
    t.rW[b] = (long long*)take(8 * cap);
  }
  t.l0 = (int*)take(4 * cap);
  t.l1 = (int*)take(4 * cap);
  for (int b = 0; b < 2; ++b) {
    t.bp[b] = (long long*)take(8 * cap);
    t.bb[b] = (long long*)take(8 * cap);
    t.wn[b] = (long long*)take(8 * cap);
  }
  if (bytes) *bytes = o;
  return t;
}
inline size_t px_step_smem() {
  size_t b = 0;
  px_tabs(nullptr, PX_GCAP, &b);
  return b;
}

// Block-wide exclusive segmented scan (PXS threads, thread order): F = a
// segment starts at this thread's element, X = its two packed counters.
// Returns the sum since the last segment start before this thread (and
// whether one occurred), and the block aggregate.
__device__ void seg_scan_block(bool F, unsigned long long X0, unsigned long long X1, bool& Fex,
                               unsigned long long& E0, unsigned long long& E1, bool& Ft, unsigned long long& T0,
                               unsigned long long& T1) {
  __shared__ unsigned long long sx0[32], sx1[32];
  __shared__ int sf[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  bool f = F;
  unsigned long long x0 = X0, x1 = X1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool fy = __shfl_up_sync(FULL, (int)f, o) != 0;
    const unsigned long long y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
    if (lane >= o) {
      if (!f) { x0 += y0; x1 += y1; }
      f = f || fy;
    }
  }
  __syncthreads();  // the previous call's readers are done with sx/sf
  if (lane == 31) {
    sx0[wid] = x0;
    sx1[wid] = x1;
    sf[wid] = f;
  }
  __syncthreads();
  // every warp scans the warp aggregates (lane j: warp j)
  bool wf = lane < (PXS / 32) && sf[lane] != 0;
  unsigned long long w0 = lane < (PXS / 32) ? sx0[lane] : 0ull, w1 = lane < (PXS / 32) ? sx1[lane] : 0ull;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool fy = __shfl_up_sync(FULL, (int)wf, o) != 0;
    const unsigned long long y0 = __shfl_up_sync(FULL, w0, o), y1 = __shfl_up_sync(FULL, w1, o);
    if (lane >= o) {
      if (!wf) { w0 += y0; w1 += y1; }
      wf = wf || fy;
    }
  }
  Ft = __shfl_sync(FULL, (int)wf, 31) != 0;
  T0 = __shfl_sync(FULL, w0, 31);
  T1 = __shfl_sync(FULL, w1, 31);
  // prefix of the warps before this one
  // (every shuffle is executed by the whole warp; the lane / warp conditions apply after)
  const int pfv = __shfl_sync(FULL, (int)wf, (wid + 31) & 31);
  unsigned long long p0 = __shfl_sync(FULL, w0, (wid + 31) & 31), p1 = __shfl_sync(FULL, w1, (wid + 31) & 31);
  const bool pf = wid > 0 && pfv != 0;
  if (wid == 0) { p0 = 0; p1 = 0; }
  // exclusive within the warp
  const int lfv = __shfl_up_sync(FULL, (int)f, 1);
  unsigned long long l0 = __shfl_up_sync(FULL, x0, 1), l1 = __shfl_up_sync(FULL, x1, 1);
  const bool lf = lane > 0 && lfv != 0;
  if (lane == 0) { l0 = 0; l1 = 0; }
  Fex = pf || lf;
  E0 = lf ? l0 : p0 + l0;
  E1 = lf ? l1 : p1 + l1;
}

template <int JPT>
__global__ void __launch_bounds__(PXS) k_px_step(View v, cudaGraphConditionalHandle cond, int max_steps) {
  Counters* c = v.ctr;
  if (c->px_done) return;
  const int tid = threadIdx.x;
  const int step = (int)c->step;
  const ts_config& cf = v.cfg;
  const int n = v.n_local, W = v.pworld, me = v.prank;
  const unsigned long long epoch = px_epoch(v, step);
  __shared__ int s_go;
  __shared__ long long s_alo, s_ahi;
  __shared__ int shi[5 * 32];
  __shared__ long long shl[5 * 32];
  if (tid == 0) px_stamp(v, step, 0);
#ifdef TS_PX_PROF
  unsigned long long pp_t = globaltimer();
  long long pp_c = clock64();
#define PX_MARK(slot)                                                   \
  do {                                                                  \
    __syncthreads();                                                    \
    if (tid == 0) {                                                     \
      const unsigned long long t_ = globaltimer();                      \
      atomicAdd(&v.ctr->prof[slot], t_ - pp_t);                         \
      pp_t = t_;                                                        \
    }                                                                   \
  } while (0)
#define PX_WMARK(slot)                                                  \
  do {                                                                  \
    __syncwarp();                                                       \
    if (tid == 0) {                                                     \
      const long long c_ = clock64();                                   \
      if (slot > 11) atomicAdd(&v.ctr->prof[slot], (unsigned long long)(c_ - pp_c)); \
      pp_c = c_;                                                        \
    }                                                                   \
  } while (0)
#else
#define PX_MARK(slot) do { } while (0)
#define PX_WMARK(slot) do { } while (0)
#endif
  if (step >= max_steps || step >= v.log1p_n) {
    if (tid == 0) px_finish(v, cond, 0);
    return;
  }
  // ---- admit_jobs (scheduler.py:131-140) over every rank's counts ----
  if (px_adm_active(v, step)) {
    if (tid == 0) {
      int lo = 0, hi = n;  // arrivals are non-decreasing: upper_bound(arrival, step)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v.arrival[mid] <= step) lo = mid + 1;
        else hi = mid;
      }
      const long long run = c->running, pend = (long long)lo - c->head, unf = (long long)n - c->finished;
      for (int p = 0; p < W; ++p) {
        long long* d = xh(v, p)->cnt[me];
        d[0] = run;
        d[1] = pend;
        d[2] = unf;
      }
      for (int p = 0; p < W; ++p) st_release_sys(&xh(v, p)->fa[me], epoch);
    }
    const XHdr* x = xh(v, me);
    if (!px_wait(v, x->fa, epoch)) {
      if (tid == 0) px_finish(v, cond, 1);
      return;
    }
    if (tid == 0) {
      long long run_g = 0, pend_g = 0, before = 0, unf_g = 0;
      for (int r = 0; r < W; ++r) {
        const long long c0 = __ldcg(&x->cnt[r][0]), c1 = __ldcg(&x->cnt[r][1]), c2 = __ldcg(&x->cnt[r][2]);
        run_g += c0;
        pend_g += c1;
        unf_g += c2;
        if (r < me) before += c1;
      }
      s_go = unf_g > 0;
      if (unf_g == 0) {
        px_finish(v, cond, 0);
      } else {
        long long A = (long long)cf.max_concurrency - run_g;
        if (A > pend_g) A = pend_g;
        if (A < 0) A = 0;
        long long q = A - before;
        const long long mine = __ldcg(&x->cnt[me][1]);
        if (q > mine) q = mine;
        if (q < 0) q = 0;
        s_alo = c->head;
        s_ahi = c->head + q;
        c->head += q;
        c->running += q;
      }
    }
    __syncthreads();
    if (!s_go) return;
  } else {
    if (tid == 0) s_alo = s_ahi = c->head;
    __syncthreads();
  }
  PX_MARK(0);
  const long long alo = s_alo, ahi = s_ahi;
  // ---- this rank's searches: thread t holds the contiguous jobs [t*JPT, t*JPT+JPT) ----
  const bool fold = cf.beta == 0.0;  // the boosted flag does not change the score: one list
  unsigned code[JPT];  // start | running << 1 | ungated << 2 | list << 3 | segment end << 4
  int comp[JPT], arr[JPT], qv[JPT], ent[JPT];
  const int lo = tid * JPT;
  {
    // the record each search's wave wrote for this step (write_next_record:
    // running, ungated, boosted, completed), contiguous 16-byte rows; the
    // SearchState row only for a stale record or a search admitted now
    ts_sched_record rr[JPT];
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int i = lo + u;
      if (i < n) {
        rr[u] = v.nrec[i];
        arr[u] = v.arrival[i];
      }
    }
    const int aprev = (lo > 0 && lo - 1 < n) ? v.arrival[lo - 1] : 0;
    const int anext = lo + JPT < n ? v.arrival[lo + JPT] : 0;
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int i = lo + u;
      code[u] = 0;
      comp[u] = 0;
      if (i >= n) continue;
      const bool adm = i >= alo && i < ahi;
      const uint32_t tag = rr[u].flags >> 8;
      bool run, ung, boosted;
      int done;
      if (!adm && (tag == (uint32_t)step || tag == NREC_FINAL)) {
        run = rr[u].flags & 1u;
        ung = (rr[u].flags & 2u) != 0;
        boosted = (rr[u].flags & 4u) != 0;
        done = (int)rr[u]._pad;
      } else {
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(v.st + i);  // state, completed, job_best
        int state = (int)(uint32_t)w.x;
        if (adm) {
          state = ST_RUNNING;
          v.st[i].state = ST_RUNNING;
          v.st[i].admit_step = step;
        }
        run = state == ST_RUNNING;
        done = (int)(uint32_t)(w.x >> 32);
        ung = done >= cf.obs_threshold;
        boosted = __longlong_as_double((long long)w.y) / cf.positive_exit_threshold > cf.proximity;  // scheduler.py:126
      }
      const int ap = u > 0 ? arr[u - 1] : (i > 0 ? aprev : arr[u]);
      const int an = u + 1 < JPT ? arr[u + 1] : anext;
      if (arr[u] < ap) c->sched_error = 1;
      unsigned cd = (i == 0 || arr[u] != ap) ? 1u : 0u;
      if (i == n - 1 || an != arr[u]) cd |= 16u;
      if (run) {
        cd |= 2u | (ung ? 4u : 0u) | ((boosted && !fold) ? 8u : 0u);
        comp[u] = done;
      }
      code[u] = cd;
    }
  }
  PX_MARK(1);
  // arrival segments: (running | ungated << 16) of list 0 and of list 1, one
  // block-wide segmented scan over the threads' aggregates
  auto xv = [](unsigned cd, int b) -> unsigned long long {
    if (!(cd & 2u) || (int)((cd >> 3) & 1u) != b) return 0ull;
    return 1ull | ((cd & 4u) ? (1ull << 16) : 0ull);
  };
  bool fex;
  unsigned long long e0, e1;
  {
    bool F = false, ft;
    unsigned long long X0 = 0, X1 = 0, t0, t1;
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      if (code[u] & 1u) { F = true; X0 = X1 = 0; }
      X0 += xv(code[u], 0);
      X1 += xv(code[u], 1);
    }
    seg_scan_block(F, X0, X1, fex, e0, e1, ft, t0, t1);
  }
  PX_MARK(2);
  // entries: segment ends with a running search, numbered in arrival order
  int fl1[1] = {0}, tot1[1];
  {
    unsigned long long y0 = e0, y1 = e1;
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const unsigned cd = code[u];
      if (cd & 1u) y0 = y1 = 0;
      y0 += xv(cd, 0);
      y1 += xv(cd, 1);
      if ((cd & 16u) && (((uint32_t)y0 & 0xFFFFu) + ((uint32_t)y1 & 0xFFFFu)) > 0) ++fl1[0];
    }
  }
  scan1_add<1>(fl1, tot1, shi);
  const int nent = tot1[0];
  {
    unsigned long long y0 = e0, y1 = e1;
    int id = fl1[0];
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const unsigned cd = code[u];
      if (cd & 1u) y0 = y1 = 0;
      qv[u] = (int)((((cd & 8u) ? y1 : y0) >> 16) & 0xFFFFu);  // ungated of its list before it in its segment
      ent[u] = id;
      y0 += xv(cd, 0);
      y1 += xv(cd, 1);
      if ((cd & 16u) && (((uint32_t)y0 & 0xFFFFu) + ((uint32_t)y1 & 0xFFFFu)) > 0) {
        PxEnt en;
        en.a = arr[u];
        en.nr0 = (int)(y0 & 0xFFFFu);
        en.nu0 = (int)((y0 >> 16) & 0xFFFFu);
        en.nr1 = (int)(y1 & 0xFFFFu);
        en.nu1 = (int)((y1 >> 16) & 0xFFFFu);
        en._p0 = en._p1 = en._p2 = 0;
        for (int p = 0; p < W; ++p) xent(v, p)[v.goff + id] = en;
        ++id;
      }
    }
  }
  PX_MARK(3);
  // every entry store above happens before the release below (bar.sync, then
  // a cumulative st.release.sys per peer)
  __syncthreads();
  if (tid < W) {
    XHdr* h = xh(v, tid);
    h->nent[me] = nent;
    h->goff[me] = v.goff;
    h->unf[me] = (long long)n - c->finished;
    st_release_sys(&h->fb[me], epoch);
  }
  const XHdr* x = xh(v, me);
  if (!px_wait(v, x->fb, epoch)) {
    if (tid == 0) px_finish(v, cond, 1);
    return;
  }
  PX_MARK(4);
  if (tid == 0) px_stamp(v, step, 1);
  // ---- compute_targets (scheduler.py:143-187) from the merged group tables (see k_px_sched) ----
  __shared__ int off[TS_MAX_PEERS + 1];
  __shared__ long long gof[TS_MAX_PEERS], s_unf, h_u[TS_MAX_PEERS], h_n[TS_MAX_PEERS];
  if (tid < W) {  // every rank's header words at once
    h_u[tid] = __ldcg(&x->unf[tid]);
    h_n[tid] = __ldcg(&x->nent[tid]);
    gof[tid] = __ldcg(&x->goff[tid]);
  }
  __syncthreads();
  if (tid == 0) {
    long long u = 0;
    off[0] = 0;
    for (int r = 0; r < W; ++r) {
      u += h_u[r];
      off[r + 1] = off[r] + (int)h_n[r];
    }
    s_unf = u;
  }
  __syncthreads();
  const long long unf_g = s_unf;
  if (unf_g == 0) {
    if (tid == 0) px_finish(v, cond, 0);
    return;
  }
  const int G = off[W];
  const PxEnt* tab = xent(v, me);
  // Outputs for the per-search pass: per concatenated entry its merged entry
  // and the ungated of each list in that merged entry before it (lower
  // ranks), per merged entry and list the sorted position and Σ(want-1) of
  // its run's first job, and want.
  __shared__ int w_gm[32], w_low0[32], w_low1[32];
  __shared__ long long w_bp0[32], w_bp1[32], w_bb0[32], w_bb1[32], w_wn0[32], w_wn1[32];
  __shared__ long long s_R, s_rrq, s_rrr;
  __shared__ int s_boost, s_err;
  extern __shared__ __align__(16) unsigned char psm[];
  const PxTabs Tb = px_tabs(G <= PX_GCAP ? psm : v.pscr, G <= PX_GCAP ? PX_GCAP : v.n_global, nullptr);
  const int *J_gm, *J_low0, *J_low1;
  const long long *J_bp0, *J_bp1, *J_bb0, *J_bb1, *J_wn0, *J_wn1;
  const long long M = cf.max_concurrency;
  if (G <= v.pgwarp) {
    // ---- one warp: every table entry in a lane ----
    J_gm = w_gm; J_low0 = w_low0; J_low1 = w_low1;
    J_bp0 = w_bp0; J_bp1 = w_bp1; J_bb0 = w_bb0; J_bb1 = w_bb1; J_wn0 = w_wn0; J_wn1 = w_wn1;
    PX_MARK(11);
    if (tid < 32) {
      const int lane = tid, g = lane;
      const bool has = g < G;
      int ea = 0, nr0 = 0, nu0 = 0, nr1 = 0, nu1 = 0;
      if (has) {
        int r = 0;
        while (r + 1 < W && off[r + 1] <= g) ++r;
        const int4* e4 = (const int4*)(tab + gof[r] + (g - off[r]));
        const int4 u4 = __ldcg(e4), w4 = __ldcg(e4 + 1);
        ea = u4.x; nr0 = u4.y; nu0 = u4.z; nr1 = u4.w; nu1 = w4.x;
      }
      PX_WMARK(12);
      const int aprev = __shfl_up_sync(FULL, ea, 1);
      const bool nw = has && (g == 0 || ea != aprev);
      const unsigned nwb = __ballot_sync(FULL, nw);
      const int Gm = __popc(nwb);
      const int m = __popc(nwb & ((2u << g) - 1u)) - 1;  // merged entry of lane g
      // segmented inclusive scans of the counts (reset where a merged entry starts)
      int i0 = nr0, i1 = nu0, i2 = nr1, i3 = nu1;
      bool f = nw;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y0 = __shfl_up_sync(FULL, i0, o), y1 = __shfl_up_sync(FULL, i1, o);
        const int y2 = __shfl_up_sync(FULL, i2, o), y3 = __shfl_up_sync(FULL, i3, o);
        const bool fy = __shfl_up_sync(FULL, (int)f, o) != 0;
        if (lane >= o && !f) { i0 += y0; i1 += y1; i2 += y2; i3 += y3; }
        if (lane >= o) f = f || fy;
      }
      if (has) {
        w_gm[g] = m;
        w_low0[g] = i1 - nu0;
        w_low1[g] = i3 - nu1;
      }
      PX_WMARK(13);
      // lane mm: merged entry mm (its first and last concatenated entries)
      const int mm = lane;
      const bool mh = mm < Gm;
      const int first = mh ? (int)__fns(nwb, 0, mm + 1) : 0;
      const int last = mh ? ((mm + 1 < Gm ? (int)__fns(nwb, 0, mm + 2) : G) - 1) : 0;
      const int ma = __shfl_sync(FULL, ea, first);
      const int Mr0 = __shfl_sync(FULL, i0, last), Mu0 = __shfl_sync(FULL, i1, last);
      const int Mr1 = __shfl_sync(FULL, i2, last), Mu1 = __shfl_sync(FULL, i3, last);
      double S0 = 0.0, S1 = 0.0;
      u128 fx = 0;
      bool bad = false;
      if (mh) {
        S0 = v.log1p_tab[step - ma] + 0.0;  // parallelism_score (scheduler.py:118-128)
        S1 = v.log1p_tab[step - ma] + cf.beta;
        u128 q;
        if (Mr0) { if (to_fixed(S0, q)) fx += q * (u128)(unsigned)Mr0; else bad = true; }
        if (Mr1) { if (to_fixed(S1, q)) fx += q * (u128)(unsigned)Mr1; else bad = true; }
      }
      PX_WMARK(14);
      long long run = mh ? (long long)Mr0 + Mr1 : 0, l0 = mh ? Mu0 : 0, l1 = mh ? Mu1 : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t h = __shfl_xor_sync(FULL, (uint64_t)(fx >> 64), o);
        const uint64_t l = __shfl_xor_sync(FULL, (uint64_t)fx, o);
        fx += ((u128)h << 64) | l;
        run += __shfl_xor_sync(FULL, run, o);
        l0 += __shfl_xor_sync(FULL, l0, o);
        l1 += __shfl_xor_sync(FULL, l1, o);
      }
      bad = __any_sync(FULL, bad);
      const double T = fixed_to_double(fx);
      const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
      const bool err = bad || (double)run * u2 >= 0x1p-10;  // would need the sequential sum (targets_block)
      const long long R = M - run;
      const bool boost_on = cf.boosting_enabled != 0 && run > 0 && R > 0 && l0 + l1 > 0;
      long long wn0 = 1, wn1 = 1;
      if (T > 0.0) {
        const double f0 = floor(S0 / T * (double)M), f1 = floor(S1 / T * (double)M);  // scheduler.py:173-175
        wn0 = f0 > 1.0 ? (long long)f0 : 1;
        wn1 = f1 > 1.0 ? (long long)f1 : 1;
      }
      const long long wv0 = mh ? (long long)Mu0 * (wn0 - 1) : 0, wv1 = mh ? (long long)Mu1 * (wn1 - 1) : 0;
      PX_WMARK(15);
      // sorted position / Σ(want-1) of each run's first job: own-list runs of
      // earlier arrival, other-list runs of higher score (equal: earlier arrival)
      long long bp0 = 0, bb0 = 0, bp1 = 0, bb1 = 0, twt = 0;
      for (int j = 0; j < Gm; ++j) {
        const double T0 = __shfl_sync(FULL, S0, j), T1 = __shfl_sync(FULL, S1, j);
        const int aj = __shfl_sync(FULL, ma, j);
        const long long u0 = __shfl_sync(FULL, (long long)Mu0, j), u1 = __shfl_sync(FULL, (long long)Mu1, j);
        const long long x0 = __shfl_sync(FULL, wv0, j), x1 = __shfl_sync(FULL, wv1, j);
        twt += x0 + x1;
        if (j < mm) { bp0 += u0; bb0 += x0; bp1 += u1; bb1 += x1; }
        if (u1 > 0 && (T1 > S0 || (T1 == S0 && aj < ma))) { bp0 += u1; bb0 += x1; }
        if (u0 > 0 && (T0 > S1 || (T0 == S1 && aj < ma))) { bp1 += u0; bb1 += x0; }
      }
      PX_WMARK(16);
      if (mh) {
        w_bp0[mm] = bp0; w_bb0[mm] = bb0; w_wn0[mm] = wn0;
        w_bp1[mm] = bp1; w_bb1[mm] = bb1; w_wn1[mm] = wn1;
      }
      if (lane == 0) {
        const long long U = l0 + l1;
        long long Rp = R - twt;
        if (Rp < 0) Rp = 0;
        s_R = R;
        s_boost = boost_on;
        s_rrq = U > 0 ? Rp / U : 0;
        s_rrr = U > 0 ? Rp % U : 0;
        s_err = err;
      }
    }
    __syncthreads();
  } else {
    // ---- many entries: block-wide scans over the staged tables ----
    J_gm = Tb.gm; J_low0 = Tb.l0; J_low1 = Tb.l1;
    J_bp0 = Tb.bp[0]; J_bp1 = Tb.bp[1]; J_bb0 = Tb.bb[0]; J_bb1 = Tb.bb[1];
    J_wn0 = Tb.wn[0]; J_wn1 = Tb.wn[1];
    for (int g = tid; g < G; g += PXS) {
      int r = 0;
      while (r + 1 < W && off[r + 1] <= g) ++r;
      const int4* e4 = (const int4*)(tab + gof[r] + (g - off[r]));
      const int4 u = __ldcg(e4), w2 = __ldcg(e4 + 1);
      Tb.a[g] = u.x;
      Tb.c0[g] = (unsigned long long)(uint32_t)u.y | ((unsigned long long)(uint32_t)u.z << 32);
      Tb.c1[g] = (unsigned long long)(uint32_t)u.w | ((unsigned long long)(uint32_t)w2.x << 32);
    }
    __syncthreads();
    PX_MARK(5);
    // merged entries and exclusive prefixes of the counts over the concatenated table
    const int pg = (G + PXS - 1) / PXS, g0 = min(G, tid * pg), g1 = min(G, g0 + pg);
    long long cg[5] = {0, 0, 0, 0, 0}, tg[5];  // new, run0, ung0, run1, ung1 — 64-bit sums of the 32-bit halves
    {
      long long acc[3] = {0, 0, 0};
      for (int g = g0; g < g1; ++g) {
        acc[0] += (g == 0 || Tb.a[g] != Tb.a[g - 1]) ? 1 : 0;
        cg[1] += (uint32_t)Tb.c0[g];
        cg[2] += (long long)(Tb.c0[g] >> 32);
        cg[3] += (uint32_t)Tb.c1[g];
        cg[4] += (long long)(Tb.c1[g] >> 32);
      }
      cg[0] = acc[0];
    }
    scan1_add<5>(cg, tg, shl);
    for (int g = g0; g < g1; ++g) {
      if (g == 0 || Tb.a[g] != Tb.a[g - 1]) Tb.mfirst[cg[0]++] = g;
      Tb.gm[g] = (int)cg[0] - 1;
      Tb.p0[g] = (unsigned long long)cg[1] | ((unsigned long long)cg[2] << 32);
      Tb.p1[g] = (unsigned long long)cg[3] | ((unsigned long long)cg[4] << 32);
      cg[1] += (uint32_t)Tb.c0[g];
      cg[2] += (long long)(Tb.c0[g] >> 32);
      cg[3] += (uint32_t)Tb.c1[g];
      cg[4] += (long long)(Tb.c1[g] >> 32);
    }
    PX_MARK(6);
    const int Gm = (int)tg[0];
    const long long tot_run = tg[1] + tg[3], len0 = tg[2], len1 = tg[4];
    const unsigned long long pt0 = (unsigned long long)tg[1] | ((unsigned long long)tg[2] << 32);
    const unsigned long long pt1 = (unsigned long long)tg[3] | ((unsigned long long)tg[4] << 32);
    __syncthreads();
    const int pm = (Gm + PXS - 1) / PXS, m0 = min(Gm, tid * pm), m1 = min(Gm, m0 + pm);
    auto mcount = [&](int m, int& a, unsigned long long& k0, unsigned long long& k1) {
      const int ga = Tb.mfirst[m], gb = m + 1 < Gm ? Tb.mfirst[m + 1] : G;
      k0 = (gb < G ? Tb.p0[gb] : pt0) - Tb.p0[ga];
      k1 = (gb < G ? Tb.p1[gb] : pt1) - Tb.p1[ga];
      a = Tb.a[ga];
    };
    u128 fx = 0;
    bool bad = false;
    int cr[2] = {0, 0}, tr[2];
    for (int m = m0; m < m1; ++m) {
      int a;
      unsigned long long k0, k1;
      mcount(m, a, k0, k1);
      const double S0 = v.log1p_tab[step - a] + 0.0, S1 = v.log1p_tab[step - a] + cf.beta;
      u128 q;
      if ((uint32_t)k0) {
        if (to_fixed(S0, q)) fx += q * (u128)(uint32_t)k0;
        else bad = true;
      }
      if ((uint32_t)k1) {
        if (to_fixed(S1, q)) fx += q * (u128)(uint32_t)k1;
        else bad = true;
      }
      cr[0] += (k0 >> 32) ? 1 : 0;
      cr[1] += (k1 >> 32) ? 1 : 0;
    }
    scan1_add<2>(cr, tr, shi);
    const u128 fsum = block_sum_u128(fx, bad);
    for (int m = m0; m < m1; ++m) {
      int a;
      unsigned long long k0, k1;
      mcount(m, a, k0, k1);
      const double S0 = v.log1p_tab[step - a] + 0.0, S1 = v.log1p_tab[step - a] + cf.beta;
      int2 mr = make_int2(-1, -1);
      if (k0 >> 32) {
        Tb.rS[0][cr[0]] = S0;
        Tb.rA[0][cr[0]] = a;
        Tb.rC[0][cr[0]] = (int)(k0 >> 32);
        mr.x = cr[0]++;
      }
      if (k1 >> 32) {
        Tb.rS[1][cr[1]] = S1;
        Tb.rA[1][cr[1]] = a;
        Tb.rC[1][cr[1]] = (int)(k1 >> 32);
        mr.y = cr[1]++;
      }
      Tb.mrun[m] = mr;
    }
    const int nrun0 = tr[0], nrun1 = tr[1];
    const double T = fixed_to_double(fsum);
    {
      const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
      if (bad || (double)tot_run * u2 >= 0x1p-10) {  // would need the sequential sum (targets_block)
        if (tid == 0) px_finish(v, cond, 2);
        return;  // block-uniform
      }
    }
    __syncthreads();
    PX_MARK(7);
    const long long R = M - tot_run;
    const bool boost_on = cf.boosting_enabled != 0 && tot_run > 0 && R > 0 && len0 + len1 > 0;
    long long tw0 = 0, tw1 = 0;
    if (boost_on) {
      long long pre[4] = {0, 0, 0, 0}, tot4[4];
      int a0[2], a1[2];
  #pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int nr = b ? nrun1 : nrun0;
        const int pr = (nr + PXS - 1) / PXS;
        a0[b] = min(nr, tid * pr);
        a1[b] = min(nr, a0[b] + pr);
        for (int k = a0[b]; k < a1[b]; ++k) {
          long long want = 1;
          if (T > 0.0) {
            const double f = floor(Tb.rS[b][k] / T * (double)M);  // scheduler.py:173-175
            want = f > 1.0 ? (long long)f : 1;
          }
          Tb.rWant[b][k] = want;
          pre[2 * b] += Tb.rC[b][k];
          pre[2 * b + 1] += (long long)Tb.rC[b][k] * (want - 1);
        }
      }
      __syncthreads();
      scan1_add<4>(pre, tot4, shl);
  #pragma unroll
      for (int b = 0; b < 2; ++b) {
        long long u = pre[2 * b], w = pre[2 * b + 1];
        for (int k = a0[b]; k < a1[b]; ++k) {
          Tb.rU[b][k] = u;
          Tb.rW[b][k] = w;
          u += Tb.rC[b][k];
          w += (long long)Tb.rC[b][k] * (Tb.rWant[b][k] - 1);
        }
      }
      tw0 = tot4[1];
      tw1 = tot4[3];
      __syncthreads();
    }
    PX_MARK(8);
    // per merged entry and list: the run's first job's sorted position and Σ(want-1)
    for (int m = m0; m < m1; ++m) {
      const int2 mr = Tb.mrun[m];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int kr = b ? mr.y : mr.x;
        long long bp = 0, bb = 0, wn = 1;
        if (kr >= 0 && boost_on) {
          const double* oS = b ? Tb.rS[0] : Tb.rS[1];
          const int* oA = b ? Tb.rA[0] : Tb.rA[1];
          const long long* oU = b ? Tb.rU[0] : Tb.rU[1];
          const long long* oW = b ? Tb.rW[0] : Tb.rW[1];
          const int on = b ? nrun0 : nrun1;
          const double S = (b ? Tb.rS[1] : Tb.rS[0])[kr];
          const int a = (b ? Tb.rA[1] : Tb.rA[0])[kr];
          wn = (b ? Tb.rWant[1] : Tb.rWant[0])[kr];
          bp = (b ? Tb.rU[1] : Tb.rU[0])[kr];
          bb = (b ? Tb.rW[1] : Tb.rW[0])[kr];
          int kk = runs_lower(oS, on, S);  // other-list runs with a higher score
          if (kk < on && oS[kk] == S && oA[kk] < a) ++kk;  // equal score: earlier arrival first
          bp += kk < on ? oU[kk] : (b ? len0 : len1);
          bb += kk < on ? oW[kk] : (b ? tw0 : tw1);
        }
        (b ? Tb.bp[1] : Tb.bp[0])[m] = bp;
        (b ? Tb.bb[1] : Tb.bb[0])[m] = bb;
        (b ? Tb.wn[1] : Tb.wn[0])[m] = wn;
      }
    }
    for (int g = g0; g < g1; ++g) {
      const int m = Tb.gm[g], f = Tb.mfirst[m];
      Tb.l0[g] = (int)((Tb.p0[g] >> 32) - (Tb.p0[f] >> 32));
      Tb.l1[g] = (int)((Tb.p1[g] >> 32) - (Tb.p1[f] >> 32));
    }
    if (tid == 0) {
      const long long U = len0 + len1;
      long long Rp = R - (tw0 + tw1);
      if (Rp < 0) Rp = 0;
      s_R = R;
      s_boost = boost_on;
      s_rrq = U > 0 ? Rp / U : 0;
      s_rrr = U > 0 ? Rp % U : 0;
      s_err = 0;
    }
    __syncthreads();
  }
  if (s_err) {
    if (tid == 0) px_finish(v, cond, 2);
    return;
  }
  PX_MARK(8);
  const long long R = s_R, rr_q = s_rrq, rr_r = s_rrr;
  const bool boost_on = s_boost != 0;
  int nl2[2] = {0, 0}, tl2[2];
  unsigned hv = 0;  // bit u: job lo+u is in the pipelined-mode list
#pragma unroll
  for (int u = 0; u < JPT; ++u) {
    const int i = lo + u;
    const unsigned cd = code[u];
    if (i >= n) continue;
    if (!(cd & 2u)) {
      v.tgt[i] = 0;
      continue;
    }
    long long tgt = 1;
    if ((cd & 4u) && boost_on) {
      const bool b = (cd & 8u) != 0;
      const int g = off[me] + ent[u], m = J_gm[g];
      const long long qt = (long long)qv[u] + (b ? J_low1 : J_low0)[g];
      const long long want = (b ? J_wn1 : J_wn0)[m];
      const long long pos = (b ? J_bp1 : J_bp0)[m] + qt;
      const long long before = (b ? J_bb1 : J_bb0)[m] + qt * (want - 1);
      long long extra = R - before;
      if (extra < 0) extra = 0;
      if (extra > want - 1) extra = want - 1;
      tgt = 1 + extra + rr_q + (pos < rr_r ? 1 : 0);
    }
    v.tgt[i] = (int)tgt;
    const bool h = v.heavy_on && min(tgt, (long long)(cf.rollout_budget - comp[u])) >= HEAVY_P;
    if (h) hv |= 1u << u;
    ++nl2[h ? 0 : 1];
  }
  PX_MARK(9);
  // the two work lists in run-queue order (one scan: the chunks are contiguous)
  scan1_add<2>(nl2, tl2, shi);
  {
    int ph = nl2[0], pl = nl2[1];
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      const int i = lo + u;
      if (i >= n || !(code[u] & 2u)) continue;
      if ((hv >> u) & 1u) v.work_heavy[ph++] = i;
      else v.work[pl++] = i;
    }
  }
  PX_MARK(10);
  if (tid == 0) {
    c->work_count = tl2[1];
    c->work_next = 0;
    c->heavy_count = tl2[0];
    c->heavy_next = c->heavy_next2 = 0;
    c->cur_step = step;
    c->step = step + 1;
    px_stamp(v, step, 2);
  }
}
#undef PX_MARK
#undef PX_WMARK

// ---- compute_targets over many CTAs (multi-GPU runs: all n_global records) ----
// The same algorithm as targets_block, with every cross-thread scan split into
// an in-CTA scan plus a scan over CTA totals in a one-CTA kernel between
// phases.  Thread t owns records [t*MT_CH, (t+1)*MT_CH); its running state
// between phases (list positions, run ids, the previous score of each list)
// lives in a global scratch row.
constexpr int MT_T = 256, MT_CH = 8, MT_REC = MT_T * MT_CH;
constexpr int MT_RUNCAP = 128;  // runs per list k_mt_all stages in shared memory (else read from global)
constexpr int MT_RB = 256;      // run blocks per list whose offsets k_mt_all keeps in shared memory
struct MtBlk1 {
  long long nrun, cnt0, cnt1;
  unsigned long long flo, fhi;
  int bad, _p;
  double min0, min1;
};
struct MtOff1 {
  long long p0, p1;
  double prev0, prev1;
};
struct MtThr {
  long long pos0, pos1, rid0, rid1;
  double prev0, prev1;
};
struct MtState {
  double T;
  long long tot_run, len0, len1, nr0, nr1, tw0, tw1;
  int boost_on, _p;
};
struct MtLayout {
  MtBlk1* b1;
  MtOff1* o1;
  MtThr* thr;
  long long* b2;  // run counts per CTA, list 0 then list 1
  long long* b3;  // Σ cnt*(want-1) per run-CTA, list 0 then list 1
  long long* b3p; // exclusive prefixes of b3 (k_mt_all with more run blocks than MT_RB)
  MtState* st;
  uint8_t* hflag; // pipelined-mode flag per local search
};
__host__ __device__ inline size_t mt_align(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ inline int mt_blocks(int n) { return (n + MT_REC - 1) / MT_REC; }
__host__ __device__ inline int mt_run_blocks(int n) { return (n + MT_T - 1) / MT_T; }
__host__ __device__ inline size_t mt_layout(unsigned char* base, int n, int n_local, MtLayout* L) {
  const int G = mt_blocks(n), G3 = mt_run_blocks(n);
  size_t o = 0;
  if (L) L->b1 = (MtBlk1*)(base + o);
  o = mt_align(o + sizeof(MtBlk1) * G);
  if (L) L->o1 = (MtOff1*)(base + o);
  o = mt_align(o + sizeof(MtOff1) * G);
  if (L) L->thr = (MtThr*)(base + o);
  o = mt_align(o + sizeof(MtThr) * (size_t)G * MT_T);
  if (L) L->b2 = (long long*)(base + o);
  o = mt_align(o + sizeof(long long) * 2 * G);
  if (L) L->b3 = (long long*)(base + o);
  o = mt_align(o + sizeof(long long) * 2 * G3);
  if (L) L->b3p = (long long*)(base + o);
  o = mt_align(o + sizeof(long long) * 2 * G3);
  if (L) L->st = (MtState*)(base + o);
  o = mt_align(o + sizeof(MtState));
  if (L) L->hflag = (uint8_t*)(base + o);
  o = mt_align(o + (size_t)n_local);
  return o;
}

// Exclusive (+) scans of K values per thread over an MT_T-thread CTA; totals out.
template <int K>
__device__ void mt_scan(long long (&x)[K], long long (&tot)[K]) {
  __shared__ long long sw[K][MT_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    incl[q] = x[q];
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, incl[q], o);
      if (lane >= o) incl[q] += y;
    }
    if (lane == 31) sw[q][wid] = incl[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < K; ++q) {
    long long base = 0, t = 0;
    for (int w = 0; w < MT_T / 32; ++w) {
      if (w < wid) base += sw[q][w];
      t += sw[q][w];
    }
    tot[q] = t;
    x[q] = base + incl[q] - x[q];
  }
  __syncthreads();
}
// Exclusive min-scan of two doubles per thread over the CTA (identity +inf); CTA mins out.
__device__ void mt_scan_min2(double& a, double& b, double& ta, double& tb) {
  __shared__ double sw[2][MT_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double ia = a, ib = b;
  for (int o = 1; o < 32; o <<= 1) {
    const double ya = __shfl_up_sync(FULL, ia, o), yb = __shfl_up_sync(FULL, ib, o);
    if (lane >= o) {
      ia = fmin(ia, ya);
      ib = fmin(ib, yb);
    }
  }
  double ea = __shfl_up_sync(FULL, ia, 1), eb = __shfl_up_sync(FULL, ib, 1);
  if (lane == 0) ea = eb = INFINITY;
  if (lane == 31) {
    sw[0][wid] = ia;
    sw[1][wid] = ib;
  }
  __syncthreads();
  double pa = INFINITY, pb = INFINITY;
  ta = tb = INFINITY;
  for (int w = 0; w < MT_T / 32; ++w) {
    if (w < wid) {
      pa = fmin(pa, sw[0][w]);
      pb = fmin(pb, sw[1][w]);
    }
    ta = fmin(ta, sw[0][w]);
    tb = fmin(tb, sw[1][w]);
  }
  a = fmin(pa, ea);
  b = fmin(pb, eb);
  __syncthreads();
}

// phase 1: per-CTA counts, exact partial score sums, list minima
__global__ void __launch_bounds__(MT_T) k_mt_count(View v, int step, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  if (step < 0) step = v.ctr->cur_step;
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global;
  if (blockIdx.x == 0 && threadIdx.x == 0 && step < v.step_times_cap) v.step_times[step] = globaltimer();
  const int t = blockIdx.x * MT_T + threadIdx.x;
  const int lo = min(n, t * MT_CH), hi = min(n, lo + MT_CH);
  long long c[3] = {0, 0, 0}, tot[3];
  u128 fx = 0;
  bool bad = false;
  double m0 = INFINITY, m1 = INFINITY;
  for (int i = lo; i < hi; ++i) {
    const ts_sched_record r = rec[i];
    if (!(r.flags & 1u)) continue;
    ++c[0];
    u128 q;
    if (to_fixed(r.score, q)) fx += q;
    else bad = true;
    if (r.flags & 2u) {
      if (r.flags & 4u) { ++c[2]; m1 = fmin(m1, r.score); }
      else { ++c[1]; m0 = fmin(m0, r.score); }
    }
  }
  mt_scan<3>(c, tot);
  double tm0, tm1;
  mt_scan_min2(m0, m1, tm0, tm1);
  __shared__ u128 sq[MT_T / 32];
  __shared__ int sbad;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) sbad = 0;
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t h = __shfl_down_sync(FULL, (uint64_t)(fx >> 64), o);
    const uint64_t l = __shfl_down_sync(FULL, (uint64_t)fx, o);
    fx += ((u128)h << 64) | l;
  }
  if (lane == 0) sq[wid] = fx;
  __syncthreads();
  if (bad) sbad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    u128 s = 0;
    for (int w = 0; w < MT_T / 32; ++w) s += sq[w];
    MtBlk1 b;
    b.nrun = tot[0];
    b.cnt0 = tot[1];
    b.cnt1 = tot[2];
    b.flo = (unsigned long long)s;
    b.fhi = (unsigned long long)(s >> 64);
    b.bad = sbad;
    b._p = 0;
    b.min0 = tm0;
    b.min1 = tm1;
    L.b1[blockIdx.x] = b;
  }
}

// phase 2 (one CTA): CTA offsets, the score sum T, the totals
__global__ void __launch_bounds__(1024) k_mt_scan1(View v, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global, G = mt_blocks(n);
  __shared__ long long shl[264];
  __shared__ double shd[80];
  __shared__ u128 sq[32];
  __shared__ int sbad;
  const int b = threadIdx.x, lane = b & 31, wid = b >> 5;
  if (b == 0) sbad = 0;
  __syncthreads();
  MtBlk1 x{};
  x.min0 = x.min1 = INFINITY;
  if (b < G) x = L.b1[b];
  long long c4[4] = {x.nrun, x.cnt0, x.cnt1, 0}, t4[4];
  block_scan_add4(c4, t4, shl);
  const double p0 = block_scan_min(x.min0, shd);
  const double p1 = block_scan_min(x.min1, shd);
  u128 fx = b < G ? (((u128)x.fhi << 64) | x.flo) : 0;
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t h = __shfl_down_sync(FULL, (uint64_t)(fx >> 64), o);
    const uint64_t l = __shfl_down_sync(FULL, (uint64_t)fx, o);
    fx += ((u128)h << 64) | l;
  }
  if (lane == 0) sq[wid] = fx;
  if (b < G && x.bad) sbad = 1;
  __syncthreads();
  if (b < G) {
    MtOff1 o;
    o.p0 = c4[1];
    o.p1 = c4[2];
    o.prev0 = p0;
    o.prev1 = p1;
    L.o1[b] = o;
  }
  if (b == 0) {
    u128 s = 0;
    for (int w = 0; w < 32; ++w) s += sq[w];
    const long long tot_run = t4[0];
    bool fallback = sbad != 0;
    double T = 0.0;
    if (!fallback) {
      T = fixed_to_double(s);
      const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
      if ((double)tot_run * u2 >= 0x1p-10) fallback = true;
    }
    if (fallback) {  // sequential Neumaier sum in run-queue order
      double f = 0.0, cc = 0.0;
      bool first = true;
      for (int i = 0; i < n; ++i) {
        const ts_sched_record r = rec[i];
        if (!(r.flags & 1u)) continue;
        const double x2 = r.score;
        if (first) { f = x2; first = false; continue; }
        const double y = f + x2;
        if (fabs(f) >= fabs(x2)) cc += (f - y) + x2;
        else cc += (x2 - y) + f;
        f = y;
      }
      if (cc != 0.0 && isfinite(cc)) f += cc;
      T = f;
      atomicAdd(&v.ctr->sum_fallbacks, 1);
    }
    MtState st{};
    st.T = T;
    st.tot_run = tot_run;
    st.len0 = t4[1];
    st.len1 = t4[2];
    const long long R = (long long)v.cfg.max_concurrency - tot_run;
    st.boost_on = (v.cfg.boosting_enabled != 0 && tot_run > 0 && R > 0 && t4[1] + t4[2] > 0) ? 1 : 0;
    *L.st = st;
  }
}

// phase 3: per-thread list positions and previous scores; runs of equal score
__global__ void __launch_bounds__(MT_T) k_mt_runs(View v, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global;
  const int t = blockIdx.x * MT_T + threadIdx.x;
  const int lo = min(n, t * MT_CH), hi = min(n, lo + MT_CH);
  const bool boost_on = L.st->boost_on != 0;
  long long c[2] = {0, 0}, tot[2];
  double m0 = INFINITY, m1 = INFINITY;
  for (int i = lo; i < hi; ++i) {
    const ts_sched_record r = rec[i];
    if ((r.flags & 3u) != 3u) continue;
    if (r.flags & 4u) { ++c[1]; m1 = fmin(m1, r.score); }
    else { ++c[0]; m0 = fmin(m0, r.score); }
  }
  mt_scan<2>(c, tot);
  double tm0, tm1;
  mt_scan_min2(m0, m1, tm0, tm1);
  const MtOff1 o = L.o1[blockIdx.x];
  MtThr th;
  th.pos0 = o.p0 + c[0];
  th.pos1 = o.p1 + c[1];
  th.prev0 = fmin(o.prev0, m0);
  th.prev1 = fmin(o.prev1, m1);
  long long rs[2] = {0, 0};
  if (boost_on) {
    double p0 = th.prev0, p1 = th.prev1;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = rec[i];
      if ((r.flags & 3u) != 3u) continue;
      if (r.flags & 4u) { if (r.score != p1) ++rs[1]; if (r.score > p1) v.ctr->sched_error = 1; p1 = r.score; }
      else { if (r.score != p0) ++rs[0]; if (r.score > p0) v.ctr->sched_error = 1; p0 = r.score; }
    }
  }
  long long rt[2];
  mt_scan<2>(rs, rt);
  th.rid0 = rs[0];
  th.rid1 = rs[1];
  L.thr[t] = th;
  if (threadIdx.x == 0) {
    L.b2[blockIdx.x] = rt[0];
    L.b2[gridDim.x + blockIdx.x] = rt[1];
  }
}

// phase 4 (one CTA): run offsets of the CTAs; run totals
__global__ void __launch_bounds__(1024) k_mt_scan2(View v, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int G = mt_blocks(v.n_global);
  __shared__ long long shl[264];
  const int b = threadIdx.x;
  long long c4[4] = {b < G ? L.b2[b] : 0, b < G ? L.b2[G + b] : 0, 0, 0}, t4[4];
  block_scan_add4(c4, t4, shl);
  if (b < G) {
    L.b2[b] = c4[0];
    L.b2[G + b] = c4[1];
  }
  if (b == 0) {
    L.st->nr0 = t4[0];
    L.st->nr1 = t4[1];
  }
}

// phase 5: run records (score, start position) of the runs starting in each chunk
__global__ void __launch_bounds__(MT_T) k_mt_write_runs(View v, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global, G = gridDim.x;
  const int t = blockIdx.x * MT_T + threadIdx.x;
  MtThr th = L.thr[t];
  th.rid0 += L.b2[blockIdx.x];
  th.rid1 += L.b2[G + blockIdx.x];
  L.thr[t] = th;
  if (!L.st->boost_on) return;
  const int lo = min(n, t * MT_CH), hi = min(n, lo + MT_CH);
  const int stride = n;
  double p0 = th.prev0, p1 = th.prev1;
  long long q0 = th.pos0, q1 = th.pos1, k0 = th.rid0, k1 = th.rid1;
  for (int i = lo; i < hi; ++i) {
    const ts_sched_record r = rec[i];
    if ((r.flags & 3u) != 3u) continue;
    if (r.flags & 4u) {
      if (r.score != p1) { v.g_runS[stride + k1] = r.score; v.g_runStart[stride + k1] = (int)q1; ++k1; }
      p1 = r.score;
      ++q1;
    } else {
      if (r.score != p0) { v.g_runS[k0] = r.score; v.g_runStart[k0] = (int)q0; ++k0; }
      p0 = r.score;
      ++q0;
    }
  }
}

__device__ __forceinline__ long long mt_want(double s, double T, long long M) {
  long long want = 1;
  if (T > 0.0) {
    const double f = floor(s / T * (double)M);
    want = f > 1.0 ? (long long)f : 1;
  }
  return want;
}

// phase 6: want per run and the per-CTA sums of cnt*(want-1) (one run per thread, both lists)
__global__ void __launch_bounds__(MT_T) k_mt_want(View v, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global, G3 = gridDim.x;
  const MtState st = *L.st;
  const long long M = v.cfg.max_concurrency;
  const int k = blockIdx.x * MT_T + threadIdx.x;
  long long w[2] = {0, 0}, tot[2];
  if (st.boost_on) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const long long nr = b ? st.nr1 : st.nr0, len = b ? st.len1 : st.len0;
      const int off = b ? n : 0;
      if (k < nr) {
        const long long want = mt_want(v.g_runS[off + k], st.T, M);
        const long long cnt = (k + 1 < nr ? v.g_runStart[off + k + 1] : len) - v.g_runStart[off + k];
        v.g_runWant[off + k] = want;
        w[b] = cnt * (want - 1);
      }
    }
  }
  mt_scan<2>(w, tot);
  if (st.boost_on) {
    if (k < st.nr0) v.g_runPW[k] = w[0];
    if (k < st.nr1) v.g_runPW[n + k] = w[1];
  }
  if (threadIdx.x == 0) {
    L.b3[blockIdx.x] = tot[0];
    L.b3[G3 + blockIdx.x] = tot[1];
  }
}

// phase 7 (one CTA): scan of the run-CTA sums; tw0, tw1
__global__ void __launch_bounds__(1024) k_mt_scan3(View v, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int G3 = mt_run_blocks(v.n_global);
  __shared__ long long shl[264];
  __shared__ long long carry[2];
  if (threadIdx.x == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  for (int base = 0; base < G3; base += 1024) {
    const int b = base + threadIdx.x;
    long long c4[4] = {b < G3 ? L.b3[b] : 0, b < G3 ? L.b3[G3 + b] : 0, 0, 0}, t4[4];
    block_scan_add4(c4, t4, shl);
    if (b < G3) {
      L.b3[b] = carry[0] + c4[0];
      L.b3[G3 + b] = carry[1] + c4[1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] += t4[0];
      carry[1] += t4[1];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    L.st->tw0 = carry[0];
    L.st->tw1 = carry[1];
  }
}

// phase 8: targets of the local slice (closed-form clamp + round-robin, merge
// rank by binary search in the other list's runs); pipelined-mode flags
__global__ void __launch_bounds__(MT_T) k_mt_targets(View v, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  const int n = v.n_global, G3 = mt_run_blocks(n);
  const int t = blockIdx.x * MT_T + threadIdx.x;
  const int lo = min(n, t * MT_CH), hi = min(n, lo + MT_CH);
  const int glo = v.goff, ghi = v.goff + v.n_local;
  if (hi <= glo || lo >= ghi) return;  // no local search in this chunk: nothing to write
  const MtState st = *L.st;
  const MtThr th = L.thr[t];
  const ts_config& cf = v.cfg;
  const long long M = cf.max_concurrency, R = M - st.tot_run;
  const long long U = st.len0 + st.len1;
  long long Rp = R - (st.tw0 + st.tw1);
  if (Rp < 0) Rp = 0;
  const int stride = n;
  const double* runS = v.g_runS;
  const int32_t* runStart = v.g_runStart;
  const long long* runWant = v.g_runWant;
  const long long* runPWl = v.g_runPW;
  auto runPW = [&](int off, long long k) { return runPWl[off + k] + L.b3[(off ? G3 : 0) + k / MT_T]; };
  long long q0 = th.pos0, q1 = th.pos1, k0 = th.rid0 - 1, k1 = th.rid1 - 1;
  double p0 = th.prev0, p1 = th.prev1;
  for (int i = lo; i < hi; ++i) {
    const ts_sched_record r = rec[i];
    const bool local = i >= glo && i < ghi;
    if (!(r.flags & 1u)) {
      if (local) {
        v.tgt[i - glo] = 0;
        L.hflag[i - glo] = 0;
      }
      continue;
    }
    long long tgt = 1;
    if ((r.flags & 2u) && st.boost_on) {
      const int b = (r.flags & 4u) ? 1 : 0;
      long long pos, k;
      if (b) { if (r.score != p1) ++k1; p1 = r.score; pos = q1++; k = k1; }
      else { if (r.score != p0) ++k0; p0 = r.score; pos = q0++; k = k0; }
      if (local) {
        const int off = b ? stride : 0, oo = b ? 0 : stride;
        const long long want = runWant[off + k];
        long long before = runPW(off, k) + (pos - runStart[off + k]) * (want - 1);
        const long long nro = b ? st.nr0 : st.nr1, leno = b ? st.len0 : st.len1, two = b ? st.tw0 : st.tw1;
        const long long obefore = b ? q0 : q1;
        int lo2 = 0, hi2 = (int)nro;  // first run of the other list with runS <= S
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (runS[oo + mid] > r.score) lo2 = mid + 1;
          else hi2 = mid;
        }
        const int kk = lo2;
        long long c, cw;
        if (kk < nro && runS[oo + kk] == r.score) {
          const long long st0 = runStart[oo + kk];
          const long long cntk = (kk + 1 < nro ? runStart[oo + kk + 1] : leno) - st0;
          long long part = obefore - st0;
          if (part < 0) part = 0;
          if (part > cntk) part = cntk;
          c = st0 + part;
          cw = runPW(oo, kk) + part * (runWant[oo + kk] - 1);
        } else if (kk < nro) {
          c = runStart[oo + kk];
          cw = runPW(oo, kk);
        } else {
          c = leno;
          cw = two;
        }
        const long long spos = pos + c;
        before += cw;
        long long extra = R - before;
        if (extra < 0) extra = 0;
        if (extra > want - 1) extra = want - 1;
        long long rr = 0;
        if (U > 0) rr = Rp / U + (spos < Rp % U ? 1 : 0);
        tgt = 1 + extra + rr;
      }
    }
    if (local) {
      v.tgt[i - glo] = (int)tgt;
      L.hflag[i - glo] = (v.heavy_on && min(tgt, (long long)(cf.rollout_budget - (int)r._pad)) >= HEAVY_P) ? 1 : 0;
    }
  }
}

// phase 9 (one CTA over the local slice): single-warp and pipelined work lists
__global__ void __launch_bounds__(TT) k_mt_split(View v, int step, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  if (step < 0) step = v.ctr->cur_step;
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  __shared__ long long shl[264];
  const int tid = threadIdx.x, nl = v.n_local, glo = v.goff;
  const int per = (nl + TT - 1) / TT;
  const int lo = min(nl, tid * per), hi = min(nl, lo + per);
  long long nh = 0, nlt = 0;
  for (int i = lo; i < hi; ++i) {
    if (!(rec[i + glo].flags & 1u)) continue;
    if (L.hflag[i]) ++nh;
    else ++nlt;
  }
  long long sc2[4] = {nh, nlt, 0, 0}, tt2[4];
  block_scan_add4(sc2, tt2, shl);
  long long ph = sc2[0], pl = sc2[1];
  for (int i = lo; i < hi; ++i) {
    if (!(rec[i + glo].flags & 1u)) continue;
    if (L.hflag[i]) v.work_heavy[ph++] = i;
    else v.work[pl++] = i;
  }
  if (tid == 0) {
    v.ctr->work_count = (int)tt2[1];
    v.ctr->work_next = 0;
    v.ctr->heavy_count = (int)tt2[0];
    v.ctr->heavy_next = v.ctr->heavy_next2 = 0;
    v.ctr->cur_step = step;
  }
}

// All phases of the multi-CTA targets in ONE cooperative launch (grid-wide
// barriers between phases; every CTA keeps its 2048 records in shared memory
// across phases, read from HBM once).  Used when the grid (one CTA per 2048
// records) fits on the device at once; the per-phase kernels above are the
// fallback.
__global__ void __launch_bounds__(MT_T) k_mt_all(View v, int step, const ts_sched_record* rec, unsigned char* mt) {
  if (v.pworld && v.ctr->px_done) return;  // ts_run_sharded: the batch has ended
  if (step < 0) step = v.ctr->cur_step;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
#ifdef TS_SCHED_PROF
  const unsigned long long mt_t0 = globaltimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11] += 1;
#endif
  MtLayout L;
  mt_layout(mt, v.n_global, v.n_local, &L);
  __shared__ ts_sched_record srec[MT_REC];
  __shared__ long long sfl[4];
  __shared__ double s_runS[2 * MT_RUNCAP];
  __shared__ int32_t s_runStart[2 * MT_RUNCAP];
  __shared__ long long s_runWant[2 * MT_RUNCAP];
  __shared__ long long s_runPW[2 * MT_RUNCAP];
  const int n = v.n_global, G = gridDim.x, G3 = mt_run_blocks(n);
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int base = b * MT_REC;
  const int nb = min(MT_REC, n - base);
  for (int i = tid; i < nb; i += MT_T) srec[i] = rec[base + i];
  if (b == 0 && tid == 0 && step < v.step_times_cap) v.step_times[step] = globaltimer();
  __syncthreads();
  const int lo = min(nb, tid * MT_CH), hi = min(nb, lo + MT_CH);  // this thread's records, CTA-local
  const ts_config& cf = v.cfg;

  // ---- phase 1: CTA counts, exact partial sums, list minima
  {
    long long c[3] = {0, 0, 0}, tot[3];
    u128 fx = 0;
    bool bad = false;
    double m0 = INFINITY, m1 = INFINITY;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = srec[i];
      if (!(r.flags & 1u)) continue;
      ++c[0];
      u128 q;
      if (to_fixed(r.score, q)) fx += q;
      else bad = true;
      if (r.flags & 2u) {
        if (r.flags & 4u) { ++c[2]; m1 = fmin(m1, r.score); }
        else { ++c[1]; m0 = fmin(m0, r.score); }
      }
    }
    mt_scan<3>(c, tot);
    double tm0, tm1;
    mt_scan_min2(m0, m1, tm0, tm1);
    __shared__ u128 sq[MT_T / 32];
    __shared__ int sbad;
    if (tid == 0) sbad = 0;
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t h = __shfl_down_sync(FULL, (uint64_t)(fx >> 64), o);
      const uint64_t l = __shfl_down_sync(FULL, (uint64_t)fx, o);
      fx += ((u128)h << 64) | l;
    }
    if (lane == 0) sq[wid] = fx;
    __syncthreads();
    if (bad) sbad = 1;
    __syncthreads();
    if (tid == 0) {
      u128 s = 0;
      for (int w = 0; w < MT_T / 32; ++w) s += sq[w];
      MtBlk1 x;
      x.nrun = tot[0];
      x.cnt0 = tot[1];
      x.cnt1 = tot[2];
      x.flo = (unsigned long long)s;
      x.fhi = (unsigned long long)(s >> 64);
      x.bad = sbad;
      x._p = 0;
      x.min0 = tm0;
      x.min1 = tm1;
      L.b1[b] = x;
    }
  }
  grid.sync();
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 1] += globaltimer() - mt_t0;
#endif
  // ---- phase 2 (every CTA, redundantly): CTA offsets, T, totals from the
  // G summaries (no further grid barrier: each CTA keeps its own copy)
  __shared__ MtOff1 s_off;
  __shared__ MtState s_st;
  {
    MtBlk1 x{};
    x.min0 = x.min1 = INFINITY;
    if (tid < G) x = L.b1[tid];
    long long c[3] = {x.nrun, x.cnt0, x.cnt1}, tot[3];
    mt_scan<3>(c, tot);
    double m0 = x.min0, m1 = x.min1, tm0, tm1;
    mt_scan_min2(m0, m1, tm0, tm1);
    __shared__ u128 sq2[MT_T / 32];
    __shared__ int sbad2;
    if (tid == 0) sbad2 = 0;
    u128 fx = tid < G ? (((u128)x.fhi << 64) | x.flo) : 0;
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t h = __shfl_down_sync(FULL, (uint64_t)(fx >> 64), o);
      const uint64_t l = __shfl_down_sync(FULL, (uint64_t)fx, o);
      fx += ((u128)h << 64) | l;
    }
    if (lane == 0) sq2[wid] = fx;
    __syncthreads();
    if (tid < G && x.bad) sbad2 = 1;
    if (tid == b) {
      MtOff1 o;
      o.p0 = c[1];
      o.p1 = c[2];
      o.prev0 = m0;
      o.prev1 = m1;
      s_off = o;
    }
    __syncthreads();
    if (tid == 0) {
      u128 sum = 0;
      for (int w = 0; w < MT_T / 32; ++w) sum += sq2[w];
      const long long tot_run = tot[0];
      bool fallback = sbad2 != 0;
      double T = 0.0;
      if (!fallback) {
        T = fixed_to_double(sum);
        const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
        if ((double)tot_run * u2 >= 0x1p-10) fallback = true;
      }
      if (fallback) {  // sequential Neumaier sum in run-queue order
        double f = 0.0, cc = 0.0;
        bool first = true;
        for (int i = 0; i < n; ++i) {
          const ts_sched_record r = rec[i];
          if (!(r.flags & 1u)) continue;
          const double x2 = r.score;
          if (first) { f = x2; first = false; continue; }
          const double y = f + x2;
          if (fabs(f) >= fabs(x2)) cc += (f - y) + x2;
          else cc += (x2 - y) + f;
          f = y;
        }
        if (cc != 0.0 && isfinite(cc)) f += cc;
        T = f;
        if (b == 0) atomicAdd(&v.ctr->sum_fallbacks, 1);
      }
      MtState st{};
      st.T = T;
      st.tot_run = tot_run;
      st.len0 = tot[1];
      st.len1 = tot[2];
      const long long R = (long long)cf.max_concurrency - tot_run;
      st.boost_on = (cf.boosting_enabled != 0 && tot_run > 0 && R > 0 && tot[1] + tot[2] > 0) ? 1 : 0;
      s_st = st;
    }
    __syncthreads();
  }
  const bool boost_on = s_st.boost_on != 0;
  // ---- phase 3: positions, previous scores, run counts
  MtThr th;
  {
    long long c[2] = {0, 0}, tot[2];
    double m0 = INFINITY, m1 = INFINITY;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = srec[i];
      if ((r.flags & 3u) != 3u) continue;
      if (r.flags & 4u) { ++c[1]; m1 = fmin(m1, r.score); }
      else { ++c[0]; m0 = fmin(m0, r.score); }
    }
    mt_scan<2>(c, tot);
    double tm0, tm1;
    mt_scan_min2(m0, m1, tm0, tm1);
    const MtOff1 o = s_off;
    th.pos0 = o.p0 + c[0];
    th.pos1 = o.p1 + c[1];
    th.prev0 = fmin(o.prev0, m0);
    th.prev1 = fmin(o.prev1, m1);
    long long rs[2] = {0, 0};
    if (boost_on) {
      double p0 = th.prev0, p1 = th.prev1;
      for (int i = lo; i < hi; ++i) {
        const ts_sched_record r = srec[i];
        if ((r.flags & 3u) != 3u) continue;
        if (r.flags & 4u) { if (r.score != p1) ++rs[1]; if (r.score > p1) v.ctr->sched_error = 1; p1 = r.score; }
        else { if (r.score != p0) ++rs[0]; if (r.score > p0) v.ctr->sched_error = 1; p0 = r.score; }
      }
    }
    long long rt[2];
    mt_scan<2>(rs, rt);
    th.rid0 = rs[0];
    th.rid1 = rs[1];
    if (tid == 0) {
      L.b2[b] = rt[0];
      L.b2[G + b] = rt[1];
    }
  }
  grid.sync();
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 2] += globaltimer() - mt_t0;
#endif
  // ---- phase 4 (every CTA): run offsets of the CTAs, run totals
  {
    long long c[2] = {tid < G ? L.b2[tid] : 0, tid < G ? L.b2[G + tid] : 0}, tot[2];
    mt_scan<2>(c, tot);
    __shared__ long long s_roff[2];
    if (tid == b) {
      s_roff[0] = c[0];
      s_roff[1] = c[1];
    }
    if (tid == 0) {
      s_st.nr0 = tot[0];
      s_st.nr1 = tot[1];
    }
    __syncthreads();
    th.rid0 += s_roff[0];
    th.rid1 += s_roff[1];
  }
  // ---- phase 5: run records
  if (boost_on) {
    double p0 = th.prev0, p1 = th.prev1;
    long long q0 = th.pos0, q1 = th.pos1, k0 = th.rid0, k1 = th.rid1;
    for (int i = lo; i < hi; ++i) {
      const ts_sched_record r = srec[i];
      if ((r.flags & 3u) != 3u) continue;
      if (r.flags & 4u) {
        if (r.score != p1) { v.g_runS[n + k1] = r.score; v.g_runStart[n + k1] = (int)q1; ++k1; }
        p1 = r.score;
        ++q1;
      } else {
        if (r.score != p0) { v.g_runS[k0] = r.score; v.g_runStart[k0] = (int)q0; ++k0; }
        p0 = r.score;
        ++q0;
      }
    }
  }
  grid.sync();
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 3] += globaltimer() - mt_t0;
#endif
  const long long M = cf.max_concurrency;
  // ---- phase 6: want per run, per-run-block sums
  if (boost_on) {
    const MtState st = s_st;
    const long long nrmax = st.nr0 > st.nr1 ? st.nr0 : st.nr1;
    const int g3 = (int)((nrmax + MT_T - 1) / MT_T);
    for (int rb = b; rb < g3; rb += G) {
      const long long k = (long long)rb * MT_T + tid;
      long long w[2] = {0, 0}, tot[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long nr = q ? st.nr1 : st.nr0, len = q ? st.len1 : st.len0;
        const int off = q ? n : 0;
        if (k < nr) {
          const long long want = mt_want(v.g_runS[off + k], st.T, M);
          const long long cnt = (k + 1 < nr ? v.g_runStart[off + k + 1] : len) - v.g_runStart[off + k];
          v.g_runWant[off + k] = want;
          w[q] = cnt * (want - 1);
        }
      }
      mt_scan<2>(w, tot);
      if (k < st.nr0) v.g_runPW[k] = w[0];
      if (k < st.nr1) v.g_runPW[n + k] = w[1];
      if (tid == 0) {
        L.b3[rb] = tot[0];
        L.b3[G3 + rb] = tot[1];
      }
    }
  }
  grid.sync();
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 4] += globaltimer() - mt_t0;
#endif
  // ---- phase 7 (every CTA): run-block offsets into shared memory, tw0/tw1
  __shared__ long long s_b3[2 * MT_RB];
  const bool b3_smem = G3 <= MT_RB;
  {
    const MtState st = s_st;
    const long long nrmax = st.nr0 > st.nr1 ? st.nr0 : st.nr1;
    const int g3 = boost_on ? (int)((nrmax + MT_T - 1) / MT_T) : 0;
    long long carry0 = 0, carry1 = 0;
    for (int base3 = 0; base3 < g3; base3 += MT_T) {
      const int rb = base3 + tid;
      long long c[2] = {rb < g3 ? L.b3[rb] : 0, rb < g3 ? L.b3[G3 + rb] : 0}, tot[2];
      mt_scan<2>(c, tot);
      if (rb < g3) {
        if (b3_smem) {
          s_b3[rb] = carry0 + c[0];
          s_b3[MT_RB + rb] = carry1 + c[1];
        } else if (b == 0) {
          // a separate array: the other CTAs are still reading the totals in b3
          L.b3p[rb] = carry0 + c[0];
          L.b3p[G3 + rb] = carry1 + c[1];
        }
      }
      carry0 += tot[0];
      carry1 += tot[1];
    }
    if (tid == 0) {
      s_st.tw0 = carry0;
      s_st.tw1 = carry1;
    }
    __syncthreads();
  }
  if (!b3_smem) grid.sync();  // CTA 0 wrote the global run-block offsets
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 5] += globaltimer() - mt_t0;
#endif
  // ---- phase 8: targets of the local records, pipelined-mode flags, per-CTA list counts
  const int glo = v.goff, ghi = v.goff + v.n_local;
  long long nh = 0, nlt = 0;
  if (base + nb > glo && base < ghi) {  // this CTA holds local records (CTA-uniform: the staging syncs)
    const MtState st = s_st;
    const long long R = M - st.tot_run, U = st.len0 + st.len1;
    long long Rp = R - (st.tw0 + st.tw1);
    if (Rp < 0) Rp = 0;
    // the runs of both lists (score, start, want, Σ before) in shared memory when
    // they fit: the binary searches below then never leave the SM
    const bool in_smem = st.nr0 <= MT_RUNCAP && st.nr1 <= MT_RUNCAP;
    const double* runS = v.g_runS;
    const int32_t* runStart = v.g_runStart;
    const long long* runWant = v.g_runWant;
    const long long* runPWg = v.g_runPW;
    int off1 = n;
    if (in_smem) {
      off1 = MT_RUNCAP;
      for (int q = 0; q < 2; ++q) {
        const long long nr = q ? st.nr1 : st.nr0;
        const int go = q ? n : 0, so = q ? MT_RUNCAP : 0;
        for (int k = tid; k < nr; k += MT_T) {
          s_runS[so + k] = v.g_runS[go + k];
          s_runStart[so + k] = v.g_runStart[go + k];
          s_runWant[so + k] = v.g_runWant[go + k];
          s_runPW[so + k] = v.g_runPW[go + k] + (b3_smem ? s_b3[(q ? MT_RB : 0) + k / MT_T] : L.b3p[(q ? G3 : 0) + k / MT_T]);
        }
      }
      runS = s_runS;
      runStart = s_runStart;
      runWant = s_runWant;
      runPWg = s_runPW;
    }
    __syncthreads();
    auto runPW = [&](int off, long long k) {
      if (in_smem) return runPWg[off + k];
      const long long blk = b3_smem ? s_b3[(off ? MT_RB : 0) + k / MT_T] : L.b3p[(off ? G3 : 0) + k / MT_T];
      return runPWg[off + k] + blk;
    };
    long long q0 = th.pos0, q1 = th.pos1, k0 = th.rid0 - 1, k1 = th.rid1 - 1;
    double p0 = th.prev0, p1 = th.prev1;
    for (int ii = lo; ii < hi; ++ii) {
      const ts_sched_record r = srec[ii];
      const int i = base + ii;
      const bool local = i >= glo && i < ghi;
      if (!(r.flags & 1u)) {
        if (local) {
          v.tgt[i - glo] = 0;
          L.hflag[i - glo] = 0;
        }
        continue;
      }
      long long tgt = 1;
      if ((r.flags & 2u) && boost_on) {
        const int lb = (r.flags & 4u) ? 1 : 0;
        long long pos, k;
        if (lb) { if (r.score != p1) ++k1; p1 = r.score; pos = q1++; k = k1; }
        else { if (r.score != p0) ++k0; p0 = r.score; pos = q0++; k = k0; }
        if (local) {
          const int off = lb ? off1 : 0, oo = lb ? 0 : off1;
          const long long want = runWant[off + k];
          long long before = runPW(off, k) + (pos - runStart[off + k]) * (want - 1);
          const long long nro = lb ? st.nr0 : st.nr1, leno = lb ? st.len0 : st.len1, two = lb ? st.tw0 : st.tw1;
          const long long obefore = lb ? q0 : q1;
          int lo2 = 0, hi2 = (int)nro;
          while (lo2 < hi2) {
            const int mid = (lo2 + hi2) >> 1;
            if (runS[oo + mid] > r.score) lo2 = mid + 1;
            else hi2 = mid;
          }
          const int kk = lo2;
          long long c, cw;
          if (kk < nro && runS[oo + kk] == r.score) {
            const long long st0 = runStart[oo + kk];
            const long long cntk = (kk + 1 < nro ? runStart[oo + kk + 1] : leno) - st0;
            long long part = obefore - st0;
            if (part < 0) part = 0;
            if (part > cntk) part = cntk;
            c = st0 + part;
            cw = runPW(oo, kk) + part * (runWant[oo + kk] - 1);
          } else if (kk < nro) {
            c = runStart[oo + kk];
            cw = runPW(oo, kk);
          } else {
            c = leno;
            cw = two;
          }
          const long long spos = pos + c;
          before += cw;
          long long extra = R - before;
          if (extra < 0) extra = 0;
          if (extra > want - 1) extra = want - 1;
          long long rr = 0;
          if (U > 0) rr = Rp / U + (spos < Rp % U ? 1 : 0);
          tgt = 1 + extra + rr;
        }
      }
      if (local) {
        v.tgt[i - glo] = (int)tgt;
        const bool hv = v.heavy_on && min(tgt, (long long)(cf.rollout_budget - (int)r._pad)) >= HEAVY_P;
        L.hflag[i - glo] = hv ? 1 : 0;
        if (hv) ++nh;
        else ++nlt;
      }
    }
  }
  {
    long long c[2] = {nh, nlt}, tot[2];
    mt_scan<2>(c, tot);
    nh = c[0];
    nlt = c[1];
    if (tid == 0) {
      L.b1[b].nrun = tot[0];  // b1 is free after phase 2: per-CTA list counts
      L.b1[b].cnt0 = tot[1];
    }
  }
  grid.sync();
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[11 + 6] += globaltimer() - mt_t0;
#endif
  // ---- phase 9: work lists in run-queue order
  {
    if (tid == 0) {
      long long h = 0, l = 0;
      for (int j = 0; j < b; ++j) {
        h += L.b1[j].nrun;
        l += L.b1[j].cnt0;
      }
      sfl[0] = h;
      sfl[1] = l;
      if (b == G - 1) {
        v.ctr->heavy_count = (int)(h + L.b1[b].nrun);
        v.ctr->work_count = (int)(l + L.b1[b].cnt0);
        v.ctr->work_next = 0;
        v.ctr->heavy_next = v.ctr->heavy_next2 = 0;
        v.ctr->cur_step = step;
      }
    }
    __syncthreads();
    long long ph = sfl[0] + nh, pl = sfl[1] + nlt;
    for (int ii = lo; ii < hi; ++ii) {
      const int i = base + ii;
      if (i < glo || i >= ghi || !(srec[ii].flags & 1u)) continue;
      if (L.hflag[i - glo]) v.work_heavy[ph++] = i - glo;
      else v.work[pl++] = i - glo;
    }
  }
#ifdef TS_SCHED_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) v.ctr->prof[18] += globaltimer() - mt_t0;
#endif
}

// Caller-provided parallelism targets (an external scheduler): P_i for every
// local search, then the work lists of the wave exactly as compute_targets'
// phase 5 builds them.  Running searches get max(1, P_i), others 0.
__global__ void __launch_bounds__(TT) k_set_targets(View v, int step, const int32_t* __restrict__ P) {
  __shared__ long long shl[264];
  const int tid = threadIdx.x, nl = v.n_local;
  if (tid == 0 && step < v.step_times_cap) v.step_times[step] = globaltimer();
  const int per = (nl + TT - 1) / TT;
  const int lo = min(nl, tid * per), hi = min(nl, lo + per);
  const ts_config& cf = v.cfg;
  long long nh = 0, nlt = 0;
  for (int i = lo; i < hi; ++i) {
    SearchState* st = v.st + i;
    if (st->state != ST_RUNNING) {
      v.tgt[i] = 0;
      continue;
    }
    const int t = max(1, P[i]);
    v.tgt[i] = t;
    if (v.heavy_on && min(t, cf.rollout_budget - st->completed) >= HEAVY_P) ++nh;
    else ++nlt;
  }
  long long sc2[4] = {nh, nlt, 0, 0}, tt2[4];
  block_scan_add4(sc2, tt2, shl);
  long long ph = sc2[0], pl = sc2[1];
  for (int i = lo; i < hi; ++i) {
    const SearchState* st = v.st + i;
    if (st->state != ST_RUNNING) continue;
    if (v.heavy_on && min(v.tgt[i], cf.rollout_budget - st->completed) >= HEAVY_P) v.work_heavy[ph++] = i;
    else v.work[pl++] = i;
  }
  if (tid == 0) {
    v.ctr->work_count = (int)tt2[1];
    v.ctr->work_next = 0;
    v.ctr->heavy_count = (int)tt2[0];
    v.ctr->heavy_next = v.ctr->heavy_next2 = 0;
    v.ctr->cur_step = step;
  }
}

// The scheduler's view of the local searches (Job fields, scheduler.py:63-74)
// for an external scheduler: running flag, completed_rollouts, best_score.
__global__ void k_read_jobs(View v, int32_t* running, int32_t* completed, double* best) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.n_local) return;
  const SearchState* st = v.st + i;
  if (running) running[i] = st->state == ST_RUNNING ? 1 : 0;
  if (completed) completed[i] = st->completed;
  if (best) best[i] = st->job_best;
}

// Number of requests with arrival_step <= step (arrivals are non-decreasing),
// by one warp: a 32-way split per round instead of a binary search.
__device__ int arrived_count(const View& v, int step) {
  if (step >= v.max_arrival) return v.n_local;
  const int lane = threadIdx.x & 31;
  // invariant: arrival[i] <= step for i < lo, arrival[i] > step for i >= hi
  int lo = 0, hi = v.n_local;
  while (hi - lo > 32) {
    const int span = (hi - lo + 31) / 32;
    const int p = lo + lane * span;
    const int t = __popc(__ballot_sync(FULL, p < hi && v.arrival[p] <= step));  // a prefix of the samples
    if (t == 0) { hi = lo; break; }
    const int nhi = min(hi, lo + t * span);  // sample t (if any) is past step
    lo = lo + (t - 1) * span + 1;            // sample t-1 is not
    hi = nhi;
  }
  return lo + __popc(__ballot_sync(FULL, lo + lane < hi && v.arrival[lo + lane] <= step));
}

// One scheduler pass of a single-GPU run, fused: the loop test of the wave
// driver, admit_jobs, parallelism_score records and compute_targets.  The
// step counter lives on the device, so a CUDA-graph while-loop of
// {k_sched, k_wave} runs a whole batch without host round trips.
__global__ void __launch_bounds__(SCHED_T) k_sched(View v, ts_sched_record* rec, cudaGraphConditionalHandle cond,
                                              int use_cond) {
  __shared__ int s_go, s_min, s_fast, s_wlo, s_whi;
  __shared__ long long s_alo, s_ahi;
  Counters* c = v.ctr;
#ifdef TS_SCHED_PROF
  unsigned long long sp_t = globaltimer();
  if (threadIdx.x == 0 && c->prof[20] && !c->prof[30]) {  // 30: the batch has ended (empty passes follow)
    c->prof[0] += sp_t - c->prof[20];
    c->prof[1] += c->prof[20] - c->prof[21];
    c->prof[2] += c->prof[21] - c->prof[22];
  }
#endif
  const int step = (int)c->step;
  int arrived = 0;
  if (threadIdx.x < 32) arrived = arrived_count(v, step);
  if (threadIdx.x == 0) {
    const int lo = arrived;
    // every counter in one round of loads; the pass's bounds go to the other
    // threads through shared memory
    const long long fin = c->finished, max_steps = c->max_steps, running = c->running, head = c->head,
                    win_lo = c->win_lo;
    const long long unfinished = (long long)v.n_local - fin;
    const bool go = unfinished > 0 && step < max_steps && step < v.log1p_n;
    if (go) {
      long long q = (long long)v.cfg.max_concurrency - running;
      if (q > (long long)lo - head) q = (long long)lo - head;
      if (q < 0) q = 0;
      c->admit_lo = head;
      c->admit_hi = head + q;
      c->head = head + q;
      c->running = running + q;
      s_alo = head;
      s_ahi = head + q;
      s_wlo = (int)win_lo;
      s_whi = (int)(head + q);
      s_min = (int)(head + q);
      // no free slot, or boosting off: compute_targets gives every running job
      // P = 1 (scheduler.py:160-163) whatever the scores, so the pass only
      // needs the list of running searches
      s_fast = (long long)v.cfg.max_concurrency - (running + q) <= 0 || v.cfg.boosting_enabled == 0;
    } else {
      c->work_count = 0;
      c->work_next = 0;
      c->heavy_count = 0;
      c->heavy_next = c->heavy_next2 = 0;
      c->free_run = 0;
      if (use_cond) cudaGraphSetConditional(cond, 0);
#ifdef TS_SCHED_PROF
      c->prof[30] = 1;
#endif
    }
    s_go = go;
  }
  __syncthreads();
  if (!s_go) return;
  SP_MARK(3, sp_t);
  const long long alo = s_alo, ahi = s_ahi;
  const ts_config& cf = v.cfg;
  // the run queue is the window [win_lo, head): searches below win_lo have
  // exited, searches from head on are not admitted yet
  const int wlo = s_wlo, whi = s_whi;
  const int nw = whi - wlo;
  // one GPU: the window's records stay in shared memory when they fit
  extern __shared__ __align__(16) unsigned char smem[];
  ts_sched_record* srec = nw <= SREC_MAX ? (ts_sched_record*)(smem + targets_smem_dev()) : rec;
  // Records.  targets_block gives thread t the records [t*per, (t+1)*per), so
  // warp w's threads own the chunk [32*w*per, 32*(w+1)*per): the warp fills
  // its chunk with lane-consecutive (coalesced) loads, four in flight per
  // lane, and a warp barrier replaces a block barrier before the call.
  const int per = (nw + SCHED_T - 1) / SCHED_T;
  const int lane = threadIdx.x & 31;
  const int c0 = min(nw, (int)(threadIdx.x >> 5) * 32 * per), c1 = min(nw, c0 + 32 * per);
  int my_min = whi;
  bool ungated = false;  // a running search past the observation gate
  for (int j0 = c0; j0 < c1; j0 += 4 * 32) {
    // the record the search's last wave wrote, else (admitted now, or written
    // for another step by the step API) gathered from the SearchState
    ts_sched_record rr[4];
    bool slow[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * 32 + lane, i = wlo + j;
      slow[u] = false;
      if (j < c1) rr[u] = v.nrec[i];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * 32 + lane, i = wlo + j;
      const uint32_t tag = rr[u].flags >> 8;
      slow[u] = j < c1 && ((i >= alo && i < ahi) || (tag != (uint32_t)step && tag != NREC_FINAL));
    }
    if (slow[0] | slow[1] | slow[2] | slow[3]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!slow[u]) continue;
        const int i = wlo + j0 + u * 32 + lane;
        const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(v.st + i);
        const bool adm = i >= alo && i < ahi;
        const int state = adm ? (int)ST_RUNNING : (int)(uint32_t)w.x;
        const int done = (int)(uint32_t)(w.x >> 32);
        const double jb = __longlong_as_double((long long)w.y);
        if (adm) {
          v.st[i].state = ST_RUNNING;
          v.st[i].admit_step = step;
        }
        ts_sched_record r;
        r.score = 0.0;
        r.flags = 0;
        r._pad = 0;
        if (state == ST_RUNNING) {
          const double ratio = jb / cf.positive_exit_threshold;
          const bool boosted = ratio > cf.proximity;
          r.score = v.log1p_tab[step - v.arrival[i]] + (boosted ? cf.beta : 0.0);
          r.flags = 1u | (done >= cf.obs_threshold ? 2u : 0u) | (boosted ? 4u : 0u);
          r._pad = (uint32_t)done;
        }
        rr[u] = r;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * 32 + lane, i = wlo + j;
      if (j >= c1) break;
      rr[u].flags &= 7u;
      if (rr[u].flags & 1u) my_min = min(my_min, i);
      ungated |= (rr[u].flags & 3u) == 3u;
      srec[j] = rr[u];
    }
  }
  __syncwarp();
  for (int o = 16; o > 0; o >>= 1) my_min = min(my_min, __shfl_xor_sync(FULL, my_min, o));
  if ((threadIdx.x & 31) == 0) atomicMin(&s_min, my_min);
  SP_MARK(4, sp_t);
  static_assert(HEAVY_P > 1, "P = 1 searches run in single-warp mode");
  // nobody past the observation gate: the extra and leftover loops of
  // compute_targets run over an empty list (scheduler.py:166-186), P = 1 again
  const bool fast = __syncthreads_or(ungated) == 0 || s_fast;
  if (fast) {
    // the running searches of the warp's chunk, in run-queue order, onto the
    // single-warp work list
    __shared__ int s_wcnt[SCHED_W];
    const int wid = threadIdx.x >> 5;
    int cnt = 0;
    for (int j = c0 + lane; j < c1; j += 32) cnt += (int)(srec[j].flags & 1u);
    cnt = __reduce_add_sync(FULL, cnt);
    if (lane == 0) s_wcnt[wid] = cnt;
    if (threadIdx.x == 0 && step < v.step_times_cap) v.step_times[step] = globaltimer();
    __syncthreads();
    const int wt = lane < SCHED_W ? s_wcnt[lane] : 0;
    int pos = __reduce_add_sync(FULL, lane < wid ? wt : 0);
    const int total = __reduce_add_sync(FULL, wt);
    __shared__ int s_cmin, s_cmax;
    if (threadIdx.x == 0) { s_cmin = 0x7FFFFFFF; s_cmax = -1; }
    __syncthreads();
    int cmin = 0x7FFFFFFF, cmax = -1;
    for (int j0 = c0; j0 < c1; j0 += 32) {
      const int j = j0 + lane;
      const bool run = j < c1 && (srec[j].flags & 1u);
      const unsigned b = __ballot_sync(FULL, run);
      if (run) {
        v.work[pos + __popc(b & ((1u << lane) - 1u))] = wlo + j;
        const int done = (int)srec[j]._pad;  // completed_rollouts
        cmin = min(cmin, done);
        cmax = max(cmax, done);
        if (v.free_ok) v.fdone[wlo + j] = 0;
      }
      if (j < c1) v.tgt[wlo + j] = run ? 1 : 0;
      pos += __popc(b);
    }
    cmin = __reduce_min_sync(FULL, cmin);
    cmax = __reduce_max_sync(FULL, cmax);
    if (lane == 0) {
      atomicMin(&s_cmin, cmin);
      atomicMax(&s_cmax, cmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c->work_count = total;
      c->work_next = 0;
      c->heavy_count = 0;
      c->heavy_next = c->heavy_next2 = 0;
      c->cur_step = step;
      // Free-running waves.  When every search is admitted, nobody can exit
      // before its budget (no positive/negative exit; the trees are too deep
      // to be exhausted within the budget, v.free_ok) and the next passes can
      // only give P = 1 again (boosting off, or no free slot while every
      // running search has the same remaining budget, so that nobody exits
      // before the others), each search's remaining waves are one rollout each
      // and independent of every other search: the wave kernel runs them back
      // to back, each search's rollouts in wave order (step = t0 + r), without
      // a scheduler pass or a grid-wide barrier per wave.
      const int rem = cf.rollout_budget - s_cmin;
      const bool freerun = v.free_ok && total > 0 && c->head == (long long)v.n_local && rem > 0 &&
                           (cf.boosting_enabled == 0 ||
                            ((long long)cf.max_concurrency - c->running <= 0 && s_cmin == s_cmax)) &&
                           (long long)step + rem <= c->max_steps;
      c->free_run = freerun ? 1 : 0;
      if (freerun) {
        c->free_t0 = step;
        c->free_rem = rem;
        c->free_next = 0;
      }
    }
    SP_MARK(9, sp_t);
  } else {
    if (threadIdx.x == 0) c->free_run = 0;
    if (srec != rec) {
      // the window's running searches compacted in place (shared memory, run-
      // queue order kept, the window offset in flags bits 8+): compute_targets
      // only sees running jobs, so the passes below touch the few still
      // running (config 2's last waves: 297 and 39 of a 4096-search window)
      // instead of the window.  srec is in shared memory only for nw <=
      // SREC_MAX = 4 * SCHED_T, so a lane holds at most 4 records of its
      // warp's chunk while every warp reads before any writes.
      static_assert(SREC_MAX <= 4 * SCHED_T, "in-place compaction holds 4 records per lane");
      __shared__ int s_ccnt[SCHED_W];
      const int wid = threadIdx.x >> 5;
      ts_sched_record rr[4];
      unsigned bal[4];
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = c0 + u * 32 + lane;
        rr[u].flags = 0;
        if (j < c1) rr[u] = srec[j];
        bal[u] = __ballot_sync(FULL, j < c1 && (rr[u].flags & 1u));
        cnt += __popc(bal[u]);
        if (j < c1 && !(rr[u].flags & 1u)) v.tgt[wlo + j] = 0;
      }
      if (lane == 0) s_ccnt[wid] = cnt;
      __syncthreads();
      const int wt = lane < SCHED_W ? s_ccnt[lane] : 0;
      int pos = __reduce_add_sync(FULL, lane < wid ? wt : 0);
      const int nrun = __reduce_add_sync(FULL, wt);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if ((bal[u] >> lane) & 1u) {
          ts_sched_record r = rr[u];
          r.flags |= (uint32_t)(c0 + u * 32 + lane) << 8;
          srec[pos + __popc(bal[u] & ((1u << lane) - 1u))] = r;
        }
        pos += __popc(bal[u]);
      }
      __syncthreads();
      targets_block(v, step, srec, nrun, 0, nrun, wlo, true);
    } else {
      targets_block(v, step, srec, nw, 0, nw, wlo);
    }
  }
  if (threadIdx.x == 0) {
    c->win_lo = s_min;  // no running search below this index
    c->step = c->free_run ? step + c->free_rem : step + 1;
    c->passes += 1;
#ifdef TS_SCHED_PROF
    c->prof[10] += 1;
    c->prof[20] = 0;
    c->prof[21] = ~0ull;
    c->prof[22] = globaltimer();
#endif
  }
}

// ---- the wave: one warp per running search ----------------------------------
struct WaveStats {
  unsigned long long rollouts, launched, nodes, scored, levels, path_nodes, tokens;
};

constexpr int WAVE_THREADS = 128;
constexpr int WAVE_WARPS = WAVE_THREADS / 32;

// One wave of one search, executed by one warp.
//
// Per rollout the warp walks root→leaf (select_leaf) and leaf→terminal
// (simulate_to_terminal).  Each selection level is one round of child loads,
// WU-PUCT and an argmax.  Each simulation level computes, lane j = child j,
// everything generate_steps draws for the child (reward, raw prior, tokens,
// terminal flag) from the running fold states; greedy_child needs only the
// rewards, the other draws fill the issue slots the dependent chain leaves
// idle and are staged in shared memory.  After the descent one lane-parallel
// batch (lane l = the expansion at depth l) normalises the priors with
// CPython's Neumaier sum, writes the node records and parent links and counts
// negative-exit leaves.
//
// Lane l also keeps path node l+1 in registers (id, meta, N|O word, W, reward,
// prefix aggregate, golden flag, chosen child index), so registration and a
// single-rollout backup are pure stores, and subtree exhaustion propagates up
// the path without loads.  WT = compile-time width (0: runtime, <= 32).
template <int NSLOT, int WT, bool SINGLE = false, bool PROD = false>
__device__ void search_wave(const View& v, int s, int step, WaveStats& ws, double* s_raw, double* s_rew) {
  constexpr int WS = WT ? WT : TS_MAX_WIDTH;  // shared-memory row stride
  const int lane = threadIdx.x & 31;
  const ts_config& cf = v.cfg;
  SearchState* S = v.st + s;
  const ts_problem* pb = v.prob + s;
  const size_t base = (size_t)s * (size_t)v.cap;
  uint64_t* NO = v.no + base;
  double* Wv = v.W + base;
  double* PR = v.prior + base;
  double* RW = v.reward + base;
  double* QQ = v.Q + base;
  uint64_t* MF = v.mf + base;
  uint32_t* ME = (uint32_t*)MF;  // ME[2*i]: meta word of node i
  int32_t* PA = v.parent + base;

  const uint64_t seed = pb->seed;
  const int bdepth = pb->base_depth;
  const int glen = pb->golden_len;
  const int hidden = pb->hidden_until_depth;
  const bool has_shared = pb->has_shared != 0;
  const double off_lo = pb->off_lo, off_hi = pb->off_hi;
  const double sh_lo = pb->shared_lo, sh_hi = pb->shared_hi;
  const int width = WT ? WT : min(cf.expand_width, pb->branching);
  const int scheme = cf.scheme;
  const bool strict = cf.strict_negative_exit != 0;
  const bool prefix_bound = cf.futility_bound == TS_BOUND_PREFIX_AGGREGATE;
  const double tau = cf.accept_threshold, theta1 = cf.first_step_threshold;
  const double c_puct = cf.c_puct;
  // lane l holds golden_path[l] and its lifted reward
  const int gstep = lane < glen ? (int)pb->golden_path[lane] : -1;
  const double grew = lane < glen ? pb->golden_rewards[lane] : 0.0;

  int completed = S->completed;
  int nnodes = S->nodes;
  int viable = S->viable;
  int best_term = S->best_term;
  double best = S->best;
  int launched = S->launched, cancelled = S->cancelled;
  int status = TS_OK;
  const int budget = cf.rollout_budget;
  // SINGLE: one rollout this wave (free-running waves), the multi-rollout
  // bookkeeping compiled out
  const int count = SINGLE ? min(1, budget - completed) : min(v.tgt[s], budget - completed);
  const bool multi = !SINGLE && count > 1;
  int32_t* SPs = v.sp + (size_t)s * (size_t)budget * 32;
  double* SSs = v.ss + (size_t)s * budget;
  int32_t* SLs = v.sl + (size_t)s * budget;

  // root fold states fold(seed, tag, len) for this lane's slots
  uint64_t root_h[NSLOT];
  {
    const uint64_t h0 = sm64(MIX_INIT ^ seed);
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
      uint64_t tag, len;
      slot_header<NSLOT>(lane, k, tag, len);
      root_h[k] = sm64(sm64(h0 ^ tag) ^ len);
    }
  }
  // the root's record lives in registers for the whole wave (sole writer)
  const uint64_t rmf = MF[0];
  uint32_t root_meta = (uint32_t)rmf;
  uint64_t rno = NO[0];
  double rW = Wv[0];
  const double rQ = QQ[0];  // W/N of the root (N > 0), constant during a wave
  int rfc = (int)(rmf >> 32);
  int decision = TS_EXIT_NONE;
  int nl = 0;
  long long tok_acc = 0;  // per-lane token tally, reduced once per wave
  // last rollout's path registers (the P=1 backup uses them directly)
  int pnode = -1, plen = 0, pj = 0;
  uint32_t pmeta = 0, lvl_term = 0;
  uint64_t pno = 0;
  double pW = 0.0, prew = 0.0, pagg = 1.0, pscore = 0.0;
  bool pgold = false;
  unsigned long long scored = 0, levels = 0, created = 0, pathn = 0;

  for (int r = 0; r < count && status == TS_OK; ++r) {
    if (!meta_expandable(root_meta)) {  // NoExpandableLeafError (tree.py:273-274)
      if (r == 0) decision = -1;        // exhausted: decide below
      break;
    }
    uint64_t h[NSLOT];
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) h[k] = root_h[k];
    int node = 0, depth = 0, nfc = rfc;
    uint32_t nmeta = root_meta;
    uint64_t nno = rno;
    double nW = rW, nQ = rQ, nrew = 1.0;
    pnode = -1;
    Agg agg;
    agg.init();
    bool golden = glen >= 0;
    double d1r = 1.0;

    // --- select_leaf (tree.py:264-284): one round of child loads per level ---
    while (nmeta & M_KIDS) {
      const unsigned pN = (uint32_t)nno, pO = (uint32_t)(nno >> 32);
      const double psq = sqrt((double)(pN + pO));
      const double pq = pN == 0 ? 0.5 : nQ;  // parent.mean_value(default=0.5)
      const int fc = nfc;
      bool valid = lane < width;
      double sc = -INFINITY, cr = 0.0, cw = 0.0, cq = 0.0;
      uint32_t cm = 0;
      uint64_t cno = 0;
      int cfc = -1;
      if (valid) {
        const int c = fc + lane;
        cno = NO[c];
        cw = Wv[c];
        cq = QQ[c];
        const double cp = PR[c];
        const uint64_t cmf = MF[c];
        cm = (uint32_t)cmf;
        cr = RW[c];
        cfc = (int)(cmf >> 32);
        valid = meta_expandable(cm);
        // branch-free, so all loads issue together; masked by `valid`
        const unsigned cN = (uint32_t)cno, cO = (uint32_t)(cno >> 32);
        // _child_q (tree.py:235-239): W/N, kept as Q since the last backup
        const double q = cN == 0 ? pq : cq;
        // wu_puct_score (tree.py:232): q + c*P*sqrt(N_s+O_s)/(1+N_sa+O_sa)
        const double u = c_puct * cp * psq / (double)(1u + cN + cO);
        if (valid && (!(q >= 0.0 && q <= 1.0) || !(cp >= 0.0 && cp <= 1.0))) status = TS_INVALID_ARGUMENT;
        sc = valid ? q + u : -INFINITY;
      }
      const unsigned vb = __ballot_sync(FULL, valid);
      if (__any_sync(FULL, status != TS_OK)) { status = TS_INVALID_ARGUMENT; break; }
      if (!vb) { status = TS_EXHAUSTED; break; }
      scored += __popc(vb);
      ++levels;
      const int j = warp_argmax(sc, valid, 0);
      node = fc + j;
      ++depth;
      nmeta = __shfl_sync(FULL, cm, j);
      nrew = __shfl_sync(FULL, cr, j);
      nno = __shfl_sync(FULL, cno, j);
      nW = __shfl_sync(FULL, cw, j);
      nQ = __shfl_sync(FULL, cq, j);
      nfc = __shfl_sync(FULL, cfc, j);
      if constexpr (PROD) {  // math.prod (scoring.py:113), the scheme fixed at compile time
        agg.a = agg.a * nrew;
        ++agg.n;
      } else {
        agg.add(nrew, scheme);
      }
      if (depth == 1) d1r = nrew;
      golden = golden && depth <= glen && __shfl_sync(FULL, gstep, depth - 1) == j;
      if (lane == depth - 1) {
        pnode = node; pmeta = nmeta; pno = nno; pW = nW; prew = nrew; pagg = agg.a; pgold = golden; pj = j;
      }
#pragma unroll
      for (int k = 0; k < NSLOT; ++k) h[k] = sm64(h[k] ^ (uint64_t)j);
    }
    if (status != TS_OK) break;
    const int d0 = depth;  // the selected non-terminal leaf
    const int fc0 = nnodes;

    // --- simulate_to_terminal (tree.py:322-349) with generate_steps replayed
    //     (backend.py:230-269); lane j = child j ---
    bool forced = false;
    uint64_t snap[NSLOT];
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) snap[k] = 0;
    while (true) {
      if (depth >= cf.depth_cap) { forced = true; break; }  // tree.py:340-343
      // (the pool holds every node a search's budget can create, ts_load_problems;
      // the single-rollout build leaves the check out)
      if (!SINGLE && nnodes + width > v.cap) { status = TS_POOL_OVERFLOW; break; }
      const int d = depth;
      const int len = d + 1;
      const uint64_t hr = state_at<NSLOT, 1>(h, d);
      snap_take<NSLOT>(snap, h, d);
      const double graw = __shfl_sync(FULL, grew, d);
      const int gnext = __shfl_sync(FULL, gstep, d);
      const bool gchild = golden && len <= glen && lane == gnext;
      const uint64_t jj = (uint64_t)lane;
      double rew;
      if (gchild) {
        rew = graw;
      } else {
        const bool shr = has_shared && len <= hidden;
        const double lo = shr ? sh_lo : off_lo, hi = shr ? sh_hi : off_hi;
        rew = lo + (hi - lo) * u53(sm64(hr ^ jj));
      }
      bool term;
      if (len < bdepth) {
        term = false;
      } else if (len >= bdepth + 1) {
        term = true;
      } else {
        const uint64_t he = state_at<NSLOT, 3>(h, d);
        term = gchild || (sm64(he ^ jj) & 1ull) != 0;  // not _branch_extends
      }
      const bool vl = lane < width;
      const int j = warp_argmax(rew, vl, 0);  // greedy_child (tree.py:307-319)
      const unsigned tmask = __ballot_sync(FULL, vl && term);
      if (vl) s_rew[d * WS + lane] = rew;
      if (lane == d) lvl_term = tmask;
      const bool jterm = (tmask >> j) & 1u;
      node = nnodes + j;
      nnodes += width;
      ++depth;
      nrew = __shfl_sync(FULL, rew, j);
      nmeta = (uint32_t)depth | ((uint32_t)j << SH_REF) | (jterm ? M_TERM : 0u);
      if constexpr (PROD) {  // math.prod (scoring.py:113), the scheme fixed at compile time
        agg.a = agg.a * nrew;
        ++agg.n;
      } else {
        agg.add(nrew, scheme);
      }
      if (depth == 1) d1r = nrew;
      golden = golden && depth <= glen && gnext == j;
      if (lane == depth - 1) {
        pnode = node; pmeta = nmeta; pno = O_ONE; pW = 0.0; prew = nrew; pagg = agg.a; pgold = golden; pj = j;
      }
#pragma unroll
      for (int k = 0; k < NSLOT; ++k) h[k] = sm64(h[k] ^ (uint64_t)j);
      if (jterm) break;
    }
    if (status != TS_OK) break;
    __syncwarp();
    const int dend = depth;      // terminal (or force-terminated) node depth
    const int nlev = dend - d0;  // expansions happened at depths d0 .. dend-1
    plen = dend;
    pscore = PROD ? agg.a : agg.value(scheme);

    // --- deferred expansion batch: lane l writes the children of depth l ---
    // values of path node l (the expanded node) come from lane l-1
    const int up_node = __shfl_up_sync(FULL, pnode, 1);
    const uint32_t up_meta = __shfl_up_sync(FULL, pmeta, 1);
    const double up_rew = __shfl_up_sync(FULL, prew, 1);
    const double up_agg = __shfl_up_sync(FULL, pagg, 1);
    const int upj = __shfl_up_sync(FULL, pj, 1);
    const int node_l = lane == 0 ? 0 : up_node;
    const uint32_t leaf_meta = lane == 0 ? root_meta : up_meta;
    const double rew_l = lane == 0 ? 1.0 : up_rew;
    const double agg_l = lane == 0 ? 1.0 : up_agg;
    const bool act = lane >= d0 && lane < d0 + nlev;
    int live = 0;    // non-terminal children of this level
    int ne_cnt = 0;  // NE: check-relevant viable new leaves
    uint32_t meta_l = 0;
    uint64_t hp, hk;
    snap_prior_tokens<NSLOT>(snap, hp, hk);
    if (act) {
      const int l = lane;
      const int len = l + 1;
      const int fcl = fc0 + (l - d0) * width;
      // raw priors and token counts of this level's children (generate_steps);
      // widths up to 4 keep them in registers with the loops unrolled, wider
      // levels stage them in shared memory with the loops unrolled by 2 (code
      // size: config 4's width-8 kernel stalled on instruction fetch)
      constexpr bool RREG = WT > 0 && WT <= 4;
      constexpr int UR = RREG ? WT : 2;
      double rv[RREG ? WT : 1];
      double* rawl = s_raw + l * WS;
#pragma unroll UR
      for (int i = 0; i < WS; ++i) {
        if (i >= width) break;
        const double x = draw_raw_prior(hp, i);
        if constexpr (RREG) rv[i] = x;
        else rawl[i] = x;
        tok_acc += draw_tokens(hk, i);
      }
#define rawv(i) pick_raw<RREG ? WT : 0>(rv, rawl, i)
      const double* rewl = s_rew + l * WS;
      // total = sum(raw_priors): CPython Neumaier sum in child order
      double tot = rawv(0), cc = 0.0;
#pragma unroll UR
      for (int i = 1; i < WS; ++i) {
        if (i >= width) break;
        const double x = rawv(i);
        const double t = tot + x;
        if (fabs(tot) >= fabs(x)) cc += (tot - t) + x;
        else cc += (x - t) + tot;
        tot = t;
      }
      if (cc != 0.0 && isfinite(cc)) tot += cc;
      const bool last = l == dend - 1;
      const bool rel_d1 = strict || d1r >= theta1;
#pragma unroll UR
      for (int j = 0; j < WS; ++j) {
        if (j >= width) break;
        const double rew = rewl[j];
        const bool term = (lvl_term >> j) & 1u;
        const int c = fcl + j;
        const bool onpath = j == pj;
        NO[c] = onpath ? O_ONE : 0ull;
        Wv[c] = 0.0;
        PR[c] = rawv(j) / tot;
#undef rawv
        RW[c] = rew;
        PA[c] = node_l;
        // the on-path child expanded at the next level gets its fc/meta from lane l+1
        if (!onpath || last) {
          uint32_t m = (uint32_t)len | ((uint32_t)j << SH_REF) | (term ? M_TERM : 0u);
          if (onpath && forced) m |= M_TERM | M_FORCED;
          MF[c] = mk_mf(-1, m);
        }
        if (!term) {
          ++live;
          // NE: a new non-terminal leaf, check-relevant and viable (scoring.py:119-175)
          const bool rel = len == 1 ? (strict || rew >= theta1) : rel_d1;
          double bound = rew;
          if (prefix_bound && l > 0) {
            const double pre = scheme == TS_SCHEME_PRODUCT ? agg_l * rew : (rew < agg_l ? rew : agg_l);
            bound = fmin(rew, pre);
          }
          if (rel && !(bound < tau)) ++ne_cnt;
        }
      }
      // the expanded node (path node l) stops being a leaf
      if (l >= 1) {
        const double bound = prefix_bound ? fmin(rew_l, agg_l) : rew_l;
        if (rel_d1 && !(bound < tau)) --ne_cnt;
      }
      const uint32_t m = l == d0 ? leaf_meta : ((uint32_t)l | ((uint32_t)upj << SH_REF));
      meta_l = m | M_KIDS | ((uint32_t)live << SH_NEXP);
      MF[node_l] = mk_mf(fcl, meta_l);
    }
    // refresh the path meta registers (lane l-1 holds path node l)
    {
      const uint32_t dn = __shfl_down_sync(FULL, meta_l, 1);
      const bool dn_act = (lane + 1) >= d0 && (lane + 1) < d0 + nlev;
      if (dn_act) pmeta = dn;
      if (d0 == 0 && nlev > 0) root_meta = __shfl_sync(FULL, meta_l, 0);
      if (forced && lane == dend - 1) pmeta |= M_TERM | M_FORCED;
    }
    if (forced && nlev == 0) {
      // the selected leaf itself hit the depth cap (d0 >= 1 since depth_cap >= 1)
      const uint32_t m = __shfl_sync(FULL, pmeta, dend - 1);
      const int lid = __shfl_sync(FULL, pnode, dend - 1);
      if (lane == 0) ME[2 * lid] = m;
    }
    viable += (int)__reduce_add_sync(FULL, (unsigned)(ne_cnt + 64)) - 64 * 32;
    if (forced) {
      // NE: the force-terminated leaf leaves the leaf set
      const bool rel = strict || d1r >= theta1;
      const double bound = prefix_bound ? fmin(nrew, PROD ? agg.a : agg.value(scheme)) : nrew;
      if (rel && !(bound < tau)) --viable;
    }
    created += (unsigned long long)nlev * width;
    if (nlev > 0 && d0 == 0) rfc = fc0;
    __syncwarp();
    // subtree exhaustion: forced node, or a last expansion with no live child
    int dead_from = -1;
    if (forced) dead_from = dend;
    else if (nlev > 0 && __shfl_sync(FULL, live, dend - 1) == 0) dead_from = dend - 1;
    if (dead_from >= 0) {
      for (int i = dead_from - 1; i >= 0; --i) {
        uint32_t m = i == 0 ? root_meta : __shfl_sync(FULL, pmeta, i - 1);
        const int pid = i == 0 ? 0 : __shfl_sync(FULL, pnode, i - 1);
        m -= NEXP_ONE;
        if (lane == 0) ME[2 * pid] = m;
        if (i == 0) root_meta = m;
        else if (lane == i - 1) pmeta = m;
        if (meta_nexp(m) > 0) break;
      }
    }
    // in-flight registration of root..leaf (tree.py:282-283); the simulated
    // path was written with O = 1 above (tree.py:347-348)
    rno += O_ONE;
    if (lane < d0) pno += O_ONE;
    if (multi) {
      if (lane < d0) NO[pnode] = pno;
      if (lane == 0) NO[0] = rno;
      SPs[(size_t)nl * 32 + lane] = pnode;
      if (lane == 0) { SSs[nl] = pscore; SLs[nl] = plen; }
    }
    ++nl;
    __syncwarp();
  }
  {
    long long t = tok_acc;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    tok_acc = t;
  }

  // --- finish_rollout → backpropagate (tree.py:352-371) → decide_exit in
  //     launch order; cancel_inflight for the rest on exit ---
  launched += nl;
  const bool exhausted = decision == -1;
  if (exhausted) decision = TS_EXIT_NONE;
  unsigned long long done = 0;
  auto decide = [&](bool exh) -> int {
    if (cf.positive_exit && best_term >= 0 && best >= cf.positive_exit_threshold) return TS_EXIT_POSITIVE;
    if (cf.negative_exit && (root_meta & M_KIDS) && viable == 0) return TS_EXIT_NEGATIVE;
    if (exh || completed >= budget) return TS_EXIT_BUDGET;
    return TS_EXIT_NONE;
  };
  if (status == TS_OK && exhausted) decision = decide(true);
  for (int r = 0; r < nl && status == TS_OK; ++r) {
    int pn, len;
    double sc;
    bool bad = false;
    if (completed >= budget) { status = TS_ACCOUNTING; break; }
    if (multi) {
      len = SLs[r];
      sc = SSs[r];
      pn = lane < len ? SPs[(size_t)r * 32 + lane] : -1;
      if (lane < len) {
        const uint64_t x = NO[pn];
        if ((x >> 32) < 1) bad = true;
        const uint64_t nx = x + 1 - O_ONE;
        const double w2 = Wv[pn] + sc;
        NO[pn] = nx;
        Wv[pn] = w2;
        QQ[pn] = w2 / (double)(uint32_t)nx;
      }
    } else {
      // single rollout: the path's N|O and W are still the registers' values
      len = plen;
      sc = pscore;
      pn = pnode;
      if (lane < len) {
        if ((pno >> 32) < 1) bad = true;
        const uint64_t nx = pno + 1 - O_ONE;
        const double w2 = pW + sc;
        NO[pn] = nx;
        Wv[pn] = w2;
        QQ[pn] = w2 / (double)(uint32_t)nx;
      }
    }
    if ((rno >> 32) < 1) bad = true;
    rno = rno + 1 - O_ONE;
    rW += sc;
    if (lane == 0) { NO[0] = rno; Wv[0] = rW; QQ[0] = rW / (double)(uint32_t)rno; }
    if (__any_sync(FULL, bad)) { status = TS_ACCOUNTING; break; }
    __syncwarp();
    ++completed;
    ++done;
    pathn += len + 1;
    if (best_term < 0 || sc > best) {
      best = sc;
      best_term = __shfl_sync(FULL, pn, len - 1);
    }
    decision = decide(false);
    if (decision != TS_EXIT_NONE) {
      for (int r2 = r + 1; r2 < nl; ++r2) {
        const int len2 = SLs[r2];
        const int pn2 = lane < len2 ? SPs[(size_t)r2 * 32 + lane] : -1;
        bool bad2 = lane < len2 && (NO[pn2] >> 32) < 1;
        if ((rno >> 32) < 1) bad2 = true;
        if (__any_sync(FULL, bad2)) { status = TS_ACCOUNTING; break; }
        if (lane < len2) NO[pn2] -= O_ONE;
        rno -= O_ONE;
        if (lane == 0) NO[0] = rno;
        __syncwarp();
        ++cancelled;
        pathn += len2 + 1;
      }
      break;
    }
  }

  if (lane == 0) {
    S->completed = completed;
    S->nodes = nnodes;
    S->viable = viable;
    S->best_term = best_term;
    S->best = best;
    S->tokens += tok_acc;
    ws.tokens += (unsigned long long)tok_acc;  // Counters::tokens once per warp at the kernel's end
    S->launched = launched;
    S->cancelled = cancelled;
    // on_rollout_complete (scheduler.py:217-233): refresh Job.best_score
    double jb = S->job_best;
    if (best_term >= 0 && best > jb) S->job_best = jb = best;
    write_next_record(v, s, step, status != TS_OK || decision != TS_EXIT_NONE, completed, jb);
    if (status != TS_OK || decision != TS_EXIT_NONE) {
      S->state = ST_FINISHED;
      S->exit_kind = status == TS_OK ? decision : TS_EXIT_NONE;
      S->status = status;
      S->exit_step = step;
      S->t_exit = globaltimer();
      atomicAdd((unsigned long long*)&v.ctr->running, (unsigned long long)-1ll);
      atomicAdd((unsigned long long*)&v.ctr->finished, 1ull);
      atomicMax(&v.ctr->last_exit_step, (long long)step);
    }
  }
  ws.rollouts += done;
  ws.launched += nl;
  ws.nodes += created;
  ws.scored += scored;
  ws.levels += levels;
  ws.path_nodes += pathn;
}



// Free-running waves (k_sched decides): items (search, chunk of FREE_C
// rollouts) in chunk-major order; a warp runs an item's rollouts as single-
// rollout waves at steps t0 + r after the search's previous chunk is done
// (acquire), then publishes its own (release).  Items of one chunk level
// outnumber the resident warps, so a predecessor has normally finished long
// before its successor is taken.
#ifndef TS_FREE_C
#define TS_FREE_C 4
#endif
constexpr int FREE_C = TS_FREE_C;
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int x;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
  return x;
}
__device__ __forceinline__ void st_release_gpu(int* p, int x) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
template <int NSLOT, int WT, bool SINGLE, bool PROD = false>
__device__ void free_run_waves(const View& v, WaveStats& ws, double* s_raw, double* s_rew) {
  const int lane = threadIdx.x & 31;
  Counters* c = v.ctr;
  const int nw = c->work_count, t0 = c->free_t0, rem = c->free_rem;
  const int nch = (rem + FREE_C - 1) / FREE_C;
  const unsigned long long total = (unsigned long long)nw * (unsigned long long)nch;
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(&c->free_next, 1ull);
    it = __shfl_sync(FULL, it, 0);
    if (it >= total) break;
    const int k = (int)(it / (unsigned long long)nw), s = v.work[it % (unsigned long long)nw];
    if (lane == 0)
      while (ld_acquire_gpu(v.fdone + s) < k) __nanosleep(64);
    __syncwarp();
    const int r1 = min(rem, (k + 1) * FREE_C);
    for (int r = k * FREE_C; r < r1; ++r) {
      if (v.st[s].state != ST_RUNNING) break;
      search_wave<NSLOT, WT, SINGLE, PROD>(v, s, t0 + r, ws, s_raw, s_rew);
      __syncwarp();
    }
    if (lane == 0) st_release_gpu(v.fdone + s, k + 1);
  }
}

// PROD: the product aggregation scheme fixed at compile time (the default
// ScoringConfig; no Neumaier compensation state along the path)
template <int NSLOT, int WT, bool PROD>
#ifndef TS_WAVE_MINB
#define TS_WAVE_MINB 4  // resident CTAs of 4 warps per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(WAVE_THREADS, TS_WAVE_MINB) k_wave(View v, int step) {
  constexpr int WS = WT ? WT : TS_MAX_WIDTH;
  extern __shared__ double wsm[];  // per warp: raw priors and rewards, [32 depths][WS]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* s_raw = wsm + (size_t)warp * 2 * 32 * WS;
  double* s_rew = s_raw + 32 * WS;
  WaveStats ws = {0, 0, 0, 0, 0, 0, 0};
#ifdef TS_SCHED_PROF
  if (threadIdx.x == 0) atomicMin(&v.ctr->prof[21], globaltimer());
#endif
  if (step < 0 && v.free_ok && v.ctr->free_run) {
    if (!v.free_kernel) free_run_waves<NSLOT, WT, false, PROD>(v, ws, s_raw, s_rew);
  } else {
  const int count = v.ctr->work_count;
  if (step < 0) step = v.ctr->cur_step;
  // the first item of every warp is its global warp index (no burst of
  // same-address atomics at launch); later items come from the shared counter
  const int nwarps = gridDim.x * WAVE_WARPS;
  int item = blockIdx.x * WAVE_WARPS + warp;
  while (item < count) {
    search_wave<NSLOT, WT, false, PROD>(v, v.work[item], step, ws, s_raw, s_rew);
    if (lane == 0) item = nwarps + atomicAdd(&v.ctr->work_next, 1);
    item = __shfl_sync(FULL, item, 0);
  }
  }
#ifdef TS_SCHED_PROF
  if (lane == 0) atomicMax(&v.ctr->prof[20], globaltimer());
#endif
  if (lane == 0 && ws.launched) {
    atomicAdd(&v.ctr->rollouts, ws.rollouts);
    atomicAdd(&v.ctr->launched, ws.launched);
    atomicAdd(&v.ctr->nodes, ws.nodes);
    atomicAdd(&v.ctr->scored, ws.scored);
    atomicAdd(&v.ctr->levels, ws.levels);
    atomicAdd(&v.ctr->path_nodes, ws.path_nodes);
    if (ws.tokens) atomicAdd(&v.ctr->tokens, ws.tokens);
  }
}

// Free-running waves get their own kernel: every wave is one rollout, so the
// multi-rollout bookkeeping is compiled out (search_wave<..., SINGLE>) and 5
// CTAs of 4 warps fit per SM (96 registers) where k_wave keeps 4.
#ifndef TS_FREE_MINB
#define TS_FREE_MINB 5
#endif
template <int NSLOT, int WT, bool PROD>
__global__ void __launch_bounds__(WAVE_THREADS, TS_FREE_MINB) k_wave_free(View v) {
  constexpr int WS = WT ? WT : TS_MAX_WIDTH;
  extern __shared__ double wsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!(v.free_ok && v.ctr->free_run)) return;
  double* s_raw = wsm + (size_t)warp * 2 * 32 * WS;
  double* s_rew = s_raw + 32 * WS;
  WaveStats ws = {0, 0, 0, 0, 0, 0, 0};
  free_run_waves<NSLOT, WT, true, PROD>(v, ws, s_raw, s_rew);
  if (lane == 0 && ws.launched) {
    atomicAdd(&v.ctr->rollouts, ws.rollouts);
    atomicAdd(&v.ctr->launched, ws.launched);
    atomicAdd(&v.ctr->nodes, ws.nodes);
    atomicAdd(&v.ctr->scored, ws.scored);
    atomicAdd(&v.ctr->levels, ws.levels);
    atomicAdd(&v.ctr->path_nodes, ws.path_nodes);
    if (ws.tokens) atomicAdd(&v.ctr->tokens, ws.tokens);
  }
}
// [scheme is product][nslot 1/2/4][width 2/4/8/runtime]
#define TS_KWF(P, A)                                                                                   \
  {(const void*)k_wave_free<A, 2, P>, (const void*)k_wave_free<A, 4, P>, (const void*)k_wave_free<A, 8, P>, \
   (const void*)k_wave_free<A, 0, P>}
static const void* kWaveFree[2][3][4] = {
    {TS_KWF(false, 1), TS_KWF(false, 2), TS_KWF(false, 4)},
    {TS_KWF(true, 1), TS_KWF(true, 2), TS_KWF(true, 4)},
};
#undef TS_KWF

// kernel table: [nslot 1/2/4][width 2/4/8/runtime]
typedef void (*wave_kernel_t)(View, int);
__device__ __host__ inline int wkind_of_width(int w) { return w == 2 ? 0 : w == 4 ? 1 : w == 8 ? 2 : 3; }
static const wave_kernel_t kWave[2][3][4] = {
    {{k_wave<1, 2, false>, k_wave<1, 4, false>, k_wave<1, 8, false>, k_wave<1, 0, false>},
     {k_wave<2, 2, false>, k_wave<2, 4, false>, k_wave<2, 8, false>, k_wave<2, 0, false>},
     {k_wave<4, 2, false>, k_wave<4, 4, false>, k_wave<4, 8, false>, k_wave<4, 0, false>}},
    {{k_wave<1, 2, true>, k_wave<1, 4, true>, k_wave<1, 8, true>, k_wave<1, 0, true>},
     {k_wave<2, 2, true>, k_wave<2, 4, true>, k_wave<2, 8, true>, k_wave<2, 0, true>},
     {k_wave<4, 2, true>, k_wave<4, 4, true>, k_wave<4, 8, true>, k_wave<4, 0, true>}},
};

// ---- pipelined CTA mode for searches with many rollouts in one wave ----------
//
// A wave's rollouts are sequential by definition: rollout k+1 selects against
// the in-flight registrations (and expansions) of rollouts <= k.  But a
// simulation only depends on its own selected leaf and path, and a later
// selection only needs it once it reaches that leaf.  So one warp selects and
// registers rollout after rollout while HEAVY_SIM warps simulate them, and the
// simulators commit in rollout order (node ids in creation order, records,
// subtree exhaustion, negative-exit counts).  Two waits keep this exactly the
// sequential semantics:
//  * the selector that arrives at a leaf whose expansion is not committed yet
//    waits for that commit and then keeps descending;
//  * a job whose exhaustion can propagate into pre-existing nodes ("risky":
//    leaf depth >= min(base_depth, depth_cap) - 1, or width 1 — below that a
//    fresh expansion always leaves a live child) is committed before the next
//    selection starts.
// 8 warps: warp 0 selects; warp 4, which shares warp 0's SM sub-partition
// (scheduler = warp id % 4), stays idle so the latency-bound selection chain
// never competes for issue slots; the other 6 warps simulate.
#ifndef TS_HEAVY_WARPS
#define TS_HEAVY_WARPS 8
#endif
#ifndef TS_HEAVY_MINB
#define TS_HEAVY_MINB 2
#endif
constexpr int HEAVY_WARPS = TS_HEAVY_WARPS;
constexpr int HEAVY_SIM = HEAVY_WARPS - 2;
constexpr int HEAVY_THREADS = 32 * HEAVY_WARPS;
__device__ __forceinline__ int heavy_sim_of_warp(int w) { return w < 4 ? w - 1 : w - 2; }
constexpr int HEAVY_RING = 16;

struct HeavyJob {
  int leaf, d0, risky, golden;
  uint32_t leaf_meta, _pad;
  double nrew, agg_a, agg_c, d1r;
  int agg_n, _pad2;
  int pnode[32];   // path node l+1 for l < d0 (the leaf is pnode[d0-1])
  int pj[32];      // child index chosen at depth l
};

constexpr int HEAVY_ZERO_O_MAX = 1 << 16;  // trees up to this size clear O with the whole CTA at an exit

struct HeavyCtl {
  volatile int issued, committed, done, status;
  int zero_o;  // set by heavy_finish: clear O of every node of the search (exit with cancellations)
  volatile int nnodes, viable;
  unsigned long long created, tokens;
  // the root's word (meta | first child << 32) after the commits so far: the
  // committing simulator updates it with MF[0], so the selector refreshes its
  // copy from shared memory instead of global memory
  volatile unsigned long long root_mf;
};

// CTA-scope acquire load / release store on shared-memory counters
__device__ __forceinline__ int ld_acquire_cta(const volatile int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared((const void*)p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(volatile int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared((const void*)p)), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_ge(volatile int* p, int v) {
  while (ld_acquire_cta(p) < v) __nanosleep(32);
}

#ifdef TS_HEAVY_PROF
#define HPROF_T0(x) long long x = clock64()
#define HPROF_ACC(acc, t0) acc += clock64() - (t0)
#else
#define HPROF_T0(x) (void)0
#define HPROF_ACC(acc, t0) (void)0
#endif

// If `node` is the selected leaf of a job that is issued but not committed,
// wait for that commit (acquire) and return true: the caller must reload the
// node's meta and first child.  Jobs [committed, issued) are checked lane-parallel.
// Lane l holds the leaf of job (issued - 1 - l) for the last 32 jobs (lleaf),
// so the check is a compare and a ballot.
__device__ __forceinline__ bool heavy_wait_inflight(HeavyCtl* ctl, int lleaf, int c0, int issued, int node) {
  const int lane = threadIdx.x & 31;
  const int job = issued - 1 - lane;
  const bool hit = job >= c0 && lleaf == node;
  const unsigned hm = __ballot_sync(FULL, hit);
  if (!hm) return false;
  spin_until_ge(&ctl->committed, issued - __ffs(hm) + 1);  // the most recent matching job
  return true;
}

// A reload that must stay behind its (warp-uniform) condition: a plain load
// would be if-converted into an unconditional load plus a select, putting a
// memory round trip on the selection chain of every level.
__device__ __forceinline__ uint64_t reload_u64(const uint64_t* p) { return *(const volatile uint64_t*)p; }

// sqrt(k) for k < SQRT_TAB in shared memory (IEEE sqrt is exact-rounded).
// Every count the selector takes a root of is N + O of one node, and
// N + O <= completed + in flight <= rollout_budget, so with the pipelined mode
// enabled only for budgets below SQRT_TAB (ts_load) the lookup needs no range
// check: a branch here stalled the selection chain on every scored node.
constexpr int SQRT_TAB = 2048;
__device__ __forceinline__ double isqrt_tab(const double* sqt, long long n) { return sqt[(int)n]; }
// the same lookup through a 32-bit shared-window address computed once per
// search: a generic pointer costs a window conversion (S2UR of the CTA id) at
// every use on the selection chain
__device__ __forceinline__ double isqrt_s(uint32_t sqs, uint32_t n) {
  double r;
  asm("ld.shared.f64 %0, [%1];" : "=d"(r) : "r"(sqs + 8u * n));
  return r;
}

template <int NSLOT, int WT, bool PROD>
__device__ __forceinline__ void heavy_select(const View& v, int s, HeavyCtl* ctl, HeavyJob* ring, const double* sqt, int count,
                             WaveStats& ws, uint64_t& rno_out, double& rW_out, int& decision_out) {
  const int lane = threadIdx.x & 31;
  const ts_config& cf = v.cfg;
  const ts_problem* pb = v.prob + s;
  const size_t base = (size_t)s * (size_t)v.cap;
  uint64_t* NO = v.no + base;
  double* Wv = v.W + base;
  double* PR = v.prior + base;
  double* RW = v.reward + base;
  uint64_t* MF = v.mf + base;
  const double* QQ = v.Q + base;
  const int bdepth = pb->base_depth;
  const int glen = pb->golden_len;
  const int width = WT;
  const int scheme = cf.scheme;
  const double c_puct = cf.c_puct;
  const int gstep = lane < glen ? (int)pb->golden_path[lane] : -1;
  const int risky_depth = min(bdepth, cf.depth_cap) - 1;
  uint64_t rno = NO[0];
  const double rW = Wv[0];
  const long long rN = (long long)(uint32_t)rno;
  const double rq = rN == 0 ? 0.5 : QQ[0];  // the root's mean (constant during a wave)
  const uint32_t sqs = (uint32_t)__cvta_generic_to_shared(sqt);
  uint64_t rmf = 0;  // the root's word, refreshed from ctl->root_mf per rollout
  int decision = TS_EXIT_NONE;
  int last_risky = -1;
  int lleaf = -1;  // lane l: leaf of job k-1-l
  int k = 0;
  unsigned long long scored = 0, levels = 0;
#ifdef TS_HEAVY_PROF
  long long p_total = 0, p_risky = 0, p_infl = 0, p_ring = 0, p_load = 0, p_math = 0;
  long long q_l1 = 0, q_l2 = 0, q_sc = 0, q_t1 = 0, q_l2t = 0, q_rounds = 0, q_math = 0;
  long long q_root_l1 = 0, q_root_l2 = 0, q_root_rounds = 0;
  HPROF_T0(p_start);
#endif
  for (; k < count; ++k) {
    HPROF_T0(t_r);
    if (last_risky >= 0) {
      spin_until_ge(&ctl->committed, last_risky + 1);
      last_risky = -1;
    }
    HPROF_ACC(p_risky, t_r);
    // jobs < cs are committed and visible from here on; jobs [cs, k) may commit
    // while this selection reads the tree (they are checked at every node entered)
    HPROF_T0(t_pro);
    const int cs = ld_acquire_cta(&ctl->committed);
    // the root's word changes only at the commit of a job that had the root as
    // its leaf (waited for below) or was risky (waited for above); the
    // committing simulator keeps it in shared memory.  The three shared loads
    // are issued back to back.
    rmf = ctl->root_mf;
    if (ctl->status != TS_OK) break;
    if (heavy_wait_inflight(ctl, lleaf, cs, k, 0)) rmf = ctl->root_mf;
    uint32_t nmeta = (uint32_t)rmf;
    if (!meta_expandable(nmeta)) {  // NoExpandableLeafError (tree.py:273-274)
      if (k == 0) decision = -1;
      break;
    }
    HPROF_ACC(p_load, t_pro);
    HPROF_T0(t_desc);
    int node = 0, depth = 0, nfc = (int)(rmf >> 32);
    // the current node's mean W/N (0.5 unvisited) and sqrt(N+O), ready before its children are scored
    double pq = rq, psq = isqrt_s(sqs, (uint32_t)(rN + (long long)(rno >> 32)));
    int pnode = -1, pj = 0;
    uint64_t pno = 0;
    double nrew = 1.0;
    Agg agg;
    agg.init();
    double d1r = 1.0;
    int status = TS_OK;
    // per-lane record of a scored node; `take` moves the descent into the node scored by lane `src`
    auto take = [&](int src, int child_index, int fc_parent, uint64_t xno, uint64_t xmf, double xr, double xnq,
                    double xnsq) {
      node = fc_parent + child_index;
      ++depth;
      const uint64_t wmf = __shfl_sync(FULL, xmf, src);
      nmeta = (uint32_t)wmf;
      nfc = (int)(wmf >> 32);
      nrew = __shfl_sync(FULL, xr, src);
      const uint64_t nno = __shfl_sync(FULL, xno, src);
      pq = __shfl_sync(FULL, xnq, src);
      psq = __shfl_sync(FULL, xnsq, src);
      if constexpr (PROD) {
        agg.a = agg.a * nrew;
        ++agg.n;
      } else {
        agg.add(nrew, scheme);
      }
      if (depth == 1) d1r = nrew;
      if (lane == depth - 1) { pnode = node; pno = nno; pj = child_index; }
      // entering a leaf whose expansion may be in flight: its word and children
      // are only valid after that job's commit (acquired in the wait)
      const bool waited = heavy_wait_inflight(ctl, lleaf, cs, k, node);
      if (waited) {
        const uint64_t x = reload_u64(MF + node);
        nmeta = (uint32_t)x;
        nfc = (int)(x >> 32);
      }
      return waited;
    };
    if constexpr (WT * (WT + 1) <= 32) {
      // two levels per round: lanes [0, W) score the children, lanes
      // [W, W + W*W) the children of every child; the second argmax runs in the
      // group of the child the first one picked
      const bool l1 = lane < WT;
      const bool l2lane = lane >= WT && lane < WT + WT * WT;
      const int gj = l2lane ? (lane - WT) / WT : 0, gi = l2lane ? (lane - WT) % WT : 0;
      while (nmeta & M_KIDS) {
        const int fc = nfc;
#ifdef TS_HEAVY_PROF
        long long t_a = clock64();
#endif
        // branch-free: every lane loads a real node (the other lanes the first
        // child's record, the same lines), so no divergent branch sits on the chain
        const int c1 = fc + (l1 ? lane : 0);
        uint64_t xno = NO[c1], xmf = MF[c1];
        double xq = QQ[c1], xp = PR[c1], xr = RW[c1];
        // the grandchild lanes read their parent child's record
        const int src = l1 ? lane : gj;
#ifdef TS_HEAVY_PROF
        {
          unsigned long long w_;
          asm volatile("xor.b64 %0, %1, %2;\n\txor.b64 %0, %0, %3;" : "=l"(w_) : "l"(xmf), "l"(xno), "l"(__double_as_longlong(xq + xp + xr)) : "memory");
          if (lane == 0) {
            const long long dt_ = clock64() - t_a + (w_ == 12345 ? 1 : 0);
            q_l1 += dt_;
            if (depth == 0) q_root_l1 += dt_;
          }
        }
        long long t_b = clock64();
#endif
        const uint64_t gpmf = __shfl_sync(FULL, xmf, src);
        const uint64_t gpno = __shfl_sync(FULL, xno, src);
        const double gpq = __shfl_sync(FULL, xq, src);
        const bool l2 = l2lane & (((uint32_t)gpmf & M_KIDS) != 0);
        {
          const int c2 = l2 ? (int)(gpmf >> 32) + gi : c1;
          const uint64_t yno = NO[c2], ymf = MF[c2];
          const double yq = QQ[c2], yp = PR[c2], yr = RW[c2];
          xno = l2 ? yno : xno;
          xmf = l2 ? ymf : xmf;
          xq = l2 ? yq : xq;
          xp = l2 ? yp : xp;
          xr = l2 ? yr : xr;
        }
        // the scored node's parent terms: the current node for l1, the child for l2
#ifdef TS_HEAVY_PROF
        {
          unsigned long long w_;
          asm volatile("xor.b64 %0, %1, %2;\n\txor.b64 %0, %0, %3;" : "=l"(w_) : "l"(xmf), "l"(xno), "l"(__double_as_longlong(xq + xp + xr)) : "memory");
          if (lane == 0) {
            const long long dt_ = clock64() - t_b + (w_ == 12345 ? 1 : 0);
            q_l2 += dt_;
            if (depth == 0) { q_root_l2 += dt_; ++q_root_rounds; }
          }
        }
        long long t_c = clock64();
#endif
        const unsigned gN = (uint32_t)gpno, gO = (uint32_t)(gpno >> 32);
        const double ppq = l1 ? pq : (gN == 0 ? 0.5 : gpq);
        const double gsq = isqrt_s(sqs, gN + gO);
        const double ppsq = l1 ? psq : gsq;
        const bool valid = (l1 | l2) & meta_expandable((uint32_t)xmf);
        const unsigned xN = (uint32_t)xno, xO = (uint32_t)(xno >> 32);
        const double xnq = xN == 0 ? 0.5 : xq;
        const double xnsq = isqrt_s(sqs, xN + xO);
        // _child_q (tree.py:235-239); wu_puct_score (tree.py:232); computed on
        // every lane (finite inputs everywhere) and masked afterwards
        const double q = xN == 0 ? ppq : xq;
        const double u = c_puct * xp * ppsq / (double)(1u + xN + xO);
        const double sc = valid ? q + u : -INFINITY;
        // non-short-circuit: four compares and no branch on the selection chain
        const bool bad = valid & (!(q >= 0.0) | !(q <= 1.0) | !(xp >= 0.0) | !(xp <= 1.0));
#ifdef TS_HEAVY_PROF
        {
          unsigned long long w_;
          asm volatile("xor.b64 %0, %1, %2;" : "=l"(w_) : "l"(__double_as_longlong(sc)), "l"(__double_as_longlong(xnsq + ppsq)) : "memory");
          if (lane == 0) q_math += clock64() - t_c + (w_ == 12345 ? 1 : 0);
        }
        t_c = clock64();
#endif
        // level 1; one ballot of each flag per round, the levels mask their lanes
        constexpr unsigned L1M = (1u << WT) - 1u;
        const unsigned vball = __ballot_sync(FULL, valid), bball = __ballot_sync(FULL, bad);
        const unsigned vb1 = vball & L1M;
        if ((bball & L1M) | (vb1 == 0u)) { status = (bball & L1M) ? TS_INVALID_ARGUMENT : TS_EXHAUSTED; break; }
        scored += __popc(vb1);
        ++levels;
        // every group's level-2 argmax, issued with level 1's: a butterfly over
        // the W lanes of each group (aligned), keys as in warp_argmax_nonneg,
        // ties to the lower lane (the first child); read for group j1 below
        int g2 = lane;
        {
          const uint64_t b = (uint64_t)__double_as_longlong(sc);
          uint64_t key = valid ? ((b >> 63) ? ~b : (b | (1ull << 63))) : 0ull;
#pragma unroll
          for (int o = 1; o < WT; o <<= 1) {
            const uint64_t pk = __shfl_xor_sync(FULL, key, o);
            const int pl = __shfl_xor_sync(FULL, g2, o);
            const bool tk = pk > key || (pk == key && pl < g2);
            key = tk ? pk : key;
            g2 = tk ? pl : g2;
          }
        }
        const int j1 = warp_argmax_nonneg(sc, valid && l1);
        const int s2 = __shfl_sync(FULL, g2, WT + j1 * WT);
#ifdef TS_HEAVY_PROF
        if (lane == 0) q_sc += clock64() - t_c;
        long long t_d = clock64();
#endif
        const bool stale1 = take(j1, j1, fc, xno, xmf, xr, xnq, xnsq);
#ifdef TS_HEAVY_PROF
        if (lane == 0) q_t1 += clock64() - t_d + (nfc == -7 ? 1 : 0);
        long long t_e = clock64();
        ++q_rounds;
#endif
        if (stale1) continue;  // the group is stale after a commit
        if (!(nmeta & M_KIDS)) break;
        // level 2, within the group of child j1
        const unsigned gm = L1M << (WT + j1 * WT);
        const unsigned vb2 = vball & gm;
        if ((bball & gm) | (vb2 == 0u)) { status = (bball & gm) ? TS_INVALID_ARGUMENT : TS_EXHAUSTED; break; }
        scored += __popc(vb2);
        ++levels;
        take(s2, (s2 - WT) % WT, nfc, xno, xmf, xr, xnq, xnsq);
#ifdef TS_HEAVY_PROF
        if (lane == 0) q_l2t += clock64() - t_e + (nfc == -7 ? 1 : 0);
#endif
      }
    } else {
    while (nmeta & M_KIDS) {
      const int fc = nfc;
      bool valid = lane < width;
      double sc = -INFINITY, cr = 0.0, nq = 0.5, nsq = 0.0;
      uint64_t cno = 0, cmf = 0;
#ifdef TS_HEAVY_PROF
      long long t_l0 = clock64();
#endif
      if (valid) {
        const int c = fc + lane;
        cno = NO[c];
        const double cq = QQ[c];
        const double cp = PR[c];
        cmf = MF[c];
        cr = RW[c];
        valid = meta_expandable((uint32_t)cmf);
#ifdef TS_HEAVY_PROF
        if (lane == 0) p_load += clock64() - t_l0 + (cq == -1.0 ? 1 : 0) + (cp == -1.0 ? 1 : 0) + (cr == -1.0 ? 1 : 0);
#endif
        // branch-free, so all five loads issue together; masked by `valid`
        const unsigned cN = (uint32_t)cno, cO = (uint32_t)(cno >> 32);
        nq = cN == 0 ? 0.5 : cq;  // this child's mean, the next level's parent term
        nsq = isqrt_tab(sqt, (long long)cN + cO);
        // _child_q (tree.py:235-239); wu_puct_score (tree.py:232)
        const double q = cN == 0 ? pq : cq;
        const double u = c_puct * cp * psq / (double)(1u + cN + cO);
        if (valid && (!(q >= 0.0 && q <= 1.0) || !(cp >= 0.0 && cp <= 1.0))) status = TS_INVALID_ARGUMENT;
        sc = valid ? q + u : -INFINITY;
      }
      const unsigned vb = __ballot_sync(FULL, valid);
      if (__any_sync(FULL, status != TS_OK)) { status = TS_INVALID_ARGUMENT; break; }
      if (!vb) { status = TS_EXHAUSTED; break; }
      scored += __popc(vb);
      ++levels;
      const int j = warp_argmax_nonneg(sc, valid);
#ifdef TS_HEAVY_PROF
      if (lane == 0) p_math += clock64() - t_l0;
#endif
      node = fc + j;
      ++depth;
      const uint64_t wmf = __shfl_sync(FULL, cmf, j);
      nmeta = (uint32_t)wmf;
      nfc = (int)(wmf >> 32);
      nrew = __shfl_sync(FULL, cr, j);
      const uint64_t nno = __shfl_sync(FULL, cno, j);
      pq = __shfl_sync(FULL, nq, j);
      psq = __shfl_sync(FULL, nsq, j);
      if constexpr (PROD) {
        agg.a = agg.a * nrew;
        ++agg.n;
      } else {
        agg.add(nrew, scheme);
      }
      if (depth == 1) d1r = nrew;
      if (lane == depth - 1) { pnode = node; pno = nno; pj = j; }
      // entering a leaf whose expansion may be in flight: its word and children
      // are only valid after that job's commit (acquired in the wait)
      HPROF_T0(t_i);
      const bool waited = heavy_wait_inflight(ctl, lleaf, cs, k, node);
      HPROF_ACC(p_infl, t_i);
      if (waited) {
        const uint64_t x = reload_u64(MF + node);
        nmeta = (uint32_t)x;
        nfc = (int)(x >> 32);
      }
    }
    }
    HPROF_ACC(p_math, t_desc);
    HPROF_T0(t_epi);
    if (status != TS_OK) {
      if (lane == 0) atomicCAS((int*)&ctl->status, TS_OK, status);
      break;
    }
    // hand the rollout to its simulator
    HPROF_T0(t_g);
    if (k - cs >= HEAVY_RING && k - ctl->committed >= HEAVY_RING) spin_until_ge(&ctl->committed, k - HEAVY_RING + 1);
    HPROF_ACC(p_ring, t_g);
#ifdef TS_HEAVY_PROF
    const long long e0 = clock64();
#endif
    // on the golden path iff every level's child is the golden step (lane
    // l holds the child index chosen at depth l + 1); checked once per rollout
    const bool on_golden = __all_sync(FULL, lane >= depth || pj == gstep);
    const bool golden = glen >= 0 && depth <= glen && on_golden;
    HeavyJob& jb = ring[k % HEAVY_RING];
    jb.pnode[lane] = pnode;
    jb.pj[lane] = pj;
    if (lane == 0) {
      jb.leaf = node;
      jb.d0 = depth;
      jb.risky = (width == 1 || depth >= risky_depth || v.heavy_sync) ? 1 : 0;
      jb.golden = golden ? 1 : 0;
      jb.leaf_meta = nmeta;
      jb.nrew = nrew;
      jb.agg_a = agg.a;
      jb.agg_c = agg.c;
      jb.agg_n = agg.n;
      jb.d1r = d1r;
    }
    __syncwarp();
#ifdef TS_HEAVY_PROF
    const long long e1 = clock64();
#endif
    if (lane == 0) st_release_cta(&ctl->issued, k + 1);
#ifdef TS_HEAVY_PROF
    const long long e2 = clock64();
#endif
    if (width == 1 || depth >= risky_depth || v.heavy_sync) last_risky = k;
    // in-flight registration of root..leaf (tree.py:282-283); only this warp
    // reads N|O of pre-existing nodes during the wave
    rno += O_ONE;
    if (lane < depth) NO[pnode] = pno + O_ONE;
    if (lane == 0) NO[0] = rno;
    lleaf = __shfl_up_sync(FULL, lleaf, 1);
    if (lane == 0) lleaf = node;
    __syncwarp();
#ifdef TS_HEAVY_PROF
    if (lane == 0) {
      const long long e3 = clock64();
      atomicAdd(&v.ctr->prof[23], (unsigned long long)(e1 - e0));
      atomicAdd(&v.ctr->prof[24], (unsigned long long)(e2 - e1));
      atomicAdd(&v.ctr->prof[25], (unsigned long long)(e3 - e2));
    }
#endif
    HPROF_ACC(p_infl, t_epi);
  }
  if (lane == 0) ctl->done = 1;
#ifdef TS_HEAVY_PROF
  HPROF_ACC(p_total, p_start);
  HPROF_T0(t_end);
#endif
  spin_until_ge(&ctl->committed, k);
#ifdef TS_HEAVY_PROF
  long long p_drain = 0;
  HPROF_ACC(p_drain, t_end);
  if (lane == 0) {
    atomicAdd(&v.ctr->prof[0], (unsigned long long)p_total);
    atomicAdd(&v.ctr->prof[1], (unsigned long long)p_risky);
    atomicAdd(&v.ctr->prof[2], (unsigned long long)p_infl);
    atomicAdd(&v.ctr->prof[3], (unsigned long long)p_ring);
    atomicAdd(&v.ctr->prof[4], (unsigned long long)p_drain);
    atomicMax(&v.ctr->prof[13], (unsigned long long)p_total);
    atomicMax(&v.ctr->prof[14], (unsigned long long)p_drain);
    atomicAdd(&v.ctr->prof[5], (unsigned long long)k);
    atomicAdd(&v.ctr->prof[6], (unsigned long long)p_load);
    atomicAdd(&v.ctr->prof[7], (unsigned long long)p_math);
    atomicAdd(&v.ctr->prof[12], (unsigned long long)levels);
    atomicAdd(&v.ctr->prof[16], (unsigned long long)q_l1);
    atomicAdd(&v.ctr->prof[17], (unsigned long long)q_l2);
    atomicAdd(&v.ctr->prof[18], (unsigned long long)q_sc);
    atomicAdd(&v.ctr->prof[19], (unsigned long long)q_t1);
    atomicAdd(&v.ctr->prof[20], (unsigned long long)q_l2t);
    atomicAdd(&v.ctr->prof[21], (unsigned long long)q_rounds);
    atomicAdd(&v.ctr->prof[22], (unsigned long long)q_math);
    atomicAdd(&v.ctr->prof[26], (unsigned long long)q_root_l1);
    atomicAdd(&v.ctr->prof[27], (unsigned long long)q_root_l2);
    atomicAdd(&v.ctr->prof[28], (unsigned long long)q_root_rounds);
  }
#endif
  rno_out = rno;
  rW_out = rW;
  decision_out = decision;
  ws.scored += scored;
  ws.levels += levels;
}

template <int NSLOT, int WT, bool PROD>
__device__ __forceinline__ void heavy_simulate(const View& v, int s, HeavyCtl* ctl, HeavyJob* ring, double* s_raw, double* s_rew,
                               int si, int nsim) {
  constexpr int WS = WT;
  const int lane = threadIdx.x & 31;
  const ts_config& cf = v.cfg;
  const ts_problem* pb = v.prob + s;
  const size_t base = (size_t)s * (size_t)v.cap;
  uint64_t* NO = v.no + base;
  double* Wv = v.W + base;
  double* PR = v.prior + base;
  double* RW = v.reward + base;
  uint64_t* MF = v.mf + base;
  uint32_t* ME = (uint32_t*)MF;
  int32_t* PA = v.parent + base;
  const uint64_t seed = pb->seed;
  const int bdepth = pb->base_depth;
  const int glen = pb->golden_len;
  const int hidden = pb->hidden_until_depth;
  const bool has_shared = pb->has_shared != 0;
  const double off_lo = pb->off_lo, off_hi = pb->off_hi;
  const double sh_lo = pb->shared_lo, sh_hi = pb->shared_hi;
  const int width = WT;
  const int scheme = cf.scheme;
  const bool strict = cf.strict_negative_exit != 0;
  const bool prefix_bound = cf.futility_bound == TS_BOUND_PREFIX_AGGREGATE;
  const double tau = cf.accept_threshold, theta1 = cf.first_step_threshold;
  const int gstep = lane < glen ? (int)pb->golden_path[lane] : -1;
  const double grew = lane < glen ? pb->golden_rewards[lane] : 0.0;
  const int budget = cf.rollout_budget;
  int32_t* SPs = v.sp + (size_t)s * (size_t)budget * 32;
  double* SSs = v.ss + (size_t)s * budget;
  int32_t* SLs = v.sl + (size_t)s * budget;
  uint64_t root_h[NSLOT];
  {
    const uint64_t h0 = sm64(MIX_INIT ^ seed);
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
      uint64_t tag, len;
      slot_header<NSLOT>(lane, k, tag, len);
      root_h[k] = sm64(sm64(h0 ^ tag) ^ len);
    }
  }
  long long tok_acc = 0;
  unsigned long long created = 0;
#ifdef TS_HEAVY_PROF
  long long q_issue = 0, q_comp = 0, q_cwait = 0, q_commit = 0;
#endif
  for (int k = si;; k += nsim) {
    HPROF_T0(t_a);
    while (ld_acquire_cta(&ctl->issued) <= k && !ctl->done) __nanosleep(32);
    HPROF_ACC(q_issue, t_a);
    HPROF_T0(t_b);
    if (ld_acquire_cta(&ctl->issued) <= k) break;
    const HeavyJob& jb = ring[k % HEAVY_RING];
    const int d0 = jb.d0;
    int pnode = jb.pnode[lane], pj = jb.pj[lane];
    uint64_t h[NSLOT];
#pragma unroll
    for (int q = 0; q < NSLOT; ++q) h[q] = root_h[q];
    for (int i = 0; i < d0; ++i) {
      const uint64_t j = (uint64_t)jb.pj[i];
#pragma unroll
      for (int q = 0; q < NSLOT; ++q) h[q] = sm64(h[q] ^ j);
    }
    Agg agg;
    agg.a = jb.agg_a;
    agg.c = jb.agg_c;
    agg.n = jb.agg_n;
    bool golden = jb.golden != 0;
    double d1r = jb.d1r, nrew = jb.nrew;
    uint32_t pmeta = 0, lvl_term = 0;
    double prew = 0.0, pagg = 1.0;
    if (lane == d0 - 1) { pmeta = jb.leaf_meta; prew = jb.nrew; pagg = jb.agg_a; }
    const int leaf = jb.leaf;
    const bool risky = jb.risky != 0;
    int depth = d0, nrel = 0, node = leaf;
    bool forced = false;
    uint64_t snap[NSLOT];
#pragma unroll
    for (int q = 0; q < NSLOT; ++q) snap[q] = 0;
    // --- simulate_to_terminal, critical path (node ids relative to the commit base) ---
    while (true) {
      if (depth >= cf.depth_cap) { forced = true; break; }
      const int d = depth;
      const int len = d + 1;
      const uint64_t hr = state_at<NSLOT, 1>(h, d);
      snap_take<NSLOT>(snap, h, d);
      const double graw = __shfl_sync(FULL, grew, d);
      const int gnext = __shfl_sync(FULL, gstep, d);
      const bool gchild = golden && len <= glen && lane == gnext;
      const uint64_t jj = (uint64_t)lane;
      double rew;
      if (gchild) {
        rew = graw;
      } else {
        const bool shr = has_shared && len <= hidden;
        const double lo = shr ? sh_lo : off_lo, hi = shr ? sh_hi : off_hi;
        rew = lo + (hi - lo) * u53(sm64(hr ^ jj));
      }
      bool term;
      if (len < bdepth) {
        term = false;
      } else if (len >= bdepth + 1) {
        term = true;
      } else {
        const uint64_t he = state_at<NSLOT, 3>(h, d);
        term = gchild || (sm64(he ^ jj) & 1ull) != 0;
      }
      const bool vl = lane < width;
      const int j = warp_argmax(rew, vl, 0);
      const unsigned tmask = __ballot_sync(FULL, vl && term);
      if (vl) s_rew[d * WS + lane] = rew;
      if (lane == d) lvl_term = tmask;
      const bool jterm = (tmask >> j) & 1u;
      node = nrel + j;  // relative id
      nrel += width;
      ++depth;
      nrew = __shfl_sync(FULL, rew, j);
      const uint32_t nm = (uint32_t)depth | ((uint32_t)j << SH_REF) | (jterm ? M_TERM : 0u);
      if constexpr (PROD) {
        agg.a = agg.a * nrew;
        ++agg.n;
      } else {
        agg.add(nrew, scheme);
      }
      if (depth == 1) d1r = nrew;
      golden = golden && depth <= glen && gnext == j;
      if (lane == depth - 1) { pnode = node; pmeta = nm; prew = nrew; pagg = agg.a; pj = j; }
#pragma unroll
      for (int q = 0; q < NSLOT; ++q) h[q] = sm64(h[q] ^ (uint64_t)j);
      if (jterm) break;
    }
    __syncwarp();
    const int dend = depth;
    const int nlev = dend - d0;
    const double pscore = PROD ? agg.a : agg.value(scheme);
    // --- everything that does not depend on the node ids, before the commit turn ---
    const double up_rew = __shfl_up_sync(FULL, prew, 1);
    const double up_agg = __shfl_up_sync(FULL, pagg, 1);
    const int upj = __shfl_up_sync(FULL, pj, 1);
    const uint32_t up_meta = __shfl_up_sync(FULL, pmeta, 1);
    const double rew_l = lane == 0 ? 1.0 : up_rew;
    const double agg_l = lane == 0 ? 1.0 : up_agg;
    const bool act = lane >= d0 && lane < d0 + nlev;
    int live = 0, ne_cnt = 0;
    uint32_t meta_l = 0;  // word of path node l (expanded at depth l), minus the root's case
    uint64_t hp, hk;
    snap_prior_tokens<NSLOT>(snap, hp, hk);
    if (act) {
      const int l = lane;
      const int len = l + 1;
      double* rawl = s_raw + l * WS;
      const double* rewl = s_rew + l * WS;
      // raw priors and token counts of this level's children (generate_steps)
#pragma unroll
      for (int i = 0; i < WS; ++i) {
        rawl[i] = draw_raw_prior(hp, i);
        tok_acc += draw_tokens(hk, i);
      }
      double tot = rawl[0], cc = 0.0;
#pragma unroll
      for (int i = 1; i < WS; ++i) {
        const double x = rawl[i];
        const double t = tot + x;
        if (fabs(tot) >= fabs(x)) cc += (tot - t) + x;
        else cc += (x - t) + tot;
        tot = t;
      }
      if (cc != 0.0 && isfinite(cc)) tot += cc;
      const bool rel_d1 = strict || d1r >= theta1;
#pragma unroll
      for (int j = 0; j < WS; ++j) {
        rawl[j] = rawl[j] / tot;  // the normalised prior, in place
        if (!((lvl_term >> j) & 1u)) {
          const double rew = rewl[j];
          ++live;
          // NE: a new non-terminal leaf, check-relevant and viable (scoring.py:119-175)
          const bool rel = len == 1 ? (strict || rew >= theta1) : rel_d1;
          double bound = rew;
          if (prefix_bound && l > 0) {
            const double pre = scheme == TS_SCHEME_PRODUCT ? agg_l * rew : (rew < agg_l ? rew : agg_l);
            bound = fmin(rew, pre);
          }
          if (rel && !(bound < tau)) ++ne_cnt;
        }
      }
      if (l >= 1) {  // the expanded node stops being a leaf
        const double bound = prefix_bound ? fmin(rew_l, agg_l) : rew_l;
        if (rel_d1 && !(bound < tau)) --ne_cnt;
      }
      const uint32_t m = l == d0 ? (d0 == 0 ? 0u : up_meta) : ((uint32_t)l | ((uint32_t)upj << SH_REF));
      meta_l = m | M_KIDS | ((uint32_t)live << SH_NEXP);
    }
    int dv = (int)__reduce_add_sync(FULL, (unsigned)(ne_cnt + 64)) - 64 * 32;
    if (forced) {
      const bool rel = strict || d1r >= theta1;
      const double bound = prefix_bound ? fmin(nrew, PROD ? agg.a : agg.value(scheme)) : nrew;
      if (rel && !(bound < tau)) --dv;
    }
    __syncwarp();
    // --- commit in rollout order: node ids, records, parent links, exhaustion ---
    HPROF_ACC(q_comp, t_b);
    HPROF_T0(t_c);
    spin_until_ge(&ctl->committed, k);
    HPROF_ACC(q_cwait, t_c);
    HPROF_T0(t_d);
    int cbase = ctl->nnodes;
    bool ok = ctl->status == TS_OK;
    if (ok && cbase + nlev * width > v.cap) {
      ok = false;
      if (lane == 0) ctl->status = TS_POOL_OVERFLOW;
    }
    if (ok) {
      if (lane >= d0 && lane < dend) pnode += cbase;  // final ids of the new path nodes
      const int fc0 = cbase;
      uint32_t root_meta = (uint32_t)ctl->root_mf;
      if (d0 == 0 && lane == 0) meta_l |= root_meta;  // the root was the selected leaf
      if (risky && lane < d0 - 1) pmeta = ME[2 * pnode];  // current metas for the propagation
      const int up_node = __shfl_up_sync(FULL, pnode, 1);
      const int node_l = lane == 0 ? 0 : up_node;
      if (act) {
        const int l = lane;
        const int len = l + 1;
        const int fcl = fc0 + (l - d0) * width;
        const double* prl = s_raw + l * WS;
        const double* rewl = s_rew + l * WS;
        const bool last = l == dend - 1;
        const int par = l == d0 ? leaf : node_l;
#pragma unroll
        for (int j = 0; j < WS; ++j) {
          const int c = fcl + j;
          const bool onpath = j == pj;
          NO[c] = onpath ? O_ONE : 0ull;
          Wv[c] = 0.0;
          PR[c] = prl[j];
          RW[c] = rewl[j];
          PA[c] = par;
          // the on-path child expanded at the next level gets its word from lane l+1
          if (!onpath || last) {
            uint32_t m = (uint32_t)len | ((uint32_t)j << SH_REF) | (((lvl_term >> j) & 1u) ? M_TERM : 0u);
            if (onpath && forced) m |= M_TERM | M_FORCED;
            MF[c] = mk_mf(-1, m);
          }
        }
      }
      // the selector reads this job's nodes only after acquiring its commit
      if (act) MF[lane == d0 ? leaf : node_l] = mk_mf(fc0 + (lane - d0) * width, meta_l);
      if (d0 == 0 && nlev > 0 && lane == 0) ctl->root_mf = mk_mf(fc0, meta_l);
      {
        const uint32_t dn = __shfl_down_sync(FULL, meta_l, 1);
        const bool dn_act = (lane + 1) >= d0 && (lane + 1) < d0 + nlev;
        if (dn_act) pmeta = dn;
        if (d0 == 0 && nlev > 0) root_meta = __shfl_sync(FULL, meta_l, 0);
        if (forced && lane == dend - 1) pmeta |= M_TERM | M_FORCED;
      }
      if (forced && nlev == 0) {
        const uint32_t m = __shfl_sync(FULL, pmeta, dend - 1);
        const int lid = __shfl_sync(FULL, pnode, dend - 1);
        if (lane == 0) ME[2 * lid] = m;
      }
      __syncwarp();
      int dead_from = -1;
      if (forced) dead_from = dend;
      else if (nlev > 0 && __shfl_sync(FULL, live, dend - 1) == 0) dead_from = dend - 1;
      if (dead_from >= 0) {
        for (int i = dead_from - 1; i >= 0; --i) {
          uint32_t m = i == 0 ? root_meta : __shfl_sync(FULL, pmeta, i - 1);
          const int pid = i == 0 ? 0 : __shfl_sync(FULL, pnode, i - 1);
          m -= NEXP_ONE;
          if (lane == 0) ME[2 * pid] = m;
          if (i == 0 && lane == 0) ctl->root_mf = (ctl->root_mf & 0xFFFFFFFF00000000ull) | m;
          if (i == 0) root_meta = m;
          else if (lane == i - 1) pmeta = m;
          if (meta_nexp(m) > 0) break;
        }
      }
      SPs[(size_t)k * 32 + lane] = pnode;
      if (lane == 0) {
        SSs[k] = pscore;
        SLs[k] = dend;
        ctl->nnodes = cbase + nlev * width;
        ctl->viable = ctl->viable + dv;
      }
      created += (unsigned long long)nlev * width;
    }
    __syncwarp();
    if (lane == 0) st_release_cta(&ctl->committed, k + 1);
    HPROF_ACC(q_commit, t_d);
  }
#ifdef TS_HEAVY_PROF
  if (lane == 0) {
    atomicAdd(&v.ctr->prof[8], (unsigned long long)q_issue);
    atomicAdd(&v.ctr->prof[9], (unsigned long long)q_comp);
    atomicAdd(&v.ctr->prof[10], (unsigned long long)q_cwait);
    atomicAdd(&v.ctr->prof[11], (unsigned long long)q_commit);
  }
#endif
  long long t = tok_acc;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&ctl->tokens, (unsigned long long)t);
    atomicAdd((unsigned long long*)&ctl->created, created);
  }
}

// warp 0 after all commits: backups, exit decisions, cancellations (as the
// single-warp mode's multi-rollout path) and the search-state write-back
__device__ __forceinline__ void heavy_finish(const View& v, int s, int step, HeavyCtl* ctl, int nl, uint64_t rno, double rW,
                             int decision, WaveStats& ws) {
  const int lane = threadIdx.x & 31;
  const ts_config& cf = v.cfg;
  SearchState* S = v.st + s;
  const size_t base = (size_t)s * (size_t)v.cap;
  uint64_t* NO = v.no + base;
  double* Wv = v.W + base;
  const uint32_t* ME = (const uint32_t*)(v.mf + base);
  double* QQ = v.Q + base;
  const int budget = cf.rollout_budget;
  int32_t* SPs = v.sp + (size_t)s * (size_t)budget * 32;
  double* SSs = v.ss + (size_t)s * budget;
  int32_t* SLs = v.sl + (size_t)s * budget;
  int completed = S->completed;
  int best_term = S->best_term;
  double best = S->best;
  int launched = S->launched + nl, cancelled = S->cancelled;
  int status = ctl->status;
  const int viable = ctl->viable;
  const uint32_t root_meta = ME[0];
  unsigned long long done = 0, pathn = 0;
  const bool exhausted = decision == -1;
  if (exhausted) decision = TS_EXIT_NONE;
  auto decide = [&](bool exh) -> int {
    if (cf.positive_exit && best_term >= 0 && best >= cf.positive_exit_threshold) return TS_EXIT_POSITIVE;
    if (cf.negative_exit && (root_meta & M_KIDS) && viable == 0) return TS_EXIT_NEGATIVE;
    if (exh || completed >= budget) return TS_EXIT_BUDGET;
    return TS_EXIT_NONE;
  };
  if (status == TS_OK && exhausted) decision = decide(true);
  if (status == TS_OK && !exhausted && nl > 0) {
    // All expansions of the wave are done, so the viable-leaf count and the
    // root are final: the first backup after which decide_exit fires
    // (scoring.py:184-207) depends only on the scores.  PE fires at the first
    // score >= theta, NE at the first backup, the budget at the last allowed one.
    int rstar = budget - completed - 1;  // nl <= budget - completed
    if (cf.negative_exit && (root_meta & M_KIDS) && viable == 0) rstar = 0;
    if (cf.positive_exit) {
      for (int r0 = 0; r0 < nl && r0 <= rstar; r0 += 32) {
        const int r = r0 + lane;
        const unsigned m = __ballot_sync(FULL, r < nl && SSs[r] >= cf.positive_exit_threshold);
        if (m) {
          rstar = min(rstar, r0 + __ffs(m) - 1);
          break;
        }
      }
    }
    const int nb = min(rstar, nl - 1) + 1;  // rollouts backed up, in launch order
    // best trajectory: the first of the maximal scores, if it beats the old best (tree.py:370)
    {
      double mx = -INFINITY;
      for (int r = lane; r < nb; r += 32) mx = fmax(mx, SSs[r]);
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
      int rb = nb;
      for (int r0 = 0; r0 < nb; r0 += 32) {
        const unsigned m = __ballot_sync(FULL, r0 + lane < nb && SSs[r0 + lane] == mx);
        if (m) { rb = r0 + __ffs(m) - 1; break; }
      }
      if (best_term < 0 || mx > best) {
        best = mx;
        best_term = SPs[(size_t)rb * 32 + SLs[rb] - 1];
      }
    }
    // backpropagate (tree.py:352-371) of rollouts [0, nb): lane i owns depth
    // i+1 (a node has one depth, so lanes never share a node) and adds the
    // scores in launch order, keeping runs of the same node in registers
    // The rollouts are read 4 at a time: their lengths, scores, this lane's
    // node ids and those nodes' N|O and W load together (independent, one
    // round trip); a node this lane already wrote back in the same batch is
    // re-read after its write-back instead (the prefetched copy is older).
    bool bad = false;
    int cur = -1;
    uint64_t cno = 0;
    double cw = 0.0;
    unsigned long long pl = 0;
    constexpr int BB = 4;
    for (int r0 = 0; r0 < nb; r0 += BB) {
      int lenb[BB], idb[BB];
      double scb[BB], wb[BB];
      uint64_t nob[BB];
#pragma unroll
      for (int k = 0; k < BB; ++k) {
        const int r = min(r0 + k, nb - 1);
        lenb[k] = SLs[r];
        scb[k] = SSs[r];
        idb[k] = SPs[(size_t)r * 32 + lane];
      }
#pragma unroll
      for (int k = 0; k < BB; ++k) {
        const bool use = r0 + k < nb && lane < lenb[k];
        if (!use) idb[k] = -1;
        nob[k] = use ? NO[idb[k]] : 0ull;
        wb[k] = use ? Wv[idb[k]] : 0.0;
      }
      const int cur0 = cur;  // the run carried into this batch (written back in it if left)
#pragma unroll
      for (int k = 0; k < BB; ++k) {
        if (r0 + k >= nb) break;
        const double sc = scb[k];
        pl += lenb[k] + 1;
        if ((rno >> 32) < 1) bad = true;
        rno = rno + 1 - O_ONE;
        rW += sc;
        const int nd = idb[k];
        if (nd >= 0) {
          if (nd != cur) {
            if (cur >= 0) {
              NO[cur] = cno;
              Wv[cur] = cw;
              QQ[cur] = cw / (double)(uint32_t)cno;
            }
            // the carried run or a node seen earlier in this batch, left since:
            // written back after the prefetch
            bool again = nd == cur0;
#pragma unroll
            for (int j = 0; j < k; ++j) again |= idb[j] == nd;
            cur = nd;
            if (again) {  // written back earlier in this batch: the prefetched copy is stale
              cno = NO[nd];
              cw = Wv[nd];
            } else {
              cno = nob[k];
              cw = wb[k];
            }
          }
          if ((cno >> 32) < 1) bad = true;
          cno = cno + 1 - O_ONE;
          cw += sc;
        }
      }
    }
    if (cur >= 0) {
      NO[cur] = cno;
      Wv[cur] = cw;
      QQ[cur] = cw / (double)(uint32_t)cno;
    }
    if (lane == 0) { NO[0] = rno; Wv[0] = rW; QQ[0] = rW / (double)(uint32_t)rno; }
    if (__any_sync(FULL, bad)) status = TS_ACCOUNTING;
    completed += nb;
    done += nb;
    pathn += pl;
    if (status == TS_OK) decision = decide(false);
    __syncwarp();
    if (status == TS_OK && nb < nl && ctl->nnodes <= HEAVY_ZERO_O_MAX) {
      // cancel_inflight (tree.py:374-380) for the wave's remaining rollouts,
      // at an exit.  Every wave ends with no rollout in flight, so O was 0 on
      // every node when this wave started; after the backups above the only
      // in-flight counts left are exactly the cancelled rollouts', and
      // removing them returns every node to O = 0.  The whole CTA clears the
      // O half of the search's N|O words after this call (coalesced), instead
      // of one warp decrementing ~17 scattered nodes per cancelled rollout.
      const int first = nb, ncan = nl - first;
      long long pc = 0;
      for (int r2 = first + lane; r2 < nl; r2 += 32) pc += SLs[r2] + 1;
      for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(FULL, pc, o);
      if ((long long)(rno >> 32) < ncan) status = TS_ACCOUNTING;
      rno -= (uint64_t)ncan * O_ONE;
      if (lane == 0) {
        NO[0] = rno;
        ctl->zero_o = 1;
      }
      __syncwarp();
      cancelled += ncan;
      pathn += (unsigned long long)pc;
    } else if (status == TS_OK && nb < nl) {
      // cancel_inflight (tree.py:374-380) for the wave's remaining rollouts.
      // Their order does not matter (O -= 1 on each path node), so lanes take
      // whole rollouts and decrement with atomics; a node's in-flight count
      // must not underflow (AccountingError), checked after all decrements.
      const int first = nb, ncan = nl - first;
      long long pc = 0;
      for (int r2 = first + lane; r2 < nl; r2 += 32) {
        const int len2 = SLs[r2];
        const int32_t* row = SPs + (size_t)r2 * 32;
        for (int i = 0; i < len2; ++i)
          atomicAdd((unsigned long long*)&NO[row[i]], (unsigned long long)(0ull - O_ONE));
        pc += len2 + 1;
      }
      for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(FULL, pc, o);
      __threadfence_block();
      __syncwarp();
      bool bad2 = (long long)(rno >> 32) < ncan;
      for (int r2 = first + lane; r2 < nl; r2 += 32) {
        const int len2 = SLs[r2];
        const int32_t* row = SPs + (size_t)r2 * 32;
        for (int i = 0; i < len2; ++i)
          if ((NO[row[i]] >> 32) > (uint64_t)budget) bad2 = true;  // wrapped below zero
      }
      if (__any_sync(FULL, bad2)) status = TS_ACCOUNTING;
      rno -= (uint64_t)ncan * O_ONE;
      if (lane == 0) NO[0] = rno;
      __syncwarp();
      cancelled += ncan;
      pathn += (unsigned long long)pc;
    }
  }
  if (lane == 0) {
    S->completed = completed;
    S->nodes = ctl->nnodes;
    S->viable = viable;
    S->best_term = best_term;
    S->best = best;
    S->tokens += (long long)ctl->tokens;
    atomicAdd(&v.ctr->tokens, ctl->tokens);
    S->launched = launched;
    S->cancelled = cancelled;
    double jb = S->job_best;
    if (best_term >= 0 && best > jb) S->job_best = jb = best;
    write_next_record(v, s, step, status != TS_OK || decision != TS_EXIT_NONE, completed, jb);
    if (status != TS_OK || decision != TS_EXIT_NONE) {
      S->state = ST_FINISHED;
      S->exit_kind = status == TS_OK ? decision : TS_EXIT_NONE;
      S->status = status;
      S->exit_step = step;
      S->t_exit = globaltimer();
      atomicAdd((unsigned long long*)&v.ctr->running, (unsigned long long)-1ll);
      atomicAdd((unsigned long long*)&v.ctr->finished, 1ull);
      atomicMax(&v.ctr->last_exit_step, (long long)step);
    }
  }
  ws.rollouts += done;
  ws.launched += nl;
  ws.nodes += ctl->created;
  ws.path_nodes += pathn;
}

// One search's wave in the pipelined CTA mode, run by a unit of the CTA:
// the whole CTA (8 warps: warp 0 selects, warp 4 idles on its scheduler
// partition, 6 simulators), or, in the paired mode (DUAL), the 4 warps of one
// parity (warp g selects, warps g+2, g+4, g+6 simulate), so that one CTA runs
// two searches side by side with named barriers.
template <bool DUAL>
__device__ __forceinline__ void heavy_bar(int g) {
  if constexpr (DUAL) asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
  else __syncthreads();
}

template <int NSLOT, int WT, bool PROD, bool DUAL>
__device__ __forceinline__ void heavy_item(const View& v, int step, int item, HeavyCtl& ctl, HeavyJob* ring, const double* sqt,
                           double* hsm, WaveStats& ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = DUAL ? (warp & 1) : 0;
  const int gw = DUAL ? (warp >> 1) : warp;  // warp index in the unit
  constexpr int UT = DUAL ? 128 : HEAVY_THREADS;
  const int ut = gw * 32 + lane;
  const int s = v.work_heavy[item];
  const SearchState* S = v.st + s;
  const int count = min(v.tgt[s], v.cfg.rollout_budget - S->completed);
  if (ut == 0) {
    ctl.issued = 0;
    ctl.committed = 0;
    ctl.done = 0;
    ctl.zero_o = 0;
    ctl.status = TS_OK;
    ctl.nnodes = S->nodes;
    ctl.viable = S->viable;
    ctl.created = 0;
    ctl.tokens = 0;
    ctl.root_mf = v.mf[(size_t)s * (size_t)v.cap];
  }
  heavy_bar<DUAL>(g);
  uint64_t rno = 0;
  double rW = 0.0;
  int decision = TS_EXIT_NONE;
  if (gw == 0) {
    heavy_select<NSLOT, WT, PROD>(v, s, &ctl, ring, sqt, count, ws, rno, rW, decision);
  } else if (DUAL || gw != 4) {
    const int si = DUAL ? gw - 1 : heavy_sim_of_warp(gw);
    const int slot = DUAL ? g * 3 + si : si;  // staging rows of this simulator
    double* s_raw = hsm + (size_t)slot * 2 * 32 * WT;
    heavy_simulate<NSLOT, WT, PROD>(v, s, &ctl, ring, s_raw, s_raw + 32 * WT, si, DUAL ? 3 : HEAVY_SIM);
  }
  heavy_bar<DUAL>(g);
#ifdef TS_HEAVY_PROF
  long long t_fin = clock64();
#endif
  if (gw == 0) heavy_finish(v, s, step, &ctl, ctl.issued, rno, rW, decision, ws);
  heavy_bar<DUAL>(g);
  if (ctl.zero_o) {  // the cancellation of an exit: O back to 0 on every node but the root
    uint64_t* NO = v.no + (size_t)s * (size_t)v.cap;
    const int nn = ctl.nnodes;
    // 8 independent loads in flight per thread, then the stores
    constexpr int U = 8;
    for (int i0 = 1 + ut; i0 < nn; i0 += U * UT) {
      uint64_t w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * UT;
        w[u] = i < nn ? NO[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * UT;
        if (i < nn && (w[u] >> 32)) NO[i] = w[u] & 0xffffffffull;
      }
    }
  }
#ifdef TS_HEAVY_PROF
  if (ut == 0) atomicMax(&v.ctr->prof[15], (unsigned long long)(clock64() - t_fin));
#endif
  heavy_bar<DUAL>(g);
}

// Work: items [0, n) of the wave's pipelined-mode list over G resident CTAs.
// Each CTA claims c from a counter and takes item c (claim order: the first
// CTAs to start, one per SM before a second on the same SM, as far as the
// block scheduler spreads them); when the wave has more items than CTAs
// (config 2's third wave: 297 boosted searches for 296 CTAs), claims c < n - G
// also take item G + c and run both side by side in the paired mode instead
// of one after the other (the wave is as long as its longest CTA).  Items
// from 2G on are claimed one at a time from a second counter (a CTA that
// starts late must still get its first-round claim).
template <int NSLOT, int WT, bool PROD>
#ifdef TS_HEAVY_MAXNREG
__global__ void __maxnreg__(TS_HEAVY_MAXNREG) k_heavy(View v, int step) {
#else
__global__ void __launch_bounds__(HEAVY_THREADS, TS_HEAVY_MINB) k_heavy(View v, int step) {
#endif
  extern __shared__ double hsm[];
  __shared__ HeavyCtl ctl[2];
  __shared__ HeavyJob ring[2][HEAVY_RING];
  __shared__ int s_item;
  __shared__ double sqt[SQRT_TAB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WaveStats ws = {0, 0, 0, 0, 0, 0, 0};
  const int count_items = v.ctr->heavy_count;
  if (count_items == 0) return;  // most waves have no pipelined-mode search
  if (step < 0) step = v.ctr->cur_step;
  const int G = gridDim.x;
  if (threadIdx.x == 0) s_item = atomicAdd(&v.ctr->heavy_next, 1);
  __syncthreads();
  const int b = s_item;
  if (b >= count_items) return;  // no item for this CTA: skip the table set-up
#ifdef TS_SCHED_PROF
  if (threadIdx.x == 0) atomicMin(&v.ctr->prof[21], globaltimer());
#endif
  for (int i = threadIdx.x; i < SQRT_TAB; i += HEAVY_THREADS) sqt[i] = sqrt((double)i);
  __syncthreads();
  if (b < count_items - G) {
    const int g = warp & 1;
    heavy_item<NSLOT, WT, PROD, true>(v, step, g == 0 ? b : G + b, ctl[g], ring[g], sqt, hsm, ws);
    __syncthreads();
  } else {
    heavy_item<NSLOT, WT, PROD, false>(v, step, b, ctl[0], ring[0], sqt, hsm, ws);
  }
  for (;;) {  // items from 2G on, one at a time
    if (count_items <= 2 * G) break;
    if (threadIdx.x == 0) s_item = 2 * G + atomicAdd(&v.ctr->heavy_next2, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= count_items) break;
    heavy_item<NSLOT, WT, PROD, false>(v, step, item, ctl[0], ring[0], sqt, hsm, ws);
  }
#ifdef TS_SCHED_PROF
  if (threadIdx.x == 0) atomicMax(&v.ctr->prof[20], globaltimer());
#endif
  if (lane == 0 && ws.launched) {  // the selector warps' statistics
    atomicAdd(&v.ctr->rollouts, ws.rollouts);
    atomicAdd(&v.ctr->launched, ws.launched);
    atomicAdd(&v.ctr->nodes, ws.nodes);
    atomicAdd(&v.ctr->scored, ws.scored);
    atomicAdd(&v.ctr->levels, ws.levels);
    atomicAdd(&v.ctr->path_nodes, ws.path_nodes);
    if (ws.tokens) atomicAdd(&v.ctr->tokens, ws.tokens);
  }
}

static const wave_kernel_t kHeavy[2][3][3] = {
    {{k_heavy<1, 2, false>, k_heavy<1, 4, false>, k_heavy<1, 8, false>},
     {k_heavy<2, 2, false>, k_heavy<2, 4, false>, k_heavy<2, 8, false>},
     {k_heavy<4, 2, false>, k_heavy<4, 4, false>, k_heavy<4, 8, false>}},
    {{k_heavy<1, 2, true>, k_heavy<1, 4, true>, k_heavy<1, 8, true>},
     {k_heavy<2, 2, true>, k_heavy<2, 4, true>, k_heavy<2, 8, true>},
     {k_heavy<4, 2, true>, k_heavy<4, 4, true>, k_heavy<4, 8, true>}},
};
size_t heavy_smem_of(int wkind) {
  const int ws = wkind == 0 ? 2 : wkind == 1 ? 4 : 8;
  return (size_t)HEAVY_SIM * 2 * 32 * ws * sizeof(double);
}

__global__ void k_latency(View v, unsigned long long* out, int n) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const SearchState& st = v.st[s];
  unsigned long long r = 0;
  if (st.exit_step >= 0 && st.admit_step >= 0 && st.admit_step < v.step_times_cap) {
    unsigned long long t0 = v.step_times[st.admit_step];
    r = st.t_exit > t0 ? st.t_exit - t0 : 0;
  }
  out[s] = r;
}

// SearchOutcome (search.py:32-42): best path by parent walk, solved flag.
__global__ void k_outcomes(View v, ts_outcome* out, int n) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const SearchState st = v.st[s];
  const ts_problem* pb = v.prob + s;
  ts_outcome o;
  memset(&o, 0, sizeof(o));
  o.exit_kind = st.exit_kind;
  o.rollouts_completed = st.completed;
  o.tokens_generated = st.tokens;
  o.best_score = st.best_term >= 0 ? st.best : 0.0;
  o.exit_step = st.exit_step;
  o.admit_step = st.admit_step;
  o.launched = st.launched;
  o.cancelled = st.cancelled;
  o.nodes = st.nodes;
  o.status = st.status;
  if (st.best_term >= 0) {
    const size_t base = (size_t)s * (size_t)v.cap;
    int ids[TS_MAX_DEPTH + 1];
    int n2 = 0;
    for (int c = st.best_term; c > 0 && n2 <= TS_MAX_DEPTH; c = v.parent[base + c]) ids[n2++] = c;
    o.best_len = n2;
    for (int i = 0; i < n2; ++i)
      o.best_path[i] = (uint8_t)(((uint32_t)v.mf[base + ids[n2 - 1 - i]] >> SH_REF) & 31u);
    if (pb->golden_len >= 0 && o.best_len == pb->golden_len) {
      o.solved = 1;
      for (int i = 0; i < n2; ++i)
        if (o.best_path[i] != pb->golden_path[i]) o.solved = 0;
    }
  }
  out[s] = o;
}

// ---- invariant checks (ts_engine_set_checks) ----------------------------------
// The reference's run-time invariants, asserted on the device state of every
// wave (test_acceptance.py:167-187, test_simulator.py:58-64, simulator.py:252-260):
//  * capacity: Σ_i min(P_i, budget - completed_i) <= M rollouts in flight per
//    wave (Engine._check_capacity), and |running| <= M;
//  * serial gate: a search below the observation gate runs one rollout;
//  * every wave ends with no rollout in flight: O == 0 on every node of every
//    search the wave touched (each launch is backed up or cancelled);
//  * conservation: launched == completed + cancelled per search, root N ==
//    completed_rollouts.
enum { INV_WAVES = 0, INV_CAPACITY, INV_GATE, INV_INFLIGHT, INV_CONSERVATION, INV_ROOT, INV_MAX_LAUNCH,
       INV_MAX_RUNNING };

__global__ void __launch_bounds__(1024) k_check_pre(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  long long sum = 0, gate = 0;
  for (int i = threadIdx.x; i < nw + nh; i += blockDim.x) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    const int done = v.st[s].completed;
    const int P = v.tgt[s];
    sum += min(P, v.cfg.rollout_budget - done);
    if (done < v.cfg.obs_threshold && P > 1) ++gate;
  }
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(FULL, sum, o);
    gate += __shfl_xor_sync(FULL, gate, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long*)&c->inv_wave, (unsigned long long)sum);
    if (gate) atomicAdd((unsigned long long*)&c->inv[INV_GATE], (unsigned long long)gate);
  }
  if (threadIdx.x == 0 && nw + nh > 0) {
    const long long run = c->running;
    if (run > c->inv[INV_MAX_RUNNING]) c->inv[INV_MAX_RUNNING] = run;
    if (run > v.cfg.max_concurrency) c->inv[INV_CAPACITY] += 1;
  }
}

__global__ void __launch_bounds__(256) k_check_post(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  __shared__ unsigned long long s_bad;
  if (blockIdx.x == 0 && threadIdx.x == 0 && nw + nh > 0) {
    const long long w = c->inv_wave;
    c->inv_wave = 0;
    c->inv[INV_WAVES] += 1;
    if (w > c->inv[INV_MAX_LAUNCH]) c->inv[INV_MAX_LAUNCH] = w;
    if (w > v.cfg.max_concurrency) c->inv[INV_CAPACITY] += 1;
  }
  for (int i = blockIdx.x; i < nw + nh; i += gridDim.x) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    const SearchState st = v.st[s];
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    const size_t base = (size_t)s * (size_t)v.cap;
    unsigned long long bad = 0;
    for (int k = threadIdx.x; k < st.nodes; k += blockDim.x) bad += (v.no[base + k] >> 32) != 0 ? 1 : 0;
    bad = __reduce_add_sync(FULL, (unsigned)bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&s_bad, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_bad) atomicAdd((unsigned long long*)&c->inv[INV_INFLIGHT], s_bad);
      if (st.status == TS_OK) {
        if (st.launched != st.completed + st.cancelled)
          atomicAdd((unsigned long long*)&c->inv[INV_CONSERVATION], 1ull);
        if ((int)(uint32_t)v.no[base] != st.completed) atomicAdd((unsigned long long*)&c->inv[INV_ROOT], 1ull);
      }
    }
    __syncthreads();
  }
}

// ---- allocation trace (ts_engine_set_trace) -------------------------------------
// One row per running search per scheduler pass, written between the pass and
// the wave: the fields of the reference's per-pass "allocation" record
// (simulator.py:314-330): parallelism_score at the pass (the same expressions
// as the pass's records, scheduler.py:118-128), the target, and the active
// rollouts (0: every wave ends with none in flight).  The host sorts the rows
// into run-queue order and adds the "action" records reconcile() would emit.
__global__ void __launch_bounds__(256) k_trace(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  const int step = c->cur_step;
  const ts_config& cf = v.cfg;
  for (int i = threadIdx.x; i < nw + nh; i += blockDim.x) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    const double ratio = v.st[s].job_best / cf.positive_exit_threshold;
    ts_trace_row r;
    r.step = step;
    r.job = v.goff + s;
    r.target = v.tgt[s];
    r.active = 0;
    r.score = v.log1p_tab[step - v.arrival[s]] + (ratio > cf.proximity ? cf.beta : 0.0);
    const unsigned long long k = atomicAdd(&c->trace_n, 1ull);
    if (k < (unsigned long long)v.trace_cap) v.trace[k] = r;
    else atomicAdd(&c->trace_drop, 1ull);
  }
}

// ---- the wave clock of a cost model (ts_engine_set_cost_model) ---------------------
// SURVEY §8(f4), a wave-level restatement of the reference's simulated time
// (backend.py:287-311, simulator.py:443-463): every generation request of a
// launched rollout (one expansion of its simulation) takes
//     max(service_time(token_count, cost, load) for the candidates) + reward_latency
//   = ((max_tokens * per_token_latency) * contention) + reward_latency,
// contention = max(1, load / engine_capacity), accumulated onto the wave's
// start clock in expansion order like the reference's event times.  load is
// the wave's in-flight candidate count: sum over the wave's launched rollouts
// of the expansion width.  A search's wave ends with its last rollout; the
// clock advances to the latest end (idle steps take no time).  The wave
// kernels are untouched: after the wave, the expansions are recovered from the
// node pool (a wave's new nodes are its expansions in creation order, `width`
// children each; an expansion continues the previous one's rollout iff its
// parent is the previous expansion's greedy child, since a rollout stops only
// at a terminal greedy child, which no later selection can expand) and their
// token counts are redrawn from the keyed RNG (backend.py:261-263).

// Between the pass and the wave: the clock of this step, per-search snapshots.
__global__ void __launch_bounds__(256) k_cost_pre(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  if (threadIdx.x == 0) {
    const double cm = __longlong_as_double((long long)c->clock_max);
    double clk = c->clock;
    if (cm > clk) clk = cm;
    c->clock = clk;
    c->cost_load = 0;
    // a pass after the batch has ended repeats the last step: keep its start
    const int step = c->cur_step;
    if (c->clock_step1 != (long long)step + 1) {
      if (step < v.step_times_cap) v.clock_at[step] = clk;
      c->clock_step1 = (long long)step + 1;
    }
  }
  for (int i = threadIdx.x; i < nw + nh; i += blockDim.x) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    v.cost_snap[s] = make_int2(v.st[s].nodes, v.st[s].launched);
  }
}

__device__ __forceinline__ int cost_width(const View& v, int s) {
  return min(v.cfg.expand_width, v.prob[s].branching);
}

// After the wave: load = sum of width x launched rollouts over the wave.
__global__ void __launch_bounds__(1024) k_cost_load(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  long long x = 0;
  for (int i = threadIdx.x; i < nw + nh; i += blockDim.x) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    x += (long long)cost_width(v, s) * (long long)(v.st[s].launched - v.cost_snap[s].y);
  }
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long*)&c->cost_load, (unsigned long long)x);
}

// After k_cost_load: one warp per search of the wave.  Lane k of a round of
// 32 expansions recovers expansion g = 32*round + k (parent, greedy child, max
// token count of its candidates); the warp then folds the round's durations
// in expansion order.
__global__ void __launch_bounds__(256) k_cost_wave(View v) {
  Counters* c = v.ctr;
  const int nw = c->work_count, nh = c->heavy_count;
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * (size_t)blockDim.x) >> 5);
  const double clock = c->clock;
  double cont = (double)c->cost_load / (double)v.cost_cap;  // inflight_load / engine_capacity
  if (!(cont > 1.0)) cont = 1.0;                            // max(1.0, ...)
  const double pt = v.cost_pt, rl = v.cost_rl;
  const int step = c->cur_step;
  for (int i = warp; i < nw + nh; i += nwarps) {
    const int s = i < nw ? v.work[i] : v.work_heavy[i - nw];
    const int w = cost_width(v, s);
    const SearchState& S = v.st[s];
    const int nb = v.cost_snap[s].x;
    const int G = (S.nodes - nb) / w;
    const size_t base = (size_t)s * (size_t)v.cap;
    const int32_t* PA = v.parent + base;
    const double* RW = v.reward + base;
    const uint64_t* MF = v.mf + base;
    const uint64_t seed = v.prob[s].seed;
    double t = clock, end = clock;
    int prev_greedy = -1;
    for (int g0 = 0; g0 < G; g0 += 32) {
      const int g = g0 + lane;
      int par = -1, greedy = -1, mt = 0;
      if (g < G) {
        const int fc = nb + g * w;
        par = PA[fc];
        // greedy_child (tree.py:307-319): strict '>', first wins
        greedy = fc;
        double br = RW[fc];
        for (int j = 1; j < w; ++j)
          if (RW[fc + j] > br) { br = RW[fc + j]; greedy = fc + j; }
        // the index path of the expanded node, root first
        const uint32_t pm = (uint32_t)MF[par];
        const int d = (int)(pm & M_DEPTH);
        uint8_t refs[TS_MAX_DEPTH + 1];
        int x = par;
        for (int k = d - 1; k >= 0; --k) {
          refs[k] = (uint8_t)((((uint32_t)MF[x]) >> SH_REF) & 31u);
          x = PA[x];
        }
        // token counts: randint(40, 120, seed, 3, len(cp), *cp) (backend.py:261-263)
        uint64_t h = sm64(MIX_INIT ^ seed);
        h = sm64(h ^ 3ull);
        h = sm64(h ^ (uint64_t)(d + 1));
        for (int k = 0; k < d; ++k) h = sm64(h ^ (uint64_t)refs[k]);
        for (int j = 0; j < w; ++j) {
          const int tok = 40 + (int)(sm64(h ^ (uint64_t)j) % 81ull);
          mt = tok > mt ? tok : mt;
        }
      }
      const int m = min(32, G - g0);
      for (int k = 0; k < m; ++k) {
        const int pk = __shfl_sync(FULL, par, k);
        const int gk = __shfl_sync(FULL, greedy, k);
        const int tk = __shfl_sync(FULL, mt, k);
        if (pk != prev_greedy) t = clock;  // a new rollout's first expansion
        t = t + ((double)tk * pt * cont + rl);
        if (t > end) end = t;
        prev_greedy = gk;
      }
    }
    if (lane == 0) {
      atomicMax(&c->clock_max, (unsigned long long)__double_as_longlong(end));
      if (S.state == ST_FINISHED && S.exit_step == step) v.sim_done[s] = end;
    }
  }
}

}  // namespace

// ============================================================================
// host side
// ============================================================================
struct ts_engine {
  int device = 0;
  ts_config cfg{};
  std::string err;
  int sm_count = 148;
  int wave_blocks[12] = {0};
  int wkind = 3;
  bool heavy_off = false;  // TS_NO_PIPELINE=1 disables the pipelined CTA mode (diagnostics)
  int mt_min = 6144;       // TS_MT_MIN: largest run queue for the one-CTA targets kernel
  int coop_ctas = -1;      // co-resident CTAs of k_mt_all (cooperative launch), 0 = unavailable
  bool heavy_sync = false; // TS_PIPELINE_SYNC=1 serialises it (diagnostics)
  // sizes
  int n_local = 0, goff = 0, n_global = 0, cap_searches = 0, cap_global = 0;
  long long cap = 0, pool_nodes = 0;
  int nslot = 4;
  bool loaded = false;
  // device buffers
  uint64_t* no = nullptr;
  double* W = nullptr;
  double* Q = nullptr;
  double* prior = nullptr;
  double* reward = nullptr;
  uint64_t* mf = nullptr;
  int32_t* parent = nullptr;
  SearchState* st = nullptr;
  ts_problem* prob = nullptr;
  int32_t* arrival = nullptr;
  Counters* ctr = nullptr;
  int32_t* work = nullptr;
  int32_t* work_heavy = nullptr;
  int32_t* tgt = nullptr;
  ts_sched_record* nrec = nullptr;
  int heavy_blocks = 0;
  int32_t* sp = nullptr;
  double* ss = nullptr;
  int32_t* sl = nullptr;
  size_t scratch_rows = 0;
  double* log1p_tab = nullptr;
  int log1p_n = 0;
  unsigned long long* step_times = nullptr;
  int step_times_cap = 0;
  double* g_runS = nullptr;
  int32_t* g_runStart = nullptr;
  long long* g_runWant = nullptr;
  long long* g_runPW = nullptr;
  unsigned char* mt = nullptr;      // multi-CTA targets scratch (mt_layout)
  size_t mt_bytes = 0;
  long long* counts = nullptr;      // 3
  ts_sched_record* records = nullptr;
  ts_outcome* outcomes = nullptr;
  int outcomes_cap = 0;
  int max_arrival = 0;
  long long launches = 0;
  void* pin = nullptr;  // pinned staging for host tables (problems in, outcomes out)
  size_t pin_bytes = 0;
  void* pin_out = nullptr;  // pinned staging of ts_run_batch_host's outcomes
  size_t pin_out_bytes = 0;
  Counters* pin_ctr = nullptr;  // pinned copy of the counters read after a run
  std::vector<cudaEvent_t> wave_ev;  // start/stop pairs of every wave since load
  size_t wave_ev_used = 0;
  // ts_run: CUDA graph with a device-driven while loop over {k_sched, k_wave}
  cudaGraph_t run_graph = nullptr;
  cudaGraphExec_t run_exec = nullptr;
  View run_view;
  bool graph_failed = false;
  int checks = 0;        // ts_engine_set_checks
  ts_trace_row* trace = nullptr;  // ts_engine_set_trace
  long long trace_cap = 0;
  double cost_pt = 0.0, cost_rl = 0.0;  // ts_engine_set_cost_model
  int cost_cap = 0;
  int2* cost_snap = nullptr;
  double* sim_done = nullptr;
  int cost_n = 0;
  double* clock_at = nullptr;  // step_times_cap entries
  int graph_unroll = 3;  // scheduler passes + waves per iteration of the graph's while loop (TS_GRAPH_UNROLL)
  // ts_run_sharded: this rank's exchange buffer and every rank's (IPC mappings
  // of other processes' buffers, or in-process pointers), the batch generation
  unsigned char* xbuf = nullptr;
  unsigned long long* xstamp = nullptr;  // PX_STAMP_WAVES x 3 timestamps
  unsigned char* xscr = nullptr;         // group scheduler scratch (px_scr)
  size_t xbytes = 0;
  int xworld = 0, xrank = 0, xgen = 0;
  unsigned char* xpeer[TS_MAX_PEERS] = {};
  bool xipc[TS_MAX_PEERS] = {};
  bool xconnected = false;
  cudaGraph_t px_graph = nullptr;
  cudaGraphExec_t px_exec = nullptr;
  View px_view;
  int px_max_steps = -1;
  bool free_ok = false;          // free-running waves allowed for the loaded batch (see k_sched)
  bool free_off = false;         // TS_NO_FREE=1 (diagnostics)
  bool free_kernel_off = false;  // TS_NO_FREE_KERNEL=1: k_wave runs the free-running waves itself (diagnostics)
  int32_t* fdone = nullptr;      // n_local: chunks of a search's rollouts done (free-running waves)
  int fdone_cap = 0;
  bool px_two_kernels = false;  // TS_PX_TWO_KERNELS=1: k_px_groups + k_px_sched instead of k_px_step (diagnostics)
  int px_gwarp = 32;            // TS_PX_GWARP: k_px_step's one-warp scheduler up to this many group entries
};

namespace {

int fail(ts_engine* e, int code, const std::string& msg) {
  if (e) e->err = msg;
  return code;
}
int cuda_fail(ts_engine* e, cudaError_t rc, const char* where) {
  return fail(e, TS_CUDA, std::string(where) + ": " + cudaGetErrorString(rc));
}
#define TS_CUDA_TRY(e, expr)                                   \
  do {                                                         \
    cudaError_t rc_ = (expr);                                  \
    if (rc_ != cudaSuccess) return cuda_fail((e), rc_, #expr); \
  } while (0)
#define TS_LAUNCH_CHECK(e, name)                                  \
  do {                                                            \
    ++(e)->launches;                                              \
    cudaError_t rc_ = cudaGetLastError();                         \
    if (rc_ != cudaSuccess) return cuda_fail((e), rc_, name);     \
  } while (0)

template <class T>
int grow(ts_engine* e, T*& p, size_t n, size_t& have, const char* what) {
  if (n <= have && p) return TS_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cudaError_t rc = cudaMalloc((void**)&p, std::max<size_t>(n, 1) * sizeof(T));
  if (rc != cudaSuccess) {
    have = 0;
    return cuda_fail(e, rc, what);
  }
  have = n;
  return TS_OK;
}

View make_view(ts_engine* e) {
  View v;
  memset(&v, 0, sizeof(v));
  v.no = e->no;
  v.W = e->W;
  v.Q = e->Q;
  v.prior = e->prior;
  v.reward = e->reward;
  v.mf = e->mf;
  v.parent = e->parent;
  v.cap = e->cap;
  v.st = e->st;
  v.prob = e->prob;
  v.arrival = e->arrival;
  v.ctr = e->ctr;
  v.work = e->work;
  v.work_heavy = e->work_heavy;
  v.tgt = e->tgt;
  v.nrec = e->nrec;
  v.heavy_on = (e->wkind != 3 && !e->heavy_off && e->n_local <= HBITS_WORDS * 32 &&
                 e->cfg.rollout_budget < SQRT_TAB) ? 1 : 0;
  v.heavy_sync = e->heavy_sync ? 1 : 0;
  v.max_arrival = e->max_arrival;
  v.sp = e->sp;
  v.ss = e->ss;
  v.sl = e->sl;
  v.log1p_tab = e->log1p_tab;
  v.log1p_n = e->log1p_n;
  v.checks = e->checks;
  v.free_ok = (e->free_ok && !e->checks && !e->trace && !(e->cost_cap > 0 && e->cost_snap && e->cost_n >= e->n_local))
                  ? 1 : 0;
  v.fdone = e->fdone;
  v.free_kernel = (v.free_ok && !e->free_kernel_off) ? 1 : 0;
  v.trace = e->trace;
  v.trace_cap = e->trace_cap;
  if (e->cost_cap > 0 && e->cost_snap && e->cost_n >= e->n_local) {
    v.cost_pt = e->cost_pt;
    v.cost_rl = e->cost_rl;
    v.cost_cap = e->cost_cap;
    v.cost_snap = e->cost_snap;
    v.sim_done = e->sim_done;
  }
  v.clock_at = e->clock_at;
  v.n_local = e->n_local;
  v.goff = e->goff;
  v.n_global = e->n_global;
  v.step_times = e->step_times;
  v.step_times_cap = e->step_times_cap;
  v.g_runS = e->g_runS;
  v.g_runStart = e->g_runStart;
  v.g_runWant = e->g_runWant;
  v.g_runPW = e->g_runPW;
  v.cfg = e->cfg;
  return v;
}

size_t targets_smem() { return TGT_SCR + 32 * 16 + HBITS_WORDS * 4 + (size_t)2 * RUNCAP * (8 + 4 + 8 + 8); }
size_t sched_smem() { return targets_smem() + (size_t)SREC_MAX * sizeof(ts_sched_record); }

// log1p(k) for k < n from the host libm (the reference calls math.log1p,
// scheduler.py:128, which is the same C library function).
int ensure_log1p(ts_engine* e, int need, cudaStream_t s) {
  if (need <= e->log1p_n) return TS_OK;
  int n = std::max(need, std::max(1024, e->log1p_n * 2));
  std::vector<double> h((size_t)n);
  for (int k = 0; k < n; ++k) h[k] = std::log1p((double)k);
  double* p = nullptr;
  TS_CUDA_TRY(e, cudaMalloc((void**)&p, sizeof(double) * n));
  TS_CUDA_TRY(e, cudaMemcpyAsync(p, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  if (e->log1p_tab) cudaFree(e->log1p_tab);
  e->log1p_tab = p;
  e->log1p_n = n;
  return TS_OK;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_pinned(ts_engine* e, size_t bytes) {
  if (bytes <= e->pin_bytes && e->pin) return TS_OK;
  if (e->pin) cudaFreeHost(e->pin);
  e->pin = nullptr;
  e->pin_bytes = 0;
  TS_CUDA_TRY(e, cudaMallocHost(&e->pin, bytes));
  e->pin_bytes = bytes;
  return TS_OK;
}

int ensure_step_times(ts_engine* e, int need, cudaStream_t s) {
  if (need <= e->step_times_cap) return TS_OK;
  int n = std::max(need, std::max(4096, e->step_times_cap * 2));
  unsigned long long* p = nullptr;
  TS_CUDA_TRY(e, cudaMalloc((void**)&p, sizeof(unsigned long long) * n));
  TS_CUDA_TRY(e, cudaMemsetAsync(p, 0, sizeof(unsigned long long) * n, s));
  if (e->step_times) {
    TS_CUDA_TRY(e, cudaMemcpyAsync(p, e->step_times, sizeof(unsigned long long) * e->step_times_cap,
                                   cudaMemcpyDeviceToDevice, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
    cudaFree(e->step_times);
  }
  e->step_times = p;
  double* ca = nullptr;  // the wave clock per step (cost model), same capacity
  TS_CUDA_TRY(e, cudaMalloc((void**)&ca, sizeof(double) * n));
  TS_CUDA_TRY(e, cudaMemsetAsync(ca, 0, sizeof(double) * n, s));
  if (e->clock_at) {
    TS_CUDA_TRY(e, cudaMemcpyAsync(ca, e->clock_at, sizeof(double) * e->step_times_cap, cudaMemcpyDeviceToDevice, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
    cudaFree(e->clock_at);
  }
  e->clock_at = ca;
  e->step_times_cap = n;
  return TS_OK;
}

// Per-search buffers of the cost model's wave clock (ts_engine_set_cost_model).
int ensure_cost(ts_engine* e) {
  if (e->cost_cap <= 0) return TS_OK;
  if (e->n_global != e->n_local)
    return fail(e, TS_INVALID_ARGUMENT, "the cost model's wave clock needs the whole run queue on one engine");
  if (e->n_local <= e->cost_n) return TS_OK;
  if (e->cost_snap) cudaFree(e->cost_snap);
  if (e->sim_done) cudaFree(e->sim_done);
  e->cost_snap = nullptr;
  e->sim_done = nullptr;
  e->cost_n = 0;
  TS_CUDA_TRY(e, cudaMalloc((void**)&e->cost_snap, sizeof(int2) * (size_t)e->n_local));
  TS_CUDA_TRY(e, cudaMalloc((void**)&e->sim_done, sizeof(double) * (size_t)e->n_local));
  e->cost_n = e->n_local;
  return TS_OK;
}

int validate_config(ts_engine* e, const ts_config& c) {
  if (c.scheme < 0 || c.scheme > 3) return fail(e, TS_INVALID_ARGUMENT, "unknown aggregation scheme");
  if (c.futility_bound < 0 || c.futility_bound > 1) return fail(e, TS_INVALID_ARGUMENT, "unknown futility bound");
  // ScoringConfig.__post_init__ (scoring.py:93-103)
  if (!(c.accept_threshold > 0.0 && c.accept_threshold < 1.0))
    return fail(e, TS_INVALID_ARGUMENT, "accept_threshold out of (0,1)");
  if (!(c.positive_exit_threshold > 0.0 && c.positive_exit_threshold < 1.0))
    return fail(e, TS_INVALID_ARGUMENT, "positive_exit_threshold out of (0,1)");
  if (!(c.first_step_threshold >= 0.0 && c.first_step_threshold < 1.0))
    return fail(e, TS_INVALID_ARGUMENT, "first_step_threshold out of [0,1)");
  // SelectionParams (tree.py:98-100)
  if (!(c.c_puct > 0.0)) return fail(e, TS_INVALID_ARGUMENT, "c_puct must be positive");
  // SchedulerConfig (scheduler.py:85-93)
  if (c.max_concurrency < 1) return fail(e, TS_INVALID_ARGUMENT, "max_concurrency must be >= 1");
  if (!(c.beta > 0.0)) return fail(e, TS_INVALID_ARGUMENT, "beta must be positive");
  if (!(c.proximity > 0.0 && c.proximity < 1.0)) return fail(e, TS_INVALID_ARGUMENT, "proximity must lie in (0,1)");
  if (c.obs_threshold < 1) return fail(e, TS_INVALID_ARGUMENT, "obs_threshold must be >= 1");
  if (c.rollout_budget < 1) return fail(e, TS_INVALID_ARGUMENT, "rollout_budget must be positive");
  if (c.depth_cap < 1) return fail(e, TS_INVALID_ARGUMENT, "depth_cap must be positive");
  if (c.expand_width < 1) return fail(e, TS_INVALID_ARGUMENT, "width must be >= 1");
  // classify_leaf (scoring.py:124-127), raised up front (simulator.py:106-110)
  if (c.negative_exit && c.scheme != TS_SCHEME_MINIMUM && c.scheme != TS_SCHEME_PRODUCT)
    return fail(e, TS_UNSUPPORTED_SCHEME, "negative exit is unsound under this aggregation scheme");
  return TS_OK;
}

int wave_index(ts_engine* e) { return (e->nslot == 1 ? 0 : e->nslot == 2 ? 1 : 2) * 4 + e->wkind; }
size_t wave_smem_of(int wkind) {
  const int ws = wkind == 0 ? 2 : wkind == 1 ? 4 : wkind == 2 ? 8 : TS_MAX_WIDTH;
  return (size_t)WAVE_WARPS * 2 * 32 * ws * sizeof(double);
}

int wave_grid(ts_engine* e, int& blocks_out) {
  const int k = wave_index(e);
  int blocks = e->wave_blocks[k];
  if (blocks <= 0) {
    int per = 0;
    cudaError_t rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)kWave[0][k / 4][k % 4],
                                                                   WAVE_THREADS, wave_smem_of(k % 4));
    if (rc != cudaSuccess) return cuda_fail(e, rc, "occupancy");
    blocks = std::max(1, per) * e->sm_count;
    e->wave_blocks[k] = blocks;
  }
  blocks = std::min(blocks, (e->n_local + WAVE_WARPS - 1) / WAVE_WARPS);
  blocks_out = std::max(blocks, 1);
  return TS_OK;
}

void* wave_fn(ts_engine* e) {
  const int k = wave_index(e);
  return (void*)kWave[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][k % 4];
}

int heavy_grid(ts_engine* e, int& blocks_out) {
  if (e->heavy_blocks <= 0) {
    int per = 0;
    const int k = wave_index(e);
    cudaError_t rc = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per, (const void*)kHeavy[0][k / 4][std::min(k % 4, 2)], HEAVY_THREADS, heavy_smem_of(std::min(e->wkind, 2)));
    if (rc != cudaSuccess) return cuda_fail(e, rc, "occupancy");
    e->heavy_blocks = std::max(1, per) * e->sm_count;
    const char* env = getenv("TS_HEAVY_BLOCKS");  // experiments: fewer resident pipelined-mode CTAs
    if (env && atoi(env) > 0) e->heavy_blocks = std::min(e->heavy_blocks, atoi(env));
  }
  blocks_out = std::max(1, std::min(e->heavy_blocks, e->n_local));
  return TS_OK;
}

void* heavy_fn(ts_engine* e) {
  const int k = wave_index(e);
  return (void*)kHeavy[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][std::min(k % 4, 2)];
}

int launch_heavy(ts_engine* e, const View& v, int step, cudaStream_t s) {
  if (!v.heavy_on) return TS_OK;
  int blocks = 0, rc;
  if ((rc = heavy_grid(e, blocks))) return rc;
  const int k = wave_index(e);
  kHeavy[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][std::min(k % 4, 2)]<<<blocks, HEAVY_THREADS,
                                                                                 heavy_smem_of(std::min(e->wkind, 2)), s>>>(v, step);
  TS_LAUNCH_CHECK(e, "k_heavy");
  return TS_OK;
}

void destroy_run_graph(ts_engine* e) {
  if (e->run_exec) cudaGraphExecDestroy(e->run_exec);
  if (e->run_graph) cudaGraphDestroy(e->run_graph);
  e->run_exec = nullptr;
  e->run_graph = nullptr;
}

// while (cond) { k_sched; k_wave }, cond cleared by k_sched when the batch is done
int build_run_graph(ts_engine* e, const View& v) {
  destroy_run_graph(e);
  int blocks = 0, rc;
  if ((rc = wave_grid(e, blocks))) return rc;
  cudaGraph_t g = nullptr;
  TS_CUDA_TRY(e, cudaGraphCreate(&g, 0));
  e->run_graph = g;
  cudaGraphConditionalHandle h;
  TS_CUDA_TRY(e, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  TS_CUDA_TRY(e, cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  View vv = v;
  ts_sched_record* rec = e->records;
  int use_cond = 1, stepm1 = -1;
  void* a1[] = {(void*)&vv, (void*)&rec, (void*)&h, (void*)&use_cond};
  cudaKernelNodeParams k1;
  memset(&k1, 0, sizeof(k1));
  k1.func = (void*)k_sched;
  k1.gridDim = dim3(1);
  k1.blockDim = dim3(SCHED_T);
  k1.sharedMemBytes = (unsigned)sched_smem();
  k1.kernelParams = a1;
  void* a2[] = {(void*)&vv, (void*)&stepm1};
  void* a4f[] = {(void*)&vv};
  cudaKernelNodeParams k2;
  memset(&k2, 0, sizeof(k2));
  k2.func = wave_fn(e);
  k2.gridDim = dim3(blocks);
  k2.blockDim = dim3(WAVE_THREADS);
  k2.sharedMemBytes = (unsigned)wave_smem_of(e->wkind);
  k2.kernelParams = a2;
  cudaKernelNodeParams kf = k2;
  if (v.free_kernel) {
    const int k = wave_index(e);
    const void* f = kWaveFree[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][k % 4];
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, WAVE_THREADS, wave_smem_of(e->wkind));
    kf.func = (void*)f;
    kf.gridDim = dim3(std::max(1, per) * e->sm_count);
    kf.kernelParams = a4f;
  }
  cudaKernelNodeParams k3 = k2;
  if (v.heavy_on) {
    int hb = 0;
    if ((rc = heavy_grid(e, hb))) return rc;
    k3.func = heavy_fn(e);
    k3.gridDim = dim3(hb);
    k3.blockDim = dim3(HEAVY_THREADS);
    k3.sharedMemBytes = (unsigned)heavy_smem_of(e->wkind);
  }
  // The body holds `graph_unroll` scheduler passes and waves: an edge inside
  // the body is cheaper than the loop's back edge (conditional node + launch).
  // A pass after the batch is done finds nothing to do (empty work lists).
  // invariant checks (ts_engine_set_checks): k_check_pre after the pass,
  // k_check_post after the wave kernels
  void* a4[] = {(void*)&vv};
  cudaKernelNodeParams kc1;
  memset(&kc1, 0, sizeof(kc1));
  kc1.func = (void*)k_check_pre;
  kc1.gridDim = dim3(1);
  kc1.blockDim = dim3(1024);
  kc1.kernelParams = a4;
  cudaKernelNodeParams kc2 = kc1;
  kc2.func = (void*)k_check_post;
  kc2.gridDim = dim3(2 * e->sm_count);
  kc2.blockDim = dim3(256);
  cudaKernelNodeParams kt = kc1;
  kt.func = (void*)k_trace;
  kt.blockDim = dim3(256);
  cudaKernelNodeParams kq1 = kt, kq2 = kc1, kq3 = kt;  // the cost model's wave clock
  kq1.func = (void*)k_cost_pre;
  kq2.func = (void*)k_cost_load;
  kq3.func = (void*)k_cost_wave;
  kq3.gridDim = dim3(2 * e->sm_count);
  cudaGraphNode_t prev[2];
  int nprev = 0;
  for (int u = 0; u < e->graph_unroll; ++u) {
    cudaGraphNode_t n1, n2, n3;
    TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n1, body, nprev ? prev : nullptr, nprev, &k1));
    if (v.checks) {
      cudaGraphNode_t nc;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nc, body, &n1, 1, &kc1));
      n1 = nc;
    }
    if (v.trace) {
      cudaGraphNode_t nt;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nt, body, &n1, 1, &kt));
      n1 = nt;
    }
    if (v.cost_cap) {
      cudaGraphNode_t nq;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nq, body, &n1, 1, &kq1));
      n1 = nq;
    }
    TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n2, body, &n1, 1, &k2));
    prev[0] = n2;
    nprev = 1;
    if (v.free_kernel) {
      cudaGraphNode_t nf;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nf, body, &n1, 1, &kf));
      TS_CUDA_TRY(e, cudaGraphAddDependencies(body, &nf, &n2, 1));
    }
    if (v.heavy_on) {
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n3, body, &n1, 1, &k3));
      prev[1] = n3;
      nprev = 2;
    }
    if (v.checks) {
      cudaGraphNode_t nc;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nc, body, prev, nprev, &kc2));
      prev[0] = nc;
      nprev = 1;
    }
    if (v.cost_cap) {
      cudaGraphNode_t nq2, nq3;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nq2, body, prev, nprev, &kq2));
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&nq3, body, &nq2, 1, &kq3));
      prev[0] = nq3;
      nprev = 1;
    }
  }
  TS_CUDA_TRY(e, cudaGraphInstantiate(&e->run_exec, g, 0));
  e->run_view = v;
  return TS_OK;
}

int launch_wave(ts_engine* e, const View& v, int step, cudaStream_t s) {
  int blocks = 0, rc;
  if ((rc = wave_grid(e, blocks))) return rc;
  if (e->wave_ev_used + 2 > e->wave_ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t ev;
      if (cudaEventCreate(&ev) != cudaSuccess) return fail(e, TS_CUDA, "cudaEventCreate");
      e->wave_ev.push_back(ev);
    }
  }
  if (v.checks) {
    k_check_pre<<<1, 1024, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_check_pre");
  }
  if (v.trace) {
    k_trace<<<1, 256, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_trace");
  }
  if (v.cost_cap) {
    k_cost_pre<<<1, 256, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_cost_pre");
  }
  cudaEventRecord(e->wave_ev[e->wave_ev_used], s);
  const int k = wave_index(e);
  kWave[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][k % 4]<<<blocks, WAVE_THREADS, wave_smem_of(k % 4), s>>>(v, step);
  TS_LAUNCH_CHECK(e, "k_wave");
  if (v.free_kernel && step < 0) {  // host-driven loop: the free-running waves' kernel (returns unless k_sched chose them)
    const void* f = kWaveFree[e->cfg.scheme == TS_SCHEME_PRODUCT ? 1 : 0][k / 4][k % 4];
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, WAVE_THREADS, wave_smem_of(k % 4));
    View vf = v;
    void* args[] = {(void*)&vf};
    TS_CUDA_TRY(e, cudaLaunchKernel(f, dim3(std::max(1, per) * e->sm_count), dim3(WAVE_THREADS), args,
                                    wave_smem_of(k % 4), s));
    TS_LAUNCH_CHECK(e, "k_wave_free");
  }
  if ((rc = launch_heavy(e, v, step, s))) return rc;
  cudaEventRecord(e->wave_ev[e->wave_ev_used + 1], s);
  e->wave_ev_used += 2;
  if (v.checks) {
    k_check_post<<<2 * e->sm_count, 256, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_check_post");
  }
  if (v.cost_cap) {
    k_cost_load<<<1, 1024, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_cost_load");
    k_cost_wave<<<2 * e->sm_count, 256, 0, s>>>(v);
    TS_LAUNCH_CHECK(e, "k_cost_wave");
  }
  return TS_OK;
}

void destroy_px_graph(ts_engine* e) {
  if (e->px_exec) cudaGraphExecDestroy(e->px_exec);
  if (e->px_graph) cudaGraphDestroy(e->px_graph);
  e->px_exec = nullptr;
  e->px_graph = nullptr;
}

void xchg_release(ts_engine* e) {
  destroy_px_graph(e);
  for (int p = 0; p < TS_MAX_PEERS; ++p) {
    if (e->xipc[p] && e->xpeer[p]) cudaIpcCloseMemHandle(e->xpeer[p]);
    e->xipc[p] = false;
    e->xpeer[p] = nullptr;
  }
  if (e->xbuf) cudaFree(e->xbuf);
  if (e->xstamp) cudaFree(e->xstamp);
  if (e->xscr) cudaFree(e->xscr);
  e->xbuf = nullptr;
  e->xstamp = nullptr;
  e->xscr = nullptr;
  e->xbytes = 0;
  e->xconnected = false;
}

// while (cond) { counts -> admit -> records -> wait -> compute_targets -> waves }:
// ts_run's loop with the scheduler's global terms exchanged over peer memory
View px_make_view(ts_engine* e) {
  View v = make_view(e);
  for (int p = 0; p < e->xworld; ++p) v.px[p] = e->xpeer[p];
  v.pworld = e->xworld;
  v.prank = e->xrank;
  v.padm_all = (long long)e->cfg.max_concurrency < (long long)e->n_global ? 1 : 0;
  v.pstamp = e->xstamp;
  v.pscr = e->xscr;
  v.pgwarp = e->px_gwarp;
  return v;
}

int build_px_graph(ts_engine* e, const View& v, int max_steps) {
  destroy_px_graph(e);
  int blocks = 0, rc;
  if ((rc = wave_grid(e, blocks))) return rc;
  cudaGraph_t g = nullptr;
  TS_CUDA_TRY(e, cudaGraphCreate(&g, 0));
  e->px_graph = g;
  cudaGraphConditionalHandle h;
  TS_CUDA_TRY(e, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  TS_CUDA_TRY(e, cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  View vv = v;
  int ms = max_steps, stepm1 = -1;
  void* a_v[] = {(void*)&vv};
  void* a_vc[] = {(void*)&vv, (void*)&h};
  void* a_vcm[] = {(void*)&vv, (void*)&h, (void*)&ms};
  void* a_wave[] = {(void*)&vv, (void*)&stepm1};
  auto kp = [](void* f, dim3 grid, dim3 block, size_t sm, void** args) {
    cudaKernelNodeParams k;
    memset(&k, 0, sizeof(k));
    k.func = f;
    k.gridDim = grid;
    k.blockDim = block;
    k.sharedMemBytes = (unsigned)sm;
    k.kernelParams = args;
    return k;
  };
  std::vector<cudaKernelNodeParams> chain;
  chain.push_back(kp((void*)k_px_counts, dim3(1), dim3(32), 0, a_v));
  chain.push_back(kp((void*)k_px_admit, dim3(1), dim3(32), 0, a_vcm));
  if (e->n_local <= 16 * PXS && !e->px_two_kernels) {
    // the whole exchange and scheduler pass in one kernel
    chain.clear();
    const int jpt = (e->n_local + PXS - 1) / PXS;
    void* f = jpt <= 1 ? (void*)k_px_step<1> : jpt <= 2 ? (void*)k_px_step<2> : jpt <= 4 ? (void*)k_px_step<4>
            : jpt <= 8 ? (void*)k_px_step<8> : (void*)k_px_step<16>;
    chain.push_back(kp(f, dim3(1), dim3(PXS), px_step_smem(), a_vcm));
  } else {
    chain.push_back(kp((void*)k_px_groups, dim3(1), dim3(PXT), 0, a_v));
    chain.push_back(kp((void*)k_px_sched, dim3(1), dim3(PXT), 0, a_vc));
  }
  cudaKernelNodeParams kw = kp(wave_fn(e), dim3(blocks), dim3(WAVE_THREADS), wave_smem_of(e->wkind), a_wave);
  cudaKernelNodeParams kh = kw;
  if (v.heavy_on) {
    int hb = 0;
    if ((rc = heavy_grid(e, hb))) return rc;
    kh = kp(heavy_fn(e), dim3(hb), dim3(HEAVY_THREADS), heavy_smem_of(e->wkind), a_wave);
  }
  cudaGraphNode_t prev[2];
  int nprev = 0;
  for (int u = 0; u < e->graph_unroll; ++u) {
    for (const cudaKernelNodeParams& k : chain) {
      cudaGraphNode_t n;
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n, body, nprev ? prev : nullptr, nprev, &k));
      prev[0] = n;
      nprev = 1;
    }
    const cudaGraphNode_t sched = prev[0];
    cudaGraphNode_t n2, n3;
    TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n2, body, &sched, 1, &kw));
    prev[0] = n2;
    nprev = 1;
    if (v.heavy_on) {
      TS_CUDA_TRY(e, cudaGraphAddKernelNode(&n3, body, &sched, 1, &kh));
      prev[1] = n3;
      nprev = 2;
    }
  }
  TS_CUDA_TRY(e, cudaGraphInstantiate(&e->px_exec, g, 0));
  e->px_view = v;
  e->px_max_steps = max_steps;
  return TS_OK;
}

void host_stats(const Counters& c, ts_run_stats* o) {
  o->steps = (int32_t)(c.last_exit_step + 1);
  o->finished = (int32_t)c.finished;
  o->rollouts = (int64_t)c.rollouts;
  o->launched = (int64_t)c.launched;
  o->nodes = (int64_t)c.nodes;
  o->children_scored = (int64_t)c.scored;
  o->select_levels = (int64_t)c.levels;
  o->path_nodes = (int64_t)c.path_nodes;
  o->kernel_launches = 0;
  o->tokens = (int64_t)c.tokens;
}

}  // namespace

extern "C" {

int ts_abi_version(void) { return TS_ABI_VERSION; }

const char* ts_last_error(const ts_engine* eng) { return eng ? eng->err.c_str() : "null engine"; }

int ts_engine_create(const ts_config* cfg, int32_t device, ts_engine** out) {
  if (!cfg || !out) return TS_INVALID_ARGUMENT;
  *out = nullptr;
  ts_engine* e = new ts_engine();
  int rc = validate_config(e, *cfg);
  if (rc != TS_OK) {
    // keep the engine so the caller can read the message, then destroy it
    *out = e;
    return rc;
  }
  e->cfg = *cfg;
  e->device = device;
  cudaError_t cr = cudaSetDevice(device);
  if (cr != cudaSuccess) {
    *out = e;
    return cuda_fail(e, cr, "cudaSetDevice");
  }
  cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, device);
  cr = cudaMalloc((void**)&e->ctr, sizeof(Counters));
  if (cr == cudaSuccess) cr = cudaMalloc((void**)&e->counts, sizeof(long long) * 3);
  if (cr == cudaSuccess)
    cr = cudaFuncSetAttribute(k_targets, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)targets_smem());
  if (cr == cudaSuccess)
    cr = cudaFuncSetAttribute(k_sched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sched_smem());
  {
    void* fs[] = {(void*)k_px_step<1>, (void*)k_px_step<2>, (void*)k_px_step<4>, (void*)k_px_step<8>,
                  (void*)k_px_step<16>};
    for (void* f : fs)
      if (cr == cudaSuccess) cr = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)px_step_smem());
  }
  for (int a = 0; a < 3 && cr == cudaSuccess; ++a)
    for (int b = 0; b < 4 && cr == cudaSuccess; ++b)
      for (int pr = 0; pr < 2 && cr == cudaSuccess; ++pr)
        cr = cudaFuncSetAttribute(kWaveFree[pr][a][b], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)wave_smem_of(b));
  for (int a = 0; a < 3 && cr == cudaSuccess; ++a)
    for (int b = 0; b < 4 && cr == cudaSuccess; ++b)
      for (int pr = 0; pr < 2 && cr == cudaSuccess; ++pr)
        cr = cudaFuncSetAttribute((const void*)kWave[pr][a][b], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)wave_smem_of(b));
  for (int a = 0; a < 3 && cr == cudaSuccess; ++a)
    for (int b = 0; b < 3 && cr == cudaSuccess; ++b)
      for (int pr = 0; pr < 2 && cr == cudaSuccess; ++pr)
        cr = cudaFuncSetAttribute((const void*)kHeavy[pr][a][b], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)heavy_smem_of(b));
  {
    const char* env = getenv("TS_NO_PIPELINE");
    e->heavy_off = env && env[0] == '1';
    const char* env2 = getenv("TS_PIPELINE_SYNC");
    const char* env3 = getenv("TS_MT_MIN");
    if (env3) e->mt_min = atoi(env3);
    int coop = 0, per = 0, sms = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k_mt_all, MT_T, 0) != cudaSuccess) per = 0;
    const char* env4 = getenv("TS_MT_COOP");
    e->coop_ctas = (coop && !(env4 && env4[0] == '0')) ? per * sms : 0;
    cudaGetLastError();
    e->heavy_sync = env2 && env2[0] == '1';
    const char* env5 = getenv("TS_NO_GRAPH");  // host-driven stepping (diagnostics: ncu cannot see graph kernels)
    e->graph_failed = env5 && env5[0] == '1';
    const char* envf = getenv("TS_NO_FREE");
    e->free_off = envf && envf[0] == '1';
    const char* envk = getenv("TS_NO_FREE_KERNEL");
    e->free_kernel_off = envk && envk[0] == '1';
    const char* env8 = getenv("TS_PX_TWO_KERNELS");
    e->px_two_kernels = env8 && env8[0] == '1';
    const char* env9 = getenv("TS_PX_GWARP");
    if (env9) e->px_gwarp = std::max(0, std::min(32, atoi(env9)));
    const char* env6 = getenv("TS_GRAPH_UNROLL");
    if (env6) e->graph_unroll = std::max(1, std::min(8, atoi(env6)));
  }
  if (cr != cudaSuccess) {
    *out = e;
    return cuda_fail(e, cr, "engine allocation");
  }
  *out = e;
  return TS_OK;
}

int ts_engine_destroy(ts_engine* e) {
  if (!e) return TS_OK;
  void* ptrs[] = {e->no, e->W, e->Q, e->prior, e->reward, e->mf, e->parent, e->st, e->prob,
                  e->arrival, e->ctr, e->work, e->sp, e->ss, e->sl, e->log1p_tab, e->step_times,
                  e->g_runS, e->g_runStart, e->g_runWant, e->g_runPW, e->counts, e->records, e->outcomes,
                  e->work_heavy, e->mt, e->tgt, e->nrec, e->trace, e->cost_snap, e->sim_done,
                  e->clock_at, e->fdone};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (cudaEvent_t ev : e->wave_ev) cudaEventDestroy(ev);
  destroy_run_graph(e);
  xchg_release(e);
  if (e->pin) cudaFreeHost(e->pin);
  if (e->pin_out) cudaFreeHost(e->pin_out);
  if (e->pin_ctr) cudaFreeHost(e->pin_ctr);
  delete e;
  return TS_OK;
}

int ts_load_problems(ts_engine* e, const ts_problem* hp, int32_t n_local, int32_t global_offset,
                     int32_t n_global, void* stream) {
  if (!e) return TS_INVALID_ARGUMENT;
  if (!hp || n_local < 1) return fail(e, TS_INVALID_ARGUMENT, "need at least one problem");
  if (global_offset < 0 || n_global < global_offset + n_local)
    return fail(e, TS_INVALID_ARGUMENT, "bad shard placement");
  cudaStream_t s = (cudaStream_t)stream;
  TS_CUDA_TRY(e, cudaSetDevice(e->device));
  const ts_config& c = e->cfg;
  int rc;
  // The problem table's DMA is enqueued first and the host validates the
  // table while it is in flight (one pass over the rows; a strided host pass
  // costs about as much as the copy itself).  A table that fails validation
  // leaves the engine unloaded.
  if (n_local > e->cap_searches || !e->st) {
    size_t h0 = 0, h1 = 0, h2 = 0, h3 = 0, h4 = 0, h5 = 0, h6 = 0, h7 = 0, h8 = 0;
    e->loaded = false;
    if ((rc = grow(e, e->st, n_local, h0, "search state")) ||
        (rc = grow(e, e->prob, n_local, h1, "problem table")) ||
        (rc = grow(e, e->arrival, n_local, h2, "arrivals")) ||
        (rc = grow(e, e->work, n_local, h3, "work list")) ||
        (rc = grow(e, e->work_heavy, n_local, h6, "work list")) ||
        (rc = grow(e, e->tgt, n_local, h7, "targets")) ||
        (rc = grow(e, e->nrec, n_local, h8, "records")) ||
        (rc = grow(e, e->records, n_local, h4, "records")) ||
        (rc = grow(e, e->outcomes, n_local, h5, "outcomes")))
      return rc;
    e->cap_searches = n_local;
    e->outcomes_cap = n_local;
  }
  {
    // one DMA at full PCIe rate: directly from pinned caller memory, else via pinned staging
    const size_t bytes = sizeof(ts_problem) * (size_t)n_local;
    e->loaded = false;
    if (is_pinned(hp)) {
      TS_CUDA_TRY(e, cudaMemcpyAsync(e->prob, hp, bytes, cudaMemcpyHostToDevice, s));
    } else {
      if ((rc = ensure_pinned(e, bytes))) return rc;
      TS_CUDA_TRY(e, cudaStreamSynchronize(s));  // the staging buffer may still feed an earlier copy
      memcpy(e->pin, hp, bytes);
      TS_CUDA_TRY(e, cudaMemcpyAsync(e->prob, e->pin, bytes, cudaMemcpyHostToDevice, s));
    }
  }
  int max_len = 1, max_width = 1, prev_arr = 0;
  int wmin = TS_MAX_WIDTH, dmin = TS_MAX_DEPTH;
  const int w0 = std::min(c.expand_width, hp[0].branching);
  bool same = true;
  for (int i = 0; i < n_local; ++i) {
    const ts_problem& p = hp[i];
    if (p.branching < 1 || p.branching > TS_MAX_WIDTH)
      return fail(e, TS_INVALID_ARGUMENT, "branching must lie in [1, 32]");
    if (p.base_depth < 1 || p.base_depth > TS_MAX_DEPTH - 1)
      return fail(e, TS_INVALID_ARGUMENT, "base_depth must lie in [1, 31]");
    if (p.golden_len > p.base_depth) return fail(e, TS_INVALID_ARGUMENT, "golden path longer than base depth");
    if (p.arrival_step < 0 || p.arrival_step < prev_arr)
      return fail(e, TS_INVALID_ARGUMENT, "arrival steps must be non-negative and non-decreasing");
    prev_arr = p.arrival_step;
    const int w = std::min(c.expand_width, p.branching);
    max_len = std::max(max_len, std::min(c.depth_cap, p.base_depth + 1));
    max_width = std::max(max_width, w);
    wmin = std::min(wmin, w);
    dmin = std::min(dmin, std::min(c.depth_cap, p.base_depth));
    same = same && w == w0;
  }
  e->max_arrival = prev_arr;
  e->nslot = max_len <= 8 ? 1 : max_len <= 16 ? 2 : 4;
  {
    // Exhausting a root needs every node of depth Dmin-1 = min(base_depth,
    // depth_cap)-1 expanded (nodes above never become terminal or forced),
    // one per rollout: impossible within the budget if budget < w^(Dmin-1).
    double need = 1.0;
    for (int d = 1; d < dmin; ++d) need *= (double)wmin;
    // with boosting on, P = 1 for every running search needs no free slot: a
    // run queue smaller than max_concurrency never free-runs
    e->free_ok = !e->free_off && !c.positive_exit && !c.negative_exit && wmin >= 2 &&
                 (double)c.rollout_budget < need && n_global == n_local &&
                 (!c.boosting_enabled || (long long)c.max_concurrency <= (long long)n_local);
    if (e->fdone_cap < n_local) {
      if (e->fdone) cudaFree(e->fdone);
      e->fdone = nullptr;
      e->fdone_cap = 0;
      TS_CUDA_TRY(e, cudaMalloc((void**)&e->fdone, sizeof(int32_t) * (size_t)std::max(1, n_local)));
      e->fdone_cap = n_local;
    }
  }
  e->wkind = same ? wkind_of_width(w0) : 3;
  // nodes a search can create: every launched rollout (<= budget) expands at
  // most min(depth_cap, base_depth+1) levels of `width` children
  const long long cap = 1 + (long long)c.rollout_budget * max_width * max_len;
  const size_t pool = (size_t)cap * (size_t)n_local;
  if (pool > (size_t)e->pool_nodes || !e->no) {
    void* ptrs[] = {e->no, e->W, e->Q, e->prior, e->reward, e->mf, e->parent};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    e->no = nullptr; e->W = nullptr; e->Q = nullptr; e->prior = nullptr; e->reward = nullptr;
    e->mf = nullptr; e->parent = nullptr;
    e->pool_nodes = 0;
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->no, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->W, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->Q, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->prior, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->reward, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->mf, pool * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->parent, pool * 4));
    e->pool_nodes = (long long)pool;
  }
  e->cap = cap;
  const size_t rows = (size_t)n_local * (size_t)c.rollout_budget;
  if (rows > e->scratch_rows || !e->sp) {
    if (e->sp) cudaFree(e->sp);
    if (e->ss) cudaFree(e->ss);
    if (e->sl) cudaFree(e->sl);
    e->sp = nullptr; e->ss = nullptr; e->sl = nullptr;
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->sp, rows * 32 * 4));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->ss, rows * 8));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->sl, rows * 4));
    e->scratch_rows = rows;
  }
  if (n_global > e->cap_global || !e->g_runS) {
    size_t a = 0, b = 0, cc = 0, d = 0;
    if ((rc = grow(e, e->g_runS, (size_t)2 * n_global, a, "runs")) ||
        (rc = grow(e, e->g_runStart, (size_t)2 * n_global, b, "runs")) ||
        (rc = grow(e, e->g_runWant, (size_t)2 * n_global, cc, "runs")) ||
        (rc = grow(e, e->g_runPW, (size_t)2 * n_global, d, "runs")))
      return rc;
    e->cap_global = n_global;
  }
  {
    const size_t need = mt_layout(nullptr, n_global, n_local, nullptr);
    if (need > e->mt_bytes) {
      if (e->mt) cudaFree(e->mt);
      e->mt = nullptr;
      TS_CUDA_TRY(e, cudaMalloc((void**)&e->mt, need));
      e->mt_bytes = need;
    }
  }
  e->n_local = n_local;
  e->goff = global_offset;
  e->n_global = n_global;
  if ((rc = ensure_log1p(e, 1024, s))) return rc;
  if ((rc = ensure_step_times(e, 4096, s))) return rc;
  if ((rc = ensure_cost(e))) return rc;
  View v = make_view(e);
  e->launches = 0;
  e->wave_ev_used = 0;
  // 64-thread CTAs: the root records are scattered stores, spread them over more SMs
  k_init<<<(n_local + 63) / 64, 64, 0, s>>>(v);
  TS_LAUNCH_CHECK(e, "k_init");
  e->loaded = true;
  return TS_OK;
}

int ts_step_counts(ts_engine* e, int32_t step, int64_t* dev_counts, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!dev_counts || step < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  View v = make_view(e);
  k_counts<<<1, 1, 0, (cudaStream_t)stream>>>(v, step, (long long*)dev_counts);
  TS_LAUNCH_CHECK(e, "k_counts");
  return TS_OK;
}

int ts_step_admit(ts_engine* e, int32_t step, const int64_t* dev_all_counts, int32_t world, int32_t rank,
                  void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!dev_all_counts || world < 1 || rank < 0 || rank >= world || step < 0)
    return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  View v = make_view(e);
  k_admit<<<1, 1, 0, (cudaStream_t)stream>>>(v, (const long long*)dev_all_counts, world, rank);
  TS_LAUNCH_CHECK(e, "k_admit");
  return TS_OK;
}

int ts_step_records(ts_engine* e, int32_t step, ts_sched_record* dev_records, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!dev_records || step < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure_log1p(e, step + 1, s))) return rc;
  View v = make_view(e);
  k_records<<<(e->n_local + 255) / 256, 256, 0, s>>>(v, step, dev_records);
  TS_LAUNCH_CHECK(e, "k_records");
  return TS_OK;
}

int ts_step_targets(ts_engine* e, int32_t step, const ts_sched_record* dev_all, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!dev_all || step < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure_step_times(e, step + 1, s))) return rc;
  View v = make_view(e);
  if (v.n_global <= e->mt_min) {
    k_targets<<<1, SCHED_T, targets_smem(), s>>>(v, step, dev_all);
    TS_LAUNCH_CHECK(e, "k_targets");
    return TS_OK;
  }
  // many CTAs: the run queue of a multi-GPU job (every rank scans all records)
  const int G = mt_blocks(v.n_global), G3 = mt_run_blocks(v.n_global);
  unsigned char* mt = e->mt;
  if (G <= e->coop_ctas) {  // one cooperative launch, grid-wide barriers between phases
    void* args[] = {(void*)&v, (void*)&step, (void*)&dev_all, (void*)&mt};
    const cudaError_t rc2 = cudaLaunchCooperativeKernel((const void*)k_mt_all, dim3(G), dim3(MT_T), args, 0, s);
    if (rc2 == cudaSuccess) {
      TS_LAUNCH_CHECK(e, "k_mt_all");
      return TS_OK;
    }
    cudaGetLastError();
    e->coop_ctas = 0;  // not available: per-phase kernels from now on
  }
  k_mt_count<<<G, MT_T, 0, s>>>(v, step, dev_all, mt);
  k_mt_scan1<<<1, 1024, 0, s>>>(v, dev_all, mt);
  k_mt_runs<<<G, MT_T, 0, s>>>(v, dev_all, mt);
  k_mt_scan2<<<1, 1024, 0, s>>>(v, mt);
  k_mt_write_runs<<<G, MT_T, 0, s>>>(v, dev_all, mt);
  k_mt_want<<<G3, MT_T, 0, s>>>(v, mt);
  k_mt_scan3<<<1, 1024, 0, s>>>(v, mt);
  k_mt_targets<<<G, MT_T, 0, s>>>(v, dev_all, mt);
  k_mt_split<<<1, TT, 0, s>>>(v, step, dev_all, mt);
  e->launches += 8;
  TS_LAUNCH_CHECK(e, "k_mt_*");
  return TS_OK;
}

int ts_step_set_targets(ts_engine* e, int32_t step, const int32_t* dev_targets, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!dev_targets || step < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if ((rc = ensure_step_times(e, step + 1, s))) return rc;
  View v = make_view(e);
  k_set_targets<<<1, TT, 0, s>>>(v, step, dev_targets);
  TS_LAUNCH_CHECK(e, "k_set_targets");
  return TS_OK;
}

int ts_read_jobs(ts_engine* e, int32_t* dev_running, int32_t* dev_completed, double* dev_best, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  View v = make_view(e);
  if (v.n_local == 0) return TS_OK;
  k_read_jobs<<<(v.n_local + 255) / 256, 256, 0, (cudaStream_t)stream>>>(v, dev_running, dev_completed, dev_best);
  TS_LAUNCH_CHECK(e, "k_read_jobs");
  return TS_OK;
}

int ts_step_wave(ts_engine* e, int32_t step, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  View v = make_view(e);
  return launch_wave(e, v, step, (cudaStream_t)stream);
}

// ts_run, and with host_out the outcome readout too: k_outcomes and both
// device-to-host copies (outcomes, counters; pinned) are queued behind the
// graph launch so the batch ends in one stream synchronisation.
static int run_impl(ts_engine* e, int32_t max_steps, ts_run_stats* stats_out, cudaStream_t s, ts_outcome* host_out,
             int32_t n_out) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (max_steps < 0) return fail(e, TS_INVALID_ARGUMENT, "max_steps must be >= 0");
  int rc;
  const size_t out_bytes = sizeof(ts_outcome) * (size_t)std::max(0, n_out);
  const bool out_direct = host_out && is_pinned(host_out);
  if (host_out && n_out > 0 && !out_direct && out_bytes > e->pin_out_bytes) {
    if (e->pin_out) cudaFreeHost(e->pin_out);
    e->pin_out = nullptr;
    e->pin_out_bytes = 0;
    TS_CUDA_TRY(e, cudaMallocHost(&e->pin_out, out_bytes));
    e->pin_out_bytes = out_bytes;
  }
  if (!e->pin_ctr) TS_CUDA_TRY(e, cudaMallocHost((void**)&e->pin_ctr, sizeof(Counters)));
  if ((rc = ensure_log1p(e, 1 << 16, s))) return rc;
  if ((rc = ensure_step_times(e, e->log1p_n + 1, s))) return rc;
  Counters c;
  long long step0 = 0;  // device scheduler-pass count before this graph launch
  for (;;) {
    k_set_max_steps<<<1, 1, 0, s>>>(e->ctr, max_steps);
    TS_LAUNCH_CHECK(e, "k_set_max_steps");
    View v = make_view(e);
    bool graphed = false;
    if (!e->graph_failed) {
      if (!e->run_exec || memcmp(&v, &e->run_view, sizeof(View)) != 0) {
        if (build_run_graph(e, v) != TS_OK) {
          destroy_run_graph(e);
          e->graph_failed = true;
          cudaGetLastError();
        }
      }
      if (e->run_exec) {
        TS_CUDA_TRY(e, cudaGraphLaunch(e->run_exec, s));
        graphed = true;
      }
    }
    if (!graphed) {
      // host-driven stepping (same kernels) when conditional graphs are unavailable
      int blocks = 0;
      if ((rc = wave_grid(e, blocks))) return rc;
      for (int it = 0;; ++it) {
        k_sched<<<1, SCHED_T, sched_smem(), s>>>(v, e->records, cudaGraphConditionalHandle(), 0);
        TS_LAUNCH_CHECK(e, "k_sched");
        if ((rc = launch_wave(e, v, -1, s))) return rc;
        if (it % 8 == 7) {
          TS_CUDA_TRY(e, cudaMemcpyAsync(&c, e->ctr, sizeof(c), cudaMemcpyDeviceToHost, s));
          TS_CUDA_TRY(e, cudaStreamSynchronize(s));
          if (c.finished >= e->n_local || c.step >= max_steps || c.step >= e->log1p_n) break;
        }
      }
    }  // graphed: the loop's kernels are counted from the device step count below
    if (host_out && n_out > 0) {
      k_outcomes<<<(n_out + 127) / 128, 128, 0, s>>>(v, e->outcomes, n_out);
      TS_LAUNCH_CHECK(e, "k_outcomes");
      TS_CUDA_TRY(e, cudaMemcpyAsync(out_direct ? (void*)host_out : e->pin_out, e->outcomes, out_bytes,
                                     cudaMemcpyDeviceToHost, s));
    }
    TS_CUDA_TRY(e, cudaMemcpyAsync(e->pin_ctr, e->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
    c = *e->pin_ctr;
    if (graphed) {
      // every iteration runs graph_unroll passes of {k_sched, k_wave[, k_heavy]}; the
      // last one contains the pass that ended the loop
      const long long iters = (c.passes - step0) / e->graph_unroll + 1;
      e->launches += iters * e->graph_unroll * ((v.heavy_on ? 3 : 2) + (v.free_kernel ? 1 : 0) + (v.checks ? 2 : 0) +
                                                (v.trace ? 1 : 0) + (v.cost_cap ? 3 : 0));
    }
    step0 = c.passes;
    if (c.finished >= e->n_local || c.step >= max_steps) break;
    // the log1p table bounds the device loop: grow it and continue
    if ((rc = ensure_log1p(e, e->log1p_n * 2, s))) return rc;
    if ((rc = ensure_step_times(e, e->log1p_n + 1, s))) return rc;
  }
  if (stats_out) {
    // the counters were read after the last launch above: no second round trip
    host_stats(c, stats_out);
    stats_out->kernel_launches = e->launches;
    stats_out->wave_ms = 0.0;
    if (c.sched_error) return fail(e, TS_INVALID_ARGUMENT, "run queue scores not ordered by arrival");
  }
  if (host_out && n_out > 0 && !out_direct) memcpy(host_out, e->pin_out, out_bytes);
  return TS_OK;
}

int ts_run(ts_engine* e, int32_t max_steps, ts_run_stats* stats_out, void* stream) {
  return run_impl(e, max_steps, stats_out, (cudaStream_t)stream, nullptr, 0);
}

int ts_read_stats(ts_engine* e, ts_run_stats* o, void* stream) {
  if (!e || !o) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  Counters c;
  TS_CUDA_TRY(e, cudaMemcpyAsync(&c, e->ctr, sizeof(c), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  TS_CUDA_TRY(e, cudaStreamSynchronize((cudaStream_t)stream));
  host_stats(c, o);
  o->kernel_launches = e->launches;
  o->wave_ms = 0.0;
  for (size_t i = 0; i + 1 < e->wave_ev_used; i += 2) {
    float ms = 0.f;
    TS_CUDA_TRY(e, cudaEventSynchronize(e->wave_ev[i + 1]));
    TS_CUDA_TRY(e, cudaEventElapsedTime(&ms, e->wave_ev[i], e->wave_ev[i + 1]));
    o->wave_ms += ms;
  }
  if (c.sched_error) return fail(e, TS_INVALID_ARGUMENT, "run queue scores not ordered by arrival");
  return TS_OK;
}

int ts_read_outcomes(ts_engine* e, ts_outcome* host_out, int32_t n, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!host_out || n < 0 || n > e->n_local) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  View v = make_view(e);
  k_outcomes<<<(n + 127) / 128, 128, 0, s>>>(v, e->outcomes, n);
  TS_LAUNCH_CHECK(e, "k_outcomes");
  const size_t bytes = sizeof(ts_outcome) * (size_t)n;
  if (is_pinned(host_out)) {
    TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, e->outcomes, bytes, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  } else {
    int rc;
    if ((rc = ensure_pinned(e, bytes))) return rc;
    TS_CUDA_TRY(e, cudaMemcpyAsync(e->pin, e->outcomes, bytes, cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
    memcpy(host_out, e->pin, bytes);
  }
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  return TS_OK;
}

int ts_read_targets(ts_engine* e, int32_t* host_out, int32_t n, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!host_out || n < 0 || n > e->n_local) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, e->tgt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  return TS_OK;
}

#if defined(TS_HEAVY_PROF) || defined(TS_SCHED_PROF) || defined(TS_PX_PROF)
// diagnostics build only (not part of the C-ABI): the phase counters
int ts_debug_prof(ts_engine* e, uint64_t* host16) {
  Counters c;
  TS_CUDA_TRY(e, cudaMemcpy(&c, e->ctr, sizeof(c), cudaMemcpyDeviceToHost));
  memcpy(host16, c.prof, sizeof(c.prof));
  return TS_OK;
}
#endif

int ts_read_latencies(ts_engine* e, uint64_t* host_out, int32_t n, void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!host_out || n < 0 || n > e->n_local) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (n == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  View v = make_view(e);
  // scratch: the outcome buffer is large enough (sizeof(ts_outcome) >= 8)
  unsigned long long* d = (unsigned long long*)e->outcomes;
  k_latency<<<(n + 255) / 256, 256, 0, s>>>(v, d, n);
  TS_LAUNCH_CHECK(e, "k_latency");
  TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  return TS_OK;
}

int ts_read_step_times(ts_engine* e, uint64_t* host_out, int32_t n, void* stream) {
  if (!e || !host_out || n < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  n = std::min(n, e->step_times_cap);
  cudaStream_t s = (cudaStream_t)stream;
  TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, e->step_times, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  return TS_OK;
}

int ts_run_batch_host(ts_engine* e, const ts_problem* hp, int32_t n, int32_t max_steps, ts_outcome* host_out,
                      ts_run_stats* stats_out, void* stream) {
  int rc;
  if ((rc = ts_load_problems(e, hp, n, 0, n, stream))) return rc;
  if (!host_out) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  return run_impl(e, max_steps, stats_out, (cudaStream_t)stream, host_out, n);
}

int ts_tree_size(ts_engine* e, int32_t search, int32_t* nodes_out) {
  if (!e || !e->loaded || !nodes_out || search < 0 || search >= e->n_local)
    return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  SearchState st;
  TS_CUDA_TRY(e, cudaMemcpy(&st, e->st + search, sizeof(st), cudaMemcpyDeviceToHost));
  *nodes_out = st.nodes;
  return TS_OK;
}

int ts_dump_tree(ts_engine* e, int32_t search, int32_t* parent, double* reward, double* prior, int32_t* visits,
                 int32_t* inflight, double* value_sum, uint8_t* terminal, int32_t* depth, int32_t* step_ref) {
  int32_t n = 0;
  int rc = ts_tree_size(e, search, &n);
  if (rc) return rc;
  const size_t b = (size_t)search * (size_t)e->cap;
  std::vector<uint64_t> no(n);
  std::vector<uint64_t> me(n);
  TS_CUDA_TRY(e, cudaMemcpy(no.data(), e->no + b, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  TS_CUDA_TRY(e, cudaMemcpy(me.data(), e->mf + b, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  if (parent) TS_CUDA_TRY(e, cudaMemcpy(parent, e->parent + b, 4 * (size_t)n, cudaMemcpyDeviceToHost));
  if (reward) TS_CUDA_TRY(e, cudaMemcpy(reward, e->reward + b, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  if (prior) TS_CUDA_TRY(e, cudaMemcpy(prior, e->prior + b, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  if (value_sum) TS_CUDA_TRY(e, cudaMemcpy(value_sum, e->W + b, 8 * (size_t)n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) {
    if (visits) visits[i] = (int32_t)(uint32_t)no[i];
    if (inflight) inflight[i] = (int32_t)(no[i] >> 32);
    const uint32_t m = (uint32_t)me[i];
    if (terminal) terminal[i] = (m & M_TERM) ? 1 : 0;
    if (depth) depth[i] = (int32_t)(m & M_DEPTH);
    if (step_ref) step_ref[i] = i == 0 ? -1 : (int32_t)((m >> SH_REF) & 31u);
  }
  return TS_OK;
}

int ts_engine_set_checks(ts_engine* e, int32_t enable) {
  if (!e) return TS_INVALID_ARGUMENT;
  e->checks = enable ? 1 : 0;
  return TS_OK;
}

int ts_engine_set_trace(ts_engine* e, int64_t capacity) {
  if (!e || capacity < 0) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (e->trace) cudaFree(e->trace);
  e->trace = nullptr;
  e->trace_cap = 0;
  if (capacity > 0) {
    TS_CUDA_TRY(e, cudaSetDevice(e->device));
    TS_CUDA_TRY(e, cudaMalloc((void**)&e->trace, sizeof(ts_trace_row) * (size_t)capacity));
    e->trace_cap = capacity;
  }
  return TS_OK;
}

int ts_engine_set_cost_model(ts_engine* e, double per_token_latency, int32_t engine_capacity,
                             double reward_latency) {
  if (!e) return TS_INVALID_ARGUMENT;
  if (engine_capacity == 0) {
    e->cost_cap = 0;
    return TS_OK;
  }
  // CostModel.__post_init__ (backend.py:299-301)
  if (!(per_token_latency > 0) || engine_capacity < 1 || !(reward_latency >= 0))
    return fail(e, TS_INVALID_ARGUMENT, "cost model parameters must be positive");
  if (e->loaded && e->n_global != e->n_local)
    return fail(e, TS_INVALID_ARGUMENT, "the cost model's wave clock needs the whole run queue on one engine");
  e->cost_pt = per_token_latency;
  e->cost_cap = engine_capacity;
  e->cost_rl = reward_latency;
  if (e->loaded) {
    e->cost_n = 0;  // fresh buffers: sim_done is only zeroed by a load
    int rc = ensure_cost(e);
    if (rc) return rc;
    TS_CUDA_TRY(e, cudaMemset(e->sim_done, 0, sizeof(double) * (size_t)e->n_local));
  }
  return TS_OK;
}

int ts_read_sim_times(ts_engine* e, double* host_completion, double* host_arrival, int32_t n, void* stream) {
  if (!e || n < 0 || n > e->n_local) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (!e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (e->cost_cap <= 0 || !e->sim_done) return fail(e, TS_INVALID_ARGUMENT, "no cost model set");
  if (n == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> arr(n);
  std::vector<double> clk(e->step_times_cap);
  TS_CUDA_TRY(e, cudaMemcpyAsync(arr.data(), e->arrival, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaMemcpyAsync(clk.data(), e->clock_at, sizeof(double) * clk.size(), cudaMemcpyDeviceToHost, s));
  if (host_completion)
    TS_CUDA_TRY(e, cudaMemcpyAsync(host_completion, e->sim_done, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  if (host_arrival)
    for (int i = 0; i < n; ++i) host_arrival[i] = arr[i] >= 0 && arr[i] < (int)clk.size() ? clk[arr[i]] : 0.0;
  return TS_OK;
}

int ts_read_trace(ts_engine* e, ts_trace_row* host_out, int64_t cap, int64_t* n_out, int64_t* dropped,
                  void* stream) {
  if (!e || !n_out || cap < 0 || (cap > 0 && !host_out)) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (!e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  Counters c;
  TS_CUDA_TRY(e, cudaMemcpyAsync(&c, e->ctr, sizeof(c), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  TS_CUDA_TRY(e, cudaStreamSynchronize((cudaStream_t)stream));
  const long long have = std::min<long long>((long long)c.trace_n, e->trace_cap);
  *n_out = have;
  if (dropped) *dropped = (int64_t)c.trace_drop;
  const long long k = std::min<long long>(have, cap);
  if (k > 0) {
    TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, e->trace, sizeof(ts_trace_row) * (size_t)k, cudaMemcpyDeviceToHost,
                                   (cudaStream_t)stream));
    TS_CUDA_TRY(e, cudaStreamSynchronize((cudaStream_t)stream));
  }
  return TS_OK;
}

int64_t ts_xchg_bytes(int32_t n_global) { return n_global < 0 ? -1 : (int64_t)xchg_bytes(n_global); }

int ts_xchg_create(ts_engine* e, int32_t world, int32_t rank, void** dev_ptr_out, uint8_t* ipc_handle_out) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (world < 1 || world > TS_MAX_PEERS || rank < 0 || rank >= world || !dev_ptr_out)
    return fail(e, TS_INVALID_ARGUMENT, "bad world/rank");
  TS_CUDA_TRY(e, cudaSetDevice(e->device));
  xchg_release(e);
  e->xbytes = xchg_bytes(e->n_global);
  TS_CUDA_TRY(e, cudaMalloc((void**)&e->xbuf, e->xbytes));
  TS_CUDA_TRY(e, cudaMemset(e->xbuf, 0, e->xbytes));
  TS_CUDA_TRY(e, cudaMalloc((void**)&e->xstamp, sizeof(unsigned long long) * 3 * PX_STAMP_WAVES));
  TS_CUDA_TRY(e, cudaMemset(e->xstamp, 0, sizeof(unsigned long long) * 3 * PX_STAMP_WAVES));
  size_t scr = 0, scr2 = 0;
  px_scr(nullptr, e->n_local, e->n_global, &scr);
  px_tabs(nullptr, e->n_global, &scr2);
  scr = std::max(scr, scr2);
  TS_CUDA_TRY(e, cudaMalloc((void**)&e->xscr, scr));
  TS_CUDA_TRY(e, cudaDeviceSynchronize());  // zeroed before any peer can write
  e->xworld = world;
  e->xrank = rank;
  e->xgen = 0;
  if (ipc_handle_out) {
    static_assert(sizeof(cudaIpcMemHandle_t) == TS_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    TS_CUDA_TRY(e, cudaIpcGetMemHandle(&h, e->xbuf));
    memcpy(ipc_handle_out, &h, sizeof(h));
  }
  *dev_ptr_out = e->xbuf;
  return TS_OK;
}

int ts_xchg_connect(ts_engine* e, const uint8_t* ipc_handles, void* const* dev_ptrs) {
  if (!e || !e->xbuf) return fail(e, TS_INVALID_ARGUMENT, "ts_xchg_create first");
  if (!ipc_handles && !dev_ptrs) return fail(e, TS_INVALID_ARGUMENT, "no peer buffers");
  TS_CUDA_TRY(e, cudaSetDevice(e->device));
  destroy_px_graph(e);
  for (int p = 0; p < e->xworld; ++p) {
    if (e->xipc[p] && e->xpeer[p]) cudaIpcCloseMemHandle(e->xpeer[p]);
    e->xipc[p] = false;
    e->xpeer[p] = nullptr;
    if (p == e->xrank) {
      e->xpeer[p] = e->xbuf;
    } else if (dev_ptrs && dev_ptrs[p]) {
      e->xpeer[p] = (unsigned char*)dev_ptrs[p];  // a rank emulated in this process
    } else if (ipc_handles) {
      cudaIpcMemHandle_t h;
      memcpy(&h, ipc_handles + (size_t)p * TS_IPC_HANDLE_BYTES, sizeof(h));
      void* q = nullptr;
      TS_CUDA_TRY(e, cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
      e->xpeer[p] = (unsigned char*)q;
      e->xipc[p] = true;
    } else {
      return fail(e, TS_INVALID_ARGUMENT, "missing peer buffer");
    }
  }
  // everything ts_run_sharded needs is allocated here: an allocation or free
  // while another rank's loop spins on this rank's flags (several ranks on
  // one device) would wait for that loop and never signal it
  int rc;
  cudaStream_t s0 = nullptr;
  if ((rc = ensure_log1p(e, PX_MAX_WAVES, s0))) return rc;
  if ((rc = ensure_step_times(e, e->log1p_n + 1, s0))) return rc;
  if (!e->pin_ctr) TS_CUDA_TRY(e, cudaMallocHost((void**)&e->pin_ctr, sizeof(Counters)));
  TS_CUDA_TRY(e, cudaDeviceSynchronize());
  e->xconnected = true;
  // the graph for the default max_steps, instantiated before any rank runs
  if ((rc = build_px_graph(e, px_make_view(e), INT32_MAX)) != TS_OK) {
    destroy_px_graph(e);
    return rc;
  }
  return TS_OK;
}

int ts_read_px_times(ts_engine* e, uint64_t* host_out, int32_t n, void* stream) {
  if (!e || !e->xstamp || !host_out || n < 0 || n > PX_STAMP_WAVES) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  TS_CUDA_TRY(e, cudaMemcpyAsync(host_out, e->xstamp, sizeof(uint64_t) * 3 * (size_t)n, cudaMemcpyDeviceToHost, s));
  TS_CUDA_TRY(e, cudaStreamSynchronize(s));
  return TS_OK;
}

int ts_run_sharded(ts_engine* e, int32_t max_steps, int32_t last_arrival_global, ts_run_stats* stats_out,
                   void* stream) {
  if (!e || !e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  if (!e->xconnected || e->xbytes != xchg_bytes(e->n_global))
    return fail(e, TS_INVALID_ARGUMENT, "exchange not connected for this run queue (ts_xchg_create/connect)");
  if (max_steps < 0) return fail(e, TS_INVALID_ARGUMENT, "max_steps must be >= 0");
  if (e->checks || e->trace || e->cost_cap > 0)
    return fail(e, TS_INVALID_ARGUMENT,
                "ts_run_sharded: checked mode, the allocation trace and the cost-model clock are single-engine "
                "features (ts_run)");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  ++e->xgen;
  Counters c;
  long long step0 = 0;
  {
    k_px_reset<<<1, 1, 0, s>>>(e->ctr, e->xgen, last_arrival_global);
    TS_LAUNCH_CHECK(e, "k_px_reset");
    const View v = px_make_view(e);
    if (!e->px_exec || e->px_max_steps != max_steps || memcmp(&v, &e->px_view, sizeof(View)) != 0) {
      if ((rc = build_px_graph(e, v, max_steps)) != TS_OK) {
        destroy_px_graph(e);
        return rc;
      }
    }
    TS_CUDA_TRY(e, cudaGraphLaunch(e->px_exec, s));
    TS_CUDA_TRY(e, cudaMemcpyAsync(e->pin_ctr, e->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    TS_CUDA_TRY(e, cudaStreamSynchronize(s));
    c = *e->pin_ctr;
    const long long waves = c.step - step0;
    e->launches += 1 + (waves / e->graph_unroll + 1) * e->graph_unroll *
                           ((e->n_local <= 16 * PXS && !e->px_two_kernels ? 1 : 4) + (v.heavy_on ? 2 : 1));
    step0 = c.step;
    if (c.px_err) return fail(e, TS_CUDA, "a peer rank did not signal (peer exchange timed out)");
    if (c.step < max_steps && c.step >= e->log1p_n && c.finished < e->n_local)
      return fail(e, TS_INVALID_ARGUMENT, "ts_run_sharded: more than 2^20 waves");
  }
  if (stats_out) {
    host_stats(c, stats_out);
    stats_out->steps = (int32_t)c.step;  // waves of the global loop (the same on every rank)
    stats_out->kernel_launches = e->launches;
    stats_out->wave_ms = 0.0;
  }
  if (c.sched_error) return fail(e, TS_INVALID_ARGUMENT, "run queue scores not ordered by arrival");
  return TS_OK;
}

int ts_read_invariants(ts_engine* e, ts_invariants* o, void* stream) {
  if (!e || !o) return fail(e, TS_INVALID_ARGUMENT, "bad arguments");
  if (!e->loaded) return fail(e, TS_INVALID_ARGUMENT, "no problems loaded");
  Counters c;
  TS_CUDA_TRY(e, cudaMemcpyAsync(&c, e->ctr, sizeof(c), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  TS_CUDA_TRY(e, cudaStreamSynchronize((cudaStream_t)stream));
  o->waves = c.inv[INV_WAVES];
  o->capacity_violations = c.inv[INV_CAPACITY];
  o->gate_violations = c.inv[INV_GATE];
  o->inflight_nodes = c.inv[INV_INFLIGHT];
  o->conservation_violations = c.inv[INV_CONSERVATION];
  o->root_mismatches = c.inv[INV_ROOT];
  o->max_wave_launched = c.inv[INV_MAX_LAUNCH];
  o->max_running = c.inv[INV_MAX_RUNNING];
  return TS_OK;
}

// make_problem (backend.py:144-166) + golden_step_rewards (201-215), host side.
int ts_fill_problem(uint64_t seed, int32_t solvable, int32_t depth_lo, int32_t depth_hi, int32_t branching,
                    double golden_lo, double golden_hi, double off_lo, double off_hi, int32_t hidden_until_depth,
                    int32_t has_shared, double shared_lo, double shared_hi, double target_aggregate,
                    ts_problem* out) {
  if (!out || depth_hi < depth_lo || branching < 1 || branching > TS_MAX_WIDTH) return TS_INVALID_ARGUMENT;
  auto mix = [](std::initializer_list<uint64_t> keys) {
    uint64_t h = MIX_INIT;
    for (uint64_t k : keys) h = sm64(h ^ k);
    return h;
  };
  memset(out, 0, sizeof(*out));
  out->seed = seed;
  out->branching = branching;
  out->base_depth = depth_lo + (int32_t)(mix({seed, 4}) % (uint64_t)(depth_hi - depth_lo + 1));
  out->hidden_until_depth = hidden_until_depth;
  out->has_shared = has_shared;
  out->off_lo = off_lo;
  out->off_hi = off_hi;
  out->shared_lo = shared_lo;
  out->shared_hi = shared_hi;
  out->golden_len = -1;
  if (!solvable) return TS_OK;
  const int depth = out->base_depth;
  if (depth > TS_MAX_DEPTH) return TS_INVALID_ARGUMENT;
  out->golden_len = depth;
  for (int d = 0; d < depth; ++d) out->golden_path[d] = (uint8_t)(mix({seed, 5, (uint64_t)d}) % (uint64_t)branching);
  double r[TS_MAX_DEPTH];
  for (int d = 0; d < depth; ++d) {
    const int len = d + 1;  // _raw_golden_reward(spec, d+1)
    uint64_t h = sm64(sm64(sm64(MIX_INIT ^ seed) ^ 1ull) ^ (uint64_t)len);
    for (int i = 0; i < len; ++i) h = sm64(h ^ (uint64_t)out->golden_path[i]);
    const bool shr = has_shared && len <= hidden_until_depth;
    const double lo = shr ? shared_lo : golden_lo, hi = shr ? shared_hi : golden_hi;
    r[d] = lo + (hi - lo) * u53(h);
  }
  for (int it = 0; it < 4; ++it) {
    double prod = 1.0;
    for (int d = 0; d < depth; ++d) prod = prod * r[d];
    if (prod >= target_aggregate) break;
    const double lift = std::pow(target_aggregate / prod, 1.0 / (double)depth);
    for (int d = 0; d < depth; ++d) {
      const double x = r[d] * lift * 1.001;
      r[d] = x < 0.99 ? x : 0.99;
    }
  }
  for (int d = 0; d < depth; ++d) out->golden_rewards[d] = r[d];
  return TS_OK;
}

}  // extern "C"
