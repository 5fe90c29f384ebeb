// policy.cu — standalone batched policy operators of the drop-in boundary
// (SURVEY.md §8(b)): the reference's scheduler and exit-policy entry points
// applied to caller-supplied state, for callers that keep their own run queue
// or trees instead of running whole searches in the engine.
//
//   ts_parallelism_scores  parallelism_score    scheduler.py:118-128
//   ts_compute_targets     compute_targets      scheduler.py:143-187
//   ts_exit_policy         check_negative_exit  scoring.py:153-175
//                          check_positive_exit  scoring.py:178-181
//                          decide_exit          scoring.py:184-207
//   ts_reconcile           reconcile            scheduler.py:199-214
//                          choose_preemption_victims  scheduler.py:190-196
//
// Same numerics contract as engine.cu: compiled with -fmad=false, every
// expression in the reference's order, log1p bit-identical to the host libm.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/treeserve_b200.h"
#include "exact.cuh"

namespace {

using tsx::fixed_to_double;
using tsx::libm_log1p;
using tsx::to_fixed;
using tsx::u128;

constexpr unsigned FULL = 0xffffffffu;
constexpr int SORT_TILE = 1024;  // elements sorted per CTA before the global merge passes

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(TS_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(x)                                    \
  do {                                           \
    cudaError_t _e = (x);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, #x); \
  } while (0)

// ---- compute_targets -----------------------------------------------------------

// Device-side scalars of one compute_targets call.
struct CtState {
  double T;               // Σ S in run-queue order (CPython sum semantics)
  long long U;            // ungated jobs
  long long tw;           // Σ over ungated of (want - 1)
  int first_bad;          // lowest run-queue index with now < arrival (n if none)
  int fallback;           // the exact fixed-point sum was not usable
};

// Sort key of an ungated job: (-S, arrival_time, job_id) (scheduler.py:167);
// gated jobs sort after every ungated one.
struct CtKey {
  double S, arrival;
  long long id;
  int gated, idx;
};
__device__ __forceinline__ bool key_less(const CtKey& a, const CtKey& b) {
  if (a.gated != b.gated) return a.gated < b.gated;
  if (a.S != b.S) return a.S > b.S;  // -S ascending
  if (a.arrival != b.arrival) return a.arrival < b.arrival;
  return a.id < b.id;
}

// parallelism_score (scheduler.py:118-128) per job; ungated = completed >= obs.
__device__ __forceinline__ double pscore(double now, double arrival, double best, double theta, double beta,
                                         double proximity) {
  const double waited = now - arrival;
  const double ratio = best / theta;
  const double boost = ratio > proximity ? beta : 0.0;
  return libm_log1p(waited) + boost;
}

__global__ void k_scores(int n, double now, double theta, double beta, double proximity, int obs,
                         const double* __restrict__ arrival, const double* __restrict__ best,
                         const int32_t* __restrict__ completed, const int64_t* __restrict__ job_id,
                         double* __restrict__ S, CtKey* __restrict__ keys, CtState* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = arrival[i];
  if (now < a) atomicMin(&st->first_bad, i);  // parallelism_score raises ValueError
  const double s = pscore(now, a, best[i], theta, beta, proximity);
  S[i] = s;
  if (keys) {
    CtKey k;
    k.S = s;
    k.arrival = a;
    k.id = job_id[i];
    k.gated = completed[i] >= obs ? 0 : 1;
    k.idx = i;
    keys[i] = k;
  }
}

// Σ S over the run queue, equal to CPython's sum() (Neumaier since 3.12):
// exact in 128-bit fixed point when every compensation term is exact (all
// scores are multiples of 2^-64 and n * ulp(2T) < 2^-10), else
// the sequential loop.  Phase 1: per-CTA partial fixed-point sums and
// ungated counts; phase 2 (one CTA): the total, its exactness test, and the
// sequential fallback.
struct SumPart {
  uint64_t lo, hi;
  long long ungated;
  int bad, _pad;
};

__device__ __forceinline__ void warp_u128_add(u128& x) {
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t h = __shfl_down_sync(FULL, (uint64_t)(x >> 64), o);
    const uint64_t l = __shfl_down_sync(FULL, (uint64_t)x, o);
    x += ((u128)h << 64) | l;
  }
}

__global__ void __launch_bounds__(256) k_sum_part(int n, int obs, const double* __restrict__ S,
                                                  const int32_t* __restrict__ completed, SumPart* part) {
  __shared__ u128 sq[8];
  __shared__ long long su[8];
  __shared__ int sbad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) sbad = 0;
  __syncthreads();
  u128 fx = 0;
  long long u = 0;
  bool bad = false;
  for (int i = blockIdx.x * 256 + tid; i < n; i += gridDim.x * 256) {
    u128 q;
    if (to_fixed(S[i], q)) fx += q;
    else bad = true;
    u += completed[i] >= obs ? 1 : 0;
  }
  warp_u128_add(fx);
  for (int o = 16; o > 0; o >>= 1) u += __shfl_down_sync(FULL, u, o);
  if (lane == 0) {
    sq[wid] = fx;
    su[wid] = u;
  }
  if (bad) sbad = 1;
  __syncthreads();
  if (tid == 0) {
    u128 t = 0;
    long long uu = 0;
    for (int w = 0; w < 8; ++w) {
      t += sq[w];
      uu += su[w];
    }
    SumPart r;
    r.lo = (uint64_t)t;
    r.hi = (uint64_t)(t >> 64);
    r.ungated = uu;
    r.bad = sbad;
    r._pad = 0;
    part[blockIdx.x] = r;
  }
}

__global__ void __launch_bounds__(32) k_sum_final(int n, int nparts, const SumPart* __restrict__ part,
                                                  const double* __restrict__ S, CtState* st) {
  const int lane = threadIdx.x;
  u128 t = 0;
  long long uu = 0;
  int bad = 0;
  for (int b = lane; b < nparts; b += 32) {
    const SumPart r = part[b];
    t += ((u128)r.hi << 64) | r.lo;
    uu += r.ungated;
    bad |= r.bad;
  }
  warp_u128_add(t);
  for (int o = 16; o > 0; o >>= 1) uu += __shfl_down_sync(FULL, uu, o);
  bad = __any_sync(FULL, bad);
  if (lane == 0) {
    bool fallback = bad != 0;
    double T = 0.0;
    if (!fallback) {
      T = fixed_to_double(t);
      const double u2 = T > 0 ? ldexp(1.0, ilogb(2.0 * T) - 52) : 0.0;
      if ((double)n * u2 >= 0x1p-10) fallback = true;
    }
    if (fallback) {  // builtin sum() over floats, run-queue order
      double f = 0.0, c = 0.0;
      for (int i = 0; i < n; ++i) {
        const double x = S[i];
        const double y = f + x;
        if (fabs(f) >= fabs(x)) c += (f - y) + x;
        else c += (x - y) + f;
        f = y;
      }
      if (c != 0.0 && isfinite(c)) f += c;
      T = f;
    }
    st->T = T;
    st->U = uu;
    st->fallback = fallback ? 1 : 0;
  }
}

// Stable merge sort of the keys: each CTA sorts one tile in shared memory,
// then global merge passes double the run width (merge by rank: an element's
// output slot is its index in its own run plus its rank in the sibling run).
__global__ void __launch_bounds__(SORT_TILE) k_sort_tile(int n, CtKey* __restrict__ keys) {
  extern __shared__ __align__(16) unsigned char smem[];
  CtKey* a = (CtKey*)smem;
  CtKey* b = a + SORT_TILE;
  const int base = blockIdx.x * SORT_TILE;
  const int m = min(SORT_TILE, n - base);
  const int t = threadIdx.x;
  if (t < m) a[t] = keys[base + t];
  __syncthreads();
  for (int w = 1; w < m; w <<= 1) {
    if (t < m) {
      const CtKey k = a[t];
      const int pb = (t / (2 * w)) * (2 * w);
      const bool left = t < pb + w;
      const int o0 = left ? min(pb + w, m) : pb;
      const int o1 = left ? min(pb + 2 * w, m) : pb + w;
      int lo = o0, hi = o1;  // left: # sibling < k; right: # sibling <= k
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const bool before = left ? key_less(a[mid], k) : !key_less(k, a[mid]);
        if (before) lo = mid + 1;
        else hi = mid;
      }
      const int own = left ? t - pb : t - (pb + w);
      b[pb + own + (lo - o0)] = k;
    }
    __syncthreads();
    CtKey* tmp = a;
    a = b;
    b = tmp;
  }
  if (t < m) keys[base + t] = a[t];
}

__global__ void k_merge_pass(int n, int w, const CtKey* __restrict__ in, CtKey* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const CtKey k = in[t];
  const int pb = (t / (2 * w)) * (2 * w);
  const bool left = t < pb + w;
  const int o0 = left ? min(pb + w, n) : pb;
  const int o1 = left ? min(pb + 2 * w, n) : pb + w;
  int lo = o0, hi = o1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool before = left ? key_less(in[mid], k) : !key_less(k, in[mid]);
    if (before) lo = mid + 1;
    else hi = mid;
  }
  const int own = left ? t - pb : t - (pb + w);
  out[pb + own + (lo - o0)] = k;
}

__device__ __forceinline__ long long want_of(double s, double T, long long M) {
  if (!(T > 0.0)) return 1;
  const double f = floor(s / T * (double)M);  // (S/T)*M, scheduler.py:173-175
  if (!(f > 1.0)) return 1;
  return f >= 9.2e18 ? (long long)9.2e18 : (long long)f;
}

// The allocation loops of compute_targets (scheduler.py:169-186) in closed
// form over the sorted ungated jobs: extra_k = clamp(R - Σ_{j<k}(want_j - 1),
// 0, want_k - 1); the leftover R' = R - Σ extra is dealt round-robin in sorted
// order: floor(R'/U) + [k < R' mod U].  Gated jobs keep 1.  Three phases: a
// per-CTA scan of (want - 1) in sorted order, a scan of the CTA totals, and
// the targets.
constexpr int AT = 256;

__device__ __forceinline__ long long block_excl_scan(long long x, long long* total) {
  __shared__ long long sw[AT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sw[wid] = incl;
  __syncthreads();
  long long base = 0, tot = 0;
  for (int w = 0; w < AT / 32; ++w) {
    if (w < wid) base += sw[w];
    tot += sw[w];
  }
  *total = tot;
  __syncthreads();
  return base + incl - x;
}

__global__ void __launch_bounds__(AT) k_want_scan(int n, long long M, const CtKey* __restrict__ sorted,
                                                  const CtState* __restrict__ st, long long* __restrict__ pre,
                                                  long long* __restrict__ blk) {
  const long long U = st->U;
  const double T = st->T;
  const int k = blockIdx.x * AT + threadIdx.x;
  const long long w = k < U ? want_of(sorted[k].S, T, M) - 1 : 0;
  long long tot;
  const long long e = block_excl_scan(w, &tot);
  if (k < n) pre[k] = e;
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_blk_scan(int nb, long long* __restrict__ blk, CtState* st) {
  __shared__ long long sw[32];
  __shared__ long long carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const long long x = i < nb ? blk[i] : 0;
    long long incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) sw[wid] = incl;
    __syncthreads();
    long long off = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < wid) off += sw[w];
      tot += sw[w];
    }
    if (i < nb) blk[i] = carry + off + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) st->tw = carry;
}

__global__ void k_targets_out(int n, long long M, const CtKey* __restrict__ sorted, const CtState* __restrict__ st,
                              const long long* __restrict__ pre, const long long* __restrict__ blk,
                              int32_t* __restrict__ targets) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long U = st->U;
  if (k >= U) {
    targets[sorted[k].idx] = 1;
    return;
  }
  const long long R = M - (long long)n;
  const long long tw = st->tw;
  const long long given = R > 0 ? (tw < R ? tw : R) : 0;
  const long long Rp = R > 0 ? R - given : 0;
  const long long want = want_of(sorted[k].S, st->T, M);
  const long long before = blk[k / AT] + pre[k];
  long long extra = R - before;
  if (extra < 0) extra = 0;
  if (extra > want - 1) extra = want - 1;
  long long rr = 0;
  if (U > 0 && Rp > 0) rr = Rp / U + ((long long)k < Rp % U ? 1 : 0);
  const long long t = 1 + extra + rr;
  targets[sorted[k].idx] = t > 0x7fffffffLL ? 0x7fffffff : (int32_t)t;
}

__global__ void k_fill(int n, int32_t v, int32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

__global__ void k_init_state(CtState* st, int n) {
  st->T = 0.0;
  st->U = 0;
  st->tw = 0;
  st->first_bad = n;
  st->fallback = 0;
}

// ---- exit policy over a forest ----------------------------------------------------

struct PolicyCounts {
  int32_t fire;      // candidate NE result (root has children and no viable leaf seen)
  int32_t relevant;  // check-relevant leaves seen (classify_leaf would be called)
};

// Per tree: NE starts as "fires" iff the root has children (scoring.py:160-161).
__global__ void k_ne_init(int n_trees, const int32_t* __restrict__ off, const uint8_t* __restrict__ flags,
                          PolicyCounts* pc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_trees) return;
  const int r = off[t];
  PolicyCounts p;
  p.fire = (off[t + 1] > r && (flags[r] & TS_NODE_HAS_CHILDREN)) ? 1 : 0;
  p.relevant = 0;
  pc[t] = p;
}

// One thread per node: expandable leaves (non-terminal, childless,
// scoring.py:137-138), filtered in selective mode by the depth-1 ancestor's
// reward (164-170), classified by classify_leaf (119-134) on the prefix
// aggregate of path_to_root(leaf)[1:] (148-150).  A viable leaf clears the
// tree's fire flag.
__global__ void k_ne_leaves(int n_nodes, int scheme, int bound, int strict, double tau, double theta_first,
                            const int32_t* __restrict__ tree_of, const int32_t* __restrict__ parent,
                            const double* __restrict__ reward, const int32_t* __restrict__ depth,
                            const uint8_t* __restrict__ flags, PolicyCounts* pc) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_nodes) return;
  const uint8_t fl = flags[g];
  if (fl & (TS_NODE_HAS_CHILDREN | TS_NODE_TERMINAL)) return;
  const int t = tree_of[g];
  if (!pc[t].fire) return;  // root without children: never fires, no leaf is classified
  if (!strict) {
    int a = g;
    while (depth[a] > 1) a = parent[a];  // _depth_one_ancestor (scoring.py:141-145)
    if (!(reward[a] >= theta_first)) return;
  }
  atomicAdd(&pc[t].relevant, 1);
  if (scheme != TS_SCHEME_MINIMUM && scheme != TS_SCHEME_PRODUCT) return;  // raises on the host
  const double leaf = reward[g];
  double b;
  if (bound == TS_BOUND_LEAF_REWARD) {
    b = leaf;
  } else {
    // prefix aggregate in root-to-leaf order (math.prod left to right / min)
    constexpr int KEEP = 64;
    double rs[KEEP];
    int d = 0;
    for (int a = g; parent[a] >= 0; a = parent[a]) {
      if (d < KEEP) rs[d] = reward[a];
      ++d;
    }
    double agg = 1.0;
    if (d <= KEEP) {
      for (int j = d - 1; j >= 0; --j) {
        const double r = rs[j];
        if (scheme == TS_SCHEME_PRODUCT) agg = agg * r;
        else agg = (j == d - 1 || r < agg) ? r : agg;
      }
    } else {  // deep leaf: walk from the top, O(d^2) loads
      for (int j = d - 1; j >= 0; --j) {
        int a = g;
        for (int s = 0; s < j; ++s) a = parent[a];
        const double r = reward[a];
        if (scheme == TS_SCHEME_PRODUCT) agg = agg * r;
        else agg = (j == d - 1 || r < agg) ? r : agg;
      }
    }
    b = agg < leaf ? agg : leaf;  // min(leaf_reward, prefix_aggregate)
  }
  if (!(b < tau)) pc[t].fire = 0;  // VIABLE (classify_leaf: futile iff bound < tau)
}

// decide_exit (scoring.py:184-207): PE > NE > budget/exhaustion > CONTINUE.
__global__ void k_decide(int n_trees, double theta_pos, int pe_on, int ne_on, int scheme_ok,
                         const PolicyCounts* __restrict__ pc, const double* __restrict__ best,
                         const uint8_t* __restrict__ has_best, const int32_t* __restrict__ completed,
                         const int32_t* __restrict__ budget, const uint8_t* __restrict__ exhausted,
                         int32_t* __restrict__ kind, uint8_t* __restrict__ ne_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_trees) return;
  const PolicyCounts p = pc[t];
  const bool unsupported = !scheme_ok && p.relevant > 0;
  const bool ne = p.fire != 0;
  if (ne_out) ne_out[t] = unsupported ? 2 : (ne ? 1 : 0);
  if (!kind) return;
  const bool hb = has_best && has_best[t];
  int k;
  if (pe_on && hb && best[t] >= theta_pos) k = TS_EXIT_POSITIVE;
  else if (ne_on && unsupported) k = -TS_UNSUPPORTED_SCHEME;
  else if (ne_on && ne) k = TS_EXIT_NEGATIVE;
  else if ((exhausted && exhausted[t]) || (completed && budget && completed[t] >= budget[t])) k = TS_EXIT_BUDGET;
  else k = TS_EXIT_NONE;
  kind[t] = k;
}

inline int blocks(long long n, int t) { return (int)((n + t - 1) / t); }

// Grow-only per-device workspace of ts_compute_targets (one host thread per
// engine/device, as everywhere in this ABI).
struct Workspace {
  int cap = 0;
  bool attr = false;
  CtState* st = nullptr;
  CtState* host = nullptr;  // pinned read-back of st
  double* S = nullptr;
  CtKey *ka = nullptr, *kb = nullptr;
  long long *pre = nullptr, *blk = nullptr;
  SumPart* part = nullptr;
};

int workspace_for(int n, Workspace** out) {
  static Workspace wss[64];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(TS_INVALID_ARGUMENT, "device index out of range");
  Workspace& w = wss[dev];
  if (w.cap < n) {
    cudaFree(w.st);
    cudaFree(w.S);
    cudaFree(w.ka);
    cudaFree(w.kb);
    cudaFree(w.pre);
    cudaFree(w.blk);
    cudaFree(w.part);
    if (!w.host) CK(cudaMallocHost((void**)&w.host, sizeof(CtState)));
    const int cap = n < 4096 ? 4096 : n;
    CK(cudaMalloc((void**)&w.st, sizeof(CtState)));
    CK(cudaMalloc((void**)&w.S, sizeof(double) * (size_t)cap));
    CK(cudaMalloc((void**)&w.ka, sizeof(CtKey) * (size_t)cap));
    CK(cudaMalloc((void**)&w.kb, sizeof(CtKey) * (size_t)cap));
    CK(cudaMalloc((void**)&w.pre, sizeof(long long) * (size_t)cap));
    CK(cudaMalloc((void**)&w.blk, sizeof(long long) * (size_t)((cap + AT - 1) / AT + 1)));
    CK(cudaMalloc((void**)&w.part, sizeof(SumPart) * 1184));
    w.cap = cap;
  }
  *out = &w;
  return TS_OK;
}

// ---- reconcile / choose_preemption_victims --------------------------------------
// One warp per job.  gap = target - active (active = the job's in-flight
// rollouts [off[j], off[j+1])): gap > 0 is LaunchAction(gap); gap < 0 ranks
// the in-flight rollouts by (prefix_score, rollout_id) (sorted(...) with the
// tuple key, scheduler.py:195) and the -gap lowest are the victims, emitted in
// rank order.  A rollout's rank = # rollouts ordered before it (lanes stride
// the segment; the comparisons of one rollout are a warp-wide count).
// Non-running jobs produce no action.  Ties on both keys cannot occur for
// distinct rollout ids; equal ids keep their input order.
__global__ void __launch_bounds__(256) k_reconcile(int n, const int32_t* __restrict__ running,
                                                   const int32_t* __restrict__ target,
                                                   const int64_t* __restrict__ off,
                                                   const double* __restrict__ score,
                                                   const int64_t* __restrict__ rid, int32_t* __restrict__ launch,
                                                   int32_t* __restrict__ victim_rank) {
  const int lane = threadIdx.x & 31;
  const int j = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (j >= n) return;
  const long long a = off[j], b = off[j + 1];
  const long long active = b - a;
  const bool run = running == nullptr || running[j] != 0;
  const long long gap = run ? (long long)target[j] - active : 0;
  if (lane == 0) launch[j] = gap > 0 ? (int32_t)gap : 0;
  const long long victims = gap < 0 ? -gap : 0;
  for (long long r = a; r < b; ++r) {
    int32_t out = -1;
    if (victims > 0) {
      const double sr = score[r];
      const int64_t ir = rid[r];
      unsigned cnt = 0;
      for (long long q = a + lane; q < b; q += 32) {
        const double sq = score[q];
        const int64_t iq = rid[q];
        cnt += (sq < sr || (sq == sr && (iq < ir || (iq == ir && q < r)))) ? 1u : 0u;
      }
      const long long rank = (long long)__reduce_add_sync(FULL, cnt);
      if (rank < victims) out = (int32_t)rank;
    }
    if (lane == 0) victim_rank[r] = out;
  }
}

}  // namespace

extern "C" {

const char* ts_policy_last_error(void) { return g_err.c_str(); }

int ts_parallelism_scores(double now, double positive_exit_threshold, double beta, double proximity,
                          const double* dev_arrival, const double* dev_best, int32_t n, double* dev_scores,
                          int32_t* host_first_bad, void* stream) {
  if (n < 0 || (n > 0 && (!dev_arrival || !dev_best || !dev_scores)))
    return fail(TS_INVALID_ARGUMENT, "ts_parallelism_scores: bad arguments");
  if (host_first_bad) *host_first_bad = n;
  if (n == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  CtState* st = nullptr;
  CK(cudaMallocAsync((void**)&st, sizeof(CtState), s));
  k_init_state<<<1, 1, 0, s>>>(st, n);
  k_scores<<<blocks(n, 256), 256, 0, s>>>(n, now, positive_exit_threshold, beta, proximity, 0, dev_arrival,
                                          dev_best, nullptr, nullptr, dev_scores, nullptr, st);
  CtState h;
  CK(cudaMemcpyAsync(&h, st, sizeof(CtState), cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(st, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  if (host_first_bad) *host_first_bad = h.first_bad;
  if (h.first_bad < n) return fail(TS_INVALID_ARGUMENT, "parallelism_score: now precedes arrival");
  return TS_OK;
}

int ts_compute_targets(const ts_sched_params* p, double now, const double* dev_arrival, const double* dev_best,
                       const int32_t* dev_completed, const int64_t* dev_job_id, int32_t n, int32_t* dev_targets,
                       ts_targets_info* host_info, void* stream) {
  if (!p || n < 0 || (n > 0 && (!dev_arrival || !dev_best || !dev_completed || !dev_job_id || !dev_targets)))
    return fail(TS_INVALID_ARGUMENT, "ts_compute_targets: bad arguments");
  if (n == 0) return fail(TS_INVALID_ARGUMENT, "run queue holds no running jobs");
  if (p->max_concurrency < 1) return fail(TS_INVALID_ARGUMENT, "max_concurrency must be >= 1");
  if (!(p->beta > 0)) return fail(TS_INVALID_ARGUMENT, "beta must be positive");
  if (!(p->proximity > 0.0 && p->proximity < 1.0)) return fail(TS_INVALID_ARGUMENT, "proximity must lie in (0,1)");
  if (p->obs_threshold < 1) return fail(TS_INVALID_ARGUMENT, "obs_threshold must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  ts_targets_info info{};
  info.first_bad = n;
  if (!p->boosting_enabled) {  // scheduler.py:158-160: no scores are computed
    k_fill<<<blocks(n, 256), 256, 0, s>>>(n, 1, dev_targets);
    CK(cudaGetLastError());
    info.kernel_launches = 1;
    if (host_info) *host_info = info;
    return TS_OK;
  }
  Workspace* ws = nullptr;
  int rc = workspace_for(n, &ws);
  if (rc) return rc;
  const int nparts = blocks(n, 256) < 1184 ? blocks(n, 256) : 1184;  // 8 x 148 SMs
  const int nb = blocks(n, AT);
  CtKey* ka = ws->ka;
  CtKey* kb = ws->kb;
  k_init_state<<<1, 1, 0, s>>>(ws->st, n);
  k_scores<<<blocks(n, 256), 256, 0, s>>>(n, now, p->positive_exit_threshold, p->beta, p->proximity,
                                          p->obs_threshold, dev_arrival, dev_best, dev_completed, dev_job_id, ws->S,
                                          ka, ws->st);
  k_sum_part<<<nparts, 256, 0, s>>>(n, p->obs_threshold, ws->S, dev_completed, ws->part);
  k_sum_final<<<1, 32, 0, s>>>(n, nparts, ws->part, ws->S, ws->st);
  const size_t sm = 2 * SORT_TILE * sizeof(CtKey);
  if (!ws->attr) {
    CK(cudaFuncSetAttribute(k_sort_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    ws->attr = true;
  }
  k_sort_tile<<<blocks(n, SORT_TILE), SORT_TILE, sm, s>>>(n, ka);
  int passes = 0;
  for (long long w = SORT_TILE; w < n; w <<= 1, ++passes) {
    k_merge_pass<<<blocks(n, 256), 256, 0, s>>>(n, (int)w, ka, kb);
    CtKey* t = ka;
    ka = kb;
    kb = t;
  }
  const long long M = (long long)p->max_concurrency;
  k_want_scan<<<nb, AT, 0, s>>>(n, M, ka, ws->st, ws->pre, ws->blk);
  k_blk_scan<<<1, 1024, 0, s>>>(nb, ws->blk, ws->st);
  k_targets_out<<<blocks(n, 256), 256, 0, s>>>(n, M, ka, ws->st, ws->pre, ws->blk, dev_targets);
  CK(cudaMemcpyAsync(ws->host, ws->st, sizeof(CtState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  const CtState h = *ws->host;
  info.first_bad = h.first_bad;
  info.total_score = h.T;
  info.ungated = h.U;
  info.sum_fallback = h.fallback;
  info.kernel_launches = 9 + passes;
  if (host_info) *host_info = info;
  if (h.first_bad < n) return fail(TS_INVALID_ARGUMENT, "parallelism_score: now precedes arrival");
  return TS_OK;
}

int ts_exit_policy(const ts_config* cfg, const ts_forest* f, int32_t* dev_kind, uint8_t* dev_ne, void* stream) {
  if (!cfg || !f || f->n_trees < 0 || f->n_nodes < 0)
    return fail(TS_INVALID_ARGUMENT, "ts_exit_policy: bad arguments");
  if (f->n_trees == 0) return TS_OK;
  if (!f->offsets || !f->tree_of || !f->parent || !f->reward || !f->depth || !f->flags)
    return fail(TS_INVALID_ARGUMENT, "ts_exit_policy: missing forest arrays");
  cudaStream_t s = (cudaStream_t)stream;
  PolicyCounts* pc = nullptr;
  CK(cudaMallocAsync((void**)&pc, sizeof(PolicyCounts) * f->n_trees, s));
  k_ne_init<<<blocks(f->n_trees, 256), 256, 0, s>>>(f->n_trees, f->offsets, f->flags, pc);
  if (f->n_nodes > 0)
    k_ne_leaves<<<blocks(f->n_nodes, 256), 256, 0, s>>>(
        f->n_nodes, cfg->scheme, cfg->futility_bound, cfg->strict_negative_exit, cfg->accept_threshold,
        cfg->first_step_threshold, f->tree_of, f->parent, f->reward, f->depth, f->flags, pc);
  const int scheme_ok = cfg->scheme == TS_SCHEME_MINIMUM || cfg->scheme == TS_SCHEME_PRODUCT;
  k_decide<<<blocks(f->n_trees, 256), 256, 0, s>>>(f->n_trees, cfg->positive_exit_threshold, cfg->positive_exit,
                                                   cfg->negative_exit, scheme_ok, pc, f->best_score, f->has_best,
                                                   f->completed, f->budget, f->exhausted, dev_kind, dev_ne);
  CK(cudaFreeAsync(pc, s));
  CK(cudaGetLastError());
  return TS_OK;
}

int ts_reconcile(const int32_t* dev_running, const int32_t* dev_targets, const int64_t* dev_offsets,
                 const double* dev_prefix_score, const int64_t* dev_rollout_id, int32_t n_jobs, int32_t* dev_launch,
                 int32_t* dev_victim_rank, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && (!dev_targets || !dev_offsets || !dev_launch)))
    return fail(TS_INVALID_ARGUMENT, "ts_reconcile: bad arguments");
  if (n_jobs == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  k_reconcile<<<blocks((long long)n_jobs * 32, 256), 256, 0, s>>>(n_jobs, dev_running, dev_targets, dev_offsets,
                                                                  dev_prefix_score, dev_rollout_id, dev_launch,
                                                                  dev_victim_rank);
  CK(cudaGetLastError());
  return TS_OK;
}

}  // extern "C"
