// beam.cu — the paper's beam-search baseline (reference beam.py:143-176) for
// many problems at once, on the same replayed synthetic backend as the tree
// search.
//
// One warp per problem; lane j is candidate j of the step (beam j / C, sample
// j % C), so the default 8 beams x 4 samples fill one warp.  A step is:
//   * generate_steps for every candidate (backend.py:230-269): the reward,
//     token and extend keys share the prefix fold of the beam's path, so each
//     lane folds (seed, tag, len, path) for the three tags with independent
//     chains and finishes with one splitmix64 on its own step index;
//   * the accumulated score (aggregate_trajectory, incremental in the
//     reference's order: math.prod / min / CPython sum);
//   * best_finished over the terminal candidates in candidate order (first
//     maximum; strict '>' against the running best, beam.py:134-140);
//   * prune_candidates (beam.py:107-117): each open lane's rank under
//     (-score, order) is a 32-way shuffle count; rank < beam_width writes the
//     surviving beam to slot `rank` of the other shared-memory buffer.
// The best beam's rewards are recomputed at the end from its path (they are a
// pure function of the path), so beams carry only their path bytes and the
// running aggregate.
//
// Same numerics contract as engine.cu (-fmad=false, reference order).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/treeserve_b200.h"
#include "exact.cuh"
#include "rng.cuh"

namespace {

using tsx::Agg;
using tsx::MIX_INIT;
using tsx::sm64;
using tsx::u53;

constexpr unsigned FULL = 0xffffffffu;
constexpr int BEAM_WARPS = 4;  // warps (problems in flight) per CTA
constexpr int MAXB = TS_BEAM_MAX_CANDIDATES;

struct BeamSmem {
  uint8_t path[2][MAXB][TS_MAX_DEPTH];  // beam index paths, double-buffered across steps
  double a[2][MAXB], c[2][MAXB];        // running aggregate (Agg a, c) of every beam
  uint8_t gold[2][MAXB];                // beam path is a golden prefix (_is_golden_prefix)
  uint8_t best[TS_MAX_DEPTH];           // best finished beam's path
};

// First lane holding the maximum of v among valid lanes (ties: lowest lane).
__device__ __forceinline__ int warp_argmax_first(double v, bool valid) {
  const uint64_t b = (uint64_t)__double_as_longlong(v + 0.0);
  const uint64_t key = (b >> 63) ? ~b : (b | (1ull << 63));
  const unsigned hi = valid ? (unsigned)(key >> 32) : 0u;
  const unsigned lo = valid ? (unsigned)key : 0u;
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  const unsigned win = __ballot_sync(FULL, valid && hi == mh && lo == ml);
  return __ffs(win) - 1;
}

__device__ __forceinline__ uint64_t fold3(uint64_t seed, uint64_t tag, uint64_t len) {
  return sm64(sm64(sm64(MIX_INIT ^ seed) ^ tag) ^ len);
}

__global__ void __launch_bounds__(32 * BEAM_WARPS) k_beam(ts_beam_config cfg, const ts_problem* __restrict__ probs,
                                                          int n, ts_beam_result* __restrict__ out) {
  __shared__ BeamSmem smem[BEAM_WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  BeamSmem& S = smem[wid];
  const int B = cfg.beam_width, C = cfg.candidates_per_beam, scheme = cfg.scheme;
  for (int pi = blockIdx.x * BEAM_WARPS + wid; pi < n; pi += gridDim.x * BEAM_WARPS) {
    const ts_problem& P = probs[pi];
    const uint64_t seed = P.seed;
    const int branching = P.branching, base = P.base_depth, glen = P.golden_len;
    const int hidden = P.hidden_until_depth;
    const bool shared = P.has_shared != 0;
    const double off_lo = P.off_lo, off_hi = P.off_hi, sh_lo = P.shared_lo, sh_hi = P.shared_hi;

    if (lane == 0) {  // the root beam: empty path, score 0.0, aggregate identity
      S.a[0][0] = 1.0;
      S.c[0][0] = 0.0;
      S.gold[0][0] = glen >= 0 ? 1 : 0;
    }
    __syncwarp();
    int na = 1, cur = 0, L = 0, steps = 0, best_len = 0;
    bool has_best = false;
    double best_score = 0.0;
    long long tokens = 0;
    while (na > 0 && steps < cfg.max_depth) {
      const int nc = na * C;
      const bool act = lane < nc;
      const int b = act ? lane / C : 0;
      const int idx = (lane % C) % branching;
      // expand_beams: candidate (b, i) = generate_steps(problem, path_b, C)[i]
      const int depth = L + 1;
      uint64_t hr = fold3(seed, 1, depth), ht = fold3(seed, 3, depth), he = fold3(seed, 6, depth);
      for (int d = 0; d < L; ++d) {
        const uint64_t s = S.path[cur][b][d];
        hr = sm64(hr ^ s);
        ht = sm64(ht ^ s);
        he = sm64(he ^ s);
      }
      hr = sm64(hr ^ (uint64_t)idx);
      ht = sm64(ht ^ (uint64_t)idx);
      he = sm64(he ^ (uint64_t)idx);
      const bool gold = S.gold[cur][b] && depth <= glen && idx == (int)P.golden_path[depth - 1];
      double reward;
      if (gold) {
        reward = P.golden_rewards[depth - 1];  // golden_step_rewards (host-lifted)
      } else {
        const bool sr = shared && depth <= hidden;
        const double lo = sr ? sh_lo : off_lo, hi = sr ? sh_hi : off_hi;
        reward = lo + (hi - lo) * u53(hr);
      }
      bool term;  // _is_terminal (backend.py:179-188)
      if (depth < base) term = false;
      else if (depth >= base + 1) term = true;
      else if (gold) term = true;
      else term = !((he % 2u) == 0u);
      const int tok = 40 + (int)(ht % 81u);  // randint_in(40, 120, ...)
      Agg g;
      g.a = S.a[cur][b];
      g.c = S.c[cur][b];
      g.n = L;
      g.add(reward, scheme);
      const double score = g.value(scheme);
      tokens += __reduce_add_sync(FULL, act ? (unsigned)tok : 0u);

      // finished pool: best_finished over this step's terminal candidates in order
      const bool fin = act && term;
      if (__ballot_sync(FULL, fin)) {
        const int w = warp_argmax_first(score, fin);
        const double ws = __shfl_sync(FULL, score, w);
        if (!has_best || ws > best_score) {
          has_best = true;
          best_score = ws;
          best_len = depth;
          const int wb = w / C, widx = (w % C) % branching;
          if (lane < L) S.best[lane] = S.path[cur][wb][lane];
          if (lane == 0) S.best[L] = (uint8_t)widx;
        }
      }
      // prune_candidates: top B open candidates by (-score, order)
      const bool open = act && !term;
      const unsigned om = __ballot_sync(FULL, open);
      int rank = 0;
      for (int k = 0; k < nc; ++k) {
        const double sk = __shfl_sync(FULL, score, k);
        rank += (((om >> k) & 1u) && (sk > score || (sk == score && k < lane))) ? 1 : 0;
      }
      const int nxt = cur ^ 1;
      if (open && rank < B) {
        for (int d = 0; d < L; ++d) S.path[nxt][rank][d] = S.path[cur][b][d];
        S.path[nxt][rank][L] = (uint8_t)idx;
        S.a[nxt][rank] = g.a;
        S.c[nxt][rank] = g.c;
        S.gold[nxt][rank] = gold ? 1 : 0;
      }
      __syncwarp();
      const int nopen = __popc(om);
      na = nopen < B ? nopen : B;
      cur = nxt;
      ++L;
      ++steps;
      if (cfg.positive_exit_enabled && has_best && best_score >= cfg.positive_exit_threshold) break;
    }

    // the result beam: best finished, else the best surviving partial
    ts_beam_result* r = out + pi;
    int rlen = 0;
    bool have = has_best;
    double rscore = best_score;
    if (!has_best && na > 0) {
      double s = 0.0;
      if (lane < na) {
        Agg g;
        g.a = S.a[cur][lane];
        g.c = S.c[cur][lane];
        g.n = L;
        s = g.value(scheme);
      }
      const int w = warp_argmax_first(s, lane < na);
      rscore = __shfl_sync(FULL, s, w);
      if (lane < L) S.best[lane] = S.path[cur][w][lane];
      have = true;
      rlen = L;
    } else if (has_best) {
      rlen = best_len;
    }
    __syncwarp();
    if (lane < rlen) {  // rewards along the path: _child_reward of every prefix
      const int d = lane + 1;
      uint64_t h = fold3(seed, 1, d);
      bool g = glen >= d;
      for (int k = 0; k < d; ++k) {
        const uint8_t s = S.best[k];
        h = sm64(h ^ (uint64_t)s);
        if (g && P.golden_path[k] != s) g = false;
      }
      double rw;
      if (g) {
        rw = P.golden_rewards[d - 1];
      } else {
        const bool sr = shared && d <= hidden;
        const double lo = sr ? sh_lo : off_lo, hi = sr ? sh_hi : off_hi;
        rw = lo + (hi - lo) * u53(h);
      }
      r->best_rewards[lane] = rw;
      r->best_path[lane] = S.best[lane];
    }
    if (lane == 0) {
      r->complete = has_best ? 1 : 0;
      r->has_best = have ? 1 : 0;
      r->is_terminal = has_best ? 1 : 0;
      r->best_len = rlen;
      r->steps = steps;
      r->status = TS_OK;
      r->tokens_generated = tokens;
      r->best_score = have ? rscore : 0.0;
    }
    for (int k = rlen + lane; k < TS_MAX_DEPTH; k += 32) {
      r->best_rewards[k] = 0.0;
      r->best_path[k] = 0;
    }
    __syncwarp();
  }
}


// ---- step-level operators -------------------------------------------------------

// expand_beams + prune ranks for one problem per warp (candidate j in lane j).
__global__ void __launch_bounds__(32 * BEAM_WARPS) k_beam_expand(ts_beam_config cfg, const ts_problem* __restrict__ probs,
                                                                 int n, const ts_beam* __restrict__ beams,
                                                                 const int32_t* __restrict__ counts,
                                                                 ts_beam_candidate* __restrict__ out,
                                                                 int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pi = blockIdx.x * BEAM_WARPS + wid;
  if (pi >= n) return;
  const ts_problem& P = probs[pi];
  const int C = cfg.candidates_per_beam, nb = counts[pi], nc = nb * C;
  const int branching = P.branching, base = P.base_depth, glen = P.golden_len;
  const bool act = lane < nc;
  const int b = act ? lane / C : 0;
  const ts_beam& bm = beams[(size_t)pi * MAXB + b];
  const int L = bm.len;
  // generate_steps raises on a terminal or too-deep context (backend.py:244-246)
  bool bad = act && (L > base + 1 || L < 0 || L >= TS_MAX_DEPTH);
  bool pgold = glen >= 0 && L <= glen;
  uint64_t he0 = fold3(P.seed, 6, (uint64_t)L);
  for (int d = 0; d < L && !bad; ++d) {
    const uint64_t s = bm.path[d];
    he0 = sm64(he0 ^ s);
    if (pgold && P.golden_path[d] != bm.path[d]) pgold = false;
  }
  if (act && !bad && L > 0) {  // _is_terminal(context)
    bool term;
    if (L < base) term = false;
    else if (L >= base + 1) term = true;
    else if (pgold) term = true;
    else term = !((he0 % 2u) == 0u);
    bad = term;
  }
  const unsigned badm = __ballot_sync(FULL, bad);
  if (lane == 0) status[pi] = badm ? TS_INVALID_ARGUMENT : TS_OK;
  if (badm) return;
  const int idx = (lane % C) % branching;
  const int depth = L + 1;
  uint64_t hr = fold3(P.seed, 1, depth), ht = fold3(P.seed, 3, depth), he = fold3(P.seed, 6, depth);
  Agg g;
  g.init();
  for (int d = 0; act && d < L; ++d) {
    const uint64_t s = bm.path[d];
    hr = sm64(hr ^ s);
    ht = sm64(ht ^ s);
    he = sm64(he ^ s);
    g.add(bm.rewards[d], cfg.scheme);
  }
  hr = sm64(hr ^ (uint64_t)idx);
  ht = sm64(ht ^ (uint64_t)idx);
  he = sm64(he ^ (uint64_t)idx);
  const bool gold = pgold && depth <= glen && idx == (int)P.golden_path[depth - 1];
  double reward;
  if (gold) {
    reward = P.golden_rewards[depth - 1];
  } else {
    const bool sr = P.has_shared && depth <= P.hidden_until_depth;
    const double lo = sr ? P.shared_lo : P.off_lo, hi = sr ? P.shared_hi : P.off_hi;
    reward = lo + (hi - lo) * u53(hr);
  }
  bool term;
  if (depth < base) term = false;
  else if (depth >= base + 1) term = true;
  else if (gold) term = true;
  else term = !((he % 2u) == 0u);
  g.add(reward, cfg.scheme);
  const double score = g.value(cfg.scheme);
  const bool open = act && !term;
  const unsigned om = __ballot_sync(FULL, open);
  int rank = 0;
  for (int k = 0; k < nc; ++k) {
    const double sk = __shfl_sync(FULL, score, k);
    rank += (((om >> k) & 1u) && (sk > score || (sk == score && k < lane))) ? 1 : 0;
  }
  if (act) {
    ts_beam_candidate c;
    c.beam = b;
    c.order = lane;
    c.step_ref = idx;
    c.token_count = 40 + (int)(ht % 81u);
    c.prm_reward = reward;
    c.score = score;
    c.is_terminal = term ? 1 : 0;
    c.rank = term ? -2 : (rank < cfg.beam_width ? rank : -1);
    out[(size_t)pi * MAXB + lane] = c;
  }
}

// prune_candidates over caller candidates: rank among the open ones by (-score, order).
__global__ void __launch_bounds__(1024) k_beam_prune(ts_beam_candidate* c, int n, int width) {
  __shared__ double ss[1024];
  __shared__ int so[1024];
  __shared__ unsigned char sopen[1024];
  const int t = threadIdx.x;
  if (t < n) {
    ss[t] = c[t].score;
    so[t] = c[t].order;
    sopen[t] = c[t].is_terminal ? 0 : 1;
  }
  __syncthreads();
  if (t >= n) return;
  if (!sopen[t]) {
    c[t].rank = -2;
    return;
  }
  const double s = ss[t];
  const int o = so[t];
  int rank = 0;
  for (int k = 0; k < n; ++k)
    rank += (sopen[k] && (ss[k] > s || (ss[k] == s && (so[k] < o || (so[k] == o && k < t))))) ? 1 : 0;
  c[t].rank = rank < width ? rank : -1;
}

thread_local std::string g_beam_err;

int beam_check(const ts_beam_config* c) {
  if (!c) return TS_INVALID_ARGUMENT;
  if (c->beam_width < 1 || c->candidates_per_beam < 1 || c->max_depth < 1) {
    g_beam_err = "beam parameters must be positive";
    return TS_INVALID_ARGUMENT;
  }
  if ((long long)c->beam_width * c->candidates_per_beam > MAXB) {
    g_beam_err = "beam_width * candidates_per_beam exceeds TS_BEAM_MAX_CANDIDATES";
    return TS_INVALID_ARGUMENT;
  }
  if (c->scheme < TS_SCHEME_MINIMUM || c->scheme > TS_SCHEME_AVERAGE) {
    g_beam_err = "unknown aggregation scheme";
    return TS_INVALID_ARGUMENT;
  }
  return TS_OK;
}

int beam_grid(int n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int need = (n + BEAM_WARPS - 1) / BEAM_WARPS;
  const int cap = sms * 8;  // 8 CTAs x 4 warps resident per SM
  return need < cap ? need : cap;
}

}  // namespace

extern "C" {

int ts_beam_search(const ts_beam_config* cfg, const ts_problem* dev_problems, int32_t n, ts_beam_result* dev_results,
                   void* stream) {
  int rc = beam_check(cfg);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!dev_problems || !dev_results))) return TS_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  k_beam<<<beam_grid(n), 32 * BEAM_WARPS, 0, (cudaStream_t)stream>>>(*cfg, dev_problems, n, dev_results);
  return cudaGetLastError() == cudaSuccess ? TS_OK : TS_CUDA;
}

int ts_beam_search_host(const ts_beam_config* cfg, const ts_problem* host_problems, int32_t n,
                        ts_beam_result* host_results, void* stream) {
  int rc = beam_check(cfg);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!host_problems || !host_results))) return TS_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ts_problem* dp = nullptr;
  ts_beam_result* dr = nullptr;
  if (cudaMallocAsync((void**)&dp, sizeof(ts_problem) * (size_t)n, s) != cudaSuccess) return TS_CUDA;
  if (cudaMallocAsync((void**)&dr, sizeof(ts_beam_result) * (size_t)n, s) != cudaSuccess) return TS_CUDA;
  cudaMemcpyAsync(dp, host_problems, sizeof(ts_problem) * (size_t)n, cudaMemcpyHostToDevice, s);
  k_beam<<<beam_grid(n), 32 * BEAM_WARPS, 0, s>>>(*cfg, dp, n, dr);
  cudaMemcpyAsync(host_results, dr, sizeof(ts_beam_result) * (size_t)n, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(dp, s);
  cudaFreeAsync(dr, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? TS_OK : TS_CUDA;
}

int ts_beam_expand(const ts_beam_config* cfg, const ts_problem* dev_problems, int32_t n, const ts_beam* dev_beams,
                   const int32_t* dev_counts, ts_beam_candidate* dev_cands, int32_t* dev_status, void* stream) {
  int rc = beam_check(cfg);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!dev_problems || !dev_beams || !dev_counts || !dev_cands || !dev_status)))
    return TS_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  k_beam_expand<<<(n + BEAM_WARPS - 1) / BEAM_WARPS, 32 * BEAM_WARPS, 0, (cudaStream_t)stream>>>(
      *cfg, dev_problems, n, dev_beams, dev_counts, dev_cands, dev_status);
  return cudaGetLastError() == cudaSuccess ? TS_OK : TS_CUDA;
}

int ts_beam_prune(ts_beam_candidate* dev_cands, int32_t n, int32_t beam_width, void* stream) {
  if (n < 0 || n > 1024 || beam_width < 1 || (n > 0 && !dev_cands)) return TS_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  k_beam_prune<<<1, 1024, 0, (cudaStream_t)stream>>>(dev_cands, n, beam_width);
  return cudaGetLastError() == cudaSuccess ? TS_OK : TS_CUDA;
}

}  // extern "C"
