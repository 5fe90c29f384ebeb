// steps.cu — generate_steps (reference backend.py:230-269) as a batched device
// operator: the synthetic LLM/PRM backend the engine replays inside its wave
// kernels, exposed for callers that expand their own trees.
//
// One warp per (problem, context path); lane j is candidate j (width <= 32).
// Every key of the reference's RNG table (backend.py:49-57) is a mix() fold
// of (seed, tag, len, path..., [i]); the lanes fold the shared prefix for
// their tags and finish with their own child index.  The prior total is
// CPython's float sum (Neumaier) over the distinct children in order, on one
// lane, so the normalised priors are bit-identical.  -fmad=false.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/treeserve_b200.h"
#include "exact.cuh"
#include "rng.cuh"

namespace {

using tsx::MIX_INIT;
using tsx::sm64;
using tsx::u53;

constexpr unsigned FULL = 0xffffffffu;
constexpr int SW = 4;  // warps per CTA

__device__ __forceinline__ uint64_t fold3(uint64_t seed, uint64_t tag, uint64_t len) {
  return sm64(sm64(sm64(MIX_INIT ^ seed) ^ tag) ^ len);
}

__global__ void __launch_bounds__(32 * SW) k_generate_steps(const ts_problem* __restrict__ probs, int n,
                                                            const uint8_t* __restrict__ paths,
                                                            const int32_t* __restrict__ lens, int width,
                                                            ts_step_candidate* __restrict__ out,
                                                            int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31, w = blockIdx.x * SW + (threadIdx.x >> 5);
  if (w >= n) return;
  const ts_problem& P = probs[w];
  const uint8_t* path = paths + (size_t)w * TS_MAX_DEPTH;
  const int L = lens[w];
  const int b = P.branching, base = P.base_depth, glen = P.golden_len;
  // context checks (backend.py:244-246): too deep, or terminal
  bool bad = L < 0 || L > base + 1 || L >= TS_MAX_DEPTH;
  bool pgold = !bad && glen >= 0 && L <= glen;
  uint64_t hx = fold3(P.seed, 6, (uint64_t)L), hp = fold3(P.seed, 2, (uint64_t)L);
  const int depth = L + 1;
  uint64_t hr = fold3(P.seed, 1, (uint64_t)depth), ht = fold3(P.seed, 3, (uint64_t)depth),
           he = fold3(P.seed, 6, (uint64_t)depth);
  for (int d = 0; !bad && d < L; ++d) {
    const uint64_t s = path[d];
    hx = sm64(hx ^ s);
    hp = sm64(hp ^ s);
    hr = sm64(hr ^ s);
    ht = sm64(ht ^ s);
    he = sm64(he ^ s);
    if (pgold && P.golden_path[d] != path[d]) pgold = false;
  }
  if (!bad && L > 0) {
    bool term;
    if (L < base) term = false;
    else if (L >= base + 1) term = true;
    else if (pgold) term = true;
    else term = !((hx % 2u) == 0u);
    bad = term;
  }
  if (lane == 0) status[w] = bad ? TS_INVALID_ARGUMENT : TS_OK;
  if (bad) return;
  const int distinct = width < b ? width : b;
  // raw priors of the distinct children, then sum() in child order on lane 0
  const double raw = lane < distinct ? 0.5 + u53(sm64(hp ^ (uint64_t)lane)) : 0.0;
  double total = 0.0;
  {
    double f = 0.0, c = 0.0;
    for (int i = 0; i < distinct; ++i) {
      const double x = __shfl_sync(FULL, raw, i);
      if (i == 0) { f = x; continue; }
      const double t = f + x;
      if (fabs(f) >= fabs(x)) c += (f - t) + x;
      else c += (x - t) + f;
      f = t;
    }
    if (c != 0.0 && isfinite(c)) f += c;
    total = f;
  }
  const int index = lane % b;
  const double prior = __shfl_sync(FULL, raw, index % distinct) / total;
  if (lane >= width) return;
  hr = sm64(hr ^ (uint64_t)index);
  ht = sm64(ht ^ (uint64_t)index);
  he = sm64(he ^ (uint64_t)index);
  const bool gold = pgold && depth <= glen && index == (int)P.golden_path[depth - 1];
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
  ts_step_candidate o;
  o.step_ref = index;
  o.token_count = 40 + (int)(ht % 81u);
  o.prior = prior;
  o.prm_reward = reward;
  o.is_terminal = term ? 1 : 0;
  o._pad = 0;
  out[(size_t)w * width + lane] = o;
}

}  // namespace

extern "C" {

int ts_generate_steps(const ts_problem* dev_problems, int32_t n, const uint8_t* dev_paths, const int32_t* dev_lens,
                      int32_t width, ts_step_candidate* dev_out, int32_t* dev_status, void* stream) {
  if (width < 1 || width > TS_MAX_WIDTH || n < 0) return TS_INVALID_ARGUMENT;
  if (n > 0 && (!dev_problems || !dev_paths || !dev_lens || !dev_out || !dev_status)) return TS_INVALID_ARGUMENT;
  if (n == 0) return TS_OK;
  k_generate_steps<<<(n + SW - 1) / SW, 32 * SW, 0, (cudaStream_t)stream>>>(dev_problems, n, dev_paths, dev_lens,
                                                                          width, dev_out, dev_status);
  return cudaGetLastError() == cudaSuccess ? TS_OK : TS_CUDA;
}

}  // extern "C"
