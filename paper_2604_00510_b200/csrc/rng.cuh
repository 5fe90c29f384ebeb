// rng.cuh — the reference's keyed RNG primitives (rng.py:15-32), shared by the
// engine and the beam kernel.
#pragma once
#include <cstdint>

namespace tsx {

// ---- rng.py ------------------------------------------------------------------
// _splitmix64 (rng.py:15-19)
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x = x + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
constexpr uint64_t MIX_INIT = 0x8E12F5A34C29D96Bull;  // mix() initial state (rng.py:24)
// uniform (rng.py:30-32): top 53 bits scaled by 2^-53 (exact)
__host__ __device__ __forceinline__ double u53(uint64_t h) { return (double)(h >> 11) * 0x1p-53; }


}  // namespace tsx
