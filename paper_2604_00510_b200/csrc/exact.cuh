// exact.cuh — bit-exact numerics shared by the engine and the standalone
// policy kernels: the exact fixed-point image of CPython's float sum() and a
// device log1p equal to the host libm's.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/treeserve_b200.h"

namespace tsx {

typedef unsigned __int128 u128;

// Exact fixed-point image of a score (LSB 2^-64).  Returns false when the
// score has bits below 2^-64 (then the sum falls back to the sequential loop).
__device__ __forceinline__ bool to_fixed(double x, u128& out) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  int ex = (int)((b >> 52) & 0x7FF);
  uint64_t m = b & ((1ull << 52) - 1);
  if (ex == 0) {
    out = 0;
    return m == 0;
  }
  m |= 1ull << 52;
  int sh = ex - 1075 + 64;  // value = m * 2^(ex-1075) = (m << sh) * 2^-64
  if (sh < 0 || sh > 74) return false;
  out = (u128)m << sh;
  return true;
}
// Round-to-nearest-even of fixed-point value × 2^-64.
__device__ inline double fixed_to_double(u128 v) {
  if (v == 0) return 0.0;
  uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
  int p = hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
  if (p <= 52) return (double)lo * 0x1p-64;
  int sh = p - 52;
  uint64_t mant = (uint64_t)(v >> sh);
  u128 rem = v & (((u128)1 << sh) - 1);
  u128 half = (u128)1 << (sh - 1);
  if (rem > half || (rem == half && (mant & 1))) {
    ++mant;
    if (mant == (1ull << 53)) { mant >>= 1; ++sh; }
  }
  return ldexp((double)mant, sh - 64);
}
// log1p equal, bit for bit, to the host libm CPython's math.log1p calls
// (scheduler.py:128).  glibc 2.39 on x86-64 dispatches log1p to its FMA build
// of the fdlibm algorithm with the Estrin-form polynomial; the fused
// operations below are exactly the ones that build contracts (read from its
// code generation) and the file is compiled with -fmad=false so nothing else
// fuses.  Validated against the host libm on 3.4e7 arguments
// (tests/test_policy_cpu.py pins the host-side restatement; the GPU test
// compares the device with math.log1p).
__host__ __device__ inline double libm_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               two54 = 1.80143985094819840000e+16, Lp1 = 6.666666666666735130e-01,
               Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01,
               Lp6 = 1.531383769920937332e-01, Lp7 = 1.479819860511658591e-01;
#ifdef __CUDA_ARCH__
#define TSX_FMA(a, b, c) __fma_rn((a), (b), (c))
  const uint64_t bx = (uint64_t)__double_as_longlong(x);
#else
#define TSX_FMA(a, b, c) std::fma((a), (b), (c))
  uint64_t bx;
  std::memcpy(&bx, &x, 8);
#endif
  auto hi_of = [](double v) -> int32_t {
#ifdef __CUDA_ARCH__
    return (int32_t)((uint64_t)__double_as_longlong(v) >> 32);
#else
    uint64_t b;
    std::memcpy(&b, &v, 8);
    return (int32_t)(b >> 32);
#endif
  };
  auto set_hi = [](double v, int32_t h) -> double {
#ifdef __CUDA_ARCH__
    uint64_t b = (uint64_t)__double_as_longlong(v);
    b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
    return __longlong_as_double((long long)b);
#else
    uint64_t b;
    std::memcpy(&b, &v, 8);
    b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
    std::memcpy(&v, &b, 8);
    return v;
#endif
  };
  const int32_t hx = (int32_t)(bx >> 32), ax = hx & 0x7fffffff;
  double f = 0.0, c = 0.0, u;
  int32_t k = 1, hu = 0;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) {  // x <= -1
      if (x == -1.0) return -two54 / 0.0;
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (two54 + x > 0.0 && ax < 0x3c900000) return x;
      return TSX_FMA(-(x * x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec4) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = hi_of(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = hi_of(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = set_hi(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = set_hi(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (0.5 * f) * f;
  const double dk = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = TSX_FMA(dk, ln2_lo, c);
      return TSX_FMA(dk, ln2_hi, c);
    }
    const double R = TSX_FMA(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    return TSX_FMA(dk, ln2_hi, -((R - TSX_FMA(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = TSX_FMA(z, Lp3, Lp2), R3 = TSX_FMA(z, Lp5, Lp4), R4 = TSX_FMA(z, Lp7, Lp6);
  const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
  const double R = TSX_FMA(z6, R4, TSX_FMA(z4, R3, TSX_FMA(z, Lp1, z2 * R2)));
  const double sh = s * (hfsq + R);
  if (k == 0) return f - (hfsq - sh);
  return TSX_FMA(dk, ln2_hi, -((hfsq - (TSX_FMA(dk, ln2_lo, c) + sh)) - f));
#undef TSX_FMA
}
// ---- aggregate_trajectory (scoring.py:106-116), incremental along a path ----
struct Agg {
  double a, c;
  int n;
  __device__ __forceinline__ void init() { a = 1.0; c = 0.0; n = 0; }
  __device__ __forceinline__ void add(double r, int scheme) {
    if (scheme == TS_SCHEME_PRODUCT) {
      a = a * r;  // math.prod: 1 * r0 * r1 ... left to right
    } else if (scheme == TS_SCHEME_MINIMUM) {
      a = (n == 0 || r < a) ? r : a;
    } else if (n == 0) {  // builtin sum(): 0 + r0, then Neumaier (CPython >= 3.12)
      a = r;
      c = 0.0;
    } else {
      double t = a + r;
      if (fabs(a) >= fabs(r)) c += (a - t) + r;
      else c += (r - t) + a;
      a = t;
    }
    ++n;
  }
  __device__ __forceinline__ double value(int scheme) const {
    if (scheme == TS_SCHEME_PRODUCT || scheme == TS_SCHEME_MINIMUM) return a;
    double s = a;
    if (c != 0.0 && isfinite(c)) s += c;
    if (scheme == TS_SCHEME_SUM) return s;
    return s / (double)n;
  }
};

}  // namespace tsx
