// Dependent-chain latency (cycles per op) of the primitives on the wave
// kernel's critical path, one warp, B200.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cstdint>

__global__ void k(long long* out, double* sink, int n) {
  const int lane = threadIdx.x;
  double x = 1.0 + lane * 1e-3, y = 3.0 + lane;
  long long t0, t1;
  unsigned long long u = 0x1234567ull + lane;
  int iv = 7 + lane;
  long long lv = 7 + lane;
#define MEASURE(idx, body)            \
  t0 = clock64();                     \
  for (int i = 0; i < n; ++i) { body; } \
  t1 = clock64();                     \
  if (lane == 0) out[idx] = (t1 - t0) / n;
  MEASURE(0, x = x * 1.0000001 + 1e-9)                    // DFMA-ish (mul+add, no contraction)
  MEASURE(1, x = y / x)                                    // DDIV
  MEASURE(2, x = sqrt(x + 1.0))                            // DSQRT
  MEASURE(3, x = (double)(lv + (long long)(x > 1.0)))      // I2F.F64.S64
  MEASURE(4, x = (double)(iv + (int)(x > 1.0)))            // I2F.F64.S32
  MEASURE(5, u = (u ^ (u >> 30)) * 0xBF58476D1CE4E5B9ull)  // 64-bit xorshift-multiply
  MEASURE(6, iv = __reduce_max_sync(0xffffffffu, (unsigned)iv) + 1)  // REDUX
  MEASURE(7, iv = __shfl_sync(0xffffffffu, iv, (lane + 1) & 31) + 1)  // SHFL
  MEASURE(8, x = (double)(u >> 11) * 0x1p-53 + x; u += (unsigned long long)x)  // u53 + chain
  sink[lane] = x + y + (double)u + iv;
}

int main() {
  long long* out;
  double* sink;
  cudaMalloc(&out, 16 * sizeof(long long));
  cudaMalloc(&sink, 32 * sizeof(double));
  k<<<1, 32>>>(out, sink, 1000);
  k<<<1, 32>>>(out, sink, 10000);
  long long h[16];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"dmul+dadd", "ddiv", "dsqrt", "i2f.f64.s64", "i2f.f64.s32", "xorshift-mul64",
                         "redux.max", "shfl", "u53+f2i chain"};
  for (int i = 0; i < 9; ++i) printf("%-16s %lld cycles\n", names[i], h[i]);
  return 0;
}
