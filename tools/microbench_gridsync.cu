// Cost of a grid-wide barrier (cooperative launch) on this GPU: K syncs in one kernel.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(sink, 1);
    g.sync();
  }
}
int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  for (int G : {2, 16, 32, 148}) {
    for (int iters : {1, 101}) {
      void* args[] = {&iters, &sink};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) cudaLaunchCooperativeKernel((void*)k, G, 256, args, 0, 0);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) cudaLaunchCooperativeKernel((void*)k, G, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("G=%d iters=%d: %.2f us per launch\n", G, iters, ms * 100.0f);
    }
  }
  return 0;
}
