// Cost of cooperative grid.sync() on this GPU, by grid size (tools/r2; informs eig_sym.cu).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int n, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) *sink = n;
}
int main() {
  int* s; cudaMalloc(&s, 4);
  for (int blocks : {32, 64, 128, 148, 296, 592}) {
    for (int threads : {256, 1024}) {
      int n = 2000;
      void* args[] = {&n, &s};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("blocks %d threads %d: %s %.3f us per grid.sync\n", blocks, threads, cudaGetErrorString(e), ms * 1e3 / n);
    }
  }
  return 0;
}
