// Microbenchmark: cost of a grid-wide barrier in a persistent cooperative kernel on
// B200 -- cooperative_groups grid.sync() vs a hand-rolled sense-reversing barrier
// (one relaxed atomic arrive per CTA + acquire spin on a generation word).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int *sink) {
  cg::grid_group g = cg::this_grid();
  int acc = 0;
  for (int i = 0; i < iters; i++) { acc += threadIdx.x; g.sync(); }
  if (acc == -1) *sink = acc;
}

struct Bar { unsigned int count; unsigned int gen; };

__device__ __forceinline__ void bar_sync(Bar *b, unsigned int nblocks, unsigned int &gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int my = gen;
    __threadfence();
    const unsigned int arrived = atomicAdd(&b->count, 1u) + 1;
    if (arrived == nblocks) {
      b->count = 0;
      __threadfence();
      atomicExch(&b->gen, my + 1);
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&b->gen));
      } while (cur == my);
    }
  }
  gen++;
  __syncthreads();
}

__global__ void k_custom(int iters, Bar *b, int *sink) {
  unsigned int gen = 0;
  int acc = 0;
  for (int i = 0; i < iters; i++) { acc += threadIdx.x; bar_sync(b, gridDim.x, gen); }
  if (acc == -1) *sink = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int *sink; cudaMalloc(&sink, 4);
  Bar *b; cudaMalloc(&b, sizeof(Bar)); cudaMemset(b, 0, sizeof(Bar));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  for (int nt : {256, 512, 1024}) {
    for (int per : {1, 2, 4}) {
      if (nt * per > 2048) continue;
      int grid = sms * per;
      void *args[] = {(void *)&iters, (void *)&sink};
      cudaLaunchCooperativeKernel((void *)k_cg, grid, nt, args, 0, 0);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void *)k_cg, grid, nt, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      void *args2[] = {(void *)&iters, (void *)&b, (void *)&sink};
      cudaMemset(b, 0, sizeof(Bar));
      cudaLaunchCooperativeKernel((void *)k_custom, grid, nt, args2, 0, 0);
      cudaMemset(b, 0, sizeof(Bar));
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void *)k_custom, grid, nt, args2, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms2; cudaEventElapsedTime(&ms2, e0, e1);
      printf("threads %4d x %d/SM (grid %d): cg %.2f us/sync, custom %.2f us/sync  %s\n", nt, per, grid,
             1e3 * ms / iters, 1e3 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
