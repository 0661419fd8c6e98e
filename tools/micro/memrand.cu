// Microbenchmark: random-access costs that bound the batch-update and discharge
// phases on B200 -- random 4-B loads / atomics (with and without return) into a
// 512 MB array, dependent-chain latency, and single-address claim counters.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// each thread: `per` random accesses, all independent (mode 0 ldcg, 1 atomicAdd ret, 2 red)
__global__ void k_rand(int *a, uint32_t mask, int per, int mode, int *sink) {
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0;
  for (int j = 0; j < per; j++) {
    const uint32_t i = hash32(gt * 977u + j * 0x9e3779b9u) & mask;
    if (mode == 0) acc += __ldcg(a + i);
    else if (mode == 1) acc += atomicAdd(a + i, 1);
    else atomicAdd(a + i, 1);
  }
  if (acc == 0x7fffffff) *sink = acc;
}

// dependent chain: next index = f(loaded value)
__global__ void k_chain(const int *a, uint32_t mask, int steps, int *sink) {
  uint32_t i = hash32(blockIdx.x * blockDim.x + threadIdx.x) & mask;
  for (int s = 0; s < steps; s++) i = (uint32_t)(__ldcg(a + i) + hash32(i)) & mask;
  if (i == 0xffffffffu) *sink = i;
}

// claims: every group of `g` lanes does one atomicAdd on a single counter
__global__ void k_claim(int *c, int g) {
  if ((threadIdx.x % g) == 0) atomicAdd(c, 1);
}
__global__ void k_claim_ret(int *c, int g, int *sink) {
  if ((threadIdx.x % g) == 0) { int x = atomicAdd(c, 1); if (x == -5) *sink = x; }
}

int main() {
  const size_t N = 1ull << 27;  // 128M ints = 512 MB
  int *a, *sink, *c;
  cudaMalloc(&a, N * 4); cudaMemset(a, 0, N * 4);
  cudaMalloc(&sink, 4); cudaMalloc(&c, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 2, nt = 512;
  const double nthr = (double)grid * nt;
  auto tm = [&](auto launch) {
    launch(); cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms * 1e3;  // us
  };
  const char *names[3] = {"ldcg", "atomicAdd(ret)", "red"};
  for (uint32_t mbits : {20u, 27u}) {
    for (int mode = 0; mode < 3; mode++)
      for (int per : {1, 4, 16}) {
        float us = tm([&] { k_rand<<<grid, nt>>>(a, (1u << mbits) - 1, per, mode, sink); });
        printf("rand %-15s span %4d MB per-thread %2d: %8.1f us  %6.1f G acc/s\n", names[mode], (4 << mbits) >> 20, per,
               us, nthr * per / us * 1e-3);
      }
  }
  for (int steps : {16}) {
    float us = tm([&] { k_chain<<<1, 1>>>(a, (1u << 27) - 1, steps, sink); });
    printf("chain 1 thread, 512 MB: %.0f ns/step\n", us * 1e3 / steps);
    us = tm([&] { k_chain<<<1, 1>>>(a, (1u << 20) - 1, steps, sink); });
    printf("chain 1 thread, 4 MB (L2): %.0f ns/step\n", us * 1e3 / steps);
    us = tm([&] { k_chain<<<grid, nt>>>(a, (1u << 27) - 1, steps, sink); });
    printf("chain all threads, 512 MB: %.0f ns/step (%.1f G acc/s)\n", us * 1e3 / steps, nthr * steps / us * 1e-3);
  }
  for (int g : {512, 32, 8, 1}) {
    float us = tm([&] { k_claim<<<grid, nt>>>(c, g); });
    float us2 = tm([&] { k_claim_ret<<<grid, nt>>>(c, g, sink); });
    printf("single-address claims: %7.0f ops: red %.1f us, atomic-ret %.1f us\n", nthr / g, us, us2);
  }
  float us = tm([&] { k_claim<<<1, 32>>>(c, 32); });
  printf("empty-ish launch: %.1f us\n", us);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
