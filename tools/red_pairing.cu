// red_pairing.cu -- does one RED instruction whose lanes hit the x and abar words of the
// same 16-byte {x, abar} pair (lanes 2k, 2k+1) cost the L2 one request instead of two?
// Per "entry": x += 1, abar += 1 on a random pair of a d-pair table.
//   A (the update kernel today): lane j owns entry j; two RED instructions (x, then abar)
//   B (paired): lane j adds word (j & 1) of entry (j >> 1); two RED instructions cover
//     the same 32 entries (each instruction: 16 entries x 2 words)
// hot: k pairs 1 KiB apart, one pair load + the two adds per update, lane 0 (A) or lanes
// 0-1 (B) of each warp.  Prints one JSON object.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/red_pairing tools/red_pairing.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ void red(double* a, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__global__ void k_cold(double* tab, uint32_t d, int iters, int paired) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31, wbase = tid - lane;
  for (int it = 0; it < iters; ++it) {
    if (!paired) {
      const uint32_t v = hash32((wbase + lane) * 977u + it * 0x9E3779B9u) % d;
      red(tab + 2 * (size_t)v, 1.0);
      red(tab + 2 * (size_t)v + 1, 1.0);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t e = 16 * h + (lane >> 1);
        const uint32_t v = hash32((wbase + e) * 977u + it * 0x9E3779B9u) % d;
        red(tab + 2 * (size_t)v + (lane & 1), 1.0);
      }
    }
  }
}
__global__ void k_hot(double* tab, uint32_t k, int iters, int paired) {
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (lane >= (paired ? 2u : 1u)) return;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double* a = tab + (size_t)((wid + it) % k) * 128;
    double v0, v1;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v0), "=d"(v1) : "l"(a));
    acc += v0 + v1;
    if (!paired) {
      red(a, 1.0 + acc * 0.0);
      red(a + 1, 1.0 + acc * 0.0);
    } else {
      red(a + lane, 1.0 + acc * 0.0);
    }
  }
}
template <class F> float best_ms(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d", sms);
  for (uint32_t d : {47236u, 3231961u}) {
    double* tab; CK(cudaMalloc(&tab, (size_t)d * 16)); CK(cudaMemset(tab, 0, (size_t)d * 16));
    const int blocks = sms * 8, threads = 256, iters = 256;
    const double entries = (double)blocks * threads * iters;
    for (int paired : {0, 1}) {
      float ms = best_ms([&] { k_cold<<<blocks, threads>>>(tab, d, iters, paired); });
      printf(", \"cold_d%u_%s_entries_per_s\": %.4g", d, paired ? "paired" : "split", entries / ms * 1e3);
    }
    CK(cudaFree(tab));
  }
  for (uint32_t k : {1u, 10u}) {
    double* tab; CK(cudaMalloc(&tab, (size_t)k * 1024)); CK(cudaMemset(tab, 0, (size_t)k * 1024));
    const int blocks = sms * 8, threads = 256, iters = 32;
    const double upd = (double)blocks * (threads / 32) * iters;
    for (int paired : {0, 1}) {
      float ms = best_ms([&] { k_hot<<<blocks, threads>>>(tab, k, iters, paired); });
      printf(", \"hot_k%u_%s_updates_per_s_per_pair\": %.4g", k, paired ? "paired" : "split", upd / ms * 1e3 / k);
    }
    CK(cudaFree(tab));
  }
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
