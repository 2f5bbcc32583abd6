// red_issue.cu -- issue cost of one warp's red.global.add.f64 instructions (one warp per SM,
// K back-to-back reductions, clock64 around the loop), by address pattern:
//   rand32   32 lanes, 32 random lines (the update kernel's unpaired scatter)
//   paired   32 lanes, 16 random lines, lanes 2k/2k+1 on one 16-B pair (the paired scatter)
//   line     32 lanes, one 32-B sector (8 words)
//   half     16 active lanes, 16 random lines
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/red_issue tools/red_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int PAT>
__global__ void k(double* tab, uint32_t d, int K, unsigned long long* cyc) {
  const uint32_t lane = threadIdx.x & 31;
  double* a[64];
#pragma unroll
  for (int it = 0; it < 64; ++it) {
    uint32_t v;
    if (PAT == 0) v = hash32(blockIdx.x * 7919u + it * 32u + lane) % d * 2;
    else if (PAT == 1) v = (hash32(blockIdx.x * 7919u + it * 32u + (lane >> 1)) % d) * 2 + (lane & 1);
    else if (PAT == 2) v = (hash32(blockIdx.x * 7919u + it) % d) * 4 + (lane & 3);
    else v = hash32(blockIdx.x * 7919u + it * 32u + lane) % d * 2;
    a[it] = tab + v;
  }
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll
  for (int it = 0; it < 64; ++it) {
    if (PAT != 3 || lane < 16)
      asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a[it]), "d"(1.0) : "memory");
  }
  const long long t1 = clock64();
  if (lane == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t d = 3231961;
  double* tab; cudaMalloc(&tab, (size_t)d * 32); cudaMemset(tab, 0, (size_t)d * 32);
  unsigned long long* cyc; cudaMalloc(&cyc, 8);
  const char* names[4] = {"rand32", "paired", "line", "half"};
  printf("{");
  for (int pat = 0; pat < 4; ++pat) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      if (pat == 0) k<0><<<sms, 32>>>(tab, d, 64, cyc);
      if (pat == 1) k<1><<<sms, 32>>>(tab, d, 64, cyc);
      if (pat == 2) k<2><<<sms, 32>>>(tab, d, 64, cyc);
      if (pat == 3) k<3><<<sms, 32>>>(tab, d, 64, cyc);
      cudaDeviceSynchronize();
    }
    unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s\"%s_cycles_per_red_instr\": %.1f", pat ? ", " : "", names[pat], (double)c / sms / 64.0);
  }
  printf("}\n");
  return 0;
}
