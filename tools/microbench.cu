// microbench.cu -- roofline denominators for the ASAGA update kernel on B200
// (SURVEY.md section 8(d), M1-M5).  Prints one JSON object.
//   M0 hbm_copy      cudaMemcpy D2D (r+w bytes), sanity vs MEASURED_PEAKS.json
//   M1 hbm_rows      random rows of s entries (int32 index + fp64 value) from a
//                    4+ GB CSR-like array: the A3 row fetch
//   M2 l2_gather     random 256-bit .cg loads of 32-byte {x, abar, D} records,
//                    L2-resident tables of d records: the A4/A6 gathers
//   M3 red_distinct  red.global.add.f64 to uniformly random records (d records)
//   M4 red_same      red.global.add.f64 to k in {1, 10} addresses (hot columns)
//   M5 red_zipf      red.global.add.f64 with Zipf(s) column popularity over d
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      fprintf(stderr, "%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__);   \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

struct __align__(32) Rec { double a, b, c, d; };

__global__ void k_rows(const int32_t* __restrict__ idx, const double* __restrict__ val, uint64_t N,
                       int s, int rows_per_warp, uint32_t salt, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double acc = 0;
  for (int r = 0; r < rows_per_warp; ++r) {
    uint64_t start = ((uint64_t)hash32((uint32_t)(w * rows_per_warp + r) ^ salt) * 2654435761ull) % (N - s);
    for (int k = lane; k < s; k += 32) acc += __ldg(idx + start + k) * __ldg(val + start + k);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_gather(const Rec* __restrict__ tab, uint32_t d, int iters, uint32_t salt, double* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    uint32_t v = hash32(tid * 977u + it * 0x9E3779B9u + salt) % d;
    double a, b, c, e;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(e) : "l"(tab + v));
    acc += a + b + c;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_red_random(double* tab, uint32_t d, uint32_t stride, int iters, uint32_t salt) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    uint32_t v = hash32(tid * 977u + it * 0x9E3779B9u + salt) % d;
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(tab + (size_t)v * stride), "d"(1.0) : "memory");
  }
}

__global__ void k_red_same(double* tab, uint32_t k, uint32_t stride, int iters) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint32_t v = (tid + it) % k;
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(tab + (size_t)v * stride), "d"(1.0) : "memory");
  }
}

// one address per warp: lane 0 loads (.cg) then REDs -- the per-line service rate
// of the update kernel's hot-feature pattern (1 load + 1 RED per update per line)
__global__ void k_ldred_hot(double* tab, uint32_t k, uint32_t stride, int iters, int do_load) {
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double* a = tab + (size_t)((wid + it) % k) * stride;
    double v = 0;
    if (do_load) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(a));
    acc += v;
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a), "d"(1.0 + acc * 0.0) : "memory");
  }
}

// the update kernel's exact hot-feature pattern: one 16-byte {x, abar} .na load
// + two REDs (x, abar) into that pair, per "update", k pairs 1 KiB apart
__global__ void k_pair_hot(double* tab, uint32_t k, int iters) {
  const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double* a = tab + (size_t)((wid + it) % k) * 128;
    double v0, v1;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v0), "=d"(v1) : "l"(a));
    acc += v0 + v1;
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a), "d"(1.0 + acc * 0.0) : "memory");
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a + 1), "d"(1.0 + acc * 0.0) : "memory");
  }
}

// TMA bulk reduction: one cp.reduce.async.bulk .add.f64 of 16 bytes per pair
// (both x and abar) from shared memory -- UBLKRED, issued lane by lane.
// hot: lane 0 of each warp on k pairs 1 KiB apart (with the pair load);
// random: every lane on a random pair of a d-pair table.
__global__ void k_bulk_pair(double* tab, uint32_t k, uint32_t d, int iters, int hot, int load = 1) {
  __shared__ __align__(16) double s[2 * 256];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (hot && (threadIdx.x & 31) != 0) return;
  s[2 * threadIdx.x] = 1.0;
  s[2 * threadIdx.x + 1] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s + 2 * threadIdx.x);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double* a = hot ? tab + (size_t)(((tid >> 5) + it) % k) * 128
                    : tab + (size_t)(hash32(tid * 977u + it * 0x9E3779B9u) % d) * 2;
    if (hot && load) {
      double v0, v1;
      asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v0), "=d"(v1) : "l"(a));
      acc += v0 + v1;
    }
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 16;" ::"l"(a),
                 "r"(sa + (acc == 12345.0 ? 16u : 0u)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// latency of one "sample's" gathers: a warp issues NCH x 32-lane scattered 16-byte
// .na loads (a row of NCH*32 entries), waits, and derives the next addresses from
// the data -- cycles per round, one warp per SM (the W = 148 regime)
__global__ void k_gather_lat(const double2* tab, uint32_t d, int nch, int rounds,
                             unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  uint32_t seed = blockIdx.x * 7919u + lane;
  double acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    double2 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < nch) {
        uint32_t c = hash32(seed + j * 131u + r * 977u) % d;
        asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[j].x), "=d"(v[j].y) : "l"(tab + c) : "memory");
      } else {
        v[j] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j].x + v[j].y;
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    seed += (uint32_t)(acc == 1.2345 ? 1 : 0);  // true data dependence of the next round
  }
  long long t1 = clock64();
  if (lane == 0) atomicAdd(out, (unsigned long long)(t1 - t0));
  if (acc == 1.2345) out[1] = 1;  // keep the loads
}

__global__ void k_red_list(double* tab, const uint32_t* __restrict__ list, uint64_t m, uint32_t stride) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x)
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(tab + (size_t)__ldg(list + j) * stride), "d"(1.0) : "memory");
}

template <typename F>
float best_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  CK(cudaGetLastError());
  return best;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  int clk = 0, memclk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, dev);
  std::string js = "{";
  char buf[512];
  snprintf(buf, sizeof buf,
           "\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"persisting_l2_max\": %d, "
           "\"smem_per_sm\": %zu, \"sm_clock_khz\": %d, \"mem_clock_khz\": %d",
           prop.name, sms, prop.l2CacheSize, prop.persistingL2CacheMaxSize,
           prop.sharedMemPerMultiprocessor, clk, memclk);
  js += buf;

  // M0 copy
  {
    size_t bytes = (size_t)2 << 30;
    void *a, *b;
    CK(cudaMalloc(&a, bytes));
    CK(cudaMalloc(&b, bytes));
    CK(cudaMemset(a, 1, bytes));
    float ms = best_ms([&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice)); });
    snprintf(buf, sizeof buf, ", \"hbm_copy_gbs\": %.1f", 2.0 * bytes / ms / 1e6);
    js += buf;
    CK(cudaFree(a));
    CK(cudaFree(b));
  }
  double* out;
  CK(cudaMalloc(&out, 64));
  // M1 random rows
  {
    const uint64_t N = (uint64_t)1 << 28;  // 268M entries: 1 GiB idx + 2 GiB val
    int32_t* idx;
    double* val;
    CK(cudaMalloc(&idx, N * 4));
    CK(cudaMalloc(&val, N * 8));
    CK(cudaMemset(idx, 0, N * 4));
    CK(cudaMemset(val, 0, N * 8));
    js += ", \"hbm_rows\": {";
    int first = 1;
    for (int s : {12, 73, 116}) {
      const int rpw = 64;
      const int blocks = sms * 8, threads = 256;
      const double rows = (double)blocks * threads / 32 * rpw;
      float ms = best_ms([&] { k_rows<<<blocks, threads>>>(idx, val, N, s, rpw, 17u, out); });
      snprintf(buf, sizeof buf, "%s\"s%d\": {\"rows_per_s\": %.4g, \"useful_gbs\": %.1f}", first ? "" : ", ", s,
               rows / ms * 1e3, rows * s * 12.0 / ms / 1e6);
      js += buf;
      first = 0;
    }
    js += "}";
    CK(cudaFree(idx));
    CK(cudaFree(val));
  }
  // M2 gathers, M3 random REDs
  {
    js += ", \"l2_gather\": {";
    int first = 1;
    for (uint32_t d : {54u, 47236u, 3231961u}) {
      Rec* tab;
      CK(cudaMalloc(&tab, (size_t)d * sizeof(Rec)));
      CK(cudaMemset(tab, 0, (size_t)d * sizeof(Rec)));
      const int blocks = sms * 8, threads = 256, iters = 256;
      const double g = (double)blocks * threads * iters;
      float ms = best_ms([&] { k_gather<<<blocks, threads>>>(tab, d, iters, 3u, out); });
      snprintf(buf, sizeof buf, "%s\"d%u\": {\"gathers_per_s\": %.4g, \"sector_gbs\": %.1f}", first ? "" : ", ", d,
               g / ms * 1e3, g * 32.0 / ms / 1e6);
      js += buf;
      first = 0;
      CK(cudaFree(tab));
    }
    js += "}, \"red_distinct\": {";
    first = 1;
    for (uint32_t d : {47236u, 3231961u}) {
      double* tab;
      CK(cudaMalloc(&tab, (size_t)d * 32));
      CK(cudaMemset(tab, 0, (size_t)d * 32));
      const int blocks = sms * 8, threads = 256, iters = 256;
      const double g = (double)blocks * threads * iters;
      float ms = best_ms([&] { k_red_random<<<blocks, threads>>>(tab, d, 4, iters, 5u); });
      snprintf(buf, sizeof buf, "%s\"d%u\": {\"reds_per_s\": %.4g}", first ? "" : ", ", d, g / ms * 1e3);
      js += buf;
      first = 0;
      CK(cudaFree(tab));
    }
    js += "}, \"red_same\": {";
    first = 1;
    for (uint32_t k : {1u, 10u, 54u}) {
      double* tab;
      CK(cudaMalloc(&tab, (size_t)k * 32));
      CK(cudaMemset(tab, 0, (size_t)k * 32));
      const int blocks = sms * 4, threads = 256, iters = 64;
      const double g = (double)blocks * threads * iters;
      float ms = best_ms([&] { k_red_same<<<blocks, threads>>>(tab, k, 4, iters); });
      snprintf(buf, sizeof buf, "%s\"k%u\": {\"reds_per_s\": %.4g, \"per_address\": %.4g}", first ? "" : ", ", k,
               g / ms * 1e3, g / ms * 1e3 / k);
      js += buf;
      first = 0;
      CK(cudaFree(tab));
    }
    js += "}, \"red_same_stride\": {";
    first = 1;
    for (uint32_t k : {10u, 20u}) {
      for (uint32_t stride : {1u, 4u, 16u, 32u, 128u}) {
        double* tab;
        CK(cudaMalloc(&tab, (size_t)k * stride * 8 + 64));
        CK(cudaMemset(tab, 0, (size_t)k * stride * 8 + 64));
        const int blocks = sms * 4, threads = 256, iters = 64;
        const double g = (double)blocks * threads * iters;
        float ms = best_ms([&] { k_red_same<<<blocks, threads>>>(tab, k, stride, iters); });
        snprintf(buf, sizeof buf, "%s\"k%u_stride%uB\": {\"reds_per_s\": %.4g, \"per_address\": %.4g}",
                 first ? "" : ", ", k, stride * 8, g / ms * 1e3, g / ms * 1e3 / k);
        js += buf;
        first = 0;
        CK(cudaFree(tab));
      }
    }
    js += "}";
  }
  // M4b single-lane load+RED per address (request rate per hot line)
  {
    js += ", \"hot_line\": {";
    int first = 1;
    for (int do_load : {0, 1}) {
      for (uint32_t k : {1u, 10u}) {
        double* tab;
        CK(cudaMalloc(&tab, (size_t)k * 128 * 8));
        CK(cudaMemset(tab, 0, (size_t)k * 128 * 8));
        const int blocks = sms * 8, threads = 256, iters = 32;
        const double g = (double)blocks * (threads / 32) * iters;
        float ms = best_ms([&] { k_ldred_hot<<<blocks, threads>>>(tab, k, 128, iters, do_load); });
        snprintf(buf, sizeof buf, "%s\"%s_k%u\": {\"reds_per_s\": %.4g, \"per_line\": %.4g}", first ? "" : ", ",
                 do_load ? "ld_red" : "red", k, g / ms * 1e3, g / ms * 1e3 / k);
        js += buf;
        first = 0;
        CK(cudaFree(tab));
      }
    }
    js += "}, \"hot_pair\": {";
    first = 1;
    for (uint32_t k : {1u, 10u}) {
      double* tab;
      CK(cudaMalloc(&tab, (size_t)k * 128 * 8));
      CK(cudaMemset(tab, 0, (size_t)k * 128 * 8));
      const int blocks = sms * 8, threads = 256, iters = 32;
      const double g = (double)blocks * (threads / 32) * iters;
      float ms = best_ms([&] { k_pair_hot<<<blocks, threads>>>(tab, k, iters); });
      snprintf(buf, sizeof buf, "%s\"k%u\": {\"updates_per_s_per_pair\": %.4g}", first ? "" : ", ", k,
               g / ms * 1e3 / k);
      js += buf;
      first = 0;
      CK(cudaFree(tab));
    }
    js += "}";
  }
  // M4c TMA bulk 16-byte reductions (x and abar in one op)
  {
    double* tab;
    const uint32_t d = 47236;
    CK(cudaMalloc(&tab, (size_t)d * 128 * 8));
    CK(cudaMemset(tab, 0, (size_t)d * 128 * 8));
    const int blocks = sms * 8, threads = 256, iters = 32;
    float ms_hot = best_ms([&] { k_bulk_pair<<<blocks, threads>>>(tab, 10, d, iters, 1); });
    const double g_hot = (double)blocks * (threads / 32) * iters;
    float ms_rnd = best_ms([&] { k_bulk_pair<<<blocks, threads>>>(tab, 10, d, iters, 0); });
    const double g_rnd = (double)blocks * threads * iters;
    float ms_hot_nl = best_ms([&] { k_bulk_pair<<<blocks, threads>>>(tab, 10, d, iters, 1, 0); });
    snprintf(buf, sizeof buf, ", \"bulk_pair\": {\"hot_k10_updates_per_s_per_pair\": %.4g, \"random_pairs_per_s\": %.4g, "
             "\"hot_k10_bulk_only_per_s_per_pair\": %.4g}",
             g_hot / ms_hot * 1e3 / 10, g_rnd / ms_rnd * 1e3, g_hot / ms_hot_nl * 1e3 / 10);
    js += buf;
    CK(cudaFree(tab));
  }
  // M2b latency of a sample's gathers (one warp per SM)
  {
    const uint32_t d = 47236;
    double2* tab;
    unsigned long long* acc;
    CK(cudaMalloc(&tab, (size_t)d * 16));
    CK(cudaMemset(tab, 0, (size_t)d * 16));
    CK(cudaMalloc(&acc, 16));
    js += ", \"gather_latency_cycles\": {";
    for (int nch = 1; nch <= 4; ++nch) {
      const int rounds = 2000;
      k_gather_lat<<<sms, 32>>>(tab, d, nch, 50, acc);  // warm
      CK(cudaMemset(acc, 0, 8));
      k_gather_lat<<<sms, 32>>>(tab, d, nch, rounds, acc);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      unsigned long long h = 0;
      CK(cudaMemcpy(&h, acc, 8, cudaMemcpyDeviceToHost));
      snprintf(buf, sizeof buf, "%s\"chunks%d\": %.1f", nch == 1 ? "" : ", ", nch, (double)h / sms / rounds);
      js += buf;
    }
    js += "}";
    CK(cudaFree(tab));
    CK(cudaFree(acc));
  }
  // M5 Zipf RED pattern
  {
    js += ", \"red_zipf\": {";
    int first = 1;
    struct Z { uint32_t d; double s; const char* name; };
    for (Z z : {Z{47236u, 1.1, "c3"}, Z{3231961u, 1.0, "c4"}}) {
      std::vector<double> cdf(z.d);
      double acc = 0;
      for (uint32_t k = 0; k < z.d; ++k) { acc += std::pow((double)(k + 1), -z.s); cdf[k] = acc; }
      for (auto& c : cdf) c /= acc;
      std::mt19937_64 rng(160604809);
      std::uniform_real_distribution<double> U(0.0, 1.0);
      std::vector<uint32_t> perm(z.d);
      for (uint32_t k = 0; k < z.d; ++k) perm[k] = k;
      std::shuffle(perm.begin(), perm.end(), rng);
      const uint64_t m = (uint64_t)1 << 26;
      std::vector<uint32_t> list(m);
      for (uint64_t j = 0; j < m; ++j)
        list[j] = perm[std::min<uint32_t>((uint32_t)(std::upper_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin()), z.d - 1)];
      uint32_t* dl;
      double* tab;
      CK(cudaMalloc(&dl, m * 4));
      CK(cudaMemcpy(dl, list.data(), m * 4, cudaMemcpyHostToDevice));
      CK(cudaMalloc(&tab, (size_t)z.d * 32));
      CK(cudaMemset(tab, 0, (size_t)z.d * 32));
      float ms = best_ms([&] { k_red_list<<<sms * 16, 256>>>(tab, dl, m, 4); });
      snprintf(buf, sizeof buf, "%s\"%s\": {\"reds_per_s\": %.4g}", first ? "" : ", ", z.name, (double)m / ms * 1e3);
      js += buf;
      first = 0;
      CK(cudaFree(dl));
      CK(cudaFree(tab));
    }
    js += "}";
  }
  js += "}";
  printf("%s\n", js.c_str());
  return 0;
}
