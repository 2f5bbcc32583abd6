// asaga_kernels.cuh -- sm_100a device code of the ASAGA hot path.
//
// Paper: Leblond, Pedregosa, Lacoste-Julien, "ASAGA: Asynchronous Parallel
// SAGA", arXiv 1606.04809 (PAPER.md; cited "P:<line>").  Kernel map
// (DESIGN.md "Kernels"):
//   ingest_tile_kernel   A0+A1: validate the CSR (read-only), n_v, ||a_i||^2, longest row
//   profile_kernel       A1: D_v = n/n_v, coordinate state {x, abar} init, Delta_r
//   expand_d_kernel      A1: D per stored entry for the plain update kernel's row stream
//   asaga_update_kernel  A2..A8: Philox sample -> row -> gather-dot -> sigma -> SAGA
//                        correction -> red.global.add.f64 scatter (Alg. 2)
//   asaga_combine_kernel A2..A8 with the hot features combined per thread block (R23)
//   margin_*_kernel      A9: m_i = b_i a_i.x, softplus(-m_i), sigma~_i (Section 4.1)
//   colseg_kernel        A9: sum_i sigma~_i a~_iv over fixed column segments (CSC)
// No tensor cores: nothing here is a dense contraction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace asaga {

// Coordinate state:
//   xa[v*S] = {x_v, abar_v}  one 16-byte pair per feature (S = pair stride: 1, or
//           8 / 64 for small d so every feature owns an L2 line / slice and hot
//           features do not share a line's atomic unit): an update gathers both
//           with ONE 128-bit L2 load (LDG.E.NA.128) and adds to both with two REDs
//           into the same sector; abar_v = (1/n) sum_i alpha_i a_iv
//   D[v]    reweighting 1/p_v = n / n_v
//   dv[k]   D_{c_k} replicated per stored entry, so the row stream (cp.async,
//           coalesced) carries D and the gather is a single wavefront per entry
// (profiles/r01_update_kernel.md: per-entry L1TEX wavefronts, not bytes, set the
// per-sample latency at the concurrency ASAGA converges at).

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) -- own implementation (the oracle has its
// own; pin P1 checks both against cuRAND).  Sampling before any read: P:265.
__device__ __forceinline__ uint2 philox_lo64(uint64_t t, uint64_t seed) {
  uint32_t c0 = (uint32_t)t, c1 = (uint32_t)(t >> 32), c2 = 0u, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint2(c0, c1);
}

// Sample-stream checksum (record_samples): sum over processed t of
// mix(t, i_t) mod 2^64 (a splitmix64 finaliser of t * phi + i_t): it holds the t -> i_t map
// itself, not just the per-row visit histogram.  The tests recompute it from the oracle's
// stream (their own copy of this public mixing function: test infrastructure, no method
// arithmetic).
__device__ __forceinline__ unsigned long long sample_mix(uint64_t t, int64_t i) {
  uint64_t z = t * 0x9E3779B97F4A7C15ull + (uint64_t)i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// i_t = floor(r * n / 2^64), r = (w1 << 32) | w0 (reading R2).
__device__ __forceinline__ int64_t sample_row(uint64_t seed, uint64_t t, uint64_t n) {
  const uint2 w = philox_lo64(t, seed);
  const uint64_t r = ((uint64_t)w.y << 32) | (uint64_t)w.x;
  return (int64_t)__umul64hi(r, n);
}

// ---------------------------------------------------------------------------
// Memory-access helpers.  Shared state (Coord, alpha) is read with .cg
// (LDG.STRONG.GPU: L1 bypass), so a read never returns a stale L1 line of a
// coordinate another SM has since added to -- the paper's "inconsistent read"
// is still unsynchronised, but bounded by in-flight updates.
__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// Gathers of shared state: weak loads that never allocate in L1 (LDG.E.NA), so
// they always come from L2 (no stale L1 line) without the ordering cost of a
// .STRONG.GPU load behind the warp's own outstanding REDs (profiles/r01_*.md).
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
#ifdef ASAGA_STRONG_GATHER
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
#else
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ double2 ld_na2(const double2* p) {
  double2 v;
#ifdef ASAGA_STRONG_GATHER
  asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
#else
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
#endif
  return v;
}
// The 32-byte coordinate record {x_v, abar_v, D_v, .} (S >= 2): the {x, abar} pair and D_v
// in ONE sector, gathered by one 256-bit load (LDG.E.NA.ENL2.256 on sm_100; D_v is never
// written after A1) -- D needs no per-entry stream.  ASAGA_REC_TWO_LOADS (measurement
// variant): a 128-bit and a 64-bit load.  (Round 2: on c3 at 384 in flight the record layout
// -- with either load -- sat at a noise floor of f - f* ~ 1e-4 unless the run was perturbed;
// profiles/r02_update_kernel.md sections 7 and 11.)
struct Rec3 {
  double x, ab, D;
};
__device__ __forceinline__ Rec3 ld_na_rec(const double2* p) {
  Rec3 r;
#ifndef ASAGA_REC_TWO_LOADS  // one 256-bit load: one request for the record's sector
  double s;
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.ab), "=d"(r.D), "=d"(s) : "l"(p));
#else  // measurement variant: {x, abar} + D (profiles/r02_update_kernel.md section 7)
  const double2 a = ld_na2(p);
  r.x = a.x;
  r.ab = a.y;
  r.D = ld_na(&p[1].x);
#endif
  return r;
}

// Hot-split membership table (record layout with hot_split_min_freq): the features with
// 0 < D_v <= hot_dmax, open addressing with linear probing in 2^log slots (-1 = free),
// filled to at most 1/8 by construction (asaga.cu: slots >= 8 x the bound
// nnz/n x hot_dmax on their number).  Membership is exact whatever the insertion order.
__device__ __forceinline__ unsigned hot_hash(int v, int log) {
  return ((unsigned)v * 0x9E3779B1u) >> (32 - log);
}
__device__ __forceinline__ void hot_insert(int32_t* tab, int log, int v) {
  const unsigned mask = (1u << log) - 1u;
  for (unsigned h = hot_hash(v, log);; h = (h + 1u) & mask) {
    const int prev = atomicCAS(tab + h, -1, v);
    if (prev == -1 || prev == v) return;
  }
}
__device__ __forceinline__ bool hot_lookup(const int32_t* tab, int log, int c) {
  const unsigned mask = (1u << log) - 1u;
  unsigned h = hot_hash(c, log);
  int e = tab[h];
  while (e != c && e != -1) {
    h = (h + 1u) & mask;
    e = tab[h];
  }
  return e == c;
}
// A1: coordinate v's state init (x = abar = 0), D_v, its record copy (S >= 2) and its
// hot-table entry
__device__ __forceinline__ void init_coord(int64_t v, int cnt, int64_t n, double2* __restrict__ xa, int S,
                                           double* __restrict__ habar, double* __restrict__ D,
                                           int32_t* __restrict__ hot_tab, int hot_log, double hot_dmax) {
  const double Dv = cnt > 0 ? (double)n / (double)cnt : 0.0;
  xa[v * S] = make_double2(0.0, 0.0);
  if (S >= 2) xa[v * S + 1] = make_double2(Dv, 0.0);
  habar[v] = 0.0;
  D[v] = Dv;
  if (hot_tab != nullptr && Dv > 0.0 && Dv <= hot_dmax) hot_insert(hot_tab, hot_log, (int)v);
}

__device__ __forceinline__ void st_cg(double* p, double v) {
  asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// Atomic coordinate add (Property 3): fire-and-forget reduction at L2.
__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
// The same add under a predicate, as ONE predicated instruction (no branch around it), so
// that lanes taking different roles in the paired scatter still issue it together.
__device__ __forceinline__ void red_add_if(double* p, double v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.relaxed.gpu.global.add.f64 [%0], %1;\n\t}"
               ::"l"(p), "d"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void red_add_u32(int32_t* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// cp.async (LDGSTS) helpers: rows are copied global -> shared while earlier ones are
// processed (update kernels: the next sample's row; ingest: the next row batches).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
// Streaming copies (row data read once per sample) marked L2 evict-first, so they do not
// push the shared state ({x, abar} pairs: 52 MB on c4) out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async4_ef(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async8_ef(void* smem, const void* gmem, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ int ld_nc_i32(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ double ld_nc_f64(const double* p) { return __ldg(p); }

// A5 (Alg. 2 lines 6-8; folded logistic P:483-485): sigma~(m) = -1 / (1 + exp(m)) in
// fp64, ~28 instructions: t = exp(-|m|) by Cody-Waite reduction (k = rint(-|m| / ln 2),
// r = -|m| - k ln 2 with ln 2 in two parts, |r| <= ln2/2), the degree-12 Taylor polynomial
// (truncation < 1.6e-16 relative; coefficients 1/j! from constant memory, so the DFMAs take
// them as operands instead of materialising 64-bit immediates), 2^k added to the exponent
// field; then 1/(1+t) (1+t in (1, 2]) from the MUFU reciprocal seed and two Newton steps;
// sigma~ = -t/(1+t) for m >= 0, -1/(1+t) for m < 0.  |m| is clamped at 700 (exp(-700) ~ 1e-304:
// t stays normal; the lost tail is below 1e-304 absolute).  The library exp + __drcp_rn took
// 61 warp instructions per sample pair in the combine kernel (ncu, profiles/r01_combine_kernel.md).
__constant__ double c_inv_fact[13] = {
    1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0, 1.0 / 40320.0,
    1.0 / 5040.0,      1.0 / 720.0,      1.0 / 120.0,     1.0 / 24.0,     1.0 / 6.0,
    0.5,               1.0,              1.0};
__device__ __forceinline__ double sigma_folded(double m) {
  const double x = fmax(-fabs(m), -700.0);
  const double kd = fma(x, 1.4426950408889634, 6755399441055744.0);  // 1.5 * 2^52: rint in the low word
  const double kf = kd - 6755399441055744.0;
  double r = fma(kf, -6.93147180559945286227e-01, x);  // ln 2, high part
  r = fma(kf, -2.31904681384629955842e-17, r);          // ln 2, low part
  double p = c_inv_fact[0];
#pragma unroll
  for (int j = 1; j < 13; ++j) p = fma(p, r, c_inv_fact[j]);
  const int ki = __double2loint(kd);
  const double t = __hiloint2double(__double2hiint(p) + (ki << 20), __double2loint(p));
  const double dd = 1.0 + t;
  double rc;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(dd));
  double e = fma(-dd, rc, 1.0);
  e = fma(e, e, e);
  rc = fma(rc, e, rc);
  e = fma(-dd, rc, 1.0);
  rc = fma(rc, e, rc);
  // a NaN margin stays NaN (fmax above would drop it), so divergence reaches alpha and abar too
  return m != m ? m : (m >= 0.0 ? -t * rc : -rc);
}

// Test hook (asaga_debug_sigma): sigma_folded over a device array.
__global__ void sigma_kernel(const double* __restrict__ m, double* __restrict__ out, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = sigma_folded(m[k]);
}

template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off);
  return v;
}

// ---------------------------------------------------------------------------
// A0 + A1: validation, label folding, column counts, squared row norms.
enum : int { ERR_ENDS = 0, ERR_ROW_BOUNDS, ERR_EMPTY_ROW, ERR_INDEX_RANGE, ERR_INDEX_ORDER,
             ERR_NONFINITE, ERR_LABEL, ERR_COUNT };

struct IngestParams {
  // the matrix is read, never written: the context keeps these arrays (the caller's
  // device arrays, or its own after a host copy) and applies b_i per sample / row
  const int64_t* indptr;  // n+1
  const int32_t* indices; // nnz
  const double* data;     // nnz
  const double* y;        // n
  int32_t* counts;        // out (pre-zeroed): n_v
  unsigned long long* err_row;   // [ERR_COUNT], pre-set to ULLONG_MAX; atomicMin(row)
  unsigned long long* max_sq;    // bits of max_i ||a_i||^2 (>= 0 doubles order as u64)
  unsigned long long* max_len;   // longest row
  int64_t n, d, nnz;
  size_t stage_off;       // ingest_tile_kernel<true>: byte offset of the warp stages in smem
  // fused A1 finish (d <= 4096): the last block to finish runs profile_small + the report
  int fuse;
  double2* xa;
  int S;
  double* habar;
  double* D;
  double comb_dmax;
  int max_h;
  int32_t* slot_of;
  int32_t* hot_id;
  int* flag;              // [1] max n_v, [2] hot count, [3] run guard, [4] finished blocks
  unsigned long long* host_out;
  int64_t row_cap;
  int hot_expected;
  int guard;
  int smem_hist;          // 1: per-block shared histogram of all d columns; 0: a per-block
                          // shared hash cache of 2^hash_log columns (the popular ones claim it)
  int hash_log;           // !smem_hist: log2 of the hash cache's slots (kHashLog, or larger)
  // self_init (fused, d <= kSelfInitMaxD): no ingest_init launch -- every block stores its
  // histogram into part[block][d] (no atomics, no zeroed counts), zeroes alpha for its rows,
  // and the last block sums the parts into counts, then (after the report) resets the error
  // rows, the maxima and its ticket for the next ingest (set once at allocation)
  int self_init;
  int32_t* part;
  double* alpha;
  int32_t* hot_tab;       // record layout's hot-split table (pre-set to -1), or NULL
  int hot_log;
  double hot_dmax;
};

// ---------------------------------------------------------------------------
// Row tiles (A0+A1 ingest, A9 margins).  A warp owns 32 consecutive rows and streams
// their entries [rowptr[r0], rowptr[r0+32]) flat, 32 per chunk (coalesced loads, many
// chunks in flight), instead of one row per lane group (three dependent round trips
// per row: the per-row kernels were latency-bound at 0.8-1 TB/s).  Lane j holds the
// tile-relative start of row r0+j; an entry finds its row by a 5-step binary search
// over the lanes, and per-row sums use a segmented warp reduction whose segment heads
// add into the warp's shared row accumulators (fixed order: deterministic).
__device__ __forceinline__ int tile_row_of(int off, int rel, int nr) {
  int j = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int cand = j + step;
    const int rc = __shfl_sync(0xffffffffu, rel, cand & 31);
    if (cand < nr && rc <= off) j = cand;
  }
  return j;
}
// Segmented sum over lanes with equal keys (keys non-decreasing across lanes): the
// first lane of each segment receives the segment's total.
__device__ __forceinline__ double seg_sum_head(double v, int key, bool* head) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, v, d);
    const int ok = __shfl_down_sync(0xffffffffu, key, d);
    if (lane + d < 32 && ok == key) v += ov;
  }
  const int pk = __shfl_up_sync(0xffffffffu, key, 1);
  *head = lane == 0 || pk != key;
  return v;
}

constexpr int kHashLog = 12, kHashSlots = 1 << kHashLog;  // ingest hash cache (32 KiB)

// (defined below; the ingest's last block runs them when the A1 finish is fused)
__device__ __forceinline__ void profile_small_body(const int32_t* __restrict__ counts, double2* __restrict__ xa, int S,
                     double* __restrict__ habar, double* __restrict__ D, int d, int64_t n,
                     int* __restrict__ max_count, double comb_dmax, int max_h,
                     int32_t* __restrict__ slot_of, int32_t* __restrict__ hot_id,
                     int* __restrict__ n_hot, int32_t* __restrict__ hot_tab,
                     int hot_log, double hot_dmax);
__device__ __forceinline__ void report_body(const unsigned long long* __restrict__ scratch,
                                            int* __restrict__ flag, unsigned long long* host_out,
                                            int64_t row_cap, int hot_expected, int guard);

// A0 + A1 over row tiles, reading the matrix only: validate, count n_v (shared histogram
// when d fits), max ||a_i||^2, longest row.
// STAGED (short rows): a tile whose entries fit kStageCap is copied into the warp's
// shared stage by cp.async, each row is then checked / counted by its OWNER lane from
// shared memory (the previous index and ||a_i||^2 in registers: a few instructions per
// entry instead of the flat path's per-chunk row search and segmented reduction).
// Larger tiles take the flat path.
// ROWS (long rows, mean >= 32 entries, n_v through the hash cache): the warp walks the
// tile row by row, 32 entries of one row per chunk: the row, label and previous column
// are warp-uniform, so the flat path's per-chunk row search and segmented reduction (186
// warp instructions per chunk on c4, ncu) become one warp sum per row (117 per chunk).
enum : int { kIngestFlat = 0, kIngestStaged = 1, kIngestRows = 2 };
constexpr int kStageCap = 512;  // entries per warp stage (int32 index + fp64 value: 6 KiB)
#ifdef ASAGA_INGEST_ROWS_BLOCKING  // measurement variant: the blocking rows loop
constexpr bool kIngestRowsPipe = false;
#else
constexpr bool kIngestRowsPipe = true;
#endif
constexpr int kIngestPF = 512;  // rows-mode L2 prefetch distance (entries)

template <int MODE>
__global__ void __launch_bounds__(1024) ingest_tile_kernel(IngestParams p) {
  constexpr bool STAGED = MODE == kIngestStaged;
  extern __shared__ __align__(16) int32_t hist[];
  __shared__ double rsq[32][32];
  __shared__ double blk_max[32];
  __shared__ long long blk_len[32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* hkey = hist;                  // !smem_hist: hash cache keys (-1 = free) ...
  const int hslots = 1 << p.hash_log;
  int32_t* hcnt = hist + hslots;         // ... and counts
  // STAGED: per-warp stages after the histogram (p.stage_off bytes into dynamic smem)
  double* stage_v = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(hist) + p.stage_off) +
                    (size_t)wib * kStageCap;
  int32_t* stage_c = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(hist) + p.stage_off +
                                                (size_t)(blockDim.x >> 5) * kStageCap * sizeof(double)) +
                     (size_t)wib * kStageCap;
  auto count_col = [&](int c) {
    if (p.smem_hist) {
      atomicAdd(&hist[c], 1);
    } else {
      // n_v: a Zipf-popular column would take ~1e6 serialised global atomics (c4: 4.8 ms
      // of the ingest); the first column to hash into a free slot keeps it per block
      const int slot = (int)(((unsigned)c * 2654435761u) >> (32 - p.hash_log));
      int k = hkey[slot];
      if (k == -1) {
        const int prev = atomicCAS(&hkey[slot], -1, c);
        k = prev == -1 ? c : prev;
      }
      if (k == c) atomicAdd(&hcnt[slot], 1);
      else red_add_u32(p.counts + c, 1u);  // REDG: no response traffic (ATOMG returns a sector)
    }
  };
  if (p.smem_hist) {
    for (int64_t v = threadIdx.x; v < p.d; v += blockDim.x) hist[v] = 0;
  } else {
    for (int k = threadIdx.x; k < hslots; k += blockDim.x) {
      hkey[k] = -1;
      hcnt[k] = 0;
    }
  }
  __syncthreads();
  double my_max = 0.0;
  long long my_len = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && (p.indptr[0] != 0 || p.indptr[p.n] != p.nnz))
    atomicMin(&p.err_row[ERR_ENDS], 0ull);  // indptr[0] = 0 and indptr[n] = nnz
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; tile * 32 < p.n; tile += nwarps) {
    const int64_t r0 = tile * 32;
    const int nr = (int)((p.n - r0) < 32 ? (p.n - r0) : 32);
    const int64_t i = r0 + lane;
    const bool row = lane < nr;
    const int64_t lo = row ? p.indptr[i] : 0;
    const int64_t hi = row ? p.indptr[i + 1] : 0;
    const double b = row ? p.y[i] : 1.0;
    if (row && b != 1.0 && b != -1.0) atomicMin(&p.err_row[ERR_LABEL], (unsigned long long)i);
    if (p.self_init && row) p.alpha[i] = 0.0;
    // bounds: every row inside [0, nnz], monotone, contiguous with the next row
    const int64_t next_lo = __shfl_down_sync(0xffffffffu, lo, 1);
    const bool bad_b = row && (lo < 0 || hi > p.nnz || hi < lo || (lane + 1 < nr && next_lo != hi));
    if (bad_b) atomicMin(&p.err_row[ERR_ROW_BOUNDS], (unsigned long long)i);
    if (__any_sync(0xffffffffu, bad_b)) continue;  // the tile cannot be streamed
    if (row && hi == lo) atomicMin(&p.err_row[ERR_EMPTY_ROW], (unsigned long long)i);
    if (row) my_len = max(my_len, (long long)(hi - lo));
    const int64_t base = __shfl_sync(0xffffffffu, lo, 0);
    const int64_t end = __shfl_sync(0xffffffffu, hi, nr - 1);
    const int rel = (int)((row ? lo : end) - base);
    if (STAGED && end - base <= kStageCap) {
      const int cnt = (int)(end - base);
      {
        const int32_t* gi = p.indices + base;
        const double* gv = p.data + base;
        for (int e = lane; e < cnt; e += 32) {  // every copy in flight at once (cp.async)
          cp_async4(stage_c + e, gi + e);
          cp_async8(stage_v + e, gv + e);
        }
      }
      cp_async_commit();
      cp_async_wait_all();
      __syncwarp();
      if (row) {
        // one "defect" flag per row in the hot loop (range or order; a non-finite value
        // shows in sq), classified by a rescan only when set
        const unsigned ud = (unsigned)(p.d < (int64_t)INT32_MAX + 1 ? p.d : (int64_t)INT32_MAX + 1);
        int prevc = -1;
        double sq = 0.0;
        bool bad = false;
        const int kend = rel + (int)(hi - lo);
        for (int k = rel; k < kend; ++k) {
          const int32_t c = stage_c[k];
          const double v = stage_v[k];
          const bool br = (unsigned)c >= ud;
          bad |= br | (prevc >= c);
          prevc = c;
          sq = fma(v, v, sq);
          if (!br) count_col(c);
        }
        if (bad || !isfinite(sq)) {
          bool br_any = false, bo_any = false, bv_any = false;
          prevc = -1;
          for (int k = rel; k < kend; ++k) {
            const int32_t c = stage_c[k];
            const double v = stage_v[k];
            br_any |= (c < 0) || ((int64_t)c >= p.d);
            bo_any |= prevc >= c;
            bv_any |= !isfinite(v);
            prevc = c;
          }
          if (br_any) atomicMin(&p.err_row[ERR_INDEX_RANGE], (unsigned long long)i);
          if (bo_any) atomicMin(&p.err_row[ERR_INDEX_ORDER], (unsigned long long)i);
          if (bv_any) atomicMin(&p.err_row[ERR_NONFINITE], (unsigned long long)i);
        }
        my_max = fmax(my_max, sq);
      }
      __syncwarp();  // the stage is refilled by the next tile
      continue;
    }
    if (MODE == kIngestRows && kIngestRowsPipe) {
      // software pipeline over the tile's row groups of kRQ x 32 entries: the next group (the
      // rest of this row, or the start of the next one) is loaded into the second register
      // set before the current group is checked and counted, so the loads of one group are in
      // flight while the previous one is processed (the blocking version loaded 4 chunks,
      // waited, processed: latency-bound, long-scoreboard stalls at one block per SM)
      constexpr int kRQ = 2;
      int32_t cA[kRQ], cB[kRQ];
      double vA[kRQ], vB[kRQ];
      auto load_group = [&](int64_t e00, int64_t rhi, int32_t (&cq)[kRQ], double (&vq)[kRQ]) {
#pragma unroll
        for (int qq = 0; qq < kRQ; ++qq) {
          const int64_t e = e00 + 32 * qq + lane;
          cq[qq] = e < rhi ? __ldcs(p.indices + e) : INT32_MAX;
          vq[qq] = e < rhi ? __ldcs(p.data + e) : 0.0;
        }
      };
      int jc = 0;
      int64_t rlo = __shfl_sync(0xffffffffu, lo, 0);
      int64_t ec = rlo, hc = __shfl_sync(0xffffffffu, hi, 0);
      load_group(ec, hc, cA, vA);
      int carry = -1;
      double sq = 0.0;
      bool br_any = false, bo_any = false, bv_any = false;
      // one step: load the next group into (cn, vn), process (cc, vc); false after the last
      // row.  Called alternately with the two register sets swapped (no register copies:
      // a copy of a load's destination waits for the load -- 47 % of the stall samples)
      auto step = [&](const int32_t (&cc)[kRQ], const double (&vc)[kRQ], int32_t (&cn)[kRQ],
                      double (&vn)[kRQ]) -> bool {
        int jn = jc;
        int64_t en = ec + 32 * kRQ, hn = hc;
        const bool row_end = en >= hc;  // warp-uniform
        if (row_end) {
          jn = jc + 1;
          if (jn < nr) {
            en = __shfl_sync(0xffffffffu, lo, jn);
            hn = __shfl_sync(0xffffffffu, hi, jn);
          }
        }
        if (jn < nr) load_group(en, hn, cn, vn);
#ifndef ASAGA_INGEST_NO_PF
        {  // L2 prefetch of the warp's entries kIngestPF ahead in the tile (rows are
           // contiguous): the register loads one group ahead then come from L2
          const int64_t pf = ec + kIngestPF;
          if (lane < 8 && pf < end) {
            const char* a = lane < 3 ? reinterpret_cast<const char*>(p.indices + pf) + lane * 128
                                     : reinterpret_cast<const char*>(p.data + pf) + (lane - 3) * 128;
            prefetch_l2(a);
          }
        }
#endif
#pragma unroll
        for (int qq = 0; qq < kRQ; ++qq) {
          const int64_t e0 = ec + 32 * qq;
          if (e0 >= hc) break;  // warp-uniform
          const int64_t e = e0 + lane;
          const int32_t c = cc[qq];
          const double v = vc[qq];
          int prev = __shfl_up_sync(0xffffffffu, c, 1);
          if (lane == 0) prev = carry;
          carry = __shfl_sync(0xffffffffu, c, 31);
          if (e < hc) {
            const bool br = (c < 0) || ((int64_t)c >= p.d);
            br_any |= br;
            bo_any |= e > rlo && prev >= c;
            bv_any |= !isfinite(v);
            sq = fma(v, v, sq);
            if (!br) count_col(c);
          }
        }
        if (row_end) {
          sq = group_sum<32>(sq, 0xffffffffu);
          const bool bad = __any_sync(0xffffffffu, br_any), bado = __any_sync(0xffffffffu, bo_any),
                     badv = __any_sync(0xffffffffu, bv_any);
          if (lane == jc) {
            my_max = fmax(my_max, sq);
            if (bad) atomicMin(&p.err_row[ERR_INDEX_RANGE], (unsigned long long)i);
            if (bado) atomicMin(&p.err_row[ERR_INDEX_ORDER], (unsigned long long)i);
            if (badv) atomicMin(&p.err_row[ERR_NONFINITE], (unsigned long long)i);
          }
          if (jn >= nr) return false;
          carry = -1;
          sq = 0.0;
          br_any = bo_any = bv_any = false;
          rlo = en;
        }
        jc = jn;
        ec = en;
        hc = hn;
        return true;
      };
      while (step(cA, vA, cB, vB) && step(cB, vB, cA, vA)) {
      }
      continue;
    }
    if (MODE == kIngestRows) {
      for (int j = 0; j < nr; ++j) {
        const int64_t rlo = __shfl_sync(0xffffffffu, lo, j);
        const int64_t rhi = __shfl_sync(0xffffffffu, hi, j);
        int carry = -1;
        double sq = 0.0;
        bool br_any = false, bo_any = false, bv_any = false;
        // 4 chunks (128 entries) are loaded before any is processed: loads in flight
        // (a cp.async ring of 128-entry units, two ahead, measured slower on c4, 2.92 vs
        // 2.81 ms: the kernel is LSU/MIO-bound, l1tex 69 %, and the ring adds a shared load)
        for (int64_t e00 = rlo; e00 < rhi; e00 += 128) {
          int32_t cq[4];
          double vq[4];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int64_t e = e00 + 32 * qq + lane;
            cq[qq] = e < rhi ? p.indices[e] : INT32_MAX;
            vq[qq] = e < rhi ? p.data[e] : 0.0;
          }
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int64_t e0 = e00 + 32 * qq;
            if (e0 >= rhi) break;  // warp-uniform
            const int64_t e = e0 + lane;
            const int32_t c = cq[qq];
            const double v = vq[qq];
            int prev = __shfl_up_sync(0xffffffffu, c, 1);
            if (lane == 0) prev = carry;
            carry = __shfl_sync(0xffffffffu, c, 31);
            if (e < rhi) {
              const bool br = (c < 0) || ((int64_t)c >= p.d);
              br_any |= br;
              bo_any |= e > rlo && prev >= c;
              bv_any |= !isfinite(v);
              sq = fma(v, v, sq);
              if (!br) count_col(c);
            }
          }
        }
        sq = group_sum<32>(sq, 0xffffffffu);
        const bool bad = __any_sync(0xffffffffu, br_any), bado = __any_sync(0xffffffffu, bo_any),
                   badv = __any_sync(0xffffffffu, bv_any);
        if (lane == j) {
          my_max = fmax(my_max, sq);
          if (bad) atomicMin(&p.err_row[ERR_INDEX_RANGE], (unsigned long long)i);
          if (bado) atomicMin(&p.err_row[ERR_INDEX_ORDER], (unsigned long long)i);
          if (badv) atomicMin(&p.err_row[ERR_NONFINITE], (unsigned long long)i);
        }
      }
      continue;
    }
    rsq[wib][lane] = 0.0;
    __syncwarp();
    int carry = -1;
    bool bad_range = false, bad_order = false, bad_val = false;
    int first_bad_range = INT32_MAX, first_bad_order = INT32_MAX, first_bad_val = INT32_MAX;
    // 4 chunks (128 entries) are loaded before any is processed: loads in flight
    for (int64_t e00 = base; e00 < end; e00 += 128) {
    int32_t cq[4];
    double vq[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int64_t e = e00 + 32 * qq + lane;
      cq[qq] = e < end ? p.indices[e] : INT32_MAX;
      vq[qq] = e < end ? p.data[e] : 0.0;
    }
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int64_t e0 = e00 + 32 * qq;
      if (e0 >= end) break;  // warp-uniform
      const int64_t e = e0 + lane;
      const bool in = e < end;
      const int32_t c = cq[qq];
      const double v = vq[qq];
      const int off = (int)(e - base);
      const int j = tile_row_of(off, rel, nr);
      const int rs = __shfl_sync(0xffffffffu, rel, j);
      int prev = __shfl_up_sync(0xffffffffu, c, 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(0xffffffffu, c, 31);
      if (in) {
        const bool br = (c < 0) || ((int64_t)c >= p.d);
        const bool bo = off > rs && prev >= c;
        const bool bv = !isfinite(v);
        if (br) first_bad_range = min(first_bad_range, j);
        if (bo) first_bad_order = min(first_bad_order, j);
        if (bv) first_bad_val = min(first_bad_val, j);
        bad_range |= br; bad_order |= bo; bad_val |= bv;
        if (!br) count_col(c);
      }
      bool head;
      const double sq = seg_sum_head(in ? v * v : 0.0, in ? j : 32 + lane, &head);
      if (in && head) rsq[wib][j] += sq;
    }
    }
    if (bad_range) atomicMin(&p.err_row[ERR_INDEX_RANGE], (unsigned long long)(r0 + first_bad_range));
    if (bad_order) atomicMin(&p.err_row[ERR_INDEX_ORDER], (unsigned long long)(r0 + first_bad_order));
    if (bad_val) atomicMin(&p.err_row[ERR_NONFINITE], (unsigned long long)(r0 + first_bad_val));
    __syncwarp();
    if (row) my_max = fmax(my_max, rsq[wib][lane]);
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) {
    my_max = fmax(my_max, __shfl_xor_sync(0xffffffffu, my_max, off));
    my_len = max(my_len, __shfl_xor_sync(0xffffffffu, my_len, off));
  }
  if (lane == 0) {
    blk_max[wib] = my_max;
    blk_len[wib] = my_len;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    long long L = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      m = fmax(m, blk_max[w]);
      L = max(L, blk_len[w]);
    }
    atomicMax(p.max_sq, (unsigned long long)__double_as_longlong(m));
    atomicMax(p.max_len, (unsigned long long)L);
  }
  __syncthreads();
  if (p.self_init) {
    for (int64_t v = threadIdx.x; v < p.d; v += blockDim.x) p.part[(int64_t)blockIdx.x * p.d + v] = hist[v];
  } else if (p.smem_hist) {
    for (int64_t v = threadIdx.x; v < p.d; v += blockDim.x)
      if (hist[v]) atomicAdd(&p.counts[v], hist[v]);
  } else {
    for (int k = threadIdx.x; k < hslots; k += blockDim.x)
      if (hkey[k] >= 0 && hcnt[k]) atomicAdd(&p.counts[hkey[k]], hcnt[k]);
  }
  if (p.fuse) {  // the last block to finish runs A1's finish and the report (d <= 4096)
    __shared__ int is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(&p.flag[4], 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (is_last) {
      __threadfence();
      if (p.self_init) {  // n_v = the sum of the blocks' parts, in block order
        for (int64_t v = threadIdx.x; v < p.d; v += blockDim.x) {
          int c = 0;
          for (int bk = 0; bk < (int)gridDim.x; ++bk) c += __ldcg(p.part + (int64_t)bk * p.d + v);
          p.counts[v] = c;
        }
        __syncthreads();
      }
      profile_small_body(p.counts, p.xa, p.S, p.habar, p.D, (int)p.d, p.n, p.flag + 1, p.comb_dmax, p.max_h,
                         p.slot_of, p.hot_id, p.flag + 2, p.hot_tab, p.hot_log, p.hot_dmax);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        report_body(p.err_row, p.flag, p.host_out, p.row_cap, p.hot_expected, p.guard);
        if (p.self_init) {  // ready for the next ingest
          for (int q = 0; q < ERR_COUNT; ++q) p.err_row[q] = ~0ull;
          p.err_row[ERR_COUNT] = 0ull;
          p.err_row[ERR_COUNT + 1] = 0ull;
          p.flag[4] = 0;
        }
      }
    }
  }
}

// A1 finish: D_v = n / n_v (IEEE division, reading R4), state init, Delta_r.
__global__ void profile_kernel(const int32_t* __restrict__ counts, double2* __restrict__ xa,
                               int S, double* __restrict__ habar, double* __restrict__ D, int64_t d,
                               int64_t n, int* __restrict__ max_count, int32_t* __restrict__ hot_tab,
                               int hot_log, double hot_dmax) {
  int my = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int c = counts[v];
    init_coord(v, c, n, xa, S, habar, D, hot_tab, hot_log, hot_dmax);
    my = max(my, c);
  }
  for (int off = 16; off > 0; off >>= 1) my = max(my, __shfl_xor_sync(0xffffffffu, my, off));
  if ((threadIdx.x & 31) == 0) atomicMax(max_count, my);
}

// A1: dv[k] = D[cols[k]] (the row stream carries D; see the layout note above).
// Hot split (hot_dmax > 0): an entry of a popular feature (D_c <= hot_dmax, i.e.
// p_c >= 1/hot_dmax) carries -D_c: its abar lives in the separate `habar` array, so
// x_c and abar_c sit on different L2 lines (2 operations per line per update, not 3).
// Combining (asaga_combine_kernel): eslot[k] = slot of the entry's feature (-1 cold),
// written only when some but not all features are hot (*n_hot < d).
__global__ void expand_d_kernel(const int32_t* __restrict__ cols, const double* __restrict__ D,
                                int64_t nnz, double hot_dmax, double* __restrict__ dv,
                                const int32_t* __restrict__ slot_of, const int* __restrict__ n_hot,
                                int64_t d, int32_t* __restrict__ eslot) {
  const bool want_slot = eslot != nullptr && *n_hot > 0 && (int64_t)*n_hot < d;
  // 4 consecutive entries per thread per step, every load of a step issued before any use
  // (one column load -> D gather -> store chain per entry was latency-bound: c4 1.07 ms)
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; k0 < nnz; k0 += stride) {
    int c[U];  // entries k0 + u * blockDim.x: every load instruction of the warp coalesced
    double Dc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * blockDim.x;
      c[u] = k < nnz ? __ldcs(cols + k) : 0;
      // an asynchronous reload expands before its validation is read back: an index out of
      // [0, d) must not be dereferenced (the data is rejected; dv is never used then)
      if ((unsigned long long)(unsigned)c[u] >= (unsigned long long)d) c[u] = 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) Dc[u] = __ldg(D + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + (int64_t)u * blockDim.x;
      if (k < nnz) {
        __stcs(dv + k, (hot_dmax > 0.0 && Dc[u] <= hot_dmax) ? -Dc[u] : Dc[u]);
        if (want_slot) eslot[k] = __ldg(slot_of + c[u]);
      }
    }
  }
}

__global__ void set_flag_kernel(int* flag, int v) { *flag = v; }

// A0's state reset in one launch (instead of five memsets): n_v = 0, alpha = 0, the error
// rows = "none", max ||a||^2 = max row = 0, the small flags = 0.
__global__ void ingest_init_kernel(int32_t* __restrict__ counts, int64_t d, double* __restrict__ alpha,
                                   int64_t n, unsigned long long* __restrict__ scratch,
                                   int* __restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t v = t0; v < d; v += stride) counts[v] = 0;
  for (int64_t i = t0; i < n; i += stride) alpha[i] = 0.0;
  if (t0 < ERR_COUNT) scratch[t0] = ~0ull;
  if (t0 < 2) scratch[ERR_COUNT + t0] = 0ull;
  if (t0 < 8) flag[t0] = 0;  // [4]: the ingest's finished-block count
}

// The ingest's report, written straight into mapped pinned host memory (no copies):
// error rows, max ||a||^2, longest row, max n_v, hot count; and the run guard for an
// asynchronous reload (valid data that fits the launch shape), when guard != 0.
__device__ __forceinline__ void report_body(const unsigned long long* __restrict__ scratch,
                                            int* __restrict__ flag, unsigned long long* host_out,
                                            int64_t row_cap, int hot_expected, int guard) {
  bool good = true;
  for (int e = 0; e < ERR_COUNT + 2; ++e) {
    host_out[e] = scratch[e];
    if (e < ERR_COUNT) good = good && scratch[e] == ~0ull;
  }
  host_out[ERR_COUNT + 2] = (unsigned long long)(unsigned)flag[1] | ((unsigned long long)(unsigned)flag[2] << 32);
  good = good && (int64_t)scratch[ERR_COUNT + 1] <= row_cap;
  if (hot_expected >= 0) good = good && flag[2] == hot_expected;
  if (guard) flag[3] = good ? 1 : 0;
}
__global__ void ingest_report_kernel(const unsigned long long* __restrict__ scratch,
                                     int* __restrict__ flag, unsigned long long* host_out,
                                     int64_t row_cap, int hot_expected, int guard) {
  report_body(scratch, flag, host_out, row_cap, hot_expected, guard);
}

// Small d (<= 1024 * 4): A1's finish and the combine hot set by ONE block (the ingest's
// last) -- D_v, state init, Delta_r, hot flags, their exclusive scan (slots in feature
// order, as the CUB path gives) and the slot tables -- instead of five launches.
__device__ __forceinline__ void profile_small_body(const int32_t* __restrict__ counts, double2* __restrict__ xa, int S,
                     double* __restrict__ habar, double* __restrict__ D, int d, int64_t n,
                     int* __restrict__ max_count, double comb_dmax, int max_h,
                     int32_t* __restrict__ slot_of, int32_t* __restrict__ hot_id,
                     int* __restrict__ n_hot, int32_t* __restrict__ hot_tab,
                     int hot_log, double hot_dmax) {
  __shared__ int warp_tot[32];
  __shared__ int warp_max[32];
  constexpr int PER = 4;  // features per thread (d <= 4096)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int flag[PER], mine = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int v = threadIdx.x * PER + q;
    flag[q] = 0;
    if (v < d) {
      const int c = counts[v];
      const double Dv = c > 0 ? (double)n / (double)c : 0.0;
      init_coord(v, c, n, xa, S, habar, D, hot_tab, hot_log, hot_dmax);
      mx = max(mx, c);
      flag[q] = (comb_dmax > 0.0 && Dv > 0.0 && Dv <= comb_dmax) ? 1 : 0;
      mine += flag[q];
    }
  }
  // block exclusive scan of the per-thread hot counts (features in thread order = id order)
  int incl = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 31) warp_tot[wib] = incl;
  if (lane == 0) warp_max[wib] = mx;
  __syncthreads();
  if (wib == 0) {
    const int nw = (int)(blockDim.x >> 5);
    int t = lane < nw ? warp_tot[lane] : 0;
    int m = lane < nw ? warp_max[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t += o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane < nw) warp_tot[lane] = t;  // inclusive over warps
    if (lane == 0) *max_count = m;
    if (lane == 31) *n_hot = t;  // inclusive total (nw <= 32)
  }
  __syncthreads();
  int slot = (wib > 0 ? warp_tot[wib - 1] : 0) + incl - mine;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int v = threadIdx.x * PER + q;
    if (v < d && slot_of != nullptr) {  // NULL when combining is off
      const bool hot = flag[q] != 0 && slot < max_h;
      slot_of[v] = hot ? slot : -1;
      if (hot) hot_id[slot] = v;
      slot += flag[q];
    }
  }
}

// Combining: hot features are those with 0 < D_v <= comb_dmax (p_v >= combine_min_freq).
__global__ void hot_flag_kernel(const double* __restrict__ D, int64_t d, double comb_dmax,
                                int32_t* __restrict__ flag) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x)
    flag[v] = (D[v] > 0.0 && D[v] <= comb_dmax) ? 1 : 0;
}

// slot of a hot feature = number of hot features before it (exclusive scan `excl`);
// slot_of[v] = -1 for cold ones and for slots beyond max_h; n_hot = the total.
__global__ void hot_slot_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ excl,
                                int64_t d, int max_h, int32_t* __restrict__ slot_of,
                                int32_t* __restrict__ hot_id, int* __restrict__ n_hot) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int s = excl[v];
    const bool hot = flag[v] != 0;
    slot_of[v] = (hot && s < max_h) ? s : -1;
    if (hot && s < max_h) hot_id[s] = (int32_t)v;
    if (v == d - 1) *n_hot = s + (hot ? 1 : 0);
  }
}

// ---------------------------------------------------------------------------
// A2..A8: the ASAGA update loop (Algorithm 2, + Section 4.2 l2 term).
//
// Worker w (a group of G lanes) processes t = t0 + w, t0 + w + W, ... (W workers
// = samples in flight).  Per sample, in the folded form a~ = b a (the label b_i comes
// with the row and multiplies the margin and dalpha: exact, b = +-1) and folded memory
// alpha~_i = b_i alpha_i:
//   i      = Philox(seed, t)                               line 3 (sample first)
//   x^, abar^ on S_i (.cg loads), D (L1)                   lines 5, 7
//   m      = sum a~_k x^_{c_k}   (group shuffle reduce)
//   dalpha = -1/(1+exp(m)) - alpha~^_i                     lines 6, 8
//   x_v   += -gamma (dalpha a~_k + D_v (abar^_v + lambda x^_v))   lines 9, 11
//   abar_v += dalpha a~_k / n                              line 13
//   alpha~_i += dalpha                                     line 12 (reading R9)
// The samples are known in advance (counter-based sampler), so the row data of
// sample t+W is prefetched into L1 while sample t computes, and the row bounds
// of sample t+2W one step earlier: the HBM row fetch leaves the critical path,
// which becomes gather (L2) -> reduce -> exp -> RED.
// The first NR*G entries of a row keep (c, a~, q = D(abar + lambda x)) in
// registers; longer rows stash q in shared memory and re-read c, a~ (read-only).
// DET: one worker; a gpu-scope fence + __syncwarp between samples makes sample
// t+1 read every write of sample t, i.e. sequential Sparse SAGA.
struct UpdateParams {
  const int64_t* rowptr;
  const int32_t* cols;
  const double* vals;   // a (the caller's values; the label is applied per sample)
  const double* y;      // b_i in {-1, +1}
  const double* dv;     // D_{c_k} per stored entry (not read by the FULL combine kernel)
  const double* D;      // D_v (combine kernel: the hot features' table)
  double2* xa;          // {x_v, abar_v} at xa[v * S]
  int S;                // pair stride
  double* habar;        // abar_v of hot-split features (entries with dv < 0)
  double* alpha;        // folded alpha~
  int32_t* visits;      // NULL unless record_samples
  unsigned long long* shash;  // NULL unless record_samples: sum over processed t of mix(t, i_t)
  unsigned long long* ov;  // NULL, or overlap instrumentation (NEXT-1, App. D):
                           // [0] sparse global progress counter (+100 per 100 local samples),
                           // [1] sum and [2] count of per-sample overlap estimates, [3] max
  int ov_every;            // measure every ov_every-th local sample
  int repl_d;              // REPL: features held in the per-CTA shared-memory replica (= d)
  int repl_every;          // REPL: a group refreshes G replica entries every repl_every samples
  int frozen;              // 1: the memory (alpha, abar) is read but never written --
                           // KROMAGNON inner steps (alpha = sigma(x~), abar = mu) and
                           // HOGWILD (alpha = abar = 0), NEXT-2
  uint64_t n;
  double gamma, lambda_, inv_n;
  uint64_t seed, t0, T;
  int64_t workers;
  int overflow;         // shared-memory q slots per group (>= max_row - NR*G, or 0)
  double bulk_dmax;     // MODE 2: entries with D_c <= bulk_dmax (popular features,
                        // p_c >= 1/bulk_dmax) use the TMA bulk pair reduction, others REDs
  int debug_mode;       // profiling build only: bit0 skip the scatter, bit1 skip exp/div
  // asaga_combine_kernel only
  int H;                  // hot features combined per block (slots 0..H-1)
  int nwb;                // worker groups per block
  const int32_t* hot_id;  // slot -> feature (NULL when every feature is hot: slot = feature)
  const int32_t* eslot;   // per stored entry: slot of its feature, or -1 (cold)
  unsigned long long* comm_passes;  // += communication-warp passes (asaga_stats)
  int wt;                 // combine_write_through: hot adds go straight to L2 (replica reads only)
  int split;              // hot split in use (entries with dv < 0 keep abar in habar)
  double late_dmax;       // asaga_pipe_kernel: entries with |D_c| <= late_dmax are hot (read late)
  double hot_dmax;        // asaga_pipe_kernel: hot split of features with D_c <= hot_dmax
  int merge_ts;           // asaga_pipe_kernel<CMB>: merge-table positions (power of 2 >= 2H)
  int merge_ns;           // ... flush period of the communication warp (ns)
  int bulk_rows;          // asaga_update_kernel: stage rows by 1-D TMA bulk copies (cols, vals, dv
                          // 16-B aligned); 0 = per-element cp.async
  int64_t nnz;            // stored entries (bulk copies never read past them)
  const int* ok;          // run guard: 0 = skip (an asynchronous reload's data does not fit)
  // asaga_update_kernel<REC>: D_v from the 32-byte record (no dv stream); hot split by
  // membership in hot_tab (2^hot_log slots, copied to shared memory), NULL = no split
  const int32_t* hot_tab;
  int hot_log;
  int pair_red;           // asaga_update_kernel (REDs, no record layout): paired scatter
};

// Shared memory per group: a P-entry {dx, dabar} source buffer for the TMA bulk
// scatter (16-B aligned, first), 2 stages of the first P = NR*G row entries, then
// `overflow` fp64 q slots for rows longer than P.  A stage holds the row's values, D's and
// columns from 16-B aligned starts (a bulk copy moves whole 16-B units: up to 1 leading
// fp64 / 3 leading int32 of the previous row come along, so entry e of the row sits at
// slot (lo & 1) + e / (lo & 3) + e), then b_i and the stage's mbarrier.
template <int G, int NR>
struct GroupSmem {
  static constexpr int P = NR * G;
  static constexpr int PV = P + 2;  // fp64 slots: 1 leading + 1 trailing of alignment slack
  static constexpr int PC = P + 4;  // int32 slots: 3 leading + 1 trailing
  static constexpr size_t delta_bytes = (size_t)P * 2 * sizeof(double);
  static constexpr size_t vals_off = 0;
  static constexpr size_t dv_off = (size_t)PV * sizeof(double);
  static constexpr size_t cols_off = 2 * (size_t)PV * sizeof(double);
  static constexpr size_t label_off = cols_off + (size_t)PC * sizeof(int32_t);  // 16-B multiple
  static constexpr size_t mbar_off = label_off + 8;
  static constexpr size_t stage_bytes = label_off + 16;
  static __host__ __device__ size_t bytes(int overflow) {
    return delta_bytes + 2 * stage_bytes + (size_t)overflow * sizeof(double);
  }
};

// 1-D TMA (cp.async.bulk) helpers: a global -> shared copy completing on an mbarrier
// (transaction bytes), issued by one lane; the group waits on the barrier's phase.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, void* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

// TMA bulk reduction of one {x, abar} pair: a single 16-byte .add.f64 performed at
// L2 by the async proxy (UBLKRED) -- one L2 operation instead of two REDs on the
// feature's line, and no LSU wavefronts (profiles/r01_update_kernel.md).
__device__ __forceinline__ void bulk_red_pair(double2* gdst, const double2* ssrc) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 16;" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Row staging of the plain update kernel: the first P entries of the row (values, D per
// entry unless dv is NULL -- the record layout --, columns) into a stage.  bulk: lane 0 issues three 1-D TMA copies of the 16-B
// aligned supersets (UBLKCP: three instructions per row instead of 3 ceil(len/G) LDGSTS per
// lane), completing on the stage's mbarrier; otherwise (misaligned caller arrays, or the
// last rows, whose aligned superset would read past nnz) per-element cp.async, and lane 0
// arrives on the barrier without transaction bytes.  b_i always by cp.async.
template <int G, int NR>
__device__ __forceinline__ void issue_row_copy(unsigned char* base, int stage, const int32_t* cols,
                                               const double* vals, const double* dv, const double* b_i,
                                               int64_t lo, int64_t hi, int g, int bulk, int64_t nnz) {
  using GS = GroupSmem<G, NR>;
  constexpr int P = NR * G;
  unsigned char* sb = base + GS::delta_bytes + stage * GS::stage_bytes;
  double* sv = reinterpret_cast<double*>(sb + GS::vals_off);
  double* sd = reinterpret_cast<double*>(sb + GS::dv_off);
  int32_t* sc = reinterpret_cast<int32_t*>(sb + GS::cols_off);
  void* bar = sb + GS::mbar_off;
  if (g == 0) cp_async8(sb + GS::label_off, b_i);
  const uint64_t pol = policy_evict_first();
  const int64_t hs = hi - lo > P ? lo + P : hi;  // staged entries [lo, hs)
  const int64_t lo_c = lo & ~(int64_t)3, hi_c = (hs + 3) & ~(int64_t)3;
  const int64_t lo_v = lo & ~(int64_t)1, hi_v = (hs + 1) & ~(int64_t)1;
  // (the caller has synchronised the group since the previous sample's scatter read the
  // stage this copy overwrites: asaga_update_kernel's loop top)
  if (bulk && hi_c <= nnz && hi_v <= nnz) {  // group-uniform
    if (g == 0) {
      const unsigned bc = (unsigned)((hi_c - lo_c) * 4), bv = (unsigned)((hi_v - lo_v) * 8);
      fence_proxy_async_smem();  // earlier generic reads of this stage before the async writes
      mbar_arrive_tx(bar, bc + (dv != nullptr ? 2 : 1) * bv);
      bulk_g2s(sc, cols + lo_c, bc, bar, pol);
      bulk_g2s(sv, vals + lo_v, bv, bar, pol);
      if (dv != nullptr) bulk_g2s(sd, dv + lo_v, bv, bar, pol);
    }
  } else {
    const int len = (int)(hs - lo);
    const int oc = (int)(lo & 3), ov = (int)(lo & 1);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;  // group-uniform: no predicated-off chunks
      const int64_t k = lo + j * G + g;
      if (j * G + g < len) {
        cp_async4_ef(sc + oc + j * G + g, cols + k, pol);
        cp_async8_ef(sv + ov + j * G + g, vals + k, pol);
        if (dv != nullptr) cp_async8_ef(sd + ov + j * G + g, dv + k, pol);
      }
    }
    if (g == 0) mbar_arrive(bar);  // (the data is waited for with cp.async.wait_all)
  }
  cp_async_commit();
}

#ifdef ASAGA_TIMING
// Profiling build only (tools/timing_build.py): per-phase SM-cycle sums of group
// leaders: [0] row wait, [1] gathers+dot, [2] reduce+exp, [3] scatter issue,
// [4] loop tail, [5] iterations.
__device__ unsigned long long g_phase_cycles[12];
#define TMARK(k)                                     \
  do {                                               \
    long long now_ = clock64();                      \
    ph[k] += (unsigned long long)(now_ - tprev);     \
    tprev = now_;                                    \
  } while (0)
#else
#define TMARK(k) \
  do {           \
  } while (0)
#endif

// MODE: 0 = plain load + store (non-atomic ablation), 1 = red.global.add.f64 per
// element (LSU), 2 = hybrid: one TMA bulk 16-byte reduction per {x, abar} pair of
// a popular feature (D_c <= bulk_dmax: its L2 line is the bottleneck), REDs for the
// rest (the bulk op is issued lane by lane, ~64 cycles each).
// REPL (small d, async only): every CTA keeps a shared-memory replica of all {x_v, abar_v}
// pairs; gathers read the replica (30-cycle LDS instead of an L2 round trip on the hot
// lines) while every write still goes to the shared state in L2.  Each group refreshes G
// replica entries from L2 every repl_every samples, so a replica value is a past value of
// the shared state of bounded age: the reads stay the paper's inconsistent reads (P:137,
// P:266-268) with a larger, still bounded, overlap (Assumption 1).
// REC (record layout, MODE 1, no replica): D_v comes with the gather of the 32-byte
// coordinate record (no per-entry D stream, no expand pass); a hot-split entry is found
// in the block's shared copy of the membership table.
// (REC keeps x, abar, D and a hot entry's abar of every chunk in flight: 8 registers per
// chunk instead of 4, so one resident 256-thread block per SM -- 8 samples, beyond the
// ~3 per SM the convergent concurrency asks for -- and no spills at NR = 8)
template <int G, int NR, bool DET, int MODE, bool REPL, bool REC>
// One resident 256-thread block per SM is all the launch shape uses (the convergent numbers
// in flight are 3-4 groups per SM), so the register cap is 255: at the former cap of 128
// (2 blocks per SM) the kernel spilled as soon as anything was added, and ran ~2 % slower on
// c4 at 128 (profiles/r02_update_kernel.md section 18).  ASAGA_UPD_MIN_BLOCKS: measurement
// variant.
#ifndef ASAGA_UPD_MIN_BLOCKS
#define ASAGA_UPD_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(256, ASAGA_UPD_MIN_BLOCKS) asaga_update_kernel(UpdateParams p) {
  constexpr bool ATOMIC = MODE != 0;
  static_assert(!REC || (MODE == 1 && !REPL), "record layout: REDs, no replica");
  if (p.ok != nullptr && *reinterpret_cast<const volatile int*>(p.ok) == 0) return;  // run guard
#ifdef ASAGA_TIMING
  unsigned long long ph[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#endif
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int P = NR * G;
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (unsigned)(lane & ~(G - 1)));
  // groups are dealt to blocks round robin (w = group slot * grid + block): with at least
  // as many workers as SMs every SM runs some (launch_shape puts one block on each)
  const int64_t w = (int64_t)(threadIdx.x / G) * gridDim.x + blockIdx.x;
  double2* rx = reinterpret_cast<double2*>(smem_raw);  // REPL replica (first in smem)
  const size_t repl_bytes = REPL ? (((size_t)p.repl_d * sizeof(double2) + 15) & ~(size_t)15)
                            : (REC && p.hot_tab != nullptr) ? ((size_t)sizeof(int32_t) << p.hot_log) : 0;
  if (REPL) {  // fill before any early exit: the whole block takes part in the barrier
    for (int v = threadIdx.x; v < p.repl_d; v += blockDim.x) rx[v] = ld_na2(p.xa + (int64_t)v * p.S);
    __syncthreads();
  }
  int32_t* ht = reinterpret_cast<int32_t*>(smem_raw);  // REC: the hot-split table (first in smem)
  if (REC && p.hot_tab != nullptr) {
    for (int q = threadIdx.x; q < (1 << p.hot_log); q += blockDim.x) ht[q] = __ldg(p.hot_tab + q);
    __syncthreads();
  }
  const double* const dvs = REC ? nullptr : p.dv;  // the row stream's D (not with REC)
  if (w >= p.workers) return;
  unsigned char* gbase =
      smem_raw + repl_bytes + (size_t)(threadIdx.x / G) * GroupSmem<G, NR>::bytes(p.overflow);
  int rcur = REPL ? (int)(((threadIdx.x / G) * G) % (p.repl_d > 0 ? p.repl_d : 1)) : 0;
  int rtick = 0;
  double2* dbuf = reinterpret_cast<double2*>(gbase);
  double* qs = reinterpret_cast<double*>(gbase + GroupSmem<G, NR>::delta_bytes +
                                         2 * GroupSmem<G, NR>::stage_bytes);

  const uint64_t tend = p.t0 + p.T;
  uint64_t t = p.t0 + (uint64_t)w;
  if (t >= tend) return;
  const uint64_t W = (uint64_t)p.workers;
  const uint64_t t_first = t;
  // the two stages' mbarriers (one arrival per use: lane 0's expect_tx or plain arrive)
  using GS = GroupSmem<G, NR>;
  if (g == 0) {
    mbar_init(gbase + GS::delta_bytes + GS::mbar_off, 1);
    mbar_init(gbase + GS::delta_bytes + GS::stage_bytes + GS::mbar_off, 1);
    mbar_init_fence();
  }
  __syncwarp(gmask);
  unsigned phase_bits = 0;  // bit s: parity of stage s's next completion
  // sample indices in batches of G: lane j draws sample mb + j of this worker (one Philox
  // per lane per G samples), shuffled out in order (group-uniform calls)
  int64_t bi = 0;
  auto draw_batch = [&](uint64_t mb) {
    const uint64_t ts = t_first + (mb + (uint64_t)g) * W;
    bi = ts < tend ? sample_row(p.seed, ts, p.n) : 0;
  };
  auto sample_of = [&](uint64_t ms) -> int64_t {
    return __shfl_sync(gmask, bi, (int)(ms & (uint64_t)(G - 1)), G);
  };
  static_assert(G >= 4, "a batch covers the prologue's three samples");
  uint64_t m = 0;  // this worker's sample count
  draw_batch(0);
  // prologue: current row bounds + its copy; next row bounds; next-next index
  int64_t i = sample_of(0);
  int64_t lo = __ldg(&p.rowptr[i]), hi = __ldg(&p.rowptr[i + 1]);
  int stage = 0;
  issue_row_copy<G, NR>(gbase, stage, p.cols, p.vals, dvs, p.y + i, lo, hi, g, p.bulk_rows, p.nnz);
  int64_t in1 = 0, lo1 = 0, hi1 = 0, in2 = 0;
  in1 = sample_of(1);
  in2 = sample_of(2);
  if (t + W < tend) {
    lo1 = __ldg(&p.rowptr[in1]);
    hi1 = __ldg(&p.rowptr[in1 + 1]);
  }

  unsigned long long ov_sum = 0, ov_cnt = 0, ov_max = 0;
  unsigned long long shash = 0;
  int ov_local = 0, ov_iter = 0;
  while (true) {
    // overlap estimate (App. D): progress counter at the read and after the write
    bool ov_meas = false;
    if (p.ov != nullptr) ov_meas = (ov_iter++ % p.ov_every) == 0;
    unsigned long long ov_c0 = 0;
    if (ov_meas) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(ov_c0) : "l"(p.ov));
    // ---- pass 1: row entries (shared memory), gathers, dot product
    const int len = (int)(hi - lo);
    cp_async_wait_all();
    unsigned char* sbase = gbase + GS::delta_bytes + stage * GS::stage_bytes;
    mbar_wait(sbase + GS::mbar_off, (phase_bits >> stage) & 1u);
    phase_bits ^= 1u << stage;
    // The group synchronises here: (1) b_i is lane 0's cp.async (the mbarrier tracks the
    // bulk bytes only, and lane 0 arrives before its per-element copies land), so the other
    // lanes may read it only after lane 0's wait above; (2) this iteration's look-ahead copy
    // overwrites the stage the previous sample scattered from, slots other lanes read (the
    // bulk path writes the whole stage from lane 0; a row at another 16-B offset shifts every
    // slot of the per-element path).  Nothing else orders the group's lanes between that
    // scatter and here: without it, c3 at its operating point plateaued at f - f* ~ 1e-4
    // once the record layout changed the code's timing (a stale b_i flips a lane's signs).
#ifndef ASAGA_NO_GROUP_SYNC  // (measurement variant only)
    __syncwarp(gmask);
#endif
    TMARK(0);
    const double* sv = reinterpret_cast<const double*>(sbase + GS::vals_off) + (lo & 1);
    const double* sd = reinterpret_cast<const double*>(sbase + GS::dv_off) + (lo & 1);
    const int32_t* sc = reinterpret_cast<const int32_t*>(sbase + GS::cols_off) + (lo & 3);
    // b_i came with the row (carrying it in registers next to the row bounds measured 9 %
    // slower on c3; a plain load next to alpha_i's, 2 %)
    const double yb = *reinterpret_cast<const double*>(sbase + GS::label_off);
    // gathers of x^, abar^ and D for every resident chunk are issued before any use
    double qq[NR];
    double2 xb[NR];
    double Dr[NR], hb[NR];  // REC: D_c from the record; abar_c of a hot-split entry
    unsigned hm = 0;        // REC: bit j = chunk j's entry is hot-split
    if (REC) {
      // every record gather first, then the table lookups and the hot entries' abar gathers
      // (separate registers: no load waits on another in-flight load's destination)
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;  // group-uniform
        if (j * G + g < len) {
          const Rec3 r = ld_na_rec(p.xa + (int64_t)sc[j * G + g] * p.S);
          xb[j] = make_double2(r.x, r.ab);
          Dr[j] = r.D;
        }
      }
      if (p.hot_tab != nullptr) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          if (j * G >= len) break;  // group-uniform
          if (j * G + g < len) {
            const int c = sc[j * G + g];
            if (hot_lookup(ht, p.hot_log, c)) {
              hb[j] = ld_na(p.habar + c);
              hm |= 1u << j;
            }
          }
        }
      }
    } else
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;  // group-uniform
      const int64_t k = lo + j * G + g;
      if (j * G + g < len) {
        const int c = sc[j * G + g];
        if (!REC && dvs == nullptr) qq[j] = __ldg(p.D + c);  // d_gather: D_c with the gather
        if (REPL)
          xb[j] = rx[c];
        else if (p.split && sd[j * G + g] < 0.0)  // hot split: x and abar on separate lines
#ifdef ASAGA_TIMING
          // bit7: no load of a hot entry's x (its RED stays): the hot lines carry REDs only
          xb[j] = make_double2((p.debug_mode & 128) ? 0.0 : ld_na(&p.xa[(int64_t)c * p.S].x),
                               (p.debug_mode & (8 | 256)) ? 0.0 : ld_na(p.habar + c));  // bit3: no hot abar ops
          // (bit8: no load of a hot entry's abar, its RED stays)
#else
          xb[j] = make_double2(ld_na(&p.xa[(int64_t)c * p.S].x), ld_na(p.habar + c));
#endif
        else
#ifdef ASAGA_TIMING
          // bit6: no cold gathers (with bit5: a kernel of the hot features' operations only,
          // whose rate at a large number in flight is the hot lines' ceiling in situ)
          xb[j] = (p.debug_mode & 64) ? make_double2(0.0, 0.0) : ld_na2(p.xa + (int64_t)c * p.S);
#else
          xb[j] = ld_na2(p.xa + (int64_t)c * p.S);
#endif
      }
    }
    const double ai = ld_na(p.alpha + i);
    // REPL: refresh G replica entries from the shared state every repl_every samples
    const bool refresh = REPL && (++rtick >= p.repl_every);
    double2 rv = make_double2(0.0, 0.0);
    int rf = 0;
    if (refresh) {
      rf = rcur + g;
      if (rf >= p.repl_d) rf -= p.repl_d;
      if (g < p.repl_d) rv = ld_na2(p.xa + (int64_t)rf * p.S);
    }
    // ---- look-ahead (read-only data): copy row t+W, load bounds of t+2W
    const bool has1 = t + W < tend, has2 = t + 2 * W < tend;
#ifdef ASAGA_TIMING
    const bool copy_late = (p.debug_mode & 4) != 0;
#else
    constexpr bool copy_late = false;
#endif
    if (has1 && !copy_late)
      issue_row_copy<G, NR>(gbase, stage ^ 1, p.cols, p.vals, dvs, p.y + in1, lo1, hi1, g, p.bulk_rows, p.nnz);
    int64_t lo2 = 0, hi2 = 0;
    if (has2) {
      lo2 = __ldg(&p.rowptr[in2]);
      hi2 = __ldg(&p.rowptr[in2 + 1]);
    }
    double dot = 0.0;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;  // group-uniform
      const int64_t k = lo + j * G + g;
      if (j * G + g < len) {
        dot = fma(sv[j * G + g], xb[j].x, dot);
        if (REC)
          qq[j] = Dr[j] * fma(p.lambda_, xb[j].x, ((hm >> j) & 1u) ? hb[j] : xb[j].y);
        else
          qq[j] = (dvs == nullptr ? qq[j] : fabs(sd[j * G + g])) * fma(p.lambda_, xb[j].x, xb[j].y);
      }
    }
    if (len > P)  // group-uniform: long rows only
    for (int64_t k = lo + P + g; k < hi; k += G) {
      const int c = ld_nc_i32(p.cols + k);
      const double a = ld_nc_f64(p.vals + k);
      if (REC) {
        const Rec3 r = ld_na_rec(p.xa + (int64_t)c * p.S);
        const bool hot = p.hot_tab != nullptr && hot_lookup(ht, p.hot_log, c);
        const double ab = hot ? ld_na(p.habar + c) : r.ab;
        dot = fma(a, r.x, dot);
        qs[k - lo - P] = r.D * fma(p.lambda_, r.x, ab);
        continue;
      }
      const double Dv = dvs == nullptr ? __ldg(p.D + c) : ld_nc_f64(p.dv + k);
      const double2 v = REPL ? rx[c]
                        : Dv < 0.0 ? make_double2(ld_na(&p.xa[(int64_t)c * p.S].x), ld_na(p.habar + c))
                                   : ld_na2(p.xa + (int64_t)c * p.S);
      dot = fma(a, v.x, dot);
      qs[k - lo - P] = fabs(Dv) * fma(p.lambda_, v.x, v.y);
    }
    if (has1 && copy_late)
      issue_row_copy<G, NR>(gbase, stage ^ 1, p.cols, p.vals, dvs, p.y + in1, lo1, hi1, g, p.bulk_rows, p.nnz);
    TMARK(1);
    // ---- scalar derivative (folded logistic) and memory difference
    dot = group_sum<G>(dot, gmask) * yb;  // folded margin b_i a_i . x^ (exact: b = +-1)
#ifdef ASAGA_TIMING
    const double sig = (p.debug_mode & 2) ? -0.5 + 0.0 * dot : sigma_folded(dot);
#else
    const double sig = sigma_folded(dot);
#endif
    const double da = sig - ai;
    const double db = da * yb;  // dalpha a~_k = (dalpha b_i) a_k, exact
    const double ngam = -p.gamma;
    TMARK(2);
#ifdef ASAGA_TIMING
    if (!(p.debug_mode & 1)) {
#endif
    // ---- pass 2: unlocked scatter (Property 3: atomic adds, no locks); row entries
    //      are re-read from the stage buffer, which is only overwritten next iteration
    if (MODE == 2) bulk_wait_read();  // the previous sample's bulk ops have read dbuf
    TMARK(6);
    if (MODE == 1 && (!REC || p.hot_tab == nullptr) && p.pair_red && !p.frozen) {
      // Paired scatter: lanes g and g^1 (partners) hold entries e0 (even lane) and e1 (odd
      // lane).  Each lane adds x of its own entry and abar of its partner's (the partner's
      // column, value and D are in the stage; abar's add needs no gathered value), in the
      // order that puts the x and abar adds of ONE entry into the same instruction:
      //   instruction 1: x(e0) by the even lane, abar(e0) by the odd lane
      //   instruction 2: abar(e1) by the even lane, x(e1) by the odd lane
      // Both words of a {x, abar} pair share a 32-byte sector, and L2 serves the lanes of
      // one reduction instruction that hit one sector as one request: half the requests of
      // one instruction per word (tools/red_pairing.cu: 2x the cold-entry rate, 1.65x the
      // rate of a popular pair).  Same adds, same values (Property 3).
      const bool odd = (g & 1) != 0;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;  // group-uniform
        const int e = j * G + g, ep = e ^ 1;
        const bool own = e < len, pin = ep < len;
        double* xv;
        double* abp;
        double dx, dyp;
        if (REC) {
          // branch-free (the record layout has no hot split here): the stage's slots past the
          // row's end hold stale data, never dereferenced -- those lanes' reductions are
          // predicated off.  The scatter phase halves (c3: 1.87e8 -> 1.94e8); on the default
          // layout (c4) the same form is slower (profiles/r02_update_kernel.md section 24).
          const int c = sc[e], cp = sc[ep];
          xv = &p.xa[(int64_t)c * p.S].x;
          abp = &p.xa[(int64_t)cp * p.S].x + 1;
          dx = ngam * fma(db, sv[e], qq[j]);
          dyp = db * sv[ep] * p.inv_n;
        } else {
          xv = &p.xa->x;  // (any valid address: the add is predicated off)
          dx = 0.0;
          if (own) {
            xv = &p.xa[(int64_t)sc[e] * p.S].x;
            dx = ngam * fma(db, sv[e], qq[j]);
          }
          abp = &p.xa->x;
          dyp = 0.0;
          if (pin) {
            const int cp = sc[ep];
            abp = (p.split && sd[ep] < 0.0) ? p.habar + cp : &p.xa[(int64_t)cp * p.S].x + 1;  // hot split
            dyp = db * sv[ep] * p.inv_n;
          }
        }
        red_add_if(odd ? abp : xv, odd ? dyp : dx, odd ? pin : own);
        red_add_if(odd ? xv : abp, odd ? dx : dyp, odd ? own : pin);
      }
    } else
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;  // group-uniform
      const int64_t k = lo + j * G + g;
      if (j * G + g < len) {
        const int c = sc[j * G + g];
        const double a = sv[j * G + g];
        const double u = fma(db, a, qq[j]);
        double* xv = &p.xa[(int64_t)c * p.S].x;
        double* abv = REC ? (((hm >> j) & 1u) ? p.habar + c : xv + 1)
                          : (p.split && sd[j * G + g] < 0.0) ? p.habar + c : xv + 1;  // hot split
        if (MODE == 2 && sd[j * G + g] <= p.bulk_dmax) {
          dbuf[j * G + g] = make_double2(ngam * u, p.frozen ? 0.0 : db * a * p.inv_n);
        } else if (MODE >= 1) {
#ifdef ASAGA_TIMING
          // bit4: no x RED for hot (split) entries; bit5: no REDs at all for cold entries
          const bool hot_e = abv != xv + 1;
          if (!((p.debug_mode & 16) && hot_e) && !((p.debug_mode & 32) && !hot_e)) red_add(xv, ngam * u);
          if (!p.frozen && !((p.debug_mode & 8) && hot_e) && !((p.debug_mode & 32) && !hot_e))
            red_add(abv, db * a * p.inv_n);
#else
          red_add(xv, ngam * u);
          if (!p.frozen) red_add(abv, db * a * p.inv_n);
#endif
        } else {
          st_cg(xv, ld_cg(xv) + ngam * u);
          if (!p.frozen) st_cg(abv, ld_cg(abv) + db * a * p.inv_n);
        }
      }
    }
    if (MODE == 2) {
      TMARK(7);
      fence_proxy_async_smem();
      TMARK(8);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;
        const int64_t k = lo + j * G + g;
        if (j * G + g < len && sd[j * G + g] <= p.bulk_dmax)
          bulk_red_pair(p.xa + (int64_t)sc[j * G + g] * p.S, dbuf + j * G + g);
      }
      bulk_commit();
    }
    if (len > P)  // group-uniform: long rows only
    for (int64_t k = lo + P + g; k < hi; k += G) {
      const int c = ld_nc_i32(p.cols + k);
      const double a = ld_nc_f64(p.vals + k);
      const double u = fma(db, a, qs[k - lo - P]);
      double* xv = &p.xa[(int64_t)c * p.S].x;
      const bool hot = REC ? (p.hot_tab != nullptr && hot_lookup(ht, p.hot_log, c))
                           : (dvs != nullptr && ld_nc_f64(p.dv + k) < 0.0);
      double* abv = hot ? p.habar + c : xv + 1;  // hot split
      if (ATOMIC) {
        red_add(xv, ngam * u);
        if (!p.frozen) red_add(abv, db * a * p.inv_n);
      } else {
        st_cg(xv, ld_cg(xv) + ngam * u);
        if (!p.frozen) st_cg(abv, ld_cg(abv) + db * a * p.inv_n);
      }
    }
#ifdef ASAGA_TIMING
    }
#endif
    if (refresh) {
      if (g < p.repl_d) rx[rf] = rv;
      rcur += G;
      if (rcur >= p.repl_d) rcur -= p.repl_d;
      rtick = 0;
    }
    TMARK(3);
    if (g == 0) {
      if (p.frozen) {
      } else if (ATOMIC) {
        red_add(p.alpha + i, da);
      } else {
        st_cg(p.alpha + i, ai + da);
      }
      if (p.visits) {
        atomicAdd(p.visits + i, 1);
        shash += sample_mix(t, i);
      }
      if (p.ov != nullptr) {
        if (++ov_local == 100) {  // sparse counter: one +100 per 100 local updates
          atomicAdd(p.ov, 100ull);
          ov_local = 0;
        }
        if (ov_meas) {
          unsigned long long c1;
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c1) : "l"(p.ov));
          const unsigned long long o = c1 - ov_c0;
          ov_sum += o;
          ov_cnt += 1;
          ov_max = max(ov_max, o);
        }
      }
    }
    if (DET) {
      if (MODE == 2) {
        bulk_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __threadfence();
      __syncwarp(gmask);
    }
#ifdef ASAGA_TIMING
    ph[5] += 1;
#endif
    TMARK(4);
    if (!has1) break;
    t += W;
    i = in1; lo = lo1; hi = hi1;
    in1 = in2; lo1 = lo2; hi1 = hi2;
    ++m;
    if (t + 2 * W < tend) {  // group-uniform
      if (((m + 2) & (uint64_t)(G - 1)) == 0) draw_batch(m + 2);
      in2 = sample_of(m + 2);
    }
    stage ^= 1;
  }
  cp_async_wait_all();
  if (MODE == 2) bulk_wait_all();
  if (p.visits && g == 0) atomicAdd(p.shash, shash);
  if (p.ov != nullptr && g == 0 && ov_cnt > 0) {
    atomicAdd(p.ov + 1, ov_sum);
    atomicAdd(p.ov + 2, ov_cnt);
    atomicMax(p.ov + 3, ov_max);
  }
#ifdef ASAGA_TIMING
  if (g == 0)
    for (int k = 0; k < 9; ++k) atomicAdd(&g_phase_cycles[k], ph[k]);
#endif
}

// ---------------------------------------------------------------------------
// A2..A8 with CTA-level combining of the hot features (async only; option
// combine_hot).  Every update touches the few most popular features, and L2 serves
// one line's operations serially, so with every sample sending its adds straight to
// L2 the hottest line caps the update rate (profiles/r01_update_kernel.md).  Here
// each thread block keeps, for H hot features (slot s -> feature hot_id[s], or all
// d features with slot = feature when FULL):
//   xr[s]   a replica of {x_v, abar_v} the workers read (an LDS, no L2 round trip)
//   pend[s] the block's adds not yet sent to L2 (shared-memory atomic adds)
// and one communication warp loops: take pend[s] (atomic exchange with 0), send it
// to the shared state with red.global.add.f64, re-read the shared pair and store
// xr[s] = shared + pend[s].  The shared state therefore receives one add per hot
// feature per block per pass instead of one per sample, and every coordinate a
// worker reads is the shared value of a recent moment plus some of the block's own
// recent adds: x^ = x_t minus a bounded set of recent updates -- the paper's
// inconsistent read with a larger, still bounded, overlap (Assumption 1, P:316-322;
// DESIGN.md reading R23).  Cold features (slot -1) are read from / added to L2 per
// sample exactly as in asaga_update_kernel.  Every add reaches the shared state
// (the comm warp flushes pend after the block's workers finish), so the quiescent
// identity abar = (1/n) sum_i alpha_i a_i holds as in the plain kernel.
// Worker w = blockIdx.x * nwb + (thread / G), processes t = t0 + w + kW as in
// asaga_update_kernel (same t -> worker map).  alpha_i is copied with its row, KS = 3
// samples ahead of its use (about 3W updates before this worker adds to it): the read of
// the memory alpha^_i is inconsistent by that bounded window, counted in
// DESIGN.md reading R23 (a repeat of i within ~3W updates, probability ~3W/n, sees the
// older alpha^_i; the atomic add still applies every dalpha exactly once).
template <int G, int NR, bool FULL>
struct CombSmem {
  static constexpr int P = NR * G;
  static constexpr int KS = 3;  // row stages: rows are copied KS samples ahead
  // per stage: fp64 value, [fp64 D, !FULL], int32 column, [int32 slot, !FULL], then alpha_i
  // (FULL: every feature has a slot and D_v comes from the block's table, not the stream)
  static constexpr size_t alpha_off = FULL ? (size_t)P * (sizeof(double) + sizeof(int32_t))
                                           : (size_t)P * (2 * sizeof(double) + 2 * sizeof(int32_t));
  static constexpr size_t stage_bytes = (alpha_off + 2 * sizeof(double) + 15) & ~(size_t)15;  // + alpha_i, b_i
  // bounds ring: {lo, hi, i} of samples fetched 2 KS ahead (cp.async, no register waits)
  static constexpr int NB = 2 * KS;
  static constexpr size_t ring_off = KS * stage_bytes;
  static constexpr size_t ring_bytes = NB * 32;
  static __host__ __device__ size_t bytes(int overflow) {
    return ((ring_off + ring_bytes + (size_t)overflow * sizeof(double)) + 15) & ~(size_t)15;
  }
};

__device__ __forceinline__ double2 lds_vol2(const double2* p) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
// Thread-block-cluster helpers (DSMEM): addresses are 32-bit shared::cluster windows.
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa_shared(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a)
               : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
  return a;
}
// all (non-exited) threads of all blocks of the cluster; release / acquire
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ double exch_cluster_f64(unsigned a) {
  unsigned long long old;
  asm volatile("atom.shared::cluster.exch.b64 %0, [%1], %2;" : "=l"(old) : "r"(a), "l"(0ull) : "memory");
  return __longlong_as_double((long long)old);
}
__device__ __forceinline__ double ld_cluster_f64(unsigned a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_cluster_v2(unsigned a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int ld_cluster_volatile_s32(unsigned a) {
  int v;
  asm volatile("ld.volatile.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void atomic_add_cluster_s32(unsigned a, int v) {
  asm volatile("red.shared::cluster.add.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ double exch_shared(double* p) {
  return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long*>(p), 0ull));
}

template <int G, int NR, bool FULL>
__device__ __forceinline__ void issue_row_copy_c(unsigned char* base, int stage, const int32_t* cols,
                                                 const int32_t* eslot, const double* vals,
                                                 const double* dv, const double* alpha_i, const double* b_i,
                                                 int64_t lo, int64_t hi, int g) {
  constexpr int P = NR * G;
  unsigned char* sb = base + stage * CombSmem<G, NR, FULL>::stage_bytes;
  if (g == 0) {
    cp_async8(sb + CombSmem<G, NR, FULL>::alpha_off, alpha_i);
    cp_async8(sb + CombSmem<G, NR, FULL>::alpha_off + sizeof(double), b_i);
  }
  double* sv = reinterpret_cast<double*>(sb);
  double* sd = sv + P;  // !FULL only
  int32_t* sc = reinterpret_cast<int32_t*>(sv + (FULL ? P : 2 * P));
  int32_t* ss = sc + P;
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (lo + j * G >= hi) break;  // group-uniform
    const int64_t k = lo + j * G + g;
    if (k < hi) {
      cp_async4(sc + j * G + g, cols + k);
      if (!FULL && eslot != nullptr) cp_async4(ss + j * G + g, eslot + k);
      cp_async8(sv + j * G + g, vals + k);
      if (!FULL) cp_async8(sd + j * G + g, dv + k);
    }
  }
  cp_async_commit();
}

// Block size (launch bounds): 768 threads -- up to 46 workers of 16 lanes + the
// communication warp per SM at <= 80 registers, no spills (512-thread blocks capped c2 at
// W = 4440, 1024 forced 64 registers; profiles/r01_combine_kernel.md); 512 for NR = 8 (long
// rows), whose register queues would spill at 80.
__host__ __device__ constexpr int comb_block_threads(int nr) { return nr >= 8 ? 512 : 768; }
template <int G, int NR, bool FULL>
__global__ void __launch_bounds__(comb_block_threads(NR), 1) asaga_combine_kernel(UpdateParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (p.ok != nullptr && *reinterpret_cast<const volatile int*>(p.ok) == 0) return;  // run guard (whole grid)
  constexpr int P = NR * G;
  __shared__ int done;  // rank 0's copy counts the finished worker groups of the cluster
  const int H = p.H;
  double2* xr = reinterpret_cast<double2*>(smem_raw);
  double2* pend = xr + H;
  double* Ds = reinterpret_cast<double*>(pend + H);  // FULL: D_v of every feature
  unsigned char* stage_base = smem_raw + (size_t)H * (2 * sizeof(double2) + sizeof(double));
  const int nwb = p.nwb;  // worker groups in this block (nwb * G is a multiple of 32)
  const unsigned crank = cluster_ctarank(), csize = cluster_nctarank();
  const bool solo = csize == 1;  // one block per cluster: block barriers, plain shared memory
  // The block's hot-slot tables; every thread runs this once, from its role's code, after
  // a worker has issued its prologue loads (they overlap), then the start barrier.
  // The replica holds {x_v, q_v = D_v (abar_v + lambda x_v)}: the correction term is formed
  // once per refresh here instead of once per entry by every worker (same expression, same
  // rounding).
  auto replica_of = [&](double2 xab, double Dv) {
    return make_double2(xab.x, Dv * fma(p.lambda_, xab.x, xab.y));
  };
  auto init_slots = [&]() {
    for (int s = threadIdx.x; s < H; s += blockDim.x) {
      const int64_t v = FULL ? s : p.hot_id[s];
      const double Dv = p.D[v];
      xr[s] = replica_of(ld_relaxed2(p.xa + v * p.S), Dv);
      pend[s] = make_double2(0.0, 0.0);
      Ds[s] = Dv;
    }
    if (threadIdx.x == 0) done = 0;
  };
  // every block's replica and counter exist before any (remote) access
  auto start_sync = [&]() {
    if (solo) asm volatile("bar.sync 2;" ::: "memory");
    else cluster_sync_all();
  };
  auto end_sync = [&]() {
    if (solo) asm volatile("bar.sync 3;" ::: "memory");
    else cluster_sync_all();
  };
  const unsigned done0 = mapa_shared(&done, 0);

  if ((int)threadIdx.x >= nwb * G) {
    // ---------------- communication warp of cluster rank r: slots s = r (mod csize).
    // Per pass, for each of its slots: take the pending pair of EVERY block of the
    // cluster (remote atomic exchanges over DSMEM), send the sum with red.global.add.f64
    // (one add per hot feature per cluster per pass), re-read the shared pair and store
    // it into every block's replica.
    const int lane = threadIdx.x & 31;
    init_slots();
    start_sync();
    const int total = nwb * (int)csize;
    constexpr int B = 4;  // slots per lane per batch (their loads in flight together)
    unsigned long long passes = 0;
    const volatile int* vdone = &done;
    while ((solo ? *vdone : ld_cluster_volatile_s32(done0)) < total) {
      ++passes;
      for (int s0 = (int)crank + (int)csize * lane; s0 < H; s0 += (int)csize * 32 * B) {
        double2 gv[B], gd[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const int s = s0 + (int)csize * 32 * b;
          if (s < H) {
            const int64_t v = FULL ? s : p.hot_id[s];
            double2* gp = p.xa + v * p.S;
            double dx = 0.0, dy = 0.0;
            if (p.wt) {  // write-through: the workers' adds went to L2; refresh only
            } else if (solo) {
              dx = exch_shared(&pend[s].x);
              dy = exch_shared(&pend[s].y);
            } else {
              for (unsigned k = 0; k < csize; ++k) {
                const unsigned a = mapa_shared(&pend[s], k);
                dx += exch_cluster_f64(a);
                dy += exch_cluster_f64(a + 8);
              }
            }
            // read the shared pair BEFORE sending this pass's adds (the load then does not
            // queue behind them at the line) and count them in locally: g + d
            gv[b] = ld_relaxed2(gp);
            if (dx != 0.0) red_add(&gp->x, dx);
            if (dy != 0.0) red_add(&gp->y, dy);
            gd[b] = make_double2(dx, dy);
          }
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const int s = s0 + (int)csize * 32 * b;
          if (s < H) {
            if (solo) {  // + this pass's adds + the adds that arrived since the exchange
              const double2 q = lds_vol2(pend + s);
              xr[s] = replica_of(make_double2(gv[b].x + gd[b].x + q.x, gv[b].y + gd[b].y + q.y), Ds[s]);
            } else {
              const double2 r = replica_of(make_double2(gv[b].x + gd[b].x, gv[b].y + gd[b].y), Ds[s]);
              for (unsigned k = 0; k < csize; ++k) st_cluster_v2(mapa_shared(&xr[s], k), r);
            }
          }
        }
      }
    }
    end_sync();  // every worker of the cluster has finished its adds to pend
    if (lane == 0 && p.comm_passes != nullptr) atomicAdd(p.comm_passes, passes);
    for (int s = (int)crank + (int)csize * lane; s < H; s += (int)csize * 32) {
      const int64_t v = FULL ? s : p.hot_id[s];
      double2* gp = p.xa + v * p.S;
      double dx = 0.0, dy = 0.0;
      for (unsigned k = 0; k < csize; ++k) {
        const unsigned a = mapa_shared(&pend[s], k);
        dx += ld_cluster_f64(a);
        dy += ld_cluster_f64(a + 8);
      }
      if (dx != 0.0) red_add(&gp->x, dx);
      if (dy != 0.0) red_add(&gp->y, dy);
    }
    end_sync();  // no block exits while another may still read its pend
    return;
  }

  // ---------------- workers
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (unsigned)(lane & ~(G - 1)));
  const int grp = threadIdx.x / G;
  const int64_t w = (int64_t)blockIdx.x * nwb + grp;
  using SM = CombSmem<G, NR, FULL>;
  constexpr int KS = SM::KS;
  unsigned char* gbase = stage_base + (size_t)grp * SM::bytes(p.overflow);
  double* qs = reinterpret_cast<double*>(gbase + SM::ring_off + SM::ring_bytes);
  int64_t* ring = reinterpret_cast<int64_t*>(gbase + SM::ring_off);  // slot k: ring[4k..4k+2]
  const uint64_t tend = p.t0 + p.T;
  const uint64_t W = (uint64_t)p.workers;
  const uint64_t t_first = p.t0 + (uint64_t)w;
  uint64_t t = t_first;
  const bool active = w < p.workers && t < tend;
  {
    // Pipeline over this worker's samples m = 0, 1, ... (t = t_first + mW), all of it
    // read-only data, so fetching early changes nothing but latency:
    //   the row (+ alpha_i) of sample m + KS is copied at iteration m (KS stages),
    //   the bounds {lo, hi} (+ i) of sample m + 2KS are copied at iteration m (ring).
    // One cp.async group per iteration; wait_group<KS-1> at iteration m completes the
    // group of iteration m - KS, which holds the row of m and the bounds of m + KS.
    // (A register queue of bounds made the loop wait on the newest rowptr load.)
    // Sample indices come in batches of G: lane j draws sample mb + j (one Philox per
    // lane per G samples instead of one per sample), shuffled out in order.
    int64_t bi = 0;
    auto draw_batch = [&](uint64_t mb) {
      const uint64_t ts = t_first + (mb + (uint64_t)g) * W;
      bi = ts < tend ? sample_row(p.seed, ts, p.n) : 0;
    };
    auto sample_of = [&](uint64_t ms) -> int64_t {  // group-uniform call; batch of ms drawn
      return __shfl_sync(gmask, bi, (int)(ms & (uint64_t)(G - 1)), G);
    };
    static_assert(G >= 2 * KS, "a batch covers the prologue's samples");
    auto fetch_bounds = [&](uint64_t m, int slot_k) {
      const uint64_t ts = t_first + m * W;
      const int64_t is = sample_of(m);
      if (g == 0 && ts < tend) {
        int64_t* slot = ring + 4 * slot_k;
        slot[2] = is;
        cp_async8(slot, p.rowptr + is);
        cp_async8(slot + 1, p.rowptr + is + 1);
      }
    };
    if (active) {
      // prologue: rows of samples 0..KS-1 (their bounds loaded together: one round trip),
      // bounds of KS..2KS-1
      draw_batch(0);
      int64_t pis[KS], plo[KS], phi[KS];
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        pis[k] = sample_of((uint64_t)k);
        const bool in = t_first + (uint64_t)k * W < tend;
        plo[k] = in ? __ldg(&p.rowptr[pis[k]]) : 0;
        phi[k] = in ? __ldg(&p.rowptr[pis[k] + 1]) : 0;
      }
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        fetch_bounds((uint64_t)(k + KS), k + KS);
        if (t_first + (uint64_t)k * W < tend) {
          if (g == 0) { ring[4 * k] = plo[k]; ring[4 * k + 1] = phi[k]; ring[4 * k + 2] = pis[k]; }
          issue_row_copy_c<G, NR, FULL>(gbase, k, p.cols, p.eslot, p.vals, p.dv, p.alpha + pis[k], p.y + pis[k], plo[k],
                                        phi[k], g);
        } else {
          cp_async_commit();
        }
      }
    }
    init_slots();
    start_sync();
    if (active) {
    unsigned long long ov_sum = 0, ov_cnt = 0, ov_max = 0;
    unsigned long long shash = 0;
    int ov_local = 0, ov_iter = 0;
    int stage = 0, rs = 0;  // row stage and bounds-ring slot of sample m
    // this worker's samples: t_first + mW < tend  (32-bit counts from here on)
    const int nsamp = (int)((tend - t_first + W - 1) / W);
    for (int m = 0;; ++m) {
      bool ov_meas = false;
    if (p.ov != nullptr) ov_meas = (ov_iter++ % p.ov_every) == 0;
      unsigned long long ov_c0 = 0;
      if (ov_meas) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(ov_c0) : "l"(p.ov));
      cp_async_wait_group<KS - 1>();  // this sample's stage (and bounds of m + KS) landed
      __syncwarp(gmask);             // lane 0 copied alpha_i and the bounds
      const int64_t* cur = ring + 4 * rs;
      const int64_t lo = cur[0], hi = cur[1], i = cur[2];
      const int len = (int)(hi - lo);
      const double* sv = reinterpret_cast<const double*>(gbase + stage * SM::stage_bytes);
      const double* sd = sv + P;  // !FULL only
      const int32_t* sc = reinterpret_cast<const int32_t*>(sv + (FULL ? P : 2 * P));
      const int32_t* ss = sc + P;
      const double ai = *reinterpret_cast<const double*>(gbase + stage * SM::stage_bytes + SM::alpha_off);
      const double yb = *reinterpret_cast<const double*>(gbase + stage * SM::stage_bytes + SM::alpha_off + 8);
      double2 xb[NR];
      double qq[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;  // group-uniform
        if (j * G + g < len) {
          const int c = sc[j * G + g];
          const int s = FULL ? c : (H > 0 ? ss[j * G + g] : -1);
          xb[j] = s >= 0 ? lds_vol2(xr + s) : ld_na2(p.xa + (int64_t)c * p.S);
        }
      }
      double dot = 0.0;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;  // group-uniform
        if (j * G + g < len) {
          dot = fma(sv[j * G + g], xb[j].x, dot);
          // hot slot: the replica's second word is already D (abar + lambda x)
          qq[j] = FULL || (H > 0 && ss[j * G + g] >= 0) ? xb[j].y
                                                        : sd[j * G + g] * fma(p.lambda_, xb[j].x, xb[j].y);
        }
      }
      if (len > P)  // group-uniform: long rows only
      for (int kk = P + g; kk < len; kk += G) {
        const int64_t k = lo + kk;
        const int c = ld_nc_i32(p.cols + k);
        const int s = FULL ? c : (H > 0 ? ld_nc_i32(p.eslot + k) : -1);
        const double2 v = s >= 0 ? lds_vol2(xr + s) : ld_na2(p.xa + (int64_t)c * p.S);
        dot = fma(ld_nc_f64(p.vals + k), v.x, dot);
        qs[kk - P] = s >= 0 ? v.y : ld_nc_f64(p.dv + k) * fma(p.lambda_, v.x, v.y);
      }
      dot = group_sum<G>(dot, gmask) * yb;  // folded margin (exact: b = +-1)
      const double da = sigma_folded(dot) - ai;  // sigma~ = -1/(1+exp(m))
      const double db = da * yb;  // dalpha a~_k = (dalpha b_i) a_k, exact
      const double ngam = -p.gamma;
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len) break;  // group-uniform
        if (j * G + g < len) {
          const int c = sc[j * G + g];
          const int s = FULL ? c : (H > 0 ? ss[j * G + g] : -1);
          const double a = sv[j * G + g];
          double dx = ngam * fma(db, a, qq[j]);
          double dy = p.frozen ? 0.0 : db * a * p.inv_n;
          if (s >= 0 && !p.wt) {
            // groups of this warp that add to the same hot slot in this chunk merge their
            // adds first (xor partners; only lanes converged here take part)
            bool mine = true;
            if (G < 32) {
              const unsigned am = __activemask();
#pragma unroll
              for (int off = G; off < 32; off <<= 1) {
                const int ps = __shfl_xor_sync(am, mine ? s : -1, off);
                const double px = __shfl_xor_sync(am, dx, off), py = __shfl_xor_sync(am, dy, off);
                if (((am >> (lane ^ off)) & 1u) && mine && ps == s) {
                  if (lane & off) mine = false;
                  else { dx += px; dy += py; }
                }
              }
            }
            // (atomicAdd on shared f64 compiles to the ATOMS.CAST.SPIN loop; a hand-written
            // interleaved CAS pair measured 3x slower)
            if (mine) {
              atomicAdd(&pend[s].x, dx);
              if (dy != 0.0) atomicAdd(&pend[s].y, dy);
            }
          } else {
            double* xv = &p.xa[(int64_t)c * p.S].x;
            red_add(xv, dx);
            if (!p.frozen) red_add(xv + 1, db * a * p.inv_n);
          }
        }
      }
      if (len > P)  // group-uniform: long rows only
      for (int kk = P + g; kk < len; kk += G) {
        const int64_t k = lo + kk;
        const int c = ld_nc_i32(p.cols + k);
        const int s = FULL ? c : (H > 0 ? ld_nc_i32(p.eslot + k) : -1);
        const double a = ld_nc_f64(p.vals + k);
        const double dx = ngam * fma(db, a, qs[kk - P]);
        if (s >= 0 && !p.wt) {
          atomicAdd(&pend[s].x, dx);
          if (!p.frozen) atomicAdd(&pend[s].y, db * a * p.inv_n);
        } else {
          double* xv = &p.xa[(int64_t)c * p.S].x;
          red_add(xv, dx);
          if (!p.frozen) red_add(xv + 1, db * a * p.inv_n);
        }
      }
      if (g == 0) {
        if (!p.frozen) red_add(p.alpha + i, da);
        if (p.visits) {
          atomicAdd(p.visits + i, 1);
          shash += sample_mix(t, i);
        }
        if (p.ov != nullptr) {
          if (++ov_local == 100) {
            atomicAdd(p.ov, 100ull);
            ov_local = 0;
          }
          if (ov_meas) {
            unsigned long long c1;
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c1) : "l"(p.ov));
            const unsigned long long o = c1 - ov_c0;
            ov_sum += o;
            ov_cnt += 1;
            ov_max = max(ov_max, o);
          }
        }
      }
      if (m + 1 >= nsamp) break;
      // advance: this stage is free (every lane is past its reads of it); refill it with
      // the row of sample m + KS (bounds in the ring) and fetch the bounds of m + 2KS
      __syncwarp(gmask);
      const int mf = m + KS;
      const int rf = rs + KS >= SM::NB ? rs + KS - SM::NB : rs + KS;  // slot of m + KS
      if (((mf + KS) & (G - 1)) == 0) draw_batch((uint64_t)(mf + KS));
      if (mf < nsamp) {
        const int64_t* nb = ring + 4 * rf;
        const int64_t nlo = nb[0], nhi = nb[1], ni = nb[2];
        fetch_bounds((uint64_t)(mf + KS), rs);  // slot of m + 2KS == slot of m
        issue_row_copy_c<G, NR, FULL>(gbase, stage, p.cols, p.eslot, p.vals, p.dv, p.alpha + ni, p.y + ni,
                                      nlo, nhi, g);
      } else {
        cp_async_commit();
      }
      t += W;
      stage = (stage + 1 == KS) ? 0 : stage + 1;
      rs = (rs + 1 == SM::NB) ? 0 : rs + 1;
    }
    cp_async_wait_all();
    if (p.visits && g == 0) atomicAdd(p.shash, shash);
    if (p.ov != nullptr && g == 0 && ov_cnt > 0) {
      atomicAdd(p.ov + 1, ov_sum);
      atomicAdd(p.ov + 2, ov_cnt);
      atomicMax(p.ov + 3, ov_max);
    }
    }  // active
  }
  __syncwarp(gmask);
  if (g == 0) {
    if (solo) atomicAdd(&done, 1);
    else atomic_add_cluster_s32(done0, 1);
  }
  end_sync();  // matches the comm warps': they then flush pend
  end_sync();
}

// ---------------------------------------------------------------------------
// A9: objective / gradient (Section 4.1).  Deterministic: fixed grid, fixed
// per-group row order, fixed-order block partials.
// Per row: m_i = a~_i . x, loss_i = softplus(-m_i) = log(1+exp(-b_i a_i.x)),
// sigma~_i = -1/(1+exp(m_i)) (so sigma_i a_i = sigma~_i a~_i).
// A9 block partials in a fixed order: block_out[b] = this block's loss sum and
// block_out[gridDim.x + b] = its share of ||x||^2 (x strided over the whole grid).
// A9 finish, fused into the margin kernels: the last block to finish (ticket in ctr, reset
// by that block) sums the block partials in a fixed order -- f is deterministic.
struct ObjFinish {
  int* ctr;
  int64_t n;
  double lambda_;
  double* f_out;     // f = loss / n + lambda/2 ||x||^2 (nullable)
  double* loss_out;  // sum of the losses (nullable)
};

__device__ __forceinline__ void block_partials(double acc, const double* __restrict__ x, int xs, int64_t d,
                                               double* __restrict__ block_out, double* wl, double* wq,
                                               const ObjFinish& fin) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double sq = 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d; v += (int64_t)gridDim.x * blockDim.x)
    sq = fma(x[(int64_t)xs * v], x[(int64_t)xs * v], sq);
  acc = group_sum<32>(acc, 0xffffffffu);
  sq = group_sum<32>(sq, 0xffffffffu);
  if (lane == 0) {
    wl[wib] = acc;
    wq[wib] = sq;
  }
  __syncthreads();
  __shared__ int is_last;
  if (threadIdx.x == 0) {
    double s = 0.0, q = 0.0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) {
      s += wl[j];
      q += wq[j];
    }
    block_out[blockIdx.x] = s;
    block_out[gridDim.x + blockIdx.x] = q;
    __threadfence();
    is_last = atomicAdd(fin.ctr, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  __shared__ double s_loss[256], s_sq[256];
  const int nb = (int)gridDim.x;
  double a = 0.0, b = 0.0;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    a += __ldcg(block_out + j);
    b += __ldcg(block_out + nb + j);
  }
  s_loss[threadIdx.x] = a;
  s_sq[threadIdx.x] = b;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      s_loss[threadIdx.x] += s_loss[threadIdx.x + off];
      s_sq[threadIdx.x] += s_sq[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (fin.f_out) *fin.f_out = s_loss[0] / (double)fin.n + 0.5 * fin.lambda_ * s_sq[0];
    if (fin.loss_out) *fin.loss_out = s_loss[0];
    *fin.ctr = 0;  // ready for the next evaluation
  }
}

// A9 margins for short rows (mean <= 16): one thread per row (see ingest_thread_kernel).
__global__ void __launch_bounds__(256)
margin_thread_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                     const double* __restrict__ vals, const double* __restrict__ y,
                     const double* __restrict__ x, int xs, int64_t n,
                     double* __restrict__ sig, double* __restrict__ block_out, int64_t d, ObjFinish fin) {
  __shared__ double wl[8], wq[8];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = rowptr[i], hi = rowptr[i + 1];
    double m = 0.0;
#pragma unroll 4
    for (int64_t k = lo; k < hi; ++k) m = fma(vals[k], __ldg(x + (int64_t)xs * cols[k]), m);
    m *= y[i];  // folded margin b_i a_i . x (exact: b = +-1)
    // softplus(-m) = max(-m, 0) + log1p(exp(-|m|))
    acc += fmax(-m, 0.0) + log1p(exp(-fabs(m)));
    if (sig != nullptr) sig[i] = -1.0 / (1.0 + exp(m));
  }
  block_partials(acc, x, xs, d, block_out, wl, wq, fin);
}

// A9 margins over row tiles (see "Row tiles" above): m_i = b_i a_i . x per row by a
// segmented warp reduction, then loss_i = softplus(-m_i), sigma~_i.
__global__ void __launch_bounds__(256)
margin_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
              const double* __restrict__ vals, const double* __restrict__ y,
              const double* __restrict__ x, int xs, int64_t n,
              double* __restrict__ sig, double* __restrict__ block_loss, int64_t d, ObjFinish fin) {
  __shared__ double rsum[8][32];
  __shared__ double wl[8], wq[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  double acc = 0.0;
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; tile * 32 < n; tile += nwarps) {
    const int64_t r0 = tile * 32;
    const int nr = (int)((n - r0) < 32 ? (n - r0) : 32);
    const bool row = lane < nr;
    const int64_t lo = row ? rowptr[r0 + lane] : 0;
    const int64_t base = __shfl_sync(0xffffffffu, lo, 0);
    const int64_t end = rowptr[r0 + nr];
    const int rel = (int)((row ? lo : end) - base);
    rsum[wib][lane] = 0.0;
    __syncwarp();
#pragma unroll 4
    for (int64_t e0 = base; e0 < end; e0 += 32) {
      const int64_t e = e0 + lane;
      const bool in = e < end;
      const double prod = in ? vals[e] * __ldg(x + (int64_t)xs * cols[e]) : 0.0;
      const int j = tile_row_of((int)(e - base), rel, nr);
      bool head;
      const double sm = seg_sum_head(prod, in ? j : 32 + lane, &head);
      if (in && head) rsum[wib][j] += sm;
    }
    __syncwarp();
    if (row) {
      const double mu = rsum[wib][lane] * y[r0 + lane];  // folded margin
      // softplus(-m) = max(-m, 0) + log1p(exp(-|m|))
      acc += fmax(-mu, 0.0) + log1p(exp(-fabs(mu)));
      if (sig != nullptr) sig[r0 + lane] = -1.0 / (1.0 + exp(mu));
    }
    __syncwarp();
  }
  block_partials(acc, x, xs, d, block_loss, wl, wq, fin);
}

// A9 margins for short rows (mean <= 32): G lanes per row, a warp streams U batches of
// 32/G CONSECUTIVE rows (coalesced), the first chunk of every row issued before any
// reduction.  Per row it costs a few warp instructions instead of the tile kernel's
// per-chunk binary search and segmented reduction.
template <int G, int U>
__global__ void __launch_bounds__(256)
margin_rows_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                   const double* __restrict__ vals, const double* __restrict__ y,
                   const double* __restrict__ x, int xs, int64_t n,
                   double* __restrict__ sig, double* __restrict__ block_loss, int64_t d, ObjFinish fin) {
  constexpr int RG = 32 / G, RPW = RG * U;  // rows per warp batch / per warp iteration
  __shared__ double wl[8], wq[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int q = lane / G, g = lane & (G - 1);
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (unsigned)(lane & ~(G - 1)));
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  double acc = 0.0;
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; tile * RPW < n; tile += nwarps) {
    const int64_t r0 = tile * RPW;
    int64_t lo[U], hi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = r0 + u * RG + q;
      lo[u] = i < n ? rowptr[i] : 0;
      hi[u] = i < n ? rowptr[i + 1] : 0;
    }
    double m[U];
    if (G == 32) {
      // long rows: the first C chunks of all U rows are loaded before any use (U x C
      // column loads, then U x C gathers of x in flight per lane; one row's chunks at a time
      // left the warp waiting on its gathers: c4 1.55 ms)
      constexpr int C = 4;
      int c[U][C];
      double a[U][C], xv[U][C];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < C; ++j) {
          const int64_t k = lo[u] + j * G + g;
          c[u][j] = k < hi[u] ? __ldcs(cols + k) : -1;
          a[u][j] = k < hi[u] ? __ldcs(vals + k) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < C; ++j) xv[u][j] = c[u][j] >= 0 ? __ldg(x + (int64_t)xs * c[u][j]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        m[u] = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) m[u] = fma(a[u][j], xv[u][j], m[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll 4
        for (int64_t k = lo[u] + C * G + g; k < hi[u]; k += G) m[u] = fma(vals[k], __ldg(x + (int64_t)xs * cols[k]), m[u]);
      }
    } else {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = lo[u] + g;
      m[u] = k < hi[u] ? vals[k] * __ldg(x + (int64_t)xs * cols[k]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll 4
      for (int64_t k = lo[u] + G + g; k < hi[u]; k += G) m[u] = fma(vals[k], __ldg(x + (int64_t)xs * cols[k]), m[u]);
    }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = r0 + u * RG + q;
      const double mu = group_sum<G>(m[u], gmask) * (i < n ? y[i] : 1.0);  // folded margin
      if (i < n && g == 0) {
        // softplus(-m) = max(-m, 0) + log1p(exp(-|m|))
        acc += fmax(-mu, 0.0) + log1p(exp(-fabs(mu)));
        if (sig != nullptr) sig[i] = -1.0 / (1.0 + exp(mu));
      }
    }
  }
  block_partials(acc, x, xs, d, block_loss, wl, wq, fin);
}

// CSC segments: segment s covers csc entries [seg_lo[s], seg_hi[s]) of one column.
__global__ void __launch_bounds__(256)
colseg_kernel(const int64_t* __restrict__ seg_lo, const int64_t* __restrict__ seg_hi,
              int64_t nseg, const int32_t* __restrict__ csc_rows,
              const double* __restrict__ csc_vals, const double* __restrict__ sig,
              double* __restrict__ seg_sum) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nseg;
       s += warps) {
    const int64_t lo = seg_lo[s], hi = seg_hi[s];
    double acc = 0.0;
    for (int64_t k = lo + lane; k < hi; k += 32) acc = fma(__ldg(sig + csc_rows[k]), csc_vals[k], acc);
    acc = group_sum<32>(acc, 0xffffffffu);
    if (lane == 0) seg_sum[s] = acc;
  }
}

// g_v = scale * (sum of v's segments, in order) + lambda x_v.
__global__ void colsum_kernel(const int64_t* __restrict__ seg_ptr,
                              const double* __restrict__ seg_sum, const double* __restrict__ x,
                              int xs, int64_t d, double inv_scale_div, double lambda_,
                              double* __restrict__ g, int divide) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t j = seg_ptr[v]; j < seg_ptr[v + 1]; ++j) s += seg_sum[j];
    g[v] = divide ? s / inv_scale_div + lambda_ * x[xs * v] : s;
  }
}

// CSC construction helpers (init-time, lazily on the first gradient call).
__global__ void row_of_kernel(const int64_t* __restrict__ rowptr, int64_t n,
                              int32_t* __restrict__ row_of) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += warps)
    for (int64_t k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) row_of[k] = (int32_t)i;
}

__global__ void iota_kernel(int64_t* __restrict__ out, int64_t m) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = k;
}

__global__ void csc_gather_kernel(const int64_t* __restrict__ perm,
                                  const int32_t* __restrict__ row_of,
                                  const double* __restrict__ vals, const double* __restrict__ y, int64_t m,
                                  int32_t* __restrict__ csc_rows, double* __restrict__ csc_vals) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = perm[k];
    const int32_t r = row_of[j];
    csc_rows[k] = r;
    csc_vals[k] = vals[j] * y[r];  // folded a~ = b a (exact)
  }
}

// seg_cnt[v] = ceil(n_v / SEG)
__global__ void segcount_kernel(const int32_t* __restrict__ counts, int64_t d, int seg,
                                int64_t* __restrict__ seg_cnt) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x)
    seg_cnt[v] = ((int64_t)counts[v] + seg - 1) / seg;
}

__global__ void segfill_kernel(const int64_t* __restrict__ colptr,
                               const int64_t* __restrict__ seg_ptr, int64_t d, int seg,
                               int64_t* __restrict__ seg_lo, int64_t* __restrict__ seg_hi) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c0 = colptr[v], c1 = colptr[v + 1];
    int64_t s = seg_ptr[v];
    for (int64_t a = c0; a < c1; a += seg, ++s) {
      seg_lo[s] = a;
      seg_hi[s] = min(a + (int64_t)seg, c1);
    }
  }
}

// K5 divergence guard: flag if any x_v is not finite.
__global__ void nonfinite_kernel(const double2* __restrict__ xa, int S, int64_t d, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(xa[v * S].x);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void sample_kernel(uint64_t seed, uint64_t t0, uint64_t count, uint64_t n,
                              int64_t* __restrict__ out) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x)
    out[k] = sample_row(seed, t0 + k, n);
}

// State conversions between the paper's alpha and the folded alpha~ = b alpha.
__global__ void fold_alpha_kernel(const double* __restrict__ in, const double* __restrict__ y,
                                  double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = y[i] * in[i];
}

// abar_v lives in habar[v] for hot-split features (D_v <= hot_dmax), else in xa[v*S].y
__global__ void unpack_xa_kernel(const double2* __restrict__ xa, int S, const double* __restrict__ habar,
                                 const double* __restrict__ D, double hot_dmax,
                                 double* __restrict__ x, double* __restrict__ ab, int64_t d) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (x) x[v] = xa[v * S].x;
    if (ab) ab[v] = (hot_dmax > 0.0 && D[v] <= hot_dmax) ? habar[v] : xa[v * S].y;
  }
}

// writes abar to both homes (the pair slot and habar): correct whatever the split
__global__ void pack_xa_kernel(double2* __restrict__ xa, int S, double* __restrict__ habar,
                               const double* __restrict__ x, const double* __restrict__ ab, int64_t d) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < d;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (x) xa[v * S].x = x[v];
    if (ab) {
      xa[v * S].y = ab[v];
      habar[v] = ab[v];
    }
  }
}

}  // namespace asaga
