// asaga.cu -- the C-ABI of include/asaga.h: context, ingest, launch logic.
//
// Every step of the hot path runs in the kernels of asaga_kernels.cuh; this
// file only validates arguments, owns device memory, picks launch shapes and
// moves results across the host/device boundary.  The one library primitive
// used is CUB's radix sort + scan, at init time only, to build the
// column-major copy the deterministic gradient pass reads.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <map>
#include <mutex>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/asaga.h"
#include "asaga_kernels.cuh"
#include "asaga_pipe.cuh"

using namespace asaga;

namespace {

constexpr int kBlock = 256;
constexpr int kColSeg = 2048;         // CSC entries per gradient segment
constexpr int64_t kSmemHistMax = 48 * 1024;  // columns held in a shared histogram
constexpr int64_t kSelfInitMaxD = 1024;      // the ingest initialises itself (no init launch)
constexpr int kIngestHashLogRows = 14;        // rows-mode ingest: 16K-slot hash cache (128 KiB)

thread_local std::string g_thread_err = "no error";

}  // namespace

struct asaga_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sms = 148;
  int64_t n = 0, d = 0, nnz = 0;
  double lambda = 0, gamma = 0, L = 0;
  int64_t delta_r = 0, max_row = 0;
  uint64_t t = 0;
  int deterministic = 0, atomic_mode = 1, record = 0;
  int64_t concurrency_opt = 0;
  int lanes_opt = 0;
  // device data.  The matrix the kernels read is never copied on the device: the caller's
  // device arrays (borrowed by asaga_init_device / asaga_reload_device*: they must outlive
  // their use) or the context's own copies of host arrays (own_*, allocated on first use).
  // Values are the caller's a_ik; the label b_i is applied per sample / row (exact).
  const int64_t* rowptr = nullptr;
  const int32_t* cols = nullptr;
  const double* vals = nullptr;
  const double* y = nullptr;
  int64_t* own_rowptr = nullptr;
  int32_t* own_cols = nullptr;
  double* own_vals = nullptr;
  double* own_y = nullptr;
  // asaga_reload_async (host arrays): two device copies used in turn, filled on copy_stream
  // while the compute stream still works on the other one
  struct HostSet {
    int64_t* rowptr = nullptr;
    int32_t* cols = nullptr;
    double* vals = nullptr;
    double* y = nullptr;
    cudaEvent_t copied = nullptr;  // H2D into this set done (copy stream)
    cudaEvent_t free = nullptr;    // the compute stream's last use of this set done
    bool used = false;
  } hs[2];
  int hs_next = 0;
  cudaStream_t copy_stream = nullptr;
  double2* xa = nullptr;   // {x_v, abar_v} pairs at xa[v * S]
  int S = 1;               // pair stride
  double bulk_dmax = 0.0;  // hybrid scatter threshold on D_c (MODE 2)
  double hot_dmax = 0.0;   // hot split threshold on D_c (abar in habar)
  int replica_every = 0;   // > 0: shared-memory replica of {x, abar} (small d, async)
  double comb_freq = 0.0;  // > 0: CTA-level combining of features with p_v >= comb_freq
  double hot_freq = 0.0;   // > 0: the ingest computes the hot set p_v >= hot_freq (slot_of, hot_id):
                           // comb_freq when combining, pipe_freq with pipe_merge
  int pipe_merge = 0;      // > 0: asaga_pipe_kernel<CMB>, hot adds merged per block, flushed every this many ns
  int comb_H = 0;          // ... the number of such (hot) features after ingest
  int32_t* slot_of = nullptr;  // d: slot of a hot feature, -1 if cold
  int32_t* hot_id = nullptr;   // kCombMaxH: slot -> feature
  int32_t* eslot = nullptr;    // nnz: slot_of[cols[k]] (allocated when 0 < comb_H < d)
  int comb_nwb = 0;            // worker groups per block of the combine kernel
  int comb_csize = 1;          // blocks per cluster of the combine kernel
  int comb_cluster_opt = 0;    // requested cluster size (0 = 1)
  int comb_max_blocks = 0;     // cap on the combine kernel's blocks (0 = resident capacity)
  int l2_persist = 0;          // plain kernel: L2 access-policy window (persisting) over xa
  double pipe_freq = 0.0;      // > 0: asaga_pipe_kernel, features with p_v >= it read late
  int row_copy_elementwise = 0;  // plain kernel: per-element cp.async row staging (no TMA bulk)
  int scatter_unpaired = 0;      // plain kernel: one reduction instruction per word (no pairing)
  int d_gather = 0;              // plain kernel: D_c gathered per entry (no dv stream)
  int rec_layout = 0;            // plain kernel: the record layout (D from the coordinate record, no dv stream)
  int32_t* hot_tab = nullptr;    // record layout + hot split: membership table of the hot-split features
  int hot_log = 0;               // ... log2 of its slots
  int comb_wt = 0;             // write-through (replica reads only)
  bool shape_valid = false;    // launch shape computed for shape_key
  int64_t row_cap = 0;         // longest row the launch shape holds (nr * lanes + overflow)
  unsigned long long* h_ing = nullptr;  // mapped pinned: ingest validation results (ERR_COUNT + 3)
  unsigned long long* h_ing_dev = nullptr;  // ... its device address
  cudaEvent_t ev_ing = nullptr;         // recorded after the ingest's readback copies
  bool ing_pending = false;             // an asynchronous reload awaits ingest_resolve
  // the arrays the kernels read passed validation (false from an ingest's enqueue until its
  // resolve succeeds): every entry point that launches a kernel on the matrix refuses to
  // run on rejected data (ASAGA_E_STATE) until a reload succeeds
  bool data_valid = false;
  bool dv_ready = false;                // dv (and eslot) expanded for the current matrix
  std::string reject_msg;               // why the last ingest was rejected
  cudaEvent_t ev_part = nullptr;        // asaga_partial_obj_grad: caller stream <-> ctx stream
  bool ing_fused = false;               // the last ingest launch ran A1's finish and the report
  long long shape_key[6] = {0, 0, 0, 0, 0, 0};
  int32_t* comb_flag = nullptr;  // d scratch: hot flags, then their exclusive scan
  int32_t* comb_excl = nullptr;
  void* cub_temp = nullptr;
  size_t cub_temp_bytes = 0;
  double* habar = nullptr; // abar of hot-split features
  double* D = nullptr;     // reweighting n / n_v
  double* dv = nullptr;    // D_{c_k} per stored entry
  double* alpha = nullptr;  // folded alpha~ = b alpha
  int32_t* counts = nullptr;
  int32_t* visits = nullptr;
  unsigned long long* shash = nullptr;  // record_samples: sum of mix(t, i_t)
  unsigned long long* ov = nullptr;  // overlap instrumentation (4 counters)
  int algorithm = ASAGA_ALG_ASAGA;
  bool snapshot_valid = false;       // KROMAGNON: alpha / abar hold a snapshot
  int ov_every = 0;
  // scratch
  double* sig = nullptr;
  double* block_loss = nullptr;
  double* scal = nullptr;  // [0] f, [1] loss sum
  int* flag = nullptr;
  unsigned long long* scratch = nullptr;
  double* tmp_n = nullptr;  // n doubles (state conversions)
  double* tmp_d = nullptr;  // d doubles
  double* tmp_d2 = nullptr; // d doubles
  double* xdense = nullptr; // d doubles: A9's dense copy of the current x (d > 4096)
  int obj_blocks = 0;
  bool margin_tiles = false;
  bool self_init_ready = false;    // small d: the ingest kernel resets its own scratch
  int32_t* ingest_part = nullptr;  // small d: per-block column counts (grid x d)
  int ingest_grid = 0;
  // CSC (built lazily)
  bool csc_built = false;
  int32_t* csc_rows = nullptr;
  double* csc_vals = nullptr;
  int64_t* seg_ptr = nullptr;
  int64_t* seg_lo = nullptr;
  int64_t* seg_hi = nullptr;
  double* seg_sum = nullptr;
  int64_t nseg = 0;
  // update-kernel launch shape
  int lanes = 32, nr = 1;
  int overflow = 0;
  size_t smem = 0;         // dynamic shared memory of a full (kBlock) block
  size_t group_bytes = 0;  // dynamic shared memory per group
  int grid = 1, block = kBlock;
  int max_tpb = kBlock;    // largest update-kernel block the shared memory allows
  int64_t workers = 1;
  int max_resident_groups = 1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  std::string err = "no error";
  std::vector<void*> allocs;
};

namespace {

asaga_status fail(asaga_ctx* ctx, asaga_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_thread_err = buf;
  return s;
}

#define CK(ctx, call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail((ctx), e_ == cudaErrorMemoryAllocation ? ASAGA_E_OOM : ASAGA_E_CUDA,    \
                  "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,       \
                  __LINE__);                                                              \
    }                                                                                     \
  } while (0)

template <typename T>
asaga_status dalloc(asaga_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess)
    return fail(ctx, e == cudaErrorMemoryAllocation ? ASAGA_E_OOM : ASAGA_E_CUDA,
                "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  ctx->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return ASAGA_OK;
}

template <typename T>
void dfree(asaga_ctx* ctx, T** p) {
  if (!*p) return;
  auto it = std::find(ctx->allocs.begin(), ctx->allocs.end(), (void*)*p);
  if (it != ctx->allocs.end()) ctx->allocs.erase(it);
  cudaFree(*p);
  *p = nullptr;
}

#define TRY(expr)                    \
  do {                               \
    asaga_status s_ = (expr);        \
    if (s_ != ASAGA_OK) return s_;   \
  } while (0)

// cudaFuncAttributeMaxDynamicSharedMemorySize, raised only when a launch needs more than was
// set before (per device and function, process-wide): the attribute call cost host time on
// every launch of the 0.1-epoch convergence loops
cudaError_t ensure_smem_attr(int device, const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(device, fn);
  const auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

int grid_for(const asaga_ctx* ctx, int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)ctx->sms * 8;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

using UpdFn = void (*)(UpdateParams);

template <int G, int NR, bool DET, bool REPL>
UpdFn pick_mode(int mode) {
  switch (mode) {
    case 0: return asaga_update_kernel<G, NR, DET, 0, REPL, false>;
    case 2: return asaga_update_kernel<G, NR, DET, 2, REPL, false>;
    default: return asaga_update_kernel<G, NR, DET, 1, REPL, false>;
  }
}

template <int G, int NR>
UpdFn pick_upd(bool det, int mode, bool repl, bool rec) {
  if (rec)  // record layout (MODE 1, no replica)
    return det ? asaga_update_kernel<G, NR, true, 1, false, true> : asaga_update_kernel<G, NR, false, 1, false, true>;
  if (det) return pick_mode<G, NR, true, false>(mode);  // deterministic mode reads L2 directly
  return repl ? pick_mode<G, NR, false, true>(mode) : pick_mode<G, NR, false, false>(mode);
}

template <int G>
UpdFn pick_upd_nr(int nr, bool det, int mode, bool repl, bool rec) {
  switch (nr) {
    case 1: return pick_upd<G, 1>(det, mode, repl, rec);
    case 2: return pick_upd<G, 2>(det, mode, repl, rec);
    case 4: return pick_upd<G, 4>(det, mode, repl, rec);
    default: return pick_upd<G, 8>(det, mode, repl, rec);
  }
}

// scatter mode: 0 non-atomic ablation, 1 LSU REDs, 2 TMA bulk pair reductions
int scatter_mode(const asaga_ctx* ctx);

bool use_replica(const asaga_ctx* ctx);
bool use_pipe(const asaga_ctx* ctx);
bool use_rec(const asaga_ctx* ctx);
UpdFn pipe_fn(const asaga_ctx* ctx, int lanes, int nr);

UpdFn update_fn(const asaga_ctx* ctx, int lanes, int nr) {
  if (use_pipe(ctx)) return pipe_fn(ctx, lanes, nr);
  const bool det = ctx->deterministic != 0;
  const int mode = scatter_mode(ctx);
  const bool repl = use_replica(ctx);
  const bool rec = use_rec(ctx);
  switch (lanes) {
    case 8: return pick_upd_nr<8>(nr, det, mode, repl, rec);
    case 16: return pick_upd_nr<16>(nr, det, mode, repl, rec);
    default: return pick_upd_nr<32>(nr, det, mode, repl, rec);
  }
}

constexpr int64_t kReplicaMaxD = 4096;  // 64 KiB of {x, abar} pairs per block
constexpr int kPipeMaxH = 512;          // pipe_merge: hot features in the per-block merge table
constexpr int kCombMaxH = 4096;         // hot features combined per block: 128 KiB of xr + pend

bool use_combine(const asaga_ctx* ctx) {
  // comb_H == 0 (no feature that popular): the same pipelined kernel, no communication warp
  return ctx->comb_freq > 0.0 && !ctx->deterministic && ctx->atomic_mode;
}

template <int G, int NR>
UpdFn pick_comb(bool full) {
  return full ? asaga_combine_kernel<G, NR, true> : asaga_combine_kernel<G, NR, false>;
}

template <int G>
UpdFn pick_comb_nr(int nr, bool full) {
  switch (nr) {
    case 1: return pick_comb<G, 1>(full);
    case 2: return pick_comb<G, 2>(full);
    case 4: return pick_comb<G, 4>(full);
    default: return pick_comb<G, 8>(full);
  }
}

UpdFn combine_fn(const asaga_ctx* ctx, int lanes, int nr) {
  const bool full = ctx->comb_H == ctx->d;
  switch (lanes) {
    case 8: return pick_comb_nr<8>(nr, full);
    case 16: return pick_comb_nr<16>(nr, full);
    default: return pick_comb_nr<32>(nr, full);
  }
}

size_t comb_group_bytes(const asaga_ctx* ctx) {  // CombSmem<G, NR, FULL>::bytes
  const bool full = ctx->comb_H == ctx->d;
  const size_t P = (size_t)ctx->nr * ctx->lanes;
  const size_t alpha_off = full ? P * (sizeof(double) + sizeof(int32_t)) : P * (2 * sizeof(double) + 2 * sizeof(int32_t));
  const size_t stage = (alpha_off + 2 * sizeof(double) + 15) & ~(size_t)15;  // + alpha_i, b_i
  // KS = 3 row stages + a bounds ring of 2 KS 32-byte slots + overflow q slots
  return (3 * stage + 6 * 32 + (size_t)ctx->overflow * sizeof(double) + 15) & ~(size_t)15;
}

size_t comb_smem(const asaga_ctx* ctx, int nwb) {  // xr, pend, D table, worker groups
  return (size_t)ctx->comb_H * (2 * 16 + 8) + (size_t)nwb * comb_group_bytes(ctx);
}

// Combine launch shape: blocks in clusters of C (C blocks share one set of hot-feature
// adds per pass, DSMEM); at most one block per SM and only as many clusters as can be
// resident at once (every block runs for the whole launch).  nwb = worker groups per block.
asaga_status comb_shape(asaga_ctx* ctx, int64_t workers, int* nwb, int* blocks, int* csize,
                        int64_t* workers_out) {
  const int kCombBlock = comb_block_threads(ctx->nr);  // launch bounds of the instance
  const int per_warp = 32 / ctx->lanes;
  int C = ctx->comb_cluster_opt > 0 ? ctx->comb_cluster_opt : 1;
  C = std::max(1, std::min(C, 8));
  int64_t groups_needed = workers;
  // resident clusters of C blocks (1 block per SM: launch bounds + large shared memory)
  UpdFn fn = combine_fn(ctx, ctx->lanes, ctx->nr);
  int cap_clusters = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C * ctx->sms);
    cfg.blockDim = dim3(kCombBlock);
    cfg.dynamicSmemBytes = 200 * 1024;  // forces one block per SM
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(ctx, ensure_smem_attr(ctx->device, (const void*)fn, 200 * 1024));
    CK(ctx, cudaOccupancyMaxActiveClusters(&cap_clusters, (const void*)fn, &cfg));
  }
  if (cap_clusters < 1) return fail(ctx, ASAGA_E_INVALID_ARG, "no cluster of %d blocks fits the device", C);
  int64_t cap_blocks = (int64_t)cap_clusters * C;
  if (ctx->comb_max_blocks > 0)
    cap_blocks = std::max<int64_t>(C, std::min<int64_t>(cap_blocks, ctx->comb_max_blocks / C * C));
  if (workers <= 0)  // auto: every resident block full of workers
    workers = cap_blocks * ((kCombBlock - 32) / ctx->lanes);
  // blocks: enough that every block has <= kCombBlock - 32 worker threads
  groups_needed = workers;
  int64_t b = std::min<int64_t>((groups_needed + per_warp - 1) / per_warp, cap_blocks);
  b = std::max<int64_t>(b, 1);
  int64_t w = (groups_needed + b - 1) / b;
  w = (w + per_warp - 1) / per_warp * per_warp;
  if (w * ctx->lanes > kCombBlock - 32)
    return fail(ctx, ASAGA_E_INVALID_ARG, "combine: %lld samples in flight need %lld worker threads per block "
                "(max %d with %lld resident blocks)", (long long)workers, (long long)(w * ctx->lanes),
                kCombBlock - 32, (long long)cap_blocks);
  b = (groups_needed + w - 1) / w;
  const int Ce = (int)std::min<int64_t>(C, b);
  b = (b + Ce - 1) / Ce * Ce;
  *nwb = (int)w;
  *blocks = (int)b;
  *csize = Ce;
  *workers_out = workers;
  return ASAGA_OK;
}

bool use_replica(const asaga_ctx* ctx) {
  return ctx->replica_every > 0 && !ctx->deterministic && ctx->d <= kReplicaMaxD;
}
// the pipelined kernel: ASAGA (not the frozen-memory methods), atomic adds, no overlap counter
bool use_pipe(const asaga_ctx* ctx) {
  return ctx->pipe_freq > 0.0 && ctx->atomic_mode && ctx->algorithm == ASAGA_ALG_ASAGA && ctx->ov == nullptr &&
         !use_combine(ctx);
}
template <int G, int NR>
UpdFn pick_pipe(bool det, bool cmb) {
  return det ? (cmb ? asaga_pipe_kernel<G, NR, true, true> : asaga_pipe_kernel<G, NR, true, false>)
             : (cmb ? asaga_pipe_kernel<G, NR, false, true> : asaga_pipe_kernel<G, NR, false, false>);
}
template <int G>
UpdFn pick_pipe_nr(int nr, bool det, bool cmb) {
  switch (nr) {
    case 1: return pick_pipe<G, 1>(det, cmb);
    case 2: return pick_pipe<G, 2>(det, cmb);
    case 4: return pick_pipe<G, 4>(det, cmb);
    default: return pick_pipe<G, 8>(det, cmb);
  }
}
bool use_merge(const asaga_ctx* ctx) {
  return use_pipe(ctx) && ctx->pipe_merge > 0 && ctx->comb_H > 0 && !ctx->deterministic;
}
UpdFn pipe_fn(const asaga_ctx* ctx, int lanes, int nr) {
  const bool det = ctx->deterministic != 0;
  const bool cmb = use_merge(ctx);
  switch (lanes) {
    case 8: return pick_pipe_nr<8>(nr, det, cmb);
    case 16: return pick_pipe_nr<16>(nr, det, cmb);
    default: return pick_pipe_nr<32>(nr, det, cmb);
  }
}
// pipe_merge: positions of the per-block merge table (power of two >= 2H, >= 4)
int merge_ts(const asaga_ctx* ctx) {
  int ts = 4;
  while (ts < 2 * ctx->comb_H) ts *= 2;
  return ts;
}
// its bytes for gpb worker groups: keys + home flags + per group a row of running sums and
// a row of sent sums (2 x {dx, dabar}) + the finished-groups count
size_t merge_bytes(const asaga_ctx* ctx, int gpb) {
  if (!use_merge(ctx)) return 0;
  const size_t ts = (size_t)merge_ts(ctx);
  return ts * 2 * sizeof(int32_t) + (size_t)gpb * 2 * ts * 2 * sizeof(double) + 16;
}

size_t replica_bytes(const asaga_ctx* ctx) {
  return use_replica(ctx) ? (((size_t)ctx->d * 16 + 15) & ~(size_t)15) : 0;
}

int scatter_mode(const asaga_ctx* ctx) {
  if (!ctx->atomic_mode) return 0;
  return ctx->bulk_dmax > 0.0 ? 2 : 1;
}

// The record layout (asaga_update_kernel<REC>): D_v read from the 32-byte coordinate record
// {x_v, abar_v, D_v, .} with the gather itself (no per-entry D stream, no expand pass).
// The plain kernel with REDs and no replica, S >= 2, and (hot split) a membership table.
bool use_rec(const asaga_ctx* ctx) {
  return ctx->rec_layout && !use_pipe(ctx) && !use_combine(ctx) && scatter_mode(ctx) == 1 && !use_replica(ctx) &&
         ctx->S >= 2 && (ctx->hot_dmax == 0.0 || ctx->hot_tab != nullptr);
}
// d_gather: the plain kernel (REDs, default layout, no hot split, no replica) gathers D_c from
// the d-vector with each entry's coordinate gather: no per-entry D stream, no expand pass.
bool use_dg(const asaga_ctx* ctx) {
  return ctx->d_gather && !ctx->rec_layout && !use_pipe(ctx) && !use_combine(ctx) && scatter_mode(ctx) == 1 &&
         !use_replica(ctx) && ctx->hot_dmax == 0.0;
}
size_t rec_tab_bytes(const asaga_ctx* ctx) {  // the kernel's shared copy of the table
  return ctx->hot_tab != nullptr ? (size_t)sizeof(int32_t) << ctx->hot_log : 0;
}
// shared memory ahead of the worker groups: the replica, or the record layout's table
// (reserved whenever the table exists: set_algorithm may switch the kernel later)
size_t pre_bytes(const asaga_ctx* ctx, bool launch) {
  return replica_bytes(ctx) + ((!launch || use_rec(ctx)) && ctx->rec_layout ? rec_tab_bytes(ctx) : 0);
}

// Spread `workers` groups over all SMs: the smallest power-of-two block (>= one
// warp, <= kBlock threads) that still gives every SM a block.  Workers packed
// onto few SMs queue behind each other's row copies and REDs in the SM's LSU
// (profiles/r01_update_kernel.md), so a low concurrency must not mean few SMs.
// The smallest power-of-two block that lets one block per SM hold every worker; then one
// block per SM (or per worker, below the SM count): the kernels deal worker groups to blocks
// round robin, so W workers spread over min(W, #SMs) SMs (packing them into full blocks left
// 36 of 148 SMs idle at c4's W = 448 in round 1).
void launch_shape(const asaga_ctx* ctx, int64_t workers, int* grid, int* block) {
  if (use_merge(ctx)) {  // gpb groups (whole warps) per block + the communication warp
    const int64_t per_warp = 32 / ctx->lanes;
    int64_t gpb = (workers + ctx->sms - 1) / ctx->sms;
    gpb = (gpb + per_warp - 1) / per_warp * per_warp;
    gpb = std::min<int64_t>(std::max<int64_t>(gpb, per_warp), ctx->max_tpb / ctx->lanes);
    *block = (int)(gpb * ctx->lanes + 32);
    *grid = (int)((workers + gpb - 1) / gpb);
    return;
  }
  const int64_t threads = workers * ctx->lanes;
  int64_t tpb = 32;
  while (tpb < ctx->max_tpb && tpb * ctx->sms < threads) tpb *= 2;
  *block = (int)tpb;
  const int64_t gpb = tpb / ctx->lanes;
  int64_t g = (workers + gpb - 1) / gpb;
  if (g < ctx->sms) g = std::min<int64_t>(ctx->sms, workers);
  *grid = (int)g;
}

// Pick lanes per sample and register chunks from the row-length profile, then
// the launch shape for the requested number of samples in flight.
asaga_status configure_update(asaga_ctx* ctx) {
  const double mean = ctx->n ? (double)ctx->nnz / (double)ctx->n : 1.0;
  int lanes = ctx->lanes_opt;
  if (lanes == 0) lanes = mean <= 8.0 ? 8 : (mean <= 16.0 ? 16 : 32);
  if (lanes != 8 && lanes != 16 && lanes != 32)
    return fail(ctx, ASAGA_E_INVALID_ARG, "lanes_per_sample must be 0, 8, 16 or 32 (got %d)", lanes);
  int nr = 1;
  // register chunks for about twice the mean row, but no more than the longest row needs
  while (nr < 8 && (double)(nr * lanes) < 2.0 * mean && (int64_t)nr * lanes < ctx->max_row) nr *= 2;
  if ((int64_t)nr * lanes < ctx->max_row && ctx->max_row <= (int64_t)2 * nr * lanes && nr < 8) nr *= 2;
  int overflow = (int)std::max<int64_t>(0, ctx->max_row - (int64_t)nr * lanes);
  overflow = (overflow + 1) & ~1;  // keep every group's smem block 16-byte aligned
  // a reload of data with the same launch-relevant profile keeps the launch shape (the
  // occupancy queries cost host time on every re-ingest otherwise)
  const long long key[6] = {lanes, nr, overflow, ctx->comb_H, (long long)ctx->concurrency_opt,
                            (long long)(use_combine(ctx) ? 1 : 0) + 2 * ctx->deterministic};
  if (ctx->shape_valid && std::memcmp(key, ctx->shape_key, sizeof(key)) == 0) return ASAGA_OK;
  ctx->shape_valid = false;
  ctx->lanes = lanes;
  ctx->nr = nr;
  ctx->overflow = overflow;
  ctx->row_cap = (int64_t)nr * lanes + overflow;
  // per group: 2 stages of nr*lanes row entries (int32 + fp64) + overflow q slots
  // (GroupSmem in asaga_kernels.cuh)
  // (GroupSmem: bulk-scatter source buffer + 2 row stages + overflow q slots)
  // GroupSmem in asaga_kernels.cuh: the bulk-scatter source buffer + 2 stages (values and
  // D with 2 slots of 16-B alignment slack, columns with 4, b_i + the stage's mbarrier) +
  // the overflow q slots
  const size_t P = (size_t)nr * lanes;
  size_t group_bytes = P * 2 * sizeof(double) +
                       2 * (2 * (P + 2) * sizeof(double) + (P + 4) * sizeof(int32_t) + 16) +
                       (size_t)ctx->overflow * sizeof(double);
  if (ctx->pipe_freq > 0.0)  // the pipelined kernel's 4 stages + bounds ring (PipeSmem); the
    // context may switch between it and the plain kernel (set_algorithm), so take the larger
    group_bytes = std::max(group_bytes, (size_t)4 * (((size_t)nr * lanes * (sizeof(int32_t) + 2 * sizeof(double)) +
                                                      16 + 15) & ~(size_t)15) +
                                            8 * 32 + (((size_t)ctx->overflow * sizeof(double) + 15) & ~(size_t)15));
  ctx->group_bytes = group_bytes;
  if (use_combine(ctx)) {
    int64_t workers = ctx->concurrency_opt > 0 ? ctx->concurrency_opt : 0;
    int nwb = 1, blocks = 1, csize = 1;
    TRY(comb_shape(ctx, workers, &nwb, &blocks, &csize, &workers));
    if (ctx->concurrency_opt <= 0)  // auto: as many workers as the shared memory allows
      while (nwb > 32 / lanes && comb_smem(ctx, nwb) > 226 * 1024) {
        workers = (int64_t)blocks * (nwb - 32 / lanes);
        TRY(comb_shape(ctx, workers, &nwb, &blocks, &csize, &workers));
      }
    ctx->smem = comb_smem(ctx, nwb);
    if (ctx->smem > 226 * 1024)
      return fail(ctx, ASAGA_E_INVALID_ARG,
                  "combine: %d hot features and %d workers per block need %zu B of shared memory "
                  "(raise combine_min_freq or lower the concurrency)", ctx->comb_H, nwb, ctx->smem);
    UpdFn cfn = combine_fn(ctx, lanes, nr);
    CK(ctx, ensure_smem_attr(ctx->device, (const void*)cfn, (int)ctx->smem));
    ctx->comb_nwb = nwb;
    ctx->comb_csize = csize;
    ctx->workers = workers;
    ctx->block = nwb * lanes + (ctx->comb_H > 0 ? 32 : 0);
    ctx->grid = blocks;
    ctx->max_resident_groups = (int)std::min<int64_t>(INT32_MAX, workers);
    std::memcpy(ctx->shape_key, key, sizeof(key));
    ctx->shape_valid = true;
    return ASAGA_OK;
  }
  // blocks of up to kBlock threads, fewer when long rows' overflow slots need the room
  // (pipe_merge: up to kBlock - 32 worker threads + the communication warp)
  const bool mg = use_merge(ctx);
  const int comm = mg ? 32 : 0;
  int tpb_max = kBlock - comm;
  while (tpb_max > 32 &&
         pre_bytes(ctx, false) + (size_t)(tpb_max / lanes) * group_bytes + merge_bytes(ctx, tpb_max / lanes) > 226 * 1024)
    tpb_max = mg ? tpb_max - 32 : tpb_max / 2;
  ctx->max_tpb = tpb_max;
  const int gpb = tpb_max / lanes;
  ctx->smem = pre_bytes(ctx, false) + (size_t)gpb * group_bytes + merge_bytes(ctx, gpb);
  UpdFn fn = update_fn(ctx, lanes, nr);
  if (ctx->smem > 226 * 1024)
    return fail(ctx, ASAGA_E_INVALID_ARG, "row of %lld entries too long for the update kernel",
                (long long)ctx->max_row);
  CK(ctx, ensure_smem_attr(ctx->device, (const void*)fn, (int)ctx->smem));
  int per_sm = 0;
  CK(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, tpb_max + comm, ctx->smem));
  per_sm = std::max(per_sm, 1);
  ctx->max_resident_groups = per_sm * ctx->sms * gpb;
  int64_t workers;
  if (ctx->deterministic) workers = 1;
  else if (ctx->concurrency_opt > 0) workers = std::min<int64_t>(ctx->concurrency_opt, ctx->max_resident_groups);
  else workers = ctx->max_resident_groups;
  ctx->workers = workers;
  launch_shape(ctx, workers, &ctx->grid, &ctx->block);
  std::memcpy(ctx->shape_key, key, sizeof(key));
  ctx->shape_valid = true;
  return ASAGA_OK;
}

// Device buffers of a context (sizes fixed by n, d, nnz).
asaga_status alloc_state(asaga_ctx* ctx) {
  const int64_t n = ctx->n, d = ctx->d, nnz = ctx->nnz;
  // Small d (every feature hot, e.g. c2's d = 54): give every feature its own
  // 1 KiB block so hot features spread over L2 slices (2.2x at 1024 in flight,
  // profiles/r01_update_kernel.md); larger d keeps pairs dense (S = 8 measured no gain on c3).
  // Larger d: dense 16-byte pairs, or 32-byte records {x_v, abar_v, D_v, .} (S = 2) for the
  // record layout.
  ctx->S = d <= 4096 ? 64 : (ctx->rec_layout ? 2 : 1);
#ifdef ASAGA_TIMING
  if (const char* e = getenv("ASAGA_PAIR_STRIDE")) ctx->S = std::max(1, atoi(e));  // experiments
#endif
  TRY(dalloc(ctx, &ctx->xa, (size_t)d * ctx->S));
  TRY(dalloc(ctx, &ctx->D, d));
  TRY(dalloc(ctx, &ctx->habar, d));
  // (dv, D per stored entry: allocated by the first expand -- the record layout needs none)
  if (ctx->hot_dmax > 0.0 && ctx->S >= 2 && ctx->rec_layout) {
    // hot-split table: the features with D_v <= hot_dmax number at most nnz/n x hot_dmax
    // (sum_v n_v = nnz) and at most d; >= 8 slots per such feature keep the linear probes short
    const double hmax = std::min((n > 0 ? (double)nnz / (double)n : 0.0) * ctx->hot_dmax, (double)d) + 8.0;
    int log = 8;
    while (log < 14 && (double)(1 << log) < 8.0 * hmax) ++log;
    if ((double)(1 << log) >= 8.0 * hmax) {  // else (> 16K slots): the dv stream carries the split
      TRY(dalloc(ctx, &ctx->hot_tab, (size_t)1 << log));
      ctx->hot_log = log;
    }
  }
  TRY(dalloc(ctx, &ctx->alpha, n));
  TRY(dalloc(ctx, &ctx->counts, d));
  TRY(dalloc(ctx, &ctx->tmp_n, n));
  TRY(dalloc(ctx, &ctx->tmp_d, d));
  TRY(dalloc(ctx, &ctx->tmp_d2, d));
  if (d > 4096) TRY(dalloc(ctx, &ctx->xdense, d));  // A9's dense copy of x
  {  // A9 grid: one full wave of the margin kernel picked by the mean row length (fixed per
     // context, so the block partials are summed in a fixed order: deterministic f)
    const double mean = n ? (double)nnz / (double)n : 1.0;
    ctx->margin_tiles = getenv("ASAGA_MARGIN_TILES") != nullptr;  // experiment: 32-row tiles for long rows
    const void* mfn = mean <= 16.0 ? (const void*)margin_thread_kernel
                      : mean <= 24.0 ? (const void*)margin_rows_kernel<8, 4>
                      : ctx->margin_tiles ? (const void*)margin_kernel : (const void*)margin_rows_kernel<32, 4>;
    int per_sm = 1;
    CK(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mfn, kBlock, 0));
    ctx->obj_blocks = ctx->sms * std::max(1, std::min(per_sm, 8));
  }
  TRY(dalloc(ctx, &ctx->block_loss, 2 * (size_t)ctx->obj_blocks));  // loss partials, ||x||^2 partials
  TRY(dalloc(ctx, &ctx->scal, 4));
  TRY(dalloc(ctx, &ctx->flag, 8));  // [0] non-finite, [1] max n_v, [2] hot count, [3] run guard, [4] ingest blocks, [5] objective blocks
  TRY(dalloc(ctx, &ctx->scratch, ERR_COUNT + 3));  // err rows, max ||a||^2, max row, comm passes
  if (ctx->record) {
    TRY(dalloc(ctx, &ctx->visits, n));
    TRY(dalloc(ctx, &ctx->shash, 1));
  }
  if (ctx->ov_every > 0) TRY(dalloc(ctx, &ctx->ov, 4));
  CK(ctx, cudaHostAlloc(&ctx->h_ing, sizeof(unsigned long long) * (ERR_COUNT + 3), cudaHostAllocMapped));
  CK(ctx, cudaHostGetDevicePointer(&ctx->h_ing_dev, ctx->h_ing, 0));
  CK(ctx, cudaEventCreateWithFlags(&ctx->ev_ing, cudaEventDisableTiming));
  if (ctx->hot_freq > 0.0) {
    TRY(dalloc(ctx, &ctx->slot_of, d));
    TRY(dalloc(ctx, &ctx->hot_id, kCombMaxH));
    TRY(dalloc(ctx, &ctx->comb_flag, d));
    TRY(dalloc(ctx, &ctx->comb_excl, d));
    if (ctx->comb_freq > 0.0) TRY(dalloc(ctx, &ctx->eslot, nnz));  // combine: written when some stay cold
    CK(ctx, cub::DeviceScan::ExclusiveSum(nullptr, ctx->cub_temp_bytes, ctx->comb_flag, ctx->comb_excl,
                                          (int)d, ctx->stream));
    unsigned char* tb = nullptr;
    TRY(dalloc(ctx, &tb, ctx->cub_temp_bytes));
    ctx->cub_temp = tb;
  }
  return ASAGA_OK;
}

// A0 + A1 on data already in device memory (the caller's device arrays, or the context's
// own copy of host arrays): read-only validation and column counts; from here on the
// kernels read these arrays.  Resets the state to x = 0, alpha = 0, abar = 0, t = 0
// (reading R1).
asaga_status ingest_enqueue(asaga_ctx* ctx, const int64_t* indptr_in, const int32_t* indices_in,
                            const double* data_in, const double* y_in, bool guard) {
  const int64_t n = ctx->n, d = ctx->d, nnz = ctx->nnz;
  unsigned long long* scratch = ctx->scratch;
  if (ctx->visits) CK(ctx, cudaMemsetAsync(ctx->visits, 0, sizeof(int32_t) * n, ctx->stream));
  if (ctx->shash) CK(ctx, cudaMemsetAsync(ctx->shash, 0, sizeof(unsigned long long), ctx->stream));
  if (ctx->ov) CK(ctx, cudaMemsetAsync(ctx->ov, 0, 4 * sizeof(unsigned long long), ctx->stream));
  // small d: the ingest kernel initialises itself (IngestParams::self_init) once the state
  // has been reset the first time; otherwise one init launch per ingest
  const bool self_init = d <= kSelfInitMaxD;
  if (!self_init || !ctx->self_init_ready) {
    ingest_init_kernel<<<grid_for(ctx, std::max(n, d), kBlock), kBlock, 0, ctx->stream>>>(
        ctx->counts, d, ctx->alpha, n, scratch, ctx->flag);
    CK(ctx, cudaGetLastError());
    ctx->self_init_ready = self_init;
  }
  ctx->t = 0;
  ctx->snapshot_valid = false;
  ctx->data_valid = false;
  ctx->dv_ready = false;
  if (ctx->csc_built) {  // a new matrix invalidates the column-major copy
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    dfree(ctx, &ctx->csc_rows);
    dfree(ctx, &ctx->csc_vals);
    dfree(ctx, &ctx->seg_ptr);
    dfree(ctx, &ctx->seg_lo);
    dfree(ctx, &ctx->seg_hi);
    dfree(ctx, &ctx->seg_sum);
    dfree(ctx, &ctx->sig);
    ctx->csc_built = false;
  }

  IngestParams ip;
  ip.indptr = indptr_in;
  ip.indices = indices_in;
  ip.data = data_in;
  ip.y = y_in;
  // from here on the kernels read these arrays (no device-side copy)
  ctx->rowptr = indptr_in;
  ctx->cols = indices_in;
  ctx->vals = data_in;
  ctx->y = y_in;
  ip.counts = ctx->counts;
  ip.err_row = scratch;
  ip.max_sq = scratch + ERR_COUNT;
  ip.max_len = scratch + ERR_COUNT + 1;
  ip.n = n;
  ip.d = d;
  ip.nnz = nnz;
  ip.smem_hist = d <= kSmemHistMax ? 1 : 0;
  const double mean_row = n > 0 ? (double)nnz / (double)n : 0.0;
  // the hash cache of n_v for large d: long rows (one row per warp step) take a larger one
  // (more of the Zipf-popular columns counted in shared memory instead of global atomics)
  ip.hash_log = (!ip.smem_hist && mean_row >= 32.0) ? kIngestHashLogRows : kHashLog;
  const size_t hist_bytes =
      ((ip.smem_hist ? (size_t)d * sizeof(int32_t) : 2 * ((size_t)1 << ip.hash_log) * sizeof(int32_t)) + 15) &
      ~(size_t)15;
  // short rows: warp stages (kStageCap entries per warp) when they fit next to the histogram
  const size_t stage_bytes = 32 * (size_t)kStageCap * (sizeof(double) + sizeof(int32_t));
  const bool staged = n > 0 && mean_row <= 16.0 && hist_bytes + stage_bytes <= 200 * 1024;
  // long rows counted through the hash cache: one row per warp step (kIngestRows; c4 ingest
  // kernel 3.13 -> 2.81 ms).  With a shared histogram (c3) the flat path stays ahead.
  const bool rows = !staged && !ip.smem_hist && mean_row >= 32.0;
  const size_t hsmem = hist_bytes + (staged ? stage_bytes : 0);
  ip.stage_off = hist_bytes;
  // 32-row tiles per warp streamed flat (measured against a G-lanes-per-row variant, 77 vs
  // 69 us on c2, and a thread-per-row variant, 102 us: uncoalesced, 1.3x the DRAM bytes)
  const void* kfn = staged ? (const void*)ingest_tile_kernel<kIngestStaged>
                  : rows   ? (const void*)ingest_tile_kernel<kIngestRows>
                           : (const void*)ingest_tile_kernel<kIngestFlat>;
  const int kIngestBlock = 1024;
  const int rows_per_warp = 32;
  // (the attribute is per function, shared by every context: set it on every launch)
  CK(ctx, ensure_smem_attr(ctx->device, kfn, (int)hsmem));
  if (ctx->ingest_grid == 0) {  // once per context (n, d fixed)
    int per_sm = 1;
    CK(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kIngestBlock, hsmem));
    per_sm = std::max(per_sm, 1);
    const int64_t want = (n + rows_per_warp * (kIngestBlock / 32) - 1) / (rows_per_warp * (kIngestBlock / 32));
    ctx->ingest_grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sms * per_sm));
  }
  const int grid = ctx->ingest_grid;
  // d <= 4096: the ingest's last block also runs A1's finish (D, state, Delta_r, the combine
  // hot set) and writes the validation report -- two launches fewer per ingest
  ip.fuse = d <= 4096 ? 1 : 0;
  ip.self_init = self_init ? 1 : 0;
  ip.alpha = ctx->alpha;
  if (self_init && !ctx->ingest_part) TRY(dalloc(ctx, &ctx->ingest_part, (size_t)grid * d));
  ip.part = ctx->ingest_part;
  ip.xa = ctx->xa;
  ip.S = ctx->S;
  ip.habar = ctx->habar;
  ip.D = ctx->D;
  ip.comb_dmax = ctx->hot_freq > 0.0 ? 1.0 / ctx->hot_freq : 0.0;
  ip.max_h = kCombMaxH;
  ip.slot_of = ctx->slot_of;
  ip.hot_id = ctx->hot_id;
  ip.flag = ctx->flag;
  ip.host_out = ctx->h_ing_dev;
  ip.row_cap = ctx->row_cap;
  ip.hot_expected = ctx->hot_freq > 0.0 ? ctx->comb_H : -1;
  ip.guard = guard ? 1 : 0;
  ip.hot_tab = ctx->hot_tab;
  ip.hot_log = ctx->hot_log;
  ip.hot_dmax = ctx->hot_dmax;
  if (ctx->hot_tab) CK(ctx, cudaMemsetAsync(ctx->hot_tab, 0xff, sizeof(int32_t) << ctx->hot_log, ctx->stream));
  ctx->ing_fused = ip.fuse != 0;
  void* iargs[] = {&ip};
  CK(ctx, cudaLaunchKernel(kfn, dim3(grid), dim3(kIngestBlock), iargs, hsmem, ctx->stream));
  if (!ip.fuse) {
    profile_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, ctx->stream>>>(
        ctx->counts, ctx->xa, ctx->S, ctx->habar, ctx->D, d, n, ctx->flag + 1, ctx->hot_tab, ctx->hot_log,
        ctx->hot_dmax);
    CK(ctx, cudaGetLastError());
  }
  if (ctx->hot_freq > 0.0 && !ip.fuse) {  // hot set (combine kernel / pipe merge): p_v >= hot_freq
    hot_flag_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, ctx->stream>>>(ctx->D, d, 1.0 / ctx->hot_freq,
                                                                          ctx->comb_flag);
    CK(ctx, cudaGetLastError());
    CK(ctx, cub::DeviceScan::ExclusiveSum(ctx->cub_temp, ctx->cub_temp_bytes, ctx->comb_flag, ctx->comb_excl,
                                          (int)d, ctx->stream));
    hot_slot_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, ctx->stream>>>(
        ctx->comb_flag, ctx->comb_excl, d, kCombMaxH, ctx->slot_of, ctx->hot_id, ctx->flag + 2);
    CK(ctx, cudaGetLastError());
  }
  return ASAGA_OK;
}

// The validation results -> mapped pinned host memory (read by ingest_resolve now, or at
// the next blocking call after an asynchronous reload); guard: also set the run guard.
asaga_status enqueue_report(asaga_ctx* ctx, bool guard) {
  if (!ctx->ing_fused) {  // (fused: written by the ingest's last block)
    ingest_report_kernel<<<1, 1, 0, ctx->stream>>>(ctx->scratch, ctx->flag, ctx->h_ing_dev, ctx->row_cap,
                                                   ctx->hot_freq > 0.0 ? ctx->comb_H : -1, guard ? 1 : 0);
    CK(ctx, cudaGetLastError());
  }
  CK(ctx, cudaEventRecord(ctx->ev_ing, ctx->stream));
  return ASAGA_OK;
}

// D per stored entry: read by the plain kernel and by the combine kernel unless every feature
// is hot (D from its block table); the pipelined kernel gathers D_v from the d-vector itself
bool needs_dv(const asaga_ctx* ctx) {
  return !(use_combine(ctx) && ctx->comb_H == ctx->d) && !use_pipe(ctx) && !use_rec(ctx) && !use_dg(ctx);
}

// D per stored entry (+ the entry's combine slot): every kernel but the combine kernel
// with every feature hot (which reads D from its block table) streams it with the row
// (also lazily, from enqueue_run, when the kernel about to run needs it and the current
// matrix has not been expanded -- e.g. after set_algorithm leaves the pipelined kernel)
asaga_status enqueue_expand(asaga_ctx* ctx) {
  if (!needs_dv(ctx)) return ASAGA_OK;
  if (!ctx->dv) TRY(dalloc(ctx, &ctx->dv, ctx->nnz));
  expand_d_kernel<<<grid_for(ctx, ctx->nnz, kBlock), kBlock, 0, ctx->stream>>>(
      ctx->cols, ctx->D, ctx->nnz, ctx->hot_dmax, ctx->dv, ctx->slot_of, ctx->flag + 2, ctx->d, ctx->eslot);
  CK(ctx, cudaGetLastError());
  ctx->dv_ready = true;
  return ASAGA_OK;
}

// Read back an enqueued ingest's validation: errors (with the first bad row), L, the
// longest row, Delta_r and the combine hot count.  Blocks on the ingest's event only.
asaga_status ingest_resolve_impl(asaga_ctx* ctx);
asaga_status ingest_resolve(asaga_ctx* ctx) {
  const asaga_status s = ingest_resolve_impl(ctx);
  ctx->data_valid = s == ASAGA_OK;
  if (s != ASAGA_OK) ctx->reject_msg = ctx->err;
  if (s != ASAGA_OK && s != ASAGA_E_CUDA && s != ASAGA_E_OOM) {
    // rejected data: close the device-side run guard as well, so no update kernel already
    // or later enqueued (run_async) reads it, whatever the last good ingest left there
    set_flag_kernel<<<1, 1, 0, ctx->stream>>>(ctx->flag + 3, 0);
    (void)cudaGetLastError();
  }
  return s;
}

// Refuse kernels on a matrix that failed validation (the context still points at
// the rejected arrays) -- unless an asynchronous reload is pending, whose run guard decides
// on the device.
asaga_status require_data(asaga_ctx* ctx) {
  if (ctx->data_valid || ctx->ing_pending) return ASAGA_OK;
  return fail(ctx, ASAGA_E_STATE, "no valid data: the last reload failed validation (%s); reload valid data first",
              ctx->reject_msg.c_str());
}

asaga_status ingest_resolve_impl(asaga_ctx* ctx) {
  CK(ctx, cudaEventSynchronize(ctx->ev_ing));
  ctx->ing_pending = false;
  const volatile unsigned long long* hv = ctx->h_ing;  // written by the device (mapped)
  unsigned long long h[ERR_COUNT + 3];
  for (int e = 0; e < ERR_COUNT + 3; ++e) h[e] = hv[e];
  const int hflag[2] = {(int)(unsigned)(h[ERR_COUNT + 2] & 0xffffffffu),  // max_v n_v
                        (int)(unsigned)(h[ERR_COUNT + 2] >> 32)};        // number of hot features
  const int64_t d = ctx->d;
  static const char* what[ERR_COUNT] = {"indptr[0] must be 0 and indptr[n] must be nnz",
                                        "row pointers out of order or out of [0, nnz]",
                                        "empty row (rows must be non-empty)",
                                        "column index out of [0, d)",
                                        "column indices not strictly increasing",
                                        "non-finite value",
                                        "label not in {-1, +1}"};
  for (int e = 0; e < ERR_COUNT; ++e) {
    if (h[e] != ULLONG_MAX) {
      ctx->shape_valid = false;
      asaga_status s = e == ERR_LABEL ? ASAGA_E_BAD_LABEL : ASAGA_E_BAD_CSR;
      if (e == ERR_ENDS) return fail(ctx, s, "%s (nnz=%lld)", what[e], (long long)ctx->nnz);
      return fail(ctx, s, "row %llu: %s", h[e], what[e]);
    }
  }
  double max_sq;
  std::memcpy(&max_sq, &h[ERR_COUNT], sizeof(double));
  ctx->L = max_sq / 4.0 + ctx->lambda;
  ctx->max_row = (int64_t)h[ERR_COUNT + 1];
  ctx->delta_r = hflag[0];
  if (ctx->comb_freq > 0.0) {
    if (hflag[1] > kCombMaxH && hflag[1] < d)
      return fail(ctx, ASAGA_E_INVALID_ARG,
                  "combine_min_freq=%g selects %d features; at most %d fit a block (raise it)",
                  ctx->comb_freq, hflag[1], kCombMaxH);
    ctx->comb_H = hflag[1];
    if (ctx->comb_H == d && d > kCombMaxH)
      return fail(ctx, ASAGA_E_INVALID_ARG, "combine_min_freq=%g selects all %lld features; at most %d fit",
                  ctx->comb_freq, (long long)d, kCombMaxH);
  } else if (ctx->hot_freq > 0.0) {  // pipe_merge
    if (hflag[1] > kPipeMaxH)
      return fail(ctx, ASAGA_E_INVALID_ARG,
                  "pipe_late_min_freq=%g selects %d features; pipe_merge takes at most %d (raise it)",
                  ctx->hot_freq, hflag[1], kPipeMaxH);
    ctx->comb_H = hflag[1];
  }
  return ASAGA_OK;
}

// Blocking A0-A1: enqueue, resolve, per-entry D, launch shape; the run guard opens.
asaga_status ingest(asaga_ctx* ctx, const int64_t* indptr_in, const int32_t* indices_in,
                    const double* data_in, const double* y_in) {
  TRY(ingest_enqueue(ctx, indptr_in, indices_in, data_in, y_in, false));
  TRY(enqueue_report(ctx, false));
  TRY(ingest_resolve(ctx));
  TRY(enqueue_expand(ctx));
  TRY(configure_update(ctx));
  set_flag_kernel<<<1, 1, 0, ctx->stream>>>(ctx->flag + 3, 1);  // data and launch shape agree
  CK(ctx, cudaGetLastError());
  return ASAGA_OK;
}

// An asynchronous reload's pending validation: resolved by every blocking entry point.
asaga_status resolve_pending(asaga_ctx* ctx) {
  if (!ctx->ing_pending) return ASAGA_OK;
  const bool had_shape = ctx->shape_valid;
  const long long key_before[6] = {ctx->shape_key[0], ctx->shape_key[1], ctx->shape_key[2],
                                   ctx->shape_key[3], ctx->shape_key[4], ctx->shape_key[5]};
  const int H_before = ctx->comb_H;
  const bool dv_before = needs_dv(ctx);
  TRY(ingest_resolve(ctx));
  const bool dv_after = needs_dv(ctx);
  TRY(configure_update(ctx));
  const bool same = had_shape && std::memcmp(key_before, ctx->shape_key, sizeof(key_before)) == 0 &&
                    H_before == ctx->comb_H && dv_before == dv_after;
  if (!same) {  // the guarded runs enqueued since the reload were skipped on the device
    if (dv_after && !dv_before) TRY(enqueue_expand(ctx));
    set_flag_kernel<<<1, 1, 0, ctx->stream>>>(ctx->flag + 3, 1);
    CK(ctx, cudaGetLastError());
    return fail(ctx, ASAGA_E_STATE,
                "the asynchronously reloaded data changed the launch profile (longest row / hot set); "
                "the runs enqueued since the reload were skipped -- run them again");
  }
  return ASAGA_OK;
}

asaga_status make_ctx(asaga_ctx** out, const asaga_csr_view* A, const double* y, double lambda,
                      double gamma, const asaga_options* opt, asaga_ctx** ctx_out) {
  if (!out) return fail(nullptr, ASAGA_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!A || !y) return fail(nullptr, ASAGA_E_INVALID_ARG, "A or y is NULL");
  if (!A->indptr || (A->nnz > 0 && (!A->indices || !A->data)))
    return fail(nullptr, ASAGA_E_INVALID_ARG, "CSR arrays are NULL");
  if (A->n <= 0 || A->d <= 0 || A->nnz < 0)
    return fail(nullptr, ASAGA_E_INVALID_ARG, "need n > 0, d > 0, nnz >= 0 (n=%lld d=%lld nnz=%lld)",
                (long long)A->n, (long long)A->d, (long long)A->nnz);
  if (A->d > INT32_MAX) return fail(nullptr, ASAGA_E_INVALID_ARG, "d exceeds int32 indices");
  if (!(lambda > 0.0) || !std::isfinite(lambda))
    return fail(nullptr, ASAGA_E_INVALID_ARG, "lambda must be > 0 (got %g)", lambda);
  if (!(gamma > 0.0) || !std::isfinite(gamma))
    return fail(nullptr, ASAGA_E_INVALID_ARG, "gamma must be > 0 (got %g)", gamma);
  asaga_options o;
  asaga_options_default(&o);
  if (opt) o = *opt;
  asaga_ctx* ctx = new asaga_ctx();
  ctx->device = o.device;
  ctx->n = A->n;
  ctx->d = A->d;
  ctx->nnz = A->nnz;
  ctx->lambda = lambda;
  ctx->gamma = gamma;
  ctx->deterministic = o.deterministic ? 1 : 0;
  ctx->atomic_mode = o.atomic_mode ? 1 : 0;
  ctx->record = o.record_samples ? 1 : 0;
  ctx->ov_every = o.measure_overlap > 0 ? o.measure_overlap : 0;
  ctx->concurrency_opt = o.concurrency;
  ctx->lanes_opt = o.lanes_per_sample;
  if (!(o.bulk_scatter_min_freq >= 0.0) || o.bulk_scatter_min_freq > 1.0) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG, "bulk_scatter_min_freq must be in [0, 1] (got %g)",
                o.bulk_scatter_min_freq);
  }
  // p_v = n_v / n >= f  <=>  D_v = n / n_v <= 1 / f
  ctx->bulk_dmax = o.bulk_scatter_min_freq > 0.0 ? 1.0 / o.bulk_scatter_min_freq : 0.0;
  if (!(o.hot_split_min_freq >= 0.0) || o.hot_split_min_freq > 1.0 ||
      (o.hot_split_min_freq > 0.0 && o.bulk_scatter_min_freq > 0.0)) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG,
                "hot_split_min_freq must be in [0, 1] and cannot be combined with bulk_scatter_min_freq");
  }
  ctx->hot_dmax = o.hot_split_min_freq > 0.0 ? 1.0 / o.hot_split_min_freq : 0.0;
  ctx->replica_every = o.smem_replica_refresh > 0 ? o.smem_replica_refresh : 0;
  if (!(o.combine_min_freq >= 0.0) || o.combine_min_freq > 1.0 ||
      (o.combine_min_freq > 0.0 && (o.hot_split_min_freq > 0.0 || o.bulk_scatter_min_freq > 0.0 ||
                                    o.smem_replica_refresh > 0))) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG,
                "combine_min_freq must be in [0, 1] and cannot be combined with the bulk scatter, "
                "the hot split or the replica");
  }
  ctx->comb_freq = o.combine_min_freq;
  if (o.combine_cluster < 0 || o.combine_cluster > 8) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG, "combine_cluster must be in [0, 8] (got %d)", o.combine_cluster);
  }
  ctx->comb_cluster_opt = o.combine_cluster;
  if (o.combine_max_blocks < 0) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG, "combine_max_blocks must be >= 0 (got %d)", o.combine_max_blocks);
  }
  ctx->comb_max_blocks = o.combine_max_blocks;
  ctx->l2_persist = o.l2_persist_state ? 1 : 0;
  if (!(o.pipe_late_min_freq >= 0.0) || !std::isfinite(o.pipe_late_min_freq) ||
      (o.pipe_late_min_freq > 0.0 && (o.combine_min_freq > 0.0 || o.bulk_scatter_min_freq > 0.0 ||
                                      o.smem_replica_refresh > 0))) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG,
                "pipe_late_min_freq must be finite and >= 0, and cannot be combined with combining, "
                "the bulk scatter or the replica");
  }
  ctx->pipe_freq = o.pipe_late_min_freq;
  if (o.pipe_merge_ns < 0 || o.pipe_merge_ns > 1000000 || (o.pipe_merge_ns > 0 && !(o.pipe_late_min_freq > 0.0))) {
    *ctx_out = ctx;
    return fail(ctx, ASAGA_E_INVALID_ARG, "pipe_merge_ns must be in [0, 1e6] and needs pipe_late_min_freq > 0");
  }
  ctx->pipe_merge = o.pipe_merge_ns;
  ctx->row_copy_elementwise = o.row_copy_elementwise ? 1 : 0;
  ctx->scatter_unpaired = o.scatter_unpaired ? 1 : 0;
  ctx->d_gather = o.d_gather ? 1 : 0;
  ctx->rec_layout = o.record_layout ? 1 : 0;
  ctx->hot_freq = o.combine_min_freq > 0.0 ? o.combine_min_freq : (ctx->pipe_merge ? ctx->pipe_freq : 0.0);
  ctx->comb_wt = o.combine_write_through ? 1 : 0;
  *ctx_out = ctx;
  cudaError_t e = cudaSetDevice(o.device);
  if (e != cudaSuccess) return fail(ctx, ASAGA_E_CUDA, "cudaSetDevice(%d): %s", o.device, cudaGetErrorString(e));
  CK(ctx, cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, o.device));
  if (o.stream) {
    ctx->stream = (cudaStream_t)o.stream;
  } else {
    CK(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  CK(ctx, cudaEventCreate(&ctx->ev0));
  CK(ctx, cudaEventCreate(&ctx->ev1));
  return ASAGA_OK;
}

asaga_status finish_init(asaga_ctx** out, asaga_ctx* ctx, asaga_status s) {
  if (s != ASAGA_OK) {
    if (ctx) {
      g_thread_err = ctx->err;
      asaga_destroy(ctx);
    }
    *out = nullptr;
    return s;
  }
  *out = ctx;
  return ASAGA_OK;
}

asaga_status ensure_csc(asaga_ctx* ctx) {
  TRY(require_data(ctx));
  if (ctx->csc_built) return ASAGA_OK;
  const int64_t d = ctx->d, nnz = ctx->nnz, n = ctx->n;
  cudaStream_t s = ctx->stream;
  int64_t *colptr = nullptr, *cnt64 = nullptr, *perm_in = nullptr, *perm_out = nullptr;
  int32_t *keys_out = nullptr, *row_of = nullptr;
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    for (void* p : {(void*)colptr, (void*)cnt64, (void*)perm_in, (void*)perm_out, (void*)keys_out,
                    (void*)row_of})
      if (p) cudaFree(p);
  };
#define CKC(call)                                                                           \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      cleanup();                                                                            \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? ASAGA_E_OOM : ASAGA_E_CUDA,        \
                  "%s failed: %s", #call, cudaGetErrorString(e_));                          \
    }                                                                                       \
  } while (0)
  CKC(cudaMalloc(&colptr, sizeof(int64_t) * (d + 1)));
  CKC(cudaMalloc(&cnt64, sizeof(int64_t) * (d + 1)));
  CKC(cudaMalloc(&perm_in, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
  CKC(cudaMalloc(&perm_out, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
  CKC(cudaMalloc(&keys_out, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  CKC(cudaMalloc(&row_of, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  // colptr = exclusive scan of n_v
  CKC(cudaMemsetAsync(cnt64, 0, sizeof(int64_t) * (d + 1), s));
  segcount_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, s>>>(ctx->counts, d, 1, cnt64);
  CKC(cudaGetLastError());
  size_t tb = 0, tb2 = 0;
  CKC(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt64, colptr, d + 1, s));
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < d) ++end_bit;
  CKC(cub::DeviceRadixSort::SortPairs(nullptr, tb2, ctx->cols, keys_out, perm_in, perm_out, nnz, 0,
                                      end_bit, s));
  void* temp = nullptr;
  CKC(cudaMalloc(&temp, std::max(tb, tb2)));
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt64, colptr, d + 1, s);
  if (e == cudaSuccess) {
    iota_kernel<<<grid_for(ctx, nnz, kBlock), kBlock, 0, s>>>(perm_in, nnz);
    e = cub::DeviceRadixSort::SortPairs(temp, tb2, ctx->cols, keys_out, perm_in, perm_out, nnz, 0,
                                        end_bit, s);
  }
  cudaStreamSynchronize(s);
  cudaFree(temp);
  CKC(e);
  asaga_status st;
  if ((st = dalloc(ctx, &ctx->csc_rows, nnz)) != ASAGA_OK) { cleanup(); return st; }
  if ((st = dalloc(ctx, &ctx->csc_vals, nnz)) != ASAGA_OK) { cleanup(); return st; }
  row_of_kernel<<<grid_for(ctx, n * 32, kBlock), kBlock, 0, s>>>(ctx->rowptr, n, row_of);
  csc_gather_kernel<<<grid_for(ctx, nnz, kBlock), kBlock, 0, s>>>(perm_out, row_of, ctx->vals, ctx->y, nnz,
                                                                    ctx->csc_rows, ctx->csc_vals);
  CKC(cudaGetLastError());
  // fixed segments of <= kColSeg entries per column (deterministic summation order)
  if ((st = dalloc(ctx, &ctx->seg_ptr, d + 1)) != ASAGA_OK) { cleanup(); return st; }
  CKC(cudaMemsetAsync(cnt64, 0, sizeof(int64_t) * (d + 1), s));
  segcount_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, s>>>(ctx->counts, d, kColSeg, cnt64);
  CKC(cudaMalloc(&temp, tb));
  e = cub::DeviceScan::ExclusiveSum(temp, tb, cnt64, ctx->seg_ptr, d + 1, s);
  cudaStreamSynchronize(s);
  cudaFree(temp);
  CKC(e);
  CKC(cudaMemcpy(&ctx->nseg, ctx->seg_ptr + d, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if ((st = dalloc(ctx, &ctx->seg_lo, ctx->nseg)) != ASAGA_OK) { cleanup(); return st; }
  if ((st = dalloc(ctx, &ctx->seg_hi, ctx->nseg)) != ASAGA_OK) { cleanup(); return st; }
  if ((st = dalloc(ctx, &ctx->seg_sum, ctx->nseg)) != ASAGA_OK) { cleanup(); return st; }
  if ((st = dalloc(ctx, &ctx->sig, n)) != ASAGA_OK) { cleanup(); return st; }
  segfill_kernel<<<grid_for(ctx, d, kBlock), kBlock, 0, s>>>(colptr, ctx->seg_ptr, d, kColSeg,
                                                             ctx->seg_lo, ctx->seg_hi);
  CKC(cudaGetLastError());
  cleanup();
#undef CKC
  ctx->csc_built = true;
  return ASAGA_OK;
}

// Enqueue margins (+ sigma~ if want_sig) and the objective finish for device x
// (element stride xs: 1 for a dense vector, 2 for the {x, abar} pairs).
asaga_status enqueue_objective(asaga_ctx* ctx, const double* x_dev, int xs, double* f_dev,
                               double* loss_sum_dev, bool want_sig, cudaStream_t s) {
  TRY(require_data(ctx));
  double* sig = want_sig ? ctx->sig : nullptr;
  // the margin kernel's last block also finishes f (ticket in flag[5], reset by that block)
  const ObjFinish fin{ctx->flag + 5, ctx->n, ctx->lambda, f_dev, loss_sum_dev};
  // short rows: G lanes per row (G ~ mean/3); long rows: 32-row tiles streamed flat
  const double mean = (double)ctx->nnz / (double)ctx->n;
  if (mean <= 16.0)
    margin_thread_kernel<<<ctx->obj_blocks, kBlock, 0, s>>>(ctx->rowptr, ctx->cols, ctx->vals, ctx->y, x_dev, xs,
                                                            ctx->n, sig, ctx->block_loss, ctx->d, fin);
  else if (mean <= 24.0)
    margin_rows_kernel<8, 4><<<ctx->obj_blocks, kBlock, 0, s>>>(ctx->rowptr, ctx->cols, ctx->vals, ctx->y, x_dev, xs,
                                                                 ctx->n, sig, ctx->block_loss, ctx->d, fin);
  else if (ctx->margin_tiles)
    margin_kernel<<<ctx->obj_blocks, kBlock, 0, s>>>(ctx->rowptr, ctx->cols, ctx->vals, ctx->y, x_dev, xs, ctx->n, sig,
                                                     ctx->block_loss, ctx->d, fin);
  else
    margin_rows_kernel<32, 4><<<ctx->obj_blocks, kBlock, 0, s>>>(ctx->rowptr, ctx->cols, ctx->vals, ctx->y, x_dev, xs,
                                                                  ctx->n, sig, ctx->block_loss, ctx->d, fin);
  CK(ctx, cudaGetLastError());
  return ASAGA_OK;
}

// Enqueue sum_i sigma~_i a~_i (raw, divide=0) or the full gradient (divide=1) into g_dev.
asaga_status enqueue_gradient(asaga_ctx* ctx, const double* x_dev, int xs, double* g_dev, int divide,
                              cudaStream_t s) {
  colseg_kernel<<<grid_for(ctx, ctx->nseg * 32, kBlock), kBlock, 0, s>>>(
      ctx->seg_lo, ctx->seg_hi, ctx->nseg, ctx->csc_rows, ctx->csc_vals, ctx->sig, ctx->seg_sum);
  CK(ctx, cudaGetLastError());
  colsum_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, s>>>(
      ctx->seg_ptr, ctx->seg_sum, x_dev, xs, ctx->d, (double)ctx->n, ctx->lambda, g_dev, divide);
  CK(ctx, cudaGetLastError());
  return ASAGA_OK;
}

// The current iterate for A9: for large d a dense copy (one pass over the pair array, then
// the margins gather 8-B x values instead of 16-B pairs -- c4: 1.6 -> ~0.6 ms); small d reads
// the pairs in place (element stride 2 S).
const double* current_x(asaga_ctx* ctx, int* xs, cudaStream_t s) {
  if (ctx->d > 4096 && ctx->xdense != nullptr) {
    unpack_xa_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, s>>>(
        ctx->xa, ctx->S, ctx->habar, ctx->D, ctx->hot_dmax, ctx->xdense, nullptr, ctx->d);
    *xs = 1;
    return ctx->xdense;
  }
  *xs = 2 * ctx->S;
  return &ctx->xa[0].x;
}

asaga_status enqueue_run(asaga_ctx* ctx, uint64_t n_updates, uint64_t seed, bool timed) {
  TRY(require_data(ctx));
  if (n_updates == 0) return ASAGA_OK;
  if (ctx->algorithm == ASAGA_ALG_KROMAGNON && !ctx->snapshot_valid)
    return fail(ctx, ASAGA_E_STATE, "KROMAGNON needs asaga_snapshot() before asaga_run");
  UpdateParams p;
  p.rowptr = ctx->rowptr;
  p.cols = ctx->cols;
  p.vals = ctx->vals;
  p.y = ctx->y;
  p.dv = (use_rec(ctx) || use_dg(ctx)) ? nullptr : ctx->dv;
  p.D = ctx->D;
  p.xa = ctx->xa;
  p.S = ctx->S;
  p.habar = ctx->habar;
  p.alpha = ctx->alpha;
  p.visits = ctx->visits;
  p.shash = ctx->shash;
  p.ov = ctx->ov;
  p.frozen = ctx->algorithm != ASAGA_ALG_ASAGA ? 1 : 0;
  p.repl_d = use_replica(ctx) ? (int)ctx->d : 0;
  p.repl_every = ctx->replica_every > 0 ? ctx->replica_every : 1;
  p.ov_every = ctx->ov_every > 0 ? ctx->ov_every : 1;
  p.n = (uint64_t)ctx->n;
  p.gamma = ctx->gamma;
  p.lambda_ = ctx->lambda;
  p.inv_n = 1.0 / (double)ctx->n;
  p.seed = seed;
  p.t0 = ctx->t;
  p.T = n_updates;
  p.workers = ctx->workers;
  p.overflow = ctx->overflow;
  p.bulk_dmax = ctx->bulk_dmax;
  p.debug_mode = 0;
#ifdef ASAGA_TIMING
  if (const char* m = getenv("ASAGA_DEBUG_MODE")) p.debug_mode = atoi(m);
#endif
  p.H = ctx->comb_H;
  p.nwb = ctx->comb_nwb;
  p.hot_id = ctx->hot_id;
  p.eslot = ctx->comb_H > 0 ? ctx->eslot : nullptr;
  p.comm_passes = ctx->comb_freq > 0.0 ? ctx->scratch + ERR_COUNT + 2 : nullptr;
  p.wt = ctx->comb_wt;
  p.split = ctx->hot_dmax > 0.0 ? 1 : 0;
  p.pair_red = ctx->scatter_unpaired ? 0 : 1;
  p.late_dmax = ctx->pipe_freq > 0.0 ? 1.0 / ctx->pipe_freq : 0.0;
  p.hot_dmax = ctx->hot_dmax;
  p.merge_ts = use_merge(ctx) ? merge_ts(ctx) : 0;
  p.merge_ns = ctx->pipe_merge;
  // 1-D TMA row staging when the arrays the kernel streams are 16-B aligned (the caller's
  // borrowed arrays may be offset views)
  p.nnz = ctx->nnz;
  p.bulk_rows = ((((uintptr_t)ctx->cols) | ((uintptr_t)ctx->vals) | ((uintptr_t)p.dv)) & 15) == 0 &&
                !ctx->row_copy_elementwise;
  p.hot_tab = use_rec(ctx) && ctx->hot_dmax > 0.0 ? ctx->hot_tab : nullptr;
  p.hot_log = ctx->hot_log;
  p.ok = ctx->flag + 3;  // 0 while an asynchronous reload's data does not fit this launch
  if (needs_dv(ctx) && !ctx->dv_ready) TRY(enqueue_expand(ctx));
  if (p.comm_passes && use_combine(ctx))
    CK(ctx, cudaMemsetAsync(p.comm_passes, 0, sizeof(unsigned long long), ctx->stream));
  if (use_combine(ctx)) {
    const int64_t need = std::min<int64_t>(ctx->workers, (int64_t)std::min<uint64_t>(n_updates, (uint64_t)INT64_MAX));
    int grid = (int)((need + ctx->comb_nwb - 1) / ctx->comb_nwb);
    grid = (grid + ctx->comb_csize - 1) / ctx->comb_csize * ctx->comb_csize;
    UpdFn cfn = combine_fn(ctx, ctx->lanes, ctx->nr);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ctx->comb_csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ctx->block);
    cfg.dynamicSmemBytes = ctx->smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(ctx, ensure_smem_attr(ctx->device, (const void*)cfn, (int)ctx->smem));
    if (timed) CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    CK(ctx, cudaLaunchKernelEx(&cfg, cfn, p));
    if (timed) CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->t += n_updates;
    return ASAGA_OK;
  }
  UpdFn fn = update_fn(ctx, ctx->lanes, ctx->nr);
  // Fewer updates than workers: launch only what is needed.  The stride stays W,
  // so the t -> worker map does not depend on the launch.
  int64_t workers = std::min<int64_t>(ctx->workers, (int64_t)std::min<uint64_t>(n_updates, (uint64_t)INT64_MAX));
  int grid = 1, block = 32;
  launch_shape(ctx, workers, &grid, &block);
  const int groups = (block - (use_merge(ctx) ? 32 : 0)) / ctx->lanes;
  const size_t smem = pre_bytes(ctx, true) + (size_t)groups * ctx->group_bytes + merge_bytes(ctx, groups);
  CK(ctx, ensure_smem_attr(ctx->device, (const void*)fn, (int)smem));
  if (timed) CK(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  if (ctx->l2_persist) {
    // the {x, abar} pairs as a persisting L2 window for this launch only
    // (the device's persisting carve-out is set once per context, at most its maximum)
    int max_win = 0, max_persist = 0;
    CK(ctx, cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
    CK(ctx, cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
    const size_t bytes = std::min<size_t>((size_t)ctx->d * ctx->S * sizeof(double2), (size_t)max_win);
    size_t cur = 0;
    CK(ctx, cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
    const size_t want = std::min<size_t>(bytes, (size_t)max_persist);
    if (cur < want) CK(ctx, cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = ctx->xa;
    attr[0].val.accessPolicyWindow.num_bytes = bytes;
    attr[0].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)want / (double)bytes);
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(ctx, cudaLaunchKernelEx(&cfg, fn, p));
  } else {
    void* args[] = {&p};
    CK(ctx, cudaLaunchKernel((const void*)fn, dim3(grid), dim3(block), args, smem, ctx->stream));
  }
  if (timed) CK(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->t += n_updates;
  return ASAGA_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

void asaga_options_default(asaga_options* opt) {
  if (!opt) return;
  opt->device = 0;
  opt->deterministic = 0;
  opt->concurrency = 0;
  opt->lanes_per_sample = 0;
  opt->atomic_mode = 1;
  opt->record_samples = 0;
  opt->measure_overlap = 0;
  opt->stream = nullptr;
  opt->bulk_scatter_min_freq = 0.0;
  opt->hot_split_min_freq = 0.0;
  opt->smem_replica_refresh = 0;
  opt->combine_min_freq = 0.0;
  opt->combine_cluster = 0;
  opt->combine_write_through = 0;
  opt->combine_max_blocks = 0;
  opt->l2_persist_state = 0;
  opt->pipe_late_min_freq = 0.0;
  opt->pipe_merge_ns = 0;
  opt->row_copy_elementwise = 0;
  opt->record_layout = 0;
  opt->scatter_unpaired = 0;
  opt->d_gather = 0;
}

asaga_status asaga_init(asaga_ctx** out, const asaga_csr_view* A, const double* y, double lambda,
                        double gamma, const asaga_options* opt) {
  asaga_ctx* ctx = nullptr;
  asaga_status s = make_ctx(out, A, y, lambda, gamma, opt, &ctx);
  if (s != ASAGA_OK) return finish_init(out, ctx, s);
  s = alloc_state(ctx);
  if (s == ASAGA_OK) s = asaga_reload(ctx, A, y);
  return finish_init(out, ctx, s);
}

asaga_status asaga_init_device(asaga_ctx** out, const asaga_csr_view* A, const double* y,
                               double lambda, double gamma, const asaga_options* opt) {
  asaga_ctx* ctx = nullptr;
  asaga_status s = make_ctx(out, A, y, lambda, gamma, opt, &ctx);
  if (s != ASAGA_OK) return finish_init(out, ctx, s);
  s = alloc_state(ctx);
  if (s == ASAGA_OK) s = asaga_reload_device(ctx, A, y);
  return finish_init(out, ctx, s);
}

static asaga_status check_same_shape(asaga_ctx* ctx, const asaga_csr_view* A, const double* y) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  if (!A || !y || !A->indptr || (A->nnz > 0 && (!A->indices || !A->data)))
    return fail(ctx, ASAGA_E_INVALID_ARG, "NULL CSR array or labels");
  if (A->n != ctx->n || A->d != ctx->d || A->nnz != ctx->nnz)
    return fail(ctx, ASAGA_E_INVALID_ARG, "reload needs the context's shape (n=%lld d=%lld nnz=%lld)",
                (long long)ctx->n, (long long)ctx->d, (long long)ctx->nnz);
  return ASAGA_OK;
}

asaga_status asaga_reload(asaga_ctx* ctx, const asaga_csr_view* A, const double* y) {
  TRY(check_same_shape(ctx, A, y));
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  if (A->indptr[0] != 0 || A->indptr[A->n] != A->nnz)
    return fail(ctx, ASAGA_E_BAD_CSR, "indptr[0] must be 0 and indptr[n] must be nnz (got %lld and %lld, nnz=%lld)",
                (long long)A->indptr[0], (long long)A->indptr[A->n], (long long)A->nnz);
  // host -> device: the host/device boundary, into the context's own arrays
  if (!ctx->own_rowptr) {
    TRY(dalloc(ctx, &ctx->own_rowptr, ctx->n + 1));
    TRY(dalloc(ctx, &ctx->own_cols, ctx->nnz));
    TRY(dalloc(ctx, &ctx->own_vals, ctx->nnz));
    TRY(dalloc(ctx, &ctx->own_y, ctx->n));
  }
  CK(ctx, cudaMemcpyAsync(ctx->own_rowptr, A->indptr, sizeof(int64_t) * (ctx->n + 1),
                          cudaMemcpyHostToDevice, ctx->stream));
  CK(ctx, cudaMemcpyAsync(ctx->own_cols, A->indices, sizeof(int32_t) * ctx->nnz, cudaMemcpyHostToDevice,
                          ctx->stream));
  CK(ctx, cudaMemcpyAsync(ctx->own_vals, A->data, sizeof(double) * ctx->nnz, cudaMemcpyHostToDevice,
                          ctx->stream));
  CK(ctx, cudaMemcpyAsync(ctx->own_y, y, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
  return ingest(ctx, ctx->own_rowptr, ctx->own_cols, ctx->own_vals, ctx->own_y);
}

asaga_status asaga_reload_device(asaga_ctx* ctx, const asaga_csr_view* A, const double* y) {
  TRY(check_same_shape(ctx, A, y));
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  // the ingest pass itself checks indptr[0] = 0, indptr[n] = nnz (no extra round trip);
  // the context then reads the caller's arrays (borrowed until the next reload / destroy)
  return ingest(ctx, A->indptr, A->indices, A->data, y);
}

asaga_status asaga_reload_device_async(asaga_ctx* ctx, const asaga_csr_view* A, const double* y) {
  TRY(check_same_shape(ctx, A, y));
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));
  if (!ctx->shape_valid) return ingest(ctx, A->indptr, A->indices, A->data, y);  // no shape to keep
  TRY(ingest_enqueue(ctx, A->indptr, A->indices, A->data, y, true));
  TRY(enqueue_expand(ctx));
  // the run guard opens on the device iff the data is valid and fits the current launch
  TRY(enqueue_report(ctx, true));
  ctx->t = 0;
  ctx->ing_pending = true;
  return ASAGA_OK;
}

asaga_status asaga_reload_async(asaga_ctx* ctx, const asaga_csr_view* A, const double* y) {
  TRY(check_same_shape(ctx, A, y));
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // (also: the previous asynchronous copy has landed)
  if (!ctx->shape_valid) return asaga_reload(ctx, A, y);  // no launch shape to keep yet
  if (!ctx->copy_stream) CK(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  const int b = ctx->hs_next;
  asaga_ctx::HostSet& h = ctx->hs[b];
  if (!h.rowptr) {
    TRY(dalloc(ctx, &h.rowptr, ctx->n + 1));
    TRY(dalloc(ctx, &h.cols, ctx->nnz));
    TRY(dalloc(ctx, &h.vals, ctx->nnz));
    TRY(dalloc(ctx, &h.y, ctx->n));
    CK(ctx, cudaEventCreateWithFlags(&h.copied, cudaEventDisableTiming));
    CK(ctx, cudaEventCreateWithFlags(&h.free, cudaEventDisableTiming));
  }
  // the copy may start once the compute stream is done with this set's previous contents
  if (h.used) CK(ctx, cudaStreamWaitEvent(ctx->copy_stream, h.free, 0));
  CK(ctx, cudaMemcpyAsync(h.rowptr, A->indptr, sizeof(int64_t) * (ctx->n + 1), cudaMemcpyHostToDevice,
                          ctx->copy_stream));
  CK(ctx, cudaMemcpyAsync(h.cols, A->indices, sizeof(int32_t) * ctx->nnz, cudaMemcpyHostToDevice,
                          ctx->copy_stream));
  CK(ctx, cudaMemcpyAsync(h.vals, A->data, sizeof(double) * ctx->nnz, cudaMemcpyHostToDevice,
                          ctx->copy_stream));
  CK(ctx, cudaMemcpyAsync(h.y, y, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, ctx->copy_stream));
  CK(ctx, cudaEventRecord(h.copied, ctx->copy_stream));
  // compute stream: everything enqueued so far read the other set (or the caller's arrays)
  asaga_ctx::HostSet& o = ctx->hs[1 - b];
  if (o.used) CK(ctx, cudaEventRecord(o.free, ctx->stream));
  CK(ctx, cudaStreamWaitEvent(ctx->stream, h.copied, 0));
  h.used = true;
  ctx->hs_next = 1 - b;
  TRY(ingest_enqueue(ctx, h.rowptr, h.cols, h.vals, h.y, true));
  TRY(enqueue_expand(ctx));
  TRY(enqueue_report(ctx, true));
  ctx->t = 0;
  ctx->ing_pending = true;
  return ASAGA_OK;
}

asaga_status asaga_run_async(asaga_ctx* ctx, uint64_t n_updates, uint64_t seed) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  return enqueue_run(ctx, n_updates, seed, false);
}

asaga_status asaga_run(asaga_ctx* ctx, uint64_t n_updates, uint64_t seed) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  if (n_updates == 0) return ASAGA_OK;
  TRY(enqueue_run(ctx, n_updates, seed, true));
  CK(ctx, cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  nonfinite_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, ctx->stream>>>(ctx->xa, ctx->S, ctx->d, ctx->flag);
  CK(ctx, cudaGetLastError());
  int bad = 0;
  CK(ctx, cudaMemcpyAsync(&bad, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  CK(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->last_ms = ms;
  if (bad) return fail(ctx, ASAGA_E_DIVERGED, "non-finite iterate after %llu updates (gamma=%g too large?)",
                       (unsigned long long)ctx->t, ctx->gamma);
  return ASAGA_OK;
}

asaga_status asaga_objective_device(asaga_ctx* ctx, const double* x_dev, double* f_dev) {
  if (!ctx || !f_dev) return fail(ctx, ASAGA_E_INVALID_ARG, "ctx or f_dev is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  if (x_dev) return enqueue_objective(ctx, x_dev, 1, f_dev, nullptr, false, ctx->stream);
  int xs = 1;
  const double* xd = current_x(ctx, &xs, ctx->stream);
  return enqueue_objective(ctx, xd, xs, f_dev, nullptr, false, ctx->stream);
}

asaga_status asaga_objective(asaga_ctx* ctx, const double* x, double* f_out) {
  if (!ctx || !f_out) return fail(ctx, ASAGA_E_INVALID_ARG, "ctx or f_out is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  int xs = 1;
  const double* xd = x ? nullptr : current_x(ctx, &xs, ctx->stream);
  if (x) {
    CK(ctx, cudaMemcpyAsync(ctx->tmp_d, x, sizeof(double) * ctx->d, cudaMemcpyHostToDevice, ctx->stream));
    xd = ctx->tmp_d;
    xs = 1;
  }
  TRY(enqueue_objective(ctx, xd, xs, ctx->scal, nullptr, false, ctx->stream));
  CK(ctx, cudaMemcpyAsync(f_out, ctx->scal, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  return ASAGA_OK;
}

asaga_status asaga_full_grad(asaga_ctx* ctx, const double* x, double* g_out) {
  if (!ctx || !g_out) return fail(ctx, ASAGA_E_INVALID_ARG, "ctx or g_out is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  TRY(ensure_csc(ctx));
  int xs = 1;
  const double* xd = x ? nullptr : current_x(ctx, &xs, ctx->stream);
  if (x) {
    CK(ctx, cudaMemcpyAsync(ctx->tmp_d, x, sizeof(double) * ctx->d, cudaMemcpyHostToDevice, ctx->stream));
    xd = ctx->tmp_d;
    xs = 1;
  }
  TRY(enqueue_objective(ctx, xd, xs, ctx->scal, nullptr, true, ctx->stream));
  TRY(enqueue_gradient(ctx, xd, xs, ctx->tmp_d2, 1, ctx->stream));
  CK(ctx, cudaMemcpyAsync(g_out, ctx->tmp_d2, sizeof(double) * ctx->d, cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  return ASAGA_OK;
}

asaga_status asaga_partial_obj_grad(asaga_ctx* ctx, const double* x_dev, double* out_dev, void* stream) {
  if (!ctx || !x_dev || !out_dev) return fail(ctx, ASAGA_E_INVALID_ARG, "NULL argument");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  TRY(ensure_csc(ctx));
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
  // the partial shares the context's A9 scratch (finish ticket, block partials, sigma,
  // segment sums) with asaga_objective on ctx->stream: order the two streams both ways
  const bool other = s != ctx->stream;
  if (other) {
    if (!ctx->ev_part) CK(ctx, cudaEventCreateWithFlags(&ctx->ev_part, cudaEventDisableTiming));
    CK(ctx, cudaEventRecord(ctx->ev_part, ctx->stream));
    CK(ctx, cudaStreamWaitEvent(s, ctx->ev_part, 0));
  }
  TRY(enqueue_objective(ctx, x_dev, 1, nullptr, out_dev + ctx->d, true, s));
  TRY(enqueue_gradient(ctx, x_dev, 1, out_dev, 0, s));
  if (other) {
    CK(ctx, cudaEventRecord(ctx->ev_part, s));
    CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_part, 0));
  }
  return ASAGA_OK;
}

asaga_status asaga_get_state(asaga_ctx* ctx, double* x, double* alpha, double* alpha_bar, uint64_t* t) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  cudaStream_t s = ctx->stream;
  if (x || alpha_bar) {
    unpack_xa_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, s>>>(
        ctx->xa, ctx->S, ctx->habar, ctx->D, ctx->hot_dmax, x ? ctx->tmp_d : nullptr,
        alpha_bar ? ctx->tmp_d2 : nullptr, ctx->d);
    CK(ctx, cudaGetLastError());
    if (x) CK(ctx, cudaMemcpyAsync(x, ctx->tmp_d, sizeof(double) * ctx->d, cudaMemcpyDeviceToHost, s));
    if (alpha_bar)
      CK(ctx, cudaMemcpyAsync(alpha_bar, ctx->tmp_d2, sizeof(double) * ctx->d, cudaMemcpyDeviceToHost, s));
  }
  if (alpha) {
    fold_alpha_kernel<<<grid_for(ctx, ctx->n, kBlock), kBlock, 0, s>>>(ctx->alpha, ctx->y, ctx->tmp_n, ctx->n);
    CK(ctx, cudaGetLastError());
    CK(ctx, cudaMemcpyAsync(alpha, ctx->tmp_n, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, s));
  }
  CK(ctx, cudaStreamSynchronize(s));
  if (t) *t = ctx->t;
  return ASAGA_OK;
}

asaga_status asaga_set_state(asaga_ctx* ctx, const double* x, const double* alpha,
                             const double* alpha_bar, const uint64_t* t) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  cudaStream_t s = ctx->stream;
  if (x) CK(ctx, cudaMemcpyAsync(ctx->tmp_d, x, sizeof(double) * ctx->d, cudaMemcpyHostToDevice, s));
  if (alpha_bar)
    CK(ctx, cudaMemcpyAsync(ctx->tmp_d2, alpha_bar, sizeof(double) * ctx->d, cudaMemcpyHostToDevice, s));
  if (x || alpha_bar) {
    pack_xa_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, s>>>(
        ctx->xa, ctx->S, ctx->habar, x ? ctx->tmp_d : nullptr, alpha_bar ? ctx->tmp_d2 : nullptr, ctx->d);
    CK(ctx, cudaGetLastError());
  }
  if (alpha) {
    CK(ctx, cudaMemcpyAsync(ctx->tmp_n, alpha, sizeof(double) * ctx->n, cudaMemcpyHostToDevice, s));
    fold_alpha_kernel<<<grid_for(ctx, ctx->n, kBlock), kBlock, 0, s>>>(ctx->tmp_n, ctx->y, ctx->alpha, ctx->n);
    CK(ctx, cudaGetLastError());
  }
  CK(ctx, cudaStreamSynchronize(s));
  if (t) ctx->t = *t;
  return ASAGA_OK;
}

asaga_status asaga_get_profile(asaga_ctx* ctx, int32_t* counts, double* D) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  cudaStream_t s = ctx->stream;
  if (counts)
    CK(ctx, cudaMemcpyAsync(counts, ctx->counts, sizeof(int32_t) * ctx->d, cudaMemcpyDeviceToHost, s));
  if (D) CK(ctx, cudaMemcpyAsync(D, ctx->D, sizeof(double) * ctx->d, cudaMemcpyDeviceToHost, s));
  CK(ctx, cudaStreamSynchronize(s));
  return ASAGA_OK;
}

asaga_status asaga_get_sample_counts(asaga_ctx* ctx, int32_t* visits, int reset) {
  if (!ctx || !visits) return fail(ctx, ASAGA_E_INVALID_ARG, "NULL argument");
  if (!ctx->visits) return fail(ctx, ASAGA_E_STATE, "context was created without record_samples");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  CK(ctx, cudaMemcpyAsync(visits, ctx->visits, sizeof(int32_t) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
  if (reset) CK(ctx, cudaMemsetAsync(ctx->visits, 0, sizeof(int32_t) * ctx->n, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  return ASAGA_OK;
}

asaga_status asaga_get_sample_hash(asaga_ctx* ctx, uint64_t* hash, int reset) {
  if (!ctx || !hash) return fail(ctx, ASAGA_E_INVALID_ARG, "NULL argument");
  if (!ctx->shash) return fail(ctx, ASAGA_E_STATE, "context was created without record_samples");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  unsigned long long h = 0;
  CK(ctx, cudaMemcpyAsync(&h, ctx->shash, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  if (reset) CK(ctx, cudaMemsetAsync(ctx->shash, 0, sizeof(h), ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  *hash = (uint64_t)h;
  return ASAGA_OK;
}

asaga_status asaga_set_gamma(asaga_ctx* ctx, double gamma) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  if (!(gamma > 0.0) || !std::isfinite(gamma))
    return fail(ctx, ASAGA_E_INVALID_ARG, "gamma must be > 0 (got %g)", gamma);
  ctx->gamma = gamma;
  return ASAGA_OK;
}

asaga_status asaga_set_concurrency(asaga_ctx* ctx, int64_t concurrency) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  if (concurrency < 0) return fail(ctx, ASAGA_E_INVALID_ARG, "concurrency must be >= 0");
  if (ctx->deterministic) return fail(ctx, ASAGA_E_STATE, "deterministic context has concurrency 1");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  ctx->concurrency_opt = concurrency;
  return configure_update(ctx);
}

asaga_status asaga_stats(const asaga_ctx* cctx, asaga_stats_t* out) {
  if (!cctx || !out) return fail(nullptr, ASAGA_E_INVALID_ARG, "NULL argument");
  asaga_ctx* ctx = const_cast<asaga_ctx*>(cctx);  // resolving a pending reload updates L, Delta_r
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));
  out->n = ctx->n;
  out->d = ctx->d;
  out->nnz = ctx->nnz;
  out->lambda = ctx->lambda;
  out->gamma = ctx->gamma;
  out->L = ctx->L;
  out->delta_r = ctx->delta_r;
  out->t = ctx->t;
  out->concurrency = ctx->workers;
  out->lanes_per_sample = ctx->lanes;
  out->deterministic = ctx->deterministic;
  out->max_row = ctx->max_row;
  out->grid = ctx->grid;
  out->block = ctx->block;
  out->last_run_ms = ctx->last_ms;
  out->bulk_scatter_min_freq = ctx->bulk_dmax > 0.0 ? 1.0 / ctx->bulk_dmax : 0.0;
  out->algorithm = ctx->algorithm;
  out->hot_split_min_freq = ctx->hot_dmax > 0.0 ? 1.0 / ctx->hot_dmax : 0.0;
  out->smem_replica = use_replica(ctx) ? 1 : 0;
  out->combine_hot = use_combine(ctx) ? ctx->comb_H : 0;
  out->combine_blocks = use_combine(ctx) ? ctx->grid : 0;
  out->combine_cluster = use_combine(ctx) ? ctx->comb_csize : 0;
  out->record_layout = use_rec(ctx) ? 1 : 0;
  out->hot_table_slots = ctx->hot_tab != nullptr ? 1 << ctx->hot_log : 0;
  out->combine_passes = 0;
  if (use_combine(ctx)) {
    unsigned long long c = 0;
    if (cudaMemcpy(&c, ctx->scratch + ERR_COUNT + 2, sizeof(c), cudaMemcpyDeviceToHost) == cudaSuccess)
      out->combine_passes = (int64_t)c;
  }
  out->overlap_mean = 0.0;
  out->overlap_max = 0;
  out->overlap_samples = 0;
  if (ctx->ov) {
    unsigned long long h[4] = {0, 0, 0, 0};
    if (cudaMemcpy(h, ctx->ov, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess && h[2] > 0) {
      out->overlap_mean = (double)h[1] / (double)h[2];
      out->overlap_max = (int64_t)h[3];
      out->overlap_samples = (int64_t)h[2];
    }
  }
  return ASAGA_OK;
}

asaga_status asaga_sample_indices(int device, uint64_t seed, uint64_t t0, uint64_t count, uint64_t n,
                                  int64_t* out_dev, void* stream) {
  if (!out_dev || n == 0) return fail(nullptr, ASAGA_E_INVALID_ARG, "out_dev NULL or n == 0");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, ASAGA_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  if (count == 0) return ASAGA_OK;
  int grid = (int)std::min<uint64_t>((count + kBlock - 1) / kBlock, 148 * 16);
  sample_kernel<<<grid, kBlock, 0, (cudaStream_t)stream>>>(seed, t0, count, n, out_dev);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(nullptr, ASAGA_E_CUDA, "sample_kernel: %s", cudaGetErrorString(e));
  return ASAGA_OK;
}

asaga_status asaga_debug_sigma(int device, const double* m_dev, double* out_dev, int64_t n, void* stream) {
  if ((!m_dev || !out_dev) && n > 0) return fail(nullptr, ASAGA_E_INVALID_ARG, "NULL buffer");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, ASAGA_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  if (n <= 0) return ASAGA_OK;
  int grid = (int)std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 16);
  sigma_kernel<<<grid, kBlock, 0, (cudaStream_t)stream>>>(m_dev, out_dev, n);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(nullptr, ASAGA_E_CUDA, "sigma_kernel: %s", cudaGetErrorString(e));
  return ASAGA_OK;
}

void* asaga_stream(const asaga_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

const char* asaga_last_error(const asaga_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

const char* asaga_status_string(asaga_status s) {
  switch (s) {
    case ASAGA_OK: return "ASAGA_OK";
    case ASAGA_E_INVALID_ARG: return "ASAGA_E_INVALID_ARG";
    case ASAGA_E_BAD_CSR: return "ASAGA_E_BAD_CSR";
    case ASAGA_E_BAD_LABEL: return "ASAGA_E_BAD_LABEL";
    case ASAGA_E_CUDA: return "ASAGA_E_CUDA";
    case ASAGA_E_OOM: return "ASAGA_E_OOM";
    case ASAGA_E_DIVERGED: return "ASAGA_E_DIVERGED";
    case ASAGA_E_STATE: return "ASAGA_E_STATE";
  }
  return "ASAGA_E_UNKNOWN";
}

asaga_status asaga_set_algorithm(asaga_ctx* ctx, int algorithm) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  if (algorithm != ASAGA_ALG_ASAGA && algorithm != ASAGA_ALG_KROMAGNON && algorithm != ASAGA_ALG_HOGWILD)
    return fail(ctx, ASAGA_E_INVALID_ARG, "unknown algorithm %d", algorithm);
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  ctx->algorithm = algorithm;
  ctx->snapshot_valid = false;
  if (algorithm == ASAGA_ALG_HOGWILD) {  // HOGWILD's memory is identically zero
    CK(ctx, cudaMemsetAsync(ctx->alpha, 0, sizeof(double) * ctx->n, ctx->stream));
    CK(ctx, cudaMemsetAsync(ctx->tmp_d2, 0, sizeof(double) * ctx->d, ctx->stream));
    pack_xa_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, ctx->stream>>>(ctx->xa, ctx->S, ctx->habar,
                                                                              nullptr, ctx->tmp_d2, ctx->d);
    CK(ctx, cudaGetLastError());
    CK(ctx, cudaStreamSynchronize(ctx->stream));
  }
  return ASAGA_OK;
}

asaga_status asaga_snapshot(asaga_ctx* ctx) {
  if (!ctx) return fail(nullptr, ASAGA_E_INVALID_ARG, "ctx is NULL");
  if (ctx->algorithm != ASAGA_ALG_KROMAGNON)
    return fail(ctx, ASAGA_E_STATE, "asaga_snapshot is the KROMAGNON synchronised phase");
  CK(ctx, cudaSetDevice(ctx->device));
  TRY(resolve_pending(ctx));  // an asynchronous reload's validation
  TRY(ensure_csc(ctx));
  cudaStream_t s = ctx->stream;
  // alpha~_i := sigma~_i(x) (folded memory), abar := (1/n) sum_i alpha~_i a~_i
  int xs = 1;
  const double* xcur = current_x(ctx, &xs, s);
  TRY(enqueue_objective(ctx, xcur, xs, ctx->scal, nullptr, true, s));
  CK(ctx, cudaMemcpyAsync(ctx->alpha, ctx->sig, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, s));
  const double lam = ctx->lambda;
  ctx->lambda = 0.0;  // the data part only: colsum adds lambda x, so zero it for this pass
  asaga_status st = enqueue_gradient(ctx, xcur, xs, ctx->tmp_d2, 1, s);
  ctx->lambda = lam;
  TRY(st);
  pack_xa_kernel<<<grid_for(ctx, ctx->d, kBlock), kBlock, 0, s>>>(ctx->xa, ctx->S, ctx->habar, nullptr,
                                                                  ctx->tmp_d2, ctx->d);
  CK(ctx, cudaGetLastError());
  CK(ctx, cudaStreamSynchronize(s));
  ctx->snapshot_valid = true;
  return ASAGA_OK;
}

int asaga_abi_version(void) { return ASAGA_ABI_VERSION; }

#ifdef ASAGA_TIMING
// Profiling build only: read and reset the per-phase cycle sums (not part of asaga.h).
__attribute__((visibility("default"))) int asaga_debug_timing(unsigned long long* out9) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out9, g_phase_cycles, 9 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  unsigned long long z[12] = {0};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  return 0;
}
#endif

void asaga_destroy(asaga_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->l2_persist) {  // give the persisting L2 carve-out this context raised back to the device
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev_ing) cudaEventDestroy(ctx->ev_ing);
  if (ctx->ev_part) cudaEventDestroy(ctx->ev_part);
  if (ctx->h_ing) cudaFreeHost(ctx->h_ing);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  for (auto& h : ctx->hs) {
    if (h.copied) cudaEventDestroy(h.copied);
    if (h.free) cudaEventDestroy(h.free);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

}  // extern "C"
