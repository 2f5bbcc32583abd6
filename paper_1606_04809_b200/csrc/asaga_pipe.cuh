// asaga_pipe.cuh -- A2..A8 for long-row data (c3, c4): the pipelined update kernel.
//
// Same method as asaga_update_kernel (Algorithm 2, with the Section 4.2 l2
// term P:519-522; folded labels, reading R9 atomic alpha), same t -> worker map (worker w
// processes t = t0 + w + kW), same arithmetic per entry.  What changes is WHEN each read
// and write of a sample happens, so that the window between reading a POPULAR ("hot")
// coordinate and writing it back is as short as the dependency chain allows:
//
//   iteration m of a worker (G lanes, NR register chunks of the row):
//     1. gathers of row m's HOT entries (|D_v| <= late_dmax: features in >= 1/late_dmax of
//        the rows) and alpha^_i                                   (Alg. 2 lines 5-8, read)
//     2. the deferred COLD scatter of sample m-1                  (lines 9-13, write)
//     3. copy of the row of sample m+3 (cp.async, 4 stages) + bounds of m+5 (ring)
//     4. dot over row m (hot values just loaded, cold ones loaded one iteration ago),
//        q_v = D_v (abar^_v + lambda x^_v) per entry
//     5. sigma~, dalpha
//     6. HOT scatter of sample m + alpha_i add                      (write)
//     7. D_v of row m+1 (loaded one iteration earlier) into its stage, gathers of row
//        m+1's COLD entries (their values arrive during iteration m+1's steps 1-3, so an L2
//        miss on a rarely used feature is off the critical path), then the loads of D_v for
//        row m+2 (read-only during a run: __ldg, L1-cached for the popular features)
//
// D_v is gathered from the d-vector in the kernel, two samples ahead, instead of streamed
// per stored entry: no expand pass over the matrix, and the row stream is the algorithmic
// 12 B per entry.
// Every read is still an unsynchronised read of the shared state and
// every write an atomic add (Property 3), so an execution is an ASAGA run with a
// bounded overlap (Assumption 1): a cold coordinate is read about one
// iteration earlier and written about one iteration later than in the plain kernel
// (reading R24) -- harmless for features that few in-flight samples share --
// while a hot coordinate's read-to-write window shrinks to steps 1-6.  Throughput is
// W / (iteration time), and ASAGA's convergence caps the overlap on the hot coordinates
// (profiles/r01_operating_point.md), so shortening both is what raises the update rate.
//
// DET = true: one worker, no deferral (every gather of row m at step 1, every write at
// step 6, a gpu-scope fence between samples): sequential Sparse SAGA computed by this
// kernel's own expressions, for exact parity against the oracle.
//
// CMB = true (option pipe_merge_ns, async only): at step 6 a worker adds its HOT entries'
// {dx, dabar} into ITS OWN row of the block's table in shared memory (feature -> position
// by a shared-memory hash of the hot set; plain loads and stores, no atomics: a row has
// one writer and only grows), and every merge_ns nanoseconds the block's communication
// warp sends, per position, the growth of every worker row since its previous look (row
// value minus the value it last sent, kept in its own array) to L2 with one
// red.global.add.f64 per coordinate.  (Shared f64 atomicAdd is a CAS loop on sm_100a:
// the first version, one shared pending sum per position, spent ~3k cycles per sample in
// those loops.)  Reads stay fresh
// loads from L2 (steps 1 and 7): only the hot ADDS wait, by at most one flush period plus
// the pass, in the block before they reach the shared state -- an iteration counted "in
// progress to the end of the writing of its update" (Assumption 1), so the
// overlap grows by about the updates of one period (reading R25) -- while each
// hot line takes one RED per block per flush instead of one per sample.  (Measured on c4:
// the REDs on the popular features' x lines, together with their per-sample loads, cap the
// plain kernel at ~1.5e8 updates/s whatever the number in flight; without them the rate
// grows with it -- profiles/r02_update_kernel.md.)  A synchronous variant (block rounds,
// merged at a barrier) measured 2.5x slower: every round waits for its slowest sample.
#pragma once

namespace asaga {

template <int G, int NR>
struct PipeSmem {
  static constexpr int P = NR * G;
  static constexpr int KS = 4;  // row stages: the row of sample m+3 is copied at iteration m
  // stage: P fp64 values, P fp64 D (filled in the kernel; negative: hot split), P int32
  // columns, then b_i
  static constexpr size_t label_off = (size_t)P * (2 * sizeof(double) + sizeof(int32_t));
  static constexpr size_t stage_bytes = (label_off + 16 + 15) & ~(size_t)15;
  // bounds ring {lo, hi, i, -}: the bounds of sample m+5 are fetched at iteration m
  static constexpr int NB = 8;
  static constexpr int BA = 5;  // bounds fetched BA samples ahead
  static constexpr size_t ring_off = KS * stage_bytes;
  static constexpr size_t ring_bytes = NB * 32;
  static constexpr size_t q_off = ring_off + ring_bytes;
  static __host__ __device__ size_t bytes(int overflow) {
    return (q_off + (size_t)overflow * sizeof(double) + 15) & ~(size_t)15;
  }
};

template <int G, int NR>
__device__ __forceinline__ void pipe_row_copy(unsigned char* gbase, int stage, const int32_t* cols,
                                              const double* vals, const double* b_i,
                                              int64_t lo, int64_t hi, int g, uint64_t pol) {
  using SM = PipeSmem<G, NR>;
  constexpr int P = SM::P;
  unsigned char* sb = gbase + stage * SM::stage_bytes;
  double* sv = reinterpret_cast<double*>(sb);
  int32_t* sc = reinterpret_cast<int32_t*>(sv + 2 * P);
  if (g == 0) cp_async8(sb + SM::label_off, b_i);
  const int len = (int)(hi - lo);
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    if (j * G >= len) break;  // group-uniform
    const int64_t k = lo + j * G + g;
    if (j * G + g < len) {
      cp_async4_ef(sc + j * G + g, cols + k, pol);
      cp_async8_ef(sv + j * G + g, vals + k, pol);
    }
  }
}

// CMB: the per-block merge table after the worker groups' blocks (asaga.cu sizes it):
// keys[TS] (feature, -1 empty), home[TS] (1: abar in habar), acc[groups][TS] {dx, dabar}
// (each worker's running sums), sent[groups][TS] (what the communication warp has sent of
// them), and the count of finished worker groups; the block's last warp communicates
__device__ __forceinline__ unsigned hot_hash(int v) { return (unsigned)v * 2654435761u; }

template <int G, int NR, bool DET, bool CMB>
__global__ void __launch_bounds__(256, 1) asaga_pipe_kernel(UpdateParams p) {
  if (p.ok != nullptr && *reinterpret_cast<const volatile int*>(p.ok) == 0) return;  // run guard
  using SM = PipeSmem<G, NR>;
  constexpr int P = SM::P;
  constexpr int KS = SM::KS, NB = SM::NB, BA = SM::BA;
  static_assert(G >= 8, "a Philox batch covers the prologue's samples 0..BA-1");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int g = lane & (G - 1);
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (unsigned)(lane & ~(G - 1)));
  const int ngrp = CMB ? (int)(blockDim.x - 32) / G : (int)blockDim.x / G;  // worker groups
  const int grp = threadIdx.x / G;
  const bool comm_warp = CMB && (int)threadIdx.x >= ngrp * G;  // the block's last warp
  const int64_t w = (int64_t)grp * gridDim.x + blockIdx.x;  // round robin (launch_shape)
  const uint64_t tend = p.t0 + p.T;
  const uint64_t W = (uint64_t)p.workers;
  const uint64_t t_first = p.t0 + (uint64_t)w;
  const bool active = grp < ngrp && w < p.workers && t_first < tend;
  const int TS = CMB ? p.merge_ts : 0;
  int32_t* mkey = reinterpret_cast<int32_t*>(smem_raw + (size_t)ngrp * SM::bytes(p.overflow));
  int32_t* mhome = mkey + TS;
  double2* macc = reinterpret_cast<double2*>(mhome + TS);  // [ngrp][TS], 16-B aligned (TS >= 4)
  double2* msent = macc + (size_t)ngrp * TS;                // [ngrp][TS]
  int* mdone = reinterpret_cast<int*>(msent + (size_t)ngrp * TS);
  if (CMB) {
    for (int k = threadIdx.x; k < TS; k += blockDim.x) {
      mkey[k] = -1;
      mhome[k] = 0;
    }
    for (int k = threadIdx.x; k < ngrp * TS; k += blockDim.x) {
      macc[k] = make_double2(0.0, 0.0);
      msent[k] = make_double2(0.0, 0.0);
    }
    if (threadIdx.x == 0) *mdone = 0;
    __syncthreads();
    for (int s = threadIdx.x; s < p.H; s += blockDim.x) {  // insert the hot set (linear probing)
      const int v = p.hot_id[s];
      unsigned h = hot_hash(v) & (unsigned)(TS - 1);
      while (atomicCAS(&mkey[h], -1, v) != -1) h = (h + 1) & (unsigned)(TS - 1);
      mhome[h] = (p.split && __ldg(p.D + v) <= p.hot_dmax) ? 1 : 0;
    }
    __syncthreads();
    if (comm_warp) {
      // ---------------- communication warp: flush the pending sums every merge_ns
      const int lane_c = threadIdx.x & 31;
      auto flush = [&]() {
        for (int k = lane_c; k < TS; k += 32) {
          const int v = mkey[k];
          if (v < 0) continue;
          double dx = 0.0, dy = 0.0;
          for (int q = 0; q < ngrp; ++q) {  // the growth of every worker's running sum
            const volatile double* a = reinterpret_cast<const volatile double*>(macc + (size_t)q * TS + k);
            const double ax = a[0], ay = a[1];
            double2* sp = msent + (size_t)q * TS + k;
            dx += ax - sp->x;
            dy += ay - sp->y;
            *sp = make_double2(ax, ay);
          }
          double* xv = &p.xa[(int64_t)v * p.S].x;
          if (dx != 0.0) red_add(xv, dx);
          if (dy != 0.0) red_add(mhome[k] ? p.habar + v : xv + 1, dy);
        }
      };
      const volatile int* vdone = mdone;
      while (*vdone < ngrp) {
        flush();
        __nanosleep(p.merge_ns);
      }
      __syncwarp();
      flush();  // every worker group has finished its adds
      return;
    }
  }
  if (!active) {  // an unused worker group of the block: counts as finished at once
    if (CMB && (threadIdx.x & (G - 1)) == 0) atomicAdd(mdone, 1);
    return;
  }
  unsigned char* gbase = smem_raw + (size_t)grp * SM::bytes(p.overflow);
  int64_t* ring = reinterpret_cast<int64_t*>(gbase + SM::ring_off);
  double* qs = reinterpret_cast<double*>(gbase + SM::q_off);  // overflow entries' q
  const int nsamp = (int)((tend - t_first + W - 1) / W);  // this worker's samples
  auto mpos = [&](int v) -> int {  // position of a hot feature in the merge table, -1 if absent
    unsigned h = hot_hash(v) & (unsigned)(TS - 1);
    for (int k = 0; k < TS; ++k) {
      const int key = mkey[h];
      if (key == v) return (int)h;
      if (key < 0) return -1;
      h = (h + 1) & (unsigned)(TS - 1);
    }
    return -1;
  };
  const uint64_t pol = policy_evict_first();
  const double ngam = -p.gamma;
  const double late = p.late_dmax;
#ifdef ASAGA_TIMING
  // profiling build only (tools/phase_timing.py --pipe): [0] hot gathers issue, [1] deferred
  // cold scatter, [2] wait + row copy, [3] dot (waits for the gathers), [4] reduce + sigma,
  // [5] iterations, [6] hot scatter, [7] D store + cold gathers issue, [8] wait + D loads
  unsigned long long ph[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#endif

  int64_t bi = 0;  // sample indices in batches of G: lane j draws sample mb + j
  auto draw_batch = [&](int mb) {
    const uint64_t ts = t_first + (uint64_t)(mb + g) * W;
    bi = ts < tend ? sample_row(p.seed, ts, p.n) : 0;
  };
  auto sample_of = [&](int ms) -> int64_t { return __shfl_sync(gmask, bi, ms & (G - 1), G); };
  auto stage_ptr = [&](int k) { return gbase + (k % KS) * SM::stage_bytes; };
  auto fetch_bounds = [&](int k) {  // sample k (< nsamp): {lo, hi, i} into ring slot k % NB
    const int64_t is = sample_of(k);
    if (g == 0) {
      int64_t* slot = ring + 4 * (k % NB);
      slot[2] = is;
      cp_async8(slot, p.rowptr + is);
      cp_async8(slot + 1, p.rowptr + is + 1);
    }
  };
  auto copy_row = [&](int k) {  // sample k (< nsamp), bounds in the ring
    const int64_t* b = ring + 4 * (k % NB);
    pipe_row_copy<G, NR>(gbase, k % KS, p.cols, p.vals, p.y + b[2], b[0], b[1], g, pol);
  };
  // D_v of a staged row: loaded into dd (read-only d-vector), later stored into the stage
  // with the hot split's sign (-D: abar in habar), which the per-entry code reads
  double dd[NR];
  auto load_d = [&](int k) {
    unsigned char* sb = gbase + (k % KS) * SM::stage_bytes;
    const int64_t* b = ring + 4 * (k % NB);
    const int len = (int)(b[1] - b[0]);
    const int32_t* sc = reinterpret_cast<const int32_t*>(reinterpret_cast<const double*>(sb) + 2 * P);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;
      if (j * G + g < len) dd[j] = __ldg(p.D + sc[j * G + g]);
    }
  };
  auto store_d = [&](int k) {
    unsigned char* sb = gbase + (k % KS) * SM::stage_bytes;
    const int64_t* b = ring + 4 * (k % NB);
    const int len = (int)(b[1] - b[0]);
    double* sd = reinterpret_cast<double*>(sb) + P;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;
      if (j * G + g < len) sd[j * G + g] = (p.split && dd[j] <= p.hot_dmax) ? -dd[j] : dd[j];
    }
  };
  auto tail_dv = [&](int c) {  // entries past P (long rows): the same encoding, loaded directly
    const double Dv = __ldg(p.D + c);
    return (p.split && Dv <= p.hot_dmax) ? -Dv : Dv;
  };
  // per-entry accessors of a staged row
  auto sval = [&](unsigned char* sb, int e) { return reinterpret_cast<const double*>(sb)[e]; };
  auto sdv = [&](unsigned char* sb, int e) { return reinterpret_cast<const double*>(sb)[P + e]; };
  auto scol = [&](unsigned char* sb, int e) {
    return reinterpret_cast<const int32_t*>(reinterpret_cast<const double*>(sb) + 2 * P)[e];
  };
  auto gather = [&](int c, double dvv) -> double2 {  // {x^_c, abar^_c} (hot split: abar in habar)
    return (p.split && dvv < 0.0) ? make_double2(ld_na(&p.xa[(int64_t)c * p.S].x), ld_na(p.habar + c))
                                  : ld_na2(p.xa + (int64_t)c * p.S);
  };
  auto scatter = [&](int c, double dvv, double a, double q, double db) {
    double* xv = &p.xa[(int64_t)c * p.S].x;
    double* abv = (p.split && dvv < 0.0) ? p.habar + c : xv + 1;
    red_add(xv, ngam * fma(db, a, q));
    red_add(abv, db * a * p.inv_n);
  };

  double2 xc[NR], xh[NR];
  double qq[NR];
  double qp[NR];  // deferred cold scatter of the previous sample: its q per entry
  double db_prev = 0.0;
  int len_prev = 0;
  int64_t lo_prev = 0;
  unsigned long long shash = 0;
  // ---- prologue: bounds of samples 0..2 (direct), rows 0..2 (groups -3..-1), bounds 3, 4
  draw_batch(0);
  for (int k = 0; k < 3; ++k) {
    if (k < nsamp) {
      const int64_t is = sample_of(k);
      if (g == 0) {
        int64_t* slot = ring + 4 * (k % NB);
        slot[0] = __ldg(p.rowptr + is);
        slot[1] = __ldg(p.rowptr + is + 1);
        slot[2] = is;
      }
    }
  }
  __syncwarp(gmask);
  for (int k = 0; k < 3; ++k) {  // group (k - 3): row k, bounds k + 2 (k >= 1)
    if (k < nsamp) copy_row(k);
    if (k >= 1 && k + 2 < nsamp) fetch_bounds(k + 2);
    cp_async_commit();
  }
  cp_async_wait_group<1>();  // groups -3, -2: rows 0, 1
  __syncwarp(gmask);
  load_d(0);
  store_d(0);
  if (1 < nsamp) load_d(1);
  __syncwarp(gmask);

  // cold and hot gathers land in DIFFERENT registers (xc, xh): a (predicated) load into a
  // register with a load still in flight waits for it (write-after-write on the
  // scoreboard), which made step 1 wait for the previous iteration's cold gathers
  // (measured: 2.6-5.6k cycles at step 1 with one shared array)
  // cold gathers of row 0 (iteration -1's step 7)
  {
    unsigned char* sb = stage_ptr(0);
    const int len0 = (int)(ring[1] - ring[0]);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len0) break;
      const int e = j * G + g;
      if (e < len0) {
        const double dvv = sdv(sb, e);
        if (DET || fabs(dvv) > late) xc[j] = gather(scol(sb, e), dvv);
      }
    }
  }

  for (int m = 0; m < nsamp; ++m) {
    unsigned char* sb = stage_ptr(m);
    const int64_t* cur = ring + 4 * (m % NB);
    const int64_t lo = cur[0], hi = cur[1], i = cur[2];
    const int len = (int)(hi - lo);
    const double yb = *reinterpret_cast<const double*>(sb + SM::label_off);
    // ---- 1. hot gathers of row m (late reads) + alpha^_i
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;  // group-uniform
      const int e = j * G + g;
      if (e < len) {
        const double dvv = sdv(sb, e);
        if (!DET && fabs(dvv) <= late) xh[j] = gather(scol(sb, e), dvv);
      }
    }
    const double ai = ld_na(p.alpha + i);
    TMARK(0);
    // ---- 2. deferred cold scatter of sample m-1 (its stage is still intact)
    if (!DET && m > 0) {
      unsigned char* sp = stage_ptr(m - 1);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= len_prev) break;
        const int e = j * G + g;
        if (e < len_prev) {
          const double dvv = sdv(sp, e);
          if (fabs(dvv) > late) scatter(scol(sp, e), dvv, sval(sp, e), qp[j], db_prev);
        }
      }
    }
    __syncwarp(gmask);  // every lane is done with stage m-1 (= the stage of m+3)
    TMARK(1);
    // ---- 3. row m+3 into the free stage, bounds of m+5 into the ring
    cp_async_wait_group<1>();  // groups up to m-2: row m+1, bounds m+3
    __syncwarp(gmask);
    if (((m + BA) & (G - 1)) == 0 && m + BA < nsamp) draw_batch(m + BA);
    if (m + 3 < nsamp) copy_row(m + 3);
    if (m + BA < nsamp) fetch_bounds(m + BA);
    cp_async_commit();
    (void)lo_prev;
    TMARK(2);
    // ---- 4. dot product and q over row m
    double dot = 0.0;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;
      const int e = j * G + g;
      if (e < len) {
        const double dvv = sdv(sb, e);
        const double2 v = (!DET && fabs(dvv) <= late) ? xh[j] : xc[j];
        dot = fma(sval(sb, e), v.x, dot);
        qq[j] = fabs(dvv) * fma(p.lambda_, v.x, v.y);
      }
    }
    if (len > P)  // group-uniform: long rows, gathered and written at once (no deferral)
      for (int64_t k = lo + P + g; k < hi; k += G) {
        const int c = ld_nc_i32(p.cols + k);
        const double dvv = tail_dv(c);
        const double2 v = gather(c, dvv);
        dot = fma(ld_nc_f64(p.vals + k), v.x, dot);
        qs[k - lo - P] = fabs(dvv) * fma(p.lambda_, v.x, v.y);
      }
    TMARK(3);
    // ---- 5. scalar derivative (folded logistic) and memory difference
    dot = group_sum<G>(dot, gmask) * yb;
    const double da = sigma_folded(dot) - ai;
    const double db = da * yb;
    TMARK(4);
    // ---- 6. hot scatter (every entry in DET) + alpha_i, long-row tail
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len) break;
      const int e = j * G + g;
      if (e < len) {
        const double dvv = sdv(sb, e);
        if (DET || fabs(dvv) <= late) {
          const int c = scol(sb, e);
          const int pos = (CMB && fabs(dvv) <= late) ? mpos(c) : -1;
          if (pos >= 0) {  // this worker's running sum (sent by the communication warp)
            const double a = sval(sb, e);
            volatile double* acc = reinterpret_cast<volatile double*>(macc + (size_t)grp * TS + pos);
            acc[0] = acc[0] + ngam * fma(db, a, qq[j]);
            acc[1] = acc[1] + db * a * p.inv_n;
          } else {
            scatter(c, dvv, sval(sb, e), qq[j], db);
          }
        }
      }
    }
    if (len > P)
      for (int64_t k = lo + P + g; k < hi; k += G) {
        const int c = ld_nc_i32(p.cols + k);
        scatter(c, tail_dv(c), ld_nc_f64(p.vals + k), qs[k - lo - P], db);
      }
    if (g == 0) {
      red_add(p.alpha + i, da);
      if (p.visits) {
        atomicAdd(p.visits + i, 1);
        shash += sample_mix(t_first + (uint64_t)m * W, i);
      }
    }
    if (DET) {
      __threadfence();
      __syncwarp(gmask);
    }
    TMARK(6);
    // this sample's cold adds are issued at the next iteration's step 2
#pragma unroll
    for (int j = 0; j < NR; ++j) qp[j] = qq[j];
    db_prev = db;
    len_prev = len;
    lo_prev = lo;

    // ---- 7. D of row m+1 into its stage, cold gathers of row m+1 (landed: waited for at
    //         step 3), then the D loads of row m+2
    if (m + 1 < nsamp) {
      store_d(m + 1);
      __syncwarp(gmask);
      unsigned char* sn = stage_ptr(m + 1);
      const int64_t* nb = ring + 4 * ((m + 1) % NB);
      const int lenn = (int)(nb[1] - nb[0]);
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j * G >= lenn) break;
        const int e = j * G + g;
        if (e < lenn) {
          const double dvv = sdv(sn, e);
          if (DET || fabs(dvv) > late) xc[j] = gather(scol(sn, e), dvv);
        }
      }
    }
    TMARK(7);
    if (m + 2 < nsamp) {
      cp_async_wait_group<1>();  // groups up to m-1: row m+2
      __syncwarp(gmask);
      load_d(m + 2);
    }
    TMARK(8);
#ifdef ASAGA_TIMING
    ph[5] += 1;
#endif
  }
  // ---- epilogue: the last sample's deferred cold scatter
  if (!DET) {
    unsigned char* sp = stage_ptr(nsamp - 1);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (j * G >= len_prev) break;
      const int e = j * G + g;
      if (e < len_prev) {
        const double dvv = sdv(sp, e);
        if (fabs(dvv) > late) scatter(scol(sp, e), dvv, sval(sp, e), qp[j], db_prev);
      }
    }
  }
  cp_async_wait_all();
  if (p.visits && g == 0) atomicAdd(p.shash, shash);
  if (CMB) {
    __threadfence_block();  // this lane's running sums are visible to the communication warp
    __syncwarp(gmask);
    if (g == 0) atomicAdd(mdone, 1);
  }
#ifdef ASAGA_TIMING
  if (g == 0)
    for (int k = 0; k < 9; ++k) atomicAdd(&g_phase_cycles[k], ph[k]);
#endif
}

}  // namespace asaga
