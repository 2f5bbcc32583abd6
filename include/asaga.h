/*
 * asaga.h -- C-ABI of the B200 ASAGA hot path (libasaga.so).
 *
 * Problem (Leblond, Pedregosa, Lacoste-Julien, arXiv 1606.04809, Section 4.1,
 * PAPER.md:483-486):
 *     min_x f(x) = (1/n) sum_i log(1 + exp(-b_i a_i^T x)) + (lambda/2) ||x||^2
 * solved by Sparse SAGA (Eq. 3) with the exact l2 term of
 * Section 4.2, run as ASAGA (Algorithm 2):
 * per sampled row i, with D_v = n / n_v,
 *     dalpha = f_i'(x^) - alpha^_i                      (scalar memory, App. E)
 *     x_v    += -gamma (dalpha a_iv + D_v abar^_v + lambda D_v x^_v)   v in S_i
 *     alpha_i += dalpha ;  abar_v += dalpha a_iv / n                   v in S_i
 * with lock-free, unsynchronised reads and atomic coordinate adds
 * (Property 3).
 *
 * Conventions for every entry point:
 *  - Host pointers are caller-owned and only borrowed for the duration of the
 *    call unless stated otherwise.  "_dev" pointers are device pointers on the
 *    context's device.  The library never frees caller memory.
 *  - All floating point is IEEE fp64; indices are 0-based int32; row pointers int64.
 *  - Every function returns an asaga_status; no C++ exception crosses the ABI.
 *    After a failure asaga_last_error(ctx) (or asaga_last_error(NULL) when no
 *    context exists, e.g. a failed asaga_init) returns a message naming the
 *    offending row where one exists.
 *  - One context per device per host thread; a context is not thread-safe.
 *  - Blocking calls synchronise the context's stream before returning;
 *    "_async" / "_device" calls only enqueue work on it.
 */
#ifndef ASAGA_H
#define ASAGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASAGA_ABI_VERSION 3

#if defined(__GNUC__)
#define ASAGA_API __attribute__((visibility("default")))
#else
#define ASAGA_API
#endif

typedef struct asaga_ctx asaga_ctx;

/* The update rule run by asaga_run (NEXT-2: the paper's comparison methods, Section
 * 4.3 PAPER.md:539-546, on the same kernel).  All three share the D_i-projected
 * l2 term of Section 4.2 (reading R21). */
typedef enum {
  ASAGA_ALG_ASAGA = 0,     /* Algorithm 2 (default) */
  ASAGA_ALG_KROMAGNON = 1, /* sparse SVRG: inner steps use the memory frozen at the last
                              asaga_snapshot (alpha_i = sigma_i(x~), abar = data gradient) */
  ASAGA_ALG_HOGWILD = 2    /* sparse SGD: memory frozen at zero */
} asaga_algorithm;

typedef enum {
  ASAGA_OK = 0,
  ASAGA_E_INVALID_ARG = 1, /* NULL pointer, lambda <= 0, gamma <= 0, n or d out of range */
  ASAGA_E_BAD_CSR = 2,     /* indptr not monotone / not ending at nnz, empty row,
                              index out of [0,d), indices not strictly increasing in a row,
                              non-finite value (rows must be non-empty: SPEC S:24-27) */
  ASAGA_E_BAD_LABEL = 3,   /* some y_i not in {-1, +1} (b_i in {-1,+1}) */
  ASAGA_E_CUDA = 4,        /* a CUDA runtime error (message carries cudaGetErrorString) */
  ASAGA_E_OOM = 5,         /* device allocation failed */
  ASAGA_E_DIVERGED = 6,    /* non-finite iterate after asaga_run (divergence guard) */
  ASAGA_E_STATE = 7        /* call not valid in the context's state (e.g. no sample record) */
} asaga_status;

/* A CSR matrix: row i holds indices[indptr[i] .. indptr[i+1]) (strictly
 * increasing, each in [0, d)) with values data[...]; indptr has n+1 entries,
 * indptr[0] = 0, indptr[n] = nnz.  The support S_i of f_i is the set of
 * stored entries of row i (reading R3). */
typedef struct {
  int64_t n, d, nnz;
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
} asaga_csr_view;

typedef struct {
  int device;            /* CUDA device ordinal (default 0) */
  int deterministic;     /* 1: a single sample in flight, updates applied in t order; the
                            iterate then equals sequential Sparse SAGA (tau = 1). Default 0. */
  int64_t concurrency;   /* async mode: number of samples in flight (the paper's number of
                            cores p; overlap tau >= p - 1).  0 = auto
                            (every resident worker of the update kernel). */
  int lanes_per_sample;  /* lanes of a warp that cooperate on one sample: 8, 16 or 32;
                            0 = auto from the mean row length */
  int atomic_mode;       /* 1 (default): red.global.add.f64 coordinate adds (Property 3).
                            0: plain load + store (lost updates; test-only ablation of
                            App. E "non-thread safe") */
  int record_samples;    /* 1: count visits per row (int32[n]) to check the sample stream */
  void* stream;          /* cudaStream_t to run on (e.g. torch's current stream);
                            NULL = a stream owned by the context */
  double bulk_scatter_min_freq; /* features present in at least this fraction of rows
                            (p_v >= it) are updated with one TMA bulk 16-byte reduction of
                            the {x_v, abar_v} pair instead of two red.global.add.f64: one L2
                            operation on the feature's line instead of two (the hot line is
                            the throughput bound), at a higher issue latency.  0 (default) =
                            never; 1e-300 = always.  Same arithmetic either way. */
  int measure_overlap;   /* k > 0: estimate the overlap tau (App. D): a
                            sparse global counter is advanced by 100 per 100 updates of each
                            worker, and every k-th sample of a worker records the counter's
                            advance between its read and its write; mean / max in
                            asaga_stats.  0 (default) = off (no counter traffic). */
  double hot_split_min_freq; /* features present in at least this fraction of rows keep
                            abar_v in a separate array, so x_v and abar_v sit on different L2
                            lines: each line then takes 2 operations per update (load + RED)
                            instead of 3; one extra 8-byte gather per such entry.  0 (default)
                            = off.  Exclusive with bulk_scatter_min_freq (ASAGA_E_INVALID_ARG). */
  int smem_replica_refresh; /* r > 0 and d <= 4096, async mode: every thread block keeps a
                            shared-memory replica of all {x_v, abar_v}; gathers read it, writes
                            still go to the shared state, and each worker refreshes G replica
                            entries from L2 every r samples.  Reads become older but stay
                            bounded-delay inconsistent reads (Assumption 1).
                            0 (default) = off. */
  double combine_min_freq;  /* f > 0, async mode: features present in at least this fraction
                            of rows (p_v >= f; at most 4096 of them, else ASAGA_E_INVALID_ARG at
                            ingest) are combined per thread block: workers read a shared-memory
                            replica of {x_v, abar_v} and add into a block-local pending pair;
                            one warp per block sends the pending adds to the shared state
                            (red.global.add.f64) and refreshes the replica, continuously.  The
                            shared state then takes one add per hot feature per block per pass
                            instead of one per sample.  Reads stay bounded-delay inconsistent
                            reads (Assumption 1; reading R23); every
                            add reaches the shared state before asaga_run returns.  Exclusive with
                            the bulk scatter, hot split and replica options.  0 (default) = off;
                            1e-300 = every used feature (small d). */
  int combine_cluster;   /* combining: thread blocks per cluster (1..8; 0 = 8).  The blocks of
                            a cluster share one communication pass over distributed shared
                            memory, so the shared state takes one add per hot feature per
                            CLUSTER per pass. */
  int combine_write_through; /* combining: 1 = the hot features' replica is kept for READS only;
                            every add goes straight to the shared state (red.global.add.f64),
                            so the hot lines lose their per-update loads but no add is held
                            back.  0 (default) = adds are combined per block. */
  int combine_max_blocks; /* combining: at most this many thread blocks (replicas), >= 0; the
                            samples in flight are packed into fewer, fuller blocks so each
                            communication pass carries more combined adds.  0 (default) = one
                            block per SM (per resident cluster slot). */
  int l2_persist_state;  /* 1: the plain update kernel is launched with an L2 access-policy
                            window marking the {x, abar} pair array persisting (up to the
                            device's persisting carve-out, which this raises for the process;
                            SURVEY 8(d) M6).  0 (default) = off. */
  double pipe_late_min_freq; /* > 0: the PIPELINED update kernel (async ASAGA with the plain
                            layout; long rows): features present in at least this fraction of
                            rows are read as late and written as early as the sample's
                            dependency chain allows, the other (cold) entries of the next row are
                            gathered one sample ahead and their adds issued while the next
                            sample's hot reads are in flight (reading R24: a bounded
                            extra overlap on rarely shared coordinates).  Same arithmetic; with
                            deterministic = 1 the same kernel runs sequentially.  A value above
                            1 defers every entry.  0 (default) = the plain kernel. */
  int pipe_merge_ns;     /* with pipe_late_min_freq > 0 (async): k > 0 = the adds to the hot
                            features (p_v >= pipe_late_min_freq, at most 512 of them) are summed
                            in the thread block's shared memory and sent to the shared state by
                            its communication warp every k ns, one red.global.add.f64 per
                            coordinate per block and flush; reads stay fresh (DESIGN.md reading
                            R25: an add reaches the shared state up to ~k ns later).  0 (default)
                            = every sample adds on its own.  At most 1e6. */
  int row_copy_elementwise; /* plain update kernel's row staging: 0 (default) = 1-D TMA bulk
                            copies (cp.async.bulk, completing on an mbarrier; three per row,
                            issued by one lane) when the column / value / D arrays are 16-B
                            aligned, else per-element cp.async; 1 = always per-element cp.async.
                            Same data, same arithmetic. */
  int record_layout;     /* plain update kernel (REDs, no replica): 1 = the record layout -- each
                            coordinate is a 32-byte record {x_v, abar_v, D_v, .} (D_v = n/n_v,
                            PAPER.md:108-110) and the gather of an entry returns D_v with x and
                            abar from the same sector: no per-entry D array (nnz x 8 bytes) and
                            no expand pass per reload; the hot split's features are found in a
                            per-block shared-memory table.  The record is gathered with one
                            256-bit load and, without the hot split, scattered with the paired
                            reductions: c3's operating point; slower on c4,
                            whose 3.2M records (103 MB) crowd the L2.
                            0 (default) = D_{c_k} streamed with the row from a per-entry copy.
                            Same arithmetic. */
  int scatter_unpaired;  /* plain update kernel (REDs, default layout): 0 (default) = paired
                            scatter -- partner lanes g, g^1 each add x of their own entry and
                            abar of the partner's, so ONE reduction instruction carries both
                            words of one {x, abar} pair (one 32-byte sector: L2 serves them as
                            one request); 1 = one instruction per word (x, then abar).  Same
                            adds, same values. */
  int d_gather;          /* plain update kernel (REDs, default layout, no hot split, no replica):
                            1 = D_c = n/n_c is gathered from the d-vector (read-only path) with
                            each entry's coordinate gather, so there is no per-entry D array
                            (nnz x 8 bytes) and no expand pass per reload (c4's operating point).
                            Ignored where it does not apply (record layout, hot split, replica,
                            combine or pipelined kernel).  0 (default) = D_c streamed with the
                            row from the per-entry copy.  Same arithmetic. */
} asaga_options;

typedef struct {
  int64_t n, d, nnz;
  double lambda, gamma;
  double L;               /* max_i ||a_i||^2 / 4 + lambda (reading R7) */
  int64_t delta_r;        /* max_v n_v (Section 3.4 sparsity measure) */
  uint64_t t;             /* global update counter: next update uses sample i_t */
  int64_t concurrency;    /* samples in flight used by the last asaga_run */
  int lanes_per_sample;
  int deterministic;
  int64_t max_row;        /* longest row */
  int grid, block;        /* launch shape of the update kernel */
  double last_run_ms;     /* device time of the last blocking asaga_run (CUDA events) */
  double bulk_scatter_min_freq;
  double overlap_mean;    /* measure_overlap: mean per-sample overlap estimate since ingest */
  int64_t overlap_max;    /* ... and the largest one */
  int64_t overlap_samples;
  int algorithm;          /* asaga_algorithm */
  double hot_split_min_freq;
  int smem_replica;       /* 1 when the shared-memory replica is in use */
  int combine_hot;        /* number of features combined per block (0 = combining off) */
  int combine_blocks;     /* thread blocks (replicas) of the combine kernel */
  int64_t combine_passes; /* communication-warp passes, summed over blocks, of the last run
                             (pass period = last_run_ms * combine_blocks / combine_passes) */
  int combine_cluster;    /* blocks per cluster of the combine kernel */
  int record_layout;      /* 1 when asaga_run uses the record layout (option record_layout, the
                             plain kernel with REDs and no replica) */
  int hot_table_slots;    /* the record layout's hot-split table (0 = none) */
} asaga_stats_t;

/* Fill *opt with the defaults listed above. */
ASAGA_API void asaga_options_default(asaga_options* opt);

/* Copy a HOST CSR matrix and labels y[n] (each +-1) to the device, validate it
 * (see ASAGA_E_BAD_CSR / _BAD_LABEL), and run the column-frequency pass: n_v, D_v = n/n_v
 * (0 when n_v = 0), Delta_r, L (Section 2).  State
 * starts at x = 0, alpha = 0, abar = 0, t = 0 (reading R1).  On success *out
 * owns all device memory; on failure *out = NULL. */
ASAGA_API asaga_status asaga_init(asaga_ctx** out, const asaga_csr_view* A, const double* y,
                        double lambda, double gamma, const asaga_options* opt);

/* As asaga_init, but A's three arrays and y are DEVICE pointers (e.g. torch
 * tensors).  They are BORROWED, not copied: the context reads them (never writes)
 * until the work enqueued before the next reload has completed on the context's stream
 * (asaga_stream), or asaga_destroy, so the caller keeps them allocated and unchanged
 * until then (a reload returns before earlier asaga_run_async work is done: order the
 * arrays' release after an event recorded on asaga_stream, as the Python binding does).  Validation runs on the device.  (The labels are applied per
 * sample and per row in the kernels -- a~_i = b_i a_i is never materialised -- so an
 * ingest moves the matrix once, read-only.) */
ASAGA_API asaga_status asaga_init_device(asaga_ctx** out, const asaga_csr_view* A_dev,
                               const double* y_dev, double lambda, double gamma,
                               const asaga_options* opt);

/* Re-ingest a new matrix of the SAME shape (n, d, nnz) into an existing
 * context, reusing its device memory: HOST arrays (asaga_reload; copied into the
 * context's own device arrays) or DEVICE arrays (asaga_reload_device; borrowed as
 * in asaga_init_device, in place of the previous ones).  Runs A0-A1 again and resets the state to
 * x = 0, alpha = 0, abar = 0, t = 0.  Errors as asaga_init; a different shape
 * gives ASAGA_E_INVALID_ARG.  Blocking (the validation result is read back).
 * REJECTED DATA: after a reload (blocking or asynchronous) fails validation, every call
 * that would launch a kernel on the matrix -- asaga_run[_async], asaga_objective[_device],
 * asaga_full_grad, asaga_partial_obj_grad, asaga_snapshot -- returns ASAGA_E_STATE until
 * a reload succeeds, and the device-side run guard is closed, so no update kernel reads
 * the rejected arrays. */
ASAGA_API asaga_status asaga_reload(asaga_ctx* ctx, const asaga_csr_view* A, const double* y);
ASAGA_API asaga_status asaga_reload_device(asaga_ctx* ctx, const asaga_csr_view* A_dev,
                                           const double* y_dev);

/* As asaga_reload_device, but NON-blocking: A0-A1 are enqueued on the context's stream
 * and the call returns at once (x = 0, alpha = 0, abar = 0, t = 0 as above); the
 * arrays are borrowed as in asaga_init_device.  The
 * validation is read back by the next BLOCKING call on the context (asaga_run,
 * asaga_objective[_device], asaga_get_state, asaga_stats, ...), which returns its error
 * (ASAGA_E_BAD_CSR / _BAD_LABEL with the row, as asaga_reload would).  Until then every
 * asaga_run_async launch is guarded on the device: it does nothing unless the new data is
 * valid and fits the context's launch shape (same longest-row capacity, same hot set);
 * if it did not fit, the resolving call returns ASAGA_E_STATE and those runs must be
 * repeated.  Without a previous successful ingest it behaves as asaga_reload_device. */
ASAGA_API asaga_status asaga_reload_device_async(asaga_ctx* ctx, const asaga_csr_view* A_dev,
                                                 const double* y_dev);

/* As asaga_reload, but NON-blocking: the HOST arrays are copied on the context's own copy
 * stream into one of two device buffers used in turn, so the copy of the next matrix runs
 * while the compute stream still works on the previous one (page-locked host memory is
 * needed for the copy to be asynchronous; pageable memory works but the copy then blocks
 * the caller).  The caller keeps the host arrays unchanged until the next blocking call.
 * Validation, the run guard and ASAGA_E_STATE are as in asaga_reload_device_async; without
 * a previous successful ingest it behaves as asaga_reload. */
ASAGA_API asaga_status asaga_reload_async(asaga_ctx* ctx, const asaga_csr_view* A, const double* y);

/* Process the global update counters t = t0 .. t0+n_updates-1 (t0 = the
 * context's counter, then t0 += n_updates).  Update t uses row
 * i_t = floor(r_t * n / 2^64), r_t = the first two 32-bit words of
 * Philox4x32-10(counter = (lo32 t, hi32 t, 0, 0), key = (lo32 seed, hi32 seed))
 * (reading R2), so run(T1); run(T2) processes the same samples as run(T1+T2),
 * and in deterministic mode yields the same iterate.  Blocks until done and
 * then checks x for non-finite values (ASAGA_E_DIVERGED). */
ASAGA_API asaga_status asaga_run(asaga_ctx* ctx, uint64_t n_updates, uint64_t seed);

/* Enqueue the same work on the context's stream and return immediately
 * (no divergence check, last_run_ms not updated). */
ASAGA_API asaga_status asaga_run_async(asaga_ctx* ctx, uint64_t n_updates, uint64_t seed);

/* f(x) (Section 4.1 objective, full lambda/2 ||x||^2).  x: HOST d-vector, or NULL
 * for the current iterate.  Blocking. */
ASAGA_API asaga_status asaga_objective(asaga_ctx* ctx, const double* x, double* f_out);

/* grad f(x) = (1/n) sum_i sigma_i(x) a_i + lambda x, sigma_i = -b_i/(1+exp(b_i a_i.x))
 * (gradient of Eq. 1 with the l2 term).  x: HOST d-vector or NULL (current
 * iterate); g_out: HOST d-vector.  Blocking.  The first call builds a
 * column-major copy of A on the device (deterministic summation order). */
ASAGA_API asaga_status asaga_full_grad(asaga_ctx* ctx, const double* x, double* g_out);

/* Enqueue f(x) for DEVICE x (NULL = current iterate) into DEVICE *f_dev. */
ASAGA_API asaga_status asaga_objective_device(asaga_ctx* ctx, const double* x_dev, double* f_dev);

/* Row-shard partial of the objective/gradient for a context built on a block
 * of rows: out_dev[0..d) = sum_{i in shard} sigma_i(x) a_i and
 * out_dev[d] = sum_{i in shard} log(1+exp(-b_i a_i.x)) (no 1/n, no lambda).
 * x_dev, out_dev: DEVICE pointers; enqueued on `stream` (NULL = context
 * stream).  Summing the outputs of all shards (an all-reduce) and then
 * f = out[d]/n + lambda/2 ||x||^2, grad = out[:d]/n + lambda x gives the full
 * objective and gradient. */
ASAGA_API asaga_status asaga_partial_obj_grad(asaga_ctx* ctx, const double* x_dev, double* out_dev,
                                    void* stream);

/* Copy the state to HOST buffers (any may be NULL): x[d], alpha[n] (the
 * paper's alpha_i, i.e. labels unfolded), alpha_bar[d], t. */
ASAGA_API asaga_status asaga_get_state(asaga_ctx* ctx, double* x, double* alpha, double* alpha_bar,
                             uint64_t* t);

/* Overwrite the state from HOST buffers (NULL leaves that part unchanged). */
ASAGA_API asaga_status asaga_set_state(asaga_ctx* ctx, const double* x, const double* alpha,
                             const double* alpha_bar, const uint64_t* t);

/* Column profile to HOST buffers (either may be NULL): counts[d] = n_v, D[d] = D_v. */
ASAGA_API asaga_status asaga_get_profile(asaga_ctx* ctx, int32_t* counts, double* D);

/* Per-row visit counts (HOST int32[n]) since init or the last reset; needs
 * options.record_samples = 1, else ASAGA_E_STATE. reset != 0 zeroes them after the copy. */
ASAGA_API asaga_status asaga_get_sample_counts(asaga_ctx* ctx, int32_t* visits, int reset);

/* Checksum of the processed sample stream itself (the t -> i_t map, not only the per-row
 * histogram): *hash = sum over every processed update t of mix(t, i_t) mod
 * 2^64, mix(t, i) = splitmix64's finaliser applied to t * 0x9E3779B97F4A7C15 + i (z ^= z>>30;
 * z *= 0xBF58476D1CE4E5B9; z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31), since init /
 * the last ingest / the last reset.  Sampling rule: Alg. 2 line 3 under reading
 * R2.  Needs options.record_samples = 1, else ASAGA_E_STATE.  reset != 0 zeroes it. */
ASAGA_API asaga_status asaga_get_sample_hash(asaga_ctx* ctx, uint64_t* hash, int reset);

/* Select the update rule (asaga_algorithm).  Switching to HOGWILD zeroes alpha and abar
 * (its memory is identically 0); switching to KROMAGNON requires asaga_snapshot()
 * before the next run (ASAGA_E_STATE otherwise).  x is kept. */
ASAGA_API asaga_status asaga_set_algorithm(asaga_ctx* ctx, int algorithm);

/* KROMAGNON's synchronised phase (Mania et al.): at the current x,
 * alpha_i := sigma_i(x) for every i and abar := (1/n) sum_i alpha_i a_i (one row pass,
 * one column pass), then the inner steps of asaga_run read this frozen memory.
 * Blocking.  ASAGA_E_STATE unless the algorithm is KROMAGNON. */
ASAGA_API asaga_status asaga_snapshot(asaga_ctx* ctx);

/* Change the step size gamma (> 0) for subsequent runs. */
ASAGA_API asaga_status asaga_set_gamma(asaga_ctx* ctx, double gamma);

/* Change the number of samples in flight (async mode; 0 = auto). */
ASAGA_API asaga_status asaga_set_concurrency(asaga_ctx* ctx, int64_t concurrency);

ASAGA_API asaga_status asaga_stats(const asaga_ctx* ctx, asaga_stats_t* out);

/* The sampler alone: out_dev[k] = i_{t0+k} for n rows (same map as asaga_run),
 * DEVICE int64 buffer of `count` entries, enqueued on `stream` (NULL = default
 * stream of `device`). */
ASAGA_API asaga_status asaga_sample_indices(int device, uint64_t seed, uint64_t t0, uint64_t count,
                                  uint64_t n, int64_t* out_dev, void* stream);

/* The scalar derivative alone (A5; Alg. 2 lines 6-8, folded logistic
 * PAPER.md:483-485): out_dev[k] = -1 / (1 + exp(m_dev[k])) as the update kernels compute it
 * (fp64, a few ulp), for n DEVICE doubles, enqueued on `stream` (NULL = default stream of
 * `device`).  A test hook: the kernels use the same device function. */
ASAGA_API asaga_status asaga_debug_sigma(int device, const double* m_dev, double* out_dev, int64_t n,
                                         void* stream);

/* Device pointer of the context's stream (cudaStream_t). */
ASAGA_API void* asaga_stream(const asaga_ctx* ctx);

/* Message for the last failure on ctx (or the calling thread's last failure
 * outside a context when ctx == NULL).  Never NULL; valid until the next call. */
ASAGA_API const char* asaga_last_error(const asaga_ctx* ctx);

ASAGA_API const char* asaga_status_string(asaga_status s);

ASAGA_API int asaga_abi_version(void);

/* Free all device memory of ctx (NULL-safe). */
ASAGA_API void asaga_destroy(asaga_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* ASAGA_H */
