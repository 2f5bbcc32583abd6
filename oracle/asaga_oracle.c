/*
 * oracle/asaga_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential fp64 CPU implementation of what the ASAGA hot
 * path computes, written from the paper (Leblond, Pedregosa, Lacoste-Julien,
 * "ASAGA: Asynchronous Parallel SAGA", arXiv 1606.04809; /root/reference/PAPER.md,
 * cited below as P:<line>).  It exists to check the CUDA path and nothing else:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load it.  It shares no code, header, table or constant
 * generator with paper_1606_04809_b200/csrc (which has its own Philox, its own
 * index map, its own column-count pass, ...).
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math):
 * every sum is sequential in CSR order.  No blocking, fusion or reordering.
 *
 * Pinned by tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Sampler (reading R2; the paper only says "uniformly at random",
 * P:243).  Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), written
 * out round by round:  one round maps (c0,c1,c2,c3) with key (k0,k1) to
 *   (hi(M1*c2) ^ c1 ^ k0,  lo(M1*c2),  hi(M0*c0) ^ c3 ^ k1,  lo(M0*c0))
 * and the key is bumped by the Weyl constants between rounds.              */
#define ORACLE_PHILOX_M0 0xD2511F53u
#define ORACLE_PHILOX_M1 0xCD9E8D57u
#define ORACLE_PHILOX_W0 0x9E3779B9u
#define ORACLE_PHILOX_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                          uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += ORACLE_PHILOX_W0;
      k1 += ORACLE_PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)ORACLE_PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)ORACLE_PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* i_t = floor(r * n / 2^64), r = (out1 << 32) | out0, counter (lo32 t, hi32 t, 0, 0),
 * key (lo32 seed, hi32 seed).  Uniform on {0..n-1} up to bias n/2^64 (reading R2).
 * "Sample i uniformly at random" happens before any read (Alg. 2 line 3). */
uint64_t oracle_sample_index(uint64_t seed, uint64_t t, uint64_t n) {
  uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), 0u, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  oracle_philox4x32_10(ctr, key, out);
  uint64_t r = ((uint64_t)out[1] << 32) | (uint64_t)out[0];
  unsigned __int128 prod = (unsigned __int128)r * (unsigned __int128)n;
  return (uint64_t)(prod >> 64);
}

/* Raw Philox words for counters (lo32 t, hi32 t, 0, 0), t = t0..t0+count-1. */
void oracle_philox_stream(uint64_t seed, uint64_t t0, uint64_t count, uint32_t* out) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (uint64_t k = 0; k < count; ++k) {
    uint64_t t = t0 + k;
    uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(t >> 32), 0u, 0u};
    oracle_philox4x32_10(ctr, key, out + 4 * k);
  }
}

void oracle_sample_stream(uint64_t seed, uint64_t t0, uint64_t count, uint64_t n,
                          int64_t* out) {
  for (uint64_t k = 0; k < count; ++k) out[k] = (int64_t)oracle_sample_index(seed, t0 + k, n);
}

/* ------------------------------------------------------------------------ */
/* Sparsity profile ("D ... coefficients 1/p_v ... p_v is the
 * probability that dimension v belongs to S_i"; "first pass").
 * n_v = #{i : v in S_i}; S_i = the stored entries of row i (reading R3).   */
void oracle_column_counts(int64_t n, int64_t d, const int64_t* indptr,
                          const int32_t* indices, int64_t* counts) {
  for (int64_t v = 0; v < d; ++v) counts[v] = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) counts[indices[k]] += 1;
}

/* D_v = 1/p_v = n / n_v (IEEE division); D_v = 0 when n_v = 0 (reading R4). */
void oracle_reweight(int64_t n, int64_t d, const int64_t* counts, double* D) {
  for (int64_t v = 0; v < d; ++v)
    D[v] = counts[v] > 0 ? (double)n / (double)counts[v] : 0.0;
}

/* L = max_i ||a_i||^2 / 4 + lambda: the smoothness constant of the logistic f_i
 * plus the l2 term ("L-Lipschitz", Table 1 L=0.25 for normalised RCV1). */
double oracle_lipschitz(int64_t n, const int64_t* indptr, const double* data,
                        double lambda) {
  double best = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double sq = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) sq += data[k] * data[k];
    if (sq > best) best = sq;
  }
  return best / 4.0 + lambda;
}

/* ------------------------------------------------------------------------ */
/* Logistic pieces (Section 4.1).
 * f_i(x) = log(1 + exp(-b_i a_i^T x)); f_i'(x) = sigma_i(x) a_i with
 * sigma_i(x) = -b_i / (1 + exp(b_i a_i^T x)) (the scalar memory of App. E). */
static double oracle_softplus(double m) { /* log(1+exp(m)), stable form */
  double am = m < 0 ? -m : m;
  return (m > 0 ? m : 0.0) + log1p(exp(-am));
}

double oracle_sigma(double b, double z) { return -b / (1.0 + exp(b * z)); }

/* f(x) = (1/n) sum_i log(1+exp(-b_i a_i.x)) + (lambda/2)||x||^2. */
double oracle_objective(int64_t n, int64_t d, const int64_t* indptr,
                        const int32_t* indices, const double* data, const double* y,
                        double lambda, const double* x) {
  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double z = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) z += data[k] * x[indices[k]];
    loss += oracle_softplus(-y[i] * z);
  }
  double sq = 0.0;
  for (int64_t v = 0; v < d; ++v) sq += x[v] * x[v];
  return loss / (double)n + 0.5 * lambda * sq;
}

/* grad f(x) = (1/n) sum_i sigma_i(x) a_i + lambda x  (gradient of Eq. 1 with the
 * l2 term of Section 4.1). */
void oracle_full_grad(int64_t n, int64_t d, const int64_t* indptr,
                      const int32_t* indices, const double* data, const double* y,
                      double lambda, const double* x, double* g) {
  for (int64_t v = 0; v < d; ++v) g[v] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double z = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) z += data[k] * x[indices[k]];
    double s = oracle_sigma(y[i], z);
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) g[indices[k]] += s * data[k];
  }
  for (int64_t v = 0; v < d; ++v) g[v] = g[v] / (double)n + lambda * x[v];
}

/* ------------------------------------------------------------------------ */
/* Sparse SAGA (Eq. 3) with the exact l2 term of Section 4.2
 * (P:519-522), one sample at a time, in the order of Algorithm 2:
 *   3: sample i                                (oracle_sample_index, before any read)
 *   5: [x]_{S_i}; 6: alpha_i; 7: [abar]_{S_i}  (sequential: reads are exact)
 *   8: dalpha = f_i'(x) - alpha_i              (scalar form, App. E)
 *   9: dx = -gamma (dalpha a_i + D_i abar + lambda D_i x)
 *  11: x_v += dx_v;  12: alpha_i += dalpha;  13: abar_v += dalpha a_iv / n
 * Every term of u uses the pre-step x and abar (reading R8).  State (x, alpha,
 * abar) is updated in place; updates t0 .. t0+T-1 use samples i_t.          */
/* One Sparse SAGA step on sample i (lines 4-13 of Alg. 2 executed without
 * interleaving).  u is scratch of at least |S_i| doubles. */
void oracle_saga_step(int64_t n, const int64_t* indptr, const int32_t* indices,
                      const double* data, const double* y, const double* D,
                      double lambda, double gamma, int64_t i, double* x, double* alpha,
                      double* alpha_bar, double* u) {
  const double inv_n = 1.0 / (double)n;
  int64_t lo = indptr[i], hi = indptr[i + 1];
  double z = 0.0;
  for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
  double s = oracle_sigma(y[i], z);
  double dalpha = s - alpha[i];
  for (int64_t k = lo; k < hi; ++k) {
    int32_t v = indices[k];
    u[k - lo] = dalpha * data[k] + D[v] * (alpha_bar[v] + lambda * x[v]);
  }
  for (int64_t k = lo; k < hi; ++k) {
    int32_t v = indices[k];
    x[v] = x[v] - gamma * u[k - lo];
    alpha_bar[v] = alpha_bar[v] + dalpha * data[k] * inv_n;
  }
  alpha[i] = alpha[i] + dalpha;
}

void oracle_sparse_saga(int64_t n, int64_t d, const int64_t* indptr,
                        const int32_t* indices, const double* data, const double* y,
                        const double* D, double lambda, double gamma, uint64_t seed,
                        uint64_t t0, uint64_t T, double* x, double* alpha,
                        double* alpha_bar) {
  (void)d;
  int64_t maxrow = 1;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] - indptr[i] > maxrow) maxrow = indptr[i + 1] - indptr[i];
  double* u = (double*)malloc(sizeof(double) * (size_t)maxrow);
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    oracle_saga_step(n, indptr, indices, data, y, D, lambda, gamma, i, x, alpha, alpha_bar, u);
  }
  free(u);
}

/* ------------------------------------------------------------------------ */
/* Bounded-delay Sparse SAGA (NEXT-1 tool, Assumption 1 P:316-322 taken at its
 * bound): update t reads x, alpha_i and abar as they stand after updates
 * 0..t-tau-1 have been written, i.e. every update is applied tau steps after
 * its read.  tau = 0 is exactly oracle_sparse_saga.  Used to predict the
 * convergence knee in the number of in-flight samples.  Pending updates are
 * kept in a ring of tau slots (each stores the row, dalpha and u).           */
typedef struct {
  int64_t i, lo, hi;
  double dalpha;
  double* u;
} oracle_pending;

void oracle_delayed_saga(int64_t n, int64_t d, const int64_t* indptr,
                         const int32_t* indices, const double* data, const double* y,
                         const double* D, double lambda, double gamma, uint64_t seed,
                         uint64_t t0, uint64_t T, int64_t tau, double* x, double* alpha,
                         double* alpha_bar) {
  (void)d;
  const double inv_n = 1.0 / (double)n;
  int64_t maxrow = 0;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] - indptr[i] > maxrow) maxrow = indptr[i + 1] - indptr[i];
  int64_t slots = tau + 1;
  oracle_pending* ring = (oracle_pending*)calloc((size_t)slots, sizeof(oracle_pending));
  for (int64_t s = 0; s < slots; ++s) {
    ring[s].u = (double*)malloc(sizeof(double) * (size_t)(maxrow > 0 ? maxrow : 1));
    ring[s].i = -1;
  }
  for (uint64_t step = 0; step < T + (uint64_t)tau + 1; ++step) {
    int64_t slot = (int64_t)(step % (uint64_t)slots);
    /* write the update read tau steps ago (it occupies this slot) */
    oracle_pending* p = &ring[slot];
    if (p->i >= 0) {
      for (int64_t k = p->lo; k < p->hi; ++k) {
        int32_t v = indices[k];
        x[v] = x[v] - gamma * p->u[k - p->lo];
        alpha_bar[v] = alpha_bar[v] + p->dalpha * data[k] * inv_n;
      }
      alpha[p->i] = alpha[p->i] + p->dalpha;
      p->i = -1;
    }
    if (step >= T) continue;
    /* read + compute update t = t0 + step */
    int64_t i = (int64_t)oracle_sample_index(seed, t0 + step, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double s = oracle_sigma(y[i], z);
    double dalpha = s - alpha[i];
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      p->u[k - lo] = dalpha * data[k] + D[v] * (alpha_bar[v] + lambda * x[v]);
    }
    p->i = i; p->lo = lo; p->hi = hi; p->dalpha = dalpha;
  }
  for (int64_t s = 0; s < slots; ++s) free(ring[s].u);
  free(ring);
}

/* ------------------------------------------------------------------------ */
/* Replicated Sparse SAGA with periodic exchange (NEXT-3 tool; Section 5, P:569:
 * "limiting communications can be interpreted as artificially increasing the delay").
 * N replicas (GPUs) each hold a copy of (x, abar); the global update counter t is dealt
 * round robin, update t runs on replica r = (t - t0) mod N.  An update reads replica r's
 * copy and alpha_i, computes Alg. 2's step exactly as oracle_saga_step (pre-step values,
 * reading R8) and applies it to replica r's copy at once; every E global updates (and
 * after the last) the replicas exchange: the shared (x, abar) receives the sum of every
 * replica's changes since the previous exchange and every copy becomes the shared value.
 * A replica's copy is kept as the shared value plus its own pending changes (x_r =
 * x + dx_r), with the pending coordinates listed, so an exchange costs the coordinates
 * touched.  alpha is one shared array (a sample's memory; reading R26: a repeat of i on
 * two replicas inside one exchange window, probability ~E/n, reads the current alpha_i).
 * N = 1, or E = 1, is sequential Sparse SAGA up to the rounding of x + dx (pinned).   */
void oracle_replica_saga(int64_t n, int64_t d, const int64_t* indptr,
                         const int32_t* indices, const double* data, const double* y,
                         const double* D, double lambda, double gamma, uint64_t seed,
                         uint64_t t0, uint64_t T, int64_t N, int64_t E, double* x,
                         double* alpha, double* alpha_bar) {
  const double inv_n = 1.0 / (double)n;
  int64_t maxrow = 1;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] - indptr[i] > maxrow) maxrow = indptr[i + 1] - indptr[i];
  double* u = (double*)malloc(sizeof(double) * (size_t)maxrow);
  double* dx = (double*)calloc((size_t)(N * d), sizeof(double));
  double* dab = (double*)calloc((size_t)(N * d), sizeof(double));
  unsigned char* mark = (unsigned char*)calloc((size_t)(N * d), 1);
  int32_t* list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N * d));
  int64_t* cnt = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  for (uint64_t step = 0; step < T; ++step) {
    const int64_t r = (int64_t)(step % (uint64_t)N);
    double* dxr = dx + r * d;
    double* dabr = dab + r * d;
    int64_t i = (int64_t)oracle_sample_index(seed, t0 + step, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      z += data[k] * (x[v] + dxr[v]);
    }
    double s = oracle_sigma(y[i], z);
    double dalpha = s - alpha[i];
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      u[k - lo] = dalpha * data[k] + D[v] * ((alpha_bar[v] + dabr[v]) + lambda * (x[v] + dxr[v]));
    }
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      dxr[v] = dxr[v] - gamma * u[k - lo];
      dabr[v] = dabr[v] + dalpha * data[k] * inv_n;
      if (!mark[r * d + v]) {
        mark[r * d + v] = 1;
        list[r * d + cnt[r]++] = v;
      }
    }
    alpha[i] = alpha[i] + dalpha;
    if ((step + 1) % (uint64_t)E == 0 || step + 1 == T) {  /* exchange, replicas in order */
      for (int64_t q = 0; q < N; ++q) {
        for (int64_t j = 0; j < cnt[q]; ++j) {
          int32_t v = list[q * d + j];
          x[v] = x[v] + dx[q * d + v];
          alpha_bar[v] = alpha_bar[v] + dab[q * d + v];
          dx[q * d + v] = 0.0;
          dab[q * d + v] = 0.0;
          mark[q * d + v] = 0;
        }
        cnt[q] = 0;
      }
    }
  }
  free(u); free(dx); free(dab); free(mark); free(list); free(cnt);
}

/* ------------------------------------------------------------------------ */
/* Comparison methods of Section 4.3, NEXT-2.  Both follow SPEC's
 * serial forms with the D_i-projected regulariser of
 * Section 4.2 applied uniformly (reading R21).
 *
 * HOGWILD (Niu et al.): sparse SGD with constant step,
 *   x_v <- x_v - gamma (sigma_i(x) a_iv + lambda D_v x_v),  v in S_i.          */
void oracle_hogwild(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                    const double* data, const double* y, const double* D, double lambda,
                    double gamma, uint64_t seed, uint64_t t0, uint64_t T, double* x) {
  (void)d;
  int64_t maxrow = 1;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] - indptr[i] > maxrow) maxrow = indptr[i + 1] - indptr[i];
  double* u = (double*)malloc(sizeof(double) * (size_t)maxrow);
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double s = oracle_sigma(y[i], z);
    for (int64_t k = lo; k < hi; ++k) u[k - lo] = s * data[k] + lambda * D[indices[k]] * x[indices[k]];
    for (int64_t k = lo; k < hi; ++k) x[indices[k]] = x[indices[k]] - gamma * u[k - lo];
  }
  free(u);
}

/* KROMAGNON (sparse SVRG of Mania et al.): the synchronised phase
 * caches s_i = sigma_i(x~) for every i and mu = (1/n) sum_i s_i a_i (the data part
 * of grad f(x~)); the inner steps are
 *   x_v <- x_v - gamma ((sigma_i(x) - s_i) a_iv + D_v mu_v + lambda D_v x_v).     */
void oracle_svrg_snapshot(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                          const double* data, const double* y, const double* xref, double* s,
                          double* mu) {
  for (int64_t v = 0; v < d; ++v) mu[v] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double z = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) z += data[k] * xref[indices[k]];
    s[i] = oracle_sigma(y[i], z);
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) mu[indices[k]] += s[i] * data[k];
  }
  for (int64_t v = 0; v < d; ++v) mu[v] = mu[v] / (double)n;
}

void oracle_svrg_inner(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                       const double* data, const double* y, const double* D, double lambda,
                       double gamma, uint64_t seed, uint64_t t0, uint64_t T, const double* s,
                       const double* mu, double* x) {
  (void)d;
  int64_t maxrow = 1;
  for (int64_t i = 0; i < n; ++i)
    if (indptr[i + 1] - indptr[i] > maxrow) maxrow = indptr[i + 1] - indptr[i];
  double* u = (double*)malloc(sizeof(double) * (size_t)maxrow);
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double dsig = oracle_sigma(y[i], z) - s[i];
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      u[k - lo] = dsig * data[k] + D[v] * mu[v] + lambda * D[v] * x[v];
    }
    for (int64_t k = lo; k < hi; ++k) x[indices[k]] = x[indices[k]] - gamma * u[k - lo];
  }
  free(u);
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the paper's other serial algorithms, at desk scale (off the hot path).
 *
 * Dense SAGA (Eq. 2) on f_i + (lambda/2)||x||^2: the full gradient
 * estimate f'_i(x) a_i - alpha_i a_i + abar + lambda x is applied to EVERY
 * coordinate (O(d) per step); abar_v += dalpha a_iv / n; alpha_i = sigma_i.      */
void oracle_dense_saga(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                       const double* data, const double* y, double lambda, double gamma,
                       uint64_t seed, uint64_t t0, uint64_t T, double* x, double* alpha,
                       double* alpha_bar) {
  const double inv_n = 1.0 / (double)n;
  double* g = (double*)malloc(sizeof(double) * (size_t)d);
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double dalpha = oracle_sigma(y[i], z) - alpha[i];
    for (int64_t v = 0; v < d; ++v) g[v] = alpha_bar[v] + lambda * x[v];
    for (int64_t k = lo; k < hi; ++k) g[indices[k]] = g[indices[k]] + dalpha * data[k];
    for (int64_t v = 0; v < d; ++v) x[v] = x[v] - gamma * g[v];
    for (int64_t k = lo; k < hi; ++k)
      alpha_bar[indices[k]] = alpha_bar[indices[k]] + dalpha * data[k] * inv_n;
    alpha[i] = alpha[i] + dalpha;
  }
  free(g);
}

/* SAGA with lagged ("just-in-time") updates (App. C):
 * the dense part of the step, x_v <- x_v - gamma (abar_v + lambda x_v), is
 * deferred until x_v is next read.  last[v] = the step up to which x_v is current;
 * abar_v does not change while v is outside the sampled supports, so k deferred
 * steps of x <- r x - gamma abar (r = 1 - gamma lambda) collapse to
 *   x <- r^k x - gamma abar (1 + r + ... + r^(k-1)),
 * summed here term by term (no closed-form division: k is small on desk data).
 * Sequentially this is the dense iteration ("strictly the same"), up to
 * rounding.  On return every coordinate is brought to t0 + T.       */
static void oracle_catch_up(int64_t v, uint64_t t, double lambda, double gamma,
                            uint64_t* last, double* x, const double* alpha_bar) {
  for (uint64_t s = last[v]; s < t; ++s) x[v] = x[v] - gamma * (alpha_bar[v] + lambda * x[v]);
  last[v] = t;
}

void oracle_lagged_saga(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                        const double* data, const double* y, double lambda, double gamma,
                        uint64_t seed, uint64_t t0, uint64_t T, double* x, double* alpha,
                        double* alpha_bar) {
  const double inv_n = 1.0 / (double)n;
  uint64_t* last = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)d);
  for (int64_t v = 0; v < d; ++v) last[v] = t0;
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    for (int64_t k = lo; k < hi; ++k) oracle_catch_up(indices[k], t, lambda, gamma, last, x, alpha_bar);
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double dalpha = oracle_sigma(y[i], z) - alpha[i];
    /* step t on the support: the sparse part plus step t's own dense part */
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      double gv = alpha_bar[v] + lambda * x[v];
      gv = gv + dalpha * data[k];
      x[v] = x[v] - gamma * gv;
      last[v] = t + 1;
    }
    for (int64_t k = lo; k < hi; ++k)
      alpha_bar[indices[k]] = alpha_bar[indices[k]] + dalpha * data[k] * inv_n;
    alpha[i] = alpha[i] + dalpha;
  }
  for (int64_t v = 0; v < d; ++v) oracle_catch_up(v, t0 + T, lambda, gamma, last, x, alpha_bar);
  free(last);
}

/* Algorithm 1 (the analysed ASAGA) run sequentially: every step
 * recomputes [abar]_{S_i} = (1/n) sum_k [alpha_k]_{S_i} from the whole memory
 * table (line 7; O(nnz) per step -- "too expensive to be practical"), then
 * dx = -gamma (f'_i(x) - alpha_i + D_i abar) on S_i with the exact l2 term
 * lambda D_i x of Section 4.2, alpha_i <- f'_i(x) (line 12, overwrite).
 * In the GLM case alpha_k = (scalar alpha_k) a_k.  Sequentially this equals Sparse
 * SAGA (whose abar is maintained incrementally), up to rounding.             */
void oracle_alg1_saga(int64_t n, int64_t d, const int64_t* indptr, const int32_t* indices,
                      const double* data, const double* y, const double* D, double lambda,
                      double gamma, uint64_t seed, uint64_t t0, uint64_t T, double* x,
                      double* alpha) {
  const double inv_n = 1.0 / (double)n;
  double* abar = (double*)malloc(sizeof(double) * (size_t)d);
  for (uint64_t t = t0; t < t0 + T; ++t) {
    int64_t i = (int64_t)oracle_sample_index(seed, t, (uint64_t)n);
    int64_t lo = indptr[i], hi = indptr[i + 1];
    /* line 7: abar from scratch (all coordinates; only S_i is used) */
    for (int64_t v = 0; v < d; ++v) abar[v] = 0.0;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k)
        abar[indices[k]] = abar[indices[k]] + alpha[r] * data[k];
    for (int64_t v = 0; v < d; ++v) abar[v] = abar[v] * inv_n;
    double z = 0.0;
    for (int64_t k = lo; k < hi; ++k) z += data[k] * x[indices[k]];
    double s = oracle_sigma(y[i], z);
    double dalpha = s - alpha[i];
    for (int64_t k = lo; k < hi; ++k) {
      int32_t v = indices[k];
      double u = dalpha * data[k] + D[v] * (abar[v] + lambda * x[v]);
      x[v] = x[v] - gamma * u;
    }
    alpha[i] = s;
  }
  free(abar);
}
