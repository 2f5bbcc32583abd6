"""Pins for the CPU oracle (``-m "not gpu"``): each test fixes a part of the
oracle against something other than itself -- a value the paper prints, a
closed form, an invariant the paper states, an independent library, or brute
force on tiny inputs -- so that a dropped term, a wrong sign/index or a
transposed operand fails at least one of them.  Pin ids (P1..P14) follow
DESIGN.md "Oracle pins"; "P:<line>" cites /root/reference/PAPER.md.
"""
import ctypes
import json
import math
import os

import numpy as np
import pytest
import scipy.optimize
import scipy.sparse
import scipy.stats

import datagen
import oracle

SEED = datagen.SAMPLE_SEED
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def csr(p):
    return scipy.sparse.csr_matrix((p.data, p.indices, p.indptr), shape=(p.n, p.d))


def fresh(p):
    return oracle.State(p.n, p.d)


def newton_opt(p, iters=60):
    """x* of f by damped Newton on the dense matrix (independent of the oracle)."""
    A = datagen.to_dense(p)
    b = p.y
    x = np.zeros(p.d)
    for _ in range(iters):
        m = b * (A @ x)
        s = -b / (1.0 + np.exp(m))  # dl/dz per sample
        g = A.T @ s / p.n + p.lam * x
        w = np.exp(m) / (1.0 + np.exp(m)) ** 2
        H = (A.T * w) @ A / p.n + p.lam * np.eye(p.d)
        x = x - np.linalg.solve(H, g)
    return x


# --------------------------------------------------------------------------- P1, P2 sampler
def test_p1_philox_matches_curand(curand_ref):
    """P1: oracle Philox4x32-10 == cuRAND's (independent implementation), 1e6 counters."""
    for seed, t0 in [(SEED, 0), (0, 0), (2**64 - 1, 2**32 - 500_000), (123456789, 2**40)]:
        count = 250_000
        ours = oracle.philox_stream(seed, t0, count)
        ref = np.empty((count, 4), dtype=np.uint32)
        curand_ref.curand_ref_philox_stream(seed, t0, count,
                                            ref.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
        assert np.array_equal(ours, ref)


def test_p2_index_map_exact_cases():
    """P2: floor(r*n/2^64): n=1 -> 0; n=2^k -> top k bits of r (exact integer arithmetic)."""
    words = oracle.philox_stream(SEED, 0, 2000).astype(np.uint64)
    r = (words[:, 1] << np.uint64(32)) | words[:, 0]
    assert (oracle.sample_stream(SEED, 0, 2000, 1) == 0).all()
    for k in (1, 7, 20, 33):
        got = oracle.sample_stream(SEED, 0, 2000, 2**k)
        assert np.array_equal(got.astype(np.uint64), r >> np.uint64(64 - k))
    # an n that is not a power of two, checked with Python big integers on a few draws
    n = 697_641
    got = oracle.sample_stream(SEED, 0, 200, n)
    for j in range(200):
        assert got[j] == (int(r[j]) * n) >> 64


@pytest.mark.parametrize("n", [3, 1000, 697_641])
def test_p2_index_map_uniform(n):
    """P2: chi^2 uniformity of 1e7 draws (with replacement, 'uniformly at random')."""
    draws = oracle.sample_stream(SEED, 0, 10_000_000, n)
    assert draws.min() >= 0 and draws.max() < n
    if n > 100_000:  # fold into 1000 equal-probability-ish bins of consecutive ids
        counts = np.bincount(draws * 1000 // n, minlength=1000)
        expected = np.bincount(np.arange(n) * 1000 // n, minlength=1000) * (1e7 / n)
    else:
        counts = np.bincount(draws, minlength=n)
        expected = np.full(n, 1e7 / n)
    chi2 = ((counts - expected) ** 2 / expected).sum()
    dof = len(counts) - 1
    assert scipy.stats.chi2.sf(chi2, dof) > 1e-4


def test_sample_stream_continuation():
    a = oracle.sample_stream(SEED, 0, 1000, 977)
    b = np.concatenate([oracle.sample_stream(SEED, 0, 400, 977),
                        oracle.sample_stream(SEED, 400, 600, 977)])
    assert np.array_equal(a, b)


# --------------------------------------------------------------------------- P3 profile
def test_p3_spec_example():
    """P3: n=2, d=2, rows {0,1} and {0}: p=(1, 1/2), D=(1, 2), Delta_r=2."""
    p = datagen.Problem("ex", 2, 2, np.array([0, 2, 3]), np.array([0, 1, 0], dtype=np.int32),
                        np.array([1.0, 1.0, 1.0]), np.array([1.0, -1.0]), 0.5)
    cnt = oracle.column_counts(p)
    assert cnt.tolist() == [2, 1]
    assert oracle.reweight(2, cnt).tolist() == [1.0, 2.0]
    assert cnt.max() == 2


@pytest.mark.parametrize("cfg,n_rows", [("c1", None), ("c2", 20_000), ("c3", 20_000)])
def test_p3_counts_match_scipy(cfg, n_rows):
    p = datagen.make(cfg, n_rows=n_rows)
    cnt = oracle.column_counts(p)
    assert np.array_equal(cnt, csr(p).getnnz(axis=0))
    D = oracle.reweight(p.n, cnt)
    used = cnt > 0
    # D_v * n_v == n within one ulp; D_v == 0 for unused columns (reading R4)
    assert np.all(np.abs(D[used] * cnt[used] - p.n) <= np.spacing(float(p.n)))
    assert np.all(D[~used] == 0.0)


def test_p3_unused_column_reweight_zero():
    p = datagen.Problem("gap", 2, 3, np.array([0, 1, 2]), np.array([0, 2], dtype=np.int32),
                        np.array([1.0, 1.0]), np.array([1.0, 1.0]), 0.5)
    assert oracle.reweight(2, oracle.column_counts(p)).tolist() == [2.0, 0.0, 2.0]


def test_p3_lipschitz_unit_rows_matches_table1():
    """Unit-norm rows give L = 1/4 + lambda; Table 1 prints L = 0.25 for normalised RCV1."""
    tab = json.load(open(os.path.join(GOLDEN, "paper_tables.json")))
    p = datagen.make("c1")
    L = oracle.lipschitz(p, p.lam)
    assert abs((L - p.lam) - tab["table1"]["RCV1"]["L"]) < 1e-12
    # a row of norm 2 -> L = 4/4 + lambda
    q = datagen.Problem("nrm", 1, 2, np.array([0, 2]), np.array([0, 1], dtype=np.int32),
                        np.array([2.0 * 0.6, 2.0 * 0.8]), np.array([1.0]), 0.25)
    assert abs(oracle.lipschitz(q, 0.25) - 1.25) < 1e-12


# --------------------------------------------------------------------------- P6 loss / sigma / grad
def test_p6_closed_forms():
    p = datagen.make("c1")
    assert oracle.objective(p, p.y, p.lam, np.zeros(p.d)) == pytest.approx(math.log(2), rel=1e-13)
    assert oracle.sigma(1.0, 0.0) == -0.5 and oracle.sigma(-1.0, 0.0) == 0.5
    assert abs(oracle.sigma(1.0, 800.0)) < 1e-300  # saturated correct classification
    assert oracle.sigma(-1.0, 800.0) == pytest.approx(1.0)
    one = datagen.Problem("one", 1, 1, np.array([0, 1]), np.array([0], dtype=np.int32),
                          np.array([1.0]), np.array([1.0]), 1.0)
    assert oracle.objective(one, one.y, 1.0, np.zeros(1)) == pytest.approx(math.log(2))
    # huge margins stay finite (stable softplus)
    assert math.isfinite(oracle.objective(one, one.y, 1.0, np.array([-1e6])))


def test_p6_objective_fsum():
    """f to 1e-12 against a compensated (math.fsum) summation written independently."""
    p = datagen.make("c1")
    x = np.random.default_rng(1).standard_normal(p.d)
    terms = []
    for i in range(p.n):
        lo, hi = p.indptr[i], p.indptr[i + 1]
        z = math.fsum(p.data[k] * x[p.indices[k]] for k in range(lo, hi))
        m = -p.y[i] * z
        terms.append(max(m, 0.0) + math.log1p(math.exp(-abs(m))))
    f = math.fsum(terms) / p.n + 0.5 * p.lam * math.fsum(x * x)
    assert oracle.objective(p, p.y, p.lam, x) == pytest.approx(f, rel=1e-12)


def test_p6_gradient_finite_differences():
    """P6: analytic grad vs central differences, rel err <= 1e-6, 100 random instances."""
    rng = np.random.default_rng(7)
    for trial in range(100):
        n = int(rng.integers(1, 51))
        d = int(rng.integers(1, 21))
        p = datagen.random_tiny(1000 + trial, n, d, density=0.4)
        lam = float(rng.uniform(0.01, 1.0))
        x = rng.standard_normal(d)
        g = oracle.full_grad(p, p.y, lam, x)
        fd = np.empty(d)
        for v in range(d):
            h = 1e-6 * (1.0 + abs(x[v]))
            e = np.zeros(d)
            e[v] = h
            fd[v] = (oracle.objective(p, p.y, lam, x + e) - oracle.objective(p, p.y, lam, x - e)) / (2 * h)
        assert np.linalg.norm(g - fd) <= 1e-6 * max(np.linalg.norm(g), 1e-3)


def test_p6_gradient_lambda_linearity_and_convexity():
    p = datagen.random_tiny(5, 30, 12)
    rng = np.random.default_rng(3)
    x, z = rng.standard_normal(12), rng.standard_normal(12)
    g1, g2 = oracle.full_grad(p, p.y, 0.1, x), oracle.full_grad(p, p.y, 0.7, x)
    assert np.allclose(g2 - g1, 0.6 * x, rtol=0, atol=1e-12)
    lam = 0.3
    fx, fz = oracle.objective(p, p.y, lam, x), oracle.objective(p, p.y, lam, z)
    gx = oracle.full_grad(p, p.y, lam, x)
    assert fz >= fx + gx @ (z - x) + 0.5 * lam * np.sum((z - x) ** 2) - 1e-12


# --------------------------------------------------------------------------- P4 unbiasedness
def test_p4_reweighted_abar_unbiased():
    """Eq. 14: (1/n) sum_i D_i abar = abar, by enumeration of all i."""
    for seed in range(5):
        p = datagen.random_tiny(seed, 40, 15, density=0.25)
        D = oracle.reweight(p.n, oracle.column_counts(p))
        abar = np.random.default_rng(seed).standard_normal(p.d)
        acc = np.zeros(p.d)
        for i in range(p.n):
            S = p.indices[p.indptr[i]:p.indptr[i + 1]]
            acc[S] += D[S] * abar[S]
        acc /= p.n
        used = D > 0
        assert np.allclose(acc[used], abar[used], rtol=1e-12, atol=1e-14)


def test_p4_increment_unbiased():
    """E_i[x+ - x] = -gamma grad f(x) when abar = (1/n) sum alpha_i a_i.

    Built from the oracle's own step: enumerate every i from one state."""
    p = datagen.random_tiny(11, 30, 10, density=0.3)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    rng = np.random.default_rng(0)
    st = fresh(p)
    st.x = rng.standard_normal(p.d)
    st.alpha = rng.standard_normal(p.n)
    A = datagen.to_dense(p)
    st.alpha_bar = A.T @ st.alpha / p.n
    gamma = 0.3
    mean_dx = np.zeros(p.d)
    for i in range(p.n):
        s = st.copy()
        oracle.saga_step(p, p.y, p.lam, gamma, i, s, D)
        mean_dx += (s.x - st.x) / p.n
    g = oracle.full_grad(p, p.y, p.lam, st.x)
    assert np.allclose(mean_dx, -gamma * g, rtol=1e-11, atol=1e-13)


# --------------------------------------------------------------------------- P5 SAGA identity
def test_p5_abar_identity_every_step():
    """abar == (1/n) sum_i alpha_i a_i after every step (P:88-89 'updated ... online')."""
    p = datagen.random_tiny(21, 25, 8, density=0.4)
    A = datagen.to_dense(p)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    st = fresh(p)
    L = oracle.lipschitz(p, p.lam)
    for _ in range(300):
        oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 1, st, D)
        assert np.allclose(st.alpha_bar, A.T @ st.alpha / p.n, rtol=0, atol=1e-12)


def test_p5_abar_identity_c1_long():
    p = datagen.make("c1")
    L = oracle.lipschitz(p, p.lam)
    st = oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 20 * p.n)
    ref = csr(p).T @ st.alpha / p.n
    assert np.linalg.norm(st.alpha_bar - ref) <= 1e-10 * np.linalg.norm(ref)


# --------------------------------------------------------------------------- P7 first update
def test_p7_first_update_closed_form():
    p = datagen.make("c1")
    L = oracle.lipschitz(p, p.lam)
    gamma = 1 / (3 * L)
    st = oracle.sparse_saga(p, p.y, p.lam, gamma, SEED, 1)
    i = oracle.sample_index(SEED, 0, p.n)
    lo, hi = p.indptr[i], p.indptr[i + 1]
    x = np.zeros(p.d)
    x[p.indices[lo:hi]] = gamma * p.y[i] / 2 * p.data[lo:hi]
    ab = np.zeros(p.d)
    ab[p.indices[lo:hi]] = -p.y[i] / (2 * p.n) * p.data[lo:hi]
    assert np.allclose(st.x, x, rtol=1e-15, atol=0)
    assert np.allclose(st.alpha_bar, ab, rtol=1e-15, atol=0)
    al = np.zeros(p.n)
    al[i] = -p.y[i] / 2
    assert np.array_equal(st.alpha, al)


# --------------------------------------------------------------------------- P8 dense reduction
def dense_saga_l2(A, b, lam, gamma, seed, T):
    """Dense SAGA (Eq. 2) with the l2 gradient lam*x added: test helper, numpy."""
    n, d = A.shape
    x = np.zeros(d)
    alpha = np.zeros(n)
    for i in oracle.sample_stream(seed, 0, T, n):
        z = A[i] @ x
        s = -b[i] / (1.0 + np.exp(b[i] * z))
        abar = A.T @ alpha / n  # recomputed from the memory table every step
        x = x - gamma * (s * A[i] - alpha[i] * A[i] + abar + lam * x)
        alpha[i] = s
    return x, alpha


def test_p8_dense_data_reduces_to_saga():
    p = datagen.random_tiny(31, 20, 6, dense=True)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    assert np.all(D == 1.0)
    L = oracle.lipschitz(p, p.lam)
    st = oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 400, D=D)
    x, alpha = dense_saga_l2(datagen.to_dense(p), p.y, p.lam, 1 / (3 * L), SEED, 400)
    assert np.allclose(st.x, x, rtol=1e-12, atol=1e-13)
    assert np.allclose(st.alpha, alpha, rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- P9 fixed point
def test_p9_fixed_point_is_stationary():
    """At (x*, alpha_i = sigma_i(x*), abar = mean alpha_i a_i) every update is zero."""
    p = datagen.make("c1")
    xs = newton_opt(p)
    assert np.abs(oracle.full_grad(p, p.y, p.lam, xs)).max() < 1e-14
    A = csr(p)
    st = fresh(p)
    st.x = xs.copy()
    z = A @ xs
    st.alpha = -p.y / (1.0 + np.exp(p.y * z))
    st.alpha_bar = A.T @ st.alpha / p.n
    L = oracle.lipschitz(p, p.lam)
    x0 = st.x.copy()
    oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 10 * p.n, st)
    assert np.abs(st.x - x0).max() <= 1e-10


# --------------------------------------------------------------------------- P10 1-D instance
def test_p10_one_dimensional_bisection():
    n = 20
    y = np.where(np.arange(n) % 3 == 0, -1.0, 1.0)
    p = datagen.Problem("1d", n, 1, np.arange(n + 1, dtype=np.int64), np.zeros(n, dtype=np.int32),
                        np.ones(n), y, 1.0 / n)

    def fprime(x):  # d/dx of (1/n) sum log(1+exp(-b x)) + lam/2 x^2
        return np.mean(-y / (1.0 + np.exp(y * x))) + p.lam * x

    lo, hi = -50.0, 50.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if fprime(mid) < 0 else (lo, mid)
    L = oracle.lipschitz(p, p.lam)
    st = oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 4000 * n)
    assert st.x[0] == pytest.approx(0.5 * (lo + hi), abs=1e-10)


# --------------------------------------------------------------------------- P11 f* / x*
def test_p11_optimum_matches_lbfgs():
    p = datagen.make("c1")
    A = csr(p)

    def fg(x):
        m = p.y * (A @ x)
        f = np.mean(np.logaddexp(0.0, -m)) + 0.5 * p.lam * x @ x
        s = -p.y / (1.0 + np.exp(m))
        return f, A.T @ s / p.n + p.lam * x

    res = scipy.optimize.minimize(fg, np.zeros(p.d), jac=True, method="L-BFGS-B",
                                  options=dict(maxiter=10000, gtol=1e-13, ftol=1e-16))
    L = oracle.lipschitz(p, p.lam)
    st = oracle.sparse_saga(p, p.y, p.lam, 1 / (3 * L), SEED, 300 * p.n)
    f_or = oracle.objective(p, p.y, p.lam, st.x)
    gn = np.linalg.norm(oracle.full_grad(p, p.y, p.lam, st.x))
    assert gn ** 2 / (2 * p.lam) <= 1e-12  # certificate (reading R13)
    assert f_or == pytest.approx(res.fun, abs=1e-10)
    assert np.linalg.norm(st.x - res.x) <= 1e-5 * np.linalg.norm(res.x)


# --------------------------------------------------------------------------- P12 Thm 1 slope
def test_p12_theorem1_rate():
    """||x_t - x*||^2 decays at least like (1 - rho)^t, rho = (1/5) min(1/n, a/kappa)."""
    p = datagen.make("c1")
    xs = newton_opt(p)
    L = oracle.lipschitz(p, p.lam)
    a = 1.0
    gamma = a / (5 * L)
    kappa = L / p.lam
    rho = 0.2 * min(1.0 / p.n, a / kappa)
    st = fresh(p)
    errs = []
    for _ in range(30):
        oracle.sparse_saga(p, p.y, p.lam, gamma, SEED, p.n, st)
        errs.append(np.sum((st.x - xs) ** 2))
    t = np.arange(1, 31) * p.n
    slope = np.polyfit(t[5:25], np.log(errs[5:25]), 1)[0]
    assert slope <= -rho / 2


# --------------------------------------------------------------------------- continuation, delay tool
def test_run_split_equals_whole():
    p = datagen.make("c1")
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    a = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 3000)
    b = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 1234)
    oracle.sparse_saga(p, p.y, p.lam, g, SEED, 3000 - 1234, b)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.alpha, b.alpha)
    assert np.array_equal(a.alpha_bar, b.alpha_bar)


def test_delayed_tau0_is_sequential_and_quiescent_identity():
    p = datagen.make("c1")
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    a = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 5000)
    b = oracle.delayed_saga(p, p.y, p.lam, g, SEED, 5000, 0)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.alpha_bar, b.alpha_bar)
    c = oracle.delayed_saga(p, p.y, p.lam, g, SEED, 5000, 17)
    # quiescent: every write applied -> abar consistent with alpha
    assert np.allclose(c.alpha_bar, csr(p).T @ c.alpha / p.n, rtol=0, atol=1e-12)
    assert not np.array_equal(a.x, c.x)


def test_delayed_tau1_by_hand():
    """tau=1 on a 3-sample problem against a hand-unrolled two-slot schedule."""
    p = datagen.random_tiny(3, 3, 4, density=0.6)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    g = 0.5
    T = 6
    got = oracle.delayed_saga(p, p.y, p.lam, g, SEED, T, 1, D=D)
    # reference: update t computed on the state with updates < t-1 applied
    st = fresh(p)
    snaps = []
    idx = oracle.sample_stream(SEED, 0, T, p.n)
    pending = None
    for t in range(T):
        s = st.copy()
        before = s.copy()
        oracle.saga_step(p, p.y, p.lam, g, int(idx[t]), s, D)
        delta = (s.x - before.x, s.alpha - before.alpha, s.alpha_bar - before.alpha_bar)
        if pending is not None:
            st.x += pending[0]; st.alpha += pending[1]; st.alpha_bar += pending[2]
        pending = delta
        snaps.append(delta)
    st.x += pending[0]; st.alpha += pending[1]; st.alpha_bar += pending[2]
    assert np.allclose(got.x, st.x, rtol=1e-14, atol=1e-15)
    assert np.allclose(got.alpha, st.alpha, rtol=1e-14, atol=1e-15)


# --------------------------------------------------------------------------- NEXT-3 replicated model
def test_replica_reduces_to_sequential():
    """One replica (any exchange period) or an exchange after every update is sequential
    Sparse SAGA: E = 1 bit for bit (x + 0 is exact), N = 1 up to the rounding of x + dx."""
    p = datagen.make("c1")
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    a = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 5000)
    for N in (2, 5):
        b = oracle.replica_saga(p, p.y, p.lam, g, SEED, 5000, N, 1)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.alpha, b.alpha)
        assert np.array_equal(a.alpha_bar, b.alpha_bar)
    for E in (7, 1000, 10**9):
        c = oracle.replica_saga(p, p.y, p.lam, g, SEED, 5000, 1, E)
        for u, v in ((c.x, a.x), (c.alpha, a.alpha), (c.alpha_bar, a.alpha_bar)):
            assert np.linalg.norm(u - v) <= 1e-13 * np.linalg.norm(v)


def test_replica_schedule_by_hand_and_quiescent_identity():
    """N = 3 replicas exchanging every E = 4 updates on a tiny problem, against the schedule
    written out with explicit copies (each replica steps its own copy with the shared alpha;
    at an exchange the shared state gains every copy's change); then the quiescent identity
    abar = (1/n) sum alpha_i a_i holds after the final exchange."""
    p = datagen.random_tiny(5, 6, 8, density=0.5)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    g, N, E, T = 0.4, 3, 4, 23
    got = oracle.replica_saga(p, p.y, p.lam, g, SEED, T, N, E, D=D)
    idx = oracle.sample_stream(SEED, 0, T, p.n)
    shared = fresh(p)
    copies = [shared.copy() for _ in range(N)]
    for t in range(T):
        r = t % N
        c = copies[r]
        c.alpha = shared.alpha  # one shared memory of alpha (reading R26)
        oracle.saga_step(p, p.y, p.lam, g, int(idx[t]), c, D)
        if (t + 1) % E == 0 or t + 1 == T:
            base_x, base_ab = shared.x.copy(), shared.alpha_bar.copy()
            for q in range(N):
                shared.x = shared.x + (copies[q].x - base_x)
                shared.alpha_bar = shared.alpha_bar + (copies[q].alpha_bar - base_ab)
            for q in range(N):
                copies[q].x, copies[q].alpha_bar = shared.x.copy(), shared.alpha_bar.copy()
    assert np.allclose(got.x, shared.x, rtol=1e-12, atol=1e-15)
    assert np.allclose(got.alpha, shared.alpha, rtol=1e-12, atol=1e-15)
    assert np.allclose(got.alpha_bar, shared.alpha_bar, rtol=1e-12, atol=1e-15)
    q = datagen.make("c1")
    gq = 1 / (3 * oracle.lipschitz(q, q.lam))
    st = oracle.replica_saga(q, q.y, q.lam, gq, SEED, 7 * q.n + 3, 4, 64)
    assert np.allclose(st.alpha_bar, csr(q).T @ st.alpha / q.n, rtol=0, atol=1e-12)


def test_replica_fixed_point_is_stationary():
    """P9 for the replicated model: at (x*, alpha_i = sigma_i(x*), abar = mean) every
    replica's every update is zero, whatever the exchange period."""
    p = datagen.make("c1")
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    x = newton_opt(p)
    A = csr(p)
    alpha = -p.y / (1.0 + np.exp(p.y * (A @ x)))
    st = fresh(p)
    st.x = x.copy()
    st.alpha = alpha
    st.alpha_bar = A.T @ alpha / p.n
    oracle.replica_saga(p, p.y, p.lam, g, SEED, 10 * p.n, 8, 256, st)
    assert np.abs(st.x - x).max() <= 1e-10


# --------------------------------------------------------------------------- NEXT-2 comparison methods
def test_svrg_first_inner_step_reference_identity():
    """At x = x~ the data difference vanishes: the step is -gamma (D mu + lambda D x) on S_i."""
    p = datagen.random_tiny(41, 30, 12, density=0.4)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    x0 = np.random.default_rng(1).standard_normal(p.d)
    s, mu = oracle.svrg_snapshot(p, p.y, x0)
    x = oracle.svrg_inner(p, p.y, p.lam, 0.3, SEED, 0, 1, s, mu, x0.copy(), D)
    i = oracle.sample_index(SEED, 0, p.n)
    S = p.indices[p.indptr[i]:p.indptr[i + 1]]
    want = x0.copy()
    want[S] = x0[S] - 0.3 * (D[S] * mu[S] + p.lam * D[S] * x0[S])
    assert np.allclose(x, want, rtol=1e-15, atol=1e-15)


def test_svrg_snapshot_is_data_gradient():
    p = datagen.random_tiny(42, 25, 9)
    x0 = np.random.default_rng(2).standard_normal(p.d)
    s, mu = oracle.svrg_snapshot(p, p.y, x0)
    # mu + lambda x~ is grad f(x~) (pinned by finite differences, P6)
    assert np.allclose(mu + p.lam * x0, oracle.full_grad(p, p.y, p.lam, x0), rtol=1e-13, atol=1e-15)
    A = datagen.to_dense(p)
    assert np.allclose(s, -p.y / (1 + np.exp(p.y * (A @ x0))), rtol=1e-14)


def test_svrg_and_hogwild_are_saga_with_frozen_memory():
    """Cross-check of three independently written oracle updates: SVRG's inner step equals
    the Sparse SAGA step with the memory frozen at (s, mu); HOGWILD's with (0, 0)."""
    p = datagen.random_tiny(43, 40, 15, density=0.3)
    D = oracle.reweight(p.n, oracle.column_counts(p))
    x0 = np.random.default_rng(3).standard_normal(p.d)
    s, mu = oracle.svrg_snapshot(p, p.y, x0)
    T = 300
    xs = oracle.svrg_inner(p, p.y, p.lam, 0.2, SEED, 0, T, s, mu, x0.copy(), D)
    xh = oracle.hogwild(p, p.y, p.lam, 0.2, SEED, 0, T, x0.copy(), D)
    for frozen_a, frozen_ab, got in ((s, mu, xs), (np.zeros(p.n), np.zeros(p.d), xh)):
        st = fresh(p)
        st.x = x0.copy()
        for i in oracle.sample_stream(SEED, 0, T, p.n):
            st.alpha, st.alpha_bar = frozen_a.copy(), frozen_ab.copy()
            oracle.saga_step(p, p.y, p.lam, 0.2, int(i), st, D)
        assert np.allclose(got, st.x, rtol=1e-13, atol=1e-14)


def test_svrg_hogwild_dense_reduce_to_textbook():
    """On 100%-dense data (D = I): textbook SVRG inner steps and textbook SGD."""
    p = datagen.random_tiny(44, 20, 6, dense=True)
    A = datagen.to_dense(p)
    b = p.y
    x0 = np.random.default_rng(4).standard_normal(p.d)
    s, mu = oracle.svrg_snapshot(p, p.y, x0)
    T, g = 200, 0.25
    x_svrg, x_sgd = x0.copy(), x0.copy()
    for i in oracle.sample_stream(SEED, 0, T, p.n):
        sig = -b[i] / (1 + np.exp(b[i] * (A[i] @ x_svrg)))
        x_svrg = x_svrg - g * ((sig - s[i]) * A[i] + mu + p.lam * x_svrg)
        sig2 = -b[i] / (1 + np.exp(b[i] * (A[i] @ x_sgd)))
        x_sgd = x_sgd - g * (sig2 * A[i] + p.lam * x_sgd)
    assert np.allclose(oracle.svrg_inner(p, p.y, p.lam, g, SEED, 0, T, s, mu, x0.copy()), x_svrg,
                       rtol=1e-12, atol=1e-13)
    assert np.allclose(oracle.hogwild(p, p.y, p.lam, g, SEED, 0, T, x0.copy()), x_sgd,
                       rtol=1e-12, atol=1e-13)


def test_hogwild_stalls_where_saga_converges():
    """Constant-step SGD plateaus at a variance floor; SAGA/SVRG converge linearly
    (the paper measures HOGWILD only to 1e-3)."""
    p = datagen.make("c1")
    L = oracle.lipschitz(p, p.lam)
    g = 1 / (3 * L)
    fstar = json.load(open(os.path.join(GOLDEN, "fstar_c1.json")))["f_star"]
    x = oracle.hogwild(p, p.y, p.lam, g, SEED, 0, 50 * p.n, np.zeros(p.d))
    saga = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 50 * p.n)
    xk = np.zeros(p.d)
    t = 0
    for _ in range(25):  # KROMAGNON: snapshot every 2 epochs
        s, mu = oracle.svrg_snapshot(p, p.y, xk)
        oracle.svrg_inner(p, p.y, p.lam, g, SEED, t, 2 * p.n, s, mu, xk)
        t += 2 * p.n
    assert oracle.objective(p, p.y, p.lam, x) - fstar > 1e-6
    assert oracle.objective(p, p.y, p.lam, saga.x) - fstar < 1e-10
    assert oracle.objective(p, p.y, p.lam, xk) - fstar < 1e-10


# --------------------------------------------------------------------------- NEXT-4 serial variants
def test_next4_dense_saga_is_the_textbook_iteration():
    """oracle.dense_saga (C) == the numpy textbook SAGA with l2 (Eq. 2) on SPARSE data,
    where the two share nothing but the sampler (the numpy side recomputes abar)."""
    p = datagen.random_tiny(41, 25, 9, density=0.3)
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    st = oracle.dense_saga(p, p.y, p.lam, g, SEED, 500)
    x, alpha = dense_saga_l2(datagen.to_dense(p), p.y, p.lam, g, SEED, 500)
    assert np.allclose(st.x, x, rtol=1e-12, atol=1e-14)
    assert np.allclose(st.alpha, alpha, rtol=1e-12, atol=1e-14)


def test_next4_lagged_updates_equal_dense_updates():
    """App. C: sequentially, deferring the dense part until a coordinate is
    read is 'strictly the same' as applying it every step -- bit for bit here, since the
    deferred steps are applied with the same formula in the same order; checked also
    after a split run (the catch-up at the end of each call)."""
    for seed, (n, d, dens) in ((3, (40, 30, 0.1)), (4, (60, 12, 0.4))):
        p = datagen.random_tiny(seed, n, d, density=dens)
        g = 1 / (3 * oracle.lipschitz(p, p.lam))
        a = oracle.dense_saga(p, p.y, p.lam, g, SEED, 7 * n)
        b = oracle.lagged_saga(p, p.y, p.lam, g, SEED, 3 * n)
        b = oracle.lagged_saga(p, p.y, p.lam, g, SEED, 4 * n, state=b)
        assert np.array_equal(a.x, b.x) and np.array_equal(a.alpha, b.alpha)
        assert np.array_equal(a.alpha_bar, b.alpha_bar)


def test_next4_alg1_equals_sparse_saga_sequentially():
    """Alg. 1 (abar recomputed from the whole memory every step, alpha_i overwritten)
    and Alg. 2's Sparse SAGA (abar maintained incrementally, alpha_i += dalpha) give
    the same sequential iterates up to rounding."""
    p = datagen.random_tiny(5, 50, 20, density=0.25)
    g = 1 / (3 * oracle.lipschitz(p, p.lam))
    a = oracle.alg1_saga(p, p.y, p.lam, g, SEED, 10 * p.n)
    b = oracle.sparse_saga(p, p.y, p.lam, g, SEED, 10 * p.n)
    assert np.linalg.norm(a.x - b.x) <= 1e-12 * np.linalg.norm(b.x)
    assert np.linalg.norm(a.alpha - b.alpha) <= 1e-12 * np.linalg.norm(b.alpha)


def test_next4_dense_lagged_and_sparse_saga_converge_alike():
    """P:129 / P:1959: dense (lagged) and sparse SAGA 'had similar convergence in terms of
    number of iterations': on c1 both reach the certified f* + 1e-6 (golden, oracle-written)
    within a factor 2 of each other's epoch count."""
    p = datagen.make("c1")
    fstar = json.load(open(os.path.join(GOLDEN, "fstar_c1.json")))["f_star"]
    g = 1 / (3 * oracle.lipschitz(p, p.lam))

    def epochs(run):
        st = None
        for j in range(1, 401):
            st = run(p.n // 10, st)
            if oracle.objective(p, p.y, p.lam, st.x) - fstar <= 1e-6:
                return j / 10
        return math.inf

    e_sparse = epochs(lambda T, st: oracle.sparse_saga(p, p.y, p.lam, g, SEED, T, st))
    e_lagged = epochs(lambda T, st: oracle.lagged_saga(p, p.y, p.lam, g, SEED, T, st))
    assert e_sparse < 40 and e_lagged < 40
    assert 0.5 <= e_lagged / e_sparse <= 2.0, (e_lagged, e_sparse)
