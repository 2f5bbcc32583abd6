"""ASAGA oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, sequential fp64 CPU implementation of the ASAGA hot path written
from the paper (arXiv 1606.04809, /root/reference/PAPER.md; "P:<line>" below).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_1606_04809_b200``) never imports it and shares no code
with it; the two meet only through the seeded input generators in ``datagen``.

Arithmetic lives in ``asaga_oracle.c`` (compiled with gcc ``-O2
-ffp-contract=off``); this module only marshals numpy arrays through ctypes.

Functions and the passages they follow:
  sample_index / sample_stream  Alg. 2 line 3, Philox4x32-10 (reading R2)
  column_counts / reweight      P:108-110 (D = diag(1/p_v)), P:128 (first pass), R4
  lipschitz                     P:38, Table 1, reading R7
  objective / full_grad         Section 4.1
  sparse_saga                   Eq. 3 + Section 4.2, Alg. 2 order
  delayed_saga                  Assumption 1 at its bound; NEXT-1 tool
  replica_saga                  Section 5 periodic exchange between replicas; NEXT-3 tool
  hogwild / svrg_*              Section 4.3 comparison methods, SPEC S:230-237,
                                S:306-307, regulariser projected as in Section 4.2 (R21)
All are pinned in tests/test_oracle_pins.py; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "asaga_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)
_U32P = ctypes.POINTER(ctypes.c_uint32)
_F64P = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile asaga_oracle.c into liboracle.so (gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
             "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        u64, i64, f64 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double
        sig = {
            "oracle_philox4x32_10": (None, [_U32P, _U32P, _U32P]),
            "oracle_sample_index": (u64, [u64, u64, u64]),
            "oracle_sample_stream": (None, [u64, u64, u64, u64, _I64P]),
            "oracle_philox_stream": (None, [u64, u64, u64, _U32P]),
            "oracle_saga_step": (None, [i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64, i64,
                                        _F64P, _F64P, _F64P, _F64P]),
            "oracle_column_counts": (None, [i64, i64, _I64P, _I32P, _I64P]),
            "oracle_reweight": (None, [i64, i64, _I64P, _F64P]),
            "oracle_lipschitz": (f64, [i64, _I64P, _F64P, f64]),
            "oracle_sigma": (f64, [f64, f64]),
            "oracle_objective": (f64, [i64, i64, _I64P, _I32P, _F64P, _F64P, f64, _F64P]),
            "oracle_full_grad": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, f64, _F64P, _F64P]),
            "oracle_sparse_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                          u64, u64, u64, _F64P, _F64P, _F64P]),
            "oracle_delayed_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                           u64, u64, u64, i64, _F64P, _F64P, _F64P]),
            "oracle_replica_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                           u64, u64, u64, i64, i64, _F64P, _F64P, _F64P]),
            "oracle_hogwild": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                      u64, u64, u64, _F64P]),
            "oracle_svrg_snapshot": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, _F64P,
                                            _F64P]),
            "oracle_svrg_inner": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                         u64, u64, u64, _F64P, _F64P, _F64P]),
            "oracle_dense_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, f64, f64, u64, u64,
                                         u64, _F64P, _F64P, _F64P]),
            "oracle_lagged_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, f64, f64, u64, u64,
                                          u64, _F64P, _F64P, _F64P]),
            "oracle_alg1_saga": (None, [i64, i64, _I64P, _I32P, _F64P, _F64P, _F64P, f64, f64,
                                        u64, u64, u64, _F64P, _F64P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _p(a: np.ndarray, ptype):
    return a.ctypes.data_as(ptype)


def _csr(A):
    """(n, d, indptr i64, indices i32, data f64) views of a Problem-like object."""
    indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(A.indices, dtype=np.int32)
    data = np.ascontiguousarray(A.data, dtype=np.float64)
    return int(A.n), int(A.d), indptr, indices, data


# --------------------------------------------------------------------------- sampler
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().oracle_philox4x32_10(_p(c, _U32P), _p(k, _U32P), _p(out, _U32P))
    return out


def philox_stream(seed: int, t0: int, count: int) -> np.ndarray:
    """Raw Philox4x32-10 words, shape (count, 4), for counters t0..t0+count-1."""
    out = np.empty((count, 4), dtype=np.uint32)
    _load().oracle_philox_stream(seed, t0, count, _p(out, _U32P))
    return out


def sample_index(seed: int, t: int, n: int) -> int:
    return int(_load().oracle_sample_index(seed, t, n))


def sample_stream(seed: int, t0: int, count: int, n: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    _load().oracle_sample_stream(seed, t0, count, n, _p(out, _I64P))
    return out


# --------------------------------------------------------------------------- profile
def column_counts(A) -> np.ndarray:
    n, d, indptr, indices, _ = _csr(A)
    out = np.empty(d, dtype=np.int64)
    _load().oracle_column_counts(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(out, _I64P))
    return out


def reweight(n: int, counts: np.ndarray) -> np.ndarray:
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    D = np.empty(counts.shape[0], dtype=np.float64)
    _load().oracle_reweight(n, counts.shape[0], _p(counts, _I64P), _p(D, _F64P))
    return D


def lipschitz(A, lam: float) -> float:
    n, _, indptr, _, data = _csr(A)
    return float(_load().oracle_lipschitz(n, _p(indptr, _I64P), _p(data, _F64P), lam))


def sigma(b: float, z: float) -> float:
    return float(_load().oracle_sigma(b, z))


# --------------------------------------------------------------------------- objective
def objective(A, y: np.ndarray, lam: float, x: np.ndarray) -> float:
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_load().oracle_objective(n, d, _p(indptr, _I64P), _p(indices, _I32P),
                                          _p(data, _F64P), _p(y, _F64P), lam, _p(x, _F64P)))


def full_grad(A, y: np.ndarray, lam: float, x: np.ndarray) -> np.ndarray:
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    g = np.empty(d, dtype=np.float64)
    _load().oracle_full_grad(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                             _p(y, _F64P), lam, _p(x, _F64P), _p(g, _F64P))
    return g


# --------------------------------------------------------------------------- solver
class State:
    """(x, alpha, alpha_bar, t) of a sequential Sparse SAGA run (reading R1: zeros)."""

    def __init__(self, n: int, d: int):
        self.x = np.zeros(d, dtype=np.float64)
        self.alpha = np.zeros(n, dtype=np.float64)
        self.alpha_bar = np.zeros(d, dtype=np.float64)
        self.t = 0

    def copy(self) -> "State":
        s = State(0, 0)
        s.x, s.alpha, s.alpha_bar, s.t = self.x.copy(), self.alpha.copy(), self.alpha_bar.copy(), self.t
        return s


def sparse_saga(A, y, lam: float, gamma: float, seed: int, T: int, state: State | None = None,
                D: np.ndarray | None = None) -> State:
    """Run T sequential Sparse SAGA updates (t = state.t .. state.t+T-1) in place."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if state is None:
        state = State(n, d)
    if D is None:
        D = reweight(n, column_counts(A))
    _load().oracle_sparse_saga(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                               _p(y, _F64P), _p(D, _F64P), lam, gamma, seed, state.t, T,
                               _p(state.x, _F64P), _p(state.alpha, _F64P),
                               _p(state.alpha_bar, _F64P))
    state.t += T
    return state


def saga_step(A, y, lam: float, gamma: float, i: int, state: State, D: np.ndarray) -> State:
    """Apply one Sparse SAGA step on sample i to ``state`` in place (t is not advanced)."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.float64)
    u = np.empty(max(int(np.diff(indptr).max()), 1), dtype=np.float64)
    _load().oracle_saga_step(n, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                             _p(y, _F64P), _p(D, _F64P), lam, gamma, i, _p(state.x, _F64P),
                             _p(state.alpha, _F64P), _p(state.alpha_bar, _F64P), _p(u, _F64P))
    return state


def delayed_saga(A, y, lam, gamma, seed, T: int, tau: int, state: State | None = None, D=None):
    """Sparse SAGA where every update is written tau updates after its read."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if state is None:
        state = State(n, d)
    if D is None:
        D = reweight(n, column_counts(A))
    _load().oracle_delayed_saga(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                                _p(y, _F64P), _p(D, _F64P), lam, gamma, seed, state.t, T, tau,
                                _p(state.x, _F64P), _p(state.alpha, _F64P),
                                _p(state.alpha_bar, _F64P))
    state.t += T
    return state


def replica_saga(A, y, lam, gamma, seed, T: int, N: int, E: int, state: State | None = None, D=None):
    """NEXT-3 model (Section 5): N replicas of (x, abar), update t on replica t mod N,
    each replica's own updates applied to its copy at once, every copy reset to the shared
    value plus everyone's changes every E updates (and at the end)."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if state is None:
        state = State(n, d)
    if D is None:
        D = reweight(n, column_counts(A))
    assert N >= 1 and E >= 1
    _load().oracle_replica_saga(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                                _p(y, _F64P), _p(D, _F64P), lam, gamma, seed, state.t, T, N, E,
                                _p(state.x, _F64P), _p(state.alpha, _F64P),
                                _p(state.alpha_bar, _F64P))
    state.t += T
    return state


def hogwild(A, y, lam, gamma, seed, t0: int, T: int, x: np.ndarray, D=None) -> np.ndarray:
    """HOGWILD's serial form (sparse SGD), updates t0..t0+T-1, x in place."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if D is None:
        D = reweight(n, column_counts(A))
    _load().oracle_hogwild(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                           _p(y, _F64P), _p(D, _F64P), lam, gamma, seed, t0, T, _p(x, _F64P))
    return x


def svrg_snapshot(A, y, xref: np.ndarray):
    """KROMAGNON's synchronised phase: (s_i = sigma_i(x~), mu = (1/n) sum s_i a_i)."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    xref = np.ascontiguousarray(xref, dtype=np.float64)
    s = np.empty(n)
    mu = np.empty(d)
    _load().oracle_svrg_snapshot(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                                 _p(y, _F64P), _p(xref, _F64P), _p(s, _F64P), _p(mu, _F64P))
    return s, mu


def svrg_inner(A, y, lam, gamma, seed, t0: int, T: int, s, mu, x: np.ndarray, D=None):
    """KROMAGNON inner steps t0..t0+T-1 against a snapshot (s, mu); x in place."""
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if D is None:
        D = reweight(n, column_counts(A))
    _load().oracle_svrg_inner(n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P),
                              _p(y, _F64P), _p(D, _F64P), lam, gamma, seed, t0, T,
                              _p(s, _F64P), _p(mu, _F64P), _p(x, _F64P))
    return x


# --------------------------------------------------------------------------- NEXT-4
def _serial(fn, A, y, lam, gamma, seed, T, state, with_D):
    n, d, indptr, indices, data = _csr(A)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if state is None:
        state = State(n, d)
    args = [n, d, _p(indptr, _I64P), _p(indices, _I32P), _p(data, _F64P), _p(y, _F64P)]
    if with_D:
        args.append(_p(reweight(n, column_counts(A)), _F64P))
    args += [lam, gamma, seed, state.t, T, _p(state.x, _F64P), _p(state.alpha, _F64P)]
    if fn != "oracle_alg1_saga":
        args.append(_p(state.alpha_bar, _F64P))
    getattr(_load(), fn)(*args)
    state.t += T
    return state


def dense_saga(A, y, lam, gamma, seed, T: int, state: State | None = None) -> State:
    """Dense SAGA (Eq. 2) with the l2 term: O(d) per step (NEXT-4, desk scale)."""
    return _serial("oracle_dense_saga", A, y, lam, gamma, seed, T, state, False)


def lagged_saga(A, y, lam, gamma, seed, T: int, state: State | None = None) -> State:
    """SAGA with lagged (just-in-time) dense updates, App. C (NEXT-4)."""
    return _serial("oracle_lagged_saga", A, y, lam, gamma, seed, T, state, False)


def alg1_saga(A, y, lam, gamma, seed, T: int, state: State | None = None) -> State:
    """Algorithm 1 run sequentially: abar recomputed from the memory every step (NEXT-4).
    state.alpha_bar is not maintained (Alg. 1 has no stored abar)."""
    return _serial("oracle_alg1_saga", A, y, lam, gamma, seed, T, state, True)
