"""Thin Python binding of include/asaga.h (argument marshalling only).

Every step of the hot path runs in libasaga.so's CUDA kernels.  There is no
CPU fallback: if the library cannot be loaded, importing this module raises.
numpy arrays are passed as host pointers; torch CUDA tensors (used only for
device memory and streams) as device pointers.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB

_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)
_F64P = ctypes.POINTER(ctypes.c_double)
_U64P = ctypes.POINTER(ctypes.c_uint64)

STATUS = {0: "ASAGA_OK", 1: "ASAGA_E_INVALID_ARG", 2: "ASAGA_E_BAD_CSR", 3: "ASAGA_E_BAD_LABEL",
          4: "ASAGA_E_CUDA", 5: "ASAGA_E_OOM", 6: "ASAGA_E_DIVERGED", 7: "ASAGA_E_STATE"}


ALGORITHMS = {"asaga": 0, "kromagnon": 1, "hogwild": 2}


class AsagaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class CsrView(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p),
                ("data", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("deterministic", ctypes.c_int),
                ("concurrency", ctypes.c_int64), ("lanes_per_sample", ctypes.c_int),
                ("atomic_mode", ctypes.c_int), ("record_samples", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("bulk_scatter_min_freq", ctypes.c_double),
                ("measure_overlap", ctypes.c_int), ("hot_split_min_freq", ctypes.c_double),
                ("smem_replica_refresh", ctypes.c_int), ("combine_min_freq", ctypes.c_double),
                ("combine_cluster", ctypes.c_int), ("combine_write_through", ctypes.c_int),
                ("combine_max_blocks", ctypes.c_int), ("l2_persist_state", ctypes.c_int),
                ("pipe_late_min_freq", ctypes.c_double), ("pipe_merge_ns", ctypes.c_int),
                ("row_copy_elementwise", ctypes.c_int),
                ("record_layout", ctypes.c_int), ("scatter_unpaired", ctypes.c_int),
                ("d_gather", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("lambda_", ctypes.c_double), ("gamma", ctypes.c_double), ("L", ctypes.c_double),
                ("delta_r", ctypes.c_int64), ("t", ctypes.c_uint64),
                ("concurrency", ctypes.c_int64), ("lanes_per_sample", ctypes.c_int),
                ("deterministic", ctypes.c_int), ("max_row", ctypes.c_int64),
                ("grid", ctypes.c_int), ("block", ctypes.c_int), ("last_run_ms", ctypes.c_double),
                ("bulk_scatter_min_freq", ctypes.c_double), ("overlap_mean", ctypes.c_double),
                ("overlap_max", ctypes.c_int64), ("overlap_samples", ctypes.c_int64),
                ("algorithm", ctypes.c_int), ("hot_split_min_freq", ctypes.c_double),
                ("smem_replica", ctypes.c_int), ("combine_hot", ctypes.c_int),
                ("combine_blocks", ctypes.c_int), ("combine_passes", ctypes.c_int64),
                ("combine_cluster", ctypes.c_int), ("record_layout", ctypes.c_int),
                ("hot_table_slots", ctypes.c_int)]


ABI_FUNCTIONS = {
    # name: (restype, argtypes)
    "asaga_options_default": (None, [ctypes.POINTER(Options)]),
    "asaga_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(CsrView),
                                  ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                  ctypes.POINTER(Options)]),
    "asaga_init_device": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(CsrView),
                                         ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                         ctypes.POINTER(Options)]),
    "asaga_reload": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CsrView), ctypes.c_void_p]),
    "asaga_reload_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CsrView),
                                           ctypes.c_void_p]),
    "asaga_reload_device_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CsrView),
                                                 ctypes.c_void_p]),
    "asaga_reload_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CsrView),
                                                 ctypes.c_void_p]),
    "asaga_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64]),
    "asaga_run_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64]),
    "asaga_objective": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _F64P]),
    "asaga_full_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "asaga_objective_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "asaga_partial_obj_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p]),
    "asaga_get_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, _U64P]),
    "asaga_set_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, _U64P]),
    "asaga_get_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "asaga_get_sample_counts": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "asaga_get_sample_hash": (ctypes.c_int, [ctypes.c_void_p, _U64P, ctypes.c_int]),
    "asaga_set_gamma": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double]),
    "asaga_set_algorithm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "asaga_snapshot": (ctypes.c_int, [ctypes.c_void_p]),
    "asaga_set_concurrency": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "asaga_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Stats)]),
    "asaga_debug_sigma": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_void_p]),
    "asaga_sample_indices": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                            ctypes.c_void_p]),
    "asaga_stream": (ctypes.c_void_p, [ctypes.c_void_p]),
    "asaga_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "asaga_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "asaga_abi_version": (ctypes.c_int, []),
    "asaga_destroy": (None, [ctypes.c_void_p]),
}


def _load():
    # ASAGA_LIB selects a profiling build (tools/phase_timing.py); default: the in-tree build
    path = os.environ.get("ASAGA_LIB", LIB)
    if not os.path.exists(path):
        raise ImportError(
            f"libasaga.so not found at {path}: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in ABI_FUNCTIONS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


def lib():
    return _lib


def _check(status: int, ctx=None):
    if status != 0:
        msg = _lib.asaga_last_error(ctx)
        raise AsagaError(status, msg.decode() if msg else "")


def _ptr(a) -> int:
    """Address of a numpy array or a torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def _is_cuda(a) -> bool:
    return (not isinstance(a, np.ndarray)) and getattr(a, "is_cuda", False)


def _host(a, dtype):
    """numpy arrays are made contiguous/typed; host torch tensors (e.g. pinned) pass as-is."""
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=dtype)
    assert a.is_contiguous() and a.element_size() == np.dtype(dtype).itemsize, "bad host tensor"
    return a


class Asaga:
    """One ASAGA context (C-ABI ``asaga_ctx``) on one device.

    ``Asaga(indptr, indices, data, y, d, lam, gamma, ...)`` with numpy arrays uses
    ``asaga_init`` (host CSR, copied to the device); with CUDA torch tensors it uses
    ``asaga_init_device`` (device-resident inputs, copied device-to-device).
    """

    def __init__(self, indptr, indices, data, y, d: int, lam: float, gamma: float, *,
                 deterministic: bool = False, concurrency: int = 0, lanes_per_sample: int = 0,
                 atomic: bool = True, record_samples: bool = False, device: int = 0,
                 stream=None, bulk_scatter_min_freq: float = 0.0, measure_overlap: int = 0,
                 hot_split_min_freq: float = 0.0, smem_replica_refresh: int = 0,
                 combine_min_freq: float = 0.0, combine_cluster: int = 0,
                 combine_write_through: bool = False, combine_max_blocks: int = 0,
                 l2_persist_state: bool = False, pipe_late_min_freq: float = 0.0,
                 pipe_merge_ns: int = 0, row_copy_elementwise: bool = False,
                 record_layout: bool = False, scatter_unpaired: bool = False,
                 d_gather: bool = False):
        n = int(indptr.shape[0]) - 1
        nnz = int(indices.shape[0])
        device_inputs = _is_cuda(indptr)
        if not device_inputs:
            indptr, indices = _host(indptr, np.int64), _host(indices, np.int32)
            data, y = _host(data, np.float64), _host(y, np.float64)
        self._keep = (indptr, indices, data, y)
        view = CsrView(n, int(d), nnz, _ptr(indptr), _ptr(indices), _ptr(data))
        opt = Options()
        _lib.asaga_options_default(ctypes.byref(opt))
        opt.device = device
        opt.deterministic = int(bool(deterministic))
        opt.concurrency = int(concurrency)
        opt.lanes_per_sample = int(lanes_per_sample)
        opt.atomic_mode = int(bool(atomic))
        opt.record_samples = int(bool(record_samples))
        opt.stream = stream
        opt.bulk_scatter_min_freq = float(bulk_scatter_min_freq)
        opt.measure_overlap = int(measure_overlap)
        opt.hot_split_min_freq = float(hot_split_min_freq)
        opt.smem_replica_refresh = int(smem_replica_refresh)
        opt.combine_min_freq = float(combine_min_freq)
        opt.combine_cluster = int(combine_cluster)
        opt.combine_write_through = int(bool(combine_write_through))
        opt.combine_max_blocks = int(combine_max_blocks)
        opt.l2_persist_state = int(bool(l2_persist_state))
        opt.pipe_late_min_freq = float(pipe_late_min_freq)
        opt.pipe_merge_ns = int(pipe_merge_ns)
        opt.row_copy_elementwise = int(bool(row_copy_elementwise))
        opt.record_layout = int(bool(record_layout))
        opt.scatter_unpaired = int(bool(scatter_unpaired))
        opt.d_gather = int(bool(d_gather))
        h = ctypes.c_void_p()
        fn = _lib.asaga_init_device if device_inputs else _lib.asaga_init
        st = fn(ctypes.byref(h), ctypes.byref(view), _ptr(y), float(lam), float(gamma),
                ctypes.byref(opt))
        self._h = None
        _check(st, None)
        self._h = h
        # device arrays are borrowed by the context (read until the next reload / close)
        self._keep = (indptr, indices, data, y) if device_inputs else None
        self.n, self.d, self.nnz = n, int(d), nnz
        self.lam = float(lam)
        self.device = device

    @classmethod
    def from_problem(cls, p, gamma: float, lam: float | None = None, **kw) -> "Asaga":
        return cls(p.indptr, p.indices, p.data, p.y, p.d, p.lam if lam is None else lam, gamma, **kw)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            _lib.asaga_destroy(self._h)  # synchronises the context's streams
            self._h = None
            self._retired = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ hot path
    def reload(self, indptr, indices, data, y) -> None:
        """Re-ingest a same-shape matrix (numpy: host path; CUDA tensors: device path)."""
        dev = _is_cuda(indptr)
        if not dev:
            indptr, indices = _host(indptr, np.int64), _host(indices, np.int32)
            data, y = _host(data, np.float64), _host(y, np.float64)
        view = CsrView(int(indptr.shape[0]) - 1, self.d, int(indices.shape[0]), _ptr(indptr),
                       _ptr(indices), _ptr(data))
        fn = _lib.asaga_reload_device if dev else _lib.asaga_reload
        _check(fn(self._h, ctypes.byref(view), _ptr(y)), self._h)
        self._borrow((indptr, indices, data, y) if dev else None)  # borrowed device arrays

    def reload_async(self, indptr, indices, data, y) -> None:
        """Non-blocking re-ingest; validation is reported by the next blocking call.
        CUDA tensors: borrowed by the context until the next reload / close
        (asaga_reload_device_async).  Host arrays (page-locked for the copy to overlap
        earlier work): copied on the context's copy stream into one of two device buffers
        (asaga_reload_async); they must stay unchanged until the next blocking call."""
        dev = _is_cuda(indptr)
        if not dev:
            indptr, indices = _host(indptr, np.int64), _host(indices, np.int32)
            data, y = _host(data, np.float64), _host(y, np.float64)
        view = CsrView(int(indptr.shape[0]) - 1, self.d, int(indices.shape[0]), _ptr(indptr),
                       _ptr(indices), _ptr(data))
        fn = _lib.asaga_reload_device_async if dev else _lib.asaga_reload_async
        _check(fn(self._h, ctypes.byref(view), _ptr(y)), self._h)
        # (references replaced only after the call: it first waits for the previous host
        # copy, which reads the previous host arrays)
        if dev:
            self._borrow((indptr, indices, data, y))
        else:
            self._keep_host = (indptr, indices, data, y)

    def _borrow(self, arrays) -> None:
        """Replace the borrowed device arrays.  Work already enqueued on the context's stream
        (e.g. an earlier run_async) may still read the previous ones, and torch's caching
        allocator does not know that stream: keep them alive, with an event recorded on the
        context's stream now, until that event has completed (checked at every reload; all
        released at close, which synchronises the stream)."""
        old = getattr(self, "_keep", None)
        if old is not None and self._h:
            import torch

            ev = torch.cuda.Event()
            ev.record(torch.cuda.ExternalStream(self.stream, device=old[0].device))
            self._retired = [(e, k) for e, k in getattr(self, "_retired", []) if not e.query()]
            self._retired.append((ev, old))
        self._keep = arrays

    def run(self, n_updates: int, seed: int) -> None:
        _check(_lib.asaga_run(self._h, int(n_updates), int(seed)), self._h)

    def run_async(self, n_updates: int, seed: int) -> None:
        _check(_lib.asaga_run_async(self._h, int(n_updates), int(seed)), self._h)

    def objective(self, x: np.ndarray | None = None) -> float:
        f = ctypes.c_double()
        xx = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        _check(_lib.asaga_objective(self._h, _ptr(xx), ctypes.byref(f)), self._h)
        return f.value

    def objective_device(self, f_dev, x_dev=None) -> None:
        _check(_lib.asaga_objective_device(self._h, _ptr(x_dev), _ptr(f_dev)), self._h)

    def full_grad(self, x: np.ndarray | None = None) -> np.ndarray:
        g = np.empty(self.d, dtype=np.float64)
        xx = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        _check(_lib.asaga_full_grad(self._h, _ptr(xx), _ptr(g)), self._h)
        return g

    def partial_obj_grad(self, x_dev, out_dev, stream=None) -> None:
        _check(_lib.asaga_partial_obj_grad(self._h, _ptr(x_dev), _ptr(out_dev), stream), self._h)

    # ------------------------------------------------------------------ state
    def get_state(self):
        x = np.empty(self.d)
        alpha = np.empty(self.n)
        ab = np.empty(self.d)
        t = ctypes.c_uint64()
        _check(_lib.asaga_get_state(self._h, _ptr(x), _ptr(alpha), _ptr(ab), ctypes.byref(t)),
               self._h)
        return x, alpha, ab, t.value

    def set_state(self, x=None, alpha=None, alpha_bar=None, t: int | None = None) -> None:
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64)
                for a in (x, alpha, alpha_bar)]
        tt = None if t is None else ctypes.byref(ctypes.c_uint64(int(t)))
        _check(_lib.asaga_set_state(self._h, *[_ptr(a) for a in arrs], tt), self._h)

    def profile(self):
        counts = np.empty(self.d, dtype=np.int32)
        D = np.empty(self.d, dtype=np.float64)
        _check(_lib.asaga_get_profile(self._h, _ptr(counts), _ptr(D)), self._h)
        return counts, D

    def sample_counts(self, reset: bool = False) -> np.ndarray:
        v = np.empty(self.n, dtype=np.int32)
        _check(_lib.asaga_get_sample_counts(self._h, _ptr(v), int(reset)), self._h)
        return v

    def sample_hash(self, reset: bool = False) -> int:
        """sum over processed t of mix(t, i_t) mod 2^64 (include/asaga.h asaga_get_sample_hash)."""
        h = ctypes.c_uint64()
        _check(_lib.asaga_get_sample_hash(self._h, ctypes.byref(h), int(reset)), self._h)
        return h.value

    def set_gamma(self, gamma: float) -> None:
        _check(_lib.asaga_set_gamma(self._h, float(gamma)), self._h)

    def set_algorithm(self, name: str) -> None:
        """'asaga' | 'kromagnon' | 'hogwild' (NEXT-2 comparison methods on the same kernel)."""
        _check(_lib.asaga_set_algorithm(self._h, ALGORITHMS[name]), self._h)

    def snapshot(self) -> None:
        """KROMAGNON's synchronised phase at the current iterate."""
        _check(_lib.asaga_snapshot(self._h), self._h)

    def set_concurrency(self, c: int) -> None:
        _check(_lib.asaga_set_concurrency(self._h, int(c)), self._h)

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.asaga_stats(self._h, ctypes.byref(s)), self._h)
        out = {f: getattr(s, f) for f, _ in Stats._fields_}
        out["lambda"] = out.pop("lambda_")
        return out

    @property
    def stream(self) -> int:
        return _lib.asaga_stream(self._h)


def sample_indices(seed: int, t0: int, count: int, n: int, out_dev, device: int = 0,
                   stream=None) -> None:
    """Fill the int64 CUDA tensor ``out_dev`` with i_{t0..t0+count-1} (the kernel's sampler)."""
    _check(_lib.asaga_sample_indices(device, int(seed), int(t0), int(count), int(n),
                                     _ptr(out_dev), stream))


def debug_sigma(m_dev, out_dev, device: int = 0, stream=None) -> None:
    """out_dev = -1 / (1 + exp(m_dev)) by the update kernels' device function (CUDA float64
    tensors of equal length; a test hook)."""
    assert m_dev.numel() == out_dev.numel()
    _check(_lib.asaga_debug_sigma(device, _ptr(m_dev), _ptr(out_dev), int(m_dev.numel()), stream))
