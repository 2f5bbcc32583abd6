"""B200-native ASAGA hot path (arXiv 1606.04809): lock-free Sparse SAGA on sm_100a.

The product is ``libasaga.so`` (C-ABI in ``include/asaga.h``); this package is
its thin Python binding plus the multi-GPU plumbing (``sharded``) that uses
``torch.distributed`` over NCCL.  Importing it loads the CUDA library and fails
loudly if it is missing -- there is no CPU fallback.
"""
from .asaga import Asaga, AsagaError, debug_sigma, sample_indices  # noqa: F401

__all__ = ["Asaga", "AsagaError", "debug_sigma", "sample_indices"]
