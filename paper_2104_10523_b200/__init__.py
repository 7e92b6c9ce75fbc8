"""B200-native sliced tensor-network contraction path of arXiv:2104.10523 (TNQVM/ExaTN).

The compute path is libtnqvm.so (C-ABI, include/tnqvm.h; CUDA kernels for sm_100a);
``tnqvm`` is its thin ctypes binding.  Build with ``__graft_entry__.build()``.
"""
from .tnqvm import Circuit, Context, Plan, TnqvmError, nccl_unique_id  # noqa: F401
