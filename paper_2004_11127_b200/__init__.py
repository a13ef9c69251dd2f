"""paper_2004_11127_b200 -- B200-native Genred hot path (KeOps, arXiv 2004.11127).

a_i = Reduction_{j=1..N} F(p, x_i, y_j)   (Eq. 1)

``libgenred.so`` (csrc/, C ABI in include/genred.h) holds every kernel; ``genred`` is the thin
ctypes binding and ``dist`` the one-process-per-GPU i-shard / j-shard orchestration over NCCL.
"""
from . import genred  # noqa: F401

__all__ = ["genred"]
