"""B200-native ring KV-cache replication (KevlarFlow, arXiv 2601.22438).

libkvring.so (C ABI, include/kvring.h) holds the allocator, the step
protocol and the sm_100a kernels; ``kvring`` is its thin ctypes binding and
``runtime`` places logical nodes on GPUs and links them into a ring.
"""
from . import kvring

__all__ = ["kvring"]
