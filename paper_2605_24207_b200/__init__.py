"""paper_2605_24207_b200 -- B200-native lifted join-aggregate of RelaNN's Neuro-Relational Algebra.

The product is librnn.so (C ABI, include/rnn.h, CUDA kernels for sm_100a under csrc/);
``rnn`` is its thin ctypes binding and ``programs`` drives the paper's workloads (GCN,
HGT, hypergraph, DHN) through it.  PyTorch provides device memory, streams and
process groups only.
"""
from . import rnn  # noqa: F401

__all__ = ["rnn"]
