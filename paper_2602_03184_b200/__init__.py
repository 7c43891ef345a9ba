"""B200-native DynSplit-KV hot path (arXiv 2602.03184).

The compute lives in libdynsplit.so (hand-written sm_100a CUDA behind the C
ABI in include/dynsplit.h); `dynsplit` is the thin ctypes binding and
`parallel` the multi-GPU plumbing (torch.distributed).
"""
from . import dynsplit  # noqa: F401

__all__ = ["dynsplit"]
