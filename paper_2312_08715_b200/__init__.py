"""B200-native Bayes3D pose-enumeration hot path (arXiv 2312.08715).

C ABI: include/b3d_b200.h, implemented by _lib/libb3d_b200.so (csrc/).
"""
from . import b3d, configs, synth  # noqa: F401

__all__ = ["b3d", "configs", "synth"]
