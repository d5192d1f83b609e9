"""B200-native (sm_100a) MEM fusion library: the data-parallel hot path of arXiv 2309.16818.

The product is libmem.so (C-ABI in include/mem.h, CUDA kernels in csrc/); `mem` is the thin
ctypes binding.  There is no CPU fallback.
"""
__all__ = ["mem", "build"]
