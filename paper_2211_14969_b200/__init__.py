"""B200-native HPS leaf stage (arXiv 2211.14969): batched static condensation of
p x p Chebyshev leaves on sm_100a, behind the reference's leaf/assembly interface.

The product is libhps_leaf_b200.so (CUDA kernels + C-ABI, include/hps_leaf_gpu.h)
and its C++ API (include/hps/leaf_gpu.hpp).  ``leaf_gpu`` is the ctypes binding
used by tests and bench.py; ``problems`` samples b, f, g on the leaf grid.
"""
__all__ = ["leaf_gpu", "problems"]
