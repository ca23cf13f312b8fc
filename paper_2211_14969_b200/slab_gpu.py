"""ctypes binding of the GPU SlabLU solver (include/hps_slablu.h, libhps_slablu_b200.so;
SURVEY.md §8f row f1): the reference's slablu module on the B200 --
partition_slabs / factor / solve of the reduced interface system given in its BSR view
(leaf_gpu.LeafStage.reduced_bsr_pattern + assemble_reduced_bsr).  Errors follow
proj/include/hps/errors.hpp: ParameterError, SingularBlockError(block_index)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .leaf_gpu import CudaError, ParameterError, _f64, _ptr

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhps_slablu_b200.so")
HPS_OK, HPS_ERR_PARAM, HPS_ERR_CUDA, HPS_ERR_SINGULAR_BLOCK = 0, 2, 3, 4


class SingularBlockError(RuntimeError):
    """hps::SingularBlockError(block_index) (errors.hpp:30-38): interface k >= 0, or
    -1 - s for the interior of slab s."""

    def __init__(self, block_index, msg):
        super().__init__(msg)
        self.block_index = block_index


class _Info(C.Structure):
    _fields_ = [("slab_width", C.c_int32), ("n_slabs", C.c_int32), ("n_active", C.c_int64),
                ("max_interior", C.c_int64), ("n_interface", C.c_int64), ("device_bytes", C.c_int64),
                ("ms_factor", C.c_float), ("ms_solve", C.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.hps_slablu_last_error.restype = C.c_char_p
        L.hps_slablu_last_error.argtypes = [C.c_void_p]
        L.hps_slablu_factor.argtypes = [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.hps_slablu_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.hps_slablu_get_info.argtypes = [C.c_void_p, C.POINTER(_Info)]
        L.hps_slablu_destroy.argtypes = [C.c_void_p]
        L.hps_slablu_default_width.restype = C.c_int32
        L.hps_slablu_default_width.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64]
        _lib = L
    return _lib


def default_width(p, nx, ny, budget_bytes):
    """SPEC.md:421 default width ceil(n_active_per_column^(1/3)) clamped to [1, nx/2], reduced
    until the dense factorization fits `budget_bytes` (> 0: no GPU query)."""
    return lib().hps_slablu_default_width(p, nx, ny, int(budget_bytes))


def _raise(rc, msg):
    if rc == HPS_ERR_PARAM:
        raise ParameterError(msg)
    if rc == HPS_ERR_SINGULAR_BLOCK:
        raise SingularBlockError(lib().hps_slablu_last_block(), msg)
    raise CudaError(msg)


class SlabLU:
    """factor() at construction from the BSR view of the reduced system; solve(rhs)."""

    def __init__(self, p, nx, ny, brow_ptr, bcol_idx, blocks, slab_width=0, device=0):
        L = lib()
        rp = np.ascontiguousarray(brow_ptr, np.int64); ci = np.ascontiguousarray(bcol_idx, np.int32)
        bl = _f64(blocks)
        h = C.c_void_p()
        rc = L.hps_slablu_factor(device, p, nx, ny, slab_width, _ptr(rp), _ptr(ci), _ptr(bl), C.byref(h))
        if rc != HPS_OK:
            _raise(rc, L.hps_slablu_last_error(None).decode())
        self._h = h
        self.info = self.get_info()

    def get_info(self):
        i = _Info()
        lib().hps_slablu_get_info(self._h, C.byref(i))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def solve(self, rhs):
        rhs = _f64(rhs, (-1,))
        if rhs.size != self.info["n_active"]:
            raise ParameterError(f"rhs: {rhs.size} values, {self.info['n_active']} expected")
        x = np.empty_like(rhs)
        rc = lib().hps_slablu_solve(self._h, _ptr(rhs), _ptr(x))
        if rc != HPS_OK:
            _raise(rc, lib().hps_slablu_last_error(self._h).decode())
        return x

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_slablu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
