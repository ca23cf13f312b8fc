"""ctypes wrapper of the CPU oracle (oracle/_build/libhps_oracle.so).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg; the product package never imports it.  The
oracle restates /root/reference/SPEC.md (see oracle/hps_oracle.hpp for the
file:line map and SURVEY.md Appendix A for the interpretations it pins).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhps_oracle.so")
_lib = None

_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.hpso_last_error.restype = C.c_char_p
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _ck(rc):
    if rc != 0:
        raise OracleError(rc, lib().hpso_last_error().decode())


def _p(a, t=_d):
    return None if a is None else a.ctypes.data_as(t)


def cheb_nodes(p, allow_small=False):
    x = np.empty(p)
    _ck(lib().hpso_cheb_nodes(p, int(allow_small), _p(x)))
    return x


def cheb_diff(p, allow_small=False):
    D = np.empty((p, p))
    _ck(lib().hpso_cheb_diff(p, int(allow_small), _p(D)))
    return D


def scale_to_interval(D, a):
    D = np.ascontiguousarray(D, dtype=np.float64)
    out = np.empty_like(D)
    _ck(lib().hpso_scale_to_interval(D.shape[0], _p(D), C.c_double(a), _p(out)))
    return out


def leaf_constants(p, a, kappa):
    Ds = np.empty((p, p)); D2 = np.empty((p, p))
    _ck(lib().hpso_leaf_constants(p, C.c_double(a), C.c_double(kappa), _p(Ds), _p(D2)))
    return Ds, D2


def leaf_index(p):
    ni, nb = (p - 2) ** 2, 4 * (p - 1)
    it = np.empty(ni, np.int32); bd = np.empty(nb, np.int32)
    _ck(lib().hpso_leaf_index(p, _p(it, _i32), _p(bd, _i32)))
    return it, bd


def build_leaf(p, a, kappa, b):
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(p * p)
    A = np.empty((p * p, p * p)); Dn = np.empty((4 * (p - 1), p * p))
    _ck(lib().hpso_build_leaf(p, C.c_double(a), C.c_double(kappa), _p(b), _p(A), _p(Dn)))
    return A, Dn


def batched_condense(p, a, kappa, b, f, want_S=False, want_lu=False, workers=0, inject=(),
                     raise_on_resonance=True):
    """b, f: (n_leaves, p*p).  Returns dict with T (n, nb, nb), w (n, nb), S, lu, ipiv, status."""
    b = np.ascontiguousarray(b, dtype=np.float64); f = np.ascontiguousarray(f, dtype=np.float64)
    n = b.shape[0]
    ni, nb = (p - 2) ** 2, 4 * (p - 1)
    T = np.empty((n, nb, nb)); w = np.empty((n, nb))
    S = np.empty((n, ni, nb)) if want_S else None
    lu = np.empty((n, ni, ni)) if want_lu else None  # column-major per leaf
    ipiv = np.empty((n, ni), np.int32) if want_lu else None
    status = np.zeros(n, np.int32); ratio = np.empty(n)
    inj = np.asarray(inject, np.int32)
    rc = lib().hpso_batched_condense(p, C.c_double(a), C.c_double(kappa), n, _p(b), _p(f), _p(T), _p(w),
                                     _p(S), _p(lu), _p(ipiv, _i32), _p(status, _i32), _p(ratio), workers,
                                     _p(inj, _i32), len(inj))
    if rc != 0 and (rc != 1 or raise_on_resonance):
        _ck(rc)
    return dict(T=T, w=w, S=S, lu=lu, ipiv=ipiv, status=status, min_pivot_ratio=ratio)


def batched_leaf_solve(p, a, kappa, b, f, v, lu=None, ipiv=None, workers=0, inject=()):
    b = np.ascontiguousarray(b, dtype=np.float64); f = np.ascontiguousarray(f, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    n = b.shape[0]
    u = np.empty((n, p * p)); status = np.zeros(n, np.int32)
    inj = np.asarray(inject, np.int32)
    _ck(lib().hpso_batched_leaf_solve(p, C.c_double(a), C.c_double(kappa), n, _p(b), _p(f), _p(v), _p(u),
                                      _p(lu), _p(ipiv, _i32), _p(status, _i32), workers,
                                      _p(inj, _i32), len(inj)))
    return u


def mesh_info(nx, ny, p):
    N = C.c_int64(); ne = C.c_int32(); na = C.c_int64()
    _ck(lib().hpso_mesh_info(nx, ny, p, C.byref(N), C.byref(ne), C.byref(na)))
    return N.value, ne.value, na.value


def mesh_maps(nx, ny, p):
    _, ne, _ = mesh_info(nx, ny, p)
    ee = np.empty((nx * ny, 4), np.int32); el = np.empty((ne, 2), np.int32); sd = np.empty((ne, 2), np.int32)
    _ck(lib().hpso_mesh_maps(nx, ny, p, _p(ee, _i32), _p(el, _i32), _p(sd, _i32)))
    return ee, el, sd


def element_node_index(nx, ny, p, e):
    out = np.empty(p * p, np.int64)
    _ck(lib().hpso_element_node_index(nx, ny, p, e, _p(out, _i64)))
    return out


def active_of_global(nx, ny, p, g):
    g = np.ascontiguousarray(g, dtype=np.int64)
    out = np.empty_like(g)
    _ck(lib().hpso_active_of_global(nx, ny, p, g.size, _p(g, _i64), _p(out, _i64)))
    return out


def reduced_pattern(nx, ny, p):
    _, _, na = mesh_info(nx, ny, p)
    nnz = C.c_int64()
    _ck(lib().hpso_reduced_nnz(nx, ny, p, C.byref(nnz)))
    rp = np.empty(na + 1, np.int64); ci = np.empty(nnz.value, np.int32)
    _ck(lib().hpso_reduced_pattern(nx, ny, p, _p(rp, _i64), _p(ci, _i32)))
    return rp, ci


def assemble_reduced(nx, ny, p, T, w, g_bnd):
    rp, ci = reduced_pattern(nx, ny, p)
    T = np.ascontiguousarray(T, dtype=np.float64); w = np.ascontiguousarray(w, dtype=np.float64)
    g_bnd = np.ascontiguousarray(g_bnd, dtype=np.float64)
    vals = np.empty(ci.size); rhs = np.empty(rp.size - 1)
    _ck(lib().hpso_assemble_reduced(nx, ny, p, _p(T), _p(w), _p(g_bnd), _p(vals), _p(rhs)))
    return rp, ci, vals, rhs


def hardware_workers():
    return lib().hpso_hardware_workers()


def build_info():
    """Which batching/error headers the oracle was compiled against (the reference's own
    proj/include/hps/{parallel,errors}.hpp when /root/reference was present at build time)."""
    f = lib().hpso_build_info
    f.restype = C.c_char_p
    return f().decode()
