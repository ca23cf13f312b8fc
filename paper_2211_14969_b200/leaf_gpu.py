"""ctypes binding of the C-ABI in include/hps_leaf_gpu.h (libhps_leaf_b200.so).

Python-side handle on the B200 leaf stage for tests and bench.py.  It mirrors
the reference's operation set: ``batched_condense``,
``leaf_solve``, ``assemble_reduced``, with ParameterError / ResonanceError as in
proj/include/hps/errors.hpp:10-26.  There is no CPU fallback: if the CUDA
library is missing or no GPU is visible the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPS_LIB_PATH: load an alternative build of the same library (kernel-variant A/B runs).
LIB_PATH = os.environ.get("HPS_LIB_PATH") or os.path.join(_HERE, "_lib", "libhps_leaf_b200.so")

HPS_OK, HPS_ERR_RESONANCE, HPS_ERR_PARAM, HPS_ERR_CUDA = 0, 1, 2, 3
OPT_SMALL_KERNEL, OPT_LOCKSTEP = 1, 2
STORAGE_RECOMPUTE, STORAGE_STORE, STORAGE_S_SOLVE = 0, 1, 2


class ParameterError(ValueError):
    """hps::ParameterError (errors.hpp:10-13)."""


class ResonanceError(RuntimeError):
    """hps::ResonanceError(element_id) (errors.hpp:18-26)."""

    def __init__(self, element_id, msg, failing=()):
        super().__init__(msg)
        self.element_id = element_id
        self.failing = list(failing)


class CudaError(RuntimeError):
    pass


class _Desc(C.Structure):
    _fields_ = [("p", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("storage", C.c_int32),
                ("a", C.c_double), ("kappa", C.c_double), ("workspace_bytes", C.c_int64)]


class _Info(C.Structure):
    _fields_ = [("p", C.c_int32), ("n_i", C.c_int32), ("n_b", C.c_int32), ("n_leaves", C.c_int32),
                ("chunk_leaves", C.c_int32), ("resident_ctas", C.c_int32),
                ("workspace_bytes_per_leaf", C.c_int64), ("n_active", C.c_int64), ("N", C.c_int64)]


class _Timing(C.Structure):
    _fields_ = [("ms_total", C.c_float), ("ms_assemble", C.c_float), ("ms_lu_schur", C.c_float),
                ("ms_scatter", C.c_float), ("kernels", C.c_int32), ("chunks", C.c_int32)]


_lib = None
EXPORTED = ["hps_gpu_create", "hps_gpu_destroy", "hps_gpu_last_error", "hps_gpu_get_info",
            "hps_gpu_get_timing", "hps_gpu_reset_timing", "hps_gpu_condense", "hps_gpu_condense_device", "hps_gpu_leaf_solve",
            "hps_gpu_reduced_pattern", "hps_gpu_assemble_reduced", "hps_gpu_assemble_reduced_device",
            "hps_gpu_set_fault_injection", "hps_host_alloc", "hps_host_free", "hps_gpu_version",
            "hps_gpu_sample_crystal", "hps_gpu_residual", "hps_gpu_residual_device",
            "hps_gpu_reduced_bsr_pattern", "hps_gpu_assemble_reduced_bsr",
            "hps_gpu_assemble_reduced_bsr_device", "hps_gpu_scatter_indices",
            "hps_gpu_build_leaf_operator", "hps_gpu_condense_operator", "hps_gpu_leaf_solve_operator",
            "hps_gpu_multi_create", "hps_gpu_multi_destroy", "hps_gpu_multi_last_error", "hps_gpu_multi_shards",
            "hps_gpu_multi_ctx", "hps_gpu_multi_condense", "hps_gpu_multi_leaf_solve",
            "hps_gpu_multi_assemble_reduced", "hps_shard_range", "hps_reduced_cut_edges",
            "hps_reduced_host_edges", "hps_gpu_condense_assemble", "hps_gpu_reconstruct",
            "hps_gpu_reconstruct_device", "hps_gpu_fp64_peak_tflops", "hps_gpu_fp64_peak_tflops_sustained",
            "hps_gpu_set_option"]


def lib():
    """Load libhps_leaf_b200.so (fails loudly when the CUDA build is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.hps_gpu_last_error.restype = C.c_char_p
        L.hps_gpu_last_error.argtypes = [C.c_void_p]
        L.hps_gpu_version.restype = C.c_char_p
        L.hps_gpu_fp64_peak_tflops.restype = C.c_double
        L.hps_gpu_fp64_peak_tflops.argtypes = [C.c_int]
        L.hps_gpu_fp64_peak_tflops_sustained.restype = C.c_double
        L.hps_gpu_fp64_peak_tflops_sustained.argtypes = [C.c_int, C.c_double]
        L.hps_gpu_create.argtypes = [C.c_int, C.POINTER(_Desc), C.POINTER(C.c_void_p)]
        L.hps_gpu_destroy.argtypes = [C.c_void_p]
        L.hps_host_alloc.restype = C.c_void_p
        L.hps_host_alloc.argtypes = [C.c_size_t]
        L.hps_host_free.argtypes = [C.c_void_p]
        L.hps_gpu_multi_last_error.restype = C.c_char_p
        L.hps_gpu_multi_last_error.argtypes = [C.c_void_p]
        L.hps_gpu_multi_create.argtypes = [C.c_void_p, C.c_int32, C.POINTER(_Desc), C.POINTER(C.c_void_p)]
        L.hps_gpu_multi_destroy.argtypes = [C.c_void_p]
        L.hps_gpu_multi_ctx.restype = C.c_void_p
        for name in ("hps_gpu_condense", "hps_gpu_condense_device", "hps_gpu_leaf_solve",
                     "hps_gpu_reduced_pattern", "hps_gpu_assemble_reduced",
                     "hps_gpu_assemble_reduced_device", "hps_gpu_set_fault_injection",
                     "hps_gpu_get_info", "hps_gpu_get_timing", "hps_gpu_reset_timing",
                     "hps_gpu_sample_crystal", "hps_gpu_residual", "hps_gpu_residual_device",
                     "hps_gpu_reduced_bsr_pattern", "hps_gpu_assemble_reduced_bsr",
                     "hps_gpu_assemble_reduced_bsr_device", "hps_gpu_scatter_indices",
                     "hps_gpu_build_leaf_operator", "hps_gpu_condense_operator",
                     "hps_gpu_leaf_solve_operator", "hps_gpu_multi_shards", "hps_gpu_multi_condense",
                     "hps_gpu_multi_leaf_solve", "hps_gpu_multi_assemble_reduced", "hps_shard_range",
                     "hps_reduced_cut_edges", "hps_reduced_host_edges", "hps_gpu_condense_assemble",
                     "hps_gpu_reconstruct", "hps_gpu_reconstruct_device", "hps_gpu_set_option"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        try:
            a = a.reshape(shape)
        except ValueError as e:
            raise ParameterError(f"input of shape {a.shape} cannot be viewed as {shape}") from e
    return a


def _rows(a, n, name):
    """Inputs handed to the C-ABI must cover exactly the n leaves of the call."""
    if a.shape[0] != n:
        raise ParameterError(f"{name}: {a.shape[0]} leaves given, {n} expected")
    return a


def _out(a, shape, dtype, name):
    """Caller-provided outputs are written through raw pointers: they must be C-contiguous,
    of the exact dtype and shape, and writeable (ParameterError otherwise)."""
    if not isinstance(a, np.ndarray) or a.dtype != np.dtype(dtype) or tuple(a.shape) != tuple(shape) \
            or not a.flags.c_contiguous or not a.flags.writeable:
        got = (getattr(a, "shape", None), getattr(a, "dtype", None))
        raise ParameterError(f"{name}: need a writeable C-contiguous {np.dtype(dtype)} array of shape "
                             f"{tuple(shape)}, got {got}")
    return a


class LeafStage:
    """One GPU context (hps_gpu_ctx) for an nx x ny mesh of p x p leaves."""

    def __init__(self, p, nx, ny, kappa, a=None, storage=STORAGE_RECOMPUTE, device=0,
                 workspace_bytes=0):
        L = lib()
        d = _Desc(p=p, nx=nx, ny=ny, storage=storage, a=(1.0 / nx if a is None else a),
                  kappa=kappa, workspace_bytes=int(workspace_bytes))
        h = C.c_void_p()
        rc = L.hps_gpu_create(device, C.byref(d), C.byref(h))
        if rc != HPS_OK:
            msg = L.hps_gpu_last_error(None).decode()
            raise (ParameterError if rc == HPS_ERR_PARAM else CudaError)(msg)
        self._h = h
        self.p, self.nx, self.ny, self.kappa = p, nx, ny, kappa
        self.n_leaves = nx * ny
        self.n_i, self.n_b = (p - 2) ** 2, 4 * (p - 1)

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_gpu_destroy(self._h)
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

    # -- errors -------------------------------------------------------------------------------
    def _check(self, rc, status=None, e0=0):
        if rc == HPS_OK:
            return
        msg = lib().hps_gpu_last_error(self._h).decode()
        if rc == HPS_ERR_RESONANCE:
            failing = [] if status is None else [e0 + int(i) for i in np.nonzero(status)[0]]
            raise ResonanceError(failing[0] if failing else -1, msg, failing)
        if rc == HPS_ERR_PARAM:
            raise ParameterError(msg)
        raise CudaError(msg)

    # -- info ---------------------------------------------------------------------------------
    def info(self):
        i = _Info()
        self._check(lib().hps_gpu_get_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def timing(self):
        t = _Timing()
        self._check(lib().hps_gpu_get_timing(self._h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in _Timing._fields_}

    def reset_timing(self):
        self._check(lib().hps_gpu_reset_timing(self._h))

    def set_option(self, option, value):
        """Kernel-path selection (hps_gpu_set_option): OPT_SMALL_KERNEL / OPT_LOCKSTEP,
        value -1 default, 0 off, 1 on."""
        self._check(lib().hps_gpu_set_option(self._h, option, value))

    def set_fault_injection(self, elements):
        el = np.asarray(elements, np.int32)
        self._check(lib().hps_gpu_set_fault_injection(self._h, _ptr(el), el.size))

    # -- batched_condense ---------------------------------------------------------------------
    def condense(self, b, f, e0=0, out=None, raise_on_resonance=True, want_S=False):
        """b, f: (n, p*p) host arrays for elements [e0, e0+n).  Returns (T, w, status), plus
        S_solve (n, n_i, n_b) when want_S."""
        pp = self.p * self.p
        b = _f64(b, (-1, pp)); f = _f64(f, (-1, pp))
        n = b.shape[0]
        _rows(f, n, "f")
        if e0 < 0 or e0 + n > self.n_leaves:
            raise ParameterError(f"element range [{e0}, {e0 + n}) outside the mesh of {self.n_leaves} leaves")
        if out is None:
            # pageable: the library stages it through pinned double buffers (a fresh pinned
            # allocation per call costs more than it saves; reuse PinnedArray for speed,
            # tools/py_condense_timing.py)
            T = np.empty((n, self.n_b, self.n_b)); w = np.empty((n, self.n_b))
        else:
            T, w = out
            _out(T, (n, self.n_b, self.n_b), np.float64, "out T")
            _out(w, (n, self.n_b), np.float64, "out w")
        S = np.empty((n, self.n_i, self.n_b)) if want_S else None
        st = np.zeros(n, np.int32)
        rc = lib().hps_gpu_condense(self._h, e0, e0 + n, _ptr(b), _ptr(f), _ptr(T), _ptr(w), _ptr(S), _ptr(st))
        if rc != HPS_OK and (rc != HPS_ERR_RESONANCE or raise_on_resonance):
            self._check(rc, st, e0)
        return (T, w, st, S) if want_S else (T, w, st)

    def condense_device(self, e0, n, d_b, d_f, d_T, d_w, d_status, stream=0):
        """Device-resident variant: arguments are raw device pointers (ints)."""
        rc = lib().hps_gpu_condense_device(self._h, e0, n, C.c_void_p(d_b), C.c_void_p(d_f), C.c_void_p(d_T),
                                           C.c_void_p(d_w), C.c_void_p(d_status), C.c_void_p(stream))
        self._check(rc)

    def sample_crystal_device(self, e0, n, d_b, centres=None, sigma=0.02, depth=0.9, stream=0):
        """Device-side crystal b(x) samples of elements [e0, e0+n) into the device buffer d_b
        (raw pointer), the layout condense_device reads."""
        if centres is None:
            from . import problems
            centres = problems.crystal_centres()
        c = np.ascontiguousarray(np.asarray(centres, dtype=np.float64).reshape(-1, 2))
        rc = lib().hps_gpu_sample_crystal(self._h, e0, n, _ptr(c), c.shape[0], C.c_double(sigma),
                                          C.c_double(depth), C.c_void_p(d_b), C.c_void_p(stream))
        self._check(rc)

    def residual(self, b, f, u_leaf):
        """Matrix-free residual pieces of the global collocation system for local solutions
        u_leaf (n_leaves x p^2): dict(r_int2, r_flux2, f_int2) (Eq. 7)."""
        pp = self.p * self.p
        b = _f64(b, (-1, pp)); f = _f64(f, (-1, pp)); u = _f64(u_leaf, (-1, pp))
        for a, nm in ((b, "b"), (f, "f"), (u, "u")):
            _rows(a, self.n_leaves, nm)
        out = np.zeros(3)
        self._check(lib().hps_gpu_residual(self._h, _ptr(b), _ptr(f), _ptr(u), _ptr(out)))
        return dict(r_int2=out[0], r_flux2=out[1], f_int2=out[2])

    # -- leaf_solve ---------------------------------------------------------------------------
    def leaf_solve(self, b, f, v, e0=0, out=None):
        """Batched leaf_solve for elements [e0, e0+n): (n, p*p) local
        solutions.  `out`: optional caller-owned (n, p*p) float64 array (pinned for overlap)."""
        pp = self.p * self.p
        b = _f64(b, (-1, pp)); f = _f64(f, (-1, pp)); v = _f64(v, (-1, self.n_b))
        n = b.shape[0]
        _rows(f, n, "f"); _rows(v, n, "v")
        if e0 < 0 or e0 + n > self.n_leaves:
            raise ParameterError(f"element range [{e0}, {e0 + n}) outside the mesh of {self.n_leaves} leaves")
        u = np.empty((n, pp)) if out is None else _out(out, (n, pp), np.float64, "out u")
        st = np.zeros(n, np.int32)
        rc = lib().hps_gpu_leaf_solve(self._h, e0, e0 + n, _ptr(b), _ptr(f), _ptr(v), _ptr(u), _ptr(st))
        self._check(rc, st, e0)
        return u

    # -- the SPEC's per-leaf operations on operators held as values ----------
    def build_leaf_operator(self, b, e0=0):
        """build_leaf_operator for elements [e0, e0+n) from their b samples: A_loc (n, p^2, p^2)
        and D_normal (n, 4, p, p^2) (edges S, E, N, W, edge nodes ascending)."""
        pp = self.p * self.p
        b = _f64(b, (-1, pp))
        n = b.shape[0]
        if e0 < 0 or e0 + n > self.n_leaves:
            raise ParameterError(f"element range [{e0}, {e0 + n}) outside the mesh of {self.n_leaves} leaves")
        A = np.empty((n, pp, pp)); Dn = np.empty((n, 4, self.p, pp))
        self._check(lib().hps_gpu_build_leaf_operator(self._h, e0, e0 + n, _ptr(b), _ptr(A), _ptr(Dn)))
        return A, Dn

    def condense_operator(self, A, Dn, f, e0=0, want_S=False, raise_on_resonance=True):
        """condense_leaf of given operators: (T, w, status[, S])."""
        pp = self.p * self.p
        A = _f64(A, (-1, pp, pp)); n = A.shape[0]
        Dn = _rows(_f64(Dn, (-1, 4, self.p, pp)), n, "D_normal"); f = _rows(_f64(f, (-1, pp)), n, "f")
        if e0 < 0 or e0 + n > self.n_leaves:
            raise ParameterError(f"element range [{e0}, {e0 + n}) outside the mesh of {self.n_leaves} leaves")
        T = np.empty((n, self.n_b, self.n_b)); w = np.empty((n, self.n_b)); st = np.zeros(n, np.int32)
        S = np.empty((n, self.n_i, self.n_b)) if want_S else None
        rc = lib().hps_gpu_condense_operator(self._h, e0, e0 + n, _ptr(A), _ptr(Dn), _ptr(f), _ptr(T), _ptr(w),
                                             _ptr(S), _ptr(st))
        if rc != HPS_OK and (rc != HPS_ERR_RESONANCE or raise_on_resonance):
            self._check(rc, st, e0)
        return (T, w, st, S) if want_S else (T, w, st)

    def leaf_solve_operator(self, A, f, v, e0=0):
        """leaf_solve with given A_loc: (n, p^2) local solutions."""
        pp = self.p * self.p
        A = _f64(A, (-1, pp, pp)); n = A.shape[0]
        f = _rows(_f64(f, (-1, pp)), n, "f"); v = _rows(_f64(v, (-1, self.n_b)), n, "v")
        if e0 < 0 or e0 + n > self.n_leaves:
            raise ParameterError(f"element range [{e0}, {e0 + n}) outside the mesh of {self.n_leaves} leaves")
        u = np.empty((n, pp)); st = np.zeros(n, np.int32)
        rc = lib().hps_gpu_leaf_solve_operator(self._h, e0, e0 + n, _ptr(A), _ptr(f), _ptr(v), _ptr(u), _ptr(st))
        self._check(rc, st, e0)
        return u

    def reconstruct(self, u_active, g_bnd, b, f):
        """reconstruct_full_solution on the GPU: the full-grid solution
        (N values, g = gy*Nx + gx) from the reduced solution and g_bnd; b, f all leaves."""
        pp = self.p * self.p
        b = _rows(_f64(b, (-1, pp)), self.n_leaves, "b"); f = _rows(_f64(f, (-1, pp)), self.n_leaves, "f")
        ua = _f64(u_active, (-1,)); g_bnd = _f64(g_bnd, (-1,))
        info = self.info()
        if ua.size != info["n_active"]:
            raise ParameterError(f"u_active: {ua.size} values, {info['n_active']} expected")
        u = np.empty(info["N"]); st = np.zeros(self.n_leaves, np.int32)
        self._check(lib().hps_gpu_reconstruct(self._h, _ptr(ua), _ptr(g_bnd), _ptr(b), _ptr(f), _ptr(u), _ptr(st)),
                    st, 0)
        return u

    # -- assemble_reduced ---------------------------------------------------------------------
    def reduced_pattern(self):
        nnz = C.c_int64()
        self._check(lib().hps_gpu_reduced_pattern(self._h, C.byref(nnz), None, None))
        na = self.info()["n_active"]
        rp = np.empty(na + 1, np.int64); ci = np.empty(max(nnz.value, 1), np.int32)
        self._check(lib().hps_gpu_reduced_pattern(self._h, C.byref(nnz), _ptr(rp), _ptr(ci)))
        return rp, ci[:nnz.value]

    def scatter_indices(self, e0=0, e1=None):
        """Per-leaf scatter map (hps_gpu_scatter_indices): slot (n, nb, nb) int64 positions
        in the CSR values (-1 = not in the reduced matrix) and row (n, nb) active rows."""
        e1 = self.n_leaves if e1 is None else e1
        n = max(e1 - e0, 0)
        slot = np.empty((n, self.n_b, self.n_b), np.int64); row = np.empty((n, self.n_b), np.int64)
        self._check(lib().hps_gpu_scatter_indices(self._h, e0, e1, _ptr(slot), _ptr(row)))
        return slot, row

    def _reduced_inputs(self, T, w, g_bnd):
        T = _f64(T, (-1, self.n_b, self.n_b)); w = _f64(w, (-1, self.n_b)); g_bnd = _f64(g_bnd, (-1,))
        _rows(T, self.n_leaves, "T"); _rows(w, self.n_leaves, "w")
        ng = 2 * (self.nx * (self.p - 1) + 1) + 2 * (self.ny * (self.p - 1) + 1)
        if g_bnd.size != ng:
            raise ParameterError(f"g_bnd: {g_bnd.size} values given, {ng} expected ([S | N | W | E])")
        return T, w, g_bnd

    def assemble_reduced(self, T, w, g_bnd):
        rp, ci = self.reduced_pattern()
        T, w, g_bnd = self._reduced_inputs(T, w, g_bnd)
        vals = np.empty(ci.size); rhs = np.empty(rp.size - 1)
        self._check(lib().hps_gpu_assemble_reduced(self._h, _ptr(T), _ptr(w), _ptr(g_bnd), _ptr(vals), _ptr(rhs)))
        return rp, ci, vals, rhs

    def condense_assemble(self, b, f, g_bnd, want_T=False, out=None, raise_on_resonance=True):
        """batched_condense + assemble_reduced of the whole mesh with T resident in HBM
        (hps_gpu_condense_assemble): (row_ptr, col_idx, values, rhs, status[, T, w]).
        `out`: optional caller-owned (values, rhs) arrays (pinned for full overlap)."""
        pp = self.p * self.p
        b = _rows(_f64(b, (-1, pp)), self.n_leaves, "b"); f = _rows(_f64(f, (-1, pp)), self.n_leaves, "f")
        g_bnd = _f64(g_bnd, (-1,))
        rp, ci = self.reduced_pattern()
        if out is None:
            vals = np.empty(ci.size); rhs = np.empty(rp.size - 1)
        else:
            vals = _out(out[0], (ci.size,), np.float64, "out values")
            rhs = _out(out[1], (rp.size - 1,), np.float64, "out rhs")
        T = np.empty((self.n_leaves, self.n_b, self.n_b)) if want_T else None
        w = np.empty((self.n_leaves, self.n_b)) if want_T else None
        st = np.zeros(self.n_leaves, np.int32)
        rc = lib().hps_gpu_condense_assemble(self._h, _ptr(b), _ptr(f), _ptr(g_bnd), _ptr(vals), _ptr(rhs),
                                             _ptr(T), _ptr(w), _ptr(st))
        if rc != HPS_OK and (rc != HPS_ERR_RESONANCE or raise_on_resonance):
            self._check(rc, st, 0)
        return (rp, ci, vals, rhs, st, T, w) if want_T else (rp, ci, vals, rhs, st)

    def reduced_bsr_pattern(self):
        """BSR pattern of the reduced system (SPEC.md:331 ReducedSystem.blocks): block row =
        interface edge, q x q blocks, q = p-2. Returns (q, brow_ptr, bcol_idx)."""
        q = C.c_int32(); nnzb = C.c_int64()
        self._check(lib().hps_gpu_reduced_bsr_pattern(self._h, C.byref(q), C.byref(nnzb), None, None))
        nbr = self.info()["n_active"] // max(q.value, 1)
        rp = np.empty(nbr + 1, np.int64); ci = np.empty(max(nnzb.value, 1), np.int32)
        self._check(lib().hps_gpu_reduced_bsr_pattern(self._h, C.byref(q), C.byref(nnzb), _ptr(rp), _ptr(ci)))
        return q.value, rp, ci[:nnzb.value]

    def assemble_reduced_bsr(self, T, w, g_bnd):
        """assemble_reduced in BSR: (brow_ptr, bcol_idx, blocks[nnzb, q, q], rhs); the entries
        are bit-identical to assemble_reduced's CSR values."""
        q, rp, ci = self.reduced_bsr_pattern()
        T, w, g_bnd = self._reduced_inputs(T, w, g_bnd)
        vals = np.empty((ci.size, q, q)); rhs = np.empty((rp.size - 1) * q)
        self._check(lib().hps_gpu_assemble_reduced_bsr(self._h, _ptr(T), _ptr(w), _ptr(g_bnd), _ptr(vals), _ptr(rhs)))
        return rp, ci, vals, rhs


def fp64_peak_tflops(device=0, sustained_s=0.0):
    """FP64 tensor (DMMA) peak of the GPU measured now: burst (hps_gpu_fp64_peak_tflops) or,
    with sustained_s > 0, after that many seconds of continuous load
    (hps_gpu_fp64_peak_tflops_sustained)."""
    v = (lib().hps_gpu_fp64_peak_tflops_sustained(device, float(sustained_s)) if sustained_s > 0
         else lib().hps_gpu_fp64_peak_tflops(device))
    if not v > 0:
        raise CudaError("FP64 peak probe failed")
    return v


def shard_range(n, k, i):
    """Leaf range [lo, hi) of shard i of k (hps_shard_range: contiguous, balanced to +-1)."""
    lo, hi = C.c_int32(), C.c_int32()
    if lib().hps_shard_range(n, k, i, C.byref(lo), C.byref(hi)) != HPS_OK:
        raise ParameterError(f"shard_range({n}, {k}, {i})")
    return lo.value, hi.value


def reduced_cut_edges(p, nx, ny, shard_lo):
    """Interface edges whose two elements lie on different shards (host only)."""
    lo = np.ascontiguousarray(shard_lo, np.int32)
    n = C.c_int64()
    if lib().hps_reduced_cut_edges(p, nx, ny, _ptr(lo), lo.size, None, C.byref(n)) != HPS_OK:
        raise ParameterError("reduced_cut_edges")
    out = np.empty(max(n.value, 1), np.int32)
    lib().hps_reduced_cut_edges(p, nx, ny, _ptr(lo), lo.size, _ptr(out), C.byref(n))
    return out[:n.value]


def reduced_host_edges(p, nx, ny, edges, T, w, g_bnd, values, rhs):
    """K4's values/rhs of `edges` on the host, in K4's operation order, into the CSR arrays
    values/rhs (modified in place)."""
    e = np.ascontiguousarray(edges, np.int32)
    T = _f64(T); w = _f64(w); g_bnd = _f64(g_bnd)
    _out(values, values.shape, np.float64, "values"); _out(rhs, rhs.shape, np.float64, "rhs")
    if lib().hps_reduced_host_edges(p, nx, ny, _ptr(e), e.size, _ptr(T), _ptr(w), _ptr(g_bnd), _ptr(values),
                                    _ptr(rhs)) != HPS_OK:
        raise ParameterError("reduced_host_edges")


class MultiLeafStage:
    """Leaf-range sharding of one mesh over several GPU contexts (hps_gpu_multi_*): one host
    thread per ctx, contiguous +-1-balanced ranges, no collective; bitwise equal to a single
    LeafStage.  `devices` may repeat a GPU (several ctxs on one device)."""

    def __init__(self, p, nx, ny, kappa, devices, a=None, storage=STORAGE_RECOMPUTE, workspace_bytes=0):
        L = lib()
        d = _Desc(p=p, nx=nx, ny=ny, storage=storage, a=(1.0 / nx if a is None else a),
                  kappa=kappa, workspace_bytes=int(workspace_bytes))
        dv = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        rc = L.hps_gpu_multi_create(_ptr(dv), dv.size, C.byref(d), C.byref(h))
        if rc != HPS_OK:
            msg = L.hps_gpu_multi_last_error(None).decode()
            raise (ParameterError if rc == HPS_ERR_PARAM else CudaError)(msg)
        self._h = h
        self.p, self.nx, self.ny, self.kappa = p, nx, ny, kappa
        self.n_leaves = nx * ny
        self.n_i, self.n_b = (p - 2) ** 2, 4 * (p - 1)

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_gpu_multi_destroy(self._h)
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

    def _check(self, rc, status=None, e0=0):
        if rc == HPS_OK:
            return
        msg = lib().hps_gpu_multi_last_error(self._h).decode()
        if rc == HPS_ERR_RESONANCE:
            failing = [] if status is None else [e0 + int(i) for i in np.nonzero(status)[0]]
            raise ResonanceError(failing[0] if failing else -1, msg, failing)
        if rc == HPS_ERR_PARAM:
            raise ParameterError(msg)
        raise CudaError(msg)

    def shards(self):
        k = lib().hps_gpu_multi_shards(self._h, None, None)
        lo = np.empty(k, np.int32); hi = np.empty(k, np.int32)
        lib().hps_gpu_multi_shards(self._h, _ptr(lo), _ptr(hi))
        return list(zip(lo.tolist(), hi.tolist()))

    def condense(self, b, f, e0=0, out=None, raise_on_resonance=True):
        pp = self.p * self.p
        b = _f64(b, (-1, pp)); f = _rows(_f64(f, (-1, pp)), b.shape[0], "f")
        n = b.shape[0]
        if out is None:
            T = np.empty((n, self.n_b, self.n_b)); w = np.empty((n, self.n_b))
        else:
            T = _out(out[0], (n, self.n_b, self.n_b), np.float64, "out T")
            w = _out(out[1], (n, self.n_b), np.float64, "out w")
        st = np.zeros(n, np.int32)
        rc = lib().hps_gpu_multi_condense(self._h, e0, e0 + n, _ptr(b), _ptr(f), _ptr(T), _ptr(w), _ptr(st))
        if rc != HPS_OK and (rc != HPS_ERR_RESONANCE or raise_on_resonance):
            self._check(rc, st, e0)
        return T, w, st

    def leaf_solve(self, b, f, v, e0=0):
        pp = self.p * self.p
        b = _f64(b, (-1, pp)); n = b.shape[0]
        f = _rows(_f64(f, (-1, pp)), n, "f"); v = _rows(_f64(v, (-1, self.n_b)), n, "v")
        u = np.empty((n, pp)); st = np.zeros(n, np.int32)
        rc = lib().hps_gpu_multi_leaf_solve(self._h, e0, e0 + n, _ptr(b), _ptr(f), _ptr(v), _ptr(u), _ptr(st))
        self._check(rc, st, e0)
        return u

    def assemble_reduced(self, T, w, g_bnd, pattern_from=None):
        """(row_ptr, col_idx, values, rhs); the pattern comes from shard 0's context."""
        ctx = lib().hps_gpu_multi_ctx(self._h, 0)
        nnz = C.c_int64()
        lib().hps_gpu_reduced_pattern(C.c_void_p(ctx), C.byref(nnz), None, None)
        i = _Info()
        lib().hps_gpu_get_info(C.c_void_p(ctx), C.byref(i))
        na = i.n_active
        rp = np.empty(na + 1, np.int64); ci = np.empty(max(nnz.value, 1), np.int32)
        lib().hps_gpu_reduced_pattern(C.c_void_p(ctx), C.byref(nnz), _ptr(rp), _ptr(ci))
        T = _rows(_f64(T, (-1, self.n_b, self.n_b)), self.n_leaves, "T")
        w = _rows(_f64(w, (-1, self.n_b)), self.n_leaves, "w")
        g_bnd = _f64(g_bnd, (-1,))
        vals = np.empty(nnz.value); rhs = np.empty(na)
        self._check(lib().hps_gpu_multi_assemble_reduced(self._h, _ptr(T), _ptr(w), _ptr(g_bnd), _ptr(vals),
                                                         _ptr(rhs)))
        return rp, ci[:nnz.value], vals, rhs


class _PinnedOwner:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().hps_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float64):
    """numpy array in pinned host memory (hps_host_alloc), freed when the last view of it
    is garbage-collected."""
    count = int(np.prod(shape))
    n = max(count * np.dtype(dtype).itemsize, 1)
    ptr = lib().hps_host_alloc(n)
    if not ptr:
        raise CudaError("hps_host_alloc failed")
    buf = (C.c_char * n).from_address(ptr)
    buf._owner = _PinnedOwner(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)


class PinnedArray:
    """Page-locked host array from hps_host_alloc (for overlapped H2D/D2H)."""

    def __init__(self, shape, dtype=np.float64):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self._p = lib().hps_host_alloc(max(n, 1))
        if not self._p:
            raise CudaError("hps_host_alloc failed")
        buf = (C.c_char * max(n, 1)).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if self._p:
            self.array = None
            lib().hps_host_free(C.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def write_reduced_coo(path, row_ptr, col_idx, values, rhs=None):
    """Coordinate-triplet dump of the reduced system for external solver debugging
    (SPEC.md assembly module, "External Interfaces: optional dump of the reduced system in
    coordinate-triplet text format").  Writes Matrix Market `coordinate real general`
    (1-based i j value, %.17g so every double round-trips bit for bit) to `path`, and the
    rhs, when given, as a Matrix Market `array` to `path + ".rhs"`.  Host-side plumbing
    over the CSR that assemble_reduced returns; nothing here touches the GPU."""
    row_ptr = np.asarray(row_ptr, np.int64)
    n = row_ptr.size - 1
    rows = np.repeat(np.arange(1, n + 1, dtype=np.int64), np.diff(row_ptr))
    cols = np.asarray(col_idx, np.int64) + 1
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{n} {n} {rows.size}\n")
        np.savetxt(fh, np.column_stack([rows, cols, np.asarray(values, np.float64)]),
                   fmt=["%d", "%d", "%.17g"])
    if rhs is not None:
        with open(str(path) + ".rhs", "w") as fh:
            fh.write("%%MatrixMarket matrix array real general\n")
            fh.write(f"{n} 1\n")
            np.savetxt(fh, np.asarray(rhs, np.float64), fmt="%.17g")
