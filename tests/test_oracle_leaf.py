"""Oracle pinned against the SPEC.md known-answer examples: leaf + assembly modules.

SPEC.md:250-324 (leaf), :326-389 (assembly), acceptance 1, 4, 9, 10 (:583-592).
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2211_14969_b200 import problems as P
import hps_harness as H


def _leaf_xy(p, a, x0=0.0, y0=0.0):
    xh = P.cheb_nodes(p)
    off = (xh + 1.0) * (a / 2.0)
    X = np.broadcast_to(x0 + off[None, :], (p, p)).ravel()
    Y = np.broadcast_to(y0 + off[:, None], (p, p)).ravel()
    return X, Y


def test_leaf_operator_examples():
    p, a = 8, 0.5
    it, bd = O.leaf_index(p)
    X, Y = _leaf_xy(p, a)
    A, Dn = O.build_leaf(p, a, 0.0, np.zeros(p * p))
    assert np.max(np.abs((A @ X)[it])) <= 1e-10
    assert np.max(np.abs((A @ np.ones(p * p))[it])) <= 1e-11 * p ** 3
    A1, _ = O.build_leaf(p, a, 1.0, np.ones(p * p))
    assert np.max(np.abs((A1 @ np.ones(p * p))[it] + 1.0)) <= 1e-11
    # a=0.5, u = sin(2x)cosh(y).  The stated 1e-6 is not reachable at p=6: the
    # degree-5 truncation error of this field on [0, 0.5]^2 is 1.3e-4 for ANY collocation code
    # (measured here).  Checked at p=6 with the truncation
    # bound and at p=8 with the SPEC's 1e-6.
    for p6, tol in ((6, 2e-4), (8, 1e-6)):
        it6, _ = O.leaf_index(p6)
        X6, Y6 = _leaf_xy(p6, 0.5)
        A6, _ = O.build_leaf(p6, 0.5, 0.0, np.zeros(p6 * p6))
        u = np.sin(2 * X6) * np.cosh(Y6)
        want = -(-4 * np.sin(2 * X6) * np.cosh(Y6) + np.sin(2 * X6) * np.cosh(Y6))
        assert np.max(np.abs((A6 @ u)[it6] - want[it6])) <= tol
    # D_normal exact on linear fields
    al, be, ga = 0.3, -1.7, 2.5
    lin = al + be * X + ga * Y
    dn = Dn @ lin
    nb = 4 * (p - 1)
    expect = np.empty(nb)
    for k in range(nb):
        if k < p: expect[k] = -ga                 # S
        elif k < 2 * p - 1: expect[k] = be        # E
        elif k < 3 * p - 2: expect[k] = ga        # N
        else: expect[k] = -be                     # W
    assert np.max(np.abs(dn - expect)) <= 1e-10
    # partition of local indices
    assert np.array_equal(np.sort(np.concatenate([it, bd])), np.arange(p * p))
    # corner positions SW=0, SE=p-1, NE=2p-2, NW=2p-1
    assert list(bd[[0, p - 1, 2 * p - 2, 2 * p - 1]]) == [0, p - 1, p * p - 1, (p - 1) * p]


def _condense_one(p, a, kappa, b, f):
    r = O.batched_condense(p, a, kappa, b[None], f[None], want_S=True)
    return r["T"][0], r["w"][0], r["S"][0]


def _noncorner(p):
    nb = 4 * (p - 1)
    return np.array([k for k in range(nb) if k not in (0, p - 1, 2 * p - 2, 2 * p - 1)])


def test_condense_linear_and_constant_fields():
    p, a = 12, 0.25
    it, bd = O.leaf_index(p)
    X, Y = _leaf_xy(p, a)
    T, w, S = _condense_one(p, a, 0.0, np.zeros(p * p), np.zeros(p * p))
    nc = _noncorner(p)
    flux = T @ X[bd]
    # right edge (E) +1, left edge (W) -1, S/N 0
    for k in nc:
        e = 0 if k < p else 1 if k < 2 * p - 1 else 2 if k < 3 * p - 2 else 3
        want = {0: 0.0, 1: 1.0, 2: 0.0, 3: -1.0}[e]
        assert abs(flux[k] - want) <= 1e-9
    assert np.max(np.abs((T @ np.ones(4 * (p - 1)))[nc])) <= 1e-9
    assert np.max(np.abs(w)) == 0.0


def test_condense_j0_interior_and_leaf_solve():
    """p=16, a=0.25, kappa=2pi, b=1, boundary data u_true."""
    p, a, kappa = 16, 0.25, 2 * math.pi
    it, bd = O.leaf_index(p)
    X, Y = _leaf_xy(p, a)
    ut = P.analytic_j0(kappa)(X, Y)
    b = np.ones(p * p); f = np.zeros(p * p)
    T, w, S = _condense_one(p, a, kappa, b, f)
    rec = S @ ut[bd]
    assert np.max(np.abs(rec - ut[it])) / np.max(np.abs(ut[it])) <= 1e-8
    u = O.batched_leaf_solve(p, a, kappa, b[None], f[None], ut[bd][None])[0]
    assert np.max(np.abs(u - ut)) <= 1e-8


def test_reconstruction_consistency_and_schur():
    """SPEC.md:266 (interior equations hold) and :308 (Schur vs dense block solve, p<=10)."""
    rng = np.random.default_rng(0)
    for p in (6, 8, 10):
        a, kappa = 0.2, 7.0
        b = rng.uniform(0, 1, p * p); f = rng.uniform(-1, 1, p * p)
        it, bd = O.leaf_index(p)
        A, Dn = O.build_leaf(p, a, kappa, b)
        T, w, S = _condense_one(p, a, kappa, b, f)
        v = rng.uniform(-1, 1, 4 * (p - 1))
        u = np.empty(p * p); u[bd] = v; u[it] = S @ v
        res = (A @ u)[it]
        assert np.max(np.abs(res)) <= 1e-9 * np.max(np.abs(A[it])) * np.max(np.abs(u))
        Aii = A[np.ix_(it, it)]; Aib = A[np.ix_(it, bd)]
        Di = Dn[:, it]; Db = Dn[:, bd]
        Tref = Db - Di @ np.linalg.solve(Aii, Aib)
        assert np.linalg.norm(T - Tref) <= 1e-11 * np.linalg.norm(Tref)
        wref = Di @ np.linalg.solve(Aii, f[it])
        assert np.linalg.norm(w - wref) <= 1e-11 * max(1.0, np.linalg.norm(wref))


def test_flux_antisymmetry():
    """outward fluxes of two neighbours cancel on the shared edge (p=16)."""
    p, a = 16, 0.25
    kappa = 2 * math.pi
    nc = np.arange(1, p - 1)
    ut = P.analytic_j0(kappa)
    it, bd = O.leaf_index(p)
    XL, YL = _leaf_xy(p, a, 0.25, 0.25); XR, YR = _leaf_xy(p, a, 0.5, 0.25)
    TL, _, _ = _condense_one(p, a, kappa, np.ones(p * p), np.zeros(p * p))
    fl = TL @ ut(XL, YL)[bd]; fr = TL @ ut(XR, YR)[bd]
    east = p + (nc - 1)            # E positions of non-corner nodes
    west = 3 * p - 2 + (nc - 1)    # W positions
    assert np.max(np.abs(fl[east] + fr[west])) <= 1e-7


def test_batched_shapes_and_determinism():
    """SPEC.md:294-295, acceptance 9: 16 leaves of 28x28; serial == parallel bitwise."""
    nx = ny = 4; p = 8
    _, _, b, f = H.leaf_inputs(nx, ny, p, lambda x, y: 0.5 + 0.5 * np.sin(7 * x) * np.cos(5 * y),
                               lambda x, y: np.cos(3 * x + y))
    r1 = O.batched_condense(p, 0.25, 9.0, b, f, want_S=True, workers=1)
    r8 = O.batched_condense(p, 0.25, 9.0, b, f, want_S=True, workers=8)
    assert r1["T"].shape == (16, 28, 28)
    for k in ("T", "w", "S"):
        assert np.array_equal(r1[k], r8[k])


def test_store_equals_recompute_bitwise():
    """SPEC.md:305, acceptance 10."""
    rng = np.random.default_rng(3)
    p, n = 10, 5
    b = rng.uniform(0, 1, (n, p * p)); f = rng.uniform(-1, 1, (n, p * p))
    r = O.batched_condense(p, 0.1, 20.0, b, f, want_lu=True)
    v = rng.uniform(-1, 1, (n, 4 * (p - 1)))
    u1 = O.batched_leaf_solve(p, 0.1, 20.0, b, f, v)
    u2 = O.batched_leaf_solve(p, 0.1, 20.0, b, f, v, lu=r["lu"], ipiv=r["ipiv"])
    assert np.array_equal(u1, u2)


def test_leaf_solve_constant():
    p = 10
    c = 0.731
    u = O.batched_leaf_solve(p, 0.3, 0.0, np.ones((1, p * p)), np.zeros((1, p * p)),
                             np.full((1, 4 * (p - 1)), c))[0]
    assert np.max(np.abs(u - c)) <= 1e-10


def test_resonance_injection_reports_element():
    p, n = 8, 6
    b = np.ones((n, p * p)); f = np.zeros((n, p * p))
    with pytest.raises(O.OracleError) as ei:
        O.batched_condense(p, 0.25, 3.0, b, f, inject=[4, 2])
    assert ei.value.code == 1 and "element 2" in str(ei.value)
    r = O.batched_condense(p, 0.25, 3.0, b, f, inject=[4, 2], raise_on_resonance=False)
    assert list(np.nonzero(r["status"])[0]) == [2, 4]


# ------------------------------------------------------------------ assembly / end to end

def _g_const(c):
    return lambda x, y: np.full(np.broadcast(x, y).shape, c)


def test_reduced_constant_and_linear():
    nx = ny = 2; p = 8
    _, _, b, f = H.leaf_inputs(nx, ny, p, lambda x, y: 1.0 + 0 * x, lambda x, y: 0 * x)
    gb = P.boundary_samples(nx, ny, p, _g_const(1.0))
    r = O.batched_condense(p, 0.5, 0.0, b, f)
    ua, _ = H.reduced_solve(nx, ny, p, r["T"], r["w"], gb)
    assert ua.size == 24
    assert np.max(np.abs(ua - 1.0)) <= 1e-10
    gb = P.boundary_samples(nx, ny, p, lambda x, y: x + 0 * y)
    ua, _ = H.reduced_solve(nx, ny, p, r["T"], r["w"], gb)
    N, _, _ = O.mesh_info(nx, ny, p)
    act = O.active_of_global(nx, ny, p, np.arange(N))
    GX, GY = H.global_coords(nx, ny, p)
    xs = np.empty(ua.size); xs[act[act >= 0]] = GX[act >= 0]
    assert np.max(np.abs(ua - xs)) <= 1e-9


def test_reduced_pattern_structure():
    nx, ny, p = 3, 4, 6
    rp, ci = O.reduced_pattern(nx, ny, p)
    q = p - 2
    assert np.all(np.diff(rp) <= 7 * q)
    for j in range(rp.size - 1):
        row = ci[rp[j]:rp[j + 1]]
        assert np.all(np.diff(row) > 0)
    # structural symmetry
    import scipy.sparse as sp
    A = sp.csr_matrix((np.ones(ci.size), ci, rp))
    assert (A - A.T).nnz == 0


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("p", [6, 8, 10])
@pytest.mark.parametrize("kappa", [0.0, 2 * math.pi])
def test_oracle_equivalence_dense_global(n, p, kappa):
    """Acceptance 1: HPS pipeline == dense global solve to 1e-9 (inf-norm)."""
    nx = ny = n
    ut = P.analytic_j0(max(kappa, 1.0))
    _, _, b, f = H.leaf_inputs(nx, ny, p, lambda x, y: 1.0 + 0 * x,
                               lambda x, y: np.sin(3 * x) * np.cos(2 * y))
    gb = P.boundary_samples(nx, ny, p, ut)
    u, _ = H.hps_pipeline(nx, ny, p, kappa, b, f, gb)
    A, rhs, cls = H.assemble_global_dense(nx, ny, p, kappa, b, f, gb)
    ud = np.linalg.solve(A, rhs)
    m = cls != 3
    err = np.max(np.abs(u[m] - ud[m])) / np.max(np.abs(ud[m]))
    assert err <= 1e-9, err


def test_true_accuracy_p16():
    """analytic Helmholtz, p=16, 8x8, kappa=2pi*4 -> relerr_true <= 1e-6."""
    nx = ny = 8; p = 16; kappa = 2 * math.pi * 4
    ut = P.analytic_j0(kappa)
    _, _, b, f = H.leaf_inputs(nx, ny, p, lambda x, y: 1.0 + 0 * x, lambda x, y: 0 * x)
    gb = P.boundary_samples(nx, ny, p, ut)
    u, _ = H.hps_pipeline(nx, ny, p, kappa, b, f, gb)
    GX, GY = H.global_coords(nx, ny, p)
    cls = H.classify(nx, ny, p)
    m = cls != 3
    ue = ut(GX, GY)
    rel = np.linalg.norm(u[m] - ue[m]) / np.linalg.norm(ue[m])
    assert rel <= 1e-6, rel


def test_reduced_coo_triplet_dump_roundtrip(tmp_path):
    """SPEC assembly 'External Interfaces': the coordinate-triplet dump of the reduced system
    reads back (scipy Matrix Market reader) as the same matrix and rhs, bit for bit."""
    import scipy.io
    import scipy.sparse as sp
    from paper_2211_14969_b200.leaf_gpu import write_reduced_coo
    nx, ny, p = 3, 2, 6
    rng = np.random.default_rng(5)
    nb = 4 * (p - 1)
    T = rng.standard_normal((nx * ny, nb, nb)); w = rng.standard_normal((nx * ny, nb))
    gb = P.boundary_samples(nx, ny, p, lambda x, y: x - 2 * y)
    rp, ci, v, r = O.assemble_reduced(nx, ny, p, T, w, gb)
    path = tmp_path / "reduced.mtx"
    write_reduced_coo(str(path), rp, ci, v, r)
    A = scipy.io.mmread(str(path)).tocsr()
    A.sort_indices()
    ref = sp.csr_matrix((v, ci, rp), shape=(r.size, r.size))
    assert A.shape == ref.shape and A.nnz == ref.nnz
    assert np.array_equal(A.indptr, ref.indptr) and np.array_equal(A.indices, ref.indices)
    assert np.array_equal(A.data.view(np.int64), ref.data.view(np.int64))
    rr = np.asarray(scipy.io.mmread(str(path) + ".rhs")).ravel()
    assert np.array_equal(rr.view(np.int64), r.view(np.int64))
