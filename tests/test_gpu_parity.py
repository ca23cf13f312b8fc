"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north star): Schur complements T_flux within relative
Frobenius 1e-10 per leaf, interface indices bit-exact, final PDE solution within
1e-9 relative.  Also: bitwise determinism across chunking / leaf ranges
(parallel.hpp:21-22), store == recompute bitwise,
resonance error reporting (errors.hpp:18-26).
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2211_14969_b200 import problems as P
import hps_harness as H

pytestmark = pytest.mark.gpu

TOL_T = 1e-10      # relative Frobenius per leaf (north star)
TOL_U = 1e-9       # final solution (north star)


def G():
    from paper_2211_14969_b200 import leaf_gpu
    return leaf_gpu


def rel_fro(a, b):
    num = np.linalg.norm((a - b).reshape(a.shape[0], -1), axis=1)
    den = np.linalg.norm(b.reshape(b.shape[0], -1), axis=1)
    return num / np.maximum(den, 1e-300)


def random_leaves(p, n, seed, lo=0.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, (n, p * p)), rng.uniform(-1, 1, (n, p * p))


@pytest.mark.parametrize("p,kappa,n", [(4, 2.0, 5), (5, 3.0, 4), (6, 7.0, 6), (8, 10.0, 9), (12, 20.0, 7),
                                       (13, 15.0, 3), (16, 40.0, 5), (22, 100.0, 6), (27, 80.0, 3),
                                       (32, 250.0, 3), (37, 300.0, 2), (42, 500.0, 3)])
def test_condense_parity_random(p, kappa, n):
    b, f = random_leaves(p, n, seed=p)
    a = 1.0 / max(n, 2)
    ref = O.batched_condense(p, a, kappa, b, f)
    with G().LeafStage(p, n, 1, kappa, a=a) as st:
        T, w, s = st.condense(b, f)
    assert not s.any()
    eT = rel_fro(T, ref["T"])
    ew = rel_fro(w, ref["w"])
    assert eT.max() <= TOL_T, eT
    assert ew.max() <= TOL_T, ew


def test_c1_fixtures_parity_and_solution():
    """C1 (p=12, 16x16, Poisson, b=1) with the SURVEY §8d fixtures: f = 2pi^2 sin(pi x) sin(pi y)
    (exact u = sin sin, g = 0) and f ~ U(-1,1) seed 0."""
    cfg = P.config("C1")
    p, nx, ny = cfg["p"], cfg["nx"], cfg["ny"]
    X, Y = P.leaf_coords(nx, ny, p)
    b = np.ones_like(X)
    f1 = 2 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y)
    f2 = np.random.default_rng(0).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: 0 * x)
    with G().LeafStage(p, nx, ny, 0.0) as st:
        for f in (f1, f2):
            ref = O.batched_condense(p, cfg["a"], 0.0, b, f)
            T, w, s = st.condense(b, f)
            assert rel_fro(T, ref["T"]).max() <= TOL_T
            assert rel_fro(w, ref["w"]).max() <= TOL_T
        # end to end with the GPU leaf stage vs the oracle pipeline, and vs the exact solution
        gpu = lambda bb, ff: st.condense(bb, ff)[:2]
        u_g, _ = H.hps_pipeline(nx, ny, p, 0.0, b, f1, gb, condense=gpu,
                                leaf_solve=lambda bb, ff, vv: st.leaf_solve(bb, ff, vv),
                                assemble=lambda T, w, g: st.assemble_reduced(T, w, g))
    u_o, _ = H.hps_pipeline(nx, ny, p, 0.0, b, f1, gb)
    cls = H.classify(nx, ny, p)
    m = cls != 3
    assert np.max(np.abs(u_g[m] - u_o[m])) / np.max(np.abs(u_o[m])) <= TOL_U
    GX, GY = H.global_coords(nx, ny, p)
    exact = np.sin(math.pi * GX) * np.sin(math.pi * GY)
    assert np.max(np.abs(u_g[m] - exact[m])) <= 1e-8


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 6), (2, 2, 4), (2, 2, 8), (3, 4, 6), (5, 3, 12), (16, 16, 12),
                                     (7, 9, 22), (12, 10, 42)])
def test_reduced_pattern_bit_exact(nx, ny, p):
    with G().LeafStage(p, nx, ny, 1.0) as st:
        rp, ci = st.reduced_pattern()
    if nx * ny == 1:
        assert rp.size == 1 and ci.size == 0
        return
    rpo, cio = O.reduced_pattern(nx, ny, p)
    assert rp.dtype == np.int64 and ci.dtype == np.int32
    assert np.array_equal(rp, rpo)
    assert np.array_equal(ci, cio)


@pytest.mark.parametrize("nx,ny,p", [(2, 2, 8), (3, 5, 10), (6, 4, 12)])
def test_reduced_values_bit_exact_given_T(nx, ny, p):
    """K4 scatter reproduces the oracle's assemble_reduced bit for bit on the same T, w, g."""
    rng = np.random.default_rng(11)
    nb = 4 * (p - 1)
    T = rng.standard_normal((nx * ny, nb, nb)); w = rng.standard_normal((nx * ny, nb))
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.cos(3 * x) + y * y)
    rpo, cio, vo, ro = O.assemble_reduced(nx, ny, p, T, w, gb)
    with G().LeafStage(p, nx, ny, 1.0) as st:
        rp, ci, v, r = st.assemble_reduced(T, w, gb)
    assert np.array_equal(rp, rpo) and np.array_equal(ci, cio)
    assert np.array_equal(v.view(np.int64), vo.view(np.int64))
    assert np.array_equal(r.view(np.int64), ro.view(np.int64))


def oracle_bsr(nx, ny, p, rp, ci, vals):
    """BSR view of the oracle's CSR (SPEC.md:331 ReducedSystem.blocks): block row = interface
    edge (q = p-2 rows), block columns = the distinct column edges of its rows, q x q blocks."""
    q = p - 2
    nbr = (rp.size - 1) // q
    brp = [0]; bci = []; blocks = []
    for br in range(nbr):
        lo, hi = rp[br * q], rp[br * q + q]
        ne = (rp[br * q + 1] - lo) // q
        cols = ci[lo:hi].reshape(q, ne, q)
        v = vals[lo:hi].reshape(q, ne, q)
        assert (cols == cols[0]).all()                     # every row of the edge shares columns
        assert (cols[0] // q == cols[0, :, :1] // q).all() and (cols[0] % q == np.arange(q)).all()
        bci += list(cols[0, :, 0] // q)
        blocks.append(v.transpose(1, 0, 2))
        brp.append(brp[-1] + ne)
    return (np.array(brp, np.int64), np.array(bci, np.int32),
            np.concatenate(blocks) if blocks else np.zeros((0, q, q)))


@pytest.mark.parametrize("nx,ny,p", [(2, 2, 4), (2, 2, 8), (3, 5, 10), (6, 4, 12), (5, 3, 22), (4, 4, 42)])
def test_reduced_bsr_view_bit_exact(nx, ny, p):
    """BSR view: pattern equal to the oracle CSR regrouped by edge blocks, block
    entries bit-identical to the oracle's CSR values, rhs identical, and the BSR matrix equals
    the CSR matrix."""
    import scipy.sparse as sp
    rng = np.random.default_rng(12)
    nb = 4 * (p - 1)
    T = rng.standard_normal((nx * ny, nb, nb)); w = rng.standard_normal((nx * ny, nb))
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.sin(2 * x) - y)
    rpo, cio, vo, ro = O.assemble_reduced(nx, ny, p, T, w, gb)
    ebrp, ebci, eblk = oracle_bsr(nx, ny, p, rpo, cio, vo)
    with G().LeafStage(p, nx, ny, 1.0) as st:
        q, brp, bci = st.reduced_bsr_pattern()
        brp2, bci2, blk, r = st.assemble_reduced_bsr(T, w, gb)
    assert q == p - 2
    assert brp.dtype == np.int64 and bci.dtype == np.int32
    assert np.array_equal(brp, ebrp) and np.array_equal(bci, ebci)
    assert np.array_equal(brp2, brp) and np.array_equal(bci2, bci)
    assert np.array_equal(blk.view(np.int64), eblk.view(np.int64))
    assert np.array_equal(r.view(np.int64), ro.view(np.int64))
    A_bsr = sp.bsr_matrix((blk, bci, brp), shape=(ro.size, ro.size)).tocsr()
    A_csr = sp.csr_matrix((vo, cio, rpo), shape=(ro.size, ro.size))
    assert (A_bsr != A_csr).nnz == 0


@pytest.mark.parametrize("p,kappa", [(8, 5.0), (12, 20.0), (22, 100.0), (27, 60.0)])
def test_leaf_solve_parity_and_store_equals_recompute(p, kappa):
    n = 5
    b, f = random_leaves(p, n, seed=100 + p)
    v = np.random.default_rng(7).uniform(-1, 1, (n, 4 * (p - 1)))
    a = 0.2
    uo = O.batched_leaf_solve(p, a, kappa, b, f, v)
    with G().LeafStage(p, n, 1, kappa, a=a) as st:
        ur = st.leaf_solve(b, f, v)
    assert rel_fro(ur, uo).max() <= TOL_T
    with G().LeafStage(p, n, 1, kappa, a=a, storage=G().STORAGE_STORE) as st:
        st.condense(b, f)
        us = st.leaf_solve(b, f, v)
        us2 = st.leaf_solve(b, f, v)            # repeated solves on kept factors
    assert np.array_equal(ur.view(np.int64), us.view(np.int64))
    assert np.array_equal(us.view(np.int64), us2.view(np.int64))


def test_bitwise_independent_of_chunking_and_range():
    """Results do not depend on chunk size, leaf range or batch position."""
    p, nx, ny, kappa = 22, 6, 5, 100.0
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X, Y); f = np.sin(X) * np.cos(Y)
    with G().LeafStage(p, nx, ny, kappa) as st:
        T1, w1, _ = st.condense(b, f)
    with G().LeafStage(p, nx, ny, kappa, workspace_bytes=7 * 3_000_000) as st:   # tiny chunks
        assert st.info()["chunk_leaves"] < nx * ny
        T2, w2, _ = st.condense(b, f)
        T3, w3, _ = st.condense(b[11:23], f[11:23], e0=11)
    assert np.array_equal(T1.view(np.int64), T2.view(np.int64))
    assert np.array_equal(w1.view(np.int64), w2.view(np.int64))
    assert np.array_equal(T1[11:23].view(np.int64), T3.view(np.int64))


def test_resonance_error_reports_smallest_element():
    p, nx, ny = 10, 4, 3
    b, f = random_leaves(p, nx * ny, seed=5)
    with G().LeafStage(p, nx, ny, 3.0) as st:
        st.set_fault_injection([9, 4, 7])
        with pytest.raises(G().ResonanceError) as ei:
            st.condense(b, f)
        assert ei.value.element_id == 4
        assert ei.value.failing == [4, 7, 9]
        assert "element 4" in str(ei.value) and "4,7,9" in str(ei.value)
        T, w, s = st.condense(b, f, raise_on_resonance=False)
        assert list(np.nonzero(s)[0]) == [4, 7, 9]
        # the same injection in the oracle agrees
        r = O.batched_condense(p, 1.0 / nx, 3.0, b, f, inject=[9, 4, 7], raise_on_resonance=False)
        assert list(np.nonzero(r["status"])[0]) == [4, 7, 9]
        ok = s == 0
        assert rel_fro(T[ok], r["T"][ok]).max() <= TOL_T
        st.set_fault_injection([])
        st.condense(b, f)
        with pytest.raises(G().ResonanceError):
            st.set_fault_injection([2])
            st.leaf_solve(b, f, np.zeros((nx * ny, 4 * (p - 1))))


@pytest.mark.parametrize("p,kappa", [(24, 60.0), (25, 60.0), (26, 70.0), (44, 300.0), (45, 300.0)])
def test_condense_parity_kernel_boundaries(p, kappa):
    """Leaf sizes at the kernel boundaries: p = 24/25 are the largest leaves of the 4-warp
    lock-step build (R <= 640), p = 26 the smallest of the 8-warp build, p = 44/45 the largest
    the 8-warp build accepts (R = 2025 <= 2048 rows, 8 strip rows per thread).  Crystal-like
    variable b, random f, three leaves against the oracle."""
    n = 3
    b, f = random_leaves(p, n, seed=100 + p, lo=0.2, hi=0.7)
    a = 1.0 / n
    ref = O.batched_condense(p, a, kappa, b, f)
    with G().LeafStage(p, n, 1, kappa, a=a) as st:
        T, w, s = st.condense(b, f)
    assert not s.any()
    assert rel_fro(T, ref["T"]).max() <= TOL_T
    assert rel_fro(w, ref["w"]).max() <= TOL_T


def test_parameter_errors():
    with pytest.raises(G().ParameterError):
        G().LeafStage(46, 2, 2, 1.0)     # beyond the largest leaf the blocked kernel holds
    with pytest.raises(G().ParameterError):
        G().LeafStage(3, 2, 2, 1.0)
    with pytest.raises(G().ParameterError):
        G().LeafStage(8, 2, 2, 1.0, a=0.0)
    with pytest.raises(G().ParameterError):
        G().LeafStage(8, 2, 2, -1.0)
    with G().LeafStage(8, 2, 2, 1.0) as st:
        b, f = random_leaves(8, 5, 0)
        with pytest.raises(G().ParameterError):
            st.condense(b, f)        # 5 leaves on a 4-leaf mesh


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("p", [6, 10])
@pytest.mark.parametrize("kappa", [0.0, 2 * math.pi])
def test_pipeline_matches_dense_global_solve(n, p, kappa):
    """Acceptance 1 with the GPU leaf stage."""
    nx = ny = n
    ut = P.analytic_j0(max(kappa, 1.0))
    _, _, b, f = H.leaf_inputs(nx, ny, p, lambda x, y: 1.0 + 0 * x, lambda x, y: np.sin(3 * x) * np.cos(2 * y))
    gb = P.boundary_samples(nx, ny, p, ut)
    with G().LeafStage(p, nx, ny, kappa) as st:
        u, _ = H.hps_pipeline(nx, ny, p, kappa, b, f, gb, condense=lambda bb, ff: st.condense(bb, ff)[:2],
                              leaf_solve=lambda bb, ff, vv: st.leaf_solve(bb, ff, vv),
                              assemble=lambda T, w, g: st.assemble_reduced(T, w, g))
    A, rhs, cls = H.assemble_global_dense(nx, ny, p, kappa, b, f, gb)
    ud = np.linalg.solve(A, rhs)
    m = cls != 3
    assert np.max(np.abs(u[m] - ud[m])) / np.max(np.abs(ud[m])) <= TOL_U


def test_c2_full_scale():
    """C2 (p=22, 48x48, kappa=100, crystal b) at full size: no resonance flags, a seeded
    subset of leaves matches the oracle, two runs are bitwise identical, and the constant
    field is annihilated on non-corner rows where b is irrelevant (kappa-free check below)."""
    cfg = P.config("C2")
    p, nx, ny = cfg["p"], cfg["nx"], cfg["ny"]
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X, Y)
    f = np.random.default_rng(2).uniform(-1, 1, X.shape)
    with G().LeafStage(p, nx, ny, cfg["kappa"]) as st:
        T, w, s = st.condense(b, f)
        T2, w2, _ = st.condense(b, f)
    assert not s.any()
    assert np.array_equal(T.view(np.int64), T2.view(np.int64))
    idx = np.random.default_rng(3).choice(nx * ny, 24, replace=False)
    ref = O.batched_condense(p, cfg["a"], cfg["kappa"], b[idx], f[idx])
    assert rel_fro(T[idx], ref["T"]).max() <= TOL_T
    assert rel_fro(w[idx], ref["w"]).max() <= TOL_T


def test_c4_subset_and_laplace_property():
    """C4 shapes (p=42, kappa=500, crystal b): a leaf subset vs the oracle; at kappa=0 the
    DtN map annihilates constants on non-corner rows for every leaf of a 16x16 mesh."""
    cfg = P.config("C4")
    p = cfg["p"]
    el = np.array([0, 97, 4801, 9603])
    X, Y = P.leaf_coords(cfg["nx"], cfg["ny"], p, elements=el)
    b = P.crystal_field(X, Y); f = np.random.default_rng(4).uniform(-1, 1, X.shape)
    ref = O.batched_condense(p, cfg["a"], cfg["kappa"], b, f)
    with G().LeafStage(p, cfg["nx"], cfg["ny"], cfg["kappa"]) as st:
        for i, e in enumerate(el):
            T, w, s = st.condense(b[i:i + 1], f[i:i + 1], e0=int(e))
            assert rel_fro(T, ref["T"][i:i + 1]).max() <= TOL_T
            assert rel_fro(w, ref["w"][i:i + 1]).max() <= TOL_T
    n = 16
    Xl, Yl = P.leaf_coords(n, n, p)
    with G().LeafStage(p, n, n, 0.0) as st:
        T, w, s = st.condense(P.crystal_field(Xl, Yl), np.zeros_like(Xl))
    nc = [k for k in range(4 * (p - 1)) if k not in (0, p - 1, 2 * p - 2, 2 * p - 1)]
    flux = T @ np.ones(4 * (p - 1))
    assert np.max(np.abs(flux[:, nc])) <= 1e-9 * np.max(np.abs(T))


@pytest.mark.parametrize("p,kappa,n", [(6, 5.0, 3), (12, 20.0, 4), (13, 9.0, 3), (22, 100.0, 3), (42, 500.0, 2)])
def test_s_solve_parity(p, kappa, n):
    """K3: S_solve = -A_ii^{-1} A_ib vs the oracle (dgetrs), relFro <= 1e-10,
    and T = D_b + D_i S_solve holds for the GPU's own S."""
    b, f = random_leaves(p, n, seed=200 + p)
    a = 1.0 / n
    ref = O.batched_condense(p, a, kappa, b, f, want_S=True)
    with G().LeafStage(p, n, 1, kappa, a=a) as st:
        T, w, s, S = st.condense(b, f, want_S=True)
    assert rel_fro(S, ref["S"]).max() <= TOL_T
    it, bd = O.leaf_index(p)
    for e in range(n):
        _, Dn = O.build_leaf(p, a, kappa, b[e])
        Tchk = Dn[:, bd] + Dn[:, it] @ S[e]
        assert np.linalg.norm(Tchk - T[e]) <= 1e-10 * np.linalg.norm(T[e])


@pytest.mark.parametrize("p", [4, 5, 6, 7, 8, 9, 10, 11, 12])
def test_small_kernel_matches_oracle_and_blocked_path(p):
    """K2s (register-resident, fused assembly, p <= 12) against the oracle (1e-10 relFro) and
    against the blocked K1+K2 path (OPT_SMALL_KERNEL off); chunk-independent bitwise; crystal b near
    resonance-free range and f ~ U(-1,1) so w is exercised."""
    nx, ny, kappa = 7, 5, 4.0 * p
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X * 0.4 + 0.3, Y * 0.4 + 0.3)
    f = np.random.default_rng(p).uniform(-1, 1, b.shape)
    ref = O.batched_condense(p, 1.0 / nx, kappa, b, f)
    with G().LeafStage(p, nx, ny, kappa) as st:
        st.set_option(G().OPT_SMALL_KERNEL, 1)
        T1, w1, s1 = st.condense(b, f)
        T3, w3, _ = st.condense(b[5:17], f[5:17], e0=5)
    assert not s1.any()
    assert rel_fro(T1, ref["T"]).max() <= TOL_T
    assert rel_fro(w1, ref["w"]).max() <= TOL_T
    assert np.array_equal(T1[5:17].view(np.int64), T3.view(np.int64))
    assert np.array_equal(w1[5:17].view(np.int64), w3.view(np.int64))
    with G().LeafStage(p, nx, ny, kappa) as st:
        st.set_option(G().OPT_SMALL_KERNEL, 0)   # blocked K1 + K2 path
        T2, w2, _ = st.condense(b, f)
    assert rel_fro(T1, T2).max() <= 1e-12
    assert rel_fro(w1, w2).max() <= 1e-12


@pytest.mark.parametrize("p", [6, 12])
def test_small_kernel_resonance_injection(p):
    nx, ny = 4, 3
    b, f = random_leaves(p, nx * ny, seed=11)
    with G().LeafStage(p, nx, ny, 3.0) as st:
        st.set_option(G().OPT_SMALL_KERNEL, 1)
        st.set_fault_injection([9, 4, 7])
        T, w, s = st.condense(b, f, raise_on_resonance=False)
        assert list(np.nonzero(s)[0]) == [4, 7, 9]
        r = O.batched_condense(p, 1.0 / nx, 3.0, b, f, inject=[9, 4, 7], raise_on_resonance=False)
        ok = s == 0
        assert rel_fro(T[ok], r["T"][ok]).max() <= TOL_T


@pytest.mark.parametrize("p", [16, 22])
def test_lockstep_kernel_bitwise_equals_persistent(p):
    """The lock-step multi-leaf K2 kernel runs the same per-leaf code as the one-leaf-per-CTA
    persistent kernel: T, w bitwise equal (lock-step on vs off), including a partial last
    round (leaf count not a multiple of 4 x #SM) and a single-leaf call (OPT_LOCKSTEP on/off)."""
    nx, ny, kappa = 7, 3, 5.0 * p
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X * 0.4 + 0.3, Y * 0.4 + 0.3)
    f = np.random.default_rng(p).uniform(-1, 1, b.shape)
    out = {}
    for ls in ("0", "1"):
        with G().LeafStage(p, nx, ny, kappa) as st:
            st.set_option(G().OPT_LOCKSTEP, int(ls))
            T, w, s = st.condense(b, f)
            T1, w1, _ = st.condense(b[3:4], f[3:4], e0=3)
        assert not s.any()
        out[ls] = (T, w, T1, w1)
    for x, y in zip(out["0"], out["1"]):
        assert np.array_equal(x.view(np.int64), y.view(np.int64))
    ref = O.batched_condense(p, 1.0 / nx, kappa, b, f)
    assert rel_fro(out["1"][0], ref["T"]).max() <= TOL_T


@pytest.mark.parametrize("cfg_name,n", [("C2", 2297), ("C4", 300)])
def test_device_crystal_sampler(cfg_name, n):
    """K0: device-side crystal b(x) at every leaf node equals the host
    restatement problems.crystal_field to the last ulps (exp/sin may differ by 1 ulp), and
    condensing from device-sampled b matches condensing from host-sampled b."""
    import torch
    cfg = P.config(cfg_name)
    p, nx, ny = cfg["p"], cfg["nx"], cfg["ny"]
    e0 = 7
    X, Y = P.leaf_coords(nx, ny, p, a=cfg["a"], elements=np.arange(e0, e0 + n))
    b_host = P.crystal_field(X, Y)
    with G().LeafStage(p, nx, ny, cfg["kappa"], a=cfg["a"]) as st:
        d_b = torch.empty((n, p * p), dtype=torch.float64, device="cuda")
        st.sample_crystal_device(e0, n, d_b.data_ptr())
        torch.cuda.synchronize()
        b_dev = d_b.cpu().numpy()
        assert np.abs(b_dev - b_host).max() <= 1e-14
        assert b_dev.min() >= 0.0 and b_dev.max() <= 1.0
        m = min(n, 64)
        f = np.zeros((m, p * p))
        T1, w1, _ = st.condense(b_host[:m], f, e0=e0)
        T2, w2, _ = st.condense(b_dev[:m], f, e0=e0)
    assert rel_fro(T2, T1).max() <= 1e-12


@pytest.mark.parametrize("n,p,kappa", [(2, 6, 3.0), (3, 8, 10.0), (4, 10, 2 * math.pi)])
def test_residual_matches_dense_global_system(n, p, kappa):
    """K6: the matrix-free device residual of the global collocation system
    equals the dense assemble_global residual, row class by row class, for an arbitrary
    (non-solution) globally consistent u; and the HPS pipeline solution has relerr_res <= 1e-9."""
    nx = ny = n
    rng = np.random.default_rng(n * 100 + p)
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X * 0.4 + 0.3, Y * 0.4 + 0.3)
    f = rng.uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.cos(3 * x) + y * y)
    N, _, _ = O.mesh_info(nx, ny, p)
    ug = rng.uniform(-1, 1, N)
    ul = np.stack([ug[O.element_node_index(nx, ny, p, e)] for e in range(nx * ny)])
    A, rhs, cls = H.assemble_global_dense(nx, ny, p, kappa, b, f, gb)
    r = A @ ug - rhs
    with G().LeafStage(p, nx, ny, kappa) as st:
        res = st.residual(b, f, ul)
        assert abs(res["r_int2"] - np.sum(r[cls == 0] ** 2)) <= 1e-11 * np.sum(r[cls == 0] ** 2)
        assert abs(res["r_flux2"] - np.sum(r[cls == 1] ** 2)) <= 1e-11 * np.sum(r[cls == 1] ** 2)
        assert abs(res["f_int2"] - np.sum(rhs[cls == 0] ** 2)) <= 1e-12 * np.sum(rhs[cls == 0] ** 2)
        u, parts = H.hps_pipeline(nx, ny, p, kappa, b, f, gb, condense=lambda bb, ff: st.condense(bb, ff)[:2],
                                  leaf_solve=lambda bb, ff, vv: st.leaf_solve(bb, ff, vv),
                                  assemble=lambda T, w, g: st.assemble_reduced(T, w, g))
        res = st.residual(b, f, parts["u_leaf"])
    g2 = np.sum(rhs[cls == 2] ** 2)
    relerr_res = math.sqrt((res["r_int2"] + res["r_flux2"]) / (res["f_int2"] + g2))
    assert relerr_res <= 1e-9, relerr_res


def test_residual_full_pipeline_mid_scale():
    """Eq. 7 relerr_res of the whole pipeline (GPU condense -> GPU scatter -> host SuperLU ->
    GPU leaf solve) on a 16x16 mesh at p=16 with the crystal field and the Gaussian pulse,
    evaluated matrix-free on the device."""
    nx = ny = 16; p = 16; kappa = 40.0
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(X, Y); f = np.random.default_rng(2).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, P.gaussian_pulse)
    with G().LeafStage(p, nx, ny, kappa) as st:
        _, parts = H.hps_pipeline(nx, ny, p, kappa, b, f, gb, condense=lambda bb, ff: st.condense(bb, ff)[:2],
                                  leaf_solve=lambda bb, ff, vv: st.leaf_solve(bb, ff, vv),
                                  assemble=lambda T, w, g: st.assemble_reduced(T, w, g))
        res = st.residual(b, f, parts["u_leaf"])
    cls = H.classify(nx, ny, p)
    Nx = nx * (p - 1) + 1
    gx, gy = H.global_coords(nx, ny, p)
    g2 = float(np.sum(P.gaussian_pulse(gx, gy)[cls == 2] ** 2))
    relerr_res = math.sqrt((res["r_int2"] + res["r_flux2"]) / (res["f_int2"] + g2))
    assert relerr_res <= 1e-9, relerr_res


@pytest.mark.parametrize("p", [16, 22, 32])
def test_resonance_injection_blocked_kernels(p):
    """Fault injection through the lock-step (p=16, 22) and persistent 8-warp (p=32) K2
    kernels: exactly the injected leaves are flagged and the others still match the oracle."""
    nx, ny = 3, 3
    b, f = random_leaves(p, nx * ny, seed=p + 1)
    with G().LeafStage(p, nx, ny, 4.0) as st:
        st.set_fault_injection([5, 1])
        T, w, s = st.condense(b, f, raise_on_resonance=False)
    assert list(np.nonzero(s)[0]) == [1, 5]
    r = O.batched_condense(p, 1.0 / nx, 4.0, b, f)
    ok = s == 0
    assert rel_fro(T[ok], r["T"][ok]).max() <= TOL_T


@pytest.mark.parametrize("p,nx,ny,kappa", [(8, 6, 5, 12.0), (16, 5, 4, 40.0), (22, 6, 6, 100.0)])
def test_condense_assemble_fused_equals_separate(p, nx, ny, kappa):
    """hps_gpu_condense_assemble (T resident in HBM, only the reduced system comes back) is
    bitwise condense + assemble_reduced; with want_T the T/w are the separate call's too."""
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    f = np.random.default_rng(3).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.exp(x) * np.cos(y))
    with G().LeafStage(p, nx, ny, kappa) as st:
        T, w, s = st.condense(b, f)
        rp, ci, va, rh = st.assemble_reduced(T, w, gb)
        rp2, ci2, va2, rh2, s2 = st.condense_assemble(b, f, gb)
        rp3, ci3, va3, rh3, s3, T3, w3 = st.condense_assemble(b, f, gb, want_T=True)
    assert np.array_equal(va, va2) and np.array_equal(rh, rh2) and not s2.any()
    assert np.array_equal(va, va3) and np.array_equal(rh, rh3)
    assert np.array_equal(T, T3) and np.array_equal(w, w3)


@pytest.mark.parametrize("p,nx,ny,kappa", [(8, 4, 3, 9.0), (14, 5, 4, 30.0), (22, 3, 3, 60.0)])
def test_reconstruct_on_device(p, nx, ny, kappa):
    """hps_gpu_reconstruct (K7 + batched leaf_solve): every non-corner node is
    bitwise the GPU leaf_solve of the host-built boundary vectors, element corners on Gamma are
    g, and interior corners follow the corner policy -- restated here in the same
    IEEE operation order, so they agree bit for bit."""
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    f = np.random.default_rng(9).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.cos(2 * x) * (1 + y))
    _, _, na = O.mesh_info(nx, ny, p)
    ua = np.random.default_rng(4).uniform(-1, 1, na)
    with G().LeafStage(p, nx, ny, kappa) as st:
        u = st.reconstruct(ua, gb, b, f)
        v = H.leaf_boundary_values(nx, ny, p, ua, gb)
        ul = st.leaf_solve(b, f, v)
    ref = H.scatter_full(nx, ny, p, ul)
    cls = H.classify(nx, ny, p)
    Nx = nx * (p - 1) + 1
    gx = np.arange(u.size) % Nx; gy = np.arange(u.size) // Nx
    corner = (gx % (p - 1) == 0) & (gy % (p - 1) == 0)
    assert np.array_equal(u[~corner], ref[~corner])
    # corner policy restated (hps_api.cpp / k7_corner_kernel order)
    xh = P.cheb_nodes(p)
    wts = [1.0 / np.prod([xh[j] - xh[k] for k in range(1, p - 1) if k != j]) for j in range(1, p - 1)]
    act = lambda x, y: O.active_of_global(nx, ny, p, np.array([y * Nx + x]))[0]
    for cy in range(ny + 1):
        for cx in range(nx + 1):
            X0, Y0 = cx * (p - 1), cy * (p - 1)
            g = Y0 * Nx + X0
            if cls[g] == 2:
                assert u[g] == ref[g]
                continue
            s = 0.0
            for d in range(4):
                t = 1.0 if d in (0, 2) else -1.0
                num = den = 0.0
                for j in range(1, p - 1):
                    x, y = X0, Y0
                    if d == 0: x = X0 - (p - 1) + j
                    if d == 1: x = X0 + j
                    if d == 2: y = Y0 - (p - 1) + j
                    if d == 3: y = Y0 + j
                    c = wts[j - 1] / (t - xh[j])
                    num = num + c * ua[act(x, y)]
                    den = den + c
                s = s + num / den
            assert u[g] == s / 4.0, (cx, cy)


@pytest.mark.parametrize("p,nx,ny,kappa", [(8, 4, 3, 9.0), (16, 4, 3, 30.0), (22, 3, 3, 60.0), (42, 2, 2, 120.0)])
def test_stored_s_solve_policy(p, nx, ny, kappa):
    """HPS_STORAGE_S_SOLVE: condense keeps
    [S_solve | A_ii^-1 f] per leaf; leaf_solve is one GEMV per leaf (K5s) and agrees with the
    recompute policy to 1e-10; condense's S_solve output is bitwise the recompute-mode K3 one;
    reconstruct_full_solution works from the store."""
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    f = np.random.default_rng(5).uniform(-1, 1, X.shape)
    v = np.random.default_rng(6).uniform(-1, 1, (nx * ny, 4 * (p - 1)))
    gb = P.boundary_samples(nx, ny, p, lambda x, y: x - y)
    _, _, na = O.mesh_info(nx, ny, p)
    ua = np.random.default_rng(7).uniform(-1, 1, na)
    with G().LeafStage(p, nx, ny, kappa) as st:
        T0, w0, _, S0 = st.condense(b, f, want_S=True)
        u0 = st.leaf_solve(b, f, v)
        r0 = st.reconstruct(ua, gb, b, f)
    with G().LeafStage(p, nx, ny, kappa, storage=G().STORAGE_S_SOLVE) as st:
        T1, w1, s1, S1 = st.condense(b, f, want_S=True)
        u1 = st.leaf_solve(np.zeros_like(b), np.zeros_like(f), v)   # b, f are not read
        r1 = st.reconstruct(ua, gb, b, f)
    assert not s1.any()
    assert np.array_equal(T0, T1) and np.array_equal(w0, w1) and np.array_equal(S0, S1)
    assert rel_fro(u1.reshape(1, -1), u0.reshape(1, -1))[0] <= 1e-10
    assert np.linalg.norm(r1 - r0) / np.linalg.norm(r0) <= 1e-10


def test_stored_s_solve_budget_and_range():
    p, nx, ny = 42, 3, 3
    with pytest.raises(G().ParameterError):
        G().LeafStage(p, nx, ny, 10.0, storage=G().STORAGE_S_SOLVE, workspace_bytes=8 << 20)
    b, f = random_leaves(p, 9, seed=3)
    with G().LeafStage(p, nx, ny, 10.0, storage=G().STORAGE_S_SOLVE) as st:
        st.condense(b[:4], f[:4])
        with pytest.raises(G().ParameterError):   # leaves 4.. were not condensed
            st.leaf_solve(b, f, np.zeros((9, 4 * (p - 1))))
