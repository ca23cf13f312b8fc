"""GPU SlabLU against the host sparse direct solve of the same
reduced system (SPEC.md:455 equivalence with the oracle: inf-norm relative <= 1e-9), plus the
SPEC examples: round trip, rhs = 0 -> 0 exactly, linearity, widths, remainder slab, error on
widths leaving fewer than 2 slabs."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2211_14969_b200 import problems as P

pytestmark = pytest.mark.gpu


def G():
    from paper_2211_14969_b200 import leaf_gpu
    return leaf_gpu


def S():
    from paper_2211_14969_b200 import slab_gpu
    return slab_gpu


def reduced(p, nx, ny, kappa, seed=0):
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y) if kappa > 0 else np.ones_like(X)
    f = np.random.default_rng(seed).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.sin(3 * x) + y)
    with G().LeafStage(p, nx, ny, kappa) as st:
        T, w, s = st.condense(b, f)
        rp, ci, va, rh = st.assemble_reduced(T, w, gb)
        brp, bci, bva, brh = st.assemble_reduced_bsr(T, w, gb)
    A = sp.csr_matrix((va, ci, rp), shape=(rp.size - 1, rp.size - 1))
    return A, rh, (brp, bci, bva)


@pytest.mark.parametrize("p,nx,ny,kappa,width", [(8, 4, 4, 0.0, 1), (8, 4, 4, 0.0, 2), (10, 7, 3, 12.0, 2),
                                                 (12, 8, 5, 2 * np.pi * 2, 1), (16, 8, 8, 2 * np.pi * 4, 0),
                                                 (22, 6, 4, 60.0, 3)])
def test_slablu_matches_sparse_direct(p, nx, ny, kappa, width):
    A, rhs, (brp, bci, bva) = reduced(p, nx, ny, kappa)
    x_ref = spla.spsolve(A.tocsc(), rhs)
    with S().SlabLU(p, nx, ny, brp, bci, bva, slab_width=width) as lu:
        x = lu.solve(rhs)
        info = lu.info
        w = info["slab_width"]
        assert info["n_slabs"] == nx // w and nx // w >= 2
        assert info["n_interface"] == ny * (p - 2)
        err = np.max(np.abs(x - x_ref)) / np.max(np.abs(x_ref))
        assert err <= 1e-9, err
        # round trip: rhs = A v -> v
        v = np.random.default_rng(1).uniform(-1, 1, rhs.size)
        assert np.max(np.abs(lu.solve(A @ v) - v)) / np.max(np.abs(v)) <= 1e-9
        # rhs = 0 -> 0 exactly; linearity
        assert not lu.solve(np.zeros_like(rhs)).any()
        r2 = np.random.default_rng(2).uniform(-1, 1, rhs.size)
        assert np.max(np.abs(lu.solve(rhs) + lu.solve(r2) - lu.solve(rhs + r2))) <= 1e-12 * np.max(np.abs(x))


def test_slablu_partition_rules():
    A, rhs, (brp, bci, bva) = reduced(8, 7, 3, 0.0)
    with S().SlabLU(8, 7, 3, brp, bci, bva, slab_width=2) as lu:   # {2, 2, 3}
        assert lu.info["n_slabs"] == 3
        assert lu.info["max_interior"] == (3 * 2 + 2 * 3) * 6   # 3 columns: 6 horizontal + 2x3 vertical edges
    with pytest.raises(G().ParameterError):
        S().SlabLU(8, 7, 3, brp, bci, bva, slab_width=4)   # 1 slab < 2


def test_slablu_singular_interface_block():
    """A reduced system whose interface block is singular after elimination raises
    SingularBlockError with that interface's index (errors.hpp:30-38)."""
    p, nx, ny = 8, 4, 3
    A, rhs, (brp, bci, bva) = reduced(p, nx, ny, 0.0)
    q = p - 2
    bva = bva.copy()
    # interface 0 (width 1): the vertical edges at x-column 1 = edge ids [ny-1, 2ny-1)
    for ed in range(ny - 1, 2 * ny - 1):
        bva[brp[ed]:brp[ed + 1]] = 0.0
    with pytest.raises(S().SingularBlockError) as ei:
        S().SlabLU(p, nx, ny, brp, bci, bva, slab_width=1)
    assert ei.value.block_index == 0
