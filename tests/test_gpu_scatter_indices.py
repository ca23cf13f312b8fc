"""hps_gpu_scatter_indices: the per-leaf COO view of assemble_reduced's CSR
 must be bit-exact with the CPU oracle's mesh maps and reduced pattern,
and accumulating T through it must reproduce the oracle's reduced values bit for bit."""
import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


def G():
    from paper_2211_14969_b200 import leaf_gpu
    return leaf_gpu


@pytest.mark.parametrize("nx,ny,p", [(1, 1, 6), (2, 2, 8), (3, 2, 6), (4, 3, 12), (5, 5, 22), (2, 3, 42)])
def test_scatter_indices_match_oracle(nx, ny, p):
    nb = 4 * (p - 1)
    n = nx * ny
    rng = np.random.default_rng(nx * 100 + ny * 10 + p)
    T = rng.uniform(-1, 1, (n, nb, nb)); w = rng.uniform(-1, 1, (n, nb))
    N = (nx * (p - 1) + 1) + (ny * (p - 1) + 1)
    g = rng.uniform(-1, 1, 2 * N)
    with G().LeafStage(p, nx, ny, 1.0) as st:
        slot, row = st.scatter_indices()
        s_part, r_part = st.scatter_indices(1, n) if n > 1 else (slot[1:], row[1:])
        rp, ci = st.reduced_pattern()
    assert slot.dtype == np.int64 and row.dtype == np.int64
    # leaf sub-ranges give the same rows of the map
    assert np.array_equal(s_part, slot[1:]) and np.array_equal(r_part, row[1:])

    # rows: active index of each local boundary node (independent derivation via oracle maps)
    _, bd = O.leaf_index(p)
    for e in range(n):
        gid = O.element_node_index(nx, ny, p, e)[bd]
        assert np.array_equal(row[e], O.active_of_global(nx, ny, p, gid)), e

    # slots: inside the row's CSR range, pointing at the column's active index
    orp, oci = O.reduced_pattern(nx, ny, p)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    both = (row[:, :, None] >= 0) & (row[:, None, :] >= 0)
    assert np.array_equal(slot >= 0, both)
    rr = np.broadcast_to(row[:, :, None], slot.shape)[both]
    cc = np.broadcast_to(row[:, None, :], slot.shape)[both]
    sv = slot[both]
    assert np.all(sv >= orp[rr]) and np.all(sv < orp[rr + 1])
    assert np.array_equal(oci[sv], cc)
    # every CSR entry receives 1 or 2 contributions (edge shared by <= 2 leaves)
    cnt = np.bincount(sv, minlength=oci.size)
    assert oci.size == 0 or (cnt.min() >= 1 and cnt.max() <= 2)

    # accumulating T in ascending leaf order reproduces the oracle's values bit for bit
    vals = np.zeros(oci.size)
    np.add.at(vals, sv, T[both])
    _, _, ovals, _ = O.assemble_reduced(nx, ny, p, T, w, g)
    assert np.array_equal(vals, ovals)


def test_scatter_indices_range_errors():
    with G().LeafStage(8, 2, 2, 1.0) as st:
        with pytest.raises(G().ParameterError):
            st.scatter_indices(0, 5)
        s, r = st.scatter_indices(2, 2)
        assert s.shape == (0, 28, 28) and r.shape == (0, 28)
