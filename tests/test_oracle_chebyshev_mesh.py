"""Oracle pinned against the SPEC.md known-answer examples: chebyshev + mesh modules.

SPEC.md:44-104 (chebyshev), :106-163 (mesh), acceptance 4 and 7 (:586, :589).
"""
import math

import numpy as np
import pytest

from oracle import pyoracle as O


def test_cheb_nodes_examples():
    # SPEC.md:50-52
    assert np.allclose(O.cheb_nodes(3, allow_small=True), [-1.0, 0.0, 1.0], atol=0, rtol=0)
    assert np.allclose(O.cheb_nodes(4), [-1.0, -0.5, 0.5, 1.0], atol=1e-15)
    s = math.sqrt(2.0) / 2.0
    assert np.allclose(O.cheb_nodes(5), [-1.0, -s, 0.0, s, 1.0], atol=1e-15)


@pytest.mark.parametrize("p", [4, 5, 8, 12, 16, 22, 33, 42])
def test_cheb_nodes_invariants(p):
    x = O.cheb_nodes(p)
    assert x[0] == -1.0 and x[-1] == 1.0
    assert np.all(np.diff(x) > 0)
    assert np.array_equal(x, -x[::-1])                          # exact symmetry
    ref = np.cos(np.pi * np.arange(p - 1, -1, -1) / (p - 1))   # SPEC.md:33 formula
    assert np.max(np.abs(x - ref)) < 1e-15


def test_cheb_nodes_rejects_small_p():
    with pytest.raises(O.OracleError) as ei:
        O.cheb_nodes(3)
    assert ei.value.code == 2


def test_diff_matrix_examples():
    D3 = O.cheb_diff(3, allow_small=True)
    assert np.allclose(D3 @ np.ones(3), 0.0, atol=1e-15)
    x3 = O.cheb_nodes(3, allow_small=True)
    assert np.allclose(D3 @ x3 ** 2, [-2.0, 0.0, 2.0], atol=1e-14)
    x8 = O.cheb_nodes(8); D8 = O.cheb_diff(8)
    assert np.max(np.abs(D8 @ x8 ** 7 - 7 * x8 ** 6)) <= 1e-10


@pytest.mark.parametrize("p", list(range(4, 43)))
def test_diff_matrix_exactness(p):
    """Acceptance 4 and the invariants at :39-40, :83-84."""
    x = O.cheb_nodes(p); D = O.cheb_diff(p)
    assert np.max(np.abs(D.sum(axis=1))) <= 1e-13 * p * p
    for i in range(p):                                              # negative-sum diagonal, j ascending
        acc = 0.0
        for j in range(p):
            if j != i:
                acc += D[i, j]
        assert D[i, i] == -acc
    for k in range(0, p):
        d = k * x ** (k - 1) if k > 0 else np.zeros(p)
        err = np.max(np.abs(D @ x ** k - d))
        assert err <= 1e-10 * max(1.0, np.max(np.abs(d))), (p, k, err)


def test_scale_to_interval():
    D = O.cheb_diff(6)
    assert np.array_equal(O.scale_to_interval(D, 2.0), D)
    assert np.array_equal(O.scale_to_interval(D, 1.0), 2.0 * D)
    x = O.cheb_nodes(6)
    xm = 0.25 * (x + 1.0)                                          # nodes mapped to [0, 0.5]
    assert np.allclose(O.scale_to_interval(D, 0.5) @ xm, 1.0, atol=1e-13)
    for bad in (0.0, -1.0):
        with pytest.raises(O.OracleError) as ei:
            O.scale_to_interval(D, bad)
        assert ei.value.code == 2


def test_mesh_counts():
    assert O.mesh_info(2, 2, 4)[0] == 49
    assert O.mesh_info(4, 2, 8)[0] == 435
    assert O.mesh_info(2, 2, 8)[2] == 24
    assert O.mesh_info(2, 2, 4)[2] == 8
    assert O.mesh_info(3, 3, 6)[0] == 256


def _classes(nx, ny, p):
    from hps_harness import classify
    return np.bincount(classify(nx, ny, p), minlength=4)


def test_node_classification():
    c = _classes(2, 2, 4)
    assert c[0] == 16 and c[2] == 24 and c[1] == 8 and c[3] == 1
    c = _classes(3, 3, 6)
    assert c.sum() == 256


@pytest.mark.parametrize("nx,ny,p", [(2, 2, 4), (3, 2, 6), (4, 4, 8), (5, 3, 12), (16, 16, 12), (7, 9, 22)])
def test_mesh_invariants(nx, ny, p):
    N, ne, na = O.mesh_info(nx, ny, p)
    assert N == (nx * (p - 1) + 1) * (ny * (p - 1) + 1)
    assert na == (nx - 1) * ny * (p - 2) + (ny - 1) * nx * (p - 2)  # corner policy
    assert na <= 2.5 * N / p                                       # acceptance 7
    # active_index is a bijection onto 0..n_active-1
    act = O.active_of_global(nx, ny, p, np.arange(N))
    v = np.sort(act[act >= 0])
    assert np.array_equal(v, np.arange(na))
    # element_node_index: shared edge nodes in exactly 2 lists, corners up to 4
    cnt = np.zeros(N, np.int64)
    for e in range(nx * ny):
        cnt[O.element_node_index(nx, ny, p, e)] += 1
    from hps_harness import classify
    cls = classify(nx, ny, p)
    assert np.all(cnt[cls == 1] == 2)
    assert np.all(cnt[cls == 0] == 1)
    assert np.all(cnt[cls == 3] == 4)


def test_active_ordering_is_edge_major_by_x_then_y():
    nx, ny, p = 3, 2, 6
    from paper_2211_14969_b200 import problems as P
    a = 1.0 / nx
    N, _, na = O.mesh_info(nx, ny, p)
    act = O.active_of_global(nx, ny, p, np.arange(N))
    xs = P.global_axis(nx, p, a); ys = P.global_axis(ny, p, a)
    Nx = nx * (p - 1) + 1
    g = np.nonzero(act >= 0)[0]
    order = g[np.argsort(act[g])]
    q = p - 2
    mids = []
    for ed in range(na // q):
        nodes = order[ed * q:(ed + 1) * q]
        X = xs[nodes % Nx]; Y = ys[nodes // Nx]
        mids.append((X.mean(), Y.mean()))
        # ascending along the edge
        assert np.all(np.diff(X) > 0) or np.all(np.diff(Y) > 0)
    mids = np.array(mids)
    key = np.lexsort((mids[:, 1], mids[:, 0]))
    assert np.array_equal(key, np.arange(len(mids)))


def test_oracle_uses_reference_headers_when_present():
    """The oracle's batching and error classes are the reference's own headers
    (proj/include/hps/parallel.hpp, errors.hpp) whenever they exist at build time."""
    import os
    info = O.build_info()
    if os.path.exists("/root/reference/proj/include/hps/parallel.hpp"):
        assert info.startswith("reference headers"), info
    else:
        assert "restated" in info or info.startswith("reference headers"), info
