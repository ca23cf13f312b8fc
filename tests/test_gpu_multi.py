"""Leaf-range sharding inside the product (hps_gpu_multi_*, parallel.hpp:21-24,
SPEC.md:291): several contexts, one host thread each, driven through the CUDA library.
Only one GPU is available here, so the shards are contexts on the same device -- the
code path (per-shard ctx, thread, disjoint pinned/host slots, per-shard K4 over the edges
inside the shard, host merge of the cut edges) is the one a multi-GPU box runs.
Everything must be bitwise equal to a single context."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2211_14969_b200 import problems as P

pytestmark = pytest.mark.gpu


def G():
    from paper_2211_14969_b200 import leaf_gpu
    return leaf_gpu


@pytest.mark.parametrize("p,nx,ny,kappa,devs", [(14, 5, 4, 30.0, [0, 0]), (8, 7, 3, 12.0, [0, 0, 0]),
                                                (22, 4, 4, 100.0, [0, 0, 0])])
def test_multi_bitwise_equals_single(p, nx, ny, kappa, devs):
    X, Y = P.leaf_coords(nx, ny, p)
    b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    f = np.random.default_rng(p).uniform(-1, 1, X.shape)
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.cos(3 * x) + y)
    v = np.random.default_rng(1).uniform(-1, 1, (nx * ny, 4 * (p - 1)))
    with G().LeafStage(p, nx, ny, kappa) as st:
        T1, w1, s1 = st.condense(b, f)
        u1 = st.leaf_solve(b, f, v)
        rp1, ci1, va1, rh1 = st.assemble_reduced(T1, w1, gb)
    with G().MultiLeafStage(p, nx, ny, kappa, devs) as ms:
        sh = ms.shards()
        assert len(sh) == len(devs) and sh[0][0] == 0 and sh[-1][1] == nx * ny
        sizes = [hi - lo for lo, hi in sh]
        assert max(sizes) - min(sizes) <= 1
        T2, w2, s2 = ms.condense(b, f)
        u2 = ms.leaf_solve(b, f, v)
        rp2, ci2, va2, rh2 = ms.assemble_reduced(T2, w2, gb)
    assert np.array_equal(T1, T2) and np.array_equal(w1, w2) and np.array_equal(s1, s2)
    assert np.array_equal(u1, u2)
    assert np.array_equal(rp1, rp2) and np.array_equal(ci1, ci2)
    assert np.array_equal(va1, va2) and np.array_equal(rh1, rh2)
    cut = G().reduced_cut_edges(p, nx, ny, [lo for lo, _ in sh])
    assert cut.size > 0   # the host merge path really ran


def test_multi_resonance_reports_all_shards():
    p, nx, ny, kappa = 12, 4, 3, 10.0
    X, Y = P.leaf_coords(nx, ny, p)
    b = np.ones_like(X); f = np.zeros_like(X)
    with G().MultiLeafStage(p, nx, ny, kappa, [0, 0]) as ms:
        for sh in range(2):
            ctx = G().lib().hps_gpu_multi_ctx(ms._h, sh)
            el = np.array([2, 9], np.int32)
            G().lib().hps_gpu_set_fault_injection(G().C.c_void_p(ctx), G()._ptr(el), el.size)
        with pytest.raises(G().ResonanceError) as ei:
            ms.condense(b, f)
    assert ei.value.element_id == 2 and ei.value.failing == [2, 9]
