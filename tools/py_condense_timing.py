"""Python-API condense timing at C2 (p=22, 48x48 leaves) for three output-buffer choices:
pageable numpy, pinned allocated per call, pinned reused (G.PinnedArray)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2211_14969_b200 import leaf_gpu as G, problems as P  # noqa: E402

p, nx = 22, 48
X, Y = P.leaf_coords(nx, nx, p)
b = P.crystal_field(X, Y); f = np.zeros_like(b)
n, nb = nx * nx, 4 * (p - 1)
with G.LeafStage(p, nx, nx, 100.0) as st:
    pT, pw = G.PinnedArray((n, nb, nb)), G.PinnedArray((n, nb))
    pb, pf = G.PinnedArray(b.shape), G.PinnedArray(f.shape)
    pb.array[:] = b; pf.array[:] = f
    for name, mk, inp in [("pageable out", lambda: (np.empty((n, nb, nb)), np.empty((n, nb))), (b, f)),
                          ("pinned per call", lambda: (G.pinned_empty((n, nb, nb)), G.pinned_empty((n, nb))), (b, f)),
                          ("pinned reused", lambda: (pT.array, pw.array), (b, f)),
                          ("pinned reused + pinned in", lambda: (pT.array, pw.array), (pb.array, pf.array))]:
        ts = []
        for i in range(4):
            t = time.perf_counter()
            st.condense(*inp, out=mk())
            ts.append(time.perf_counter() - t)
        dt = min(ts[1:])
        print(f"{name:<28} {dt*1e3:7.2f} ms  {n/dt:9.0f} leaves/s")

    v = np.random.default_rng(0).uniform(-1, 1, (n, nb))
    for name in ("leaf_solve pageable u",):
        ts = []
        for i in range(4):
            t = time.perf_counter()
            st.leaf_solve(b, f, v)
            ts.append(time.perf_counter() - t)
        dt = min(ts[1:])
        print(f"{name:<28} {dt*1e3:7.2f} ms  {n/dt:9.0f} leaves/s")
