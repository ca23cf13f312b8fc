"""First GPU bring-up: condense a few small configs and compare with the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
from paper_2211_14969_b200 import leaf_gpu as G

rng = np.random.default_rng(0)
for (p, n, kappa) in [(4, 3, 1.0), (6, 4, 3.0), (8, 5, 10.0), (12, 6, 20.0), (13, 3, 5.0), (22, 4, 100.0), (27, 2, 50.0), (42, 2, 500.0)]:
    nx = n; ny = 1
    a = 1.0 / nx
    b = rng.uniform(0, 1, (n, p * p)); f = rng.uniform(-1, 1, (n, p * p))
    t0 = time.time()
    r = O.batched_condense(p, a, kappa, b, f)
    t1 = time.time()
    with G.LeafStage(p, nx, ny, kappa, a=a) as st:
        T, w, s = st.condense(b, f, raise_on_resonance=False)
        tm = st.timing()
    t2 = time.time()
    eT = np.linalg.norm(T - r["T"], axis=(1, 2)) / np.linalg.norm(r["T"], axis=(1, 2))
    ew = np.linalg.norm(w - r["w"], axis=1) / np.maximum(np.linalg.norm(r["w"], axis=1), 1e-300)
    print(f"p={p:2d} n={n} kappa={kappa}: relFro T max {eT.max():.3e}  w max {ew.max():.3e}  status {s.tolist()}  "
          f"oracle {t1-t0:.3f}s gpu {t2-t1:.3f}s timing {tm}", flush=True)
