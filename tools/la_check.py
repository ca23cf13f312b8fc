"""Quick check of the lookahead kernel vs the 2-CTA kernel and the oracle (small cases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
from paper_2211_14969_b200 import leaf_gpu as G

rng = np.random.default_rng(1)
for (p, n, kappa) in [(6, 3, 2.0), (8, 4, 5.0), (12, 5, 20.0), (13, 3, 5.0), (22, 6, 100.0), (27, 3, 50.0), (42, 3, 500.0)]:
    b = rng.uniform(0, 1, (n, p * p)); f = rng.uniform(-1, 1, (n, p * p))
    r = O.batched_condense(p, 1.0 / n, kappa, b, f)
    os.environ["HPS_LOOKAHEAD"] = "1"
    with G.LeafStage(p, n, 1, kappa, a=1.0 / n) as st:
        T1, w1, s1 = st.condense(b, f)
    os.environ["HPS_LOOKAHEAD"] = "0"
    with G.LeafStage(p, n, 1, kappa, a=1.0 / n) as st:
        T0, w0, s0 = st.condense(b, f)
    e1 = np.max(np.linalg.norm(T1 - r["T"], axis=(1, 2)) / np.linalg.norm(r["T"], axis=(1, 2)))
    ew = np.max(np.linalg.norm(w1 - r["w"], axis=1) / np.linalg.norm(r["w"], axis=1))
    print(f"p={p} n={n}: LA relFro T {e1:.2e} w {ew:.2e}  status {s1.tolist()}  LA==2CTA bitwise: {np.array_equal(T1, T0)}", flush=True)
