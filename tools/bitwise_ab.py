"""T/w of a few configs from the library selected by HPS_LIB_PATH, saved for a bitwise A/B
between builds (kernel-layout changes must not change a single bit):
  HPS_LIB_PATH=... python tools/bitwise_ab.py out.npz ; python tools/bitwise_ab.py --cmp a.npz b.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k].view(np.int64), b[k].view(np.int64))]
    print("bitwise equal" if not bad else f"DIFFER: {bad}")
    sys.exit(1 if bad else 0)
from paper_2211_14969_b200 import leaf_gpu as G, problems as P
out = {}
for name, n in (("C4", 300), ("C3", 300), ("C2", 700), ("C1", 128)):
    cfg = P.config(name)
    p = cfg["p"]
    X, Y = P.leaf_coords(cfg["nx"], cfg["ny"], p, elements=np.arange(cfg["n_leaves"] // 2, cfg["n_leaves"] // 2 + n))
    b = P.crystal_field(X, Y); f = np.random.default_rng(2).uniform(-1, 1, X.shape)
    with G.LeafStage(p, cfg["nx"], cfg["ny"], cfg["kappa"], a=cfg["a"]) as st:
        T, w, s = st.condense(b, f, e0=cfg["n_leaves"] // 2)
        if p <= 12:
            st.set_option(G.OPT_SMALL_KERNEL, 0)
            T2, w2, _ = st.condense(b, f, e0=cfg["n_leaves"] // 2)
            out[name + "_blocked_T"] = T2; out[name + "_blocked_w"] = w2
    out[name + "_T"] = T; out[name + "_w"] = w
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
