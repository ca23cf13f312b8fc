"""Profiling driver: condense `n` leaves of config C4 (or --p) through the device-resident
C-ABI twice (the second launch is the one ncu captures with -s/-c)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2211_14969_b200 import leaf_gpu as G, problems as P

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=296)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = P.config(a.config)
p, n = cfg["p"], a.n
X, Y = P.leaf_coords(cfg["nx"], cfg["ny"], p, elements=np.arange(n))
b = torch.from_numpy(P.crystal_field(X, Y)).cuda(); f = torch.zeros_like(b)
nb = 4 * (p - 1)
T = torch.empty((n, nb, nb), dtype=torch.float64, device="cuda"); w = torch.empty((n, nb), dtype=torch.float64, device="cuda")
s = torch.empty(n, dtype=torch.int32, device="cuda")
st = G.LeafStage(p, cfg["nx"], cfg["ny"], cfg["kappa"], a=cfg["a"])
strm = torch.cuda.Stream()
print("resident K2 CTAs:", st.info()["resident_ctas"], flush=True)
torch.cuda.synchronize()
for r in range(a.reps):
    st.reset_timing()
    st.condense_device(0, n, b.data_ptr(), f.data_ptr(), T.data_ptr(), w.data_ptr(), s.data_ptr(), strm.cuda_stream)
    tm = st.timing()
    k2 = tm["ms_lu_schur"]
    print(f"rep {r}: K1 {tm['ms_assemble']:.2f} ms  K2 {k2:.2f} ms  K2 {n*P.flops_condense(p)/k2/1e9:.2f} TF/s")
torch.cuda.synchronize()
st.close()
