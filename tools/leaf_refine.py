"""Accuracy of T for the worst C4 leaf (near-resonant) against an extended-precision
reference: T_ref = D_b - D_i X with X = A_ii^{-1} A_ib from float64 LU plus iterative
refinement whose residuals are computed in long double (x87 80-bit).  Reports the relative
Frobenius error of the GPU's T and of the CPU oracle's T against T_ref, i.e. which of the two
backward-stable computations is closer to the exact Schur complement.
  python tools/leaf_refine.py [--leaf 4543] [--out gpurun_out/leaf_refine.json]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.linalg as sl
from oracle import pyoracle as O
from paper_2211_14969_b200 import problems as P

ap = argparse.ArgumentParser()
ap.add_argument("--leaf", type=int, default=4543)
ap.add_argument("--out", default="")
a = ap.parse_args()
cfg = P.config("C4")
p, nx, kappa = cfg["p"], cfg["nx"], cfg["kappa"]
X, Y = P.leaf_coords(nx, nx, p, elements=np.array([a.leaf]))
b = P.crystal_field(X, Y); f = np.zeros_like(b)
it, bd = O.leaf_index(p)
A, Dn = O.build_leaf(p, cfg["a"], kappa, b[0])
Aii, Aib = A[np.ix_(it, it)], A[np.ix_(it, bd)]
Di, Db = Dn[:, it], Dn[:, bd]
lu = sl.lu_factor(Aii)
Xs = sl.lu_solve(lu, Aib)
L = np.longdouble
XL = Xs.astype(L)
AiiL, AibL = Aii.astype(L), Aib.astype(L)
hist = []
for k in range(3):
    R = AibL - AiiL @ XL
    dX = sl.lu_solve(lu, R.astype(np.float64))
    XL = XL + dX.astype(L)
    hist.append(float(np.linalg.norm(dX) / np.linalg.norm(Xs)))
T_ref = (Db.astype(L) - Di.astype(L) @ XL)
T_o = O.batched_condense(p, cfg["a"], kappa, b, f)["T"][0]
from paper_2211_14969_b200 import leaf_gpu as G
with G.LeafStage(p, nx, nx, kappa, a=cfg["a"], workspace_bytes=4 << 30) as st:
    T_g = st.condense(b, f, e0=a.leaf)[0][0]
nrm = float(np.sqrt(np.sum(T_ref.astype(np.float64) ** 2)))
err = lambda T: float(np.sqrt(np.sum((T.astype(L) - T_ref) ** 2)) / nrm)
out = dict(leaf=a.leaf, b_min=float(b.min()), b_max=float(b.max()), refinement_steps_rel=hist,
           cond_est=float(np.linalg.cond(Aii, 1)), relfro_gpu_vs_ref=err(T_g), relfro_oracle_vs_ref=err(T_o),
           relfro_gpu_vs_oracle=float(np.linalg.norm(T_g - T_o) / np.linalg.norm(T_o)))
print(json.dumps(out))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
