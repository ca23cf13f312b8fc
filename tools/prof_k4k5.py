"""Profiling driver for K4 (scatter into the reduced system) and K5 (leaf solve):
C4-sized scatter on device-resident T/w, and a C2-sized batched leaf solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
from paper_2211_14969_b200 import leaf_gpu as G, problems as P

cfg = P.config("C4")
p, nx, ny = cfg["p"], cfg["nx"], cfg["ny"]
nb = 4 * (p - 1)
st = G.LeafStage(p, nx, ny, cfg["kappa"], a=cfg["a"], workspace_bytes=8 << 30)
rp, ci = st.reduced_pattern()
T = torch.randn((nx * ny, nb, nb), dtype=torch.float64, device="cuda")
w = torch.randn((nx * ny, nb), dtype=torch.float64, device="cuda")
g = torch.from_numpy(P.boundary_samples(nx, ny, p, P.gaussian_pulse)).cuda()
vals = torch.empty(ci.size, dtype=torch.float64, device="cuda")
rhs = torch.empty(rp.size - 1, dtype=torch.float64, device="cuda")
L = G.lib()
s = torch.cuda.Stream()
torch.cuda.synchronize()
for r in range(2):
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    rc = L.hps_gpu_assemble_reduced_device(st._h, C.c_void_p(T.data_ptr()), C.c_void_p(w.data_ptr()),
                                           C.c_void_p(g.data_ptr()), C.c_void_p(vals.data_ptr()),
                                           C.c_void_p(rhs.data_ptr()), C.c_void_p(s.cuda_stream))
    ev1.record(s); torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    qq = p - 2
    byts = 8 * (nx * ny) * (nb * nb + nb + (4 * qq) ** 2 + 4 * qq)   # B_K4(p) per leaf
    print(f"K4 rep {r}: rc={rc} {ms:.3f} ms, nnz={ci.size}, B_K4 {byts/1e9:.2f} GB -> {byts/ms/1e6:.1f} GB/s")
st.close()
c2 = P.config("C2")
p2, n2 = c2["p"], c2["n_leaves"]
X, Y = P.leaf_coords(c2["nx"], c2["ny"], p2)
b2 = P.crystal_field(X, Y); f2 = np.zeros_like(X)
v2 = np.random.default_rng(0).uniform(-1, 1, (n2, 4 * (p2 - 1)))
with G.LeafStage(p2, c2["nx"], c2["ny"], c2["kappa"], a=c2["a"]) as s2:
    for r in range(2):
        u = s2.leaf_solve(b2, f2, v2)
        print(f"K5 leaf_solve C2 rep {r}: {s2.timing()}")
