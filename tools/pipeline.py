"""Whole HPS pipeline on one config with per-stage timing (BASELINE north star: the leaf stage
on the GPU, the reduced sparse direct solve unchanged on the host and timed separately):

  condense (GPU, C-ABI host buffers) -> assemble_reduced (GPU, CSR) -> SuperLU (host)
  -> leaf_solve (GPU) -> matrix-free residual (GPU, Eq. 7 relerr_res)

  python tools/pipeline.py --config C2 [--out profiles/r01_pipeline_c2.json]
Gaussian-pulse Dirichlet data, crystal b(x), f ~ U(-1,1) seed 2 (SURVEY §8d parity inputs).
"""
import argparse, json, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from paper_2211_14969_b200 import leaf_gpu as G, problems as P
import hps_harness as H

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--out", default="")
ap.add_argument("--slab-width", type=int, default=0)
ap.add_argument("--no-superlu", action="store_true", help="skip the host sparse solve (hours at C4)")
ap.add_argument("--workspace-gb", type=float, default=0.0, help="leaf-stage HBM budget (0: 70%% of free)")
a = ap.parse_args()
cfg = P.config(a.config)
p, nx, ny, kappa = cfg["p"], cfg["nx"], cfg["ny"], cfg["kappa"]
X, Y = P.leaf_coords(nx, ny, p)
b = P.crystal_field(X, Y); f = np.random.default_rng(2).uniform(-1, 1, X.shape)
gb = P.boundary_samples(nx, ny, p, P.gaussian_pulse)
t = {}
with G.LeafStage(p, nx, ny, kappa, workspace_bytes=int(a.workspace_gb * 2**30)) as st:
    st.condense(b[:1], f[:1])                               # warm-up (module load, workspace)
    t0 = time.perf_counter(); T, w, s = st.condense(b, f); t["condense_s"] = time.perf_counter() - t0
    t0 = time.perf_counter(); rp, ci, vals, rhs = st.assemble_reduced(T, w, gb); t["assemble_reduced_s"] = time.perf_counter() - t0
    t["k4_ms"] = st.timing()["ms_scatter"]
    # fused: T stays in HBM, only the reduced system comes back (pinned outputs)
    pv = G.pinned_empty(vals.shape); pr = G.pinned_empty(rhs.shape)
    st.condense_assemble(b, f, gb, out=(pv, pr))            # warm-up of the resident buffers
    t0 = time.perf_counter(); st.condense_assemble(b, f, gb, out=(pv, pr))
    t["condense_assemble_fused_s"] = time.perf_counter() - t0
    tf = st.timing(); t["fused_k4_ms"] = tf["ms_scatter"]; t["fused_device_ms"] = tf["ms_total"]
    assert np.array_equal(pv, vals) and np.array_equal(pr, rhs)
    A = sp.csr_matrix((vals, ci, rp), shape=(rp.size - 1, rp.size - 1))
    ua = None
    if not a.no_superlu:
        t0 = time.perf_counter(); ua = spla.spsolve(A.tocsc(), rhs); t["host_superlu_s"] = time.perf_counter() - t0
    # GPU SlabLU on the BSR view of the same system
    from paper_2211_14969_b200 import slab_gpu as SG
    brp, bci, bva, brh = st.assemble_reduced_bsr(T, w, gb)
    with SG.SlabLU(p, nx, ny, brp, bci, bva, slab_width=a.slab_width) as lu:   # warm-up: library
        lu.solve(rhs)                                                           # handles, JIT, workspaces
    t0 = time.perf_counter()
    with SG.SlabLU(p, nx, ny, brp, bci, bva, slab_width=a.slab_width) as lu:
        t["slablu_factor_s"] = time.perf_counter() - t0
        t0 = time.perf_counter(); ua_s = lu.solve(rhs); t["slablu_solve_s"] = time.perf_counter() - t0
        t["slablu_info"] = lu.get_info()
    if ua is not None:
        t["slablu_vs_superlu_relerr"] = float(np.max(np.abs(ua_s - ua)) / np.max(np.abs(ua)))
    else:
        ua = ua_s
        t["slablu_reduced_residual"] = float(np.linalg.norm(A @ ua_s - rhs) / np.linalg.norm(rhs))
    v = H.leaf_boundary_values(nx, ny, p, ua, gb)
    t0 = time.perf_counter(); ul = st.leaf_solve(b, f, v); t["leaf_solve_s"] = time.perf_counter() - t0
    t0 = time.perf_counter(); res = st.residual(b, f, ul); t["residual_s"] = time.perf_counter() - t0
cls = H.classify(nx, ny, p)
gx, gy = H.global_coords(nx, ny, p)
g2 = float(np.sum(P.gaussian_pulse(gx, gy)[cls == 2] ** 2))
relerr = math.sqrt((res["r_int2"] + res["r_flux2"]) / (res["f_int2"] + g2))
N = (nx * (p - 1) + 1) * (ny * (p - 1) + 1)
out = dict(config=a.config, p=p, nx=nx, ny=ny, kappa=kappa, dof=N, n_active=int(rp.size - 1), nnz=int(ci.size),
           resonant=int(s.sum()), relerr_res=relerr, **{k: (round(v_, 4) if isinstance(v_, float) and k.endswith(("_s", "_ms")) else v_) for k, v_ in t.items()})
print(json.dumps(out))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
