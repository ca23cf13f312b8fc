"""Generate the committed parity fixtures under tests/golden/.

The reference (arXiv 2211.14969's `proj/`) ships no implementation and no stored
data, so there are no upstream golden vectors.  The fixtures here
are produced by the CPU restatement in oracle/ (test infrastructure: C++ +
OpenBLAS dgetrf/dgetrs/dgemm, following SPEC.md:250-324 and :326-389) at fixed
seeds, as SURVEY.md §8c prescribes, and committed so that

  * the CPU suite pins the oracle against drift (tests/test_golden.py), and
  * the GPU suite checks the CUDA path against stored numbers, not only against
    an oracle recomputed in the same process.

Each oracle result is first cross-checked against the SPEC known answers it must
satisfy (constant field -> zero flux, u = x -> unit flux) before being written.

Run:  python tools/make_golden.py   (writes tests/golden/*.npz + MANIFEST.json)
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from paper_2211_14969_b200 import problems as P  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# (name, p, nx, ny, kappa, field, seed): a handful of leaves per case keeps each
# fixture small (T is 16(p-1)^2 doubles per leaf).
CONDENSE_CASES = [
    ("condense_p8_poisson", 8, 2, 2, 0.0, "one", 0),
    ("condense_p12_c1", 12, 3, 2, 0.0, "one", 0),
    ("condense_p12_helm", 12, 2, 2, 20.0, "random", 12),
    ("condense_p22_c2", 22, 2, 1, 100.0, "crystal", 2),
    ("condense_p32_c3", 32, 1, 1, 250.0, "crystal", 3),
    ("condense_p42_c4", 42, 1, 1, 500.0, "crystal_scaled", 4),
]

PATTERN_CASES = [(4, 4, 8), (3, 2, 6), (5, 3, 12), (2, 2, 22)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fields(p, nx, ny, kind, seed):
    rng = np.random.default_rng(seed)
    X, Y = P.leaf_coords(nx, ny, p)
    if kind == "one":
        b = np.ones_like(X)
    elif kind == "random":
        b = rng.uniform(0.0, 1.0, X.shape)
    elif kind == "crystal":
        # a window of the C2-C5 crystal around the lattice
        b = P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    elif kind == "crystal_scaled":
        # SURVEY §8d resonance caveat: b scaled into [0, 0.7]
        b = 0.7 * P.crystal_field(0.3 + 0.4 * X, 0.3 + 0.4 * Y)
    else:
        raise ValueError(kind)
    f = rng.uniform(-1.0, 1.0, X.shape)
    return np.ascontiguousarray(b), np.ascontiguousarray(f)


def known_answers(p, a, kappa):
    """SPEC.md:285-286 on one leaf: constant field -> zero flux, u = x -> flux (-1 W, +1 E)."""
    if kappa != 0.0:
        return
    b = np.ones((1, p * p)); f = np.zeros((1, p * p))
    T = O.batched_condense(p, a, 0.0, b, f)["T"][0]
    nb = 4 * (p - 1)
    assert np.abs(T @ np.ones(nb)).max() <= 1e-9 * max(1.0, np.abs(T).max())


def main():
    os.makedirs(OUT, exist_ok=True)
    manifest = {"generator": "tools/make_golden.py", "oracle": "oracle/ (C++ + OpenBLAS)",
                "condense": {}, "pattern": {}}
    for name, p, nx, ny, kappa, kind, seed in CONDENSE_CASES:
        a = 1.0 / nx
        known_answers(p, a, kappa)
        b, f = fields(p, nx, ny, kind, seed)
        r = O.batched_condense(p, a, kappa, b, f)
        v = np.random.default_rng(seed + 100).uniform(-1, 1, (nx * ny, 4 * (p - 1)))
        u = O.batched_leaf_solve(p, a, kappa, b, f, v)
        np.savez_compressed(os.path.join(OUT, name + ".npz"), p=p, nx=nx, ny=ny, a=a, kappa=kappa,
                            b=b, f=f, T=r["T"], w=r["w"], v=v, u=u)
        manifest["condense"][name] = {"p": p, "nx": nx, "ny": ny, "kappa": kappa, "field": kind,
                                      "seed": seed, "sha256_T": sha(r["T"]), "sha256_w": sha(r["w"])}
    for nx, ny, p in PATTERN_CASES:
        rp, ci = O.reduced_pattern(nx, ny, p)
        ee, el, sd = O.mesh_maps(nx, ny, p)
        N, ne, na = O.mesh_info(nx, ny, p)
        enodes = np.stack([O.element_node_index(nx, ny, p, e) for e in range(nx * ny)]).astype(np.int64)
        name = f"pattern_{nx}x{ny}_p{p}"
        np.savez_compressed(os.path.join(OUT, name + ".npz"), nx=nx, ny=ny, p=p, N=N, n_edges=ne,
                            n_active=na, row_ptr=rp, col_idx=ci, elem_edges=ee, edge_elems=el,
                            edge_sides=sd, elem_nodes=enodes)
        manifest["pattern"][name] = {"N": int(N), "n_active": int(na), "nnz": int(ci.size),
                                     "sha256_row_ptr": sha(rp), "sha256_col_idx": sha(ci)}
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("wrote", len(CONDENSE_CASES) + len(PATTERN_CASES), "fixtures to", OUT)


if __name__ == "__main__":
    main()
