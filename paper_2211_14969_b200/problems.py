"""Problem data on the leaf grid (host side, numpy).

Mirrors the reference ``problems`` module as far as the leaf
stage needs it: pointwise sampling of b(x) and f(x) at every leaf's p*p local
Chebyshev nodes ("sampled pointwise at collocation nodes"), the
Dirichlet data g on the four sides of the unit square, and the presets used by
the BASELINE configs.  Sampling is outside the product timing:
the C-ABI consumes per-leaf samples.
"""
from __future__ import annotations

import math

import numpy as np


def cheb_nodes(p: int) -> np.ndarray:
    """Ascending Chebyshev-Gauss-Lobatto nodes on [-1, 1]."""
    k = np.arange(p, dtype=np.float64)
    return np.sin(math.pi * (2.0 * k - (p - 1)) / (2.0 * (p - 1)))


def leaf_coords(nx: int, ny: int, p: int, a: float | None = None, elements=None):
    """Physical (x, y) of every leaf's local nodes, shape (n_leaves, p*p) each.

    Local order l = iy*p + ix; element e = ey*nx + ex.
    """
    if a is None:
        a = 1.0 / nx
    xh = cheb_nodes(p)
    off = (xh + 1.0) * (a / 2.0)
    if elements is None:
        elements = np.arange(nx * ny)
    elements = np.asarray(elements)
    ex = (elements % nx).astype(np.float64)
    ey = (elements // nx).astype(np.float64)
    X = ex[:, None, None] * a + off[None, None, :]          # (n, 1, p) -> varies with ix
    Y = ey[:, None, None] * a + off[None, :, None]          # (n, p, 1) -> varies with iy
    X = np.broadcast_to(X, (elements.size, p, p)).reshape(elements.size, p * p)
    Y = np.broadcast_to(Y, (elements.size, p, p)).reshape(elements.size, p * p)
    return np.ascontiguousarray(X), np.ascontiguousarray(Y)


def global_axis(n_el: int, p: int, a: float) -> np.ndarray:
    """Coordinates of the n_el*(p-1)+1 global grid lines along one axis, taken from
    the lexicographically first element that holds each node."""
    xh = cheb_nodes(p)
    off = (xh + 1.0) * (a / 2.0)
    g = np.arange(n_el * (p - 1) + 1)
    e = np.maximum(0, (g - 1) // (p - 1))
    i = g - e * (p - 1)
    return e * a + off[i]


def boundary_samples(nx: int, ny: int, p: int, g, a: float | None = None) -> np.ndarray:
    """g_bnd = [south(Nx), north(Nx), west(Ny), east(Ny)] (the C-ABI layout)."""
    if a is None:
        a = 1.0 / nx
    xs = global_axis(nx, p, a)
    ys = global_axis(ny, p, a)
    X1, Y1 = nx * a, ny * a
    return np.concatenate([g(xs, np.zeros_like(xs)), g(xs, np.full_like(xs, Y1)),
                           g(np.zeros_like(ys), ys), g(np.full_like(ys, X1), ys)]).astype(np.float64)


# ---- presets -------------------------------------------------------------------------------

def crystal_centres() -> np.ndarray:
    """6x6 lattice at spacing 0.08 inside [0.3, 0.7]^2."""
    c = 0.3 + 0.08 * np.arange(6)
    cx, cy = np.meshgrid(c, c, indexing="xy")
    return np.stack([cx.ravel(), cy.ravel()], axis=1)


def crystal_field(x, y, sigma: float = 0.02, depth: float = 0.9):
    """b(x) = clamp(1 - sum_i depth*exp(-|x-c_i|^2/sigma^2), 0, 1)."""
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64)
    s = np.zeros(np.broadcast(x, y).shape)
    inv = 1.0 / (sigma * sigma)
    for cx, cy in crystal_centres():
        s += depth * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) * inv)
    return np.clip(1.0 - s, 0.0, 1.0)


def gaussian_pulse(x, y):
    """g = exp(-2000 (y - 0.5)^2) on x = 0, else 0 (Eq. 8)."""
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64)
    return np.where(x == 0.0, np.exp(-2000.0 * (y - 0.5) ** 2), 0.0)


def analytic_j0(kappa: float):
    """u_true = J0(kappa |x - (-0.1, 0.5)|) (Eq. 6)."""
    from scipy.special import j0

    def u(x, y):
        return j0(kappa * np.hypot(np.asarray(x) + 0.1, np.asarray(y) - 0.5))
    return u


def config(name: str):
    """BASELINE.json configs restated as inputs."""
    table = {
        "C1": dict(p=12, nx=16, ny=16, kappa=0.0),
        "C2": dict(p=22, nx=48, ny=48, kappa=100.0),
        "C3": dict(p=32, nx=64, ny=64, kappa=250.0),
        "C4": dict(p=42, nx=98, ny=98, kappa=500.0),
    }
    c = dict(table[name])
    c["a"] = 1.0 / c["nx"]
    c["n_leaves"] = c["nx"] * c["ny"]
    c["N"] = (c["nx"] * (c["p"] - 1) + 1) * (c["ny"] * (c["p"] - 1) + 1)
    return c


def flops_condense(p: int) -> float:
    """F_condense(p) = 2/3 n_i^3 + 2 n_i^2 n_b + 2 n_b^2 n_i."""
    ni, nb = (p - 2) ** 2, 4 * (p - 1)
    return (2.0 / 3.0) * ni ** 3 + 2.0 * ni ** 2 * nb + 2.0 * nb ** 2 * ni


def flops_leaf_solve(p: int) -> float:
    """F_leafsolve(p) = 2/3 n_i^3 + 2 n_i^2 + 2 n_i n_b with the recompute policy."""
    ni, nb = (p - 2) ** 2, 4 * (p - 1)
    return (2.0 / 3.0) * ni ** 3 + 2.0 * ni ** 2 + 2.0 * ni * nb
