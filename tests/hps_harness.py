"""Shared test plumbing: the reduced-system pipeline and the global dense oracle.

Test infrastructure.  ``assemble_global`` restates SPEC.md:337-342,354-362 (the
oracle/residual path, out of the product scope) and ``dense_solve`` the oracle
module; both exist only to check the leaf stage end to end
(acceptance 1 at :583).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import pyoracle as O
from paper_2211_14969_b200 import problems as P


def leaf_inputs(nx, ny, p, bfun, ffun, a=None):
    X, Y = P.leaf_coords(nx, ny, p, a)
    b = np.broadcast_to(bfun(X, Y), X.shape).astype(np.float64).copy()
    f = np.broadcast_to(ffun(X, Y), X.shape).astype(np.float64).copy()
    return X, Y, b, f


def global_coords(nx, ny, p, a=None):
    if a is None:
        a = 1.0 / nx
    xs = P.global_axis(nx, p, a); ys = P.global_axis(ny, p, a)
    GX, GY = np.meshgrid(xs, ys, indexing="xy")
    return GX.ravel(), GY.ravel()


def classify(nx, ny, p):
    """Per global node: 0 element-interior, 1 active, 2 Dirichlet, 3 interior corner."""
    N, _, _ = O.mesh_info(nx, ny, p)
    Nx = nx * (p - 1) + 1; Ny = ny * (p - 1) + 1
    g = np.arange(N)
    gx = g % Nx; gy = g // Nx
    cls = np.zeros(N, np.int32)
    onx = gx % (p - 1) == 0; ony = gy % (p - 1) == 0
    bnd = (gx == 0) | (gy == 0) | (gx == Nx - 1) | (gy == Ny - 1)
    cls[(onx | ony)] = 1
    cls[onx & ony] = 3
    cls[bnd] = 2
    return cls


def reduced_solve(nx, ny, p, T, w, g_bnd, assemble=None):
    """assemble_reduced + host sparse direct solve (SuperLU, the paper's comparison solver)."""
    if assemble is None:
        rp, ci, vals, rhs = O.assemble_reduced(nx, ny, p, T, w, g_bnd)
    else:
        rp, ci, vals, rhs = assemble(T, w, g_bnd)
    A = sp.csr_matrix((vals, ci, rp), shape=(rp.size - 1, rp.size - 1))
    u = spla.spsolve(A.tocsc(), rhs)
    return u, (rp, ci, vals, rhs)


def leaf_boundary_values(nx, ny, p, u_active, g_bnd):
    """Per leaf boundary vector v (n_b, SPEC boundary order) from the reduced solution and g.
    Interior corners get 0 (their T/A_ib columns are exactly zero)."""
    n = nx * ny
    nb = 4 * (p - 1)
    _, bd = O.leaf_index(p)
    v = np.zeros((n, nb))
    Nx = nx * (p - 1) + 1
    gS = g_bnd[:Nx]; gN = g_bnd[Nx:2 * Nx]; gW = g_bnd[2 * Nx:2 * Nx + (ny * (p - 1) + 1)]
    gE = g_bnd[2 * Nx + (ny * (p - 1) + 1):]
    for e in range(n):
        gid = O.element_node_index(nx, ny, p, e)[bd]
        act = O.active_of_global(nx, ny, p, gid)
        gx = gid % Nx; gy = gid // Nx
        Ny = ny * (p - 1) + 1
        for k in range(nb):
            if act[k] >= 0:
                v[e, k] = u_active[act[k]]
            elif gy[k] == 0:
                v[e, k] = gS[gx[k]]
            elif gy[k] == Ny - 1:
                v[e, k] = gN[gx[k]]
            elif gx[k] == 0:
                v[e, k] = gW[gy[k]]
            elif gx[k] == Nx - 1:
                v[e, k] = gE[gy[k]]
    return v


def scatter_full(nx, ny, p, u_leaf):
    """Leaf-local solutions -> global vector (first writer wins; shared nodes agree)."""
    N, _, _ = O.mesh_info(nx, ny, p)
    u = np.full(N, np.nan)
    for e in range(nx * ny):
        gid = O.element_node_index(nx, ny, p, e)
        m = np.isnan(u[gid])
        u[gid[m]] = u_leaf[e][m]
    return u


def assemble_global_dense(nx, ny, p, kappa, b_leaf, f_leaf, g_bnd, a=None):
    """Dense N x N collocation system: interior collocation rows,
    flux-continuity rows at active nodes, identity rows at Dirichlet nodes; interior corner
    rows are identity with zero data (decoupled, corner policy SPEC.md:152)."""
    if a is None:
        a = 1.0 / nx
    N, _, _ = O.mesh_info(nx, ny, p)
    it, bd = O.leaf_index(p)
    A = np.zeros((N, N)); rhs = np.zeros(N)
    cls = classify(nx, ny, p)
    Nx = nx * (p - 1) + 1; Ny = ny * (p - 1) + 1
    for e in range(nx * ny):
        gid = O.element_node_index(nx, ny, p, e)
        Al, Dn = O.build_leaf(p, a, kappa, b_leaf[e])
        for i in it:
            A[gid[i], gid] += Al[i]
            rhs[gid[i]] = f_leaf[e][i]
        for k, l in enumerate(bd):
            if cls[gid[l]] == 1:
                A[gid[l], gid] += Dn[k]
    gS = g_bnd[:Nx]; gN = g_bnd[Nx:2 * Nx]; gW = g_bnd[2 * Nx:2 * Nx + Ny]; gE = g_bnd[2 * Nx + Ny:]
    for g in np.nonzero(cls >= 2)[0]:
        A[g, :] = 0.0; A[g, g] = 1.0
        gx, gy = g % Nx, g // Nx
        if cls[g] == 3:
            rhs[g] = 0.0
        elif gy == 0:
            rhs[g] = gS[gx]
        elif gy == Ny - 1:
            rhs[g] = gN[gx]
        elif gx == 0:
            rhs[g] = gW[gy]
        else:
            rhs[g] = gE[gy]
    return A, rhs, cls


def hps_pipeline(nx, ny, p, kappa, b_leaf, f_leaf, g_bnd, condense=None, leaf_solve=None,
                 assemble=None):
    """condense -> assemble_reduced -> sparse solve -> leaf_solve; returns global u (corners NaN-free
    only where defined) and the pieces.  `condense`/`leaf_solve`/`assemble` default to the oracle."""
    a = 1.0 / nx
    if condense is None:
        r = O.batched_condense(p, a, kappa, b_leaf, f_leaf)
        T, w = r["T"], r["w"]
    else:
        T, w = condense(b_leaf, f_leaf)
    ua, red = reduced_solve(nx, ny, p, T, w, g_bnd, assemble)
    v = leaf_boundary_values(nx, ny, p, ua, g_bnd)
    if leaf_solve is None:
        u_leaf = O.batched_leaf_solve(p, a, kappa, b_leaf, f_leaf, v)
    else:
        u_leaf = leaf_solve(b_leaf, f_leaf, v)
    return scatter_full(nx, ny, p, u_leaf), dict(T=T, w=w, u_active=ua, reduced=red, v=v, u_leaf=u_leaf)
