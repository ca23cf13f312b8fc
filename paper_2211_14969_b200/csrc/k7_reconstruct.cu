// ============================================================================
//  K7 — reconstruct_full_solution on the device:
//    K7a  per-leaf boundary vectors v (SPEC boundary order) from the reduced solution
//         (active nodes) and the Dirichlet data g on Gamma; interior
//         element corners get 0 (their T / A_ib columns are exact zeros);
//    (batched leaf_solve: K1s + K2 + K5, hps_host.cpp)
//    K7b  placement of every leaf's p*p local solution into the full grid, each global
//         node written by exactly one element (its S/W sides and interior, plus the N/E
//         side on the top row / right column of elements);
//    K7c  element corners: Dirichlet data on Gamma; interior corners by the corner policy
//         (SPEC.md:152): the average of the degree-(p-3) interpolants of the four adjacent
//         interface edges (through their p-2 active nodes) evaluated at the corner, in the
//         C++ API's host operation order with _rn intrinsics (bit-identical to it).
//  All HBM-bound gathers / scatters over N values.
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

// active index of global node (gx, gy) or -1 (hps_api.cpp MeshTopology::active_of_global)
__device__ __forceinline__ long long active_of(int p, int nx, int ny, long long gx, long long gy) {
  const long long rx = gx % (p - 1), ry = gy % (p - 1), cx = gx / (p - 1), cy = gy / (p - 1);
  if (rx == 0 && ry != 0 && cx >= 1 && cx <= nx - 1)
    return ((cx - 1) * (2 * ny - 1) + (ny - 1) + cy) * (p - 2) + (ry - 1);
  if (ry == 0 && rx != 0 && cy >= 1 && cy <= ny - 1) return (cx * (2 * ny - 1) + (cy - 1)) * (p - 2) + (rx - 1);
  return -1;
}

// Dirichlet value at a boundary node; g_bnd = [S(Nx) | N(Nx) | W(Ny) | E(Ny)].
__device__ __forceinline__ double g_value(const double* __restrict__ g, long long Nx, long long Ny, long long gx,
                                          long long gy) {
  if (gy == 0) return __ldg(g + gx);
  if (gy == Ny - 1) return __ldg(g + Nx + gx);
  if (gx == 0) return __ldg(g + 2 * Nx + gy);
  return __ldg(g + 2 * Nx + Ny + gy);
}

// grid = n leaves (from e0), block 128
__global__ void __launch_bounds__(128) k7_leaf_boundary_kernel(int p, int nx, int ny, int e0,
                                                               const double* __restrict__ ua,
                                                               const double* __restrict__ g,
                                                               double* __restrict__ v) {
  const int le = blockIdx.x, e = e0 + le, nb = 4 * (p - 1);
  const int ex = e % nx, ey = e / nx;
  const long long Nx = (long long)nx * (p - 1) + 1, Ny = (long long)ny * (p - 1) + 1;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    int edge;
    const int l = boundary_local(k, p, &edge);
    const int iy = l / p, ix = l - iy * p;
    const long long gx = (long long)ex * (p - 1) + ix, gy = (long long)ey * (p - 1) + iy;
    const long long act = active_of(p, nx, ny, gx, gy);
    double val = 0.0;
    if (act >= 0) val = __ldg(ua + act);
    else if (gx == 0 || gy == 0 || gx == Nx - 1 || gy == Ny - 1) val = g_value(g, Nx, Ny, gx, gy);
    v[(size_t)le * nb + k] = val;
  }
}

// grid = n leaves, block 256
__global__ void __launch_bounds__(256) k7_place_kernel(int p, int nx, int ny, int e0, const double* __restrict__ ul,
                                                       double* __restrict__ u) {
  const int le = blockIdx.x, e = e0 + le, pp = p * p;
  const int ex = e % nx, ey = e / nx;
  const long long Nx = (long long)nx * (p - 1) + 1;
  for (int l = threadIdx.x; l < pp; l += blockDim.x) {
    const int iy = l / p, ix = l - iy * p;
    if ((iy < p - 1 || ey == ny - 1) && (ix < p - 1 || ex == nx - 1))
      u[((long long)ey * (p - 1) + iy) * Nx + (long long)ex * (p - 1) + ix] = __ldg(ul + (size_t)le * pp + l);
  }
}

// one thread per element corner (cx, cy) in [0, nx] x [0, ny].  xh: ascending CGL nodes,
// wts[j-1] = 1 / prod_{k != j} (xh[j] - xh[k]) over the p-2 interior nodes (host-computed).
__global__ void __launch_bounds__(256) k7_corner_kernel(int p, int nx, int ny, const double* __restrict__ xh,
                                                        const double* __restrict__ wts,
                                                        const double* __restrict__ ua,
                                                        const double* __restrict__ g, double* __restrict__ u) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long ncx = nx + 1;
  if (idx >= ncx * (ny + 1)) return;
  const int cx = int(idx % ncx), cy = int(idx / ncx);
  const long long Nx = (long long)nx * (p - 1) + 1, Ny = (long long)ny * (p - 1) + 1;
  const long long gx = (long long)cx * (p - 1), gy = (long long)cy * (p - 1);
  if (cx == 0 || cy == 0 || cx == nx || cy == ny) {
    u[gy * Nx + gx] = g_value(g, Nx, Ny, gx, gy);
    return;
  }
  double s = 0.0;
  for (int dir = 0; dir < 4; ++dir) {   // left, right (horizontal line), down, up (vertical)
    const double t = (dir == 0 || dir == 2) ? 1.0 : -1.0;
    double num = 0.0, den = 0.0;
    for (int j = 1; j <= p - 2; ++j) {
      long long x = gx, y = gy;
      if (dir == 0) x = gx - (p - 1) + j;
      if (dir == 1) x = gx + j;
      if (dir == 2) y = gy - (p - 1) + j;
      if (dir == 3) y = gy + j;
      const double val = __ldg(ua + active_of(p, nx, ny, x, y));
      const double c = __ddiv_rn(__ldg(wts + j - 1), __dsub_rn(t, __ldg(xh + j)));
      num = __dadd_rn(num, __dmul_rn(c, val));
      den = __dadd_rn(den, c);
    }
    s = __dadd_rn(s, __ddiv_rn(num, den));
  }
  u[gy * Nx + gx] = __ddiv_rn(s, 4.0);
}

void launch_leaf_boundary(int p, int nx, int ny, int e0, int n, const double* ua, const double* g, double* v,
                          cudaStream_t st) {
  if (n <= 0) return;
  k7_leaf_boundary_kernel<<<n, 128, 0, st>>>(p, nx, ny, e0, ua, g, v);
}

void launch_place(int p, int nx, int ny, int e0, int n, const double* ul, double* u, cudaStream_t st) {
  if (n <= 0) return;
  k7_place_kernel<<<n, 256, 0, st>>>(p, nx, ny, e0, ul, u);
}

void launch_corners(int p, int nx, int ny, const double* xh, const double* wts, const double* ua, const double* g,
                    double* u, cudaStream_t st) {
  const long long nc = (long long)(nx + 1) * (ny + 1);
  k7_corner_kernel<<<unsigned((nc + 255) / 256), 256, 0, st>>>(p, nx, ny, xh, wts, ua, g, u);
}

}  // namespace hpsg
