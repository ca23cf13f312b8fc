// ============================================================================
//  K6 — matrix-free residual of the global collocation system on the device
//  ("residual evaluation at larger N
//  uses matrix-free row application"; Eq. 7 relerr_res).
//
//  Rows of the global system (assemble_global, tests/hps_harness.py):
//    interior node (iy, ix) of element e:  (A_loc u_e)(iy,ix) - f_e(iy,ix)
//        = -sum_k D2[iy][k] u(k,ix) - sum_k D2[ix][k] u(iy,k) - kappa^2 b u - f
//    active interface node: sum over its two elements of the outward normal derivative
//        (D_n u_e)[k]  (S: -d/dy, E: +d/dx, N: +d/dy, W: -d/dx)
//    Dirichlet / interior-corner rows: identity rows, exactly satisfied by construction.
//  Inputs are leaf-major local solutions u_e (p*p, the hps_gpu_leaf_solve output), b, f.
//  Pass 1 (one CTA per element): interior residual sum of squares and sum f^2 per element,
//  and the element's outward fluxes at the interior nodes of its four edges.  Pass 2 (one
//  CTA per interface edge): flux rows = F[e0] + F[e1] (ascending element ids, fixed order),
//  sum of squares per edge.  Partials are reduced in a fixed order on the host: the
//  result is bitwise reproducible.  HBM bound (reads u, b, f once).
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

__device__ __forceinline__ int edge_side_base(int p, int side) {
  return side == 0 ? 1 : side == 1 ? p : side == 2 ? 2 * p : 3 * p - 2;
}

// Block sum of one double per thread (fixed tree order).
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, red[w]);
  __syncthreads();
  return s;   // valid on thread 0
}

// grid = n_leaves, block 256, dynamic smem = 3 p^2 doubles (u, D2, Ds)
__global__ void __launch_bounds__(256) k6_leaf_residual_kernel(int p, double k2, const double* __restrict__ D2,
                                                               const double* __restrict__ Ds,
                                                               const double* __restrict__ b,
                                                               const double* __restrict__ f,
                                                               const double* __restrict__ u,
                                                               double* __restrict__ flux,
                                                               double* __restrict__ part) {
  extern __shared__ double sm6[];
  __shared__ double red[8];
  const int e = blockIdx.x, pp = p * p, q = p - 2, nb = 4 * (p - 1);
  double* us = sm6;
  double* d2 = sm6 + pp;
  double* ds = sm6 + 2 * pp;
  for (int t = threadIdx.x; t < pp; t += blockDim.x) {
    us[t] = __ldg(u + (size_t)e * pp + t);
    d2[t] = __ldg(D2 + t);
    ds[t] = __ldg(Ds + t);
  }
  __syncthreads();
  double rr = 0.0, ff = 0.0;
  for (int i = threadIdx.x; i < q * q; i += blockDim.x) {
    const int iy = i / q + 1, ix = i % q + 1, l = iy * p + ix;
    double s = 0.0;
    for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(d2[iy * p + k], us[k * p + ix]));
    for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(d2[ix * p + k], us[iy * p + k]));
    const double fl = __ldg(f + (size_t)e * pp + l);
    const double au = __dsub_rn(-s, __dmul_rn(__dmul_rn(k2, __ldg(b + (size_t)e * pp + l)), us[l]));
    const double r = __dsub_rn(au, fl);
    rr = __dadd_rn(rr, __dmul_rn(r, r));
    ff = __dadd_rn(ff, __dmul_rn(fl, fl));
  }
  // outward fluxes at the interior nodes of the four edges (boundary positions base+kk)
  for (int t = threadIdx.x; t < 4 * q; t += blockDim.x) {
    const int side = t / q, kk = t % q, j = kk + 1;
    double s = 0.0;
    switch (side) {
      case 0: for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(ds[k], us[k * p + j])); s = -s; break;            // S
      case 1: for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(ds[(p - 1) * p + k], us[j * p + k])); break;      // E
      case 2: for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(ds[(p - 1) * p + k], us[k * p + j])); break;      // N
      default: for (int k = 0; k < p; ++k) s = __dadd_rn(s, __dmul_rn(ds[k], us[j * p + k])); s = -s; break;          // W
    }
    flux[(size_t)e * nb + edge_side_base(p, side) + kk] = s;
  }
  const double a0 = block_sum(rr, red);
  const double a1 = block_sum(ff, red);
  if (threadIdx.x == 0) {
    part[2 * e] = a0;
    part[2 * e + 1] = a1;
  }
}

// grid = n_edges, block 64
__global__ void __launch_bounds__(64) k6_flux_residual_kernel(MeshDev m, const double* __restrict__ flux,
                                                              double* __restrict__ part) {
  __shared__ double red[8];
  const int ed = blockIdx.x, p = m.p, q = p - 2, nb = 4 * (p - 1);
  const int e0 = m.edge_elems[2 * ed], e1 = m.edge_elems[2 * ed + 1];
  const int s0 = m.edge_sides[2 * ed], s1 = m.edge_sides[2 * ed + 1];
  double rr = 0.0;
  for (int kk = threadIdx.x; kk < q; kk += blockDim.x) {
    const double r = __dadd_rn(__ldg(flux + (size_t)e0 * nb + edge_side_base(p, s0) + kk),
                               __ldg(flux + (size_t)e1 * nb + edge_side_base(p, s1) + kk));
    rr = __dadd_rn(rr, __dmul_rn(r, r));
  }
  const double a = block_sum(rr, red);
  if (threadIdx.x == 0) part[ed] = a;
}

void launch_residual(const MeshDev& m, double k2, const double* D2, const double* Ds, const double* b,
                     const double* f, const double* u, double* flux, double* part_leaf, double* part_edge,
                     int n_leaves, cudaStream_t st) {
  const int p = m.p;
  k6_leaf_residual_kernel<<<n_leaves, 256, 3 * p * p * sizeof(double), st>>>(p, k2, D2, Ds, b, f, u, flux,
                                                                             part_leaf);
  if (m.n_edges > 0) k6_flux_residual_kernel<<<m.n_edges, 64, 0, st>>>(m, flux, part_edge);
}

}  // namespace hpsg
