// ============================================================================
//  K5 — batched leaf-solution recovery (north star #5; replaces leaf_solve,
//  SPEC.md:297-305, and the interior part of reconstruct_full_solution,
//  SPEC.md:363-367).
//
//  Pipeline per chunk (hps_host.cpp):
//    recompute policy: K1s [A_ii | f_i - A_ib v] -> K2 (factor + trailing column,
//                      y = L^{-1} P rhs) -> K5 back substitution
//    store policy    : rhs into the kept condense workspace -> K2 trailing-only
//                      -> K5 (same code on the same factors: bitwise equal)
//  K5 (this file): one CTA per leaf.  Blocked back substitution over the
//  64-row blocks of U (physical rows through perm): a warp-per-row GEMV
//  against the already-solved tail, then a one-warp triangular solve of the
//  64x64 diagonal block.  Finally the p*p local vector u (interior from the
//  solve, boundary = v) in local order.  HBM bound: reads U once (ni^2/2).
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

__global__ void __launch_bounds__(256) k5_backsolve_kernel(LeafDims d, const double* __restrict__ ws,
                                                           const short* __restrict__ perm,
                                                           const double* __restrict__ v,
                                                           double* __restrict__ u) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* x = reinterpret_cast<double*>(smem_raw);
  short* ps = reinterpret_cast<short*>(x + d.ni);
  const int leaf = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* M = ws + (size_t)leaf * d.leaf_stride;
  const short* P = perm + (size_t)leaf * d.Rpad;
  const int ni = d.ni, ld = d.ld;
  for (int k = tid; k < ni; k += 256) {
    ps[k] = P[k];
    x[k] = M[(size_t)P[k] * ld + d.tb0];
  }
  __syncthreads();
  for (int I = d.nblk - 1; I >= 0; --I) {
    const int r0 = 64 * I;
    const int nr = min(64, ni - r0);
    const int c1 = r0 + nr;
    if (c1 < ni) {
      for (int k = r0 + warp; k < c1; k += 8) {
        const double* urow = M + (size_t)ps[k] * ld;
        double s = 0.0;
        for (int j = c1 + lane; j < ni; j += 32) s = fma(urow[j], x[j], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) x[k] -= s;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double y0 = lane < nr ? x[r0 + lane] : 0.0;
      double y1 = lane + 32 < nr ? x[r0 + lane + 32] : 0.0;
      const double* row0 = M + (size_t)ps[r0 + min(lane, nr - 1)] * ld;
      const double* row1 = M + (size_t)ps[r0 + min(lane + 32, nr - 1)] * ld;
      for (int kk = nr - 1; kk >= 0; --kk) {
        const double own = (kk < 32) ? y0 : y1;
        const double val = __shfl_sync(0xffffffffu, own, kk & 31);
        const double xk = val / M[(size_t)ps[r0 + kk] * ld + r0 + kk];
        if (lane == (kk & 31)) {
          if (kk < 32) y0 = xk; else y1 = xk;
        }
        if (lane < kk) y0 = fma(-row0[r0 + kk], xk, y0);
        if (lane + 32 < kk) y1 = fma(-row1[r0 + kk], xk, y1);
      }
      if (lane < nr) x[r0 + lane] = y0;
      if (lane + 32 < nr) x[r0 + lane + 32] = y1;
    }
    __syncthreads();
  }
  const int p = d.p, q = p - 2, nb = 4 * (p - 1);
  const double* vl = v + (size_t)leaf * nb;
  double* ul = u + (size_t)leaf * p * p;
  for (int l = tid; l < p * p; l += 256) {
    const int iy = l / p, ix = l % p;
    double val;
    if (iy >= 1 && iy <= p - 2 && ix >= 1 && ix <= p - 2) val = x[(iy - 1) * q + (ix - 1)];
    else if (iy == 0) val = vl[ix];                          // S
    else if (ix == p - 1) val = vl[p - 1 + iy];              // E (incl. NE corner)
    else if (iy == p - 1) val = vl[2 * p - 1 + ix];          // N (incl. NW corner)
    else val = vl[3 * p - 3 + iy];                           // W
    ul[l] = val;
  }
}

void launch_backsolve(const LeafDims& d, const double* ws, const short* perm, const double* v,
                      double* u, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  const size_t smem = (size_t)d.ni * sizeof(double) + (size_t)d.ni * sizeof(short) + 16;
  // a per-device function attribute: set on every launch (several GPUs in one process)
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k5_backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k5_backsolve_kernel<<<n_leaves, 256, smem, st>>>(d, ws, perm, v, u);
}

// K5s — leaf_solve from a stored S_solve (HPS_STORAGE_S_SOLVE; SPEC.md:263,297-305,313;
// PAPER.md:162-165): interior = A_ii^{-1} f_i + S_solve v with [S_solve | A_ii^{-1} f_i] kept
// per leaf (n_i x (n_b + 1), row-major) by the condense call.  One CTA per leaf, one warp per
// interior row: lanes stride the n_b + 1 row entries, fixed shuffle tree (deterministic).  HBM
// bound: reads the stored row block once (8 n_i (n_b + 1) bytes per leaf).
__global__ void __launch_bounds__(256) k5s_apply_kernel(int p, const double* __restrict__ S,
                                                        const double* __restrict__ v, double* __restrict__ u) {
  const int leaf = blockIdx.x;
  const int q = p - 2, ni = q * q, nb = 4 * (p - 1), pp = p * p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane >> 3, l8 = lane & 7;   // 4 rows per warp, 8 lanes per row
  const double* Sl = S + (size_t)leaf * ni * (nb + 1);
  const double* vl = v + (size_t)leaf * nb;
  double* ul = u + (size_t)leaf * pp;
  __shared__ double vs[4 * 64];   // nb <= 4 (p - 1) <= 256 for p <= 65
  for (int k = threadIdx.x; k < nb; k += 256) {
    const double x = __ldg(vl + k);
    vs[k] = x;
    int e;
    ul[boundary_local(k, p, &e)] = x;
  }
  __syncthreads();
  // u_i = [S_solve | A_ii^{-1} f]_i . [v ; 1]: 8 lanes stride a row with three independent
  // partial sums (more loads in flight per warp than one warp per row), then a 3-step
  // shuffle reduction inside the 8-lane group.
  for (int b = 4 * warp; b < ni; b += 32) {   // warp-uniform trip count (full-mask shuffles)
    const int i = b + sub;
    const bool ok = i < ni;
    const double* row = Sl + (size_t)(ok ? i : ni - 1) * (nb + 1);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    int k = l8;
    for (; k + 16 < nb; k += 24) {
      a0 = fma(__ldcs(row + k), vs[k], a0);
      a1 = fma(__ldcs(row + k + 8), vs[k + 8], a1);
      a2 = fma(__ldcs(row + k + 16), vs[k + 16], a2);
    }
    for (; k < nb; k += 8) a0 = fma(__ldcs(row + k), vs[k], a0);
    double acc = (a0 + a1) + a2;
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (ok && l8 == 0) ul[interior_local(i, p)] = __dadd_rn(__ldcs(row + nb), acc);
  }
}

void launch_stored_solve(int p, const double* S, const double* v, double* u, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  k5s_apply_kernel<<<n_leaves, 256, 0, st>>>(p, S, v, u);
}

}  // namespace hpsg
