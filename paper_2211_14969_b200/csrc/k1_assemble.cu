// ============================================================================
//  K1 — leaf operator assembly (north star #1; replaces build_leaf_operator,
//  SPEC.md:270-278, and the block extraction in condense_leaf).
//
//  Writes every leaf's augmented matrix (hps_device.cuh layout) straight into
//  the HBM workspace: interior rows of -(D2 (x) I) - (I (x) D2) - kappa^2 diag(b)
//   and the outward-normal rows D_n.
//  HBM-write bound: every 16-byte store is a coalesced double2 of one row.
//  Entries are evaluated with explicit _rn intrinsics in the same operation
//  order as the CPU oracle (oracle/hps_oracle.cpp a_entry/dn_entry), so A is
//  bit-identical to the oracle's.
// ============================================================================
#include "hps_assembly.cuh"
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

// grid (ceil(Rpad / kRows), n_leaves), block 256.
constexpr int kRows = 8;

// Boundary position of local node (y, x) on the leaf boundary (SPEC.md:314 order).
__device__ __forceinline__ int boundary_pos(int y, int x, int p) {
  if (y == 0) return x;                   // S (incl. SW, SE)
  if (x == p - 1) return p - 1 + y;       // E (incl. NE)
  if (y == p - 1) return 2 * p - 1 + x;   // N (incl. NW)
  return 3 * p - 3 + y;                   // W
}
// Column of local node (y, x) in the augmented layout.
__device__ __forceinline__ int node_col(int y, int x, int p, int tb0) {
  if (y >= 1 && y <= p - 2 && x >= 1 && x <= p - 2) return (y - 1) * (p - 2) + (x - 1);
  return tb0 + boundary_pos(y, x, p);
}

// K1: one CTA per kRows rows of one leaf, one warp per row.  Each warp first evaluates
// its row's <= 2p+1 structural nonzeros into registers (table loads in flight), then all
// threads stream zeros over the CTA's rows with 16-byte stores (the operator is >95%
// zeros: HBM-write bound), and after the barrier the warps scatter their nonzeros --
// exactly the entries a_entry / dn_entry evaluate (same IEEE sequence as the oracle).
__global__ void __launch_bounds__(256) k1_assemble_kernel(
    LeafDims d, const int* __restrict__ rowcode, const int* __restrict__ colcode,
    const double* __restrict__ Ds, const double* __restrict__ D2, double k2,
    const double* __restrict__ b, const double* __restrict__ f, double* __restrict__ ws,
    const int* __restrict__ inject) {
  const int leaf = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  const int p = d.p, q = p - 2, pp = p * p;
  const double* bl = b + (size_t)leaf * pp;
  const double* fl = f + (size_t)leaf * pp;
  const bool inj = inject && inject[leaf];
  double* W = ws + (size_t)leaf * d.leaf_stride;
  const int half = d.ld >> 1;
  const int nrows = min(kRows, d.Rpad - r0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = r0 + warp;
  // ---- phase 0: this warp's row nonzeros into registers (2 line positions per lane) ----
  double val[2][2];
  int col[2][2];   // -1: nothing to write
  double fval = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) col[h][0] = col[h][1] = -1;
  if (warp < nrows && r < d.R) {
    const int rc = __ldg(rowcode + r);
    const int iy = rc & 255, ix = (rc >> 8) & 255;
    if (r < d.ni) {
      const int l = iy * p + ix;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j >= p) continue;
        // row line (jy == iy): node (iy, j)
        const bool int_row = j >= 1 && j <= q;
        if (!(int_row && inj && r == 0)) {
          double v;
          if (j == ix) {
            v = -__ldg(D2 + iy * p + iy);
            v = __dsub_rn(v, __ldg(D2 + ix * p + ix));
            v = __dsub_rn(v, __dmul_rn(k2, __ldg(bl + l)));
          } else {
            v = -__ldg(D2 + ix * p + j);
          }
          val[h][0] = v;
          col[h][0] = node_col(iy, j, p, d.tb0);
        }
        // column line (jx == ix, jy != iy): node (j, ix)
        const bool int_col = j >= 1 && j <= q;
        if (j != iy && !(int_col && inj && r == 0)) {
          val[h][1] = -__ldg(D2 + iy * p + j);
          col[h][1] = node_col(j, ix, p, d.tb0);
        }
      }
      if (lane == 0) fval = __ldg(fl + l);
    } else {
      const int edge = (rc >> 18) & 3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        if (j >= p) continue;
        if (edge == 0 || edge == 2) {   // S: -d/dy, N: +d/dy along the column line
          const double v = __ldg(Ds + iy * p + j);
          val[h][0] = edge == 0 ? -v : v;
          col[h][0] = node_col(j, ix, p, d.tb0);
        } else {                        // E: +d/dx, W: -d/dx along the row line
          const double v = __ldg(Ds + ix * p + j);
          val[h][0] = edge == 3 ? -v : v;
          col[h][0] = node_col(iy, j, p, d.tb0);
        }
      }
    }
  }
  // ---- phase 1: stream zeros over the CTA's rows ----
  double2* W2 = reinterpret_cast<double2*>(W + (size_t)r0 * d.ld);
  for (int idx = threadIdx.x; idx < nrows * half; idx += blockDim.x) W2[idx] = make_double2(0.0, 0.0);
  __syncthreads();
  // ---- phase 2: scatter the nonzeros ----
  if (warp >= nrows || r >= d.R) return;
  double* row = W + (size_t)r * d.ld;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (col[h][t] >= 0) row[col[h][t]] = val[h][t];
  if (r < d.ni && lane == 0) row[d.tb0 + d.nb] = fval;
}

// ||A_ii||_inf per leaf: row sums over the sparse cross stencil in
// ascending column order (bit-identical to the oracle's dense ascending sum).
__global__ void __launch_bounds__(256) k1_aii_norm_kernel(LeafDims d, const double* __restrict__ D2,
                                                          double k2, const double* __restrict__ b,
                                                          const int* __restrict__ inject,
                                                          double* __restrict__ norms) {
  const int leaf = blockIdx.x;
  const int p = d.p, q = p - 2;
  const double* bl = b + (size_t)leaf * p * p;
  const bool inj = inject && inject[leaf];
  double best = 0.0;
  for (int i = threadIdx.x; i < d.ni; i += blockDim.x) {
    if (inj && i == 0) continue;
    const int iy = i / q + 1, ix = i % q + 1;
    double s = 0.0;
    for (int jy = 1; jy <= q; ++jy) {
      if (jy != iy) {
        s = __dadd_rn(s, fabs(__ldg(D2 + iy * p + jy)));
      } else {
        for (int jx = 1; jx <= q; ++jx)
          s = __dadd_rn(s, fabs(a_entry(iy, ix, iy, jx, p, D2, k2, __ldg(bl + iy * p + ix))));
      }
    }
    best = fmax(best, s);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    norms[leaf] = m;
  }
}

// Leaf-solve right-hand side  f_i - A_ib v: the four boundary
// neighbours of interior node (iy, ix) in ascending boundary position
// (S: ix, E: p-1+iy, N: 2p-1+ix, W: 3p-3+iy), same operation order as the oracle.
__device__ __forceinline__ double solve_rhs(int iy, int ix, int p, const double* __restrict__ D2,
                                            const double* __restrict__ fl,
                                            const double* __restrict__ vl) {
  double s = __ldg(fl + iy * p + ix);
  const double aS = -__ldg(D2 + iy * p + 0), aE = -__ldg(D2 + ix * p + p - 1);
  const double aN = -__ldg(D2 + iy * p + p - 1), aW = -__ldg(D2 + ix * p + 0);
  if (aS != 0.0) s = __dsub_rn(s, __dmul_rn(aS, __ldg(vl + ix)));
  if (aE != 0.0) s = __dsub_rn(s, __dmul_rn(aE, __ldg(vl + p - 1 + iy)));
  if (aN != 0.0) s = __dsub_rn(s, __dmul_rn(aN, __ldg(vl + 2 * p - 1 + ix)));
  if (aW != 0.0) s = __dsub_rn(s, __dmul_rn(aW, __ldg(vl + 3 * p - 3 + iy)));
  return s;
}

// Recompute-policy leaf solve: [A_ii | gap | f_i - A_ib v] (no D rows).
__global__ void __launch_bounds__(256) k1_assemble_solve_kernel(
    LeafDims d, const int* __restrict__ rowcode, const int* __restrict__ colcode,
    const double* __restrict__ Ds, const double* __restrict__ D2, double k2,
    const double* __restrict__ b, const double* __restrict__ f, const double* __restrict__ v,
    double* __restrict__ ws, const int* __restrict__ inject) {
  const int leaf = blockIdx.y;
  const int r0 = blockIdx.x * kRows;
  const int pp = d.p * d.p;
  const double* bl = b + (size_t)leaf * pp;
  const double* fl = f + (size_t)leaf * pp;
  const double* vl = v + (size_t)leaf * 4 * (d.p - 1);
  const bool inj = inject && inject[leaf];
  double* W = ws + (size_t)leaf * d.leaf_stride;
  const int half = d.ld >> 1;
  for (int idx = threadIdx.x; idx < kRows * half; idx += blockDim.x) {
    const int r = r0 + idx / half;
    if (r >= d.Rpad) break;
    const int c = (idx % half) * 2;
    const int rc = __ldg(rowcode + r);
    const bool zrow = inj && r == 0;
    double out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cc = __ldg(colcode + c + h);
      if (((rc >> 16) & 3) == 0 && ((cc >> 16) & 3) == 2)
        out[h] = solve_rhs(rc & 255, (rc >> 8) & 255, d.p, D2, fl, vl);
      else
        out[h] = aug_value(rc, cc, d.p, Ds, D2, k2, bl, fl, zrow);
    }
    reinterpret_cast<double2*>(W + (size_t)r * d.ld)[c >> 1] = make_double2(out[0], out[1]);
  }
}

// Store-policy leaf solve: write f_i - A_ib v into column `col` of the kept
// condense workspace (interior rows are physical rows 0..ni-1).
__global__ void __launch_bounds__(256) k1_write_rhs_kernel(LeafDims d, int col,
                                                           const double* __restrict__ D2,
                                                           const double* __restrict__ f,
                                                           const double* __restrict__ v,
                                                           double* __restrict__ ws) {
  const int leaf = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.ni) return;
  const int q = d.p - 2;
  const int iy = i / q + 1, ix = i % q + 1;
  ws[(size_t)leaf * d.leaf_stride + (size_t)i * d.ld + col] =
      solve_rhs(iy, ix, d.p, D2, f + (size_t)leaf * d.p * d.p, v + (size_t)leaf * 4 * (d.p - 1));
}

void launch_assemble(const LeafDims& d, const int* rowcode, const int* colcode, const double* Ds,
                     const double* D2, double k2, const double* b, const double* f, double* ws,
                     double* norms, const int* inject, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  dim3 grid((d.Rpad + kRows - 1) / kRows, n_leaves);
  k1_assemble_kernel<<<grid, 256, 0, st>>>(d, rowcode, colcode, Ds, D2, k2, b, f, ws, inject);
  k1_aii_norm_kernel<<<n_leaves, 256, 0, st>>>(d, D2, k2, b, inject, norms);
}

void launch_assemble_solve(const LeafDims& d, const int* rowcode, const int* colcode,
                           const double* Ds, const double* D2, double k2, const double* b,
                           const double* f, const double* v, double* ws, double* norms,
                           const int* inject, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  dim3 grid((d.Rpad + kRows - 1) / kRows, n_leaves);
  k1_assemble_solve_kernel<<<grid, 256, 0, st>>>(d, rowcode, colcode, Ds, D2, k2, b, f, v, ws,
                                                 inject);
  k1_aii_norm_kernel<<<n_leaves, 256, 0, st>>>(d, D2, k2, b, inject, norms);
}

void launch_write_rhs(const LeafDims& d, int col, const double* D2, const double* f,
                      const double* v, double* ws, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  dim3 grid((d.ni + 255) / 256, n_leaves);
  k1_write_rhs_kernel<<<grid, 256, 0, st>>>(d, col, D2, f, v, ws);
}

}  // namespace hpsg
