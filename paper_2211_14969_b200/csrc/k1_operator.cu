// ============================================================================
//  K1op — the SPEC's single-leaf operator surface on the GPU:
//    build_leaf_operator: dense A_loc (p^2 x p^2) and the four
//      outward-normal maps D_normal (4 x p x p^2, S, E, N, W, each edge's p nodes
//      ascending) of a batch of leaves, from their b samples;
//    condense_leaf / leaf_solve on a CALLER-GIVEN operator:
//      gather [A_ii | A_ib | f_i ; D_i | D_b | 0] (or [A_ii | f_i - A_ib v]) from
//      A_loc / D_normal into the K2 workspace layout (hps_device.cuh), plus
//      ||A_ii||_inf as a dense ascending row sum.
//  The batched hot path (hps_gpu_condense) assembles from b directly (K1/K2s);
//  these kernels serve the reference's per-leaf operations, which take the
//  operator as a value.  Entries come from hps_assembly.cuh (a_entry/dn_entry:
//  the oracle's IEEE operation sequence), so an operator built here and gathered
//  back reproduces the b-path workspace bit for bit.
// ============================================================================
#include "hps_assembly.cuh"
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

// Node (y, x) of position t along edge `edge` (S: (0, t), E: (t, p-1), N: (p-1, t), W: (t, 0)).
__device__ __forceinline__ void edge_node(int edge, int t, int p, int* y, int* x) {
  switch (edge) {
    case 0: *y = 0; *x = t; break;
    case 1: *y = t; *x = p - 1; break;
    case 2: *y = p - 1; *x = t; break;
    default: *y = t; *x = 0; break;
  }
}

// grid (ceil(rows / 8), n), block 256: rows = p^2 operator rows then 4p normal rows;
// each warp writes one row with coalesced stores.
__global__ void __launch_bounds__(256) k1_leaf_operator_kernel(int p, const double* __restrict__ Ds,
                                                               const double* __restrict__ D2, double k2,
                                                               const double* __restrict__ b,
                                                               double* __restrict__ A,
                                                               double* __restrict__ Dn) {
  const int leaf = blockIdx.y;
  const int pp = p * p;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= pp + 4 * p) return;
  const double* bl = b + (size_t)leaf * pp;
  if (row < pp) {
    const int iy = row / p, ix = row - iy * p;
    const double bv = __ldg(bl + row);
    double* out = A + ((size_t)leaf * pp + row) * pp;
    for (int m = lane; m < pp; m += 32) out[m] = a_entry(iy, ix, m / p, m % p, p, D2, k2, bv);
  } else {
    const int r = row - pp, edge = r / p, t = r - edge * p;
    int iy, ix;
    edge_node(edge, t, p, &iy, &ix);
    double* out = Dn + ((size_t)leaf * 4 * p + r) * pp;
    for (int m = lane; m < pp; m += 32) out[m] = dn_entry(edge, iy, ix, m / p, m % p, p, Ds);
  }
}

// Gather a given operator into the K2 workspace.  solve = 0: condense layout
// [A_ii | gap | A_ib | f_i ; D_i | gap | D_b | 0]; solve = 1: [A_ii | gap | f_i - A_ib v]
// (no D rows).  Boundary position k of the D rows reads D_normal[edge(k)][t(k)] (the owning
// edge of a corner).  f_i - A_ib v sums the nonzero A_ib entries in ascending
// boundary position, the order of the b path's solve_rhs (k1_assemble.cu).
__global__ void __launch_bounds__(256) k1_gather_operator_kernel(LeafDims d, int solve,
                                                                 const double* __restrict__ A,
                                                                 const double* __restrict__ Dn,
                                                                 const double* __restrict__ f,
                                                                 const double* __restrict__ v,
                                                                 double* __restrict__ ws) {
  const int leaf = blockIdx.y;
  const int p = d.p, pp = p * p, nb = 4 * (p - 1);
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= d.Rpad) return;
  double* W = ws + (size_t)leaf * d.leaf_stride + (size_t)r * d.ld;
  const double* Al = A + (size_t)leaf * pp * pp;
  const double* fl = f + (size_t)leaf * pp;
  const double* row = nullptr;
  int lrow = -1;
  if (r < d.ni) {
    lrow = interior_local(r, p);
    row = Al + (size_t)lrow * pp;
  } else if (r < d.R) {
    int edge;
    const int l = boundary_local(r - d.ni, p, &edge);
    const int y = l / p, x = l - y * p;
    const int t = (edge == 0 || edge == 2) ? x : y;
    row = Dn + ((size_t)leaf * 4 * p + edge * p + t) * pp;
  }
  for (int c = lane; c < d.ld; c += 32) {
    double val = 0.0;
    if (row) {
      if (c < d.ni) {
        val = __ldg(row + interior_local(c, p));
      } else if (!solve && c >= d.tb0 && c < d.tb0 + nb) {
        int e;
        val = __ldg(row + boundary_local(c - d.tb0, p, &e));
      } else if (r < d.ni && c == (solve ? d.tb0 : d.tb0 + nb)) {
        double s = __ldg(fl + lrow);
        if (solve) {
          const double* vl = v + (size_t)leaf * nb;
          for (int k = 0; k < nb; ++k) {
            int e;
            const double a = __ldg(row + boundary_local(k, p, &e));
            if (a != 0.0) s = __dsub_rn(s, __dmul_rn(a, __ldg(vl + k)));
          }
        }
        val = s;
      }
    }
    W[c] = val;
  }
}

// ||A_ii||_inf of a given operator: dense row sums of |A_ii| in ascending column order
// (equal, bit for bit, to k1_aii_norm_kernel's sparse sum for the standard operator: the
// skipped entries are exact zeros).
__global__ void __launch_bounds__(256) k1_operator_norm_kernel(LeafDims d, const double* __restrict__ A,
                                                               double* __restrict__ norms) {
  const int leaf = blockIdx.x;
  const int p = d.p, pp = p * p;
  const double* Al = A + (size_t)leaf * pp * pp;
  double best = 0.0;
  for (int i = threadIdx.x; i < d.ni; i += blockDim.x) {
    const double* row = Al + (size_t)interior_local(i, p) * pp;
    double s = 0.0;
    for (int c = 0; c < d.ni; ++c) s = __dadd_rn(s, fabs(__ldg(row + interior_local(c, p))));
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

void launch_leaf_operator(int p, const double* Ds, const double* D2, double k2, const double* b, double* A,
                          double* Dn, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  dim3 grid((p * p + 4 * p + 7) / 8, n_leaves);
  k1_leaf_operator_kernel<<<grid, 256, 0, st>>>(p, Ds, D2, k2, b, A, Dn);
}

void launch_gather_operator(const LeafDims& d, bool solve, const double* A, const double* Dn, const double* f,
                            const double* v, double* ws, double* norms, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  dim3 grid((d.Rpad + 7) / 8, n_leaves);
  k1_gather_operator_kernel<<<grid, 256, 0, st>>>(d, solve ? 1 : 0, A, Dn, f, v, ws);
  k1_operator_norm_kernel<<<n_leaves, 256, 0, st>>>(d, A, norms);
}

}  // namespace hpsg
