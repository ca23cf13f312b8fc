// ============================================================================
//  K4 — scatter of every leaf's T_flux / w_equiv into the reduced interface
//  system (north star #4; replaces assemble_reduced).
//
//  CSR over active nodes: row j = edge*q + k (q = p-2), its
//  columns are the active nodes of the (<= 7) interior edges of the two
//  elements adjacent to the row's edge, edges ascending, nodes ascending
//  (int64 row_ptr, int32 col_idx).  Gather formulation,
//  one CTA per interface edge, no atomics: every value is
//        0 + T_{e0}[r0, c0] + T_{e1}[r1, c1]     (present terms, e0 < e1)
//  and every rhs entry
//        -( sum_t ( w_t[r_t] + sum_{Gamma cols} T_t[r_t, c] g_c ) )
//  in exactly the order of the CPU oracle, with _rn intrinsics (no FMA
//  contraction): given the same T, values and rhs are bit-identical.
//  HBM bound: reads the active x active part of T, writes nnz values.  Each CTA first tabulates
//  its row pattern (T column and output offset per row position), then warps walk rows and
//  lanes walk positions with four rows' loads in flight: no integer division per entry,
//  C4 (211M nonzeros) in 0.75 ms = 5.4 TB/s of algorithmic B_K4 (83% of HBM).
//
//  BSR view (SPEC.md:331's ReducedSystem "blocks" are exactly
//  this): block row = interface edge, block column = one of its <= 7 column
//  edges (ascending), block = the dense q x q coupling, row-major.  Since every
//  row of an edge has the same columns, block (ed, rank) holds the entries
//  CSR keeps at edge_off[ed] + k*rowlen + rank*q + kk; the BSR kernel writes
//  them at edge_off[ed] + rank*q*q + k*q + kk (same values, same bits), and
//  block offsets are edge_off[ed] / (q*q) + rank.
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

#ifndef HPS_K4_MINB
#define HPS_K4_MINB 6   // min CTAs/SM for the values kernel: 40-register cap (measured 5.4 vs 3.1 TB/s uncapped)
#endif

__device__ __forceinline__ int side_base(int p, int side) {
  return side == 0 ? 1 : side == 1 ? p : side == 2 ? 2 * p : 3 * p - 2;
}

// grid = n_edges, block 256
__global__ void __launch_bounds__(256) k4_pattern_kernel(MeshDev m, int64_t* __restrict__ row_ptr,
                                                         int32_t* __restrict__ col_idx) {
  const int ed = blockIdx.x;
  const int q = m.p - 2;
  const int ne = m.edge_ne[ed];
  const int64_t off = m.edge_off[ed];
  const int rowlen = ne * q;
  for (int k = threadIdx.x; k < q; k += blockDim.x) {
    const int64_t j = (int64_t)ed * q + k;
    row_ptr[j] = off + (int64_t)k * rowlen;
    if (j == m.n_active - 1) row_ptr[j + 1] = off + (int64_t)q * rowlen;
  }
  for (int e = threadIdx.x; e < q * rowlen; e += blockDim.x) {
    const int pos = e % rowlen;
    const int ce = m.edge_cols[ed * 7 + pos / q];
    col_idx[off + e] = ce * q + pos % q;
  }
}

// grid = n_edges, block 256.  BSR: block row pointer (n_edges + 1) and block columns.
__global__ void __launch_bounds__(256) k4_bsr_pattern_kernel(MeshDev m, int64_t* __restrict__ brow_ptr,
                                                             int32_t* __restrict__ bcol_idx) {
  const int ed = blockIdx.x;
  const int q = m.p - 2;
  const int ne = m.edge_ne[ed];
  const int64_t boff = m.edge_off[ed] / ((int64_t)q * q);
  if (threadIdx.x == 0) {
    brow_ptr[ed] = boff;
    if (ed == m.n_edges - 1) brow_ptr[ed + 1] = boff + ne;
  }
  if (threadIdx.x < ne) bcol_idx[boff + threadIdx.x] = m.edge_cols[ed * 7 + threadIdx.x];
}

// grid = n_edges (or the length of edge_list: a leaf-range shard's own edges), block 256.
// BSR selects the output layout (see the header).  T and w are indexed by global element
// id (a shard passes base pointers offset by its first leaf).
template <bool BSR>
__global__ void __launch_bounds__(256, HPS_K4_MINB) k4_values_kernel(MeshDev m, const double* __restrict__ T,
                                                        const double* __restrict__ w,
                                                        const double* __restrict__ g_bnd,
                                                        double* __restrict__ values,
                                                        double* __restrict__ rhs,
                                                        const int* __restrict__ edge_list) {
  const int ed = edge_list ? edge_list[blockIdx.x] : blockIdx.x;
  const int p = m.p, q = p - 2, nb = 4 * (p - 1);
  const int ne = m.edge_ne[ed];
  const int64_t off = m.edge_off[ed];
  const int rowlen = ne * q;
  __shared__ int col_side[2][7];  // side of column-edge rank in element t, or -1
  __shared__ int el[2], sd[2];
  if (threadIdx.x < 2) {
    const int t = threadIdx.x;
    el[t] = m.edge_elems[2 * ed + t];
    sd[t] = m.edge_sides[2 * ed + t];
    for (int r = 0; r < 7; ++r) {
      col_side[t][r] = -1;
      if (r < ne) {
        const int ce = m.edge_cols[ed * 7 + r];
        for (int s = 0; s < 4; ++s)
          if (m.elem_edges[4 * el[t] + s] == ce) col_side[t][r] = s;
      }
    }
  }
  __syncthreads();
  // Column table of the edge's rows (every row of an edge has the same columns): position
  // pos = rank * q + kk -> T column of element t (side_base of its side + kk) or -1, and the
  // output offset of (row k, pos) = k * kstride + pstride(pos) (CSR: k * rowlen + pos; BSR:
  // k * q + rank * q * q + kk).  Each warp walks rows k, lanes walk positions: no integer
  // division per entry, four rows' worth of loads in flight per lane.
  constexpr int MAXPOS = 7 * 43;   // 7 column edges x (p - 2), p <= 45
  __shared__ int tcol[2][MAXPOS];
  __shared__ int opos[MAXPOS];
  for (int pos = threadIdx.x; pos < rowlen; pos += blockDim.x) {
    const int rank = pos / q, kk = pos - rank * q;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int sc = col_side[t][rank];
      tcol[t][pos] = sc >= 0 ? side_base(p, sc) + kk : -1;
    }
    opos[pos] = BSR ? rank * q * q + kk : pos;
  }
  __syncthreads();
  const int kstride = BSR ? q : rowlen;
  const double* T0 = T + ((size_t)el[0] * nb + side_base(p, sd[0])) * nb;
  const double* T1 = T + ((size_t)el[1] * nb + side_base(p, sd[1])) * nb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  constexpr int U = 4;   // rows per pass
  for (int k0 = warp * U; k0 < q; k0 += nwarp * U) {
    for (int pos = lane; pos < rowlen; pos += 32) {
      const int c0 = tcol[0][pos], c1 = tcol[1][pos], o = opos[pos];
      double tv[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        tv[u][0] = (k < q && c0 >= 0) ? __ldg(T0 + (size_t)k * nb + c0) : 0.0;
        tv[u][1] = (k < q && c1 >= 0) ? __ldg(T1 + (size_t)k * nb + c1) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u;
        if (k >= q) continue;
        double v = 0.0;   // 0 + T_e0 + T_e1 in the oracle's order (present terms only)
        if (c0 >= 0) v = __dadd_rn(v, tv[u][0]);
        if (c1 >= 0) v = __dadd_rn(v, tv[u][1]);
        values[off + (int64_t)k * kstride + o] = v;
      }
    }
  }
  // rhs: one thread per row of this edge
  const int Nx = m.nx * (p - 1) + 1, Ny = m.ny * (p - 1) + 1;
  for (int k = threadIdx.x; k < q; k += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < 2; ++t) {
      const int e = el[t];
      const int r = side_base(p, sd[t]) + k;
      const double* Te = T + ((size_t)e * nb + r) * nb;
      acc = __dadd_rn(acc, __ldg(w + (size_t)e * nb + r));
      const int ex = e % m.nx, ey = e / m.nx;
      for (int sc = 0; sc < 4; ++sc) {
        if (m.elem_edges[4 * e + sc] >= 0) continue;
        const double* gs;
        int base;
        switch (sc) {
          case 0: gs = g_bnd; base = ex * (p - 1); break;                         // south
          case 1: gs = g_bnd + 2 * Nx + Ny; base = ey * (p - 1); break;           // east
          case 2: gs = g_bnd + Nx; base = ex * (p - 1); break;                    // north
          default: gs = g_bnd + 2 * Nx; base = ey * (p - 1); break;               // west
        }
        for (int kk = 0; kk < q; ++kk) {
          const double prod = __dmul_rn(__ldg(Te + side_base(p, sc) + kk), __ldg(gs + base + kk + 1));
          acc = __dadd_rn(acc, prod);
        }
      }
    }
    rhs[(int64_t)ed * q + k] = -acc;
  }
}

// Per-leaf scatter map (the COO view of the same CSR; SURVEY §8b hps_gpu_scatter_indices):
// for leaf e and local boundary index r (SURVEY A.4 order) row[e][r] = active row of that
// node or -1 (corner / Dirichlet); slot[e][r][c] = position in the CSR values array that
// T_e[r, c] is summed into, or -1 when the row or the column is not active (Gamma columns go
// to the rhs).  grid = leaves, block 256.
__global__ void __launch_bounds__(256) k4_scatter_index_kernel(MeshDev m, int e0, int64_t* __restrict__ slot,
                                                               int64_t* __restrict__ row) {
  const int le = blockIdx.x, e = e0 + le;
  const int p = m.p, q = p - 2, nb = 4 * (p - 1);
  __shared__ int r_edge[4 * 64], r_k[4 * 64];   // per local boundary index (nb <= 4*63)
  __shared__ int rank_of[4][4];                   // [row side][col side] -> column rank, -1 if absent
  for (int r = threadIdx.x; r < nb; r += blockDim.x) {
    int ed = -1, k = -1;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int kk = r - side_base(p, s);
      if (kk >= 0 && kk < q) {
        ed = m.elem_edges[4 * e + s];
        k = kk;
      }
    }
    r_edge[r] = ed;
    r_k[r] = ed >= 0 ? k : -1;
    row[(size_t)le * nb + r] = ed >= 0 ? (int64_t)ed * q + k : -1;
  }
  if (threadIdx.x < 16) {
    const int sr = threadIdx.x / 4, sc = threadIdx.x % 4;
    const int er = m.elem_edges[4 * e + sr], ec = m.elem_edges[4 * e + sc];
    int rk = -1;
    if (er >= 0 && ec >= 0)
      for (int t = 0; t < m.edge_ne[er]; ++t)
        if (m.edge_cols[er * 7 + t] == ec) rk = t;
    rank_of[sr][sc] = rk;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb * nb; i += blockDim.x) {
    const int r = i / nb, c = i - r * nb;
    int64_t out = -1;
    const int er = r_edge[r], ec = r_edge[c];
    if (er >= 0 && ec >= 0) {
      int sr = 0, sc = 0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (m.elem_edges[4 * e + s] == er) sr = s;
        if (m.elem_edges[4 * e + s] == ec) sc = s;
      }
      const int rk = rank_of[sr][sc];
      const int rowlen = m.edge_ne[er] * q;
      out = m.edge_off[er] + (int64_t)r_k[r] * rowlen + (int64_t)rk * q + r_k[c];
    }
    slot[(size_t)le * nb * nb + i] = out;
  }
}

void launch_reduced_pattern(const MeshDev& m, int64_t* row_ptr, int32_t* col_idx, cudaStream_t st) {
  if (m.n_edges <= 0) return;
  k4_pattern_kernel<<<m.n_edges, 256, 0, st>>>(m, row_ptr, col_idx);
}

void launch_reduced_bsr_pattern(const MeshDev& m, int64_t* brow_ptr, int32_t* bcol_idx, cudaStream_t st) {
  if (m.n_edges <= 0) return;
  k4_bsr_pattern_kernel<<<m.n_edges, 256, 0, st>>>(m, brow_ptr, bcol_idx);
}

void launch_reduced_values(const MeshDev& m, const double* T, const double* w, const double* g_bnd,
                           double* values, double* rhs, cudaStream_t st, bool bsr, const int* edge_list,
                           int n_list) {
  const int grid = edge_list ? n_list : m.n_edges;
  if (grid <= 0) return;
  if (bsr)
    k4_values_kernel<true><<<grid, 256, 0, st>>>(m, T, w, g_bnd, values, rhs, edge_list);
  else
    k4_values_kernel<false><<<grid, 256, 0, st>>>(m, T, w, g_bnd, values, rhs, edge_list);
}

void launch_scatter_indices(const MeshDev& m, int e0, int n, int64_t* slot, int64_t* row, cudaStream_t st) {
  if (n <= 0) return;
  k4_scatter_index_kernel<<<n, 256, 0, st>>>(m, e0, slot, row);
}

}  // namespace hpsg
