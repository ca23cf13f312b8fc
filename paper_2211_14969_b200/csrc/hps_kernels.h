// Launch wrappers of the sm_100a kernels (internal to libhps_leaf_b200.so).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hps_device.cuh"

namespace hpsg {

// K0: crystal-field b(x) samples of leaves [e0, e0+n) (k0_fields.cu); off = (xh+1)*(a/2),
// centres = 2*ncent doubles (cx, cy), inv_s2 = 1/sigma^2.
void launch_crystal(int p, int nx, double a, const double* off, const double* centres, int ncent,
                    double inv_s2, double depth, int e0, int n, double* b, cudaStream_t st);

// K1: augmented leaf matrices + ||A_ii||_inf.
void launch_assemble(const LeafDims& d, const int* rowcode, const int* colcode, const double* Ds,
                     const double* D2, double k2, const double* b, const double* f, double* ws,
                     double* norms, const int* inject, int n_leaves, cudaStream_t st);

// K1 (leaf-solve variant): [A_ii | f_i - A_ib v] with no D rows (rows ni..Rpad zero).
void launch_assemble_solve(const LeafDims& d, const int* rowcode, const int* colcode,
                           const double* Ds, const double* D2, double k2, const double* b,
                           const double* f, const double* v, double* ws, double* norms,
                           const int* inject, int n_leaves, cudaStream_t st);

// K1op (k1_operator.cu): dense A_loc (p^2 x p^2) + D_normal (4 x p x p^2) of a batch of leaves
// from b, and the gather of a given operator into the K2 workspace (+ ||A_ii||_inf).
void launch_leaf_operator(int p, const double* Ds, const double* D2, double k2, const double* b, double* A,
                          double* Dn, int n_leaves, cudaStream_t st);
void launch_gather_operator(const LeafDims& d, bool solve, const double* A, const double* Dn, const double* f,
                            const double* v, double* ws, double* norms, int n_leaves, cudaStream_t st);

// Store-policy leaf solve: rhs into column `col` of a kept condense workspace.
void launch_write_rhs(const LeafDims& d, int col, const double* D2, const double* f,
                      const double* v, double* ws, int n_leaves, cudaStream_t st);

// K2+K3: blocked LU + triangular solves + Schur GEMM -> T, w, status.
constexpr int PHASE_SLOTS = 20;   // per-leaf profiling counters (LuArgs::phase_cycles)
struct LuArgs;
struct LuArgs {
  LeafDims d;           // geometry; R = ni and ntb = 1 for leaf solves
  double* ws;           // leaf workspaces (leaf_stride apart)
  double* linv;         // nblk * 64 * 64 per leaf
  short* perm;          // Rpad per leaf: written when factor = 1, read when factor = 0
  const double* norms;  // ||A_ii||_inf per leaf (factor = 1)
  double* T_out;        // nb*nb per leaf (D rows of the trailing columns)
  double* w_out;        // nb per leaf
  int* status;          // per leaf (factor = 1)
  double* minratio;     // per leaf, nullable
  int factor;           // 1: factor A_ii then trailing columns; 0: trailing columns only
  long long* phase_cycles = nullptr;  // optional PHASE_SLOTS counters per leaf (profiling)
  int lockstep = 0;                   // factor: lock-step multi-leaf kernel (panels aligned)
  int s_with_load = 0;                // K3: S rows hold n_b + 1 entries, the last = +A_ii^{-1} f_i
  const int* inject = nullptr;         // per leaf, nullable
  int* sched = nullptr;               // persistent K2: leaf-claim counter, zeroed before the
                                      // launch (nullptr: static leaf split)
};
// Two builds of k2_lu_schur.cu: g256 (8-warp CTAs, R <= 2048) and g128 (4-warp CTAs,
// R <= 640, more leaves per SM).  K3: S_solve = -A_ii^{-1} A_ib from a factored workspace
// (after K2); uinv_ws holds 4096 doubles per resident CTA (<= 4 per SM).
#define HPS_K2_DECL(ns)                                                                       \
  namespace ns {                                                                              \
  size_t lu_smem_bytes();                                                                     \
  int lu_ctas_per_sm(const LeafDims& d);                                                      \
  void launch_lu_schur(const LuArgs& a, int n_leaves, cudaStream_t st);                       \
  void launch_ssolve(const LuArgs& a, double* S_out, double* uinv_ws, int n_leaves,           \
                     cudaStream_t st);                                                        \
  }
HPS_K2_DECL(g256)
HPS_K2_DECL(g128)
#undef HPS_K2_DECL

// Config choice: the 4-warp build for small leaves (R <= 640, p <= 24) unless forced.
inline bool use_g128(const LeafDims& d, int force) {
  if (force == 128) return d.R <= 640;
  if (force == 256) return false;
  return d.R <= 640;
}
inline void launch_lu_schur(const LuArgs& a, int n_leaves, cudaStream_t st, int force = 0) {
  if (use_g128(a.d, force)) g128::launch_lu_schur(a, n_leaves, st);
  else g256::launch_lu_schur(a, n_leaves, st);
}
// Co-resident K2 CTAs per SM for leaves of shape d (occupancy query, not an assumption).
inline int lu_ctas_per_sm(const LeafDims& d, int force = 0) {
  return use_g128(d, force) ? g128::lu_ctas_per_sm(d) : g256::lu_ctas_per_sm(d);
}
inline void launch_ssolve(const LuArgs& a, double* S_out, double* uinv_ws, int n_leaves,
                          cudaStream_t st, int force = 0) {
  if (use_g128(a.d, force)) g128::launch_ssolve(a, S_out, uinv_ws, n_leaves, st);
  else g256::launch_ssolve(a, S_out, uinv_ws, n_leaves, st);
}

// K2s: register-resident condensation of small leaves (p <= 12), assembly fused
// (k2s_small.cu).  T, w, status, minratio (nullable), ||A_ii|| (nullable) per leaf.
struct SmallArgs {
  const double* Ds = nullptr;
  const double* D2 = nullptr;
  double k2 = 0.0;
  const double* b = nullptr;   // p*p per leaf
  const double* f = nullptr;   // p*p per leaf
  double* T_out = nullptr;
  double* w_out = nullptr;
  int* status = nullptr;
  double* minratio = nullptr;
  double* norms = nullptr;
  const int* inject = nullptr;
  long long* trace = nullptr;  // diagnostics: clock64 per step of leaf 0 (HPS_K2S_TRACE)
};
bool small_condense_supported(int p);
bool small_condense_preferred(int p);
int small_condense_warps(int p);
int small_condense_block(int p);   // pivot columns factored per warp block (BW)
void launch_small_condense(const SmallArgs& a, int p, int n_leaves, cudaStream_t st);

// K5: back substitution u_i = U^{-1} y (y = L^{-1} P rhs in column tb0) and the
// local solution vector u (p*p per leaf): interior from the solve, boundary = v.
void launch_backsolve(const LeafDims& d, const double* ws, const short* perm, const double* v,
                      double* u, int n_leaves, cudaStream_t st);

// K5s: u = [A_ii^{-1} f + S_solve v on the interior, v on the boundary] from stored
// [S_solve | A_ii^{-1} f] (n_i x (n_b + 1) per leaf).
void launch_stored_solve(int p, const double* S, const double* v, double* u, int n_leaves, cudaStream_t st);

// Mesh tables for K4 (device pointers).
struct MeshDev {
  int nx, ny, p, n_edges;
  int64_t n_active;
  const int* elem_edges;   // 4 per element (S,E,N,W), -1 on Gamma
  const int* edge_elems;   // 2 per edge, ascending element id
  const int* edge_sides;   // 2 per edge
  const int* edge_cols;    // 7 per edge: sorted column edges of the row block, -1 padded
  const int* edge_ne;      // number of column edges
  const int64_t* edge_off; // first nonzero of the edge's rows
};
void launch_reduced_pattern(const MeshDev& m, int64_t* row_ptr, int32_t* col_idx, cudaStream_t st);
// bsr: values in BSR layout (block row = interface edge, q x q row-major blocks).
// edge_list (device, n_list ids): only those edges (a leaf-range shard's own edges).
void launch_reduced_values(const MeshDev& m, const double* T, const double* w, const double* g_bnd,
                           double* values, double* rhs, cudaStream_t st, bool bsr = false,
                           const int* edge_list = nullptr, int n_list = 0);
void launch_reduced_bsr_pattern(const MeshDev& m, int64_t* brow_ptr, int32_t* bcol_idx, cudaStream_t st);
// Per-leaf scatter map for leaves [e0, e0+n): slot (n x nb x nb) into the CSR values, row (n x nb).
void launch_scatter_indices(const MeshDev& m, int e0, int n, int64_t* slot, int64_t* row, cudaStream_t st);

// K7 (k7_reconstruct.cu): reconstruct_full_solution pieces.
void launch_leaf_boundary(int p, int nx, int ny, int e0, int n, const double* ua, const double* g, double* v,
                          cudaStream_t st);
void launch_place(int p, int nx, int ny, int e0, int n, const double* ul, double* u, cudaStream_t st);
void launch_corners(int p, int nx, int ny, const double* xh, const double* wts, const double* ua, const double* g,
                    double* u, cudaStream_t st);

// FP64 tensor peak probe (k9_fp64_peak.cu): TF/s of a register-only DMMA loop on `device`;
// sustain_s <= 0: burst rate, else the rate after sustain_s seconds of continuous load.
double measure_dmma_peak_tflops(int device, double sustain_s = 0.0);

// K6: matrix-free residual of the global collocation system (k6_residual.cu): per-leaf
// [sum r_int^2, sum f_int^2] into part_leaf (2 per leaf), per-edge sum r_flux^2 into
// part_edge, outward fluxes (nb per leaf) into the flux scratch.
void launch_residual(const MeshDev& m, double k2, const double* D2, const double* Ds, const double* b,
                     const double* f, const double* u, double* flux, double* part_leaf, double* part_edge,
                     int n_leaves, cudaStream_t st);

}  // namespace hpsg
