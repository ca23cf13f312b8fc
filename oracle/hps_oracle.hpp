// ============================================================================
//  hps_oracle.hpp — CPU restatement of the reference's HPS leaf stage.
//
//  TEST INFRASTRUCTURE ONLY.  This is the parity oracle: only tests/,
//  __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
//  may load it, and only as the checker or the timed CPU baseline.  The
//  product (paper_2211_14969_b200/) never links or calls it.
//
//  The reference (/root/reference) is a specification plus two
//  headers (proj/include/hps/{errors,parallel}.hpp); it has no implementation
//  and no tests, so this file restates SPEC.md with the interpretations pinned
//  in SURVEY.md Appendix A.  Dense LU/solve/GEMM come from the OpenBLAS that
//  ships inside the scipy wheel (scipy_dgetrf_/dgetrs_/dgemm_), the stand-in
//  for the reference's Eigen3 3.4 dependency (proj/CMakeLists.txt:13), which
//  is neither vendored nor installed.
//
//  Parity pinning: the reference ships no golden vectors.  The oracle is pinned
//  against every known-answer example in SPEC.md (tests/test_oracle_*.py) and
//  against a dense global solve (acceptance 1 :583).
// ============================================================================
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <stdexcept>

#ifdef HPSO_REFERENCE_HEADERS
#include <hps/errors.hpp>   // the reference's own taxonomy (proj/include/hps/errors.hpp)
#endif

namespace hpso {

// Error taxonomy: the reference's classes when its headers are on the include path,
// else a restatement of proj/include/hps/errors.hpp:10-26 (ParameterError is an
// invalid_argument, ResonanceError carries the element id).
#ifdef HPSO_REFERENCE_HEADERS
using ParameterError = hps::ParameterError;
using ResonanceError = hps::ResonanceError;
#else
struct ParameterError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ResonanceError : std::runtime_error {
  ResonanceError(int e, const std::string& m) : std::runtime_error(m), element_id_(e) {}
  int element_id() const { return element_id_; }

 private:
  int element_id_;
};
#endif

// ---- chebyshev --------------------------------------------
// x_k = sin(pi*(2k-(p-1)) / (2(p-1))): ascending CGL nodes, exactly antisymmetric
// (SURVEY Appendix A.1).
std::vector<double> cheb_nodes(int p, bool allow_small = false);
// D_ij = (c_i/c_j)(-1)^{i+j}/(x_i-x_j), D_ii = -sum_{j!=i} D_ij.
// Row-major p x p.
std::vector<double> cheb_diff_matrix(const std::vector<double>& x);
// (2/a) * D; rejects a <= 0.
std::vector<double> scale_to_interval(const std::vector<double>& D, double a);

// ---- leaf geometry ------------
struct LeafIndex {
  int p, n_i, n_b;
  std::vector<int> interior;   // (p-2)^2 local ids l = iy*p + ix, row-major
  std::vector<int> boundary;   // 4(p-1) local ids: S(ix 0..p-1) E(iy 1..p-1) N(ix 0..p-2) W(iy 1..p-2)
  std::vector<int> bnd_edge;   // edge owning boundary position k: 0=S 1=E 2=N 3=W
  std::vector<char> bnd_corner;// 1 if boundary position k is a leaf corner
};
LeafIndex leaf_index(int p);

// Per-(p, a, kappa) constants: scaled D and D2 = Ds*Ds (row-major).
struct LeafConstants {
  int p;
  double a, kappa;
  std::vector<double> x, Ds, D2;
  LeafIndex idx;
};
LeafConstants leaf_constants(int p, double a, double kappa);

// build_leaf_operator: dense A_loc (p^2 x p^2, row-major) and
// the boundary-ordered outward-normal rows Dn (4(p-1) x p^2, row-major).
void build_leaf_operator(const LeafConstants& c, const double* b, double* A_loc, double* Dn);

// condense_leaf via dgetrf + dgetrs + dgemm.
//   T  : n_b x n_b row-major (T_flux = D_b + D_i S_solve)
//   w  : n_b                 (w_equiv = D_i A_ii^{-1} f_i)
//   S  : n_i x n_b row-major (S_solve = -A_ii^{-1} A_ib), nullable
//   lu : n_i x n_i column-major LU factors + ipiv, nullable ("store" policy)
// Returns 0, or 1 on resonance (pivot < 1e-12 ||A_ii||_inf).
int condense_leaf(const LeafConstants& c, const double* b, const double* f, double* T, double* w,
                  double* S, double* lu, int32_t* ipiv, bool inject_singular, double* min_pivot_ratio);

// leaf_solve: p^2 local values, interior = A_ii^{-1}(f_i - A_ib v),
// boundary = v.  With lu/ipiv non-null the stored factors are used ("store"),
// otherwise A_ii is rebuilt and refactored ("recompute").
int leaf_solve(const LeafConstants& c, const double* b, const double* f, const double* v, double* u,
               const double* lu, const int32_t* ipiv, bool inject_singular);

// ---- mesh indexing (SURVEY Appendix A.6-8,13) -------------
struct MeshIndex {
  int nx, ny, p;
  int64_t N;           // (nx(p-1)+1)(ny(p-1)+1)
  int n_edges;         // interior edges
  int64_t n_active;    // n_edges * (p-2)
  // Per element: interior edge id for S,E,N,W or -1 if that side lies on Gamma.
  std::vector<int32_t> elem_edges;   // 4 * nx*ny
  // Per edge: the two adjacent elements (lower id first) and the side index of the
  // edge within each (0=S 1=E 2=N 3=W).
  std::vector<int32_t> edge_elems;   // 2 * n_edges
  std::vector<int32_t> edge_sides;   // 2 * n_edges
};
MeshIndex mesh_index(int nx, int ny, int p);
// element_node_index: p^2 global ids per element in local order.
void element_node_index(const MeshIndex& m, int e, int64_t* out);
// active_index of global node g, or -1.
int64_t active_of_global(const MeshIndex& m, int64_t g);

// ---- assemble_reduced ----------------------------
struct ReducedCSR {
  int64_t n;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
};
ReducedCSR reduced_pattern(const MeshIndex& m);
// values[nnz], rhs[n]. T (n_b^2 per leaf) and w (n_b per leaf) leaf-major.
// g_bnd = [south(Nx), north(Nx), west(Ny), east(Ny)] Dirichlet samples along the
// four sides of the unit square indexed by global gx / gy.
void assemble_reduced(const MeshIndex& m, const ReducedCSR& pat, const double* T, const double* w,
                      const double* g_bnd, double* values, double* rhs);

// Dirichlet sample for a boundary position of an element from g_bnd.
double dirichlet_value(const MeshIndex& m, int e, int side, int k_along, const double* g_bnd);

// ---- batching (proj/include/hps/parallel.hpp:25-58) ------------------------
// Dynamic-dispatch thread pool: every index runs on exactly one worker, so
// per-index outputs are bitwise-independent of the worker count; the first
// exception is rethrown after all workers join.
#ifndef HPSO_REFERENCE_HEADERS   // else hps::hardware_workers / hps::parallel_for (.inl)
int hardware_workers();
template <class Fn> void parallel_for(int n, int workers, Fn&& fn);
#endif

}  // namespace hpso

#include "hps_oracle_parallel.inl"
