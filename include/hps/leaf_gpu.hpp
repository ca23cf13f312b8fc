// ============================================================================
//  hps/leaf_gpu.hpp — SPEC-shaped C++ API of the B200 leaf stage (drop-in for
//  the reference's `leaf` and `assembly` operations).
//
//  Same operation names, argument meaning and error behaviour as the
//  reference specification, as free functions in namespace hps:
//    build_leaf_operator(topo, spec, e)
//    condense_leaf(ops, f_local)
//    batched_condense(topo, spec, f)
//    leaf_solve(ops-or-recipe, condensed, v, f) SPEC.md:297-305
//    assemble_reduced(topo, leaves, spec)
//    reconstruct_full_solution(topo, leaves, u, spec, f)
//  (each thread keeps one GPU context per mesh/problem shape; set_leaf_config picks the
//  device, storage policy and worker count), and as the explicit
//  one-context-per-GPU class hps::b200::LeafStage.
//  Errors: hps::ParameterError (std::invalid_argument) and
//  hps::ResonanceError(element_id) exactly as proj/include/hps/errors.hpp:10-26
//  declares them; when that header is included first its classes are used.
//  The compute path is libhps_leaf_b200.so's C-ABI (include/hps_leaf_gpu.h):
//  there is no CPU fallback — a missing GPU raises.
// ============================================================================
#pragma once
#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hps_leaf_gpu.h"

#ifndef HPS_ERRORS_HPP  // reference header proj/include/hps/errors.hpp not included
namespace hps {
class ParameterError : public std::invalid_argument {
 public:
  explicit ParameterError(const std::string& m) : std::invalid_argument(m) {}
};
class ResonanceError : public std::runtime_error {
 public:
  ResonanceError(int element_id, const std::string& m) : std::runtime_error(m), id_(element_id) {}
  int element_id() const { return id_; }

 private:
  int id_;
};
}  // namespace hps
#endif

namespace hps {

// Recompute (default) re-forms the leaf factors in leaf_solve; Store keeps them;
// SSolve keeps [S_solve | A_ii^-1 f] so leaf_solve is one GEMV per leaf.
enum class StoragePolicy {
  Recompute = HPS_STORAGE_RECOMPUTE,
  Store = HPS_STORAGE_STORE,
  SSolve = HPS_STORAGE_S_SOLVE
};

// MeshParams: unit-size square elements of side a on an
// nx x ny grid starting at the origin.
struct MeshParams {
  double x_extent = 1.0, y_extent = 1.0;
  int nx = 2, ny = 2, p = 8;
  double a() const { return x_extent / nx; }
};

// MeshTopology, the index maps the leaf stage needs.
struct MeshTopology {
  MeshParams params;
  int64_t N = 0;          // (nx(p-1)+1)(ny(p-1)+1)
  int64_t n_active = 0;   // interface nodes minus corners
  // Global ids of element e's p*p local nodes (local l = iy*p + ix).
  std::vector<int64_t> element_node_index(int e) const;
  // Physical coordinates of element e's local nodes.
  void element_coords(int e, std::vector<double>& x, std::vector<double>& y) const;
  // active index of global node g, or -1 (SPEC.md:154 ordering).
  int64_t active_of_global(int64_t g) const;
};
MeshTopology build_mesh(const MeshParams& params);

// ProblemSpec.
struct ProblemSpec {
  double kappa = 0.0;
  std::function<double(double, double)> b_field = [](double, double) { return 1.0; };
  std::function<double(double, double)> dirichlet_g = [](double, double) { return 0.0; };
  std::function<double(double, double)> body_load_f = [](double, double) { return 0.0; };
};

// CondensedLeaf.  load_map is the recompute recipe (element id).
struct CondensedLeaf {
  int element_id = -1;
  int n_b = 0;
  std::vector<double> T_flux;   // n_b x n_b row-major
  std::vector<double> w_equiv;  // n_b
  std::vector<double> S_solve;  // n_i x n_b row-major, -A_ii^{-1} A_ib (LeafStageConfig::want_s_solve)
};

// ReducedSystem in CSR over MeshTopology::active_of_global order.
struct ReducedSystem {
  int64_t n_active = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col_idx;
  std::vector<double> values;
  std::vector<double> rhs;
};

// The same system as SPEC.md:331's block structure ("(interface edge, interface edge)
// pairs sharing an element -> dense (p-2)x(p-2) coupling blocks"), in BSR: block row i =
// interface edge i, bcol_idx = column edges ascending, blocks row-major q x q.
struct ReducedBlocks {
  int64_t n_active = 0;
  int32_t block_size = 0;
  std::vector<int64_t> brow_ptr;
  std::vector<int32_t> bcol_idx;
  std::vector<double> blocks;  // nnzb * q * q
  std::vector<double> rhs;
};

// LeafOperators.
struct LeafOperators {
  int element_id = -1;
  int p = 0;
  std::vector<double> A_loc;                    // p^2 x p^2 row-major, local order l = iy*p + ix
  std::vector<int> interior_idx;                // (p-2)^2 local ids, ascending
  std::vector<int> boundary_idx;                // 4(p-1) local ids: S, E, N, W (corners on the first edge)
  std::array<std::vector<double>, 4> D_normal;  // S, E, N, W: p x p^2 row-major, edge nodes ascending
};

// Recompute recipe of a CondensedLeaf's load_map: the element is rebuilt
// from the mesh and the problem (element id = CondensedLeaf::element_id).
struct LeafRecipe {
  MeshTopology topo;
  ProblemSpec spec;
};

// Configuration of the free functions (worker count, storage policy) plus the
// GPU they run on.  Applies to the calling thread's contexts created afterwards.
struct LeafConfig {
  int device = 0;
  StoragePolicy storage = StoragePolicy::Recompute;
  int workers = 0;                     // host sampling threads (parallel.hpp semantics)
  int64_t workspace_bytes = int64_t(16) << 30;   // device budget per context
};
void set_leaf_config(const LeafConfig& cfg);
LeafConfig leaf_config();

LeafOperators build_leaf_operator(const MeshTopology& topo, const ProblemSpec& spec, int element_id);
CondensedLeaf condense_leaf(const LeafOperators& ops, const std::vector<double>& f_local);
// f: full-grid load (N values), or empty to sample spec.body_load_f.  Throws ResonanceError
// for the smallest failing element id (message lists all of them).
std::vector<CondensedLeaf> batched_condense(const MeshTopology& topo, const ProblemSpec& spec,
                                            const std::vector<double>& f = {});
std::vector<double> leaf_solve(const LeafOperators& ops, const CondensedLeaf& condensed,
                               const std::vector<double>& boundary_values, const std::vector<double>& f_local);
std::vector<double> leaf_solve(const LeafRecipe& recipe, const CondensedLeaf& condensed,
                               const std::vector<double>& boundary_values, const std::vector<double>& f_local);
ReducedSystem assemble_reduced(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves,
                               const ProblemSpec& spec);
std::vector<double> reconstruct_full_solution(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves,
                                              const std::vector<double>& reduced_solution,
                                              const ProblemSpec& spec, const std::vector<double>& f = {});

namespace b200 {

struct LeafStageConfig {
  int device = 0;
  StoragePolicy storage = StoragePolicy::Recompute;  // SPEC.md:313 default
  int64_t workspace_bytes = 0;                       // 0: 70% of free HBM
  int workers = 0;                                   // host sampling threads (parallel.hpp semantics)
  bool want_s_solve = false;                         // also return S_solve (K3 back substitution)
};

// One GPU context for one mesh/problem.  Not reentrant (one host thread per ctx).
class LeafStage {
 public:
  LeafStage(const MeshTopology& topo, const ProblemSpec& spec, LeafStageConfig cfg = {});
  ~LeafStage();
  LeafStage(const LeafStage&) = delete;
  LeafStage& operator=(const LeafStage&) = delete;

  // batched_condense(topo, spec, f): f is the full-grid load (N values) or empty
  // to sample spec.body_load_f.  Throws ResonanceError for the smallest failing id.
  std::vector<CondensedLeaf> batched_condense(const std::vector<double>& f_full = {});
  // assemble_reduced(topo, leaves, spec).
  ReducedSystem assemble_reduced(const std::vector<CondensedLeaf>& leaves);
  // assemble_reduced in the BSR block view (entries bit-identical to the CSR values).
  ReducedBlocks assemble_reduced_blocks(const std::vector<CondensedLeaf>& leaves);
  // Batched leaf_solve: boundary values v (n_b per element, SPEC boundary order)
  // for elements [e0, e0 + n) -> p*p local values each.
  std::vector<double> leaf_solve(int e0, int n, const std::vector<double>& v,
                                 const std::vector<double>& f_full = {});
  // reconstruct_full_solution: full-grid values from the reduced solution u_active
  // (interfaces), g (Dirichlet) and batched leaf solves (interiors).  Interior
  // corner nodes get the average of the adjacent edge interpolants.
  std::vector<double> reconstruct_full_solution(const std::vector<double>& u_active,
                                                const std::vector<double>& f_full = {});

  // Eq. 7 relerr_res = ||A u - f||_2 / ||f||_2 of the full collocation system
  // (SPEC.md:337-342,354-362 compute_errors) for a full-grid solution u (N values, e.g.
  // reconstruct_full_solution's output), evaluated matrix-free on the GPU (K6).
  double relerr_res(const std::vector<double>& u_full, const std::vector<double>& f_full = {});

  hps_gpu_ctx* raw() { return ctx_; }
  const MeshTopology& topology() const { return topo_; }

 private:
  void sample(int e0, int n, const std::vector<double>& f_full, std::vector<double>& b,
              std::vector<double>& f) const;
  MeshTopology topo_;
  ProblemSpec spec_;
  LeafStageConfig cfg_;
  hps_gpu_ctx* ctx_ = nullptr;
};

}  // namespace b200
}  // namespace hps
