// ============================================================================
//  hps_oracle_capi.cpp — extern "C" surface of the CPU oracle for ctypes.
//  TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
//  bench.py CPU-baseline leg.  Return codes follow the product C-ABI:
//  0 ok, 1 resonance (see status[]), 2 parameter error.
// ============================================================================
#include <cstring>
#include <string>

#include "hps_oracle.hpp"

extern "C" void scipy_openblas_set_num_threads(int);

namespace {
thread_local std::string g_err;
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
struct BlasInit {
  BlasInit() { scipy_openblas_set_num_threads(1); }  // one BLAS thread per worker
} g_blas_init;
}  // namespace

#define ORACLE_TRY try {
#define ORACLE_CATCH                                               \
  }                                                                \
  catch (const hpso::ParameterError& e) { return fail(2, e.what()); } \
  catch (const std::exception& e) { return fail(3, e.what()); }

extern "C" {

const char* hpso_last_error() { return g_err.c_str(); }
// Which batching/error headers the oracle was compiled against.
const char* hpso_build_info() {
#ifdef HPSO_REFERENCE_HEADERS
  return "reference headers: proj/include/hps/parallel.hpp + errors.hpp";
#else
  return "restated parallel.hpp/errors.hpp (reference headers absent at build time)";
#endif
}
int hpso_hardware_workers() { return hpso::hardware_workers(); }

int hpso_cheb_nodes(int p, int allow_small, double* x) {
  ORACLE_TRY
  auto v = hpso::cheb_nodes(p, allow_small != 0);
  std::memcpy(x, v.data(), sizeof(double) * v.size());
  return 0;
  ORACLE_CATCH
}

int hpso_cheb_diff(int p, int allow_small, double* D) {
  ORACLE_TRY
  auto v = hpso::cheb_diff_matrix(hpso::cheb_nodes(p, allow_small != 0));
  std::memcpy(D, v.data(), sizeof(double) * v.size());
  return 0;
  ORACLE_CATCH
}

int hpso_scale_to_interval(int p, const double* D, double a, double* out) {
  ORACLE_TRY
  std::vector<double> v(D, D + size_t(p) * p);
  auto s = hpso::scale_to_interval(v, a);
  std::memcpy(out, s.data(), sizeof(double) * s.size());
  return 0;
  ORACLE_CATCH
}

int hpso_leaf_constants(int p, double a, double kappa, double* Ds, double* D2) {
  ORACLE_TRY
  auto c = hpso::leaf_constants(p, a, kappa);
  if (Ds) std::memcpy(Ds, c.Ds.data(), sizeof(double) * c.Ds.size());
  if (D2) std::memcpy(D2, c.D2.data(), sizeof(double) * c.D2.size());
  return 0;
  ORACLE_CATCH
}

int hpso_leaf_index(int p, int32_t* interior, int32_t* boundary) {
  ORACLE_TRY
  auto L = hpso::leaf_index(p);
  for (size_t i = 0; i < L.interior.size(); ++i) interior[i] = L.interior[i];
  for (size_t i = 0; i < L.boundary.size(); ++i) boundary[i] = L.boundary[i];
  return 0;
  ORACLE_CATCH
}

int hpso_build_leaf(int p, double a, double kappa, const double* b, double* A_loc, double* Dn) {
  ORACLE_TRY
  auto c = hpso::leaf_constants(p, a, kappa);
  hpso::build_leaf_operator(c, b, A_loc, Dn);
  return 0;
  ORACLE_CATCH
}

// batched_condense.  Leaf-major arrays: b, f (p^2), T (n_b^2),
// w (n_b), S (n_i*n_b, nullable), lu (n_i^2 column-major, nullable), ipiv (n_i, nullable),
// status (1 int per leaf: 0 ok / 1 resonance), min_ratio (nullable).
int hpso_batched_condense(int p, double a, double kappa, int n_leaves, const double* b,
                          const double* f, double* T, double* w, double* S, double* lu,
                          int32_t* ipiv, int32_t* status, double* min_ratio, int workers,
                          const int32_t* inject, int n_inject) {
  ORACLE_TRY
  auto c = hpso::leaf_constants(p, a, kappa);
  const size_t P = size_t(p) * p, ni = c.idx.n_i, nb = c.idx.n_b;
  std::vector<char> inj(n_leaves, 0);
  for (int t = 0; t < n_inject; ++t)
    if (inject[t] >= 0 && inject[t] < n_leaves) inj[inject[t]] = 1;
  hpso::parallel_for(n_leaves, workers, [&](int e) {
    status[e] = hpso::condense_leaf(c, b + e * P, f + e * P, T + e * nb * nb, w + e * nb,
                                    S ? S + e * ni * nb : nullptr, lu ? lu + e * ni * ni : nullptr,
                                    ipiv ? ipiv + e * ni : nullptr, inj[e] != 0,
                                    min_ratio ? min_ratio + e : nullptr);
  });
  for (int e = 0; e < n_leaves; ++e)
    if (status[e]) return fail(1, "resonance in element " + std::to_string(e));
  return 0;
  ORACLE_CATCH
}

// batched leaf_solve.  v: n_b per leaf (boundary order), u: p^2 per leaf.
int hpso_batched_leaf_solve(int p, double a, double kappa, int n_leaves, const double* b,
                            const double* f, const double* v, double* u, const double* lu,
                            const int32_t* ipiv, int32_t* status, int workers,
                            const int32_t* inject, int n_inject) {
  ORACLE_TRY
  auto c = hpso::leaf_constants(p, a, kappa);
  const size_t P = size_t(p) * p, ni = c.idx.n_i, nb = c.idx.n_b;
  std::vector<char> inj(n_leaves, 0);
  for (int t = 0; t < n_inject; ++t)
    if (inject[t] >= 0 && inject[t] < n_leaves) inj[inject[t]] = 1;
  hpso::parallel_for(n_leaves, workers, [&](int e) {
    status[e] = hpso::leaf_solve(c, b + e * P, f + e * P, v + e * nb, u + e * P,
                                 lu ? lu + e * ni * ni : nullptr, ipiv ? ipiv + e * ni : nullptr,
                                 inj[e] != 0);
  });
  for (int e = 0; e < n_leaves; ++e)
    if (status[e]) return fail(1, "resonance in element " + std::to_string(e));
  return 0;
  ORACLE_CATCH
}

int hpso_mesh_info(int nx, int ny, int p, int64_t* N, int32_t* n_edges, int64_t* n_active) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  *N = m.N;
  *n_edges = m.n_edges;
  *n_active = m.n_active;
  return 0;
  ORACLE_CATCH
}

int hpso_mesh_maps(int nx, int ny, int p, int32_t* elem_edges, int32_t* edge_elems,
                   int32_t* edge_sides) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  std::memcpy(elem_edges, m.elem_edges.data(), 4 * m.elem_edges.size());
  std::memcpy(edge_elems, m.edge_elems.data(), 4 * m.edge_elems.size());
  std::memcpy(edge_sides, m.edge_sides.data(), 4 * m.edge_sides.size());
  return 0;
  ORACLE_CATCH
}

int hpso_element_node_index(int nx, int ny, int p, int e, int64_t* out) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  if (e < 0 || e >= nx * ny) return fail(2, "element out of range");
  hpso::element_node_index(m, e, out);
  return 0;
  ORACLE_CATCH
}

int hpso_active_of_global(int nx, int ny, int p, int64_t n, const int64_t* g, int64_t* out) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  for (int64_t i = 0; i < n; ++i) out[i] = hpso::active_of_global(m, g[i]);
  return 0;
  ORACLE_CATCH
}

int hpso_reduced_nnz(int nx, int ny, int p, int64_t* nnz) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  auto r = hpso::reduced_pattern(m);
  *nnz = r.row_ptr[r.n];
  return 0;
  ORACLE_CATCH
}

int hpso_reduced_pattern(int nx, int ny, int p, int64_t* row_ptr, int32_t* col_idx) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  auto r = hpso::reduced_pattern(m);
  std::memcpy(row_ptr, r.row_ptr.data(), 8 * r.row_ptr.size());
  std::memcpy(col_idx, r.col_idx.data(), 4 * r.col_idx.size());
  return 0;
  ORACLE_CATCH
}

int hpso_assemble_reduced(int nx, int ny, int p, const double* T, const double* w,
                          const double* g_bnd, double* values, double* rhs) {
  ORACLE_TRY
  auto m = hpso::mesh_index(nx, ny, p);
  auto r = hpso::reduced_pattern(m);
  hpso::assemble_reduced(m, r, T, w, g_bnd, values, rhs);
  return 0;
  ORACLE_CATCH
}

}  // extern "C"
