// ============================================================================
//  hps_api.cpp — SPEC-shaped C++ API (include/hps/leaf_gpu.hpp) over the C-ABI.
//  Host work here is sampling, index maps and
//  placement; every leaf operation runs through hps_gpu_* on the B200.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <exception>
#include <list>
#include <mutex>
#include <thread>
#include <tuple>

#include "hps/leaf_gpu.hpp"

namespace hps {

namespace {

std::vector<double> cheb_nodes(int p) {
  std::vector<double> x(p);
  for (int k = 0; k < p; ++k) x[k] = std::sin(M_PI * double(2 * k - (p - 1)) / (2.0 * double(p - 1)));
  return x;
}

// Element-parallel loop with the reference's contract (parallel.hpp:25-58): dynamic
// dispatch, each index on exactly one worker (outputs per index, so results do not depend
// on the worker count), and the first exception thrown by any task is rethrown on the
// calling thread after every worker has joined (parallel.hpp:42-57).
template <class Fn>
void for_elements(int n, int workers, Fn&& fn) {
  if (n <= 0) return;
  if (workers <= 0) workers = std::max(1u, std::thread::hardware_concurrency());
  if (workers == 1 || n == 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  workers = std::min(workers, n);
  std::atomic<int> next{0};
  std::atomic<bool> failed{false};
  std::exception_ptr first;
  std::mutex mu;
  auto body = [&] {
    for (;;) {
      const int i = next.fetch_add(1, std::memory_order_relaxed);
      if (i >= n || failed.load(std::memory_order_relaxed)) return;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
        failed.store(true, std::memory_order_relaxed);
        return;
      }
    }
  };
  std::vector<std::thread> th;
  th.reserve(size_t(workers) - 1);
  for (int t = 1; t < workers; ++t) th.emplace_back(body);
  body();
  for (auto& t : th) t.join();
  if (first) std::rethrow_exception(first);
}

// Return code -> hps:: exception.  ResonanceError carries the smallest failing element id,
// taken from the per-leaf status words of the call (element e0 + i has status[i]).
void throw_rc(int rc, hps_gpu_ctx* ctx, const int32_t* status = nullptr, int e0 = 0, int n = 0) {
  if (rc == HPS_OK) return;
  const std::string msg = hps_gpu_last_error(ctx);
  if (rc == HPS_ERR_PARAM) throw ParameterError(msg);
  if (rc == HPS_ERR_RESONANCE) {
    int id = -1;
    for (int i = 0; status && i < n; ++i)
      if (status[i]) {
        id = e0 + i;
        break;
      }
    throw ResonanceError(id, msg);
  }
  throw std::runtime_error(msg);
}

// b and f samples at the p*p local nodes of elements [e0, e0 + n): b from
// spec.b_field, f from the full-grid load (N values) or spec.body_load_f when empty.
void sample_leaves(const MeshTopology& topo, const ProblemSpec& spec, int e0, int n,
                   const std::vector<double>& f_full, int workers, std::vector<double>& b,
                   std::vector<double>& f) {
  const int p = topo.params.p;
  const size_t pp = size_t(p) * p;
  if (!f_full.empty() && int64_t(f_full.size()) != topo.N)
    throw ParameterError("f must have N = " + std::to_string(topo.N) + " values");
  b.resize(size_t(n) * pp);
  f.resize(size_t(n) * pp);
  for_elements(n, workers, [&](int i) {
    std::vector<double> x, y;
    topo.element_coords(e0 + i, x, y);
    std::vector<int64_t> gid;
    if (!f_full.empty()) gid = topo.element_node_index(e0 + i);
    for (size_t l = 0; l < pp; ++l) {
      b[i * pp + l] = spec.b_field(x[l], y[l]);
      f[i * pp + l] = f_full.empty() ? spec.body_load_f(x[l], y[l]) : f_full[gid[l]];
    }
  });
}

}  // namespace

// ---------------------------------------------------------------- mesh
MeshTopology build_mesh(const MeshParams& prm) {
  if (prm.p < 4) throw ParameterError("build_mesh: p must be >= 4");
  if (prm.nx < 1 || prm.ny < 1) throw ParameterError("build_mesh: nx, ny must be >= 1");
  const double ax = prm.x_extent / prm.nx, ay = prm.y_extent / prm.ny;
  if (!(ax > 0.0) || std::fabs(ax - ay) > 1e-12 * std::max(ax, ay))
    throw ParameterError("build_mesh: elements must be square (SPEC.md:114)");
  MeshTopology t;
  t.params = prm;
  t.N = int64_t(prm.nx * (prm.p - 1) + 1) * int64_t(prm.ny * (prm.p - 1) + 1);
  t.n_active = int64_t((prm.nx - 1) * prm.ny + prm.nx * (prm.ny - 1)) * (prm.p - 2);
  return t;
}

std::vector<int64_t> MeshTopology::element_node_index(int e) const {
  const int p = params.p, ex = e % params.nx, ey = e / params.nx;
  const int64_t Nx = int64_t(params.nx) * (p - 1) + 1;
  std::vector<int64_t> g(size_t(p) * p);
  for (int iy = 0; iy < p; ++iy)
    for (int ix = 0; ix < p; ++ix)
      g[iy * p + ix] = (int64_t(ey) * (p - 1) + iy) * Nx + int64_t(ex) * (p - 1) + ix;
  return g;
}

void MeshTopology::element_coords(int e, std::vector<double>& x, std::vector<double>& y) const {
  const int p = params.p, ex = e % params.nx, ey = e / params.nx;
  const double a = params.a();
  const auto xh = cheb_nodes(p);
  x.resize(size_t(p) * p);
  y.resize(size_t(p) * p);
  for (int iy = 0; iy < p; ++iy)
    for (int ix = 0; ix < p; ++ix) {
      x[iy * p + ix] = ex * a + (xh[ix] + 1.0) * (a / 2.0);
      y[iy * p + ix] = ey * a + (xh[iy] + 1.0) * (a / 2.0);
    }
}

int64_t MeshTopology::active_of_global(int64_t g) const {
  const int p = params.p, nx = params.nx, ny = params.ny;
  const int64_t Nx = int64_t(nx) * (p - 1) + 1;
  const int64_t gx = g % Nx, gy = g / Nx, rx = gx % (p - 1), ry = gy % (p - 1);
  const int64_t cx = gx / (p - 1), cy = gy / (p - 1);
  if (rx == 0 && ry != 0 && cx >= 1 && cx <= nx - 1)
    return ((cx - 1) * (2 * ny - 1) + (ny - 1) + cy) * (p - 2) + (ry - 1);
  if (ry == 0 && rx != 0 && cy >= 1 && cy <= ny - 1)
    return (cx * (2 * ny - 1) + (cy - 1)) * (p - 2) + (rx - 1);
  return -1;
}

namespace {

hps_gpu_ctx* create_ctx(const MeshParams& mp, double kappa, int device, StoragePolicy storage,
                        int64_t workspace_bytes) {
  hps_leaf_desc d{};
  d.p = mp.p;
  d.nx = mp.nx;
  d.ny = mp.ny;
  d.storage = int32_t(storage);
  d.a = mp.a();
  d.kappa = kappa;
  d.workspace_bytes = workspace_bytes;
  hps_gpu_ctx* ctx = nullptr;
  const int rc = hps_gpu_create(device, &d, &ctx);
  if (rc != HPS_OK) {
    const std::string m = hps_gpu_last_error(nullptr);
    if (rc == HPS_ERR_PARAM) throw ParameterError(m);
    throw std::runtime_error(m);
  }
  return ctx;
}

std::vector<double> boundary_samples(const MeshTopology& t, const ProblemSpec& s) {
  const int p = t.params.p, nx = t.params.nx, ny = t.params.ny;
  const double a = t.params.a();
  const auto xh = cheb_nodes(p);
  auto axis = [&](int nel) {
    std::vector<double> c(size_t(nel) * (p - 1) + 1);
    for (size_t g = 0; g < c.size(); ++g) {
      const int e = g == 0 ? 0 : int((g - 1) / (p - 1));
      c[g] = e * a + (xh[g - size_t(e) * (p - 1)] + 1.0) * (a / 2.0);
    }
    return c;
  };
  const auto xs = axis(nx), ys = axis(ny);
  std::vector<double> g;
  for (double x : xs) g.push_back(s.dirichlet_g(x, 0.0));
  for (double x : xs) g.push_back(s.dirichlet_g(x, ny * a));
  for (double y : ys) g.push_back(s.dirichlet_g(0.0, y));
  for (double y : ys) g.push_back(s.dirichlet_g(nx * a, y));
  return g;
}

// Gathers the leaves' T and w leaf-major (SPEC.md:349's ordering guard).
void gather_leaves(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves, std::vector<double>& T,
                   std::vector<double>& w) {
  const int n = topo.params.nx * topo.params.ny;
  const int nb = 4 * (topo.params.p - 1);
  if (int(leaves.size()) != n) throw ParameterError("assemble_reduced: one condensed leaf per element");
  T.resize(size_t(n) * nb * nb);
  w.resize(size_t(n) * nb);
  for (int e = 0; e < n; ++e) {
    if (leaves[e].element_id != e || int(leaves[e].T_flux.size()) != nb * nb ||
        int(leaves[e].w_equiv.size()) != nb)
      throw ParameterError("assemble_reduced: inconsistent leaf ordering");
    std::copy(leaves[e].T_flux.begin(), leaves[e].T_flux.end(), T.begin() + size_t(e) * nb * nb);
    std::copy(leaves[e].w_equiv.begin(), leaves[e].w_equiv.end(), w.begin() + size_t(e) * nb);
  }
}

// Pinned staging of the leaf-major T/w the GPU writes (grow-only, one per thread): a fresh
// cudaHostAlloc of 2 GB at C4 costs about a second per call.
struct PinnedScratch {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedScratch() { hps_host_free(p); }
  double* get(size_t n) {
    if (n * sizeof(double) > bytes) {
      hps_host_free(p);
      p = hps_host_alloc(n * sizeof(double));
      bytes = p ? n * sizeof(double) : 0;
      if (!p) throw std::runtime_error("batched_condense: pinned host allocation failed");
    }
    return static_cast<double*>(p);
  }
};
thread_local PinnedScratch t_pinned_T, t_pinned_w;

std::vector<CondensedLeaf> condense_on(hps_gpu_ctx* ctx, const MeshTopology& topo, const ProblemSpec& spec,
                                       int workers, bool want_s, const std::vector<double>& f_full) {
  const int n = topo.params.nx * topo.params.ny;
  const int nb = 4 * (topo.params.p - 1), ni = (topo.params.p - 2) * (topo.params.p - 2);
  std::vector<double> b, f;
  sample_leaves(topo, spec, 0, n, f_full, workers, b, f);
  double* T = t_pinned_T.get(size_t(n) * nb * nb);
  double* w = t_pinned_w.get(size_t(n) * nb);
  std::vector<double> S(want_s ? size_t(n) * ni * nb : 0);
  std::vector<int32_t> st(n);
  const int rc = hps_gpu_condense(ctx, 0, n, b.data(), f.data(), T, w, want_s ? S.data() : nullptr, st.data());
  std::vector<CondensedLeaf> out;
  if (rc == HPS_OK) {
    out.resize(n);
    // one value per element, filled in parallel
    for_elements(n, workers, [&](int e) {
      out[e].element_id = e;
      out[e].n_b = nb;
      out[e].T_flux.assign(T + size_t(e) * nb * nb, T + size_t(e + 1) * nb * nb);
      out[e].w_equiv.assign(w + size_t(e) * nb, w + size_t(e + 1) * nb);
      if (want_s) out[e].S_solve.assign(S.begin() + size_t(e) * ni * nb, S.begin() + size_t(e + 1) * ni * nb);
    });
  }
  throw_rc(rc, ctx, st.data(), 0, n);
  return out;
}

ReducedSystem assemble_on(hps_gpu_ctx* ctx, const MeshTopology& topo, const ProblemSpec& spec,
                          const std::vector<CondensedLeaf>& leaves) {
  std::vector<double> T, w;
  gather_leaves(topo, leaves, T, w);
  ReducedSystem r;
  r.n_active = topo.n_active;
  int64_t nnz = 0;
  throw_rc(hps_gpu_reduced_pattern(ctx, &nnz, nullptr, nullptr), ctx);
  r.row_ptr.resize(size_t(r.n_active) + 1);
  r.col_idx.resize(size_t(nnz));
  r.values.resize(size_t(nnz));
  r.rhs.resize(size_t(r.n_active));
  throw_rc(hps_gpu_reduced_pattern(ctx, &nnz, r.row_ptr.data(), r.col_idx.data()), ctx);
  const auto g = boundary_samples(topo, spec);
  throw_rc(hps_gpu_assemble_reduced(ctx, T.data(), w.data(), g.data(), r.values.data(), r.rhs.data()), ctx);
  return r;
}

std::vector<double> leaf_solve_on(hps_gpu_ctx* ctx, const MeshTopology& topo, const ProblemSpec& spec,
                                  int workers, int e0, int n, const std::vector<double>& v,
                                  const std::vector<double>& f_full) {
  const int p = topo.params.p, nb = 4 * (p - 1);
  if (int64_t(v.size()) != int64_t(n) * nb) throw ParameterError("leaf_solve: v needs n_b values per leaf");
  std::vector<double> b, f;
  sample_leaves(topo, spec, e0, n, f_full, workers, b, f);
  std::vector<double> u(size_t(n) * p * p);
  std::vector<int32_t> st(n);
  throw_rc(hps_gpu_leaf_solve(ctx, e0, e0 + n, b.data(), f.data(), v.data(), u.data(), st.data()), ctx,
           st.data(), e0, n);
  return u;
}

// reconstruct_full_solution on the GPU (hps_gpu_reconstruct: K7 boundary
// vectors, batched leaf_solve, placement, corner policy SPEC.md:152); the host only samples
// b, f and g.
std::vector<double> reconstruct_on(hps_gpu_ctx* ctx, const MeshTopology& topo, const ProblemSpec& spec,
                                   int workers, const std::vector<double>& u_active,
                                   const std::vector<double>& f_full) {
  const int n = topo.params.nx * topo.params.ny;
  if (int64_t(u_active.size()) != topo.n_active) throw ParameterError("reduced solution size");
  std::vector<double> b, f;
  sample_leaves(topo, spec, 0, n, f_full, workers, b, f);
  const auto g = boundary_samples(topo, spec);
  std::vector<double> u(size_t(topo.N));
  std::vector<int32_t> st(n);
  throw_rc(hps_gpu_reconstruct(ctx, u_active.data(), g.data(), b.data(), f.data(), u.data(), st.data()), ctx,
           st.data(), 0, n);
  return u;
}

// ---- per-thread context cache of the free functions ----------------------------------
// One hps_gpu_ctx per (device, p, nx, ny, a, kappa, storage, budget) on each thread (the
// C-ABI's one-ctx-one-thread rule), least recently used first out beyond kMaxCtx.
thread_local LeafConfig t_cfg;
using CtxKey = std::tuple<int, int, int, int, double, double, int, int64_t>;
struct CtxEntry {
  CtxKey key;
  hps_gpu_ctx* ctx;
};
struct CtxCache {
  static constexpr size_t kMaxCtx = 4;
  std::list<CtxEntry> lru;
  ~CtxCache() {
    for (auto& e : lru) hps_gpu_destroy(e.ctx);
  }
  hps_gpu_ctx* get(const MeshParams& mp, double kappa) {
    const LeafConfig& c = t_cfg;
    const CtxKey key{c.device, mp.p, mp.nx, mp.ny, mp.a(), kappa, int(c.storage), c.workspace_bytes};
    for (auto it = lru.begin(); it != lru.end(); ++it)
      if (it->key == key) {
        lru.splice(lru.begin(), lru, it);
        return lru.front().ctx;
      }
    hps_gpu_ctx* ctx = create_ctx(mp, kappa, c.device, c.storage, c.workspace_bytes);
    lru.push_front({key, ctx});
    if (lru.size() > kMaxCtx) {
      hps_gpu_destroy(lru.back().ctx);
      lru.pop_back();
    }
    return ctx;
  }
};
thread_local CtxCache t_ctx;

hps_gpu_ctx* ctx_for(const MeshTopology& topo, double kappa) { return t_ctx.get(topo.params, kappa); }
// Operator-path entry points only use p (the operator arrives as a value).
hps_gpu_ctx* ctx_for_p(int p) {
  MeshParams mp;
  mp.p = p;
  mp.nx = mp.ny = 1;
  return t_ctx.get(mp, 0.0);
}

std::vector<int> interior_index(int p) {
  std::vector<int> it;
  for (int iy = 1; iy <= p - 2; ++iy)
    for (int ix = 1; ix <= p - 2; ++ix) it.push_back(iy * p + ix);
  return it;
}
std::vector<int> boundary_index(int p) {
  std::vector<int> bd;
  for (int ix = 0; ix <= p - 1; ++ix) bd.push_back(ix);                // S
  for (int iy = 1; iy <= p - 1; ++iy) bd.push_back(iy * p + p - 1);    // E
  for (int ix = 0; ix <= p - 2; ++ix) bd.push_back((p - 1) * p + ix);  // N
  for (int iy = 1; iy <= p - 2; ++iy) bd.push_back(iy * p);            // W
  return bd;
}

// Operator of `ops` in the C-ABI layout: A_loc (p^4) and D_normal (4 p p^2).
void check_ops(const LeafOperators& ops) {
  const int p = ops.p;
  const size_t pp = size_t(p) * p;
  if (p < 4) throw ParameterError("condense_leaf: LeafOperators.p must be >= 4");
  if (ops.A_loc.size() != pp * pp) throw ParameterError("condense_leaf: A_loc must be p^2 x p^2");
  for (const auto& d : ops.D_normal)
    if (d.size() != size_t(p) * pp) throw ParameterError("condense_leaf: D_normal[edge] must be p x p^2");
}

}  // namespace

// ---------------------------------------------------------------- SPEC free functions
void set_leaf_config(const LeafConfig& cfg) { t_cfg = cfg; }
LeafConfig leaf_config() { return t_cfg; }

LeafOperators build_leaf_operator(const MeshTopology& topo, const ProblemSpec& spec, int element_id) {
  const int p = topo.params.p, n = topo.params.nx * topo.params.ny;
  if (element_id < 0 || element_id >= n) throw ParameterError("build_leaf_operator: element does not exist");
  hps_gpu_ctx* ctx = ctx_for(topo, spec.kappa);
  std::vector<double> b, f;
  sample_leaves(topo, spec, element_id, 1, {}, 1, b, f);
  const size_t pp = size_t(p) * p;
  LeafOperators ops;
  ops.element_id = element_id;
  ops.p = p;
  ops.A_loc.resize(pp * pp);
  std::vector<double> dn(4 * size_t(p) * pp);
  throw_rc(hps_gpu_build_leaf_operator(ctx, element_id, element_id + 1, b.data(), ops.A_loc.data(), dn.data()),
           ctx);
  for (int e = 0; e < 4; ++e) ops.D_normal[e].assign(dn.begin() + e * p * pp, dn.begin() + (e + 1) * p * pp);
  ops.interior_idx = interior_index(p);
  ops.boundary_idx = boundary_index(p);
  return ops;
}

CondensedLeaf condense_leaf(const LeafOperators& ops, const std::vector<double>& f_local) {
  check_ops(ops);
  const int p = ops.p, nb = 4 * (p - 1), ni = (p - 2) * (p - 2);
  const size_t pp = size_t(p) * p;
  if (f_local.size() != pp) throw ParameterError("condense_leaf: f_local needs p^2 values");
  hps_gpu_ctx* ctx = ctx_for_p(p);
  std::vector<double> dn(4 * size_t(p) * pp);
  for (int e = 0; e < 4; ++e) std::copy(ops.D_normal[e].begin(), ops.D_normal[e].end(), dn.begin() + e * p * pp);
  CondensedLeaf c;
  c.element_id = ops.element_id;
  c.n_b = nb;
  c.T_flux.resize(size_t(nb) * nb);
  c.w_equiv.resize(nb);
  c.S_solve.resize(size_t(ni) * nb);
  int32_t st = 0;
  const int rc = hps_gpu_condense_operator(ctx, 0, 1, ops.A_loc.data(), dn.data(), f_local.data(), c.T_flux.data(),
                                           c.w_equiv.data(), c.S_solve.data(), &st);
  if (rc == HPS_ERR_RESONANCE) throw ResonanceError(ops.element_id, hps_gpu_last_error(ctx));
  throw_rc(rc, ctx);
  return c;
}

std::vector<CondensedLeaf> batched_condense(const MeshTopology& topo, const ProblemSpec& spec,
                                            const std::vector<double>& f) {
  return condense_on(ctx_for(topo, spec.kappa), topo, spec, t_cfg.workers, false, f);
}

std::vector<double> leaf_solve(const LeafOperators& ops, const CondensedLeaf& condensed,
                               const std::vector<double>& v, const std::vector<double>& f_local) {
  check_ops(ops);
  const int p = ops.p, nb = 4 * (p - 1);
  if (int(v.size()) != nb) throw ParameterError("leaf_solve: boundary values need 4(p-1) entries");
  if (f_local.size() != size_t(p) * p) throw ParameterError("leaf_solve: f_local needs p^2 values");
  if (condensed.n_b != 0 && condensed.n_b != nb) throw ParameterError("leaf_solve: condensed leaf of another p");
  hps_gpu_ctx* ctx = ctx_for_p(p);
  std::vector<double> u(size_t(p) * p);
  int32_t st = 0;
  const int rc = hps_gpu_leaf_solve_operator(ctx, 0, 1, ops.A_loc.data(), f_local.data(), v.data(), u.data(), &st);
  if (rc == HPS_ERR_RESONANCE) throw ResonanceError(ops.element_id, hps_gpu_last_error(ctx));
  throw_rc(rc, ctx);
  return u;
}

std::vector<double> leaf_solve(const LeafRecipe& recipe, const CondensedLeaf& condensed,
                               const std::vector<double>& v, const std::vector<double>& f_local) {
  const MeshTopology& topo = recipe.topo;
  const int p = topo.params.p, e = condensed.element_id;
  if (e < 0 || e >= topo.params.nx * topo.params.ny) throw ParameterError("leaf_solve: element does not exist");
  if (f_local.size() != size_t(p) * p) throw ParameterError("leaf_solve: f_local needs p^2 values");
  hps_gpu_ctx* ctx = ctx_for(topo, recipe.spec.kappa);
  std::vector<double> b, f;
  sample_leaves(topo, recipe.spec, e, 1, {}, 1, b, f);
  if (int(v.size()) != 4 * (p - 1)) throw ParameterError("leaf_solve: boundary values need 4(p-1) entries");
  std::vector<double> u(size_t(p) * p);
  int32_t st = 0;
  throw_rc(hps_gpu_leaf_solve(ctx, e, e + 1, b.data(), f_local.data(), v.data(), u.data(), &st), ctx, &st, e, 1);
  return u;
}

ReducedSystem assemble_reduced(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves,
                               const ProblemSpec& spec) {
  return assemble_on(ctx_for(topo, spec.kappa), topo, spec, leaves);
}

std::vector<double> reconstruct_full_solution(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves,
                                              const std::vector<double>& reduced_solution,
                                              const ProblemSpec& spec, const std::vector<double>& f) {
  if (int64_t(leaves.size()) != int64_t(topo.params.nx) * topo.params.ny)
    throw ParameterError("reconstruct_full_solution: one condensed leaf per element");
  return reconstruct_on(ctx_for(topo, spec.kappa), topo, spec, t_cfg.workers, reduced_solution, f);
}

// ---------------------------------------------------------------- b200::LeafStage
namespace b200 {

LeafStage::LeafStage(const MeshTopology& topo, const ProblemSpec& spec, LeafStageConfig cfg)
    : topo_(topo), spec_(spec), cfg_(cfg) {
  ctx_ = create_ctx(topo.params, spec.kappa, cfg.device, cfg.storage, cfg.workspace_bytes);
}

LeafStage::~LeafStage() { hps_gpu_destroy(ctx_); }

void LeafStage::sample(int e0, int n, const std::vector<double>& f_full, std::vector<double>& b,
                       std::vector<double>& f) const {
  sample_leaves(topo_, spec_, e0, n, f_full, cfg_.workers, b, f);
}

std::vector<CondensedLeaf> LeafStage::batched_condense(const std::vector<double>& f_full) {
  return condense_on(ctx_, topo_, spec_, cfg_.workers, cfg_.want_s_solve, f_full);
}

ReducedSystem LeafStage::assemble_reduced(const std::vector<CondensedLeaf>& leaves) {
  return assemble_on(ctx_, topo_, spec_, leaves);
}

ReducedBlocks LeafStage::assemble_reduced_blocks(const std::vector<CondensedLeaf>& leaves) {
  std::vector<double> T, w;
  gather_leaves(topo_, leaves, T, w);
  ReducedBlocks r;
  r.n_active = topo_.n_active;
  int64_t nnzb = 0;
  throw_rc(hps_gpu_reduced_bsr_pattern(ctx_, &r.block_size, &nnzb, nullptr, nullptr), ctx_);
  const int64_t q = r.block_size;
  r.brow_ptr.resize(size_t(q > 0 ? r.n_active / q : 0) + 1);
  r.bcol_idx.resize(size_t(nnzb));
  r.blocks.resize(size_t(nnzb * q * q));
  r.rhs.resize(size_t(r.n_active));
  throw_rc(hps_gpu_reduced_bsr_pattern(ctx_, &r.block_size, &nnzb, r.brow_ptr.data(), r.bcol_idx.data()), ctx_);
  const auto g = boundary_samples(topo_, spec_);
  throw_rc(hps_gpu_assemble_reduced_bsr(ctx_, T.data(), w.data(), g.data(), r.blocks.data(), r.rhs.data()), ctx_);
  return r;
}

std::vector<double> LeafStage::leaf_solve(int e0, int n, const std::vector<double>& v,
                                          const std::vector<double>& f_full) {
  return leaf_solve_on(ctx_, topo_, spec_, cfg_.workers, e0, n, v, f_full);
}

double LeafStage::relerr_res(const std::vector<double>& u_full, const std::vector<double>& f_full) {
  const int p = topo_.params.p, nx = topo_.params.nx, ny = topo_.params.ny, n = nx * ny;
  const size_t pp = size_t(p) * p;
  if (int64_t(u_full.size()) != topo_.N) throw ParameterError("relerr_res: u needs N values");
  std::vector<double> b, f;
  sample(0, n, f_full, b, f);
  std::vector<double> ul(size_t(n) * pp);
  for_elements(n, cfg_.workers, [&](int e) {
    const auto gid = topo_.element_node_index(e);
    for (size_t l = 0; l < pp; ++l) ul[size_t(e) * pp + l] = u_full[gid[l]];
  });
  double out[3] = {0.0, 0.0, 0.0};
  throw_rc(hps_gpu_residual(ctx_, b.data(), f.data(), ul.data(), out), ctx_);
  // Dirichlet rows (identity, data g) enter ||f|| once per boundary node.
  const int64_t Nx = int64_t(nx) * (p - 1) + 1, Ny = int64_t(ny) * (p - 1) + 1;
  const auto g = boundary_samples(topo_, spec_);   // [S(Nx), N(Nx), W(Ny), E(Ny)]
  double g2 = 0.0;
  for (int64_t i = 0; i < 2 * Nx; ++i) g2 += g[i] * g[i];
  for (int64_t i = 1; i < Ny - 1; ++i) g2 += g[2 * Nx + i] * g[2 * Nx + i] + g[2 * Nx + Ny + i] * g[2 * Nx + Ny + i];
  return std::sqrt((out[0] + out[1]) / (out[2] + g2));
}

std::vector<double> LeafStage::reconstruct_full_solution(const std::vector<double>& u_active,
                                                         const std::vector<double>& f_full) {
  return reconstruct_on(ctx_, topo_, spec_, cfg_.workers, u_active, f_full);
}

}  // namespace b200
}  // namespace hps
