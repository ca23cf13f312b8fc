// ============================================================================
//  hps_api.cpp — SPEC-shaped C++ API (include/hps/leaf_gpu.hpp) over the C-ABI.
//  Host work here is sampling, index maps and
//  placement; every leaf operation runs through hps_gpu_* on the B200.
// ============================================================================
#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>

#include "hps/leaf_gpu.hpp"

namespace hps {

namespace {

std::vector<double> cheb_nodes(int p) {
  std::vector<double> x(p);
  for (int k = 0; k < p; ++k) x[k] = std::sin(M_PI * double(2 * k - (p - 1)) / (2.0 * double(p - 1)));
  return x;
}

// Element-parallel loop with the reference's contract (parallel.hpp:25-58):
// each index on exactly one worker, outputs per index.
template <class Fn>
void for_elements(int n, int workers, Fn&& fn) {
  if (workers <= 0) workers = std::max(1u, std::thread::hardware_concurrency());
  workers = std::min(workers, std::max(n, 1));
  if (workers <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  auto body = [&] {
    for (int i; (i = next.fetch_add(1)) < n;) fn(i);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < workers; ++t) th.emplace_back(body);
  body();
  for (auto& t : th) t.join();
}

void throw_rc(int rc, hps_gpu_ctx* ctx) {
  if (rc == HPS_OK) return;
  const std::string msg = hps_gpu_last_error(ctx);
  if (rc == HPS_ERR_PARAM) throw ParameterError(msg);
  if (rc == HPS_ERR_RESONANCE) {
    // message: "ResonanceError: element <id>: ..."
    int id = -1;
    const auto pos = msg.find("element ");
    if (pos != std::string::npos) id = std::atoi(msg.c_str() + pos + 8);
    throw ResonanceError(id, msg);
  }
  throw std::runtime_error(msg);
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

namespace b200 {

LeafStage::LeafStage(const MeshTopology& topo, const ProblemSpec& spec, LeafStageConfig cfg)
    : topo_(topo), spec_(spec), cfg_(cfg) {
  hps_leaf_desc d{};
  d.p = topo.params.p;
  d.nx = topo.params.nx;
  d.ny = topo.params.ny;
  d.storage = int32_t(cfg.storage);
  d.a = topo.params.a();
  d.kappa = spec.kappa;
  d.workspace_bytes = cfg.workspace_bytes;
  const int rc = hps_gpu_create(cfg.device, &d, &ctx_);
  if (rc != HPS_OK) {
    const std::string m = hps_gpu_last_error(nullptr);
    if (rc == HPS_ERR_PARAM) throw ParameterError(m);
    throw std::runtime_error(m);
  }
}

LeafStage::~LeafStage() { hps_gpu_destroy(ctx_); }

void LeafStage::sample(int e0, int n, const std::vector<double>& f_full, std::vector<double>& b,
                       std::vector<double>& f) const {
  const int p = topo_.params.p;
  const size_t pp = size_t(p) * p;
  if (!f_full.empty() && int64_t(f_full.size()) != topo_.N)
    throw ParameterError("f must have N = " + std::to_string(topo_.N) + " values");
  b.resize(size_t(n) * pp);
  f.resize(size_t(n) * pp);
  for_elements(n, cfg_.workers, [&](int i) {
    std::vector<double> x, y;
    topo_.element_coords(e0 + i, x, y);
    std::vector<int64_t> gid;
    if (!f_full.empty()) gid = topo_.element_node_index(e0 + i);
    for (size_t l = 0; l < pp; ++l) {
      b[i * pp + l] = spec_.b_field(x[l], y[l]);
      f[i * pp + l] = f_full.empty() ? spec_.body_load_f(x[l], y[l]) : f_full[gid[l]];
    }
  });
}

std::vector<CondensedLeaf> LeafStage::batched_condense(const std::vector<double>& f_full) {
  const int n = topo_.params.nx * topo_.params.ny;
  const int nb = 4 * (topo_.params.p - 1);
  std::vector<double> b, f;
  sample(0, n, f_full, b, f);
  double* T = static_cast<double*>(hps_host_alloc(sizeof(double) * size_t(n) * nb * nb));
  double* w = static_cast<double*>(hps_host_alloc(sizeof(double) * size_t(n) * nb));
  const int ni = (topo_.params.p - 2) * (topo_.params.p - 2);
  std::vector<double> S(cfg_.want_s_solve ? size_t(n) * ni * nb : 0);
  std::vector<int32_t> st(n);
  const int rc = hps_gpu_condense(ctx_, 0, n, b.data(), f.data(), T, w,
                                  cfg_.want_s_solve ? S.data() : nullptr, st.data());
  std::vector<CondensedLeaf> out;
  if (rc == HPS_OK) {
    out.resize(n);
    for (int e = 0; e < n; ++e) {
      out[e].element_id = e;
      out[e].n_b = nb;
      out[e].T_flux.assign(T + size_t(e) * nb * nb, T + size_t(e + 1) * nb * nb);
      out[e].w_equiv.assign(w + size_t(e) * nb, w + size_t(e + 1) * nb);
      if (cfg_.want_s_solve)
        out[e].S_solve.assign(S.begin() + size_t(e) * ni * nb, S.begin() + size_t(e + 1) * ni * nb);
    }
  }
  hps_host_free(T);
  hps_host_free(w);
  throw_rc(rc, ctx_);
  return out;
}

static std::vector<double> boundary_samples(const MeshTopology& t, const ProblemSpec& s) {
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
static void gather_leaves(const MeshTopology& topo, const std::vector<CondensedLeaf>& leaves,
                          std::vector<double>& T, std::vector<double>& w) {
  const int n = topo.params.nx * topo.params.ny;
  const int nb = 4 * (topo.params.p - 1);
  if (int(leaves.size()) != n) throw ParameterError("assemble_reduced: one condensed leaf per element");
  T.resize(size_t(n) * nb * nb);
  w.resize(size_t(n) * nb);
  for (int e = 0; e < n; ++e) {
    if (leaves[e].element_id != e || int(leaves[e].T_flux.size()) != nb * nb)
      throw ParameterError("assemble_reduced: inconsistent leaf ordering");
    std::copy(leaves[e].T_flux.begin(), leaves[e].T_flux.end(), T.begin() + size_t(e) * nb * nb);
    std::copy(leaves[e].w_equiv.begin(), leaves[e].w_equiv.end(), w.begin() + size_t(e) * nb);
  }
}

ReducedSystem LeafStage::assemble_reduced(const std::vector<CondensedLeaf>& leaves) {
  std::vector<double> T, w;
  gather_leaves(topo_, leaves, T, w);
  ReducedSystem r;
  r.n_active = topo_.n_active;
  int64_t nnz = 0;
  throw_rc(hps_gpu_reduced_pattern(ctx_, &nnz, nullptr, nullptr), ctx_);
  r.row_ptr.resize(size_t(r.n_active) + 1);
  r.col_idx.resize(size_t(nnz));
  r.values.resize(size_t(nnz));
  r.rhs.resize(size_t(r.n_active));
  throw_rc(hps_gpu_reduced_pattern(ctx_, &nnz, r.row_ptr.data(), r.col_idx.data()), ctx_);
  const auto g = boundary_samples(topo_, spec_);
  throw_rc(hps_gpu_assemble_reduced(ctx_, T.data(), w.data(), g.data(), r.values.data(), r.rhs.data()),
           ctx_);
  return r;
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
  throw_rc(hps_gpu_reduced_bsr_pattern(ctx_, &r.block_size, &nnzb, r.brow_ptr.data(), r.bcol_idx.data()),
           ctx_);
  const auto g = boundary_samples(topo_, spec_);
  throw_rc(hps_gpu_assemble_reduced_bsr(ctx_, T.data(), w.data(), g.data(), r.blocks.data(), r.rhs.data()),
           ctx_);
  return r;
}

std::vector<double> LeafStage::leaf_solve(int e0, int n, const std::vector<double>& v,
                                          const std::vector<double>& f_full) {
  const int p = topo_.params.p, nb = 4 * (p - 1);
  if (int64_t(v.size()) != int64_t(n) * nb) throw ParameterError("leaf_solve: v needs n_b values per leaf");
  std::vector<double> b, f;
  sample(e0, n, f_full, b, f);
  std::vector<double> u(size_t(n) * p * p);
  std::vector<int32_t> st(n);
  throw_rc(hps_gpu_leaf_solve(ctx_, e0, e0 + n, b.data(), f.data(), v.data(), u.data(), st.data()), ctx_);
  return u;
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
  const int p = topo_.params.p, nx = topo_.params.nx, ny = topo_.params.ny, nb = 4 * (p - 1);
  const int n = nx * ny;
  if (int64_t(u_active.size()) != topo_.n_active) throw ParameterError("reduced solution size");
  const int64_t Nx = int64_t(nx) * (p - 1) + 1, Ny = int64_t(ny) * (p - 1) + 1;
  const auto g = boundary_samples(topo_, spec_);
  auto gval = [&](int64_t gx, int64_t gy) {
    if (gy == 0) return g[gx];
    if (gy == Ny - 1) return g[Nx + gx];
    if (gx == 0) return g[2 * Nx + gy];
    return g[2 * Nx + Ny + gy];
  };
  // boundary vectors per leaf (corners of interior edges do not enter: exact zero columns)
  std::vector<double> v(size_t(n) * nb, 0.0);
  for_elements(n, cfg_.workers, [&](int e) {
    const auto gid = topo_.element_node_index(e);
    for (int k = 0; k < nb; ++k) {
      int iy, ix;
      if (k < p) { iy = 0; ix = k; }
      else if (k < 2 * p - 1) { iy = k - p + 1; ix = p - 1; }
      else if (k < 3 * p - 2) { iy = p - 1; ix = k - 2 * p + 1; }
      else { iy = k - 3 * p + 3; ix = 0; }
      const int64_t gg = gid[iy * p + ix];
      const int64_t act = topo_.active_of_global(gg);
      const int64_t gx = gg % Nx, gy = gg / Nx;
      if (act >= 0) v[size_t(e) * nb + k] = u_active[act];
      else if (gx == 0 || gy == 0 || gx == Nx - 1 || gy == Ny - 1) v[size_t(e) * nb + k] = gval(gx, gy);
    }
  });
  const auto ul = leaf_solve(0, n, v, f_full);
  std::vector<double> u(size_t(topo_.N), 0.0);
  for (int e = 0; e < n; ++e) {
    const auto gid = topo_.element_node_index(e);
    for (int l = 0; l < p * p; ++l) u[gid[l]] = ul[size_t(e) * p * p + l];
  }
  // Interior corners: average of the degree-(p-3) interpolants of the
  // adjacent interface edges (through their p-2 active nodes) evaluated at the corner.
  const auto xh = cheb_nodes(p);
  std::vector<double> wts(p - 2);
  for (int j = 1; j <= p - 2; ++j) {
    double prod = 1.0;
    for (int k = 1; k <= p - 2; ++k)
      if (k != j) prod *= (xh[j] - xh[k]);
    wts[j - 1] = 1.0 / prod;
  }
  auto edge_extrap = [&](const double* vals, double t) {  // barycentric (2nd form) at t
    double num = 0.0, den = 0.0;
    for (int j = 0; j < p - 2; ++j) {
      const double c = wts[j] / (t - xh[j + 1]);
      num += c * vals[j];
      den += c;
    }
    return num / den;
  };
  std::vector<double> vals(p - 2);
  for (int cy = 1; cy < ny; ++cy)
    for (int cx = 1; cx < nx; ++cx) {
      const int64_t gx = int64_t(cx) * (p - 1), gy = int64_t(cy) * (p - 1);
      double s = 0.0;
      int cnt = 0;
      for (int dir = 0; dir < 4; ++dir) {  // left, right (horizontal line), down, up (vertical)
        for (int j = 1; j <= p - 2; ++j) {
          int64_t x = gx, y = gy;
          if (dir == 0) x = gx - (p - 1) + j;
          if (dir == 1) x = gx + j;
          if (dir == 2) y = gy - (p - 1) + j;
          if (dir == 3) y = gy + j;
          vals[j - 1] = u_active[topo_.active_of_global(y * Nx + x)];
        }
        s += edge_extrap(vals.data(), (dir == 0 || dir == 2) ? 1.0 : -1.0);
        ++cnt;
      }
      u[gy * Nx + gx] = s / cnt;
    }
  // Element corners on Gamma take the Dirichlet data.
  for (int64_t gx = 0; gx < Nx; gx += p - 1) {
    u[gx] = gval(gx, 0);
    u[(Ny - 1) * Nx + gx] = gval(gx, Ny - 1);
  }
  for (int64_t gy = 0; gy < Ny; gy += p - 1) {
    u[gy * Nx] = gval(0, gy);
    u[gy * Nx + Nx - 1] = gval(Nx - 1, gy);
  }
  return u;
}

}  // namespace b200
}  // namespace hps
