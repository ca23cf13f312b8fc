// C++ API test (include/hps/leaf_gpu.hpp) — the reference-facing SPEC-shaped interface.
// Run on a GPU by tests/test_gpu_cxx_api.py.  Exit code 0 = all checks passed.
//   1. analytic Helmholtz: batched_condense -> assemble_reduced ->
//      dense solve (test-only) -> reconstruct_full_solution matches J0 to 1e-6.
//   2. ParameterError for p < 4 and a mismatched f (programming guard).
//   3. ResonanceError carries the smallest failing element id (errors.hpp:18-26).
#include <cmath>
#include <cstdio>
#include <vector>

#include "hps/leaf_gpu.hpp"

static std::vector<double> dense_solve(int n, const hps::ReducedSystem& r) {
  std::vector<double> A(size_t(n) * n, 0.0), x(r.rhs);
  for (int i = 0; i < n; ++i)
    for (int64_t k = r.row_ptr[i]; k < r.row_ptr[i + 1]; ++k) A[size_t(i) * n + r.col_idx[k]] = r.values[k];
  for (int c = 0; c < n; ++c) {
    int pv = c;
    for (int i = c + 1; i < n; ++i)
      if (std::fabs(A[size_t(i) * n + c]) > std::fabs(A[size_t(pv) * n + c])) pv = i;
    for (int j = 0; j < n; ++j) std::swap(A[size_t(c) * n + j], A[size_t(pv) * n + j]);
    std::swap(x[c], x[pv]);
    for (int i = c + 1; i < n; ++i) {
      const double l = A[size_t(i) * n + c] / A[size_t(c) * n + c];
      for (int j = c; j < n; ++j) A[size_t(i) * n + j] -= l * A[size_t(c) * n + j];
      x[i] -= l * x[c];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < n; ++j) s -= A[size_t(i) * n + j] * x[j];
    x[i] = s / A[size_t(i) * n + i];
  }
  return x;
}

int main() {
  int fails = 0;
  const double kappa = 2.0 * M_PI * 2.0;
  auto ut = [kappa](double x, double y) { return std::cyl_bessel_j(0.0, kappa * std::hypot(x + 0.1, y - 0.5)); };
  hps::MeshParams mp;
  mp.nx = mp.ny = 4;
  mp.p = 14;
  const auto topo = hps::build_mesh(mp);
  hps::ProblemSpec spec;
  spec.kappa = kappa;
  spec.b_field = [](double, double) { return 1.0; };
  spec.dirichlet_g = ut;
  {
    hps::b200::LeafStage stage(topo, spec);
    const auto leaves = stage.batched_condense();
    const auto red = stage.assemble_reduced(leaves);
    {  // BSR view (SPEC.md:331 blocks): every block entry equals its CSR entry bit for bit
      const auto blk = stage.assemble_reduced_blocks(leaves);
      const int64_t q = blk.block_size;
      int64_t bad = (q != mp.p - 2) || (blk.rhs != red.rhs) ? 1 : 0;
      for (int64_t br = 0; br + 1 < int64_t(blk.brow_ptr.size()); ++br)
        for (int64_t b = blk.brow_ptr[br]; b < blk.brow_ptr[br + 1]; ++b)
          for (int64_t k = 0; k < q; ++k) {
            const int64_t row = br * q + k, rank = b - blk.brow_ptr[br];
            const int64_t rowlen = (blk.brow_ptr[br + 1] - blk.brow_ptr[br]) * q;
            for (int64_t kk = 0; kk < q; ++kk) {
              const int64_t c = red.row_ptr[row] + rank * q + kk;
              bad += red.col_idx[c] != blk.bcol_idx[b] * q + kk;
              bad += red.values[c] != blk.blocks[(b * q + k) * q + kk];
            }
            bad += red.row_ptr[row + 1] - red.row_ptr[row] != rowlen;
          }
      std::printf("BSR view: %zu blocks, mismatches %lld\n", blk.bcol_idx.size(), (long long)bad);
      if (bad) { std::printf("FAIL BSR view\n"); ++fails; }
    }
    const auto ua = dense_solve(int(red.n_active), red);
    const auto u = stage.reconstruct_full_solution(ua);
    const int64_t Nx = mp.nx * (mp.p - 1) + 1;
    double num = 0, den = 0, cmax = 0;
    std::vector<double> xs, ys;
    for (int e = 0; e < mp.nx * mp.ny; ++e) {
      topo.element_coords(e, xs, ys);
      const auto gid = topo.element_node_index(e);
      for (size_t l = 0; l < gid.size(); ++l) {
        const double d = u[gid[l]] - ut(xs[l], ys[l]);
        num += d * d;
        den += ut(xs[l], ys[l]) * ut(xs[l], ys[l]);
        const int64_t gx = gid[l] % Nx, gy = gid[l] / Nx;
        if (gx % (mp.p - 1) == 0 && gy % (mp.p - 1) == 0) cmax = std::max(cmax, std::fabs(d));
      }
    }
    const double rel = std::sqrt(num / den);
    std::printf("analytic J0 p=%d 4x4: relerr_true %.3e, max corner error %.3e\n", mp.p, rel, cmax);
    if (!(rel <= 1e-6)) { std::printf("FAIL relerr_true\n"); ++fails; }
    if (!(cmax <= 1e-5)) { std::printf("FAIL corner recovery\n"); ++fails; }
    const double rres = stage.relerr_res(u);   // Eq. 7, matrix-free on the GPU (K6)
    std::printf("relerr_res %.3e\n", rres);
    if (!(rres <= 1e-9)) { std::printf("FAIL relerr_res\n"); ++fails; }
    try {
      stage.batched_condense(std::vector<double>(5, 0.0));
      std::printf("FAIL no ParameterError for bad f\n");
      ++fails;
    } catch (const hps::ParameterError&) {
    }
    const int32_t inj[2] = {11, 6};
    hps_gpu_set_fault_injection(stage.raw(), inj, 2);
    try {
      stage.batched_condense();
      std::printf("FAIL no ResonanceError\n");
      ++fails;
    } catch (const hps::ResonanceError& e) {
      if (e.element_id() != 6) { std::printf("FAIL element_id %d\n", e.element_id()); ++fails; }
    }
  }
  try {
    hps::MeshParams bad = mp;
    bad.p = 3;
    hps::build_mesh(bad);
    std::printf("FAIL no ParameterError for p=3\n");
    ++fails;
  } catch (const hps::ParameterError&) {
  }
  std::printf(fails ? "FAILED %d\n" : "cxx api ok\n", fails);
  return fails ? 1 : 0;
}
