// Host cost of the SPEC-shaped C++ API at a headline config: wall time of
// hps::batched_condense(topo, spec, f) -- b/f sampling through the std::function callbacks on
// all host threads, the GPU condensation, and the copy of T/w into one CondensedLeaf value per
// element (SPEC.md:262-267 value types) -- against the C-ABI device time of the same call.
//   build: make api_timing ; run: build/api_timing [p nx kappa]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "hps/leaf_gpu.hpp"

int main(int argc, char** argv) {
  hps::MeshParams mp;
  mp.p = argc > 1 ? std::atoi(argv[1]) : 42;
  mp.nx = mp.ny = argc > 2 ? std::atoi(argv[2]) : 98;
  hps::ProblemSpec spec;
  spec.kappa = argc > 3 ? std::atof(argv[3]) : 500.0;
  spec.b_field = [](double x, double y) {   // crystal field, 6x6 lattice
    double s = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        const double dx = x - (0.3 + 0.08 * i), dy = y - (0.3 + 0.08 * j);
        s += 0.9 * std::exp(-(dx * dx + dy * dy) / 4e-4);
      }
    return std::fmin(1.0, std::fmax(0.0, 1.0 - s));
  };
  const auto topo = hps::build_mesh(mp);
  using clk = std::chrono::steady_clock;
  for (int rep = 0; rep < 3; ++rep) {
    const auto t0 = clk::now();
    const auto leaves = hps::batched_condense(topo, spec);
    const double s = std::chrono::duration<double>(clk::now() - t0).count();
    std::printf("rep %d: hps::batched_condense p=%d %dx%d: %.3f s wall (%zu leaves, %.0f leaves/s)\n", rep, mp.p,
                mp.nx, mp.ny, s, leaves.size(), leaves.size() / s);
  }
  return 0;
}
