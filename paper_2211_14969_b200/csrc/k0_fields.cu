// ============================================================================
//  K0 — device-side sampling of the coefficient field b(x) at every leaf's p*p
//  Chebyshev nodes (removes the H2D of the b samples).
//
//  Node coordinates follow problems.leaf_coords / SPEC.md:115-118 (local order
//  l = iy*p + ix, element e = ey*nx + ex):  x = ex*a + (xh[ix]+1)*(a/2), the
//  offsets (xh+1)*(a/2) computed once on the host with the same operations.
//  crystal_field:
//      b = clamp(1 - sum_i depth * exp(-((x-cx_i)^2 + (y-cy_i)^2) / sigma^2), 0, 1)
//  summed over the 36 centres in the host order, each term with the same IEEE
//  operation sequence as the numpy restatement (explicit _rn, no contraction); only
//  exp() may differ from the host libm in the last ulp.
//  HBM-write bound (8 p^2 bytes per leaf); one thread per node.
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

__global__ void __launch_bounds__(256) k0_crystal_kernel(int p, int nx, double a, const double* __restrict__ off,
                                                         const double* __restrict__ centres, int ncent,
                                                         double inv_s2, double depth, int e0, long long total,
                                                         double* __restrict__ b) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int pp = p * p;
  const int e = e0 + static_cast<int>(t / pp), l = static_cast<int>(t % pp);
  const int iy = l / p, ix = l - iy * p;
  const double ex = static_cast<double>(e % nx), ey = static_cast<double>(e / nx);
  const double x = __dadd_rn(__dmul_rn(ex, a), __ldg(off + ix));
  const double y = __dadd_rn(__dmul_rn(ey, a), __ldg(off + iy));
  double s = 0.0;
  for (int i = 0; i < ncent; ++i) {
    const double dx = __dsub_rn(x, __ldg(centres + 2 * i)), dy = __dsub_rn(y, __ldg(centres + 2 * i + 1));
    const double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
    s = __dadd_rn(s, __dmul_rn(depth, exp(__dmul_rn(-r2, inv_s2))));
  }
  const double v = __dsub_rn(1.0, s);
  b[t] = fmin(fmax(v, 0.0), 1.0);
}

void launch_crystal(int p, int nx, double a, const double* off, const double* centres, int ncent,
                    double inv_s2, double depth, int e0, int n, double* b, cudaStream_t st) {
  const long long total = (long long)n * p * p;
  if (total <= 0) return;
  const int blocks = static_cast<int>((total + 255) / 256);
  k0_crystal_kernel<<<blocks, 256, 0, st>>>(p, nx, a, off, centres, ncent, inv_s2, depth, e0, total, b);
}

}  // namespace hpsg
