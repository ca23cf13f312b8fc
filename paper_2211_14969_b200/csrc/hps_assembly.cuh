// ============================================================================
//  hps_assembly.cuh — entries of the augmented leaf operator,
//  shared by K1 (materialise in HBM) and K2 (fused first-touch assembly).
//  Same IEEE operation sequence as the CPU oracle (oracle/hps_oracle.cpp a_entry /
//  dn_entry): the entries are bit-identical to the oracle's.
// ============================================================================
#pragma once
#include "hps_device.cuh"

namespace hpsg {

// Column/row code (built on the host once per p, see hps_host.cpp):
//   bits 0..7  : jy (or iy)      bits 8..15 : jx (or ix)
//   bits 16..17: kind  0 interior node, 1 boundary node, 2 load column, 3 zero
//   bits 18..19: owning edge of a boundary node (rows only)
__device__ __forceinline__ double a_entry(int iy, int ix, int jy, int jx, int p,
                                          const double* __restrict__ D2, double k2, double bl) {
  if (jy == iy && jx == ix) {
    double v = -__ldg(D2 + iy * p + iy);
    v = __dsub_rn(v, __ldg(D2 + ix * p + ix));
    return __dsub_rn(v, __dmul_rn(k2, bl));
  }
  if (jx == ix) return -__ldg(D2 + iy * p + jy);
  if (jy == iy) return -__ldg(D2 + ix * p + jx);
  return 0.0;
}

__device__ __forceinline__ double dn_entry(int edge, int iy, int ix, int jy, int jx, int p,
                                           const double* __restrict__ Ds) {
  switch (edge) {
    case 0: return jx == ix ? -__ldg(Ds + iy * p + jy) : 0.0;   // S: -d/dy
    case 1: return jy == iy ? __ldg(Ds + ix * p + jx) : 0.0;    // E: +d/dx
    case 2: return jx == ix ? __ldg(Ds + iy * p + jy) : 0.0;    // N: +d/dy
    default: return jy == iy ? -__ldg(Ds + ix * p + jx) : 0.0;  // W: -d/dx
  }
}

__device__ __forceinline__ double aug_value(int rcode, int ccode, int p, const double* __restrict__ Ds,
                                            const double* __restrict__ D2, double k2,
                                            const double* __restrict__ bl,
                                            const double* __restrict__ fl, bool zero_aii_row) {
  const int rkind = (rcode >> 16) & 3, ckind = (ccode >> 16) & 3;
  if (rkind == 3 || ckind == 3) return 0.0;
  const int iy = rcode & 255, ix = (rcode >> 8) & 255;
  const int jy = ccode & 255, jx = (ccode >> 8) & 255;
  if (rkind == 0) {  // interior collocation row
    if (ckind == 2) return __ldg(fl + iy * p + ix);
    if (ckind == 0 && zero_aii_row) return 0.0;
    return a_entry(iy, ix, jy, jx, p, D2, k2, __ldg(bl + iy * p + ix));
  }
  if (ckind == 2) return 0.0;  // flux row, load column
  return dn_entry((rcode >> 18) & 3, iy, ix, jy, jx, p, Ds);
}

// The same row/column codes the host builds (hps_host.cpp layout_codes), computed
// arithmetically: K2's first-touch assembly avoids dependent table loads.
__device__ __forceinline__ int make_code(int y, int x, int kind, int edge) {
  return y | (x << 8) | (kind << 16) | (edge << 18);
}
__device__ __forceinline__ int row_code_of(int phys, int p, int ni, int R) {
  const int q = p - 2;
  if (phys < ni) {
    const int iy = phys / q;
    return make_code(iy + 1, phys - iy * q + 1, 0, 0);
  }
  if (phys < R) {
    int edge;
    const int l = boundary_local(phys - ni, p, &edge);
    const int iy = l / p;
    return make_code(iy, l - iy * p, 1, edge);
  }
  return 3 << 16;
}
__device__ __forceinline__ int col_code_of(int c, int p, int ni, int tb0, int nb) {
  const int q = p - 2;
  if (c < ni) {
    const int jy = c / q;
    return make_code(jy + 1, c - jy * q + 1, 0, 0);
  }
  if (c >= tb0 && c < tb0 + nb) {
    int edge;
    const int l = boundary_local(c - tb0, p, &edge);
    const int jy = l / p;
    return make_code(jy, l - jy * p, 1, 0);
  }
  if (c == tb0 + nb) return 2 << 16;
  return 3 << 16;
}

}  // namespace hpsg
