// ============================================================================
//  hps_device.cuh — shared device-side definitions for the HPS leaf-stage
//  kernels (sm_100a).
//
//  FP64 tensor work on sm_100a is warp-level mma.sync m8n8k4.f64, which ptxas
//  lowers to DMMA.8x8x4 (tcgen05/UMMA has no f64 kind).
//  Measured on the pool's B200: 37.1 TF/s DMMA vs 34.1 TF/s DFMA
//  (profiles/r01_fp64_peak.log), so the dense contractions go through DMMA.
// ============================================================================
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hpsg {

// ---------------------------------------------------------------------------
// Per-(p) leaf geometry.  Interior index i <-> local l = (i/(p-2)+1)*p + i%(p-2)+1.
// Boundary position k (S: ix 0..p-1, E: iy 1..p-1, N: ix 0..p-2, W: iy 1..p-2)
// (SURVEY Appendix A.4).  Augmented leaf matrix (row-major, ld):
//   rows [0, ni)      : [ A_ii | A_ib | f_i ]
//   rows [ni, ni+nb)  : [ D_i  | D_b  | 0   ]
// Partial LU of the first ni columns (pivots only among the first ni rows)
// leaves T_flux in the D_b block and -w_equiv in the last column:
//   D_b - D_i A_ii^{-1} A_ib = T_flux   (S_solve = -A_ii^{-1} A_ib)
//   0   - D_i A_ii^{-1} f_i  = -w_equiv
// ---------------------------------------------------------------------------
// Column layout: [0, ni) A_ii / D_i ; [ni, tb0) zero gap (keeps the trailing
// block 64-aligned) ; [tb0, tb0+nb) A_ib / D_b ; tb0+nb : f_i / 0 ; zero pad to ld.
struct LeafDims {
  int p, ni, nb;
  int R;      // ni + nb            (rows used)
  int Rpad;   // rows allocated     (multiple of 64)
  int tb0;    // first trailing column = 64 * nblk
  int ld;     // row stride in doubles (multiple of 64, >= tb0 + nb + 1)
  int nblk;   // 64-wide column blocks of A_ii
  int ntb;    // 64-wide trailing column blocks ([A_ib | f])
  long long leaf_stride;  // doubles per leaf workspace (Rpad * ld)
};

inline LeafDims make_dims(int p) {
  LeafDims d;
  d.p = p;
  d.ni = (p - 2) * (p - 2);
  d.nb = 4 * (p - 1);
  d.R = d.ni + d.nb;
  d.Rpad = (d.R + 63) / 64 * 64;
  d.nblk = (d.ni + 63) / 64;
  d.tb0 = 64 * d.nblk;
  d.ld = (d.tb0 + d.nb + 1 + 63) / 64 * 64;
  d.ntb = (d.nb + 1 + 63) / 64;
  d.leaf_stride = (long long)d.Rpad * d.ld;
  return d;
}

__device__ __forceinline__ int interior_local(int i, int p) {
  const int q = p - 2;
  return (i / q + 1) * p + (i % q) + 1;
}

// Boundary position k -> local id l and owning edge (0 S, 1 E, 2 N, 3 W).
__device__ __forceinline__ int boundary_local(int k, int p, int* edge) {
  if (k < p) { *edge = 0; return k; }                               // S: (0, k)
  if (k < 2 * p - 1) { *edge = 1; return (k - p + 1) * p + (p - 1); } // E: (k-p+1, p-1)
  if (k < 3 * p - 2) { *edge = 2; return (p - 1) * p + (k - 2 * p + 1); } // N: (p-1, k-2p+1)
  *edge = 3; return (k - 3 * p + 3) * p;                             // W: (k-3p+3, 0)
}

// ---------------------------------------------------------------------------
// DMMA m8n8k4 f64:  D = A(8x4) * B(4x8) + C.
// Fragments (cute SM80_8x8x4_F64F64F64F64_TN): lane g = lane>>2, t = lane&3;
//   A: A[g][t]   B: B[t][g]   C/D: C[g][2t], C[g][2t+1].
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: 16-byte global -> shared copies.
// ---------------------------------------------------------------------------
#ifndef HPS_L2_PREFETCH
#define HPS_L2_PREFETCH ".L2::256B"
#endif
// .L2::256B: every 16-byte request also pulls the rest of its 256-byte segment into L2,
// so a row's next K chunk is an L2 hit and DRAM sees 256-byte bursts.
// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): one 32-byte row segment per thread.
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ void ld_v4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p)
               : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global" HPS_L2_PREFETCH " [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// ---- mbarrier helpers (shared::cta) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar))
               : "memory");
}
// Arrive once this thread's prior cp.async copies have landed (count pre-set at init).
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1/x for a pivot: MUFU.RCP64H seed + two Newton steps, no special-case branch (IEEE
// division and __drcp_rn carry one, and a CALL to a slow path, on the pivot chain).
// Relative error ~1 ulp; x is a nonzero finite pivot (a zero or tiny pivot is a
// resonance and is flagged through min |pivot| / ||A_ii||).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

}  // namespace hpsg
