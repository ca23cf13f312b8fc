// K2 tile-job mainloop with TMA operand staging (tile::gather4) vs the cp.async mainloop.
// Every CTA runs `reps` tile jobs C(TMxTN) -= A(TMxK) B(KxTN) on its own 2048 x ld block of
// rows, rows gathered through a per-CTA permutation (as K2's perm[]).
//   A stage: TM x 16 doubles, SWIZZLE_128B (16-byte chunk j of row r at chunk j ^ (r & 7)),
//            one gather4 per 4 rows.
//   B stage: TN/8 column blocks of 16 x 8 doubles, unswizzled (a 4-row fragment read is 256
//            contiguous bytes), one gather4 per block per 4 rows.
// Each warp's lane 0 stages its share of a chunk (expect_tx on the stage's full barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2211_14969_b200/csrc \
//        tools/microbench/tma_bench.cu -o tools/microbench/tma_bench
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2211_14969_b200/csrc/k2_lu_schur.cu"

using namespace hpsg;
using namespace hpsg::g256;

#ifndef SWZ_ROW
#define SWZ_ROW(r) ((r) & 7)   // swizzle row phase as seen by the fragment reads
#endif

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, unsigned long long* bar, int col,
                                            int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

template <int TM_, int TN_>
struct TT {
  static constexpr int WM = TM_ / 32, WN = TN_ / 32, K = 16;
  static constexpr int A_DBL = TM_ * 16, B_DBL = 16 * TN_;
  static constexpr int STAGE = A_DBL + B_DBL;                 // multiple of 128 doubles (1 KB)
  static constexpr int A_G4_PER_WARP = TM_ / 4 / 8;            // gather4s of A rows per warp
  static constexpr int B_BLK_PER_WARP = TN_ / 8 / 8;           // 8-column B blocks per warp
#ifndef DIAG
#define DIAG 0   // 1: stage A only, 2: stage B only (throughput diagnostics; results wrong)
#endif
  static constexpr unsigned BYTES_PER_WARP =
      ((DIAG == 2 ? 0 : A_G4_PER_WARP * 4 * 16) + (DIAG == 1 ? 0 : B_BLK_PER_WARP * 16 * 8)) * 8;
};
#ifndef TNS
#define TNS 3
#endif
constexpr int NS = TNS;

struct TSmem {
  alignas(1024) double pipe[NS * (128 * 16 + 16 * 64)];
  unsigned long long full[NS], empty[NS];
  int perm[2048];
};

// rows: global row of logical row i = base + perm[i]
template <class T>
__device__ void tma_tile(Acc& acc, const CUtensorMap* mA, const CUtensorMap* mB, TSmem* sm, int base, int arow0,
                         int bcol, int K, unsigned& gch) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % T::WM, wn = warp / T::WM;
  const int nch = K / 16;
  const int* perm = sm->perm;
  auto fill = [&](int c) {
    const unsigned gf = gch + c;
    const int st = gf % NS;
    if (gf >= NS) mbar_wait(&sm->empty[st], ((gf - NS) / NS) & 1u);
    if (lane == 0) {
      double* As = sm->pipe + st * T::STAGE;
      double* Bs = As + T::A_DBL;
      mbar_expect_tx(&sm->full[st], T::BYTES_PER_WARP);
#pragma unroll
      for (int j = 0; j < (DIAG == 2 ? 0 : T::A_G4_PER_WARP); ++j) {
        const int r = (warp * T::A_G4_PER_WARP + j) * 4;
        tma_gather4(As + r * 16, mA, &sm->full[st], c * 16, base + perm[arow0 + r], base + perm[arow0 + r + 1],
                    base + perm[arow0 + r + 2], base + perm[arow0 + r + 3]);
      }
#pragma unroll
      for (int b = 0; b < (DIAG == 1 ? 0 : T::B_BLK_PER_WARP); ++b) {
        const int blk = warp * T::B_BLK_PER_WARP + b;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = c * 16 + 4 * j;
          tma_gather4(Bs + blk * 128 + 4 * j * 8, mB, &sm->full[st], bcol + 8 * blk, base + perm[k],
                      base + perm[k + 1], base + perm[k + 2], base + perm[k + 3]);
        }
      }
    }
  };
  for (int s = 0; s < NS - 1; ++s)
    if (s < nch) fill(s);
  acc_zero(acc);
  int aoff[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) aoff[kk] = ((((2 * kk + (t >> 1)) ^ SWZ_ROW(g))) << 1) + (t & 1);
  for (int c = 0; c < nch; ++c) {
    const unsigned gc = gch + c;
    const int st = gc % NS;
    mbar_wait(&sm->full[st], (gc / NS) & 1u);
    const double* As = sm->pipe + st * T::STAGE;
    const double* Bs = As + T::A_DBL;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (kk == 3 && c + NS - 1 < nch) fill(c + NS - 1);
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = -As[(32 * wm + 8 * mi + g) * 16 + aoff[kk]];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(4 * wn + ni) * 128 + (4 * kk + t) * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm->empty[st]);
  }
  gch += nch;
}

template <class T>
__global__ void __launch_bounds__(256, 2) tma_bench_kernel(const __grid_constant__ CUtensorMap mA,
                                                           const __grid_constant__ CUtensorMap mB, double* ws,
                                                           int ld, int K, int reps, const int* perm_g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TSmem* sm = reinterpret_cast<TSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 2048; i += 256) sm->perm[i] = perm_g ? perm_g[i] : i;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&sm->full[s], 8);
      mbar_init(&sm->empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int base = blockIdx.x * 2048;
  double* M = ws + (size_t)base * ld;
  constexpr int TM_ = T::WM * 32;
  unsigned gch = 0;
  for (int r = 0; r < reps; ++r) {
    const int rt = (r % 4) * TM_;
    Acc acc;
    tma_tile<T>(acc, &mA, &mB, sm, base, rt, 1024, K, gch);
    // C rows (logical rt + i) at columns 1536..: C -= A B
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % T::WM, wn = warp / T::WM;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = 32 * wm + 8 * mi + (lane >> 2);
      double* crow = M + (size_t)sm->perm[rt + i] * ld + 1536;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int c = 32 * wn + 8 * ni + 2 * (lane & 3);
        double2 v = *reinterpret_cast<double2*>(crow + c);
        v.x += acc.v[mi][ni][0];
        v.y += acc.v[mi][ni][1];
        *reinterpret_cast<double2*>(crow + c) = v;
      }
    }
    __syncthreads();
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<EncodeFn>(fn);
}

static CUtensorMap make_map(double* ws, size_t rows, int ld, int box_cols, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ws, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

template <class T>
void run(const char* name, int ctas, int K, int reps, double* ws, int ld, const CUtensorMap& mA,
         const CUtensorMap& mB, const int* perm) {
  auto k = tma_bench_kernel<T>;
  const int smem = sizeof(TSmem) + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<ctas, 256, smem>>>(mA, mB, ws, ld, K, 1, perm);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<<<ctas, 256, smem>>>(mA, mB, ws, ld, K, reps, perm);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * T::WM * 32 * T::WN * 32 * (double)K * reps * ctas;
  printf("TMA %s ctas=%d K=%d: %.3f ms  %.2f TF/s  (%s)\n", name, ctas, K, ms, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

// Correctness: one CTA, random values, random permutation, one job; C compared on the host.
template <class T>
bool check(const char* name, double* ws, int ld, const CUtensorMap& mA, const CUtensorMap& mB, int* perm_d) {
  const int rows = 2048, K = 256;
  std::vector<double> h((size_t)rows * ld);
  srand(7);
  for (auto& x : h) x = (rand() % 2001 - 1000) / 1000.0;
  std::vector<int> perm(2048);
  for (int i = 0; i < 2048; ++i) perm[i] = i;
  for (int i = 2047; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
  cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(perm_d, perm.data(), 2048 * 4, cudaMemcpyHostToDevice);
  auto k = tma_bench_kernel<T>;
  const int smem = sizeof(TSmem) + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 256, smem>>>(mA, mB, ws, ld, K, 1, perm_d);
  std::vector<double> out((size_t)rows * ld);
  cudaMemcpy(out.data(), ws, out.size() * 8, cudaMemcpyDeviceToHost);
  constexpr int TM_ = T::WM * 32, TN_ = T::WN * 32;
  double err = 0;
  for (int i = 0; i < TM_; ++i)
    for (int j = 0; j < TN_; ++j) {
      double s = 0;
      for (int kk = 0; kk < K; ++kk) s += h[(size_t)perm[i] * ld + kk] * h[(size_t)perm[kk] * ld + 1024 + j];
      const double ref = h[(size_t)perm[i] * ld + 1536 + j] - s;
      err = std::max(err, std::abs(out[(size_t)perm[i] * ld + 1536 + j] - ref));
    }
  printf("check %s: max abs err %.3e (%s)\n", name, err, cudaGetErrorString(cudaGetLastError()));
  return err < 1e-9;
}

int main() {
  const int ld = 2048;
  const int ctas_max = 296;
  const size_t rows = (size_t)ctas_max * 2048;
  double* ws;
  cudaMalloc(&ws, rows * ld * 8 + (1 << 20));
  cudaMemset(ws, 0, rows * ld * 8);
  int* perm_d;
  cudaMalloc(&perm_d, 2048 * 4);
  CUtensorMap mA = make_map(ws, rows, ld, 16, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap mB = make_map(ws, rows, ld, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
  bool ok = check<TT<128, 64>>("128x64", ws, ld, mA, mB, perm_d);
  ok &= check<TT<64, 128>>("64x128", ws, ld, mA, mB, perm_d);
  cudaMemset(ws, 0, rows * ld * 8);
  for (int ctas : {148, 296}) {
    run<TT<128, 64>>("128x64", ctas, 1024, 40, ws, ld, mA, mB, nullptr);
    run<TT<64, 128>>("64x128", ctas, 1024, 40, ws, ld, mA, mB, nullptr);
    run<TT<128, 64>>("128x64", ctas, 256, 160, ws, ld, mA, mB, nullptr);
    run<TT<128, 64>>("128x64", ctas, 64, 400, ws, ld, mA, mB, nullptr);
  }
  return ok ? 0 : 1;
}
