// Isolated throughput of the K2 tile-job mainloop (tile_mma) on B200: every CTA runs
// `reps` tile jobs C(TMxTN) -= A(TMxK) B(KxTN) on its own rows (perm = identity).
#include <cstdio>
// TB_BLK = 0: row-major leaf rows (stride ld).  TB_BLK > 0: column-blocked layout, 16-column
// blocks of TB_BLK doubles each (all rows of a block contiguous, 128 B per row).
#ifndef TB_BLK
#define TB_BLK 0
#endif
#if TB_BLK
#define HPS_KOFF(k) (((k) / 16) * (long long)TB_BLK)
#define HPS_COFF(c) (((c) / 16) * (long long)TB_BLK + (c) % 16)
#endif
#include "../../paper_2211_14969_b200/csrc/k2_lu_schur.cu"

using namespace hpsg;
using namespace hpsg::HPS_CFG;

template <class TL, bool HOT = false>
#ifndef TB_MINB
#define TB_MINB 2
#endif
__global__ void __launch_bounds__(NT, TB_MINB) tile_bench_kernel(double* ws, int ld, int K, int reps) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < MAX_RPAD; i += NT) sm->perm[i] = (short)i;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm->full[s], NT);
      mbar_init(&sm->empty[s], NT / 32);
    }
    sm->gchunk = 0;
  }
  __syncthreads();
  const double* M = ws + (size_t)blockIdx.x * 2048 * ld;
  const short* perm = sm->perm;
  constexpr int TM_ = TL::WM * 32;
  for (int r = 0; r < reps; ++r) {
    const int rt = (r % 4) * TM_;
    const double* MA = HOT ? ws : M;
    const int ldh = HOT ? 0 : (TB_BLK ? 16 : ld);   // HOT: every row aliases row 0 -> L1/L2-resident operands
    auto arow = [=](int i) -> const double* { return MA + (size_t)perm[rt + i] * ldh; };
    auto brow = [=](int k) -> const double* { return MA + (size_t)perm[k] * ldh + HPS_COFF(1024); };
    auto crow = [=](int i) -> double* { return const_cast<double*>(M) + (size_t)perm[rt + i] * ld + 1536; };
    Acc acc;
    auto init = [&](Acc& x) { acc_load<TL>(x, crow, TM_); };
    tile_mma<TL>(Grp{(int)threadIdx.x, 0}, acc, init, arow, brow, K, -1.0, sm->pipe, sm->full, sm->empty,
                 &sm->gchunk);
    acc_store<TL>(acc, crow, TM_, TL::WN * 32);
  }
}

template <class TL, bool HOT = false>
void run(const char* name, int ctas, int K, int reps, double* ws, int ld) {
  cudaFuncSetAttribute(tile_bench_kernel<TL, HOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  tile_bench_kernel<TL, HOT><<<ctas, NT, sizeof(Smem)>>>(ws, ld, K, 1);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  tile_bench_kernel<TL, HOT><<<ctas, NT, sizeof(Smem)>>>(ws, ld, K, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * TL::WM * 32 * TL::WN * 32 * (double)K * reps * ctas;
  printf("%s%s ctas=%d K=%d: %.3f ms  %.2f TF/s  (%s)\n", name, HOT ? " HOT" : "", ctas, K, ms, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}



// Compute-only variants of the same mainloop: fragments from shared memory, no global loads.
template <class TL, bool BARRIER>
__global__ void __launch_bounds__(NT, 2) compute_only_kernel(double* out, int nch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  for (int i = threadIdx.x; i < PIPE_DBL; i += NT) sm->pipe[i] = 1e-3 * (i % 17);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % TL::WM, wn = warp / TL::WM;
  Acc acc;
  acc_zero(acc);
  for (int c = 0; c < nch; ++c) {
    if (BARRIER) __syncthreads();
    const double* As = sm->pipe + (c % NSTAGE) * TL::STAGE;
    const double* Bs = As + (TL::WM * 32) * TL::LDA;
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = -As[(32 * wm + 8 * mi + g) * TL::LDA + 4 * kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(4 * kk + t) * TL::LDB + 32 * wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
  }
  double s = 0;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) s += acc.v[mi][ni][0] + acc.v[mi][ni][1];
  out[blockIdx.x * NT + threadIdx.x] = s;
}

template <class TL, bool BARRIER>
void run_compute(const char* name, int ctas, int nch) {
  double* out;
  cudaMalloc(&out, ctas * NT * 8);
  auto k = compute_only_kernel<TL, BARRIER>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  k<<<ctas, NT, sizeof(Smem)>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<ctas, NT, sizeof(Smem)>>>(out, nch);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * TL::WM * 32 * TL::WN * 32 * (double)KC * nch * ctas;
  printf("compute-only %s barrier=%d ctas=%d: %.2f TF/s\n", name, (int)BARRIER, ctas, fl / ms / 1e9);
  cudaFree(out);
}

void run_all_compute() {
  for (int ctas : {148, 296}) {
    run_compute<TileL, true>("128x64", ctas, 20000);
    run_compute<TileL, false>("128x64", ctas, 20000);
  }
}

int main() {
  run_all_compute();
  const int ld = 2048;
  double* ws;
  cudaMalloc(&ws, (size_t)592 * 2048 * ld * 8 + (1 << 20));
  cudaMemset(ws, 0, (size_t)592 * 2048 * ld * 8);
#ifdef TB_G128   // -DHPS_NT=128 -DHPS_CFG=g128 -DHPS_MAX_ROWS=640 -DHPS_NSTAGE=2 -DTB_MINB=4 -DTB_G128
  for (int ctas : {148, 296, 592}) {
    run<TileL>("64x64", ctas, 400, 100, ws, ld);
    run<TileL>("64x64", ctas, 192, 200, ws, ld);
    run<TileL>("64x64", ctas, 64, 400, ws, ld);
  }
  return 0;
#endif
  for (int ctas : {148, 296}) {
    run<TileL>("128x64", ctas, 1024, 40, ws, ld);
    run<TileU>("64x128", ctas, 1024, 40, ws, ld);
    run<TileL>("128x64", ctas, 256, 160, ws, ld);
    run<TileL>("128x64", ctas, 64, 400, ws, ld);
    run<TileL, true>("128x64", ctas, 1024, 40, ws, ld);
  }
  return 0;
}
