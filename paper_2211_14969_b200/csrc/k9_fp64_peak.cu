// ============================================================================
//  FP64 tensor peak probe (the roofline denominator of K2/K3, measured in the same
//  process and on the same GPU as the bench; MEASURED_PEAKS.json has no FP64 entry).
//  A register-only loop of independent mma.sync.m8n8k4.f64 (DMMA.8x8x4) chains,
//  16 warps per CTA, 2 CTAs per SM: 512 flop per DMMA per warp.
//  Two figures, as MEASURED_PEAKS.json gives for bf16: the burst rate (best of three
//  ~10 ms launches after a warm-up) for kernels timed alone, and the sustained rate
//  (launches back to back for `sustain_s` seconds, rate of the last third) for kernels
//  timed inside a long step -- the B200 power cap lowers the SM clock under a
//  continuous FP64 tensor load.
// ============================================================================
#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

__global__ void __launch_bounds__(512) k9_dmma_peak_kernel(double* out, int iters) {
  const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;   // keep the loop alive
}

double measure_dmma_peak_tflops(int device, double sustain_s) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, 512 * sizeof(double)) != cudaSuccess) return 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000, blocks = 2 * sms, threads = 512;
  k9_dmma_peak_kernel<<<blocks, threads>>>(out, iters);   // warm-up (clocks up)
  float best = 1e30f;
  int launches = 1;
  if (sustain_s <= 0.0) {
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      k9_dmma_peak_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
  } else {
    // ~10 ms per launch: 2/3 of the launches bring the board to its power-limited steady
    // state, the last third is timed as one interval.
    cudaEventRecord(e0);
    k9_dmma_peak_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms1 = 10.0f;
    cudaEventElapsedTime(&ms1, e0, e1);
    const int total = static_cast<int>(sustain_s * 1e3 / (ms1 > 0.1f ? ms1 : 0.1f)) + 3;
    launches = total / 3;
    for (int r = 0; r < total - launches; ++r) k9_dmma_peak_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < launches; ++r) k9_dmma_peak_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&best, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = double(launches) * double(blocks) * (threads / 32) * double(iters) * 8.0 * 512.0;
  return cudaGetLastError() == cudaSuccess && best < 1e29f ? flops / (best * 1e-3) / 1e12 : 0.0;
}

}  // namespace hpsg
