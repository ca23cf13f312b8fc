// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Used to pin the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double run(K kern, int blocks, int threads, int iters, double flop_per_thread_iter, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = (double)blocks * threads * iters * flop_per_thread_iter;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* out; cudaMalloc(&out, 1 << 26);
  const int iters = 20000;
  // DMMA m8n8k4: 8*8*4 FMA per warp = 512 flop per warp = 16 flop per thread per mma
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      double t4 = run(dmma_loop<4>, sms * bps, 32 * warps, iters, 16.0 * 4, out);
      double t8 = run(dmma_loop<8>, sms * bps, 32 * warps, iters, 16.0 * 8, out);
      printf("DMMA m8n8k4 warps/blk %2d blk/SM %d : NACC4 %.2f TF  NACC8 %.2f TF\n", warps, bps, t4, t8);
    }
  }
  for (int warps : {8, 16, 32}) {
    double t = run(dfma_loop<8>, sms * 2, 32 * warps, iters, 2.0 * 8, out);
    printf("DFMA warps/blk %2d blk/SM 2 NACC8 : %.2f TF\n", warps, t);
  }
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
