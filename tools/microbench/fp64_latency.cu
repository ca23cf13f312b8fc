// Dependent-chain latency of FP64 ops (DFMA, DMUL, reciprocal, SHFL, REDUX) on one warp, alone
// and with K co-resident warps streaming DMMA.m8n8k4 (contention on the SM's FP64 datapath).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int OP>
__global__ void lat(double* out, long long* cyc, int iters, int same_smsp, int lds_mix) {
  __shared__ double sm[1024];
  sm[threadIdx.x % 1024] = threadIdx.x;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp == 0) {
    double x = 1.0 + threadIdx.x * 1e-9, y = 0.999999;
    unsigned u = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (OP == 0) x = fma(x, y, 1e-9);
      else if (OP == 1) x = x * y;
      else if (OP == 2) x = 1.0 / x;
      else if (OP == 3) u = __reduce_max_sync(0xffffffffu, u) + 1;
      else if (OP == 4) x = __shfl_xor_sync(0xffffffffu, x, 1) * 1.0000001;
      else if (OP == 5) { double c1 = 0.0; dmma(x, c1, y, 1.0); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { *cyc = t1 - t0; done = 1; }
    out[threadIdx.x] = x + u;
  } else if (warp % 4 == 0 || !same_smsp) {
    double c[8][2] = {};
    double a = 1.0 + threadIdx.x, b = 0.5;
    while (!done) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (lds_mix) a = sm[(threadIdx.x * 5 + r * 33) & 1023];
        dmma(c[r][0], c[r][1], a, b);
      }
    }
    double s = 0;
    for (int r = 0; r < 8; ++r) s += c[r][0] + c[r][1];
    out[1024 + threadIdx.x] = s;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8 << 20); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DMUL", "1.0/x", "REDUX", "SHFL+DMUL", "DMMA-chain"};
  const int iters = 2048;
  for (int mix = 0; mix < 2; ++mix)
  for (int op : {0, 2, 5}) {
    for (int m : {0, 1, 2, 3}) {   // m DMMA warps on the probe warp's SMSP (warps 4, 8, 12)
      long long h = 0;
      const int nthr = 32 * (1 + 4 * m);
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: lat<0><<<1, nthr>>>(out, cyc, iters, 1, mix); break;
          case 2: lat<2><<<1, nthr>>>(out, cyc, iters, 1, mix); break;
          case 5: lat<5><<<1, nthr>>>(out, cyc, iters, 1, mix); break;
        }
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      }
      printf("%-10s  co-SMSP DMMA warps %d (lds mix %d): %8.1f cycles/op\n", names[op], m, mix, double(h) / iters);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
