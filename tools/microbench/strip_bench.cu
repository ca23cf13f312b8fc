// Per-column cost of K2's pivot strip (base_strip) in isolation, and next to a co-resident
// CTA streaming DMMA on the same SM (the second K2 CTA's tile jobs).
//   blocks [0, sms): a leaf-like matrix of R rows; 16 strips (64 columns) of base_strip,
//                    thread 0 times each strip with clock64
//   blocks [sms, 2 sms) (co = 1): register-only DMMA loop for about as long
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2211_14969_b200/csrc \
//        tools/microbench/strip_bench.cu -o tools/microbench/strip_bench
#include <cstdio>
#include <vector>
#include "../../paper_2211_14969_b200/csrc/k2_lu_schur.cu"

using namespace hpsg;
using namespace hpsg::HPS_CFG;

template <int NSLOT>
__global__ void __launch_bounds__(NT, 2) strip_kernel(double* ws, int R, int ld, int co, long long* cyc,
                                                      double* sink) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  const int sms = gridDim.x / 2;
  if ((int)blockIdx.x >= sms) {
    if (!co) return;
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < co; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) sink[threadIdx.x] = s;
    return;
  }
  for (int i = threadIdx.x; i < MAX_RPAD; i += NT) {
    sm->perm[i] = (short)(i < R ? i : R - 1);
    sm->iperm[i] = (short)i;
  }
  __syncthreads();
  LeafCtx L;
  L.M = ws + (size_t)blockIdx.x * R * ld;
  L.ld = ld;
  L.R = R;
  L.ni = R;
  L.perm = sm->perm;
  L.iperm = sm->iperm;
  L.scratch = sm->pipe;
  L.wrow = &sm->wrow[0][0][0];
  L.redk = &sm->redk[0][0];
  const Grp G{(int)threadIdx.x, 0};
  double minpiv = 1e300;
  long long tp = 0;
  double* sbuf = L.scratch + 2 * 32 * XS;   // strip hand-off buffer, as panel_factor
  for (int s = 0; s < 16; ++s) {
    // as after an in-panel update: the strip's rows arrive in shared memory (untimed copy)
    for (int i = threadIdx.x; i < R - 4 * s; i += NT) {
      const double* src = L.M + (size_t)sm->perm[4 * s + i] * ld + 4 * s;
      for (int j = 0; j < 4; ++j) sbuf[4 * i + j] = src[j];
    }
    __syncthreads();
    const long long t0 = clock64();
    base_strip<NSLOT>(G, L, 4 * s, 4, minpiv, sbuf, nullptr, tp);
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x * 16 + s] = t1 - t0;
  }
  if (threadIdx.x == 0 && minpiv == 12345.0) sink[0] = minpiv;
}

template <int NSLOT>
void run(int R, int co, int sms) {
  const int ld = 128;
  double* ws;
  cudaMalloc(&ws, (size_t)sms * R * ld * 8);
  std::vector<double> h((size_t)sms * R * ld);
  unsigned s = 12345;
  for (auto& x : h) {
    s = s * 1664525u + 1013904223u;
    x = (double)(s >> 8) / (1 << 24) - 0.5;
  }
  cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  long long* cyc;
  cudaMalloc(&cyc, sms * 16 * 8);
  double* sink;
  cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(strip_kernel<NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  strip_kernel<NSLOT><<<2 * sms, NT, sizeof(Smem)>>>(ws, R, ld, co, cyc, sink);
  cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  strip_kernel<NSLOT><<<2 * sms, NT, sizeof(Smem)>>>(ws, R, ld, co, cyc, sink);
  std::vector<long long> c(sms * 16);
  cudaMemcpy(c.data(), cyc, c.size() * 8, cudaMemcpyDeviceToHost);
  double tot = 0;
  for (int b = 0; b < sms; ++b)
    for (int k = 1; k < 16; ++k) tot += c[b * 16 + k];
  printf("NT=%d NSLOT=%d R=%d co-resident DMMA CTA=%s: %.0f cycles per pivot column (%s)\n", NT, NSLOT, R,
         co ? "yes" : "no", tot / (sms * 15.0) / 4.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(ws);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#if HPS_NT == 256
  for (int co : {0, 400000}) {
    run<8>(1764, co, sms);
    run<4>(1024, co, sms);
    run<2>(484, co, sms);
  }
#else
  for (int co : {0, 400000}) {
    run<4>(484, co, sms);
    run<2>(256, co, sms);
  }
#endif
  return 0;
}
