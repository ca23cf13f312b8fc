// ============================================================================
//  GPU SlabLU — the reference's two-level direct solver of the reduced interface
//  system, on one B200.
//
//  Layout.  With the active ordering of SPEC.md:154 (interface edges sorted by
//  x-midpoint, then y-midpoint) the unknowns of element column c are its horizontal
//  edges followed by the vertical edges on its right, so contiguous element-column
//  slabs give the reduced unknowns as [I_0 | B_0 | I_1 | B_1 | ... | I_{S-1}]:
//  slab interiors I_s, slab interfaces B_k (the vertical edge column between slabs
//  k and k+1, ny*(p-2) unknowns).  Every block below is dense, column-major, in HBM.
//
//  factor:  per slab   A_II = P L U (getrf), X_l = A_II^-1 A_{I,B(s-1)}, X_r = A_II^-1 A_{I,B(s)}
//           per iface  T_k = A_{BkBk} - A_{Bk,Ik} X_r(k) - A_{Bk,Ik+1} X_l(k+1)
//                      U_k = A_{Bk,Bk+1} - A_{Bk,Ik+1} X_r(k+1),  L_k+1 = A_{Bk+1,Bk} - A_{Bk+1,Ik+1} X_l(k+1)
//           sweep      D_0 = T_0; E_k-1 = D_k-1^-1 U_k-1; D_k = T_k - L_k E_k-1 (getrf each D_k:
//                      no pivoting across blocks, the "limited pivoting scheme")
//  solve:   y_s = A_II^-1 f_Is; w_k = f_Bk - A_{Bk,Ik} y_k - A_{Bk,Ik+1} y_k+1;
//           s_k = D_k^-1 (w_k - L_k s_k-1); x_Blast = s_last, x_Bk = s_k - E_k x_Bk+1;
//           x_Is = y_s - X_l x_B(s-1) - X_r x_B(s)
//  The dense LU / solves / GEMMs are cuSOLVER + cuBLAS; the BSR gathers and the pivot
//  checks (min |U_kk| < 1e-12 ||block||_inf -> SingularBlockError) are kernels
//  of this file.  Deterministic: fixed operation order, no atomics.
// ============================================================================
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <memory>
#include <string>
#include <vector>

#include "hps_slablu.h"

#define HPS_OK_ 0
#define HPS_ERR_PARAM_ 2
#define HPS_ERR_CUDA_ 3

namespace {

// ---- kernels ---------------------------------------------------------------
// Dense column-major gather of the BSR rows [r0, r1) x block columns [c0, c1) (edge ids)
// into out (ld = (r1 - r0) q).  grid = r1 - r0 block rows, block 128.
__global__ void densify_kernel(const int64_t* __restrict__ brow_ptr, const int32_t* __restrict__ bcol_idx,
                               const double* __restrict__ blocks, int q, int64_t r0, int64_t c0, int64_t c1,
                               double* __restrict__ out, int64_t ld) {
  const int64_t br = r0 + blockIdx.x;
  const int64_t b0 = brow_ptr[br], b1 = brow_ptr[br + 1];
  const int qq = q * q;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t bc = bcol_idx[b];
    if (bc < c0 || bc >= c1) continue;
    const double* blk = blocks + b * qq;
    for (int t = threadIdx.x; t < qq; t += blockDim.x) {
      const int k = t / q, kk = t - k * q;   // block row-major: (k, kk)
      out[((bc - c0) * q + kk) * ld + blockIdx.x * (int64_t)q + k] = blk[t];
    }
  }
}

// ||A||_inf of an n x n column-major block (one thread per row, ascending columns).
__global__ void row_abs_sum_kernel(const double* __restrict__ A, int64_t n, double* __restrict__ rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = 0; j < n; ++j) s += fabs(A[j * n + i]);
  rows[i] = s;
}

// out[0] = max(rows), out[1] = min |diag(LU)| (single CTA, fixed-order reduction).
__global__ void pivot_check_kernel(const double* __restrict__ rows, const double* __restrict__ LU, int64_t n,
                                   double* __restrict__ out) {
  __shared__ double smax[256], smin[256];
  double mx = 0.0, mn = INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    mx = fmax(mx, rows[i]);
    mn = fmin(mn, fabs(LU[i * n + i]));
  }
  smax[threadIdx.x] = mx;
  smin[threadIdx.x] = mn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + o]);
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = smax[0];
    out[1] = smin[0];
  }
}

struct DBuf {
  double* p = nullptr;
  int64_t rows = 0, cols = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(int64_t r, int64_t c) {
    rows = r;
    cols = c;
    return cudaMalloc(&p, size_t(std::max<int64_t>(1, r * c)) * 8);
  }
  size_t bytes() const { return size_t(rows * cols) * 8; }
};
struct IBuf {
  int64_t* p = nullptr;
  ~IBuf() {
    if (p) cudaFree(p);
  }
};

thread_local std::string g_err;
thread_local int32_t g_block = 0;

int64_t edges_per_col(int ny) { return 2 * int64_t(ny) - 1; }

// Device bytes the factorization holds for width w (blocks + the largest getrf workspace
// excluded: a small fraction).
double factor_bytes(int p, int nx, int ny, int w) {
  const int64_t q = p - 2, S = nx / w, nB = int64_t(ny) * q;
  double tot = 0.0;
  for (int64_t s = 0; s < S; ++s) {
    const int64_t cb = s * w, ce = (s == S - 1) ? nx : (s + 1) * w;
    const int64_t nI = ((ce - 1) * edges_per_col(ny) + ny - 1 - cb * edges_per_col(ny)) * q;
    tot += double(nI) * nI + 4.0 * double(nI) * nB;
  }
  tot += double(S - 1) * 3.0 * double(nB) * nB;
  return tot * 8.0;
}

}  // namespace

struct hps_slablu {
  int device = 0, p = 0, nx = 0, ny = 0, w = 0, S = 0;
  int64_t q = 0, n_active = 0, nB = 0;
  std::vector<int64_t> i0, nI, b0;   // slab interior offsets/sizes, interface offsets
  std::vector<std::unique_ptr<DBuf>> A, Xl, Xr, BL, BR, D, E, L;
  std::vector<std::unique_ptr<IBuf>> ipA, ipD;
  cudaStream_t st = nullptr;
  cublasHandle_t cb = nullptr;
  cusolverDnHandle_t cs = nullptr;
  cusolverDnParams_t prm = nullptr;
  DBuf work, x, rows, chk;
  int* d_info = nullptr;
  size_t work_bytes = 0;
  hps_slablu_info_t info{};
  std::string err;
  ~hps_slablu() {
    if (d_info) cudaFree(d_info);
    if (prm) cusolverDnDestroyParams(prm);
    if (cs) cusolverDnDestroy(cs);
    if (cb) cublasDestroy(cb);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

#define CKC(call)                                                                                     \
  do {                                                                                                \
    cudaError_t e__ = (call);                                                                         \
    if (e__ != cudaSuccess) {                                                                         \
      g_err = std::string("CUDA error in ") + #call + ": " + cudaGetErrorString(e__);                \
      return HPS_ERR_CUDA_;                                                                           \
    }                                                                                                 \
  } while (0)
#define CKS(call)                                                                                     \
  do {                                                                                                \
    if ((call) != 0) {                                                                                \
      g_err = std::string("cuSOLVER/cuBLAS error in ") + #call;                                      \
      return HPS_ERR_CUDA_;                                                                           \
    }                                                                                                 \
  } while (0)

int densify(hps_slablu* s, const int64_t* d_rp, const int32_t* d_ci, const double* d_bl, int64_t r0, int64_t r1,
            int64_t c0, int64_t c1, DBuf& out) {
  CKC(out.alloc((r1 - r0) * s->q, (c1 - c0) * s->q));
  CKC(cudaMemsetAsync(out.p, 0, out.bytes(), s->st));
  if (r1 > r0) densify_kernel<<<unsigned(r1 - r0), 128, 0, s->st>>>(d_rp, d_ci, d_bl, int(s->q), r0, c0, c1, out.p,
                                                                    (r1 - r0) * s->q);
  CKC(cudaGetLastError());
  return HPS_OK_;
}

// LU in place with the pivot check; block index reported on failure.
int factor_block(hps_slablu* s, DBuf& M, std::unique_ptr<IBuf>& ip, int32_t block_index) {
  const int64_t n = M.rows;
  ip = std::make_unique<IBuf>();
  CKC(cudaMalloc(&ip->p, size_t(std::max<int64_t>(1, n)) * 8));
  if (n == 0) return HPS_OK_;
  CKC(s->rows.p ? cudaSuccess : cudaErrorInvalidValue);
  row_abs_sum_kernel<<<unsigned((n + 255) / 256), 256, 0, s->st>>>(M.p, n, s->rows.p);
  size_t dws = 0, hws = 0;
  CKS(cusolverDnXgetrf_bufferSize(s->cs, s->prm, n, n, CUDA_R_64F, M.p, n, CUDA_R_64F, &dws, &hws));
  if (dws > s->work_bytes) {
    if (s->work.p) cudaFree(s->work.p);
    s->work.p = nullptr;
    CKC(cudaMalloc(&s->work.p, dws));
    s->work_bytes = dws;
  }
  std::vector<char> hbuf(std::max<size_t>(1, hws));
  CKS(cusolverDnXgetrf(s->cs, s->prm, n, n, CUDA_R_64F, M.p, n, ip->p, CUDA_R_64F, s->work.p, dws, hbuf.data(), hws,
                       s->d_info));
  pivot_check_kernel<<<1, 256, 0, s->st>>>(s->rows.p, M.p, n, s->chk.p);
  double h[2];
  int info = 0;
  CKC(cudaMemcpyAsync(h, s->chk.p, 16, cudaMemcpyDeviceToHost, s->st));
  CKC(cudaMemcpyAsync(&info, s->d_info, 4, cudaMemcpyDeviceToHost, s->st));
  CKC(cudaStreamSynchronize(s->st));
  if (info != 0 || !(h[1] >= 1e-12 * h[0])) {
    g_block = block_index;
    g_err = "SingularBlockError: block " + std::to_string(block_index) + " (" +
            (block_index >= 0 ? "interface " + std::to_string(block_index)
                              : "interior of slab " + std::to_string(-1 - block_index)) +
            "): pivot " + std::to_string(h[1]) + " below 1e-12 * ||block||_inf = " + std::to_string(1e-12 * h[0]);
    return HPS_ERR_SINGULAR_BLOCK;
  }
  return HPS_OK_;
}

// B <- M^{-1} B with M factored (getrs, n x nrhs, column-major, ldb = n).
int solve_block(hps_slablu* s, const DBuf& M, const IBuf& ip, double* B, int64_t nrhs) {
  const int64_t n = M.rows;
  if (n == 0 || nrhs == 0) return HPS_OK_;
  CKS(cusolverDnXgetrs(s->cs, s->prm, CUBLAS_OP_N, n, nrhs, CUDA_R_64F, M.p, n, ip.p, CUDA_R_64F, B, n, s->d_info));
  return HPS_OK_;
}

// C <- C - A B  (column-major, A m x k, B k x n, C m x n)
int gemm_sub(hps_slablu* s, const double* A, const double* B, double* C, int64_t m, int64_t n, int64_t k) {
  if (m == 0 || n == 0 || k == 0) return HPS_OK_;
  const double alpha = -1.0, beta = 1.0;
  CKS(cublasDgemm(s->cb, CUBLAS_OP_N, CUBLAS_OP_N, int(m), int(n), int(k), &alpha, A, int(m), B, int(k), &beta, C,
                  int(m)));
  return HPS_OK_;
}
// y <- y - A x
int gemv_sub(hps_slablu* s, const double* A, const double* x, double* y, int64_t m, int64_t n) {
  if (m == 0 || n == 0) return HPS_OK_;
  const double alpha = -1.0, beta = 1.0;
  CKS(cublasDgemv(s->cb, CUBLAS_OP_N, int(m), int(n), &alpha, A, int(m), x, 1, &beta, y, 1));
  return HPS_OK_;
}

}  // namespace

extern "C" {

int32_t hps_slablu_default_width(int32_t p, int32_t nx, int32_t ny, int64_t budget) {
  if (p < 4 || nx < 2 || ny < 1) return 1;
  const double na = double((int64_t(nx) - 1) * ny + int64_t(nx) * (ny - 1)) * (p - 2);
  int w = int(std::ceil(std::cbrt(na / nx)));
  w = std::max(1, std::min(w, nx / 2));
  if (budget <= 0) {
    size_t fr = 0, tot = 0;
    budget = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? int64_t(0.7 * double(fr)) : (int64_t(64) << 30);
  }
  while (w > 1 && factor_bytes(p, nx, ny, w) > double(budget)) --w;
  return w;
}

const char* hps_slablu_last_error(const hps_slablu* s) { return s ? s->err.c_str() : g_err.c_str(); }
int32_t hps_slablu_last_block(void) { return g_block; }

int hps_slablu_factor(int device, int32_t p, int32_t nx, int32_t ny, int32_t slab_width, const int64_t* brow_ptr,
                      const int32_t* bcol_idx, const double* blocks, hps_slablu** out) {
  if (!out || !brow_ptr || !bcol_idx || !blocks) {
    g_err = "ParameterError: null argument";
    return HPS_ERR_PARAM_;
  }
  *out = nullptr;
  if (p < 4 || nx < 1 || ny < 1) {
    g_err = "ParameterError: p >= 4, nx, ny >= 1";
    return HPS_ERR_PARAM_;
  }
  CKC(cudaSetDevice(device));
  const int w = slab_width > 0 ? slab_width : hps_slablu_default_width(p, nx, ny, 0);
  if (w < 1 || nx / w < 2) {   // rejects widths leaving fewer than 2 slabs
    g_err = "ParameterError: slab width " + std::to_string(w) + " leaves fewer than 2 slabs (nx = " +
            std::to_string(nx) + ")";
    return HPS_ERR_PARAM_;
  }
  auto s = std::make_unique<hps_slablu>();
  s->device = device;
  s->p = p; s->nx = nx; s->ny = ny; s->w = w;
  s->q = p - 2;
  s->S = nx / w;
  const int64_t epc = edges_per_col(ny), q = s->q;
  const int64_t n_edges = (int64_t(nx) - 1) * ny + int64_t(nx) * (ny - 1);
  s->n_active = n_edges * q;
  s->nB = int64_t(ny) * q;
  const int S = s->S;
  // partition: edge ranges of I_s and B_s
  std::vector<int64_t> Ie0(S), Ie1(S), Be0(S), Be1(S);
  for (int k = 0; k < S; ++k) {
    const int64_t cb = int64_t(k) * w, ce = (k == S - 1) ? nx : int64_t(k + 1) * w;
    Ie0[k] = cb * epc;
    Ie1[k] = (ce - 1) * epc + ny - 1;
    Be0[k] = Ie1[k];
    Be1[k] = (k == S - 1) ? Ie1[k] : ce * epc;
  }
  s->i0.resize(S); s->nI.resize(S); s->b0.resize(S);
  for (int k = 0; k < S; ++k) {
    s->i0[k] = Ie0[k] * q;
    s->nI[k] = (Ie1[k] - Ie0[k]) * q;
    s->b0[k] = Be0[k] * q;
  }
  CKC(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
  CKS(cublasCreate(&s->cb));
  CKS(cublasSetStream(s->cb, s->st));
  CKS(cusolverDnCreate(&s->cs));
  CKS(cusolverDnSetStream(s->cs, s->st));
  CKS(cusolverDnCreateParams(&s->prm));
  CKC(cudaMalloc(&s->d_info, 4));
  CKC(s->chk.alloc(2, 1));
  int64_t maxn = s->nB;
  for (int k = 0; k < S; ++k) maxn = std::max(maxn, s->nI[k]);
  CKC(s->rows.alloc(maxn, 1));
  CKC(s->x.alloc(std::max<int64_t>(1, s->n_active), 1));
  // upload the BSR view
  const int64_t nnzb = brow_ptr[n_edges];
  int64_t* d_rp = nullptr;
  int32_t* d_ci = nullptr;
  double* d_bl = nullptr;
  struct Tmp {
    void* a; void* b; void* c;
    ~Tmp() { if (a) cudaFree(a); if (b) cudaFree(b); if (c) cudaFree(c); }
  } tmp{nullptr, nullptr, nullptr};
  CKC(cudaMalloc(&d_rp, size_t(n_edges + 1) * 8)); tmp.a = d_rp;
  CKC(cudaMalloc(&d_ci, size_t(std::max<int64_t>(1, nnzb)) * 4)); tmp.b = d_ci;
  CKC(cudaMalloc(&d_bl, size_t(std::max<int64_t>(1, nnzb)) * q * q * 8)); tmp.c = d_bl;
  CKC(cudaMemcpyAsync(d_rp, brow_ptr, size_t(n_edges + 1) * 8, cudaMemcpyHostToDevice, s->st));
  CKC(cudaMemcpyAsync(d_ci, bcol_idx, size_t(nnzb) * 4, cudaMemcpyHostToDevice, s->st));
  CKC(cudaMemcpyAsync(d_bl, blocks, size_t(nnzb) * q * q * 8, cudaMemcpyHostToDevice, s->st));
  cudaEvent_t e0, e1;
  CKC(cudaEventCreate(&e0));
  CKC(cudaEventCreate(&e1));
  CKC(cudaEventRecord(e0, s->st));
  s->A.resize(S); s->Xl.resize(S); s->Xr.resize(S); s->BL.resize(S); s->BR.resize(S); s->ipA.resize(S);
  s->D.resize(std::max(0, S - 1)); s->E.resize(std::max(0, S - 1)); s->L.resize(std::max(0, S - 1));
  s->ipD.resize(std::max(0, S - 1));
  int rc;
  // ---- slab interiors (independent; here one stream, in slab order) ----
  for (int k = 0; k < S; ++k) {
    s->A[k] = std::make_unique<DBuf>();
    if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Ie0[k], Ie1[k], Ie0[k], Ie1[k], *s->A[k]))) return rc;
    if ((rc = factor_block(s.get(), *s->A[k], s->ipA[k], -1 - k))) return rc;
    if (k > 0) {   // left interface B_{k-1}
      s->Xl[k] = std::make_unique<DBuf>();
      s->BL[k] = std::make_unique<DBuf>();
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Ie0[k], Ie1[k], Be0[k - 1], Be1[k - 1], *s->Xl[k]))) return rc;
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Be0[k - 1], Be1[k - 1], Ie0[k], Ie1[k], *s->BL[k]))) return rc;
      if ((rc = solve_block(s.get(), *s->A[k], *s->ipA[k], s->Xl[k]->p, s->nB))) return rc;
    }
    if (k < S - 1) {   // right interface B_k
      s->Xr[k] = std::make_unique<DBuf>();
      s->BR[k] = std::make_unique<DBuf>();
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Ie0[k], Ie1[k], Be0[k], Be1[k], *s->Xr[k]))) return rc;
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Be0[k], Be1[k], Ie0[k], Ie1[k], *s->BR[k]))) return rc;
      if ((rc = solve_block(s.get(), *s->A[k], *s->ipA[k], s->Xr[k]->p, s->nB))) return rc;
    }
  }
  // ---- interface blocks + block Thomas forward sweep (SPEC.md:446; sequential, :449) ----
  const int64_t nB = s->nB;
  for (int k = 0; k < S - 1; ++k) {
    s->D[k] = std::make_unique<DBuf>();
    if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Be0[k], Be1[k], Be0[k], Be1[k], *s->D[k]))) return rc;
    // T_k = A_BkBk - A_{Bk,Ik} X_r(k) - A_{Bk,Ik+1} X_l(k+1)
    if ((rc = gemm_sub(s.get(), s->BR[k]->p, s->Xr[k]->p, s->D[k]->p, nB, nB, s->nI[k]))) return rc;
    if ((rc = gemm_sub(s.get(), s->BL[k + 1]->p, s->Xl[k + 1]->p, s->D[k]->p, nB, nB, s->nI[k + 1]))) return rc;
    if (k > 0) {
      // L_k = A_{Bk,Bk-1} - A_{Bk,Ik} X_l(k) ;  D_k = T_k - L_k E_{k-1}
      s->L[k] = std::make_unique<DBuf>();
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Be0[k], Be1[k], Be0[k - 1], Be1[k - 1], *s->L[k]))) return rc;
      if ((rc = gemm_sub(s.get(), s->BR[k]->p, s->Xl[k]->p, s->L[k]->p, nB, nB, s->nI[k]))) return rc;
      if ((rc = gemm_sub(s.get(), s->L[k]->p, s->E[k - 1]->p, s->D[k]->p, nB, nB, nB))) return rc;
    }
    if ((rc = factor_block(s.get(), *s->D[k], s->ipD[k], k))) return rc;
    if (k < S - 2) {
      // U_k = A_{Bk,Bk+1} - A_{Bk,Ik+1} X_r(k+1) ;  E_k = D_k^{-1} U_k
      s->E[k] = std::make_unique<DBuf>();
      if ((rc = densify(s.get(), d_rp, d_ci, d_bl, Be0[k], Be1[k], Be0[k + 1], Be1[k + 1], *s->E[k]))) return rc;
      if ((rc = gemm_sub(s.get(), s->BL[k + 1]->p, s->Xr[k + 1]->p, s->E[k]->p, nB, nB, s->nI[k + 1]))) return rc;
      if ((rc = solve_block(s.get(), *s->D[k], *s->ipD[k], s->E[k]->p, nB))) return rc;
    }
  }
  CKC(cudaEventRecord(e1, s->st));
  CKC(cudaStreamSynchronize(s->st));
  cudaEventElapsedTime(&s->info.ms_factor, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  s->info.slab_width = w;
  s->info.n_slabs = S;
  s->info.n_active = s->n_active;
  s->info.n_interface = nB;
  int64_t mx = 0, bytes = 0;
  for (int k = 0; k < S; ++k) mx = std::max(mx, s->nI[k]);
  s->info.max_interior = mx;
  for (auto* v : {&s->A, &s->Xl, &s->Xr, &s->BL, &s->BR, &s->D, &s->E, &s->L})
    for (auto& b : *v)
      if (b) bytes += int64_t(b->bytes());
  s->info.device_bytes = bytes;
  *out = s.release();
  return HPS_OK_;
}

int hps_slablu_solve(hps_slablu* s, const double* rhs, double* x) {
  if (!s) return HPS_ERR_PARAM_;
  if (!rhs || !x) {
    s->err = "ParameterError: null vector";
    return HPS_ERR_PARAM_;
  }
  g_err.clear();
  auto fail = [&](int rc) {
    s->err = g_err;
    return rc;
  };
  if (cudaSetDevice(s->device) != cudaSuccess) return fail(HPS_ERR_CUDA_);
  const int S = s->S;
  const int64_t nB = s->nB;
  double* X = s->x.p;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rc = HPS_OK_;
  auto run = [&]() -> int {
    CKC(cudaMemcpyAsync(X, rhs, size_t(s->n_active) * 8, cudaMemcpyHostToDevice, s->st));
    CKC(cudaEventRecord(e0, s->st));
    int r;
    // y_s = A_II^{-1} f_Is
    for (int k = 0; k < S; ++k)
      if ((r = solve_block(s, *s->A[k], *s->ipA[k], X + s->i0[k], 1))) return r;
    // w_k = f_Bk - A_{Bk,Ik} y_k - A_{Bk,Ik+1} y_k+1 ; forward sweep s_k = D_k^{-1}(w_k - L_k s_k-1)
    for (int k = 0; k < S - 1; ++k) {
      double* xb = X + s->b0[k];
      if ((r = gemv_sub(s, s->BR[k]->p, X + s->i0[k], xb, nB, s->nI[k]))) return r;
      if ((r = gemv_sub(s, s->BL[k + 1]->p, X + s->i0[k + 1], xb, nB, s->nI[k + 1]))) return r;
      if (k > 0 && (r = gemv_sub(s, s->L[k]->p, X + s->b0[k - 1], xb, nB, nB))) return r;
      if ((r = solve_block(s, *s->D[k], *s->ipD[k], xb, 1))) return r;
    }
    // back sweep x_Bk = s_k - E_k x_Bk+1
    for (int k = S - 3; k >= 0; --k)
      if ((r = gemv_sub(s, s->E[k]->p, X + s->b0[k + 1], X + s->b0[k], nB, nB))) return r;
    // interiors x_Is = y_s - X_l x_B(s-1) - X_r x_B(s)
    for (int k = 0; k < S; ++k) {
      if (k > 0 && (r = gemv_sub(s, s->Xl[k]->p, X + s->b0[k - 1], X + s->i0[k], s->nI[k], nB))) return r;
      if (k < S - 1 && (r = gemv_sub(s, s->Xr[k]->p, X + s->b0[k], X + s->i0[k], s->nI[k], nB))) return r;
    }
    CKC(cudaEventRecord(e1, s->st));
    CKC(cudaMemcpyAsync(x, X, size_t(s->n_active) * 8, cudaMemcpyDeviceToHost, s->st));
    CKC(cudaStreamSynchronize(s->st));
    return HPS_OK_;
  };
  rc = run();
  if (rc == HPS_OK_) cudaEventElapsedTime(&s->info.ms_solve, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc == HPS_OK_ ? rc : fail(rc);
}

int hps_slablu_get_info(const hps_slablu* s, hps_slablu_info_t* out) {
  if (!s || !out) return HPS_ERR_PARAM_;
  *out = s->info;
  return HPS_OK_;
}

void hps_slablu_destroy(hps_slablu* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  delete s;
}

}  // extern "C"
