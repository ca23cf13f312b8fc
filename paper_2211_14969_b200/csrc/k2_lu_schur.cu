// ============================================================================
//  K2 + K3 — batched blocked FP64 LU of A_ii with partial pivoting, fused with
//  the multi-RHS triangular solve and the Schur-complement GEMM
//  (north star #2 and #3; replaces condense_leaf).
//
//  One CTA (256 threads, 8 warps) owns one leaf; two CTAs share an SM.  The
//  augmented leaf matrix M = [[A_ii, A_ib, f_i], [D_i, D_b, 0]] lives in the HBM
//  workspace written by K1.  A left-looking blocked LU over 64-wide column blocks
//  of A_ii turns every dense contraction into a "tile job"
//        C(64x64) <- C - A(64xK) * B(Kx64)        (DMMA m8n8k4, cp.async 4-stage)
//  and, continued over the trailing columns [A_ib | f], leaves
//        T_flux  = D_b - D_i A_ii^{-1} A_ib     in the D rows of the A_ib columns,
//        -w_equiv = -D_i A_ii^{-1} f_i          in the D rows of the f column,
//  i.e. exactly 2/3 ni^3 + 2 ni^2 nb + 2 nb^2 ni flops (getrf + getrs + gemm).
//
//  Pivoting never moves data: perm[] (shared memory) maps logical row -> physical
//  row and every tile load gathers rows through it.  Pivot candidates are the
//  not-yet-pivoted A_ii rows (physical < ni); D rows (physical >= ni) are carried
//  along as extra L rows.  Panels (64 columns) are factorised recursively: 4-wide
//  register strips with a warp-shuffle + shared-memory arg-max pivot search, and
//  the recursion's triangular/skinny updates.  The unit-lower diagonal block of
//  each panel is inverted once (Linv) so the U-part of later columns is two tile
//  jobs instead of a 64-step substitution.
//
//  Resonance: status = 1 when min |U_kk| < 1e-12 ||A_ii||_inf.
// ============================================================================
#include <climits>

#include "hps_device.cuh"
#include "hps_kernels.h"

namespace hpsg {

constexpr int NT = 256;              // threads per CTA
constexpr int TM = 64, TN = 64;      // tile job shape
constexpr int KC = 16;               // K chunk per pipeline stage
constexpr int NSTAGE = 4;
constexpr int LDA_S = KC + 4;        // 20 doubles: conflict-free A fragment loads
constexpr int LDB_S = TN + 4;        // 68 doubles: conflict-free B fragment loads
constexpr int STAGE_DBL = TM * LDA_S + KC * LDB_S;   // 2368 doubles
constexpr int PIPE_DBL = NSTAGE * STAGE_DBL;         // 9472 doubles = 75.8 KB
constexpr int NSLOT = 8;             // strip rows per thread: R <= 2048 (p <= 45)
constexpr int MAX_RPAD = 2048;

struct Smem {
  double pipe[PIPE_DBL];             // tile-job pipeline, re-used by the panel code
  double piv[4];                     // current pivot row (strip)
  double redv[NT / 32];
  int redl[NT / 32];
  int redp[NT / 32];
  short perm[MAX_RPAD];
};

// ---------------------------------------------------------------------------
// Tile job: acc = Cinit - A * B  (or + when sign = +1)
// ---------------------------------------------------------------------------
struct Acc {
  double v[2][4][2];
};

template <class ARow, class BRow>
__device__ __forceinline__ void load_chunk(double* st, const ARow& arow, const BRow& brow, int k0,
                                           int K) {
  double* As = st;
  double* Bs = st + TM * LDA_S;
  const int tid = threadIdx.x;
  if (k0 + KC <= K) {
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
      const int g = tid + rep * NT;
      const int row = g >> 3, seg = g & 7;
      cp_async16(As + row * LDA_S + 2 * seg, arow(row) + k0 + 2 * seg);
    }
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
      const int g = tid + rep * NT;
      const int row = g >> 5, seg = g & 31;
      cp_async16(Bs + row * LDB_S + 2 * seg, brow(k0 + row) + 2 * seg);
    }
  } else {  // K tail: predicated element loads, zero fill (k >= K contributes nothing)
    for (int e = tid; e < TM * KC; e += NT) {
      const int row = e / KC, col = e % KC;
      As[row * LDA_S + col] = (k0 + col < K) ? arow(row)[k0 + col] : 0.0;
    }
    for (int e = tid; e < KC * TN; e += NT) {
      const int row = e / TN, col = e % TN;
      Bs[row * LDB_S + col] = (k0 + row < K) ? brow(k0 + row)[col] : 0.0;
    }
  }
}

template <class ARow, class BRow>
__device__ void tile_mma(Acc& acc, const ARow& arow, const BRow& brow, int K, double sign,
                         double* pipe) {
  const int nch = (K + KC - 1) / KC;
  if (nch == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;
#pragma unroll
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < nch) load_chunk(pipe + s * STAGE_DBL, arow, brow, s * KC, K);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    {
      const int cn = c + NSTAGE - 1;
      if (cn < nch) load_chunk(pipe + (cn % NSTAGE) * STAGE_DBL, arow, brow, cn * KC, K);
      cp_async_commit();
    }
    const double* As = pipe + (c % NSTAGE) * STAGE_DBL;
    const double* Bs = As + TM * LDA_S;
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      double a[2], b[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) a[mi] = sign * As[(16 * wm + 8 * mi + g) * LDA_S + 4 * kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(4 * kk + t) * LDB_S + 32 * wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Fragment element (mi, ni, h) <-> tile row/col.
__device__ __forceinline__ int acc_row(int mi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  return 16 * (warp & 3) + 8 * mi + (lane >> 2);
}
__device__ __forceinline__ int acc_col(int ni) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  return 32 * (warp >> 2) + 8 * ni + 2 * (lane & 3);
}

template <class CRow>
__device__ __forceinline__ void acc_load(Acc& acc, const CRow& crow, int nrows) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int r = acc_row(mi);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      if (r < nrows) {
        const double2 v = *reinterpret_cast<const double2*>(crow(r) + acc_col(ni));
        acc.v[mi][ni][0] = v.x;
        acc.v[mi][ni][1] = v.y;
      } else {
        acc.v[mi][ni][0] = 0.0;
        acc.v[mi][ni][1] = 0.0;
      }
    }
  }
}

__device__ __forceinline__ void acc_zero(Acc& acc) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc.v[mi][ni][0] = acc.v[mi][ni][1] = 0.0;
}

template <class CRow>
__device__ __forceinline__ void acc_store(const Acc& acc, const CRow& crow, int nrows) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int r = acc_row(mi);
    if (r >= nrows) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(crow(r) + acc_col(ni)) =
          make_double2(acc.v[mi][ni][0], acc.v[mi][ni][1]);
  }
}

// ---------------------------------------------------------------------------
// Panel factorisation pieces
// ---------------------------------------------------------------------------
struct LeafCtx {
  double* M;         // leaf workspace
  int ld, R, ni;
  short* perm;       // shared
  Smem* sm;
};

__device__ __forceinline__ double* mrow(const LeafCtx& L, int logical) {
  return L.M + (size_t)L.perm[logical] * L.ld;
}

// Factor columns [e, e+sw) (sw <= 4) over logical rows [e, R): pivot search among
// not-yet-pivoted A_ii rows, register-resident rows, 2 barriers per column.
__device__ void base_strip(const LeafCtx& L, int e, int sw, double& minpiv) {
  Smem* sm = L.sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrows = L.R - e;
  double x[NSLOT][4];
  int phys[NSLOT], lpos[NSLOT];
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int idx = tid + s * NT;
    phys[s] = -1;
    lpos[s] = INT_MAX;
    x[s][0] = x[s][1] = x[s][2] = x[s][3] = 0.0;
    if (idx < nrows) {
      lpos[s] = e + idx;
      phys[s] = L.perm[e + idx];
      const double* src = L.M + (size_t)phys[s] * L.ld + e;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < sw) x[s][j] = src[j];
    }
  }
  __syncthreads();  // everyone has read perm[] before thread 0 starts swapping
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= sw) break;
    const int col = e + j;
    const int p_old = L.perm[col];
    double best = -1.0;
    int bl = INT_MAX, bp = -1;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      if (phys[s] >= 0 && phys[s] < L.ni && lpos[s] >= col) {
        const double v = fabs(x[s][j]);
        if (v > best || (v == best && lpos[s] < bl)) { best = v; bl = lpos[s]; bp = phys[s]; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ov > best || (ov == best && ol < bl)) { best = ov; bl = ol; bp = op; }
    }
    if (lane == 0) { sm->redv[warp] = best; sm->redl[warp] = bl; sm->redp[warp] = bp; }
    __syncthreads();
    best = sm->redv[0]; bl = sm->redl[0]; bp = sm->redp[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) {
      const double ov = sm->redv[w];
      const int ol = sm->redl[w];
      if (ov > best || (ov == best && ol < bl)) { best = ov; bl = ol; bp = sm->redp[w]; }
    }
    // pivot row owner publishes its (already updated) strip row
#pragma unroll
    for (int s = 0; s < NSLOT; ++s)
      if (phys[s] == bp) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) sm->piv[jj] = x[s][jj];
      }
    if (tid == 0) {
      L.perm[col] = (short)bp;
      L.perm[bl] = (short)p_old;
    }
    __syncthreads();
    const double piv = sm->piv[j];
    if (tid == 0) minpiv = fmin(minpiv, fabs(piv));
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      if (phys[s] == bp) lpos[s] = col;
      else if (phys[s] == p_old) lpos[s] = bl;
      if (phys[s] >= 0 && lpos[s] > col) {
        const double l = x[s][j] / piv;
        x[s][j] = l;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (jj > j && jj < sw) x[s][jj] = fma(-l, sm->piv[jj], x[s][jj]);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    if (phys[s] < 0) continue;
    double* dst = L.M + (size_t)phys[s] * L.ld + e;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < sw) dst[j] = x[s][j];
  }
  __syncthreads();
}

// Recursive-LU update inside a panel: source columns [s0, s0+h) are factored,
// destination columns [d0, d0+nd) (d0 = s0+h) have all earlier updates.
//   U part (rows s0..s0+h-1):  X = L_hh^{-1} X         (forward substitution)
//   L part (rows d0..R-1)   :  C -= A[:, src] * X       (skinny FMA update)
__device__ void panel_update(const LeafCtx& L, int s0, int h, int d0, int nd) {
  Smem* sm = L.sm;
  double* Ls = sm->pipe;              // h x h   (stride 33)
  double* X = sm->pipe + 33 * 32;     // h x nd  (stride 33)
  const int tid = threadIdx.x;
  for (int e = tid; e < h * h; e += NT) {
    const int i = e / h, k = e % h;
    Ls[i * 33 + k] = (k < i) ? mrow(L, s0 + i)[s0 + k] : 0.0;
  }
  for (int e = tid; e < h * nd; e += NT) {
    const int i = e / nd, j = e % nd;
    X[i * 33 + j] = mrow(L, s0 + i)[d0 + j];
  }
  __syncthreads();
  for (int k = 0; k < h - 1; ++k) {
    for (int e = tid; e < (h - 1 - k) * nd; e += NT) {
      const int i = k + 1 + e / nd, j = e % nd;
      X[i * 33 + j] = fma(-Ls[i * 33 + k], X[k * 33 + j], X[i * 33 + j]);
    }
    __syncthreads();
  }
  for (int e = tid; e < h * nd; e += NT) {
    const int i = e / nd, j = e % nd;
    mrow(L, s0 + i)[d0 + j] = X[i * 33 + j];
  }
  // L part: rows logical [d0, R)
  for (int r = d0 + tid; r < L.R; r += NT) {
    double* row = mrow(L, r);
    for (int j0 = 0; j0 < nd; j0 += 8) {
      double acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = (j0 + j < nd) ? row[d0 + j0 + j] : 0.0;
      for (int k = 0; k < h; ++k) {
        const double a = row[s0 + k];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fma(-a, X[k * 33 + j0 + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < nd) row[d0 + j0 + j] = acc[j];
    }
  }
  __syncthreads();
}

// Inverse of the unit-lower diagonal block of panel [c0, c0+w) -> Linv (64x64,
// identity-padded, row-major).
__device__ void panel_linv(const LeafCtx& L, int c0, int w, double* linv) {
  double* Ls = L.sm->pipe;            // 64 x 65
  double* X = L.sm->pipe + 64 * 65;   // 64 x 65
  const int tid = threadIdx.x;
  for (int e = tid; e < 64 * 64; e += NT) {
    const int i = e >> 6, k = e & 63;
    Ls[i * 65 + k] = (i < w && k < i) ? mrow(L, c0 + i)[c0 + k] : 0.0;
    X[i * 65 + k] = (i == k) ? 1.0 : 0.0;
  }
  __syncthreads();
  // X <- L^{-1}: for k, rows i > k: X[i, :k+1] -= L[i,k] * X[k, :k+1]
  for (int k = 0; k < w - 1; ++k) {
    const int nr = w - 1 - k, ncol = k + 1;
    for (int e = tid; e < nr * ncol; e += NT) {
      const int i = k + 1 + e / ncol, j = e % ncol;
      X[i * 65 + j] = fma(-Ls[i * 65 + k], X[k * 65 + j], X[i * 65 + j]);
    }
    __syncthreads();
  }
  for (int e = tid; e < 64 * 64; e += NT) linv[e] = X[(e >> 6) * 65 + (e & 63)];
  __syncthreads();
}

__device__ void panel_factor(const LeafCtx& L, int c0, int w, double& minpiv) {
  for (int e = c0; e < c0 + w;) {
    const int sw = min(4, c0 + w - e);
    base_strip(L, e, sw, minpiv);
    e += sw;
    const int done = e - c0;
    if (done < w) {
      const int h = done & (-done);      // lowest set bit: recursive-LU schedule
      panel_update(L, e - h, h, e, min(h, c0 + w - e));
    }
  }
}

// ---------------------------------------------------------------------------
// Kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 2) k2_lu_schur_kernel(LuArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  const LeafDims d = a.d;
  const int leaf = blockIdx.x;
  LeafCtx L;
  L.M = a.ws + (size_t)leaf * d.leaf_stride;
  L.ld = d.ld;
  L.R = d.R;
  L.ni = d.ni;
  L.perm = sm->perm;
  L.sm = sm;
  double* Linv = a.linv + (size_t)leaf * d.nblk * 4096;
  short* perm_g = a.perm + (size_t)leaf * d.Rpad;
  // Entries past Rpad are read by masked-out tile rows (e.g. the D-row tiles start at ni, which
  // need not be 64-aligned): point them at a valid row so the gathers stay in bounds.
  for (int i = threadIdx.x; i < MAX_RPAD; i += NT)
    sm->perm[i] = i < d.Rpad ? (a.factor ? (short)i : perm_g[i]) : (short)(d.Rpad - 1);
  __syncthreads();
  double minpiv = INFINITY;  // meaningful on thread 0

  const double* M = L.M;
  const int ld = d.ld;
  const short* perm = sm->perm;
  auto lrow = [&](int base) {  // rows gathered through perm, starting at logical `base`
    return [=](int i) -> const double* { return M + (size_t)perm[base + i] * ld; };
  };

  // ---------------- A_ii block columns ----------------
  for (int J = 0; J < (a.factor ? d.nblk : 0); ++J) {
    const int c0 = 64 * J;
    const int w = min(64, d.ni - c0);
    // (a) U part: logical rows [64 I, 64 I + 64), I < J
    for (int I = 0; I < J; ++I) {
      const int r0 = 64 * I;
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[r0 + i] * ld + c0; };
      Acc acc;
      acc_load(acc, crow, TM);
      auto arow = lrow(r0);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
      tile_mma(acc, arow, brow, r0, -1.0, sm->pipe);
      acc_store(acc, crow, TM);
      __threadfence_block();
      __syncthreads();
      // X <- Linv_I * X
      const double* li = Linv + (size_t)I * 4096;
      acc_zero(acc);
      auto arow2 = [=](int i) -> const double* { return li + i * 64; };
      auto brow2 = [=](int k) -> const double* { return M + (size_t)perm[r0 + k] * ld + c0; };
      tile_mma(acc, arow2, brow2, 64, 1.0, sm->pipe);
      acc_store(acc, crow, TM);
      __threadfence_block();
      __syncthreads();
    }
    // (b) L part: logical rows [c0, R)
    for (int rt = c0; rt < d.R; rt += TM) {
      const int nr = min(TM, d.R - rt);
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[rt + i] * ld + c0; };
      Acc acc;
      acc_load(acc, crow, nr);
      auto arow = lrow(rt);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
      tile_mma(acc, arow, brow, c0, -1.0, sm->pipe);
      acc_store(acc, crow, nr);
    }
    __threadfence_block();
    __syncthreads();
    // (c) panel factorisation + inverse of its unit-lower diagonal block
    panel_factor(L, c0, w, minpiv);
    panel_linv(L, c0, w, Linv + (size_t)J * 4096);
  }

  // ---------------- trailing columns [A_ib | f] ----------------
  for (int tb = 0; tb < d.ntb; ++tb) {
    const int c0 = d.tb0 + 64 * tb;
    for (int I = 0; I < d.nblk; ++I) {
      const int r0 = 64 * I;
      const int nr = min(TM, d.ni - r0);
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[r0 + i] * ld + c0; };
      Acc acc;
      acc_load(acc, crow, TM);
      auto arow = lrow(r0);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
      tile_mma(acc, arow, brow, r0, -1.0, sm->pipe);
      acc_store(acc, crow, nr);
      __threadfence_block();
      __syncthreads();
      const double* li = Linv + (size_t)I * 4096;
      acc_zero(acc);
      auto arow2 = [=](int i) -> const double* { return li + i * 64; };
      auto brow2 = [=](int k) -> const double* { return M + (size_t)perm[r0 + k] * ld + c0; };
      tile_mma(acc, arow2, brow2, 64, 1.0, sm->pipe);
      acc_store(acc, crow, nr);
      __threadfence_block();
      __syncthreads();
    }
    // D rows: T = D_b - L21 U12 ; -w = 0 - L21 (L^{-1} f)
    double* Tl = a.T_out + (size_t)leaf * d.nb * d.nb;
    double* wl = a.w_out + (size_t)leaf * d.nb;
    for (int rt = d.ni; rt < d.R; rt += TM) {
      const int nr = min(TM, d.R - rt);
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[rt + i] * ld + c0; };
      Acc acc;
      acc_load(acc, crow, nr);
      auto arow = lrow(rt);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
      tile_mma(acc, arow, brow, d.ni, -1.0, sm->pipe);
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const int r = acc_row(mi);
        if (r >= nr) continue;
        const int trow = rt + r - d.ni;
#pragma unroll
        for (int ni2 = 0; ni2 < 4; ++ni2) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int tc = 64 * tb + acc_col(ni2) + hh;
            if (tc < d.nb) Tl[(size_t)trow * d.nb + tc] = acc.v[mi][ni2][hh];
            else if (tc == d.nb) wl[trow] = -acc.v[mi][ni2][hh];
          }
        }
      }
    }
  }
  if (!a.factor) return;
  __syncthreads();
  for (int i = threadIdx.x; i < d.Rpad; i += NT) perm_g[i] = sm->perm[i];
  if (threadIdx.x == 0) {
    const double nrm = a.norms[leaf];
    const double ratio = nrm > 0.0 ? minpiv / nrm : 0.0;
    if (a.minratio) a.minratio[leaf] = ratio;
    a.status[leaf] = (ratio >= 1e-12) ? 0 : 1;
  }
}

size_t lu_smem_bytes() { return sizeof(Smem); }

void launch_lu_schur(const LuArgs& a, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  cudaFuncSetAttribute(k2_lu_schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(Smem));
  k2_lu_schur_kernel<<<n_leaves, NT, sizeof(Smem), st>>>(a);
}

}  // namespace hpsg
