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

#include "hps_assembly.cuh"
#include "hps_device.cuh"
#include "hps_kernels.h"

#ifndef HPS_NT
#define HPS_NT 256
#endif
#ifndef HPS_CFG
#define HPS_CFG g256
#endif

namespace hpsg {
// Two builds of this file (Makefile), each in its own namespace:
//   g256: HPS_NT=256 (8-warp CTAs, 2 per SM, 3 stages, R <= 2048)  -- large p
//   g128: HPS_NT=128 (4-warp CTAs, more leaves per SM, R <= 1024)   -- small p, where the
//         latency-bound pivot panels dominate and more co-resident leaves hide them.
namespace HPS_CFG {

// Optional per-phase cycle counters (LuArgs::phase_cycles != nullptr): thread 0
// accumulates clock64() deltas between CTA-wide barriers into 8 slots per leaf:
// 0 U-part tiles, 1 L-part tiles, 2 panel strips+updates, 3 Linv, 4 trailing.
#ifdef HPS_STRIP_MARKS
#define STRIP_MARK(slot) PHASE_MARK(slot)
#else
#define STRIP_MARK(slot) do { } while (0)
#endif
#define PHASE_MARK(slot)                                                     \
  do {                                                                       \
    if (pc && G.tid == 0) {                                                  \
      const long long now__ = clock64();                                     \
      pc[slot] += now__ - t_phase;                                           \
      t_phase = now__;                                                       \
    }                                                                        \
  } while (0)

constexpr int NT = HPS_NT;           // threads per CTA / group (32x32 warp tiles)
constexpr int NWARP = NT / 32;
#ifndef HPS_NSTAGE
#define HPS_NSTAGE 3
#endif
#ifndef HPS_CTAS
#define HPS_CTAS 2
#endif
#ifndef HPS_MAX_ROWS
#define HPS_MAX_ROWS 2048
#endif
#ifndef HPS_DIST
#define HPS_DIST 0   // tile-job prefetch distance in chunks (0: NSTAGE - 1)
#endif
#ifndef HPS_UNR4_MAXH
#define HPS_UNR4_MAXH 8
#endif
#ifndef HPS_KC
#define HPS_KC 16
#endif
#ifndef HPS_OWNER_SWITCH
#define HPS_OWNER_SWITCH 1   // pivot-row publish: switch on the slot instead of a select chain
#endif
#ifndef HPS_LPF
#define HPS_LPF (HPS_NT != 256)   // L-part tile init prefetches the C tile into L1 (measured: helps g128, not g256)
#endif
#ifndef HPS_TPF
#define HPS_TPF 1   // D-row (trailing) tile init prefetches the C tile into L1
#endif
#ifndef HPS_UPF
#define HPS_UPF 1   // U-part tile init: 0 prefetch the C tile into L1, 1 none (measured best), 2 prefetch Linv_J rows
#endif
#ifndef HPS_STRIP_REDUX2
#define HPS_STRIP_REDUX2 1   // cross-warp pivot arg-max with redux.sync on the lanes
#endif
#ifndef HPS_STRIP_LEAN
#define HPS_STRIP_LEAN 1   // candidate carried through the arg-max, key bits fixed per strip
#endif

// Column offset inside a row of the leaf matrix (row-major).  The tile microbenchmark
// redefines these to measure a column-blocked layout (tools/microbench/tile_bench.cu).
#ifndef HPS_KOFF
#define HPS_KOFF(k) (k)
#define HPS_COFF(c) (c)
#endif
constexpr int KC = HPS_KC;           // K chunk per stage
constexpr int NSTAGE = HPS_NSTAGE;   // pipeline stages
constexpr int MAX_NSTAGE = 4;
constexpr int MAX_NSLOT = 8;
static_assert(MAX_NSLOT * NT >= HPS_MAX_ROWS, "strip rows per thread");         // strip rows per thread: R <= 2048 (p <= 45)
constexpr int MAX_RPAD = HPS_MAX_ROWS + 128;  // perm entries (tile gathers may run past R)

// A group of NT threads sharing a named barrier.  The one-leaf-per-CTA kernel uses the whole
// CTA (barrier 0); the lock-step multi-leaf kernel runs several groups (barriers 1..).
// gtid(): thread index within its group (the tile/panel helpers are group-local).
__device__ __forceinline__ int gtid() { return static_cast<int>(threadIdx.x) & (NT - 1); }

struct Grp {
  int tid;   // thread index within the group
  int bar;   // named barrier id
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(NT) : "memory");
  }
};

// Tile jobs C(TM x TN) <- C -/+ A(TM x K) B(K x TN): 128x64 for the L part and the
// D rows (row-tall), 64x128 for the U part (row-wide).  Stage: A TM x KC (+4 pad),
// B KC x TN (+4 pad); both pads make the m8n8k4 fragment loads bank-conflict free.
template <int TM_, int TN_, int KC_ = KC, int NS_ = NSTAGE>
struct Tile {
  static constexpr int WM = TM_ / 32, WN = TN_ / 32;   // warp grid, WM * WN == 8
  static constexpr int K = KC_;                       // K chunk
  static constexpr int NS = NS_;                      // pipeline stages
  static constexpr int LDA = KC_ + 4;                 // == 4 mod 16: conflict-free A fragments
  static constexpr int LDB = TN_ + 4;
  static constexpr int STAGE = TM_ * LDA + KC_ * LDB;
  static constexpr int AGR = TM_ * KC_ / 2 / NT;      // 16-byte A granules / thread / chunk
  static constexpr int BGR = KC_ * TN_ / 2 / NT;      // 16-byte B granules / thread / chunk
  static constexpr int BROW = TN_ / 2;                // granules per B row
  static_assert(WM * WN == NT / 32, "one 32x32 warp tile per warp");
  static_assert(NS_ <= MAX_NSTAGE, "stages");
};
#if HPS_NT == 256
using TileL = Tile<128, 64>;
using TileU = Tile<64, 128>;
#else
using TileL = Tile<64, 64>;
using TileU = Tile<64, 64>;
#endif
constexpr int TLM = TileL::WM * 32;  // L-part / D-row tile rows
constexpr int TUN = TileU::WN * 32;  // U-part tile columns
constexpr int LS_U = TUN + 4;        // Linv-apply staging of a 64 x TUN U tile (== 4 mod 16)
constexpr int cmax(int a, int b) { return a > b ? a : b; }
// The pipeline region doubles as panel scratch: in-panel update blocks (2 x 32 x 36),
// the strip hand-off (4 x rows) and the Linv/Uinv staging (64 x 65).
constexpr int PANEL_DBL = cmax(2 * 32 * 36 + 4 * HPS_MAX_ROWS, 64 * 65);
constexpr int PIPE_DBL =
    cmax(cmax(cmax(NSTAGE * TileL::STAGE, NSTAGE * TileU::STAGE), 64 * LS_U), PANEL_DBL);

struct Smem {
  double pipe[PIPE_DBL];             // tile-job pipeline, re-used by the panel code
  unsigned long long full[NSTAGE];   // stage filled (256 thread arrivals)
  unsigned long long empty[NSTAGE];  // stage consumed (8 warp arrivals)
  unsigned gchunk;                   // running K-chunk counter of this CTA
  int next_leaf;                     // dynamic leaf schedule (LuArgs::sched)
  alignas(16) double wrow[2][NWARP][8];          // per-warp pivot candidate rows + 1/pivot (double-buffered)
  unsigned long long redk[2][NWARP];
  short perm[MAX_RPAD];              // logical -> physical row
  short iperm[MAX_RPAD];             // physical -> logical row
};

// Accumulator of one 32x32 warp tile: 4x4 DMMA 8x8 tiles, 2 doubles per lane each.
struct Acc {
  double v[4][4][2];
};

template <class TL>
__device__ __forceinline__ int acc_row(int mi) {
  const int warp = gtid() >> 5, lane = threadIdx.x & 31;
  return 32 * (warp % TL::WM) + 8 * mi + (lane >> 2);
}
template <class TL>
__device__ __forceinline__ int acc_col(int ni) {
  const int warp = gtid() >> 5, lane = threadIdx.x & 31;
  return 32 * (warp / TL::WM) + 8 * ni + 2 * (lane & 3);
}

// Stage one K chunk.  Full chunks: per-thread A row pointers fixed for the whole tile
// job, B rows re-gathered through perm each chunk.  K tail: predicated element loads
// with zero fill (k >= K contributes nothing).
// Stage one K chunk.  Full chunks: per-thread A row pointers fixed for the whole tile
// job, B rows re-gathered through perm each chunk, cp.async with an mbarrier arrival on
// completion.  K tail: predicated element loads with zero fill (k >= K contributes
// nothing) followed by a plain arrival.
template <class TL, class ARow, class BRow>
__device__ __forceinline__ void load_chunk(double* st, unsigned long long* full, const double* const* pa,
                                           const ARow& arow, const BRow& brow, int k0, int K) {
  double* As = st;
  double* Bs = st + (TL::WM * 32) * TL::LDA;
  const int tid = gtid();
  constexpr int TM_ = TL::WM * 32, TN_ = TL::WN * 32, KC_ = TL::K;
  if (k0 + KC_ <= K) {
#pragma unroll
    for (int r = 0; r < TL::AGR; ++r) {
      const int gi = tid + r * NT;
      cp_async16(As + (gi / (KC_ / 2)) * TL::LDA + 2 * (gi % (KC_ / 2)), pa[r] + HPS_KOFF(k0));
    }
#pragma unroll
    for (int r = 0; r < TL::BGR; ++r) {
      const int gi = tid + r * NT;
      const int row = gi / TL::BROW, seg = gi % TL::BROW;
      cp_async16(Bs + row * TL::LDB + 2 * seg, brow(k0 + row) + HPS_COFF(2 * seg));
    }
    cp_async_mbar_arrive(full);
  } else {
    for (int e = tid; e < TM_ * KC_; e += NT) {
      const int row = e / KC_, col = e % KC_;
      As[row * TL::LDA + col] = (k0 + col < K) ? arow(row)[k0 + col] : 0.0;
    }
    for (int e = tid; e < KC_ * TN_; e += NT) {
      const int row = e / TN_, col = e % TN_;
      Bs[row * TL::LDB + col] = (k0 + row < K) ? brow(k0 + row)[col] : 0.0;
    }
    mbar_arrive(full);
  }
}

// Tile job mainloop: NSTAGE-deep cp.async pipeline synchronised by per-stage mbarriers
// (full: 256 thread arrivals as copies land; empty: 8 warp arrivals as a stage is
// consumed) instead of a CTA-wide barrier per K chunk.  Chunks are numbered per CTA
// (sm->gchunk) across tile jobs so the barrier phases stay consistent.
template <class TL, class ARow, class BRow, class Init>
__device__ void tile_mma(const Grp& G, Acc& acc, const Init& init, const ARow& arow, const BRow& brow,
                         int K, double sign, double* pipe, unsigned long long* full,
                         unsigned long long* empty, unsigned* gchunk, int mact = TL::WM * 32,
                         int nact = TL::WN * 32) {
  constexpr int KC_ = TL::K, NS_ = TL::NS;
  const int nch = (K + KC_ - 1) / KC_;
  if (nch == 0) {
    init(acc);
    return;
  }
  const int warp = gtid() >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % TL::WM, wn = warp / TL::WM;
  // Warps whose 32x32 tile lies wholly in the padding of a remainder tile (fewer than
  // mact rows / nact columns are real) only stage operands: no DMMA on padding.
  const bool act = 32 * wm < mact && 32 * wn < nact;
  const unsigned g0 = *gchunk;
  const double* pa[TL::AGR];
#pragma unroll
  for (int r = 0; r < TL::AGR; ++r) {
    const int gi = gtid() + r * NT;
    pa[r] = arow(gi / (KC_ / 2)) + 2 * (gi % (KC_ / 2));
  }
  auto fill = [&](int c) {
    const unsigned gf = g0 + c;
    const int st = gf % NS_;
    if (gf >= NS_) mbar_wait(&empty[st], ((gf - NS_) / NS_) & 1u);
    load_chunk<TL>(pipe + st * TL::STAGE, &full[st], pa, arow, brow, c * KC_, K);
  };
#pragma unroll
  // Prefetch distance DIST <= NS-1 chunks: the refill of chunk c+DIST goes into the stage
  // of chunk c+DIST-NS, released NS-DIST chunks earlier (slack for slow warps).
  constexpr int DIST = (HPS_DIST > 0 && HPS_DIST < NS_) ? HPS_DIST : NS_ - 1;
  for (int s = 0; s < DIST; ++s)
    if (s < nch) fill(s);
  init(acc);   // C-init (load or first-touch assembly) overlaps the prologue copies
  // The refill of the stage freed by chunk c-1 is issued while computing chunk c (before its
  // last k-step): the wait for the slowest warp to release that stage is then mostly hidden.
  for (int c = 0; c < nch; ++c) {
    const unsigned gc = g0 + c;
    const int st = gc % NS_;
    mbar_wait(&full[st], (gc / NS_) & 1u);
    const double* As = pipe + st * TL::STAGE;
    const double* Bs = As + (TL::WM * 32) * TL::LDA;
    if (!act) {
      if (c + DIST < nch) fill(c + DIST);
    } else
#pragma unroll
    for (int kk = 0; kk < KC_ / 4; ++kk) {
      if (kk == KC_ / 4 - 1 && c + DIST < nch) fill(c + DIST);
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sign * As[(32 * wm + 8 * mi + g) * TL::LDA + 4 * kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[(4 * kk + t) * TL::LDB + 32 * wn + 8 * ni + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc.v[mi][ni][0], acc.v[mi][ni][1], a[mi], b[ni]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  G.sync();
  if (G.tid == 0) *gchunk = g0 + nch;
  G.sync();
}

// C tile element access, rows masked by nrows, columns by ncols.
template <class TL, class CRow>
__device__ __forceinline__ void acc_load(Acc& acc, const CRow& crow, int nrows) {
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = acc_row<TL>(mi);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      if (r < nrows) {
        const double2 v = *reinterpret_cast<const double2*>(crow(r) + acc_col<TL>(ni));
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
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc.v[mi][ni][0] = acc.v[mi][ni][1] = 0.0;
}

// Accuracy: a tile job accumulates its K-range product sum from ZERO and adds the original
// entries once at the end (C <- C + (-sum A B)), instead of subtracting every product from a
// running value initialised with C.  With near-singular A_ii (leaves next to a resonance) the
// running-value form loses an order of magnitude: at C4's worst leaf (cond(A_ii) ~ 2e8) T was
// 5.0e-11 from an extended-precision reference against LAPACK's 2.0e-12; the separate sum is
// what blocked LAPACK effectively does (tools/leaf_refine.py, profiles/r02_leaf_refine_*.json).
// Only the tile jobs need it (the in-panel updates sum at most 32 products: measured no gain,
// profiles/r02_k2_accuracy_ab.log).  The C tile is prefetched into L1 when the job starts so
// the epilogue's load hits.
template <class TL, class CRow>
__device__ __forceinline__ void acc_prefetch_l1(const CRow& crow, int nrows) {
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = acc_row<TL>(mi);
    if (r >= nrows) continue;
    asm volatile("prefetch.global.L1 [%0];" ::"l"(crow(r) + acc_col<TL>(0)));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(crow(r) + acc_col<TL>(2)));
  }
}
template <class TL, class CRow>
__device__ __forceinline__ void acc_add(Acc& acc, const CRow& crow, int nrows) {
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = acc_row<TL>(mi);
    if (r >= nrows) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double2 c = *reinterpret_cast<const double2*>(crow(r) + acc_col<TL>(ni));
      acc.v[mi][ni][0] = __dadd_rn(c.x, acc.v[mi][ni][0]);
      acc.v[mi][ni][1] = __dadd_rn(c.y, acc.v[mi][ni][1]);
    }
  }
}

template <class TL, class CRow>
__device__ __forceinline__ void acc_store(const Acc& acc, const CRow& crow, int nrows, int ncols) {
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = acc_row<TL>(mi);
    if (r >= nrows) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int c = acc_col<TL>(ni);
      if (c + 1 < ncols)
        *reinterpret_cast<double2*>(crow(r) + c) = make_double2(acc.v[mi][ni][0], acc.v[mi][ni][1]);
      else if (c < ncols)
        crow(r)[c] = acc.v[mi][ni][0];
    }
  }
}

// U-part epilogue: acc (64x128 tile) <- Linv (64x64) * acc.  The tile goes through
// shared memory; Linv fragments come straight from global (32 KB per block row, L1/L2
// resident across the block row's tiles).  TRI = 1: Linv is lower triangular (zeros above
// the diagonal), TRI = 2: upper; the k-steps that only meet those zeros are skipped
// (72 of 128 DMMA groups remain).
constexpr int TRI_FULL = 0, TRI_LOWER = 1, TRI_UPPER = 2;
#ifndef HPS_NACT
#define HPS_NACT (HPS_NT == 256)   // skip DMMA on warp tiles made only of column padding
#endif
#ifndef HPS_TRI_SKIP
#define HPS_TRI_SKIP 1
#endif

// acc = Linv[32 WMI .. 32 WMI + 31, :] * Cs[:, 32 wn ..]: fully unrolled so the triangular
// k-range of every 8-row group is a compile-time constant.
template <int TRI, int WMI>
__device__ __forceinline__ void linv_core(Acc& acc, const double* __restrict__ linv, const double* Cs,
                                          int wn, int g, int t, int ls) {
  acc_zero(acc);
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    // rows of group mi: [32 WMI + 8 mi, +8); k-step covers k in [4 kk, 4 kk + 4)
    bool need[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
      need[mi] = !HPS_TRI_SKIP || TRI == TRI_FULL ||
                 (TRI == TRI_LOWER ? 4 * kk <= 32 * WMI + 8 * mi + 7 : 4 * kk + 3 >= 32 * WMI + 8 * mi);
    if (!(need[0] || need[1] || need[2] || need[3])) continue;
    double av[4], bv[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
      if (need[mi]) av[mi] = linv[(32 * WMI + 8 * mi + g) * 64 + 4 * kk + t];  // coherent: written in-kernel
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bv[ni] = Cs[(4 * kk + t) * ls + 32 * wn + 8 * ni + g];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      if (!need[mi]) continue;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc.v[mi][ni][0], acc.v[mi][ni][1], av[mi], bv[ni]);
    }
  }
}

template <int TRI = TRI_FULL>
__device__ __forceinline__ void linv_apply(const Grp& G, Acc& acc, const double* __restrict__ linv,
                                           double* pipe, int nact = TUN) {
  static_assert(TileU::WM == 2, "linv_apply: two 32-row warp groups");
  double* Cs = pipe;   // 64 x LS_U
  const int warp = gtid() >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = warp % TileU::WM, wn = warp / TileU::WM;
  const bool act = 32 * wn < nact;   // each warp reads only its own 32 columns of Cs
  if (act)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(Cs + acc_row<TileU>(mi) * LS_U + acc_col<TileU>(ni)) =
          make_double2(acc.v[mi][ni][0], acc.v[mi][ni][1]);
  G.sync();
  if (act) {
    if (wm == 0) linv_core<TRI, 0>(acc, linv, Cs, wn, g, t, LS_U);
    else linv_core<TRI, 1>(acc, linv, Cs, wn, g, t, LS_U);
  }
  G.sync();
}

// ---------------------------------------------------------------------------
// Panel factorisation pieces
// ---------------------------------------------------------------------------
struct LeafCtx {
  double* M;                 // leaf workspace
  int ld, R, ni;
  short* perm;               // shared: logical -> physical
  short* iperm;              // shared: physical -> logical
  double* scratch;           // shared: panel scratch (>= 64*65 doubles)
  double* wrow;              // shared: [2][NWARP][8] pivot candidate rows, [4] = 1/pivot
  unsigned long long* redk;  // shared: [2][8] pivot keys
};

__device__ __forceinline__ double* mrow(const LeafCtx& L, int logical) {
  return L.M + (size_t)L.perm[logical] * L.ld;
}

// Factor columns [e, e+sw) (sw <= 4) over logical rows [e, R) with register-resident
// rows and ONE barrier per column.  Pivot search: every candidate (not yet pivoted A_ii
// row, physical id < ni <= 2047) becomes a 64-bit key  bits(|v|) with its low 11 mantissa
// bits replaced by (2047 - phys)  -- an order-preserving, symmetric arg-max that costs one
// integer max per comparison; magnitudes closer than 2^-41 relative are treated as ties
// and resolved by the smaller physical row (deterministic for any thread mapping).  Each
// warp publishes its winner and that row's strip values (double-buffered slots), so the
// pivot row needs no second broadcast round.  Interchanges are bookkeeping only: thread 0
// swaps perm/iperm after the barrier; nobody else reads them inside the strip.
// Integer-only (the sign bit is masked, no fabs): FP64 instructions here would queue
// behind the co-resident CTA's DMMA on the shared FP64 pipe.
__device__ __forceinline__ unsigned long long pivot_key(double v, int phys) {
  return (static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7FFFFFFFFFFFF800ull) |
         static_cast<unsigned long long>(0x7FF - phys);
}

template <int NSLOT>
__device__ void base_strip(const Grp& G, const LeafCtx& L, int e, int sw, double& minpiv,
                           const double* sbuf, long long* pc, long long& t_phase) {
  const int tid = G.tid, lane = tid & 31, warp = tid >> 5;
  const int nrows = L.R - e;
  double x[NSLOT][4];
  int phys[NSLOT];
  unsigned active = 0;   // bit s: slot holds a row that is not yet pivoted
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    const int idx = tid + s * NT;
    phys[s] = 0x7FFF;
    x[s][0] = x[s][1] = x[s][2] = x[s][3] = 0.0;
    if (idx < nrows) {
      phys[s] = L.perm[e + idx];
      active |= 1u << s;
      if (sbuf) {   // handed over in shared memory by the preceding panel_update
        const double2 v0 = *reinterpret_cast<const double2*>(sbuf + 4 * idx);
        const double2 v1 = *reinterpret_cast<const double2*>(sbuf + 4 * idx + 2);
        x[s][0] = v0.x; x[s][1] = v0.y; x[s][2] = v1.x; x[s][3] = v1.y;
      } else {
        const double* src = L.M + (size_t)phys[s] * L.ld + e;
        if (sw == 4) {
          ld_v4(src, x[s][0], x[s][1], x[s][2], x[s][3]);   // e % 4 == 0, ld % 64 == 0
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < sw) x[s][j] = src[j];
        }
      }
    }
  }
#if HPS_STRIP_LEAN
  unsigned elig = 0;
  unsigned klo[NSLOT];
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    if (((active >> s) & 1u) && phys[s] < L.ni) elig |= 1u << s;
    klo[s] = static_cast<unsigned>(0x7FF - phys[s]);
  }
#endif
  G.sync();  // all perm reads done before thread 0 starts swapping
  PHASE_MARK(8);
  int pivrow[4];
  double pivval[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= sw) break;
    const int buf = j & 1;
    unsigned long long best = 0ull;
    int bs = 0;
#if HPS_STRIP_LEAN
    // The candidate value rides along with the arg-max; eligibility and the low key bits were
    // fixed when the strip was loaded (elig tracks the pivoted rows).
    double cand = 0.0;
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const unsigned long long k = ((elig >> s) & 1u)
          ? (static_cast<unsigned long long>(__double_as_longlong(x[s][j])) & 0x7FFFFFFFFFFFF800ull) | klo[s]
          : 0ull;
      if (k > best) { best = k; bs = s; cand = x[s][j]; }
    }
#else
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      const unsigned long long k =
          ((active >> s) & 1u) && phys[s] < L.ni ? pivot_key(x[s][j], phys[s]) : 0ull;
      if (k > best) { best = k; bs = s; }
    }
    // Every lane takes the reciprocal of its own candidate now, so the FP64 division chain
    // overlaps the warp arg-max instead of following it (only the winner's is published).
    double cand = x[0][j];
#pragma unroll
    for (int s = 1; s < NSLOT; ++s)
      if (s == bs) cand = x[s][j];
#endif
    const double rcand = best != 0ull ? fast_rcp(cand) : 0.0;
    // Warp arg-max of the 64-bit keys with two redux.sync (high word, then low word among
    // the lanes holding the maximal high word).
    const unsigned hi = static_cast<unsigned>(best >> 32);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? static_cast<unsigned>(best) : 0u);
    const unsigned long long wbest = (static_cast<unsigned long long>(mhi) << 32) | mlo;
    STRIP_MARK(11);
    if (lane == 0) L.redk[buf * NWARP + warp] = wbest;
    if (best == wbest && best != 0ull) {  // this lane owns the warp's candidate row
      double* wr = L.wrow + (buf * NWARP + warp) * 8;
#if HPS_OWNER_SWITCH
      // One indirect branch to the slot's two stores instead of a select chain over all slots
      // (the chain is issued by the whole warp for one active lane).
      switch (bs) {
#define HPS_PUB(S)                                                                    \
  case S:                                                                           \
    if (S < NSLOT) {                                                                \
      *reinterpret_cast<double2*>(wr) = make_double2(x[S % NSLOT][0], x[S % NSLOT][1]); \
      *reinterpret_cast<double2*>(wr + 2) = make_double2(x[S % NSLOT][2], x[S % NSLOT][3]); \
    }                                                                               \
    break;
        HPS_PUB(0) HPS_PUB(1) HPS_PUB(2) HPS_PUB(3) HPS_PUB(4) HPS_PUB(5) HPS_PUB(6) HPS_PUB(7)
#undef HPS_PUB
      }
#else
      double r0 = x[0][0], r1 = x[0][1], r2 = x[0][2], r3 = x[0][3];
#pragma unroll
      for (int s = 1; s < NSLOT; ++s)
        if (s == bs) { r0 = x[s][0]; r1 = x[s][1]; r2 = x[s][2]; r3 = x[s][3]; }
      *reinterpret_cast<double2*>(wr) = make_double2(r0, r1);
      *reinterpret_cast<double2*>(wr + 2) = make_double2(r2, r3);
#endif
      wr[4] = rcand;   // dgetf2-style reciprocal 1/pivot
    }
    STRIP_MARK(12);
    G.sync();
    STRIP_MARK(13);
#if HPS_STRIP_REDUX2
    // Cross-warp arg-max on the lanes: lane w reads warp w's key, two redux.sync as above, the
    // winner is the lowest lane holding the maximum (keys are unique per row).
    const unsigned long long kw = lane < NWARP ? L.redk[buf * NWARP + lane] : 0ull;
    const unsigned khi = static_cast<unsigned>(kw >> 32);
    const unsigned kmhi = __reduce_max_sync(0xffffffffu, khi);
    const unsigned kmlo = __reduce_max_sync(0xffffffffu, khi == kmhi ? static_cast<unsigned>(kw) : 0u);
    const unsigned long long kb = (static_cast<unsigned long long>(kmhi) << 32) | kmlo;
    const int ww = __ffs(__ballot_sync(0xffffffffu, lane < NWARP && kw == kb)) - 1;
#else
    unsigned long long kb = L.redk[buf * NWARP];
    int ww = 0;
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) {
      const unsigned long long k = L.redk[buf * NWARP + w];
      if (k > kb) { kb = k; ww = w; }
    }
#endif
    const int pphys = 0x7FF - static_cast<int>(kb & 0x7FFull);
    const double* wr = L.wrow + (buf * NWARP + ww) * 8;
    const double2 p01 = *reinterpret_cast<const double2*>(wr);
    const double2 p23 = *reinterpret_cast<const double2*>(wr + 2);
    const double rpiv = wr[4];
    const double prow[4] = {p01.x, p01.y, p23.x, p23.y};
    pivrow[j] = pphys;
    pivval[j] = prow[j];
    STRIP_MARK(14);
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) {
      if (phys[s] == pphys) {
        active &= ~(1u << s);
#if HPS_STRIP_LEAN
        elig &= ~(1u << s);
#endif
      }
      if ((active >> s) & 1u) {
        const double l = x[s][j] * rpiv;
        x[s][j] = l;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          if (jj > j && jj < sw) x[s][jj] = fma(-l, prow[jj], x[s][jj]);
      }
    }
    STRIP_MARK(15);
  }
  // Row interchanges (bookkeeping only, in column order) and the pivot minimum, once per strip.
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= sw) break;
      const int col = e + j, pphys = pivrow[j];
      minpiv = fmin(minpiv, fabs(pivval[j]));
      const int q = L.iperm[pphys];
      const int pold = L.perm[col];
      L.perm[col] = (short)pphys;
      L.perm[q] = (short)pold;
      L.iperm[pphys] = (short)col;
      L.iperm[pold] = (short)q;
    }
  }
  PHASE_MARK(9);
#pragma unroll
  for (int s = 0; s < NSLOT; ++s) {
    if (phys[s] == 0x7FFF) continue;
    double* dst = L.M + (size_t)phys[s] * L.ld + e;
    if (sw == 4) {
      st_v4(dst, x[s][0], x[s][1], x[s][2], x[s][3]);       // one 32-byte segment per row
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < sw) dst[j] = x[s][j];
    }
  }
  G.sync();   // bar.sync orders the global stores for the CTA's readers
}

constexpr int XS = 36;  // stride of the in-panel h x nd blocks (== 4 mod 16: conflict-free B fragments)

// Recursive-LU update inside a panel: source columns [s0, s0+h) are factored,
// destination columns [d0, d0+nd) (d0 = s0+h) carry all earlier updates.
//   U part (rows s0..s0+h-1):  X = L_hh^{-1} X     one warp, column per lane, no barriers
//   L part (rows d0..R-1)   :  C -= A[:, src] X    DMMA m8n8k4, one 8-row group per warp
template <int H>
__device__ void panel_update_t(const Grp& G, const LeafCtx& L, int s0, int d0, int nd, long long* pc,
                               long long& t_phase, double* sbuf) {
  constexpr int NTILE = (H + 7) / 8;        // 8-wide DMMA column tiles (nd <= H)
  constexpr int UNR = H <= HPS_UNR4_MAXH ? 4 : 2;   // 8-row groups in flight per warp
  constexpr int KS = H / 4;                 // DMMA k-steps
  double* Ls = L.scratch;              // H x H   (stride XS)
  double* X = L.scratch + 32 * XS;     // H x 8*NTILE (stride XS), zero padded
  const int tid = G.tid, lane = tid & 31, warp = tid >> 5;
  // Ls (strictly lower part of the factored h x h block) and X (the block above the
  // destination columns) in 32-byte row segments: s0, d0 are multiples of 4.
  for (int e = tid; e < H * (H / 4); e += NT) {
    const int i = e / (H / 4), k = 4 * (e % (H / 4));
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (k < i) ld_v4(mrow(L, s0 + i) + s0 + k, v0, v1, v2, v3);
    double* q = Ls + i * XS + k;
    q[0] = k < i ? v0 : 0.0;
    q[1] = k + 1 < i ? v1 : 0.0;
    q[2] = k + 2 < i ? v2 : 0.0;
    q[3] = k + 3 < i ? v3 : 0.0;
  }
  for (int e = tid; e < H * 2 * NTILE; e += NT) {
    const int i = e / (2 * NTILE), j = 4 * (e % (2 * NTILE));
    const double* src = mrow(L, s0 + i) + d0 + j;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (j + 3 < nd) {
      ld_v4(src, v0, v1, v2, v3);
    } else if (j < nd) {
      v0 = src[0];
      if (j + 1 < nd) v1 = src[1];
      if (j + 2 < nd) v2 = src[2];
    }
    double* q = X + i * XS + j;
    q[0] = v0; q[1] = v1; q[2] = v2; q[3] = v3;
  }
  G.sync();
  if (warp == 0 && lane < nd) {  // U part: one column per lane, registers, no barriers
    double x[H];
#pragma unroll
    for (int i = 0; i < H; ++i) x[i] = X[i * XS + lane];
#pragma unroll
    for (int k = 0; k < H - 1; ++k)
#pragma unroll
      for (int i = k + 1; i < H; ++i) x[i] = fma(-Ls[i * XS + k], x[k], x[i]);
#pragma unroll
    for (int i = 0; i < H; ++i) X[i * XS + lane] = x[i];
  }
  G.sync();
  for (int e = tid; e < H * 2 * NTILE; e += NT) {
    const int i = e / (2 * NTILE), j = 4 * (e % (2 * NTILE));
    if (j >= nd) continue;
    double* dst = mrow(L, s0 + i) + d0 + j;
    const double* q = X + i * XS + j;
    if (j + 3 < nd) {
      st_v4(dst, q[0], q[1], q[2], q[3]);
    } else {
      for (int jj = 0; j + jj < nd; ++jj) dst[jj] = q[jj];
    }
  }
  PHASE_MARK(6);
  // L part with DMMA: rows logical [d0, R) in 8-row groups; each warp keeps UNR groups'
  // loads in flight before computing.
  const int g = lane >> 2, t = lane & 3;
  for (int base = d0 + 8 * warp; base < L.R; base += 8 * (NT / 32) * UNR) {
    double acc[UNR][NTILE][2];
    double a[UNR][KS];
    double* row[UNR];
    bool ok[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int r0 = base + 8 * (NT / 32) * u;
      const int r = r0 + g;
      ok[u] = r < L.R;
      row[u] = L.M + (size_t)L.perm[ok[u] ? r : min(r0, L.R - 1)] * L.ld;
#pragma unroll
      for (int ni = 0; ni < NTILE; ++ni) {
        const double2 c = *reinterpret_cast<const double2*>(row[u] + d0 + 8 * ni + 2 * t);
        acc[u][ni][0] = c.x;
        acc[u][ni][1] = c.y;
      }
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) a[u][kk] = -row[u][s0 + 4 * kk + t];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int ni = 0; ni < NTILE; ++ni)
          dmma(acc[u][ni][0], acc[u][ni][1], a[u][kk], X[(4 * kk + t) * XS + 8 * ni + g]);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (!ok[u]) continue;
#pragma unroll
      for (int ni = 0; ni < NTILE; ++ni) {
        const int c = 8 * ni + 2 * t;
        if (c + 1 < nd) {
          *reinterpret_cast<double2*>(row[u] + d0 + c) = make_double2(acc[u][ni][0], acc[u][ni][1]);
        } else if (c < nd) {
          row[u][d0 + c] = acc[u][ni][0];
        }
      }
      // the next base strip (columns d0..d0+3, rows d0..R-1) reads these from shared memory
      if (t < 2) {
        const int r = base + 8 * (NT / 32) * u + g;
        *reinterpret_cast<double2*>(sbuf + 4 * (r - d0) + 2 * t) = make_double2(acc[u][0][0], acc[u][0][1]);
      }
    }
  }
  __threadfence_block();
  G.sync();
  PHASE_MARK(7);
}

// Recursive-LU update inside a panel: source columns [s0, s0+h) are factored,
// destination columns [d0, d0+nd) (d0 = s0+h) carry all earlier updates.
//   U part (rows s0..s0+h-1):  X = L_hh^{-1} X     one warp, column per lane, registers
//   L part (rows d0..R-1)   :  C -= A[:, src] X    DMMA m8n8k4 over 8-row groups
__device__ void panel_update(const Grp& G, const LeafCtx& L, int s0, int h, int d0, int nd,
                             long long* pc, long long& t_phase, double* sbuf) {
  switch (h) {
    case 4: panel_update_t<4>(G, L, s0, d0, nd, pc, t_phase, sbuf); break;
    case 8: panel_update_t<8>(G, L, s0, d0, nd, pc, t_phase, sbuf); break;
    case 16: panel_update_t<16>(G, L, s0, d0, nd, pc, t_phase, sbuf); break;
    default: panel_update_t<32>(G, L, s0, d0, nd, pc, t_phase, sbuf); break;
  }
}

// Inverse of the unit-lower diagonal block of panel [c0, c0+w) -> Linv (64x64,
// identity-padded, row-major).  Warp w owns columns 8w..8w+7; the four lanes of a
// column hold 16 rows each in registers and step through k with a shuffle
// broadcast of X[k][j] -- no block barriers inside.
__device__ void panel_linv(const Grp& G, const LeafCtx& L, int c0, int w, double* linv) {
  double* Ls = L.scratch;             // 64 x 65
  const int tid = G.tid, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 64 * 16; e += NT) {
    const int i = e >> 4, k = 4 * (e & 15);
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (i < w && k < i) ld_v4(mrow(L, c0 + i) + c0 + k, v0, v1, v2, v3);   // c0 % 64 == 0
    double* q = Ls + i * 65 + k;
    q[0] = (i < w && k < i) ? v0 : 0.0;
    q[1] = (i < w && k + 1 < i) ? v1 : 0.0;
    q[2] = (i < w && k + 2 < i) ? v2 : 0.0;
    q[3] = (i < w && k + 3 < i) ? v3 : 0.0;
  }
  G.sync();
  // lane (jj, q): column j = jb + 8 warp + jj, rows i = 4 r + q (r < 16).  Rows interleaved by
  // quarter so the four quarters' Ls reads hit four different banks.
  for (int jb = 0; jb < 64; jb += 8 * NWARP) {
    const int j = jb + 8 * warp + (lane >> 2), q = lane & 3;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = (4 * r + q == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 63; ++k) {
      const double xk = __shfl_sync(0xffffffffu, x[k >> 2], (lane & ~3) | (k & 3));
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (4 * r + q > k) x[r] = fma(-Ls[(4 * r + q) * 65 + k], xk, x[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) linv[(4 * r + q) * 64 + j] = x[r];
  }
  G.sync();
}

template <int NSLOT>
__device__ void panel_factor(const Grp& G, const LeafCtx& L, int c0, int w, double& minpiv,
                             long long* pc, long long& t_phase) {
  double* sbuf = L.scratch + 2 * 32 * XS;   // R x 4 strip hand-off (after the update's Ls/X)
  bool handed = false;
  for (int e = c0; e < c0 + w;) {
    const int sw = min(4, c0 + w - e);
    base_strip<NSLOT>(G, L, e, sw, minpiv, handed ? sbuf : nullptr, pc, t_phase);
    PHASE_MARK(10);
    e += sw;
    const int done = e - c0;
    handed = false;
    if (done < w) {
      const int h = done & (-done);      // lowest set bit: recursive-LU schedule
      panel_update(G, L, e - h, h, e, min(h, c0 + w - e), pc, t_phase, sbuf);
      handed = true;
    }
  }
}

// ---------------------------------------------------------------------------
// Kernel
// ---------------------------------------------------------------------------
// lock_nt > 0 (lock-step multi-leaf kernel): before every panel all groups of the CTA meet
// at named barrier 15 (lock_nt threads), so the co-resident leaves factor their panels at
// the same time and run their tile jobs at the same time: the latency-bound panels' scalar
// FP64 work then does not queue behind the other leaves' DMMA streams.
__device__ __forceinline__ void lock_sync(int lock_nt) {
  if (lock_nt > 0) asm volatile("bar.sync 15, %0;\n" ::"r"(lock_nt) : "memory");
}

template <int NSLOT>
__device__ void process_leaf(const LuArgs& a, Smem* sm, const int leaf, const Grp G = Grp{(int)threadIdx.x, 0},
                             int lock_nt = 0) {
  const LeafDims d = a.d;
  LeafCtx L;
  L.M = a.ws + (size_t)leaf * d.leaf_stride;
  L.ld = d.ld;
  L.R = d.R;
  L.ni = d.ni;
  L.perm = sm->perm;
  L.iperm = sm->iperm;
  L.scratch = sm->pipe;
  L.wrow = &sm->wrow[0][0][0];
  L.redk = &sm->redk[0][0];
  double* Linv = a.linv + (size_t)leaf * d.nblk * 4096;
  short* perm_g = a.perm + (size_t)leaf * d.Rpad;
  // Entries past Rpad are read by masked-out tile rows (e.g. the D-row tiles start at ni, which
  // need not be 64-aligned): point them at a valid row so the gathers stay in bounds.
  for (int i = G.tid; i < MAX_RPAD; i += NT) {
    sm->perm[i] = i < d.Rpad ? (a.factor ? (short)i : perm_g[i]) : (short)(d.Rpad - 1);
    sm->iperm[i] = (short)i;   // only used while factoring (perm starts as the identity)
  }
  G.sync();
  double minpiv = INFINITY;  // meaningful on thread 0
  long long* pc = a.phase_cycles ? a.phase_cycles + (size_t)leaf * PHASE_SLOTS : nullptr;
  long long t_phase = clock64();
  const long long t_leaf0 = t_phase;
  unsigned long long ns_leaf0 = 0;
  if (pc && G.tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_leaf0));

  const double* M = L.M;
  const int ld = d.ld;
  const short* perm = sm->perm;
  auto lrow = [&](int base) {  // rows gathered through perm, starting at logical `base`
    return [=](int i) -> const double* { return M + (size_t)perm[base + i] * ld; };
  };

  // Crout-ordered blocked LU over 64-wide blocks J of A_ii:
  //   (b) L part of block column J   rows [c0, R)      -= L[:, 0:c0] U[0:c0, J]   (K = c0)
  //   (c) panel J factorisation (pivoting) + Linv_J
  //   (a) U part of block row J      cols right of J   = Linv_J (A - L[J, 0:c0] U[0:c0, :])
  // The U-part tiles of one block row are independent (no sequential block-row chain), and
  // the Linv_J product is fused into the tile epilogue (shared memory, no HBM round trip).
#ifdef HPS_EPI_MARKS
  long long epi_main = 0, epi_tail = 0, lpt_main = 0, lpt_tail = 0, njobs = 0;
#endif
  for (int J = 0; J < d.nblk; ++J) {
    const int c0 = 64 * J;
    const int w = min(64, d.ni - c0);
    if (a.factor) {
      for (int rt = c0; rt < d.R; rt += TLM) {
        const int nr = min(TLM, d.R - rt);
        auto crow = [=](int i) -> double* { return L.M + (size_t)perm[rt + i] * ld + c0; };
        Acc acc;
        auto init = [&](Acc& x) { acc_zero(x); if (HPS_LPF) acc_prefetch_l1<TileL>(crow, nr); };
        auto arow = lrow(rt);
        auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
        // columns c0 + w .. c0 + 63 of the last block are A_ii padding (zero): no DMMA there
#ifdef HPS_EPI_MARKS
        const long long tl0 = clock64();
#endif
        tile_mma<TileL>(G, acc, init, arow, brow, c0, -1.0, sm->pipe, sm->full, sm->empty, &sm->gchunk,
                        nr, HPS_NACT ? w : 64);
#ifdef HPS_EPI_MARKS
        const long long tl1 = clock64();
#endif
        acc_add<TileL>(acc, crow, nr);
        acc_store<TileL>(acc, crow, nr, 64);
#ifdef HPS_EPI_MARKS
        if (G.tid == 0) { lpt_main += tl1 - tl0; lpt_tail += clock64() - tl1; ++njobs; }
#endif
      }
      __threadfence_block();
      G.sync();
      lock_sync(lock_nt);
      PHASE_MARK(1);
      panel_factor<NSLOT>(G, L, c0, w, minpiv, pc, t_phase);
      PHASE_MARK(2);
      panel_linv(G, L, c0, w, Linv + (size_t)J * 4096);
      PHASE_MARK(3);
    }
    const double* li = Linv + (size_t)J * 4096;
    const int ct_begin = a.factor ? c0 + 64 : d.tb0;
    const int ct_end = d.tb0 + 64 * d.ntb;
    for (int ct = ct_begin; ct < ct_end; ct += TUN) {
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[c0 + i] * ld + ct; };
      Acc acc;
#if HPS_UPF == 0
      auto init = [&](Acc& x) { acc_zero(x); acc_prefetch_l1<TileU>(crow, 64); };
#elif HPS_UPF == 1
      auto init = [&](Acc& x) { acc_zero(x); };
#else
      // keep Linv_J (32 KB, re-read by every tile of the block row) in L1 instead of the C tile
      auto init = [&](Acc& x) {
        acc_zero(x);
        const int wm_ = (G.tid >> 5) % TileU::WM, ln = threadIdx.x & 31;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(li + (32 * wm_ + ln) * 64));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(li + (32 * wm_ + ln) * 64 + 16));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(li + (32 * wm_ + ln) * 64 + 32));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(li + (32 * wm_ + ln) * 64 + 48));
      };
#endif
      auto arow = lrow(c0);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + ct; };
      // Real (non-padding) columns of this tile: A_ii columns end at ni, the trailing block
      // [A_ib | f] at tb0 + nb + 1; padding columns stay zero without DMMA work.
      const int real_end = ct + TUN > d.tb0 ? d.tb0 + d.nb + 1 : d.ni;
      const int nc = HPS_NACT ? min(TUN, real_end - ct) : TUN;
#ifdef HPS_EPI_MARKS
      const long long te0 = clock64();
#endif
      tile_mma<TileU>(G, acc, init, arow, brow, c0, -1.0, sm->pipe, sm->full, sm->empty, &sm->gchunk,
                      64, nc);
#ifdef HPS_EPI_MARKS
      const long long te1 = clock64();
#endif
      acc_add<TileU>(acc, crow, 64);
      linv_apply<TRI_LOWER>(G, acc, li, sm->pipe, nc);
      acc_store<TileU>(acc, crow, w, min(TUN, ct_end - ct));
#ifdef HPS_EPI_MARKS
      if (G.tid == 0) { epi_main += te1 - te0; epi_tail += clock64() - te1; }
#endif
    }
    __threadfence_block();
    G.sync();
    PHASE_MARK(0);
  }

#ifdef HPS_EPI_MARKS
  if (pc && G.tid == 0) { pc[11] += epi_main; pc[12] += epi_tail; pc[13] += lpt_main; pc[14] += lpt_tail; pc[15] += njobs; }
#endif
  // ---------------- D rows of the trailing columns ----------------
  // T = D_b - L21 U12 ; -w = 0 - L21 (L^{-1} f)      (K = ni)
  for (int tb = 0; tb < d.ntb; ++tb) {
    const int c0 = d.tb0 + 64 * tb;
    double* Tl = a.T_out + (size_t)leaf * d.nb * d.nb;
    double* wl = a.w_out + (size_t)leaf * d.nb;
    for (int rt = d.ni; rt < d.R; rt += TLM) {
      const int nr = min(TLM, d.R - rt);
      auto crow = [=](int i) -> double* { return L.M + (size_t)perm[rt + i] * ld + c0; };
      Acc acc;
      auto init = [&](Acc& x) { acc_zero(x); if (HPS_TPF) acc_prefetch_l1<TileL>(crow, nr); };
      auto arow = lrow(rt);
      auto brow = [=](int k) -> const double* { return M + (size_t)perm[k] * ld + c0; };
      tile_mma<TileL>(G, acc, init, arow, brow, d.ni, -1.0, sm->pipe, sm->full, sm->empty, &sm->gchunk,
                      nr, HPS_NACT ? d.nb + 1 - 64 * tb : 64);
      acc_add<TileL>(acc, crow, nr);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = acc_row<TileL>(mi);
        if (r >= nr) continue;
        const int trow = rt + r - d.ni;
#pragma unroll
        for (int ni2 = 0; ni2 < 4; ++ni2) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int tc = 64 * tb + acc_col<TileL>(ni2) + hh;
            if (tc < d.nb) Tl[(size_t)trow * d.nb + tc] = acc.v[mi][ni2][hh];
            else if (tc == d.nb) wl[trow] = -acc.v[mi][ni2][hh];
          }
        }
      }
    }
  }
  G.sync();
  PHASE_MARK(4);
  if (!a.factor) {
    G.sync();
    return;
  }
  G.sync();
  for (int i = G.tid; i < d.Rpad; i += NT) perm_g[i] = sm->perm[i];
  if (G.tid == 0) {
    if (pc) {   // whole-leaf clock64 cycles and globaltimer ns (effective SM clock)
      unsigned long long ns1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      pc[5] += clock64() - t_leaf0;
      pc[16] += (long long)(ns1 - ns_leaf0);
      pc[17] = blockIdx.x;
      pc[18] = smid;
    }
    const double nrm = a.norms[leaf];
    const double ratio = nrm > 0.0 ? minpiv / nrm : 0.0;
    if (a.minratio) a.minratio[leaf] = ratio;
    a.status[leaf] = (ratio >= 1e-12) ? 0 : 1;
  }
  G.sync();
}

// Persistent: grid = 2 CTAs per SM, each walks leaves blockIdx.x, +gridDim.x, ...
constexpr int CTAS_PER_SM = HPS_CTAS;

template <int NSLOT>
__global__ void __launch_bounds__(NT, CTAS_PER_SM) k2_lu_schur_kernel(LuArgs a, int n_leaves) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm->full[s], NT);
      mbar_init(&sm->empty[s], NT / 32);
    }
    sm->gchunk = 0;
  }
  __syncthreads();
  // Dynamic schedule (a.sched, zeroed before the launch): after its first leaf a CTA claims the
  // next unclaimed one.  The two CTAs sharing an SM do not progress at the same rate (one
  // persistently gets more of the DMMA pipe: 521 vs 693 ms of busy time for 16 leaves each at
  // C4, profiles/r02_k2_balance.log), so a static leaf split leaves the faster CTA idle for the
  // last ~12% of the launch.  A leaf's result does not depend on which CTA computes it.
  int leaf = blockIdx.x;
  while (leaf < n_leaves) {
    process_leaf<NSLOT>(a, sm, leaf);
    if (a.sched) {
      if (threadIdx.x == 0) sm->next_leaf = (int)gridDim.x + atomicAdd(a.sched, 1);
      __syncthreads();
      leaf = sm->next_leaf;
      __syncthreads();
    } else {
      leaf += gridDim.x;
    }
  }
}

// Lock-step multi-leaf kernel: one CTA per SM with CTAS_PER_SM groups of NT threads, each
// group a leaf (own shared-memory slice, pipeline mbarriers and named barrier 1 + group),
// all groups aligned before every panel (process_leaf lock_nt).  Groups without a leaf in
// the last round still meet the lock barriers (nblk of them per leaf of the round).
constexpr int NGRP = CTAS_PER_SM;
constexpr size_t SMEM_GRP = (sizeof(Smem) + 127) / 128 * 128;

template <int NSLOT>
__global__ void __launch_bounds__(NT * NGRP, 1) k2_lu_lockstep_kernel(LuArgs a, int n_leaves) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int grp = threadIdx.x / NT;
  Smem* sm = reinterpret_cast<Smem*>(smem_raw + grp * SMEM_GRP);
  const Grp G{gtid(), 1 + grp};
  if (G.tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm->full[s], NT);
      mbar_init(&sm->empty[s], NT / 32);
    }
    sm->gchunk = 0;
  }
  __syncthreads();
  const int per_round = gridDim.x * NGRP;
  for (int base = 0; base < n_leaves; base += per_round) {
    const int in_round = min(per_round, n_leaves - base);
    // leaves of this CTA in this round: base + blockIdx.x * NGRP + [0, NGRP) ∩ [0, in_round)
    const int first = blockIdx.x * NGRP;
    const int mine = max(0, min(NGRP, in_round - first));
    if (mine == 0) break;   // no later round has leaves for this CTA either
    const int lock_nt = NT * mine;
    if (grp < mine) process_leaf<NSLOT>(a, sm, base + first + grp, G, a.factor && mine > 1 ? lock_nt : 0);
  }
}


size_t lu_smem_bytes() { return sizeof(Smem); }

// ===========================================================================
// K3 (standalone): S_solve = -A_ii^{-1} A_ib = -U^{-1} (L^{-1} P A_ib)
// Runs after K2 on the same workspace.  Blocked back substitution over the 64-row blocks
// of U, last to first:  X_I = Uinv_I (Y_I - U[I, >I] X_{>I}),  X stored in place of Y
// (row k of X at the physical row of logical row k).  Uinv_I (upper, non-unit 64x64) is
// formed warp-synchronously like Linv; the GEMM and the Uinv product reuse the K2 tile
// code (64x128 tiles, DMMA).  Output row-major n_i x n_b per leaf.
// ===========================================================================
__device__ void block_uinv(const Grp& G, const double* M, const short* perm, int ld, int r0, int w,
                           double* Us, double* uinv) {
  const int tid = G.tid, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 64 * 64; e += NT) {
    const int i = e >> 6, k = e & 63;
    Us[i * 65 + k] = (i < w && k < w) ? (k >= i ? M[(size_t)perm[r0 + i] * ld + r0 + k] : 0.0)
                                      : (i == k ? 1.0 : 0.0);
  }
  G.sync();
  for (int jb = 0; jb < 64; jb += 8 * NWARP) {
    const int j = jb + 8 * warp + (lane >> 2), q = lane & 3;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = (4 * r + q == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 63; k >= 0; --k) {
      if (q == (k & 3)) x[k >> 2] = x[k >> 2] / Us[k * 65 + k];
      const double xk = __shfl_sync(0xffffffffu, x[k >> 2], (lane & ~3) | (k & 3));
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (4 * r + q < k) x[r] = fma(-Us[(4 * r + q) * 65 + k], xk, x[r]);
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) uinv[(4 * r + q) * 64 + j] = x[r];
  }
  __threadfence_block();
  G.sync();
}

__global__ void __launch_bounds__(NT, CTAS_PER_SM) k3_ssolve_kernel(LuArgs a, double* __restrict__ S_out,
                                                         double* __restrict__ uinv_ws, int n_leaves) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem* sm = reinterpret_cast<Smem*>(smem_raw);
  const Grp G{(int)threadIdx.x, 0};
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm->full[s], NT);
      mbar_init(&sm->empty[s], NT / 32);
    }
    sm->gchunk = 0;
  }
  __syncthreads();
  const LeafDims d = a.d;
  const int ld = d.ld;
  for (int leaf = blockIdx.x; leaf < n_leaves; leaf += gridDim.x) {
    double* Mw = a.ws + (size_t)leaf * d.leaf_stride;
    const double* M = Mw;
    const short* perm_g = a.perm + (size_t)leaf * d.Rpad;
    double* uinv = uinv_ws + (size_t)blockIdx.x * 4096;
    for (int i = threadIdx.x; i < MAX_RPAD; i += NT) sm->perm[i] = i < d.Rpad ? perm_g[i] : (short)(d.Rpad - 1);
    __syncthreads();
    const short* perm = sm->perm;
    const int sc = d.nb + a.s_with_load;   // S columns: A_ib (and the load column)
    const int ct_end = d.tb0 + sc;
    for (int I = d.nblk - 1; I >= 0; --I) {
      const int r0 = 64 * I, w = min(64, d.ni - r0);
      block_uinv(G, M, perm, ld, r0, w, sm->pipe, uinv);
      const int K = max(0, d.ni - r0 - 64);
      for (int ct = d.tb0; ct < ct_end; ct += TUN) {
        auto crow = [=](int i) -> double* { return Mw + (size_t)perm[r0 + i] * ld + ct; };
        auto arow = [=](int i) -> const double* { return M + (size_t)perm[r0 + i] * ld + r0 + 64; };
        auto brow = [=](int k) -> const double* { return M + (size_t)perm[r0 + 64 + k] * ld + ct; };
        Acc acc;
        auto init = [&](Acc& x) { acc_zero(x); acc_prefetch_l1<TileU>(crow, 64); };
        tile_mma<TileU>(G, acc, init, arow, brow, K, -1.0, sm->pipe, sm->full, sm->empty, &sm->gchunk);
        acc_add<TileU>(acc, crow, 64);
        linv_apply<TRI_UPPER>(G, acc, uinv, sm->pipe);
        acc_store<TileU>(acc, crow, w, min(TUN, ct_end - ct));
      }
      __threadfence_block();
      __syncthreads();
    }
    double* Sl = S_out + (size_t)leaf * d.ni * sc;
    for (int e = threadIdx.x; e < d.ni * sc; e += NT) {
      const int k = e / sc, c = e - sc * (e / sc);
      const double x = M[(size_t)perm[k] * ld + d.tb0 + c];
      Sl[e] = c < d.nb ? -x : x;   // S_solve = -A_ii^{-1} A_ib ; +A_ii^{-1} f_i
    }
    __syncthreads();
  }
}

void launch_ssolve(const LuArgs& a, double* S_out, double* uinv_ws, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  cudaFuncSetAttribute(k3_ssolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = n_leaves < CTAS_PER_SM * sms ? n_leaves : CTAS_PER_SM * sms;
  k3_ssolve_kernel<<<grid, NT, sizeof(Smem), st>>>(a, S_out, uinv_ws, n_leaves);
}

template <int NSLOT>
static void launch_ns(const LuArgs& a, int n_leaves, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (a.lockstep && a.factor) {
    const int smem = int(SMEM_GRP * NGRP);
    cudaFuncSetAttribute(k2_lu_lockstep_kernel<NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int need = (n_leaves + NGRP - 1) / NGRP;
    const int grid = need < sms ? need : sms;
    k2_lu_lockstep_kernel<NSLOT><<<grid, NT * NGRP, smem, st>>>(a, n_leaves);
    return;
  }
  cudaFuncSetAttribute(k2_lu_schur_kernel<NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(Smem));
  // Persistent grid = what is actually co-resident (a grid larger than that would leave
  // whole CTAs, each owning several leaves, waiting for a second wave).
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_lu_schur_kernel<NSLOT>, NT, sizeof(Smem));
  if (per_sm < 1) per_sm = 1;
  const int grid = n_leaves < per_sm * sms ? n_leaves : per_sm * sms;
  k2_lu_schur_kernel<NSLOT><<<grid, NT, sizeof(Smem), st>>>(a, n_leaves);
}

template <int NSLOT>
static int ctas_ns() {
  cudaFuncSetAttribute(k2_lu_schur_kernel<NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(Smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2_lu_schur_kernel<NSLOT>, NT, sizeof(Smem));
  return per_sm < 1 ? 1 : per_sm;
}

int lu_ctas_per_sm(const LeafDims& d) {
  const int need = (d.R + NT - 1) / NT;
  return need <= 2 ? ctas_ns<2>() : need <= 4 ? ctas_ns<4>() : ctas_ns<8>();
}

// Strip rows per thread = ceil(R / NT): register-resident pivot strips sized to p.
void launch_lu_schur(const LuArgs& a, int n_leaves, cudaStream_t st) {
  if (n_leaves <= 0) return;
  const int need = (a.d.R + NT - 1) / NT;
  if (need <= 2) launch_ns<2>(a, n_leaves, st);
  else if (need <= 4) launch_ns<4>(a, n_leaves, st);
  else launch_ns<8>(a, n_leaves, st);
}

}  // namespace HPS_CFG
}  // namespace hpsg
