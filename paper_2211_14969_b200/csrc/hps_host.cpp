// ============================================================================
//  hps_host.cpp — host runtime behind the C-ABI (include/hps_leaf_gpu.h).
//
//  Replaces the reference's CPU batching (proj/include/hps/parallel.hpp:25-58:
//  one std::thread worker per leaf) with one context per GPU that streams leaf
//  chunks through HBM:  H2D(b, f) -> K1 assemble -> K2/K3 LU+Schur -> D2H(T, w)
//  on three streams with double-buffered I/O, so copies overlap the FP64 work.
//  Chunk size is derived from the device budget (180 GB HBM on B200) and is a
//  multiple of the resident-CTA count (2 leaves per SM) so waves stay full.
//  Results never depend on chunking: every leaf is computed by one CTA with a
//  schedule that depends on p only.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "hps_kernels.h"
#include "hps_leaf_gpu.h"

using hpsg::LeafDims;

namespace {

constexpr int kMaxP = 45;

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    release();
    cudaError_t e = cudaMalloc(&ptr, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// Pinned host staging (the per-leaf status words): a D2H into caller memory that may be
// pageable would block the host thread inside the chunk loop and serialise the pipeline.
struct HostBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ~HostBuf() { release(); }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    release();
    cudaError_t e = cudaHostAlloc(&ptr, n, cudaHostAllocPortable);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// ---- 1-D Chebyshev primitives -------
// Same formulas and summation order as the CPU oracle (bit-identical tables).
void cheb_tables(int p, double a, std::vector<double>& Ds, std::vector<double>& D2) {
  std::vector<double> x(p);
  const double den = 2.0 * double(p - 1);
  for (int k = 0; k < p; ++k) x[k] = std::sin(M_PI * double(2 * k - (p - 1)) / den);
  std::vector<double> D(size_t(p) * p, 0.0);
  for (int i = 0; i < p; ++i) {
    const double ci = (i == 0 || i == p - 1) ? 2.0 : 1.0;
    double s = 0.0;
    for (int j = 0; j < p; ++j) {
      if (j == i) continue;
      const double cj = (j == 0 || j == p - 1) ? 2.0 : 1.0;
      const double sgn = ((i + j) & 1) ? -1.0 : 1.0;
      const double v = (ci / cj) * sgn / (x[i] - x[j]);
      D[size_t(i) * p + j] = v;
      s += v;
    }
    D[size_t(i) * p + i] = -s;
  }
  const double sc = 2.0 / a;
  Ds.resize(D.size());
  for (size_t i = 0; i < D.size(); ++i) Ds[i] = D[i] * sc;
  D2.assign(size_t(p) * p, 0.0);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int k = 0; k < p; ++k) s += Ds[size_t(i) * p + k] * Ds[size_t(k) * p + j];
      D2[size_t(i) * p + j] = s;
    }
}

int code(int y, int x, int kind, int edge = 0) { return y | (x << 8) | (kind << 16) | (edge << 18); }

void boundary_node(int k, int p, int* iy, int* ix, int* edge) {
  if (k < p) { *edge = 0; *iy = 0; *ix = k; return; }
  if (k < 2 * p - 1) { *edge = 1; *iy = k - p + 1; *ix = p - 1; return; }
  if (k < 3 * p - 2) { *edge = 2; *iy = p - 1; *ix = k - 2 * p + 1; return; }
  *edge = 3; *iy = k - 3 * p + 3; *ix = 0;
}

// Row/column codes of the augmented layout (hps_device.cuh).
void layout_codes(const LeafDims& d, bool solve, std::vector<int>& rows, std::vector<int>& cols) {
  const int p = d.p, q = p - 2;
  rows.assign(d.Rpad, code(0, 0, 3));
  cols.assign(d.ld, code(0, 0, 3));
  for (int r = 0; r < d.ni; ++r) rows[r] = code(r / q + 1, r % q + 1, 0);
  for (int c = 0; c < d.ni; ++c) cols[c] = code(c / q + 1, c % q + 1, 0);
  if (solve) {
    cols[d.tb0] = code(0, 0, 2);
    return;
  }
  for (int k = 0; k < d.nb; ++k) {
    int iy, ix, e;
    boundary_node(k, p, &iy, &ix, &e);
    rows[d.ni + k] = code(iy, ix, 1, e);
    cols[d.tb0 + k] = code(iy, ix, 1);
  }
  cols[d.tb0 + d.nb] = code(0, 0, 2);
}

LeafDims solve_dims(int p) {
  LeafDims d = hpsg::make_dims(p);
  d.nb = 0;
  d.R = d.ni;
  d.Rpad = (d.ni + 63) / 64 * 64;
  d.ld = (d.tb0 + 1 + 63) / 64 * 64;
  d.ntb = 1;
  d.leaf_stride = (long long)d.Rpad * d.ld;
  return d;
}

// ---- mesh tables ------------------
struct MeshHost {
  int nx, ny, p, n_edges;
  int64_t n_active, nnz;
  std::vector<int> elem_edges, edge_elems, edge_sides, edge_cols, edge_ne;
  std::vector<int64_t> edge_off;
};

MeshHost mesh_tables(int nx, int ny, int p) {
  MeshHost m;
  m.nx = nx; m.ny = ny; m.p = p;
  m.n_edges = (nx - 1) * ny + nx * (ny - 1);
  m.n_active = int64_t(m.n_edges) * (p - 2);
  auto id_h = [&](int c, int ey) { return c * (2 * ny - 1) + (ey - 1); };
  auto id_v = [&](int ex, int ey) { return (ex - 1) * (2 * ny - 1) + (ny - 1) + ey; };
  m.elem_edges.assign(size_t(4) * nx * ny, -1);
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      int* s = &m.elem_edges[size_t(4) * (ey * nx + ex)];
      if (ey >= 1) s[0] = id_h(ex, ey);
      if (ex + 1 <= nx - 1) s[1] = id_v(ex + 1, ey);
      if (ey + 1 <= ny - 1) s[2] = id_h(ex, ey + 1);
      if (ex >= 1) s[3] = id_v(ex, ey);
    }
  m.edge_elems.assign(size_t(2) * m.n_edges, -1);
  m.edge_sides.assign(size_t(2) * m.n_edges, -1);
  for (int c = 0; c < nx; ++c)
    for (int ey = 1; ey < ny; ++ey) {
      const int id = id_h(c, ey);
      m.edge_elems[2 * id] = (ey - 1) * nx + c; m.edge_sides[2 * id] = 2;
      m.edge_elems[2 * id + 1] = ey * nx + c;   m.edge_sides[2 * id + 1] = 0;
    }
  for (int ex = 1; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      const int id = id_v(ex, ey);
      m.edge_elems[2 * id] = ey * nx + ex - 1; m.edge_sides[2 * id] = 1;
      m.edge_elems[2 * id + 1] = ey * nx + ex; m.edge_sides[2 * id + 1] = 3;
    }
  const int q = p - 2;
  m.edge_cols.assign(size_t(7) * m.n_edges, -1);
  m.edge_ne.assign(m.n_edges, 0);
  m.edge_off.assign(size_t(m.n_edges) + 1, 0);
  for (int ed = 0; ed < m.n_edges; ++ed) {
    int buf[8], n = 0;
    for (int t = 0; t < 2; ++t) {
      const int e = m.edge_elems[2 * ed + t];
      for (int s = 0; s < 4; ++s) {
        const int x = m.elem_edges[size_t(4) * e + s];
        if (x >= 0) buf[n++] = x;
      }
    }
    std::sort(buf, buf + n);
    n = int(std::unique(buf, buf + n) - buf);
    for (int i = 0; i < n; ++i) m.edge_cols[size_t(7) * ed + i] = buf[i];
    m.edge_ne[ed] = n;
    m.edge_off[ed + 1] = m.edge_off[ed] + int64_t(n) * q * q;
  }
  m.nnz = m.edge_off[m.n_edges];
  return m;
}

}  // namespace

// ============================================================================
struct hps_gpu_ctx {
  int device = 0;
  hps_leaf_desc desc{};
  LeafDims d{}, ds{};
  int sms = 148;
  int n_leaves = 0;
  int chunk = 0;
  int k2_ctas = 2;               // co-resident K2 CTAs per SM (occupancy query at create)
  int io_pieces = 4;             // host-buffer transfer pieces when the range fits (io_schedule)
  size_t per_leaf = 0;
  std::string err;
  double k2 = 0.0;
  DevBuf rowcode, colcode, rowcode_s, colcode_s, Ds, D2;
  DevBuf ws, linv, perm, norms, minratio, status, inject_all;
  DevBuf in_b[2], in_f[2], in_v[2], out_T[2], out_w[2], out_st[2], out_u[2], out_S[2], uinv;
  MeshHost mesh;
  DevBuf m_elem_edges, m_edge_elems, m_edge_sides, m_edge_cols, m_edge_ne, m_edge_off;
  cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in_ready[2]{}, ev_in_free[2]{}, ev_out_ready[2]{}, ev_out_free[2]{};
  // Last use of the shared device scratch (ws, linv, perm, norms, minratio) by any call,
  // on whichever stream it ran: device-resident calls run on the caller's stream, host-buffer
  // calls on s_comp, so every entry waits on it and every exit records it.
  cudaEvent_t ev_scratch = nullptr;
  std::vector<cudaEvent_t> tev;  // timing events, 3 per chunk (before K1, K1|K2, after K2)
  int tslots = 0;                // chunk triplets recorded since the last fold
  hps_gpu_timing_t tacc{};       // intervals folded out of the event ring since the last reset
  int tkernels = 0;              // kernels launched since the last reset
  float ms_scatter = 0.0f;
  hps_gpu_timing_t timing{};
  bool has_inject = false;
  // Lock-step multi-leaf K2 kernel (4 leaves per CTA, panels aligned): measured faster for
  // the 4-warp build (C2: 14.05 -> 13.25 ms), slower for the 8-warp build (C3/C4), so it runs
  // wherever the 4-warp build does.
  // Experiment knobs (phase timers, forced K2 build/path, K2s trace, no staging) exist only in
  // HPS_DEBUG_KNOBS builds (`make EXTRA=-DHPS_DEBUG_KNOBS`), read once at ctx creation.
  bool phase_timers = false;
  int lockstep_env = -1;
  int force_cfg = 0;
  int small_env = -1;
  bool k2s_trace = false;
  bool no_stage = false;
  bool no_direct = false;   // debug: D2H copies even for mapped pinned outputs
  DevBuf phase_buf;
  DevBuf sched;                  // persistent-K2 leaf-claim counter (LuArgs::sched)
  DevBuf field_off, field_cent;   // K0 crystal sampler: node offsets, centres
  DevBuf op_A, op_Dn, op_b, op_f, op_v, op_T, op_w, op_st, op_S, op_u;   // operator-path staging
  DevBuf k4_T, k4_w, k4_g, k4_vals, k4_rhs, k4_list;   // assemble_reduced (host buffers), persistent
  DevBuf rc_ua, rc_g, rc_b, rc_f, rc_v, rc_ul, rc_u, rc_st, rc_tab;   // reconstruct_full_solution
  DevBuf s_store;                 // HPS_STORAGE_S_SOLVE: [S_solve | A_ii^{-1} f] of every leaf
  DevBuf ls_v, ls_u, ls_st;       // stored-S_solve leaf_solve I/O
  bool s_solve() const { return desc.storage == HPS_STORAGE_S_SOLVE; }
  DevBuf res_flux, res_pl, res_pe, res_in;   // K6 residual scratch
  int store_e0 = -1, store_e1 = -1;
  HostBuf h_status;               // pinned staging of status[] (see HostBuf)
  HostBuf h_T[2], h_w[2];         // pinned staging of T/w pieces for pageable caller buffers
  HostBuf h_u[2];                 // same for leaf_solve's u

  ~hps_gpu_ctx() {
    for (auto e : tev) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
      if (ev_in_ready[i]) cudaEventDestroy(ev_in_ready[i]);
      if (ev_in_free[i]) cudaEventDestroy(ev_in_free[i]);
      if (ev_out_ready[i]) cudaEventDestroy(ev_out_ready[i]);
      if (ev_out_free[i]) cudaEventDestroy(ev_out_free[i]);
    }
    if (ev_scratch) cudaEventDestroy(ev_scratch);
    if (s_comp) cudaStreamDestroy(s_comp);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
  }
  int fail(int code, const std::string& m) {
    err = m;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* where) {
    return fail(HPS_ERR_CUDA, std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
  }
  hpsg::MeshDev mesh_dev() const {
    hpsg::MeshDev m;
    m.nx = mesh.nx; m.ny = mesh.ny; m.p = mesh.p; m.n_edges = mesh.n_edges;
    m.n_active = mesh.n_active;
    m.elem_edges = m_elem_edges.as<int>();
    m.edge_elems = m_edge_elems.as<int>();
    m.edge_sides = m_edge_sides.as<int>();
    m.edge_cols = m_edge_cols.as<int>();
    m.edge_ne = m_edge_ne.as<int>();
    m.edge_off = m_edge_off.as<int64_t>();
    return m;
  }
  cudaEvent_t timing_event(size_t i) {
    while (tev.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      tev.push_back(e);
    }
    return tev[i];
  }
};

#define CK(call)                                                  \
  do {                                                            \
    cudaError_t e__ = (call);                                     \
    if (e__ != cudaSuccess) return ctx->cuda_fail(e__, #call);    \
  } while (0)

namespace {

template <class T>
cudaError_t upload(DevBuf& b, const std::vector<T>& v) {
  cudaError_t e = b.ensure(std::max<size_t>(1, v.size() * sizeof(T)));
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  return cudaMemcpy(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

std::string id_list(const std::vector<int>& ids) {
  std::string s;
  for (size_t i = 0; i < ids.size() && i < 64; ++i) s += (i ? "," : "") + std::to_string(ids[i]);
  if (ids.size() > 64) s += ",...";
  return s;
}

int resonance_error(hps_gpu_ctx* ctx, const std::vector<int>& bad) {
  return ctx->fail(HPS_ERR_RESONANCE,
                   "ResonanceError: element " + std::to_string(bad.front()) +
                       ": interior block singular (pivot < 1e-12*||A_ii||_inf); failing elements [" +
                       id_list(bad) + "]");
}

void reset_timing(hps_gpu_ctx* ctx) {
  ctx->tslots = 0;
  ctx->tacc = hps_gpu_timing_t{};
  ctx->tkernels = 0;
  ctx->ms_scatter = 0.0f;
}

// Move the intervals of the recorded event triplets into ctx->tacc and empty the ring
// (synchronizes on the last recorded event).
void fold_timing(hps_gpu_ctx* ctx) {
  const int n = ctx->tslots;
  if (n == 0) return;
  hps_gpu_timing_t& t = ctx->tacc;
  cudaEventSynchronize(ctx->tev[3 * n - 1]);
  for (int c = 0; c < n; ++c) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ctx->tev[3 * c], ctx->tev[3 * c + 1]);
    cudaEventElapsedTime(&b, ctx->tev[3 * c + 1], ctx->tev[3 * c + 2]);
    t.ms_assemble += a;
    t.ms_lu_schur += b;
  }
  float span = 0;
  cudaEventElapsedTime(&span, ctx->tev[0], ctx->tev[3 * n - 1]);
  t.ms_total += span;
  t.chunks += n;
  ctx->tslots = 0;
}

// Timing-event slot for the next chunk.  The ring is bounded (kTimingSlots triplets): a
// long loop of device-resident calls that never resets folds it instead of growing it.
constexpr int kTimingSlots = 256;
int next_timing_slot(hps_gpu_ctx* ctx) {
  if (ctx->tslots >= kTimingSlots) fold_timing(ctx);
  return ctx->tslots++;
}

// Sum the per-chunk CUDA-event intervals recorded since the last reset.
void finish_timing(hps_gpu_ctx* ctx) {
  fold_timing(ctx);
  hps_gpu_timing_t t = ctx->tacc;
  t.kernels = ctx->tkernels;
  t.ms_scatter = ctx->ms_scatter;
  t.ms_total += t.ms_scatter;
  ctx->timing = t;
}

// K2 launch with the dynamic leaf schedule: the claim counter is zeroed on the launch stream
// (the persistent kernel falls back to a static split if the counter cannot be allocated).
static void launch_k2(hps_gpu_ctx* ctx, hpsg::LuArgs a, int n, cudaStream_t st, int force) {
  if (ctx->sched.ensure(sizeof(int)) == cudaSuccess &&
      cudaMemsetAsync(ctx->sched.ptr, 0, sizeof(int), st) == cudaSuccess)
    a.sched = ctx->sched.as<int>();
  hpsg::launch_lu_schur(a, n, st, force);
}

// Device pipeline for one chunk of `n` leaves starting at element e (K1 + K2).
bool use_small(const hps_gpu_ctx* ctx, bool need_factors) {
  if (ctx->small_env == 0 || need_factors || ctx->phase_timers) return false;
  return ctx->small_env == 1 ? hpsg::small_condense_supported(ctx->d.p)
                             : hpsg::small_condense_preferred(ctx->d.p);
}

void enqueue_condense_chunk(hps_gpu_ctx* ctx, int e, int n, const double* d_b, const double* d_f,
                            double* d_T, double* d_w, int* d_status, cudaStream_t st,
                            bool need_factors) {
  const LeafDims& d = ctx->d;
  const int* inj = ctx->has_inject ? ctx->inject_all.as<int>() + e : nullptr;
  const int ci = next_timing_slot(ctx);
  if (use_small(ctx, need_factors)) {
    // K2s: one kernel, assembly + norm + elimination + T/w/status (no workspace).
    ctx->tkernels += 1;
    cudaEventRecord(ctx->timing_event(3 * ci), st);
    cudaEventRecord(ctx->timing_event(3 * ci + 1), st);
    hpsg::SmallArgs a;
    a.Ds = ctx->Ds.as<double>();
    a.D2 = ctx->D2.as<double>();
    a.k2 = ctx->k2;
    a.b = d_b;
    a.f = d_f;
    a.T_out = d_T;
    a.w_out = d_w;
    a.status = d_status;
    a.minratio = ctx->minratio.as<double>();
    a.norms = ctx->norms.as<double>();
    a.inject = inj;
    const bool trace = ctx->k2s_trace;
    const int NW = hpsg::small_condense_warps(d.p), BW = hpsg::small_condense_block(d.p);
    const int NPB = (d.ni + BW - 1) / BW;
    const size_t ntr = size_t(3) * NPB * NW + NPB + 2 * NW + 1;
    if (trace) {
      ctx->phase_buf.ensure(ntr * 8);
      cudaMemsetAsync(ctx->phase_buf.ptr, 0, ntr * 8, st);
      a.trace = ctx->phase_buf.as<long long>();
    }
    hpsg::launch_small_condense(a, d.p, n, st);
    cudaEventRecord(ctx->timing_event(3 * ci + 2), st);
    if (trace) {
      std::vector<long long> h(ntr);
      cudaMemcpyAsync(h.data(), ctx->phase_buf.ptr, ntr * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      const long long* pub = h.data() + 3 * size_t(NPB) * NW;   // block published (owner)
      const long long* wst = pub + NPB;                          // warp start / after assembly
      const long long t0 = wst[0];
      long long asm_max = 0;
      for (int q = 0; q < NW; ++q) asm_max = std::max(asm_max, wst[NW + q] - wst[q]);
      const double per = NPB > 1 ? double(pub[NPB - 1] - pub[0]) / (NPB - 1) : 0.0;
      double wake = 0, bulk = 0;
      int nw = 0;
      for (int kb = 0; kb < NPB; ++kb)
        for (int q = 0; q < NW; ++q) {
          const long long r = h[3 * (size_t(kb) * NW + q)], e = h[3 * (size_t(kb) * NW + q) + 1];
          if (r == 0) continue;
          wake += double(r - pub[kb]);
          bulk += double(e - r);
          ++nw;
        }
      std::fprintf(stderr,
                   "[k2s trace p=%d NW=%d BW=%d] assembly %lld cyc, pivot blocks %d, period %.0f cyc/block "
                   "(%.0f/step), recv-publish %.0f, block body %.0f, total %lld cyc\n",
                   d.p, NW, BW, asm_max, NPB, per, per / BW, wake / std::max(1, nw), bulk / std::max(1, nw),
                   wst[2 * NW] - t0);
    }
    return;
  }
  ctx->tkernels += 3;
  cudaEventRecord(ctx->timing_event(3 * ci), st);
  hpsg::launch_assemble(d, ctx->rowcode.as<int>(), ctx->colcode.as<int>(), ctx->Ds.as<double>(),
                        ctx->D2.as<double>(), ctx->k2, d_b, d_f, ctx->ws.as<double>(),
                        ctx->norms.as<double>(), inj, n, st);
  cudaEventRecord(ctx->timing_event(3 * ci + 1), st);
  hpsg::LuArgs a;
  a.d = d;
  a.ws = ctx->ws.as<double>();
  a.linv = ctx->linv.as<double>();
  a.perm = ctx->perm.as<short>();
  a.norms = ctx->norms.as<double>();
  a.T_out = d_T;
  a.w_out = d_w;
  a.status = d_status;
  a.minratio = ctx->minratio.as<double>();
  a.factor = 1;
  a.lockstep = ctx->lockstep_env == 1 || (ctx->lockstep_env != 0 && hpsg::use_g128(d, ctx->force_cfg));
  a.inject = inj;
  if (ctx->phase_timers) {
    ctx->phase_buf.ensure(size_t(ctx->chunk) * hpsg::PHASE_SLOTS * sizeof(long long));
    cudaMemsetAsync(ctx->phase_buf.ptr, 0, size_t(n) * hpsg::PHASE_SLOTS * sizeof(long long), st);
    a.phase_cycles = ctx->phase_buf.as<long long>();
  }
  launch_k2(ctx, a, n, st, ctx->force_cfg);
  cudaEventRecord(ctx->timing_event(3 * ci + 2), st);
  if (ctx->phase_timers) {
    constexpr int NS = hpsg::PHASE_SLOTS;
    std::vector<long long> h(size_t(n) * NS);
    cudaMemcpyAsync(h.data(), ctx->phase_buf.ptr, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double sum[NS] = {0};
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < NS; ++k) sum[k] += double(h[size_t(i) * NS + k]);
    std::fprintf(stderr,
                 "[hps phase cycles/leaf] U-part %.3g  L-part %.3g  panel %.3g (strips %.3g [start %.3g "
                 "columns %.3g end %.3g] upd-U %.3g upd-L %.3g)  linv %.3g  trailing %.3g\n",
                 sum[0] / n, sum[1] / n,
                 (sum[2] + sum[8] + sum[9] + sum[10] + sum[6] + sum[7]) / n,
                 (sum[8] + sum[9] + sum[10]) / n, sum[8] / n, sum[9] / n, sum[10] / n, sum[6] / n,
                 sum[7] / n, sum[3] / n, sum[4] / n);
    if (sum[16] > 0)
      std::fprintf(stderr, "[hps leaf totals] cycles/leaf %.4g  ns/leaf %.4g  effective SM clock %.0f MHz\n",
                   sum[5] / n, sum[16] / n, 1e3 * sum[5] / sum[16]);
    if (sum[16] > 0) {   // busy time per CTA and per SM (load balance of the persistent grid)
      std::vector<double> cta(4096, 0.0), sm(512, 0.0);
      for (int i = 0; i < n; ++i) {
        cta[size_t(h[size_t(i) * NS + 17]) & 4095] += double(h[size_t(i) * NS + 16]);
        sm[size_t(h[size_t(i) * NS + 18]) & 511] += double(h[size_t(i) * NS + 16]);
      }
      auto stats = [](const std::vector<double>& v, double& mn, double& mean, double& mx) {
        mn = 1e300; mx = 0; mean = 0; int k = 0;
        for (double x : v) if (x > 0) { mn = std::min(mn, x); mx = std::max(mx, x); mean += x; ++k; }
        mean /= std::max(1, k);
      };
      double a0, a1, a2, b0, b1, b2;
      stats(cta, a0, a1, a2);
      stats(sm, b0, b1, b2);
      std::fprintf(stderr, "[hps balance] busy ms per CTA min %.2f mean %.2f max %.2f | per SM min %.2f mean %.2f max %.2f\n",
                   a0 * 1e-6, a1 * 1e-6, a2 * 1e-6, b0 * 1e-6, b1 * 1e-6, b2 * 1e-6);
    }
    if (sum[11] + sum[12] + sum[13] + sum[14] + sum[15] > 0)
      std::fprintf(stderr,
                   "[hps strip column cycles/leaf] keys+redux %.3g  publish %.3g  barrier %.3g  "
                   "select %.3g  update %.3g\n",
                   sum[11] / n, sum[12] / n, sum[13] / n, sum[14] / n, sum[15] / n);
  }
}

}  // namespace

// ============================================================================
extern "C" {

const char* hps_gpu_version(void) { return "hps_leaf_b200 0.2 (sm_100a, DMMA f64)"; }

double hps_gpu_fp64_peak_tflops(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return 0.0;
  return hpsg::measure_dmma_peak_tflops(device);
}

double hps_gpu_fp64_peak_tflops_sustained(int device, double seconds) {
  if (cudaSetDevice(device) != cudaSuccess) return 0.0;
  return hpsg::measure_dmma_peak_tflops(device, seconds > 0.0 ? seconds : 3.0);
}

void* hps_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return p;
}
void hps_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

static thread_local std::string g_create_error;

// ctx == NULL returns the message of the last failed hps_gpu_create on this thread.
const char* hps_gpu_last_error(const hps_gpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int hps_gpu_create(int device, const hps_leaf_desc* desc, hps_gpu_ctx** out) {
  if (!out || !desc) return HPS_ERR_PARAM;
  *out = nullptr;
  auto ctx = std::make_unique<hps_gpu_ctx>();
  auto reject = [&](int code, const std::string& m) {
    g_create_error = m;
    return code;
  };
  ctx->device = device;
  ctx->desc = *desc;
  const hps_leaf_desc& D = *desc;
  // ParameterError conventions: cheb_nodes p < 4, scale_to_interval a <= 0 (:66).
  if (D.p < 4 || D.p > kMaxP)
    return reject(HPS_ERR_PARAM, "ParameterError: p must be in [4, 45]");
  if (!(D.a > 0.0))
    return reject(HPS_ERR_PARAM, "ParameterError: a must be > 0");
  if (!(D.kappa >= 0.0) || !std::isfinite(D.kappa))
    return reject(HPS_ERR_PARAM, "ParameterError: kappa must be >= 0");
  if (D.nx < 1 || D.ny < 1)
    return reject(HPS_ERR_PARAM, "ParameterError: nx, ny must be >= 1");
  if (D.storage != HPS_STORAGE_RECOMPUTE && D.storage != HPS_STORAGE_STORE && D.storage != HPS_STORAGE_S_SOLVE)
    return reject(HPS_ERR_PARAM, "ParameterError: unknown storage policy");
  hps_gpu_ctx* c = ctx.get();
#ifdef HPS_DEBUG_KNOBS
  auto env_int = [](const char* k, int dflt) { const char* v = std::getenv(k); return v ? std::atoi(v) : dflt; };
  c->io_pieces = env_int("HPS_IO_PIECES", c->io_pieces);
  c->phase_timers = std::getenv("HPS_PHASE_TIMERS") != nullptr;
  c->lockstep_env = env_int("HPS_LOCKSTEP", -1);
  c->force_cfg = env_int("HPS_K2_CFG", 0);
  c->small_env = env_int("HPS_SMALL", -1);
  c->k2s_trace = std::getenv("HPS_K2S_TRACE") != nullptr;
  c->no_stage = std::getenv("HPS_NO_STAGE") != nullptr;
  c->no_direct = std::getenv("HPS_NO_DIRECT") != nullptr;
#endif
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return reject(HPS_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->d = hpsg::make_dims(D.p);
  c->ds = solve_dims(D.p);
  c->n_leaves = D.nx * D.ny;
  c->k2 = D.kappa * D.kappa;
  std::vector<double> Ds, D2;
  cheb_tables(D.p, D.a, Ds, D2);
  std::vector<int> rows, cols, rows_s, cols_s;
  layout_codes(c->d, false, rows, cols);
  layout_codes(c->ds, true, rows_s, cols_s);
  c->mesh = mesh_tables(D.nx, D.ny, D.p);

#undef CK
#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess)                                                             \
      return reject(HPS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)
  {
    CK(upload(c->Ds, Ds));
    CK(upload(c->D2, D2));
    CK(upload(c->rowcode, rows));
    CK(upload(c->colcode, cols));
    CK(upload(c->rowcode_s, rows_s));
    CK(upload(c->colcode_s, cols_s));
    CK(upload(c->m_elem_edges, c->mesh.elem_edges));
    CK(upload(c->m_edge_elems, c->mesh.edge_elems));
    CK(upload(c->m_edge_sides, c->mesh.edge_sides));
    CK(upload(c->m_edge_cols, c->mesh.edge_cols));
    CK(upload(c->m_edge_ne, c->mesh.edge_ne));
    CK(upload(c->m_edge_off, c->mesh.edge_off));
    CK(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_scratch, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&c->ev_in_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_in_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_out_ready[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_out_free[i], cudaEventDisableTiming));
    }
  }
  // Memory plan: per in-flight leaf = workspace + Linv + perm + scalars + 2x I/O.
  const LeafDims& d = c->d;
  const size_t pp = size_t(D.p) * D.p;
  const size_t io = (2 * pp + size_t(d.nb) * d.nb + 2 * d.nb + pp + 4) * sizeof(double);
  c->per_leaf = size_t(d.leaf_stride) * 8 + size_t(d.nblk) * 4096 * 8 + size_t(d.Rpad) * 2 + 32 +
                2 * io;
  size_t budget = size_t(D.workspace_bytes);
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    budget = size_t(double(fr) * 0.7);
  }
  const size_t s_bytes = D.storage == HPS_STORAGE_S_SOLVE
                             ? size_t(c->n_leaves) * size_t(d.ni) * size_t(d.nb + 1) * sizeof(double) : 0;
  if (s_bytes) {
    if (budget < s_bytes + c->per_leaf)
      return reject(HPS_ERR_PARAM, "ParameterError: storage policy 's_solve' needs " + std::to_string(s_bytes >> 20) +
                                       " MiB for the stored S_solve blocks; exceeds the device budget");
    budget -= s_bytes;
  }
  int chunk = int(std::min<size_t>(size_t(c->n_leaves), budget / c->per_leaf));
  c->k2_ctas = hpsg::lu_ctas_per_sm(d, c->force_cfg);
  const int slots = c->k2_ctas * c->sms;
  // Several chunks: make each a whole number of waves.  Everything resident: one chunk.
  if (chunk < c->n_leaves && chunk > slots) chunk = chunk / slots * slots;
  if (D.storage == HPS_STORAGE_STORE && chunk < c->n_leaves)
    return reject(HPS_ERR_PARAM, "ParameterError: storage policy 'store' needs the factors of all " +
                                     std::to_string(c->n_leaves) +
                                     " leaves resident; exceeds the device budget (use recompute)");
  if (chunk < 1)
    return reject(HPS_ERR_PARAM, "ParameterError: device budget below one leaf");
  c->chunk = chunk;
  {
    // + 2 rows of slack: 128-wide U tiles may read up to 64 doubles past the last row.
    CK(c->ws.ensure((size_t(chunk) * d.leaf_stride + 2 * size_t(d.ld)) * 8));
    CK(c->linv.ensure(size_t(chunk) * d.nblk * 4096 * 8));
    CK(c->perm.ensure(size_t(chunk) * d.Rpad * 2));
    CK(c->norms.ensure(size_t(chunk) * 8));
    CK(c->minratio.ensure(size_t(chunk) * 8));
    CK(c->status.ensure(size_t(chunk) * 4));
    CK(c->inject_all.ensure(size_t(c->n_leaves) * 4));
    if (s_bytes) CK(c->s_store.ensure(s_bytes));
    CK(cudaMemset(c->inject_all.ptr, 0, size_t(c->n_leaves) * 4));
    CK(cudaMemset(c->ws.ptr, 0, (size_t(chunk) * d.leaf_stride + 2 * size_t(d.ld)) * 8));
  }
  *out = ctx.release();
  return HPS_OK;
}
#undef CK
#define CK(call)                                                  \
  do {                                                            \
    cudaError_t e__ = (call);                                     \
    if (e__ != cudaSuccess) return ctx->cuda_fail(e__, #call);    \
  } while (0)

void hps_gpu_destroy(hps_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  delete ctx;
}

int hps_gpu_get_info(const hps_gpu_ctx* ctx, hps_gpu_info_t* out) {
  if (!ctx || !out) return HPS_ERR_PARAM;
  out->p = ctx->d.p;
  out->n_i = ctx->d.ni;
  out->n_b = ctx->d.nb;
  out->n_leaves = ctx->n_leaves;
  out->chunk_leaves = ctx->chunk;
  out->resident_ctas = ctx->k2_ctas * ctx->sms;
  out->workspace_bytes_per_leaf = int64_t(ctx->per_leaf);
  out->n_active = ctx->mesh.n_active;
  out->N = int64_t(ctx->desc.nx * (ctx->d.p - 1) + 1) * int64_t(ctx->desc.ny * (ctx->d.p - 1) + 1);
  return HPS_OK;
}

int hps_gpu_get_timing(hps_gpu_ctx* ctx, hps_gpu_timing_t* out) {
  if (!ctx || !out) return HPS_ERR_PARAM;
  cudaSetDevice(ctx->device);
  finish_timing(ctx);
  *out = ctx->timing;
  return HPS_OK;
}

int hps_gpu_reset_timing(hps_gpu_ctx* ctx) {
  if (!ctx) return HPS_ERR_PARAM;
  reset_timing(ctx);
  return HPS_OK;
}

int hps_gpu_set_option(hps_gpu_ctx* ctx, int32_t option, int32_t value) {
  if (!ctx) return HPS_ERR_PARAM;
  if (value < -1 || value > 1) return ctx->fail(HPS_ERR_PARAM, "ParameterError: option value must be -1, 0 or 1");
  switch (option) {
    case HPS_OPT_SMALL_KERNEL:
      if (value == 1 && !hpsg::small_condense_supported(ctx->d.p))
        return ctx->fail(HPS_ERR_PARAM, "ParameterError: the register-resident kernel needs 4 <= p <= 12");
      ctx->small_env = value;
      return HPS_OK;
    case HPS_OPT_LOCKSTEP:
      if (value == 1 && ctx->d.R > 640)
        return ctx->fail(HPS_ERR_PARAM, "ParameterError: the lock-step kernel needs (p-2)^2 + 4(p-1) <= 640");
      ctx->lockstep_env = value;
      return HPS_OK;
    default:
      return ctx->fail(HPS_ERR_PARAM, "ParameterError: unknown option");
  }
}

int hps_gpu_set_fault_injection(hps_gpu_ctx* ctx, const int32_t* elements, int32_t n) {
  if (!ctx) return HPS_ERR_PARAM;
  cudaSetDevice(ctx->device);
  std::vector<int> flags(ctx->n_leaves, 0);
  for (int i = 0; i < n; ++i)
    if (elements[i] >= 0 && elements[i] < ctx->n_leaves) flags[elements[i]] = 1;
  CK(cudaMemcpy(ctx->inject_all.ptr, flags.data(), flags.size() * 4, cudaMemcpyHostToDevice));
  ctx->has_inject = n > 0;
  return HPS_OK;
}

static int check_range(hps_gpu_ctx* ctx, int e0, int e1) {
  if (e0 < 0 || e1 > ctx->n_leaves || e0 > e1)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: element range [" + std::to_string(e0) + ", " +
                                        std::to_string(e1) + ") outside the mesh");
  return HPS_OK;
}

// Host-buffer transfer schedule (piece sizes, each <= chunk) so the H2D of piece i+1 and the
// D2H of piece i-1 overlap the compute of piece i.  Streaming (range > workspace chunk):
// full chunks, remainder last (measured best at C4: one-wave pieces lose more to per-launch
// imbalance than they save in exposed copies).  Range fits: a one-wave first piece (its H2D
// is exposed), a one-wave last piece (its D2H is exposed), the middle in >= io_pieces-2
// pieces of whole waves of resident CTAs (C2: e2e 134k -> 151k leaves/s).  'store' keeps one
// chunk (its factors stay resident).
static std::vector<int> io_schedule(int total, int chunk, int wave, int io_pieces, bool store) {
  std::vector<int> out;
  if (total <= 0) return out;
  wave = std::max(1, std::min(wave, chunk));
  if (store || io_pieces <= 1 || total > chunk) {
    for (int r = total; r > 0; r -= chunk) out.push_back(std::min(r, chunk));
    return out;
  }
  const int first = std::min(wave, total);
  const int last = std::min(wave, total - first);
  int mid = total - first - last;
  out.push_back(first);
  if (mid > 0) {
    const int nm = std::max((mid + chunk - 1) / chunk, std::max(1, io_pieces - 2));
    int piece = (mid + nm - 1) / nm;
    piece = std::min(chunk, (piece + wave - 1) / wave * wave);
    for (; mid > 0; mid -= piece) out.push_back(std::min(mid, piece));
    // fold a fragment shorter than half a wave into the previous middle piece
    if (out.size() > 2 && out.back() < wave / 2 && out[out.size() - 2] + out.back() <= chunk) {
      out[out.size() - 2] += out.back();
      out.pop_back();
    }
  }
  if (last > 0) out.push_back(last);
  return out;
}

// Host copy-out of a staged piece: split across threads above 8 MB (one thread's memcpy into
// freshly faulted pageable pages runs far below the host's memory bandwidth).
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t kMin = size_t(8) << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = int(std::min<size_t>(std::min(8u, hw), std::max<size_t>(1, bytes / kMin)));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t part = (bytes + nt - 1) / nt;
  std::vector<std::thread> th;
  size_t done = std::min(part, bytes);   // bytes from here on are copied by the calling thread
  try {
    for (int i = 1; i < nt; ++i) {
      const size_t o = size_t(i) * part;
      if (o >= bytes) break;
      th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                                        std::min(part, bytes - o)); });
      done = std::min(bytes, o + part);
    }
  } catch (...) {   // no thread could be started: nothing may propagate out of the C-ABI
  }
  std::memcpy(dst, src, std::min(part, bytes));
  if (done < bytes) std::memcpy(static_cast<char*>(dst) + done, static_cast<const char*>(src) + done,
                                bytes - done);
  for (auto& t : th) t.join();
}

static bool host_pinned(const void* ptr) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// HPS_STORAGE_S_SOLVE: K3 back-substitutes the factored chunk's [A_ib | f] columns into the
// resident store at the leaves' slots (element c0 .. c0 + n).
static void enqueue_s_store(hps_gpu_ctx* ctx, int c0, int n, cudaStream_t st) {
  const LeafDims& d = ctx->d;
  hpsg::LuArgs a3;
  a3.d = d;
  a3.ws = ctx->ws.as<double>();
  a3.perm = ctx->perm.as<short>();
  a3.s_with_load = 1;
  hpsg::launch_ssolve(a3, ctx->s_store.as<double>() + size_t(c0) * d.ni * (d.nb + 1), ctx->uinv.as<double>(), n,
                      st, ctx->force_cfg);
  ctx->tkernels += 1;
}

// Host-buffer condense pipeline.  dT_res/dw_res (device, nullable): keep every leaf's T/w
// resident in HBM at (e - e0) instead of the double-buffered staging (hps_gpu_condense_assemble
// runs K4 on them afterwards); T/w (host) may then be null (no D2H of T at all).
static int condense_pipeline(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, const double* f,
                             double* T, double* w, double* S, int32_t* status, double* dT_res, double* dw_res) {
  if (ctx->desc.storage == HPS_STORAGE_STORE && (e1 - e0) > ctx->chunk)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: store policy range exceeds resident factors");
  CK(cudaSetDevice(ctx->device));
  const LeafDims& d = ctx->d;
  const size_t pp = size_t(d.p) * d.p, nb2 = size_t(d.nb) * d.nb;
  const int chunk = ctx->chunk;
  for (int i = 0; i < 2; ++i) {
    CK(ctx->in_b[i].ensure(size_t(chunk) * pp * 8));
    CK(ctx->in_f[i].ensure(size_t(chunk) * pp * 8));
    if (!dT_res) {
      CK(ctx->out_T[i].ensure(size_t(chunk) * nb2 * 8));
      CK(ctx->out_w[i].ensure(size_t(chunk) * d.nb * 8));
    }
    CK(ctx->out_st[i].ensure(size_t(chunk) * 4));
    if (S && !ctx->s_solve()) CK(ctx->out_S[i].ensure(size_t(chunk) * d.ni * d.nb * 8));
  }
  if (S || ctx->s_solve()) CK(ctx->uinv.ensure(size_t(4 * ctx->sms) * 4096 * 8));
  const size_t nis = size_t(d.ni) * d.nb;
  const std::vector<int> pieces =
      io_schedule(e1 - e0, chunk, ctx->k2_ctas * ctx->sms, ctx->io_pieces,
                  ctx->desc.storage == HPS_STORAGE_STORE);
  CK(ctx->h_status.ensure(size_t(e1 - e0) * 4));
  // A D2H into pageable memory blocks the host thread until it completes, which would
  // serialise the pieces: pageable T/w land in pinned double buffers instead and are copied
  // out on the host while the next piece computes.
  const bool want_T = T != nullptr;
  const bool pinned_out = want_T && host_pinned(T) && host_pinned(w);
  const bool stage = want_T && !pieces.empty() && !ctx->no_stage && !pinned_out;
  // Pinned caller outputs mapped into the device address space: the register-resident K2s
  // (p <= 12) writes T/w straight into host memory as each leaf finishes (the north star's "S
  // blocks straight into pinned host memory"; C1 e2e 1.00M -> 1.19M leaves/s), so no D2H copy
  // trails the last piece.  The blocked K2's D-row epilogue stores are too scattered for the
  // host link (C2 e2e 145k -> 74k when tried): it keeps the staged D2H copies.
  double* T_map = nullptr;
  double* w_map = nullptr;
  if (pinned_out && !dT_res && !ctx->no_direct &&
      use_small(ctx, S != nullptr || ctx->desc.storage != HPS_STORAGE_RECOMPUTE)) {
    void* pt = nullptr;
    void* pw = nullptr;
    if (cudaHostGetDevicePointer(&pt, T, 0) == cudaSuccess && cudaHostGetDevicePointer(&pw, w, 0) == cudaSuccess) {
      T_map = static_cast<double*>(pt);
      w_map = static_cast<double*>(pw);
    } else {
      cudaGetLastError();
    }
  }
  if (stage) {
    const int maxp = *std::max_element(pieces.begin(), pieces.end());
    for (int i = 0; i < 2; ++i) {
      CK(ctx->h_T[i].ensure(size_t(maxp) * nb2 * 8));
      CK(ctx->h_w[i].ensure(size_t(maxp) * d.nb * 8));
    }
  }
  auto drain = [&](int ci, size_t off, int n) -> cudaError_t {
    cudaError_t e = cudaEventSynchronize(ctx->ev_out_free[ci & 1]);
    if (e != cudaSuccess) return e;
    par_memcpy(T + off * nb2, ctx->h_T[ci & 1].ptr, size_t(n) * nb2 * 8);
    std::memcpy(w + off * d.nb, ctx->h_w[ci & 1].ptr, size_t(n) * d.nb * 8);
    return cudaSuccess;
  };
  reset_timing(ctx);
  CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_scratch, 0));
  int c0 = e0;
  for (int ci = 0; ci < int(pieces.size()); c0 += pieces[ci], ++ci) {
    const int n = pieces[ci];
    const int k = ci & 1;
    const size_t off = size_t(c0 - e0);
    double* T_dst = stage ? ctx->h_T[k].as<double>() : want_T ? T + off * nb2 : nullptr;
    double* w_dst = stage ? ctx->h_w[k].as<double>() : want_T ? w + off * d.nb : nullptr;
    double* dT = dT_res ? dT_res + off * nb2 : T_map ? T_map + off * nb2 : ctx->out_T[k].as<double>();
    double* dw = dw_res ? dw_res + off * d.nb : w_map ? w_map + off * d.nb : ctx->out_w[k].as<double>();
    CK(cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_in_free[k], 0));
    CK(cudaMemcpyAsync(ctx->in_b[k].ptr, b + off * pp, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_h2d));
    CK(cudaMemcpyAsync(ctx->in_f[k].ptr, f + off * pp, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_h2d));
    CK(cudaEventRecord(ctx->ev_in_ready[k], ctx->s_h2d));
    CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_in_ready[k], 0));
    CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_out_free[k], 0));
    enqueue_condense_chunk(ctx, c0, n, ctx->in_b[k].as<double>(), ctx->in_f[k].as<double>(), dT, dw,
                           ctx->out_st[k].as<int>(), ctx->s_comp,
                           S != nullptr || ctx->desc.storage != HPS_STORAGE_RECOMPUTE);
    if (ctx->s_solve()) {   // K3 into the resident store: [S_solve | A_ii^{-1} f] of these leaves
      enqueue_s_store(ctx, c0, n, ctx->s_comp);
    } else if (S) {  // K3: S_solve from the factored workspace
      hpsg::LuArgs a3;
      a3.d = d;
      a3.ws = ctx->ws.as<double>();
      a3.perm = ctx->perm.as<short>();
      hpsg::launch_ssolve(a3, ctx->out_S[k].as<double>(), ctx->uinv.as<double>(), n, ctx->s_comp,
                          ctx->force_cfg);
      ctx->tkernels += 1;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_in_free[k], ctx->s_comp));
    CK(cudaEventRecord(ctx->ev_out_ready[k], ctx->s_comp));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_out_ready[k], 0));
    if (want_T && !T_map) {
      CK(cudaMemcpyAsync(T_dst, dT, n * nb2 * 8, cudaMemcpyDeviceToHost, ctx->s_d2h));
      CK(cudaMemcpyAsync(w_dst, dw, n * size_t(d.nb) * 8, cudaMemcpyDeviceToHost, ctx->s_d2h));
    }
    CK(cudaMemcpyAsync(ctx->h_status.as<int32_t>() + off, ctx->out_st[k].ptr, n * 4, cudaMemcpyDeviceToHost,
                       ctx->s_d2h));
    if (S && ctx->s_solve())   // the n_b S_solve columns of the stored (n_b + 1)-wide rows
      CK(cudaMemcpy2DAsync(S + off * nis, size_t(d.nb) * 8,
                           ctx->s_store.as<double>() + size_t(c0) * d.ni * (d.nb + 1), size_t(d.nb + 1) * 8,
                           size_t(d.nb) * 8, size_t(n) * d.ni, cudaMemcpyDeviceToHost, ctx->s_d2h));
    else if (S)
      CK(cudaMemcpyAsync(S + off * nis, ctx->out_S[k].ptr, n * nis * 8, cudaMemcpyDeviceToHost, ctx->s_d2h));
    CK(cudaEventRecord(ctx->ev_out_free[k], ctx->s_d2h));
    if (stage && ci > 0) CK(drain(ci - 1, off - size_t(pieces[ci - 1]), pieces[ci - 1]));
  }
  CK(cudaEventRecord(ctx->ev_scratch, ctx->s_comp));
  CK(cudaStreamSynchronize(ctx->s_d2h));
  CK(cudaStreamSynchronize(ctx->s_comp));
  if (stage) {
    const int last = int(pieces.size()) - 1;
    CK(drain(last, size_t(c0 - e0) - size_t(pieces[last]), pieces[last]));
  }
  std::memcpy(status, ctx->h_status.ptr, size_t(e1 - e0) * 4);
  finish_timing(ctx);
  if (ctx->desc.storage != HPS_STORAGE_RECOMPUTE) {
    ctx->store_e0 = e0;
    ctx->store_e1 = e1;
  }
  std::vector<int> bad;
  for (int i = 0; i < e1 - e0; ++i)
    if (status[i]) bad.push_back(e0 + i);
  if (!bad.empty()) return resonance_error(ctx, bad);
  return HPS_OK;
}

int hps_gpu_condense(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, const double* f,
                     double* T, double* w, double* S, int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e1)) return rc;
  if (!b || !f || !T || !w || !status) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  return condense_pipeline(ctx, e0, e1, b, f, T, w, S, status, nullptr, nullptr);
}

// batched_condense + assemble_reduced in one call with T resident in HBM:
// the host receives only the reduced system (CSR values + rhs) and, when asked, T/w.
int hps_gpu_condense_assemble(hps_gpu_ctx* ctx, const double* b, const double* f, const double* g_bnd,
                              double* values, double* rhs, double* T, double* w, int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (!b || !f || !g_bnd || !values || !rhs || !status || (!T) != (!w))
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer (T and w: both or neither)");
  CK(cudaSetDevice(ctx->device));
  const LeafDims& d = ctx->d;
  const size_t nl = size_t(ctx->n_leaves), nb = size_t(d.nb);
  const size_t ng = 2 * size_t(ctx->desc.nx * (d.p - 1) + 1) + 2 * size_t(ctx->desc.ny * (d.p - 1) + 1);
  const int64_t na = ctx->mesh.n_active, nnz = ctx->mesh.nnz;
  CK(ctx->k4_T.ensure(nl * nb * nb * 8));
  CK(ctx->k4_w.ensure(nl * nb * 8));
  CK(ctx->k4_g.ensure(ng * 8));
  CK(ctx->k4_vals.ensure(size_t(std::max<int64_t>(1, nnz)) * 8));
  CK(ctx->k4_rhs.ensure(size_t(std::max<int64_t>(1, na)) * 8));
  CK(cudaMemcpyAsync(ctx->k4_g.ptr, g_bnd, ng * 8, cudaMemcpyHostToDevice, ctx->s_comp));
  const int rc = condense_pipeline(ctx, 0, int(nl), b, f, T, w, nullptr, status, ctx->k4_T.as<double>(),
                                   ctx->k4_w.as<double>());
  if (rc != HPS_OK) return rc;   // resonance: the reduced system is not formed
  if (na == 0) return HPS_OK;
  cudaStream_t st = ctx->s_comp;
  cudaEvent_t t0 = ctx->timing_event(3 * kTimingSlots), t1 = ctx->timing_event(3 * kTimingSlots + 1);
  CK(cudaEventRecord(t0, st));
  hpsg::launch_reduced_values(ctx->mesh_dev(), ctx->k4_T.as<double>(), ctx->k4_w.as<double>(), ctx->k4_g.as<double>(),
                              ctx->k4_vals.as<double>(), ctx->k4_rhs.as<double>(), st, false);
  CK(cudaEventRecord(t1, st));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(values, ctx->k4_vals.ptr, size_t(nnz) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(rhs, ctx->k4_rhs.ptr, size_t(na) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, t0, t1);
  ctx->ms_scatter = ms;
  ctx->tkernels += 1;
  ctx->timing.ms_scatter = ms;
  ctx->timing.ms_total += ms;
  ctx->timing.kernels = ctx->tkernels;
  return HPS_OK;
}

int hps_gpu_condense_device(hps_gpu_ctx* ctx, int32_t e0, int32_t n, const double* d_b,
                            const double* d_f, double* d_T, double* d_w, int32_t* d_status,
                            void* stream) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e0 + n)) return rc;
  CK(cudaSetDevice(ctx->device));
  if (n > 0 && (!d_b || !d_f || !d_T || !d_w || !d_status))
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: null device buffer");
  const bool store = ctx->desc.storage == HPS_STORAGE_STORE;
  if (store && n > ctx->chunk)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: store policy range exceeds resident factors");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->s_comp;
  const LeafDims& d = ctx->d;
  const size_t pp = size_t(d.p) * d.p, nb2 = size_t(d.nb) * d.nb;
  if (ctx->s_solve()) CK(ctx->uinv.ensure(size_t(4 * ctx->sms) * 4096 * 8));
  CK(cudaStreamWaitEvent(st, ctx->ev_scratch, 0));
  for (int c0 = 0; c0 < n; c0 += ctx->chunk) {
    const int m = std::min(ctx->chunk, n - c0);
    enqueue_condense_chunk(ctx, e0 + c0, m, d_b + c0 * pp, d_f + c0 * pp, d_T + c0 * nb2,
                           d_w + size_t(c0) * d.nb, d_status + c0, st, ctx->desc.storage != HPS_STORAGE_RECOMPUTE);
    if (ctx->s_solve()) enqueue_s_store(ctx, e0 + c0, m, st);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(ctx->ev_scratch, st));
  // 'store' / 's_solve': the kept factors / S_solve blocks are now those of [e0, e0 + n).
  if (ctx->desc.storage != HPS_STORAGE_RECOMPUTE) {
    ctx->store_e0 = e0;
    ctx->store_e1 = e0 + n;
  }
  return HPS_OK;
}

int hps_gpu_sample_crystal(hps_gpu_ctx* ctx, int32_t e0, int32_t n, const double* centres, int32_t ncent,
                           double sigma, double depth, double* d_b, void* stream) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e0 + n)) return rc;
  if (!d_b || (ncent > 0 && !centres) || ncent < 0 || !(sigma > 0.0))
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: crystal sampler needs d_b, centres and sigma > 0");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->s_comp;
  const int p = ctx->d.p;
  const double a = ctx->desc.a;
  // off[k] = (x_k + 1) * (a / 2), x_k the ascending CGL nodes (problems.leaf_coords).
  std::vector<double> off(p);
  const double den = 2.0 * double(p - 1);
  for (int k = 0; k < p; ++k) off[k] = (std::sin(M_PI * double(2 * k - (p - 1)) / den) + 1.0) * (a / 2.0);
  CK(ctx->field_off.ensure(size_t(p) * 8));
  CK(ctx->field_cent.ensure(size_t(std::max(1, ncent)) * 16));
  CK(cudaMemcpyAsync(ctx->field_off.ptr, off.data(), size_t(p) * 8, cudaMemcpyHostToDevice, st));
  if (ncent > 0)
    CK(cudaMemcpyAsync(ctx->field_cent.ptr, centres, size_t(ncent) * 16, cudaMemcpyHostToDevice, st));
  hpsg::launch_crystal(p, ctx->desc.nx, a, ctx->field_off.as<double>(), ctx->field_cent.as<double>(), ncent,
                       1.0 / (sigma * sigma), depth, e0, n, d_b, st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));   // the host tables above are pageable temporaries
  return HPS_OK;
}

int hps_gpu_residual_device(hps_gpu_ctx* ctx, const double* d_b, const double* d_f, const double* d_u,
                            double* out, void* stream) {
  if (!ctx) return HPS_ERR_PARAM;
  if (!d_b || !d_f || !d_u || !out) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->s_comp;
  const int n = ctx->n_leaves, nb = ctx->d.nb;
  const int ne = ctx->mesh.n_edges;
  CK(ctx->res_flux.ensure(size_t(n) * nb * 8));
  CK(ctx->res_pl.ensure(size_t(n) * 16));
  CK(ctx->res_pe.ensure(size_t(std::max(1, ne)) * 8));
  hpsg::launch_residual(ctx->mesh_dev(), ctx->k2, ctx->D2.as<double>(), ctx->Ds.as<double>(), d_b, d_f, d_u,
                        ctx->res_flux.as<double>(), ctx->res_pl.as<double>(), ctx->res_pe.as<double>(), n, st);
  CK(cudaGetLastError());
  std::vector<double> pl(size_t(n) * 2), pe(size_t(std::max(0, ne)));
  CK(cudaMemcpyAsync(pl.data(), ctx->res_pl.ptr, pl.size() * 8, cudaMemcpyDeviceToHost, st));
  if (ne > 0) CK(cudaMemcpyAsync(pe.data(), ctx->res_pe.ptr, pe.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double ri = 0.0, fi = 0.0, rf = 0.0;   // fixed order: elements, then edges
  for (int e = 0; e < n; ++e) {
    ri += pl[2 * size_t(e)];
    fi += pl[2 * size_t(e) + 1];
  }
  for (int k = 0; k < ne; ++k) rf += pe[k];
  out[0] = ri;
  out[1] = rf;
  out[2] = fi;
  return HPS_OK;
}

int hps_gpu_residual(hps_gpu_ctx* ctx, const double* b, const double* f, const double* u, double* out) {
  if (!ctx) return HPS_ERR_PARAM;
  if (!b || !f || !u || !out) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  CK(cudaSetDevice(ctx->device));
  const size_t pp = size_t(ctx->d.p) * ctx->d.p, n = size_t(ctx->n_leaves);
  CK(ctx->res_in.ensure(3 * n * pp * 8));
  double* d = ctx->res_in.as<double>();
  CK(cudaMemcpyAsync(d, b, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_comp));
  CK(cudaMemcpyAsync(d + n * pp, f, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_comp));
  CK(cudaMemcpyAsync(d + 2 * n * pp, u, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_comp));
  return hps_gpu_residual_device(ctx, d, d + n * pp, d + 2 * n * pp, out, ctx->s_comp);
}

// One chunk of batched leaf_solve on device buffers (elements [c0, c0 + n), n <= chunk):
// recompute policy K1s [A_ii | f_i - A_ib v] -> K2 -> K5; store policy: rhs into the kept
// condense workspace -> K2 trailing-only -> K5.
static cudaError_t enqueue_leaf_solve_chunk(hps_gpu_ctx* ctx, int c0, int n, const double* d_b, const double* d_f,
                                            const double* d_v, double* d_u, int* d_st, cudaStream_t st) {
  const LeafDims& d = ctx->d;
  if (ctx->s_solve()) {   // K5s: one GEMV per leaf from the stored [S_solve | A_ii^{-1} f]
    const int slot = next_timing_slot(ctx);
    ctx->tkernels += 1;
    cudaEventRecord(ctx->timing_event(3 * slot), st);
    cudaEventRecord(ctx->timing_event(3 * slot + 1), st);
    hpsg::launch_stored_solve(d.p, ctx->s_store.as<double>() + size_t(c0) * d.ni * (d.nb + 1), d_v, d_u, n, st);
    cudaMemsetAsync(d_st, 0, size_t(n) * 4, st);
    cudaEventRecord(ctx->timing_event(3 * slot + 2), st);
    return cudaGetLastError();
  }
  const bool store = ctx->desc.storage == HPS_STORAGE_STORE;
  const int slot = next_timing_slot(ctx);
  ctx->tkernels += store ? 3 : 4;
  cudaEventRecord(ctx->timing_event(3 * slot), st);
  hpsg::LuArgs a;
  a.ws = ctx->ws.as<double>();
  a.linv = ctx->linv.as<double>();
  a.perm = ctx->perm.as<short>();
  a.norms = ctx->norms.as<double>();
  a.T_out = nullptr;
  a.w_out = nullptr;
  a.status = d_st;
  a.minratio = nullptr;
  LeafDims dsolve;
  if (store) {
    // Kept condense factors: rhs into column tb0, trailing-only LU pass.
    const size_t lo = size_t(c0 - ctx->store_e0);
    dsolve = d;
    dsolve.R = d.ni;
    dsolve.ntb = 1;
    a.ws += lo * d.leaf_stride;
    a.linv += lo * d.nblk * 4096;
    a.perm += lo * d.Rpad;
    hpsg::launch_write_rhs(d, d.tb0, ctx->D2.as<double>(), d_f,
                           d_v, a.ws, n, st);
    cudaMemsetAsync(a.status, 0, n * 4, st);
    a.factor = 0;
  } else {
    dsolve = ctx->ds;
    const int* inj = ctx->has_inject ? ctx->inject_all.as<int>() + c0 : nullptr;
    hpsg::launch_assemble_solve(dsolve, ctx->rowcode_s.as<int>(), ctx->colcode_s.as<int>(),
                                ctx->Ds.as<double>(), ctx->D2.as<double>(), ctx->k2,
                                d_b, d_f,
                                d_v, a.ws, ctx->norms.as<double>(), inj, n, st);
    a.factor = 1;
  }
  cudaEventRecord(ctx->timing_event(3 * slot + 1), st);
  a.d = dsolve;
  // (lock-step measured no faster for the leaf-solve factorisation: 10.63 vs 10.45 ms at C2)
  launch_k2(ctx, a, n, st, 0);
  hpsg::launch_backsolve(dsolve, a.ws, a.perm, d_v, d_u,
                         n, st);
  cudaEventRecord(ctx->timing_event(3 * slot + 2), st);
  return cudaGetLastError();
}

int hps_gpu_leaf_solve(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, const double* f,
                       const double* v, double* u, int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e1)) return rc;
  if (!b || !f || !v || !u || !status) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  if (ctx->desc.storage != HPS_STORAGE_RECOMPUTE && (e0 < ctx->store_e0 || e1 > ctx->store_e1))
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: store policy: no kept factors for [" +
                                        std::to_string(e0) + ", " + std::to_string(e1) + ")");
  CK(cudaSetDevice(ctx->device));
  const LeafDims& d = ctx->d;
  const size_t pp = size_t(d.p) * d.p, nb = size_t(d.nb);
  const int chunk = ctx->chunk;
  for (int i = 0; i < 2; ++i) {
    CK(ctx->in_b[i].ensure(size_t(chunk) * pp * 8));
    CK(ctx->in_f[i].ensure(size_t(chunk) * pp * 8));
    CK(ctx->in_v[i].ensure(size_t(chunk) * nb * 8));
    CK(ctx->out_u[i].ensure(size_t(chunk) * pp * 8));
    CK(ctx->out_st[i].ensure(size_t(chunk) * 4));
  }
  // Transfer pipeline granularity: at least ~4 chunks (whole waves of resident CTAs) so the
  // H2D of chunk i+1 and the D2H of chunk i-1 overlap the compute of chunk i even when the
  // whole range fits the workspace.  'store' keeps one chunk (its factors stay resident).
  int io_chunk = chunk;
  if (ctx->desc.storage != HPS_STORAGE_STORE) {
    const int slots = ctx->k2_ctas * ctx->sms;
    const int quarter = (e1 - e0 + 3) / 4;
    io_chunk = std::min(chunk, std::max(slots, (quarter + slots - 1) / slots * slots));
  }
  CK(ctx->h_status.ensure(size_t(e1 - e0) * 4));
  const bool stage = e1 > e0 && !ctx->no_stage && !host_pinned(u);   // see hps_gpu_condense
  if (stage)
    for (int i = 0; i < 2; ++i) CK(ctx->h_u[i].ensure(size_t(std::min(io_chunk, e1 - e0)) * pp * 8));
  auto drain = [&](int ci, size_t off, int n) -> cudaError_t {
    cudaError_t e = cudaEventSynchronize(ctx->ev_out_free[ci & 1]);
    if (e == cudaSuccess) par_memcpy(u + off * pp, ctx->h_u[ci & 1].ptr, size_t(n) * pp * 8);
    return e;
  };
  reset_timing(ctx);
  CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_scratch, 0));
  int ci = 0;
  for (int c0 = e0; c0 < e1; c0 += io_chunk, ++ci) {
    const int n = std::min(io_chunk, e1 - c0);
    const int k = ci & 1;
    const size_t off = size_t(c0 - e0);
    CK(cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_in_free[k], 0));
    if (!ctx->s_solve()) {   // the stored policy reads only v
      CK(cudaMemcpyAsync(ctx->in_b[k].ptr, b + off * pp, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_h2d));
      CK(cudaMemcpyAsync(ctx->in_f[k].ptr, f + off * pp, n * pp * 8, cudaMemcpyHostToDevice, ctx->s_h2d));
    }
    CK(cudaMemcpyAsync(ctx->in_v[k].ptr, v + off * nb, n * nb * 8, cudaMemcpyHostToDevice, ctx->s_h2d));
    CK(cudaEventRecord(ctx->ev_in_ready[k], ctx->s_h2d));
    CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_in_ready[k], 0));
    CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_out_free[k], 0));
    cudaStream_t st = ctx->s_comp;
    CK(enqueue_leaf_solve_chunk(ctx, c0, n, ctx->in_b[k].as<double>(), ctx->in_f[k].as<double>(),
                                ctx->in_v[k].as<double>(), ctx->out_u[k].as<double>(), ctx->out_st[k].as<int>(), st));
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_in_free[k], st));
    CK(cudaEventRecord(ctx->ev_out_ready[k], st));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_out_ready[k], 0));
    CK(cudaMemcpyAsync(stage ? ctx->h_u[k].as<double>() : u + off * pp, ctx->out_u[k].ptr, n * pp * 8,
                       cudaMemcpyDeviceToHost, ctx->s_d2h));
    CK(cudaMemcpyAsync(ctx->h_status.as<int32_t>() + off, ctx->out_st[k].ptr, n * 4, cudaMemcpyDeviceToHost,
                       ctx->s_d2h));
    CK(cudaEventRecord(ctx->ev_out_free[k], ctx->s_d2h));
    if (stage && ci > 0) CK(drain(ci - 1, off - size_t(io_chunk), io_chunk));
  }
  CK(cudaEventRecord(ctx->ev_scratch, ctx->s_comp));
  CK(cudaStreamSynchronize(ctx->s_d2h));
  CK(cudaStreamSynchronize(ctx->s_comp));
  if (stage) {
    const int last = ci - 1;
    const size_t loff = size_t(last) * io_chunk;
    CK(drain(last, loff, (e1 - e0) - int(loff)));
  }
  std::memcpy(status, ctx->h_status.ptr, size_t(e1 - e0) * 4);
  finish_timing(ctx);
  std::vector<int> bad;
  for (int i = 0; i < e1 - e0; ++i)
    if (status[i]) bad.push_back(e0 + i);
  if (!bad.empty()) return resonance_error(ctx, bad);
  return HPS_OK;
}

int hps_gpu_reduced_pattern(hps_gpu_ctx* ctx, int64_t* nnz, int64_t* row_ptr, int32_t* col_idx) {
  if (!ctx || !nnz) return HPS_ERR_PARAM;
  *nnz = ctx->mesh.nnz;
  if (!row_ptr) return HPS_OK;
  if (!col_idx) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null col_idx");
  CK(cudaSetDevice(ctx->device));
  const int64_t na = ctx->mesh.n_active;
  if (na == 0) {
    row_ptr[0] = 0;
    return HPS_OK;
  }
  DevBuf rp, ci;
  CK(rp.ensure(size_t(na + 1) * 8));
  CK(ci.ensure(size_t(std::max<int64_t>(1, ctx->mesh.nnz)) * 4));
  hpsg::launch_reduced_pattern(ctx->mesh_dev(), rp.as<int64_t>(), ci.as<int32_t>(), ctx->s_comp);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(row_ptr, rp.ptr, size_t(na + 1) * 8, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaMemcpyAsync(col_idx, ci.ptr, size_t(ctx->mesh.nnz) * 4, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaStreamSynchronize(ctx->s_comp));
  return HPS_OK;
}

int hps_gpu_scatter_indices(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, int64_t* slot, int64_t* row) {
  if (!ctx) return HPS_ERR_PARAM;
  if (e0 < 0 || e1 < e0 || e1 > ctx->n_leaves)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: element range out of bounds");
  if (e1 == e0) return HPS_OK;
  if (!slot || !row) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null output");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = e1 - e0, nb = 4 * (ctx->d.p - 1);
  DevBuf ds, dr;
  CK(ds.ensure(size_t(n * nb * nb) * 8));
  CK(dr.ensure(size_t(n * nb) * 8));
  hpsg::launch_scatter_indices(ctx->mesh_dev(), e0, int(n), ds.as<int64_t>(), dr.as<int64_t>(), ctx->s_comp);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(slot, ds.ptr, size_t(n * nb * nb) * 8, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaMemcpyAsync(row, dr.ptr, size_t(n * nb) * 8, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaStreamSynchronize(ctx->s_comp));
  return HPS_OK;
}

int hps_gpu_reduced_bsr_pattern(hps_gpu_ctx* ctx, int32_t* block_size, int64_t* nnzb,
                                int64_t* brow_ptr, int32_t* bcol_idx) {
  if (!ctx || !block_size || !nnzb) return HPS_ERR_PARAM;
  const int64_t q = ctx->d.p - 2;
  *block_size = int32_t(q);
  *nnzb = ctx->mesh.nnz / (q * q);
  if (!brow_ptr) return HPS_OK;
  if (!bcol_idx) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null bcol_idx");
  CK(cudaSetDevice(ctx->device));
  const int64_t nbr = ctx->mesh.n_active / q;
  if (nbr == 0) {
    brow_ptr[0] = 0;
    return HPS_OK;
  }
  DevBuf rp, ci;
  CK(rp.ensure(size_t(nbr + 1) * 8));
  CK(ci.ensure(size_t(std::max<int64_t>(1, *nnzb)) * 4));
  hpsg::launch_reduced_bsr_pattern(ctx->mesh_dev(), rp.as<int64_t>(), ci.as<int32_t>(), ctx->s_comp);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(brow_ptr, rp.ptr, size_t(nbr + 1) * 8, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaMemcpyAsync(bcol_idx, ci.ptr, size_t(*nnzb) * 4, cudaMemcpyDeviceToHost, ctx->s_comp));
  CK(cudaStreamSynchronize(ctx->s_comp));
  return HPS_OK;
}

static int assemble_reduced_device(hps_gpu_ctx* ctx, const double* d_T, const double* d_w,
                                   const double* d_g_bnd, double* d_values, double* d_rhs,
                                   void* stream, bool bsr) {
  if (!ctx) return HPS_ERR_PARAM;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->s_comp;
  hpsg::launch_reduced_values(ctx->mesh_dev(), d_T, d_w, d_g_bnd, d_values, d_rhs, st, bsr);
  CK(cudaGetLastError());
  return HPS_OK;
}

int hps_gpu_assemble_reduced_device(hps_gpu_ctx* ctx, const double* d_T, const double* d_w,
                                    const double* d_g_bnd, double* d_values, double* d_rhs,
                                    void* stream) {
  return assemble_reduced_device(ctx, d_T, d_w, d_g_bnd, d_values, d_rhs, stream, false);
}

int hps_gpu_assemble_reduced_bsr_device(hps_gpu_ctx* ctx, const double* d_T, const double* d_w,
                                        const double* d_g_bnd, double* d_bvalues, double* d_rhs,
                                        void* stream) {
  return assemble_reduced_device(ctx, d_T, d_w, d_g_bnd, d_bvalues, d_rhs, stream, true);
}

static int assemble_reduced_host(hps_gpu_ctx* ctx, const double* T, const double* w,
                                 const double* g_bnd, double* values, double* rhs, bool bsr) {
  if (!ctx || !T || !w || !g_bnd || !values || !rhs) return HPS_ERR_PARAM;
  CK(cudaSetDevice(ctx->device));
  const LeafDims& d = ctx->d;
  const size_t nl = size_t(ctx->n_leaves), nb = size_t(d.nb);
  const size_t ng = 2 * size_t(ctx->desc.nx * (d.p - 1) + 1) + 2 * size_t(ctx->desc.ny * (d.p - 1) + 1);
  const int64_t na = ctx->mesh.n_active, nnz = ctx->mesh.nnz;
  if (na == 0) return HPS_OK;
  CK(ctx->k4_T.ensure(nl * nb * nb * 8));
  CK(ctx->k4_w.ensure(nl * nb * 8));
  CK(ctx->k4_g.ensure(ng * 8));
  CK(ctx->k4_vals.ensure(size_t(nnz) * 8));
  CK(ctx->k4_rhs.ensure(size_t(na) * 8));
  cudaStream_t st = ctx->s_comp;
  CK(cudaMemcpyAsync(ctx->k4_T.ptr, T, nl * nb * nb * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->k4_w.ptr, w, nl * nb * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->k4_g.ptr, g_bnd, ng * 8, cudaMemcpyHostToDevice, st));
  reset_timing(ctx);
  cudaEvent_t t0 = ctx->timing_event(0), t1 = ctx->timing_event(1);
  cudaEventRecord(t0, st);
  hpsg::launch_reduced_values(ctx->mesh_dev(), ctx->k4_T.as<double>(), ctx->k4_w.as<double>(),
                              ctx->k4_g.as<double>(), ctx->k4_vals.as<double>(), ctx->k4_rhs.as<double>(), st,
                              bsr);
  cudaEventRecord(t1, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(values, ctx->k4_vals.ptr, size_t(nnz) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(rhs, ctx->k4_rhs.ptr, size_t(na) * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaEventElapsedTime(&ctx->ms_scatter, t0, t1);
  ctx->tkernels = 1;
  finish_timing(ctx);
  return HPS_OK;
}

int hps_gpu_assemble_reduced(hps_gpu_ctx* ctx, const double* T, const double* w,
                             const double* g_bnd, double* values, double* rhs) {
  return assemble_reduced_host(ctx, T, w, g_bnd, values, rhs, false);
}

int hps_gpu_assemble_reduced_bsr(hps_gpu_ctx* ctx, const double* T, const double* w,
                                 const double* g_bnd, double* bvalues, double* rhs) {
  return assemble_reduced_host(ctx, T, w, g_bnd, bvalues, rhs, true);
}

// ---------------------------------------------------------------------------
// reconstruct_full_solution on the device (K7 + batched leaf_solve).
// ---------------------------------------------------------------------------
int hps_gpu_reconstruct_device(hps_gpu_ctx* ctx, const double* d_u_active, const double* d_g_bnd,
                               const double* d_b, const double* d_f, double* d_u_full, double* d_u_leaf,
                               int32_t* d_status, void* stream) {
  if (!ctx) return HPS_ERR_PARAM;
  if (!d_u_active || !d_g_bnd || !d_b || !d_f || !d_u_full || !d_status)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: null device buffer");
  const int n = ctx->n_leaves;
  if (ctx->desc.storage != HPS_STORAGE_RECOMPUTE && (ctx->store_e0 > 0 || ctx->store_e1 < n))
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: store policy: no kept factors for the whole mesh");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->s_comp;
  const int p = ctx->d.p, nx = ctx->desc.nx, ny = ctx->desc.ny, nb = ctx->d.nb;
  const size_t pp = size_t(p) * p;
  // corner-policy tables: nodes and barycentric weights of the p-2 interior nodes
  std::vector<double> tab(size_t(2 * p), 0.0);
  {
    const double den = 2.0 * double(p - 1);
    for (int k = 0; k < p; ++k) tab[k] = std::sin(M_PI * double(2 * k - (p - 1)) / den);
    for (int j = 1; j <= p - 2; ++j) {
      double prod = 1.0;
      for (int k = 1; k <= p - 2; ++k)
        if (k != j) prod *= (tab[j] - tab[k]);
      tab[p + j - 1] = 1.0 / prod;
    }
  }
  CK(ctx->rc_tab.ensure(tab.size() * 8));
  CK(ctx->rc_v.ensure(size_t(n) * nb * 8));
  if (!d_u_leaf) {
    CK(ctx->rc_ul.ensure(size_t(n) * pp * 8));
    d_u_leaf = ctx->rc_ul.as<double>();
  }
  CK(cudaMemcpyAsync(ctx->rc_tab.ptr, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, st));
  CK(cudaStreamWaitEvent(st, ctx->ev_scratch, 0));
  hpsg::launch_leaf_boundary(p, nx, ny, 0, n, d_u_active, d_g_bnd, ctx->rc_v.as<double>(), st);
  for (int c0 = 0; c0 < n; c0 += ctx->chunk) {
    const int m = std::min(ctx->chunk, n - c0);
    CK(enqueue_leaf_solve_chunk(ctx, c0, m, d_b + size_t(c0) * pp, d_f + size_t(c0) * pp,
                                ctx->rc_v.as<double>() + size_t(c0) * nb, d_u_leaf + size_t(c0) * pp, d_status + c0,
                                st));
  }
  hpsg::launch_place(p, nx, ny, 0, n, d_u_leaf, d_u_full, st);
  hpsg::launch_corners(p, nx, ny, ctx->rc_tab.as<double>(), ctx->rc_tab.as<double>() + p, d_u_active, d_g_bnd,
                       d_u_full, st);
  ctx->tkernels += 3;
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_scratch, st));
  CK(cudaStreamSynchronize(st));   // the host tables above are temporaries
  return HPS_OK;
}

int hps_gpu_reconstruct(hps_gpu_ctx* ctx, const double* u_active, const double* g_bnd, const double* b,
                        const double* f, double* u_full, int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (!u_active || !g_bnd || !b || !f || !u_full || !status)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  CK(cudaSetDevice(ctx->device));
  const int p = ctx->d.p, n = ctx->n_leaves;
  const size_t pp = size_t(p) * p;
  const int64_t na = ctx->mesh.n_active;
  const int64_t Nx = int64_t(ctx->desc.nx) * (p - 1) + 1, Ny = int64_t(ctx->desc.ny) * (p - 1) + 1;
  const size_t ng = size_t(2 * Nx + 2 * Ny), N = size_t(Nx * Ny);
  CK(ctx->rc_ua.ensure(size_t(std::max<int64_t>(1, na)) * 8));
  CK(ctx->rc_g.ensure(ng * 8));
  CK(ctx->rc_b.ensure(size_t(n) * pp * 8));
  CK(ctx->rc_f.ensure(size_t(n) * pp * 8));
  CK(ctx->rc_u.ensure(N * 8));
  CK(ctx->rc_st.ensure(size_t(n) * 4));
  cudaStream_t st = ctx->s_comp;
  reset_timing(ctx);
  if (na > 0) CK(cudaMemcpyAsync(ctx->rc_ua.ptr, u_active, size_t(na) * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->rc_g.ptr, g_bnd, ng * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->rc_b.ptr, b, size_t(n) * pp * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->rc_f.ptr, f, size_t(n) * pp * 8, cudaMemcpyHostToDevice, st));
  const int rc = hps_gpu_reconstruct_device(ctx, ctx->rc_ua.as<double>(), ctx->rc_g.as<double>(),
                                            ctx->rc_b.as<double>(), ctx->rc_f.as<double>(), ctx->rc_u.as<double>(),
                                            nullptr, ctx->rc_st.as<int>(), st);
  if (rc != HPS_OK) return rc;
  CK(cudaMemcpyAsync(u_full, ctx->rc_u.ptr, N * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(status, ctx->rc_st.ptr, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  finish_timing(ctx);
  std::vector<int> bad;
  for (int i = 0; i < n; ++i)
    if (status[i]) bad.push_back(i);
  if (!bad.empty()) return resonance_error(ctx, bad);
  return HPS_OK;
}

// ---------------------------------------------------------------------------
// The reference's per-leaf operations on operators given as values:
// build_leaf_operator -> (A_loc, D_normal), condense_leaf(ops, f), leaf_solve(ops, ...).
// Synchronous, in sub-batches sized to a staging budget; K2/K3/K5 are the hot-path kernels.
// ---------------------------------------------------------------------------
static int op_batch(const hps_gpu_ctx* ctx, size_t bytes_per_leaf) {
  const size_t budget = size_t(2) << 30;   // 2 GB of operator staging per sub-batch
  return int(std::max<size_t>(1, std::min<size_t>(size_t(ctx->chunk), budget / std::max<size_t>(1, bytes_per_leaf))));
}

int hps_gpu_build_leaf_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* b, double* A_loc,
                                double* D_normal) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e1)) return rc;
  if (e1 == e0) return HPS_OK;
  if (!b || !A_loc || !D_normal) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  CK(cudaSetDevice(ctx->device));
  const int p = ctx->d.p;
  const size_t pp = size_t(p) * p, na = pp * pp, nd = 4 * size_t(p) * pp;
  const int sub = op_batch(ctx, (na + nd + pp) * 8);
  CK(ctx->op_A.ensure(size_t(sub) * na * 8));
  CK(ctx->op_Dn.ensure(size_t(sub) * nd * 8));
  CK(ctx->op_b.ensure(size_t(sub) * pp * 8));
  cudaStream_t st = ctx->s_comp;
  CK(cudaStreamWaitEvent(st, ctx->ev_scratch, 0));
  for (int c0 = e0; c0 < e1; c0 += sub) {
    const int n = std::min(sub, e1 - c0);
    const size_t off = size_t(c0 - e0);
    CK(cudaMemcpyAsync(ctx->op_b.ptr, b + off * pp, n * pp * 8, cudaMemcpyHostToDevice, st));
    hpsg::launch_leaf_operator(p, ctx->Ds.as<double>(), ctx->D2.as<double>(), ctx->k2, ctx->op_b.as<double>(),
                               ctx->op_A.as<double>(), ctx->op_Dn.as<double>(), n, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(A_loc + off * na, ctx->op_A.ptr, n * na * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(D_normal + off * nd, ctx->op_Dn.ptr, n * nd * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaEventRecord(ctx->ev_scratch, st));
  return HPS_OK;
}

// Shared body of condense_operator / leaf_solve_operator.
static int operator_pass(hps_gpu_ctx* ctx, bool solve, int32_t e0, int32_t e1, const double* A_loc,
                         const double* D_normal, const double* f, const double* v, double* T, double* w,
                         double* S, double* u, int32_t* status) {
  CK(cudaSetDevice(ctx->device));
  const LeafDims d = solve ? ctx->ds : ctx->d;
  const int p = d.p, nb = 4 * (p - 1);
  const size_t pp = size_t(p) * p, na = pp * pp, nd = 4 * size_t(p) * pp;
  const int sub = op_batch(ctx, (na + (solve ? 0 : nd) + 2 * pp + nb) * 8);
  CK(ctx->op_A.ensure(size_t(sub) * na * 8));
  if (!solve) CK(ctx->op_Dn.ensure(size_t(sub) * nd * 8));
  CK(ctx->op_f.ensure(size_t(sub) * pp * 8));
  CK(ctx->op_st.ensure(size_t(sub) * 4));
  if (solve) {
    CK(ctx->op_v.ensure(size_t(sub) * nb * 8));
    CK(ctx->op_u.ensure(size_t(sub) * pp * 8));
  } else {
    CK(ctx->op_T.ensure(size_t(sub) * nb * nb * 8));
    CK(ctx->op_w.ensure(size_t(sub) * nb * 8));
    if (S) {
      CK(ctx->op_S.ensure(size_t(sub) * d.ni * nb * 8));
      CK(ctx->uinv.ensure(size_t(4 * ctx->sms) * 4096 * 8));
    }
  }
  cudaStream_t st = ctx->s_comp;
  reset_timing(ctx);
  CK(cudaStreamWaitEvent(st, ctx->ev_scratch, 0));
  for (int c0 = e0; c0 < e1; c0 += sub) {
    const int n = std::min(sub, e1 - c0);
    const size_t off = size_t(c0 - e0);
    CK(cudaMemcpyAsync(ctx->op_A.ptr, A_loc + off * na, n * na * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->op_f.ptr, f + off * pp, n * pp * 8, cudaMemcpyHostToDevice, st));
    if (solve) CK(cudaMemcpyAsync(ctx->op_v.ptr, v + off * nb, n * size_t(nb) * 8, cudaMemcpyHostToDevice, st));
    else CK(cudaMemcpyAsync(ctx->op_Dn.ptr, D_normal + off * nd, n * nd * 8, cudaMemcpyHostToDevice, st));
    const int slot = next_timing_slot(ctx);
    cudaEventRecord(ctx->timing_event(3 * slot), st);
    hpsg::launch_gather_operator(d, solve, ctx->op_A.as<double>(), ctx->op_Dn.as<double>(), ctx->op_f.as<double>(),
                                 ctx->op_v.as<double>(), ctx->ws.as<double>(), ctx->norms.as<double>(), n, st);
    cudaEventRecord(ctx->timing_event(3 * slot + 1), st);
    hpsg::LuArgs a;
    a.d = d;
    a.ws = ctx->ws.as<double>();
    a.linv = ctx->linv.as<double>();
    a.perm = ctx->perm.as<short>();
    a.norms = ctx->norms.as<double>();
    a.T_out = solve ? nullptr : ctx->op_T.as<double>();
    a.w_out = solve ? nullptr : ctx->op_w.as<double>();
    a.status = ctx->op_st.as<int>();
    a.minratio = nullptr;
    a.factor = 1;
    a.lockstep = !solve && hpsg::use_g128(d, ctx->force_cfg);
    launch_k2(ctx, a, n, st, ctx->force_cfg);
    ctx->tkernels += 3;
    if (solve) {
      hpsg::launch_backsolve(d, a.ws, a.perm, ctx->op_v.as<double>(), ctx->op_u.as<double>(), n, st);
      ctx->tkernels += 1;
    } else if (S) {
      hpsg::launch_ssolve(a, ctx->op_S.as<double>(), ctx->uinv.as<double>(), n, st, ctx->force_cfg);
      ctx->tkernels += 1;
    }
    cudaEventRecord(ctx->timing_event(3 * slot + 2), st);
    CK(cudaGetLastError());
    if (solve) {
      CK(cudaMemcpyAsync(u + off * pp, ctx->op_u.ptr, n * pp * 8, cudaMemcpyDeviceToHost, st));
    } else {
      CK(cudaMemcpyAsync(T + off * nb * nb, ctx->op_T.ptr, n * size_t(nb) * nb * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(w + off * nb, ctx->op_w.ptr, n * size_t(nb) * 8, cudaMemcpyDeviceToHost, st));
      if (S)
        CK(cudaMemcpyAsync(S + off * d.ni * nb, ctx->op_S.ptr, n * size_t(d.ni) * nb * 8, cudaMemcpyDeviceToHost,
                           st));
    }
    CK(cudaMemcpyAsync(status + off, ctx->op_st.ptr, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaEventRecord(ctx->ev_scratch, st));
  finish_timing(ctx);
  // the kept LU factors (if any) were overwritten (a stored S_solve is not touched)
  if (ctx->desc.storage == HPS_STORAGE_STORE) ctx->store_e0 = ctx->store_e1 = -1;
  std::vector<int> bad;
  for (int i = 0; i < e1 - e0; ++i)
    if (status[i]) bad.push_back(e0 + i);
  if (!bad.empty()) return resonance_error(ctx, bad);
  return HPS_OK;
}

int hps_gpu_condense_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* A_loc,
                              const double* D_normal, const double* f, double* T, double* w, double* S,
                              int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e1)) return rc;
  if (e1 == e0) return HPS_OK;
  if (!A_loc || !D_normal || !f || !T || !w || !status)
    return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  return operator_pass(ctx, false, e0, e1, A_loc, D_normal, f, nullptr, T, w, S, nullptr, status);
}

int hps_gpu_leaf_solve_operator(hps_gpu_ctx* ctx, int32_t e0, int32_t e1, const double* A_loc, const double* f,
                                const double* v, double* u, int32_t* status) {
  if (!ctx) return HPS_ERR_PARAM;
  if (int rc = check_range(ctx, e0, e1)) return rc;
  if (e1 == e0) return HPS_OK;
  if (!A_loc || !f || !v || !u || !status) return ctx->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  return operator_pass(ctx, true, e0, e1, A_loc, nullptr, f, v, nullptr, nullptr, nullptr, u, status);
}

}  // extern "C"

// ============================================================================
// Leaf-range sharding across GPUs of one box (parallel.hpp:21-24,42-57;
// SPEC.md:291,317): one ctx per device entry, one host thread per ctx, contiguous element
// ranges balanced to +-1 leaf, each shard's outputs written into its disjoint slots of the
// caller's buffers.  No collective: the only cross-shard data are the interface edges whose
// two elements sit on different shards, summed on the host in the K4 order (bit-identical).
// A device may be listed more than once (several ctxs on one GPU, e.g. for tests).
// ============================================================================
struct hps_gpu_multi {
  std::vector<hps_gpu_ctx*> ctx;
  std::vector<int> lo, hi;          // leaf range of each shard (whole mesh)
  MeshHost mesh;
  int p = 0, nb = 0, n_leaves = 0;
  std::string err;
  ~hps_gpu_multi() {
    for (auto* c : ctx) hps_gpu_destroy(c);
  }
  int fail(int code, const std::string& m) {
    err = m;
    return code;
  }
};

namespace {

// Contiguous ranges of [e0, e1) over k shards, sizes balanced to +-1 (first shards larger).
void split_range(int e0, int e1, int k, std::vector<int>& lo, std::vector<int>& hi) {
  const int n = e1 - e0, base = n / k, rem = n % k;
  lo.assign(k, 0);
  hi.assign(k, 0);
  int a = e0;
  for (int i = 0; i < k; ++i) {
    lo[i] = a;
    a += base + (i < rem ? 1 : 0);
    hi[i] = a;
  }
}

// Runs fn(i) for every shard on its own thread (serially when threads cannot be started);
// returns the first nonzero return code in shard order.
template <class Fn>
std::vector<int> for_shards(int k, Fn&& fn) {
  std::vector<int> rc(k, HPS_OK);
  std::vector<std::thread> th;
  int started = 0;
  try {
    for (int i = 1; i < k; ++i, ++started) th.emplace_back([&, i] { rc[i] = fn(i); });
  } catch (...) {
  }
  if (k > 0) rc[0] = fn(0);
  for (int i = 1 + started; i < k; ++i) rc[i] = fn(i);
  for (auto& t : th) t.join();
  return rc;
}

// K4's entry arithmetic for one interface edge on the host (k4_values_kernel, same IEEE
// sequence: v = (0 + T_e0) + T_e1 over present terms; rhs = -((0 + w + sum T g) + ...)).
void host_edge_values(const MeshHost& m, const double* T, const double* w, const double* g_bnd, int ed,
                      double* values, double* rhs) {
  const int p = m.p, q = p - 2, nb = 4 * (p - 1);
  auto side_base = [p](int side) { return side == 0 ? 1 : side == 1 ? p : side == 2 ? 2 * p : 3 * p - 2; };
  const int ne = m.edge_ne[ed];
  const int64_t off = m.edge_off[ed];
  const int rowlen = ne * q;
  int el[2], sd[2], col_side[2][7];
  for (int t = 0; t < 2; ++t) {
    el[t] = m.edge_elems[2 * ed + t];
    sd[t] = m.edge_sides[2 * ed + t];
    for (int r = 0; r < 7; ++r) {
      col_side[t][r] = -1;
      if (r < ne)
        for (int s4 = 0; s4 < 4; ++s4)
          if (m.elem_edges[size_t(4) * el[t] + s4] == m.edge_cols[size_t(7) * ed + r]) col_side[t][r] = s4;
    }
  }
  for (int k = 0; k < q; ++k)
    for (int pos = 0; pos < rowlen; ++pos) {
      const int rank = pos / q, kk = pos - rank * q;
      double v = 0.0;
      for (int t = 0; t < 2; ++t) {
        const int sc = col_side[t][rank];
        if (sc < 0) continue;
        const int r = side_base(sd[t]) + k;
        v = v + T[(size_t(el[t]) * nb + r) * nb + side_base(sc) + kk];
      }
      values[off + int64_t(k) * rowlen + pos] = v;
    }
  const int Nx = m.nx * (p - 1) + 1, Ny = m.ny * (p - 1) + 1;
  for (int k = 0; k < q; ++k) {
    double acc = 0.0;
    for (int t = 0; t < 2; ++t) {
      const int e = el[t];
      const int r = side_base(sd[t]) + k;
      const double* Te = T + (size_t(e) * nb + r) * nb;
      acc = acc + w[size_t(e) * nb + r];
      const int ex = e % m.nx, ey = e / m.nx;
      for (int sc = 0; sc < 4; ++sc) {
        if (m.elem_edges[size_t(4) * e + sc] >= 0) continue;
        const double* gs;
        int base;
        switch (sc) {
          case 0: gs = g_bnd; base = ex * (p - 1); break;
          case 1: gs = g_bnd + 2 * Nx + Ny; base = ey * (p - 1); break;
          case 2: gs = g_bnd + Nx; base = ex * (p - 1); break;
          default: gs = g_bnd + 2 * Nx; base = ey * (p - 1); break;
        }
        for (int kk = 0; kk < q; ++kk) {
          const double prod = Te[side_base(sc) + kk] * gs[base + kk + 1];
          acc = acc + prod;
        }
      }
    }
    rhs[int64_t(ed) * q + k] = -acc;
  }
}

}  // namespace

extern "C" {

// ---- host-only pieces of the sharded path (no GPU needed) ----
int hps_shard_range(int32_t n, int32_t k, int32_t i, int32_t* lo, int32_t* hi) {
  if (n < 0 || k < 1 || i < 0 || i >= k || !lo || !hi) return HPS_ERR_PARAM;
  std::vector<int> L, H;
  split_range(0, n, k, L, H);
  *lo = L[i];
  *hi = H[i];
  return HPS_OK;
}

int hps_reduced_cut_edges(int32_t p, int32_t nx, int32_t ny, const int32_t* shard_lo, int32_t k, int32_t* edges,
                          int64_t* n_cut) {
  if (p < 4 || nx < 1 || ny < 1 || k < 1 || !shard_lo || !n_cut) return HPS_ERR_PARAM;
  const MeshHost mh = mesh_tables(nx, ny, p);
  auto shard = [&](int e) {
    int s = 0;
    while (s + 1 < k && e >= shard_lo[s + 1]) ++s;
    return s;
  };
  int64_t c = 0;
  for (int ed = 0; ed < mh.n_edges; ++ed)
    if (shard(mh.edge_elems[2 * ed]) != shard(mh.edge_elems[2 * ed + 1])) {
      if (edges) edges[c] = ed;
      ++c;
    }
  *n_cut = c;
  return HPS_OK;
}

int hps_reduced_host_edges(int32_t p, int32_t nx, int32_t ny, const int32_t* edges, int64_t n, const double* T,
                           const double* w, const double* g_bnd, double* values, double* rhs) {
  if (p < 4 || nx < 1 || ny < 1 || (n > 0 && (!edges || !T || !w || !g_bnd || !values || !rhs)))
    return HPS_ERR_PARAM;
  const MeshHost mh = mesh_tables(nx, ny, p);
  for (int64_t i = 0; i < n; ++i) {
    if (edges[i] < 0 || edges[i] >= mh.n_edges) return HPS_ERR_PARAM;
    host_edge_values(mh, T, w, g_bnd, edges[i], values, rhs);
  }
  return HPS_OK;
}

int hps_gpu_multi_create(const int32_t* devices, int32_t n_devices, const hps_leaf_desc* desc,
                         hps_gpu_multi** out) {
  if (!out || !desc || !devices || n_devices < 1) {
    g_create_error = "ParameterError: hps_gpu_multi_create needs >= 1 device and a descriptor";
    return HPS_ERR_PARAM;
  }
  *out = nullptr;
  auto m = std::make_unique<hps_gpu_multi>();
  const int n = desc->nx * desc->ny;
  const int k = std::min<int>(n_devices, std::max(1, n));
  m->ctx.assign(k, nullptr);
  split_range(0, n, k, m->lo, m->hi);
  // each ctx budgets for its own shard (the shard decides chunking; ctxs on one device
  // share its memory, so the default budget is split between them)
  std::vector<int> per_dev(k, 0);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) per_dev[i] += devices[j] == devices[i];
  std::vector<std::string> errs(k);
  for (int i = 0; i < k; ++i) {   // sequential: cudaMemGetInfo-based budgets see earlier ctxs
    hps_leaf_desc d = *desc;
    if (d.workspace_bytes == 0 && per_dev[i] > 1) {
      size_t fr = 0, tot = 0;
      cudaSetDevice(devices[i]);
      cudaMemGetInfo(&fr, &tot);
      const int remaining = [&] { int c = 0; for (int j = i; j < k; ++j) c += devices[j] == devices[i]; return c; }();
      d.workspace_bytes = int64_t(double(fr) * 0.7 / remaining);
    }
    const int rc = hps_gpu_create(devices[i], &d, &m->ctx[i]);
    if (rc != HPS_OK) {
      g_create_error = "shard " + std::to_string(i) + " (device " + std::to_string(devices[i]) + "): " +
                       g_create_error;
      return rc;
    }
  }
  m->mesh = mesh_tables(desc->nx, desc->ny, desc->p);
  m->p = desc->p;
  m->nb = 4 * (desc->p - 1);
  m->n_leaves = n;
  *out = m.release();
  return HPS_OK;
}

void hps_gpu_multi_destroy(hps_gpu_multi* m) { delete m; }

const char* hps_gpu_multi_last_error(const hps_gpu_multi* m) { return m ? m->err.c_str() : g_create_error.c_str(); }

int hps_gpu_multi_shards(const hps_gpu_multi* m, int32_t* lo, int32_t* hi) {
  if (!m) return HPS_ERR_PARAM;
  const int k = int(m->ctx.size());
  for (int i = 0; i < k && lo && hi; ++i) {
    lo[i] = m->lo[i];
    hi[i] = m->hi[i];
  }
  return k;
}

hps_gpu_ctx* hps_gpu_multi_ctx(hps_gpu_multi* m, int32_t shard) {
  if (!m || shard < 0 || shard >= int(m->ctx.size())) return nullptr;
  return m->ctx[shard];
}

// Resonance ids of all shards (status of the whole range) -> one message; other errors:
// the first failing shard's message.
static int multi_result(hps_gpu_multi* m, const std::vector<int>& rc, const int32_t* status, int e0, int e1) {
  for (size_t i = 0; i < rc.size(); ++i)
    if (rc[i] != HPS_OK && rc[i] != HPS_ERR_RESONANCE)
      return m->fail(rc[i], "shard " + std::to_string(i) + ": " + m->ctx[i]->err);
  std::vector<int> bad;
  for (int i = 0; status && i < e1 - e0; ++i)
    if (status[i]) bad.push_back(e0 + i);
  if (bad.empty()) return HPS_OK;
  return m->fail(HPS_ERR_RESONANCE,
                 "ResonanceError: element " + std::to_string(bad.front()) +
                     ": interior block singular (pivot < 1e-12*||A_ii||_inf); failing elements [" + id_list(bad) +
                     "]");
}

int hps_gpu_multi_condense(hps_gpu_multi* m, int32_t e0, int32_t e1, const double* b, const double* f, double* T,
                           double* w, int32_t* status) {
  if (!m) return HPS_ERR_PARAM;
  if (e0 < 0 || e1 > m->n_leaves || e0 > e1)
    return m->fail(HPS_ERR_PARAM, "ParameterError: element range outside the mesh");
  if (!b || !f || !T || !w || !status) return m->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  const int k = int(m->ctx.size());
  std::vector<int> lo, hi;
  split_range(e0, e1, k, lo, hi);
  const size_t pp = size_t(m->p) * m->p, nb = size_t(m->nb);
  const auto rc = for_shards(k, [&](int i) {
    const size_t o = size_t(lo[i] - e0);
    if (hi[i] == lo[i]) return int(HPS_OK);
    return hps_gpu_condense(m->ctx[i], lo[i], hi[i], b + o * pp, f + o * pp, T + o * nb * nb, w + o * nb, nullptr,
                            status + o);
  });
  return multi_result(m, rc, status, e0, e1);
}

int hps_gpu_multi_leaf_solve(hps_gpu_multi* m, int32_t e0, int32_t e1, const double* b, const double* f,
                             const double* v, double* u, int32_t* status) {
  if (!m) return HPS_ERR_PARAM;
  if (e0 < 0 || e1 > m->n_leaves || e0 > e1)
    return m->fail(HPS_ERR_PARAM, "ParameterError: element range outside the mesh");
  if (!b || !f || !v || !u || !status) return m->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  const int k = int(m->ctx.size());
  std::vector<int> lo, hi;
  split_range(e0, e1, k, lo, hi);
  const size_t pp = size_t(m->p) * m->p, nb = size_t(m->nb);
  const auto rc = for_shards(k, [&](int i) {
    const size_t o = size_t(lo[i] - e0);
    if (hi[i] == lo[i]) return int(HPS_OK);
    return hps_gpu_leaf_solve(m->ctx[i], lo[i], hi[i], b + o * pp, f + o * pp, v + o * nb, u + o * pp, status + o);
  });
  return multi_result(m, rc, status, e0, e1);
}

// assemble_reduced over shards: shard i runs K4 on the interface edges whose two elements
// both lie in its leaf range (its T/w slice on its device), copying those edges' CSR rows
// back; edges cut by a shard boundary are summed on the host in K4's order.
int hps_gpu_multi_assemble_reduced(hps_gpu_multi* m, const double* T, const double* w, const double* g_bnd,
                                   double* values, double* rhs) {
  if (!m) return HPS_ERR_PARAM;
  if (!T || !w || !g_bnd || !values || !rhs) return m->fail(HPS_ERR_PARAM, "ParameterError: null buffer");
  const MeshHost& mh = m->mesh;
  if (mh.n_active == 0) return HPS_OK;
  const int k = int(m->ctx.size()), q = m->p - 2;
  const size_t nb = size_t(m->nb);
  std::vector<int> shard_of(m->n_leaves);
  for (int i = 0; i < k; ++i)
    for (int e = m->lo[i]; e < m->hi[i]; ++e) shard_of[e] = i;
  std::vector<std::vector<int>> own(k);
  std::vector<int> cut;
  for (int ed = 0; ed < mh.n_edges; ++ed) {
    const int s0 = shard_of[mh.edge_elems[2 * ed]], s1 = shard_of[mh.edge_elems[2 * ed + 1]];
    if (s0 == s1) own[s0].push_back(ed);
    else cut.push_back(ed);
  }
  const size_t ng = 2 * size_t(mh.nx * (m->p - 1) + 1) + 2 * size_t(mh.ny * (m->p - 1) + 1);
  const auto rc = for_shards(k, [&](int i) -> int {
    hps_gpu_ctx* ctx = m->ctx[i];
    if (own[i].empty()) return HPS_OK;
    CK(cudaSetDevice(ctx->device));
    const size_t n = size_t(m->hi[i] - m->lo[i]);
    CK(ctx->k4_T.ensure(n * nb * nb * 8));
    CK(ctx->k4_w.ensure(n * nb * 8));
    CK(ctx->k4_g.ensure(ng * 8));
    CK(ctx->k4_vals.ensure(size_t(mh.nnz) * 8));
    CK(ctx->k4_rhs.ensure(size_t(mh.n_active) * 8));
    CK(ctx->k4_list.ensure(own[i].size() * 4));
    cudaStream_t st = ctx->s_comp;
    const size_t lo = size_t(m->lo[i]);
    CK(cudaMemcpyAsync(ctx->k4_T.ptr, T + lo * nb * nb, n * nb * nb * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->k4_w.ptr, w + lo * nb, n * nb * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->k4_g.ptr, g_bnd, ng * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->k4_list.ptr, own[i].data(), own[i].size() * 4, cudaMemcpyHostToDevice, st));
    // T/w of element e live at (e - lo): shift the base pointers (only own-edge elements are read)
    hpsg::launch_reduced_values(ctx->mesh_dev(), ctx->k4_T.as<double>() - lo * nb * nb,
                                ctx->k4_w.as<double>() - lo * nb, ctx->k4_g.as<double>(), ctx->k4_vals.as<double>(),
                                ctx->k4_rhs.as<double>(), st, false, ctx->k4_list.as<int>(), int(own[i].size()));
    CK(cudaGetLastError());
    // copy back maximal runs of consecutive own edges (CSR rows of consecutive edges are contiguous)
    const auto& L = own[i];
    for (size_t a = 0; a < L.size();) {
      size_t b2 = a + 1;
      while (b2 < L.size() && L[b2] == L[b2 - 1] + 1) ++b2;
      const int ea = L[a], eb = L[b2 - 1] + 1;
      const int64_t v0 = mh.edge_off[ea], v1 = mh.edge_off[eb];
      CK(cudaMemcpyAsync(values + v0, ctx->k4_vals.as<double>() + v0, size_t(v1 - v0) * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(rhs + int64_t(ea) * q, ctx->k4_rhs.as<double>() + int64_t(ea) * q, size_t(eb - ea) * q * 8,
                         cudaMemcpyDeviceToHost, st));
      a = b2;
    }
    CK(cudaStreamSynchronize(st));
    return HPS_OK;
  });
  for (int ed : cut) host_edge_values(mh, T, w, g_bnd, ed, values, rhs);
  for (int i = 0; i < k; ++i)
    if (rc[i] != HPS_OK) return m->fail(rc[i], "shard " + std::to_string(i) + ": " + m->ctx[i]->err);
  return HPS_OK;
}

}  // extern "C"
