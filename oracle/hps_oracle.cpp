// ============================================================================
//  hps_oracle.cpp — CPU restatement of the reference HPS leaf stage.
//  TEST INFRASTRUCTURE ONLY (header comment in hps_oracle.hpp says why).
//
//  Every function cites the SPEC.md lines it restates.  Compiled with
//  -ffp-contract=off so that assembly arithmetic is exactly the written
//  sequence of IEEE operations (the GPU assembly kernel uses explicit _rn
//  intrinsics for the same sequence, which makes A bit-identical).
// ============================================================================
#include "hps_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>

extern "C" {
// OpenBLAS bundled in the scipy wheel (32-bit integer LAPACK interface).
void scipy_dgetrf_(const int* m, const int* n, double* a, const int* lda, int* ipiv, int* info);
void scipy_dgetrs_(const char* tr, const int* n, const int* nrhs, const double* a, const int* lda,
                   const int* ipiv, double* b, const int* ldb, int* info, size_t);
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
                  const double* alpha, const double* a, const int* lda, const double* b,
                  const int* ldb, const double* beta, double* c, const int* ldc, size_t, size_t);
void scipy_dgemv_(const char* t, const int* m, const int* n, const double* alpha, const double* a,
                  const int* lda, const double* x, const int* incx, const double* beta, double* y,
                  const int* incy, size_t);
void scipy_openblas_set_num_threads(int);
}

namespace hpso {

// ---------------------------------------------------------------- chebyshev
// SPEC.md:44-52 (cheb_nodes), :32-33 (endpoints, ascending), :82 (exact symmetry).
std::vector<double> cheb_nodes(int p, bool allow_small) {
  if (p < (allow_small ? 2 : 4)) throw ParameterError("cheb_nodes: p must be >= 4");
  std::vector<double> x(p);
  const double den = 2.0 * double(p - 1);
  for (int k = 0; k < p; ++k) {
    const double m = double(2 * k - (p - 1));
    x[k] = std::sin(M_PI * m / den);
  }
  return x;
}

// SPEC.md:53-61 (cheb_diff_matrix), :84,89 (negative-sum diagonal).
std::vector<double> cheb_diff_matrix(const std::vector<double>& x) {
  const int p = int(x.size());
  std::vector<double> D(size_t(p) * p, 0.0);
  auto c = [p](int i) { return (i == 0 || i == p - 1) ? 2.0 : 1.0; };
  for (int i = 0; i < p; ++i) {
    double s = 0.0;
    for (int j = 0; j < p; ++j) {
      if (j == i) continue;
      const double sgn = ((i + j) & 1) ? -1.0 : 1.0;
      const double v = (c(i) / c(j)) * sgn / (x[i] - x[j]);
      D[size_t(i) * p + j] = v;
      s += v;
    }
    D[size_t(i) * p + i] = -s;
  }
  return D;
}

// SPEC.md:62-70.
std::vector<double> scale_to_interval(const std::vector<double>& D, double a) {
  if (!(a > 0.0)) throw ParameterError("scale_to_interval: a must be > 0");
  const double s = 2.0 / a;
  std::vector<double> out(D.size());
  for (size_t i = 0; i < D.size(); ++i) out[i] = D[i] * s;
  return out;
}

// ------------------------------------------------------------ leaf geometry
// SPEC.md:256,314 and SURVEY Appendix A.3-4.
LeafIndex leaf_index(int p) {
  LeafIndex L;
  L.p = p;
  L.n_i = (p - 2) * (p - 2);
  L.n_b = 4 * (p - 1);
  for (int iy = 1; iy <= p - 2; ++iy)
    for (int ix = 1; ix <= p - 2; ++ix) L.interior.push_back(iy * p + ix);
  auto add = [&](int iy, int ix, int edge) {
    L.boundary.push_back(iy * p + ix);
    L.bnd_edge.push_back(edge);
    const bool corner = (iy == 0 || iy == p - 1) && (ix == 0 || ix == p - 1);
    L.bnd_corner.push_back(corner ? 1 : 0);
  };
  for (int ix = 0; ix <= p - 1; ++ix) add(0, ix, 0);        // S
  for (int iy = 1; iy <= p - 1; ++iy) add(iy, p - 1, 1);    // E
  for (int ix = 0; ix <= p - 2; ++ix) add(p - 1, ix, 2);    // N
  for (int iy = 1; iy <= p - 2; ++iy) add(iy, 0, 3);        // W
  return L;
}

LeafConstants leaf_constants(int p, double a, double kappa) {
  if (p < 4) throw ParameterError("p must be >= 4");
  if (!(a > 0.0)) throw ParameterError("a must be > 0");
  if (!(kappa >= 0.0)) throw ParameterError("kappa must be >= 0");
  LeafConstants c;
  c.p = p;
  c.a = a;
  c.kappa = kappa;
  c.x = cheb_nodes(p);
  c.Ds = scale_to_interval(cheb_diff_matrix(c.x), a);
  c.D2.assign(size_t(p) * p, 0.0);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int k = 0; k < p; ++k) s += c.Ds[size_t(i) * p + k] * c.Ds[size_t(k) * p + j];
      c.D2[size_t(i) * p + j] = s;
    }
  c.idx = leaf_index(p);
  return c;
}

// Entry A_loc[l, m] of -(D2 (x) I) - (I (x) D2) - kappa^2 diag(b).
// The diagonal is evaluated as ((-D2[iy,iy]) - D2[ix,ix]) - (kappa^2 * b).
static inline double a_entry(const LeafConstants& c, const double* b, int l, int m) {
  const int p = c.p;
  const int iy = l / p, ix = l % p, jy = m / p, jx = m % p;
  if (l == m) {
    double v = -c.D2[size_t(iy) * p + iy];
    v = v - c.D2[size_t(ix) * p + ix];
    const double kb = (c.kappa * c.kappa) * b[l];
    return v - kb;
  }
  if (jx == ix) return -c.D2[size_t(iy) * p + jy];
  if (jy == iy) return -c.D2[size_t(ix) * p + jx];
  return 0.0;
}

// Outward normal derivative row at boundary position k, column m
// (S: -d/dy, E: +d/dx, N: +d/dy, W: -d/dx; corners use the owning edge).
static inline double dn_entry(const LeafConstants& c, int k, int m) {
  const int p = c.p;
  const int l = c.idx.boundary[k];
  const int iy = l / p, ix = l % p, jy = m / p, jx = m % p;
  switch (c.idx.bnd_edge[k]) {
    case 0: return jx == ix ? -c.Ds[size_t(iy) * p + jy] : 0.0;
    case 1: return jy == iy ? c.Ds[size_t(ix) * p + jx] : 0.0;
    case 2: return jx == ix ? c.Ds[size_t(iy) * p + jy] : 0.0;
    default: return jy == iy ? -c.Ds[size_t(ix) * p + jx] : 0.0;
  }
}

// SPEC.md:270-278.
void build_leaf_operator(const LeafConstants& c, const double* b, double* A_loc, double* Dn) {
  const int P = c.p * c.p;
  if (A_loc)
    for (int l = 0; l < P; ++l)
      for (int m = 0; m < P; ++m) A_loc[size_t(l) * P + m] = a_entry(c, b, l, m);
  if (Dn)
    for (int k = 0; k < c.idx.n_b; ++k)
      for (int m = 0; m < P; ++m) Dn[size_t(k) * P + m] = dn_entry(c, k, m);
}

// Column-major blocks of the interior rows.
static void build_blocks(const LeafConstants& c, const double* b, std::vector<double>& Aii,
                         std::vector<double>* Aib, std::vector<double>* Di, std::vector<double>* Db) {
  const int ni = c.idx.n_i, nb = c.idx.n_b;
  Aii.resize(size_t(ni) * ni);
  for (int j = 0; j < ni; ++j)
    for (int i = 0; i < ni; ++i)
      Aii[size_t(j) * ni + i] = a_entry(c, b, c.idx.interior[i], c.idx.interior[j]);
  if (Aib) {
    Aib->resize(size_t(ni) * nb);
    for (int j = 0; j < nb; ++j)
      for (int i = 0; i < ni; ++i)
        (*Aib)[size_t(j) * ni + i] = a_entry(c, b, c.idx.interior[i], c.idx.boundary[j]);
  }
  if (Di) {
    Di->resize(size_t(nb) * ni);
    for (int j = 0; j < ni; ++j)
      for (int k = 0; k < nb; ++k) (*Di)[size_t(j) * nb + k] = dn_entry(c, k, c.idx.interior[j]);
  }
  if (Db) {
    Db->resize(size_t(nb) * nb);
    for (int j = 0; j < nb; ++j)
      for (int k = 0; k < nb; ++k) (*Db)[size_t(j) * nb + k] = dn_entry(c, k, c.idx.boundary[j]);
  }
}

// LU with partial pivoting + resonance test.
// Test hook: inject_singular zeroes interior row 0 of A_ii before factoring, which
// deterministically produces a zero final pivot.
static int factor_aii(const LeafConstants& c, std::vector<double>& Aii, std::vector<int>& ipiv,
                      bool inject_singular, double* min_ratio) {
  const int ni = c.idx.n_i;
  if (inject_singular)
    for (int j = 0; j < ni; ++j) Aii[size_t(j) * ni] = 0.0;
  double norm_inf = 0.0;
  for (int i = 0; i < ni; ++i) {
    double s = 0.0;
    for (int j = 0; j < ni; ++j) s += std::fabs(Aii[size_t(j) * ni + i]);
    norm_inf = std::max(norm_inf, s);
  }
  ipiv.resize(ni);
  int info = 0;
  scipy_dgetrf_(&ni, &ni, Aii.data(), &ni, ipiv.data(), &info);
  double pmin = INFINITY;
  for (int k = 0; k < ni; ++k) pmin = std::min(pmin, std::fabs(Aii[size_t(k) * ni + k]));
  const double ratio = norm_inf > 0.0 ? pmin / norm_inf : 0.0;
  if (min_ratio) *min_ratio = ratio;
  if (info > 0 || !(ratio >= 1e-12)) return 1;
  return 0;
}

// SPEC.md:279-287.
int condense_leaf(const LeafConstants& c, const double* b, const double* f, double* T, double* w,
                  double* S, double* lu, int32_t* ipiv_out, bool inject_singular, double* min_ratio) {
  const int ni = c.idx.n_i, nb = c.idx.n_b;
  std::vector<double> Aii, Aib, Di, Db;
  build_blocks(c, b, Aii, &Aib, &Di, &Db);
  std::vector<int> ipiv;
  if (factor_aii(c, Aii, ipiv, inject_singular, min_ratio)) return 1;
  if (lu) std::memcpy(lu, Aii.data(), sizeof(double) * Aii.size());
  if (ipiv_out)
    for (int k = 0; k < ni; ++k) ipiv_out[k] = ipiv[k];
  int info = 0;
  const char N = 'N';
  // X = A_ii^{-1} A_ib ; S_solve = -X
  std::vector<double>& X = Aib;
  scipy_dgetrs_(&N, &ni, &nb, Aii.data(), &ni, ipiv.data(), X.data(), &ni, &info, 1);
  for (auto& v : X) v = -v;
  // T = D_b + D_i * S_solve
  const double one = 1.0;
  scipy_dgemm_(&N, &N, &nb, &nb, &ni, &one, Di.data(), &nb, X.data(), &ni, &one, Db.data(), &nb, 1, 1);
  for (int r = 0; r < nb; ++r)
    for (int cc = 0; cc < nb; ++cc) T[size_t(r) * nb + cc] = Db[size_t(cc) * nb + r];
  if (S)
    for (int i = 0; i < ni; ++i)
      for (int cc = 0; cc < nb; ++cc) S[size_t(i) * nb + cc] = X[size_t(cc) * ni + i];
  // w = D_i A_ii^{-1} f_i
  std::vector<double> y(ni);
  for (int i = 0; i < ni; ++i) y[i] = f[c.idx.interior[i]];
  const int onei = 1;
  scipy_dgetrs_(&N, &ni, &onei, Aii.data(), &ni, ipiv.data(), y.data(), &ni, &info, 1);
  const double zero = 0.0;
  scipy_dgemv_(&N, &nb, &ni, &one, Di.data(), &nb, y.data(), &onei, &zero, w, &onei, 1);
  return 0;
}

// SPEC.md:297-305.  rhs_i = f_i - sum_c A_ib[i,c] v[c] (c ascending), then
// interior = A_ii^{-1} rhs with stored ("store") or recomputed ("recompute") factors.
int leaf_solve(const LeafConstants& c, const double* b, const double* f, const double* v, double* u,
               const double* lu, const int32_t* ipiv_in, bool inject_singular) {
  const int ni = c.idx.n_i, nb = c.idx.n_b;
  std::vector<double> Aii;
  std::vector<int> ipiv(ni);
  if (lu) {
    Aii.assign(lu, lu + size_t(ni) * ni);
    for (int k = 0; k < ni; ++k) ipiv[k] = ipiv_in[k];
  } else {
    build_blocks(c, b, Aii, nullptr, nullptr, nullptr);
    if (factor_aii(c, Aii, ipiv, inject_singular, nullptr)) return 1;
  }
  std::vector<double> rhs(ni);
  for (int i = 0; i < ni; ++i) {
    double s = f[c.idx.interior[i]];
    for (int k = 0; k < nb; ++k) {
      const double a = a_entry(c, b, c.idx.interior[i], c.idx.boundary[k]);
      if (a != 0.0) s = s - a * v[k];
    }
    rhs[i] = s;
  }
  int info = 0;
  const char N = 'N';
  const int onei = 1;
  scipy_dgetrs_(&N, &ni, &onei, Aii.data(), &ni, ipiv.data(), rhs.data(), &ni, &info, 1);
  for (int i = 0; i < ni; ++i) u[c.idx.interior[i]] = rhs[i];
  for (int k = 0; k < nb; ++k) u[c.idx.boundary[k]] = v[k];
  return 0;
}

// ---------------------------------------------------------------- mesh
// Interior edges sorted by (x-midpoint, y-midpoint):
// column c contributes its ny-1 horizontal edges, then the ny vertical edges on x=(c+1)a.
static inline int id_h(int ny, int c, int ey) { return c * (2 * ny - 1) + (ey - 1); }
static inline int id_v(int ny, int ex, int ey) { return (ex - 1) * (2 * ny - 1) + (ny - 1) + ey; }

MeshIndex mesh_index(int nx, int ny, int p) {
  if (p < 4) throw ParameterError("p must be >= 4");
  if (nx < 1 || ny < 1) throw ParameterError("nx, ny must be >= 1");
  MeshIndex m;
  m.nx = nx;
  m.ny = ny;
  m.p = p;
  m.N = int64_t(nx * (p - 1) + 1) * int64_t(ny * (p - 1) + 1);
  m.n_edges = (nx - 1) * ny + nx * (ny - 1);
  m.n_active = int64_t(m.n_edges) * (p - 2);
  m.elem_edges.assign(size_t(4) * nx * ny, -1);
  m.edge_elems.assign(size_t(2) * m.n_edges, -1);
  m.edge_sides.assign(size_t(2) * m.n_edges, -1);
  for (int ey = 0; ey < ny; ++ey)
    for (int ex = 0; ex < nx; ++ex) {
      const int e = ey * nx + ex;
      int32_t* s = &m.elem_edges[size_t(4) * e];
      if (ey >= 1) s[0] = id_h(ny, ex, ey);
      if (ex + 1 <= nx - 1) s[1] = id_v(ny, ex + 1, ey);
      if (ey + 1 <= ny - 1) s[2] = id_h(ny, ex, ey + 1);
      if (ex >= 1) s[3] = id_v(ny, ex, ey);
    }
  // Adjacent elements per edge, lower element id first.
  for (int c = 0; c < nx; ++c)
    for (int ey = 1; ey < ny; ++ey) {
      const int id = id_h(ny, c, ey);
      m.edge_elems[2 * id] = (ey - 1) * nx + c;  m.edge_sides[2 * id] = 2;      // N side of lower
      m.edge_elems[2 * id + 1] = ey * nx + c;    m.edge_sides[2 * id + 1] = 0;  // S side of upper
    }
  for (int ex = 1; ex < nx; ++ex)
    for (int ey = 0; ey < ny; ++ey) {
      const int id = id_v(ny, ex, ey);
      m.edge_elems[2 * id] = ey * nx + ex - 1;   m.edge_sides[2 * id] = 1;      // E side of left
      m.edge_elems[2 * id + 1] = ey * nx + ex;   m.edge_sides[2 * id + 1] = 3;  // W side of right
    }
  return m;
}

// SPEC.md:115,118 (g = gy*(nx(p-1)+1) + gx; local l = iy*p + ix).
void element_node_index(const MeshIndex& m, int e, int64_t* out) {
  const int p = m.p, ex = e % m.nx, ey = e / m.nx;
  const int64_t Nx = int64_t(m.nx) * (p - 1) + 1;
  for (int iy = 0; iy < p; ++iy)
    for (int ix = 0; ix < p; ++ix)
      out[iy * p + ix] = (int64_t(ey) * (p - 1) + iy) * Nx + int64_t(ex) * (p - 1) + ix;
}

int64_t active_of_global(const MeshIndex& m, int64_t g) {
  const int p = m.p;
  const int64_t Nx = int64_t(m.nx) * (p - 1) + 1;
  const int64_t gx = g % Nx, gy = g / Nx;
  const int64_t rx = gx % (p - 1), ry = gy % (p - 1);
  const int64_t cx = gx / (p - 1), cy = gy / (p - 1);
  if (rx == 0 && ry != 0 && cx >= 1 && cx <= m.nx - 1)  // vertical interior line
    return int64_t(id_v(m.ny, int(cx), int(cy))) * (p - 2) + (ry - 1);
  if (ry == 0 && rx != 0 && cy >= 1 && cy <= m.ny - 1)  // horizontal interior line
    return int64_t(id_h(m.ny, int(cx), int(cy))) * (p - 2) + (rx - 1);
  return -1;
}

// ------------------------------------------------------------ assemble_reduced
static inline int side_base(int p, int side) {
  switch (side) {
    case 0: return 1;
    case 1: return p;
    case 2: return 2 * p;
    default: return 3 * p - 2;
  }
}

// Sorted union of the interior edges of the (one or two) elements adjacent to edge `ed`.
static int row_edges(const MeshIndex& m, int ed, int* out) {
  int n = 0;
  for (int t = 0; t < 2; ++t) {
    const int e = m.edge_elems[2 * ed + t];
    for (int s = 0; s < 4; ++s) {
      const int x = m.elem_edges[size_t(4) * e + s];
      if (x >= 0) out[n++] = x;
    }
  }
  std::sort(out, out + n);
  return int(std::unique(out, out + n) - out);
}

// CSR pattern of A~: columns sorted ascending, int64 row_ptr,
// int32 col_idx.
ReducedCSR reduced_pattern(const MeshIndex& m) {
  ReducedCSR r;
  const int q = m.p - 2;
  r.n = m.n_active;
  r.row_ptr.assign(size_t(r.n) + 1, 0);
  int buf[8];
  for (int ed = 0; ed < m.n_edges; ++ed) {
    const int ne = row_edges(m, ed, buf);
    for (int k = 0; k < q; ++k) {
      const int64_t j = int64_t(ed) * q + k;
      r.row_ptr[j + 1] = r.row_ptr[j] + int64_t(ne) * q;
    }
  }
  r.col_idx.resize(size_t(r.row_ptr[r.n]));
  for (int ed = 0; ed < m.n_edges; ++ed) {
    const int ne = row_edges(m, ed, buf);
    for (int k = 0; k < q; ++k) {
      int64_t pos = r.row_ptr[int64_t(ed) * q + k];
      for (int t = 0; t < ne; ++t)
        for (int kk = 0; kk < q; ++kk) r.col_idx[pos++] = int32_t(int64_t(buf[t]) * q + kk);
    }
  }
  return r;
}

double dirichlet_value(const MeshIndex& m, int e, int side, int k, const double* g_bnd) {
  const int p = m.p, ex = e % m.nx, ey = e / m.nx;
  const int64_t Nx = int64_t(m.nx) * (p - 1) + 1, Ny = int64_t(m.ny) * (p - 1) + 1;
  const double* gS = g_bnd;
  const double* gN = g_bnd + Nx;
  const double* gW = g_bnd + 2 * Nx;
  const double* gE = g_bnd + 2 * Nx + Ny;
  switch (side) {
    case 0: return gS[int64_t(ex) * (p - 1) + k + 1];
    case 1: return gE[int64_t(ey) * (p - 1) + k + 1];
    case 2: return gN[int64_t(ex) * (p - 1) + k + 1];
    default: return gW[int64_t(ey) * (p - 1) + k + 1];
  }
}

// SPEC.md:345-353,378-379,382.  For active row j on edge ed (local side s_t in each
// adjacent element e_t, t = 0,1 in ascending element id):
//   A~[j, c] = 0 + T_{e0}[r0, c0] + T_{e1}[r1, c1]           (only present terms)
//   f~[j]    = -( sum_t ( w_t[r_t] + sum_{Gamma cols} T_t[r_t, c] g_c ) )
// with the accumulation order written here (GPU K4 follows it exactly).
void assemble_reduced(const MeshIndex& m, const ReducedCSR& pat, const double* T, const double* w,
                      const double* g_bnd, double* values, double* rhs) {
  const int p = m.p, q = p - 2, nb = 4 * (p - 1);
  std::fill(values, values + pat.row_ptr[pat.n], 0.0);
  int buf[8];
  for (int ed = 0; ed < m.n_edges; ++ed) {
    const int ne = row_edges(m, ed, buf);
    for (int k = 0; k < q; ++k) {
      const int64_t j = int64_t(ed) * q + k;
      const int64_t rp = pat.row_ptr[j];
      double acc = 0.0;
      for (int t = 0; t < 2; ++t) {
        const int e = m.edge_elems[2 * ed + t];
        const int s = m.edge_sides[2 * ed + t];
        const int r = side_base(p, s) + k;
        const double* Te = T + size_t(e) * nb * nb + size_t(r) * nb;
        acc = acc + w[size_t(e) * nb + r];
        for (int sc = 0; sc < 4; ++sc) {
          const int ce = m.elem_edges[size_t(4) * e + sc];
          if (ce >= 0) {
            const int rank = int(std::lower_bound(buf, buf + ne, ce) - buf);
            double* dst = values + rp + int64_t(rank) * q;
            for (int kk = 0; kk < q; ++kk) dst[kk] = dst[kk] + Te[side_base(p, sc) + kk];
          } else {
            for (int kk = 0; kk < q; ++kk) {
              const double g = dirichlet_value(m, e, sc, kk, g_bnd);
              const double prod = Te[side_base(p, sc) + kk] * g;
              acc = acc + prod;
            }
          }
        }
      }
      rhs[j] = -acc;
    }
  }
}

}  // namespace hpso
