// =====================================================================================
//  CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  Plain, slow, obviously-correct fp64 implementation of what the hot path computes:
//  quadratic B-spline cloth membrane (FEM Baraff–Witkin) + quadratic (Laplacian) bending
//  energy, gradient and Hessian at the paper's reduced quadrature points, scattered into a
//  3x3-block sparse (BSR) matrix whose pattern is the set union of the structural stencils.
//
//  Paper: arXiv 2506.18867, /root/reference/PAPER.md (cited as PAPER.md:<line>).
//  Readings where the paper is silent/garbled: DESIGN.md §"Readings" (Q1..Q12, D4, D6, D7).
//
//  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
//  load this library.  It shares NO code with paper_2506_18867_b200/ (the CUDA path).
//
//  Route (deliberately the plain one):
//   * Cox–de Boor recursion evaluated per point (Eq. `eq: B-spline basis`),
//     derivatives by differentiating the recursion (Piegl & Tiller, cited PAPER.md:151);
//   * inverse map by the inverse function theorem, incl. second derivatives;
//   * dense local matrices H_loc = w B^T A B (membrane), w mu L L^T (x) I3 (bending);
//   * optional PSD projection of each FBW term by cyclic Jacobi eigen-decomposition (D7);
//   * scatter into the oracle's own set-union BSR pattern by binary search.
//
//  Parity status of each function: see the headers of tests/test_oracle_pins.py, (incremental
//  potential: lumped mass, inertia, gravity, pinned elimination) tests/test_oracle_ip.py and (contact pullback)
//  tests/test_oracle_contact.py; every function
//  below is pinned (no "parity unpinned" entries) except the membrane stiffness convention
//  mu_st/mu_sh of oracle_material_from_young (D6, a naming convention: "parity unpinned").
// =====================================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err = "ok";
int fail(const std::string& m, int code = -1) { g_err = m; return code; }

// ------------------------------------------------------------------ knots
// Open uniform integer knot vector, p = 2 ("open"/"uniform", PAPER.md:189 integer,
// starts at 0): (0,0,0,1,...,S-1,S,S,S) with n = S + 2 control points.
bool knots_ok(const double* k, int n) {
  const int S = n - 2;
  if (S < 1) return false;
  for (int i = 0; i < 3; ++i)
    if (k[i] != 0.0 || k[S + 2 + i] != (double)S) return false;
  for (int t = 0; t <= S; ++t)
    if (k[2 + t] != (double)t) return false;
  return true;
}

// ------------------------------------------------------------------ basis
// All quadratic bases N_{i,2}, i in [0, nk-3), with first and second derivatives at x.
// N_{i,0}(x) = 1 iff xi_i <= x < xi_{i+1} (half-open); at the right end x = xi_last
// the last non-empty span is used (closure, left limit — DESIGN.md Q8).  0/0 := 0.
// Derivative recursion: N^{(d)}_{i,p} = p [ N^{(d-1)}_{i,p-1}/(xi_{i+p}-xi_i)
//                                         - N^{(d-1)}_{i+1,p-1}/(xi_{i+p+1}-xi_{i+1}) ].
inline double sdiv(double a, double b) { return b == 0.0 ? 0.0 : a / b; }

void cox_de_boor(const double* xi, int nk, double x, double* N, double* dN, double* ddN) {
  const int nb0 = nk - 1, nb1 = nk - 2, nb2 = nk - 3;
  std::vector<double> N0(nb0, 0.0), N1(nb1, 0.0), dN1(nb1, 0.0);
  int s = -1;
  for (int i = 0; i < nb0; ++i)
    if (xi[i] <= x && x < xi[i + 1]) { s = i; break; }
  if (s < 0 && x == xi[nk - 1])
    for (int i = nb0 - 1; i >= 0; --i)
      if (xi[i] < xi[i + 1]) { s = i; break; }
  if (s >= 0) N0[s] = 1.0;
  for (int i = 0; i < nb1; ++i) {
    N1[i] = sdiv(x - xi[i], xi[i + 1] - xi[i]) * N0[i] + sdiv(xi[i + 2] - x, xi[i + 2] - xi[i + 1]) * N0[i + 1];
    dN1[i] = 1.0 * (sdiv(N0[i], xi[i + 1] - xi[i]) - sdiv(N0[i + 1], xi[i + 2] - xi[i + 1]));
  }
  for (int i = 0; i < nb2; ++i) {
    N[i] = sdiv(x - xi[i], xi[i + 2] - xi[i]) * N1[i] + sdiv(xi[i + 3] - x, xi[i + 3] - xi[i + 1]) * N1[i + 1];
    dN[i] = 2.0 * (sdiv(N1[i], xi[i + 2] - xi[i]) - sdiv(N1[i + 1], xi[i + 3] - xi[i + 1]));
    ddN[i] = 2.0 * (sdiv(dN1[i], xi[i + 2] - xi[i]) - sdiv(dN1[i + 1], xi[i + 3] - xi[i + 1]));
  }
}

// ------------------------------------------------------------------ Gauss–Legendre (Q6)
// Exact nodes/weights on [a,b] (1, 2 or 3 points).
void gauss(int m, double a, double b, double* x, double* w) {
  const double c = 0.5 * (a + b), h = 0.5 * (b - a);
  if (m == 1) { x[0] = c; w[0] = b - a; return; }
  if (m == 2) {
    const double t = 1.0 / std::sqrt(3.0);
    x[0] = c - h * t; x[1] = c + h * t; w[0] = w[1] = h;
    return;
  }
  const double t = std::sqrt(0.6);
  x[0] = c - h * t; x[1] = c; x[2] = c + h * t;
  w[0] = w[2] = h * 5.0 / 9.0; w[1] = h * 8.0 / 9.0;
}

// ------------------------------------------------------------------ rules
enum { RULE_REDUCED = 0, RULE_G2_INTERIOR = 1, RULE_G3_FULL = 2 };

struct QP {           // one quadrature point
  double u, v, w;     // parametric coordinates and parametric weight w_hat
  int onknot_u, onknot_v;  // 1 if the coordinate is an interior knot (structural stencil differs)
};

// Per-direction structural index sets:
//  x strictly inside span s:  V = D2 = {s, s+1, s+2};
//  x on interior knot p:      V = {p, p+1} (value/first-derivative), D2 = {p, p+1, p+2} (right limit).
void dir_sets(double x, int onknot, std::vector<int>& V, std::vector<int>& D2) {
  V.clear(); D2.clear();
  if (onknot) {
    const int p = (int)x;
    V = {p, p + 1};
    D2 = {p, p + 1, p + 2};
  } else {
    const int s = (int)std::floor(x);
    V = {s, s + 1, s + 2};
    D2 = V;
  }
}

void push_tensor(std::vector<QP>& out, int mu, double au, double bu, int mv, double av, double bv) {
  double xu[3], wu[3], xv[3], wv[3];
  gauss(mu, au, bu, xu, wu);
  gauss(mv, av, bv, xv, wv);
  for (int j = 0; j < mv; ++j)
    for (int i = 0; i < mu; ++i) out.push_back({xu[i], xv[j], wu[i] * wv[j], 0, 0});
}

// Membrane rules.  REDUCED = PAPER.md:290-293 and Fig. `fig: quadrature`:
//  corner spans G3xG3; bottom/top side spans G2(u)xG3(v); left/right side spans G3(u)xG2(v);
//  interior region [1,Su-1]x[1,Sv-1] split into dual cells centred on knots (p,q), clipped to the
//  region (Q2); full cells alternate: p+q even -> u = p, v = G2 on [q-1/2, q+1/2]; odd -> v = q,
//  u = G2 on [p-1/2, p+1/2] (Q1); half cells on the region's edges keep the knot-line point pair
//  with half the weight; corner quarter cells get one point at the knot with weight 1/4.
void membrane_rule(int kind, int Su, int Sv, std::vector<QP>& out) {
  out.clear();
  if (kind == RULE_G3_FULL) {
    for (int j = 0; j < Sv; ++j)
      for (int i = 0; i < Su; ++i) push_tensor(out, 3, i, i + 1, 3, j, j + 1);
    return;
  }
  // boundary frame (shared by REDUCED and G2_INTERIOR)
  for (int j = 0; j < Sv; ++j)
    for (int i = 0; i < Su; ++i) {
      const bool bu = (i == 0 || i == Su - 1), bv = (j == 0 || j == Sv - 1);
      if (bu && bv) push_tensor(out, 3, i, i + 1, 3, j, j + 1);
      else if (bv) push_tensor(out, 2, i, i + 1, 3, j, j + 1);
      else if (bu) push_tensor(out, 3, i, i + 1, 2, j, j + 1);
      else if (kind == RULE_G2_INTERIOR) push_tensor(out, 2, i, i + 1, 2, j, j + 1);
    }
  if (kind == RULE_G2_INTERIOR) return;
  double g[2], gw[2];
  for (int q = 1; q <= Sv - 1; ++q)
    for (int p = 1; p <= Su - 1; ++p) {
      const bool eu = (p == 1 || p == Su - 1), ev = (q == 1 || q == Sv - 1);
      if (eu && ev) { out.push_back({(double)p, (double)q, 0.25, 1, 1}); continue; }
      bool along_v;  // two Gauss points along v (u = p fixed)?
      double wscale = 1.0;
      if (eu) { along_v = true; wscale = 0.5; }
      else if (ev) { along_v = false; wscale = 0.5; }
      else along_v = ((p + q) % 2 == 0);
      if (along_v) {
        gauss(2, q - 0.5, q + 0.5, g, gw);
        for (int t = 0; t < 2; ++t) out.push_back({(double)p, g[t], gw[t] * wscale, 1, 0});
      } else {
        gauss(2, p - 0.5, p + 0.5, g, gw);
        for (int t = 0; t < 2; ++t) out.push_back({g[t], (double)q, gw[t] * wscale, 0, 1});
      }
    }
}

// Bending rules.  REDUCED = PAPER.md:571-573 and Fig. `fig: quadrature` right:
//  one point at the centre of every boundary span (w = 1); one point at every interior knot (the
//  centre of its dual cell), w = omega_p*omega_q with omega = 1/2 at the first/last interior knot
//  (the clipped half cells, Q2) and 1 otherwise.
void bending_rule(int kind, int Su, int Sv, std::vector<QP>& out) {
  out.clear();
  if (kind == RULE_G3_FULL) {
    for (int j = 0; j < Sv; ++j)
      for (int i = 0; i < Su; ++i) push_tensor(out, 3, i, i + 1, 3, j, j + 1);
    return;
  }
  for (int j = 0; j < Sv; ++j)
    for (int i = 0; i < Su; ++i) {
      const bool bnd = (i == 0 || i == Su - 1 || j == 0 || j == Sv - 1);
      if (bnd) push_tensor(out, 1, i, i + 1, 1, j, j + 1);
      else if (kind == RULE_G2_INTERIOR) push_tensor(out, 2, i, i + 1, 2, j, j + 1);
    }
  if (kind == RULE_G2_INTERIOR) return;
  for (int q = 1; q <= Sv - 1; ++q)
    for (int p = 1; p <= Su - 1; ++p) {
      const double wu = (p == 1 || p == Su - 1) ? 0.5 : 1.0;
      const double wv = (q == 1 || q == Sv - 1) ? 0.5 : 1.0;
      out.push_back({(double)p, (double)q, wu * wv, 1, 1});
    }
}

// Structural stencil of a point: membrane V(u) x V(v); bending (D2(u) x V(v)) u (V(u) x D2(v))
// u (V(u) x V(v)) — the cps whose N, N_u, N_v, N_uu, N_vv or N_uv can be nonzero (Q3/D4, Q10).
// Returned as a sorted list of (i, j).
void stencil(const QP& q, bool bending, std::vector<std::pair<int, int>>& st) {
  std::vector<int> Vu, Du, Vv, Dv;
  dir_sets(q.u, q.onknot_u, Vu, Du);
  dir_sets(q.v, q.onknot_v, Vv, Dv);
  st.clear();
  for (int j : Vv) for (int i : Vu) st.push_back({i, j});
  if (bending) {
    for (int j : Vv) for (int i : Du) st.push_back({i, j});
    for (int j : Dv) for (int i : Vu) st.push_back({i, j});
  }
  std::sort(st.begin(), st.end(), [](auto a, auto b) { return a.second != b.second ? a.second < b.second : a.first < b.first; });
  st.erase(std::unique(st.begin(), st.end()), st.end());
}

// ------------------------------------------------------------------ per-point precompute
struct Point {
  bool bending;
  double w;                 // w = w_hat * det J  (integral over material space, Q9)
  std::vector<int> cp;      // global cp index a = j*n_u + i
  std::vector<int> row;     // cp row j of each stencil entry
  std::vector<double> b;    // membrane: b_a = (dN_a/dX1, dN_a/dX2), 2 per cp
  std::vector<double> L;    // bending: Laplacian coefficient L_a (Eq. `eq: Laplacian in parametric space`)
  int row_min, row_max;
};

struct Oracle {
  int n_u, n_v, Su, Sv;
  std::vector<double> ku, kv, rest;  // rest [n_v][n_u][2]
  double mu_st1, mu_st2, mu_sh, mu_bd;
  int mrule, brule;
  int r0, r1;          // owned cp rows [r0, r1)
  int lo, hi;          // rows present in x: [lo, hi)
  std::vector<Point> pts;
  std::vector<int32_t> row_ptr, col_idx;   // owned block rows, global column indices
};

// Material-map derivatives at (u,v): PAPER.md:277-288 (Eq. `eq: deformation gradient`) and
// PAPER.md:560-568.  J_{c p} = dX_c/dp (p in {u,v}); G = J^{-1}, G_{r c} = dr/dX_c;
// second order (inverse function theorem, derivation in DESIGN.md):
//   d^2 r / dX_a dX_b = - sum_{c,p,q} G_{r c} X_{c,pq} G_{p a} G_{q b},  X_{c,pq} = sum N_{,pq} X_c.
int precompute_point(const Oracle& o, const QP& q, bool bending, Point& P) {
  const int nu = o.n_u, nv = o.n_v;
  std::vector<double> Nu(nu), dNu(nu), ddNu(nu), Nv(nv), dNv(nv), ddNv(nv);
  cox_de_boor(o.ku.data(), nu + 3, q.u, Nu.data(), dNu.data(), ddNu.data());
  cox_de_boor(o.kv.data(), nv + 3, q.v, Nv.data(), dNv.data(), ddNv.data());
  // J and second derivatives of X, summed over all cps (zero outside the support by Eq. 1).
  double J[2][2] = {{0, 0}, {0, 0}}, X2[2][2][2] = {};
  const int iu0 = std::max(0, (int)std::floor(q.u) - 1), iu1 = std::min(nu - 1, (int)std::floor(q.u) + 3);
  const int jv0 = std::max(0, (int)std::floor(q.v) - 1), jv1 = std::min(nv - 1, (int)std::floor(q.v) + 3);
  for (int j = jv0; j <= jv1; ++j)
    for (int i = iu0; i <= iu1; ++i) {
      const double* X = &o.rest[2 * ((size_t)j * nu + i)];
      const double Na_u = dNu[i] * Nv[j], Na_v = Nu[i] * dNv[j];
      const double Na_uu = ddNu[i] * Nv[j], Na_vv = Nu[i] * ddNv[j], Na_uv = dNu[i] * dNv[j];
      for (int c = 0; c < 2; ++c) {
        J[c][0] += Na_u * X[c];
        J[c][1] += Na_v * X[c];
        X2[c][0][0] += Na_uu * X[c];
        X2[c][1][1] += Na_vv * X[c];
        X2[c][0][1] += Na_uv * X[c];
        X2[c][1][0] += Na_uv * X[c];
      }
    }
  const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  if (!(det > 0.0)) return fail("degenerate geometry: det J <= 0 at a quadrature point", -4);
  double G[2][2];  // G[r][c] = d r / d X_c ; r: 0=u,1=v
  G[0][0] = J[1][1] / det; G[0][1] = -J[0][1] / det;
  G[1][0] = -J[1][0] / det; G[1][1] = J[0][0] / det;
  double R2[2][2][2];  // R2[r][a][b] = d^2 r / dX_a dX_b
  for (int r = 0; r < 2; ++r)
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double s = 0;
        for (int c = 0; c < 2; ++c)
          for (int p = 0; p < 2; ++p)
            for (int qq = 0; qq < 2; ++qq) s += G[r][c] * X2[c][p][qq] * G[p][a] * G[qq][b];
        R2[r][a][b] = -s;
      }
  const double u1 = G[0][0], u2 = G[0][1], v1 = G[1][0], v2 = G[1][1];
  const double u11 = R2[0][0][0], u22 = R2[0][1][1], v11 = R2[1][0][0], v22 = R2[1][1][1];
  P.bending = bending;
  P.w = q.w * det;
  std::vector<std::pair<int, int>> st;
  stencil(q, bending, st);
  P.cp.clear(); P.row.clear(); P.b.clear(); P.L.clear();
  P.row_min = 1 << 30; P.row_max = -1;
  for (auto [i, j] : st) {
    if (i < 0 || i >= nu || j < 0 || j >= nv) return fail("internal: stencil outside grid", -1);
    P.cp.push_back(j * nu + i);
    P.row.push_back(j);
    P.row_min = std::min(P.row_min, j);
    P.row_max = std::max(P.row_max, j);
    const double Na_u = dNu[i] * Nv[j], Na_v = Nu[i] * dNv[j];
    if (!bending) {
      // b_a = (N_a,u u1 + N_a,v v1, N_a,u u2 + N_a,v v2)   (Eq. `eq: deformation gradient`)
      P.b.push_back(Na_u * u1 + Na_v * v1);
      P.b.push_back(Na_u * u2 + Na_v * v2);
    } else {
      const double Na_uu = ddNu[i] * Nv[j], Na_vv = Nu[i] * ddNv[j], Na_uv = dNu[i] * dNv[j];
      // Eq. `eq: Laplacian in parametric space`
      P.L.push_back((u1 * u1 + u2 * u2) * Na_uu + (v1 * v1 + v2 * v2) * Na_vv + (u11 + u22) * Na_u +
                    (v11 + v22) * Na_v + 2.0 * (u1 * v1 + u2 * v2) * Na_uv);
    }
  }
  return 0;
}

// ------------------------------------------------------------------ energies (templated for complex step)
// FBW: I5(e1)=f1.f1, I5(e2)=f2.f2, I6=f1.f2 with f_beta = F e_beta;
// Psi = mu_sh I6^2 + mu_st1 (sqrt(I5_1)-1)^2 + mu_st2 (sqrt(I5_2)-1)^2.
// No conjugation anywhere: the expressions stay holomorphic for the complex-step checks.
template <class T>
void deformation_gradient(const Point& P, const std::vector<T>& xs, T f[2][3]) {
  for (int be = 0; be < 2; ++be)
    for (int c = 0; c < 3; ++c) f[be][c] = T(0);
  for (size_t k = 0; k < P.cp.size(); ++k)
    for (int be = 0; be < 2; ++be)
      for (int c = 0; c < 3; ++c) f[be][c] += xs[3 * k + c] * P.b[2 * k + be];
}

template <class T>
T membrane_psi(const Oracle& o, const T f[2][3]) {
  T I51 = T(0), I52 = T(0), I6 = T(0);
  for (int c = 0; c < 3; ++c) { I51 += f[0][c] * f[0][c]; I52 += f[1][c] * f[1][c]; I6 += f[0][c] * f[1][c]; }
  const T s1 = std::sqrt(I51) - T(1), s2 = std::sqrt(I52) - T(1);
  return o.mu_sh * I6 * I6 + o.mu_st1 * s1 * s1 + o.mu_st2 * s2 * s2;
}

// P = dPsi/dF, columns: P_1 = 2 mu_st1 (1 - 1/|f1|) f1 + 2 mu_sh I6 f2 ; P_2 symmetric.
template <class T>
void membrane_P(const Oracle& o, const T f[2][3], T Pm[2][3]) {
  T I51 = T(0), I52 = T(0), I6 = T(0);
  for (int c = 0; c < 3; ++c) { I51 += f[0][c] * f[0][c]; I52 += f[1][c] * f[1][c]; I6 += f[0][c] * f[1][c]; }
  const T a1 = T(2.0 * o.mu_st1) * (T(1) - T(1) / std::sqrt(I51));
  const T a2 = T(2.0 * o.mu_st2) * (T(1) - T(1) / std::sqrt(I52));
  for (int c = 0; c < 3; ++c) {
    Pm[0][c] = a1 * f[0][c] + T(2.0 * o.mu_sh) * I6 * f[1][c];
    Pm[1][c] = a2 * f[1][c] + T(2.0 * o.mu_sh) * I6 * f[0][c];
  }
}

template <class T>
void gather_x(const Oracle& o, const Point& P, const T* x, std::vector<T>& xs) {
  xs.resize(3 * P.cp.size());
  for (size_t k = 0; k < P.cp.size(); ++k) {
    const int j = P.row[k], i = P.cp[k] - j * o.n_u;
    const T* src = x + 3 * ((size_t)(j - o.lo) * o.n_u + i);
    for (int c = 0; c < 3; ++c) xs[3 * k + c] = src[c];
  }
}

template <class T>
T point_energy(const Oracle& o, const Point& P, const std::vector<T>& xs) {
  if (!P.bending) {
    T f[2][3];
    deformation_gradient(P, xs, f);
    return T(P.w) * membrane_psi(o, f);
  }
  // Psi_bd = 1/2 mu_bd <Lap phi, Lap phi>
  T lap[3] = {T(0), T(0), T(0)};
  for (size_t k = 0; k < P.cp.size(); ++k)
    for (int c = 0; c < 3; ++c) lap[c] += P.L[k] * xs[3 * k + c];
  return T(0.5 * P.w * o.mu_bd) * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]);
}

template <class T>
void point_gradient(const Oracle& o, const Point& P, const std::vector<T>& xs, std::vector<T>& g) {
  g.assign(3 * P.cp.size(), T(0));
  if (!P.bending) {
    T f[2][3], Pm[2][3];
    deformation_gradient(P, xs, f);
    membrane_P(o, f, Pm);
    // g_a = w P b_a
    for (size_t k = 0; k < P.cp.size(); ++k)
      for (int c = 0; c < 3; ++c) g[3 * k + c] = T(P.w) * (Pm[0][c] * P.b[2 * k] + Pm[1][c] * P.b[2 * k + 1]);
    return;
  }
  T lap[3] = {T(0), T(0), T(0)};
  for (size_t k = 0; k < P.cp.size(); ++k)
    for (int c = 0; c < 3; ++c) lap[c] += P.L[k] * xs[3 * k + c];
  for (size_t k = 0; k < P.cp.size(); ++k)
    for (int c = 0; c < 3; ++c) g[3 * k + c] = T(P.w * o.mu_bd * P.L[k]) * lap[c];
}

// ------------------------------------------------------------------ Jacobi eigen (for PSD projection, D7)
// Cyclic Jacobi on a symmetric n x n matrix (row-major); returns eigenvalues in d, vectors in V (columns).
void jacobi_eig(int n, std::vector<double> A, std::vector<double>& d, std::vector<double>& V) {
  V.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0, tot = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) { tot += A[i * n + j] * A[i * n + j]; if (i != j) off += A[i * n + j] * A[i * n + j]; }
    if (off <= 1e-34 * tot || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- A J (columns p,q)
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^T A (rows p,q)
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  d.resize(n);
  for (int i = 0; i < n; ++i) d[i] = A[i * n + i];
}

// PSD(M) = sum_i max(lambda_i, 0) v_i v_i^T
void psd_project(int n, std::vector<double>& M) {
  std::vector<double> d, V;
  jacobi_eig(n, M, d, V);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0;
      for (int k = 0; k < n; ++k) s += std::max(d[k], 0.0) * V[i * n + k] * V[j * n + k];
      M[i * n + j] = s;
    }
}

// F-space Hessian A = d^2 Psi / d vecF^2 (6x6, vecF = (f1, f2)), per term (D7):
//  stretch_j: 2 mu_j [ (1 - 1/|f_j|) I3 + f_j f_j^T / |f_j|^3 ] on the f_j block;
//  shear:     2 mu_sh [ g g^T + I6 [[0, I3],[I3, 0]] ],  g = (f2, f1).
void membrane_A(const Oracle& o, const double f[2][3], bool project, double A[6][6]) {
  double I5[2], I6 = 0;
  for (int be = 0; be < 2; ++be) { I5[be] = 0; for (int c = 0; c < 3; ++c) I5[be] += f[be][c] * f[be][c]; }
  for (int c = 0; c < 3; ++c) I6 += f[0][c] * f[1][c];
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) A[i][j] = 0;
  const double mus[2] = {o.mu_st1, o.mu_st2};
  for (int be = 0; be < 2; ++be) {
    const double nrm = std::sqrt(I5[be]);
    std::vector<double> H(9);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        H[a * 3 + b] = 2.0 * mus[be] * ((a == b ? 1.0 - 1.0 / nrm : 0.0) + f[be][a] * f[be][b] / (nrm * nrm * nrm));
    if (project) psd_project(3, H);
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) A[3 * be + a][3 * be + b] += H[a * 3 + b];
  }
  std::vector<double> Hs(36);
  double g[6];
  for (int c = 0; c < 3; ++c) { g[c] = f[1][c]; g[3 + c] = f[0][c]; }
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      const double S = ((a < 3) != (b < 3) && (a % 3) == (b % 3)) ? 1.0 : 0.0;
      Hs[a * 6 + b] = 2.0 * o.mu_sh * (g[a] * g[b] + I6 * S);
    }
  if (project) psd_project(6, Hs);
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) A[a][b] += Hs[a * 6 + b];
}

// Dense local Hessian (3k x 3k, row-major).
void point_hessian(const Oracle& o, const Point& P, const std::vector<double>& xs, bool project, std::vector<double>& H) {
  const int k = (int)P.cp.size(), m = 3 * k;
  H.assign((size_t)m * m, 0.0);
  if (!P.bending) {
    double f[2][3], A[6][6];
    deformation_gradient(P, xs, f);
    membrane_A(o, f, project, A);
    // B (6 x 3k): vecF = B c, B[3*be + c][3*a + c] = b_a,be
    std::vector<double> B((size_t)6 * m, 0.0), AB((size_t)6 * m, 0.0);
    for (int a = 0; a < k; ++a)
      for (int be = 0; be < 2; ++be)
        for (int c = 0; c < 3; ++c) B[(size_t)(3 * be + c) * m + 3 * a + c] = P.b[2 * a + be];
    for (int r = 0; r < 6; ++r)
      for (int col = 0; col < m; ++col) {
        double s = 0;
        for (int t = 0; t < 6; ++t) s += A[r][t] * B[(size_t)t * m + col];
        AB[(size_t)r * m + col] = s;
      }
    for (int r = 0; r < m; ++r)
      for (int col = 0; col < m; ++col) {
        double s = 0;
        for (int t = 0; t < 6; ++t) s += B[(size_t)t * m + r] * AB[(size_t)t * m + col];
        H[(size_t)r * m + col] = P.w * s;
      }
    return;
  }
  // bending: w mu_bd L_a L_b I3 (constant, PSD; never projected — DESIGN.md D7)
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b)
      for (int c = 0; c < 3; ++c) H[(size_t)(3 * a + c) * m + 3 * b + c] = P.w * o.mu_bd * P.L[a] * P.L[b];
}

enum { FLAG_PROJECT = 1, FLAG_NO_MEMBRANE = 2, FLAG_NO_BENDING = 4, FLAG_ABS_SUM = 8 };
// FLAG_ABS_SUM: accumulate |local Hessian entries| instead of the entries (sum_q |H_q,blk|, the
// cancellation scale of every block, used by the parity tolerance).

bool skip(const Point& P, int flags) {
  return (P.bending && (flags & FLAG_NO_BENDING)) || (!P.bending && (flags & FLAG_NO_MEMBRANE));
}
bool touches(const Point& P, int ra, int rb) { return P.row_max >= ra && P.row_min < rb; }

}  // namespace

// =====================================================================================
extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// All quadratic bases at x: N, dN, ddN of length nk - 3.
int oracle_basis_all(const double* knots, int nk, double x, double* N, double* dN, double* ddN) {
  if (nk < 4) return fail("nk < 4");
  cox_de_boor(knots, nk, x, N, dN, ddN);
  return 0;
}

int oracle_gauss(int m, double a, double b, double* x, double* w) {
  if (m < 1 || m > 3) return fail("m must be 1..3");
  gauss(m, a, b, x, w);
  return 0;
}

// Rule points: returns the count; fills up to cap points (u, v, w_hat) and stencils
// (st_n[k] entries of (i,j) pairs in st[k*18 ...]) when the pointers are non-null.
int oracle_rule(int kind, int bending, int Su, int Sv, int cap, double* u, double* v, double* w,
                int32_t* st_n, int32_t* st) {
  if (kind < 0 || kind > 2) return fail("bad rule kind");
  if (kind != RULE_G3_FULL && (Su < 3 || Sv < 3)) return fail("reduced rules need >= 3 spans per direction", -3);
  std::vector<QP> q;
  if (bending) bending_rule(kind, Su, Sv, q); else membrane_rule(kind, Su, Sv, q);
  std::vector<std::pair<int, int>> s;
  for (int k = 0; k < (int)q.size() && k < cap; ++k) {
    if (u) u[k] = q[k].u;
    if (v) v[k] = q[k].v;
    if (w) w[k] = q[k].w;
    if (st_n) {
      stencil(q[k], bending != 0, s);
      st_n[k] = (int)s.size();
      for (size_t t = 0; t < s.size(); ++t) { st[k * 18 + 2 * t] = s[t].first; st[k * 18 + 2 * t + 1] = s[t].second; }
    }
  }
  return (int)q.size();
}

// Material map (D6 / Q4): mu_st1 = mu_st2 = E h / 2; mu_sh = G h / 2 with
// G = shear_E if shear_E >= 0 else E / (2 (1 + nu)); mu_bd = E_b h^3 / (12 (1 - nu^2)),
// E_b = bend_E if >= 0 else E.  (mu_bd pinned by the plate formula PAPER.md:1149.)
int oracle_material_from_young(double E, double nu, double h, double shear_E, double bend_E, double* mu4) {
  if (!(E > 0) || !(h > 0) || !(nu > -1 && nu < 0.5)) return fail("bad material");
  const double G = shear_E >= 0 ? shear_E : E / (2.0 * (1.0 + nu));
  const double Eb = bend_E >= 0 ? bend_E : E;
  mu4[0] = E * h / 2.0;
  mu4[1] = E * h / 2.0;
  mu4[2] = G * h / 2.0;
  mu4[3] = Eb * h * h * h / (12.0 * (1.0 - nu * nu));
  return 0;
}

// Create: precompute rules, per-point coefficients and the pattern of owned rows [r0, r1).
void* oracle_create(int n_u, int n_v, const double* knots_u, const double* knots_v, const double* rest_xy,
                    const double* mu4, int mrule, int brule, int r0, int r1) {
  if (n_u < 3 || n_v < 3) { fail("grid too small", -3); return nullptr; }
  if (!knots_ok(knots_u, n_u) || !knots_ok(knots_v, n_v)) { fail("knots must be open, uniform, integer", -2); return nullptr; }
  if (r0 < 0 || r1 > n_v || r0 >= r1) { fail("bad row range"); return nullptr; }
  auto* o = new Oracle();
  o->n_u = n_u; o->n_v = n_v; o->Su = n_u - 2; o->Sv = n_v - 2;
  o->ku.assign(knots_u, knots_u + n_u + 3);
  o->kv.assign(knots_v, knots_v + n_v + 3);
  o->rest.assign(rest_xy, rest_xy + (size_t)2 * n_u * n_v);
  o->mu_st1 = mu4[0]; o->mu_st2 = mu4[1]; o->mu_sh = mu4[2]; o->mu_bd = mu4[3];
  o->mrule = mrule; o->brule = brule;
  o->r0 = r0; o->r1 = r1;
  o->lo = std::max(0, r0 - 2); o->hi = std::min(n_v, r1 + 2);
  std::vector<QP> qm, qb;
  if ((mrule != RULE_G3_FULL && (o->Su < 3 || o->Sv < 3)) || (brule != RULE_G3_FULL && (o->Su < 3 || o->Sv < 3))) {
    fail("reduced rules need >= 3 spans per direction", -3); delete o; return nullptr;
  }
  membrane_rule(mrule, o->Su, o->Sv, qm);
  bending_rule(brule, o->Su, o->Sv, qb);
  // keep only points touching owned rows (row reach of a stencil: floor(v)-1 .. floor(v)+2)
  auto keep = [&](const QP& q) { const int j = (int)std::floor(q.v); return j + 2 >= r0 && j - 1 < r1; };
  int err = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (const QP& q : (pass == 0 ? qm : qb)) {
      if (!keep(q)) continue;
      Point P;
      const int rc = precompute_point(*o, q, pass == 1, P);
      if (rc) { err = rc; break; }
      if (touches(P, r0, r1)) o->pts.push_back(std::move(P));
    }
  if (err) { delete o; return nullptr; }
  // Pattern: diagonal u union over points of stencil x stencil (Q10), owned rows only, sorted.
  const int nrows = (r1 - r0) * n_u;
  std::vector<std::vector<int32_t>> cols(nrows);
  for (int a = 0; a < nrows; ++a) cols[a].push_back(r0 * n_u + a);
  for (const Point& P : o->pts)
    for (size_t k = 0; k < P.cp.size(); ++k) {
      if (P.row[k] < r0 || P.row[k] >= r1) continue;
      auto& c = cols[P.cp[k] - r0 * n_u];
      for (int b : P.cp) c.push_back(b);
    }
  o->row_ptr.assign(nrows + 1, 0);
  for (int a = 0; a < nrows; ++a) {
    auto& c = cols[a];
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    o->row_ptr[a + 1] = o->row_ptr[a] + (int32_t)c.size();
  }
  o->col_idx.resize(o->row_ptr[nrows]);
  for (int a = 0; a < nrows; ++a) std::copy(cols[a].begin(), cols[a].end(), o->col_idx.begin() + o->row_ptr[a]);
  return o;
}

void oracle_destroy(void* h) { delete static_cast<Oracle*>(h); }

int64_t oracle_nnzb(void* h) { return (int64_t)static_cast<Oracle*>(h)->col_idx.size(); }
int oracle_num_points(void* h, int* n_membrane, int* n_bending) {
  auto* o = static_cast<Oracle*>(h);
  int m = 0, b = 0;
  for (auto& P : o->pts) (P.bending ? b : m)++;
  *n_membrane = m; *n_bending = b;
  return 0;
}

int oracle_pattern(void* h, int32_t* row_ptr, int32_t* col_idx) {
  auto* o = static_cast<Oracle*>(h);
  std::copy(o->row_ptr.begin(), o->row_ptr.end(), row_ptr);
  std::copy(o->col_idx.begin(), o->col_idx.end(), col_idx);
  return 0;
}

// Point coefficient dump (for inverse-map pins): point k of the owned set: w, stencil size, cps,
// and b (2 per cp) or L (1 per cp).  Returns bending flag.
int oracle_point(void* h, int k, double* w, int32_t* n, int32_t* cps, double* coef) {
  auto* o = static_cast<Oracle*>(h);
  if (k < 0 || k >= (int)o->pts.size()) return fail("bad point index");
  const Point& P = o->pts[k];
  *w = P.w;
  *n = (int)P.cp.size();
  for (size_t t = 0; t < P.cp.size(); ++t) {
    cps[t] = P.cp[t];
    if (P.bending) coef[t] = P.L[t];
    else { coef[2 * t] = P.b[2 * t]; coef[2 * t + 1] = P.b[2 * t + 1]; }
  }
  return P.bending ? 1 : 0;
}

// Energy, gradient (owned rows) and Hessian values (owned block rows).  x: rows [lo, hi).
// Energy counts the points whose lowest stencil row is owned (so slabs sum to the total).
// Any of E, g, vals may be null.
int oracle_eval(void* h, const double* x, int flags, double* E, double* g, double* vals, int nthreads) {
  auto* o = static_cast<Oracle*>(h);
  const bool project = flags & FLAG_PROJECT;
  const int nu = o->n_u, r0 = o->r0, r1 = o->r1;
  if (nthreads <= 0) nthreads = 1;
  if (E) {
    double e = 0;
    std::vector<double> xs;
    for (const Point& P : o->pts) {
      if (skip(P, flags) || P.row_min < r0 || P.row_min >= r1) continue;
      gather_x(*o, P, x, xs);
      e += point_energy(*o, P, xs);
    }
    *E = e;
  }
  // Row chunks: each chunk scatters only into its own rows; every block accumulates its points in
  // the global point order, so results are independent of the thread count.
  const int chunk = 4;
  const int nchunks = (r1 - r0 + chunk - 1) / chunk;
  if (g) std::fill(g, g + (size_t)3 * (r1 - r0) * nu, 0.0);
  if (vals) std::fill(vals, vals + (size_t)9 * o->col_idx.size(), 0.0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
  for (int cchunk = 0; cchunk < nchunks; ++cchunk) {
    const int ra = r0 + cchunk * chunk, rb = std::min(r1, ra + chunk);
    std::vector<double> xs, gl, Hl;
    for (const Point& P : o->pts) {
      if (skip(P, flags) || !touches(P, ra, rb)) continue;
      gather_x(*o, P, x, xs);
      const int k = (int)P.cp.size(), m = 3 * k;
      if (g) {
        point_gradient(*o, P, xs, gl);
        for (int a = 0; a < k; ++a) {
          if (P.row[a] < ra || P.row[a] >= rb) continue;
          double* dst = g + 3 * (size_t)(P.cp[a] - r0 * nu);
          for (int c = 0; c < 3; ++c) dst[c] += gl[3 * a + c];
        }
      }
      if (vals) {
        point_hessian(*o, P, xs, project, Hl);
        if (flags & FLAG_ABS_SUM)
          for (double& hv : Hl) hv = std::fabs(hv);
        for (int a = 0; a < k; ++a) {
          if (P.row[a] < ra || P.row[a] >= rb) continue;
          const int row = P.cp[a] - r0 * nu;
          const int32_t* c0 = o->col_idx.data() + o->row_ptr[row];
          const int32_t* c1 = o->col_idx.data() + o->row_ptr[row + 1];
          for (int b = 0; b < k; ++b) {
            const int32_t* it = std::lower_bound(c0, c1, P.cp[b]);
            double* blk = vals + 9 * (size_t)(it - o->col_idx.data());
            for (int r = 0; r < 3; ++r)
              for (int c = 0; c < 3; ++c) blk[3 * r + c] += Hl[(size_t)(3 * a + r) * m + 3 * b + c];
          }
        }
      }
    }
  }
  return 0;
}

// Complex-step helpers: energy and analytic gradient in std::complex<double> (holomorphic).
int oracle_energy_cplx(void* h, const double* x_re, const double* x_im, int flags, double* E_re, double* E_im) {
  auto* o = static_cast<Oracle*>(h);
  const size_t n = (size_t)3 * (o->hi - o->lo) * o->n_u;
  std::vector<std::complex<double>> x(n), xs;
  for (size_t i = 0; i < n; ++i) x[i] = {x_re[i], x_im[i]};
  std::complex<double> e = 0;
  for (const Point& P : o->pts) {
    if (skip(P, flags) || P.row_min < o->r0 || P.row_min >= o->r1) continue;
    gather_x(*o, P, x.data(), xs);
    e += point_energy(*o, P, xs);
  }
  *E_re = e.real(); *E_im = e.imag();
  return 0;
}

int oracle_gradient_cplx(void* h, const double* x_re, const double* x_im, int flags, double* g_re, double* g_im) {
  auto* o = static_cast<Oracle*>(h);
  const int nu = o->n_u;
  const size_t n = (size_t)3 * (o->hi - o->lo) * nu, ng = (size_t)3 * (o->r1 - o->r0) * nu;
  std::vector<std::complex<double>> x(n), xs, gl, g(ng, 0.0);
  for (size_t i = 0; i < n; ++i) x[i] = {x_re[i], x_im[i]};
  for (const Point& P : o->pts) {
    if (skip(P, flags)) continue;
    gather_x(*o, P, x.data(), xs);
    point_gradient(*o, P, xs, gl);
    for (size_t a = 0; a < P.cp.size(); ++a) {
      if (P.row[a] < o->r0 || P.row[a] >= o->r1) continue;
      for (int c = 0; c < 3; ++c) g[3 * (size_t)(P.cp[a] - o->r0 * nu) + c] += gl[3 * a + c];
    }
  }
  for (size_t i = 0; i < ng; ++i) { g_re[i] = g[i].real(); g_im[i] = g[i].imag(); }
  return 0;
}

// ------------------------------------------------------------------ incremental potential
// Lumped mass of the owned control points, step by step as the paper states it:
//   consistent mass  M_ab = int_Omega0 R0 N_a N_b dX
//   quadrature       3x3 Gauss per knot span (exact for N_a N_b per span)
//   lumping          m_a = sum_b M_ab, off-diagonals dropped     (Eq. lumped mass)
// R0 = areal (reference) density, dX = det J du dv.  m: [owned rows][n_u].
int oracle_lumped_mass(void* h, double R0, double* m) {
  auto* o = static_cast<Oracle*>(h);
  const int nu = o->n_u, nv = o->n_v;
  std::vector<double> Nu(nu), dNu(nu), ddNu(nu), Nv(nv), dNv(nv), ddNv(nv);
  std::fill(m, m + (size_t)(o->r1 - o->r0) * nu, 0.0);
  double gx[3], gw[3], hx[3], hw[3];
  for (int t = 0; t < o->Sv; ++t)
    for (int s = 0; s < o->Su; ++s) {
      // bases active on span (s, t): i in [s, s+2], j in [t, t+2]
      if (t + 2 < o->r0 || t >= o->r1) continue;
      gauss(3, s, s + 1, gx, gw);
      gauss(3, t, t + 1, hx, hw);
      double Mloc[9][9] = {};
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          cox_de_boor(o->ku.data(), nu + 3, gx[a], Nu.data(), dNu.data(), ddNu.data());
          cox_de_boor(o->kv.data(), nv + 3, hx[b], Nv.data(), dNv.data(), ddNv.data());
          double J[2][2] = {{0, 0}, {0, 0}};
          for (int j = t; j <= t + 2; ++j)
            for (int i = s; i <= s + 2; ++i) {
              const double* X = &o->rest[2 * ((size_t)j * nu + i)];
              for (int c = 0; c < 2; ++c) { J[c][0] += dNu[i] * Nv[j] * X[c]; J[c][1] += Nu[i] * dNv[j] * X[c]; }
            }
          const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
          if (!(det > 0.0)) return fail("degenerate geometry: det J <= 0 at a mass quadrature point", -4);
          const double wq = gw[a] * hw[b] * det * R0;
          for (int e = 0; e < 9; ++e)
            for (int f = 0; f < 9; ++f)
              Mloc[e][f] += wq * Nu[s + e % 3] * Nv[t + e / 3] * Nu[s + f % 3] * Nv[t + f / 3];
        }
      for (int e = 0; e < 9; ++e) {
        const int j = t + e / 3, i = s + e % 3;
        if (j < o->r0 || j >= o->r1) continue;
        for (int f = 0; f < 9; ++f) m[(size_t)(j - o->r0) * nu + i] += Mloc[e][f];   // row sum
      }
    }
  return 0;
}

// Incremental potential (Eq. `eq:incremental_potential`) with the lumped mass and a
// uniform gravity field ("handled similarly to standard FEM"; Q13):
//   E = E_elastic(x) + sum_a m_a/(2 dt^2) |x_a - xhat_a|^2 - sum_a m_a g.x_a
//   g_a += m_a/dt^2 (x_a - xhat_a) - m_a g,   H_aa += m_a/dt^2 I3.
// Pinned control points (Dirichlet, Q14): gradient row zeroed; Hessian rows and columns zeroed
// and the diagonal block set to I3 (energy unchanged).  x: rows [lo, hi); xhat, m, pinned: owned rows
// (pinned over ALL rows [n_v][n_u], since columns of other slabs' rows are masked too).
int oracle_eval_ip(void* h, const double* x, const double* xhat, const double* m, double dt, const double* grav,
                   const uint8_t* pinned, int flags, double* E, double* g, double* vals, int nthreads) {
  auto* o = static_cast<Oracle*>(h);
  const int rc = oracle_eval(h, x, flags, E, g, vals, nthreads);
  if (rc) return rc;
  const int nu = o->n_u;
  const double k = 1.0 / (dt * dt);
  for (int j = o->r0; j < o->r1; ++j)
    for (int i = 0; i < nu; ++i) {
      const size_t a = (size_t)(j - o->r0) * nu + i;
      const double* xa = x + 3 * ((size_t)(j - o->lo) * nu + i);
      const double* ha = xhat + 3 * a;
      double d2 = 0, gx = 0;
      for (int c = 0; c < 3; ++c) { d2 += (xa[c] - ha[c]) * (xa[c] - ha[c]); gx += grav[c] * xa[c]; }
      if (E) *E += 0.5 * k * m[a] * d2 - m[a] * gx;
      if (g)
        for (int c = 0; c < 3; ++c) g[3 * a + c] += k * m[a] * (xa[c] - ha[c]) - m[a] * grav[c];
      if (vals) {
        const int32_t* c0 = o->col_idx.data() + o->row_ptr[a];
        const int32_t* c1 = o->col_idx.data() + o->row_ptr[a + 1];
        double* blk = vals + 9 * (size_t)(std::lower_bound(c0, c1, (int32_t)(j * nu + i)) - o->col_idx.data());
        for (int c = 0; c < 3; ++c) blk[4 * c] += k * m[a];
      }
    }
  if (pinned) {
    for (int j = o->r0; j < o->r1; ++j)
      for (int i = 0; i < nu; ++i) {
        const size_t a = (size_t)(j - o->r0) * nu + i;
        const bool pa = pinned[(size_t)j * nu + i] != 0;
        if (g && pa)
          for (int c = 0; c < 3; ++c) g[3 * a + c] = 0.0;
        if (!vals) continue;
        for (int32_t q = o->row_ptr[a]; q < o->row_ptr[a + 1]; ++q) {
          const int b = o->col_idx[q];
          if (!pa && !pinned[b]) continue;
          double* blk = vals + 9 * (size_t)q;
          for (int e = 0; e < 9; ++e) blk[e] = 0.0;
          if (b == j * nu + i)
            for (int c = 0; c < 3; ++c) blk[4 * c] = 1.0;
        }
      }
  }
  return 0;
}

// Exposed for the projection pins: the 6x6 F-space Hessian of the FBW density at F = (f1, f2).
int oracle_membrane_A(const double* mu4, const double* f6, int project, double* A36) {
  Oracle o;
  o.mu_st1 = mu4[0]; o.mu_st2 = mu4[1]; o.mu_sh = mu4[2]; o.mu_bd = mu4[3];
  double f[2][3] = {{f6[0], f6[1], f6[2]}, {f6[3], f6[4], f6[5]}}, A[6][6];
  membrane_A(o, f, project != 0, A);
  for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) A36[6 * i + j] = A[i][j];
  return 0;
}

// ------------------------------------------------------------------ contact pullback
// A contact-mesh vertex alpha sits at a fixed parametric point (u_alpha, v_alpha) of the sheet and moves with it,
//   x^alpha = sum_ij N_ij(u_alpha, v_alpha) C^ij       (Eq. `eq: trig mesh node from control
// points`), so a barrier B(x) on the mesh has, by the chain rule (Eq. `eq: gradient and hessian of
// contact barrier`; the second-derivative term vanishes because x is linear in C),
//   dB/dC^i = sum_alpha N_i(alpha) dB/dx^alpha,   d2B/dC^i dC^j = sum_{alpha,beta} N_i(alpha) d2B/dx^alpha dx^beta N_j(beta).
// The plain route: the dense weight of every control point for every vertex (Cox-de Boor over all bases), and a
// dense (3 n_cp)^2 Hessian that every pair's 3x3 vertex blocks are scattered into term by term.
// W: [nvert][n_v * n_u] (row-major, control point a = j n_u + i).
int oracle_contact_weights(void* h, int nvert, const double* uv, double* W) {
  auto* o = static_cast<Oracle*>(h);
  const int nu = o->n_u, nv = o->n_v;
  std::vector<double> Nu(nu), dNu(nu), ddNu(nu), Nv(nv), dNv(nv), ddNv(nv);
  for (int a = 0; a < nvert; ++a) {
    const double u = uv[2 * a], v = uv[2 * a + 1];
    if (!(u >= 0.0 && u <= o->Su && v >= 0.0 && v <= o->Sv)) return fail("contact vertex outside the parameter domain");
    cox_de_boor(o->ku.data(), nu + 3, u, Nu.data(), dNu.data(), ddNu.data());
    cox_de_boor(o->kv.data(), nv + 3, v, Nv.data(), dNv.data(), ddNv.data());
    for (int j = 0; j < nv; ++j)
      for (int i = 0; i < nu; ++i) W[(size_t)a * nu * nv + (size_t)j * nu + i] = Nu[i] * Nv[j];
  }
  return 0;
}

// Pairs: verts [npairs][4] (mesh vertex indices, -1 = a slot without control-point DOFs, e.g. an obstacle vertex),
// H [npairs][12][12] (the barrier Hessian of the pair w.r.t. its 4 vertex slots), gv [npairs][12] (its gradient; may
// be NULL).  Hcp: dense [3 n_cp][3 n_cp], gcp: [3 n_cp] (may be NULL); both overwritten.
int oracle_contact_pullback(void* h, int nvert, const double* uv, int npairs, const int32_t* verts, const double* H,
                            const double* gv, double* Hcp, double* gcp) {
  auto* o = static_cast<Oracle*>(h);
  const size_t ncp = (size_t)o->n_u * o->n_v, N3 = 3 * ncp;
  std::vector<double> W((size_t)nvert * ncp);
  if (oracle_contact_weights(h, nvert, uv, W.data())) return -1;
  std::fill(Hcp, Hcp + N3 * N3, 0.0);
  if (gcp) std::fill(gcp, gcp + N3, 0.0);
  for (int c = 0; c < npairs; ++c) {
    for (int sa = 0; sa < 4; ++sa) {
      const int al = verts[4 * c + sa];
      if (al < 0) continue;
      if (al >= nvert) return fail("contact pair vertex out of range");
      const double* wa = &W[(size_t)al * ncp];
      for (size_t i = 0; i < ncp; ++i) {
        if (wa[i] == 0.0) continue;
        if (gcp && gv)
          for (int r = 0; r < 3; ++r) gcp[3 * i + r] += wa[i] * gv[12 * c + 3 * sa + r];
        for (int sb = 0; sb < 4; ++sb) {
          const int be = verts[4 * c + sb];
          if (be < 0) continue;
          const double* wb = &W[(size_t)be * ncp];
          for (size_t j = 0; j < ncp; ++j) {
            if (wb[j] == 0.0) continue;
            for (int r = 0; r < 3; ++r)
              for (int q = 0; q < 3; ++q)
                Hcp[(3 * i + r) * N3 + 3 * j + q] += wa[i] * wb[j] * H[(size_t)144 * c + (3 * sa + r) * 12 + 3 * sb + q];
          }
        }
      }
    }
  }
  return 0;
}

int oracle_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
