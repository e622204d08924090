// Host-side precompute for the B200 library: basis tables, rules, rest-map coefficients, pattern.
// Independent implementation (no code shared with oracle/).  Paper: /root/reference/PAPER.md.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <string>

namespace bsf {

// ------------------------------------------------------------------ basis (A2.2 / A2.3, p = 2)
// Knot vector U (0-indexed) of the open uniform integer sheet: U[0..2] = 0, U[2+t] = t, U[S+2..S+4] = S.
static inline double knot(int S, int k) {
  if (k <= 2) return 0.0;
  if (k >= S + 2) return (double)S;
  return (double)(k - 2);
}

void basis1(int S, double x, Basis1& out) {
  const int p = 2;
  int s = (int)std::floor(x);
  if (s >= S) s = S - 1;
  if (s < 0) s = 0;
  const int i = s + 2;  // knot-span index: U[i] <= x < U[i+1]
  double ndu[3][3], left[3], right[3];
  ndu[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = x - knot(S, i + 1 - j);
    right[j] = knot(S, i + j) - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];       // knot differences (lower triangle)
      const double temp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * temp;      // basis values (upper triangle)
      saved = left[j - r] * temp;
    }
    ndu[j][j] = saved;
  }
  double ders[3][3];
  for (int j = 0; j <= p; ++j) ders[0][j] = ndu[j][p];
  double a[2][3];
  for (int r = 0; r <= p; ++r) {
    int s1 = 0, s2 = 1;
    a[0][0] = 1.0;
    for (int k = 1; k <= 2; ++k) {
      double d = 0.0;
      const int rk = r - k, pk = p - k;
      if (r >= k) {
        a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
        d = a[s2][0] * ndu[rk][pk];
      }
      const int j1 = (rk >= -1) ? 1 : -rk;
      const int j2 = (r - 1 <= pk) ? k - 1 : p - r;
      for (int j = j1; j <= j2; ++j) {
        a[s2][j] = (a[s1][j] - a[s1][j - 1]) / ndu[pk + 1][rk + j];
        d += a[s2][j] * ndu[rk + j][pk];
      }
      if (r <= pk) {
        a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
        d += a[s2][k] * ndu[r][pk];
      }
      ders[k][r] = d;
      std::swap(s1, s2);
    }
  }
  out.span = s;
  for (int j = 0; j < 3; ++j) {
    out.N[j] = ders[0][j];
    out.d1[j] = ders[1][j] * 2.0;   // multiply by p
    out.d2[j] = ders[2][j] * 2.0;   // multiply by p (p-1)
  }
}

// ------------------------------------------------------------------ rules
namespace {
const double kG2 = 0.28867513459481288225;   // sqrt(3)/6: G2 nodes at centre -/+ h*kG2*2 ... (see g2)
void g2(double a, double b, double* x, double* w) {
  const double c = 0.5 * (a + b), h = b - a;
  x[0] = c - h * kG2;
  x[1] = c + h * kG2;
  w[0] = w[1] = 0.5 * h;
}
void g3(double a, double b, double* x, double* w) {
  const double c = 0.5 * (a + b), h = b - a;
  const double o = 0.38729833462074168852;   // sqrt(15)/10
  x[0] = c - h * o; x[1] = c; x[2] = c + h * o;
  w[0] = w[2] = h * (5.0 / 18.0);
  w[1] = h * (8.0 / 18.0);
}
void tensor(std::vector<RulePoint>& out, int nu, int nv, int s, int t) {
  double xu[3], wu[3], xv[3], wv[3];
  if (nu == 3) g3(s, s + 1, xu, wu); else if (nu == 2) g2(s, s + 1, xu, wu); else { xu[0] = s + 0.5; wu[0] = 1; }
  if (nv == 3) g3(t, t + 1, xv, wv); else if (nv == 2) g2(t, t + 1, xv, wv); else { xv[0] = t + 0.5; wv[0] = 1; }
  for (int b = 0; b < nv; ++b)
    for (int a = 0; a < nu; ++a) out.push_back({xu[a], xv[b], wu[a] * wv[b], false, false});
}
}  // namespace

void make_rule(int kind, bool bending, int Su, int Sv, std::vector<RulePoint>& out) {
  out.clear();
  // Span-anchored points.  Boundary frame of the REDUCED rules (Fig. 4 grey spans):
  // membrane 3x3 at corner spans, (2 along the edge) x 3 on side spans; bending one point at the
  // centre of every boundary span.
  for (int t = 0; t < Sv; ++t)
    for (int s = 0; s < Su; ++s) {
      const bool eu = (s == 0 || s == Su - 1), ev = (t == 0 || t == Sv - 1);
      if (kind == RULE_G3_FULL) { tensor(out, 3, 3, s, t); continue; }
      if (eu || ev) {
        if (bending) tensor(out, 1, 1, s, t);
        else tensor(out, eu ? 3 : 2, ev ? 3 : 2, s, t);
      } else if (kind == RULE_G2_INTERIOR) {
        tensor(out, 2, 2, s, t);
      }
    }
  if (kind != RULE_REDUCED) return;
  // Knot-anchored points of the interior region [1, Su-1] x [1, Sv-1] (dual grid).
  for (int q = 1; q < Sv; ++q)
    for (int p = 1; p < Su; ++p) {
      const double cu = (p == 1 || p == Su - 1) ? 0.5 : 1.0;   // clipped dual-cell extents (Q2)
      const double cv = (q == 1 || q == Sv - 1) ? 0.5 : 1.0;
      if (bending) {  // one point at the dual-cell centre = the knot
        out.push_back({(double)p, (double)q, cu * cv, true, true});
        continue;
      }
      if (cu < 1.0 && cv < 1.0) {  // quarter cell: a single point at the knot
        out.push_back({(double)p, (double)q, 0.25, true, true});
        continue;
      }
      // Gauss pair along v (u = p on the knot line) or along u (v = q), alternating on the dual
      // grid by the parity of p+q (Q1); half cells on the region's edges keep their knot line.
      const bool along_v = (cu < 1.0) ? true : (cv < 1.0) ? false : ((p + q) % 2 == 0);
      double x[2], w[2];
      if (along_v) {
        g2(q - 0.5, q + 0.5, x, w);
        for (int k = 0; k < 2; ++k) out.push_back({(double)p, x[k], w[k] * cu * cv, true, false});
      } else {
        g2(p - 0.5, p + 0.5, x, w);
        for (int k = 0; k < 2; ++k) out.push_back({x[k], (double)q, w[k] * cu * cv, false, true});
      }
    }
}

// ------------------------------------------------------------------ per-point coefficients
uint16_t stencil_mask(bool bending, bool ku, bool kv) {
  // value/first-derivative entries: {0,1} on a knot line, {0,1,2} inside a span;
  // second-derivative entries (right limit): always {0,1,2}.
  const int vu = ku ? 0x3 : 0x7, vv = kv ? 0x3 : 0x7, du = 0x7, dv = 0x7;
  uint16_t m = 0;
  for (int jv = 0; jv < 3; ++jv)
    for (int iu = 0; iu < 3; ++iu) {
      const bool Vu = (vu >> iu) & 1, Vv = (vv >> jv) & 1, Du = (du >> iu) & 1, Dv = (dv >> jv) & 1;
      const bool in = bending ? ((Du && Vv) || (Vu && Dv)) : (Vu && Vv);
      if (in) m |= (uint16_t)(1u << win_entry(iu, jv));
    }
  return m;
}

static int eval_point(const Sheet& sh, const RulePoint& q, bool bending, Point& P, std::string& err) {
  P.bending = bending;
  basis1(sh.Su, q.u, P.bu);
  basis1(sh.Sv, q.v, P.bv);
  P.ou = P.bu.span;
  P.ov = P.bv.span;
  P.mask = stencil_mask(bending, q.knot_u, q.knot_v);
  // rest-map derivatives over the 3x3 window (all bases that can be nonzero at the point)
  double Xu[2] = {0, 0}, Xv[2] = {0, 0}, Xuu[2] = {0, 0}, Xvv[2] = {0, 0}, Xuv[2] = {0, 0};
  for (int jv = 0; jv < 3; ++jv)
    for (int iu = 0; iu < 3; ++iu) {
      const double* X = &sh.rest[2 * ((size_t)(P.ov + jv) * sh.n_u + (P.ou + iu))];
      for (int c = 0; c < 2; ++c) {
        Xu[c] += P.bu.d1[iu] * P.bv.N[jv] * X[c];
        Xv[c] += P.bu.N[iu] * P.bv.d1[jv] * X[c];
        Xuu[c] += P.bu.d2[iu] * P.bv.N[jv] * X[c];
        Xvv[c] += P.bu.N[iu] * P.bv.d2[jv] * X[c];
        Xuv[c] += P.bu.d1[iu] * P.bv.d1[jv] * X[c];
      }
    }
  const double det = Xu[0] * Xv[1] - Xv[0] * Xu[1];
  if (!(det > 0.0)) {
    err = "degenerate rest geometry: det(dX/d(u,v)) <= 0 at parametric point (" + std::to_string(q.u) + ", " +
          std::to_string(q.v) + ")";
    return -4;
  }
  // G = (dX/d(u,v))^{-1}: rows are grad u and grad v in material space (inverse function theorem)
  P.G[0][0] = Xv[1] / det;  P.G[0][1] = -Xv[0] / det;
  P.G[1][0] = -Xu[1] / det; P.G[1][1] = Xu[0] / det;
  P.what = q.what;
  P.detJ = det;
  P.w = q.what * det;
  // Laplacian coefficients: grad u . grad u, grad v . grad v, 2 grad u . grad v, Lap u, Lap v.
  // Lap r = - sum_c G[r][c] tr(G^T Hess(X_c) G)   (second-order inverse function theorem)
  P.c_uu = P.G[0][0] * P.G[0][0] + P.G[0][1] * P.G[0][1];
  P.c_vv = P.G[1][0] * P.G[1][0] + P.G[1][1] * P.G[1][1];
  P.c_uv = 2.0 * (P.G[0][0] * P.G[1][0] + P.G[0][1] * P.G[1][1]);
  double trc[2];
  for (int c = 0; c < 2; ++c) {
    // tr(G^T Hc G) = sum_k (G e_k)^T Hc (G e_k) with columns of G: (G[0][k], G[1][k])
    double t = 0;
    for (int k = 0; k < 2; ++k) {
      const double a = P.G[0][k], b = P.G[1][k];
      t += a * a * Xuu[c] + 2.0 * a * b * Xuv[c] + b * b * Xvv[c];
    }
    trc[c] = t;
  }
  P.c_u = -(P.G[0][0] * trc[0] + P.G[0][1] * trc[1]);
  P.c_v = -(P.G[1][0] * trc[0] + P.G[1][1] * trc[1]);
  for (int jv = 0; jv < 3; ++jv)
    for (int iu = 0; iu < 3; ++iu) {
      const int e = win_entry(iu, jv);
      const bool in = (P.mask >> e) & 1;
      const double Nu_ = P.bu.d1[iu] * P.bv.N[jv], Nv_ = P.bu.N[iu] * P.bv.d1[jv];
      P.b[e][0] = in ? Nu_ * P.G[0][0] + Nv_ * P.G[1][0] : 0.0;
      P.b[e][1] = in ? Nu_ * P.G[0][1] + Nv_ * P.G[1][1] : 0.0;
      const double Nuu = P.bu.d2[iu] * P.bv.N[jv], Nvv = P.bu.N[iu] * P.bv.d2[jv], Nuv = P.bu.d1[iu] * P.bv.d1[jv];
      P.L[e] = in ? P.c_uu * Nuu + P.c_vv * Nvv + P.c_uv * Nuv + P.c_u * Nu_ + P.c_v * Nv_ : 0.0;
    }
  return 0;
}

int lumped_mass(const Sheet& sh, double R0, std::vector<double>& m, std::string& err) {
  const int nu = sh.n_u;
  m.assign((size_t)(sh.r1 - sh.r0) * nu, 0.0);
  double xu[3], wu[3], xv[3], wv[3];
  for (int t = std::max(0, sh.r0 - 2); t < std::min(sh.Sv, sh.r1); ++t) {   // spans touching owned rows
    g3(t, t + 1, xv, wv);
    for (int s = 0; s < sh.Su; ++s) {
      g3(s, s + 1, xu, wu);
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          Basis1 bu, bv;
          basis1(sh.Su, xu[a], bu);
          basis1(sh.Sv, xv[b], bv);
          double Xu[2] = {0, 0}, Xv[2] = {0, 0};
          for (int jv = 0; jv < 3; ++jv)
            for (int iu = 0; iu < 3; ++iu) {
              const double* X = &sh.rest[2 * ((size_t)(bv.span + jv) * nu + (bu.span + iu))];
              for (int c = 0; c < 2; ++c) {
                Xu[c] += bu.d1[iu] * bv.N[jv] * X[c];
                Xv[c] += bu.N[iu] * bv.d1[jv] * X[c];
              }
            }
          const double det = Xu[0] * Xv[1] - Xv[0] * Xu[1];
          if (!(det > 0.0)) { err = "degenerate rest geometry at a mass quadrature point"; return -4; }
          const double w = wu[a] * wv[b] * det * R0;
          for (int jv = 0; jv < 3; ++jv) {
            const int j = bv.span + jv;
            if (j < sh.r0 || j >= sh.r1) continue;
            for (int iu = 0; iu < 3; ++iu) m[(size_t)(j - sh.r0) * nu + bu.span + iu] += w * bu.N[iu] * bv.N[jv];
          }
        }
    }
  }
  return 0;
}

int build_sheet(int n_u, int n_v, const double* ku, const double* kv, const double* rest_xy, int mrule,
                int brule, int r0, int r1, Sheet& sh, std::string& err) {
  if (n_u < 3 || n_v < 3) { err = "need at least 3 control points per direction"; return -3; }
  for (int d = 0; d < 2; ++d) {
    const int n = d ? n_v : n_u, S = n - 2;
    const double* k = d ? kv : ku;
    for (int t = 0; t < n + 3; ++t)
      if (k[t] != knot(S, t)) { err = "knot vectors must be open, uniform and integer: (0,0,0,1,...,S,S,S)"; return -2; }
  }
  if (mrule < 0 || mrule > 2 || brule < 0 || brule > 2) { err = "unknown quadrature rule"; return -1; }
  if ((mrule != RULE_G3_FULL || brule != RULE_G3_FULL) && (n_u < 5 || n_v < 5)) {
    err = "reduced / G2-interior rules need at least 3 knot spans per direction";
    return -3;
  }
  if (r0 < 0 || r1 > n_v || r0 >= r1) { err = "invalid owned row range"; return -1; }
  sh.n_u = n_u; sh.n_v = n_v; sh.Su = n_u - 2; sh.Sv = n_v - 2;
  sh.r0 = r0; sh.r1 = r1;
  sh.mrule = mrule; sh.brule = brule;
  sh.xlo = std::max(0, r0 - 2); sh.xhi = std::min(n_v, r1 + 2);
  sh.rest.assign(rest_xy, rest_xy + (size_t)2 * n_u * n_v);
  sh.mem.clear(); sh.bend.clear(); sh.mem_eown.clear(); sh.bend_eown.clear();
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<RulePoint> rp;
    make_rule(pass ? brule : mrule, pass == 1, sh.Su, sh.Sv, rp);
    for (const RulePoint& q : rp) {
      const int ov = std::min((int)std::floor(q.v), sh.Sv - 1);
      if (ov < r0 - 2 || ov > r1 - 1) continue;   // anchor rows of the slab window
      Point P;
      const int rc = eval_point(sh, q, pass == 1, P, err);
      if (rc) return rc;
      // keep every point anchored in rows [r0-2, r1): the anchors of a slab are then complete, so
      // gather programs built for one control point are valid for every control point of its class
      int jmin = 3;
      for (int e = 0; e < 9; ++e)
        if ((P.mask >> e) & 1) jmin = std::min(jmin, e / 3);
      if (P.ov < r0 - 2 || P.ov > r1 - 1) continue;
      const uint8_t own = (P.ov + jmin >= r0 && P.ov + jmin < r1) ? 1 : 0;
      if (pass) { sh.bend.push_back(P); sh.bend_eown.push_back(own); }
      else { sh.mem.push_back(P); sh.mem_eown.push_back(own); }
    }
  }
  // affine detection: constant G and det J, vanishing second-order terms, up to the rounding of the
  // rest-map evaluation (it grows with the parametric coordinate: 2.3e-13 relative at 1024^2; a
  // Greville sheet stays affine up to ~1e5 spans with the 1e-11 bound)
  {
    bool aff = true;
    const std::vector<Point>* lists[2] = {&sh.mem, &sh.bend};
    const Point* ref = sh.mem.empty() ? (sh.bend.empty() ? nullptr : &sh.bend[0]) : &sh.mem[0];
    if (ref) {
      const double gs = std::fabs(ref->G[0][0]) + std::fabs(ref->G[0][1]) + std::fabs(ref->G[1][0]) + std::fabs(ref->G[1][1]);
      for (auto* L : lists)
        for (const Point& P : *L) {
          for (int r = 0; r < 2 && aff; ++r)
            for (int c = 0; c < 2; ++c)
              if (std::fabs(P.G[r][c] - ref->G[r][c]) > 1e-11 * gs) aff = false;
          if (std::fabs(P.c_u) > 1e-11 * gs * gs || std::fabs(P.c_v) > 1e-11 * gs * gs) aff = false;
          if (!aff) break;
        }
    }
    sh.affine = aff;
  }
  // pattern: diagonal + union over points of (stencil x stencil), restricted to owned rows
  const int nrows = (r1 - r0) * n_u;
  std::vector<std::vector<int32_t>> cols(nrows);
  for (int a = 0; a < nrows; ++a) cols[a].push_back(r0 * n_u + a);
  const std::vector<Point>* lists[2] = {&sh.mem, &sh.bend};
  for (auto* L : lists)
    for (const Point& P : *L) {
      int members[9], nm = 0;
      for (int e = 0; e < 9; ++e)
        if ((P.mask >> e) & 1) members[nm++] = (P.ov + e / 3) * n_u + P.ou + e % 3;
      for (int x = 0; x < nm; ++x) {
        const int row = members[x] / n_u;
        if (row < r0 || row >= r1) continue;
        auto& c = cols[members[x] - r0 * n_u];
        c.insert(c.end(), members, members + nm);
      }
    }
  sh.row_ptr.assign(nrows + 1, 0);
  for (int a = 0; a < nrows; ++a) {
    auto& c = cols[a];
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    sh.row_ptr[a + 1] = sh.row_ptr[a] + (int32_t)c.size();
  }
  sh.col_idx.resize(sh.row_ptr[nrows]);
  for (int a = 0; a < nrows; ++a) std::copy(cols[a].begin(), cols[a].end(), sh.col_idx.begin() + sh.row_ptr[a]);
  return 0;
}

// Step a2 for a flat affine rest sheet (J = dX/d(u,v), G = J^-1, w = what det J): the rest
// map evaluated at the centre of every knot span must have one constant J (to 1e-11 of |J|, the test
// build_sheet applies) and vanishing second derivatives (no Laplacian coefficients c_u, c_v).  out[9] =
// G00 G01 G10 G11 det J mu_st1 mu_st2 mu_sh mu_bd, the per-item layout of bsf_eval_all_batch_params.
int affine_params(int n_u, int n_v, const double* rest_xy, const double mu[4], double out[9], std::string& err) {
  if (n_u < 3 || n_v < 3) { err = "need at least 3 control points per direction"; return -3; }
  const int Su = n_u - 2, Sv = n_v - 2;
  double J0[2][2] = {{0, 0}, {0, 0}}, jn = 0.0;
  for (int t = 0; t < Sv; ++t)
    for (int s = 0; s < Su; ++s) {
      Basis1 bu, bv;
      basis1(Su, s + 0.5, bu);
      basis1(Sv, t + 0.5, bv);
      double Xu[2] = {0, 0}, Xv[2] = {0, 0}, X2[3][2] = {{0, 0}, {0, 0}, {0, 0}};
      for (int jv = 0; jv < 3; ++jv)
        for (int iu = 0; iu < 3; ++iu) {
          const double* X = &rest_xy[2 * ((size_t)(bv.span + jv) * n_u + (bu.span + iu))];
          for (int c = 0; c < 2; ++c) {
            Xu[c] += bu.d1[iu] * bv.N[jv] * X[c];
            Xv[c] += bu.N[iu] * bv.d1[jv] * X[c];
            X2[0][c] += bu.d2[iu] * bv.N[jv] * X[c];
            X2[1][c] += bu.N[iu] * bv.d2[jv] * X[c];
            X2[2][c] += bu.d1[iu] * bv.d1[jv] * X[c];
          }
        }
      const double det = Xu[0] * Xv[1] - Xv[0] * Xu[1];
      if (!(det > 0.0)) {
        err = "degenerate rest geometry: det(dX/d(u,v)) <= 0 in span (" + std::to_string(s) + ", " + std::to_string(t) + ")";
        return -4;
      }
      if (s == 0 && t == 0) {
        J0[0][0] = Xu[0]; J0[1][0] = Xu[1]; J0[0][1] = Xv[0]; J0[1][1] = Xv[1];
        jn = std::fabs(Xu[0]) + std::fabs(Xu[1]) + std::fabs(Xv[0]) + std::fabs(Xv[1]);
        continue;
      }
      bool ok = std::fabs(Xu[0] - J0[0][0]) <= 1e-11 * jn && std::fabs(Xu[1] - J0[1][0]) <= 1e-11 * jn &&
                std::fabs(Xv[0] - J0[0][1]) <= 1e-11 * jn && std::fabs(Xv[1] - J0[1][1]) <= 1e-11 * jn;
      for (int k = 0; k < 3 && ok; ++k) ok = std::fabs(X2[k][0]) + std::fabs(X2[k][1]) <= 1e-11 * jn;
      if (!ok) {
        err = "rest map is not affine (span (" + std::to_string(s) + ", " + std::to_string(t) + ") differs)";
        return -1;
      }
    }
  const double det = J0[0][0] * J0[1][1] - J0[0][1] * J0[1][0];
  out[0] = J0[1][1] / det;  out[1] = -J0[0][1] / det;
  out[2] = -J0[1][0] / det; out[3] = J0[0][0] / det;
  out[4] = det;
  for (int k = 0; k < 4; ++k) out[5 + k] = mu[k];
  return 0;
}

}  // namespace bsf
