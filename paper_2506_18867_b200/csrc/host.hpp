// Host-side precompute of the B200 assembly library (bsf_create).  Shares no code with oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bsf {

// Values and first/second derivatives of the three quadratic bases that are active on the
// (right-limit) span containing x: bases span, span+1, span+2.
struct Basis1 {
  int span;
  double N[3], d1[3], d2[3];
};

// Evaluate on the open uniform integer knot vector of S spans with the
// textbook span-local algorithm (Piegl & Tiller A2.2/A2.3; the paper cites that book at
// PAPER.md:151).  The span is chosen with the half-open convention of Eq. `eq: B-spline basis`
// (PAPER.md:156): x in [s, s+1) -> s, so quantities at a knot are right limits; x == S -> S-1.
void basis1(int S, double x, Basis1& out);

enum RuleKind { RULE_REDUCED = 0, RULE_G2_INTERIOR = 1, RULE_G3_FULL = 2 };

struct RulePoint {
  double u, v, what;     // parametric position, parametric weight
  bool knot_u, knot_v;   // coordinate lies on an interior knot line
};

// Quadrature points of one energy on an Su x Sv-span sheet (Fig. 4).
void make_rule(int kind, bool bending, int Su, int Sv, std::vector<RulePoint>& out);

// One quadrature point with everything the kernels need.  The stencil lives in the 3x3 window of
// bases [ou, ou+2] x [ov, ov+2]; bit (3*jv + iu) of `mask` marks the structural members.
struct Point {
  bool bending;
  int ou, ov;
  uint16_t mask;
  Basis1 bu, bv;
  double what, detJ;              // parametric weight and det(dX/d(u,v))
  double w;                       // what * det J
  double G[2][2];                 // G[r][c] = d r / d X_c, r in {u, v}
  double c_uu, c_vv, c_uv, c_u, c_v;  // Laplacian coefficients
  // stencil coefficients for window entry e = 3*jv + iu:
  double b[9][2];                 // membrane: b_e = G^T (dN/du, dN/dv)
  double L[9];                    // bending:  Laplacian coefficient
};

struct Geometry {  // result of validating and evaluating the rest map at a point
  int status;
  std::string msg;
};

struct Sheet {
  int n_u, n_v, Su, Sv;
  int r0, r1;          // owned cp rows
  int xlo, xhi;        // rows present in the position array
  std::vector<double> rest;  // [n_v][n_u][2]
  std::vector<Point> mem, bend;       // points whose stencil touches the owned rows
  std::vector<uint8_t> mem_eown, bend_eown;  // 1 if the point's energy is counted by this slab
  std::vector<int32_t> row_ptr, col_idx;     // owned block rows
  bool affine = false;                        // G, det J constant and no second-order terms
  int mrule = 0, brule = 0;
};

// Build the sheet: validates knots (status -2), sizes (-3), rest geometry (-4); returns 0 or the
// negative status with a message in err.
int build_sheet(int n_u, int n_v, const double* ku, const double* kv, const double* rest_xy,
                int mrule, int brule, int r0, int r1, Sheet& sh, std::string& err);

// Lumped mass of the owned control points (Q13): m_a = int R0 N_a dX (the row
// sum of the consistent mass matrix) by 3x3 Gauss per knot span.
// m: [owned rows][n_u].  Returns 0 or -4 (det J <= 0 at a mass point, message in err).
int lumped_mass(const Sheet& sh, double R0, std::vector<double>& m, std::string& err);

// Per-item parameters of a flat affine rest sheet (step a2; bsf_affine_params): out[9] = G00 G01 G10 G11
// det J mu[0..3].  Returns 0, -3 (too small), -4 (det J <= 0) or -1 (the rest map is not affine).
int affine_params(int n_u, int n_v, const double* rest_xy, const double mu[4], double out[9], std::string& err);

// Index helpers
inline int win_entry(int iu, int jv) { return 3 * jv + iu; }

// Structural stencil mask of a point (bit 3*jv+iu of its 3x3 window; Q10, D4).
uint16_t stencil_mask(bool bending, bool knot_u, bool knot_v);

}  // namespace bsf
