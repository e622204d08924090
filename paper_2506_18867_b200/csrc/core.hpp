// Core path: the uniform interior of an affine sheet with the REDUCED rules (DESIGN.md §5 "k_core").
//
// In the interior every control point a = (i, j) sees the same quadrature configuration up to the
// parity pi = (i + j) & 1 of a (Fig. `fig: quadrature`; Q1):
//   - the dual cell centred on knot (p, q) holds two membrane Gauss points, along v on the knot line
//     u = p when p + q is even ("V-", "V+"), along u on v = q when p + q is odd ("H-", "H+");
//   - one bending point sits at every knot (8-cp right-limit stencil, D4).
// So the incidence of a's 12 membrane points on a's 23 BSR blocks is a compile-time table per parity
// (below), and every coefficient d_a,mu d_b,nu of H_ab = sum_q sum_{mu,nu} d_a,mu d_b,nu A~_mu,nu(q)
// (the paper's per-block gather) is a constant of the sheet, taken from the exact basis
// tables and verified against every control point at create time (core.cu, build_core).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>

#include "dev.hpp"
#include "host.hpp"

namespace bsf {
namespace core {

constexpr int kW = 32;            // strip width (control points); a warp = 32 same-parity cps of 2 rows
constexpr int kRows = 2;          // output rows per step
constexpr int kNB = 23;           // BSR blocks of an interior row
constexpr int kKC = kW + 3;       // knot columns of a strip window: p in [i0-2, i0+kW]
constexpr int kKH = (kKC + 1) / 2;  // entries of a parity-split knot array
constexpr int kRing = 7;          // knot rows resident: q in [j-2, j+4] (gather of step k, points of k+1)
constexpr int kGatherWarps = 9;   // one warp per block entry (r, c), both parities in turn
constexpr int kPointWarps = 7;    // the next step's 210 quadrature points (7 x 30 lanes)
constexpr int kThreads = 32 * (kGatherWarps + kPointWarps);
// channels of one membrane point record (SoA, stride kKH):
//   [0,6) A~uu (sym 3x3)   [6,12) A~vv (sym)   [12,21) A~uv (3r+c)   [21,24) P~u   [24,27) P~v
constexpr int kChan = 27;
constexpr int kSetD = kChan * kKH;            // doubles per membrane set of one ring row
constexpr int kBendD = 3 * kKH;               // doubles per bending parity array of one ring row
constexpr int kRowD = 4 * kSetD + 2 * kBendD; // doubles per ring row
constexpr int kPosC = kW + 6;                 // staged position columns: [i0-3, i0+kW+3)
constexpr int kPosStep = 5 * kPosC * 3;       // positions of the cp rows of 2 knot rows
constexpr int kPosD = 2 * kPosStep;           // double buffer (the 5-knot-row prologue uses 8 rows of it)
constexpr int kStageRow = kW * kNB * 9 + 2;   // doubles per staged output row (+ alignment slack)

// sets: 0 V- (u = p, v = q - g, anchor (p, q-1), stencil 2x3), 1 V+ (u = p, v = q + g, anchor (p, q)),
//       2 H- (u = p - g, v = q, anchor (p-1, q), 3x2),          3 H+ (u = p + g, v = q, anchor (p, q))
constexpr int set_adu(int set) { return set == 2 ? -1 : 0; }
constexpr int set_adv(int set) { return set == 0 ? -1 : 0; }
constexpr int set_nu(int set) { return set < 2 ? 2 : 3; }
constexpr int set_nv(int set) { return set < 2 ? 3 : 2; }

// Block index of column offset (di, dj) in an interior row (columns ascending; (-2,-2), (2,2) absent).
constexpr int block_index(int di, int dj) {
  if (dj == -2) return (di >= -1 && di <= 2) ? di + 1 : -1;
  if (dj == -1) return (di >= -2 && di <= 2) ? 4 + di + 2 : -1;
  if (dj == 0) return (di >= -2 && di <= 2) ? 9 + di + 2 : -1;
  if (dj == 1) return (di >= -2 && di <= 2) ? 14 + di + 2 : -1;
  if (dj == 2) return (di >= -2 && di <= 1) ? 19 + di + 2 : -1;
  return -1;
}
constexpr int block_di(int k) { return k < 4 ? k - 1 : k < 19 ? ((k - 4) % 5) - 2 : k - 21; }
constexpr int block_dj(int k) { return k < 4 ? -2 : k < 9 ? -1 : k < 14 ? 0 : k < 19 ? 1 : 2; }

constexpr int kMaxSlots = 12;
constexpr int kMaxContrib = 80;

// Membrane incidence of a control point of parity pi: its slots (incident points) and, per slot,
// the blocks b the point reaches (contributions).
struct Template {
  int nslot = 0, ncontrib = 0;
  int s_dp[kMaxSlots] = {}, s_dq[kMaxSlots] = {}, s_set[kMaxSlots] = {}, s_ea[kMaxSlots] = {};
  int s_c0[kMaxSlots] = {}, s_nc[kMaxSlots] = {};
  int c_blk[kMaxContrib] = {}, c_eb[kMaxContrib] = {}, c_slot[kMaxContrib] = {};
};

constexpr Template make_template(int pi) {
  Template T{};
  for (int set = 0; set < 4; ++set)           // slots grouped by point set (shared coefficient table)
  for (int dq = -2; dq <= 1; ++dq)
    for (int dp = -2; dp <= 1; ++dp) {
      const int kappa = (pi + dp + dq) & 1;   // knot (i+dp, j+dq): even -> V pair, odd -> H pair
      {
        if ((set >> 1) != kappa) continue;
        const int s = dp + set_adu(set), t = dq + set_adv(set);   // anchor relative to a
        const int iu = -s, jv = -t;                                 // a's window entry
        if (iu < 0 || iu >= set_nu(set) || jv < 0 || jv >= set_nv(set)) continue;
        const int k = T.nslot++;
        T.s_dp[k] = dp; T.s_dq[k] = dq; T.s_set[k] = set; T.s_ea[k] = iu + 3 * jv;
        T.s_c0[k] = T.ncontrib;
        for (int jb = 0; jb < set_nv(set); ++jb)
          for (int ib = 0; ib < set_nu(set); ++ib) {
            const int c = T.ncontrib++;
            T.c_blk[c] = block_index(s + ib, t + jb);
            T.c_eb[c] = ib + 3 * jb;
            T.c_slot[c] = k;
          }
        T.s_nc[k] = T.ncontrib - T.s_c0[k];
      }
    }
  return T;
}

// Per-set parametric d-vectors (dN/du Nv, Nu dN/dv) of the 9 window entries of an interior point:
// uniform quadratic bases on a span with local coordinate x, N = ((1-x)^2/2, (1+2x-2x^2)/2, x^2/2),
// N' = (x-1, 1-2x, x); at a knot (right limit, x = 0) N = (1/2, 1/2, 0), N' = (-1, 1, 0); the Gauss
// pair of a dual cell sits at x = g (span q / p) and x = 1-g (span q-1 / p-1), g = sqrt(3)/6 (the
// rule's node literal, host.cpp).  Compile-time, so the gather's coefficients are immediates; create
// time verifies every interior point's own tables against it (relative 1e-12).
struct SetTable { double v[4][9][2]; };
constexpr double kGauss = 0.28867513459481288225;
constexpr SetTable make_set_table() {
  SetTable T{};
  const double xs[2] = {1.0 - kGauss, kGauss};   // set w = 0 (minus), 1 (plus)
  for (int set = 0; set < 4; ++set) {
    const double x = xs[set & 1];
    const double Ng[3] = {0.5 * (1.0 - x) * (1.0 - x), 0.5 * (1.0 + 2.0 * x - 2.0 * x * x), 0.5 * x * x};
    const double dg[3] = {x - 1.0, 1.0 - 2.0 * x, x};
    const double Nk[3] = {0.5, 0.5, 0.0}, dk[3] = {-1.0, 1.0, 0.0};
    for (int e = 0; e < 9; ++e) {
      const int iu = e % 3, jv = e / 3;
      const bool V = set < 2;   // V: u on the knot line, v at the Gauss node; H: the reverse
      const double Nu = V ? Nk[iu] : Ng[iu], du = V ? dk[iu] : dg[iu];
      const double Nv = V ? Ng[jv] : Nk[jv], dv = V ? dg[jv] : dk[jv];
      const bool in = V ? iu < 2 : jv < 2;
      T.v[set][e][0] = in ? du * Nv : 0.0;
      T.v[set][e][1] = in ? Nu * dv : 0.0;
    }
  }
  return T;
}
constexpr SetTable kSetTable = make_set_table();

// Bending incidence: knots (i+dp, j+dq), dp, dq in [-2, 0], a at window entry (-dp, -dq) != (2, 2).
constexpr int kBSlots = 8;
constexpr int bslot_dp(int k) { return -(k % 3); }   // slot k: a sits at window entry k of the point
constexpr int bslot_dq(int k) { return -(k / 3); }

}  // namespace core

struct CoreTables {
  int ok = 0;
  int CI0 = 0, CI1 = 0, CJ0 = 0, CJ1 = 0;   // interior rectangle of control points (global indices)
  int RJ0 = 0, RJ1 = 0;                      // owned rows of the rectangle ([CJ0,CJ1) ∩ [r0,r1))
  int nstrips = 0;
  size_t smem = 0;
  // host copies of the constant tables (uploaded to __constant__ memory at every launch's first use)
  double K[2][core::kMaxContrib][4] = {};   // k_uu, k_vv, (k_uv + k_vu)/2, (k_uv - k_vu)/2
  double D[2][core::kMaxSlots][2] = {};     // d_a of the slot's point (gradient)
  double S[4][9][2] = {};                   // per set: (dN/du Nv, Nu dN/dv) per window entry
  double LA[9] = {}, LB[9] = {}, LC[9] = {}; // bending: N''u Nv, Nu N''v, N'u N'v per window entry
  double what[5] = {};                       // parametric weights: sets 0-3, bending
  double G[4] = {}, detJ = 0;                // handle's own affine map
  int32_t* row_ptr = nullptr;                // device copy (owned rows)
  int64_t rp_base = 0, rp_stride = 0;        // row_ptr of (CI0, j) = rp_base + (j - RJ0) * rp_stride
  double* d_tabs = nullptr;                  // device copy of S | LA | LB | LC | what
  // Curved (non-affine) rest map (round 2): the interior template is the same (it is parametric), but G, w and the
  // Laplacian coefficients vary per point, and the bending Hessian is no longer one table per CTA.  The kernel
  // streams them from these device tables ("can be precomputed"):
  int curved = 0;
  int64_t kp = 0;                   // knot pitch: Su + 1
  double* mtab = nullptr;           // [Sv+1][2][5][Su+1]: the two membrane points (minus, plus) of the dual cell of
                                    // knot (p, q): G00 G01 G10 G11 w
  double* btab = nullptr;           // [Sv+1][10][Su+1]: the bending point at knot (p, q): L_0..L_8 (G-contracted), w
  int64_t cw = 0;                   // core columns CI1 - CI0
  double* beta = nullptr;           // [RJ1-RJ0][23][cw]: sum over the cp's bending points of w L_a L_b (x mu_bd at run time)
  double* gw = nullptr;             // [RJ1-RJ0][8][cw]: w L_a of the cp's 8 bending slots (x mu_bd at run time)
  size_t table_bytes = 0;           // bytes of the four tables (read once per call)
};

// Build (and verify) the interior tables; returns 0 with ok = 1, 1 if the sheet has no usable
// interior (ok = 0, the tile path covers everything), < 0 on an internal error.
int build_core(const Sheet& sh, const int32_t* d_row_ptr, CoreTables& ct, std::string& err,
               const std::function<void*(size_t)>& dalloc);

// Launch the core kernel over nbatch items.  e_part: per-item energy partials at
// e_part[item * e_stride + e_off + cta]; the number of CTAs per item is returned in *nctas.
int core_eval(const CoreTables& ct, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, double* e_part,
              int64_t e_stride, int64_t e_off, int nchunks, const double* d_params, double detJ_ref,
              cudaStream_t st, const struct IpFused* ip = nullptr, int row_begin = -1, int row_end = -1);

int core_ctas_per_item(const CoreTables& ct, int nchunks);
// Row chunks per (strip, item).  reserved_sms: SMs the band / corner kernels beside k_core occupy (a small
// problem runs one wave of k_core next to them).
int core_pick_chunks(const CoreTables& ct, int nbatch, int rows = -1, int reserved_sms = 0);

}  // namespace bsf
