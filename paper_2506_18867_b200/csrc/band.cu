// k_band: the four edge bands of the frame (DESIGN.md §5 "k_band").
//
// Between the core rectangle and a sheet edge the quadrature configuration changes with the distance to
// the edge (clipped dual cells, boundary Gauss rules, open-knot end bases) but
// not along the edge, except for the knot parity: a band cp (s, t) (s along the edge, t across) sees the
// same points as (s + 2, t) shifted by two spans.  The host therefore builds, per band,
//   - point classes: the points of one anchor cell, keyed by (anchor along parity, anchor depth, index),
//     verified bit for bit against every anchor cell of the band (basis values, weight, stencil mask);
//   - one template per (parity, depth row): the incident points of a representative cp as
//     (class, anchor pair offset, position ea of the cp in the point's 3x3 window).
// One CTA per (band, 16 along cps, batch item):
//   1. stage positions; evaluate every point of the CTA's anchor window into shared memory in the
//      parametric frame (A~ = w (G (x) I) A (G (x) I)^T, P~ = w G P; bending
//      sqrt(w mu) Lap phi), one record channel per stride kMS (lanes read consecutive
//      anchor pairs);
//   2. gather: a warp = 8 same-parity cps x 4 block entries (r, c) of one depth row; per incident point
//          Y_u = d_a,u A~uu[r][c] + d_a,v A~uv[c][r],   Y_v = d_a,u A~uv[r][c] + d_a,v A~vv[r][c]
//          H_ab[r][c] += d_b,u Y_u + d_b,v Y_v   for the 9 cps b of the point's window
//      (H_ab = sum_q sum_{mu,nu} d_a,mu d_b,nu A~_mu,nu(q), the per-block gather of PAPER.md:705), with
//      the 25 block accumulators in registers (a switch on the warp-uniform ea makes every index a
//      compile-time constant); the bending part sum_q' w mu L_a L_b I3 is added on the diagonal entries,
//      and 3 more lanes per cp gather g_a = sum_q d_a . P~(q) + sum_q' sqrt(w mu) L_a sqrt(w mu) Lap phi;
//   3. each lane stores its entries of its cp's row (no staging: a warp store covers 8 rows x 4
//      adjacent doubles).
// Band rows are disjoint from the core's and from the corner tiles of k_frame.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "core.hpp"
#include "fbw.cuh"
#include "frame.hpp"
#include "ip.hpp"

namespace bsf {

namespace {
using namespace band;

struct BandArgs {
  const double* x;
  int64_t xs;
  double* g;
  int64_t gs;
  double* vals;
  int64_t vs;
  double* epart;
  int64_t e_stride, e_off;
  const int32_t* row_ptr;
  const double* params;
  int n_u, xlo, xhi, r0;
  int project, flags, dbg;
  unsigned long long* sflag;   // singular-stretch word (fbw.cuh)
  EFinal ef;                   // fused energy reduction of the call
  double G00, G01, G10, G11, detJ, mu1, mu2, mush, mubd;
  const double2* mcf;
  const int2* mcls;
  const double* mwhat;
  const double* bcf;
  const int2* bcls;
  const double* bwhat;
  // band descriptors in the kernel parameter space (constant bank)
  int nbands;
  int cfirst[5];                  // first CTA (blockIdx.x) of each band
  BandDesc desc[4];
  const uint32_t* ent;            // template entries of all bands
  const double2* entd;            // per entry (d_a,u, d_a,v) at its window position (membrane; 0 for bending)
  // incremental-potential terms (Q13; xhat == nullptr: elastic only)
  const double* xhat;
  int64_t xhs;
  const double* mass;
  double ipk, grav[3];
  const double* ipar;      // optional per-item parameters: masses scale by ipar[9 item + 4] / ip_detJ
  double ip_detJ;
};

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Membrane records are anchor-pair major: rec[class][m][kRecP], channel ch at kRecPos[ch]. A gather load
// instruction reads 4 channels (one per lane group) x 8 consecutive anchor pairs; this permutation (found
// by exhaustive search over the 12 (channel group, load) combinations and both pair offsets) puts every
// such load at the 2-wavefront minimum (no bank conflicts).
constexpr int kRecP = 30, kRecC = kMS * kRecP;
// Run-time channels (the gather's per-task offsets) read a constant-bank table: the switch below becomes a jump
// table there, which the compiler rematerialised inside the gather loops (5 % of the band kernel's stall samples).
struct RecPosTable { unsigned char p[27]; };
constexpr RecPosTable kRecPos = {{5, 15, 0, 27, 23, 24, 9, 14, 19, 2, 26, 8, 1, 20, 13, 4, 16, 21, 7, 18, 12, 25, 29, 28, 11,
                                  3, 10}};
__constant__ RecPosTable kRecPosDev = kRecPos;
__host__ __device__ __forceinline__ constexpr int rec_pos(int ch) {   // compile-time channels
  switch (ch) {
    case 0: return 5;   case 1: return 15;  case 2: return 0;   case 3: return 27;  case 4: return 23;
    case 5: return 24;  case 6: return 9;   case 7: return 14;  case 8: return 19;  case 9: return 2;
    case 10: return 26; case 11: return 8;  case 12: return 1;  case 13: return 20; case 14: return 13;
    case 15: return 4;  case 16: return 16; case 17: return 21; case 18: return 7;  case 19: return 18;
    case 20: return 12; case 21: return 25; case 22: return 29; case 23: return 28; case 24: return 11;
    case 25: return 3;  default: return 10;
  }
}
__device__ __forceinline__ int rec_pos_rt(int ch) { return kRecPosDev.p[ch]; }   // run-time channels

constexpr int kPA = kNA + 4;                       // staged along cps: [S0 - 2, S0 + kNA + 2)
constexpr int kPosMax = (kMaxD + 4) * kPA * 3;     // staged depth rows: [od0, od1 + 1]

// acc[slot(b)] += d_b,u Y_u + d_b,v Y_v over the 9 window entries b = (bi, bj) of a point in which a sits at
// EA, with the tensor-product coefficients d_b,u = N'u[bi] Nv[bj], d_b,v = Nu[bi] N'v[bj] (masked entries
// are zero in the 1D factors; checked at build time): per window row bj, Au = Nv[bj] Y_u, Av = N'v[bj] Y_v,
// then acc += N'u[bi] Au + Nu[bi] Av.  cu[i] = (N'u[i], Nu[i]), cv[j] = (Nv[j], N'v[j]).
template <int EA>
__device__ __forceinline__ void upd_mem(double (&acc)[kSl], const double2* cu, const double2* cv, double Yu,
                                        double Yv) {
  const double2 u0 = cu[0], u1 = cu[1], u2 = cu[2];
#pragma unroll
  for (int bj = 0; bj < 3; ++bj) {
    const double2 v = cv[bj];
    const double au = v.x * Yu, av = v.y * Yv;
    double* row = acc + (bj - EA / 3 + 2) * 5 + (2 - EA % 3);
    row[0] = fma(u0.x, au, fma(u0.y, av, row[0]));
    row[1] = fma(u1.x, au, fma(u1.y, av, row[1]));
    row[2] = fma(u2.x, au, fma(u2.y, av, row[2]));
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_band(const BandArgs A) {
  extern __shared__ __align__(16) double bsm[];
  BSF_POISON_SMEM(bsm);
  const int cta = blockIdx.x, item = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int band = 0;   // uniform (blockIdx and parameters only)
  while (band + 1 < A.nbands && cta >= A.cfirst[band + 1]) ++band;
  const BandDesc& D = A.desc[band];
  const int S0 = (D.sa0 & ~1) + kNA * (cta - A.cfirst[band]);
  const int axis = D.axis, sa0 = D.sa0, sa1 = D.sa1, t0 = D.t0, t1 = D.t1, od0 = D.od0, od1 = D.od1;
  const int ncls = D.ncls, nbcls = D.nbcls;
  const int PD = od1 - od0 + 2;
  double* pos = bsm;                                   // [PD][kPA][3]
  double2* cf = reinterpret_cast<double2*>(pos + kPosMax);   // [ncls][6] 1D factors (N'u, Nu) x 3, (Nv, N'v) x 3
  double* lw = pos + kPosMax + 12 * ncls;              // [nbcls][9] sqrt(w mu) L_e (item constants)
  double* rec = lw + ((9 * nbcls + 1) & ~1);           // [ncls][kMS][kRecP] (channel ch at rec_pos(ch))
  double* brec = rec + kRecC * ncls;                   // [nbcls][3][kMS] sqrt(w mu) Lap phi
  double* kc = brec + 3 * kMS * nbcls;                 // [16] per-item constants
  double* red = kc + 16;                               // [32] per-warp energy partials
  double* beta = red + 32;                             // [2][kMaxD][kSl] bending Hessian per block slot
  double2* sda = reinterpret_cast<double2*>(beta + 2 * kMaxD * kSl);     // [D.nent] entry window coefficients
  uint32_t* sent = reinterpret_cast<uint32_t*>(sda + D.nent);             // [D.nent] template entries
  const double* __restrict__ x = A.x + item * A.xs;

  if (tid == 0) {
    double G00 = A.G00, G01 = A.G01, G10 = A.G10, G11 = A.G11, det = A.detJ;
    double mu1 = A.mu1, mu2 = A.mu2, mush = A.mush, mubd = A.mubd;
    if (A.params) {
      const double* pp = A.params + 9 * (int64_t)item;
      G00 = pp[0]; G01 = pp[1]; G10 = pp[2]; G11 = pp[3]; det = pp[4];
      mu1 = (A.flags & 2) ? 0.0 : pp[5];
      mu2 = (A.flags & 2) ? 0.0 : pp[6];
      mush = (A.flags & 2) ? 0.0 : pp[7];
      mubd = (A.flags & 4) ? 0.0 : pp[8];
    }
    kc[0] = G00; kc[1] = G01; kc[2] = G10; kc[3] = G11; kc[4] = det; kc[5] = mu1; kc[6] = mu2; kc[7] = mush;
    kc[8] = mubd; kc[9] = G00 * G00 + G01 * G01; kc[10] = G10 * G10 + G11 * G11; kc[11] = 2.0 * (G00 * G10 + G01 * G11);
  }
  // ---- 1. positions, class coefficients, template entries
  for (int k = tid; k < PD * kPA * 3; k += kThreads) {
    const int row = k / (kPA * 3), rem = k - row * (kPA * 3);
    const int col = rem / 3, c = rem - col * 3;
    const int dep = od0 + row, al = S0 - 2 + col;
    const int i = axis ? dep : al, j = axis ? al : dep;
    double v = 0.0;
    if (j >= A.xlo && j < A.xhi && i >= 0 && i < A.n_u) v = x[((int64_t)(j - A.xlo) * A.n_u + i) * 3 + c];
    pos[k] = v;
  }
  for (int k = tid; k < 6 * ncls; k += kThreads) cf[k] = A.mcf[6 * D.cls0 + k];
  for (int k = tid; k < D.nent; k += kThreads) { sent[k] = A.ent[D.ent0 + k]; sda[k] = A.entd[D.ent0 + k]; }
  __syncthreads();
  for (int k = tid; k < 9 * nbcls; k += kThreads) {   // sqrt(w mu) L_e, L_e = G-contracted Laplacian coefficient
    const int bc = k / 9, e = k - bc * 9;
    const double* c3 = A.bcf + 27 * (int64_t)(D.bcls0 + bc);
    const double L = kc[9] * c3[e] + kc[10] * c3[9 + e] + kc[11] * c3[18 + e];
    lw[k] = sqrt(A.bwhat[D.bcls0 + bc] * kc[4] * kc[8]) * L;
  }
  __syncthreads();

  // beta[pi][td][slot] = sum over the bending entries of (pi, td) of w mu L_a L_b (position independent)
  for (int k = tid; k < 2 * (t1 - t0) * kSl; k += kThreads) {
    const int sl = k % kSl, pt = k / kSl, pi = pt & 1, td = pt >> 1;
    const int di = sl % 5 - 2, dj = sl / 5 - 2;
    const uint32_t* eb = sent + D.eoff[pi][td] + D.ment[pi][td];
    double b = 0.0;
    for (int q = 0; q < D.bent[pi][td]; ++q) {
      const uint32_t E = eb[q];
      const int ea = E >> 28, bi = ea % 3 + di, bj = ea / 3 + dj;   // b's window position
      if (bi < 0 || bi > 2 || bj < 0 || bj > 2) continue;
      const double* l9 = lw + ((E >> 16) & 0xFFF);
      b = fma(l9[ea], l9[3 * bj + bi], b);
    }
    beta[(pi * kMaxD + td) * kSl + sl] = b;
  }

  // ---- 2. points of the anchor window [max(S0, sa0) - 2, min(S0 + kNA, sa1)) x [od0, od1)
  const int olo = max(S0, sa0) - 2, ohi = min(S0 + kNA, sa1);
  const int own_lo = olo + 2;
  double e_acc = 0.0;
  const int nmt = ncls * kMS, ntask = (A.dbg & 16) ? 0 : nmt + nbcls * kMS;
  for (int tk = tid; tk < ntask; tk += kThreads) {
    const bool mem = tk < nmt;
    const int cls = mem ? tk / kMS : (tk - nmt) / kMS;
    const int m = mem ? tk - cls * kMS : (tk - nmt) - cls * kMS;
    const int2 ci = mem ? A.mcls[D.cls0 + cls] : A.bcls[D.bcls0 + cls];
    const int oa = S0 - 2 + 2 * m + ci.x, od = ci.y;
    if (oa < olo || oa >= ohi) continue;
    const bool own = oa >= own_lo && od >= t0 && od < t1;
    // window entry e = (ei, ej) = (e % 3, e / 3) in (i, j); staged at along col, depth row
    const int cb = 2 * m + ci.x, rb = od - od0;
    if (mem) {
      double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0};
      const double2* c6 = cf + 6 * cls;
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        const double2 fu = c6[e % 3], fv = c6[3 + e / 3];
        const double2 d = make_double2(fu.x * fv.x, fu.y * fv.y);   // (dN/du Nv, Nu dN/dv)
        const int ea = axis ? e / 3 : e % 3, ed = axis ? e % 3 : e / 3;
        const double* C = pos + ((rb + ed) * kPA + cb + ea) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) { Fu[c] = fma(C[c], d.x, Fu[c]); Fv[c] = fma(C[c], d.y, Fv[c]); }
      }
      const double wq = A.mwhat[D.cls0 + cls] * kc[4];
      double f1[3], f2[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { f1[c] = fma(Fu[c], kc[0], Fv[c] * kc[2]); f2[c] = fma(Fu[c], kc[1], Fv[c] * kc[3]); }
      double* r = rec + kRecC * cls + kRecP * m;
      const auto emit_p = [&](int c, double P1c, double P2c) {   // P~_mu = w sum_beta G_mu,beta P_beta
        r[rec_pos(21 + c)] = wq * fma(kc[0], P1c, kc[1] * P2c);
        r[rec_pos(24 + c)] = wq * fma(kc[2], P1c, kc[3] * P2c);
      };
      const double wG00 = wq * kc[0], wG01 = wq * kc[1], wG10 = wq * kc[2], wG11 = wq * kc[3];
      const double a11 = wG00 * kc[0], a12 = wG00 * kc[1], a22 = wG01 * kc[1];
      const double b11 = wG10 * kc[2], b12 = wG10 * kc[3], b22 = wG11 * kc[3];
      const double c11 = wG00 * kc[2], c12 = wG00 * kc[3], c21 = wG01 * kc[2], c22 = wG01 * kc[3];
      double i5 = 1.0;
      const double psi = !A.vals   // no Hessian values requested: Psi and P only (explicit FMAs: the same bits)
          ? fbw_emit(f1, f2, kc[5], kc[6], kc[7], false, emit_p, [](int, int, double, double, double, double) {}, &i5)
          : fbw_emit(f1, f2, kc[5], kc[6], kc[7], A.project != 0, emit_p,
                                  [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
        const int e6 = sym3(r3, c3);
        r[rec_pos(e6)] = a11 * A11 + a12 * (A12rc + A12cr) + a22 * A22;
        r[rec_pos(6 + e6)] = b11 * A11 + b12 * (A12rc + A12cr) + b22 * A22;
        r[rec_pos(12 + 3 * r3 + c3)] = c11 * A11 + c12 * A12rc + c21 * A12cr + c22 * A22;
        if (r3 != c3) r[rec_pos(12 + 3 * c3 + r3)] = c11 * A11 + c12 * A12cr + c21 * A12rc + c22 * A22;
      }, &i5);
      if (own) {
        e_acc += wq * psi;
        fbw_flag_singular(A.sflag, i5, item, axis ? od : oa, axis ? oa : od);
      }
    } else {
      const double* l9 = lw + 9 * cls;
      double lap[3] = {0, 0, 0};
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        const int ea = axis ? e / 3 : e % 3, ed = axis ? e % 3 : e / 3;
        const double* C = pos + ((rb + ed) * kPA + cb + ea) * 3;
        const double L = l9[e];
        lap[0] = fma(L, C[0], lap[0]); lap[1] = fma(L, C[1], lap[1]); lap[2] = fma(L, C[2], lap[2]);
      }
      double* r = brec + 3 * kMS * cls + m;
      r[0] = lap[0]; r[kMS] = lap[1]; r[2 * kMS] = lap[2];
      if (own) e_acc += 0.5 * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]);
    }
  }
  __syncthreads();

  // ---- 3. gather: warp task = (depth row, parity, channel group); lane = (channel k, along l)
  const int nd = t1 - t0, ntw = (A.dbg & 32) ? 0 : nd * 6;
  const int k4 = lane >> 3, l = lane & 7;
  for (int kt = 0; kt < 6 && ntw > 0; ++kt) {
    const int wt = D.wtask[warp][kt];
    if (wt == 255) break;
    const int td = wt / 6, pi = (wt / 3) & 1, grp = wt % 3;
    // groups 0, 1 are Hessian entries only; group 2 holds entry (2, 2) and the gradient lanes (and the IP energy)
    if (!A.vals && (grp < 2 || (!A.g && !A.xhat))) continue;
    const int lc = grp * kLC + k4;                   // 0..8: block entry (r, c); 9..11: gradient component
    const int s = S0 + pi + 2 * l, t = t0 + td;
    const bool valid = s >= sa0 && s < sa1;
    const int r3 = lc / 3, c3 = lc - 3 * (lc / 3);
    const bool hess = lc < 9;
    // record channels of this lane: Hessian lanes A~uu[rc], A~uv[cr], A~uv[rc], A~vv[rc]; gradient lanes
    // P~u[c], P~v[c] (their Y_u is the gradient contribution; their block accumulators are not used)
    const int o_uu = rec_pos_rt(hess ? sym3(r3, c3) : 21 + lc - 9) + kRecP * l;
    const int o_cr = rec_pos_rt(hess ? 12 + 3 * c3 + r3 : 24 + lc - 9) + kRecP * l;
    const int o_rc = hess ? rec_pos_rt(12 + 3 * r3 + c3) + kRecP * l : o_uu;
    const int o_vv = hess ? rec_pos_rt(6 + sym3(r3, c3)) + kRecP * l : o_cr;
    double acc[kSl];
#pragma unroll
    for (int k = 0; k < kSl; ++k) acc[k] = 0.0;
    double gacc = 0.0;
    // membrane entries, grouped by ea: compile-time accumulator indices, no divergence (every lane runs
    // the same instructions)
    const uint32_t* ep = sent + D.eoff[pi][td];
    const unsigned char* mc = D.mcnt[pi][td];
    // software pipeline across entries (and ea groups): the entry word two ahead, the record channels and
    // the window factors of the next entry are loaded while the current one is accumulated
    const double2* dp = sda + D.eoff[pi][td];   // (d_a,u, d_a,v) of each entry
    uint32_t E1 = ep[0], E2 = ep[1];
    double p_uu, p_cr, p_rc, p_vv;
    double2 p_da;
    {
      const double* rb = rec + (E1 & 0xFFFF);
      p_uu = rb[o_uu]; p_cr = rb[o_cr]; p_rc = rb[o_rc]; p_vv = rb[o_vv];
      p_da = dp[0];
    }
    int k = 0;
    static_for<0, 9>([&](auto EA_) {
      constexpr int EA = decltype(EA_)::value;
      const int n = mc[EA];
      for (int q = 0; q < n; ++q) {
        const uint32_t E = E1;
        const double ruu = p_uu, rcr = p_cr, rrc = p_rc, rvv = p_vv;
        const double dau = p_da.x, dav = p_da.y;
        E1 = E2;
        E2 = ep[k + 2];
        ++k;
        {
          const double* rb = rec + (E1 & 0xFFFF);
          p_uu = rb[o_uu]; p_cr = rb[o_cr]; p_rc = rb[o_rc]; p_vv = rb[o_vv];
          p_da = dp[k];
        }
        const double2* c6 = cf + ((E >> 16) & 0xFFF);
        const double Yu = fma(dau, ruu, dav * rcr);
        const double Yv = fma(dau, rrc, dav * rvv);
        upd_mem<EA>(acc, c6, c6 + 3, Yu, Yv);
        gacc += Yu;
      }
    });
    // bending: the Hessian part sum_q' w mu L_a L_b is position independent (beta table of the CTA,
    // diagonal entries only); the gradient lanes gather sqrt(w mu) L_a sqrt(w mu) Lap phi
    {
      const double* bt = beta + (pi * kMaxD + td) * kSl;
      const double dl = (hess && r3 == c3) ? 1.0 : 0.0;
#pragma unroll
      for (int k2 = 0; k2 < kSl; ++k2) acc[k2] = fma(dl, bt[k2], acc[k2]);
      const int go = (hess ? 0 : lc - 9) * kMS + l;
      const int nb = D.bent[pi][td];
      const uint32_t* eb = ep + D.ment[pi][td];
      for (int q = 0; q < nb; ++q) {
        const uint32_t E = eb[q];
        gacc = fma(lw[((E >> 16) & 0xFFF) + (E >> 28)], brec[(E & 0xFFFF) + go], gacc);
      }
    }
    if (valid && A.xhat) {   // incremental potential: diagonal m/dt^2, gradient and energy (gradient lanes)
      const int ai = axis ? t : s, aj = axis ? s : t;
      const int64_t aloc = (int64_t)(aj - A.r0) * A.n_u + ai;
      const double mm = A.mass[aloc] * (A.ipar ? A.ipar[9 * (int64_t)item + 4] / A.ip_detJ : 1.0);
      if (hess) {
        if (r3 == c3) acc[12] += A.ipk * mm;
      } else {
        const int c = lc - 9;
        const double xa = pos[((t - od0) * kPA + (s - S0 + 2)) * 3 + c];
        const double d = xa - A.xhat[item * A.xhs + aloc * 3 + c];
        gacc += A.ipk * mm * d - mm * A.grav[c];
        e_acc += 0.5 * A.ipk * mm * d * d - mm * A.grav[c] * xa;
      }
    }
    if (valid && !(A.dbg & 64)) {
      const int ai = axis ? t : s, aj = axis ? s : t;
      const int64_t aloc = (int64_t)(aj - A.r0) * A.n_u + ai;
      if (hess && A.vals) {
        double* dst = A.vals + item * A.vs + (int64_t)A.row_ptr[aloc] * 9 + lc;
        const unsigned char* rk = D.rank[td];
#pragma unroll
        for (int k = 0; k < kSl; ++k) {
          const int q = rk[k];
          if (q != 255) dst[9 * q] = acc[k];
        }
      } else if (!hess && A.g) {
        A.g[item * A.gs + 3 * aloc + (lc - 9)] = gacc;
      }
    }
  }
  // ---- energy partial of this CTA
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  if (lane == 0) red[warp] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += red[w];
    A.epart[item * A.e_stride + A.e_off + cta] = sum;
  }
  energy_final_fused(A.ef, A.epart, item);
}

template <class T>
bool upload_v(const std::function<void*(size_t)>& dalloc, T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return true;
  void* p = dalloc(v.size() * sizeof(T));
  if (!p) return false;
  if (cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  *dst = static_cast<T*>(p);
  return true;
}

// Classes are represented by one cell's points; every other cell must match them to 1e-12 (the same
// reading as k_core's representative interior coefficients: the "same" point of two cells
// differs in the last bits of its double-rounded coordinate).
bool close1(double a, double b) { return std::fabs(a - b) <= 1e-12 * std::max(1.0, std::fabs(b)); }

bool close_basis(const Basis1& a, const Basis1& b) {
  for (int k = 0; k < 3; ++k)
    if (!close1(a.N[k], b.N[k]) || !close1(a.d1[k], b.d1[k]) || !close1(a.d2[k], b.d2[k])) return false;
  return true;
}

bool close_point(const Point& p, const Point& q) {
  return p.mask == q.mask && close1(p.what, q.what) && close_basis(p.bu, q.bu) && close_basis(p.bv, q.bv);
}

}  // namespace

int build_band(const Sheet& sh, const CoreTables& ct, BandTables& bt, std::string& err,
               const std::function<void*(size_t)>& dalloc) {
  bt = BandTables();
  if (!ct.ok || !sh.affine || getenv("BSF_NO_BAND")) return 0;
  const int nu = sh.n_u, Su = sh.Su, Sv = sh.Sv, r0 = sh.r0, r1 = sh.r1;
  // anchor buckets (points in list order)
  const int nanch = Su * Sv;
  std::vector<int32_t> mh(nanch + 1, 0), bh(nanch + 1, 0);
  for (const Point& P : sh.mem) ++mh[P.ov * Su + P.ou + 1];
  for (const Point& P : sh.bend) ++bh[P.ov * Su + P.ou + 1];
  for (int a = 0; a < nanch; ++a) { mh[a + 1] += mh[a]; bh[a + 1] += bh[a]; }
  std::vector<int32_t> mi(sh.mem.size()), bi(sh.bend.size());
  {
    std::vector<int32_t> f(mh.begin(), mh.end() - 1), fb(bh.begin(), bh.end() - 1);
    for (size_t k = 0; k < sh.mem.size(); ++k) mi[f[sh.mem[k].ov * Su + sh.mem[k].ou]++] = (int32_t)k;
    for (size_t k = 0; k < sh.bend.size(); ++k) bi[fb[sh.bend[k].ov * Su + sh.bend[k].ou]++] = (int32_t)k;
  }
  struct Geo { int axis, sa0, sa1, t0, t1; };
  const Geo geos[4] = {{0, ct.CI0, ct.CI1, r0, ct.RJ0}, {0, ct.CI0, ct.CI1, ct.RJ1, r1},
                       {1, ct.RJ0, ct.RJ1, 0, ct.CI0}, {1, ct.RJ0, ct.RJ1, ct.CI1, nu}};
  std::vector<BandDesc> descs;
  std::vector<int2> ctas, mcls, bcls;
  std::vector<double2> mcf;
  std::vector<double> mwhat, bcf, bwhat;
  std::vector<uint32_t> ent;
  std::vector<double2> entd;
  size_t smem_max = 0;
  for (int b = 0; b < 4; ++b) {
    const Geo& G = geos[b];
    if (G.sa1 <= G.sa0 || G.t1 <= G.t0) continue;
    const int D = G.t1 - G.t0;
    const int Sal = G.axis ? Sv : Su, Sdp = G.axis ? Su : Sv;
    if (D > kMaxD || G.sa0 - 2 < 0 || G.sa1 > Sal || G.sa1 - G.sa0 < 8) continue;
    const int od0 = std::max(G.t0 - 2, 0), od1 = std::min(G.t1, Sdp);
    if (od1 <= od0) continue;
    // cell (oa, od) -> bucket range
    auto cell = [&](bool bend, int oa, int od, int& k0, int& k1) {
      const int ou = G.axis ? od : oa, ov = G.axis ? oa : od;
      const std::vector<int32_t>& hh = bend ? bh : mh;
      k0 = hh[ov * Su + ou]; k1 = hh[ov * Su + ou + 1];
    };
    // classes from reference cells near the middle of the band
    const int mid = ((G.sa0 + G.sa1) / 2) & ~1;
    bool okb = true;
    int ccount[2] = {0, 0};
    std::vector<int> cfirst[2];   // [bend][par * ndep + (od - od0)] -> first class index (band relative)
    std::vector<int> ccnt[2];
    const int ndep = od1 - od0;
    for (int bend = 0; bend < 2 && okb; ++bend) {
      cfirst[bend].assign(2 * ndep, 0);
      ccnt[bend].assign(2 * ndep, 0);
      for (int par = 0; par < 2; ++par)
        for (int od = od0; od < od1; ++od) {
          int k0, k1;
          cell(bend, mid + par, od, k0, k1);
          cfirst[bend][par * ndep + od - od0] = ccount[bend];
          ccnt[bend][par * ndep + od - od0] = k1 - k0;
          ccount[bend] += k1 - k0;
          // verify every cell of the band's anchor range with this parity and depth
          for (int oa = G.sa0 - 2; oa < G.sa1 && okb; ++oa) {
            if ((oa & 1) != par) continue;
            int q0, q1;
            cell(bend, oa, od, q0, q1);
            if (q1 - q0 != k1 - k0) { okb = false; break; }
            const std::vector<Point>& L = bend ? sh.bend : sh.mem;
            const std::vector<int32_t>& ii = bend ? bi : mi;
            uint32_t used = 0;
            for (int k = 0; k < k1 - k0 && okb; ++k) {
              int hit = -1;
              for (int q = 0; q < q1 - q0 && hit < 0; ++q)
                if (!((used >> q) & 1) && close_point(L[ii[q0 + q]], L[ii[k0 + k]])) hit = q;
              if (hit < 0) okb = false;
              else used |= 1u << hit;
            }
          }
        }
    }
    if (!okb || ccount[0] > 255 || ccount[1] > 255 || 9 * ccount[0] > 4095 || kRecC * ccount[0] > 65535) {
      if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "k_band: band %d rejected (point classes)\n", b);
      continue;
    }
    BandDesc d;
    std::memset(&d, 0, sizeof d);
    d.axis = G.axis; d.sa0 = G.sa0; d.sa1 = G.sa1; d.t0 = G.t0; d.t1 = G.t1; d.od0 = od0; d.od1 = od1;
    d.ncls = ccount[0]; d.nbcls = ccount[1];
    d.cls0 = (int)mcls.size(); d.bcls0 = (int)bcls.size(); d.ent0 = (int)ent.size();
    // class data (from the reference cells)
    for (int bend = 0; bend < 2; ++bend)
      for (int par = 0; par < 2; ++par)
        for (int od = od0; od < od1; ++od) {
          int k0, k1;
          cell(bend, mid + par, od, k0, k1);
          for (int k = k0; k < k1; ++k) {
            const Point& P = bend ? sh.bend[bi[k]] : sh.mem[mi[k]];
            if (!bend) {
              mcls.push_back(make_int2(par, od));
              mwhat.push_back(P.what);
              for (int e = 0; e < 9; ++e) {
                const int iu = e % 3, jv = e / 3;
                const bool in = (P.mask >> e) & 1;
                // tensor-product form: a masked entry must have zero 1D products
                if (!in && (P.bu.d1[iu] * P.bv.N[jv] != 0.0 || P.bu.N[iu] * P.bv.d1[jv] != 0.0)) okb = false;
              }
              for (int i = 0; i < 3; ++i) mcf.push_back(make_double2(P.bu.d1[i], P.bu.N[i]));
              for (int j = 0; j < 3; ++j) mcf.push_back(make_double2(P.bv.N[j], P.bv.d1[j]));
            } else {
              bcls.push_back(make_int2(par, od));
              bwhat.push_back(P.what);
              double LA[9], LB[9], LC[9];
              for (int e = 0; e < 9; ++e) {
                const int iu = e % 3, jv = e / 3;
                const bool in = (P.mask >> e) & 1;
                LA[e] = in ? P.bu.d2[iu] * P.bv.N[jv] : 0.0;
                LB[e] = in ? P.bu.N[iu] * P.bv.d2[jv] : 0.0;
                LC[e] = in ? P.bu.d1[iu] * P.bv.d1[jv] : 0.0;
              }
              bcf.insert(bcf.end(), LA, LA + 9);
              bcf.insert(bcf.end(), LB, LB + 9);
              bcf.insert(bcf.end(), LC, LC + 9);
            }
          }
        }
    // templates per (parity, depth row) from a representative cp; pattern rows checked for every cp
    for (int td = 0; td < D && okb; ++td) {
      const int t = G.t0 + td;
      std::vector<int> ref_off;   // slot per rank of the row
      for (int s = G.sa0; s < G.sa1 && okb; ++s) {
        const int ai = G.axis ? t : s, aj = G.axis ? s : t;
        const int64_t al = (int64_t)(aj - r0) * nu + ai;
        std::vector<int> off;
        for (int32_t q = sh.row_ptr[al]; q < sh.row_ptr[al + 1]; ++q) {
          const int bcol = sh.col_idx[q], bi_ = bcol % nu, bj_ = bcol / nu;
          const int di = bi_ - ai, dj = bj_ - aj;
          if (di < -2 || di > 2 || dj < -2 || dj > 2) { okb = false; break; }
          off.push_back((dj + 2) * 5 + di + 2);
        }
        if (s == G.sa0) ref_off = off;
        else if (off != ref_off) okb = false;
      }
      if (!okb) break;
      std::memset(d.rank[td], 255, kSl);
      for (size_t k = 0; k < ref_off.size(); ++k) d.rank[td][ref_off[k]] = (unsigned char)k;
      for (int pi = 0; pi < 2; ++pi) {
        const int sr = mid + pi;   // representative cp (anchors [sr - 2, sr] inside the verified range)
        const int ai = G.axis ? t : sr, aj = G.axis ? sr : t;
        d.eoff[pi][td] = (int)ent.size() - d.ent0;
        for (int bend = 0; bend < 2; ++bend) {
          std::vector<uint32_t> grp[9];
          for (int od = t - 2; od <= t; ++od) {
            if (od < od0 || od >= od1) continue;
            for (int oa = sr - 2; oa <= sr; ++oa) {
              int k0, k1;
              cell(bend, oa, od, k0, k1);
              const int cbase = cfirst[bend][(oa & 1) * ndep + od - od0];
              int r0k, r1k;
              cell(bend, mid + (oa & 1), od, r0k, r1k);   // the class representatives of this cell
              for (int k = k0; k < k1; ++k) {
                const Point& P = bend ? sh.bend[bi[k]] : sh.mem[mi[k]];
                const int ea = (ai - P.ou) + 3 * (aj - P.ov);
                if (!((P.mask >> ea) & 1)) continue;
                int cl = -1;
                for (int q = r0k; q < r1k && cl < 0; ++q)
                  if (close_point(P, bend ? sh.bend[bi[q]] : sh.mem[mi[q]])) cl = q - r0k;
                if (cl < 0) { okb = false; break; }
                const int dm = (pi - (sr - oa) + 2) >> 1;
                const uint32_t c = (uint32_t)(cbase + cl);
                const uint32_t roff = bend ? 3u * kMS * c + (uint32_t)dm : (uint32_t)(kRecC * c + kRecP * dm);
                grp[ea].push_back(roff | (((bend ? 9u : 6u) * c) << 16) | ((uint32_t)ea << 28));
              }
            }
          }
          int cnt = 0;
          for (int ea = 0; ea < 9; ++ea) {
            if (grp[ea].size() > 255) okb = false;
            (bend ? d.bcnt : d.mcnt)[pi][td][ea] = (unsigned char)grp[ea].size();
            ent.insert(ent.end(), grp[ea].begin(), grp[ea].end());
            for (uint32_t E : grp[ea]) {   // the entry's window coefficients (membrane; bending: unused)
              const size_t f = 6 * (size_t)d.cls0 + ((E >> 16) & 0xFFF);
              entd.push_back(bend ? make_double2(0.0, 0.0)
                                  : make_double2(mcf[f + ea % 3].x * mcf[f + 3 + ea / 3].x,
                                                 mcf[f + ea % 3].y * mcf[f + 3 + ea / 3].y));
            }
            cnt += (int)grp[ea].size();
          }
          (bend ? d.bent : d.ment)[pi][td] = cnt;
        }
      }
    }
    if (!okb) {   // roll back this band's data
      if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "k_band: band %d rejected (templates / pattern)\n", b);
      mcls.resize(d.cls0); mwhat.resize(d.cls0); mcf.resize(6 * (size_t)d.cls0);
      bcls.resize(d.bcls0); bwhat.resize(d.bcls0); bcf.resize(27 * (size_t)d.bcls0);
      ent.resize(d.ent0);
      entd.resize(d.ent0);
      continue;
    }
    {   // gather tasks to warps: longest first onto the least loaded warp (cost ~ membrane entries + 1/3 bending)
      const int nt = 6 * D;
      std::vector<int> order(nt);
      for (int k = 0; k < nt; ++k) order[k] = k;
      auto cost = [&](int wt) { const int td = wt / 6, pi = (wt / 3) & 1; return 3 * d.ment[pi][td] + d.bent[pi][td]; };
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost(x) > cost(y); });
      constexpr int nw = kThreads / 32;
      int load[nw] = {}, cnt[nw] = {};
      std::memset(d.wtask, 255, sizeof d.wtask);
      for (int wt : order) {
        int best = -1;
        for (int w = 0; w < nw; ++w)
          if (cnt[w] < 6 && (best < 0 || load[w] < load[best])) best = w;
        if (best < 0) { okb = false; break; }
        d.wtask[best][cnt[best]++] = (unsigned char)wt;
        load[best] += cost(wt);
      }
    }
    ent.push_back(0u);   // padding: the membrane loop prefetches two entries ahead
    ent.push_back(0u);
    entd.push_back(make_double2(0.0, 0.0));
    entd.push_back(make_double2(0.0, 0.0));
    d.nent = (int)ent.size() - d.ent0;
    const size_t smem = sizeof(double) * ((size_t)kPosMax + 12 * d.ncls + ((9 * d.nbcls + 1) & ~1) +
                                          (size_t)kRecC * d.ncls + 3 * kMS * d.nbcls + 48 + 2 * kMaxD * kSl) +
                        (sizeof(double2) + sizeof(uint32_t)) * (size_t)d.nent;
    smem_max = std::max(smem_max, smem);
    bt.h_cfirst.push_back((int)ctas.size());
    for (int S0 = G.sa0 & ~1; S0 < G.sa1; S0 += kNA) ctas.push_back(make_int2((int)descs.size(), S0));
    bt.covered[b] = 1;
    descs.push_back(d);
  }
  if (descs.empty() || smem_max > 227 * 1024) {
    if (getenv("BSF_CORE_DEBUG") && !descs.empty()) fprintf(stderr, "k_band: over the smem / parameter budget\n");
    bt = BandTables();
    return 0;
  }
  bt.h_cfirst.push_back((int)ctas.size());
  bt.h_desc = descs;

  const bool ok = upload_v(dalloc, &bt.mcf, mcf) && upload_v(dalloc, &bt.mcls, mcls) &&
                  upload_v(dalloc, &bt.mwhat, mwhat) && upload_v(dalloc, &bt.bcf, bcf) &&
                  upload_v(dalloc, &bt.bcls, bcls) && upload_v(dalloc, &bt.bwhat, bwhat) &&
                  upload_v(dalloc, &bt.ent, ent) && upload_v(dalloc, &bt.entd, entd);
  if (!ok) { err = "band: device allocation failed"; return -7; }
  if (cudaFuncSetAttribute(k_band, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max) != cudaSuccess) {
    cudaGetLastError();
    bt = BandTables();
    return 0;
  }
  bt.smem = smem_max;
  bt.nbands = (int)descs.size();
  bt.nctas = (int)ctas.size();
  if (getenv("BSF_CORE_DEBUG")) {
    fprintf(stderr, "k_band: %d bands, %d CTAs per item, smem %zu\n", bt.nbands, bt.nctas, bt.smem);
    for (const BandDesc& d : descs)
      fprintf(stderr, "  axis %d along [%d,%d) depth [%d,%d) classes %d+%d entries %d\n", d.axis, d.sa0, d.sa1, d.t0,
              d.t1, d.ncls, d.nbcls, d.nent);
  }
  bt.ok = 1;
  return 0;
}

int band_eval(const BandTables& bt, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const int32_t* d_row_ptr,
              double* e_part, int64_t e_stride, int64_t e_off, const double* d_params, const double* G4, double detJ,
              cudaStream_t st, const IpFused* ip) {
  if (!bt.ok || bt.nctas == 0) return 0;
  static_assert(sizeof(BandArgs) <= 32000, "kernel parameter budget");
  BandArgs A;
  A.sflag = call_sflag();
  A.ef = call_efinal();
  A.x = d_x; A.xs = x_stride; A.g = d_g; A.gs = g_stride; A.vals = d_vals; A.vs = v_stride;
  A.epart = e_part; A.e_stride = e_stride; A.e_off = e_off;
  A.row_ptr = d_row_ptr; A.params = d_params;
  A.n_u = sh.n_u; A.xlo = sh.xlo; A.xhi = sh.xhi; A.r0 = sh.r0;
  A.project = (flags & 1) ? 1 : 0; A.flags = flags;
  {   // profiling switches (read once per process): 16 no points, 32 no gather
    static const int dbg = getenv("BSF_CORE_DEBUG") ? atoi(getenv("BSF_CORE_DEBUG")) : 0;
    A.dbg = dbg;
  }
  A.G00 = G4[0]; A.G01 = G4[1]; A.G10 = G4[2]; A.G11 = G4[3]; A.detJ = detJ;
  A.mu1 = (flags & 2) ? 0.0 : mat.mu_st1;
  A.mu2 = (flags & 2) ? 0.0 : mat.mu_st2;
  A.mush = (flags & 2) ? 0.0 : mat.mu_sh;
  A.mubd = (flags & 4) ? 0.0 : mat.mu_bd;
  A.mcf = bt.mcf; A.mcls = bt.mcls; A.mwhat = bt.mwhat;
  A.bcf = bt.bcf; A.bcls = bt.bcls; A.bwhat = bt.bwhat;
  A.nbands = bt.nbands;
  for (int b = 0; b <= bt.nbands; ++b) A.cfirst[b] = bt.h_cfirst[b];
  std::memcpy(A.desc, bt.h_desc.data(), sizeof(BandDesc) * bt.h_desc.size());
  A.ent = bt.ent; A.entd = bt.entd;
  A.xhat = ip ? ip->xhat : nullptr; A.xhs = ip ? ip->xhs : 0; A.mass = ip ? ip->mass : nullptr;
  A.ipk = ip ? ip->k : 0.0;
  for (int c = 0; c < 3; ++c) A.grav[c] = ip ? ip->grav[c] : 0.0;
  A.ipar = ip ? ip->params : nullptr;
  A.ip_detJ = ip ? ip->detJ_ref : 1.0;
  dim3 grid(bt.nctas, nbatch);
  k_band<<<grid, kThreads, bt.smem, st>>>(A);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

}  // namespace bsf
