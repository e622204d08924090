// k_core: the fused interior kernel.  See core.hpp for the configuration it exploits.
//
// One CTA owns a strip of kW = 32 control-point columns over a chunk of rows of one sheet (grid.z =
// batch item) and walks it kRows = 2 rows per step:
//   1. point phase: the quadrature points of the two new knot rows of the strip window — membrane
//      F~ = sum_e C_e d_e, F = F~ G, FBW Psi, P, A with the optional per-term PSD
//      projection (fbw.cuh), stored in the parametric frame as
//      A~ = w (G (x) I) A (G (x) I)^T split into A~uu, A~vv, S = A~uv + A~uv^T, D = A~uv - A~uv^T and
//      P~ = w G P; bending Lap phi = sum_e L_e C_e — into a shared-memory ring of
//      5 knot rows, channel-major (SoA), V / H point sets split by knot parity;
//   2. gather: warp (parity pi, role) — 32 same-parity control points of the 2 rows — accumulates ONE
//      entry (r, c) (and its transpose) of all 23 blocks of each lane's block row over the 12
//      incident membrane points, with the compile-time incidence table of parity pi and constant
//      coefficients k_uu, k_vv, k_s, k_a (core.hpp), in registers:
//          H_ab[r][c] = sum_q k_uu A~uu[rc] + k_vv A~vv[rc] + k_s S[rc] + k_a D[rc]
//      plus the constant bending blocks beta_ab I3 (the bending Hessian of an affine interior is
//      state independent: sum_q w mu L_a L_b); diagonal roles also gather g_a[r];
//   3. the two rows' outputs are staged in shared memory in their final BSR order and written with
//      two TMA bulk copies (cp.async.bulk shared -> global), overlapping the next step's point phase.
// Every block row is computed completely by its own control point (no transposes across rows), so
// rows, slabs and chunks are independent and no atomics are used.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <type_traits>
#include <vector>

#include "core.hpp"
#include "ip.hpp"
#include "fbw.cuh"

namespace bsf {

namespace {
using namespace core;

struct CoreArgs {
  const double* x;
  int64_t xs;
  double* g;
  int64_t gs;
  double* vals;
  int64_t vs;
  double* epart;
  int64_t e_stride, e_off;
  const int32_t* row_ptr;
  int64_t rp_base, rp_stride;
  const double* params;
  int n_u, xlo, xhi, r0;
  int CI0, CI1, RJ0, RJ1, nstrips, nchunks;
  int JA, JB;              // rows of this launch ([RJ0, RJ1) or a sub-range; addressing stays relative to RJ0)
  int project, flags, dbg, layout;
  unsigned long long* sflag;   // singular-stretch word (fbw.cuh)
  EFinal ef;                   // fused energy reduction of the call
  double G00, G01, G10, G11, detJ, mu1, mu2, mush, mubd;
  // curved rest map (CoreTables): per-point / per-cp tables, knot pitch, core columns
  const double* mtab;
  const double* btab;
  const double* beta;
  const double* gw;
  int64_t kp, cw;
  int Su, Sv;
  const double* tabs;      // device [104]: S[4][9][2] | LA[9] | LB[9] | LC[9] | what[5]
  double what[5];
  // incremental-potential terms (Q13; xhat == nullptr: elastic only)
  const double* xhat;
  int64_t xhs;
  const double* mass;
  double ipk, grav[3];
  const double* ipar;      // optional per-item parameters: masses scale by ipar[9 item + 4] / ip_detJ
  double ip_detJ;
};

// shared constants block (doubles)
constexpr int kCstL = 0;        // [9]  L_e  (bending Laplacian coefficients of this item)
constexpr int kCstLw = 9;       // [9]  w_b mu_bd L_e
constexpr int kCstBeta = 18;    // [23] bending Hessian blocks beta_ab
constexpr int kCstS = 41;       // [72] S[set][e][2]
constexpr int kCstRed = 113;    // [24] energy reduction
constexpr int kCstW = 137;      // [5]  parametric weights of the sets and of the bending points
constexpr int kCstP = 142;      // [10] G00 G01 G10 G11 detJ mu1 mu2 mush mubd w_b of this item
constexpr int kCstN = 152;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Bulk-store issuer: lane 0 of a gather warp.  The issuing thread is the only one that can wait for the
// store's shared-memory reads (bulk async-groups are per thread), and the gather warps are the ones that
// overwrite the staging buffer, so the wait sits in a gather warp right before its staging stores (a point
// warp there would couple the gather to the point phase).
// Warp layouts.  Warps are issued by the SM sub-partition (scheduler) warp % 4, so which role sits on which warp
// decides how the per-step work is spread over the four schedulers.  A layout gives the gather warps' block
// entries (role = 3 r + c), the warp that issues the bulk stores, the point-item block of each point warp
// (items 30 pw .. 30 pw + 29: pw 0-3 membrane, 4 mixed, 5-6 bending) and its gradient rounds
// [g0, g0 + gn) (round = 3 parity + component).  Selected with BSF_CORE_LAYOUT (default 6: C4 k_core 451 us with layout 1, 444 with 0, 431 with 4, 429 with 5, 428 with 6;
// the per-warp busy cycles of scripts/core_timers.py --c4 show the gather warps as the limit from layout 4 on).
struct CoreLayout {
  int8_t role[kGatherWarps];
  int8_t tma_warp;
  int8_t pw[kPointWarps];
  int8_t g0[kPointWarps], gn[kPointWarps];
};
__constant__ CoreLayout kLayouts[8] = {
    // 0: diagonal roles on warps 0-2, one gradient round on every point warp but warp 12
    {{0, 4, 8, 1, 2, 3, 5, 6, 7}, 3, {0, 1, 2, 3, 4, 5, 6}, {0, 1, 2, 0, 3, 4, 5}, {1, 1, 1, 0, 1, 1, 1}},
    // 1: the round-2 layout: role = warp, bulk stores on warp 1, gradient rounds on warps 9-14
    {{0, 1, 2, 3, 4, 5, 6, 7, 8}, 1, {0, 1, 2, 3, 4, 5, 6}, {0, 1, 2, 3, 4, 5, 0}, {1, 1, 1, 1, 1, 1, 0}},
    // 2: as 0, the mixed item block on warp 12, three gradient rounds on each bending warp
    {{0, 4, 8, 1, 2, 3, 5, 6, 7}, 3, {0, 1, 2, 4, 3, 5, 6}, {0, 0, 0, 0, 0, 0, 3}, {0, 0, 0, 0, 0, 3, 3}},
    // 3: off-diagonal roles on scheduler 0 (warps 0, 4, 8), diagonal ones on warps 1-3; point warps as 2
    {{1, 0, 4, 8, 2, 3, 5, 6, 7}, 5, {0, 1, 2, 4, 3, 5, 6}, {0, 0, 0, 0, 0, 0, 3}, {0, 0, 0, 0, 0, 3, 3}},
    // 4: as 3, two gradient rounds on each bending warp and one on warps 10, 11
    {{1, 0, 4, 8, 2, 3, 5, 6, 7}, 5, {0, 1, 2, 4, 3, 5, 6}, {0, 4, 5, 0, 0, 0, 2}, {0, 1, 1, 0, 0, 2, 2}},
    // 5: as 4, a bending block on warp 12 (scheduler 0) and the mixed block on warp 14
    {{1, 0, 4, 8, 2, 3, 5, 6, 7}, 5, {0, 1, 2, 5, 3, 4, 6}, {0, 4, 5, 0, 0, 0, 2}, {0, 1, 1, 2, 0, 0, 2}},
    // 6: as 5, no gradient round on scheduler 2 (warps 10, 14): warps 11 (one), 12 (two), 15 (three)
    {{1, 0, 4, 8, 2, 3, 5, 6, 7}, 5, {0, 1, 2, 5, 3, 4, 6}, {0, 0, 5, 0, 0, 0, 2}, {0, 0, 1, 2, 0, 0, 3}},
    // 7: as 5, one gradient round on warp 12 and three on warp 15
    {{1, 0, 4, 8, 2, 3, 5, 6, 7}, 5, {0, 1, 2, 5, 3, 4, 6}, {0, 4, 5, 0, 0, 0, 1}, {0, 1, 1, 1, 0, 0, 3}},
};

// Staged positions: per cp row, the strip's kPosC columns split by column parity ([even | odd] halves of
// kPosH columns, 3 doubles each), so the lanes of a point set — consecutive knots of one parity, 2 columns
// apart — read 3 doubles apart (an odd stride: no shared-memory bank conflicts).
constexpr int kPosH = kPosC / 2;
static_assert(kPosC % 2 == 0, "even staged column count");
__device__ __forceinline__ int pos_col(int col) { return (col & 1) * kPosH + (col >> 1); }

__device__ __forceinline__ int ring_slot(int q) { return (unsigned)(q + 7 * kRing) % kRing; }   // q >= -49

#ifdef BSF_PHASE_TIMERS
__device__ unsigned long long g_core_t[16];
__device__ unsigned long long g_warp_t[32];
#define CT_MARK(v) const long long v = clock64()
#define CT_ADD(i, d) atomicAdd(&g_core_t[i], (unsigned long long)(d))
#else
#define CT_MARK(v)
#define CT_ADD(i, d)
#endif

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Gather of one warp: PI = parity of the lanes' control points; the warp's role is one entry (r, c)
// of the 3x3 blocks.  For every incident point q (slot) of the lane's control point a:
//     Yu = d_a,u A~uu[rc] + d_a,v A~vu[rc],   Yv = d_a,u A~uv[rc] + d_a,v A~vv[rc]
//     H_ab[r][c] += d_b,u Yu + d_b,v Yv            for each block b of q's stencil
// (= sum_{mu,nu} d_a,mu d_b,nu A~_mu,nu[r][c]).  d comes from the 4 x 9 x 2 per-set basis table S,
// indexed at compile time (static_for over the parity's incidence table), so the 23 accumulators live
// in registers and every coefficient is a uniform-register operand.  base0[d] / base1[d]
// (d = dq + 2): lane's record pointer for knot row j+h+dq for even / odd knot-column offsets dp.
// Diagonal roles (r == c) add the constant bending blocks and gather g_a[r]; bb0 / bb1 address the
// bending arrays (channel r).  Staging stores wait on `bar` (previous bulk store has read the buffer).
template <int IMM>
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(IMM));
  return v;
}

// Gradient of one component r for the lanes' control points (parity PI): g_a[r] = sum_q d_a . P~(q)[r]
// over the 12 incident membrane points + sum_q' w mu L_a(q') Lap phi(q')[r] over the 8 bending points.
// base0/1: shared byte addresses of the knot rows (channel 0) for even / odd dp; bb0/1: bending arrays
// at channel r.  Run by the point warps with spare time (the gather warps carry the blocks).
template <int PI, bool CURVED>
__device__ __forceinline__ void gather_grad(const uint32_t (&base0)[4], const uint32_t (&base1)[4],
                                            const double* const (&bb0)[3], const double* const (&bb1)[3],
                                            uint32_t o_pu, uint32_t o_pv, const double* __restrict__ cst,
                                            double* gdst, double g0, const double* __restrict__ gw, int64_t gws,
                                            double mubd) {
  double g = g0;
  static_for<0, make_template(PI).nslot>([&](auto SI) {
    constexpr int s = decltype(SI)::value;
    constexpr Template T = make_template(PI);
    constexpr int dp = T.s_dp[s], dq = T.s_dq[s], set = T.s_set[s], ea = T.s_ea[s];
    constexpr int imm = 8 * (set * kSetD + ((dp + 2) >> 1));
    const uint32_t bu = (dp & 1) ? base1[dq + 2] : base0[dq + 2];
    constexpr double dau = kSetTable.v[set][ea][0], dav = kSetTable.v[set][ea][1];
    g = fma(dau, lds_f64<imm>(bu + o_pu), fma(dav, lds_f64<imm>(bu + o_pv), g));
  });
  static_for<0, kBSlots>([&](auto KI) {
    constexpr int k = decltype(KI)::value;
    constexpr int dp = bslot_dp(k), dq = bslot_dq(k);
    const double* b = ((dp & 1) ? bb1[dq + 2] : bb0[dq + 2]) + ((dp + 2) >> 1);
    // curved: w mu L_a of this cp's own bending slot k (per-cp table); affine: one value per slot
    g = fma(CURVED ? mubd * __ldg(gw + k * gws) : cst[kCstLw + k], b[0], g);
  });
  if (gdst) *gdst = g;
}

template <int PI, bool CURVED>
__device__ __forceinline__ void gather_role(const uint32_t (&base0)[4],
                                            const uint32_t (&base1)[4], int o_rc, int o_cr, bool diag,
                                            const double* __restrict__ cst, double* st_lane, bool active,
                                            uint32_t bar, uint32_t parity, double dshift,
                                            const double* __restrict__ beta, int64_t bs, double mubd, bool tma) {
  double acc[kNB];
#pragma unroll
  for (int k = 0; k < kNB; ++k) acc[k] = 0.0;
  if (CURVED && diag) {   // the per-cp bending blocks are read after the loop: start their trip to L1 now
#pragma unroll
    for (int k = 0; k < kNB; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(beta + k * bs));
  }
  static_for<0, make_template(PI).nslot>([&](auto SI) {
    constexpr int s = decltype(SI)::value;
    constexpr Template T = make_template(PI);
    constexpr int dp = T.s_dp[s], dq = T.s_dq[s], set = T.s_set[s], ea = T.s_ea[s];
    constexpr int imm = 8 * (set * kSetD + ((dp + 2) >> 1));   // byte offset within the knot row
    const uint32_t bu = (dp & 1) ? base1[dq + 2] : base0[dq + 2];   // shared byte address (+ role uu)
    const double auu = lds_f64<imm>(bu), avv = lds_f64<imm + 8 * 6 * kKH>(bu);
    const double arc = lds_f64<imm>(bu + o_rc), acr = lds_f64<imm>(bu + o_cr);
    // (Yu, Yv) = dau (auu, arc) + dav (acr, avv), with the larger of dau, dav factored out into the block
    // coefficients (compile-time constants): Y = f (Y1, Y2), one DFMA each instead of a DMUL + DFMA
    constexpr double dau = kSetTable.v[set][ea][0], dav = kSetTable.v[set][ea][1];
    constexpr bool FU = (dau < 0 ? -dau : dau) >= (dav < 0 ? -dav : dav);
    constexpr double f = FU ? dau : dav, ra = FU ? dav / dau : dau / dav;
    const double Y1 = FU ? fma(ra, acr, auu) : fma(ra, auu, acr);
    const double Y2 = FU ? fma(ra, avv, arc) : fma(ra, arc, avv);
    static_for<T.s_c0[s], T.s_c0[s] + T.s_nc[s]>([&](auto CI) {
      constexpr int c = decltype(CI)::value;
      constexpr Template T2 = make_template(PI);
      constexpr int k = T2.c_blk[c], eb = T2.c_eb[c];
      constexpr double bu = kSetTable.v[set][eb][0] * f, bv = kSetTable.v[set][eb][1] * f;
      acc[k] = fma(bu, Y1, fma(bv, Y2, acc[k]));
    });
  });
  if (diag) {   // the state-independent bending blocks beta_ab I3 (+ inertia m_a/dt^2); adding them at the end
                // measured faster than starting the accumulators from them (508 vs 490 us on C4)
    if constexpr (CURVED) {   // this cp's own bending blocks (per-cp table, w L_a L_b summed over its points)
#pragma unroll
      for (int k = 0; k < kNB; ++k) acc[k] = fma(mubd, __ldg(beta + k * bs), acc[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kNB; ++k) acc[k] += cst[kCstBeta + k];
    }
    acc[block_index(0, 0)] += dshift;
  }
  if (!st_lane) return;
  if (PI == 0 && tma) {   // the previous step's bulk store has read the staging buffer
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
  }
  mbar_wait(bar, parity);
  if (!active) return;
  // Lanes m and m + 8 of a half-warp are 8 control points (an even multiple of 207 doubles) apart, i.e. on the
  // same bank: lanes 8-15 store block (k + 1) mod 23 when the others store block k (9 doubles further: an odd
  // bank offset), so every store wavefront is conflict-free (measured: 516 -> 490 us on C4).
  const bool rot = (threadIdx.x & 8) != 0;
  double* const sb = st_lane + (rot ? 9 : 0);   // block k (or k + 1) at sb + 9 k: one base, immediate offsets
#pragma unroll
  for (int k = 0; k < kNB - 1; ++k) sb[k * 9] = rot ? acc[k + 1] : acc[k];
  st_lane[rot ? 0 : (kNB - 1) * 9] = rot ? acc[0] : acc[kNB - 1];
}

// Stage the positions of cp rows [prow0, prow0 + nrows), cols [i0-3, i0+kW+3) (zero outside the array)
// with asynchronous 8-byte copies (cp.async; the caller waits before the barrier that publishes them).
// Thread tid copies elements tid, tid + kThreads, ... of the [nrows][kPosC][3] block.
__device__ __forceinline__ void load_pos_async(double* pos, const double* __restrict__ x, const CoreArgs& A, int i0,
                                               int prow0, int nrows, int tid) {
  for (int k = tid; k < nrows * kPosC * 3; k += kThreads) {
    const int row = k / (kPosC * 3), rem = k - row * (kPosC * 3);
    const int col = rem / 3, c = rem - col * 3;
    const int R = prow0 + row, Cc = i0 - 3 + col;
    const bool in = R >= A.xlo && R < A.xhi && Cc >= 0 && Cc < A.n_u;
    const double* src = in ? &x[((int64_t)(R - A.xlo) * A.n_u + Cc) * 3 + c] : x;
    double* dst = pos + (row * kPosC + pos_col(col)) * 3 + c;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(in ? 8 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Same for the 5-row blocks of the main loop, with the element -> (row, col, component) map of this
// thread precomputed (kPosStep <= 2 kThreads: at most two elements per thread).
struct PosMap {
  int n;            // elements of this thread (0..2)
  int off[2];       // (row * n_u + col - (i0 - 3)) * 3 + c relative to the block origin, or -1 if the column is off the sheet
  int row[2];
  uint32_t dst[2];  // shared offsets (bytes) within a block
};

__device__ __forceinline__ void load_pos_step(uint32_t pos_s, const double* __restrict__ x, const CoreArgs& A,
                                              const PosMap& pm, int i0, int prow0) {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (e < pm.n) {
      const int R = prow0 + pm.row[e];
      const bool in = pm.off[e] >= 0 && R >= A.xlo && R < A.xhi;
      const double* src = in ? x + ((int64_t)(prow0 - A.xlo) * A.n_u + (i0 - 3)) * 3 + pm.off[e] : x;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(pos_s + pm.dst[e]), "l"(src),
                   "r"(in ? 8 : 0)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

struct PointCtx {
  double G00, G01, G10, G11, det, mu1, mu2, mush, mubd, wb;
  int i0, i1, ja, jb;
  bool project;
  bool diagG;      // G01 == G10 == 0 (axis-aligned rest sheet): F, A~ and P~ by scaling
  unsigned long long* sflag;
  int item;
  // curved rest map: per-point tables (CoreTables::mtab / btab), knot pitch, last knot indices
  const double* mtab;
  const double* btab;
  int64_t kp;
  int Su, Sv;
};

// Quadrature points of two consecutive knot rows q0, q0+1: item it in [0, 6 kKC) =
//   [membrane of row q0 (V- nV, V+ nV, H- nH, H+ nH) | membrane of row q0+1 | bending q0 | bending q0+1],
// each set ordered by its knot index k = lp >> 1 (conflict-free record writes; membrane items first so
// that warps do not diverge between the two kinds).  pos holds cp rows from prow0.
// Returns the point's owned energy.
template <bool CURVED, bool HESS>
__device__ __forceinline__ double eval_item(double* ring, const double* pos, int prow0, const double* cst,
                                         const PointCtx& P, int q0, int it) {
  const int nmem = 2 * kKC;
  if (it >= 2 * nmem) {
    // bending: per row lp even knots then lp odd knots
    const int rb = it - 2 * nmem, r = rb >= kKC, rr = rb - r * kKC, q = q0 + r, nE = (kKC + 1) / 2;
    const int lp = rr < nE ? 2 * rr : 2 * (rr - nE) + 1;
    const int p = P.i0 - 2 + lp;
    double* row = ring + ring_slot(q) * kRowD;
    // curved: this knot's own Laplacian coefficients and weight (clamped: knots past the sheet feed only lanes
    // that store nothing)
    const double* bt = CURVED ? P.btab + (int64_t)min(max(q, 0), P.Sv) * 10 * P.kp + min(max(p, 0), P.Su) : nullptr;
    double lap[3] = {0, 0, 0};
#pragma unroll
    for (int jv = 0; jv < 3; ++jv)
#pragma unroll
      for (int iu = 0; iu < 3; ++iu) {
        const int e = 3 * jv + iu;
        if (e == 8) continue;
        const double L = CURVED ? __ldg(bt + e * P.kp) : cst[kCstL + e];
        const double* C = pos + ((q + jv - prow0) * kPosC + pos_col(p + iu - (P.i0 - 3))) * 3;
        lap[0] = fma(L, C[0], lap[0]); lap[1] = fma(L, C[1], lap[1]); lap[2] = fma(L, C[2], lap[2]);
      }
    double* rec = row + 4 * kSetD + (lp & 1) * kBendD + (lp >> 1);
    rec[0] = lap[0];
    rec[kKH] = lap[1];
    rec[2 * kKH] = lap[2];
    if (p >= P.i0 && p < P.i1 && q >= P.ja && q < P.jb)
      return 0.5 * (CURVED ? __ldg(bt + 9 * P.kp) : cst[kCstP + 9]) * cst[kCstP + 8] *
             fma(lap[0], lap[0], fma(lap[1], lap[1], lap[2] * lap[2]));
    return 0.0;
  }
  const int r = it >= nmem, mi = it - r * nmem, q = q0 + r;
  double* row = ring + ring_slot(q) * kRowD;
  const int pv = (q + P.i0) & 1;                 // lp parity of the V knots of this row (p + q even)
  const int nV = (kKC - pv + 1) / 2, nH = kKC - nV;
  int set, k;
  if (mi < 2 * nV) { set = mi >= nV; k = mi - set * nV; }
  else { const int x = mi - 2 * nV; set = 2 + (x >= nH); k = x - (set - 2) * nH; }
  const int lp = 2 * k + ((set < 2) ? pv : 1 - pv), p = P.i0 - 2 + lp;
  const int s = p + (set == 2 ? -1 : 0), tq = q + (set == 0 ? -1 : 0);   // anchor
  const double* Sset = cst + kCstS + set * 18;
  double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0};
  // the 6 structural window entries of the point (V sets: columns iu = 0, 1 x rows jv = 0..2; H sets: iu = 0..2 x
  // jv = 0, 1); the other 3 entries have d = 0
  const bool vset = set < 2;
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const int iu = vset ? (t & 1) : (t % 3), jv = vset ? (t >> 1) : (t / 3);
    const int e = 3 * jv + iu;
    const double du = Sset[2 * e], dv = Sset[2 * e + 1];
    const double* C = pos + ((tq + jv - prow0) * kPosC + pos_col(s + iu - (P.i0 - 3))) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) { Fu[c] = fma(C[c], du, Fu[c]); Fv[c] = fma(C[c], dv, Fv[c]); }
  }
  double wq, G00, G01, G10, G11;
  if constexpr (CURVED) {   // this point's G = (dX/d(u,v))^-1 and w from the table of its knot (minus / plus point)
    const double* gm = P.mtab + ((int64_t)min(max(q, 0), P.Sv) * 2 + (set & 1)) * 5 * P.kp + min(max(p, 0), P.Su);
    G00 = __ldg(gm); G01 = __ldg(gm + P.kp); G10 = __ldg(gm + 2 * P.kp); G11 = __ldg(gm + 3 * P.kp);
    wq = __ldg(gm + 4 * P.kp);
  } else {
    wq = cst[kCstW + set] * cst[kCstP + 4];
    G00 = cst[kCstP + 0]; G01 = cst[kCstP + 1]; G10 = cst[kCstP + 2]; G11 = cst[kCstP + 3];
  }
  double f1[3], f2[3];   // F_beta = sum_mu F~_mu G_mu,beta
  if (!CURVED && P.diagG) {
#pragma unroll
    for (int c = 0; c < 3; ++c) { f1[c] = Fu[c] * G00; f2[c] = Fv[c] * G11; }
  } else {
#pragma unroll
    for (int c = 0; c < 3; ++c) { f1[c] = fma(Fu[c], G00, Fv[c] * G10); f2[c] = fma(Fu[c], G01, Fv[c] * G11); }
  }
  double* rec = row + set * kSetD + k;
  double psi, i5 = 1.0;
  // P~_mu = w sum_beta G_mu,beta P_beta;  A~_mu,nu = w sum_{beta,gamma} G_mu,beta G_nu,gamma A_beta,gamma,
  // streamed into the record as fbw_emit forms each F-space entry
  const auto emit_p = [&](int c, double P1c, double P2c) {   // explicit FMAs (see fbw_emit)
    rec[(21 + c) * kKH] = wq * fma(G00, P1c, G01 * P2c);
    rec[(24 + c) * kKH] = wq * fma(G10, P1c, G11 * P2c);
  };
  if constexpr (!HESS) {   // no Hessian requested: Psi and P only (the A entries and the projection are dead code)
    psi = fbw_emit(f1, f2, cst[kCstP + 5], cst[kCstP + 6], cst[kCstP + 7], false, emit_p,
                   [](int, int, double, double, double, double) {}, &i5);
  } else if (!CURVED && P.diagG) {   // A~uu = w G00^2 A11, A~vv = w G11^2 A22, A~uv = w G00 G11 A12
    const double auu = wq * G00 * G00, avv = wq * G11 * G11;
    const double auv = wq * G00 * G11;
    psi = fbw_emit(f1, f2, cst[kCstP + 5], cst[kCstP + 6], cst[kCstP + 7], P.project, emit_p,
                   [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
      const int e6 = sym3(r3, c3);
      rec[e6 * kKH] = auu * A11;
      rec[(6 + e6) * kKH] = avv * A22;
      rec[(12 + 3 * r3 + c3) * kKH] = auv * A12rc;
      if (r3 != c3) rec[(12 + 3 * c3 + r3) * kKH] = auv * A12cr;
    }, &i5);
  } else {
    psi = fbw_emit(f1, f2, cst[kCstP + 5], cst[kCstP + 6], cst[kCstP + 7], P.project, emit_p,
                   [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
      const int e6 = sym3(r3, c3);
      const double sym12 = A12rc + A12cr;
      rec[e6 * kKH] = wq * (G00 * G00 * A11 + G00 * G01 * sym12 + G01 * G01 * A22);
      rec[(6 + e6) * kKH] = wq * (G10 * G10 * A11 + G10 * G11 * sym12 + G11 * G11 * A22);
      rec[(12 + 3 * r3 + c3) * kKH] = wq * (G00 * G10 * A11 + G00 * G11 * A12rc + G01 * G10 * A12cr + G01 * G11 * A22);
      if (r3 != c3)
        rec[(12 + 3 * c3 + r3) * kKH] = wq * (G00 * G10 * A11 + G00 * G11 * A12cr + G01 * G10 * A12rc + G01 * G11 * A22);
    }, &i5);
  }
  if (s >= P.i0 && s < P.i1 && tq >= P.ja && tq < P.jb) {
    fbw_flag_singular(P.sflag, i5, P.item, s, tq);
    return wq * psi;
  }
  return 0.0;
}

// IP: the incremental-potential terms (compiled out of the elastic kernel); CURVED: a non-affine rest map (per-point
// G, w and Laplacian coefficients and per-cp bending blocks from the CoreTables device tables)
template <bool IP, bool CURVED, bool HESS>
__global__ void __launch_bounds__(kThreads, 1) k_core(const CoreArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);   // [kRing][kRowD]
  double* stage = ring + kRing * kRowD;                  // [2][kStageRow]  (16-B aligned: kRing*kRowD even)
  double* posb = stage + 2 * kStageRow;                  // [kPosD]
  double* cst = posb + kPosD;                            // [kCstN]
  BSF_POISON_SMEM(smem_raw);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(cst + kCstN);
  const int tid = threadIdx.x;
  CT_MARK(TK0);
  const int strip = blockIdx.x, chunk = blockIdx.y, item = blockIdx.z;
  const int i0 = A.CI0 + strip * kW, i1 = min(i0 + kW, A.CI1);
  const int nsteps = (A.JB - A.JA + kRows - 1) / kRows;
  const int sa = chunk * nsteps / A.nchunks, sb = (chunk + 1) * nsteps / A.nchunks;
  const int ja = A.JA + kRows * sa, jb = min(A.JA + kRows * sb, A.JB);
  const double* __restrict__ x = A.x + item * A.xs;
  double* vals = A.vals ? A.vals + item * A.vs : nullptr;
  // incremental potential: per-item mass scale (det J of the item's affine rest map over the handle's)
  const double msc = (IP && A.ipar) ? A.ipar[9 * (int64_t)item + 4] / A.ip_detJ : 1.0, ipk_m = A.ipk * msc;
  double* gout = A.g ? A.g + item * A.gs : nullptr;

  // ---- per-item affine map and stiffness
  PointCtx P;
  P.G00 = A.G00; P.G01 = A.G01; P.G10 = A.G10; P.G11 = A.G11; P.det = A.detJ;
  P.mu1 = A.mu1; P.mu2 = A.mu2; P.mush = A.mush; P.mubd = A.mubd;
  if (A.params) {
    const double* pp = A.params + 9 * (int64_t)item;
    P.G00 = pp[0]; P.G01 = pp[1]; P.G10 = pp[2]; P.G11 = pp[3]; P.det = pp[4];
    P.mu1 = (A.flags & 2) ? 0.0 : pp[5];
    P.mu2 = (A.flags & 2) ? 0.0 : pp[6];
    P.mush = (A.flags & 2) ? 0.0 : pp[7];
    P.mubd = (A.flags & 4) ? 0.0 : pp[8];
  }
  P.i0 = i0; P.i1 = i1; P.ja = ja; P.jb = jb; P.project = A.project != 0;
  P.sflag = A.sflag; P.item = item;
  P.mtab = A.mtab; P.btab = A.btab; P.kp = A.kp; P.Su = A.Su; P.Sv = A.Sv;
  P.diagG = (P.G01 == 0.0 && P.G10 == 0.0);
  const double cuu = P.G00 * P.G00 + P.G01 * P.G01, cvv = P.G10 * P.G10 + P.G11 * P.G11;
  const double cuv = 2.0 * (P.G00 * P.G10 + P.G01 * P.G11);
  P.wb = A.what[4] * P.det;
  if (tid < 9) {
    const double L = (tid == 8) ? 0.0 : cuu * A.tabs[72 + tid] + cvv * A.tabs[81 + tid] + cuv * A.tabs[90 + tid];
    cst[kCstL + tid] = L;
    cst[kCstLw + tid] = P.wb * P.mubd * L;
  }
  if (tid < 72) cst[kCstS + tid] = A.tabs[tid];
  if (tid == 0) {   // per-item doubles of the point phase live in shared memory (registers go to the gather)
    cst[kCstP + 0] = P.G00; cst[kCstP + 1] = P.G01; cst[kCstP + 2] = P.G10; cst[kCstP + 3] = P.G11;
    cst[kCstP + 4] = P.det; cst[kCstP + 5] = P.mu1; cst[kCstP + 6] = P.mu2; cst[kCstP + 7] = P.mush;
    cst[kCstP + 8] = P.mubd; cst[kCstP + 9] = P.wb;
  }
  if (tid < 5) cst[kCstW + tid] = A.tabs[99 + tid];
  const uint32_t bar = smem_u32(mbar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < kNB) {   // beta_ab = w mu sum_{bending q containing a, b} L_a(q) L_b(q)
    double s = 0.0;
    for (int k = 0; k < kBSlots; ++k)
      for (int e = 0; e < 8; ++e) {
        const int di = bslot_dp(k) + e % 3, dj = bslot_dq(k) + e / 3;
        if (block_index(di, dj) == tid) s += cst[kCstL + k] * cst[kCstL + e];
      }
    cst[kCstBeta + tid] = P.wb * P.mubd * s;
  }

  double e_acc = 0.0;
  // ---- warp roles: warps 0-8 gather block entry (r, c) = warp_role(warp) for both parities (warp 3, entry
  // (0, 1), also waits for the bulk stores); warps 9-15 evaluate the quadrature points of the next step
  // (7 x 30 lanes = the 210 points).  (Measured alternative, slower: one warp per entry pair (r,c) + (c,r) and
  // parity, sharing the record loads (A~uu, A~vv symmetric, A~vu[rc] = A~uv[cr]); 46 accumulators per lane and
  // twice the gather code: 705 vs 495 us on C4.  Also slower: a separate diagonal-role variant loading
  // A~uv[rr] once, 562 us, from the register allocation of the extra instantiations.)
  const int warp = tid >> 5, lane = tid & 31;
  const CoreLayout& LY = kLayouts[A.layout];
  const int role = warp < kGatherWarps ? LY.role[warp] : 0;
  const int tma = 32 * LY.tma_warp;   // the bulk-store issuing thread
  const int rr = role / 3, cc = role - 3 * (role / 3);
  const bool diag = rr == cc;
  const int o_uu = sym3(rr, cc) * kKH;
  const int o_rc = (12 + 3 * rr + cc) * kKH, o_cr = (12 + 3 * cc + rr) * kKH;
  const int h = lane >> 4, m = lane & 15;
  const int pw = warp >= kGatherWarps ? LY.pw[warp - kGatherWarps] : -1;   // point item block

  CT_MARK(TK1);
  if (ja < jb) {
    // Iteration m evaluates the quadrature points of knot rows q0 = ja-3+2m, q0+1 ("pair m") and, for
    // m >= 3, gathers the rows of step k = m-3 (j = ja+2k, needing knot rows j-2 .. j+2 = pairs k..k+2).
    // Pairs 0-2 form the prologue.  Positions of pair m+1 are fetched asynchronously during m.
    const int nst = (jb - ja + kRows - 1) / kRows;
    PosMap pm;
    pm.n = 0;
    for (int e = 0; e < 2; ++e) {
      const int kk = tid + e * kThreads;
      if (kk < kPosStep) {
        const int row = kk / (kPosC * 3), rem = kk - row * (kPosC * 3), col = rem / 3, c = rem - col * 3;
        const int Cc = i0 - 3 + col;
        pm.row[e] = row;
        pm.off[e] = (Cc >= 0 && Cc < A.n_u) ? (row * A.n_u + col) * 3 + c : -1;
        pm.dst[e] = ((row * kPosC + pos_col(col)) * 3 + c) * 8;
        pm.n = e + 1;
      }
    }
    const uint32_t pos_s = smem_u32(posb);
    // Prologue (pairs 0-2) in ONE phase on all 16 warps (round 2; it took three point-only iterations on the 7
    // point warps): the 9 cp rows [ja-4, ja+5) of its positions go to the staging buffer, idle until the first
    // bulk store, while pair 3's rows go to position buffer 1 as the main loop expects.
    double* ppos = stage;
    load_pos_async(ppos, x, A, i0, ja - 4, 9, tid);
    if (nst >= 2) load_pos_async(posb + kPosStep, x, A, i0, ja + 2, 5, tid);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // the 3 pairs' 420 membrane items first, then their 210 bending items: the second round over the 512 threads
    // holds only the cheap bending items (one membrane round instead of two)
    for (int it = tid; it < 3 * 6 * kKC; it += kThreads) {
      const bool mem = it < 3 * 4 * kKC;
      const int b = it - 3 * 4 * kKC;
      const int pr = mem ? it / (4 * kKC) : b / (2 * kKC);
      const int item = mem ? it - pr * (4 * kKC) : 4 * kKC + b - pr * (2 * kKC);
      e_acc += eval_item<CURVED, HESS>(ring, ppos + 2 * pr * (kPosC * 3), ja - 4 + 2 * pr, cst, P, ja - 3 + 2 * pr, item);
    }
    __syncthreads();
    for (int mi = 3; mi <= nst + 2; ++mi) {
      const int q0 = ja - 3 + 2 * mi, k = mi - 3, j = ja + kRows * k;
      CT_MARK(T0);
#ifdef BSF_PHASE_TIMERS
      if (tid == 0 && mi == 3) CT_ADD(12, T0 - TK1);
#endif
      // (a) positions of the next pair (async) and the quadrature points of this pair
      if (mi + 1 <= nst + 1) load_pos_step(pos_s + ((mi + 1) & 1) * (kPosStep * 8), x, A, pm, i0, q0 + 1);
      if (mi <= nst + 1 && pw >= 0 && lane < 30 && !((A.dbg & 1) && k >= 0))
        e_acc += eval_item<CURVED, HESS>(ring, posb + (mi & 1) * kPosStep, q0 - 1, cst, P, q0, pw * 30 + lane);
      CT_MARK(T1);
      if (k >= 0) {
        // (b) profiling mode without the gather: the issuing thread releases the staging buffer here (else the
        // gather warp 0 does, right before its staging stores)
        if (tid == tma && (A.dbg & 6)) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
        }
        // (c) gather of rows j, j+1: lanes = 16 control points of parity PI in each of the two rows
        if (HESS && warp < kGatherWarps && !(A.dbg & 2)) {
          // ring rows of knot rows jr-2 .. jr+1 of this lane's row jr = j + h (parity independent)
          const double* rowp[4];
          {
            int sl = ring_slot(j + h - 2);
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              rowp[d] = ring + sl * kRowD + m;
              sl = (sl == kRing - 1) ? 0 : sl + 1;
            }
          }
#pragma unroll 1
          for (int PI = 0; PI < 2; ++PI) {
            const int jr = j + h;
            const int sigma = (PI + jr + i0) & 1;
            const int i = i0 + 2 * m + sigma;
            const bool active = (i < i1) && (jr < jb);
            uint32_t base0[4], base1[4];   // shared byte addresses of the role's A~uu channel
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              base0[d] = smem_u32(rowp[d]) + 8 * o_uu;
              base1[d] = base0[d] + 8 * sigma;
            }
            // staging: row h of the step; base parity matched to the global address (TMA needs equal
            // alignment mod 16 on both sides)
            double* st_lane = nullptr;
            if (vals && !(A.dbg & 4)) {
              const int64_t g0 = (A.rp_base + (int64_t)(jr - A.RJ0) * A.rp_stride + (int64_t)(i0 - A.CI0) * kNB) * 9;
              const int pad = (int)(((uintptr_t)(vals + g0) >> 3) & 1);
              st_lane = stage + h * kStageRow + pad + (i - i0) * (kNB * 9) + 3 * rr + cc;
            }
            const uint32_t par = k & 1;
            const double dshift = (IP && diag && active) ? ipk_m * A.mass[(int64_t)(jr - A.r0) * A.n_u + i] : 0.0;
            const int orc = 8 * (o_rc - o_uu), ocr = 8 * (o_cr - o_uu);
            // curved: the lane's row of the per-cp bending table (a valid row for inactive lanes)
            const double* bsrc = CURVED ? A.beta + ((int64_t)(active ? jr - A.RJ0 : 0) * kNB) * A.cw + (active ? i - A.CI0 : 0)
                                        : nullptr;
            if (PI == 0)
              gather_role<0, CURVED>(base0, base1, orc, ocr, diag, cst, st_lane, active, bar, par, dshift, bsrc, A.cw,
                                     P.mubd, tid == tma);
            else
              gather_role<1, CURVED>(base0, base1, orc, ocr, diag, cst, st_lane, active, bar, par, dshift, bsrc, A.cw,
                                     P.mubd, tid == tma);
          }
        }
      }
      // (c') gradient rows of step k: the point warps take the six (parity, component) rounds (layout)
      const int gr0 = warp >= kGatherWarps ? LY.g0[warp - kGatherWarps] : 0;
      const int gr1 = warp >= kGatherWarps ? gr0 + LY.gn[warp - kGatherWarps] : 0;
#pragma unroll 1
      for (int gw = gr0; gw < gr1; ++gw)
      if (k >= 0 && (gout || IP) && !(A.dbg & 2)) {
        const int PI = gw / 3, rg = gw % 3;
        const int jr = j + h;
        const int sigma = (PI + jr + i0) & 1;
        const int i = i0 + 2 * m + sigma;
        if ((i < i1) && (jr < jb)) {
          uint32_t gb0[4], gb1[4];
          int sl = ring_slot(jr - 2);
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            gb0[d] = smem_u32(ring + sl * kRowD + m);
            gb1[d] = gb0[d] + 8 * sigma;
            sl = (sl == kRing - 1) ? 0 : sl + 1;
          }
          {
            const int r = rg;
            const double* bb0[3];
            const double* bb1[3];
            int s2 = ring_slot(jr - 2);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double* rb = ring + s2 * kRowD + 4 * kSetD + r * kKH + m;
              bb0[d] = rb + sigma * kBendD;
              bb1[d] = rb + (1 - sigma) * kBendD + sigma;
              s2 = (s2 == kRing - 1) ? 0 : s2 + 1;
            }
            const int64_t al = (int64_t)(jr - A.r0) * A.n_u + i;
            double* gdst = gout ? gout + al * 3 + r : nullptr;
            // incremental potential: m/dt^2 (x - xhat) - m g on the gradient, its energy on this lane
            double g0 = 0.0;
            if constexpr (IP) {
              const double mm = A.mass[al] * msc, xa = x[((int64_t)(jr - A.xlo) * A.n_u + i) * 3 + r];
              const double d = xa - A.xhat[item * A.xhs + al * 3 + r], gr = A.grav[r];
              g0 = A.ipk * mm * d - mm * gr;
              e_acc += 0.5 * A.ipk * mm * d * d - mm * gr * xa;
            }
            if (gout) {
              const uint32_t opu = 8 * (21 + r) * kKH, opv = 8 * (24 + r) * kKH;
              const double* gsrc = CURVED ? A.gw + ((int64_t)(jr - A.RJ0) * kBSlots) * A.cw + (i - A.CI0) : nullptr;
              if (PI == 0) gather_grad<0, CURVED>(gb0, gb1, bb0, bb1, opu, opv, cst, gdst, g0, gsrc, A.cw, P.mubd);
              else gather_grad<1, CURVED>(gb0, gb1, bb0, bb1, opu, opv, cst, gdst, g0, gsrc, A.cw, P.mubd);
            }
          }
        }
      }
      CT_MARK(T2);
      asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      CT_MARK(T3);
      __syncthreads();
      CT_MARK(T4);
#ifdef BSF_PHASE_TIMERS
      if (k >= 0 && lane == 0) atomicAdd(&g_warp_t[warp], (unsigned long long)(T3 - T0));
      if (k >= 0 && lane == 0) {
        if (warp == kGatherWarps) { CT_ADD(0, T1 - T0); CT_ADD(7, T2 - T1); }
        if (warp == 0) { CT_ADD(1, T2 - T1); CT_ADD(3, T3 - T2); CT_ADD(4, T4 - T3); CT_ADD(5, T4 - T0); CT_ADD(6, 1); }
        if (warp == 2) CT_ADD(2, T2 - T1);
      }
#endif
      // (d) bulk stores of the step's rows (head / tail doubles off the 16-B grid by plain stores)
      if (k >= 0 && vals && tid >= tma && tid < tma + 5) {
        for (int hh = 0; hh < kRows; ++hh) {
          const int jr2 = j + hh;
          if (jr2 >= jb) break;
          const int64_t g0 = (A.rp_base + (int64_t)(jr2 - A.RJ0) * A.rp_stride + (int64_t)(i0 - A.CI0) * kNB) * 9;
          double* gd = vals + g0;
          const int pad = (int)(((uintptr_t)gd >> 3) & 1);
          const double* sp = stage + hh * kStageRow + pad;
          const int64_t nd = (int64_t)(i1 - i0) * (kNB * 9);
          const int head = pad;                                  // 1 double if gd is 8 mod 16
          const int tail = (int)((nd - head) & 1);               // 1 double if the end is 8 mod 16
          if (tid == tma) {
            const int64_t nb = (A.dbg & 8) ? 0 : nd - head - tail;
            if (nb > 0)
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gd + head),
                           "r"(smem_u32(sp + head)), "r"((uint32_t)(nb * 8))
                           : "memory");
          } else if (tid == tma + 1 + hh) {
            if (head) gd[0] = sp[0];
          } else if (tid == tma + 3 + hh) {
            if (tail) gd[nd - 1] = sp[nd - 1];
          }
        }
        if (tid == tma) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
#ifdef BSF_PHASE_TIMERS
      if (k >= 0 && (tid == 0 || tid == 32)) { CT_MARK(T5); CT_ADD(tid ? 14 : 13, T5 - T4); }
#endif
    }
  }
  CT_MARK(TK2);
  if (tid == tma) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef BSF_PHASE_TIMERS
  if (tid == 0) { CT_ADD(8, TK1 - TK0); CT_ADD(9, TK2 - TK1); CT_ADD(10, 1); CT_ADD(11, clock64() - TK0); }
#endif
  // ---- energy partial of this CTA (fixed-order tree)
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  __syncthreads();
  if ((tid & 31) == 0) cst[kCstRed + (tid >> 5)] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += cst[kCstRed + w];
    A.epart[item * A.e_stride + A.e_off + (int64_t)chunk * A.nstrips + strip] = s;
  }
  energy_final_fused(A.ef, A.epart, item);
}

// Energy-only calls on affine sheets (the line search): the quadrature points whose anchor lies in the
// CTA's [i0, i1) x [ja, jb) (k_core's ownership), one thread per anchor (s, t): its 2 membrane points (V+ and H-
// when s + t is even, V- and H+ when odd; Q1) and its bending point, straight from the positions in
// global memory (no ring, no staging, no gather), plus the incremental-potential terms of the control point
// (s, t).  Same per-point arithmetic as eval_item; the per-CTA sum is in another order than k_core's.
constexpr int kEThreads = 256;

template <bool IP>
__global__ void __launch_bounds__(kEThreads) k_core_energy(const CoreArgs A) {
  __shared__ double c[kCstN];
  __shared__ double red[kEThreads / 32];
  const int tid = threadIdx.x;
  const int strip = blockIdx.x, chunk = blockIdx.y, item = blockIdx.z;
  const int i0 = A.CI0 + strip * kW, i1 = min(i0 + kW, A.CI1);
  const int nsteps = (A.JB - A.JA + kRows - 1) / kRows;
  const int sa = chunk * nsteps / A.nchunks, sb = (chunk + 1) * nsteps / A.nchunks;
  const int ja = A.JA + kRows * sa, jb = min(A.JA + kRows * sb, A.JB);
  const double* __restrict__ x = A.x + item * A.xs;
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
  const bool diagG = (G01 == 0.0 && G10 == 0.0);
  const double cuu = G00 * G00 + G01 * G01, cvv = G10 * G10 + G11 * G11, cuv = 2.0 * (G00 * G10 + G01 * G11);
  const double wb = A.what[4] * det;
  if (tid < 9) c[kCstL + tid] = (tid == 8) ? 0.0 : cuu * A.tabs[72 + tid] + cvv * A.tabs[81 + tid] + cuv * A.tabs[90 + tid];
  if (tid < 72) c[kCstS + tid] = A.tabs[tid];
  if (tid < 5) c[kCstW + tid] = A.tabs[99 + tid];
  __syncthreads();
  const double msc = (IP && A.ipar) ? A.ipar[9 * (int64_t)item + 4] / A.ip_detJ : 1.0;
  double e_acc = 0.0;
  const int nw = i1 - i0, na = nw * max(0, jb - ja);
  for (int a = tid; a < na; a += kEThreads) {
    const int t = ja + a / nw, s = i0 + a - (a / nw) * nw;
    const double* xw = x + ((int64_t)(t - A.xlo) * A.n_u + s) * 3;   // window origin (s, t)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int set = ((s + t) & 1) ? (h ? 3 : 0) : (h ? 2 : 1);
      const bool vset = set < 2;
      const double* Sset = c + kCstS + set * 18;
      double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0};
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int iu = vset ? (q & 1) : (q % 3), jv = vset ? (q >> 1) : (q / 3);
        const int e = 3 * jv + iu;
        const double du = Sset[2 * e], dv = Sset[2 * e + 1];
        const double* C = xw + ((int64_t)jv * A.n_u + iu) * 3;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) { Fu[cc] = fma(__ldg(C + cc), du, Fu[cc]); Fv[cc] = fma(__ldg(C + cc), dv, Fv[cc]); }
      }
      double f1[3], f2[3];
      if (diagG) {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) { f1[cc] = Fu[cc] * G00; f2[cc] = Fv[cc] * G11; }
      } else {
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) { f1[cc] = fma(Fu[cc], G00, Fv[cc] * G10); f2[cc] = fma(Fu[cc], G01, Fv[cc] * G11); }
      }
      double i5 = 1.0;
      const double psi = fbw_emit(f1, f2, mu1, mu2, mush, false, [](int, double, double) {},
                                  [](int, int, double, double, double, double) {}, &i5);
      e_acc += c[kCstW + set] * det * psi;
      fbw_flag_singular(A.sflag, i5, item, s, t);
    }
    double lap[3] = {0, 0, 0};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double L = c[kCstL + e];
      const double* C = xw + ((int64_t)(e / 3) * A.n_u + e % 3) * 3;
      lap[0] = fma(L, __ldg(C), lap[0]); lap[1] = fma(L, __ldg(C + 1), lap[1]); lap[2] = fma(L, __ldg(C + 2), lap[2]);
    }
    e_acc += 0.5 * wb * mubd * fma(lap[0], lap[0], fma(lap[1], lap[1], lap[2] * lap[2]));
    if constexpr (IP) {
      const int64_t al = (int64_t)(t - A.r0) * A.n_u + s;
      const double mm = A.mass[al] * msc;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const double xa = xw[r], d = xa - A.xhat[item * A.xhs + al * 3 + r];
        e_acc += 0.5 * A.ipk * mm * d * d - mm * A.grav[r] * xa;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kEThreads / 32; ++w) sum += red[w];
    A.epart[item * A.e_stride + A.e_off + (int64_t)chunk * A.nstrips + strip] = sum;
  }
  energy_final_fused(A.ef, A.epart, item);
}

}  // namespace

// ------------------------------------------------------------------------------------------ host
namespace {

int set_of(const Point& P) {   // -1: not an interior-template membrane point
  const uint16_t V = 0xDB;      // window entries iu in {0,1}: a point on a knot line u = p (2x3 stencil)
  const uint16_t H = 0x3F;      // entries jv in {0,1}: a point on v = q (3x2)
  const int par = (P.ou + P.ov) & 1;
  if (P.mask == V) return par ? 0 : 1;          // V-: anchor (p, q-1), p+q even -> s+t odd
  if (P.mask == H) return par ? 3 : 2;          // H-: anchor (p-1, q), p+q odd -> s+t even
  return -1;
}

void point_du_dv(const Point& P, double (&S)[9][2]) {
  for (int e = 0; e < 9; ++e) {
    const int iu = e % 3, jv = e / 3;
    const bool in = (P.mask >> e) & 1;
    S[e][0] = in ? P.bu.d1[iu] * P.bv.N[jv] : 0.0;
    S[e][1] = in ? P.bu.N[iu] * P.bv.d1[jv] : 0.0;
  }
}

}  // namespace

int build_core(const Sheet& sh, const int32_t* d_row_ptr, CoreTables& ct, std::string& err,
               const std::function<void*(size_t)>& dalloc) {
  ct = CoreTables();
  ct.row_ptr = const_cast<int32_t*>(d_row_ptr);
  if (sh.mrule != RULE_REDUCED || sh.brule != RULE_REDUCED || (!sh.affine && getenv("BSF_NO_CURVED_CORE"))) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  const int nu = sh.n_u, Su = sh.Su, Sv = sh.Sv;
  if (nu < 16 || sh.n_v < 16) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  // ---- anchor buckets
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
  // ---- representatives near the middle of the owned rows
  const int jc = (sh.r0 + sh.r1) / 2, ic = nu / 2;
  bool have[5] = {false, false, false, false, false};
  for (int t = std::max(0, jc - 3); t <= std::min(Sv - 1, jc + 1); ++t)
    for (int s = std::max(0, ic - 3); s <= std::min(Su - 1, ic + 1); ++s) {
      const int an = t * Su + s;
      for (int k = mh[an]; k < mh[an + 1]; ++k) {
        const Point& P = sh.mem[mi[k]];
        const int set = set_of(P);
        if (set < 0 || have[set]) continue;
        std::memcpy(ct.S[set], kSetTable.v[set], sizeof(ct.S[set]));
        ct.what[set] = P.what;
        have[set] = true;
      }
      for (int k = bh[an]; k < bh[an + 1]; ++k) {
        const Point& P = sh.bend[bi[k]];
        if (have[4] || P.mask != 0xFF) continue;
        for (int e = 0; e < 9; ++e) {
          const int iu = e % 3, jv = e / 3;
          const bool in = (P.mask >> e) & 1;
          ct.LA[e] = in ? P.bu.d2[iu] * P.bv.N[jv] : 0.0;
          ct.LB[e] = in ? P.bu.N[iu] * P.bv.d2[jv] : 0.0;
          ct.LC[e] = in ? P.bu.d1[iu] * P.bv.d1[jv] : 0.0;
        }
        ct.what[4] = P.what;
        have[4] = true;
      }
    }
  for (bool hv : have)
    if (!hv) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  // ---- per-control-point conformance with the template (owned rows)
  const double tol = 1e-12;
  auto close = [&](double a, double b) { return std::fabs(a - b) <= tol * std::max(1.0, std::fabs(b)); };
  constexpr Template T0 = make_template(0), T1 = make_template(1);
  auto conforms = [&](int i, int j) -> bool {
    if (i < 2 || j < 2 || i > nu - 3 || j > sh.n_v - 3) return false;
    const Template& T = ((i + j) & 1) ? T1 : T0;
    // membrane: exactly the template's 12 points
    int found = 0;
    for (int t = j - 2; t <= j; ++t)
      for (int s = i - 2; s <= i; ++s) {
        if (s < 0 || t < 0 || s >= Su || t >= Sv) continue;
        const int an = t * Su + s;
        for (int k = mh[an]; k < mh[an + 1]; ++k) {
          const Point& P = sh.mem[mi[k]];
          const int ea = (i - s) + 3 * (j - t);
          if (!((P.mask >> ea) & 1)) continue;
          const int set = set_of(P);
          if (set < 0) return false;
          int slot = -1;
          for (int z = 0; z < T.nslot; ++z)
            if (T.s_set[z] == set && T.s_ea[z] == ea) slot = z;
          if (slot < 0) return false;
          if (!close(P.what, ct.what[set])) return false;
          double S[9][2];
          point_du_dv(P, S);
          for (int e = 0; e < 9; ++e)
            if (!close(S[e][0], ct.S[set][e][0]) || !close(S[e][1], ct.S[set][e][1])) return false;
          ++found;
        }
      }
    if (found != T.nslot) return false;
    int bfound = 0;
    for (int t = j - 2; t <= j; ++t)
      for (int s = i - 2; s <= i; ++s) {
        if (s < 0 || t < 0 || s >= Su || t >= Sv) continue;
        const int an = t * Su + s;
        for (int k = bh[an]; k < bh[an + 1]; ++k) {
          const Point& P = sh.bend[bi[k]];
          const int ea = (i - s) + 3 * (j - t);
          if (!((P.mask >> ea) & 1)) continue;
          if (P.mask != 0xFF || !close(P.what, ct.what[4])) return false;
          for (int e = 0; e < 9; ++e) {
            const int iu = e % 3, jv = e / 3;
            const bool in = (P.mask >> e) & 1;
            if (!close(in ? P.bu.d2[iu] * P.bv.N[jv] : 0.0, ct.LA[e]) ||
                !close(in ? P.bu.N[iu] * P.bv.d2[jv] : 0.0, ct.LB[e]) ||
                !close(in ? P.bu.d1[iu] * P.bv.d1[jv] : 0.0, ct.LC[e]))
              return false;
          }
          ++bfound;
        }
      }
    if (bfound != kBSlots) return false;
    // pattern row: the 23 standard columns
    const int64_t al = (int64_t)(j - sh.r0) * nu + i;
    if (sh.row_ptr[al + 1] - sh.row_ptr[al] != kNB) return false;
    for (int k = 0; k < kNB; ++k)
      if (sh.col_idx[sh.row_ptr[al] + k] != (j + block_dj(k)) * nu + i + block_di(k)) return false;
    return true;
  };
  // rectangle: conformant columns of the middle owned row, then the owned rows on which all of them conform
  const int jm = std::min(std::max(jc, sh.r0), sh.r1 - 1);
  int c0 = ic, c1 = ic;
  if (!conforms(ic, jm)) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  while (c0 - 1 >= 0 && conforms(c0 - 1, jm)) --c0;
  while (c1 + 1 < nu && conforms(c1 + 1, jm)) ++c1;
  ++c1;
  auto row_ok = [&](int j) {
    for (int i = c0; i < c1; ++i)
      if (!conforms(i, j)) return false;
    return true;
  };
  int j0 = jm, j1 = jm;
  while (j0 - 1 >= sh.r0 && row_ok(j0 - 1)) --j0;
  while (j1 + 1 < sh.r1 && row_ok(j1 + 1)) ++j1;
  ++j1;
  if (!row_ok(jm)) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  if (c1 - c0 < 8 || j1 - j0 < 1) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  ct.CI0 = c0; ct.CI1 = c1; ct.CJ0 = j0; ct.CJ1 = j1; ct.RJ0 = j0; ct.RJ1 = j1;
  {   // row starts of the rectangle: affine in the row (every core row has the same frame columns)
    auto rp = [&](int i, int j) { return (int64_t)sh.row_ptr[(int64_t)(j - sh.r0) * nu + i]; };
    ct.rp_base = rp(c0, j0);
    ct.rp_stride = (j1 - j0 > 1) ? rp(c0, j0 + 1) - rp(c0, j0) : 0;
    for (int j = j0; j < j1; ++j)
      for (int i = c0; i < c1; ++i)
        if (rp(i, j) != ct.rp_base + (int64_t)(j - j0) * ct.rp_stride + (int64_t)(i - c0) * kNB) { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  }
  ct.nstrips = (c1 - c0 + kW - 1) / kW;
  // ---- coefficient tables
  for (int pi = 0; pi < 2; ++pi) {
    const Template T = make_template(pi);
    for (int s = 0; s < T.nslot; ++s) {
      const double* da = ct.S[T.s_set[s]][T.s_ea[s]];
      ct.D[pi][s][0] = da[0];
      ct.D[pi][s][1] = da[1];
      for (int c = T.s_c0[s]; c < T.s_c0[s] + T.s_nc[s]; ++c) {
        const double* db = ct.S[T.s_set[s]][T.c_eb[c]];
        const double k11 = da[0] * db[0], k22 = da[1] * db[1], k12 = da[0] * db[1], k21 = da[1] * db[0];
        ct.K[pi][c][0] = k11;
        ct.K[pi][c][1] = k22;
        ct.K[pi][c][2] = 0.5 * (k12 + k21);
        ct.K[pi][c][3] = 0.5 * (k12 - k21);
      }
    }
  }
  {
    const Point& ref = sh.mem.empty() ? sh.bend[0] : sh.mem[0];
    ct.G[0] = ref.G[0][0]; ct.G[1] = ref.G[0][1]; ct.G[2] = ref.G[1][0]; ct.G[3] = ref.G[1][1];
    ct.detJ = ref.detJ;
  }
  if (!sh.affine) {   // curved rest map: per-point rest tables (see CoreTables)
    ct.curved = 1;
    const int64_t kp = Su + 1, nq = Sv + 1;
    ct.kp = kp;
    ct.cw = c1 - c0;
    std::vector<double> mt((size_t)nq * 2 * 5 * kp, 0.0), bt((size_t)nq * 10 * kp, 0.0);
    for (const Point& P : sh.mem) {
      const int set = set_of(P);
      if (set < 0) continue;
      const int p = P.ou + (set == 2 ? 1 : 0), q = P.ov + (set == 0 ? 1 : 0), pm = set & 1;
      double* d = &mt[(((size_t)q * 2 + pm) * 5) * kp + p];
      d[0] = P.G[0][0]; d[kp] = P.G[0][1]; d[2 * kp] = P.G[1][0]; d[3 * kp] = P.G[1][1]; d[4 * kp] = P.w;
    }
    std::vector<int32_t> bidx((size_t)nq * kp, -1);   // interior bending point of knot (p, q)
    for (size_t k = 0; k < sh.bend.size(); ++k) {
      const Point& P = sh.bend[k];
      if (P.mask != 0xFF) continue;
      bidx[(size_t)P.ov * kp + P.ou] = (int32_t)k;
      for (int e = 0; e < 9; ++e) bt[((size_t)P.ov * 10 + e) * kp + P.ou] = P.L[e];
      bt[((size_t)P.ov * 10 + 9) * kp + P.ou] = P.w;
    }
    const int64_t nr = j1 - j0, cw = c1 - c0;
    std::vector<double> be((size_t)nr * kNB * cw, 0.0), gwv((size_t)nr * kBSlots * cw, 0.0);
    for (int j = j0; j < j1; ++j)
      for (int i = c0; i < c1; ++i)
        for (int k = 0; k < kBSlots; ++k) {
          const int p = i + bslot_dp(k), q = j + bslot_dq(k);
          const int32_t bk = bidx[(size_t)q * kp + p];
          if (bk < 0) { err = "core: curved tables: missing bending point"; return -1; }
          const Point& P = sh.bend[bk];
          gwv[((size_t)(j - j0) * kBSlots + k) * cw + (i - c0)] = P.w * P.L[k];
          for (int eb = 0; eb < 8; ++eb) {
            const int blk = block_index(bslot_dp(k) + eb % 3, bslot_dq(k) + eb / 3);
            if (blk >= 0) be[((size_t)(j - j0) * kNB + blk) * cw + (i - c0)] += P.w * P.L[k] * P.L[eb];
          }
        }
    auto up = [&](double** dst, const std::vector<double>& v) {
      void* p = dalloc(v.size() * sizeof(double));
      if (!p || cudaMemcpy(p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) return false;
      *dst = static_cast<double*>(p);
      return true;
    };
    if (!up(&ct.mtab, mt) || !up(&ct.btab, bt) || !up(&ct.beta, be) || !up(&ct.gw, gwv)) {
      err = "core: curved table upload failed";
      return -7;
    }
    ct.table_bytes = sizeof(double) * (mt.size() + bt.size() + be.size() + gwv.size());
  }
  {
    std::vector<double> tabs(104, 0.0);
    std::memcpy(tabs.data(), ct.S, sizeof(ct.S));
    std::memcpy(tabs.data() + 72, ct.LA, sizeof(ct.LA));
    std::memcpy(tabs.data() + 81, ct.LB, sizeof(ct.LB));
    std::memcpy(tabs.data() + 90, ct.LC, sizeof(ct.LC));
    std::memcpy(tabs.data() + 99, ct.what, sizeof(ct.what));
    void* p = dalloc(tabs.size() * sizeof(double));
    if (!p || cudaMemcpy(p, tabs.data(), tabs.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
      err = "core: table upload failed";
      return -7;
    }
    ct.d_tabs = static_cast<double*>(p);
  }
  ct.smem = sizeof(double) * ((size_t)kRing * kRowD + 2 * kStageRow + kPosD + kCstN) + 16;
  if (ct.smem > 227 * 1024) { err = "core: shared memory budget"; return -1; }
  const auto attr = [&](auto fn) {
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ct.smem) == cudaSuccess;
  };
  if (!attr(k_core<false, false, true>) || !attr(k_core<true, false, true>) || !attr(k_core<false, true, true>) ||
      !attr(k_core<true, true, true>) || !attr(k_core<false, false, false>) || !attr(k_core<true, false, false>) ||
      !attr(k_core<false, true, false>) || !attr(k_core<true, true, false>)) {
    cudaGetLastError();
    { if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_core: no core (line %d)\n", __LINE__); return 1; }
  }
  if (getenv("BSF_CORE_DEBUG")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_core<false, false, true>);
    int nb = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_core<false, false, true>, kThreads, ct.smem);
    fprintf(stderr, "k_core: regs %d maxthreads %d local %zu static smem %zu dyn %zu maxdyn %d occ %d\n", fa.numRegs,
            fa.maxThreadsPerBlock, fa.localSizeBytes, fa.sharedSizeBytes, ct.smem, fa.maxDynamicSharedSizeBytes, nb);
  }
  ct.ok = 1;
  (void)err;
  return 0;
}

int core_ctas_per_item(const CoreTables& ct, int nchunks) { return ct.nstrips * nchunks; }

constexpr int kOneWaveRows = 192;    // longest row chunk of the one-wave choice
constexpr double kSideRoundRows = 24;   // one round of band CTAs (2 per SM, ~43 us) in k_core row steps (~1.8 us)

int core_pick_chunks(const CoreTables& ct, int nbatch, int rows_override, int reserved_sms) {
  // row chunks per (strip, item): minimise (waves of 1 CTA per SM) x (rows per chunk + the 6-row prologue
  // of a chunk); chunks of >= 16 rows.  The band / corner kernels run beside k_core and fill a partial
  // last wave, so large batches prefer few long chunks and small ones many.
  // Small problems (one strip row of CTAs fits beside the band / corner kernels, e.g. one C2 or C3 sheet): the
  // most chunks that still run in ONE wave on the SMs the band / corner kernels leave free, chunks of >= 6
  // rows (measured on C2 / C3: more chunks starve the band kernel, shorter chunks pay the prologue again).
  static const int nsm = [] {
    int d = 0, n = 0;
    cudaGetDevice(&d);
    return cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) == cudaSuccess && n > 0 ? n : 148;
  }();
  // experiment switches (read once): BSF_CORE_MINROWS (shortest chunk, rows), BSF_CORE_PROLOGUE (row cost of
  // a chunk's prologue)
  static const int min_rows = getenv("BSF_CORE_MINROWS") ? std::max(2, atoi(getenv("BSF_CORE_MINROWS"))) : 16;
  static const double prologue = getenv("BSF_CORE_PROLOGUE") ? atof(getenv("BSF_CORE_PROLOGUE")) : 6.0;
  static const int force_nch = getenv("BSF_CORE_NCH") ? atoi(getenv("BSF_CORE_NCH")) : 0;
  if (force_nch > 0) return std::min(force_nch, std::max(1, (rows_override >= 0 ? rows_override : ct.RJ1 - ct.RJ0) / 2));
  const int rows = rows_override >= 0 ? rows_override : ct.RJ1 - ct.RJ0;
  const int per = std::max(1, ct.nstrips * std::max(1, nbatch));
  if (reserved_sms > 0 && per <= 16 && per + reserved_sms < nsm)
    return std::max(1, std::min((nsm - reserved_sms) / per, rows / 6));
  // One wave when the chunks stay short enough (row slabs of a multi-GPU split): the chunk count minimising
  // max(chunk rows + prologue, rounds of the band / corner kernels on the SMs k_core leaves free x
  // kSideRoundRows), with all core CTAs in one wave.  Measured on C4 row slabs against the multi-wave choice
  // below (whose second wave starts late behind the side kernels): 512 rows 263 -> 251 us, 256 rows
  // 162 -> 142 us; an N = 8 edge slab (92 core rows, 76 band CTAs) is faster in 3 chunks than in 4 (the band
  // kernel gets one round); a whole 1024^2 sheet, 256 rows per chunk, is faster in two waves (430 vs 466 us).
  if (per < nsm) {
    int best1 = 0;
    double c1 = 1e300;
    for (int nch = 1; per * nch < nsm && nch <= std::max(1, rows / 6); ++nch) {
      const int free_sms = nsm - per * nch;
      const int rounds = reserved_sms > 0 ? (reserved_sms + free_sms - 1) / free_sms : 0;
      const double cost = std::max((double)rows / nch + prologue, (double)rounds * kSideRoundRows);
      if (cost < c1 - 1e-9) { c1 = cost; best1 = nch; }
    }
    if (best1 > 0 && rows <= kOneWaveRows * best1) return best1;
  }
  const int maxch = std::max(1, rows / min_rows);
  int best = 1;
  double bcost = 1e300;
  for (int nch = 1; nch <= maxch; ++nch) {
    const long long nctas = (long long)per * nch;
    const long long waves = (nctas + 147) / 148;
    const double cost = (double)waves * ((double)rows / nch + prologue);
    if (cost < bcost - 1e-9) { bcost = cost; best = nch; }
  }
  return best;
}

int core_eval(const CoreTables& ct, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, double* e_part,
              int64_t e_stride, int64_t e_off, int nchunks, const double* d_params, double detJ_ref,
              cudaStream_t st, const IpFused* ip, int row_begin, int row_end) {
  (void)detJ_ref;
  CoreArgs A;
  A.JA = row_begin >= 0 ? row_begin : ct.RJ0;
  A.JB = row_end >= 0 ? row_end : ct.RJ1;
  if (A.JB <= A.JA) return 0;
  A.xhat = ip ? ip->xhat : nullptr; A.xhs = ip ? ip->xhs : 0; A.mass = ip ? ip->mass : nullptr;
  A.ipk = ip ? ip->k : 0.0;
  for (int c = 0; c < 3; ++c) A.grav[c] = ip ? ip->grav[c] : 0.0;
  A.ipar = ip ? ip->params : nullptr;
  A.ip_detJ = ip ? ip->detJ_ref : 1.0;
  A.x = d_x; A.xs = x_stride; A.g = d_g; A.gs = g_stride; A.vals = d_vals; A.vs = v_stride;
  A.epart = e_part; A.e_stride = e_stride; A.e_off = e_off;
  A.row_ptr = ct.row_ptr; A.rp_base = ct.rp_base; A.rp_stride = ct.rp_stride; A.params = d_params;
  A.n_u = sh.n_u; A.xlo = sh.xlo; A.xhi = sh.xhi; A.r0 = sh.r0;
  A.CI0 = ct.CI0; A.CI1 = ct.CI1; A.RJ0 = ct.RJ0; A.RJ1 = ct.RJ1; A.nstrips = ct.nstrips; A.nchunks = nchunks;
  A.project = (flags & 1) ? 1 : 0; A.flags = flags; A.sflag = call_sflag(); A.ef = call_efinal();
  {   // profiling switches (read once per process): 1 no points, 2 no gather, 4 no stores
    static const int dbg = getenv("BSF_CORE_DEBUG") ? atoi(getenv("BSF_CORE_DEBUG")) : 0;
    A.dbg = dbg;
    static const int layout = getenv("BSF_CORE_LAYOUT") ? std::min(7, std::max(0, atoi(getenv("BSF_CORE_LAYOUT")))) : 6;
    A.layout = layout;
  }
  A.G00 = ct.G[0]; A.G01 = ct.G[1]; A.G10 = ct.G[2]; A.G11 = ct.G[3]; A.detJ = ct.detJ;
  A.mu1 = (flags & 2) ? 0.0 : mat.mu_st1;
  A.mu2 = (flags & 2) ? 0.0 : mat.mu_st2;
  A.mush = (flags & 2) ? 0.0 : mat.mu_sh;
  A.mubd = (flags & 4) ? 0.0 : mat.mu_bd;
  A.tabs = ct.d_tabs;
  std::memcpy(A.what, ct.what, sizeof(A.what));

  dim3 grid(ct.nstrips, nchunks, nbatch);
  A.mtab = ct.mtab; A.btab = ct.btab; A.beta = ct.beta; A.gw = ct.gw; A.kp = ct.kp; A.cw = ct.cw;
  A.Su = sh.Su; A.Sv = sh.Sv;
  if (ct.curved) {
    if (A.vals) {
      if (A.xhat) k_core<true, true, true><<<grid, kThreads, ct.smem, st>>>(A);
      else k_core<false, true, true><<<grid, kThreads, ct.smem, st>>>(A);
    } else {
      if (A.xhat) k_core<true, true, false><<<grid, kThreads, ct.smem, st>>>(A);
      else k_core<false, true, false><<<grid, kThreads, ct.smem, st>>>(A);
    }
  } else {
    static const bool no_ekernel = getenv("BSF_CORE_NO_EKERNEL") != nullptr;   // test switch
    if (A.vals) {
      if (A.xhat) k_core<true, false, true><<<grid, kThreads, ct.smem, st>>>(A);
      else k_core<false, false, true><<<grid, kThreads, ct.smem, st>>>(A);
    } else if (!A.g && !no_ekernel) {   // energy only: no ring, no gather (k_core_energy)
      if (A.xhat) k_core_energy<true><<<grid, kEThreads, 0, st>>>(A);
      else k_core_energy<false><<<grid, kEThreads, 0, st>>>(A);
    } else {   // energy / gradient calls: no Hessian gather, no A entries
      if (A.xhat) k_core<true, false, false><<<grid, kThreads, ct.smem, st>>>(A);
      else k_core<false, false, false><<<grid, kThreads, ct.smem, st>>>(A);
    }
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

#ifdef BSF_PHASE_TIMERS
extern "C" int bsf_debug_core_timers(unsigned long long* out48, int reset) {
  cudaMemcpyFromSymbol(out48, g_core_t, sizeof(unsigned long long) * 16);
  cudaMemcpyFromSymbol(out48 + 16, g_warp_t, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(g_core_t, z, sizeof(unsigned long long) * 16);
    cudaMemcpyToSymbol(g_warp_t, z, sizeof(z));
  }
  return 0;
}
#endif
}  // namespace bsf
