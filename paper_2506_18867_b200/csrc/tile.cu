// Fused tile path of the assembly (the hot path).
//
// One CTA owns a strip of kTX control-point columns over a chunk of rows of one sheet (grid.z =
// batch item).  It walks the chunk kRS output rows at a time:
//   1. stage the positions of the rows the new anchor rows need (coalesced loads);
//   2. point phase: evaluate every quadrature point whose stencil origin ("anchor") lies in the two
//      new anchor rows of the strip window — F = F~ G, FBW Psi, P, A
//       with optional per-term PSD projection — and keep the parametric-frame
//      data  A~ = w (G (x) I) A (G (x) I)^T,  P~ = w G P  (membrane) or  L^ = sqrt(w mu) L,
//      D^ = sqrt(w mu) Lap phi  (bending)  in a shared-memory ring of 4 anchor rows;
//   3. gather: each thread owns one (control point a, row offset dj) task = the <=5 contiguous BSR
//      blocks of row a whose columns lie in row j+dj; it walks the host-built incidence program of
//      a's boundary/parity class, loading each incident point's A~ once and accumulating
//      H_ab = sum_q sum_{mu,nu} d_a,mu d_b,nu A~_mu,nu  (+ sum_q' L^_a L^_b I3)  in registers
//      (the paper's per-block gather, without atomics); a 6th task per point
//      gathers g_a = sum_q d_a . P~ + sum_q' L^_a D^;
//   4. the strip's row segments are staged in shared memory and written to HBM coalesced.
// The energy is reduced per CTA (points owned by anchor) and summed per item by k_energy_final.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

#include "core.hpp"
#include "fbw.cuh"
#include "frame.hpp"
#include "tile.hpp"
#include "ip.hpp"

namespace bsf {

namespace {

constexpr int kPosCols = kTX + 4;
constexpr int kPosRows = kRS + 2;
constexpr int kAC = kTX + 2;   // anchor columns of a strip window

__host__ __device__ inline int bclass(int i, int n) {
  if (i < 6) return i;
  if (i >= n - 6) return 7 + (i - (n - 6));
  return 6;
}

struct TileArgs {
  const double* x;
  int64_t xs;
  double* g;
  int64_t gs;
  double* vals;
  int64_t vs;
  double* epart;
  int n_u, n_v, Su, Sv, r0, r1, xlo, xhi;
  int capm, capb, nchunks_total, nstrips, chunk_base;
  int affine, project;
  unsigned long long* sflag;   // singular-stretch word (fbw.cuh)
  double G00, G01, G10, G11, detJ;
  double mu1, mu2, mush, mubd;
  const int32_t* m_aoff;
  const int32_t* b_aoff;
  const uint2* m_info;     // (uc | vc << 16, shape | ou << 16)
  const uint2* b_info;
  const double* utab;      // [nu_cls][9]: N[3] dN[3] ddN[3]
  const double* vtab;      // [nv_cls][9]
  const double* stab;      // [nshape][2]: w (affine) , mask
  const double* m_geo;
  const double* b_geo;
  int64_t Mm, Bm;
  const int16_t* lut;
  const int4* tasks;
  const unsigned long long* ent;
  const int32_t* row_ptr;
  const int2* chunks;      // (ra, rb) per chunk of this launch
  const int2* work;        // frame mode: (strip, chunk of this launch) per CTA; nullptr = full grid
  int sk_i0, sk_i1, sk_j0, sk_j1;   // control points whose rows k_core writes (no gather here)
  int ex_i0, ex_i1, ex_j0, ex_j1;   // anchors whose energy k_core counts
  int64_t e_stride;        // energy partial slots per item
  const double* params;    // optional per-item [9]: G00 G01 G10 G11 detJ mu_st1 mu_st2 mu_sh mu_bd
  double detJ_ref;         // det J the class weights were built with
  int flags;
};

// point records in shared memory (array of structures, odd strides -> conflict-free 8-byte access)
constexpr int kMS = 45;    // membrane: [0,21) A~  [21,39) d_e (e*2 + mu)  [39,45) P~
constexpr int kBS = 13;    // bending:  [0,9) L^_e  [9,12) D^  [12] pad

__device__ __forceinline__ int wrap(int q, int cap) { return q >= cap ? q - cap : q; }

#ifdef BSF_PHASE_TIMERS
__device__ unsigned long long g_phase[16];
#endif

// Warp-cooperative store of one 3x3 block per lane: lanes 9k..9k+8 store block 3r+k of round r
// (72 contiguous bytes each); pos < 0 skips.  `transpose` selects H^T.
__device__ __forceinline__ void warp_store_block(double* wb, const double (&blk)[9], bool transpose, int pos,
                                                 double* vals, int lane) {
#pragma unroll
  for (int q = 0; q < 9; ++q) wb[lane * 9 + q] = transpose ? blk[3 * (q % 3) + q / 3] : blk[q];
  __syncwarp();
  const int sub = lane / 9, el = lane - sub * 9;
#pragma unroll
  for (int rr = 0; rr < 11; ++rr) {
    const int owner = min(3 * rr + sub, 31);
    const int po = __shfl_sync(0xffffffffu, pos, owner);
    if (lane < 27 && 3 * rr + sub < 32 && po >= 0) vals[(int64_t)po * 9 + el] = wb[owner * 9 + el];
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 2) k_tile(const TileArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BSF_POISON_SMEM(smem_raw);
  const int tid = threadIdx.x;
  int strip = blockIdx.x, cl = blockIdx.y;
  if (A.work) { const int2 w = A.work[blockIdx.x]; strip = w.x; cl = w.y; }
  const int chunk = A.chunk_base + cl, item = blockIdx.z;
  const int i0 = strip * kTX;
  const int2 chr = A.chunks[cl];
  const int ra = chr.x, rb = chr.y;
  const int slo = max(0, i0 - 2), shi = min(A.Su - 1, i0 + kTX - 1);
  const double* __restrict__ x = A.x + item * A.xs;

  // ---- shared memory carve-up
  double* pos = reinterpret_cast<double*>(smem_raw);                   // [kPosRows][kPosCols][3]
  double* pm = pos + kPosRows * kPosCols * 3;                          // [capm][kMS]
  double* pb = pm + (int64_t)kMS * A.capm;                             // [capb][kBS]
  double* wbuf = pb + (int64_t)kBS * A.capb;                           // [kThreads/32][288]
  double* red = wbuf + (kThreads / 32) * 288;                          // [32]
  int* astm = reinterpret_cast<int*>(red + 32);                        // [kRing][kAC]
  int* astb = astm + kRing * kAC;                                      // [kRing][kAC]

  const bool want_h = A.vals != nullptr, want_g = A.g != nullptr;
  double e_acc = 0.0;
  // affine geometry and stiffness of this batch item (per-item parameters for batches of sheets)
  double pG00 = A.G00, pG01 = A.G01, pG10 = A.G10, pG11 = A.G11, pdet = A.detJ;
  double pmu1 = A.mu1, pmu2 = A.mu2, pmush = A.mush, pmubd = A.mubd;
  if (A.params) {
    const double* pp = A.params + 9 * (int64_t)item;
    pG00 = pp[0]; pG01 = pp[1]; pG10 = pp[2]; pG11 = pp[3];
    pdet = pp[4] / A.detJ_ref;
    pmu1 = (A.flags & 2) ? 0.0 : pp[5];
    pmu2 = (A.flags & 2) ? 0.0 : pp[6];
    pmush = (A.flags & 2) ? 0.0 : pp[7];
    pmubd = (A.flags & 4) ? 0.0 : pp[8];
  }
  int head_m = 0, head_b = 0;

  for (int j0 = ra - 2; j0 < rb; j0 += kRS) {
#ifdef BSF_PHASE_TIMERS
    const long long T0 = clock64();
#endif
    // ---------------- 1. positions of cp rows j0 .. j0+kRS+1, cols i0-2 .. i0+kTX+1
    for (int k = tid; k < kPosRows * kPosCols * 3; k += kThreads) {
      const int row = k / (kPosCols * 3), rem = k - row * kPosCols * 3;
      const int col = rem / 3, c = rem - col * 3;
      const int R = j0 + row, Cc = i0 - 2 + col;
      double v = 0.0;
      if (R >= A.xlo && R < A.xhi && Cc >= 0 && Cc < A.n_u) v = x[((int64_t)(R - A.xlo) * A.n_u + Cc) * 3 + c];
      pos[k] = v;
    }
    // ---------------- 2. ring bookkeeping for anchor rows j0, j0+1 (uniform in every thread)
    int P0m[kRS], Nm[kRS], Hm[kRS], P0b[kRS], Nb[kRS], Hb[kRS];
#pragma unroll
    for (int r = 0; r < kRS; ++r) {
      const int t = j0 + r;
      const bool valid = (t >= 0 && t < A.Sv && slo <= shi);
      P0m[r] = valid ? A.m_aoff[t * A.Su + slo] : 0;
      Nm[r] = valid ? A.m_aoff[t * A.Su + shi + 1] - P0m[r] : 0;
      P0b[r] = valid ? A.b_aoff[t * A.Su + slo] : 0;
      Nb[r] = valid ? A.b_aoff[t * A.Su + shi + 1] - P0b[r] : 0;
      Hm[r] = head_m;
      Hb[r] = head_b;
      head_m = wrap(head_m + Nm[r], A.capm);   // Nm <= capm
      head_b = wrap(head_b + Nb[r], A.capb);
      if (tid < kAC) {
        const int s = i0 - 2 + tid, slot = (t + 4) & 3;
        int sm = 0, sb = 0;
        if (valid && s >= slo && s <= shi) {
          sm = wrap(Hm[r] + (A.m_aoff[t * A.Su + s] - P0m[r]), A.capm);
          sb = wrap(Hb[r] + (A.b_aoff[t * A.Su + s] - P0b[r]), A.capb);
        }
        astm[slot * kAC + tid] = sm;
        astb[slot * kAC + tid] = sb;
      }
    }
    __syncthreads();
#ifdef BSF_PHASE_TIMERS
    const long long T1 = clock64();
#endif
    // ---------------- 3. point phase
    const int nmem = Nm[0] + Nm[1], ntot = nmem + Nb[0] + Nb[1];
    for (int k = tid; k < ntot; k += kThreads) {
      if (k < nmem) {
        const int r = k < Nm[0] ? 0 : 1;
        const int kk = r ? k - Nm[0] : k;
        const int64_t p = P0m[r] + kk;
        double* rec = pm + (int64_t)kMS * wrap(Hm[r] + kk, A.capm);
        const int t = j0 + r;
        const uint2 info = A.m_info[p];
        const int ou = info.y >> 16;
        const double* tu = A.utab + (info.x & 0xFFFF) * 9;
        const double* tv = A.vtab + (info.x >> 16) * 9;
        const double* sh = A.stab + (info.y & 0xFFFF) * 2;
        double Nu[3], dNu[3], Nv[3], dNv[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) { Nu[q] = tu[q]; dNu[q] = tu[3 + q]; Nv[q] = tv[q]; dNv[q] = tv[3 + q]; }
        const int mask = (int)sh[1];
        // d_e = (dN/du, dN/dv) of window entry e (zero outside the structural stencil);
        // F~ = [dphi/du, dphi/dv] = sum_e C_e d_e^T
        double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0};
#pragma unroll
        for (int jv = 0; jv < 3; ++jv)
#pragma unroll
          for (int iu = 0; iu < 3; ++iu) {
            const int e = 3 * jv + iu;
            const bool in = (mask >> e) & 1;
            const double du = in ? dNu[iu] * Nv[jv] : 0.0, dv = in ? Nu[iu] * dNv[jv] : 0.0;
            rec[21 + 2 * e] = du;
            rec[22 + 2 * e] = dv;
            const double* C = pos + ((t + jv - j0) * kPosCols + (ou + iu - (i0 - 2))) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) { Fu[c] = fma(C[c], du, Fu[c]); Fv[c] = fma(C[c], dv, Fv[c]); }
          }
        double G00, G01, G10, G11, w;
        if (A.affine) { G00 = pG00; G01 = pG01; G10 = pG10; G11 = pG11; w = sh[0] * pdet; }
        else {
          G00 = A.m_geo[p]; G01 = A.m_geo[A.Mm + p]; G10 = A.m_geo[2 * A.Mm + p]; G11 = A.m_geo[3 * A.Mm + p];
          w = A.m_geo[4 * A.Mm + p];
        }
        double f1[3], f2[3];   // F_beta = sum_mu F~_mu G_mu,beta
#pragma unroll
        for (int c = 0; c < 3; ++c) { f1[c] = Fu[c] * G00 + Fv[c] * G10; f2[c] = Fu[c] * G01 + Fv[c] * G11; }
        FSpace o;
        fbw_point(f1, f2, pmu1, pmu2, pmush, A.project != 0, o);
        if (ou >= i0 && ou < i0 + kTX && t >= ra && t < rb &&
            !(ou >= A.ex_i0 && ou < A.ex_i1 && t >= A.ex_j0 && t < A.ex_j1)) {
          e_acc += w * o.psi;
          fbw_flag_singular(A.sflag, o.i5min, item, ou, t);
        }
        // P~_mu = w sum_beta G_mu,beta P_beta
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          rec[39 + c] = w * (G00 * o.P1[c] + G01 * o.P2[c]);
          rec[42 + c] = w * (G10 * o.P1[c] + G11 * o.P2[c]);
        }
        // A~_mu,nu = w sum_{beta,gamma} G_mu,beta G_nu,gamma A_beta,gamma
        const double a11 = w * G00 * G00, a12 = w * G00 * G01, a22 = w * G01 * G01;  // for mu=nu=u
        const double b11 = w * G10 * G10, b12 = w * G10 * G11, b22 = w * G11 * G11;  // mu=nu=v
        const double c11 = w * G00 * G10, c12 = w * G00 * G11, c21 = w * G01 * G10, c22 = w * G01 * G11;  // u,v
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
          for (int c3 = r3; c3 < 3; ++c3) {
            const int s6 = sym3(r3, c3);
            const double A11 = o.A11[s6], A22 = o.A22[s6];
            const double A12rc = o.A12[3 * r3 + c3], A12cr = o.A12[3 * c3 + r3];  // A21[r][c] = A12[c][r]
            rec[s6] = a11 * A11 + a12 * (A12rc + A12cr) + a22 * A22;
            rec[6 + s6] = b11 * A11 + b12 * (A12rc + A12cr) + b22 * A22;
          }
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
          for (int c3 = 0; c3 < 3; ++c3)
            rec[12 + 3 * r3 + c3] =
                c11 * o.A11[sym3(r3, c3)] + c12 * o.A12[3 * r3 + c3] + c21 * o.A12[3 * c3 + r3] + c22 * o.A22[sym3(r3, c3)];
      } else {
        const int kb = k - nmem;
        const int r = kb < Nb[0] ? 0 : 1;
        const int kk = r ? kb - Nb[0] : kb;
        const int64_t p = P0b[r] + kk;
        double* rec = pb + (int64_t)kBS * wrap(Hb[r] + kk, A.capb);
        const int t = j0 + r;
        const uint2 info = A.b_info[p];
        const int ou = info.y >> 16;
        const double* tu = A.utab + (info.x & 0xFFFF) * 9;
        const double* tv = A.vtab + (info.x >> 16) * 9;
        const double* sh = A.stab + (info.y & 0xFFFF) * 2;
        double cuu, cvv, cuv, cu, cv, w;
        if (A.affine) {
          cuu = pG00 * pG00 + pG01 * pG01;
          cvv = pG10 * pG10 + pG11 * pG11;
          cuv = 2.0 * (pG00 * pG10 + pG01 * pG11);
          cu = 0.0; cv = 0.0;
          w = sh[0] * pdet;
        } else {
          w = A.b_geo[p]; cuu = A.b_geo[A.Bm + p]; cvv = A.b_geo[2 * A.Bm + p]; cuv = A.b_geo[3 * A.Bm + p];
          cu = A.b_geo[4 * A.Bm + p]; cv = A.b_geo[5 * A.Bm + p];
        }
        const int mask = (int)sh[1];
        const double sw = sqrt(w * pmubd);
        double lap[3] = {0, 0, 0};
#pragma unroll
        for (int jv = 0; jv < 3; ++jv)
#pragma unroll
          for (int iu = 0; iu < 3; ++iu) {
            const int e = 3 * jv + iu;
            double L = 0.0;
            if ((mask >> e) & 1) {
              // Eq. `eq: Laplacian in parametric space`
              L = cuu * tu[6 + iu] * tv[jv] + cvv * tu[iu] * tv[6 + jv] + cuv * tu[3 + iu] * tv[3 + jv] +
                  cu * tu[3 + iu] * tv[jv] + cv * tu[iu] * tv[3 + jv];
              const double* C = pos + ((t + jv - j0) * kPosCols + (ou + iu - (i0 - 2))) * 3;
              lap[0] += L * C[0]; lap[1] += L * C[1]; lap[2] += L * C[2];
            }
            rec[e] = sw * L;
          }
        if (ou >= i0 && ou < i0 + kTX && t >= ra && t < rb &&
            !(ou >= A.ex_i0 && ou < A.ex_i1 && t >= A.ex_j0 && t < A.ex_j1))
          e_acc += 0.5 * w * pmubd * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]);
        rec[9] = sw * lap[0];
        rec[10] = sw * lap[1];
        rec[11] = sw * lap[2];
      }
    }
    __syncthreads();
    // prologue step (anchor rows ra-2, ra-1): no output, except the two halo rows above a slab whose
    // forward pairs reach into the first owned rows (transpose-only)
#ifdef BSF_PHASE_TIMERS
    const long long T2 = clock64();
    if (tid == 0) { atomicAdd(&g_phase[0], (unsigned long long)(T1 - T0)); atomicAdd(&g_phase[1], (unsigned long long)(T2 - T1)); }
#endif
    const bool halo_step = (j0 < ra);
    if (halo_step && !(ra == A.r0 && A.r0 > 0)) continue;
    // ---------------- 4. gather: symmetric forward tasks (b after a), both H_ab and H_ab^T written.
    // warps 0-1: group 0 (diagonal row) for control points 0-15 / 16-31 of the step, the entry list
    // split between lane halves; warps 2-5: groups 1-4; warp 6: gradient.
    {
      const int warp = tid >> 5, lane = tid & 31;
      const bool split = (warp < 2);
      const int cpi = split ? warp * 16 + (lane & 15) : lane;
      const int half = split ? (lane >> 4) : 0;
      const int task = split ? 0 : (warp < 6 ? warp - 1 : 5);
      const int r = cpi / kTX, c = cpi - r * kTX;
      const int i = i0 + c, j = j0 + r;
      const bool owned_row = (j >= A.r0);
      bool active = (i < A.n_u) && (j < rb) && (j >= 0) &&
                    !(i >= A.sk_i0 && i < A.sk_i1 && j >= A.sk_j0 && j < A.sk_j1);
      if (task == 0 || task == 5) active = active && owned_row;        // group 0 / gradient: owned rows only
      active = active && ((task < 5) ? want_h : want_g);
      const int anchor_min = max(0, ra - 2);
      int4 h0 = make_int4(0, 0, 0, 0), h1 = make_int4(0, 0, 0, 0);
      int a_loc = 0;
      if (active) {
        const int pid = A.lut[(bclass(i, A.n_u) * kNCls + bclass(j, A.n_v)) * 2 + ((i + j) & 1)];
        h0 = A.tasks[(pid * kTasks + task) * 2];
        h1 = A.tasks[(pid * kTasks + task) * 2 + 1];
        a_loc = (j - A.r0) * A.n_u + i;
      }
      const int n_m = active ? (h0.y & 0xFFFF) : 0, n_b = active ? (h0.y >> 16) : 0;
      const int nmax_m = __reduce_max_sync(0xffffffffu, n_m), nmax_b = __reduce_max_sync(0xffffffffu, n_b);
      const unsigned long long* ent = A.ent + h0.x;
      if (task < 5) {
        double acc0[9], acc1[9], acc2[9];
        double dg0 = 0.0, dg1 = 0.0, dg2 = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) { acc0[q] = 0.0; acc1[q] = 0.0; acc2[q] = 0.0; }
        const int estep = split ? 2 : 1;
        unsigned long long Ea = (half < n_m) ? __ldg(ent + half) : 0ull;
        unsigned long long Eb = (half + estep < n_m) ? __ldg(ent + half + estep) : 0ull;
        for (int e = half; e < nmax_m; e += estep) {
          const unsigned long long E = Ea;
          Ea = Eb;
          Eb = (e + 2 * estep < n_m) ? __ldg(ent + e + 2 * estep) : 0ull;
          if (e < n_m) {
            const int dt = E & 3, dc = (E >> 2) & 3, idx = (E >> 5) & 15, la = (E >> 9) & 15;
            const int t = j - 2 + dt;
            if (t >= anchor_min) {
              const double* rec = pm + kMS * wrap(astm[((t + 4) & 3) * kAC + c + dc] + idx, A.capm);
              const double da1 = rec[21 + 2 * la], da2 = rec[22 + 2 * la];
              double Am[21];
#pragma unroll
              for (int k = 0; k < 21; ++k) Am[k] = rec[k];
              const int lb0 = (E >> 13) & 15, lb1 = (E >> 17) & 15, lb2 = (E >> 21) & 15;
              // contributions to the task's <= 3 blocks; a missing block (lb == 15) reads entry 0 and
              // gets zero coefficients (branch-free body)
#define BSF_BLOCK(ACC, LB)                                                                          \
  {                                                                                                 \
    const bool ok = (LB) != 15;                                                                     \
    const int l2 = ok ? (LB) : 0;                                                                   \
    const double db1 = ok ? rec[21 + 2 * l2] : 0.0, db2 = ok ? rec[22 + 2 * l2] : 0.0;              \
    const double k11 = da1 * db1, k22 = da2 * db2, k12 = da1 * db2, k21 = da2 * db1;                \
    _Pragma("unroll") for (int r3 = 0; r3 < 3; ++r3)                                                \
    _Pragma("unroll") for (int c3 = 0; c3 < 3; ++c3) {                                              \
      double v = ACC[3 * r3 + c3];                                                                  \
      v = fma(k11, Am[sym3(r3, c3)], v);                                                            \
      v = fma(k22, Am[6 + sym3(r3, c3)], v);                                                        \
      v = fma(k12, Am[12 + 3 * r3 + c3], v);                                                        \
      v = fma(k21, Am[12 + 3 * c3 + r3], v);                                                        \
      ACC[3 * r3 + c3] = v;                                                                         \
    }                                                                                               \
  }
              BSF_BLOCK(acc0, lb0)
              BSF_BLOCK(acc1, lb1)
              BSF_BLOCK(acc2, lb2)
#undef BSF_BLOCK
            }
          }
        }
        const unsigned long long* entb = ent + n_m;
        for (int e = half; e < nmax_b; e += estep) {
          if (e < n_b) {
            const unsigned long long E = __ldg(entb + e);
            const int dt = E & 3, dc = (E >> 2) & 3, idx = (E >> 5) & 15, la = (E >> 9) & 15;
            const int t = j - 2 + dt;
            if (t >= anchor_min) {
              const double* rec = pb + kBS * wrap(astb[((t + 4) & 3) * kAC + c + dc] + idx, A.capb);
              const double La = rec[la];
              const int lb0 = (E >> 13) & 15, lb1 = (E >> 17) & 15, lb2 = (E >> 21) & 15;
              dg0 = fma(La, lb0 != 15 ? rec[lb0 != 15 ? lb0 : 0] : 0.0, dg0);
              dg1 = fma(La, lb1 != 15 ? rec[lb1 != 15 ? lb1 : 0] : 0.0, dg1);
              dg2 = fma(La, lb2 != 15 ? rec[lb2 != 15 ? lb2 : 0] : 0.0, dg2);
            }
          }
        }
        acc0[0] += dg0; acc0[4] += dg0; acc0[8] += dg0;
        acc1[0] += dg1; acc1[4] += dg1; acc1[8] += dg1;
        acc2[0] += dg2; acc2[4] += dg2; acc2[8] += dg2;
        if (split) {   // combine the two lane halves (same control point, complementary entries)
#pragma unroll
          for (int q = 0; q < 9; ++q) {
            acc0[q] += __shfl_xor_sync(0xffffffffu, acc0[q], 16);
            acc1[q] += __shfl_xor_sync(0xffffffffu, acc1[q], 16);
            acc2[q] += __shfl_xor_sync(0xffffffffu, acc2[q], 16);
          }
        }
        // ---- warp-cooperative writes (72-byte blocks).  Split warps: the lower half stores H_ab, the
        // upper half H_ab^T of the same block in one pass.
        const int nb = active ? (h0.z & 0xF) : 0;
        const int nbmax = __reduce_max_sync(0xffffffffu, nb);
        double* wb = wbuf + warp * 288;
        double* vals = A.vals + item * A.vs;
        const int rpa = (active && owned_row) ? A.row_ptr[a_loc] : 0;
#define BSF_OUT(M, ACC)                                                                             \
  if ((M) < nbmax) {                                                                                \
    const int kab = (h1.x >> (8 * (M))) & 0xFF, kba = (h1.y >> (8 * (M))) & 0xFF;                   \
    const int dpk = (h1.z >> (5 * (M))) & 31, di = (dpk & 7) - 2, dj = dpk >> 3;                    \
    const bool mv = ((M) < nb);                                                                     \
    const int jb = j + dj;                                                                          \
    const int pf = (mv && owned_row) ? rpa + kab : -1;                                              \
    int pt = -1;                                                                                    \
    if (mv && !(di == 0 && dj == 0) && jb >= A.r0 && jb < A.r1) pt = A.row_ptr[a_loc + di + dj * A.n_u] + kba; \
    if (split) {                                                                                    \
      warp_store_block(wb, ACC, half == 1, half ? pt : pf, vals, lane);                             \
    } else {                                                                                        \
      warp_store_block(wb, ACC, false, pf, vals, lane);                                             \
      warp_store_block(wb, ACC, true, pt, vals, lane);                                              \
    }                                                                                               \
  }
        BSF_OUT(0, acc0)
        BSF_OUT(1, acc1)
        BSF_OUT(2, acc2)
#undef BSF_OUT
      } else {
        double g0 = 0.0, g1 = 0.0, g2 = 0.0;
        for (int e = 0; e < nmax_m; ++e) {
          if (e < n_m) {
            const unsigned long long E = __ldg(ent + e);
            const int dt = E & 3, dc = (E >> 2) & 3, idx = (E >> 5) & 15, la = (E >> 9) & 15;
            const int t = j - 2 + dt;
            const double* rec = pm + kMS * wrap(astm[((t + 4) & 3) * kAC + c + dc] + idx, A.capm);
            const double da1 = rec[21 + 2 * la], da2 = rec[22 + 2 * la];
            g0 = fma(da1, rec[39], fma(da2, rec[42], g0));
            g1 = fma(da1, rec[40], fma(da2, rec[43], g1));
            g2 = fma(da1, rec[41], fma(da2, rec[44], g2));
          }
        }
        const unsigned long long* entb = ent + n_m;
        for (int e = 0; e < nmax_b; ++e) {
          if (e < n_b) {
            const unsigned long long E = __ldg(entb + e);
            const int dt = E & 3, dc = (E >> 2) & 3, idx = (E >> 5) & 15, la = (E >> 9) & 15;
            const int t = j - 2 + dt;
            const double* rec = pb + kBS * wrap(astb[((t + 4) & 3) * kAC + c + dc] + idx, A.capb);
            const double La = rec[la];
            g0 = fma(La, rec[9], g0);
            g1 = fma(La, rec[10], g1);
            g2 = fma(La, rec[11], g2);
          }
        }
        if (active) {
          double* gd = A.g + item * A.gs + 3 * (int64_t)a_loc;
          gd[0] = g0; gd[1] = g1; gd[2] = g2;
        }
      }
    }
#ifdef BSF_PHASE_TIMERS
    {
      const long long T3 = clock64();
      if ((tid & 31) == 0) atomicAdd(&g_phase[2 + (tid >> 5)], (unsigned long long)(T3 - T2));
      __syncthreads();
      if (tid == 0) { atomicAdd(&g_phase[9], (unsigned long long)(clock64() - T2)); atomicAdd(&g_phase[10], 1ull); }
    }
#endif
    __syncthreads();
  }
  // ---------------- energy partial of this CTA (fixed-order tree)
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    A.epart[(int64_t)item * A.e_stride + (int64_t)chunk * A.nstrips + strip] = s;
  }
}

__global__ void __launch_bounds__(256) k_energy_final(const double* __restrict__ epart, int per_item, double* E) {
  __shared__ double sm[8];
  const double* p = epart + (int64_t)blockIdx.x * per_item;
  double s = 0.0;
  for (int k = threadIdx.x; k < per_item; k += blockDim.x) s += p[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
    E[blockIdx.x] = t;
  }
}

// ------------------------------------------------------------------ host side
template <class T>
bool upload(const std::function<void*(size_t)>& dalloc, T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return true;
  void* p = dalloc(v.size() * sizeof(T));
  if (!p) return false;
  if (cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  *dst = static_cast<T*>(p);
  return true;
}

}  // namespace

int build_tiles(const Sheet& sh, TileTables& tt, std::string& err, const std::function<void*(size_t)>& dalloc) {
  tt = TileTables();
  const int Su = sh.Su, Sv = sh.Sv, nu = sh.n_u;
  tt.n_u = nu; tt.n_v = sh.n_v; tt.Su = Su; tt.Sv = Sv; tt.r0 = sh.r0; tt.r1 = sh.r1; tt.xlo = sh.xlo;
  const int nanch = Su * Sv;
  // ---- sort points by anchor (stable)
  auto sort_by_anchor = [&](const std::vector<Point>& P, std::vector<int32_t>& aoff, std::vector<int>& order) {
    aoff.assign(nanch + 1, 0);
    for (const Point& p : P) ++aoff[p.ov * Su + p.ou + 1];
    for (int a = 0; a < nanch; ++a) aoff[a + 1] += aoff[a];
    order.assign(P.size(), 0);
    std::vector<int32_t> fill(aoff.begin(), aoff.end() - 1);
    for (size_t k = 0; k < P.size(); ++k) order[fill[P[k].ov * Su + P[k].ou]++] = (int)k;
    int mx = 0;
    for (int a = 0; a < nanch; ++a) mx = std::max(mx, aoff[a + 1] - aoff[a]);
    return mx;
  };
  std::vector<int32_t> m_aoff, b_aoff;
  std::vector<int> m_ord, b_ord;
  if (sort_by_anchor(sh.mem, m_aoff, m_ord) > 15 || sort_by_anchor(sh.bend, b_aoff, b_ord) > 15) return 1;
  // ---- basis tables, keyed by their exact bits: one table per distinct 1D evaluation (x - span is
  // the same double for every span of a binade, so the tables stay few), plus a small "shape" table
  // (weight for the affine case, stencil mask).  No rounding of any coefficient.
  const double detJ_ref = sh.mem.empty() ? (sh.bend.empty() ? 1.0 : sh.bend[0].detJ) : sh.mem[0].detJ;
  std::map<std::vector<double>, int> ucls, vcls, scls;
  std::vector<double> utab, vtab, stab;
  auto intern = [](std::map<std::vector<double>, int>& M, std::vector<double>& tab, std::vector<double> key) {
    auto it = M.find(key);
    if (it != M.end()) return it->second;
    const int id = (int)M.size();
    M.emplace(key, id);
    tab.insert(tab.end(), key.begin(), key.end());
    return id;
  };
  auto b9 = [](const Basis1& b) {
    std::vector<double> k(b.N, b.N + 3);
    k.insert(k.end(), b.d1, b.d1 + 3);
    k.insert(k.end(), b.d2, b.d2 + 3);
    return k;
  };
  std::vector<uint2> m_info(sh.mem.size()), b_info(sh.bend.size());
  for (int kind = 0; kind < 2; ++kind) {
    const std::vector<Point>& P = kind ? sh.bend : sh.mem;
    const std::vector<int>& ord = kind ? b_ord : m_ord;
    std::vector<uint2>& info = kind ? b_info : m_info;
    for (size_t k = 0; k < ord.size(); ++k) {
      const Point& p = P[ord[k]];
      const int uc = intern(ucls, utab, b9(p.bu)), vc = intern(vcls, vtab, b9(p.bv));
      const int sc = intern(scls, stab, {sh.affine ? p.what * detJ_ref : 0.0, (double)p.mask});
      info[k] = make_uint2((uint32_t)uc | ((uint32_t)vc << 16), (uint32_t)sc | ((uint32_t)p.ou << 16));
    }
  }
  if (ucls.size() > 65535 || vcls.size() > 65535 || scls.size() > 65535 || nu > 65535) return 1;
  // affine: the kernel multiplies the class weight by detJ; classes already hold w, so detJ = 1
  tt.affine = sh.affine ? 1 : 0;
  if (sh.affine) {
    const Point& ref = sh.mem.empty() ? sh.bend[0] : sh.mem[0];
    tt.G[0] = ref.G[0][0]; tt.G[1] = ref.G[0][1]; tt.G[2] = ref.G[1][0]; tt.G[3] = ref.G[1][1];
    tt.detJ = 1.0;
  }
  tt.detJ_ref = detJ_ref;
  std::vector<double> m_geo, b_geo;
  if (!sh.affine) {
    const size_t M = sh.mem.size(), B = sh.bend.size();
    m_geo.resize(5 * M);
    b_geo.resize(6 * B);
    for (size_t k = 0; k < M; ++k) {
      const Point& p = sh.mem[m_ord[k]];
      m_geo[k] = p.G[0][0]; m_geo[M + k] = p.G[0][1]; m_geo[2 * M + k] = p.G[1][0]; m_geo[3 * M + k] = p.G[1][1];
      m_geo[4 * M + k] = p.w;
    }
    for (size_t k = 0; k < B; ++k) {
      const Point& p = sh.bend[b_ord[k]];
      b_geo[k] = p.w; b_geo[B + k] = p.c_uu; b_geo[2 * B + k] = p.c_vv; b_geo[3 * B + k] = p.c_uv;
      b_geo[4 * B + k] = p.c_u; b_geo[5 * B + k] = p.c_v;
    }
  }
  // ---- strips and row chunks.  Chunks whose anchor ring can hold the heavy boundary anchor rows
  // (t = 0: side spans, t = Sv-1: side spans + knot half cells) form a separate launch with a larger
  // point pool; interior chunks keep the pool small so two CTAs fit on an SM.
  tt.nstrips = (nu + kTX - 1) / kTX;
  std::vector<int> cm(Sv, 0), cb(Sv, 0);   // max points per anchor row over strips
  for (int st = 0; st < tt.nstrips; ++st) {
    const int i0 = st * kTX, slo = std::max(0, i0 - 2), shi = std::min(Su - 1, i0 + kTX - 1);
    if (slo > shi) continue;
    for (int t = 0; t < Sv; ++t) {
      cm[t] = std::max(cm[t], m_aoff[t * Su + shi + 1] - m_aoff[t * Su + slo]);
      cb[t] = std::max(cb[t], b_aoff[t * Su + shi + 1] - b_aoff[t * Su + slo]);
    }
  }
  auto ring_need = [&](int ra, int rb, int& pm_, int& pb_) {   // pool need of one chunk
    pm_ = 1; pb_ = 1;
    for (int j0 = ra - 2; j0 < rb; j0 += kRS) {
      int sm = 0, sb = 0;
      for (int t = j0 - 2; t <= j0 + 1; ++t)
        if (t >= 0 && t < Sv) { sm += cm[t]; sb += cb[t]; }
      pm_ = std::max(pm_, sm);
      pb_ = std::max(pb_, sb);
    }
  };
  std::vector<int2> cl[2];   // 0 interior, 1 boundary
  {
    const int r0 = sh.r0, r1 = sh.r1;
    std::vector<int> cuts{r0};
    const int lo_edge = std::min(r1, std::max(r0, 6)), hi_edge = std::max(lo_edge, std::min(r1, Sv - 4));
    if (lo_edge > r0) cuts.push_back(lo_edge);
    const int span = hi_edge - lo_edge;
    if (span > 0) {
      const int n = (span + 31) / 32;
      for (int k = 1; k < n; ++k) cuts.push_back(lo_edge + ((span * k / n) & ~1));
      cuts.push_back(hi_edge);
    }
    if (r1 > cuts.back()) cuts.push_back(r1);
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
      if (cuts[k + 1] <= cuts[k]) continue;
      int pm_, pb_;
      ring_need(cuts[k], cuts[k + 1], pm_, pb_);
      const bool heavy = (cuts[k] - 4 <= 0) || (cuts[k + 1] + 1 >= Sv - 1);
      cl[heavy ? 1 : 0].push_back(make_int2(cuts[k], cuts[k + 1]));
    }
  }
  tt.nchunks = (int)(cl[0].size() + cl[1].size());
  for (int L = 0; L < 2; ++L) {
    int capm = 1, capb = 1;
    for (const int2& ch : cl[L]) {
      int pm_, pb_;
      ring_need(ch.x, ch.y, pm_, pb_);
      capm = std::max(capm, pm_);
      capb = std::max(capb, pb_);
    }
    tt.capm_l[L] = capm;
    tt.capb_l[L] = capb;
    tt.nch_l[L] = (int)cl[L].size();
    tt.smem_l[L] = sizeof(double) * (kPosRows * kPosCols * 3 + (size_t)kMS * capm + (size_t)kBS * capb +
                                     (kThreads / 32) * 288 + 32) +
                   sizeof(int) * (2 * kRing * kAC);
    if (!cl[L].empty() && tt.smem_l[L] > 227 * 1024) return 1;
  }
  std::vector<int2> chunks(cl[0]);
  chunks.insert(chunks.end(), cl[1].begin(), cl[1].end());
  // ---- gather programs: one per (boundary class u, boundary class v, parity).  Forward blocks of a
  // control point a = (i, j): b = (i+di, j+dj) after a in storage order, split into 5 tasks of <= 3
  // blocks: T0 dj=0 di 0..2 | T1a dj=1 di -2..0 | T1b dj=1 di 1..2 | T2a dj=2 di -2..-1 | T2b dj=2 di 0..2.
  // Task 5 gathers the gradient.  Block ranks come from the structural pattern of ANY row (also rows
  // outside the slab), so one program serves every control point of its class.
  static const int grp_n[5] = {3, 3, 3, 3, 1};
  static const int grp_off[5][3][2] = {{{0, 0}, {1, 0}, {2, 0}},
                                       {{-2, 1}, {-1, 1}, {0, 1}},
                                       {{1, 1}, {2, 1}, {-2, 2}},
                                       {{-1, 2}, {0, 2}, {1, 2}},
                                       {{2, 2}, {0, 0}, {0, 0}}};
  struct SPt { int ou, ov; uint16_t mask; };
  std::vector<SPt> spts;
  std::vector<int32_t> s_aoff(nanch + 1, 0);
  {
    std::vector<RulePoint> rp;
    std::vector<SPt> tmp;
    for (int kind = 0; kind < 2; ++kind) {
      make_rule(kind ? sh.brule : sh.mrule, kind == 1, Su, Sv, rp);
      for (const RulePoint& q : rp) {
        const int ou = std::min((int)std::floor(q.u), Su - 1), ov = std::min((int)std::floor(q.v), Sv - 1);
        tmp.push_back({ou, ov, stencil_mask(kind == 1, q.knot_u, q.knot_v)});
      }
    }
    for (const SPt& p : tmp) ++s_aoff[p.ov * Su + p.ou + 1];
    for (int a = 0; a < nanch; ++a) s_aoff[a + 1] += s_aoff[a];
    spts.resize(tmp.size());
    std::vector<int32_t> fill(s_aoff.begin(), s_aoff.end() - 1);
    for (const SPt& p : tmp) spts[fill[p.ov * Su + p.ou]++] = p;
  }
  auto row_cols = [&](int i, int j) {   // structural column list of block row (i, j), global indices
    std::vector<int> cols{j * nu + i};
    for (int t = std::max(0, j - 2); t <= std::min(Sv - 1, j); ++t)
      for (int s2 = std::max(0, i - 2); s2 <= std::min(Su - 1, i); ++s2)
        for (int k = s_aoff[t * Su + s2]; k < s_aoff[t * Su + s2 + 1]; ++k) {
          const SPt& p = spts[k];
          const int la = (i - s2) + 3 * (j - t);
          if (!((p.mask >> la) & 1)) continue;
          for (int e = 0; e < 9; ++e)
            if ((p.mask >> e) & 1) cols.push_back((t + e / 3) * nu + s2 + e % 3);
        }
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    return cols;
  };
  std::vector<int16_t> lut(kNCls * kNCls * 2, -1);
  std::vector<int4> tasks;
  std::vector<unsigned long long> ents;
  auto build_prog = [&](int i, int j) {
    const std::vector<int> ca = row_cols(i, j);
    const int a = j * nu + i;
    int nb[5], kab[5][3], kba[5][3], dpk[5][3], bcol[5][3];
    for (int tk = 0; tk < 5; ++tk) {
      nb[tk] = 0;
      for (int g = 0; g < grp_n[tk]; ++g) {
        const int di = grp_off[tk][g][0], dj = grp_off[tk][g][1];
        if (i + di < 0 || i + di >= nu || j + dj >= sh.n_v) continue;
        const int b = (j + dj) * nu + i + di;
        const int k = (int)(std::lower_bound(ca.begin(), ca.end(), b) - ca.begin());
        if (k >= (int)ca.size() || ca[k] != b) continue;
        const std::vector<int> cb = row_cols(b % nu, b / nu);
        const int kb = (int)(std::lower_bound(cb.begin(), cb.end(), a) - cb.begin());
        if (kb >= (int)cb.size() || cb[kb] != a || k > 255 || kb > 255) return false;
        kab[tk][nb[tk]] = k;
        kba[tk][nb[tk]] = kb;
        dpk[tk][nb[tk]] = (di + 2) | (dj << 3);
        bcol[tk][nb[tk]] = b;
        ++nb[tk];
      }
    }
    {   // every forward block of the row must belong to a group
      int fwd = 0, tot = 0;
      for (int b : ca) if (b > a) ++fwd;
      for (int tk = 0; tk < 5; ++tk) tot += nb[tk];
      if (tot != fwd + 1) return false;
    }
    std::vector<unsigned long long> lists[kTasks][2];
    for (int kind = 0; kind < 2; ++kind) {
      const std::vector<int32_t>& aoff = kind ? b_aoff : m_aoff;
      const std::vector<int>& ord = kind ? b_ord : m_ord;
      const std::vector<Point>& P = kind ? sh.bend : sh.mem;
      for (int dt = 0; dt < 3; ++dt)
        for (int dc = 0; dc < 3; ++dc) {
          const int t = j - 2 + dt, s2 = i - 2 + dc;
          if (t < 0 || t >= Sv || s2 < 0 || s2 >= Su) continue;
          const int an = t * Su + s2;
          const int npts = aoff[an + 1] - aoff[an];
          for (int idx = 0; idx < npts; ++idx) {
            const Point& p = P[ord[aoff[an] + idx]];
            const int la = (i - s2) + 3 * (j - t);
            if (!((p.mask >> la) & 1)) continue;
            const unsigned long long base = (unsigned long long)dt | ((unsigned long long)dc << 2) |
                                            ((unsigned long long)kind << 4) | ((unsigned long long)idx << 5) |
                                            ((unsigned long long)la << 9);
            lists[5][kind].push_back(base | (0xFFFull << 13));
            for (int tk = 0; tk < 5; ++tk) {
              unsigned long long lbs = 0;
              bool any = false;
              for (int m = 0; m < 3; ++m) {
                unsigned long long lb = 15;
                if (m < nb[tk]) {
                  const int b = bcol[tk][m], ib = b % nu - s2, jb = b / nu - t;
                  if (ib >= 0 && ib < 3 && jb >= 0 && jb < 3 && ((p.mask >> (ib + 3 * jb)) & 1)) {
                    lb = (unsigned long long)(ib + 3 * jb);
                    any = true;
                  }
                }
                lbs |= lb << (4 * m);
              }
              if (any) lists[tk][kind].push_back(base | (lbs << 13));
            }
          }
        }
    }
    for (int tk = 0; tk < kTasks; ++tk) {
      int4 h0, h1;
      h0.x = (int)ents.size();
      h0.y = (int)lists[tk][0].size() | ((int)lists[tk][1].size() << 16);
      h0.z = tk < 5 ? nb[tk] : 0;
      h0.w = 0;
      h1 = make_int4(0, 0, 0, 0);
      if (tk < 5)
        for (int m = 0; m < nb[tk]; ++m) {
          h1.x |= kab[tk][m] << (8 * m);
          h1.y |= kba[tk][m] << (8 * m);
          h1.z |= dpk[tk][m] << (5 * m);
        }
      ents.insert(ents.end(), lists[tk][0].begin(), lists[tk][0].end());
      ents.insert(ents.end(), lists[tk][1].begin(), lists[tk][1].end());
      tasks.push_back(h0);
      tasks.push_back(h1);
    }
    return true;
  };
  // representatives: owned rows first (their anchor windows lie inside the slab's point list, so
  // their programs are complete); the two halo rows above a slab only add classes not seen yet
  // (entries below the slab window are skipped at run time anyway)
  int nprog = 0;
  std::vector<int> rows;
  for (int j = sh.r0; j < sh.r1; ++j) rows.push_back(j);
  for (int j = std::max(0, sh.r0 - 2); j < sh.r0; ++j) rows.push_back(j);
  for (int j : rows) {
    const int cv = bclass(j, sh.n_v);
    for (int i = 0; i < nu; ++i) {
      const int key = (bclass(i, nu) * kNCls + cv) * 2 + ((i + j) & 1);
      if (lut[key] >= 0) continue;
      lut[key] = (int16_t)nprog++;
      if (!build_prog(i, j)) return 1;
    }
  }
  // consistency: the structural pattern equals the slab's pattern on every owned row
  for (int j = sh.r0; j < sh.r1; j += std::max(1, (sh.r1 - sh.r0) / 7))
    for (int i = 0; i < nu; i += std::max(1, nu / 7)) {
      const std::vector<int> c = row_cols(i, j);
      const int64_t al = (int64_t)(j - sh.r0) * nu + i;
      if ((int)c.size() != sh.row_ptr[al + 1] - sh.row_ptr[al] ||
          !std::equal(c.begin(), c.end(), sh.col_idx.begin() + sh.row_ptr[al])) {
        err = "internal: structural pattern mismatch";
        return -1;
      }
    }
  // ---- upload
  std::vector<int32_t> rp(sh.row_ptr.begin(), sh.row_ptr.end());
  bool ok = upload(dalloc, &tt.m_aoff, m_aoff) && upload(dalloc, &tt.b_aoff, b_aoff) &&
            upload(dalloc, &tt.m_info, m_info) && upload(dalloc, &tt.b_info, b_info) &&
            upload(dalloc, &tt.utab, utab) && upload(dalloc, &tt.vtab, vtab) && upload(dalloc, &tt.stab, stab) &&
            upload(dalloc, &tt.m_geo, m_geo) && upload(dalloc, &tt.b_geo, b_geo) && upload(dalloc, &tt.lut, lut) &&
            upload(dalloc, &tt.tasks, tasks) && upload(dalloc, &tt.ent, ents) && upload(dalloc, &tt.row_ptr, rp) &&
            upload(dalloc, &tt.chunks, chunks);
  if (!ok) { err = "tile tables: device allocation failed"; return -7; }
  const size_t smax = std::max(tt.smem_l[0], tt.smem_l[1]);
  if (cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  tt.ok = 1;
  return 0;
}

int tile_set_core(TileTables& tt, const Sheet& sh, const CoreTables& ct, const std::function<void*(size_t)>& dalloc) {
  // rows k_core writes completely: every control point of its rectangle; the tile kernel still
  // processes those whose forward blocks reach owned frame rows (their transposes live there)
  tt.sk[0] = ct.CI0 + 2;
  tt.sk[1] = ct.CI1 - 2;
  tt.sk[2] = ct.RJ0;
  tt.sk[3] = (ct.RJ1 == sh.r1) ? sh.r1 : ct.RJ1 - 2;
  tt.ex[0] = ct.CI0; tt.ex[1] = ct.CI1; tt.ex[2] = ct.RJ0; tt.ex[3] = ct.RJ1;
  std::vector<int2> chunks(tt.nchunks);
  if (cudaMemcpy(chunks.data(), tt.chunks, sizeof(int2) * tt.nchunks, cudaMemcpyDeviceToHost) != cudaSuccess) return -6;
  int base = 0;
  for (int L = 0; L < 2; ++L) {
    std::vector<int2> work;
    for (int c = 0; c < tt.nch_l[L]; ++c) {
      const int2 ch = chunks[base + c];
      for (int st = 0; st < tt.nstrips; ++st) {
        const int i0 = st * kTX, i1 = std::min(tt.n_u, i0 + kTX);
        bool need = false;
        for (int j = ch.x; j < ch.y && !need; ++j)
          for (int i = i0; i < i1 && !need; ++i) {
            const bool skipped = i >= tt.sk[0] && i < tt.sk[1] && j >= tt.sk[2] && j < tt.sk[3];
            const bool anchor = i < tt.Su && j < tt.Sv;
            const bool excl = i >= tt.ex[0] && i < tt.ex[1] && j >= tt.ex[2] && j < tt.ex[3];
            if (!skipped || (anchor && !excl)) need = true;
          }
        if (need) work.push_back(make_int2(st, c));
      }
    }
    tt.nwork_l[L] = (int)work.size();
    if (!work.empty() && !upload(dalloc, &tt.work_l[L], work)) return -7;
    base += tt.nch_l[L];
  }
  tt.core = 1;
  return 0;
}

int tile_eval(TileTables& tt, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_E, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride,
              cudaStream_t st, int* launches, const std::function<void*(size_t)>& dalloc, const double* d_params,
              const CoreTables* ct, const FrameTables* ft, const IpFused* ip, const HaloOverlap* halo) {
  const bool core = ct && tt.core && ct->ok;
  if (ip && !(core && ft && ft->ok)) return -1;   // the fused incremental potential needs core + band + corners
  if (core && ft && ft->ok) {
    // frame kernel (full frame rows) + core kernel (full core rows): disjoint rows, one energy array
    // [item][frame tiles | core CTAs]; every slot is written on every call
    // halo overlap: the interior core rows [ja, jb) first (own chunking), then the two boundary row
    // ranges with one chunk each; energy slots [frame tiles | band CTAs | core CTAs of each launch]
    const bool ov = halo && halo->jb > halo->ja && halo->ja >= ct->RJ0 && halo->jb <= ct->RJ1;
    // SMs held by the band (2 CTAs per SM) and corner kernels running beside k_core
    const int reserved = (int)std::min<int64_t>(1 << 20, ((int64_t)ft->band.nctas * nbatch + 1) / 2 +
                                                            (int64_t)ft->ntiles * nbatch);
    const int core_nch = ov ? core_pick_chunks(*ct, nbatch, halo->jb - halo->ja, reserved)
                            : core_pick_chunks(*ct, nbatch, -1, reserved);
    if (getenv("BSF_DEBUG_CHUNKS"))
      fprintf(stderr, "chunks: band %d ctas, frame %d tiles, reserved %d, core rows %d strips %d nch %d\n",
              (int)ft->band.nctas, (int)ft->ntiles, reserved, ct->RJ1 - ct->RJ0, ct->nstrips, core_nch);
    const int64_t nfb = ft->ntiles + ft->band.nctas;   // energy slots: [frame tiles | band CTAs | core CTAs]
    const int64_t nb_lo = (ov && halo->ja > ct->RJ0) ? core_ctas_per_item(*ct, 1) : 0;   // boundary launches
    const int64_t nb_hi = (ov && halo->jb < ct->RJ1) ? core_ctas_per_item(*ct, 1) : 0;
    const int64_t e_stride = nfb + core_ctas_per_item(*ct, core_nch) + nb_lo + nb_hi;
    const int64_t need = (int64_t)nbatch * e_stride;
    if (need > tt.e_cap) {
      void* p = dalloc(need * sizeof(double));
      if (!p) return -7;
      tt.e_part = static_cast<double*>(p);
      tt.e_cap = need;
    }
    // fused energy reduction: the last CTA of the call's core / band / corner kernels writes each item's energy
    // (no separate reduction launch after the join); its counters are zeroed first on the caller's stream
    if (d_E && nbatch > tt.e_cnt_cap) {
      void* p = dalloc(sizeof(unsigned) * (size_t)nbatch);
      if (!p) return -7;
      tt.e_cnt = static_cast<unsigned*>(p);
      tt.e_cnt_cap = nbatch;
    }
    if (d_E && cudaMemsetAsync(tt.e_cnt, 0, sizeof(unsigned) * (size_t)nbatch, st) != cudaSuccess) return -6;
    struct EfScope {   // the launch functions below read call_efinal(); reset on every exit path
      explicit EfScope(const EFinal& e) { call_efinal() = e; }
      ~EfScope() { call_efinal() = EFinal(); }
    } ef_scope(d_E ? EFinal{tt.e_cnt, d_E, (int)e_stride, (int)e_stride} : EFinal());
    // the two kernels write disjoint rows: the frame runs on a side stream forked from / joined to st
    // (event fork-join, CUDA-graph capturable)
    if (!tt.side) {
      if (cudaStreamCreateWithFlags(&tt.side, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamCreateWithFlags(&tt.side2, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&tt.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&tt.ev_join, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&tt.ev_join2, cudaEventDisableTiming) != cudaSuccess)
        return -6;
    }
    int rc = 0;
    if (ov) {   // interior rows while the halo is in flight, then wait for it
      rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.e_part, e_stride,
                     nfb, core_nch, d_params, tt.detJ_ref, st, ip, halo->ja, halo->jb);
      if (rc) return rc;
      if (cudaStreamWaitEvent(st, halo->ready, 0) != cudaSuccess) return -6;
    }
    // corners (k_frame) and bands (k_band) run beside the core on side streams.  Small problems (a few core
    // strips: one C2 / C3 sheet) put them on two streams, since the three kernels have similar latencies;
    // large ones queue the corners before the bands on one stream (fewer SMs held back from k_core at its start)
    // (row slabs of a multi-GPU split count as small: their corner and band kernels are a large share of the slab;
    // C4 at N = 8, edge slab of 96 rows: 96 -> 85 us)
    static const int side_mode = getenv("BSF_SIDE_STREAMS") ? atoi(getenv("BSF_SIDE_STREAMS")) : 0;   // experiment
    const bool slab = sh.r0 > 0 || sh.r1 < sh.n_v;
    const bool small = side_mode == 2 || (side_mode != 1 && ((int64_t)ct->nstrips * nbatch <= 16 || slab));
    cudaStream_t fst = small ? tt.side2 : tt.side;
    if (cudaEventRecord(tt.ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(tt.side, tt.ev_fork, 0) != cudaSuccess ||
        (small && cudaStreamWaitEvent(tt.side2, tt.ev_fork, 0) != cudaSuccess))
      return -6;
    // Small problems whose core, band and corner CTAs together exceed the SMs (one C3 sheet: 112 + 56 + 4): launch
    // k_core first.  The CTA scheduler spreads a kernel's CTAs over idle SMs before doubling up, so band CTAs that
    // start first hold one SM each and push the last core CTAs into a second wave (C3 graph replays 63 -> 46 us;
    // direct calls, where the memset in front already lines the three up, are unchanged).
    const bool cf = !ov && small &&
                    (int64_t)core_ctas_per_item(*ct, core_nch) * nbatch + (int64_t)ft->band.nctas * nbatch +
                            (int64_t)ft->ntiles * nbatch > 148;
    cudaEvent_t* tv = nullptr;   // [core start, core end, band start, band end] of this call
    if (tt.tev_n > 0) {
      tv = tt.tev.data() + 4 * tt.tev_next;
      tt.tev_next = (tt.tev_next + 1) % tt.tev_n;
      tt.tev_count = std::min(tt.tev_count + 1, tt.tev_n);
    }
    if (cf) {
      if (tv && cudaEventRecord(tv[0], st) != cudaSuccess) return -6;
      rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.e_part, e_stride,
                     nfb, core_nch, d_params, tt.detJ_ref, st, ip);
      if (rc) return rc;
    }
    rc = frame_eval(*ft, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.row_ptr,
                        tt.e_part, e_stride, 0, d_params, ct->G, ct->detJ, fst, ip);
    if (rc) return rc;
    if (tv && cudaEventRecord(tv[2], tt.side) != cudaSuccess) return -6;
    rc = band_eval(ft->band, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.row_ptr,
                   tt.e_part, e_stride, ft->ntiles, d_params, ct->G, ct->detJ, tt.side, ip);
    if (rc) return rc;
    if (tv && (cudaEventRecord(tv[3], tt.side) != cudaSuccess || (!cf && cudaEventRecord(tv[0], st) != cudaSuccess)))
      return -6;
    if (ov) {
      const int64_t o1 = nfb + core_ctas_per_item(*ct, core_nch), o2 = o1 + nb_lo;
      rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.e_part, e_stride,
                     o1, 1, d_params, tt.detJ_ref, st, ip, ct->RJ0, halo->ja);
      if (rc) return rc;
      rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.e_part, e_stride,
                     o2, 1, d_params, tt.detJ_ref, st, ip, halo->jb, ct->RJ1);
    } else if (!cf) {
      rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, tt.e_part, e_stride,
                     nfb, core_nch, d_params, tt.detJ_ref, st, ip);
    }
    if (rc) return rc;
    if (tv && cudaEventRecord(tv[1], st) != cudaSuccess) return -6;
    if (cudaEventRecord(tt.ev_join, tt.side) != cudaSuccess || cudaStreamWaitEvent(st, tt.ev_join, 0) != cudaSuccess)
      return -6;
    if (small && (cudaEventRecord(tt.ev_join2, tt.side2) != cudaSuccess ||
                  cudaStreamWaitEvent(st, tt.ev_join2, 0) != cudaSuccess))
      return -6;
    const int nl = 1 + (ft->ntiles > 0) + (ft->band.ok && ft->band.nctas > 0) + (ov && halo->ja > ct->RJ0) +
                   (ov && halo->jb < ct->RJ1);
    if (launches) *launches = nl;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
  }
  const int64_t tile_slots = (int64_t)tt.nstrips * tt.nchunks;
  int core_nch = 0, core_slots = 0;
  if (core) {
    core_nch = core_pick_chunks(*ct, nbatch);
    core_slots = core_ctas_per_item(*ct, core_nch);
  }
  const int64_t e_stride = tile_slots + core_slots;
  double* epart = nullptr;
  if (core) {
    // tile slots of (strip, chunk) pairs outside the work lists are never written: keep them zero
    const int64_t need = (int64_t)nbatch * e_stride;
    if (need > tt.e_core_cap || core_slots != tt.core_ctas) {
      void* p = dalloc(need * sizeof(double));
      if (!p) return -7;
      if (cudaMemsetAsync(p, 0, need * sizeof(double), st) != cudaSuccess) return -6;
      tt.e_part_core = static_cast<double*>(p);
      tt.e_core_cap = need;
      tt.core_ctas = core_slots;
    }
    epart = tt.e_part_core;
  } else {
    const int64_t need = (int64_t)nbatch * tile_slots;
    if (need > tt.e_cap) {
      void* p = dalloc(need * sizeof(double));
      if (!p) return -7;
      tt.e_part = static_cast<double*>(p);
      tt.e_cap = need;
    }
    epart = tt.e_part;
  }
  TileArgs A;
  A.sflag = call_sflag();
  A.x = d_x; A.xs = x_stride; A.g = d_g; A.gs = g_stride; A.vals = d_vals; A.vs = v_stride; A.epart = epart;
  A.e_stride = e_stride;
  A.n_u = tt.n_u; A.n_v = tt.n_v; A.Su = tt.Su; A.Sv = tt.Sv; A.r0 = tt.r0; A.r1 = tt.r1;
  A.xlo = sh.xlo; A.xhi = sh.xhi;
  A.nchunks_total = tt.nchunks; A.nstrips = tt.nstrips;
  A.affine = tt.affine; A.project = (flags & 1) ? 1 : 0;
  A.G00 = tt.G[0]; A.G01 = tt.G[1]; A.G10 = tt.G[2]; A.G11 = tt.G[3]; A.detJ = tt.detJ;
  A.mu1 = (flags & 2) ? 0.0 : mat.mu_st1;
  A.mu2 = (flags & 2) ? 0.0 : mat.mu_st2;
  A.mush = (flags & 2) ? 0.0 : mat.mu_sh;
  A.mubd = (flags & 4) ? 0.0 : mat.mu_bd;
  A.m_aoff = tt.m_aoff; A.b_aoff = tt.b_aoff;
  A.m_info = tt.m_info;
  A.b_info = tt.b_info;
  A.utab = tt.utab; A.vtab = tt.vtab; A.stab = tt.stab; A.m_geo = tt.m_geo; A.b_geo = tt.b_geo;
  A.Mm = (int64_t)sh.mem.size(); A.Bm = (int64_t)sh.bend.size();
  A.lut = tt.lut; A.tasks = tt.tasks; A.ent = tt.ent; A.row_ptr = tt.row_ptr;
  A.params = d_params; A.detJ_ref = tt.detJ_ref; A.flags = flags;
  const int big = 1 << 30;
  A.sk_i0 = core ? tt.sk[0] : big; A.sk_i1 = core ? tt.sk[1] : big;
  A.sk_j0 = core ? tt.sk[2] : big; A.sk_j1 = core ? tt.sk[3] : big;
  A.ex_i0 = core ? tt.ex[0] : big; A.ex_i1 = core ? tt.ex[1] : big;
  A.ex_j0 = core ? tt.ex[2] : big; A.ex_j1 = core ? tt.ex[3] : big;
  int nl = 0;
  int base = 0;
  for (int L = 0; L < 2; ++L) {   // interior chunks, then boundary chunks
    if (tt.nch_l[L] == 0) continue;
    A.capm = tt.capm_l[L];
    A.capb = tt.capb_l[L];
    A.chunk_base = base;
    A.chunks = tt.chunks + base;
    if (core) {
      A.work = tt.work_l[L];
      if (tt.nwork_l[L] > 0) {
        dim3 grid(tt.nwork_l[L], 1, nbatch);
        k_tile<<<grid, kThreads, tt.smem_l[L], st>>>(A);
        ++nl;
      }
    } else {
      A.work = nullptr;
      dim3 grid(tt.nstrips, tt.nch_l[L], nbatch);
      k_tile<<<grid, kThreads, tt.smem_l[L], st>>>(A);
      ++nl;
    }
    base += tt.nch_l[L];
  }
  if (core) {
    const int rc = core_eval(*ct, sh, d_x, x_stride, mat, flags, nbatch, d_g, g_stride, d_vals, v_stride, epart,
                             e_stride, tile_slots, core_nch, d_params, tt.detJ_ref, st);
    if (rc) return rc;
    ++nl;
  }
  if (d_E) {
    k_energy_final<<<nbatch, 256, 0, st>>>(epart, (int)e_stride, d_E);
    ++nl;
  }
  if (launches) *launches = nl;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

#ifdef BSF_PHASE_TIMERS
extern "C" int bsf_debug_phase_timers(unsigned long long* out16, int reset) {
  cudaMemcpyFromSymbol(out16, g_phase, sizeof(unsigned long long) * 16);
  if (reset) { unsigned long long z[16] = {}; cudaMemcpyToSymbol(g_phase, z, sizeof(z)); }
  return 0;
}
#endif
}  // namespace bsf
