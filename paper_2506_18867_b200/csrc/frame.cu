// k_frame: full-row assembly of the frame control points (see frame.hpp).
//
// One CTA per (tile of <= 16 control points, batch item):
//   1. stage the positions of the tile window (cps [i0-2, i0+tw+2) x [j0-2, j0+th+2)) and the tile's
//      contribution lists;
//   2. point phase: every quadrature point incident to a tile control point (host list): membrane
//      F~ = sum_e C_e d_e, F = F~ G, FBW Psi / P / A with the optional per-term projection
//      (PAPER.md:264-288), kept in the parametric frame as A~uu, A~vv, A~uv (w (G (x) I) A (G (x) I)^T)
//      and P~ = w G P; bending sqrt(w mu) L_e and sqrt(w mu) Lap phi;
//   3. gather: one thread per (control point a, block b of a's row) sums, in registers, the 3x3 block
//          H_ab = sum_q sum_{mu,nu} d_a,mu(q) d_b,nu(q) A~_mu,nu(q)  +  sum_q' w mu L_a(q') L_b(q') I3
//      over the host-built list of the points q containing a and b (the paper's per-block gather,
//      PAPER.md:705), and writes it; one more thread per control point gathers the gradient
//          g_a = sum_q d_a . P~(q) + sum_q' w mu L_a(q') Lap phi(q').
// Every frame row is written completely by this kernel and no core row is touched, so k_frame and
// k_core are independent.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "core.hpp"
#include "fbw.cuh"
#include "frame.hpp"
#include "ip.hpp"

namespace bsf {

namespace {
using namespace frame;

struct FrameArgs {
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
  int maxM, maxB;
  int project, flags, dbg;
  unsigned long long* sflag;   // singular-stretch word (fbw.cuh)
  EFinal ef;                   // fused energy reduction of the call
  double G00, G01, G10, G11, detJ, mu1, mu2, mush, mubd;
  const int4* tile;
  const int32_t* tpm;
  const int32_t* tpb;
  const int2* m_anc;
  const int32_t* m_own;
  const double* m_coef;
  const double* m_what;
  const int2* b_anc;
  const int32_t* b_own;
  const double* b_coef;
  const double* b_what;
  const uint4* lst;       // [ntiles * kTasks] per task: (first | count << 20, output, transposed output, 0):
                          // output = global block index (row_ptr + rank) or ~a_loc for the gradient;
                          // transposed output = block of H_ab^T in row b (frame pairs computed once) or -1
  const uint32_t* ent;    // tile-relative contribution entries
  const int32_t* tent;    // [ntiles+1]
  // incremental-potential terms (Q13; xhat == nullptr: elastic only)
  const double* xhat;
  int64_t xhs;
  const double* mass;
  double ipk, grav[3];
  const double* ipar;      // optional per-item parameters: masses scale by ipar[9 item + 4] / ip_detJ
  double ip_detJ;
};

constexpr int kPosD = 8 * 8 * 3;    // (tw + 4) * (th + 4) * 3 for 4x4 tiles
// record strides in doubles are odd so that lanes reading different points hit different banks
constexpr int kMRec = 29;           // 27 channels + pad
constexpr int kMCf = 19;            // 18 d-vector entries + pad
constexpr int kBRec = 13;           // 12 bending channels + pad

__global__ void __launch_bounds__(kThreads, 3) k_frame(const FrameArgs A) {
  extern __shared__ __align__(16) double fsm[];
  BSF_POISON_SMEM(fsm);
  const int tile = blockIdx.x, item = blockIdx.y, tid = threadIdx.x;
  const int4 ti = A.tile[tile];
  const int i0 = ti.x, j0 = ti.y, tw = ti.z & 255, th = ti.z >> 8, ncp = ti.w;
  const int PW = tw + 4;
  const int maxM = A.maxM, maxB = A.maxB;
  double* pos = fsm;                       // [(th+4)][(tw+4)][3]
  double* mch = pos + kPosD;               // [maxM][kMRec]  A~uu 6 | A~vv 6 | A~uv 9 | P~u 3 | P~v 3
  double* mcf = mch + kMRec * maxM;        // [maxM][kMCf]   (du, dv) per window entry
  double* bch = mcf + kMCf * maxM;         // [maxB][kBRec]  sqrt(w mu) L_e 9 | sqrt(w mu) Lap phi 3
  double* red = bch + kBRec * maxB;        // [16] energy reduction
  double* kc = red + 16;                   // [16] per-item constants (kept out of registers)
  uint32_t* sent = reinterpret_cast<uint32_t*>(kc + 16);   // [tile entries]
  const double* __restrict__ x = A.x + item * A.xs;

  // ---- per-item affine map and stiffness
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
  if (tid == 0) {
    kc[0] = G00; kc[1] = G01; kc[2] = G10; kc[3] = G11; kc[4] = det; kc[5] = mu1; kc[6] = mu2; kc[7] = mush;
    kc[8] = mubd; kc[9] = G00 * G00 + G01 * G01; kc[10] = G10 * G10 + G11 * G11; kc[11] = 2.0 * (G00 * G10 + G01 * G11);
  }


  // ---- 1. positions and the tile's contribution entries
  const int npos = (th + 4) * PW * 3;
  for (int k = tid; k < npos; k += kThreads) {
    const int row = k / (PW * 3), rem = k - row * (PW * 3);
    const int col = rem / 3, c = rem - col * 3;
    const int R = j0 - 2 + row, C = i0 - 2 + col;
    double v = 0.0;
    if (R >= A.xlo && R < A.xhi && C >= 0 && C < A.n_u) v = x[((int64_t)(R - A.xlo) * A.n_u + C) * 3 + c];
    pos[k] = v;
  }
  {
    const int e0 = A.tent[tile], ne = A.tent[tile + 1] - e0;
    for (int k = tid; k < ne; k += kThreads) sent[k] = A.ent[e0 + k];
  }
  __syncthreads();

  // ---- 2. quadrature points of the tile
  const int m0 = A.tpm[tile], M = A.tpm[tile + 1] - m0, b0 = A.tpb[tile], B = A.tpb[tile + 1] - b0;
  double e_acc = 0.0;
  // points on the threads at the end of the task order (the shortest gather lists)
  for (int t = kThreads - 1 - tid; t < ((A.dbg & 16) ? 0 : M + B); t += kThreads) {
    if (t < M) {
      const int p = m0 + t;
      const int2 an = A.m_anc[p];
      const double* cf = A.m_coef + (int64_t)kMCoef * p;
      double* rec = mch + t * kMRec;
      double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0};
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        const double du = cf[2 * e], dv = cf[2 * e + 1];
        mcf[t * kMCf + 2 * e] = du;
        mcf[t * kMCf + 2 * e + 1] = dv;
        const double* C = pos + ((an.y + e / 3 - (j0 - 2)) * PW + (an.x + e % 3 - (i0 - 2))) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) { Fu[c] = fma(C[c], du, Fu[c]); Fv[c] = fma(C[c], dv, Fv[c]); }
      }
      const double wq = A.m_what[p] * kc[4];
      double f1[3], f2[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { f1[c] = fma(Fu[c], kc[0], Fv[c] * kc[2]); f2[c] = fma(Fu[c], kc[1], Fv[c] * kc[3]); }
      double psi, i5 = 1.0;
      const auto emit_p = [&](int c, double P1c, double P2c) {   // P~_mu = w sum_beta G_mu,beta P_beta
        rec[21 + c] = wq * fma(kc[0], P1c, kc[1] * P2c);
        rec[24 + c] = wq * fma(kc[2], P1c, kc[3] * P2c);
      };
      if (!A.vals) {   // no Hessian values requested: Psi and P only (explicit FMAs: the same bits as below)
        psi = fbw_emit(f1, f2, kc[5], kc[6], kc[7], false, emit_p, [](int, int, double, double, double, double) {},
                       &i5);
      } else if (kc[1] == 0.0 && kc[2] == 0.0) {   // axis-aligned rest map: A~ by entrywise scaling
        const double auu = wq * kc[0] * kc[0], avv = wq * kc[3] * kc[3], auv = wq * kc[0] * kc[3];
        psi = fbw_emit(f1, f2, kc[5], kc[6], kc[7], A.project != 0, emit_p,
                       [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
          const int e6 = sym3(r3, c3);
          rec[e6] = auu * A11;
          rec[6 + e6] = avv * A22;
          rec[12 + 3 * r3 + c3] = auv * A12rc;
          if (r3 != c3) rec[12 + 3 * c3 + r3] = auv * A12cr;
        }, &i5);
      } else {
        const double wG00 = wq * kc[0], wG01 = wq * kc[1], wG10 = wq * kc[2], wG11 = wq * kc[3];
        const double a11 = wG00 * kc[0], a12 = wG00 * kc[1], a22 = wG01 * kc[1];
        const double b11 = wG10 * kc[2], b12 = wG10 * kc[3], b22 = wG11 * kc[3];
        const double c11 = wG00 * kc[2], c12 = wG00 * kc[3], c21 = wG01 * kc[2], c22 = wG01 * kc[3];
        psi = fbw_emit(f1, f2, kc[5], kc[6], kc[7], A.project != 0, emit_p,
                       [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
          const int e6 = sym3(r3, c3);
          rec[e6] = a11 * A11 + a12 * (A12rc + A12cr) + a22 * A22;
          rec[6 + e6] = b11 * A11 + b12 * (A12rc + A12cr) + b22 * A22;
          rec[12 + 3 * r3 + c3] = c11 * A11 + c12 * A12rc + c21 * A12cr + c22 * A22;
          if (r3 != c3) rec[12 + 3 * c3 + r3] = c11 * A11 + c12 * A12cr + c21 * A12rc + c22 * A22;
        }, &i5);
      }
      if (A.m_own[p]) {
        e_acc += wq * psi;
        fbw_flag_singular(A.sflag, i5, item, an.x, an.y);
      }
    } else {
      const int tb = t - M, q = b0 + tb;
      const int2 an = A.b_anc[q];
      const double* cf = A.b_coef + 27 * (int64_t)q;
      const double w = A.b_what[q] * kc[4];
      const double sw = sqrt(w * kc[8]);
      double* rec = bch + tb * kBRec;
      double lap[3] = {0, 0, 0};
#pragma unroll
      for (int e = 0; e < 9; ++e) {
        const double L = kc[9] * cf[e] + kc[10] * cf[9 + e] + kc[11] * cf[18 + e];
        const double* C = pos + ((an.y + e / 3 - (j0 - 2)) * PW + (an.x + e % 3 - (i0 - 2))) * 3;
        lap[0] = fma(L, C[0], lap[0]); lap[1] = fma(L, C[1], lap[1]); lap[2] = fma(L, C[2], lap[2]);
        rec[e] = sw * L;
      }
      if (A.b_own[q]) e_acc += 0.5 * w * kc[8] * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) rec[9 + c] = sw * lap[c];
    }
  }
  __syncthreads();

  // ---- 3. gather: tasks = (control point, block) or (control point, gradient), sorted by list length on
  // the host; thread tid takes tasks tid, tid + kThreads, ... (lanes of a warp run loops of similar length)
  for (int tk = tid; tk < ((A.dbg & 32) ? 0 : kTasks); tk += kThreads) {
  const uint4 task = A.lst[tile * kTasks + tk];
  const int first = task.x & 0xFFFFF, cnt = task.x >> 20;
  const int out = (int)task.y, outT = (int)task.z;
  if (out >= 0 && !A.vals) continue;   // a Hessian block task of a call without Hessian values
  if (cnt > 0 && out >= 0) {
    double h[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) h[k] = 0.0;
    double hb = 0.0;
    for (int e = 0; e < cnt; ++e) {
      const uint32_t E = sent[first + e];
      const int pt = E & 1023, ea = (E >> 10) & 15, eb = (E >> 14) & 15;
      if (!(E >> 18)) {
        const double* rec = mch + pt * kMRec;
        const double* cf = mcf + pt * kMCf;
        const double au = cf[2 * ea], av = cf[2 * ea + 1], bu = cf[2 * eb], bv = cf[2 * eb + 1];
        const double k11 = au * bu, k22 = av * bv, k12 = au * bv, k21 = av * bu;
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
          for (int c3 = 0; c3 < 3; ++c3) {
            const int e6 = sym3(r3, c3);
            h[3 * r3 + c3] = fma(k11, rec[e6], fma(k22, rec[6 + e6], fma(k12, rec[12 + 3 * r3 + c3],
                                 fma(k21, rec[12 + 3 * c3 + r3], h[3 * r3 + c3]))));
          }
      } else {
        const double* rec = bch + pt * kBRec;
        hb = fma(rec[ea], rec[eb], hb);
      }
    }
    if (A.xhat && task.w)   // diagonal block: inertia m_a/dt^2
      hb += A.ipk * A.mass[task.w - 1] * (A.ipar ? A.ipar[9 * (int64_t)item + 4] / A.ip_detJ : 1.0);
    h[0] += hb; h[4] += hb; h[8] += hb;
    if (A.vals) {
      double* dst = A.vals + item * A.vs + (int64_t)out * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) dst[k] = h[k];
      if (outT >= 0) {   // H_ba = H_ab^T (b a later frame control point)
        double* dt = A.vals + item * A.vs + (int64_t)outT * 9;
#pragma unroll
        for (int k = 0; k < 9; ++k) dt[k] = h[3 * (k % 3) + k / 3];
      }
    }
  } else if (out < 0 && (A.g || A.xhat)) {
    double g0 = 0.0, g1 = 0.0, g2 = 0.0;
    for (int e = 0; e < cnt; ++e) {
      const uint32_t E = sent[first + e];
      const int pt = E & 1023, ea = (E >> 10) & 15;
      if (!(E >> 18)) {
        const double* rec = mch + pt * kMRec;
        const double au = mcf[pt * kMCf + 2 * ea], av = mcf[pt * kMCf + 2 * ea + 1];
        g0 = fma(au, rec[21], fma(av, rec[24], g0));
        g1 = fma(au, rec[22], fma(av, rec[25], g1));
        g2 = fma(au, rec[23], fma(av, rec[26], g2));
      } else {
        const double* rec = bch + pt * kBRec;
        const double La = rec[ea];
        g0 = fma(La, rec[9], g0);
        g1 = fma(La, rec[10], g1);
        g2 = fma(La, rec[11], g2);
      }
    }
    const int64_t al = ~out;
    if (A.xhat) {   // incremental potential: m/dt^2 (x - xhat) - m g and its energy
      const int aj = (int)(al / A.n_u) + A.r0, ai = (int)(al % A.n_u);
      const double* xa = pos + ((aj - (j0 - 2)) * PW + (ai - (i0 - 2))) * 3;
      const double* xh = A.xhat + item * A.xhs + 3 * al;
      const double mm = A.mass[al] * (A.ipar ? A.ipar[9 * (int64_t)item + 4] / A.ip_detJ : 1.0);
      double gi[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double d = xa[c] - xh[c];
        gi[c] = A.ipk * mm * d - mm * A.grav[c];
        e_acc += 0.5 * A.ipk * mm * d * d - mm * A.grav[c] * xa[c];
      }
      g0 += gi[0]; g1 += gi[1]; g2 += gi[2];
    }
    if (A.g) {
      double* gd = A.g + item * A.gs + 3 * al;
      gd[0] = g0; gd[1] = g1; gd[2] = g2;
    }
  }
  }
  // ---- energy partial of this CTA
  const int lane = tid & 31, warp = tid >> 5;
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  if (lane == 0) red[warp] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) sum += red[w];
    A.epart[item * A.e_stride + A.e_off + tile] = sum;
  }
  energy_final_fused(A.ef, A.epart, item);
}

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

int build_frame(const Sheet& sh, const CoreTables& ct, FrameTables& ft, std::string& err,
                const std::function<void*(size_t)>& dalloc) {
  ft = FrameTables();
  if (!ct.ok || !sh.affine) return 1;
  const int nu = sh.n_u, Su = sh.Su, Sv = sh.Sv, r0 = sh.r0, r1 = sh.r1;
  // ---- edge bands (band.cu); the rest of the frame (corners, bands that are not translation invariant)
  // is cut into 4x4 tiles
  {
    const int brc = build_band(sh, ct, ft.band, err, dalloc);
    if (brc < 0) return brc;
  }
  const int* cov = ft.band.covered;
  struct Rect { int i0, i1, j0, j1; };
  std::vector<Rect> rects;
  for (int side = 0; side < 2; ++side) {   // bottom, top (full width, or the two corners when banded)
    const int j0 = side ? ct.RJ1 : r0, j1 = side ? r1 : ct.RJ0;
    if (cov[side]) {
      rects.push_back({0, ct.CI0, j0, j1});
      rects.push_back({ct.CI1, nu, j0, j1});
    } else {
      rects.push_back({0, nu, j0, j1});
    }
  }
  if (!cov[2]) rects.push_back({0, ct.CI0, ct.RJ0, ct.RJ1});
  if (!cov[3]) rects.push_back({ct.CI1, nu, ct.RJ0, ct.RJ1});
  std::vector<Rect> tiles;
  for (const Rect& R : rects) {
    if (R.i1 <= R.i0 || R.j1 <= R.j0) continue;
    for (int j = R.j0; j < R.j1; j += 4)
      for (int i = R.i0; i < R.i1; i += 4) tiles.push_back({i, std::min(i + 4, R.i1), j, std::min(j + 4, R.j1)});
  }
  if (tiles.empty()) {   // the bands cover the whole frame
    if (!ft.band.ok) return 1;
    ft.ntiles = 0;
    ft.ok = 1;
    return 0;
  }
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
  std::vector<int4> tinfo;
  std::vector<uint4> tasks;
  std::vector<int32_t> tpm{0}, tpb{0}, tent{0};
  std::vector<int2> m_anc, b_anc;
  std::vector<int32_t> m_own, b_own;
  std::vector<double> m_coef, m_what, b_coef, b_what;
  std::vector<uint32_t> ent;
  int max_te = 1;
  for (const Rect& T : tiles) {
    const int tw = T.i1 - T.i0, th = T.j1 - T.j0, ncp = tw * th;
    tinfo.push_back(make_int4(T.i0, T.j0, tw | (th << 8), ncp));
    std::map<int, int> loc[2];   // global point -> local index, per kind
    auto in_tile = [&](int i, int j) { return i >= T.i0 && i < T.i1 && j >= T.j0 && j < T.j1; };
    const size_t tbase = ent.size();
    std::vector<uint4> ttask;
    for (int slot = 0; slot < ncp; ++slot) {
      const int i = T.i0 + slot % tw, j = T.j0 + slot / tw;
      const int64_t al = (int64_t)(j - r0) * nu + i;
      const int32_t* c0 = sh.col_idx.data() + sh.row_ptr[al];
      const int32_t* c1 = sh.col_idx.data() + sh.row_ptr[al + 1];
      const int nb = (int)(c1 - c0);
      if (nb > kMaxNB) { err = "frame: row with more than 25 blocks"; return -1; }
      std::vector<std::vector<uint32_t>> per(kSlots);   // per block rank + gradient
      for (int kind = 0; kind < 2; ++kind) {
        const std::vector<Point>& L = kind ? sh.bend : sh.mem;
        const std::vector<int32_t>& hh = kind ? bh : mh;
        const std::vector<int32_t>& ii = kind ? bi : mi;
        for (int t = j - 2; t <= j; ++t)
          for (int s = i - 2; s <= i; ++s) {
            if (s < 0 || t < 0 || s >= Su || t >= Sv) continue;
            const int an = t * Su + s;
            for (int k = hh[an]; k < hh[an + 1]; ++k) {
              const int gp = ii[k];
              const Point& P = L[gp];
              const int ea = (i - s) + 3 * (j - t);
              if (!((P.mask >> ea) & 1)) continue;
              auto it = loc[kind].find(gp);
              const int lp = it == loc[kind].end() ? (int)loc[kind].size() : it->second;
              if (it == loc[kind].end()) loc[kind].emplace(gp, lp);
              const uint32_t head = (uint32_t)lp | ((uint32_t)ea << 10) | ((uint32_t)kind << 18);
              per[kSlots - 1].push_back(head);
              for (int e = 0; e < 9; ++e) {
                if (!((P.mask >> e) & 1)) continue;
                const int32_t b = (P.ov + e / 3) * nu + P.ou + e % 3;
                const int32_t* pb = std::lower_bound(c0, c1, b);
                if (pb == c1 || *pb != b) { err = "frame: stencil member outside the pattern"; return -1; }
                per[pb - c0].push_back(head | ((uint32_t)e << 14));
              }
            }
          }
      }
      const int32_t a_glob = j * nu + i;
      for (int k = 0; k < kSlots; ++k) {
        if (k < kMaxNB && k >= nb) continue;
        int32_t outT = -1;
        if (k < kMaxNB) {   // frame-frame pairs: computed once, by the earlier control point
          const int32_t b = c0[k];
          const int bi = b % nu, bj = b / nu;
          bool bframe = false;   // b's row is written by this kernel (a tile cp; not core, not band)
          for (const Rect& R : rects) bframe = bframe || (bi >= R.i0 && bi < R.i1 && bj >= R.j0 && bj < R.j1);
          if (bframe && b < a_glob) continue;
          if (bframe && b > a_glob) {
            const int64_t bl = (int64_t)(bj - r0) * nu + bi;
            const int32_t* d0 = sh.col_idx.data() + sh.row_ptr[bl];
            const int32_t* d1 = sh.col_idx.data() + sh.row_ptr[bl + 1];
            const int32_t* pa = std::lower_bound(d0, d1, a_glob);
            if (pa == d1 || *pa != a_glob) { err = "frame: pattern not symmetric"; return -1; }
            outT = sh.row_ptr[bl] + (int32_t)(pa - d0);
          }
        }
        const size_t f = ent.size() - tbase;
        if (f >= (1u << 20) || per[k].size() >= 4096) { err = "frame: program too long"; return -1; }
        const int32_t outi = (k == kSlots - 1) ? ~(int32_t)al : sh.row_ptr[al] + k;
        const uint32_t dg = (k < kMaxNB && c0[k] == a_glob) ? (uint32_t)al + 1u : 0u;   // diagonal block: a_loc + 1
        ttask.push_back(make_uint4((uint32_t)f | ((uint32_t)per[k].size() << 20), (uint32_t)outi, (uint32_t)outT, dg));
        ent.insert(ent.end(), per[k].begin(), per[k].end());
      }
    }
    std::stable_sort(ttask.begin(), ttask.end(), [](const uint4& a, const uint4& b) { return (a.x >> 20) > (b.x >> 20); });
    if ((int)ttask.size() > kTasks) { err = "frame: too many tasks per tile"; return -1; }
    ttask.resize(kTasks, make_uint4(0u, 0u, 0xFFFFFFFFu, 0u));
    tasks.insert(tasks.end(), ttask.begin(), ttask.end());
    if (loc[0].size() > 1023 || loc[1].size() > 1023) { err = "frame: too many points per tile"; return -1; }
    std::vector<int> mg(loc[0].size()), bg(loc[1].size());
    for (auto& kv : loc[0]) mg[kv.second] = kv.first;
    for (auto& kv : loc[1]) bg[kv.second] = kv.first;
    for (int gp : mg) {
      const Point& P = sh.mem[gp];
      m_anc.push_back(make_int2(P.ou, P.ov));
      m_own.push_back(in_tile(P.ou, P.ov) && P.ov >= r0 && P.ov < r1 ? 1 : 0);
      for (int e = 0; e < 9; ++e) {
        const int iu = e % 3, jv = e / 3;
        const bool in = (P.mask >> e) & 1;
        m_coef.push_back(in ? P.bu.d1[iu] * P.bv.N[jv] : 0.0);
        m_coef.push_back(in ? P.bu.N[iu] * P.bv.d1[jv] : 0.0);
      }
      m_what.push_back(P.what);
    }
    for (int gp : bg) {
      const Point& P = sh.bend[gp];
      b_anc.push_back(make_int2(P.ou, P.ov));
      b_own.push_back(in_tile(P.ou, P.ov) && P.ov >= r0 && P.ov < r1 ? 1 : 0);
      double LA[9], LB[9], LC[9];
      for (int e = 0; e < 9; ++e) {
        const int iu = e % 3, jv = e / 3;
        const bool in = (P.mask >> e) & 1;
        LA[e] = in ? P.bu.d2[iu] * P.bv.N[jv] : 0.0;
        LB[e] = in ? P.bu.N[iu] * P.bv.d2[jv] : 0.0;
        LC[e] = in ? P.bu.d1[iu] * P.bv.d1[jv] : 0.0;
      }
      b_coef.insert(b_coef.end(), LA, LA + 9);
      b_coef.insert(b_coef.end(), LB, LB + 9);
      b_coef.insert(b_coef.end(), LC, LC + 9);
      b_what.push_back(P.what);
    }
    ft.maxM = std::max(ft.maxM, (int)mg.size());
    ft.maxB = std::max(ft.maxB, (int)bg.size());
    tpm.push_back((int32_t)m_anc.size());
    tpb.push_back((int32_t)b_anc.size());
    max_te = std::max(max_te, (int)(ent.size() - tbase));
    tent.push_back((int32_t)ent.size());
  }
  ft.ntiles = (int)tiles.size();
  ft.maxM = std::max(ft.maxM, 1);
  ft.maxB = std::max(ft.maxB, 1);
  ft.smem = sizeof(double) * ((size_t)kPosD + (size_t)(kMRec + kMCf) * ft.maxM + (size_t)kBRec * ft.maxB + 32) +
            sizeof(uint32_t) * (size_t)max_te;
  if (ft.smem > 227 * 1024) { err = "frame: shared memory budget"; return 1; }
  const bool ok = upload(dalloc, &ft.tile, tinfo) && upload(dalloc, &ft.tpm, tpm) && upload(dalloc, &ft.tpb, tpb) &&
                  upload(dalloc, &ft.m_anc, m_anc) && upload(dalloc, &ft.m_own, m_own) &&
                  upload(dalloc, &ft.m_coef, m_coef) && upload(dalloc, &ft.m_what, m_what) &&
                  upload(dalloc, &ft.b_anc, b_anc) && upload(dalloc, &ft.b_own, b_own) &&
                  upload(dalloc, &ft.b_coef, b_coef) && upload(dalloc, &ft.b_what, b_what) &&
                  upload(dalloc, &ft.lst, tasks) && upload(dalloc, &ft.ent, ent) &&
                  upload(dalloc, &ft.tent, tent);
  if (!ok) { err = "frame: device allocation failed"; return -7; }
  if (cudaFuncSetAttribute(k_frame, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ft.smem) != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  if (getenv("BSF_CORE_DEBUG"))
    fprintf(stderr, "k_frame: %d tiles, maxM %d maxB %d, max tile entries %d, avg entries/cp %.1f, smem %zu\n",
            ft.ntiles, ft.maxM, ft.maxB, max_te, (double)ent.size() / (16.0 * ft.ntiles), ft.smem);
  ft.ok = 1;
  return 0;
}

int frame_eval(const FrameTables& ft, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
               int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const int32_t* d_row_ptr,
               double* e_part, int64_t e_stride, int64_t e_off, const double* d_params, const double* G4, double detJ,
               cudaStream_t st, const IpFused* ip) {
  if (ft.ntiles == 0) return 0;
  FrameArgs A;
  A.sflag = call_sflag();
  A.ef = call_efinal();
  A.xhat = ip ? ip->xhat : nullptr; A.xhs = ip ? ip->xhs : 0; A.mass = ip ? ip->mass : nullptr;
  A.ipk = ip ? ip->k : 0.0;
  for (int c = 0; c < 3; ++c) A.grav[c] = ip ? ip->grav[c] : 0.0;
  A.ipar = ip ? ip->params : nullptr;
  A.ip_detJ = ip ? ip->detJ_ref : 1.0;
  A.x = d_x; A.xs = x_stride; A.g = d_g; A.gs = g_stride; A.vals = d_vals; A.vs = v_stride;
  A.epart = e_part; A.e_stride = e_stride; A.e_off = e_off;
  A.row_ptr = d_row_ptr; A.params = d_params;
  A.n_u = sh.n_u; A.xlo = sh.xlo; A.xhi = sh.xhi; A.r0 = sh.r0;
  A.maxM = ft.maxM; A.maxB = ft.maxB;
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
  A.tile = ft.tile; A.tpm = ft.tpm; A.tpb = ft.tpb;
  A.m_anc = ft.m_anc; A.m_own = ft.m_own; A.m_coef = ft.m_coef; A.m_what = ft.m_what;
  A.b_anc = ft.b_anc; A.b_own = ft.b_own; A.b_coef = ft.b_coef; A.b_what = ft.b_what;
  A.lst = ft.lst; A.ent = ft.ent; A.tent = ft.tent;
  dim3 grid(ft.ntiles, nbatch);
  k_frame<<<grid, kThreads, ft.smem, st>>>(A);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

}  // namespace bsf
