// k_g3: energy, gradient and BSR Hessian under the G3-FULL rule on affine sheets (DESIGN.md §5 "k_g3").
//
// G3-FULL puts a 3x3 Gauss rule on every knot span for both energies (the paper's
// full-quadrature comparison).  On an affine sheet the basis values at the nodes of a
// span depend only on the span's position relative to the open ends (5 one-dimensional span classes per
// direction: the first two, the interior, the last two), so the host keeps, per class, the values
// N, N', N'' of the 3 local bases at the 3 nodes, verified against every point's own Cox-de Boor tables.
//
// One CTA (16 warps) per strip of 16 control-point columns x a chunk of rows, 2 rows per step:
//   1. points: the 2 new span rows of the strip window (18 spans x 9 nodes each), from positions staged in
//      shared memory: F~ = sum_e C_e (dN_e/du, dN_e/dv), F = F~ G, the FBW Psi, P and A with the optional
//      per-term projection, stored in the parametric frame as A~ = w (G (x) I) A (G (x)
//      I)^T and P~ = w G P; the bending Lap phi = sum_e L_e C_e as w mu Lap phi.  A ring
//      of 4 span rows, channel-major with the span column fastest (conflict-free gather loads);
//   2. gather: warp (r, c) accumulates entry (r, c) of the 25 blocks of each lane's block row (lanes = 16
//      columns x 2 rows) over the 81 incident points:
//          Y_u = d_a,u A~uu[rc] + d_a,v A~uv[cr],   Y_v = d_a,u A~uv[rc] + d_a,v A~vv[rc]
//          H_ab[r][c] += d_b,u Y_u + d_b,v Y_v   for the 9 control points b of the span
//      (PAPER.md:705's per-block gather, row-complete, no atomics); the bending Hessian sum_q w mu L_a L_b
//      I3 is state independent and comes from host tables per control-point class (6 parametric parts
//      combined with the item's G and mu); 3 more warps gather g_a.
// Interior CTAs (every span of the window in the interior class) take the node derivatives once per node
// (template UNI); the others look them up per span.  Outputs go straight from registers to the BSR rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "fbw.cuh"
#include "g3.hpp"

namespace bsf {

namespace {
using namespace g3;

struct G3Args {
  const double* x;
  int64_t xs;
  double* g;
  int64_t gs;
  double* vals;
  int64_t vs;
  double* epart;
  int64_t e_stride, e_off;
  const int4* ctas;       // frame CTAs: (i0, i1, ja, jb); interior: the strips (i0, i1, -, -)
  int nch, uj0, uj1;       // interior: row chunks per strip and the interior rows [uj0, uj1)
  const int32_t* row_ptr;
  const double* params;
  const double* tabs;     // [2][kMaxCls * 27]
  const int8_t* ucls;
  const int8_t* vcls;
  const double* beta;
  int n_u, n_v, Su, Sv, r0, xlo, xhi, tlo, thi, cint_u, cint_v;
  int project, flags, dbg;
  unsigned long long* sflag;   // singular-stretch word (fbw.cuh)
  double G00, G01, G10, G11, detJ, mu1, mu2, mush, mubd;
  double what[kNG];
};

constexpr int kCS = kNG * kSC;                 // channel stride of a record slot
constexpr int kSlotD = kCh * kCS;              // doubles per span row slot
constexpr int kPosC = kSC + 2;                 // staged position columns [i0 - 2, i0 + 18)
constexpr int kTabD = kMaxCls * 27;
// per-CTA constants (doubles)
constexpr int kKG = 0;      // G00 G01 G10 G11
constexpr int kKDet = 4, kKMu = 5;   // det, mu1 mu2 mush mubd (5..8)
constexpr int kKC = 9;      // cuu cvv cuv
constexpr int kKB = 12;     // beta coefficients [6]
constexpr int kKW = 18;     // what * det [9]
constexpr int kKN = 28;

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

__host__ __device__ __forceinline__ int cp_class(int i, int n) {   // bending-Hessian class of a cp index
  if (i < 4) return i;
  if (i >= n - 4) return 8 - (n - 1 - i);
  return 4;
}

__device__ __forceinline__ int slot_of(int t) { return (t + 8) & (kSlots - 1); }

// Points of span rows t0, t0 + 1 of the strip window into the ring (positions: cp rows t0 .. t0 + 3).
__device__ __forceinline__ double span_rows(const G3Args& A, const double* __restrict__ x, double* rec, double* pos,
                                            const double* tab, const double* kc, int i0, int i1, int ja, int jb,
                                            int t0, int tid) {
  if (tid < 4 * kPosC * 3) {
    const int rr = tid / (kPosC * 3), rem = tid - rr * (kPosC * 3), cc = rem / 3, c = rem - 3 * cc;
    const int R = t0 + rr, C = i0 - 2 + cc;
    pos[tid] = (R >= A.xlo && R < A.xhi && C >= 0 && C < A.n_u) ? x[((int64_t)(R - A.xlo) * A.n_u + C) * 3 + c] : 0.0;
  }
  __syncthreads();
  double e = 0.0;
  if (tid < 2 * kCS) {
    const int r = tid / kCS, rem = tid - r * kCS, g = rem / kSC, col = rem - g * kSC;
    const int t = t0 + r, s = i0 - 2 + col;
    double* R = rec + slot_of(t) * kSlotD + g * kSC + col;
    if (!(s >= 0 && s < A.Su && t >= A.tlo && t < A.thi)) {
#pragma unroll
      for (int ch = 0; ch < kCh; ++ch) R[ch * kCS] = 0.0;
      return 0.0;
    }
    const int gu = g % 3, gv = g / 3;
    const double* tu = tab + (A.ucls[s] * 3 + gu) * 9;           // N[3] | d1[3] | d2[3]
    const double* tv = tab + kTabD + (A.vcls[t] * 3 + gv) * 9;
    const double cuu = kc[kKC], cvv = kc[kKC + 1], cuv = kc[kKC + 2];
    double Fu[3] = {0, 0, 0}, Fv[3] = {0, 0, 0}, lap[3] = {0, 0, 0};
#pragma unroll
    for (int ev = 0; ev < 3; ++ev)
#pragma unroll
      for (int eu = 0; eu < 3; ++eu) {
        const double du = tu[3 + eu] * tv[ev], dv = tu[eu] * tv[3 + ev];
        const double L = cuu * tu[6 + eu] * tv[ev] + cvv * tu[eu] * tv[6 + ev] + cuv * tu[3 + eu] * tv[3 + ev];
        const double* C = pos + ((r + ev) * kPosC + col + eu) * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          Fu[c] = fma(C[c], du, Fu[c]);
          Fv[c] = fma(C[c], dv, Fv[c]);
          lap[c] = fma(C[c], L, lap[c]);
        }
      }
    const double G00 = kc[kKG], G01 = kc[kKG + 1], G10 = kc[kKG + 2], G11 = kc[kKG + 3];
    const double w = kc[kKW + g];
    double f1[3], f2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) { f1[c] = Fu[c] * G00 + Fv[c] * G10; f2[c] = Fu[c] * G01 + Fv[c] * G11; }
    const auto emit_p = [&](int c, double P1c, double P2c) {   // P~_mu = w sum_beta G_mu,beta P_beta
      R[(21 + c) * kCS] = w * (G00 * P1c + G01 * P2c);
      R[(24 + c) * kCS] = w * (G10 * P1c + G11 * P2c);
    };
    double i5 = 1.0;
    const double psi = fbw_emit(f1, f2, kc[kKMu], kc[kKMu + 1], kc[kKMu + 2], A.project != 0, emit_p,
                                [&](int r3, int c3, double A11, double A22, double A12rc, double A12cr) {
      const int e6 = sym3(r3, c3);
      const double sym12 = A12rc + A12cr;
      R[e6 * kCS] = w * (G00 * G00 * A11 + G00 * G01 * sym12 + G01 * G01 * A22);
      R[(6 + e6) * kCS] = w * (G10 * G10 * A11 + G10 * G11 * sym12 + G11 * G11 * A22);
      R[(12 + 3 * r3 + c3) * kCS] = w * (G00 * G10 * A11 + G00 * G11 * A12rc + G01 * G10 * A12cr + G01 * G11 * A22);
      if (r3 != c3)
        R[(12 + 3 * c3 + r3) * kCS] = w * (G00 * G10 * A11 + G00 * G11 * A12cr + G01 * G10 * A12rc + G01 * G11 * A22);
    }, &i5);
    const double wm = w * kc[kKMu + 3];
#pragma unroll
    for (int c = 0; c < 3; ++c) R[(27 + c) * kCS] = wm * lap[c];
    if (s >= i0 && s < i1 && t >= ja && t < jb) {
      e = w * psi + 0.5 * wm * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]);
      fbw_flag_singular(A.sflag, i5, blockIdx.y, s, t);
    }
  }
  return e;
}

// node derivatives (d_e,u, d_e,v) of the 9 window entries e = eu + 3 ev and the parametric Laplacian
// coefficients, from the 1D tables of one span and node
struct NodeD {
  double du[9], dv[9];
};

__device__ __forceinline__ void node_d(const double* tu, const double* tv, NodeD& d) {
  const double Nu0 = tu[0], Nu1 = tu[1], Nu2 = tu[2], Du0 = tu[3], Du1 = tu[4], Du2 = tu[5];
  const double Nv0 = tv[0], Nv1 = tv[1], Nv2 = tv[2], Dv0 = tv[3], Dv1 = tv[4], Dv2 = tv[5];
  const double Nu[3] = {Nu0, Nu1, Nu2}, Du[3] = {Du0, Du1, Du2}, Nv[3] = {Nv0, Nv1, Nv2}, Dv[3] = {Dv0, Dv1, Dv2};
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    d.du[e] = Du[e % 3] * Nv[e / 3];
    d.dv[e] = Nu[e % 3] * Dv[e / 3];
  }
}

template <bool UNI>
__global__ void __launch_bounds__(kThreads, 1) k_g3(const G3Args A) {
  extern __shared__ __align__(16) double sm[];
  double* rec = sm;                            // [kSlots][kCh][kNG][kSC]
  double* pos = rec + kSlots * kSlotD;         // [4][kPosC][3]
  double* tab = pos + 4 * kPosC * 3;           // [2][kTabD]
  double* kc = tab + 2 * kTabD;                // [kKN]
  double* red = kc + kKN;                      // [16]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // interior CTAs derive their chunk from blockIdx.x and the launch's chunk count (nothing batch-size
  // dependent lives in device memory, so graphs captured at any batch size replay correctly)
  int4 cta;
  if constexpr (UNI) {
    const int s = blockIdx.x / A.nch, c = blockIdx.x - s * A.nch, rows = A.uj1 - A.uj0;
    const int4 sp = A.ctas[s];
    cta = make_int4(sp.x, sp.y, A.uj0 + ((rows * c / A.nch) & ~1),
                    (c + 1 == A.nch) ? A.uj1 : A.uj0 + ((rows * (c + 1) / A.nch) & ~1));
  } else {
    cta = A.ctas[blockIdx.x];
  }
  const int item = blockIdx.y;
  if (cta.z >= cta.w) {   // empty chunk: its energy slot is still written
    if (threadIdx.x == 0) A.epart[item * A.e_stride + A.e_off + blockIdx.x] = 0.0;
    return;
  }
  BSF_POISON_SMEM(sm);
  const int i0 = cta.x, i1 = cta.y, ja = cta.z, jb = cta.w;
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
    kc[kKG] = G00; kc[kKG + 1] = G01; kc[kKG + 2] = G10; kc[kKG + 3] = G11; kc[kKDet] = det;
    kc[kKMu] = mu1; kc[kKMu + 1] = mu2; kc[kKMu + 2] = mush; kc[kKMu + 3] = mubd;
    const double cuu = G00 * G00 + G01 * G01, cvv = G10 * G10 + G11 * G11, cuv = 2.0 * (G00 * G10 + G01 * G11);
    kc[kKC] = cuu; kc[kKC + 1] = cvv; kc[kKC + 2] = cuv;
    const double s = det * mubd;
    kc[kKB] = s * cuu * cuu; kc[kKB + 1] = s * cvv * cvv; kc[kKB + 2] = s * cuv * cuv;
    kc[kKB + 3] = s * cuu * cvv; kc[kKB + 4] = s * cuu * cuv; kc[kKB + 5] = s * cvv * cuv;
    for (int g = 0; g < kNG; ++g) kc[kKW + g] = A.what[g] * det;
  }
  for (int k = tid; k < 2 * kTabD; k += kThreads) tab[k] = A.tabs[k];
  __syncthreads();

  double e_acc = 0.0;
  const int h = lane >> 4, m = lane & 15;
  const bool hess_warp = warp < 9 && A.vals, grad_warp = warp >= 9 && warp < 12 && A.g;
  const int r3 = warp / 3, c3 = warp - 3 * (warp / 3);
  const int rg = warp - 9;   // gradient component of a gradient warp
  // step j: span rows j, j+1 into the ring, then the gather of cp rows j, j+1 (spans j-2 .. j+1); the first
  // step (j = ja - 2) only fills the ring.  One call site of span_rows: every span row is evaluated by the
  // same instructions whatever the chunking (bit-identical results across launch configurations).
  for (int j = ja - 2; j < jb; j += 2) {
    __syncthreads();
    if (!(A.dbg & 1) || j < ja) e_acc += span_rows(A, x, rec, pos, tab, kc, i0, i1, ja, jb, j, tid);
    __syncthreads();
    if (j < ja || (!hess_warp && !grad_warp) || (A.dbg & 2)) continue;
    const int i = i0 + m, jr = j + h;
    const bool active = i < i1 && jr < jb;
    int sl[3];
#pragma unroll
    for (int dv = 0; dv < 3; ++dv) sl[dv] = slot_of(jr - 2 + dv);
    // span classes of the lane's 3 x 3 spans (general CTAs; spans off the sheet have zero records)
    int cu[3] = {A.cint_u, A.cint_u, A.cint_u}, cv[3] = {A.cint_v, A.cint_v, A.cint_v};
    if constexpr (!UNI) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        cu[d] = A.ucls[min(max(i - 2 + d, 0), A.Su - 1)];
        cv[d] = max((int)A.vcls[min(max(jr - 2 + d, 0), A.Sv - 1)], 0);
      }
    }
    if (hess_warp) {
      const int o_uu = sym3(r3, c3) * kCS, o_vv = (6 + sym3(r3, c3)) * kCS;
      const int o_rc = (12 + 3 * r3 + c3) * kCS, o_cr = (12 + 3 * c3 + r3) * kCS;
      double acc[25];
#pragma unroll
      for (int k = 0; k < 25; ++k) acc[k] = 0.0;
#pragma unroll 1
      for (int g = 0; g < kNG; ++g) {
        const int gu = g % 3, gv = g / 3;
        NodeD d;
        if constexpr (UNI) node_d(tab + (A.cint_u * 3 + gu) * 9, tab + kTabD + (A.cint_v * 3 + gv) * 9, d);
        static_for<0, 3>([&](auto DV_) {
          constexpr int DV = decltype(DV_)::value;
          static_for<0, 3>([&](auto DU_) {
            constexpr int DU = decltype(DU_)::value;
            if constexpr (!UNI) node_d(tab + (cu[DU] * 3 + gu) * 9, tab + kTabD + (cv[DV] * 3 + gv) * 9, d);
            const double* b = rec + sl[DV] * kSlotD + g * kSC + m + DU;
            const double auu = b[o_uu], avv = b[o_vv], arc = b[o_rc], acr = b[o_cr];
            constexpr int EA = (2 - DU) + 3 * (2 - DV);
            const double Yu = fma(d.du[EA], auu, d.dv[EA] * acr), Yv = fma(d.du[EA], arc, d.dv[EA] * avv);
            static_for<0, 9>([&](auto EB_) {
              constexpr int EB = decltype(EB_)::value;
              constexpr int k = (EB / 3 + DV) * 5 + (EB % 3 + DU);
              acc[k] = fma(d.du[EB], Yu, fma(d.dv[EB], Yv, acc[k]));
            });
          });
        });
      }
      if (r3 == c3) {   // bending: beta_ab = sum_p coef_p T_p[class(a)][b - a]
        const double* T = A.beta + (cp_class(min(i, A.n_u - 1), A.n_u) * 9 + cp_class(min(jr, A.n_v - 1), A.n_v)) * 150;
#pragma unroll
        for (int k = 0; k < 25; ++k) {
          double bsum = 0.0;
#pragma unroll
          for (int p = 0; p < kBetaParts; ++p) bsum = fma(kc[kKB + p], __ldg(T + p * 25 + k), bsum);
          acc[k] += bsum;
        }
      }
      if (active) {
        const int64_t al = (int64_t)(jr - A.r0) * A.n_u + i;
        double* out = A.vals + item * A.vs + (int64_t)A.row_ptr[al] * 9 + 3 * r3 + c3;
        if constexpr (UNI) {
#pragma unroll
          for (int k = 0; k < 25; ++k) out[k * 9] = acc[k];
        } else {
          const int dimin = max(-2, -i), dimax = min(2, A.n_u - 1 - i);
          const int djmin = max(-2, -jr), djmax = min(2, A.n_v - 1 - jr);
          const int nd = dimax - dimin + 1;
#pragma unroll
          for (int k = 0; k < 25; ++k) {
            const int di = k % 5 - 2, dj = k / 5 - 2;
            if (di >= dimin && di <= dimax && dj >= djmin && dj <= djmax)
              out[((dj - djmin) * nd + (di - dimin)) * 9] = acc[k];
          }
        }
      }
    } else {   // gradient component rg: g_a = sum_q d_a . P~(q) + sum_q L_a (w mu Lap phi)(q)
      const double cuu = kc[kKC], cvv = kc[kKC + 1], cuv = kc[kKC + 2];
      double gacc = 0.0;
#pragma unroll 1
      for (int g = 0; g < kNG; ++g) {
        const int gu = g % 3, gv = g / 3;
        static_for<0, 3>([&](auto DV_) {
          constexpr int DV = decltype(DV_)::value;
          static_for<0, 3>([&](auto DU_) {
            constexpr int DU = decltype(DU_)::value;
            constexpr int eu = 2 - DU, ev = 2 - DV;
            const double* tu = tab + ((UNI ? A.cint_u : cu[DU]) * 3 + gu) * 9;
            const double* tv = tab + kTabD + ((UNI ? A.cint_v : cv[DV]) * 3 + gv) * 9;
            const double dau = tu[3 + eu] * tv[ev], dav = tu[eu] * tv[3 + ev];
            const double La = cuu * tu[6 + eu] * tv[ev] + cvv * tu[eu] * tv[6 + ev] + cuv * tu[3 + eu] * tv[3 + ev];
            const double* b = rec + sl[DV] * kSlotD + g * kSC + m + DU;
            gacc = fma(dau, b[(21 + rg) * kCS], fma(dav, b[(24 + rg) * kCS], fma(La, b[(27 + rg) * kCS], gacc)));
          });
        });
      }
      if (active) A.g[item * A.gs + ((int64_t)(jr - A.r0) * A.n_u + i) * 3 + rg] = gacc;
    }
  }
  // energy partial of this CTA (fixed-order tree)
  for (int o = 16; o > 0; o >>= 1) e_acc += __shfl_xor_sync(0xffffffffu, e_acc, o);
  __syncthreads();
  if (lane == 0) red[warp] = e_acc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    A.epart[item * A.e_stride + A.e_off + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) k_g3_energy(const double* __restrict__ part, int n, int64_t stride,
                                                   double* __restrict__ E) {
  __shared__ double sm[8];
  const double* p = part + blockIdx.x * stride;
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += p[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sm[w];
    E[blockIdx.x] = t;
  }
}

bool close(double a, double b) { return std::fabs(a - b) <= 1e-12 * std::max(1.0, std::fabs(b)); }

template <class T>
bool upload_vec(const std::function<void*(size_t)>& dalloc, T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return true;
  void* p = dalloc(v.size() * sizeof(T));
  if (!p || cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return false;
  *dst = static_cast<T*>(p);
  return true;
}

using Node = std::array<double, 9>;   // N[3] | d1[3] | d2[3] of the 3 local bases at one node

Node node_of(const Basis1& b) {
  return {b.N[0], b.N[1], b.N[2], b.d1[0], b.d1[1], b.d1[2], b.d2[0], b.d2[1], b.d2[2]};
}
bool node_close(const Node& a, const Node& b) {
  for (int k = 0; k < 9; ++k)
    if (!close(a[k], b[k])) return false;
  return true;
}

// 1D classes of one direction: spans[k] = the 3 nodes of span k (sorted along the span); returns false if
// a span does not have exactly 3 nodes or there are more than kMaxCls classes.
bool make_classes(const std::vector<std::vector<Node>>& spans, std::vector<std::array<Node, 3>>& cls,
                  std::vector<int8_t>& of) {
  of.assign(spans.size(), -1);
  for (size_t s = 0; s < spans.size(); ++s) {
    if (spans[s].empty()) continue;
    if (spans[s].size() != 3) return false;
    std::array<Node, 3> key = {spans[s][0], spans[s][1], spans[s][2]};
    std::sort(key.begin(), key.end(), [](const Node& a, const Node& b) { return a[0] > b[0]; });   // N_left decreases along the span
    int id = -1;
    for (size_t c = 0; c < cls.size() && id < 0; ++c)
      if (node_close(cls[c][0], key[0]) && node_close(cls[c][1], key[1]) && node_close(cls[c][2], key[2])) id = (int)c;
    if (id < 0) {
      if ((int)cls.size() >= kMaxCls) return false;
      id = (int)cls.size();
      cls.push_back(key);
    }
    of[s] = (int8_t)id;
  }
  return true;
}

int node_index(const std::array<Node, 3>& c, const Node& n) {
  for (int k = 0; k < 3; ++k)
    if (node_close(c[k], n)) return k;
  return -1;
}

}  // namespace

int build_g3(const Sheet& sh, G3Tables& gt, std::string& err, const std::function<void*(size_t)>& dalloc) {
  gt = G3Tables();
  auto no = [&](int line) {
    if (getenv("BSF_CORE_DEBUG")) fprintf(stderr, "build_g3: not applicable (line %d)\n", line);
    return 1;
  };
  if (!sh.affine || sh.mrule != RULE_G3_FULL || sh.brule != RULE_G3_FULL) return no(__LINE__);
  const int nu = sh.n_u, nv = sh.n_v, Su = sh.Su, Sv = sh.Sv;
  const int tlo = std::max(0, sh.r0 - 2), thi = std::min(Sv, sh.r1);
  if (Su < 1 || thi <= tlo) return no(__LINE__);
  const size_t npts = (size_t)9 * Su * (thi - tlo);
  if (sh.mem.size() != npts || sh.bend.size() != npts) return no(__LINE__);
  // ---- 1D node tables per span (u from the first window row, v from the first column)
  std::vector<std::vector<Node>> us(Su), vs(Sv);
  auto add = [](std::vector<Node>& v, const Node& n) {
    for (const Node& m : v)
      if (node_close(m, n)) return;
    v.push_back(n);
  };
  for (const Point& P : sh.mem) {
    if (P.ov == tlo) add(us[P.ou], node_of(P.bu));
    if (P.ou == 0) add(vs[P.ov], node_of(P.bv));
  }
  std::vector<std::array<Node, 3>> cu, cv;
  std::vector<int8_t> ucls, vcls;
  if (!make_classes(us, cu, ucls) || !make_classes(vs, cv, vcls)) return no(__LINE__);
  for (int s = 0; s < Su; ++s)
    if (ucls[s] < 0) return no(__LINE__);
  for (int t = tlo; t < thi; ++t)
    if (vcls[t] < 0) return no(__LINE__);
  // ---- every point: its nodes, weight and geometry against the tables
  const Point& p0 = sh.mem[0];
  const double G[4] = {p0.G[0][0], p0.G[0][1], p0.G[1][0], p0.G[1][1]};
  bool have_w[kNG] = {};
  for (int pass = 0; pass < 2; ++pass)
    for (const Point& P : pass ? sh.bend : sh.mem) {
      if (P.mask != 0x1FF || P.ou < 0 || P.ou >= Su || P.ov < tlo || P.ov >= thi) return no(__LINE__);
      const int gu = node_index(cu[ucls[P.ou]], node_of(P.bu)), gv = node_index(cv[vcls[P.ov]], node_of(P.bv));
      if (gu < 0 || gv < 0) return no(__LINE__);
      const int g = gu + 3 * gv;
      if (!have_w[g]) { gt.what[g] = P.what; have_w[g] = true; }
      if (!close(P.what, gt.what[g])) return no(__LINE__);   // G and det J: constant up to sh.affine's bound
      if (pass && (std::fabs(P.c_u) > 1e-9 * std::max(1.0, P.c_uu) || std::fabs(P.c_v) > 1e-9 * std::max(1.0, P.c_vv)))
        return no(__LINE__);
    }
  for (bool hw : have_w)
    if (!hw) return no(__LINE__);
  // ---- pattern: every owned row holds the full (clipped) 5 x 5 offsets in (dj, di) order
  for (int j = sh.r0; j < sh.r1; ++j)
    for (int i = 0; i < nu; ++i) {
      const int64_t al = (int64_t)(j - sh.r0) * nu + i;
      int k = sh.row_ptr[al];
      for (int dj = std::max(-2, -j); dj <= std::min(2, nv - 1 - j); ++dj)
        for (int di = std::max(-2, -i); di <= std::min(2, nu - 1 - i); ++di) {
          if (k >= sh.row_ptr[al + 1] || sh.col_idx[k] != (j + dj) * nu + i + di) return no(__LINE__);
          ++k;
        }
      if (k != sh.row_ptr[al + 1]) return no(__LINE__);
    }
  gt.n_u = nu; gt.n_v = nv; gt.Su = Su; gt.Sv = Sv; gt.r0 = sh.r0; gt.r1 = sh.r1; gt.xlo = sh.xlo; gt.xhi = sh.xhi;
  gt.tlo = tlo; gt.thi = thi;
  gt.ncls_u = (int)cu.size(); gt.ncls_v = (int)cv.size();
  for (int k = 0; k < 4; ++k) gt.G[k] = G[k];
  gt.detJ = p0.detJ;
  for (size_t c = 0; c < cu.size(); ++c)
    for (int n = 0; n < 3; ++n)
      for (int k = 0; k < 9; ++k) gt.utab[c * 27 + n * 9 + k] = cu[c][n][k];
  for (size_t c = 0; c < cv.size(); ++c)
    for (int n = 0; n < 3; ++n)
      for (int k = 0; k < 9; ++k) gt.vtab[c * 27 + n * 9 + k] = cv[c][n][k];
  // interior class: spans [2, S - 3] (every span whose three bases are the uniform B-spline)
  auto interior = [](const std::vector<int8_t>& of, int S, int lo, int hi) -> int {
    if (S < 5) return -1;
    const int c = of[std::max(2, lo)];
    for (int s = std::max(2, lo); s <= std::min(S - 3, hi - 1); ++s)
      if (of[s] != c) return -1;
    return c;
  };
  gt.cint_u = interior(ucls, Su, 0, Su);
  gt.cint_v = interior(vcls, Sv, tlo, thi);
  // ---- bending Hessian parts per control-point class pair (representatives: first cp of each class)
  std::vector<double> beta((size_t)81 * 150, 0.0);
  {
    const double* UT = gt.utab;
    const double* VT = gt.vtab;
    for (int pu = 0; pu < 9; ++pu)
      for (int pv = 0; pv < 9; ++pv) {
        int i = -1, j = -1;
        for (int q = 0; q < nu && i < 0; ++q)
          if (cp_class(q, nu) == pu) i = q;
        for (int q = sh.r0; q < sh.r1 && j < 0; ++q)
          if (cp_class(q, nv) == pv) j = q;
        if (i < 0 || j < 0) continue;
        double* T = beta.data() + (pu * 9 + pv) * 150;
        for (int t = std::max(0, j - 2); t <= std::min(Sv - 1, j); ++t)
          for (int s = std::max(0, i - 2); s <= std::min(Su - 1, i); ++s)
            for (int g = 0; g < kNG; ++g) {
              const double* tu = UT + (ucls[s] * 3 + g % 3) * 9;
              const double* tv = VT + (vcls[t] * 3 + g / 3) * 9;
              const int eau = i - s, eav = j - t;
              const double LA_a = tu[6 + eau] * tv[eav], LB_a = tu[eau] * tv[6 + eav], LC_a = tu[3 + eau] * tv[3 + eav];
              const double wh = gt.what[g];
              for (int ebv = 0; ebv < 3; ++ebv)
                for (int ebu = 0; ebu < 3; ++ebu) {
                  const int k = (t + ebv - j + 2) * 5 + (s + ebu - i + 2);
                  const double LA_b = tu[6 + ebu] * tv[ebv], LB_b = tu[ebu] * tv[6 + ebv], LC_b = tu[3 + ebu] * tv[3 + ebv];
                  T[0 * 25 + k] += wh * LA_a * LA_b;
                  T[1 * 25 + k] += wh * LB_a * LB_b;
                  T[2 * 25 + k] += wh * LC_a * LC_b;
                  T[3 * 25 + k] += wh * (LA_a * LB_b + LB_a * LA_b);
                  T[4 * 25 + k] += wh * (LA_a * LC_b + LC_a * LA_b);
                  T[5 * 25 + k] += wh * (LB_a * LC_b + LC_a * LB_b);
                }
            }
      }
  }
  // ---- CTA lists: interior strips [16, n_u - 16) x rows [4, n_v - 4) take the uniform path
  struct Seg { int a, b; bool uni; };
  std::vector<Seg> cs, rs;
  const bool cuni = gt.cint_u >= 0 && gt.cint_v >= 0 && nu >= 2 * kW + 4;
  if (cuni) {
    cs.push_back({0, kW, false});
    for (int a = kW; a < nu - kW; a += kW) cs.push_back({a, std::min(a + kW, nu - kW), true});
    cs.push_back({nu - kW, nu, false});
  } else {
    for (int a = 0; a < nu; a += kW) cs.push_back({a, std::min(a + kW, nu), false});
  }
  const int ru0 = std::max(sh.r0, 4), ru1 = std::min(sh.r1, nv - 4);
  auto add_rows = [&](int a, int b, bool uni) {
    for (int q = a; q < b; q += 32) rs.push_back({q, std::min(q + 32, b), uni});
  };
  if (cuni && ru1 > ru0) {
    if (ru0 > sh.r0) add_rows(sh.r0, ru0, false);
    gt.uni_j0 = ru0; gt.uni_j1 = ru1;
    if (ru1 < sh.r1) add_rows(ru1, sh.r1, false);
  } else {
    add_rows(sh.r0, sh.r1, false);
  }
  for (const Seg& c : cs) {
    if (c.uni && gt.uni_j1 > gt.uni_j0) gt.h_uni_strips.push_back(make_int4(c.a, c.b, 0, 0));
    for (const Seg& r : rs) gt.h_gen.push_back(make_int4(c.a, c.b, r.a, r.b));
    if (!c.uni && gt.uni_j1 > gt.uni_j0)   // general strips also cover the interior rows
      for (int q = gt.uni_j0; q < gt.uni_j1; q += 32) gt.h_gen.push_back(make_int4(c.a, c.b, q, std::min(q + 32, gt.uni_j1)));
  }
  gt.n_gen = (int)gt.h_gen.size();
  // ---- device tables
  std::vector<double> tabs(2 * kTabD, 0.0);
  std::memcpy(tabs.data(), gt.utab, sizeof(double) * kTabD);
  std::memcpy(tabs.data() + kTabD, gt.vtab, sizeof(double) * kTabD);
  std::vector<int32_t> rp(sh.row_ptr.begin(), sh.row_ptr.end());
  double* d_tabs = nullptr;
  if (!upload_vec(dalloc, &d_tabs, tabs) || !upload_vec(dalloc, &gt.ucls, ucls) || !upload_vec(dalloc, &gt.vcls, vcls) ||
      !upload_vec(dalloc, &gt.beta, beta) || !upload_vec(dalloc, &gt.row_ptr, rp) ||
      !upload_vec(dalloc, &gt.cta_gen, gt.h_gen) || !upload_vec(dalloc, &gt.cta_uni, gt.h_uni_strips)) {
    err = "g3 tables: device allocation failed";
    return -7;
  }
  gt.d_tabs = d_tabs;
  gt.smem = sizeof(double) * ((size_t)kSlots * kSlotD + 4 * kPosC * 3 + 2 * kTabD + kKN + 16);
  if (cudaFuncSetAttribute(k_g3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gt.smem) != cudaSuccess ||
      cudaFuncSetAttribute(k_g3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gt.smem) != cudaSuccess) {
    cudaGetLastError();
    return no(__LINE__);
  }
  gt.ok = 1;
  return 0;
}

int g3_eval(G3Tables& gt, const double* d_x, int64_t x_stride, const Mat& mat, int flags, int nbatch, double* d_E,
            double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const double* d_params, cudaStream_t st,
            int* launches, const std::function<void*(size_t)>& dalloc) {
  int nl = 0;
  // interior row chunks for this batch size: minimise (waves of 1 CTA per SM) x (rows per chunk + 1 prologue
  // step), chunks of >= 8 rows.  The chunk count is a launch argument (no per-batch device list).
  int nch = 1;
  if (!gt.h_uni_strips.empty()) {
    const int rows = gt.uni_j1 - gt.uni_j0;
    const long long per = (long long)gt.h_uni_strips.size() * nbatch, gen = (long long)gt.n_gen * nbatch;
    double bc = 1e300;
    for (int c = 1; c <= std::max(1, rows / 8); ++c) {
      const long long waves = (per * c + gen + 147) / 148;
      const double cost = (double)waves * ((double)rows / c + 2.0);
      if (cost < bc - 1e-9) { bc = cost; nch = c; }
    }
  }
  gt.n_uni = (int)gt.h_uni_strips.size() * nch;
  const int64_t nct = gt.n_uni + gt.n_gen;
  if ((int64_t)nbatch * nct > gt.e_cap) {
    void* p = dalloc(sizeof(double) * (size_t)nbatch * nct);
    if (!p) return -7;
    gt.e_part = static_cast<double*>(p);
    gt.e_cap = (int64_t)nbatch * nct;
  }
  G3Args A;
  A.sflag = call_sflag();
  A.x = d_x; A.xs = x_stride; A.g = d_g; A.gs = g_stride; A.vals = d_vals; A.vs = v_stride;
  A.epart = gt.e_part; A.e_stride = nct;
  A.row_ptr = gt.row_ptr; A.params = d_params; A.tabs = gt.d_tabs; A.ucls = gt.ucls; A.vcls = gt.vcls; A.beta = gt.beta;
  A.n_u = gt.n_u; A.n_v = gt.n_v; A.Su = gt.Su; A.Sv = gt.Sv; A.r0 = gt.r0; A.xlo = gt.xlo; A.xhi = gt.xhi;
  A.tlo = gt.tlo; A.thi = gt.thi; A.cint_u = std::max(gt.cint_u, 0); A.cint_v = std::max(gt.cint_v, 0);
  A.project = (flags & 1) ? 1 : 0; A.flags = flags;
  {   // profiling switches (read once per process): 1 no point phase after the first step, 2 no gather
    static const int dbg = getenv("BSF_G3_DEBUG") ? atoi(getenv("BSF_G3_DEBUG")) : 0;
    A.dbg = dbg;
  }
  A.G00 = gt.G[0]; A.G01 = gt.G[1]; A.G10 = gt.G[2]; A.G11 = gt.G[3]; A.detJ = gt.detJ;
  A.mu1 = (flags & 2) ? 0.0 : mat.mu_st1;
  A.mu2 = (flags & 2) ? 0.0 : mat.mu_st2;
  A.mush = (flags & 2) ? 0.0 : mat.mu_sh;
  A.mubd = (flags & 4) ? 0.0 : mat.mu_bd;
  std::memcpy(A.what, gt.what, sizeof(A.what));
  if (gt.n_gen > 0) {
    A.ctas = gt.cta_gen; A.e_off = 0;
    k_g3<false><<<dim3(gt.n_gen, nbatch), kThreads, gt.smem, st>>>(A);
    ++nl;
  }
  if (gt.n_uni > 0) {
    A.ctas = gt.cta_uni; A.e_off = gt.n_gen; A.nch = nch; A.uj0 = gt.uni_j0; A.uj1 = gt.uni_j1;
    k_g3<true><<<dim3(gt.n_uni, nbatch), kThreads, gt.smem, st>>>(A);
    ++nl;
  }
  if (d_E) {
    k_g3_energy<<<nbatch, 256, 0, st>>>(gt.e_part, (int)nct, nct, d_E);
    ++nl;
  }
  if (launches) *launches = nl;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

}  // namespace bsf
