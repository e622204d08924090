// Generic assembly path (any rule, any rest shape): per-point kernels write the F-space data of
// every quadrature point to scratch, then block-owner gather kernels sum each BSR block and each
// gradient row over its incidence list (the paper's "per-block parallel gather"),
// deterministically and without atomics.
#include <cuda_runtime.h>

#include "dev.hpp"
#include "fbw.cuh"

namespace bsf {

// ---- membrane point: F = sum_e x_e b_e^T, then FBW quantities -------------
__global__ void __launch_bounds__(128) k_membrane_points(GenericTables t, const double* __restrict__ x, Mat mat,
                                                         int project) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= t.Mm) return;
  const int64_t M = t.Mm;
  double f1[3] = {0, 0, 0}, f2[3] = {0, 0, 0};
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const int xi = t.m_xi[e * M + q];
    if (xi < 0) continue;
    const double b0 = t.m_b[(2 * e) * M + q], b1 = t.m_b[(2 * e + 1) * M + q];
    const double* p = x + 3 * (int64_t)xi;
    const double c0 = p[0], c1 = p[1], c2 = p[2];
    f1[0] += c0 * b0; f1[1] += c1 * b0; f1[2] += c2 * b0;
    f2[0] += c0 * b1; f2[1] += c1 * b1; f2[2] += c2 * b1;
  }
  FSpace o;
  fbw_point(f1, f2, mat.mu_st1, mat.mu_st2, mat.mu_sh, project != 0, o);
  const double w = t.m_w[q];
  t.s_E[q] = t.m_eown[q] ? w * o.psi : 0.0;
  if (t.m_eown[q]) fbw_flag_singular(t.sflag, o.i5min, 0, (int)(q & 0x3FFFFF), 0x3FFFFF);   // t field: point index marker
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    t.s_P[c * M + q] = w * o.P1[c];
    t.s_P[(3 + c) * M + q] = w * o.P2[c];
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    t.s_A[k * M + q] = w * o.A11[k];
    t.s_A[(6 + k) * M + q] = w * o.A22[k];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) t.s_A[(12 + k) * M + q] = w * o.A12[k];
}

// ---- bending point: Lap phi = sum_e L_e x_e ---------------------------------
__global__ void __launch_bounds__(128) k_bending_points(GenericTables t, const double* __restrict__ x, Mat mat) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= t.Bm) return;
  const int64_t B = t.Bm;
  double lap[3] = {0, 0, 0};
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const int xi = t.b_xi[e * B + q];
    if (xi < 0) continue;
    const double L = t.b_L[e * B + q];
    const double* p = x + 3 * (int64_t)xi;
    lap[0] += L * p[0]; lap[1] += L * p[1]; lap[2] += L * p[2];
  }
  const double wm = t.b_w[q] * mat.mu_bd;
  t.s_E[t.Mm + q] = t.b_eown[q] ? 0.5 * wm * (lap[0] * lap[0] + lap[1] * lap[1] + lap[2] * lap[2]) : 0.0;
  t.s_D[q] = wm * lap[0];
  t.s_D[B + q] = wm * lap[1];
  t.s_D[2 * B + q] = wm * lap[2];
}

// ---- Hessian block gather: H_ab = sum_q sum_{be,ga} b_a,be b_b,ga (wA)_{be,ga}
//                                   + sum_q' w mu_bd L_a L_b I3  -------------------------------
__global__ void __launch_bounds__(256) k_hessian_gather(GenericTables t, int64_t nnzb, double* __restrict__ vals,
                                                        Mat mat) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nnzb) return;
  const int64_t M = t.Mm, B = t.Bm;
  double H[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  double diag = 0.0;
  for (int64_t s = t.h_ptr[k], e = t.h_ptr[k + 1]; s < e; ++s) {
    const uint32_t inc = t.h_inc[s];
    const int64_t q = (inc & ~kIncBend) >> 8;
    const int la = (inc >> 4) & 15, lb = inc & 15;
    if (inc & kIncBend) {
      diag += t.b_w[q] * t.b_L[la * B + q] * t.b_L[lb * B + q];
      continue;
    }
    const double ba0 = t.m_b[(2 * la) * M + q], ba1 = t.m_b[(2 * la + 1) * M + q];
    const double bb0 = t.m_b[(2 * lb) * M + q], bb1 = t.m_b[(2 * lb + 1) * M + q];
    const double c11 = ba0 * bb0, c22 = ba1 * bb1, c12 = ba0 * bb1, c21 = ba1 * bb0;
    double A11[6], A22[6], A12[9];
#pragma unroll
    for (int i = 0; i < 6; ++i) { A11[i] = t.s_A[i * M + q]; A22[i] = t.s_A[(6 + i) * M + q]; }
#pragma unroll
    for (int i = 0; i < 9; ++i) A12[i] = t.s_A[(12 + i) * M + q];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        H[3 * r + c] += c11 * A11[sym3(r, c)] + c22 * A22[sym3(r, c)] + c12 * A12[3 * r + c] + c21 * A12[3 * c + r];
  }
  diag *= mat.mu_bd;
  H[0] += diag; H[4] += diag; H[8] += diag;
  double* out = vals + 9 * k;
#pragma unroll
  for (int i = 0; i < 9; ++i) out[i] = H[i];
}

// ---- gradient gather: g_a = sum_q (wP) b_a + sum_q' (w mu_bd Lap phi) L_a ---------------------
__global__ void __launch_bounds__(256) k_gradient_gather(GenericTables t, int64_t nrows, double* __restrict__ grad) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= nrows) return;
  const int64_t M = t.Mm, B = t.Bm;
  double g[3] = {0, 0, 0};
  for (int64_t s = t.g_ptr[a], e = t.g_ptr[a + 1]; s < e; ++s) {
    const uint32_t inc = t.g_inc[s];
    const int64_t q = (inc & ~kIncBend) >> 8;
    const int la = (inc >> 4) & 15;
    if (inc & kIncBend) {
      const double L = t.b_L[la * B + q];
      g[0] += L * t.s_D[q]; g[1] += L * t.s_D[B + q]; g[2] += L * t.s_D[2 * B + q];
    } else {
      const double b0 = t.m_b[(2 * la) * M + q], b1 = t.m_b[(2 * la + 1) * M + q];
#pragma unroll
      for (int c = 0; c < 3; ++c) g[c] += t.s_P[c * M + q] * b0 + t.s_P[(3 + c) * M + q] * b1;
    }
  }
  grad[3 * a] = g[0]; grad[3 * a + 1] = g[1]; grad[3 * a + 2] = g[2];
}

// ---- deterministic energy reduction: fixed-shape tree over the per-point contributions --------
__global__ void __launch_bounds__(256) k_reduce_partials(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  __shared__ double sm[8];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) s += v[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) k_reduce_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sm[8];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
  }
}

// ---- launch orchestration ------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

int generic_eval(const GenericTables& t, const double* d_x, const Mat& mat, int flags, int64_t nnzb, int64_t nrows,
                 double* d_E, double* d_g, double* d_vals, cudaStream_t st, int* launches) {
  const bool proj = flags & 1, nomem = flags & 2, nobend = flags & 4;
  int nl = 0;
  GenericTables tt = t;
  tt.sflag = call_sflag();
  Mat m = mat;
  if (nomem) { m.mu_st1 = m.mu_st2 = m.mu_sh = 0.0; }
  if (nobend) { m.mu_bd = 0.0; }
  if (t.Mm > 0) { k_membrane_points<<<nblk(t.Mm, 128), 128, 0, st>>>(tt, d_x, m, proj ? 1 : 0); ++nl; }
  if (t.Bm > 0) { k_bending_points<<<nblk(t.Bm, 128), 128, 0, st>>>(tt, d_x, m); ++nl; }
  if (d_vals && nnzb > 0) { k_hessian_gather<<<nblk(nnzb, 256), 256, 0, st>>>(tt, nnzb, d_vals, m); ++nl; }
  if (d_g && nrows > 0) { k_gradient_gather<<<nblk(nrows, 256), 256, 0, st>>>(tt, nrows, d_g); ++nl; }
  if (d_E) {
    const int64_t n = t.Mm + t.Bm;
    if (n > 0) {
      k_reduce_partials<<<t.e_nblocks, 256, 0, st>>>(t.s_E, n, t.e_part);
      k_reduce_final<<<1, 256, 0, st>>>(t.e_part, t.e_nblocks, d_E);
      nl += 2;
    } else {
      cudaMemsetAsync(d_E, 0, sizeof(double), st);
    }
  }
  if (launches) *launches = nl;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

}  // namespace bsf
