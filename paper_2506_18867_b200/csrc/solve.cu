// Linear algebra on the assembled BSR Hessian (closing the Newton step on the GPU).
//
// The projected Newton step (Eq. `eq: per iteration solve`) solves
//     (H_inertia + H_elasticity) dC = -g
// with the matrix this library assembles.  The paper factorises it (CHOLMOD); here it is solved by
// block-Jacobi preconditioned conjugate gradients on the device (the PSD projection plus the lumped
// inertia make the matrix SPD).  Also: y = H x (BSR SpMV) and the Gershgorin spectrum bound the paper uses
// to gate its Neumann split.
//
// Kernels (FP64, HBM-bound: the matrix streams once per product, 72 B per block):
//   k_spmv       one warp per block row: lane k multiplies block k of the row (rows have <= 25 blocks)
//                by x_col, a 3-value warp reduction gives y_a; optional fused dot p.(Ap) partials
//   k_diag_inv   3x3 inverses of the diagonal blocks (adjugate / determinant)
//   k_cg_update  x += alpha p, r -= alpha q, z = D^-1 r, partial sums of r.z and r.r
//   k_cg_dir     p = z + beta p
//   k_cg_scalar  one thread: fixed-order sums of the partials, alpha / beta / convergence flag
//   k_gersh      per scalar row: a_ii -/+ sum_{j != i} |a_ij|, reduced to min / max
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "solve.hpp"

namespace bsf {

namespace {

constexpr int kWarpsPerBlk = 8;
constexpr int kVecThreads = 256;

// y[a] = sum_b H_ab x[b]; rows = owned cps (global index r0*n_u + a), x in the position layout (rows
// [xlo, ...)).  dot: if non-null, partial[blockIdx.x] = sum over the CTA's rows of p[a].y[a] with p = x
// restricted to owned rows.
__global__ void __launch_bounds__(32 * kWarpsPerBlk) k_spmv(const int32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col_idx,
                                                            const double* __restrict__ vals,
                                                            const double* __restrict__ x, double* __restrict__ y,
                                                            int nrows, int n_u, int r0, int xlo,
                                                            double* __restrict__ dot_part) {
  __shared__ double red[kWarpsPerBlk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x * kWarpsPerBlk + warp;
  double d = 0.0;
  if (a < nrows) {
    const int q0 = row_ptr[a], q1 = row_ptr[a + 1];
    double y0 = 0.0, y1 = 0.0, y2 = 0.0;
    for (int q = q0 + lane; q < q1; q += 32) {
      const int b = col_idx[q] - xlo * n_u;
      const double* h = vals + (int64_t)q * 9;
      const double x0 = x[3 * (int64_t)b], x1 = x[3 * (int64_t)b + 1], x2 = x[3 * (int64_t)b + 2];
      y0 = fma(h[0], x0, fma(h[1], x1, fma(h[2], x2, y0)));
      y1 = fma(h[3], x0, fma(h[4], x1, fma(h[5], x2, y1)));
      y2 = fma(h[6], x0, fma(h[7], x1, fma(h[8], x2, y2)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      y0 += __shfl_xor_sync(0xffffffffu, y0, o);
      y1 += __shfl_xor_sync(0xffffffffu, y1, o);
      y2 += __shfl_xor_sync(0xffffffffu, y2, o);
    }
    if (lane == 0) {
      y[3 * (int64_t)a] = y0; y[3 * (int64_t)a + 1] = y1; y[3 * (int64_t)a + 2] = y2;
      if (dot_part) {
        const double* p = x + 3 * ((int64_t)(r0 - xlo) * n_u + a);
        d = p[0] * y0 + p[1] * y1 + p[2] * y2;
      }
    }
  }
  if (!dot_part) return;
  if (lane == 0) red[warp] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarpsPerBlk; ++w) s += red[w];
    dot_part[blockIdx.x] = s;
  }
}

__global__ void k_diag_inv(const int32_t* __restrict__ diag, const double* __restrict__ vals, double* __restrict__ dinv,
                           int nrows, int* __restrict__ bad) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nrows) return;
  const double* m = vals + (int64_t)diag[a] * 9;
  const double c00 = m[4] * m[8] - m[5] * m[7], c01 = m[5] * m[6] - m[3] * m[8], c02 = m[3] * m[7] - m[4] * m[6];
  const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  double* o = dinv + (int64_t)a * 9;
  if (!(det > 0.0)) { atomicExch(bad, 1); for (int k = 0; k < 9; ++k) o[k] = (k % 4 == 0) ? 1.0 : 0.0; return; }
  const double r = 1.0 / det;
  o[0] = c00 * r; o[1] = (m[2] * m[7] - m[1] * m[8]) * r; o[2] = (m[1] * m[5] - m[2] * m[4]) * r;
  o[3] = c01 * r; o[4] = (m[0] * m[8] - m[2] * m[6]) * r; o[5] = (m[2] * m[3] - m[0] * m[5]) * r;
  o[6] = c02 * r; o[7] = (m[1] * m[6] - m[0] * m[7]) * r; o[8] = (m[0] * m[4] - m[1] * m[3]) * r;
}

// z = D^-1 r and the partial sums of r.z, r.r (mode 0: initial, no update; mode 1: x += a p, r -= a q first)
__global__ void __launch_bounds__(kVecThreads) k_cg_update(int mode, const double* __restrict__ S, double* __restrict__ xs,
                                                           const double* __restrict__ p, const double* __restrict__ q,
                                                           double* __restrict__ r, double* __restrict__ z,
                                                           const double* __restrict__ dinv, int nrows,
                                                           double* __restrict__ part) {
  __shared__ double red[2][kVecThreads / 32];
  const int a = blockIdx.x * kVecThreads + threadIdx.x;
  double rz = 0.0, rr = 0.0;
  if (a < nrows && !(mode && S[kSDone] != 0.0)) {
    double rv[3];
    const double al = mode ? S[kSAlpha] : 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int64_t k = 3 * (int64_t)a + c;
      double rk = r[k];
      if (mode) {
        xs[k] = fma(al, p[k], xs[k]);
        rk = fma(-al, q[k], rk);
        r[k] = rk;
      }
      rv[c] = rk;
    }
    const double* m = dinv + (int64_t)a * 9;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double zc = m[3 * c] * rv[0] + m[3 * c + 1] * rv[1] + m[3 * c + 2] * rv[2];
      z[3 * (int64_t)a + c] = zc;
      rz = fma(rv[c], zc, rz);
      rr = fma(rv[c], rv[c], rr);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rz += __shfl_xor_sync(0xffffffffu, rz, o);
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = rz; red[1][threadIdx.x >> 5] = rr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kVecThreads / 32; ++w) { s0 += red[0][w]; s1 += red[1][w]; }
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// p = z + beta p (mode 0: p = z); p lives in the position layout of a single-slab sheet (= owned layout)
__global__ void __launch_bounds__(kVecThreads) k_cg_dir(int mode, const double* __restrict__ S, const double* __restrict__ z,
                                                        double* __restrict__ p, int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * kVecThreads + threadIdx.x;
  if (k >= n || (mode && S[kSDone] != 0.0)) return;
  p[k] = mode ? fma(S[kSBeta], p[k], z[k]) : z[k];
}

// Fixed-order block reduction of `nparts` partials with stride `stride` (offset `off`): thread t sums
// partials t, t + 1024, ... in order, then a shared-memory tree (deterministic for a given nparts).
constexpr int kRedThreads = 1024;
__device__ __forceinline__ double block_sum(const double* __restrict__ part, int nparts, int stride, int off,
                                            double* sh) {
  double s = 0.0;
  for (int k = threadIdx.x; k < nparts; k += kRedThreads) s += part[(int64_t)k * stride + off];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kRedThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// which: 0 = after the product (alpha = rz / pq), 1 = after the update (beta, convergence), 2 = initial
__global__ void __launch_bounds__(kRedThreads) k_cg_scalar(int which, double* __restrict__ S,
                                                           const double* __restrict__ part, int nparts, double rtol2) {
  __shared__ double sh[kRedThreads];
  if (which != 2 && S[kSDone] != 0.0) return;   // uniform over the block
  if (which == 0) {
    const double pq = block_sum(part, nparts, 1, 0, sh);
    if (threadIdx.x == 0) {
      S[kSAlpha] = (pq > 0.0) ? S[kSRz] / pq : 0.0;
      if (!(pq > 0.0)) S[kSDone] = 2.0;   // not SPD along p (or p = 0)
    }
    return;
  }
  const double rz = block_sum(part, nparts, 2, 0, sh);
  const double rr = block_sum(part, nparts, 2, 1, sh);
  if (threadIdx.x != 0) return;
  if (which == 2) {
    S[kSRz] = rz; S[kSRr] = rr; S[kSRr0] = rr; S[kSIter] = 0.0;
    S[kSDone] = (rr == 0.0) ? 1.0 : 0.0;
    return;
  }
  S[kSBeta] = (S[kSRz] != 0.0) ? rz / S[kSRz] : 0.0;
  S[kSRz] = rz;
  S[kSRr] = rr;
  S[kSIter] += 1.0;
  if (rr <= rtol2 * S[kSBnorm2]) S[kSDone] = 1.0;
  else if (S[kSIter] >= S[kSMaxIt]) S[kSDone] = 3.0;   // iteration budget spent
}

__global__ void __launch_bounds__(kVecThreads) k_dot(const double* __restrict__ u, const double* __restrict__ v, int64_t n,
                                                     double* __restrict__ part) {
  __shared__ double red[kVecThreads / 32];
  double s = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * kVecThreads + threadIdx.x; k < n; k += (int64_t)gridDim.x * kVecThreads)
    s = fma(u[k], v[k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kVecThreads / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kRedThreads) k_set_bnorm(double* __restrict__ S, const double* __restrict__ part,
                                                           int nparts, double max_iter) {
  __shared__ double sh[kRedThreads];
  const double s = block_sum(part, nparts, 1, 0, sh);
  if (threadIdx.x == 0) { S[kSBnorm2] = s; S[kSMaxIt] = max_iter; }
}

// r = b - r (r holds A x)
__global__ void __launch_bounds__(kVecThreads) k_residual(const double* __restrict__ b, double* __restrict__ r, int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * kVecThreads + threadIdx.x;
  if (k < n) r[k] = b[k] - r[k];
}

// Gershgorin discs of the scalar rows: lo = min_i (a_ii - R_i), hi = max_i (a_ii + R_i); one warp per block row
__global__ void __launch_bounds__(32 * kWarpsPerBlk) k_gersh(const int32_t* __restrict__ row_ptr,
                                                             const int32_t* __restrict__ col_idx,
                                                             const double* __restrict__ vals, int nrows, int g0,
                                                             double* __restrict__ part) {
  __shared__ double red[2][kWarpsPerBlk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x * kWarpsPerBlk + warp;
  double lo = INFINITY, hi = -INFINITY;
  if (a < nrows) {
    double R[3] = {0, 0, 0}, dg[3] = {0, 0, 0};
    for (int q = row_ptr[a] + lane; q < row_ptr[a + 1]; q += 32) {
      const double* h = vals + (int64_t)q * 9;
      const bool isd = col_idx[q] == g0 + a;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (isd && r == c) dg[r] = h[4 * r];
          else R[r] += fabs(h[3 * r + c]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        R[r] += __shfl_xor_sync(0xffffffffu, R[r], o);
        dg[r] += __shfl_xor_sync(0xffffffffu, dg[r], o);
      }
#pragma unroll
    for (int r = 0; r < 3; ++r) { lo = fmin(lo, dg[r] - R[r]); hi = fmax(hi, dg[r] + R[r]); }
  }
  if (lane == 0) { red[0][warp] = lo; red[1][warp] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kWarpsPerBlk; ++w) { lo = fmin(lo, red[0][w]); hi = fmax(hi, red[1][w]); }
    part[2 * blockIdx.x] = lo;
    part[2 * blockIdx.x + 1] = hi;
  }
}

}  // namespace

int spmv(const SolveArgs& A, const double* d_vals, const double* d_x, double* d_y, double* dot_part, cudaStream_t st) {
  const int nb = (A.nrows + kWarpsPerBlk - 1) / kWarpsPerBlk;
  if (nb == 0) return 0;
  k_spmv<<<nb, 32 * kWarpsPerBlk, 0, st>>>(A.row_ptr, A.col_idx, d_vals, d_x, d_y, A.nrows, A.n_u, A.r0, A.xlo, dot_part);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

int gershgorin(const SolveArgs& A, const double* d_vals, double* d_part, double* lo, double* hi, cudaStream_t st) {
  const int nb = (A.nrows + kWarpsPerBlk - 1) / kWarpsPerBlk;
  if (nb == 0) { *lo = *hi = 0.0; return 0; }
  k_gersh<<<nb, 32 * kWarpsPerBlk, 0, st>>>(A.row_ptr, A.col_idx, d_vals, A.nrows, A.r0 * A.n_u, d_part);
  if (cudaPeekAtLastError() != cudaSuccess) return -6;
  std::vector<double> h(2 * (size_t)nb);
  if (cudaMemcpyAsync(h.data(), d_part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return -6;
  double l = INFINITY, u = -INFINITY;
  for (int k = 0; k < nb; ++k) { l = std::fmin(l, h[2 * k]); u = std::fmax(u, h[2 * k + 1]); }
  *lo = l; *hi = u;
  return 0;
}

int solve_parts(int nrows) {
  const int a = (nrows + kWarpsPerBlk - 1) / kWarpsPerBlk, b = (nrows + kVecThreads - 1) / kVecThreads;
  return 2 * (a > b ? a : b) + 64;
}

int pcg(const SolveArgs& A, const double* d_vals, const double* d_b, double* d_x, const CgWork& W, int max_iter,
        double rtol, int check_every, int* iters, double* relres, int* status, cudaStream_t st) {
  const int n3 = 3 * A.nrows;
  const int nbv = (A.nrows + kVecThreads - 1) / kVecThreads;
  const int nbs = (A.nrows + kWarpsPerBlk - 1) / kWarpsPerBlk;
  const int nbn = (n3 + kVecThreads - 1) / kVecThreads;
  if (cudaMemsetAsync(W.bad, 0, sizeof(int), st) != cudaSuccess) return -6;
  k_diag_inv<<<(A.nrows + 127) / 128, 128, 0, st>>>(A.diag, d_vals, W.dinv, A.nrows, W.bad);
  // |b|^2
  k_dot<<<nbv, kVecThreads, 0, st>>>(d_b, d_b, n3, W.part);
  k_set_bnorm<<<1, kRedThreads, 0, st>>>(W.S, W.part, nbv, (double)max_iter);
  // r = b - A x, z = D^-1 r, p = z
  if (spmv(A, d_vals, d_x, W.r, nullptr, st)) return -6;
  k_residual<<<nbn, kVecThreads, 0, st>>>(d_b, W.r, n3);
  k_cg_update<<<nbv, kVecThreads, 0, st>>>(0, W.S, d_x, W.p, W.q, W.r, W.z, W.dinv, A.nrows, W.part);
  k_cg_scalar<<<1, kRedThreads, 0, st>>>(2, W.S, W.part, nbv, rtol * rtol);
  k_cg_dir<<<nbn, kVecThreads, 0, st>>>(0, W.S, W.z, W.p, n3);
  // iterations in chunks of check_every, recorded once as a CUDA graph on an internal stream (one launch
  // per chunk instead of 5 per iteration; after convergence or the budget the kernels return at once)
  auto chunk = [&](cudaStream_t s) {
    for (int k = 0; k < check_every; ++k) {
      spmv(A, d_vals, W.p, W.q, W.part, s);   // q = A p, partials of p.q
      k_cg_scalar<<<1, kRedThreads, 0, s>>>(0, W.S, W.part, nbs, rtol * rtol);
      k_cg_update<<<nbv, kVecThreads, 0, s>>>(1, W.S, d_x, W.p, W.q, W.r, W.z, W.dinv, A.nrows, W.part);
      k_cg_scalar<<<1, kRedThreads, 0, s>>>(1, W.S, W.part, nbv, rtol * rtol);
      k_cg_dir<<<nbn, kVecThreads, 0, s>>>(1, W.S, W.z, W.p, n3);
    }
  };
  CgGraph* Gr = W.graph;
  cudaStream_t run = st;
  if (Gr) {
    if (!Gr->cs && (cudaStreamCreateWithFlags(&Gr->cs, cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&Gr->e0, cudaEventDisableTiming) != cudaSuccess ||
                    cudaEventCreateWithFlags(&Gr->e1, cudaEventDisableTiming) != cudaSuccess))
      return -6;
    const bool same = Gr->exec && Gr->key[0] == d_vals && Gr->key[1] == d_b && Gr->key[2] == d_x &&
                      Gr->key_rtol == rtol && Gr->key_max == check_every;
    if (!same) {
      if (Gr->exec) { cudaGraphExecDestroy(Gr->exec); Gr->exec = nullptr; }
      cudaGraph_t g = nullptr;
      if (cudaStreamBeginCapture(Gr->cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return -6;
      chunk(Gr->cs);
      if (cudaStreamEndCapture(Gr->cs, &g) != cudaSuccess) return -6;
      const cudaError_t ie = cudaGraphInstantiate(&Gr->exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) { Gr->exec = nullptr; return -6; }
      Gr->key[0] = d_vals; Gr->key[1] = d_b; Gr->key[2] = d_x; Gr->key_rtol = rtol; Gr->key_max = check_every;
    }
    if (cudaEventRecord(Gr->e0, st) != cudaSuccess || cudaStreamWaitEvent(Gr->cs, Gr->e0, 0) != cudaSuccess) return -6;
    run = Gr->cs;
  }
  double hs[kSN];
  *status = 0;
  for (int it = 0;; it += check_every) {
    if (max_iter <= 0) {   // no iterations: report the initial residual
      if (cudaMemcpyAsync(hs, W.S, sizeof(hs), cudaMemcpyDeviceToHost, run) != cudaSuccess ||
          cudaStreamSynchronize(run) != cudaSuccess)
        return -6;
      break;
    }
    if (Gr) { if (cudaGraphLaunch(Gr->exec, run) != cudaSuccess) return -6; }
    else chunk(run);
    if (cudaPeekAtLastError() != cudaSuccess) return -6;
    if (cudaMemcpyAsync(hs, W.S, sizeof(hs), cudaMemcpyDeviceToHost, run) != cudaSuccess ||
        cudaStreamSynchronize(run) != cudaSuccess)
      return -6;
    if (hs[kSDone] != 0.0 || it + check_every >= max_iter) break;
  }
  if (Gr && (cudaEventRecord(Gr->e1, run) != cudaSuccess || cudaStreamWaitEvent(st, Gr->e1, 0) != cudaSuccess))
    return -6;
  // the diagonal-block check ran on st before the iterations, which `run` has been synchronised behind
  int bad = 0;
  if (cudaMemcpyAsync(&bad, W.bad, sizeof(int), cudaMemcpyDeviceToHost, run) != cudaSuccess ||
      cudaStreamSynchronize(run) != cudaSuccess)
    return -6;
  *iters = (int)hs[kSIter];
  *relres = hs[kSBnorm2] > 0.0 ? std::sqrt(hs[kSRr] / hs[kSBnorm2]) : 0.0;
  // 0 converged, 1 iteration budget spent, 2 not SPD
  *status = (hs[kSDone] == 1.0 || hs[kSRr] == 0.0) ? 0 : ((hs[kSDone] == 2.0 || bad) ? 2 : 1);
  return 0;
}

}  // namespace bsf
