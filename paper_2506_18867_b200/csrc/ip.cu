// Incremental-potential epilogue (Q13/Q14).
//
// After the elastic assembly of a batch, per owned control point a and item:
//   E  += m_a/(2 dt^2) |x_a - xhat_a|^2 - m_a g.x_a        (lumped mass PAPER.md:613-615)
//   g_a += m_a/dt^2 (x_a - xhat_a) - m_a g
//   H_aa += m_a/dt^2 I3                                      (diagonal block, always in the pattern)
// then the pinned control points are eliminated (gradient rows 0; Hessian rows and columns 0, diagonal
// block I3).  One thread per (control point, item); the energy partials are summed per item in a fixed
// order (deterministic).  Bytes per control point: x, xhat, m, g (read + write) and 3 diagonal doubles.
#include <cuda_runtime.h>

#include "ip.hpp"

namespace bsf {

namespace {

constexpr int kIpThreads = 256;

__global__ void __launch_bounds__(kIpThreads) k_ip(IpArgs A) {
  __shared__ double red[kIpThreads / 32];
  const int a = blockIdx.x * kIpThreads + threadIdx.x, item = blockIdx.y;
  double e = 0.0;
  if (a < A.ncp) {
    const int j = a / A.n_u, i = a - j * A.n_u;   // owned-row index j (row r0 + j)
    const double* x = A.x + item * A.xs + ((int64_t)(j + A.r0 - A.xlo) * A.n_u + i) * 3;
    const double* xh = A.xhat + item * A.xhs + (int64_t)a * 3;
    const double msc = A.params ? A.params[9 * (int64_t)item + 4] / A.detJ_ref : 1.0;   // per-item det J
    const double m = A.mass[a] * msc, km = A.k * m;
    double d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      d[c] = x[c] - xh[c];
      e = fma(0.5 * km * d[c], d[c], e);
      e = fma(-m * A.grav[c], x[c], e);
    }
    if (A.g) {
      double* g = A.g + item * A.gs + (int64_t)a * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) g[c] += km * d[c] - m * A.grav[c];
    }
    if (A.vals) {
      double* blk = A.vals + item * A.vs + (int64_t)A.diag[a] * 9;
      blk[0] += km;
      blk[4] += km;
      blk[8] += km;
    }
  }
  if (!A.epart) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kIpThreads / 32; ++w) s += red[w];
    A.epart[(int64_t)item * gridDim.x + blockIdx.x] = s;
  }
}

// pinned elimination: tasks [0, nzero) zero a block, [nzero, nzero + npin) set the diagonal block of a pinned
// row to I3 and zero its gradient row
__global__ void __launch_bounds__(kIpThreads) k_ip_pin(IpArgs A) {
  const int t = blockIdx.x * kIpThreads + threadIdx.x, item = blockIdx.y;
  if (t < A.nzero) {
    if (A.vals) {
      double* blk = A.vals + item * A.vs + (int64_t)A.zero_blk[t] * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) blk[k] = 0.0;
    }
  } else if (t < A.nzero + A.npin) {
    const int p = t - A.nzero;
    if (A.vals) {
      double* blk = A.vals + item * A.vs + (int64_t)A.diag[A.pin_cp[p]] * 9;
#pragma unroll
      for (int k = 0; k < 9; ++k) blk[k] = (k % 4 == 0) ? 1.0 : 0.0;
    }
    if (A.g) {
      double* g = A.g + item * A.gs + (int64_t)A.pin_cp[p] * 3;
      g[0] = g[1] = g[2] = 0.0;
    }
  }
}

__global__ void __launch_bounds__(256) k_ip_energy(const double* __restrict__ epart, int per_item, double* E) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int k = 0; k < per_item; ++k) s += epart[(int64_t)blockIdx.x * per_item + k];
  E[blockIdx.x] += s;
}

}  // namespace

int ip_eval(IpArgs A, int nbatch, double* d_energy, cudaStream_t st, int* launches) {
  int nl = 0;
  const int nblk = (A.ncp + kIpThreads - 1) / kIpThreads;
  if (nblk == 0 || nbatch == 0) return 0;
  if (!d_energy) A.epart = nullptr;
  k_ip<<<dim3(nblk, nbatch), kIpThreads, 0, st>>>(A);
  ++nl;
  if (A.nzero + A.npin > 0 && (A.vals || A.g)) {
    k_ip_pin<<<dim3((A.nzero + A.npin + kIpThreads - 1) / kIpThreads, nbatch), kIpThreads, 0, st>>>(A);
    ++nl;
  }
  if (d_energy) {
    k_ip_energy<<<nbatch, 32, 0, st>>>(A.epart, nblk, d_energy);
    ++nl;
  }
  if (launches) *launches = nl;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

int ip_pin(IpArgs A, int nbatch, cudaStream_t st, int* launches) {
  if (launches) *launches = 0;
  if (A.nzero + A.npin == 0 || nbatch == 0 || !(A.vals || A.g)) return 0;
  k_ip_pin<<<dim3((A.nzero + A.npin + kIpThreads - 1) / kIpThreads, nbatch), kIpThreads, 0, st>>>(A);
  if (launches) *launches = 1;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

int ip_partials(int ncp) { return (ncp + kIpThreads - 1) / kIpThreads; }

}  // namespace bsf
