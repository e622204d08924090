// BSR products, the Gershgorin bound and block-Jacobi PCG on the assembled Hessian (solve.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace bsf {

struct SolveArgs {
  const int32_t* row_ptr;   // owned block rows (device)
  const int32_t* col_idx;
  const int32_t* diag;      // block index of (a, a) per owned row (PCG only)
  int nrows, n_u, r0, xlo;
};

// device scalar slots of the PCG
enum { kSRz = 0, kSRr, kSRr0, kSAlpha, kSBeta, kSDone, kSIter, kSBnorm2, kSMaxIt, kSN };

// CUDA graph of a chunk of PCG iterations (replayed until convergence; rebuilt when the operands change)
struct CgGraph {
  cudaStream_t cs = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaGraphExec_t exec = nullptr;
  const void* key[3] = {nullptr, nullptr, nullptr};
  double key_rtol = 0.0;
  int key_max = 0;
};

struct CgWork {
  CgGraph* graph = nullptr;   // owned by the handle
  double *r, *z, *p, *q;   // [3 nrows] each
  double* dinv;            // [nrows][9]
  double* part;            // [solve_parts(nrows)] partial sums
  double* S;               // [kSN]
  int* bad;                // non-positive diagonal block determinant seen
};

int spmv(const SolveArgs& A, const double* d_vals, const double* d_x, double* d_y, double* dot_part, cudaStream_t st);
int gershgorin(const SolveArgs& A, const double* d_vals, double* d_part, double* lo, double* hi, cudaStream_t st);
int solve_parts(int nrows);
// Solves H x = b (in: initial guess in d_x); status 0 converged (|r| <= rtol |b|), 1 max_iter reached,
// 2 not SPD (p.Hp <= 0 or a diagonal block not positive definite).  Synchronises `st` every check_every
// iterations to test convergence.
int pcg(const SolveArgs& A, const double* d_vals, const double* d_b, double* d_x, const CgWork& W, int max_iter,
        double rtol, int check_every, int* iters, double* relres, int* status, cudaStream_t st);

}  // namespace bsf
