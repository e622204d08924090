// Banded Cholesky of the assembled Hessian and the Gershgorin-gated Neumann split (chol.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace bsf {

struct CholState {
  bool ready = false, factored = false;
  int64_t n = 0, kd = 0, nb = 0, ldab = 0, nnzb = 0;
  int lwork = 0, npanels = 0;
  double* ab = nullptr;       // [n][ldab] lower band (+ nb zero rows)
  double* work = nullptr;     // potrf workspace
  int* info = nullptr;        // [npanels] potrf status per panel
  int32_t* brow = nullptr;    // [nnzb] block row of every block
  double* tmp = nullptr;      // [n]
  double* part = nullptr;     // reduction partials
  void* blas = nullptr;       // cublasHandle_t
  void* dn = nullptr;         // cusolverDnHandle_t
  double lam_min_D = 0.0;     // Gershgorin lower bound of the factorised matrix's spectrum
};

using SpmvFn = std::function<int(const double* x, double* y, cudaStream_t st)>;

int chol_setup(CholState& C, const std::vector<int32_t>& row_ptr, const std::vector<int32_t>& col_idx, int nrows,
               size_t max_bytes, std::string& err);
int chol_factor(CholState& C, const int32_t* d_col_idx, const double* d_vals, cudaStream_t st, std::string& err);
int chol_solve(CholState& C, const double* d_b, double* d_x, cudaStream_t st, std::string& err);
int neumann_solve(CholState& C, const SpmvFn& spmv_b, const double* d_b, double* d_x, int max_terms, double rtol,
                  int* terms, double* step, cudaStream_t st, std::string& err);
void chol_free(CholState& C);

}  // namespace bsf
