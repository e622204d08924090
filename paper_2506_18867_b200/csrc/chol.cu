// Direct solve of the Newton system on the device ("projected Newton" with a
// Cholesky factorisation, PAPER.md:857-890 the Neumann split gated by a Gershgorin bound).
//
// The assembled Hessian of a whole sheet is banded in the control-point-major DOF order (a = j n_u + i, DOF
// 3a + r): every block couples control points at most 2 n_u + 1 apart, so the half-bandwidth is
// kd = max over the pattern of 3 (a - b) + 2 (= 6 n_u + 5 for the reduced rules).  Cholesky keeps that band
// (no fill outside it), so the factor is stored as a lower band [N][ldab] (element (i, j), i >= j, at
// ab[(i - j) + j ldab]) with ldab = kd + nb + 1: the nb extra rows of zeros make every panel rectangle of the
// blocked right-looking algorithm a plain column-major matrix with leading dimension ldab - 1 (the LAPACK
// dpbtrf view), so the panel steps are the library calls potrf (diagonal block), trsm (the kd rows below it)
// and syrk (their rank-nb update of the trailing band).  Solves walk the same panels (trsv on the diagonal
// block, gemv with the rows below it).
// cuBLAS / cuSOLVER are loaded at run time from the process (torch ships both), like NCCL (halo.cpp).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "chol.hpp"

namespace bsf {

namespace {

struct Lib {
  bool ok = false;
  std::string err;
  decltype(&cublasCreate_v2) create = nullptr;
  decltype(&cublasDestroy_v2) destroy = nullptr;
  decltype(&cublasSetStream_v2) set_stream = nullptr;
  decltype(&cublasDtrsm_v2) trsm = nullptr;
  decltype(&cublasDsyrk_v2) syrk = nullptr;
  decltype(&cublasDtbsv_v2) tbsv = nullptr;
  decltype(&cublasDtrsv_v2) trsv = nullptr;
  decltype(&cublasDgemv_v2) gemv = nullptr;
  decltype(&cusolverDnCreate) s_create = nullptr;
  decltype(&cusolverDnDestroy) s_destroy = nullptr;
  decltype(&cusolverDnSetStream) s_set_stream = nullptr;
  decltype(&cusolverDnDpotrf_bufferSize) potrf_buf = nullptr;
  decltype(&cusolverDnDpotrf) potrf = nullptr;
};

const Lib& lib() {
  static Lib L;
  static std::once_flag once;
  std::call_once(once, [] {
    auto open = [](const char* a, const char* b) {
      void* h = dlopen(a, RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen(a, RTLD_NOW | RTLD_GLOBAL);
      if (!h && b) h = dlopen(b, RTLD_NOW | RTLD_GLOBAL);
      return h;
    };
    void* hb = open("libcublas.so.12", "libcublas.so");
    void* hs = open("libcusolver.so.11", "libcusolver.so");
    if (!hb || !hs) { L.err = std::string("cannot load cuBLAS / cuSOLVER: ") + dlerror(); return; }
#define BSF_SYM(h, f, n) L.f = reinterpret_cast<decltype(L.f)>(dlsym(h, n))
    BSF_SYM(hb, create, "cublasCreate_v2");
    BSF_SYM(hb, destroy, "cublasDestroy_v2");
    BSF_SYM(hb, set_stream, "cublasSetStream_v2");
    BSF_SYM(hb, trsm, "cublasDtrsm_v2");
    BSF_SYM(hb, syrk, "cublasDsyrk_v2");
    BSF_SYM(hb, tbsv, "cublasDtbsv_v2");
    BSF_SYM(hb, trsv, "cublasDtrsv_v2");
    BSF_SYM(hb, gemv, "cublasDgemv_v2");
    BSF_SYM(hs, s_create, "cusolverDnCreate");
    BSF_SYM(hs, s_destroy, "cusolverDnDestroy");
    BSF_SYM(hs, s_set_stream, "cusolverDnSetStream");
    BSF_SYM(hs, potrf_buf, "cusolverDnDpotrf_bufferSize");
    BSF_SYM(hs, potrf, "cusolverDnDpotrf");
#undef BSF_SYM
    L.ok = L.create && L.destroy && L.set_stream && L.trsm && L.syrk && L.tbsv && L.trsv && L.gemv && L.s_create &&
           L.s_destroy &&
           L.s_set_stream && L.potrf_buf && L.potrf;
    if (!L.ok) L.err = "cuBLAS / cuSOLVER lack a required symbol";
  });
  return L;
}

// Lower band of the BSR values: entry (3a + r, 3b + c) with 3a + r >= 3b + c goes to ab[(i - j) + j ldab].
__global__ void k_bsr_to_band(const int32_t* __restrict__ brow, const int32_t* __restrict__ col_idx,
                              const double* __restrict__ vals, int64_t nnzb, double* __restrict__ ab, int64_t ldab) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnzb * 9) return;
  const int64_t k = t / 9;
  const int rc = (int)(t - 9 * k), r = rc / 3, c = rc - 3 * (rc / 3);
  const int64_t i = 3 * (int64_t)brow[k] + r, j = 3 * (int64_t)col_idx[k] + c;
  if (i >= j) ab[(i - j) + j * ldab] = vals[t];
}

// y = b - y   (Neumann / fixed-point residual)
__global__ void k_sub_from(const double* __restrict__ b, double* __restrict__ y, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) y[t] = b[t] - y[t];
}

// part[blk] = (sum (x - y)^2, sum x^2) over the block's entries; x <- y afterwards
__global__ void k_step_norm(double* __restrict__ x, const double* __restrict__ y, int64_t n, double* __restrict__ part) {
  __shared__ double s0[256], s1[256];
  double d2 = 0.0, x2 = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double d = y[t] - x[t];
    d2 += d * d;
    x2 += y[t] * y[t];
    x[t] = y[t];
  }
  s0[threadIdx.x] = d2;
  s1[threadIdx.x] = x2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) { s0[threadIdx.x] += s0[threadIdx.x + o]; s1[threadIdx.x] += s1[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = s0[0]; part[2 * blockIdx.x + 1] = s1[0]; }
}

}  // namespace

void chol_free(CholState& C) {
  const Lib& L = lib();
  if (C.blas && L.ok) L.destroy(static_cast<cublasHandle_t>(C.blas));
  if (C.dn && L.ok) L.s_destroy(static_cast<cusolverDnHandle_t>(C.dn));
  for (void* p : {(void*)C.ab, (void*)C.work, (void*)C.info, (void*)C.brow, (void*)C.tmp, (void*)C.part}) cudaFree(p);
  C = CholState();
}

int chol_setup(CholState& C, const std::vector<int32_t>& row_ptr, const std::vector<int32_t>& col_idx, int nrows,
               size_t max_bytes, std::string& err) {
  const Lib& L = lib();
  if (!L.ok) { err = L.err; return -6; }
  if (C.ready) return 0;
  // half-bandwidth of the pattern in DOFs
  int64_t kd = 0;
  std::vector<int32_t> brow(col_idx.size());
  for (int a = 0; a < nrows; ++a)
    for (int32_t k = row_ptr[a]; k < row_ptr[a + 1]; ++k) {
      brow[k] = a;
      kd = std::max<int64_t>(kd, 3 * (int64_t)(a - col_idx[k]) + 2);
    }
  C.n = 3 * (int64_t)nrows;
  C.kd = kd;
  static const int nb_env = getenv("BSF_CHOL_NB") ? atoi(getenv("BSF_CHOL_NB")) : 0;
  C.nb = nb_env > 0 ? nb_env : 512;   // measured: 128 / 256 / 512 give the same factor time, the solve 50 / 27 / 16 ms on C2
  C.ldab = kd + C.nb + 1;
  const size_t bytes = sizeof(double) * (size_t)C.n * (size_t)C.ldab;
  if (bytes > max_bytes) {
    err = "banded factor needs " + std::to_string(bytes >> 20) + " MiB (half-bandwidth " + std::to_string(kd) +
          " DOFs), above the limit";
    return -7;
  }
  C.npanels = (int)((C.n + C.nb - 1) / C.nb);
  if (cudaMalloc(&C.ab, bytes) != cudaSuccess || cudaMalloc(&C.info, sizeof(int) * C.npanels) != cudaSuccess ||
      cudaMalloc(&C.brow, sizeof(int32_t) * brow.size()) != cudaSuccess ||
      cudaMalloc(&C.tmp, sizeof(double) * (size_t)C.n) != cudaSuccess ||
      cudaMalloc(&C.part, sizeof(double) * 2 * 1024) != cudaSuccess) {
    cudaGetLastError();
    chol_free(C);
    err = "cudaMalloc failed (banded factor)";
    return -7;
  }
  if (cudaMemcpy(C.brow, brow.data(), sizeof(int32_t) * brow.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    chol_free(C);
    err = "upload failed";
    return -6;
  }
  cublasHandle_t hb = nullptr;
  cusolverDnHandle_t hs = nullptr;
  if (L.create(&hb) != CUBLAS_STATUS_SUCCESS || L.s_create(&hs) != CUSOLVER_STATUS_SUCCESS) {
    chol_free(C);
    err = "cuBLAS / cuSOLVER handle creation failed";
    return -6;
  }
  C.blas = hb;
  C.dn = hs;
  int lwork = 0;
  if (L.potrf_buf(hs, CUBLAS_FILL_MODE_LOWER, (int)std::min<int64_t>(C.nb, C.n), C.ab, (int)(C.ldab - 1), &lwork) !=
          CUSOLVER_STATUS_SUCCESS ||
      cudaMalloc(&C.work, sizeof(double) * std::max(lwork, 1)) != cudaSuccess) {
    chol_free(C);
    err = "potrf workspace";
    return -6;
  }
  C.lwork = lwork;
  C.nnzb = (int64_t)col_idx.size();
  C.ready = true;
  return 0;
}

int chol_factor(CholState& C, const int32_t* d_col_idx, const double* d_vals, cudaStream_t st, std::string& err) {
  const Lib& L = lib();
  auto hb = static_cast<cublasHandle_t>(C.blas);
  auto hs = static_cast<cusolverDnHandle_t>(C.dn);
  C.factored = false;
  if (cudaMemsetAsync(C.ab, 0, sizeof(double) * (size_t)C.n * (size_t)C.ldab, st) != cudaSuccess ||
      cudaMemsetAsync(C.info, 0, sizeof(int) * C.npanels, st) != cudaSuccess) { err = "memset"; return -6; }
  const int64_t nt = C.nnzb * 9;
  k_bsr_to_band<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(C.brow, d_col_idx, d_vals, C.nnzb, C.ab, C.ldab);
  if (L.set_stream(hb, st) != CUBLAS_STATUS_SUCCESS || L.s_set_stream(hs, st) != CUSOLVER_STATUS_SUCCESS) {
    err = "set stream";
    return -6;
  }
  const int lda = (int)(C.ldab - 1);
  const double one = 1.0, mone = -1.0;
  for (int64_t j0 = 0; j0 < C.n; j0 += C.nb) {
    const int jb = (int)std::min<int64_t>(C.nb, C.n - j0);
    double* a11 = C.ab + j0 * C.ldab;   // (j0, j0)
    if (L.potrf(hs, CUBLAS_FILL_MODE_LOWER, jb, a11, lda, C.work, C.lwork, C.info + j0 / C.nb) !=
        CUSOLVER_STATUS_SUCCESS) {
      err = "potrf failed";
      return -6;
    }
    const int i2 = (int)std::min<int64_t>(C.kd, C.n - j0 - jb);
    if (i2 <= 0) continue;
    double* a21 = a11 + jb;                       // (j0 + jb, j0)
    double* a22 = C.ab + (j0 + jb) * C.ldab;      // (j0 + jb, j0 + jb)
    if (L.trsm(hb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, i2, jb, &one, a11,
               lda, a21, lda) != CUBLAS_STATUS_SUCCESS ||
        L.syrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, i2, jb, &mone, a21, lda, &one, a22, lda) !=
            CUBLAS_STATUS_SUCCESS) {
      err = "trsm / syrk failed";
      return -6;
    }
  }
  std::vector<int> info(C.npanels);
  if (cudaMemcpyAsync(info.data(), C.info, sizeof(int) * C.npanels, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    err = "factorisation did not complete";
    return -6;
  }
  for (int p = 0; p < C.npanels; ++p)
    if (info[p] != 0) {   // potrf: the leading minor of that order of the panel's updated block is not positive
      err = "matrix not positive definite (pivot " + std::to_string((int64_t)p * C.nb + info[p] - 1) + ")";
      return -1;
    }
  C.factored = true;
  return 0;
}

int chol_solve(CholState& C, const double* d_b, double* d_x, cudaStream_t st, std::string& err) {
  const Lib& L = lib();
  if (!C.factored) { err = "no factorisation (bsf_chol_factor)"; return -1; }
  auto hb = static_cast<cublasHandle_t>(C.blas);
  if (d_x != d_b && cudaMemcpyAsync(d_x, d_b, sizeof(double) * (size_t)C.n, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    err = "copy";
    return -6;
  }
  if (L.set_stream(hb, st) != CUBLAS_STATUS_SUCCESS) { err = "set stream"; return -6; }
  // blocked banded triangular solves over the factor's panels (the dense views of the factorisation): forward
  // L y = b: y1 = L11^-1 y1, y2 -= A21 y1; backward L^T x = y: x1 -= A21^T x2, x1 = L11^-T x1
  const int lda = (int)(C.ldab - 1);
  const double one = 1.0, mone = -1.0;
  for (int64_t j0 = 0; j0 < C.n; j0 += C.nb) {
    const int jb = (int)std::min<int64_t>(C.nb, C.n - j0);
    const int i2 = (int)std::min<int64_t>(C.kd, C.n - j0 - jb);
    const double* a11 = C.ab + j0 * C.ldab;
    if (L.trsv(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, jb, a11, lda, d_x + j0, 1) !=
            CUBLAS_STATUS_SUCCESS ||
        (i2 > 0 && L.gemv(hb, CUBLAS_OP_N, i2, jb, &mone, a11 + jb, lda, d_x + j0, 1, &one, d_x + j0 + jb, 1) !=
                       CUBLAS_STATUS_SUCCESS)) {
      err = "forward solve failed";
      return -6;
    }
  }
  for (int64_t p = (C.n + C.nb - 1) / C.nb - 1; p >= 0; --p) {
    const int64_t j0 = p * C.nb;
    const int jb = (int)std::min<int64_t>(C.nb, C.n - j0);
    const int i2 = (int)std::min<int64_t>(C.kd, C.n - j0 - jb);
    const double* a11 = C.ab + j0 * C.ldab;
    if ((i2 > 0 && L.gemv(hb, CUBLAS_OP_T, i2, jb, &mone, a11 + jb, lda, d_x + j0 + jb, 1, &one, d_x + j0, 1) !=
                       CUBLAS_STATUS_SUCCESS) ||
        L.trsv(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, jb, a11, lda, d_x + j0, 1) !=
            CUBLAS_STATUS_SUCCESS) {
      err = "backward solve failed";
      return -6;
    }
  }
  return 0;
}

int neumann_solve(CholState& C, const SpmvFn& spmv_b, const double* d_b, double* d_x, int max_terms, double rtol,
                  int* terms, double* step, cudaStream_t st, std::string& err) {
  // x_0 = D^-1 b; x_{k+1} = D^-1 (b - B x_k): the partial sums of sum_k (-D^-1 B)^k D^-1 b (PAPER.md Eq.
  // `eq: Neumann expansion`), stopped when |x_{k+1} - x_k| <= rtol |x_{k+1}|
  if (chol_solve(C, d_b, d_x, st, err)) return -6;
  const int nblk = (int)std::min<int64_t>(1024, (C.n + 255) / 256);
  std::vector<double> h(2 * (size_t)nblk);
  int k = 0;
  double rel = 0.0;
  for (; k < max_terms; ++k) {
    if (spmv_b(d_x, C.tmp, st)) { err = "spmv"; return -6; }
    k_sub_from<<<(unsigned)((C.n + 255) / 256), 256, 0, st>>>(d_b, C.tmp, C.n);
    if (chol_solve(C, C.tmp, C.tmp, st, err)) return -6;
    k_step_norm<<<nblk, 256, 0, st>>>(d_x, C.tmp, C.n, C.part);
    if (cudaMemcpyAsync(h.data(), C.part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      err = "sync";
      return -6;
    }
    double d2 = 0.0, x2 = 0.0;
    for (int b = 0; b < nblk; ++b) { d2 += h[2 * b]; x2 += h[2 * b + 1]; }
    rel = x2 > 0.0 ? std::sqrt(d2 / x2) : std::sqrt(d2);
    if (rel <= rtol) { ++k; break; }
  }
  if (terms) *terms = k;
  if (step) *step = rel;
  return 0;
}

}  // namespace bsf
