// k_g3: the G3-FULL rule (3x3 Gauss on every span for both energies, SURVEY §8(c).2 "G3-FULL", the paper's
// full-quadrature baseline) on affine sheets (g3.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "dev.hpp"
#include "host.hpp"

namespace bsf {

namespace g3 {
constexpr int kW = 16;          // control-point columns per CTA strip (2 rows x 16 = the 32 lanes)
constexpr int kSC = 18;         // span columns of a strip window: [i0 - 2, i0 + 16)
constexpr int kNG = 9;          // Gauss nodes per span (gu + 3 gv)
constexpr int kCh = 30;         // record channels: A~uu (6), A~vv (6), A~uv (9), P~u (3), P~v (3), w mu Lap phi (3)
constexpr int kSlots = 4;       // span-row ring
constexpr int kThreads = 512;
constexpr int kMaxCls = 8;      // 1D span classes per direction (5 for S >= 5)
constexpr int kBetaParts = 6;   // bending Hessian parts (cuu^2, cvv^2, cuv^2, cuu cvv, cuu cuv, cvv cuv)
}  // namespace g3

struct G3Tables {
  int ok = 0;
  int n_u = 0, n_v = 0, Su = 0, Sv = 0, r0 = 0, r1 = 0, xlo = 0, xhi = 0, tlo = 0, thi = 0;
  int ncls_u = 0, ncls_v = 0, cint_u = -1, cint_v = -1;
  double G[4] = {0, 0, 0, 0}, detJ = 1.0;
  double what[g3::kNG] = {};
  double utab[g3::kMaxCls * 27] = {}, vtab[g3::kMaxCls * 27] = {};   // [cls][g][N | d1 | d2][e]
  double* d_tabs = nullptr;        // device copy of utab | vtab
  int8_t* ucls = nullptr;          // device [Su]: 1D class of each span column
  int8_t* vcls = nullptr;          // device [Sv]: of each span row (-1 outside the slab window)
  double* beta = nullptr;          // device [9 x 9 cp classes][6][25]: parametric bending Hessian parts
  int32_t* row_ptr = nullptr;      // device [owned rows * n_u + 1]
  int4* cta_uni = nullptr;         // device: interior strips (i0, i1, -, -), row chunks from the launch
  int4* cta_gen = nullptr;         // device: frame CTAs (i0, i1, ja, jb)
  int n_uni = 0, n_gen = 0;
  std::vector<int4> h_uni_strips, h_gen;   // interior strips (rows chunked per call) and the frame CTAs
  int uni_j0 = 0, uni_j1 = 0;
  double* e_part = nullptr;        // energy partials [nbatch][n_uni + n_gen]
  int64_t e_cap = 0;
  size_t smem = 0;
};

// 0: built; 1: not applicable (not affine, not G3-FULL for both energies, tables failed verification);
// < 0 error.
int build_g3(const Sheet& sh, G3Tables& gt, std::string& err, const std::function<void*(size_t)>& dalloc);

int g3_eval(G3Tables& gt, const double* d_x, int64_t x_stride, const Mat& mat, int flags, int nbatch, double* d_E,
            double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const double* d_params, cudaStream_t st,
            int* launches, const std::function<void*(size_t)>& dalloc);

}  // namespace bsf
