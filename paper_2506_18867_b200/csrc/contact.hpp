// Contact Hessian pullback to the control points (contact.cu, Alg. 1).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "host.hpp"

namespace bsf {

struct ContactState {
  bool ready = false, assembled = false;
  int nvert = 0, ncp = 0, n_u = 0;
  // static: the embedded mesh
  int2* vwin = nullptr;        // [nvert] (span u, span v) of the vertex's 3x3 control-point window
  double* vw = nullptr;        // [9][nvert] N_ij(u_alpha, v_alpha), window entry e = 3 jv + iu
  int32_t* cp_ptr = nullptr;   // [ncp + 1] control point -> (vertex, entry) lists with nonzero weight
  int2* cp_list = nullptr;
  // per call: sort scratch and the off-diagonal contact BSR
  uint64_t *k1 = nullptr, *k2 = nullptr;
  uint32_t *v1 = nullptr, *v2 = nullptr;
  int32_t *flag = nullptr, *id = nullptr, *start = nullptr, *rank = nullptr;
  double* hlin = nullptr;      // [unique vertex pairs][9] H_lin blocks
  int2* ab = nullptr;          // [unique vertex pairs] (alpha, beta)
  int32_t* wps = nullptr;      // [window pairs + 1] run starts into wpu
  uint32_t* wpu = nullptr;     // [unique vertex pairs] vertex pairs sorted by window pair
  int2* wpo = nullptr;         // [window pairs] the two window origins (linear control-point index)
  double* wblk = nullptr;      // [window pairs][81][9] the window pairs' control-point blocks
  int32_t *row_ptr = nullptr, *col = nullptr;
  double* vals = nullptr;
  double* gv = nullptr;        // [nvert][3] per-vertex gradient
  uint8_t* tmp = nullptr;      // CUB temporary storage
  int* bad = nullptr;          // a pair vertex index >= nvert was seen
  int64_t k1_cap = 0, k2_cap = 0, v1_cap = 0, v2_cap = 0, flag_cap = 0, id_cap = 0, start_cap = 0, rank_cap = 0,
          hlin_cap = 0, ab_cap = 0, row_cap = 0, col_cap = 0, vals_cap = 0, gv_cap = 0, tmp_cap = 0,
          bad_cap = 0, wps_cap = 0, wpu_cap = 0, wpo_cap = 0, wblk_cap = 0;
  int64_t nnz = 0;             // off-diagonal blocks of the last assembly
  int nrows = 0;
};

int contact_mesh(ContactState& S, const Sheet& sh, int nvert, const double* uv, std::string& err);
int contact_positions(const ContactState& S, const double* d_x, double* d_xv, cudaStream_t st);
int contact_assemble(ContactState& S, int npairs, const int32_t* d_verts, const double* d_H, const double* d_g,
                     double* d_grad_cp, double* d_vals, const int32_t* d_diag_pos, int64_t* nnz_off, cudaStream_t st,
                     std::string& err);
void contact_free(ContactState& S);

}  // namespace bsf
