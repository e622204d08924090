// Device-side tables of one handle, shared by the kernels and the C-ABI layer.
#pragma once
#include <cstdint>

namespace bsf {

struct Mat {
  double mu_st1, mu_st2, mu_sh, mu_bd;
};

// Generic path tables (SoA, [entry][point]).
struct GenericTables {
  int64_t Mm = 0, Bm = 0;          // membrane / bending points touching the owned rows
  int32_t* m_xi = nullptr;         // [9][Mm] x-local cp index of window entry (or -1)
  double* m_b = nullptr;           // [18][Mm] b coefficients (entry*2 + beta)
  double* m_w = nullptr;           // [Mm]
  uint8_t* m_eown = nullptr;       // [Mm]
  int32_t* b_xi = nullptr;         // [9][Bm]
  double* b_L = nullptr;           // [9][Bm]
  double* b_w = nullptr;           // [Bm]
  uint8_t* b_eown = nullptr;       // [Bm]
  // scratch written by the point kernels
  double* s_A = nullptr;           // [21][Mm]  w * A (F-space Hessian)
  double* s_P = nullptr;           // [6][Mm]   w * P
  double* s_E = nullptr;           // [Mm + Bm] owned energy contributions
  double* s_D = nullptr;           // [3][Bm]   w mu_bd Lap(phi)
  // gather incidence lists
  int64_t* h_ptr = nullptr;        // [nnzb+1]
  uint32_t* h_inc = nullptr;       // packed (kind:1 | point:23 | la:4 | lb:4)
  int64_t* g_ptr = nullptr;        // [n_rows+1]
  uint32_t* g_inc = nullptr;       // packed (kind:1 | point:23 | la:4 | 0:4)
  double* e_part = nullptr;        // energy partial sums
  int e_nblocks = 0;
  unsigned long long* sflag = nullptr;   // singular-stretch word of the call (set per launch)
};

// Singular-stretch word of the handle whose call is being enqueued (mapped host memory, device address;
// fbw.cuh fbw_flag_singular).  Set by the C-ABI layer around each dispatch on the calling thread; every
// launch function copies it into its kernel's arguments.
inline unsigned long long*& call_sflag() {
  static thread_local unsigned long long* p = nullptr;
  return p;
}

// Fused energy reduction of a call (fbw.cuh energy_final_fused): the launch functions of the core / band / corner
// kernels copy the calling thread's current value into their kernel arguments.
struct EFinal {
  unsigned* cnt = nullptr;   // [nbatch] CTAs done (zeroed at the start of every call)
  double* out = nullptr;     // [nbatch] energies (nullptr: no fused reduction)
  int total = 0;             // CTAs per item over all kernels of the call (= energy slots per item)
  int per_item = 0;          // energy slots per item
};
inline EFinal& call_efinal() {
  static thread_local EFinal e;
  return e;
}

constexpr uint32_t kIncBend = 1u << 31;
inline __host__ __device__ uint32_t pack_inc(bool bend, uint32_t pt, uint32_t la, uint32_t lb) {
  return (bend ? kIncBend : 0u) | (pt << 8) | (la << 4) | lb;
}

}  // namespace bsf
