// Incremental-potential epilogue kernels (ip.cu; Q13/Q14).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace bsf {

struct IpArgs {
  const double* x;       // positions, rows [xlo, ...) of the slab window, item stride xs
  int64_t xs;
  const double* xhat;    // [owned cps][3], item stride xhs
  int64_t xhs;
  double* g;             // [owned cps][3] or null, item stride gs
  int64_t gs;
  double* vals;          // BSR values or null, item stride vs
  int64_t vs;
  double* epart;         // energy partials [item][ip_partials(ncp)] (scratch)
  const double* mass;    // [owned cps]
  const int32_t* diag;   // [owned cps] block index of (a, a)
  const int32_t* zero_blk;   // blocks zeroed by the pinned elimination
  const int32_t* pin_cp;     // owned pinned control points
  int nzero, npin;
  int ncp, n_u, r0, xlo;
  double k;              // 1 / dt^2
  double grav[3];
  const double* params;  // optional per-item affine parameters [item][9]: masses scale by params[4] / detJ_ref
  double detJ_ref;
};

// Fused form (the assembly kernels add the terms themselves: core, band and corner kernels): the
// predicted positions, masses and constants they read.  k = 1/dt^2.
struct IpFused {
  const double* xhat;    // [owned cps][3] per item, item stride xhs
  int64_t xhs;
  const double* mass;    // [owned cps]
  double k;
  double grav[3];
  const double* params;  // optional per-item affine parameters: masses scale by params[9 item + 4] / detJ_ref
  double detJ_ref;
};

int ip_eval(IpArgs A, int nbatch, double* d_energy, cudaStream_t st, int* launches);
// only the pinned elimination (after a fused assembly)
int ip_pin(IpArgs A, int nbatch, cudaStream_t st, int* launches);
int ip_partials(int ncp);

}  // namespace bsf
