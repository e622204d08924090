// Fused tile path: one kernel evaluates the quadrature points of a column strip row by row into a
// shared-memory ring and gathers every BSR block / gradient row of the strip from it (see tile.cu
// and DESIGN.md §5).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "dev.hpp"
#include "host.hpp"

namespace bsf {

constexpr int kTX = 16;        // strip width (control points)
constexpr int kRS = 2;         // output rows per step
constexpr int kRing = kRS + 2; // anchor rows resident in the ring
constexpr int kTasks = 6;      // program tasks per control point: 5 forward-block groups + gradient
constexpr int kThreads = 32 * 7;   // warps 0-1 group 0 (split), 2-5 groups 1-4, 6 gradient
constexpr int kNCls = 13;      // boundary-distance classes per direction

struct TileTables {
  int ok = 0;
  int n_u = 0, n_v = 0, Su = 0, Sv = 0, r0 = 0, r1 = 0, xlo = 0;
  int nstrips = 0, nchunks = 0;
  int capm_l[2] = {1, 1}, capb_l[2] = {1, 1}, nch_l[2] = {0, 0};   // per chunk list (interior, boundary)
  size_t smem_l[2] = {0, 0};
  int2* chunks = nullptr;          // [nchunks] (ra, rb): interior chunks then boundary chunks
  int affine = 0;
  double G[4] = {0, 0, 0, 0};      // affine: G[r*2+c]
  double detJ = 0;
  double detJ_ref = 1.0;           // det J folded into the class weights (affine)
  int32_t* m_aoff = nullptr;       // [Sv*Su+1] anchor -> first membrane point (points sorted by anchor)
  int32_t* b_aoff = nullptr;
  uint2* m_info = nullptr;         // per sorted point: (u-table | v-table << 16, shape | anchor column << 16)
  uint2* b_info = nullptr;
  double* utab = nullptr;          // [n][9]: N[3] dN[3] ddN[3] of one exact 1D evaluation
  double* vtab = nullptr;
  double* stab = nullptr;          // [n][2]: w = what*detJ (affine) or 0, stencil mask
  double* m_geo = nullptr;         // general path: [5][Mm] G00 G01 G10 G11 w
  double* b_geo = nullptr;         // general path: [6][Bm] w c_uu c_vv c_uv c_u c_v
  int16_t* lut = nullptr;          // [kNCls][kNCls][2] -> program id
  int4* tasks = nullptr;           // [nprog][kTasks]: (entry offset, n_mem | n_bend<<16, k_lo | nb<<8, 0)
  unsigned long long* ent = nullptr;
  int32_t* row_ptr = nullptr;      // owned rows' pattern (device copy)
  double* e_part = nullptr;        // per-CTA energy partials (grown on demand)
  int64_t e_cap = 0;
  unsigned* e_cnt = nullptr;       // [nbatch] fused energy reduction counters (core path; grown on demand)
  int64_t e_cnt_cap = 0;
  // frame mode (the interior core kernel covers a rectangle): CTAs of the tile kernel
  // restricted to the (strip, chunk) pairs that touch the frame, per chunk list
  int core = 0;
  int sk[4] = {0, 0, 0, 0};        // skipped control points [i0,i1) x [j0,j1): rows written by k_core
  int ex[4] = {0, 0, 0, 0};        // anchors whose energy k_core counts
  int2* work_l[2] = {nullptr, nullptr};
  int nwork_l[2] = {0, 0};
  int core_ctas = 0;               // k_core CTAs per item (energy partial slots)
  int core_nchunks = 0;
  double* e_part_core = nullptr;   // [item][tile slots | core slots], tile slots of dropped pairs stay 0
  int64_t e_core_cap = 0;
  cudaStream_t side = nullptr;     // band kernel stream (fork / join with the caller's stream)
  cudaStream_t side2 = nullptr;    // corner (frame) kernel stream: runs beside the band and core kernels
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  // live per-kernel timing (bsf_set_kernel_timing): per call, event pairs around the core launch (caller's
  // stream) and the band launch (side stream), in a ring of tev_n calls
  std::vector<cudaEvent_t> tev;
  int tev_n = 0, tev_next = 0, tev_count = 0;
};

struct CoreTables;

// Switch a tile table set to frame mode around the core rectangle (uploads the work lists).
int tile_set_core(TileTables& tt, const Sheet& sh, const CoreTables& ct, const std::function<void*(size_t)>& dalloc);

int build_tiles(const Sheet& sh, TileTables& tt, std::string& err, const std::function<void*(size_t)>& dalloc);

// Batched evaluation: item b uses x + b*x_stride, grad + b*g_stride, vals + b*v_stride, E + b.
int tile_eval(TileTables& tt, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_E, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride,
              cudaStream_t st, int* launches, const std::function<void*(size_t)>& dalloc,
              const double* d_params = nullptr, const CoreTables* ct = nullptr,
              const struct FrameTables* ft = nullptr, const struct IpFused* ip = nullptr,
              const struct HaloOverlap* halo = nullptr);

// Overlap of the slab halo exchange with the assembly: the core rows [ja, jb), which read
// owned positions only, are launched first; `ready` (recorded after the exchange on another stream) is
// waited for before every launch that reads halo rows (the remaining core rows, bands, corners).
struct HaloOverlap {
  int ja, jb;
  cudaEvent_t ready;
};

}  // namespace bsf
