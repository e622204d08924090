// Frame path: the control points around the core rectangle (DESIGN.md §5 "k_frame").
//
// Near the sheet's edges the quadrature configuration changes from control point to control point
// (clipped dual cells, boundary spans with 2x3 / 3x3 Gauss rules, non-uniform end bases; PAPER.md:290-
// 293, 571-573), so the frame is assembled from host-built per-block contribution lists instead of the
// core's compile-time table.  The frame is cut into 4x4 tiles; one CTA per (tile, batch item) evaluates
// the tile's incident quadrature points into shared memory and gathers every block of every tile row
// in full (one thread per block; no transposes), so frame rows and core rows are written by disjoint
// kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "dev.hpp"
#include "host.hpp"

namespace bsf {

struct CoreTables;

namespace frame {
constexpr int kMaxCp = 16;      // control points per tile (4 x 4)
constexpr int kMaxNB = 25;      // blocks of a frame row
constexpr int kSlots = kMaxNB + 1;          // threads per control point: one per block + the gradient
constexpr int kTasks = kMaxCp * kSlots;     // 416 task slots per tile
constexpr int kThreads = 224;               // 7 warps, <= 2 tasks per thread, 4 CTAs per SM
constexpr int kMChan = 27;      // membrane record: A~uu 6 | A~vv 6 | A~uv 9 | P~u 3 | P~v 3
constexpr int kMCoef = 18;      // (dN/du Nv, Nu dN/dv) per window entry
constexpr int kBChan = 12;      // bending record: sqrt(w mu) L_e 9 | sqrt(w mu) Lap phi 3
}  // namespace frame

// Band path (band.cu): the four edge bands of the frame (between the core rectangle and the sheet edge,
// corners excluded) are translation invariant along the edge with period 2 (knot parity), so each band
// is assembled from one host-built template per (parity, depth row) with the core's channel split
// (one lane per control point x block entry (r, c)) and the y-formulation of the gather.
namespace band {
constexpr int kLA = 8;            // along lanes: same-parity control points s = S0 + pi + 2 l
constexpr int kLC = 4;            // channel lanes (a warp = 8 control points x 4 block entries)
constexpr int kNA = 2 * kLA;      // along control points per CTA
constexpr int kMS = kLA + 1;      // anchor pair slots: m = (oa - (S0 - 2)) >> 1
constexpr int kMaxD = 6;          // band depth (control points)
constexpr int kSl = 25;           // block column offsets (di, dj) in [-2, 2]^2
constexpr int kChan = 27;         // membrane record channels (as k_core)
constexpr int kThreads = 256;   // 2 CTAs per SM (measured: 512 threads, 1 CTA per SM, cut a single band CTA's
                                // latency by ~20 % but cost batched throughput: C2 x 100 1.06 -> 1.12 ms)
}  // namespace band

struct BandDesc {
  int axis;                       // 0: along i, depth j (bottom / top); 1: along j, depth i (left / right)
  int sa0, sa1, t0, t1;           // control points [sa0, sa1) along x [t0, t1) in depth
  int od0, od1;                   // anchor depth range of the classes
  int ncls, nbcls;                // membrane / bending point classes
  int cls0, bcls0;                // first class in the class arrays
  int ent0, nent;                 // entries of the band in the entry array
  int eoff[2][band::kMaxD];       // per (parity, depth row): first entry (band relative); membrane entries
                                  // grouped by ea = 0..8, then bending entries grouped by ea
  int ment[2][band::kMaxD], bent[2][band::kMaxD];   // entry counts
  unsigned char mcnt[2][band::kMaxD][9], bcnt[2][band::kMaxD][9];
  unsigned char rank[band::kMaxD][band::kSl];   // block rank of offset slot in the row, 255 = not in the pattern
  unsigned char wtask[band::kThreads / 32][6];  // gather tasks (depth row * 6 + parity * 3 + group) of each warp,
                                                // balanced by entry count on the host; 255 = none
};

struct BandTables {
  int ok = 0;
  int nbands = 0, nctas = 0;
  int covered[4] = {0, 0, 0, 0};  // bottom, top, left, right
  size_t smem = 0;
  double2* mcf = nullptr;         // [classes][9] parametric (dN/du Nv, Nu dN/dv) per window entry (masked)
  int2* mcls = nullptr;           // [classes] (anchor along parity, anchor depth)
  double* mwhat = nullptr;
  double* bcf = nullptr;          // [bending classes][27] LA | LB | LC
  int2* bcls = nullptr;
  double* bwhat = nullptr;
  // host copies of the warp-uniform gather data (passed in the kernel parameters)
  std::vector<BandDesc> h_desc;
  std::vector<int> h_cfirst;
  uint32_t* ent = nullptr;        // record offset (16 bits) | coefficient offset << 16 (12 bits) | ea << 28
  double2* entd = nullptr;        // per entry: (d_a,u, d_a,v) at its window position (membrane)
};

struct FrameTables {
  int ok = 0;
  BandTables band;
  int ntiles = 0;
  int maxM = 0, maxB = 0;      // per tile: membrane / bending points
  size_t smem = 0;
  int4* tile = nullptr;        // [ntiles] (i0, j0, tw | th << 8, ncp)
  int32_t* tpm = nullptr;      // [ntiles+1] first membrane point of each tile
  int32_t* tpb = nullptr;      // [ntiles+1] first bending point
  int2* m_anc = nullptr;       // [M] anchor (ou, ov)
  int32_t* m_own = nullptr;    // [M] 1 if the point's energy is counted by its tile
  double* m_coef = nullptr;    // [M][18] parametric d-vectors (masked), [M] what at m_what
  double* m_what = nullptr;
  int2* b_anc = nullptr;
  int32_t* b_own = nullptr;
  double* b_coef = nullptr;    // [B][27] LA | LB | LC per window entry (masked)
  double* b_what = nullptr;
  uint4* lst = nullptr;        // [ntiles * kTasks] tasks: (first | count << 20, block or ~a_loc, transposed block or -1, 0)
  uint32_t* ent = nullptr;     // entries: local point | ea << 10 | eb << 14 | bending << 18
  int32_t* tent = nullptr;     // [ntiles+1] first entry of each tile
};

// Build the frame tables for the control points of the owned rows outside the core rectangle.
// Returns 0 (ok = 1), 1 if not applicable (ok = 0), < 0 on errors.
int build_frame(const Sheet& sh, const CoreTables& ct, FrameTables& ft, std::string& err,
                const std::function<void*(size_t)>& dalloc);

// Band tables (called by build_frame). Returns 0 (ok = 1 if any band is covered), < 0 on errors.
int build_band(const Sheet& sh, const CoreTables& ct, BandTables& bt, std::string& err,
               const std::function<void*(size_t)>& dalloc);

int band_eval(const BandTables& bt, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
              int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const int32_t* d_row_ptr,
              double* e_part, int64_t e_stride, int64_t e_off, const double* d_params, const double* G4, double detJ,
              cudaStream_t st, const struct IpFused* ip = nullptr);

int frame_eval(const FrameTables& ft, const Sheet& sh, const double* d_x, int64_t x_stride, const Mat& mat, int flags,
               int nbatch, double* d_g, int64_t g_stride, double* d_vals, int64_t v_stride, const int32_t* d_row_ptr,
               double* e_part, int64_t e_stride, int64_t e_off, const double* d_params, const double* G4, double detJ,
               cudaStream_t st, const struct IpFused* ip = nullptr);

}  // namespace bsf
