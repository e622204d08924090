// Contact Hessian pullback and assembly on the device (PAPER.md:584-603 and Alg. 1,
// PAPER.md:792-846).
//
// The contact mesh is embedded in the sheet: vertex alpha at a fixed parametric point moves as
// x^alpha = sum_ij N_ij(u_alpha, v_alpha) C^ij (Eq. `eq: trig mesh node from control points`), so a barrier's
// gradient and Hessian on the mesh pull back to the control points by the chain rule (Eq. `eq: gradient and
// hessian of contact barrier`).  The barrier and the contact detection that produce the pairs are out of scope;
// the inputs are the active pairs (up to 4 mesh vertices, -1 = no DOFs) with their 12x12 Hessians and gradients.
//
// Alg. 1 builds hash maps keyed by vertex pairs, then by control-point pairs, with spatial blocks to limit write
// conflicts.  The B200 version keeps its two levels but replaces hashing by sorting, which is deterministic and
// conflict-free: (1) the pairs' vertex-pair blocks are keyed by (alpha, beta), radix-sorted (stable: equal keys
// keep their emission order) and summed per key in that order (the linear-mesh Hessian H_lin); (1b) the H_lin
// blocks are grouped by their pair of 3x3 control-point windows (every vertex inside one knot span has the same
// window), and each window pair's 9 x 9 control-point blocks sum_{vertex pairs} N_i(alpha) N_j(beta) H_lin(alpha,
// beta) are formed by one CTA; (2) those blocks are keyed by their control-point pair (i, j), sorted and summed the
// same way.  The sorted unique keys ARE the BSR pattern (rows i, columns j
// ascending): diagonal blocks (i == j) are added into the elastic matrix's diagonal blocks (the paper's D, which
// keeps the elastic pattern), the rest is the off-diagonal contact matrix B in its own BSR pattern (the paper's
// B = H_barrier,od of the Neumann split).  The gradient goes through per-vertex sums and a static control-point
// -> vertex list.  No atomics: every output value is summed by one thread in a fixed order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <vector>

#include "contact.hpp"
#include "host.hpp"

namespace bsf {

namespace {

// Keys are a * m + b with m the number of vertices (control points); the sentinel m^2 (m for the vertex keys) sorts
// after every valid key, and the radix sort only visits the bits up to it.
inline int key_bits(uint64_t sentinel) {
  int b = 1;
  while (b < 64 && (sentinel >> b)) ++b;
  return b;
}

// level 1: (pair, slot a, slot b) -> key (alpha, beta); invalid slots -> the sentinel (sorted to the end)
template <class K>
__global__ void k_emit_lin(const int32_t* __restrict__ verts, int npairs, int nvert, K* __restrict__ key,
                           uint32_t* __restrict__ val, int* __restrict__ bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)npairs * 16) return;
  const int c = (int)(t >> 4), sa = (int)(t >> 2) & 3, sb = (int)t & 3;
  const int32_t a = verts[4 * c + sa], b = verts[4 * c + sb];
  const bool ok = a < nvert && b < nvert;
  if (!ok && sb == 0) atomicOr(bad, 1);
  // key a * nvert + b; the sentinel nvert^2 sorts after every valid key within the sorted bit range
  const uint64_t m = (uint64_t)nvert;
  key[t] = (K)((ok && a >= 0 && b >= 0) ? (uint64_t)a * m + (uint64_t)b : m * m);
  val[t] = (uint32_t)t;
}

// run heads of a sorted key array (first of each distinct valid key): flag[t] = 1
template <class K>
__global__ void k_heads(const K* __restrict__ key, int64_t n, K nokey, int32_t* __restrict__ flag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  flag[t] = (key[t] != nokey && (t == 0 || key[t] != key[t - 1])) ? 1 : 0;
}

// run starts: start[id[t] - 1] = t for heads; start[nruns] = end of the valid keys
template <class K>
__global__ void k_run_starts(const int32_t* __restrict__ flag, const int32_t* __restrict__ id, int64_t n,
                             const K* __restrict__ key, K nokey, int32_t* __restrict__ start) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (flag[t]) start[id[t] - 1] = (int32_t)t;
  if (key[t] != nokey && (t + 1 == n || key[t + 1] == nokey)) start[id[t]] = (int32_t)(t + 1);
}

// H_lin[u] = sum over the run of the pairs' (alpha, beta) blocks, in sorted (= emission) order
template <class K>
__global__ void k_sum_lin(const int32_t* __restrict__ start, int nruns, const uint32_t* __restrict__ val,
                          const double* __restrict__ H, const K* __restrict__ key, int nvert,
                          double* __restrict__ hlin, int2* __restrict__ ab) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nruns) return;
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int k = start[u]; k < start[u + 1]; ++k) {
    const uint32_t v = val[k];
    const int c = (int)(v >> 4), sa = (int)(v >> 2) & 3, sb = (int)v & 3;
    const double* h = H + (int64_t)144 * c + (3 * sa) * 12 + 3 * sb;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) s[3 * r + q] += h[12 * r + q];
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) hlin[9 * (int64_t)u + e] = s[e];
  const uint64_t kk = key[start[u]];
  ab[u] = make_int2((int)(kk / (uint64_t)nvert), (int)(kk % (uint64_t)nvert));
}

// level 1b: the vertex-pair blocks grouped by their pair of control-point windows (all vertices inside one knot
// span share a window), so that level 2 emits 81 control-point pairs per window pair, not per vertex pair
template <class K>
__global__ void k_emit_wp(const int2* __restrict__ ab, int nlin, const int2* __restrict__ vwin, int n_u, int ncp,
                          K* __restrict__ key, uint32_t* __restrict__ val) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nlin) return;
  const int2 p = ab[u], oa = vwin[p.x], ob = vwin[p.y];
  key[u] = (K)((uint64_t)(oa.y * n_u + oa.x) * (uint64_t)ncp + (uint64_t)(ob.y * n_u + ob.x));
  val[u] = (uint32_t)u;
}

// window pair w: its run of vertex pairs [wps[w], wps[w+1]) in wpu, and its two window origins (linear cp index)
template <class K>
__global__ void k_wp_info(const K* __restrict__ key, const int32_t* __restrict__ start, int nwp, int ncp,
                          int32_t* __restrict__ wps, int2* __restrict__ wpo) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwp) return;
  const uint64_t kk = key[start[w]];
  wpo[w] = make_int2((int)(kk / (uint64_t)ncp), (int)(kk % (uint64_t)ncp));
  wps[w] = start[w];
  if (w == nwp - 1) wps[nwp] = start[nwp];
}

// level 2, one CTA per window pair w, one thread per pair of window entries (ea, eb): the 3x3 block
// sum over w's vertex pairs of N_ea(alpha) N_eb(beta) H_lin(alpha, beta), in run order, and its key (i, j),
// emitted when some vertex pair of w has both weights nonzero (the oracle's structural pattern)
constexpr int kWpChunk = 32;   // vertex pairs of a window pair staged in shared memory at a time

template <class K>
__global__ void __launch_bounds__(96) k_wp_blocks(const int32_t* __restrict__ wps, const uint32_t* __restrict__ wpu,
                                                  const int2* __restrict__ wpo, const int2* __restrict__ ab,
                                                  const double* __restrict__ hlin, const double* __restrict__ vw,
                                                  int nvert, int n_u, int ncp, int nwp, double* __restrict__ wblk,
                                                  K* __restrict__ key, uint32_t* __restrict__ val) {
  // the run's weights and H_lin blocks are staged by all threads (independent loads in flight), then every
  // thread sums its block over them in run order
  __shared__ double sa[kWpChunk][9], sb[kWpChunk][9], sh[kWpChunk][9], so[729];
  const int e = threadIdx.x;
  const int ea = e / 9, eb = e - 9 * (e / 9);
  for (int w = blockIdx.x; w < nwp; w += gridDim.x) {   // grid-stride: the window pairs are many and short
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool nz = false;
  const int k0 = wps[w], k1 = wps[w + 1];
  for (int c0 = k0; c0 < k1; c0 += kWpChunk) {
    const int nc = min(kWpChunk, k1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < 27 * nc; t += blockDim.x) {
      const int k = t / 27, c = t - 27 * k;
      const uint32_t u = wpu[c0 + k];
      const int2 p = ab[u];
      if (c < 9) sa[k][c] = vw[(int64_t)c * nvert + p.x];
      else if (c < 18) sb[k][c - 9] = vw[(int64_t)(c - 9) * nvert + p.y];
      else sh[k][c - 18] = hlin[9 * (int64_t)u + c - 18];
    }
    __syncthreads();
    if (e < 81)
      for (int k = 0; k < nc; ++k) {
        const double wa = sa[k][ea], wb = sb[k][eb];
        nz |= wa != 0.0 && wb != 0.0;
        const double wt = wa * wb;
#pragma unroll
        for (int q = 0; q < 9; ++q) s[q] = fma(wt, sh[k][q], s[q]);
      }
  }
  // the window pair's 81 blocks are one contiguous 5,832-byte range of wblk: written through shared memory so
  // that every warp store is coalesced
  if (e < 81) {
#pragma unroll
    for (int q = 0; q < 9; ++q) so[9 * e + q] = s[q];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < 729; q += blockDim.x) wblk[729 * (int64_t)w + q] = so[q];
  if (e < 81) {
    const int64_t t = 81 * (int64_t)w + e;
    const uint64_t m = (uint64_t)ncp;
    val[t] = (uint32_t)t;
    const int2 o = wpo[w];
    const uint32_t i = (uint32_t)(o.x + (ea / 3) * n_u + ea % 3);
    const uint32_t j = (uint32_t)(o.y + (eb / 3) * n_u + eb % 3);
    key[t] = (K)(nz ? (uint64_t)i * m + j : m * m);
  }
  }
}

// Control-point blocks: sum of the run's window-pair blocks in sorted order; diagonal blocks go into the elastic
// matrix's diagonal (vals_d, nullable), off-diagonal ones into the contact BSR at their rank.
constexpr int kSumThreads = 128;

template <class K>
__global__ void __launch_bounds__(kSumThreads) k_sum_cp(const int32_t* __restrict__ start, int nruns,
                                                         const uint32_t* __restrict__ val, const K* __restrict__ key,
                                                         const double* __restrict__ wblk, int ncp,
                                                         const int32_t* __restrict__ offd_rank,
                                                         double* __restrict__ bvals, int32_t* __restrict__ bcol,
                                                         double* __restrict__ vals_d,
                                                         const int32_t* __restrict__ diag_pos) {
  // the CTA's off-diagonal blocks are consecutive in the output: staged in shared memory, then written coalesced
  __shared__ double so[9 * kSumThreads];
  const int r0 = blockIdx.x * kSumThreads, r = r0 + threadIdx.x;
  const int rl = min(nruns, r0 + kSumThreads) - 1;
  const int o0 = offd_rank[r0];
  if (r < nruns) {
    double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = start[r]; k < start[r + 1]; ++k) {
      const double* b = wblk + 9 * (int64_t)val[k];
#pragma unroll
      for (int q = 0; q < 9; ++q) s[q] += b[q];
    }
    const uint64_t kk = key[start[r]];
    const int i = (int)(kk / (uint64_t)ncp), j = (int)(kk % (uint64_t)ncp);
    if (i == j) {
      if (vals_d) {
        double* d = vals_d + 9 * (int64_t)diag_pos[i];
#pragma unroll
        for (int q = 0; q < 9; ++q) d[q] += s[q];
      }
    } else {
      const int32_t o = offd_rank[r];
      bcol[o] = j;
#pragma unroll
      for (int q = 0; q < 9; ++q) so[9 * (o - o0) + q] = s[q];
    }
  }
  __syncthreads();
  // off-diagonal blocks of this CTA: ranks [o0, o1)
  const uint64_t kl = key[start[rl]];
  const int o1 = offd_rank[rl] + ((kl / (uint64_t)ncp) != (kl % (uint64_t)ncp) ? 1 : 0);
  for (int t = threadIdx.x; t < 9 * (o1 - o0); t += kSumThreads) bvals[9 * (int64_t)o0 + t] = so[t];
}

template <class K>
__global__ void k_offd_flags(const K* __restrict__ key, const int32_t* __restrict__ start, int nruns, int ncp,
                             int32_t* __restrict__ flag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  const uint64_t kk = key[start[r]];
  flag[r] = kk / (uint64_t)ncp != kk % (uint64_t)ncp;
}

// row_ptr of the off-diagonal contact BSR from the sorted unique keys (rows ascending): one thread per row
// finds its first entry by binary search over the off-diagonal ranks
template <class K>
__global__ void k_row_ptr(const K* __restrict__ key, const int32_t* __restrict__ start,
                          const int32_t* __restrict__ flag, const int32_t* __restrict__ rank, int nruns, int nrows,
                          int ncp, int32_t* __restrict__ row_ptr) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a > nrows) return;
  // first run whose row is >= a
  int lo = 0, hi = nruns;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int)(key[start[mid]] / (uint64_t)ncp) < a) lo = mid + 1; else hi = mid;
  }
  // off-diagonal entries before run lo
  row_ptr[a] = lo < nruns ? rank[lo] : (nruns > 0 ? rank[nruns - 1] + flag[nruns - 1] : 0);
}

// gradient: per-vertex sums (k_sum_vert over runs of the sorted (alpha, slot) keys), scattered into a dense
// per-vertex array, then gathered per control point through the static cp -> (vertex, entry) lists
template <class K>
__global__ void k_emit_vert(const int32_t* __restrict__ verts, int npairs, int nvert, K* __restrict__ key,
                            uint32_t* __restrict__ val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)npairs * 4) return;
  const int32_t a = verts[t];
  key[t] = (K)((a >= 0 && a < nvert) ? (uint64_t)a : (uint64_t)nvert);
  val[t] = (uint32_t)t;
}

template <class K>
__global__ void k_sum_vert(const int32_t* __restrict__ start, int nruns, const uint32_t* __restrict__ val,
                           const K* __restrict__ key, const double* __restrict__ g, double* __restrict__ gv) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nruns) return;
  double s[3] = {0, 0, 0};
  for (int k = start[u]; k < start[u + 1]; ++k) {
    const uint32_t v = val[k];   // pair c = v / 4, slot = v % 4
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] += g[3 * (int64_t)v + r];
  }
  const int a = (int)key[start[u]];
#pragma unroll
  for (int r = 0; r < 3; ++r) gv[3 * (int64_t)a + r] = s[r];
}

__global__ void k_grad_cp(const int32_t* __restrict__ cp_ptr, const int2* __restrict__ cp_list,
                          const double* __restrict__ vw, int nvert, const double* __restrict__ gv, int ncp,
                          double* __restrict__ gcp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncp) return;
  double s[3] = {0, 0, 0};
  for (int k = cp_ptr[i]; k < cp_ptr[i + 1]; ++k) {
    const int2 ve = cp_list[k];   // (vertex, window entry)
    const double w = vw[(int64_t)ve.y * nvert + ve.x];
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] = fma(w, gv[3 * (int64_t)ve.x + r], s[r]);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) gcp[3 * (int64_t)i + r] += s[r];
}

__global__ void k_positions(const int2* __restrict__ vwin, const double* __restrict__ vw, int nvert, int n_u,
                            const double* __restrict__ x, double* __restrict__ xv) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nvert) return;
  const int2 o = vwin[a];
  double s[3] = {0, 0, 0};
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const double w = vw[(int64_t)e * nvert + a];
    const double* c = x + 3 * ((int64_t)(o.y + e / 3) * n_u + o.x + e % 3);
#pragma unroll
    for (int r = 0; r < 3; ++r) s[r] = fma(w, c[r], s[r]);
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) xv[3 * (int64_t)a + r] = s[r];
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)std::max<int64_t>(1, (n + b - 1) / b); }

template <class T>
bool grow(T** p, int64_t* cap, int64_t need) {
  if (need <= *cap) return true;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (size_t)std::max<int64_t>(need, 1)) != cudaSuccess) return false;
  *cap = need;
  return true;
}

}  // namespace

void contact_free(ContactState& S) {
  for (void* p : {(void*)S.vwin, (void*)S.vw, (void*)S.cp_ptr, (void*)S.cp_list, (void*)S.k1, (void*)S.k2,
                  (void*)S.v1, (void*)S.v2, (void*)S.flag, (void*)S.id, (void*)S.start, (void*)S.hlin, (void*)S.ab,
                  (void*)S.rank, (void*)S.row_ptr, (void*)S.col, (void*)S.vals, (void*)S.gv, (void*)S.tmp, (void*)S.bad,
                  (void*)S.wps, (void*)S.wpu, (void*)S.wpo, (void*)S.wblk})
    cudaFree(p);
  S = ContactState();
}

int contact_mesh(ContactState& S, const Sheet& sh, int nvert, const double* uv, std::string& err) {
  contact_free(S);
  const int nu = sh.n_u, nv = sh.n_v;
  std::vector<int2> win(nvert);
  std::vector<double> w((size_t)9 * nvert);
  std::vector<std::vector<int2>> lists((size_t)nu * nv);
  for (int a = 0; a < nvert; ++a) {
    const double u = uv[2 * a], v = uv[2 * a + 1];
    if (!(u >= 0.0 && u <= sh.Su && v >= 0.0 && v <= sh.Sv)) { err = "contact vertex outside the parameter domain"; return -1; }
    Basis1 bu, bv;
    basis1(sh.Su, u, bu);
    basis1(sh.Sv, v, bv);
    win[a] = make_int2(bu.span, bv.span);
    for (int e = 0; e < 9; ++e) {
      const double we = bu.N[e % 3] * bv.N[e / 3];
      w[(size_t)e * nvert + a] = we;
      if (we != 0.0) lists[(size_t)(bv.span + e / 3) * nu + bu.span + e % 3].push_back(make_int2(a, e));
    }
  }
  std::vector<int32_t> ptr((size_t)nu * nv + 1, 0);
  std::vector<int2> flat;
  for (size_t i = 0; i < lists.size(); ++i) {
    ptr[i + 1] = ptr[i] + (int32_t)lists[i].size();
    flat.insert(flat.end(), lists[i].begin(), lists[i].end());
  }
  auto up = [](auto** dst, const auto& v) {
    using T = std::remove_reference_t<decltype(v[0])>;
    if (cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * std::max<size_t>(v.size(), 1)) != cudaSuccess) return false;
    return v.empty() || cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up(&S.vwin, win) || !up(&S.vw, w) || !up(&S.cp_ptr, ptr) || !up(&S.cp_list, flat)) {
    contact_free(S);
    err = "contact mesh upload failed";
    return -7;
  }
  S.nvert = nvert;
  S.ncp = nu * nv;
  S.n_u = nu;
  S.ready = true;
  return 0;
}

int contact_positions(const ContactState& S, const double* d_x, double* d_xv, cudaStream_t st) {
  k_positions<<<nblk(S.nvert, 128), 128, 0, st>>>(S.vwin, S.vw, S.nvert, S.n_u, d_x, d_xv);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

// sorts (key, val) of n entries with CUB (stable LSD radix sort), then marks the runs of equal valid keys:
// returns the number of runs (host), run starts in S.start[0 .. nruns] (device)
template <class K>
static int sort_runs(ContactState& S, K* k_in, uint32_t* v_in, K* k_out, uint32_t* v_out, int64_t n, uint64_t nokey64,
                     cudaStream_t st, int* nruns, std::string& err) {
  const int nbits = key_bits(nokey64);
  const K nokey = (K)nokey64;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k_in, k_out, v_in, v_out, (int)n, 0, nbits, st);
  size_t tb2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb2, S.flag, S.id, (int)n, st);
  if (!grow(&S.tmp, &S.tmp_cap, (int64_t)std::max(tb, tb2)) || !grow(&S.flag, &S.flag_cap, n) ||
      !grow(&S.id, &S.id_cap, n) || !grow(&S.start, &S.start_cap, n + 1)) {
    err = "contact scratch allocation failed";
    return -7;
  }
  tb = (size_t)S.tmp_cap;
  if (cub::DeviceRadixSort::SortPairs(S.tmp, tb, k_in, k_out, v_in, v_out, (int)n, 0, nbits, st) != cudaSuccess) {
    err = "radix sort failed";
    return -6;
  }
  k_heads<<<nblk(n, 256), 256, 0, st>>>(k_out, n, nokey, S.flag);
  tb2 = (size_t)S.tmp_cap;
  if (cub::DeviceScan::InclusiveSum(S.tmp, tb2, S.flag, S.id, (int)n, st) != cudaSuccess) { err = "scan failed"; return -6; }
  int last = 0;
  if (cudaMemcpyAsync(&last, S.id + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    err = "run count";
    return -6;
  }
  *nruns = last;
  if (last > 0) k_run_starts<<<nblk(n, 256), 256, 0, st>>>(S.flag, S.id, n, k_out, nokey, S.start);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

// K1: key type of the vertex keys (level 1, gradient), K2: of the control-point keys (levels 1b, 2); 32-bit when
// the sentinel fits (fewer radix passes and half the key traffic)
template <class K1, class K2>
static int assemble_impl(ContactState& S, int npairs, const int32_t* d_verts, const double* d_H, const double* d_g,
                         double* d_grad_cp, double* d_vals, const int32_t* d_diag_pos, int64_t* nnz_off,
                         cudaStream_t st, std::string& err) {
  const auto K1p = [](uint64_t* p) { return reinterpret_cast<K1*>(p); };
  const auto K2p = [](uint64_t* p) { return reinterpret_cast<K2*>(p); };
  S.nnz = 0;
  S.nrows = S.ncp;
  if (!grow(&S.row_ptr, &S.row_cap, S.ncp + 1)) { err = "allocation"; return -7; }
  int rc = 0;
  // ---- level 1: vertex-pair blocks
  const int64_t n1 = (int64_t)npairs * 16;
  int nlin = 0;
  if (npairs > 0) {
    if (!grow(&S.k1, &S.k1_cap, n1) || !grow(&S.v1, &S.v1_cap, n1) || !grow(&S.k2, &S.k2_cap, n1) ||
        !grow(&S.v2, &S.v2_cap, n1)) { err = "allocation"; return -7; }
    if (!grow(&S.bad, &S.bad_cap, 1) || cudaMemsetAsync(S.bad, 0, sizeof(int), st) != cudaSuccess) {
      err = "allocation";
      return -7;
    }
    k_emit_lin<<<nblk(n1, 256), 256, 0, st>>>(d_verts, npairs, S.nvert, K1p(S.k1), S.v1, S.bad);
    if ((rc = sort_runs(S, K1p(S.k1), S.v1, K1p(S.k2), S.v2, n1, (uint64_t)S.nvert * S.nvert, st, &nlin, err))) return rc;
    int bad = 0;
    if (cudaMemcpy(&bad, S.bad, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) { err = "copy"; return -6; }
    if (bad) { err = "contact pair vertex index >= n_vert"; return -1; }
    if ((int64_t)nlin * 81 > (int64_t)INT32_MAX) { err = "too many distinct contact vertex pairs (> 26.5M)"; return -1; }
  }
  if (nlin > 0) {
    if (!grow(&S.hlin, &S.hlin_cap, 9 * (int64_t)nlin) || !grow(&S.ab, &S.ab_cap, nlin)) { err = "allocation"; return -7; }
    k_sum_lin<<<nblk(nlin, 128), 128, 0, st>>>(S.start, nlin, S.v2, d_H, K1p(S.k2), S.nvert, S.hlin, S.ab);
  }
  // ---- level 1b: window pairs
  int nwp = 0;
  if (nlin > 0) {
    k_emit_wp<<<nblk(nlin, 256), 256, 0, st>>>(S.ab, nlin, S.vwin, S.n_u, S.ncp, K2p(S.k1), S.v1);
    if ((rc = sort_runs(S, K2p(S.k1), S.v1, K2p(S.k2), S.v2, nlin, (uint64_t)S.ncp * S.ncp, st, &nwp, err))) return rc;
    if (!grow(&S.wps, &S.wps_cap, nwp + 1) || !grow(&S.wpo, &S.wpo_cap, nwp) || !grow(&S.wpu, &S.wpu_cap, nlin)) {
      err = "allocation";
      return -7;
    }
    k_wp_info<<<nblk(nwp, 256), 256, 0, st>>>(K2p(S.k2), S.start, nwp, S.ncp, S.wps, S.wpo);
    if (cudaMemcpyAsync(S.wpu, S.v2, sizeof(uint32_t) * nlin, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      err = "copy";
      return -6;
    }
  }
  // ---- level 2: control-point blocks
  const int64_t n2 = (int64_t)nwp * 81;
  int ncpb = 0;
  if (n2 > 0) {
    if (!grow(&S.k1, &S.k1_cap, n2) || !grow(&S.v1, &S.v1_cap, n2) || !grow(&S.k2, &S.k2_cap, n2) ||
        !grow(&S.v2, &S.v2_cap, n2)) { err = "allocation"; return -7; }
    if (!grow(&S.wblk, &S.wblk_cap, 9 * n2)) { err = "allocation"; return -7; }
    k_wp_blocks<<<std::min(nwp, 148 * 16), 96, 0, st>>>(S.wps, S.wpu, S.wpo, S.ab, S.hlin, S.vw, S.nvert, S.n_u, S.ncp,
                                                        nwp, S.wblk, K2p(S.k1), S.v1);
    if ((rc = sort_runs(S, K2p(S.k1), S.v1, K2p(S.k2), S.v2, n2, (uint64_t)S.ncp * S.ncp, st, &ncpb, err))) return rc;
  }
  if (ncpb > 0) {
    // off-diagonal ranks (exclusive scan of the off-diagonal flags of the runs), pattern, values
    if (!grow(&S.rank, &S.rank_cap, ncpb + 1)) { err = "allocation"; return -7; }
    int32_t* offflag = S.flag;   // reuse: the run flags of the level-2 sort are no longer needed
    k_offd_flags<<<nblk(ncpb, 256), 256, 0, st>>>(K2p(S.k2), S.start, ncpb, S.ncp, offflag);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, offflag, S.rank, ncpb, st);
    if (!grow(&S.tmp, &S.tmp_cap, (int64_t)tb)) { err = "allocation"; return -7; }
    tb = (size_t)S.tmp_cap;
    if (cub::DeviceScan::ExclusiveSum(S.tmp, tb, offflag, S.rank, ncpb, st) != cudaSuccess) { err = "scan"; return -6; }
    int lastr = 0, lastf = 0;
    if (cudaMemcpyAsync(&lastr, S.rank + ncpb - 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&lastf, offflag + ncpb - 1, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) { err = "count"; return -6; }
    S.nnz = lastr + lastf;
    if (!grow(&S.col, &S.col_cap, std::max<int64_t>(S.nnz, 1)) || !grow(&S.vals, &S.vals_cap, 9 * std::max<int64_t>(S.nnz, 1))) {
      err = "allocation";
      return -7;
    }
    k_sum_cp<<<nblk(ncpb, kSumThreads), kSumThreads, 0, st>>>(S.start, ncpb, S.v2, K2p(S.k2), S.wblk, S.ncp, S.rank, S.vals, S.col,
                                              d_vals, d_diag_pos);
    k_row_ptr<<<nblk(S.ncp + 1, 256), 256, 0, st>>>(K2p(S.k2), S.start, offflag, S.rank, ncpb, S.ncp, S.ncp, S.row_ptr);
  } else if (cudaMemsetAsync(S.row_ptr, 0, sizeof(int32_t) * (S.ncp + 1), st) != cudaSuccess) {
    err = "memset";
    return -6;
  }
  // ---- gradient
  if (d_g && d_grad_cp && npairs > 0) {
    const int64_t n3 = (int64_t)npairs * 4;
    if (!grow(&S.k1, &S.k1_cap, n3) || !grow(&S.v1, &S.v1_cap, n3) || !grow(&S.k2, &S.k2_cap, n3) ||
        !grow(&S.v2, &S.v2_cap, n3) || !grow(&S.gv, &S.gv_cap, 3 * (int64_t)S.nvert)) { err = "allocation"; return -7; }
    if (cudaMemsetAsync(S.gv, 0, sizeof(double) * 3 * (size_t)S.nvert, st) != cudaSuccess) { err = "memset"; return -6; }
    k_emit_vert<<<nblk(n3, 256), 256, 0, st>>>(d_verts, npairs, S.nvert, K1p(S.k1), S.v1);
    int nv = 0;
    if ((rc = sort_runs(S, K1p(S.k1), S.v1, K1p(S.k2), S.v2, n3, (uint64_t)S.nvert, st, &nv, err))) return rc;
    if (nv > 0) k_sum_vert<<<nblk(nv, 128), 128, 0, st>>>(S.start, nv, S.v2, K1p(S.k2), d_g, S.gv);
    k_grad_cp<<<nblk(S.ncp, 128), 128, 0, st>>>(S.cp_ptr, S.cp_list, S.vw, S.nvert, S.gv, S.ncp, d_grad_cp);
  }
  if (getenv("BSF_DEBUG_CONTACT"))
    fprintf(stderr, "contact: pairs %d, vertex pairs %d, window pairs %d, cp pairs %d, off-diagonal %lld\n", npairs,
            nlin, nwp, ncpb, (long long)S.nnz);
  if (nnz_off) *nnz_off = S.nnz;
  S.assembled = true;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

int contact_assemble(ContactState& S, int npairs, const int32_t* d_verts, const double* d_H, const double* d_g,
                     double* d_grad_cp, double* d_vals, const int32_t* d_diag_pos, int64_t* nnz_off, cudaStream_t st,
                     std::string& err) {
  static const bool force64 = getenv("BSF_CONTACT_KEYS64") && atoi(getenv("BSF_CONTACT_KEYS64")) != 0;   // test switch
  const bool v32 = !force64 && (uint64_t)S.nvert * S.nvert <= 0xffffffffull;
  const bool c32 = !force64 && (uint64_t)S.ncp * S.ncp <= 0xffffffffull;
  if (v32 && c32)
    return assemble_impl<uint32_t, uint32_t>(S, npairs, d_verts, d_H, d_g, d_grad_cp, d_vals, d_diag_pos, nnz_off, st, err);
  if (v32)
    return assemble_impl<uint32_t, uint64_t>(S, npairs, d_verts, d_H, d_g, d_grad_cp, d_vals, d_diag_pos, nnz_off, st, err);
  if (c32)
    return assemble_impl<uint64_t, uint32_t>(S, npairs, d_verts, d_H, d_g, d_grad_cp, d_vals, d_diag_pos, nnz_off, st, err);
  return assemble_impl<uint64_t, uint64_t>(S, npairs, d_verts, d_H, d_g, d_grad_cp, d_vals, d_diag_pos, nnz_off, st, err);
}

}  // namespace bsf
