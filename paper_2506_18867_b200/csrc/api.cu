// C-ABI of libbsfem (include/bsfem.h): handle creation, table upload and call dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <string>
#include <vector>

#include "../../include/bsfem.h"
#include "dev.hpp"
#include "host.hpp"
#include "core.hpp"
#include "frame.hpp"
#include "tile.hpp"
#include "ip.hpp"
#include "solve.hpp"
#include "g3.hpp"
#include "chol.hpp"
#include "contact.hpp"

namespace bsf {
int generic_eval(const GenericTables& t, const double* d_x, const Mat& mat, int flags, int64_t nnzb, int64_t nrows,
                 double* d_E, double* d_g, double* d_vals, cudaStream_t st, int* launches);
}

namespace {
thread_local std::string g_err = "ok";
bsf_status fail(bsf_status s, const std::string& m) {
  g_err = m;
  return s;
}
}  // namespace

struct bsf_sheet {
  int device = 0;
  bsf::Sheet sh;
  bsf::Mat mat{};
  bsf::GenericTables gt;
  bsf::TileTables tt;
  bool tile_ok = false;
  bsf::CoreTables ct;
  bool core_ok = false;
  bsf::FrameTables ft;
  bsf::G3Tables g3;                     // G3-FULL rule on affine sheets (g3.cu)
  bool g3_ok = false;
  bool generic_ok = false;              // generic gather path built (point count fits its index packing)
  cudaStream_t copy_stream = nullptr;   // host-buffer calls: position uploads
  cudaEvent_t ev_copy = nullptr, ev_start = nullptr;
  struct StageUse { const void* ptr; cudaEvent_t done; };   // BSF_ASYNC_STAGE: last reader of each stage
  std::vector<StageUse> stage_uses;
  // incremental potential (bsf_set_inertia)
  bool ip_set = false;
  double ip_k = 0.0, ip_g[3] = {0.0, 0.0, 0.0};
  std::vector<double> h_mass;
  double* d_mass = nullptr;
  int32_t *d_diag = nullptr, *d_zero = nullptr, *d_pin = nullptr;
  size_t cap_mass = 0, cap_diag = 0, cap_zero = 0, cap_pin = 0;
  int nzero = 0, npin = 0;
  double* d_ip_epart = nullptr;
  int64_t ip_epart_cap = 0;
  // linear algebra on the assembled Hessian (solve.cu)
  int32_t *d_rp = nullptr, *d_ci = nullptr, *d_sdiag = nullptr;
  bsf::CgWork cg{};
  bsf::CgGraph cg_graph;
  bsf::CholState chol;                  // banded Cholesky of the Newton matrix (chol.cu)
  bsf::ContactState contact;            // embedded contact mesh and its pulled-back Hessian (contact.cu)
  cudaStream_t comm_stream = nullptr;   // bsf_eval_all_slab: halo exchange
  cudaEvent_t ev_halo0 = nullptr, ev_halo = nullptr;
  bool solve_ready = false, cg_ready = false;
  std::vector<void*> allocs;
  int last_launches = 0;
  bool host_only = false;
  // singular-stretch word (fbw.cuh fbw_flag_singular): page-locked, mapped host memory the kernels store to
  unsigned long long* sflag_host = nullptr;
  unsigned long long* sflag_dev = nullptr;
  ~bsf_sheet() {
    if (host_only) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (sflag_host) cudaFreeHost(sflag_host);
    bsf::chol_free(chol);
    bsf::contact_free(contact);
    if (tt.side) cudaStreamDestroy(tt.side);
    if (tt.side2) cudaStreamDestroy(tt.side2);
    if (tt.ev_join2) cudaEventDestroy(tt.ev_join2);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ev_copy) cudaEventDestroy(ev_copy);
    if (ev_start) cudaEventDestroy(ev_start);
    if (tt.ev_fork) cudaEventDestroy(tt.ev_fork);
    if (tt.ev_join) cudaEventDestroy(tt.ev_join);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (ev_halo0) cudaEventDestroy(ev_halo0);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (cg_graph.exec) cudaGraphExecDestroy(cg_graph.exec);
    if (cg_graph.cs) cudaStreamDestroy(cg_graph.cs);
    if (cg_graph.e0) cudaEventDestroy(cg_graph.e0);
    if (cg_graph.e1) cudaEventDestroy(cg_graph.e1);
    for (StageUse& u : stage_uses) cudaEventDestroy(u.done);
    for (cudaEvent_t e : tt.tev) cudaEventDestroy(e);
    for (void* p : allocs) cudaFree(p);
    cudaSetDevice(prev);
  }
  template <class T>
  bsf_status upload(T** dst, const std::vector<T>& src) {
    *dst = nullptr;
    if (src.empty()) return BSF_OK;
    void* p = nullptr;
    if (cudaMalloc(&p, src.size() * sizeof(T)) != cudaSuccess) return fail(BSF_E_OOM, "cudaMalloc failed");
    allocs.push_back(p);
    if (cudaMemcpy(p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(BSF_E_CUDA, "cudaMemcpy failed");
    *dst = static_cast<T*>(p);
    return BSF_OK;
  }
  // upload into an existing allocation when it is large enough (set_inertia may be called every step)
  template <class T>
  bsf_status upload_reuse(T** dst, size_t* cap, const std::vector<T>& src) {
    if (src.empty()) return BSF_OK;
    if (!*dst || *cap < src.size()) {
      bsf_status s = upload(dst, src);
      if (s == BSF_OK) *cap = src.size();
      return s;
    }
    if (cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(BSF_E_CUDA, "cudaMemcpy failed");
    return BSF_OK;
  }
  std::function<void*(size_t)> dalloc() {
    return [this](size_t bytes) -> void* {
      void* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
      allocs.push_back(p);
      return p;
    };
  }
  template <class T>
  bsf_status alloc(T** dst, size_t n) {
    *dst = nullptr;
    if (n == 0) return BSF_OK;
    void* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return fail(BSF_E_OOM, "cudaMalloc failed");
    allocs.push_back(p);
    *dst = static_cast<T*>(p);
    return BSF_OK;
  }
};

namespace {

bsf_status build_generic(bsf_sheet* h) {
  const bsf::Sheet& sh = h->sh;
  bsf::GenericTables& t = h->gt;
  const int64_t M = (int64_t)sh.mem.size(), B = (int64_t)sh.bend.size();
  // the incidence lists pack point indices in 23 bits: larger handles run on the tile / G3 kernels only
  h->generic_ok = !(M >= (1 << 23) || B >= (1 << 23));
  if (!h->generic_ok) return BSF_OK;
  t.Mm = M;
  t.Bm = B;
  const int nu = sh.n_u;
  auto xloc = [&](const bsf::Point& P, int e) { return (P.ov + e / 3 - sh.xlo) * nu + P.ou + e % 3; };
  std::vector<int32_t> m_xi(9 * M), b_xi(9 * B);
  std::vector<double> m_b(18 * M), m_w(M), b_L(9 * B), b_w(B);
  for (int64_t q = 0; q < M; ++q) {
    const bsf::Point& P = sh.mem[q];
    m_w[q] = P.w;
    for (int e = 0; e < 9; ++e) {
      const bool in = (P.mask >> e) & 1;
      m_xi[e * M + q] = in ? xloc(P, e) : -1;
      m_b[(2 * e) * M + q] = P.b[e][0];
      m_b[(2 * e + 1) * M + q] = P.b[e][1];
    }
  }
  for (int64_t q = 0; q < B; ++q) {
    const bsf::Point& P = sh.bend[q];
    b_w[q] = P.w;
    for (int e = 0; e < 9; ++e) {
      const bool in = (P.mask >> e) & 1;
      b_xi[e * B + q] = in ? xloc(P, e) : -1;
      b_L[e * B + q] = P.L[e];
    }
  }
  // incidence lists (counting sort by block / by row; within a list: membrane points then bending
  // points in creation order -> deterministic)
  const int r0 = sh.r0, r1 = sh.r1;
  const int64_t nrows = (int64_t)(r1 - r0) * nu, nnzb = (int64_t)sh.col_idx.size();
  std::vector<int64_t> hp(nnzb + 1, 0), gp(nrows + 1, 0);
  auto for_each_inc = [&](auto&& fn) {
    for (int pass = 0; pass < 2; ++pass) {
      const auto& L = pass ? sh.bend : sh.mem;
      for (int64_t q = 0; q < (int64_t)L.size(); ++q) {
        const bsf::Point& P = L[q];
        for (int ea = 0; ea < 9; ++ea) {
          if (!((P.mask >> ea) & 1)) continue;
          const int ra = P.ov + ea / 3;
          if (ra < r0 || ra >= r1) continue;
          const int64_t row = (int64_t)(ra - r0) * nu + P.ou + ea % 3;
          fn(pass == 1, q, ea, row, -1, -1);
          const int32_t* c0 = sh.col_idx.data() + sh.row_ptr[row];
          const int32_t* c1 = sh.col_idx.data() + sh.row_ptr[row + 1];
          for (int eb = 0; eb < 9; ++eb) {
            if (!((P.mask >> eb) & 1)) continue;
            const int32_t b = (P.ov + eb / 3) * nu + P.ou + eb % 3;
            const int64_t k = std::lower_bound(c0, c1, b) - sh.col_idx.data();
            fn(pass == 1, q, ea, row, eb, k);
          }
        }
      }
    }
  };
  for_each_inc([&](bool, int64_t, int, int64_t row, int eb, int64_t k) {
    if (eb < 0) ++gp[row + 1]; else ++hp[k + 1];
  });
  for (int64_t i = 0; i < nnzb; ++i) hp[i + 1] += hp[i];
  for (int64_t i = 0; i < nrows; ++i) gp[i + 1] += gp[i];
  std::vector<uint32_t> hinc(hp[nnzb]), ginc(gp[nrows]);
  std::vector<int64_t> hf(hp.begin(), hp.end() - 1), gf(gp.begin(), gp.end() - 1);
  for_each_inc([&](bool bend, int64_t q, int ea, int64_t row, int eb, int64_t k) {
    if (eb < 0) ginc[gf[row]++] = bsf::pack_inc(bend, (uint32_t)q, ea, 0);
    else hinc[hf[k]++] = bsf::pack_inc(bend, (uint32_t)q, ea, eb);
  });
  std::vector<uint8_t> me(sh.mem_eown), be(sh.bend_eown);
  bsf_status s;
  if ((s = h->upload(&t.m_xi, m_xi)) || (s = h->upload(&t.m_b, m_b)) || (s = h->upload(&t.m_w, m_w)) ||
      (s = h->upload(&t.m_eown, me)) || (s = h->upload(&t.b_xi, b_xi)) || (s = h->upload(&t.b_L, b_L)) ||
      (s = h->upload(&t.b_w, b_w)) || (s = h->upload(&t.b_eown, be)) || (s = h->upload(&t.h_ptr, hp)) ||
      (s = h->upload(&t.h_inc, hinc)) || (s = h->upload(&t.g_ptr, gp)) || (s = h->upload(&t.g_inc, ginc)))
    return s;
  if ((s = h->alloc(&t.s_A, 21 * M)) || (s = h->alloc(&t.s_P, 6 * M)) || (s = h->alloc(&t.s_E, M + B)) ||
      (s = h->alloc(&t.s_D, 3 * B)))
    return s;
  t.e_nblocks = (int)std::max<int64_t>(1, std::min<int64_t>(592, (M + B + 255) / 256));
  if ((s = h->alloc(&t.e_part, t.e_nblocks))) return s;
  return BSF_OK;
}

// Sets the singular-stretch word of the handle for the launches enqueued in this scope (dev.hpp call_sflag).
struct SflagScope {
  explicit SflagScope(unsigned long long* p) { bsf::call_sflag() = p; }
  ~SflagScope() { bsf::call_sflag() = nullptr; }
};

// A completed earlier call found a singular stretch (|F e_beta| < 1e-12 at a membrane point; SURVEY §8(b),
// SPEC.md:290): report it once, naming the point, and clear the word.  Host read, no synchronisation.
bsf_status take_singular(bsf_sheet* h) {
  if (!h->sflag_host) return BSF_OK;
  const unsigned long long c = *(volatile unsigned long long*)h->sflag_host;
  if (!(c >> 63)) return BSF_OK;
  *(volatile unsigned long long*)h->sflag_host = 0ull;
  const int item = (int)((c >> 44) & 0x7FFFF), t = (int)((c >> 22) & 0x3FFFFF), s = (int)(c & 0x3FFFFF);
  std::string where = t == 0x3FFFFF ? "membrane point #" + std::to_string(s) + " of the generic path"
                                    : "a membrane point anchored at knot span (" + std::to_string(s) + ", " +
                                          std::to_string(t) + ") of batch item " + std::to_string(item);
  return fail(BSF_E_SINGULAR_STRETCH, "singular stretch |F e_beta| < 1e-12 (FBW undefined) at " + where +
                                          " in an earlier call; its outputs hold inf / NaN there");
}

bsf_status check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BSF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return BSF_OK;
}

}  // namespace

extern "C" {

const char* bsf_last_error(void) { return g_err.c_str(); }

bsf_status bsf_material_from_young(double E, double nu, double h, double shear_E, double bend_E, bsf_material* out) {
  if (!out || !(E > 0.0) || !(h > 0.0) || !(nu > -1.0 && nu < 0.5)) return fail(BSF_E_INVALID_ARG, "invalid material");
  const double G = shear_E >= 0.0 ? shear_E : E / (2.0 * (1.0 + nu));
  const double Eb = bend_E >= 0.0 ? bend_E : E;
  out->mu_st1 = 0.5 * E * h;
  out->mu_st2 = 0.5 * E * h;
  out->mu_sh = 0.5 * G * h;
  out->mu_bd = Eb * h * h * h / (12.0 * (1.0 - nu * nu));
  return BSF_OK;
}

bsf_status bsf_create(int n_u, int n_v, const double* knots_u, const double* knots_v, const double* rest_xy,
                      const bsf_material* mat, int membrane_rule, int bending_rule, int row_begin, int row_end,
                      int device, bsf_handle* out) {
  if (!out || !knots_u || !knots_v || !rest_xy || !mat) return fail(BSF_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const bool host_only = (device == -1);   // host-only handle: pattern / sizes queries, no compute
  if (!host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      return fail(BSF_E_NO_DEVICE, "no CUDA device");
    }
    if (device < 0 || device >= ndev) return fail(BSF_E_INVALID_ARG, "bad device ordinal");
  }
  auto* h = new (std::nothrow) bsf_sheet();
  if (!h) return fail(BSF_E_OOM, "host allocation failed");
  h->device = device;
  std::string err;
  const int rc = bsf::build_sheet(n_u, n_v, knots_u, knots_v, rest_xy, membrane_rule, bending_rule, row_begin,
                                  row_end, h->sh, err);
  if (rc) {
    delete h;
    return fail((bsf_status)rc, err);
  }
  h->mat = {mat->mu_st1, mat->mu_st2, mat->mu_sh, mat->mu_bd};
  if (host_only) {
    h->host_only = true;
    *out = h;
    return BSF_OK;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  bsf_status s = BSF_OK;
  if (cudaHostAlloc(reinterpret_cast<void**>(&h->sflag_host), sizeof(unsigned long long), cudaHostAllocMapped) !=
          cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->sflag_dev), h->sflag_host, 0) != cudaSuccess) {
    cudaGetLastError();
    s = fail(BSF_E_CUDA, "mapped host allocation failed");
  } else {
    *h->sflag_host = 0ull;
  }
  if (s == BSF_OK) s = build_generic(h);
  if (s == BSF_OK) {
    std::string terr;
    const int trc = bsf::build_tiles(h->sh, h->tt, terr, h->dalloc());
    h->tile_ok = (trc == 0);
    if (trc < 0) s = fail(BSF_E_OOM, terr);
    if (h->tile_ok) {   // interior core kernel (affine sheets, REDUCED rules): optional
      const int crc = bsf::build_core(h->sh, h->tt.row_ptr, h->ct, terr, h->dalloc());
      if (crc < 0) s = fail(BSF_E_CUDA, terr);
      else if (crc == 0 && h->ct.ok) {
        const int src = bsf::tile_set_core(h->tt, h->sh, h->ct, h->dalloc());
        if (src < 0) s = fail(BSF_E_OOM, "frame work lists");
        else h->core_ok = true;
        if (h->core_ok && !getenv("BSF_FRAME_TILE")) {   // frame kernel (else: tile kernel on the frame)
          const int frc = bsf::build_frame(h->sh, h->ct, h->ft, terr, h->dalloc());
          if (frc < 0) s = fail(BSF_E_CUDA, terr);
        }
      }
    }
    if (s == BSF_OK) {   // G3-FULL on affine sheets: its own kernel (else tile / generic)
      const int grc = bsf::build_g3(h->sh, h->g3, terr, h->dalloc());
      if (grc < 0) s = fail(BSF_E_OOM, terr);
      h->g3_ok = (grc == 0);
    }
    if (s == BSF_OK && !h->generic_ok && !h->tile_ok && !h->g3_ok)
      s = fail(BSF_E_INVALID_ARG, "too many quadrature points per handle (use slabs)");
  }
  cudaSetDevice(prev);
  if (s != BSF_OK) {
    delete h;
    return s;
  }
  *out = h;
  return BSF_OK;
}

bsf_status bsf_destroy(bsf_handle h) {
  delete h;
  return BSF_OK;
}

bsf_status bsf_set_material(bsf_handle h, const bsf_material* mat) {
  if (!h || !mat) return fail(BSF_E_INVALID_ARG, "null argument");
  h->mat = {mat->mu_st1, mat->mu_st2, mat->mu_sh, mat->mu_bd};
  return BSF_OK;
}

bsf_status bsf_get_sizes(bsf_handle h, int64_t* n_rows, int64_t* nnzb, int64_t* n_membrane, int64_t* n_bending) {
  if (!h) return fail(BSF_E_INVALID_ARG, "null handle");
  if (n_rows) *n_rows = (int64_t)(h->sh.r1 - h->sh.r0) * h->sh.n_u;
  if (nnzb) *nnzb = (int64_t)h->sh.col_idx.size();
  if (n_membrane) *n_membrane = (int64_t)h->sh.mem.size();
  if (n_bending) *n_bending = (int64_t)h->sh.bend.size();
  return BSF_OK;
}

bsf_status bsf_get_pattern(bsf_handle h, int32_t* row_ptr, int32_t* col_idx) {
  if (!h) return fail(BSF_E_INVALID_ARG, "null handle");
  if (row_ptr) std::memcpy(row_ptr, h->sh.row_ptr.data(), h->sh.row_ptr.size() * sizeof(int32_t));
  if (col_idx) std::memcpy(col_idx, h->sh.col_idx.data(), h->sh.col_idx.size() * sizeof(int32_t));
  return BSF_OK;
}

static bool use_g3(bsf_handle h, int flags) { return h->g3_ok && !(flags & (BSF_GENERIC_PATH | BSF_TILE_ONLY)); }

bsf_status bsf_eval_all(bsf_handle h, const double* d_x, double* d_energy, double* d_grad, double* d_vals, int flags,
                        bsf_stream stream) {
  if (!h || !d_x) return fail(BSF_E_INVALID_ARG, "null argument");
  if (flags & ~31) return fail(BSF_E_INVALID_ARG, "unknown flag bits");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return fail(BSF_E_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(pe));
  if (bsf_status ss = take_singular(h)) return ss;
  SflagScope sfs(h->sflag_dev);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  const bsf::Mat m = h->mat;
  const int64_t nrows = (int64_t)(h->sh.r1 - h->sh.r0) * h->sh.n_u, nnzb = (int64_t)h->sh.col_idx.size();
  auto st = static_cast<cudaStream_t>(stream);
  int nl = 0;
  int rc;
  if (use_g3(h, flags))
    rc = bsf::g3_eval(h->g3, d_x, 0, m, flags, 1, d_energy, d_grad, 0, d_vals, 0, nullptr, st, &nl, h->dalloc());
  else if (h->tile_ok && !(flags & BSF_GENERIC_PATH))
    rc = bsf::tile_eval(h->tt, h->sh, d_x, 0, m, flags, 1, d_energy, d_grad, 0, d_vals, 0, st, &nl, h->dalloc(), nullptr,
                        (h->core_ok && !(flags & BSF_TILE_ONLY)) ? &h->ct : nullptr, &h->ft);
  else if (!h->generic_ok) {
    if (prev != h->device) cudaSetDevice(prev);
    return fail(BSF_E_INVALID_ARG, "generic path not built for this handle (too many points; use slabs)");
  } else
    rc = bsf::generic_eval(h->gt, d_x, m, flags, nnzb, nrows, d_energy, d_grad, d_vals, st, &nl);
  h->last_launches = nl;
  if (prev != h->device) cudaSetDevice(prev);
  if (rc) return check_cuda("kernel launch") == BSF_OK ? fail(BSF_E_CUDA, "launch failed") : BSF_E_CUDA;
  return BSF_OK;
}

static bool ip_epilogue_forced() {   // debug / comparison switch, read once
  static const bool v = getenv("BSF_IP_EPILOGUE") != nullptr;
  return v;
}

static bsf_status eval_batch_impl(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride, double* d_energy,
                                  double* d_grad, int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags,
                                  bsf_stream stream, const double* d_params, const bsf::IpFused* ip = nullptr) {
  if (h && nbatch == 0) return BSF_OK;   // empty batch: no-op (its pointers may be NULL)
  if (!h || !d_x || nbatch < 0) return fail(BSF_E_INVALID_ARG, "null argument / negative batch");
  if (flags & ~31) return fail(BSF_E_INVALID_ARG, "unknown flag bits");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  const int64_t xn = (int64_t)(h->sh.xhi - h->sh.xlo) * h->sh.n_u * 3;
  const int64_t gn = (int64_t)(h->sh.r1 - h->sh.r0) * h->sh.n_u * 3, vn = (int64_t)h->sh.col_idx.size() * 9;
  if (nbatch > 1 && (x_stride < xn || (d_grad && grad_stride < gn) || (d_vals && vals_stride < vn)))
    return fail(BSF_E_INVALID_ARG, "batch strides smaller than one item");
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return fail(BSF_E_CUDA, std::string("pending CUDA error: ") + cudaGetErrorString(pe));
  if (bsf_status ss = take_singular(h)) return ss;
  SflagScope sfs(h->sflag_dev);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  int nl = 0, rc = 0;
  if (d_params && !use_g3(h, flags) && !(h->tile_ok && h->sh.affine && !(flags & BSF_GENERIC_PATH))) {
    if (prev != h->device) cudaSetDevice(prev);
    return fail(BSF_E_INVALID_ARG, "per-item parameters need an affine sheet on the tile path");
  }
  if (use_g3(h, flags)) {
    if (ip) rc = -1;   // the incremental potential takes the epilogue path on this kernel
    else
      rc = bsf::g3_eval(h->g3, d_x, x_stride, h->mat, flags, nbatch, d_energy, d_grad, grad_stride, d_vals, vals_stride,
                        d_params, st, &nl, h->dalloc());
  } else if (h->tile_ok && !(flags & BSF_GENERIC_PATH)) {
    rc = bsf::tile_eval(h->tt, h->sh, d_x, x_stride, h->mat, flags, nbatch, d_energy, d_grad, grad_stride, d_vals,
                        vals_stride, st, &nl, h->dalloc(), d_params,
                        (h->core_ok && !(flags & BSF_TILE_ONLY)) ? &h->ct : nullptr, &h->ft, ip);
  } else if (!h->generic_ok) {
    if (prev != h->device) cudaSetDevice(prev);
    return fail(BSF_E_INVALID_ARG, "generic path not built for this handle (too many points; use slabs)");
  } else {
    const int64_t nrows = (int64_t)(h->sh.r1 - h->sh.r0) * h->sh.n_u, nnzb = (int64_t)h->sh.col_idx.size();
    for (int b = 0; b < nbatch && rc == 0; ++b) {
      int l = 0;
      rc = bsf::generic_eval(h->gt, d_x + b * x_stride, h->mat, flags, nnzb, nrows, d_energy ? d_energy + b : nullptr,
                             d_grad ? d_grad + b * grad_stride : nullptr, d_vals ? d_vals + b * vals_stride : nullptr,
                             st, &l);
      nl += l;
    }
  }
  h->last_launches = nl;
  if (prev != h->device) cudaSetDevice(prev);
  if (rc) return check_cuda("kernel launch") == BSF_OK ? fail(BSF_E_CUDA, "launch failed") : BSF_E_CUDA;
  return BSF_OK;
}

bsf_status bsf_eval_all_batch(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride, double* d_energy,
                              double* d_grad, int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags,
                              bsf_stream stream) {
  return eval_batch_impl(h, nbatch, d_x, x_stride, d_energy, d_grad, grad_stride, d_vals, vals_stride, flags, stream,
                         nullptr);
}

bsf_status bsf_eval_all_batch_params(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride,
                                     const double* d_params, double* d_energy, double* d_grad, int64_t grad_stride,
                                     double* d_vals, int64_t vals_stride, int flags, bsf_stream stream) {
  if (!d_params) return fail(BSF_E_INVALID_ARG, "null parameters");
  return eval_batch_impl(h, nbatch, d_x, x_stride, d_energy, d_grad, grad_stride, d_vals, vals_stride, flags, stream,
                         d_params);
}

bsf_status bsf_set_inertia(bsf_handle h, double areal_density, double dt, const double* gravity,
                           const uint8_t* pinned) {
  if (!h) return fail(BSF_E_INVALID_ARG, "null handle");
  if (!(dt > 0.0) || !(areal_density >= 0.0)) return fail(BSF_E_INVALID_ARG, "need dt > 0 and areal_density >= 0");
  const bsf::Sheet& sh = h->sh;
  std::vector<double> m;
  std::string err;
  const int rc = bsf::lumped_mass(sh, areal_density, m, err);
  if (rc) return fail(BSF_E_DEGENERATE_GEOMETRY, err);
  const int nu = sh.n_u, nrows = (sh.r1 - sh.r0) * nu;
  std::vector<int32_t> diag(nrows), zero, pin;
  for (int a = 0; a < nrows; ++a) {
    const int32_t ga = sh.r0 * nu + a;
    const int32_t* c0 = sh.col_idx.data() + sh.row_ptr[a];
    const int32_t* c1 = sh.col_idx.data() + sh.row_ptr[a + 1];
    const int32_t* it = std::lower_bound(c0, c1, ga);
    if (it == c1 || *it != ga) return fail(BSF_E_INVALID_ARG, "pattern without a diagonal block");
    diag[a] = (int32_t)(it - sh.col_idx.data());
    if (!pinned) continue;
    const bool pa = pinned[ga] != 0;
    if (pa) pin.push_back(a);
    for (const int32_t* q = c0; q < c1; ++q)
      if ((pa || pinned[*q]) && !(pa && *q == ga)) zero.push_back((int32_t)(q - sh.col_idx.data()));
  }
  if (!h->host_only) {   // a host-only handle keeps the masses (bsf_get_lumped_mass) but cannot evaluate
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != h->device) cudaSetDevice(h->device);
    // in-flight calls may still read the previous tables: finish them before overwriting in place
    if (h->ip_set && cudaDeviceSynchronize() != cudaSuccess) {
      if (prev != h->device) cudaSetDevice(prev);
      return fail(BSF_E_CUDA, "device synchronisation failed");
    }
    bsf_status s = h->upload_reuse(&h->d_mass, &h->cap_mass, m);
    if (s == BSF_OK) s = h->upload_reuse(&h->d_diag, &h->cap_diag, diag);
    if (s == BSF_OK) s = h->upload_reuse(&h->d_zero, &h->cap_zero, zero);
    if (s == BSF_OK) s = h->upload_reuse(&h->d_pin, &h->cap_pin, pin);
    if (prev != h->device) cudaSetDevice(prev);
    if (s != BSF_OK) return s;
  }
  h->h_mass = m;
  h->nzero = (int)zero.size();
  h->npin = (int)pin.size();
  h->ip_k = 1.0 / (dt * dt);
  for (int c = 0; c < 3; ++c) h->ip_g[c] = gravity ? gravity[c] : 0.0;
  h->ip_set = true;
  return BSF_OK;
}

bsf_status bsf_get_lumped_mass(bsf_handle h, double* m) {
  if (!h || !m) return fail(BSF_E_INVALID_ARG, "null argument");
  if (!h->ip_set) return fail(BSF_E_INVALID_ARG, "bsf_set_inertia has not been called");
  std::memcpy(m, h->h_mass.data(), h->h_mass.size() * sizeof(double));
  return BSF_OK;
}

bsf_status bsf_eval_ip_batch(bsf_handle h, int nbatch, const double* d_x, int64_t x_stride, const double* d_xhat,
                             int64_t xhat_stride, const double* d_params, double* d_energy, double* d_grad,
                             int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags, bsf_stream stream) {
  if (h && nbatch == 0) return BSF_OK;   // empty batch: no-op
  if (!h || !d_x || !d_xhat || nbatch < 0) return fail(BSF_E_INVALID_ARG, "null argument / negative batch");
  if (!h->ip_set) return fail(BSF_E_INVALID_ARG, "bsf_set_inertia has not been called");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  const int64_t ncp = (int64_t)(h->sh.r1 - h->sh.r0) * h->sh.n_u;
  if (nbatch > 1 && xhat_stride < 3 * ncp) return fail(BSF_E_INVALID_ARG, "batch strides smaller than one item");
  // fused into the core / band / corner kernels when that path runs (every affine REDUCED sheet), else an
  // epilogue pass after the assembly; the pinned elimination always runs after
  const bool fused = h->tile_ok && h->core_ok && h->ft.ok && !(flags & (BSF_TILE_ONLY | BSF_GENERIC_PATH)) &&
                     !ip_epilogue_forced();
  if (d_params && !(h->sh.affine && h->tt.detJ_ref > 0.0))
    return fail(BSF_E_INVALID_ARG, "per-item parameters need an affine sheet");
  bsf::IpFused ipf;
  ipf.xhat = d_xhat; ipf.xhs = xhat_stride; ipf.mass = h->d_mass; ipf.k = h->ip_k;
  for (int c = 0; c < 3; ++c) ipf.grav[c] = h->ip_g[c];
  ipf.params = d_params; ipf.detJ_ref = h->tt.detJ_ref > 0.0 ? h->tt.detJ_ref : 1.0;   // the sheet's det J
  bsf_status s = eval_batch_impl(h, nbatch, d_x, x_stride, d_energy, d_grad, grad_stride, d_vals, vals_stride, flags,
                                 stream, d_params, fused ? &ipf : nullptr);
  if (s != BSF_OK || nbatch == 0) return s;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  const int64_t need = (int64_t)nbatch * bsf::ip_partials((int)ncp);
  if (!fused && d_energy && need > h->ip_epart_cap) {
    s = h->alloc(&h->d_ip_epart, (size_t)need);
    if (s == BSF_OK) h->ip_epart_cap = need;
  }
  if (s == BSF_OK) {
    bsf::IpArgs A;
    A.x = d_x; A.xs = x_stride; A.xhat = d_xhat; A.xhs = xhat_stride;
    A.g = d_grad; A.gs = grad_stride; A.vals = d_vals; A.vs = vals_stride;
    A.epart = h->d_ip_epart; A.mass = h->d_mass; A.diag = h->d_diag; A.zero_blk = h->d_zero; A.pin_cp = h->d_pin;
    A.nzero = h->nzero; A.npin = h->npin;
    A.ncp = (int)ncp; A.n_u = h->sh.n_u; A.r0 = h->sh.r0; A.xlo = h->sh.xlo;
    A.k = h->ip_k;
    for (int c = 0; c < 3; ++c) A.grav[c] = h->ip_g[c];
    A.params = d_params; A.detJ_ref = ipf.detJ_ref;
    int nl = 0;
    if (fused ? bsf::ip_pin(A, nbatch, static_cast<cudaStream_t>(stream), &nl)
              : bsf::ip_eval(A, nbatch, d_energy, static_cast<cudaStream_t>(stream), &nl))
      s = check_cuda("kernel launch") == BSF_OK ? fail(BSF_E_CUDA, "launch failed") : BSF_E_CUDA;
    h->last_launches += nl;
  }
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

static bsf_status solve_setup(bsf_handle h, bool cg, bsf::SolveArgs& A) {
  const bsf::Sheet& sh = h->sh;
  const int nu = sh.n_u, nrows = (sh.r1 - sh.r0) * nu;
  if (!h->solve_ready) {
    std::vector<int32_t> diag(nrows);
    for (int a = 0; a < nrows; ++a) {
      const int32_t ga = sh.r0 * nu + a;
      const int32_t* c0 = sh.col_idx.data() + sh.row_ptr[a];
      const int32_t* c1 = sh.col_idx.data() + sh.row_ptr[a + 1];
      diag[a] = (int32_t)(std::lower_bound(c0, c1, ga) - sh.col_idx.data());
    }
    bsf_status s = h->upload(&h->d_rp, sh.row_ptr);
    if (s == BSF_OK) s = h->upload(&h->d_ci, sh.col_idx);
    if (s == BSF_OK) s = h->upload(&h->d_sdiag, diag);
    if (s == BSF_OK) s = h->alloc(&h->cg.part, (size_t)bsf::solve_parts(nrows));
    if (s != BSF_OK) return s;
    h->solve_ready = true;
  }
  if (cg && !h->cg_ready) {
    const size_t n3 = 3 * (size_t)nrows;
    bsf_status s = h->alloc(&h->cg.r, n3);
    if (s == BSF_OK) s = h->alloc(&h->cg.z, n3);
    if (s == BSF_OK) s = h->alloc(&h->cg.p, n3);
    if (s == BSF_OK) s = h->alloc(&h->cg.q, n3);
    if (s == BSF_OK) s = h->alloc(&h->cg.dinv, 9 * (size_t)nrows);
    if (s == BSF_OK) s = h->alloc(&h->cg.S, (size_t)bsf::kSN);
    if (s == BSF_OK) s = h->alloc(&h->cg.bad, 1);
    if (s != BSF_OK) return s;
    h->cg.graph = &h->cg_graph;
    h->cg_ready = true;
  }
  A.row_ptr = h->d_rp; A.col_idx = h->d_ci; A.diag = h->d_sdiag;
  A.nrows = nrows; A.n_u = nu; A.r0 = sh.r0; A.xlo = sh.xlo;
  return BSF_OK;
}

bsf_status bsf_bsr_spmv(bsf_handle h, const double* d_vals, const double* d_x, double* d_y, bsf_stream stream) {
  if (!h || !d_vals || !d_x || !d_y) return fail(BSF_E_INVALID_ARG, "null argument");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  if (s == BSF_OK && bsf::spmv(A, d_vals, d_x, d_y, nullptr, static_cast<cudaStream_t>(stream)))
    s = fail(BSF_E_CUDA, "spmv launch failed");
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_gershgorin(bsf_handle h, const double* d_vals, double* lo, double* hi, bsf_stream stream) {
  if (!h || !d_vals || !lo || !hi) return fail(BSF_E_INVALID_ARG, "null argument");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  if (s == BSF_OK && bsf::gershgorin(A, d_vals, h->cg.part, lo, hi, static_cast<cudaStream_t>(stream)))
    s = fail(BSF_E_CUDA, "gershgorin failed");
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_pcg(bsf_handle h, const double* d_vals, const double* d_b, double* d_x, int max_iter, double rtol,
                   int* iters, double* relres, bsf_stream stream) {
  if (!h || !d_vals || !d_b || !d_x) return fail(BSF_E_INVALID_ARG, "null argument");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  if (h->sh.r0 != 0 || h->sh.r1 != h->sh.n_v) return fail(BSF_E_INVALID_ARG, "bsf_pcg needs a whole-sheet handle");
  if (max_iter < 0 || !(rtol > 0.0)) return fail(BSF_E_INVALID_ARG, "need max_iter >= 0 and rtol > 0");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, true, A);
  int it = 0, status = 0;
  double rr = 0.0;
  if (s == BSF_OK && bsf::pcg(A, d_vals, d_b, d_x, h->cg, max_iter, rtol, 16, &it, &rr, &status,
                              static_cast<cudaStream_t>(stream)))
    s = fail(BSF_E_CUDA, "pcg failed");
  if (prev != h->device) cudaSetDevice(prev);
  if (s != BSF_OK) return s;
  if (iters) *iters = it;
  if (relres) *relres = rr;
  if (status == 2) return fail(BSF_E_INVALID_ARG, "matrix not SPD (p.Hp <= 0 or a diagonal block not positive definite)");
  return BSF_OK;
}

bsf_status bsf_chol_factor(bsf_handle h, const double* d_vals, bsf_stream stream) {
  if (!h || !d_vals) return fail(BSF_E_INVALID_ARG, "null argument");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  if (h->sh.r0 != 0 || h->sh.r1 != h->sh.n_v) return fail(BSF_E_INVALID_ARG, "bsf_chol_factor needs a whole-sheet handle");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  std::string err;
  if (s == BSF_OK && !h->chol.ready) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const int rc = bsf::chol_setup(h->chol, h->sh.row_ptr, h->sh.col_idx, A.nrows, fr / 2, err);
    if (rc) s = fail(rc == -7 ? BSF_E_OOM : BSF_E_CUDA, err);
  }
  // the spectrum's Gershgorin lower bound of the factorised matrix (the Neumann gate's denominator)
  double lo = 0.0, hi = 0.0;
  if (s == BSF_OK && bsf::gershgorin(A, d_vals, h->cg.part, &lo, &hi, st)) s = fail(BSF_E_CUDA, "gershgorin failed");
  if (s == BSF_OK) {
    const int rc = bsf::chol_factor(h->chol, h->d_ci, d_vals, st, err);
    if (rc) s = fail(rc == -1 ? BSF_E_INVALID_ARG : BSF_E_CUDA, err);
    h->chol.lam_min_D = lo;
  }
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_chol_solve(bsf_handle h, const double* d_b, double* d_x, bsf_stream stream) {
  if (!h || !d_b || !d_x) return fail(BSF_E_INVALID_ARG, "null argument");
  if (!h->chol.factored) return fail(BSF_E_INVALID_ARG, "no factorisation (bsf_chol_factor)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  std::string err;
  const int rc = bsf::chol_solve(h->chol, d_b, d_x, static_cast<cudaStream_t>(stream), err);
  if (prev != h->device) cudaSetDevice(prev);
  return rc ? fail(BSF_E_CUDA, err) : BSF_OK;
}

bsf_status bsf_neumann_solve(bsf_handle h, const double* d_vals_B, const double* d_b, double* d_x, int max_terms,
                             double rtol, double* gate, int* terms, bsf_stream stream) {
  if (!h || !d_vals_B || !d_b || !d_x || max_terms < 0 || !(rtol > 0.0)) return fail(BSF_E_INVALID_ARG, "bad arguments");
  if (!h->chol.factored) return fail(BSF_E_INVALID_ARG, "no factorisation of D (bsf_chol_factor)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  double lo = 0.0, hi = 0.0;
  if (s == BSF_OK && bsf::gershgorin(A, d_vals_B, h->cg.part, &lo, &hi, st)) s = fail(BSF_E_CUDA, "gershgorin failed");
  // |D^-1 B|_op <= lambda_max(B) / lambda_min(D), both bounded by Gershgorin discs
  const double lmaxB = std::max(std::fabs(lo), std::fabs(hi)), lminD = h->chol.lam_min_D;
  const double g = lminD > 0.0 ? lmaxB / lminD : INFINITY;
  if (gate) *gate = g;
  if (s == BSF_OK && !(g < 1.0))
    s = fail(BSF_E_INVALID_ARG, "Neumann gate not met: lambda_max(B) / lambda_min(D) bound = " + std::to_string(g) +
                                    " >= 1 (factorise D + B instead)");
  if (s == BSF_OK) {
    std::string err;
    const bsf::SpmvFn spmv_b = [&](const double* x, double* y, cudaStream_t ss) {
      return bsf::spmv(A, d_vals_B, x, y, nullptr, ss);
    };
    if (bsf::neumann_solve(h->chol, spmv_b, d_b, d_x, max_terms, rtol, terms, nullptr, st, err))
      s = fail(BSF_E_CUDA, err);
  }
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

// ---- contact pullback (contact.cu, Alg. 1) ----
static bsf_status contact_check(bsf_handle h, const char* what) {
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  if (h->sh.r0 != 0 || h->sh.r1 != h->sh.n_v) return fail(BSF_E_INVALID_ARG, std::string(what) + " needs a whole-sheet handle");
  return BSF_OK;
}

bsf_status bsf_contact_mesh(bsf_handle h, int n_vert, const double* uv) {
  if (!h || n_vert < 0 || (n_vert > 0 && !uv)) return fail(BSF_E_INVALID_ARG, "bad arguments");
  bsf_status s = contact_check(h, "bsf_contact_mesh");
  if (s != BSF_OK) return s;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  std::string err;
  const int rc = bsf::contact_mesh(h->contact, h->sh, n_vert, uv, err);
  if (prev != h->device) cudaSetDevice(prev);
  return rc ? fail(rc == -7 ? BSF_E_OOM : BSF_E_INVALID_ARG, err) : BSF_OK;
}

bsf_status bsf_contact_positions(bsf_handle h, const double* d_x, double* d_xv, bsf_stream stream) {
  if (!h || !d_x || !d_xv) return fail(BSF_E_INVALID_ARG, "null argument");
  if (!h->contact.ready) return fail(BSF_E_INVALID_ARG, "no contact mesh (bsf_contact_mesh)");
  if (h->contact.nvert == 0) return BSF_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  const int rc = bsf::contact_positions(h->contact, d_x, d_xv, static_cast<cudaStream_t>(stream));
  if (prev != h->device) cudaSetDevice(prev);
  return rc ? fail(BSF_E_CUDA, "contact positions launch failed") : BSF_OK;
}

bsf_status bsf_contact_assemble(bsf_handle h, int n_pairs, const int32_t* d_verts, const double* d_H,
                                const double* d_g, double* d_grad, double* d_vals, int64_t* nnzb_off,
                                bsf_stream stream) {
  if (!h || n_pairs < 0 || (n_pairs > 0 && (!d_verts || !d_H))) return fail(BSF_E_INVALID_ARG, "bad arguments");
  if (!h->contact.ready) return fail(BSF_E_INVALID_ARG, "no contact mesh (bsf_contact_mesh)");
  if ((int64_t)n_pairs * 16 > (int64_t)INT32_MAX) return fail(BSF_E_INVALID_ARG, "too many contact pairs");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  if (s == BSF_OK) {
    std::string err;
    const int rc = bsf::contact_assemble(h->contact, n_pairs, d_verts, d_H, d_g, d_grad, d_vals, h->d_sdiag, nnzb_off,
                                         static_cast<cudaStream_t>(stream), err);
    if (rc) s = fail(rc == -7 ? BSF_E_OOM : rc == -1 ? BSF_E_INVALID_ARG : BSF_E_CUDA, err);
  }
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_contact_get(bsf_handle h, int32_t* d_row_ptr, int32_t* d_col_idx, double* d_vals, bsf_stream stream) {
  if (!h) return fail(BSF_E_INVALID_ARG, "null handle");
  const bsf::ContactState& C = h->contact;
  if (!C.assembled) return fail(BSF_E_INVALID_ARG, "no contact assembly (bsf_contact_assemble)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  bool ok = true;
  if (d_row_ptr)
    ok &= cudaMemcpyAsync(d_row_ptr, C.row_ptr, sizeof(int32_t) * (C.ncp + 1), cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  if (d_col_idx && C.nnz)
    ok &= cudaMemcpyAsync(d_col_idx, C.col, sizeof(int32_t) * C.nnz, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  if (d_vals && C.nnz)
    ok &= cudaMemcpyAsync(d_vals, C.vals, sizeof(double) * 9 * C.nnz, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
  if (prev != h->device) cudaSetDevice(prev);
  return ok ? BSF_OK : fail(BSF_E_CUDA, "contact copy failed");
}

bsf_status bsf_contact_neumann_solve(bsf_handle h, const double* d_b, double* d_x, int max_terms, double rtol,
                                     double* gate, int* terms, bsf_stream stream) {
  if (!h || !d_b || !d_x || max_terms < 0 || !(rtol > 0.0)) return fail(BSF_E_INVALID_ARG, "bad arguments");
  if (!h->chol.factored) return fail(BSF_E_INVALID_ARG, "no factorisation of D (bsf_chol_factor)");
  if (!h->contact.assembled) return fail(BSF_E_INVALID_ARG, "no contact assembly (bsf_contact_assemble)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  bsf::SolveArgs A;
  bsf_status s = solve_setup(h, false, A);
  // B = H_barrier,od in its own pattern (no diagonal blocks: those were merged into D)
  bsf::SolveArgs B = A;
  B.row_ptr = h->contact.row_ptr; B.col_idx = h->contact.col; B.diag = nullptr;
  double lo = 0.0, hi = 0.0;
  if (s == BSF_OK && h->contact.nnz > 0 && bsf::gershgorin(B, h->contact.vals, h->cg.part, &lo, &hi, st))
    s = fail(BSF_E_CUDA, "gershgorin failed");
  const double lmaxB = std::max(std::fabs(lo), std::fabs(hi)), lminD = h->chol.lam_min_D;
  const double g = lminD > 0.0 ? lmaxB / lminD : INFINITY;
  if (gate) *gate = g;
  if (s == BSF_OK && !(g < 1.0))
    s = fail(BSF_E_INVALID_ARG, "Neumann gate not met: lambda_max(B) / lambda_min(D) bound = " + std::to_string(g) +
                                    " >= 1 (factorise D + B instead)");
  if (s == BSF_OK) {
    std::string err;
    const double* vb = h->contact.vals;
    const bsf::SpmvFn spmv_b = [&](const double* x, double* y, cudaStream_t ss) {
      return bsf::spmv(B, vb, x, y, nullptr, ss);
    };
    if (bsf::neumann_solve(h->chol, spmv_b, d_b, d_x, max_terms, rtol, terms, nullptr, st, err))
      s = fail(BSF_E_CUDA, err);
  }
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_eval_all_batch_host(bsf_handle h, int nbatch, const double* h_x, int64_t x_stride, double* d_x_stage,
                                   const double* d_params, double* h_energy, double* d_energy, double* d_grad,
                                   int64_t grad_stride, double* d_vals, int64_t vals_stride, int flags, int chunk,
                                   bsf_stream stream) {
  if (h && nbatch == 0) return BSF_OK;   // empty batch: no-op
  if (!h || !h_x || !d_x_stage || nbatch < 0) return fail(BSF_E_INVALID_ARG, "null argument / negative batch");
  if (h_energy && !d_energy) return fail(BSF_E_INVALID_ARG, "h_energy needs the device energy buffer");
  const bool async_stage = (flags & BSF_ASYNC_STAGE) != 0;
  flags &= ~BSF_ASYNC_STAGE;
  if (nbatch == 0) return BSF_OK;
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle (device = -1) cannot compute");
  const int64_t xn = (int64_t)(h->sh.xhi - h->sh.xlo) * h->sh.n_u * 3;
  if (nbatch > 1 && x_stride < xn) return fail(BSF_E_INVALID_ARG, "batch strides smaller than one item");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  if (!h->copy_stream) {
    if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_copy, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) != cudaSuccess) {
      if (prev != h->device) cudaSetDevice(prev);
      return fail(BSF_E_CUDA, "stream creation failed");
    }
  }
  // chunk plan: fixed size if given, else geometric (nbatch/10, then doubling) so that each chunk's
  // assembly covers the next, larger upload while the first exposed upload stays small
  // (BSF_ASYNC_STAGE: one chunk by default, the previous call's assembly already covers this upload)
  int ch = chunk > 0 ? chunk : (async_stage ? nbatch : std::max(1, (nbatch + 9) / 10));
  // the uploads run on the copy stream, after the work already queued on `stream` (stage reuse)
  bsf_status s = BSF_OK;
  bsf_sheet::StageUse* use = nullptr;
  if (async_stage) {
    for (bsf_sheet::StageUse& u : h->stage_uses)
      if (u.ptr == d_x_stage) use = &u;
    if (!use) {
      if (h->stage_uses.size() >= 8) {   // bounded: forget the oldest stage (its event is released on completion)
        cudaEventDestroy(h->stage_uses.front().done);
        h->stage_uses.erase(h->stage_uses.begin());
      }
      bsf_sheet::StageUse u{d_x_stage, nullptr};
      if (cudaEventCreateWithFlags(&u.done, cudaEventDisableTiming) != cudaSuccess) {
        if (prev != h->device) cudaSetDevice(prev);
        return fail(BSF_E_CUDA, "event creation failed");
      }
      // first use of this stage: order after everything queued so far (as without the flag)
      if (cudaEventRecord(u.done, st) != cudaSuccess) s = fail(BSF_E_CUDA, "event");
      h->stage_uses.push_back(u);
      use = &h->stage_uses.back();
    }
    if (s == BSF_OK && cudaStreamWaitEvent(h->copy_stream, use->done, 0) != cudaSuccess) s = fail(BSF_E_CUDA, "event");
  } else if (cudaEventRecord(h->ev_start, st) != cudaSuccess ||
             cudaStreamWaitEvent(h->copy_stream, h->ev_start, 0) != cudaSuccess) {
    s = fail(BSF_E_CUDA, "event");
  }
  int launches = 0;
  for (int b0 = 0, nb = 0; b0 < nbatch && s == BSF_OK; b0 += nb, ch = chunk > 0 ? ch : 2 * ch) {
    nb = std::min(ch, nbatch - b0);
    const size_t bytes = sizeof(double) * (size_t)((int64_t)(nb - 1) * x_stride + xn);
    if (cudaMemcpyAsync(d_x_stage + b0 * x_stride, h_x + b0 * x_stride, bytes, cudaMemcpyHostToDevice,
                        h->copy_stream) != cudaSuccess ||
        cudaEventRecord(h->ev_copy, h->copy_stream) != cudaSuccess || cudaStreamWaitEvent(st, h->ev_copy, 0) != cudaSuccess) {
      s = fail(BSF_E_CUDA, "position upload");
      break;
    }
    s = eval_batch_impl(h, nb, d_x_stage + b0 * x_stride, x_stride, d_energy ? d_energy + b0 : nullptr,
                        d_grad ? d_grad + b0 * grad_stride : nullptr, grad_stride,
                        d_vals ? d_vals + b0 * vals_stride : nullptr, vals_stride, flags, stream,
                        d_params ? d_params + 9 * (int64_t)b0 : nullptr);
    launches += h->last_launches;
  }
  if (s == BSF_OK && use && cudaEventRecord(use->done, st) != cudaSuccess) s = fail(BSF_E_CUDA, "event");
  if (s == BSF_OK && h_energy &&
      cudaMemcpyAsync(h_energy, d_energy, sizeof(double) * nbatch, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    s = fail(BSF_E_CUDA, "energy download");
  h->last_launches = launches;
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

bsf_status bsf_eval_energy(bsf_handle h, const double* d_x, double* d_energy, int flags, bsf_stream stream) {
  if (!d_energy) return fail(BSF_E_INVALID_ARG, "null energy");
  return bsf_eval_all(h, d_x, d_energy, nullptr, nullptr, flags, stream);
}
bsf_status bsf_eval_gradient(bsf_handle h, const double* d_x, double* d_grad, int flags, bsf_stream stream) {
  if (!d_grad) return fail(BSF_E_INVALID_ARG, "null gradient");
  return bsf_eval_all(h, d_x, nullptr, d_grad, nullptr, flags, stream);
}
bsf_status bsf_assemble_hessian(bsf_handle h, const double* d_x, double* d_vals, int flags, bsf_stream stream) {
  if (!d_vals) return fail(BSF_E_INVALID_ARG, "null values");
  return bsf_eval_all(h, d_x, nullptr, nullptr, d_vals, flags, stream);
}

int bsf_last_launch_count(bsf_handle h) { return h ? h->last_launches : 0; }

bsf_status bsf_poll_status(bsf_handle h) {
  if (!h) return fail(BSF_E_INVALID_ARG, "null handle");
  return take_singular(h);
}

bsf_status bsf_affine_params(int n_u, int n_v, const double* rest_xy, const bsf_material* mat, double* out9) {
  if (!rest_xy || !mat || !out9) return fail(BSF_E_INVALID_ARG, "null argument");
  const double mu[4] = {mat->mu_st1, mat->mu_st2, mat->mu_sh, mat->mu_bd};
  std::string err;
  const int rc = bsf::affine_params(n_u, n_v, rest_xy, mu, out9, err);
  return rc ? fail((bsf_status)rc, err) : BSF_OK;
}

bsf_status bsf_get_core_rect(bsf_handle h, int32_t* rect4) {
  if (!h || !rect4) return fail(BSF_E_INVALID_ARG, "null argument");
  const bool on = h->core_ok;
  rect4[0] = on ? h->ct.CI0 : 0;
  rect4[1] = on ? h->ct.CI1 : 0;
  rect4[2] = on ? h->ct.RJ0 : 0;
  rect4[3] = on ? h->ct.RJ1 : 0;
  return BSF_OK;
}

}  // extern "C"

namespace bsf {
int nccl_unique_id(void* out128, std::string& err);
int nccl_comm_init(void** comm, int nranks, const void* id128, int rank, std::string& err);
int nccl_comm_destroy(void* comm, std::string& err);
int nccl_halo_exchange(double* d_x, int n_u, int r0, int r1, int xlo, int xhi, int rank, int nranks, void* comm,
                       void* stream, std::string& err);
int nccl_allreduce_sum(double* d_buf, size_t n, void* comm, void* stream, std::string& err);
void halo_plan(int n_u, int r0, int r1, int xlo, int xhi, int rank, int nranks, int64_t plan[8]);
}  // namespace bsf

extern "C" bsf_status bsf_halo_plan(bsf_handle h, int rank, int nranks, int64_t* plan8) {
  if (!h || !plan8 || nranks < 1 || rank < 0 || rank >= nranks) return fail(BSF_E_INVALID_ARG, "bad plan arguments");
  const bsf::Sheet& sh = h->sh;
  if (nranks > 1 && sh.r1 - sh.r0 < 2) return fail(BSF_E_INVALID_ARG, "every slab must own at least 2 rows");
  bsf::halo_plan(sh.n_u, sh.r0, sh.r1, sh.xlo, sh.xhi, rank, nranks, plan8);
  return BSF_OK;
}

extern "C" bsf_status bsf_nccl_get_unique_id(void* out128) {
  if (!out128) return fail(BSF_E_INVALID_ARG, "null id buffer");
  std::string err;
  return bsf::nccl_unique_id(out128, err) ? fail(BSF_E_NCCL, err) : BSF_OK;
}

extern "C" bsf_status bsf_nccl_comm_init(int nranks, const void* id128, int rank, int device, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(BSF_E_INVALID_ARG, "bad comm arguments");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  std::string err;
  const int rc = bsf::nccl_comm_init(comm, nranks, id128, rank, err);
  cudaSetDevice(prev);
  return rc ? fail(BSF_E_NCCL, err) : BSF_OK;
}

extern "C" bsf_status bsf_nccl_comm_destroy(void* comm) {
  if (!comm) return BSF_OK;
  std::string err;
  return bsf::nccl_comm_destroy(comm, err) ? fail(BSF_E_NCCL, err) : BSF_OK;
}

extern "C" bsf_status bsf_halo_exchange(bsf_handle h, double* d_x, void* nccl_comm, int rank, int nranks,
                                        bsf_stream stream) {
  if (!h || !d_x || !nccl_comm || rank < 0 || rank >= nranks) return fail(BSF_E_INVALID_ARG, "bad halo arguments");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle");
  const bsf::Sheet& sh = h->sh;
  if ((rank > 0 && sh.r1 - sh.r0 < 2) || (rank < nranks - 1 && sh.r1 - sh.r0 < 2))
    return fail(BSF_E_INVALID_ARG, "every slab must own at least 2 rows");
  std::string err;
  const int rc = bsf::nccl_halo_exchange(d_x, sh.n_u, sh.r0, sh.r1, sh.xlo, sh.xhi, rank, nranks, nccl_comm, stream, err);
  return rc ? fail(BSF_E_NCCL, err) : BSF_OK;
}

extern "C" bsf_status bsf_eval_all_slab(bsf_handle h, double* d_x, void* nccl_comm, int rank, int nranks,
                                        double* d_energy, double* d_grad, double* d_vals, int flags,
                                        bsf_stream stream) {
  if (!h || !d_x || rank < 0 || rank >= nranks) return fail(BSF_E_INVALID_ARG, "bad slab arguments");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle");
  if (flags & ~31) return fail(BSF_E_INVALID_ARG, "unknown flag bits");
  const bsf::Sheet& sh = h->sh;
  const bool exchange = nranks > 1;
  if (exchange && !nccl_comm) return fail(BSF_E_INVALID_ARG, "null communicator");
  if (exchange && sh.r1 - sh.r0 < 2) return fail(BSF_E_INVALID_ARG, "every slab must own at least 2 rows");
  if (bsf_status ss = take_singular(h)) return ss;
  SflagScope sfs(h->sflag_dev);
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  auto st = static_cast<cudaStream_t>(stream);
  bsf_status s = BSF_OK;
  const bool fused = h->tile_ok && h->core_ok && h->ft.ok && !(flags & (BSF_TILE_ONLY | BSF_GENERIC_PATH));
  // interior core rows: the gather of row j reads control-point rows j-4 .. j+3 (knot-row pairs of the
  // prologue), so rows [r0+4, r1-4) need no halo; the boundary rows wait for the exchange
  bsf::HaloOverlap ov{0, 0, nullptr};
  static const bool force_split = getenv("BSF_SLAB_SPLIT") != nullptr;   // test switch: split without exchange
  if (fused && (exchange || force_split)) {
    ov.ja = std::max(h->ct.RJ0, rank > 0 ? sh.r0 + 4 : h->ct.RJ0);
    ov.jb = std::min(h->ct.RJ1, rank < nranks - 1 ? sh.r1 - 4 : h->ct.RJ1);
  }
  if (!exchange && ov.jb > ov.ja) {   // forced split on one rank: `ready` is an already-reached point of st
    if (!h->ev_halo && cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess)
      s = fail(BSF_E_CUDA, "event");
    if (s == BSF_OK && cudaEventRecord(h->ev_halo, st) != cudaSuccess) s = fail(BSF_E_CUDA, "event");
    ov.ready = h->ev_halo;
    ov.ja = std::max(h->ct.RJ0, sh.r0 + 4);
    ov.jb = std::min(h->ct.RJ1, sh.r1 - 4);
  }
  if (exchange) {
    if (!h->comm_stream &&
        (cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&h->ev_halo0, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess))
      s = fail(BSF_E_CUDA, "stream creation failed");
    std::string err;
    if (s == BSF_OK && (cudaEventRecord(h->ev_halo0, st) != cudaSuccess ||
                        cudaStreamWaitEvent(h->comm_stream, h->ev_halo0, 0) != cudaSuccess))
      s = fail(BSF_E_CUDA, "event");
    if (s == BSF_OK && bsf::nccl_halo_exchange(d_x, sh.n_u, sh.r0, sh.r1, sh.xlo, sh.xhi, rank, nranks, nccl_comm,
                                               h->comm_stream, err))
      s = fail(BSF_E_NCCL, err);
    if (s == BSF_OK && cudaEventRecord(h->ev_halo, h->comm_stream) != cudaSuccess) s = fail(BSF_E_CUDA, "event");
    ov.ready = h->ev_halo;
    if (s == BSF_OK && !(ov.jb > ov.ja) && cudaStreamWaitEvent(st, h->ev_halo, 0) != cudaSuccess)   // no overlap
      s = fail(BSF_E_CUDA, "event");
  }
  int nl = 0;
  if (s == BSF_OK) {
    int rc;
    if (use_g3(h, flags)) {
      if (ov.jb > ov.ja && cudaStreamWaitEvent(st, ov.ready, 0) != cudaSuccess) rc = -6;   // no split on this path
      else rc = bsf::g3_eval(h->g3, d_x, 0, h->mat, flags, 1, d_energy, d_grad, 0, d_vals, 0, nullptr, st, &nl, h->dalloc());
    } else if (h->tile_ok && !(flags & BSF_GENERIC_PATH))
      rc = bsf::tile_eval(h->tt, sh, d_x, 0, h->mat, flags, 1, d_energy, d_grad, 0, d_vals, 0, st, &nl, h->dalloc(),
                          nullptr, (h->core_ok && !(flags & BSF_TILE_ONLY)) ? &h->ct : nullptr, &h->ft, nullptr,
                          (ov.jb > ov.ja) ? &ov : nullptr);
    else if (!h->generic_ok)
      rc = -100;
    else
      rc = bsf::generic_eval(h->gt, d_x, h->mat, flags, (int64_t)sh.col_idx.size(), (int64_t)(sh.r1 - sh.r0) * sh.n_u,
                             d_energy, d_grad, d_vals, st, &nl);
    if (rc == -100) s = fail(BSF_E_INVALID_ARG, "generic path not built for this handle (too many points; use slabs)");
    else if (rc) s = check_cuda("kernel launch") == BSF_OK ? fail(BSF_E_CUDA, "launch failed") : BSF_E_CUDA;
  }
  h->last_launches = nl;
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

extern "C" bsf_status bsf_set_kernel_timing(bsf_handle h, int ncalls) {
  if (!h || ncalls < 0) return fail(BSF_E_INVALID_ARG, "bad arguments");
  if (h->host_only) return fail(BSF_E_NO_DEVICE, "host-only handle");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (cudaEvent_t e : h->tt.tev) cudaEventDestroy(e);
  h->tt.tev.assign(4 * (size_t)ncalls, nullptr);
  bsf_status s = BSF_OK;
  for (cudaEvent_t& e : h->tt.tev)
    if (cudaEventCreate(&e) != cudaSuccess) { s = fail(BSF_E_CUDA, "event creation failed"); break; }
  h->tt.tev_n = s == BSF_OK ? ncalls : 0;
  h->tt.tev_next = h->tt.tev_count = 0;
  if (prev != h->device) cudaSetDevice(prev);
  return s;
}

extern "C" int bsf_get_kernel_timing(bsf_handle h, float* core_ms, float* band_ms, int n) {
  if (!h || h->tt.tev_n == 0) return 0;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != h->device) cudaSetDevice(h->device);
  const int cnt = std::min(n, h->tt.tev_count);
  // oldest first: the ring's last `cnt` calls
  for (int k = 0; k < cnt; ++k) {
    const int slot = ((h->tt.tev_next - cnt + k) % h->tt.tev_n + h->tt.tev_n) % h->tt.tev_n;
    cudaEvent_t* tv = h->tt.tev.data() + 4 * slot;
    cudaEventSynchronize(tv[1]);
    cudaEventSynchronize(tv[3]);
    if (core_ms && cudaEventElapsedTime(&core_ms[k], tv[0], tv[1]) != cudaSuccess) core_ms[k] = -1.0f;
    if (band_ms && cudaEventElapsedTime(&band_ms[k], tv[2], tv[3]) != cudaSuccess) band_ms[k] = -1.0f;
  }
  if (prev != h->device) cudaSetDevice(prev);
  return cnt;
}

extern "C" bsf_status bsf_allreduce_sum(double* d_buf, int64_t n, void* nccl_comm, bsf_stream stream) {
  if (!d_buf || !nccl_comm || n < 0) return fail(BSF_E_INVALID_ARG, "bad allreduce arguments");
  std::string err;
  return bsf::nccl_allreduce_sum(d_buf, (size_t)n, nccl_comm, stream, err) ? fail(BSF_E_NCCL, err) : BSF_OK;
}
