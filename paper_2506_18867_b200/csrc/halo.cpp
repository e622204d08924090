// Multi-GPU row-slab plumbing: NCCL is loaded at run time (dlopen of
// the process's libnccl.so.2, e.g. the one torch ships), so the library has no link-time NCCL
// dependency.  A slab owns control-point rows [r0, r1); its position buffer holds rows
// [max(0, r0-2), min(n_v, r1+2)).  The exchange sends the first / last two owned rows to the
// previous / next slab and receives their rows into the halo, all inside one NCCL group.
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

namespace bsf_nccl {

// Minimal NCCL ABI (stable since NCCL 2.x): opaque handles, enums as int.
typedef void* ncclComm_t;
typedef void* cudaStream_t_;
struct ncclUniqueId { char internal[128]; };
typedef int (*GetUniqueId_t)(ncclUniqueId*);
typedef int (*CommInitRank_t)(ncclComm_t*, int, ncclUniqueId, int);
typedef int (*CommDestroy_t)(ncclComm_t);
typedef int (*Send_t)(const void*, size_t, int, int, ncclComm_t, cudaStream_t_);
typedef int (*Recv_t)(void*, size_t, int, int, ncclComm_t, cudaStream_t_);
typedef int (*Group_t)();
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t_);
typedef const char* (*GetErrorString_t)(int);

struct Api {
  bool ok = false;
  std::string err;
  GetUniqueId_t getUniqueId = nullptr;
  CommInitRank_t commInitRank = nullptr;
  CommDestroy_t commDestroy = nullptr;
  Send_t send = nullptr;
  Recv_t recv = nullptr;
  Group_t groupStart = nullptr, groupEnd = nullptr;
  AllReduce_t allReduce = nullptr;
  GetErrorString_t errStr = nullptr;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { a.err = std::string("cannot load libnccl.so.2: ") + dlerror(); return; }
    a.getUniqueId = (GetUniqueId_t)dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (CommInitRank_t)dlsym(h, "ncclCommInitRank");
    a.commDestroy = (CommDestroy_t)dlsym(h, "ncclCommDestroy");
    a.send = (Send_t)dlsym(h, "ncclSend");
    a.recv = (Recv_t)dlsym(h, "ncclRecv");
    a.groupStart = (Group_t)dlsym(h, "ncclGroupStart");
    a.groupEnd = (Group_t)dlsym(h, "ncclGroupEnd");
    a.allReduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
    a.errStr = (GetErrorString_t)dlsym(h, "ncclGetErrorString");
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.send && a.recv && a.groupStart && a.groupEnd &&
           a.allReduce;
    if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

}  // namespace bsf_nccl

namespace bsf {
// ncclDataType_t ncclFloat64 = 8 (ncclDouble), ncclRedOp_t ncclSum = 0
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

int nccl_unique_id(void* out128, std::string& err) {
  const auto& a = bsf_nccl::api();
  if (!a.ok) { err = a.err; return -8; }
  bsf_nccl::ncclUniqueId id;
  const int rc = a.getUniqueId(&id);
  if (rc) { err = "ncclGetUniqueId failed"; return -8; }
  std::memcpy(out128, id.internal, 128);
  return 0;
}

int nccl_comm_init(void** comm, int nranks, const void* id128, int rank, std::string& err) {
  const auto& a = bsf_nccl::api();
  if (!a.ok) { err = a.err; return -8; }
  bsf_nccl::ncclUniqueId id;
  std::memcpy(id.internal, id128, 128);
  bsf_nccl::ncclComm_t c = nullptr;
  const int rc = a.commInitRank(&c, nranks, id, rank);
  if (rc) { err = std::string("ncclCommInitRank failed: ") + (a.errStr ? a.errStr(rc) : "?"); return -8; }
  *comm = c;
  return 0;
}

int nccl_comm_destroy(void* comm, std::string& err) {
  const auto& a = bsf_nccl::api();
  if (!a.ok) { err = a.err; return -8; }
  return a.commDestroy(comm) ? -8 : 0;
}

// The exchange plan of a slab: rows owned [r0, r1), buffer rows [xlo, xhi), n_u cps per row,
// 3 doubles per cp.  plan[4 d + 0..3] for d = 0 (peer rank-1, below) and d = 1 (peer rank+1, above):
// peer rank (-1: none), send offset, receive offset, count — offsets and count in doubles of the buffer.
// The slab sends its first / last nlo / nhi owned rows and receives the peer's into its halo rows.
void halo_plan(int n_u, int r0, int r1, int xlo, int xhi, int rank, int nranks, int64_t plan[8]) {
  const int64_t row = (int64_t)n_u * 3;
  const int nlo = r0 - xlo, nhi = xhi - r1;   // halo rows below / above (0..2)
  for (int k = 0; k < 8; ++k) plan[k] = 0;
  plan[0] = plan[4] = -1;
  if (rank > 0 && nlo > 0) {
    plan[0] = rank - 1; plan[1] = (int64_t)(r0 - xlo) * row; plan[2] = 0; plan[3] = (int64_t)nlo * row;
  }
  if (rank < nranks - 1 && nhi > 0) {
    plan[4] = rank + 1; plan[5] = (int64_t)(r1 - nhi - xlo) * row; plan[6] = (int64_t)(r1 - xlo) * row;
    plan[7] = (int64_t)nhi * row;
  }
}

int nccl_halo_exchange(double* d_x, int n_u, int r0, int r1, int xlo, int xhi, int rank, int nranks, void* comm,
                       void* stream, std::string& err) {
  const auto& a = bsf_nccl::api();
  if (!a.ok) { err = a.err; return -8; }
  int64_t plan[8];
  halo_plan(n_u, r0, r1, xlo, xhi, rank, nranks, plan);
  int rc = a.groupStart();
  for (int d = 0; d < 2; ++d) {
    const int64_t* p = plan + 4 * d;
    if (p[0] < 0) continue;
    rc |= a.send(d_x + p[1], (size_t)p[3], kNcclFloat64, (int)p[0], comm, stream);
    rc |= a.recv(d_x + p[2], (size_t)p[3], kNcclFloat64, (int)p[0], comm, stream);
  }
  rc |= a.groupEnd();
  if (rc) { err = "NCCL halo exchange failed"; return -8; }
  return 0;
}

int nccl_allreduce_sum(double* d_buf, size_t n, void* comm, void* stream, std::string& err) {
  const auto& a = bsf_nccl::api();
  if (!a.ok) { err = a.err; return -8; }
  return a.allReduce(d_buf, d_buf, n, kNcclFloat64, kNcclSum, comm, stream) ? (err = "ncclAllReduce failed", -8) : 0;
}

}  // namespace bsf
