// Multi-GPU plumbing of the Z-sub-part sharding: one NCCL
// communicator per rank, the one-known-plane halo exchange between
// neighbouring ranks and the gather of every rank's core planes on rank 0,
// as grouped point-to-point sends / receives on the caller's stream.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2") so the library has no
// link-time NCCL dependency and shares the NCCL a host process (torch)
// already loaded.  The communicator is created from a unique id the host
// broadcasts (torch.distributed, MPI, a file ...).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cstdint>
#include <cstring>
#include <string>
#include "../../include/volkrig_b200.h"

namespace vk {
int comm_set_err(int status, const std::string& msg);   // vk_api.cu
}

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
#define VK_SYM(field, name)                                                  \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));             \
  if (!a.field) {                                                            \
    a.why = std::string("NCCL symbol missing: ") + name;                     \
    return a;                                                                \
  }
    VK_SYM(get_unique_id, "ncclGetUniqueId")
    VK_SYM(comm_init_rank, "ncclCommInitRank")
    VK_SYM(comm_destroy, "ncclCommDestroy")
    VK_SYM(comm_count, "ncclCommCount")
    VK_SYM(comm_user_rank, "ncclCommUserRank")
    VK_SYM(group_start, "ncclGroupStart")
    VK_SYM(group_end, "ncclGroupEnd")
    VK_SYM(send, "ncclSend")
    VK_SYM(recv, "ncclRecv")
    VK_SYM(error_string, "ncclGetErrorString")
#undef VK_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

int nccl_err(const char* what, ncclResult_t r) {
  return vk::comm_set_err(VK_E_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

#define VK_NCCL(call)                                        \
  do {                                                       \
    const ncclResult_t r_ = (call);                          \
    if (r_ != ncclSuccess) return nccl_err(#call, r_);       \
  } while (0)

// inside ncclGroupStart/End: keep the first failure, carry on to group_end
// (an open group would capture the process's later NCCL calls, torch's too)
#define VK_NCCL_G(first, call)                               \
  do {                                                       \
    const ncclResult_t r_ = (call);                          \
    if (r_ != ncclSuccess && first.r == ncclSuccess) {       \
      first.r = r_;                                          \
      first.what = #call;                                    \
    }                                                        \
  } while (0)

struct GroupErr {
  ncclResult_t r = ncclSuccess;
  const char* what = "";
};

int need_nccl() {
  if (!nccl().ok) return vk::comm_set_err(VK_E_UNSUPPORTED, nccl().why);
  return VK_OK;
}

}  // namespace

extern "C" {

int vk_comm_unique_id(unsigned char* id) {
  if (!id) return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "null id");
  if (int e = need_nccl()) return e;
  ncclUniqueId u;
  VK_NCCL(nccl().get_unique_id(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return VK_OK;
}

int vk_comm_create(const unsigned char* id, int32_t world, int32_t rank, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world)
    return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_comm_create: id, comm, 0 <= rank < world");
  if (int e = need_nccl()) return e;
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  VK_NCCL(nccl().comm_init_rank(&c, world, u, rank));
  *comm = c;
  return VK_OK;
}

int vk_comm_destroy(void* comm) {
  if (!comm) return VK_OK;
  if (int e = need_nccl()) return e;
  VK_NCCL(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
  return VK_OK;
}

int vk_halo_exchange(void* comm, const float* first_plane, float* halo, int64_t n, void* stream) {
  if (!comm || n < 0) return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_halo_exchange: comm, n");
  if (int e = need_nccl()) return e;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 0, rank = 0;
  VK_NCCL(nccl().comm_count(c, &world));
  VK_NCCL(nccl().comm_user_rank(c, &rank));
  if ((rank > 0 && !first_plane) || (rank < world - 1 && !halo))
    return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_halo_exchange: null plane");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GroupErr ge;
  VK_NCCL(nccl().group_start());
  if (rank > 0) VK_NCCL_G(ge, nccl().send(first_plane, (size_t)n, ncclFloat32, rank - 1, c, st));
  if (rank < world - 1) VK_NCCL_G(ge, nccl().recv(halo, (size_t)n, ncclFloat32, rank + 1, c, st));
  VK_NCCL(nccl().group_end());
  if (ge.r != ncclSuccess) return nccl_err(ge.what, ge.r);
  return VK_OK;
}

int vk_gather_core(void* comm, const float* core, const int64_t* counts, float* out, void* stream) {
  if (!comm || !counts) return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_gather_core: comm, counts");
  if (int e = need_nccl()) return e;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 0, rank = 0;
  VK_NCCL(nccl().comm_count(c, &world));
  VK_NCCL(nccl().comm_user_rank(c, &rank));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rank == 0) {
    if (!out || (counts[0] > 0 && !core)) return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_gather_core: out");
    if (counts[0] > 0) {
      const cudaError_t ce = cudaMemcpyAsync(out, core, (size_t)counts[0] * sizeof(float),
                                             cudaMemcpyDeviceToDevice, st);
      if (ce != cudaSuccess) return vk::comm_set_err(VK_E_CUDA, cudaGetErrorString(ce));
    }
    int64_t off = counts[0];
    GroupErr ge;
    VK_NCCL(nccl().group_start());
    for (int r = 1; r < world; ++r) {
      if (counts[r] > 0) VK_NCCL_G(ge, nccl().recv(out + off, (size_t)counts[r], ncclFloat32, r, c, st));
      off += counts[r];
    }
    VK_NCCL(nccl().group_end());
    if (ge.r != ncclSuccess) return nccl_err(ge.what, ge.r);
  } else if (counts[rank] > 0) {
    if (!core) return vk::comm_set_err(VK_E_INVALID_ARGUMENT, "vk_gather_core: core");
    VK_NCCL(nccl().send(core, (size_t)counts[rank], ncclFloat32, 0, c, st));
  }
  return VK_OK;
}

}  // extern "C"
