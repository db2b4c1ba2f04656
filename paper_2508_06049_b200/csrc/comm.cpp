// NCCL binding at run time.  See comm.hpp.
#include "comm.hpp"

#include <dlfcn.h>

#include <string>

#include "common.hpp"

namespace kb {
namespace {

// the subset of nccl.h the sharded solver uses (ABI-stable since NCCL 2.7)
using nccl_result = int;
using nccl_comm = void*;
struct nccl_uid {
  char internal[128];
};
constexpr int kNcclFloat64 = 8;

struct Nccl {
  nccl_result (*get_unique_id)(nccl_uid*) = nullptr;
  nccl_result (*comm_init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  nccl_result (*comm_destroy)(nccl_comm) = nullptr;
  nccl_result (*send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
};

const Nccl& nccl() {
  static Nccl api;
  static bool loaded = false;
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(KB_CUDA, std::string("NCCL not available: ") + dlerror());
  auto sym = [&](const char* name) {
    void* p = dlsym(h, name);
    if (!p) fail(KB_CUDA, std::string("NCCL symbol missing: ") + name);
    return p;
  };
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
  api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
  api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  loaded = true;
  return api;
}

void check(nccl_result r, const char* what) {
  if (r != 0) fail(KB_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

void NcclComm::unique_id(unsigned char out[128]) {
  nccl_uid id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  for (int i = 0; i < 128; ++i) out[i] = static_cast<unsigned char>(id.internal[i]);
}

NcclComm::NcclComm(int nranks, int rank, const unsigned char id[128]) : nranks_(nranks), rank_(rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(KB_STRUCTURAL, "communicator rank out of range");
  nccl_uid uid;
  for (int i = 0; i < 128; ++i) uid.internal[i] = static_cast<char>(id[i]);
  check(nccl().comm_init_rank(&comm_, nranks, uid, rank), "ncclCommInitRank");
}

NcclComm::~NcclComm() {
  if (comm_) nccl().comm_destroy(comm_);
}

void NcclComm::group_start() { check(nccl().group_start(), "ncclGroupStart"); }
void NcclComm::group_end() { check(nccl().group_end(), "ncclGroupEnd"); }
void NcclComm::send(const double* buf, size_t count, int peer, cudaStream_t st) {
  check(nccl().send(buf, count, kNcclFloat64, peer, comm_, st), "ncclSend");
}
void NcclComm::recv(double* buf, size_t count, int peer, cudaStream_t st) {
  check(nccl().recv(buf, count, kNcclFloat64, peer, comm_, st), "ncclRecv");
}

}  // namespace kb
