// NCCL communicator of the sharded 3-d solver (one process per GPU).  NCCL is
// bound at run time (dlopen of libnccl.so.2 -- in a torch process the library
// torch.distributed already loaded), so the library itself has no link-time
// NCCL dependency and loads on hosts without it.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace kb {

class NcclComm {
 public:
  static void unique_id(unsigned char out[128]);
  NcclComm(int nranks, int rank, const unsigned char id[128]);
  ~NcclComm();
  NcclComm(const NcclComm&) = delete;
  NcclComm& operator=(const NcclComm&) = delete;
  int rank() const { return rank_; }
  int size() const { return nranks_; }
  void group_start();
  void group_end();
  void send(const double* buf, size_t count, int peer, cudaStream_t st);
  void recv(double* buf, size_t count, int peer, cudaStream_t st);

 private:
  void* comm_ = nullptr;
  int nranks_ = 1, rank_ = 0;
};

}  // namespace kb
