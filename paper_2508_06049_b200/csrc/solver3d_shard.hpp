// Macro-sharded 3-d FMG + estimator: the operation sequence
// of Solver3D (proj/src/multigrid.cpp:231-321, estimator.cpp:8-45 structure)
// over macro shards, bit-identical to the one-device solver.
//
// Each shard holds the lattices of its slot range on the sharded levels and
// everything on the replicated coarse levels (<= rep_level).  Every group
// operation is preceded by one exchange of the member contributions of the
// groups that span shards (shard3d.hpp); every shard then sums all members in
// ascending slot order, as the one-device kernels do.  The crossing from a
// sharded to a replicated level is one all-gather of the restricted residual
// blocks; the estimator's per-macro sums are all-gathered the same way and
// reduced on the host in slot order.
//
// Two transports move the same buffers:
//   * in-process: several shards on one device, one stream, device copies
//     (the parity harness: bitwise equal to Solver3D on one GPU);
//   * NCCL: one shard per process/GPU, grouped ncclSend/ncclRecv per peer.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "comm.hpp"
#include "shard3d.hpp"
#include "solver3d.hpp"

namespace kb {

struct Shard3D {
  ShardPlan3D plan;
  std::vector<DevLevel3D> lev;
  DeviceArena tables, data;
  std::vector<const int*> pack_pos, pack_slot, pack_ijk;
  std::vector<double*> u, b, w, vu, vb, r, gbnd, ftab;
  double *sendbuf = nullptr, *ghost = nullptr, *cg_scratch = nullptr, *est_all = nullptr, *est_a = nullptr,
         *est_b = nullptr, *est_c = nullptr;
  DevStatus* status = nullptr;
  DevStatus* status_host = nullptr;
};

class ShardedSolver3D {
 public:
  // comm == nullptr: `nshards` shards in this process on the current device;
  // otherwise one shard, rank comm->rank() of comm->size()
  ShardedSolver3D(std::shared_ptr<DeviceHierarchy3D> h, Problem3D p, SolverConfig2D cfg, int nshards, int rep_level,
                  std::shared_ptr<NcclComm> comm);
  ~ShardedSolver3D();

  cudaStream_t stream() const { return stream_; }
  int shards_total() const { return P_; }
  int rep_level() const { return rep_; }
  void fmg_enqueue();
  void fmg();
  void sync_and_check();
  void estimate_enqueue(int offset);
  EstimateReport2D estimate_finish(int offset, int kind);
  // the full level array (M * S) gathered from the local shards; with NCCL
  // only this rank's block (and replicated levels) are written
  void state_read(int which, int level, double* host_out);
  int launches_per_fmg() const { return fmg_launches_; }
  int launches_per_estimate() const { return est_launches_; }
  // bytes one FMG exchanges between shards (all shards, both directions counted once)
  double exchange_bytes_per_fmg() const { return xbytes_fmg_; }

 private:
  bool sharded(int l) const { return P_ > 1 && l > rep_; }
  int off(const Shard3D& sh, int l) const { return sharded(l) ? sh.plan.s0 : 0; }
  int mloc(const Shard3D& sh, int l) const { return sharded(l) ? sh.plan.count : M_; }
  size_t lsize(const Shard3D& sh, int l) const;
  void exchange(int l, int c0, int c1);
  void allgather(const std::vector<double*>& arrays, size_t per_macro);
  void pack(int l, int mode, const std::vector<double*>& x, int c0, int c1);
  void rhs(int l);
  void set_boundary(int l, int which, int zero_rest);
  void vcycle(int l, bool top);
  void prolong(int lc, const std::vector<const double*>& c, const std::vector<double*>& f, int mode);
  void enqueue_fmg_body();
  void load_problem();

  std::shared_ptr<DeviceHierarchy3D> H_;
  Problem3D prob_;
  SolverConfig2D cfg_;
  std::shared_ptr<NcclComm> comm_;
  int P_ = 1, rep_ = 0, L_ = 0, M_ = 0;
  std::vector<std::unique_ptr<Shard3D>> sh_;
  cudaStream_t stream_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
  double* sums_host_ = nullptr;
  int launches_ = 0, fmg_launches_ = 0, est_launches_ = 0;
  double xbytes_ = 0.0, xbytes_fmg_ = 0.0;
  bool has_source_ = false;
};

}  // namespace kb
