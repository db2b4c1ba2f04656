// Host orchestration of the 3-d hot path: device-resident hierarchy, problem
// data and the FMG / V-cycle / estimator drivers enqueueing the kernels of
// kernels3d.cu on one CUDA stream (captured once as a CUDA graph).  Same
// structure as Solver2D (proj/src/multigrid.cpp:113-321, estimator.cpp:8-45).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "dev3d.hpp"
#include "hier3d.hpp"
#include "solver2d.hpp"

namespace kb {

struct DeviceHierarchy3D {
  Hierarchy3D host;
  std::vector<DevLevel3D> lev;
  DeviceArena arena;
  static std::unique_ptr<DeviceHierarchy3D> create(const Mesh3D& mesh, int max_level);
};

enum Problem3Kind : int { P3_ZERO = 0, P3_SIN = 3, P3_GAUSS = 4, P3_SERIES = 5, P3_HOST = 6 };

struct Problem3D {
  int kind = P3_ZERO;
  std::vector<double> params;  // series coefficients C_abc (64, a fastest)
  std::function<double(double, double, double)> source, boundary;
  static Problem3D builtin(int kind);
  void set_params(const double* p, int count);
};

// f of problem p per copy of macros [s0, s1) of level l at the owner copy's
// node coordinates (like proj/src/fem.cpp:183-186, host libm), into out[(s - s0) * S + idx];
// host threads split the macros (the values do not depend on the split)
void tabulate_source3(const Hierarchy3D& hh, int l, const Problem3D& p, int s0, int s1, double* out);

class Solver3D {
 public:
  Solver3D(std::shared_ptr<DeviceHierarchy3D> h, Problem3D p, SolverConfig2D cfg);
  ~Solver3D();

  const Hierarchy3D& hier() const { return H_->host; }
  cudaStream_t stream() const { return stream_; }
  void set_stream(cudaStream_t st) { stream_ = st ? st : own_stream_; }
  std::size_t load_problem(const Problem3D& p);

  void fmg_enqueue();
  void fmg();
  void sync_and_check();
  void estimate_enqueue(int offset);
  EstimateReport2D estimate_finish(int offset, int kind);
  EstimateReport2D estimate(int offset, int kind) {
    estimate_enqueue(offset);
    return estimate_finish(offset, kind);
  }
  double* state(int which, int level);
  size_t level_size(int level) const;
  int launches_per_fmg() const { return fmg_launches_; }
  int launches_per_estimate() const { return est_launches_; }
  int last_cg_iters() const { return status_host_ ? status_host_->iters : 0; }
  void set_profiling(bool on);
  void kernel_stats(int kind, double* ms, int* launches, double* bytes);

  // single operations
  void apply(int level, int op_mass, const double* x, double* y);
  void residual(int level, const double* u, const double* b, double* r);
  void gauss_seidel(int level, double* u, const double* b, int sweeps);
  void restrict_to(int fine_level, const double* r, double* rc);
  void prolongate(int coarse_level, const double* c, double* f);
  void cg_level0(double* u, const double* b);
  double dot_unique(int level, const double* a, const double* b);
  void interface_sync(int level, double* f, int additive);

 private:
  struct Probe {
    int kind;
    double bytes;
    int ev0, ev1;
  };
  void vcycle(int l, double* u, const double* b);
  void enqueue_fmg_body();
  void mark(int kind, double bytes, int nlaunch = 1);
  void probe_begin(std::vector<Probe>* list);
  cudaEvent_t event_at(int idx);
  double dofs(int l) const { return static_cast<double>(H_->host.levels[l].dofs); }

  std::shared_ptr<DeviceHierarchy3D> H_;
  Problem3D prob_;
  SolverConfig2D cfg_;
  cudaStream_t stream_ = nullptr, own_stream_ = nullptr;
  DeviceArena arena_;
  int L_ = 0;
  bool has_source_ = false;
  std::vector<double*> u_, b_, w_, vu_, vb_, r_, gbnd_, ftab_;
  double *cg_scratch_ = nullptr, *est_sums_ = nullptr, *est_a_ = nullptr, *est_b_ = nullptr, *est_c_ = nullptr;
  double *dot_partial_ = nullptr, *dot_out_ = nullptr;
  DevStatus* status_ = nullptr;
  DevStatus* status_host_ = nullptr;
  double* sums_host_ = nullptr;
  double* stage_ = nullptr;
  double *corners_ = nullptr, *params_ = nullptr;  // device: macro corners, series coefficients (fast-mode f)
  std::size_t stage_count_ = 0;
  cudaGraphExec_t exec_ = nullptr;
  int launches_ = 0, fmg_launches_ = 0, est_launches_ = 0;
  bool profiling_ = false, capturing_ = false;
  std::vector<cudaEvent_t> events_;
  int next_event_ = 0, last_event_ = -1;
  std::vector<Probe>* probes_ = nullptr;
  std::vector<Probe> fmg_probes_, est_probes_;
};

}  // namespace kb
