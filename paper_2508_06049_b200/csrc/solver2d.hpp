// Host orchestration of the 2-d hot path: device-resident hierarchy, problem
// data, and the FMG / V-cycle / estimator drivers that enqueue the sm_100a
// kernels of kernels2d.cu on one CUDA stream (optionally as a CUDA graph).
//
// Mirrors MultigridSolver (proj/include/klref/multigrid.hpp:64-99,
// proj/src/multigrid.cpp:113-321) and error_estimate
// (proj/src/estimator.cpp:8-45).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <functional>
#include <memory>
#include <vector>

#include "dev2d.hpp"
#include "hier2d.hpp"

namespace kb {

// Bump allocator over one cudaMalloc'd arena.
class DeviceArena {
 public:
  DeviceArena() = default;
  DeviceArena(const DeviceArena&) = delete;
  DeviceArena& operator=(const DeviceArena&) = delete;
  ~DeviceArena();
  void reserve(size_t bytes);
  void* take(size_t bytes);
  template <typename T>
  T* upload(const std::vector<T>& v) {
    if (v.empty()) return nullptr;
    T* p = static_cast<T*>(take(v.size() * sizeof(T)));
    KB_CUDA_CHECK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }
  size_t used() const { return used_; }

 private:
  char* base_ = nullptr;
  size_t cap_ = 0, used_ = 0;
  bool pooled_ = false;  // from the stream-ordered pool (cudaMallocAsync)
};

struct DeviceHierarchy2D {
  Hierarchy2D host;
  std::vector<DevLevel2D> lev;
  DevHier2D dh{};
  int* gs_done = nullptr;
  DeviceArena arena;
  static std::unique_ptr<DeviceHierarchy2D> create(const Mesh2D& mesh, int max_level);
};

enum ProblemKind : int { PROB_ZERO = 0, PROB_SIN2D = 1, PROB_LSHAPE = 2, PROB_HOST = 3 };

struct Problem2D {
  int kind = PROB_ZERO;
  std::function<double(double, double)> source;    // host (glibc) evaluation
  std::function<double(double, double)> boundary;
  std::function<double(double, double)> exact;
  bool has_exact = false;
  static Problem2D builtin(int kind);
};

struct SolverConfig2D {
  int nu = 2, pre_smooth = 2, post_smooth = 2;
  double coarse_rel_tol = 1e-9, coarse_abs_floor = 1e-12;
  int coarse_max_iter = 100000;
  int finest_policy = 0;  // 0 = None, 1 = ValidationTwoDigits (proj/include/klref/multigrid.hpp:12-17)
  int max_extra_cycles = 60;
  int faithful_source = 0;  // 1: host-tabulated f (bitwise-faithful RHS)
  int use_graph = 1;
};

struct EstimateReport2D {
  int offset = 1, base_level = 0, kind = 0;
  double norm_coarser = 0.0, norm_base = 0.0, conv_factor = 0.0, eta = 0.0;
  std::vector<double> eta_local;
};

class Solver2D {
 public:
  Solver2D(std::shared_ptr<DeviceHierarchy2D> h, Problem2D p, SolverConfig2D cfg);
  ~Solver2D();

  const Hierarchy2D& hier() const { return H_->host; }
  cudaStream_t stream() const { return stream_; }
  // launch on a caller-owned stream from now on (nullptr: back to the solver's own)
  void set_stream(cudaStream_t st);
  // (re)tabulate the problem's f and g on the host and copy them to the device
  // through pinned staging buffers; returns the bytes copied host->device
  std::size_t load_problem(const Problem2D& p);

  // Per-kernel CUDA-event probes (roofline evidence): when enabled, every
  // kernel of the FMG graph / estimator is bracketed by event records, and
  // kernel_stats() sums the device time and algorithmic bytes per kernel kind
  // over the most recent FMG + estimate.
  void set_profiling(bool on);
  void kernel_stats(int kind, double* ms, int* launches, double* bytes);

  // FMG (proj/src/multigrid.cpp:248-321) into the solver-owned FmgState.
  void fmg_enqueue();
  void fmg();
  void sync_and_check();
  EstimateReport2D estimate(int offset, int kind);
  void estimate_enqueue(int offset);
  EstimateReport2D estimate_finish(int offset, int kind);

  // state access: which 0 = u, 1 = b, 2 = w (w[l] lives on level l+1)
  double* state(int which, int level);
  size_t level_size(int level) const;

  // single operations on device arrays (API parity with the reference)
  void apply(int level, int op_mass, const double* x, double* y);
  void residual(int level, const double* u, const double* b, double* r);
  void gauss_seidel(int level, double* u, const double* b, int sweeps);
  void restrict_to(int fine_level, const double* r, double* rc);
  void prolongate(int coarse_level, const double* c, double* f);
  void cg_level0(double* u, const double* b);
  double dot_unique(int level, const double* a, const double* b);
  void interface_sync(int level, double* f, int additive);
  // ExactErrorEvaluator at the finest level (proj/src/fem.cpp:358-476):
  // global / per-macro ||u - u_L||; three-term moment form, pointwise fallback
  struct ExactNorms {
    double global = 0.0;
    std::vector<double> per_macro;
  };
  // of the solver's u_L, or of any level-L device function u
  ExactNorms exact_error(const double* u = nullptr);
  // MultigridSolver::solve_direct(l), proj/src/multigrid.cpp:323-357: b = level_rhs(l),
  // u = g on the boundary; level 0 by cg_level0, l > 0 by the unpreconditioned CG
  // of the reference (tolerance relative to the initial residual, no throw)
  void solve_direct(int level, double* u);
  int extra_cycles() const { return extra_cycles_; }
  int launches_per_fmg() const { return fmg_launches_; }
  int launches_per_estimate() const { return est_launches_; }
  int last_cg_iters() const;

 private:
  void vcycle(int l, double* u, const double* b);
  void enqueue_fmg_body();
  struct Probe {
    int kind;
    double bytes;
    int ev0, ev1;
  };
  // after a kernel launch: count it and, when profiling, close its probe
  void mark(int kind, double bytes, int nlaunch = 1);
  void probe_begin(std::vector<Probe>* list);
  cudaEvent_t event_at(int idx);
  void tabulate(const Problem2D& p);
  double l2_norm_mass(int level, const double* f, double* tmp);
  double dot_seq(int level, const double* a, const double* b);  // sqrt(max(0, dot_unique(f, M f)))
  void finest_residual_vs_estimate();
  double* scratch(int slot, int level);  // level-sized device scratch vectors (slot 0..3)
  void exact_setup();
  ExactNorms exact_pointwise(const double* u = nullptr);
  double dofs(int l) const { return static_cast<double>(H_->host.levels[l].dofs); }

  std::shared_ptr<DeviceHierarchy2D> H_;
  Problem2D prob_;
  SolverConfig2D cfg_;
  cudaStream_t stream_ = nullptr;
  DeviceArena arena_;
  int L_ = 0;
  std::vector<double*> u_, b_, w_, vu_, vb_, r_, gbnd_, ftab_;
  double* cg_scratch_ = nullptr;
  double* est_sums_ = nullptr;
  double* est_tmp_a_ = nullptr;
  double* est_tmp_b_ = nullptr;
  double* dot_partial_ = nullptr;
  double* dot_out_ = nullptr;
  DevStatus* status_ = nullptr;
  int* gs_done_ = nullptr;
  DevStatus* status_host_ = nullptr;
  double* sums_host_ = nullptr;
  int src_kind_ = SRC_ZERO;
  cudaGraphExec_t exec_ = nullptr;
  int launches_ = 0, fmg_launches_ = 0, est_launches_ = 0;
  cudaStream_t own_stream_ = nullptr;
  // pinned staging of the problem tables (Dirichlet g per level, f table per level)
  double* stage_ = nullptr;
  bool stage_pinned_ = true;
  std::size_t stage_count_ = 0;
  std::vector<std::size_t> gbnd_count_, ftab_count_;
  // profiling probes
  bool profiling_ = false;
  bool capturing_ = false;
  std::vector<cudaEvent_t> events_;
  int next_event_ = 0, last_event_ = -1;
  std::vector<Probe>* probes_ = nullptr;
  std::vector<Probe> fmg_probes_, est_probes_;
  // exact-error evaluator state (built on first use; host moments per copy)
  std::unique_ptr<DeviceArena> ex_arena_;
  double* ex_moments_ = nullptr;
  double* ex_out_ = nullptr;
  std::vector<double> ex_usq_;
  std::unique_ptr<DeviceArena> scr_arena_;
  std::vector<double*> scr_;
  int scr_level_ = -1;
  int extra_cycles_ = 0;
};

}  // namespace kb
