// klref_b200/klref.hpp -- C++ drop-in facade of the reference hot-path API
// (proj/include/klref/{hhg,fem,multigrid,estimator}.hpp) over the C-ABI of
// libklref_b200.so (include/klref_b200.h).  Header-only; link with -lklref_b200.
//
// Source compatibility with the reference's callers (proj/src/amr.cpp) is the
// goal: the same namespace, class and function names, argument meaning and
// exception types.  Put include/klref_b200/dropin first on the include path
// and the reference's own headers after it: "klref/{hhg,fem,multigrid,
// estimator}.hpp" then resolve to this facade, while the reference's
// macro_mesh.hpp / errors.hpp / amr.hpp / mesh_io.hpp / problems.hpp stay the
// reference's (the exception classes and Point / Index are the reference's
// own when its headers are visible; identical definitions otherwise).
// Differences, all forced by the device design:
//   * GridHierarchy::build is a template over the mesh type: any type with the
//     accessors of the reference MacroMesh that the hot path reads -- dim(),
//     num_vertices(), vertex(id).coords, active(), element(id).v
//     (proj/include/klref/macro_mesh.hpp:64-79) -- so the reference's own
//     MacroMesh is accepted unchanged;
//   * grid functions live on the device; GridFunction::macro(slot) hands out a
//     host mirror that is downloaded on first access and uploaded again
//     before the next device operation (proj/include/klref/hhg.hpp:41-42);
//   * FmgState's u / b / w are views of the solver's device state, copied to
//     the host on access (the reference copies them by value); running fmg()
//     again on the same solver updates them;
//   * ExactErrorEvaluator evaluates functions of its hierarchy's finest level
//     (the reference's callers only use that level).
#ifndef KLREF_B200_KLREF_HPP
#define KLREF_B200_KLREF_HPP

#include <array>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../klref_b200.h"

namespace klref {

// ---------------------------------------------------------------- errors
// proj/include/klref/errors.hpp:10-53; Point / Index, proj/include/klref/macro_mesh.hpp:16-19
}  // namespace klref
#if __has_include("klref/macro_mesh.hpp")
#include "klref/macro_mesh.hpp"  // the reference's errors.hpp, Index, Point
namespace klref {
#else
#include <stdexcept>
namespace klref {
using Index = std::int32_t;
inline constexpr Index kNoIndex = -1;
using Point = std::array<double, 3>;
class StructuralError : public std::runtime_error {
 public:
  explicit StructuralError(const std::string& what) : std::runtime_error(what) {}
};
class DomainError : public std::domain_error {
 public:
  explicit DomainError(const std::string& what) : std::domain_error(what) {}
};
class SolverError : public std::runtime_error {
 public:
  SolverError(const std::string& what, double last_residual) : std::runtime_error(what), last_(last_residual) {}
  double last_residual() const { return last_; }

 private:
  double last_ = 0.0;
};
class IoError : public std::runtime_error {
 public:
  explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
class InternalError : public std::logic_error {
 public:
  explicit InternalError(const std::string& what) : std::logic_error(what) {}
};
class ResourceError : public std::runtime_error {
 public:
  ResourceError(const std::string& what, int level) : std::runtime_error(what), level_(level) {}
  int level() const { return level_; }

 private:
  int level_ = -1;
};
#endif
// CUDA failure or no device (no reference counterpart)
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(int rc) {
  if (rc == KLREF_OK) return;
  const std::string msg = klref_last_error();
  switch (rc) {
    case KLREF_ERR_STRUCTURAL: throw StructuralError(msg);
    case KLREF_ERR_DOMAIN: throw DomainError(msg);
    case KLREF_ERR_SOLVER: throw SolverError(msg, klref_last_error_residual());
    case KLREF_ERR_IO: throw IoError(msg);
    case KLREF_ERR_RESOURCE: throw ResourceError(msg, klref_last_error_level());
    case KLREF_ERR_CUDA: throw DeviceError(msg);
    default: throw InternalError(msg);
  }
}
template <typename H, void (*Destroy)(H)>
struct Handle {
  H h = nullptr;
  Handle() = default;
  explicit Handle(H x) : h(x) {}
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() {
    if (h) Destroy(h);
  }
};
}  // namespace detail

// ---------------------------------------------------------------- hhg.hpp
inline int lattice_index(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }
inline int lattice_size(int n) { return (n + 1) * (n + 2) / 2; }

enum class SyncMode { ReplaceFromOwner, Additive };
enum class OperatorKind { Stiffness, Mass };
enum class FinestPolicy { None, ValidationTwoDigits, ResidualVsEstimate };
enum class EstimatorKind { Unscaled, Scaled };

class GridHierarchy;
class GridFunction;
using HierarchyPtr = std::shared_ptr<const GridHierarchy>;

class GridHierarchy : public std::enable_shared_from_this<GridHierarchy> {
 public:
  // GridHierarchy::build, proj/src/hhg.cpp:48-144 (+ upload to the device)
  template <typename Mesh>
  static HierarchyPtr build(const Mesh& macro, int max_level) {
    const int dim = macro.dim();
    std::vector<double> coords;
    for (std::size_t v = 0; v < macro.num_vertices(); ++v) {
      const auto& p = macro.vertex(static_cast<std::int32_t>(v)).coords;
      for (int d = 0; d < dim; ++d) coords.push_back(p[d]);
    }
    std::vector<int> corners;
    for (auto id : macro.active())
      for (int c = 0; c <= dim; ++c) corners.push_back(static_cast<int>(macro.element(id).v[c]));
    klref_mesh m = nullptr;
    detail::check(klref_mesh_create(dim, static_cast<int>(macro.num_vertices()), coords.data(),
                                    static_cast<int>(macro.active().size()), corners.data(), &m));
    detail::Handle<klref_mesh, klref_mesh_destroy> mesh(m);
    klref_hierarchy h = nullptr;
    detail::check(klref_hierarchy_build(m, max_level, &h));
    std::shared_ptr<GridHierarchy> out(new GridHierarchy(h));
    return out;
  }

  int max_level() const { return query_int(klref_hierarchy_max_level); }
  int num_macros() const { return query_int(klref_hierarchy_num_macros); }
  std::int64_t dof_count(int l) const {
    int64_t v = 0;
    detail::check(klref_hierarchy_dof_count(h_->h, l, &v));
    return v;
  }
  std::int64_t fine_element_count(int l) const {
    int64_t v = 0;
    detail::check(klref_hierarchy_fine_element_count(h_->h, l, &v));
    return v;
  }
  int lattice_size_at(int l) const {
    int v = 0;
    detail::check(klref_hierarchy_lattice_size(h_->h, l, &v));
    return v;
  }
  inline GridFunction create_function(int l) const;

  klref_hierarchy handle() const { return h_->h; }
  // solver context for the single operations of the free functions below
  klref_solver ops() const {
    if (!ops_) {
      klref_problem p = nullptr;
      detail::check(klref_problem_create(KLREF_PROBLEM_ZERO, &p));
      detail::Handle<klref_problem, klref_problem_destroy> hp(p);
      klref_solver_config cfg;
      klref_solver_config_default(&cfg);
      klref_solver s = nullptr;
      detail::check(klref_solver_create(h_->h, p, &cfg, &s));
      ops_ = std::make_shared<detail::Handle<klref_solver, klref_solver_destroy>>(s);
    }
    return ops_->h;
  }

 private:
  explicit GridHierarchy(klref_hierarchy h)
      : h_(std::make_shared<detail::Handle<klref_hierarchy, klref_hierarchy_destroy>>(h)) {}
  int query_int(int (*fn)(klref_hierarchy, int*)) const {
    int v = 0;
    detail::check(fn(h_->h, &v));
    return v;
  }
  std::shared_ptr<detail::Handle<klref_hierarchy, klref_hierarchy_destroy>> h_;
  mutable std::shared_ptr<detail::Handle<klref_solver, klref_solver_destroy>> ops_;
};

// GridFunction (proj/include/klref/hhg.hpp:33-53): device data + lazy host mirror.
class GridFunction {
 public:
  GridFunction() = default;
  GridFunction(HierarchyPtr h, int level) : h_(std::move(h)), level_(level) {
    klref_gf g = nullptr;
    detail::check(klref_gf_create(h_->handle(), level_, &g));
    d_ = std::make_shared<detail::Handle<klref_gf, klref_gf_destroy>>(g);
    S_ = h_->lattice_size_at(level_);
  }
  GridFunction(const GridFunction& o) : GridFunction(o.h_, o.level_) { assign(o); }
  GridFunction& operator=(const GridFunction& o) {
    if (this != &o) {
      if (!d_ || o.h_ != h_ || o.level_ != level_) *this = GridFunction(o.h_, o.level_);
      assign(o);
    }
    return *this;
  }
  GridFunction(GridFunction&&) = default;
  GridFunction& operator=(GridFunction&&) = default;

  int level() const { return level_; }
  const HierarchyPtr& hierarchy() const { return h_; }
  std::size_t num_macros() const { return h_ ? static_cast<std::size_t>(h_->num_macros()) : 0; }
  std::vector<double>& macro(int slot) {
    pull();
    host_dirty_ = true;
    return host_[static_cast<std::size_t>(slot)];
  }
  const std::vector<double>& macro(int slot) const {
    pull();
    return host_[static_cast<std::size_t>(slot)];
  }
  // BLAS-1 of the reference (proj/src/hhg.cpp:27-46) on the host mirror
  void fill(double value) {
    for (int s = 0; s < static_cast<int>(num_macros()); ++s)
      for (auto& v : macro(s)) v = value;
  }
  void scale(double alpha) {
    for (int s = 0; s < static_cast<int>(num_macros()); ++s)
      for (auto& v : macro(s)) v *= alpha;
  }
  void add_scaled(const GridFunction& x, double alpha) {
    for (int s = 0; s < static_cast<int>(num_macros()); ++s) {
      auto& y = macro(s);
      const auto& xs = x.macro(s);
      for (std::size_t k = 0; k < y.size(); ++k) y[k] += alpha * xs[k];
    }
  }
  // the device handle, after pushing host-side edits
  klref_gf device() const {
    push();
    return d_->h;
  }
  // the device copy changed (a kernel wrote it): drop the host mirror
  void device_written() { host_valid_ = host_dirty_ = false; }
  // flat host copy in the reference layout (macro-major)
  std::vector<double> flat() const {
    pull();
    std::vector<double> out;
    for (const auto& m : host_) out.insert(out.end(), m.begin(), m.end());
    return out;
  }
  void assign_flat(const std::vector<double>& v) {
    detail::check(klref_gf_upload(d_->h, v.data()));
    device_written();
  }

 private:
  void assign(const GridFunction& o) { assign_flat(o.flat()); }
  void pull() const {
    if (host_valid_) return;
    std::vector<double> flat(static_cast<std::size_t>(num_macros()) * S_);
    detail::check(klref_gf_download(d_->h, flat.data()));
    host_.assign(num_macros(), {});
    for (std::size_t s = 0; s < num_macros(); ++s)
      host_[s].assign(flat.begin() + s * S_, flat.begin() + (s + 1) * S_);
    host_valid_ = true;
  }
  void push() const {
    if (!host_dirty_) return;
    std::vector<double> flat;
    for (const auto& m : host_) flat.insert(flat.end(), m.begin(), m.end());
    detail::check(klref_gf_upload(d_->h, flat.data()));
    host_dirty_ = false;
  }
  HierarchyPtr h_;
  int level_ = -1;
  std::size_t S_ = 0;
  std::shared_ptr<detail::Handle<klref_gf, klref_gf_destroy>> d_;
  mutable std::vector<std::vector<double>> host_;
  mutable bool host_valid_ = false, host_dirty_ = false;
};

inline GridFunction GridHierarchy::create_function(int l) const { return GridFunction(shared_from_this(), l); }

// interface_sync / dot_unique, proj/src/hhg.cpp:206-257
inline void interface_sync(GridFunction& f, SyncMode mode) {
  detail::check(klref_interface_sync(f.hierarchy()->ops(), f.device(),
                                     mode == SyncMode::Additive ? KLREF_SYNC_ADDITIVE : KLREF_SYNC_REPLACE));
  f.device_written();
}
inline double dot_unique(const GridFunction& a, const GridFunction& b) {
  double v = 0.0;
  detail::check(klref_dot_unique(a.hierarchy()->ops(), a.device(), b.device(), &v));
  return v;
}

// ---------------------------------------------------------------- fem.hpp
class OperatorP1 {
 public:
  OperatorP1(HierarchyPtr h, OperatorKind kind, int level) : h_(std::move(h)), kind_(kind), level_(level) {}
  OperatorKind kind() const { return kind_; }
  int level() const { return level_; }
  const HierarchyPtr& hierarchy() const { return h_; }
  // OperatorP1::apply, proj/src/fem.cpp:95-126 (x interface-consistent)
  void apply(const GridFunction& x, GridFunction& y) const {
    if (x.level() != level_ || y.level() != level_) throw StructuralError("operator level mismatch");
    detail::check(klref_apply(h_->ops(), kind_ == OperatorKind::Mass ? KLREF_MASS : KLREF_STIFFNESS, x.device(),
                              y.device()));
    y.device_written();
  }

 private:
  HierarchyPtr h_;
  OperatorKind kind_;
  int level_;
};

// ProblemSpec, proj/include/klref/fem.hpp:55-64 (host callbacks; f and g are
// tabulated on the host -- glibc -- when a solver is created)
struct ProblemSpec {
  std::string name;
  std::function<double(double, double)> exact;
  std::function<double(double, double)> source;
  std::function<double(double, double)> boundary;
  bool has_exact = true;
  bool has_corner = false;
  Point corner{0.0, 0.0, 0.0};
  double domain_volume = 1.0;
};

// ---------------------------------------------------------------- multigrid.hpp: config
struct SolverConfig {
  int nu = 2;
  int pre_smooth = 2;
  int post_smooth = 2;
  double coarse_rel_tol = 1e-9;
  double coarse_abs_floor = 1e-12;
  int coarse_max_iter = 100000;
  FinestPolicy finest_policy = FinestPolicy::ValidationTwoDigits;  // the reference default
  int max_extra_cycles = 60;
  bool record_residuals = false;
};

// ---------------------------------------------------------------- fem.hpp: exact error
struct ErrorNorms {
  double global = 0.0;
  std::vector<double> per_macro;
};

namespace detail {
struct HostProblem {
  std::function<double(double, double)> source, boundary, exact;
};
inline double src_cb(double x, double y, void* p) { return static_cast<HostProblem*>(p)->source(x, y); }
inline double bnd_cb(double x, double y, void* p) { return static_cast<HostProblem*>(p)->boundary(x, y); }
inline double exact_cb(double x, double y, void* p) { return static_cast<HostProblem*>(p)->exact(x, y); }
using SolverHandle = std::shared_ptr<Handle<klref_solver, klref_solver_destroy>>;
// a device solver for the host problem p; the callbacks' owner (hp) must
// outlive it, so it is shared with whoever keeps the solver
inline SolverHandle make_solver(klref_hierarchy h, const ProblemSpec& p, const klref_solver_config& c,
                                std::shared_ptr<HostProblem>& hp) {
  hp = std::make_shared<HostProblem>(HostProblem{p.source, p.boundary, p.exact});
  klref_problem prob = nullptr;
  check(klref_problem_create_host(src_cb, bnd_cb, hp.get(), &prob));
  Handle<klref_problem, klref_problem_destroy> hprob(prob);
  if (p.has_exact && p.exact) check(klref_problem_set_exact(prob, exact_cb, hp.get()));
  klref_solver s = nullptr;
  check(klref_solver_create(h, prob, &c, &s));
  return std::make_shared<Handle<klref_solver, klref_solver_destroy>>(s);
}
}  // namespace detail

// ExactErrorEvaluator (proj/include/klref/fem.hpp:101-114, proj/src/fem.cpp:358-476):
// ||u - u_h|| by the 6-point rule in the reference's three-term moment form
// (pointwise fallback on cancellation); moments tabulated on the host, the
// per-macro sums on the device.  `level` must be the hierarchy's finest level.
class ExactErrorEvaluator {
 public:
  ExactErrorEvaluator(HierarchyPtr h, const ProblemSpec& p, int level) : h_(std::move(h)), level_(level) {
    if (level_ != h_->max_level())
      throw StructuralError("ExactErrorEvaluator: the device evaluator works on the hierarchy's finest level");
    if (!p.has_exact || !p.exact) throw StructuralError("the problem has no closed-form solution");
    klref_solver_config c;
    klref_solver_config_default(&c);
    c.finest_policy = 0;
    c.faithful_source = 1;
    s_ = detail::make_solver(h_->handle(), p, c, hp_);
  }
  ErrorNorms evaluate(const GridFunction& u_h) const {
    if (u_h.level() != level_) throw StructuralError("ExactErrorEvaluator: level mismatch");
    ErrorNorms out;
    out.per_macro.assign(static_cast<std::size_t>(h_->num_macros()), 0.0);
    detail::check(klref_solver_exact_error_of(s_->h, u_h.device(), &out.global, out.per_macro.data()));
    return out;
  }

 private:
  friend class MultigridSolver;
  ExactErrorEvaluator(HierarchyPtr h, int level, detail::SolverHandle s, std::shared_ptr<detail::HostProblem> hp)
      : h_(std::move(h)), level_(level), s_(std::move(s)), hp_(std::move(hp)) {}
  HierarchyPtr h_;
  int level_;
  detail::SolverHandle s_;
  std::shared_ptr<detail::HostProblem> hp_;
};

// exact_error_norm(p, u_h), proj/include/klref/fem.hpp:116
inline ErrorNorms exact_error_norm(const ProblemSpec& p, const GridFunction& u_h) {
  return ExactErrorEvaluator(u_h.hierarchy(), p, u_h.level()).evaluate(u_h);
}

// ---------------------------------------------------------------- multigrid.hpp
class MultigridSolver;

// FmgState (proj/include/klref/multigrid.hpp:43-53): views of the solver's
// device state; u[l], b[l] on level l, w[l] = P u[l] on level l + 1.
class FmgState {
 public:
  class Levels {
   public:
    Levels(detail::SolverHandle s, HierarchyPtr h, int which, int count, int shift)
        : s_(std::move(s)), h_(std::move(h)), which_(which), count_(count), shift_(shift) {}
    std::size_t size() const { return static_cast<std::size_t>(count_); }
    GridFunction operator[](std::size_t l) const {
      const int level = static_cast<int>(l) + shift_;
      GridFunction f(h_, level);
      std::vector<double> flat(static_cast<std::size_t>(h_->num_macros()) * h_->lattice_size_at(level));
      detail::check(klref_solver_state_read(s_->h, which_, level, flat.data()));
      f.assign_flat(flat);
      return f;
    }
    GridFunction back() const { return (*this)[size() - 1]; }

   private:
    detail::SolverHandle s_;
    HierarchyPtr h_;
    int which_, count_, shift_;
  };

  HierarchyPtr h;
  SolverConfig config;
  Levels u, b, w;
  int extra_cycles = 0;
  std::shared_ptr<const ExactErrorEvaluator> error_eval;  // set in validation mode (problem with exact)

 private:
  friend class MultigridSolver;
  friend struct EstimateAccess;
  FmgState(detail::SolverHandle s, HierarchyPtr hh, SolverConfig cfg)
      : h(hh),
        config(cfg),
        u(s, hh, KLREF_STATE_U, hh->max_level() + 1, 0),
        b(s, hh, KLREF_STATE_B, hh->max_level() + 1, 0),
        w(s, hh, KLREF_STATE_W, hh->max_level(), 1),
        solver_(std::move(s)) {}
  detail::SolverHandle solver_;
};

class MultigridSolver {
 public:
  // MultigridSolver(h, p, cfg), proj/src/multigrid.cpp:113-119.  Like the
  // reference, p is not owned; f and g are tabulated here.
  MultigridSolver(HierarchyPtr h, const ProblemSpec& p, SolverConfig cfg) : h_(std::move(h)), p_(&p), cfg_(cfg) {
    klref_solver_config c;
    klref_solver_config_default(&c);
    c.nu = cfg.nu;
    c.pre_smooth = cfg.pre_smooth;
    c.post_smooth = cfg.post_smooth;
    c.coarse_rel_tol = cfg.coarse_rel_tol;
    c.coarse_abs_floor = cfg.coarse_abs_floor;
    c.coarse_max_iter = cfg.coarse_max_iter;
    c.finest_policy = cfg.finest_policy == FinestPolicy::ValidationTwoDigits  ? 1
                      : cfg.finest_policy == FinestPolicy::ResidualVsEstimate ? 2
                                                                              : 0;
    c.max_extra_cycles = cfg.max_extra_cycles;
    c.faithful_source = 1;
    s_ = detail::make_solver(h_->handle(), p, c, hp_);
  }
  const HierarchyPtr& hierarchy() const { return h_; }
  const ProblemSpec& problem() const { return *p_; }
  const SolverConfig& config() const { return cfg_; }

  // MultigridSolver::fmg, proj/src/multigrid.cpp:248-321 (finest-level policy included)
  FmgState fmg() {
    detail::check(klref_solver_fmg(s_->h));
    FmgState st(s_, h_, cfg_);
    detail::check(klref_solver_extra_cycles(s_->h, &st.extra_cycles));
    if (cfg_.finest_policy == FinestPolicy::ValidationTwoDigits && p_->has_exact && p_->exact)
      st.error_eval = std::shared_ptr<const ExactErrorEvaluator>(
          new ExactErrorEvaluator(h_, h_->max_level(), s_, hp_));
    return st;
  }
  // MultigridSolver::solve_direct(l), proj/src/multigrid.cpp:323-357
  GridFunction solve_direct(int l) {
    GridFunction u(h_, l);
    detail::check(klref_solver_solve_direct(s_->h, l, u.device()));
    u.device_written();
    return u;
  }
  // single operations, proj/src/multigrid.cpp:127-229
  void gauss_seidel(int l, GridFunction& u, const GridFunction& b, int sweeps) {
    if (u.level() != l || b.level() != l) throw StructuralError("grid function level mismatch");
    detail::check(klref_gauss_seidel(s_->h, u.device(), b.device(), sweeps));
    u.device_written();
  }
  void residual(int l, const GridFunction& u, const GridFunction& b, GridFunction& r) const {
    if (u.level() != l || b.level() != l || r.level() != l) throw StructuralError("grid function level mismatch");
    detail::check(klref_residual(s_->h, u.device(), b.device(), r.device()));
    r.device_written();
  }
  void cg_level0(GridFunction& u, const GridFunction& b) {
    detail::check(klref_cg_level0(s_->h, u.device(), b.device()));
    u.device_written();
  }
  klref_solver handle() const { return s_->h; }

 private:
  HierarchyPtr h_;
  const ProblemSpec* p_;
  SolverConfig cfg_;
  std::shared_ptr<detail::HostProblem> hp_;
  detail::SolverHandle s_;
  friend struct EstimateAccess;
};

// prolongate / restrict_transpose / prolongate_to, proj/src/multigrid.cpp:22-111
inline GridFunction prolongate(const GridFunction& coarse) {
  GridFunction fine(coarse.hierarchy(), coarse.level() + 1);
  detail::check(klref_prolongate(coarse.hierarchy()->ops(), coarse.device(), fine.device()));
  fine.device_written();
  return fine;
}
inline GridFunction restrict_transpose(const GridFunction& fine) {
  GridFunction coarse(fine.hierarchy(), fine.level() - 1);
  detail::check(klref_restrict_transpose(fine.hierarchy()->ops(), fine.device(), coarse.device()));
  coarse.device_written();
  return coarse;
}
inline GridFunction prolongate_to(const GridFunction& coarse, int target_level) {
  GridFunction f = coarse;
  while (f.level() < target_level) f = prolongate(f);
  return f;
}

// ---------------------------------------------------------------- estimator.hpp
struct EstimateReport {
  int offset = 1;
  int base_level = 0;
  EstimatorKind kind = EstimatorKind::Unscaled;
  double norm_coarser = 0.0;
  double norm_base = 0.0;
  double conv_factor = 0.0;
  double eta = 0.0;
  std::vector<double> eta_local;
};

struct EstimateAccess {
  static klref_solver solver(const FmgState& s) { return s.solver_->h; }
};

// error_estimate(state, j, kind), proj/src/estimator.cpp:8-45 (on the device state)
inline EstimateReport error_estimate(const FmgState& state, int offset, EstimatorKind kind) {
  klref_estimate_report r{};
  EstimateReport out;
  out.eta_local.assign(static_cast<std::size_t>(state.h->num_macros()), 0.0);
  detail::check(klref_error_estimate(EstimateAccess::solver(state), offset,
                                     kind == EstimatorKind::Scaled ? KLREF_SCALED : KLREF_UNSCALED, &r,
                                     out.eta_local.data()));
  out.offset = r.offset;
  out.base_level = r.base_level;
  out.kind = kind;
  out.norm_coarser = r.norm_coarser;
  out.norm_base = r.norm_base;
  out.conv_factor = r.conv_factor;
  out.eta = r.eta;
  return out;
}

// ---------------------------------------------------------------- estimator.hpp: effectivity
// proj/include/klref/estimator.hpp:27-68 (host formulas, C-ABI klref_effectivity_*)
struct EquivalenceConstants {
  double lower = 0.0;  // C1
  double upper = 0.0;  // C2
};
inline EquivalenceConstants effectivity_constants(double theta, double eps, int offset) {
  EquivalenceConstants c;
  detail::check(klref_effectivity_constants(theta, eps, offset, &c.lower, &c.upper));
  return c;
}
inline double local_spread_bound_scaled(double theta_max, double eps, int offset) {
  double v = 0.0;
  detail::check(klref_local_spread_bound_scaled(theta_max, eps, offset, &v));
  return v;
}
inline double local_spread_bound_unscaled(double theta_min, double theta_max, int offset) {
  double v = 0.0;
  detail::check(klref_local_spread_bound_unscaled(theta_min, theta_max, offset, &v));
  return v;
}
struct BoundsConstants {
  double theta = 0.25;
  double eps = 0.0;
  int offset = 1;
  int order = 2;
  double theta_eps = 0.25;
  EquivalenceConstants equivalence;
  double theta_min = 0.25;
  double theta_max = 0.25;
  double spread_scaled = 0.0;
  double spread_unscaled = 0.0;
};
inline BoundsConstants make_bounds(double theta, double eps, int offset) {
  BoundsConstants b;
  b.theta = theta;
  b.eps = eps;
  b.offset = offset;
  b.order = static_cast<int>(std::lround(-std::log2(theta)));
  b.theta_eps = (1.0 + eps) * theta;
  b.equivalence = effectivity_constants(theta, eps, offset);
  b.theta_min = theta;
  b.theta_max = theta;
  b.spread_scaled = local_spread_bound_scaled(theta, eps, offset);
  b.spread_unscaled = local_spread_bound_unscaled(theta, theta, offset);
  return b;
}
inline BoundsConstants make_bounds_from_order(int order, double eps, int offset) {
  BoundsConstants b = make_bounds(std::pow(2.0, -static_cast<double>(order)), eps, offset);
  b.order = order;
  return b;
}
struct EffectivityReport {
  double gamma = 0.0;
  bool gamma_valid = false;
  std::vector<double> gamma_local;
  double spread = 0.0;
  bool spread_valid = false;
};
inline EffectivityReport effectivity_index(const EstimateReport& report, const ErrorNorms& exact) {
  EffectivityReport out;
  out.gamma_local.assign(report.eta_local.size(), 0.0);
  int gv = 0, sv = 0;
  detail::check(klref_effectivity_index(report.eta, static_cast<int>(report.eta_local.size()), report.eta_local.data(),
                                        exact.global, static_cast<int>(exact.per_macro.size()),
                                        exact.per_macro.data(), &out.gamma, &gv, out.gamma_local.data(),
                                        &out.spread, &sv));
  out.gamma_valid = gv != 0;
  out.spread_valid = sv != 0;
  return out;
}

}  // namespace klref

#endif  // KLREF_B200_KLREF_HPP
