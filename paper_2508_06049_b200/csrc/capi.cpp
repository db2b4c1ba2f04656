// extern "C" boundary of libklref_b200.so (include/klref_b200.h).  Converts
// the internal C++ exceptions (kb::Error, mirroring the reference's
// errors.hpp) into status codes plus a thread-local message.
#include "../../include/klref_b200.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "solver2d.hpp"
#include "solver3d.hpp"
#include "solver3d_shard.hpp"

struct klref_mesh_s {
  int dim = 2;
  kb::Mesh2D mesh;
  kb::Mesh3D mesh3;
};
struct klref_hierarchy_s {
  int dim = 2;
  std::shared_ptr<kb::DeviceHierarchy2D> dev;   // 2-d (lev empty for host-only builds)
  std::shared_ptr<kb::DeviceHierarchy3D> dev3;  // 3-d
  bool on_device = false;
};
struct klref_problem_s {
  kb::Problem2D p;
  kb::Problem3D p3;
  int dims = 1;  // bit mask of the dimensions this problem is defined for (1: 2-d, 2: 3-d)
};
struct klref_solver_s {
  std::unique_ptr<kb::Solver2D> s;
  std::unique_ptr<kb::Solver3D> s3;
  klref_hierarchy_s* h = nullptr;
};
struct klref_comm_s {
  std::shared_ptr<kb::NcclComm> c;
};
struct klref_sharded_s {
  std::unique_ptr<kb::ShardedSolver3D> s;
};
struct klref_gf_s {
  double* d = nullptr;
  size_t count = 0;
  int level = 0;
  klref_hierarchy_s* h = nullptr;
};

namespace {

thread_local std::string g_msg;
thread_local double g_residual = 0.0;
thread_local int g_level = -1;

int set_error(int code, const std::string& msg, double residual = 0.0, int level = -1) {
  g_msg = msg;
  g_residual = residual;
  g_level = level;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return KLREF_OK;
  } catch (const kb::Error& e) {
    return set_error(e.code, e.what(), e.residual, e.level);
  } catch (const std::bad_alloc&) {
    return set_error(KLREF_ERR_RESOURCE, "host allocation failed");
  } catch (const std::exception& e) {
    return set_error(KLREF_ERR_INTERNAL, e.what());
  }
}

void require_device() {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    kb::fail(kb::KB_CUDA, std::string("no CUDA device available (the hot path has no CPU fallback): ") +
                              (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
}

void need(const void* p, const char* what) {
  if (!p) kb::fail(kb::KB_STRUCTURAL, std::string("null argument: ") + what);
}

const kb::Hierarchy2D& host_of(klref_hierarchy h) {
  if (h->dim != 2) kb::fail(kb::KB_STRUCTURAL, "this query needs a 2-d hierarchy");
  return h->dev->host;
}
int max_level_of(klref_hierarchy h) { return h->dim == 3 ? h->dev3->host.L : h->dev->host.L; }
int macros_of(klref_hierarchy h) { return h->dim == 3 ? h->dev3->host.M : h->dev->host.M; }
int lattice_size_of(klref_hierarchy h, int l) {
  return h->dim == 3 ? h->dev3->host.levels[l].S : h->dev->host.levels[l].S;
}

void check_level(klref_hierarchy h, int level) {
  if (level < 0 || level > max_level_of(h)) kb::fail(kb::KB_STRUCTURAL, "level out of range");
}

// run f on the solver of either dimension (same method names)
template <typename F>
void on_solver(klref_solver s, F&& f) {
  if (s->s3)
    f(*s->s3);
  else
    f(*s->s);
}

void same_hier(klref_solver s, klref_gf f) {
  need(f, "grid function");
  if (f->h != s->h) kb::fail(kb::KB_STRUCTURAL, "grid function belongs to another hierarchy");
}

}  // namespace

extern "C" {

const char* klref_last_error(void) { return g_msg.c_str(); }
double klref_last_error_residual(void) { return g_residual; }
int klref_last_error_level(void) { return g_level; }
int klref_abi_version(void) { return 1; }
int klref_device_init(void) {
  return guarded([&] { KB_CUDA_CHECK(cudaFree(nullptr)); });
}

int klref_mesh_create(int dim, int num_vertices, const double* coords, int num_elements, const int* corners,
                      klref_mesh* out) {
  return guarded([&] {
    need(coords, "coords");
    need(corners, "corners");
    need(out, "out");
    if (dim != 2 && dim != 3) kb::fail(kb::KB_STRUCTURAL, "macro meshes are 2-d (triangles) or 3-d (tetrahedra)");
    auto m = std::make_unique<klref_mesh_s>();
    m->dim = dim;
    if (dim == 2)
      m->mesh = kb::Mesh2D::create(num_vertices, coords, num_elements, corners);
    else
      m->mesh3 = kb::Mesh3D::create(num_vertices, coords, num_elements, corners);
    *out = m.release();
  });
}

void klref_mesh_destroy(klref_mesh mesh) { delete mesh; }

static int build_impl(klref_mesh mesh, int max_level, klref_hierarchy* out, bool device) {
  return guarded([&] {
    need(mesh, "mesh");
    need(out, "out");
    auto h = std::make_unique<klref_hierarchy_s>();
    h->dim = mesh->dim;
    if (mesh->dim == 3) {
      if (device) {
        require_device();
        h->dev3 = kb::DeviceHierarchy3D::create(mesh->mesh3, max_level);
        h->on_device = true;
      } else {
        h->dev3 = std::make_shared<kb::DeviceHierarchy3D>();
        h->dev3->host = kb::Hierarchy3D::build(mesh->mesh3, max_level);
      }
    } else if (device) {
      require_device();
      h->dev = kb::DeviceHierarchy2D::create(mesh->mesh, max_level);
      h->on_device = true;
    } else {
      h->dev = std::make_shared<kb::DeviceHierarchy2D>();
      h->dev->host = kb::Hierarchy2D::build(mesh->mesh, max_level);
    }
    *out = h.release();
  });
}

int klref_hierarchy_build(klref_mesh mesh, int max_level, klref_hierarchy* out) {
  return build_impl(mesh, max_level, out, true);
}
int klref_hierarchy_build_host(klref_mesh mesh, int max_level, klref_hierarchy* out) {
  return build_impl(mesh, max_level, out, false);
}
void klref_hierarchy_destroy(klref_hierarchy h) { delete h; }

int klref_hierarchy_num_macros(klref_hierarchy h, int* out) {
  return guarded([&] {
    need(h, "h");
    *out = macros_of(h);
  });
}
int klref_hierarchy_max_level(klref_hierarchy h, int* out) {
  return guarded([&] {
    need(h, "h");
    *out = max_level_of(h);
  });
}
int klref_hierarchy_dof_count(klref_hierarchy h, int level, int64_t* out) {
  return guarded([&] {
    need(h, "h");
    check_level(h, level);
    *out = h->dim == 3 ? h->dev3->host.levels[level].dofs : host_of(h).levels[level].dofs;
  });
}
int klref_hierarchy_fine_element_count(klref_hierarchy h, int level, int64_t* out) {
  return guarded([&] {
    need(h, "h");
    *out = static_cast<int64_t>(macros_of(h)) << (h->dim * level);
  });
}
int klref_hierarchy_lattice_size(klref_hierarchy h, int level, int* out) {
  return guarded([&] {
    need(h, "h");
    check_level(h, level);
    *out = lattice_size_of(h, level);
  });
}
int klref_hierarchy_dag_depth(klref_hierarchy h, int* out) {
  return guarded([&] {
    need(h, "h");
    *out = h->dim == 3 ? 0 : host_of(h).dag_depth;
  });
}
int klref_hierarchy_groups(klref_hierarchy h, int level, int* num_groups, int* num_members, int* ptr,
                           int* members) {
  return guarded([&] {
    need(h, "h");
    check_level(h, level);
    if (h->dim == 3) {
      const kb::Level3D& l3 = h->dev3->host.levels[level];
      if (num_groups) *num_groups = static_cast<int>(l3.grp_ptr.size()) - 1;
      if (num_members) *num_members = static_cast<int>(l3.mem_slot.size());
      if (ptr) std::copy(l3.grp_ptr.begin(), l3.grp_ptr.end(), ptr);
      if (members)
        for (size_t k = 0; k < l3.mem_slot.size(); ++k) {
          members[4 * k] = l3.mem_slot[k];
          members[4 * k + 1] = l3.mem_idx[k];
          members[4 * k + 2] = members[4 * k + 3] = 0;
        }
      return;
    }
    const kb::Level2D& lv = host_of(h).levels[level];
    if (num_groups) *num_groups = static_cast<int>(lv.grp_ptr.size()) - 1;
    if (num_members) *num_members = static_cast<int>(lv.mem_slot.size());
    if (ptr) std::copy(lv.grp_ptr.begin(), lv.grp_ptr.end(), ptr);
    if (members)
      for (size_t k = 0; k < lv.mem_slot.size(); ++k) {
        members[4 * k] = lv.mem_slot[k];
        members[4 * k + 1] = lv.mem_idx[k];
        members[4 * k + 2] = lv.mem_i[k];
        members[4 * k + 3] = lv.mem_j[k];
      }
  });
}
int klref_hierarchy_element_matrices(klref_hierarchy h, int level, int kind, double* mats, double* stencil) {
  return guarded([&] {
    need(h, "h");
    check_level(h, level);
    if (h->dim == 3) {  // mats[96 M] (six micro-tet types, 4x4), stencil[15 M]
      const kb::Level3D& l3 = h->dev3->host.levels[level];
      if (mats) {
        const auto& src = kind == KLREF_MASS ? l3.kmass : l3.kstiff;
        std::copy(src.begin(), src.end(), mats);
      }
      if (stencil) std::copy(l3.stencil.begin(), l3.stencil.end(), stencil);
      return;
    }
    const kb::Level2D& lv = host_of(h).levels[level];
    if (mats) {
      const auto& src = kind == KLREF_MASS ? lv.kmass : lv.kstiff;
      std::copy(src.begin(), src.end(), mats);
    }
    if (stencil) std::copy(lv.stencil.begin(), lv.stencil.end(), stencil);
  });
}

int klref_problem_create(int kind, klref_problem* out) {
  return guarded([&] {
    need(out, "out");
    auto p = std::make_unique<klref_problem_s>();
    if (kind == KLREF_PROBLEM_ZERO) {
      p->p = kb::Problem2D::builtin(kind);
      p->p3 = kb::Problem3D::builtin(kb::P3_ZERO);
      p->dims = 3;
    } else if (kind >= KLREF_PROBLEM_SIN3D) {
      p->p3 = kb::Problem3D::builtin(kind);
      p->dims = 2;
    } else {
      p->p = kb::Problem2D::builtin(kind);
      p->dims = 1;
    }
    *out = p.release();
  });
}

int klref_problem_create_host(double (*source)(double, double, void*), double (*boundary)(double, double, void*),
                              void* ctx, klref_problem* out) {
  return guarded([&] {
    need(out, "out");
    need(reinterpret_cast<const void*>(source), "source");
    need(reinterpret_cast<const void*>(boundary), "boundary");
    auto p = std::make_unique<klref_problem_s>();
    p->p.kind = kb::PROB_HOST;
    p->p.source = [source, ctx](double x, double y) { return source(x, y, ctx); };
    p->p.boundary = [boundary, ctx](double x, double y) { return boundary(x, y, ctx); };
    p->p.has_exact = false;
    *out = p.release();
  });
}
int klref_problem_set_exact(klref_problem p, double (*exact)(double, double, void*), void* ctx) {
  return guarded([&] {
    need(p, "problem");
    need(reinterpret_cast<const void*>(exact), "exact");
    p->p.exact = [exact, ctx](double x, double y) { return exact(x, y, ctx); };
    p->p.has_exact = true;
  });
}
int klref_problem_create_host3(double (*source)(double, double, double, void*),
                               double (*boundary)(double, double, double, void*), void* ctx, klref_problem* out) {
  return guarded([&] {
    need(out, "out");
    need(reinterpret_cast<const void*>(source), "source");
    need(reinterpret_cast<const void*>(boundary), "boundary");
    auto p = std::make_unique<klref_problem_s>();
    p->p3.kind = kb::P3_HOST;
    p->p3.source = [source, ctx](double x, double y, double z) { return source(x, y, z, ctx); };
    p->p3.boundary = [boundary, ctx](double x, double y, double z) { return boundary(x, y, z, ctx); };
    p->dims = 2;
    *out = p.release();
  });
}
int klref_problem_set_params(klref_problem p, const double* params, int count) {
  return guarded([&] {
    need(p, "problem");
    need(params, "params");
    if (!(p->dims & 2)) kb::fail(kb::KB_STRUCTURAL, "parameters belong to 3-d series problems");
    p->p3.set_params(params, count);
  });
}
void klref_problem_destroy(klref_problem p) { delete p; }

void klref_solver_config_default(klref_solver_config* cfg) {
  if (!cfg) return;
  cfg->nu = 2;
  cfg->pre_smooth = 2;
  cfg->post_smooth = 2;
  cfg->coarse_rel_tol = 1e-9;
  cfg->coarse_abs_floor = 1e-12;
  cfg->coarse_max_iter = 100000;
  cfg->finest_policy = 0;
  cfg->faithful_source = 0;
  cfg->use_graph = 1;
  cfg->max_extra_cycles = 60;
}

int klref_solver_create(klref_hierarchy h, klref_problem p, const klref_solver_config* cfg, klref_solver* out) {
  return guarded([&] {
    need(h, "h");
    need(p, "problem");
    need(out, "out");
    require_device();
    if (!h->on_device) kb::fail(kb::KB_STRUCTURAL, "hierarchy was built host-only");
    kb::SolverConfig2D c;
    if (cfg) {
      c.nu = cfg->nu;
      c.pre_smooth = cfg->pre_smooth;
      c.post_smooth = cfg->post_smooth;
      c.coarse_rel_tol = cfg->coarse_rel_tol;
      c.coarse_abs_floor = cfg->coarse_abs_floor;
      c.coarse_max_iter = cfg->coarse_max_iter;
      c.finest_policy = cfg->finest_policy;
      c.faithful_source = cfg->faithful_source;
      c.use_graph = cfg->use_graph;
      c.max_extra_cycles = cfg->max_extra_cycles;
    }
    auto s = std::make_unique<klref_solver_s>();
    if (h->dim == 3) {
      if (!(p->dims & 2)) kb::fail(kb::KB_STRUCTURAL, "a 2-d problem cannot drive a 3-d hierarchy");
      s->s3 = std::make_unique<kb::Solver3D>(h->dev3, p->p3, c);
    } else {
      if (!(p->dims & 1)) kb::fail(kb::KB_STRUCTURAL, "a 3-d problem cannot drive a 2-d hierarchy");
      s->s = std::make_unique<kb::Solver2D>(h->dev, p->p, c);
    }
    s->h = h;
    *out = s.release();
  });
}
void klref_solver_destroy(klref_solver s) { delete s; }

int klref_solver_fmg(klref_solver s) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.fmg(); });
  });
}
int klref_solver_fmg_enqueue(klref_solver s) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.fmg_enqueue(); });
  });
}
int klref_solver_synchronize(klref_solver s) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.sync_and_check(); });
  });
}
int klref_solver_stream(klref_solver s, void** stream) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { *stream = reinterpret_cast<void*>(v.stream()); });
  });
}
int klref_solver_launch_count(klref_solver s, int* out) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { *out = v.launches_per_fmg(); });
  });
}
int klref_solver_last_cg_iterations(klref_solver s, int* out) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { *out = v.last_cg_iters(); });
  });
}
int klref_solver_estimate_launch_count(klref_solver s, int* out) {
  return guarded([&] {
    need(s, "solver");
    need(out, "out");
    on_solver(s, [&](auto& v) { *out = v.launches_per_estimate(); });
  });
}
int klref_solver_set_stream(klref_solver s, void* stream) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.set_stream(reinterpret_cast<cudaStream_t>(stream)); });
  });
}
int klref_solver_set_problem(klref_solver s, klref_problem p, int64_t* h2d_bytes) {
  return guarded([&] {
    need(s, "solver");
    need(p, "problem");
    size_t b;
    if (s->s3)
      b = s->s3->load_problem(p->p3);
    else
      b = s->s->load_problem(p->p);
    if (h2d_bytes) *h2d_bytes = static_cast<int64_t>(b);
  });
}
int klref_solver_set_profiling(klref_solver s, int on) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.set_profiling(on != 0); });
  });
}
int klref_solver_kernel_stats(klref_solver s, int kind, double* ms, int* launches, double* bytes) {
  return guarded([&] {
    need(s, "solver");
    if (kind < KLREF_KERNEL_ALL || kind >= kb::KK_COUNT) kb::fail(kb::KB_STRUCTURAL, "unknown kernel kind");
    on_solver(s, [&](auto& v) { v.kernel_stats(kind, ms, launches, bytes); });
  });
}
int klref_solver_state_read(klref_solver s, int which, int level, double* host_out) {
  return guarded([&] {
    need(s, "solver");
    need(host_out, "host_out");
    on_solver(s, [&](auto& v) {
      const double* d = v.state(which, level);
      const size_t count = v.level_size(level);
      KB_CUDA_CHECK(cudaMemcpyAsync(host_out, d, count * 8, cudaMemcpyDeviceToHost, v.stream()));
      KB_CUDA_CHECK(cudaStreamSynchronize(v.stream()));
    });
  });
}

int klref_solver_exact_error(klref_solver s, double* global, double* per_macro) {
  return guarded([&] {
    need(s, "solver");
    if (!s->s) kb::fail(kb::KB_STRUCTURAL, "the exact-error evaluator is defined for 2-d hierarchies");
    const auto e = s->s->exact_error();
    if (global) *global = e.global;
    if (per_macro) std::copy(e.per_macro.begin(), e.per_macro.end(), per_macro);
  });
}
int klref_solver_exact_error_of(klref_solver s, klref_gf u, double* global, double* per_macro) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, u);
    if (!s->s) kb::fail(kb::KB_STRUCTURAL, "the exact-error evaluator is defined for 2-d hierarchies");
    if (u->level != s->s->hier().L) kb::fail(kb::KB_STRUCTURAL, "the exact-error evaluator works on the finest level");
    const auto e = s->s->exact_error(u->d);
    if (global) *global = e.global;
    if (per_macro) std::copy(e.per_macro.begin(), e.per_macro.end(), per_macro);
  });
}
int klref_solver_solve_direct(klref_solver s, int level, klref_gf u) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, u);
    if (!s->s) kb::fail(kb::KB_STRUCTURAL, "solve_direct is defined for 2-d hierarchies");
    if (u->level != level) kb::fail(kb::KB_STRUCTURAL, "grid function level mismatch");
    s->s->solve_direct(level, u->d);
  });
}
int klref_solver_extra_cycles(klref_solver s, int* out) {
  return guarded([&] {
    need(s, "solver");
    need(out, "out");
    *out = s->s ? s->s->extra_cycles() : 0;
  });
}

static void fill_report(const kb::EstimateReport2D& r, klref_estimate_report* out, double* eta_local) {
  if (out) {
    out->offset = r.offset;
    out->base_level = r.base_level;
    out->kind = r.kind;
    out->norm_coarser = r.norm_coarser;
    out->norm_base = r.norm_base;
    out->conv_factor = r.conv_factor;
    out->eta = r.eta;
  }
  if (eta_local) std::copy(r.eta_local.begin(), r.eta_local.end(), eta_local);
}

int klref_error_estimate(klref_solver s, int offset, int kind, klref_estimate_report* out, double* eta_local) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { fill_report(v.estimate(offset, kind), out, eta_local); });
  });
}
int klref_error_estimate_enqueue(klref_solver s, int offset) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { v.estimate_enqueue(offset); });
  });
}
int klref_error_estimate_finish(klref_solver s, int offset, int kind, klref_estimate_report* out,
                                double* eta_local) {
  return guarded([&] {
    need(s, "solver");
    on_solver(s, [&](auto& v) { fill_report(v.estimate_finish(offset, kind), out, eta_local); });
  });
}

int klref_gf_create(klref_hierarchy h, int level, klref_gf* out) {
  return guarded([&] {
    need(h, "h");
    need(out, "out");
    require_device();
    check_level(h, level);
    auto f = std::make_unique<klref_gf_s>();
    f->count = static_cast<size_t>(macros_of(h)) * lattice_size_of(h, level);
    f->level = level;
    f->h = h;
    KB_CUDA_CHECK(cudaMalloc(&f->d, f->count * 8));
    KB_CUDA_CHECK(cudaMemset(f->d, 0, f->count * 8));
    *out = f.release();
  });
}
void klref_gf_destroy(klref_gf f) {
  if (!f) return;
  if (f->d) cudaFree(f->d);
  delete f;
}
int klref_gf_upload(klref_gf f, const double* host) {
  return guarded([&] {
    need(f, "f");
    need(host, "host");
    KB_CUDA_CHECK(cudaMemcpy(f->d, host, f->count * 8, cudaMemcpyHostToDevice));
  });
}
int klref_gf_download(klref_gf f, double* host) {
  return guarded([&] {
    need(f, "f");
    need(host, "host");
    KB_CUDA_CHECK(cudaMemcpy(host, f->d, f->count * 8, cudaMemcpyDeviceToHost));
  });
}

int klref_apply(klref_solver s, int kind, klref_gf x, klref_gf y) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, x);
    same_hier(s, y);
    if (x->level != y->level) kb::fail(kb::KB_STRUCTURAL, "operator level mismatch");
    on_solver(s, [&](auto& v) { v.apply(x->level, kind == KLREF_MASS, x->d, y->d); });
  });
}
int klref_residual(klref_solver s, klref_gf u, klref_gf b, klref_gf r) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, u);
    same_hier(s, b);
    same_hier(s, r);
    if (u->level != b->level || u->level != r->level) kb::fail(kb::KB_STRUCTURAL, "grid function level mismatch");
    on_solver(s, [&](auto& v) { v.residual(u->level, u->d, b->d, r->d); });
  });
}
int klref_gauss_seidel(klref_solver s, klref_gf u, klref_gf b, int sweeps) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, u);
    same_hier(s, b);
    if (u->level != b->level) kb::fail(kb::KB_STRUCTURAL, "grid function level mismatch");
    on_solver(s, [&](auto& v) { v.gauss_seidel(u->level, u->d, b->d, sweeps); });
  });
}
int klref_restrict_transpose(klref_solver s, klref_gf fine, klref_gf coarse) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, fine);
    same_hier(s, coarse);
    if (coarse->level + 1 != fine->level) kb::fail(kb::KB_STRUCTURAL, "restriction level mismatch");
    on_solver(s, [&](auto& v) { v.restrict_to(fine->level, fine->d, coarse->d); });
  });
}
int klref_prolongate(klref_solver s, klref_gf coarse, klref_gf fine) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, fine);
    same_hier(s, coarse);
    if (coarse->level + 1 != fine->level) kb::fail(kb::KB_STRUCTURAL, "prolongation level mismatch");
    on_solver(s, [&](auto& v) { v.prolongate(coarse->level, coarse->d, fine->d); });
  });
}
int klref_cg_level0(klref_solver s, klref_gf u, klref_gf b) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, u);
    same_hier(s, b);
    if (u->level != 0 || b->level != 0) kb::fail(kb::KB_STRUCTURAL, "cg_level0 works on level 0");
    on_solver(s, [&](auto& v) { v.cg_level0(u->d, b->d); });
  });
}
int klref_dot_unique(klref_solver s, klref_gf a, klref_gf b, double* out) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, a);
    same_hier(s, b);
    need(out, "out");
    if (a->level != b->level) kb::fail(kb::KB_STRUCTURAL, "grid function level mismatch");
    on_solver(s, [&](auto& v) { *out = v.dot_unique(a->level, a->d, b->d); });
  });
}
int klref_interface_sync(klref_solver s, klref_gf f, int mode) {
  return guarded([&] {
    need(s, "solver");
    same_hier(s, f);
    on_solver(s, [&](auto& v) { v.interface_sync(f->level, f->d, mode == KLREF_SYNC_ADDITIVE); });
  });
}

// ---- effectivity constants and indices (host, O(1) / O(M)) -------------
// proj/src/estimator.cpp:47-123: the equivalence constants C1, C2 of the
// error bound, the local spread bounds, and the validation-mode effectivity
// indices against the exact error.
int klref_effectivity_constants(double theta, double eps, int offset, double* lower, double* upper) {
  return guarded([&] {
    need(lower, "lower");
    need(upper, "upper");
    const double theta_eps = (1.0 + eps) * theta;
    if (!(theta > 0.0) || eps < 0.0 || offset < 1)
      kb::fail(kb::KB_DOMAIN, "effectivity constants need theta > 0, eps >= 0, offset >= 1");
    if (theta_eps >= 1.0) kb::fail(kb::KB_DOMAIN, "saturation requires (1 + eps) * theta < 1");
    const double j = static_cast<double>(offset);
    *lower = std::pow(1.0 + eps, -j) * std::pow(1.0 - std::pow(theta_eps, j), j + 1.0) /
             std::pow(1.0 + std::pow(theta_eps, j + 1.0), j);
    *upper = std::pow(1.0 + eps, j) * std::pow(1.0 + std::pow(theta_eps, j), j + 1.0) /
             std::pow(1.0 - std::pow(theta_eps, j + 1.0), j);
  });
}

int klref_local_spread_bound_scaled(double theta_max, double eps, int offset, double* out) {
  return guarded([&] {
    need(out, "out");
    if (!(theta_max > 0.0) || eps < 0.0 || offset < 1 || (1.0 + eps) * theta_max >= 1.0)
      kb::fail(kb::KB_DOMAIN, "spread bound requires (1 + eps) * theta_max < 1");
    const double j = static_cast<double>(offset);
    const double tj = std::pow(theta_max, j), tj1 = std::pow(theta_max, j + 1.0);
    *out = std::pow(1.0 + eps, 2.0 * j) * std::pow((1.0 + tj1) / (1.0 - tj1), j) *
           std::pow((1.0 + tj) / (1.0 - tj), j + 1.0);
  });
}

int klref_local_spread_bound_unscaled(double theta_min, double theta_max, int offset, double* out) {
  return guarded([&] {
    need(out, "out");
    if (!(theta_min > 0.0) || theta_min > theta_max || offset < 1)
      kb::fail(kb::KB_DOMAIN, "spread bound requires 0 < theta_min <= theta_max");
    if (theta_max >= 1.0) kb::fail(kb::KB_DOMAIN, "spread bound requires theta_max < 1");
    const double j = static_cast<double>(offset);
    *out = (std::pow(theta_min, -j) + 1.0) / (std::pow(theta_max, -j) - 1.0);
  });
}

int klref_effectivity_index(double eta, int num_local, const double* eta_local, double exact_global,
                            int num_exact, const double* exact_local, double* gamma, int* gamma_valid,
                            double* gamma_local, double* spread, int* spread_valid) {
  return guarded([&] {
    need(gamma, "gamma");
    need(gamma_valid, "gamma_valid");
    need(spread, "spread");
    need(spread_valid, "spread_valid");
    if (num_local > 0) {
      need(eta_local, "eta_local");
      need(gamma_local, "gamma_local");
    }
    if (num_exact > 0) need(exact_local, "exact_local");
    const double nan = std::numeric_limits<double>::quiet_NaN();
    *gamma_valid = exact_global > 0.0;
    *gamma = *gamma_valid ? eta / exact_global : nan;
    double lo = std::numeric_limits<double>::infinity(), hi = 0.0;
    bool any = false;
    const double cutoff = 1e-14 * exact_global;
    for (int t = 0; t < num_local; ++t) {
      gamma_local[t] = nan;
      if (t >= num_exact) continue;
      if (exact_local[t] <= cutoff || exact_local[t] == 0.0) continue;
      const double g = eta_local[t] / exact_local[t];
      gamma_local[t] = g;
      lo = std::min(lo, g);
      hi = std::max(hi, g);
      any = true;
    }
    *spread_valid = any && lo > 0.0;
    *spread = *spread_valid ? hi / lo : nan;
  });
}

int klref_mark(int rule, double fraction, int num_active, const int* active_ids, const int* green_parent,
               const double* indicator, int num_reverted, const int* reverted_ids, int* marks_out, int* num_marks) {
  return guarded([&] {
    need(active_ids, "active_ids");
    need(indicator, "indicator");
    need(reverted_ids, "reverted_ids");
    need(marks_out, "marks_out");
    need(num_marks, "num_marks");
    // aggregation on the green-reverted set, proj/src/amr.cpp:45-65
    std::map<int, double> by_id;
    for (int t = 0; t < num_active; ++t) by_id[active_ids[t]] = indicator[t];
    std::vector<double> agg(num_reverted, 0.0);
    for (int t = 0; t < num_reverted; ++t) {
      const int id = reverted_ids[t];
      auto it = by_id.find(id);
      if (it != by_id.end()) {
        agg[t] = it->second;
        continue;
      }
      double sq = 0.0;
      for (int a = 0; a < num_active; ++a)
        if (green_parent && green_parent[a] == id) sq += indicator[a] * indicator[a];
      agg[t] = std::sqrt(sq);
    }
    std::vector<int> marks;
    if (rule == KLREF_MARK_TOP_FRACTION) {
      // mark_top_fraction, proj/src/macro_mesh.cpp:678-695
      if (!(fraction > 0.0) || fraction > 1.0) kb::fail(kb::KB_STRUCTURAL, "mark fraction must be in (0, 1]");
      const size_t count = static_cast<size_t>(std::ceil(fraction * static_cast<double>(num_reverted)));
      std::vector<size_t> order(num_reverted);
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        if (agg[a] != agg[b]) return agg[a] > agg[b];
        return reverted_ids[a] < reverted_ids[b];
      });
      for (size_t i = 0; i < count; ++i) marks.push_back(reverted_ids[order[i]]);
    } else if (rule == KLREF_MARK_HALF_MAX) {
      double mx = 0.0;
      for (double v : agg) mx = std::max(mx, v);
      for (int t = 0; t < num_reverted; ++t)
        if (agg[t] >= 0.5 * mx) marks.push_back(reverted_ids[t]);
    } else {
      kb::fail(kb::KB_STRUCTURAL, "unknown marking rule");
    }
    std::sort(marks.begin(), marks.end());
    std::copy(marks.begin(), marks.end(), marks_out);
    *num_marks = static_cast<int>(marks.size());
  });
}

int klref_comm_unique_id(unsigned char id[128]) {
  return guarded([&] {
    need(id, "id");
    kb::NcclComm::unique_id(id);
  });
}
int klref_comm_create(int nranks, int rank, const unsigned char id[128], klref_comm* out) {
  return guarded([&] {
    need(id, "id");
    need(out, "out");
    require_device();
    auto c = std::make_unique<klref_comm_s>();
    c->c = std::make_shared<kb::NcclComm>(nranks, rank, id);
    *out = c.release();
  });
}
void klref_comm_destroy(klref_comm c) { delete c; }

int klref_sharded_create(klref_hierarchy h, klref_problem p, const klref_solver_config* cfg, klref_comm comm,
                         int local_shards, int rep_level, klref_sharded* out) {
  return guarded([&] {
    need(h, "h");
    need(p, "problem");
    need(out, "out");
    require_device();
    if (!h->on_device) kb::fail(kb::KB_STRUCTURAL, "hierarchy was built host-only");
    if (h->dim != 3) kb::fail(kb::KB_STRUCTURAL, "sharding is defined for 3-d hierarchies (the 2-d path is exact-order)");
    if (!(p->dims & 2)) kb::fail(kb::KB_STRUCTURAL, "a 2-d problem cannot drive a 3-d hierarchy");
    kb::SolverConfig2D c;
    if (cfg) {
      c.nu = cfg->nu;
      c.pre_smooth = cfg->pre_smooth;
      c.post_smooth = cfg->post_smooth;
      c.coarse_rel_tol = cfg->coarse_rel_tol;
      c.coarse_abs_floor = cfg->coarse_abs_floor;
      c.coarse_max_iter = cfg->coarse_max_iter;
      c.finest_policy = cfg->finest_policy;
      c.faithful_source = cfg->faithful_source;
      c.use_graph = cfg->use_graph;
    }
    auto s = std::make_unique<klref_sharded_s>();
    s->s = std::make_unique<kb::ShardedSolver3D>(h->dev3, p->p3, c, local_shards, rep_level,
                                                 comm ? comm->c : nullptr);
    *out = s.release();
  });
}
void klref_sharded_destroy(klref_sharded s) { delete s; }
int klref_sharded_fmg(klref_sharded s) {
  return guarded([&] {
    need(s, "solver");
    s->s->fmg();
  });
}
int klref_sharded_fmg_enqueue(klref_sharded s) {
  return guarded([&] {
    need(s, "solver");
    s->s->fmg_enqueue();
  });
}
int klref_sharded_synchronize(klref_sharded s) {
  return guarded([&] {
    need(s, "solver");
    s->s->sync_and_check();
  });
}
int klref_sharded_stream(klref_sharded s, void** stream) {
  return guarded([&] {
    need(s, "solver");
    need(stream, "stream");
    *stream = reinterpret_cast<void*>(s->s->stream());
  });
}
int klref_sharded_counts(klref_sharded s, int* fmg_launches, int* estimate_launches, double* exchange_bytes) {
  return guarded([&] {
    need(s, "solver");
    if (fmg_launches) *fmg_launches = s->s->launches_per_fmg();
    if (estimate_launches) *estimate_launches = s->s->launches_per_estimate();
    if (exchange_bytes) *exchange_bytes = s->s->exchange_bytes_per_fmg();
  });
}
int klref_sharded_error_estimate_enqueue(klref_sharded s, int offset) {
  return guarded([&] {
    need(s, "solver");
    s->s->estimate_enqueue(offset);
  });
}
int klref_sharded_error_estimate_finish(klref_sharded s, int offset, int kind, klref_estimate_report* out,
                                        double* eta_local) {
  return guarded([&] {
    need(s, "solver");
    fill_report(s->s->estimate_finish(offset, kind), out, eta_local);
  });
}
int klref_sharded_state_read(klref_sharded s, int which, int level, double* host_out) {
  return guarded([&] {
    need(s, "solver");
    need(host_out, "host_out");
    s->s->state_read(which, level, host_out);
  });
}
int klref_shard_plan(klref_hierarchy h, int nshards, int rank, int rep_level, int level, int* colors,
                     int64_t* send_counts, int64_t* recv_counts, int* send_keys, int* recv_keys) {
  return guarded([&] {
    need(h, "h");
    if (h->dim != 3) kb::fail(kb::KB_STRUCTURAL, "sharding is defined for 3-d hierarchies");
    check_level(h, level);
    const kb::Hierarchy3D& hh = h->dev3->host;
    const kb::ShardPlan3D plan = kb::build_shard_plan(hh, nshards, rank, rep_level);
    if (colors) *colors = hh.colors;
    const int C = hh.colors;
    const kb::ShardLevel3D& sl = plan.lev[level];
    for (int p = 0; p < nshards; ++p)
      for (int c = 0; c < C; ++c) {
        const size_t o = static_cast<size_t>(p) * (C + 1) + c;
        if (send_counts) send_counts[p * C + c] = plan.sharded(level) ? sl.send_off[o + 1] - sl.send_off[o] : 0;
        if (recv_counts) recv_counts[p * C + c] = plan.sharded(level) ? sl.recv_off[o + 1] - sl.recv_off[o] : 0;
      }
    if (!plan.sharded(level)) return;
    if (send_keys)
      for (size_t e = 0; e < sl.pack_pos.size(); ++e) {
        int* k = send_keys + 3 * static_cast<size_t>(sl.pack_pos[e]);
        k[0] = sl.pack_gid[e];
        k[1] = sl.pack_slot[e] + plan.s0;
        k[2] = sl.pack_idx[e];
      }
    if (recv_keys) {
      const kb::Level3D& lv = hh.levels[level];
      for (int g = 0; g < sl.ng; ++g) {
        const int gg = sl.gid[g];
        for (int q = sl.grp_ptr[g]; q < sl.grp_ptr[g + 1]; ++q) {
          if (sl.mem_slot[q] >= 0) continue;
          const int gq = lv.grp_ptr[gg] + (q - sl.grp_ptr[g]);
          int* k = recv_keys + 3 * static_cast<size_t>(~sl.mem_slot[q]);
          k[0] = gg;
          k[1] = lv.mem_slot[gq];
          k[2] = lv.mem_idx[gq];
        }
      }
    }
  });
}
int klref_shard_starts(int num_macros, int nshards, int* starts) {
  return guarded([&] {
    need(starts, "starts");
    if (nshards < 1 || nshards > num_macros) kb::fail(kb::KB_STRUCTURAL, "shard count out of range");
    const std::vector<int> st = kb::shard_starts(num_macros, nshards);
    std::copy(st.begin(), st.end(), starts);
  });
}

}  // extern "C"
