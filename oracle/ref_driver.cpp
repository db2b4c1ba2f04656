// Test infrastructure (oracle), not product code.
//
// Driver that links the *patched* reference (oracle/build_ref.sh) and runs its
// hot path through the reference's own public API:
//   GridHierarchy::build        proj/src/hhg.cpp:48
//   MultigridSolver::fmg        proj/src/multigrid.cpp:248
//   error_estimate              proj/src/estimator.cpp:8
//   OperatorP1::apply           proj/src/fem.cpp:95
//   MultigridSolver::gauss_seidel/residual   proj/src/multigrid.cpp:127,183
//   restrict_transpose/prolongate            proj/src/multigrid.cpp:55,22
// It writes golden data (raw little-endian fp64 per macro lattice, text
// reports) consumed by tests/gen_golden.py, and times the reference for the
// CPU baseline leg of bench.py.  It never runs inside the product path.
//
// Commands:
//   ref_driver mesh  <cfg1|cfg2> <out.mesh>
//   ref_driver solve <mesh> <sin|lshape|zero> <L> <nu> <outdir>
//   ref_driver amr   <mesh> <sin|lshape> <L> <nu> <K> <halfmax|top10> <outdir>
//   ref_driver ops   <mesh> <L> <seed> <outdir>
//   ref_driver time  <mesh> <sin|lshape> <L> <nu> <reps> [budget_s]
//   ref_driver solvevtd <mesh> <sin|lshape> <L> <nu> <outdir>   (FinestPolicy::ValidationTwoDigits)
//   ref_driver solverve <mesh> <sin|lshape> <L> <nu> <l_direct> <outdir>
//       (FinestPolicy::ResidualVsEstimate; solve_direct(0) and solve_direct(l_direct))
//   ref_driver bounds      (stdin: "theta eps offset" lines -> effectivity_constants,
//                          local spread bounds, make_bounds order; "ERR" on DomainError)
//   ref_driver effidx <file>  (eta, n, eta_local[n], exact global, m, exact per_macro[m]
//                          -> effectivity_index: gamma valid spread valid gamma_local...)
//   ref_driver amr3d <L> <nu> <K> <outdir>
//       BASELINE.json config 4: the unit cube as 6 Kuhn tetrahedra, K steps of
//       (3-d estimate -> marks >= 0.5 max on the green-reverted set ->
//       refine_rg_3d, proj/src/macro_mesh.cpp:662-676).  The reference has no
//       3-d solver: eta_T comes from the builder's 3-d C oracle
//       (klref_oracle3d.c, Gaussian peak problem) on the mesh as written and re-read.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "klref/amr.hpp"
#include "klref/estimator.hpp"
#include "klref/fem.hpp"
#include "klref/hhg.hpp"
#include "klref/macro_mesh.hpp"
#include "klref/mesh_io.hpp"
#include "klref/multigrid.hpp"
#include "klref/problems.hpp"

using namespace klref;

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// splitmix64 -> uniform(-1, 1); mirrored bit-for-bit by tests/_rng.py.
struct SplitMix {
  std::uint64_t s;
  double next() {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    return 2.0 * u - 1.0;
  }
};

MacroMesh cfg1_mesh() {
  // square_grid_mesh pattern, proj/src/problems.cpp:58-70, nx = ny = 2 on [0,1]^2.
  const int nx = 2, ny = 2;
  std::vector<Point> verts;
  std::vector<std::array<Index, 4>> elems;
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) verts.push_back({double(i) / nx, double(j) / ny, 0.0});
  auto at = [&](int i, int j) { return static_cast<Index>(j * (nx + 1) + i); };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      elems.push_back({at(i, j), at(i + 1, j), at(i + 1, j + 1), kNoIndex});
      elems.push_back({at(i, j), at(i + 1, j + 1), at(i, j + 1), kNoIndex});
    }
  return MacroMesh::create(2, verts, elems);
}

MacroMesh cfg2_mesh() {
  // lshape_initial_mesh algorithm (proj/src/problems.cpp:81-109), 1x1 cells per quadrant.
  std::vector<Point> verts{{0, 0, 0}, {1, 0, 0}, {0, 1, 0},   {1, 1, 0},
                           {-1, 0, 0}, {-1, 1, 0}, {-1, -1, 0}, {0, -1, 0}};
  std::vector<std::array<Index, 4>> elems{{0, 1, 3, kNoIndex}, {0, 3, 2, kNoIndex},
                                          {4, 0, 2, kNoIndex}, {4, 2, 5, kNoIndex},
                                          {6, 7, 0, kNoIndex}, {6, 0, 4, kNoIndex}};
  return MacroMesh::create(2, verts, elems);
}

ProblemSpec make_problem(const std::string& name) {
  if (name == "lshape") return make_lshape_spec();
  ProblemSpec p;
  if (name == "sin") {
    // cfg1: u = sin(pi x) sin(pi y), f = 2 pi^2 sin(pi x) sin(pi y), g = u.
    p.name = "sin";
    p.exact = [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
    p.source = [](double x, double y) {
      return 2.0 * M_PI * M_PI * std::sin(M_PI * x) * std::sin(M_PI * y);
    };
    p.boundary = p.exact;
    p.has_exact = true;
    p.domain_volume = 1.0;
    return p;
  }
  if (name == "zero") {
    p.name = "zero";
    p.exact = [](double, double) { return 0.0; };
    p.source = p.exact;
    p.boundary = p.exact;
    return p;
  }
  std::fprintf(stderr, "unknown problem %s\n", name.c_str());
  std::exit(2);
}

void dump(const GridFunction& f, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  for (std::size_t s = 0; s < f.num_macros(); ++s) {
    const auto& m = f.macro(static_cast<int>(s));
    out.write(reinterpret_cast<const char*>(m.data()),
              static_cast<std::streamsize>(m.size() * sizeof(double)));
  }
}

std::string fmt(double x) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", x);
  return buf;
}

std::string join(const std::vector<double>& v) {
  std::string s;
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? " " : "") + fmt(v[i]);
  return s;
}
std::string join_ids(const std::vector<Index>& v) {
  std::string s;
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? " " : "") + std::to_string(v[i]);
  return s;
}

// Indicator aggregation on the green-reverted set, as mark_and_refine
// (proj/src/amr.cpp:41-65) does before marking.
std::pair<MacroMesh, std::vector<double>> reverted_indicator(const MacroMesh& mesh,
                                                             const std::vector<double>& ind) {
  auto [reverted, ignored] = revert_green(mesh, MarkSet{});
  (void)ignored;
  std::map<Index, double> by_id;
  for (std::size_t t = 0; t < mesh.active().size(); ++t) by_id[mesh.active()[t]] = ind[t];
  std::vector<double> agg(reverted.num_active(), 0.0);
  for (std::size_t t = 0; t < reverted.active().size(); ++t) {
    const Index id = reverted.active()[t];
    auto it = by_id.find(id);
    if (it != by_id.end()) {
      agg[t] = it->second;
      continue;
    }
    double sq = 0.0;
    for (Index old_id : mesh.active()) {
      const MacroElement& el = mesh.element(old_id);
      if (el.state == ElementState::GreenChild && el.parent == id) sq += by_id[old_id] * by_id[old_id];
    }
    agg[t] = std::sqrt(sq);
  }
  return {std::move(reverted), std::move(agg)};
}

// Marking rule of BASELINE.json configs 2/4: agg >= 0.5 * max(agg). Not in the
// reference; same reversion/aggregation as above.
MarkSet mark_half_max(const MacroMesh& reverted, const std::vector<double>& agg) {
  double mx = 0.0;
  for (double v : agg) mx = std::max(mx, v);
  MarkSet m;
  for (std::size_t t = 0; t < agg.size(); ++t)
    if (agg[t] >= 0.5 * mx) m.ids.push_back(reverted.active()[t]);
  return m;
}

struct SolveOut {
  std::string report;
  MarkSet marks_top10_eta, marks_halfmax_eta, marks_top10_exact;
  MacroMesh reverted;
};

SolveOut solve_and_report(const MacroMesh& mesh, const ProblemSpec& p, int L, int nu,
                          const std::string& outdir, bool dump_all) {
  SolverConfig sc;
  sc.nu = nu;
  sc.finest_policy = FinestPolicy::None;
  auto h = GridHierarchy::build(mesh, L);
  MultigridSolver solver(h, p, sc);
  FmgState st = solver.fmg();
  std::ostringstream r;
  r << "num_macros " << h->num_macros() << "\n";
  r << "dofs " << h->dof_count(L) << "\n";
  r << "active_ids " << join_ids(mesh.active()) << "\n";
  {
    std::vector<Index> gp;
    for (Index id : mesh.active()) {
      const MacroElement& el = mesh.element(id);
      gp.push_back(el.state == ElementState::GreenChild ? el.parent : kNoIndex);
    }
    r << "active_green_parent " << join_ids(gp) << "\n";
  }
  if (dump_all) {
    for (int l = 0; l <= L; ++l) {
      dump(st.u[l], outdir + "/u_" + std::to_string(l) + ".bin");
      dump(st.b[l], outdir + "/b_" + std::to_string(l) + ".bin");
      if (l < L) dump(st.w[l], outdir + "/w_" + std::to_string(l) + ".bin");
    }
  } else {
    dump(st.u[L], outdir + "/u_" + std::to_string(L) + ".bin");
  }
  SolveOut out;
  for (int j = 1; j <= L - 1; ++j) {
    for (int kind = 0; kind < 2; ++kind) {
      const EstimatorKind ek = kind == 0 ? EstimatorKind::Unscaled : EstimatorKind::Scaled;
      const EstimateReport er = error_estimate(st, j, ek);
      const std::string tag = std::string(kind == 0 ? "u" : "s") + std::to_string(j);
      r << "est_" << tag << " " << fmt(er.norm_base) << " " << fmt(er.norm_coarser) << " "
        << fmt(er.conv_factor) << " " << fmt(er.eta) << "\n";
      r << "eta_local_" << tag << " " << join(er.eta_local) << "\n";
      if (j == 1 && kind == 0) {
        auto [rev, agg] = reverted_indicator(mesh, er.eta_local);
        out.marks_top10_eta = mark_top_fraction(rev, agg, 0.10);
        out.marks_halfmax_eta = mark_half_max(rev, agg);
        r << "agg_eta " << join(agg) << "\n";
        r << "reverted_ids " << join_ids(rev.active()) << "\n";
        out.reverted = rev;
      }
    }
  }
  if (p.has_exact) {
    const ErrorNorms ex = exact_error_norm(p, st.u[L]);
    r << "exact_global " << fmt(ex.global) << "\n";
    r << "exact_local " << join(ex.per_macro) << "\n";
    auto [rev, agg] = reverted_indicator(mesh, ex.per_macro);
    out.marks_top10_exact = mark_top_fraction(rev, agg, 0.10);
  }
  r << "marks_top10_eta " << join_ids(out.marks_top10_eta.ids) << "\n";
  r << "marks_halfmax_eta " << join_ids(out.marks_halfmax_eta.ids) << "\n";
  r << "marks_top10_exact " << join_ids(out.marks_top10_exact.ids) << "\n";
  out.report = r.str();
  return out;
}

void write_text(const std::string& path, const std::string& s) {
  std::ofstream o(path);
  o << s;
}

int cmd_solve(int argc, char** argv) {
  if (argc < 7) return 2;
  const MacroMesh mesh = read_mesh_file(argv[2]);
  const ProblemSpec p = make_problem(argv[3]);
  const int L = std::atoi(argv[4]), nu = std::atoi(argv[5]);
  const std::string outdir = argv[6];
  std::filesystem::create_directories(outdir);
  SolveOut s = solve_and_report(mesh, p, L, nu, outdir, true);
  write_text(outdir + "/report.txt", s.report);
  // one refinement step with the reference default marking (top 10 %)
  MacroMesh refined = refine_rg_2d(s.reverted, s.marks_top10_eta);
  write_mesh_file(refined, outdir + "/refined_top10_eta.mesh");
  return 0;
}

int cmd_amr(int argc, char** argv) {
  if (argc < 9) return 2;
  MacroMesh mesh = read_mesh_file(argv[2]);
  const ProblemSpec p = make_problem(argv[3]);
  const int L = std::atoi(argv[4]), nu = std::atoi(argv[5]), K = std::atoi(argv[6]);
  const std::string rule = argv[7], outdir = argv[8];
  for (int k = 0; k <= K; ++k) {
    const std::string pre = outdir + "/k" + std::to_string(k) + "_";
    std::filesystem::create_directories(outdir + "/k" + std::to_string(k));
    write_mesh_file(mesh, pre + "mesh.txt");
    SolveOut s = solve_and_report(mesh, p, L, nu, outdir + "/k" + std::to_string(k), true);
    write_text(pre + "report.txt", s.report);
    if (k == K) break;
    const MarkSet& m = rule == "halfmax" ? s.marks_halfmax_eta : s.marks_top10_eta;
    mesh = refine_rg_2d(s.reverted, m);
  }
  return 0;
}

extern "C" {
struct o3h;
o3h* o3_build(int nv, const double* xyz, int ne, const int* tet_in, int L);
void o3_free(o3h* h);
int o3_level_size(const o3h* h, int l);
long long o3_dofs(const o3h* h, int l);
int o3_fmg(const o3h* h, int prob, const double* par, int nu, int pre, int post, double rel, double absf, int maxit,
           double** u, double** b, double** w);
int o3_estimate(const o3h* h, const double* uL, double** w, double* out4, double* local_sums);
}

MacroMesh kuhn_unit_cube() {
  std::vector<Point> verts;
  for (int k = 0; k <= 1; ++k)
    for (int j = 0; j <= 1; ++j)
      for (int i = 0; i <= 1; ++i) verts.push_back({double(i), double(j), double(k)});
  auto at = [](int i, int j, int k) { return static_cast<Index>((k * 2 + j) * 2 + i); };
  // the Kuhn subdivision of proj/src/problems.cpp:122-133 on one cube
  static const int perms[6][3][3] = {
      {{1, 0, 0}, {1, 1, 0}, {1, 1, 1}}, {{1, 0, 0}, {1, 0, 1}, {1, 1, 1}},
      {{0, 1, 0}, {1, 1, 0}, {1, 1, 1}}, {{0, 1, 0}, {0, 1, 1}, {1, 1, 1}},
      {{0, 0, 1}, {1, 0, 1}, {1, 1, 1}}, {{0, 0, 1}, {0, 1, 1}, {1, 1, 1}}};
  std::vector<std::array<Index, 4>> elems;
  for (const auto& p : perms)
    elems.push_back({at(0, 0, 0), at(p[0][0], p[0][1], p[0][2]), at(p[1][0], p[1][1], p[1][2]),
                     at(p[2][0], p[2][1], p[2][2])});
  return MacroMesh::create(3, std::move(verts), std::move(elems));
}

int cmd_amr3d(int argc, char** argv) {
  if (argc < 6) return 2;
  const int L = std::atoi(argv[2]), nu = std::atoi(argv[3]), K = std::atoi(argv[4]);
  const std::string outdir = argv[5];
  std::filesystem::create_directories(outdir);
  MacroMesh mesh = kuhn_unit_cube();
  for (int k = 0; k <= K; ++k) {
    const std::string path = outdir + "/cfg4_k" + std::to_string(k) + ".mesh";
    write_mesh_file(mesh, path);
    const MacroMesh fm = read_mesh_file(path);  // the numbering the solvers see
    std::vector<double> xyz;
    for (Index v = 0; v < static_cast<Index>(fm.num_vertices()); ++v)
      for (int a = 0; a < 3; ++a) xyz.push_back(fm.vertex(v).coords[a]);
    std::vector<int> tets;
    for (Index id : fm.active())
      for (int a = 0; a < 4; ++a) tets.push_back(fm.element(id).v[a]);
    o3h* h = o3_build(static_cast<int>(fm.num_vertices()), xyz.data(), static_cast<int>(fm.num_active()),
                      tets.data(), L);
    std::vector<std::vector<double>> U(L + 1), B(L + 1), W(L + 1);
    std::vector<double*> up(L + 1), bp(L + 1), wp(L + 1);
    for (int l = 0; l <= L; ++l) {
      U[l].assign(o3_level_size(h, l), 0.0);
      B[l].assign(o3_level_size(h, l), 0.0);
      up[l] = U[l].data();
      bp[l] = B[l].data();
      if (l < L) {
        W[l].assign(o3_level_size(h, l + 1), 0.0);
        wp[l] = W[l].data();
      }
    }
    const int st = o3_fmg(h, 2 /* gauss */, nullptr, nu, 2, 2, 1e-9, 1e-12, 100000, up.data(), bp.data(), wp.data());
    if (st != 0) throw std::runtime_error("3-d oracle FMG failed");
    double out4[4];
    std::vector<double> sums(2 * fm.num_active());
    o3_estimate(h, up[L], wp.data(), out4, sums.data());
    std::vector<double> eta_local(fm.num_active());
    for (std::size_t t = 0; t < eta_local.size(); ++t) eta_local[t] = std::sqrt(std::max(0.0, sums[2 * t]));
    std::ostringstream r;
    r << "num_macros " << fm.num_active() << "\n";
    r << "dofs " << o3_dofs(h, L) << "\n";
    r << "active_ids " << join_ids(mesh.active()) << "\n";
    {
      std::vector<Index> gp;
      for (Index id : mesh.active()) {
        const MacroElement& el = mesh.element(id);
        gp.push_back(el.state == ElementState::GreenChild ? el.parent : -1);
      }
      r << "green_parent " << join_ids(gp) << "\n";
    }
    r << "eta " << fmt(out4[3]) << "\n";
    r << "norm_base " << fmt(out4[0]) << "\n";
    r << "norm_coarser " << fmt(out4[1]) << "\n";
    r << "eta_local " << join(eta_local) << "\n";
    o3_free(h);
    if (k < K) {
      auto [rev, agg] = reverted_indicator(mesh, eta_local);
      const MarkSet m = mark_half_max(rev, agg);
      r << "reverted_ids " << join_ids(rev.active()) << "\n";
      r << "marks_halfmax_eta " << join_ids(m.ids) << "\n";
      mesh = refine_rg_3d(rev, m);
    }
    write_text(outdir + "/cfg4_k" + std::to_string(k) + "_report.txt", r.str());
    std::fprintf(stderr, "amr3d k=%d: %zu macros, eta %.6e\n", k, fm.num_active(), out4[3]);
  }
  return 0;
}

// FinestPolicy::ValidationTwoDigits (the reference default, multigrid.cpp:282-293)
int cmd_solvevtd(int argc, char** argv) {
  if (argc < 7) return 2;
  const MacroMesh mesh = read_mesh_file(argv[2]);
  const ProblemSpec p = make_problem(argv[3]);
  const int L = std::atoi(argv[4]), nu = std::atoi(argv[5]);
  const std::string outdir = argv[6];
  std::filesystem::create_directories(outdir);
  SolverConfig sc;
  sc.nu = nu;
  sc.finest_policy = FinestPolicy::ValidationTwoDigits;
  auto h = GridHierarchy::build(mesh, L);
  MultigridSolver solver(h, p, sc);
  FmgState st = solver.fmg();
  dump(st.u[L], outdir + "/u_" + std::to_string(L) + ".bin");
  const ErrorNorms ex = st.error_eval ? st.error_eval->evaluate(st.u[L]) : exact_error_norm(p, st.u[L]);
  std::ostringstream r;
  r << "extra_cycles " << st.extra_cycles << "\n";
  r << "exact_global " << fmt(ex.global) << "\n";
  r << "exact_local " << join(ex.per_macro) << "\n";
  write_text(outdir + "/report.txt", r.str());
  return 0;
}

// FinestPolicy::ResidualVsEstimate (proj/src/multigrid.cpp:294-319) and
// MultigridSolver::solve_direct(l) (proj/src/multigrid.cpp:323-357) on the same mesh
int cmd_solverve(int argc, char** argv) {
  if (argc < 8) return 2;
  const MacroMesh mesh = read_mesh_file(argv[2]);
  const ProblemSpec p = make_problem(argv[3]);
  const int L = std::atoi(argv[4]), nu = std::atoi(argv[5]), ld = std::atoi(argv[6]);
  const std::string outdir = argv[7];
  std::filesystem::create_directories(outdir);
  SolverConfig sc;
  sc.nu = nu;
  sc.finest_policy = FinestPolicy::ResidualVsEstimate;
  auto h = GridHierarchy::build(mesh, L);
  MultigridSolver solver(h, p, sc);
  FmgState st = solver.fmg();
  dump(st.u[L], outdir + "/u_" + std::to_string(L) + ".bin");
  for (int l : {0, ld}) dump(solver.solve_direct(l), outdir + "/direct_" + std::to_string(l) + ".bin");
  std::ostringstream r;
  r << "extra_cycles " << st.extra_cycles << "\n";
  write_text(outdir + "/report.txt", r.str());
  return 0;
}

int cmd_ops(int argc, char** argv) {
  if (argc < 6) return 2;
  const MacroMesh mesh = read_mesh_file(argv[2]);
  const int L = std::atoi(argv[3]);
  SplitMix rng{std::strtoull(argv[4], nullptr, 10)};
  const std::string outdir = argv[5];
  std::filesystem::create_directories(outdir);
  auto h = GridHierarchy::build(mesh, L);
  ProblemSpec p = make_problem("zero");
  SolverConfig sc;
  sc.finest_policy = FinestPolicy::None;
  MultigridSolver solver(h, p, sc);
  for (int l = 0; l <= L; ++l) {
    const std::string tag = std::to_string(l);
    auto rand_fn = [&]() {
      GridFunction f = h->create_function(l);
      for (int s = 0; s < h->num_macros(); ++s)
        for (double& v : f.macro(s)) v = rng.next();
      interface_sync(f, SyncMode::ReplaceFromOwner);
      return f;
    };
    GridFunction x = rand_fn(), bb = rand_fn();
    dump(x, outdir + "/x_" + tag + ".bin");
    dump(bb, outdir + "/bb_" + tag + ".bin");
    GridFunction y = h->create_function(l);
    solver.stiffness(l).apply(x, y);
    dump(y, outdir + "/Ax_" + tag + ".bin");
    solver.mass(l).apply(x, y);
    dump(y, outdir + "/Mx_" + tag + ".bin");
    GridFunction r = h->create_function(l);
    solver.residual(l, x, bb, r);
    dump(r, outdir + "/res_" + tag + ".bin");
    {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", dot_unique(x, bb));
      write_text(outdir + "/dot_" + tag + ".txt", buf);
    }
    if (l >= 1) {
      GridFunction u = x;
      solver.gauss_seidel(l, u, bb, 1);
      dump(u, outdir + "/gs1_" + tag + ".bin");
      solver.gauss_seidel(l, u, bb, 1);
      dump(u, outdir + "/gs2_" + tag + ".bin");
      GridFunction rc = restrict_transpose(x);
      dump(rc, outdir + "/restrict_" + tag + ".bin");
    }
    if (l < L) {
      GridFunction pf = prolongate(x);
      dump(pf, outdir + "/prolong_" + tag + ".bin");
    }
    if (l == 0) {
      GridFunction u0 = h->create_function(0);
      GridFunction b0 = bb;
      solver.cg_level0(u0, b0);
      dump(u0, outdir + "/cg0.bin");
    }
  }
  return 0;
}

int cmd_time(int argc, char** argv) {
  if (argc < 7) return 2;
  const MacroMesh mesh = read_mesh_file(argv[2]);
  const ProblemSpec p = make_problem(argv[3]);
  const int L = std::atoi(argv[4]), nu = std::atoi(argv[5]), reps = std::atoi(argv[6]);
  const double budget = argc > 7 ? std::atof(argv[7]) : 1e30;
  SolverConfig sc;
  sc.nu = nu;
  sc.finest_policy = FinestPolicy::None;
  double best_build = 1e30, best_fmg = 1e30, best_est = 1e30, sum_total = 0.0;
  std::vector<double> totals;
  std::int64_t dofs = 0;
  const auto t_start = Clock::now();
  for (int rep = 0; rep <= reps; ++rep) {  // rep 0 is the warm-up
    const auto t0 = Clock::now();
    auto h = GridHierarchy::build(mesh, L);
    MultigridSolver solver(h, p, sc);
    const auto t1 = Clock::now();
    FmgState st = solver.fmg();
    const auto t2 = Clock::now();
    EstimateReport er = error_estimate(st, 1, EstimatorKind::Unscaled);
    const auto t3 = Clock::now();
    (void)er;
    dofs = h->dof_count(L);
    if (rep > 0) {
      best_build = std::min(best_build, secs(t0, t1));
      best_fmg = std::min(best_fmg, secs(t1, t2));
      best_est = std::min(best_est, secs(t2, t3));
      totals.push_back(secs(t0, t3));
      sum_total += secs(t0, t3);
    }
    if (rep > 0 && secs(t_start, Clock::now()) > budget) break;
  }
  std::printf("{\"dofs\": %lld, \"reps\": %zu, \"build_s\": %.9g, \"fmg_s\": %.9g, \"est_s\": %.9g, "
              "\"mean_total_s\": %.9g}\n",
              static_cast<long long>(dofs), totals.size(), best_build, best_fmg, best_est,
              totals.empty() ? 0.0 : sum_total / totals.size());
  return 0;
}

// timeall <sin|lshape|zero> <L> <nu> <steps> <warmup> <mesh>...: one "step" is
// MultigridSolver::fmg() + error_estimate(j=1) on every listed mesh in turn
// (the hot path of the AMR loop, proj/src/amr.cpp:176-213; hierarchy build
// and solver construction happen once, outside the timed region).
int cmd_timeall(int argc, char** argv) {
  if (argc < 8) return 2;
  const ProblemSpec p = make_problem(argv[2]);
  const int L = std::atoi(argv[3]), nu = std::atoi(argv[4]);
  const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
  SolverConfig sc;
  sc.nu = nu;
  sc.finest_policy = FinestPolicy::None;
  std::vector<std::shared_ptr<const GridHierarchy>> hs;
  std::vector<std::unique_ptr<MultigridSolver>> solvers;
  std::int64_t dofs = 0;
  for (int a = 7; a < argc; ++a) {
    hs.push_back(GridHierarchy::build(read_mesh_file(argv[a]), L));
    solvers.push_back(std::make_unique<MultigridSolver>(hs.back(), p, sc));
    dofs += hs.back()->dof_count(L);
  }
  std::vector<double> times;
  double fmg_s = 0.0, est_s = 0.0;
  for (int it = 0; it < warmup + steps; ++it) {
    double f = 0.0, e = 0.0;
    for (auto& s : solvers) {
      const auto t0 = Clock::now();
      FmgState st = s->fmg();
      const auto t1 = Clock::now();
      EstimateReport er = error_estimate(st, 1, EstimatorKind::Unscaled);
      const auto t2 = Clock::now();
      (void)er;
      f += secs(t0, t1);
      e += secs(t1, t2);
    }
    if (it >= warmup) {
      times.push_back(f + e);
      fmg_s += f;
      est_s += e;
    }
  }
  std::printf("{\"dofs_per_step\": %lld, \"steps\": %d, \"fmg_s\": %.9g, \"est_s\": %.9g, \"step_s\": [",
              static_cast<long long>(dofs), steps, fmg_s, est_s);
  for (size_t i = 0; i < times.size(); ++i) std::printf("%s%.9g", i ? ", " : "", times[i]);
  std::printf("]}\n");
  return 0;
}

// effectivity constants / spread bounds (proj/src/estimator.cpp:47-99) for
// the (theta, eps, offset) triples on stdin
int cmd_bounds() {
  double theta = 0.0, eps = 0.0;
  int offset = 0;
  while (std::scanf("%lf %lf %d", &theta, &eps, &offset) == 3) {
    try {
      const BoundsConstants b = make_bounds(theta, eps, offset);
      std::printf("%.17g %.17g %.17g %.17g %d\n", b.equivalence.lower, b.equivalence.upper, b.spread_scaled,
                  b.spread_unscaled, b.order);
    } catch (const DomainError&) {
      std::printf("ERR\n");
    }
  }
  return 0;
}

// effectivity_index (proj/src/estimator.cpp:100-123) of the report in <file>
int cmd_effidx(int argc, char** argv) {
  if (argc < 3) return 2;
  std::ifstream in(argv[2]);
  EstimateReport r;
  ErrorNorms ex;
  int n = 0, m = 0;
  in >> r.eta >> n;
  r.eta_local.resize(n);
  for (auto& v : r.eta_local) in >> v;
  in >> ex.global >> m;
  ex.per_macro.resize(m);
  for (auto& v : ex.per_macro) in >> v;
  const EffectivityReport e = effectivity_index(r, ex);
  std::printf("%.17g %d %.17g %d", e.gamma, e.gamma_valid ? 1 : 0, e.spread, e.spread_valid ? 1 : 0);
  for (double g : e.gamma_local) std::printf(" %.17g", g);
  std::printf("\n");
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver mesh|solve|amr|ops|time ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "mesh") {
      if (argc < 4) return 2;
      const std::string which = argv[2];
      const MacroMesh m = which == "cfg1" ? cfg1_mesh() : cfg2_mesh();
      write_mesh_file(m, argv[3]);
      return 0;
    }
    if (cmd == "solve") return cmd_solve(argc, argv);
    if (cmd == "amr") return cmd_amr(argc, argv);
    if (cmd == "solverve") return cmd_solverve(argc, argv);
    if (cmd == "ops") return cmd_ops(argc, argv);
    if (cmd == "amr3d") return cmd_amr3d(argc, argv);
    if (cmd == "solvevtd") return cmd_solvevtd(argc, argv);
    if (cmd == "time") return cmd_time(argc, argv);
    if (cmd == "timeall") return cmd_timeall(argc, argv);
    if (cmd == "bounds") return cmd_bounds();
    if (cmd == "effidx") return cmd_effidx(argc, argv);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
