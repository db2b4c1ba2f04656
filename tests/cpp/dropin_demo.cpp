// Drop-in demo / GPU test of the C++ facade include/klref_b200/klref.hpp:
// the reference's own call sequence of run_kl (proj/src/amr.cpp:176-213) --
// GridHierarchy::build, MultigridSolver(h, p, cfg), fmg(), error_estimate --
// against a mesh type exposing the reference MacroMesh accessors.
//
//   dropin_demo <mesh file> <sin|lshape> <L> <nu> <u_L output .bin>
// prints one JSON line {dofs, eta, norm_base, norm_coarser, conv, eta_local}.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "klref_b200/klref.hpp"

namespace {

// Minimal stand-in with the accessors of the reference MacroMesh
// (proj/include/klref/macro_mesh.hpp:64-79) read from the mesh_io format.
struct DemoMesh {
  struct V {
    std::array<double, 3> coords{0, 0, 0};
  };
  struct E {
    std::array<std::int32_t, 4> v{-1, -1, -1, -1};
  };
  int d = 2;
  std::vector<V> verts;
  std::vector<E> elems;
  std::vector<std::int32_t> act;
  int dim() const { return d; }
  std::size_t num_vertices() const { return verts.size(); }
  const V& vertex(std::int32_t id) const { return verts.at(static_cast<std::size_t>(id)); }
  const E& element(std::int32_t id) const { return elems.at(static_cast<std::size_t>(id)); }
  const std::vector<std::int32_t>& active() const { return act; }
};

DemoMesh read_mesh(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw klref::IoError("cannot open " + path);
  std::vector<std::string> lines;
  for (std::string ln; std::getline(in, ln);)
    if (!ln.empty() && ln[0] != '#') lines.push_back(ln);
  DemoMesh m;
  std::size_t p = 0;
  std::string tag;
  std::istringstream(lines[p++]) >> tag >> m.d;
  int nv = 0, ne = 0;
  std::istringstream(lines[p++]) >> tag >> nv;
  m.verts.resize(nv);
  for (int v = 0; v < nv; ++v) {
    std::istringstream s(lines[p++]);
    int id;
    s >> id;
    for (int c = 0; c < m.d; ++c) s >> m.verts[id].coords[c];
  }
  std::istringstream(lines[p++]) >> tag >> ne;
  m.elems.resize(ne);
  for (int e = 0; e < ne; ++e) {
    std::istringstream s(lines[p++]);
    int id;
    s >> id;
    for (int c = 0; c <= m.d; ++c) s >> m.elems[id].v[c];
    m.act.push_back(id);
  }
  return m;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: dropin_demo <mesh> <sin|lshape> <L> <nu> <out.bin>\n");
    return 2;
  }
  try {
    const DemoMesh mesh = read_mesh(argv[1]);
    const std::string prob = argv[2];
    const int L = std::atoi(argv[3]), nu = std::atoi(argv[4]);
    klref::ProblemSpec p;
    if (prob == "sin") {  // BASELINE.json config 1
      p.exact = [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
      p.source = [](double x, double y) { return 2.0 * M_PI * M_PI * std::sin(M_PI * x) * std::sin(M_PI * y); };
    } else {  // make_lshape_spec, proj/src/problems.cpp:36-53
      p.exact = [](double x, double y) {
        const double r = std::hypot(x, y);
        if (r == 0.0) return 0.0;
        double phi = std::atan2(y, x);
        if (phi < 0.0) phi += 2.0 * M_PI;
        return std::pow(r, 2.0 / 3.0) * std::sin(2.0 * phi / 3.0);
      };
      p.source = [](double, double) { return 0.0; };
    }
    p.boundary = p.exact;
    klref::SolverConfig cfg;
    cfg.nu = nu;
    cfg.finest_policy = klref::FinestPolicy::None;
    // run_kl's per-iteration sequence, proj/src/amr.cpp:176-201
    auto h = klref::GridHierarchy::build(mesh, L);
    klref::MultigridSolver solver(h, p, cfg);
    klref::FmgState st = solver.fmg();
    const klref::EstimateReport er = klref::error_estimate(st, 1, klref::EstimatorKind::Unscaled);
    // validation rows of run_kl, proj/src/amr.cpp:188-204: exact error and effectivity
    const klref::ErrorNorms exact = klref::exact_error_norm(p, st.u.back());
    const klref::EffectivityReport eff = klref::effectivity_index(er, exact);
    const klref::BoundsConstants bounds = klref::make_bounds_from_order(2, 0.0, 1);
    const klref::GridFunction uL = st.u.back();
    const std::vector<double> flat = uL.flat();
    std::FILE* f = std::fopen(argv[5], "wb");
    if (!f) throw klref::IoError("cannot write output");
    std::fwrite(flat.data(), sizeof(double), flat.size(), f);
    std::fclose(f);
    std::printf("{\"dofs\": %lld, \"eta\": %.17g, \"norm_base\": %.17g, \"norm_coarser\": %.17g, \"conv\": %.17g, "
                "\"exact\": %.17g, \"gamma\": %.17g, \"spread\": %.17g, \"c1\": %.17g, \"c2\": %.17g, "
                "\"eta_local\": [",
                static_cast<long long>(h->dof_count(L)), er.eta, er.norm_base, er.norm_coarser, er.conv_factor,
                exact.global, eff.gamma, eff.spread, bounds.equivalence.lower, bounds.equivalence.upper);
    for (std::size_t s = 0; s < er.eta_local.size(); ++s) std::printf("%s%.17g", s ? ", " : "", er.eta_local[s]);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "dropin_demo: %s\n", e.what());
    return 1;
  }
  return 0;
}
