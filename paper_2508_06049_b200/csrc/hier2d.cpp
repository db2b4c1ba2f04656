// Host-side construction of the 2-d HHG tables.  See hier2d.hpp.
#include "hier2d.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <new>

namespace kb {
namespace {

constexpr int kLocalEdges[3][2] = {{0, 1}, {0, 2}, {1, 2}};

double signed_area(double ax, double ay, double bx, double by, double cx, double cy) {
  return 0.5 * ((bx - ax) * (cy - ay) - (by - ay) * (cx - ax));
}

// P1 stiffness on one micro triangle; D1 fix: |area| (proj/src/fem.cpp:30-41).
std::array<double, 9> stiffness_matrix(double p0x, double p0y, double p1x, double p1y, double p2x,
                                       double p2y) {
  const double area2 = (p1x - p0x) * (p2y - p0y) - (p1y - p0y) * (p2x - p0x);
  const double area = 0.5 * std::fabs(area2);
  const double gx[3] = {-(p2y - p1y) / area2, -(p0y - p2y) / area2, -(p1y - p0y) / area2};
  const double gy[3] = {(p2x - p1x) / area2, (p0x - p2x) / area2, (p1x - p0x) / area2};
  std::array<double, 9> k{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) k[3 * i + j] = area * (gx[i] * gx[j] + gy[i] * gy[j]);
  return k;
}

std::array<double, 9> mass_matrix(double area) {
  const double d = area / 6.0, o = area / 12.0;
  return {d, o, o, o, d, o, o, o, d};
}

int edge_lattice_index(int n, int le, int t) {
  switch (le) {
    case 0: return lattice_index(n, t, 0);
    case 1: return lattice_index(n, 0, t);
    default: return lattice_index(n, n - t, t);
  }
}

int direction_code(int di, int dj) {
  if (di == 1 && dj == 0) return 0;    // E
  if (di == -1 && dj == 0) return 1;   // W
  if (di == 0 && dj == 1) return 2;    // N
  if (di == 0 && dj == -1) return 3;   // S
  if (di == -1 && dj == 1) return 4;   // NW
  if (di == 1 && dj == -1) return 5;   // SE
  return -1;
}

bool on_lattice_boundary(int n, int i, int j) { return i == 0 || j == 0 || i + j == n; }

std::uint64_t pack32(std::int32_t lo, std::int32_t hi) {
  return static_cast<std::uint64_t>(static_cast<std::uint32_t>(lo)) |
         (static_cast<std::uint64_t>(static_cast<std::uint32_t>(hi)) << 32);
}
std::uint64_t pack16(std::int16_t a, std::int16_t b, std::int16_t c, std::int16_t d) {
  return static_cast<std::uint64_t>(static_cast<std::uint16_t>(a)) |
         (static_cast<std::uint64_t>(static_cast<std::uint16_t>(b)) << 16) |
         (static_cast<std::uint64_t>(static_cast<std::uint16_t>(c)) << 32) |
         (static_cast<std::uint64_t>(static_cast<std::uint16_t>(d)) << 48);
}

std::uint64_t dbits(double d) {
  std::uint64_t w;
  std::memcpy(&w, &d, 8);
  return w;
}

// One pre-decoded lane record (layout in hier2d.hpp, kProgLaneWords): the
// compact partial_row of member `rec` (may be null: no record) of node k.
void put_lane(std::uint64_t* w, const MemberRec* rec, const Level2D& lvl, int k, int flags, int wr0, int wr1,
              int wb, int wc, int xb, double diag, double inv) {
  // absent cells / members: zero coefficients reading the zero ghost slot
  // (index max_ghosts), so the partial-row chain needs no selects
  const int zero = -1 - lvl.max_ghosts;
  double c[6] = {0, 0, 0, 0, 0, 0};
  int loc[6] = {zero, zero, zero, zero, zero, zero};
  int nc = 0;
  if (rec) {
    const double* ku = &lvl.kstiff[18 * static_cast<std::size_t>(rec->slot)];
    static const int ci[12] = {1, 2, 3, 5, 6, 7, 10, 11, 12, 14, 15, 16};
    for (int cell = 0; cell < 6; ++cell) {
      if (!((rec->mask >> cell) & 1)) continue;
      if (nc == 3) fail(KB_INTERNAL, "boundary node with more than three cells in one macro");
      for (int q = 0; q < 2; ++q) {
        c[2 * nc + q] = ku[ci[2 * cell + q]];
        loc[2 * nc + q] = rec->loc[2 * cell + q];
      }
      ++nc;
    }
  }
  for (int q = 0; q < 6; ++q) w[q] = dbits(c[q]);
  w[6] = dbits(diag);
  w[7] = dbits(inv);
  w[8] = pack32(loc[0], loc[1]);
  w[9] = pack32(loc[2], loc[3]);
  w[10] = pack32(loc[4], loc[5]);
  w[11] = pack32(k, flags);
  w[12] = pack32(wr0, wr1);
  w[13] = pack32(wb, wc);
  // the same reads as slots of the concatenated [ghosts | lattice] shared-memory
  // region of k_gs_pipe / k_gs_macro (ghost g -> g, lattice index l -> G + 1 + l)
  std::uint16_t a[6];
  for (int q = 0; q < 6; ++q) {
    const long long v = loc[q] >= 0 ? lvl.max_ghosts + 1LL + loc[q] : -1LL - loc[q];
    if (v < 0 || v > 0xffff) fail(KB_INTERNAL, "step-program slot does not fit 16 bits");
    a[q] = static_cast<std::uint16_t>(v);
  }
  w[14] = pack32(xb, static_cast<int>(a[4] | (static_cast<unsigned>(a[5]) << 16)));
  w[15] = static_cast<std::uint64_t>(a[0]) | (static_cast<std::uint64_t>(a[1]) << 16) |
          (static_cast<std::uint64_t>(a[2]) << 32) | (static_cast<std::uint64_t>(a[3]) << 48);
  (void)nc;
}

// Step programs (layout in hier2d.hpp, Level2D::prog).
void build_programs(Level2D& lvl, int M) {
  const int n = lvl.n;
  const std::size_t per_macro = static_cast<std::size_t>(2 * n + 1) * kProgStepWords;
  lvl.prog.assign(per_macro * M, 0);
  lvl.prog_ptr.assign(M, 0);
  lvl.prog_extra.clear();
  lvl.xtra_ptr.assign(M + 1, 0);
  lvl.max_extra = 0;
  for (int m = 0; m < M; ++m) {
    lvl.prog_ptr[m] = static_cast<long long>(per_macro * m);
    int nextra = 0;
    for (int t = 0; t <= 2 * n; ++t) {
      int ti[3], tj[3];
      bool big = false;
      for (int type = 0; type < 3; ++type) {
        ti[type] = tj[type] = -1;
        if (type == 0 && t <= n) {
          ti[type] = t;
          tj[type] = 0;
        } else if (type == 1 && !(t & 1) && t >= 2) {
          ti[type] = 0;
          tj[type] = t / 2;
        } else if (type == 2 && t > n && t < 2 * n) {
          tj[type] = t - n;
          ti[type] = n - tj[type];
        }
        if (ti[type] >= 0) {
          const BNode& bn = lvl.bnode[static_cast<std::size_t>(m) * 3 * n + bpos(n, ti[type], tj[type])];
          big = big || (!bn.domain && bn.rec_count > 2);
        }
      }
      for (int type = 0; type < 3; ++type) {
        std::uint64_t* w = &lvl.prog[per_macro * m + static_cast<std::size_t>(t) * kProgStepWords +
                                     static_cast<std::size_t>(2 * type) * kProgLaneWords];
        const int i = ti[type], j = tj[type];
        if (i < 0) {
          for (int mem = 0; mem < 2; ++mem)
            put_lane(w + mem * kProgLaneWords, nullptr, lvl, -1, big ? 1 << 16 : 0, 0, 0, 0, 0, 0, 1.0, 1.0);
          continue;
        }
        const BNode& bn = lvl.bnode[static_cast<std::size_t>(m) * 3 * n + bpos(n, i, j)];
        const int k = lattice_index(n, i, j);
        const int rc = bn.domain ? 0 : bn.rec_count;
        // flags: bit 0 domain boundary, bits 8..15 member count, bit 16 a vertex group of > 2 members this step
        const int flags = (bn.domain ? 1 : 0) | (rc << 8) | (big ? 1 << 16 : 0);
        const int wr0 = bn.wr_count > 0 ? lvl.wr[bn.wr_begin] : 0;
        const int wr1 = bn.wr_count > 1 ? lvl.wr[bn.wr_begin + 1] : 0;
        const double inv = bn.diag != 0.0 ? 1.0 / bn.diag : 0.0;
        for (int mem = 0; mem < 2; ++mem)
          put_lane(w + mem * kProgLaneWords, mem < rc ? &lvl.rec[bn.rec_begin + mem] : nullptr, lvl, k, flags, wr0,
                   wr1, bn.wr_begin, bn.wr_count, nextra, bn.diag, inv);
        for (int r = 2; r < rc; ++r) {
          std::uint64_t x[kProgLaneWords];
          put_lane(x, &lvl.rec[bn.rec_begin + r], lvl, k, flags, wr0, wr1, bn.wr_begin, bn.wr_count, nextra, bn.diag,
                   inv);
          lvl.prog_extra.insert(lvl.prog_extra.end(), x, x + kProgLaneWords);
        }
        nextra += std::max(0, rc - 2);
      }
    }
    lvl.xtra_ptr[m + 1] = static_cast<int>(lvl.prog_extra.size());
    lvl.max_extra = std::max(lvl.max_extra, nextra);
  }
}

}  // namespace

Mesh2D Mesh2D::create(int nv, const double* xy, int ne, const int* tri3) {
  if (nv <= 0 || ne <= 0) fail(KB_STRUCTURAL, "mesh has no vertices or no elements");
  Mesh2D m;
  m.x.resize(nv);
  m.y.resize(nv);
  for (int v = 0; v < nv; ++v) {
    m.x[v] = xy[2 * v];
    m.y[v] = xy[2 * v + 1];
    if (!std::isfinite(m.x[v]) || !std::isfinite(m.y[v]))
      fail(KB_STRUCTURAL, "vertex coordinates must be finite");
  }
  m.tri.resize(ne);
  m.area.resize(ne);
  std::map<std::pair<int, int>, int> edge_count;
  for (int e = 0; e < ne; ++e) {
    std::array<int, 3> v{tri3[3 * e], tri3[3 * e + 1], tri3[3 * e + 2]};
    for (int k = 0; k < 3; ++k)
      if (v[k] < 0 || v[k] >= nv) fail(KB_STRUCTURAL, "element references unknown vertex");
    if (v[0] == v[1] || v[0] == v[2] || v[1] == v[2])
      fail(KB_STRUCTURAL, "element vertices must be distinct");
    // orient_positive, proj/src/macro_mesh.cpp:206-210
    if (signed_area(m.x[v[0]], m.y[v[0]], m.x[v[1]], m.y[v[1]], m.x[v[2]], m.y[v[2]]) < 0.0)
      std::swap(v[1], v[2]);
    m.tri[e] = v;
    m.area[e] = signed_area(m.x[v[0]], m.y[v[0]], m.x[v[1]], m.y[v[1]], m.x[v[2]], m.y[v[2]]);
    if (!(m.area[e] > 0.0)) fail(KB_STRUCTURAL, "degenerate element in input");
    for (const auto& le : kLocalEdges) {
      const int a = v[le[0]], b = v[le[1]];
      edge_count[{std::min(a, b), std::max(a, b)}]++;
    }
  }
  m.boundary.assign(nv, 0);
  for (const auto& [k, c] : edge_count) {
    if (c > 2) fail(KB_STRUCTURAL, "edge shared by more than two elements");
    if (c == 1) m.boundary[k.first] = m.boundary[k.second] = 1;
  }
  return m;
}

int Hierarchy2D::boundary_group(int slot, int l, int i, int j) const {
  const Level2D& lvl = levels[l];
  const int n = lvl.n;
  const MacroLevel& ml = lvl.macros[slot];
  const auto& ids = mesh.tri[slot];
  if (i == 0 && j == 0) return ml.corner_group[0];
  if (i == n && j == 0) return ml.corner_group[1];
  if (i == 0 && j == n) return ml.corner_group[2];
  // D2 fix: the group index counts from the edge's lower-id corner.
  auto pos = [&](int le, int t) { return ids[kLocalEdges[le][0]] < ids[kLocalEdges[le][1]] ? t : n - t; };
  if (j == 0) return ml.edge[0].group_start + (pos(0, i) - 1);
  if (i == 0) return ml.edge[1].group_start + (pos(1, j) - 1);
  if (i + j == n) return ml.edge[2].group_start + (pos(2, j) - 1);
  fail(KB_STRUCTURAL, "node is not on the lattice boundary");
}

bool Hierarchy2D::on_domain_boundary(int slot, int l, int i, int j) const {
  const Level2D& lvl = levels[l];
  const int n = lvl.n;
  const MacroLevel& ml = lvl.macros[slot];
  if (i == 0 && j == 0) return ml.corner_boundary[0];
  if (i == n && j == 0) return ml.corner_boundary[1];
  if (i == 0 && j == n) return ml.corner_boundary[2];
  if (j == 0) return ml.edge[0].domain_boundary;
  if (i == 0) return ml.edge[1].domain_boundary;
  if (i + j == n) return ml.edge[2].domain_boundary;
  return false;
}

bool Hierarchy2D::owns_boundary_node(int slot, int l, int i, int j) const {
  const Level2D& lvl = levels[l];
  const int n = lvl.n;
  const MacroLevel& ml = lvl.macros[slot];
  if (i == 0 && j == 0) return ml.corner_owner[0];
  if (i == n && j == 0) return ml.corner_owner[1];
  if (i == 0 && j == n) return ml.corner_owner[2];
  if (j == 0) return ml.edge[0].owner;
  if (i == 0) return ml.edge[1].owner;
  if (i + j == n) return ml.edge[2].owner;
  return true;
}

void Hierarchy2D::node_coordinates(int slot, int l, int i, int j, double& x, double& y) const {
  const int n = levels[l].n;
  const auto& v = mesh.tri[slot];
  const double xi = static_cast<double>(i) / n;
  const double yj = static_cast<double>(j) / n;
  x = mesh.x[v[0]] + xi * (mesh.x[v[1]] - mesh.x[v[0]]) + yj * (mesh.x[v[2]] - mesh.x[v[0]]);
  y = mesh.y[v[0]] + xi * (mesh.y[v[1]] - mesh.y[v[0]]) + yj * (mesh.y[v[2]] - mesh.y[v[0]]);
}

Hierarchy2D Hierarchy2D::build(const Mesh2D& mesh, int max_level) {
  const auto tb = std::chrono::steady_clock::now();
  if (max_level < 0) fail(KB_STRUCTURAL, "hierarchy level must be nonnegative");
  if (max_level > 9) fail(KB_STRUCTURAL, "2-d wavefront smoother supports levels <= 9");
  Hierarchy2D h;
  h.mesh = mesh;
  h.L = max_level;
  h.M = static_cast<int>(mesh.tri.size());
  const int M = h.M;

  // Global vertex and edge incidence ordered by vertex id / edge key
  // (proj/src/hhg.cpp:73-83).
  std::map<int, std::vector<std::pair<int, int>>> vertex_use;
  std::map<std::pair<int, int>, std::vector<std::pair<int, int>>> edge_use;
  for (int s = 0; s < M; ++s) {
    const auto& ids = mesh.tri[s];
    for (int c = 0; c < 3; ++c) vertex_use[ids[c]].push_back({s, c});
    for (int le = 0; le < 3; ++le) {
      const int a = ids[kLocalEdges[le][0]], b = ids[kLocalEdges[le][1]];
      edge_use[{std::min(a, b), std::max(a, b)}].push_back({s, le});
    }
  }
  for (const auto& [k, uses] : edge_use)
    if (uses.size() > 2) fail(KB_STRUCTURAL, "hierarchy requires a conforming macro mesh");

  // Vertex-sharing neighbours and the Gauss-Seidel dependency depth
  // (SURVEY.md Appendix A.3).
  {
    std::vector<std::vector<int>> nb(M);
    for (const auto& [vid, uses] : vertex_use)
      for (const auto& a : uses)
        for (const auto& b : uses)
          if (a.first != b.first) nb[a.first].push_back(b.first);
    h.nb_lo_ptr.assign(1, 0);
    h.nb_hi_ptr.assign(1, 0);
    std::vector<int> depth(M, 0);
    for (int s = 0; s < M; ++s) {
      auto& v = nb[s];
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      int d = 0;
      for (int o : v) {
        if (o < s) {
          h.nb_lo.push_back(o);
          d = std::max(d, depth[o]);
        } else {
          h.nb_hi.push_back(o);
        }
      }
      depth[s] = d + 1;
      h.dag_depth = std::max(h.dag_depth, depth[s]);
      h.nb_lo_ptr.push_back(static_cast<int>(h.nb_lo.size()));
      h.nb_hi_ptr.push_back(static_cast<int>(h.nb_hi.size()));
    }
    h.dag_ptr.assign(h.dag_depth + 1, 0);
    for (int s = 0; s < M; ++s) ++h.dag_ptr[depth[s]];
    for (int d = 1; d <= h.dag_depth; ++d) h.dag_ptr[d] += h.dag_ptr[d - 1];
    h.dag_list.assign(M, 0);
    std::vector<int> fill(h.dag_ptr.begin(), h.dag_ptr.end() - 1);
    for (int s = 0; s < M; ++s) h.dag_list[fill[depth[s] - 1]++] = s;
  }

  try {
    for (int l = 0; l <= max_level; ++l) {
      Level2D lvl;
      lvl.n = 1 << l;
      const int n = lvl.n;
      lvl.S = lattice_size(n);
      const int S = lvl.S;
      lvl.macros.resize(M);
      lvl.grp_ptr.push_back(0);
      const int corner_idx[3] = {lattice_index(n, 0, 0), lattice_index(n, n, 0), lattice_index(n, 0, n)};
      const int corner_ij[3][2] = {{0, 0}, {n, 0}, {0, n}};
      auto push_member = [&](int s, int idx, int i, int j) {
        lvl.mem_slot.push_back(s);
        lvl.mem_idx.push_back(idx);
        lvl.mem_i.push_back(i);
        lvl.mem_j.push_back(j);
      };
      // vertex groups (proj/src/hhg.cpp:95-109)
      for (const auto& [vid, uses] : vertex_use) {
        const int gid = static_cast<int>(lvl.grp_ptr.size()) - 1;
        for (const auto& [s, c] : uses) {
          push_member(s, corner_idx[c], corner_ij[c][0], corner_ij[c][1]);
          lvl.macros[s].corner_group[c] = gid;
          lvl.macros[s].corner_boundary[c] = mesh.boundary[vid] != 0;
        }
        lvl.macros[uses.front().first].corner_owner[uses.front().second] = true;
        lvl.grp_ptr.push_back(static_cast<int>(lvl.mem_slot.size()));
      }
      // edge groups (proj/src/hhg.cpp:111-132)
      for (const auto& [key, uses] : edge_use) {
        const bool bnd = uses.size() == 1;
        const int group_start = static_cast<int>(lvl.grp_ptr.size()) - 1;
        for (int s = 1; s <= n - 1; ++s) {
          for (const auto& [slot, le] : uses) {
            const int first = mesh.tri[slot][kLocalEdges[le][0]];
            const int t = (first == key.first) ? s : n - s;
            const int ii = le == 0 ? t : (le == 1 ? 0 : n - t);
            const int jj = le == 0 ? 0 : t;
            push_member(slot, edge_lattice_index(n, le, t), ii, jj);
          }
          lvl.grp_ptr.push_back(static_cast<int>(lvl.mem_slot.size()));
        }
        for (const auto& [slot, le] : uses) {
          auto& info = lvl.macros[slot].edge[le];
          info.group_start = group_start;
          info.owner = (slot == uses.front().first && le == uses.front().second);
          info.domain_boundary = bnd;
        }
      }
      const std::int64_t interior = static_cast<std::int64_t>(n - 1) * (n - 2) / 2;
      lvl.dofs = static_cast<std::int64_t>(vertex_use.size()) +
                 static_cast<std::int64_t>(edge_use.size()) * (n - 1) +
                 static_cast<std::int64_t>(M) * interior;
      h.levels.push_back(std::move(lvl));
    }
  } catch (const std::bad_alloc&) {
    Error e(KB_RESOURCE, "out of memory while building hierarchy level");
    e.level = static_cast<int>(h.levels.size());
    throw e;
  }

  // Derived tables: the levels are independent, one host thread each.
  auto derive = [&](int l) {
    Level2D& lvl = h.levels[l];
    const auto tl0 = std::chrono::steady_clock::now();
    const int n = lvl.n, S = lvl.S;
    lvl.node_gid.assign(static_cast<std::size_t>(M) * S, -1);
    lvl.node_flags.assign(static_cast<std::size_t>(M) * S, 4);  // interior: owner
    for (int s = 0; s < M; ++s) {
      for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n - j; ++i) {
          if (!on_lattice_boundary(n, i, j)) continue;
          const std::size_t k = static_cast<std::size_t>(s) * S + lattice_index(n, i, j);
          lvl.node_gid[k] = h.boundary_group(s, l, i, j);
          std::uint8_t f = 1;
          if (h.on_domain_boundary(s, l, i, j)) f |= 2;
          if (h.owns_boundary_node(s, l, i, j)) f |= 4;
          lvl.node_flags[k] = f;
        }
    }
    // element matrices and stencils (proj/src/fem.cpp:62-93)
    lvl.kstiff.assign(static_cast<std::size_t>(M) * 18, 0.0);
    lvl.kmass.assign(static_cast<std::size_t>(M) * 18, 0.0);
    lvl.stencil.assign(static_cast<std::size_t>(M) * 7, 0.0);
    lvl.inv_c.assign(M, 0.0);
    for (int s = 0; s < M; ++s) {
      double p[3][2];
      const int cij[3][2] = {{0, 0}, {1, 0}, {0, 1}};
      for (int c = 0; c < 3; ++c) h.node_coordinates(s, l, cij[c][0], cij[c][1], p[c][0], p[c][1]);
      const auto up = stiffness_matrix(p[0][0], p[0][1], p[1][0], p[1][1], p[2][0], p[2][1]);
      std::array<double, 9> down{};
      if (n >= 2) {
        double q[3][2];
        const int dij[3][2] = {{1, 0}, {0, 1}, {1, 1}};
        for (int c = 0; c < 3; ++c) h.node_coordinates(s, l, dij[c][0], dij[c][1], q[c][0], q[c][1]);
        down = stiffness_matrix(q[0][0], q[0][1], q[1][0], q[1][1], q[2][0], q[2][1]);
      }
      const double cell_area = mesh.area[s] / (static_cast<double>(n) * n);
      const auto mu = mass_matrix(cell_area);
      const auto md = n >= 2 ? mass_matrix(cell_area) : std::array<double, 9>{};
      for (int k = 0; k < 9; ++k) {
        lvl.kstiff[18 * s + k] = up[k];
        lvl.kstiff[18 * s + 9 + k] = down[k];
        lvl.kmass[18 * s + k] = mu[k];
        lvl.kmass[18 * s + 9 + k] = md[k];
      }
      const auto& ku = up;
      const auto& kd = down;
      double* st = &lvl.stencil[7 * s];
      st[0] = ku[0] + ku[4] + ku[8] + kd[0] + kd[4] + kd[8];
      st[1] = ku[1] + kd[5];
      st[2] = ku[3] + kd[7];
      st[3] = ku[2] + kd[2];
      st[4] = ku[6] + kd[6];
      st[5] = ku[5] + kd[1];
      st[6] = ku[7] + kd[3];
      lvl.inv_c[s] = 1.0 / st[0];
    }
    // owner dot order (proj/src/hhg.cpp:233-255)
    for (int s = 0; s < M; ++s) {
      const std::size_t base = static_cast<std::size_t>(s) * S;
      for (int j = 1; j < n; ++j)
        for (int i = 1; i < n - j; ++i) lvl.dot_order.push_back(static_cast<int>(base + lattice_index(n, i, j)));
      const MacroLevel& ml = lvl.macros[s];
      const int corner_idx[3] = {lattice_index(n, 0, 0), lattice_index(n, n, 0), lattice_index(n, 0, n)};
      for (int c = 0; c < 3; ++c)
        if (ml.corner_owner[c]) lvl.dot_order.push_back(static_cast<int>(base + corner_idx[c]));
      for (int le = 0; le < 3; ++le) {
        if (!ml.edge[le].owner) continue;
        for (int t = 1; t <= n - 1; ++t) lvl.dot_order.push_back(static_cast<int>(base + edge_lattice_index(n, le, t)));
      }
    }
    if (l == 0) return;

    // Wavefront Gauss-Seidel tables.
    lvl.bnode.assign(static_cast<std::size_t>(M) * 3 * n, BNode{});
    lvl.ghost_ptr.assign(1, 0);
    for (int m = 0; m < M; ++m) {
      std::map<int, int> ghost_of;
      std::vector<int> ghosts;
      auto visit = [&](int i, int j) {
        BNode bn{};
        const int gid = h.boundary_group(m, l, i, j);
        const int own_off = m * S + lattice_index(n, i, j);
        bn.domain = h.on_domain_boundary(m, l, i, j) ? 1 : 0;
        bn.wr_begin = static_cast<int>(lvl.wr.size());
        for (int k = lvl.grp_ptr[gid]; k < lvl.grp_ptr[gid + 1]; ++k) {
          const int off = lvl.mem_slot[k] * S + lvl.mem_idx[k];
          if (off != own_off) lvl.wr.push_back(off);
        }
        bn.wr_count = static_cast<int>(lvl.wr.size()) - bn.wr_begin;
        bn.rec_begin = static_cast<int>(lvl.rec.size());
        double diag = 0.0;
        if (!bn.domain) {
          for (int k = lvl.grp_ptr[gid]; k < lvl.grp_ptr[gid + 1]; ++k) {
            const int sp = lvl.mem_slot[k], ip = lvl.mem_i[k], jp = lvl.mem_j[k];
            const double* ku = &lvl.kstiff[18 * sp];
            const double* kd = ku + 9;
            MemberRec r{};
            r.slot = sp;
            // cells of partial_row in order (proj/src/fem.cpp:138-172)
            const bool cell[6] = {ip + jp <= n - 1,
                                  ip >= 1 && ip - 1 + jp <= n - 1,
                                  jp >= 1 && ip + jp - 1 <= n - 1,
                                  ip >= 1 && ip + jp <= n - 1,
                                  jp >= 1 && ip + jp <= n - 1,
                                  ip >= 1 && jp >= 1 && ip + jp <= n};
            const double dg[6] = {ku[0], ku[4], ku[8], kd[0], kd[4], kd[8]};
            const int rd[12][2] = {{ip + 1, jp}, {ip, jp + 1}, {ip - 1, jp}, {ip - 1, jp + 1},
                                   {ip, jp - 1}, {ip + 1, jp - 1}, {ip - 1, jp + 1}, {ip, jp + 1},
                                   {ip + 1, jp - 1}, {ip + 1, jp}, {ip, jp - 1}, {ip - 1, jp}};
            double d = 0.0;
            for (int c = 0; c < 6; ++c) {
              r.code[2 * c] = r.code[2 * c + 1] = -1;
              r.loc[2 * c] = r.loc[2 * c + 1] = -1;
              if (!cell[c]) continue;
              r.mask |= 1 << c;
              d += dg[c];
              for (int q = 0; q < 2; ++q) {
                const int xi = rd[2 * c + q][0], xj = rd[2 * c + q][1];
                int code = -1;
                if (sp == m) {
                  code = direction_code(xi - i, xj - j);
                } else {
                  if (on_lattice_boundary(n, xi, xj)) {
                    const int g2 = h.boundary_group(sp, l, xi, xj);
                    for (int k2 = lvl.grp_ptr[g2]; k2 < lvl.grp_ptr[g2 + 1]; ++k2)
                      if (lvl.mem_slot[k2] == m) code = direction_code(lvl.mem_i[k2] - i, lvl.mem_j[k2] - j);
                    if (code < 0) {
                      bool shared = false;
                      for (int k2 = lvl.grp_ptr[g2]; k2 < lvl.grp_ptr[g2 + 1]; ++k2)
                        shared = shared || lvl.mem_slot[k2] == m;
                      if (shared) fail(KB_INTERNAL, "shared neighbour is not lattice-adjacent");
                    }
                  }
                  if (code < 0) {
                    const int goff = sp * S + lattice_index(n, xi, xj);
                    auto it = ghost_of.find(goff);
                    int gi;
                    if (it == ghost_of.end()) {
                      gi = static_cast<int>(ghosts.size());
                      ghosts.push_back(goff);
                      ghost_of[goff] = gi;
                    } else {
                      gi = it->second;
                    }
                    code = 6 + gi;
                  }
                }
                if (code < 0) fail(KB_INTERNAL, "unresolved partial-row read");
                if (code > 32767) fail(KB_INTERNAL, "too many ghost values");
                r.code[2 * c + q] = static_cast<std::int16_t>(code);
                int loc;
                if (code < 6) {
                  static const int dij[6][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {-1, 1}, {1, -1}};
                  loc = lattice_index(n, i + dij[code][0], j + dij[code][1]);
                } else {
                  loc = -1 - (code - 6);
                }
                // only used by the shared-memory smoother (lattices up to n = 128)
                r.loc[2 * c + q] = (loc > 32767 || loc < -32768) ? 0 : static_cast<std::int16_t>(loc);
              }
            }
            diag += d;
            lvl.rec.push_back(r);
          }
        }
        bn.rec_count = static_cast<int>(lvl.rec.size()) - bn.rec_begin;
        bn.diag = diag;
        lvl.bnode[static_cast<std::size_t>(m) * 3 * n + bpos(n, i, j)] = bn;
      };
      for (int i = 0; i <= n; ++i) visit(i, 0);
      for (int j = 1; j <= n; ++j) visit(0, j);
      for (int j = 1; j <= n - 1; ++j) visit(n - j, j);
      lvl.ghost_off.insert(lvl.ghost_off.end(), ghosts.begin(), ghosts.end());
      lvl.ghost_ptr.push_back(static_cast<int>(lvl.ghost_off.size()));
      lvl.max_ghosts = std::max(lvl.max_ghosts, static_cast<int>(ghosts.size()));
    }
    const auto tp0 = std::chrono::steady_clock::now();
    build_programs(lvl, M);
    if (getenv("KB_BUILD_TRACE"))
      fprintf(stderr, "  level %d: tables %.1f ms, programs %.1f ms (prog %zu KB, rec %zu, bnode %zu)\n", l,
              1e3 * std::chrono::duration<double>(tp0 - tl0).count(),
              1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tp0).count(),
              lvl.prog.size() * sizeof(lvl.prog[0]) / 1024, lvl.rec.size(), lvl.bnode.size());
  };
  parallel_levels(0, max_level, derive);
  const bool trace = getenv("KB_BUILD_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  h.build_gs_schedules();
  const auto t1 = std::chrono::steady_clock::now();
  h.build_pipe_tables();
  const auto t2 = std::chrono::steady_clock::now();
  if (trace)
    fprintf(stderr, "hierarchy build: tables+programs %.1f ms, gs schedules %.1f ms, pipe tables %.1f ms\n",
            1e3 * std::chrono::duration<double>(t0 - tb).count(), 1e3 * std::chrono::duration<double>(t1 - t0).count(),
            1e3 * std::chrono::duration<double>(t2 - t1).count());
  return h;
}

}  // namespace kb
