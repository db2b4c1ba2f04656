// Host-side 3-d HHG tables.  See hier3d.hpp for the design.
#include "hier3d.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <new>
#include <set>

namespace kb {

int dir_index(int di, int dj, int dk) {
  for (int d = 0; d < 15; ++d)
    if (kDir[d][0] == di && kDir[d][1] == dj && kDir[d][2] == dk) return d;
  return -1;
}

namespace {

double det3(const double a[3], const double b[3], const double c[3]) {
  return a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) + a[2] * (b[0] * c[1] - b[1] * c[0]);
}

bool in_lattice(int n, int i, int j, int k) { return i >= 0 && j >= 0 && k >= 0 && i + j + k <= n; }

}  // namespace

void tet_matrices(const double p[4][3], double* K, double* Mm) {
  double e[3][3];
  for (int r = 0; r < 3; ++r)
    for (int d = 0; d < 3; ++d) e[r][d] = p[r + 1][d] - p[0][d];
  const double det = det3(e[0], e[1], e[2]);
  const double vol = std::fabs(det) / 6.0;
  // gradients of the barycentric functions 1..3: rows of J^{-1} = cof(J)^T / det, J = [e0 e1 e2] (columns)
  double g[4][3];
  for (int a = 0; a < 3; ++a) {
    const double* u = e[(a + 1) % 3];
    const double* v = e[(a + 2) % 3];
    const double c[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    for (int d = 0; d < 3; ++d) g[a + 1][d] = c[d] / det;
  }
  for (int d = 0; d < 3; ++d) g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      K[4 * a + b] = vol * (g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2]);
      Mm[4 * a + b] = (a == b ? vol / 10.0 : vol / 20.0);
    }
}

Mesh3D Mesh3D::create(int nv, const double* xyz, int ne, const int* t4) {
  if (nv <= 0 || ne <= 0) fail(KB_STRUCTURAL, "empty 3-d macro mesh");
  Mesh3D m;
  m.x.resize(nv);
  m.y.resize(nv);
  m.z.resize(nv);
  for (int v = 0; v < nv; ++v) {
    m.x[v] = xyz[3 * v];
    m.y[v] = xyz[3 * v + 1];
    m.z[v] = xyz[3 * v + 2];
  }
  for (int e = 0; e < ne; ++e) {
    std::array<int, 4> c{t4[4 * e], t4[4 * e + 1], t4[4 * e + 2], t4[4 * e + 3]};
    for (int q = 0; q < 4; ++q)
      if (c[q] < 0 || c[q] >= nv) fail(KB_STRUCTURAL, "tetrahedron corner out of range");
    auto signed_vol = [&](const std::array<int, 4>& t) {
      const double a[3] = {m.x[t[1]] - m.x[t[0]], m.y[t[1]] - m.y[t[0]], m.z[t[1]] - m.z[t[0]]};
      const double b[3] = {m.x[t[2]] - m.x[t[0]], m.y[t[2]] - m.y[t[0]], m.z[t[2]] - m.z[t[0]]};
      const double d[3] = {m.x[t[3]] - m.x[t[0]], m.y[t[3]] - m.y[t[0]], m.z[t[3]] - m.z[t[0]]};
      return det3(a, b, d) / 6.0;
    };
    double v = signed_vol(c);
    if (v < 0.0) {  // orient positively (corners 2 and 3 swapped)
      std::swap(c[2], c[3]);
      v = -v;
    }
    if (!(v > 0.0)) fail(KB_STRUCTURAL, "degenerate tetrahedron");
    m.tet.push_back(c);
    m.vol.push_back(v);
  }
  return m;
}

Hierarchy3D Hierarchy3D::build(const Mesh3D& mesh, int max_level) {
  if (max_level < 0 || max_level > 8) fail(KB_STRUCTURAL, "3-d levels must be in [0, 8]");
  Hierarchy3D h;
  h.mesh = mesh;
  h.L = max_level;
  const int M = static_cast<int>(mesh.tet.size());
  h.M = M;
  const int NV = static_cast<int>(mesh.x.size());

  // primitives: edges and faces keyed by sorted vertex ids, with their tets
  std::map<std::pair<int, int>, int> edge_id;
  std::map<std::array<int, 3>, int> face_id;
  std::vector<int> vert_use(NV, 0), edge_use, face_use;
  for (int s = 0; s < M; ++s) {
    const auto& t = mesh.tet[s];
    ++vert_use[t[0]], ++vert_use[t[1]], ++vert_use[t[2]], ++vert_use[t[3]];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) {
        const auto key = std::make_pair(std::min(t[a], t[b]), std::max(t[a], t[b]));
        if (!edge_id.count(key)) edge_id[key] = 0;
      }
    for (int o = 0; o < 4; ++o) {
      std::array<int, 3> f{};
      int q = 0;
      for (int a = 0; a < 4; ++a)
        if (a != o) f[q++] = t[a];
      std::sort(f.begin(), f.end());
      ++face_id[f];  // temporarily the use count
    }
  }
  {
    int e = 0;
    for (auto& kv : edge_id) kv.second = e++;
    edge_use.assign(e, 0);
    int f = 0;
    face_use.reserve(face_id.size());
    for (auto& kv : face_id) {
      if (kv.second > 2) fail(KB_STRUCTURAL, "non-manifold 3-d macro mesh (face in more than two tets)");
      face_use.push_back(kv.second);
      kv.second = f++;
    }
  }
  for (int s = 0; s < M; ++s) {
    const auto& t = mesh.tet[s];
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b) ++edge_use[edge_id[{std::min(t[a], t[b]), std::max(t[a], t[b])}]];
  }
  // domain boundary: boundary faces and their vertices / edges
  std::vector<std::uint8_t> vbnd(NV, 0);
  std::set<std::pair<int, int>> ebnd;
  for (const auto& kv : face_id)
    if (face_use[kv.second] == 1) {
      const auto& f = kv.first;
      vbnd[f[0]] = vbnd[f[1]] = vbnd[f[2]] = 1;
      ebnd.insert({f[0], f[1]});
      ebnd.insert({f[0], f[2]});
      ebnd.insert({f[1], f[2]});
    }

  // per tet: ids / boundary flags of its 6 edges (by local vertex pair) and 4
  // faces (by the local vertex they miss), so the per-node loops below do no
  // map look-ups
  std::vector<std::array<int, 16>> tet_edge(M);
  std::vector<std::array<std::uint8_t, 16>> tet_edge_bnd(M);
  std::vector<std::array<int, 4>> tet_face(M), tet_face_use(M);
  for (int s = 0; s < M; ++s) {
    const auto& t = mesh.tet[s];
    tet_edge[s].fill(-1);
    tet_edge_bnd[s].fill(0);
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) {
        if (a == b) continue;
        const auto key = std::make_pair(std::min(t[a], t[b]), std::max(t[a], t[b]));
        tet_edge[s][4 * a + b] = edge_id.at(key);
        tet_edge_bnd[s][4 * a + b] = ebnd.count(key) > 0;
      }
    for (int o = 0; o < 4; ++o) {
      std::array<int, 3> f{};
      int q = 0;
      for (int a = 0; a < 4; ++a)
        if (a != o) f[q++] = t[a];
      std::sort(f.begin(), f.end());
      tet_face[s][o] = face_id.at(f);
      tet_face_use[s][o] = face_use[tet_face[s][o]];
    }
  }

  // vertex colouring in Z_2^m: grid parity when the vertices sit on a uniform
  // axis-aligned grid (Kuhn meshes: 8 colours), else greedy by ascending id
  std::vector<int> vcol(NV, 0);
  int ncol = 0;
  {
    double hmin = 1e300, xmin = 1e300, ymin = 1e300, zmin = 1e300;
    for (int v = 0; v < NV; ++v) {
      xmin = std::min(xmin, mesh.x[v]);
      ymin = std::min(ymin, mesh.y[v]);
      zmin = std::min(zmin, mesh.z[v]);
    }
    for (const auto& kv : edge_id) {
      const int a = kv.first.first, b = kv.first.second;
      hmin = std::min(hmin, std::max({std::fabs(mesh.x[a] - mesh.x[b]), std::fabs(mesh.y[a] - mesh.y[b]),
                                      std::fabs(mesh.z[a] - mesh.z[b])}));
    }
    bool grid = hmin > 0.0;
    for (int v = 0; v < NV && grid; ++v) {
      const double q[3] = {(mesh.x[v] - xmin) / hmin, (mesh.y[v] - ymin) / hmin, (mesh.z[v] - zmin) / hmin};
      int c = 0;
      for (int d = 0; d < 3; ++d) {
        const double r = std::round(q[d]);
        if (std::fabs(q[d] - r) > 1e-9) grid = false;
        c |= (static_cast<long long>(r) & 1) << d;
      }
      vcol[v] = c;
    }
    for (int s = 0; s < M && grid; ++s) {
      const auto& t = mesh.tet[s];
      for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b)
          if (vcol[t[a]] == vcol[t[b]]) grid = false;
      // the interior octahedron diagonal flips all four weights
      if ((vcol[t[0]] ^ vcol[t[1]] ^ vcol[t[2]] ^ vcol[t[3]]) == 0) grid = false;
    }
    if (grid) {
      ncol = 8;
    } else {
      // greedy by ascending vertex id: smallest colour differing from every
      // lower-id tet neighbour and, in tets where v is the highest id, from
      // the XOR of the other three corners
      std::vector<std::vector<int>> tets_of(NV);
      for (int s = 0; s < M; ++s)
        for (int a = 0; a < 4; ++a) tets_of[mesh.tet[s][a]].push_back(s);
      int mx = 0;
      for (int v = 0; v < NV; ++v) {
        int c = 0;
        for (bool ok = false; !ok;) {
          ok = true;
          for (int s : tets_of[v]) {
            const auto& t = mesh.tet[s];
            bool lower = true;
            int x = c;
            for (int a = 0; a < 4; ++a) {
              if (t[a] == v) continue;
              if (t[a] > v) lower = false;
              if (t[a] < v && vcol[t[a]] == c) ok = false;
            }
            if (ok && lower) {
              for (int a = 0; a < 4; ++a)
                if (t[a] != v) x ^= vcol[t[a]];
              if (x == 0) ok = false;
            }
            if (!ok) break;
          }
          if (!ok) ++c;
        }
        vcol[v] = c;
        mx = std::max(mx, c);
      }
      ncol = 2;
      while (ncol < mx + 1) ncol <<= 1;
    }
  }
  h.colors = ncol;

  try {
    h.levels.resize(static_cast<std::size_t>(max_level) + 1);
    parallel_levels(0, max_level, [&](int l) {  // the levels are independent: one host thread each
      Level3D lv;
      const int n = 1 << l;
      lv.n = n;
      lv.S = tet_size(n);
      const int S = lv.S;
      const int nE = static_cast<int>(edge_id.size()), nF = static_cast<int>(face_id.size());
      const long long per_face = n >= 3 ? static_cast<long long>(n - 1) * (n - 2) / 2 : 0;
      const long long nG = NV + static_cast<long long>(nE) * (n - 1) + nF * per_face;
      // group layout: vertices, edges (t = weight on the higher-id end), faces (lattice of size n-3)
      auto gid_of = [&](int s, const int* vid, const int* w) -> long long {
        int loc[4], sw[4], cnt = 0;
        for (int q = 0; q < 4; ++q)
          if (w[q] > 0) {
            loc[cnt] = q;
            sw[cnt] = w[q];
            ++cnt;
          }
        for (int a = 0; a < cnt; ++a)  // sort the support by vertex id
          for (int b = a + 1; b < cnt; ++b)
            if (vid[loc[b]] < vid[loc[a]]) std::swap(loc[a], loc[b]), std::swap(sw[a], sw[b]);
        if (cnt == 1) return vid[loc[0]];
        if (cnt == 2) return NV + static_cast<long long>(tet_edge[s][4 * loc[0] + loc[1]]) * (n - 1) + (sw[1] - 1);
        return NV + static_cast<long long>(nE) * (n - 1) +
               static_cast<long long>(tet_face[s][6 - loc[0] - loc[1] - loc[2]]) * per_face +
               lattice_index(n - 3, sw[1] - 1, sw[2] - 1);
      };
      auto gcolor = [&](const int* vid, const int* w) {
        int c = 0;
        for (int q = 0; q < 4; ++q)
          if (w[q] & 1) c ^= vcol[vid[q]];
        return c;
      };
      // members per group (CSR), in slot order
      if (nG >= (1ll << 31)) fail(KB_RESOURCE, "too many shared-node groups");
      std::vector<int> cnt(nG + 1, 0);
      lv.node_gid.assign(static_cast<size_t>(M) * S, -1);
      std::vector<int>& node_g = lv.node_gid;
      for (int s = 0; s < M; ++s) {
        const int* vid = mesh.tet[s].data();
        for (int k = 0; k <= n; ++k)
          for (int j = 0; j <= n - k; ++j)
            for (int i = 0; i <= n - k - j; ++i) {
              const int w[4] = {n - i - j - k, i, j, k};
              if (w[0] > 0 && i > 0 && j > 0 && k > 0) continue;
              const int g = static_cast<int>(gid_of(s, vid, w));
              node_g[static_cast<size_t>(s) * S + lattice_index3(n, i, j, k)] = g;
              ++cnt[g + 1];
            }
      }
      for (long long g = 0; g < nG; ++g) cnt[g + 1] += cnt[g];
      lv.grp_ptr.assign(cnt.begin(), cnt.end());
      lv.mem_slot.assign(cnt[nG], 0);
      lv.mem_idx.assign(cnt[nG], 0);
      lv.grp_domain.assign(nG, 0);
      lv.grp_color.assign(nG, 0);
      std::vector<int> fill(cnt.begin(), cnt.end() - 1);
      lv.node_flags.assign(static_cast<size_t>(M) * S, 4);
      lv.pat_color.assign(8 * static_cast<size_t>(M), 0);
      for (int s = 0; s < M; ++s) {
        const int* vid = mesh.tet[s].data();
        for (int p = 0; p < 8; ++p) {
          const int pi = p & 1, pj = (p >> 1) & 1, pk = (p >> 2) & 1;
          const int w[4] = {(n + pi + pj + pk) & 1, pi, pj, pk};
          lv.pat_color[8 * s + p] = gcolor(vid, w);
        }
        for (int k = 0; k <= n; ++k)
          for (int j = 0; j <= n - k; ++j)
            for (int i = 0; i <= n - k - j; ++i) {
              const size_t off = static_cast<size_t>(s) * S + lattice_index3(n, i, j, k);
              const int g = node_g[off];
              if (g < 0) continue;
              const int w[4] = {n - i - j - k, i, j, k};
              const int first = lv.grp_ptr[g];
              const bool owner = fill[g] == first;
              lv.mem_slot[fill[g]] = s;
              lv.mem_idx[fill[g]] = lattice_index3(n, i, j, k);
              ++fill[g];
              // domain boundary: the node's support lies in a boundary face
              int loc[4], c = 0;
              for (int q = 0; q < 4; ++q)
                if (w[q] > 0) loc[c++] = q;
              bool dom;
              if (c == 1)
                dom = vbnd[vid[loc[0]]];
              else if (c == 2)
                dom = tet_edge_bnd[s][4 * loc[0] + loc[1]] != 0;
              else
                dom = tet_face_use[s][6 - loc[0] - loc[1] - loc[2]] == 1;
              lv.grp_domain[g] = dom;
              lv.grp_color[g] = gcolor(vid, w);
              lv.node_flags[off] = static_cast<std::uint8_t>(1 | (dom ? 2 : 0) | (owner ? 4 : 0));
            }
      }
      const long long interior = n >= 4 ? static_cast<long long>(n - 1) * (n - 2) * (n - 3) / 6 : 0;
      lv.dofs = NV + static_cast<long long>(nE) * (n - 1) + nF * per_face + M * interior;

      // element matrices (six Kuhn types) and the interior 15-point stencil
      lv.kstiff.assign(96 * static_cast<size_t>(M), 0.0);
      lv.kmass.assign(96 * static_cast<size_t>(M), 0.0);
      lv.stencil.assign(15 * static_cast<size_t>(M), 0.0);
      lv.inv_c.assign(M, 0.0);
      for (int s = 0; s < M; ++s) {
        const auto& t = mesh.tet[s];
        const double P[4][3] = {{mesh.x[t[0]], mesh.y[t[0]], mesh.z[t[0]]},
                                {mesh.x[t[1]], mesh.y[t[1]], mesh.z[t[1]]},
                                {mesh.x[t[2]], mesh.y[t[2]], mesh.z[t[2]]},
                                {mesh.x[t[3]], mesh.y[t[3]], mesh.z[t[3]]}};
        auto node_x = [&](int i, int j, int k, double* out) {
          for (int d = 0; d < 3; ++d)
            out[d] = P[0][d] + (static_cast<double>(i) / n) * (P[1][d] - P[0][d]) +
                     (static_cast<double>(j) / n) * (P[2][d] - P[0][d]) +
                     (static_cast<double>(k) / n) * (P[3][d] - P[0][d]);
        };
        for (int ty = 0; ty < 6; ++ty) {
          double p[4][3];
          for (int r = 0; r < 4; ++r) {
            int di, dj, dk;
            cell_vertex(ty, r, di, dj, dk);
            node_x(di, dj, dk, p[r]);
          }
          tet_matrices(p, &lv.kstiff[96 * s + 16 * ty], &lv.kmass[96 * s + 16 * ty]);
        }
        double* st = &lv.stencil[15 * s];
        for (int ty = 0; ty < 6; ++ty)
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
              int ri, rj, rk, ci, cj, ck;
              cell_vertex(ty, r, ri, rj, rk);
              cell_vertex(ty, c, ci, cj, ck);
              const int d = dir_index(ci - ri, cj - rj, ck - rk);
              if (d < 0) fail(KB_INTERNAL, "micro-cell edge outside the 15-point stencil");
              st[d] += lv.kstiff[96 * s + 16 * ty + 4 * r + c];
            }
        lv.inv_c[s] = 1.0 / st[0];
      }
      // partial stencils per boundary signature: from the first node (lattice
      // order) carrying it, the sum over its existing cells in (type, role,
      // column) order; every other node of that signature is checked on small
      // levels to have the same cells
      lv.psK.assign(240 * static_cast<size_t>(M), 0.0);
      lv.psM.assign(240 * static_cast<size_t>(M), 0.0);
      auto cells_of = [&](int i, int j, int k, auto&& visit) {
        for (int ty = 0; ty < 6; ++ty)
          for (int r = 0; r < 4; ++r) {
            int ri, rj, rk;
            cell_vertex(ty, r, ri, rj, rk);
            bool ok = true;
            for (int c = 0; c < 4 && ok; ++c) {
              int ci, cj, ck;
              cell_vertex(ty, c, ci, cj, ck);
              ok = in_lattice(n, i - ri + ci, j - rj + cj, k - rk + ck);
            }
            if (ok) visit(ty, r);
          }
      };
      for (int s = 0; s < M; ++s) {
        int done = 0;
        std::vector<int> cellmask(16, 0);
        for (int k = 0; k <= n; ++k)
          for (int j = 0; j <= n - k; ++j)
            for (int i = 0; i <= n - k - j; ++i) {
              const int sg = boundary_signature(n, i, j, k);
              if (sg == 0) continue;
              int mask = 0;
              if (!((done >> sg) & 1) || n <= 16) cells_of(i, j, k, [&](int ty, int r) { mask |= 1 << (4 * ty + r); });
              if ((done >> sg) & 1) {
                if (n <= 16 && mask != cellmask[sg]) fail(KB_INTERNAL, "boundary signature does not fix the cells");
                continue;
              }
              done |= 1 << sg;
              cellmask[sg] = mask;
              double* pk = &lv.psK[240 * static_cast<size_t>(s) + 15 * sg];
              double* pm = &lv.psM[240 * static_cast<size_t>(s) + 15 * sg];
              cells_of(i, j, k, [&](int ty, int r) {
                int ri, rj, rk;
                cell_vertex(ty, r, ri, rj, rk);
                for (int c = 0; c < 4; ++c) {
                  int ci, cj, ck;
                  cell_vertex(ty, c, ci, cj, ck);
                  const int d = dir_index(ci - ri, cj - rj, ck - rk);
                  pk[d] += lv.kstiff[96 * s + 16 * ty + 4 * r + c];
                  pm[d] += lv.kmass[96 * s + 16 * ty + 4 * r + c];
                }
              });
            }
      }
      // group diagonals: sum over members of the partial-stencil centres
      lv.grp_diag.assign(nG, 0.0);
      {
        std::vector<int> ii(S), jj(S), kk(S);
        for (int k = 0; k <= n; ++k)
          for (int j = 0; j <= n - k; ++j)
            for (int i = 0; i <= n - k - j; ++i) {
              const int idx = lattice_index3(n, i, j, k);
              ii[idx] = i, jj[idx] = j, kk[idx] = k;
            }
        for (long long g = 0; g < nG; ++g) {
          double diag = 0.0;
          for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
            const int idx = lv.mem_idx[q];
            diag += lv.psK[240 * static_cast<size_t>(lv.mem_slot[q]) + 15 * boundary_signature(n, ii[idx], jj[idx], kk[idx])];
          }
          lv.grp_diag[g] = diag;
        }
      }
      // boundary groups by colour
      lv.color_grp_ptr.assign(ncol + 1, 0);
      for (long long g = 0; g < nG; ++g) ++lv.color_grp_ptr[lv.grp_color[g] + 1];
      for (int c = 0; c < ncol; ++c) lv.color_grp_ptr[c + 1] += lv.color_grp_ptr[c];
      lv.color_grp.assign(nG, 0);
      {
        std::vector<int> f2(lv.color_grp_ptr.begin(), lv.color_grp_ptr.end() - 1);
        for (long long g = 0; g < nG; ++g) lv.color_grp[f2[lv.grp_color[g]]++] = static_cast<int>(g);
      }
      h.levels[static_cast<std::size_t>(l)] = std::move(lv);
    });
  } catch (const std::bad_alloc&) {
    Error e(KB_RESOURCE, "out of memory while building a 3-d hierarchy level");
    e.level = max_level;
    throw e;
  }
  return h;
}

}  // namespace kb
