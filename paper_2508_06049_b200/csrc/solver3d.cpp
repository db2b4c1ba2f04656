// Host orchestration of the 3-d hot path.  See solver3d.hpp.
#include "solver3d.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <thread>

namespace kb {

void launch3_ftab(const DevLevel3D& lv, const double* corners, int kind, const double* params, double* f,
                  cudaStream_t st);  // kernels3d.cu

namespace {
size_t r256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }

double sin3(double x, double y, double z) { return std::sin(M_PI * x) * std::sin(M_PI * y) * std::sin(M_PI * z); }
double gauss3(double x, double y, double z) {
  const double dx = x - 0.5, dy = y - 0.5, dz = z - 0.5;
  return std::exp(-1000.0 * (dx * dx + dy * dy + dz * dz));
}
}  // namespace

// ------------------------------------------------------------------ hierarchy upload
std::unique_ptr<DeviceHierarchy3D> DeviceHierarchy3D::create(const Mesh3D& mesh, int max_level) {
  auto d = std::make_unique<DeviceHierarchy3D>();
  d->host = Hierarchy3D::build(mesh, max_level);
  const Hierarchy3D& h = d->host;
  std::vector<std::vector<int>> ijk(h.L + 1), own(h.L + 1), col_pat(h.L + 1), pat_ptr(h.L + 1), pat_node(h.L + 1);
  std::vector<int> pat_max(h.L + 1, 0);
  size_t bytes = 0;
  for (int l = 0; l <= h.L; ++l) {
    const Level3D& lv = h.levels[l];
    const int n = lv.n;
    ijk[l].resize(lv.mem_slot.size());
    // member (i, j, k) from the lattice index
    std::vector<int> ii(lv.S), jj(lv.S), kk(lv.S);
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n - k; ++j)
        for (int i = 0; i <= n - k - j; ++i) {
          const int idx = lattice_index3(n, i, j, k);
          ii[idx] = i, jj[idx] = j, kk[idx] = k;
        }
    for (size_t q = 0; q < lv.mem_slot.size(); ++q) {
      const int idx = lv.mem_idx[q];
      ijk[l][q] = ii[idx] | (jj[idx] << 10) | (kk[idx] << 20);
    }
    const int ng = static_cast<int>(lv.grp_ptr.size()) - 1;
    own[l].resize(ng);
    for (int g = 0; g < ng; ++g) {
      const int q = lv.grp_ptr[g];
      own[l][g] = lv.mem_slot[q] * lv.S + lv.mem_idx[q];
    }
    // colour -> parity pattern per macro
    col_pat[l].assign(static_cast<size_t>(h.M) * h.colors, -1);
    for (int s = 0; s < h.M; ++s)
      for (int p = 0; p < 8; ++p) col_pat[l][static_cast<size_t>(h.colors) * s + lv.pat_color[8 * s + p]] = p;
    // the interior relaxations of a macro in the smoother's order: step (plane k,
    // parity class q) at [pat_ptr[4 (k - 1) + q], ...), entry = lat2(n - k, i, j) | j << 16
    if (n >= 4 && n <= 64) {
      pat_ptr[l].assign(1, 0);
      for (int k = 1; k <= n - 3; ++k)
        for (int q = 0; q < 4; ++q) {
          // The nodes of a step are independent, so their order is free: runs of
          // 8 consecutive class nodes of a row (16-byte stride) are paired, one
          // with an even and one with an odd in-plane index, per half-warp — the
          // two runs then fall on disjoint shared-memory banks for every one of
          // the 14 neighbour loads (all offsets shift both runs alike).
          std::vector<std::vector<int>> run[2];
          std::vector<int> rest;
          for (int j = 1 + (q >> 1); j <= n - 2 - k; j += 2) {
            std::vector<int> row;
            for (int i = 1 + (q & 1); i <= n - 1 - k - j; i += 2)
              row.push_back((j * (n - k + 1) - (j * (j - 1)) / 2 + i) | j << 16);
            size_t t = 0;
            for (; t + 8 <= row.size(); t += 8)
              run[(row[t] & 0xffff) & 1].emplace_back(row.begin() + t, row.begin() + t + 8);
            rest.insert(rest.end(), row.begin() + t, row.end());
          }
          const size_t pairs = std::min(run[0].size(), run[1].size());
          for (size_t t = 0; t < pairs; ++t)
            for (int h = 0; h < 2; ++h) pat_node[l].insert(pat_node[l].end(), run[h][t].begin(), run[h][t].end());
          for (int h = 0; h < 2; ++h)
            for (size_t t = pairs; t < run[h].size(); ++t)
              pat_node[l].insert(pat_node[l].end(), run[h][t].begin(), run[h][t].end());
          pat_node[l].insert(pat_node[l].end(), rest.begin(), rest.end());
          const int end = static_cast<int>(pat_node[l].size());
          pat_max[l] = std::max(pat_max[l], end - pat_ptr[l].back());
          pat_ptr[l].push_back(end);
        }
    }
    auto vb = [](auto& v) { return r256(v.size() * sizeof(v[0])); };
    bytes += vb(lv.grp_ptr) + vb(lv.mem_slot) + vb(ijk[l]) + vb(lv.grp_domain) + vb(lv.grp_diag) +
             vb(lv.color_grp_ptr) + vb(lv.color_grp) + vb(lv.kstiff) + vb(lv.kmass) + 2 * vb(lv.stencil) +
             vb(lv.inv_c) + vb(lv.pat_color) + vb(own[l]) + r256(4 * h.colors) + vb(col_pat[l]) +
             vb(pat_ptr[l]) + vb(pat_node[l]) + r256(lv.color_grp.size() * 16) + r256(lv.color_grp.size() * 32) +
             r256(lv.mem_slot.size() * 8 + 8);
  }
  // level-0 CG program: for every vertex group, its members' partial stencils
  // as (coefficient, global vertex) terms, centre first (level-0 groups are the
  // macro vertices in id order)
  std::vector<int> cg_gmem(1, 0), cg_mterm(1, 0), cg_vid;
  std::vector<double> cg_coef;
  {
    const Level3D& lv = h.levels[0];
    const int ng = static_cast<int>(lv.grp_ptr.size()) - 1;
    for (int g = 0; g < ng; ++g) {
      for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
        const int s = lv.mem_slot[q], idx = lv.mem_idx[q];
        const int i = idx == 1, j = idx == 2, k = idx == 3;  // n = 1: lattice index = local vertex
        const double* ps = &lv.psK[240 * static_cast<size_t>(s) + 15 * boundary_signature(1, i, j, k)];
        for (int dd = 0; dd < 15; ++dd) {
          const int a = i + kDir[dd][0], b = j + kDir[dd][1], c = k + kDir[dd][2];
          if (a < 0 || b < 0 || c < 0 || a + b + c > 1) continue;
          cg_coef.push_back(ps[dd]);
          cg_vid.push_back(h.mesh.tet[s][lattice_index3(1, a, b, c)]);
        }
        cg_mterm.push_back(static_cast<int>(cg_coef.size()));
      }
      cg_gmem.push_back(static_cast<int>(cg_mterm.size()) - 1);
      if (lv.grp_ptr[g + 1] == lv.grp_ptr[g]) fail(KB_STRUCTURAL, "macro vertex used by no tetrahedron");
    }
    bytes += r256(cg_gmem.size() * 4) + r256(cg_mterm.size() * 4) + r256(cg_vid.size() * 4) + r256(cg_coef.size() * 8);
    // compact program (upper bounds: every row distinct)
    bytes += r256(cg_coef.size() * 8) + r256(cg_mterm.size() * 2) + r256(cg_vid.size() * 2);
  }
  for (int l = 0; l <= h.L; ++l) bytes += 2 * r256(h.levels[l].psK.size() * 8);
  d->arena.reserve(bytes + 4096);
  for (int l = 0; l <= h.L; ++l) {
    const Level3D& lv = h.levels[l];
    DevLevel3D dl{};
    dl.n = lv.n;
    dl.S = lv.S;
    dl.M = h.M;
    dl.ng = static_cast<int>(lv.grp_ptr.size()) - 1;
    dl.colors = h.colors;
    dl.grp_ptr = d->arena.upload(lv.grp_ptr);
    dl.mem_slot = d->arena.upload(lv.mem_slot);
    dl.mem_ijk = d->arena.upload(ijk[l]);
    dl.grp_domain = d->arena.upload(lv.grp_domain);
    dl.grp_diag = d->arena.upload(lv.grp_diag);
    dl.color_grp_ptr = d->arena.upload(lv.color_grp_ptr);
    {
      // within a colour the groups are independent: wide ones first (warp
      // relaxation), then the narrow ones, each part ascending
      std::vector<int> cg(lv.color_grp.size()), wide_end(h.colors);
      for (int c = 0; c < h.colors; ++c) {
        int w = lv.color_grp_ptr[c];
        for (int t = lv.color_grp_ptr[c]; t < lv.color_grp_ptr[c + 1]; ++t) {
          const int g = lv.color_grp[t];
          if (lv.grp_ptr[g + 1] - lv.grp_ptr[g] > 4) cg[w++] = g;
        }
        wide_end[c] = w;
        for (int t = lv.color_grp_ptr[c]; t < lv.color_grp_ptr[c + 1]; ++t) {
          const int g = lv.color_grp[t];
          if (lv.grp_ptr[g + 1] - lv.grp_ptr[g] <= 4) cg[w++] = g;
        }
      }
      dl.color_grp = d->arena.upload(cg);
      dl.color_wide_end = d->arena.upload(wide_end);
      dl.max_color_groups = 0;
      for (int c = 0; c < h.colors; ++c)
        dl.max_color_groups = std::max(dl.max_color_groups, lv.color_grp_ptr[c + 1] - lv.color_grp_ptr[c]);
      // flat records of the groups at their colour-list position
      std::vector<int4> hdr(cg.size(), make_int4(0, 0, 0, 0));
      std::vector<int2> mem(4 * cg.size(), make_int2(-1, 0)), wide;
      for (size_t t = 0; t < cg.size(); ++t) {
        const int g = cg[t], beg = lv.grp_ptr[g], cnt = lv.grp_ptr[g + 1] - beg;
        if (cnt > 0xffff) fail(KB_STRUCTURAL, "shared-node group with more than 65535 members");
        std::int32_t w[2];
        std::memcpy(w, &lv.grp_diag[g], 8);
        hdr[t] = make_int4(w[0], w[1], cnt | (lv.grp_domain[g] ? 1 << 16 : 0), static_cast<int>(wide.size()));
        for (int q = 0; q < cnt; ++q) {
          const int2 rec = make_int2(lv.mem_slot[beg + q], ijk[l][beg + q]);
          if (cnt <= 4)
            mem[4 * t + q] = rec;
          else
            wide.push_back(rec);
        }
      }
      if (wide.empty()) wide.push_back(make_int2(0, 0));
      dl.nar_hdr = d->arena.upload(hdr);
      dl.nar_mem = d->arena.upload(mem);
      dl.wide_mem = d->arena.upload(wide);
    }
    dl.kstiff = d->arena.upload(lv.kstiff);
    dl.kmass = d->arena.upload(lv.kmass);
    // interior stencils: stiffness from the host tables, mass summed the same way
    std::vector<double> stM(15 * static_cast<size_t>(h.M), 0.0);
    for (int s = 0; s < h.M; ++s)
      for (int ty = 0; ty < 6; ++ty)
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) {
            int ri, rj, rk, ci, cj, ck;
            cell_vertex(ty, r, ri, rj, rk);
            cell_vertex(ty, c, ci, cj, ck);
            stM[15 * s + dir_index(ci - ri, cj - rj, ck - rk)] += lv.kmass[96 * s + 16 * ty + 4 * r + c];
          }
    dl.stK = d->arena.upload(lv.stencil);
    dl.stM = d->arena.upload(stM);
    dl.inv_c = d->arena.upload(lv.inv_c);
    dl.pat_color = d->arena.upload(lv.pat_color);
    dl.col_pat = d->arena.upload(col_pat[l]);
    if (!pat_node[l].empty()) {
      dl.pat_ptr = d->arena.upload(pat_ptr[l]);
      dl.pat_node = d->arena.upload(pat_node[l]);
      dl.pat_max = pat_max[l];
    }
    dl.own_dot = d->arena.upload(own[l]);
    dl.psK = d->arena.upload(lv.psK);
    dl.psM = d->arena.upload(lv.psM);
    if (l == 0) {
      // assembled level-0 operator: row g adds the members' partial stencils in
      // slot order (terms centre first), coefficients of one column added in
      // that order, columns in first-appearance order (oracle apply0)
      std::vector<int> rowptr(1, 0);
      std::vector<unsigned short> col;
      std::vector<double> val;
      for (size_t g = 0; g + 1 < cg_gmem.size(); ++g) {
        const size_t start = col.size();
        for (int q = cg_gmem[g]; q < cg_gmem[g + 1]; ++q)
          for (int t = cg_mterm[q]; t < cg_mterm[q + 1]; ++t) {
            const int v = cg_vid[t];
            if (v < 0 || v >= 65536) fail(KB_STRUCTURAL, "coarse mesh too large for the level-0 CG (vertex id >= 65536)");
            size_t pos = start;
            while (pos < col.size() && col[pos] != v) ++pos;
            if (pos == col.size()) {
              col.push_back(static_cast<unsigned short>(v));
              val.push_back(cg_coef[t]);
            } else {
              val[pos] = val[pos] + cg_coef[t];
            }
          }
        rowptr.push_back(static_cast<int>(col.size()));
      }
      dl.cg_rowptr = d->arena.upload(rowptr);
      dl.cg_col = d->arena.upload(col);
      dl.cg_val = d->arena.upload(val);
      dl.cg_nnz = static_cast<int>(col.size());
    }
    d->lev.push_back(dl);
  }
  return d;
}

// ------------------------------------------------------------------ problems
Problem3D Problem3D::builtin(int kind) {
  Problem3D p;
  p.kind = kind;
  switch (kind) {
    case P3_ZERO:
      p.source = p.boundary = [](double, double, double) { return 0.0; };
      break;
    case P3_SIN:  // BASELINE.json config 3: u = prod sin(pi x_i), f = 3 pi^2 u
      p.boundary = sin3;
      p.source = [](double x, double y, double z) { return 3.0 * M_PI * M_PI * sin3(x, y, z); };
      break;
    case P3_GAUSS:  // config 4: u = exp(-1000 |x - c|^2), f = (6a - 4a^2 r^2) u
      p.boundary = gauss3;
      p.source = [](double x, double y, double z) {
        const double dx = x - 0.5, dy = y - 0.5, dz = z - 0.5, r2 = dx * dx + dy * dy + dz * dz;
        return (6.0 * 1000.0 - 4.0 * 1000.0 * 1000.0 * r2) * gauss3(x, y, z);
      };
      break;
    case P3_SERIES:  // config 5: f = sum C_abc sin(a pi x) sin(b pi y) sin(c pi z), g = 0
      p.params.assign(64, 0.0);
      p.boundary = [](double, double, double) { return 0.0; };
      break;
    default:
      fail(KB_STRUCTURAL, "unknown built-in 3-d problem kind");
  }
  return p;
}

void Problem3D::set_params(const double* v, int count) {
  if (kind != P3_SERIES || count != 64) fail(KB_STRUCTURAL, "series problems take 64 coefficients");
  params.assign(v, v + count);
}

// acc += C_abc * ((sin(a pi x) * sin(b pi y)) * sin(c pi z)) in (c, b, a) order;
// the twelve sines are formed once per point (same values, same bits)
double series_value(const std::vector<double>& C, double x, double y, double z) {
  double sx[5], sy[5], sz[5];
  for (int a = 1; a <= 4; ++a) {
    sx[a] = std::sin(a * M_PI * x);
    sy[a] = std::sin(a * M_PI * y);
    sz[a] = std::sin(a * M_PI * z);
  }
  double acc = 0.0;
  for (int c = 1; c <= 4; ++c)
    for (int b = 1; b <= 4; ++b)
      for (int a = 1; a <= 4; ++a) acc += C[(a - 1) + 4 * (b - 1) + 16 * (c - 1)] * (sx[a] * sy[b] * sz[c]);
  return acc;
}

void tabulate_source3(const Hierarchy3D& hh, int l, const Problem3D& p, int s0, int s1, double* out) {
  const Level3D& lv = hh.levels[l];
  const int n = lv.n, S = lv.S;
  std::vector<int> ii(S), jj(S), kk(S);
  for (int k = 0; k <= n; ++k)
    for (int j = 0; j <= n - k; ++j)
      for (int i = 0; i <= n - k - j; ++i) {
        const int idx = lattice_index3(n, i, j, k);
        ii[idx] = i, jj[idx] = j, kk[idx] = k;
      }
  auto work = [&](int a, int b) {
    for (int s = a; s < b; ++s)
      for (int idx = 0; idx < S; ++idx) {
        const size_t off = static_cast<size_t>(s) * S + idx;
        int os = s, oidx = idx;
        const int g = lv.node_gid[off];
        if (g >= 0) {
          os = lv.mem_slot[lv.grp_ptr[g]];
          oidx = lv.mem_idx[lv.grp_ptr[g]];
        }
        const auto& t = hh.mesh.tet[os];
        double x[3];
        const double P[4][3] = {{hh.mesh.x[t[0]], hh.mesh.y[t[0]], hh.mesh.z[t[0]]},
                                {hh.mesh.x[t[1]], hh.mesh.y[t[1]], hh.mesh.z[t[1]]},
                                {hh.mesh.x[t[2]], hh.mesh.y[t[2]], hh.mesh.z[t[2]]},
                                {hh.mesh.x[t[3]], hh.mesh.y[t[3]], hh.mesh.z[t[3]]}};
        for (int c = 0; c < 3; ++c)
          x[c] = P[0][c] + (static_cast<double>(ii[oidx]) / n) * (P[1][c] - P[0][c]) +
                 (static_cast<double>(jj[oidx]) / n) * (P[2][c] - P[0][c]) +
                 (static_cast<double>(kk[oidx]) / n) * (P[3][c] - P[0][c]);
        out[static_cast<size_t>(s - s0) * S + idx] =
            p.kind == P3_SERIES ? series_value(p.params, x[0], x[1], x[2]) : p.source(x[0], x[1], x[2]);
      }
  };
  const long long nodes = static_cast<long long>(s1 - s0) * S;
  int nt = static_cast<int>(std::min<long long>(std::max(1u, std::thread::hardware_concurrency()), nodes / 200000 + 1));
  // host problems wrap caller callbacks (e.g. Python through ctypes): one thread
  if (p.kind == P3_HOST) nt = 1;
  if (nt <= 1) {
    work(s0, s1);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) {
    const int a = s0 + static_cast<int>(static_cast<long long>(s1 - s0) * t / nt);
    const int b = s0 + static_cast<int>(static_cast<long long>(s1 - s0) * (t + 1) / nt);
    pool.emplace_back(work, a, b);
  }
  for (auto& th : pool) th.join();
}

// ------------------------------------------------------------------ solver
Solver3D::Solver3D(std::shared_ptr<DeviceHierarchy3D> h, Problem3D p, SolverConfig2D cfg)
    : H_(std::move(h)), prob_(std::move(p)), cfg_(cfg) {
  const Hierarchy3D& hh = H_->host;
  L_ = hh.L;
  const int M = hh.M;
  if (cfg_.finest_policy != 0) fail(KB_STRUCTURAL, "only FinestPolicy::None is available on the device path");
  // host-callback problems have no device form: always tabulated on the host
  if (prob_.kind == P3_HOST) cfg_.faithful_source = 1;
  has_source_ = prob_.kind != P3_ZERO;
  auto lsize = [&](int l) { return static_cast<size_t>(M) * hh.levels[l].S; };
  size_t bytes = 0;
  for (int l = 0; l <= L_; ++l) {
    bytes += 2 * r256(lsize(l) * 8);
    if (l < L_) bytes += r256(lsize(l + 1) * 8) + 2 * r256(lsize(l) * 8);
    if (l >= 1) bytes += r256(lsize(l) * 8);
    bytes += r256((hh.levels[l].grp_ptr.size()) * 8);
    if (has_source_) bytes += r256(lsize(l) * 8);
  }
  bytes += r256(3 * lsize(0) * 8) + r256(2 * M * 8) + 3 * r256(lsize(L_) * 8) + r256(64 * 8) + r256(8) +
           r256(sizeof(DevStatus)) + r256(12 * M * 8) + r256(64 * 8);
  arena_.reserve(bytes);
  u_.assign(L_ + 1, nullptr);
  b_ = w_ = vu_ = vb_ = r_ = gbnd_ = ftab_ = u_;
  for (int l = 0; l <= L_; ++l) {
    u_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    b_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    if (l < L_) {
      w_[l] = static_cast<double*>(arena_.take(lsize(l + 1) * 8));
      vu_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
      vb_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    }
    if (l >= 1) r_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    gbnd_[l] = static_cast<double*>(arena_.take(hh.levels[l].grp_ptr.size() * 8));
    if (has_source_) ftab_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
  }
  cg_scratch_ = static_cast<double*>(arena_.take(3 * lsize(0) * 8));
  est_sums_ = static_cast<double*>(arena_.take(2 * M * 8));
  est_a_ = static_cast<double*>(arena_.take(lsize(L_) * 8));
  est_b_ = static_cast<double*>(arena_.take(lsize(L_) * 8));
  est_c_ = static_cast<double*>(arena_.take(lsize(L_) * 8));
  dot_partial_ = static_cast<double*>(arena_.take(64 * 8));
  dot_out_ = static_cast<double*>(arena_.take(8));
  status_ = static_cast<DevStatus*>(arena_.take(sizeof(DevStatus)));
  corners_ = static_cast<double*>(arena_.take(12 * M * 8));
  params_ = static_cast<double*>(arena_.take(64 * 8));
  KB_CUDA_CHECK(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  stream_ = own_stream_;
  KB_CUDA_CHECK(cudaMallocHost(&status_host_, sizeof(DevStatus)));
  KB_CUDA_CHECK(cudaMallocHost(&sums_host_, 2 * M * sizeof(double)));
  KB_CUDA_CHECK(cudaMemset(status_, 0, sizeof(DevStatus)));
  // macro corners + series coefficients for the device source tables (fast mode)
  std::vector<double> cv(12 * static_cast<size_t>(M));
  for (int s = 0; s < M; ++s)
    for (int c = 0; c < 4; ++c) {
      const int v = hh.mesh.tet[s][c];
      cv[12 * s + 3 * c] = hh.mesh.x[v];
      cv[12 * s + 3 * c + 1] = hh.mesh.y[v];
      cv[12 * s + 3 * c + 2] = hh.mesh.z[v];
    }
  KB_CUDA_CHECK(cudaMemcpy(corners_, cv.data(), cv.size() * 8, cudaMemcpyHostToDevice));
  for (int l = 0; l <= L_; ++l) stage_count_ = std::max(stage_count_, std::max(lsize(l), hh.levels[l].grp_ptr.size()));
  KB_CUDA_CHECK(cudaMallocHost(&stage_, stage_count_ * sizeof(double)));
  load_problem(prob_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

Solver3D::~Solver3D() {
  if (exec_) cudaGraphExecDestroy(exec_);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  if (own_stream_) cudaStreamDestroy(own_stream_);
  if (status_host_) cudaFreeHost(status_host_);
  if (sums_host_) cudaFreeHost(sums_host_);
  if (stage_) cudaFreeHost(stage_);
}

size_t Solver3D::level_size(int level) const {
  return static_cast<size_t>(H_->host.M) * H_->host.levels.at(level).S;
}

// Dirichlet values g per group and (faithful mode) f per copy, both at the
// owner copy's node coordinates, host libm (like proj/src/fem.cpp:212-228).
size_t Solver3D::load_problem(const Problem3D& p) {
  if (p.kind != prob_.kind) fail(KB_STRUCTURAL, "set_problem: the problem kind must match the solver's");
  if (&p != &prob_) prob_ = p;
  const Hierarchy3D& hh = H_->host;
  const int M = hh.M;
  size_t bytes = 0;
  for (int l = 0; l <= L_; ++l) {
    const Level3D& lv = hh.levels[l];
    const int n = lv.n, S = lv.S;
    auto coords = [&](int s, int i, int j, int k, double* out) {
      const auto& t = hh.mesh.tet[s];
      const double P[4][3] = {{hh.mesh.x[t[0]], hh.mesh.y[t[0]], hh.mesh.z[t[0]]},
                              {hh.mesh.x[t[1]], hh.mesh.y[t[1]], hh.mesh.z[t[1]]},
                              {hh.mesh.x[t[2]], hh.mesh.y[t[2]], hh.mesh.z[t[2]]},
                              {hh.mesh.x[t[3]], hh.mesh.y[t[3]], hh.mesh.z[t[3]]}};
      for (int a = 0; a < 3; ++a)
        out[a] = P[0][a] + (static_cast<double>(i) / n) * (P[1][a] - P[0][a]) +
                 (static_cast<double>(j) / n) * (P[2][a] - P[0][a]) + (static_cast<double>(k) / n) * (P[3][a] - P[0][a]);
    };
    std::vector<int> ii(S), jj(S), kk(S);
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n - k; ++j)
        for (int i = 0; i <= n - k - j; ++i) {
          const int idx = lattice_index3(n, i, j, k);
          ii[idx] = i, jj[idx] = j, kk[idx] = k;
        }
    const int ng = static_cast<int>(lv.grp_ptr.size()) - 1;
    KB_CUDA_CHECK(cudaStreamSynchronize(stream_));  // the staging buffer may feed an earlier copy
    for (int g = 0; g < ng; ++g) {
      double v = 0.0;
      if (lv.grp_domain[g]) {
        const int q = lv.grp_ptr[g], s = lv.mem_slot[q], idx = lv.mem_idx[q];
        double x[3];
        coords(s, ii[idx], jj[idx], kk[idx], x);
        v = prob_.boundary(x[0], x[1], x[2]);
      }
      stage_[g] = v;
    }
    KB_CUDA_CHECK(cudaMemcpyAsync(gbnd_[l], stage_, ng * 8, cudaMemcpyHostToDevice, stream_));
    bytes += ng * 8;
    if (has_source_ && cfg_.faithful_source) {
      KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
      const size_t N = level_size(l);
      tabulate_source3(hh, l, prob_, 0, M, stage_);
      KB_CUDA_CHECK(cudaMemcpyAsync(ftab_[l], stage_, N * 8, cudaMemcpyHostToDevice, stream_));
      bytes += N * 8;
    }
  }
  if (has_source_ && !cfg_.faithful_source) {
    // fast mode: f from the device tables of the (possibly new) coefficients
    KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
    std::fill(stage_, stage_ + 64, 0.0);
    std::copy(prob_.params.begin(), prob_.params.begin() + std::min<size_t>(64, prob_.params.size()), stage_);
    KB_CUDA_CHECK(cudaMemcpyAsync(params_, stage_, 64 * 8, cudaMemcpyHostToDevice, stream_));
    bytes += 64 * 8;
    for (int l = 0; l <= L_; ++l) launch3_ftab(H_->lev[l], corners_, prob_.kind, params_, ftab_[l], stream_);
  }
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return bytes;
}

double* Solver3D::state(int which, int level) {
  if (level < 0 || level > L_) fail(KB_STRUCTURAL, "level out of range");
  if (which == 0) return u_[level];
  if (which == 1) return b_[level];
  if (which == 2) {
    if (level < 1) fail(KB_STRUCTURAL, "w lives on levels 1..L");
    return w_[level - 1];
  }
  fail(KB_STRUCTURAL, "unknown state component");
}

// ------------------------------------------------------------------ probes (as Solver2D)
void Solver3D::set_profiling(bool on) {
  if (on == profiling_) return;
  profiling_ = on;
  if (exec_) {
    cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
  }
  fmg_probes_.clear();
  est_probes_.clear();
}
cudaEvent_t Solver3D::event_at(int idx) {
  while (static_cast<int>(events_.size()) <= idx) {
    cudaEvent_t e;
    KB_CUDA_CHECK(cudaEventCreate(&e));
    events_.push_back(e);
  }
  return events_[idx];
}
void Solver3D::probe_begin(std::vector<Probe>* list) {
  probes_ = list;
  list->clear();
  if (!profiling_) return;
  next_event_ = (list == &fmg_probes_) ? 0 : 4096;
  last_event_ = next_event_++;
  cudaEvent_t e = event_at(last_event_);
  if (capturing_)
    KB_CUDA_CHECK(cudaEventRecordWithFlags(e, stream_, cudaEventRecordExternal));
  else
    KB_CUDA_CHECK(cudaEventRecord(e, stream_));
}
void Solver3D::mark(int kind, double bytes, int nlaunch) {
  launches_ += nlaunch;
  if (!profiling_ || !probes_) return;
  const int e = next_event_++;
  if (capturing_)
    KB_CUDA_CHECK(cudaEventRecordWithFlags(event_at(e), stream_, cudaEventRecordExternal));
  else
    KB_CUDA_CHECK(cudaEventRecord(event_at(e), stream_));
  probes_->push_back({kind, bytes, last_event_, e});
  last_event_ = e;
}
void Solver3D::kernel_stats(int kind, double* ms, int* launches, double* bytes) {
  double t = 0.0, b = 0.0;
  int c = 0;
  for (const auto* list : {&fmg_probes_, &est_probes_})
    for (const Probe& p : *list) {
      if (p.kind != kind && kind >= 0) continue;
      float f = 0.f;
      KB_CUDA_CHECK(cudaEventElapsedTime(&f, events_[p.ev0], events_[p.ev1]));
      t += f;
      b += p.bytes;
      ++c;
    }
  if (ms) *ms = t;
  if (launches) *launches = c;
  if (bytes) *bytes = b;
}

// ------------------------------------------------------------------ FMG
void Solver3D::vcycle(int l, double* u, const double* b) {
  const auto& lev = H_->lev;
  if (l == 0) {
    launch3_cg0(lev[0], u, b, cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
                status_, stream_);
    mark(KK_CG0, 0.0);
    return;
  }
  // algorithmic bytes per unique DoF: GS 24/sweep, residual 24,
  // restriction 8 fine + 8 coarse, prolongation+correction 16 fine + 8 coarse
  if (cfg_.pre_smooth > 0) {
    launch3_gs(lev[l], u, b, cfg_.pre_smooth, stream_);
    mark(KK_GS, 24.0 * cfg_.pre_smooth * dofs(l), launch3_gs_count(lev[l], cfg_.pre_smooth));
  }
  launch3_apply(lev[l], false, u, r_[l], b, A3_RES_OWNER, stream_);
  mark(KK_RESIDUAL, 24.0 * dofs(l), launch3_apply_count(lev[l]));
  // the restriction also writes the coarse level's zero initial guess (no memset node)
  launch3_restrict(lev[l], lev[l - 1], r_[l], vb_[l - 1], 1, stream_, vu_[l - 1]);
  mark(KK_RESTRICT, 8.0 * dofs(l) + 16.0 * dofs(l - 1), 2);
  vcycle(l - 1, vu_[l - 1], vb_[l - 1]);
  launch3_prolong(lev[l - 1], lev[l], vu_[l - 1], u, P3_ADD, stream_);
  mark(KK_PROLONG, 16.0 * dofs(l) + 8.0 * dofs(l - 1));
  if (cfg_.post_smooth > 0) {
    launch3_gs(lev[l], u, b, cfg_.post_smooth, stream_);
    mark(KK_GS, 24.0 * cfg_.post_smooth * dofs(l), launch3_gs_count(lev[l], cfg_.post_smooth));
  }
}

void Solver3D::enqueue_fmg_body() {
  const auto& lev = H_->lev;
  launches_ = 0;
  probe_begin(&fmg_probes_);
  KB_CUDA_CHECK(cudaMemsetAsync(status_, 0, sizeof(DevStatus), stream_));
  mark(KK_OTHER, 0.0, 0);
  for (int l = 0; l <= L_; ++l) {
    // b = M f_I, then the Dirichlet rows g
    if (has_source_) {
      launch3_apply(lev[l], true, ftab_[l], b_[l], nullptr, A3_PLAIN, stream_);
      launch3_set_boundary(lev[l], b_[l], gbnd_[l], 0, stream_);
      mark(KK_RHS, 16.0 * dofs(l), 1 + launch3_apply_count(lev[l]));
    } else {
      launch3_set_boundary(lev[l], b_[l], gbnd_[l], 1, stream_);
      mark(KK_RHS, 8.0 * dofs(l), 1);
    }
  }
  launch3_set_boundary(lev[0], u_[0], gbnd_[0], 1, stream_);
  mark(KK_OTHER, 8.0 * dofs(0));
  launch3_cg0(lev[0], u_[0], b_[0], cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
              status_, stream_);
  mark(KK_CG0, 0.0);
  for (int l = 0; l < L_; ++l) {
    // w[l] = P u[l] (snapshot before the Dirichlet reset); next = w with g on the boundary
    launch3_prolong(lev[l], lev[l + 1], u_[l], w_[l], P3_ASSIGN, stream_);
    KB_CUDA_CHECK(cudaMemcpyAsync(u_[l + 1], w_[l], level_size(l + 1) * 8, cudaMemcpyDeviceToDevice, stream_));
    launch3_set_boundary(lev[l + 1], u_[l + 1], gbnd_[l + 1], 0, stream_);
    mark(KK_PROLONG, 24.0 * dofs(l + 1) + 8.0 * dofs(l), 2);
    for (int c = 0; c < cfg_.nu; ++c) vcycle(l + 1, u_[l + 1], b_[l + 1]);
  }
  fmg_launches_ = launches_;
  probes_ = nullptr;
}

void Solver3D::fmg_enqueue() {
  if (L_ < 1) fail(KB_STRUCTURAL, "full multigrid requires at least one level above the coarse grid");
  if (!cfg_.use_graph) {
    enqueue_fmg_body();
    return;
  }
  if (!exec_) {
    cudaGraph_t graph = nullptr;
    KB_CUDA_CHECK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    capturing_ = true;
    try {
      enqueue_fmg_body();
    } catch (...) {
      capturing_ = false;
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    capturing_ = false;
    KB_CUDA_CHECK(cudaStreamEndCapture(stream_, &graph));
    KB_CUDA_CHECK(cudaGraphInstantiate(&exec_, graph, 0));
    cudaGraphDestroy(graph);
  }
  KB_CUDA_CHECK(cudaGraphLaunch(exec_, stream_));
}

void Solver3D::sync_and_check() {
  KB_CUDA_CHECK(cudaMemcpyAsync(status_host_, status_, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (status_host_->code) {
    Error e(KB_SOLVER, status_host_->code == 1 ? "coarse-grid CG did not converge"
                                               : "coarse-grid CG lost positive definiteness");
    e.residual = status_host_->residual;
    throw e;
  }
}

void Solver3D::fmg() {
  fmg_enqueue();
  sync_and_check();
}

// error_estimate (proj/src/estimator.cpp:8-45): e_base = u_L - P^(j-1) w[L-j],
// e_coarser = u_L - P^j w[L-j-1]
void Solver3D::estimate_enqueue(int offset) {
  if (offset < 1 || offset > L_ - 1) fail(KB_STRUCTURAL, "estimate offset must satisfy 1 <= j <= L-1");
  const auto& lev = H_->lev;
  const int base = L_ - offset;
  const int saved = launches_;
  probe_begin(&est_probes_);
  auto lift = [&](const double* src, int from_level, double* out) -> const double* {
    // prolongate from `from_level` to L through the scratch vectors
    const double* cur = src;
    for (int l = from_level; l < L_; ++l) {
      double* dst = (l + 1 == L_) ? out : (l % 2 ? vu_[l + 1] : vb_[l + 1]);
      launch3_prolong(lev[l], lev[l + 1], cur, dst, P3_ASSIGN, stream_);
      mark(KK_ESTIMATE, 8.0 * dofs(l + 1) + 8.0 * dofs(l));
      cur = dst;
    }
    return cur;
  };
  const double* wb = lift(w_[base], base + 1, est_a_);
  const double* wc = lift(w_[base - 1], base, est_b_);
  launch3_estimate(lev[L_], u_[L_], wb, wc, est_sums_, est_c_, stream_);  // est_c_: per-plane partials
  mark(KK_ESTIMATE, 24.0 * dofs(L_), launch3_estimate_count(lev[L_]));
  KB_CUDA_CHECK(cudaMemcpyAsync(sums_host_, est_sums_, 2 * H_->host.M * sizeof(double), cudaMemcpyDeviceToHost,
                                stream_));
  probes_ = nullptr;
  est_launches_ = launches_ - saved;
  launches_ = saved;
}

EstimateReport2D Solver3D::estimate_finish(int offset, int kind) {
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  const int M = H_->host.M;
  EstimateReport2D rep;
  rep.offset = offset;
  rep.base_level = L_ - offset;
  rep.kind = kind;
  double gb = 0.0, gc = 0.0;
  for (int s = 0; s < M; ++s) {
    gb += sums_host_[2 * s];
    gc += sums_host_[2 * s + 1];
  }
  rep.norm_base = std::sqrt(std::max(0.0, gb));
  rep.norm_coarser = std::sqrt(std::max(0.0, gc));
  rep.conv_factor = rep.norm_coarser > 0.0 ? rep.norm_base / rep.norm_coarser : 0.0;
  rep.eta = std::pow(rep.conv_factor, offset) * rep.norm_base;
  rep.eta_local.resize(M);
  const double floor = 1e-14 * rep.norm_coarser;
  for (int s = 0; s < M; ++s) {
    const double lb = std::sqrt(std::max(0.0, sums_host_[2 * s]));
    if (kind == 0) {
      rep.eta_local[s] = lb;
    } else {
      const double lc = std::sqrt(std::max(0.0, sums_host_[2 * s + 1]));
      rep.eta_local[s] = std::pow(lc > floor ? lb / lc : rep.conv_factor, offset) * lb;
    }
  }
  return rep;
}

// ------------------------------------------------------------------ single operations
void Solver3D::apply(int level, int op_mass, const double* x, double* y) {
  launch3_apply(H_->lev.at(level), op_mass != 0, x, y, nullptr, A3_PLAIN, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}
void Solver3D::residual(int level, const double* u, const double* b, double* r) {
  launch3_apply(H_->lev.at(level), false, u, r, b, A3_RESIDUAL, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}
void Solver3D::gauss_seidel(int level, double* u, const double* b, int sweeps) {
  if (level < 1) fail(KB_STRUCTURAL, "Gauss-Seidel runs on levels >= 1");
  launch3_gs(H_->lev.at(level), u, b, sweeps, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}
void Solver3D::restrict_to(int fine_level, const double* r, double* rc) {
  if (fine_level < 1) fail(KB_STRUCTURAL, "restriction below level 0");
  launch3_owner_mask(H_->lev.at(fine_level), r, est_c_, stream_);
  launch3_restrict(H_->lev.at(fine_level), H_->lev.at(fine_level - 1), est_c_, rc, 0, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}
void Solver3D::prolongate(int coarse_level, const double* c, double* f) {
  if (coarse_level + 1 > L_) fail(KB_STRUCTURAL, "prolongation beyond the finest level");
  launch3_prolong(H_->lev.at(coarse_level), H_->lev.at(coarse_level + 1), c, f, P3_ASSIGN, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}
void Solver3D::cg_level0(double* u, const double* b) {
  KB_CUDA_CHECK(cudaMemsetAsync(status_, 0, sizeof(DevStatus), stream_));
  launch3_cg0(H_->lev.at(0), u, b, cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
              status_, stream_);
  sync_and_check();
}
double Solver3D::dot_unique(int level, const double* a, const double* b) {
  launch3_dot(H_->lev.at(level), a, b, dot_partial_, dot_out_, stream_);
  double out = 0.0;
  KB_CUDA_CHECK(cudaMemcpyAsync(&out, dot_out_, 8, cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return out;
}
void Solver3D::interface_sync(int level, double* f, int additive) {
  launch3_sync(H_->lev.at(level), f, additive, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

}  // namespace kb
