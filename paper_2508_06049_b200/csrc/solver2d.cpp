// Host orchestration of the 2-d hot path.  See solver2d.hpp.
#include "solver2d.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>

namespace kb {

// ------------------------------------------------------------------ arena
// The arenas come from the device's default stream-ordered memory pool with
// the release threshold lifted, so an AMR loop that rebuilds hierarchy and
// solver per step reuses the freed blocks instead of paying cudaMalloc /
// cudaFree (2 - 40 ms per 100 MB arena, measured) every time.  The allocation
// is made usable from every stream by synchronising the allocating (legacy
// default) stream; the free is preceded by a device synchronise, like cudaFree.
namespace {
bool arena_pool_ready() {
  static const bool ok = [] {
    const char* e = getenv("KB_ARENA_POOL");
    if (e && e[0] == '0') return false;
    int dev = 0, supported = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    if (cudaDeviceGetAttribute(&supported, cudaDevAttrMemoryPoolsSupported, dev) != cudaSuccess || !supported) {
      cudaGetLastError();
      return false;
    }
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    unsigned long long keep = ~0ull;
    if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return true;
  }();
  return ok;
}
}  // namespace

DeviceArena::~DeviceArena() {
  if (!base_) return;
  if (pooled_) {
    cudaDeviceSynchronize();
    cudaFreeAsync(base_, nullptr);
  } else {
    cudaFree(base_);
  }
}

void DeviceArena::reserve(size_t bytes) {
  if (base_) fail(KB_INTERNAL, "arena already reserved");
  cap_ = bytes + 256;
  cudaError_t e;
  if (cap_ <= (size_t(1) << 30) && arena_pool_ready()) {  // large arenas: plain cudaMalloc (nothing retained)
    e = cudaMallocAsync(reinterpret_cast<void**>(&base_), cap_, nullptr);
    if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
    pooled_ = e == cudaSuccess;
  } else {
    e = cudaMalloc(&base_, cap_);
  }
  if (e != cudaSuccess) {
    base_ = nullptr;
    Error err(KB_RESOURCE, std::string("device allocation failed: ") + cudaGetErrorString(e));
    throw err;
  }
  used_ = 0;
}

void* DeviceArena::take(size_t bytes) {
  const size_t off = (used_ + 255) & ~static_cast<size_t>(255);
  if (off + bytes > cap_) fail(KB_INTERNAL, "device arena exhausted");
  used_ = off + bytes;
  return base_ + off;
}


namespace {
size_t round256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }
template <typename T>
size_t vbytes(const std::vector<T>& v) {
  return round256(v.size() * sizeof(T));
}
}  // namespace

// ------------------------------------------------------------------ hierarchy upload
std::unique_ptr<DeviceHierarchy2D> DeviceHierarchy2D::create(const Mesh2D& mesh, int max_level) {
  auto d = std::make_unique<DeviceHierarchy2D>();
  const auto tc0 = std::chrono::steady_clock::now();
  d->host = Hierarchy2D::build(mesh, max_level);
  const auto tc1 = std::chrono::steady_clock::now();
  const Hierarchy2D& h = d->host;
  const int M = h.M;
  std::vector<std::vector<int>> mem_off(h.L + 1), mem_ij(h.L + 1);
  std::vector<std::vector<double>> geo(h.L + 1), wq(h.L + 1);
  size_t bytes = vbytes(h.nb_lo_ptr) + vbytes(h.nb_lo) + vbytes(h.nb_hi_ptr) + vbytes(h.nb_hi) +
                 vbytes(h.dag_ptr) + vbytes(h.dag_list);
  for (int l = 0; l <= h.L; ++l) {
    const Level2D& lv = h.levels[l];
    const int n = lv.n;
    for (size_t k = 0; k < lv.mem_slot.size(); ++k) {
      mem_off[l].push_back(lv.mem_slot[k] * lv.S + lv.mem_idx[k]);
      mem_ij[l].push_back(lv.mem_i[k] | (lv.mem_j[k] << 16));
    }
    for (int s = 0; s < M; ++s) {
      const auto& v = mesh.tri[s];
      // RHS quadrature map, proj/src/fem.cpp:183-186
      geo[l].push_back(mesh.x[v[0]]);
      geo[l].push_back(mesh.y[v[0]]);
      geo[l].push_back((mesh.x[v[1]] - mesh.x[v[0]]) / n);
      geo[l].push_back((mesh.y[v[1]] - mesh.y[v[0]]) / n);
      geo[l].push_back((mesh.x[v[2]] - mesh.x[v[0]]) / n);
      geo[l].push_back((mesh.y[v[2]] - mesh.y[v[0]]) / n);
      const double cell_area = mesh.area[s] / (static_cast<double>(n) * n);
      wq[l].push_back(cell_area / 3.0);
    }
    bytes += vbytes(lv.node_gid) + vbytes(lv.node_flags) + vbytes(lv.grp_ptr) + vbytes(mem_off[l]) +
             vbytes(mem_ij[l]) + vbytes(lv.mem_slot) + vbytes(lv.kstiff) + vbytes(lv.kmass) +
             vbytes(lv.stencil) + vbytes(lv.inv_c) + vbytes(lv.bnode) + vbytes(lv.rec) + vbytes(lv.wr) +
             vbytes(lv.ghost_ptr) + vbytes(lv.ghost_off) + vbytes(lv.dot_order) + vbytes(geo[l]) +
             vbytes(wq[l]) + vbytes(lv.prog) + vbytes(lv.prog_ptr) + vbytes(lv.prog_extra) + vbytes(lv.xtra_ptr) +
             vbytes(lv.sc_cell_copy) + vbytes(lv.sc_copy_cell) + vbytes(lv.sc_mtab) + vbytes(lv.sc_gtab) +
             vbytes(lv.sched[0].blocks) + vbytes(lv.sched[0].lev_off) + vbytes(lv.sched[1].blocks) +
             vbytes(lv.sched[1].lev_off) + vbytes(lv.pipe.rec);
  }
  // level-0 CG tables (k_cg0): the gather of OperatorP1::apply at n = 1 -- every
  // node is a macro corner whose one cell up(0,0) contributes row r (its role)
  // of K_up, proj/src/fem.cpp:106-115 -- expressed over the unique DoF in the
  // owner order of dot_unique (proj/src/hhg.cpp:227-257)
  std::vector<int> cg_mem_ptr, cg_mem_dof, cg_copy_ptr, cg_copy;
  std::vector<double> cg_mem_coef;
  {
    const Level2D& l0 = h.levels[0];
    const int cnt = static_cast<int>(l0.dot_order.size());
    std::vector<int> dof_of_group(l0.grp_ptr.size(), -1);
    for (int dd = 0; dd < cnt; ++dd) {
      const int g = l0.node_gid[l0.dot_order[dd]];
      if (g < 0) fail(KB_INTERNAL, "level-0 node outside a group");
      dof_of_group[g] = dd;
    }
    auto dof_of_copy = [&](int k) {
      const int g = l0.node_gid[k];
      if (g < 0 || dof_of_group[g] < 0) fail(KB_INTERNAL, "level-0 copy without a DoF");
      return dof_of_group[g];
    };
    cg_mem_ptr.push_back(0);
    cg_copy_ptr.push_back(0);
    for (int dd = 0; dd < cnt; ++dd) {
      const int g = l0.node_gid[l0.dot_order[dd]];
      for (int q = l0.grp_ptr[g]; q < l0.grp_ptr[g + 1]; ++q) {
        const int slot = l0.mem_slot[q];
        const int role = l0.mem_j[q] == 1 ? 2 : l0.mem_i[q];  // (0,0) a, (1,0) b, (0,1) c
        for (int c = 0; c < 3; ++c) {
          cg_mem_coef.push_back(l0.kstiff[18 * static_cast<size_t>(slot) + 3 * role + c]);
          cg_mem_dof.push_back(dof_of_copy(slot * l0.S + c));  // lattice index of corner c at n = 1
        }
        cg_copy.push_back(slot * l0.S + l0.mem_idx[q]);
      }
      cg_mem_ptr.push_back(static_cast<int>(cg_mem_coef.size() / 3));
      cg_copy_ptr.push_back(static_cast<int>(cg_copy.size()));
    }
    bytes += vbytes(cg_mem_ptr) + vbytes(cg_mem_dof) + vbytes(cg_copy_ptr) + vbytes(cg_copy) + vbytes(cg_mem_coef);
  }
  const auto tc2 = std::chrono::steady_clock::now();
  d->arena.reserve(bytes + 4096);
  const auto tc3 = std::chrono::steady_clock::now();
  d->dh.M = M;
  d->dh.L = h.L;
  d->dh.nb_lo_ptr = d->arena.upload(h.nb_lo_ptr);
  d->dh.nb_lo = d->arena.upload(h.nb_lo);
  d->dh.nb_hi_ptr = d->arena.upload(h.nb_hi_ptr);
  d->dh.nb_hi = d->arena.upload(h.nb_hi);
  d->dh.dag_depth = h.dag_depth;
  d->dh.dag_width = 0;
  for (int k = 0; k < h.dag_depth; ++k) d->dh.dag_width = std::max(d->dh.dag_width, h.dag_ptr[k + 1] - h.dag_ptr[k]);
  d->dh.dag_ptr = d->arena.upload(h.dag_ptr);
  d->dh.dag_list = d->arena.upload(h.dag_list);
  for (int l = 0; l <= h.L; ++l) {
    const Level2D& lv = h.levels[l];
    DevLevel2D dl{};
    dl.n = lv.n;
    dl.S = lv.S;
    dl.M = M;
    dl.node_gid = d->arena.upload(lv.node_gid);
    dl.node_flags = d->arena.upload(lv.node_flags);
    dl.grp_ptr = d->arena.upload(lv.grp_ptr);
    dl.mem_off = d->arena.upload(mem_off[l]);
    dl.mem_ij = d->arena.upload(mem_ij[l]);
    dl.mem_slot = d->arena.upload(lv.mem_slot);
    dl.kstiff = d->arena.upload(lv.kstiff);
    dl.kmass = d->arena.upload(lv.kmass);
    dl.stencil = d->arena.upload(lv.stencil);
    dl.inv_c = d->arena.upload(lv.inv_c);
    dl.bnode = d->arena.upload(lv.bnode);
    dl.rec = d->arena.upload(lv.rec);
    dl.wr = d->arena.upload(lv.wr);
    dl.ghost_ptr = d->arena.upload(lv.ghost_ptr);
    dl.ghost_off = d->arena.upload(lv.ghost_off);
    dl.max_ghosts = lv.max_ghosts;
    dl.num_groups = static_cast<int>(lv.grp_ptr.size()) - 1;
    dl.dot_order = d->arena.upload(lv.dot_order);
    dl.dot_count = static_cast<int>(lv.dot_order.size());
    dl.prog = reinterpret_cast<const unsigned long long*>(d->arena.upload(lv.prog));
    dl.prog_ptr = d->arena.upload(lv.prog_ptr);
    dl.prog_extra = reinterpret_cast<const unsigned long long*>(d->arena.upload(lv.prog_extra));
    dl.xtra_ptr = d->arena.upload(lv.xtra_ptr);
    dl.max_extra = lv.max_extra;
    if (l == 0) {
      dl.cg_nmem = static_cast<int>(cg_mem_coef.size() / 3);
      dl.cg_ncopy = static_cast<int>(cg_copy.size());
      dl.cg_mem_ptr = d->arena.upload(cg_mem_ptr);
      dl.cg_mem_dof = d->arena.upload(cg_mem_dof);
      dl.cg_mem_coef = d->arena.upload(cg_mem_coef);
      dl.cg_copy_ptr = d->arena.upload(cg_copy_ptr);
      dl.cg_copy = d->arena.upload(cg_copy);
    }
    dl.geo = d->arena.upload(geo[l]);
    dl.wq = d->arena.upload(wq[l]);
    if (lv.pipe.ok) {
      dl.pipe_rec = d->arena.upload(lv.pipe.rec);
      dl.pipe_rec_words = lv.pipe.rec_words;
      dl.pipe_maxreq = lv.pipe.maxreq;
    }
    dl.sc_nu = lv.sc_nu;
    if (lv.sc_nu > 0) {
      dl.sc_cell_copy = d->arena.upload(lv.sc_cell_copy);
      dl.sc_copy_cell = d->arena.upload(lv.sc_copy_cell);
      dl.sc_mtab = d->arena.upload(lv.sc_mtab);
      dl.sc_gtab = d->arena.upload(lv.sc_gtab);
      for (int q = 0; q < 2; ++q) {
        dl.sc_blocks[q] = d->arena.upload(lv.sched[q].blocks);
        dl.sc_lev_off[q] = d->arena.upload(lv.sched[q].lev_off);
        dl.sc_levels[q] = lv.sched[q].levels;
        dl.sc_max_width[q] = lv.sched[q].max_width;
        dl.sc_max_block[q] = lv.sched[q].max_block_words;
        dl.sc_max_members[q] = lv.sched[q].max_members;
      }
    }
    d->lev.push_back(dl);
  }
  if (getenv("KB_BUILD_TRACE")) {
    auto ms = [](auto a, auto b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
    fprintf(stderr, "device hierarchy: host build %.1f ms, host tables %.1f ms, arena %.1f ms (%zu MB), upload %.1f ms\n",
            ms(tc0, tc1), ms(tc1, tc2), ms(tc2, tc3), bytes >> 20, ms(tc3, std::chrono::steady_clock::now()));
  }
  return d;
}

// ------------------------------------------------------------------ problems
Problem2D Problem2D::builtin(int kind) {
  Problem2D p;
  p.kind = kind;
  switch (kind) {
    case PROB_ZERO:
      p.source = p.boundary = p.exact = [](double, double) { return 0.0; };
      p.has_exact = true;
      break;
    case PROB_SIN2D:
      // BASELINE.json config 1: u = sin(pi x) sin(pi y), f = 2 pi^2 u
      p.exact = [](double x, double y) { return std::sin(M_PI * x) * std::sin(M_PI * y); };
      p.source = [](double x, double y) {
        return 2.0 * M_PI * M_PI * std::sin(M_PI * x) * std::sin(M_PI * y);
      };
      p.boundary = p.exact;
      p.has_exact = true;
      break;
    case PROB_LSHAPE:
      // make_lshape_spec, proj/src/problems.cpp:36-53
      p.exact = [](double x, double y) {
        const double r = std::hypot(x, y);
        if (r == 0.0) return 0.0;
        double phi = std::atan2(y, x);
        if (phi < 0.0) phi += 2.0 * M_PI;
        return std::pow(r, 2.0 / 3.0) * std::sin(2.0 * phi / 3.0);
      };
      p.source = [](double, double) { return 0.0; };
      p.boundary = p.exact;
      p.has_exact = true;
      break;
    default:
      fail(KB_STRUCTURAL, "unknown built-in problem kind");
  }
  return p;
}

// ------------------------------------------------------------------ solver
Solver2D::Solver2D(std::shared_ptr<DeviceHierarchy2D> h, Problem2D p, SolverConfig2D cfg)
    : H_(std::move(h)), prob_(std::move(p)), cfg_(cfg) {
  const Hierarchy2D& hh = H_->host;
  L_ = hh.L;
  const int M = hh.M;
  if (cfg_.finest_policy < 0 || cfg_.finest_policy > 2) fail(KB_STRUCTURAL, "unknown finest-level policy");
  if (prob_.kind == PROB_ZERO || prob_.kind == PROB_LSHAPE)
    src_kind_ = SRC_ZERO;
  else if (prob_.kind == PROB_SIN2D && !cfg_.faithful_source)
    src_kind_ = SRC_SIN2D;
  else
    src_kind_ = SRC_TABLE;

  auto lsize = [&](int l) { return static_cast<size_t>(M) * hh.levels[l].S; };
  auto fsize = [&](int l) {
    const size_t n2 = 2 * static_cast<size_t>(hh.levels[l].n);
    return static_cast<size_t>(M) * (n2 + 1) * (n2 + 2) / 2;
  };
  size_t bytes = 0;
  for (int l = 0; l <= L_; ++l) {
    bytes += 2 * round256(lsize(l) * 8);                               // u, b
    if (l < L_) bytes += round256(lsize(l + 1) * 8) + 2 * round256(lsize(l) * 8);  // w, vu, vb
    if (l >= 1) bytes += round256(lsize(l) * 8);                       // r
    bytes += round256(static_cast<size_t>(M) * 3 * hh.levels[l].n * 8);  // gbnd
    if (src_kind_ != SRC_ZERO) bytes += round256(fsize(l) * 8);
  }
  bytes += round256(3 * lsize(0) * 8) + round256(2 * M * 8) + round256(lsize(L_) * 8) +
           round256(lsize(std::max(L_ - 1, 0)) * 8) + round256(64 * 8) + round256(8) +
           round256(sizeof(DevStatus)) + round256((M + 3) / 4 * 16);
  const auto ts0 = std::chrono::steady_clock::now();
  arena_.reserve(bytes);
  const auto ts1 = std::chrono::steady_clock::now();
  u_.assign(L_ + 1, nullptr);
  b_.assign(L_ + 1, nullptr);
  w_.assign(L_ + 1, nullptr);
  vu_.assign(L_ + 1, nullptr);
  vb_.assign(L_ + 1, nullptr);
  r_.assign(L_ + 1, nullptr);
  gbnd_.assign(L_ + 1, nullptr);
  ftab_.assign(L_ + 1, nullptr);
  for (int l = 0; l <= L_; ++l) {
    u_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    b_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    if (l < L_) {
      w_[l] = static_cast<double*>(arena_.take(lsize(l + 1) * 8));
      vu_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
      vb_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    }
    if (l >= 1) r_[l] = static_cast<double*>(arena_.take(lsize(l) * 8));
    gbnd_[l] = static_cast<double*>(arena_.take(static_cast<size_t>(M) * 3 * hh.levels[l].n * 8));
    if (src_kind_ != SRC_ZERO) ftab_[l] = static_cast<double*>(arena_.take(fsize(l) * 8));
  }
  cg_scratch_ = static_cast<double*>(arena_.take(3 * lsize(0) * 8));
  est_sums_ = static_cast<double*>(arena_.take(2 * M * 8));
  est_tmp_a_ = static_cast<double*>(arena_.take(lsize(L_) * 8));
  est_tmp_b_ = static_cast<double*>(arena_.take(lsize(std::max(L_ - 1, 0)) * 8));
  dot_partial_ = static_cast<double*>(arena_.take(64 * 8));
  dot_out_ = static_cast<double*>(arena_.take(8));
  status_ = static_cast<DevStatus*>(arena_.take(sizeof(DevStatus)));
  gs_done_ = static_cast<int*>(arena_.take((M + 3) / 4 * 16));  // k_gs_pipe polls 16-byte chunks

  KB_CUDA_CHECK(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  stream_ = own_stream_;
  KB_CUDA_CHECK(cudaMallocHost(&status_host_, sizeof(DevStatus)));
  KB_CUDA_CHECK(cudaMallocHost(&sums_host_, 2 * M * sizeof(double)));

  gbnd_count_.assign(L_ + 1, 0);
  ftab_count_.assign(L_ + 1, 0);
  for (int l = 0; l <= L_; ++l) {
    gbnd_count_[l] = static_cast<size_t>(M) * 3 * hh.levels[l].n;
    if (src_kind_ == SRC_TABLE) ftab_count_[l] = fsize(l);
    stage_count_ += gbnd_count_[l] + ftab_count_[l];
  }
  const auto ts2 = std::chrono::steady_clock::now();
  // small staging buffers are pinned; a large source table (tens of MB) goes
  // through pageable memory (pinning it costs more than the staged copy saves)
  stage_pinned_ = stage_count_ * sizeof(double) <= (8u << 20);
  if (stage_pinned_) {
    KB_CUDA_CHECK(cudaMallocHost(&stage_, stage_count_ * sizeof(double)));
  } else {
    stage_ = static_cast<double*>(std::malloc(stage_count_ * sizeof(double)));
    if (!stage_) fail(KB_RESOURCE, "host allocation of the problem tables failed");
  }
  const auto ts3 = std::chrono::steady_clock::now();
  load_problem(prob_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (getenv("KB_BUILD_TRACE")) {
    auto ms = [](auto a, auto b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
    fprintf(stderr, "solver: arena %.1f ms (%zu MB), misc %.1f ms, pinned stage %.1f ms (%zu MB), tabulate + copy %.1f ms\n",
            ms(ts0, ts1), bytes >> 20, ms(ts1, ts2), ms(ts2, ts3), (stage_count_ * 8) >> 20,
            ms(ts3, std::chrono::steady_clock::now()));
  }
  KB_CUDA_CHECK(cudaMemset(status_, 0, sizeof(DevStatus)));
}

Solver2D::~Solver2D() {
  if (exec_) cudaGraphExecDestroy(exec_);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  if (own_stream_) cudaStreamDestroy(own_stream_);
  if (status_host_) cudaFreeHost(status_host_);
  if (sums_host_) cudaFreeHost(sums_host_);
  if (stage_) {
    if (stage_pinned_) cudaFreeHost(stage_);
    else std::free(stage_);
  }
}

void Solver2D::tabulate(const Problem2D& p) {
  // Dirichlet data: g at the owner copy's node coordinates for every
  // domain-boundary copy (set_domain_boundary_values + ReplaceFromOwner,
  // proj/src/fem.cpp:212-228), evaluated with the host libm like the reference.
  const Hierarchy2D& hh = H_->host;
  const int M = hh.M;
  double* dst = stage_;
  for (int l = 0; l <= L_; ++l) {
    const Level2D& lv = hh.levels[l];
    const int n = lv.n;
    double* g = dst;
    std::fill(g, g + gbnd_count_[l], 0.0);
    // the problem's callbacks are evaluated macro-parallel on host threads (pure
    // functions of (x, y) like the reference's problems; KB_HOST_THREADS=0: in order)
    parallel_for(M, [&](int s) {
      auto visit = [&](int i, int j) {
        if (!hh.on_domain_boundary(s, l, i, j)) return;
        const int gid = hh.boundary_group(s, l, i, j);
        const int first = lv.grp_ptr[gid];
        double x, y;
        hh.node_coordinates(lv.mem_slot[first], l, lv.mem_i[first], lv.mem_j[first], x, y);
        g[static_cast<size_t>(s) * 3 * n + bpos(n, i, j)] = p.boundary(x, y);
      };
      for (int i = 0; i <= n; ++i) visit(i, 0);
      for (int j = 1; j <= n; ++j) visit(0, j);
      for (int j = 1; j <= n - 1; ++j) visit(n - j, j);
    }, gbnd_count_[l] >= 20000);
    dst += gbnd_count_[l];
    if (ftab_count_[l]) {
      // f at the cell edge midpoints through the RHS map (proj/src/fem.cpp:183-194)
      const int n2 = 2 * n;
      const int SF = lattice_size(n2);
      double* f = dst;
      std::fill(f, f + ftab_count_[l], 0.0);
      parallel_for(M, [&](int s) {
        const auto& v = hh.mesh.tri[s];
        const double c0x = hh.mesh.x[v[0]], c0y = hh.mesh.y[v[0]];
        const double ux = (hh.mesh.x[v[1]] - c0x) / n, uy = (hh.mesh.y[v[1]] - c0y) / n;
        const double wx = (hh.mesh.x[v[2]] - c0x) / n, wy = (hh.mesh.y[v[2]] - c0y) / n;
        for (int J = 0; J <= n2; ++J)
          for (int I = 0; I <= n2 - J; ++I) {
            if (((I | J) & 1) == 0) continue;  // only edge midpoints are used
            const double hi = 0.5 * I, hj = 0.5 * J;
            f[static_cast<size_t>(s) * SF + lattice_index(n2, I, J)] =
                p.source(c0x + hi * ux + hj * wx, c0y + hi * uy + hj * wy);
          }
      }, ftab_count_[l] >= 20000);
      dst += ftab_count_[l];
    }
  }
}

size_t Solver2D::load_problem(const Problem2D& p) {
  // the device source path (table / zero / device-evaluated) was fixed at construction
  if (p.kind != prob_.kind) fail(KB_STRUCTURAL, "set_problem: the problem kind must match the solver's");
  if (&p != &prob_) prob_ = p;
  ex_moments_ = nullptr;  // the exact-error moments belong to the previous problem
  ex_arena_.reset();
  // the staging buffer may still feed an earlier copy
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  tabulate(prob_);
  size_t bytes = 0;
  const double* src = stage_;
  for (int l = 0; l <= L_; ++l) {
    KB_CUDA_CHECK(cudaMemcpyAsync(gbnd_[l], src, gbnd_count_[l] * 8, cudaMemcpyHostToDevice, stream_));
    src += gbnd_count_[l];
    bytes += gbnd_count_[l] * 8;
    if (ftab_count_[l]) {
      KB_CUDA_CHECK(cudaMemcpyAsync(ftab_[l], src, ftab_count_[l] * 8, cudaMemcpyHostToDevice, stream_));
      src += ftab_count_[l];
      bytes += ftab_count_[l] * 8;
    }
  }
  return bytes;
}

void Solver2D::set_stream(cudaStream_t st) { stream_ = st ? st : own_stream_; }

void Solver2D::set_profiling(bool on) {
  if (on == profiling_) return;
  profiling_ = on;
  if (exec_) {
    cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
  }
  fmg_probes_.clear();
  est_probes_.clear();
}

cudaEvent_t Solver2D::event_at(int idx) {
  while (static_cast<int>(events_.size()) <= idx) {
    cudaEvent_t e;
    KB_CUDA_CHECK(cudaEventCreate(&e));
    events_.push_back(e);
  }
  return events_[idx];
}

static void record_event(cudaEvent_t e, cudaStream_t st, bool capturing) {
  if (capturing)
    KB_CUDA_CHECK(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
  else
    KB_CUDA_CHECK(cudaEventRecord(e, st));
}

void Solver2D::probe_begin(std::vector<Probe>* list) {
  probes_ = list;
  list->clear();
  if (!profiling_) return;
  // FMG probes use events [0, 1024); estimator probes start at 1024
  next_event_ = (list == &fmg_probes_) ? 0 : 1024;
  last_event_ = next_event_++;
  record_event(event_at(last_event_), stream_, capturing_);
}

void Solver2D::mark(int kind, double bytes, int nlaunch) {
  launches_ += nlaunch;
  if (!profiling_ || !probes_) return;
  const int e = next_event_++;
  record_event(event_at(e), stream_, capturing_);
  probes_->push_back({kind, bytes, last_event_, e});
  last_event_ = e;
}

void Solver2D::kernel_stats(int kind, double* ms, int* launches, double* bytes) {
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

size_t Solver2D::level_size(int level) const {
  return static_cast<size_t>(H_->host.M) * H_->host.levels.at(level).S;
}

double* Solver2D::state(int which, int level) {
  if (level < 0 || level > L_) fail(KB_STRUCTURAL, "level out of range");
  if (which == 0) return u_[level];
  if (which == 1) return b_[level];
  if (which == 2) {
    if (level < 1) fail(KB_STRUCTURAL, "w lives on levels 1..L");
    return w_[level - 1];
  }
  fail(KB_STRUCTURAL, "unknown state component");
}

void Solver2D::vcycle(int l, double* u, const double* b) {
  // v_cycle, proj/src/multigrid.cpp:231-246
  const auto& lev = H_->lev;
  if (l == 0) {
    launch_cg0(lev[0], u, b, cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
               status_, stream_);
    mark(KK_CG0, 0.0);
    return;
  }
  // algorithmic bytes per unique DoF: GS 24/sweep, residual 24,
  // restriction 8 fine + 8 coarse, prolongation+correction 16 fine + 8 coarse
  if (cfg_.pre_smooth > 0) {
    launch_gs(H_->dh, lev[l], u, b, cfg_.pre_smooth, gs_done_, stream_);
    mark(KK_GS, 24.0 * cfg_.pre_smooth * dofs(l));
  }
  launch_apply(lev[l], lev[l].kstiff, u, r_[l], b, APPLY_RESIDUAL, stream_);
  mark(KK_RESIDUAL, 24.0 * dofs(l));
  // the restriction also writes the coarse level's zero initial guess (no memset node)
  launch_restrict(lev[l], lev[l - 1], r_[l], vb_[l - 1], 1, stream_, vu_[l - 1]);
  mark(KK_RESTRICT, 8.0 * dofs(l) + 16.0 * dofs(l - 1));
  vcycle(l - 1, vu_[l - 1], vb_[l - 1]);
  launch_prolong(lev[l - 1], lev[l], vu_[l - 1], u, nullptr, nullptr, PROLONG_ADD, stream_);
  mark(KK_PROLONG, 16.0 * dofs(l) + 8.0 * dofs(l - 1));
  if (cfg_.post_smooth > 0) {
    launch_gs(H_->dh, lev[l], u, b, cfg_.post_smooth, gs_done_, stream_);
    mark(KK_GS, 24.0 * cfg_.post_smooth * dofs(l));
  }
}

void Solver2D::enqueue_fmg_body() {
  // MultigridSolver::fmg, proj/src/multigrid.cpp:248-279
  const auto& lev = H_->lev;
  launches_ = 0;
  probe_begin(&fmg_probes_);
  KB_CUDA_CHECK(cudaMemsetAsync(status_, 0, sizeof(DevStatus), stream_));
  mark(KK_OTHER, 0.0, 0);
  for (int l = 0; l <= L_; ++l) {
    launch_rhs(lev[l], src_kind_, ftab_[l], ftab_[l], gbnd_[l], b_[l], stream_);
    // write b (8 B/DoF) + read the f table (4 midpoints per node) when one is used
    mark(KK_RHS, 8.0 * dofs(l) + (src_kind_ == SRC_TABLE ? 32.0 * dofs(l) : 0.0), src_kind_ == SRC_SIN2D ? 2 : 1);
  }
  launch_set_boundary(lev[0], u_[0], gbnd_[0], 1, stream_);
  mark(KK_OTHER, 8.0 * dofs(0));
  launch_cg0(lev[0], u_[0], b_[0], cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
             status_, stream_);
  mark(KK_CG0, 0.0);
  for (int l = 0; l < L_; ++l) {
    // w[l] = P u[l] (snapshot before the Dirichlet reset); next = w with g on the boundary
    launch_prolong(lev[l], lev[l + 1], u_[l], w_[l], u_[l + 1], gbnd_[l + 1], PROLONG_W_NEXT, stream_);
    mark(KK_PROLONG, 16.0 * dofs(l + 1) + 8.0 * dofs(l));
    for (int c = 0; c < cfg_.nu; ++c) vcycle(l + 1, u_[l + 1], b_[l + 1]);
  }
  fmg_launches_ = launches_;
  probes_ = nullptr;
}

void Solver2D::fmg_enqueue() {
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

void Solver2D::sync_and_check() {
  KB_CUDA_CHECK(cudaMemcpyAsync(status_host_, status_, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (status_host_->code == 1) {
    Error e(KB_SOLVER, "coarse-grid CG did not converge");
    e.residual = status_host_->residual;
    throw e;
  }
  if (status_host_->code == 2) {
    Error e(KB_SOLVER, "coarse-grid CG lost positive definiteness");
    e.residual = status_host_->residual;
    throw e;
  }
}

int Solver2D::last_cg_iters() const { return status_host_ ? status_host_->iters : 0; }

void Solver2D::fmg() {
  fmg_enqueue();
  sync_and_check();
  extra_cycles_ = 0;
  // FinestPolicy::ValidationTwoDigits, proj/src/multigrid.cpp:282-293: extra
  // finest V-cycles until the leading two digits of ||u - u_L|| settle
  if (cfg_.finest_policy == 1 && prob_.has_exact) {
    auto round_two_digits = [](double x) {  // proj/src/multigrid.cpp:13-18
      if (x == 0.0 || !std::isfinite(x)) return x;
      const double e = std::floor(std::log10(std::abs(x)));
      const double scale = std::pow(10.0, e - 1.0);
      return std::round(x / scale) * scale;
    };
    double prev = round_two_digits(exact_error().global);
    for (int extra = 0; extra < cfg_.max_extra_cycles; ++extra) {
      if (prev == 0.0 || prev < 1e-14) break;
      vcycle(L_, u_[L_], b_[L_]);
      sync_and_check();
      ++extra_cycles_;
      const double cur = round_two_digits(exact_error().global);
      if (cur == prev) break;
      prev = cur;
    }
  } else if (cfg_.finest_policy == 2) {
    finest_residual_vs_estimate();
  }
}

double* Solver2D::scratch(int slot, int level) {
  if (scr_level_ != level) {
    scr_arena_ = std::make_unique<DeviceArena>();
    scr_arena_->reserve(4 * (level_size(level) * 8 + 256) + 256);
    scr_.assign(4, nullptr);
    for (auto& p : scr_) p = static_cast<double*>(scr_arena_->take(level_size(level) * 8));
    scr_level_ = level;
  }
  return scr_.at(slot);
}

// l2_norm (proj/src/fem.cpp:320-325): sqrt(max(0, dot_unique(f, M f)))
double Solver2D::l2_norm_mass(int level, const double* f, double* tmp) {
  const auto& lv = H_->lev[level];
  launch_apply(lv, lv.kmass, f, tmp, nullptr, APPLY_PLAIN, stream_);
  return std::sqrt(std::max(0.0, dot_unique(level, f, tmp)));
}

// FinestPolicy::ResidualVsEstimate, proj/src/multigrid.cpp:294-319: eta_1 from
// the stored coarse solutions, then extra finest V-cycles until the mass norm
// of the update falls below 1e-2 eta_1
void Solver2D::finest_residual_vs_estimate() {
  const auto& lev = H_->lev;
  const size_t N = level_size(L_);
  double* e = scratch(0, L_);
  double* mf = scratch(1, L_);
  double* before = scratch(2, L_);
  double* pc = scratch(3, L_);
  double eta1 = 0.0;
  if (L_ >= 2) {
    // e_fine = u_L + (-1) w[L-1]
    KB_CUDA_CHECK(cudaMemcpyAsync(e, u_[L_], N * 8, cudaMemcpyDeviceToDevice, stream_));
    launch_axpy(e, w_[L_ - 1], -1.0, static_cast<std::int64_t>(N), stream_);
    const double n_fine = l2_norm_mass(L_, e, mf);
    // e_coarse = u_L + (-1) prolongate_to(w[L-2], L) (w[L-2] lives on level L-1)
    launch_prolong(lev[L_ - 1], lev[L_], w_[L_ - 2], pc, nullptr, nullptr, PROLONG_ASSIGN, stream_);
    KB_CUDA_CHECK(cudaMemcpyAsync(e, u_[L_], N * 8, cudaMemcpyDeviceToDevice, stream_));
    launch_axpy(e, pc, -1.0, static_cast<std::int64_t>(N), stream_);
    const double n_coarse = l2_norm_mass(L_, e, mf);
    eta1 = n_coarse > 0.0 ? (n_fine / n_coarse) * n_fine : 0.0;
  }
  for (int extra = 0; extra < cfg_.max_extra_cycles; ++extra) {
    KB_CUDA_CHECK(cudaMemcpyAsync(before, u_[L_], N * 8, cudaMemcpyDeviceToDevice, stream_));
    vcycle(L_, u_[L_], b_[L_]);
    sync_and_check();
    ++extra_cycles_;
    // delta = u_L + (-1) before
    KB_CUDA_CHECK(cudaMemcpyAsync(e, u_[L_], N * 8, cudaMemcpyDeviceToDevice, stream_));
    launch_axpy(e, before, -1.0, static_cast<std::int64_t>(N), stream_);
    const double update = l2_norm_mass(L_, e, mf);
    const double target = eta1 > 0.0 ? 1e-2 * eta1 : 1e-10 * std::max(1.0, l2_norm_mass(L_, u_[L_], mf));
    if (update < target) break;
  }
}

// dot_unique with the reference's sequential summation order (solve_direct's
// level CG: its iterates are compared bit for bit)
double Solver2D::dot_seq(int level, const double* a, const double* b) {
  launch_dot_seq(H_->lev.at(level), a, b, dot_out_, stream_);
  double out = 0.0;
  KB_CUDA_CHECK(cudaMemcpyAsync(&out, dot_out_, 8, cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return out;
}

void Solver2D::solve_direct(int l, double* u) {
  if (l < 0 || l > L_) fail(KB_STRUCTURAL, "level out of range");
  const auto& lev = H_->lev;
  const auto& lv = lev[l];
  // b = level_rhs(l); u = g on the domain boundary, 0 elsewhere
  launch_rhs(lv, src_kind_, ftab_[l], ftab_[l], gbnd_[l], b_[l], stream_);
  launch_set_boundary(lv, u, gbnd_[l], 1, stream_);
  if (l == 0) {
    KB_CUDA_CHECK(cudaMemsetAsync(status_, 0, sizeof(DevStatus), stream_));
    launch_cg0(lv, u, b_[0], cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
               status_, stream_);
    sync_and_check();
    return;
  }
  const size_t N = level_size(l);
  const std::int64_t n64 = static_cast<std::int64_t>(N);
  double* r = scratch(0, l);
  double* p = scratch(1, l);
  double* ap = scratch(2, l);
  launch_apply(lv, lv.kstiff, u, r, b_[l], APPLY_RESIDUAL, stream_);
  KB_CUDA_CHECK(cudaMemcpyAsync(p, r, N * 8, cudaMemcpyDeviceToDevice, stream_));
  double rr = dot_seq(l, r, r);
  const double tol = std::max(cfg_.coarse_rel_tol * std::sqrt(rr), cfg_.coarse_abs_floor);
  int it = 0;
  while (std::sqrt(rr) > tol && it < cfg_.coarse_max_iter) {
    ++it;
    // ap = A p, zero domain boundary (apply + zero_domain_boundary)
    launch_apply(lv, lv.kstiff, p, ap, nullptr, APPLY_ZERO_BND, stream_);
    const double pap = dot_seq(l, p, ap);
    if (pap <= 0.0) break;
    const double alpha = rr / pap;
    launch_axpy(u, p, alpha, n64, stream_);
    launch_axpy(r, ap, -alpha, n64, stream_);
    const double rr_new = dot_seq(l, r, r);
    // p.scale(rr_new / rr); p.add_scaled(r, 1.0)
    launch_scale_add(p, rr_new / rr, r, n64, stream_);
    rr = rr_new;
  }
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

// ExactErrorEvaluator constructor, proj/src/fem.cpp:358-392: moments of the
// exact solution per lattice copy and the per-macro integral of its square,
// by the 6-point degree-4 rule per fine cell (host, the reference's order)
void Solver2D::exact_setup() {
  if (ex_moments_) return;
  if (!prob_.has_exact) fail(KB_STRUCTURAL, "the problem has no closed-form solution");
  const Hierarchy2D& hh = H_->host;
  const int M = hh.M, n = hh.levels[L_].n, S = hh.levels[L_].S;
  constexpr double kQa = 0.445948490915965, kQwa = 0.223381589678011;
  constexpr double kQb = 0.091576213509771, kQwb = 0.109951743655322;
  const double quad[6][4] = {{1 - 2 * kQa, kQa, kQa, kQwa}, {kQa, 1 - 2 * kQa, kQa, kQwa},
                             {kQa, kQa, 1 - 2 * kQa, kQwa}, {1 - 2 * kQb, kQb, kQb, kQwb},
                             {kQb, 1 - 2 * kQb, kQb, kQwb}, {kQb, kQb, 1 - 2 * kQb, kQwb}};
  std::vector<double> mom(static_cast<size_t>(M) * S, 0.0);
  ex_usq_.assign(M, 0.0);
  for (int slot = 0; slot < M; ++slot) {
    const double cell_area = hh.mesh.area[slot] / (static_cast<double>(n) * n);
    double* mm = &mom[static_cast<size_t>(slot) * S];
    double& usq = ex_usq_[slot];
    const auto& t = hh.mesh.tri[slot];
    const double c0x = hh.mesh.x[t[0]], c0y = hh.mesh.y[t[0]];
    const double ux = (hh.mesh.x[t[1]] - c0x) / n, uy = (hh.mesh.y[t[1]] - c0y) / n;
    const double wx = (hh.mesh.x[t[2]] - c0x) / n, wy = (hh.mesh.y[t[2]] - c0y) / n;
    auto cell = [&](int a, int b, int c, double i0, double j0, double i1, double j1, double i2, double j2) {
      for (const auto& q : quad) {
        const double ii = q[0] * i0 + q[1] * i1 + q[2] * i2;
        const double jj = q[0] * j0 + q[1] * j1 + q[2] * j2;
        const double x = c0x + ii * ux + jj * wx;
        const double y = c0y + ii * uy + jj * wy;
        const double uval = prob_.exact(x, y);
        const double wa = q[3] * cell_area;
        mm[a] += wa * uval * q[0];
        mm[b] += wa * uval * q[1];
        mm[c] += wa * uval * q[2];
        usq += wa * uval * uval;
      }
    };
    for (int j = 0; j < n; ++j) {
      const int r0 = lattice_index(n, 0, j), r1 = lattice_index(n, 0, j + 1);
      for (int i = 0; i < n - j; ++i) cell(r0 + i, r0 + i + 1, r1 + i, i, j, i + 1, j, i, j + 1);
      for (int i = 0; i + 1 < n - j; ++i) cell(r0 + i + 1, r1 + i, r1 + i + 1, i + 1, j, i, j + 1, i + 1, j + 1);
    }
  }
  ex_arena_ = std::make_unique<DeviceArena>();
  ex_arena_->reserve(mom.size() * 8 + 2 * static_cast<size_t>(M) * 8 + 1024);
  ex_moments_ = ex_arena_->upload(mom);
  ex_out_ = static_cast<double*>(ex_arena_->take(2 * static_cast<size_t>(M) * 8));
}

// ExactErrorEvaluator::evaluate, proj/src/fem.cpp:395-420 (device per-macro
// terms, host sums in slot order, pointwise fallback on cancellation)
Solver2D::ExactNorms Solver2D::exact_error(const double* u) {
  exact_setup();
  const int M = H_->host.M;
  launch_exact_eval(H_->lev[L_], u ? u : u_[L_], ex_moments_, ex_out_, stream_);
  std::vector<double> terms(2 * static_cast<size_t>(M));
  KB_CUDA_CHECK(cudaMemcpyAsync(terms.data(), ex_out_, terms.size() * 8, cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  ExactNorms out;
  out.per_macro.assign(M, 0.0);
  double total = 0.0, scale = 0.0;
  for (int s = 0; s < M; ++s) {
    const double e2 = ex_usq_[s] - 2.0 * terms[2 * s] + terms[2 * s + 1];
    out.per_macro[s] = e2;
    total += e2;
    scale += ex_usq_[s] + terms[2 * s + 1];
  }
  if (total < 1e-12 * scale) return exact_pointwise(u);  // proj/src/fem.cpp:416-417
  for (double& v : out.per_macro) v = std::sqrt(std::max(0.0, v));
  out.global = std::sqrt(std::max(0.0, total));
  return out;
}

// ExactErrorEvaluator::evaluate_pointwise, proj/src/fem.cpp:422-455 (host,
// the cancellation fallback)
Solver2D::ExactNorms Solver2D::exact_pointwise(const double* ud) {
  const Hierarchy2D& hh = H_->host;
  const int M = hh.M, n = hh.levels[L_].n, S = hh.levels[L_].S;
  std::vector<double> u(static_cast<size_t>(M) * S);
  KB_CUDA_CHECK(cudaMemcpy(u.data(), ud ? ud : u_[L_], u.size() * 8, cudaMemcpyDeviceToHost));
  constexpr double kQa = 0.445948490915965, kQwa = 0.223381589678011;
  constexpr double kQb = 0.091576213509771, kQwb = 0.109951743655322;
  const double quad[6][4] = {{1 - 2 * kQa, kQa, kQa, kQwa}, {kQa, 1 - 2 * kQa, kQa, kQwa},
                             {kQa, kQa, 1 - 2 * kQa, kQwa}, {1 - 2 * kQb, kQb, kQb, kQwb},
                             {kQb, 1 - 2 * kQb, kQb, kQwb}, {kQb, kQb, 1 - 2 * kQb, kQwb}};
  ExactNorms out;
  out.per_macro.assign(M, 0.0);
  double total = 0.0;
  for (int slot = 0; slot < M; ++slot) {
    const double* cm = &u[static_cast<size_t>(slot) * S];
    const double cell_area = hh.mesh.area[slot] / (static_cast<double>(n) * n);
    const auto& t = hh.mesh.tri[slot];
    const double c0x = hh.mesh.x[t[0]], c0y = hh.mesh.y[t[0]];
    const double ux = (hh.mesh.x[t[1]] - c0x) / n, uy = (hh.mesh.y[t[1]] - c0y) / n;
    const double wx = (hh.mesh.x[t[2]] - c0x) / n, wy = (hh.mesh.y[t[2]] - c0y) / n;
    double sum = 0.0;
    auto cell = [&](int a, int b, int c, double i0, double j0, double i1, double j1, double i2, double j2) {
      const double ca = cm[a], cb = cm[b], cc = cm[c];
      for (const auto& q : quad) {
        const double ii = q[0] * i0 + q[1] * i1 + q[2] * i2;
        const double jj = q[0] * j0 + q[1] * j1 + q[2] * j2;
        const double x = c0x + ii * ux + jj * wx;
        const double y = c0y + ii * uy + jj * wy;
        const double diff = prob_.exact(x, y) - (q[0] * ca + q[1] * cb + q[2] * cc);
        sum += q[3] * cell_area * diff * diff;
      }
    };
    for (int j = 0; j < n; ++j) {
      const int r0 = lattice_index(n, 0, j), r1 = lattice_index(n, 0, j + 1);
      for (int i = 0; i < n - j; ++i) cell(r0 + i, r0 + i + 1, r1 + i, i, j, i + 1, j, i, j + 1);
      for (int i = 0; i + 1 < n - j; ++i) cell(r0 + i + 1, r1 + i, r1 + i + 1, i + 1, j, i, j + 1, i + 1, j + 1);
    }
    out.per_macro[slot] = std::sqrt(sum);
    total += sum;
  }
  out.global = std::sqrt(total);
  return out;
}

void Solver2D::estimate_enqueue(int offset) {
  // error_estimate, proj/src/estimator.cpp:8-29
  if (offset < 1 || offset > L_ - 1) fail(KB_STRUCTURAL, "estimate offset must satisfy 1 <= j <= L-1");
  const auto& lev = H_->lev;
  const int base = L_ - offset;
  const int saved = launches_;
  probe_begin(&est_probes_);
  // e_base = u_L - prolongate_to(w[base], L): w[base] lives on level base+1
  const double* wb = w_[base];
  for (int l = base + 1; l < L_; ++l) {
    double* dst = (l + 1 == L_) ? est_tmp_a_ : vu_[l + 1];
    launch_prolong(lev[l], lev[l + 1], wb, dst, nullptr, nullptr, PROLONG_ASSIGN, stream_);
    mark(KK_ESTIMATE, 8.0 * dofs(l + 1) + 8.0 * dofs(l));
    wb = dst;
  }
  // e_coarser = u_L - prolongate_to(w[base-1], L); the last prolongation is inline
  const double* wc = w_[base - 1];
  for (int l = base; l < L_ - 1; ++l) {
    double* dst = (l + 1 == L_ - 1) ? est_tmp_b_ : vb_[l + 1];
    launch_prolong(lev[l], lev[l + 1], wc, dst, nullptr, nullptr, PROLONG_ASSIGN, stream_);
    mark(KK_ESTIMATE, 8.0 * dofs(l + 1) + 8.0 * dofs(l));
    wc = dst;
  }
  launch_estimate(lev[L_], u_[L_], wb, wc, est_sums_, stream_);
  // one fused pass reads u_L, w[L-1] and w[L-2] (inline prolongation): 18 B per fine DoF (2-d)
  mark(KK_ESTIMATE, 16.0 * dofs(L_) + 8.0 * dofs(L_ - 1));
  est_launches_ = launches_ - saved;
  launches_ = saved;
  KB_CUDA_CHECK(cudaMemcpyAsync(sums_host_, est_sums_, 2 * H_->host.M * sizeof(double), cudaMemcpyDeviceToHost,
                                stream_));
  probes_ = nullptr;
}

EstimateReport2D Solver2D::estimate_finish(int offset, int kind) {
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
      const double conv_t = lc > floor ? lb / lc : rep.conv_factor;
      rep.eta_local[s] = std::pow(conv_t, offset) * lb;
    }
  }
  return rep;
}

EstimateReport2D Solver2D::estimate(int offset, int kind) {
  estimate_enqueue(offset);
  return estimate_finish(offset, kind);
}

// ------------------------------------------------------------------ single operations
void Solver2D::apply(int level, int op_mass, const double* x, double* y) {
  const auto& lv = H_->lev.at(level);
  launch_apply(lv, op_mass ? lv.kmass : lv.kstiff, x, y, nullptr, APPLY_PLAIN, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Solver2D::residual(int level, const double* u, const double* b, double* r) {
  const auto& lv = H_->lev.at(level);
  launch_apply(lv, lv.kstiff, u, r, b, APPLY_RESIDUAL, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Solver2D::gauss_seidel(int level, double* u, const double* b, int sweeps) {
  if (level < 1) fail(KB_STRUCTURAL, "Gauss-Seidel runs on levels >= 1");
  launch_gs(H_->dh, H_->lev.at(level), u, b, sweeps, gs_done_, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Solver2D::restrict_to(int fine_level, const double* r, double* rc) {
  if (fine_level < 1) fail(KB_STRUCTURAL, "restriction below level 0");
  launch_restrict(H_->lev.at(fine_level), H_->lev.at(fine_level - 1), r, rc, 0, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Solver2D::prolongate(int coarse_level, const double* c, double* f) {
  if (coarse_level + 1 > L_) fail(KB_STRUCTURAL, "prolongation beyond the finest level");
  launch_prolong(H_->lev.at(coarse_level), H_->lev.at(coarse_level + 1), c, f, nullptr, nullptr, PROLONG_ASSIGN,
                 stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Solver2D::cg_level0(double* u, const double* b) {
  KB_CUDA_CHECK(cudaMemsetAsync(status_, 0, sizeof(DevStatus), stream_));
  launch_cg0(H_->lev.at(0), u, b, cg_scratch_, {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter},
             status_, stream_);
  sync_and_check();
}

double Solver2D::dot_unique(int level, const double* a, const double* b) {
  launch_dot(H_->lev.at(level), a, b, dot_partial_, dot_out_, stream_);
  double out = 0.0;
  KB_CUDA_CHECK(cudaMemcpyAsync(&out, dot_out_, 8, cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return out;
}

void Solver2D::interface_sync(int level, double* f, int additive) {
  launch_sync(H_->lev.at(level), f, additive, stream_);
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

}  // namespace kb
