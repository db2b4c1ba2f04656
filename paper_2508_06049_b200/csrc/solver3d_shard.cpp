// Macro-sharded 3-d FMG + estimator.  See solver3d_shard.hpp.
#include "solver3d_shard.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace kb {

void launch3_ftab(const DevLevel3D& lv, const double* corners, int kind, const double* params, double* f,
                  cudaStream_t st);  // kernels3d.cu

namespace {
size_t r256(size_t b) { return (b + 255) & ~static_cast<size_t>(255); }
template <typename T>
size_t vb(const std::vector<T>& v) {
  return r256(v.size() * sizeof(T));
}

}  // namespace

size_t ShardedSolver3D::lsize(const Shard3D& sh, int l) const {
  return static_cast<size_t>(mloc(sh, l)) * H_->host.levels[l].S;
}

ShardedSolver3D::ShardedSolver3D(std::shared_ptr<DeviceHierarchy3D> h, Problem3D p, SolverConfig2D cfg, int nshards,
                                 int rep_level, std::shared_ptr<NcclComm> comm)
    : H_(std::move(h)), prob_(std::move(p)), cfg_(cfg), comm_(std::move(comm)) {
  const Hierarchy3D& hh = H_->host;
  L_ = hh.L;
  M_ = hh.M;
  if (cfg_.finest_policy != 0) fail(KB_STRUCTURAL, "only FinestPolicy::None is available on the device path");
  // host-callback problems have no device form: always tabulated on the host
  if (prob_.kind == P3_HOST) cfg_.faithful_source = 1;
  P_ = comm_ ? comm_->size() : nshards;
  if (P_ < 1 || P_ > M_) fail(KB_STRUCTURAL, "shard count must be in [1, number of macro elements]");
  rep_ = std::min(std::max(rep_level, 0), L_);
  has_source_ = prob_.kind != P3_ZERO;
  const int C = hh.colors;
  std::vector<int> ranks;
  if (comm_)
    ranks.push_back(comm_->rank());
  else
    for (int r = 0; r < P_; ++r) ranks.push_back(r);

  for (int r : ranks) {
    auto shp = std::make_unique<Shard3D>();
    Shard3D& sh = *shp;
    sh.plan = build_shard_plan(hh, P_, r, rep_);
    // ---- tables
    size_t tb = 0;
    long long smax = 1, rmax = 1;
    for (int l = 0; l <= L_; ++l) {
      if (!sharded(l)) continue;
      const ShardLevel3D& s = sh.plan.lev[l];
      tb += vb(s.grp_ptr) + vb(s.mem_slot) + vb(s.mem_ijk) + vb(s.grp_domain) + vb(s.grp_diag) + vb(s.color_grp_ptr) +
            vb(s.color_grp) + vb(s.color_wide_end) + vb(s.pack_pos) + vb(s.pack_slot) + vb(s.pack_ijk);
      smax = std::max(smax, s.send_total);
      rmax = std::max(rmax, s.recv_total);
    }
    sh.tables.reserve(tb + 4096);
    sh.pack_pos.assign(L_ + 1, nullptr);
    sh.pack_slot = sh.pack_ijk = sh.pack_pos;
    // ---- data
    size_t db = 0;
    for (int l = 0; l <= L_; ++l) {
      db += 2 * r256(lsize(sh, l) * 8);
      if (l < L_) db += r256(lsize(sh, l + 1) * 8) + 2 * r256(lsize(sh, l) * 8);
      if (l >= 1) db += r256(lsize(sh, l) * 8);
      db += r256((sharded(l) ? sh.plan.lev[l].ng : hh.levels[l].grp_ptr.size()) * 8 + 8);
      if (has_source_) db += r256(lsize(sh, l) * 8);
    }
    db += r256(smax * 8) + r256(rmax * 8) + r256(3 * lsize(sh, 0) * 8) + r256(2 * M_ * 8) + 3 * r256(lsize(sh, L_) * 8) +
          r256(sizeof(DevStatus)) + r256(12 * M_ * 8) + r256(64 * 8);
    sh.data.reserve(db + 4096);
    sh.sendbuf = static_cast<double*>(sh.data.take(smax * 8));
    sh.ghost = static_cast<double*>(sh.data.take(rmax * 8));

    for (int l = 0; l <= L_; ++l) {
      DevLevel3D dl = H_->lev[l];
      dl.ghost = nullptr;
      if (sharded(l)) {
        const ShardLevel3D& s = sh.plan.lev[l];
        const size_t s0 = static_cast<size_t>(sh.plan.s0);
        dl.M = sh.plan.count;
        dl.ng = s.ng;
        dl.grp_ptr = sh.tables.upload(s.grp_ptr);
        dl.mem_slot = sh.tables.upload(s.mem_slot);
        dl.mem_ijk = sh.tables.upload(s.mem_ijk);
        dl.grp_domain = sh.tables.upload(s.grp_domain);
        dl.grp_diag = sh.tables.upload(s.grp_diag);
        dl.color_grp_ptr = sh.tables.upload(s.color_grp_ptr);
        dl.color_grp = sh.tables.upload(s.color_grp);
        dl.color_wide_end = sh.tables.upload(s.color_wide_end);
        dl.nar_hdr = nullptr;  // shard tables: the chained group tables
        dl.max_color_groups = 0;
        dl.nar_mem = nullptr;
        dl.wide_mem = nullptr;
        // per-macro tables of the full hierarchy, from this shard's first slot
        dl.kstiff += 96 * s0;
        dl.kmass += 96 * s0;
        dl.stK += 15 * s0;
        dl.stM += 15 * s0;
        dl.inv_c += s0;
        dl.pat_color += 8 * s0;
        dl.col_pat += static_cast<size_t>(C) * s0;
        dl.psK += 240 * s0;
        dl.psM += 240 * s0;
        dl.own_dot = nullptr;  // owner dots are not defined on a shard
        dl.ghost = sh.ghost;
        sh.pack_pos[l] = sh.tables.upload(s.pack_pos);
        sh.pack_slot[l] = sh.tables.upload(s.pack_slot);
        sh.pack_ijk[l] = sh.tables.upload(s.pack_ijk);
      }
      sh.lev.push_back(dl);
    }
    sh.u.assign(L_ + 1, nullptr);
    sh.b = sh.w = sh.vu = sh.vb = sh.r = sh.gbnd = sh.ftab = sh.u;
    for (int l = 0; l <= L_; ++l) {
      sh.u[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
      sh.b[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
      if (l < L_) {
        sh.w[l] = static_cast<double*>(sh.data.take(lsize(sh, l + 1) * 8));
        sh.vu[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
        sh.vb[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
      }
      if (l >= 1) sh.r[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
      sh.gbnd[l] = static_cast<double*>(sh.data.take(static_cast<size_t>(sh.lev[l].ng) * 8 + 8));
      if (has_source_) sh.ftab[l] = static_cast<double*>(sh.data.take(lsize(sh, l) * 8));
    }
    sh.cg_scratch = static_cast<double*>(sh.data.take(3 * lsize(sh, 0) * 8));
    sh.est_all = static_cast<double*>(sh.data.take(2 * static_cast<size_t>(M_) * 8));
    sh.est_a = static_cast<double*>(sh.data.take(lsize(sh, L_) * 8));
    sh.est_b = static_cast<double*>(sh.data.take(lsize(sh, L_) * 8));
    sh.est_c = static_cast<double*>(sh.data.take(lsize(sh, L_) * 8));
    sh.status = static_cast<DevStatus*>(sh.data.take(sizeof(DevStatus)));
    KB_CUDA_CHECK(cudaMemset(sh.status, 0, sizeof(DevStatus)));
    KB_CUDA_CHECK(cudaMallocHost(&sh.status_host, sizeof(DevStatus)));
    // device source tables (fast mode): every copy at its own macro's coordinates
    if (has_source_ && !cfg_.faithful_source) {
      double* corners = static_cast<double*>(sh.data.take(12 * static_cast<size_t>(M_) * 8));
      double* params = static_cast<double*>(sh.data.take(64 * 8));
      std::vector<double> cv(12 * static_cast<size_t>(M_));
      for (int s = 0; s < M_; ++s)
        for (int c = 0; c < 4; ++c) {
          const int v = hh.mesh.tet[s][c];
          cv[12 * s + 3 * c] = hh.mesh.x[v];
          cv[12 * s + 3 * c + 1] = hh.mesh.y[v];
          cv[12 * s + 3 * c + 2] = hh.mesh.z[v];
        }
      KB_CUDA_CHECK(cudaMemcpy(corners, cv.data(), cv.size() * 8, cudaMemcpyHostToDevice));
      std::vector<double> par(64, 0.0);
      if (!prob_.params.empty()) std::copy(prob_.params.begin(), prob_.params.end(), par.begin());
      KB_CUDA_CHECK(cudaMemcpy(params, par.data(), 64 * 8, cudaMemcpyHostToDevice));
      for (int l = 0; l <= L_; ++l)
        launch3_ftab(sh.lev[l], corners + 12 * static_cast<size_t>(off(sh, l)), prob_.kind, params, sh.ftab[l],
                     nullptr);
    }
    sh_.push_back(std::move(shp));
  }
  KB_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  KB_CUDA_CHECK(cudaMallocHost(&sums_host_, 2 * static_cast<size_t>(M_) * sizeof(double)));
  KB_CUDA_CHECK(cudaDeviceSynchronize());
  load_problem();
}

ShardedSolver3D::~ShardedSolver3D() {
  if (exec_) cudaGraphExecDestroy(exec_);
  if (stream_) cudaStreamDestroy(stream_);
  if (sums_host_) cudaFreeHost(sums_host_);
  for (auto& sh : sh_)
    if (sh->status_host) cudaFreeHost(sh->status_host);
}

// Dirichlet g per group and (faithful mode) f per copy at the owner copy's
// node coordinates -- the tables Solver3D::load_problem builds, sliced per shard
void ShardedSolver3D::load_problem() {
  const Hierarchy3D& hh = H_->host;
  for (int l = 0; l <= L_; ++l) {
    const Level3D& lv = hh.levels[l];
    const int n = lv.n, S = lv.S;
    std::vector<int> ii(S), jj(S), kk(S);
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n - k; ++j)
        for (int i = 0; i <= n - k - j; ++i) {
          const int idx = lattice_index3(n, i, j, k);
          ii[idx] = i, jj[idx] = j, kk[idx] = k;
        }
    auto coords = [&](int s, int idx, double* out) {
      const auto& t = hh.mesh.tet[s];
      const double P[4][3] = {{hh.mesh.x[t[0]], hh.mesh.y[t[0]], hh.mesh.z[t[0]]},
                              {hh.mesh.x[t[1]], hh.mesh.y[t[1]], hh.mesh.z[t[1]]},
                              {hh.mesh.x[t[2]], hh.mesh.y[t[2]], hh.mesh.z[t[2]]},
                              {hh.mesh.x[t[3]], hh.mesh.y[t[3]], hh.mesh.z[t[3]]}};
      for (int a = 0; a < 3; ++a)
        out[a] = P[0][a] + (static_cast<double>(ii[idx]) / n) * (P[1][a] - P[0][a]) +
                 (static_cast<double>(jj[idx]) / n) * (P[2][a] - P[0][a]) +
                 (static_cast<double>(kk[idx]) / n) * (P[3][a] - P[0][a]);
    };
    const int NG = static_cast<int>(lv.grp_ptr.size()) - 1;
    std::vector<double> g(NG, 0.0);
    for (int q = 0; q < NG; ++q)
      if (lv.grp_domain[q]) {
        double x[3];
        coords(lv.mem_slot[lv.grp_ptr[q]], lv.mem_idx[lv.grp_ptr[q]], x);
        g[q] = prob_.boundary(x[0], x[1], x[2]);
      }
    for (auto& shp : sh_) {
      Shard3D& sh = *shp;
      std::vector<double> gl;
      if (sharded(l)) {
        for (int gid : sh.plan.lev[l].gid) gl.push_back(g[gid]);
      } else {
        gl = g;
      }
      if (!gl.empty()) KB_CUDA_CHECK(cudaMemcpy(sh.gbnd[l], gl.data(), gl.size() * 8, cudaMemcpyHostToDevice));
      if (has_source_ && cfg_.faithful_source) {
        const int s0 = off(sh, l), cnt = mloc(sh, l);
        std::vector<double> f(static_cast<size_t>(cnt) * S);
        tabulate_source3(hh, l, prob_, s0, s0 + cnt, f.data());
        KB_CUDA_CHECK(cudaMemcpy(sh.ftab[l], f.data(), f.size() * 8, cudaMemcpyHostToDevice));
      }
    }
  }
}

// ------------------------------------------------------------------ transport
void ShardedSolver3D::exchange(int l, int c0, int c1) {
  const int C = H_->host.colors;
  auto seg = [&](const std::vector<long long>& off, int p, int c) { return off[static_cast<size_t>(p) * (C + 1) + c]; };
  if (comm_) {
    const Shard3D& sh = *sh_[0];
    const ShardLevel3D& s = sh.plan.lev[l];
    const int r = sh.plan.r;
    comm_->group_start();
    for (int p = 0; p < P_; ++p) {
      if (p == r) continue;
      const long long ns = seg(s.send_off, p, c1) - seg(s.send_off, p, c0);
      const long long nr = seg(s.recv_off, p, c1) - seg(s.recv_off, p, c0);
      if (ns > 0) comm_->send(sh.sendbuf + seg(s.send_off, p, c0), ns, p, stream_);
      if (nr > 0) comm_->recv(sh.ghost + seg(s.recv_off, p, c0), nr, p, stream_);
      xbytes_ += 8.0 * ns;
    }
    comm_->group_end();
    return;
  }
  for (auto& qs : sh_) {  // receiver
    const ShardLevel3D& rq = qs->plan.lev[l];
    for (auto& ps : sh_) {  // sender
      const int p = ps->plan.r, q = qs->plan.r;
      if (p == q) continue;
      const ShardLevel3D& sp = ps->plan.lev[l];
      const long long nr = seg(rq.recv_off, p, c1) - seg(rq.recv_off, p, c0);
      if (nr <= 0) continue;
      KB_CUDA_CHECK(cudaMemcpyAsync(qs->ghost + seg(rq.recv_off, p, c0), ps->sendbuf + seg(sp.send_off, q, c0), nr * 8,
                                    cudaMemcpyDeviceToDevice, stream_));
      xbytes_ += 8.0 * nr;
    }
  }
}

void ShardedSolver3D::allgather(const std::vector<double*>& a, size_t per) {
  const std::vector<int>& st = sh_[0]->plan.starts;
  if (comm_) {
    const int r = sh_[0]->plan.r;
    comm_->group_start();
    for (int p = 0; p < P_; ++p) {
      if (p == r) continue;
      comm_->send(a[0] + st[r] * per, (st[r + 1] - st[r]) * per, p, stream_);
      comm_->recv(a[0] + st[p] * per, (st[p + 1] - st[p]) * per, p, stream_);
      xbytes_ += 8.0 * (st[r + 1] - st[r]) * per;
    }
    comm_->group_end();
    return;
  }
  for (size_t q = 0; q < sh_.size(); ++q)
    for (size_t p = 0; p < sh_.size(); ++p) {
      if (p == q) continue;
      const int rp = sh_[p]->plan.r;
      KB_CUDA_CHECK(cudaMemcpyAsync(a[q] + st[rp] * per, a[p] + st[rp] * per, (st[rp + 1] - st[rp]) * per * 8,
                                    cudaMemcpyDeviceToDevice, stream_));
      xbytes_ += 8.0 * (st[rp + 1] - st[rp]) * per;
    }
}

void ShardedSolver3D::pack(int l, int mode, const std::vector<double*>& x, int c0, int c1) {
  for (size_t q = 0; q < sh_.size(); ++q) {
    Shard3D& sh = *sh_[q];
    const ShardLevel3D& s = sh.plan.lev[l];
    launch3_pack(sh.lev[l], mode, x[q], sh.pack_pos[l], sh.pack_slot[l], sh.pack_ijk[l], s.pack_col_ptr[c0],
                 s.pack_col_ptr[c1], sh.sendbuf, stream_);
    ++launches_;
  }
}

// ------------------------------------------------------------------ FMG pieces
namespace {
template <typename F>
std::vector<double*> each(const std::vector<std::unique_ptr<Shard3D>>& sh, F f) {
  std::vector<double*> v;
  for (auto& s : sh) v.push_back(f(*s));
  return v;
}
}  // namespace

void ShardedSolver3D::set_boundary(int l, int which, int zero_rest) {
  for (auto& sh : sh_) {
    double* f = which == 0 ? sh->u[l] : sh->b[l];
    launch3_set_boundary(sh->lev[l], f, sh->gbnd[l], zero_rest, stream_);
    launches_ += 1 + zero_rest;
  }
}

void ShardedSolver3D::rhs(int l) {
  const int C = H_->host.colors;
  if (!has_source_) {
    set_boundary(l, 1, 1);
    return;
  }
  if (sharded(l)) {
    pack(l, PK3_FULL_M, each(sh_, [&](Shard3D& s) { return s.ftab[l]; }), 0, C);
    exchange(l, 0, C);
  }
  for (auto& sh : sh_) {
    launch3_apply(sh->lev[l], true, sh->ftab[l], sh->b[l], nullptr, A3_PLAIN, stream_);
    ++launches_;
  }
  set_boundary(l, 1, 0);
}

void ShardedSolver3D::prolong(int lc, const std::vector<const double*>& c, const std::vector<double*>& f, int mode) {
  const bool cross = sharded(lc + 1) && !sharded(lc);
  const size_t Sc = H_->host.levels[lc].S;
  for (size_t q = 0; q < sh_.size(); ++q) {
    const Shard3D& sh = *sh_[q];
    launch3_prolong(sh.lev[lc], sh.lev[lc + 1], c[q] + (cross ? sh.plan.s0 * Sc : 0), f[q], mode, stream_);
    ++launches_;
  }
}

void ShardedSolver3D::vcycle(int l, bool top) {
  const int C = H_->host.colors;
  auto U = [&](Shard3D& s) { return top ? s.u[l] : s.vu[l]; };
  auto B = [&](Shard3D& s) { return top ? s.b[l] : s.vb[l]; };
  if (l == 0) {
    for (auto& sh : sh_) {
      launch3_cg0(sh->lev[0], U(*sh), B(*sh), sh->cg_scratch,
                  {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter}, sh->status, stream_);
      ++launches_;
    }
    return;
  }
  auto smooth = [&](int sweeps) {
    if (sweeps <= 0) return;
    if (!sharded(l)) {
      for (auto& sh : sh_) {
        launch3_gs(sh->lev[l], U(*sh), B(*sh), sweeps, stream_);
        launches_ += launch3_gs_count(sh->lev[l], sweeps);
      }
      return;
    }
    for (int s = 0; s < sweeps; ++s) {
      for (int c = 0; c < C; ++c) {
        pack(l, PK3_OFF_K, each(sh_, U), c, c + 1);
        exchange(l, c, c + 1);
        for (auto& sh : sh_) {
          launch3_gs_color_groups(sh->lev[l], U(*sh), B(*sh), c, stream_);
          ++launches_;
        }
      }
      for (auto& sh : sh_) {
        launch3_gs_interior(sh->lev[l], U(*sh), B(*sh), stream_);
        launches_ += sh->lev[l].n >= 4 ? C : 0;
      }
    }
  };
  smooth(cfg_.pre_smooth);
  // residual for the restriction (non-owner and domain copies 0)
  if (sharded(l)) {
    pack(l, PK3_FULL_K, each(sh_, U), 0, C);
    exchange(l, 0, C);
  }
  for (auto& sh : sh_) {
    launch3_apply(sh->lev[l], false, U(*sh), sh->r[l], B(*sh), A3_RES_OWNER, stream_);
    ++launches_;
  }
  // restriction + coarse additive sync (domain copies 0)
  const size_t Sc = H_->host.levels[l - 1].S;
  if (sharded(l - 1)) {
    for (auto& sh : sh_) launch3_restrict_only(sh->lev[l], sh->lev[l - 1], sh->r[l], sh->vb[l - 1], stream_);
    pack(l - 1, PK3_VALUE, each(sh_, [&](Shard3D& s) { return s.vb[l - 1]; }), 0, C);
    exchange(l - 1, 0, C);
    for (auto& sh : sh_) launch3_sync_zero(sh->lev[l - 1], sh->vb[l - 1], 1, 1, stream_);
    launches_ += 2 * static_cast<int>(sh_.size());
  } else if (sharded(l)) {
    for (auto& sh : sh_) {
      DevLevel3D cv = sh->lev[l - 1];
      cv.M = sh->plan.count;
      launch3_restrict_only(sh->lev[l], cv, sh->r[l], sh->vb[l - 1] + sh->plan.s0 * Sc, stream_);
    }
    allgather(each(sh_, [&](Shard3D& s) { return s.vb[l - 1]; }), Sc);
    for (auto& sh : sh_) launch3_sync_zero(sh->lev[l - 1], sh->vb[l - 1], 1, 1, stream_);
    launches_ += 2 * static_cast<int>(sh_.size());
  } else {
    for (auto& sh : sh_) launch3_restrict(sh->lev[l], sh->lev[l - 1], sh->r[l], sh->vb[l - 1], 1, stream_);
    launches_ += 2 * static_cast<int>(sh_.size());
  }
  for (auto& sh : sh_) {
    KB_CUDA_CHECK(cudaMemsetAsync(sh->vu[l - 1], 0, lsize(*sh, l - 1) * 8, stream_));
  }
  vcycle(l - 1, false);
  std::vector<const double*> cc;
  for (auto& sh : sh_) cc.push_back(sh->vu[l - 1]);
  prolong(l - 1, cc, each(sh_, U), P3_ADD);
  smooth(cfg_.post_smooth);
}

void ShardedSolver3D::enqueue_fmg_body() {
  launches_ = 0;
  xbytes_ = 0.0;
  for (auto& sh : sh_) KB_CUDA_CHECK(cudaMemsetAsync(sh->status, 0, sizeof(DevStatus), stream_));
  for (int l = 0; l <= L_; ++l) rhs(l);
  set_boundary(0, 0, 1);
  for (auto& sh : sh_) {
    launch3_cg0(sh->lev[0], sh->u[0], sh->b[0], sh->cg_scratch,
                {cfg_.coarse_rel_tol, cfg_.coarse_abs_floor, cfg_.coarse_max_iter}, sh->status, stream_);
    ++launches_;
  }
  for (int l = 0; l < L_; ++l) {
    // w[l] = P u[l] (snapshot before the Dirichlet reset); next = w with g on the boundary
    std::vector<const double*> cu;
    for (auto& sh : sh_) cu.push_back(sh->u[l]);
    prolong(l, cu, each(sh_, [&](Shard3D& s) { return s.w[l]; }), P3_ASSIGN);
    for (auto& sh : sh_)
      KB_CUDA_CHECK(cudaMemcpyAsync(sh->u[l + 1], sh->w[l], lsize(*sh, l + 1) * 8, cudaMemcpyDeviceToDevice, stream_));
    set_boundary(l + 1, 0, 0);
    for (int c = 0; c < cfg_.nu; ++c) vcycle(l + 1, true);
  }
  fmg_launches_ = launches_;
  xbytes_fmg_ = xbytes_;
}

void ShardedSolver3D::fmg_enqueue() {
  if (L_ < 1) fail(KB_STRUCTURAL, "full multigrid requires at least one level above the coarse grid");
  if (!cfg_.use_graph) {
    enqueue_fmg_body();
    return;
  }
  if (!exec_) {
    cudaGraph_t graph = nullptr;
    KB_CUDA_CHECK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_fmg_body();
    } catch (...) {
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    KB_CUDA_CHECK(cudaStreamEndCapture(stream_, &graph));
    KB_CUDA_CHECK(cudaGraphInstantiate(&exec_, graph, 0));
    cudaGraphDestroy(graph);
  }
  KB_CUDA_CHECK(cudaGraphLaunch(exec_, stream_));
}

void ShardedSolver3D::sync_and_check() {
  for (auto& sh : sh_)
    KB_CUDA_CHECK(cudaMemcpyAsync(sh->status_host, sh->status, sizeof(DevStatus), cudaMemcpyDeviceToHost, stream_));
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  for (auto& sh : sh_)
    if (sh->status_host->code) {
      Error e(KB_SOLVER, sh->status_host->code == 1 ? "coarse-grid CG did not converge"
                                                    : "coarse-grid CG lost positive definiteness");
      e.residual = sh->status_host->residual;
      throw e;
    }
}

void ShardedSolver3D::fmg() {
  fmg_enqueue();
  sync_and_check();
}

// error_estimate (proj/src/estimator.cpp:8-45), as Solver3D::estimate_enqueue
void ShardedSolver3D::estimate_enqueue(int offset) {
  if (offset < 1 || offset > L_ - 1) fail(KB_STRUCTURAL, "estimate offset must satisfy 1 <= j <= L-1");
  const int base = L_ - offset;
  const int saved = launches_;
  auto lift = [&](int wl, int from_level, double* Shard3D::*out) {
    std::vector<const double*> cur;
    for (auto& sh : sh_) cur.push_back(sh->w[wl]);
    for (int l = from_level; l < L_; ++l) {
      std::vector<double*> dst;
      for (auto& sh : sh_) dst.push_back((l + 1 == L_) ? (*sh).*out : (l % 2 ? sh->vu[l + 1] : sh->vb[l + 1]));
      prolong(l, cur, dst, P3_ASSIGN);
      cur.assign(dst.begin(), dst.end());
    }
    return cur;
  };
  const std::vector<const double*> wb = lift(base, base + 1, &Shard3D::est_a);
  const std::vector<const double*> wc = lift(base - 1, base, &Shard3D::est_b);
  for (size_t q = 0; q < sh_.size(); ++q) {
    Shard3D& sh = *sh_[q];
    launch3_estimate(sh.lev[L_], sh.u[L_], wb[q], wc[q], sh.est_all + 2 * static_cast<size_t>(off(sh, L_)), sh.est_c,
                     stream_);
    launches_ += 2;
  }
  if (sharded(L_)) allgather(each(sh_, [&](Shard3D& s) { return s.est_all; }), 2);
  KB_CUDA_CHECK(cudaMemcpyAsync(sums_host_, sh_[0]->est_all, 2 * static_cast<size_t>(M_) * sizeof(double),
                                cudaMemcpyDeviceToHost, stream_));
  est_launches_ = launches_ - saved;
  launches_ = saved;
}

EstimateReport2D ShardedSolver3D::estimate_finish(int offset, int kind) {
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  EstimateReport2D rep;
  rep.offset = offset;
  rep.base_level = L_ - offset;
  rep.kind = kind;
  double gb = 0.0, gc = 0.0;
  for (int s = 0; s < M_; ++s) {
    gb += sums_host_[2 * s];
    gc += sums_host_[2 * s + 1];
  }
  rep.norm_base = std::sqrt(std::max(0.0, gb));
  rep.norm_coarser = std::sqrt(std::max(0.0, gc));
  rep.conv_factor = rep.norm_coarser > 0.0 ? rep.norm_base / rep.norm_coarser : 0.0;
  rep.eta = std::pow(rep.conv_factor, offset) * rep.norm_base;
  rep.eta_local.resize(M_);
  const double floor = 1e-14 * rep.norm_coarser;
  for (int s = 0; s < M_; ++s) {
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

void ShardedSolver3D::state_read(int which, int level, double* host_out) {
  if (level < 0 || level > L_) fail(KB_STRUCTURAL, "level out of range");
  if (which == 2 && level < 1) fail(KB_STRUCTURAL, "w lives on levels 1..L");
  if (which < 0 || which > 2) fail(KB_STRUCTURAL, "unknown state component");
  KB_CUDA_CHECK(cudaStreamSynchronize(stream_));
  const size_t S = H_->host.levels[level].S;
  for (auto& sh : sh_) {
    const double* src = which == 0 ? sh->u[level] : which == 1 ? sh->b[level] : sh->w[level - 1];
    KB_CUDA_CHECK(cudaMemcpy(host_out + off(*sh, level) * S, src, lsize(*sh, level) * 8, cudaMemcpyDeviceToHost));
    if (!sharded(level)) break;
  }
}

}  // namespace kb
