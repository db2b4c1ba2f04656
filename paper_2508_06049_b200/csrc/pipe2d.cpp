// Tables of the fine-grained pipelined 2-d smoother.  See PipeTables2D in
// hier2d.hpp.  The dependences are derived by replaying the reference's
// sequential relaxation order (proj/src/multigrid.cpp:152-178)
// over the global memory locations that cross macros: every interface copy
// (relax_boundary_node writes all copies, :132-150) and every ghost value (a
// neighbouring lattice's node read by a member's partial_row,
// proj/src/fem.cpp:128-173, written through by its owner when relaxed).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hier2d.hpp"

namespace kb {

namespace {
constexpr int kDij2[6][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {-1, 1}, {1, -1}};  // E W N S NW SE

int min_pipe_n() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_GS_PIPE_MIN_N");
    v = e ? atoi(e) : 8;
  }
  return v;
}

void build_level(const Hierarchy2D& h, Level2D& lv) {
  const int n = lv.n, S = lv.S, M = h.M, T = 2 * n + 1;
  const std::size_t copies = static_cast<std::size_t>(M) * S;
  // global locations that cross macros: interface copies and ghosts
  std::vector<char> tracked(copies, 0);
  for (std::size_t q = 0; q < lv.mem_slot.size(); ++q)
    tracked[static_cast<std::size_t>(lv.mem_slot[q]) * S + lv.mem_idx[q]] = 1;
  for (int off : lv.ghost_off) tracked[off] = 2;
  // per location: last write (serial, macro, step) and global readers since
  struct Reader {
    int m, th;
  };
  // the per-location state is kept for the tracked locations only (a few per
  // cent of the copies): loc_id maps a copy offset to its compact index
  std::vector<int> loc_id(copies, -1);
  int ntracked = 0;
  for (std::size_t L = 0; L < copies; ++L)
    if (tracked[L]) loc_id[L] = ntracked++;
  std::vector<long long> w_serial_c(ntracked, 0);
  std::vector<int> w_m_c(ntracked, -1), w_t_c(ntracked, 0);
  std::vector<std::vector<Reader>> readers_c(ntracked);
  struct LocView {  // indexable by copy offset (tracked locations only)
    std::vector<int>& id;
    std::vector<long long>& serial;
    long long& operator[](std::size_t L) { return serial[id[L]]; }
  };
  LocView w_serial{loc_id, w_serial_c};
  struct IntView {
    std::vector<int>& id;
    std::vector<int>& v;
    int& operator[](std::size_t L) { return v[id[L]]; }
  };
  IntView w_m{loc_id, w_m_c}, w_t{loc_id, w_t_c};
  struct ReadersView {
    std::vector<int>& id;
    std::vector<std::vector<Reader>>& v;
    std::vector<Reader>& operator[](std::size_t L) { return v[id[L]]; }
  };
  ReadersView readers{loc_id, readers_c};
  // initial loads: every macro reads its lattice and its ghosts before its step
  // 0; semantically at (sweep 0, m), so only later writers wait for them
  auto initial_loads = [&](int m) {
    auto add = [&](std::size_t L) {
      if (w_m[L] < 0) readers[L].push_back({m, 2});
    };
    for (int p = 0; p < 3 * n; ++p) {
      int i, j;
      if (p <= n) i = p, j = 0;
      else if (p <= 2 * n) i = 0, j = p - n;
      else j = p - 2 * n, i = n - j;
      add(static_cast<std::size_t>(m) * S + lattice_index(n, i, j));
    }
    for (int x = lv.ghost_ptr[m]; x < lv.ghost_ptr[m + 1]; ++x) add(lv.ghost_off[x]);
  };
  // what each macro holds: per boundary position and per ghost slot, the write serial
  std::vector<std::vector<long long>> know_b(M, std::vector<long long>(3 * n, 0));
  std::vector<std::vector<long long>> know_g(M);
  for (int m = 0; m < M; ++m) know_g[m].assign(lv.ghost_ptr[m + 1] - lv.ghost_ptr[m], 0);
  long long serial = 0;

  // per step: requirements (macro, progress) and fetches (destination, source),
  // fixed capacity kPipeLanes each (more is not supported by the kernel: the
  // macro-DAG smoother runs then); counts keep counting past the capacity
  struct StepRec {
    int nreq = 0, nfetch = 0;
    std::pair<int, int> req[kPipeLanes], fetch[kPipeLanes];
  };
  std::vector<StepRec> recs(static_cast<std::size_t>(M) * 2 * T);
  auto bpos_of = [&](int i, int j) { return bpos(n, i, j); };
  auto is_bnd = [&](int i, int j) { return i == 0 || j == 0 || i + j == n; };

  for (int s = 0; s < 2; ++s)
    for (int m = 0; m < M; ++m) {
      if (s == 0) initial_loads(m);
      std::vector<char> seen_b(3 * n, 0), written_b(3 * n, 0);
      std::vector<char> seen_g(know_g[m].size(), 0);
      const int gb = lv.ghost_ptr[m];
      for (int t = 0; t < T; ++t) {
        StepRec& R = recs[(static_cast<std::size_t>(m) * 2 + s) * T + t];
        const int tau = s * T + t;
        auto need = [&](int m2, int p) {
          if (m2 == m) return;
          const int have = std::min(R.nreq, kPipeLanes);
          for (int e = 0; e < have; ++e)
            if (R.req[e].first == m2) {
              if (R.req[e].second < p) R.req[e].second = p;
              return;
            }
          if (R.nreq < kPipeLanes) R.req[R.nreq] = {m2, p};
          ++R.nreq;
        };
        auto first_use = [&](std::size_t L, int dst, long long& know) {
          if (w_serial[L] == know) return;
          if (w_m[L] >= 0) need(w_m[L], w_t[L] + 2);
          if (R.nfetch < kPipeLanes) R.fetch[R.nfetch] = {dst, static_cast<int>(L)};
          ++R.nfetch;
          readers[L].push_back({m, tau + 2});
          know = w_serial[L];
        };
        auto read_lattice = [&](int i, int j) {
          if (!is_bnd(i, j)) return;
          const int bp = bpos_of(i, j);
          if (written_b[bp] || seen_b[bp]) return;
          seen_b[bp] = 1;
          first_use(static_cast<std::size_t>(m) * S + lattice_index(n, i, j), lattice_index(n, i, j), know_b[m][bp]);
        };
        auto read_ghost = [&](int x) {
          if (seen_g[x]) return;
          seen_g[x] = 1;
          first_use(static_cast<std::size_t>(lv.ghost_off[gb + x]), -1 - x, know_g[m][x]);
        };
        auto write = [&](std::size_t L) {
          if (!tracked[L]) return;
          for (const Reader& r : readers[L]) need(r.m, r.th);
          if (w_m[L] >= 0) need(w_m[L], w_t[L] + 2);
          w_serial[L] = ++serial;
          w_m[L] = m;
          w_t[L] = tau;
          readers[L].clear();
        };
        // the relaxations of wavefront step t: reads first (no node reads a
        // node of its own step), then writes
        // only lattice-boundary nodes and their inner neighbours (i, j or
        // n - i - j equal to 1) read or write tracked locations: the rows
        // j = 0, 1, the columns i = 0, 1 and the diagonals i + j = n, n - 1 of
        // the wavefront i + 2 j = t, in ascending j like the full wavefront
        int cand[6] = {0, 1, t / 2, (t - 1) / 2, t - n, t - n + 1}, nc = 0;
        if (t & 1) cand[2] = -1; else cand[3] = -1;
        std::sort(cand, cand + 6);
        std::pair<int, int> nodes[6];
        for (int c = 0; c < 6; ++c) {
          const int j = cand[c];
          if (j < 0 || j > n || (c > 0 && cand[c - 1] == j)) continue;
          const int i = t - 2 * j;
          if (i < 0 || i > n - j) continue;
          if (!(is_bnd(i, j) || i == 1 || j == 1 || i + j == n - 1)) continue;
          nodes[nc++] = {i, j};
        }
        for (int c = 0; c < nc; ++c) {
          const int i = nodes[c].first, j = nodes[c].second;
          if (!is_bnd(i, j)) {
            for (int d = 0; d < 6; ++d) read_lattice(i + kDij2[d][0], j + kDij2[d][1]);
            continue;
          }
          const BNode& bn = lv.bnode[static_cast<std::size_t>(m) * 3 * n + bpos_of(i, j)];
          if (bn.domain) continue;
          for (int q = 0; q < bn.rec_count; ++q) {
            const MemberRec& mr = lv.rec[bn.rec_begin + q];
            for (int c = 0; c < 6; ++c) {
              if (!((mr.mask >> c) & 1)) continue;
              for (int z = 0; z < 2; ++z) {
                const int code = mr.code[2 * c + z];
                if (code < 6)
                  read_lattice(i + kDij2[code][0], j + kDij2[code][1]);
                else
                  read_ghost(code - 6);
              }
            }
          }
        }
        for (int c = 0; c < nc; ++c) {
          const int i = nodes[c].first, j = nodes[c].second;
          if (is_bnd(i, j)) {
            const int bp = bpos_of(i, j);
            const int g = lv.node_gid[static_cast<std::size_t>(m) * S + lattice_index(n, i, j)];
            for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q)
              write(static_cast<std::size_t>(lv.mem_slot[q]) * S + lv.mem_idx[q]);
            written_b[bp] = 1;
            know_b[m][bp] = w_serial[static_cast<std::size_t>(m) * S + lattice_index(n, i, j)];  // m's own write
          } else if (i == 1 || j == 1 || i + j == n - 1) {
            write(static_cast<std::size_t>(m) * S + lattice_index(n, i, j));  // exported (write-through)
          }
        }
      }
    }
  PipeTables2D& P = lv.pipe;
  P = PipeTables2D{};
  for (StepRec& R : recs) {
    P.maxreq = std::max(P.maxreq, R.nreq);
    P.maxfetch = std::max(P.maxfetch, R.nfetch);
    std::sort(R.req, R.req + std::min(R.nreq, kPipeLanes));
  }
  if (P.maxreq > kPipeLanes || P.maxfetch > kPipeLanes) {  // not supported: the macro-DAG smoother runs
    if (getenv("KB_PIPE_DEBUG"))
      std::fprintf(stderr, "pipe tables M=%d n=%d: maxreq %d maxfetch %d exceed %d lanes\n", M, n, P.maxreq, P.maxfetch,
                   kPipeLanes);
    return;
  }
  P.rec_words = 4 * kPipeLanes;
  P.rec.assign(recs.size() * P.rec_words, 0);
  for (std::size_t r = 0; r < recs.size(); ++r) {
    std::int32_t* w = &P.rec[r * P.rec_words];
    for (int k = 0; k < kPipeLanes; ++k) w[4 * k] = -1, w[4 * k + 2] = -1;
    for (int k = 0; k < recs[r].nreq; ++k) {
      w[4 * k] = recs[r].req[k].first;
      w[4 * k + 1] = recs[r].req[k].second;
    }
    for (int f = 0; f < recs[r].nfetch; ++f) {
      w[4 * f + 2] = recs[r].fetch[f].second;
      w[4 * f + 3] = recs[r].fetch[f].first;
    }
  }
  P.ok = true;
  if (getenv("KB_PIPE_DEBUG")) {
    long long nr = 0, nf = 0;
    for (const StepRec& R : recs) nr += R.nreq, nf += R.nfetch;
    std::fprintf(stderr, "pipe tables M=%d n=%d: maxreq %d maxfetch %d, total req %lld fetch %lld (%.2f / %.2f per step)\n", M, n,
                 P.maxreq, P.maxfetch, nr, nf, double(nr) / recs.size(), double(nf) / recs.size());
    // critical path of the two sweeps under a unit model: a step costs c, a
    // cross-macro requirement adds the hand-off latency h (development aid)
    for (double h : {0.0, 1.0, 2.0, 4.0}) {
      std::vector<double> F(static_cast<std::size_t>(M) * 2 * T, 0.0);
      std::vector<int> hops(F.size(), 0);
      for (int sw = 0; sw < 2; ++sw)
        for (int m = 0; m < M; ++m)
          for (int t = 0; t < T; ++t) {
            const int tau = sw * T + t;
            const std::size_t e = static_cast<std::size_t>(m) * 2 * T + tau;
            double start = tau > 0 ? F[e - 1] : 0.0;
            int hp = tau > 0 ? hops[e - 1] : 0;
            const StepRec& RR = recs[(static_cast<std::size_t>(m) * 2 + sw) * T + t];
            for (int qq = 0; qq < RR.nreq; ++qq) {
              const int m2 = RR.req[qq].first, p = RR.req[qq].second;
              const std::size_t e2 = static_cast<std::size_t>(m2) * 2 * T + (p - 2);
              if (F[e2] + h > start) start = F[e2] + h, hp = hops[e2] + 1;
            }
            F[e] = start + 1.0;
            hops[e] = hp;
          }
      std::size_t best = 0;
      for (std::size_t e = 0; e < F.size(); ++e)
        if (F[e] > F[best]) best = e;
      std::fprintf(stderr, "  critical path (h = %.0f c): %.0f c, %d hand-offs (%d steps per macro)\n", h, F[best], hops[best], 2 * T);
    }
  }
}
}  // namespace

void Hierarchy2D::build_pipe_tables() {
  parallel_levels(1, L, [&](int l) {
    Level2D& lv = levels[l];
    if (lv.n < min_pipe_n() || lv.sc_nu > 0 || lv.n > 128) return;
    build_level(*this, lv);
  });
}

}  // namespace kb
