// Static exact-order Gauss-Seidel schedules of small 2-d levels.  See
// GsSched2D in hier2d.hpp.  The relaxation semantics are the reference's
// (proj/src/multigrid.cpp:127-181): interior
// nodes use the 7-point form of :170-175, lattice-boundary nodes
// relax_boundary_node (:132-150) over the group members' partial rows
// (proj/src/fem.cpp:128-173), written to every copy.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "hier2d.hpp"

namespace kb {

namespace {
constexpr int kDij[6][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {-1, 1}, {1, -1}};  // E W N S NW SE

void build_one(const Hierarchy2D& h, Level2D& lv, int sweeps, GsSched2D& out) {
  const int n = lv.n, S = lv.S, M = h.M;
  struct Relax {
    int level;
    std::vector<std::int32_t> head;
    std::vector<std::int32_t> mem;  // member records (8 words each)
  };
  std::vector<Relax> rel;
  // dependence bookkeeping per unique node: level of the last write, highest
  // level of a read since that write
  std::vector<int> last_w(lv.sc_nu, 0), last_r(lv.sc_nu, 0);
  std::vector<int> reads;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int m = 0; m < M; ++m)
      for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n - j; ++i) {
          const int k = lattice_index(n, i, j);
          const int cell = lv.sc_copy_cell[static_cast<std::size_t>(m) * S + k];
          Relax r;
          reads.clear();
          const bool bnd = i == 0 || j == 0 || i + j == n;
          if (!bnd) {
            r.head = {cell, m, 0, 0, 0, 0, 0, 0};
            for (int d = 0; d < 6; ++d) {
              const int c = lv.sc_copy_cell[static_cast<std::size_t>(m) * S + lattice_index(n, i + kDij[d][0], j + kDij[d][1])];
              r.head[2 + d] = c;
              reads.push_back(c);
            }
          } else {
            const BNode& bn = lv.bnode[static_cast<std::size_t>(m) * 3 * n + bpos(n, i, j)];
            const int g = lv.node_gid[static_cast<std::size_t>(m) * S + k];
            if (g != cell) fail(KB_INTERNAL, "schedule: group numbering");
            const double inv = bn.diag != 0.0 ? 1.0 / bn.diag : 0.0;
            r.head = {cell, -1 - g, 0, bn.domain ? -1 : bn.rec_count, 0, 0, 0, 0};
            std::memcpy(&r.head[4], &bn.diag, 8);
            std::memcpy(&r.head[6], &inv, 8);
            if (!bn.domain) out.max_members = std::max(out.max_members, bn.rec_count);
            if (!bn.domain) {
              // partial_row coefficient positions of the six cells (put_lane, hier2d.cpp)
              static const int ci[12] = {1, 2, 3, 5, 6, 7, 10, 11, 12, 14, 15, 16};
              for (int q = 0; q < bn.rec_count; ++q) {
                const MemberRec& mr = lv.rec[bn.rec_begin + q];
                std::int32_t rec[kSchedMemberWords] = {};
                for (int z = 12; z < 18; ++z) rec[z] = lv.sc_nu;  // absent terms read the zero slot
                double coef[6] = {0, 0, 0, 0, 0, 0};
                int nc = 0;
                for (int c = 0; c < 6; ++c) {
                  if (!((mr.mask >> c) & 1)) continue;
                  if (nc == 3) fail(KB_INTERNAL, "schedule: more than three cells of one member");
                  for (int t = 0; t < 2; ++t) {
                    const int code = mr.code[2 * c + t];
                    int off;
                    if (code < 6)
                      off = m * S + lattice_index(n, i + kDij[code][0], j + kDij[code][1]);
                    else
                      off = lv.ghost_off[lv.ghost_ptr[m] + code - 6];
                    const int cc = lv.sc_copy_cell[off];
                    coef[2 * nc + t] = lv.kstiff[18 * static_cast<std::size_t>(mr.slot) + ci[2 * c + t]];
                    rec[12 + 2 * nc + t] = cc;
                    reads.push_back(cc);
                  }
                  ++nc;
                }
                std::memcpy(rec, coef, sizeof coef);
                rec[18] = nc;
                r.mem.insert(r.mem.end(), rec, rec + kSchedMemberWords);
              }
            }
          }
          int L = std::max(last_w[cell], last_r[cell]);
          for (int c : reads)
            if (c != cell) L = std::max(L, last_w[c]);
          ++L;
          r.level = L;
          last_w[cell] = L;
          last_r[cell] = 0;
          for (int c : reads)
            if (c != cell) last_r[c] = std::max(last_r[c], L);
          rel.push_back(std::move(r));
        }
  int levels = 0;
  for (const Relax& r : rel) levels = std::max(levels, r.level);
  std::vector<std::vector<int>> by_level(levels);
  for (std::size_t q = 0; q < rel.size(); ++q) by_level[rel[q].level - 1].push_back(static_cast<int>(q));
  const int max_members = out.max_members;
  out = GsSched2D{};
  out.max_members = max_members;
  out.sweeps = sweeps;
  out.levels = levels;
  for (int L = 0; L < levels; ++L) {
    const auto& list = by_level[L];
    out.lev_off.push_back(static_cast<std::int32_t>(out.blocks.size()));
    const std::size_t b0 = out.blocks.size();
    out.blocks.push_back(static_cast<std::int32_t>(list.size()));
    out.blocks.insert(out.blocks.end(), 7, 0);
    const std::size_t hb = out.blocks.size();
    out.blocks.resize(hb + 8 * list.size(), 0);
    for (std::size_t t = 0; t < list.size(); ++t) {
      Relax& r = rel[list[t]];
      if (r.head[1] < 0) r.head[2] = static_cast<std::int32_t>(out.blocks.size() - b0);
      std::copy(r.head.begin(), r.head.end(), out.blocks.begin() + hb + 8 * t);
      out.blocks.insert(out.blocks.end(), r.mem.begin(), r.mem.end());
    }
    out.max_width = std::max(out.max_width, static_cast<int>(list.size()));
    out.max_block_words = std::max(out.max_block_words, static_cast<int>(out.blocks.size() - b0));
  }
  out.lev_off.push_back(static_cast<std::int32_t>(out.blocks.size()));
}
}  // namespace

void Hierarchy2D::build_gs_schedules() {
  parallel_levels(1, L, [&](int l) {
    Level2D& lv = levels[l];
    const int n = lv.n, S = lv.S;
    const int NG = static_cast<int>(lv.grp_ptr.size()) - 1;
    const std::size_t copies = static_cast<std::size_t>(M) * S;
    // unique nodes: groups, then interiors
    const std::size_t interior = copies - static_cast<std::size_t>(M) * 3 * n;
    const std::size_t nu = NG + interior;
    const std::size_t table = 16 * (nu + 1) + 8 * 26 * static_cast<std::size_t>(M) + 16 * NG;
    static const std::size_t table_max =
        getenv("KB_SCHED_TABLE_KB") ? static_cast<std::size_t>(atoi(getenv("KB_SCHED_TABLE_KB"))) * 1024 : kSchedTableBytes;
    if (table > table_max) return;
    lv.sc_nu = static_cast<int>(nu);
    lv.sc_copy_cell.assign(copies, -1);
    lv.sc_cell_copy.assign(nu, -1);
    for (int g = 0; g < NG; ++g) {
      lv.sc_cell_copy[g] = lv.mem_slot[lv.grp_ptr[g]] * S + lv.mem_idx[lv.grp_ptr[g]];
      for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) lv.sc_copy_cell[lv.mem_slot[q] * S + lv.mem_idx[q]] = g;
    }
    int next = NG;
    for (std::size_t c = 0; c < copies; ++c)
      if (lv.sc_copy_cell[c] < 0) {
        lv.sc_copy_cell[c] = next;
        lv.sc_cell_copy[next] = static_cast<int>(c);
        ++next;
      }
    if (static_cast<std::size_t>(next) != nu) fail(KB_INTERNAL, "schedule: unique node count");
    lv.sc_mtab.assign(26 * static_cast<std::size_t>(M), 0.0);
    for (int m = 0; m < M; ++m) {
      double* t = &lv.sc_mtab[26 * static_cast<std::size_t>(m)];
      for (int q = 1; q <= 6; ++q) t[q - 1] = lv.stencil[7 * m + q];
      t[6] = lv.inv_c[m];
      for (int q = 0; q < 18; ++q) t[8 + q] = lv.kstiff[18 * m + q];
    }
    lv.sc_gtab.assign(2 * static_cast<std::size_t>(NG), 0.0);
    for (int m = 0; m < M; ++m)
      for (int p = 0; p < 3 * n; ++p) {
        const BNode& bn = lv.bnode[static_cast<std::size_t>(m) * 3 * n + p];
        int i, j;
        if (p <= n) i = p, j = 0;
        else if (p <= 2 * n) i = 0, j = p - n;
        else j = p - 2 * n, i = n - j;
        const int g = lv.node_gid[static_cast<std::size_t>(m) * S + lattice_index(n, i, j)];
        lv.sc_gtab[2 * g] = bn.diag;
        lv.sc_gtab[2 * g + 1] = bn.diag != 0.0 ? 1.0 / bn.diag : 0.0;
      }
    for (int s = 1; s <= 2; ++s) {
      lv.sched[s - 1].max_members = 0;
      build_one(*this, lv, s, lv.sched[s - 1]);
    }
    if (getenv("KB_SCHED_DEBUG"))
      std::fprintf(stderr, "gs schedule M=%d l=%d nu=%zu: 1 sweep %d levels (width %d, block %d words), 2 sweeps %d levels\n",
                   M, l, nu, lv.sched[0].levels, lv.sched[0].max_width, lv.sched[0].max_block_words, lv.sched[1].levels);
  });
}

}  // namespace kb
