// Shard plans of the 3-d hierarchy.  See shard3d.hpp.
#include "shard3d.hpp"

#include <algorithm>

namespace kb {

std::vector<int> shard_starts(int M, int P) {
  std::vector<int> st(P + 1);
  for (int r = 0; r <= P; ++r) st[r] = static_cast<int>((static_cast<long long>(M) * r) / P);
  return st;
}

ShardPlan3D build_shard_plan(const Hierarchy3D& h, int P, int r, int rep_level) {
  if (P < 1 || r < 0 || r >= P) fail(KB_STRUCTURAL, "shard rank out of range");
  if (P > h.M) fail(KB_STRUCTURAL, "more shards than macro elements");
  ShardPlan3D plan;
  plan.P = P;
  plan.r = r;
  plan.rep_level = std::max(0, rep_level);
  plan.colors = h.colors;
  plan.starts = shard_starts(h.M, P);
  plan.s0 = plan.starts[r];
  plan.count = plan.starts[r + 1] - plan.starts[r];
  plan.lev.resize(h.L + 1);
  const int C = h.colors;
  std::vector<int> owner(h.M);
  for (int p = 0; p < P; ++p)
    for (int s = plan.starts[p]; s < plan.starts[p + 1]; ++s) owner[s] = p;

  for (int l = 0; l <= h.L; ++l) {
    if (!plan.sharded(l)) continue;
    const Level3D& lv = h.levels[l];
    ShardLevel3D& sl = plan.lev[l];
    const int n = lv.n;
    std::vector<int> ijk_of(lv.S);
    for (int k = 0; k <= n; ++k)
      for (int j = 0; j <= n - k; ++j)
        for (int i = 0; i <= n - k - j; ++i) ijk_of[lattice_index3(n, i, j, k)] = i | (j << 10) | (k << 20);
    const int NG = static_cast<int>(lv.grp_ptr.size()) - 1;

    // local groups (ascending global id) and their members
    std::vector<int> lid(NG, -1);
    sl.grp_ptr.assign(1, 0);
    for (int g = 0; g < NG; ++g) {
      bool mine = false;
      for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) mine = mine || owner[lv.mem_slot[q]] == r;
      if (!mine) continue;
      lid[g] = static_cast<int>(sl.gid.size());
      sl.gid.push_back(g);
      for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
        sl.mem_slot.push_back(0);  // filled below
        sl.mem_ijk.push_back(ijk_of[lv.mem_idx[q]]);
      }
      sl.grp_ptr.push_back(static_cast<int>(sl.mem_slot.size()));
      sl.grp_domain.push_back(lv.grp_domain[g]);
      sl.grp_diag.push_back(lv.grp_diag[g]);
    }
    sl.ng = static_cast<int>(sl.gid.size());

    // segment sizes: recv[p][c] = members on p of local groups of colour c;
    // send[p][c] = local members of colour-c groups that also have a member on p
    std::vector<long long> rc(static_cast<size_t>(P) * C, 0), sc(static_cast<size_t>(P) * C, 0);
    std::vector<char> has(P);
    auto peers_of = [&](int g) {
      std::fill(has.begin(), has.end(), 0);
      for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) has[owner[lv.mem_slot[q]]] = 1;
    };
    for (int c = 0; c < C; ++c)
      for (int t = lv.color_grp_ptr[c]; t < lv.color_grp_ptr[c + 1]; ++t) {
        const int g = lv.color_grp[t];
        if (lid[g] < 0) continue;
        peers_of(g);
        int mine = 0;
        for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
          const int p = owner[lv.mem_slot[q]];
          if (p == r)
            ++mine;
          else
            ++rc[static_cast<size_t>(p) * C + c];
        }
        for (int p = 0; p < P; ++p)
          if (p != r && has[p]) sc[static_cast<size_t>(p) * C + c] += mine;
      }
    sl.send_off.assign(static_cast<size_t>(P) * (C + 1), 0);
    sl.recv_off.assign(static_cast<size_t>(P) * (C + 1), 0);
    long long so = 0, ro = 0;
    for (int p = 0; p < P; ++p)
      for (int c = 0; c <= C; ++c) {
        sl.send_off[static_cast<size_t>(p) * (C + 1) + c] = so;
        sl.recv_off[static_cast<size_t>(p) * (C + 1) + c] = ro;
        if (c < C) {
          so += sc[static_cast<size_t>(p) * C + c];
          ro += rc[static_cast<size_t>(p) * C + c];
        }
      }
    sl.send_total = so;
    sl.recv_total = ro;
    if (so > (1ll << 31) - 1 || ro > (1ll << 31) - 1) fail(KB_RESOURCE, "shard exchange too large");

    // fill member slots (local or ghost) and the pack entries, both in the
    // (peer, colour, group ascending, member ascending) enumeration
    std::vector<long long> rcur(sl.recv_off), scur(sl.send_off);
    sl.pack_col_ptr.assign(C + 1, 0);
    for (int c = 0; c < C; ++c) {
      for (int t = lv.color_grp_ptr[c]; t < lv.color_grp_ptr[c + 1]; ++t) {
        const int g = lv.color_grp[t];
        if (lid[g] < 0) continue;
        peers_of(g);
        const int base = sl.grp_ptr[lid[g]];
        for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
          const int s = lv.mem_slot[q], p = owner[s];
          int& ms = sl.mem_slot[base + (q - lv.grp_ptr[g])];
          if (p == r)
            ms = s - plan.s0;
          else
            ms = ~static_cast<int>(rcur[static_cast<size_t>(p) * (C + 1) + c]++);
        }
        // sends: for every peer sharing the group, my members ascending
        for (int p = 0; p < P; ++p) {
          if (p == r || !has[p]) continue;
          for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
            const int s = lv.mem_slot[q];
            if (owner[s] != r) continue;
            sl.pack_pos.push_back(static_cast<int>(scur[static_cast<size_t>(p) * (C + 1) + c]++));
            sl.pack_slot.push_back(s - plan.s0);
            sl.pack_ijk.push_back(ijk_of[lv.mem_idx[q]]);
            sl.pack_gid.push_back(g);
            sl.pack_idx.push_back(lv.mem_idx[q]);
          }
        }
      }
      sl.pack_col_ptr[c + 1] = static_cast<int>(sl.pack_pos.size());
    }

    // colour lists of the local groups: wide groups first, each part ascending
    sl.color_grp_ptr.assign(C + 1, 0);
    sl.color_wide_end.assign(C, 0);
    for (int c = 0; c < C; ++c) {
      for (int wide = 1; wide >= 0; --wide) {
        for (int t = lv.color_grp_ptr[c]; t < lv.color_grp_ptr[c + 1]; ++t) {
          const int g = lv.color_grp[t];
          if (lid[g] < 0) continue;
          if ((lv.grp_ptr[g + 1] - lv.grp_ptr[g] > 4) == (wide == 1)) sl.color_grp.push_back(lid[g]);
        }
        if (wide) sl.color_wide_end[c] = static_cast<int>(sl.color_grp.size());
      }
      sl.color_grp_ptr[c + 1] = static_cast<int>(sl.color_grp.size());
    }
  }
  return plan;
}

}  // namespace kb
