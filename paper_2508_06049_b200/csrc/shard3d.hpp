// Macro sharding of the 3-d hierarchy (PAPER.md:949-954:
// macro elements are independent units, the interface primitives are the only
// coupling).  Shard r owns the contiguous slot range [starts[r], starts[r+1])
// (cube-major Kuhn meshes: z-slabs).  On a sharded level a shard keeps the
// lattices of its own macros and the shared-node groups with at least one
// local member; a member on another shard is a ghost entry whose
// contribution (partial row or copy value) that shard computes and sends.
//
// Exchange layout (both ends enumerate the same list): for the pair
// (sender a, receiver b) and colour c, the groups of colour c in ascending
// global id that have members on both a and b, and for each the members on a
// in ascending slot.  Buffers are peer-major, then colour, so an exchange of a
// colour range is one contiguous segment per peer.
//
// Levels <= rep_level are replicated: every shard holds all macros there
// (the coarse levels are < 1% of the work; level 0 carries the CG).
#pragma once

#include <cstdint>
#include <vector>

#include "hier3d.hpp"

namespace kb {

struct ShardLevel3D {
  int ng = 0;
  std::vector<int> gid;                     // local group -> global group
  std::vector<int> grp_ptr, mem_slot, mem_ijk;  // mem_slot: local slot, or ~ghost index
  std::vector<std::uint8_t> grp_domain;
  std::vector<double> grp_diag;
  std::vector<int> color_grp_ptr, color_grp, color_wide_end;  // local group ids, wide (> 4 members) first
  // send / receive segment offsets: off[p * (C + 1) + c], colour c of peer p
  std::vector<long long> send_off, recv_off;
  // pack entries, colour-major (then peer): buffer position, local slot, (i, j, k)
  std::vector<int> pack_pos, pack_slot, pack_ijk, pack_col_ptr;
  std::vector<int> pack_gid, pack_idx;  // host only: global group and lattice index of each entry (plan checks)
  long long send_total = 0, recv_total = 0;
};

struct ShardPlan3D {
  int P = 1, r = 0, rep_level = 0, colors = 8;
  int s0 = 0, count = 0;       // this shard's slot range
  std::vector<int> starts;     // P + 1
  std::vector<ShardLevel3D> lev;  // per level; empty tables on replicated levels
  bool sharded(int l) const { return l > rep_level && P > 1; }
};

// balanced contiguous slot ranges
std::vector<int> shard_starts(int M, int P);
ShardPlan3D build_shard_plan(const Hierarchy3D& h, int P, int r, int rep_level);

}  // namespace kb
