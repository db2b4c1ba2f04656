// Host-side hierarchical hybrid grid (HHG) over a conforming 2-d macro mesh:
// shared-node groups, ownership, per-macro element matrices and the derived
// device tables used by the sm_100a kernels (kernels2d.cu).
//
// Semantics follow the reference GridHierarchy (proj/src/hhg.cpp:48-144) and
// OperatorP1 (proj/src/fem.cpp:62-93) with the two defects fixed:
//   D1: element matrices use |area| (proj/src/fem.cpp:32);
//   D2: edge-node groups are addressed by the position counted from the edge's
//       lower-id corner (proj/src/hhg.cpp:170-172 vs :114-123).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>

#include "common.hpp"

namespace kb {

// Conforming 2-d macro mesh in slot order (ascending active element id).
// Equivalent of the parts of MacroMesh (proj/include/klref/macro_mesh.hpp:62)
// the hot path reads: vertex coordinates, vertex boundary flags, element
// corner ids (oriented counter-clockwise as MacroMesh::create does,
// proj/src/macro_mesh.cpp:206-216) and element areas.
struct Mesh2D {
  std::vector<double> x, y;
  std::vector<std::uint8_t> boundary;   // recomputed from edge use, proj/src/macro_mesh.cpp:306-318
  std::vector<std::array<int, 3>> tri;  // corner vertex ids per slot
  std::vector<double> area;             // signed_area, proj/src/macro_mesh.cpp:28-30

  static Mesh2D create(int num_vertices, const double* xy, int num_elements, const int* tri3);
};

struct MacroEdgeInfo {
  int group_start = -1;
  bool owner = false;
  bool domain_boundary = false;
};
struct MacroLevel {
  std::array<int, 3> corner_group{-1, -1, -1};
  std::array<bool, 3> corner_owner{false, false, false};
  std::array<bool, 3> corner_boundary{false, false, false};
  std::array<MacroEdgeInfo, 3> edge{};
};

// Relaxation record of one group member for the wavefront Gauss-Seidel:
// partial_row (proj/src/fem.cpp:128-173) of member `slot` at its local node,
// with every x-read resolved either to a neighbour of the relaxing node in the
// relaxing macro (codes 0..5 = E, W, N, S, NW, SE) or to a ghost value of a
// node the relaxing macro does not hold (code 6 + ghost index).
struct MemberRec {
  std::int32_t slot;
  std::int32_t mask;       // existing cells, bit k in the partial_row order
  std::int16_t code[12];   // two reads per cell, in partial_row order
  // the same reads as lattice indices of the relaxing macro (>= 0) or ghost
  // values (-1 - ghost index), for the shared-memory smoother
  std::int16_t loc[12];
};
struct BNode {
  std::int32_t rec_begin, rec_count;
  std::int32_t wr_begin, wr_count;  // other copies to write
  std::int32_t domain;              // on the domain boundary: u = b
  std::int32_t pad;
  double diag;                      // sum over members of the partial diagonals
};

// lane record: c[6] diag inv (8 doubles) | loc[6] k flags wr0 wr1 wb wc xb nc (16 int32)
constexpr int kProgLaneWords = 16;                        // 128 bytes
constexpr int kProgStepWords = 6 * kProgLaneWords;        // 3 node types x 2 members
// shared-memory budget of the static schedule's resident tables (u, b, macro and group tables)
constexpr std::size_t kSchedTableBytes = 80 * 1024;  // end of round 2: above it the pipelined smoother is faster (sweep in DESIGN.md)
constexpr int kSchedMemberWords = 20;

// Exact-order Gauss-Seidel of a small level as a static schedule
// (gs_sched2d.cpp, kernels2d.cu k_gs_sched).  The reference's sequential
// relaxations (sweep, slot, row j, node i; an interface node is
// re-relaxed by every member macro) are levelled by their true data
// dependences on the unique node values (read-after-write, write-after-read,
// write-after-write), so every dependence-level is a set of independent
// relaxations and executing the levels in order with a barrier between them
// reproduces the sequential result bit for bit -- with far fewer barrier
// steps than the macro DAG x wavefront schedule (cfg2 k=5, 2 sweeps: 152
// levels at l = 1, 372 at l = 3).
//
// Block of one level (int32 words, 16-byte aligned): [count, 0 x 7], then
// `count` 8-word headers, then the member records of its group relaxations:
//   interior  {cell, macro, E, W, N, S, NW, SE}        (cells of the neighbours)
//   group     {cell, -1 - group, member word offset in the block, members (-1: domain
//              boundary, u = b), diag (double), RN(1/diag) (double)}
//   member    {c0 .. c5 (doubles), r0 .. r5, cells, 0}  (partial_row terms in order:
//              coefficient, read; 20 words)
struct GsSched2D {
  int sweeps = 0, levels = 0, max_width = 0, max_block_words = 0, max_members = 0;
  std::vector<std::int32_t> blocks;
  std::vector<std::int32_t> lev_off;  // word offset of each level block (levels + 1)
};

// Fine-grained pipelined smoother of larger levels (pipe2d.cpp, kernels2d.cu
// k_gs_pipe): one CTA per macro sweeps its lattice in shared memory along the
// wavefront while the other macros run concurrently; the
// reference's sequential order across macros (A.1/A.3) is enforced per
// wavefront step instead of per sweep.  For every macro m, sweep s (0, 1) and
// step t a record lists the gate of the step -- progress[m2] >= p for the
// other macros whose writes this step's reads need (RAW) or whose reads of
// global values this step's writes would clobber (WAR, WAW) -- and the values
// to re-read from global memory before the step (interface copies other
// macros relaxed, ghost values of neighbouring lattices).  progress[m] counts
// completed steps + 1 (published after every step); a fetch for step tau is
// done by the end of step tau - 1 of its macro.
//   record: kPipeLanes int4 entries (rec_words = 4 kPipeLanes), entry k =
//   {k-th requirement: macro or -1, progress; k-th fetch: source global
//   offset or -1, destination: lattice index >= 0 or -1 - ghost slot}
constexpr int kPipeLanes = 16;
struct PipeTables2D {
  bool ok = false;
  int maxreq = 0, maxfetch = 0, rec_words = 0;
  std::vector<std::int32_t> rec;  // [M][sweep 0, 1][2n + 1] records
};

struct Level2D {
  int n = 1, S = 3;
  // shared-node groups (vertex groups first, then edge groups), members ascending slot
  std::vector<int> grp_ptr;
  std::vector<int> mem_slot, mem_i, mem_j, mem_idx;
  std::vector<MacroLevel> macros;
  std::int64_t dofs = 0;
  // dense per-copy tables (M * S)
  std::vector<int> node_gid;               // -1 for lattice-interior nodes
  std::vector<std::uint8_t> node_flags;    // bit0 lattice boundary, bit1 domain boundary, bit2 owner
  // per macro element matrices: [up(9), down(9)]
  std::vector<double> kstiff, kmass;
  std::vector<double> stencil;             // 7 per macro (C, E, W, N, S, NW, SE), proj/src/fem.cpp:85-91
  std::vector<double> inv_c;               // 1 / stencil[0]
  // wavefront Gauss-Seidel tables (levels >= 1)
  std::vector<BNode> bnode;                // M * 3n, boundary position order (see bpos())
  std::vector<MemberRec> rec;
  std::vector<int> wr;                     // global copy offsets
  std::vector<int> ghost_ptr, ghost_off;   // per macro ghost lists (global offsets)
  int max_ghosts = 0;
  // Step programs of the shared-memory smoother (kernels2d.cu, k_gs_*): for
  // every macro and wavefront step t = 0..2n, six pre-decoded lane records
  // (boundary-node type x group member 0/1) of kProgLaneBytes: the compact
  // partial_row of that member (existing cells only, in the order of
  // proj/src/fem.cpp:138-172; reads are lattice indices of the relaxing macro
  // or ghost slots -1-g) plus the node's lattice index, flags, copy targets,
  // diag and RN(1/diag).  Members beyond the second (vertex groups) are lane
  // records in prog_extra; prog_ptr[m] / xtra_ptr[m] are 8-byte-word offsets.
  std::vector<std::uint64_t> prog, prog_extra;
  std::vector<long long> prog_ptr;
  std::vector<int> xtra_ptr;
  int max_extra = 0;  // most extra records of one macro
  // owner dot order (dot_unique, proj/src/hhg.cpp:227-257): offsets in summation order
  std::vector<int> dot_order;
  // static Gauss-Seidel schedules (sched[s - 1]: s sweeps; empty when the level
  // does not fit one CTA's shared memory).  Unique node values: groups first,
  // then lattice-interior nodes in copy order.
  int sc_nu = 0;
  std::vector<int> sc_cell_copy;   // per unique node: the owner copy (gather)
  std::vector<int> sc_copy_cell;   // per copy: its unique node (scatter)
  std::vector<double> sc_mtab;     // per macro: s1..s6, 1/s0, 0, K_up(9), K_down(9)
  std::vector<double> sc_gtab;     // per group: diag, RN(1/diag)
  GsSched2D sched[2];
  PipeTables2D pipe;
};

// Boundary position of lattice-boundary node (i, j): row 0 first, then the
// i = 0 edge, then the hypotenuse.
inline int bpos(int n, int i, int j) {
  if (j == 0) return i;
  if (i == 0) return n + j;
  return 2 * n + j;
}

struct Hierarchy2D {
  Mesh2D mesh;
  int L = 0;
  int M = 0;
  std::vector<Level2D> levels;
  // vertex-sharing neighbours per macro (level independent): lower and higher slots
  std::vector<int> nb_lo_ptr, nb_lo, nb_hi_ptr, nb_hi;
  int dag_depth = 0;
  // macros grouped by DAG level: dag_list[dag_ptr[d] .. dag_ptr[d+1])
  std::vector<int> dag_ptr, dag_list;

  static Hierarchy2D build(const Mesh2D& mesh, int max_level);
  // static Gauss-Seidel schedules of the levels that fit (gs_sched2d.cpp)
  void build_gs_schedules();
  // pipelined-smoother tables of the levels the schedule does not cover (pipe2d.cpp)
  void build_pipe_tables();

  // boundary_group with the D2 fix (proj/src/hhg.cpp:163-174)
  int boundary_group(int slot, int l, int i, int j) const;
  bool on_domain_boundary(int slot, int l, int i, int j) const;
  bool owns_boundary_node(int slot, int l, int i, int j) const;
  // node_coordinates, proj/src/hhg.cpp:146-154
  void node_coordinates(int slot, int l, int i, int j, double& x, double& y) const;
};

}  // namespace kb
