// Host-side hierarchical hybrid grid over a conforming 3-d macro mesh of
// tetrahedra (BASELINE.json configs 3-5).  The reference has no 3-d solver
// (proj/src/hhg.cpp:49-50 throws for dim != 2), so this
// is the builder's design, written in the style of the 2-d reference
// (proj/src/hhg.cpp:48-144, proj/src/fem.cpp:62-93) and restated
// independently by the CPU oracle (oracle/klref_oracle3d.c):
//
//  * each macro tet carries the structured lattice {(i,j,k) >= 0, i+j+k <= n},
//    n = 2^l, node x = P0 + (i/n)(P1-P0) + (j/n)(P2-P0) + (k/n)(P3-P0); index
//    k-major, each k-plane a 2-d lattice of size n-k (lattice_index3);
//  * micro-tets are the Freudenthal (Kuhn) refinement: base node + one of six
//    step orders of u1 = (1,0,0), u2 = (-1,1,0), u3 = (0,-1,1) (kKuhn), n^3
//    cells per macro, nested across levels; 15-point stencil (kDir);
//  * interface copies: every lattice-boundary node belongs to a shared-node
//    group identified by its integer barycentric weights on global vertex ids
//    (vertex groups, then edge groups, then face groups, each in key order);
//    members in ascending slot, owner = lowest slot (as proj/src/hhg.cpp:95-132);
//  * smoother colouring: a vertex colouring g(v) of the macro mesh in Z_2^m
//    (tet vertices pairwise distinct); node colour = XOR of g(v) over vertices
//    with odd weight -- stencil neighbours always differ in colour.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace kb {

inline int tet_size(int n) { return (n + 1) * (n + 2) * (n + 3) / 6; }
// k-major: plane k is a 2-d lattice of size n - k
inline int lattice_index3(int n, int i, int j, int k) {
  const int m = n - k;
  return tet_size(n) - tet_size(n - k) + j * (m + 1) - (j * (j - 1)) / 2 + i;
}

// the six Freudenthal step orders (permutations of u1, u2, u3)
constexpr int kKuhn[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
constexpr int kStep[3][3] = {{1, 0, 0}, {-1, 1, 0}, {0, -1, 1}};
// the 15 stencil directions: centre, then +/- (u1, u2, u3, u1+u2, u2+u3, u1+u3, u1+u2+u3)
constexpr int kDir[15][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0}, {-1, 1, 0}, {1, -1, 0},
                             {0, -1, 1}, {0, 1, -1}, {0, 1, 0},  {0, -1, 0}, {-1, 0, 1},
                             {1, 0, -1}, {1, -1, 1}, {-1, 1, -1}, {0, 0, 1}, {0, 0, -1}};
int dir_index(int di, int dj, int dk);  // -1 if not a stencil direction

// vertex r of micro-cell (base, type): base + prefix sum of its first r steps
inline void cell_vertex(int type, int r, int& di, int& dj, int& dk) {
  di = dj = dk = 0;
  for (int q = 0; q < r; ++q) {
    di += kStep[kKuhn[type][q]][0];
    dj += kStep[kKuhn[type][q]][1];
    dk += kStep[kKuhn[type][q]][2];
  }
}

struct Mesh3D {
  std::vector<double> x, y, z;
  std::vector<std::array<int, 4>> tet;  // corner vertex ids per slot (positively oriented)
  std::vector<double> vol;
  static Mesh3D create(int num_vertices, const double* xyz, int num_elements, const int* tet4);
};

struct Level3D {
  int n = 1, S = 4;
  std::int64_t dofs = 0;
  // shared-node groups (vertex, edge, face), members ascending slot
  std::vector<int> grp_ptr, mem_slot, mem_idx;
  std::vector<std::uint8_t> grp_domain;  // group on the domain boundary
  std::vector<int> grp_color;
  // dense per-copy tables (M * S)
  std::vector<int> node_gid;             // -1 for lattice-interior nodes
  std::vector<std::uint8_t> node_flags;  // bit0 lattice boundary, bit1 domain boundary, bit2 owner
  // per macro: element matrices [type][4][4] (stiffness, mass), interior stencil, 1/s0
  std::vector<double> kstiff, kmass;     // 96 per macro each
  std::vector<double> stencil;           // 15 per macro (kDir order)
  // partial stencils of lattice-boundary nodes, by boundary signature
  // (i == 0 | j == 0 << 1 | k == 0 << 2 | w0 == 0 << 3): 16 x 15 per macro
  std::vector<double> psK, psM;
  std::vector<double> inv_c;
  std::vector<int> pat_color;            // 8 per macro: colour of the parity pattern (i&1 | (j&1)<<1 | (k&1)<<2)
  std::vector<int> color_grp_ptr, color_grp;  // boundary groups by colour
  std::vector<double> grp_diag;          // sum over members of the partial diagonals
};

struct Hierarchy3D {
  Mesh3D mesh;
  int L = 0, M = 0, colors = 8;
  std::vector<Level3D> levels;
  static Hierarchy3D build(const Mesh3D& mesh, int max_level);
};

inline int boundary_signature(int n, int i, int j, int k) {
  return (i == 0) | ((j == 0) << 1) | ((k == 0) << 2) | ((i + j + k == n) << 3);
}

// element matrices of one micro-tet with physical vertices p[4][3]
void tet_matrices(const double p[4][3], double* K16, double* M16);

}  // namespace kb
