// Device-side views of the 3-d HHG tables and the 3-d kernel launch API
// (kernels3d.cu).  Grid functions are fp64 arrays of M * S_l doubles,
// macro-major, each macro a k-major tet lattice (lattice_index3) with
// interface copies.  Unlike the 2-d path there are no dense per-copy tables:
// lattice-interior nodes are recognised from (i, j, k), every
// lattice-boundary copy is reached through its shared-node group.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dev2d.hpp"
#include "hier3d.hpp"

namespace kb {

struct DevLevel3D {
  int n, S, M, ng, colors;
  const int* grp_ptr;
  const int* mem_slot;
  const int* mem_ijk;          // i | j << 10 | k << 20
  const std::uint8_t* grp_domain;
  const double* grp_diag;
  const int* color_grp_ptr;    // boundary groups by colour
  const int* color_grp;         // per colour: wide groups (> 4 members) first
  const int* color_wide_end;    // per colour: end of its wide groups in color_grp
  int max_color_groups;         // largest colour (groups): sizes the cooperative smoother's grid
  // flat records of the groups at their position t in color_grp: header
  // (diagonal lo, hi, members | domain << 16, first member in wide_mem) and, for
  // narrow groups (<= 4 members), four member slots (macro slot, i | j << 10 |
  // k << 20) at 4 t; wide groups keep theirs contiguous in wide_mem; null on
  // shard tables
  const int4* nar_hdr;
  const int2* nar_mem;
  const int2* wide_mem;
  const double* kstiff;        // 96 per macro: [type][4][4]
  const double* kmass;
  const double* stK;           // 15 per macro (kDir order)
  const double* stM;
  const double* inv_c;
  const int* pat_color;        // 8 per macro
  const int* col_pat;          // colors per macro: the parity pattern of that colour, -1 none
  // 4 <= n <= 64: a macro's lattice-interior nodes (lat2(n - k, i, j) | j << 16)
  // in the smoother's order, step (plane k, parity class q) at
  // [pat_ptr[4 (k - 1) + q], pat_ptr[4 (k - 1) + q + 1]); pat_max nodes at most; else null
  const int* pat_ptr;
  const int* pat_node;
  int pat_max;
  const int* own_dot;          // group owner copy offsets (dot order)
  const double* psK;           // boundary partial stencils: 16 signatures x 15 per macro
  const double* psM;
  // level-0 CG on the unique macro-vertex values (level 0 only): the assembled
  // operator rows (row g = group g = macro vertex g; columns are vertex ids)
  const int* cg_rowptr;        // ng + 1
  const unsigned short* cg_col;
  const double* cg_val;
  int cg_nnz;
  // sharded levels (solver3d_shard.cpp): a member with mem_slot < 0 lives on
  // another shard; its contribution (partial row or copy value, as the
  // operation needs) is ghost[~mem_slot], received by the exchange before the
  // kernel runs, and its copy is written by its own shard
  const double* ghost;
};

enum Apply3Mode : int {
  A3_PLAIN = 0,     // y = Op x, every copy
  A3_RESIDUAL = 1,  // r = b - A u, domain-boundary copies 0
  A3_RES_OWNER = 2, // residual for restriction: non-owner and domain copies 0
};
enum Prolong3Mode : int { P3_ASSIGN = 0, P3_ADD = 1 };

void launch3_apply(const DevLevel3D& lv, bool mass, const double* x, double* y, const double* b, int mode,
                   cudaStream_t st);
// smoother: one cooperative launch (boundary colours, then per-macro interior
// colours; KB_GS3_SPLIT=1 selects the per-colour launches)
void launch3_gs(const DevLevel3D& lv, double* u, const double* b, int sweeps, cudaStream_t st);
int launch3_gs_count(const DevLevel3D& lv, int sweeps);
int launch3_apply_count(const DevLevel3D& lv);     // kernels per launch3_apply
int launch3_estimate_count(const DevLevel3D& lv);  // kernels per launch3_estimate
void launch3_prolong(const DevLevel3D& coarse, const DevLevel3D& fine, const double* c, double* f, int mode,
                     cudaStream_t st);
// restriction of an owner-masked fine vector (A3_RES_OWNER residual), then
// coarse additive sync; zero_domain: coarse domain-boundary copies 0
void launch3_restrict(const DevLevel3D& fine, const DevLevel3D& coarse, const double* rf, double* rc,
                      int zero_domain, cudaStream_t st, double* zero_out = nullptr);
// the restriction alone over coarse.M macros (no sync; sharded levels)
void launch3_restrict_only(const DevLevel3D& fine, const DevLevel3D& coarse, const double* rf, double* rc,
                           cudaStream_t st);
// interface sync with optional zero of the domain-boundary copies
void launch3_sync_zero(const DevLevel3D& lv, double* f, int additive, int zero_domain, cudaStream_t st);
// zero the non-owner copies of f into out (single-operation restriction)
void launch3_owner_mask(const DevLevel3D& lv, const double* f, double* out, cudaStream_t st);
// set domain-boundary copies to g (per group); zero_rest: other nodes 0
void launch3_set_boundary(const DevLevel3D& lv, double* f, const double* g_grp, int zero_rest, cudaStream_t st);
void launch3_sync(const DevLevel3D& lv, double* f, int additive, cudaStream_t st);
void launch3_cg0(const DevLevel3D& lv0, double* u, const double* b, double* scratch, CgParams prm,
                 DevStatus* status, cudaStream_t st);
// per-macro sums of e^T M e for e_base = uL - wb and e_coarser = uL - wc (all on level L)
// part: scratch of 2 M (n + 1) doubles
void launch3_estimate(const DevLevel3D& lv, const double* uL, const double* wb, const double* wc, double* sums,
                      double* part, cudaStream_t st);
void launch3_dot(const DevLevel3D& lv, const double* a, const double* b, double* partial, double* out,
                 cudaStream_t st);
// exchange pack: out[pos[e]] = contribution of local member e (slot, ijk) for
// the entries [e0, e1): mode 0 copy value of x, 1 stiffness partial row of x,
// 2 mass partial row of x, 3 off-diagonal stiffness partial row (smoother)
enum Pack3Mode : int { PK3_VALUE = 0, PK3_FULL_K = 1, PK3_FULL_M = 2, PK3_OFF_K = 3 };
void launch3_pack(const DevLevel3D& lv, int mode, const double* x, const int* pos, const int* slot, const int* ijk,
                  int e0, int e1, double* out, cudaStream_t st);
// boundary colour c of the smoother alone (one group per thread)
void launch3_gs_color_groups(const DevLevel3D& lv, double* u, const double* b, int c, cudaStream_t st);
// interior phase of the smoother alone (every macro, all colours, one sweep)
void launch3_gs_interior(const DevLevel3D& lv, double* u, const double* b, cudaStream_t st);
void launch3_axpy(double* y, const double* x, double alpha, std::int64_t count, cudaStream_t st);

}  // namespace kb
