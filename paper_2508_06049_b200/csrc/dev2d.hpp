// Device-side views of the 2-d HHG tables and the kernel launch API
// (implemented in kernels2d.cu).  Everything is fp64; grid functions are
// stored macro-major with interface copies, each macro in the reference's
// row-major lattice order (proj/include/klref/hhg.hpp:13, :33-53), so a
// level-l function is one contiguous array of M * S_l doubles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "hier2d.hpp"

namespace kb {

// Dynamic shared memory above 48 KB needs the per-kernel opt-in, which is a
// per-device attribute.  The high-water mark is kept per (device, kernel)
// under a mutex and only ever grows: graph nodes captured earlier keep their
// (larger) launch sizes valid when a later launch of the same kernel needs less.
template <typename K>
inline void ensure_dynamic_smem(K kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> high;
  if (smem <= 48 * 1024) return;
  int dev = 0;
  KB_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& hw = high[{dev, reinterpret_cast<const void*>(kernel)}];
  if (smem <= hw) return;
  KB_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  hw = smem;
}

struct DevLevel2D {
  int n, S, M;
  const int* node_gid;
  const std::uint8_t* node_flags;
  const int* grp_ptr;
  const int* mem_off;
  const int* mem_ij;   // i | (j << 16)
  const int* mem_slot;
  const double* kstiff;
  const double* kmass;
  const double* stencil;
  const double* inv_c;
  const BNode* bnode;
  const MemberRec* rec;
  const int* wr;
  const int* ghost_ptr;
  const int* ghost_off;
  int max_ghosts;
  int num_groups;
  const int* dot_order;
  int dot_count;
  const unsigned long long* prog;        // smoother step programs (Level2D::prog)
  const long long* prog_ptr;
  const unsigned long long* prog_extra;  // vertex-group members beyond the second
  const int* xtra_ptr;
  int max_extra;
  const double* geo;   // per macro: c0x, c0y, ux, uy, wx, wy (RHS quadrature map, proj/src/fem.cpp:183-186)
  const double* wq;    // per macro: cell_area / 3
  // static Gauss-Seidel schedules (Level2D::sched; sc_blocks[s - 1] null when absent)
  int sc_nu;
  const int* sc_cell_copy;
  const int* sc_copy_cell;
  const double* sc_mtab;
  const double* sc_gtab;
  const int* sc_blocks[2];
  const int* sc_lev_off[2];
  int sc_levels[2], sc_max_width[2], sc_max_block[2], sc_max_members[2];
  // pipelined smoother tables (Level2D::pipe; null when absent)
  const int* pipe_rec;
  int pipe_rec_words, pipe_maxreq;
  // level 0 only: the coarse operator over unique DoF in dot_unique order
  // (k_cg0): per DoF the member range, per member the three (coefficient,
  // DoF) terms of its cell row, per DoF the copy offsets to write back
  int cg_nmem, cg_ncopy;
  const int* cg_mem_ptr;      // dot_count + 1
  const int* cg_mem_dof;      // 3 per member
  const double* cg_mem_coef;  // 3 per member
  const int* cg_copy_ptr;     // dot_count + 1
  const int* cg_copy;         // copy offsets
};

struct DevHier2D {
  int M, L;
  const int* nb_lo_ptr;
  const int* nb_lo;
  const int* nb_hi_ptr;
  const int* nb_hi;
  int dag_depth, dag_width;  // number of DAG levels, most macros in one level
  const int* dag_ptr;
  const int* dag_list;
};

// Kernel kinds for the per-kernel probes (KLREF_KERNEL_* in include/klref_b200.h).
enum KernelKind : int {
  KK_GS = 0,        // Gauss-Seidel sweeps
  KK_RESIDUAL = 1,  // r = b - A u
  KK_RESTRICT = 2,
  KK_PROLONG = 3,   // prolongation (+ correction / w snapshot)
  KK_RHS = 4,       // right-hand side + Dirichlet rows
  KK_CG0 = 5,       // level-0 CG
  KK_ESTIMATE = 6,  // fused estimator norms (+ its prolongations)
  KK_OTHER = 7,     // boundary init, memsets
  KK_COUNT = 8
};

enum ApplyMode : int { APPLY_PLAIN = 0, APPLY_RESIDUAL = 1, APPLY_ZERO_BND = 2 };
enum ProlongMode : int { PROLONG_ASSIGN = 0, PROLONG_ADD = 1, PROLONG_W_NEXT = 2 };

// Device problem descriptor for the source term (fast mode); faithful mode
// passes a host-tabulated f instead (RHS).
enum SourceKind : int { SRC_ZERO = 0, SRC_TABLE = 1, SRC_SIN2D = 2 };

struct CgParams {
  double rel_tol, abs_floor;
  int max_iter;
};

// status word written by device code (level-0 CG failures)
struct DevStatus {
  int code;       // 0 ok, 1 not converged, 2 lost positive definiteness
  int iters;
  double residual;
};

// y = Op x (+ residual / boundary modes); K = kstiff or kmass of the level
void launch_apply(const DevLevel2D& lv, const double* K, const double* x, double* y, const double* b,
                  int mode, cudaStream_t st);
void launch_restrict(const DevLevel2D& fine, const DevLevel2D& coarse, const double* r, double* rc,
                     int zero_boundary, cudaStream_t st, double* zero_out = nullptr);
void launch_prolong(const DevLevel2D& coarse, const DevLevel2D& fine, const double* c, double* f,
                    double* next, const double* gbnd, int mode, cudaStream_t st);
void launch_set_boundary(const DevLevel2D& lv, double* f, const double* gbnd, int zero_rest,
                         cudaStream_t st);
void launch_rhs(const DevLevel2D& lv, int src_kind, const double* ftab, double* ftab_scratch,
                const double* gbnd, double* b, cudaStream_t st);
void launch_cg0(const DevLevel2D& lv0, double* u, const double* b, double* scratch, CgParams prm,
                DevStatus* status, cudaStream_t st);
void launch_gs(const DevHier2D& hd, const DevLevel2D& lv, double* u, const double* b, int sweeps,
               int* done, cudaStream_t st);
// ExactErrorEvaluator::evaluate terms (proj/src/fem.cpp:395-420): per macro
// cross = sum_k moments[k] u[k] and uh_sq = sum over cells of the mass form,
// both in the reference's sequential order (one thread per macro);
// out[2 m] = cross, out[2 m + 1] = uh_sq
void launch_exact_eval(const DevLevel2D& lv, const double* uL, const double* moments, double* out, cudaStream_t st);
void launch_estimate(const DevLevel2D& lv, const double* uL, const double* wb, const double* wc,
                     double* sums, cudaStream_t st);
void launch_dot(const DevLevel2D& lv, const double* a, const double* b, double* partial,
                double* out, cudaStream_t st);
// dot_unique in the reference's sequential owner order (single warp)
void launch_dot_seq(const DevLevel2D& lv, const double* a, const double* b, double* out, cudaStream_t st);
void launch_sync(const DevLevel2D& lv, double* f, int additive, cudaStream_t st);
void launch_axpy(double* y, const double* x, double alpha, std::int64_t count, cudaStream_t st);
// y = y * beta; y = y + 1.0 * x  (GridFunction::scale then add_scaled(x, 1.0))
void launch_scale_add(double* y, double beta, const double* x, std::int64_t count, cudaStream_t st);
int gs_block_threads(int n);

}  // namespace kb
