// sm_100a kernels of the 2-d hot path (fp64, memory/latency bound, no tensor
// cores).  Compiled with -fmad=false: every kernel reproduces the reference's
// floating-point operation order so that results are
// bitwise identical to the (patched) reference.
//
//   apply / residual     OperatorP1::apply + interface_sync(Additive)   proj/src/fem.cpp:95-126
//                        MultigridSolver::residual                      proj/src/multigrid.cpp:183-190
//   restrict             restrict_transpose                             proj/src/multigrid.cpp:55-104
//   prolong              prolongate / u += P e / FMG w snapshot          proj/src/multigrid.cpp:22-53, 243, 265-268
//   rhs                  assemble_rhs + set_domain_boundary_values      proj/src/fem.cpp:175-228
//   cg0                  MultigridSolver::cg_level0                     proj/src/multigrid.cpp:198-229
//   gs                   MultigridSolver::gauss_seidel                  proj/src/multigrid.cpp:127-181
//   estimate             error_estimate norms                           proj/src/estimator.cpp:8-45, fem.cpp:320-356
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include "dev2d.hpp"

// Measurement traces (per-step clock stamps, printf timelines) are compiled in
// only with -DKB_GS_TRACE (Makefile NVDEFS); production kernels carry none.
#ifdef KB_GS_TRACE
#define KB_TRACING(x) (x)
#else
#define KB_TRACING(x) false
#endif

namespace kb {
namespace {

constexpr int kThreads = 256;

#ifdef KB_GS_TRACE
__device__ int g_lvl_item;
__device__ long long g_gs_trace[4][1 << 12];  // debug builds only: per-step clocks of block 0
__device__ int g_dbg_S, g_dbg_G, g_dbg_MS;
#define KB_CHECK(cond, code, a, b)                                                        \
  do {                                                                                    \
    if (!(cond) && atomicCAS(reinterpret_cast<unsigned long long*>(&g_gs_trace[3][4000]), 0ull, 1ull) == 0ull) { \
      g_gs_trace[3][4001] = (code);                                                       \
      g_gs_trace[3][4002] = (a);                                                          \
      g_gs_trace[3][4003] = (b);                                                          \
    }                                                                                     \
  } while (0)
#else
#define KB_CHECK(cond, code, a, b) \
  do {                             \
  } while (0)
#endif

// KB_GS_CHECK builds (verification, not product): the shared-memory slots,
// lattice indices and global offsets the smoothers take from host tables are
// bounds-checked on the device; a violation traps (the parity tests then fail
// with an illegal-instruction error instead of reading or writing out of range)
#ifdef KB_GS_CHECK
#define KB_ASSERT(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define KB_ASSERT(cond) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ int dlat(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }

__device__ __forceinline__ void decode(int n, int idx, int& i, int& j) {
  const double a = 2.0 * n + 3.0;
  int jj = static_cast<int>((a - sqrt(a * a - 8.0 * idx)) * 0.5);
  jj = max(0, min(jj, n));
  while (jj < n && dlat(n, 0, jj + 1) <= idx) ++jj;
  while (jj > 0 && dlat(n, 0, jj) > idx) --jj;
  j = jj;
  i = idx - dlat(n, 0, jj);
}

// Gather form of the reference element scatter: the <= 6 incident cells of
// node (p, q) in the reference's visit order (SURVEY.md A.5 "apply").
__device__ __forceinline__ double gather_apply(const double* __restrict__ x, int n, int p, int q,
                                               const double* __restrict__ K) {
  const double* ku = K;
  const double* kd = K + 9;
  double acc = 0.0;
  if (q >= 1 && p + q <= n)  // up(p, q-1) as c
    acc += (ku[6] * x[dlat(n, p, q - 1)] + ku[7] * x[dlat(n, p + 1, q - 1)]) + ku[8] * x[dlat(n, p, q)];
  if (p >= 1 && q >= 1 && p + q <= n)  // down(p-1, q-1) as c
    acc += (kd[6] * x[dlat(n, p, q - 1)] + kd[7] * x[dlat(n, p - 1, q)]) + kd[8] * x[dlat(n, p, q)];
  if (q >= 1 && p + q <= n - 1)  // down(p, q-1) as b
    acc += (kd[3] * x[dlat(n, p + 1, q - 1)] + kd[4] * x[dlat(n, p, q)]) + kd[5] * x[dlat(n, p + 1, q)];
  if (p >= 1 && p + q <= n)  // up(p-1, q) as b
    acc += (ku[3] * x[dlat(n, p - 1, q)] + ku[4] * x[dlat(n, p, q)]) + ku[5] * x[dlat(n, p - 1, q + 1)];
  if (p + q <= n - 1)  // up(p, q) as a
    acc += (ku[0] * x[dlat(n, p, q)] + ku[1] * x[dlat(n, p + 1, q)]) + ku[2] * x[dlat(n, p, q + 1)];
  if (p >= 1 && p + q <= n - 1)  // down(p-1, q) as a
    acc += (kd[0] * x[dlat(n, p, q)] + kd[1] * x[dlat(n, p - 1, q + 1)]) + kd[2] * x[dlat(n, p, q + 1)];
  return acc;
}

__device__ __forceinline__ void write_out(int mode, double v, int k, double* y, const double* b,
                                          const std::uint8_t* flags) {
  if (mode == APPLY_RESIDUAL) {
    // r = (-y) + 1.0 * b, then zero_domain_boundary (proj/src/multigrid.cpp:185-188)
    y[k] = (flags[k] & 2) ? 0.0 : (b[k] - v);
  } else if (mode == APPLY_ZERO_BND) {
    y[k] = (flags[k] & 2) ? 0.0 : v;
  } else {
    y[k] = v;
  }
}

// One copy k of the level: interior nodes directly; lattice-boundary nodes are
// produced by the group leader (first member) as the ascending-slot sum of the
// members' macro-local products, written to every copy (interface_sync Additive).
__device__ __forceinline__ void apply_node(const DevLevel2D& lv, const double* __restrict__ K,
                                           const double* __restrict__ x, double* y,
                                           const double* b, int mode, int k) {
  const int S = lv.S, n = lv.n;
  const int slot = k / S;
  const int idx = k - slot * S;
  int i, j;
  decode(n, idx, i, j);
  const std::uint8_t fl = lv.node_flags[k];
  if (!(fl & 1)) {
    write_out(mode, gather_apply(x + static_cast<size_t>(slot) * S, n, i, j, K + 18 * slot), k, y, b,
              lv.node_flags);
    return;
  }
  const int gid = lv.node_gid[k];
  const int beg = lv.grp_ptr[gid], end = lv.grp_ptr[gid + 1];
  if (lv.mem_off[beg] != k) return;
  double v;
  if (end - beg == 1) {
    v = gather_apply(x + static_cast<size_t>(slot) * S, n, i, j, K + 18 * slot);
  } else {
    v = 0.0;
    for (int m = beg; m < end; ++m) {
      const int ms = lv.mem_slot[m], ij = lv.mem_ij[m];
      v += gather_apply(x + static_cast<size_t>(ms) * S, n, ij & 0xffff, ij >> 16, K + 18 * ms);
    }
  }
  for (int m = beg; m < end; ++m) write_out(mode, v, lv.mem_off[m], y, b, lv.node_flags);
}

__global__ void k_apply(DevLevel2D lv, const double* __restrict__ K, const double* __restrict__ x,
                        double* y, const double* b, int mode) {
  const int total = lv.M * lv.S;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x)
    apply_node(lv, K, x, y, b, mode, k);
}

// Level-wide apply / residual, split by node kind in one launch:
//  * blocks [0, interior_blocks): 256 consecutive lattice indices of one macro
//    each; lattice-interior nodes evaluate the reference's six-cell gather with
//    all cells present (no branches, 7 loads, the same operation order as
//    gather_apply), lattice-boundary nodes are skipped;
//  * the remaining blocks: one shared-node group per thread -- members'
//    partial gathers summed in ascending slot (interface_sync Additive),
//    written to every copy.
__device__ __forceinline__ void decode_fast(int n, int idx, int& i, int& j) {
  const float a = 2.0f * n + 3.0f;
  int jj = static_cast<int>((a - sqrtf(a * a - 8.0f * idx)) * 0.5f);
  jj = max(0, min(jj, n));
  while (jj < n && dlat(n, 0, jj + 1) <= idx) ++jj;
  while (jj > 0 && dlat(n, 0, jj) > idx) --jj;
  j = jj;
  i = idx - dlat(n, 0, jj);
}

__global__ void __launch_bounds__(256) k_apply2(DevLevel2D lv, const double* __restrict__ K,
                                                const double* __restrict__ x, double* y,
                                                const double* __restrict__ b, int mode, int chunks_per_macro,
                                                int interior_blocks) {
  const int n = lv.n, S = lv.S;
  if (static_cast<int>(blockIdx.x) < interior_blocks) {
    const int m = blockIdx.x / chunks_per_macro;
    const int idx = (blockIdx.x - m * chunks_per_macro) * 256 + threadIdx.x;
    if (idx >= S) return;
    int p, q;
    decode_fast(n, idx, p, q);
    if (p == 0 || q == 0 || p + q == n) return;
    const double* ku = K + 18 * m;
    const double* kd = ku + 9;
    const double* xm = x + static_cast<size_t>(m) * S;
    const int k = idx;
    const double C = xm[k], E = xm[k + 1], W = xm[k - 1];
    const double N = xm[k + n + 1 - q], NW = xm[k + n - q];
    const double Sv = xm[k - (n + 2 - q)], SE = xm[k - (n + 1 - q)];
    // gather_apply order: up(p,q-1) c, down(p-1,q-1) c, down(p,q-1) b,
    // up(p-1,q) b, up(p,q) a, down(p-1,q) a
    double acc = 0.0;
    acc += (__ldg(ku + 6) * Sv + __ldg(ku + 7) * SE) + __ldg(ku + 8) * C;
    acc += (__ldg(kd + 6) * Sv + __ldg(kd + 7) * W) + __ldg(kd + 8) * C;
    acc += (__ldg(kd + 3) * SE + __ldg(kd + 4) * C) + __ldg(kd + 5) * E;
    acc += (__ldg(ku + 3) * W + __ldg(ku + 4) * C) + __ldg(ku + 5) * NW;
    acc += (__ldg(ku + 0) * C + __ldg(ku + 1) * E) + __ldg(ku + 2) * N;
    acc += (__ldg(kd + 0) * C + __ldg(kd + 1) * NW) + __ldg(kd + 2) * N;
    const size_t off = static_cast<size_t>(m) * S + k;
    if (mode == APPLY_RESIDUAL)
      y[off] = b[off] - acc;  // interior nodes are never on the domain boundary
    else
      y[off] = acc;
    return;
  }
  const int g = (blockIdx.x - interior_blocks) * 256 + threadIdx.x;
  if (g >= lv.num_groups) return;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  double v;
  if (end - beg == 1) {
    const int ms = lv.mem_slot[beg], ij = lv.mem_ij[beg];
    v = gather_apply(x + static_cast<size_t>(ms) * S, n, ij & 0xffff, ij >> 16, K + 18 * ms);
  } else {
    v = 0.0;
    for (int q = beg; q < end; ++q) {
      const int ms = lv.mem_slot[q], ij = lv.mem_ij[q];
      v += gather_apply(x + static_cast<size_t>(ms) * S, n, ij & 0xffff, ij >> 16, K + 18 * ms);
    }
  }
  for (int q = beg; q < end; ++q) write_out(mode, v, lv.mem_off[q], y, b, lv.node_flags);
}

// ---------------------------------------------------------------- restrict
__device__ __forceinline__ double gather_restrict(const double* __restrict__ f,
                                                  const std::uint8_t* __restrict__ fl, int nf, int I,
                                                  int J) {
  double c = 0.0;
  // fine visit order (SURVEY.md A.5 "restrict_transpose")
  const int ii[7] = {2 * I, 2 * I + 1, 2 * I - 1, 2 * I, 2 * I + 1, 2 * I - 1, 2 * I};
  const int jj[7] = {2 * J - 1, 2 * J - 1, 2 * J, 2 * J, 2 * J, 2 * J + 1, 2 * J + 1};
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    const int i = ii[t], j = jj[t];
    if (i < 0 || j < 0 || i + j > nf) continue;
    const int k = dlat(nf, i, j);
    const double v = (fl[k] & 4) ? f[k] : 0.0;  // non-owner copies masked (multigrid.cpp:63-76)
    if (v == 0.0) continue;
    c += (t == 3) ? v : 0.5 * v;
  }
  return c;
}

__global__ void k_restrict(DevLevel2D fine, DevLevel2D coarse, const double* __restrict__ r, double* rc,
                           int zero_boundary, double* zero_out) {
  const int total = coarse.M * coarse.S;
  const int Sc = coarse.S, Sf = fine.S, nc = coarse.n, nf = fine.n;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    if (zero_out) zero_out[k] = 0.0;  // the V-cycle's zero initial guess on the coarse level (one launch less)
    const int slot = k / Sc;
    int I, J;
    decode(nc, k - slot * Sc, I, J);
    const std::uint8_t fl = coarse.node_flags[k];
    if (!(fl & 1)) {
      rc[k] = gather_restrict(r + static_cast<size_t>(slot) * Sf, fine.node_flags + static_cast<size_t>(slot) * Sf,
                              nf, I, J);
      continue;
    }
    const int gid = coarse.node_gid[k];
    const int beg = coarse.grp_ptr[gid], end = coarse.grp_ptr[gid + 1];
    if (coarse.mem_off[beg] != k) continue;
    double v;
    if (end - beg == 1) {
      v = gather_restrict(r + static_cast<size_t>(slot) * Sf, fine.node_flags + static_cast<size_t>(slot) * Sf, nf,
                          I, J);
    } else {
      v = 0.0;
      for (int m = beg; m < end; ++m) {
        const int ms = coarse.mem_slot[m], ij = coarse.mem_ij[m];
        v += gather_restrict(r + static_cast<size_t>(ms) * Sf, fine.node_flags + static_cast<size_t>(ms) * Sf, nf,
                             ij & 0xffff, ij >> 16);
      }
    }
    for (int m = beg; m < end; ++m) {
      const int o = coarse.mem_off[m];
      rc[o] = (zero_boundary && (coarse.node_flags[o] & 2)) ? 0.0 : v;
    }
  }
}

// ---------------------------------------------------------------- prolong
__device__ __forceinline__ double prolong_value(const double* __restrict__ c, int nc, int i, int j) {
  if ((i & 1) == 0 && (j & 1) == 0) return c[dlat(nc, i / 2, j / 2)];
  if ((j & 1) == 0) return 0.5 * (c[dlat(nc, (i - 1) / 2, j / 2)] + c[dlat(nc, (i + 1) / 2, j / 2)]);
  if ((i & 1) == 0) return 0.5 * (c[dlat(nc, i / 2, (j - 1) / 2)] + c[dlat(nc, i / 2, (j + 1) / 2)]);
  return 0.5 * (c[dlat(nc, (i + 1) / 2, (j - 1) / 2)] + c[dlat(nc, (i - 1) / 2, (j + 1) / 2)]);
}

__device__ __forceinline__ int bpos_dev(int n, int i, int j) {
  if (j == 0) return i;
  if (i == 0) return n + j;
  return 2 * n + j;
}

__global__ void k_prolong(DevLevel2D coarse, DevLevel2D fine, const double* __restrict__ c, double* f,
                          double* next, const double* __restrict__ gbnd, int mode) {
  const int total = fine.M * fine.S;
  const int Sf = fine.S, Sc = coarse.S, nf = fine.n, nc = coarse.n;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int slot = k / Sf;
    int i, j;
    decode(nf, k - slot * Sf, i, j);
    const double v = prolong_value(c + static_cast<size_t>(slot) * Sc, nc, i, j);
    if (mode == PROLONG_ADD) {
      f[k] = f[k] + v;  // u.add_scaled(ef, 1.0)
    } else {
      f[k] = v;
      if (mode == PROLONG_W_NEXT) {
        const bool dom = fine.node_flags[k] & 2;
        next[k] = dom ? gbnd[static_cast<size_t>(slot) * 3 * nf + bpos_dev(nf, i, j)] : v;
      }
    }
  }
}

// Dirichlet values: f = g (owner-evaluated, replace-synced) on domain-boundary
// copies; optionally zero everything else (u0 initialisation).
__global__ void k_set_boundary(DevLevel2D lv, double* f, const double* __restrict__ gbnd, int zero_rest) {
  const int total = lv.M * lv.S;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const std::uint8_t fl = lv.node_flags[k];
    if (fl & 2) {
      const int slot = k / lv.S;
      int i, j;
      decode(lv.n, k - slot * lv.S, i, j);
      f[k] = gbnd[static_cast<size_t>(slot) * 3 * lv.n + bpos_dev(lv.n, i, j)];
    } else if (zero_rest) {
      f[k] = 0.0;
    }
  }
}

// ---------------------------------------------------------------- rhs
__global__ void k_ftab(DevLevel2D lv, int kind, double* ftab) {
  const int n2 = 2 * lv.n;
  const int SF = (n2 + 1) * (n2 + 2) / 2;
  const int total = lv.M * SF;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int slot = k / SF;
    int I, J;
    decode(n2, k - slot * SF, I, J);
    const double* g = lv.geo + 6 * slot;
    const double hi = 0.5 * I, hj = 0.5 * J;
    const double x = g[0] + hi * g[2] + hj * g[4];
    const double y = g[1] + hi * g[3] + hj * g[5];
    double f = 0.0;
    if (kind == SRC_SIN2D) f = 2.0 * M_PI * M_PI * sin(M_PI * x) * sin(M_PI * y);
    ftab[k] = f;
  }
}

__device__ __forceinline__ double gather_rhs(const double* __restrict__ F, int n, int p, int q, double hw) {
  const int n2 = 2 * n;
  auto f = [&](int I, int J) { return F[dlat(n2, I, J)]; };
  double acc = 0.0;
  if (q >= 1 && p + q <= n) {  // up(p, q-1) as c
    const int i = p, j = q - 1;
    acc += hw * (f(2 * i, 2 * j + 1) + f(2 * i + 1, 2 * j + 1));
  }
  if (p >= 1 && q >= 1 && p + q <= n) {  // down(p-1, q-1) as c
    const int i = p - 1, j = q - 1;
    acc += hw * (f(2 * i + 2, 2 * j + 1) + f(2 * i + 1, 2 * j + 2));
  }
  if (q >= 1 && p + q <= n - 1) {  // down(p, q-1) as b
    const int i = p, j = q - 1;
    acc += hw * (f(2 * i + 1, 2 * j + 1) + f(2 * i + 1, 2 * j + 2));
  }
  if (p >= 1 && p + q <= n) {  // up(p-1, q) as b
    const int i = p - 1, j = q;
    acc += hw * (f(2 * i + 1, 2 * j) + f(2 * i + 1, 2 * j + 1));
  }
  if (p + q <= n - 1) {  // up(p, q) as a
    acc += hw * (f(2 * p + 1, 2 * q) + f(2 * p, 2 * q + 1));
  }
  if (p >= 1 && p + q <= n - 1) {  // down(p-1, q) as a
    const int i = p - 1, j = q;
    acc += hw * (f(2 * i + 1, 2 * j + 1) + f(2 * i + 2, 2 * j + 1));
  }
  return acc;
}

__global__ void k_rhs(DevLevel2D lv, const double* __restrict__ ftab, const double* __restrict__ gbnd,
                      double* b, int src_zero) {
  const int total = lv.M * lv.S;
  const int S = lv.S, n = lv.n;
  const int SF = (2 * n + 1) * (2 * n + 2) / 2;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += gridDim.x * blockDim.x) {
    const int slot = k / S;
    int i, j;
    decode(n, k - slot * S, i, j);
    const std::uint8_t fl = lv.node_flags[k];
    if (fl & 2) {
      b[k] = gbnd[static_cast<size_t>(slot) * 3 * n + bpos_dev(n, i, j)];
      continue;
    }
    if (src_zero) {
      b[k] = 0.0;
      continue;
    }
    if (!(fl & 1)) {
      b[k] = gather_rhs(ftab + static_cast<size_t>(slot) * SF, n, i, j, lv.wq[slot] * 0.5);
      continue;
    }
    const int gid = lv.node_gid[k];
    const int beg = lv.grp_ptr[gid], end = lv.grp_ptr[gid + 1];
    if (lv.mem_off[beg] != k) continue;
    double v;
    if (end - beg == 1) {
      v = gather_rhs(ftab + static_cast<size_t>(slot) * SF, n, i, j, lv.wq[slot] * 0.5);
    } else {
      v = 0.0;
      for (int m = beg; m < end; ++m) {
        const int ms = lv.mem_slot[m], ij = lv.mem_ij[m];
        v += gather_rhs(ftab + static_cast<size_t>(ms) * SF, n, ij & 0xffff, ij >> 16, lv.wq[ms] * 0.5);
      }
    }
    for (int m = beg; m < end; ++m) b[lv.mem_off[m]] = v;
  }
}

// ---------------------------------------------------------------- level-0 CG
// One CTA runs the whole unpreconditioned CG of MultigridSolver::cg_level0;
// dot_unique is a sequential sum in the reference's owner order.
__device__ double seq_dot(const DevLevel2D& lv, const double* a, const double* b, bool zero_bnd) {
  double s = 0.0;
  for (int t = 0; t < lv.dot_count; ++t) {
    const int k = lv.dot_order[t];
    double x = a[k], y = b[k];
    if (zero_bnd && (lv.node_flags[k] & 2)) x = y = 0.0;
    s += x * y;
  }
  return s;
}

// cg_level0 (proj/src/multigrid.cpp:198-229) by one CTA over the unique DoF
// of level 0, numbered in the owner order of dot_unique (every copy of a node
// holds the same value throughout the CG, so the copy-wise arithmetic of the
// reference is the DoF-wise arithmetic here, bit for bit):
//   apply   OperatorP1::apply at n = 1: member m of a node contributes
//           acc_m = 0.0 + ((k0 x_a + k1 x_b) + k2 x_c) (row `role` of its K_up,
//           the gather order of proj/src/fem.cpp:106-115); a single member is
//           the row value, several are summed 0.0 + acc_0 + acc_1 ... in slot
//           order (interface_sync Additive); domain rows zeroed;
//   dot     the products in parallel, then s = s + x y in DoF order by one
//           thread from 16-byte shared-memory loads issued ahead of the
//           dependent additions (measured: the dependent chain of additions
//           is the cost of the CG, ~ 8-9 cycles per DoF and dot).
constexpr int kCg0Threads = 128;

__device__ __forceinline__ double cg_seq_sum(const double* prod, int cnt) {
  double acc = 0.0;
  int t = 0;
  for (; t + 16 <= cnt; t += 16) {
    double v[16];
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(prod + t));
#pragma unroll
    for (int q = 0; q < 16; q += 2)
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[q]), "=d"(v[q + 1]) : "r"(a + 8u * q) : "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = acc + v[q];
  }
  for (; t < cnt; ++t) acc = acc + prod[t];
  return acc;
}

__global__ void __launch_bounds__(kCg0Threads) k_cg0(DevLevel2D lv, double* ug, const double* bg, CgParams prm,
                                                      DevStatus* status) {
  extern __shared__ __align__(16) double cg_smem[];
  const int cnt = lv.dot_count, nmem = lv.cg_nmem, tid = threadIdx.x;
  const int cnt2 = (cnt + 1) & ~1;  // 16-byte aligned arrays
  double* u = cg_smem;
  double* b = u + cnt2;
  double* r = b + cnt2;
  double* p = r + cnt2;
  double* ap = p + cnt2;
  double* prod = ap + cnt2;
  double* acc_m = prod + cnt2;                                  // nmem
  double* coef = acc_m + nmem;                                  // 3 nmem
  int* mdof = reinterpret_cast<int*>(coef + 3 * static_cast<size_t>(nmem));  // 3 nmem
  int* mptr = mdof + 3 * nmem;                                  // cnt + 1
  unsigned char* dom = reinterpret_cast<unsigned char*>(mptr + cnt + 1);
  __shared__ double sh_s;
  for (int d = tid; d < cnt; d += kCg0Threads) {
    const int k = lv.dot_order[d];
    u[d] = ug[k];
    b[d] = bg[k];
    dom[d] = lv.node_flags[k] & 2;
  }
  for (int q = tid; q < 3 * nmem; q += kCg0Threads) {
    coef[q] = lv.cg_mem_coef[q];
    mdof[q] = lv.cg_mem_dof[q];
  }
  for (int d = tid; d <= cnt; d += kCg0Threads) mptr[d] = lv.cg_mem_ptr[d];
  __syncthreads();
  // y = A x (residual: y = b - A x); domain rows zeroed
  auto apply = [&](const double* x, double* y, bool residual) {
    for (int m = tid; m < nmem; m += kCg0Threads) {
      const int q = 3 * m;
      acc_m[m] = 0.0 + ((coef[q] * x[mdof[q]] + coef[q + 1] * x[mdof[q + 1]]) + coef[q + 2] * x[mdof[q + 2]]);
    }
    __syncthreads();
    for (int d = tid; d < cnt; d += kCg0Threads) {
      const int m0 = mptr[d], m1 = mptr[d + 1];
      double v;
      if (m1 - m0 == 1) {
        v = acc_m[m0];
      } else {
        v = 0.0;
        for (int m = m0; m < m1; ++m) v += acc_m[m];
      }
      y[d] = dom[d] ? 0.0 : (residual ? b[d] - v : v);
    }
    __syncthreads();
  };
  // dot_unique in its sequential order; `zero_dom` zeroes domain rows of both operands
  auto dot = [&](const double* x, const double* y, bool zero_dom) {
    for (int d = tid; d < cnt; d += kCg0Threads) {
      double xv = x[d], yv = y[d];
      if (zero_dom && dom[d]) xv = yv = 0.0;
      prod[d] = xv * yv;
    }
    __syncthreads();
    if (tid == 0) sh_s = cg_seq_sum(prod, cnt);
    __syncthreads();
    return sh_s;
  };
  apply(u, r, true);
  for (int d = tid; d < cnt; d += kCg0Threads) p[d] = r[d];
  double rr = dot(r, r, false);
  const double bnorm = sqrt(fmax(0.0, dot(b, b, true)));
  const double tl = prm.rel_tol * bnorm;
  const double tol = (tl < prm.abs_floor) ? prm.abs_floor : tl;
  int it = 0, code = 0;
  while (sqrt(rr) > tol) {
    if (++it > prm.max_iter) {
      code = 1;
      break;
    }
    apply(p, ap, false);
    const double pap = dot(p, ap, false);
    if (pap <= 0.0) {
      code = 2;
      break;
    }
    const double alpha = rr / pap;
    // the products of (r + (-alpha) ap)^2 from the values the update stores
    for (int d = tid; d < cnt; d += kCg0Threads) {
      const double rn = r[d] + (-alpha) * ap[d];
      u[d] = u[d] + alpha * p[d];
      r[d] = rn;
      prod[d] = rn * rn;
    }
    __syncthreads();
    if (tid == 0) sh_s = cg_seq_sum(prod, cnt);
    __syncthreads();
    const double rr_new = sh_s;
    const double beta = rr_new / rr;
    for (int d = tid; d < cnt; d += kCg0Threads) p[d] = p[d] * beta + r[d];
    // (the next apply reads p after its own first barrier)
    rr = rr_new;
  }
  if (tid == 0) {
    status->iters = it;
    if (code != 0 && status->code == 0) {
      status->code = code;
      status->residual = sqrt(rr);
    }
  }
  __syncthreads();
  // every copy of each DoF
  for (int d = tid; d < cnt; d += kCg0Threads)
    for (int c = lv.cg_copy_ptr[d]; c < lv.cg_copy_ptr[d + 1]; ++c) ug[lv.cg_copy[c]] = u[d];
}

// ---------------------------------------------------------------- Gauss-Seidel
// Exact-order forward Gauss-Seidel.  Work items are (sweep, macro) in the
// reference's sequential order; macro m's sweep s starts once every
// vertex-sharing macro m' < m finished sweep s and every m'' > m finished
// sweep s-1 (bitwise identical to the sequential order).
// Inside a macro one lane owns one lattice row j and walks the hyperplane
// wavefront t = i + 2j (A.2): W comes from the lane's own previous result,
// S/SE from lane j-1 by shuffle (SMEM hand-off across warps), and the
// not-yet-updated E/N/NW/b values are prefetched kPf steps ahead from L2.
constexpr int kPf = 8;     // prefetch distance (wavefront steps)
constexpr int kRing = 16;  // cross-warp hand-off ring

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double pick(int c, double E, double W, double N, double S, double NW, double SE,
                                       const double* gh) {
  switch (c) {
    case 0: return E;
    case 1: return W;
    case 2: return N;
    case 3: return S;
    case 4: return NW;
    case 5: return SE;
    default: return gh[c - 6];
  }
}

__device__ __noinline__ double relax_interface(const DevLevel2D& lv, const BNode& bn, double B, double E,
                                               double W, double N, double S, double NW, double SE,
                                               const double* gh) {
  double off = 0.0;
  for (int r = 0; r < bn.rec_count; ++r) {
    const MemberRec rec = lv.rec[bn.rec_begin + r];
    const double* ku = lv.kstiff + 18 * rec.slot;
    const double* kd = ku + 9;
    double o = 0.0;
    // partial_row cell order, proj/src/fem.cpp:138-172
    if (rec.mask & 1) o += ku[1] * pick(rec.code[0], E, W, N, S, NW, SE, gh) + ku[2] * pick(rec.code[1], E, W, N, S, NW, SE, gh);
    if (rec.mask & 2) o += ku[3] * pick(rec.code[2], E, W, N, S, NW, SE, gh) + ku[5] * pick(rec.code[3], E, W, N, S, NW, SE, gh);
    if (rec.mask & 4) o += ku[6] * pick(rec.code[4], E, W, N, S, NW, SE, gh) + ku[7] * pick(rec.code[5], E, W, N, S, NW, SE, gh);
    if (rec.mask & 8) o += kd[1] * pick(rec.code[6], E, W, N, S, NW, SE, gh) + kd[2] * pick(rec.code[7], E, W, N, S, NW, SE, gh);
    if (rec.mask & 16) o += kd[3] * pick(rec.code[8], E, W, N, S, NW, SE, gh) + kd[5] * pick(rec.code[9], E, W, N, S, NW, SE, gh);
    if (rec.mask & 32) o += kd[6] * pick(rec.code[10], E, W, N, S, NW, SE, gh) + kd[7] * pick(rec.code[11], E, W, N, S, NW, SE, gh);
    off += o;
  }
  return (B - off) / bn.diag;
}

__global__ void __launch_bounds__(576, 1) k_gs(DevHier2D hd, DevLevel2D lv, double* u, const double* __restrict__ b,
                                             int sweeps, int* done) {
  extern __shared__ double smem[];
  const int n = lv.n, S = lv.S, M = lv.M;
  const int nwarps = blockDim.x >> 5;
  double* gh = smem;
  double* xfer = smem + lv.max_ghosts;                                 // [nwarps][kRing]
  volatile int* prog = reinterpret_cast<int*>(xfer + nwarps * kRing);  // [nwarps]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = tid;
  const bool row_ok = j <= n;
  const int len = n - j;
  const int rowj = row_ok ? dlat(n, 0, j) : 0;
  const int rowj1 = (j + 1 <= n) ? dlat(n, 0, j + 1) : 0;
  const int nitems = sweeps * M;

  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int s = item / M, m = item - s * M;
    if (tid == 0) {
      for (int q = hd.nb_lo_ptr[m]; q < hd.nb_lo_ptr[m + 1]; ++q)
        while (ld_acquire(done + hd.nb_lo[q]) < s + 1) {}
      for (int q = hd.nb_hi_ptr[m]; q < hd.nb_hi_ptr[m + 1]; ++q)
        while (ld_acquire(done + hd.nb_hi[q]) < s) {}
      __threadfence();
    }
    __syncthreads();
    const int gbeg = lv.ghost_ptr[m], gcnt = lv.ghost_ptr[m + 1] - gbeg;
    for (int g = tid; g < gcnt; g += blockDim.x) gh[g] = __ldcg(u + lv.ghost_off[gbeg + g]);
    if (tid < nwarps) prog[tid] = 0;
    __syncthreads();

    double* um = u + static_cast<size_t>(m) * S;
    const double* bm = b + static_cast<size_t>(m) * S;
    const BNode* bnm = lv.bnode + static_cast<size_t>(m) * 3 * n;
    const double* st = lv.stencil + 7 * m;
    const double s1 = st[1], s2 = st[2], s3 = st[3], s4 = st[4], s5 = st[5], s6 = st[6];
    const double inv_c = lv.inv_c[m];

    double eR[kPf], nR[kPf], bR[kPf];
    auto fetch = [&](int t, double& e, double& nn, double& bb) {
      const int i = t - 2 * j;
      e = nn = bb = 0.0;
      if (row_ok && i >= 0 && i <= len) {
        bb = __ldcg(bm + rowj + i);
        if (i + 1 <= len) e = __ldcg(um + rowj + i + 1);
        if (i <= len - 1) nn = __ldcg(um + rowj1 + i);
      }
    };
#pragma unroll
    for (int k = 0; k < kPf; ++k) fetch(k, eR[k], nR[k], bR[k]);

    double prev = 0.0, se_prev = 0.0, n_prev = 0.0;
    const int tmax = 2 * n;
    for (int t0 = 0; t0 <= tmax; t0 += kPf) {
#pragma unroll
      for (int k = 0; k < kPf; ++k) {
        const int t = t0 + k;
        if (t > tmax) break;
        const double E = eR[k], N = nR[k], B = bR[k];
        fetch(t + kPf, eR[k], nR[k], bR[k]);
        double se = __shfl_up_sync(0xffffffffu, prev, 1);
        if (warp > 0) {
          // lane 0 takes row 32w-1's result of step t-1 from the previous warp
          while (prog[warp - 1] < t) {}
          __threadfence_block();
          const double hand = xfer[(warp - 1) * kRing + ((t - 1) & (kRing - 1))];
          if (lane == 0) se = hand;
        }
        const double Sv = se_prev, W = prev, NW = n_prev;
        const int i = t - 2 * j;
        double res = 0.0;
        if (row_ok && i >= 0 && i <= len) {
          if (j >= 1 && i >= 1 && i <= len - 1) {
            double acc = s1 * E + s2 * W;
            acc = acc + s3 * N;
            acc = acc + s4 * Sv;
            acc = acc + s5 * NW;
            acc = acc + s6 * se;
            res = (B - acc) * inv_c;
          } else {
            const BNode bn = bnm[bpos_dev(n, i, j)];
            res = bn.domain ? B : relax_interface(lv, bn, B, E, W, N, Sv, NW, se, gh);
            for (int q = 0; q < bn.wr_count; ++q) u[lv.wr[bn.wr_begin + q]] = res;
          }
          um[rowj + i] = res;
        }
        prev = res;
        se_prev = se;
        n_prev = N;
        if (warp + 1 < nwarps) {
          // ring overrun guard: the next warp must have consumed step t-kRing+1
          while (prog[warp + 1] < t - kRing + 2) {}
          if (lane == 31) xfer[warp * kRing + (t & (kRing - 1))] = res;
          __syncwarp();
          __threadfence_block();
          if (lane == 0) prog[warp] = t + 1;
        } else if (lane == 0) {
          prog[warp] = t + 1;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(done + m, s + 1);
    }
  }
}


// ------------------------------------------------ Gauss-Seidel, shared-memory
// One group of warps relaxes one macro lattice held in shared memory, along
// the hyperplane wavefront t = i + 2j (every stencil neighbour
// of a step-t node belongs to step t +- 1 or t +- 2, so a named barrier per
// step is the only synchronisation).  Warp roles:
//   warp 0  boundary warp: the (at most three) lattice-boundary nodes of step t,
//           lane 8 type + q evaluating the partial row of group member q;
//   warp 1  program warp: streams the precompiled step programs
//           (Level2D::prog) into a shared-memory ring with cp.async, kRingSteps
//           steps ahead, so the boundary warp never waits on L2;
//   warp 2+ interior warps, one lattice row per lane (7-point form of
//           proj/src/multigrid.cpp:170-175).
constexpr int kRingSteps = 8;
// in shared memory the six 128-byte lane records of a step are padded to 144
// bytes so that the six boundary lanes' vector loads hit distinct banks
constexpr int kLaneStride = 144;
constexpr int kStepBytes = 6 * kLaneStride;  // 864 per ring slot
static_assert(kProgLaneWords * 8 == 128, "lane records are eight 16-byte chunks");

__device__ __forceinline__ void bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double ld_s64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_s64(unsigned a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_s64u(unsigned a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}

// One pre-decoded lane record of a step program (Level2D::prog, 128 bytes).
struct PNode {
  double c[6], diag, inv, B;
  int loc[6], k, flags, wr0, wr1, wb, wc, xb, nc;
  unsigned slot01, slot23, slot45;  // [ghosts | lattice] slots of the six reads, 16 bits each
};

__device__ __forceinline__ void ld_s_v2f64(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void ld_s_v4s32(unsigned a, int& x, int& y, int& z, int& w) {
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a) : "memory");
}

__device__ __forceinline__ void load_lane(PNode& p, unsigned a) {
  ld_s_v2f64(a, p.c[0], p.c[1]);
  ld_s_v2f64(a + 16, p.c[2], p.c[3]);
  ld_s_v2f64(a + 32, p.c[4], p.c[5]);
  ld_s_v2f64(a + 48, p.diag, p.inv);
  ld_s_v4s32(a + 64, p.loc[0], p.loc[1], p.loc[2], p.loc[3]);
  ld_s_v4s32(a + 80, p.loc[4], p.loc[5], p.k, p.flags);
  ld_s_v4s32(a + 96, p.wr0, p.wr1, p.wb, p.wc);
  int s45, s01, s23;
  ld_s_v4s32(a + 112, p.xb, s45, s01, s23);
  p.slot01 = static_cast<unsigned>(s01);
  p.slot23 = static_cast<unsigned>(s23);
  p.slot45 = static_cast<unsigned>(s45);
  p.nc = 0;
}

// lane (type, mem): member `mem` of the step's node of this type.  Members 0/1
// come from the ring slot; members >= 2 (vertex groups, flag bit 16 set on
// every record of such a step) from the staged extra records.
__device__ __forceinline__ void load_pnode(PNode& p, unsigned slot, unsigned xs, unsigned bs_s, int type, int mem) {
  load_lane(p, slot + static_cast<unsigned>(kLaneStride) * static_cast<unsigned>(2 * type + (mem < 2 ? mem : 0)));
  p.B = ld_s64(bs_s + 8u * (p.k >= 0 ? p.k : 0));  // b is constant during the sweep
  if (p.flags & (1 << 16)) {
    const int rc = p.k >= 0 ? ((p.flags >> 8) & 0xff) : 0;
    if (mem >= 2 && mem < rc) load_lane(p, xs + 128u * static_cast<unsigned>(p.xb + mem - 2));
  }
  if (mem >= 2 && !(p.flags & (1 << 16))) p.nc = 0;
}

// Relax the boundary nodes of one step (relax_boundary_node,
// proj/src/multigrid.cpp:132-150): member off-diagonal sums o (cells in the
// order of proj/src/fem.cpp:138-172), summed over members in slot order,
// (b - off) / diag correctly rounded, written to every copy.
__device__ __forceinline__ void relax_nodes(const PNode& p, unsigned us_s, unsigned bs_s, unsigned gh_s,
                                            double* copies, const int* wr_global, int lane,
                                            double* own_copy = nullptr) {
  const int type = lane >> 3, mem = lane & 7;
  const bool lane_ok = type < 3;
  const int rc = (lane_ok && p.k >= 0) ? ((p.flags >> 8) & 0xff) : 0;
  // reads: lattice values of this macro, or ghost values (constant during the sweep)
  double x[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int l = p.loc[q];
    x[q] = ld_s64(l >= 0 ? us_s + 8u * l : gh_s + 8u * (-1 - l));
  }
  const double B = p.B;
  // absent cells carry zero coefficients and read the zero slot: o + 0 == o
  // bitwise, since o = 0.0 + ... is never -0.0 (no selects on the chain)
  double o = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) o = o + (p.c[2 * c] * x[2 * c] + p.c[2 * c + 1] * x[2 * c + 1]);
  o = mem < rc ? o : 0.0;
  double off = 0.0;
  if (p.flags & (1 << 16)) {
    // a vertex group with more than two members: sequential sum over members
    // (members >= rc contribute +0.0)
#pragma unroll
    for (int r = 0; r < 8; ++r) off = off + __shfl_sync(0xffffffffu, o, (lane & ~7) + r);
  } else {
    const double o1 = __shfl_down_sync(0xffffffffu, o, 1);
    off = (off + o) + o1;  // rc < 2: o1 = +0.0
  }
  if (lane_ok && mem == 0 && p.k >= 0) {
    double res = B;
    if (!(p.flags & 1)) {
      // (B - off) / diag correctly rounded: q = x y, r = x - q d exactly (FMA),
      // RN(q + r y) = RN(x / d) for y = RN(1 / d) (Markstein); a zero
      // numerator keeps its sign through x * y.
      const double xn = B - off;
      const double q = xn * p.inv;
      const double r = __fma_rn(-q, p.diag, xn);
      res = xn == 0.0 ? q : __fma_rn(r, p.inv, q);
    }
    st_s64(us_s + 8u * p.k, res);
    if (own_copy) own_copy[p.k] = res;  // pipelined smoother: global copies are the record
    if (copies) {
      if (p.wc > 0) copies[p.wr0] = res;
      if (p.wc > 1) copies[p.wr1] = res;
      for (int q = p.wb + 2; q < p.wb + p.wc; ++q) copies[wr_global[q]] = res;
    }
  }
}

// Lane record of the pipelined smoother (k_gs_pipe), loaded in two parts so
// that neither sits between the gate and the relaxation: pnode_issue (the
// record's vector loads, issued right after the current step's six lattice
// reads) and pnode_finish (the dependent part: b, the extra record of a
// vertex-group member, the six read addresses), done after the current
// step's stores.
struct PipeNode {
  double c[6], diag, inv, B;
  int k, flags, wr0, wr1, wb, wc, xb;
  unsigned s01, s23, s45;  // [ghosts | lattice] slots of the six reads, 16 bits each
  unsigned a[6];           // their shared-memory addresses
};

__device__ __forceinline__ void ld_s_v2s32(unsigned a, int& x, int& y) {
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(x), "=r"(y) : "r"(a) : "memory");
}

__device__ __forceinline__ void pnode_issue(PipeNode& p, unsigned rec) {
  ld_s_v2f64(rec, p.c[0], p.c[1]);
  ld_s_v2f64(rec + 16, p.c[2], p.c[3]);
  ld_s_v2f64(rec + 32, p.c[4], p.c[5]);
  ld_s_v2f64(rec + 48, p.diag, p.inv);
  ld_s_v2s32(rec + 88, p.k, p.flags);
  ld_s_v4s32(rec + 96, p.wr0, p.wr1, p.wb, p.wc);
  int s45, s01, s23;
  ld_s_v4s32(rec + 112, p.xb, s45, s01, s23);
  p.s01 = static_cast<unsigned>(s01);
  p.s23 = static_cast<unsigned>(s23);
  p.s45 = static_cast<unsigned>(s45);
}
// lane (type, mem): member `mem` of the step's node of this type; members 0/1
// come from the ring slot, members >= 2 of vertex groups (flag bit 16 set on
// every record of such a step) from the staged extra records
__device__ __forceinline__ unsigned pnode_rec(unsigned slot, int type, int mem) {
  return slot + static_cast<unsigned>(kLaneStride) * static_cast<unsigned>(2 * type + (mem < 2 ? mem : 0));
}
__device__ __forceinline__ void pnode_finish(PipeNode& p, unsigned xs, unsigned bs_s, unsigned gx_s, int mem) {
  if (p.flags & (1 << 16)) {
    const int rc = p.k >= 0 ? ((p.flags >> 8) & 0xff) : 0;
    if (mem >= 2 && mem < rc) pnode_issue(p, xs + 128u * static_cast<unsigned>(p.xb + mem - 2));
  }
  p.B = ld_s64(bs_s + 8u * (p.k >= 0 ? p.k : 0));  // b is constant during the sweep
  p.a[0] = gx_s + 8u * (p.s01 & 0xffffu), p.a[1] = gx_s + 8u * (p.s01 >> 16);
  p.a[2] = gx_s + 8u * (p.s23 & 0xffffu), p.a[3] = gx_s + 8u * (p.s23 >> 16);
  p.a[4] = gx_s + 8u * (p.s45 & 0xffffu), p.a[5] = gx_s + 8u * (p.s45 >> 16);
}

// relax_nodes for k_gs_pipe, with the shortest dependent path after the gate:
// the six read addresses are precomputed (slots of the [ghosts | lattice]
// region), no selects, absent members / cells are zero coefficients on the
// zero slot (o = +0.0), the two-member sum is one shuffle.  The own copy and
// up to two other copies are stored to global memory; vertex groups (> 2
// members, `big` steps) take the general sum and the remaining copies.
// `mid` runs after the six reads are issued (the next record's loads), `tail`
// after the stores (its dependent part).
template <class Mid, class Tail>
__device__ __forceinline__ void relax_pipe(const PipeNode& p, unsigned us_s, double* u, const int* wr_global, int lane,
                                           double* own_copy, int g_chk_slots, int g_chk_S, int g_chk_MS,
                                           unsigned gx_s, Mid&& mid, Tail&& tail) {
  (void)g_chk_slots, (void)g_chk_S, (void)g_chk_MS, (void)gx_s;  // bounds of the KB_GS_CHECK build
  const int type = lane >> 3, mem = lane & 7;
#ifdef KB_GS_CHECK
  {
    const unsigned lim = gx_s + 8u * static_cast<unsigned>(g_chk_slots);
    KB_ASSERT(p.a[0] < lim && p.a[1] < lim && p.a[2] < lim && p.a[3] < lim && p.a[4] < lim && p.a[5] < lim);
    KB_ASSERT(p.k < g_chk_S);
  }
#endif
  const double x0 = ld_s64(p.a[0]), x1 = ld_s64(p.a[1]), x2 = ld_s64(p.a[2]);
  const double x3 = ld_s64(p.a[3]), x4 = ld_s64(p.a[4]), x5 = ld_s64(p.a[5]);
  mid();
  double o = 0.0;
  o = o + (p.c[0] * x0 + p.c[1] * x1);
  o = o + (p.c[2] * x2 + p.c[3] * x3);
  o = o + (p.c[4] * x4 + p.c[5] * x5);
  double off = 0.0;
  const bool big = (p.flags >> 16) & 1;  // the same on every lane of the step
  if (!big) {
    const double o1 = __shfl_down_sync(0xffffffffu, o, 1);
    off = (off + o) + o1;  // a single member: o1 = +0.0
  } else {
    const int rc = (type < 3 && p.k >= 0) ? ((p.flags >> 8) & 0xff) : 0;
    o = mem < rc ? o : 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) off = off + __shfl_sync(0xffffffffu, o, (lane & ~7) + r);
  }
  if (type < 3 && mem == 0 && p.k >= 0) {
    // (B - off) / diag correctly rounded (Markstein; a zero numerator keeps its sign)
    const double xn = p.B - off;
    const double q = xn * p.inv;
    const double r = __fma_rn(-q, p.diag, xn);
    const double quot = xn == 0.0 ? q : __fma_rn(r, p.inv, q);
    const double res = (p.flags & 1) ? p.B : quot;
    KB_ASSERT(p.wc <= 0 || (p.wr0 >= 0 && p.wr0 < g_chk_MS));
    KB_ASSERT(p.wc <= 1 || (p.wr1 >= 0 && p.wr1 < g_chk_MS));
    st_s64(us_s + 8u * static_cast<unsigned>(p.k), res);
    own_copy[p.k] = res;
    if (p.wc > 0) u[p.wr0] = res;
    if (p.wc > 1) u[p.wr1] = res;
    // more than two other copies: vertex groups (also domain-boundary ones, rc = 0)
    for (int q2 = p.wb + 2; q2 < p.wb + p.wc; ++q2) u[wr_global[q2]] = res;
  }
  tail();
}

// Issue the cp.async copies of step program `t` (if it exists) into its ring slot.
__device__ __forceinline__ void issue_step(const unsigned long long* prog_m, unsigned ring_s, int n, int t, int lane) {
  if (t <= 2 * n) {
    const char* src = reinterpret_cast<const char*>(prog_m + static_cast<size_t>(t) * kProgStepWords);
    const unsigned dst = ring_s + static_cast<unsigned>(t % kRingSteps) * kStepBytes;
    for (int c = lane; c < 48; c += 32)  // 6 records x 8 chunks
      cp_async16(dst + static_cast<unsigned>(kLaneStride) * (c >> 3) + 16u * (c & 7), src + 16 * c);
  }
}
// ... and commit it as one group (group counting stays uniform)
__device__ __forceinline__ void stream_step(const unsigned long long* prog_m, unsigned ring_s, int n, int t, int lane) {
  issue_step(prog_m, ring_s, n, t, lane);
  cp_async_commit();
}

// Static inputs of the group's next macro (level mode): its first step
// programs, ghost offsets and extra records, streamed while this one sweeps.
struct NextPrefetch {
  const unsigned long long* prog_m;  // null: no next macro
  unsigned ring_s;
  const int* go_src;
  int* go_dst;
  int go_count;
  const unsigned long long* xs_src;
  unsigned long long* xs_dst;
  int xs_words;
};

__device__ __forceinline__ void issue_next(const NextPrefetch& nx, int n, int t, int lane) {
  if (!nx.prog_m || t >= kRingSteps - 1) return;
  if (t == 0) {
    for (int x = lane; x < nx.go_count; x += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(nx.go_dst + x)), "l"(nx.go_src + x)
                   : "memory");
    for (int x = lane; x < nx.xs_words; x += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(nx.xs_dst + x)), "l"(nx.xs_src + x)
                   : "memory");
  }
  issue_step(nx.prog_m, nx.ring_s, n, t, lane);
}

// Per-macro inputs of one sweep.  `head_ready`: the first kRingSteps - 1 step
// programs are already in the ring (streamed ahead during the previous sweep).
struct SweepArgs {
  int m;
  const unsigned long long* prog_m;  // this macro's step programs (global)
  const double* st;                  // 7-point stencil (C, E, W, N, S, NW, SE)
  double inv_c;
  bool head_ready;
  NextPrefetch next;
};

__device__ __forceinline__ void group_sweep(const DevLevel2D& lv, const SweepArgs& a, double* us, const double* bs,
                                            const double* gh, const unsigned long long* xs, unsigned char* ring,
                                            double* copies, int gw, int lane, int bar_id, int bar_threads) {
  const int n = lv.n;
  const unsigned ring_s = smem_addr(ring);

  if (gw == 1) {
    const unsigned long long* prog_m = a.prog_m;
    // lookahead kRingSteps - 1: during step t the slot of step t - 1 is refilled
    // (the boundary warp read it before the barrier that ended step t - 1)
    if (!a.head_ready) {
#pragma unroll 1
      for (int t = 0; t < kRingSteps - 1; ++t) stream_step(prog_m, ring_s, n, t, lane);
    }
    cp_async_wait<kRingSteps - 3>();  // steps 0 and 1 landed
    bar_sync(bar_id, bar_threads);
    for (int t = 0; t <= 2 * n; ++t) {
      issue_step(prog_m, ring_s, n, t + kRingSteps - 1, lane);
      issue_next(a.next, n, t, lane);  // same commit group: counting unchanged
      cp_async_commit();
      cp_async_wait<kRingSteps - 3>();  // step t + 2 landed
      bar_sync(bar_id, bar_threads);
    }
    for (int t = 2 * n + 1; t < kRingSteps - 1; ++t) issue_next(a.next, n, t, lane);  // short sweeps
    cp_async_commit();
    cp_async_wait<0>();
  } else if (gw == 0) {
    const unsigned us_s = smem_addr(us), bs_s = smem_addr(bs), gh_s = smem_addr(gh), xs_s = smem_addr(xs);
    const int type = lane >> 3, mem = lane & 7;
    const int tl = type < 3 ? type : 0;
    bar_sync(bar_id, bar_threads);
    // two register sets, ping-pong (no copies); the slot after the last step
    // holds stale shared memory and is never decoded
    PNode p0, p1;
    load_pnode(p0, ring_s, xs_s, bs_s, tl, mem);
#ifdef KB_GS_TRACE
    const bool trc = blockIdx.x == 0 && lane == 0 && bar_id == 1;
#define KB_STAMP(row, t, dep) \
  if (trc) g_gs_trace[row][t] = clock64() + ((dep) == 12345.0 ? 1 : 0)
#else
#define KB_STAMP(row, t, dep)
#endif
    for (int t = 0; t <= 2 * n; t += 2) {
      KB_STAMP(0, t, 0.0);
      if (t + 1 <= 2 * n)
        load_pnode(p1, ring_s + static_cast<unsigned>((t + 1) % kRingSteps) * kStepBytes, xs_s, bs_s, tl, mem);
      KB_STAMP(1, t, p0.c[0]);
      relax_nodes(p0, us_s, bs_s, gh_s, copies, lv.wr, lane);
      KB_STAMP(2, t, ld_s64(us_s));
      bar_sync(bar_id, bar_threads);
      if (t + 1 > 2 * n) break;
      KB_STAMP(0, t + 1, 0.0);
      if (t + 2 <= 2 * n)
        load_pnode(p0, ring_s + static_cast<unsigned>((t + 2) % kRingSteps) * kStepBytes, xs_s, bs_s, tl, mem);
      KB_STAMP(1, t + 1, p1.c[0]);
      relax_nodes(p1, us_s, bs_s, gh_s, copies, lv.wr, lane);
      KB_STAMP(2, t + 1, ld_s64(us_s));
      bar_sync(bar_id, bar_threads);
    }
  } else {
    const double* st = a.st;
    const double s1 = st[1], s2 = st[2], s3 = st[3], s4 = st[4], s5 = st[5], s6 = st[6];
    const double inv_c = a.inv_c;
    const int j = 32 * (gw - 2) + lane + 1;
    const bool row = j <= n - 1;
    const int rowk = row ? dlat(n, 0, j) : 0;
    const int dn = n + 1 - j, dnw = n - j, ds = n + 2 - j;
    bar_sync(bar_id, bar_threads);
    for (int t = 0; t <= 2 * n; ++t) {
      const int i = t - 2 * j;
      if (row && i >= 1 && i <= n - j - 1) {
        const int k = rowk + i;
        const double B = bs[k];
        const double E = us[k + 1], W = us[k - 1], N = us[k + dn], S = us[k - ds];
        const double NW = us[k + dnw], SE = us[k - dn];
        double acc = s1 * E + s2 * W;
        acc = acc + s3 * N;
        acc = acc + s4 * S;
        acc = acc + s5 * NW;
        acc = acc + s6 * SE;
        us[k] = (B - acc) * inv_c;
      }
#ifdef KB_GS_TRACE
      if (blockIdx.x == 0 && gw == 2 && lane == 0 && bar_id == 1) g_gs_trace[3][t] = clock64();
#endif
      bar_sync(bar_id, bar_threads);
    }
  }
}

// warps per macro group: boundary warp, program warp, one interior warp per 32 rows
__host__ __device__ __forceinline__ int gs_group_warps(int n) { return 2 + (n - 1 + 31) / 32; }
constexpr int kMaxLevelGroups = 8;
constexpr int kRingBytes = kRingSteps * kStepBytes;

// per-group shared scratch: ring | extra records | ghosts (8-byte words)
__host__ __device__ __forceinline__ size_t gs_group_words(const DevLevel2D& lv) {
  const size_t w = kRingBytes / 8 + static_cast<size_t>(lv.max_extra) * kProgLaneWords + lv.max_ghosts + 1;
  return (w + 1) & ~static_cast<size_t>(1);  // keeps every group's ring 16-byte aligned
}

// Mode "level": the whole level (u and b of every macro) in one CTA's shared
// memory.  Groups of W warps take the macros of one DAG level at a time
// and a __syncthreads separates DAG levels.  The small
// per-level tables are staged once; while a group sweeps one macro, its
// program warp already streams the next macro's static inputs (ghost offsets,
// extra records, first step programs) into the group's second buffer set.
struct LevelTables {  // shared-memory copies of the per-macro tables
  int *dag_ptr, *dag_list, *ghost_ptr, *xtra_ptr, *prog_off;
  double *stencil, *inv_c;
};

__host__ __device__ __forceinline__ size_t gs_level_table_bytes(int M, int D) {
  // ints: dag_ptr D+1, dag_list M, ghost_ptr M+1, xtra_ptr M+1, prog_off M (padded to 8 bytes) + doubles 8 M
  const size_t ints = (D + 1) + M + (M + 1) + (M + 1) + M;
  return ((ints * 4 + 7) & ~static_cast<size_t>(7)) + static_cast<size_t>(8) * M * 8;
}
// per-group buffers: 2 rings | 2 extra-record sets | 2 ghost-offset lists | ghost values
__host__ __device__ __forceinline__ size_t gs_level_group_bytes(const DevLevel2D& lv) {
  const size_t ring = kRingBytes;
  const size_t xs = static_cast<size_t>(lv.max_extra) * kProgLaneWords * 8;
  const size_t go = ((static_cast<size_t>(lv.max_ghosts) * 4 + 15) & ~static_cast<size_t>(15));
  const size_t gv = static_cast<size_t>(lv.max_ghosts + 1) * 8;
  return (2 * (ring + xs + go) + gv + 15) & ~static_cast<size_t>(15);
}

__global__ void __launch_bounds__(512, 1) k_gs_level(DevHier2D hd, DevLevel2D lv, double* u,
                                                      const double* __restrict__ b, int sweeps) {
  extern __shared__ __align__(16) double smem[];
  const int S = lv.S, M = lv.M, n = lv.n, D = hd.dag_depth;
  const int W = gs_group_warps(n);
  const int G = blockDim.x / (32 * W);
  const size_t total = static_cast<size_t>(M) * S;
  double* lu = smem;
  double* lb = lu + total;
  unsigned char* tb = reinterpret_cast<unsigned char*>(lb + total);  // 16-byte aligned (2 total doubles)
  LevelTables T;
  {
    int* ip = reinterpret_cast<int*>(tb);
    T.dag_ptr = ip;
    T.dag_list = T.dag_ptr + (D + 1);
    T.ghost_ptr = T.dag_list + M;
    T.xtra_ptr = T.ghost_ptr + (M + 1);
    T.prog_off = T.xtra_ptr + (M + 1);
    const size_t ints = (D + 1) + M + (M + 1) + (M + 1) + M;
    T.stencil = reinterpret_cast<double*>(tb + ((ints * 4 + 7) & ~static_cast<size_t>(7)));
    T.inv_c = T.stencil + 7 * M;
  }
  unsigned char* gbase = tb + ((gs_level_table_bytes(M, D) + 15) & ~static_cast<size_t>(15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp / W, gw = warp - g * W, gt = gw * 32 + lane;
  const size_t gbytes = gs_level_group_bytes(lv);
  const size_t xs_bytes = static_cast<size_t>(lv.max_extra) * kProgLaneWords * 8;
  const size_t go_bytes = ((static_cast<size_t>(lv.max_ghosts) * 4 + 15) & ~static_cast<size_t>(15));
  unsigned char* gb = gbase + static_cast<size_t>(g) * gbytes;
  // buffer set `c` (0/1): ring, extra records, ghost offsets
  auto ringb = [&](int c) { return gb + c * kRingBytes; };
  auto xsb = [&](int c) { return reinterpret_cast<unsigned long long*>(gb + 2 * kRingBytes + c * xs_bytes); };
  auto gob = [&](int c) { return reinterpret_cast<int*>(gb + 2 * kRingBytes + 2 * xs_bytes + c * go_bytes); };
  double* gh = reinterpret_cast<double*>(gb + 2 * kRingBytes + 2 * xs_bytes + 2 * go_bytes);
  if (gw == 0 && lane == 0) gh[lv.max_ghosts] = 0.0;  // zero slot of absent partial-row terms

  for (size_t k = threadIdx.x; k < total; k += blockDim.x) {
    lu[k] = __ldcg(u + k);
    lb[k] = __ldg(b + k);
  }
  for (int k = threadIdx.x; k <= D; k += blockDim.x) T.dag_ptr[k] = hd.dag_ptr[k];
  for (int k = threadIdx.x; k < M; k += blockDim.x) {
    T.dag_list[k] = hd.dag_list[k];
    T.prog_off[k] = static_cast<int>(lv.prog_ptr[k]);
    T.inv_c[k] = lv.inv_c[k];
  }
  for (int k = threadIdx.x; k <= M; k += blockDim.x) {
    T.ghost_ptr[k] = lv.ghost_ptr[k];
    T.xtra_ptr[k] = lv.xtra_ptr[k];
  }
  for (int k = threadIdx.x; k < 7 * M; k += blockDim.x) T.stencil[k] = lv.stencil[k];
  __syncthreads();

  const int gthreads = 32 * W;
  // the group's macros in schedule order: (s, d, q = dag_ptr[d] + g + G i)
  auto next_item = [&](int& s, int& d, int& q) -> bool {
    q += G;
    while (q >= T.dag_ptr[d + 1]) {
      if (++d == D) {
        d = 0;
        if (++s == sweeps) return false;
      }
      q = T.dag_ptr[d] + g;
    }
    return true;
  };
  auto next_args = [&](int m, int buf) {
    NextPrefetch nx;
    nx.prog_m = lv.prog + T.prog_off[m];
    nx.ring_s = smem_addr(ringb(buf));
    nx.go_src = lv.ghost_off + T.ghost_ptr[m];
    nx.go_dst = gob(buf);
    nx.go_count = T.ghost_ptr[m + 1] - T.ghost_ptr[m];
    nx.xs_src = lv.prog_extra + T.xtra_ptr[m];
    nx.xs_dst = xsb(buf);
    nx.xs_words = T.xtra_ptr[m + 1] - T.xtra_ptr[m];
    return nx;
  };
  if (g < G && gw == 1) {
    int s0 = 0, d0 = 0, q0 = g - G;
    if (next_item(s0, d0, q0)) {
      const NextPrefetch nx = next_args(T.dag_list[q0], 0);
      for (int t = 0; t < kRingSteps - 1; ++t) issue_next(nx, n, t, lane);
      cp_async_commit();
    }
  }
  int cur = 0;
  for (int s = 0; s < sweeps; ++s) {
    for (int d = 0; d < D; ++d) {
      if (g < G) {
        for (int q = T.dag_ptr[d] + g; q < T.dag_ptr[d + 1]; q += G) {
          const int m = T.dag_list[q];
          if (gw == 1) cp_async_wait<0>();  // this macro's inputs landed
          bar_sync(1 + g, gthreads);
          const int gc = T.ghost_ptr[m + 1] - T.ghost_ptr[m];
          for (int x = gt; x < gc; x += gthreads) gh[x] = lu[gob(cur)[x]];
          bar_sync(1 + g, gthreads);
          SweepArgs args{m, lv.prog + T.prog_off[m], T.stencil + 7 * m, T.inv_c[m], true, NextPrefetch{}};
          int ns = s, nd = d, nq = q;
          if (next_item(ns, nd, nq)) args.next = next_args(T.dag_list[nq], cur ^ 1);
          group_sweep(lv, args, lu + static_cast<size_t>(m) * S, lb + static_cast<size_t>(m) * S, gh, xsb(cur),
                      ringb(cur), lu, gw, lane, 1 + g, gthreads);
          bar_sync(1 + g, gthreads);
          cur ^= 1;
        }
      }
      __syncthreads();
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  for (size_t k = threadIdx.x; k < total; k += blockDim.x) u[k] = lu[k];
}

// Mode "macro": one CTA (a group of W warps) per macro sweep with the macro's
// u, b, ghosts and step-program ring in shared memory; macro m's sweep s
// starts once every vertex-sharing macro m' < m finished sweep s and every
// m'' > m finished sweep s-1.
__global__ void __launch_bounds__(192, 1) k_gs_macro(DevHier2D hd, DevLevel2D lv, double* u,
                                                     const double* __restrict__ b, int sweeps, int* done) {
  extern __shared__ __align__(16) double smem[];
  const int S = lv.S, M = lv.M, n = lv.n;
  unsigned char* ring = reinterpret_cast<unsigned char*>(smem);
  unsigned long long* xs = reinterpret_cast<unsigned long long*>(ring + kRingBytes);
  double* gh = reinterpret_cast<double*>(xs + static_cast<size_t>(lv.max_extra) * kProgLaneWords);
  double* us = gh + lv.max_ghosts + 1;
  double* bs = us + S;
  const int tid = threadIdx.x, gw = tid >> 5, lane = tid & 31;
  const int nitems = sweeps * M;
  int cur = -1;
  if (tid == 0) gh[lv.max_ghosts] = 0.0;  // zero slot of absent partial-row terms
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int s = item / M, m = item - s * M;
    if (tid == 0) {
      for (int q = hd.nb_lo_ptr[m]; q < hd.nb_lo_ptr[m + 1]; ++q)
        while (ld_acquire(done + hd.nb_lo[q]) < s + 1) {}
      for (int q = hd.nb_hi_ptr[m]; q < hd.nb_hi_ptr[m + 1]; ++q)
        while (ld_acquire(done + hd.nb_hi[q]) < s) {}
    }
    __syncthreads();
    double* um = u + static_cast<size_t>(m) * S;
    if (m != cur) {
      const double* bm = b + static_cast<size_t>(m) * S;
#pragma unroll 4
      for (int k = tid; k < S; k += blockDim.x) {
        us[k] = __ldcg(um + k);
        bs[k] = __ldg(bm + k);
      }
      const int xb = lv.xtra_ptr[m], xc = lv.xtra_ptr[m + 1] - xb;
      for (int x = tid; x < xc; x += blockDim.x) xs[x] = lv.prog_extra[xb + x];
    } else {
      // only the interface copies of this macro can have changed since its last sweep
      for (int p = tid; p < 3 * n; p += blockDim.x) {
        const int k = p <= n ? p : (p <= 2 * n ? dlat(n, 0, p - n) : dlat(n, 3 * n - p, p - 2 * n));
        us[k] = __ldcg(um + k);
      }
    }
    const int gbeg = lv.ghost_ptr[m], gcnt = lv.ghost_ptr[m + 1] - gbeg;
    for (int x = tid; x < gcnt; x += blockDim.x) gh[x] = __ldcg(u + lv.ghost_off[gbeg + x]);
    __syncthreads();
    const SweepArgs args{m, lv.prog + lv.prog_ptr[m], lv.stencil + 7 * m, lv.inv_c[m], false, NextPrefetch{}};
    group_sweep(lv, args, us, bs, gh, xs, ring, u, gw, lane, 1, blockDim.x);
#pragma unroll 4
    for (int k = tid; k < S; k += blockDim.x) um[k] = us[k];
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(done + m, s + 1);
    }
    cur = m;
  }
}

// ------------------------------------------------ Gauss-Seidel, static schedule
// Small levels (GsSched2D, gs_sched2d.cpp): the unique node values u, b, the
// per-macro stencils / element matrices and the per-group diagonals live in
// shared memory; the dependence-levels of the reference's sequential
// relaxation order are executed in order, one relaxation per thread, one
// __syncthreads per level.  The level blocks stream from L2 into a ring of
// shared-memory slots by TMA bulk copies (thread 0 issues block g + K once
// every thread is past level g), completion tracked by one mbarrier per slot.
constexpr int kSchedMaxThreads = 1024;

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_block(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ int4 ld_s_int4(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

__device__ long long g_sched_trace[8][512];

// One relaxation per SG-lane subgroup: lane q evaluates member q's partial
// row (group relaxations), lane 0 sums the members in slot order and writes
// the value.  The producer (last thread) issues the TMA copy of block g + K
// after the barrier that ends level g.
template <int SG>
__global__ void __launch_bounds__(kSchedMaxThreads, 1) k_gs_sched(DevLevel2D lv, double* u,
                                                                 const double* __restrict__ b, int si, int reps, int K,
                                                                 int slot_bytes, int trace) {
  extern __shared__ __align__(16) double smem[];
  const int nu = lv.sc_nu, M = lv.M, NG = lv.num_groups, levels = lv.sc_levels[si];
  double* su = smem;  // nu unique values + the zero slot
  double* sb = su + nu + 1;
  double* mt = sb + nu + 1;
  double* gt = mt + 26 * static_cast<size_t>(M);
  int* loff = reinterpret_cast<int*>(gt + 2 * static_cast<size_t>(NG));
  unsigned long long* mbar =
      reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(loff + levels + 1) + 15) & ~uintptr_t(15));
  unsigned char* ring = reinterpret_cast<unsigned char*>(mbar + 2 * ((K + 1) / 2));
  const unsigned ring_s = smem_addr(ring), mbar_s = smem_addr(mbar);
  const unsigned su_s = smem_addr(su), sb_s = smem_addr(sb), mt_s = smem_addr(mt);
  const int* blocks = lv.sc_blocks[si];
  const int tid = threadIdx.x, nthreads = blockDim.x, producer = nthreads - 1;
  const int total = reps * levels;
  const int q = tid & (SG - 1), sg = tid / SG, R = nthreads / SG;
  const unsigned submask = SG == 32 ? 0xffffffffu : (((1u << SG) - 1u) << ((tid & 31) & ~(SG - 1)));

  for (int k = tid; k <= levels; k += nthreads) loff[k] = lv.sc_lev_off[si][k];
  if (tid == producer) {
    for (int k = 0; k < K; ++k) mbar_init(mbar_s + 8u * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == producer)
    for (int g = 0; g < K && g < total; ++g) {
      const int lvl = g % levels;
      tma_load_block(ring_s + static_cast<unsigned>(g) * slot_bytes, blocks + loff[lvl],
                     4u * static_cast<unsigned>(loff[lvl + 1] - loff[lvl]), mbar_s + 8u * g);
    }
  for (int c = tid; c < nu; c += nthreads) {
    const int o = lv.sc_cell_copy[c];
    su[c] = __ldcg(u + o);
    sb[c] = __ldg(b + o);
  }
  if (tid == 0) su[nu] = 0.0;
  for (int k = tid; k < 26 * M; k += nthreads) mt[k] = lv.sc_mtab[k];
  for (int k = tid; k < 2 * NG; k += nthreads) gt[k] = lv.sc_gtab[k];
  __syncthreads();

  const int kshift = __ffs(K) - 1;
  const int tmax = (slot_bytes - 64) / 32;  // header loads stay inside the slot
  for (int g = 0; g < total; ++g) {
    const int slot = g & (K - 1);  // K is a power of two
    if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[0][g] = clock64();
    mbar_wait(mbar_s + 8u * slot, static_cast<unsigned>((g >> kshift) & 1));
    if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[1][g] = clock64();
    const unsigned blk = ring_s + static_cast<unsigned>(slot) * slot_bytes;
    // warp-uniform trip count: every lane reaches the member-sum shuffles; the
    // first header is loaded together with the count (slot 0 exists in every block)
    int count = 1;
    for (int t0 = 0; t0 < count; t0 += R) {
      const int t = t0 + sg;
      const unsigned hd = blk + 32u + 32u * min(t, tmax);
      const int4 c4 = ld_s_int4(blk);
      const int4 h0 = ld_s_int4(hd), h1 = ld_s_int4(hd + 16);
      count = c4.x;
      const bool act = t < count;
      const int cell = h0.x;
      const bool interior = h0.y >= 0;
      const int nm = (!act || interior) ? 0 : h0.w;  // group members (-1: domain boundary)
      const double B = ld_s64(sb_s + 8u * (act ? cell : 0));
      if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[3][g] = clock64() + (cell == -12345 ? 1 : 0);
      double o = 0.0;
      if (q < nm) {
        // member q's partial_row (proj/src/fem.cpp:138-172 cell order, coefficients inline)
        const unsigned mr = blk + 4u * static_cast<unsigned>(h0.z) + 4u * kSchedMemberWords * q;
        double k[6];
        ld_s_v2f64(mr, k[0], k[1]);
        ld_s_v2f64(mr + 16, k[2], k[3]);
        ld_s_v2f64(mr + 32, k[4], k[5]);
        const int4 ra = ld_s_int4(mr + 48), rb = ld_s_int4(mr + 64);
        const int nc = rb.z;
        const int rd[6] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y};
        double x[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) x[c] = ld_s64(su_s + 8u * rd[c]);
        // absent terms: zero coefficient x zero slot, o + 0 == o (o is never -0.0)
        (void)nc;
#pragma unroll
        for (int c = 0; c < 3; ++c) o = o + (k[2 * c] * x[2 * c] + k[2 * c + 1] * x[2 * c + 1]);
      }
      if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[4][g] = clock64() + (o == 12345.0 ? 1 : 0);
      // members summed in ascending slot; lanes beyond a group's members hold
      // +0.0, the bound is warp-uniform (the whole warp shuffles, converged)
      double ov[SG];
#pragma unroll
      for (int r = 0; r < SG; ++r) ov[r] = __shfl_sync(0xffffffffu, o, r, SG);
      double off = 0.0;
#pragma unroll
      for (int r = 0; r < SG; ++r) off = off + ov[r];
      if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[5][g] = clock64() + (off == 12345.0 ? 1 : 0) + (nm << 20);
      if (act && q == 0) {
        double res;
        if (interior) {
          // interior node, proj/src/multigrid.cpp:170-175 (SURVEY.md A.5 order)
          const unsigned st = mt_s + 208u * h0.y;
          const double E = ld_s64(su_s + 8u * h0.z), W = ld_s64(su_s + 8u * h0.w);
          const double N = ld_s64(su_s + 8u * h1.x), Sv = ld_s64(su_s + 8u * h1.y);
          const double NW = ld_s64(su_s + 8u * h1.z), SE = ld_s64(su_s + 8u * h1.w);
          double s1, s2, s3, s4, s5, s6, ic, pad;
          ld_s_v2f64(st, s1, s2);
          ld_s_v2f64(st + 16, s3, s4);
          ld_s_v2f64(st + 32, s5, s6);
          ld_s_v2f64(st + 48, ic, pad);
          double acc = s1 * E + s2 * W;
          acc = acc + s3 * N;
          acc = acc + s4 * Sv;
          acc = acc + s5 * NW;
          acc = acc + s6 * SE;
          res = (B - acc) * ic;
        } else if (h0.w < 0) {
          res = B;  // domain boundary: u = b
        } else {
          // relax_boundary_node, proj/src/multigrid.cpp:132-150
          const double diag = __longlong_as_double(static_cast<long long>(static_cast<unsigned>(h1.x)) |
                                                   (static_cast<long long>(h1.y) << 32));
          const double inv = __longlong_as_double(static_cast<long long>(static_cast<unsigned>(h1.z)) |
                                                  (static_cast<long long>(h1.w) << 32));
          const double xn = B - off;
          const double qq = xn * inv;
          const double r = __fma_rn(-qq, diag, xn);
          res = xn == 0.0 ? qq : __fma_rn(r, inv, qq);
        }
        st_s64(su_s + 8u * cell, res);
      }
    }
    if (KB_TRACING(trace) && tid == 0 && g < 512) g_sched_trace[2][g] = clock64();
    __syncthreads();
    if (tid == producer && g + K < total) {
      const int lvl = (g + K) % levels;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma_load_block(blk, blocks + loff[lvl], 4u * static_cast<unsigned>(loff[lvl + 1] - loff[lvl]),
                     mbar_s + 8u * slot);
    }
  }
  const size_t copies = static_cast<size_t>(M) * lv.S;
  for (size_t k = tid; k < copies; k += nthreads) u[k] = su[lv.sc_copy_cell[k]];
  if (KB_TRACING(trace) && tid == 0) {
    for (int g = 0; g < total && g < 40; ++g)
      printf("level %d: wait %lld hdr %lld member %lld sum %lld final %lld barrier+issue %lld nm %lld\n", g,
             g_sched_trace[1][g] - g_sched_trace[0][g], g_sched_trace[3][g] - g_sched_trace[1][g],
             g_sched_trace[4][g] - g_sched_trace[3][g], (g_sched_trace[5][g] & 0xfffff) - (g_sched_trace[4][g] & 0xfffff),
             g_sched_trace[2][g] - g_sched_trace[5][g], g + 1 < total ? g_sched_trace[0][g + 1] - g_sched_trace[2][g] : 0ll,
             g_sched_trace[5][g] >> 20);
  }
}

// ------------------------------------------------ Gauss-Seidel, pipelined
// One CTA per macro (all resident), the macro's lattice in shared memory, all
// sweeps of the call in one pass over global steps tau = s T + t.  The warps
// of group_sweep (boundary, program, interior) are the consumers; per step
// they bar.arrive on barrier A (step done) and bar.sync on barrier B (gate of
// the next step).  The sync warp owns the gates (PipeTables2D): it waits until
// the step's requirements hold (other macros' progress), re-reads the step's
// remote values from global memory into the lattice / ghost slots, then
// arrives on B; after A it publishes this macro's progress (st.release.gpu).
// Requirements of step tau + 2 are polled and its values fetched during step
// tau, so the gate normally opens at once; when it does not, progress is
// published first and the gate waits (no cyclic wait: every requirement names
// an event that precedes the step in the sequential order).
constexpr int kPipeBarB = 1, kPipeBarA0 = 2, kPipeBarAs = 8;  // gate; ring of step-done barriers (power of two)
constexpr int kPipePubs = 4;  // publisher warps
constexpr int kPipeRing = 16;  // step programs + gate records in flight
constexpr int kPipePRing = 16;  // record ring of the prefetch / gate warps (power of two)
constexpr int kPipePAhead = 4;  // record pairs requested ahead of the prefetch warp
constexpr int kPipeStage = 8;   // prefetched steps in flight (power of two, <= kPipePRing - 2 kPipePAhead)
constexpr int kPipeKnown = 64;  // observed-progress cache entries

__device__ __forceinline__ void bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void issue_prog(const unsigned long long* prog_m, unsigned ring_s, int t, int slot, int lane) {
  const char* src = reinterpret_cast<const char*>(prog_m + static_cast<size_t>(t) * kProgStepWords);
  const unsigned dst = ring_s + static_cast<unsigned>(slot) * kStepBytes;
  for (int c = lane; c < 48; c += 32)
    cp_async16(dst + static_cast<unsigned>(kLaneStride) * (c >> 3) + 16u * (c & 7), src + 16 * c);
}

__global__ void __launch_bounds__(384, 1) k_gs_pipe(DevLevel2D lv, double* u, const double* __restrict__ b,
                                                    int sweeps, int* progress, const int* __restrict__ rec,
                                                    int rec_words, int maxreq, int trace) {
  extern __shared__ __align__(16) double smem[];
#ifdef KB_GS_ABLATE
  // measurement builds only (results are wrong): drop one role's work per bit
  const int abl = trace >> 4;
#else
  constexpr int abl = 0;
#endif
  const int S = lv.S, n = lv.n, T = 2 * n + 1, m = blockIdx.x, total = sweeps * T;
  const int Wc = gs_group_warps(n), cthreads = 32 * Wc, bthreads = cthreads + 32;
  unsigned char* ring = reinterpret_cast<unsigned char*>(smem);
  int* pring = reinterpret_cast<int*>(ring + (kPipeRing * kStepBytes));  // gate records (prefetch warp's ring)
  unsigned long long* xs = reinterpret_cast<unsigned long long*>(pring + kPipePRing * 4 * kPipeLanes);
  double* gh = reinterpret_cast<double*>(xs + static_cast<size_t>(lv.max_extra) * kProgLaneWords);
  double* us = gh + lv.max_ghosts + 1;
  double* bs = us + S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned ring_s = smem_addr(ring);
  __shared__ int pub_last[kPipePubs];  // last step-done barrier each publisher passed
  __shared__ __align__(16) double fstage[kPipeStage][kPipeLanes][2];  // prefetched remote values (16-byte copies)
  __shared__ __align__(8) unsigned long long fbar[kPipeStage];  // slot filled (32 async arrivals)
  __shared__ int2 known[kPipeKnown];  // prefetch warp: last observed progress per macro (direct mapped)
  __shared__ int gate_pos;            // last gate opened
  const unsigned fbar_s = smem_addr(fbar);
#ifdef KB_GS_TRACE
  // per-step timeline of macro m for steps 64..127 (KB_PIPE_TRACE, trace builds):
  // 0 sync ready at B, 1 sync past B, 2 boundary past B, 3 boundary done,
  // 4 boundary ready at B, 5 interior warp 2 done, 6 last interior warp done,
  // 7 program warp at A, 8 publisher past A.  "Past" stamps are taken after a
  // shared load that the barrier orders (a clock read right after a deferred
  // BAR.SYNC records its issue, not its release)
  __shared__ long long ptr_t[12][64];
  __shared__ int ptr_dummy;
  if (tid == 0) ptr_dummy = 0;
#define PTR(row, st)                                                                     \
  do {                                                                                   \
    if ((trace & 1) && lane == 0 && (st) >= 64 && (st) < 128) {                                \
      if (*reinterpret_cast<volatile int*>(&ptr_dummy) != 12345) ptr_t[row][(st) - 64] = clock64(); \
    }                                                                                    \
  } while (0)
#else
#define PTR(row, st) \
  do {               \
  } while (0)
#endif
  if (tid < kPipePubs) pub_last[tid] = -1;
  if (tid < kPipeStage) mbar_init(fbar_s + 8u * tid, kPipeLanes);
  if (tid < kPipeKnown) known[tid] = make_int2(-1, 0);
  if (tid == 0) gate_pos = -1;
  const unsigned long long* prog_m = lv.prog + lv.prog_ptr[m];
  // sweep-0 records, then sweep-1 records (sweeps <= 2): step tau's record is rec_m0[tau]
  const int4* rec_m0 = reinterpret_cast<const int4*>(rec) + static_cast<size_t>(m) * 2 * T * kPipeLanes;
  double* um = u + static_cast<size_t>(m) * S;

  // initial state: lattice, b, extra records, ghosts; the head of the step stream
  {
    const double* bm = b + static_cast<size_t>(m) * S;
    for (int k = tid; k < S; k += blockDim.x) {
      us[k] = __ldcg(um + k);
      bs[k] = __ldg(bm + k);
    }
    const int xb = lv.xtra_ptr[m], xc = lv.xtra_ptr[m + 1] - xb;
    for (int x = tid; x < xc; x += blockDim.x) xs[x] = lv.prog_extra[xb + x];
    const int gbeg = lv.ghost_ptr[m], gcnt = lv.ghost_ptr[m + 1] - gbeg;
    for (int x = tid; x < gcnt; x += blockDim.x) gh[x] = __ldcg(u + lv.ghost_off[gbeg + x]);
    if (tid == 0) gh[lv.max_ghosts] = 0.0;
    if (warp == 1) {
      for (int tau = 0; tau < kPipeRing - 1 && tau < total; ++tau) {
        issue_prog(prog_m, ring_s, tau % T, tau & (kPipeRing - 1), lane);
        cp_async_commit();
      }
      cp_async_wait<0>();
    }
  }
  __syncthreads();

  if (warp > Wc + 1) {
    // ------------------------------------------------ publisher warps (off the gate barrier B): warp
    // Wc + 2 + w takes the step-done barriers A of steps tau = w mod kPipePubs and raises
    // progress[m] to tau + 2 (red.release.gpu.max: the release may finish out of order)
    const int w = warp - Wc - 2;
    for (int tau = w; tau < total; tau += kPipePubs) {
      bar_sync(kPipeBarA0 + (tau & (kPipeBarAs - 1)), bthreads);
      PTR(8, tau);
      if (lane == 0) {
        *reinterpret_cast<volatile int*>(&pub_last[w]) = tau;
        if (abl & 128) {
        } else if (abl & 32)
          asm volatile("red.relaxed.gpu.global.max.s32 [%0], %1;" ::"l"(progress + m), "r"(tau + 2) : "memory");
        else
          asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(progress + m), "r"(tau + 2) : "memory");
      }
    }
  } else if (warp == Wc + 1) {
    // ------------------------------------------------ prefetch warp
    // Runs up to kPipeStage steps ahead of the gate.  Per step s: wait until
    // the step's requirements hold (other macros' progress; an observed
    // progress value is remembered, so a requirement already met costs no
    // load), copy the step's remote values from L2 into stage slot
    // s % kPipeStage (cp.async, issued after the acquire that observed the
    // producer's release) and arrive on the slot's mbarrier when the copies
    // -- and every earlier cp.async of the lane, among them the step's record
    // the gate reads -- have landed (cp.async.mbarrier.arrive).  Records
    // (one int4 per lane, PipeTables2D) stream into a ring kPipePAhead steps
    // ahead.
    // Two steps per iteration: lanes 0-15 take the entries of step st, lanes
    // 16-31 those of step st + 1 (records of consecutive steps are adjacent).
    const unsigned pring_s = smem_addr(pring);
    const int4* prg = reinterpret_cast<const int4*>(pring);
    const int half = lane >> 4, ent = lane & (kPipeLanes - 1);
    auto issue_recs = [&](int st) {  // records st, st + 1 (st even), one 16-byte entry per lane
      if (st + half < total)
        cp_async16(pring_s + static_cast<unsigned>((st & (kPipePRing - 1)) * kPipeLanes + lane) * 16u,
                   rec_m0 + static_cast<size_t>(st) * kPipeLanes + lane);
    };
    for (int st = 0; st < 2 * kPipePAhead; st += 2) {
      issue_recs(st);
      cp_async_commit();
    }
    long long t_wait = 0, t_start = clock64();
    int n_wait = 0;
    for (int st = 0; st < total; st += 2) {
      cp_async_wait<kPipePAhead - 1>();  // records st, st + 1 landed (every lane's part)
      __syncwarp();
      const int sl = st + half;  // this lane's step
      // slot reuse: the gate of step st + 1 - kPipeStage has read its values and
      // the records the ring slots of st + 2 kPipePAhead (+1) held
      if (st + 1 >= kPipeStage)
        while (*reinterpret_cast<volatile int*>(&gate_pos) < st + 1 - kPipeStage) {
        }
      PTR(9, st);
      const int4 e = sl < total ? prg[(st & (kPipePRing - 1)) * kPipeLanes + lane] : make_int4(-1, 0, -1, 0);
      if (e.x >= 0 && !(abl & 8)) {
        const int2 kn = known[e.x & (kPipeKnown - 1)];
        if (kn.x != e.x || kn.y < e.y) {
          const int* pm = progress + e.x;
          int v;
          long long spins = 0;
          if (KB_TRACING(trace & 1)) ++n_wait, t_wait -= clock64();
          while ((v = ld_acquire(pm)) < e.y) {
            if (++spins == (1ll << 24)) {  // a broken table would deadlock: fail loudly instead
              printf("k_gs_pipe: macro %d step %d waits for macro %d progress %d (has %d)\n", m, sl, e.x, e.y, v);
              __trap();
            }
          }
          if (KB_TRACING(trace & 1)) t_wait += clock64();
          known[e.x & (kPipeKnown - 1)] = make_int2(e.x, v);
        }
      }
      // each half goes on as soon as its own step's requirements hold: step st
      // must not wait for the requirements of step st + 1 (a cycle otherwise)
      __syncwarp(half ? 0xffff0000u : 0x0000ffffu);
      PTR(10, st);
      const int slot = sl & (kPipeStage - 1);
      if (e.z >= 0 && !(abl & 64)) {
        KB_ASSERT(e.z < lv.M * S);
        cp_async16(smem_addr(&fstage[slot][ent][0]), u + (e.z & ~1));
      }
      if (sl < total)
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fbar_s + 8u * slot) : "memory");
      issue_recs(st + 2 * kPipePAhead);
      cp_async_commit();
      PTR(11, st);
    }
    cp_async_wait<0>();
    if (KB_TRACING(trace & 1) && lane == 0 && (m % 20 == 0 || m == gridDim.x - 1))
      printf("pipe macro %d: steps %d, prefetch waits %d, cycles waiting %lld of %lld\n", m, total, n_wait, t_wait,
             clock64() - t_start);
  } else if (warp == Wc) {
    // ------------------------------------------------ gate warp
    // gate of step g: wait for the prefetched values of step g (slot mbarrier,
    // which also covers the step's record), store them into the lattice /
    // ghost slots, arrive on B
    const int2* prg = reinterpret_cast<const int2*>(pring);
    for (int g = 0, slot = 0, ph = 0; g < total; ++g) {
      mbar_wait(fbar_s + 8u * slot, ph);
      if (lane < kPipeLanes) {
        const int2 e = prg[((g & (kPipePRing - 1)) * kPipeLanes + lane) * 2 + 1];  // {source, destination}
        if (e.x >= 0) {
          const double v = fstage[slot][lane][e.x & 1];
          KB_ASSERT(e.y < S && -1 - e.y <= lv.max_ghosts);
          if (e.y >= 0)
            us[e.y] = v;
          else
            gh[-1 - e.y] = v;
        }
      }
      __syncwarp();
      if (lane == 0) *reinterpret_cast<volatile int*>(&gate_pos) = g;
      if (++slot == kPipeStage) slot = 0, ph ^= 1;
      // the step-done barrier of step g reuses the one of step g - kPipeBarAs: its
      // publisher must have passed it (flow control only)
      if (g >= kPipeBarAs && !(abl & 512)) {
        const int gp = g - kPipeBarAs;
        while (*reinterpret_cast<volatile int*>(&pub_last[gp & (kPipePubs - 1)]) < gp) {
        }
      }
      __syncwarp();
      PTR(0, g);
      bar_sync(kPipeBarB, bthreads);  // gate of step g opens
      PTR(1, g);
    }
  } else {
    // ------------------------------------------------ consumers (group_sweep roles)
    const int gw = warp;
    const unsigned us_s = smem_addr(us), bs_s = smem_addr(bs), gh_s = smem_addr(gh), xs_s = smem_addr(xs);
    bar_sync(kPipeBarB, bthreads);  // gate of step 0
    if (gw == 1) {
      for (int tau = 0, tn = (kPipeRing - 1) % T; tau < total; ++tau, tn = (tn + 1 == T ? 0 : tn + 1)) {
        const int nx = tau + kPipeRing - 1;  // step nx = tn mod T
        if (nx < total && !(abl & 16))
          issue_prog(prog_m, ring_s, tn, nx & (kPipeRing - 1), lane);
        cp_async_commit();
        if (!(abl & 256)) cp_async_wait<kPipeRing - 7>();  // steps and records <= tau + 6 landed (read by the sync warp after A)
        PTR(7, tau);
        bar_arrive(kPipeBarA0 + (tau & (kPipeBarAs - 1)), bthreads);
        if (tau + 1 < total) bar_sync(kPipeBarB, bthreads);
      }
      cp_async_wait<0>();
    } else if (gw == 0) {
      const int type = lane >> 3, mem = lane & 7;
      const int tl = type < 3 ? type : 0;
      // the next step's lane records are read while waiting for its gate, so
      // they do not queue in front of this step's lattice reads
      PipeNode p0, p1;
      const unsigned gx_s = gh_s;
      auto slot_of = [&](int tau) { return ring_s + static_cast<unsigned>(tau & (kPipeRing - 1)) * kStepBytes; };
      auto relax = [&](const PipeNode& p, PipeNode& nx, int tau) {
        const bool more = tau + 1 < total && !(abl & 4);
        relax_pipe(
            p, us_s, u, lv.wr, lane, um, lv.max_ghosts + 1 + S, S, lv.M * S, gx_s,
            [&] {
              if (more) pnode_issue(nx, pnode_rec(slot_of(tau + 1), tl, mem));
            },
            [&] {
              if (more) pnode_finish(nx, xs_s, bs_s, gx_s, mem);
            });
      };
      pnode_issue(p0, pnode_rec(ring_s, tl, mem));
      pnode_finish(p0, xs_s, bs_s, gx_s, mem);
      for (int tau = 0; tau < total; tau += 2) {
        PTR(2, tau);
        if (!(abl & 2)) relax(p0, p1, tau);
        PTR(3, tau);
        bar_arrive(kPipeBarA0 + (tau & (kPipeBarAs - 1)), bthreads);
        if (tau + 1 >= total) break;
        PTR(4, tau + 1);
        bar_sync(kPipeBarB, bthreads);
        PTR(2, tau + 1);
        if (!(abl & 2)) relax(p1, p0, tau + 1);
        PTR(3, tau + 1);
        bar_arrive(kPipeBarA0 + ((tau + 1) & (kPipeBarAs - 1)), bthreads);
        if (tau + 2 >= total) break;
        PTR(4, tau + 2);
        bar_sync(kPipeBarB, bthreads);
      }
    } else {
      const double* st = lv.stencil + 7 * m;
      const double s1 = st[1], s2 = st[2], s3 = st[3], s4 = st[4], s5 = st[5], s6 = st[6];
      const double inv_c = lv.inv_c[m];
      const int j = 32 * (gw - 2) + lane + 1;
      const bool row = j <= n - 1;
      const int rowk = row ? dlat(n, 0, j) : 0;
      const int dn = n + 1 - j, dnw = n - j, ds = n + 2 - j;
      int t = 0;  // tau mod T, kept incrementally (no division on the step path)
      for (int tau = 0; tau < total; ++tau, t = (t + 1 == T ? 0 : t + 1)) {
        const int i = t - 2 * j;
        if (!(abl & 1) && row && i >= 1 && i <= n - j - 1) {
          const int k = rowk + i;
          const double B = bs[k];
          const double E = us[k + 1], W = us[k - 1], N = us[k + dn], Sv = us[k - ds];
          const double NW = us[k + dnw], SE = us[k - dn];
          double acc = s1 * E + s2 * W;
          acc = acc + s3 * N;
          acc = acc + s4 * Sv;
          acc = acc + s5 * NW;
          acc = acc + s6 * SE;
          const double v = (B - acc) * inv_c;
          us[k] = v;
          if (j == 1 || i == 1 || i + j == n - 1) um[k] = v;  // exported: ghost of a neighbour
        }
        if (gw == 2) PTR(5, tau);
        if (gw == Wc - 1) PTR(6, tau);
        bar_arrive(kPipeBarA0 + (tau & (kPipeBarAs - 1)), bthreads);
        if (tau + 1 < total) bar_sync(kPipeBarB, bthreads);
      }
    }
  }
  __syncthreads();
#ifdef KB_GS_TRACE
  if ((trace & 1) && tid == 0 && m % 20 == 0) printf("trace end m %d\n", m);
  if ((trace & 1) && (m == 0 || m == gridDim.x / 2) && tid == 0)
    for (int q = 0; q < 24; ++q) {
      const long long b0 = ptr_t[2][q];  // boundary past B of step 64 + q
      printf("m %d step %d: %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld | next B %6lld\n", m, 64 + q,
             ptr_t[0][q] - b0, ptr_t[1][q] - b0, ptr_t[2][q] - b0, ptr_t[3][q] - b0, ptr_t[4][q] - b0,
             ptr_t[5][q] - b0, ptr_t[6][q] - b0, ptr_t[7][q] - b0, ptr_t[8][q] - b0, ptr_t[2][q + 1] - b0);
      printf("m %d step %d: prefetch %6lld %6lld %6lld\n", m, 64 + q, ptr_t[9][q] - b0, ptr_t[10][q] - b0,
             ptr_t[11][q] - b0);
    }
#endif
#undef PTR
  // lattice-interior nodes back to global memory (interface copies are kept
  // current by every relaxation)
  for (int k = tid; k < S; k += blockDim.x) {
    int i, j;
    decode(n, k, i, j);
    if (i >= 1 && j >= 1 && i + j <= n - 1) um[k] = us[k];
  }
}

// ---------------------------------------------------------------- exact error (validation)
// ExactErrorEvaluator::evaluate, proj/src/fem.cpp:395-420: one thread per
// macro keeps the reference's sequential sums (the three-term form cancels,
// so the order matters at the 1e-9 level)
__global__ void k_exact_eval(DevLevel2D lv, const double* __restrict__ uL, const double* __restrict__ mom,
                             double* out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= lv.M) return;
  const int n = lv.n, S = lv.S;
  const double* cm = uL + static_cast<size_t>(m) * S;
  const double* mm = mom + static_cast<size_t>(m) * S;
  double cross = 0.0;
  for (int k = 0; k < S; ++k) cross += mm[k] * cm[k];
  const double* ku = lv.kmass + 18 * static_cast<size_t>(m);  // the up-cell mass matrix for every cell
  const double k0 = ku[0], k1 = ku[1], k2 = ku[2], k3 = ku[3], k4 = ku[4], k5 = ku[5], k6 = ku[6], k7 = ku[7],
               k8 = ku[8];
  double uh_sq = 0.0;
  auto cell = [&](int a, int b, int c) {
    const double xa = cm[a], xb = cm[b], xc = cm[c];
    uh_sq += xa * (k0 * xa + k1 * xb + k2 * xc) + xb * (k3 * xa + k4 * xb + k5 * xc) +
             xc * (k6 * xa + k7 * xb + k8 * xc);
  };
  for (int j = 0; j < n; ++j) {
    const int r0 = dlat(n, 0, j), r1 = dlat(n, 0, j + 1);
    for (int i = 0; i < n - j; ++i) cell(r0 + i, r0 + i + 1, r1 + i);
    for (int i = 0; i + 1 < n - j; ++i) cell(r0 + i + 1, r1 + i, r1 + i + 1);
  }
  out[2 * m] = cross;
  out[2 * m + 1] = uh_sq;
}

// ---------------------------------------------------------------- estimator
__device__ __forceinline__ double quad_form(const double* k, double a, double b, double c) {
  return a * (k[0] * a + k[1] * b + k[2] * c) + b * (k[3] * a + k[4] * b + k[5] * c) +
         c * (k[6] * a + k[7] * b + k[8] * c);
}

// One CTA per macro: e_base = u_L - wb and e_coarser = u_L - P wc (inline
// prolongation from level L-1); per-macro sums of e^T M_T e over all cells
// (local_l2_norms, proj/src/fem.cpp:327-356) in a fixed reduction order.
__global__ void k_estimate(DevLevel2D lv, const double* __restrict__ uL, const double* __restrict__ wb,
                           const double* __restrict__ wc, double* sums) {
  const int slot = blockIdx.x;
  const int n = lv.n, S = lv.S, nc = n / 2, Sc = (nc + 1) * (nc + 2) / 2;
  const double* u = uL + static_cast<size_t>(slot) * S;
  const double* w1 = wb + static_cast<size_t>(slot) * S;
  const double* w2 = wc + static_cast<size_t>(slot) * Sc;
  const double* K = lv.kmass + 18 * slot;  // up == down for the mass matrix
  double qb = 0.0, qc = 0.0;
  for (int idx = threadIdx.x; idx < S; idx += blockDim.x) {
    int i, j;
    decode(n, idx, i, j);
    if (i + j > n - 1) continue;
    const int a = dlat(n, i, j), bq = dlat(n, i + 1, j), c = dlat(n, i, j + 1);
    const double ua = u[a], ub = u[bq], uc = u[c];
    const double eba = ua - w1[a], ebb = ub - w1[bq], ebc = uc - w1[c];
    const double eca = ua - prolong_value(w2, nc, i, j), ecb = ub - prolong_value(w2, nc, i + 1, j),
                 ecc = uc - prolong_value(w2, nc, i, j + 1);
    qb += quad_form(K, eba, ebb, ebc);
    qc += quad_form(K, eca, ecb, ecc);
    if (i + j <= n - 2) {
      const int d = dlat(n, i + 1, j + 1);
      const double ud = u[d];
      const double ebd = ud - w1[d];
      const double ecd = ud - prolong_value(w2, nc, i + 1, j + 1);
      qb += quad_form(K + 9, ebb, ebc, ebd);
      qc += quad_form(K + 9, ecb, ecc, ecd);
    }
  }
  __shared__ double rb[kThreads], rcq[kThreads];
  rb[threadIdx.x] = qb;
  rcq[threadIdx.x] = qc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      rb[threadIdx.x] += rb[threadIdx.x + w];
      rcq[threadIdx.x] += rcq[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sums[2 * slot] = rb[0];
    sums[2 * slot + 1] = rcq[0];
  }
}

// ---------------------------------------------------------------- misc
__global__ void k_dot_partial(DevLevel2D lv, const double* a, const double* b, double* partial) {
  double s = 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < lv.dot_count; t += gridDim.x * blockDim.x) {
    const int k = lv.dot_order[t];
    s += a[k] * b[k];
  }
  __shared__ double red[kThreads];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// dot_unique in the reference's exact sequential order (proj/src/hhg.cpp:227-257):
// lanes form 32 products at a time, lane 0 adds them in order
__global__ void k_dot_seq(DevLevel2D lv, const double* a, const double* b, double* out) {
  const int lane = threadIdx.x;
  double s = 0.0;
  for (int t0 = 0; t0 < lv.dot_count; t0 += 32) {
    const int t = t0 + lane;
    double p = 0.0;
    if (t < lv.dot_count) {
      const int k = lv.dot_order[t];
      p = a[k] * b[k];
    }
    const int cnt = min(32, lv.dot_count - t0);
    for (int r = 0; r < cnt; ++r) {
      const double v = __shfl_sync(0xffffffffu, p, r);
      s = s + v;
    }
  }
  if (lane == 0) *out = s;
}

__global__ void k_dot_final(const double* partial, int count, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += partial[i];
    *out = s;
  }
}

__global__ void k_sync(DevLevel2D lv, double* f, int additive, int ngroups) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ngroups; g += gridDim.x * blockDim.x) {
    const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
    if (end - beg < 2) continue;
    if (additive) {
      double sum = 0.0;
      for (int m = beg; m < end; ++m) sum += f[lv.mem_off[m]];
      for (int m = beg; m < end; ++m) f[lv.mem_off[m]] = sum;
    } else {
      const double v = f[lv.mem_off[beg]];
      for (int m = beg + 1; m < end; ++m) f[lv.mem_off[m]] = v;
    }
  }
}

__global__ void k_axpy(double* y, const double* x, double alpha, long long count) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    y[k] = y[k] + alpha * x[k];
}

__global__ void k_scale_add(double* y, double beta, const double* x, long long count) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double t = y[k] * beta;
    y[k] = t + 1.0 * x[k];
  }
}

int grid_for(long long total) {
  long long g = (total + kThreads - 1) / kThreads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g);
}

void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(KB_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void launch_apply(const DevLevel2D& lv, const double* K, const double* x, double* y, const double* b,
                  int mode, cudaStream_t st) {
  const int chunks = (lv.S + 255) / 256;
  const int interior_blocks = lv.M * chunks;
  const int group_blocks = (lv.num_groups + 255) / 256;
  k_apply2<<<interior_blocks + group_blocks, 256, 0, st>>>(lv, K, x, y, b, mode, chunks, interior_blocks);
  check_launch("k_apply");
}

void launch_restrict(const DevLevel2D& fine, const DevLevel2D& coarse, const double* r, double* rc,
                     int zero_boundary, cudaStream_t st, double* zero_out) {
  k_restrict<<<grid_for(static_cast<long long>(coarse.M) * coarse.S), kThreads, 0, st>>>(fine, coarse, r, rc,
                                                                                         zero_boundary, zero_out);
  check_launch("k_restrict");
}

void launch_prolong(const DevLevel2D& coarse, const DevLevel2D& fine, const double* c, double* f,
                    double* next, const double* gbnd, int mode, cudaStream_t st) {
  k_prolong<<<grid_for(static_cast<long long>(fine.M) * fine.S), kThreads, 0, st>>>(coarse, fine, c, f, next,
                                                                                    gbnd, mode);
  check_launch("k_prolong");
}

void launch_set_boundary(const DevLevel2D& lv, double* f, const double* gbnd, int zero_rest, cudaStream_t st) {
  k_set_boundary<<<grid_for(static_cast<long long>(lv.M) * lv.S), kThreads, 0, st>>>(lv, f, gbnd, zero_rest);
  check_launch("k_set_boundary");
}

void launch_rhs(const DevLevel2D& lv, int src_kind, const double* ftab, double* ftab_scratch,
                const double* gbnd, double* b, cudaStream_t st) {
  const double* F = ftab;
  if (src_kind != SRC_ZERO && src_kind != SRC_TABLE) {
    const long long SF = static_cast<long long>(2 * lv.n + 1) * (2 * lv.n + 2) / 2;
    k_ftab<<<grid_for(lv.M * SF), kThreads, 0, st>>>(lv, src_kind, ftab_scratch);
    check_launch("k_ftab");
    F = ftab_scratch;
  }
  k_rhs<<<grid_for(static_cast<long long>(lv.M) * lv.S), kThreads, 0, st>>>(lv, F, gbnd, b,
                                                                            src_kind == SRC_ZERO ? 1 : 0);
  check_launch("k_rhs");
}

namespace {
template <typename K>
void set_smem(K kernel, size_t smem);
}  // namespace

void launch_cg0(const DevLevel2D& lv0, double* u, const double* b, double* scratch, CgParams prm,
                DevStatus* status, cudaStream_t st) {
  (void)scratch;
  const size_t cnt2 = (static_cast<size_t>(lv0.dot_count) + 1) & ~size_t(1), nmem = static_cast<size_t>(lv0.cg_nmem);
  const size_t smem = 6 * cnt2 * 8 + nmem * 8 + 3 * nmem * 8 + 3 * nmem * 4 + (cnt2 + 1) * 4 + cnt2 + 16;
  if (smem > 200 * 1024) fail(KB_STRUCTURAL, "coarse mesh too large for the level-0 CG");
  set_smem(k_cg0, smem);
  k_cg0<<<1, kCg0Threads, smem, st>>>(lv0, u, b, prm, status);
  check_launch("k_cg0");
}

int gs_block_threads(int n) { return 32 * ((n + 1 + 31) / 32); }

namespace {
int device_attr(cudaDeviceAttr a) {
  int dev = 0, v = 0;
  KB_CUDA_CHECK(cudaGetDevice(&dev));
  KB_CUDA_CHECK(cudaDeviceGetAttribute(&v, a, dev));
  return v;
}

template <typename K>
void set_smem(K kernel, size_t smem) {
  ensure_dynamic_smem(kernel, smem);
}

void launch_gs_level(const DevHier2D& hd, const DevLevel2D& lv, double* u, const double* b, int sweeps,
                     cudaStream_t st, size_t smem, int groups) {
  set_smem(k_gs_level, smem);
  k_gs_level<<<1, 32 * gs_group_warps(lv.n) * groups, smem, st>>>(hd, lv, u, b, sweeps);
  check_launch("k_gs_level");
}

void launch_gs_macro(const DevHier2D& hd, const DevLevel2D& lv, double* u, const double* b, int sweeps, int* done,
                     cudaStream_t st, size_t smem, int num_sms) {
  const int threads = 32 * gs_group_warps(lv.n);
  set_smem(k_gs_macro, smem);
  int occ = 0;
  KB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gs_macro, threads, smem));
  if (occ < 1) fail(KB_CUDA, "k_gs_macro cannot be resident");
  int grid = lv.M;
  if (grid > occ * num_sms) grid = occ * num_sms;
  KB_CUDA_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * lv.M, st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_gs_macro, hd, lv, u, b, sweeps, done));
}
}  // namespace

// Smoother dispatch: the whole level in one CTA's shared memory when it fits,
// else one shared-memory CTA per macro, else (n > 128) the register-wavefront
// kernel with the lattice in L2.
// shared memory of k_gs_sched for schedule si with K ring slots (0: does not fit)
size_t gs_sched_smem(const DevLevel2D& lv, int si, int smem_max, int* K_out, int* slot_out) {
  if (lv.sc_nu <= 0 || !lv.sc_blocks[si] || lv.sc_max_members[si] > 32) return 0;
  const size_t tables = 16 * static_cast<size_t>(lv.sc_nu + 1) + 8 * 26 * static_cast<size_t>(lv.M) +
                        16 * static_cast<size_t>(lv.num_groups) + 4 * static_cast<size_t>(lv.sc_levels[si] + 1);
  const size_t head = ((tables + 15) & ~size_t(15)) + 8 * 8;  // mbarriers (<= 8)
  const size_t slot = (4 * static_cast<size_t>(lv.sc_max_block[si]) + 15) & ~size_t(15);
  if (head + 2 * slot > static_cast<size_t>(smem_max)) return 0;
  const size_t fit = (static_cast<size_t>(smem_max) - head) / slot;
  const int K = fit >= 8 ? 8 : fit >= 4 ? 4 : 2;  // a power of two
  *K_out = K;
  *slot_out = static_cast<int>(slot);
  return head + K * slot;
}

bool gs_sched_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_GS_SCHED");
    v = e ? (e[0] != '0') : 1;
  }
  return v == 1;
}

bool gs_pipe_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_GS_PIPE");
    v = e ? (e[0] != '0') : 1;
  }
  return v == 1;
}

void launch_gs(const DevHier2D& hd, const DevLevel2D& lv, double* u, const double* b, int sweeps, int* done,
               cudaStream_t st) {
  if (sweeps <= 0) return;
  static int num_sms = 0, smem_max = 0;
  if (num_sms == 0) {
    num_sms = device_attr(cudaDevAttrMultiProcessorCount);
    smem_max = device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin);
  }
  if (gs_sched_enabled()) {
    // the static dependence-level schedule (small levels)
    const int si = sweeps == 2 ? 1 : 0, reps = sweeps == 2 ? 1 : sweeps;
    int K = 0, slot = 0;
    const size_t smem = gs_sched_smem(lv, si, smem_max, &K, &slot);
    if (smem > 0) {
      static int trace = getenv("KB_SCHED_TRACE") ? 1 : 0;
      const int SG = lv.sc_max_members[si] <= 4 ? 4 : lv.sc_max_members[si] <= 8 ? 8 : lv.sc_max_members[si] <= 16 ? 16 : 32;
      // at most 512 threads: wider levels take a second pass, every level's block
      // barrier is cheaper (cfg2 k = 5, level 3: 277 -> 264 us per 2-sweep call)
      static const int cap = getenv("KB_SCHED_THREADS") ? atoi(getenv("KB_SCHED_THREADS")) : 512;
      const int threads = static_cast<int>(
          std::min<long long>(cap, std::max<long long>(64, ((static_cast<long long>(lv.sc_max_width[si]) * SG + 31) / 32) * 32)));
      auto go = [&](auto kern) {
        set_smem(kern, smem);
        kern<<<1, threads, smem, st>>>(lv, u, b, si, reps, K, slot, trace);
      };
      if (SG == 4) go(k_gs_sched<4>);
      else if (SG == 8) go(k_gs_sched<8>);
      else if (SG == 16) go(k_gs_sched<16>);
      else go(k_gs_sched<32>);
      trace = 0;
      check_launch("k_gs_sched");
      return;
    }
  }
  if (lv.pipe_rec && sweeps <= 2 && gs_pipe_enabled()) {
    // fine-grained pipelined smoother: one resident CTA per macro
    const int threads = 32 * (gs_group_warps(lv.n) + 2 + kPipePubs);
    const size_t smem = kPipeRing * kStepBytes + static_cast<size_t>(kPipePRing) * kPipeLanes * 16 +
                        static_cast<size_t>(lv.max_extra) * kProgLaneWords * 8 + (lv.max_ghosts + 1) * 8 +
                        2 * static_cast<size_t>(lv.S) * 8;
    static size_t pipe_static = 0;
    if (!pipe_static) {
      cudaFuncAttributes fa{};
      KB_CUDA_CHECK(cudaFuncGetAttributes(&fa, k_gs_pipe));
      pipe_static = fa.sharedSizeBytes;
    }
    if (threads <= 384 && smem + pipe_static <= static_cast<size_t>(smem_max)) {
      set_smem(k_gs_pipe, smem);
      int occ = 0;
      KB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gs_pipe, threads, smem));
      if (occ * num_sms >= lv.M) {
        KB_CUDA_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * lv.M, st));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(lv.M);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // every macro's CTA resident at once
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        static int trace = getenv("KB_PIPE_TRACE") ? 1 : 0;
        static const int ablate = getenv("KB_PIPE_ABLATE") ? atoi(getenv("KB_PIPE_ABLATE")) : 0;  // KB_GS_ABLATE builds
        KB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_gs_pipe, lv, u, b, sweeps, done, lv.pipe_rec, lv.pipe_rec_words,
                                         lv.pipe_maxreq, trace | (ablate << 4)));
        trace &= ~1;
        return;
      }
    }
  }
  const size_t S = static_cast<size_t>(lv.S), M = static_cast<size_t>(lv.M);
  const int W = gs_group_warps(lv.n);
  if (W <= 6) {
    // groups per CTA: named barriers 1..kMaxLevelGroups, at most 512 threads
    const int groups = std::max(1, std::min(std::min(kMaxLevelGroups, 16 / W), hd.dag_width));
    const size_t gwords = gs_group_words(lv);
    const size_t level_smem = 2 * M * S * sizeof(double) + ((gs_level_table_bytes(lv.M, hd.dag_depth) + 15) & ~15ull) +
                              static_cast<size_t>(groups) * gs_level_group_bytes(lv);
    if (level_smem <= static_cast<size_t>(smem_max)) {
      launch_gs_level(hd, lv, u, b, sweeps, st, level_smem, groups);
      return;
    }
    const size_t macro_smem = gwords * 8 + 2 * S * sizeof(double);
    if (macro_smem <= static_cast<size_t>(smem_max)) {
      launch_gs_macro(hd, lv, u, b, sweeps, done, st, macro_smem, num_sms);
      return;
    }
  }
  const int threads = gs_block_threads(lv.n);
  if (threads > 576) fail(KB_STRUCTURAL, "wavefront smoother supports n <= 575");
  const int nwarps = threads / 32;
  const size_t smem = sizeof(double) * (lv.max_ghosts + nwarps * kRing) + sizeof(int) * nwarps + 16;
  set_smem(k_gs, smem);
  int occ = 0;
  KB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gs, threads, smem));
  if (occ < 1) fail(KB_CUDA, "k_gs cannot be resident");
  int grid = lv.M;
  if (grid > occ * num_sms) grid = occ * num_sms;
  KB_CUDA_CHECK(cudaMemsetAsync(done, 0, sizeof(int) * lv.M, st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_gs, hd, lv, u, b, sweeps, done));
}

void launch_exact_eval(const DevLevel2D& lv, const double* uL, const double* moments, double* out, cudaStream_t st) {
  k_exact_eval<<<(lv.M + 63) / 64, 64, 0, st>>>(lv, uL, moments, out);
  check_launch("k_exact_eval");
}

void launch_estimate(const DevLevel2D& lv, const double* uL, const double* wb, const double* wc, double* sums,
                     cudaStream_t st) {
  k_estimate<<<lv.M, kThreads, 0, st>>>(lv, uL, wb, wc, sums);
  check_launch("k_estimate");
}

void launch_dot(const DevLevel2D& lv, const double* a, const double* b, double* partial, double* out,
                cudaStream_t st) {
  const int blocks = 64;
  k_dot_partial<<<blocks, kThreads, 0, st>>>(lv, a, b, partial);
  k_dot_final<<<1, 32, 0, st>>>(partial, blocks, out);
  check_launch("k_dot");
}

void launch_dot_seq(const DevLevel2D& lv, const double* a, const double* b, double* out, cudaStream_t st) {
  k_dot_seq<<<1, 32, 0, st>>>(lv, a, b, out);
  check_launch("k_dot_seq");
}

void launch_sync(const DevLevel2D& lv, double* f, int additive, cudaStream_t st) {
  k_sync<<<grid_for(lv.num_groups), kThreads, 0, st>>>(lv, f, additive, lv.num_groups);
  check_launch("k_sync");
}

#ifdef KB_GS_TRACE
extern "C" int klref_debug_gs_trace(long long* host, int count) {
  return cudaMemcpyFromSymbol(host, g_gs_trace, sizeof(long long) * count) == cudaSuccess ? 0 : 1;
}
#endif

void launch_scale_add(double* y, double beta, const double* x, std::int64_t count, cudaStream_t st) {
  k_scale_add<<<grid_for(count), kThreads, 0, st>>>(y, beta, x, count);
  check_launch("k_scale_add");
}

void launch_axpy(double* y, const double* x, double alpha, std::int64_t count, cudaStream_t st) {
  k_axpy<<<grid_for(count), kThreads, 0, st>>>(y, x, alpha, count);
  check_launch("k_axpy");
}

}  // namespace kb
