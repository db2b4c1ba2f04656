// sm_100a kernels of the 3-d hot path (fp64, HBM-bound, no tensor cores).
// The reference has no 3-d solver; the operation orders below are the
// builder's specification, restated sequentially by oracle/klref_oracle3d.c
// (tests compare bit for bit).  Compiled with -fmad=false like the 2-d path.
//
//   apply / residual    15-point stencil on lattice-interior nodes (plane-
//                       parallel), member partial rows + additive sync on the
//                       shared-node groups (like proj/src/fem.cpp:95-173)
//   gauss_seidel        multicolour: boundary groups colour by colour, then
//                       every macro's interior colour by colour (one launch
//                       per colour, rows to warps, read-only path for u)
//   restrict / prolong  Freudenthal linear interpolation and its transpose
//   cg0                 level-0 CG in one CTA (proj/src/multigrid.cpp:198-229 order)
//   estimate            fused per-macro e^T M e over all micro-cells
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dev3d.hpp"

namespace kb {
namespace {

constexpr int kT = 256;

__constant__ int c_cv[6][4][3];  // vertex r of a type-t micro-cell relative to its base
__constant__ int c_dir[15][3];
__constant__ int c_pdir[8];      // parity pattern -> direction index (prolongation)
__device__ unsigned long long g_gs3_trace[64];  // measurement trace of k3_gs_sweeps (globaltimer ns)
// compile-time tables (indices resolve in unrolled loops; no local memory)
__device__ __forceinline__ constexpr int row_dk(int t) {
  constexpr int v[7] = {0, 0, 0, 1, -1, 1, -1};
  return v[t];
}
__device__ __forceinline__ constexpr int row_dj(int t) {
  constexpr int v[7] = {0, 1, -1, -1, 1, 0, 0};
  return v[t];
}
__device__ __forceinline__ constexpr int dir_row(int d) {  // neighbour row (0..6) of direction d
  constexpr int v[15] = {0, 0, 0, 1, 2, 3, 4, 1, 2, 5, 6, 3, 4, 5, 6};
  return v[d];
}
__device__ __forceinline__ constexpr int dir_di(int d) {  // i offset of direction d (kDir[d][0])
  constexpr int v[15] = {0, 1, -1, -1, 1, 0, 0, 0, 0, -1, 1, 1, -1, 0, 0};
  return v[d];
}

__device__ __forceinline__ int tsz(int n) { return (n + 1) * (n + 2) * (n + 3) / 6; }
__device__ __forceinline__ int lat2(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }
__device__ __forceinline__ int lat3(int n, int i, int j, int k) { return tsz(n) - tsz(n - k) + lat2(n - k, i, j); }
__device__ __forceinline__ bool inl(int n, int i, int j, int k) {
  return i >= 0 && j >= 0 && k >= 0 && i + j + k <= n;
}
__device__ __forceinline__ bool interior3(int n, int i, int j, int k) {
  return i >= 1 && j >= 1 && k >= 1 && i + j + k <= n - 1;
}
// (i, j) of the 2-d index q in a plane lattice of size m
__device__ __forceinline__ void decode2(int m, int q, int& i, int& j) {
  const float a = 2.0f * m + 3.0f;
  int jj = static_cast<int>((a - sqrtf(a * a - 8.0f * q)) * 0.5f);
  jj = max(0, min(jj, m));
  while (jj < m && lat2(m, 0, jj + 1) <= q) ++jj;
  while (jj > 0 && lat2(m, 0, jj) > q) --jj;
  j = jj;
  i = q - lat2(m, 0, jj);
}

// decode2 for m <= 1024 with one correction step each way (float sqrt is within one row)
__device__ __forceinline__ void decode2_fast(int m, int q, int& i, int& j) {
  const float a = 2.0f * m + 3.0f;
  int jj = static_cast<int>((a - sqrtf(fmaxf(a * a - 8.0f * q, 0.0f))) * 0.5f);
  jj = jj + (jj < m && lat2(m, 0, jj + 1) <= q);
  jj = jj - (jj > 0 && lat2(m, 0, jj) > q);
  j = jj;
  i = q - lat2(m, 0, jj);
}

__device__ __forceinline__ int sig3(int n, int i, int j, int k) {
  return (i == 0) | ((j == 0) << 1) | ((k == 0) << 2) | ((i + j + k == n) << 3);
}

// 15 independent fp64 loads issued back to back (see partial_row)
__device__ __forceinline__ void load15(double (&v)[15], const double* const (&a)[15]) {
  asm volatile(
      "ld.global.f64 %0, [%15];\n\t"
      "ld.global.f64 %1, [%16];\n\t"
      "ld.global.f64 %2, [%17];\n\t"
      "ld.global.f64 %3, [%18];\n\t"
      "ld.global.f64 %4, [%19];\n\t"
      "ld.global.f64 %5, [%20];\n\t"
      "ld.global.f64 %6, [%21];\n\t"
      "ld.global.f64 %7, [%22];\n\t"
      "ld.global.f64 %8, [%23];\n\t"
      "ld.global.f64 %9, [%24];\n\t"
      "ld.global.f64 %10, [%25];\n\t"
      "ld.global.f64 %11, [%26];\n\t"
      "ld.global.f64 %12, [%27];\n\t"
      "ld.global.f64 %13, [%28];\n\t"
      "ld.global.f64 %14, [%29];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]), "=d"(v[8]),
        "=d"(v[9]), "=d"(v[10]), "=d"(v[11]), "=d"(v[12]), "=d"(v[13]), "=d"(v[14])
      : "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(a[4]), "l"(a[5]), "l"(a[6]), "l"(a[7]), "l"(a[8]), "l"(a[9]),
        "l"(a[10]), "l"(a[11]), "l"(a[12]), "l"(a[13]), "l"(a[14])
      : "memory");
}
// 15 consecutive fp64 values
__device__ __forceinline__ void load15_seq(double (&v)[15], const double* p) {
  asm volatile(
      "ld.global.f64 %0, [%15];\n\t"
      "ld.global.f64 %1, [%15+8];\n\t"
      "ld.global.f64 %2, [%15+16];\n\t"
      "ld.global.f64 %3, [%15+24];\n\t"
      "ld.global.f64 %4, [%15+32];\n\t"
      "ld.global.f64 %5, [%15+40];\n\t"
      "ld.global.f64 %6, [%15+48];\n\t"
      "ld.global.f64 %7, [%15+56];\n\t"
      "ld.global.f64 %8, [%15+64];\n\t"
      "ld.global.f64 %9, [%15+72];\n\t"
      "ld.global.f64 %10, [%15+80];\n\t"
      "ld.global.f64 %11, [%15+88];\n\t"
      "ld.global.f64 %12, [%15+96];\n\t"
      "ld.global.f64 %13, [%15+104];\n\t"
      "ld.global.f64 %14, [%15+112];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]), "=d"(v[8]),
        "=d"(v[9]), "=d"(v[10]), "=d"(v[11]), "=d"(v[12]), "=d"(v[13]), "=d"(v[14])
      : "l"(p)
      : "memory");
}

// Offsets of the 7 lattice rows around node (., j, k) — rows (k + row_dk(t),
// j + row_dj(t)) — and their last i (-1 when the row is outside the macro).
__device__ __forceinline__ void node_rows(int n, int j, int k, int (&ra)[7], int (&len)[7]) {
  const int T = tsz(n);
  const int pb0 = T - tsz(n - k);                              // plane k
  const int pbp = pb0 + (n - k + 1) * (n - k + 2) / 2;         // plane k + 1
  const int pbm = pb0 - (n - k + 2) * (n - k + 3) / 2;         // plane k - 1
#pragma unroll
  for (int t = 0; t < 7; ++t) {
    const int dk = row_dk(t), kk = k + dk, jj = j + row_dj(t), m2 = n - kk;
    const int pb = dk == 0 ? pb0 : (dk > 0 ? pbp : pbm);
    const bool valid = kk >= 0 && kk <= n && jj >= 0 && jj <= m2;
    ra[t] = valid ? pb + jj * (m2 + 1) - (jj * (jj - 1)) / 2 : pb0;
    len[t] = valid ? m2 - jj : -1;
  }
}

// Lattice-boundary signature bits (sig3) that put the neighbour along
// direction d outside the macro: i = 0 and di < 0, j = 0 and dj < 0, k = 0 and
// dk < 0, i + j + k = n and di + dj + dk > 0 (compile time per direction).
__device__ __forceinline__ constexpr int dir_bad(int d) {
  constexpr int v[15] = {0, 8, 1, 1, 2, 2, 4, 8, 2, 1, 4, 10, 5, 8, 4};
  return v[d];
}
// Row starts (shared-memory plane slots) of the 7 rows around (., j) of plane
// k with m2 = n - k; base[0..2]: slot bases of planes k - 1, k, k + 1.  Rows
// outside the lattice get an address that is never loaded.
__device__ __forceinline__ void slot_rows(const int (&base)[3], int m2, int j, int (&ra)[7]) {
  const int r0 = lat2(m2, 0, j);
  ra[0] = base[1] + r0;
  ra[1] = ra[0] + (m2 + 1 - j);
  ra[2] = ra[0] - (m2 + 2 - j);
  ra[5] = base[2] + r0 - j;      // plane k + 1: lat2(m2 - 1, 0, j)
  ra[3] = ra[5] - (m2 + 1 - j);  // lat2(m2 - 1, 0, j - 1)
  ra[6] = base[0] + r0 + j;      // plane k - 1: lat2(m2 + 1, 0, j)
  ra[4] = ra[6] + (m2 + 2 - j);  // lat2(m2 + 1, 0, j + 1)
}

// partial row of a lattice-boundary node of one macro: its signature's partial
// stencil over the neighbours inside the macro, centre first.  All loads are
// issued together (clamped to the node itself when the neighbour is outside
// the macro); the sum keeps the specification's order and terms.
template <bool kOff>
__device__ __forceinline__ double partial_row(const double* __restrict__ ps_m, const double* xm, int n, int i, int j,
                                              int k) {
  const int sig = sig3(n, i, j, k);
  const double* ps = ps_m + 15 * sig;
  // row starts from the plane offsets; a neighbour is inside the macro unless the
  // node's boundary signature excludes its direction (dir_bad)
  const int m2 = n - k, pb0 = tsz(n) - tsz(m2);
  const int base[3] = {pb0 - (m2 + 2) * (m2 + 3) / 2, pb0, pb0 + (m2 + 1) * (m2 + 2) / 2};
  int ra[7];
  slot_rows(base, m2, j, ra);
  const int c0 = ra[0] + i;
  double x[15], cf[15];
  bool ok[15];
  const double* ad[15];
#pragma unroll
  for (int d = 0; d < 15; ++d) {
    ok[d] = (sig & dir_bad(d)) == 0;
    ad[d] = xm + (ok[d] ? ra[dir_row(d)] + i + dir_di(d) : c0);
  }
  // ptxas sinks plain loads to just before their use, serialising the L2 round
  // trips of the 15 terms; issued from one asm block they are all in flight
  load15(x, ad);
  load15_seq(cf, ps);
  double acc = kOff ? 0.0 : cf[0] * x[0];
#pragma unroll
  for (int d = 1; d < 15; ++d) {
    const double t = acc + cf[d] * x[d];
    acc = ok[d] ? t : acc;
  }
  return acc;
}
__device__ double partial_full(const double* __restrict__ ps_m, const double* xm, int n, int i, int j, int k) {
  return partial_row<false>(ps_m, xm, n, i, j, k);
}
// off-diagonal part (Gauss-Seidel)
__device__ double partial_off3(const double* __restrict__ ps_m, const double* xm, int n, int i, int j, int k) {
  return partial_row<true>(ps_m, xm, n, i, j, k);
}

__device__ __forceinline__ void unpack_ijk(int p, int& i, int& j, int& k) {
  i = p & 1023;
  j = (p >> 10) & 1023;
  k = (p >> 20) & 1023;
}

// k-plane streaming helpers (TMA bulk copies into shared-memory plane slots)
__device__ __forceinline__ void p3_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void p3_mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ int plane_base(int n, int k) { return tsz(n) - tsz(n - k); }
// doubles per plane slot: the largest plane (k = 0), +1 alignment pad, 16-byte multiple
__host__ __device__ __forceinline__ int plane_stride(int n) { return ((n + 1) * (n + 2) / 2 + 3) & ~1; }

// ---------------------------------------------------------------- apply / residual
// blocks [0, M (n+1)): one k-plane of one macro, lattice-interior nodes;
// remaining blocks: one shared-node group per thread.
__global__ void __launch_bounds__(kT) k3_apply(DevLevel3D lv, int mass, const double* __restrict__ x, double* y,
                                               const double* __restrict__ b, int mode, int plane_blocks) {
  const int n = lv.n, S = lv.S;
  const double* __restrict__ st_all = mass ? lv.stM : lv.stK;
  if (static_cast<int>(blockIdx.x) < plane_blocks) {
    const int m = blockIdx.x / (n + 1), k = blockIdx.x - m * (n + 1);
    const int m2 = n - k;
    if (k < 1 || m2 < 3) return;
    const double* st = st_all + 15 * m;
    double s[15];
#pragma unroll
    for (int d = 0; d < 15; ++d) s[d] = __ldg(st + d);
    const double* xm = x + static_cast<size_t>(m) * S;
    const int base = tsz(n) - tsz(n - k);
    const int np = (m2 + 1) * (m2 + 2) / 2;
    for (int q = threadIdx.x; q < np; q += blockDim.x) {
      int i, j;
      decode2(m2, q, i, j);
      if (!interior3(n, i, j, k)) continue;
      double acc = s[0] * xm[base + q];
#pragma unroll
      for (int d = 1; d < 15; ++d) acc = acc + s[d] * xm[lat3(n, i + c_dir[d][0], j + c_dir[d][1], k + c_dir[d][2])];
      const size_t off = static_cast<size_t>(m) * S + base + q;
      y[off] = mode == A3_PLAIN ? acc : b[off] - acc;
    }
    return;
  }
  const int g = (blockIdx.x - plane_blocks) * blockDim.x + threadIdx.x;
  if (g >= lv.ng) return;
  const double* K = mass ? lv.psM : lv.psK;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  double v;
  auto part = [&](int q) {
    const int s = lv.mem_slot[q];
    if (s < 0) return lv.ghost[~s];  // another shard's member (sharded levels)
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    return partial_full(K + 240 * s, x + static_cast<size_t>(s) * S, n, i, j, k);
  };
  if (end - beg == 1) {
    v = part(beg);
  } else {
    v = 0.0;
    for (int q = beg; q < end; ++q) v += part(q);
  }
  const bool dom = lv.grp_domain[g];
  for (int q = beg; q < end; ++q) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    const size_t off = static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k);
    if (mode == A3_PLAIN)
      y[off] = v;
    else if (mode == A3_RESIDUAL)
      y[off] = dom ? 0.0 : b[off] - v;
    else
      y[off] = (dom || q != beg) ? 0.0 : b[off] - v;
  }
}

// Group part of k3_apply on small levels (n < 8, where it is latency-bound):
// one warp per group, lane q evaluates member q's partial row, every lane sums
// the members in slot order from shuffles (the sequence of k3_apply), the
// lanes write their members' copies.
__global__ void __launch_bounds__(kT) k3_apply_groups_warp(DevLevel3D lv, int mass, const double* __restrict__ x,
                                                           double* y, const double* __restrict__ b, int mode) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (g >= lv.ng) return;  // warp-uniform
  const int n = lv.n, S = lv.S;
  const double* K = mass ? lv.psM : lv.psK;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  const bool dom = lv.grp_domain[g];
  double v = 0.0;
  for (int q0 = beg; q0 < end; q0 += 32) {
    const int q = q0 + lane;
    double part = 0.0;
    if (q < end) {
      const int s = lv.mem_slot[q];
      if (s < 0) {
        part = lv.ghost[~s];
      } else {
        int i, j, k;
        unpack_ijk(lv.mem_ijk[q], i, j, k);
        part = partial_full(K + 240 * s, x + static_cast<size_t>(s) * S, n, i, j, k);
      }
    }
    const int cnt = min(32, end - q0);
    if (end - beg == 1) {
      v = __shfl_sync(0xffffffffu, part, 0);
    } else {
      for (int t = 0; t < cnt; ++t) v += __shfl_sync(0xffffffffu, part, t);
    }
  }
  for (int q = beg + lane; q < end; q += 32) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    const size_t off = static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k);
    if (mode == A3_PLAIN)
      y[off] = v;
    else if (mode == A3_RESIDUAL)
      y[off] = dom ? 0.0 : b[off] - v;
    else
      y[off] = (dom || q != beg) ? 0.0 : b[off] - v;
  }
}

// Streaming form of the same operator (levels n >= 8), two kernels:
//  k3_apply_stream  one CTA per macro streams the k-planes of x through a
//                   4-slot shared-memory ring (TMA bulk copies two planes
//                   ahead) and writes, for every node of the macro, its full
//                   stencil row (lattice interior; y or b - y) or its partial
//                   row (lattice boundary copies; raw) — each x, b, y value
//                   moves once;
//  k3_apply_groups  per shared-node group: the member partial rows summed in
//                   slot order (the additive sync of k3_apply) and the mode's
//                   write to every copy.
// Same operations and orders as k3_apply / partial_row (bit-identical).
constexpr int kAsSlots = 4;
constexpr int kAsPF = 6;  // L2 prefetch distance (planes) ahead of the TMA stream

template <int kAsThreads>
__global__ void __launch_bounds__(kAsThreads) k3_apply_stream(DevLevel3D lv, int mass, const double* __restrict__ x,
                                                              double* y, const double* __restrict__ b, int mode) {
  extern __shared__ __align__(128) unsigned long long as_smem[];
  const int n = lv.n, S = lv.S, m = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int nwarps = kAsThreads / 32;
  const int stride = plane_stride(n);
  double* ps = reinterpret_cast<double*>(as_smem + kAsSlots);  // 16 signatures x 15
  double* ring = ps + 240;
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(as_smem));
  const unsigned ring_s = static_cast<unsigned>(__cvta_generic_to_shared(ring));
  const double* xm = x + static_cast<size_t>(m) * S;
  auto issue = [&](int k) {
    const size_t a = reinterpret_cast<size_t>(xm + plane_base(n, k));
    const int off = static_cast<int>((a >> 3) & 1);
    const int len = (n - k + 1) * (n - k + 2) / 2;
    const unsigned bytes = static_cast<unsigned>(((off + len) * 8 + 15) & ~15);
    const int slot = k % kAsSlots;
    const unsigned bar = bar_s + 8u * slot;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            ring_s + 8u * static_cast<unsigned>(slot * stride)),
        "l"(a - 8 * off), "r"(bytes), "r"(bar)
        : "memory");
  };
  if (tid == 0) {
    for (int t = 0; t < kAsSlots; ++t) p3_mbar_init(bar_s + 8u * t, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < 2 && k <= n; ++k) issue(k);
  }
  const double* psg = (mass ? lv.psM : lv.psK) + 240 * static_cast<size_t>(m);
  for (int t = tid; t < 240; t += kAsThreads) ps[t] = __ldg(psg + t);
  double s[15];
  {
    const double* st = (mass ? lv.stM : lv.stK) + 15 * m;
#pragma unroll
    for (int d = 0; d < 15; ++d) s[d] = __ldg(st + d);
  }
  __syncthreads();
  const size_t gm = static_cast<size_t>(m) * S;
  auto l2_prefetch = [&](const double* v, int k) {
    const int len = (n - k + 1) * (n - k + 2) / 2;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<size_t>(v + plane_base(n, k)) &
                                                                    ~size_t(15)),
                 "r"(static_cast<unsigned>((len * 8 + 31) & ~15))
                 : "memory");
  };
  if (tid == 32)
    for (int k = 2; k < 2 + kAsPF && k <= n; ++k) l2_prefetch(xm, k);
  if (tid == 64 && b)
    for (int k = 1; k < 1 + kAsPF && k <= n; ++k) l2_prefetch(b + static_cast<size_t>(m) * S, k);
  for (int k = 0; k <= n; ++k) {
    if (tid == 0 && k + 2 <= n) issue(k + 2);  // its slot held plane k - 2, done last step
    if (tid == 32 && k + 2 + kAsPF <= n) l2_prefetch(xm, k + 2 + kAsPF);
    if (tid == 64 && b && k + 1 + kAsPF <= n) l2_prefetch(b + static_cast<size_t>(m) * S, k + 1 + kAsPF);
    if (k + 1 <= n) p3_mbar_wait(bar_s + 8u * ((k + 1) % kAsSlots), ((k + 1) / kAsSlots) & 1);
    if (k == 0) p3_mbar_wait(bar_s, 0);
    const int m2 = n - k;
    int base[3];  // slot base (+ alignment offset) of planes k-1, k, k+1 (clamped to k)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int kk = min(max(k - 1 + d, 0), n);
      base[d] = (kk % kAsSlots) * stride + static_cast<int>((reinterpret_cast<size_t>(xm + plane_base(n, kk)) >> 3) & 1);
    }
    const size_t gp = gm + plane_base(n, k);
    // lattice-interior nodes, flattened in pairs (i, i + 1) of a row: the
    // plane's interior is the triangle lattice of size mi = m2 - 3 shifted by
    // (1, 1); rows 2c and 2c + 1 hold mi + 1 - 2c pairs together.  The two
    // nodes share their row starts and most neighbour loads (the compiler
    // merges the equal shared-memory addresses); each keeps the full
    // stencil's term order.
    int npairs = 0;
    if (k >= 1 && m2 >= 3) {
      const int mi = m2 - 3, nc = (mi + 2) / 2;  // row couples
      npairs = nc * (mi + 1) - nc * (nc - 1);
      const float A = static_cast<float>(mi + 2);
      for (int e = tid; e < npairs; e += kAsThreads) {
        // couple c: pairs before it = c (mi + 1) - c (c - 1) = c (mi + 2 - c)
        int c = static_cast<int>((A - sqrtf(fmaxf(A * A - 4.0f * e, 0.0f))) * 0.5f);
        c = c + (c + 1 <= nc - 1 && (c + 1) * (mi + 1 - c) <= e);
        c = c - (c > 0 && c * (mi + 2 - c) > e);
        const int e1 = e - c * (mi + 2 - c);
        const int L0 = mi + 1 - 2 * c, P0 = (L0 + 1) >> 1;  // first row of the couple: L0 nodes, P0 pairs
        const int r = e1 < P0 ? 2 * c : 2 * c + 1;
        const int p = e1 < P0 ? e1 : e1 - P0;
        const int L = mi + 1 - r;
        const int j = r + 1, i = 1 + 2 * p;
        const bool two = 2 * p + 1 < L;
        int ra[7];
        slot_rows(base, m2, j, ra);
        const size_t off = gp + (ra[0] - base[1]) + i;
        const double bv0 = mode == A3_PLAIN ? 0.0 : __ldg(b + off);
        const double bv1 = mode == A3_PLAIN || !two ? 0.0 : __ldg(b + off + 1);
        double acc0 = s[0] * ring[ra[0] + i];
        double acc1 = s[0] * ring[ra[0] + i + 1];
#pragma unroll
        for (int d = 1; d < 15; ++d) {
          acc0 = acc0 + s[d] * ring[ra[dir_row(d)] + i + dir_di(d)];
          acc1 = acc1 + s[d] * ring[ra[dir_row(d)] + i + 1 + dir_di(d)];
        }
        y[off] = mode == A3_PLAIN ? acc0 : bv0 - acc0;
        if (two) y[off + 1] = mode == A3_PLAIN ? acc1 : bv1 - acc1;
      }
    }
    // lattice-boundary nodes of the plane: partial rows (raw)
    const int nb = k == 0 ? (m2 + 1) * (m2 + 2) / 2 : (m2 >= 1 ? 3 * m2 : 1);
    // boundary nodes continue the interior's thread rotation (balanced per plane)
    for (int e = (tid - npairs % kAsThreads + kAsThreads) % kAsThreads; e < nb; e += kAsThreads) {
      int i, j;
      if (k == 0) {
        decode2(m2, e, i, j);
      } else if (m2 == 0) {
        i = 0, j = 0;
      } else if (e < m2 + 1) {  // row j = 0
        i = e, j = 0;
      } else if (e < 2 * m2) {  // i = 0, j = 1 .. m2 - 1
        i = 0, j = e - m2;
      } else {                  // i = m2 - j, j = 1 .. m2
        j = e - 2 * m2 + 1, i = m2 - j;
      }
      const int sig = sig3(n, i, j, k);
      const double* cf = ps + 15 * sig;
      int ra[7];
      slot_rows(base, m2, j, ra);
      const int c0 = ra[0] + i;
      double acc = cf[0] * ring[c0];
#pragma unroll
      for (int d = 1; d < 15; ++d) {
        const bool ok = (sig & dir_bad(d)) == 0;
        const double t = acc + cf[d] * ring[ok ? ra[dir_row(d)] + i + dir_di(d) : c0];
        acc = ok ? t : acc;
      }
      y[gp + lat2(m2, 0, j) + i] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kT) k3_apply_groups(DevLevel3D lv, double* y, const double* __restrict__ b,
                                                      int mode) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= lv.ng) return;
  const int n = lv.n, S = lv.S;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  auto copy = [&](int q) {
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    return static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k);
  };
  double v;
  if (end - beg == 1) {
    v = y[copy(beg)];
  } else {
    v = 0.0;
    for (int q = beg; q < end; ++q) {
      const int s = lv.mem_slot[q];
      v += s < 0 ? lv.ghost[~s] : y[copy(q)];
    }
  }
  const bool dom = lv.grp_domain[g];
  for (int q = beg; q < end; ++q) {
    if (lv.mem_slot[q] < 0) continue;
    const size_t off = copy(q);
    if (mode == A3_PLAIN)
      y[off] = v;
    else if (mode == A3_RESIDUAL)
      y[off] = dom ? 0.0 : b[off] - v;
    else
      y[off] = (dom || q != beg) ? 0.0 : b[off] - v;
  }
}

// ---------------------------------------------------------------- Gauss-Seidel
// relaxation of one shared-node group (all copies get the same value)
__device__ __forceinline__ void stamp(long long* tr, int slot) {
  if (tr) tr[slot] = clock64();
}
__device__ void gs_group(const DevLevel3D& lv, double* u, const double* __restrict__ b, int g,
                         long long* tr = nullptr) {
  const int n = lv.n, S = lv.S;
  stamp(tr, 0);
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  int ql = beg;  // first member on this shard: b's copies are interface-consistent
  while (lv.mem_slot[ql] < 0) ++ql;
  int i0, j0, k0;
  unpack_ijk(lv.mem_ijk[ql], i0, j0, k0);
  const size_t own = static_cast<size_t>(lv.mem_slot[ql]) * S + lat3(n, i0, j0, k0);
  double val;
  if (lv.grp_domain[g]) {
    val = b[own];
  } else {
    double off = 0.0;
    for (int q = beg; q < end; ++q) {
      const int s = lv.mem_slot[q];
      if (s < 0) {
        off = off + lv.ghost[~s];
        continue;
      }
      int i, j, k;
      unpack_ijk(lv.mem_ijk[q], i, j, k);
      stamp(tr, 1 + 2 * (q - beg));
      off = off + partial_off3(lv.psK + 240 * s, u + static_cast<size_t>(s) * S, n, i, j, k);
      if (tr) tr[2 + 2 * (q - beg)] = clock64() + (off == 12345.0 ? 1 : 0);
    }
    val = (b[own] - off) / lv.grp_diag[g];
  }
  if (tr) tr[8] = clock64() + (val == 12345.0 ? 1 : 0);
  for (int q = beg; q < end; ++q) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    u[static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k)] = val;
  }
  stamp(tr, 9);
}

// Relaxation of a narrow group (<= 4 members) by W lanes (W = 4 on small
// levels, where the colour phases are latency-bound; W = 2 on large levels,
// where most narrow groups are 2-member face groups): lane q of the W
// evaluates the partial rows of members q and q + W, every lane forms the
// member sum in slot order from shuffles (the sequential order of gs_group),
// the lanes write their own members' copies.  All 32 lanes of the warp call it
// (valid = false for lane groups without a group).
template <int W>
__device__ __forceinline__ void gs_group_lanes(const DevLevel3D& lv, double* u, const double* __restrict__ b, int t,
                                               bool valid, int sub) {
  constexpr int R = 4 / W;  // members per lane
  const int n = lv.n, S = lv.S;
  int cnt = 0, slot[R], i[R], j[R], k[R];
  double part[R], diag = 1.0;
  bool dom = false;
  // One round trip for the group's data: its flat record (header: diagonal,
  // member count, domain flag; four member slots of (macro slot, i j k)) at
  // the group's position in the colour list; without records (shard tables)
  // the chain colour list -> group -> member tables.
  if (lv.nar_hdr) {
    int4 hd = make_int4(0, 0, 0, 0);
    if (valid) hd = __ldg(lv.nar_hdr + t);
    cnt = hd.z & 0xffff;
    dom = (hd.z >> 16) != 0;
    diag = __hiloint2double(hd.y, hd.x);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = sub + W * r;
      int2 mm = make_int2(-1, 0);
      if (valid && q < cnt) mm = __ldg(lv.nar_mem + 4 * static_cast<size_t>(t) + q);
      slot[r] = q < cnt ? mm.x : -1;
      unpack_ijk(mm.y, i[r], j[r], k[r]);
    }
  } else {
    int beg = 0;
    if (valid) {
      const int g = lv.color_grp[t];
      beg = lv.grp_ptr[g];
      cnt = lv.grp_ptr[g + 1] - beg;
      dom = lv.grp_domain[g];
      diag = lv.grp_diag[g];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = sub + W * r;
      slot[r] = -1;
      i[r] = j[r] = k[r] = 0;
      if (valid && q < cnt) {
        slot[r] = lv.mem_slot[beg + q];
        if (slot[r] >= 0) unpack_ijk(lv.mem_ijk[beg + q], i[r], j[r], k[r]);
      }
    }
  }
  const int qbase = (threadIdx.x & 31) & ~(W - 1);
  // the first member on this shard holds b (b's copies are interface-consistent);
  // its load goes out before the partial rows
  unsigned mine = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) mine |= (valid && sub + W * r < cnt && slot[r] >= 0) ? 1u << r : 0u;
  int first = 4;
#pragma unroll
  for (int r = R - 1; r >= 0; --r) {
    const unsigned here = __ballot_sync(0xffffffffu, (mine >> r) & 1u);
    const unsigned bits = (here >> qbase) & ((1u << W) - 1u);
    if (bits) first = min(first, W * r + __ffs(bits) - 1);
  }
  double bown = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (valid && sub + W * r == first) bown = __ldg(b + static_cast<size_t>(slot[r]) * S + lat3(n, i[r], j[r], k[r]));
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int q = sub + W * r;
    part[r] = 0.0;
    if (valid && q < cnt) {
      if (slot[r] < 0)
        part[r] = lv.ghost[~slot[r]];
      else if (!dom)
        part[r] = partial_off3(lv.psK + 240 * slot[r], u + static_cast<size_t>(slot[r]) * S, n, i[r], j[r], k[r]);
    }
  }
  double off = 0.0;
#pragma unroll
  for (int t4 = 0; t4 < 4; ++t4) {
    const double v = __shfl_sync(0xffffffffu, part[t4 / W], qbase + t4 % W);
    if (t4 < cnt) off = off + v;
  }
  const double bq = __shfl_sync(0xffffffffu, bown, qbase + (first < 4 ? first % W : 0));
  if (!valid) return;
  const double val = dom ? bq : (bq - off) / diag;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (sub + W * r < cnt && slot[r] >= 0) u[static_cast<size_t>(slot[r]) * S + lat3(n, i[r], j[r], k[r])] = val;
}

// boundary phase of colour c: one group per thread
__global__ void __launch_bounds__(kT) k3_gs_groups(DevLevel3D lv, double* u, const double* __restrict__ b, int c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int p0 = lv.color_grp_ptr[c], p1 = lv.color_grp_ptr[c + 1];
  if (p0 + t >= p1) return;
  gs_group(lv, u, b, lv.color_grp[p0 + t]);
}

// Interior relaxation (the specification's order, oracle o3_gauss_seidel):
// every macro plane by plane (k ascending), inside a plane the four (i, j)
// parity classes q = 0..3 — i = 1 + (q & 1) + 2 a, j = 1 + (q >> 1) + 2 r —
// one after the other; nodes of a class are never stencil neighbours.  The row
// is two fused chains (directions 1..7 and 8..14) added last.
__device__ __forceinline__ double gs_row_fma(const double (&s)[15], const double (&x)[15]) {
  double a0 = s[1] * x[1], a1 = s[8] * x[8];
#pragma unroll
  for (int d = 2; d < 8; ++d) a0 = __fma_rn(s[d], x[d], a0);
#pragma unroll
  for (int d = 9; d < 15; ++d) a1 = __fma_rn(s[d], x[d], a1);
  return a0 + a1;
}
// Neighbour offsets of lattice-interior node c = lat2(m2, i, j) of plane k
// (m2 = n - k) relative to the starts of planes k - 1, k, k + 1: with
// rs = c - i the row start, the pairs (d: offset) are
//   plane k     1: c+1  2: c-1  3: c+m2-j  7: c+m2-j+1  8: c-(m2+2-j)  4: c-(m2+2-j)+1
//   plane k+1   5: c-m2-1  11: c-m2  9: c-j-1  13: c-j       (lat2(m2 - 1, ., .))
//   plane k-1  14: c+j  10: c+j+1  12: c+m2+1  6: c+m2+2      (lat2(m2 + 1, ., .))
template <typename Ld>
__device__ __forceinline__ void gs_gather(double (&x)[15], Ld ld, int bm, int b0, int bp, int c, int j, int m2) {
  const int e0 = b0 + c, e1 = e0 + (m2 - j), e2 = e0 - (m2 + 2 - j);
  const int p0 = bp + c - m2 - 1, p1 = bp + c - j - 1, q0 = bm + c + j, q1 = bm + c + m2 + 1;
  x[1] = ld(e0 + 1), x[2] = ld(e0 - 1), x[3] = ld(e1), x[4] = ld(e2 + 1), x[5] = ld(p0), x[6] = ld(q1 + 1);
  x[7] = ld(e1 + 1), x[8] = ld(e2), x[9] = ld(p1), x[10] = ld(q0 + 1), x[11] = ld(p0 + 1), x[12] = ld(q1);
  x[13] = ld(p1 + 1), x[14] = ld(q0);
}

// Small levels (n <= 16, inside the cooperative smoother): the CTA's macros
// (every active-th one) together, step by step (plane k, class q) with block
// barriers; the items of a step are (macro, node) from the level's step lists.
__device__ void gs_interior_batch(const DevLevel3D& lv, double* u, const double* __restrict__ b, int active,
                                  int group) {
  const int n = lv.n, S = lv.S, T = tsz(n), per = lv.pat_max, steps = 4 * (n - 3);
  const int mine = (lv.M - static_cast<int>(blockIdx.x) + active - 1) / active;  // macros of this CTA
  for (int g0 = 0; g0 < mine; g0 += group)
    for (int st = 0; st < steps; ++st) {
      const int nm = min(group, mine - g0);
      const int q0 = __ldg(lv.pat_ptr + st), cnt = __ldg(lv.pat_ptr + st + 1) - q0;
      for (int t = threadIdx.x; t < nm * per; t += blockDim.x) {
        const int mi = t / per, idx = t - mi * per;
        if (idx >= cnt) continue;
        const int m = blockIdx.x + (g0 + mi) * active;
        const int ent = __ldg(lv.pat_node + q0 + idx), c = ent & 0xffff, j = ent >> 16, k = (st >> 2) + 1;
        const int m2 = n - k, pb0 = T - tsz(m2);
        double* um = u + static_cast<size_t>(m) * S;
        double sc[15], x[15];
#pragma unroll
        for (int d = 1; d < 15; ++d) sc[d] = __ldg(lv.stK + 15 * m + d);
        gs_gather(x, [&](int o) { return um[o]; }, pb0 - (m2 + 2) * (m2 + 3) / 2, pb0, pb0 + (m2 + 1) * (m2 + 2) / 2, c,
                  j, m2);
        um[pb0 + c] = (__ldg(b + static_cast<size_t>(m) * S + pb0 + c) - gs_row_fma(sc, x)) * __ldg(lv.inv_c + m);
      }
      __syncthreads();
    }
}

// Relaxation of a group with many members (macro vertices, edges): one warp,
// a lane per member partial row, the member sum in slot order by shuffles.
__device__ void gs_group_warp(const DevLevel3D& lv, double* u, const double* __restrict__ b, int t, int lane) {
  const int n = lv.n, S = lv.S;
  if (lv.nar_hdr) {
    // flat record: header at the colour-list position, members contiguous from hd.w
    const int4 hd = __ldg(lv.nar_hdr + t);
    const int cnt = hd.z & 0xffff;
    const bool dom = (hd.z >> 16) != 0;
    const int2* mem = lv.wide_mem + hd.w;
    double off = 0.0, bown = 0.0;
    int2 first = make_int2(0, 0);
    for (int q0 = 0; q0 < cnt; q0 += 32) {
      double part = 0.0;
      int2 mm = make_int2(0, 0);
      if (q0 + lane < cnt) {
        mm = __ldg(mem + q0 + lane);
        int i, j, k;
        unpack_ijk(mm.y, i, j, k);
        if (q0 + lane == 0) bown = __ldg(b + static_cast<size_t>(mm.x) * S + lat3(n, i, j, k));
        if (!dom) part = partial_off3(lv.psK + 240 * mm.x, u + static_cast<size_t>(mm.x) * S, n, i, j, k);
      }
      if (q0 == 0) first = mm;
      const int c32 = min(32, cnt - q0);
      if (!dom)
        for (int q = 0; q < c32; ++q) off = off + __shfl_sync(0xffffffffu, part, q);
    }
    bown = __shfl_sync(0xffffffffu, bown, 0);
    const double val = dom ? bown : (bown - off) / __hiloint2double(hd.y, hd.x);
    for (int q = lane; q < cnt; q += 32) {
      const int2 mm = q < 32 ? first : __ldg(mem + q);
      int i, j, k;
      unpack_ijk(mm.y, i, j, k);
      u[static_cast<size_t>(mm.x) * S + lat3(n, i, j, k)] = val;
    }
    return;
  }
  const int g = lv.color_grp[t];
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  int ql = beg;
  while (lv.mem_slot[ql] < 0) ++ql;
  int i0, j0, k0;
  unpack_ijk(lv.mem_ijk[ql], i0, j0, k0);
  const size_t own = static_cast<size_t>(lv.mem_slot[ql]) * S + lat3(n, i0, j0, k0);
  double val;
  if (lv.grp_domain[g]) {
    val = b[own];
  } else {
    double off = 0.0;
    for (int q0 = beg; q0 < end; q0 += 32) {
      double part = 0.0;
      const int q = q0 + lane;
      if (q < end) {
        const int s = lv.mem_slot[q];
        if (s < 0) {
          part = lv.ghost[~s];
        } else {
          int i, j, k;
          unpack_ijk(lv.mem_ijk[q], i, j, k);
          part = partial_off3(lv.psK + 240 * s, u + static_cast<size_t>(s) * S, n, i, j, k);
        }
      }
      const int cnt = min(32, end - q0);
      for (int t = 0; t < cnt; ++t) off = off + __shfl_sync(0xffffffffu, part, t);
    }
    val = (b[own] - off) / lv.grp_diag[g];
  }
  for (int q = beg + lane; q < end; q += 32) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    u[static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k)] = val;
  }
}

// Whole smoother (sweeps x [boundary colours, interior]) in one cooperative
// launch: grid barriers between the boundary colours and between the phases.
// Per colour the group list holds the wide groups (warp each) first, then the
// narrow ones (thread each).  The interior phase runs at most `active` CTAs
// (one macro each at a time) so that the macros being smoothed stay in L2
// across their colours.
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k3_gs_sweeps(DevLevel3D lv, double* u, const double* __restrict__ b,
                                                         int sweeps, int phases, int active, int group) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nthreads = gridDim.x * NT;
  const int tid = blockIdx.x * NT + threadIdx.x;
  const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nthreads >> 5;
#ifdef KB_GS_TRACE
  if ((phases & 4) && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_gs3_trace[63]));
#endif
  // colour ranges once (not a dependent load at the head of every phase)
  __shared__ int s_cptr[65], s_cwide[64];
  for (int c = threadIdx.x; c <= lv.colors && c <= 64; c += NT) {
    s_cptr[c] = lv.color_grp_ptr[c];
    if (c < lv.colors) s_cwide[c] = lv.color_wide_end[c];
  }
  __syncthreads();
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int c = 0; c < lv.colors; ++c) {
      const bool cached = lv.colors <= 64;
      const int p0 = cached ? s_cptr[c] : lv.color_grp_ptr[c], p1 = cached ? s_cptr[c + 1] : lv.color_grp_ptr[c + 1],
                pw = cached ? s_cwide[c] : lv.color_wide_end[c];
      if (phases & 1) {
        for (int t = p0 + gw; t < pw; t += nw) gs_group_warp(lv, u, b, t, lane);
#ifdef KB_GS_TRACE
        if (phases & 8) {  // measurement trace: one thread per group
          for (int t = pw + tid; t < p1; t += nthreads)
            gs_group(lv, u, b, lv.color_grp[t],
                     tid == 0 && sw == 0 ? reinterpret_cast<long long*>(g_gs3_trace + 16 + 10 * c) : nullptr);
        } else
#endif
        {
          if (lv.n <= 8) {  // four lanes per narrow group up to n = 8, two from n = 16 (0.354 -> 0.335 ms there)
            for (int t0 = pw + 8 * gw; t0 < p1; t0 += 8 * nw) {
              const int t = t0 + (lane >> 2);
              gs_group_lanes<4>(lv, u, b, t, t < p1, lane & 3);
            }
          } else {
            for (int t0 = pw + 16 * gw; t0 < p1; t0 += 16 * nw) {
              const int t = t0 + (lane >> 1);
              gs_group_lanes<2>(lv, u, b, t, t < p1, lane & 1);
            }
          }
        }
      }
#ifdef KB_GS_TRACE
      if (phases & 4) {  // measurement trace (KB_GS3_PHASES bit 2): work end vs barrier exit
        __syncthreads();
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (sw == 0 && threadIdx.x == 0) atomicMax(&g_gs3_trace[2 * c], t);
      }
#endif
      if (p1 > p0) grid.sync();
#ifdef KB_GS_TRACE
      if ((phases & 4) && threadIdx.x == 0 && blockIdx.x == 0 && sw == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_gs3_trace[2 * c + 1] = t;
      }
#endif
    }
    if (lv.n >= 4 && lv.n <= 16) {
      if ((phases & 2) && static_cast<int>(blockIdx.x) < active) {
        gs_interior_batch(lv, u, b, active, group);  // levels with step lists (the host launches k3_gs_planes otherwise)
      }
      if (sw + 1 < sweeps) grid.sync();
    }
  }
#ifdef KB_GS_TRACE
  if (phases & 4) {
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int c = 0; c < lv.colors; ++c)
        printf("colour %d: groups %d wide %d, last work done %llu ns, barrier passed (blk0) %llu ns\n", c,
               lv.color_grp_ptr[c + 1] - lv.color_grp_ptr[c], lv.color_wide_end[c] - lv.color_grp_ptr[c],
               g_gs3_trace[2 * c] - g_gs3_trace[63], g_gs3_trace[2 * c + 1] - g_gs3_trace[63]);
    if ((phases & 8) && blockIdx.x == 0 && threadIdx.x == 0)
      for (int c = 0; c < 4; ++c) {
        const unsigned long long* t = g_gs3_trace + 16 + 10 * c;
        printf("colour %d first narrow group (cycles from start): meta %llu  m0 %llu..%llu  m1 %llu..%llu  div %llu  "
               "store %llu\n",
               c, t[1] - t[0], t[1] - t[0], t[2] - t[0], t[3] - t[0], t[4] - t[0], t[8] - t[0], t[9] - t[0]);
      }
  }
#endif
}

// Interior phase as a k-plane stream (4 <= n <= 64): one CTA per macro keeps
// planes k - 1, k, k + 1 of u and plane k of b in shared memory (TMA bulk
// copies: u two planes ahead in a 4-slot ring, b one plane ahead in a 2-slot
// ring), relaxes the four parity classes of plane k with a block barrier after
// each and writes every new value to the ring and to global memory; u and b are
// read once and u written once per sweep.  The nodes of a step come from the
// level's step lists (entry = in-plane index | j << 16), one per thread.
template <int NT, int US, int BS>
__global__ void __launch_bounds__(NT, 1024 / NT) k3_gs_planes(DevLevel3D lv, double* u, const double* __restrict__ b) {
  // US u slots (plane k in slot k % US, US - 2 planes ahead), BS b slots (plane
  // k in slot (k - 1) % BS, BS - 1 planes ahead); one mbarrier per slot
  extern __shared__ __align__(128) unsigned long long gp_smem[];
  constexpr int PF = 6;  // L2 prefetch distance beyond the TMA stream (planes)
  const int n = lv.n, S = lv.S, m = blockIdx.x, tid = threadIdx.x;
  const int stride = plane_stride(n);
  const int steps = 4 * (n - 3);
  int* sp = reinterpret_cast<int*>(gp_smem + US + BS);  // step starts (steps + 1, padded to 16 bytes)
  double* ring_u = reinterpret_cast<double*>(gp_smem + US + BS) + ((steps + 4) >> 2 << 1);
  double* ring_b = ring_u + US * stride;
  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(gp_smem));
  const unsigned ringu_s = static_cast<unsigned>(__cvta_generic_to_shared(ring_u));
  const unsigned ringb_s = static_cast<unsigned>(__cvta_generic_to_shared(ring_b));
  double* um = u + static_cast<size_t>(m) * S;
  const double* bm = b + static_cast<size_t>(m) * S;
  auto issue = [&](const double* src, int k, unsigned dst_s, unsigned bar) {
    const size_t a = reinterpret_cast<size_t>(src + plane_base(n, k));
    const int off = static_cast<int>((a >> 3) & 1);
    const int len = (n - k + 1) * (n - k + 2) / 2;
    const unsigned bytes = static_cast<unsigned>(((off + len) * 8 + 15) & ~15);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_s),
                 "l"(a - 8 * off), "r"(bytes), "r"(bar)
                 : "memory");
  };
  auto issue_u = [&](int k) {
    if (k <= n - 2) issue(um, k, ringu_s + 8u * static_cast<unsigned>((k % US) * stride), bar_s + 8u * (k % US));
  };
  auto issue_b = [&](int k) {
    if (k <= n - 3)
      issue(bm, k, ringb_s + 8u * static_cast<unsigned>(((k - 1) % BS) * stride), bar_s + 8u * (US + (k - 1) % BS));
  };
  auto l2_prefetch = [&](const double* v, int k) {
    if (k > n - 2) return;
    const int len = (n - k + 1) * (n - k + 2) / 2;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<size_t>(v + plane_base(n, k)) &
                                                                    ~size_t(15)),
                 "r"(static_cast<unsigned>((len * 8 + 31) & ~15))
                 : "memory");
  };
  auto align_u = [&](int k) { return static_cast<int>((reinterpret_cast<size_t>(um + plane_base(n, k)) >> 3) & 1); };
  if (tid == 0) {
    for (int t = 0; t < US + BS; ++t) p3_mbar_init(bar_s + 8u * t, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k <= US - 2; ++k) issue_u(k);
    for (int k = 1; k <= BS - 1; ++k) issue_b(k);
  }
  if (tid == 0) {
    for (int k = US - 1; k < US - 1 + PF; ++k) l2_prefetch(um, k);
    for (int k = BS; k < BS + PF; ++k) l2_prefetch(bm, k);
  }
  double s[15];
#pragma unroll
  for (int d = 1; d < 15; ++d) s[d] = __ldg(lv.stK + 15 * m + d);
  s[0] = 0.0;
  const double inv_c = __ldg(lv.inv_c + m);
  for (int t = tid; t <= steps; t += NT) sp[t] = __ldg(lv.pat_ptr + t);
  __syncthreads();
  // step starts in a rolling register window w0..w4 = sp[st .. st + 4]; this
  // thread's entries of the next three steps are loaded ahead (L2 latency)
  auto spc = [&](int t) { return sp[min(t, steps)]; };
  int w0 = spc(0), w1 = spc(1), w2 = spc(2), w3 = spc(3), w4 = spc(4);
  auto entry = [&](int lo, int hi) { return tid < hi - lo ? __ldg(lv.pat_node + lo + tid) : 0; };
  int e1 = entry(w0, w1), e2 = entry(w1, w2), e3 = entry(w2, w3);
  const int warp = tid >> 5;
  for (int k = 1; k <= n - 3; ++k) {
    // The steps shrink with k: a warp beyond the plane's largest step has no
    // node left in this or any later plane and leaves; the others meet at a
    // named barrier sized for the warps that remain.
    int need;
    {
      const int st = 4 * (k - 1);
      const int big = max(max(w1 - w0, w2 - w1), max(w3 - w2, w4 - w3));
      need = min(NT / 32, (big + 31) >> 5);
      (void)st;
    }
    if (warp >= need) break;
    if (tid == 0) {
      issue_u(k + US - 2);  // its slot held plane k - 2
      issue_b(k + BS - 1);  // its slot held plane k - 1
      l2_prefetch(um, k + US - 2 + PF);
      l2_prefetch(bm, k + BS - 1 + PF);
    }
    if (k == 1) {
      p3_mbar_wait(bar_s, 0);
      p3_mbar_wait(bar_s + 8u, 0);
    }
    p3_mbar_wait(bar_s + 8u * ((k + 1) % US), ((k + 1) / US) & 1);
    p3_mbar_wait(bar_s + 8u * (US + (k - 1) % BS), ((k - 1) / BS) & 1);
    const int m2 = n - k;
    const int bm1 = ((k - 1) % US) * stride + align_u(k - 1), b0 = (k % US) * stride + align_u(k),
              bp1 = ((k + 1) % US) * stride + align_u(k + 1);
    const int gp = plane_base(n, k);
    const double* bk =
        ring_b + ((k - 1) % BS) * stride + static_cast<int>((reinterpret_cast<size_t>(bm + gp) >> 3) & 1);
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      const int st = 4 * (k - 1) + q, p0 = w0, cnt = w1 - w0;
      int ent = e1;
      e1 = e2, e2 = e3, e3 = entry(w3, w4);
      w0 = w1, w1 = w2, w2 = w3, w3 = w4, w4 = spc(st + 5);
      for (int e = tid; e < cnt; e += NT) {
        if (e != tid) ent = __ldg(lv.pat_node + p0 + e);
        const int c = ent & 0xffff, j = ent >> 16;
        double x[15];
        gs_gather(x, [&](int o) { return ring_u[o]; }, bm1, b0, bp1, c, j, m2);
        const double v = (bk[c] - gs_row_fma(s, x)) * inv_c;
        ring_u[b0 + c] = v;
        um[gp + c] = v;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * need) : "memory");
    }
  }
}
// The same order straight on global memory (n > 64): one CTA per macro, rows
// to warps, block barriers between the classes.
__global__ void __launch_bounds__(kT) k3_gs_planes_global(DevLevel3D lv, double* u, const double* __restrict__ b) {
  const int n = lv.n, S = lv.S, m = blockIdx.x, T = tsz(n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  double* um = u + static_cast<size_t>(m) * S;
  const double* bm = b + static_cast<size_t>(m) * S;
  double s[15];
#pragma unroll
  for (int d = 1; d < 15; ++d) s[d] = __ldg(lv.stK + 15 * m + d);
  s[0] = 0.0;
  const double inv_c = __ldg(lv.inv_c + m);
  for (int k = 1; k <= n - 3; ++k) {
    const int m2 = n - k, pb0 = T - tsz(m2);
    const int pbm = pb0 - (m2 + 2) * (m2 + 3) / 2, pbp = pb0 + (m2 + 1) * (m2 + 2) / 2;
    for (int q = 0; q < 4; ++q) {
      for (int j = 1 + (q >> 1) + 2 * warp; j <= n - 2 - k; j += 2 * nwarps)
        for (int i = 1 + (q & 1) + 2 * lane; i + j + k <= n - 1; i += 64) {
          const int c = lat2(m2, i, j);
          double x[15];
          gs_gather(x, [&](int o) { return um[o]; }, pbm, pb0, pbp, c, j, m2);
          um[pb0 + c] = (__ldg(bm + pb0 + c) - gs_row_fma(s, x)) * inv_c;
        }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- transfers
// Fine node (i, j, k) of parity pattern p = (i&1, j&1, k&1) != 0 lies on the
// coarse edge along the Freudenthal direction D(p) (the c_pdir table:
// (1,0,0) (0,1,0) (-1,1,0) (0,0,1) (-1,0,1) (0,-1,1) (1,-1,1) for p = 1..7):
// di = pi ? (pj ^ pk ? -1 : 1) : 0, dj = pj ? (pk ? -1 : 1) : 0, dk = pk.
__global__ void __launch_bounds__(kT) k3_prolong(DevLevel3D cv, DevLevel3D fv, const double* __restrict__ c, double* f,
                                                 int mode) {
  const int nf = fv.n, nc = cv.n;
  const int m = blockIdx.x / (nf + 1), k = blockIdx.x - m * (nf + 1);
  const int m2 = nf - k;
  const int np = (m2 + 1) * (m2 + 2) / 2;
  const int base = tsz(nf) - tsz(nf - k);
  const double* cm = c + static_cast<size_t>(m) * cv.S;
  const int pk = k & 1;
  // coarse planes (k - dk) / 2 and (k + dk) / 2: starts and sizes
  const int ka = (k - pk) >> 1, kb = (k + pk) >> 1;
  const int ca = tsz(nc) - tsz(nc - ka), cb = tsz(nc) - tsz(nc - kb);
  const int ma = nc - ka, mb = nc - kb;
  double* fm = f + static_cast<size_t>(m) * fv.S + base;
  for (int q = threadIdx.x; q < np; q += blockDim.x) {
    int i, j;
    decode2_fast(m2, q, i, j);
    const int pi = i & 1, pj = j & 1;
    double v;
    if ((pi | pj | pk) == 0) {
      v = cm[ca + lat2(ma, i >> 1, j >> 1)];
    } else {
      const int di = pi ? ((pj ^ pk) ? -1 : 1) : 0, dj = pj ? (pk ? -1 : 1) : 0;
      v = 0.5 * (cm[ca + lat2(ma, (i - di) >> 1, (j - dj) >> 1)] + cm[cb + lat2(mb, (i + di) >> 1, (j + dj) >> 1)]);
    }
    fm[q] = mode == P3_ADD ? fm[q] + v : v;
  }
}

// restriction (transpose of k3_prolong): coarse node (i, j, k) gathers the fine
// value at (2i, 2j, 2k) and half of each fine neighbour along the 14
// directions, in direction order (the oracle's order)
__global__ void __launch_bounds__(kT) k3_restrict(DevLevel3D fv, DevLevel3D cv, const double* __restrict__ rf,
                                                  double* rc, double* zero_out) {
  const int nf = fv.n, nc = cv.n;
  const int m = blockIdx.x / (nc + 1), k = blockIdx.x - m * (nc + 1);
  const int m2 = nc - k;
  const int np = (m2 + 1) * (m2 + 2) / 2;
  const int base = tsz(nc) - tsz(nc - k);
  const double* fm = rf + static_cast<size_t>(m) * fv.S;
  const int kf = 2 * k, T = tsz(nf);
  // fine planes kf - 1, kf, kf + 1 (sizes mf + 1, mf, mf - 1)
  const int mf = nf - kf;
  const int p0 = T - tsz(nf - kf);
  const int pp = p0 + (mf + 1) * (mf + 2) / 2, pm = kf > 0 ? p0 - (mf + 2) * (mf + 3) / 2 : 0;
  for (int q = threadIdx.x; q < np; q += blockDim.x) {
    int i, j;
    decode2_fast(m2, q, i, j);
    const int fi = 2 * i, fj = 2 * j;
    // row starts of the 7 fine rows around (fj, kf)
    const int r0 = lat2(mf, 0, fj);
    int ra[7], len[7];
    ra[0] = p0 + r0, len[0] = mf - fj;
    ra[1] = ra[0] + (mf + 1 - fj), len[1] = mf - fj - 1;                         // (kf, fj + 1)
    ra[2] = ra[0] - (mf + 2 - fj), len[2] = fj >= 1 ? mf - fj + 1 : -1;          // (kf, fj - 1)
    const bool up = kf + 1 <= nf, dn = kf >= 1;
    ra[5] = pp + r0 - fj, len[5] = up ? mf - 1 - fj : -1;                        // (kf + 1, fj)
    ra[3] = ra[5] - (mf + 1 - fj), len[3] = up && fj >= 1 ? mf - fj : -1;       // (kf + 1, fj - 1)
    ra[6] = pm + r0 + fj, len[6] = dn ? mf + 1 - fj : -1;                        // (kf - 1, fj)
    ra[4] = ra[6] + (mf + 2 - fj), len[4] = dn ? mf - fj : -1;                  // (kf - 1, fj + 1)
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < 15; ++d) {
      const int r = dir_row(d), ii = fi + dir_di(d);
      if (ii < 0 || ii > len[r]) continue;
      const double v = fm[ra[r] + ii];
      acc = acc + (d == 0 ? v : 0.5 * v);
    }
    rc[static_cast<size_t>(m) * cv.S + base + q] = acc;
    if (zero_out) zero_out[static_cast<size_t>(m) * cv.S + base + q] = 0.0;  // the coarse zero initial guess
  }
}

// shared-node groups: additive / replace sync, optional zero of domain copies
__global__ void __launch_bounds__(kT) k3_sync(DevLevel3D lv, double* f, int additive, int zero_domain) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= lv.ng) return;
  const int n = lv.n, S = lv.S;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  auto off_of = [&](int q) {
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    return static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k);
  };
  auto val_of = [&](int q) { return lv.mem_slot[q] < 0 ? lv.ghost[~lv.mem_slot[q]] : f[off_of(q)]; };
  if (zero_domain && lv.grp_domain[g]) {
    for (int q = beg; q < end; ++q)
      if (lv.mem_slot[q] >= 0) f[off_of(q)] = 0.0;
    return;
  }
  if (end - beg < 2) return;
  double v;
  if (additive) {
    v = 0.0;
    for (int q = beg; q < end; ++q) v += val_of(q);
  } else {
    v = val_of(beg);
  }
  for (int q = beg; q < end; ++q)
    if (lv.mem_slot[q] >= 0) f[off_of(q)] = v;
}

// k3_sync on small levels (n < 8, latency-bound): one warp per group, the
// member loads in parallel, the slot-order sum from shuffles (same sequence)
__global__ void __launch_bounds__(kT) k3_sync_warp(DevLevel3D lv, double* f, int additive, int zero_domain) {
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (g >= lv.ng) return;  // warp-uniform
  const int n = lv.n, S = lv.S;
  const int beg = lv.grp_ptr[g], end = lv.grp_ptr[g + 1];
  auto off_of = [&](int q) {
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    return static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k);
  };
  if (zero_domain && lv.grp_domain[g]) {
    for (int q = beg + lane; q < end; q += 32)
      if (lv.mem_slot[q] >= 0) f[off_of(q)] = 0.0;
    return;
  }
  if (end - beg < 2) return;
  double v = 0.0;
  if (additive) {
    for (int q0 = beg; q0 < end; q0 += 32) {
      const int q = q0 + lane;
      double x = 0.0;
      if (q < end) x = lv.mem_slot[q] < 0 ? lv.ghost[~lv.mem_slot[q]] : f[off_of(q)];
      const int cnt = min(32, end - q0);
      for (int t = 0; t < cnt; ++t) v += __shfl_sync(0xffffffffu, x, t);
    }
  } else {
    v = lv.mem_slot[beg] < 0 ? lv.ghost[~lv.mem_slot[beg]] : f[off_of(beg)];
  }
  __syncwarp();  // every lane has read before any copy is overwritten
  for (int q = beg + lane; q < end; q += 32)
    if (lv.mem_slot[q] >= 0) f[off_of(q)] = v;
}

__global__ void __launch_bounds__(kT) k3_owner_mask(DevLevel3D lv, double* f) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= lv.ng) return;
  const int n = lv.n, S = lv.S;
  for (int q = lv.grp_ptr[g] + 1; q < lv.grp_ptr[g + 1]; ++q) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    f[static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k)] = 0.0;
  }
}

__global__ void __launch_bounds__(kT) k3_set_boundary(DevLevel3D lv, double* f, const double* __restrict__ g_grp) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= lv.ng || !lv.grp_domain[g]) return;
  const int n = lv.n, S = lv.S;
  const double v = g_grp[g];
  for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
    if (lv.mem_slot[q] < 0) continue;
    int i, j, k;
    unpack_ijk(lv.mem_ijk[q], i, j, k);
    f[static_cast<size_t>(lv.mem_slot[q]) * S + lat3(n, i, j, k)] = v;
  }
}

// exchange pack of a sharded level: the contribution of each local member of a
// group that spans shards, computed by the same functions the group kernels
// use, so that every shard sums bit-identical member terms in slot order
__global__ void __launch_bounds__(kT) k3_pack(DevLevel3D lv, int mode, const double* __restrict__ x,
                                              const int* __restrict__ pos, const int* __restrict__ slot,
                                              const int* __restrict__ ijk, int e0, int e1, double* out) {
  const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e1) return;
  const int n = lv.n, s = slot[e];
  int i, j, k;
  unpack_ijk(ijk[e], i, j, k);
  const double* xm = x + static_cast<size_t>(s) * lv.S;
  double v;
  if (mode == PK3_VALUE)
    v = xm[lat3(n, i, j, k)];
  else if (mode == PK3_OFF_K)
    v = partial_off3(lv.psK + 240 * s, xm, n, i, j, k);
  else
    v = partial_full((mode == PK3_FULL_M ? lv.psM : lv.psK) + 240 * s, xm, n, i, j, k);
  out[pos[e]] = v;
}

// ---------------------------------------------------------------- level-0 CG (one CTA)
// CG on the unique macro-vertex values in shared memory (cg_level0's loop,
// proj/src/multigrid.cpp:198-229).  The level-0 operator is assembled (round 2
// specification, oracle apply0): row g adds, over the group's members in slot
// order, their partial stencils (centre first, then the directions inside the
// macro), coefficients of one column added in that order, columns in
// first-appearance order; y_g is the sequential sum over the row.  One thread
// per row; the rows sit in shared memory when they fit.
__device__ void cg0_apply_csr(int ng, const int* rp, const unsigned short* col, const double* val, const double* x,
                              double* y, const double* b, const unsigned char* dom, int residual) {
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    const int p0 = rp[g], p1 = rp[g + 1];
    double v = val[p0] * x[col[p0]];
    for (int t = p0 + 1; t < p1; ++t) v = v + val[t] * x[col[t]];
    y[g] = dom[g] ? 0.0 : (residual ? b[g] - v : v);
  }
}

// 3-d dot order (oracle o3_dot): chunks of 32 terms summed in order, then the
// chunk sums in order.  The products are formed in parallel first, the chunk
// sums are unrolled (loads in flight), thread 0 adds the chunk sums.
__device__ double cg0_dot(int ng, const double* a, const double* b, const unsigned char* dom, bool zero_dom,
                          double* chunks, double* prod) {
  const int nch = (ng + 31) / 32;
  __syncthreads();
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    double x = a[g], y = b[g];
    if (zero_dom && dom[g]) x = y = 0.0;
    prod[g] = x * y;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    double t[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) t[q] = 32 * c + q < ng ? prod[32 * c + q] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (32 * c + q < ng) s += t[q];
    chunks[c] = s;
  }
  __syncthreads();
  __shared__ double total;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int c = 0; c < nch; ++c) t += chunks[c];
    total = t;
  }
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(1024) k3_cg0(DevLevel3D lv, double* uc, const double* bc, CgParams prm,
                                               DevStatus* status, int staged) {
  extern __shared__ double sm[];
  const int ng = lv.ng;
  double* u = sm;
  double* b = u + ng;
  double* r = b + ng;
  double* p = r + ng;
  double* ap = p + ng;
  double* prod = ap + ng;  // dot-product terms
  double* chunks = prod + ng;
  // staged != 0: the assembled rows in shared memory behind the vectors
  const int nnz = lv.cg_nnz;
  double* sval = chunks + (ng + 31) / 32;
  int* srp = reinterpret_cast<int*>(sval + (staged ? nnz : 0));
  unsigned short* scol = reinterpret_cast<unsigned short*>(srp + (staged ? ng + 1 : 0));
  unsigned char* dom = reinterpret_cast<unsigned char*>(scol + (staged ? ((nnz + 3) & ~3) : 0));
  if (staged) {
    for (int t = threadIdx.x; t < nnz; t += blockDim.x) {
      sval[t] = lv.cg_val[t];
      scol[t] = lv.cg_col[t];
    }
    for (int t = threadIdx.x; t <= ng; t += blockDim.x) srp[t] = lv.cg_rowptr[t];
  }
  const int* rp = staged ? srp : lv.cg_rowptr;
  const unsigned short* col = staged ? scol : lv.cg_col;
  const double* val = staged ? sval : lv.cg_val;
  auto cg0_op = [&](const double* x, double* y, const double* bb, int residual) {
    cg0_apply_csr(ng, rp, col, val, x, y, bb, dom, residual);
  };
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    u[g] = uc[lv.own_dot[g]];
    b[g] = bc[lv.own_dot[g]];
    dom[g] = lv.grp_domain[g];
  }
  __syncthreads();
  cg0_op(u, r, b, 1);
  __syncthreads();
  for (int g = threadIdx.x; g < ng; g += blockDim.x) p[g] = r[g];
  double rr = cg0_dot(ng, r, r, dom, false, chunks, prod);
  const double bn = sqrt(fmax(0.0, cg0_dot(ng, b, b, dom, true, chunks, prod)));
  const double tol = prm.rel_tol * bn < prm.abs_floor ? prm.abs_floor : prm.rel_tol * bn;
  int it = 0;
  while (sqrt(rr) > tol) {
    if (++it > prm.max_iter) {
      if (threadIdx.x == 0 && status->code == 0) {
        status->code = 1;
        status->residual = sqrt(rr);
      }
      break;
    }
    cg0_op(p, ap, nullptr, 0);
    const double pap = cg0_dot(ng, p, ap, dom, false, chunks, prod);
    if (pap <= 0.0) {
      if (threadIdx.x == 0 && status->code == 0) {
        status->code = 2;
        status->residual = sqrt(rr);
      }
      break;
    }
    const double alpha = rr / pap;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
      u[g] = u[g] + alpha * p[g];
      r[g] = r[g] + (-alpha) * ap[g];
    }
    const double rn = cg0_dot(ng, r, r, dom, false, chunks, prod);
    const double beta = rn / rr;
    rr = rn;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) p[g] = p[g] * beta + r[g];
    __syncthreads();
  }
  if (threadIdx.x == 0) status->iters = it;
  __syncthreads();
  // scatter to every copy
  for (int g = threadIdx.x; g < ng; g += blockDim.x)
    for (int q = lv.grp_ptr[g]; q < lv.grp_ptr[g + 1]; ++q) {
      int i, j, k;
      unpack_ijk(lv.mem_ijk[q], i, j, k);
      uc[static_cast<size_t>(lv.mem_slot[q]) * lv.S + lat3(lv.n, i, j, k)] = u[g];
    }
}

// ---------------------------------------------------------------- estimator
// vertex c of a type-t micro-cell relative to its base, axis a (compile time)
__device__ __forceinline__ constexpr int cell_off(int t, int c, int a) {
  constexpr int v[6][4][3] = {{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
                              {{0, 0, 0}, {1, 0, 0}, {1, -1, 1}, {0, 0, 1}},
                              {{0, 0, 0}, {-1, 1, 0}, {0, 1, 0}, {0, 0, 1}},
                              {{0, 0, 0}, {-1, 1, 0}, {-1, 0, 1}, {0, 0, 1}},
                              {{0, 0, 0}, {0, -1, 1}, {1, -1, 1}, {0, 0, 1}},
                              {{0, 0, 0}, {0, -1, 1}, {-1, 0, 1}, {0, 0, 1}}};
  return v[t][c][a];
}

// one block per (macro, base plane k): rows to warps, base nodes to lanes, the
// six cell types per base node; per-block partial sums, reduced per macro in
// plane order by k3_estimate_reduce
__global__ void __launch_bounds__(kT) k3_estimate(DevLevel3D lv, const double* __restrict__ uL,
                                                  const double* __restrict__ wb, const double* __restrict__ wc,
                                                  double* part) {
  const int n = lv.n, S = lv.S, T = tsz(n);
  const int m = blockIdx.x / (n + 1), k = blockIdx.x - m * (n + 1);
  const int m2 = n - k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const size_t mo = static_cast<size_t>(m) * S;
  double Mt[6][16];
#pragma unroll
  for (int t = 0; t < 6; ++t)
#pragma unroll
    for (int e = 0; e < 16; ++e) Mt[t][e] = __ldg(lv.kmass + 96 * m + 16 * t + e);
  double qb = 0.0, qc = 0.0;
  for (int j = warp; j <= m2; j += nwarps) {
    // starts of rows (dk, dj) for dk in {0, 1}, dj in {-1, 0, 1}
    int rs[2][3];
#pragma unroll
    for (int dk = 0; dk < 2; ++dk)
#pragma unroll
      for (int dj = -1; dj <= 1; ++dj) {
        const int kk = k + dk, jj = j + dj;
        rs[dk][dj + 1] = (kk <= n && jj >= 0) ? T - tsz(n - kk) + lat2(n - kk, 0, jj) : 0;
      }
    for (int i = lane; i <= m2 - j; i += 32) {
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        bool ok = true;
        int vi[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int a = i + cell_off(t, c, 0), bb = j + cell_off(t, c, 1), cc = k + cell_off(t, c, 2);
          ok = ok && a >= 0 && bb >= 0 && a + bb + cc <= n;
          vi[c] = rs[cell_off(t, c, 2)][cell_off(t, c, 1) + 1] + a;
        }
        if (!ok) continue;
        double eb[4], ec[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double uu = uL[mo + vi[c]];
          eb[c] = uu - wb[mo + vi[c]];
          ec[c] = uu - wc[mo + vi[c]];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double* Tm = Mt[t];
          const double rb = ((Tm[4 * a] * eb[0] + Tm[4 * a + 1] * eb[1]) + Tm[4 * a + 2] * eb[2]) + Tm[4 * a + 3] * eb[3];
          const double rc = ((Tm[4 * a] * ec[0] + Tm[4 * a + 1] * ec[1]) + Tm[4 * a + 2] * ec[2]) + Tm[4 * a + 3] * ec[3];
          qb = qb + eb[a] * rb;
          qc = qc + ec[a] * rc;
        }
      }
    }
  }
  __shared__ double rb[kT], rcs[kT];
  rb[threadIdx.x] = qb;
  rcs[threadIdx.x] = qc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      rb[threadIdx.x] += rb[threadIdx.x + w];
      rcs[threadIdx.x] += rcs[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * static_cast<size_t>(blockIdx.x)] = rb[0];
    part[2 * static_cast<size_t>(blockIdx.x) + 1] = rcs[0];
  }
}

// Node-centric form of the same sums: over a macro, sum_cells e_c^T M_c e_c
// = sum_nodes e_i (M_m e)_i with M_m the macro's assembled mass matrix (the
// interior stencil stM, the signature partial stencils psM on the lattice
// boundary).  One block per (macro, plane k), rows to warps, nodes to lanes
// (coalesced); e = uL - w formed at each load.  Same sums as the cell form up
// to rounding (the tests bound the difference).
__global__ void __launch_bounds__(kT) k3_estimate_nodes(DevLevel3D lv, const double* __restrict__ uL,
                                                        const double* __restrict__ wb,
                                                        const double* __restrict__ wc, double* part) {
  const int n = lv.n, S = lv.S;
  const int m = blockIdx.x / (n + 1), k = blockIdx.x - m * (n + 1);
  const int m2 = n - k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const size_t mo = static_cast<size_t>(m) * S;
  const double* um = uL + mo;
  const double* bm = wb + mo;
  const double* cm = wc + mo;
  double qb = 0.0, qc = 0.0;
  for (int j = warp; j <= m2; j += nwarps) {
    int ra[7], len[7];
    node_rows(n, j, k, ra, len);
    for (int i = lane; i <= m2 - j; i += 32) {
      const int sig = sig3(n, i, j, k);
      const double* cf = sig ? lv.psM + 240 * static_cast<size_t>(m) + 15 * sig : lv.stM + 15 * static_cast<size_t>(m);
      const int c0 = ra[0] + i;
      bool ok[15];
      const double *au[15], *ab[15], *ac[15];
#pragma unroll
      for (int d = 0; d < 15; ++d) {
        const int r = dir_row(d), ii = i + dir_di(d);
        ok[d] = ii >= 0 && ii <= len[r];
        const int o = ok[d] ? ra[r] + ii : c0;
        au[d] = um + o;
        ab[d] = bm + o;
        ac[d] = cm + o;
      }
      double xu[15], xb[15], xc[15], c[15];
      load15(xu, au);
      load15(xb, ab);
      load15(xc, ac);
      load15_seq(c, cf);
      const double eb0 = xu[0] - xb[0], ec0 = xu[0] - xc[0];
      double mb = c[0] * eb0, mc = c[0] * ec0;
#pragma unroll
      for (int d = 1; d < 15; ++d) {
        const double tb = mb + c[d] * (xu[d] - xb[d]);
        const double tc = mc + c[d] * (xu[d] - xc[d]);
        mb = ok[d] ? tb : mb;
        mc = ok[d] ? tc : mc;
      }
      qb = qb + eb0 * mb;
      qc = qc + ec0 * mc;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    qb += __shfl_xor_sync(0xffffffffu, qb, o);
    qc += __shfl_xor_sync(0xffffffffu, qc, o);
  }
  __shared__ double rb[kT / 32], rcs[kT / 32];
  if (lane == 0) {
    rb[warp] = qb;
    rcs[warp] = qc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sb = 0.0, sc = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      sb += rb[w];
      sc += rcs[w];
    }
    part[2 * static_cast<size_t>(blockIdx.x)] = sb;
    part[2 * static_cast<size_t>(blockIdx.x) + 1] = sc;
  }
}

// Streaming form of k3_estimate_nodes (levels n >= 8): one CTA per macro
// walks its k-planes once; e_b = uL - wb and e_c = uL - wc of plane k + 2 are
// loaded (coalesced, issued before the plane-k work so their latency hides
// behind it) and stored into 3-slot shared-memory rings; plane k's nodes take
// their mass rows (interior stencil / boundary partial stencil) from the rings.
// Each of uL, wb, wc is read once.  Writes the macro's two sums directly.
constexpr int kEsThreads = 256;
constexpr int kEsPer = 9;  // plane nodes per thread (n <= 64: <= 2145 nodes)

__global__ void __launch_bounds__(kEsThreads, 2) k3_estimate_stream(DevLevel3D lv, const double* __restrict__ uL,
                                                                    const double* __restrict__ wb,
                                                                    const double* __restrict__ wc, double* sums) {
  extern __shared__ __align__(128) unsigned long long es_smem[];
  const int n = lv.n, S = lv.S, m = blockIdx.x, tid = threadIdx.x;
  const int stride = plane_stride(n);
  double* ps = reinterpret_cast<double*>(es_smem);  // 16 signatures x 15
  double* rb = ps + 240;                             // e_b ring, 2 slots (planes k, k + 1)
  double* rc = rb + 2 * stride;                      // e_c ring, 2 slots
  const size_t mo = static_cast<size_t>(m) * S;
  for (int t = tid; t < 240; t += kEsThreads)
    ps[t] = __ldg(lv.psM + 240 * static_cast<size_t>(m) + t) * (t % 15 == 0 ? 1.0 : 2.0);
  // e^T M e over the macro's (symmetric) assembled mass matrix as the diagonal
  // plus twice the forward half: the odd directions are the lexicographically
  // positive ones (planes k and k + 1 only), their coefficients doubled here
  double s[15];
#pragma unroll
  for (int d = 0; d < 15; ++d) s[d] = __ldg(lv.stM + 15 * static_cast<size_t>(m) + d) * (d == 0 ? 1.0 : 2.0);
  double lu[kEsPer], lb[kEsPer], lc[kEsPer];
  auto load = [&](int k) {  // plane k of uL, wb, wc into registers
    if (k > n) return;
    const size_t o = mo + plane_base(n, k);
    const int len = (n - k + 1) * (n - k + 2) / 2;
#pragma unroll
    for (int t = 0; t < kEsPer; ++t) {
      const int q = tid + t * kEsThreads;
      if (q < len) {
        lu[t] = __ldg(uL + o + q);
        lb[t] = __ldg(wb + o + q);
        lc[t] = __ldg(wc + o + q);
      }
    }
  };
  auto store = [&](int k) {  // e of plane k into its ring slot
    if (k > n) return;
    const int len = (n - k + 1) * (n - k + 2) / 2, sl = (k & 1) * stride;
#pragma unroll
    for (int t = 0; t < kEsPer; ++t) {
      const int q = tid + t * kEsThreads;
      if (q < len) {
        rb[sl + q] = lu[t] - lb[t];
        rc[sl + q] = lu[t] - lc[t];
      }
    }
  };
  load(0);
  store(0);
  load(1);
  store(1);
  __syncthreads();
  double qb = 0.0, qc = 0.0;
  for (int k = 0; k <= n; ++k) {
    load(k + 2);
    const int m2 = n - k;
    int base[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) base[d] = ((k - 1 + d) & 1) * stride;  // base[0] (plane k - 1) is not read
    if (k >= 1 && m2 >= 3) {
      const int mi = m2 - 3, ni = (mi + 1) * (mi + 2) / 2;
      for (int e = tid; e < ni; e += kEsThreads) {
        int i, j;
        decode2_fast(mi, e, i, j);
        ++i, ++j;
        const int r0 = lat2(m2, 0, j);
        int ra[7];
        ra[0] = base[1] + r0;
        ra[1] = ra[0] + (m2 + 1 - j);
        ra[2] = ra[0] - (m2 + 2 - j);
        ra[5] = base[2] + r0 - j;
        ra[3] = ra[5] - (m2 + 1 - j);
        ra[6] = ra[4] = 0;
        const double eb0 = rb[ra[0] + i], ec0 = rc[ra[0] + i];
        double mb = s[0] * eb0, mc = s[0] * ec0;
#pragma unroll
        for (int d = 1; d < 15; d += 2) {
          const int a = ra[dir_row(d)] + i + dir_di(d);
          mb = mb + s[d] * rb[a];
          mc = mc + s[d] * rc[a];
        }
        qb = qb + eb0 * mb;
        qc = qc + ec0 * mc;
      }
    }
    const int nb = k == 0 ? (m2 + 1) * (m2 + 2) / 2 : (m2 >= 1 ? 3 * m2 : 1);
    // boundary nodes continue the interior's thread rotation (balanced per plane)
    const int ni_all = k >= 1 && m2 >= 3 ? (m2 - 2) * (m2 - 1) / 2 : 0;
    for (int e = (tid - ni_all % kEsThreads + kEsThreads) % kEsThreads; e < nb; e += kEsThreads) {
      int i, j;
      if (k == 0) {
        decode2_fast(m2, e, i, j);
      } else if (m2 == 0) {
        i = 0, j = 0;
      } else if (e < m2 + 1) {
        i = e, j = 0;
      } else if (e < 2 * m2) {
        i = 0, j = e - m2;
      } else {
        j = e - 2 * m2 + 1, i = m2 - j;
      }
      const int sig = sig3(n, i, j, k);
      const double* cf = ps + 15 * sig;
      int ra[7];
      slot_rows(base, m2, j, ra);
      const int c0 = ra[0] + i;
      const double eb0 = rb[c0], ec0 = rc[c0];
      double mb = cf[0] * eb0, mc = cf[0] * ec0;
#pragma unroll
      for (int d = 1; d < 15; d += 2) {
        const bool ok = (sig & dir_bad(d)) == 0;
        const int a = ok ? ra[dir_row(d)] + i + dir_di(d) : c0;
        const double tb = mb + cf[d] * rb[a], tc = mc + cf[d] * rc[a];
        mb = ok ? tb : mb;
        mc = ok ? tc : mc;
      }
      qb = qb + eb0 * mb;
      qc = qc + ec0 * mc;
    }
    __syncthreads();  // plane k - 1's slot is free
    store(k + 2);
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    qb += __shfl_xor_sync(0xffffffffu, qb, o);
    qc += __shfl_xor_sync(0xffffffffu, qc, o);
  }
  __shared__ double wsum[2][kEsThreads / 32];
  if ((tid & 31) == 0) {
    wsum[0][tid >> 5] = qb;
    wsum[1][tid >> 5] = qc;
  }
  __syncthreads();
  if (tid == 0) {
    double sb = 0.0, sc = 0.0;
    for (int w = 0; w < kEsThreads / 32; ++w) {
      sb += wsum[0][w];
      sc += wsum[1][w];
    }
    sums[2 * m] = sb;
    sums[2 * m + 1] = sc;
  }
}

__global__ void k3_estimate_reduce(int M, int planes, const double* part, double* sums) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  double b = 0.0, c = 0.0;
  for (int k = 0; k < planes; ++k) {
    b += part[2 * (static_cast<size_t>(m) * planes + k)];
    c += part[2 * (static_cast<size_t>(m) * planes + k) + 1];
  }
  sums[2 * m] = b;
  sums[2 * m + 1] = c;
}

// ---------------------------------------------------------------- dot (owner copies + interiors)
__global__ void __launch_bounds__(kT) k3_dot_partial(DevLevel3D lv, const double* a, const double* b, double* part) {
  const int n = lv.n, S = lv.S;
  double s = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < lv.ng; t += stride) {
    const int o = lv.own_dot[t];
    s += a[o] * b[o];
  }
  const long long total = static_cast<long long>(lv.M) * S;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total; t += stride) {
    const int m = static_cast<int>(t / S), idx = static_cast<int>(t - static_cast<long long>(m) * S);
    int k = 0;
    while (idx >= tsz(n) - tsz(n - k - 1)) ++k;
    int i, j;
    decode2(n - k, idx - (tsz(n) - tsz(n - k)), i, j);
    if (interior3(n, i, j, k)) s += a[t] * b[t];
  }
  __shared__ double red[kT];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k3_dot_final(const double* part, int count, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < count; ++i) s += part[i];
    *out = s;
  }
}

__global__ void k3_axpy(double* y, const double* x, double alpha, long long count) {
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < count;
       q += static_cast<long long>(gridDim.x) * blockDim.x)
    y[q] = y[q] + alpha * x[q];
}

// source table f at every copy's own node coordinates (device libm; fast mode)
__global__ void __launch_bounds__(kT) k3_ftab(DevLevel3D lv, const double* __restrict__ corners, int kind,
                                              const double* __restrict__ par, double* f) {
  const int n = lv.n;
  const int m = blockIdx.x / (n + 1), k = blockIdx.x - m * (n + 1);
  const int m2 = n - k;
  const int np = (m2 + 1) * (m2 + 2) / 2;
  const int base = tsz(n) - tsz(n - k);
  const double* P = corners + 12 * m;
  for (int q = threadIdx.x; q < np; q += blockDim.x) {
    int i, j;
    decode2(m2, q, i, j);
    double X[3];
    for (int a = 0; a < 3; ++a)
      X[a] = P[a] + (static_cast<double>(i) / n) * (P[3 + a] - P[a]) + (static_cast<double>(j) / n) * (P[6 + a] - P[a]) +
             (static_cast<double>(k) / n) * (P[9 + a] - P[a]);
    double v = 0.0;
    if (kind == 3) {
      v = 3.0 * M_PI * M_PI * (sin(M_PI * X[0]) * sin(M_PI * X[1]) * sin(M_PI * X[2]));
    } else if (kind == 4) {
      const double dx = X[0] - 0.5, dy = X[1] - 0.5, dz = X[2] - 0.5, r2 = dx * dx + dy * dy + dz * dz;
      v = (6.0 * 1000.0 - 4.0 * 1000.0 * 1000.0 * r2) * exp(-1000.0 * r2);
    } else if (kind == 5) {
      double sx[4], sy[4], sz[4];
      for (int a = 0; a < 4; ++a) {
        sx[a] = sin((a + 1) * M_PI * X[0]);
        sy[a] = sin((a + 1) * M_PI * X[1]);
        sz[a] = sin((a + 1) * M_PI * X[2]);
      }
      for (int c = 0; c < 4; ++c)
        for (int b = 0; b < 4; ++b)
          for (int a = 0; a < 4; ++a) v += par[a + 4 * b + 16 * c] * (sx[a] * sy[b] * sz[c]);
    }
    f[static_cast<size_t>(m) * lv.S + base + q] = v;
  }
}

void check3(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(KB_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void init_constants() {
  static bool done = false;
  if (done) return;
  int cv[6][4][3];
  for (int ty = 0; ty < 6; ++ty)
    for (int r = 0; r < 4; ++r) cell_vertex(ty, r, cv[ty][r][0], cv[ty][r][1], cv[ty][r][2]);
  KB_CUDA_CHECK(cudaMemcpyToSymbol(c_cv, cv, sizeof(cv)));
  KB_CUDA_CHECK(cudaMemcpyToSymbol(c_dir, kDir, sizeof(kDir)));
  int pdir[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = 1; p < 8; ++p)
    for (int d = 1; d < 15; ++d) {
      const int* v = kDir[d];
      // the positive direction whose parities are p
      if (((v[0] & 1) | ((v[1] & 1) << 1) | ((v[2] & 1) << 2)) == p && (d & 1)) pdir[p] = d;
    }
  KB_CUDA_CHECK(cudaMemcpyToSymbol(c_pdir, pdir, sizeof(pdir)));
  done = true;
}

int device_attr3(cudaDeviceAttr a) {
  int dev = 0, v = 0;
  KB_CUDA_CHECK(cudaGetDevice(&dev));
  KB_CUDA_CHECK(cudaDeviceGetAttribute(&v, a, dev));
  return v;
}

// KB_GS3_SPLIT=1: the per-colour launches (k3_gs_groups + k3_gs_color), kept
// as a same-result variant for measurement
bool gs_split() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_GS3_SPLIT");
    v = e && e[0] == '1';
  }
  return v == 1;
}

// largest n whose smoother runs whole (boundary colours and interior steps) in
// one cooperative launch; above it the sweeps alternate the cooperative
// boundary kernel with the plane-stream interior (experiment: KB_GS3_WHOLE_N)
int gs_whole_n() {
  // n = 16 split: 0.214 -> 0.174 ms per 2 sweeps on 384 macros, 0.335 -> 0.323 ms on 3072; n = 8 split is slower on 3072
  static const int v = getenv("KB_GS3_WHOLE_N") ? atoi(getenv("KB_GS3_WHOLE_N")) : 8;
  return std::min(v, 16);
}

// KB_GS3_PHASES (measurement only): 1 boundary phase, 2 interior phase, 3 both
int gs_phases() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_GS3_PHASES");
    v = e ? atoi(e) : 3;
  }
  return v;
}

// streaming apply / estimator for levels with 8 <= n <= 64 (KB_APPLY3_STREAM=0: plane-block kernels)
bool apply_streams(const DevLevel3D& lv) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KB_APPLY3_STREAM");
    v = e ? atoi(e) : 1;
  }
  return v && lv.n >= 8 && lv.n <= 64 && lv.M > 0;
}
bool estimate_cells() {
  static int cells = -1;
  if (cells < 0) {
    const char* e = getenv("KB_EST3_CELLS");  // measurement: the cell-by-cell form
    cells = e && e[0] == '1';
  }
  return cells == 1;
}

// threads of a (macro, k-plane) block: the average plane of a level-n lattice
// holds (n + 1)(n + 2) / 6 nodes (experiment: KB_PLANE_NT)
int plane_threads(int n) {
  static const int forced = getenv("KB_PLANE_NT") ? atoi(getenv("KB_PLANE_NT")) : 0;
  if (forced) return forced;
  return n >= 64 ? 256 : n >= 32 ? 128 : 64;
}

int blocks_for(long long count) { return static_cast<int>(std::max(1ll, (count + kT - 1) / kT)); }

}  // namespace

void launch3_apply(const DevLevel3D& lv, bool mass, const double* x, double* y, const double* b, int mode,
                   cudaStream_t st) {
  init_constants();
  if (apply_streams(lv)) {
    const size_t smem = (kAsSlots + 240 + kAsSlots * static_cast<size_t>(plane_stride(lv.n))) * 8;
    // threads per macro by plane size: the per-plane barrier and TMA wait cost
    // less with fewer warps and more CTAs per SM on the small planes (residual on
    // 3072 macros: n = 32 0.51 -> 0.36 ms with 128 threads, n = 16 0.22 -> 0.13 ms
    // and n = 8 0.12 -> 0.08 ms with 64; n = 64 keeps 256)
    static const int nt_exp = getenv("KB_AS_NT") ? atoi(getenv("KB_AS_NT")) : 0;
    const int nt = nt_exp ? nt_exp : (lv.n >= 64 ? 256 : lv.n >= 32 ? 128 : 64);
    if (nt == 64) {
      ensure_dynamic_smem(k3_apply_stream<64>, smem);
      k3_apply_stream<64><<<lv.M, 64, smem, st>>>(lv, mass ? 1 : 0, x, y, b, mode);
    } else if (nt == 128) {
      ensure_dynamic_smem(k3_apply_stream<128>, smem);
      k3_apply_stream<128><<<lv.M, 128, smem, st>>>(lv, mass ? 1 : 0, x, y, b, mode);
    } else {
      ensure_dynamic_smem(k3_apply_stream<256>, smem);
      k3_apply_stream<256><<<lv.M, 256, smem, st>>>(lv, mass ? 1 : 0, x, y, b, mode);
    }
    check3("k3_apply_stream");
    if (lv.ng > 0) {
      k3_apply_groups<<<blocks_for(lv.ng), kT, 0, st>>>(lv, y, b, mode);
      check3("k3_apply_groups");
    }
    return;
  }
  const int planes = lv.M * (lv.n + 1);
  if (lv.n < 8 && lv.ng > 0) {  // small levels: the groups by warps (latency-bound), planes as before
    k3_apply<<<planes, kT, 0, st>>>(lv, mass ? 1 : 0, x, y, b, mode, planes);
    check3("k3_apply");
    k3_apply_groups_warp<<<blocks_for(32ll * lv.ng), kT, 0, st>>>(lv, mass ? 1 : 0, x, y, b, mode);
    check3("k3_apply_groups_warp");
    return;
  }
  k3_apply<<<planes + blocks_for(lv.ng), kT, 0, st>>>(lv, mass ? 1 : 0, x, y, b, mode, planes);
  check3("k3_apply");
}

// interior phase of one sweep (levels without step lists, the sharded path, KB_GS3_SPLIT)
template <int NT, int US, int BS>
void launch_gs_planes(const DevLevel3D& lv, double* u, const double* b, cudaStream_t st) {
  const int steps = 4 * (lv.n - 3);
  const int smem = 8 * (US + BS) + 8 * ((steps + 4) >> 2 << 1) + (US + BS) * plane_stride(lv.n) * 8;
  ensure_dynamic_smem(k3_gs_planes<NT, US, BS>, static_cast<size_t>(smem));
  k3_gs_planes<NT, US, BS><<<lv.M, NT, smem, st>>>(lv, u, b);
  check3("k3_gs_planes");
}

void launch3_gs_interior(const DevLevel3D& lv, double* u, const double* b, cudaStream_t st) {
  init_constants();
  if (lv.n < 4 || lv.M <= 0) return;  // no lattice-interior nodes
  if (!lv.pat_node) {  // n > 64
    k3_gs_planes_global<<<lv.M, kT, 0, st>>>(lv, u, b);
    check3("k3_gs_planes_global");
  } else if (lv.n == 64) {
    launch_gs_planes<512, 4, 2>(lv, u, b, st);  // 103 KB: two CTAs per SM
  } else if (lv.n == 32) {
    // CTAs per SM matter more than the prefetch depth here (27 KB, eight CTAs
    // per SM: 0.44 ms per 2 sweeps on 3072 macros; 54 KB with 8 + 4 slots: 0.62 ms)
    launch_gs_planes<128, 4, 2>(lv, u, b, st);
  } else {
    launch_gs_planes<32, 4, 2>(lv, u, b, st);
  }
}

void launch3_gs(const DevLevel3D& lv, double* u, const double* b, int sweeps, cudaStream_t st) {
  init_constants();
  if (sweeps <= 0) return;
  if (gs_split()) {
    for (int s = 0; s < sweeps; ++s) {
      for (int c = 0; c < lv.colors; ++c) {
        k3_gs_groups<<<blocks_for(lv.ng), kT, 0, st>>>(lv, u, b, c);
        check3("k3_gs_groups");
      }
      launch3_gs_interior(lv, u, b, st);
    }
    return;
  }
  // 256-thread CTAs, three per SM (cooperative: grid barriers between the colours)
  static int sms = 0, occ = 0;
  if (sms == 0) {
    sms = device_attr3(cudaDevAttrMultiProcessorCount);
    KB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_gs_sweeps<256, 3>, 256, 0));
    if (occ < 1) fail(KB_CUDA, "k3_gs_sweeps cannot be resident");
  }
  // grid by the largest colour phase: lanes of its groups / 256, in whole
  // multiples of the SM count, at least one CTA per SM (fewer CTAs: cheaper grid
  // barriers; 384 macros at n = 8: 0.141 -> 0.110 ms per 2 sweeps with 148 CTAs)
  int grid = occ * sms;
  if (lv.max_color_groups > 0) {
    const long long lanes = static_cast<long long>(lv.max_color_groups) * (lv.n <= 8 ? 4 : 2);
    const int want = static_cast<int>((lanes + 255) / 256);
    grid = std::min(grid, std::max(sms, (want + sms - 1) / sms * sms));
  }
  if (lv.n <= 4) grid = std::min(grid, sms);  // tiny levels: one CTA per SM
  if (const char* e = getenv("KB_GS3_GRID")) grid = std::max(1, std::min(grid, atoi(e)));
  int active = grid;
  if (const char* e = getenv("KB_GS3_ACTIVE")) active = std::max(1, std::min(grid, atoi(e)));
  int group = lv.M;  // macros of a CTA taken together per interior step
  if (const char* e = getenv("KB_GS3_G")) group = std::max(1, atoi(e));
  // levels with step lists (n <= 16) run whole in one launch; larger levels
  // alternate the boundary colours (cooperative) with the plane-stream interior
  const bool whole = lv.n <= gs_whole_n();
  const int calls = whole ? 1 : sweeps;
  for (int s = 0; s < calls; ++s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int ph = gs_phases();
    if (ph & 1 || whole)
      KB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k3_gs_sweeps<256, 3>, lv, u, b, whole ? sweeps : 1, whole ? ph : (ph & ~2),
                                       active, group));
    if (!whole && (ph & 2)) launch3_gs_interior(lv, u, b, st);
  }
}

int launch3_apply_count(const DevLevel3D& lv) { return apply_streams(lv) || (lv.n < 8 && lv.ng > 0) ? 1 + (lv.ng > 0) : 1; }
int launch3_estimate_count(const DevLevel3D& lv) { return !estimate_cells() && apply_streams(lv) ? 1 : 2; }

int launch3_gs_count(const DevLevel3D& lv, int sweeps) {
  if (sweeps <= 0) return 0;
  const int interior = lv.n >= 4 ? 1 : 0;
  if (gs_split()) return sweeps * (lv.colors + interior);
  return lv.n <= gs_whole_n() ? 1 : sweeps * (1 + interior);
}

void launch3_prolong(const DevLevel3D& coarse, const DevLevel3D& fine, const double* c, double* f, int mode,
                     cudaStream_t st) {
  init_constants();
  k3_prolong<<<fine.M * (fine.n + 1), plane_threads(fine.n), 0, st>>>(coarse, fine, c, f, mode);
  check3("k3_prolong");
}

void launch3_restrict(const DevLevel3D& fine, const DevLevel3D& coarse, const double* rf, double* rc,
                      int zero_domain, cudaStream_t st, double* zero_out) {
  init_constants();
  k3_restrict<<<coarse.M * (coarse.n + 1), plane_threads(coarse.n), 0, st>>>(fine, coarse, rf, rc, zero_out);
  check3("k3_restrict");
  launch3_sync_zero(coarse, rc, 1, zero_domain, st);
}

void launch3_restrict_only(const DevLevel3D& fine, const DevLevel3D& coarse, const double* rf, double* rc,
                           cudaStream_t st) {
  init_constants();
  k3_restrict<<<coarse.M * (coarse.n + 1), plane_threads(coarse.n), 0, st>>>(fine, coarse, rf, rc, nullptr);
  check3("k3_restrict");
}

void launch3_sync_zero(const DevLevel3D& lv, double* f, int additive, int zero_domain, cudaStream_t st) {
  if (lv.n < 8)
    k3_sync_warp<<<blocks_for(32ll * lv.ng), kT, 0, st>>>(lv, f, additive, zero_domain);
  else
    k3_sync<<<blocks_for(lv.ng), kT, 0, st>>>(lv, f, additive, zero_domain);
  check3("k3_sync");
}

void launch3_owner_mask(const DevLevel3D& lv, const double* f, double* out, cudaStream_t st) {
  KB_CUDA_CHECK(cudaMemcpyAsync(out, f, sizeof(double) * static_cast<size_t>(lv.M) * lv.S, cudaMemcpyDeviceToDevice,
                                st));
  k3_owner_mask<<<blocks_for(lv.ng), kT, 0, st>>>(lv, out);
  check3("k3_owner_mask");
}

void launch3_set_boundary(const DevLevel3D& lv, double* f, const double* g_grp, int zero_rest, cudaStream_t st) {
  if (zero_rest) KB_CUDA_CHECK(cudaMemsetAsync(f, 0, sizeof(double) * static_cast<size_t>(lv.M) * lv.S, st));
  k3_set_boundary<<<blocks_for(lv.ng), kT, 0, st>>>(lv, f, g_grp);
  check3("k3_set_boundary");
}

void launch3_sync(const DevLevel3D& lv, double* f, int additive, cudaStream_t st) {
  launch3_sync_zero(lv, f, additive, 0, st);
}

void launch3_cg0(const DevLevel3D& lv0, double* u, const double* b, double* scratch, CgParams prm,
                 DevStatus* status, cudaStream_t st) {
  (void)scratch;
  init_constants();
  const size_t base = (6 * static_cast<size_t>(lv0.ng) + (lv0.ng + 31) / 32) * sizeof(double) + lv0.ng + 16;
  if (base > 200 * 1024) fail(KB_STRUCTURAL, "coarse mesh too large for the level-0 CG (more than ~4800 vertices)");
  if (!lv0.cg_rowptr) fail(KB_INTERNAL, "level-0 operator rows missing");
  // the assembled rows staged in shared memory when they fit (no per-iteration L2 traffic)
  const size_t rows_bytes = 8 * static_cast<size_t>(lv0.cg_nnz) + 4 * static_cast<size_t>(lv0.ng + 1) +
                            2 * static_cast<size_t>((lv0.cg_nnz + 3) & ~3);
  const int staged = base + rows_bytes + 64 <= 220 * 1024 ? 1 : 0;
  const size_t smem = base + (staged ? rows_bytes + 64 : 0);
  ensure_dynamic_smem(k3_cg0, smem);
  k3_cg0<<<1, 1024, smem, st>>>(lv0, u, b, prm, status, staged);
  check3("k3_cg0");
}

void launch3_estimate(const DevLevel3D& lv, const double* uL, const double* wb, const double* wc, double* sums,
                      double* part, cudaStream_t st) {
  init_constants();
  const bool cells = estimate_cells();
  if (!cells && apply_streams(lv)) {
    const size_t smem = (240 + 4 * static_cast<size_t>(plane_stride(lv.n))) * 8;
    ensure_dynamic_smem(k3_estimate_stream, smem);
    k3_estimate_stream<<<lv.M, kEsThreads, smem, st>>>(lv, uL, wb, wc, sums);
    check3("k3_estimate_stream");
    return;
  }
  if (cells)
    k3_estimate<<<lv.M * (lv.n + 1), kT, 0, st>>>(lv, uL, wb, wc, part);
  else
    k3_estimate_nodes<<<lv.M * (lv.n + 1), kT, 0, st>>>(lv, uL, wb, wc, part);
  check3("k3_estimate");
  k3_estimate_reduce<<<(lv.M + 127) / 128, 128, 0, st>>>(lv.M, lv.n + 1, part, sums);
  check3("k3_estimate_reduce");
}

void launch3_dot(const DevLevel3D& lv, const double* a, const double* b, double* partial, double* out,
                 cudaStream_t st) {
  k3_dot_partial<<<64, kT, 0, st>>>(lv, a, b, partial);
  k3_dot_final<<<1, 32, 0, st>>>(partial, 64, out);
  check3("k3_dot");
}

void launch3_ftab(const DevLevel3D& lv, const double* corners, int kind, const double* params, double* f,
                  cudaStream_t st) {
  init_constants();
  k3_ftab<<<lv.M * (lv.n + 1), kT, 0, st>>>(lv, corners, kind, params, f);
  check3("k3_ftab");
}

void launch3_pack(const DevLevel3D& lv, int mode, const double* x, const int* pos, const int* slot, const int* ijk,
                  int e0, int e1, double* out, cudaStream_t st) {
  if (e1 <= e0) return;
  k3_pack<<<blocks_for(e1 - e0), kT, 0, st>>>(lv, mode, x, pos, slot, ijk, e0, e1, out);
  check3("k3_pack");
}

void launch3_gs_color_groups(const DevLevel3D& lv, double* u, const double* b, int c, cudaStream_t st) {
  init_constants();
  k3_gs_groups<<<blocks_for(lv.ng), kT, 0, st>>>(lv, u, b, c);
  check3("k3_gs_groups");
}

void launch3_axpy(double* y, const double* x, double alpha, std::int64_t count, cudaStream_t st) {
  k3_axpy<<<blocks_for(std::min<long long>(count, 148ll * 32 * kT)), kT, 0, st>>>(y, x, alpha, count);
  check3("k3_axpy");
}

}  // namespace kb
