// Development micro-benchmark (not product code): cost of a grid-wide barrier
// on the B200 -- cooperative_groups grid.sync() against a monotonic-counter
// barrier (one atomicAdd per CTA, thread 0 polls with ld.acquire.gpu).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  g.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__device__ __forceinline__ void ctr_bar(unsigned* ctr, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}
__global__ void k_ctr(int iters, unsigned* ctr, long long* out) {
  unsigned target = 0;
  ctr_bar(ctr, target);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) ctr_bar(ctr, target);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / iters;
}

int main() {
  long long* out;
  unsigned* ctr;
  cudaMallocManaged(&out, 16);
  cudaMalloc(&ctr, 4);
  int iters = 2000;
  for (int per = 1; per <= 3; ++per) {
    int grid = 148 * per;
    void* a1[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)k_cg, dim3(grid), dim3(256), a1, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(ctr, 0, 4);
    void* a2[] = {&iters, &ctr, &out};
    cudaLaunchCooperativeKernel((void*)k_ctr, dim3(grid), dim3(256), a2, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("grid %d x 256: grid.sync %lld cycles, counter barrier %lld cycles (%s)\n", grid, out[0], out[1],
           cudaGetErrorString(e));
  }
  return 0;
}
