// Development micro-benchmark (not product code): the per-step named-barrier
// structure of k_gs_pipe on the B200 -- consumers bar.arrive(A[t % 12]) then
// bar.sync(B); one sync warp bar.sync(B); four publisher warps bar.sync(A[t])
// for t = w mod 4.  Cycles per step for a given number of consumer warps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void k_pipe_bars(int steps, int cw, int pubs_on, long long* out) {
  const int warp = threadIdx.x >> 5;
  const int cth = 32 * cw, bth = cth + 32;
  long long t0 = clock64();
  if (warp < cw) {  // consumers
    for (int t = 0; t < steps; ++t) {
      if (pubs_on) bar_arrive(2 + t % 12, bth);
      bar_sync(1, bth);
    }
  } else if (warp == cw) {  // sync warp
    for (int t = 0; t < steps; ++t) bar_sync(1, bth);
  } else if (pubs_on) {  // publishers
    const int w = warp - cw - 1;
    for (int t = w; t < steps; t += 4) bar_sync(2 + t % 12, bth);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / steps;
}

// alternative: the gate as an mbarrier-free shared-memory counter: consumers
// spin until gate >= t (the sync warp writes it), then increment a per-step
// done counter with atomicAdd; no named barriers
__global__ void k_pipe_flags(int steps, int cw, long long* out) {
  __shared__ volatile int gate;
  __shared__ int done[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) gate = 0;
  if (threadIdx.x < 16) done[threadIdx.x] = 0;
  __syncthreads();
  long long t0 = clock64();
  if (warp < cw) {
    for (int t = 0; t < steps; ++t) {
      while (gate < t) {}
      __syncwarp();
      if (lane == 0) atomicAdd(&done[t & 15], 1);
    }
  } else if (warp == cw) {
    for (int t = 0; t < steps; ++t) {
      // open gate t once every consumer finished step t - 1
      if (t > 0) {
        while (*((volatile int*)&done[(t - 1) & 15]) < cw) {}
        if (lane == 0) done[(t - 1) & 15] = 0;
      }
      __syncwarp();
      if (lane == 0) gate = t;
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / steps;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int cw : {2, 4, 6}) {
    for (int pubs : {0, 1}) {
      const int threads = 32 * (cw + 1 + (pubs ? 4 : 0));
      k_pipe_bars<<<1, threads>>>(1000, cw, pubs, d);
      k_pipe_bars<<<1, threads>>>(20000, cw, pubs, d);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("named barriers: %d consumer warps, publishers %s: %lld cycles per step\n", cw, pubs ? "on" : "off", h[0]);
    }
    k_pipe_flags<<<1, 32 * (cw + 1)>>>(20000, cw, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("shared-memory flags: %d consumer warps: %lld cycles per step\n", cw, h[1]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
