// Development micro-benchmark (not product code): one-way latency of a
// cross-SM "data + progress flag" hand-off through L2 on the B200, for the
// publication / detection variants the pipelined smoother can use.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: data store; red.release.gpu flag / consumer ld.acquire spin, then data load (.cg)
// mode 1: data store; st.release.gpu flag / consumer ld.acquire spin, then data load
// mode 2: data store; fence.acq_rel.gpu; st.relaxed flag / consumer ld.relaxed spin; fence; data load
// mode 3: no data: flag only (st.release / ld.acquire)
__global__ void k_pingpong(int* flags, double* data, int iters, int mode, long long* out) {
  const int me = blockIdx.x, other = 1 - me;
  if (threadIdx.x != 0) return;
  int* myflag = flags + 32 * me;        // separate 128-byte lines
  int* otherflag = flags + 32 * other;
  double* mydata = data + 16 * me;
  double* otherdata = data + 16 * other;
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if ((it & 1) == me) {  // my turn to publish
      if (mode != 3) mydata[0] = acc + it;
      if (mode == 0) asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(myflag), "r"(it) : "memory");
      else if (mode == 1 || mode == 3) asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(myflag), "r"(it) : "memory");
      else {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(myflag), "r"(it) : "memory");
      }
    } else {  // wait for the other's publication of step it
      if (mode == 2) {
        while (ld_rlx(otherflag) < it) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        while (ld_acq(otherflag) < it) {}
      }
      if (mode != 3) acc += __ldcg(otherdata);
    }
  }
  long long t1 = clock64();
  out[me] = (t1 - t0) / iters;
  out[2 + me] = (long long)acc;
}

int main() {
  int* flags;
  double* data;
  long long* out;
  cudaMalloc(&flags, 4096);
  cudaMalloc(&data, 4096);
  cudaMalloc(&out, 64);
  const char* names[4] = {"red.release + ld.acquire + data .cg", "st.release + ld.acquire + data .cg",
                          "fence + st.relaxed / ld.relaxed + fence + data", "st.release / ld.acquire, flag only"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flags, 0, 4096);
      cudaMemset(data, 0, 4096);
      k_pingpong<<<2, 32>>>(flags, data, 20000, mode, out);
      cudaDeviceSynchronize();
    }
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("%-48s one-way hand-off %lld cycles\n", names[mode], (h[0] + h[1]) / 2);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
