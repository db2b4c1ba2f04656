// Development micro-benchmark: base latencies on the B200 (not product code).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_bar(long long* out, int iters, int threads) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_syncthreads(long long* out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / iters;
}
__global__ void k_dadd(long long* out, double a, int iters) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x + a; x = x + a; x = x + a; x = x + a; x = x + a; x = x + a; x = x + a; x = x + a;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[2] = (t1 - t0) / (8 * iters); out[9] = (long long)x; }
}
__global__ void k_dmul(long long* out, double a, int iters) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = x * a; x = x * a; x = x * a; x = x * a; x = x * a; x = x * a; x = x * a; x = x * a;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[3] = (t1 - t0) / (8 * iters); out[10] = (long long)x; }
}
__global__ void k_lds(long long* out, int iters) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = buf[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[4] = (t1 - t0) / iters; out[11] = p; }
}
__global__ void k_ddiv(long long* out, double a, int iters) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = (x + 1.0) / a;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[5] = (t1 - t0) / iters; out[12] = (long long)x; }
}
__global__ void k_shfl(long long* out, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_down_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[6] = (t1 - t0) / iters; out[13] = (long long)x; }
}
int main() {
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k_bar<<<1, 160>>>(d, 1000, 160);
    k_syncthreads<<<1, 160>>>(d, 1000);
    k_dadd<<<1, 32>>>(d, 1.000001, 1000);
    k_dmul<<<1, 32>>>(d, 1.000001, 1000);
    k_lds<<<1, 32>>>(d, 1000);
    k_ddiv<<<1, 32>>>(d, 3.0, 1000);
    k_shfl<<<1, 32>>>(d, 1000);
  }
  long long h[16];
  cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  printf("bar.sync(160) %lld cyc\nsyncthreads(160) %lld\nDADD dep %lld\nDMUL dep %lld\nLDS dep %lld\nDDIV dep %lld\nSHFL+DADD %lld\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
