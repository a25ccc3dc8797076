#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}
__global__ void k_rcp(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fast_rcp(x) + 1.5;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_div(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 1.5;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_mufu(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r + 1.5;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, int n, long long* cyc) {
  __shared__ double sh[64];
  sh[threadIdx.x] = threadIdx.x;
  __syncwarp();
  int idx = threadIdx.x;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = sh[idx & 63];
    acc += v;
    idx = (int)v + 1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_syncwarp(double* out, int n, long long* cyc) {
  __shared__ double sh[64];
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (threadIdx.x == (i & 31)) sh[i & 1] = x;
    __syncwarp();
    x = sh[i & 1] + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  const int n = 2048;
  k_rcp<<<1, 32>>>(out, 3.0, n, cyc); cudaDeviceSynchronize(); k_rcp<<<1, 32>>>(out, 3.0, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("fast_rcp chain: %.1f cycles\n", (double)h / n);
  k_div<<<1, 32>>>(out, 3.0, n, cyc); cudaDeviceSynchronize(); k_div<<<1, 32>>>(out, 3.0, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("IEEE div chain: %.1f cycles\n", (double)h / n);
  k_mufu<<<1, 32>>>(out, 3.0, n, cyc); cudaDeviceSynchronize(); k_mufu<<<1, 32>>>(out, 3.0, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("MUFU.RCP64H+DADD chain: %.1f cycles\n", (double)h / n);
  k_lds<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize(); k_lds<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("LDS.64 dependent chain: %.1f cycles\n", (double)h / n);
  k_syncwarp<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize(); k_syncwarp<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("STS+syncwarp+LDS: %.1f cycles\n", (double)h / n);
  return 0;
}
