// FP64 latency / throughput probe (dependent DFMA chain, independent DFMAs,
// __syncthreads round trip) on one SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double a, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3 + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void indep(double* out, double a, int n, long long* cyc) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, 1e-9);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void bar(double* out, int n, long long* cyc) {
  __shared__ double sh[256];
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    sh[threadIdx.x] = x;
    __syncthreads();
    x = sh[(threadIdx.x + 1) & 255] + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 8);
  const int n = 4096;
  chain<<<1, 32>>>(out, 0.999999, n, cyc); cudaDeviceSynchronize();
  chain<<<1, 32>>>(out, 0.999999, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DFMA latency: %.2f cycles\n", (double)h / n);
  for (int w : {1, 4, 8, 16, 32}) {
    indep<<<1, 32 * w>>>(out, 0.999999, n, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%2d warps x 8 independent chains: %.3f warp-DFMA/cycle/SM\n", w, (double)w * 8 * n / h);
  }
  for (int t : {64, 128, 256}) {
    bar<<<1, t>>>(out, n, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("STS+BAR+LDS round trip, %d threads: %.1f cycles\n", t, (double)h / n);
  }
  return 0;
}
