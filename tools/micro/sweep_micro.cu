// Microbenchmark of the 96x96 register sweep (one CTA): full kernel vs
// variants with parts removed, to locate the per-step latency.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_19892_b200/csrc/mas.cuh"

template <int VAR>
__global__ void sweep_var(const double* A, double* out, long long* cyc) {
  __shared__ double rowk[2 * 96];
  const int m = 96;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double R[SWEEP_T][SWEEP_T];
  for (int a = 0; a < SWEEP_T; ++a)
    for (int b = 0; b < SWEEP_T; ++b) R[a][b] = A[(tr + 16 * a) * m + tc + 16 * b];
  if (tr == 0) publish(R, 0, rowk, tc, m);
  long long t0 = clock64();
  for (int k = 0; k < m; ++k) {
    double* rk = rowk + (k & 1) * 96;
    __syncthreads();
    const double piv = rk[k];
    const double inv = VAR == 3 ? 1.0 / piv : fast_rcp(piv);
    double ci[SWEEP_T], cj[SWEEP_T];
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a) {
      ci[a] = rk[min(tr + 16 * a, 95)] * inv;
      cj[a] = rk[min(tc + 16 * a, 95)];
    }
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a)
#pragma unroll
      for (int b = 0; b < SWEEP_T; ++b) R[a][b] = fma(-ci[a], cj[b], R[a][b]);
    const int kr = k & 15, ka = k >> 4;
    if (VAR != 1) {
      if (tr == kr) {
        switch (ka) {
          case 0: fix_row<0>(R, cj, inv); break;
          case 1: fix_row<1>(R, cj, inv); break;
          case 2: fix_row<2>(R, cj, inv); break;
          case 3: fix_row<3>(R, cj, inv); break;
          case 4: fix_row<4>(R, cj, inv); break;
          default: fix_row<5>(R, cj, inv); break;
        }
      }
      if (tc == kr) {
        switch (ka) {
          case 0: fix_col<0>(R, ci); if (tr == kr) R[0][0] = -inv; break;
          case 1: fix_col<1>(R, ci); if (tr == kr) R[1][1] = -inv; break;
          case 2: fix_col<2>(R, ci); if (tr == kr) R[2][2] = -inv; break;
          case 3: fix_col<3>(R, ci); if (tr == kr) R[3][3] = -inv; break;
          case 4: fix_col<4>(R, ci); if (tr == kr) R[4][4] = -inv; break;
          default: fix_col<5>(R, ci); if (tr == kr) R[5][5] = -inv; break;
        }
      }
    }
    const int k1 = k + 1;
    if (VAR == 2) {
      if (k1 < m && tid < 96) rowk[(k1 & 1) * 96 + tid] = R[0][0];  // no switch
    } else {
      if (k1 < m && tr == (k1 & 15)) publish(R, k1 >> 4, rowk + (k1 & 1) * 96, tc, m);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < SWEEP_T; ++a)
    for (int b = 0; b < SWEEP_T; ++b) s += R[a][b];
  out[tid] = s;
  if (tid == 0) cyc[0] = t1 - t0;
}

int main() {
  const int m = 96;
  double h[m * m];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) h[i * m + j] = (i == j) ? 200.0 : 1.0 / (1.0 + i + j);
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, sizeof(h));
  cudaMalloc(&out, 256 * 8);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  const char* names[] = {"full", "no fix-ups", "no publish switch", "IEEE division"};
  for (int rep = 0; rep < 2; ++rep) {
    sweep_var<0><<<1, 256>>>(A, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %.0f cycles/step\n", names[0], c / 96.0);
    sweep_var<1><<<1, 256>>>(A, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %.0f cycles/step\n", names[1], c / 96.0);
    sweep_var<2><<<1, 256>>>(A, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %.0f cycles/step\n", names[2], c / 96.0);
    sweep_var<3><<<1, 256>>>(A, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-20s %.0f cycles/step\n", names[3], c / 96.0);
  }
  // the production kernel, timed end to end with events
  int* st;
  cudaMalloc(&st, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_block_sweep<<<1, 256>>>(96, A, m, 0, out, st);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) k_block_sweep<<<1, 256>>>(96, A, m, 0, out, st);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("k_block_sweep end to end: %.1f us\n", 1e3 * ms / 20);
  return 0;
}
