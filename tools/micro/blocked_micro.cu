// Per-phase clock breakdown of sweep_blocked on one 96x96 SPD block.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2604_19892_b200/csrc/mas.cuh"

template <class LOAD>
__device__ bool sweep_timed(LOAD load, int m, double* sm, double (&R)[SWEEP_T][SWEEP_T], long long* ph) {
  long long tt = clock64();
#define LAP(q) do { __syncthreads(); long long n_ = clock64(); if (threadIdx.x == 0) ph[q] += n_ - tt; tt = n_; } while (0)
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double* pk = sm;              // 2 x 16 pivot-row broadcast, [32] = SPD flag
  double* pm = sm + 40;         // 16 x 16 (-P^-1)
  double* acol = pm + 256;            // 96 x 16: A(i, 16K + d), row stride SWEEP_LD
  double* wsm = acol + 96 * SWEEP_LD; // 96 x 16: W(i, c), row stride SWEEP_LD
#pragma unroll
  for (int a = 0; a < SWEEP_T; ++a)
#pragma unroll
    for (int b = 0; b < SWEEP_T; ++b) {
      int i = tr + 16 * a, j = tc + 16 * b;
      R[a][b] = (i < m && j < m) ? load(i, j) : (i == j ? 1.0 : 0.0);
    }
  const int np = (m + 15) >> 4;
#pragma unroll
  for (int K = 0; K < SWEEP_T; ++K) {
    if (K >= np) break;
    LAP(0);
    // (1) sweep the pivot block P = R[K][K]: staged in smem, swept by warp 0
    //     alone (lane l holds row l/2, columns 8 (l%2) .. +8) with warp-level
    //     broadcasts -- no CTA barrier inside the 16 pivot steps
    pm[tr * 16 + tc] = R[K][K];
    __syncthreads();
    if (tid < 32) {
      // lane holds P(r, c0 .. c0+7); the pivot row is broadcast by register
      // shuffles (the k loop is unrolled so every register index is static)
      const int lane = tid, r = lane >> 1, c0 = (lane & 1) * 8;
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = pm[r * 16 + c0 + q];
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int kq = k & 7, kh = k >> 3;
        const double piv = __shfl_sync(WARP_ALL, v[kq], 2 * k + kh);
        const double pik = __shfl_sync(WARP_ALL, v[kq], 2 * r + kh);  // P(r, k)
        double cj[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) cj[q] = __shfl_sync(WARP_ALL, v[q], 2 * k + (lane & 1));  // P(k, c0 + q)
        ok = ok && (piv > 0.0);
        const double inv = fast_rcp(piv);
        const double ci = pik * inv;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c = c0 + q;
          double t = fma(-ci, cj[q], v[q]);
          if (r == k) t = cj[q] * inv;
          if (c == k) t = (r == k) ? -inv : ci;
          v[q] = t;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) pm[r * 16 + c0 + q] = v[q];
      if (lane == 0) pk[32] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    if (pk[32] == 0.0) return false;  // uniform across the CTA
    const double p = pm[tr * 16 + tc];
    R[K][K] = p;
    LAP(1);
    // (2) stage the column panel A(i, K.) (i outside K); -P^-1 is in pm
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a)
      if (a != K) acol[(tr + 16 * a) * SWEEP_LD + tc] = R[a][K];
    __syncthreads();
    // (3) W(i, c) = A_iK P^-1 = -sum_d A(i, Kd) pm(d, c), c = tc
    double w[SWEEP_T];
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a) {
      w[a] = 0.0;
      if (a == K) continue;
      const double* ar = acol + (tr + 16 * a) * SWEEP_LD;
#pragma unroll
      for (int d = 0; d < 16; ++d) w[a] = fma(-ar[d], pm[d * 16 + tc], w[a]);
      wsm[(tr + 16 * a) * SWEEP_LD + tc] = w[a];
    }
    __syncthreads();
    LAP(2);
    // (4) A_ij -= W(i, .) . A(j, K.) for i, j outside K
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      double wi[SWEEP_T], aj[SWEEP_T];
#pragma unroll
      for (int a = 0; a < SWEEP_T; ++a) {
        wi[a] = (a == K) ? 0.0 : wsm[(tr + 16 * a) * SWEEP_LD + d];
        aj[a] = (a == K) ? 0.0 : acol[(tc + 16 * a) * SWEEP_LD + d];
      }
#pragma unroll
      for (int a = 0; a < SWEEP_T; ++a) {
        if (a == K) continue;
#pragma unroll
        for (int b = 0; b < SWEEP_T; ++b)
          if (b != K) R[a][b] = fma(-wi[a], aj[b], R[a][b]);
      }
    }
    LAP(3);
    // (5) block column K <- W, block row K <- W^T
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a)
      if (a != K) R[a][K] = w[a];
#pragma unroll
    for (int b = 0; b < SWEEP_T; ++b)
      if (b != K) R[K][b] = wsm[(tc + 16 * b) * SWEEP_LD + tr];
    __syncthreads();  // acol / wsm / pm are rewritten by the next panel
    LAP(4);
  }
  return true;
}

__global__ void run2(const double* A, double* out, long long* ph) {
  __shared__ double swsm[SWEEP_SMEM];
  double R[SWEEP_T][SWEEP_T];
  auto load = [&](int i, int j) -> double { return A[i * 96 + j]; };
  bool ok = sweep_timed(load, 96, swsm, R, ph);
  double s = 0;
  for (int a = 0; a < SWEEP_T; ++a) for (int b = 0; b < SWEEP_T; ++b) s += R[a][b];
  out[threadIdx.x] = s + ok;
}

__global__ void run(const double* A, double* out, long long* cyc) {
  __shared__ double swsm[SWEEP_SMEM];
  double R[SWEEP_T][SWEEP_T];
  auto load = [&](int i, int j) -> double { return A[i * 96 + j]; };
  long long t0 = clock64();
  bool ok = sweep_blocked(load, 96, swsm, R);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < SWEEP_T; ++a)
    for (int b = 0; b < SWEEP_T; ++b) s += R[a][b];
  out[threadIdx.x] = s + ok;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  const int m = 96;
  static double h[m * m];
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) h[i * m + j] = (i == j) ? 200.0 : 1.0 / (1.0 + i + j);
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, sizeof(h));
  cudaMalloc(&out, 256 * 8);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  for (int rep = 0; rep < 3; ++rep) {
    run<<<1, 256>>>(A, out, cyc);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("sweep_blocked: %lld cycles (%.1f us at 1.965 GHz)\n", c, c / 1965.0);
  }
  long long* ph;
  cudaMalloc(&ph, 8 * 8);
  cudaMemset(ph, 0, 64);
  run2<<<1, 256>>>(A, out, ph);
  long long hp[8];
  cudaMemcpy(hp, ph, 64, cudaMemcpyDeviceToHost);
  const char* nm[] = {"load+pre", "P sweep (warp 0)", "stage+W", "update", "fix"};
  for (int q = 0; q < 5; ++q) printf("%-18s %lld cycles\n", nm[q], hp[q]);
  return 0;
}
