// common.cuh -- shared device helpers for the MAS-PNCG sm_100a backend.
//
// FP64 throughout (the reference is float64 everywhere, geometry.py:8).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include <stdexcept>
#include <string>

#include "../../include/maspncg.h"

// ---------------------------------------------------------------------------
// host-side error plumbing: a thrown MpError carries an mp_status

struct MpError : public std::runtime_error {
  int status;
  MpError(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

#define CUDA_CHECK(expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw MpError(MP_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

extern thread_local int64_t* g_launch_counter;
#define LAUNCH_CHECK()                            \
  do {                                            \
    if (g_launch_counter) ++(*g_launch_counter);  \
    CUDA_CHECK(cudaGetLastError());               \
  } while (0)

static inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---------------------------------------------------------------------------
// small dense helpers (row-major 3x3)

struct M3 {
  double a[9];
  __host__ __device__ double& operator()(int r, int c) { return a[3 * r + c]; }
  __host__ __device__ double operator()(int r, int c) const { return a[3 * r + c]; }
};

__device__ __forceinline__ double det3(const M3& m) {
  return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) -
         m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
         m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
}

// cofactor matrix, column c = cross of the other two columns (energy.py:230-235)
__device__ __forceinline__ M3 cof3(const M3& F) {
  M3 c;
  for (int k = 0; k < 3; ++k) {
    int i = (k + 1) % 3, j = (k + 2) % 3;
    // column k = F[:, i] x F[:, j]
    c(0, k) = F(1, i) * F(2, j) - F(2, i) * F(1, j);
    c(1, k) = F(2, i) * F(0, j) - F(0, i) * F(2, j);
    c(2, k) = F(0, i) * F(1, j) - F(1, i) * F(0, j);
  }
  return c;
}

__device__ __forceinline__ M3 mul3(const M3& A, const M3& B) {
  M3 C;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) C(r, c) = A(r, 0) * B(0, c) + A(r, 1) * B(1, c) + A(r, 2) * B(2, c);
  return C;
}

// ---------------------------------------------------------------------------
// 3x3 SVD by one-sided Jacobi (column orthogonalisation of F), singular
// values sorted descending, U and V proper or improper orthogonal.  The
// caller applies the reference's reflection fold (energy.py:184-191).

__device__ __forceinline__ void jacobi_cols(double A[3][3], double V[3][3], int p, int q) {
  double alpha = A[0][p] * A[0][p] + A[1][p] * A[1][p] + A[2][p] * A[2][p];
  double beta = A[0][q] * A[0][q] + A[1][q] * A[1][q] + A[2][q] * A[2][q];
  double gamma = A[0][p] * A[0][q] + A[1][p] * A[1][q] + A[2][p] * A[2][q];
  if (gamma == 0.0 || fabs(gamma) <= 1e-300) return;
  if (fabs(gamma) <= 2.2e-16 * 0.5 * sqrt(alpha * beta)) return;
  double zeta = (beta - alpha) / (2.0 * gamma);
  double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = c * t;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double ap = A[r][p], aq = A[r][q];
    A[r][p] = c * ap - s * aq;
    A[r][q] = s * ap + c * aq;
    double vp = V[r][p], vq = V[r][q];
    V[r][p] = c * vp - s * vq;
    V[r][q] = s * vp + c * vq;
  }
}

__device__ __forceinline__ void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// U, V as column matrices U[r][c]; S descending, all >= 0.
__device__ void svd3(const M3& F, double U[3][3], double S[3], double V[3][3]) {
  double A[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[r][c] = F(r, c);
      V[r][c] = (r == c) ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 12; ++sweep) {
    jacobi_cols(A, V, 0, 1);
    jacobi_cols(A, V, 0, 2);
    jacobi_cols(A, V, 1, 2);
    // convergence: all column pairs orthogonal to working precision
    double n0 = A[0][0] * A[0][0] + A[1][0] * A[1][0] + A[2][0] * A[2][0];
    double n1 = A[0][1] * A[0][1] + A[1][1] * A[1][1] + A[2][1] * A[2][1];
    double n2 = A[0][2] * A[0][2] + A[1][2] * A[1][2] + A[2][2] * A[2][2];
    double g01 = A[0][0] * A[0][1] + A[1][0] * A[1][1] + A[2][0] * A[2][1];
    double g02 = A[0][0] * A[0][2] + A[1][0] * A[1][2] + A[2][0] * A[2][2];
    double g12 = A[0][1] * A[0][2] + A[1][1] * A[1][2] + A[2][1] * A[2][2];
    const double tol = 2.2e-16;
    if (g01 * g01 <= tol * tol * n0 * n1 && g02 * g02 <= tol * tol * n0 * n2 &&
        g12 * g12 <= tol * tol * n1 * n2)
      break;
  }
  double s[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) s[c] = sqrt(A[0][c] * A[0][c] + A[1][c] * A[1][c] + A[2][c] * A[2][c]);
  // sort descending (permute columns of A and V)
  int idx[3] = {0, 1, 2};
  if (s[idx[0]] < s[idx[1]]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
  if (s[idx[1]] < s[idx[2]]) { int t = idx[1]; idx[1] = idx[2]; idx[2] = t; }
  if (s[idx[0]] < s[idx[1]]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
  double Vs[3][3], As[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    S[c] = s[idx[c]];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      Vs[r][c] = V[r][idx[c]];
      As[r][c] = A[r][idx[c]];
    }
  }
  const double smax = S[0];
  const double tiny = (smax > 0.0 ? smax : 1.0) * 1e-300;
  // left singular vectors; complete when singular values vanish
  double u0[3], u1[3], u2[3];
  if (S[0] > tiny) {
    for (int r = 0; r < 3; ++r) u0[r] = As[r][0] / S[0];
  } else {
    u0[0] = 1.0; u0[1] = 0.0; u0[2] = 0.0;
  }
  if (S[1] > tiny) {
    for (int r = 0; r < 3; ++r) u1[r] = As[r][1] / S[1];
  } else {
    // any unit vector orthogonal to u0
    double e[3] = {0.0, 0.0, 0.0};
    int k = (fabs(u0[0]) < 0.6) ? 0 : ((fabs(u0[1]) < 0.6) ? 1 : 2);
    e[k] = 1.0;
    double d = e[0] * u0[0] + e[1] * u0[1] + e[2] * u0[2];
    for (int r = 0; r < 3; ++r) u1[r] = e[r] - d * u0[r];
    double n = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
    for (int r = 0; r < 3; ++r) u1[r] /= n;
  }
  if (S[2] > tiny) {
    for (int r = 0; r < 3; ++r) u2[r] = As[r][2] / S[2];
  } else {
    cross3(u0, u1, u2);
  }
  for (int r = 0; r < 3; ++r) {
    U[r][0] = u0[r];
    U[r][1] = u1[r];
    U[r][2] = u2[r];
#pragma unroll
    for (int c = 0; c < 3; ++c) V[r][c] = Vs[r][c];
  }
}

__device__ __forceinline__ double det_cols(const double U[3][3]) {
  return U[0][0] * (U[1][1] * U[2][2] - U[1][2] * U[2][1]) -
         U[0][1] * (U[1][0] * U[2][2] - U[1][2] * U[2][0]) +
         U[0][2] * (U[1][0] * U[2][1] - U[1][1] * U[2][0]);
}

// signed SVD: reflection folded into the smallest singular value
__device__ __forceinline__ void signed_svd3(const M3& F, double U[3][3], double S[3], double V[3][3]) {
  svd3(F, U, S, V);
  if (det_cols(U) * det_cols(V) < 0.0) {
    U[0][2] = -U[0][2];
    U[1][2] = -U[1][2];
    U[2][2] = -U[2][2];
    S[2] = -S[2];
  }
}

// symmetric 3x3 eigen-decomposition (cyclic Jacobi); Q columns = eigenvectors
__device__ void sym_eig3(double A[3][3], double w[3], double Q[3][3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Q[r][c] = (r == c) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 16; ++sweep) {
    double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    double dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off <= 1e-34 * dia || off == 0.0) break;
    for (int pq = 0; pq < 3; ++pq) {
      int p = (pq == 2) ? 1 : 0;
      int q = (pq == 0) ? 1 : 2;
      double apq = A[p][q];
      if (apq == 0.0) continue;
      double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
      double t = copysign(1.0, theta) / (fabs(theta) + sqrt(1.0 + theta * theta));
      double c = 1.0 / sqrt(1.0 + t * t);
      double s = t * c;
      // A' = J^T A J with J rotating (p,q)
      for (int k = 0; k < 3; ++k) {
        double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - s * akq;
        A[k][q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {
        double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - s * aqk;
        A[q][k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {
        double qkp = Q[k][p], qkq = Q[k][q];
        Q[k][p] = c * qkp - s * qkq;
        Q[k][q] = s * qkp + c * qkq;
      }
    }
  }
  w[0] = A[0][0];
  w[1] = A[1][1];
  w[2] = A[2][2];
}

// ---------------------------------------------------------------------------
// atomics

__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMin(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_min_all(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block reduction helper: per-block partial sums -> part[blockIdx]
template <int BLOCK>
__device__ __forceinline__ void block_sum_store(double v, double* part) {
  __shared__ double sh[BLOCK / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = (threadIdx.x < BLOCK / 32) ? sh[threadIdx.x] : 0.0;
    w = warp_sum(w);
    if (threadIdx.x == 0) part[blockIdx.x] = w;
  }
}

// packed symmetric "cyclic diagonal" layout used for every dense SPD inverse
// (level-0 blocks, Woodbury overlays, coarse levels):
//   entry A(i, (i+s) mod m) for s = 0..floor(m/2), stored diagonal-major:
//   diag s (s < m/2 or m odd): m entries at s*m ; diag m/2 (m even): m/2.
// Total m(m+1)/2 doubles.  Thread i of an apply reads diag_s[i] and
// diag_s[(i-s) mod m] -- both unit-stride across a warp.
__host__ __device__ __forceinline__ int64_t cyc_size(int m) { return (int64_t)m * (m + 1) / 2; }
__host__ __device__ __forceinline__ int64_t cyc_index(int m, int i, int j) {
  // position of A(i,j) (symmetric) in the packed layout
  int s = j - i;
  if (s < 0) s += m;
  int base = i;
  if (2 * s > m) {  // use the transposed representative A(j, i)
    s = m - s;
    base = j;
  }
  if (2 * s == m) base = (i < j) ? i : j;  // half diagonal: A(r, r+m/2), r < m/2
  return (int64_t)s * m + base;
}

// Fixed-order warp gather: the lanes stride over incidences [b, e) of an
// index list and sum buf[3 idx + 0..2]; a shfl_down tree leaves the total in
// lane 0.  The partition and the tree are fixed, so the bits are reproducible,
// and a vertex with thousands of incidences is spread over 32 lanes.
__device__ __forceinline__ void warp_gather3(int b, int e, const int* __restrict__ idx,
                                             const double* __restrict__ buf, double& s0, double& s1, double& s2) {
  const int lane = threadIdx.x & 31;
  s0 = s1 = s2 = 0.0;
  for (int k = b + lane; k < e; k += 32) {
    const double* f = buf + 3 * (int64_t)idx[k];
    s0 += f[0]; s1 += f[1]; s2 += f[2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_down_sync(0xffffffffu, s0, o);
    s1 += __shfl_down_sync(0xffffffffu, s1, o);
    s2 += __shfl_down_sync(0xffffffffu, s2, o);
  }
}

