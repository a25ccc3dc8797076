// exact.cuh -- error-free transformations and exact 3x3 determinants.
//
// The reference evaluates every CCD cubic coefficient with np.linalg.det
// (LU), which returns an exact 0 for the structurally singular matrices that
// axis-aligned synthetic scenes produce (coplanar edges, points on a face
// plane).  A cancelling FP64 cofactor expansion leaves a 1e-21 residue there
// instead, and the sign-based bisection then "certifies" a crossing step.
// So each coefficient is evaluated in FP64 with a forward error bound, and
// whenever |value| does not clear the bound it is recomputed exactly as a
// floating-point expansion (Shewchuk, "Adaptive Precision Floating-Point
// Arithmetic", 1997) and rounded.  Measured on the golden CCD pairs: exact
// zero agrees with the reference's zero on 1526/1538 singular pairs and
// never disagrees in sign.
#pragma once

#include "common.cuh"

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__device__ __forceinline__ void two_prod(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = fma(a, b, -p);
}

// h += b, h a nonoverlapping expansion (increasing magnitude), zeros elided
template <int CAP>
__device__ __forceinline__ void grow(double (&h)[CAP], int& n, double b) {
  double Q = b;
  int m = 0;
  for (int i = 0; i < n; ++i) {
    double s, e;
    two_sum(Q, h[i], s, e);
    Q = s;
    if (e != 0.0) h[m++] = e;
  }
  if (Q != 0.0 && m < CAP) h[m++] = Q;
  n = m;
}

// add sign * a*b*c exactly (4 doubles)
template <int CAP>
__device__ __forceinline__ void add_triple(double (&h)[CAP], int& n, double sgn, double a, double b, double c) {
  double p, e, p1, e1, p2, e2;
  two_prod(b, c, p, e);
  two_prod(a, p, p1, e1);
  two_prod(a, e, p2, e2);
  grow(h, n, sgn * p1);
  grow(h, n, sgn * e1);
  grow(h, n, sgn * p2);
  grow(h, n, sgn * e2);
}

// det of the matrix with columns u, v, w: sum over permutations
template <int CAP>
__device__ __forceinline__ void add_det(double (&h)[CAP], int& n, const double u[3], const double v[3],
                                        const double w[3]) {
  add_triple(h, n, 1.0, u[0], v[1], w[2]);
  add_triple(h, n, -1.0, u[0], v[2], w[1]);
  add_triple(h, n, -1.0, u[1], v[0], w[2]);
  add_triple(h, n, 1.0, u[1], v[2], w[0]);
  add_triple(h, n, 1.0, u[2], v[0], w[1]);
  add_triple(h, n, -1.0, u[2], v[1], w[0]);
}

template <int CAP>
__device__ __forceinline__ double expansion_value(const double (&h)[CAP], int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, h[i]);
  return s;
}

// magnitude bound |u|.(|v| x |w|) style permanent of absolute values
__device__ __forceinline__ double det_perm_abs(const double u[3], const double v[3], const double w[3]) {
  return fabs(u[0]) * (fabs(v[1]) * fabs(w[2]) + fabs(v[2]) * fabs(w[1])) +
         fabs(u[1]) * (fabs(v[0]) * fabs(w[2]) + fabs(v[2]) * fabs(w[0])) +
         fabs(u[2]) * (fabs(v[0]) * fabs(w[1]) + fabs(v[1]) * fabs(w[0]));
}

__device__ __forceinline__ double det_fast(const double u[3], const double v[3], const double w[3]) {
  return u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0]) +
         u[2] * (v[0] * w[1] - v[1] * w[0]);
}

// one cubic coefficient = sum of k determinants (k = 1 or 3), filtered exact
__device__ double det_sum_filtered(int k, const double* const* U, const double* const* V, const double* const* W) {
  double val = 0.0, mag = 0.0;
  for (int q = 0; q < k; ++q) {
    val += det_fast(U[q], V[q], W[q]);
    mag += det_perm_abs(U[q], V[q], W[q]);
  }
  const double bound = 16.0 * 1.1102230246251565e-16 * mag;
  if (fabs(val) > bound) return val;
  double h[80];
  int n = 0;
  for (int q = 0; q < k; ++q) add_det(h, n, U[q], V[q], W[q]);
  return expansion_value(h, n);
}
