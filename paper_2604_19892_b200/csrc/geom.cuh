// geom.cuh -- point-triangle / edge-edge distances and the barrier.
//
// Written with explicit round-to-nearest intrinsics (no FMA contraction) in
// the same operation order as the reference's numpy batches
// (geometry.py:209-323), so distances -- and therefore the d < d_hat
// activation test and the penetration test -- are bit-identical.
#pragma once

#include "common.cuh"

#define RMUL(a, b) __dmul_rn((a), (b))
#define RADD(a, b) __dadd_rn((a), (b))
#define RSUB(a, b) __dsub_rn((a), (b))
#define RDIV(a, b) __ddiv_rn((a), (b))

__device__ __forceinline__ double rdot3(const double a[3], const double b[3]) {
  return RADD(RADD(RMUL(a[0], b[0]), RMUL(a[1], b[1])), RMUL(a[2], b[2]));
}

__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// pt_distance_batch (geometry.py:209-284); grad rows (p, t0, t1, t2)
__device__ double pt_distance(const double p[3], const double t0[3], const double t1[3], const double t2[3],
                              double grad[12]) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ab[i] = RSUB(t1[i], t0[i]);
    ac[i] = RSUB(t2[i], t0[i]);
    ap[i] = RSUB(p[i], t0[i]);
    bp[i] = RSUB(p[i], t1[i]);
    cp[i] = RSUB(p[i], t2[i]);
  }
  double d1 = rdot3(ab, ap), d2 = rdot3(ac, ap);
  double d3 = rdot3(ab, bp), d4 = rdot3(ac, bp);
  double d5 = rdot3(ab, cp), d6 = rdot3(ac, cp);
  double vc = RSUB(RMUL(d1, d4), RMUL(d3, d2));
  double vb = RSUB(RMUL(d5, d2), RMUL(d1, d6));
  double va = RSUB(RMUL(d3, d6), RMUL(d5, d4));
  double w0, w1, w2;
  if (d1 <= 0.0 && d2 <= 0.0) {
    w0 = 1.0; w1 = 0.0; w2 = 0.0;
  } else if (d3 >= 0.0 && d4 <= d3) {
    w0 = 0.0; w1 = 1.0; w2 = 0.0;
  } else if (d6 >= 0.0 && d5 <= d6) {
    w0 = 0.0; w1 = 0.0; w2 = 1.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = RDIV(d1, RSUB(d1, d3));
    w0 = RSUB(1.0, v); w1 = v; w2 = 0.0;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double v = RDIV(d2, RSUB(d2, d6));
    w0 = RSUB(1.0, v); w1 = 0.0; w2 = v;
  } else if (va <= 0.0 && RSUB(d4, d3) >= 0.0 && RSUB(d5, d6) >= 0.0) {
    double num = RSUB(d4, d3);
    double v = RDIV(num, RADD(num, RSUB(d5, d6)));
    w0 = 0.0; w1 = RSUB(1.0, v); w2 = v;
  } else {
    double denom = RADD(RADD(va, vb), vc);
    double v = RDIV(vb, denom), ww = RDIV(vc, denom);
    w0 = RSUB(RSUB(1.0, v), ww); w1 = v; w2 = ww;
  }
  double diff[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double cl = RADD(RADD(RMUL(w0, t0[i]), RMUL(w1, t1[i])), RMUL(w2, t2[i]));
    diff[i] = RSUB(p[i], cl);
  }
  double d = __dsqrt_rn(rdot3(diff, diff));
  double u[3] = {0.0, 0.0, 0.0};
  if (d > 0.0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) u[i] = RDIV(diff[i], d);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    grad[i] = u[i];
    grad[3 + i] = RMUL(-w0, u[i]);
    grad[6 + i] = RMUL(-w1, u[i]);
    grad[9 + i] = RMUL(-w2, u[i]);
  }
  return d;
}

// ee_distance_batch (geometry.py:287-323); grad rows (a0, a1, b0, b1)
__device__ double ee_distance(const double a0[3], const double a1[3], const double b0[3], const double b1[3],
                              double grad[12]) {
  double d1[3], d2[3], r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    d1[i] = RSUB(a1[i], a0[i]);
    d2[i] = RSUB(b1[i], b0[i]);
    r[i] = RSUB(a0[i], b0[i]);
  }
  double a = rdot3(d1, d1), e = rdot3(d2, d2), f = rdot3(d2, r), c = rdot3(d1, r), b = rdot3(d1, d2);
  double denom = RSUB(RMUL(a, e), RMUL(b, b));
  double s = 0.0;
  if (denom > 0.0) s = clip01(RDIV(RSUB(RMUL(b, f), RMUL(c, e)), denom));
  double t = RDIV(RADD(RMUL(b, s), f), e);
  bool low = t < 0.0, high = t > 1.0;
  t = clip01(t);
  if (low) s = clip01(RDIV(-c, a));
  if (high) s = clip01(RDIV(RSUB(b, c), a));
  double diff[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double ca = RADD(a0[i], RMUL(s, d1[i]));
    double cb = RADD(b0[i], RMUL(t, d2[i]));
    diff[i] = RSUB(ca, cb);
  }
  double d = __dsqrt_rn(rdot3(diff, diff));
  double u[3] = {0.0, 0.0, 0.0};
  if (d > 0.0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) u[i] = RDIV(diff[i], d);
  }
  double oms = RSUB(1.0, s), omt = RSUB(1.0, t);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    grad[i] = RMUL(oms, u[i]);
    grad[3 + i] = RMUL(s, u[i]);
    grad[6 + i] = RMUL(-omt, u[i]);
    grad[9 + i] = RMUL(-t, u[i]);
  }
  return d;
}

// kappa * (b, b', b'') of b(d) = -(d - dh)^2 ln(d/dh) inside (0, dh)
// (contact.py:34-64); caller guarantees 0 < d < dh
__device__ __forceinline__ void barrier3(double d, double dh, double kappa, double* b, double* db, double* ddb) {
  double t = d - dh;
  double ln = log(d / dh);
  if (b) *b = kappa * (-t * t * ln);
  if (db) *db = kappa * (-2.0 * t * ln - t * t / d);
  if (ddb) *ddb = kappa * (-2.0 * ln - 4.0 * t / d + t * t / (d * d));
}
