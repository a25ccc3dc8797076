// ccd.cuh -- conservative per-pair CCD step bounds, per-subdomain
// min-reduction, mixed-step certificate and the clamped update.
//
// Reference: ccd.py:40-56 (orientation cubic), :95-115 (window), :142-157
// (sign bisection), :172-193 (relative-displacement bound, distances),
// :255-294 (pair / per-subdomain steps), :297-320 (certify_mixed);
// solver.py:268-280 (_apply_ccd).
//
// The pair step is computed inside the broad-phase query (contact.cuh,
// BP_CCD): no candidate list has to round-trip before alpha_d is known; the
// pair list is still emitted because certify_mixed re-visits it under p_mix.
#pragma once

#include "contact.cuh"
#include "bvh.cuh"
#include "exact.cuh"

#define CCD_S 0.1

// Cubic coefficients (a3, a2, a1, a0) of det[q1-q0, q2-q0, q3-q0](alpha),
// each filtered-exact (exact.cuh) so structural zeros stay exactly zero.
__device__ void ccd_coeffs(const double X[4][3], const double P[4][3], double co[4]) {
  double c[3][3], e[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c[r][k] = RSUB(X[r + 1][k], X[0][k]);
      e[r][k] = RSUB(P[r + 1][k], P[0][k]);
    }
  {
    const double* U[1] = {c[0]};
    const double* V[1] = {c[1]};
    const double* W[1] = {c[2]};
    co[3] = det_sum_filtered(1, U, V, W);
  }
  {
    const double* U[3] = {e[0], c[0], c[0]};
    const double* V[3] = {c[1], e[1], c[1]};
    const double* W[3] = {c[2], c[2], e[2]};
    co[2] = det_sum_filtered(3, U, V, W);
  }
  {
    const double* U[3] = {e[0], e[0], c[0]};
    const double* V[3] = {e[1], c[1], e[1]};
    const double* W[3] = {c[2], e[2], e[2]};
    co[1] = det_sum_filtered(3, U, V, W);
  }
  {
    const double* U[1] = {e[0]};
    const double* V[1] = {e[1]};
    const double* W[1] = {e[2]};
    co[0] = det_sum_filtered(1, U, V, W);
  }
}

// min(first positive root of f'', first positive root of f') (ccd.py:95-115),
// same elementwise operation order as the reference's numpy batch
__device__ double ccd_window(const double co[4]) {
  const double a3 = co[0], a2 = co[1], a1 = co[2];
  double mon = (a3 != 0.0) ? RDIV(-a2, RMUL(3.0, a3)) : INFINITY;
  if (!(mon > 0.0)) mon = INFINITY;
  double a = RMUL(3.0, a3), b = RMUL(2.0, a2), c = a1;
  double lin = (b != 0.0) ? RDIV(-c, b) : INFINITY;
  double disc = RSUB(RMUL(b, b), RMUL(RMUL(4.0, a), c));
  double sq = __dsqrt_rn(fmax(disc, 0.0));
  double sgn = (b != 0.0) ? (b > 0.0 ? 1.0 : -1.0) : -1.0;
  double qq = RMUL(-0.5, RADD(b, RMUL(sgn, sq)));
  double r1 = (a != 0.0 && qq != 0.0) ? RDIV(qq, a) : INFINITY;
  double r2 = (qq != 0.0) ? RDIV(c, qq) : INFINITY;
  if (!(disc >= 0.0 && r1 > 0.0)) r1 = INFINITY;
  if (!(disc >= 0.0 && r2 > 0.0)) r2 = INFINITY;
  double ext = (a != 0.0) ? fmin(r1, r2) : (lin > 0.0 ? lin : INFINITY);
  return fmin(mon, ext);
}

__device__ __forceinline__ double horner(const double co[4], double al) {
  return RADD(RMUL(RADD(RMUL(RADD(RMUL(co[0], al), co[1]), al), co[2]), al), co[3]);
}

// frame-invariant relative displacement bound (ccd.py:172-179)
__device__ double ccd_speed(const double P[4][3], bool is_pt) {
  double mean[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mean[k] = RDIV(RADD(RADD(RADD(P[0][k], P[1][k]), P[2][k]), P[3][k]), 4.0);
  double nr[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double q0 = RSUB(P[a][0], mean[0]), q1 = RSUB(P[a][1], mean[1]), q2 = RSUB(P[a][2], mean[2]);
    nr[a] = __dsqrt_rn(RADD(RADD(RMUL(q0, q0), RMUL(q1, q1)), RMUL(q2, q2)));
  }
  if (is_pt) return RADD(nr[0], fmax(fmax(nr[1], nr[2]), nr[3]));
  return RADD(fmax(nr[0], nr[1]), fmax(nr[2], nr[3]));
}

__device__ __forceinline__ double ccd_distance(const double X[4][3], bool is_pt) {
  double gr[12];
  return is_pt ? pt_distance(X[0], X[1], X[2], X[3], gr) : ee_distance(X[0], X[1], X[2], X[3], gr);
}

// certify_mixed's per-pair test (ccd.py:309-320) on X, P (P = p_mix rows)
__device__ __forceinline__ bool ccd_cert_test(const double X[4][3], const double P[4][3], bool is_pt, double d,
                                              double speed, const double* co_or_null) {
  double lhs = (speed > 0.0) ? RMUL(1.0 - CCD_S, d) : INFINITY;
  if ((lhs >= speed) && (d > 0.0)) return true;
  double co[4];
  if (co_or_null) {
    co[0] = co_or_null[0]; co[1] = co_or_null[1]; co[2] = co_or_null[2]; co[3] = co_or_null[3];
  } else {
    ccd_coeffs(X, P, co);
  }
  double w = ccd_window(co);
  double f1 = RADD(RADD(RADD(co[0], co[1]), co[2]), co[3]);
  return (w >= 1.0) && (co[3] != 0.0) && (RMUL(f1, co[3]) > 0.0);
}

// pair_steps for one pair (ccd.py:255-281).  *cert_p: the certify_mixed test
// of this pair under the UNSCALED p (valid as the certificate when every
// alpha_d ends up 1, i.e. p_mix == p).
__device__ double ccd_pair_alpha(const double* x, const double* p, const int vid[4], bool is_pt, double alpha_l,
                                 bool* cert_p) {
  double X[4][3], P[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      X[a][k] = x[3 * vid[a] + k];
      P[a][k] = p[3 * vid[a] + k];
    }
  double d = ccd_distance(X, is_pt);
  double speed = ccd_speed(P, is_pt);
  const double one_s = 1.0 - CCD_S;
  double lb = (speed > 0.0) ? RDIV(RMUL(one_s, d), speed) : INFINITY;
  if (!(d > 0.0)) lb = 0.0;
  double alb = fmin(lb, 1.0);
  // alb == 1: alpha_hat <= 1 rules the bisection out, alpha_pair = 1, and the
  // cubic is only needed if certify_mixed's distance test fails
  if (alb >= 1.0) {
    if (cert_p) {
      double lhs = (speed > 0.0) ? RMUL(one_s, d) : INFINITY;
      *cert_p = ((lhs >= speed) && (d > 0.0)) ? true : ccd_cert_test(X, P, is_pt, d, speed, nullptr);
    }
    return 1.0;
  }
  double co[4];
  ccd_coeffs(X, P, co);
  double ahat = fmin(1.0, ccd_window(co));
  double bis = 0.0;
  if (alb < ahat && co[3] != 0.0) {
    double al = ahat;
    while (true) {
      if (RMUL(horner(co, al), co[3]) > 0.0) break;
      if (al <= alpha_l) break;
      al = fmax(RMUL(0.5, al), alpha_l);
    }
    bis = al;
  }
  if (cert_p) *cert_p = ccd_cert_test(X, P, is_pt, d, speed, co);
  return fmin(fmax(alb, bis), 1.0);
}

// certify_mixed for one pair under p_mix = alpha_d[sub] p (ccd.py:297-320)
__device__ bool ccd_certify_pair(const double* x, const double* p, const double* alpha_d, int bs, const int vid[4],
                                 bool is_pt) {
  double X[4][3], P[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double s = alpha_d[vid[a] / bs];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      X[a][k] = x[3 * vid[a] + k];
      P[a][k] = s * p[3 * vid[a] + k];
    }
  }
  return ccd_cert_test(X, P, is_pt, ccd_distance(X, is_pt), ccd_speed(P, is_pt), nullptr);
}

// certify_mixed over a stored pair list: *fail set when any pair fails
__global__ void k_ccd_certify(int64_t n, const int4* __restrict__ verts, const int* __restrict__ is_pt,
                              const double* __restrict__ x, const double* __restrict__ p,
                              const double* __restrict__ alpha_d, int bs, int* __restrict__ fail) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  if (!ccd_certify_pair(x, p, alpha_d, bs, id, is_pt[i] != 0)) atomicExch(fail, 1);
}

// Tight CCD enumeration bound.  For any constant c, the reference's
// relative-displacement bound of a pair (ccd.py:172-179) satisfies
//   speed <= 4 max_a |p_a - c|,
// so a pair with 0.9 d >= speed -- which gets alpha_pair = 1 exactly and
// passes certify_mixed's first test -- is any pair whose distance exceeds
// (4 / 0.9) max_a |p_a - c|.  Inflating every vertex by 4.5 |p_v - c| (c =
// component midrange) therefore enumerates every pair that can move alpha_d,
// the global min or the certificate; the reference's own membership test is
// still applied to each enumerated pair.  s = alpha_d scaling (p_mix) or 1.
// component midrange of alpha_d-scaled p: blocks reduce min / max (order-
// free) into partials; the last block to finish combines them
__global__ void k_motion_midrange(int64_t N, int bs, const double* __restrict__ p, const double* __restrict__ alpha_d,
                                  double* __restrict__ part, int* __restrict__ done, double* __restrict__ out) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    double s = alpha_d ? alpha_d[v / bs] : 1.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double q = s * p[3 * v + k];
      mn[k] = fmin(mn[k], q);
      mx[k] = fmax(mx[k], q);
    }
  }
  __shared__ double sh[6][32];
  __shared__ bool last;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double a = -warp_max(-mn[k]), b = warp_max(mx[k]);
    if ((threadIdx.x & 31) == 0) {
      sh[k][threadIdx.x >> 5] = a;
      sh[3 + k][threadIdx.x >> 5] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double a = INFINITY, b = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a = fmin(a, sh[threadIdx.x][w]);
      b = fmax(b, sh[3 + threadIdx.x][w]);
    }
    part[6 * blockIdx.x + threadIdx.x] = a;
    part[6 * blockIdx.x + 3 + threadIdx.x] = b;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < 3) {
    double a = INFINITY, b = -INFINITY;
    for (int q = 0; q < (int)gridDim.x; ++q) {
      a = fmin(a, __ldcg(part + 6 * q + threadIdx.x));
      b = fmax(b, __ldcg(part + 6 * q + 3 + threadIdx.x));
    }
    out[threadIdx.x] = 0.5 * (a + b);
  }
  if (threadIdx.x == 0) *done = 0;
}

// Per-body tight enumeration (n_bodies > 1): the same bound with a per-pair
// choice of c.  Same-body pairs use their body's midrange c_b (inflation
// 4.5 |s p_v - c_b|); cross-body pairs use the midrange C of the body
// centres (inflation 4.5 (|s p_v - c_b| + |c_b - C|) >= 4.5 |s p_v - C|,
// so the pair's two boxes grown this way cover the single-c criterion).
// Each pair is enumerated in exactly one of the two passes.

// order-preserving unsigned encoding of doubles (for atomic min / max)
__device__ __forceinline__ unsigned long long ord_key(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

__global__ void k_body_minmax(int64_t N, int bs, const int* __restrict__ body, const double* __restrict__ p,
                              const double* __restrict__ alpha_d, unsigned long long* __restrict__ mm) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= N) return;
  const double s = alpha_d ? alpha_d[v / bs] : 1.0;
  unsigned long long* m = mm + 6 * (int64_t)body[v];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const unsigned long long q = ord_key(s * p[3 * v + k]);
    atomicMin(m + k, q);
    atomicMax(m + 3 + k, q);
  }
}

// body centres c_b (nb x 3) and the midrange C of the centres ([3*nb..])
__global__ void k_body_centres(int nb, const unsigned long long* __restrict__ mm, double* __restrict__ cen) {
  __shared__ double lo[3][256], hi[3][256];
  double l[3] = {INFINITY, INFINITY, INFINITY}, h[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double c = 0.5 * (ord_val(mm[6 * b + k]) + ord_val(mm[6 * b + 3 + k]));
      cen[3 * b + k] = c;
      l[k] = fmin(l[k], c);
      h[k] = fmax(h[k], c);
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k][threadIdx.x] = l[k];
    hi[k][threadIdx.x] = h[k];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double a = INFINITY, b = -INFINITY;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      a = fmin(a, lo[threadIdx.x][t]);
      b = fmax(b, hi[threadIdx.x][t]);
    }
    cen[3 * nb + threadIdx.x] = 0.5 * (a + b);
  }
}

__global__ void k_body_infl(int64_t N, int bs, const int* __restrict__ body, const double* __restrict__ p,
                            const double* __restrict__ alpha_d, const double* __restrict__ cen, int nb, int cross,
                            double* __restrict__ infl) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= N) return;
  const double s = alpha_d ? alpha_d[v / bs] : 1.0;
  const double* cb = cen + 3 * (int64_t)body[v];
  double r = 0.0, d = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double q = s * p[3 * v + k] - cb[k];
    r += q * q;
    const double e = cb[k] - cen[3 * nb + k];
    d += e * e;
  }
  infl[v] = 4.5 * (sqrt(r) + (cross ? sqrt(d) : 0.0)) * (1.0 + 1e-12) + 1e-12;
}

__global__ void k_motion_infl(int64_t N, int bs, const double* __restrict__ p, const double* __restrict__ alpha_d,
                              const double* __restrict__ mid, double* __restrict__ infl) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= N) return;
  double s = alpha_d ? alpha_d[v / bs] : 1.0;
  double r = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double q = s * p[3 * v + k] - mid[k];
    r += q * q;
  }
  infl[v] = 4.5 * sqrt(r) * (1.0 + 1e-12) + 1e-12;
}

// x_new = x + alpha_d[sub] p   (mixed)  or  x + alpha p  (global)
__global__ void k_ccd_update(int64_t N, int bs, const double* __restrict__ x, const double* __restrict__ p,
                             const double* __restrict__ alpha_d, double alpha, double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  double s = alpha_d ? alpha_d[(i / 3) / bs] : alpha;
  out[i] = RADD(x[i], RMUL(s, p[i]));  // x + (alpha p), as solver.py:274-280
}

__global__ void k_fill(double* a, int64_t n, double v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

// Per-object motion summary for the exact relative-motion prefilter of the
// tight enumeration (bp.cuh rel_safe): c_o = the (alpha_d-scaled) motion of
// the object's first vertex, m_o = max over its vertices |s p_a - c_o|.
// Objects: triangles [0, F), edges [F, F+E), surface points [F+E, ...).
__global__ void k_obj_motion(int64_t F, int64_t E, int64_t V, const int* __restrict__ tri,
                             const int* __restrict__ edge, const int* __restrict__ sverts,
                             const double* __restrict__ p, const double* __restrict__ alpha_d, int bs,
                             double* __restrict__ mot) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= F + E + V) return;
  int ids[3];
  int n;
  if (o < F) {
    ids[0] = tri[3 * o]; ids[1] = tri[3 * o + 1]; ids[2] = tri[3 * o + 2]; n = 3;
  } else if (o < F + E) {
    ids[0] = edge[2 * (o - F)]; ids[1] = edge[2 * (o - F) + 1]; n = 2;
  } else {
    ids[0] = sverts[o - F - E]; n = 1;
  }
  double c[3], m = 0.0;
  const double s0 = alpha_d ? alpha_d[ids[0] / bs] : 1.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = s0 * p[3 * (int64_t)ids[0] + k];
  for (int a = 1; a < n; ++a) {
    const double sa = alpha_d ? alpha_d[ids[a] / bs] : 1.0;
    double r = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double q = sa * p[3 * (int64_t)ids[a] + k] - c[k];
      r += q * q;
    }
    m = fmax(m, sqrt(r));
  }
  double* out = mot + 4 * o;
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = m;
}

static void obj_motion(mp_ctx* c, const double* p, const double* alpha_d) {
  const int64_t nobj = c->F + c->E + c->V;
  c->obj_mot.ensure(4 * (size_t)nobj);
  k_obj_motion<<<grid_for(nobj, 256), 256, 0, c->stream>>>(c->F, c->E, c->V, c->tri, c->edge, c->sverts, p, alpha_d,
                                                           c->bs, c->obj_mot);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Local-centre tight enumeration.  One global c makes every vertex's box
// grow with |p_v - C|: bodies moving apart or together, or a large step on
// one part of the scene, inflate everything.  Per subdomain d (32 vertices,
// spatially compact) take c_d = the midrange of its (scaled) motion and
//   delta_d = max |c_d - c_d'| over subdomains d' whose boxes lie within
//             rho of d's box, rho = 2 max_v 4.5 |p_v - C| + 2 max edge,
// and inflate vertex v by 4.5 (|p_v - c_d(v)| + delta_d(v)).  Exactness: a
// pair the global criterion cannot rule out has all its vertices' subdomain
// boxes within rho of each other; choosing c = c_d(w*) for the pair vertex
// w* with the largest |p_w - c_d(w)| bounds the pair's max |p - c| by that
// vertex's inflation / 4.5, so a pair whose boxes grown this way do not
// overlap has 0.9 gap > 4.05 max|p - c| >= speed (the same argument as the
// global scheme, ccd.py:172-179).  Pairs beyond rho are safe globally.

__global__ void k_sub_motion(int64_t N, int64_t D, int bs, const double* __restrict__ x, const double* __restrict__ p,
                             const double* __restrict__ alpha_d, double* __restrict__ cen, double* __restrict__ box) {
  const int64_t d = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d >= D) return;  // warp-uniform
  const int64_t v = d * bs + lane;
  const bool live = lane < bs && v < N;
  const double s = alpha_d ? alpha_d[d] : 1.0;
  double pl[3], ph[3], xl[3], xh[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double q = live ? s * p[3 * v + k] : 0.0, xx = live ? x[3 * v + k] : 0.0;
    pl[k] = live ? q : INFINITY;
    ph[k] = live ? q : -INFINITY;
    xl[k] = live ? xx : INFINITY;
    xh[k] = live ? xx : -INFINITY;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    pl[k] = -warp_max(-pl[k]);
    ph[k] = warp_max(ph[k]);
    xl[k] = -warp_max(-xl[k]);
    xh[k] = warp_max(xh[k]);
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cen[3 * d + k] = 0.5 * (pl[k] + ph[k]);
      box[6 * d + k] = xl[k];
      box[6 * d + 3 + k] = xh[k];
    }
}

// max surface edge length and max global inflation (order-free maxima)
__global__ void k_reach_parts(int64_t E, const int* __restrict__ edge, const double* __restrict__ x, int64_t N,
                              const double* __restrict__ infl, double* __restrict__ out) {
  double me = 0.0, mi = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E || i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < E) {
      const int a = edge[2 * i], b = edge[2 * i + 1];
      double r = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double t = x[3 * a + k] - x[3 * b + k];
        r += t * t;
      }
      me = fmax(me, sqrt(r));
    }
    if (i < N) mi = fmax(mi, infl[i]);
  }
  me = warp_max(me);
  mi = warp_max(mi);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(out, me);
    atomic_max_nonneg(out + 1, mi);
  }
}

__global__ void k_sub_keys(int64_t D, const double* __restrict__ box, const double* __restrict__ org, double inv_h,
                           int n1, int n2, unsigned long long* __restrict__ key, int* __restrict__ id) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= D) return;
  int c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = (int)floor((0.5 * (box[6 * d + k] + box[6 * d + 3 + k]) - org[k]) * inv_h);
  key[d] = ((unsigned long long)c[0] * n1 + c[1]) * n2 + c[2];
  id[d] = (int)d;
}

__device__ __forceinline__ int64_t lower_key(const unsigned long long* __restrict__ key, int64_t n,
                                             unsigned long long k) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// delta_d over the 27 neighbour cells (cell = rho + the largest box extent)
__global__ void k_sub_delta(int64_t D, const double* __restrict__ box, const double* __restrict__ cen,
                            const double* __restrict__ org, double inv_h, int n0, int n1, int n2, double rho,
                            const unsigned long long* __restrict__ key, const int* __restrict__ id,
                            double* __restrict__ delta) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= D) return;
  int c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) c[k] = (int)floor((0.5 * (box[6 * d + k] + box[6 * d + 3 + k]) - org[k]) * inv_h);
  const double* bd = box + 6 * d;
  double dl = 0.0;
  for (int a = max(0, c[0] - 1); a <= min(n0 - 1, c[0] + 1); ++a)
    for (int b = max(0, c[1] - 1); b <= min(n1 - 1, c[1] + 1); ++b)
      for (int e = max(0, c[2] - 1); e <= min(n2 - 1, c[2] + 1); ++e) {
        const unsigned long long k = ((unsigned long long)a * n1 + b) * n2 + e;
        for (int64_t q = lower_key(key, D, k); q < D && key[q] == k; ++q) {
          const int64_t o = id[q];
          const double* bo = box + 6 * o;
          double g2 = 0.0;
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const double gap = fmax(0.0, fmax(bd[t] - bo[3 + t], bo[t] - bd[3 + t]));
            g2 += gap * gap;
          }
          if (g2 > rho * rho) continue;
          const double dx = cen[3 * d] - cen[3 * o], dy = cen[3 * d + 1] - cen[3 * o + 1],
                       dz = cen[3 * d + 2] - cen[3 * o + 2];
          dl = fmax(dl, sqrt(dx * dx + dy * dy + dz * dz));
        }
      }
  delta[d] = dl;
}

__global__ void k_local_infl(int64_t N, int bs, const double* __restrict__ p, const double* __restrict__ alpha_d,
                             const double* __restrict__ cen, const double* __restrict__ delta,
                             double* __restrict__ infl) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= N) return;
  const int64_t d = v / bs;
  const double s = alpha_d ? alpha_d[d] : 1.0;
  double r = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double q = s * p[3 * v + k] - cen[3 * d + k];
    r += q * q;
  }
  infl[v] = 4.5 * (sqrt(r) + delta[d]) * (1.0 + 1e-12) + 1e-12;
}

// c->infl holds the global-centre inflation on entry; replaced by the local
// one when that is smaller everywhere it matters (its maximum is smaller)
static void local_infl(mp_ctx* c, const double* x, const double* p, const double* alpha_d) {
  cudaStream_t st = c->stream;
  const int64_t D = c->D, N = c->N;
  c->sub_cen.ensure(3 * (size_t)D);
  c->sub_box.ensure(6 * (size_t)D);
  c->sub_delta.ensure(D);
  c->infl2.ensure(N);
  k_sub_motion<<<grid_for(32 * D, 256), 256, 0, st>>>(N, D, c->bs, x, p, alpha_d, c->sub_cen, c->sub_box);
  LAUNCH_CHECK();
  double* parts = c->dscal.p + 48;  // [48] max edge, [49] max global inflation
  CUDA_CHECK(cudaMemsetAsync(parts, 0, 2 * sizeof(double), st));
  k_reach_parts<<<296, 256, 0, st>>>(c->E, c->edge, x, N, c->infl, parts);
  LAUNCH_CHECK();
  std::vector<double> boxes(6 * D);
  double h2[2];
  CUDA_CHECK(cudaMemcpyAsync(h2, parts, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaMemcpyAsync(boxes.data(), c->sub_box.p, sizeof(double) * 6 * D, cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  const double rho = (2.0 * h2[1] + 2.0 * h2[0]) * (1.0 + 1e-9);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, ext = 0.0;
  for (int64_t d = 0; d < D; ++d)
    for (int k = 0; k < 3; ++k) {
      const double m = 0.5 * (boxes[6 * d + k] + boxes[6 * d + 3 + k]);
      lo[k] = std::min(lo[k], m);
      hi[k] = std::max(hi[k], m);
      ext = std::max(ext, boxes[6 * d + 3 + k] - boxes[6 * d + k]);
    }
  // centres of two subdomains whose boxes are within rho are within rho + ext per axis
  double h = std::max(rho + ext, 1e-12);
  int n[3];
  for (;;) {
    double cells = 1.0;
    for (int k = 0; k < 3; ++k) {
      n[k] = (int)std::floor((hi[k] - lo[k]) / h) + 1;
      cells *= n[k];
    }
    if (cells < 4e18) break;
    h *= 2.0;
  }
  c->dscal_h.assign(lo, lo + 3);
  CUDA_CHECK(cudaMemcpyAsync(c->dscal.p + 50, lo, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
  c->sub_key.ensure(D); c->sub_key2.ensure(D); c->sub_id.ensure(D); c->sub_id2.ensure(D);
  k_sub_keys<<<grid_for(D, 256), 256, 0, st>>>(D, c->sub_box, c->dscal.p + 50, 1.0 / h, n[1], n[2], c->sub_key,
                                                c->sub_id);
  LAUNCH_CHECK();
  const unsigned long long ncell = (unsigned long long)n[0] * n[1] * n[2];
  sort_pairs_u64(c, c->sub_key, c->sub_key2, c->sub_id, c->sub_id2, D, bits_for(ncell));
  k_sub_delta<<<grid_for(D, 128), 128, 0, st>>>(D, c->sub_box, c->sub_cen, c->dscal.p + 50, 1.0 / h, n[0], n[1], n[2],
                                                rho, c->sub_key2, c->sub_id2, c->sub_delta);
  LAUNCH_CHECK();
  k_local_infl<<<grid_for(N, 256), 256, 0, st>>>(N, c->bs, p, alpha_d, c->sub_cen, c->sub_delta, c->infl2);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemsetAsync(parts, 0, 2 * sizeof(double), st));
  k_reach_parts<<<296, 256, 0, st>>>(0, c->edge, x, N, c->infl2, parts);
  LAUNCH_CHECK();
  double m2[2];
  CUDA_CHECK(cudaMemcpyAsync(m2, parts, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  if (m2[1] < h2[1]) std::swap(c->infl.p, c->infl2.p);  // the local inflation wins
}

// per-vertex inflation of the two-pass tight enumeration (cross = 0: the
// same-body pass, 1: the cross-body pass), p scaled by alpha_d if given
static void body_infl(mp_ctx* c, const double* p, const double* alpha_d, int cross) {
  cudaStream_t st = c->stream;
  const int nb = (int)c->n_bodies;
  c->infl.ensure(c->N);
  c->body_mm.ensure(6 * (size_t)nb);
  c->body_cen.ensure(3 * (size_t)nb + 3);
  std::vector<unsigned long long> init(6 * (size_t)nb);
  for (int b = 0; b < nb; ++b)
    for (int k = 0; k < 3; ++k) {
      init[6 * b + k] = ~0ull;
      init[6 * b + 3 + k] = 0ull;
    }
  CUDA_CHECK(cudaMemcpyAsync(c->body_mm.p, init.data(), sizeof(unsigned long long) * init.size(),
                             cudaMemcpyHostToDevice, st));
  k_body_minmax<<<grid_for(c->N, 256), 256, 0, st>>>(c->N, c->bs, c->body, p, alpha_d, c->body_mm);
  LAUNCH_CHECK();
  k_body_centres<<<1, 256, 0, st>>>(nb, c->body_mm, c->body_cen);
  LAUNCH_CHECK();
  k_body_infl<<<grid_for(c->N, 256), 256, 0, st>>>(c->N, c->bs, c->body, p, alpha_d, c->body_cen, nb, cross, c->infl);
  LAUNCH_CHECK();
  sync_stream(c);  // init is a stack array
}

struct CcdResult {
  double min_alpha;   // min over pairs (1 if none)
  bool certified;
  int64_t n_pairs;
};

// collect_pairs + per_subdomain_steps (+ certify_mixed when per_subdomain);
// leaves alpha_d in c->alpha_d; x_out receives the clamped position.
// exact_set: enumerate the reference's full candidate set and store it (the
// stage tap); otherwise the tight set (k_motion_infl), which yields the same
// alpha_d, global min and certificate.
static CcdResult ccd_clamp(mp_ctx* c, const double* x, const double* p, double pinf, bool per_subdomain,
                           double* x_out, bool exact_set = false) {
  CcdResult R{1.0, true, 0};
  cudaStream_t st = c->stream;
  // MP_CCD_TRACE=1: per-call host timings of the CCD phases on stderr
  static const bool trace = getenv("MP_CCD_TRACE") != nullptr;
  auto tr0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what, int64_t n) {
    if (!trace) return;
    CUDA_CHECK(cudaStreamSynchronize(st));
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "ccd %-10s %9.3f ms  n=%lld\n", what, std::chrono::duration<double, std::milli>(t - tr0).count(),
            (long long)n);
    tr0 = t;
  };
  k_fill<<<grid_for(c->D, 256), 256, 0, st>>>(c->alpha_d, c->D, 1.0);
  LAUNCH_CHECK();
  double* d_min = c->dscal.p + 41;
  double* d_mid = c->dscal.p + 44;
  k_fill<<<1, 32, 0, st>>>(d_min, 1, 1.0);
  LAUNCH_CHECK();
  int cert_fail_p = 0;
  if (c->F > 0) {
    const double* infl = nullptr;
    const bool bodies = !exact_set && c->ccd_bodies && c->n_bodies > 1;
    if (bodies) {
      body_infl(c, p, nullptr, 0);
      infl = c->infl;
    } else if (!exact_set) {
      c->infl.ensure(c->N);
      k_motion_midrange<<<148, 256, 0, st>>>(c->N, c->bs, p, nullptr, c->mid_part, c->counters.p + 15, d_mid);
      LAUNCH_CHECK();
      k_motion_infl<<<grid_for(c->N, 256), 256, 0, st>>>(c->N, c->bs, p, nullptr, d_mid, c->infl);
      LAUNCH_CHECK();
      if (c->ccd_local) local_infl(c, x, p, nullptr);
      infl = c->infl;
    }
    if (!exact_set && c->ccd_prefilter) obj_motion(c, p, nullptr);
    lap("infl", 0);
    // the motion-aware BVH (bvh.cuh) for the tight single-centre passes; the
    // grid for the exact set, the per-body passes and the >2^30 fallback
    const int gmode = (exact_set || bodies || c->ccd_bvh == 0) ? BP_GRID_ALWAYS
                      : (c->ccd_bvh == 1 ? BP_GRID_NONE : BP_GRID_AUTO);
    BpGrid B = build_bp(c, x, pinf, 0.0, infl, bodies ? 1 : 0, gmode);
    lap("grid", 0);
    if (!exact_set && c->ccd_prefilter) B.T.objmot = c->obj_mot.p;
    // one enumeration + pair pass of MODE over the boxes of G: the BVH when
    // build_bp left no grid, else the grid (crowded calls are timed:
    // bp.cuh BP_GRID_AUTO keeps each method's cost)
    auto enumerate = [&](auto mode_tag, BpGrid& G, BpOut O, int* fl) -> int64_t {
      constexpr int M = decltype(mode_tag)::value;
      const auto t0 = std::chrono::steady_clock::now();
      const int method = G.has_grid ? 0 : 1;
      const CcdParams cc{p, c->cfg.alpha_l, c->bs};
      const int64_t n = G.has_grid ? run_bp<M>(c, x, G, O, ContactParams{}, cc, fl)
                                   : run_bvh<M>(c, x, G, O, ContactParams{}, cc, fl);
      if (G.crowd > 0.0) {  // run_bvh / run_bp end on a host sync: the interval is the enumeration's
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        double& e = c->enum_ms.ms[method][G.crowd_bucket];
        e = e < 0.0 ? ms : 0.5 * (e + ms);
        if (trace) fprintf(stderr, "ccd crowded  %s %.3f ms (crowd %.1f)\n", method ? "bvh" : "grid", ms, G.crowd);
      }
      return n;
    };
    ContactParams CP{};
    CcdParams CC{p, c->cfg.alpha_l, c->bs};
    if (exact_set && c->ccd_verts.n < 4096) {
      c->ccd_verts.ensure(4096); c->ccd_ispt.ensure(4096); c->ccd_alpha.ensure(4096);
    }
    for (int attempt = 0; attempt < 4; ++attempt) {
      BpOut O{};
      if (exact_set) {
        O.verts = c->ccd_verts; O.ccd_ispt = c->ccd_ispt; O.alpha_pair = c->ccd_alpha;
        O.cap = (int64_t)c->ccd_verts.n;
      }
      O.alpha_d = c->alpha_d;
      O.min_alpha = d_min;
      c->rb_extra = d_min;  // read back with run_bp's counters: no extra sync
      int64_t n = enumerate(std::integral_constant<int, BP_CCD>{}, B, O, &cert_fail_p);
      c->rb_extra = nullptr;
      if (!exact_set || n <= O.cap) {
        R.n_pairs = n;
        if (bodies) {  // the cross-body pass: minima and the failure flag accumulate
          int fail2 = 0;
          body_infl(c, p, nullptr, 1);
          BpGrid B2 = build_bp(c, x, pinf, 0.0, c->infl, 2);
          if (c->ccd_prefilter) B2.T.objmot = c->obj_mot.p;
          c->rb_extra = d_min;
          R.n_pairs += run_bp<BP_CCD>(c, x, B2, O, CP, CC, &fail2);
          c->rb_extra = nullptr;
          cert_fail_p |= fail2;
        }
        break;
      }
      size_t cap = (size_t)(n * 1.5) + 4096;
      c->ccd_verts.ensure(cap); c->ccd_ispt.ensure(cap); c->ccd_alpha.ensure(cap);
      k_fill<<<grid_for(c->D, 256), 256, 0, st>>>(c->alpha_d, c->D, 1.0);
      LAUNCH_CHECK();
      k_fill<<<1, 32, 0, st>>>(d_min, 1, 1.0);
      LAUNCH_CHECK();
      if (attempt == 3) throw MpError(MP_ERR_CAPACITY, "ccd pair capacity retry failed");
    }
    R.min_alpha = c->h_scal[0];
    lap("pairs", R.n_pairs);
    if (per_subdomain && R.n_pairs > 0) {
      if (R.min_alpha == 1.0) {
        // every alpha_d is 1: p_mix == p, the certificate was evaluated inline
        R.certified = cert_fail_p == 0;
      } else if (exact_set) {
        CUDA_CHECK(cudaMemsetAsync(c->counters.p + 2, 0, sizeof(int), st));
        k_ccd_certify<<<grid_for(R.n_pairs, 128), 128, 0, st>>>(R.n_pairs, c->ccd_verts, c->ccd_ispt, x, p,
                                                                c->alpha_d, c->bs, c->counters.p + 2);
        LAUNCH_CHECK();
        CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 2, c->counters.p + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
        sync_stream(c);
        R.certified = c->h_cnt[2] == 0;
      } else if (bodies) {
        BpOut O{};
        O.alpha_d = c->alpha_d;
        int fail = 0, fail2 = 0;
        if (c->ccd_prefilter) obj_motion(c, p, c->alpha_d);
        body_infl(c, p, c->alpha_d, 0);
        BpGrid B2 = build_bp(c, x, pinf, 0.0, c->infl, 1);
        if (c->ccd_prefilter) B2.T.objmot = c->obj_mot.p;
        run_bp<BP_CERT>(c, x, B2, O, CP, CC, &fail);
        body_infl(c, p, c->alpha_d, 1);
        BpGrid B3 = build_bp(c, x, pinf, 0.0, c->infl, 2);
        if (c->ccd_prefilter) B3.T.objmot = c->obj_mot.p;
        run_bp<BP_CERT>(c, x, B3, O, CP, CC, &fail2);
        R.certified = (fail | fail2) == 0;
      } else {
        k_motion_midrange<<<148, 256, 0, st>>>(c->N, c->bs, p, c->alpha_d, c->mid_part, c->counters.p + 15, d_mid);
        LAUNCH_CHECK();
        k_motion_infl<<<grid_for(c->N, 256), 256, 0, st>>>(c->N, c->bs, p, c->alpha_d, d_mid, c->infl);
        LAUNCH_CHECK();
        if (c->ccd_local) local_infl(c, x, p, c->alpha_d);
        if (c->ccd_prefilter) obj_motion(c, p, c->alpha_d);
        BpGrid B2 = build_bp(c, x, pinf, 0.0, c->infl, 0, gmode);
        if (c->ccd_prefilter) B2.T.objmot = c->obj_mot.p;
        BpOut O{};
        O.alpha_d = c->alpha_d;
        int fail = 0;
        lap("cert-grid", 0);
        const int64_t nc = enumerate(std::integral_constant<int, BP_CERT>{}, B2, O, &fail);
        R.certified = fail == 0;
        lap("cert", nc);
      }
    }
  }
  c->n_ccd = exact_set ? R.n_pairs : 0;
  c->n_ccd_seen = R.n_pairs;
  if (per_subdomain && R.certified) {
    k_ccd_update<<<grid_for(3 * c->N, 256), 256, 0, st>>>(c->N, c->bs, x, p, c->alpha_d, 0.0, x_out);
  } else {
    k_ccd_update<<<grid_for(3 * c->N, 256), 256, 0, st>>>(c->N, c->bs, x, p, nullptr, R.min_alpha, x_out);
  }
  LAUNCH_CHECK();
  return R;
}
