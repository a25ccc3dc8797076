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

// pair_steps for one pair (ccd.py:255-281)
__device__ double ccd_pair_alpha(const double* x, const double* p, const int vid[4], bool is_pt, double alpha_l) {
  double X[4][3], P[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      X[a][k] = x[3 * vid[a] + k];
      P[a][k] = p[3 * vid[a] + k];
    }
  double co[4];
  ccd_coeffs(X, P, co);
  double d = ccd_distance(X, is_pt);
  double speed = ccd_speed(P, is_pt);
  const double one_s = 1.0 - CCD_S;
  double lb = (speed > 0.0) ? RDIV(RMUL(one_s, d), speed) : INFINITY;
  if (!(d > 0.0)) lb = 0.0;
  double alb = fmin(lb, 1.0);
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
  return fmin(fmax(alb, bis), 1.0);
}

// certify_mixed (ccd.py:297-320): flag[0] cleared when any pair fails
__global__ void k_ccd_certify(int64_t n, const int4* __restrict__ verts, const int* __restrict__ is_pt,
                              const double* __restrict__ x, const double* __restrict__ p,
                              const double* __restrict__ alpha_d, int bs, int* __restrict__ fail) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  double X[4][3], P[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double s = alpha_d[id[a] / bs];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      X[a][k] = x[3 * id[a] + k];
      P[a][k] = s * p[3 * id[a] + k];
    }
  }
  const bool pt = is_pt[i] != 0;
  double d = ccd_distance(X, pt);
  double speed = ccd_speed(P, pt);
  double lhs = (speed > 0.0) ? RMUL(1.0 - CCD_S, d) : INFINITY;
  bool ok = (lhs >= speed) && (d > 0.0);
  if (ok) return;
  double co[4];
  ccd_coeffs(X, P, co);
  double w = ccd_window(co);
  double f1 = RADD(RADD(RADD(co[0], co[1]), co[2]), co[3]);
  bool ok_sign = (w >= 1.0) && (co[3] != 0.0) && (RMUL(f1, co[3]) > 0.0);
  if (!ok_sign) atomicExch(fail, 1);
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

struct CcdResult {
  double min_alpha;   // min over pairs (1 if none)
  bool certified;
  int64_t n_pairs;
};

// collect_pairs + per_subdomain_steps (+ certify when per_subdomain);
// leaves alpha_d in c->alpha_d.  x_out receives the clamped position.
static CcdResult ccd_clamp(mp_ctx* c, const double* x, const double* p, double pinf, bool per_subdomain,
                           double* x_out) {
  CcdResult R{1.0, true, 0};
  k_fill<<<grid_for(c->D, 256), 256, 0, c->stream>>>(c->alpha_d, c->D, 1.0);
  LAUNCH_CHECK();
  if (c->F > 0) {
    BpGrid B = build_bp(c, x, pinf, 0.0);
    ContactParams CP{};
    CcdParams CC{p, c->cfg.alpha_l, c->bs};
    if (c->ccd_verts.n < 4096) {
      c->ccd_verts.ensure(4096); c->ccd_ispt.ensure(4096); c->ccd_alpha.ensure(4096);
    }
    for (int attempt = 0; attempt < 4; ++attempt) {
      BpOut O{};
      O.verts = c->ccd_verts; O.ccd_ispt = c->ccd_ispt; O.alpha_pair = c->ccd_alpha; O.alpha_d = c->alpha_d;
      O.cap = (int64_t)c->ccd_verts.n;
      int64_t n = run_bp<BP_CCD>(c, x, B, O, CP, CC, nullptr);
      if (n <= O.cap) {
        R.n_pairs = n;
        break;
      }
      size_t cap = (size_t)(n * 1.5) + 4096;
      c->ccd_verts.ensure(cap); c->ccd_ispt.ensure(cap); c->ccd_alpha.ensure(cap);
      k_fill<<<grid_for(c->D, 256), 256, 0, c->stream>>>(c->alpha_d, c->D, 1.0);
      LAUNCH_CHECK();
      if (attempt == 3) throw MpError(MP_ERR_CAPACITY, "ccd pair capacity retry failed");
    }
  }
  c->n_ccd = R.n_pairs;
  if (R.n_pairs > 0) {
    // global min over pairs (deterministic: min is order independent)
    size_t bytes = 0;
    cub::DeviceReduce::Min(nullptr, bytes, c->ccd_alpha.p, c->dscal.p, (int)R.n_pairs, c->stream);
    void* tmp = cub_temp(c, bytes);
    cub::DeviceReduce::Min(tmp, bytes, c->ccd_alpha.p, c->dscal.p, (int)R.n_pairs, c->stream);
    LAUNCH_CHECK();
    CUDA_CHECK(cudaMemsetAsync(c->counters.p + 2, 0, sizeof(int), c->stream));
    if (per_subdomain) {
      k_ccd_certify<<<grid_for(R.n_pairs, 128), 128, 0, c->stream>>>(R.n_pairs, c->ccd_verts, c->ccd_ispt, x, p,
                                                                    c->alpha_d, c->bs, c->counters.p + 2);
      LAUNCH_CHECK();
    }
    CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->dscal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 2, c->counters.p + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    R.min_alpha = c->h_scal[0];
    R.certified = c->h_cnt[2] == 0;
  }
  if (per_subdomain && R.certified) {
    k_ccd_update<<<grid_for(3 * c->N, 256), 256, 0, c->stream>>>(c->N, c->bs, x, p, c->alpha_d, 0.0, x_out);
  } else {
    k_ccd_update<<<grid_for(3 * c->N, 256), 256, 0, c->stream>>>(c->N, c->bs, x, p, nullptr, R.min_alpha, x_out);
  }
  LAUNCH_CHECK();
  return R;
}
