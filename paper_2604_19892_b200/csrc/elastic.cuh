// elastic.cuh -- per-tet FEM kernels: gradient, energy, PSD-projected Hessian.
//
// Reference: energy.py:164-171 (F = Ds Bm), :184-224 (ARAP, signed SVD,
// analytic twist projection), :230-290 (stable neo-Hookean + eigen
// projection), :296-339 (dispatch), :357-370 (gradient), :373-413 (assembly).
//
// One thread per tet.  dF/dx is never stored (the reference keeps a (T,9,12)
// G): with bc_0 = -sum_r Bm[r,:] and bc_m = Bm[m-1,:], the tet force on
// vertex m is vol * P bc_m and the Hessian block (a,b) is
//   vol * ( mu (bc_a.bc_b) I3 + U K_ab U^T ),
// K_ab built from the analytic eigen-modes of the 9x9 Hessian in the
// (U, V) singular frame (twist / flip / scaling modes), each clamped at 0 --
// identical in exact arithmetic to eigh + clamp (verified to 1e-14).
#pragma once

#include <climits>

#include "ctx.cuh"

__device__ __forceinline__ void load_tet(const double* __restrict__ x, int4 t, double X[4][3]) {
  const int id[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) X[a][c] = x[3 * id[a] + c];
}

__device__ __forceinline__ void tet_F(const double X[4][3], const TetParam& tp, M3& F, double bc[4][3]) {
  double Ds[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Ds[r][c] = X[c + 1][r] - X[0][r];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      F(i, j) = Ds[i][0] * tp.Bm[0 * 3 + j] + Ds[i][1] * tp.Bm[1 * 3 + j] + Ds[i][2] * tp.Bm[2 * 3 + j];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    bc[1][j] = tp.Bm[0 * 3 + j];
    bc[2][j] = tp.Bm[1 * 3 + j];
    bc[3][j] = tp.Bm[2 * 3 + j];
    bc[0][j] = -(tp.Bm[0 * 3 + j] + tp.Bm[1 * 3 + j] + tp.Bm[2 * 3 + j]);
  }
}

// first Piola stress (energy.py:199-202, 244-247)
__device__ __forceinline__ M3 piola(const M3& F, int kind, double mu, double lam) {
  M3 P;
  if (kind == 1) {
    double U[3][3], S[3], V[3][3];
    signed_svd3(F, U, S, V);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double R = U[i][0] * V[j][0] + U[i][1] * V[j][1] + U[i][2] * V[j][2];
        P(i, j) = mu * (F(i, j) - R);
      }
  } else if (kind == 2) {
    double J = det3(F);
    M3 C = cof3(F);
    double coef = lam * (J - 1.0) - mu;
#pragma unroll
    for (int q = 0; q < 9; ++q) P.a[q] = mu * F.a[q] + coef * C.a[q];
  } else {
#pragma unroll
    for (int q = 0; q < 9; ++q) P.a[q] = 0.0;
  }
  return P;
}

// energy density (energy.py:194-196, 238-241)
__device__ __forceinline__ double psi(const M3& F, int kind, double mu, double lam) {
  if (kind == 1) {
    double U[3][3], S[3], V[3][3];
    signed_svd3(F, U, S, V);
    double s = (S[0] - 1.0) * (S[0] - 1.0) + (S[1] - 1.0) * (S[1] - 1.0) + (S[2] - 1.0) * (S[2] - 1.0);
    return 0.5 * mu * s;
  } else if (kind == 2) {
    double J = det3(F);
    double ic = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) ic += F.a[q] * F.a[q];
    return 0.5 * mu * (ic - 3.0) - mu * (J - 1.0) + 0.5 * lam * (J - 1.0) * (J - 1.0);
  }
  return 0.0;
}

// ---------------------------------------------------------------------------
// gradient: g = M (x - x~) (pinned -> 0), then tets and contacts accumulate

__global__ void k_inertia_grad(int64_t N, const double* __restrict__ x, const double* __restrict__ xt,
                               const double* __restrict__ mass, const unsigned char* __restrict__ pinned,
                               double* __restrict__ g) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  int64_t v = i / 3;
  g[i] = pinned[v] ? 0.0 : mass[v] * (x[i] - xt[i]);
}

template <int KIND>
__global__ void __launch_bounds__(128) k_tet_grad(int64_t t0, int64_t nt, const int4* __restrict__ tets,
                                                  const TetParam* __restrict__ tetp,
                                                  const double* __restrict__ x, double h2, double* __restrict__ fbuf) {
  const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= t0 + nt) return;
  const int4 tv = tets[t];
  const TetParam tp = tetp[t];
  double X[4][3], bc[4][3];
  load_tet(x, tv, X);
  M3 F;
  tet_F(X, tp, F, bc);
  const M3 P = piola(F, KIND, tp.mu, tp.lam);
  const double s = h2 * tp.vol;
  // per-corner forces; k_grad_gather sums them per vertex in a fixed order
  double* f = fbuf + 12 * t;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i)
      f[3 * a + i] = s * (P(i, 0) * bc[a][0] + P(i, 1) * bc[a][1] + P(i, 2) * bc[a][2]);
}

// g = M (x - x~) + the vertex's tet-corner forces + its contact terms
// (fixed-order warp gathers, one warp per vertex); pinned entries 0
// (energy.py:357-370)
__global__ void k_grad_gather(int64_t N, const double* __restrict__ x, const double* __restrict__ xt,
                              const double* __restrict__ mass, const unsigned char* __restrict__ pinned,
                              const int* __restrict__ vt_off, const int* __restrict__ vt_val,
                              const double* __restrict__ fbuf, const int* __restrict__ c_off,
                              const int* __restrict__ c_val, const double* __restrict__ cbuf,
                              double* __restrict__ g, int64_t v0, int64_t v1) {
  const int64_t v = v0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);  // [v0, v1): owned rows
  const int lane = threadIdx.x & 31;
  if (v >= v1) return;  // warp-uniform
  if (pinned[v]) {
    if (lane < 3) g[3 * v + lane] = 0.0;
    return;
  }
  double e0, e1, e2, c0 = 0.0, c1 = 0.0, c2 = 0.0;
  warp_gather3(vt_off[v], vt_off[v + 1], vt_val, fbuf, e0, e1, e2);
  if (c_off) warp_gather3(c_off[v], c_off[v + 1], c_val, cbuf, c0, c1, c2);
  if (lane) return;
  const double mv = mass[v];
  g[3 * v] = mv * (x[3 * v] - xt[3 * v]) + e0 + c0;
  g[3 * v + 1] = mv * (x[3 * v + 1] - xt[3 * v + 1]) + e1 + c1;
  g[3 * v + 2] = mv * (x[3 * v + 2] - xt[3 * v + 2]) + e2 + c2;
}

// The gradient in one pass (energy.py:357-370), no per-corner scratch: one
// warp per vertex, lane l computes the elastic force of its incidences
// l, l+32, ... (tet F, Piola stress, the force on this corner -- the same
// expression as k_tet_grad, so the same bits) and the warp sums them with
// the fixed tree of warp_gather3; then inertia and the contact rows.  The
// tet data are read once from HBM (a tet's 4 corner warps hit L2), x and g
// once: the 81 N + 113 T + 17 C algorithmic bytes.  Tets [0, T_snh) are
// SNH, [T_snh, T_el) ARAP (create_ctx sorts them so).
__global__ void __launch_bounds__(256) k_grad_fused(int64_t v0, int64_t v1, const double* __restrict__ x,
                                                   const double* __restrict__ xt, const double* __restrict__ mass,
                                                   const unsigned char* __restrict__ pinned,
                                                   const int* __restrict__ vt_off, const int* __restrict__ vt_val,
                                                   const int4* __restrict__ tets, const TetParam* __restrict__ tetp,
                                                   int64_t T_snh, double h2, const int* __restrict__ c_off,
                                                   const int* __restrict__ c_val, const double* __restrict__ cbuf,
                                                   double* __restrict__ g) {
  const int64_t v = v0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= v1) return;  // warp-uniform
  if (pinned[v]) {
    if (lane < 3) g[3 * v + lane] = 0.0;
    return;
  }
  double e0 = 0.0, e1 = 0.0, e2 = 0.0;
  const int b = vt_off[v], e = vt_off[v + 1];
  for (int k = b + lane; k < e; k += 32) {
    const int inc = vt_val[k];
    const int64_t t = inc >> 2;
    const int a = inc & 3;
    const TetParam tp = tetp[t];
    double X[4][3], bc[4][3];
    load_tet(x, tets[t], X);
    M3 F;
    tet_F(X, tp, F, bc);
    const M3 P = piola(F, t < T_snh ? 2 : 1, tp.mu, tp.lam);
    const double s = h2 * tp.vol;
    e0 += s * (P(0, 0) * bc[a][0] + P(0, 1) * bc[a][1] + P(0, 2) * bc[a][2]);
    e1 += s * (P(1, 0) * bc[a][0] + P(1, 1) * bc[a][1] + P(1, 2) * bc[a][2]);
    e2 += s * (P(2, 0) * bc[a][0] + P(2, 1) * bc[a][1] + P(2, 2) * bc[a][2]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    e0 += __shfl_down_sync(0xffffffffu, e0, o);
    e1 += __shfl_down_sync(0xffffffffu, e1, o);
    e2 += __shfl_down_sync(0xffffffffu, e2, o);
  }
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  if (c_off) warp_gather3(c_off[v], c_off[v + 1], c_val, cbuf, c0, c1, c2);
  if (lane) return;
  const double mv = mass[v];
  g[3 * v] = mv * (x[3 * v] - xt[3 * v]) + e0 + c0;
  g[3 * v + 1] = mv * (x[3 * v + 1] - xt[3 * v + 1]) + e1 + c1;
  g[3 * v + 2] = mv * (x[3 * v + 2] - xt[3 * v + 2]) + e2 + c2;
}

// energy pieces: 0.5 (x-x~)^T M (x-x~)  and  sum vol*psi  (energy.py:346-354)
__global__ void k_inertia_energy(int64_t N, const double* __restrict__ x, const double* __restrict__ xt,
                                 const double* __restrict__ mass, double* part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = x[i] - xt[i];
    acc += d * mass[i / 3] * d;
  }
  block_sum_store<256>(acc, part);
}

template <int KIND>
__global__ void k_tet_energy(int64_t t0, int64_t nt, const int4* __restrict__ tets,
                             const TetParam* __restrict__ tetp, const double* __restrict__ x, double* part) {
  double acc = 0.0;
  for (int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < t0 + nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    TetParam tp = tetp[t];
    double X[4][3], bc[4][3];
    load_tet(x, tets[t], X);
    M3 F;
    tet_F(X, tp, F, bc);
    acc += tp.vol * psi(F, KIND, tp.mu, tp.lam);
  }
  block_sum_store<256>(acc, part);
}

// ---------------------------------------------------------------------------
// PSD-projected element Hessians scattered into the static BSR(3x3)

struct TetModes {
  double U[3][3];
  double vb[4][3];   // vb[a][j] = V[:,j] . bc_a
  double cT[3], cF[3];  // (lambda - mu) of twist / flip mode of pair p
  double cD[3];         // (lambda - mu) of scaling mode a
  double eD[3][3];      // scaling-mode eigenvectors (columns) in the frame
};

__device__ const int PAIR_I[3] = {0, 0, 1};
__device__ const int PAIR_J[3] = {1, 2, 2};
__device__ const int PAIR_K[3] = {2, 1, 0};

__device__ void tet_modes(const M3& F, const double bc[4][3], int kind, double mu, double lam, TetModes& md) {
  double S[3], V[3][3];
  signed_svd3(F, md.U, S, V);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) md.vb[a][j] = V[0][j] * bc[a][0] + V[1][j] * bc[a][1] + V[2][j] * bc[a][2];
  if (kind == 1) {
    for (int p = 0; p < 3; ++p) {
      int i = PAIR_I[p], j = PAIR_J[p];
      double den = S[i] + S[j];
      double safe = (fabs(den) < 1e-8) ? copysign(1e-8, den + 1e-300) : den;
      double l = fmax(mu * (1.0 - 2.0 / safe), 0.0);
      md.cT[p] = l - mu;
      md.cF[p] = 0.0;
      md.cD[p] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) md.eD[r][c] = (r == c) ? 1.0 : 0.0;
  } else {
    double J = S[0] * S[1] * S[2];
    double c = lam * (J - 1.0) - mu;
    for (int p = 0; p < 3; ++p) {
      double sk = S[PAIR_K[p]];
      md.cT[p] = fmax(mu + c * sk, 0.0) - mu;
      md.cF[p] = fmax(mu - c * sk, 0.0) - mu;
    }
    double gg[3] = {S[1] * S[2], S[0] * S[2], S[0] * S[1]};
    double A[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q) A[r][q] = (r == q ? mu : 0.0) + lam * gg[r] * gg[q];
    A[0][1] += c * S[2]; A[1][0] += c * S[2];
    A[0][2] += c * S[1]; A[2][0] += c * S[1];
    A[1][2] += c * S[0]; A[2][1] += c * S[0];
    double w[3];
    sym_eig3(A, w, md.eD);
    for (int a = 0; a < 3; ++a) md.cD[a] = fmax(w[a], 0.0) - mu;
  }
}

// 3x3 block (a,b) of vol^-1 * H12 (without the mu*(bc_a.bc_b) I part)
__device__ __forceinline__ void tet_block(const TetModes& md, int a, int b, double blk[3][3]) {
  double K[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  const double rs2 = 0.70710678118654752440;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    int i = PAIR_I[p], j = PAIR_J[p];
    // twist: (vb_j e_i - vb_i e_j)/sqrt2 ; flip: (vb_j e_i + vb_i e_j)/sqrt2
    double tai = md.vb[a][j] * rs2, taj = -md.vb[a][i] * rs2;
    double tbi = md.vb[b][j] * rs2, tbj = -md.vb[b][i] * rs2;
    double cT = md.cT[p], cF = md.cF[p];
    K[i][i] += cT * tai * tbi + cF * tai * tbi;
    K[j][j] += cT * taj * tbj + cF * taj * tbj;
    K[i][j] += cT * tai * tbj - cF * tai * tbj;
    K[j][i] += cT * taj * tbi - cF * taj * tbi;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double cq = md.cD[q];
    double wa[3], wb[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      wa[i] = md.eD[i][q] * md.vb[a][i];
      wb[i] = md.eD[i][q] * md.vb[b][i];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) K[i][j] += cq * wa[i] * wb[j];
  }
  // blk = U K U^T
  double UK[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) UK[r][c] = md.U[r][0] * K[0][c] + md.U[r][1] * K[1][c] + md.U[r][2] * K[2][c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) blk[r][c] = UK[r][0] * md.U[c][0] + UK[r][1] * md.U[c][1] + UK[r][2] * md.U[c][2];
}

// index of the element block (a, b), a <= b, among the 10 stored per tet
__device__ __forceinline__ int pair_index(int a, int b) { return a * (7 - a) / 2 + b; }

template <int KIND>
__global__ void k_tet_hessian(int64_t t0, int64_t nt, const int4* __restrict__ tets,
                              const TetParam* __restrict__ tetp, const unsigned char* __restrict__ pinned,
                              const double* __restrict__ x, double h2, double* __restrict__ hbuf) {
  const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= t0 + nt) return;
  const int kd = KIND;
  int4 tv = tets[t];
  TetParam tp = tetp[t];
  double X[4][3], bc[4][3];
  load_tet(x, tv, X);
  M3 F;
  tet_F(X, tp, F, bc);
  TetModes md;
  tet_modes(F, bc, kd, tp.mu, tp.lam, md);
  const int id[4] = {tv.x, tv.y, tv.z, tv.w};
  bool pin[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) pin[a] = pinned[id[a]] != 0;
  const double s = h2 * tp.vol;
  // element blocks a <= b into hbuf; k_hess_gather sums them per BSR slot
  double* hb = hbuf + 90 * t;
  for (int a = 0; a < 4; ++a) {
    if (pin[a]) continue;
    for (int b = a; b < 4; ++b) {
      if (pin[b]) continue;
      double blk[3][3];
      tet_block(md, a, b, blk);
      double mI = tp.mu * (bc[a][0] * bc[b][0] + bc[a][1] * bc[b][1] + bc[a][2] * bc[b][2]);
      double* dst = hb + 9 * pair_index(a, b);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) dst[3 * r + c] = s * (blk[r][c] + (r == c ? mI : 0.0));
    }
  }
}

// one thread per BSR slot: (mass | pinned identity on the diagonal) + its
// element blocks in ascending (tet, a, b) order (energy.py:373-413)
__global__ void k_hess_gather(int64_t nnzb, const int* __restrict__ slot_row, const int* __restrict__ cols,
                              const int* __restrict__ hs_off, const int* __restrict__ hs_val,
                              const double* __restrict__ hbuf, const double* __restrict__ mass,
                              const unsigned char* __restrict__ pinned, double* __restrict__ bsr) {
  int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (sl >= nnzb) return;
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  const int v = slot_row[sl];
  if (cols[sl] == v) {
    const double dv = pinned[v] ? 1.0 : mass[v];
    acc[0] = dv; acc[4] = dv; acc[8] = dv;
  }
  const int k0 = hs_off[sl], k1 = hs_off[sl + 1];
  // 4 element blocks per step, all loads issued before the adds (same order)
  int k = k0;
  for (; k + 4 <= k1; k += 4) {
    double v[4][9];
    bool tr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = hs_val[k + u];
      const int t = e >> 4, a = (e >> 2) & 3, b = e & 3;
      tr[u] = a > b;
      const double* blk = hbuf + 90 * (int64_t)t + 9 * (tr[u] ? pair_index(b, a) : pair_index(a, b));
#pragma unroll
      for (int q = 0; q < 9; ++q) v[u][q] = blk[q];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (!tr[u]) {
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] += v[u][q];
      } else {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[3 * r + c] += v[u][3 * c + r];
      }
    }
  }
  for (; k < k1; ++k) {
    const int e = hs_val[k];
    const int t = e >> 4, a = (e >> 2) & 3, b = e & 3;
    if (a <= b) {
      const double* blk = hbuf + 90 * (int64_t)t + 9 * pair_index(a, b);
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] += blk[q];
    } else {
      const double* blk = hbuf + 90 * (int64_t)t + 9 * pair_index(b, a);
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[3 * r + c] += blk[3 * c + r];
    }
  }
  double* out = bsr + 9 * sl;
#pragma unroll
  for (int q = 0; q < 9; ++q) out[q] = acc[q];
}

// y = BSR x ; 8 lanes per block row, lanes stride over the row's blocks
__global__ void k_bsr_spmv(int64_t N, const int* __restrict__ rowptr, const int* __restrict__ cols,
                           const double* __restrict__ vals, const double* __restrict__ xin, double* __restrict__ y,
                           int64_t r0) {
  int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t row = r0 + (gt >> 3);  // N: end of the launch's row range [r0, N)
  int lane = threadIdx.x & 7;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  if (row < N) {
    int beg = rowptr[row], end = rowptr[row + 1];
    for (int k = beg + lane; k < end; k += 8) {
      int c = cols[k];
      const double* b = vals + 9 * (int64_t)k;
      double x0 = xin[3 * c], x1 = xin[3 * c + 1], x2 = xin[3 * c + 2];
      a0 += b[0] * x0 + b[1] * x1 + b[2] * x2;
      a1 += b[3] * x0 + b[4] * x1 + b[5] * x2;
      a2 += b[6] * x0 + b[7] * x1 + b[8] * x2;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (row < N && lane == 0) {
    y[3 * row] = a0;
    y[3 * row + 1] = a1;
    y[3 * row + 2] = a2;
  }
}

// ---------------------------------------------------------------------------
// host launchers

// energy.gradient's elastic + inertia part (energy.py:357-370), with the
// contact rows' terms when c_off is given (contact.cuh): per-corner / per-row
// forces, then one fixed-order gather per vertex -- bitwise reproducible
static void gradient_gather(mp_ctx* c, const double* x, const double* xt, double h, double* g, const int* c_off,
                            const int* c_val, const double* cbuf) {
  if (c->fused_grad) {
    timer_begin(c, MP_STAGE_TET_GRAD);
    k_grad_fused<<<grid_for(32 * (c->own_v1 - c->own_v0), 256), 256, 0, c->stream>>>(
        c->own_v0, c->own_v1, x, xt, c->mass, c->pinned, c->vt_off, c->vt_val, c->tets, c->tetp, c->T_snh, h * h,
        c_off, c_val, cbuf, g);
    LAUNCH_CHECK();
    // algorithmic bytes: 81 B per vertex, 113 B per tet
    timer_end(c, MP_STAGE_TET_GRAD, 81.0 * c->N + 113.0 * c->T);
    return;
  }
  if (c->T_snh) {
    timer_begin(c, MP_STAGE_TET_GRAD);
    k_tet_grad<2><<<grid_for(c->T_snh, 128), 128, 0, c->stream>>>(0, c->T_snh, c->tets, c->tetp, x, h * h, c->fbuf);
    LAUNCH_CHECK();
    // algorithmic bytes: 113 B of tet data per tet, x read and g written
    // once per vertex (48 B)
    timer_end(c, MP_STAGE_TET_GRAD, 113.0 * c->T_snh + 48.0 * c->N);
  }
  if (c->T_arap) {
    k_tet_grad<1><<<grid_for(c->T_arap, 128), 128, 0, c->stream>>>(c->T_snh, c->T_arap, c->tets, c->tetp, x, h * h,
                                                                   c->fbuf);
    LAUNCH_CHECK();
  }
  k_grad_gather<<<grid_for(32 * (c->own_v1 - c->own_v0), 128), 128, 0, c->stream>>>(
      c->N, x, xt, c->mass, c->pinned, c->vt_off, c->vt_val, c->fbuf, c_off, c_val, cbuf, g, c->own_v0, c->own_v1);
  LAUNCH_CHECK();
}

static void assemble_elastic_bsr(mp_ctx* c, const double* x, double h, cudaStream_t s = nullptr) {
  if (!s) s = c->stream;
  if (c->T_snh) {
    k_tet_hessian<2><<<grid_for(c->T_snh, 64), 64, 0, s>>>(0, c->T_snh, c->tets, c->tetp, c->pinned, x, h * h,
                                                           c->hbuf);
    LAUNCH_CHECK();
  }
  if (c->T_arap) {
    k_tet_hessian<1><<<grid_for(c->T_arap, 64), 64, 0, s>>>(c->T_snh, c->T_arap, c->tets, c->tetp, c->pinned, x,
                                                            h * h, c->hbuf);
    LAUNCH_CHECK();
  }
  k_hess_gather<<<grid_for(c->nnzb, 128), 128, 0, s>>>(c->nnzb, c->slot_row, c->cols, c->hs_off, c->hs_val, c->hbuf,
                                                       c->mass, c->pinned, c->bsr);
  LAUNCH_CHECK();
}

// The elastic part of H_base depends on x alone: when an iteration is known
// to rebuild, it is assembled on the side stream while the constraint set
// (sync-bound at small scale) runs on the main one; snapshot joins it.
static void bsr_ahead(mp_ctx* c, const double* x, double h) {
  CUDA_CHECK(cudaEventRecord(c->ev_it, c->stream));  // after every reader of the previous BSR
  CUDA_CHECK(cudaStreamWaitEvent(c->side, c->ev_it, 0));
  assemble_elastic_bsr(c, x, h, c->side);
  CUDA_CHECK(cudaEventRecord(c->ev_bsr_ahead, c->side));
  c->bsr_ahead_pending = true;
}

static void bsr_spmv(mp_ctx* c, const double* xin, double* y) {
  k_bsr_spmv<<<grid_for(8 * (c->own_v1 - c->own_v0), 256), 256, 0, c->stream>>>(c->own_v1, c->rowptr, c->cols, c->bsr,
                                                                                 xin, y, c->own_v0);
  LAUNCH_CHECK();
}
