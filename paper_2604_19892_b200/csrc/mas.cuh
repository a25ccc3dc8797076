// mas.cuh -- multilevel additive Schwarz preconditioner on the device.
//
// Reference: mas.py:84-90 (_spd_inverse), :123-179 (build_hierarchy),
// :182-205 (apply_preconditioner); woodbury.py:46-87 (build_update /
// apply_subdomain).
//
// Level 0: subdomain d = vertices [d*bs, d*bs + n_d) after renumbering; its
// dense block M_d = H[idx, idx] (elastic BSR blocks + mass + contact k g g^T)
// is assembled in a D x m x m scratch, factored and inverted in shared memory
// by one CTA, symmetrised, and stored packed-symmetric in the cyclic-diagonal
// layout (common.cuh) -- m(m+1)/2 doubles, the algorithmic minimum.  Padded
// dofs of a short last subdomain are identity.
// Coarse level l: aggregate a = vertices [a*span_l, (a+1)*span_l), span_l =
// bs * coarse_block^l; M_l = C H C^T accumulated from BSR blocks and contacts,
// inverted with cuSOLVER potrf/potri (dense FP64), packed the same way.
// Woodbury (Sparse-Input): for touched subdomains W = B U is formed from the
// <= 12 non-zero rows of each u column; the corrected inverse
// B~ = B - W cap^-1 W^T (== (M_d + U U^T)^-1) goes to an overlay slot the
// apply reads instead of B_d.  Large K_d falls back to refactoring
// M_d + U U^T directly (same matrix, one Cholesky-inverse).
#pragma once

#include "ctx.cuh"

// ---------------------------------------------------------------------------
// level-0 assembly

// M_d assembled in shared memory (m x m, row stride m), by the subdomain's
// own CTA: first the contact terms -- one thread per local vertex a owns
// rows 3a..3a+2 and adds its incidences' k grad_a grad_b^T (b in the same
// subdomain) in ascending (contact, partner) order -- then the BSR blocks
// whose row and column both lie in the subdomain (unique targets).  No
// atomics: the same sums in the same order on every run.
__device__ void assemble_block_smem(int64_t d, int64_t N, int bs, int m, const unsigned char* __restrict__ pinned,
                                    const int* __restrict__ off, const int* __restrict__ inc,
                                    const int4* __restrict__ verts, const double* __restrict__ grad,
                                    const double* __restrict__ k, const int* __restrict__ rowptr,
                                    const int* __restrict__ slot_row, const int* __restrict__ cols,
                                    const double* __restrict__ vals, double* S) {
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) S[e] = 0.0;
  __syncthreads();
  const int64_t v0 = d * bs;
  const int nd = (int)((N - v0) < bs ? (N - v0) : bs);
  if (off && (int)threadIdx.x < nd) {
    const int la = threadIdx.x;
    const int64_t v = v0 + la;
    if (!pinned[v]) {  // pinned rows of grad are zero
      for (int q = off[v]; q < off[v + 1]; ++q) {
        const int e = inc[q];
        const int64_t i = e >> 2;
        const int a = e & 3;
        const int4 vv = verts[i];
        const int id[4] = {vv.x, vv.y, vv.z, vv.w};
        const double kk = k[i];
        const double* ga = grad + 12 * i + 3 * a;
        for (int b = 0; b < 4; ++b) {
          if (id[b] / bs != d) continue;
          const int lb = id[b] - (int)v0;
          const double* gb = grad + 12 * i + 3 * b;
          for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) {
              const double val = kk * ga[r] * gb[cc];
              if (val != 0.0) S[(3 * la + r) * m + 3 * lb + cc] += val;
            }
        }
      }
    }
  }
  __syncthreads();
  const int s0 = rowptr[v0], s1 = rowptr[v0 + nd];
  for (int sl = s0 + threadIdx.x; sl < s1; sl += blockDim.x) {
    const int w = cols[sl];
    if (w < v0 || w >= v0 + nd) continue;
    const int lr = slot_row[sl] - (int)v0;
    const int lc = w - (int)v0;
    const double* b = vals + 9 * (int64_t)sl;
    double* dst = S + (3 * lr) * m + 3 * lc;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) dst[r * m + c] += b[3 * r + c];
  }
  __syncthreads();
}

// write a symmetric m x m smem matrix (0.5 (X + X^T)) in cyclic-diagonal packing
__device__ void store_cyc_sym(const double* X, int m, double* __restrict__ out, bool symmetrize) {
  const int tot = (int)cyc_size(m);
  for (int e = threadIdx.x; e < tot; e += blockDim.x) {
    int s = e / m;
    int i = e - s * m;
    int j = i + s;
    if (j >= m) j -= m;
    out[e] = symmetrize ? 0.5 * (X[i * m + j] + X[j * m + i]) : X[i * m + j];
  }
}

__device__ void load_cyc_full(const double* __restrict__ in, int m, double* X) {
  const int64_t tot = cyc_size(m);
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    int s = (int)(e / m);
    int i = (int)(e - (int64_t)s * m);
    int j = i + s;
    if (j >= m) j -= m;
    double v = in[e];
    X[i * m + j] = v;
    X[j * m + i] = v;
  }
}

// In-smem Cholesky (lower, A = L L^T) of A (m x m row-major). Returns false
// (via *bad) when a pivot is not positive -- LAPACK potrf's failure mode.
__device__ void smem_cholesky(double* A, int m, int* bad) {
  for (int k = 0; k < m; ++k) {
    __syncthreads();
    double piv = A[k * m + k];
    if (!(piv > 0.0)) {
      if (threadIdx.x == 0) *bad = 1;
      return;  // uniform: every thread read the same pivot
    }
    double dk = sqrt(piv);
    __syncthreads();
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) A[i * m + k] /= dk;
    if (threadIdx.x == 0) A[k * m + k] = dk;
    __syncthreads();
    // trailing update of the lower triangle
    const int rem = m - k - 1;
    const int tot = rem * rem;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      int i = k + 1 + e / rem;
      int j = k + 1 + e % rem;
      if (j <= i) A[i * m + j] -= A[i * m + k] * A[j * m + k];
    }
  }
  __syncthreads();
}

// X = A^-1 from the lower Cholesky factor in A: thread j solves column j
// (L y = e_j, L^T x = y), mirroring cho_solve(cho_factor(A), I) (mas.py:89)
__device__ void smem_chol_inverse(const double* L, int m, double* X) {
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    for (int i = 0; i < j; ++i) X[i * m + j] = 0.0;
    for (int i = j; i < m; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) s -= L[i * m + k] * X[k * m + j];
      X[i * m + j] = s / L[i * m + i];
    }
    for (int i = m - 1; i >= 0; --i) {
      double s = X[i * m + j];
      for (int k = i + 1; k < m; ++k) s -= L[k * m + i] * X[k * m + j];
      X[i * m + j] = s / L[i * m + i];
    }
  }
  __syncthreads();
}


#define SWEEP_T 6

// 1/a to ~1 ulp: MUFU reciprocal seed + two Newton steps (the IEEE division
// sits on the sweep's serial critical path)
__device__ __forceinline__ double fast_rcp(double a) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
  double e = fma(-a, r, 1.0);
  r = fma(r, e, r);
  e = fma(-a, r, 1.0);
  return fma(r, e, r);
}

// Sweep every pivot of the m x m (m <= 96) symmetric matrix held in
// registers (sweep_regs); on return it holds -M^-1.  Returns false
// (uniformly) when a pivot is not positive.  Per step the common path is 12
// shared loads and 36 DFMA per thread; the 16 threads holding row k and the
// 16 holding column k take a compile-time-indexed fix-up, and the owners of
// row k+1 publish it (raw and scaled by its reciprocal) right after their
// update.

// The pivot-row buffer of one step: raw row k [0, 96), the row scaled by
// 1 / A_kk [96, 192), 1 / A_kk at [192], A_kk at [193] (double-buffered).
#define SW_ROW 196

// Owners of row k1 (one half-warp: tr fixed, tc = 0..15) publish it raw and
// scaled for the next step; the pivot A_{k1,k1} comes from the half-warp's
// lane tc = k1 % 16 (register R[A][A]), its reciprocal is computed once here
// instead of in all 256 threads.
template <int A>
__device__ __forceinline__ void publish_row_scaled(const double (&R)[SWEEP_T][SWEEP_T], double* rk, int tc, int m,
                                                   int k1) {
  const unsigned hm = 0xFFFFu << (threadIdx.x & 16);
  const double piv = __shfl_sync(hm, R[A][A], (threadIdx.x & 16) + (k1 & 15));
  const double inv = fast_rcp(piv);
#pragma unroll
  for (int b = 0; b < SWEEP_T; ++b)
    if (tc + 16 * b < m) {
      rk[tc + 16 * b] = R[A][b];
      rk[96 + tc + 16 * b] = R[A][b] * inv;
    }
  if (tc == 0) {
    rk[192] = inv;
    rk[193] = piv;
  }
}

// The 16 pivots of register panel KA (k = 16 KA + kr): the fix-ups index
// R[KA][.] / R[.][KA] at compile time.  Per step: one barrier, 12 shared
// loads (the scaled column values, the raw row values), 36 FMA.
template <int KA>
__device__ __forceinline__ bool sweep_panel(int m, double* rowk, double (&R)[SWEEP_T][SWEEP_T], int tr, int tc) {
  for (int kr = 0; kr < 16; ++kr) {
    const int k = 16 * KA + kr;
    if (k >= m) return true;  // uniform
    const double* r = rowk + (k & 1) * SW_ROW;
    __syncthreads();
    // every shared load of the step issued before the pivot test (which
    // would otherwise serialise a second shared-memory round trip behind it)
    const double piv = r[193], inv = r[192];
    double ci[SWEEP_T], cj[SWEEP_T], rs[SWEEP_T];
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a) {
      ci[a] = r[96 + tr + 16 * a];  // A_ik / A_kk (= A_ki / A_kk)
      cj[a] = r[tc + 16 * a];       // A_kj
      rs[a] = r[96 + tc + 16 * a];  // A_kj / A_kk (row k's fix-up)
    }
    if (!(piv > 0.0)) return false;  // uniform across the CTA
#pragma unroll
    for (int a = 0; a < SWEEP_T; ++a)
#pragma unroll
      for (int b = 0; b < SWEEP_T; ++b) R[a][b] = fma(-ci[a], cj[b], R[a][b]);
    if (tr == kr)  // row k: A_kj <- A_kj / A_kk
#pragma unroll
      for (int b = 0; b < SWEEP_T; ++b) R[KA][b] = rs[b];
    if (tc == kr) {  // column k: A_ik <- A_ik / A_kk, and A_kk <- -1 / A_kk
#pragma unroll
      for (int a = 0; a < SWEEP_T; ++a) R[a][KA] = ci[a];
      if (tr == kr) R[KA][KA] = -inv;
    }
    const int k1 = k + 1;
    if (k1 < m && tr == (k1 & 15)) {
      double* rn = rowk + (k1 & 1) * SW_ROW;
      if (kr < 15) publish_row_scaled<KA>(R, rn, tc, m, k1);
      else if (KA + 1 < SWEEP_T) publish_row_scaled<(KA + 1 < SWEEP_T ? KA + 1 : KA)>(R, rn, tc, m, k1);
    }
  }
  return true;
}

// The matrix lives in R (thread (tr, tc) holds rows tr + 16a, columns
// tc + 16b); LOAD(i, j) supplies the input, all 36 loads issued at once.
// rowk: 2 x SW_ROW doubles of shared memory.
template <class LOAD>
__device__ bool sweep_regs(LOAD load, int m, double* rowk, double (&R)[SWEEP_T][SWEEP_T]) {
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
#pragma unroll
  for (int a = 0; a < SWEEP_T; ++a)
#pragma unroll
    for (int b = 0; b < SWEEP_T; ++b) {
      int i = tr + 16 * a, j = tc + 16 * b;
      R[a][b] = (i < m && j < m) ? load(i, j) : 0.0;
    }
  for (int e = tid; e < 2 * SW_ROW; e += blockDim.x) rowk[e] = 0.0;
  __syncthreads();
  if (tr == 0) publish_row_scaled<0>(R, rowk, tc, m, 0);  // row 0 for step 0
  return sweep_panel<0>(m, rowk, R, tr, tc) && sweep_panel<1>(m, rowk, R, tr, tc) &&
         sweep_panel<2>(m, rowk, R, tr, tc) && sweep_panel<3>(m, rowk, R, tr, tc) &&
         sweep_panel<4>(m, rowk, R, tr, tc) && sweep_panel<5>(m, rowk, R, tr, tc);
}

// element (i, j) of a symmetric m x m matrix is the stored representative
// of the cyclic-diagonal packing (common.cuh) at position cyc_index(m, i, j)
__device__ __forceinline__ bool cyc_rep(int m, int i, int j) {
  int s = j - i;
  if (s < 0) s += m;
  return 2 * s < m || (2 * s == m && i < j);
}

// One CTA per subdomain: M_d assembled in smem (BSR + contacts) -> Mblk
// (packed) and Bblk = sym(M^-1)
// (mas.py:84-90).  The inverse is formed by the symmetric sweep operator
// (Gauss-Jordan without pivoting, stable for SPD): after sweeping every
// pivot the matrix holds -M^-1.  Its pivots are the Schur-complement
// diagonals, i.e. the squared Cholesky pivots, so "pivot <= 0" is exactly
// cho_factor's non-SPD failure.  The m x m matrix lives in registers, a
// 6 x 6 tile per thread on a 16 x 16 thread grid (m <= 96); each step
// broadcasts the old pivot row through shared memory (double-buffered, one
// barrier per step).  The matrix stays symmetric to rounding, so the
// broadcast pivot row doubles as the pivot column.
__global__ void __launch_bounds__(256, 2)
k_mas_sweep(int64_t D, int64_t N, int bs, int m, const unsigned char* __restrict__ pinned,
            const int* __restrict__ inc_off, const int* __restrict__ inc, const int4* __restrict__ cverts,
            const double* __restrict__ cgrad, const double* __restrict__ ck, const int* __restrict__ rowptr,
            const int* __restrict__ slot_row, const int* __restrict__ cols, const double* __restrict__ bsr,
            double* __restrict__ Mblk,
            double* __restrict__ Bblk, int* __restrict__ status, int64_t d0) {
  extern __shared__ double msm[];  // m x m: M_d
  __shared__ double rowk[2 * SW_ROW];
  const int64_t d = d0 + blockIdx.x;  // d0: a shard's first owned subdomain
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
  const int nd3 = 3 * (int)((N - d * bs) < bs ? (N - d * bs) : bs);
  assemble_block_smem(d, N, bs, m, pinned, inc_off, inc, cverts, cgrad, ck, rowptr, slot_row, cols, bsr, msm);
  const int64_t csz = cyc_size(m);
  double* mout = Mblk + d * csz;
  double R[SWEEP_T][SWEEP_T];
  // M_d (padding rows of a short last subdomain = identity), packed into Mblk
  auto load = [&](int i, int j) -> double {
    double v = (i >= nd3 || j >= nd3) ? ((i == j) ? 1.0 : 0.0) : msm[i * m + j];
    if (cyc_rep(m, i, j)) mout[cyc_index(m, i, j)] = v;
    return v;
  };
  if (!sweep_regs(load, m, rowk, R)) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  // B_d = -R; R is symmetric to rounding (1 ulp), the representative of each
  // symmetric pair is stored (the reference averages the two, mas.py:90)
  double* bout = Bblk + d * csz;
#pragma unroll
  for (int a = 0; a < SWEEP_T; ++a)
#pragma unroll
    for (int b = 0; b < SWEEP_T; ++b) {
      const int i = tr + 16 * a, j = tc + 16 * b;
      if (i < m && j < m && cyc_rep(m, i, j)) bout[cyc_index(m, i, j)] = -R[a][b];
    }
}

// ---------------------------------------------------------------------------
// coarse levels

// M_l from the BSR by a static gather map: one warp per nonzero coarse block
// (A, B) sums its BSR slots in ascending order (lanes strided, fixed shuffle
// tree), then scales by 1/(|a||b|) -- no atomics, reproducible
__global__ void k_coarse_gather(int nblk, const int* __restrict__ cb_key, const int* __restrict__ cb_off,
                                const int* __restrict__ cb_slot, const double* __restrict__ bsr, int nA, int64_t N,
                                int span, int n, double* __restrict__ M) {
  // one warp per nonzero coarse block; lane l sums slots l, l + 32, ... in
  // that order (fixed), four slots' loads in flight at a time (a diagonal
  // block gathers ~|A| x 14 slots: dependent slot -> block loads otherwise
  // serialise on latency)
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= nblk) return;
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  const int k1 = cb_off[w + 1];
  for (int k = cb_off[w] + lane; k < k1; k += 4 * 32) {
    int sl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sl[u] = (k + 32 * u < k1) ? cb_slot[k + 32 * u] : -1;
    double b[4][9];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 9; ++q) b[u][q] = sl[u] >= 0 ? bsr[9 * (int64_t)sl[u] + q] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (sl[u] >= 0)
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] += b[u][q];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], o);
  if (lane) return;
  const int key = cb_key[w];
  const int A = key / nA, B = key - (key / nA) * nA;
  const int64_t na = (N - (int64_t)A * span) < span ? (N - (int64_t)A * span) : span;
  const int64_t nb = (N - (int64_t)B * span) < span ? (N - (int64_t)B * span) : span;
  const double sc = 1.0 / ((double)na * (double)nb);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) M[(int64_t)(3 * A + r) * n + 3 * B + c] = acc[3 * r + c] * sc;
}

// M_{l+1} from the finer level's dense M_l (contacts included): every coarse
// 3x3 block sums the cb x cb fine blocks it covers, weighted |a_f||b_f| /
// (|A||B|) -- the same Galerkin sum as from the BSR, from n_l^2 instead of
// nnzb reads.  One thread per coarse entry, fine blocks in ascending order.
__global__ void k_coarse_up(int nA, int cb, int nAf, const double* __restrict__ Mf, int nf, int64_t N, int span,
                            int span_f, double* __restrict__ M) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = 3 * nA;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e / n), j = (int)(e - (int64_t)(e / n) * n);
  const int A = i / 3, r = i - 3 * (i / 3), B = j / 3, c = j - 3 * (j / 3);
  auto size = [&](int a, int sp) {
    const int64_t s = N - (int64_t)a * sp;
    return (double)(s < sp ? s : sp);
  };
  double acc = 0.0;
  for (int af = A * cb; af < (A + 1) * cb && af < nAf; ++af) {
    const double wa = size(af, span_f);
    for (int bf = B * cb; bf < (B + 1) * cb && bf < nAf; ++bf)
      acc += Mf[(int64_t)(3 * af + r) * nf + 3 * bf + c] * (wa * size(bf, span_f));
  }
  M[e] = acc / (size(A, span) * size(B, span));
}

// 128-bit fixed-point accumulation: integer addition is associative, so the
// contact terms of the coarse levels sum to the same bits in any order.
// y is in units of the call's fixed-point unit (|partial sums| < 2^120).
__device__ __forceinline__ void fx_add(unsigned long long* p, double y) {
  const double yi = rint(y);
  if (yi == 0.0) return;
  __int128 v;
  const int e = ilogb(yi);
  if (e < 62) {
    v = (__int128)(long long)yi;
  } else {
    const long long m = (long long)scalbn(yi, 52 - e);  // exact 53-bit signed mantissa
    v = (__int128)m * ((__int128)1 << (e - 52));
  }
  const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
  const unsigned long long old = atomicAdd(p, lo);
  atomicAdd(p + 1, hi + (old + lo < old ? 1ull : 0ull));
}

// the two words fx_add adds (false: rounds to zero, nothing to add)
__device__ __forceinline__ bool fx_split(double y, unsigned long long& lo, unsigned long long& hi) {
  const double yi = rint(y);
  if (yi == 0.0) return false;
  __int128 v;
  const int e = ilogb(yi);
  if (e < 62) {
    v = (__int128)(long long)yi;
  } else {
    const long long m = (long long)scalbn(yi, 52 - e);
    v = (__int128)m * ((__int128)1 << (e - 52));
  }
  lo = (unsigned long long)v;
  hi = (unsigned long long)(v >> 64);
  return true;
}

__device__ __forceinline__ double fx_get(const unsigned long long* p) {
  return (double)(long long)p[1] * 18446744073709551616.0 + (double)p[0];
}

// fixed-point unit from T = sum_i k_i |grad_i|^2 >= |any coarse contact entry|:
// out[0] = 1 / unit, out[1] = unit = 2^(ilogb(T) + 1 - 120).  One block, fixed order.
#define FX_PARTS 64
__global__ void k_fx_scale_part(int64_t nc, const double* __restrict__ k, const double* __restrict__ nrm,
                                double* __restrict__ part) {
  // block b sums the fixed chunk [b c, (b + 1) c): strided lanes, fixed tree
  __shared__ double sh[256];
  const int64_t c = (nc + FX_PARTS - 1) / FX_PARTS;
  const int64_t i0 = blockIdx.x * c, i1 = min(nc, i0 + c);
  double s = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += 256) s += fabs(k[i]) * nrm[i] * nrm[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_fx_scale(const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double T = 0.0;
  for (int b = 0; b < FX_PARTS; ++b) T += part[b];
  const int e = (T > 0.0 && isfinite(T)) ? ilogb(T) + 1 - 120 : 0;
  out[0] = ldexp(1.0, -e);
  out[1] = ldexp(1.0, e);
}

// contacts -> the coarse level's 128-bit accumulators: k w_A w_B^T over the
// contact's distinct aggregates, w_A = sum_{a in A} grad_a / |A| (the same
// sum as k grad_a grad_b^T / (|A||B|) over vertex pairs).  One thread per
// (contact, aggregate pair): a contact's <= 16 blocks go to 16 threads, and
// each thread issues its 9 low-word atomics before it uses any returned
// word (a thread per contact made 144 dependent atomic round trips: ~200 us
// at C2 for 13k contacts).
__global__ void k_contact_coarse(int64_t nc, const int4* __restrict__ verts, const double* __restrict__ grad,
                                 const double* __restrict__ k, int64_t N, int span, int n,
                                 const double* __restrict__ fx, unsigned long long* __restrict__ acc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = t >> 4;
  if (i >= nc) return;
  const int pa = (int)(t & 15) >> 2, pb = (int)(t & 3);
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  const double* gr = grad + 12 * i;
  int agg[4];
  double w[4][3];
  int na = 0;
  for (int a = 0; a < 4; ++a) {
    const int A = id[a] / span;
    int q = 0;
    while (q < na && agg[q] != A) ++q;
    if (q == na) {
      agg[na] = A;
      w[na][0] = w[na][1] = w[na][2] = 0.0;
      ++na;
    }
    w[q][0] += gr[3 * a]; w[q][1] += gr[3 * a + 1]; w[q][2] += gr[3 * a + 2];
  }
  if (pa >= na || pb >= na) return;
  double wa[3], wb[3];
  {
    const int64_t sa = (N - (int64_t)agg[pa] * span) < span ? (N - (int64_t)agg[pa] * span) : span;
    const int64_t sb = (N - (int64_t)agg[pb] * span) < span ? (N - (int64_t)agg[pb] * span) : span;
    const double ia = 1.0 / (double)sa, ib = 1.0 / (double)sb;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      wa[r] = w[pa][r] * ia;
      wb[r] = w[pb][r] * ib;
    }
  }
  const double s = k[i] * fx[0];
  unsigned long long lo[9], hi[9];
  bool live[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const double val = s * wa[e / 3] * wb[e % 3];
    live[e] = fx_split(val, lo[e], hi[e]);
  }
  unsigned long long old[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    unsigned long long* p = acc + 2 * ((int64_t)(3 * agg[pa] + e / 3) * n + 3 * agg[pb] + e % 3);
    old[e] = live[e] ? atomicAdd(p, lo[e]) : 0ull;
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    if (!live[e]) continue;
    unsigned long long* p = acc + 2 * ((int64_t)(3 * agg[pa] + e / 3) * n + 3 * agg[pb] + e % 3);
    atomicAdd(p + 1, hi[e] + (old[e] + lo[e] < old[e] ? 1ull : 0ull));
  }
}

// 0.5 (M + M^T) on the lower triangle (the only half potrf reads)
// (plus the contact accumulators when acc != nullptr)
// 32 x 32 tile pairs (I, J), I >= J, through shared memory so both the
// (i, j) and the transposed (j, i) accesses are coalesced
__global__ void __launch_bounds__(256) k_sym_lower(int n, double* M, const unsigned long long* __restrict__ acc,
                                                   const double* __restrict__ fx) {
  const int nt = (n + 31) / 32;
  // blockIdx.x -> (I, J) with J <= I, row-major over the lower triangle
  const int64_t b = blockIdx.x;
  int I = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while ((int64_t)(I + 1) * (I + 2) / 2 <= b) ++I;
  while ((int64_t)I * (I + 1) / 2 > b) --I;
  const int J = (int)(b - (int64_t)I * (I + 1) / 2);
  if (I >= nt) return;
  __shared__ double ta[32][33], tb[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const double unit = acc ? fx[1] : 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int i = 32 * I + r, j = 32 * J + tx;
    if (i < n && j < n) {
      double a = M[(int64_t)i * n + j];
      if (acc) a += fx_get(acc + 2 * ((int64_t)i * n + j)) * unit;
      ta[r][tx] = a;
    }
    const int i2 = 32 * J + r, j2 = 32 * I + tx;
    if (i2 < n && j2 < n) {
      double a = M[(int64_t)i2 * n + j2];
      if (acc) a += fx_get(acc + 2 * ((int64_t)i2 * n + j2)) * unit;
      tb[r][tx] = a;
    }
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = 32 * I + r, j = 32 * J + tx;
    if (i < n && j < n) {
      // (i, j) with its transpose (j, i) = tb[tx][r]
      const double a = ta[r][tx], bt = tb[tx][r];
      M[(int64_t)i * n + j] = (i == j) ? a : 0.5 * (a + bt);
    }
    const int i2 = 32 * J + r, j2 = 32 * I + tx;
    if (I != J && i2 < n && j2 < n) {
      const double a = tb[r][tx], bt = ta[tx][r];
      M[(int64_t)i2 * n + j2] = 0.5 * (bt + a);
    }
  }
}

// ---------------------------------------------------------------------------
// apply

// raw sums of g over each level-1 aggregate (one CTA per aggregate) and the
// restriction r = C g = raw sum * (1 / |a|) (the reference's aggregation
// weights 1/len(verts), mas.py:123-135)
__global__ void k_restrict1(int64_t N, int span, const double* __restrict__ g, double* __restrict__ rsum,
                            double* __restrict__ r, int64_t a0) {
  const int64_t a = a0 + blockIdx.x;  // a0: a shard's first owned aggregate
  const int64_t v0 = a * span;
  int64_t v1 = v0 + span;
  if (v1 > N) v1 = N;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    s0 += g[3 * v];
    s1 += g[3 * v + 1];
    s2 += g[3 * v + 2];
  }
  __shared__ double sh[3][32];
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = s0; sh[1][w] = s1; sh[2][w] = s2;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sh[threadIdx.x][q];
    rsum[3 * a + threadIdx.x] = t;
    r[3 * a + threadIdx.x] = t * (1.0 / (double)(v1 - v0));
  }
}

// raw sums of a coarser level from the finer level's raw sums, and its r
__global__ void k_restrict_up(int A, int cb, int Afine, int64_t N, int span, const double* __restrict__ fine,
                              double* __restrict__ out, double* __restrict__ r) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= 3 * (int64_t)A) return;
  int a = (int)(e / 3), c = (int)(e % 3);
  double s = 0.0;
  for (int q = a * cb; q < (a + 1) * cb && q < Afine; ++q) s += fine[3 * q + c];
  out[e] = s;
  const int64_t v0 = (int64_t)a * span;
  const int64_t na = (N - v0) < span ? (N - v0) : span;
  r[e] = s * (1.0 / (double)na);
}

// y = Minv r: each (row block, diagonal chunk) CTA writes its partial; the
// row block's last CTA to finish sums the chunks in order (reproducible).
// Many small chunks keep every SM busy.
__global__ void k_coarse_mv(int n, int chunks, const double* __restrict__ P, const double* __restrict__ r,
                            double* __restrict__ ypc, double* __restrict__ y, int* __restrict__ done) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int ch = blockIdx.y;
  const int smax = n / 2;  // diagonals 0..smax
  int per = (smax + 1 + chunks - 1) / chunks;
  int s0 = ch * per, s1 = s0 + per - 1;
  if (s1 > smax) s1 = smax;
  double acc = 0.0;
  const bool even = (n % 2) == 0;
  if (i < n) {
    int s = s0;
    if (s == 0) {
      acc += P[i] * r[i];
      s = 1;
    }
    const int s_hi = (even && s1 == n / 2) ? s1 - 1 : s1;  // full diagonals
    // 4 diagonals per step, loads issued before use (latency, not a chain)
    for (; s + 3 <= s_hi; s += 4) {
      double a[4], b[4];
      int jp[4], jm[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        jp[u] = i + s + u; if (jp[u] >= n) jp[u] -= n;
        jm[u] = i - s - u; if (jm[u] < 0) jm[u] += n;
        const double* dg = P + (int64_t)(s + u) * n;
        a[u] = __ldg(dg + i);
        b[u] = __ldg(dg + jm[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += a[u] * r[jp[u]] + b[u] * r[jm[u]];
    }
    for (; s <= s1; ++s) {
      const double* dg = P + (int64_t)s * n;
      int jp = i + s; if (jp >= n) jp -= n;
      int jm = i - s; if (jm < 0) jm += n;
      if (even && 2 * s == n) {
        // half diagonal: A(i, i+n/2) stored at min(i, i+n/2)
        acc += dg[i < jp ? i : jp] * r[jp];
      } else {
        acc += __ldg(dg + i) * r[jp] + __ldg(dg + jm) * r[jm];
      }
    }
    ypc[(int64_t)ch * n + i] = acc;
  }
  __threadfence();
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done + blockIdx.x, 1) == chunks - 1;
  __syncthreads();
  if (!last) return;
  if (i < n) {
    double s = 0.0;
    for (int q = 0; q < chunks; ++q) s += __ldcg(ypc + (int64_t)q * n + i);
    y[i] = s;
  }
  if (threadIdx.x == 0) done[blockIdx.x] = 0;  // ready for the next apply
}

struct LevelView {
  const double* y;
  int n, span, ratio;  // ratio = span / bs: subdomains per aggregate
};
struct LevelViews {
  LevelView lv[8];
  int L;
  int64_t d0;  // first subdomain of this launch (a shard's owned range; 0 on one GPU)
};

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Level-0 + Woodbury overlay + coarse prolongation + pinned projection
// (mas.py:196-205, solver.py:351-352).  Persistent CTAs walk the subdomains;
// each packed block (m(m+1)/2 doubles, 37 KB at m = 96) is streamed into
// shared memory by one TMA bulk copy, double-buffered so the next block's
// copy overlaps this block's matvec.  One thread per block row reads the
// cyclic diagonals diag_s[i], diag_s[(i-s) mod m] from shared memory.
#define APPLY_THREADS 192  // two 96-thread groups split the diagonals of a block
#define APPLY_CHUNKS 4      // bulk copies per block (more TMA requests in flight)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// USE_TMA: one elected thread streams each packed block with cp.async.bulk
// (TMA, completes on an mbarrier); otherwise every thread issues 16-byte
// cp.async (LDGSTS) copies -- same double buffering, more requests in flight.
template <bool USE_TMA, int STAGES>
__global__ void __launch_bounds__(APPLY_THREADS)
k_mas_apply_l0(int64_t D, int64_t N, int bs, int m, const double* __restrict__ Bblk,
               const int* __restrict__ overlay_of, const double* __restrict__ overlay, const double* __restrict__ g,
               const unsigned char* __restrict__ pinned, LevelViews LV, double* __restrict__ z) {
  extern __shared__ __align__(16) double sm[];
  const int64_t csz = cyc_size(m);
  const int64_t cpad = (csz + 1) & ~1ll;  // 16-byte aligned stages
  double* buf[STAGES];
#pragma unroll
  for (int q = 0; q < STAGES; ++q) buf[q] = sm + q * cpad;
  double* gsh = sm + STAGES * cpad;  // 96
  double* part = gsh + 96;           // 96 partial sums of the second group
  __shared__ __align__(8) unsigned long long bar[STAGES];
  const int tid = threadIdx.x;
  const int grp = tid >= 96 ? 1 : 0;
  const int i = tid - 96 * grp;
  // chunk boundaries in doubles, multiples of 2 (16 B)
  const int64_t chunk = ((csz + APPLY_CHUNKS - 1) / APPLY_CHUNKS + 1) & ~1ll;
  auto src_of = [&](int64_t dl) -> const double* {
    const int64_t d = LV.d0 + dl;
    const int ov = overlay_of ? overlay_of[d] : -1;
    return (ov >= 0) ? overlay + (int64_t)ov * csz : Bblk + d * csz;
  };
  auto issue = [&](int stage, int64_t d) {  // TMA: thread 0 only
    const double* src = src_of(d);
    mbar_expect_tx(&bar[stage], (unsigned)(csz * sizeof(double)));
    for (int q = 0; q < APPLY_CHUNKS; ++q) {
      const int64_t b0 = q * chunk;
      const int64_t b1 = (b0 + chunk < csz) ? b0 + chunk : csz;
      if (b1 > b0) bulk_g2s(buf[stage] + b0, src + b0, (unsigned)((b1 - b0) * sizeof(double)), &bar[stage]);
    }
  };
  auto issue_async = [&](int stage, int64_t d) {  // LDGSTS: every thread
    const double* src = src_of(d);
    const int64_t n16 = csz / 2;  // 16-byte chunks (csz is even for m = 96)
    for (int64_t e = tid; e < n16; e += APPLY_THREADS) cp_async16(buf[stage] + 2 * e, src + 2 * e);
    if ((csz & 1) && tid == 0) buf[stage][csz - 1] = src[csz - 1];
    cp_async_commit();
  };
  if (USE_TMA && tid == 0) {
    for (int q = 0; q < STAGES; ++q) mbar_init(&bar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // prologue: the first STAGES-1 blocks of this CTA
  for (int q = 0; q < STAGES - 1; ++q) {
    const int64_t dq = blockIdx.x + (int64_t)q * gridDim.x;
    if (USE_TMA) {
      if (tid == 0 && dq < D) issue(q, dq);
    } else {
      if (dq < D) issue_async(q, dq);
      else cp_async_commit();
    }
  }
  int64_t d = blockIdx.x;
  const int smax = m / 2;
  const bool even = (m % 2) == 0;
  const int s_full = even ? smax - 1 : smax;
  const int s_mid = s_full / 2;  // group 0: 1..s_mid, group 1: s_mid+1..s_full (+ half diagonal)
  for (int it = 0; d < D; d += gridDim.x, ++it) {
    const int st = it % STAGES;
    const int64_t dn = d + (int64_t)(STAGES - 1) * gridDim.x;
    const int sn = (it + STAGES - 1) % STAGES;
    // prefetch STAGES-1 blocks ahead into the stage freed by iteration it-1
    if (USE_TMA) {
      if (tid == 0 && dn < D) issue(sn, dn);
    } else {
      if (dn < D) issue_async(sn, dn);
      else cp_async_commit();  // empty group keeps the wait_group count uniform
    }
    const int64_t da = LV.d0 + d;
    const int64_t v0 = da * bs;
    const int nd3 = 3 * (int)((N - v0) < bs ? (N - v0) : bs);
    if (tid < m) gsh[tid] = (tid < nd3) ? g[3 * v0 + tid] : 0.0;
    if (USE_TMA) {
      __syncthreads();
      mbar_wait(&bar[st], (unsigned)((it / STAGES) & 1));
    } else {
      cp_async_wait<STAGES - 1>();  // this block's group has landed (prefetches may still fly)
      __syncthreads();
    }
    const double* P = buf[st];
    double acc = 0.0;
    if (i < nd3) {
      const int s0 = grp ? s_mid + 1 : 1, s1 = grp ? s_full : s_mid;
      if (!grp) acc = P[i] * gsh[i];
#pragma unroll 4
      for (int s = s0; s <= s1; ++s) {
        const double* dg = P + (int64_t)s * m;
        int jp = i + s; if (jp >= m) jp -= m;
        int jm = i - s; if (jm < 0) jm += m;
        acc += dg[i] * gsh[jp] + dg[jm] * gsh[jm];
      }
      if (grp && even) {
        const double* dg = P + (int64_t)smax * m;
        int jp = i + smax; if (jp >= m) jp -= m;
        acc += dg[i < jp ? i : jp] * gsh[jp];
      }
      if (grp) part[i] = acc;
    }
    __syncthreads();
    if (!grp && i < nd3) {
      acc += part[i];
      // prolongation C^T y: y of the vertex's aggregate times 1/|a|
      const int64_t dof = 3 * v0 + i;
      const int64_t v = v0 + i / 3;
      const int c = i - 3 * (i / 3);
      for (int l = 0; l < LV.L; ++l) {
        const LevelView& L = LV.lv[l];
        const int64_t a = da / L.ratio;
        const int64_t na = (N - a * L.span) < L.span ? (N - a * L.span) : L.span;
        acc += L.y[3 * a + c] * (1.0 / (double)na);
      }
      z[dof] = pinned[v] ? 0.0 : acc;
    }
    // stage st and gsh / part are reused: the next iteration's first barrier
    // orders these reads before any overwrite (the prefetch into st waits
    // for it + 2, issued after that barrier)
  }
}

// Direct variant (default): one CTA of 192 threads per subdomain, no staging
// of the packed block -- thread i of group 0 / 1 streams diagonals 1..s_mid /
// s_mid+1.. of row i straight from HBM (two unit-stride loads per diagonal
// across the warp, 8 diagonals unrolled: 16 independent loads in flight per
// thread).  The whole D-block grid is one wave (about 10 CTAs, 60 warps per
// SM), so the loads of every block are in flight at once and no pipeline has
// to fill or drain.  Same sums, same order as the staged variants.
__global__ void __launch_bounds__(APPLY_THREADS, 10)
k_mas_apply_l0_direct(int64_t D, int64_t N, int bs, int m, const double* __restrict__ Bblk,
                      const int* __restrict__ overlay_of, const double* __restrict__ overlay,
                      const double* __restrict__ g, const unsigned char* __restrict__ pinned, LevelViews LV,
                      double* __restrict__ z) {
  __shared__ double gsh[96];
  __shared__ double part[96];
  const int64_t d = LV.d0 + blockIdx.x;
  const int tid = threadIdx.x;
  const int grp = tid >= 96 ? 1 : 0;
  const int i = tid - 96 * grp;
  const int64_t csz = cyc_size(m);
  const int ov = overlay_of ? overlay_of[d] : -1;
  const double* __restrict__ P = (ov >= 0) ? overlay + (int64_t)ov * csz : Bblk + d * csz;
  const int64_t v0 = d * bs;
  const int nd3 = 3 * (int)((N - v0) < bs ? (N - v0) : bs);
  if (tid < m) gsh[tid] = (tid < nd3) ? g[3 * v0 + tid] : 0.0;
  __syncthreads();
  const int smax = m / 2;
  const bool even = (m % 2) == 0;
  const int s_full = even ? smax - 1 : smax;
  const int s_mid = s_full / 2;
  double acc = 0.0;
  if (i < nd3) {
    const int s0 = grp ? s_mid + 1 : 1, s1 = grp ? s_full : s_mid;
    if (!grp) acc = __ldcs(P + i) * gsh[i];
    // 8 diagonals per step: all 16 loads issued before the first use, so a
    // thread waits one memory latency per 8 diagonals, not per diagonal
    int s = s0;
    for (; s + 7 <= s1; s += 8) {
      double a[8], b[8];
      int jp[8], jm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        jp[u] = i + s + u; if (jp[u] >= m) jp[u] -= m;
        jm[u] = i - s - u; if (jm[u] < 0) jm[u] += m;
        const double* dg = P + (int64_t)(s + u) * m;
        a[u] = __ldcs(dg + i);
        b[u] = __ldcs(dg + jm[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += a[u] * gsh[jp[u]] + b[u] * gsh[jm[u]];
    }
    for (; s <= s1; ++s) {
      const double* dg = P + (int64_t)s * m;
      int jp = i + s; if (jp >= m) jp -= m;
      int jm = i - s; if (jm < 0) jm += m;
      acc += __ldcs(dg + i) * gsh[jp] + __ldcs(dg + jm) * gsh[jm];
    }
    if (grp && even) {
      const double* dg = P + (int64_t)smax * m;
      int jp = i + smax; if (jp >= m) jp -= m;
      acc += __ldcs(dg + (i < jp ? i : jp)) * gsh[jp];
    }
    if (grp) part[i] = acc;
  }
  __syncthreads();
  if (!grp && i < nd3) {
    acc += part[i];
    const int64_t dof = 3 * v0 + i;
    const int64_t v = v0 + i / 3;
    const int c = i - 3 * (i / 3);
    for (int l = 0; l < LV.L; ++l) {
      const LevelView& L = LV.lv[l];
      const int64_t a = d / L.ratio;
      const int64_t na = (N - a * L.span) < L.span ? (N - a * L.span) : L.span;
      acc += L.y[3 * a + c] * (1.0 / (double)na);
    }
    z[dof] = pinned[v] ? 0.0 : acc;
  }
}

// z += C_l^T y_l over the levels (the prolongation of the level-0 kernel,
// same order), pinned rows 0; rows of [v0, v1)
__global__ void k_prolong(int64_t v0, int64_t v1, int64_t N, int bs, const unsigned char* __restrict__ pinned,
                          LevelViews LV, double* __restrict__ z) {
  const int64_t dof = 3 * v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (dof >= 3 * v1) return;
  const int64_t v = dof / 3;
  const int c = (int)(dof - 3 * v);
  const int64_t d = v / bs;
  double acc = z[dof];
  for (int l = 0; l < LV.L; ++l) {
    const LevelView& L = LV.lv[l];
    const int64_t a = d / L.ratio;
    const int64_t na = (N - a * L.span) < L.span ? (N - a * L.span) : L.span;
    acc += L.y[3 * a + c] * (1.0 / (double)na);
  }
  z[dof] = pinned[v] ? 0.0 : acc;
}

// ---------------------------------------------------------------------------
// Sparse-Input Woodbury build, one CTA per touched subdomain.
// smem: B (m x m full), U (m x K), W (m x K), cap (K x K)

__global__ void k_woodbury(int64_t N, int bs, int m, int Kmax, const double* __restrict__ Bblk,
                           const int* __restrict__ tsub, const int* __restrict__ tstart, const int* __restrict__ tlen,
                           const int* __restrict__ ecand, const int4* __restrict__ cverts,
                           const double* __restrict__ cu, double* __restrict__ overlay, int* __restrict__ status,
                           int64_t d0, int64_t d1) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  const int d = tsub[t];
  const int K = tlen[t];
  if (K > Kmax) return;       // handled by k_direct_update
  if (d < d0 || d >= d1) return;  // another shard's subdomain
  double* B = sm;
  double* U = B + m * m;
  double* W = U + m * Kmax;
  double* C = W + m * Kmax;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  load_cyc_full(Bblk + (int64_t)d * cyc_size(m), m, B);
  for (int e = threadIdx.x; e < m * K; e += blockDim.x) U[e] = 0.0;
  __syncthreads();
  // U columns: candidate rows restricted to this subdomain (woodbury.py:46-54)
  for (int col = threadIdx.x; col < K; col += blockDim.x) {
    int ci = ecand[tstart[t] + col];
    int4 v = cverts[ci];
    const int id[4] = {v.x, v.y, v.z, v.w};
    for (int a = 0; a < 4; ++a) {
      if (id[a] / bs != d) continue;
      int l = id[a] - d * bs;
      for (int r = 0; r < 3; ++r) U[(3 * l + r) * K + col] = cu[12 * (int64_t)ci + 3 * a + r];
    }
  }
  __syncthreads();
  // W = B U using only the non-zero rows of U (sparse input)
  for (int e = threadIdx.x; e < m * K; e += blockDim.x) {
    int i = e / K, col = e % K;
    double s = 0.0;
    for (int r = 0; r < m; ++r) {
      double u = U[r * K + col];
      if (u != 0.0) s += B[i * m + r] * u;
    }
    W[e] = s;
  }
  __syncthreads();
  // cap = I + U^T W, symmetrised (woodbury.py:71-72)
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    int a = e / K, b = e % K;
    double s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < m; ++r) {
      s1 += U[r * K + a] * W[r * K + b];
      s2 += U[r * K + b] * W[r * K + a];
    }
    C[e] = (a == b ? 1.0 : 0.0) + 0.5 * (s1 + s2);
  }
  smem_cholesky(C, K, &bad);
  if (bad) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  // Y = W L^-T (row i: solve L y = W[i,:]^T) written over W
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double* w = W + i * K;
    for (int a = 0; a < K; ++a) {
      double s = w[a];
      for (int b = 0; b < a; ++b) s -= C[a * K + b] * w[b];
      w[a] = s / C[a * K + a];
    }
  }
  __syncthreads();
  // B~ = B - Y Y^T, stored packed
  const int64_t tot = cyc_size(m);
  double* out = overlay + (int64_t)t * tot;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    int s = (int)(e / m);
    int i = (int)(e - (int64_t)s * m);
    int j = i + s;
    if (j >= m) j -= m;
    double acc = 0.0;
    for (int a = 0; a < K; ++a) acc += W[i * K + a] * W[j * K + a];
    out[e] = 0.5 * (B[i * m + j] + B[j * m + i]) - acc;
  }
}

// direct path for large K_d: overlay = sym((M_d + U U^T)^-1)
__global__ void k_direct_update(int64_t N, int bs, int m, const double* __restrict__ Mblk,
                                const int* __restrict__ tsub, const int* __restrict__ tstart,
                                const int* __restrict__ tlen, const int* __restrict__ ecand,
                                const int4* __restrict__ cverts, const double* __restrict__ cu, int Kthresh,
                                double* __restrict__ overlay, int* __restrict__ status, int64_t d0, int64_t d1) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  const int K = tlen[t];
  if (K <= Kthresh) return;
  const int d = tsub[t];
  if (d < d0 || d >= d1) return;  // another shard's subdomain
  double* A = sm;
  double* X = sm + m * m;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  load_cyc_full(Mblk + (int64_t)d * cyc_size(m), m, A);
  __syncthreads();
  // add u u^T restricted to the subdomain, one candidate at a time
  for (int col = 0; col < K; ++col) {
    int ci = ecand[tstart[t] + col];
    int4 v = cverts[ci];
    const int id[4] = {v.x, v.y, v.z, v.w};
    for (int e = threadIdx.x; e < 144; e += blockDim.x) {
      int p = e / 12, q = e % 12;
      int a = p / 3, r = p % 3, b = q / 3, cc = q % 3;
      if (id[a] / bs != d || id[b] / bs != d) continue;
      int la = id[a] - d * bs, lb = id[b] - d * bs;
      A[(3 * la + r) * m + 3 * lb + cc] += cu[12 * (int64_t)ci + p] * cu[12 * (int64_t)ci + q];
    }
    __syncthreads();
  }
  smem_cholesky(A, m, &bad);
  if (bad) {
    if (threadIdx.x == 0) atomicExch(status, 1);
    return;
  }
  smem_chol_inverse(A, m, X);
  store_cyc_sym(X, m, overlay + (int64_t)t * cyc_size(m), true);
}
