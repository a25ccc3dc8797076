// coarse.cuh -- dense SPD inverse of a coarse MAS level, the coarse-level
// _spd_inverse of the reference (mas.py:84-90 applied at mas.py:167), as ONE
// persistent kernel: no library calls, one launch per level per rebuild.
//
// Algorithm: the symmetric sweep operator (Gauss-Jordan without pivoting,
// stable for SPD) in 32-wide pivot panels.  After panel K is swept,
//   A_KK <- -A_KK^-1,  A_IK <- W_I = A_IK A_KK^-1,  A_KI <- W_I^T,
//   A_IJ <- A_IJ - W_I A_JK^T                          (I, J != K)
// and after the last panel A = -M^-1.  Its pivots are the Schur-complement
// diagonals (the squared Cholesky pivots), so "pivot <= 0" is exactly
// cho_factor's non-SPD failure (mas.py:86-88).
//
// Layout: only the lower triangle of 32 x 32 tiles is kept, tile-major
// (tile (I, J <= I) is 1024 contiguous doubles, row-major inside) -- n^2/2
// doubles of traffic per panel instead of n^2.  A panel's old column
// A_{., K} is kept in a double-buffered column buffer written by the
// previous phase, so the in-place update of phase K never races with its
// readers: one grid barrier per panel.
//
// Work split per phase: a unit = (row tile I, chunk of <= 8 column tiles);
// a unit recomputes W_I (32 x 32 x 32, +1/8 work) and updates its tiles
// with a 4 x 8 register tile per thread (12 shared loads per 32 FMA).
// Every CTA sweeps the 32 x 32 pivot block itself (32 barrier steps):
// redundant, but it saves a second grid barrier per panel.
#pragma once

#include "common.cuh"

#define CS_TB 32       // tile edge (= pivot panel width)
#define CS_CH 8        // column tiles per work unit
#define CS_LD 33       // padded smem row stride
#define CS_THREADS 256

struct CoarseSweepArgs {
  int n;                     // matrix order
  int nT;                    // tiles per side (n padded to 32 nT)
  int n_units;               // work units per phase
  const int2* units;         // (row tile I, first column tile J0) per unit
  int ch;                    // column tiles per unit (<= CS_CH; chosen so the units fill the SMs)
  const double* dense;       // n x n assembled M (row-major, both halves valid)
  double* tiles;             // lower tiles, tile-major
  double* colbuf;            // 2 x nT x 1024: panel column A_{I,K} (row-major (i, k))
  double* inv;               // cyc_size(n) packed sym(M^-1)
  int* status;               // set to 1 when a pivot is not positive
  unsigned* bar;             // [0] arrival count, [1] generation
  double* pmbuf;             // nT x 1024: -A_KK^-1 of each panel, published by the lookahead CTA
  double* dbuf;              // nT x 1024: diagonal tile (K+1, K+1) as phase K starts (lookahead input)
  int prof;                  // debug: CTA 0 prints per-phase %globaltimer splits (MP_CS_PROF)
};

__device__ __forceinline__ unsigned long long cs_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int64_t cs_tile(int I, int J) { return ((int64_t)I * (I + 1) / 2 + J) * 1024; }

// sense-free generation barrier over all CTAs of the (co-resident) grid
__device__ __forceinline__ void cs_grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// The whole CTA sweeps the 32 x 32 pivot block (row-major in global) ->
// Pm = -P^-1 in smem (row-major, stride CS_LD).  Thread t holds row t/8,
// columns 4(t%8)..+3 in registers; the matrix stays symmetric, so the pivot
// row (double-buffered in rk, published by its owners after their update)
// doubles as the pivot column: one barrier per pivot (~5 us for 32; a
// one-warp shuffle-only variant measured 25-31 us).  Returns false
// (uniformly) when a pivot is not positive.  Reads bypass L1 (__ldcg): the
// buffers are rewritten by other CTAs between grid barriers.
__device__ bool cs_pivot_sweep(const double* __restrict__ P, double* Pm, double* rk) {
  const int t = threadIdx.x, i = t >> 3, j0 = (t & 7) * 4;
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = __ldcg(P + i * 32 + j0 + q);
  if (i == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) rk[j0 + q] = v[q];
  for (int k = 0; k < 32; ++k) {
    const double* r = rk + (k & 1) * 32;
    __syncthreads();
    // the step's shared loads all issue before the pivot test
    const double piv = r[k], rik = r[i];
    double rkj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) rkj[q] = r[j0 + q];
    if (!(piv > 0.0)) return false;  // uniform across the CTA
    double inv;  // 1/piv to ~1 ulp: MUFU seed + two Newton steps (the IEEE
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(piv));  // division sits on the serial path)
    double e = fma(-piv, inv, 1.0);
    inv = fma(inv, e, inv);
    e = fma(-piv, inv, 1.0);
    inv = fma(inv, e, inv);
    const double cik = rik * inv;   // A_ik / A_kk (= A_ki / A_kk)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      const double ckj = rkj[q];
      v[q] = (i == k) ? ((j == k) ? -inv : ckj * inv) : ((j == k) ? cik : fma(-cik, ckj, v[q]));
    }
    if (i == k + 1 && k + 1 < 32)
#pragma unroll
      for (int q = 0; q < 4; ++q) rk[((k + 1) & 1) * 32 + j0 + q] = v[q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) Pm[i * CS_LD + j0 + q] = v[q];
  return true;
}

// W = A_IK A_KK^-1 = -C Pm (C = A_IK row-major in smem), 4 outputs per thread
__device__ __forceinline__ void cs_compute_W(const double* Csm, const double* Pm, double* Wsm) {
  const int i = threadIdx.x >> 3, j0 = (threadIdx.x & 7) * 4;
  double w4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int d = 0; d < 32; ++d) {
    const double a = Csm[i * CS_LD + d];
#pragma unroll
    for (int q = 0; q < 4; ++q) w4[q] = fma(-a, Pm[d * CS_LD + j0 + q], w4[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) Wsm[i * CS_LD + j0 + q] = w4[q];
}

// A unit's panel tiles into registers: pre[0] = A_IK, pre[1 + q] = A_{J0+q, K};
// element w = tid + 256 s of each tile.  Unrolled, predicated: every load is
// in flight at once.
__device__ __forceinline__ void cs_load_unit(const double* __restrict__ cur, int2 uc, int K, int ch,
                                             double (&pre)[1 + CS_CH][4]) {
  const int I = uc.x, J0 = uc.y, nq = min(ch, I + 1 - J0);
  const bool live = I != K;
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4) {
    const int w = threadIdx.x + CS_THREADS * s4;
    pre[0][s4] = live ? __ldcg(cur + (int64_t)I * 1024 + w) : 0.0;
#pragma unroll
    for (int q = 0; q < CS_CH; ++q) pre[1 + q][s4] = (live && q < nq) ? __ldcg(cur + (int64_t)(J0 + q) * 1024 + w) : 0.0;
  }
}

__global__ void __launch_bounds__(CS_THREADS, 1) k_coarse_sweep(CoarseSweepArgs A) {
  extern __shared__ double cs_sm[];
  double* Pm = cs_sm;                        // 32 x CS_LD: -A_KK^-1
  double* Wsm = Pm + 32 * CS_LD;             // 32 x CS_LD: W_I, then own column tile
  double* Csm = Wsm + 32 * CS_LD;            // 32 x CS_LD: own A_IK (row-major)
  double* Bsm = Csm + 32 * CS_LD;            // CS_CH x 32 x CS_LD: A_JK^T (k-major) per column tile
  const int tid = threadIdx.x;
  const int n = A.n, nT = A.nT;
  const int G = gridDim.x;

  // ---- setup: lower tiles (identity padding) and the first panel column ----
  {
    const int64_t tot = (int64_t)nT * (nT + 1) / 2 * 1024;
    for (int64_t e = blockIdx.x * (int64_t)CS_THREADS + tid; e < tot; e += (int64_t)G * CS_THREADS) {
      const int64_t t = e >> 10;
      const int w = (int)(e & 1023);
      // tile index t -> (I, J): I(I+1)/2 <= t
      int I = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
      while ((int64_t)(I + 1) * (I + 2) / 2 <= t) ++I;
      while ((int64_t)I * (I + 1) / 2 > t) --I;
      const int J = (int)(t - (int64_t)I * (I + 1) / 2);
      const int i = 32 * I + (w >> 5), j = 32 * J + (w & 31);
      const double v = (i < n && j < n) ? A.dense[(int64_t)i * n + j] : (i == j ? 1.0 : 0.0);
      A.tiles[e] = v;
      if (J == 0) A.colbuf[(int64_t)I * 1024 + w] = v;
      if (J == I) A.dbuf[(int64_t)I * 1024 + w] = v;
    }
  }
  cs_grid_sync(A.bar);

  for (int K = 0; K < nT; ++K) {
    const double* cur = A.colbuf + (int64_t)(K & 1) * nT * 1024;
    double* nxt = A.colbuf + (int64_t)((K + 1) & 1) * nT * 1024;
    // CTA 0 is the lookahead CTA (when there are others): it publishes
    // -A_{K+1,K+1}^-1 for the next phase; the units are spread over the rest
    const int G1 = G > 1 ? G - 1 : 1;
    const int self = G > 1 ? (int)blockIdx.x - 1 : 0;
    // the first unit's panel tiles are fetched before the pivot block (all
    // loads in flight in registers, hiding the L2 latency)
    double pre[1 + CS_CH][4];
    const unsigned long long t0 = A.prof ? cs_now() : 0ull;
    int u = self;
    if (self >= 0 && u < A.n_units) cs_load_unit(cur, A.units[u], K, A.ch, pre);
    // (1) Pm = -A_KK^-1: swept by every CTA at K = 0, then published one phase ahead
    if (K == 0) {
      const bool ok0 = cs_pivot_sweep(cur, Pm, Wsm);
      __syncthreads();
      if (!ok0) {  // the same bits in every CTA: all leave together
        if (blockIdx.x == 0 && tid == 0) atomicExch(A.status, 1);
        return;
      }
    } else {
      for (int w = tid; w < 1024; w += CS_THREADS) Pm[(w >> 5) * CS_LD + (w & 31)] = __ldcg(A.pmbuf + (int64_t)K * 1024 + w);
      __syncthreads();
    }
    const unsigned long long t1 = A.prof ? cs_now() : 0ull;
    // (1b) lookahead: the diagonal tile (K+1, K+1) after this phase's update
    // -- the same operations in the same order as its owner unit, so the
    // same bits -- swept at once; its inverse is the next phase's Pm
    if (blockIdx.x == 0 && K + 1 < nT) {
      const double* ck = cur + (int64_t)(K + 1) * 1024;  // A_{K+1,K}
      for (int w = tid; w < 1024; w += CS_THREADS) {
        const double a = __ldcg(ck + w);
        Csm[(w >> 5) * CS_LD + (w & 31)] = a;
        Bsm[(w & 31) * CS_LD + (w >> 5)] = a;
      }
      __syncthreads();
      cs_compute_W(Csm, Pm, Wsm);
      __syncthreads();
      const int tr = tid >> 5, tc = tid & 31;
      double acc[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = __ldcg(A.dbuf + (int64_t)(K + 1) * 1024 + (tr * 4 + r) * 32 + tc);
#pragma unroll 4
      for (int d = 0; d < 32; ++d) {
        const double b = Bsm[d * CS_LD + tc];
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r] = fma(-Wsm[(tr * 4 + r) * CS_LD + d], b, acc[r]);
      }
      double* scratch = A.pmbuf + (int64_t)(K + 1) * 1024;  // P' staged here, then overwritten by -P'^-1
#pragma unroll
      for (int r = 0; r < 4; ++r) scratch[(tr * 4 + r) * 32 + tc] = acc[r];
      __syncthreads();
      double* Pn = Bsm + 32 * CS_LD;
      const bool okn = cs_pivot_sweep(scratch, Pn, Csm);
      __syncthreads();
      if (!okn) {
        if (tid == 0) atomicExch(A.status, 1);  // every CTA leaves after this phase's barrier
      } else {
        for (int w = tid; w < 1024; w += CS_THREADS) scratch[w] = Pn[(w >> 5) * CS_LD + (w & 31)];
      }
      __syncthreads();
    }
    for (; self >= 0 && u < A.n_units; u += G1) {
      const int2 uc = A.units[u];
      const int I = uc.x, J0 = uc.y;
      const int c = J0;  // 0 for the row's first unit
      const int J1 = min(J0 + A.ch, I + 1);
      if (I == K) {  // the pivot row: only A_KK <- -P^-1
        if (c == 0)
          for (int w = tid; w < 1024; w += CS_THREADS) A.tiles[cs_tile(K, K) + w] = Pm[(w >> 5) * CS_LD + (w & 31)];
        continue;
      }
      if (u != self) cs_load_unit(cur, uc, K, A.ch, pre);
      // (2) own column tile A_IK (row-major) and the chunk's A_JK (transposed, k-major)
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int w = tid + CS_THREADS * s4;
        Csm[(w >> 5) * CS_LD + (w & 31)] = pre[0][s4];
#pragma unroll
        for (int q = 0; q < CS_CH; ++q)
          if (q < J1 - J0) Bsm[q * 32 * CS_LD + (w & 31) * CS_LD + (w >> 5)] = pre[1 + q][s4];
      }
      __syncthreads();
      // (3) the chunk's tiles into registers (rows tr*4 + r, column tc of
      // tile J0 + q) -- issued before W so their latency hides under it --
      // then W_I = A_IK A_KK^-1 = -A_IK Pm
      const int tr = tid >> 5, tc = tid & 31;
      const int nq = J1 - J0;
      double acc[4][CS_CH];
#pragma unroll
      for (int q = 0; q < CS_CH; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r)
          acc[r][q] = (q < nq && J0 + q != K) ? __ldcg(A.tiles + cs_tile(I, J0 + q) + (tr * 4 + r) * 32 + tc) : 0.0;
      cs_compute_W(Csm, Pm, Wsm);
      __syncthreads();
      // (4) the rank-32 update of the chunk's tiles
#pragma unroll 4
      for (int d = 0; d < 32; ++d) {
        double wv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) wv[r] = Wsm[(tr * 4 + r) * CS_LD + d];
#pragma unroll
        for (int q = 0; q < CS_CH; ++q) {
          if (q < nq) {
            const double b = Bsm[q * 32 * CS_LD + d * CS_LD + tc];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r][q] = fma(-wv[r], b, acc[r][q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < CS_CH; ++q) {
        if (q >= nq) continue;
        const int J = J0 + q;
        double* T = A.tiles + cs_tile(I, J);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int i = tr * 4 + r;
          const double v = (J == K) ? Wsm[i * CS_LD + tc] : acc[r][q];  // A_IK <- W_I (I > K)
          T[i * 32 + tc] = v;
          if (I == J && I == K + 2) A.dbuf[(int64_t)I * 1024 + i * 32 + tc] = v;  // next phase's lookahead input
          if (K + 1 < nT) {
            if (J == K + 1) nxt[(int64_t)I * 1024 + i * 32 + tc] = v;       // A_{I,K+1}, I >= K+1
            else if (I == K + 1) nxt[(int64_t)J * 1024 + tc * 32 + i] = v;  // A_{J,K+1} = A_{K+1,J}^T
          }
        }
      }
      // the pivot row's tile (K, I) <- W_I^T for I < K (row K owns no units)
      if (I < K && c == 0) {
        double* T = A.tiles + cs_tile(K, I);
        for (int w = tid; w < 1024; w += CS_THREADS) {
          const int i = w >> 5, j = w & 31;  // (K-row i, I-column j) = W_I(j, i)
          T[w] = Wsm[j * CS_LD + i];
        }
        // A_{I,K+1} for I < K comes from row K+1 (handled above); A_{K,K+1}
        // = W_{K+1}^T is written by row K+1's unit holding column K
      }
      __syncthreads();  // smem reused by the next unit
    }
    const unsigned long long t2 = A.prof ? cs_now() : 0ull;
    cs_grid_sync(A.bar);
    if (A.prof && blockIdx.x == 1 && tid == 0 && K < 4)
      printf("cs phase %d: pivot %llu ns, units %llu ns, barrier %llu ns\n", K, t1 - t0, t2 - t1, cs_now() - t2);
    if (*(volatile int*)A.status) return;  // the lookahead found a non-positive pivot: all leave
  }

  // ---- pack sym(-A) in the cyclic layout (common.cuh) ----
  const int64_t tot = cyc_size(n);
  for (int64_t e = blockIdx.x * (int64_t)CS_THREADS + tid; e < tot; e += (int64_t)G * CS_THREADS) {
    const int s = (int)(e / n);
    const int i = (int)(e - (int64_t)s * n);
    int j = i + s;
    if (j >= n) j -= n;
    const int r = i > j ? i : j, cc = i > j ? j : i;  // lower representative
    const int I = r >> 5, J = cc >> 5;
    double v = __ldcg(A.tiles + cs_tile(I, J) + (r & 31) * 32 + (cc & 31));
    if (I == J) v = 0.5 * (v + __ldcg(A.tiles + cs_tile(I, J) + (cc & 31) * 32 + (r & 31)));
    A.inv[e] = -v;
  }
}

static size_t coarse_sweep_smem() { return sizeof(double) * (3 * 32 * CS_LD + CS_CH * 32 * CS_LD); }
