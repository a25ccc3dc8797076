// ops.cuh -- fused vector reductions and small vector kernels.
//
// Every PNCG scalar of one iteration (norms and the dots of the 2x2
// subspace system, solver.py:357-392, 444) comes out of ONE pass over the
// vectors: k_multidot accumulates up to MAX_DOTS products per thread, writes
// per-block partials, and k_multidot_final sums them in a fixed order
// (deterministic, no atomics).
#pragma once

#include "ctx.cuh"

#define MAX_DOTS 10
#define RED_BLOCKS 296  // 2 x 148 SMs
#define RED_THREADS 256

struct DotSpec {
  const double* a[MAX_DOTS];
  const double* b[MAX_DOTS];
  int n;
};

__global__ void k_multidot(int64_t len, DotSpec S, double* __restrict__ part) {
  double acc[MAX_DOTS];
#pragma unroll
  for (int q = 0; q < MAX_DOTS; ++q) acc[q] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int q = 0; q < MAX_DOTS; ++q)
      if (q < S.n) acc[q] += S.a[q][i] * S.b[q][i];
  }
  __shared__ double sh[MAX_DOTS][RED_THREADS / 32];
#pragma unroll
  for (int q = 0; q < MAX_DOTS; ++q) {
    if (q >= S.n) break;
    double v = warp_sum(acc[q]);
    if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < S.n) {
    double t = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) t += sh[threadIdx.x][w];
    part[blockIdx.x * MAX_DOTS + threadIdx.x] = t;
  }
}

// sum partials in block order; mode per slot: 0 sum, 1 max
// one warp per dot: lanes stride over the block partials, fixed shuffle
// tree (reproducible; a single thread walking 296 partials is latency bound)
__global__ void k_multidot_final(int nblocks, int n, const double* __restrict__ part, double* __restrict__ out) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q >= n) return;  // warp-uniform
  double t = 0.0;
  for (int b = lane; b < nblocks; b += 32) t += part[b * MAX_DOTS + q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if (lane == 0) out[q] = t;
}

// returns dots in c->h_scal[0..n)
static void multidot(mp_ctx* c, int64_t len, const DotSpec& S) {
  c->red_part.ensure((size_t)RED_BLOCKS * MAX_DOTS);
  int nb = (int)grid_for(len, RED_THREADS);
  if (nb > RED_BLOCKS) nb = RED_BLOCKS;
  k_multidot<<<nb, RED_THREADS, 0, c->stream>>>(len, S, c->red_part);
  LAUNCH_CHECK();
  k_multidot_final<<<1, 32 * MAX_DOTS, 0, c->stream>>>(nb, S.n, c->red_part, c->dscal);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->dscal.p, sizeof(double) * S.n, cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
}

// p = a z + b pp ; Hp = a v + b Hpp ; partials of g.p and max|p|
__global__ void k_form_dir(int64_t len, double a, double b, const double* __restrict__ z,
                           const double* __restrict__ pp, const double* __restrict__ v,
                           const double* __restrict__ Hpp, const double* __restrict__ g, double* __restrict__ p,
                           double* __restrict__ Hp, double* __restrict__ part) {
  double gp = 0.0, mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    // (-mu z) + (nu p_prev), each product rounded as in solver.py:384-385
    double pi = __dmul_rn(a, z[i]);
    double hi = __dmul_rn(a, v[i]);
    if (pp) {
      pi = __dadd_rn(pi, __dmul_rn(b, pp[i]));
      hi = __dadd_rn(hi, __dmul_rn(b, Hpp[i]));
    }
    p[i] = pi;
    Hp[i] = hi;
    gp += g[i] * pi;
    mx = fmax(mx, fabs(pi));
  }
  __shared__ double s1[RED_THREADS / 32], s2[RED_THREADS / 32];
  gp = warp_sum(gp);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    s1[threadIdx.x >> 5] = gp;
    s2[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, m = 0.0;
    for (int w = 0; w < RED_THREADS / 32; ++w) {
      t += s1[w];
      m = fmax(m, s2[w]);
    }
    part[blockIdx.x * MAX_DOTS] = t;
    part[blockIdx.x * MAX_DOTS + 1] = m;
  }
}

__global__ void k_form_dir_final(int nblocks, const double* __restrict__ part, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  double t = 0.0, m = 0.0;
  for (int b = lane; b < nblocks; b += 32) {
    t += part[b * MAX_DOTS];
    m = fmax(m, part[b * MAX_DOTS + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  if (lane == 0) {
    out[0] = t;
    out[1] = m;
  }
}

// p, Hp formed on device; returns (g.p, max|p|) in h_scal[0..1]
static void form_direction(mp_ctx* c, double a, double b, const double* pp, const double* Hpp) {
  const int64_t len = 3 * c->N;
  c->red_part.ensure((size_t)RED_BLOCKS * MAX_DOTS);
  int nb = (int)grid_for(len, RED_THREADS);
  if (nb > RED_BLOCKS) nb = RED_BLOCKS;
  k_form_dir<<<nb, RED_THREADS, 0, c->stream>>>(len, a, b, c->z, pp, c->hv, Hpp, c->g, c->p, c->Hp, c->red_part);
  LAUNCH_CHECK();
  k_form_dir_final<<<1, 32, 0, c->stream>>>(nb, c->red_part, c->dscal);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->dscal.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
}

__global__ void k_velocity(int64_t N, const double* __restrict__ x, const double* __restrict__ x0, double h,
                           const unsigned char* __restrict__ pinned, double* __restrict__ v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  v[i] = pinned[i / 3] ? 0.0 : (x[i] - x0[i]) / h;
}

// prepare_step on device (energy.py:77-94)
__global__ void k_prepare(int64_t N, const double* __restrict__ x, double* __restrict__ v,
                          const double* __restrict__ mass, const double* __restrict__ f_ext,
                          const unsigned char* __restrict__ pinned, double h, double* __restrict__ xt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  int64_t vtx = i / 3;
  double m = mass[vtx];
  double acc = (m > 0.0) ? f_ext[i] / m : 0.0;
  if (pinned[vtx]) {
    xt[i] = x[i];
    v[i] = 0.0;
  } else {
    xt[i] = __dadd_rn(__dadd_rn(x[i], __dmul_rn(h, v[i])), __dmul_rn(__dmul_rn(h, h), acc));
  }
}

// original order <-> subdomain order (flat 3N vectors)
__global__ void k_to_new(int64_t N, const int* __restrict__ new2old, const double* __restrict__ src,
                         double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  int64_t v = i / 3;
  dst[i] = src[3 * (int64_t)new2old[v] + (i % 3)];
}

__global__ void k_to_old(int64_t N, const int* __restrict__ new2old, const double* __restrict__ src,
                         double* __restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  int64_t v = i / 3;
  dst[3 * (int64_t)new2old[v] + (i % 3)] = src[i];
}
