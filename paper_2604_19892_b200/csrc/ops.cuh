// ops.cuh -- fused vector reductions and small vector kernels.
//
// Every PNCG scalar of one iteration (norms and the dots of the 2x2
// subspace system, solver.py:357-392, 444) comes out of ONE pass over the
// vectors: k_multidot_chunks writes one partial per chunk (a level-1
// aggregate's dofs) and per dot, and the chunks are summed in chunk order on
// the host (group.cuh group_dots) -- deterministic, no atomics, and the same
// bits on one GPU and on a multi-GPU group.
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

// Per-chunk partials of up to MAX_DOTS dots: chunk q = dofs [q cl, (q+1) cl)
// (cl = 3 x one level-1 aggregate); one CTA per chunk sums in a fixed order.
// The chunks' sum in chunk order (group_dots) does not depend on how the
// chunks are spread over shards or CTAs.
__global__ void k_multidot_chunks(int64_t len, int64_t cl, int64_t q0, DotSpec S, double* __restrict__ part) {
  const int64_t q = q0 + blockIdx.x;
  const int64_t b = q * cl, e = (b + cl < len) ? b + cl : len;
  double acc[MAX_DOTS];
#pragma unroll
  for (int k = 0; k < MAX_DOTS; ++k) acc[k] = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
#pragma unroll
    for (int k = 0; k < MAX_DOTS; ++k)
      if (k < S.n) acc[k] += S.a[k][i] * S.b[k][i];
  }
  __shared__ double sh[MAX_DOTS][4];
#pragma unroll
  for (int k = 0; k < MAX_DOTS; ++k) {
    if (k >= S.n) break;
    const double v = warp_sum(acc[k]);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < S.n) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[threadIdx.x][w];
    part[q * MAX_DOTS + threadIdx.x] = t;
  }
}

// dots over this shard's owned chunks -> group-wide values in c->h_scal[0..n)
// (extra device scalars, if any, land in h_scal[MAX_DOTS..])
static void multidot(mp_ctx* c, int64_t len, const DotSpec& S, const double* extra = nullptr, int n_extra = 0);

// p = a z + b pp ; Hp = a v + b Hpp (elementwise, every row); max|p| into
// *pmax (order-free: atomicMax on the bit pattern of a non-negative double)
__global__ void k_form_dir(int64_t len, double a, double b, const double* __restrict__ z,
                           const double* __restrict__ pp, const double* __restrict__ v,
                           const double* __restrict__ Hpp, double* __restrict__ p, double* __restrict__ Hp,
                           unsigned long long* __restrict__ pmax) {
  double mx = 0.0;
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
    mx = fmax(mx, fabs(pi));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomicMax(pmax, (unsigned long long)__double_as_longlong(mx));
}

// p, Hp formed on device; returns (g.p, max|p|) in h_scal[0..1]
static void form_direction(mp_ctx* c, double a, double b, const double* pp, const double* Hpp) {
  const int64_t len = 3 * c->N;
  unsigned long long* pmax = reinterpret_cast<unsigned long long*>(c->dscal.p + 40);
  CUDA_CHECK(cudaMemsetAsync(pmax, 0, sizeof(unsigned long long), c->stream));
  k_form_dir<<<(unsigned)std::min<int64_t>(grid_for(len, RED_THREADS), RED_BLOCKS), RED_THREADS, 0, c->stream>>>(
      len, a, b, c->z, pp, c->hv, Hpp, c->p, c->Hp, pmax);
  LAUNCH_CHECK();
  DotSpec S{};
  S.a[0] = c->g;
  S.b[0] = c->p;
  S.n = 1;
  multidot(c, len, S, c->dscal.p + 40, 1);
  c->h_scal[1] = c->h_scal[MAX_DOTS];  // max|p| (the bits of a non-negative double)
}

// a - b and c - d, elementwise
__global__ void k_sub2(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ c, const double* __restrict__ d, double* __restrict__ ab,
                       double* __restrict__ cd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  ab[i] = a[i] - b[i];
  cd[i] = c[i] - d[i];
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
