// check.cuh -- the scalable penetration checker.
//
// The reference checker (cli.py:360-422) certifies an emitted frame by
//   (1) the minimum distance over all non-adjacent point-triangle and
//       edge-edge surface pairs (brute force, O(V F + E^2)), and
//   (2) a triangle-triangle intersection test over all non-adjacent
//       triangle pairs (a Python double loop, O(F^2); geometry.py:686-732).
// Here (1) runs through the solver's own broad phase and distance kernels
// (a surface-only context, mp_constraint_set with d_hat = the search radius,
// doubled until pairs are found -- exact: every pair closer than the radius
// is a candidate), and (2) is this file: triangles binned into a uniform
// grid (every cell its box covers), entries radix-sorted by cell, each pair
// tested once in the first cell both boxes share, boxes first, then the
// exact test with the reference's decision rules (touching counts, the
// coplanar case in 2-D on the dominant axes).
#pragma once

#include "bp.cuh"

struct TriBox {
  double lo[3], hi[3];
};

__global__ void k_tri_boxes(int64_t F, const double* __restrict__ x, const int* __restrict__ tri,
                            TriBox* __restrict__ box, unsigned long long* __restrict__ ext_bits) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double e = 0.0;
  if (f < F) {
    TriBox b;
    for (int k = 0; k < 3; ++k) {
      double a0 = x[3 * (int64_t)tri[3 * f] + k], a1 = x[3 * (int64_t)tri[3 * f + 1] + k],
             a2 = x[3 * (int64_t)tri[3 * f + 2] + k];
      b.lo[k] = fmin(a0, fmin(a1, a2));
      b.hi[k] = fmax(a0, fmax(a1, a2));
      e += b.hi[k] - b.lo[k];
    }
    box[f] = b;
  }
  // mean extent: sum of (sum of the 3 extents) in 2^-40 fixed point (order-free)
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0 && e > 0.0) atomicAdd(ext_bits, (unsigned long long)(e * 1099511627776.0 / 3.0));
}

struct GridSpec {
  double lo[3];
  double inv_h;
  int dim[3];
};

__device__ __forceinline__ void cell_range(const GridSpec& G, const TriBox& b, int c0[3], int c1[3]) {
  for (int k = 0; k < 3; ++k) {
    c0[k] = max(0, min(G.dim[k] - 1, (int)floor((b.lo[k] - G.lo[k]) * G.inv_h)));
    c1[k] = max(0, min(G.dim[k] - 1, (int)floor((b.hi[k] - G.lo[k]) * G.inv_h)));
  }
}

__device__ __forceinline__ unsigned long long cell_key(const GridSpec& G, int i, int j, int k) {
  return ((unsigned long long)i * G.dim[1] + j) * G.dim[2] + k;
}

__global__ void k_tri_count(int64_t F, const TriBox* __restrict__ box, GridSpec G, int* __restrict__ cnt) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= F) return;
  int c0[3], c1[3];
  cell_range(G, box[f], c0, c1);
  cnt[f] = (c1[0] - c0[0] + 1) * (c1[1] - c0[1] + 1) * (c1[2] - c0[2] + 1);
}

__global__ void k_tri_fill(int64_t F, const TriBox* __restrict__ box, GridSpec G, const int* __restrict__ off,
                           unsigned long long* __restrict__ key, int* __restrict__ val) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f >= F) return;
  int c0[3], c1[3];
  cell_range(G, box[f], c0, c1);
  int o = off[f];
  for (int i = c0[0]; i <= c1[0]; ++i)
    for (int j = c0[1]; j <= c1[1]; ++j)
      for (int k = c0[2]; k <= c1[2]; ++k) {
        key[o] = cell_key(G, i, j, k);
        val[o] = (int)f;
        ++o;
      }
}

// ---- exact triangle-triangle test (geometry.py:686-732 decision rules) ----

__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

__device__ bool seg_seg_2d(const double p0[2], const double p1[2], const double q0[2], const double q1[2]) {
  const double d1x = p1[0] - p0[0], d1y = p1[1] - p0[1], d2x = q1[0] - q0[0], d2y = q1[1] - q0[1];
  const double den = d1x * d2y - d1y * d2x;
  const double rx = q0[0] - p0[0], ry = q0[1] - p0[1];
  if (den == 0.0) {  // parallel: collinear overlap only
    if (rx * d1y - ry * d1x != 0.0) return false;
    const double tt = d1x * d1x + d1y * d1y;
    if (tt == 0.0) return false;
    const double t0 = (rx * d1x + ry * d1y) / tt;
    const double t1 = t0 + (d2x * d1x + d2y * d1y) / tt;
    return fmax(fmin(t0, t1), 0.0) <= fmin(fmax(t0, t1), 1.0);
  }
  const double s = (rx * d2y - ry * d2x) / den, t = (rx * d1y - ry * d1x) / den;
  return s >= 0.0 && s <= 1.0 && t >= 0.0 && t <= 1.0;
}

__device__ bool point_in_tri_2d(const double p[2], const double a[2], const double b[2], const double c[2]) {
  const double s1 = (b[0] - a[0]) * (p[1] - a[1]) - (b[1] - a[1]) * (p[0] - a[0]);
  const double s2 = (c[0] - b[0]) * (p[1] - b[1]) - (c[1] - b[1]) * (p[0] - b[0]);
  const double s3 = (a[0] - c[0]) * (p[1] - c[1]) - (a[1] - c[1]) * (p[0] - c[0]);
  const bool neg = s1 < 0 || s2 < 0 || s3 < 0, pos = s1 > 0 || s2 > 0 || s3 > 0;
  return !(neg && pos);
}

// the triangle's slice of the plane-plane line, projected on `axis`
__device__ void tri_interval(const double t[3][3], const double dist[3], int axis, double& lo, double& hi) {
  lo = INFINITY;
  hi = -INFINITY;
  for (int i = 0; i < 3; ++i)
    if (dist[i] == 0.0) {
      lo = fmin(lo, t[i][axis]);
      hi = fmax(hi, t[i][axis]);
    }
  for (int i = 0; i < 3; ++i) {
    if (!(dist[i] > 0.0)) continue;
    for (int j = 0; j < 3; ++j) {
      if (!(dist[j] < 0.0)) continue;
      const double f = dist[i] / (dist[i] - dist[j]);
      const double v = t[i][axis] + f * (t[j][axis] - t[i][axis]);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
  }
}

__device__ bool tri_tri_intersect(const double a[3][3], const double b[3][3], double coplanar_tol) {
  double e1[3], e2[3], n1[3], n2[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = a[1][k] - a[0][k];
    e2[k] = a[2][k] - a[0][k];
  }
  cross3(e1, e2, n1);
  for (int k = 0; k < 3; ++k) {
    e1[k] = b[1][k] - b[0][k];
    e2[k] = b[2][k] - b[0][k];
  }
  cross3(e1, e2, n2);
  double db[3], da[3];
  const double oa = dot3(a[0], n1), ob = dot3(b[0], n2);
  for (int i = 0; i < 3; ++i) db[i] = dot3(b[i], n1) - oa;
  if ((db[0] > 0 && db[1] > 0 && db[2] > 0) || (db[0] < 0 && db[1] < 0 && db[2] < 0)) return false;
  for (int i = 0; i < 3; ++i) da[i] = dot3(a[i], n2) - ob;
  if ((da[0] > 0 && da[1] > 0 && da[2] > 0) || (da[0] < 0 && da[1] < 0 && da[2] < 0)) return false;
  // coplanar to rounding (|vertex-plane distance| <= coplanar_tol x the
  // longest edge) takes the 2-D test: the reference's exact == 0 test sends
  // such pairs through the interval test along an ill-defined plane-plane
  // line and reports disjoint coplanar triangles as intersecting (DESIGN.md
  // 4: two voxel faces 1.1 mm apart flagged by ipcsim's own function)
  double L2 = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      const double ea = a[(i + 1) % 3][k] - a[i][k], eb = b[(i + 1) % 3][k] - b[i][k];
      L2 = fmax(L2, fmax(ea * ea, eb * eb));
    }
  const double tb = coplanar_tol * sqrt(L2 * dot3(n1, n1)), ta = coplanar_tol * sqrt(L2 * dot3(n2, n2));
  const bool cop_b = fabs(db[0]) <= tb && fabs(db[1]) <= tb && fabs(db[2]) <= tb;
  const bool cop_a = fabs(da[0]) <= ta && fabs(da[1]) <= ta && fabs(da[2]) <= ta;
  if (cop_b || cop_a) {
    // coplanar: drop the dominant axis of n1 and test in 2-D
    int ax = 0;
    if (fabs(n1[1]) > fabs(n1[ax])) ax = 1;
    if (fabs(n1[2]) > fabs(n1[ax])) ax = 2;
    const int u = ax == 0 ? 1 : 0, v = ax == 2 ? 1 : 2;
    double p[3][2], q[3][2];
    for (int i = 0; i < 3; ++i) {
      p[i][0] = a[i][u]; p[i][1] = a[i][v];
      q[i][0] = b[i][u]; q[i][1] = b[i][v];
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        if (seg_seg_2d(p[i], p[(i + 1) % 3], q[j], q[(j + 1) % 3])) return true;
    return point_in_tri_2d(p[0], q[0], q[1], q[2]) || point_in_tri_2d(q[0], p[0], p[1], p[2]);
  }
  double line[3];
  cross3(n1, n2, line);
  int ax = 0;
  if (fabs(line[1]) > fabs(line[ax])) ax = 1;
  if (fabs(line[2]) > fabs(line[ax])) ax = 2;
  double lo1, hi1, lo2, hi2;
  tri_interval(a, da, ax, lo1, hi1);
  tri_interval(b, db, ax, lo2, hi2);
  return fmax(lo1, lo2) <= fmin(hi1, hi2);
}

// one thread per (entry, later entry of the same cell) scan; a pair is
// tested only in the first cell both boxes cover
__global__ void k_tri_pairs(int64_t n_ent, const unsigned long long* __restrict__ key, const int* __restrict__ val,
                            const TriBox* __restrict__ box, GridSpec G, const double* __restrict__ x,
                            const int* __restrict__ tri, double coplanar_tol, unsigned long long* __restrict__ hits,
                            int* __restrict__ first_hit) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_ent) return;
  const unsigned long long k = key[e];
  const int fa = val[e];
  const TriBox ba = box[fa];
  const int ia[3] = {tri[3 * fa], tri[3 * fa + 1], tri[3 * fa + 2]};
  int ca0[3], ca1[3];
  cell_range(G, ba, ca0, ca1);
  for (int64_t o = e + 1; o < n_ent && key[o] == k; ++o) {
    const int fb = val[o];
    const TriBox bb = box[fb];
    bool overlap = true;
    for (int d = 0; d < 3; ++d) overlap = overlap && ba.lo[d] <= bb.hi[d] && bb.lo[d] <= ba.hi[d];
    if (!overlap) continue;
    const int ib[3] = {tri[3 * fb], tri[3 * fb + 1], tri[3 * fb + 2]};
    bool shared = false;
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) shared = shared || ia[p] == ib[q];
    if (shared) continue;
    int cb0[3], cb1[3];
    cell_range(G, bb, cb0, cb1);
    const unsigned long long first = cell_key(G, max(ca0[0], cb0[0]), max(ca0[1], cb0[1]), max(ca0[2], cb0[2]));
    if (first != k) continue;  // counted in the first shared cell
    double A[3][3], B[3][3];
    for (int p = 0; p < 3; ++p)
      for (int d = 0; d < 3; ++d) {
        A[p][d] = x[3 * (int64_t)ia[p] + d];
        B[p][d] = x[3 * (int64_t)ib[p] + d];
      }
    if (tri_tri_intersect(A, B, coplanar_tol)) {
      atomicAdd(hits, 1ull);
      atomicMin(first_hit, min(fa, fb));
    }
  }
}

// number of intersecting non-adjacent triangle pairs of the surface at x
// (x and tri in the caller's numbering, on the device)
static unsigned long long tri_intersections(mp_ctx* c, const double* x, const int* tri, int64_t F, int* first,
                                            double coplanar_tol) {
  cudaStream_t st = c->stream;
  DBuf<TriBox> box;
  box.ensure(F);
  c->n_pairs_dev.ensure(2);
  CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, 2 * sizeof(unsigned long long), st));
  k_tri_boxes<<<grid_for(F, 256), 256, 0, st>>>(F, x, tri, box, c->n_pairs_dev.p + 1);
  LAUNCH_CHECK();
  std::vector<TriBox> hb(F);
  unsigned long long ext = 0;
  CUDA_CHECK(cudaMemcpyAsync(hb.data(), box.p, sizeof(TriBox) * F, cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaMemcpyAsync(&ext, c->n_pairs_dev.p + 1, sizeof(ext), cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  GridSpec G{};
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = 0; k < 3; ++k) G.lo[k] = INFINITY;
  for (const TriBox& b : hb)
    for (int k = 0; k < 3; ++k) {
      G.lo[k] = std::min(G.lo[k], b.lo[k]);
      hi[k] = std::max(hi[k], b.hi[k]);
    }
  // cell = 2 x the mean triangle extent, coarsened until the grid has < 2^40 cells
  double h = std::max(2.0 * ((double)ext / 1099511627776.0) / (double)F, 1e-12);
  for (;;) {
    double cells = 1.0;
    for (int k = 0; k < 3; ++k) cells *= std::floor((hi[k] - G.lo[k]) / h) + 1.0;
    if (cells < 1099511627776.0) break;
    h *= 2.0;
  }
  G.inv_h = 1.0 / h;
  for (int k = 0; k < 3; ++k) G.dim[k] = (int)std::floor((hi[k] - G.lo[k]) * G.inv_h) + 1;
  DBuf<int> cnt, off;
  cnt.ensure(F + 1);
  off.ensure(F + 1);
  CUDA_CHECK(cudaMemsetAsync(cnt.p + F, 0, sizeof(int), st));
  k_tri_count<<<grid_for(F, 256), 256, 0, st>>>(F, box, G, cnt);
  LAUNCH_CHECK();
  exclusive_scan(c, cnt, off, F + 1);
  int n_ent = 0;
  CUDA_CHECK(cudaMemcpyAsync(&n_ent, off.p + F, sizeof(int), cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  DBuf<unsigned long long> key, key2;
  DBuf<int> val, val2, fh;
  key.ensure(n_ent); key2.ensure(n_ent); val.ensure(n_ent); val2.ensure(n_ent);
  k_tri_fill<<<grid_for(F, 256), 256, 0, st>>>(F, box, G, off, key, val);
  LAUNCH_CHECK();
  const unsigned long long ncell = (unsigned long long)G.dim[0] * G.dim[1] * G.dim[2];
  sort_pairs_u64(c, key, key2, val, val2, n_ent, bits_for(ncell));
  fh.ensure(1);
  const int big = INT32_MAX;
  CUDA_CHECK(cudaMemcpyAsync(fh.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_tri_pairs<<<grid_for(n_ent, 128), 128, 0, st>>>(n_ent, key2, val2, box, G, x, tri, coplanar_tol,
                                                    c->n_pairs_dev.p, fh);
  LAUNCH_CHECK();
  unsigned long long hits = 0;
  CUDA_CHECK(cudaMemcpyAsync(&hits, c->n_pairs_dev.p, sizeof(hits), cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaMemcpyAsync(first, fh.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  return hits;
}
