// contact.cuh -- broad phase, constraint set, contact terms, classification,
// per-subdomain Top-K.
//
// Broad phase (geometry.py:443-503).  The reference's membership is its
// exact AABB filter applied to hash-grid candidates:
//   PT (v, t):  v not in t  and  x_v >= lo_t - gap  and  x_v <= hi_t + gap
//   EE (i, j):  i < j, no shared vertex, lo_i <= hi_j + gap, lo_j <= hi_i + gap
// with gap = d_hat + 2 mb.  Here: a uniform grid over our own cell size.
//   PT: each triangle is inserted in every cell its filter box
//       [lo - gap, hi + gap] touches; a vertex queries only its own cell, so
//       each passing pair is seen exactly once (floor((v - o)/c) is monotone,
//       hence the filter box test implies the cell hit).
//   EE: edge boxes [lo, hi + gap]; a pair overlaps iff the filter passes and
//       is reported only in the cell holding max(lo_i, lo_j) (the low corner
//       of the box intersection), so once.
// The filter arithmetic is the reference's (IEEE subtract/add, compare).
#pragma once

#include <cub/cub.cuh>

#include "ctx.cuh"
#include "geom.cuh"

enum { BP_RAW = 0, BP_CONTACT = 1, BP_CCD = 2, BP_CERT = 3 };

// ---------------------------------------------------------------------------
// dense cell grid (our own cell size, independent of the reference's)
//
// Objects inserted in the grid: triangles [0, F), edges [F, F+E) and surface
// points [F+E, F+E+V), each with an ENUMERATION box.  Reference mode
// (infl == nullptr): triangle box = the reference's PT filter box
// [lo - gap, hi + gap], edge box = the EE join box [lo, hi + gap], point box
// = the point.  Tight CCD mode (infl != nullptr, per-vertex inflation):
// every box is the raw box grown by its vertices' largest inflation.  A
// candidate pair is met in every cell both boxes cover and reported only in
// the cell of the low corner of the box intersection.  The reference's own
// membership test is then applied to the pair exactly (queries below).

struct CellGrid {
  double o[3];
  double h;
  int n[3];
};

__device__ __forceinline__ int cg_coord(double v, double o, double h, int n) {
  double q = floor((v - o) / h);  // monotone in v: box overlap implies a shared cell
  if (!(q >= 0.0)) return 0;      // also catches NaN
  if (q > (double)(n - 1)) return n - 1;
  return (int)q;
}

__device__ __forceinline__ int cg_id(const CellGrid& G, int a, int b, int c) { return (a * G.n[1] + b) * G.n[2] + c; }

// Boxes of triangles and edges: raw (rlo, rhi); reference filter (flo, fhi:
// triangle [lo - gap, hi + gap], edge [lo, hi + gap]); enumeration (elo,
// ehi).  The largest raw-box diagonal (the reference's grid cell candidate,
// geometry.py:462-465, same IEEE expression) is max-reduced into *diag_max.
__global__ void k_prim_boxes(int64_t F, int64_t E, const int* __restrict__ tri, const int* __restrict__ edge,
                             const double* __restrict__ x, double gap, const double* __restrict__ infl,
                             double* __restrict__ rlo, double* __restrict__ rhi, double* __restrict__ flo,
                             double* __restrict__ fhi, double* __restrict__ elo, double* __restrict__ ehi,
                             double* __restrict__ diag_max) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double dg = 0.0;
  if (i < F + E) {
    double l[3], h[3], inf = 0.0;
    if (i < F) {
      int a = tri[3 * i], b = tri[3 * i + 1], c = tri[3 * i + 2];
      if (infl) inf = fmax(fmax(infl[a], infl[b]), infl[c]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double xa = x[3 * a + k], xb = x[3 * b + k], xc = x[3 * c + k];
        l[k] = fmin(fmin(xa, xb), xc);
        h[k] = fmax(fmax(xa, xb), xc);
      }
    } else {
      int64_t e = i - F;
      int a = edge[2 * e], b = edge[2 * e + 1];
      if (infl) inf = fmax(infl[a], infl[b]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double xa = x[3 * a + k], xb = x[3 * b + k];
        l[k] = fmin(xa, xb);
        h[k] = fmax(xa, xb);
      }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double dk = RSUB(h[k], l[k]);
      s = (k == 0) ? RMUL(dk, dk) : RADD(s, RMUL(dk, dk));
      const double fl = (i < F) ? RSUB(l[k], gap) : l[k];
      const double fh = RADD(h[k], gap);
      rlo[3 * i + k] = l[k];
      rhi[3 * i + k] = h[k];
      flo[3 * i + k] = fl;
      fhi[3 * i + k] = fh;
      elo[3 * i + k] = infl ? l[k] - inf : fl;
      ehi[3 * i + k] = infl ? h[k] + inf : fh;
    }
    dg = __dsqrt_rn(s);
  }
  dg = warp_max(dg);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(diag_max, dg);
}

// enumeration boxes of the surface points (object ids F+E+q)
__global__ void k_point_boxes(int64_t V, const int* __restrict__ sverts, const double* __restrict__ x,
                              const double* __restrict__ infl, double* __restrict__ elo, double* __restrict__ ehi) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= V) return;
  int v = sverts[q];
  double e = infl ? infl[v] : 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    elo[3 * q + k] = x[3 * v + k] - e;
    ehi[3 * q + k] = x[3 * v + k] + e;
  }
}

// stats for the grid: [0..2] min lo, [3..5] max hi, [6] sum of max extents
__global__ void k_box_stats(int64_t P, const double* __restrict__ lo, const double* __restrict__ hi,
                            double* __restrict__ part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, ext = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    double e = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double l = lo[3 * i + k], h = hi[3 * i + k];
      mn[k] = fmin(mn[k], l);
      mx[k] = fmax(mx[k], h);
      e = fmax(e, h - l);
    }
    ext += e;
  }
  __shared__ double sh[7][8];
  double vals[7] = {-mn[0], -mn[1], -mn[2], mx[0], mx[1], mx[2], ext};
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = vals[q];
    v = (q < 6) ? warp_max(v) : warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < 7; ++q) {
      double v = sh[q][0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = (q < 6) ? fmax(v, sh[q][w]) : v + sh[q][w];
      part[7 * blockIdx.x + q] = v;
    }
  }
}

__device__ __forceinline__ void box_span(const CellGrid& G, const double* lo, const double* hi, int c0[3],
                                         int c1[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c0[k] = cg_coord(lo[k], G.o[k], G.h, G.n[k]);
    c1[k] = cg_coord(hi[k], G.o[k], G.h, G.n[k]);
  }
}

// number of grid cells each object box covers
__global__ void k_cell_span(int64_t n, CellGrid G, const double* __restrict__ lo, const double* __restrict__ hi,
                            int* __restrict__ cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c0[3], c1[3];
  box_span(G, lo + 3 * i, hi + 3 * i, c0, c1);
  long long m = (long long)(c1[0] - c0[0] + 1) * (c1[1] - c0[1] + 1) * (c1[2] - c0[2] + 1);
  cnt[i] = (int)(m > (1 << 30) ? (1 << 30) : m);
}

__device__ __forceinline__ int upper_bound_i32(const int* a, int n, int k) {
  int l = 0, r = n;
  while (l < r) {
    int m = (l + r) >> 1;
    if (a[m] <= k) l = m + 1; else r = m;
  }
  return l;
}

// one thread per (object, covered cell) entry: its cell and the per-class
// per-cell histograms (class 0 triangles, 1 edges, 2 points)
__global__ void k_entry_hist(int64_t total, int64_t nobj, int64_t F, int64_t P, CellGrid G,
                             const int* __restrict__ off, const double* __restrict__ lo, const double* __restrict__ hi,
                             int* __restrict__ ecell, int* __restrict__ tri_cnt, int* __restrict__ edge_cnt,
                             int* __restrict__ pt_cnt) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  int p = upper_bound_i32(off, (int)nobj + 1, (int)e) - 1;
  int r = (int)e - off[p];
  int c0[3], c1[3];
  box_span(G, lo + 3 * (int64_t)p, hi + 3 * (int64_t)p, c0, c1);
  int sx = c1[0] - c0[0] + 1, sy = c1[1] - c0[1] + 1;
  int cell = cg_id(G, c0[0] + r % sx, c0[1] + (r / sx) % sy, c0[2] + r / (sx * sy));
  ecell[e] = cell;
  atomicAdd(p < F ? &tri_cnt[cell] : (p < P ? &edge_cnt[cell] : &pt_cnt[cell]), 1);
}

__global__ void k_entry_fill(int64_t total, int64_t nobj, int64_t F, int64_t P, const int* __restrict__ off,
                             const int* __restrict__ ecell, const int* __restrict__ tri_start,
                             const int* __restrict__ edge_start, const int* __restrict__ pt_start,
                             int* __restrict__ tri_cur, int* __restrict__ edge_cur, int* __restrict__ pt_cur,
                             int* __restrict__ tri_ent, int* __restrict__ edge_ent, int* __restrict__ pt_ent) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  int p = upper_bound_i32(off, (int)nobj + 1, (int)e) - 1;
  int cell = ecell[e];
  if (p < F) tri_ent[tri_start[cell] + atomicAdd(&tri_cur[cell], 1)] = p;
  else if (p < P) edge_ent[edge_start[cell] + atomicAdd(&edge_cur[cell], 1)] = p - (int)F;
  else pt_ent[pt_start[cell] + atomicAdd(&pt_cur[cell], 1)] = p - (int)P;
}

// work lists: cells holding points and triangles; cells holding >= 2 edges
__global__ void k_cell_lists(int ncell, const int* __restrict__ pt_start, const int* __restrict__ tri_start,
                             const int* __restrict__ edge_start, int* __restrict__ cells_pt,
                             int* __restrict__ cells_ee, int* __restrict__ ncount) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  bool a = false, b = false;
  if (c < ncell) {
    a = (pt_start[c + 1] > pt_start[c]) && (tri_start[c + 1] > tri_start[c]);
    b = (edge_start[c + 1] - edge_start[c]) >= 2;
  }
  const int lane = threadIdx.x & 31;
  unsigned ma = __ballot_sync(0xffffffffu, a), mb = __ballot_sync(0xffffffffu, b);
  int ba = 0, bb = 0;
  if (lane == 0) {
    if (ma) ba = atomicAdd(&ncount[0], __popc(ma));
    if (mb) bb = atomicAdd(&ncount[1], __popc(mb));
  }
  ba = __shfl_sync(0xffffffffu, ba, 0);
  bb = __shfl_sync(0xffffffffu, bb, 0);
  unsigned below = (1u << lane) - 1u;
  if (a) cells_pt[ba + __popc(ma & below)] = c;
  if (b) cells_ee[bb + __popc(mb & below)] = c;
}

struct BpOut {
  // raw tap mode
  int* a;
  int* b;
  // contact mode: scratch pair table
  unsigned long long* khi;
  unsigned long long* klo;
  int4* verts;
  double* d;
  double* k;
  double* nrm;
  double* grad;
  int* is_pt;
  // ccd / certificate modes (verts == nullptr: no pair list is stored)
  double* alpha_pair;
  double* alpha_d;
  double* min_alpha;  // global min over pairs (atomic)
  int* ccd_ispt;
  // common
  int* counter;    // [0] = reported pairs, [1] = flag (penetration / failed certificate)
  int64_t cap;
};

struct KeyCtx {
  const int* new2old;
  int bits;
};

__device__ __forceinline__ void make_key(const KeyCtx& K, int type, int i0, int i1, int i2, int i3,
                                         unsigned long long* hi, unsigned long long* lo) {
  unsigned long long b = (unsigned long long)K.bits;
  *hi = ((unsigned long long)type << (2 * b)) | ((unsigned long long)K.new2old[i0] << b) |
        (unsigned long long)K.new2old[i1];
  *lo = ((unsigned long long)K.new2old[i2] << b) | (unsigned long long)K.new2old[i3];
}

struct ContactParams {
  double d_hat, kappa;
  const unsigned char* pinned;
  KeyCtx key;
};

// write one active constraint (contact.py:139-165) into slot of the scratch table
__device__ void write_contact(const BpOut& O, const ContactParams& CP, int slot, int type, const int vid[4], double d,
                              double gr[12]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
    if (CP.pinned[vid[a]]) {
      gr[3 * a] = 0.0; gr[3 * a + 1] = 0.0; gr[3 * a + 2] = 0.0;
    }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 12; ++q) s += gr[q] * gr[q];
  double ddb;
  barrier3(d, CP.d_hat, CP.kappa, nullptr, nullptr, &ddb);
  unsigned long long hi, lo;
  make_key(CP.key, type, vid[0], vid[1], vid[2], vid[3], &hi, &lo);
  O.khi[slot] = hi;
  O.klo[slot] = lo;
  O.verts[slot] = make_int4(vid[0], vid[1], vid[2], vid[3]);
  O.d[slot] = d;
  O.k[slot] = ddb;
  O.nrm[slot] = sqrt(s);
  O.is_pt[slot] = type;
#pragma unroll
  for (int q = 0; q < 12; ++q) O.grad[12 * (int64_t)slot + q] = gr[q];
}

struct CcdParams {
  const double* p;
  double alpha_l;
  int bs;
};

__device__ double ccd_pair_alpha(const double* x, const double* p, const int vid[4], bool is_pt, double alpha_l,
                                 bool* cert_p);
__device__ bool ccd_certify_pair(const double* x, const double* p, const double* alpha_d, int bs, const int vid[4],
                                 bool is_pt);



// ---------------------------------------------------------------------------
// cell-centric queries: one warp per work cell, lanes stride over the cell's
// candidate pairs, warp-aggregated output slots.

// the reference hash grid's reachability (geometry.py:417-440, 465-475):
// query box [q_lo - pad, q_hi + pad] and inserted box [b_lo - pad, b_hi + pad]
// share a reference cell on every axis
struct RefGrid {
  double cell, pad;
};

__device__ __forceinline__ bool ref_reach(const RefGrid& R, const double* qlo, const double* qhi, const double* blo,
                                          const double* bhi) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double q0 = floor(RDIV(RSUB(qlo[k], R.pad), R.cell)), q1 = floor(RDIV(RADD(qhi[k], R.pad), R.cell));
    double i0 = floor(RDIV(RSUB(blo[k], R.pad), R.cell)), i1 = floor(RDIV(RADD(bhi[k], R.pad), R.cell));
    if (!(q0 <= i1 && i0 <= q1)) return false;
  }
  return true;
}

__device__ __forceinline__ int warp_slot(bool emit, int* counter) {
  const int lane = threadIdx.x & 31;
  unsigned m = __ballot_sync(0xffffffffu, emit);
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + __popc(m & ((1u << lane) - 1u));
}

struct BpTables {
  CellGrid G;
  RefGrid R;
  const int *pt_start, *pt_ent, *tri_start, *tri_ent, *edge_start, *edge_ent;
  const int *cells_pt, *cells_ee, *ncount;
  const double *flo, *fhi, *rlo, *rhi;  // (F+E)*3 reference filter / raw boxes
  const double *elo, *ehi;              // (F+E+V)*3 enumeration boxes
};

__device__ __forceinline__ bool boxes_meet(const double* al, const double* ah, const double* bl, const double* bh) {
  return al[0] <= bh[0] && bl[0] <= ah[0] && al[1] <= bh[1] && bl[1] <= ah[1] && al[2] <= bh[2] && bl[2] <= ah[2];
}

// the pair is reported in exactly one cell: the one holding the low corner
// of the intersection of the two enumeration boxes
__device__ __forceinline__ bool owns_corner(const CellGrid& G, int cell, const double* al, const double* bl) {
  const int cz = cell % G.n[2], cy = (cell / G.n[2]) % G.n[1], cx = cell / (G.n[2] * G.n[1]);
  return cg_coord(fmax(al[0], bl[0]), G.o[0], G.h, G.n[0]) == cx &&
         cg_coord(fmax(al[1], bl[1]), G.o[1], G.h, G.n[1]) == cy &&
         cg_coord(fmax(al[2], bl[2]), G.o[2], G.h, G.n[2]) == cz;
}

// per-pair work of the non-raw modes
template <int MODE>
__device__ __forceinline__ void pair_work(const BpOut& O, const ContactParams& CP, const CcdParams& CC,
                                          const double* x, bool pass, int type, int vid[4], int vid_ccd[4]) {
  if (MODE == BP_CONTACT) {
    double d = 0.0, gr[12];
    if (pass) {
      double X[4][3];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) X[a][k] = x[3 * vid[a] + k];
      d = type ? pt_distance(X[0], X[1], X[2], X[3], gr) : ee_distance(X[0], X[1], X[2], X[3], gr);
      if (d <= 0.0) O.counter[1] = 1;
    }
    const bool emit = pass && d > 0.0 && d < CP.d_hat;
    int slot = warp_slot(emit, O.counter);
    if (emit && slot < O.cap) write_contact(O, CP, slot, type, vid, d, gr);
  } else if (MODE == BP_CCD) {
    int slot = warp_slot(pass, O.counter);
    if (pass) {
      bool cert_p = true;
      double al = ccd_pair_alpha(x, CC.p, vid_ccd, type != 0, CC.alpha_l, &cert_p);
      if (al < 1.0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) atomic_min_nonneg(&O.alpha_d[vid_ccd[r] / CC.bs], al);
        atomic_min_nonneg(O.min_alpha, al);
      }
      if (!cert_p) O.counter[1] = 1;  // certificate under the unscaled p fails
      if (O.verts && slot < O.cap) {
        O.verts[slot] = make_int4(vid_ccd[0], vid_ccd[1], vid_ccd[2], vid_ccd[3]);
        O.ccd_ispt[slot] = type;
        O.alpha_pair[slot] = al;
      }
    }
  } else if (MODE == BP_CERT) {
    warp_slot(pass, O.counter);
    if (pass && !ccd_certify_pair(x, CC.p, O.alpha_d, CC.bs, vid_ccd, type != 0)) O.counter[1] = 1;
  }
}

// PT pairs (geometry.py:478-487)
template <int MODE>
__global__ void __launch_bounds__(256) k_bp_pt(BpTables T, const int* __restrict__ sverts, const int* __restrict__ tri,
                                               const int* __restrict__ tri_sorted, const double* __restrict__ x,
                                               int64_t PE, BpOut O, ContactParams CP, CcdParams CC) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ncells = T.ncount[0];
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ncells; w += nw) {
    const int cell = T.cells_pt[w];
    const int ps = T.pt_start[cell], np = T.pt_start[cell + 1] - ps;
    const int ts = T.tri_start[cell], nt = T.tri_start[cell + 1] - ts;
    const int64_t npairs = (int64_t)np * nt;
    for (int64_t b0 = 0; b0 < npairs; b0 += 32) {
      const int64_t q = b0 + lane;
      bool pass = false;
      int v = 0, t = 0, a = 0, b = 0, c = 0;
      if (q < npairs) {
        const int qi = T.pt_ent[ps + (int)(q / nt)];
        v = sverts[qi];
        t = T.tri_ent[ts + (int)(q % nt)];
        a = tri[3 * t]; b = tri[3 * t + 1]; c = tri[3 * t + 2];
        const double* pl = T.elo + 3 * (PE + qi);
        const double* ph = T.ehi + 3 * (PE + qi);
        const double* tl = T.elo + 3 * (int64_t)t;
        const double* th = T.ehi + 3 * (int64_t)t;
        pass = a != v && b != v && c != v && boxes_meet(pl, ph, tl, th) && owns_corner(T.G, cell, pl, tl);
        if (pass) {
          const double pv[3] = {x[3 * v], x[3 * v + 1], x[3 * v + 2]};
          const double* l = T.flo + 3 * (int64_t)t;
          const double* h = T.fhi + 3 * (int64_t)t;
          pass = pv[0] >= l[0] && pv[1] >= l[1] && pv[2] >= l[2] && pv[0] <= h[0] && pv[1] <= h[1] && pv[2] <= h[2];
          pass = pass && ref_reach(T.R, pv, pv, T.rlo + 3 * (int64_t)t, T.rhi + 3 * (int64_t)t);
        }
      }
      if (MODE == BP_RAW) {
        int slot = warp_slot(pass, O.counter);
        if (pass && slot < O.cap) {
          O.a[slot] = v;
          O.b[slot] = t;
        }
      } else {
        // constraint set: triangle sorted by original id (contact.py:133-135);
        // CCD: surface order (ccd.py:229-231)
        int vid[4] = {v, 0, 0, 0}, vid_ccd[4] = {v, a, b, c};
        if (MODE == BP_CONTACT && q < npairs) {
          vid[1] = tri_sorted[3 * t]; vid[2] = tri_sorted[3 * t + 1]; vid[3] = tri_sorted[3 * t + 2];
        }
        pair_work<MODE>(O, CP, CC, x, pass, 1, vid, vid_ccd);
      }
    }
  }
}

// EE pairs (geometry.py:489-499)
template <int MODE>
__global__ void __launch_bounds__(256) k_bp_ee(BpTables T, const int* __restrict__ edge, const double* __restrict__ x,
                                               int64_t F, BpOut O, ContactParams CP, CcdParams CC) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int ncells = T.ncount[1];
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ncells; w += nw) {
    const int cell = T.cells_ee[w];
    const int es = T.edge_start[cell];
    const int64_t k = T.edge_start[cell + 1] - es;
    const int64_t npairs = k * (k - 1) / 2;
    for (int64_t b0 = 0; b0 < npairs; b0 += 32) {
      const int64_t q = b0 + lane;
      bool pass = false;
      int i = 0, j = 0;
      int vid[4] = {0, 0, 0, 0};
      if (q < npairs) {
        // upper-triangle index -> (r, s), r < s
        int64_t r = k - 2 - (int64_t)floor(sqrt((double)(-8 * q + 4 * k * (k - 1) - 7)) / 2.0 - 0.5);
        int64_t s = q + r + 1 - k * (k - 1) / 2 + (k - r) * ((k - r) - 1) / 2;
        int e1 = T.edge_ent[es + (int)r], e2 = T.edge_ent[es + (int)s];
        i = min(e1, e2);
        j = max(e1, e2);
        vid[0] = edge[2 * i]; vid[1] = edge[2 * i + 1]; vid[2] = edge[2 * j]; vid[3] = edge[2 * j + 1];
        const double* eli = T.elo + 3 * (F + i);
        const double* elj = T.elo + 3 * (F + j);
        pass = !(vid[0] == vid[2] || vid[0] == vid[3] || vid[1] == vid[2] || vid[1] == vid[3]) &&
               boxes_meet(eli, T.ehi + 3 * (F + i), elj, T.ehi + 3 * (F + j)) && owns_corner(T.G, cell, eli, elj);
        if (pass) {
          const double* li = T.flo + 3 * (F + i);
          const double* hi_i = T.fhi + 3 * (F + i);
          const double* lj = T.flo + 3 * (F + j);
          const double* hj = T.fhi + 3 * (F + j);
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) pass = pass && (li[kk] <= hj[kk]) && (lj[kk] <= hi_i[kk]);
          pass = pass && ref_reach(T.R, T.rlo + 3 * (F + i), T.rhi + 3 * (F + i), T.rlo + 3 * (F + j),
                                   T.rhi + 3 * (F + j));
        }
      }
      if (MODE == BP_RAW) {
        int slot = warp_slot(pass, O.counter);
        if (pass && slot < O.cap) {
          O.a[slot] = i;
          O.b[slot] = j;
        }
      } else {
        pair_work<MODE>(O, CP, CC, x, pass, 0, vid, vid);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// CUB helpers

static void* cub_temp(mp_ctx* c, size_t bytes) {
  c->cub_tmp.ensure(bytes + 256);
  return c->cub_tmp.p;
}

static void exclusive_scan(mp_ctx* c, const int* in, int* out, int64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, c->stream);
  void* tmp = cub_temp(c, bytes);
  cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, c->stream);
  LAUNCH_CHECK();
}

static void sort_pairs_u64(mp_ctx* c, const unsigned long long* kin, unsigned long long* kout, const int* vin,
                           int* vout, int64_t n, int end_bit) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, c->stream);
  void* tmp = cub_temp(c, bytes);
  cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, c->stream);
  LAUNCH_CHECK();
}

static int bits_for(unsigned long long v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// ---------------------------------------------------------------------------
// broad-phase build (host driver)

struct BpGrid {
  BpTables T{};
  int ncell = 0;
  int64_t F = 0, PE = 0;
  bool empty = true;
};

static void sync_stream(mp_ctx* c) { CUDA_CHECK(cudaStreamSynchronize(c->stream)); }

// Everything one broad-phase call at (x, mb, d_hat) needs: boxes, the dense
// cell tables of triangles / edges / surface points and the work lists.
// infl (per vertex, device) switches to tight enumeration boxes.
static BpGrid build_bp(mp_ctx* c, const double* x, double mb, double d_hat, const double* infl = nullptr) {
  BpGrid B;
  B.F = c->F;
  const int64_t P = c->F + c->E;
  const int64_t V = c->V;
  const int64_t nobj = P + V;
  B.PE = P;
  if (c->F == 0 || P == 0) return B;
  const double gap = d_hat + 2.0 * mb;
  cudaStream_t st = c->stream;
  for (DBuf<double>* b : {&c->box_rlo, &c->box_rhi, &c->box_flo, &c->box_fhi}) b->ensure(3 * P);
  c->box_elo.ensure(3 * nobj);
  c->box_ehi.ensure(3 * nobj);
  CUDA_CHECK(cudaMemsetAsync(c->dscal.p + 40, 0, sizeof(double), st));
  k_prim_boxes<<<grid_for(P, 256), 256, 0, st>>>(c->F, c->E, c->tri, c->edge, x, gap, infl, c->box_rlo, c->box_rhi,
                                                  c->box_flo, c->box_fhi, c->box_elo, c->box_ehi, c->dscal.p + 40);
  LAUNCH_CHECK();
  if (V) {
    k_point_boxes<<<grid_for(V, 256), 256, 0, st>>>(V, c->sverts, x, infl, c->box_elo.p + 3 * P,
                                                     c->box_ehi.p + 3 * P);
    LAUNCH_CHECK();
  }
  const int nb = 64;
  c->red_part.ensure(7 * nb + 1);
  k_box_stats<<<nb, 256, 0, st>>>(P, c->box_elo, c->box_ehi, c->red_part);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(c->red_part.p + 7 * nb, c->dscal.p + 40, sizeof(double), cudaMemcpyDeviceToDevice, st));
  std::vector<double> part(7 * nb + 1);
  CUDA_CHECK(cudaMemcpyAsync(part.data(), c->red_part.p, sizeof(double) * (7 * nb + 1), cudaMemcpyDeviceToHost, st));
  sync_stream(c);
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, ext = 0.0;
  for (int b = 0; b < nb; ++b) {
    for (int k = 0; k < 3; ++k) {
      mn[k] = fmin(mn[k], -part[7 * b + k]);
      mx[k] = fmax(mx[k], part[7 * b + 3 + k]);
    }
    ext += part[7 * b + 6];
  }
  // the reference's cell and pad (geometry.py:465-466)
  B.T.R.cell = fmax(part[7 * nb], d_hat + mb);
  B.T.R.pad = 0.5 * d_hat + mb;
  double span = fmax(fmax(mx[0] - mn[0], mx[1] - mn[1]), mx[2] - mn[2]);
  double h = ext / (double)P;  // mean enumeration-box extent
  if (!(h > 0.0) || !std::isfinite(h)) h = span > 0.0 ? span : 1.0;
  h = fmax(h, span * 1e-6);
  if (!(h > 0.0)) h = 1.0;
  const double max_cells = fmax(1 << 18, fmin(1 << 24, 16.0 * (double)nobj));
  c->cell_cnt.ensure(nobj + 1);
  c->cell_off.ensure(nobj + 1);
  int total = 0, ncell = 0;
  for (int attempt = 0; attempt < 60; ++attempt, h *= 1.5) {
    CellGrid& G = B.T.G;
    G.h = h;
    double cells = 1.0;
    for (int k = 0; k < 3; ++k) {
      G.o[k] = mn[k];
      double nk = floor((mx[k] - mn[k]) / h) + 1.0;
      if (!(nk >= 1.0)) nk = 1.0;
      G.n[k] = (int)fmin(nk, 1 << 20);
      cells *= (double)G.n[k];
    }
    if (cells > max_cells) continue;
    ncell = (int)cells;
    k_cell_span<<<grid_for(nobj, 256), 256, 0, st>>>(nobj, G, c->box_elo, c->box_ehi, c->cell_cnt);
    LAUNCH_CHECK();
    CUDA_CHECK(cudaMemsetAsync(c->cell_cnt.p + nobj, 0, sizeof(int), st));
    exclusive_scan(c, c->cell_cnt, c->cell_off, nobj + 1);
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 4, c->cell_off.p + nobj, sizeof(int), cudaMemcpyDeviceToHost, st));
    sync_stream(c);
    total = c->h_cnt[4];
    if (total >= 0 && (int64_t)total <= 32 * nobj + 4096) break;
  }
  B.ncell = ncell;
  auto& g = c->grid;
  for (DBuf<int>* b : {&g.tri_cnt, &g.tri_start, &g.edge_cnt, &g.edge_start, &g.pt_cnt, &g.pt_start})
    b->ensure((size_t)ncell + 1);
  g.cells_pt.ensure(ncell);
  g.cells_ee.ensure(ncell);
  g.ecell.ensure((size_t)total + 1);
  g.tri_ent.ensure((size_t)total + 1);
  g.edge_ent.ensure((size_t)total + 1);
  g.pt_ent.ensure((size_t)total + 1);
  for (DBuf<int>* b : {&g.tri_cnt, &g.edge_cnt, &g.pt_cnt})
    CUDA_CHECK(cudaMemsetAsync(b->p, 0, sizeof(int) * ((size_t)ncell + 1), st));
  CUDA_CHECK(cudaMemsetAsync(c->counters.p + 8, 0, 2 * sizeof(int), st));
  if (total) {
    k_entry_hist<<<grid_for(total, 256), 256, 0, st>>>(total, nobj, c->F, P, B.T.G, c->cell_off, c->box_elo,
                                                       c->box_ehi, g.ecell, g.tri_cnt, g.edge_cnt, g.pt_cnt);
    LAUNCH_CHECK();
  }
  exclusive_scan(c, g.tri_cnt, g.tri_start, ncell + 1);
  exclusive_scan(c, g.edge_cnt, g.edge_start, ncell + 1);
  exclusive_scan(c, g.pt_cnt, g.pt_start, ncell + 1);
  // the counts become per-cell fill cursors
  for (DBuf<int>* b : {&g.tri_cnt, &g.edge_cnt, &g.pt_cnt})
    CUDA_CHECK(cudaMemsetAsync(b->p, 0, sizeof(int) * ((size_t)ncell + 1), st));
  if (total) {
    k_entry_fill<<<grid_for(total, 256), 256, 0, st>>>(total, nobj, c->F, P, c->cell_off, g.ecell, g.tri_start,
                                                       g.edge_start, g.pt_start, g.tri_cnt, g.edge_cnt, g.pt_cnt,
                                                       g.tri_ent, g.edge_ent, g.pt_ent);
    LAUNCH_CHECK();
  }
  k_cell_lists<<<grid_for(ncell, 256), 256, 0, st>>>(ncell, g.pt_start, g.tri_start, g.edge_start, g.cells_pt,
                                                      g.cells_ee, c->counters.p + 8);
  LAUNCH_CHECK();
  BpTables& T = B.T;
  T.pt_start = g.pt_start; T.pt_ent = g.pt_ent;
  T.tri_start = g.tri_start; T.tri_ent = g.tri_ent;
  T.edge_start = g.edge_start; T.edge_ent = g.edge_ent;
  T.cells_pt = g.cells_pt; T.cells_ee = g.cells_ee; T.ncount = c->counters.p + 8;
  T.flo = c->box_flo; T.fhi = c->box_fhi; T.rlo = c->box_rlo; T.rhi = c->box_rhi;
  T.elo = c->box_elo; T.ehi = c->box_ehi;
  B.empty = false;
  return B;
}

static unsigned bp_blocks(mp_ctx* c) {
  static int sms = 0;
  if (!sms) CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  return (unsigned)(sms * 8);  // 8 x 256-thread CTAs per SM, persistent warps
}

// Run the PT (which & 1) and EE (which & 2) queries in MODE.  Returns the
// number of reported pairs (may exceed O.cap: the caller grows and retries);
// *flag = counters[1] (penetration / failed certificate).
template <int MODE>
static int64_t run_bp(mp_ctx* c, const double* x, const BpGrid& B, BpOut O, ContactParams CP, CcdParams CC,
                      int* flag, int which = 3) {
  CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 2 * sizeof(int), c->stream));
  O.counter = c->counters.p;
  if (!B.empty) {
    if ((which & 1) && c->V) {
      k_bp_pt<MODE><<<bp_blocks(c), 256, 0, c->stream>>>(B.T, c->sverts, c->tri, c->tri_sorted, x, B.PE, O, CP,
                                                          CC);
      LAUNCH_CHECK();
    }
    if ((which & 2) && c->E > 1) {
      k_bp_ee<MODE><<<bp_blocks(c), 256, 0, c->stream>>>(B.T, c->edge, x, B.F, O, CP, CC);
      LAUNCH_CHECK();
    }
  }
  CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  if (flag) *flag = c->h_cnt[1];
  return c->h_cnt[0];
}

// ---------------------------------------------------------------------------
// constraint set: broad phase (mb = 0) + distances + compaction + key sort

__global__ void k_iota(int* a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int)i;
}

__global__ void k_gather_u64(const unsigned long long* src, const int* idx, unsigned long long* dst, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_gather_pairs(int64_t n, const int* __restrict__ idx, const unsigned long long* khi,
                               const unsigned long long* klo, const int4* verts, const double* d, const double* k,
                               const double* nrm, const double* grad, const int* is_pt, unsigned long long* okhi,
                               unsigned long long* oklo, int4* overts, double* od, double* ok, double* onrm,
                               double* ograd, int* ois_pt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = idx[i];
  okhi[i] = khi[s];
  oklo[i] = klo[s];
  overts[i] = verts[s];
  od[i] = d[s];
  ok[i] = k[s];
  onrm[i] = nrm[s];
  ois_pt[i] = is_pt[s];
#pragma unroll
  for (int q = 0; q < 12; ++q) ograd[12 * i + q] = grad[12 * (int64_t)s + q];
}

static void sort_table_into(mp_ctx* c, PairTable& src, PairTable& dst, int64_t n) {
  dst.ensure(n);
  dst.count = n;
  if (n == 0) return;
  c->sort_idx.ensure(n);
  c->sort_idx2.ensure(n);
  c->sort_k1.ensure(n);
  c->sort_k2.ensure(n);
  k_iota<<<grid_for(n, 256), 256, 0, c->stream>>>(c->sort_idx, n);
  LAUNCH_CHECK();
  const int b = c->id_bits;
  sort_pairs_u64(c, src.klo, c->sort_k1, c->sort_idx, c->sort_idx2, n, 2 * b);
  k_gather_u64<<<grid_for(n, 256), 256, 0, c->stream>>>(src.khi, c->sort_idx2, c->sort_k2, n);
  LAUNCH_CHECK();
  sort_pairs_u64(c, c->sort_k2, c->sort_k1, c->sort_idx2, c->sort_idx, n, 2 * b + 1);
  k_gather_pairs<<<grid_for(n, 128), 128, 0, c->stream>>>(n, c->sort_idx, src.khi, src.klo, src.verts, src.d, src.k,
                                                          src.nrm, src.grad, src.is_pt, dst.khi, dst.klo, dst.verts,
                                                          dst.d, dst.k, dst.nrm, dst.grad, dst.is_pt);
  LAUNCH_CHECK();
}

static BpOut table_out(PairTable& t) {
  BpOut O{};
  O.khi = t.khi; O.klo = t.klo; O.verts = t.verts; O.d = t.d; O.k = t.k; O.nrm = t.nrm; O.grad = t.grad;
  O.is_pt = t.is_pt;
  O.cap = (int64_t)t.d.n;
  return O;
}

// compute_constraint_set at x (device, new order) into c->cur (key order)
static void constraint_set(mp_ctx* c, const double* x) {
  c->cur.count = 0;
  if (c->F == 0) return;
  BpGrid B = build_bp(c, x, 0.0, c->d_hat);
  ContactParams CP{c->d_hat, c->kappa, c->pinned, KeyCtx{c->new2old, c->id_bits}};
  CcdParams CC{};
  if (c->scratch.d.n < 1024) c->scratch.ensure(1024);
  for (int attempt = 0; attempt < 4; ++attempt) {
    BpOut O = table_out(c->scratch);
    int pen = 0;
    int64_t n = run_bp<BP_CONTACT>(c, x, B, O, CP, CC, &pen);
    if (pen) throw MpError(MP_ERR_PENETRATION, "contact distance <= 0");
    if (n <= O.cap) {
      sort_table_into(c, c->scratch, c->cur, n);
      return;
    }
    c->scratch.ensure((size_t)(n * 1.5) + 1024);
  }
  throw MpError(MP_ERR_CAPACITY, "constraint set capacity retry failed");
}

// ---------------------------------------------------------------------------
// contact terms of gradient / energy / HVP

__global__ void k_contact_grad(int64_t n, const int4* __restrict__ verts, const double* __restrict__ d,
                               const double* __restrict__ grad, const unsigned char* __restrict__ pinned,
                               double dh, double kappa, double* __restrict__ g) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double db;
  barrier3(d[i], dh, kappa, nullptr, &db, nullptr);
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    if (pinned[id[a]]) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) atomicAdd(&g[3 * id[a] + k], db * grad[12 * i + 3 * a + k]);
  }
}

__global__ void k_contact_energy(int64_t n, const double* __restrict__ d, double dh, double kappa, double* part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double b;
    barrier3(d[i], dh, kappa, &b, nullptr, nullptr);
    acc += b;
  }
  block_sum_store<256>(acc, part);
}

// out += sum_i s_i w_i (w_i . vec) over rank-one terms; s == nullptr -> 1
__global__ void k_rank1_apply(int64_t n, const int4* __restrict__ verts, const double* __restrict__ w,
                              const double* __restrict__ s, const double* __restrict__ vec, double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  double dot = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) dot += w[12 * i + 3 * a + k] * vec[3 * id[a] + k];
  if (s) dot *= s[i];
  if (dot == 0.0) return;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double val = w[12 * i + 3 * a + k];
      if (val != 0.0) atomicAdd(&out[3 * id[a] + k], val * dot);
    }
}

// ---------------------------------------------------------------------------
// classification against the base snapshot (contact.py:182-214)

__device__ __forceinline__ int find_key(const unsigned long long* khi, const unsigned long long* klo, int n,
                                        unsigned long long hi, unsigned long long lo) {
  int a = 0, b = n;
  while (a < b) {
    int mid = (a + b) >> 1;
    bool less = (khi[mid] < hi) || (khi[mid] == hi && klo[mid] < lo);
    if (less) a = mid + 1; else b = mid;
  }
  if (a < n && khi[a] == hi && klo[a] == lo) return a;
  return -1;
}

__global__ void k_classify(int64_t n, const unsigned long long* __restrict__ khi, const unsigned long long* __restrict__ klo,
                           const double* __restrict__ grad, const double* __restrict__ nrm, const double* __restrict__ k,
                           int nb, const unsigned long long* __restrict__ bkhi, const unsigned long long* __restrict__ bklo,
                           const double* __restrict__ bgrad, const double* __restrict__ bnrm,
                           const double* __restrict__ bk, double eps_rot, int* __restrict__ flag,
                           double* __restrict__ scale, double* __restrict__ ds) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double nr = nrm[i];
  if (nr <= 1e-12) {
    flag[i] = 0;
    return;
  }
  int j = find_key(bkhi, bklo, nb, khi[i], klo[i]);
  if (j >= 0) {
    double bn = bnrm[j];
    double cosv = 0.0;
    if (bn > 1e-12) {
      for (int q = 0; q < 12; ++q) cosv += (grad[12 * i + q] / nr) * (bgrad[12 * (int64_t)j + q] / bn);
    }
    if (cosv >= eps_rot) {
      double delta = k[i] - bk[j];
      if (delta <= 0.0) {
        flag[i] = 0;
        return;
      }
      flag[i] = 1;
      scale[i] = sqrt(delta);
      ds[i] = delta;
      return;
    }
  }
  flag[i] = 1;
  scale[i] = sqrt(k[i]);
  ds[i] = k[i];
}

__global__ void k_compact_cands(int64_t n, const int* __restrict__ flag, const int* __restrict__ pos,
                                const double* __restrict__ scale, const double* __restrict__ ds_in,
                                const int4* __restrict__ verts, const double* __restrict__ grad,
                                int4* __restrict__ cverts, double* __restrict__ cu, double* __restrict__ cds) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  int o = pos[i];
  cverts[o] = verts[i];
  cds[o] = ds_in[i];
  double s = scale[i];
#pragma unroll
  for (int q = 0; q < 12; ++q) cu[12 * (int64_t)o + q] = s * grad[12 * i + q];
}

static void classify_all(mp_ctx* c, double eps_rot) {
  const int64_t n = c->cur.count;
  c->n_cand = 0;
  if (n == 0) return;
  c->cand_flag.ensure(n + 1);
  c->cand_pos.ensure(n + 1);
  c->tmp_scale.ensure(n);
  c->tmp_ds.ensure(n);
  k_classify<<<grid_for(n, 128), 128, 0, c->stream>>>(n, c->cur.khi, c->cur.klo, c->cur.grad, c->cur.nrm, c->cur.k,
                                                      (int)c->base.count, c->base.khi, c->base.klo, c->base.grad,
                                                      c->base.nrm, c->base.k, eps_rot, c->cand_flag, c->tmp_scale,
                                                      c->tmp_ds);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemsetAsync(c->cand_flag.p + n, 0, sizeof(int), c->stream));
  exclusive_scan(c, c->cand_flag, c->cand_pos, n + 1);
  int tot = 0;
  CUDA_CHECK(cudaMemcpyAsync(&tot, c->cand_pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  c->n_cand = tot;
  if (!tot) return;
  c->cand_verts.ensure(tot);
  c->cand_u.ensure(12 * (size_t)tot);
  c->cand_ds.ensure(tot);
  k_compact_cands<<<grid_for(n, 128), 128, 0, c->stream>>>(n, c->cand_flag, c->cand_pos, c->tmp_scale, c->tmp_ds,
                                                           c->cur.verts, c->cur.grad, c->cand_verts, c->cand_u,
                                                           c->cand_ds);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// select_top_k (contact.py:217-233): entries (subdomain, candidate) for every
// distinct subdomain owning a vertex whose u-row is non-zero; per subdomain
// order by (-delta_s, key) and keep K.

__global__ void k_topk_count(int64_t n, const int4* __restrict__ verts, const double* __restrict__ u, int bs,
                             int* __restrict__ cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  int subs[4];
  int m = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* r = u + 12 * i + 3 * a;
    if (r[0] == 0.0 && r[1] == 0.0 && r[2] == 0.0) continue;
    int s = id[a] / bs;
    bool dup = false;
    for (int q = 0; q < m; ++q) dup = dup || subs[q] == s;
    if (!dup) subs[m++] = s;
  }
  cnt[i] = m;
}

__global__ void k_topk_fill(int64_t n, const int4* __restrict__ verts, const double* __restrict__ u,
                            const double* __restrict__ ds, int bs, const int* __restrict__ off,
                            int* __restrict__ esub, int* __restrict__ ecand, unsigned long long* __restrict__ ekey) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 v = verts[i];
  const int id[4] = {v.x, v.y, v.z, v.w};
  int subs[4];
  int m = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* r = u + 12 * i + 3 * a;
    if (r[0] == 0.0 && r[1] == 0.0 && r[2] == 0.0) continue;
    int s = id[a] / bs;
    bool dup = false;
    for (int q = 0; q < m; ++q) dup = dup || subs[q] == s;
    if (!dup) subs[m++] = s;
  }
  // descending delta_s: complement of the (positive) double's bit pattern
  unsigned long long key = ~(unsigned long long)__double_as_longlong(ds[i]);
  int o = off[i];
  for (int q = 0; q < m; ++q) {
    esub[o + q] = subs[q];
    ecand[o + q] = (int)i;
    ekey[o + q] = key;
  }
}

// run starts of the (subdomain-sorted) entry list -> touched subdomains
__global__ void k_topk_runs(int64_t ne, const int* __restrict__ esub, int* __restrict__ is_start) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ne) return;
  is_start[i] = (i == 0 || esub[i] != esub[i - 1]) ? 1 : 0;
}

__global__ void k_topk_touched(int64_t ne, const int* __restrict__ esub, const int* __restrict__ is_start,
                               const int* __restrict__ run_id, int K, int* __restrict__ tsub,
                               int* __restrict__ tstart, int* __restrict__ tlen, int* __restrict__ overlay_of) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ne || !is_start[i]) return;
  int r = run_id[i];
  int64_t j = i + 1;
  while (j < ne && !is_start[j]) ++j;
  int len = (int)(j - i);
  tsub[r] = esub[i];
  tstart[r] = (int)i;
  tlen[r] = len < K ? len : K;
  overlay_of[esub[i]] = r;
}

__global__ void k_gather_sub_key(int64_t n, const int* __restrict__ sub, const int* __restrict__ idx,
                                 unsigned long long* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = (unsigned long long)sub[idx[i]];
}

__global__ void k_gather_entries(int64_t n, const int* __restrict__ idx, const int* __restrict__ sub,
                                 const int* __restrict__ cand, int* __restrict__ osub, int* __restrict__ ocand) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  osub[i] = sub[idx[i]];
  ocand[i] = cand[idx[i]];
}
