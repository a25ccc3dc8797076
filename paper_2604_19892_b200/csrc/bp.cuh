// bp.cuh -- broad phase (geometry.py:443-503) on a hierarchical grid, fused
// with the per-pair work of its three callers (constraint set, CCD steps,
// certificate).
//
// Membership is the reference's, applied exactly to every enumerated pair:
//   PT (v, t):  v not in t and lo_t - gap <= x_v <= hi_t + gap (componentwise)
//   EE (i, j):  i < j, no shared vertex, lo_i <= hi_j + gap, lo_j <= hi_i + gap
// with gap = d_hat + 2 mb, AND the reference hash grid must reach the pair
// (cell = max(largest primitive diagonal, d_hat + mb), boxes padded by
// d_hat / 2 + mb; geometry.py:417-440, 462-475).  The enumeration itself uses
// our own grid (below) over boxes that provably contain every such pair.
#pragma once

#include <chrono>
#include <cub/cub.cuh>

#include "ctx.cuh"
#include "geom.cuh"

enum { BP_RAW = 0, BP_CONTACT = 1, BP_CCD = 2, BP_CERT = 3 };

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
  int* counter;    // [0] = reported pairs, [1] = flag (penetration / failed certificate), [2] = stored
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

static void sort_pairs_i32(mp_ctx* c, const int* kin, int* kout, const int* vin, int* vout, int64_t n,
                           int end_bit) {
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



// Boxes of triangles and edges: raw (rlo, rhi); reference filter (flo, fhi:
// triangle [lo - gap, hi + gap], edge [lo, hi + gap]); enumeration (elo,
// ehi).  A tight inflation (per vertex, ccd.cuh) is capped at gap: every
// enumerated pair must also pass the reference filter (axis separation <=
// gap), and two boxes grown by min(i_a, gap), min(i_b, gap) still meet
// whenever the separation is <= min(i_a + i_b, gap) -- so the enumeration is
// never looser than the reference's own filter, whatever the motion field
// (the cap carries a 1e-9 relative margin over the rounded filter).  The
// largest raw-box diagonal (the reference's grid cell candidate,
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
      if (infl) inf = fmin(fmax(fmax(infl[a], infl[b]), infl[c]), gap * (1.0 + 1e-9));
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double xa = x[3 * a + k], xb = x[3 * b + k], xc = x[3 * c + k];
        l[k] = fmin(fmin(xa, xb), xc);
        h[k] = fmax(fmax(xa, xb), xc);
      }
    } else {
      int64_t e = i - F;
      int a = edge[2 * e], b = edge[2 * e + 1];
      if (infl) inf = fmin(fmax(infl[a], infl[b]), gap * (1.0 + 1e-9));
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
__global__ void k_point_boxes(int64_t V, const int* __restrict__ sverts, const double* __restrict__ x, double gap,
                              const double* __restrict__ infl, double* __restrict__ elo, double* __restrict__ ehi) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= V) return;
  int v = sverts[q];
  double e = infl ? fmin(infl[v], gap * (1.0 + 1e-9)) : 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    elo[3 * q + k] = x[3 * v + k] - e;
    ehi[3 * q + k] = x[3 * v + k] + e;
  }
}

// stats for the grid: [0..2] min lo, [3..5] max hi, [6] sum of max extents
// of the enumeration boxes, [7] the same of the raw boxes
#define BOX_STATS 8
__global__ void k_box_stats(int64_t P, const double* __restrict__ lo, const double* __restrict__ hi,
                            const double* __restrict__ rlo, const double* __restrict__ rhi,
                            double* __restrict__ part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, ext = 0.0, rext = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    double e = 0.0, r = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double l = lo[3 * i + k], h = hi[3 * i + k];
      mn[k] = fmin(mn[k], l);
      mx[k] = fmax(mx[k], h);
      e = fmax(e, h - l);
      r = fmax(r, rhi[3 * i + k] - rlo[3 * i + k]);
    }
    ext += e;
    rext += r;
  }
  __shared__ double sh[BOX_STATS][8];
  double vals[BOX_STATS] = {-mn[0], -mn[1], -mn[2], mx[0], mx[1], mx[2], ext, rext};
#pragma unroll
  for (int q = 0; q < BOX_STATS; ++q) {
    double v = vals[q];
    v = (q < 6) ? warp_max(v) : warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < BOX_STATS; ++q) {
      double v = sh[q][0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = (q < 6) ? fmax(v, sh[q][w]) : v + sh[q][w];
      part[BOX_STATS * blockIdx.x + q] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// hierarchical uniform grid
//
// Level l has cell size h_l = h0 * 2^l (exact scaling) over the scene box.
// Every object lives at the lowest level whose cell is at least as large as
// its enumeration box, stored ONCE, in the cell holding its box's low corner.
// A pair is found by the object of LOWER level querying the partner's level
// (or, at equal levels, by the lower index for EE): the query walks levels
// >= its own and visits the cells that can hold the low corner of a level-l
// box meeting it ([lo - h_l, hi] per axis), so every candidate is met exactly
// once -- no duplicate encounters to filter.  Small objects find large ones
// (the floor slab, boxes of fast CCD vertices) without the large ones
// enumerating anything.

#define HG_MAX_LEVELS 24

struct HGrid {
  double o[3];
  double h0, inv_h0;
  int nlev;
  int n[HG_MAX_LEVELS][3];
  int off[HG_MAX_LEVELS + 1];  // first global cell id of each level
};

__device__ __forceinline__ double hg_h(const HGrid& G, int l) { return ldexp(G.h0, l); }

// cell coordinate at level l: floor((v - o) / h_l), evaluated as a product
// with the exact power-of-two scaled reciprocal; the same monotone function
// is used for every object, query and corner, which is all consistency needs
__device__ __forceinline__ int hg_coord(const HGrid& G, int l, int k, double v) {
  double q = floor((v - G.o[k]) * ldexp(G.inv_h0, -l));
  if (!(q >= 0.0)) return 0;  // also catches NaN
  if (q > (double)(G.n[l][k] - 1)) return G.n[l][k] - 1;
  return (int)q;
}

__device__ __forceinline__ void hg_span(const HGrid& G, int l, const double* lo, const double* hi, int c0[3],
                                        int c1[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c0[k] = hg_coord(G, l, k, lo[k]);
    c1[k] = hg_coord(G, l, k, hi[k]);
  }
}

// cells a query box must visit at level l to meet every level-l object whose
// box it overlaps: objects are stored once, in the cell of their low corner,
// and their extent is <= h_l, so that corner lies in [lo - h_l, hi]
__device__ __forceinline__ void hg_query_span(const HGrid& G, int l, const double* lo, const double* hi, int c0[3],
                                              int c1[3]) {
  const double h = hg_h(G, l) * (1.0 + 1e-6);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c0[k] = hg_coord(G, l, k, lo[k] - h);
    c1[k] = hg_coord(G, l, k, hi[k]);
  }
}

__device__ __forceinline__ int hg_cell(const HGrid& G, int l, int a, int b, int c) {
  return G.off[l] + (a * G.n[l][1] + b) * G.n[l][2] + c;
}

__device__ __forceinline__ bool boxes_meet(const double* al, const double* ah, const double* bl, const double* bh) {
  return al[0] <= bh[0] && bl[0] <= ah[0] && al[1] <= bh[1] && bl[1] <= ah[1] && al[2] <= bh[2] && bl[2] <= ah[2];
}


// the reference hash grid's cell range of every object
// (floor((lo - pad) / cell), floor((hi + pad) / cell); geometry.py:421-423,
// same IEEE expressions): triangles / edges from their raw boxes, points
// from their position.  Two objects are reachable in the reference grid iff
// their ranges overlap on every axis.
__global__ void k_ref_cells(int64_t P, int64_t V, const int* __restrict__ sverts, const double* __restrict__ x,
                            const double* __restrict__ rlo, const double* __restrict__ rhi, double pad, double cell,
                            int* __restrict__ rc) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= P + V) return;
  double lo[3], hi[3];
  if (i < P) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      lo[k] = rlo[3 * i + k];
      hi[k] = rhi[3 * i + k];
    }
  } else {
    const int v = sverts[i - P];
#pragma unroll
    for (int k = 0; k < 3; ++k) lo[k] = hi[k] = x[3 * v + k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double a = floor(RDIV(RSUB(lo[k], pad), cell)), b = floor(RDIV(RADD(hi[k], pad), cell));
    rc[6 * i + k] = (int)fmax(fmin(a, 1e9), -1e9);
    rc[6 * i + 3 + k] = (int)fmax(fmin(b, 1e9), -1e9);
  }
}

__device__ __forceinline__ bool ref_reach(const int* __restrict__ rc, int64_t a, int64_t b) {
  const int* A = rc + 6 * a;
  const int* B = rc + 6 * b;
  return A[0] <= B[3] && B[0] <= A[3] && A[1] <= B[4] && B[1] <= A[4] && A[2] <= B[5] && B[2] <= A[5];
}

// level of every object and the number of cells it covers there
__global__ void k_obj_level(int64_t nobj, int64_t F, int64_t P, HGrid G, const double* __restrict__ lo,
                            const double* __restrict__ hi, int* __restrict__ level, int* __restrict__ cnt,
                            unsigned* __restrict__ lmask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nobj) return;
  const double* l0 = lo + 3 * i;
  const double* h0 = hi + 3 * i;
  double ext = fmax(fmax(h0[0] - l0[0], h0[1] - l0[1]), h0[2] - l0[2]);
  int l = 0;
  while (l < G.nlev - 1 && ext > hg_h(G, l)) ++l;
  level[i] = l;
  cnt[i] = 1;  // stored once, in the cell of its low corner
  // which levels hold any triangle / edge / point (queries skip empty ones):
  // OR-reduced per warp, one atomic per warp and class
  const int cls = i < F ? 0 : (i < P ? 1 : 2);
  const unsigned bit = 1u << l;
  const unsigned live = __activemask();
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const unsigned w = __reduce_or_sync(live, cls == q ? bit : 0u);
    if (w && (threadIdx.x & 31) == (__ffs(live) - 1)) atomicOr(lmask + q, w);
  }
}

__device__ __forceinline__ int upper_bound_i32(const int* a, int n, int k) {
  int l = 0, r = n;
  while (l < r) {
    int m = (l + r) >> 1;
    if (a[m] <= k) l = m + 1; else r = m;
  }
  return l;
}

// one thread per (object, covered cell) entry: its global cell id and the
// per-class histograms (0 triangles, 1 edges, 2 points)
__global__ void k_entry_hist(const int* __restrict__ total_dev, int64_t nobj, int64_t F, int64_t P, HGrid G,
                             const int* __restrict__ off,
                             const int* __restrict__ level, const double* __restrict__ lo,
                             const double* __restrict__ hi, int* __restrict__ ecell, int* __restrict__ tri_cnt,
                             int* __restrict__ edge_cnt, int* __restrict__ pt_cnt) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= *total_dev) return;
  int p = upper_bound_i32(off, (int)nobj + 1, (int)e) - 1;
  int r = (int)e - off[p];
  int l = level[p];
  const double* o = lo + 3 * (int64_t)p;
  (void)r;
  int cell = hg_cell(G, l, hg_coord(G, l, 0, o[0]), hg_coord(G, l, 1, o[1]), hg_coord(G, l, 2, o[2]));
  ecell[e] = cell;
  atomicAdd(p < F ? &tri_cnt[cell] : (p < P ? &edge_cnt[cell] : &pt_cnt[cell]), 1);
}

__global__ void k_entry_fill(const int* __restrict__ total_dev, int64_t nobj, int64_t F, int64_t P,
                             const int* __restrict__ off,
                             const int* __restrict__ ecell, const int* __restrict__ tri_start,
                             const int* __restrict__ edge_start, const int* __restrict__ pt_start,
                             int* __restrict__ tri_cur, int* __restrict__ edge_cur, int* __restrict__ pt_cur,
                             int* __restrict__ tri_ent, int* __restrict__ edge_ent, int* __restrict__ pt_ent,
                             const double* __restrict__ elo, const double* __restrict__ ehi,
                             double* __restrict__ tri_box, double* __restrict__ edge_box,
                             double* __restrict__ pt_box) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= *total_dev) return;
  int p = upper_bound_i32(off, (int)nobj + 1, (int)e) - 1;
  int cell = ecell[e];
  int pos;
  double* box;
  if (p < F) {
    pos = tri_start[cell] + atomicAdd(&tri_cur[cell], 1);
    tri_ent[pos] = p;
    box = tri_box;
  } else if (p < P) {
    pos = edge_start[cell] + atomicAdd(&edge_cur[cell], 1);
    edge_ent[pos] = p - (int)F;
    box = edge_box;
  } else {
    pos = pt_start[cell] + atomicAdd(&pt_cur[cell], 1);
    pt_ent[pos] = p - (int)P;
    box = pt_box;
  }
  // the box travels with the entry: the query lanes read it coalesced
  double* b = box + 6 * (int64_t)pos;
  const double* l = elo + 3 * (int64_t)p;
  const double* h = ehi + 3 * (int64_t)p;
  reinterpret_cast<double2*>(b)[0] = make_double2(l[0], l[1]);
  reinterpret_cast<double2*>(b)[1] = make_double2(l[2], h[0]);
  reinterpret_cast<double2*>(b)[2] = make_double2(h[1], h[2]);
}

// ---------------------------------------------------------------------------
// per-pair work of each mode.  pair_work is called by all 32 lanes of a warp
// (ballots / warp minimum inside); live lanes carry one reference pair:
// PT (a = surface vertex device id, b = triangle), EE (a < b edge indices).

__device__ __forceinline__ int warp_slot(bool emit, int* counter) {
  const int lane = threadIdx.x & 31;
  unsigned m = __ballot_sync(0xffffffffu, emit);
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  return base + __popc(m & ((1u << lane) - 1u));
}

struct PairArgs {
  const int* tri;         // surface order (CCD, ccd.py:229-231)
  const int* tri_sorted;  // rows sorted by original id (constraint set, contact.py:133-135)
  const int* edge;
  const double* x;
  BpOut O;
  ContactParams CP;
  CcdParams CC;
  unsigned long long* n_pairs;  // fused enumeration: reference pairs seen
  // append enumeration (HQ_APPEND): this class's list and its counter
  int *app_a, *app_b, *app_cnt;
  int64_t app_cap;
  int app_ee;  // app_cnt is counters[9] (EE) rather than [8] (PT): the overflow flag sits at counters[10]
};

template <int MODE>
__device__ __forceinline__ void pair_work(bool live, bool is_pt, int a, int b, int64_t i, const PairArgs& A) {
  const int lane = threadIdx.x & 31;
  const BpOut& O = A.O;
  const double* x = A.x;
  int vid[4] = {0, 0, 0, 0}, vid_ccd[4] = {0, 0, 0, 0};
  if (live) {
    if (is_pt) {
      vid_ccd[0] = a; vid_ccd[1] = A.tri[3 * b]; vid_ccd[2] = A.tri[3 * b + 1]; vid_ccd[3] = A.tri[3 * b + 2];
      vid[0] = a; vid[1] = A.tri_sorted[3 * b]; vid[2] = A.tri_sorted[3 * b + 1]; vid[3] = A.tri_sorted[3 * b + 2];
    } else {
      vid_ccd[0] = vid[0] = A.edge[2 * a]; vid_ccd[1] = vid[1] = A.edge[2 * a + 1];
      vid_ccd[2] = vid[2] = A.edge[2 * b]; vid_ccd[3] = vid[3] = A.edge[2 * b + 1];
    }
  }
  if (MODE == BP_CONTACT) {
    double d = 0.0, gr[12];
    if (live) {
      double X[4][3];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) X[r][k] = x[3 * vid[r] + k];
      d = is_pt ? pt_distance(X[0], X[1], X[2], X[3], gr) : ee_distance(X[0], X[1], X[2], X[3], gr);
      if (d <= 0.0) O.counter[1] = 1;
    }
    const bool emit = live && d > 0.0 && d < A.CP.d_hat;
    const int slot = warp_slot(emit, O.counter);
    if (emit && slot < O.cap) write_contact(O, A.CP, slot, is_pt ? 1 : 0, vid, d, gr);
  } else if (MODE == BP_CCD) {
    bool cert_p = true;
    const double al = live ? ccd_pair_alpha(x, A.CC.p, vid_ccd, is_pt, A.CC.alpha_l, &cert_p) : 1.0;
    if (live && al < 1.0) {
      // read before the atomic: once a subdomain's minimum has settled most
      // pairs cannot lower it, so contended atomics stay rare
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double* ad = &O.alpha_d[vid_ccd[r] / A.CC.bs];
        if (al < *(volatile double*)ad) atomic_min_nonneg(ad, al);
      }
    }
    // global minimum: warp minimum first, one filtered atomic per warp
    const double wm = warp_min_all(al);
    if (lane == 0 && wm < *(volatile double*)O.min_alpha) atomic_min_nonneg(O.min_alpha, wm);
    if (!cert_p) O.counter[1] = 1;  // certificate under the unscaled p fails
    if (live && O.verts && i >= 0 && i < O.cap) {
      O.verts[i] = make_int4(vid_ccd[0], vid_ccd[1], vid_ccd[2], vid_ccd[3]);
      O.ccd_ispt[i] = is_pt ? 1 : 0;
      O.alpha_pair[i] = al;
    }
  } else if (MODE == BP_CERT) {
    if (live && !ccd_certify_pair(x, A.CC.p, O.alpha_d, A.CC.bs, vid_ccd, is_pt)) O.counter[1] = 1;
  }
}

// the stored list: pairs [0, n_pt) are PT, [n_pt, n) are EE
template <int MODE>
__global__ void __launch_bounds__(256) k_pairs(const int* __restrict__ n_pt_dev, const int* __restrict__ n_dev,
                                               int64_t cap, const int* __restrict__ pa, const int* __restrict__ pb,
                                               PairArgs A) {
  const int64_t n_pt = *n_pt_dev;
  const int64_t n = *n_dev < cap ? *n_dev : cap;  // n > cap: the caller grows and reruns
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (pair_work ballots across the warp)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x - lane); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool live = i < n;
    pair_work<MODE>(live, i < n_pt, live ? pa[i] : 0, live ? pb[i] : 0, i, A);
  }
}

// the appended lists: PT pairs [0, n_pt) in (pa, pb), EE pairs in (ea, eb)
template <int MODE>
__global__ void __launch_bounds__(256) k_pairs_app(const int* __restrict__ cnt, int64_t cap_pt, int64_t cap_ee,
                                                   const int* __restrict__ pa, const int* __restrict__ pb,
                                                   const int* __restrict__ ea, const int* __restrict__ eb,
                                                   PairArgs A) {
  if (cnt[2]) return;  // append counter hit HQ_APPEND_LIMIT: the list is partial, the caller reruns list-free
  const int64_t n_pt = cnt[0] < cap_pt ? cnt[0] : cap_pt;  // overflow: the caller grows and reruns
  const int64_t n_ee = cnt[1] < cap_ee ? cnt[1] : cap_ee;
  const int64_t n = n_pt + n_ee;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x - lane); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool live = i < n, pt = i < n_pt;
    int a = 0, b = 0;
    if (live) {
      if (pt) {
        a = pa[i]; b = pb[i];
      } else {
        a = ea[i - n_pt]; b = eb[i - n_pt];
      }
    }
    pair_work<MODE>(live, pt, a, b, -1, A);
  }
}

// ---------------------------------------------------------------------------
// enumeration: count pass, scan, fill pass -> reference pair list
//   PT pairs (v, t): v = surface vertex (device id), t = triangle index
//   EE pairs (i, j): edge indices, i < j

struct BpTables {
  HGrid G;
  const int *pt_start, *pt_ent, *tri_start, *tri_ent, *edge_start, *edge_ent;
  const double *pt_box, *tri_box, *edge_box;  // per entry (lo, hi)
  const int* level;                     // (F+E+V)
  const unsigned* lmask;                // [3] levels holding triangles / edges / points
  const int* rc;                        // (F+E+V)*6 reference-grid cell ranges
  const double *flo, *fhi;              // (F+E)*3 reference filter / join boxes
  const double *elo, *ehi;              // (F+E+V)*3 enumeration boxes
  int64_t F, P;                         // object id bases: edges at F, points at P
  const int* body = nullptr;            // (N) body of each vertex (connected component)
  int body_mode = 0;                    // 0 all pairs, 1 same-body pairs only, 2 cross-body pairs only
  const double* objmot = nullptr;       // (F+E+V)*4 per-object motion (c, m): exact CCD prefilter, or null
  const double *rlo = nullptr, *rhi = nullptr;  // (F+E)*3 raw primitive boxes
};

// Exact relative-motion prefilter of the tight CCD enumeration.  For any
// constant c the reference's relative displacement bound (ccd.py:172-179)
// is at most 4 max_a |p_a - c| over the pair's vertices; with c = c_1 (c_2)
// that is 4 max(m_1, m_2 + |c_1 - c_2|) (resp. swapped), and the distance
// is at least the gap between the raw boxes.  A pair with 0.9 gap > that
// bound gets alpha_pair = 1 exactly and passes certify_mixed's distance
// test, so dropping it changes no alpha_d, minimum or certificate.  Unlike
// the enumeration boxes (one global c), the bound is relative: a rigidly
// moving or rotating neighbourhood keeps only its truly close pairs.
__device__ __forceinline__ bool rel_safe(const BpTables& T, int64_t o1, int64_t o2, const double* l1,
                                         const double* h1, const double* l2, const double* h2) {
  if (!T.objmot) return false;
  double g2 = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double d = fmax(0.0, fmax(l1[k] - h2[k], l2[k] - h1[k]));
    g2 += d * d;
  }
  const double* a = T.objmot + 4 * o1;
  const double* b = T.objmot + 4 * o2;
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  const double dl = sqrt(dx * dx + dy * dy + dz * dz);
  const double M = fmin(fmax(a[3], b[3] + dl), fmax(b[3], a[3] + dl));
  const double lhs = 0.9 * sqrt(g2) * (1.0 - 1e-12), rhs = 4.0 * M * (1.0 + 1e-12);
  return lhs > rhs;
}

// the body filter of the two-pass tight CCD enumeration (ccd.cuh)
__device__ __forceinline__ bool body_pass(const BpTables& T, int u, int w) {
  return T.body_mode == 0 || ((T.body[u] == T.body[w]) == (T.body_mode == 1));
}

// PT filter (geometry.py:484-486) + reference reachability, point q vs tri t
__device__ __forceinline__ bool pt_ref_pass(const BpTables& T, const int* tri, const double* x, int v, int64_t q,
                                            int t) {
  if (tri[3 * t] == v || tri[3 * t + 1] == v || tri[3 * t + 2] == v) return false;
  if (!body_pass(T, v, tri[3 * t])) return false;
  const double* l = T.flo + 3 * (int64_t)t;
  const double* h = T.fhi + 3 * (int64_t)t;
  const double p0 = x[3 * v], p1 = x[3 * v + 1], p2 = x[3 * v + 2];
  if (!(p0 >= l[0] && p1 >= l[1] && p2 >= l[2] && p0 <= h[0] && p1 <= h[1] && p2 <= h[2])) return false;
  return ref_reach(T.rc, T.P + q, t);
}

// One warp per query object: lanes stride over the entries of each visited
// cell, so a query meeting thousands of candidates (a fast CCD vertex, the
// floor slab) is spread over 32 lanes.  Every lane runs the same loop trip
// counts, so ballots are safe; the fill pass writes a query's pairs in entry
// order at the offsets of the count pass (deterministic list).
#define WARP_FULL 0xffffffffu

// EM: HQ_COUNT / HQ_FILL build the stored list (count pass, scan, fill
// pass); a BP mode fuses the per-pair work into the enumeration instead --
// order-free consumers only (CCD / certificate minima and flags, contacts
// that are key-sorted afterwards): passing pairs queue in shared memory and
// are worked 32 at a time, so no list is written and no count pass runs.
// HQ_APPEND writes an unordered list in one pass: warps queue their passing
// pairs in shared memory and reserve 32 list slots per atomic -- for the
// order-free CCD / certificate consumers, it saves the count pass.
enum { HQ_APPEND = -3, HQ_COUNT = -2, HQ_FILL = -1 };

// The 32-bit append counter must not wrap: past HQ_APPEND_LIMIT reservations
// a warp raises app_cnt[2] and stops writing; the host then reruns the call in
// the list-free fused mode (64-bit pair count).  Every slot below the limit
// was written before any warp reached it, so the list stays memory-safe.
#define HQ_APPEND_LIMIT (1 << 30)
// the limit the kernels apply (MP_OPT_APPEND_LIMIT lowers it so small scenes
// exercise the list-free rerun in tests)
__device__ int g_append_limit = HQ_APPEND_LIMIT;
__device__ __forceinline__ void hq_append_flush(int lane, int k, const int2* q, const PairArgs& A) {
  int base = 0;
  const int lim = g_append_limit;
  if (lane == 0) {
    base = atomicAdd(A.app_cnt, k);
    if (base < 0 || base > lim - k) atomicExch(A.app_cnt + (A.app_ee ? 1 : 2), 1);
  }
  base = __shfl_sync(WARP_FULL, base, 0);
  if (base < 0 || base > lim - k) return;
  if (lane < k && (int64_t)base + lane < A.app_cap) {
    const int2 pr = q[lane];
    A.app_a[base + lane] = pr.x;
    A.app_b[base + lane] = pr.y;
  }
}
#define HQ_QUEUE 64

template <int EM>
__device__ __forceinline__ void hq_emit(bool pass, bool is_pt, int lane, int& n, int o, int a, int b, int* pa, int* pb,
                                        int64_t cap, int2* q, int& qn, const PairArgs& A) {
  const unsigned m = __ballot_sync(WARP_FULL, pass);
  const int rank = __popc(m & ((1u << lane) - 1u));
  if (EM == HQ_FILL) {
    if (pass) {
      const int64_t pos = (int64_t)o + n + rank;
      if (pos < cap) {
        pa[pos] = a;
        pb[pos] = b;
      }
    }
  } else if (EM == HQ_APPEND) {
    if (pass) q[qn + rank] = make_int2(a, b);
    qn += __popc(m);
    if (qn >= 32) {
      __syncwarp();
      qn -= 32;
      hq_append_flush(lane, 32, q + qn, A);
      __syncwarp();
    }
  } else if (EM >= 0) {
    if (pass) q[qn + rank] = make_int2(a, b);
    qn += __popc(m);
    if (qn >= 32) {
      __syncwarp();
      qn -= 32;
      const int2 pr = q[qn + lane];
      __syncwarp();
      pair_work<(EM >= 0 ? EM : 0)>(true, is_pt, pr.x, pr.y, -1, A);
    }
  }
  n += __popc(m);
}

template <int EM>
__device__ __forceinline__ void hq_finish(bool is_pt, int lane, int n, int* cnt, int2* q, int qn, const PairArgs& A) {
  if (EM == HQ_COUNT) {
    if (lane == 0) *cnt = n;
  } else if (EM == HQ_APPEND) {
    __syncwarp();
    if (qn > 0) hq_append_flush(lane, qn, q, A);
  } else if (EM >= 0) {
    __syncwarp();
    if (qn > 0) {
      const int2 pr = q[lane < qn ? lane : 0];
      pair_work<(EM >= 0 ? EM : 0)>(lane < qn, is_pt, pr.x, pr.y, -1, A);
    }
    if (lane == 0 && n) atomicAdd(A.n_pairs, (unsigned long long)n);
  }
}

// A warp walks the entries of up to 32 consecutive cells FLATTENED: lane t
// of round r takes entry r*32 + t of the batch's concatenated ranges (an
// exclusive warp scan of the cell sizes, then a 5-step shuffle search for
// the lane's cell), so a batch of small cells costs one memory round trip
// per 32 entries instead of one per cell.  The order -- cells ascending,
// entries ascending -- is the per-cell walk's, so ordered lists keep their
// order.
struct CellBatch {
  int my0;    // this lane's cell: first entry
  int excl;   // entries of the batch's cells before this lane's
  int total;  // entries in the batch
};

__device__ __forceinline__ CellBatch cell_batch(int my0, int my1) {
  const int lane = threadIdx.x & 31;
  const int cnt = my1 - my0;
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(WARP_FULL, incl, d);
    if (lane >= d) incl += y;
  }
  return CellBatch{my0, incl - cnt, __shfl_sync(WARP_FULL, incl, 31)};
}

// the entry at flattened position f (all 32 lanes call; f < total for a
// valid result)
__device__ __forceinline__ int batch_entry(const CellBatch& b, int f) {
  int c = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int v = __shfl_sync(WARP_FULL, b.excl, c + step);
    if (v <= f) c += step;
  }
  return __shfl_sync(WARP_FULL, b.my0, c) + (f - __shfl_sync(WARP_FULL, b.excl, c));
}

// points query the triangles of every level >= their own
template <int EM>
__global__ void __launch_bounds__(128) k_hq_points(BpTables T, int64_t V, const int* __restrict__ sverts,
                                                   const int* __restrict__ tri, const double* __restrict__ x,
                                                   int* __restrict__ cnt, const int* __restrict__ off,
                                                   int* __restrict__ pa, int* __restrict__ pb, int64_t cap,
                                                   PairArgs A) {
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= V) return;  // warp-uniform
  const int v = sverts[q];
  const double* pl = T.elo + 3 * (T.P + q);
  const double* ph = T.ehi + 3 * (T.P + q);
  int n = 0;
  const int o = EM == HQ_FILL ? off[q] : 0;
  __shared__ int2 qbuf[4][HQ_QUEUE];
  int2* Q = qbuf[threadIdx.x >> 5];
  int qn = 0;
  const unsigned mask = T.lmask[0];
  for (int l = T.level[T.P + q]; l < T.G.nlev; ++l) {
    if (!((mask >> l) & 1u)) continue;
    int c0[3], c1[3];
    hg_query_span(T.G, l, pl, ph, c0, c1);
    // the span's cells in (a, b, c) order, 32 at a time: each lane loads one
    // cell's entry range, the warp walks the batch's entries flattened
    const int nb_ = c1[1] - c0[1] + 1, nc_ = c1[2] - c0[2] + 1;
    const int ncell_ = (c1[0] - c0[0] + 1) * nb_ * nc_;
    for (int cb_ = 0; cb_ < ncell_; cb_ += 32) {
          int my0 = 0, my1 = 0;
          {
            const int idx = cb_ + lane;
            if (idx < ncell_) {
              const int r = idx % (nb_ * nc_);
              const int cell = hg_cell(T.G, l, c0[0] + idx / (nb_ * nc_), c0[1] + r / nc_, c0[2] + r % nc_);
              my0 = T.tri_start[cell];
              my1 = T.tri_start[cell + 1];
            }
          }
          const CellBatch cbt = cell_batch(my0, my1);
          for (int base = 0; base < cbt.total; base += 32) {
            const int f = base + lane;
            const int e = batch_entry(cbt, f < cbt.total ? f : cbt.total - 1);
            bool pass = false;
            int t = 0;
            if (f < cbt.total) {
              t = T.tri_ent[e];
              const double* tl = T.tri_box + 6 * (int64_t)e;
              pass = boxes_meet(pl, ph, tl, tl + 3) &&
                     pt_ref_pass(T, tri, x, v, q, t) &&
                     !rel_safe(T, T.P + q, t, x + 3 * (int64_t)v, x + 3 * (int64_t)v, T.rlo + 3 * (int64_t)t,
                               T.rhi + 3 * (int64_t)t);
            }
            hq_emit<EM>(pass, true, lane, n, o, v, t, pa, pb, cap, Q, qn, A);
          }
        }
  }
  hq_finish<EM>(true, lane, n, cnt ? cnt + q : nullptr, Q, qn, A);
}

// triangles query the points of every level above their own
template <int EM>
__global__ void __launch_bounds__(128) k_hq_tris(BpTables T, int64_t F, const int* __restrict__ sverts,
                                                 const int* __restrict__ tri, const double* __restrict__ x,
                                                 int* __restrict__ cnt, const int* __restrict__ off,
                                                 int* __restrict__ pa, int* __restrict__ pb, int64_t cap,
                                                 PairArgs A) {
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= F) return;
  const double* tl = T.elo + 3 * t;
  const double* th = T.ehi + 3 * t;
  int n = 0;
  const int o = EM == HQ_FILL ? off[t] : 0;
  __shared__ int2 qbuf[4][HQ_QUEUE];
  int2* Q = qbuf[threadIdx.x >> 5];
  int qn = 0;
  const unsigned mask = T.lmask[2];
  for (int l = T.level[t] + 1; l < T.G.nlev; ++l) {
    if (!((mask >> l) & 1u)) continue;
    int c0[3], c1[3];
    hg_query_span(T.G, l, tl, th, c0, c1);
    // the span's cells in (a, b, c) order, 32 at a time: each lane loads one
    // cell's entry range, the warp walks the batch's entries flattened
    const int nb_ = c1[1] - c0[1] + 1, nc_ = c1[2] - c0[2] + 1;
    const int ncell_ = (c1[0] - c0[0] + 1) * nb_ * nc_;
    for (int cb_ = 0; cb_ < ncell_; cb_ += 32) {
          int my0 = 0, my1 = 0;
          {
            const int idx = cb_ + lane;
            if (idx < ncell_) {
              const int r = idx % (nb_ * nc_);
              const int cell = hg_cell(T.G, l, c0[0] + idx / (nb_ * nc_), c0[1] + r / nc_, c0[2] + r % nc_);
              my0 = T.pt_start[cell];
              my1 = T.pt_start[cell + 1];
            }
          }
          const CellBatch cbt = cell_batch(my0, my1);
          for (int base = 0; base < cbt.total; base += 32) {
            const int f = base + lane;
            const int e = batch_entry(cbt, f < cbt.total ? f : cbt.total - 1);
            bool pass = false;
            int v = 0;
            if (f < cbt.total) {
              const int q = T.pt_ent[e];
              const double* pl = T.pt_box + 6 * (int64_t)e;
              v = sverts[q];
              pass = boxes_meet(pl, pl + 3, tl, th) &&
                     pt_ref_pass(T, tri, x, v, q, (int)t) &&
                     !rel_safe(T, T.P + q, t, x + 3 * (int64_t)v, x + 3 * (int64_t)v, T.rlo + 3 * t,
                               T.rhi + 3 * t);
            }
            hq_emit<EM>(pass, true, lane, n, o, v, (int)t, pa, pb, cap, Q, qn, A);
          }
        }
  }
  hq_finish<EM>(true, lane, n, cnt ? cnt + t : nullptr, Q, qn, A);
}

// edges query the edges of every level >= their own (equal level: higher index)
template <int EM>
__global__ void __launch_bounds__(128) k_hq_edges(BpTables T, int64_t E, const int* __restrict__ edge,
                                                  int* __restrict__ cnt, const int* __restrict__ off,
                                                  int* __restrict__ pa, int* __restrict__ pb, int64_t cap,
                                                  PairArgs A) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= E) return;
  const int lv = T.level[T.F + i];
  const double* il = T.elo + 3 * (T.F + i);
  const double* ih = T.ehi + 3 * (T.F + i);
  const double* fli = T.flo + 3 * (T.F + i);
  const double* fhi = T.fhi + 3 * (T.F + i);
  const int ia = edge[2 * i], ib = edge[2 * i + 1];
  int n = 0;
  const int o = EM == HQ_FILL ? off[i] : 0;
  __shared__ int2 qbuf[4][HQ_QUEUE];
  int2* Q = qbuf[threadIdx.x >> 5];
  int qn = 0;
  const unsigned mask = T.lmask[1];
  for (int l = lv; l < T.G.nlev; ++l) {
    if (!((mask >> l) & 1u)) continue;
    int c0[3], c1[3];
    hg_query_span(T.G, l, il, ih, c0, c1);
    // the span's cells in (a, b, c) order, 32 at a time: each lane loads one
    // cell's entry range, the warp walks the batch's entries flattened
    const int nb_ = c1[1] - c0[1] + 1, nc_ = c1[2] - c0[2] + 1;
    const int ncell_ = (c1[0] - c0[0] + 1) * nb_ * nc_;
    for (int cb_ = 0; cb_ < ncell_; cb_ += 32) {
          int my0 = 0, my1 = 0;
          {
            const int idx = cb_ + lane;
            if (idx < ncell_) {
              const int r = idx % (nb_ * nc_);
              const int cell = hg_cell(T.G, l, c0[0] + idx / (nb_ * nc_), c0[1] + r / nc_, c0[2] + r % nc_);
              my0 = T.edge_start[cell];
              my1 = T.edge_start[cell + 1];
            }
          }
          const CellBatch cbt = cell_batch(my0, my1);
          for (int base = 0; base < cbt.total; base += 32) {
            const int f = base + lane;
            const int e = batch_entry(cbt, f < cbt.total ? f : cbt.total - 1);
            bool pass = false;
            int j = 0;
            if (f < cbt.total) {
              j = T.edge_ent[e];
              const double* jl = T.edge_box + 6 * (int64_t)e;
              pass = !(l == lv && j <= (int)i) && boxes_meet(il, ih, jl, jl + 3);
              if (pass) {
                const int ja = edge[2 * j], jb = edge[2 * j + 1];
                const double* flj = T.flo + 3 * (T.F + j);
                const double* fhj = T.fhi + 3 * (T.F + j);
                // reference join filter (geometry.py:491-498) + reachability
                pass = !(ia == ja || ia == jb || ib == ja || ib == jb) && body_pass(T, ia, ja) && fli[0] <= fhj[0] &&
                       fli[1] <= fhj[1] && fli[2] <= fhj[2] && flj[0] <= fhi[0] && flj[1] <= fhi[1] &&
                       flj[2] <= fhi[2] && ref_reach(T.rc, T.F + i, T.F + j) &&
                       !rel_safe(T, T.F + i, T.F + j, T.rlo + 3 * (T.F + i), T.rhi + 3 * (T.F + i),
                                 T.rlo + 3 * (T.F + j), T.rhi + 3 * (T.F + j));
              }
            }
            hq_emit<EM>(pass, false, lane, n, o, min((int)i, j), max((int)i, j), pa, pb, cap, Q, qn, A);
          }
        }
  }
  hq_finish<EM>(false, lane, n, cnt ? cnt + i : nullptr, Q, qn, A);
}

// ---------------------------------------------------------------------------
// broad-phase build (host driver)

struct BpGrid {
  BpTables T{};
  bool empty = true;
  bool has_grid = false;  // false: boxes / filters only (the BVH enumeration, bvh.cuh)
  double filter_gap = 0.0;  // the reference filter gap with a rounding margin (bvh.cuh node tests)
  double crowd = 0.0;       // BP_GRID_AUTO: the crowding probe when it ran (> BP_CROWD_LIMIT: a timed choice)
  int crowd_bucket = 0;     // ilogb(crowd)
  double raw_mean = 0.0;    // mean largest raw-box extent of the triangles and edges
};

enum { BP_GRID_NONE = 0, BP_GRID_ALWAYS = 1, BP_GRID_AUTO = 2 };
// Crowded calls: the measured times of each method per log2 bucket of the
// crowding (ctx enum_ms) give the estimates; unknown BVH -> BVH (bounded),
// unknown grid -> tried only below BP_GRID_TRY; else the faster estimate,
// the other re-measured every BP_REPROBE crowded calls when it is within 2x.
#define BP_BUCKETS 32
static bool choose_bvh(mp_ctx* c, int k, double crowd);

// BP_GRID_AUTO: when the enumeration boxes average more than BP_AUTO_RATIO
// times the raw ones, the grid is built and its crowding measured -- sum
// over cells of (objects in the cell)^2, per object, ~ the box tests per
// query.  Up to BP_CROWD_LIMIT the grid enumerates.  Past it the cheaper
// method depends on the motion: where the relative-motion prefilter rejects
// most box-overlapping pairs (bodies moving coherently: C5 restart
// directions, crowd 250-60000) the BVH prunes whole subtrees (0.05-0.13 s
// vs the grid's 0.6-15.5 s); where most of them pass (the C3 twist, up to
// 2^31 pairs) the grid's warp-wide cell scans are 1.5-3x faster.  So
// crowded calls are timed and chosen by choose_bvh below (the grid is only
// tried blind below BP_GRID_TRY, where a wrong guess costs at most ~0.2 s).
// Both emit the same pair set: the choice changes timing only.
#define BP_AUTO_RATIO 1.6
#define BP_CROWD_LIMIT 100.0
#define BP_REPROBE 32
#define BP_GRID_TRY 1000.0

static bool choose_bvh(mp_ctx* c, int k, double crowd) {
  // estimate of method m at bucket k: its time there, else extrapolated x2
  // per bucket from the nearest lower bucket it ran in, else the nearest
  // higher one as is; < 0 when it never ran
  auto estimate = [&](int m) {
    const double* t = c->enum_ms.ms[m];
    for (int j = k; j >= 0; --j)
      if (t[j] >= 0.0) return t[j] * ldexp(1.0, k - j);
    for (int j = k + 1; j < BP_BUCKETS; ++j)
      if (t[j] >= 0.0) return t[j];
    return -1.0;
  };
  const double tg = estimate(0), tb = estimate(1);
  bool bvh;
  if (tb < 0.0) bvh = true;                            // the BVH's worst cases are bounded
  else if (tg < 0.0) bvh = !(crowd < BP_GRID_TRY);     // the grid's are not
  else bvh = tb <= tg;
  if (++c->n_crowded % BP_REPROBE == 0 && tg >= 0.0 && tb >= 0.0) {
    const double chosen = bvh ? tb : tg, other = bvh ? tg : tb;
    if (other <= 2.0 * chosen) bvh = !bvh;  // re-measure a close alternative
  }
  return bvh;
}

__global__ void k_cell_crowd(int64_t ncell, const int* __restrict__ a, const int* __restrict__ b,
                             const int* __restrict__ c, unsigned long long* __restrict__ out) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncell; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long n = (unsigned long long)(a[i] + b[i] + c[i]);
    s += n * n;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// Everything one broad-phase call at (x, mb, d_hat) needs: boxes, levels,
// reference cell ranges and the per-level cell tables of triangles / edges /
// surface points.  infl (per vertex, device) switches to tight enumeration.
static BpGrid build_bp(mp_ctx* c, const double* x, double mb, double d_hat, const double* infl = nullptr,
                       int body_mode = 0, int grid_mode = BP_GRID_ALWAYS) {
  BpGrid B;
  const int64_t F = c->F, P = c->F + c->E, V = c->V, nobj = P + V;
  B.T.F = F;
  B.T.P = P;
  B.T.body = c->body.p;
  B.T.body_mode = body_mode;
  if (F == 0) return B;
  const double gap = d_hat + 2.0 * mb;
  cudaStream_t st = c->stream;
  for (DBuf<double>* b : {&c->box_rlo, &c->box_rhi, &c->box_flo, &c->box_fhi}) b->ensure(3 * P);
  c->box_elo.ensure(3 * nobj);
  c->box_ehi.ensure(3 * nobj);
  CUDA_CHECK(cudaMemsetAsync(c->dscal.p + 40, 0, sizeof(double), st));
  k_prim_boxes<<<grid_for(P, 256), 256, 0, st>>>(F, c->E, c->tri, c->edge, x, gap, infl, c->box_rlo, c->box_rhi,
                                                  c->box_flo, c->box_fhi, c->box_elo, c->box_ehi, c->dscal.p + 40);
  LAUNCH_CHECK();
  if (V) {
    k_point_boxes<<<grid_for(V, 256), 256, 0, st>>>(V, c->sverts, x, gap, infl, c->box_elo.p + 3 * P,
                                                     c->box_ehi.p + 3 * P);
    LAUNCH_CHECK();
  }
  const int nb = 64;
  c->red_part.ensure(BOX_STATS * nb + 1);
  k_box_stats<<<nb, 256, 0, st>>>(P, c->box_elo, c->box_ehi, c->box_rlo, c->box_rhi, c->red_part);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(c->red_part.p + BOX_STATS * nb, c->dscal.p + 40, sizeof(double), cudaMemcpyDeviceToDevice,
                             st));
  std::vector<double> part(BOX_STATS * nb + 1);
  CUDA_CHECK(cudaMemcpyAsync(part.data(), c->red_part.p, sizeof(double) * (BOX_STATS * nb + 1), cudaMemcpyDeviceToHost,
                             st));
  sync_stream(c);
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, ext = 0.0, rext = 0.0;
  for (int b = 0; b < nb; ++b) {
    for (int k = 0; k < 3; ++k) {
      mn[k] = fmin(mn[k], -part[BOX_STATS * b + k]);
      mx[k] = fmax(mx[k], part[BOX_STATS * b + 3 + k]);
    }
    ext += part[BOX_STATS * b + 6];
    rext += part[BOX_STATS * b + 7];
  }
  auto& g = c->grid;
  // the reference's cell and pad (geometry.py:465-466) -> per-object ranges
  const double ref_cell = fmax(part[BOX_STATS * nb], d_hat + mb);
  const double ref_pad = 0.5 * d_hat + mb;
  g.rc.ensure(6 * nobj);
  k_ref_cells<<<grid_for(nobj, 256), 256, 0, st>>>(P, V, c->sverts, x, c->box_rlo, c->box_rhi, ref_pad, ref_cell,
                                                   g.rc);
  LAUNCH_CHECK();
  {
    // the filter tests of the BVH nodes: gap plus a relative and an absolute
    // (a few ulps of the largest coordinate) rounding margin
    double amax = 0.0;
    for (int k = 0; k < 3; ++k) amax = fmax(amax, fmax(fabs(mn[k]), fabs(mx[k])));
    B.filter_gap = gap * (1.0 + 1e-9) + 1e-15 * (std::isfinite(amax) ? amax : 0.0);
    B.raw_mean = rext / (double)std::max<int64_t>(1, P);
  }
  auto boxes_only = [&]() {  // the BVH's inputs: boxes, filters, reference cell ranges
    BpTables& T = B.T;
    T.rc = g.rc;
    T.flo = c->box_flo; T.fhi = c->box_fhi;
    T.elo = c->box_elo; T.ehi = c->box_ehi;
    T.rlo = c->box_rlo; T.rhi = c->box_rhi;
    B.empty = false;
    B.has_grid = false;
  };
  if (grid_mode == BP_GRID_NONE) {
    boxes_only();
    return B;
  }
  const bool probe = grid_mode == BP_GRID_AUTO && ext > BP_AUTO_RATIO * rext;
  B.has_grid = true;
  // level 0: about the mean primitive extent, at most ~4M cells
  double span = fmax(fmax(mx[0] - mn[0], mx[1] - mn[1]), mx[2] - mn[2]);
  if (!(span > 0.0) || !std::isfinite(span)) span = 1.0;
  double h0 = ext / (double)P;
  if (!(h0 > 0.0) || !std::isfinite(h0)) h0 = span;
  h0 = fmax(h0, span * 1e-6);
  HGrid& G = B.T.G;
  for (;;) {
    double cells0 = 1.0;
    for (int k = 0; k < 3; ++k) cells0 *= floor((mx[k] - mn[k]) / h0) + 1.0;
    if (cells0 <= (double)(1 << 22)) break;
    h0 *= 2.0;
  }
  G.h0 = h0;
  G.inv_h0 = 1.0 / h0;
  for (int k = 0; k < 3; ++k) G.o[k] = mn[k];
  int64_t tot_cells = 0;
  G.nlev = 0;
  for (int l = 0; l < HG_MAX_LEVELS; ++l) {
    const double h = ldexp(h0, l);
    int small = 1;
    for (int k = 0; k < 3; ++k) {
      // as many cells as hg_coord can return (it clamps into [0, n-1])
      double nk = floor((mx[k] - mn[k]) * ldexp(G.inv_h0, -l)) + 1.0;
      if (!(nk >= 1.0)) nk = 1.0;
      G.n[l][k] = (int)nk;
      small = small && (G.n[l][k] <= 2);
    }
    G.off[l] = (int)tot_cells;
    tot_cells += (int64_t)G.n[l][0] * G.n[l][1] * G.n[l][2];
    G.nlev = l + 1;
    if (small && h >= span) break;
  }
  G.off[G.nlev] = (int)tot_cells;
  g.level.ensure(nobj);
  c->cell_cnt.ensure(nobj + 1);
  c->cell_off.ensure(nobj + 1);
  unsigned* lmask = (unsigned*)(c->counters.p + 12);
  CUDA_CHECK(cudaMemsetAsync(lmask, 0, 3 * sizeof(unsigned), st));
  k_obj_level<<<grid_for(nobj, 256), 256, 0, st>>>(nobj, F, P, G, c->box_elo, c->box_ehi, g.level, c->cell_cnt,
                                                   lmask);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemsetAsync(c->cell_cnt.p + nobj, 0, sizeof(int), st));
  exclusive_scan(c, c->cell_cnt, c->cell_off, nobj + 1);
  // one entry per object,
  // so the entry arrays are sized without reading the total back
  const int64_t total_cap = nobj;
  const int* total_dev = c->cell_off.p + nobj;
  const size_t ncell = (size_t)tot_cells;
  for (DBuf<int>* b : {&g.tri_cnt, &g.tri_start, &g.edge_cnt, &g.edge_start, &g.pt_cnt, &g.pt_start})
    b->ensure(ncell + 1);
  g.ecell.ensure((size_t)total_cap + 1);
  g.tri_ent.ensure((size_t)total_cap + 1);
  g.edge_ent.ensure((size_t)total_cap + 1);
  g.pt_ent.ensure((size_t)total_cap + 1);
  g.tri_box.ensure(6 * (size_t)F + 6);
  g.edge_box.ensure(6 * (size_t)c->E + 6);
  g.pt_box.ensure(6 * (size_t)V + 6);
  for (DBuf<int>* b : {&g.tri_cnt, &g.edge_cnt, &g.pt_cnt})
    CUDA_CHECK(cudaMemsetAsync(b->p, 0, sizeof(int) * (ncell + 1), st));
  k_entry_hist<<<grid_for(total_cap, 256), 256, 0, st>>>(total_dev, nobj, F, P, G, c->cell_off, g.level, c->box_elo,
                                                         c->box_ehi, g.ecell, g.tri_cnt, g.edge_cnt, g.pt_cnt);
  LAUNCH_CHECK();
  if (probe) {
    c->crowd_dev.ensure(1);
    CUDA_CHECK(cudaMemsetAsync(c->crowd_dev.p, 0, sizeof(unsigned long long), st));
    k_cell_crowd<<<4 * 148, 256, 0, st>>>((int64_t)ncell, g.tri_cnt, g.edge_cnt, g.pt_cnt, c->crowd_dev);
    LAUNCH_CHECK();
    unsigned long long sq = 0;
    CUDA_CHECK(cudaMemcpyAsync(&sq, c->crowd_dev.p, sizeof(sq), cudaMemcpyDeviceToHost, st));
    sync_stream(c);
    const double crowd = (double)sq / (double)std::max<int64_t>(1, nobj);
    if (getenv("MP_BP_TRACE"))
      fprintf(stderr, "  bp crowd %.1f (enumeration / raw extent %.2f)\n", crowd, ext / fmax(rext, 1e-300));
    if (crowd > BP_CROWD_LIMIT) {
      B.crowd = crowd;
      B.crowd_bucket = std::min(BP_BUCKETS - 1, std::max(0, ilogb(crowd)));
      const bool bvh = choose_bvh(c, B.crowd_bucket, crowd);
      if (bvh) {
        boxes_only();
        return B;
      }
    }
  }
  exclusive_scan(c, g.tri_cnt, g.tri_start, ncell + 1);
  exclusive_scan(c, g.edge_cnt, g.edge_start, ncell + 1);
  exclusive_scan(c, g.pt_cnt, g.pt_start, ncell + 1);
  // the counts become per-cell fill cursors
  for (DBuf<int>* b : {&g.tri_cnt, &g.edge_cnt, &g.pt_cnt})
    CUDA_CHECK(cudaMemsetAsync(b->p, 0, sizeof(int) * (ncell + 1), st));
  k_entry_fill<<<grid_for(total_cap, 256), 256, 0, st>>>(total_dev, nobj, F, P, c->cell_off, g.ecell, g.tri_start,
                                                         g.edge_start, g.pt_start, g.tri_cnt, g.edge_cnt, g.pt_cnt,
                                                         g.tri_ent, g.edge_ent, g.pt_ent, c->box_elo, c->box_ehi,
                                                         g.tri_box, g.edge_box, g.pt_box);
  LAUNCH_CHECK();
  BpTables& T = B.T;
  T.tri_box = g.tri_box; T.edge_box = g.edge_box; T.pt_box = g.pt_box;
  T.pt_start = g.pt_start; T.pt_ent = g.pt_ent;
  T.tri_start = g.tri_start; T.tri_ent = g.tri_ent;
  T.edge_start = g.edge_start; T.edge_ent = g.edge_ent;
  T.level = g.level;
  T.lmask = lmask;
  T.rc = g.rc;
  T.flo = c->box_flo; T.fhi = c->box_fhi;
  T.elo = c->box_elo; T.ehi = c->box_ehi;
  T.rlo = c->box_rlo; T.rhi = c->box_rhi;  // (after every ensure above: the pointers are final)
  B.empty = false;
  return B;
}

// 64-bit sum of the per-query pair counts of the ordered list (each count is
// a 32-bit non-negative int; their int32 scan wraps past 2^31 pairs)
__global__ void k_sum_counts(int64_t n, const int* __restrict__ cnt, unsigned long long* __restrict__ total) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned)cnt[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(total, s);
}

// The reference pair list of the grid (PT if which & 1, EE if which & 2):
// count pass, exclusive scan, fill pass into the current capacity -- no host
// sync; the counts stay on the device (qoff[V+F] = PT pairs, qoff[V+F+E] =
// all) and the caller checks the capacity at its own readback.  Deterministic
// order: points' pairs, then triangles' pairs (both PT), then edges' pairs.
static void collect_pairs(mp_ctx* c, const double* x, const BpGrid& B, int which) {
  const int64_t V = c->V, F = c->F, E = c->E;
  const int64_t nq = V + F + E;
  auto& g = c->grid;
  g.qcnt.ensure(nq + 1);
  g.qoff.ensure(nq + 1);
  cudaStream_t st = c->stream;
  CUDA_CHECK(cudaMemsetAsync(g.qcnt.p, 0, sizeof(int) * (nq + 1), st));
  if (B.empty) {
    CUDA_CHECK(cudaMemsetAsync(g.qoff.p, 0, sizeof(int) * (nq + 1), st));
    return;
  }
  if (g.pa.n < 1024) {
    g.pa.ensure(1 << 16);
    g.pb.ensure(1 << 16);
  }
  const int64_t cap = (int64_t)std::min(g.pa.n, g.pb.n);
  if ((which & 1) && V) {
    k_hq_points<HQ_COUNT><<<grid_for(32 * V, 128), 128, 0, st>>>(B.T, V, c->sverts, c->tri, x, g.qcnt.p, nullptr,
                                                                  nullptr, nullptr, 0, PairArgs{});
    LAUNCH_CHECK();
    k_hq_tris<HQ_COUNT><<<grid_for(32 * F, 128), 128, 0, st>>>(B.T, F, c->sverts, c->tri, x, g.qcnt.p + V, nullptr,
                                                                nullptr, nullptr, 0, PairArgs{});
    LAUNCH_CHECK();
  }
  if ((which & 2) && E > 1) {
    k_hq_edges<HQ_COUNT><<<grid_for(32 * E, 128), 128, 0, st>>>(B.T, E, c->edge, g.qcnt.p + V + F, nullptr, nullptr,
                                                                 nullptr, 0, PairArgs{});
    LAUNCH_CHECK();
  }
  // the int32 scan below must not wrap: a 64-bit total of the counts rides
  // on the caller's readback (h_npairs) and is checked before the list is used
  c->n_pairs_dev.ensure(1);
  CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, sizeof(unsigned long long), st));
  k_sum_counts<<<148, 256, 0, st>>>(nq, g.qcnt.p, c->n_pairs_dev.p);
  LAUNCH_CHECK();
  exclusive_scan(c, g.qcnt, g.qoff, nq + 1);
  if ((which & 1) && V) {
    k_hq_points<HQ_FILL><<<grid_for(32 * V, 128), 128, 0, st>>>(B.T, V, c->sverts, c->tri, x, nullptr, g.qoff.p, g.pa,
                                                                 g.pb, cap, PairArgs{});
    LAUNCH_CHECK();
    k_hq_tris<HQ_FILL><<<grid_for(32 * F, 128), 128, 0, st>>>(B.T, F, c->sverts, c->tri, x, nullptr, g.qoff.p + V,
                                                               g.pa, g.pb, cap, PairArgs{});
    LAUNCH_CHECK();
  }
  if ((which & 2) && E > 1) {
    k_hq_edges<HQ_FILL><<<grid_for(32 * E, 128), 128, 0, st>>>(B.T, E, c->edge, nullptr, g.qoff.p + V + F, g.pa,
                                                                g.pb, cap, PairArgs{});
    LAUNCH_CHECK();
  }
}

// Broad phase + the per-pair work of MODE.  Returns the number of reference
// pairs (CONTACT: active constraints emitted, may exceed O.cap -- the
// caller grows and retries); *flag = counters[1] (penetration / failed
// certificate).  RAW leaves the list in c->grid.pa / pb and returns n,
// with *n_pt_out the PT prefix length.
// Fused enumeration (MODE = CONTACT / CCD / CERT without a stored list): the
// hq kernels do the per-pair work themselves; the pair count lands in
// c->n_pairs_dev.
template <int MODE>
static void fused_pairs(mp_ctx* c, const double* x, const BpGrid& B, const PairArgs& A) {
  const int64_t V = c->V, F = c->F, E = c->E;
  cudaStream_t st = c->stream;
  if (B.empty) return;
  if (V) {
    k_hq_points<MODE><<<grid_for(32 * V, 128), 128, 0, st>>>(B.T, V, c->sverts, c->tri, x, nullptr, nullptr,
                                                              nullptr, nullptr, 0, A);
    LAUNCH_CHECK();
    k_hq_tris<MODE><<<grid_for(32 * F, 128), 128, 0, st>>>(B.T, F, c->sverts, c->tri, x, nullptr, nullptr, nullptr,
                                                            nullptr, 0, A);
    LAUNCH_CHECK();
  }
  if (E > 1) {
    k_hq_edges<MODE><<<grid_for(32 * E, 128), 128, 0, st>>>(B.T, E, c->edge, nullptr, nullptr, nullptr, nullptr, 0,
                                                             A);
    LAUNCH_CHECK();
  }
}

// MP_BP_TRACE=1: per-kernel host timings of the one-pass enumeration and a
// per-level summary of the grid (objects per class, largest cell) on stderr
struct BpTrace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit BpTrace(cudaStream_t s) : on(getenv("MP_BP_TRACE") != nullptr), st(s) {
    if (on) { CUDA_CHECK(cudaStreamSynchronize(st)); t0 = std::chrono::steady_clock::now(); }
  }
  void lap(const char* what) {
    if (!on) return;
    CUDA_CHECK(cudaStreamSynchronize(st));
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "  bp %-8s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

static void bp_trace_levels(mp_ctx* c, const BpGrid& B) {
  const HGrid& G = B.T.G;
  const int64_t nobj = B.T.P + c->V;
  std::vector<int> lev(nobj);
  CUDA_CHECK(cudaMemcpy(lev.data(), B.T.level, sizeof(int) * nobj, cudaMemcpyDeviceToHost));
  const int64_t ncell = G.off[G.nlev];
  std::vector<int> st[3];
  const int* starts[3] = {B.T.tri_start, B.T.edge_start, B.T.pt_start};
  for (int q = 0; q < 3; ++q) {
    st[q].resize(ncell + 1);
    CUDA_CHECK(cudaMemcpy(st[q].data(), starts[q], sizeof(int) * (ncell + 1), cudaMemcpyDeviceToHost));
  }
  fprintf(stderr, "  bp grid h0=%.4g nlev=%d\n", G.h0, G.nlev);
  for (int l = 0; l < G.nlev; ++l) {
    int64_t cnt[3] = {0, 0, 0};
    for (int64_t i = 0; i < nobj; ++i)
      if (lev[i] == l) ++cnt[i < B.T.F ? 0 : (i < B.T.P ? 1 : 2)];
    int mx[3] = {0, 0, 0};
    for (int64_t cc = G.off[l]; cc < G.off[l + 1]; ++cc)
      for (int q = 0; q < 3; ++q) mx[q] = std::max(mx[q], st[q][cc + 1] - st[q][cc]);
    if (cnt[0] + cnt[1] + cnt[2])
      fprintf(stderr, "  bp L%-2d cells %dx%dx%d  tri %lld (max/cell %d)  edge %lld (%d)  pt %lld (%d)\n", l,
              G.n[l][0], G.n[l][1], G.n[l][2], (long long)cnt[0], mx[0], (long long)cnt[1], mx[1],
              (long long)cnt[2], mx[2]);
  }
}

template <int MODE>
static int64_t run_bp(mp_ctx* c, const double* x, const BpGrid& B, BpOut O, ContactParams CP, CcdParams CC,
                      int* flag, int which = 3, int64_t* n_pt_out = nullptr) {
  const int64_t V = c->V, F = c->F, E = c->E, nq = V + F + E;
  auto& g = c->grid;
  // fused for the constraint set only: the CCD / certificate pair work needs
  // ~100 registers, and inlined into the enumeration it costs more occupancy
  // than the count pass it saves (measured: 362 vs 264 us per edge pass)
  const bool fused = c->bp_fused == 2 && MODE == BP_CONTACT && which == 3 && !n_pt_out;
  // order-free consumers (contacts are key-sorted afterwards; CCD / the
  // certificate reduce minima and flags) without a stored per-pair output:
  // one-pass unordered list, then the pair kernel
  const bool append = c->bp_fused == 1 && MODE != BP_RAW && which == 3 && !n_pt_out &&
                      !(MODE == BP_CCD && O.verts);
  for (int attempt = 0; attempt < 3; ++attempt) {
    CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 3 * sizeof(int), c->stream));
    O.counter = c->counters.p;
    if (fused) {
      // results are final after one pass (CONTACT: the caller checks O.cap)
      c->n_pairs_dev.ensure(1);
      CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, sizeof(unsigned long long), c->stream));
      PairArgs A{c->tri, c->tri_sorted, c->edge, x, O, CP, CC, c->n_pairs_dev.p, nullptr, nullptr, nullptr, 0};
      fused_pairs<MODE>(c, x, B, A);
      CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CUDA_CHECK(cudaMemcpyAsync(c->h_npairs, c->n_pairs_dev.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 c->stream));
      if (c->rb_extra)
        CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->rb_extra, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      sync_stream(c);
      if (flag) *flag = c->h_cnt[1];
      return MODE == BP_CONTACT ? c->h_cnt[0] : (int64_t)*c->h_npairs;
    }
    if (append) {
      if (g.pa.n < 1024) { g.pa.ensure(1 << 16); g.pb.ensure(1 << 16); }
      if (g.ea.n < 1024) { g.ea.ensure(1 << 16); g.eb.ensure(1 << 16); }
      int* cnt = c->counters.p + 8;  // [8] PT, [9] EE appended
      CUDA_CHECK(cudaMemsetAsync(cnt, 0, 3 * sizeof(int), c->stream));  // [10]: append overflow flag
      const int64_t cap_pt = (int64_t)std::min(g.pa.n, g.pb.n), cap_ee = (int64_t)std::min(g.ea.n, g.eb.n);
      if (!B.empty) {
        if (getenv("MP_BP_TRACE")) bp_trace_levels(c, B);
        BpTrace tr(c->stream);
        PairArgs A{c->tri, c->tri_sorted, c->edge, x, O, CP, CC, nullptr, g.pa, g.pb, cnt, cap_pt};
        if (V) {
          k_hq_points<HQ_APPEND><<<grid_for(32 * V, 128), 128, 0, c->stream>>>(B.T, V, c->sverts, c->tri, x, nullptr,
                                                                               nullptr, nullptr, nullptr, 0, A);
          LAUNCH_CHECK();
          tr.lap("points");
          k_hq_tris<HQ_APPEND><<<grid_for(32 * F, 128), 128, 0, c->stream>>>(B.T, F, c->sverts, c->tri, x, nullptr,
                                                                             nullptr, nullptr, nullptr, 0, A);
          LAUNCH_CHECK();
          tr.lap("tris");
        }
        if (E > 1) {
          PairArgs Ae = A;
          Ae.app_a = g.ea; Ae.app_b = g.eb; Ae.app_cnt = cnt + 1; Ae.app_cap = cap_ee; Ae.app_ee = 1;
          k_hq_edges<HQ_APPEND><<<grid_for(32 * E, 128), 128, 0, c->stream>>>(B.T, E, c->edge, nullptr, nullptr,
                                                                              nullptr, nullptr, 0, Ae);
          LAUNCH_CHECK();
          tr.lap("edges");
        }
        k_pairs_app<MODE><<<8 * 148, 256, 0, c->stream>>>(cnt, cap_pt, cap_ee, g.pa, g.pb, g.ea, g.eb, A);
        LAUNCH_CHECK();
        tr.lap("pairs");
      }
      CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 5, cnt, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      if (c->rb_extra)  // the caller's scalar rides on this readback (h_scal[0])
        CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->rb_extra, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      sync_stream(c);
      if (c->h_cnt[7]) {  // >= 2^30 candidate pairs: no list; rerun list-free with a 64-bit count
        CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 3 * sizeof(int), c->stream));
        c->n_pairs_dev.ensure(1);
        CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, sizeof(unsigned long long), c->stream));
        PairArgs A{c->tri, c->tri_sorted, c->edge, x, O, CP, CC, c->n_pairs_dev.p, nullptr, nullptr, nullptr, 0};
        fused_pairs<MODE>(c, x, B, A);
        CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CUDA_CHECK(cudaMemcpyAsync(c->h_npairs, c->n_pairs_dev.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                   c->stream));
        if (c->rb_extra)  // the caller's scalar (CCD minimum) as recomputed by this full pass
          CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->rb_extra, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        sync_stream(c);
        if (flag) *flag = c->h_cnt[1];
        return MODE == BP_CONTACT ? c->h_cnt[0] : (int64_t)*c->h_npairs;
      }
      const int64_t n_pt = c->h_cnt[5], n_ee = c->h_cnt[6];
      if (n_pt > cap_pt || n_ee > cap_ee) {  // grow and rerun (minima / flags are idempotent)
        if (n_pt > cap_pt) { g.pa.ensure((size_t)(n_pt * 1.25) + 1024); g.pb.ensure((size_t)(n_pt * 1.25) + 1024); }
        if (n_ee > cap_ee) { g.ea.ensure((size_t)(n_ee * 1.25) + 1024); g.eb.ensure((size_t)(n_ee * 1.25) + 1024); }
        continue;
      }
      if (flag) *flag = c->h_cnt[1];
      return MODE == BP_CONTACT ? c->h_cnt[0] : n_pt + n_ee;  // CONTACT: constraints emitted
    }
    collect_pairs(c, x, B, which);
    const int64_t cap = (int64_t)std::min(g.pa.n, g.pb.n);
    if (MODE != BP_RAW && !B.empty) {
      int sms = 148;
      PairArgs A{c->tri, c->tri_sorted, c->edge, x, O, CP, CC, nullptr, nullptr, nullptr, nullptr, 0};
      k_pairs<MODE><<<(unsigned)(8 * sms), 256, 0, c->stream>>>(g.qoff.p + V + F, g.qoff.p + nq, cap, g.pa, g.pb, A);
      LAUNCH_CHECK();
    }
    // one readback: the mode's counters and the pair-list sizes
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 5, g.qoff.p + V + F, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 6, g.qoff.p + nq, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    if (c->rb_extra)
      CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->rb_extra, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (!B.empty)
      CUDA_CHECK(cudaMemcpyAsync(c->h_npairs, c->n_pairs_dev.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 c->stream));
    sync_stream(c);
    if (!B.empty && *c->h_npairs > (unsigned long long)HQ_APPEND_LIMIT)
      throw MpError(MP_ERR_CAPACITY, "ordered broad-phase list exceeds 2^30 pairs (the default one-pass "
                                     "enumeration handles this size)");
    const int64_t n_pt = c->h_cnt[5], n = c->h_cnt[6];
    if (n > cap) {  // the list did not fit: grow and rerun (results are idempotent)
      g.pa.ensure((size_t)(n * 1.25) + 1024);
      g.pb.ensure((size_t)(n * 1.25) + 1024);
      continue;
    }
    if (n_pt_out) *n_pt_out = n_pt;
    if (flag) *flag = MODE == BP_RAW ? 0 : c->h_cnt[1];
    return MODE == BP_CONTACT ? c->h_cnt[0] : n;
  }
  throw MpError(MP_ERR_CAPACITY, "broad-phase pair list capacity retry failed");
}
