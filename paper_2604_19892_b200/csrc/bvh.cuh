// bvh.cuh -- motion-aware bounding-volume hierarchy for the tight CCD and
// certificate enumeration (the reference pair set of ccd.py:221-241 under the
// exact filters of bp.cuh).
//
// The hierarchical grid (bp.cuh) sizes its cells on the enumeration boxes.
// When a direction p is large over much of the scene (a restart direction
// before alpha_d clamps it), every box grows to ~2 |p|_inf, the grid
// collapses to a few cells holding 10^4-10^5 objects each, and the box tests
// explode quadratically (seconds per call at C5), although the exact
// relative-motion prefilter (bp.cuh rel_safe) keeps only ~10^7 pairs: most
// of a ball moves with its neighbourhood.  Here the pruning itself is
// relative.  Each node of a fixed-topology 8-ary tree over the objects
// (ordered by their smallest Morton-renumbered vertex id, so siblings are
// spatial neighbours) carries, rounded outward to float:
//   - the union of its objects' raw boxes and enumeration boxes,
//   - the box of their motion centres c_o and the largest motion radius m_o
//     (k_obj_motion),
// and a query object q skips a child whose enumeration box misses q's, whose
// raw box is beyond the reference filter gap, or for which
//   0.9 dist(raw_q, raw_node) > 4 max(m_q, m_node + max_{c in cbox} |c_q - c|),
// the node-wide form of rel_safe (M <= max(m_q, m_o + |c_q - c_o|)).  Every
// skip is implied for each object below, so the objects reached and tested
// with the unchanged per-pair predicate are a superset of the passing ones:
// the emitted pair set is the grid's, bit for bit.
//
// Scale: threads hand long traversals on as tasks (rounds, lists grown to
// the requested size, query chunks past the memory budget); past the 2^30
// one-pass list the pairs are worked where they are found (list-free), and
// the CCD then adds an exact alpha prune (run_bvh).
#pragma once

#include "bp.cuh"

#define BVH_W 8
#define BVH_MAX_LEVELS 12
// depth-first, children pushed after their parent is popped: at most
// 1 + 7 (levels - 1) entries are live
#define BVH_STACK (1 + (BVH_W - 1) * (BVH_MAX_LEVELS - 1))

struct BvhNode {
  float rlo[3], rhi[3];  // raw boxes (union)
  float elo[3], ehi[3];  // enumeration boxes (union)
  float clo[3], chi[3];  // motion centres (box)
  float m;               // largest motion radius
  float amax;            // largest alpha_d bound of its objects' subdomains (the alpha prune; 1 when unused)
};

struct BvhTree {
  const BvhNode* node;        // all levels, leaves (level 0) first
  const int* order;           // sorted position -> object index within the class
  int64_t n;                  // objects
  int nlev;                   // levels; level nlev-1 is the root
  int64_t off[BVH_MAX_LEVELS + 1];
  int64_t cnt[BVH_MAX_LEVELS];
};

__device__ __forceinline__ float f_dn(double v) { return __double2float_rd(v); }
__device__ __forceinline__ float f_up(double v) { return __double2float_ru(v); }

// leaf level: thread per object, groups of 8 lanes reduce one leaf.  base =
// object id offset of the class in the per-object arrays (tris 0, edges F).
__global__ void k_bvh_leaves(int64_t n, int64_t base, const int* __restrict__ order, const double* __restrict__ rlo,
                             const double* __restrict__ rhi, const double* __restrict__ elo,
                             const double* __restrict__ ehi, const double* __restrict__ mot,
                             BvhNode* __restrict__ leaf, const int* __restrict__ ids, int per,
                             const double* __restrict__ alpha_d, int bs) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = s < n;
  float v[19];
  float am = 1.0f;
  if (live && alpha_d) {  // the alpha prune: max over the object's vertices' subdomain bounds
    const int64_t oc = order[s];
    double a = 0.0;
    for (int k = 0; k < per; ++k) a = fmax(a, alpha_d[ids[per * oc + k] / bs]);
    am = f_up(a);
  }
  if (live) {
    const int64_t o = base + order[s];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = f_dn(rlo[3 * o + k]);
      v[3 + k] = f_up(rhi[3 * o + k]);
      v[6 + k] = f_dn(elo[3 * o + k]);
      v[9 + k] = f_up(ehi[3 * o + k]);
      const double cc = mot ? mot[4 * o + k] : 0.0;
      v[12 + k] = f_dn(cc);
      v[15 + k] = f_up(cc);
    }
    v[18] = mot ? f_up(mot[4 * o + 3]) : 0.0f;
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = v[6 + k] = v[12 + k] = INFINITY;
      v[3 + k] = v[9 + k] = v[15 + k] = -INFINITY;
    }
    v[18] = 0.0f;
  }
#pragma unroll
  for (int o = 1; o < BVH_W; o <<= 1) {
#pragma unroll
    for (int q = 0; q < 19; ++q) {
      const float w = __shfl_xor_sync(0xffffffffu, v[q], o);
      const bool is_lo = (q < 3) || (q >= 6 && q < 9) || (q >= 12 && q < 15);
      v[q] = is_lo ? fminf(v[q], w) : fmaxf(v[q], w);
    }
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  if (live && (s & (BVH_W - 1)) == 0) {
    BvhNode& d = leaf[s / BVH_W];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      d.rlo[k] = v[k]; d.rhi[k] = v[3 + k];
      d.elo[k] = v[6 + k]; d.ehi[k] = v[9 + k];
      d.clo[k] = v[12 + k]; d.chi[k] = v[15 + k];
    }
    d.m = v[18];
    d.amax = am;
  }
}

// one level up: thread per child, groups of 8 lanes reduce one parent
__global__ void k_bvh_up(int64_t nchild, const BvhNode* __restrict__ child, BvhNode* __restrict__ parent) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = s < nchild;
  float v[19];
  float am = 0.0f;
  if (live) {
    const BvhNode& c = child[s];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = c.rlo[k]; v[3 + k] = c.rhi[k];
      v[6 + k] = c.elo[k]; v[9 + k] = c.ehi[k];
      v[12 + k] = c.clo[k]; v[15 + k] = c.chi[k];
    }
    v[18] = c.m;
    am = c.amax;
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      v[k] = v[6 + k] = v[12 + k] = INFINITY;
      v[3 + k] = v[9 + k] = v[15 + k] = -INFINITY;
    }
    v[18] = 0.0f;
  }
#pragma unroll
  for (int o = 1; o < BVH_W; o <<= 1) {
#pragma unroll
    for (int q = 0; q < 19; ++q) {
      const float w = __shfl_xor_sync(0xffffffffu, v[q], o);
      const bool is_lo = (q < 3) || (q >= 6 && q < 9) || (q >= 12 && q < 15);
      v[q] = is_lo ? fminf(v[q], w) : fmaxf(v[q], w);
    }
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  if (live && (s & (BVH_W - 1)) == 0) {
    BvhNode& d = parent[s / BVH_W];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      d.rlo[k] = v[k]; d.rhi[k] = v[3 + k];
      d.elo[k] = v[6 + k]; d.ehi[k] = v[9 + k];
      d.clo[k] = v[12 + k]; d.chi[k] = v[15 + k];
    }
    d.m = v[18];
    d.amax = am;
  }
}

// the query side of a node test
struct BvhQuery {
  double elo[3], ehi[3];  // enumeration box
  double rlo[3], rhi[3];  // raw box
  double c[3], m;         // motion centre / radius (rel != 0)
  double gap;             // reference filter gap (with margin)
  bool rel;
  double amax;            // the alpha prune: the query's subdomain bound (> 1: off)
  double near_r;          // near pass: raw separation limit (<= 0: off)
};

// squared separation of two boxes
__device__ __forceinline__ double box_gap2(const double* l1, const double* h1, const double* l2, const double* h2) {
  double g2 = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double d = fmax(0.0, fmax(l1[k] - h2[k], l2[k] - h1[k]));
    g2 += d * d;
  }
  return g2;
}

// May any object below `nd` pass the per-pair predicate against q?
__device__ __forceinline__ bool bvh_visit(const BvhQuery& q, const BvhNode& nd) {
  double d2 = 0.0, c2 = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // enumeration boxes meet (boxes_meet on every object below)
    if (q.elo[k] > (double)nd.ehi[k] || (double)nd.elo[k] > q.ehi[k]) return false;
    // reference filter: per-axis separation of the raw boxes <= gap
    const double sep = fmax(0.0, fmax(q.rlo[k] - (double)nd.rhi[k], (double)nd.rlo[k] - q.rhi[k]));
    if (sep > q.gap) return false;
    d2 += sep * sep;
    const double dc = fmax(fabs(q.c[k] - (double)nd.clo[k]), fabs(q.c[k] - (double)nd.chi[k]));
    c2 += dc * dc;
  }
  if (q.near_r > 0.0 && d2 > q.near_r * q.near_r) return false;
  if (!q.rel) return true;
  const double U = fmax(q.m, (double)nd.m + sqrt(c2));
  const double D = sqrt(d2);
  if (0.9 * D * (1.0 - 1e-9) > 4.0 * U * (1.0 + 1e-9)) return false;
  // alpha prune: every pair below has alpha_pair >= 0.9 D / speed >= 0.9 D / (4 U),
  // so when that bound reaches the subdomain bounds of both sides (upper
  // bounds of their final alpha_d) no pair below can lower any minimum
  if (q.amax <= 1.0) {
    const double lb = (0.9 * D * (1.0 - 1e-9)) / (4.0 * U * (1.0 + 1e-9));
    if (lb >= fmax(q.amax, (double)nd.amax)) return false;
  }
  return true;
}

// Pair emission from divergent traversals: each thread buffers its pairs
// (BVH_BUF) and flushes a full buffer alone (one atomic per BVH_BUF pairs);
// after the traversal loop the converged warp flushes the remainders with
// one atomic per warp.  (One atomic per pair on the shared list counter
// serialises at ~1 ns each: 9 of the 10 ms of a C5 points pass.)
#define BVH_BUF 16
#define BVH_BUDGET 64          // node expansions per thread per round
#define BVH_TASKS0 (1 << 20)   // initial task-list capacity per list
#define BVH_TASKS_MAX (1ll << 27)  // largest task list grown on demand (1 GiB each, 4 lists)
// MP_BP_TRACE: [0] inner-node expansions, [1] leaf expansions, [2] objects tested, [3] queries
__device__ unsigned long long g_bvh_stats[4];
struct BvhOut {
  int2 buf[BVH_BUF];
  int n = 0;
  double amin = 1.0;              // list-free mode: this thread's smallest alpha_pair
  unsigned long long npairs = 0;  // list-free mode: pairs worked
};

__device__ __forceinline__ bool bvh_reserve(int k, int& base, const PairArgs& A) {
  const int lim = g_append_limit;
  base = atomicAdd(A.app_cnt, k);
  if (base < 0 || base > lim - k) {
    atomicExch(A.app_cnt + (A.app_ee ? 1 : 2), 1);
    return false;
  }
  return true;
}

__device__ __forceinline__ void bvh_write(int base, int k, const int2* buf, const PairArgs& A) {
  for (int r = 0; r < k; ++r)
    if ((int64_t)base + r < A.app_cap) {
      A.app_a[base + r] = buf[r].x;
      A.app_b[base + r] = buf[r].y;
    }
}

__device__ __forceinline__ void bvh_emit(BvhOut& o, int a, int b, const PairArgs& A) {
  o.buf[o.n++] = make_int2(a, b);
  if (o.n == BVH_BUF) {
    int base;
    if (bvh_reserve(BVH_BUF, base, A)) bvh_write(base, BVH_BUF, o.buf, A);
    o.n = 0;
  }
}

// One passing pair: appended to the list (FM < 0), or worked at once by this
// thread (FM = BP_CCD / BP_CERT, the list-free mode for calls past the 2^30
// list limit): pair_work's per-pair steps without its warp collectives --
// the alpha_d minima are order-free atomics, the global minimum and the pair
// count are reduced per thread and flushed once per warp at the end.
template <int FM>
__device__ __forceinline__ void bvh_take(BvhOut& o, bool is_pt, int a, int b, const PairArgs& A) {
  if (FM < 0) {
    bvh_emit(o, a, b, A);
    return;
  }
  ++o.npairs;
  int vid[4];
  if (is_pt) {
    vid[0] = a; vid[1] = A.tri[3 * b]; vid[2] = A.tri[3 * b + 1]; vid[3] = A.tri[3 * b + 2];
  } else {
    vid[0] = A.edge[2 * a]; vid[1] = A.edge[2 * a + 1]; vid[2] = A.edge[2 * b]; vid[3] = A.edge[2 * b + 1];
  }
  if (FM == BP_CCD) {
    bool cert_p = true;
    const double al = ccd_pair_alpha(A.x, A.CC.p, vid, is_pt, A.CC.alpha_l, &cert_p);
    if (al < 1.0)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double* ad = &A.O.alpha_d[vid[r] / A.CC.bs];
        if (al < *(volatile double*)ad) atomic_min_nonneg(ad, al);
      }
    o.amin = fmin(o.amin, al);
    if (!cert_p) A.O.counter[1] = 1;
  } else if (FM == BP_CERT) {
    if (!ccd_certify_pair(A.x, A.CC.p, A.O.alpha_d, A.CC.bs, vid, is_pt)) A.O.counter[1] = 1;
  }
}

// all 32 lanes, converged: the list-free mode's warp minimum and pair count
template <int FM>
__device__ __forceinline__ void bvh_finish_warp(BvhOut& o, const PairArgs& A);

// all 32 lanes, converged
__device__ __forceinline__ void bvh_flush_warp(BvhOut& o, const PairArgs& A) {
  const int lane = threadIdx.x & 31;
  int incl = o.n;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;
  int base = 0;
  bool ok = true;
  if (lane == 31) ok = bvh_reserve(total, base, A);
  base = __shfl_sync(0xffffffffu, base, 31);
  ok = __shfl_sync(0xffffffffu, ok, 31);
  if (ok) bvh_write(base + incl - o.n, o.n, o.buf, A);
}

// Load balance: a thread stops after `budget` node expansions and hands its
// remaining stack to the next round as (query, entry) tasks, so a few
// queries meeting thousands of nodes (a fast vertex among slow neighbours)
// are spread over many threads instead of one thread finishing last.
struct BvhTasks {
  const int2* in;    // this round's (query, stack entry) tasks, or null: one root task per query
  const unsigned long long* n_in;
  int64_t in_cap;    // capacity of `in` (its count may exceed it after an overflow)
  int2* out;         // entries handed to the next round
  unsigned long long* n_out;  // [0] count (64-bit: requests can pass 2^31), [1] overflow flag
  int64_t cap;
  int budget;
  bool abandon;      // on a full list: stop (the host grows the lists and reruns) or finish the traversal here
  int64_t q_base;    // root round: queries [q_base, n) (the kernel's V / E argument is the chunk's end)
};

// Hands the stack on; false when the task list is full: the thread then
// abandons (the host grows the lists to the requested total and reruns the
// enumeration from scratch -- minima and flags are idempotent) or, with a
// fixed capacity, finishes its traversal itself.  The slots a failed
// reservation still got below the capacity are marked (query -1) and
// skipped by the next round.
__device__ __forceinline__ bool bvh_dump(const BvhTasks& K, int query, const int* stack, int sp) {
  const unsigned long long base = atomicAdd(K.n_out, (unsigned long long)sp);
  if (base + sp > (unsigned long long)K.cap) {
    atomicExch(K.n_out + 1, 1ull);
    for (int r = 0; r < sp; ++r)
      if (base + r < (unsigned long long)K.cap) K.out[base + r] = make_int2(-1, 0);
    return false;
  }
  for (int r = 0; r < sp; ++r) K.out[base + r] = make_int2(query, stack[r]);
  return true;
}

template <int FM>
__device__ __forceinline__ void bvh_finish_warp(BvhOut& o, const PairArgs& A) {
  if (FM < 0) {
    bvh_flush_warp(o, A);
    return;
  }
  const int lane = threadIdx.x & 31;
  unsigned long long n = o.npairs;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) n += __shfl_down_sync(0xffffffffu, n, d);
  if (lane == 0 && n) atomicAdd(A.n_pairs, n);
  if (FM == BP_CCD) {
    const double wm = warp_min_all(o.amin);
    if (lane == 0 && wm < *(volatile double*)A.O.min_alpha) atomic_min_nonneg(A.O.min_alpha, wm);
  }
}

// Points query the triangle tree (PT pairs (v, t)); the leaf predicate is
// k_hq_points' (boxes_meet, pt_ref_pass, rel_safe).
template <int FM>
__global__ void __launch_bounds__(128) k_bvh_points(BpTables T, BvhTree TT, int64_t V, const int* __restrict__ sverts,
                                                    const int* __restrict__ tri, const double* __restrict__ x,
                                                    double gap, PairArgs A, BvhTasks K, bool stats,
                                                    const double* __restrict__ abound, double near_r) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = K.in ? min((int64_t)*K.n_in, K.in_cap) : V - K.q_base;
  if (blockIdx.x * (int64_t)blockDim.x >= nt || TT.n == 0) return;  // block-uniform
  BvhOut out;
  int2 task = K.in ? K.in[t0 < nt ? t0 : nt - 1]
                   : make_int2((int)(K.q_base + (t0 < nt ? t0 : nt - 1)), ((TT.nlev - 1) << 26) | 0);
  const bool live = t0 < nt && task.x >= 0;
  if (task.x < 0) task.x = 0;
  const int64_t q = task.x;
  const int v = sverts[q];
  const int64_t oq = T.P + q;
  BvhQuery Q;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    Q.elo[k] = T.elo[3 * oq + k];
    Q.ehi[k] = T.ehi[3 * oq + k];
    Q.rlo[k] = Q.rhi[k] = x[3 * (int64_t)v + k];
    Q.c[k] = T.objmot ? T.objmot[4 * oq + k] : 0.0;
  }
  Q.m = T.objmot ? T.objmot[4 * oq + 3] : 0.0;
  Q.rel = T.objmot != nullptr;
  Q.gap = gap;
  Q.amax = abound ? abound[v / A.CC.bs] : 2.0;
  Q.near_r = near_r;
  int stack[BVH_STACK];
  int sp = 0;
  if (live) stack[sp++] = task.y;
  unsigned n_in = 0, n_leaf = 0;
  int budget = K.budget;
  while (sp > 0) {
    if ((int)(n_in + n_leaf) >= budget) {
      if (bvh_dump(K, (int)q, stack, sp) || K.abandon) break;
      budget = INT_MAX;  // the list is full and fixed (test knob): finish here
    }
    const int e = stack[--sp];
    const int L = e >> 26;
    const int64_t k = e & ((1 << 26) - 1);
    if (L == 0) {
      ++n_leaf;
      const int64_t s1 = min((int64_t)(k + 1) * BVH_W, TT.n);
      for (int64_t s = k * BVH_W; s < s1; ++s) {
        const int t = TT.order[s];
        const double* tl = T.elo + 3 * (int64_t)t;
        const double* th = T.ehi + 3 * (int64_t)t;
        if (boxes_meet(Q.elo, Q.ehi, tl, th) && pt_ref_pass(T, tri, x, v, q, t) &&
            !rel_safe(T, oq, t, Q.rlo, Q.rhi, T.rlo + 3 * (int64_t)t, T.rhi + 3 * (int64_t)t) &&
            (near_r <= 0.0 || box_gap2(Q.rlo, Q.rhi, T.rlo + 3 * (int64_t)t, T.rhi + 3 * (int64_t)t) <= near_r * near_r))
          bvh_take<FM>(out, true, v, t, A);
      }
    } else {
      ++n_in;
      const int64_t c0 = k * BVH_W, c1 = min(c0 + BVH_W, TT.cnt[L - 1]);
      const BvhNode* base = TT.node + TT.off[L - 1];
      for (int64_t j = c1 - 1; j >= c0; --j)
        if (bvh_visit(Q, base[j])) stack[sp++] = ((L - 1) << 26) | (int)j;
    }
  }
  if (stats) {
    atomicAdd(&g_bvh_stats[0], (unsigned long long)n_in);
    atomicAdd(&g_bvh_stats[1], (unsigned long long)n_leaf);
    atomicAdd(&g_bvh_stats[3], 1ull);
  }
  __syncwarp();
  bvh_finish_warp<FM>(out, A);
}

// Edges query the edge tree at sorted positions above their own (each
// unordered pair once); the leaf predicate is k_hq_edges'.
template <int FM>
__global__ void __launch_bounds__(128) k_bvh_edges(BpTables T, BvhTree TE, int64_t E, const int* __restrict__ edge,
                                                   double gap, PairArgs A, BvhTasks K, bool stats,
                                                   const double* __restrict__ abound, double near_r) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = K.in ? min((int64_t)*K.n_in, K.in_cap) : E - K.q_base;
  if (blockIdx.x * (int64_t)blockDim.x >= nt) return;  // block-uniform
  BvhOut out;
  int2 task = K.in ? K.in[t0 < nt ? t0 : nt - 1]
                   : make_int2((int)(K.q_base + (t0 < nt ? t0 : nt - 1)), ((TE.nlev - 1) << 26) | 0);
  const bool live = t0 < nt && task.x >= 0;
  if (task.x < 0) task.x = 0;
  const int64_t si = task.x;
  const int i = TE.order[si];
  const int64_t oi = T.F + i;
  BvhQuery Q;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    Q.elo[k] = T.elo[3 * oi + k];
    Q.ehi[k] = T.ehi[3 * oi + k];
    Q.rlo[k] = T.rlo[3 * oi + k];
    Q.rhi[k] = T.rhi[3 * oi + k];
    Q.c[k] = T.objmot ? T.objmot[4 * oi + k] : 0.0;
  }
  Q.m = T.objmot ? T.objmot[4 * oi + 3] : 0.0;
  Q.rel = T.objmot != nullptr;
  Q.gap = gap;
  Q.amax = abound ? fmax(abound[edge[2 * i] / A.CC.bs], abound[edge[2 * i + 1] / A.CC.bs]) : 2.0;
  Q.near_r = near_r;
  const double* fli = T.flo + 3 * oi;
  const double* fhi = T.fhi + 3 * oi;
  const int ia = edge[2 * i], ib = edge[2 * i + 1];
  int stack[BVH_STACK];
  int sp = 0;
  if (live) stack[sp++] = task.y;
  unsigned n_in = 0, n_leaf = 0;
  int budget = K.budget;
  while (sp > 0) {
    if ((int)(n_in + n_leaf) >= budget) {
      if (bvh_dump(K, (int)si, stack, sp) || K.abandon) break;
      budget = INT_MAX;  // the list is full and fixed (test knob): finish here
    }
    const int e = stack[--sp];
    const int L = e >> 26;
    const int64_t k = e & ((1 << 26) - 1);
    if (L == 0) {
      ++n_leaf;
      const int64_t s1 = min((int64_t)(k + 1) * BVH_W, TE.n);
      for (int64_t s = max(k * BVH_W, si + 1); s < s1; ++s) {
        const int j = TE.order[s];
        const int64_t oj = T.F + j;
        if (!boxes_meet(Q.elo, Q.ehi, T.elo + 3 * oj, T.ehi + 3 * oj)) continue;
        const int ja = edge[2 * j], jb = edge[2 * j + 1];
        const double* flj = T.flo + 3 * oj;
        const double* fhj = T.fhi + 3 * oj;
        const bool pass = !(ia == ja || ia == jb || ib == ja || ib == jb) && body_pass(T, ia, ja) &&
                          fli[0] <= fhj[0] && fli[1] <= fhj[1] && fli[2] <= fhj[2] && flj[0] <= fhi[0] &&
                          flj[1] <= fhi[1] && flj[2] <= fhi[2] && ref_reach(T.rc, oi, oj) &&
                          !rel_safe(T, oi, oj, Q.rlo, Q.rhi, T.rlo + 3 * oj, T.rhi + 3 * oj) &&
                          (near_r <= 0.0 || box_gap2(Q.rlo, Q.rhi, T.rlo + 3 * oj, T.rhi + 3 * oj) <= near_r * near_r);
        if (pass) bvh_take<FM>(out, false, min(i, j), max(i, j), A);
      }
    } else {
      ++n_in;
      const int64_t c0 = k * BVH_W, c1 = min(c0 + BVH_W, TE.cnt[L - 1]);
      // a child whose last sorted position is <= si holds no partner
      int64_t per = BVH_W;  // objects per level-(L-1) node: 8^L
      for (int l = 1; l < L; ++l) per *= BVH_W;
      const BvhNode* base = TE.node + TE.off[L - 1];
      for (int64_t j = c1 - 1; j >= c0; --j) {
        if ((j + 1) * per - 1 <= si) break;
        if (bvh_visit(Q, base[j])) stack[sp++] = ((L - 1) << 26) | (int)j;
      }
    }
  }
  if (stats) {
    atomicAdd(&g_bvh_stats[0], (unsigned long long)n_in);
    atomicAdd(&g_bvh_stats[1], (unsigned long long)n_leaf);
    atomicAdd(&g_bvh_stats[3], 1ull);
  }
  __syncwarp();
  bvh_finish_warp<FM>(out, A);
}

// the class trees: order fixed at first use (by smallest vertex id -- the
// vertex ids are Morton-renumbered), boxes refit every call
__global__ void k_min_vertex_key(int64_t n, int per, const int* __restrict__ ids, int* __restrict__ key,
                                 int* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int k = ids[per * i];
  for (int a = 1; a < per; ++a) k = min(k, ids[per * i + a]);
  key[i] = k;
  val[i] = (int)i;
}

static void bvh_shape(BvhTree& T, int64_t n) {
  T.n = n;
  int64_t m = (n + BVH_W - 1) / BVH_W, off = 0;
  T.nlev = 0;
  for (;;) {
    if (T.nlev >= BVH_MAX_LEVELS) throw MpError(MP_ERR_CAPACITY, "bvh depth");
    T.off[T.nlev] = off;
    T.cnt[T.nlev] = m;
    off += m;
    ++T.nlev;
    if (m <= 1) break;
    m = (m + BVH_W - 1) / BVH_W;
  }
  T.off[T.nlev] = off;
}

static void bvh_trace_stats(bool on, const char* what, const BvhTree& T) {
  if (!on) return;
  unsigned long long h[4];
  CUDA_CHECK(cudaMemcpyFromSymbol(h, g_bvh_stats, sizeof(h)));
  fprintf(stderr, "  bvh %s: levels %d, per query %.1f inner / %.1f leaf expansions (%llu queries)\n", what, T.nlev,
          (double)h[0] / fmax(1.0, (double)h[3]), (double)h[1] / fmax(1.0, (double)h[3]), h[3]);
  const unsigned long long z[4] = {0, 0, 0, 0};
  CUDA_CHECK(cudaMemcpyToSymbol(g_bvh_stats, z, sizeof(z)));
}

// Tight CCD / certificate enumeration through the class trees: the same
// reference pair list as run_bp's one-pass append (bp.cuh), then the mode's
// pair kernel; past the 2^30 list limit the traversal reruns list-free, the
// pairs worked where they are found (64-bit count).  Returns the pair count.
template <int MODE>
static int64_t run_bvh(mp_ctx* c, const double* x, const BpGrid& B, BpOut O, ContactParams CP, CcdParams CC,
                       int* flag) {
  const int64_t V = c->V, F = c->F, E = c->E;
  cudaStream_t st = c->stream;
  auto& g = c->grid;
  BvhTree TT{}, TE{};
  bvh_shape(TT, F);
  bvh_shape(TE, E);
  if (!c->bvh_ready) {  // fixed object order, by smallest (Morton-renumbered) vertex id
    c->bvh_tri_order.ensure(F + 1);
    c->bvh_edge_order.ensure(E + 1);
    const int64_t nmax = std::max(F, E) + 1;
    c->bvh_key.ensure(2 * nmax);
    c->bvh_val.ensure(nmax);
    const int bits = bits_for((unsigned long long)std::max<int64_t>(1, c->N));
    if (F) {
      k_min_vertex_key<<<grid_for(F, 256), 256, 0, st>>>(F, 3, c->tri, c->bvh_key, c->bvh_val);
      LAUNCH_CHECK();
      sort_pairs_i32(c, c->bvh_key, c->bvh_key.p + nmax, c->bvh_val, c->bvh_tri_order, F, bits);
    }
    if (E) {
      k_min_vertex_key<<<grid_for(E, 256), 256, 0, st>>>(E, 2, c->edge, c->bvh_key, c->bvh_val);
      LAUNCH_CHECK();
      sort_pairs_i32(c, c->bvh_key, c->bvh_key.p + nmax, c->bvh_val, c->bvh_edge_order, E, bits);
    }
    c->bvh_ready = true;
  }
  c->bvh_tri_nodes.ensure(5 * (size_t)(TT.off[TT.nlev] + 1));
  c->bvh_edge_nodes.ensure(5 * (size_t)(TE.off[TE.nlev] + 1));
  BvhNode* nt = reinterpret_cast<BvhNode*>(c->bvh_tri_nodes.p);
  BvhNode* ne = reinterpret_cast<BvhNode*>(c->bvh_edge_nodes.p);
  TT.node = nt; TT.order = c->bvh_tri_order;
  TE.node = ne; TE.order = c->bvh_edge_order;
  const BpTables& T = B.T;
  auto refit = [&](BvhTree& R, BvhNode* nodes, int64_t base, const double* alpha) {
    if (R.n == 0) return;
    const bool tri_tree = base == 0;
    k_bvh_leaves<<<grid_for(R.n, 256), 256, 0, st>>>(R.n, base, R.order, T.rlo, T.rhi, T.elo, T.ehi, T.objmot,
                                                      nodes, tri_tree ? c->tri : c->edge, tri_tree ? 3 : 2, alpha,
                                                      c->bs);
    LAUNCH_CHECK();
    for (int l = 1; l < R.nlev; ++l) {
      k_bvh_up<<<grid_for(R.cnt[l - 1], 256), 256, 0, st>>>(R.cnt[l - 1], nodes + R.off[l - 1], nodes + R.off[l]);
      LAUNCH_CHECK();
    }
  };
  BpTrace tr(st);
  refit(TT, nt, 0, nullptr);
  refit(TE, ne, F, nullptr);
  tr.lap("refit");
  // task lists: [class][ping-pong]; counters: per class and buffer (count, overflow)
  const size_t want = 4 * (size_t)(c->bvh_task_cap > 0 ? c->bvh_task_cap : BVH_TASKS0);
  if (c->bvh_tasks.n < want) c->bvh_tasks.ensure(want);
  c->bvh_task_cnt.ensure(8);
  const bool fixed_cap = c->bvh_task_cap > 0;
  if (c->bvh_task_max <= 0) c->bvh_task_max = BVH_TASKS_MAX;  // test knob: overflowing threads finish their traversals
  bool list_free = false;  // set when the one-pass list would pass 2^30 pairs
  const double* abound_cur = nullptr;  // the alpha prune's subdomain bounds (list-free CCD, phase 1)
  double near_cur = 0.0;               // the near pass's separation limit (list-free CCD, phase 0)
  for (int attempt = 0; attempt < 6; ++attempt) {
    CUDA_CHECK(cudaMemsetAsync(c->counters.p, 0, 3 * sizeof(int), st));
    c->n_pairs_dev.ensure(1);
    CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, sizeof(unsigned long long), st));
    O.counter = c->counters.p;
    if (g.pa.n < 1024) { g.pa.ensure(1 << 16); g.pb.ensure(1 << 16); }
    if (g.ea.n < 1024) { g.ea.ensure(1 << 16); g.eb.ensure(1 << 16); }
    int* cnt = c->counters.p + 8;  // [8] PT, [9] EE appended, [10] overflow flag
    CUDA_CHECK(cudaMemsetAsync(cnt, 0, 3 * sizeof(int), st));
    const int64_t cap_pt = (int64_t)std::min(g.pa.n, g.pb.n), cap_ee = (int64_t)std::min(g.ea.n, g.eb.n);
    unsigned long long* tcnt = c->bvh_task_cnt.p;  // [2 * (2 * class + buffer)] count, [+1] overflow
    if (!B.empty) {
      PairArgs A{c->tri, c->tri_sorted, c->edge, x, O, CP, CC, c->n_pairs_dev.p, g.pa, g.pb, cnt, cap_pt};
      PairArgs Ae = A;
      Ae.app_a = g.ea; Ae.app_b = g.eb; Ae.app_cnt = cnt + 1; Ae.app_cap = cap_ee; Ae.app_ee = 1;
      // The rounds of one class over the queries [q0, q1); false when a round
      // overflowed the task lists (*need = the entries it requested): the
      // threads abandoned work and the caller rolls the chunk back.
      // (finish_here: a single query still overflowing at the largest lists
      // finishes its traversal in its own threads -- guaranteed progress)
      auto traverse = [&](int cls, int64_t q0, int64_t q1, int64_t* need, bool finish_here) -> bool {
        const bool keep = fixed_cap || finish_here;
        const int64_t tcap = fixed_cap ? c->bvh_task_cap
                                       : std::min<int64_t>((int64_t)(c->bvh_tasks.n / 4), c->bvh_task_max);
        int2* tb[2];
        for (int b = 0; b < 2; ++b) tb[b] = reinterpret_cast<int2*>(c->bvh_tasks.p) + (2 * cls + b) * tcap;
        unsigned long long* tc = tcnt + 4 * cls;
        int64_t n_task = q1 - q0;
        for (int round = 0; n_task; ++round) {
          const int cur = round & 1, nxt = cur ^ 1;
          CUDA_CHECK(cudaMemsetAsync(tc + 2 * nxt, 0, 2 * sizeof(unsigned long long), st));
          BvhTasks K{round ? tb[cur] : nullptr, tc + 2 * cur, tcap, tb[nxt], tc + 2 * nxt, tcap, BVH_BUDGET, !keep,
                     q0};
          if (cls == 0) {
            if (list_free)
              k_bvh_points<MODE><<<grid_for(n_task, 128), 128, 0, st>>>(T, TT, q1, c->sverts, c->tri, x,
                                                                        B.filter_gap, A, K, tr.on, abound_cur,
                                                                        near_cur);
            else
              k_bvh_points<-1><<<grid_for(n_task, 128), 128, 0, st>>>(T, TT, q1, c->sverts, c->tri, x,
                                                                      B.filter_gap, A, K, tr.on, nullptr, 0.0);
            LAUNCH_CHECK();
            tr.lap("points");
            bvh_trace_stats(tr.on, "points", TT);
          } else {
            if (list_free)
              k_bvh_edges<MODE><<<grid_for(n_task, 128), 128, 0, st>>>(T, TE, q1, c->edge, B.filter_gap, Ae, K,
                                                                       tr.on, abound_cur, near_cur);
            else
              k_bvh_edges<-1><<<grid_for(n_task, 128), 128, 0, st>>>(T, TE, q1, c->edge, B.filter_gap, Ae, K,
                                                                     tr.on, nullptr, 0.0);
            LAUNCH_CHECK();
            tr.lap("edges");
            bvh_trace_stats(tr.on, "edges", TE);
          }
          unsigned long long hh[2];
          CUDA_CHECK(cudaMemcpyAsync(hh, tc + 2 * nxt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
          sync_stream(c);
          const int64_t req = (int64_t)std::min<unsigned long long>(hh[0], 1ull << 62);
          if (hh[1] && !keep) {
            *need = req;
            return false;
          }
          n_task = std::min<int64_t>(req, tcap);
          if (tr.on && n_task)
            fprintf(stderr, "  bvh %s round %d hands on %lld tasks\n", cls ? "edges" : "points", round + 1,
                    (long long)n_task);
        }
        return true;
      };
      // List-free CCD (> 2^30 pairs: a direction huge against the gaps, the
      // reference set nearly every pair): an exact alpha prune.  Phase 0
      // works the pairs within a few mean primitive extents -- a subset, so
      // the alpha_d it leaves are upper bounds of the final ones; the trees
      // are refit with those bounds and phase 1 skips every node whose
      // pairs provably have alpha_pair >= the bounds of all their
      // subdomains (bvh_visit).  The returned count is phase 1's pairs.
      const bool prune = list_free && MODE == BP_CCD && T.objmot && O.alpha_d;
      for (int phase = prune ? 0 : 1; phase < 2; ++phase) {
      near_cur = phase == 0 ? 4.0 * B.raw_mean : 0.0;
      abound_cur = (phase == 1 && prune) ? O.alpha_d : nullptr;
      if (phase == 1 && prune) {
        CUDA_CHECK(cudaMemsetAsync(c->n_pairs_dev.p, 0, sizeof(unsigned long long), st));
        refit(TT, nt, 0, O.alpha_d);
        refit(TE, ne, F, O.alpha_d);
      }
      // each class in query chunks: a chunk whose rounds overflow is rolled
      // back (its appended pairs / list-free count dropped; minima and flags
      // are idempotent) and rerun with lists of the requested size, or --
      // past BVH_TASKS_MAX -- split in four
      for (int cls = 0; cls < 2; ++cls) {
        const int64_t nq = cls == 0 ? ((V && F) ? V : 0) : (E > 1 ? E : 0);
        int64_t q0 = 0, chunk = nq;
        while (q0 < nq) {
          const int64_t q1 = std::min(nq, q0 + chunk);
          int app0 = 0;
          unsigned long long np0 = 0;
          if (q0 > 0) {  // the chunk's starting counts (zero for a class's first chunk)
            CUDA_CHECK(cudaMemcpyAsync(&app0, cnt + cls, sizeof(int), cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaMemcpyAsync(&np0, c->n_pairs_dev.p, sizeof(np0), cudaMemcpyDeviceToHost, st));
            sync_stream(c);
          } else if (cls == 1) {
            CUDA_CHECK(cudaMemcpyAsync(&np0, c->n_pairs_dev.p, sizeof(np0), cudaMemcpyDeviceToHost, st));
            sync_stream(c);
          }
          int64_t need = 0;
          const bool at_max = (int64_t)(c->bvh_tasks.n / 4) >= c->bvh_task_max;
          if (traverse(cls, q0, q1, &need, at_max && q1 - q0 == 1)) {
            q0 = q1;
            continue;
          }
          CUDA_CHECK(cudaMemcpyAsync(cnt + cls, &app0, sizeof(int), cudaMemcpyHostToDevice, st));
          CUDA_CHECK(cudaMemcpyAsync(c->n_pairs_dev.p, &np0, sizeof(np0), cudaMemcpyHostToDevice, st));
          sync_stream(c);
          const int64_t want_n = need + need / 4 + 1024;
          if (want_n <= c->bvh_task_max && (int64_t)(c->bvh_tasks.n / 4) < want_n) {
            c->bvh_tasks.ensure(4 * (size_t)want_n);
          } else {
            if ((int64_t)(c->bvh_tasks.n / 4) < c->bvh_task_max) c->bvh_tasks.ensure(4 * (size_t)c->bvh_task_max);
            chunk = std::max<int64_t>(1, (q1 - q0) / 4);
          }
          if (tr.on)
            fprintf(stderr, "  bvh %s chunk [%lld, %lld) overflowed (%lld tasks): retry with %lld per list, chunk %lld\n",
                    cls ? "edges" : "points", (long long)q0, (long long)q1, (long long)need,
                    (long long)(c->bvh_tasks.n / 4), (long long)chunk);
        }
      }
      }  // phases
      if (!list_free) {
        k_pairs_app<MODE><<<8 * 148, 256, 0, st>>>(cnt, cap_pt, cap_ee, g.pa, g.pb, g.ea, g.eb, A);
        LAUNCH_CHECK();
        tr.lap("pairs");
      }
    }
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt, c->counters.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaMemcpyAsync(c->h_cnt + 5, cnt, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
    if (c->rb_extra)  // the caller's scalar rides on this readback (h_scal[0])
      CUDA_CHECK(cudaMemcpyAsync(c->h_scal, c->rb_extra, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (list_free)
      CUDA_CHECK(cudaMemcpyAsync(c->h_npairs, c->n_pairs_dev.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 st));
    sync_stream(c);
    if (list_free) {
      if (flag) *flag = c->h_cnt[1];
      return (int64_t)*c->h_npairs;
    }
    if (c->h_cnt[7]) {  // >= 2^30 pairs: rerun list-free (minima / flags are idempotent)
      list_free = true;
      continue;
    }
    const int64_t n_pt = c->h_cnt[5], n_ee = c->h_cnt[6];
    if (n_pt > cap_pt || n_ee > cap_ee) {  // grow and rerun (minima / flags are idempotent)
      if (n_pt > cap_pt) { g.pa.ensure((size_t)(n_pt * 1.25) + 1024); g.pb.ensure((size_t)(n_pt * 1.25) + 1024); }
      if (n_ee > cap_ee) { g.ea.ensure((size_t)(n_ee * 1.25) + 1024); g.eb.ensure((size_t)(n_ee * 1.25) + 1024); }
      continue;
    }
    if (flag) *flag = c->h_cnt[1];
    return n_pt + n_ee;
  }
  throw MpError(MP_ERR_CAPACITY, "bvh pair list capacity retry failed");
}
