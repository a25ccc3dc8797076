// contact.cuh -- constraint set, contact terms, classification, per-subdomain
// Top-K.  The broad phase under the constraint set lives in bp.cuh.
#pragma once

#include "bp.cuh"

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

// ---------------------------------------------------------------------------
// vertex -> incidence CSR of a 4-vertex row table (deterministic scatter)

__global__ void k_inc_keys(int64_t n, const int4* __restrict__ verts, int* __restrict__ cnt, int* __restrict__ key,
                           int* __restrict__ val) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= 4 * n) return;
  const int4 v = verts[e >> 2];
  const int a = (int)(e & 3);
  const int id = a == 0 ? v.x : (a == 1 ? v.y : (a == 2 ? v.z : v.w));
  key[e] = id;
  val[e] = (int)e;
  atomicAdd(&cnt[id], 1);  // integer counts: order-free
}

// I.off = per-vertex offsets, I.val2 = incidences 4i+a grouped by vertex,
// ascending within a vertex (stable radix sort of ascending input)
static void build_inc(mp_ctx* c, IncCSR& I, const int4* verts, int64_t n) {
  const int64_t N = c->N;
  I.cnt.ensure(N + 1);
  I.off.ensure(N + 1);
  CUDA_CHECK(cudaMemsetAsync(I.cnt.p, 0, sizeof(int) * (N + 1), c->stream));
  if (n > 0) {
    const size_t m = 4 * (size_t)n;
    I.key.ensure(m); I.key2.ensure(m); I.val.ensure(m); I.val2.ensure(m);
    k_inc_keys<<<grid_for((int64_t)m, 256), 256, 0, c->stream>>>(n, verts, I.cnt, I.key, I.val);
    LAUNCH_CHECK();
    sort_pairs_i32(c, I.key, I.key2, I.val, I.val2, (int64_t)m, c->id_bits);
  }
  exclusive_scan(c, I.cnt, I.off, N + 1);
}

// per-row contact gradient terms kappa b'(d) grad (pinned rows are zero)
__global__ void k_contact_grad_rows(int64_t n, const double* __restrict__ d, const double* __restrict__ grad,
                                    double dh, double kappa, double* __restrict__ cbuf) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double db;
  barrier3(d[i], dh, kappa, nullptr, &db, nullptr);
#pragma unroll
  for (int q = 0; q < 12; ++q) cbuf[12 * i + q] = db * grad[12 * i + q];
}

// per-row rank-one terms s_i w_i (w_i . vec); s == nullptr -> 1
__global__ void k_rank1_rows(int64_t n, const int4* __restrict__ verts, const double* __restrict__ w,
                             const double* __restrict__ s, const double* __restrict__ vec, double* __restrict__ rbuf) {
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
#pragma unroll
  for (int q = 0; q < 12; ++q) rbuf[12 * i + q] = w[12 * i + q] * dot;
}

// out[v] += (sum over A's incidences) + (sum over B's): one warp per vertex,
// fixed-order gathers; pinned vertices' rows are zero in every table
__global__ void k_inc_gather_add(int64_t N, const unsigned char* __restrict__ pinned,
                                 const int* __restrict__ a_off, const int* __restrict__ a_val,
                                 const double* __restrict__ a_buf, const int* __restrict__ b_off,
                                 const int* __restrict__ b_val, const double* __restrict__ b_buf,
                                 double* __restrict__ out, int64_t v0) {
  const int64_t v = v0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);  // rows [v0, N)
  const int lane = threadIdx.x & 31;
  if (v >= N || pinned[v]) return;  // warp-uniform
  const bool ha = a_off && a_off[v + 1] > a_off[v], hb = b_off && b_off[v + 1] > b_off[v];
  if (!ha && !hb) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
  if (ha) warp_gather3(a_off[v], a_off[v + 1], a_val, a_buf, a0, a1, a2);
  if (hb) warp_gather3(b_off[v], b_off[v + 1], b_val, b_buf, b0, b1, b2);
  if (lane) return;
  out[3 * v] = (out[3 * v] + a0) + b0;
  out[3 * v + 1] = (out[3 * v + 1] + a1) + b1;
  out[3 * v + 2] = (out[3 * v + 2] + a2) + b2;
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
  c->inc_cur_rows = -1;
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
      build_inc(c, c->inc_cur, c->cur.verts, n);
      c->inc_cur_rows = n;
      return;
    }
    c->scratch.ensure((size_t)(n * 1.5) + 1024);
  }
  throw MpError(MP_ERR_CAPACITY, "constraint set capacity retry failed");
}

// ---------------------------------------------------------------------------
// contact terms of gradient / energy / HVP

__global__ void k_contact_energy(int64_t n, const double* __restrict__ d, double dh, double kappa, double* part) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double b;
    barrier3(d[i], dh, kappa, &b, nullptr, nullptr);
    acc += b;
  }
  block_sum_store<256>(acc, part);
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
  build_inc(c, c->inc_cand, c->cand_verts, tot);
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
