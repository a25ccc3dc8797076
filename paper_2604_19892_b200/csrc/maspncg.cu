// maspncg.cu -- C ABI + the MAS-PNCG outer loop (Alg. 1) on sm_100a.
//
// Single translation unit: the stage headers hold the kernels and their
// launchers; this file owns context creation (partition, renumbering, static
// BSR pattern), the advance_step loop and the exported entry points
// declared in include/maspncg.h.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <functional>
#include <vector>

#include "stages.cuh"
#include "check.cuh"

thread_local int64_t* g_launch_counter = nullptr;

mp_ctx::~mp_ctx() {
  if (grp && rank == 0) {  // the group's shard 0 owns the other shards and the group
    for (size_t q = 1; q < grp->sh.size(); ++q) delete grp->sh[q];
    for (int q = 0; q < GROUP_MAX; ++q) {
      if (grp->ev[q]) cudaEventDestroy(grp->ev[q]);
      if (grp->ev2[q]) cudaEventDestroy(grp->ev2[q]);
    }
    delete grp;
  }
  for (auto* l : levels) delete l;
  if (h_scal) cudaFreeHost(h_scal);
  if (h_cnt) cudaFreeHost(h_cnt);
  for (auto& t : timers) {
    if (t.a) cudaEventDestroy(t.a);
    if (t.b) cudaEventDestroy(t.b);
  }
  if (ev_bsr) cudaEventDestroy(ev_bsr);
  if (ev_g) cudaEventDestroy(ev_g);
  if (ev_l0) cudaEventDestroy(ev_l0);
  if (ev_it) cudaEventDestroy(ev_it);
  if (ev_t0) cudaEventDestroy(ev_t0);
  if (ev_t1) cudaEventDestroy(ev_t1);
  if (ev_bsr_ahead) cudaEventDestroy(ev_bsr_ahead);
  if (side) cudaStreamDestroy(side);
  if (stream) cudaStreamDestroy(stream);
}

// ---------------------------------------------------------------------------
// Morton partition (mas.py:30-77), computed once on the host exactly as the
// reference does (same IEEE expression, stable sort)

static uint64_t part1by2(uint64_t v) {
  v = (v | (v << 32)) & 0x1F00000000FFFFull;
  v = (v | (v << 16)) & 0x1F0000FF0000FFull;
  v = (v | (v << 8)) & 0x100F00F00F00F00Full;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

static void morton_partition(const double* rest, int64_t N, int bs, std::vector<int>& new2old,
                             std::vector<int64_t>& sub_of) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < N; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], rest[3 * i + k]);
      hi[k] = std::max(hi[k], rest[3 * i + k]);
    }
  double ext[3];
  for (int k = 0; k < 3; ++k) {
    ext[k] = hi[k] - lo[k];
    if (ext[k] == 0.0) ext[k] = 1.0;
  }
  std::vector<uint64_t> code(N);
  for (int64_t i = 0; i < N; ++i) {
    uint64_t q[3];
    for (int k = 0; k < 3; ++k) {
      volatile double t = (rest[3 * i + k] - lo[k]) / ext[k];
      volatile double u = t * 1023.0;
      q[k] = (uint64_t)(double)u;
    }
    code[i] = part1by2(q[0]) | (part1by2(q[1]) << 1) | (part1by2(q[2]) << 2);
  }
  std::vector<int> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return code[a] < code[b]; });
  int64_t D = std::max<int64_t>(1, (N + bs - 1) / bs);
  new2old.assign(N, 0);
  sub_of.assign(N, 0);
  for (int64_t d = 0; d < D; ++d) {
    int64_t b = d * bs, e = std::min<int64_t>(N, b + bs);
    std::vector<int> blk(order.begin() + b, order.begin() + e);
    std::sort(blk.begin(), blk.end());
    for (int64_t r = 0; r < (int64_t)blk.size(); ++r) {
      new2old[b + r] = blk[r];
      sub_of[blk[r]] = d;
    }
  }
}

static void validate_config(const mp_solver_config& c) {
  if (!(c.eps > 0)) throw MpError(MP_ERR_CONFIG, "eps must be positive");
  if (!(c.delta > 0 && c.delta < 1)) throw MpError(MP_ERR_CONFIG, "delta must lie in (0, 1)");
  if (c.iter_max < 1) throw MpError(MP_ERR_CONFIG, "iter_max must be >= 1");
  if (c.preconditioner != MP_PRECOND_MAS && c.preconditioner != MP_PRECOND_JACOBI)
    throw MpError(MP_ERR_CONFIG, "unknown preconditioner");
  if (c.direction_rule < MP_DIR_SUBSPACE2D || c.direction_rule > MP_DIR_CD)
    throw MpError(MP_ERR_CONFIG, "unknown direction rule");
  if (c.update_strategy < 0 || c.update_strategy > 2) throw MpError(MP_ERR_CONFIG, "unknown update strategy");
  if (c.block_size < 1 || c.block_size > 32) throw MpError(MP_ERR_CONFIG, "block_size must lie in [1, 32]");
  if (c.K < 0) throw MpError(MP_ERR_CONFIG, "K must be >= 0");
  if (c.coarse_block < 1) throw MpError(MP_ERR_CONFIG, "coarse_block must be >= 1");
}

// coarse level shapes (mas.py:155-169): aggregate coarse_block units of the
// previous level; stop at the first level that does not coarsen
static void setup_levels(mp_ctx* c) {
  for (auto* l : c->levels) delete l;
  c->levels.clear();
  int64_t units = c->D;
  int64_t span = c->bs;
  const int cb = c->cfg.coarse_block;
  for (int l = 0; l < c->cfg.levels && l < 8; ++l) {
    int64_t n_agg = (units + cb - 1) / cb;
    if (n_agg == units) break;
    span *= cb;
    auto* L = new CoarseLevel();
    L->A = (int)n_agg;
    L->n = (int)(3 * n_agg);
    L->span = (int)span;
    // ~4 blocks per SM over (row block, diagonal chunk), >= 4 diagonals each
    int rowblocks = (L->n + 127) / 128;
    int maxch = std::max(1, (L->n / 2 + 1) / 4);
    int ch = std::max(1, std::min(maxch, 4 * 148 / std::max(1, rowblocks)));
    L->chunks = ch;
    L->rsum.ensure(L->n);
    L->r.ensure(L->n);
    L->ypart.ensure((size_t)L->n);
    L->ypc.ensure((size_t)ch * L->n);
    L->mv_cnt.zero((size_t)rowblocks, c->stream);
    // BSR -> M_l gather map (first coarse level only; the next levels sum
    // the previous level's blocks): slots grouped by coarse block (A, B)
    if (c->levels.empty()) {
      const int64_t N = c->N;
      const int nA = L->A;
      std::vector<std::pair<int64_t, int>> ks;
      ks.reserve(c->h_cols.size());
      for (int64_t v = 0; v < N; ++v)
        for (int k = c->h_rowptr[v]; k < c->h_rowptr[v + 1]; ++k)
          ks.emplace_back((v / span) * nA + c->h_cols[k] / span, k);
      std::stable_sort(ks.begin(), ks.end(),
                       [](const std::pair<int64_t, int>& a, const std::pair<int64_t, int>& b) { return a.first < b.first; });
      std::vector<int> key, off, slot(ks.size());
      for (size_t q = 0; q < ks.size(); ++q) {
        if (q == 0 || ks[q].first != ks[q - 1].first) {
          key.push_back((int)ks[q].first);
          off.push_back((int)q);
        }
        slot[q] = ks[q].second;
      }
      off.push_back((int)ks.size());
      L->nblk = (int)key.size();
      if (L->nblk) {
        L->cb_key.upload(key.data(), key.size(), c->stream);
        L->cb_off.upload(off.data(), off.size(), c->stream);
        L->cb_slot.upload(slot.data(), slot.size(), c->stream);
      }
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    // the coarse chain is the build's critical path: its CTAs go ahead of
    // the level-0 sweep's queued CTAs
    int prio_lo = 0, prio_hi = 0;
    CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CUDA_CHECK(cudaStreamCreateWithPriority(&L->st, cudaStreamNonBlocking, prio_hi));
    CUDA_CHECK(cudaStreamCreateWithPriority(&L->st2, cudaStreamNonBlocking, prio_hi));
    CUDA_CHECK(cudaEventCreateWithFlags(&L->done, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&L->ev_w, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&L->ev_u, cudaEventDisableTiming));
    CUDA_CHECK(cudaEventCreateWithFlags(&L->ev_asm, cudaEventDisableTiming));
    {  // coarse-inverse work units: (row tile I, first column tile J0), ch tiles J0.. <= I each;
       // ch: the narrowest that still fits one unit per SM (+ the lookahead CTA)
      const int nT = (L->n + CS_TB - 1) / CS_TB;
      int sms = 148;
      CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      // widest units: the coarse kernel then leaves SMs to the concurrent
      // level-0 sweep (narrower units filling every SM measured slower:
      // 1.08 vs 0.95 ms per MAS build at C2)
      L->cs_ch = CS_CH;
      (void)sms;
      std::vector<int2> units;
      for (int I = 0; I < nT; ++I)
        for (int j0 = 0; j0 <= I; j0 += L->cs_ch) units.push_back(make_int2(I, j0));
      L->n_units = (int)units.size();
      L->cs_units.upload(units.data(), units.size(), c->stream);
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    c->levels.push_back(L);
    units = n_agg;
  }
  c->n_levels = (int)c->levels.size();
  group_ranges(c, c->rank, c->nshards);  // owned ranges and reduction chunks follow the level-1 aggregates
}

static void set_smem_limits() {
  static bool done = false;
  if (done) return;
  int dev = 0, optin = 0;
  CUDA_CHECK(cudaGetDevice(&dev));
  CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  auto allow = [&](const void* fn) {
    cudaFuncAttributes fa{};
    CUDA_CHECK(cudaFuncGetAttributes(&fa, fn));
    int dyn = optin - (int)fa.sharedSizeBytes;
    CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  };
  allow((const void*)k_mas_apply_l0<true, 2>);
  allow((const void*)k_mas_apply_l0<false, 2>);
  allow((const void*)k_mas_apply_l0<true, 3>);
  allow((const void*)k_mas_apply_l0<false, 3>);
  allow((const void*)k_woodbury);
  allow((const void*)k_direct_update);
  allow((const void*)k_coarse_sweep);
  allow((const void*)k_mas_sweep);
  done = true;
}

static void create_ctx(const mp_scene_desc* s, const mp_solver_config* cfg, int device, mp_ctx* c) {
  validate_config(*cfg);
  c->cfg = *cfg;
  c->device = device;
  CUDA_CHECK(cudaSetDevice(device));
  CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_bsr, cudaEventDisableTiming));
  CUDA_CHECK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_g, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_l0, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_it, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreate(&c->ev_t0));
  CUDA_CHECK(cudaEventCreate(&c->ev_t1));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_bsr_ahead, cudaEventDisableTiming));
  set_smem_limits();
  CUDA_CHECK(cudaMallocHost(&c->h_scal, 64 * sizeof(double)));
  CUDA_CHECK(cudaMallocHost(&c->h_cnt, 16 * sizeof(int)));
  c->h_npairs = reinterpret_cast<unsigned long long*>(c->h_scal + 63);
  c->N = s->n_verts;
  c->T = s->n_tets;
  c->F = s->n_tris;
  c->E = s->n_edges;
  c->V = s->n_surf_verts;
  c->d_hat = s->d_hat;
  c->kappa = s->kappa;
  c->bs = cfg->block_size;
  c->m = 3 * c->bs;
  const int64_t N = c->N;
  if (N < 1) throw MpError(MP_ERR_CONFIG, "scene has no vertices");
  if (N >= (1ll << 30)) throw MpError(MP_ERR_CONFIG, "scene too large");
  morton_partition(s->rest, N, c->bs, c->h_new2old, c->h_sub_of_old);
  c->D = std::max<int64_t>(1, (N + c->bs - 1) / c->bs);
  c->h_old2new.assign(N, 0);
  for (int64_t i = 0; i < N; ++i) c->h_old2new[c->h_new2old[i]] = (int)i;
  const auto& o2n = c->h_old2new;
  const auto& n2o = c->h_new2old;
  c->id_bits = bits_for((unsigned long long)(N > 1 ? N - 1 : 1));
  cudaStream_t st = c->stream;
  c->new2old.upload(n2o.data(), N, st);
  {
    std::vector<double> mass(N), fe(3 * N);
    std::vector<unsigned char> pin(N);
    for (int64_t i = 0; i < N; ++i) {
      int o = n2o[i];
      mass[i] = s->mass[o];
      pin[i] = s->dirichlet[o] ? 1 : 0;
      for (int k = 0; k < 3; ++k) fe[3 * i + k] = s->f_ext[3 * o + k];
    }
    c->mass.upload(mass.data(), N, st);
    c->pinned.upload(pin.data(), N, st);
    c->f_ext.upload(fe.data(), 3 * N, st);
  }
  // tets and per-tet constants
  const int64_t T = c->T;
  // tets grouped by material (SNH, then ARAP, then none) so every kernel
  // runs a kind-specialised instantiation over a contiguous range
  std::vector<int64_t> torder(T);
  std::iota(torder.begin(), torder.end(), (int64_t)0);
  auto rank_of = [&](int64_t t) { return s->kind[t] == 2 ? 0 : (s->kind[t] == 1 ? 1 : 2); };
  std::stable_sort(torder.begin(), torder.end(), [&](int64_t a, int64_t b) { return rank_of(a) < rank_of(b); });
  std::vector<int4> tets(T);
  std::vector<TetParam> tp(T);
  std::vector<signed char> kind(T);
  c->T_snh = c->T_arap = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t u = torder[t];
    int id[4];
    for (int a = 0; a < 4; ++a) {
      int64_t o = s->tets[4 * u + a];
      if (o < 0 || o >= N) throw MpError(MP_ERR_CONFIG, "tet index out of range");
      id[a] = o2n[o];
    }
    tets[t] = make_int4(id[0], id[1], id[2], id[3]);
    for (int q = 0; q < 9; ++q) tp[t].Bm[q] = s->Bm[9 * u + q];
    tp[t].vol = s->vol[u];
    tp[t].mu = s->mu[u];
    tp[t].lam = s->lam[u];
    kind[t] = s->kind[u];
    if (kind[t] == 2) ++c->T_snh;
    else if (kind[t] == 1) ++c->T_arap;
  }
  c->tets.upload(tets.data(), T, st);
  c->tetp.upload(tp.data(), T, st);
  c->kind.upload(kind.data(), T, st);
  // static BSR pattern: vertex adjacency through tets (+ diagonal)
  {
    std::vector<std::vector<int>> adj(N);
    for (int64_t v = 0; v < N; ++v) adj[v].push_back((int)v);
    for (int64_t t = 0; t < T; ++t) {
      const int id[4] = {tets[t].x, tets[t].y, tets[t].z, tets[t].w};
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) adj[id[a]].push_back(id[b]);
    }
    std::vector<int> rowptr(N + 1, 0);
    for (int64_t v = 0; v < N; ++v) {
      auto& r = adj[v];
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      rowptr[v + 1] = rowptr[v] + (int)r.size();
    }
    c->nnzb = rowptr[N];
    std::vector<int> cols(c->nnzb), diag(N), slot(16 * T);
    for (int64_t v = 0; v < N; ++v) {
      std::copy(adj[v].begin(), adj[v].end(), cols.begin() + rowptr[v]);
      diag[v] = rowptr[v] + (int)(std::lower_bound(adj[v].begin(), adj[v].end(), (int)v) - adj[v].begin());
    }
    for (int64_t t = 0; t < T; ++t) {
      const int id[4] = {tets[t].x, tets[t].y, tets[t].z, tets[t].w};
      for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
          auto& r = adj[id[a]];
          slot[16 * t + 4 * a + b] =
              rowptr[id[a]] + (int)(std::lower_bound(r.begin(), r.end(), id[b]) - r.begin());
        }
    }
    c->rowptr.upload(rowptr.data(), N + 1, st);
    c->cols.upload(cols.data(), c->nnzb, st);
    c->h_rowptr = rowptr;
    c->h_cols = cols;
    c->diag_slot.upload(diag.data(), N, st);
    c->tet_slot.upload(slot.data(), 16 * T, st);
    // Deterministic assembly maps (fixed summation order, no atomics):
    //   BSR slot -> its element blocks 16t + 4a + b (t ascending), for the
    //   Hessian gather; vertex -> its tet corners 4t + a, for the gradient.
    // Tets of no material and pinned rows / columns contribute nothing.
    const int64_t T_el = c->T_snh + c->T_arap;
    std::vector<unsigned char> pinh(N);
    for (int64_t i = 0; i < N; ++i) pinh[i] = s->dirichlet[n2o[i]] ? 1 : 0;
    std::vector<int> hoff(c->nnzb + 1, 0), voff(N + 1, 0), srow(c->nnzb);
    for (int64_t v = 0; v < N; ++v)
      for (int k = rowptr[v]; k < rowptr[v + 1]; ++k) srow[k] = (int)v;
    for (int64_t t = 0; t < T_el; ++t) {
      const int id[4] = {tets[t].x, tets[t].y, tets[t].z, tets[t].w};
      for (int a = 0; a < 4; ++a) {
        if (pinh[id[a]]) continue;
        ++voff[id[a] + 1];
        for (int b = 0; b < 4; ++b)
          if (!pinh[id[b]]) ++hoff[slot[16 * t + 4 * a + b] + 1];
      }
    }
    for (int64_t k = 0; k < c->nnzb; ++k) hoff[k + 1] += hoff[k];
    for (int64_t v = 0; v < N; ++v) voff[v + 1] += voff[v];
    std::vector<int> hval(hoff[c->nnzb]), vval(voff[N]);
    std::vector<int> hcur(hoff.begin(), hoff.end() - 1), vcur(voff.begin(), voff.end() - 1);
    for (int64_t t = 0; t < T_el; ++t) {
      const int id[4] = {tets[t].x, tets[t].y, tets[t].z, tets[t].w};
      for (int a = 0; a < 4; ++a) {
        if (pinh[id[a]]) continue;
        vval[vcur[id[a]]++] = (int)(4 * t + a);
        for (int b = 0; b < 4; ++b)
          if (!pinh[id[b]]) hval[hcur[slot[16 * t + 4 * a + b]]++] = (int)(16 * t + 4 * a + b);
      }
    }
    c->hs_off.upload(hoff.data(), c->nnzb + 1, st);
    if (hval.empty()) hval.push_back(0);
    c->hs_val.upload(hval.data(), hval.size(), st);
    c->slot_row.upload(srow.data(), c->nnzb, st);
    c->vt_off.upload(voff.data(), N + 1, st);
    if (vval.empty()) vval.push_back(0);
    c->vt_val.upload(vval.data(), vval.size(), st);
    c->fbuf.ensure(12 * (size_t)std::max<int64_t>(1, T_el));
    c->hbuf.ensure(90 * (size_t)std::max<int64_t>(1, T_el));
    c->bsr.ensure(9 * (size_t)c->nnzb);
    CUDA_CHECK(cudaStreamSynchronize(st));
  }
  // surface
  {
    std::vector<int> tri(3 * c->F), tri_sorted(3 * c->F), edge(2 * c->E), sv(c->V);
    for (int64_t f = 0; f < c->F; ++f) {
      int64_t o[3] = {s->tris[3 * f], s->tris[3 * f + 1], s->tris[3 * f + 2]};
      for (int k = 0; k < 3; ++k) tri[3 * f + k] = o2n[o[k]];
      std::sort(o, o + 3);
      for (int k = 0; k < 3; ++k) tri_sorted[3 * f + k] = o2n[o[k]];
    }
    for (int64_t e = 0; e < 2 * c->E; ++e) edge[e] = o2n[s->edges[e]];
    for (int64_t v = 0; v < c->V; ++v) sv[v] = o2n[s->surf_verts[v]];
    c->tri.upload(tri.data(), 3 * c->F, st);
    c->tri_sorted.upload(tri_sorted.data(), 3 * c->F, st);
    c->edge.upload(edge.data(), 2 * c->E, st);
    c->sverts.upload(sv.data(), c->V, st);
    CUDA_CHECK(cudaStreamSynchronize(st));
  }
  {  // bodies: connected components over tets and surface triangles (union-find)
    std::vector<int> par(N);
    std::iota(par.begin(), par.end(), 0);
    std::function<int(int)> root = [&](int a) {
      while (par[a] != a) a = par[a] = par[par[a]];
      return a;
    };
    auto join = [&](int a, int b) {
      a = root(a);
      b = root(b);
      if (a != b) par[std::max(a, b)] = std::min(a, b);
    };
    for (int64_t t = 0; t < T; ++t) {
      join(tets[t].x, tets[t].y);
      join(tets[t].x, tets[t].z);
      join(tets[t].x, tets[t].w);
    }
    for (int64_t f = 0; f < c->F; ++f) {
      const int a = o2n[s->tris[3 * f]];
      join(a, o2n[s->tris[3 * f + 1]]);
      join(a, o2n[s->tris[3 * f + 2]]);
    }
    std::vector<int> id(N, -1), body(N);
    int nb = 0;
    for (int64_t v = 0; v < N; ++v) {
      const int r = root((int)v);
      if (id[r] < 0) id[r] = nb++;
      body[v] = id[r];
    }
    // one body, or too many to matter (loose points): the single-c enumeration
    c->n_bodies = (nb > 1 && nb <= 65536) ? nb : 1;
    if (c->n_bodies == 1) std::fill(body.begin(), body.end(), 0);
    c->body.upload(body.data(), N, st);
  }
  const size_t n3 = 3 * (size_t)N;
  for (DBuf<double>* b : {&c->x, &c->xt, &c->vel, &c->g, &c->g_prev, &c->z, &c->p, &c->Hp, &c->p_prev, &c->Hp_prev, &c->z_prev,
                          &c->hv, &c->x_start, &c->x_best, &c->tmp, &c->tmp2})
    b->ensure(n3);
  c->counters.zero(16, c->stream);
  c->mid_part.ensure(6 * 148);
  c->dscal.ensure(64);
  c->alpha_d.ensure(c->D);
  setup_levels(c);
}

// ---------------------------------------------------------------------------
// advance_step (solver.py:296-458)

struct LoopResult {
  std::vector<mp_iter_record> recs;
  bool converged = false;
  uint32_t flags = 0;
};

using Clock = std::chrono::steady_clock;
static double ms_since(Clock::time_point a) {
  return std::chrono::duration<double, std::milli>(Clock::now() - a).count();
}

// 2-norm condition number of a 2x2 matrix (np.linalg.cond)
static double cond2(double a, double b, double c, double d) {
  double E = 0.5 * (a + d), F = 0.5 * (a - d), G = 0.5 * (c + b), H = 0.5 * (c - b);
  double Q = std::sqrt(E * E + H * H), R = std::sqrt(F * F + G * G);
  double s1 = Q + R, s2 = std::fabs(Q - R);
  if (s2 == 0.0) return INFINITY;
  return s1 / s2;
}

// LAPACK gesv on 2x2 (partial pivoting, reciprocal pivot scaling)
static void solve2(double A[2][2], double b[2], double* x0, double* x1) {
  double a00 = A[0][0], a01 = A[0][1], a10 = A[1][0], a11 = A[1][1], b0 = b[0], b1 = b[1];
  if (std::fabs(a10) > std::fabs(a00)) {
    std::swap(a00, a10);
    std::swap(a01, a11);
    std::swap(b0, b1);
  }
  double l = a10 * (1.0 / a00);
  double u11 = a11 - l * a01;
  double y1 = b1 - l * b0;
  *x1 = y1 / u11;
  *x0 = (b0 - a01 * (*x1)) / a00;
}

static void advance_loop_body(mp_ctx* c, double h, LoopResult& R);

static void advance_loop(mp_ctx* c, double h, LoopResult& R) {
  const auto t0 = Clock::now();
  if (c->nshards > 1) {
    // every shard runs the loop (SPMD, lockstep); shard 0's records are the group's
    run_shards(c, [&](mp_ctx* sc) {
      LoopResult Rs;
      advance_loop_body(sc, h, Rs);
      if (sc->rank == 0) R = std::move(Rs);
    });
  } else {
    advance_loop_body(c, h, R);
  }
  if (c->timing) {
    c->loop_ms += ms_since(t0);
    c->n_loop += 1;
  }
}

static void advance_loop_body(mp_ctx* c, double h, LoopResult& R) {
  const mp_solver_config& cfg = c->cfg;
  const int64_t n3 = 3 * c->N;
  cudaStream_t st = c->stream;
  CUDA_CHECK(cudaMemcpyAsync(c->x_start.p, c->x.p, n3 * 8, cudaMemcpyDeviceToDevice, st));
  CUDA_CHECK(cudaMemcpyAsync(c->x_best.p, c->x.p, n3 * 8, cudaMemcpyDeviceToDevice, st));
  const bool full_every = cfg.update_strategy == MP_UPDATE_FULLREBUILD;
  bool restart = true;
  bool have_prev = false;   // p_prev / Hp_prev / z_prev valid
  double best = INFINITY;
  const bool subspace = cfg.direction_rule == MP_DIR_SUBSPACE2D;
  double prev_zg = 0.0, prev_gp = 0.0;  // g_prev.z_prev, g_prev.p_prev (baseline beta rules)
  R.recs.clear();
  R.converged = false;
  c->bsr_ahead_pending = false;
  c->mas_flags_pending = false;
  struct DeferGuard {  // the loop checks the MAS flags at its next sync; restored on any exit
    mp_ctx* c;
    explicit DeferGuard(mp_ctx* x) : c(x) { c->defer_mas_check = true; }
    ~DeferGuard() {
      c->defer_mas_check = false;
      c->mas_overlap = nullptr;  // (it captures this loop's locals)
    }
  } defer_guard(c);
  for (int64_t k = 0; k < cfg.iter_max; ++k) {
    auto t0 = Clock::now();
    const bool rebuild = restart || full_every;
    CUDA_CHECK(cudaEventRecord(c->ev_t0, st));
    if (rebuild) bsr_ahead(c, c->x, h);
    timer_begin(c, MP_STAGE_CONSTRAINT_SET);
    constraint_set(c, c->x);
    timer_end(c, MP_STAGE_CONSTRAINT_SET, 0.0);
    bool grad_done = false;
    auto grad = [&]() {
      timer_begin(c, MP_STAGE_GRADIENT);
      gradient(c, c->x, c->xt, h, c->g);
      timer_end(c, MP_STAGE_GRADIENT, gradient_bytes(c));
      grad_done = true;
    };
    if (rebuild) {
      c->mas_overlap = grad;  // launched inside mas_build, beside the coarse assembly
      snapshot(c, c->x, h, true);
      c->mas_overlap = nullptr;
    } else {
      timer_begin(c, MP_STAGE_UPDATE);
      update_build(c);
      timer_end(c, MP_STAGE_UPDATE, 0.0);
    }
    if (!grad_done) grad();
    timer_begin(c, MP_STAGE_MAS_APPLY);
    precond_apply(c, c->g, c->z, true);
    timer_end(c, MP_STAGE_MAS_APPLY, mas_apply_bytes(c));
    // (no host sync here: t_grad_ms is the CUDA-event time from the
    // iteration's start to z, read at the record)
    CUDA_CHECK(cudaEventRecord(c->ev_t1, st));

    timer_begin(c, MP_STAGE_HVP);
    hvp(c, c->z, c->hv, !rebuild);
    timer_end(c, MP_STAGE_HVP, hvp_bytes(c, !rebuild));
    DotSpec S{};
    S.n = 0;
    auto add = [&](const double* a, const double* b) {
      if (S.n >= MAX_DOTS) throw MpError(MP_ERR_CONFIG, "too many fused dots");
      S.a[S.n] = a;
      S.b[S.n] = b;
      return S.n++;
    };
    int i_zz = add(c->z, c->z), i_gg = add(c->g, c->g), i_zg = add(c->z, c->g), i_zv = add(c->z, c->hv);
    int i_zHp = -1, i_pv = -1, i_pHp = -1, i_pg = -1, i_gzp = -1;
    if (have_prev) {
      if (subspace) {  // the 2x2 system (baselines need MAX_DOTS slots for their beta dots)
        i_zHp = add(c->z, c->Hp_prev);
        i_pv = add(c->p_prev, c->hv);
        i_pHp = add(c->p_prev, c->Hp_prev);
      }
      i_pg = add(c->p_prev, c->g);
      i_gzp = add(c->g, c->z_prev);
    }
    // baseline beta rules: the differences are formed elementwise first, as
    // the reference does (g @ (z - z_prev), y = g - g_prev), not from
    // differences of dots (cancellation)
    int i_gzd = -1, i_yz = -1, i_yzd = -1, i_py = -1;
    if (have_prev && !subspace && !restart) {
      k_sub2<<<grid_for(n3, 256), 256, 0, st>>>(n3, c->z, c->z_prev, c->g, c->g_prev, c->tmp, c->tmp2);
      LAUNCH_CHECK();
      i_gzd = add(c->g, c->tmp);
      i_yz = add(c->tmp2, c->z);
      i_yzd = add(c->tmp2, c->tmp);
      i_py = add(c->p_prev, c->tmp2);
    }
    multidot(c, n3, S);
    mas_flags_check(c);  // the MAS build's non-SPD flags rode on that sync
    const auto t1 = Clock::now();
    double dots[MAX_DOTS];
    std::memcpy(dots, c->h_scal, sizeof(double) * S.n);
    const double z_norm = std::sqrt(dots[i_zz]);
    const double grad_norm = std::sqrt(dots[i_gg]);
    const double zg = dots[i_zg], zv = dots[i_zv];
    if (z_norm < best) {
      best = z_norm;
      CUDA_CHECK(cudaMemcpyAsync(c->x_best.p, c->x.p, n3 * 8, cudaMemcpyDeviceToDevice, st));
    }
    double mu = 0.0, nu = 0.0;
    double pinf = 0.0;
    double gp_now = 0.0;
    if (z_norm == 0.0) {
      CUDA_CHECK(cudaMemsetAsync(c->p.p, 0, n3 * 8, st));
      CUDA_CHECK(cudaMemsetAsync(c->Hp.p, 0, n3 * 8, st));
    } else if (!subspace) {
      // baseline_direction (solver.py:171-200, 393-400): p = -z + beta p_prev
      double beta = 0.0;
      if (!restart && have_prev) {
        const double gz = zg, pg = dots[i_pg];
        switch (cfg.direction_rule) {
          case MP_DIR_FR: beta = gz / prev_zg; break;
          case MP_DIR_PR: beta = dots[i_gzd] / prev_zg; break;
          case MP_DIR_DK: {
            const double py = dots[i_py];  // p_prev . y, y = g - g_prev
            if (py != 0.0) beta = dots[i_yz] / py - dots[i_yzd] * pg / (py * py);
            break;
          }
          default: beta = prev_gp != 0.0 ? -gz / prev_gp : 0.0; break;  // CD
        }
        beta = std::max(beta, 0.0);
      }
      form_direction(c, -1.0, beta, beta != 0.0 ? c->p_prev.p : nullptr, beta != 0.0 ? c->Hp_prev.p : nullptr);
      gp_now = c->h_scal[0];
      pinf = c->h_scal[1];
      if (!restart && have_prev && gp_now >= 0.0) {  // not a descent direction: steepest
        beta = 0.0;
        form_direction(c, -1.0, 0.0, nullptr, nullptr);
        gp_now = c->h_scal[0];
        pinf = c->h_scal[1];
      }
      mu = 1.0;
      nu = beta;
    } else if (restart || !have_prev) {
      if (zv <= 0.0) throw MpError(MP_ERR_MODEL_NOT_SPD, "z.Hz <= 0 at restart");
      mu = zg / zv;
      nu = 0.0;
      form_direction(c, -mu, 0.0, nullptr, nullptr);
      gp_now = c->h_scal[0];
      pinf = c->h_scal[1];
    } else {
      // solve_2d_subspace (solver.py:147-161)
      const double zHz = zv;
      if (zHz <= 0.0) throw MpError(MP_ERR_MODEL_NOT_SPD, "z.Hz <= 0 in subspace solve");
      double A[2][2] = {{zHz, -dots[i_zHp]}, {-dots[i_pv], dots[i_pHp]}};
      double b[2] = {zg, -dots[i_pg]};
      if (cond2(A[0][0], A[0][1], A[1][0], A[1][1]) > 1e12) {
        mu = b[0] / zHz;
        nu = 0.0;
      } else {
        solve2(A, b, &mu, &nu);
      }
      form_direction(c, -mu, nu, c->p_prev, c->Hp_prev);
      double gp = c->h_scal[0];
      pinf = c->h_scal[1];
      if (gp >= 0.0 && z_norm > 0.0) {
        if (zv <= 0.0) throw MpError(MP_ERR_MODEL_NOT_SPD, "z.Hz <= 0 in fallback");
        mu = zg / zv;
        nu = 0.0;
        form_direction(c, -mu, 0.0, nullptr, nullptr);
        pinf = c->h_scal[1];
      }
    }
    auto t2 = Clock::now();
    double min_alpha = 1.0;
    bool certified = true;
    const double e_iter = c->record_energy ? energy(c, c->x, c->xt, h) : NAN;
    if (pinf > 0.0 && subspace) {
      timer_begin(c, MP_STAGE_CCD);
      CcdResult cr = ccd_clamp(c, c->x, c->p, pinf, cfg.ccd_per_subdomain != 0, c->tmp, c->ccd_exact_set);
      timer_end(c, MP_STAGE_CCD, 0.0);
      min_alpha = cr.min_alpha;
      certified = cr.certified;
      std::swap(c->x.p, c->tmp.p);
    } else if (pinf > 0.0) {
      // baselines: global pair step, then backtracking on the incremental
      // potential with a fresh constraint set per trial (solver.py:283-293, 406-412)
      timer_begin(c, MP_STAGE_CCD);
      CcdResult cr = ccd_clamp(c, c->x, c->p, pinf, false, c->tmp, c->ccd_exact_set);
      timer_end(c, MP_STAGE_CCD, 0.0);
      min_alpha = cr.min_alpha;
      const double e0 = energy(c, c->x, c->xt, h);  // cur still holds the set at x
      double alpha = std::min(1.0, min_alpha);
      for (int it = 0; it < 40; ++it) {
        k_ccd_update<<<grid_for(n3, 256), 256, 0, st>>>(c->N, c->bs, c->x, c->p, nullptr, alpha, c->tmp);
        LAUNCH_CHECK();
        bool lower = false;
        try {
          constraint_set(c, c->tmp);
          lower = energy(c, c->tmp, c->xt, h) < e0;
        } catch (const MpError& e) {
          if (e.status != MP_ERR_PENETRATION && e.status != MP_ERR_DEGENERATE) throw;
        }
        if (lower) break;
        alpha *= 0.5;
      }
      k_ccd_update<<<grid_for(n3, 256), 256, 0, st>>>(c->N, c->bs, c->x, c->p, nullptr, alpha, c->tmp);
      LAUNCH_CHECK();
      std::swap(c->x.p, c->tmp.p);
      mu = alpha;
    }
    sync_stream(c);
    auto t3 = Clock::now();
    mp_iter_record rec{};
    rec.k = k;
    rec.grad_norm = grad_norm;
    rec.z_norm = z_norm;
    rec.r = 0.0;
    rec.restart = restart ? 1 : 0;
    rec.n_contacts = (int32_t)c->cur.count;
    rec.mu = mu;
    rec.nu = nu;
    rec.min_alpha = min_alpha;
    {
      float gms = 0.f;  // iteration start -> z, on the device (both events completed by the syncs since)
      CUDA_CHECK(cudaEventElapsedTime(&gms, c->ev_t0, c->ev_t1));
      rec.t_grad_ms = gms;
      // the direction phase: the host time to t2 less the part before z
      rec.t_dir_ms = std::max(0.0, std::chrono::duration<double, std::milli>(t2 - t0).count() - (double)gms);
    }
    (void)t1;
    rec.t_ccd_ms = std::chrono::duration<double, std::milli>(t3 - t2).count();
    rec.n_candidates = (int32_t)(rebuild ? 0 : c->n_cand);
    rec.n_ccd_pairs = (int32_t)std::min<int64_t>(c->n_ccd_seen, INT32_MAX);  // saturates (>2^31 at C3)
    rec.ccd_certified = certified ? 1 : 0;
    rec.energy = e_iter;
    const bool converged_now = z_norm <= cfg.eps;
    if (converged_now && (restart || full_every)) {
      R.recs.push_back(rec);
      R.converged = true;
      break;
    }
    if (converged_now) {
      restart = true;
    } else {
      double r = 0.0;
      if (have_prev) {
        if (zg <= 0.0) throw MpError(MP_ERR_PRECOND_NOT_SPD, "g.z <= 0 in restart ratio");
        r = std::fabs(dots[i_gzp]) / zg;
      }
      rec.r = r;
      restart = r > cfg.delta;
    }
    R.recs.push_back(rec);
    std::swap(c->z_prev.p, c->z.p);
    std::swap(c->p_prev.p, c->p.p);
    std::swap(c->Hp_prev.p, c->Hp.p);
    if (!subspace) std::swap(c->g_prev.p, c->g.p);  // history g_prev (solver.py:449)
    prev_zg = zg;
    prev_gp = gp_now;
    have_prev = true;
  }
  if (!R.converged) {
    R.flags |= MP_FLAG_NOT_CONVERGED;
    CUDA_CHECK(cudaMemcpyAsync(c->x.p, c->x_best.p, n3 * 8, cudaMemcpyDeviceToDevice, st));
  }
  k_velocity<<<grid_for(n3, 256), 256, 0, st>>>(c->N, c->x, c->x_start, h, c->pinned, c->vel);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// C ABI

static const char* status_codes[] = {"ok",
                                     "penetration-detected",
                                     "non-spd-subdomain",
                                     "capacitance-not-spd",
                                     "model-not-spd",
                                     "precond-not-spd",
                                     "non-spd-block",
                                     "degenerate-primitive",
                                     "config-error",
                                     "capacity-overflow",
                                     "cuda-error"};

template <typename Fn>
static int guarded(mp_ctx* c, Fn&& fn) {
  g_launch_counter = c ? &c->launches : nullptr;
  try {
    if (c) CUDA_CHECK(cudaSetDevice(c->device));
    if (c) c->bsr_ahead_pending = false;  // an H_base assembled ahead belongs to one loop iteration only
    if (c) c->mas_overlap = nullptr;
    fn();
    return MP_OK;
  } catch (const MpError& e) {
    if (c) c->last_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    return MP_ERR_CUDA;
  }
}

static void upload_vec_new(mp_ctx* c, const double* host, double* dev) {
  const int64_t n3 = 3 * c->N;
  c->tmp2.ensure(n3);
  CUDA_CHECK(cudaMemcpyAsync(c->tmp2.p, host, n3 * 8, cudaMemcpyHostToDevice, c->stream));
  k_to_new<<<grid_for(n3, 256), 256, 0, c->stream>>>(c->N, c->new2old, c->tmp2, dev);
  LAUNCH_CHECK();
}

static void download_vec_old(mp_ctx* c, const double* dev, double* host) {
  const int64_t n3 = 3 * c->N;
  k_to_old<<<grid_for(n3, 256), 256, 0, c->stream>>>(c->N, c->new2old, dev, c->tmp2);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemcpyAsync(host, c->tmp2.p, n3 * 8, cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
}

// sequential per-shard host work (uploads) on each shard's device
template <class Fn>
static void each_shard(mp_ctx* c, Fn&& fn) {
  if (c->nshards <= 1 || !c->grp) {
    fn(c);
    return;
  }
  int64_t* saved = g_launch_counter;
  for (mp_ctx* sc : c->grp->sh) {
    CUDA_CHECK(cudaSetDevice(sc->device));
    g_launch_counter = &sc->launches;
    fn(sc);
  }
  g_launch_counter = saved;
  CUDA_CHECK(cudaSetDevice(c->device));
}

static void prepare_on(mp_ctx* sc, double h) {
  k_prepare<<<grid_for(3 * sc->N, 256), 256, 0, sc->stream>>>(sc->N, sc->x, sc->vel, sc->mass, sc->f_ext, sc->pinned,
                                                              h, sc->xt);
  LAUNCH_CHECK();
}

// stage taps evaluate one device stage on a whole scene: single-GPU contexts
static void single_gpu_only(mp_ctx* c) {
  if (c->nshards > 1) throw MpError(MP_ERR_CONFIG, "stage taps run on single-GPU contexts (mp_create)");
}

extern "C" {

const char* mp_status_code(int status) {
  if (status < 0 || status > MP_ERR_CUDA) return "sim-error";
  return status_codes[status];
}

const char* mp_last_error(mp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

void* mp_stream(mp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t mp_launch_count(mp_ctx* ctx) {
  if (!ctx) return 0;
  if (!ctx->grp) return ctx->launches;
  int64_t n = 0;
  for (mp_ctx* sc : ctx->grp->sh) n += sc->launches;
  return n;
}

int mp_stage_timing(mp_ctx* c, int enable) {
  return guarded(c, [&] {
    for (auto& t : c->timers) {
      timer_fold(t);
      t.total_ms = 0.0;
      t.bytes = 0.0;
      t.count = 0;
    }
    c->sync_wait_ms = 0.0;
    c->n_sync = 0;
    c->loop_ms = 0.0;
    c->n_loop = 0;
    c->timing = enable != 0;
  });
}

int mp_set_option(mp_ctx* c, int option, int64_t value) {
  return guarded(c, [&] {
    if (option == MP_OPT_CCD_EXACT_SET) c->ccd_exact_set = value != 0;
    else if (option == MP_OPT_RECORD_ENERGY) c->record_energy = value != 0;
    else if (option == MP_OPT_APPLY_TMA) c->apply_mode = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
    else if (option == MP_OPT_APPLY_STAGES) c->apply_stages = value == 3 ? 3 : 2;
    else if (option == MP_OPT_BP_FUSED) c->bp_fused = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
    else if (option == MP_OPT_KEEP_COARSE) c->keep_coarse = value != 0;
    else if (option == MP_OPT_GRAD_FUSED) c->fused_grad = value != 0;
    else if (option == MP_OPT_APPLY_OVERLAP) c->overlap_apply = value != 0;
    else if (option == MP_OPT_CCD_PREFILTER) c->ccd_prefilter = value != 0;
    else if (option == MP_OPT_CCD_BODIES) c->ccd_bodies = value != 0;
    else if (option == MP_OPT_CCD_LOCAL) c->ccd_local = value != 0;
    else if (option == MP_OPT_CCD_BVH) c->ccd_bvh = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
    else if (option == MP_OPT_BVH_TASKS) {
      c->bvh_task_cap = std::max<int64_t>(0, value);
      c->bvh_task_max = value < 0 ? -value : 0;
    }
    else if (option == MP_OPT_APPEND_LIMIT) {
      const int lim = (int)std::max<int64_t>(64, std::min<int64_t>(HQ_APPEND_LIMIT, value <= 0 ? HQ_APPEND_LIMIT : value));
      CUDA_CHECK(cudaMemcpyToSymbol(g_append_limit, &lim, sizeof(int)));
    }
    else if (option == MP_OPT_APPLY_CTAS) c->apply_ctas_per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(8, value));
    else throw MpError(MP_ERR_CONFIG, "unknown option");
  });
}

int mp_stage_stats(mp_ctx* c, int stage, double* total_ms, int64_t* count, double* bytes) {
  return guarded(c, [&] {
    if (stage < 0 || stage >= MP_STAGE_COUNT) throw MpError(MP_ERR_CONFIG, "unknown stage");
    if (stage == MP_STAGE_HOST_WAIT || stage == MP_STAGE_LOOP) {
      const bool w = stage == MP_STAGE_HOST_WAIT;
      if (total_ms) *total_ms = w ? c->sync_wait_ms : c->loop_ms;
      if (count) *count = w ? c->n_sync : c->n_loop;
      if (bytes) *bytes = 0.0;
      return;
    }
    StageTimer& t = c->timers[stage];
    timer_fold(t);
    if (total_ms) *total_ms = t.total_ms;
    if (count) *count = t.count;
    if (bytes) *bytes = t.bytes;
  });
}

static thread_local std::string g_create_error;
const char* mp_create_error(void) { return g_create_error.c_str(); }

int mp_create(const mp_scene_desc* scene, const mp_solver_config* cfg, int device, mp_ctx** out) {
  *out = nullptr;
  mp_ctx* c = new mp_ctx();
  int st = guarded(c, [&] { create_ctx(scene, cfg, device, c); });
  if (st != MP_OK) {
    g_create_error = c->last_error;
    delete c;
    return st;
  }
  *out = c;
  return MP_OK;
}

int mp_create_multi(const mp_scene_desc* scene, const mp_solver_config* cfg, int n_dev, const int* dev_ids,
                    mp_ctx** out) {
  *out = nullptr;
  if (n_dev < 1 || n_dev > GROUP_MAX || !dev_ids) {
    g_create_error = "n_dev must lie in [1, 16]";
    return MP_ERR_CONFIG;
  }
  if (n_dev == 1) return mp_create(scene, cfg, dev_ids[0], out);
  std::vector<mp_ctx*> sh(n_dev, nullptr);
  for (int q = 0; q < n_dev; ++q) {
    const int st = mp_create(scene, cfg, dev_ids[q], &sh[q]);
    if (st != MP_OK) {
      for (mp_ctx* s2 : sh)
        if (s2) mp_destroy(s2);
      return st;
    }
  }
  Group* G = new Group();
  G->sh = sh;
  G->bar.n = n_dev;
  int st = guarded(sh[0], [&] {
    // peer access between distinct devices (exchanges are peer copies over NVLink)
    for (int a = 0; a < n_dev; ++a)
      for (int b = 0; b < n_dev; ++b) {
        const int da = dev_ids[a], db = dev_ids[b];
        if (da == db) continue;
        int can = 0;
        CUDA_CHECK(cudaDeviceCanAccessPeer(&can, da, db));
        if (!can) continue;
        CUDA_CHECK(cudaSetDevice(da));
        const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_CHECK(e);
        cudaGetLastError();
      }
    for (int q = 0; q < n_dev; ++q) {
      CUDA_CHECK(cudaSetDevice(dev_ids[q]));
      CUDA_CHECK(cudaEventCreateWithFlags(&G->ev[q], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&G->ev2[q], cudaEventDisableTiming));
      sh[q]->grp = G;
      sh[q]->rank = q;
      sh[q]->nshards = n_dev;
      group_ranges(sh[q], q, n_dev);
    }
    CUDA_CHECK(cudaSetDevice(dev_ids[0]));
    const size_t np = (size_t)sh[0]->n_chunks * MAX_DOTS;
    for (auto& hp : G->hpart) CUDA_CHECK(cudaMallocHost(&hp, sizeof(double) * np));
  });
  if (st != MP_OK) {
    g_create_error = sh[0]->last_error;
    mp_destroy(sh[0]);
    return st;
  }
  *out = sh[0];
  return MP_OK;
}

void mp_destroy(mp_ctx* ctx) {
  if (!ctx) return;
  if (ctx->grp && ctx->rank != 0) return;  // shards are owned by shard 0
  if (ctx->grp)
    for (mp_ctx* sc : ctx->grp->sh) {
      cudaSetDevice(sc->device);
      cudaStreamSynchronize(sc->stream);
    }
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

int mp_set_config(mp_ctx* c, const mp_solver_config* cfg) {
  return guarded(c, [&] {
    validate_config(*cfg);
    if (cfg->block_size != c->cfg.block_size)
      throw MpError(MP_ERR_CONFIG, "block_size is fixed per context (partition); create a new context");
    const bool relevel = cfg->levels != c->cfg.levels || cfg->coarse_block != c->cfg.coarse_block;
    // the hierarchy (streams, gather maps) only depends on the MAS depth; the
    // per-call config of the Python API re-sets the rest freely
    each_shard(c, [&](mp_ctx* sc) {
      sc->cfg = *cfg;
      if (relevel) setup_levels(sc);
      sc->have_mas = false;
    });
    if (relevel && c->grp) {  // the group's chunk partial buffers follow the new chunk count
      for (auto& hp : c->grp->hpart) {
        if (hp) cudaFreeHost(hp);
        CUDA_CHECK(cudaMallocHost(&hp, sizeof(double) * (size_t)c->n_chunks * MAX_DOTS));
      }
    }
  });
}

int mp_spd_inverse(int device, int64_t n, const double* A, double* inv, int32_t* not_spd) {
  static thread_local mp_ctx* tmp = nullptr;  // scratch context: streams + buffers of one coarse level
  if (n < 1 || n > (1 << 15)) return MP_ERR_CONFIG;
  if (!tmp) tmp = new mp_ctx();
  return guarded(tmp, [&] {
    mp_ctx* c = tmp;
    c->device = device;
    CUDA_CHECK(cudaSetDevice(device));
    if (!c->stream) CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    set_smem_limits();
    CoarseLevel L;
    struct Unown {  // the stream belongs to the scratch context, not to L
      CoarseLevel& l;
      ~Unown() { l.st = nullptr; }
    } unown{L};
    L.n = (int)n;
    L.st = c->stream;
    const int nT = (L.n + CS_TB - 1) / CS_TB;
    std::vector<int2> units;
    L.cs_ch = CS_CH;
    for (int ch = 1; ch <= CS_CH; ++ch) {
      int64_t nu = 0;
      for (int I = 0; I < nT; ++I) nu += (I + ch) / ch;
      if (nu + 1 <= 148) {
        L.cs_ch = ch;
        break;
      }
    }
    for (int I = 0; I < nT; ++I)
      for (int j0 = 0; j0 <= I; j0 += L.cs_ch) units.push_back(make_int2(I, j0));
    L.n_units = (int)units.size();
    L.cs_units.upload(units.data(), units.size(), c->stream);
    L.dense.upload(A, (size_t)n * n, c->stream);
    c->counters.zero(16, c->stream);
    dense_spd_inverse(c, L, c->counters.p);
    std::vector<double> packed(cyc_size(L.n));
    int flag = 0;
    CUDA_CHECK(cudaMemcpyAsync(packed.data(), L.inv.p, sizeof(double) * packed.size(), cudaMemcpyDeviceToHost,
                               c->stream));
    CUDA_CHECK(cudaMemcpyAsync(&flag, c->counters.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    *not_spd = flag;
    for (int i = 0; i < L.n; ++i)
      for (int j = 0; j < L.n; ++j) inv[(int64_t)i * n + j] = packed[cyc_index(L.n, i, j)];
  });
}

int mp_check_intersections(int device, int64_t n_verts, const double* x, int64_t n_tris, const int64_t* tris,
                           double coplanar_tol, int64_t* n_hits, int64_t* first_tri) {
  static thread_local mp_ctx* tmp = nullptr;  // scratch context: a stream and the sort helpers
  if (n_verts < 1 || n_tris < 0 || n_tris >= (1ll << 31)) return MP_ERR_CONFIG;
  if (!tmp) tmp = new mp_ctx();
  return guarded(tmp, [&] {
    mp_ctx* c = tmp;
    c->device = device;
    CUDA_CHECK(cudaSetDevice(device));
    if (!c->stream) CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    *n_hits = 0;
    *first_tri = -1;
    if (n_tris < 2) return;
    std::vector<int> t32(3 * n_tris);
    for (int64_t i = 0; i < 3 * n_tris; ++i) {
      if (tris[i] < 0 || tris[i] >= n_verts) throw MpError(MP_ERR_CONFIG, "triangle index out of range");
      t32[i] = (int)tris[i];
    }
    DBuf<double> xd;
    DBuf<int> td;
    xd.upload(x, 3 * n_verts, c->stream);
    td.upload(t32.data(), t32.size(), c->stream);
    int first = INT32_MAX;
    *n_hits = (int64_t)tri_intersections(c, xd, td, n_tris, &first, coplanar_tol);
    *first_tri = first == INT32_MAX ? -1 : first;
  });
}

int mp_set_contact(mp_ctx* c, double d_hat, double kappa) {
  return guarded(c, [&] {
    if (!(d_hat > 0) || !(kappa > 0)) throw MpError(MP_ERR_CONFIG, "d_hat and kappa must be positive");
    each_shard(c, [&](mp_ctx* sc) {
      sc->d_hat = d_hat;
      sc->kappa = kappa;
      sc->have_snapshot = sc->have_mas = false;
    });
  });
}

int mp_shard_range(int64_t n_verts, int32_t block_size, int32_t levels, int32_t coarse_block, int32_t rank,
                   int32_t nshards, int64_t* out) {
  if (n_verts < 1 || block_size < 1 || coarse_block < 1 || nshards < 1 || rank < 0 || rank >= nshards)
    return MP_ERR_CONFIG;
  // the unit group_ranges aligns to: the level-1 aggregate (mas.py:155-169)
  // when one is built, else the subdomain
  const int64_t D = (n_verts + block_size - 1) / block_size;
  const bool coarse = levels >= 1 && (D + coarse_block - 1) / coarse_block != D;
  const int64_t U = coarse ? (int64_t)block_size * coarse_block : (int64_t)block_size;
  const int64_t NU = (n_verts + U - 1) / U;
  const int64_t u0 = NU * rank / nshards, u1 = NU * (rank + 1) / nshards;
  const int64_t v0 = std::min(n_verts, u0 * U), v1 = std::min(n_verts, u1 * U);
  out[0] = v0;
  out[1] = v1;
  out[2] = v0 / block_size;
  out[3] = (v1 + block_size - 1) / block_size;
  out[4] = coarse ? u0 : 0;
  out[5] = coarse ? u1 : 0;
  out[6] = u0;  // reduction chunks
  out[7] = u1;
  return MP_OK;
}

int mp_partition_host(const double* rest, int64_t n, int32_t block_size, int64_t* subdomain_of) {
  if (n < 1 || block_size < 1) return MP_ERR_CONFIG;
  try {
    std::vector<int> n2o;
    std::vector<int64_t> sub;
    morton_partition(rest, n, block_size, n2o, sub);
    std::memcpy(subdomain_of, sub.data(), sizeof(int64_t) * n);
  } catch (...) {
    return MP_ERR_CONFIG;
  }
  return MP_OK;
}

int mp_partition(mp_ctx* c, int64_t* D, int64_t* subdomain_of) {
  return guarded(c, [&] {
    *D = c->D;
    if (subdomain_of) std::memcpy(subdomain_of, c->h_sub_of_old.data(), sizeof(int64_t) * c->N);
  });
}

static void fill_records(const LoopResult& R, mp_iter_record* recs, int64_t cap, int64_t* n_recs,
                         int32_t* converged, uint32_t* flags) {
  int64_t n = (int64_t)R.recs.size();
  if (recs) std::memcpy(recs, R.recs.data(), sizeof(mp_iter_record) * std::min(n, cap));
  if (n_recs) *n_recs = n;
  if (converged) *converged = R.converged ? 1 : 0;
  if (flags) *flags = R.flags;
}

int mp_advance(mp_ctx* c, const double* x, const double* v, const double* x_tilde, double h, double* x_out,
               double* v_out, mp_iter_record* recs, int64_t cap, int64_t* n_recs, int32_t* converged,
               uint32_t* flags) {
  return guarded(c, [&] {
    each_shard(c, [&](mp_ctx* sc) {
      upload_vec_new(sc, x, sc->x);
      upload_vec_new(sc, x_tilde, sc->xt);
    });
    LoopResult R;
    advance_loop(c, h, R);
    download_vec_old(c, c->x, x_out);
    download_vec_old(c, c->vel, v_out);
    fill_records(R, recs, cap, n_recs, converged, flags);
  });
}

int mp_step(mp_ctx* c, const double* x, const double* v, double h, double* x_out, double* v_out,
            mp_iter_record* recs, int64_t cap, int64_t* n_recs, int32_t* converged, uint32_t* flags) {
  return guarded(c, [&] {
    each_shard(c, [&](mp_ctx* sc) {
      upload_vec_new(sc, x, sc->x);
      upload_vec_new(sc, v, sc->vel);
      prepare_on(sc, h);
    });
    LoopResult R;
    advance_loop(c, h, R);
    download_vec_old(c, c->x, x_out);
    download_vec_old(c, c->vel, v_out);
    fill_records(R, recs, cap, n_recs, converged, flags);
  });
}

// device-resident variant: x, v stay on the device between calls (bench)
int mp_step_device(mp_ctx* c, double h, mp_iter_record* recs, int64_t cap, int64_t* n_recs, int32_t* converged,
                   uint32_t* flags) {
  return guarded(c, [&] {
    each_shard(c, [&](mp_ctx* sc) { prepare_on(sc, h); });
    LoopResult R;
    advance_loop(c, h, R);
    fill_records(R, recs, cap, n_recs, converged, flags);
  });
}

int mp_set_state(mp_ctx* c, const double* x, const double* v) {
  return guarded(c, [&] {
    each_shard(c, [&](mp_ctx* sc) {
      upload_vec_new(sc, x, sc->x);
      upload_vec_new(sc, v, sc->vel);
      sync_stream(sc);
    });
  });
}

int mp_get_state(mp_ctx* c, double* x, double* v) {
  return guarded(c, [&] {
    if (x) download_vec_old(c, c->x, x);
    if (v) download_vec_old(c, c->vel, v);
  });
}

int mp_shards(mp_ctx* c) { return c ? c->nshards : 0; }

int mp_broad_phase(mp_ctx* c, const double* x, double motion_bound, double d_hat, int64_t* pt, int64_t pt_cap,
                   int64_t* n_pt, int64_t* ee, int64_t ee_cap, int64_t* n_ee) {
  return guarded(c, [&] {
    single_gpu_only(c);
    *n_pt = 0;
    *n_ee = 0;
    if (c->F == 0) return;
    upload_vec_new(c, x, c->x);
    BpGrid B = build_bp(c, c->x, motion_bound, d_hat);
    int64_t npt = 0;
    BpOut O{};
    ContactParams CP{};
    CcdParams CC{};
    const int64_t n = run_bp<BP_RAW>(c, c->x, B, O, CP, CC, nullptr, 3, &npt);
    std::vector<int> a(n), b(n);
    if (n) {
      CUDA_CHECK(cudaMemcpyAsync(a.data(), c->grid.pa.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
      CUDA_CHECK(cudaMemcpyAsync(b.data(), c->grid.pb.p, n * 4, cudaMemcpyDeviceToHost, c->stream));
      sync_stream(c);
    }
    // PT rows (original vertex id, triangle), EE rows (edge i, edge j); sorted
    std::vector<std::pair<int64_t, int64_t>> pt_rows(npt), ee_rows(n - npt);
    for (int64_t i = 0; i < npt; ++i) pt_rows[i] = {c->h_new2old[a[i]], b[i]};
    for (int64_t i = npt; i < n; ++i) ee_rows[i - npt] = {a[i], b[i]};
    std::sort(pt_rows.begin(), pt_rows.end());
    std::sort(ee_rows.begin(), ee_rows.end());
    *n_pt = (int64_t)pt_rows.size();
    *n_ee = (int64_t)ee_rows.size();
    if (pt)
      for (int64_t i = 0; i < *n_pt && i < pt_cap; ++i) {
        pt[2 * i] = pt_rows[i].first;
        pt[2 * i + 1] = pt_rows[i].second;
      }
    if (ee)
      for (int64_t i = 0; i < *n_ee && i < ee_cap; ++i) {
        ee[2 * i] = ee_rows[i].first;
        ee[2 * i + 1] = ee_rows[i].second;
      }
  });
}

static void download_table(mp_ctx* c, PairTable& t, int64_t cap, int64_t* n, int64_t* verts, uint8_t* is_pt,
                           double* d, double* grad, double* k) {
  const int64_t m = t.count;
  *n = m;
  if (m == 0 || cap < m) return;
  std::vector<int4> v(m);
  std::vector<int> ip(m);
  CUDA_CHECK(cudaMemcpyAsync(v.data(), t.verts.p, m * sizeof(int4), cudaMemcpyDeviceToHost, c->stream));
  CUDA_CHECK(cudaMemcpyAsync(ip.data(), t.is_pt.p, m * 4, cudaMemcpyDeviceToHost, c->stream));
  if (d) CUDA_CHECK(cudaMemcpyAsync(d, t.d.p, m * 8, cudaMemcpyDeviceToHost, c->stream));
  if (grad) CUDA_CHECK(cudaMemcpyAsync(grad, t.grad.p, m * 96, cudaMemcpyDeviceToHost, c->stream));
  if (k) CUDA_CHECK(cudaMemcpyAsync(k, t.k.p, m * 8, cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  for (int64_t i = 0; i < m; ++i) {
    const int id[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
    if (verts)
      for (int a = 0; a < 4; ++a) verts[4 * i + a] = c->h_new2old[id[a]];
    if (is_pt) is_pt[i] = (uint8_t)ip[i];
  }
}

int mp_constraint_set(mp_ctx* c, const double* x, int64_t cap, int64_t* n, int64_t* verts, uint8_t* is_pt,
                      double* d, double* grad, double* k) {
  return guarded(c, [&] {
    single_gpu_only(c);
    upload_vec_new(c, x, c->x);
    constraint_set(c, c->x);
    download_table(c, c->cur, cap, n, verts, is_pt, d, grad, k);
  });
}

int mp_gradient(mp_ctx* c, const double* x, const double* x_tilde, double h, double* g) {
  return guarded(c, [&] {
    single_gpu_only(c);
    upload_vec_new(c, x, c->x);
    upload_vec_new(c, x_tilde, c->xt);
    constraint_set(c, c->x);
    gradient(c, c->x, c->xt, h, c->g);
    download_vec_old(c, c->g, g);
  });
}

int mp_energy(mp_ctx* c, const double* x, const double* x_tilde, double h, double* e) {
  return guarded(c, [&] {
    single_gpu_only(c);
    upload_vec_new(c, x, c->x);
    upload_vec_new(c, x_tilde, c->xt);
    constraint_set(c, c->x);
    *e = energy(c, c->x, c->xt, h);
  });
}

int mp_snapshot(mp_ctx* c, const double* x, double h, int build_mas) {
  return guarded(c, [&] {
    single_gpu_only(c);
    upload_vec_new(c, x, c->x);
    constraint_set(c, c->x);
    snapshot(c, c->x, h, build_mas != 0);
    sync_stream(c);
  });
}

int mp_hvp(mp_ctx* c, const double* vec, int with_updates, double* out) {
  return guarded(c, [&] {
    single_gpu_only(c);
    if (!c->have_snapshot) throw MpError(MP_ERR_CONFIG, "no snapshot: call mp_snapshot first");
    upload_vec_new(c, vec, c->tmp);
    hvp(c, c->tmp, c->hv, with_updates != 0);
    download_vec_old(c, c->hv, out);
  });
}

int mp_precond_apply(mp_ctx* c, const double* g, int with_updates, double* z) {
  return guarded(c, [&] {
    single_gpu_only(c);
    if (!c->have_mas) throw MpError(MP_ERR_CONFIG, "no MAS hierarchy: call mp_snapshot(build_mas=1) first");
    upload_vec_new(c, g, c->g);
    precond_apply(c, c->g, c->z, with_updates != 0);
    download_vec_old(c, c->z, z);
  });
}

int mp_update_at(mp_ctx* c, const double* x, int64_t* n_candidates, int64_t* n_touched) {
  return guarded(c, [&] {
    single_gpu_only(c);
    if (!c->have_snapshot) throw MpError(MP_ERR_CONFIG, "no snapshot: call mp_snapshot first");
    upload_vec_new(c, x, c->tmp);
    constraint_set(c, c->tmp);
    update_build(c);
    sync_stream(c);
    if (n_candidates) *n_candidates = c->n_cand;
    if (n_touched) *n_touched = c->n_touched;
  });
}

int mp_ccd(mp_ctx* c, const double* x, const double* p, double* alpha_d, double* x_new, double* min_alpha,
           int32_t* certified, int64_t* n_pairs, int32_t exact_set) {
  return guarded(c, [&] {
    single_gpu_only(c);
    upload_vec_new(c, x, c->x);
    upload_vec_new(c, p, c->p);
    // max |p| over all components (ccd.py:225), from the caller's array
    const int64_t n3 = 3 * c->N;
    double pinf = 0.0;
    for (int64_t i = 0; i < n3; ++i) pinf = std::max(pinf, std::fabs(p[i]));
    CcdResult R = ccd_clamp(c, c->x, c->p, pinf, c->cfg.ccd_per_subdomain != 0, c->tmp, exact_set != 0);
    if (alpha_d)
      CUDA_CHECK(cudaMemcpyAsync(alpha_d, c->alpha_d.p, c->D * 8, cudaMemcpyDeviceToHost, c->stream));
    download_vec_old(c, c->tmp, x_new);
    *min_alpha = R.min_alpha;
    *certified = R.certified ? 1 : 0;
    *n_pairs = R.n_pairs;
  });
}

int mp_coarse_matrix(mp_ctx* c, int level, double* out, int64_t cap, int64_t* n) {
  return guarded(c, [&] {
    single_gpu_only(c);
    if (level < 1 || level > c->n_levels) throw MpError(MP_ERR_CONFIG, "no such coarse level");
    CoarseLevel& L = *c->levels[level - 1];
    *n = L.n;
    if (!out || cap < (int64_t)L.n * L.n) return;
    if (!c->keep_coarse || !L.keep.p) throw MpError(MP_ERR_CONFIG, "enable MP_OPT_KEEP_COARSE before the build");
    for (auto* l : c->levels) CUDA_CHECK(cudaStreamSynchronize(l->st));
    CUDA_CHECK(cudaMemcpy(out, L.keep.p, sizeof(double) * (size_t)L.n * L.n, cudaMemcpyDeviceToHost));
  });
}

int mp_ccd_pairs(mp_ctx* c, int64_t cap, int64_t* n, int64_t* verts, uint8_t* is_pt, double* alpha) {
  return guarded(c, [&] {
    single_gpu_only(c);
    const int64_t m = c->n_ccd;
    *n = m;
    if (m == 0 || cap < m) return;
    std::vector<int4> v(m);
    std::vector<int> ip(m);
    CUDA_CHECK(cudaMemcpyAsync(v.data(), c->ccd_verts.p, m * sizeof(int4), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(ip.data(), c->ccd_ispt.p, m * 4, cudaMemcpyDeviceToHost, c->stream));
    if (alpha) CUDA_CHECK(cudaMemcpyAsync(alpha, c->ccd_alpha.p, m * 8, cudaMemcpyDeviceToHost, c->stream));
    sync_stream(c);
    for (int64_t i = 0; i < m; ++i) {
      const int id[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
      if (verts)
        for (int a = 0; a < 4; ++a) verts[4 * i + a] = c->h_new2old[id[a]];
      if (is_pt) is_pt[i] = (uint8_t)ip[i];
    }
  });
}

}  // extern "C"
