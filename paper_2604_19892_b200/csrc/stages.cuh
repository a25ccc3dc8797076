// stages.cuh -- host drivers of the device stages: gradient, energy,
// snapshot (H_base + MAS build), update (classify / Top-K / Woodbury),
// preconditioner apply and HVP.
#pragma once

#include "ccd.cuh"
#include "coarse.cuh"
#include "group.cuh"
#include "elastic.cuh"
#include "mas.cuh"
#include "ops.cuh"

#define WOODBURY_KMAX 48

// ALGORITHMIC bytes per stage invocation: compulsory
// unique HBM traffic, FP64 = 8 B, ids int32.
static double gradient_bytes(const mp_ctx* c) {
  return 81.0 * c->N + 113.0 * c->T + 17.0 * c->cur.count;
}
static double mas_apply_bytes(const mp_ctx* c) {
  double b = 8.0 * (double)c->D * (double)cyc_size(c->m) + 48.0 * c->N;
  for (int l = 0; l < c->n_levels; ++l) b += 8.0 * (double)cyc_size(c->levels[l]->n);
  return b;
}
static double hvp_bytes(const mp_ctx* c, bool with_cands) {
  double pairs = (double)c->base.count + (with_cands ? (double)c->n_cand : 0.0);
  return 76.0 * c->nnzb + 4.0 * (c->N + 1) + 48.0 * c->N + 116.0 * pairs;
}
static double hessian_bytes(const mp_ctx* c) {
  return 33.0 * c->N + 113.0 * c->T + 72.0 * c->nnzb;
}


// energy.gradient (energy.py:357-370) with the current constraint set
static void gradient(mp_ctx* c, const double* x, const double* xt, double h, double* g) {
  const int64_t nc = c->cur.count;
  if (nc) {
    c->cbuf.ensure(12 * (size_t)nc);
    k_contact_grad_rows<<<grid_for(nc, 128), 128, 0, c->stream>>>(nc, c->cur.d, c->cur.grad, c->d_hat, c->kappa,
                                                                   c->cbuf);
    LAUNCH_CHECK();
  }
  gradient_gather(c, x, xt, h, g, nc ? c->inc_cur.off.p : nullptr, c->inc_cur.val2.p, c->cbuf.p);
}

// energy.incremental_potential (energy.py:346-354)
static double energy(mp_ctx* c, const double* x, const double* xt, double h) {
  const int nb = 64;
  c->red_part.ensure(4 * nb);
  CUDA_CHECK(cudaMemsetAsync(c->red_part.p, 0, sizeof(double) * 4 * nb, c->stream));
  k_inertia_energy<<<nb, 256, 0, c->stream>>>(c->N, x, xt, c->mass, c->red_part.p);
  LAUNCH_CHECK();
  if (c->T_snh) {
    k_tet_energy<2><<<nb, 256, 0, c->stream>>>(0, c->T_snh, c->tets, c->tetp, x, c->red_part.p + nb);
    LAUNCH_CHECK();
  }
  if (c->T_arap) {
    k_tet_energy<1><<<nb, 256, 0, c->stream>>>(c->T_snh, c->T_arap, c->tets, c->tetp, x, c->red_part.p + 3 * nb);
    LAUNCH_CHECK();
  }
  if (c->cur.count) {
    k_contact_energy<<<nb, 256, 0, c->stream>>>(c->cur.count, c->cur.d, c->d_hat, c->kappa, c->red_part.p + 2 * nb);
    LAUNCH_CHECK();
  }
  std::vector<double> part(4 * nb);
  CUDA_CHECK(cudaMemcpyAsync(part.data(), c->red_part.p, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int q = 0; q < 4; ++q)
    for (int b = 0; b < nb; ++b) s[q] += part[q * nb + b];
  return 0.5 * s[0] + h * h * (s[1] + s[3]) + s[2];
}

static void copy_table(mp_ctx* c, PairTable& s, PairTable& d) {
  int64_t n = s.count;
  d.ensure(n > 0 ? n : 1);
  d.count = n;
  if (!n) return;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
  };
  cp(d.khi.p, s.khi.p, n * 8);
  cp(d.klo.p, s.klo.p, n * 8);
  cp(d.verts.p, s.verts.p, n * sizeof(int4));
  cp(d.d.p, s.d.p, n * 8);
  cp(d.k.p, s.k.p, n * 8);
  cp(d.nrm.p, s.nrm.p, n * 8);
  cp(d.grad.p, s.grad.p, n * 96);
  cp(d.is_pt.p, s.is_pt.p, n * 4);
}

static int read_status(mp_ctx* c, int* dev) {
  int h = 0;
  CUDA_CHECK(cudaMemcpyAsync(&h, dev, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  return h;
}

// sym(M^-1) of a coarse level's dense SPD matrix, packed in the cyclic
// layout, on the level's own stream: the coarse-level _spd_inverse
// (mas.py:84-90, :167) as one persistent cooperative kernel
// (coarse.cuh k_coarse_sweep, one grid barrier per 32-pivot panel).
static void dense_spd_inverse(mp_ctx* c, CoarseLevel& L, int* status) {
  (void)c;
  const int n = L.n, nT = (n + CS_TB - 1) / CS_TB;
  L.inv.ensure((size_t)cyc_size(n));
  L.cs_tiles.ensure((size_t)nT * (nT + 1) / 2 * 1024);
  L.cs_col.ensure(2 * (size_t)nT * 1024);
  L.cs_pm.ensure((size_t)nT * 1024);
  L.cs_diag.ensure((size_t)nT * 1024);
  L.cs_bar.zero(2, L.st);
  static int max_ctas = 0;
  if (!max_ctas) {
    int dev = 0, sms = 0, per = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coarse_sweep, CS_THREADS, coarse_sweep_smem()));
    max_ctas = std::max(1, sms * std::max(1, per));
  }
  // every unit its own CTA (+ the lookahead CTA); capping the grid to leave
  // SMs to the level-0 sweep measured slower (64 CTAs 973 us,
  // 96 CTAs 920 us per C2 build)
  const int grid = std::max(1, std::min(L.n_units + 1, max_ctas));
  static const int prof = getenv("MP_CS_PROF") ? 1 : 0;
  CoarseSweepArgs A{n, nT, L.n_units, L.cs_units.p, L.cs_ch, L.dense.p, L.cs_tiles.p, L.cs_col.p, L.inv.p, status,
                    L.cs_bar.p, L.cs_pm.p, L.cs_diag.p, prof};
  void* args[] = {&A};
  CUDA_CHECK(cudaLaunchCooperativeKernel((const void*)k_coarse_sweep, dim3(grid), dim3(CS_THREADS), args,
                                         coarse_sweep_smem(), L.st));
  if (g_launch_counter) ++(*g_launch_counter);
}

// the non-SPD flags of the last MAS build (their readback must have completed:
// after a stream sync) -- cho_factor's failure (mas.py:86-88)
static void mas_flags_check(mp_ctx* c) {
  if (!c->mas_flags_pending) return;
  c->mas_flags_pending = false;
  if (group_or(c, c->h_mas_flags[0])) throw MpError(MP_ERR_NON_SPD_SUBDOMAIN, "subdomain block not SPD");
  for (int q = 1; q < 5; ++q)
    if (c->h_mas_flags[q]) throw MpError(MP_ERR_NON_SPD_SUBDOMAIN, "coarse level not SPD");
}

// build_hierarchy (mas.py:138-179) from the BSR + base contacts
static unsigned sym_tiles(int n) {
  const int64_t nt = (n + 31) / 32;
  return (unsigned)(nt * (nt + 1) / 2);
}

// MP_MAS_TRACE=1: a CUDA-event timeline of every 50th MAS build on stderr
// (assembly and sweep end of each coarse level, level-0 sweep end, readback)
struct MasTrace {
  bool on = false;
  cudaEvent_t e[16];
  int ne = 0;
  const char* name[16];
  cudaStream_t st0 = nullptr;
  explicit MasTrace(cudaStream_t s) : st0(s) {
    static const bool want = getenv("MP_MAS_TRACE") != nullptr;
    static int64_t calls = 0;
    on = want && (calls++ % 50 == 0);
    if (on) mark("start", s);
  }
  void mark(const char* what, cudaStream_t s) {
    if (!on || ne >= 16) return;
    CUDA_CHECK(cudaEventCreate(&e[ne]));
    CUDA_CHECK(cudaEventRecord(e[ne], s));
    name[ne++] = what;
  }
  ~MasTrace() {
    if (!on) return;
    cudaEventSynchronize(e[ne - 1]);
    fprintf(stderr, "mas_build:");
    for (int i = 1; i < ne; ++i) {
      float ms = 0.f;
      cudaEventSynchronize(e[i]);
      cudaEventElapsedTime(&ms, e[0], e[i]);
      fprintf(stderr, "  %s %.1f", name[i], 1e3 * ms);
    }
    fprintf(stderr, " us\n");
    for (int i = 0; i < ne; ++i) cudaEventDestroy(e[i]);
  }
};

static void mas_build(mp_ctx* c) {
  const int m = c->m;
  const int64_t D = c->D;
  MasTrace mt(c->stream);
  if (mt.on) fprintf(stderr, "mas_build: %lld contacts, coarse n %d\n", (long long)c->base.count,
                     c->n_levels ? c->levels[0]->n : 0);
  static const char* asm_name[4] = {"asm1", "asm2", "asm3", "asm4"};
  static const char* inv_name[4] = {"inv1", "inv2", "inv3", "inv4"};
  // coarse levels: own streams, concurrent with the level-0 blocks below
  CUDA_CHECK(cudaMemsetAsync(c->counters.p + 3, 0, 8 * sizeof(int), c->stream));
  const int64_t nc = c->base.count;
  CUDA_CHECK(cudaEventRecord(c->ev_bsr, c->stream));
  // assembly: the first coarse level from the BSR (static gather map) plus
  // the contact terms (fixed point); every further level from the previous
  // level's dense matrix before that one is swept in place
  for (int l = 0; l < c->n_levels; ++l) {
    CoarseLevel& L = *c->levels[l];
    cudaStream_t st = L.st;
    if (l == 0) {
      CUDA_CHECK(cudaStreamWaitEvent(st, c->ev_bsr, 0));
      if (nc) {
        // contact terms on the level's second stream, beside the BSR gather
        CUDA_CHECK(cudaStreamWaitEvent(L.st2, c->ev_bsr, 0));
        // the fixed-point unit (off the level-0 sweep's stream)
        c->fx_scale.ensure(2 + FX_PARTS);
        k_fx_scale_part<<<FX_PARTS, 256, 0, L.st2>>>(nc, c->base.k, c->base.nrm, c->fx_scale.p + 2);
        LAUNCH_CHECK();
        k_fx_scale<<<1, 32, 0, L.st2>>>(c->fx_scale.p + 2, c->fx_scale);
        LAUNCH_CHECK();
        mt.mark("fx_scale", L.st2);
        L.fx_acc.zero(2 * (size_t)L.n * L.n, L.st2);
        k_contact_coarse<<<grid_for(16 * nc, 128), 128, 0, L.st2>>>(nc, c->base.verts, c->base.grad, c->base.k, c->N,
                                                                    L.span, L.n, c->fx_scale, L.fx_acc);
        LAUNCH_CHECK();
        CUDA_CHECK(cudaEventRecord(L.ev_w, L.st2));
        mt.mark("contact1", L.st2);
      }
      L.dense.zero((size_t)L.n * L.n, st);
      if (L.nblk) {
        k_coarse_gather<<<grid_for(32 * (int64_t)L.nblk, 128), 128, 0, st>>>(L.nblk, L.cb_key, L.cb_off, L.cb_slot,
                                                                             c->bsr, L.A, c->N, L.span, L.n, L.dense);
        LAUNCH_CHECK();
        mt.mark("gather1", st);
      }
      if (nc) CUDA_CHECK(cudaStreamWaitEvent(st, L.ev_w, 0));
      k_sym_lower<<<sym_tiles(L.n), 256, 0, st>>>(L.n, L.dense, nc ? L.fx_acc.p : nullptr, c->fx_scale.p);
    } else {
      CoarseLevel& F = *c->levels[l - 1];
      CUDA_CHECK(cudaStreamWaitEvent(st, F.ev_asm, 0));
      L.dense.ensure((size_t)L.n * L.n);
      k_coarse_up<<<grid_for((int64_t)L.n * L.n, 256), 256, 0, st>>>(L.A, c->cfg.coarse_block, F.A, F.dense, F.n,
                                                                     c->N, L.span, F.span, L.dense);
      LAUNCH_CHECK();
      k_sym_lower<<<sym_tiles(L.n), 256, 0, st>>>(L.n, L.dense, nullptr, nullptr);
    }
    LAUNCH_CHECK();
    CUDA_CHECK(cudaEventRecord(L.ev_asm, st));
    mt.mark(asm_name[std::min(l, 3)], st);
  }
  for (int l = 0; l < c->n_levels; ++l) {
    CoarseLevel& L = *c->levels[l];
    if (l + 1 < c->n_levels) CUDA_CHECK(cudaStreamWaitEvent(L.st, c->levels[l + 1]->ev_asm, 0));
    L.inv.ensure((size_t)cyc_size(L.n));
    if (c->keep_coarse) {
      L.keep.ensure((size_t)L.n * L.n);
      CUDA_CHECK(cudaMemcpyAsync(L.keep.p, L.dense.p, sizeof(double) * (size_t)L.n * L.n, cudaMemcpyDeviceToDevice,
                                 L.st));
    }
    if (l == 0) timer_begin(c, MP_STAGE_COARSE_INV, L.st);
    dense_spd_inverse(c, L, c->counters.p + 4 + std::min(l, 3));
    // work: the padded order's (32 nT)^3 FMAs of the panel sweep (2 flops each)
    if (l == 0) timer_end(c, MP_STAGE_COARSE_INV, 2.0 * std::pow(32.0 * ((L.n + 31) / 32), 3.0), L.st);
    CUDA_CHECK(cudaEventRecord(L.done, L.st));
    mt.mark(inv_name[std::min(l, 3)], L.st);
  }
  // level 0: one CTA per subdomain assembles M_d in smem and sweeps it
  c->Bblk.ensure((size_t)D * cyc_size(m));
  c->Mblk.ensure((size_t)D * cyc_size(m));
  // (a shard sweeps its owned subdomains only).  The level-0 sweep starts
  // after the coarse assembly: its 2 CTAs per SM otherwise hold every SM for
  // ~100 us and the assembly chain (the critical path into the coarse
  // inverse) waits behind them (MP_MAS_TRACE: assembly 290 us -> see DESIGN)
  // the solver loop's gradient (independent of the MAS) runs here, on the
  // main stream, while the coarse assembly runs on the level streams
  if (c->mas_overlap) {
    auto fn = std::move(c->mas_overlap);
    c->mas_overlap = nullptr;
    fn();
  }
  if (c->n_levels) CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->levels[c->n_levels - 1]->ev_asm, 0));
  if (c->own_d1 > c->own_d0) {
    timer_begin(c, MP_STAGE_MAS_SWEEP0);
    k_mas_sweep<<<(unsigned)(c->own_d1 - c->own_d0), 256, sizeof(double) * m * m, c->stream>>>(
        D, c->N, c->bs, m, c->pinned, nc ? c->inc_base.off.p : nullptr, c->inc_base.val2.p, c->base.verts,
        c->base.grad, c->base.k, c->rowptr, c->slot_row, c->cols, c->bsr, c->Mblk, c->Bblk, c->counters.p + 3,
        c->own_d0);
    LAUNCH_CHECK();
    // work: the sweep operator's m^3 FMAs per subdomain (2 flops each)
    timer_end(c, MP_STAGE_MAS_SWEEP0, 2.0 * (double)m * m * m * (double)(c->own_d1 - c->own_d0));
    mt.mark("sweep0", c->stream);
  }
  for (int l = 0; l < c->n_levels; ++l) CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->levels[l]->done, 0));
  mt.mark("joined", c->stream);
  // one readback of every level's non-SPD flag (counters 3..7); the solver
  // loop checks it at its next sync (mas_flags_check) instead of syncing here
  CUDA_CHECK(cudaMemcpyAsync(c->h_mas_flags, c->counters.p + 3, 5 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  c->mas_flags_pending = true;
  if (!c->defer_mas_check) {
    sync_stream(c);
    mas_flags_check(c);
  }
  c->have_mas = true;
}

// ---------------------------------------------------------------------------
// 3x3 block Jacobi baseline (solver.py:207-246): per vertex, the diagonal
// block of H_base (BSR diagonal slot + the vertex's own contact terms
// k g_a g_a^T) plus, for the non-rebuild branch, the candidates' u_a u_a^T
// (_blocks_with_updates); Cholesky-checked ("non-spd-block") and inverted.

__device__ __forceinline__ void add_outer3(double B[9], const double* a, const double* b, double s) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int q = 0; q < 3; ++q) B[3 * r + q] += s * a[r] * b[q];
}

__global__ void k_jacobi_blocks(int64_t v0, int64_t v1, const int* __restrict__ diag_slot,
                                const double* __restrict__ bsr, const int* __restrict__ b_off,
                                const int* __restrict__ b_val, const double* __restrict__ b_grad,
                                const double* __restrict__ b_k, const int* __restrict__ q_off,
                                const int* __restrict__ q_val, const double* __restrict__ q_u,
                                double* __restrict__ inv, int* __restrict__ status) {
  const int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= v1) return;
  double B[9];
  const double* d = bsr + 9 * (int64_t)diag_slot[v];
#pragma unroll
  for (int q = 0; q < 9; ++q) B[q] = d[q];
  if (b_off)
    for (int e = b_off[v]; e < b_off[v + 1]; ++e) {
      const int inc = b_val[e];
      const double* g = b_grad + 12 * (int64_t)(inc >> 2) + 3 * (inc & 3);
      add_outer3(B, g, g, b_k[inc >> 2]);
    }
  if (q_off)
    for (int e = q_off[v]; e < q_off[v + 1]; ++e) {
      const int inc = q_val[e];
      const double* u = q_u + 12 * (int64_t)(inc >> 2) + 3 * (inc & 3);
      if (u[0] != 0.0 || u[1] != 0.0 || u[2] != 0.0) add_outer3(B, u, u, 1.0);
    }
  // Cholesky pivots (np.linalg.cholesky's failure), then the inverse
  const double l00 = B[0];
  const double l10 = B[3], l20 = B[6];
  const double p1 = B[4] - l10 * l10 / l00;
  const double p2 = B[8] - l20 * l20 / l00 - (B[7] - l20 * l10 / l00) * (B[7] - l20 * l10 / l00) / p1;
  if (!(l00 > 0.0) || !(p1 > 0.0) || !(p2 > 0.0)) {
    atomicExch(status, 1);
    return;
  }
  const double c00 = B[4] * B[8] - B[5] * B[7], c01 = B[2] * B[7] - B[1] * B[8], c02 = B[1] * B[5] - B[2] * B[4];
  const double det = B[0] * c00 + B[3] * c01 + B[6] * c02;
  const double id = 1.0 / det;
  double* o = inv + 9 * v;
  o[0] = c00 * id; o[1] = c01 * id; o[2] = c02 * id;
  o[3] = (B[5] * B[6] - B[3] * B[8]) * id; o[4] = (B[0] * B[8] - B[2] * B[6]) * id; o[5] = (B[2] * B[3] - B[0] * B[5]) * id;
  o[6] = (B[3] * B[7] - B[4] * B[6]) * id; o[7] = (B[1] * B[6] - B[0] * B[7]) * id; o[8] = (B[0] * B[4] - B[1] * B[3]) * id;
}

__global__ void k_jacobi_apply(int64_t v0, int64_t v1, const double* __restrict__ inv, const double* __restrict__ g,
                               double* __restrict__ z) {
  const int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= v1) return;
  const double* B = inv + 9 * v;
  const double g0 = g[3 * v], g1 = g[3 * v + 1], g2 = g[3 * v + 2];
  z[3 * v] = B[0] * g0 + B[1] * g1 + B[2] * g2;
  z[3 * v + 1] = B[3] * g0 + B[4] * g1 + B[5] * g2;
  z[3 * v + 2] = B[6] * g0 + B[7] * g1 + B[8] * g2;
}

// JacobiPreconditioner(blocks) (solver.py:213-231); with_cands adds the
// update candidates (solver.py:234-241)
static void jacobi_build(mp_ctx* c, bool with_cands) {
  c->jac_inv.ensure(9 * (size_t)c->N);
  CUDA_CHECK(cudaMemsetAsync(c->counters.p + 11, 0, sizeof(int), c->stream));
  const int64_t nv = c->own_v1 - c->own_v0;
  const bool nb = c->base.count > 0, nq = with_cands && c->n_cand > 0;
  if (nv > 0)
    k_jacobi_blocks<<<grid_for(nv, 128), 128, 0, c->stream>>>(
        c->own_v0, c->own_v1, c->diag_slot, c->bsr, nb ? c->inc_base.off.p : nullptr, c->inc_base.val2.p,
        c->base.grad, c->base.k, nq ? c->inc_cand.off.p : nullptr, c->inc_cand.val2.p, c->cand_u, c->jac_inv,
        c->counters.p + 11);
  LAUNCH_CHECK();
  if (group_or(c, read_status(c, c->counters.p + 11))) throw MpError(MP_ERR_NON_SPD_BLOCK, "Jacobi block not SPD");
  c->have_mas = true;  // "a preconditioner is built"
}

// rebuild branch of advance_step (solver.py:323-335): base := cur at x,
// H_base = assemble_base_hessian, MAS hierarchy
static void snapshot(mp_ctx* c, const double* x, double h, bool build_mas) {
  timer_begin(c, MP_STAGE_HESSIAN);
  copy_table(c, c->cur, c->base);
  if (c->inc_cur_rows == c->cur.count && c->cur.count > 0) {
    // base == cur row for row: its incidence CSR is cur's
    const size_t m = 4 * (size_t)c->cur.count;
    c->inc_base.off.ensure(c->N + 1);
    c->inc_base.val2.ensure(m);
    CUDA_CHECK(cudaMemcpyAsync(c->inc_base.off.p, c->inc_cur.off.p, sizeof(int) * (c->N + 1),
                               cudaMemcpyDeviceToDevice, c->stream));
    CUDA_CHECK(cudaMemcpyAsync(c->inc_base.val2.p, c->inc_cur.val2.p, sizeof(int) * m, cudaMemcpyDeviceToDevice,
                               c->stream));
  } else {
    build_inc(c, c->inc_base, c->base.verts, c->base.count);
  }
  if (c->bsr_ahead_pending) {  // assembled ahead on the side stream (bsr_ahead) from the same x
    CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_bsr_ahead, 0));
    c->bsr_ahead_pending = false;
  } else {
    assemble_elastic_bsr(c, x, h);
  }
  timer_end(c, MP_STAGE_HESSIAN, hessian_bytes(c));
  c->have_snapshot = true;
  c->have_mas = false;
  c->have_updates = false;
  c->n_cand = 0;
  c->n_touched = 0;
  if (build_mas) {
    timer_begin(c, MP_STAGE_MAS_BUILD);
    if (c->cfg.preconditioner == MP_PRECOND_JACOBI) jacobi_build(c, false);
    else mas_build(c);
    timer_end(c, MP_STAGE_MAS_BUILD, 0.0);
  }
}

// non-rebuild branch (solver.py:337-346): classify_all, select_top_k,
// build_update, against the snapshot; cur must hold the constraint set at x
static void update_build(mp_ctx* c) {
  classify_all(c, c->cfg.eps_rot);
  c->have_updates = false;
  c->n_touched = 0;
  if (c->cfg.preconditioner == MP_PRECOND_JACOBI) {  // solver.py:344-346
    if (c->cfg.update_strategy != MP_UPDATE_FREEZE && c->have_mas) jacobi_build(c, true);
    return;
  }
  if (c->cfg.update_strategy == MP_UPDATE_FREEZE || c->n_cand == 0 || !c->have_mas) return;
  const int64_t nc = c->n_cand;
  c->ent_count.ensure(nc + 1);
  c->ent_off.ensure(nc + 1);
  k_topk_count<<<grid_for(nc, 128), 128, 0, c->stream>>>(nc, c->cand_verts, c->cand_u, c->bs, c->ent_count);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemsetAsync(c->ent_count.p + nc, 0, sizeof(int), c->stream));
  exclusive_scan(c, c->ent_count, c->ent_off, nc + 1);
  int ne = 0;
  CUDA_CHECK(cudaMemcpyAsync(&ne, c->ent_off.p + nc, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  if (ne == 0) return;
  c->ent_sub.ensure(ne); c->ent_cand.ensure(ne); c->ent_key.ensure(ne);
  c->ent_sub2.ensure(ne); c->ent_cand2.ensure(ne); c->ent_key2.ensure(ne);
  c->sort_idx.ensure(ne); c->sort_idx2.ensure(ne); c->sort_k1.ensure(ne); c->sort_k2.ensure(ne);
  k_topk_fill<<<grid_for(nc, 128), 128, 0, c->stream>>>(nc, c->cand_verts, c->cand_u, c->cand_ds, c->bs, c->ent_off,
                                                        c->ent_sub, c->ent_cand, c->ent_key);
  LAUNCH_CHECK();
  // stable LSD: by descending delta_s, then by subdomain
  k_iota<<<grid_for(ne, 256), 256, 0, c->stream>>>(c->sort_idx, ne);
  LAUNCH_CHECK();
  sort_pairs_u64(c, c->ent_key, c->ent_key2, c->sort_idx, c->sort_idx2, ne, 64);
  // subdomain key of the permuted entries
  k_gather_sub_key<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ent_sub, c->sort_idx2, c->sort_k1);
  LAUNCH_CHECK();
  sort_pairs_u64(c, c->sort_k1, c->sort_k2, c->sort_idx2, c->sort_idx, ne, bits_for((unsigned long long)c->D));
  k_gather_entries<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->sort_idx, c->ent_sub, c->ent_cand, c->ent_sub2,
                                                             c->ent_cand2);
  LAUNCH_CHECK();
  // runs -> touched subdomains
  c->ent_count.ensure(ne + 1);
  c->ent_off.ensure(ne + 1);
  k_topk_runs<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ent_sub2, c->ent_count);
  LAUNCH_CHECK();
  CUDA_CHECK(cudaMemsetAsync(c->ent_count.p + ne, 0, sizeof(int), c->stream));
  exclusive_scan(c, c->ent_count, c->ent_off, ne + 1);
  int nt = 0;
  CUDA_CHECK(cudaMemcpyAsync(&nt, c->ent_off.p + ne, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync_stream(c);
  c->touched_sub.ensure(nt); c->touched_start.ensure(nt); c->touched_len.ensure(nt);
  c->overlay_of.ensure(c->D);
  CUDA_CHECK(cudaMemsetAsync(c->overlay_of.p, 0xff, sizeof(int) * c->D, c->stream));  // -1
  k_topk_touched<<<grid_for(ne, 256), 256, 0, c->stream>>>(ne, c->ent_sub2, c->ent_count, c->ent_off, c->cfg.K,
                                                           c->touched_sub, c->touched_start, c->touched_len,
                                                           c->overlay_of);
  LAUNCH_CHECK();
  c->n_touched = nt;
  const int m = c->m;
  c->overlay.ensure((size_t)nt * cyc_size(m));
  CUDA_CHECK(cudaMemsetAsync(c->counters.p + 4, 0, sizeof(int), c->stream));
  const int kw = c->cfg.K < WOODBURY_KMAX ? c->cfg.K : WOODBURY_KMAX;
  const size_t smem_w = sizeof(double) * ((size_t)m * m + 2 * (size_t)m * kw + (size_t)kw * kw);
  k_woodbury<<<nt, 256, smem_w, c->stream>>>(c->N, c->bs, m, kw, c->Bblk, c->touched_sub, c->touched_start,
                                             c->touched_len, c->ent_cand2, c->cand_verts, c->cand_u, c->overlay,
                                             c->counters.p + 4, c->own_d0, c->own_d1);
  LAUNCH_CHECK();
  if (c->cfg.K > WOODBURY_KMAX) {
    const size_t smem_d = sizeof(double) * 2 * (size_t)m * m;
    k_direct_update<<<nt, 256, smem_d, c->stream>>>(c->N, c->bs, m, c->Mblk, c->touched_sub, c->touched_start,
                                                    c->touched_len, c->ent_cand2, c->cand_verts, c->cand_u,
                                                    WOODBURY_KMAX, c->overlay, c->counters.p + 4, c->own_d0, c->own_d1);
    LAUNCH_CHECK();
  }
  if (group_or(c, read_status(c, c->counters.p + 4))) throw MpError(MP_ERR_CAPACITANCE, "capacitance not SPD");
  c->have_updates = nt > 0;
}

// mas.apply_preconditioner + z[pinned] = 0
static void precond_apply(mp_ctx* c, const double* g, double* z, bool with_updates) {
  if (c->cfg.preconditioner == MP_PRECOND_JACOBI) {  // jac.apply (solver.py:228-229)
    const int64_t nv = c->own_v1 - c->own_v0;
    if (nv > 0) k_jacobi_apply<<<grid_for(nv, 256), 256, 0, c->stream>>>(c->own_v0, c->own_v1, c->jac_inv, g, z);
    LAUNCH_CHECK();
    if (c->nshards > 1 && z != c->z.p) throw MpError(MP_ERR_CONFIG, "group apply writes the context's z only");
    group_allgather(c, [](mp_ctx* p) { return p->z.p; },
                    [](mp_ctx* p, int64_t& lo, int64_t& hi) { lo = 3 * p->own_v0; hi = 3 * p->own_v1; });
    return;
  }
  LevelViews LV{};
  LV.L = c->n_levels;
  // overlap (MP_OPT_APPLY_OVERLAP, default): the level-0 block products
  // (no prolongation) on the side stream, beside the restriction and coarse
  // matvecs on the main stream; k_prolong adds the coarse correction
  const bool overlap = c->overlap_apply && c->n_levels > 0;
  if (overlap) {
    const bool ov0 = with_updates && c->have_updates;
    const int64_t Down0 = c->own_d1 - c->own_d0;
    LevelViews L0{};
    L0.L = 0;
    L0.d0 = c->own_d0;
    CUDA_CHECK(cudaEventRecord(c->ev_g, c->stream));
    CUDA_CHECK(cudaStreamWaitEvent(c->side, c->ev_g, 0));
    double b0 = 8.0 * (double)c->D * (double)cyc_size(c->m) + 48.0 * c->N;
    for (int l = 0; l < c->n_levels; ++l) b0 += 8.0 * c->levels[l]->n;
    timer_begin(c, MP_STAGE_MAS_L0, c->side);
    if (Down0 > 0)
      k_mas_apply_l0_direct<<<(unsigned)Down0, APPLY_THREADS, 0, c->side>>>(
          Down0, c->N, c->bs, c->m, c->Bblk, ov0 ? c->overlay_of.p : nullptr, c->overlay, g, c->pinned, L0, z);
    LAUNCH_CHECK();
    timer_end(c, MP_STAGE_MAS_L0, b0, c->side);
    CUDA_CHECK(cudaEventRecord(c->ev_l0, c->side));
  }
  for (int l = 0; l < c->n_levels; ++l) {
    CoarseLevel& L = *c->levels[l];
    if (l == 0) {
      // owned aggregates, then every shard's slice to every shard (6 doubles per aggregate)
      if (c->own_a1 > c->own_a0)
        k_restrict1<<<(unsigned)(c->own_a1 - c->own_a0), 128, 0, c->stream>>>(c->N, L.span, g, L.rsum, L.r,
                                                                              c->own_a0);
      LAUNCH_CHECK();
      auto rng = [](mp_ctx* p, int64_t& lo, int64_t& hi) { lo = 3 * p->own_a0; hi = 3 * p->own_a1; };
      group_allgather(c, [](mp_ctx* p) { return p->levels[0]->rsum.p; }, rng);
      group_allgather(c, [](mp_ctx* p) { return p->levels[0]->r.p; }, rng);
    } else {
      CoarseLevel& F = *c->levels[l - 1];
      k_restrict_up<<<grid_for(3 * (int64_t)L.A, 128), 128, 0, c->stream>>>(L.A, c->cfg.coarse_block, F.A, c->N,
                                                                             L.span, F.rsum, L.rsum, L.r);
    }
    LAUNCH_CHECK();
    dim3 grid(grid_for(L.n, 128), L.chunks);
    k_coarse_mv<<<grid, 128, 0, c->stream>>>(L.n, L.chunks, L.inv, L.r, L.ypc, L.ypart, L.mv_cnt);
    LAUNCH_CHECK();
    LV.lv[l] = LevelView{L.ypart, L.n, L.span, L.span / c->bs};
  }
  const bool ov = with_updates && c->have_updates;
  const int64_t cpad = (cyc_size(c->m) + 1) & ~1ll;
  const int stages = c->apply_stages == 3 ? 3 : 2;
  const size_t smem = sizeof(double) * (stages * cpad + 2 * 96);
  const int64_t Down = c->own_d1 - c->own_d0;  // this shard's subdomains
  LV.d0 = c->own_d0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(Down, (int64_t)c->apply_ctas_per_sm * 148));
  const int* ovp = ov ? c->overlay_of.p : nullptr;
  // algorithmic bytes of the level-0 kernel: every packed block once, g and
  // z, the coarse corrections it reads (3 A_l doubles per level)
  double l0_bytes = 8.0 * (double)c->D * (double)cyc_size(c->m) + 48.0 * c->N;
  for (int l = 0; l < c->n_levels; ++l) l0_bytes += 8.0 * c->levels[l]->n;
  auto launch_l0 = [&](cudaStream_t s, const LevelViews& V) {
    timer_begin(c, MP_STAGE_MAS_L0, s);
#define L0_ARGS Down, c->N, c->bs, c->m, c->Bblk, ovp, c->overlay, g, c->pinned, V, z
    if (Down <= 0) {
    } else if (c->apply_mode == 2) {
      k_mas_apply_l0_direct<<<(unsigned)Down, APPLY_THREADS, 0, s>>>(L0_ARGS);
    } else if (c->apply_mode == 1) {
      if (stages == 3) k_mas_apply_l0<true, 3><<<grid, APPLY_THREADS, smem, s>>>(L0_ARGS);
      else k_mas_apply_l0<true, 2><<<grid, APPLY_THREADS, smem, s>>>(L0_ARGS);
    } else {
      if (stages == 3) k_mas_apply_l0<false, 3><<<grid, APPLY_THREADS, smem, s>>>(L0_ARGS);
      else k_mas_apply_l0<false, 2><<<grid, APPLY_THREADS, smem, s>>>(L0_ARGS);
    }
#undef L0_ARGS
    LAUNCH_CHECK();
    timer_end(c, MP_STAGE_MAS_L0, l0_bytes, s);
  };
  if (!overlap) {
    launch_l0(c->stream, LV);
  } else {
    // the coarse chain is already queued on the main stream; the level-0
    // block products ran beside it on the side stream; add the coarse
    // prolongation once both are done (same sums in the same order as the
    // fused kernel: acc + C_1^T y_1 + C_2^T y_2)
    CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_l0, 0));
    const int64_t nd = 3 * (c->own_v1 - c->own_v0);
    if (nd > 0)
      k_prolong<<<grid_for(nd, 256), 256, 0, c->stream>>>(c->own_v0, c->own_v1, c->N, c->bs, c->pinned, LV, z);
    LAUNCH_CHECK();
  }
  // z on the owned rows -> every shard (the HVP reads z at every neighbour)
  // (z is always the context's z buffer; every shard swaps its buffers in lockstep)
  if (c->nshards > 1 && z != c->z.p) throw MpError(MP_ERR_CONFIG, "group apply writes the context's z only");
  group_allgather(c, [](mp_ctx* p) { return p->z.p; },
                  [](mp_ctx* p, int64_t& lo, int64_t& hi) { lo = 3 * p->own_v0; hi = 3 * p->own_v1; });
}

// HessianModel.hvp (energy.py:435-440): H_base v + sum u (u^T v)
static void hvp(mp_ctx* c, const double* vec, double* out, bool with_cands) {
  bsr_spmv(c, vec, out);  // owned rows
  const int64_t nb = c->base.count, nq = with_cands ? c->n_cand : 0;
  if (nb) {
    c->rbuf_base.ensure(12 * (size_t)nb);
    k_rank1_rows<<<grid_for(nb, 128), 128, 0, c->stream>>>(nb, c->base.verts, c->base.grad, c->base.k, vec,
                                                           c->rbuf_base);
    LAUNCH_CHECK();
  }
  if (nq) {
    c->rbuf_cand.ensure(12 * (size_t)nq);
    k_rank1_rows<<<grid_for(nq, 128), 128, 0, c->stream>>>(nq, c->cand_verts, c->cand_u, nullptr, vec, c->rbuf_cand);
    LAUNCH_CHECK();
  }
  if (nb || nq) {
    k_inc_gather_add<<<grid_for(32 * (c->own_v1 - c->own_v0), 128), 128, 0, c->stream>>>(
        c->own_v1, c->pinned, nb ? c->inc_base.off.p : nullptr, c->inc_base.val2.p, c->rbuf_base.p,
        nq ? c->inc_cand.off.p : nullptr, c->inc_cand.val2.p, c->rbuf_cand.p, out, c->own_v0);
    LAUNCH_CHECK();
  }
}
