// ctx.cuh -- the device context: every piece of solver state lives here,
// device-resident, in subdomain-renumbered vertex order.
//
// Vertex renumbering: the reference's Morton partition (mas.py:63-77) puts
// vertex `old` in subdomain d at rank r of d's sorted vertex list; here that
// vertex gets id new = d*bs + r.  A subdomain is therefore a contiguous run
// of vertices and dofs, coarse aggregates are contiguous runs of subdomains,
// and subdomain_of(new) = new / bs.  Dof order inside a subdomain equals the
// reference's B_d dof order (ascending original id, mas.py:74).
#pragma once


#include <string>
#include <thread>
#include <mutex>
#include <condition_variable>
#include <atomic>
#include <chrono>
#include <functional>
#include <vector>

#include "common.cuh"

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  // grow to at least `count` elements, geometrically (cudaFree / cudaMalloc
  // synchronise the device: buffers sized by contact counts must not
  // reallocate every time a count creeps up); contents are NOT preserved
  void ensure(size_t count) {
    if (count <= n && p) return;
    const size_t grown = n + n / 2;
    release();
    size_t c = count < 1 ? 1 : count;
    if (grown > c) c = grown;
    CUDA_CHECK(cudaMalloc(&p, c * sizeof(T)));
    n = c;
  }
  void upload(const T* host, size_t count, cudaStream_t s) {
    ensure(count);
    if (count) CUDA_CHECK(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void zero(size_t count, cudaStream_t s) {
    ensure(count);
    CUDA_CHECK(cudaMemsetAsync(p, 0, count * sizeof(T), s));
  }
  operator T*() const { return p; }
};

// per-tet constant data, 12 doubles (96 B): Bm row-major, vol, mu, lam
struct TetParam {
  double Bm[9];
  double vol, mu, lam;
};

// contact pair table (structure of arrays), key order = reference key order:
// ("ee",(a0,a1),(b0,b1)) < ("pt", v, (t0,t1,t2))  (contact.py:98-113)
struct PairTable {
  DBuf<unsigned long long> khi, klo;  // 128-bit sort key
  DBuf<int4> verts;                   // new vertex ids, canonical order
  DBuf<double> d, k, nrm;             // distance, kappa b''(d), |grad|
  DBuf<double> grad;                  // (C,12) pinned rows zeroed
  DBuf<int> is_pt;
  int64_t count = 0;
  void ensure(size_t c) {
    khi.ensure(c); klo.ensure(c); verts.ensure(c);
    d.ensure(c); k.ensure(c); nrm.ensure(c); grad.ensure(12 * c); is_pt.ensure(c);
  }
};

struct IncCSR {
  DBuf<int> cnt, off;        // (N+1)
  DBuf<int> key, key2, val, val2;  // (4 rows): vertex keys, incidences (val2 sorted)
};

// per-level cell tables of the broad phase (bp.cuh build_bp)
struct BpGridBufs {
  DBuf<int> tri_cnt, tri_start, edge_cnt, edge_start, pt_cnt, pt_start;  // (ncell+1)
  DBuf<int> level;                                                       // (objects)
  DBuf<int> rc;                                                          // (objects*6) reference cells
  DBuf<int> qcnt, qoff;                                                  // per-query pair counts
  DBuf<int> pa, pb;                                                      // reference pair list (PT in append mode)
  DBuf<int> ea, eb;                                                      // append mode: EE list
  DBuf<int> ecell, tri_ent, edge_ent, pt_ent;                            // (entries)
  DBuf<double> tri_box, edge_box, pt_box;  // (entries*6) the entry's enumeration box, in cell order
};

struct CoarseLevel {
  int A = 0;          // aggregates
  int n = 0;          // 3A dofs
  int span = 0;       // vertices per aggregate (last may be short)
  DBuf<double> dense; // n*n Galerkin matrix, swept in place
  DBuf<double> keep;  // n*n copy of the assembled matrix before the sweep (MP_OPT_KEEP_COARSE)
  DBuf<double> inv;   // cyc_size(n) packed inverse
  DBuf<double> rsum;  // 3A restricted raw sums
  DBuf<double> r;     // 3A restriction C_l g (averages)
  DBuf<double> ypart; // n: M_l^-1 r (sum of the diagonal chunks' partials, fixed order)
  DBuf<double> ypc;   // chunks*n partials
  DBuf<int> mv_cnt;   // per row block: chunks done (the last one reduces)
  DBuf<unsigned long long> fx_acc;  // n*n*2: contact terms, 128-bit fixed point
  DBuf<int> cb_key, cb_off, cb_slot;  // BSR -> M_l gather map: nonzero blocks A*nA+B, their slots
  int nblk = 0;
  // the coarse inverse (coarse.cuh): work units, lower tiles, panel columns, grid barrier
  DBuf<int2> cs_units;
  int n_units = 0;
  int cs_ch = 8;  // column tiles per unit
  DBuf<double> cs_tiles, cs_col, cs_pm, cs_diag;
  DBuf<unsigned> cs_bar;
  int chunks = 1;
  // each coarse level is built on its own stream (st2: its contact terms),
  // concurrently with level 0
  cudaStream_t st = nullptr, st2 = nullptr;
  cudaEvent_t done = nullptr, ev_w = nullptr, ev_u = nullptr, ev_asm = nullptr;
  ~CoarseLevel() {
    for (cudaEvent_t e : {done, ev_w, ev_u, ev_asm})
      if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
    if (st2) cudaStreamDestroy(st2);
  }
};

// CUDA-event timer of one solver stage on the context stream.  Events are
// recorded around the stage's launches; the elapsed time is folded in lazily
// (at the next begin or at readout), after the loop's own per-iteration sync,
// so timing adds no host stall.
struct StageTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  bool pending = false;
  double total_ms = 0.0;
  double bytes = 0.0;   // algorithmic bytes of all timed launches
  int64_t count = 0;
};

struct Group;

struct mp_ctx {
  int device = 0;
  // ---- shard of a multi-GPU group (group.cuh); one GPU: rank 0 of 1 owning everything ----
  Group* grp = nullptr;
  int rank = 0, nshards = 1;
  int64_t own_v0 = 0, own_v1 = 0;  // owned vertices (aligned to level-1 aggregates)
  int64_t own_d0 = 0, own_d1 = 0;  // owned subdomains
  int64_t own_a0 = 0, own_a1 = 0;  // owned level-1 aggregates
  int64_t chunk_v = 32;            // vertices per reduction chunk (= the alignment unit)
  int64_t n_chunks = 1, own_c0 = 0, own_c1 = 1;
  DBuf<double> chunk_part;         // n_chunks * MAX_DOTS chunk partials
  std::vector<double> h_part;      // host copy (single shard) for the ordered chunk sum
  int par_dots = 0, par_flags = 0; // double-buffer parities of the group's host exchange arrays
  bool timing = false;
  bool ccd_exact_set = false;
  bool record_energy = false;
  int apply_mode = 2;        // level-0 apply: 2 direct loads, 1 TMA-staged, 0 cp.async-staged
  int apply_stages = 2;      // level-0 apply pipeline depth (2 or 3)
  int apply_ctas_per_sm = 3; // level-0 apply persistent CTAs per SM
  bool fused_grad = false;  // gradient: one fused per-vertex pass (k_grad_fused; measured slower at C2, 98 vs 74 us) or per-tet scratch + gather (MP_OPT_GRAD_FUSED)
  bool overlap_apply = true;  // MAS apply: level 0 on the side stream beside the coarse chain (MP_OPT_APPLY_OVERLAP)
  cudaStream_t side = nullptr;  // side stream (level-0 apply, elastic H_base ahead) and its events
  cudaEvent_t ev_it = nullptr, ev_bsr_ahead = nullptr;  // bsr_ahead (elastic.cuh)
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;         // iteration start / z ready (t_grad_ms)
  bool bsr_ahead_pending = false;
  bool defer_mas_check = false;      // the solver loop checks the MAS build's flags at its next sync
  std::function<void()> mas_overlap; // launched by mas_build beside the coarse assembly (the loop's gradient)
  bool mas_flags_pending = false;
  int h_mas_flags[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaEvent_t ev_g = nullptr, ev_l0 = nullptr;   // gradient: one fused pass (k_grad_fused) or per-tet scratch + gather (MP_OPT_GRAD_FUSED)
  bool keep_coarse = false;  // keep each coarse level's assembled matrix (mp_coarse_matrix)
  int bp_fused = 1;          // 1: one-pass unordered pair lists, 2: contact work fused into the queries, 0: ordered lists
  StageTimer timers[MP_STAGE_COUNT];
  cudaStream_t stream = nullptr;
  std::string last_error;
  int64_t launches = 0;

  // ---- sizes ----
  int64_t N = 0, T = 0, F = 0, E = 0, V = 0;
  int64_t T_snh = 0, T_arap = 0;  // tets are stored SNH [0, T_snh), ARAP next, then none
  int bs = 32;   // partition block size
  int m = 96;    // dofs per (padded) subdomain block = 3*bs
  int64_t D = 0; // subdomains
  int id_bits = 1;  // bits per vertex id in pair keys
  double d_hat = 0.0, kappa = 0.0;
  mp_solver_config cfg{};

  // ---- host copies of static maps ----
  std::vector<int> h_new2old, h_old2new;
  std::vector<int64_t> h_sub_of_old;  // reference order

  // ---- static device data ----
  DBuf<int> new2old;
  DBuf<double> mass;        // (N)
  DBuf<unsigned char> pinned;
  DBuf<double> f_ext;       // (3N)
  DBuf<int4> tets;          // (T) new ids
  DBuf<TetParam> tetp;
  DBuf<signed char> kind;
  // BSR(3x3) pattern of the elastic + mass Hessian
  int64_t nnzb = 0;
  DBuf<int> rowptr, cols, tet_slot, diag_slot;
  DBuf<double> bsr;         // nnzb*9 values
  std::vector<int> h_rowptr, h_cols;  // host copy of the pattern (coarse gather maps)
  // deterministic assembly (fixed-order gathers instead of atomics)
  DBuf<int> hs_off, hs_val, slot_row;  // BSR slot -> element blocks 16t+4a+b; slot -> row
  DBuf<int> vt_off, vt_val;            // vertex -> tet corners 4t+a
  DBuf<double> fbuf;                   // (T_el,4,3) per-corner elastic forces
  DBuf<double> hbuf;                   // (T_el,10,9) element blocks a <= b
  // surface
  DBuf<int> tri;            // (F*3) new ids, surface order
  DBuf<int> tri_sorted;     // (F*3) new ids ordered by ascending original id
  DBuf<int> edge;           // (E*2) new ids (original order = ascending original id)
  DBuf<int> sverts;         // (V) new ids

  // ---- per-step vectors (3N) ----
  DBuf<double> x, xt, vel, g, g_prev, z, p, Hp, p_prev, Hp_prev, z_prev, hv, x_start, x_best, tmp, tmp2;

  // ---- contact sets ----
  PairTable cur, base, scratch;
  // vertex -> incidences (4 row + corner, ascending) of cur / base / the
  // update candidates: fixed-order per-vertex gathers instead of atomics
  IncCSR inc_cur, inc_base, inc_cand;
  int64_t inc_cur_rows = -1;  // rows of cur that inc_cur indexes (-1: stale)
  DBuf<double> cbuf, rbuf_base, rbuf_cand;  // (rows, 12) per-row terms
  DBuf<double> fx_scale;                   // coarse contact fixed-point unit
  DBuf<double> mid_part;                   // (148, 6) CCD motion midrange partials
  DBuf<int> sort_idx, sort_idx2;
  DBuf<unsigned long long> sort_k1, sort_k2;
  DBuf<unsigned char> cub_tmp;
  // update candidates (classify_all output, key order)
  int64_t n_cand = 0;
  DBuf<int4> cand_verts;
  DBuf<double> cand_u;      // (n_cand, 12)
  DBuf<double> cand_ds;
  DBuf<int> cand_flag, cand_pos;
  DBuf<double> tmp_scale, tmp_ds;
  // top-K entries
  DBuf<int> ent_count, ent_off, ent_sub, ent_cand, ent_sub2, ent_cand2;
  DBuf<unsigned long long> ent_key, ent_key2;
  DBuf<int> touched_sub, touched_start, touched_len, overlay_of;
  int64_t n_touched = 0;
  DBuf<double> overlay;     // n_touched * cyc(m)
  bool have_updates = false;

  // ---- broad phase scratch ----
  DBuf<double> box_flo, box_fhi; // (F+E)*3 reference filter / join boxes
  DBuf<double> box_rlo, box_rhi; // (F+E)*3 raw primitive boxes
  DBuf<double> box_elo, box_ehi; // (F+E+V)*3 enumeration boxes
  DBuf<double> infl;             // (N) per-vertex CCD inflation
  DBuf<int> body;                // (N) connected component (body) of each vertex
  int64_t n_bodies = 1;
  DBuf<unsigned long long> body_mm;  // per-body min / max of the motion (ordered keys)
  DBuf<double> body_cen;             // per-body motion centres + their midrange
  DBuf<double> obj_mot;              // per-object motion (c, m) for the exact CCD prefilter
  bool ccd_prefilter = true;         // MP_OPT_CCD_PREFILTER
  bool ccd_bodies = false;           // MP_OPT_CCD_BODIES: two-pass per-body tight enumeration
  int ccd_bvh = 2;                   // MP_OPT_CCD_BVH: tight CCD enumeration 0 grid, 1 BVH (bvh.cuh), 2 per call
  bool bvh_ready = false;            // class orders built (fixed topology)
  DBuf<int> bvh_tri_order, bvh_edge_order, bvh_key, bvh_val;
  DBuf<float4> bvh_tri_nodes, bvh_edge_nodes;  // BvhNode = 5 float4
  DBuf<int2> bvh_tasks;              // 4 task lists (class x ping-pong) of the load-balanced traversal
  DBuf<unsigned long long> bvh_task_cnt;
  int64_t bvh_task_cap = 0;          // MP_OPT_BVH_TASKS test knob: fixed task-list capacity (0: grown as needed)
  int64_t bvh_task_max = 0;          // largest grown task list (0: BVH_TASKS_MAX; MP_OPT_BVH_TASKS < 0 lowers it)
  DBuf<unsigned long long> crowd_dev;  // grid crowding probe (bp.cuh BP_GRID_AUTO)
  struct EnumTimes {                 // crowded CCD enumerations: ms per log2 crowding bucket, grid / BVH (< 0 unknown)
    double ms[2][32];
    EnumTimes() {
      for (auto& r : ms)
        for (double& v : r) v = -1.0;
    }
  } enum_ms;
  int64_t n_crowded = 0;
  bool ccd_local = false;            // MP_OPT_CCD_LOCAL: per-subdomain motion centres (ccd.cuh local_infl)
  DBuf<double> sub_cen, sub_box, sub_delta, infl2;
  DBuf<unsigned long long> sub_key, sub_key2;
  DBuf<int> sub_id, sub_id2;
  std::vector<double> dscal_h;
  DBuf<int> cell_cnt, cell_off;  // per-primitive covered-cell counts / offsets
  BpGridBufs grid;
  DBuf<int> cand_a, cand_b;      // raw broad-phase pairs (taps)
  DBuf<int> counters;            // device counters
  DBuf<double> dscal;            // device scalars
  DBuf<double> red_part;         // reduction partials

  // ---- MAS ----
  DBuf<double> Bblk;        // D * cyc(m) packed inverses
  DBuf<double> Mblk;        // D * cyc(m) packed subdomain blocks (direct refactor path)
  DBuf<double> jac_inv;     // N * 9 inverse diagonal blocks (Jacobi baseline)
  std::vector<CoarseLevel*> levels;
  int n_levels = 0;
  cudaEvent_t ev_bsr = nullptr;     // H_base ready (coarse streams wait on it)
  bool have_snapshot = false;
  bool have_mas = false;

  // ---- CCD ----
  DBuf<int4> ccd_verts;
  DBuf<int> ccd_ispt;
  DBuf<double> ccd_alpha;   // per pair
  DBuf<double> alpha_d;     // (D)
  int64_t n_ccd = 0;        // stored pair list length (exact-set taps)
  int64_t n_ccd_seen = 0;   // pairs enumerated by the last CCD

  // pinned host staging for scalars
  double sync_wait_ms = 0.0;  // host time blocked in sync_stream (stage timing on)
  int64_t n_sync = 0;
  double loop_ms = 0.0;       // host wall time of advance loops (stage timing on)
  int64_t n_loop = 0;
  double* h_scal = nullptr;
  int* h_cnt = nullptr;
  unsigned long long* h_npairs = nullptr;  // = h_scal[63]
  const double* rb_extra = nullptr;        // device scalar run_bp reads back into h_scal[0]
  DBuf<unsigned long long> n_pairs_dev;    // fused enumeration pair count

  ~mp_ctx();
};

// every host wait on the context stream goes through here: with
// MP_OPT stage timing on, the wall time spent blocked is accumulated
static void sync_stream(mp_ctx* c) {
  if (!c->timing) {
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return;
  }
  auto t0 = std::chrono::steady_clock::now();
  CUDA_CHECK(cudaStreamSynchronize(c->stream));
  c->sync_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->n_sync += 1;
}

static void timer_fold(StageTimer& t) {
  if (!t.pending) return;
  CUDA_CHECK(cudaEventSynchronize(t.b));
  float ms = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&ms, t.a, t.b));
  t.total_ms += ms;
  t.count += 1;
  t.pending = false;
}

static void timer_begin(mp_ctx* c, int id, cudaStream_t s = nullptr) {
  if (!c->timing) return;
  StageTimer& t = c->timers[id];
  timer_fold(t);
  if (!t.a) {
    CUDA_CHECK(cudaEventCreate(&t.a));
    CUDA_CHECK(cudaEventCreate(&t.b));
  }
  CUDA_CHECK(cudaEventRecord(t.a, s ? s : c->stream));
}

static void timer_end(mp_ctx* c, int id, double bytes, cudaStream_t s = nullptr) {
  if (!c->timing) return;
  StageTimer& t = c->timers[id];
  CUDA_CHECK(cudaEventRecord(t.b, s ? s : c->stream));
  t.pending = true;
  t.bytes += bytes;
}
