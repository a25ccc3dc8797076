/*
 * maspncg.h -- C ABI of the B200-native MAS-PNCG solver inner loop.
 *
 * The reference (ipcsim, pure Python) has no native FFI; its drop-in
 * boundary is the Python scene/solver API.  Each entry point below replaces
 * one reference function (file:line under /root/reference/pkg/src/ipcsim/)
 * and is bound from Python with ctypes (paper_2604_19892_b200/_native.py;
 * see INTEGRATION.md for the binding a maintainer would add to ipcsim).
 *
 * Conventions
 *   - plain pointers and sizes only; every array argument is HOST memory in
 *     the reference's layout (vertex ids = original ids, positions/vectors
 *     flat (3N,) xyz-interleaved, float64);
 *   - every function returns an mp_status (0 = ok); on failure
 *     mp_last_error(ctx) holds the message and mp_status_code(status) the
 *     reference error code string (errors.py:8-42);
 *   - a context owns one CUDA device, one stream and all device state; it is
 *     not re-entrant (one host thread drives it).
 */
#ifndef MASPNCG_H
#define MASPNCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mp_status {
  MP_OK = 0,
  MP_ERR_PENETRATION = 1,        /* "penetration-detected"   contact.py:41,56,137,149 */
  MP_ERR_NON_SPD_SUBDOMAIN = 2,  /* "non-spd-subdomain"      mas.py:88                */
  MP_ERR_CAPACITANCE = 3,        /* "capacitance-not-spd"    woodbury.py:76           */
  MP_ERR_MODEL_NOT_SPD = 4,      /* "model-not-spd"          solver.py:155,377,389    */
  MP_ERR_PRECOND_NOT_SPD = 5,    /* "precond-not-spd"        solver.py:167            */
  MP_ERR_NON_SPD_BLOCK = 6,      /* "non-spd-block"          solver.py:223            */
  MP_ERR_DEGENERATE = 7,         /* "degenerate-primitive"   geometry.py:68           */
  MP_ERR_CONFIG = 8,             /* "config-error"           errors.py:38-42          */
  MP_ERR_CAPACITY = 9,           /* "capacity-overflow"      (new: device buffers)    */
  MP_ERR_CUDA = 10               /* "cuda-error"             (new)                    */
} mp_status;

/* Static scene, uploaded once.  Mirrors solver.Scene (solver.py:80-114) plus
 * ElasticModel (energy.py:101-149) and SurfaceMesh (geometry.py:377-405). */
typedef struct mp_scene_desc {
  int64_t n_verts;
  const double* rest;        /* (N,3) rest positions (Morton partition input) */
  const double* mass;        /* (N,) lumped masses                             */
  const uint8_t* dirichlet;  /* (N,) pinned mask                               */
  const double* f_ext;       /* (3N,) external force                           */
  int64_t n_tets;
  const int64_t* tets;       /* (T,4)                                          */
  const int8_t* kind;        /* (T,) 0 none, 1 ARAP, 2 SNH                     */
  const double* mu;          /* (T,)                                           */
  const double* lam;         /* (T,)                                           */
  const double* Bm;          /* (T,3,3) inverse rest shape, row-major          */
  const double* vol;         /* (T,) rest volumes                              */
  int64_t n_tris;
  const int64_t* tris;       /* (F,3) surface triangles, reference order       */
  int64_t n_edges;
  const int64_t* edges;      /* (E,2) surface edges, reference order           */
  int64_t n_surf_verts;
  const int64_t* surf_verts; /* (V,) surface vertex ids                        */
  double d_hat;
  double kappa;
} mp_scene_desc;

enum { MP_PRECOND_MAS = 0, MP_PRECOND_JACOBI = 1 };
enum { MP_DIR_SUBSPACE2D = 0, MP_DIR_FR = 1, MP_DIR_PR = 2, MP_DIR_DK = 3, MP_DIR_CD = 4 };
enum { MP_UPDATE_WOODBURY = 0, MP_UPDATE_FREEZE = 1, MP_UPDATE_FULLREBUILD = 2 };

/* solver.SolverConfig (solver.py:48-77), same fields and meaning. */
typedef struct mp_solver_config {
  double eps;
  double delta;
  int64_t iter_max;
  int32_t K;
  int32_t preconditioner;
  int32_t direction_rule;
  int32_t update_strategy;
  int32_t block_size;
  int32_t levels;
  int32_t coarse_block;
  int32_t ccd_per_subdomain;
  double eps_rot;
  double alpha_l;
} mp_solver_config;

/* solver.IterRecord (solver.py:117-129) plus device-side diagnostics. */
typedef struct mp_iter_record {
  int64_t k;
  double grad_norm;
  double z_norm;
  double r;
  int32_t restart;
  int32_t n_contacts;      /* active constraint pairs this iteration       */
  double mu;
  double nu;
  double min_alpha;
  double t_grad_ms;        /* CUDA-event stage times                      */
  double t_dir_ms;
  double t_ccd_ms;
  int32_t n_candidates;    /* rank-one update candidates (non-rebuild)    */
  int32_t n_ccd_pairs;     /* CCD candidate pairs enumerated (saturates at INT32_MAX) */
  int32_t ccd_certified;   /* certify_mixed outcome (1 = mixed step kept) */
  int32_t pad_;
  double energy;           /* incremental potential at the iterate (NaN unless enabled) */
} mp_iter_record;

#define MP_FLAG_NOT_CONVERGED 1u

typedef struct mp_ctx mp_ctx;

/* Create a context on `device`: uploads the scene, builds the Morton
 * partition (mas.py:30-77), the static BSR pattern and surface tables. */
int mp_create(const mp_scene_desc* scene, const mp_solver_config* cfg, int device, mp_ctx** out);
/* A partitioned multi-GPU context ("group"): one shard
 * per entry of dev_ids (entries may repeat a device -- the equivalence tests
 * run two shards on one GPU), each owning a contiguous Morton range of
 * level-1 aggregates (mas.py:63-77).  mp_step / mp_advance / mp_step_device /
 * mp_set_state / mp_get_state run on every shard (one host thread each);
 * the results are bitwise those of a single-GPU context.  The stage taps
 * need a single-GPU context.  n_dev == 1 is mp_create. */
int mp_create_multi(const mp_scene_desc* scene, const mp_solver_config* cfg, int n_dev, const int* dev_ids,
                    mp_ctx** out);
/* number of shards of a context (1 for mp_create) */
int mp_shards(mp_ctx* ctx);
void mp_destroy(mp_ctx* ctx);
int mp_set_config(mp_ctx* ctx, const mp_solver_config* cfg);
const char* mp_status_code(int status);
const char* mp_last_error(mp_ctx* ctx);
/* the context's CUDA stream (cudaStream_t) for external event timing */
void* mp_stream(mp_ctx* ctx);
/* number of subdomains D and the partition's vertex -> subdomain map (N,) */
int mp_partition(mp_ctx* ctx, int64_t* D, int64_t* subdomain_of);

/* solver.step (solver.py:461-464): prepare_step + advance_step.
 * x, v in; x_out, v_out out (3N).  recs: caller array of `cap` records,
 * *n_recs = iterations run (records beyond cap are dropped but counted). */
int mp_step(mp_ctx* ctx, const double* x, const double* v, double h,
            double* x_out, double* v_out, mp_iter_record* recs, int64_t cap,
            int64_t* n_recs, int32_t* converged, uint32_t* flags);
/* solver.advance_step (solver.py:296-458) on a prepared state. */
int mp_advance(mp_ctx* ctx, const double* x, const double* v, const double* x_tilde, double h,
               double* x_out, double* v_out, mp_iter_record* recs, int64_t cap,
               int64_t* n_recs, int32_t* converged, uint32_t* flags);

/* ---- stage taps: one device stage on host inputs, for open-loop parity ---- */

/* geometry.broad_phase (geometry.py:443-503): sorted unique (v, tri) and
 * (edge i, edge j) pairs.  Pass NULL outputs to query counts only. */
int mp_broad_phase(mp_ctx* ctx, const double* x, double motion_bound, double d_hat,
                   int64_t* pt, int64_t pt_cap, int64_t* n_pt,
                   int64_t* ee, int64_t ee_cap, int64_t* n_ee);

/* contact.compute_constraint_set + ConstraintSet.arrays (contact.py:98-155):
 * pairs in key order; verts (C,4) original ids, is_pt (C,), d, grad (C,12),
 * k = kappa b''(d). */
int mp_constraint_set(mp_ctx* ctx, const double* x, int64_t cap, int64_t* n,
                      int64_t* verts, uint8_t* is_pt, double* d, double* grad, double* k);

/* energy.gradient (energy.py:357-370) with the constraint set at x. */
int mp_gradient(mp_ctx* ctx, const double* x, const double* x_tilde, double h, double* g);
/* energy.incremental_potential (energy.py:346-354) with the constraint set at x. */
int mp_energy(mp_ctx* ctx, const double* x, const double* x_tilde, double h, double* e);

/* Freeze a snapshot at x: H_base = assemble_base_hessian (energy.py:373-413)
 * and, if build_mas, the MAS hierarchy (mas.py:138-179). */
int mp_snapshot(mp_ctx* ctx, const double* x, double h, int build_mas);
/* HessianModel.hvp (energy.py:435-440) of the snapshot (+ candidates of the
 * last mp_update_at call when with_updates != 0). */
int mp_hvp(mp_ctx* ctx, const double* vec, int with_updates, double* out);
/* mas.apply_preconditioner (mas.py:182-205) + pinned projection
 * (solver.py:351-352); with_updates applies the Woodbury state of the last
 * mp_update_at call. */
int mp_precond_apply(mp_ctx* ctx, const double* g, int with_updates, double* z);
/* The non-rebuild branch of advance_step (solver.py:336-346) at x against
 * the snapshot: fresh constraint set, classify_all, select_top_k,
 * build_update.  Returns the number of candidates and touched subdomains. */
int mp_update_at(mp_ctx* ctx, const double* x, int64_t* n_candidates, int64_t* n_touched);

/* ccd.per_subdomain_steps + certify_mixed + _apply_ccd (ccd.py:221-320,
 * solver.py:268-280): alpha_d (D,), x_new (3N), min alpha, certificate.
 * exact_set != 0 enumerates (and keeps, for mp_ccd_pairs) the reference's
 * full candidate set, *n_pairs = its size; exact_set == 0 is the solver's
 * tight enumeration (same alpha_d / min / certificate, *n_pairs = pairs
 * enumerated). */
int mp_ccd(mp_ctx* ctx, const double* x, const double* p, double* alpha_d,
           double* x_new, double* min_alpha, int32_t* certified, int64_t* n_pairs,
           int32_t exact_set);

/* The CCD candidate pairs of the last mp_ccd / iteration with their
 * certified steps (ccd.py:244-281 alpha_pair); rows (v,t0,t1,t2) or
 * (a0,a1,b0,b1), original ids, unordered. */
int mp_ccd_pairs(mp_ctx* ctx, int64_t cap, int64_t* n, int64_t* verts, uint8_t* is_pt, double* alpha);

/* The assembled Galerkin matrix M_l = C_l H C_l^T (mas.py:155-168) of coarse
 * level `level` (1-based) as it entered the last build's factorisation,
 * row-major n x n; needs MP_OPT_KEEP_COARSE set before that build.  Pass
 * out = NULL to query n. */
int mp_coarse_matrix(mp_ctx* ctx, int level, double* out, int64_t cap, int64_t* n);

/* Number of kernels this context has launched since creation. */
int64_t mp_launch_count(mp_ctx* ctx);

/* Per-stage CUDA-event timing on the context stream (bench / profiling).
 * mp_stage_timing(ctx, 1) resets and enables; every later stage launch is
 * bracketed by events.  mp_stage_stats returns, for one stage, the summed
 * device time, the number of timed invocations and the summed ALGORITHMIC
 * bytes of those invocations (compulsory unique HBM traffic). */
enum {
  MP_STAGE_GRADIENT = 0,       /* energy.gradient          energy.py:357-370 */
  MP_STAGE_MAS_APPLY = 1,      /* mas.apply_preconditioner mas.py:182-205    */
  MP_STAGE_HVP = 2,            /* HessianModel.hvp         energy.py:435-440 */
  MP_STAGE_CONSTRAINT_SET = 3, /* broad phase + constraint set contact.py:116-165 */
  MP_STAGE_HESSIAN = 4,        /* assemble_base_hessian    energy.py:373-413 */
  MP_STAGE_MAS_BUILD = 5,      /* build_hierarchy          mas.py:138-179    */
  MP_STAGE_UPDATE = 6,         /* classify/top-K/Woodbury  solver.py:337-346 */
  MP_STAGE_CCD = 7,            /* CCD clamp                solver.py:268-280 */
  MP_STAGE_MAS_L0 = 8,         /* the level-0 kernel of the MAS apply alone   */
  MP_STAGE_TET_GRAD = 9,       /* the SNH per-tet gradient kernel alone        */
  MP_STAGE_HOST_WAIT = 10,     /* host wall time blocked on the stream (syncs) */
  MP_STAGE_LOOP = 11,          /* host wall time of advance_step loops         */
  MP_STAGE_MAS_SWEEP0 = 12,    /* the level-0 block sweep kernel alone (work = FP64 flops, not bytes) */
  MP_STAGE_COARSE_INV = 13,    /* the first coarse level's inverse kernel alone (work = FP64 flops)   */
  MP_STAGE_COUNT = 14
};
int mp_stage_timing(mp_ctx* ctx, int enable);

/* Solver options beyond SolverConfig.  MP_OPT_CCD_EXACT_SET: enumerate the
 * reference's full CCD candidate set inside the loop (default 0: the tight
 * set, same results).  MP_OPT_RECORD_ENERGY: evaluate the incremental
 * potential at every iterate into mp_iter_record.energy (default 0).
 * MP_OPT_APPLY_TMA: level-0 MAS apply variant -- 2 (default) direct
 * streaming loads, one CTA per subdomain; 1 TMA bulk staging; 0 per-thread
 * cp.async staging; MP_OPT_APPLY_STAGES (2 or 3) and
 * MP_OPT_APPLY_CTAS (persistent CTAs per SM) tune its pipeline; same results.
 * MP_OPT_BP_FUSED: broad-phase enumeration for the constraint set, CCD and
 * certificate -- 1 (default) one-pass unordered pair lists, 2 constraint-set
 * pair work fused into the grid queries, 0 ordered count/scan/fill lists;
 * same results. */
enum { MP_OPT_CCD_EXACT_SET = 1, MP_OPT_RECORD_ENERGY = 2, MP_OPT_APPLY_TMA = 3, MP_OPT_APPLY_STAGES = 4,
       MP_OPT_APPLY_CTAS = 5, MP_OPT_BP_FUSED = 6, MP_OPT_KEEP_COARSE = 7,
       MP_OPT_APPEND_LIMIT = 8 /* test knob: process-wide one-pass list limit (default and max 2^30; <= 0 resets) */,
       MP_OPT_GRAD_FUSED = 9 /* gradient: 1 one fused per-vertex pass, 0 (default, faster) per-tet scratch + gather; same bits */,
       MP_OPT_APPLY_OVERLAP = 10 /* MAS apply: 1 (default) level 0 beside the coarse chain + prolongation pass, 0 fused; same bits */,
       MP_OPT_CCD_PREFILTER = 11 /* tight CCD: 1 (default) exact relative-motion pair prefilter, 0 off; same results */,
       MP_OPT_CCD_BODIES = 12 /* tight CCD: 1 two passes (same-body / cross-body centres), 0 (default) one global centre; same results */,
       MP_OPT_CCD_LOCAL = 13 /* tight CCD: 1 per-subdomain motion centres when they inflate less, 0 (default) global; same results */,
       MP_OPT_CCD_BVH = 14 /* tight CCD / certificate enumeration: 0 hierarchical grid, 1 motion-aware BVH, 2 (default) per
                              call: the grid unless it is crowded, then the method measured faster; same results */,
       MP_OPT_BVH_TASKS = 15 /* test knob for the BVH's hand-on task lists: > 0 a fixed capacity (a full list makes
                                threads finish their own traversals); < 0 grown as needed up to -value, then the
                                queries split in chunks; 0 (default) grown up to 2^27; same results */ };
int mp_set_option(mp_ctx* ctx, int option, int64_t value);
int mp_stage_stats(mp_ctx* ctx, int stage, double* total_ms, int64_t* count, double* bytes);

/* Message of the last failed mp_create on this thread. */
const char* mp_create_error(void);

/* The coarse-level dense inverse (mas.py:84-90 `_spd_inverse` as used at
 * mas.py:167) on `device`, standalone: inv (n x n, row-major) = sym(A^-1)
 * of the symmetric n x n row-major A; *not_spd = 1 (and inv undefined) where
 * cho_factor would raise non-spd-subdomain.  Test / parity entry point. */
int mp_spd_inverse(int device, int64_t n, const double* A, double* inv, int32_t* not_spd);

/* The penetration checker's triangle-triangle part (cli.py:393-401 with
 * geometry.tri_tri_intersect, geometry.py:686-732) on `device`: the number
 * of intersecting non-adjacent triangle pairs of the surface (x: (N,3),
 * tris: (F,3)) and the smallest triangle index involved (-1 if none).
 * Uniform-grid candidates, O(F) instead of the reference's O(F^2).
 * coplanar_tol = 0 is the reference's rule (coplanar iff every
 * vertex-plane value is exactly 0); > 0 treats pairs coplanar to within
 * coplanar_tol x the longest edge as coplanar (the reference's rule reports
 * disjoint faces that are coplanar to rounding as intersecting). */
int mp_check_intersections(int device, int64_t n_verts, const double* x, int64_t n_tris, const int64_t* tris,
                           double coplanar_tol, int64_t* n_hits, int64_t* first_tri);

/* Change the barrier parameters of a context (Scene.d_hat / kappa); the
 * checker uses a surface-only context with d_hat = its search radius. */
int mp_set_contact(mp_ctx* ctx, double d_hat, double kappa);

/* Host-only: the owned ranges shard `rank` of `nshards` gets in a group
 * (mp_create_multi): out[0..1] vertices [v0, v1) (renumbered, subdomain
 * order), out[2..3] subdomains, out[4..5] level-1 aggregates, out[6..7]
 * reduction chunks.  The unit is the level-1 aggregate (coarse_block
 * subdomains) when a coarse level is built, else the subdomain. */
int mp_shard_range(int64_t n_verts, int32_t block_size, int32_t levels, int32_t coarse_block, int32_t rank,
                   int32_t nshards, int64_t* out);

/* mas.partition_domain (mas.py:63-77) on the host, no GPU needed:
 * subdomain_of (n,) for a Morton partition into blocks of block_size. */
int mp_partition_host(const double* rest, int64_t n, int32_t block_size, int64_t* subdomain_of);

/* Device-resident stepping (the bench's timed path and multi-frame drivers):
 * mp_set_state uploads x, v once; mp_step_device runs prepare_step +
 * advance_step on the resident state; mp_get_state downloads it. */
int mp_set_state(mp_ctx* ctx, const double* x, const double* v);
int mp_get_state(mp_ctx* ctx, double* x, double* v);
int mp_step_device(mp_ctx* ctx, double h, mp_iter_record* recs, int64_t cap, int64_t* n_recs,
                   int32_t* converged, uint32_t* flags);

#ifdef __cplusplus
}
#endif
#endif /* MASPNCG_H */
