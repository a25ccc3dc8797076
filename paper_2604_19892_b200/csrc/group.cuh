// group.cuh -- the partitioned multi-GPU solver.
//
// A group is one mp_ctx per GPU ("shard") inside one process, driven by one
// host thread per shard running the SAME control flow (SPMD; every branch
// decision is taken from group-wide scalars, so the shards stay in
// lockstep).  The mesh is partitioned by MAS subdomain (mas.py:63-77): shard
// s owns a contiguous Morton range of level-1 aggregates (whole subdomains,
// whole aggregates), i.e. a contiguous range of renumbered vertices.
//
// Owner-computes: the level-0 MAS build and apply (mas.py:84-90, 182-205),
// the Woodbury build (woodbury.py:46-87), the gradient gather
// (energy.py:357-370), the HVP (energy.py:435-440) and every PNCG dot run on
// the owner only.  Replicated on every shard (identical inputs, identical
// bits): positions and directions, the constraint set, H_base and the
// coarse levels, classification / top-K, CCD.
//
// Exchanges per PNCG iteration, over NVLink peer copies ordered by
// cross-device events (cudaMemcpyPeerAsync; P2P access enabled when the
// devices allow it):
//   * the level-1 restriction C_1 g: 6 doubles per owned aggregate;
//   * z = P g on the owned rows: 3 doubles per owned vertex (the "halo" is
//     the whole vector -- the HVP reads z at every neighbour);
//   * the PNCG scalars: per-chunk partials of the owned chunks (chunk = one
//     level-1 aggregate), summed on the host over ALL chunks in chunk order --
//     the same sums in the same order as on one GPU, so the group's
//     trajectory is bitwise identical to the single-GPU one;
//   * status flags (non-SPD block, capacitance) OR-ed across shards.
#pragma once

#include <exception>

#include "ops.cuh"

struct HostBarrier {
  std::mutex m;
  std::condition_variable cv;
  int n = 1, count = 0;
  uint64_t gen = 0;
  bool aborted = false;
  // false once any shard aborted (its error is reported by the caller)
  bool wait() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) return false;
    const uint64_t g = gen;
    if (++count == n) {
      count = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

#define GROUP_MAX 16

struct Group {
  std::vector<mp_ctx*> sh;
  HostBarrier bar;
  cudaEvent_t ev[GROUP_MAX] = {};   // per shard: its slice is ready
  cudaEvent_t ev2[GROUP_MAX] = {};  // per shard: its peer copies are done
  double* hpart[2] = {nullptr, nullptr};  // pinned, n_chunks * MAX_DOTS (double-buffered by call parity)
  int flags[2][GROUP_MAX] = {};
  double vals[2][GROUP_MAX] = {};
  ~Group() {
    for (double* p : hpart)
      if (p) cudaFreeHost(p);
  }
};

static void group_sync(mp_ctx* c) {
  if (c->nshards > 1 && !c->grp->bar.wait()) throw MpError(MP_ERR_CUDA, "aborted: another shard failed");
}

// Allgather of a role buffer: every shard's owned slice [lo, hi) (elements,
// from rng(shard, lo, hi)) is copied into every other shard's copy.
template <class Buf, class Rng>
static void group_allgather(mp_ctx* c, Buf buf, Rng rng) {
  if (c->nshards <= 1) return;
  Group* G = c->grp;
  CUDA_CHECK(cudaEventRecord(G->ev[c->rank], c->stream));
  group_sync(c);
  for (int q = 0; q < c->nshards; ++q) {
    if (q == c->rank) continue;
    mp_ctx* p = G->sh[q];
    int64_t lo = 0, hi = 0;
    rng(p, lo, hi);
    if (hi <= lo) continue;
    CUDA_CHECK(cudaStreamWaitEvent(c->stream, G->ev[q], 0));
    CUDA_CHECK(cudaMemcpyPeerAsync(buf(c) + lo, c->device, buf(p) + lo, p->device, sizeof(double) * (hi - lo),
                                   c->stream));
  }
  CUDA_CHECK(cudaEventRecord(G->ev2[c->rank], c->stream));
  group_sync(c);
  // my slice may be overwritten only after every peer has read it
  for (int q = 0; q < c->nshards; ++q)
    if (q != c->rank) CUDA_CHECK(cudaStreamWaitEvent(c->stream, G->ev2[q], 0));
}

// OR of a per-shard host flag over the group (one GPU: the flag itself)
static int group_or(mp_ctx* c, int v) {
  if (c->nshards <= 1) return v;
  Group* G = c->grp;
  const int b = c->par_flags ^= 1;
  G->flags[b][c->rank] = v;
  group_sync(c);
  int r = 0;
  for (int q = 0; q < c->nshards; ++q) r |= G->flags[b][q];
  return r;
}

// The PNCG scalars from per-chunk partials (device c->chunk_part, owned
// chunks filled): summed over every chunk in chunk order on the host --
// bitwise the same whatever the sharding.  extra/n_extra: device scalars
// read back in the same synchronisation (into h_scal[MAX_DOTS..]).
static void group_dots(mp_ctx* c, int n, double* out, const double* extra = nullptr, int n_extra = 0) {
  const int64_t nc = c->n_chunks;
  double* hp;
  if (c->nshards <= 1) {
    c->h_part.resize((size_t)nc * MAX_DOTS);
    hp = c->h_part.data();
    CUDA_CHECK(cudaMemcpyAsync(hp, c->chunk_part.p, sizeof(double) * nc * MAX_DOTS, cudaMemcpyDeviceToHost,
                               c->stream));
  } else {
    hp = c->grp->hpart[c->par_dots ^= 1];
    const int64_t a = c->own_c0, b = c->own_c1;
    if (b > a)
      CUDA_CHECK(cudaMemcpyAsync(hp + a * MAX_DOTS, c->chunk_part.p + a * MAX_DOTS, sizeof(double) * (b - a) * MAX_DOTS,
                                 cudaMemcpyDeviceToHost, c->stream));
  }
  if (n_extra)
    CUDA_CHECK(cudaMemcpyAsync(c->h_scal + MAX_DOTS, extra, sizeof(double) * n_extra, cudaMemcpyDeviceToHost,
                               c->stream));
  sync_stream(c);
  group_sync(c);
  for (int k = 0; k < n; ++k) {
    double t = 0.0;
    for (int64_t q = 0; q < nc; ++q) t += hp[q * MAX_DOTS + k];
    out[k] = t;
  }
}

// The owned ranges of every shard: NU alignment units (level-1 aggregates,
// or subdomains without coarse levels) split evenly; chunk = unit.
static void group_ranges(mp_ctx* c, int rank, int nshards) {
  const int64_t U = c->n_levels ? (int64_t)c->levels[0]->span : (int64_t)c->bs;
  const int64_t NU = (c->N + U - 1) / U;
  const int64_t u0 = NU * rank / nshards, u1 = NU * (rank + 1) / nshards;
  c->rank = rank;
  c->nshards = nshards;
  c->chunk_v = U;
  c->n_chunks = NU;
  c->own_c0 = u0;
  c->own_c1 = u1;
  c->own_v0 = std::min<int64_t>(c->N, u0 * U);
  c->own_v1 = std::min<int64_t>(c->N, u1 * U);
  c->own_d0 = c->own_v0 / c->bs;
  c->own_d1 = (c->own_v1 + c->bs - 1) / c->bs;
  c->own_a0 = c->n_levels ? u0 : 0;
  c->own_a1 = c->n_levels ? u1 : 0;
  c->chunk_part.ensure((size_t)NU * MAX_DOTS);
}

// Run fn on every shard, one host thread each (shard 0 on the caller's);
// the first error is rethrown, and the others are released from the
// barriers.
template <class Fn>
static void run_shards(mp_ctx* c, Fn&& fn) {
  if (c->nshards <= 1 || !c->grp) {
    fn(c);
    return;
  }
  Group* G = c->grp;
  G->bar.aborted = false;
  std::vector<std::exception_ptr> err(c->nshards);
  for (mp_ctx* sc : G->sh) sc->par_dots = sc->par_flags = 0;
  auto body = [&](int s) {
    mp_ctx* sc = G->sh[s];
    try {
      CUDA_CHECK(cudaSetDevice(sc->device));
      int64_t* saved = g_launch_counter;
      g_launch_counter = &sc->launches;
      fn(sc);
      g_launch_counter = saved;
    } catch (...) {
      err[s] = std::current_exception();
      G->bar.abort();
    }
  };
  std::vector<std::thread> th;
  for (int s = 1; s < c->nshards; ++s) th.emplace_back(body, s);
  body(0);
  for (auto& t : th) t.join();
  // prefer the error that caused the abort over the "aborted" follow-ups
  std::exception_ptr first = nullptr;
  for (auto& e : err) {
    if (!e) continue;
    try {
      std::rethrow_exception(e);
    } catch (const MpError& m) {
      if (std::string(m.what()).rfind("aborted:", 0) != 0) {
        first = e;
        break;
      }
      if (!first) first = e;
    } catch (...) {
      first = e;
      break;
    }
  }
  if (first) std::rethrow_exception(first);
}

static void multidot(mp_ctx* c, int64_t len, const DotSpec& S, const double* extra, int n_extra) {
  const int64_t nq = c->own_c1 - c->own_c0;
  if (nq > 0) {
    k_multidot_chunks<<<(unsigned)nq, 128, 0, c->stream>>>(len, 3 * c->chunk_v, c->own_c0, S, c->chunk_part);
    LAUNCH_CHECK();
  }
  group_dots(c, S.n, c->h_scal, extra, n_extra);
}
