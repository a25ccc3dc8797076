#!/usr/bin/env python
"""Benchmark of the B200 MAS-PNCG solver inner loop (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A *step* is one simulated frame: ``solver.step`` = prepare_step +
advance_step (Alg. 1, `pkg/src/ipcsim/solver.py:296-464`) of the config-2
scene (8 soft SNH cubes stacked on a pinned floor, 46,664 V / 235,830 T,
BASELINE.json ``configs[1]``), every PNCG iteration on the device.

Metric: PNCG iterations per second (whole job), with sec/frame alongside.
Both arms time the SAME frames: bench frame 6 onwards from a committed start
state (tests/golden/c2_bench.npz, this solver's own state after 5 frames from
rest, where the reference's stage taps were recorded); the CPU arms measure
iterations/s on a bounded prefix of frame 6.

* ``value``  -- device-resident frames (state resident in HBM, CUDA events on
  the context stream around each frame, L2 flushed between frames).
* ``e2e``    -- the same frames through the public API
  ``solver.step(scene, x, v, h, cfg)`` with host (pinned) numpy buffers: the
  H2D of x, v and the D2H of x, v are inside the timed region.
* ``roofline`` -- the MAS apply stage (north-star roofline kernel #1),
  algorithmic bytes per launch / CUDA-event launch time measured inside the
  timed frames; ``roofline_gradient`` the same for the gradient stage.
* ``cpu_baseline`` -- the numpy oracle (oracle/, a CPU restatement of the
  reference's algorithm) on a bounded sample of the same workload, rank 0.

N > 1 (torchrun): every rank simulates its own replica of the scene on its
own GPU ("replicas only": config 2 is a single-GPU scene per the north
star); ``value`` = all ranks' iterations / max-over-ranks time.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port; the Python reference itself cannot travel to the GPU box) on
the same frame from the same start state, rank 0 only, with 1 BLAS thread
and with every host thread (the faster is the line's value).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SCENE_DESC = ("c2_stack: 8 SNH cubes (17^3 cells, 0.2 m, E=1e5) stacked 2x2x2 with 5e-3 gaps on a pinned "
              "1.2x1.2x0.1 floor, released from rest (contacts form from frame 2); 46,664 V / 235,830 T / "
              "27,756 surface tris; h=0.01, d_hat=2e-3, kappa=1e4; SolverConfig defaults (K=8, levels=2, "
              "coarse_block=4, block 32) except iter_max")
H = 0.01
GAP = 5e-3
ITER_MAX = 500
# The timed frames start from this committed state: the GPU's own state after
# 5 frames from rest (tools/c2_dump.py; the solver is bitwise deterministic,
# so every box reaches the same bits), at which the reference's stage taps
# were recorded (tests/golden/make_c2_golden.py).  Both arms time frames
# from here, so they time the same frames whatever --warmup is.
START = ROOT / "tests" / "golden" / "c2_bench.npz"
START_FRAME = 6  # 1-based: the frame after the 5 frames that produced START


def start_state():
    with np.load(START) as z:
        return z["x0"].copy(), z["v0"].copy()


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


def _fp64_peak():
    """FP64 FMA peak measured on this GPU by tools/micro/fp64_peak (built by
    __graft_entry__.build()); else 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz."""
    exe = ROOT / "tools" / "micro" / "fp64_peak"
    try:
        out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
        return float(json.loads(out.strip().splitlines()[-1])["fp64_fma_tflops"]), "measured"
    except Exception:
        return 37.2, "nominal (148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _oracle_frame(budget_s, threads):
    """PNCG iterations of bench frame START_FRAME (from the committed start
    state) by the numpy oracle within a wall-clock budget; the scene, its
    partition and the start state are prepared outside the timed call.
    Returns (iterations, seconds)."""
    from threadpoolctl import threadpool_limits

    from oracle import solver as osolver

    from paper_2604_19892_b200 import scenes

    scene = osolver.Scene.from_scene(scenes.c2_stack(gap=GAP))
    cfg = osolver.SolverConfig(iter_max=ITER_MAX)
    scene.partition(cfg.block_size)
    x, v = start_state()
    with threadpool_limits(limits=threads):
        return osolver.timed_iterations(scene, x, v, H, cfg, budget_s=budget_s)


def cpu_baseline(budget_s=30.0, threads=1):
    """The oracle (numpy CPU restatement of the reference, oracle/) on a
    bounded sample of the same workload: the first timed frame, from the same
    start state, single BLAS thread (BLAS threading slows this
    path down).  Returns the cpu_baseline object."""
    iters, elapsed = _oracle_frame(budget_s, threads)
    return {
        "value": iters / elapsed, "unit": "iters/s", "cores": threads, "kind": "port",
        "sample": f"the first {iters} PNCG iterations of bench frame {START_FRAME} (the GPU arm's first timed "
                  f"frame, same start state) by the numpy oracle, {elapsed:.1f} s, single process, BLAS "
                  f"threads={threads}; scene/partition built outside the timed call",
    }


def _host_cpu():
    info = {"nproc": os.cpu_count()}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return info


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port: the Python reference cannot travel to the GPU box) on the
    SAME frames as the GPU arm: bench frame START_FRAME from the committed
    start state, iterations/s over one continuous bounded sample.  Measured
    with one BLAS thread (the fastest setting for this path) and, for the
    record, with every host thread; `value` is the faster of the two."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    for _ in range(max(0, min(args.warmup, 1))):
        _oracle_frame(2.0, 1)  # imports, BLAS init
    budget = float(min(200.0, max(60.0, 10.0 * args.steps)))
    it1, s1 = _oracle_frame(budget, 1)
    budget_all = min(40.0, budget / 3.0)
    itn, sn = _oracle_frame(budget_all, nthreads)
    v1, vn = it1 / s1, itn / sn
    value, threads, it, sec = (v1, 1, it1, s1) if v1 >= vn else (vn, nthreads, itn, sn)
    line = {
        "impl": "reference", "metric": "PNCG iters/sec", "value": value, "unit": "iters/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": SCENE_DESC, "iter_max": ITER_MAX, "same_frames": True,
                   "frames": f"bench frame {START_FRAME} from the committed start state (tests/golden/c2_bench.npz) "
                             "-- the GPU arm's first timed frame",
                   "sample": f"one continuous {sec:.0f} s sample ({it} PNCG iterations) split evenly over the "
                             f"{args.steps} steps"},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": f"{it} PNCG iterations of frame {START_FRAME} in {sec:.1f} s",
                         "threads_1": {"iters_per_s": v1, "iters": it1, "s": round(s1, 1)},
                         f"threads_{nthreads}": {"iters_per_s": vn, "iters": itn, "s": round(sn, 1)},
                         "host": _host_cpu()},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    from paper_2604_19892_b200 import scenes, solver

    from paper_2604_19892_b200.replicas import ReplicaGroup

    _, _, local = _dist()
    torch.cuda.set_device(local)
    grp = ReplicaGroup.from_env("nccl")
    ws, rank = grp.world_size, grp.rank
    barrier, allmax, allsum = grp.barrier, grp.allmax, grp.allsum

    scene = scenes.c2_stack(gap=GAP)
    cfg = solver.SolverConfig(iter_max=args.iter_max or ITER_MAX)
    ctx = scene.context(cfg, device=local)
    x0 = scene.mesh.rest_positions.ravel().copy()
    ctx.set_state(x0, np.zeros_like(x0))
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    for _ in range(args.warmup):
        ctx.step_device(H)
    torch.cuda.synchronize()
    xw, vw = ctx.get_state()

    # the timed frames (and the e2e leg) start from the committed state
    x_start_h, v_start_h = start_state()
    warm_equals_start = bool(args.warmup == START_FRAME - 1 and np.array_equal(xw, x_start_h)
                             and np.array_equal(vw, v_start_h)) if args.warmup == START_FRAME - 1 else None
    ctx.set_state(x_start_h, v_start_h)
    # dry run of the timed frames: the solver is bitwise deterministic, so
    # this grows every capacity-driven buffer (pair lists, contact tables) to
    # its final size -- the timed frames then allocate nothing
    for _ in range(args.steps):
        ctx.step_device(H)
    torch.cuda.synchronize()
    ctx.set_state(x_start_h, v_start_h)

    # ---- timed: device-resident frames (stage timers off: they add event
    # records and host waits; the solver is bitwise deterministic, so the
    # breakdown pass below replays exactly these frames with them on) ----
    sampler = ClockSampler()
    if rank == 0:
        sampler.start()
    ctx.stage_timing(False)
    launches0 = ctx.launches
    total_ms = 0.0
    iters = 0
    frames = []
    for _ in range(args.steps):
        flush.fill_(1)  # evict L2 between frames (outside the timed interval)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        recs, conv, _ = ctx.step_device(H)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        total_ms += ms
        iters += len(recs)
        frames.append({"iters": len(recs), "ms": round(ms, 3), "converged": conv,
                       "restarts": int(sum(r.restart for r in recs)),
                       "z_norm_last": recs[-1].z_norm if len(recs) else None})
    launches = ctx.launches - launches0
    clocks = sampler.stop() if rank == 0 else None
    t_max = allmax(total_ms)
    all_iters = allsum(float(iters))

    # ---- breakdown: the same frames again, stage timers on ----
    ctx.set_state(x_start_h, v_start_h)
    ctx.stage_timing(True)
    replay_ms = 0.0
    replay_same = True
    for f in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        recs, conv, _ = ctx.step_device(H)
        e1.record(stream)
        torch.cuda.synchronize()
        replay_ms += e0.elapsed_time(e1)
        replay_same &= len(recs) == frames[f]["iters"] and (
            not len(recs) or recs[-1].z_norm == frames[f]["z_norm_last"])
    stats = ctx.stage_stats()
    ctx.stage_timing(False)
    total_ms_timed = total_ms
    total_ms = replay_ms  # stage shares are of the replay (timers on)
    for fr in frames:
        fr.pop("z_norm_last", None)

    # ---- e2e: the same frames through the public API with host buffers ----
    xp = torch.empty(x_start_h.size, dtype=torch.float64).pin_memory().numpy()
    vp = torch.empty(v_start_h.size, dtype=torch.float64).pin_memory().numpy()
    xp[:] = x_start_h
    vp[:] = v_start_h
    e2e_s = 0.0
    e2e_iters = 0
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        st, tr = solver.step(scene, xp, vp, H, cfg)
        xp[:] = st.x  # the next frame's host input
        vp[:] = st.v
        e2e_s += time.perf_counter() - t0
        e2e_iters += tr.iterations
        barrier()
    e2e_s = allmax(e2e_s)
    e2e_all = allsum(float(e2e_iters))

    if rank != 0:
        grp.close()
        return

    peaks, peak_kind = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))

    def roof(name, kernels):
        ms, cnt, b = stats[name]
        if cnt == 0 or ms <= 0:
            return None
        ach = (b / cnt) / (ms / cnt * 1e-3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(name)
        return {"bound": "hbm", "kernel": kernels, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic, "bytes_per_launch": round(b / cnt),
                "us_per_launch": round(1e3 * ms / cnt, 2), "launches": cnt, "peak_kind": peak_kind}

    fp64_peak, fp64_kind = _fp64_peak()

    def roof_fp64(name, kernel):
        ms, cnt, f = stats[name]
        if cnt == 0 or ms <= 0:
            return None
        ach = (f / cnt) / (ms / cnt * 1e-3) / 1e12
        return {"bound": "fp64", "kernel": kernel, "achieved": round(ach, 2), "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": round(ach / fp64_peak, 4), "flops_per_launch": round(f / cnt),
                "us_per_launch": round(1e3 * ms / cnt, 2), "launches": cnt, "peak_kind": fp64_kind,
                "note": "timed in place, concurrent with the other levels' kernels of the same build"}

    host = {"loop_ms": round(stats["loop"][0], 2), "blocked_in_syncs_ms": round(stats["host_wait"][0], 2),
            "syncs": stats["host_wait"][1],
            "note": "host wall time of the advance loops and the part spent blocked on the stream"}
    stage_share = {k: {"ms": round(v[0], 2), "count": v[1], "share": round(v[0] / max(total_ms, 1e-9), 4)}
                   for k, v in stats.items() if k not in ("loop", "host_wait")}
    n3 = 3 * scene.mesh.n_vertices
    line = {
        "metric": "PNCG iters/sec", "value": all_iters / (t_max * 1e-3), "unit": "iters/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": SCENE_DESC, "step": "one frame (prepare_step + advance_step)",
                   "l2": "flushed between timed frames (512 MiB write)",
                   "parallelism": "replicas" if ws > 1 else "single-gpu", "iter_max": cfg.iter_max,
                   "frames": f"frames {START_FRAME}..{START_FRAME + args.steps - 1} from the committed start state "
                             "(tests/golden/c2_bench.npz = this solver's state after 5 frames from rest)",
                   "warmup_reaches_start_state": warm_equals_start},
        "sec_per_frame": t_max * 1e-3 / args.steps,
        "frames": frames,
        "e2e": {"value": e2e_all / e2e_s, "unit": "iters/s", "h2d_bytes_per_step": 2 * 8 * n3,
                "d2h_bytes_per_step": 2 * 8 * n3, "sec_per_frame": e2e_s / args.steps,
                "frames": "the timed frames replayed from the same start state (the solver is bitwise "
                          "deterministic: the same iterations as the device-resident pass)",
                "api": "paper_2604_19892_b200.solver.step(scene, x, v, h, cfg) with pinned numpy x, v"},
        "roofline": roof("mas_apply_l0", "k_mas_apply_l0_direct (level-0 packed block matvec + Woodbury overlay + "
                                          "coarse prolongation + pinned projection; one CTA per subdomain, "
                                          "streaming loads)"),
        "roofline_mas_stage": roof("mas_apply",
                                   "MAS apply stage: k_restrict1 + k_restrict_up + k_coarse_mv x2 + k_mas_apply_l0_direct"),
        "roofline_gradient": roof("tet_grad", "k_tet_grad<SNH> (F, Piola, per-corner forces; 113 B/tet + 48 B/vertex)"),
        "roofline_gradient_stage": roof("gradient",
                                        "gradient stage: k_contact_grad_rows + k_tet_grad x2 + k_grad_gather"),
        "roofline_hvp": roof("hvp", "HVP: k_bsr_spmv + k_rank1_rows + k_inc_gather_add"),
        "roofline_mas_sweep0": roof_fp64("mas_sweep0", "k_mas_sweep: level-0 block assembly + symmetric sweep "
                                                       "(m^3 FMA per subdomain)"),
        "roofline_coarse_inv": roof_fp64("coarse_inv", "k_coarse_sweep: first coarse level's inverse "
                                                       "((32 nT)^3 FMA, persistent, one grid barrier per panel)"),
        "stages": stage_share,
        "stages_note": ("stage times, rooflines and host stats come from a replay of the same frames with "
                        "CUDA-event stage timers on (bitwise-identical trajectory: %s; %.1f ms vs %.1f ms "
                        "timed without timers)" % (replay_same, replay_ms, total_ms_timed)),
        "host": host,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and ws == 1:
        try:
            line["cpu_baseline"] = cpu_baseline()
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "unavailable": repr(e)[:200]}
    if args.configs and ws == 1:
        line["other_configs"] = {}
        for name in [c for c in args.configs.split(",") if c]:
            try:
                line["other_configs"][name] = measure_config(name, flush, local)
            except Exception as e:  # reported, never silently replaced
                line["other_configs"][name] = {"unavailable": repr(e)[:300]}
    print(json.dumps(line), flush=True)
    grp.close()


# BASELINE.json configs 3-5 on one B200: bounded device-resident samples
# (not the headline; SURVEY 8.0 sizes).  Each: the scene built on the host,
# one untimed frame (buffers grow), then timed frames with CUDA events on
# the solver stream, L2 flushed before each; PNCG iterations/s and the
# frames' capped sec/frame; then the GPU penetration checker on the final
# positions (cli.SurfaceChecker: min PT/EE distance + tri-tri count).
OTHER = {
    "c3": {"desc": "c3_rod: SNH rod 8x8x2500 cells (202,589 V / 960,006 T with the floor), twist 5 rad/s at the ends, "
                   "h=0.01, SolverConfig defaults (levels 2, coarse_block 4)", "frames": 1, "iter_max": 40, "h": 0.01},
    "c4": {"desc": "c4_spheres_in_bowl: 64 SNH voxel balls (8,625 V each) over a pinned ARAP bowl (562,859 V / "
                   "2,804,112 T), h=0.01, coarse_block 32", "frames": 1, "iter_max": 40, "h": 0.01, "cb": 32},
    "c5": {"desc": "c5_puffer_balls: 8 SNH puffer balls (core + 410 spikes; 1,142,784 V / 2,743,680 T) closing at "
                   "0.1 m/s each, d_hat=1e-4, h=0.005, coarse_block 32", "frames": 1, "iter_max": 20, "h": 0.005,
           "cb": 32},
}


def measure_config(name, flush, local):
    import torch

    from paper_2604_19892_b200 import cli, scenes, solver

    spec = OTHER[name]
    t0 = time.perf_counter()
    if name == "c3":
        scene = scenes.c3_rod()
        v0 = scenes.c3_rod_v0(scene)
    elif name == "c4":
        scene = scenes.c4_spheres_in_bowl()
        v0 = np.zeros(3 * scene.mesh.n_vertices)
    else:
        scene = scenes.c5_puffer_balls()
        v0 = scenes.c5_puffer_v0(scene)
    build_s = time.perf_counter() - t0
    cfg = solver.SolverConfig(iter_max=spec["iter_max"], coarse_block=spec.get("cb", 4))
    ctx = scene.context(cfg, device=local)
    x0 = scene.mesh.rest_positions.ravel().copy()
    ctx.set_state(x0, v0)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    ctx.step_device(spec["h"])  # untimed: buffers grow
    ctx.set_state(x0, v0)
    frames, tot_ms, tot_it = [], 0.0, 0
    for _ in range(spec["frames"]):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        recs, conv, _ = ctx.step_device(spec["h"])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tot_ms += ms
        tot_it += len(recs)
        frames.append({"iters": len(recs), "ms": round(ms, 1), "restarts": int(sum(r.restart for r in recs)),
                       "converged": bool(conv), "min_alpha": min([1.0] + [r.min_alpha for r in recs]),
                       "contacts_last": int(recs[-1].n_contacts) if recs else 0})
    x, _ = ctx.get_state()
    # rooflines at this scale: one more frame with the stage timers on
    ctx.stage_timing(True)
    ctx.step_device(spec["h"])
    st = ctx.stage_stats()
    ctx.stage_timing(False)
    peaks, _ = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    roof = {}
    for key, label in (("mas_apply_l0", "k_mas_apply_l0_direct"), ("mas_apply", "MAS apply stage"),
                       ("tet_grad", "k_tet_grad<SNH>"), ("gradient", "gradient stage"), ("hvp", "HVP stage")):
        ms, cnt, b = st[key]
        if cnt and ms > 0:
            ach = (b / cnt) / (ms / cnt * 1e-3) / 1e9
            roof[key] = {"kernel": label, "achieved_gbs": round(ach, 1), "frac": round(ach / hbm, 4),
                         "us_per_launch": round(1e3 * ms / cnt, 2), "bytes_per_launch": round(b / cnt)}
    stage_ms = {k: round(v[0], 2) for k, v in st.items()}
    chk = cli.SurfaceChecker(scene.mesh.rest_positions, scene.surface.triangles, local)
    check = {"min_distance": chk.min_distance(x), "tri_tri_intersections": chk.intersections(x)[0]}
    return {"workload": spec["desc"], "n_verts": int(scene.mesh.n_vertices), "n_tets": int(len(scene.elastic.vol)),
            "iter_max": spec["iter_max"], "value": tot_it / (tot_ms * 1e-3), "unit": "iters/s",
            "sec_per_frame_capped": tot_ms * 1e-3 / spec["frames"], "frames": frames, "build_s": round(build_s, 1),
            "penetration_check": check, "roofline": roof, "stages_ms_one_frame": stage_ms,
            "note": "frames capped at iter_max (bounded sample), from rest"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--iter-max", type=int, default=0, help=f"PNCG iterations cap per frame (default {ITER_MAX})")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--configs", default="c3,c4,c5",
                    help="extra BASELINE configs measured after the headline at N=1 (comma list; '' for none)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
