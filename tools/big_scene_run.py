"""Configs 3-5 at full size on one B200: device-resident frames (CUDA
events on the solver stream, L2 flushed between frames), PNCG iterations/s
and sec/frame, then the scalable penetration checker on every frame's
positions.  C4/C5 use coarse_block = 32 (SURVEY.md 8(d) hard part 3).

    python tools/big_scene_run.py c5 FRAMES ITER_MAX [devices]"""

import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_19892_b200 import cli, scenes, solver  # noqa: E402

which = sys.argv[1]
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
iter_max = int(sys.argv[3]) if len(sys.argv) > 3 else 100
devices = [int(d) for d in sys.argv[4].split(",")] if len(sys.argv) > 4 else None
t0 = time.time()
if which == "c3":
    scene = scenes.c3_rod()
    v0 = scenes.c3_rod_v0(scene)
    h, cfg = 0.01, solver.SolverConfig(iter_max=iter_max)
elif which == "c4":
    scene = scenes.c4_spheres_in_bowl()
    v0 = np.zeros(3 * scene.mesh.n_vertices)
    h, cfg = 0.01, solver.SolverConfig(iter_max=iter_max, coarse_block=32)
else:
    scene = scenes.c5_puffer_balls()
    v0 = scenes.c5_puffer_v0(scene)
    h, cfg = 0.005, solver.SolverConfig(iter_max=iter_max, coarse_block=32)
build_s = time.time() - t0
print(json.dumps({"scene": which, "n_verts": int(scene.mesh.n_vertices), "n_tets": int(len(scene.elastic.vol)),
                  "build_s": round(build_s, 1)}), flush=True)
t0 = time.time()
ctx = scene.context(cfg, devices=devices) if devices else scene.context(cfg)
print(json.dumps({"context_s": round(time.time() - t0, 1)}), flush=True)
x0 = scene.mesh.rest_positions.ravel().copy()
ctx.set_state(x0, v0)
stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
chk = cli.SurfaceChecker(scene.mesh.rest_positions, scene.surface.triangles)
out = []
for f in range(frames):
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs, conv, _ = ctx.step_device(h)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    x, _ = ctx.get_state()
    t1 = time.time()
    dmin = chk.min_distance(x)
    hits = chk.intersections(x)[0]
    out.append({"frame": f + 1, "iters": len(recs), "ms": round(ms, 1), "iters_per_s": round(len(recs) / ms * 1e3, 1),
                "restarts": int(sum(r.restart for r in recs)), "converged": bool(conv),
                "min_alpha": min([1.0] + [r.min_alpha for r in recs]), "contacts_last": int(recs[-1].n_contacts),
                "check": {"min_distance": dmin, "intersections": hits, "s": round(time.time() - t1, 2)}})
    print(json.dumps(out[-1]), flush=True)
# stage breakdown: one more frame from the last state with the CUDA-event stage timers on
ctx.stage_timing(True)
recs, conv, _ = ctx.step_device(h)
st = ctx.stage_stats()
ctx.stage_timing(False)
stages = {k: {"ms": round(v[0], 2), "count": v[1]} for k, v in st.items()}
print(json.dumps({"stage_frame_iters": len(recs), "stages": stages}), flush=True)
print(json.dumps({"scene": which, "n_verts": int(scene.mesh.n_vertices), "n_tets": int(len(scene.elastic.vol)),
                  "surface_tris": int(len(scene.surface.triangles)), "devices": devices or [0], "stages": stages,
                  "build_s": round(build_s, 1), "cfg": {"iter_max": iter_max, "coarse_block": cfg.coarse_block, "h": h},
                  "frames": out}))
