"""Penetration checker on the REST state of C5 (and one puffer ball alone):
are the generated meshes intersection-free before any step?"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import cli, geometry, scenes, _native  # noqa: E402

ball = scenes.puffer_mesh()
surf = geometry.SurfaceMesh.from_tet_mesh(ball)
n, first = _native.check_intersections(ball.rest_positions, surf.triangles)
out = {"ball_tris": len(surf.triangles), "ball_intersections": n, "first": first}
if n:
    t = surf.triangles[first]
    out["first_tri"] = t.tolist()
    out["first_xyz"] = ball.rest_positions[t].tolist()
scene = scenes.c5_puffer_balls()
chk = cli.SurfaceChecker(scene.mesh.rest_positions, scene.surface.triangles)
out["c5_rest_intersections"] = chk.intersections(scene.mesh.rest_positions)[0]
out["c5_rest_min_distance"] = chk.min_distance(scene.mesh.rest_positions)
c4 = scenes.c4_spheres_in_bowl()
chk4 = cli.SurfaceChecker(c4.mesh.rest_positions, c4.surface.triangles)
out["c4_rest_intersections"] = chk4.intersections(c4.mesh.rest_positions)[0]
print(json.dumps(out))
