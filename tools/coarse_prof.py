"""Per-phase timing of the coarse inverse kernel (MP_CS_PROF=1 prints
%globaltimer splits from CTA 0) and CUDA-event timing of whole launches via
the standalone entry, on random SPD matrices of the scenes' coarse orders."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2604_19892_b200 import _native  # noqa: E402

for n in [int(a) for a in (sys.argv[1:] or ["276", "1095", "1902"])]:
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n))
    A = X @ X.T + n * np.eye(n)
    _native.spd_inverse(A)
    t0 = time.perf_counter()
    for _ in range(5):
        inv, bad = _native.spd_inverse(A)
    dt = (time.perf_counter() - t0) / 5
    err = np.abs(inv - np.linalg.inv(A)).max() / np.abs(np.linalg.inv(A)).max()
    print(f"n={n}: {dt * 1e3:.2f} ms per call incl. H2D/D2H, rel err {err:.1e}, not_spd={bad}", flush=True)
