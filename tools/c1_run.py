"""BASELINE config 1 on the device: tests/golden/c1/c1.ini (the reference's
INI schema) through this repo's `cli simulate`, 10 frames; prints the
frames.csv rows, the per-frame wall time and the penetration check.

    python tools/c1_run.py OUT_DIR"""
import sys
import time
from pathlib import Path

sys.path.insert(0, ".")
from paper_2604_19892_b200 import cli  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c1_out").resolve()
out.mkdir(parents=True, exist_ok=True)
ini = out / "c1.ini"
ini.write_text(Path("tests/golden/c1/c1.ini").read_text().replace("output_dir = out_c1", f"output_dir = {out}/sim"))
t0 = time.time()
rc = cli.main(["simulate", str(ini)])
print("simulate rc", rc, "wall s", round(time.time() - t0, 2))
print((out / "sim" / "frames.csv").read_text())
print("check rc", cli.main(["check", str(out / "sim")]))
