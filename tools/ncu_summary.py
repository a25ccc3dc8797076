"""Summarise an ncu --set full report: per-kernel duration, DRAM bytes,
achieved bandwidth, occupancy, registers (reads the raw page)."""
import csv
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_%",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_%",
    "smsp__inst_executed.sum": "inst",
}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    units = rows[1]
    ki = h.index("Kernel Name")
    cols = [(i, WANT[x]) for i, x in enumerate(h) if x in WANT]
    print("kernel | " + " | ".join(n for _, n in cols) + " | GB/s (dram r+w / time)")
    for r in rows[2:]:
        vals = {}
        for i, n in cols:
            v = r[i].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                continue
            u = units[i]
            if n.endswith("_MB"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            if n == "us":
                v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            vals[n] = v
        gbs = (vals.get("dram_read_MB", 0) + vals.get("dram_write_MB", 0)) / max(vals.get("us", 1e-9), 1e-9) * 1e3
        print(r[ki].split("(")[0][:28] + " | " + " | ".join(f"{vals.get(n, float('nan')):.4g}" for _, n in cols)
              + f" | {gbs:.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
