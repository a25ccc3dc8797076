"""From an `ncu --page raw --csv` dump: DRAM bytes per launch, warp stall
reasons (per issued instruction), issue activity, occupancy, L1/L2 hit rates."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
d = dict(zip(h, v))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


stalls = sorted(((num(k), k) for k in h if "smsp__average_warps_issue_stalled" in k and num(k)), reverse=True)
print("top stall reasons (warps per issued instruction):")
for val, k in stalls[:6]:
    print(f"  {val:8.3f} {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
          "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio"):
    print(f"  {k} = {d.get(k)}")
