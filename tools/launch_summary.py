"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total / mean device time and share."""
import collections
import csv
import sys


def summarize(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else (v * 1e3 if r[ui] in ("msecond", "ms") else v)
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"total {T:.0f} us over {sum(cnt.values())} launches (ncu, serialised, cold caches)"]
    out.append(f"{'kernel':62s} {'launches':>8s} {'total us':>12s} {'share':>7s} {'us/launch':>10s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{k[:62]:62s} {cnt[k]:8d} {v:12.1f} {100 * v / T:6.2f}% {v / cnt[k]:10.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30))
