"""Summarise an ncu --csv launch list (gpu__time_duration.sum): mean us per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    try:
        d[r[ik]].append(float(r[iv].replace(",", "")))
    except ValueError:
        pass
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
total = sum(sum(v) for v in d.values()) / steps
print(f"{'kernel':60s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1000:9.1f} {sum(v) / steps / total:7.1%}")
print(f"{'total per step':60s} {'':8s} {total / 1000:9.1f}")
