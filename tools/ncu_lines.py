"""Per-source-line summary of an ncu source page (cuda,sass mix), hottest first.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
  python tools/ncu_lines.py mix.csv [top_n]
Prints, per CUDA source line: share of warp instructions executed, lane efficiency
(thread instructions / (32 * warp instructions)) and share of warp stall samples.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lines, h, fname = [], None, ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0] and len(r) >= 9:
        try:
            ex = int(r[h.index("Instructions Executed")] or 0)
            th = int(r[h.index("Thread Instructions Executed")] or 0)
            st = int(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        if ex or st:
            lines.append((fname, int(r[0]), r[1].strip(), ex, th, st))
tot = sum(x[3] for x in lines) or 1
tst = sum(x[5] for x in lines) or 1
print(f"warp instructions {tot}, stall samples {tst}, lane eff "
      f"{sum(x[4] for x in lines) / 32 / tot:.2f}")
for f, ln, src, ex, th, st in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{f[:14]:14s}:{ln:<5d} instr {100 * ex / tot:5.1f}%  lanes {th / 32 / max(ex, 1):4.2f}  "
          f"stall {100 * st / tst:5.1f}%  {src[:80]}")
