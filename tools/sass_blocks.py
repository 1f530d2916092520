"""Group an ncu SASS source page (csv) into straight-line blocks by execution count."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
h = rows[1]
ia, isrc = h.index('Address'), h.index('Source')
iex, ist = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data) or 1
print("total warp instructions", tot, "stall samples", tst)
blocks = []
for d in data:
    if blocks and blocks[-1][2] == d[2]:
        blocks[-1][1] = d[0]; blocks[-1][3] += 1; blocks[-1][4] += d[3]; blocks[-1][5].append(d[1])
    else:
        blocks.append([d[0], d[0], d[2], 1, d[3], [d[1]]])
for b in blocks:
    if b[2] * b[3] / tot > thr or b[4] / tst > 2 * thr:
        print(f"{b[0] & 0xffff:5x}-{b[1] & 0xffff:5x} n={b[3]:4d} ex_each={b[2]:8d} "
              f"share={b[2] * b[3] / tot * 100:5.1f}% stall={b[4] / tst * 100:5.1f}%")
        if len(sys.argv) > 3:
            for s in b[5][:int(sys.argv[3])]:
                print("      ", s)
