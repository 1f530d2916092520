"""Group an ncu SASS source page (csv) into straight-line blocks by execution count.

  python tools/sass_blocks.py page.csv [threshold] [n_source_lines] [kernel_substring]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
nsrc = int(sys.argv[3]) if len(sys.argv) > 3 else 0
want = sys.argv[4] if len(sys.argv) > 4 else ""
# sections: a "Kernel Name" row, a header row, then instruction rows
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1] if len(r) > 1 else "", None, []]
        sections.append(cur)
    elif r and r[0] == "Address" and cur is not None:
        cur[1] = r
    elif cur is not None and cur[1] is not None and len(r) >= len(cur[1]):
        cur[2].append(r)
if not sections:  # single-kernel page without a name row
    sections = [["", rows[1], rows[2:]]]
name, h, body = next(s for s in sections if want in s[0])
ia, isrc = h.index("Address"), h.index("Source")
iex, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)) for r in body]
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data) or 1
print(name[:100])
print("total warp instructions", tot, "stall samples", tst)
blocks = []
for d in data:
    if blocks and blocks[-1][2] == d[2]:
        blocks[-1][1] = d[0]; blocks[-1][3] += 1; blocks[-1][4] += d[3]; blocks[-1][5].append(d[1])
    else:
        blocks.append([d[0], d[0], d[2], 1, d[3], [d[1]]])
for b in blocks:
    if b[2] * b[3] / max(tot, 1) > thr or b[4] / tst > 2 * thr:
        print(f"{b[0] & 0xffff:5x}-{b[1] & 0xffff:5x} n={b[3]:4d} ex_each={b[2]:8d} "
              f"share={b[2] * b[3] / max(tot, 1) * 100:5.1f}% stall={b[4] / tst * 100:5.1f}%")
        for s in b[5][:nsrc]:
            print("      ", s)
