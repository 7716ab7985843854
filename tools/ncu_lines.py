"""Per-source-line totals from `ncu --page source --csv --print-source cuda,sass`:
warp-stall samples and warp instructions executed, by file:line (inlined code is
attributed to its innermost source line). Usage: python tools/ncu_lines.py CSV [TOP]"""
import csv
import sys

rows, fname = [], "?"
with open(sys.argv[1]) as fh:
    for r in csv.reader(fh):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] and r[0].isdigit() and len(r) > 8:
            try:
                rows.append((fname, int(r[0]), r[1].strip(), int(r[4]), int(r[7])))
            except ValueError:
                pass
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
by_file = {}
for f, _, _, s, i in rows:
    a = by_file.setdefault(f, [0, 0])
    a[0] += s
    a[1] += i
for f, (s, i) in sorted(by_file.items(), key=lambda x: -x[1][0]):
    print(f"  {f:28s} samples {100 * s / tot_s:5.1f}%  inst {100 * i / tot_i:5.1f}%")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for f, ln, src, s, i in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{100 * s / tot_s:5.1f}% {100 * i / tot_i:5.1f}%  {f}:{ln}  {src[:90]}")
