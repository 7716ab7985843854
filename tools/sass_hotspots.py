"""Aggregate an ncu source page (--print-source sass --csv) by opcode and list
the hottest instructions: where the warp-stall samples land."""
import csv
import sys
from collections import Counter


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    samp = Counter()
    cnt = Counter()
    total = 0
    hot = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[idx["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        s = int(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
        n = int(float(r[idx["Instructions Executed"]] or 0))
        samp[op] += s
        cnt[op] += n
        total += s
        hot.append((s, r[idx["Address"]][-5:], src[:70]))
    print(f"total samples {total}")
    for op, s in samp.most_common(top):
        print(f"  {op:12s} samples {s:8d} ({100.0 * s / max(total, 1):5.1f}%)  executed {cnt[op]}")
    print("hottest instructions:")
    for s, a, src in sorted(hot, reverse=True)[:top]:
        print(f"  {s:7d} {a} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
