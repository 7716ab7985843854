"""Dynamic instruction counts per source line for chosen SASS opcodes, from
`ncu --page source --csv --print-source cuda,sass` (each SASS row belongs to the
source row above it). Usage: python tools/ncu_ops.py CSV OPCODE[,OPCODE] [TOP]"""
import collections
import csv
import re
import sys

ops = set(sys.argv[2].split(","))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cnt, fname, cur = collections.Counter(), "?", None
tot = 0
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0].isdigit():
        cur = f"{fname}:{r[0]}  {r[1].strip()[:80]}"
    elif len(r) > 8 and r[2].startswith("0x"):
        ins = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip())
        op = ins.split()[0].split(".")[0] if ins else "?"
        if op in ops:
            try:
                c = int(r[7])
            except ValueError:
                continue
            cnt[cur] += c
            tot += c
print(f"total {tot}")
for k, c in cnt.most_common(top):
    print(f"{100 * c / max(tot, 1):5.1f}%  {k}")
