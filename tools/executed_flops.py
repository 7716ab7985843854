"""Executed FP64 work of one kernel launch from an ncu source page (SASS,
--page source --csv --print-source sass): DFMA = 2 flops per thread, DMUL /
DADD = 1, DMMA.884 = 8x8x4 FMAs = 512 flops per warp instruction. Counts are
warp-level "Instructions Executed"; thread-level = x32 (the kernels run full
warps on the FP64 paths). Usage: executed_flops.py SRC.csv BATCH"""
import csv
import json
import sys
from collections import Counter


def executed(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    cnt = Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[idx["Source"]].strip()
        if not src:
            continue
        op = src.split()[1] if src.startswith("@") else src.split()[0]
        cnt[op.split(".")[0]] += int(float(r[idx["Instructions Executed"]] or 0))
    flops = 32 * (2 * cnt["DFMA"] + cnt["DMUL"] + cnt["DADD"]) + 512 * cnt["DMMA"]
    return flops, {k: cnt[k] for k in ("DFMA", "DMUL", "DADD", "DMMA")}


if __name__ == "__main__":
    f, c = executed(sys.argv[1])
    B = int(sys.argv[2])
    print(json.dumps({"flops_per_launch": f, "flops_per_solve": f / B, "warp_instructions": c}))
