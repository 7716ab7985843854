"""Per-source-line warp-stall samples from an ncu report (cuda,sass source
view), aggregated per file and per line range. Usage:
  python tools/src_hotspots.py REPORT.ncu-rep [file:start-end:name ...]"""
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur = None
    agg = {}
    for r in csv.reader(out.splitlines()):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if not r or r[0] in ("Function Name", "Line No") or cur is None or len(r) < 5:
            continue
        try:
            line, s = int(r[0]), int(float(r[4] or 0))
        except ValueError:
            continue
        if s:
            agg.setdefault(cur, {}).setdefault(line, [0, r[1][:90]])[0] += s
    return agg


def main():
    agg = load(sys.argv[1])
    tot = sum(v[0] for f in agg.values() for v in f.values())
    print(f"total samples {tot}")
    for f, lines in sorted(agg.items(), key=lambda kv: -sum(v[0] for v in kv[1].values())):
        print(f"  {f:24s} {sum(v[0] for v in lines.values()):8d}")
    for spec in sys.argv[2:]:
        f, rng, name = spec.split(":")
        a, b = map(int, rng.split("-"))
        s = sum(v[0] for l, v in agg.get(f, {}).items() if a <= l <= b)
        print(f"  range {name:20s} {s:8d} ({100.0 * s / max(tot, 1):.1f}%)")
    top = sorted(((v[0], f, l, v[1]) for f, d in agg.items() for l, v in d.items()), reverse=True)[:25]
    for s, f, l, src in top:
        print(f"  {s:7d} {f}:{l} {src}")


if __name__ == "__main__":
    main()
