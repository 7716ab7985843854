"""Print the bench lines of gpurun_out/quick.json compactly."""
import json
import sys

for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quick.json"):
    if not l.startswith("{"):
        continue
    d = json.loads(l)
    print(d["config"]["workload"][:44], f"{d['value'] / 1e6:.2f} M/s", f"{d['ms_per_step'] * 1000:.1f} us",
          d.get("roofline_binding"), round(d.get("roofline_frac_of_binding", 0), 3))
    for k, v in d.get("extra", {}).items():
        print("   ", k, f"{v['solves_per_s'] / 1e6:.3f} M/s", f"{v['ms_per_step'] * 1000:.1f} us", v["binding"],
              round(v["roofline_frac_of_binding"], 3))
