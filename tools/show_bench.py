"""Prints the key numbers of a bench.py JSON line (the last one in the file)."""
import json
import sys

for f in sys.argv[1:]:
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print(f, "value %.0f e2e %.0f ms/step %.3f launches %s checks %s" % (
        d["value"], d["e2e"]["value"], d["ms_per_step"], d.get("gpu_launches"), d.get("checks")))
    r = d.get("roofline") or {}
    print("  roofline:", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})
    for k, v in d.get("kernels", {}).items():
        print("   %-38s ms/launch %.4f share %.3f hbm %.3f alu %.3f" % (
            k, v["ms_per_launch"], v["share"], v["hbm_frac"], v["alu_frac"]))
