"""Summarise a bench.py JSON line (last line of the given log)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d[k] for k in ["value", "ms_per_step", "gpu_launches"] if k in d}, "e2e", d.get("e2e", {}).get("value"))
print(d.get("roofline"))
for k, v in sorted(d.get("kernels", {}).items(), key=lambda kv: -kv[1]["ms"]):
    print("  %-20s %6d launches %9.3f ms %8.1f us/launch %8.1f GB/s" % (k, v["launches"], v["ms"], v["ms"] * 1000 / max(1, v["launches"]), v["gbs"]))
