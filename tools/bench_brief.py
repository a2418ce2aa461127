"""One-line digest of a bench.py JSON output file."""
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "unreadable:", e); sys.exit(0)
s = d.get("stages", {})
a, c = s.get("analyze", {}), s.get("correlate_peaks", {})
print(sys.argv[1].split("/")[-1], "| %.3g samples/s" % d["value"], "| ms/step %.3f" % d["ms_per_step"],
      "| analyze %.3f ms %.0f GB/s (%.0f%%)" % (a.get("ms", 0), a.get("achieved", 0), 100 * a.get("frac", 0)),
      "| corr %.3f ms %.1f TF" % (c.get("ms", 0), (c.get("alu") or c.get("tensor") or {}).get("achieved", 0)),
      "| e2e %s" % (d.get("e2e", {}) or {}).get("value"), "| cpu %s" % (d.get("cpu_baseline", {}) or {}).get("value"),
      "| clocks", d.get("clocks"))
v = d.get("variants") or {}
if v:
    print("   variants:", {k: round(x, 3) for k, x in v.items() if k.endswith("_ms")})
