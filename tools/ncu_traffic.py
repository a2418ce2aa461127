"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per kernel
from an ncu --set full report into profiles/ncu_traffic.json[<config>][<kernel>] (bytes).
usage: python tools/ncu_traffic.py <report.ncu-rep> <config name, e.g. C2>"""
import csv, io, json, os, subprocess, sys
rep, cfg = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for row in r[2:]:
    name = row[hdr.index("Kernel Name")]
    short = name.split("<")[0].split("(")[0].replace("void ", "").strip()
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(row[i].replace(",", "")) * scale[units[i]]
    out.setdefault(short, []).append(tot)
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d.setdefault(cfg, {})
for k, v in out.items():
    d[cfg][k] = sum(v) / len(v)
json.dump(d, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(d[cfg]))
