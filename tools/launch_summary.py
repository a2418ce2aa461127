"""Per-kernel launch count / mean time / share of an ncu --metrics gpu__time_duration.sum csv.
usage: python tools/launch_summary.py <launches.csv> <title> [exclude-regex]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[i]; data = rows[i + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.OrderedDict()
for r in data:
    if len(r) <= vi:
        continue
    if len(sys.argv) > 3 and re.search(sys.argv[3], r[ki]):
        continue
    agg.setdefault(r[ki].split('(')[0], []).append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
print(sys.argv[2] + "\nncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); unit " + data[0][ui])
for k, v in agg.items():
    print("%-48s launches %4d  mean %12.1f  share %5.1f%%" % (k, len(v), sum(v) / len(v), 100 * sum(v) / tot))
