"""Hot SASS lines of an ncu report (source page): samples, executions, top stall reasons.
usage: python tools/sass_hot.py <report> [threshold_pct]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[1]; rows = r[2:]
iss = h.index('Warp Stall Sampling (All Samples)'); iex = h.index('Instructions Executed'); isrc = h.index('Source')
stall_cols = [i for i, k in enumerate(h) if k.startswith('stall_') and 'Not Issued' not in k]
tot = sum(float(x[iss] or 0) for x in rows)
ex_tot = sum(float(x[iex] or 0) for x in rows)
print("samples", tot, "instr executed", ex_tot)
for n, x in enumerate(rows):
    sm = float(x[iss] or 0)
    if sm / tot * 100 >= thr:
        st = sorted(((float(x[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
        print(n, f"{sm / tot * 100:5.1f}%", x[iex], x[isrc][:80], [(b, int(a)) for a, b in st])
