"""Attribute an ncu capture's per-instruction samples / executions to CUDA source lines:
nvdisasm --print-line-info of the kernel's cubin gives offset -> line, the ncu source page
(SASS, -lineinfo build) gives address -> samples.  Prints the hottest source lines with their
stall reasons.
usage: python tools/ncu_lines.py <report.ncu-rep> <object or .so> <mangled kernel name> [top]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, func):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cubins = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")]
        out = ""
        for cb in cubins:
            out = subprocess.run(["nvdisasm", "--print-line-info", cb], capture_output=True, text=True).stdout
            if func in out:
                break
    m, cur, on = {}, None, False
    for ln in out.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            on = ln.strip().endswith(".text." + func + " --------------------------") or (".text." + func + " ") in ln
            continue
        if not on:
            continue
        a = re.search(r'File "([^"]+)", line (\d+)', ln) if "## File" in ln else None
        if a:
            cur = (a.group(1), int(a.group(2)))
            continue
        b = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
        if b and cur is not None:
            m[int(b.group(1), 16)] = cur
    return m


def main():
    rep, obj, func = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    lm = line_map(obj, func)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, rows = r[1], r[2:]
    ia, iss, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    base = int(rows[0][ia], 16)
    agg = {}
    for x in rows:
        ln = lm.get(int(x[ia], 16) - base, ("?", -1))
        a = agg.setdefault(ln, [0.0, 0.0, {}])
        a[0] += float(x[iss] or 0)
        a[1] += float(x[iex] or 0)
        for j in stall:
            a[2][h[j][6:]] = a[2].get(h[j][6:], 0) + float(x[j] or 0)
    tot = sum(v[0] for v in agg.values())
    cache = {}
    for (fn, ln), (sm, ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        s2 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        if fn not in cache:
            cache[fn] = open(fn).read().splitlines() if os.path.exists(fn) else []
        src = cache[fn]
        text = src[ln - 1].strip()[:64] if 0 < ln <= len(src) else ""
        print(f"{sm / tot * 100:5.1f}%  {os.path.basename(fn)}:{ln:<5d} ex {int(ex):>9d}  {[(k, int(v)) for k, v in s2]}  {text}")


if __name__ == "__main__":
    main()
