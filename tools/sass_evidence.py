"""Per-kernel SASS evidence of the Blackwell-native paths in libsidwt.so: counts of the
tcgen05 / TMEM / TMA / packed-FMA mnemonics in each kernel (cuobjdump -sass), and an
excerpt of the instructions around the first tensor-core MMA of each tensor-core kernel.
usage: python tools/sass_evidence.py [libsidwt.so] [> profiles/<round>_sass_evidence.txt]"""
import collections
import os
import re
import subprocess
import sys

MNEMONICS = ("UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMASTG", "UTMALDG", "UBLKCP", "USETMAXREG", "FFMA2",
             "IMAD", "PRMT", "SYNCS")


def kernels(lib):
    """{short kernel name: [sass lines]} from cuobjdump -sass."""
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs, cur = collections.OrderedDict(), None
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(ln)
    return funcs


def short(name):
    m = re.match(r"_ZN5sidwt\d+(k_\w+?)(I|E)", name)
    return m.group(1) if m else name


def counts(lines):
    c = collections.Counter()
    for ln in lines:
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            op = m.group(1)
            for k in MNEMONICS:
                if op == k or op.startswith(k):
                    c[k] += 1
    return c


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(here, "..", "paper_cs_0607001_b200", "libsidwt.so")
    funcs = kernels(lib)
    print(f"# cuobjdump -sass {os.path.basename(lib)}: {len(funcs)} kernels, sm_100a")
    for name, lines in funcs.items():
        c = counts(lines)
        print(f"{short(name):24s} {name[:90]}")
        print("    " + "  ".join(f"{k}x{v}" for k, v in sorted(c.items())))
    for name, lines in funcs.items():
        idx = [i for i, ln in enumerate(lines) if re.search(r"\bUTC[A-Z]*MMA\b", ln)]
        if not idx:
            continue
        i = idx[0]
        print(f"\n## excerpt: {short(name)} around its first tcgen05 MMA")
        for ln in lines[max(0, i - 6): i + 6]:
            print("   " + ln.strip())
        ld = [j for j, ln in enumerate(lines) if re.search(r"\bLDTM\b", ln)]
        if ld:
            print(f"## excerpt: {short(name)} TMEM load (tcgen05.ld)")
            for ln in lines[max(0, ld[0] - 2): ld[0] + 3]:
                print("   " + ln.strip())


if __name__ == "__main__":
    main()
