"""Instruction histogram of libhetft.so's SASS: per kernel, the mnemonics
that prove the Blackwell paths (tcgen05 MMA = UTC*MMA, TMEM loads = LDTM,
TMA = UTMALDG/UBLKCP, packed FP32 = FFMA2/FADD2, cp.async = LDGSTS,
streaming loads LDG.E.NA.128.CONSTANT) and totals.

    python tools/sass_histogram.py paper_1405_2912_b200/libhetft.so > profiles/r02_sass_histogram.txt
"""
import collections
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "FFMA2", "FADD2", "FFMA",
        "DFMA", "LDGSTS", "LDG.E.NA.128.CONSTANT", "LDG.E.NA.128", "LDS.128", "STG.E.EF.128", "HMMA"]

lib = sys.argv[1]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
func = None
hist = collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and func:
        op = m.group(1)
        hist[func]["total"] += 1
        for k in KEYS:
            if op == k or op.startswith(k + ".") or (k.count(".") and op.startswith(k)):
                hist[func][k] += 1
                break
demangled = {}
try:
    out = subprocess.run(["c++filt"], input="\n".join(hist), capture_output=True, text=True).stdout.splitlines()
    demangled = dict(zip(hist, out))
except OSError:
    pass
tot = collections.Counter()
print(f"# SASS instruction histogram of {lib} (cuobjdump -sass; sm_100a)")
for f in sorted(hist, key=lambda f: demangled.get(f, f)):
    h = hist[f]
    tot.update(h)
    keys = ", ".join(f"{k} {h[k]}" for k in KEYS if h[k])
    print(f"{demangled.get(f, f)[:90]:90s} total {h['total']:6d}  {keys}")
print("\n# whole library: " + ", ".join(f"{k} {tot[k]}" for k in ["total"] + KEYS if tot[k]))
