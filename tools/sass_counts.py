"""Static SASS opcode counts per kernel of the in-tree build -> markdown table.

usage: python tools/sass_counts.py > profiles/r02/sass/opcode_counts.md
(cuobjdump -sass paper_2204_07921_b200/libcmg.so piped through c++filt)
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2204_07921_b200" / "libcmg.so"
SEL = ["UTMALDG", "UBLKCP", "SYNCS", "FFMA2", "FADD2", "FMUL2", "MUFU.RSQ64H", "MUFU.RCP64H", "MUFU.RSQ", "DFMA",
       "DADD", "DMUL", "LDS", "STS", "LDG", "STG", "BAR", "CALL"]
out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
funcs, cur = collections.OrderedDict(), None
for ln in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", ln)
    if m and cur:
        op = m.group(1)
        funcs[cur]["_n"] += 1
        for s in SEL:
            if op == s or op.startswith(s + ".") and not (s == "MUFU.RSQ" and op.startswith("MUFU.RSQ64H")):
                funcs[cur][s] += 1
                break
names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
print("# SASS opcode counts of the round-2 build (cuobjdump -sass paper_2204_07921_b200/libcmg.so, sm_100a)\n")
print("Static instruction counts per kernel instantiation (selected opcodes): UTMALDG = TMA tensor load, UBLKCP = "
      "bulk async copy (cp.async.bulk), FFMA2/FADD2/FMUL2 = packed fp32x2, MUFU.RSQ64H/RCP64H = fp64 sqrt/div seeds, "
      "DFMA/DADD/DMUL = fp64 pipe, CALL = out-of-line calls (library sqrt/div range paths).\n")
print("| kernel | instructions | selected opcodes |\n|---|---|---|")
for (mangled, cnt), nm in sorted(zip(funcs.items(), names), key=lambda t: t[1]):
    if not nm.startswith(("void cmg::", "cmg::", "void (anonymous")) and "k_" not in nm:
        continue
    sel = ", ".join(f"{s} {cnt[s]}" for s in SEL if cnt[s])
    print(f"| `{nm[:110]}` | {cnt['_n']} | {sel} |")
