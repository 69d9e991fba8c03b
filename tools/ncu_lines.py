"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python tools/ncu_lines.py <src.csv[.gz]> <kernel-substring> <cubin> [top]

The `ncu --page source --csv` export holds per-SASS-instruction samples with
absolute addresses; `nvdisasm -g` of the same build's cubin (extract it with
`cuobjdump -xelf all libcmg.so`) maps instruction offsets to the innermost
(inlined) source line.  Samples are summed over every launch of the kernel in
the export and printed per file:line, hottest first.
"""
import collections
import csv
import gzip
import io
import re
import subprocess
import sys


def sass_lines(cubin, mangled_sub):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    funcs = {}
    cur, loc = None, "?"
    for ln in out.splitlines():
        m = re.match(r"^\.text\.(\S+):", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = {}
            loc = "?"
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and cur:
            funcs[cur][int(m.group(1), 16)] = (loc, m.group(2).strip())
    return funcs


def main(src, ksub, cubin, top=40):
    raw = gzip.open(src, "rt").read() if src.endswith(".gz") else open(src).read()
    blocks, cur = [], None
    for ln in raw.splitlines():
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    agg = collections.Counter()
    inst = collections.Counter()
    name = None
    for b in blocks:
        kname = next(csv.reader([b[0]]))[1]
        if ksub not in kname:
            continue
        name = kname
        rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
        hdr = rows[0]
        ai, si, ii = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
            "Instructions Executed")
        base = None
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            a = int(r[ai], 16)
            base = a if base is None else base
            agg[a - base] += int(float(r[si] or 0))
            inst[a - base] += int(float(r[ii] or 0))
    if name is None:
        sys.exit(f"no kernel matching {ksub!r}")
    funcs = sass_lines(cubin, None)
    # pick the function whose instruction count matches the export
    nins = max(agg) // 16 + 1
    cands = [f for f, d in funcs.items() if max(d) // 16 + 1 == nins]
    want = re.findall(r"<(.*)>", name)
    f = cands[0] if len(cands) == 1 else None
    if f is None:
        sys.exit(f"ambiguous or missing function for {name}: {cands[:5]}")
    per = collections.Counter()
    peri = collections.Counter()
    for off, s in agg.items():
        loc = funcs[f].get(off, ("?", ""))[0]
        per[loc] += s
        peri[loc] += inst[off]
    tot = sum(per.values())
    print(f"== {name}  ({f})  samples={tot}")
    for loc, s in per.most_common(int(top)):
        print(f"  {100.0 * s / tot:5.1f}%  {s:6d}  inst {peri[loc]:9d}  {loc}")


if __name__ == "__main__":
    main(*sys.argv[1:])
