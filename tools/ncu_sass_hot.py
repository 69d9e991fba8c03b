"""Aggregate an `ncu --page source --csv` (SASS view) export: samples and
instructions per opcode, and the top stall reasons."""
import collections
import csv
import gzip
import io
import sys


def main(path, top=25):
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    lines = raw.splitlines()
    # the export may hold several kernels: split on "Kernel Name" lines
    blocks, cur = [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    for b in blocks:
        name = next(csv.reader([b[0]]))[1]
        rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
        hdr = rows[0]
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        src = hdr.index("Source")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        ops = collections.defaultdict(lambda: [0, 0])
        stalls = collections.Counter()
        tot = 0
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            op = r[src].strip().split()[0] if r[src].strip() else "?"
            if op.startswith("@"):
                op = r[src].strip().split()[1]
            op = op.split(".")[0]
            s = int(float(r[si] or 0))
            ops[op][0] += s
            ops[op][1] += int(float(r[ii] or 0))
            tot += s
            for c in stall_cols:
                try:
                    stalls[hdr[c]] += int(float(r[c] or 0))
                except ValueError:
                    pass
        print(f"== {name[:100]}  samples={tot}")
        for op, (s, n) in sorted(ops.items(), key=lambda x: -x[1][0])[:top]:
            print(f"   {op:12s} {100 * s / max(tot, 1):5.1f}%  inst {n}")
        if stalls:
            print("   stalls:", ", ".join(f"{k}={v}" for k, v in stalls.most_common(10)))


if __name__ == "__main__":
    main(sys.argv[1])
