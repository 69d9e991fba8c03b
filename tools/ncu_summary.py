"""Summarise an `ncu --page raw --csv` export (optionally .gz) as a markdown table."""
import csv
import gzip
import io
import sys

COLS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2_hit_%", "lts__t_sector_hit_rate.pct"),
    ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("fp64_%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fma_%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("alu_%", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    ("xu_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("lsu_%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("smem_KB", "launch__shared_mem_per_block_dynamic"),
]
SCALE = {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3,
         "Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6, "Kbyte/block": 1.0, "byte/block": 1e-3}


def load(path):
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


def main(path, out=sys.stdout):
    hdr, units, rows = load(path)
    name_i = hdr.index("Kernel Name")
    cols = [(lab, hdr.index(m)) for lab, m in COLS if m in hdr]
    out.write("| kernel | " + " | ".join(l for l, _ in cols) + " |\n")
    out.write("|---" * (len(cols) + 1) + "|\n")
    for r in rows:
        name = r[name_i].split("(")[0].replace("void ", "").replace("cmg::", "")
        vals = []
        for lab, i in cols:
            v = r[i].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[i], 1.0) if lab in ("time_us", "dram_rd_MB", "dram_wr_MB", "smem_KB") \
                    else float(v)
                vals.append(f"{x:.1f}" if abs(x) < 1e5 else f"{x:.0f}")
            except ValueError:
                vals.append(v)
        out.write(f"| `{name}` | " + " | ".join(vals) + " |\n")


if __name__ == "__main__":
    main(sys.argv[1])
