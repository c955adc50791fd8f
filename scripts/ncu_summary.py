"""Summarise .ncu-rep captures into a small text table (committed under profiles/).

usage: python scripts/ncu_summary.py OUT.txt REP1.ncu-rep [REP2 ...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_size", "cluster"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units, data = r[0], r[1], r[2:]
    for d in data:
        rec = dict(zip(head, d))
        u = dict(zip(head, units))
        yield rec, u


def fmt(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if unit == "byte":
        return f"{x / 1e9:.3f} GB"
    if unit in ("Tbyte",):
        return f"{x * 1e3:.3f} GB"
    if unit == "Kbyte":
        return f"{x / 1e6:.3f} GB"
    if unit == "Mbyte":
        return f"{x / 1e3:.3f} GB"
    if unit == "Gbyte":
        return f"{x:.3f} GB"
    if unit in ("nsecond", "ns"):
        return f"{x / 1e3:.1f} us"
    if unit in ("usecond", "us"):
        return f"{x:.1f} us"
    if unit in ("msecond", "ms"):
        return f"{x * 1e3:.1f} us"
    return f"{x:g}{'%' if unit == '%' else ''}"


def main():
    out_path, reps = sys.argv[1], sys.argv[2:]
    lines = []
    for rep in reps:
        lines.append(f"== {rep.split('/')[-1]}")
        for rec, u in rows(rep):
            name = rec.get("Kernel Name", "?")
            name = name.split("(")[0][:60]
            parts = [f"{lab}={fmt(rec.get(m, 'n/a'), u.get(m, ''))}" for m, lab in METRICS if m in rec]
            lines.append(f"{name}: " + ", ".join(parts))
    text = "\n".join(lines) + "\n"
    open(out_path, "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
