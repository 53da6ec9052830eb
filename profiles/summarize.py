"""Summarise ncu reports (gpurun_out/*.ncu-rep) into the markdown kept in profiles/.
Usage: python profiles/summarize.py OUT.md label=path.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time_us", 1.0),
    ("dram__bytes_read.sum", "dram_rd_MB", 1.0),
    ("dram__bytes_write.sum", "dram_wr_MB", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak", 1.0),
    ("smsp__inst_executed.sum", "warp_inst_M", 1e-6),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_%", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%", 1.0),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb_stall", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__grid_size", "grid", 1.0),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        yield d, u


def main():
    out = sys.argv[1]
    lines = ["| label | kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---" * (len(KEYS) + 2) + "|"]
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        for d, u in rows(path):
            vals = []
            for k, name, sc in KEYS:
                v = d.get(k, "")
                try:
                    f = float(v.replace(",", ""))
                    unit = u.get(k, "")
                    if k == "gpu__time_duration.sum":
                        f *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
                    if k.startswith("dram__bytes"):
                        f *= {"byte": 1e-6, "KB": 1e-3, "Kbyte": 1e-3, "GB": 1e3, "Gbyte": 1e3}.get(unit, 1.0)
                    vals.append(f"{f * sc:.3g}")
                except ValueError:
                    vals.append(v)
            lines.append(f"| {label} | {d.get('Kernel Name', '')[:60]} | " + " | ".join(vals) + " |")
    with open(out, "a") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
