"""Markdown table of per-launch metrics from ncu --set full reports (raw page)."""
import csv
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", "us"), ("dram__bytes_read.sum", "DRAM rd MB", "MB"),
        ("dram__bytes_write.sum", "DRAM wr MB", "MB"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", None),
        ("sm__inst_executed.avg.per_cycle_active", "IPC/SM", None),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %", None),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", None),
        ("launch__grid_size", "grid", None), ("launch__registers_per_thread", "regs", None)]
SCALE = {"nsecond": {"us": 1e-3}, "ns": {"us": 1e-3}, "usecond": {"us": 1.0}, "us": {"us": 1.0}, "msecond": {"us": 1e3}, "ms": {"us": 1e3},
         "byte": {"MB": 1e-6}, "Kbyte": {"MB": 1e-3}, "Mbyte": {"MB": 1.0}, "Gbyte": {"MB": 1e3}}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for v in r[2:]:
        yield dict(zip(h, v)), dict(zip(h, units))


print("| kernel | " + " | ".join(c[1] for c in COLS) + " |")
print("|---" * (len(COLS) + 1) + "|")
for rep in sys.argv[1:]:
    for d, u in rows(rep):
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        vals = []
        for k, _, sc in COLS:
            x = d.get(k, "")
            try:
                f = float(x.replace(',', ''))
                if sc is not None:
                    f *= SCALE.get(u.get(k, ""), {}).get(sc, float("nan"))
                vals.append(f"{f:.2f}")
            except ValueError:
                vals.append("n/a")
        print(f"| `{name}` | " + " | ".join(vals) + " |")
