"""Summarise an ncu report: key SOL metrics and the top stalled SASS lines."""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issued Ipc Active", "Executed Instructions", "Registers Per Thread",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block", "L2 Hit Rate", "Grid Size", "Block Size")


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            res.append((d["ID"], d["Kernel Name"][:50], d["Metric Name"], d["Metric Value"], d["Metric Unit"]))
    return res


def raw(rep, pats):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        for i, name in enumerate(h):
            if any(p in name for p in pats):
                res.append((name, r[i]))
    return res


def hot(rep, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            h = r
            continue
        if r and r[0] == "Kernel Name":
            if data:
                break
            continue
        if h and r:
            data.append(r)
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = [h.index(c) for c in cols]
    tot = sum(int(x[si] or 0) for x in data)
    print(f"samples {tot}, executed {sum(int(x[ei] or 0) for x in data)}")
    for x in sorted(data, key=lambda x: -int(x[si] or 0))[:n]:
        rs = sorted(((c[6:], int(x[j] or 0)) for c, j in zip(cols, idx) if int(x[j] or 0)), key=lambda t: -t[1])[:2]
        print(f"{x[0][-5:]} {x[si]:>5} {x[ei]:>8} {x[1][:70]:70} {rs}")


if __name__ == "__main__":
    rep = sys.argv[1]
    for row in details(rep):
        print(*row)
    for name, v in raw(rep, ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_op")):
        print(name, v)
    hot(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 25)
