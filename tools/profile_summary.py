"""Summarise the round's ncu captures into profiles/ (launch list share, conv
--set full metrics, DRAM traffic per launch for bench.py's roofline)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            i = int(d["ID"])
            per.setdefault(i, {"name": d["Kernel Name"]})[d["Metric Name"]] = d["Metric Value"]
    return [(i, per[i]["name"], float(per[i]["gpu__time_duration.sum"]) / 1e3) for i in sorted(per)]


CONV = ("spconv_tc_kernel", "spconv_halo_kernel")


def is_conv(name):
    return any(c in name for c in CONV)


def first_frame(ls):
    """Kernels of the first full eager frame: from the first maps launch to the
    grid writer of the fused head (rowbits_grid_kernel, after the 14th conv)."""
    out, started, nconv = [], False, 0
    for i, name, us in ls:
        if "l0_flags_kernel" in name:
            if started and nconv:
                break
            started, out, nconv = True, [], 0
        if not started or "pack_weights" in name or name.startswith("void at::") or name.startswith("at::"):
            continue  # one-time weight packing (first eager frame only; never in the graph)
        out.append((i, name, us))
        if is_conv(name):
            nconv += 1
        if "rowbits_grid" in name or nconv == 15:
            break
    return out


def raw(rep, metrics):
    """Metric values per launch; a metric may appear under a section prefix (e.g. TPC.TriageCompute.)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    col = {}
    for m in metrics:
        exact = [i for i, name in enumerate(h) if name == m]
        pref = [i for i, name in enumerate(h) if name.endswith("." + m)]
        if exact or pref:
            col[m] = (exact or pref)[0]
    return [{m: r[i] for m, i in col.items()} | {"name": r[h.index("Kernel Name")]} for r in rows[2:]]


def tensor_pct(r):
    """tcgen05 (hmma subpipe) busy cycles as a fraction of the SM's ACTIVE cycles,
    both in the SM clock domain (ncu's own pct_of_peak_sustained_active ratio;
    round 1 divided a realtime-clock count by SM-clock cycles, which could
    exceed 100 %)."""
    v = r.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active")
    try:
        return f"{float(v):.1f}"
    except (TypeError, ValueError):
        return "n/a"


def main(tag, launch_csv, conv_rep, maps_rep=None):
    md = [f"# ncu summary, {tag}", ""]
    ls = launches(launch_csv)
    fr = first_frame(ls)
    tot = sum(u for _, _, u in fr)
    conv = sum(u for _, n, u in fr if is_conv(n))
    md += [f"Launch list: `{os.path.basename(launch_csv)}` (`ncu --metrics gpu__time_duration.sum "
           "--clock-control none`, cold-cache, serialised).", "",
           f"First eager frame: {len(fr)} launches, {tot:.1f} us summed; sparse conv kernels (spconv_halo x10, "
           f"dec0b with the head fused, + spconv_tc x4: down01/12 gathers, up21/10 column blocks) "
           f"{conv:.1f} us = {100 * conv / tot:.1f}% of the frame.", "",
           "| # | kernel | us |", "|---|---|---|"]
    md += [f"| {i} | `{n[:70]}` | {u:.2f} |" for i, n, u in fr]
    mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]
    rs = raw(conv_rep, mets)
    md += ["", f"`--set full` capture `{os.path.basename(conv_rep)}` (first eager frame's 14 conv launches):", "",
           "| launch | kernel | us | DRAM read MB | DRAM write MB | grid | SM % | L2 % | tensor pipe % (of active SM cycles) |",
           "|---|---|---|---|---|---|---|---|---|"]
    dram = []
    names = ["enc0a", "enc0b", "down01", "enc1a", "enc1b", "down12", "enc2a", "enc2b", "up21", "dec1a", "dec1b",
             "up10", "dec0a", "dec0b+head"]

    def mb(v, unit_scale):
        try:
            return float(v) * unit_scale
        except ValueError:
            return 0.0
    for k, r in enumerate(rs):
        rd = mb(r.get("dram__bytes_read.sum", "0"), 1.0)
        wr = mb(r.get("dram__bytes_write.sum", "0"), 1.0)
        l2 = mb(r.get("lts__t_bytes.sum", "0"), 1.0)
        if k < 14:
            dram.append(rd + wr)
        kn = "halo" if "halo" in r["name"] else "tc"
        md.append(f"| {names[k] if k < len(names) else k} | {kn} | {r.get('gpu__time_duration.sum')} | {rd:.2f} | "
                  f"{wr:.2f} | {r.get('launch__grid_size')} | {r.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                  f"{r.get('lts__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                  f"{tensor_pct(r)} |")
    if maps_rep:
        mr = raw(maps_rep, mets)
        md += ["", f"`--set full` capture `{os.path.basename(maps_rep)}` (map kernels K1-K3 incl. every level's halo "
               "tables, and the fused head's grid writer):", "",
               "| kernel | us | DRAM read MB | grid |", "|---|---|---|---|"]
        for r in mr:
            md.append(f"| `{r['name'][:40]}` | {r.get('gpu__time_duration.sum')} | {r.get('dram__bytes_read.sum')} | "
                      f"{r.get('launch__grid_size')} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    tr = {"conv_dram_bytes_per_launch": 1e6 * sum(dram) / max(1, len(dram)),
          "source": f"profiles/{tag}_ncu_summary.md (dram__bytes_read.sum + dram__bytes_write.sum, mean of 14 conv "
                    "launches, ncu --set full, caches flushed between replays)"}
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
        json.dump(tr, fh, indent=1)
    print("\n".join(md[:8]))


if __name__ == "__main__":
    main(*sys.argv[1:])
