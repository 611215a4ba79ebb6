"""Per-CUDA-source-line instruction / stall totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(r for r in rows if r and r[0] == "Line No")
ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg, cur, fname = {}, None, ""
for r in rows:
    if not r or r[0] == "Line No":
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:100])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None or len(r) <= ie:
        continue
    try:
        agg[cur][0] += int(r[ie])
        agg[cur][1] += int(r[st])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot}, stall samples {tots}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:14]:14s}:{k[1]:<4d} {100 * v[0] / tot:5.1f}% inst {100 * v[1] / tots:5.1f}% stall  {k[2]}")
