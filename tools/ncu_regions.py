"""Group an ncu source-page CSV (``ncu -i R --page source --csv --print-source sass``)
into code regions of W SASS instructions and print, for every region above a sample
threshold, its share of the warp-stall samples, the dominant opcodes and the stall
reasons (tuning tool).

usage: python tools/ncu_regions.py SRC.csv [W] [MIN_PCT]
"""
import csv
import sys

f = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
MIN = float(sys.argv[3]) if len(sys.argv) > 3 else 0.6
rows = list(csv.reader(open(f)))
hdr, rows = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
tot = sum(int(r[2]) for r in rows)
print(f"total samples {tot}")
for s in range(0, len(rows), W):
    ch = rows[s:s + W]
    smp = sum(int(r[2]) for r in ch)
    if 100.0 * smp / tot < MIN:
        continue
    ops = {}
    for r in ch:
        t = r[1].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:6])
    rs = {k[6:]: sum(int(r[col[k]] or 0) for r in ch) for k in reasons}
    rtot = sum(rs.values()) or 1
    rtop = " ".join(f"{k}:{100 * v / rtot:.0f}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:5])
    ex = max(int(r[5]) if r[5].isdigit() else 0 for r in ch)
    print(f"{s:6d} {100 * smp / tot:5.1f}% exec={ex:>10d} | {top} | {rtop}")
