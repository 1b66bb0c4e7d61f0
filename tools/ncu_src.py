"""Summarise an ncu --page source --csv dump: top SASS instructions by warp-stall samples."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Source"); ni = hdr.index("Warp Stall Sampling (All Samples)")
tot = 0; byop = collections.Counter(); top = []
for r in rows[2:]:
    if len(r) <= ni: continue
    try: v = int(r[ni])
    except ValueError: continue
    tot += v
    op = r[si].strip().split()[0] if r[si].strip() else "?"
    if op.startswith("@"): op = r[si].strip().split()[1]
    byop[op.split(".")[0]] += v
    top.append((v, r[0], r[si].strip()))
print("total samples", tot)
for op, v in byop.most_common(15): print(f"  {op:10s} {v:7d} {100*v/tot:5.1f}%")
for v, a, s in sorted(top, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v:6d} {a[-5:]} {s[:90]}")
