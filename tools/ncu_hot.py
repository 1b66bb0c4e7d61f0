"""ncu --page source --csv dump -> SASS in address order with stall samples and the
dominant stall reason per instruction; prints windows around the hottest instructions.
usage: ncu_hot.py src.csv [min_samples] [context]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
si = hdr.index("Source"); ni = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed"); it = hdr.index("Avg. Threads Executed")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[2:] if len(r) > ni]
def val(r, i):
    try: return int(float(r[i]))
    except ValueError: return 0
hot = [k for k, r in enumerate(body) if val(r, ni) >= thr]
show = sorted({j for k in hot for j in range(max(0, k - ctx), min(len(body), k + ctx + 1))})
prev = -2
for j in show:
    if j != prev + 1: print("   ...")
    prev = j
    r = body[j]
    top = max(stalls, key=lambda s: val(r, s[0]))
    print(f"{val(r, ni):5d} {val(r, ie):8d} {r[it][:5]:>5s} {top[1][6:]:12s} {r[0][-5:]} {r[si].strip()[:100]}")
