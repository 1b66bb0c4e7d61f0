"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) into
markdown (stdout) and, with --traffic, update profiles/traffic.json with the
dominant mapping kernels' DRAM bytes per launch."""
import csv, json, sys, collections, os

def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ii = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[h + 1:]:
        if len(r) <= vi: continue
        try: v = float(r[vi].replace(",", ""))
        except ValueError: continue
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for i, m in per.items():
        name = names[i].split("(")[0].replace("void ", "")
        for k, v in m.items(): agg[name][k].append(v)
    return agg

agg = load(sys.argv[1])
tot = sum(sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"]) for m in agg.values())
print("| kernel | launches | mean us | share | DRAM read MB | DRAM write MB |")
print("|---|---|---|---|---|---|")
for name, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"]) / len(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    mean = sum(t) / len(t) / 1e3
    rd = sum(m.get("dram__bytes_read.sum", [0])) / max(1, len(m.get("dram__bytes_read.sum", [0]))) / 1e6
    wr = sum(m.get("dram__bytes_write.sum", [0])) / max(1, len(m.get("dram__bytes_write.sum", [0]))) / 1e6
    print(f"| `{name[:60]}` | {len(t)} | {mean:.1f} | {100 * mean * 1e3 / tot:.1f}% | {rd:.2f} | {wr:.2f} |")
if "--traffic" in sys.argv:
    key = sys.argv[sys.argv.index("--traffic") + 1]
    out = {}
    path = "profiles/traffic.json"
    if os.path.exists(path): out = json.load(open(path))
    for name, m in agg.items():
        if "k_gather" in name or "k_spread" in name or "k_bin" in name:
            b = [r + w for r, w in zip(m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", []))]
            if b: out.setdefault(key, {})[name.split("<")[0].split("::")[-1]] = sum(b) / len(b)
    json.dump(out, open(path, "w"), indent=1)
