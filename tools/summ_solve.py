"""Summarise an ncu per-launch CSV of one solve (tools/prof_solve.py):
per kernel class time / DRAM bytes / achieved GB/s; coarse SYMV launches
(those following a k_front_* launch) are reported per launch."""
import collections
import csv
import sys

rows = collections.OrderedDict()
for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')):
    k = int(r["ID"])
    d = rows.setdefault(k, {"name": r["Kernel Name"].split("(")[0], "grid": r["Grid Size"],
                            "block": r["Block Size"]})
    v = float(r["Metric Value"].replace(",", ""))
    d[r["Metric Name"]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
prev = ""
coarse = []
for k, d in rows.items():
    name = d["name"]
    t = d.get("gpu__time_duration.sum", 0) * 1e-9
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    cls = name
    if name.startswith("k_symv") and prev.startswith("k_front"):
        cls = name + "[coarse]"
        coarse.append((k, d["grid"], t * 1e6, b / 1e6, b / max(t, 1e-12) / 1e9))
    a = agg[cls]
    a[0] += 1
    a[1] += t
    a[2] += b
    prev = name
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':32s} {'n':>5s} {'ms':>9s} {'share':>6s} {'GB':>8s} {'GB/s':>7s}")
for cls, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{cls:32s} {n:5d} {t*1e3:9.3f} {t/tot:6.1%} {b/1e9:8.3f} {b/max(t,1e-12)/1e9:7.0f}")
print(f"total {tot*1e3:.3f} ms")
if coarse and "-v" in sys.argv:
    print("coarse symv launches: id grid us MB GB/s")
    for c in coarse:
        print("  ", c[0], c[1], f"{c[2]:.1f} {c[3]:.2f} {c[4]:.0f}")
