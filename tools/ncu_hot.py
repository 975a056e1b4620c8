"""Hot instructions of one ncu capture: the SASS lines with the most warp-stall
samples, each with its two dominant stall reasons and the instructions just
before it (where the stalled operand was produced).

  python tools/ncu_hot.py gpurun_out/x.ncu-rep [top=30] [context=2]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 2
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
st = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(int(r[iS]) for r in data)
print(f"{rows[0][1][:100]}\nsamples {tot}, instructions {sum(int(r[iE]) for r in data)}")
agg = {}
for r in data:
    for i in st:
        agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
hot = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:top]
shown = set()
for i in sorted(hot):
    r = data[i]
    reasons = sorted(((int(r[j] or 0), h[j][6:]) for j in st), reverse=True)[:2]
    for k in range(max(0, i - ctx), i):
        if k not in shown:
            print(f"      {k:5d} {data[k][1].strip()[:70]}")
            shown.add(k)
    print(f"  ->  {i:5d} {r[1].strip()[:70]:70s} {int(r[iS]):6d} ({100 * int(r[iS]) / tot:4.1f}%) "
          f"{' '.join(f'{n}:{v}' for v, n in reasons)} exec {r[iE]}")
    shown.add(i)

# per CUDA source line (needs -lineinfo): instructions executed and stall samples
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, agg = "?", "?", {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if len(r) > 7 and r[0] and r[2] == "":          # a CUDA line row
        line = (fname, r[0], r[1].strip()[:80])
        continue
    if len(r) > 7 and r[0] and r[2]:
        # combined row: Line No, Source, Address, Sass, samples..., executed at index 7
        line = (fname, r[0], r[1].strip()[:80]) if r[0] else line
    try:
        smp, ex = int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(line, [0, 0])
    a[0] += smp
    a[1] += ex
tot_s = sum(v[0] for v in agg.values()) or 1
tot_e = sum(v[1] for v in agg.values()) or 1
print("\nper source line: stall samples %, instructions %")
for k, v in sorted(agg.items(), key=lambda x: -(x[1][0] / tot_s + x[1][1] / tot_e))[:top]:
    print(f"  {k[0]}:{k[1]:>5} {100 * v[0] / tot_s:5.1f}% {100 * v[1] / tot_e:5.1f}%  {k[2]}")
