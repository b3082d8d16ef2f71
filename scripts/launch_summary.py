"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): launches, total ms, share; units normalised (ncu mixes ms/us/ns).
    python scripts/launch_summary.py gpurun_out/<tag>_launches.csv "<command line>" > profiles/..."""
import csv
import sys

SCALE = {"second": 1e3, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "s": 1e3, "ms": 1.0,
         "us": 1e-3, "ns": 1e-6}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
per, tot = {}, 0.0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    ms = float(r[vi].replace(",", "")) * SCALE[r[ui]]
    name = r[ki].split("(")[0].replace("void ", "")
    n, t = per.get(name, (0, 0.0))
    per[name] = (n + 1, t + ms)
    tot += ms
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# whole process, cold-cache and serialised per launch; ms per kernel name")
for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
    print(f"{k[-64:]:64s} {n:4d} launches {t:10.3f} ms {t / tot * 100:6.1f}%")
