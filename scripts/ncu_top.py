"""Top utilisation metrics of one kernel in an ncu report (the limiter is
usually the largest pct_of_peak): python scripts/ncu_top.py REP [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
out = []
for i, h in enumerate(hdr):
    if "pct_of_peak_sustained" in h and ".max." not in h:
        try:
            out.append((float(vals[i]), h))
        except ValueError:
            pass
for v, h in sorted(out, reverse=True)[:n]:
    print(f"{v:8.2f}  {h}")
