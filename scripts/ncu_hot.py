"""Hot SASS lines (stall samples) of one kernel in an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-kernel-base", "function",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
sec = rows[starts[0]:(starts[1] if len(starts) > 1 else len(rows))]
h = [i for i, r in enumerate(sec) if r and r[0] == "Address"][0]
hdr = sec[h]; data = [r for r in sec[h + 1:] if len(r) == len(hdr)]
si, ie, wi = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x or 0)
tot = sum(f(r[ie]) for r in data); tw = sum(f(r[wi]) for r in data) or 1
print(f"warp-instr per unit {tot / units:.1f}")
for i in sorted(range(len(data)), key=lambda i: -f(data[i][wi]))[:int(sys.argv[4]) if len(sys.argv) > 4 else 16]:
    print(f"{i:5d} {f(data[i][wi]) / tw * 100:5.1f}% {f(data[i][ie]) / units:8.1f}/unit  {data[i][si][:90]}")
