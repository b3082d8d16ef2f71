"""Stall samples per CUDA source line (ncu --print-source cuda,sass): where a
kernel's warps wait, with the dominant stall reasons of each line."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, res, tot = "?", None, [], 0.0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("",):
        f = lambda k: float(r[hdr.index(k)] or 0) if r[hdr.index(k)] not in ("-",) else 0.0
        samp = f("Warp Stall Sampling (All Samples)")
        tot += samp
        st = sorted(((f(k), k[6:]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
        res.append((samp, f"{fname}:{r[0]}", r[1][:70], ", ".join(f"{n}={v:.0f}" for v, n in st if v > 0),
                    f("Instructions Executed")))
res.sort(reverse=True)
for s, loc, src, st, ie in res[:top]:
    print(f"{s / tot * 100:5.1f}% {loc:24s} {src:70s} | {st}")
