"""Writes profiles/<tag>_*.txt/json from gpurun_out ncu artefacts:
launch list shares, per-kernel key metrics, DRAM traffic per launch."""
import csv, json, os, subprocess, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go, pr = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")
os.makedirs(pr, exist_ok=True)

# launch list -> per-kernel time shares
rows = [r for r in csv.reader(open(os.path.join(go, f"launches_{tag}.csv"))) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, per = 0.0, {}
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
    per.setdefault(name, [0, 0.0])
    per[name][0] += 1
    per[name][1] += v
    tot += v
unit = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"][0][hdr.index("Metric Unit")]
with open(os.path.join(pr, f"{tag}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    f.write(f"# python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e ; unit {unit}\n")
    f.write(f"{'kernel':40s} {'launches':>8s} {'total':>12s} {'share':>7s}\n")
    for k, (n, v) in sorted(per.items(), key=lambda x: -x[1][1]):
        f.write(f"{k:40s} {n:8d} {v:12.1f} {v / tot * 100:6.1f}%\n")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"]
traffic = {}
for kern in ("ws_factor", "ws_core16"):
    raw = subprocess.run(["ncu", "-i", os.path.join(go, f"{tag}_{kern}.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    d = {k: (v[i], u[i]) for i, k in enumerate(h)}
    with open(os.path.join(pr, f"{tag}_{kern}_ncu.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{kern} -s 1 -c 1\n")
        f.write(f"# kernel: {d['Kernel Name'][0]}\n")
        for w in want:
            if w in d:
                f.write(f"{w:75s} {d[w][0]:>20s} {d[w][1]}\n")
        st = sorted(((float(v[i] or 0), k) for i, k in enumerate(h)
                     if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")),
                    reverse=True)[:8]
        f.write("stalls per issue: " + ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={x:.2f}" for x, k in st) + "\n")
    def to_bytes(val, unit):
        x = float(val.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    b = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
    traffic[f"netflix_j32_tf32_{'core' if 'core' in kern else 'factor'}"] = b
json.dump(traffic, open(os.path.join(pr, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(pr, f"{tag}_launches.txt")).read())
print(json.dumps(traffic))
