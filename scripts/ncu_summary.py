"""Summarise an ncu report: key throughput metrics, stall reasons, hot SASS."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__inst_executed.avg.per_cycle_active", "lts__t_bytes.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
for w in want:
    if w in hdr:
        i = hdr.index(w); print(f"{w:70s} {vals[i]:>18s} {units[i]}")
st = [(float(vals[i] or 0), h) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
print("stalls per issue:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
for i, r in enumerate(rows):
    if r and r[0] == "Address":
        h = i; break
hdr = rows[h]; data = rows[h + 1:]
si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[wi] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -float(r[wi] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{float(r[wi]) / tot * 100:5.1f}%  {r[si][:100]}")
