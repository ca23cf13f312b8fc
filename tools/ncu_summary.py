"""Summarise an ncu report: headline metrics + top source lines by warp-stall samples."""
import csv, subprocess, sys, io

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]
print(f"## {rep}")
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:80s} {vals[i]:>16s} {units[i]}")
stalls = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            stalls.append((float(vals[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
stalls.sort(reverse=True)
print("stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = None
data = []
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if len(r) > 4 and r[2] == "-" and r[0].isdigit():
        try:
            data.append((int(r[4]), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
data.sort(reverse=True)
print(f"top source lines by warp-stall samples (total {tot}):")
for d in data[:top]:
    print(f"  {100 * d[0] / tot:5.1f}%  {d[1]}:{d[2]}  {d[3]}")
