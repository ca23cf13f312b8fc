"""Per-source-line warp-stall samples from an ncu report (--set full --import-source on).
Usage: python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, timeout=600).stdout
rows, hdr, f, tot = [], None, None, 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
    elif row[0] == "Line No" and hdr is None:
        hdr = row
    elif len(row) > 6 and row[2] == "-" and row[0].isdigit():
        s = int(row[4]); tot += s
        rows.append((s, f, int(row[0]), row[1].strip()[:80], row))
idx = {n[6:]: i for i, n in enumerate(hdr) if n.startswith("stall_") and "(Not" not in n}
rows.sort(key=lambda r: -r[0])
print("total samples", tot)
for s, f, l, src, row in rows[:top]:
    st = sorted(((int(row[i]) if row[i].isdigit() else 0, n) for n, i in idx.items()), reverse=True)[:3]
    print(f"{s:7d} {100 * s / tot:5.1f}% {f}:{l} {src} | " + ", ".join(f"{n}={v}" for v, n in st))
