"""DRAM traffic of the dominant kernel per config -> profiles/k2_traffic_p<p>.json (the
`roofline.traffic` source of bench.py).  Run on the GPU box:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"k2_lu|k2s_condense" -s 1 -c 1 --csv --log-file X.csv \
      python tools/prof_k2.py --config C2 --n <one wave>
  python tools/k2_traffic.py X.csv <p> <leaves> <kernel-name> <source-note>
"""
import csv, json, os, sys

path, p, leaves, kernel, note = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
rd = wr = dur = None
with open(path) as fh:
    rows = [r for r in csv.reader(fh) if len(r) > 10]
hdr = rows[0]
im, iv, iu = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1}
for r in rows[1:]:
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    if r[im] == "dram__bytes_read.sum": rd = v
    elif r[im] == "dram__bytes_write.sum": wr = v
    elif r[im] == "gpu__time_duration.sum": dur = v
out = {"kernel": kernel, "p": p, "source": note, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "duration_s": dur, "leaves": leaves, "bytes_per_leaf": (rd + wr) / leaves}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", f"k2_traffic_p{p}.json"), "w") as fh:
    json.dump(out, fh)
print(json.dumps(out))
