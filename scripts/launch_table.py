"""Per-launch table (duration us, DRAM MB read/write) from an ncu --csv
launch list with gpu__time_duration.sum and dram__bytes_{read,write}.sum."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: j for j, h in enumerate(hdr)}
k = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    d = k.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = 0.0
for i in sorted(k):
    if i < first:
        continue
    d = k[i]
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    print(f"{i:3d} {t:8.1f} us  rd {d.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB  "
          f"wr {d.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB  {d['name'][:90]}")
print(f"total {tot:.1f} us")
