"""Per-launch table from an ncu --csv --print-units base metrics log:
    python tools/launch_table.py gpurun_out/x_launches.csv [last_n]"""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
i = next(j for j, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
hdr = rows[0]
iK, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
k = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    d = k.setdefault(int(r[iID]), {"n": r[iK].split("(")[0][:48]})
    d[r[iM]] = float(r[iV].replace(",", ""))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for i in sorted(k)[-last:]:
    d = k[i]
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    rd = d.get("dram__bytes_read.sum", 0) / 1e6
    wr = d.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:4d} {d['n']:48s} {t:10.1f} us {rd:10.1f} MB r {wr:10.1f} MB w {((rd + wr) / 1e3) / (t / 1e6) if t else 0:8.0f} GB/s")
