"""Per-kernel DRAM bytes / time of one propagate from an ncu CSV (raw page,
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)
-> profiles/r01_c2_ncu_full_propagate.json + profiles/ncu_c2_summary.json.

    python tools/ncu_summarize.py gpurun_out/prop_metrics.csv
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rows = list(csv.reader(open(sys.argv[1])))
# ncu --csv --print-units base: one row per (kernel, metric)
hdr = rows[0]
iK, iM, iV, iU = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                  hdr.index("Metric Unit"))
iID = hdr.index("ID")
kern = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    k = kern.setdefault(int(r[iID]), {"Kernel Name": r[iK]})
    v = float(r[iV].replace(",", "")) if r[iV] else 0.0
    unit = r[iU]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
             "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(unit, 1)
    k[r[iM]] = v * scale
ks = [kern[i] for i in sorted(kern)]
# the kernels of ONE propagate: from the last k_init / k_pull<1 up to and including k_compress
start = max(i for i, k in enumerate(ks) if "k_init" in k["Kernel Name"] or "k_pull<1" in k["Kernel Name"])
end = next(i for i in range(start, len(ks)) if "k_compress" in ks[i]["Kernel Name"])
one = ks[start:end + 1]
rd = sum(k.get("dram__bytes_read.sum", 0) for k in one)
wr = sum(k.get("dram__bytes_write.sum", 0) for k in one)
t = sum(k.get("gpu__time_duration.sum", 0) for k in one)
(ROOT / "profiles" / "r01_c2_ncu_full_propagate.json").write_text(json.dumps(one, indent=1))
(ROOT / "profiles" / "ncu_c2_summary.json").write_text(json.dumps({
    "config": "c2",
    "source": "profiles/r01_c2_ncu_full_propagate.json (ncu, kernels of one propagate, bytes in B, times in us)",
    "dram_bytes_per_propagate": rd + wr, "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
    "kernel_time_us_serialized": t}, indent=1))
print(f"{len(one)} kernels, read {rd/1e6:.1f} MB, write {wr/1e6:.1f} MB, {t:.1f} us serialized")
for k in one:
    print(f"  {k['Kernel Name'][:60]:60s} {k.get('gpu__time_duration.sum',0):8.1f} us "
          f"R {k.get('dram__bytes_read.sum',0)/1e6:7.1f} MB W {k.get('dram__bytes_write.sum',0)/1e6:7.1f} MB")
