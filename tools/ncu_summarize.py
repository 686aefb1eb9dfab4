"""Per-kernel DRAM bytes, L2 sectors and time of ONE propagate from an ncu
CSV (tools/ncu_configs.sh: --csv --print-units base, metrics
gpu__time_duration, dram__bytes_{read,write}, lts__t_sectors_srcunit_tex_op_
{read,atom,red,write}[_lookup_hit]) -> profiles/ncu_<cfg>_summary.json, which
bench.py reads for roofline.traffic and roofline.random_access.

    python tools/ncu_summarize.py c2 [gpurun_out/ncu_c2.csv]
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
cfg = sys.argv[1]
src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / f"ncu_{cfg}.csv"
lines = src.read_text().splitlines()
start_row = next(j for j, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start_row:]))
hdr = rows[0]
iK, iM, iV, iID = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
kern = {}
for r in rows[1:]:
    if len(r) <= iV:
        continue
    k = kern.setdefault(int(r[iID]), {"kernel": r[iK].split("(")[0].replace("void ", "")})
    k[r[iM]] = float(r[iV].replace(",", "")) if r[iV] else 0.0
ks = [kern[i] for i in sorted(kern)]
# the kernels of ONE propagate: after the last L2 flush, up to the last
# compress kernel (tiled compress: copy-in / compress / copy-out per tile)
first = max(i for i, k in enumerate(ks) if k["kernel"].endswith("k_flush")) + 1
stop = next((i for i in range(first, len(ks)) if "k_gains" in ks[i]["kernel"]), len(ks))   # memoize follows
last = max(i for i in range(first, stop) if "k_compress" in ks[i]["kernel"] or "k_tile_copy" in ks[i]["kernel"])
one = ks[first:last + 1]

S = "lts__t_sectors_srcunit_tex_op_"


def tot(key):
    return sum(k.get(key, 0.0) for k in one)


groups = {}
for k in one:
    name = k["kernel"].replace("imx::", "")
    g = groups.setdefault(name, {"launches": 0, "time_us": 0.0, "dram_read_B": 0.0, "dram_write_B": 0.0,
                                 "l2_read_sectors": 0.0, "l2_read_hit_sectors": 0.0, "l2_atom_sectors": 0.0,
                                 "l2_red_sectors": 0.0, "l2_write_sectors": 0.0})
    g["launches"] += 1
    g["time_us"] += k.get("gpu__time_duration.sum", 0.0) / 1e3
    g["dram_read_B"] += k.get("dram__bytes_read.sum", 0.0)
    g["dram_write_B"] += k.get("dram__bytes_write.sum", 0.0)
    g["l2_read_sectors"] += k.get(S + "read.sum", 0.0)
    g["l2_read_hit_sectors"] += k.get(S + "read_lookup_hit.sum", 0.0)
    g["l2_atom_sectors"] += k.get(S + "atom.sum", 0.0)
    g["l2_red_sectors"] += k.get(S + "red.sum", 0.0)
    g["l2_write_sectors"] += k.get(S + "write.sum", 0.0)
rd, wr = tot("dram__bytes_read.sum"), tot("dram__bytes_write.sum")
l2 = tot(S + "read.sum") + tot(S + "atom.sum") + tot(S + "red.sum") + tot(S + "write.sum")
t_us = tot("gpu__time_duration.sum") / 1e3
sys.path.insert(0, str(ROOT))
from paper_2008_03095_b200.build import source_hash  # noqa: E402

log = src.with_suffix(".log")
stamp = next((l.split("=", 1)[1].strip() for l in (log.read_text().splitlines() if log.exists() else [])
              if l.startswith("src_hash=")), None) or source_hash()
summary = {
    "config": cfg,
    "src_hash": stamp,
    "source": f"ncu --replay-mode application (tools/ncu_configs.sh), kernels of one propagate after an L2 flush; "
              f"serialised, cold-cache launch times",
    "dram_bytes_per_propagate": rd + wr,
    "dram_read_MB": rd / 1e6,
    "dram_write_MB": wr / 1e6,
    "l2_sectors_per_propagate": l2,
    "l2_read_hit_rate": tot(S + "read_lookup_hit.sum") / max(1.0, tot(S + "read.sum")),
    "kernel_time_us_serialized": t_us,
    "kernels": groups,
}
out = ROOT / "profiles" / f"ncu_{cfg}_summary.json"
out.write_text(json.dumps(summary, indent=1))
print(f"{cfg}: {len(one)} launches, DRAM {rd / 1e6:.1f} MB read + {wr / 1e6:.1f} MB write, "
      f"L2 {l2 / 1e6:.1f} M sectors, {t_us:.1f} us serialised -> {out.relative_to(ROOT)}")
for name, g in groups.items():
    print(f"  {name:32s} x{g['launches']:<4d} {g['time_us']:9.1f} us  DRAM {(g['dram_read_B'] + g['dram_write_B']) / 1e6:9.1f} MB"
          f"  L2 rd {g['l2_read_sectors'] / 1e6:7.1f}M (hit {g['l2_read_hit_sectors'] / max(1, g['l2_read_sectors']):.2f})"
          f" atom {g['l2_atom_sectors'] / 1e6:6.1f}M red {g['l2_red_sectors'] / 1e6:6.1f}M wr {g['l2_write_sectors'] / 1e6:6.1f}M")
