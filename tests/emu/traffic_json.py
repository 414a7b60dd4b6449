"""Dev tool: profiles/ncu_traffic.json from an ncu CSV of the named launches.

ncu --nvtx --nvtx-include "walk_chunks/" ... --metrics \
  dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none --csv --log-file X.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline
python tests/emu/traffic_json.py X.csv profiles/<name>.csv [config] (the CSV is copied
there; the JSON entry of the config -- default c2 -- cites it)
"""
import csv
import collections
import json
import re
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]


def main():
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    config = sys.argv[3] if len(sys.argv) > 3 else "c2"
    command = sys.argv[4] if len(sys.argv) > 4 else f"bench.py --config {config} --steps 1 --warmup 1 --no-cpu-baseline"
    rows = [r for r in csv.reader(open(src)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    ti = next(i for i, h in enumerate(hdr) if "Push/Pop_Range" in h)
    mi, vi, ii = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.defaultdict(dict)  # launch id -> {tag, metric: value}
    for r in rows:
        if r[0] == "ID" or len(r) != len(hdr):
            continue
        m = re.search(r":([A-Za-z_]+):none", r[ti])
        if not m:
            continue
        d = per[r[ii]]
        d["tag"] = m.group(1)
        d[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: collections.Counter())
    for d in per.values():
        a = agg[d["tag"]]
        a["launches"] += 1
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
        a["ns"] += d.get("gpu__time_duration.sum", 0.0)
    shutil.copy(src, dst)
    rel = dst.relative_to(ROOT) if dst.is_absolute() else dst
    source = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              f"--clock-control none on `{command}`; "
              f"mean over the launches of the run (warm-up, step and e2e runs); {rel}")
    out = {}
    for tag, a in sorted(agg.items()):
        n = a["launches"]
        out[tag] = {"launches": n, "dram_bytes_per_launch": (a["rd"] + a["wr"]) / n,
                    "dram_read_bytes_per_launch": a["rd"] / n, "dram_write_bytes_per_launch": a["wr"] / n,
                    "ncu_ns_per_launch": a["ns"] / n, "source": source}
    db_path = ROOT / "profiles" / "ncu_traffic.json"
    db = json.loads(db_path.read_text()) if db_path.exists() else {}
    db[config] = out
    db_path.write_text(json.dumps(db, indent=1) + "\n")
    for tag, e in out.items():
        print(f"{tag:18s} x{e['launches']} {e['dram_bytes_per_launch'] / 1e9:8.2f} GB/launch "
              f"{e['ncu_ns_per_launch'] / 1e6:7.2f} ms")


if __name__ == "__main__":
    main()
