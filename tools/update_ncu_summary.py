"""Refresh profiles/ncu_summary.json (bench.py's roofline.traffic source) from a
tools/ncu_summary.py JSON of the c2 kernels.

    python tools/update_ncu_summary.py profiles/<dir>/ncu_full_c2.json
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src = Path(sys.argv[1]).resolve()
rows = [r for v in json.load(open(src)).values() for r in v]
out = {}
for key in ("refine_lowd_kernel", "count_rows_kernel", "emit_rows_kernel"):
    hit = [r for r in rows if key in r["kernel"]]
    if hit:
        r = hit[0]
        out[key] = {"kernel": r["kernel"], "dram_bytes_per_launch": r["dram_bytes_per_launch"],
                    "duration_ns": r["duration_ns"], "source": str(src.relative_to(ROOT))}
path = ROOT / "profiles" / "ncu_summary.json"
data = json.load(open(path)) if path.exists() else {}
data["c2"] = out
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data, indent=1))
