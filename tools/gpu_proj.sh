#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-proj}; mkdir -p "$out"
timeout 1500 python tools/strong_projection.py c5 2 4 8 > "$out/strong_projection.jsonl" 2> "$out/strong_projection.err"; echo "projection rc=$?"
python - "$out" <<'P'
import json,sys
for l in open(sys.argv[1]+"/strong_projection.jsonl"):
    x=json.loads(l)
    if "G" in x: print(x["G"], round(x["T_G_ms"],2), "eff", round(x["efficiency"],3), "serial", round(x["efficiency_serial_collectives"],3), {k:round(v,2) for k,v in x["slowest_rank"].items() if k.endswith("_ms")})
    else: print("T1", x["T1_ms"])
P
