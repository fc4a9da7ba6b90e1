#!/usr/bin/env bash
# Shard-rank index probe (+ launch list) and the emit check.  usage: bash tools/gpu_sh.sh <tag>
set -u
tag=${1:-sh}; out=gpurun_out/$tag; mkdir -p "$out"
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py tests/test_distributed.py -x -q \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8)) and not brute_force_configs and not every_knob" \
  > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
tail -2 "$out/pytest_gpu.log" >> "$out/status.txt"
timeout 600 python tools/shard_index_probe.py 8 7 10 >> "$out/shard_index.txt" 2>&1
timeout 600 python tools/shard_index_probe.py 2 1 6 >> "$out/shard_index.txt" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches_shard8.csv" python tools/shard_index_probe.py 8 7 2 > "$out/ncu_shard.log" 2>&1
python tools/launch_summary.py "$out/launches_shard8.csv" > "$out/launches_shard8_summary.txt" 2>&1
timeout 900 python tools/sweep.py c1 c2 c4d2 expo3d2m c5 --reps 3 --kernels tile > "$out/sweep.jsonl" 2> "$out/sweep.err"
timeout 600 python bench.py --skip-cpu > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
cat "$out/status.txt" "$out/shard_index.txt"; head -25 "$out/launches_shard8_summary.txt"
python - "$out" <<'P'
import json,sys
out=sys.argv[1]
for l in open(out+"/sweep.jsonl"):
    d=json.loads(l); print(d["config"], round(d["index_ms"],3), round(d["refine_ms"],3), round(d["finalize_ms"],3), round(d["step_ms"],3))
d=json.loads(open(out+"/bench.json").read().strip().splitlines()[-1])
print("bench", round(d["ms_per_step"],4), d.get("phases_ms"), "e2e", d["e2e"].get("seconds"))
P
timeout 900 python tools/strong_projection.py c5 2 4 8 > "$out/strong_projection.jsonl" 2> "$out/strong_projection.err"; echo "projection rc=$?" >> "$out/status.txt"
python - "$out" <<'P'
import json,sys
for l in open(sys.argv[1]+"/strong_projection.jsonl"):
    x=json.loads(l)
    if "G" in x: print(x["G"], round(x["T_G_ms"],2), "eff", round(x["efficiency"],3), "serial", round(x["efficiency_serial_collectives"],3), {k:round(v,3) for k,v in x["slowest_rank"].items() if k.endswith("_ms")})
    else: print("T1", x["T1_ms"])
P
