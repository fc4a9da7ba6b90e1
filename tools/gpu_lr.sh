#!/usr/bin/env bash
# Long-row changes: join/parity tests, Expo3D2M launch list, low-d sweep, bench line.
set -u
out=gpurun_out/${1:-lr}; mkdir -p "$out"
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py -x -q \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8)) and not brute_force_configs and not every_knob" \
  > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"; tail -1 "$out/pytest_gpu.log" >> "$out/status.txt"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches_expo.csv" python tools/sweep.py expo3d2m --reps 1 --kernels tile > "$out/ncu.log" 2>&1
python tools/launch_summary.py "$out/launches_expo.csv" > "$out/launches_expo_summary.txt" 2>&1
timeout 900 python tools/sweep.py c1 c2 c4d2 expo3d2m c5 c3 --reps 3 --kernels tile,scalar > "$out/sweep.jsonl" 2> "$out/sweep.err"
timeout 600 python bench.py --skip-cpu > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
cat "$out/status.txt"; head -8 "$out/launches_expo_summary.txt"
python - "$out" <<'P'
import json,sys
out=sys.argv[1]
for l in open(out+"/sweep.jsonl"):
    d=json.loads(l); print(d["config"], d["kernel"], round(d["index_ms"],3), round(d["refine_ms"],3), round(d["finalize_ms"],3), round(d["step_ms"],3))
d=json.loads(open(out+"/bench.json").read().strip().splitlines()[-1])
print("bench", round(d["ms_per_step"],4), d.get("phases_ms"), "e2e", d["e2e"].get("seconds"))
P
