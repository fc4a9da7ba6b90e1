#!/usr/bin/env bash
# Index-phase change check: the grid / join GPU tests, full-size digests of the low-d
# configs, then the index probe and a bench line.  usage: bash tools/gpu_ix.sh <tag>
set -u
tag=${1:-ix}; out=gpurun_out/$tag; mkdir -p "$out"
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py -x -q \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8)) and not brute_force_configs and not every_knob" \
  > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
tail -3 "$out/pytest_gpu.log" >> "$out/status.txt"
for c in c2 c5 c3 expo3d2m; do timeout 300 python tools/index_probe.py $c 10 >> "$out/index.txt" 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches_c5.csv" python tools/index_probe.py c5 2 > "$out/ncu_c5.log" 2>&1
python tools/launch_summary.py "$out/launches_c5.csv" > "$out/launches_c5_summary.txt" 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches_c2.csv" python tools/index_probe.py c2 2 > "$out/ncu_c2.log" 2>&1
python tools/launch_summary.py "$out/launches_c2.csv" > "$out/launches_c2_summary.txt" 2>&1
for c in c3 expo3d2m; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$out/launches_$c.csv" python tools/index_probe.py $c 2 > "$out/ncu_$c.log" 2>&1
  python tools/launch_summary.py "$out/launches_$c.csv" > "$out/launches_${c}_summary.txt" 2>&1
done
timeout 600 python bench.py --skip-cpu > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
cat "$out/status.txt" "$out/index.txt"; head -12 "$out/launches_c5_summary.txt"; head -12 "$out/launches_c2_summary.txt"
