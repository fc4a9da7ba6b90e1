#!/usr/bin/env bash
# Expo3D2M output-phase breakdown: launch list of one join + row-length histogram.
set -u
out=gpurun_out/${1:-expo}; mkdir -p "$out"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$out/launches_expo.csv" python tools/sweep.py expo3d2m --reps 1 --kernels tile > "$out/ncu.log" 2>&1
python tools/launch_summary.py "$out/launches_expo.csv" > "$out/launches_expo_summary.txt" 2>&1
timeout 300 python tools/rowlen_hist.py expo3d2m > "$out/rowlen.txt" 2>&1
cat "$out/launches_expo_summary.txt" | head -30; cat "$out/rowlen.txt" | tail -20
