#!/usr/bin/env bash
# Iteration loop on the GPU box: gpu tests, one bench line, launch list, full
# capture of the named kernels.  usage: bash tools/gpu_quick.sh <tag> [kernel-regex] [bench args]
set -u
tag=${1:-q}
kre=${2:-refine_|emit_rows}
shift; [ $# -gt 0 ] && shift
bargs="$*"
out=gpurun_out/$tag
mkdir -p "$out"
timeout 900 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
tail -3 "$out/pytest_gpu.log"
timeout 600 python bench.py --skip-cpu $bargs > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file "$out/launches.csv" python bench.py --steps 1 --warmup 3 --skip-cpu $bargs \
  > "$out/ncu_launch.log" 2>&1; echo "ncu launches rc=$?" >> "$out/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c 3 \
  -o "$out/full" python bench.py --steps 1 --warmup 3 --skip-cpu $bargs \
  > "$out/ncu_full.log" 2>&1; echo "ncu full rc=$?" >> "$out/status.txt"
cat "$out/status.txt"
