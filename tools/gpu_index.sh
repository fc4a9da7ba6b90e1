#!/usr/bin/env bash
# Index-phase probe: build_grid timing at c2 / c5 (+ c3), per-kernel launch list of one build.
# usage: bash tools/gpu_index.sh <tag>
set -u
tag=${1:-ix}; out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1
for c in c2 c5 c3 expo3d2m; do timeout 300 python tools/index_probe.py $c 10 >> "$out/index.txt" 2>&1; done
for c in c2 c5 c3 expo3d2m; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$out/launches_$c.csv" python tools/index_probe.py $c 2 > "$out/ncu_$c.log" 2>&1
  python tools/launch_summary.py "$out/launches_$c.csv" > "$out/launches_${c}_summary.txt" 2>&1
done
cat "$out/index.txt"; head -30 "$out/launches_c2_summary.txt"
