#!/usr/bin/env bash
# One GPU session: tests, smoke, bench lines (both arms), ncu launch list + full
# captures of the c2 hot kernels, the all-config sweep, the e2e phase probe.
# usage (from the repo root, under gpurun):  bash tools/gpu_round.sh [tag]
set -u
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi > "$out/nvidia-smi.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?" >> "$out/status.txt"
timeout 900 python bench.py > "$out/bench_c2_tile.json" 2> "$out/bench_c2_tile.err"; echo "bench rc=$?" >> "$out/status.txt"
timeout 600 python bench.py --kernel scalar --skip-cpu > "$out/bench_c2_scalar.json" 2> "$out/bench_c2_scalar.err"; echo "bench scalar rc=$?" >> "$out/status.txt"
timeout 600 python bench.py --impl reference > "$out/bench_ref.json" 2> "$out/bench_ref.err"; echo "bench ref rc=$?" >> "$out/status.txt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file "$out/launches_c2_tile.csv" python bench.py --steps 1 --warmup 3 --skip-cpu \
  > "$out/ncu_launch.log" 2>&1; echo "ncu launches rc=$?" >> "$out/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:refine_lowd|emit_rows|count_rows" -c 3 \
  -o "$out/full_c2_tile" python bench.py --steps 1 --warmup 3 --skip-cpu \
  > "$out/ncu_full.log" 2>&1; echo "ncu full rc=$?" >> "$out/status.txt"
timeout 300 python tools/e2e_probe.py c2 4 > "$out/e2e_probe.txt" 2>&1; echo "e2e probe rc=$?" >> "$out/status.txt"
timeout 1800 python tools/sweep.py --reps 2 > "$out/sweep.jsonl" 2> "$out/sweep.err"; echo "sweep rc=$?" >> "$out/status.txt"
cat "$out/status.txt"
