#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-hw}; mkdir -p "$out"
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py -x -q \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8 or c5)) and not brute_force_configs and not every_knob" \
  > "$out/pytest.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"; tail -1 "$out/pytest.log" >> "$out/status.txt"
for c in expo3d2m c3 c2; do timeout 300 python tools/index_probe.py $c 10 >> "$out/index.txt" 2>&1; done
cat "$out/status.txt" "$out/index.txt"
