#!/usr/bin/env bash
# Radix digit width A/B on the grid build (c2, c5, a c5 strong-layout rank).
set -u
out=gpurun_out/${1:-dg}; mkdir -p "$out"
for b in 8 10 11 6; do
  echo "digits<=$b" >> "$out/ab.txt"
  for c in c2 c5; do TJ_SORT_DIGIT_BITS=$b timeout 300 python tools/index_probe.py $c 10 >> "$out/ab.txt" 2>&1; done
  TJ_SORT_DIGIT_BITS=$b timeout 300 python tools/shard_index_probe.py 8 7 8 >> "$out/ab.txt" 2>&1
done
timeout 600 python -m pytest tests/test_gpu_join.py -x -q -k "grid or wide or sweep" > "$out/pytest.log" 2>&1; echo "pytest rc=$?" >> "$out/ab.txt"
tail -1 "$out/pytest.log" >> "$out/ab.txt"
cat "$out/ab.txt"
