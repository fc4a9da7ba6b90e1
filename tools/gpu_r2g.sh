#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2g}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 600 python tools/gram_probe.py 400000 16 2 > $out/gram_probe.txt 2>&1
timeout 600 python tools/gram_probe.py 200000 64 2 >> $out/gram_probe.txt 2>&1; echo "gram probe rc=$?" >> $out/status.txt
cat $out/gram_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:refine_gram" --launch-skip 1 -c 1 \
  -o $out/full_gram_d16 python tools/gram_probe.py 200000 16 1 > $out/ncu_gram.log 2>&1; echo "ncu gram rc=$?" >> $out/status.txt
timeout 900 python tools/sweep.py c4d16 c4d32 c4d64 --reps 1 --kernels tile > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep rc=$?" >> $out/status.txt
cat $out/status.txt
