#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2f}; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_join.py -m gpu -x -q -k "gram or estimate or overflow or small_join or ladder or lattice" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 600 python tools/gram_probe.py 400000 16 2 > $out/gram_probe.txt 2>&1
timeout 600 python tools/gram_probe.py 200000 64 2 >> $out/gram_probe.txt 2>&1; echo "gram probe rc=$?" >> $out/status.txt
cat $out/gram_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:refine_gram" -c 1 \
  -o $out/full_gram_d16 python tools/gram_probe.py 200000 16 1 > $out/ncu_gram.log 2>&1; echo "ncu gram rc=$?" >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
timeout 900 python tools/sweep.py c4d16 c4d32 c4d64 --reps 1 --kernels tile > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep rc=$?" >> $out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c4d16 or c4d32 or c4d64 or brute" > $out/pytest_parity_hd.log 2>&1; echo "parity hd rc=$?" >> $out/status.txt
cat $out/status.txt
