#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2j}; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py -m gpu -x -q -k "not knob" > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 900 python tools/sweep.py c1 c2 c4d2 c5 expo3d2m --reps 2 --kernels tile > $out/sweep_lowd.jsonl 2> $out/sweep_lowd.err; echo "sweep rc=$?" >> $out/status.txt
cat $out/sweep_lowd.jsonl | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_c2.csv python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $out/status.txt
timeout 600 python tools/e2e_pipeline.py c2 5 > $out/e2e_pipeline.txt 2>&1; echo "pipeline rc=$?" >> $out/status.txt
cat $out/status.txt
