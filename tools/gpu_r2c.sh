#!/usr/bin/env bash
# round-2 check: GPU suite, c2 bench (chunked D2H pipeline), Gram-kernel sweep, ncu
set -u
out=gpurun_out/${1:-r2c}; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" >> $out/status.txt
timeout 900 python tools/sweep.py c4d16 c4d32 c4d64 c4d8 c3 --reps 1 --kernels tile > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep rc=$?" >> $out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_c2.csv python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:refine_gram" -c 1 \
  -o $out/full_gram_d16 python tools/sweep.py c4d16 --reps 1 --kernels tile > $out/ncu_gram.log 2>&1; echo "ncu gram rc=$?" >> $out/status.txt
timeout 600 python tools/e2e_probe.py c2 4 > $out/e2e_probe.txt 2>&1; echo "e2e probe rc=$?" >> $out/status.txt
cat $out/status.txt
