#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2e}; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_dmma.py tests/test_distributed.py tests/test_io_cli.py -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 300 python tools/e2e_pipeline.py c2 5 > $out/e2e_pipeline.txt 2>&1; echo "pipeline rc=$?" >> $out/status.txt
cat $out/e2e_pipeline.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_pipeline.csv python tools/e2e_pipeline.py c2 1 > $out/ncu_pipeline.log 2>&1; echo "ncu pipeline rc=$?" >> $out/status.txt
timeout 600 python tools/gram_probe.py 400000 16 2 > $out/gram_probe.txt 2>&1
timeout 600 python tools/gram_probe.py 200000 64 2 >> $out/gram_probe.txt 2>&1; echo "gram probe rc=$?" >> $out/status.txt
cat $out/gram_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:refine_gram" -c 1 \
  -o $out/full_gram_d16 python tools/gram_probe.py 200000 16 1 > $out/ncu_gram.log 2>&1; echo "ncu gram rc=$?" >> $out/status.txt
timeout 900 python tools/sweep.py c4d16 c4d32 c4d64 --reps 1 --kernels tile > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep rc=$?" >> $out/status.txt
cat $out/status.txt
