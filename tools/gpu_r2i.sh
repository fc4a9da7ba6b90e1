#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2i}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" >> $out/status.txt
timeout 900 python tools/sweep.py c1 c2 c4d2 c5 expo3d2m --reps 2 --kernels tile > $out/sweep_lowd.jsonl 2> $out/sweep_lowd.err; echo "sweep rc=$?" >> $out/status.txt
TJ_SYMMETRIC=0 timeout 900 python tools/sweep.py c2 c5 --reps 2 --kernels tile > $out/sweep_lowd_nosym.jsonl 2>> $out/sweep_lowd.err; echo "sweep nosym rc=$?" >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_c2.csv python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:refine_lowd|emit_rows|count_rows" -c 3 \
  -o $out/full_c2 python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $out/status.txt
timeout 1800 python tools/sweep.py c4d2 c4d8 c3 c5 expo3d2m --reps 2 --kernels scalar,core_fma,core_expanded > $out/sweep_core.jsonl 2> $out/sweep_core.err; echo "sweep core rc=$?" >> $out/status.txt
timeout 1500 bash tools/kernel_ncu.sh $out/kncu > $out/kncu.log 2>&1; echo "kernel ncu rc=$?" >> $out/status.txt
du -sh $out >> $out/status.txt
cat $out/status.txt
