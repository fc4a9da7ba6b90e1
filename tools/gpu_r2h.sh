#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2h}; mkdir -p $out
timeout 600 python tools/gram_probe.py 400000 16 2 > $out/gram_probe.txt 2>&1
timeout 600 python tools/gram_probe.py 200000 64 2 >> $out/gram_probe.txt 2>&1; echo "gram probe rc=$?" >> $out/status.txt
cat $out/gram_probe.txt
timeout 900 python tools/sweep.py c4d16 c4d32 c4d64 --reps 1 --kernels tile > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep hd rc=$?" >> $out/status.txt
cat $out/sweep_hd.jsonl | cut -c1-200
timeout 1800 python tools/sweep.py c1 c2 c4d2 c4d8 c3 c5 expo3d2m --reps 2 --kernels tile,scalar,core_fma,core_expanded > $out/sweep_all.jsonl 2> $out/sweep_all.err; echo "sweep all rc=$?" >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
timeout 1500 bash tools/kernel_ncu.sh $out/kncu > $out/kncu.log 2>&1; echo "kernel ncu rc=$?" >> $out/status.txt
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" >> $out/status.txt
timeout 600 python bench.py --config expo3d2m --skip-cpu > $out/bench_expo3d2m.json 2> $out/bench_expo3d2m.err; echo "bench expo rc=$?" >> $out/status.txt
cat $out/status.txt
