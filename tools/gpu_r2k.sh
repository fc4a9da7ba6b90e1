#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2k}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" >> $out/status.txt
timeout 1800 python tools/sweep.py c4d16 c4d32 c4d64 --reps 1 --kernels tile,core_expanded > $out/sweep_hd.jsonl 2> $out/sweep_hd.err; echo "sweep hd rc=$?" >> $out/status.txt
cat $out/sweep_hd.jsonl | cut -c1-300
timeout 600 python tools/refine_only.py 400000:16:0.657508 core_expanded 2 > $out/rate_d16_core_expanded.txt 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:refine_" --launch-skip 1 -c 1 -o /tmp/kce python tools/refine_only.py 400000:16:0.657508 core_expanded 2 > $out/ncu_ce.log 2>&1
python tools/ncu_summary.py /tmp/kce.ncu-rep > $out/ncu_d16_core_expanded.json 2>>$out/status.txt; echo "ncu ce rc=$?" >> $out/status.txt
timeout 2400 python tools/make_bf_digests.py c4d64 > $out/bf_c4d64.log 2>&1; echo "bf c4d64 rc=$?" >> $out/status.txt
cp tests/golden/bf_digests.json $out/ 2>/dev/null
cat $out/status.txt
