#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2m}; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log
grep "pairs expansion" -r $out/pytest_gpu.log
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
cat $out/strong_projection.jsonl | cut -c1-300
TJ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > $out/bench_n2_strong_c2.json 2> $out/bench_n2_strong_c2.err; echo "bench n2 rc=$?" >> $out/status.txt
timeout 600 python -m pytest tests/test_io_cli.py -m gpu -q -s -k pairs_expansion > $out/pairs_expansion.log 2>&1
cat $out/status.txt
