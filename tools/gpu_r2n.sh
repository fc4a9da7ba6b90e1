#!/usr/bin/env bash
set -u
out=gpurun_out/${1:-r2n}; mkdir -p $out
timeout 900 python -m pytest tests/test_distributed.py -m gpu -x -q > $out/pytest_dist.log 2>&1; echo "pytest dist rc=$?" >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
cat $out/strong_projection.jsonl | cut -c1-400
cat $out/status.txt
