#!/usr/bin/env bash
# Result-pipeline schedules: e2e phases per (chunks, copies), tests of the public path, a bench line.
set -u
out=gpurun_out/${1:-e2e}; mkdir -p "$out"
timeout 900 python -m pytest tests/test_gpu_join.py tests/test_io_cli.py tests/test_gpu_parity.py -x -q -m gpu \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8 or c3 or c5)) and not brute_force_configs and not every_knob" \
  > "$out/pytest.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"; tail -1 "$out/pytest.log" >> "$out/status.txt"
timeout 900 python tools/e2e_pipeline.py c2 5 > "$out/e2e_pipeline.txt" 2>&1
timeout 600 python bench.py --skip-cpu > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
cat "$out/status.txt" "$out/e2e_pipeline.txt"
python -c "import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);print('bench',d['ms_per_step'],'e2e',d['e2e']['seconds'])"
