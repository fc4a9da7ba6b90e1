#!/usr/bin/env bash
# Emit-change check: GPU join tests + low-d full-size digests, the low-d sweep
# (DMMA kernel), a bench line and an ncu source capture of the emit kernel.
# usage: bash tools/gpu_emit.sh <tag>
set -u
tag=${1:-em}; out=gpurun_out/$tag; mkdir -p "$out"
timeout 1200 python -m pytest tests/test_gpu_join.py tests/test_gpu_parity.py -x -q \
  -k "not (full_pair_set and (c4d16 or c4d32 or c4d64 or c4d8)) and not brute_force_configs and not every_knob" \
  > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
tail -3 "$out/pytest_gpu.log" >> "$out/status.txt"
timeout 900 python tools/sweep.py c1 c2 c4d2 expo3d2m c5 --reps 3 --kernels tile > "$out/sweep.jsonl" 2> "$out/sweep.err"
timeout 600 python bench.py --skip-cpu > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:emit_rows" -c 1 \
  -o "$out/full" python bench.py --steps 1 --warmup 3 --skip-cpu > "$out/ncu_full.log" 2>&1; echo "ncu rc=$?" >> "$out/status.txt"
python tools/ncu_source.py "$out/full.ncu-rep" emit_rows 40 > "$out/source_emit.txt" 2>> "$out/status.txt"
python tools/ncu_summary.py "$out/full.ncu-rep" > "$out/summary.json" 2>> "$out/status.txt"
cat "$out/status.txt"
python - "$out" <<'P'
import json,sys
out=sys.argv[1]
for l in open(out+"/sweep.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print({k:d.get(k) for k in ("config","kernel","index_ms","refine_ms","finalize_ms","step_ms")})
d=json.loads(open(out+"/bench.json").read().strip().splitlines()[-1])
print("bench", round(d["ms_per_step"],4), d.get("phases_ms"), "e2e", d["e2e"].get("seconds"))
P
