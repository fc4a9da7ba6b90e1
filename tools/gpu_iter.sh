#!/usr/bin/env bash
# Iteration loop: selected GPU tests, a bench line, source-level ncu of one kernel.
# usage: bash tools/gpu_iter.sh <tag> <kernel-regex> <pytest -k expr> [bench args]
set -u
tag=$1; kre=$2; kexpr=$3; shift 3; bargs="$*"
out=gpurun_out/$tag; mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" > "$out/build.log" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "$kexpr" > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$out/status.txt"
tail -3 "$out/pytest_gpu.log" >> "$out/status.txt"
timeout 600 python bench.py --skip-cpu $bargs > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?" >> "$out/status.txt"
python - "$out/bench.json" >> "$out/status.txt" <<'P'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms_per_step",round(d["ms_per_step"],4),"phases",{k:round(v,4) for k,v in d.get("phases_ms",{}).items()})
r=d["roofline"];print("roofline",r.get("kernel"),round(r.get("ms",0),4),round(r["frac"],4))
print("e2e",d["e2e"].get("seconds"))
P
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c ${NCU_COUNT:-1} \
  -o "$out/full" python bench.py --steps 1 --warmup 3 --skip-cpu $bargs > "$out/ncu_full.log" 2>&1; echo "ncu rc=$?" >> "$out/status.txt"
for k in $(echo "$kre" | tr '|' ' '); do python tools/ncu_source.py "$out/full.ncu-rep" "$k" 60 > "$out/source_$k.txt" 2>> "$out/status.txt"; done
python tools/ncu_summary.py "$out/full.ncu-rep" > "$out/summary.json" 2>> "$out/status.txt"
cat "$out/status.txt"
