#!/usr/bin/env bash
# source-level ncu of the c2 emit kernel (per-line instructions / stalls)
set -u
out=gpurun_out/${1:-r2p}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:emit_rows" -c 1 \
  -o $out/emit_c2 python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_emit.log 2>&1; echo "ncu emit rc=$?" >> $out/status.txt
python tools/ncu_source.py $out/emit_c2.ncu-rep emit_rows 80 > $out/emit_source.txt 2>> $out/status.txt
python tools/ncu_summary.py $out/emit_c2.ncu-rep > $out/emit_summary.json 2>> $out/status.txt
ncu -i $out/emit_c2.ncu-rep --page details --csv > $out/emit_details.csv 2>> $out/status.txt
du -sh $out >> $out/status.txt
cat $out/status.txt
