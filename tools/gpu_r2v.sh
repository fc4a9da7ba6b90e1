#!/usr/bin/env bash
# source-level ncu of the high-d small-cell DMMA kernel (refine_tc) at c4d8
set -u
out=gpurun_out/r2v; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:refine_tc" -c 1 \
  -o $out/tc_c4d8 python tools/refine_only.py c4d8 tile 1 > $out/ncu.log 2>&1; echo "ncu rc=$?" >> $out/status.txt
python tools/ncu_source.py $out/tc_c4d8.ncu-rep refine_tc 60 > $out/source.txt 2>> $out/status.txt
python tools/ncu_summary.py $out/tc_c4d8.ncu-rep > $out/summary.json 2>> $out/status.txt
ncu -i $out/tc_c4d8.ncu-rep --page raw --csv > $out/raw.csv 2>> $out/status.txt
cat $out/status.txt
