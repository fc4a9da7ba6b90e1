#!/usr/bin/env bash
# refine_tc staging (lane per row): tests + c4d8 / c3 / d16 refine-only timings + source ncu
set -u
out=gpurun_out/${1:-r2z}; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "ladder or dim or parity or lattice or sweep or high" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -2 $out/pytest.log >> $out/status.txt
(timeout 300 python tools/refine_only.py c4d8 tile 3; timeout 300 python tools/refine_only.py c3 tile 2;
 timeout 300 python tools/refine_only.py 400000:16:0.657508 tile 2) > $out/refine_only.txt 2>&1
cat $out/refine_only.txt >> $out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:refine_tc" -c 1 \
  -o $out/tc_c4d8 python tools/refine_only.py c4d8 tile 1 > $out/ncu.log 2>&1; echo "ncu rc=$?" >> $out/status.txt
python tools/ncu_source.py $out/tc_c4d8.ncu-rep refine_tc 40 > $out/source.txt 2>> $out/status.txt
python tools/ncu_summary.py $out/tc_c4d8.ncu-rep > $out/summary.json 2>> $out/status.txt
rm -f $out/tc_c4d8.ncu-rep
cat $out/status.txt
