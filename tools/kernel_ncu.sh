#!/usr/bin/env bash
# ncu --set full of each refine kernel (DMMA tile + the three CUDA-core variants)
# at c2, c4d8 and a reduced c4d16 (400k points, same eps): FP64 tensor-pipe vs
# FP64 FMA-pipe utilisation for the dispatcher table.  The reports are reduced to
# JSON on the box (tools/ncu_summary.py) and deleted: gpurun returns <= 64 MiB.
# usage: bash tools/kernel_ncu.sh <outdir>
set -u
out=${1:-gpurun_out/kncu}; mkdir -p $out
for spec in c2 c4d8 400000:16:0.657508; do
  tag=$(echo $spec | tr ':' '_')
  for k in tile scalar core_fma core_expanded; do
    timeout 600 python tools/refine_only.py $spec $k 2 > $out/rate_${tag}_${k}.txt 2>&1
    rep=/tmp/kncu_${tag}_${k}
    timeout 900 ncu --set full --clock-control none -k "regex:refine_" --launch-skip 1 -c 1 \
      -o $rep python tools/refine_only.py $spec $k 2 > $out/ncu_${tag}_${k}.log 2>&1
    echo "$spec $k rc=$?" >> $out/status.txt
    python tools/ncu_summary.py $rep.ncu-rep > $out/ncu_${tag}_${k}.json 2>> $out/status.txt
    rm -f $rep.ncu-rep
  done
done
cat $out/rate_*.txt
