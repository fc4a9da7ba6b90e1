set -u
out=gpurun_out/route1; mkdir -p $out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/shard_index_probe.py 8 7 3 > $out/ncu.log 2>&1
python tools/launch_summary.py $out/launches.csv > $out/summary.txt 2>&1
cat $out/summary.txt | head -40
