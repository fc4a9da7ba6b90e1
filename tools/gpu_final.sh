#!/usr/bin/env bash
# round-2 final evidence: GPU suite, smoke, bench lines (both arms, N=1 and the
# 2-rank strong path), strong projection, all-config sweep, launch list + ncu of c2
set -u
out=gpurun_out/${1:-r2final}; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?" >> $out/status.txt
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -3 $out/pytest_gpu.log >> $out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/status.txt
timeout 600 python bench.py > $out/bench_c2.json 2> $out/bench_c2.err; echo "bench rc=$?" >> $out/status.txt
timeout 600 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; echo "bench ref rc=$?" >> $out/status.txt
TJ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 > $out/bench_n2_strong_c2.json 2> $out/bench_n2_strong_c2.err; echo "bench n2 rc=$?" >> $out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $out/bench_n2_ref.json 2> $out/bench_n2_ref.err; echo "bench n2 ref rc=$?" >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
timeout 2400 python tools/sweep.py c1 c2 c4d2 c4d8 c3 c5 expo3d2m --reps 2 --kernels tile,scalar > $out/sweep_all.jsonl 2> $out/sweep_all.err; echo "sweep rc=$?" >> $out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $out/launches_c2.csv python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $out/status.txt
python tools/launch_summary.py $out/launches_c2.csv > $out/launches_c2_summary.txt 2>> $out/status.txt
timeout 900 ncu -f --set full --clock-control none --import-source on -k "regex:refine_lowd|emit_rows|count_rows" -c 3 \
  -o /tmp/full_c2 python bench.py --steps 1 --warmup 3 --skip-cpu > $out/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $out/status.txt
python tools/ncu_summary.py /tmp/full_c2.ncu-rep > $out/ncu_full_c2.json 2>> $out/status.txt
timeout 600 python tools/shard_index_probe.py 8 7 10 > $out/shard_index.txt 2>&1
for c in c2 c5 c3 expo3d2m; do timeout 300 python tools/index_probe.py $c 10 >> $out/index.txt 2>&1; done
du -sh $out >> $out/status.txt
cat $out/status.txt
