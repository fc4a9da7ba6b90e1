set -u
out=gpurun_out/r2b; mkdir -p $out
timeout 1500 python tools/make_bf_digests.py > $out/bf.log 2>&1; echo "bf rc=$?" >> $out/status.txt
cp tests/golden/bf_digests.json $out/ 2>/dev/null
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_io_cli.py -m gpu -q -x > $out/pytest_parity.log 2>&1; echo "parity rc=$?" >> $out/status.txt
bash tools/run_reference_tests.sh run $out; echo "reftests done" >> $out/status.txt
cat $out/status.txt
