#!/usr/bin/env bash
# Run the reference package's OWN test files (test_join.py, test_cli.py,
# test_datasets.py, unchanged) against the GPU drop-in through the `tilejoin`
# import shim in tests/shim.
#   stage (in the build container, where /root/reference exists):
#       bash tools/run_reference_tests.sh stage
#     copies the test files into .reftests/ (git-ignored scratch, never committed;
#     it travels to the GPU box with the gpurun snapshot).
#   run (on the GPU box):   bash tools/run_reference_tests.sh run [outdir]
#   clean:                  bash tools/run_reference_tests.sh clean
set -u
cmd=${1:-run}
case "$cmd" in
  stage)
    mkdir -p .reftests
    cp /root/reference/pkg/tests/{conftest.py,test_join.py,test_cli.py,test_datasets.py} .reftests/
    ;;
  run)
    out=${2:-gpurun_out/reftests}
    mkdir -p "$out"
    PYTHONPATH="$PWD/tests/shim:$PWD" timeout 1200 python -m pytest -p no:cacheprovider -q \
      --rootdir=.reftests .reftests/test_join.py .reftests/test_cli.py .reftests/test_datasets.py \
      > "$out/reference_tests.txt" 2>&1
    echo "reference tests rc=$?" | tee -a "$out/reference_tests.txt"
    tail -5 "$out/reference_tests.txt"
    ;;
  clean)
    rm -rf .reftests
    ;;
esac
