#!/usr/bin/env bash
# strong multi-GPU path after the one-byte count exchange: 2-rank GPU tests, projection
set -u
out=gpurun_out/r2w; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 900 python -m pytest tests/test_distributed.py -m gpu -x -q > $out/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
tail -2 $out/pytest_dist.log >> $out/status.txt
timeout 900 python tools/strong_projection.py c5 1 2 4 8 > $out/strong_projection.jsonl 2> $out/strong_projection.err; echo "projection rc=$?" >> $out/status.txt
cat $out/status.txt
python - <<'P'
import json
for l in open("gpurun_out/r2w/strong_projection.jsonl"):
    d = json.loads(l)
    if "G" in d:
        w = d["slowest_rank"]
        print(d["G"], round(d["T_G_ms"], 2), "eff", round(d["efficiency"], 3), "dev", round(d["efficiency_device_only"], 3),
              "coll", round(d["collectives_ms_est"], 3), {k: round(w[k], 2) for k in ("route_ms", "index_ms", "refine_ms", "output_ms")})
P
