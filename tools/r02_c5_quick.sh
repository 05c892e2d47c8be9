#!/usr/bin/env bash
# C5 quick check: banded parity tests, then the C5 bench line (no CPU baseline) and the chain timeline.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02c5q}
timeout 1200 python -m pytest tests/test_banded_gpu.py tests/test_configs_gpu.py -x -q -k "banded or c5 or C5" 2>&1 | tail -4
timeout 600 python bench.py --workload C5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/${T}_bench_C5.json 2> $O/${T}_bench_C5.err; echo bench_rc=$?
python - <<PY
import json
d=json.loads(open("$O/${T}_bench_C5.json").read().strip().splitlines()[-1])
print("C5 ms_per_step", round(d["ms_per_step"],2), "e2e", round(d["e2e"]["value"],3))
for k,v in sorted(d["kernels"].items(), key=lambda kv:-kv[1]["total_ms"])[:8]: print("  ",k,v["launches"],round(v["total_ms"],1))
PY
