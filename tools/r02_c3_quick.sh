#!/usr/bin/env bash
# C3 quick check: dense parity tests (small sizes, C3 full batch, fuzz), then the C3 bench line twice.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02c3q}
timeout 1500 python -m pytest tests/test_dense_gpu.py tests/test_configs_gpu.py tests/test_fuzz_gpu.py tests/test_pivoting_gpu.py -x -q -k "not C4 and not c4 and not C5 and not c5 and not banded and not tridiag" 2>&1 | tail -3
for rep in 1 2; do
timeout 600 python bench.py --workload C3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 ms_per_step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']))"
done
