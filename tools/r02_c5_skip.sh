#!/usr/bin/env bash
# C5 phase split in graph mode by ablation (PFX_BD_SKIP bits: 1 back substitution, 2 rhs chain,
# 4 far trailing update, 8 diagonal LU + inverses, 16 panel products); results are wrong, times only.
cd "$(dirname "$0")/.."
for sk in ${SKIPS:-0 1 3 7}; do
  PFX_BD_SKIP=$sk timeout 600 python bench.py --workload C5 --steps 4 --warmup 2 --no-cpu-baseline --e2e-steps 0 --prof-steps 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('skip=$sk ms_per_step', round(d['ms_per_step'],2))"
done
