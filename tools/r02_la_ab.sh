#!/usr/bin/env bash
# A/B of the LU look-ahead (PFX_LU_LOOKAHEAD): C4 at 12 systems (the headline) and one
# rank's share at 8 ranks (column split), two alternations; then the large-dense parity tests.
cd "$(dirname "$0")/.."
O=gpurun_out
for rep in 1 2; do
  for la in 1 0; do
    PFX_LU_LOOKAHEAD=$la timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > $O/la${la}_r${rep}.json 2> $O/la${la}_r${rep}.err
    python - <<PY
import json
d=json.loads(open("$O/la${la}_r${rep}.json").read().strip().splitlines()[-1])
print("C4 lookahead=$la rep=$rep ms_per_step", round(d["ms_per_step"],2))
PY
    PFX_LU_LOOKAHEAD=$la timeout 300 python tools/c4_cols_prof.py 8 0 2>&1 | head -1
  done
done
timeout 900 python -m pytest tests/test_dense_large_gpu.py tests/test_colsplit_gpu.py tests/test_configs_gpu.py -x -q -k "not C5 and not c5" 2>&1 | tail -3
