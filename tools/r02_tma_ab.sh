#!/usr/bin/env bash
# zgemm tile staging A/B: TMA (default) against cp.async (PFX_ZGEMM_CPASYNC=1) on C4 and C5,
# alternating, plus the bitwise-equality test and the large-dense / band parity tests.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02tma}
timeout 900 python -m pytest tests/test_dense_large_gpu.py tests/test_banded_gpu.py -q -x > $O/${T}_pytest.log 2>&1; echo pytest_rc=$?; tail -2 $O/${T}_pytest.log
for i in 1 2; do
  for mode in tma cpasync; do
    if [ $mode = cpasync ]; then export PFX_ZGEMM_CPASYNC=1; else unset PFX_ZGEMM_CPASYNC; fi
    for w in ${WL:-C4 C5}; do
      timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/${T}_${w}_${mode}_$i.json 2> $O/${T}_${w}_${mode}_$i.err
      echo "$w $mode $i rc=$? $(python -c "import json;d=json.load(open('$O/${T}_${w}_${mode}_$i.json'));print(round(d['ms_per_step'],2))" 2>/dev/null)"
    done
  done
done
unset PFX_ZGEMM_CPASYNC
